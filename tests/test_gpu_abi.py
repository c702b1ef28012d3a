"""The C-ABI exercised without the Python wrapper: (1) the ctypes stub
INTEGRATION.md documents for the reference side, executed verbatim; (2) a C
program that dlopens libmcf.so and runs mcf_csr_build -> mcf_als_plan ->
mcf_als_half_step.  Both are compared with the oracle on config 0 (the
reference's als_half_step, factor.py:512-538, restated in oracle/)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle
from conftest import REPO

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4


def _rel(got, ref):
    return np.abs(got - ref).max() / np.abs(ref).max()


def test_integration_md_stub_runs_cfg0(golden):
    from integration_snippets import load_binding
    from paper_1108_2580_b200 import SingularSystemError, _lib
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I, D, lam = int(g["U"]), int(g["I"]), int(g["D"]), float(g["lam"])
    ns = load_binding({"SingularSystemError": SingularSystemError})
    dev = torch.device("cuda")
    # the caller's own items layout: stable CSC (oracle.side_csr == factor._side_csr)
    ptr, idx, val, _, _ = oracle.side_csr(i, u, s, I)
    ld = _lib.factor_ld(D)
    P = torch.zeros(U, ld, dtype=torch.float32, device=dev)
    P[:, :D] = torch.as_tensor(g["P0"], device=dev)
    Q = torch.zeros(I, ld, dtype=torch.float32, device=dev)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)  # noqa: E731
    ns["als_half_step"](t(ptr, torch.int64), t(idx, torch.int32), t(val, torch.float32), P, Q, D,
                        lam, weighted=True)
    torch.cuda.synchronize()
    ref, failed = oracle.als_half_step(g["P0"].astype(np.float64), g["Q0"].astype(np.float64),
                                       u, i, s, "items", lam_n=lam)
    assert failed == -1
    assert _rel(Q[:, :D].double().cpu().numpy(), ref) < REL_TOL
    assert torch.all(Q[:, D:] == 0)
    # the documented error convention: a singular row -> SingularSystemError
    Pz = torch.zeros_like(P)
    with pytest.raises(SingularSystemError, match="row 0"):
        ns["als_half_step"](t(ptr, torch.int64), t(idx, torch.int32), t(val, torch.float32), Pz,
                            Q, D, 0.0)


def test_c_driver_cfg0(golden, tmp_path):
    from paper_1108_2580_b200 import _lib
    exe = tmp_path / "mcf_driver"
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", "-std=gnu11", "-I", os.path.join(REPO, "include"),
                    "-I", os.path.join(cuda, "include"),
                    os.path.join(REPO, "tests", "c_driver", "mcf_driver.c"), "-o", str(exe),
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", "-ldl"], check=True)
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I, D, lam = int(g["U"]), int(g["I"]), int(g["D"]), float(g["lam"])
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as fh:
        fh.write(np.array([u.size, U, I, D], np.int64).tobytes())
        fh.write(np.array([lam], np.float32).tobytes())
        for a, dt in ((u, np.int32), (i, np.int32), (s, np.float32), (g["P0"], np.float32),
                      (g["Q0"], np.float32)):
            fh.write(np.ascontiguousarray(a, dtype=dt).tobytes())
    out = tmp_path / "out.bin"
    res = subprocess.run([str(exe), _lib.LIB_PATH, str(inp), str(out)], capture_output=True,
                         text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    raw = out.read_bytes()
    fail = int(np.frombuffer(raw[:8], np.int64)[0])
    Q = np.frombuffer(raw[8:], np.float32).reshape(I, D)
    assert fail == -1
    ref, _ = oracle.als_half_step(g["P0"].astype(np.float64), g["Q0"].astype(np.float64), u, i,
                                  s, "items", lam_n=lam)
    assert _rel(Q.astype(np.float64), ref) < REL_TOL
