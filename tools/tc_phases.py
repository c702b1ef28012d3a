"""Phase breakdown (cycles per row per team) of the tensor-core wide path:
a users half-step with `n` ratings per row, MCF_TC_PROF=1.  GPU box only.
    NS=8,64 python tools/tc_phases.py 100 50"""
import ctypes
import os
import sys

os.environ["MCF_TC_PROF"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import _lib  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

NAMES = ["task", "gram", "hot", "chol:diag(to barA)", "chol:trsm", "chol:lastblk", "backsub", "chol:mma", "output", "chol:split+fence"]
U, I = int(os.environ.get("U", 300_000)), 4096
L = _lib.lib()
L.mcf_tc_prof_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
for D in [int(x) for x in sys.argv[1:]] or [100]:
    for n in [int(x) for x in os.environ.get("NS", "8,64,256").split(",")]:
        g = torch.Generator(device="cuda").manual_seed(0)
        users = torch.arange(U, device="cuda", dtype=torch.int32).repeat_interleave(n)
        items = torch.randint(0, I, (U * n,), device="cuda", dtype=torch.int32, generator=g)
        scores = torch.rand(U * n, device="cuda", generator=g) * 100
        eng = AlsEngine(DeviceRatings(users, items, scores, U, I), D)
        eng.set_factors(torch.randn(U, D) * 0.1, torch.randn(I, D) * 0.1)
        eng.half_step("users", 0.0, 0.05)
        buf = (ctypes.c_ulonglong * 16)()
        L.mcf_tc_prof_read(buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.half_step("users", 0.0, 0.05)
        e1.record()
        torch.cuda.synchronize()
        L.mcf_tc_prof_read(buf)
        tot = sum(buf[k] for k in range(10))
        print(f"D={D} n={n}: {e0.elapsed_time(e1):.2f} ms, {U} rows; cycles per row per team: "
              f"total {tot / U:.0f}: " +
              ", ".join(f"{NAMES[k]} {buf[k] / U:.0f}" for k in range(10)) +
              f" | gram: issue {buf[10] / U:.0f}, wait-landed {buf[11] / U:.0f}, mma {buf[12] / U:.0f}")
