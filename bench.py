"""Benchmark of the ALS sweep on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

A step is ONE FULL SWEEP (items half-step, then users half-step; every
training rating is touched twice) over BASELINE config 1 by default:
1,000,990 users x 624,961 items, 258,806,215 training ratings, D = 20,
weighted lambda 0.065, fp32, synthetic data from this repo's seeded
generator (paper_1108_2580_b200/synth.py; the KDD-Cup data is not
available).  metric = training ratings per second per full sweep.

* value: W untimed + K timed sweeps on device-resident layouts and factors,
  CUDA events on the launching stream, barrier + synchronize on both sides,
  max over ranks.  The CSR/CSC are 2.07 GB each, far larger than the 126 MB
  L2, so no explicit flush between sweeps.
* roofline: the dominant kernel is the fused Gram + Cholesky half-step
  (k_als_pair<5,4> at D = 20, 2 launches per sweep); achieved = algorithmic
  bytes per launch (n_nnz (4D + 8) + 4D n_rows_solved) / mean
  launch time from CUDA events around each half-step.
* parity: one extra re-anchored sweep after the timed region -- the device
  half-steps vs the float64 oracle solving the same rows from the device's
  own input factors, on the 64 highest-degree rows of each side plus random
  rows (SURVEY §8(c) protocol; tolerance 1e-4 relative, north_star).
* e2e: the same metric through the public drop-in API
  ``factor.train("wals", ...)`` (``devices=N`` at N > 1) on HOST (pinned)
  arrays: H2D of the COO split, layout builds, `sweeps` sweeps with the
  per-sweep objective and held-out RMSE, D2H of the factors -- ratings *
  sweeps / wall time.
* cpu_baseline (rank 0, N = 1): the REFERENCE itself (multicf installed in
  baseline/_ref, numba, all host cores): its factor.als_half_step sweep with
  the wALS weights hook on a bounded sample workload -- the same generator at
  --ref-scale of the config (default 2 %) -- timed as-is (its per-call CSR
  rebuild included, factor.py:522) and solve-only (prebuilt _side_csr +
  run_blocks(als_solve_rows), the bench convention of parallel.py:187-231).
  Falls back to the oracle port (kind "port") when baseline/_ref is absent.
* --impl reference: that reference sweep as its own arm (rank 0 only; no GPU
  work, libmcf never loaded): every step is one as-is sweep of the sample.
* --gpus N without a torchrun environment re-launches itself under
  torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1108_2580_b200 import synth  # noqa: E402

PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(REPO, "profiles", "roofline_traffic.json")
FP32 = os.path.join(REPO, "profiles", "fp32_peak.json")   # tools/micro/fp32_peak on this pool
METRIC = "ALS ratings/sec per full sweep"


# ---------------------------------------------------------------------------
# clocks

THROTTLE_BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
                 0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler:
    def __init__(self, index: int):
        self.index, self.samples, self.reasons = index, [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                sm, mx, act = (x.strip() for x in out.split(","))
                self.samples.append(float(sm))
                self.max_mhz = float(mx)
                bits = int(act, 16)
                for b, name in THROTTLE_BITS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# helpers

def algorithmic(nnz, U, I, D):
    """bytes and flops per full sweep and per half-step."""
    b_items = nnz * (4 * D + 8) + 4 * D * I
    b_users = nnz * (4 * D + 8) + 4 * D * U
    f_rows = lambda n: n * (D ** 3 / 3 + 2 * D * D)  # noqa: E731
    f_items = nnz * (D * D + 3 * D) + f_rows(I)
    f_users = nnz * (D * D + 3 * D) + f_rows(U)
    return {"bytes_sweep": b_items + b_users, "flops_sweep": f_items + f_users,
            "bytes_launch_mean": (b_items + b_users) / 2, "flops_launch_mean": (f_items + f_users) / 2}


def fp32_peak():
    """Measured FFMA2 peak of this pool's B200 (tools/micro/fp32_peak, kept in
    profiles/fp32_peak.json); nominal 148 SM x 128 FMA x 2 x 1.965 GHz else."""
    try:
        with open(FP32) as fh:
            return float(json.load(fh)["fp32_tflops"]), "measured (tools/micro/fp32_peak)"
    except Exception:
        return 74.4, "nominal"


def kernel_name(D: int) -> str:
    from paper_1108_2580_b200.device import tc_path
    if tc_path(D):
        return ("k_als_tc<NBLK> (tcgen05 kind::f16 Gram, fp16 h/l split, TMEM-resident blocked "
                "Cholesky with negated-MMA trailing updates; + k_tc_prep, k_tc_split; rows with "
                "n <= 32 ratings: k_als_dual<1, N>, dual form on CUDA cores)")
    if D <= 20:
        return "k_als_pair<5,4> (fused Gram + lam*n + Cholesky + solve; + k_als_heavy for hot rows)"
    if D <= 28:
        return "k_als_warp (4x4 register tiles, warp Cholesky)"
    if D <= 104:
        return "k_als_tile_warp (warp per row, 8x8 register tiles, blocked register Cholesky)"
    return "k_als_cta"


def roofline_for(D, bytes_launch, flops_launch, launch_s, traffic=None, kernel=None):
    """roofline time = max(bytes / HBM, flops / compute peak) per
    launch; the bound is whichever is larger and `achieved` is reported in
    that resource's unit (GB/s or TFLOP/s), the other view beside it.  The
    compute peak is the FP32 CUDA-core peak, or -- on the tensor-core path
    (D >= 64) -- the measured dense 16-bit tensor peak / 3: every fp32
    product is three fp16 MMAs (h h + h l + l h)."""
    hbm, hbm_kind = peaks()
    f32, f32_kind = fp32_peak()
    from paper_1108_2580_b200.device import tc_path
    if tc_path(D):
        f32, f32_kind = tensor_peak_3x()
    t_hbm = bytes_launch / (hbm * 1e9)
    t_f32 = flops_launch / (f32 * 1e12)
    gbs = bytes_launch / launch_s / 1e9
    tfs = flops_launch / launch_s / 1e12
    if t_hbm >= t_f32:
        r = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
             "peak_kind": hbm_kind, "achieved_tflops": tfs, "fp32_peak_tflops": f32}
    else:
        r = {"bound": "tensor" if tc_path(D) else "fp32", "achieved": tfs, "peak": f32,
             "unit": "TFLOP/s", "frac": tfs / f32,
             "peak_kind": f32_kind, "achieved_gbs": gbs, "hbm_peak_gbs": hbm}
    r.update({"traffic": traffic, "kernel": kernel or kernel_name(D),
              "roofline_ms_per_launch": 1e3 * max(t_hbm, t_f32),
              "algorithmic_bytes_per_launch": bytes_launch,
              "algorithmic_flops_per_launch": flops_launch})
    return r


def launches_per_sweep(eng) -> int:
    """libmcf kernels per sweep: per half-step the row kernel, plus the hot-row
    reduce kernel when the layout has hot rows (D <= 20 path); on the
    tensor-core path the scale pre-pass, the table split, the tensor-core
    kernel and the short-row dual kernel."""
    from paper_1108_2580_b200.device import tc_path
    n = 0
    for lay in (eng.r.by_item, eng.r.by_user):
        info = lay.plan()[1]
        if tc_path(eng.D):
            n += 7      # k_tc_prep, k_tc_split, k_als_tc, k_als_dual<1, N> for N = 32, 24, 16, 8
        else:
            n += 1 + (1 if (eng.D <= 20 and info[4] > 0) else 0)
    return n


def tensor_peak_3x():
    """Dense 16-bit tensor peak (MEASURED_PEAKS.json bf16, the same pipe rate as
    fp16) / 3 -- the effective fp32-product rate of the 3-term fp16 split."""
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["bf16_tflops"]) / 3.0, "measured bf16 / 3 (3 fp16 MMAs per product)"
    except Exception:
        return 2250.0 / 3.0, "nominal dense 16-bit / 3"


def peaks():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_setup(n_gpus, use_cuda=True):
    """One process per GPU; the device is bound before the NCCL group is
    created.  use_cuda=False (the reference arm, --dry-run on CPU): gloo, no
    CUDA context at all."""
    use_cuda = use_cuda and torch.cuda.is_available()
    local = int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", 0)))
    if use_cuda:
        torch.cuda.set_device(local)
    if n_gpus > 1 or "RANK" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if use_cuda else "gloo")
        rank, world = dist.get_rank(), dist.get_world_size()
    else:
        rank, world = 0, 1
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# the reference itself (baseline/_ref) on a bounded sample workload

REF_DIR = os.path.join(REPO, "baseline", "_ref")


def reference_package():
    """The unmodified reference (multicf) from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "multicf")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mcf_ref_numba_cache")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import multicf
    import multicf._kernels as K
    import multicf.data as Dm
    import multicf.factor as F
    import multicf.parallel as PAR
    import numba
    return {"F": F, "Dm": Dm, "K": K, "PAR": PAR, "version": getattr(multicf, "__version__", "?"),
            "numba": numba.__version__}


class ReferenceSweep:
    """The reference's own ALS sweep -- factor.als_half_step on items, then
    users (factor.py:550-555), weighted lambda through its wALS hook
    (weights = 1/n_row, equal to lam * n_r to <= 1e-13) -- on the
    config's generator at `scale` (CPU-generated, same shape parameters:
    Zipf item popularity over a random permutation, log-normal user counts,
    N(0, 0.1) fp32 initial factors)."""

    def __init__(self, ref, cfg, scale: float, threads: int):
        self.ref, self.threads = ref, int(threads)
        F, Dm = ref["F"], ref["Dm"]
        self.cfg = synth.scaled_config(cfg, scale)
        wl = synth.generate(self.cfg, seed=0, device="cpu")
        u = wl.train_users.numpy().astype(np.int64)
        i = wl.train_items.numpy().astype(np.int64)
        s = wl.train_scores.numpy().astype(np.float64)
        U, I = self.cfg.users, self.cfg.items
        self.ds = Dm.Dataset.from_arrays(u, i, s, np.zeros(u.size, np.int64), num_users=U,
                                         num_items=I)
        self.model = F.init_model("als", self.ds, F.HyperParams(D=cfg.D, lam=cfg.lam), 0)
        P0, Q0 = synth.init_factors(U, I, cfg.D, seed=1)
        self.model.p, self.model.q = P0.astype(np.float64), Q0.astype(np.float64)
        self.lam = cfg.lam
        self.w = {"items": 1.0 / np.bincount(i, minlength=I)[i],
                  "users": 1.0 / np.bincount(u, minlength=U)[u]}
        self.nnz = int(u.size)
        self._csr = {}
        ref["K"].warmup()

    def describe(self) -> str:
        c = self.cfg
        return (f"{c.name}: the config's generator at reduced scale, {c.users} users x {c.items} "
                f"items, {self.nnz} train ratings, D = {c.D}; full reference sweeps "
                f"(multicf.factor.als_half_step, wALS weights 1/n_row, threads = {self.threads})")

    def sweep_as_is(self) -> float:
        F = self.ref["F"]
        t0 = time.perf_counter()
        for side in ("items", "users"):
            F.als_half_step(self.model, self.ds, side, self.lam, self.w[side], self.threads)
        return time.perf_counter() - t0

    def sweep_solve_only(self) -> float:
        """Prebuilt _side_csr + run_blocks(als_solve_rows) (factor.py:522-534
        without the per-call CSR rebuild)."""
        F, K, PAR = self.ref["F"], self.ref["K"], self.ref["PAR"]
        for side in ("items", "users"):
            if side not in self._csr:
                self._csr[side] = F._side_csr(self.ds, side, self.w[side])
        t0 = time.perf_counter()
        for side in ("items", "users"):
            ptr_, idx, val, wts = self._csr[side]
            fixed = self.model.q if side == "users" else self.model.p
            out = self.model.p if side == "users" else self.model.q

            def work(lo, hi, ptr_=ptr_, idx=idx, val=val, wts=wts, fixed=fixed, out=out):
                fail = np.full(1, -1, dtype=np.int64)
                K.als_solve_rows(lo, hi, ptr_, idx, val, wts, fixed, out, self.lam, fail)
                assert fail[0] < 0

            PAR.run_blocks(work, PAR.even_bounds(out.shape[0], self.threads), self.threads)
        return time.perf_counter() - t0


def reference_baseline(cfg, scale: float, steps: int = 2, warmup: int = 1):
    """cpu_baseline of our arm: a few reference sweeps of the sample."""
    ref = reference_package()
    if ref is None:
        return None
    threads = os.cpu_count() or 1
    rs = ReferenceSweep(ref, cfg, scale, threads)
    for _ in range(warmup):
        rs.sweep_as_is()
    asis = [rs.sweep_as_is() for _ in range(steps)]
    solve = [rs.sweep_solve_only() for _ in range(steps)]
    v = rs.nnz / statistics.median(asis)
    return {"value": v, "unit": "ratings/s", "cores": threads, "kind": "reference",
            "sample": rs.describe(), "variant": "as-is (factor.als_half_step, CSR rebuilt "
            "per half-step, factor.py:522)",
            "solve_only": {"value": rs.nnz / statistics.median(solve), "unit": "ratings/s",
                           "what": "prebuilt _side_csr + run_blocks(als_solve_rows)"},
            "reference": f"multicf {ref['version']} (baseline/_ref), numba {ref['numba']}"}


def port_baseline(engine, lam, threads=None):
    """Fallback cpu_baseline without baseline/_ref: the oracle port (C,
    float64, the reference's als_solve_rows with static row blocks) on 4000
    random user rows and 2000 random item rows."""
    import oracle
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(7)
    P, Q = (t.double().cpu().numpy() for t in engine.factors())
    rates, desc = {}, []
    for side, nrow in (("users", 4000), ("items", 2000)):
        lay = engine.r.layout(side)
        rows = np.sort(rng.choice(lay.n_rows, size=min(nrow, lay.n_rows), replace=False))
        sp, idx, val, n = gather_rows(lay, rows)
        t0 = time.perf_counter()
        oracle.solve_rows((sp, idx, val, None), Q if side == "users" else P, sp.size - 1,
                          lam_n=lam, threads=threads)
        rates[side] = n / (time.perf_counter() - t0)
        desc.append(f"{side}: {sp.size - 1} random rows, {n} ratings")
    v = 1.0 / (1.0 / rates["users"] + 1.0 / rates["items"])
    return {"value": v, "unit": "ratings/s", "cores": threads, "kind": "port",
            "sample": "; ".join(desc)}


# ---------------------------------------------------------------------------
# parity at the benchmarked size (re-anchored half-steps vs the oracle)

def gather_rows(lay, rows: np.ndarray):
    """Sub-CSR of `rows` (sorted int64) of a device layout, on the host:
    (ptr, idx int64, val float64, ratings)."""
    ptr_h = lay.ptr.cpu().numpy()
    starts, ends = ptr_h[rows], ptr_h[rows + 1]
    counts = ends - starts
    sub_ptr = np.zeros(rows.size + 1, np.int64)
    np.cumsum(counts, out=sub_ptr[1:])
    n = int(sub_ptr[-1])
    dev = lay.idx.device
    st = torch.as_tensor(starts, device=dev)
    cnt = torch.as_tensor(counts, device=dev)
    flat = (torch.repeat_interleave(st, cnt) + torch.arange(n, device=dev)
            - torch.repeat_interleave(torch.as_tensor(sub_ptr[:-1], device=dev), cnt))
    idx = lay.idx[flat].cpu().numpy().astype(np.int64)
    val = lay.val[flat].cpu().numpy().astype(np.float64)
    return sub_ptr, idx, val, n


def parity_rows(lay, n_random: int, n_hot: int, rng) -> np.ndarray:
    deg = lay.degrees()
    hot = torch.topk(deg, min(n_hot, lay.n_rows)).indices.cpu().numpy()
    rand = rng.choice(lay.n_rows, size=min(n_random, lay.n_rows), replace=False)
    return np.unique(np.concatenate([hot, rand])).astype(np.int64)


def rel_errors(got: np.ndarray, ref: np.ndarray):
    """row-wise |d_r| / max(|ref_r|, 1e-6 max|ref|) and
    max|d| / max|ref|."""
    rn = np.linalg.norm(ref, axis=1)
    dn = np.linalg.norm(got - ref, axis=1)
    row = float((dn / np.maximum(rn, 1e-6 * rn.max() + 1e-30)).max())
    mx = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
    return row, mx


def side_parity(lay, rows, fixed_f64, got, lam_n, y_shift=0.0, S=None, T=None, tau=0.0):
    import oracle
    threads = os.cpu_count() or 1
    sp, idx, val, n = gather_rows(lay, rows)
    ref, failed = oracle.solve_rows((sp, idx, val - y_shift, None), fixed_f64, rows.size,
                                    0.0, lam_n, tax_S=S, tax_T=T, tau=tau, threads=threads,
                                    dynamic=True)
    row, mx = rel_errors(got, ref)
    return {"rows": int(rows.size), "ratings": n, "max_row_rel": row, "max_rel": mx,
            "oracle_failed_row": int(failed)}


def summarize_parity(parts: dict, n_hot: int, hottest: dict, t0: float) -> dict:
    row = max(p["max_row_rel"] for p in parts.values())
    mx = max(p["max_rel"] for p in parts.values())
    return {"max_row_rel": row, "max_rel": mx, "tolerance": 1e-4,
            "pass": bool(row <= 1e-4 and mx <= 1e-4), "hottest_n": n_hot,
            "hottest_degree": hottest, "per_side": parts,
            "protocol": "re-anchored: device half-step vs float64 oracle (oracle/als_oracle.c) "
                        "on the same rows from the device's own input factors",
            "seconds": time.perf_counter() - t0}


def reanchored_parity(eng, lam, n_hot=64, n_random=(2000, 4000), seed=11):
    """One extra sweep, items then users, each half-step compared with the
    oracle on the hottest + random rows."""
    t0 = time.perf_counter()
    rng = np.random.default_rng(seed)
    D = eng.D
    parts, hottest = {}, {}
    for side, nr in zip(("items", "users"), n_random):
        lay = eng.r.layout(side)
        fixed = (eng.P if side == "items" else eng.Q)[:, :D].double().cpu().numpy()
        eng.half_step(side, 0.0, lam)
        eng.check()
        rows = parity_rows(lay, nr, n_hot, rng)
        out = eng.Q if side == "items" else eng.P
        got = out[torch.as_tensor(rows, device=out.device), :D].double().cpu().numpy()
        parts[side] = side_parity(lay, rows, fixed, got, lam)
        hottest[side] = int(lay.degrees().max())
    return summarize_parity(parts, n_hot, hottest, t0)


def mfitr_parity(solver, graph, w, cfg, n_hot=64, n_random=(2000, 4000), seed=11):
    """ALS-MFITR (factor blocks): the tracks layer (taxonomy S/T from the
    device's own Q) and the users half-step, each vs the oracle."""
    import oracle
    t0 = time.perf_counter()
    rng = np.random.default_rng(seed)
    eng, h = solver.eng, solver.hyper
    D, I = eng.D, eng.r.num_items
    lay = eng.r.by_item
    Q_in = eng.Q[:, :D].double().cpu().numpy()
    P_in = eng.P[:, :D].double().cpu().numpy()
    solver.solve_layer(0)                         # tracks
    eng.check()
    tracks = solver.layers[0].cpu().numpy().astype(np.int64)
    deg = lay.degrees()[solver.layers[0].long()]
    hot = tracks[torch.topk(deg, min(n_hot, tracks.size)).indices.cpu().numpy()]
    rows = np.unique(np.concatenate([hot, rng.choice(tracks, size=min(n_random[0], tracks.size),
                                                     replace=False)]))
    S, T = oracle.taxonomy_terms(graph.edge_child, graph.edge_parent, np.asarray(w, np.float64),
                                 Q_in, I)
    got = eng.Q[torch.as_tensor(rows, device=eng.device), :D].double().cpu().numpy()
    parts = {"items_tracks_layer": side_parity(lay, rows, P_in, got, h.lam2, solver.mu, S[rows],
                                               T[rows], solver.tau)}
    fixed = eng.Q[:, :D].double().cpu().numpy()
    solver.users()
    eng.check()
    urows = parity_rows(eng.r.by_user, n_random[1], n_hot, rng)
    got = eng.P[torch.as_tensor(urows, device=eng.device), :D].double().cpu().numpy()
    parts["users"] = side_parity(eng.r.by_user, urows, fixed, got, h.lam2, solver.mu)
    hottest = {"tracks": int(deg.max()), "users": int(eng.r.by_user.degrees().max())}
    return summarize_parity(parts, n_hot, hottest, t0)


# ---------------------------------------------------------------------------

def arm_config(cfg, world, extra=None):
    """The `config` object of both arms (ours and --impl reference)."""
    c = {"workload": cfg.name, "users": cfg.users, "items": cfg.items, "nnz_train": cfg.nnz,
         "D": cfg.D, "lambda_weighted": cfg.lam,
         "step": "one full sweep (items then users half-step)",
         "l2": "inputs > L2 (CSR/CSC 8 B/rating = 2.07 GB each vs 126 MB L2); no flush",
         "parallelism": f"rows sharded over {world} GPU(s)"}
    if cfg.taxonomy is not None:
        c["step"] = "one ALS-MFITR sweep: 4 item layers + users"
        c["lambda3"] = c["lambda4"] = cfg.tax_weight
    c.update(extra or {})
    return c


def run_reference(args, rank, world):
    """--impl reference: the reference's own sweep on the host cores (rank 0
    only; the other ranks exit without work).  No GPU work, libmcf is never
    loaded."""
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    ref = reference_package()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref (the reference "
                          "package multicf) is not installed"}), flush=True)
        return
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    rs = ReferenceSweep(ref, cfg, args.ref_scale, threads)
    t_prep = time.perf_counter() - t0
    for _ in range(args.warmup):
        rs.sweep_as_is()
    times = [rs.sweep_as_is() for _ in range(args.steps)]
    solve = [rs.sweep_solve_only() for _ in range(min(args.steps, 3))]
    ms = 1000.0 * statistics.mean(times)
    value = rs.nnz * args.steps / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "ratings/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, BASELINE config shapes)",
            "config": arm_config(cfg, world),
            "cpu_baseline": {"value": value, "unit": "ratings/s", "cores": threads,
                             "kind": "reference", "sample": rs.describe(),
                             "variant": "as-is (factor.als_half_step, CSR rebuilt per "
                                        "half-step, factor.py:522)"},
            "solve_only": {"value": rs.nnz / statistics.median(solve), "unit": "ratings/s",
                           "what": "prebuilt _side_csr + run_blocks(als_solve_rows), "
                                   f"median of {len(solve)} sweeps"},
            "e2e": {"value": value, "unit": "ratings/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "reference": f"multicf {ref['version']} (baseline/_ref, unmodified), numba "
                         f"{ref['numba']}",
            "step": "one as-is reference sweep (items then users) of the sample workload",
            "sample_prep_s": t_prep, "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def pinned_split(wl):
    """The workload's train / held-out arrays in pinned host memory."""
    def pinned(t):
        return t.cpu().pin_memory().numpy()
    return tuple(pinned(t) for t in (wl.train_users, wl.train_items, wl.train_scores,
                                     wl.valid_users, wl.valid_items, wl.valid_scores))


def time_e2e(call, steps: int, world: int):
    """Median wall time of `call()` over `steps` calls after one warm call
    (allocator pools, plans, NCCL communicators), synchronized, max over ranks."""
    times, res = [], None
    for s in range(steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = call()
        torch.cuda.synchronize()
        if s > 0:
            times.append(time.perf_counter() - t0)
    return max_over_ranks(statistics.median(times), world), res


def als_e2e(args, cfg, wl, P0, Q0, world):
    """e2e through the public drop-in: factor.train('wals', reg='weighted')
    on pinned host arrays (devices=N at N > 1)."""
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    dev = torch.device("cuda", torch.cuda.current_device())
    tu, ti, ts, vu, vi, vs = pinned_split(wl)
    tr = Dataset.from_arrays(tu, ti, ts, num_users=cfg.users, num_items=cfg.items, compact=True)
    va = Dataset.from_arrays(vu, vi, vs, num_users=cfg.users, num_items=cfg.items, compact=True)
    hp = factor.HyperParams(lam=cfg.lam, D=cfg.D, iters=cfg.sweeps)
    P0p, Q0p = torch.from_numpy(P0).pin_memory(), torch.from_numpy(Q0).pin_memory()
    Pn = torch.empty(cfg.users, cfg.D, dtype=torch.float32, pin_memory=True)
    Qn = torch.empty(cfg.items, cfg.D, dtype=torch.float32, pin_memory=True)

    def call():
        tr.__dict__.pop("_device_cache", None)
        model, rep = factor.train("wals", tr, va, hp, reg="weighted", init=(P0p, Q0p),
                                  device=dev, as_torch=True,
                                  devices=world if world > 1 else None)
        Pn.copy_(model.p, non_blocking=True)
        Qn.copy_(model.q, non_blocking=True)
        tr.__dict__.pop("_device_cache", None)
        return rep[-1].valid_rmse

    t, rm = time_e2e(call, max(1, args.e2e_steps), world)
    h2d = sum(a.nbytes for a in (tu, ti, ts, vu, vi, vs)) + P0.nbytes + Q0.nbytes
    d2h = Pn.numel() * 4 + Qn.numel() * 4 + 16 * cfg.sweeps
    return {"value": cfg.nnz * cfg.sweeps / t, "unit": "ratings/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "step": f"one factor.train('wals', reg='weighted'{', devices=%d' % world if world > 1 else ''}) "
                    f"call: {cfg.sweeps} sweeps + layout builds + per-sweep objective and held-out "
                    "RMSE, factors to pinned host memory",
            "seconds_per_step": t, "valid_rmse": rm}


def mfitr_e2e(args, cfg, wl, P0, Q0, world, blocks):
    """e2e through mfitr.train_mfitr on pinned host arrays (edge weights,
    layouts, `sweeps` ALS-MFITR sweeps with loss_mfitr and held-out RMSE)."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.data import Dataset
    dev = torch.device("cuda", torch.cuda.current_device())
    tu, ti, ts, vu, vi, vs = pinned_split(wl)
    tr = Dataset.from_arrays(tu, ti, ts, num_users=cfg.users, num_items=cfg.items, compact=True)
    va = Dataset.from_arrays(vu, vi, vs, num_users=cfg.users, num_items=cfg.items, compact=True)
    h = mfitr.MfitrHyper(D=cfg.D, lam1=cfg.lam if blocks == "full" else 0.0, lam2=cfg.lam,
                         lam3=cfg.tax_weight, lam4=cfg.tax_weight, iters=cfg.sweeps)

    def call():
        tr.__dict__.pop("_device_cache", None)
        model, rep = mfitr.train_mfitr("mfitr", tr, va, wl.graph, h, init=(P0, Q0), device=dev,
                                       as_torch=True, blocks=blocks,
                                       devices=world if world > 1 else None)
        out = [model.base.p.cpu(), model.base.q.cpu()]
        tr.__dict__.pop("_device_cache", None)
        return rep[-1].valid_rmse, sum(o.numel() * 4 for o in out)

    t, (rm, d2h) = time_e2e(call, max(1, args.e2e_steps), world)
    h2d = sum(a.nbytes for a in (tu, ti, ts, vu, vi, vs)) + P0.nbytes + Q0.nbytes
    return {"value": cfg.nnz * cfg.sweeps / t, "unit": "ratings/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h + 16 * cfg.sweeps),
            "step": f"one mfitr.train_mfitr(blocks='{blocks}'"
                    f"{', devices=%d' % world if world > 1 else ''}) call: edge weights, layouts, "
                    f"{cfg.sweeps} sweeps + per-sweep loss_mfitr and held-out RMSE",
            "seconds_per_step": t, "valid_rmse": rm}


def cpu_baseline_for(args, cfg, eng=None, lam=None):
    if args.skip_cpu:
        return None
    b = reference_baseline(cfg, args.ref_scale)
    if b is None and eng is not None:
        b = port_baseline(eng, lam)
    if b is not None and cfg.taxonomy is not None:
        b["note"] = ("the reference trains MFITR by SGD only: this is its ALS sweep on the "
                     "config's ratings generator (SURVEY §8(d))")
    return b


def timed_sweeps(args, world, dev, step_fns):
    """W warm-up sweeps, then K timed sweeps with a CUDA event after every
    call of step_fns; returns (per-call ms lists, total ms, clocks)."""
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        for f in step_fns:
            f()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n = len(step_fns)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n * args.steps + 1)]
    with ClockSampler(gpu_index(dev)) as clk:
        time.sleep(0.3)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev[0].record(stream)
        for s in range(args.steps):
            for k, f in enumerate(step_fns):
                f()
                ev[n * s + k + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    total = ev[0].elapsed_time(ev[-1])
    per = [[ev[n * s + k].elapsed_time(ev[n * s + k + 1]) for s in range(args.steps)]
           for k in range(n)]
    return per, total, clk.summary()


def gpu_index(dev) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    if vis and vis[0].strip().isdigit() and dev.index is not None and dev.index < len(vis):
        return int(vis[dev.index])
    return dev.index or 0


def run_ours(args, rank, world):
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings

    cfg = synth.CONFIGS[args.config]
    if args.scale != 1.0:
        cfg = synth.scaled_config(cfg, args.scale)
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    wl = synth.generate(cfg, seed=0, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    if world > 1 or args.force_sharded:
        if cfg.taxonomy is not None:
            return run_sharded_mfitr(args, rank, world, cfg, wl, t_gen)
        return run_sharded(args, rank, world, cfg, wl, t_gen)
    if cfg.taxonomy is not None:
        return run_mfitr(args, cfg, wl, t_gen)
    nnz = wl.nnz
    t0 = time.perf_counter()
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
    torch.cuda.synchronize()
    t_layout = time.perf_counter() - t0
    eng = AlsEngine(r, cfg.D)
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    eng.set_factors(P0, Q0)
    eng.r.by_user.plan()
    eng.r.by_item.plan()
    lam = cfg.lam

    per, total_ms, clocks = timed_sweeps(args, world, dev, [
        lambda: eng.half_step("items", 0.0, lam), lambda: eng.half_step("users", 0.0, lam)])
    eng.check()
    ms_per_step = max_over_ranks(total_ms / args.steps, world)
    value = nnz / (ms_per_step / 1000.0)
    half_ms = per[0] + per[1]

    alg = algorithmic(nnz, cfg.users, cfg.items, cfg.D)
    mean_launch_s = statistics.mean(half_ms) / 1000.0
    traffic = None
    if os.path.exists(TRAFFIC):
        try:
            traffic = json.load(open(TRAFFIC)).get(cfg.name)
        except Exception:
            traffic = None
    roofline = roofline_for(cfg.D, alg["bytes_launch_mean"], alg["flops_launch_mean"],
                            mean_launch_s, traffic)
    roofline["launch_ms"] = {"items": statistics.mean(per[0]), "users": statistics.mean(per[1])}

    # held-out RMSE after the timed sweeps (sanity, not timed)
    rm = float(eng.rmse(wl.valid_users, wl.valid_items, wl.valid_scores).item())
    n_launch = launches_per_sweep(eng) * args.steps

    parity = None if args.skip_parity else reanchored_parity(eng, lam)
    cpu = cpu_baseline_for(args, cfg, eng, lam) if rank == 0 else None

    e2e = None
    if not args.skip_e2e:
        del r, eng
        torch.cuda.empty_cache()
        e2e = als_e2e(args, cfg, wl, P0, Q0, world)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ratings/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": arm_config(cfg, world),
                "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": n_launch, "clocks": clocks,
                "valid_rmse_after": rm, "layout_build_s": t_layout, "datagen_s": t_gen,
                "sweep_ms_items_users": [roofline["launch_ms"]["items"],
                                         roofline["launch_ms"]["users"]]}
        print(json.dumps(line), flush=True)


def run_mfitr(args, cfg, wl, t_gen):
    """Configs 2 / 4: ALS-MFITR sweeps (layered item half-step with the
    taxonomy term, then users), device edge weights (bit-exact AC)."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
    tr = wl.train_dataset()
    tr.__dict__["_device_cache"] = {(str(dev), cfg.users, cfg.items): r}
    ew = mfitr.edge_weights(wl.graph, tr, device=dev, num_items=cfg.items)
    torch.cuda.synchronize()
    t_layout = time.perf_counter() - t0
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    full = args.mfitr_blocks == "full"
    h = mfitr.MfitrHyper(D=cfg.D, lam1=cfg.lam if full else 0.0, lam2=cfg.lam,
                         lam3=cfg.tax_weight, lam4=cfg.tax_weight, iters=cfg.sweeps)
    if full:   # every block: [q|b_i] layers, [q_a|b_a] artists, [p|b_u] users (D+1 solves)
        art = wl.graph.artist_array(cfg.items)
        solver = mfitr.MfitrFullSolver(r, wl.graph, ew.w, h, r.global_mean, art, P0, Q0)
        eng = solver
    else:
        eng = AlsEngine(r, cfg.D)
        eng.set_factors(P0, Q0)
        solver = mfitr.MfitrSolver(eng, wl.graph, ew.w, h, r.global_mean)
    per, total_ms, clocks = timed_sweeps(args, 1, dev, [solver.sweep])
    eng.check()
    ms = total_ms / args.steps
    nnz = wl.nnz
    alg = algorithmic(nnz, cfg.users, cfg.items, cfg.D)
    E = wl.graph.num_edges
    extra = E * (12 + 8 * cfg.D) + 4 * cfg.items * (cfg.D + 1)
    extra_f = 2 * E * (2 * cfg.D + 1)
    # per sweep (one step = 4 item layers + users; the layers share the launch budget)
    roof = roofline_for(cfg.D, alg["bytes_sweep"] + extra, alg["flops_sweep"] + extra_f,
                        ms / 1000.0, kernel=kernel_name(cfg.D) + " per item layer + users; "
                        "k_tax_terms per layer")
    roof["per"] = "sweep"
    if full:
        _, sse = solver.predict(wl.valid_users, wl.valid_items, wl.valid_scores)
    else:
        art = torch.as_tensor(wl.graph.artist_array(cfg.items).astype(np.int32), device=dev)
        _, sse = eng.predict(wl.valid_users, wl.valid_items, wl.valid_scores, want_pred=False,
                             mu=r.global_mean, art=art, Q_a=torch.zeros_like(eng.Q))
    rm = float(torch.sqrt(sse / wl.valid_users.numel()).item())
    parity = None
    if not full and not args.skip_parity:
        parity = mfitr_parity(solver, wl.graph, ew.w, cfg)
    cpu = cpu_baseline_for(args, cfg)
    e2e = None
    if not args.skip_e2e:
        del solver, eng, r, tr
        torch.cuda.empty_cache()
        e2e = mfitr_e2e(args, cfg, wl, P0, Q0, 1, args.mfitr_blocks)
    line = {"metric": "MFITR ratings/sec per full sweep", "value": nnz / (ms / 1000.0),
            "unit": "ratings/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator, BASELINE config shapes)",
            "config": arm_config(cfg, 1, {
                "lambda1": h.lam1, "lambda2": cfg.lam, "edges": E, "blocks": args.mfitr_blocks,
                "step": "one ALS-MFITR sweep: 4 item layers + users" + (
                    " + artists; [f|b] blocks, D+1 unknowns" if full else
                    "; factors only (biases, q_a frozen at 0)")}),
            "roofline": roof, "parity": parity,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": None, "clocks": clocks,
            "valid_rmse_after": rm, "layout_build_s": t_layout, "datagen_s": t_gen}
    print(json.dumps(line), flush=True)


def run_sharded_mfitr(args, rank, world, cfg, wl, t_gen):
    """Configs 2 / 4 at N > 1: users cut at nnz quantiles, items assigned by
    whole taxonomy subtree (no exchange inside the layered item half-step),
    one exact all-gather per half-step (parallel.ShardedMfitr).  Strong
    scaling: the same workload for every N."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.device import DeviceRatings
    from paper_1108_2580_b200.parallel import ShardedMfitr
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    # edge weights from the full ratings (every rank computes the same, bit-exact)
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
    tr = wl.train_dataset()
    tr.__dict__["_device_cache"] = {(str(dev), cfg.users, cfg.items): r}
    ew = mfitr.edge_weights(wl.graph, tr, device=dev, num_items=cfg.items)
    mu = r.global_mean
    del r, tr
    torch.cuda.empty_cache()
    run = ShardedMfitr(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items,
                       cfg.D, wl.graph, ew.w, cfg.lam, 2 * cfg.tax_weight, mu, device=dev)
    torch.cuda.synchronize()
    t_layout = time.perf_counter() - t0
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    run.set_factors(P0, Q0)
    per, total_ms, clocks = timed_sweeps(args, world, dev, [run.sweep])
    run.check()
    ms = max_over_ranks(total_ms / args.steps, world)
    nnz = wl.nnz
    D = cfg.D
    local = run.nnz_local["items"] + run.nnz_local["users"]
    roof = roofline_for(D, local * (4 * D + 8), local * (D * D + 3 * D), ms / 1000.0,
                        kernel=kernel_name(D) + " per rank: 4 item layers + users; "
                        "k_tax_terms; all-gather")
    roof["per"] = "sweep (this rank's ratings)"
    e2e = None
    if not args.skip_e2e:
        del run
        torch.cuda.empty_cache()
        e2e = mfitr_e2e(args, cfg, wl, P0, Q0, world, "q")
    if rank == 0:
        line = {"metric": "MFITR ratings/sec per full sweep", "value": nnz / (ms / 1000.0),
                "unit": "ratings/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": arm_config(cfg, world, {
                    "lambda2": cfg.lam, "edges": wl.graph.num_edges, "blocks": "q",
                    "step": "one ALS-MFITR sweep incl. the all-gather after each half-step",
                    "parallelism": f"users nnz-balanced, items by taxonomy subtree (LPT) "
                                   f"over {world} GPU(s)"}),
                "roofline": roof, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": None, "clocks": clocks, "layout_build_s": t_layout,
                "datagen_s": t_gen, "nnz_local_rank0": run.nnz_local if args.skip_e2e else None}
        print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, cfg, wl, t_gen):
    """N > 1: users and items sharded at nnz quantiles, opposite factor
    replicated, exact all-gather of the solved rows after every half-step
    (paper_1108_2580_b200/parallel.py).  Strong scaling: the same config-1
    workload for every N."""
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    from paper_1108_2580_b200.parallel import ShardedAls
    dev = torch.device("cuda", torch.cuda.current_device())
    lam = cfg.lam
    t0 = time.perf_counter()
    run = ShardedAls(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items,
                     cfg.D, device=dev, collective=args.collective)
    torch.cuda.synchronize()
    t_layout = time.perf_counter() - t0
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    run.set_factors(P0, Q0)
    per, total_ms, clocks = timed_sweeps(args, world, dev, [
        lambda: run.half_step("items", 0.0, lam), lambda: run.half_step("users", 0.0, lam)])
    run.check()
    ms_per_step = max_over_ranks(total_ms / args.steps, world)
    nnz = wl.nnz
    value = nnz / (ms_per_step / 1000.0)
    half_ms = per[0] + per[1]
    D = cfg.D
    local_bytes = (run.nnz_local["items"] + run.nnz_local["users"]) * (4 * D + 8) / 2
    local_flops = (run.nnz_local["items"] + run.nnz_local["users"]) * (D * D + 3 * D) / 2
    mean_launch_s = max_over_ranks(statistics.mean(half_ms), world) / 1000.0
    roof = roofline_for(D, local_bytes, local_flops, mean_launch_s,
                        kernel=kernel_name(D) + " per rank (local shard) + all-gather")
    P, Q = run.factors()
    z = torch.zeros(0, dtype=torch.int32, device=dev)
    ev_eng = AlsEngine(DeviceRatings(z, z, z.float(), cfg.users, cfg.items, dev), D)
    ev_eng.set_factors(P, Q)
    rm = float(ev_eng.rmse(wl.valid_users, wl.valid_items, wl.valid_scores).item())
    nnz_local = run.nnz_local
    e2e = None
    if not args.skip_e2e:
        del run, ev_eng, P, Q
        torch.cuda.empty_cache()
        e2e = als_e2e(args, cfg, wl, P0, Q0, world)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ratings/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": arm_config(cfg, world, {
                    "step": "one full sweep incl. the all-gather after each half-step",
                    "parallelism": f"rows sharded over {world} GPUs (nnz-balanced), "
                                   "opposite factor replicated",
                    "collective": args.collective}),
                "roofline": roof, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": 4 * args.steps, "clocks": clocks, "valid_rmse_after": rm,
                "layout_build_s": t_layout, "datagen_s": t_gen, "nnz_local_rank0": nnz_local}
        print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: run the same command as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """--dry-run: the launcher, process group and max-over-ranks plumbing
    only (no data, no kernels); rank 0 prints one JSON line."""
    ones = torch.ones(1, dtype=torch.float64)
    if world > 1:
        ones = ones.to("cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(ones)
    t = max_over_ranks(float(rank), world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": int(ones.item()),
                          "max_rank": t, "backend": dist.get_backend() if world > 1 else None}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-parity", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-scale", type=float, default=0.02,
                    help="size of the reference's sample workload, as a fraction of the config")
    ap.add_argument("--collective", choices=["nccl", "mcf", "peer", "multicast"], default="nccl",
                    help="N > 1 ALS: torch NCCL all-gather, libmcf's own NCCL communicator, or "
                         "the fused stores from the solve kernel (peer / NVLS multicast)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU runner even at N = 1 (exercises its host logic)")
    ap.add_argument("--mfitr-blocks", choices=["q", "full"], default="q",
                    help="configs 2/4: factor blocks only (default) or every MFITR block")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / process-group plumbing only (no data, no kernels)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch(args.gpus))
    rank, world, _ = dist_setup(args.gpus, use_cuda=args.impl == "ours")
    try:
        if args.dry_run:
            run_dry(args, rank, world)
        elif args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
