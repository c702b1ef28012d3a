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
* roofline: the dominant kernel is the fused Gram+Cholesky half-step
  (k_als_warp<5>, 2 launches per sweep); achieved = algorithmic bytes per
  launch (n_nnz (4D + 8) + 4D n_rows_solved) / mean launch
  time from CUDA events around each half-step.
* e2e: the same metric through the public drop-in API
  ``factor.train("wals", ...)`` on HOST (pinned) arrays: H2D of the COO
  split, both layout builds, `sweeps` sweeps with the per-sweep objective and
  held-out RMSE, D2H of the factors -- ratings * sweeps / wall time.
* cpu_baseline (rank 0, N = 1): the CPU oracle port (oracle/als_oracle.c, the
  reference's als_solve_rows restated in C float64, pthreads over static
  row blocks like parallel.run_blocks) on a bounded random sample of rows of
  both layouts, using all host cores.
* --impl reference: that same CPU port as its own arm (ratings/s per full
  sweep extrapolated from the timed sample sweeps).
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
    if D <= 20:
        return "k_als_pair<5,4> (fused Gram + lam*n + Cholesky + solve; + k_als_heavy for hot rows)"
    if D <= 28:
        return "k_als_warp (4x4 register tiles, warp Cholesky)"
    if D <= 104:
        return "k_als_tile_warp (warp per row, 8x8 register tiles, blocked register Cholesky)"
    return "k_als_cta"


def roofline_for(D, bytes_launch, flops_launch, launch_s, traffic=None, kernel=None):
    """roofline time = max(bytes / HBM, flops / FP32 peak) per
    launch; the bound is whichever is larger and `achieved` is reported in
    that resource's unit (GB/s or TFLOP/s), the other view beside it."""
    hbm, hbm_kind = peaks()
    f32, f32_kind = fp32_peak()
    t_hbm = bytes_launch / (hbm * 1e9)
    t_f32 = flops_launch / (f32 * 1e12)
    gbs = bytes_launch / launch_s / 1e9
    tfs = flops_launch / launch_s / 1e12
    if t_hbm >= t_f32:
        r = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
             "peak_kind": hbm_kind, "achieved_tflops": tfs, "fp32_peak_tflops": f32}
    else:
        r = {"bound": "fp32", "achieved": tfs, "peak": f32, "unit": "TFLOP/s", "frac": tfs / f32,
             "peak_kind": f32_kind, "achieved_gbs": gbs, "hbm_peak_gbs": hbm}
    r.update({"traffic": traffic, "kernel": kernel or kernel_name(D),
              "roofline_ms_per_launch": 1e3 * max(t_hbm, t_f32),
              "algorithmic_bytes_per_launch": bytes_launch,
              "algorithmic_flops_per_launch": flops_launch})
    return r


def launches_per_sweep(eng) -> int:
    """libmcf kernels per sweep: per half-step the row kernel, plus the hot-row
    reduce kernel when the layout has hot rows (D <= 20 path)."""
    n = 0
    for lay in (eng.r.by_item, eng.r.by_user):
        info = lay.plan()[1]
        n += 1 + (1 if eng.D <= 20 and info[4] > 0 else 0)
    return n


def peaks():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_setup(n_gpus):
    if n_gpus > 1 or "RANK" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        rank, world = dist.get_rank(), dist.get_world_size()
    else:
        rank, world = 0, 1
    local = int(os.environ.get("LOCAL_RANK", rank))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU baseline (oracle port) on a bounded sample

def sample_rows(lay, n_rows_target, rng):
    n = lay.n_rows
    rows = np.sort(rng.choice(n, size=min(n_rows_target, n), replace=False)).astype(np.int64)
    ptr = lay.ptr.cpu().numpy()
    starts, ends = ptr[rows], ptr[rows + 1]
    counts = ends - starts
    sub_ptr = np.zeros(rows.size + 1, np.int64)
    np.cumsum(counts, out=sub_ptr[1:])
    flat = np.concatenate([np.arange(a, b) for a, b in zip(starts, ends)]) if rows.size else \
        np.zeros(0, np.int64)
    ft = torch.from_numpy(flat).to(lay.idx.device)
    idx = lay.idx[ft].cpu().numpy().astype(np.int64)
    val = lay.val[ft].cpu().numpy().astype(np.float64)
    return sub_ptr, idx, val, int(counts.sum())


def cpu_sample_sweep(engine, lam, sample_rows_per_side=(4000, 2000), seed=7, threads=None,
                     repeats=1):
    """Time the oracle port on sampled rows of both layouts; returns
    (ratings/s per full sweep, description, cores)."""
    import oracle
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    P, Q = (t.double().cpu().numpy() for t in engine.factors())
    rates, desc = {}, []
    for side, nrow in zip(("users", "items"), sample_rows_per_side):
        lay = engine.r.layout(side)
        sp, idx, val, n = sample_rows(lay, nrow, rng)
        fixed = Q if side == "users" else P
        ts = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            oracle.solve_rows((sp, idx, val, None), fixed, sp.size - 1, lam_n=lam,
                              threads=threads)
            ts.append(time.perf_counter() - t0)
        rates[side] = n / min(ts)
        desc.append(f"{side}: {sp.size - 1} random rows, {n} ratings")
    per_sweep = 1.0 / (1.0 / rates["users"] + 1.0 / rates["items"])
    return per_sweep, "; ".join(desc), threads, rates


# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    cfg = synth.CONFIGS[args.config]
    wl = synth.generate(cfg, seed=0, device="cuda")
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items)
    eng = AlsEngine(r, cfg.D)
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    eng.set_factors(P0, Q0)
    del wl
    vals = []
    desc = cores = None
    for s in range(args.warmup + args.steps):
        v, desc, cores, _ = cpu_sample_sweep(eng, cfg.lam, seed=100 + s)
        if s >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    nnz = r.nnz
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "ratings/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * nnz / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "users": cfg.users, "items": cfg.items,
                       "nnz_train": nnz, "D": cfg.D, "lambda_weighted": cfg.lam},
            "cpu_baseline": {"value": value, "unit": "ratings/s", "cores": cores,
                             "kind": "port", "sample": desc},
            "e2e": {"value": value, "unit": "ratings/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings

    cfg = synth.CONFIGS[args.config]
    if args.scale != 1.0:
        cfg = synth.scaled_config(cfg, args.scale)
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    wl = synth.generate(cfg, seed=0, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    nnz = wl.nnz
    if world > 1 or args.force_sharded:
        if cfg.taxonomy is not None:
            return run_sharded_mfitr(args, rank, world, cfg, wl, t_gen)
        return run_sharded(args, rank, world, cfg, wl, t_gen)
    if cfg.taxonomy is not None:
        return run_mfitr(args, cfg, wl, t_gen)
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
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        eng.sweep(0.0, lam)
    eng.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(dev.index)).split(",")[0]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else dev.index
    with ClockSampler(gpu_index) as clk:
        time.sleep(0.3)
        torch.cuda.synchronize()
        ev[0].record(stream)
        for s in range(args.steps):
            eng.half_step("items", 0.0, lam)
            ev[2 * s + 1].record(stream)
            eng.half_step("users", 0.0, lam)
            ev[2 * s + 2].record(stream)
        torch.cuda.synchronize()
    eng.check()
    total_ms = ev[0].elapsed_time(ev[-1])
    half_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(2 * args.steps)]
    ms_per_step = max_over_ranks(total_ms / args.steps, world)
    value = nnz / (ms_per_step / 1000.0)

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
    roofline["launch_ms"] = {"items": statistics.mean(half_ms[0::2]),
                             "users": statistics.mean(half_ms[1::2])}

    # held-out RMSE after the timed sweeps (sanity, not timed)
    rm = float(eng.rmse(wl.valid_users, wl.valid_items, wl.valid_scores).item())
    n_launch = launches_per_sweep(eng) * args.steps

    # ---- CPU baseline (oracle port, bounded sample) ----
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        v, desc, cores, rates = cpu_sample_sweep(eng, lam)
        cpu = {"value": v, "unit": "ratings/s", "cores": cores, "kind": "port", "sample": desc,
               "per_side_ratings_per_s": rates}

    # ---- e2e through the public API on host buffers ----
    e2e = None
    if not args.skip_e2e:
        def pinned(t):
            return t.cpu().pin_memory().numpy()
        tu, ti, ts = pinned(wl.train_users), pinned(wl.train_items), pinned(wl.train_scores)
        vu, vi, vs = pinned(wl.valid_users), pinned(wl.valid_items), pinned(wl.valid_scores)
        tr = Dataset.from_arrays(tu, ti, ts, num_users=cfg.users, num_items=cfg.items,
                                 compact=True)
        va = Dataset.from_arrays(vu, vi, vs, num_users=cfg.users, num_items=cfg.items,
                                 compact=True)
        del r, eng
        torch.cuda.empty_cache()
        hp = factor.HyperParams(lam=lam, D=cfg.D, iters=cfg.sweeps)
        e2e_steps = max(1, args.e2e_steps)
        times = []
        # the step's host inputs (init factors too) and outputs live in pinned memory
        P0p = torch.from_numpy(P0).pin_memory()
        Q0p = torch.from_numpy(Q0).pin_memory()
        Pn = torch.empty(cfg.users, cfg.D, dtype=torch.float32, pin_memory=True)
        Qn = torch.empty(cfg.items, cfg.D, dtype=torch.float32, pin_memory=True)
        for s in range(e2e_steps + 1):
            tr.__dict__.pop("_device_cache", None)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            model, rep = factor.train("wals", tr, va, hp, reg="weighted", init=(P0p, Q0p),
                                      device=dev, as_torch=True)
            Pn.copy_(model.p, non_blocking=True)
            Qn.copy_(model.q, non_blocking=True)
            torch.cuda.synchronize()
            if s > 0:   # first call warms allocator/plans
                times.append(time.perf_counter() - t0)
            e2e_rmse = rep[-1].valid_rmse
            del model
            tr.__dict__.pop("_device_cache", None)
        t_e2e = max_over_ranks(statistics.median(times), world)
        h2d = tu.nbytes + ti.nbytes + ts.nbytes + vu.nbytes + vi.nbytes + vs.nbytes + \
            P0.nbytes + Q0.nbytes
        d2h = Pn.numel() * 4 + Qn.numel() * 4 + 16 * cfg.sweeps
        e2e = {"value": nnz * cfg.sweeps / t_e2e, "unit": "ratings/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "step": f"one factor.train('wals', reg='weighted') call: {cfg.sweeps} sweeps "
                       "+ layout builds + per-sweep objective and held-out RMSE",
               "seconds_per_step": t_e2e, "valid_rmse": e2e_rmse}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ratings/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": {"workload": cfg.name, "users": cfg.users, "items": cfg.items,
                           "nnz_train": nnz, "D": cfg.D, "lambda_weighted": lam,
                           "step": "one full sweep (items then users half-step)",
                           "l2": "inputs > L2 (CSR/CSC 8 B/rating = 2.07 GB each vs 126 MB L2); "
                                 "no flush",
                           "parallelism": f"rows sharded over {world} GPU(s)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": n_launch, "clocks": clk.summary(),
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
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        solver.sweep()
    eng.check()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev.index) as clk:
        time.sleep(0.2)
        torch.cuda.synchronize()
        ev[0].record(stream)
        for s in range(args.steps):
            solver.sweep()
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
    eng.check()
    ms = ev[0].elapsed_time(ev[-1]) / args.steps
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
    line = {"metric": "MFITR ratings/sec per full sweep", "value": nnz / (ms / 1000.0),
            "unit": "ratings/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator, BASELINE config shapes)",
            "config": {"workload": cfg.name, "users": cfg.users, "items": cfg.items,
                       "nnz_train": nnz, "D": cfg.D, "lambda1": h.lam1, "lambda2": cfg.lam,
                       "lambda3": cfg.tax_weight, "lambda4": cfg.tax_weight,
                       "edges": E, "blocks": args.mfitr_blocks,
                       "step": "one ALS-MFITR sweep: 4 item layers + users" + (
                           " + artists; [f|b] blocks, D+1 unknowns" if full else
                           "; factors only (biases, q_a frozen at 0)")},
            "roofline": roof,
            "cpu_baseline": None, "e2e": None, "gpu_launches": None, "clocks": clk.summary(),
            "valid_rmse_after": rm, "layout_build_s": t_layout, "datagen_s": t_gen}
    print(json.dumps(line), flush=True)


def run_sharded_mfitr(args, rank, world, cfg, wl, t_gen):
    """Configs 2 / 4 at N > 1: users cut at nnz quantiles, items assigned by
    whole taxonomy subtree (no exchange inside the layered item half-step),
    one in-place NCCL all-gather per half-step (parallel.ShardedMfitr).
    Strong scaling: the same workload for every N."""
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
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        run.sweep()
    run.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev.index) as clk:
        time.sleep(0.2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev[0].record(stream)
        for s in range(args.steps):
            run.sweep()
            ev[s + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    run.check()
    ms = max_over_ranks(ev[0].elapsed_time(ev[-1]) / args.steps, world)
    nnz = wl.nnz
    D = cfg.D
    local = run.nnz_local["items"] + run.nnz_local["users"]
    roof = roofline_for(D, local * (4 * D + 8), local * (D * D + 3 * D), ms / 1000.0,
                        kernel=kernel_name(D) + " per rank: 4 item layers + users; "
                        "k_tax_terms; all-gather")
    roof["per"] = "sweep (this rank's ratings)"
    if rank == 0:
        line = {"metric": "MFITR ratings/sec per full sweep", "value": nnz / (ms / 1000.0),
                "unit": "ratings/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": {"workload": cfg.name, "users": cfg.users, "items": cfg.items,
                           "nnz_train": nnz, "D": D, "lambda2": cfg.lam,
                           "lambda3": cfg.tax_weight, "lambda4": cfg.tax_weight,
                           "edges": wl.graph.num_edges, "blocks": "q",
                           "step": "one ALS-MFITR sweep incl. the all-gather after each half-step",
                           "parallelism": f"users nnz-balanced, items by taxonomy subtree (LPT) "
                                          f"over {world} GPU(s)"},
                "roofline": roof, "cpu_baseline": None, "e2e": None,
                "gpu_launches": None, "clocks": clk.summary(), "layout_build_s": t_layout,
                "datagen_s": t_gen, "nnz_local_rank0": run.nnz_local}
        print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, cfg, wl, t_gen):
    """N > 1: users and items sharded at nnz quantiles, opposite factor
    replicated, in-place NCCL all-gather of the solved shard after every
    half-step (paper_1108_2580_b200/parallel.py).  Strong scaling: the same
    config-1 workload for every N."""
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
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        run.sweep(0.0, lam)
    run.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    with ClockSampler(dev.index) as clk:
        time.sleep(0.2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev[0].record(stream)
        for s in range(args.steps):
            run.half_step("items", 0.0, lam)
            ev[2 * s + 1].record(stream)
            run.half_step("users", 0.0, lam)
            ev[2 * s + 2].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    run.check()
    total_ms = ev[0].elapsed_time(ev[-1])
    ms_per_step = max_over_ranks(total_ms / args.steps, world)
    nnz = wl.nnz
    value = nnz / (ms_per_step / 1000.0)
    half_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(2 * args.steps)]
    D = cfg.D
    local_bytes = (run.nnz_local["items"] + run.nnz_local["users"]) * (4 * D + 8) / 2
    local_flops = (run.nnz_local["items"] + run.nnz_local["users"]) * (D * D + 3 * D) / 2
    mean_launch_s = max_over_ranks(statistics.mean(half_ms), world) / 1000.0
    roof = roofline_for(D, local_bytes, local_flops, mean_launch_s,
                        kernel=kernel_name(D) + " per rank (local shard) + all-gather")
    P, Q = run.factors()
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    z = torch.zeros(0, dtype=torch.int32, device=dev)
    ev_eng = AlsEngine(DeviceRatings(z, z, z.float(), cfg.users, cfg.items, dev), D)
    ev_eng.set_factors(P, Q)
    rm = float(ev_eng.rmse(wl.valid_users, wl.valid_items, wl.valid_scores).item())
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "ratings/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded generator, BASELINE config shapes)",
                "config": {"workload": cfg.name, "users": cfg.users, "items": cfg.items,
                           "nnz_train": nnz, "D": D, "lambda_weighted": lam,
                           "step": "one full sweep incl. the NCCL all-gather after each half-step",
                           "l2": "inputs > L2; no flush",
                           "parallelism": f"rows sharded over {world} GPUs (nnz-balanced), "
                                          "opposite factor replicated",
                           "collective": args.collective},
                "roofline": roof,
                "cpu_baseline": None, "e2e": None, "gpu_launches": 4 * args.steps,
                "clocks": clk.summary(), "valid_rmse_after": rm, "layout_build_s": t_layout,
                "datagen_s": t_gen}
        print(json.dumps(line), flush=True)


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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--collective", choices=["nccl", "peer"], default="nccl",
                    help="N > 1 ALS: NCCL all-gather after each half-step, or the fused "
                         "peer stores from the solve kernel (symmetric memory)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU runner even at N = 1 (exercises its host logic)")
    ap.add_argument("--mfitr-blocks", choices=["q", "full"], default="q",
                    help="configs 2/4: factor blocks only (default) or every MFITR block")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, _ = dist_setup(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
