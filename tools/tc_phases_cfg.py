"""Phase breakdown of the tensor-core wide path on a full config (default 3):
per half-step and per task class (dual rows, primal rows with n < D, primal
rows, hot chunks) the clock64 phase counters summed over teams, as a share
of all team-cycles and as cycles per task.  MCF_TC_PROF=1.  GPU box only.
    MCF_TC_PROFILE=1 tools/variant.sh prof -e "" && MCF_LIB=build/var_prof.so python tools/tc_phases_cfg.py [cfg]"""
import ctypes
import os
import sys

os.environ["MCF_TC_PROF"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import _lib, synth  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

NAMES = ["task", "gram", "hot", "diag", "trsm", "lastblk", "backsub", "mma", "output", "split"]
CLASSES = ["dual", "primal n<D", "primal", "hot chunk"]
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
dev = torch.device("cuda")
wl = synth.generate(cfg, seed=0, device=dev)
r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
eng = AlsEngine(r, cfg.D)
eng.set_factors(P0, Q0)
L = _lib.lib()
L.mcf_tc_prof_read_classes.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
L.mcf_tc_prof_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 80)()
eng.sweep(0.0, cfg.lam)
L.mcf_tc_prof_read_classes(buf)
for side in ("items", "users"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.half_step(side, 0.0, cfg.lam)
    e1.record()
    torch.cuda.synchronize()
    L.mcf_tc_prof_read_classes(buf)
    cls = buf[16:]
    tot = sum(cls[16 * c + k] for c in range(4) for k in range(10))
    print(f"== {side} half-step: {e0.elapsed_time(e1):.2f} ms (profiled), "
          f"{tot / 1e9:.2f} G team-cycles")
    if buf[13]:
        print(f"  diagonal warp per block: TMEM-load wait {buf[11] / buf[13]:.0f}, "
              f"factorisation {buf[12] / buf[13]:.0f} cycles ({buf[13]} blocks)")
    for c in range(4):
        nt = cls[16 * c + 10]
        ct = sum(cls[16 * c + k] for k in range(10))
        if nt == 0:
            continue
        print(f"  {CLASSES[c]:<11} {nt:>8} tasks, {100 * ct / tot:5.1f}% of cycles, "
              f"{ct / nt:8.0f} cycles/task: " +
              ", ".join(f"{NAMES[k]} {cls[16 * c + k] / nt:.0f}" for k in range(10) if cls[16 * c + k]))
