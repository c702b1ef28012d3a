"""Config-1 sweep time vs the pair path's task length (chunk).  GPU box only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import synth  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "1"))]   # CFG=3: the wide path
wl = synth.generate(cfg, seed=0, device="cuda")
r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
for chunk in [int(c) for c in sys.argv[1:]] or [1024, 2048, 4096]:
    eng = AlsEngine(r, cfg.D, chunk=chunk)
    eng.set_factors(P0, Q0)
    for _ in range(3 if cfg.D <= 20 else 1):
        eng.sweep(0.0, cfg.lam)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    reps = 10 if cfg.D <= 20 else 2
    for _ in range(reps):
        eng.sweep(0.0, cfg.lam)
    e[1].record()
    torch.cuda.synchronize()
    print(f"D={cfg.D} chunk {chunk}: {e[0].elapsed_time(e[1]) / reps:.3f} ms per sweep", flush=True)
    del eng
