"""Device time of one config-1 layout build (both sides), for the launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import synth  # noqa: E402
from paper_1108_2580_b200.device import DeviceRatings  # noqa: E402

cfg = synth.CONFIGS[1]
wl = synth.generate(cfg, seed=0, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items)
    e1.record()
    torch.cuda.synchronize()
    print(f"layouts rep {rep}: {e0.elapsed_time(e1):.1f} ms")
    del r
