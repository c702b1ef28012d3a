"""Compare the layout build against torch's stable sort (CUB onesweep) on
config-1 keys: a yardstick for the radix passes only.  GPU box only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import synth  # noqa: E402
from paper_1108_2580_b200.device import SideLayout  # noqa: E402

cfg = synth.CONFIGS[1]
wl = synth.generate(cfg, seed=0, device="cuda")
u, i, s = (x.to(torch.int32) for x in (wl.train_users, wl.train_items)), None, wl.train_scores
u, i = wl.train_users.to(torch.int32), wl.train_items.to(torch.int32)


def timed(fn, n=3):
    out = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
        del r
    return min(out)


print(f"SideLayout(users) {timed(lambda: SideLayout(u, i, s, cfg.users)):.2f} ms")
print(f"SideLayout(items) {timed(lambda: SideLayout(i, u, s, cfg.items)):.2f} ms")
print(f"torch.sort(users, stable) {timed(lambda: torch.sort(u, stable=True)):.2f} ms")
print(f"torch.sort(items, stable) {timed(lambda: torch.sort(i, stable=True)):.2f} ms")
print(f"s.double().mean() {timed(lambda: s.double().mean()):.2f} ms")
