"""Device time of one config-1-sized layout build per side (skewed synthetic
keys, no generator), for CUDA-event timing and the ncu launch list
(`ncu -k regex:^k_ ...`).  GPU box only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200.device import SideLayout  # noqa: E402

U, I, NNZ = 1000990, 624961, 258806215
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.randint(0, U, (NNZ,), device="cuda", dtype=torch.int32, generator=g)
x = torch.rand(NNZ, device="cuda", generator=g)
i = (x.pow(3) * I).to(torch.int32).clamp_(max=I - 1)      # skewed: hot low ids
s = torch.rand(NNZ, device="cuda", generator=g) * 100
del x
for rep in range(reps):
    for name, k, c, n in (("users", u, i, U), ("items", i, u, I)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lay = SideLayout(k, c, s, n)
        e1.record()
        torch.cuda.synchronize()
        print(f"rep {rep} {name}: {e0.elapsed_time(e1):.2f} ms")
        del lay
