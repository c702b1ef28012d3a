"""Per-row solve cost of the wide paths: a users half-step where every row
has only `n` ratings (Gram work negligible), D in argv.  GPU box only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

U, I = 1_000_000, 4096
for D in [int(x) for x in sys.argv[1:]] or [50, 100]:
    for n in [int(x) for x in os.environ.get("NS", "8,64,256").split(",")]:
        g = torch.Generator(device="cuda").manual_seed(0)
        users = torch.arange(U, device="cuda", dtype=torch.int32).repeat_interleave(n)
        items = torch.randint(0, I, (U * n,), device="cuda", dtype=torch.int32, generator=g)
        scores = torch.rand(U * n, device="cuda", generator=g) * 100
        r = DeviceRatings(users, items, scores, U, I)
        eng = AlsEngine(r, D)
        eng.set_factors(torch.randn(U, D) * 0.1, torch.randn(I, D) * 0.1)
        for _ in range(2):
            eng.half_step("users", 0.0, 0.05)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            eng.half_step("users", 0.0, 0.05)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"D={D} n={n}: {ms:.2f} ms per users half-step ({U} rows, {U*n} ratings) "
              f"= {ms*1e3/U*148:.2f} us per row per SM")
        del r, eng
