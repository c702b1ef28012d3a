"""Phase timing of one ALS-MFITR full-block sweep (MfitrFullSolver) at a
config (default 2): gather-table builds, per-rating targets, taxonomy terms
and each block's solve, CUDA events on the current stream.  GPU box only.
    python tools/mfitr_phases.py [cfg]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import mfitr, synth  # noqa: E402
from paper_1108_2580_b200.device import DeviceRatings  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
dev = torch.device("cuda")
wl = synth.generate(cfg, seed=0, device=dev)
r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
tr = wl.train_dataset()
tr.__dict__["_device_cache"] = {(str(dev), cfg.users, cfg.items): r}
ew = mfitr.edge_weights(wl.graph, tr, device=dev, num_items=cfg.items)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
h = mfitr.MfitrHyper(D=cfg.D, lam1=cfg.lam, lam2=cfg.lam, lam3=cfg.tax_weight,
                     lam4=cfg.tax_weight, iters=cfg.sweeps)
s = mfitr.MfitrFullSolver(r, wl.graph, ew.w, h, r.global_mean, wl.graph.artist_array(cfg.items),
                          P0, Q0)
for _ in range(2):
    s.sweep()
torch.cuda.synchronize()
marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((name, e))


mark("start")
s._item_prep()
mark("items: [p|1] table + targets")
for k in range(len(s.layers)):
    s._solve_layer(k)
    mark(f"items: layer {k} ({int(s.layers[k].numel())} rows)")
if s.fused:
    s.artists()
    mark(f"artists: from the emitted item systems ({int(s.artist_row.numel())} artists)")
else:
    s._fixed(s.Pa, None, None, s.U, s.Xu)
    mark("artists: [p|1] table")
    s._targets(2, s.by_artist, s.art_item, s.t_art)
    mark(f"artists: targets ({s.by_artist.nnz} ratings)")
    s.solver.solve(s.by_artist, s.Xu, s.Aa, 0.0, h.lam2, fail=s.fail, val=s.t_art, bias=s._bias())
    mark("artists: solve")
if s.fused:
    s.users()
    mark("users: [q+q_a|1|b_i+b_a] table + solve")
else:
    s._fixed(s.Qa, s.Aa, s.art, s.I, s.Xi)
    mark("users: [q+q_a|1] table")
    s._targets(0, r.by_user, None, s.t_users)
    mark("users: targets")
    s.solver.solve(r.by_user, s.Xi, s.Pa, 0.0, h.lam2, fail=s.fail, val=s.t_users, bias=s._bias())
    mark("users: solve")
torch.cuda.synchronize()
s.check()
tot = marks[0][1].elapsed_time(marks[-1][1])
for (a, ea), (b, eb) in zip(marks, marks[1:]):
    print(f"{b:<40} {ea.elapsed_time(eb):7.2f} ms")
print(f"{'sweep':<40} {tot:7.2f} ms")
