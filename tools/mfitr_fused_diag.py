"""Fused MFITR item step: YSUB gather vs precomputed targets (mode 3) vs the
per-rating legacy path, one item sweep from the same state.  GPU box only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_mfitr as T  # noqa: E402
from conftest import GOLDEN  # noqa: E402

g = dict(np.load(os.path.join(GOLDEN, "mfitr_cfg2s.npz")))
D = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(20)
U, I = int(g["U"]), int(g["I"])
g["P"], g["Q"] = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
g["Qa"] = rng.normal(0, 0.05, (I, D))
g["bu"], g["bi"], g["ba"] = rng.normal(0, 1, U), rng.normal(0, 1, I), rng.normal(0, 1, I)
g["lam1"] = 0.0
if os.environ.get("ZERO_BU"):
    g["bu"] = np.zeros(U)
if os.environ.get("ZERO_MU"):
    g["mu"] = np.float64(0.0)
res = {}
for mode in ("ysub", "mode3", "legacy"):
    if mode == "legacy":
        os.environ["MCF_MFITR_LEGACY"] = "1"
    fs = T._full_solver(g)
    os.environ.pop("MCF_MFITR_LEGACY", None)
    if mode == "mode3":
        fs._fixed(fs.Pa, None, None, fs.U, fs.Xu)
        fs._targets(3, fs.r.by_item, fs.item_rows, fs.t_items)
        h = fs.hyper
        from paper_1108_2580_b200 import _lib
        from paper_1108_2580_b200._lib import ptr
        from paper_1108_2580_b200.device import stream_ptr
        for k in range(len(fs.layers)):
            rows = fs.layers[k]
            if not rows.numel():
                continue
            _lib.check(_lib.lib().mcf_taxonomy_terms(
                ptr(fs.inc_ptr), ptr(fs.inc_edge), ptr(fs.inc_other), ptr(fs.w), ptr(fs.Qa), fs.I,
                fs.D + 1, ptr(rows), rows.numel(), ptr(fs.S), ptr(fs.T), stream_ptr(fs.device)), "tax")
            fs.solver.solve(fs.r.by_item, fs.Xu, fs.Qa, 0.0, h.lam2, 0.0, fs.S, fs.T, fs.tau, rows,
                            ("layer", k), None, fs.fail, None, val=fs.t_items, bias=fs._bias(),
                            emit=(fs.emit, fs.Aa, fs.art, False))
    else:
        fs.item_layers()
    fs.check()
    res[mode] = [x.copy() for x in T._host_params(fs)]
names = ["P", "Q", "bu", "bi", "ba", "Qa"]
for a, b in (("ysub", "mode3"), ("mode3", "legacy"), ("ysub", "legacy")):
    print(D, a, "vs", b, " ".join(f"{n}:{np.abs(x - y).max():.2e}" for n, x, y in zip(names, res[a], res[b])))
