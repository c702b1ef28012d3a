"""Seeded synthetic rating workloads with the shapes of BASELINE.json configs.

The reference's own generator (pkg/src/multicf/synth.py:169-274, planted
communities + drift) is NOT the generator BASELINE names; this module writes
the one BASELINE.json/SURVEY.md §8(d) describe:

* item popularity Zipf(s) over ranks, ranks mapped to item ids by a seeded
  permutation (popularity is not id-ordered);
* per-user counts: ``min + multinomial`` (config 0) or log-normal with the
  given median, sigma solved so the total is exact (configs 1-4);
* users draw items WITHOUT replacement (successive sampling done as
  draw-with-replacement + keep first distinct draws, repeated for deficits),
  so an item's degree is at most U;
* ground truth u, v ~ N(0, std 1/sqrt(D)); rating
  r = clip(round(50 + 25 u.v + N(0, 15)), 0, 100) (integers, exact in fp32);
* 4 held-out ratings per user, uniformly random (records are stored in a
  random order, so a user's first 4 records in file order are a uniform
  choice);
* MFITR configs: ids are contiguous blocks artists | albums | tracks | genres;
  each album gets one random artist, each track one random album and that
  album's artist, and 0-3 uniform genres (carried, never regularised).

Everything is torch so the full-size workloads generate on the GPU in
seconds; on the CPU (tests, fixtures) the same code is bit-reproducible for
a given seed.  CPU and CUDA random streams differ, so a workload's device is
part of its identity.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .data import Dataset
from .taxonomy import ItemKind, TaxonomyGraph, build_graph_arrays


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    users: int
    items: int
    total: int                 # ratings including the held-out ones
    D: int
    lam: float                 # weighted-lambda (lambda * n_r on the diagonal)
    sweeps: int
    zipf_s: float
    counts: str                # "multinomial" | "lognormal"
    median: int = 120
    min_count: int = 10
    holdout: int = 4
    taxonomy: tuple | None = None   # (tracks, albums, artists, genres)
    tax_weight: float = 0.0         # lambda3 = lambda4 = tax_weight

    @property
    def nnz(self) -> int:
        return self.total - self.holdout * self.users


def _tax_split(items: int) -> tuple:
    base = (507_172, 88_909, 27_888, 992)
    tot = sum(base)
    t, al, ar = (round(items * b / tot) for b in base[:3])
    return (t, al, ar, items - t - al - ar)


CONFIGS = {
    0: WorkloadConfig("cfg0-als-small", 2_000, 1_000, 100_000, 10, 0.065, 5, 1.1,
                      "multinomial"),
    1: WorkloadConfig("cfg1-als-full", 1_000_990, 624_961, 262_810_175, 20, 0.065, 10,
                      1.2, "lognormal"),
    2: WorkloadConfig("cfg2-mfitr-full", 1_000_990, 624_961, 262_810_175, 20, 0.065, 10,
                      1.2, "lognormal", taxonomy=(507_172, 88_909, 27_888, 992),
                      tax_weight=0.1),
    3: WorkloadConfig("cfg3-als-wide", 1_000_990, 624_961, 262_810_175, 100, 0.05, 5,
                      1.2, "lognormal"),
    4: WorkloadConfig("cfg4-mfitr-scaled", 4_000_000, 2_500_000, 1_050_000_000, 50,
                      0.065, 5, 1.2, "lognormal", taxonomy=_tax_split(2_500_000),
                      tax_weight=0.1),
}


def scaled_config(cfg: WorkloadConfig, factor: float, name: str | None = None) -> WorkloadConfig:
    """Same generator at a fraction of the size (parity tests at sizes the
    CPU oracle finishes in seconds)."""
    u = max(50, int(cfg.users * factor))
    i = max(40, int(cfg.items * factor))
    tax = None
    if cfg.taxonomy is not None:
        tax = _tax_split(i)
    per_user = min(cfg.total / cfg.users, i / 8.0)     # keep the density feasible
    total = max(u * (cfg.min_count + 2), int(u * per_user))
    return WorkloadConfig(name or f"{cfg.name}-x{factor:g}", u, i, total, cfg.D, cfg.lam,
                          cfg.sweeps, cfg.zipf_s, cfg.counts, cfg.median, cfg.min_count,
                          cfg.holdout, tax, cfg.tax_weight)


@dataclass
class Workload:
    cfg: WorkloadConfig
    # torch tensors on the generation device, file order
    train_users: torch.Tensor
    train_items: torch.Tensor
    train_scores: torch.Tensor
    valid_users: torch.Tensor
    valid_items: torch.Tensor
    valid_scores: torch.Tensor
    graph: TaxonomyGraph | None
    seed: int

    @property
    def num_users(self) -> int:
        return self.cfg.users

    @property
    def num_items(self) -> int:
        return self.cfg.items

    @property
    def nnz(self) -> int:
        return int(self.train_users.numel())

    def train_dataset(self, compact: bool = True) -> Dataset:
        return Dataset.from_arrays(self.train_users.cpu().numpy(), self.train_items.cpu().numpy(),
                                   self.train_scores.cpu().numpy(), split="train",
                                   num_users=self.num_users, num_items=self.num_items,
                                   compact=compact)

    def valid_dataset(self, compact: bool = True) -> Dataset:
        return Dataset.from_arrays(self.valid_users.cpu().numpy(), self.valid_items.cpu().numpy(),
                                   self.valid_scores.cpu().numpy(), split="valid",
                                   num_users=self.num_users, num_items=self.num_items,
                                   compact=compact)


def _user_counts(cfg: WorkloadConfig, g: torch.Generator, dev) -> torch.Tensor:
    U, total, lo = cfg.users, cfg.total, cfg.min_count
    cap = max(lo, cfg.items // 4)      # keeps successive sampling cheap
    if total > U * cap or total < U * lo:
        raise ValueError(f"{cfg.name}: {total} ratings do not fit {U} users x [{lo}, {cap}]")
    if cfg.counts == "multinomial":
        extra = total - U * lo
        if extra < 0:
            raise ValueError("total below users * min_count")
        draws = torch.randint(0, U, (extra,), generator=g, device=dev)
        counts = lo + torch.bincount(draws, minlength=U)
        return counts.clamp_(max=cap).to(torch.int64)
    z = torch.randn(U, generator=g, device=dev, dtype=torch.float64)
    mu = math.log(cfg.median)

    def total_for(sig):
        c = torch.round(torch.exp(mu + sig * z)).clamp_(lo, cap)
        return float(c.sum())

    a, b = 0.0, 4.0
    for _ in range(80):
        m = 0.5 * (a + b)
        if total_for(m) < total:
            a = m
        else:
            b = m
    counts = torch.round(torch.exp(mu + a * z)).clamp_(lo, cap).to(torch.int64)
    diff = total - int(counts.sum())
    perm = torch.randperm(U, generator=g, device=dev)
    while diff != 0:
        if diff > 0:
            cand = perm[counts[perm] < cap][:diff]
            counts[cand] += 1
        else:
            cand = perm[counts[perm] > lo][:-diff]
            counts[cand] -= 1
        if cand.numel() == 0:
            raise ValueError(f"{cfg.name}: cannot meet the rating total")
        diff = total - int(counts.sum())
    return counts


def _segment_rank(keys_sorted_group: torch.Tensor) -> torch.Tensor:
    """Position of each element inside its run of equal (sorted) group ids."""
    n = keys_sorted_group.numel()
    if n == 0:
        return keys_sorted_group.new_zeros(0)
    idx = torch.arange(n, device=keys_sorted_group.device)
    start = torch.ones(n, dtype=torch.bool, device=keys_sorted_group.device)
    start[1:] = keys_sorted_group[1:] != keys_sorted_group[:-1]
    first = torch.where(start, idx, torch.zeros_like(idx))
    first = torch.cummax(first, 0).values
    return idx - first


def _sample_items(counts: torch.Tensor, cfg: WorkloadConfig, g, dev) -> tuple:
    """(user, rank) pairs: each user draws counts[u] distinct ranks, ppswor
    over Zipf(s) weights, realised as draw-with-replacement keeping the first
    distinct draws (successive sampling), repeated for users left short."""
    U, I = cfg.users, cfg.items
    w = torch.arange(1, I + 1, device=dev, dtype=torch.float64).pow_(-cfg.zipf_s)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    chosen = torch.empty(0, dtype=torch.int64, device=dev)     # sorted keys u*I + rank
    deficit = counts.clone()
    factor = 1.3
    rounds = 0
    while True:
        need_u = torch.nonzero(deficit > 0).flatten()
        if need_u.numel() == 0:
            break
        rounds += 1
        if rounds > 6:
            # users still short only miss rare items: finish them exactly with
            # Gumbel top-k over the items they do not hold yet (same ppswor
            # law), 64 users at a time
            extra = []
            logw = torch.log(w)
            lo_all = torch.searchsorted(chosen, need_u * I)
            hi_all = torch.searchsorted(chosen, (need_u + 1) * I)
            for a in range(0, need_u.numel(), 64):
                us = need_u[a:a + 64]
                lo, hi = lo_all[a:a + 64], hi_all[a:a + 64]
                B = us.numel()
                gum = -torch.log(-torch.log(torch.rand(B, I, generator=g, device=dev,
                                                       dtype=torch.float64)))
                key = logw[None, :] + gum
                lens = hi - lo
                row = torch.repeat_interleave(torch.arange(B, device=dev), lens)
                pos = torch.arange(int(lens.sum()), device=dev) - \
                    torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
                held = chosen[torch.repeat_interleave(lo, lens) + pos] - us[row] * I
                key[row, held] = -float("inf")
                dk = deficit[us]
                top = torch.topk(key, int(dk.max()), dim=1).indices
                keep = torch.arange(top.shape[1], device=dev)[None, :] < dk[:, None]
                extra.append((top + us[:, None] * I)[keep])
            chosen = torch.sort(torch.cat([chosen] + extra)).values
            break
        m = (deficit[need_u].double() * factor).ceil().to(torch.int64) + 2
        uu = torch.repeat_interleave(need_u, m)
        r = torch.searchsorted(cdf, torch.rand(uu.numel(), generator=g, device=dev,
                                               dtype=torch.float64))
        r.clamp_(max=I - 1)
        keys = uu * I + r
        del r
        # drop draws already held by the user
        if chosen.numel():
            pos = torch.searchsorted(chosen, keys).clamp_(max=chosen.numel() - 1)
            keys = keys[chosen[pos] != keys]
        # keep the first occurrence of each key in draw order
        order = torch.sort(keys, stable=True).indices
        ks = keys[order]
        first = torch.ones_like(ks, dtype=torch.bool)
        first[1:] = ks[1:] != ks[:-1]
        keep_pos = torch.sort(order[first]).values          # back to draw order
        keys = keys[keep_pos]
        del order, ks, first, keep_pos
        users_k = keys // I
        # draw order is user-major (uu ascending), so ranks inside a user are
        # positions inside its run
        rk = _segment_rank(users_k)
        acc = keys[rk < deficit[users_k]]
        deficit -= torch.bincount(acc // I, minlength=U)
        chosen = torch.sort(torch.cat([chosen, acc])).values
        factor = 2.5
    return chosen // I, chosen % I


def generate(cfg: WorkloadConfig | int, seed: int = 0, device="cpu") -> Workload:
    """Build the seeded workload of ``cfg`` on ``device``."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    U, I, D = cfg.users, cfg.items, cfg.D
    counts = _user_counts(cfg, g, dev)
    users, ranks = _sample_items(counts, cfg, g, dev)
    item_of_rank = torch.randperm(I, generator=g, device=dev)
    items = item_of_rank[ranks]
    del ranks
    # random record (file) order
    perm = torch.randperm(users.numel(), generator=g, device=dev)
    users = users[perm].to(torch.int32)
    items = items[perm].to(torch.int32)
    del perm
    # ratings from the planted model
    tu = torch.randn(U, D, generator=g, device=dev) / math.sqrt(D)
    tv = torch.randn(I, D, generator=g, device=dev) / math.sqrt(D)
    n = users.numel()
    scores = torch.empty(n, dtype=torch.float32, device=dev)
    step = 1 << 24
    for s in range(0, n, step):
        e = min(n, s + step)
        dot = (tu[users[s:e].long()] * tv[items[s:e].long()]).sum(1)
        noise = torch.randn(e - s, generator=g, device=dev) * 15.0
        scores[s:e] = torch.round(50.0 + 25.0 * dot + noise).clamp_(0.0, 100.0)
    del tu, tv
    # hold out each user's first `holdout` records in file order
    order = torch.sort(users, stable=True).indices
    pos_in_user = _segment_rank(users[order])
    held = torch.zeros(n, dtype=torch.bool, device=dev)
    held[order[pos_in_user < cfg.holdout]] = True
    del order, pos_in_user
    keep = ~held
    graph = _taxonomy(cfg, g, dev) if cfg.taxonomy is not None else None
    return Workload(cfg, users[keep], items[keep], scores[keep],
                    users[held], items[held], scores[held], graph, int(seed))


def _taxonomy(cfg: WorkloadConfig, g, dev) -> TaxonomyGraph:
    T, Al, Ar, G = cfg.taxonomy
    I = cfg.items
    assert T + Al + Ar + G == I
    art0, alb0, trk0, gen0 = 0, Ar, Ar + Al, Ar + Al + T
    kind = np.full(I, -1, dtype=np.int8)
    kind[art0:alb0] = ItemKind.ARTIST
    kind[alb0:trk0] = ItemKind.ALBUM
    kind[trk0:gen0] = ItemKind.TRACK
    kind[gen0:] = ItemKind.GENRE
    album_of = np.full(I, -1, dtype=np.int64)
    artist_link = np.full(I, -1, dtype=np.int64)
    alb_art = torch.randint(0, Ar, (Al,), generator=g, device=dev).cpu().numpy() + art0
    artist_link[alb0:trk0] = alb_art
    trk_alb = torch.randint(0, Al, (T,), generator=g, device=dev).cpu().numpy()
    album_of[trk0:gen0] = trk_alb + alb0
    artist_link[trk0:gen0] = alb_art[trk_alb]
    ng = torch.randint(0, 4, (T,), generator=g, device=dev).cpu().numpy()
    gen_ids = (torch.randint(0, max(G, 1), (int(ng.sum()),), generator=g, device=dev)
               .cpu().numpy() + gen0)
    genre_ptr = np.zeros(I + 1, dtype=np.int64)
    cnt = np.zeros(I, dtype=np.int64)
    cnt[trk0:gen0] = ng if G > 0 else 0
    np.cumsum(cnt, out=genre_ptr[1:])
    if G == 0:
        gen_ids = gen_ids[:0]
    return build_graph_arrays(kind, album_of, artist_link, genre_ptr, gen_ids)


def init_factors(num_users: int, num_items: int, D: int, seed: int = 1, std: float = 0.1):
    """Host-generated fp32 N(0, std) initial factors (Q drawn before P, the
    reference's draw order, factor.py:144-147); shared with the oracle."""
    rng = np.random.default_rng(seed)
    Q0 = (rng.standard_normal((num_items, D), dtype=np.float32) * np.float32(std))
    P0 = (rng.standard_normal((num_users, D), dtype=np.float32) * np.float32(std))
    return P0, Q0
