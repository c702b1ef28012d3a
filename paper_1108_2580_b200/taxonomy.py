"""Item taxonomy (track -> album -> artist forest) for MFITR.

Host-side mirror of the reference's ``multicf.taxonomy``
(reference: pkg/src/multicf/taxonomy.py:16-118).  The integer maps that
feed the device -- the (child, parent) edge list sorted by (child, parent)
(taxonomy.py:106-118), ``artist_array`` (taxonomy.py:82-90) and the
per-item incident-edge index used by the segmented S/T reduction -- are
built with vectorised numpy and must equal the reference's bit for bit
(tests/test_taxonomy.py pins them against fixtures made by the reference).

Genre links are carried (``genre_ptr``/``genre_ids``) but never become
edges: the reference's graph has no genre edges (taxonomy.py:3-4,106-118).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from .errors import DanglingReferenceError, ParseError, TaxonomyError, UnknownIdError


class ItemKind(IntEnum):
    TRACK = 0
    ALBUM = 1
    ARTIST = 2
    GENRE = 3


@dataclass
class TaxonomyGraph:
    kind: np.ndarray            # int8, -1 = not in the graph
    album_of: np.ndarray        # int64, -1 = none
    artist_link: np.ndarray     # int64, -1 = none
    genre_ptr: np.ndarray       # int64 [n+1] CSR of genre tags (never regularised)
    genre_ids: np.ndarray       # int64
    edge_child: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    edge_parent: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    dropped_links: int = 0

    @property
    def num_nodes(self) -> int:
        return int(self.kind.size)

    @property
    def num_edges(self) -> int:
        return int(self.edge_child.size)

    def __contains__(self, i: int) -> bool:
        return 0 <= i < self.kind.size and self.kind[i] >= 0

    @property
    def genres(self) -> dict:
        out = {}
        for i in np.flatnonzero(np.diff(self.genre_ptr) > 0):
            out[int(i)] = tuple(int(x) for x in
                                self.genre_ids[self.genre_ptr[i]:self.genre_ptr[i + 1]])
        return out

    def artist_of(self, i: int):
        if i not in self:
            raise UnknownIdError(f"item {i} not in taxonomy")
        if self.kind[i] == ItemKind.ARTIST:
            return int(i)
        a = int(self.artist_link[i])
        return a if a >= 0 else None

    def artist_array(self, num_items: int) -> np.ndarray:
        """Dense artist id per item, -1 when unknown; an artist maps to
        itself (reference taxonomy.py:82-90)."""
        out = np.full(num_items, -1, dtype=np.int64)
        n = min(num_items, self.kind.size)
        k = self.kind[:n]
        sel = k >= 0
        out[:n][sel] = self.artist_link[:n][sel]
        art = np.flatnonzero(k == ItemKind.ARTIST)
        out[art] = art
        return out

    def validate(self) -> None:
        """Every edge goes up the track < album < artist layering
        (reference taxonomy.py:92-103)."""
        if self.edge_child.size and not np.all(self.kind[self.edge_parent] >
                                                self.kind[self.edge_child]):
            raise TaxonomyError("edge violates track<album<artist layering")

    def incident_edges(self, num_items: int):
        """CSR over items of incident edges: (ptr, edge_id, other_end).

        Each edge appears twice, once under its child and once under its
        parent; inside an item the entries are in edge-list order, so the
        segmented reduction sums them in a fixed order."""
        E = self.edge_child.size
        ends = np.concatenate([self.edge_child, self.edge_parent])
        other = np.concatenate([self.edge_parent, self.edge_child])
        eid = np.concatenate([np.arange(E), np.arange(E)])
        order = np.argsort(ends, kind="stable")
        ptr = np.zeros(num_items + 1, dtype=np.int64)
        np.cumsum(np.bincount(ends, minlength=num_items), out=ptr[1:])
        return ptr, eid[order].astype(np.int64), other[order].astype(np.int64)

    def layers(self, num_items: int):
        """Item ids per solve layer: tracks, albums, artists, then every other
        item (genres, untyped, beyond the graph).  No edge joins two items of
        one layer (layering), so a layer's rows are independent given the
        others -- the exact block solve of the ALS-MFITR item half-step."""
        kind = np.full(num_items, -1, dtype=np.int8)
        n = min(num_items, self.kind.size)
        kind[:n] = self.kind[:n]
        return [np.flatnonzero(kind == ItemKind.TRACK),
                np.flatnonzero(kind == ItemKind.ALBUM),
                np.flatnonzero(kind == ItemKind.ARTIST),
                np.flatnonzero((kind < 0) | (kind == ItemKind.GENRE))]


def _edges(kind, album_of, artist_link):
    """Edge list sorted by (child, parent) (reference taxonomy.py:106-118)."""
    ids = np.flatnonzero(kind >= 0)
    k = kind[ids]
    t = ids[(k == ItemKind.TRACK) & (album_of[ids] >= 0)]
    a = ids[(k != ItemKind.ARTIST) & (artist_link[ids] >= 0)]
    child = np.concatenate([t, a]).astype(np.int64)
    parent = np.concatenate([album_of[t], artist_link[a]]).astype(np.int64)
    order = np.lexsort((parent, child))
    return child[order], parent[order]


def build_graph_arrays(kind, album_of, artist_link, genre_ptr=None, genre_ids=None,
                       dropped: int = 0) -> TaxonomyGraph:
    kind = np.asarray(kind, dtype=np.int8)
    album_of = np.asarray(album_of, dtype=np.int64)
    artist_link = np.asarray(artist_link, dtype=np.int64)
    if genre_ptr is None:
        genre_ptr = np.zeros(kind.size + 1, dtype=np.int64)
        genre_ids = np.zeros(0, dtype=np.int64)
    ec, ep = _edges(kind, album_of, artist_link)
    return TaxonomyGraph(kind, album_of, artist_link, np.asarray(genre_ptr, np.int64),
                         np.asarray(genre_ids, np.int64), ec, ep, dropped)


def build_graph(kind, album_of, artist_link, genres: dict | None = None,
                dropped: int = 0) -> TaxonomyGraph:
    """Reference-signature constructor (taxonomy.py:106): genres as a dict."""
    kind = np.asarray(kind, dtype=np.int8)
    n = kind.size
    cnt = np.zeros(n, dtype=np.int64)
    ids = []
    for i in sorted((genres or {}).keys()):
        cnt[i] = len(genres[i])
        ids.extend(genres[i])
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=ptr[1:])
    return build_graph_arrays(kind, album_of, artist_link, ptr,
                              np.asarray(ids, dtype=np.int64), dropped)


_KIND_NAMES = {"track": ItemKind.TRACK, "album": ItemKind.ALBUM, "artist": ItemKind.ARTIST}


def load_taxonomy(path, strict: bool = True) -> TaxonomyGraph:
    """Parse `kind|item|album_or_NA|artist_or_NA|genre,genre,...` lines
    (reference taxonomy.py:121-196): strict mode raises on undeclared or
    wrong-kind parents, lenient mode drops and counts them; a track with an
    album but no artist inherits the album's artist."""
    rows = []
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, line in enumerate(fh, start=1):
            line = line.rstrip("\n")
            if not line.strip() or line.startswith("#"):
                continue
            parts = line.split("|")
            if len(parts) != 5:
                raise ParseError(path, line_no, f"expected 5 '|' fields, got {len(parts)}")
            kname, id_s, alb_s, art_s, gen_s = parts
            if kname not in _KIND_NAMES:
                raise ParseError(path, line_no, f"unknown kind {kname!r}")
            try:
                item = int(id_s)
                alb = -1 if alb_s == "NA" else int(alb_s)
                art = -1 if art_s == "NA" else int(art_s)
                gens = tuple(int(g) for g in gen_s.split(",") if g)
            except ValueError as exc:
                raise ParseError(path, line_no, f"non-numeric field: {exc}") from None
            if item < 0:
                raise ParseError(path, line_no, "negative item id")
            rows.append((line_no, _KIND_NAMES[kname], item, alb, art, gens))
    if not rows:
        return build_graph(np.empty(0, np.int8), np.empty(0, np.int64), np.empty(0, np.int64), {})
    n = max(r[2] for r in rows) + 1
    kind = np.full(n, -1, dtype=np.int8)
    album_of = np.full(n, -1, dtype=np.int64)
    artist_link = np.full(n, -1, dtype=np.int64)
    genres = {}
    for line_no, k, item, _, _, _ in rows:
        if kind[item] >= 0:
            raise TaxonomyError(f"{path}:{line_no}: item {item} declared twice")
        kind[item] = k
    dropped = 0
    for line_no, k, item, alb, art, gens in rows:
        if gens:
            genres[item] = gens
        if k == ItemKind.ARTIST:
            if alb >= 0 or art >= 0:
                raise ParseError(path, line_no, "artists cannot have parents")
            continue
        if k == ItemKind.ALBUM and alb >= 0:
            raise ParseError(path, line_no, "albums cannot have an album parent")
        for ref, want, slot in ((alb, ItemKind.ALBUM, album_of), (art, ItemKind.ARTIST, artist_link)):
            if ref < 0:
                continue
            if ref < n and kind[ref] == want:
                slot[item] = ref
            elif strict:
                raise DanglingReferenceError(
                    f"{path}:{line_no}: item {item} references undeclared "
                    f"{'album' if want == ItemKind.ALBUM else 'artist'} {ref}")
            else:
                dropped += 1
    for _, k, item, _, _, _ in rows:
        if k == ItemKind.TRACK and artist_link[item] < 0 and album_of[item] >= 0:
            artist_link[item] = artist_link[album_of[item]]
    return build_graph(kind, album_of, artist_link, genres, dropped)
