"""Host-side drop-in pieces against files written / read by the reference:
load_ratings, save_model byte layout, load_taxonomy, taxonomy maps."""
import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_load_ratings_matches_reference(golden):
    from paper_1108_2580_b200.data import load_ratings
    g = golden("formats.npz")
    ds = load_ratings(os.path.join(GOLDEN, "ratings_small.tsv"))
    for k in ("users", "items", "scores", "times"):
        assert np.array_equal(getattr(ds, k), g[k])


def test_load_ratings_errors(tmp_path):
    from paper_1108_2580_b200.data import load_ratings
    from paper_1108_2580_b200.errors import ParseError, RangeError
    p = tmp_path / "bad.tsv"
    p.write_text("1\t2\t3.0\n")
    with pytest.raises(ParseError):
        load_ratings(p)
    p.write_text("1\t2\t300.0\t5\n")
    with pytest.raises(RangeError):
        load_ratings(p)
    p.write_text("-1\t2\t3.0\t5\n")
    with pytest.raises(ParseError):
        load_ratings(p)


def test_model_format_round_trip_byte_identical(golden, tmp_path):
    from paper_1108_2580_b200 import modelio
    g = golden("formats.npz")
    ref = tmp_path / "ref.bin"
    ref.write_bytes(g["als_bytes"].tobytes())
    m = modelio.load_model(ref)
    assert m.kind == "als" and m.D == 3 and m.epochs_done == 3
    out = tmp_path / "ours.bin"
    modelio.save_model(m, out)
    assert out.read_bytes() == g["als_bytes"].tobytes()
    # MFITR model
    ref.write_bytes(g["mfitr_bytes"].tobytes())
    mm = modelio.load_model(ref)
    modelio.save_model(mm, out)
    assert out.read_bytes() == g["mfitr_bytes"].tobytes()
    # fp32 device factors widen to the same bytes
    m.p = m.p.astype(np.float32)
    m.q = m.q.astype(np.float32)
    ref.write_bytes(g["als_bytes"].tobytes())
    modelio.save_model(m, out)
    assert out.read_bytes() == g["als_bytes"].tobytes()


def test_load_taxonomy_matches_reference(golden):
    from paper_1108_2580_b200.taxonomy import load_taxonomy
    g = golden("taxonomy.npz")
    t = load_taxonomy(os.path.join(GOLDEN, "taxonomy_file.tax"))
    assert np.array_equal(t.kind, g["f_kind"])
    assert np.array_equal(t.album_of, g["f_album_of"])
    assert np.array_equal(t.artist_link, g["f_artist_link"])
    assert np.array_equal(t.edge_child, g["f_ec"]) and np.array_equal(t.edge_parent, g["f_ep"])
    assert np.array_equal(t.artist_array(t.num_nodes), g["f_art"])
    assert t.genres == {1: (7, 8), 4: (7,)}


def test_taxonomy_maps_vectorised_match_reference(golden):
    from paper_1108_2580_b200.taxonomy import build_graph_arrays
    g = golden("taxonomy.npz")
    for p in ("s", "g"):
        t = build_graph_arrays(g[f"{p}_kind"], g[f"{p}_album_of"], g[f"{p}_artist_link"])
        assert np.array_equal(t.edge_child, g[f"{p}_ec"])
        assert np.array_equal(t.edge_parent, g[f"{p}_ep"])
        assert np.array_equal(t.artist_array(g[f"{p}_art"].size), g[f"{p}_art"])
        t.validate()
        # layers partition the items and no edge stays inside a layer
        layers = t.layers(t.num_nodes)
        assert sum(L.size for L in layers) == t.num_nodes
        lid = np.empty(t.num_nodes, int)
        for k, L in enumerate(layers):
            lid[L] = k
        assert np.all(lid[t.edge_child] != lid[t.edge_parent])


def test_incident_edges_cover_each_edge_twice(golden):
    from paper_1108_2580_b200.taxonomy import build_graph_arrays
    g = golden("taxonomy.npz")
    t = build_graph_arrays(g["g_kind"], g["g_album_of"], g["g_artist_link"])
    ptr, eid, other = t.incident_edges(t.num_nodes)
    assert ptr[-1] == 2 * t.num_edges
    assert np.array_equal(np.bincount(eid, minlength=t.num_edges), np.full(t.num_edges, 2))
    for i in range(0, t.num_nodes, 37):
        for e, o in zip(eid[ptr[i]:ptr[i + 1]], other[ptr[i]:ptr[i + 1]]):
            assert {t.edge_child[e], t.edge_parent[e]} == {i, o}
