"""Pin the CPU oracle against the reference's own outputs (golden vectors).

Each stage of oracle/fastbcc_oracle.c is checked on the 1,077-graph reference
corpus against what the reference computed on the same input (and, for the
stage functions, on the reference's own forest), plus the reference's
known-answer tests.  Only once this file is green is the oracle trusted as
the checker for the GPU kernels.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN


def test_cc_labels_match_reference(corpus, oracle_mod):
    # connectivity.py:593-611 labels are canonical (min id), forest-independent
    for i, name, g in corpus.items():
        label, forest, ncomp = oracle_mod.connected_components(g.offsets, g.edges)
        assert np.array_equal(label, corpus.get(i, "cc_label")), name
        assert ncomp == corpus.get(i, "num_components"), name
        assert forest.shape[0] == g.n - ncomp, name


def test_rooting_on_reference_forest(corpus, oracle_mod):
    # build_euler_tour(n, ref forest, labels): euler_tour.py:361-394.  Same
    # pairs in the same order give the same tree CSR, so positions are exact.
    for i, name, g in corpus.items():
        parent, first, last = oracle_mod.root_forest(g.n, corpus.get(i, "cc_label"),
                                                     corpus.get(i, "forest"))
        assert np.array_equal(parent, corpus.get(i, "parent")), name
        assert np.array_equal(first, corpus.get(i, "first")), name
        assert np.array_equal(last, corpus.get(i, "last")), name


def test_tags_and_fence_on_reference_forest(corpus, oracle_mod):
    # compute_tags tagging.py:300-304; skeleton_record connectivity.py:471-480
    for i, name, g in corpus.items():
        parent, first, last = (corpus.get(i, k) for k in ("parent", "first", "last"))
        w1, w2 = oracle_mod.compute_w(g.offsets, g.edges, parent, first)
        assert np.array_equal(w1, corpus.get(i, "w1")), name
        assert np.array_equal(w2, corpus.get(i, "w2")), name
        for block in (2, 16, 1000):
            low, high = oracle_mod.low_high(first, last, w1, w2, block)
            assert np.array_equal(low, corpus.get(i, "low")), (name, block)
            assert np.array_equal(high, corpus.get(i, "high")), (name, block)
        skel = oracle_mod.pack_skeleton(parent, first, last, low, high)
        assert np.array_equal((skel[:, 1] & 1).astype(np.uint8), corpus.get(i, "fence")), name


@pytest.mark.parametrize("parallel", [False, True])
def test_fast_bcc_matches_reference(corpus, oracle_mod, parallel):
    """Both oracle modes: sequential (the checker) and parallel (the CPU
    baseline: concurrent union-find, splitter list ranking)."""
    for i, name, g in corpus.items():
        r = oracle_mod.fast_bcc(g.offsets, g.edges, parallel=parallel)
        assert np.array_equal(r["label"], corpus.get(i, "label")), name
        assert np.array_equal(r["head"], corpus.get(i, "head")), name
        assert r["num_bccs"] == corpus.get(i, "num_bccs") == corpus.get(i, "ht_num_bccs"), name
        assert r["num_components"] == corpus.get(i, "num_components"), name
        assert np.array_equal(r["is_ap"], corpus.get(i, "is_ap")), name
        assert np.array_equal(r["edge_label"], corpus.get(i, "edge_label")), name


def test_list_ranking_golden(oracle_mod):
    z = np.load(GOLDEN / "listrank.npz", allow_pickle=True)
    lo = ho = 0
    for L, H in zip(z["L"], z["H"]):
        nxt = z["nxt"][lo:lo + L]
        heads = z["heads"][ho:ho + H]
        assert np.array_equal(oracle_mod.list_ranking(nxt, heads), z["ranks"][lo:lo + L])
        lo += L
        ho += H
    for nxt, heads in zip(z["bad_nxt"], z["bad_heads"]):
        with pytest.raises(ValueError):
            oracle_mod.list_ranking(nxt, heads)


def test_known_answers(oracle_mod):
    from paper_2301_01356_b200.graphs import Graph

    # chain(3): test_euler_tour.py:51-56
    g = Graph.from_edges(3, [(0, 1), (1, 2)])
    lab, forest, _ = oracle_mod.connected_components(g.offsets, g.edges)
    p, f, l = oracle_mod.root_forest(3, lab, forest)
    assert p.tolist() == [-1, 0, 1] and f.tolist() == [0, 1, 2] and l.tolist() == [5, 4, 3]
    # C4 on the explicit chain tree 0-1-2-3: test_tagging.py:52-63
    g = Graph.from_edges(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    p, f, l = oracle_mod.root_forest(4, np.zeros(4, np.int32), [(0, 1), (1, 2), (2, 3)])
    assert f.tolist() == [0, 1, 2, 3] and l.tolist() == [7, 6, 5, 4]
    w1, w2 = oracle_mod.compute_w(g.offsets, g.edges, p, f)
    assert w1.tolist() == [0, 1, 2, 0] and w2.tolist() == [3, 1, 2, 3]
    low, high = oracle_mod.low_high(f, l, w1, w2)
    assert low.tolist() == [0, 0, 0, 0] and high.tolist() == [3, 3, 3, 3]
    with pytest.raises(ValueError):
        oracle_mod.low_high(f, l, w1, w2, block=1)
    # single list: test_euler_tour.py:110-114 ; long chain :167-172
    assert oracle_mod.list_ranking([1, 2, 3, -1], [0]).tolist() == [0, 1, 2, 3]
    nxt = np.arange(1, 100_001, dtype=np.int32)
    nxt[-1] = -1
    assert np.array_equal(oracle_mod.list_ranking(nxt, [0]), np.arange(100_000))
    # bowtie heads {1:0, 3:2}, APs {2}: test_bcc.py:109-112
    g = Graph.from_edges(5, [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (4, 2)])
    r = oracle_mod.fast_bcc(g.offsets, g.edges)
    assert {int(l): int(r["head"][l]) for l in np.flatnonzero(r["head"] != -1)} == {1: 0, 3: 2}
    assert np.flatnonzero(r["is_ap"]).tolist() == [2]
    # chain(5000): 4,999 BCCs, 4,998 APs (test_bcc.py:124-128)
    i = np.arange(4999)
    g = Graph.from_edges(5000, np.column_stack([i, i + 1]))
    r = oracle_mod.fast_bcc(g.offsets, g.edges)
    assert r["num_bccs"] == 4999 and r["num_components"] == 1 and r["is_ap"].sum() == 4998
    # empty and isolated (test_bcc.py:161-168)
    r = oracle_mod.fast_bcc(np.zeros(5, np.int64), np.empty(0, np.uint32))
    assert r["num_bccs"] == 0 and r["num_components"] == 4 and r["is_ap"].sum() == 0


def test_config1_golden(oracle_mod, config_meta):
    import workloads

    g = workloads.make("1")
    meta = config_meta["1"]
    assert workloads.csr_digest(g) == meta["csr_sha256"]
    r = oracle_mod.fast_bcc(g.offsets, g.edges)
    z = np.load(GOLDEN / "config1.npz")
    for k in ("label", "head", "is_ap", "edge_label"):
        assert np.array_equal(r[k], z[k]), k
    assert r["num_bccs"] == meta["num_bccs"] == 21104
    assert r["num_components"] == meta["num_components"] == 3002
    assert int(r["is_ap"].sum()) == meta["num_ap"] == 18561


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name,parallel", [("2", False), ("3", False), ("1", True), ("2", True), ("3", True)])
def test_config_digests(oracle_mod, config_meta, name, parallel):
    """Configs 1-3 at full size: the oracle reproduces the reference's
    outputs bit for bit (sha256 of label/head/is_ap/edge_label), in both
    modes."""
    import workloads

    g = workloads.make(name)
    meta = config_meta[name]
    assert workloads.csr_digest(g) == meta["csr_sha256"]
    r = oracle_mod.fast_bcc(g.offsets, g.edges, parallel=parallel)
    assert r["num_bccs"] == meta["num_bccs"]
    assert r["num_components"] == meta["num_components"]
    assert _sha(r["label"]) == meta["label_sha256"]
    assert _sha(r["head"]) == meta["head_sha256"]
    assert _sha(r["is_ap"]) == meta["is_ap_sha256"]
    assert _sha(r["edge_label"]) == meta["edge_label_sha256"]


def _classes_from_definition(g, parent, first, last, low, high):
    """classify_edge (bcc.py:54-70) restated in numpy, per slot -- the CPU
    check of the classification fixtures (the product op runs on the GPU)."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets))
    dst = g.edges.astype(np.int64)
    tree_down = parent[dst] == src
    tree_up = parent[src] == dst
    child = np.where(tree_down, dst, src)
    pc = np.where(tree_down, src, dst)
    fence = (low[child] >= first[pc]) & (high[child] <= last[pc])
    anc = ((first[src] <= first[dst]) & (last[dst] <= last[src])) | ((first[dst] <= first[src]) & (last[src] <= last[dst]))
    out = np.where(anc, 2, 3).astype(np.int8)
    tree = tree_down | tree_up
    out[tree] = np.where(fence[tree], 1, 0)
    return src, dst, out


def test_classify_fixtures_consistent(corpus):
    """tests/golden/classify.npz holds the reference's classify_edge on its
    own forest (cross-checked there against classify_edges_oracle): the
    definition restated here agrees on every edge of the corpus."""
    z = np.load(GOLDEN / "classify.npz")
    eo = np.concatenate([[0], np.cumsum(z["E"])])
    for i, name, g in corpus.items():
        if g.m == 0:
            continue
        arrs = [corpus.get(i, k).astype(np.int64) for k in ("parent", "first", "last", "low", "high")]
        src, dst, cls = _classes_from_definition(g, *arrs)
        assert np.array_equal(cls[src < dst], z["cls"][eo[i]:eo[i + 1]]), name
