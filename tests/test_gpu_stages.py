"""GPU parity of the stand-alone stage operations against the
reference's own outputs on its test corpus (golden vectors) and its
known-answer / error-case tests."""

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2301_01356_b200 import stages  # noqa: E402
from paper_2301_01356_b200.bcc import BccLabeling, StepTimings, extract_bccs  # noqa: E402
from paper_2301_01356_b200.graphs import Graph, symmetrize  # noqa: E402


def test_connected_components_corpus(corpus, oracle_mod):
    from test_gpu_parity import _check_forest

    for i, name, g in corpus.items():
        res = stages.connected_components(g)
        assert np.array_equal(res.labels, corpus.get(i, "cc_label")), name
        assert res.num_components == corpus.get(i, "num_components"), name
        assert res.forest_edges.pairs.shape[0] == g.n - res.num_components, name
        if g.n:
            fe = np.zeros((g.n, 2), np.int32)
            hooked = np.flatnonzero(res.labels != np.arange(g.n))
            fe[hooked] = res.forest_edges.pairs
            _check_forest(g, res.labels, fe.reshape(-1))


def test_connected_components_predicate(corpus, oracle_mod):
    # test_connectivity.py:112-120: parity predicate, and a per-slot mask
    keep = lambda u, v: (u + v) % 2 == 0  # noqa: E731
    for i, name, g in list(corpus.items())[:200]:
        res = stages.connected_components(g, keep)
        pairs = g.edge_pairs()
        mask = np.array([keep(int(u), int(v)) for u, v in pairs], np.uint8)
        lab, _, nc = oracle_mod.connected_components(g.offsets, g.edges, keep_mask=mask)
        assert np.array_equal(res.labels, lab), name
        assert res.num_components == nc, name
        for u, v in res.forest_edges.pairs:
            assert keep(int(u), int(v)), name
    g = Graph.from_edges(25, [(i, i + 1) for i in range(24)])
    res = stages.connected_components(g, lambda u, v: False)
    assert res.num_components == 25


def test_list_ranking_golden_and_errors():
    z = np.load(GOLDEN / "listrank.npz", allow_pickle=True)
    lo = ho = 0
    for L, H in zip(z["L"], z["H"]):
        got = stages.list_ranking(z["nxt"][lo:lo + L], z["heads"][ho:ho + H])
        assert np.array_equal(got, z["ranks"][lo:lo + L])
        lo += L
        ho += H
    for nxt, heads in zip(z["bad_nxt"], z["bad_heads"]):
        with pytest.raises(ValueError):
            stages.list_ranking(nxt, heads)
    # test_euler_tour.py:110-172
    assert stages.list_ranking(np.array([1, 2, 3, -1]), np.array([0])).tolist() == [0, 1, 2, 3]
    assert stages.list_ranking(np.array([1, -1]), np.array([-1, 0])).tolist() == [0, 1]
    assert stages.list_ranking(np.array([], np.int32), np.array([], np.int32)).size == 0
    nxt = np.arange(1, 100_001, dtype=np.int32)
    nxt[-1] = -1
    assert np.array_equal(stages.list_ranking(nxt, np.array([0])), np.arange(100_000))


def test_build_euler_tour_matches_reference_exactly(corpus):
    for i, name, g in corpus.items():
        f = stages.build_euler_tour(g.n, corpus.get(i, "forest"), corpus.get(i, "cc_label"))
        assert np.array_equal(f.parent, corpus.get(i, "parent")), name
        assert np.array_equal(f.first, corpus.get(i, "first")), name
        assert np.array_equal(f.last, corpus.get(i, "last")), name
        f2 = stages.build_euler_tour(g.n, corpus.get(i, "forest"))  # labels derived (test_euler_tour.py:70-78)
        assert np.array_equal(f2.first, f.first) and np.array_equal(f2.last, f.last), name


def test_build_euler_tour_known_answers_and_errors():
    f = stages.build_euler_tour(3, [(0, 1), (1, 2)])
    assert f.parent.tolist() == [-1, 0, 1] and f.first.tolist() == [0, 1, 2] and f.last.tolist() == [5, 4, 3]
    f = stages.build_euler_tour(4, [(0, 1), (1, 2), (2, 3)])
    assert f.first.tolist() == [0, 1, 2, 3] and f.last.tolist() == [7, 6, 5, 4]
    f = stages.build_euler_tour(1, [])
    assert f.first[0] == 0 and f.last[0] == 1
    with pytest.raises(ValueError, match="forest"):
        stages.build_euler_tour(3, [(0, 1), (1, 2), (2, 0)])
    with pytest.raises(ValueError, match="range"):
        stages.build_euler_tour(3, [(0, 5)])
    with pytest.raises(ValueError, match="labels"):
        stages.build_euler_tour(3, [], labels=np.array([0, 0, 0], np.int32))
    assert stages.build_euler_tour(0, []).n == 0


def test_compute_tags_on_reference_forest(corpus):
    for i, name, g in corpus.items():
        forest = stages.RootedForest(corpus.get(i, "parent"), corpus.get(i, "first"), corpus.get(i, "last"),
                                     np.flatnonzero(corpus.get(i, "parent") == -1))
        t = stages.compute_tags(g, forest)
        for k in ("w1", "w2", "low", "high"):
            assert np.array_equal(getattr(t, k), corpus.get(i, k)), (name, k)
        sk = stages.skeleton_record(forest.parent, forest.first, forest.last, t.low, t.high)
        assert np.array_equal((sk[:, 1] & 1).astype(np.uint8), corpus.get(i, "fence")), name
    g = Graph.from_edges(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    f = stages.build_euler_tour(4, [(0, 1), (1, 2), (2, 3)])
    t = stages.compute_tags(g, f)  # test_tagging.py:52-63
    assert t.w1.tolist() == [0, 1, 2, 0] and t.w2.tolist() == [3, 1, 2, 3]
    assert t.low.tolist() == [0, 0, 0, 0] and t.high.tolist() == [3, 3, 3, 3]
    with pytest.raises(ValueError):
        stages.compute_tags(g, f, block=1)
    cls = stages.classify_edges(g, f, t)  # test_bcc.py:48-59: (0,1) fence, (1,2)/(2,3) plain, (3,0) back
    src = np.repeat(np.arange(4), np.diff(g.offsets))
    got = {(int(u), int(v)): int(c) for u, v, c in zip(src, g.edges, cls) if u < v}
    assert got == {(0, 1): 1, (1, 2): 0, (2, 3): 0, (0, 3): 2}


def test_extract_bccs_device_matches_reference(corpus):
    """fbcc_extract_bccs == the reference's extract_bccs (bcc.py:199-219) on
    every corpus labeling (tests/golden/extract.npz, produced by running the
    reference) -- and the host mirror agrees too."""
    z = np.load(GOLDEN / "extract.npz")
    bo = np.concatenate([[0], np.cumsum(z["nblocks"])])
    vo = np.concatenate([[0], np.cumsum(z["blen"])])
    for i, name, g in corpus.items():
        lab = BccLabeling(corpus.get(i, "label"), corpus.get(i, "head"), corpus.get(i, "num_bccs"),
                          corpus.get(i, "num_components"), StepTimings())
        want = [z["verts"][vo[b]:vo[b + 1]] for b in range(bo[i], bo[i + 1])]
        got = stages.extract_bccs_device(lab.label, lab.head)
        host = extract_bccs(lab)
        assert len(got) == len(want) == len(host) == corpus.get(i, "num_bccs"), name
        for a, b, c in zip(got, want, host):
            assert np.array_equal(a, b) and np.array_equal(c, b), name


def test_symmetrize_device(corpus):
    for i, name, g in corpus.items():
        d = stages.symmetrize_device(g.edge_pairs(), g.n)
        off, e = d._dev
        assert np.array_equal(off.cpu().numpy(), g.offsets), name
        assert np.array_equal(e.cpu().numpy().view(np.uint32), g.edges), name
    d = stages.symmetrize_device([(0, 1), (1, 0), (2, 2), (1, 3), (0, 1)], 4)
    assert d._dev[0].cpu().tolist() == [0, 1, 3, 3, 4]
    assert d._dev[1].cpu().tolist() == [1, 0, 3, 1]
    with pytest.raises(ValueError):
        stages.symmetrize_device([(0, 5)], 4)
    rng = np.random.Generator(np.random.PCG64(7))
    pairs = rng.integers(0, 5000, size=(40000, 2))
    h = symmetrize(pairs, 5000)
    d = stages.symmetrize_device(pairs, 5000)
    assert np.array_equal(d._dev[0].cpu().numpy(), h.offsets)
    assert np.array_equal(d._dev[1].cpu().numpy().view(np.uint32), h.edges)


def test_fast_bcc_on_device_graph():
    """The drop-in entry point accepts a device-symmetrized graph directly."""
    from paper_2301_01356_b200 import fast_bcc

    rng = np.random.Generator(np.random.PCG64(3))
    pairs = rng.integers(0, 3000, size=(4000, 2))
    dg = stages.symmetrize_device(pairs, 3000)
    hg = symmetrize(pairs, 3000)
    a = fast_bcc(dg)
    b = fast_bcc(hg)
    assert np.array_equal(a.label, b.label) and np.array_equal(a.head, b.head)
    assert np.array_equal(a.edge_label, b.edge_label) and a.num_bccs == b.num_bccs


def test_rmat_device_generator_matches_numpy():
    """The GPU RMAT generator (bench/test input only) reproduces the numpy
    PCG64 stream bit for bit, across chunk boundaries."""
    import workloads

    u0, v0 = workloads._rmat_pairs(scale=12, edge_factor=16, seed=0, chunk=5000)
    u1, v1 = workloads.rmat_pairs_device(scale=12, edge_factor=16, seed=0, chunk=5000)
    assert np.array_equal(u0, u1.cpu().numpy())
    assert np.array_equal(v0, v1.cpu().numpy())


def test_classify_edges_device_matches_reference(corpus):
    """fbcc_classify_edges == the reference's classify_edge (bcc.py:54-70) on
    every edge of the corpus, for the reference's forest and tags
    (tests/golden/classify.npz, made by tests/golden/make_golden.py); both
    slots of an edge get the same class."""
    z = np.load(GOLDEN / "classify.npz")
    eo = np.concatenate([[0], np.cumsum(z["E"])])
    for i, name, g in corpus.items():
        forest = stages.RootedForest(corpus.get(i, "parent"), corpus.get(i, "first"), corpus.get(i, "last"),
                                     np.flatnonzero(corpus.get(i, "parent") == -1))
        tags = stages.VertexTags(*(corpus.get(i, k) for k in ("w1", "w2", "low", "high")))
        cls = stages.classify_edges(g, forest, tags)
        assert cls.shape == (g.m,), name
        src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets))
        dst = g.edges.astype(np.int64)
        up = src < dst
        assert np.array_equal(cls[up], z["cls"][eo[i]:eo[i + 1]]), name
        # the reverse slot of every edge: same class
        key_up = src[up] * (g.n + 1) + dst[up]
        key_dn = dst[~up] * (g.n + 1) + src[~up]
        order = np.argsort(key_up)
        pos = order[np.searchsorted(key_up[order], key_dn)]
        assert np.array_equal(cls[~up], cls[up][pos]), name


def test_load_bin_to_device_roundtrip(tmp_path, config_meta):
    """load_bin(path, device=...) (graphs.py:173-204): the .bin lands in
    pinned staging buffers and goes straight to HBM; fast_bcc on the device
    graph reproduces the reference's config-1 outputs."""
    import hashlib

    import torch

    import workloads
    from paper_2301_01356_b200 import fast_bcc
    from paper_2301_01356_b200.graphs import load_bin, write_bin

    g = workloads.make("1")
    path = tmp_path / "config1.bin"
    write_bin(g, path)
    d = load_bin(path, device="cuda")
    off, adj = d._dev
    assert off.is_cuda and adj.is_cuda and off.dtype == torch.int64
    assert np.array_equal(off.cpu().numpy(), g.offsets)
    assert np.array_equal(adj.cpu().numpy().view(np.uint32), g.edges)
    lab = fast_bcc(d)
    meta = config_meta["1"]
    assert lab.num_bccs == meta["num_bccs"] and lab.num_components == meta["num_components"]
    assert hashlib.sha256(np.ascontiguousarray(lab.edge_label).tobytes()).hexdigest() == meta["edge_label_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(lab.label).tobytes()).hexdigest() == meta["label_sha256"]
