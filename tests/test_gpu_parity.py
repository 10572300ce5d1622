"""GPU parity: the sm_100a pipeline against the reference's golden outputs and
the (golden-pinned) CPU oracle, rung by rung (SURVEY §8(c) ladder).

Integer work: every comparison is bit-exact.  The GPU builds its own
spanning forest, so the stage-1..4 rungs use numbering-independent checks or
feed the GPU's own forest to the oracle; labels/heads/counts/articulation
flags/edge labels are compared to the reference outputs directly.
"""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, relaxed_w2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _run(g, debug=True):
    from paper_2301_01356_b200.bcc import run_device

    off = torch.from_numpy(g.offsets).cuda()
    adj = torch.from_numpy(g.edges.view(np.int32)).cuda()
    dbg = {} if debug else None
    res, stats = run_device(off, adj, debug=dbg)
    torch.cuda.synchronize()
    out = {k: (v.cpu().numpy() if v is not None else None) for k, v in res.items()}
    if debug:
        out["dbg"] = {k: v.cpu().numpy() for k, v in dbg.items()}
    out["num_bccs"] = int(stats.num_bccs)
    out["num_components"] = int(stats.num_components)
    out["num_edges"] = int(stats.num_edges)
    return out


def _check_forest(g, comp, forest2):
    """check_cc (test_connectivity.py:27-53): n-c edges, all in G, acyclic, spanning."""
    n = g.n
    hooked = np.flatnonzero(comp != np.arange(n))
    pairs = forest2.reshape(-1, 2)[hooked]
    ncomp = n - hooked.size
    parent = np.arange(n)

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for u, v in pairs:
        u, v = int(u), int(v)
        row = g.edges[g.offsets[u]:g.offsets[u + 1]]
        assert np.searchsorted(row, v) < row.size and row[np.searchsorted(row, v)] == v, "forest edge not in G"
        ru, rv = find(u), find(v)
        assert ru != rv, "forest has a cycle"
        parent[ru] = rv
    assert len({find(v) for v in range(n)}) == ncomp
    return pairs


def _check_rooting(n, comp, pairs, dbg, oracle, deg=None):
    # rung 2: parents are the unique rooting of the GPU forest at min-id roots
    parent_o, _, _ = oracle.root_forest(n, comp, pairs)
    assert np.array_equal(dbg["parent"][:n], parent_o)
    first, last = dbg["first"][:n], dbg["last"][:n]
    assert np.array_equal(np.sort(np.concatenate([first, last])), np.arange(2 * n))
    assert np.all(first < last)
    p = dbg["parent"][:n]
    nr = p >= 0
    assert np.all(first[p[nr]] < first[nr]) and np.all(last[nr] < last[p[nr]])
    roots = np.flatnonzero(~nr)
    listed = roots
    if deg is not None:
        from paper_2301_01356_b200 import _lib

        if _lib.get_option("detach"):
            # isolated roots (but vertex 0) are off the list: they follow it,
            # in id order (rooting.cu k_positions)
            off_list = (deg[roots] == 0) & (roots != 0)
            det, listed = roots[off_list], roots[~off_list]
            L = 2 * (n - len(det))
            assert np.array_equal(first[det], L + 2 * np.arange(len(det)))
            assert np.all(first[listed] < L)
    # trees are laid out in root-id order, root at both ends (euler_tour.py:12-17)
    assert np.all(np.diff(first[listed]) > 0)


def test_corpus_all_rungs(corpus, oracle_mod):
    for i, name, g in corpus.items():
        n = g.n
        r = _run(g)
        if n == 0:
            continue
        d = r["dbg"]
        # rung 1
        assert np.array_equal(r["comp"], corpus.get(i, "cc_label")), name
        pairs = _check_forest(g, r["comp"], d["forest"][:2 * n])
        _check_rooting(n, r["comp"], pairs, d, oracle_mod, np.diff(g.offsets))
        # rung 3/4: oracle tags on the GPU's own rooted forest
        w1, w2 = oracle_mod.compute_w(g.offsets, g.edges, d["parent"][:n], d["first"][:n])
        assert np.array_equal(d["w1"][:n], w1), name
        assert np.array_equal(d["w2"][:n], relaxed_w2(g.offsets, g.edges, d["parent"][:n], d["first"][:n])), name
        low, high = oracle_mod.low_high(d["first"][:n], d["last"][:n], w1, w2)
        assert all(np.array_equal(a, b) for a, b in
                   zip((low, high), oracle_mod.low_high(d["first"][:n], d["last"][:n], w1, d["w2"][:n]))), name
        assert np.array_equal(d["low"][:n], low), name
        assert np.array_equal(d["high"][:n], high), name
        skel = oracle_mod.pack_skeleton(d["parent"][:n], d["first"][:n], d["last"][:n], low, high)
        assert np.array_equal(d["fence"][:n], (skel[:, 1] & 1).astype(np.uint8)), name
        # rung 5/6: reference outputs
        assert np.array_equal(r["label"], corpus.get(i, "label")), name
        assert np.array_equal(r["head"], corpus.get(i, "head")), name
        assert r["num_bccs"] == corpus.get(i, "num_bccs"), name
        assert r["num_components"] == corpus.get(i, "num_components"), name
        assert np.array_equal(r["is_ap"], corpus.get(i, "is_ap")), name
        assert np.array_equal(r["edge_label"], corpus.get(i, "edge_label")), name


def test_public_api_known_answers():
    from paper_2301_01356_b200 import Graph, articulation_points, extract_bccs, fast_bcc

    lab = fast_bcc(Graph.from_edges(2, [(0, 1)]))
    assert lab.head_map() == {1: 0}
    i = np.arange(4)
    lab = fast_bcc(Graph.from_edges(5, np.column_stack([i, i + 1])))
    assert set(map(int, articulation_points(lab))) == {1, 2, 3}
    lab = fast_bcc(Graph.from_edges(5, [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (4, 2)]))
    assert lab.head_map() == {1: 0, 3: 2}
    assert [b.tolist() for b in extract_bccs(lab)] == [[0, 1, 2], [2, 3, 4]]
    g = Graph.from_edges(6, [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4), (4, 5), (5, 3)])
    lab = fast_bcc(g)
    assert lab.is_root(0) and not lab.is_root(3) and lab.head[3] == 2
    i = np.arange(4999)
    lab = fast_bcc(Graph.from_edges(5000, np.column_stack([i, i + 1])))
    assert lab.num_bccs == 4999 and lab.num_components == 1 and articulation_points(lab).size == 4998
    lab = fast_bcc(Graph.empty(0))
    assert lab.num_bccs == 0 and lab.n == 0 and extract_bccs(lab) == []
    lab = fast_bcc(Graph.empty(4))
    assert lab.num_bccs == 0 and lab.num_components == 4 and articulation_points(lab).size == 0


def test_knobs_do_not_change_output():
    from paper_2301_01356_b200 import fast_bcc
    import workloads

    g = workloads.grid(12, 12, keep_prob=0.85, seed=3)
    base = fast_bcc(g)
    for kw in ({"beta": 0.05}, {"beta": 0.9}, {"block": 2}, {"block": 4096}, {"seed": 99}):
        lab = fast_bcc(g, **kw)
        assert np.array_equal(lab.label, base.label) and np.array_equal(lab.head, base.head)
    with pytest.raises(ValueError):
        fast_bcc(g, block=1)
    with pytest.raises(ZeroDivisionError):
        fast_bcc(g, beta=0)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["1", "2", "3"])
def test_configs_match_reference(name, config_meta):
    import workloads

    g = workloads.make(name)
    meta = config_meta[name]
    assert workloads.csr_digest(g) == meta["csr_sha256"]
    r = _run(g, debug=False)
    assert r["num_bccs"] == meta["num_bccs"]
    assert r["num_components"] == meta["num_components"]
    assert r["num_edges"] == meta["E"]
    assert int(r["is_ap"].sum()) == meta["num_ap"]
    assert _sha(r["label"]) == meta["label_sha256"]
    assert _sha(r["head"]) == meta["head_sha256"]
    assert _sha(r["is_ap"]) == meta["is_ap_sha256"]
    assert _sha(r["edge_label"]) == meta["edge_label_sha256"]
    if name == "1":
        z = np.load(GOLDEN / "config1.npz")
        for k in ("label", "head", "is_ap", "edge_label"):
            assert np.array_equal(r[k], z[k]), k


def test_repeat_runs_identical():
    """Atomics make the forest and tour numbering run-dependent; the outputs
    must not be (worker-invariance analogue, test_acceptance.py:175-194)."""
    import workloads

    g = workloads.make("1")
    a = _run(g, debug=False)
    for _ in range(3):
        b = _run(g, debug=False)
        for k in ("label", "head", "is_ap", "edge_label"):
            assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", ["1", "2", "3"])
def test_public_api_paths_match_reference(name, config_meta):
    """fast_bcc on a pageable host graph, a pinned one (fbcc_run_host: streamed
    upload, Stage 1 linked per arrived range, for several range counts), a
    device-resident one and with device outputs: all equal the reference's
    digests."""
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, _lib, fast_bcc

    g = workloads.make(name)
    meta = config_meta[name]

    def check(lab):
        host = {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v))
                for k, v in (("label", lab.label), ("head", lab.head), ("edge_label", lab.edge_label),
                             ("is_ap", lab.is_ap))}
        assert lab.num_bccs == meta["num_bccs"]
        assert lab.num_components == meta["num_components"]
        assert host["edge_label"].size == meta["E"]
        assert _sha(host["label"]) == meta["label_sha256"]
        assert _sha(host["head"]) == meta["head_sha256"]
        assert _sha(host["edge_label"]) == meta["edge_label_sha256"]
        assert _sha(host["is_ap"].astype(np.uint8)) == meta["is_ap_sha256"]

    check(fast_bcc(g))  # pageable
    gp = Graph(g.offsets, g.edges).pin()
    old = _lib.get_option("stream_chunks")
    try:
        for chunks in (1, 3, 8, 64):
            _lib.set_option("stream_chunks", chunks)
            check(fast_bcc(gp))
    finally:
        _lib.set_option("stream_chunks", old)
    check(fast_bcc(gp, device_outputs=True))
    gd = Graph.from_device(torch.from_numpy(g.offsets).cuda(), torch.from_numpy(g.edges.view(np.int32)).cuda())
    check(fast_bcc(gd))
    check(fast_bcc(gd, device_outputs=True))


def test_host_offsets_widths_agree():
    """fbcc_run_host with the int32 offsets Graph.pin() keeps
    (FBCC_FLAG_HOST_OFFSETS32, widened on the device) and with the int64
    reference offsets give identical outputs."""
    import workloads
    from paper_2301_01356_b200 import Graph, fast_bcc

    for name in ("1", "3"):
        g = workloads.make(name)
        gp = Graph(g.offsets, g.edges).pin()
        assert gp._pinned_off32 is not None
        a = fast_bcc(gp)
        gp._pinned_off32 = None  # int64 upload
        b = fast_bcc(gp)
        for k in ("label", "head", "edge_label", "is_ap"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (name, k)
        assert a.num_bccs == b.num_bccs and a.num_components == b.num_components
