"""GPU parity on mid-size graphs that exercise what the 64-vertex corpus
cannot: several 4096-position tiles, multi-level list ranking, rows split
across thread chunks, hubs, long paths, many isolated vertices.  Each graph
is checked rung by rung against the (golden-pinned) oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import workloads  # noqa: E402
from paper_2301_01356_b200.graphs import symmetrize  # noqa: E402
from conftest import relaxed_w2  # noqa: E402
from test_gpu_parity import _check_forest, _check_rooting, _run  # noqa: E402


def _star(k):
    i = np.arange(1, k + 1)
    return symmetrize(np.column_stack([np.zeros(k, np.int64), i]), k + 1)


def _star_at(n, c):
    i = np.setdiff1d(np.arange(n), [c])
    return symmetrize(np.column_stack([np.full(i.size, c), i]), n)


def _wheel_at(n, c):
    i = np.setdiff1d(np.arange(n), [c])
    rim = np.column_stack([i, np.roll(i, -1)])
    return symmetrize(np.concatenate([np.column_stack([np.full(i.size, c), i]), rim]), n)


def _with_isolated(g, extra):
    p = g.edge_pairs()
    p = p[p[:, 0] < p[:, 1]]
    # spread the old ids over a bigger id space so isolated vertices interleave
    return symmetrize(p * 3 + 1, g.n * 3 + extra)


GRAPHS = {
    "chain_10k": lambda: workloads.chain(10_000),
    "chain_300k": lambda: workloads.chain(300_000),
    "cycle_50k": lambda: symmetrize(np.column_stack([np.arange(50_000), (np.arange(50_000) + 1) % 50_000]), 50_000),
    "star_100k": lambda: _star(100_000),
    # hubs that are not the tree root (rooting's split out-lists, kHubDeg)
    "star_mid_20k": lambda: _star_at(20_000, 7_777),
    "wheel_mid_30k": lambda: _wheel_at(30_000, 12_345),
    "grid_300": lambda: workloads.grid(300, 300),
    "torus_200_p07": lambda: workloads.grid(200, 200, circular=True, keep_prob=0.7, seed=5),
    "uniform_64k_d3": lambda: workloads.uniform(1 << 16, 3, seed=1),
    "uniform_64k_d1": lambda: workloads.uniform(1 << 16, 1, seed=2),
    "rmat_s16": lambda: workloads.rmat(16, 8, seed=3),
    "isolated_mix": lambda: _with_isolated(workloads.grid(100, 100, keep_prob=0.8, seed=1), 5),
}


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_mid_graph_rungs(name, oracle_mod):
    g = GRAPHS[name]()
    n = g.n
    r = _run(g)
    d = r["dbg"]
    ref = oracle_mod.fast_bcc(g.offsets, g.edges)
    lab1, _, ncomp = oracle_mod.connected_components(g.offsets, g.edges)
    assert np.array_equal(r["comp"], lab1), "rung 1: component labels"
    pairs = _check_forest(g, r["comp"], d["forest"][:2 * n])
    _check_rooting(n, r["comp"], pairs, d, oracle_mod, np.diff(g.offsets))
    p, f, l = d["parent"][:n], d["first"][:n], d["last"][:n]
    w1, w2 = oracle_mod.compute_w(g.offsets, g.edges, p, f)
    assert np.array_equal(d["w1"][:n], w1), "rung 3: w1"
    assert np.array_equal(d["w2"][:n], relaxed_w2(g.offsets, g.edges, p, f)), "rung 3: w2 (relaxed)"
    low, high = oracle_mod.low_high(f, l, w1, w2)
    bad = np.flatnonzero(d["low"][:n] != low)
    assert bad.size == 0, f"rung 3: low differs at {bad[:5]} first={f[bad[:5]]} last={l[bad[:5]]}"
    assert np.array_equal(d["high"][:n], high), "rung 3: high"
    skel = oracle_mod.pack_skeleton(p, f, l, low, high)
    assert np.array_equal(d["fence"][:n], (skel[:, 1] & 1).astype(np.uint8)), "rung 4: fence"
    # rung 5: the skeleton CC on the GPU's own forest equals the oracle's
    lab5, _, _ = oracle_mod.connected_components(g.offsets, g.edges, skel=skel)
    assert np.array_equal(r["label"], lab5), "rung 5: skeleton labels (own forest)"
    assert np.array_equal(r["label"], ref["label"]), "rung 5: labels vs oracle"
    assert np.array_equal(r["head"], ref["head"]), "rung 6: head"
    assert r["num_bccs"] == ref["num_bccs"]
    assert r["num_components"] == ref["num_components"] == ncomp
    assert np.array_equal(r["is_ap"], ref["is_ap"]), "rung 6: is_ap"
    assert np.array_equal(r["edge_label"], ref["edge_label"]), "rung 6: edge labels"


# Alternative kernel paths and tunables: every one must give the reference's
# outputs (the edge-block pass without the bitmap is what graphs with
# n > 1.6M run; max_rounds runs the adaptive sampling rounds and their skips)
OPTION_VARIANTS = [{"eb_staged": 0}, {"max_rounds": 6}, {"max_rounds": 8, "sample_rounds": 2}, {"pdl": 0},
                   {"sample_rounds": 1}, {"giant_skip": 0}, {"s0": 8, "sl": 4}, {"accept_fold": 1},
                   {"accept_fold": 1, "max_rounds": 5}, {"skel_parent": 131}, {"skel_max_rounds": 4},
                   {"compress_mask": 0}, {"detach": 0}, {"detach": 0, "s0": 8, "sl": 4},
                   # Stage 3 from the rows' first three arcs (forced: the meshes overflow the repair list and
                   # fall back to the full gather inside the same plan) and without it
                   {"witness": 2}, {"witness": 0}, {"witness": 2, "detach": 0}]


@pytest.mark.parametrize("name", ["rmat_s16", "isolated_mix", "star_mid_20k", "uniform_64k_d3", "chain_300k",
                                  "torus_200_p07"])
def test_mid_graph_option_paths(name, oracle_mod):
    from paper_2301_01356_b200 import _lib

    g = GRAPHS[name]()
    ref = oracle_mod.fast_bcc(g.offsets, g.edges)
    defaults = {k: _lib.get_option(k) for k in _lib.OPTIONS}
    try:
        for var in OPTION_VARIANTS:
            for k, v in var.items():
                _lib.set_option(k, v)
            r = _run(g, debug=False)
            for k in ("label", "head", "is_ap", "edge_label"):
                assert np.array_equal(r[k], ref[k]), (name, var, k)
            assert r["num_bccs"] == ref["num_bccs"] and r["num_components"] == ref["num_components"], (name, var)
            for k in var:
                _lib.set_option(k, defaults[k])
    finally:
        for k, v in defaults.items():
            _lib.set_option(k, v)


# Graphs past the edge pass's shared-memory bitmap (n > 1.6M vertices): the
# global-bitmap path (a giant holding >= 1/4 of Stage 5's samples) and the
# label-gather path (small giant), plus the largest graph the shared-memory
# path takes.
BIG = {
    "uniform_1p55m_d4": lambda: workloads.uniform(1_550_000, 4, seed=7),   # shared-memory bitmap, near its limit
    "uniform_1p8m_d4": lambda: workloads.uniform(1_800_000, 4, seed=8),    # global bitmap (giant ~all)
    "uniform_1p8m_d1": lambda: workloads.uniform(1_800_000, 1, seed=9),    # label gathers (no giant)
    # n >= 2^22 with >= 3/4 of the vertices hooked to a near id in round 0: the id-ordered compress
    # (k_jump_local / k_jump_list) -- a path, a torus (row chains + the column-0 chain), and paths of 4
    # whose heads hang off far, random heads (more exit targets than the list holds: the fallback)
    "chain_4p3m": lambda: workloads.chain(4_300_000),
    "torus_2100": lambda: workloads.grid(2100, 2100, circular=True),
    "paths4_far_heads_4p2m": lambda: _paths4_far_heads(1 << 20),
}


def _paths4_far_heads(k):
    rng = np.random.default_rng(11)
    i = np.arange(k, dtype=np.int64)
    inner = np.concatenate([np.column_stack([4 * i + j, 4 * i + j + 1]) for j in range(3)])
    parent = (rng.random(k - 1) * np.arange(1, k)).astype(np.int64)  # head c hangs off head parent[c - 1] < c
    heads = np.column_stack([4 * np.arange(1, k, dtype=np.int64), 4 * parent])
    return symmetrize(np.concatenate([inner, heads]), 4 * k)


@pytest.mark.parametrize("name", sorted(BIG))
def test_big_graph_edge_paths(name, oracle_mod):
    g = BIG[name]()
    ref = oracle_mod.fast_bcc(g.offsets, g.edges)
    r = _run(g, debug=False)
    for k in ("label", "head", "is_ap", "edge_label"):
        assert np.array_equal(r[k], ref[k]), (name, k)
    assert r["num_bccs"] == ref["num_bccs"] and r["num_components"] == ref["num_components"]


def _random_graph(seed):
    """Seeded mix: uniform random (sparse to dense), tori with deletions,
    paths with chords, and stars glued to them -- the shapes whose union-find
    and tour structure the round-0 rule, the adaptive rounds and the
    block-local compress treat differently."""
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 0:
        n = int(rng.integers(2, 4000))
        pairs = rng.integers(0, n, size=(int(n * rng.uniform(0.3, 6.0)), 2))
    elif kind == 1:
        r, c = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        return workloads.grid(r, c, circular=bool(rng.integers(0, 2)), keep_prob=float(rng.uniform(0.4, 1.0)),
                              seed=int(seed))
    elif kind == 2:
        n = int(rng.integers(3, 5000))
        i = np.arange(n - 1)
        chords = rng.integers(0, n, size=(int(rng.integers(0, n // 3 + 1)), 2))
        pairs = np.concatenate([np.column_stack([i, i + 1]), chords])
    else:
        n = int(rng.integers(10, 3000))
        hub = int(rng.integers(0, n))
        spokes = rng.choice(n, size=int(rng.integers(1, n)), replace=False)
        extra = rng.integers(0, n, size=(int(rng.integers(0, 2 * n)), 2))
        pairs = np.concatenate([np.column_stack([np.full(spokes.size, hub), spokes]), extra])
    return symmetrize(pairs.astype(np.int64), n)


@pytest.mark.parametrize("block", range(4))
def test_random_graphs_match_oracle(block, oracle_mod):
    """200 seeded random graphs (50 per parametrisation), full outputs vs the
    golden-pinned oracle."""
    for seed in range(block * 50, block * 50 + 50):
        g = _random_graph(seed)
        ref = oracle_mod.fast_bcc(g.offsets, g.edges)
        r = _run(g, debug=False)
        for k in ("label", "head", "is_ap", "edge_label"):
            assert np.array_equal(r[k], ref[k]), (seed, k)
        assert r["num_bccs"] == ref["num_bccs"] and r["num_components"] == ref["num_components"], seed


def _core_with_blobs(seed):
    """A dense random core with dense blobs hanging off single cut vertices: the
    blob's top tree edge is a fence whose subtree holds rows of more than three
    arcs (one of them a hub over 64), so the sampled tags leave it open and
    k_witness_fix has to rescan a few hundred rows."""
    rng = np.random.default_rng(seed)
    nc = 4096
    pairs = [rng.integers(0, nc, size=(nc * 8, 2))]
    n = nc
    for b in range(6):
        size = int(rng.integers(40, 700))
        ids = np.arange(n, n + size)
        hub = ids[int(rng.integers(0, size))]
        pairs.append(np.column_stack([np.full(size, hub), ids]))                      # a hub row
        pairs.append(ids[rng.integers(0, size, size=(size * 3, 2))])                  # dense inside
        pairs.append(np.array([[int(rng.integers(0, nc)), ids[int(rng.integers(0, size))]]]))  # one cut edge
        n += size
    p = np.concatenate(pairs).astype(np.int64)
    return symmetrize(p[p[:, 0] != p[:, 1]], n)


@pytest.mark.parametrize("seed", range(4))
def test_witness_repair_paths(seed, oracle_mod):
    from paper_2301_01356_b200 import _lib

    g = _core_with_blobs(seed)
    ref = oracle_mod.fast_bcc(g.offsets, g.edges)
    old = _lib.get_option("witness")
    try:
        for w in (2, 1, 0):
            _lib.set_option("witness", w)
            r = _run(g, debug=False)
            for k in ("label", "head", "is_ap", "edge_label"):
                assert np.array_equal(r[k], ref[k]), (seed, w, k)
            assert r["num_bccs"] == ref["num_bccs"] and r["num_components"] == ref["num_components"]
            if w:  # the host path records the rows' first arcs itself (k_record_arcs) before sampling them
                from paper_2301_01356_b200 import Graph, fast_bcc

                lab = fast_bcc(Graph(g.offsets, g.edges).pin())
                for k in ("label", "head", "is_ap", "edge_label"):
                    assert np.array_equal(np.asarray(getattr(lab, k)).astype(ref[k].dtype), ref[k]), (seed, w, "host", k)
                assert lab.num_bccs == ref["num_bccs"]
    finally:
        _lib.set_option("witness", old)


def test_random_graphs_witness_forced(oracle_mod):
    """The seeded random graphs again with the sampled tags forced on."""
    from paper_2301_01356_b200 import _lib

    old = _lib.get_option("witness")
    try:
        _lib.set_option("witness", 2)
        for seed in range(0, 200, 3):
            g = _random_graph(seed)
            ref = oracle_mod.fast_bcc(g.offsets, g.edges)
            r = _run(g, debug=False)
            for k in ("label", "head", "is_ap", "edge_label"):
                assert np.array_equal(r[k], ref[k]), (seed, k)
            assert r["num_bccs"] == ref["num_bccs"] and r["num_components"] == ref["num_components"], seed
    finally:
        _lib.set_option("witness", old)
