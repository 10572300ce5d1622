"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/fastbcc_b200.h declares, the host-side wrapper mirrors the
reference's argument errors, and Graph/symmetrize match the reference
container semantics (graphs.py:43-143).  No kernel is launched here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2301_01356_b200 import _lib, build

    build.build()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    hdr = (ROOT / "include" / "fastbcc_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fbcc_\w+)\s*\(", hdr, re.M))
    from paper_2301_01356_b200 import _lib

    assert declared == set(_lib.all_exports())
    for name in declared:
        assert hasattr(lib, name), name


def test_strerror_and_version(lib):
    assert lib.fbcc_version() >= 100
    assert b"cycle" in lib.fbcc_strerror(5)
    assert b"cover" in lib.fbcc_strerror(6)
    assert b"2**30" in lib.fbcc_strerror(2)


def test_workspace_sizes(lib):
    from paper_2301_01356_b200 import _lib

    small = _lib.workspace_bytes(1000, 4000)
    big = _lib.workspace_bytes(10**6, 4 * 10**6)
    assert 0 < small < big
    # n > 2^30 and m >= 2^31 are rejected like euler_tour.py:402-403
    with pytest.raises(ValueError, match="2\\*\\*30"):
        _lib.workspace_bytes(1 << 30, 10)
    with pytest.raises(ValueError):
        _lib.workspace_bytes(10, 1 << 31)


def test_run_rejects_bad_args_without_gpu(lib):
    from paper_2301_01356_b200 import _lib

    out = _lib.FbccOutputs()
    stats = _lib.FbccStats()
    rc = lib.fbcc_run(None, None, 4, 0, None, 0, ctypes.byref(out), None, ctypes.byref(stats), None, 0)
    assert rc == _lib.FBCC_ERR_ARG
    rc = lib.fbcc_run(ctypes.c_void_p(8), None, -1, 0, None, 0, ctypes.byref(out), None, None, None, 0)
    assert rc == _lib.FBCC_ERR_ARG


def test_knob_errors_mirror_reference():
    from paper_2301_01356_b200 import Graph, fast_bcc

    g = Graph.from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(ValueError):
        fast_bcc(g, block=1)
    with pytest.raises(ZeroDivisionError):
        fast_bcc(g, beta=0)
    with pytest.raises(ValueError):
        fast_bcc(g, beta=-1.0)


def test_empty_graph_needs_no_device():
    from paper_2301_01356_b200 import Graph, extract_bccs, fast_bcc

    lab = fast_bcc(Graph.empty(0))
    assert lab.n == 0 and lab.num_bccs == 0 and extract_bccs(lab) == []


def test_no_cpu_fallback():
    import torch

    from paper_2301_01356_b200 import Graph, fast_bcc

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        fast_bcc(Graph.from_edges(3, [(0, 1), (1, 2)]))


def test_symmetrize_and_validate():
    from paper_2301_01356_b200.graphs import Graph, symmetrize

    g = symmetrize([(0, 1), (1, 0), (2, 2), (1, 3), (0, 1)], 4)
    assert g.offsets.tolist() == [0, 1, 3, 3, 4]
    assert g.edges.tolist() == [1, 0, 3, 1]
    g.validate()
    assert g.undirected_edges().tolist() == [[0, 1], [1, 3]]
    with pytest.raises(ValueError):
        symmetrize([(0, 5)], 4)
    with pytest.raises(ValueError):
        Graph(np.array([0, 1, 1]), np.array([1], np.uint32), validate=True)  # asymmetric
    # idempotent (reference test_graphs.py:62-70)
    p = g.edge_pairs()
    g2 = symmetrize(p, 4)
    assert np.array_equal(g2.offsets, g.offsets) and np.array_equal(g2.edges, g.edges)


def test_symmetrize_matches_golden_corpus(corpus):
    from paper_2301_01356_b200.graphs import symmetrize

    for i, name, g in corpus.items():
        g2 = symmetrize(g.edge_pairs(), g.n)
        assert np.array_equal(g2.offsets, g.offsets), name
        assert np.array_equal(g2.edges, g.edges), name


def test_bin_roundtrip_and_errors(tmp_path):
    import warnings

    from paper_2301_01356_b200.graphs import Graph, load_bin, symmetrize, write_bin

    g = symmetrize([(0, 1), (1, 2), (2, 0), (2, 3)], 5)
    p = tmp_path / "g.bin"
    write_bin(g, p)
    h = load_bin(p)
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.edges, g.edges)
    raw = p.read_bytes()
    (tmp_path / "t.bin").write_bytes(raw[:10])
    with pytest.raises(ValueError, match="truncated"):
        load_bin(tmp_path / "t.bin")
    (tmp_path / "s.bin").write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="size mismatch"):
        load_bin(tmp_path / "s.bin")
    legacy = bytearray(raw)
    n, m = g.n, g.m
    legacy[16:24] = np.array([24 + 8 * (n - 1) + 4 * m], "<u8").tobytes()
    (tmp_path / "l.bin").write_bytes(bytes(legacy))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        load_bin(tmp_path / "l.bin")
        assert any("legacy" in str(x.message) for x in w)
