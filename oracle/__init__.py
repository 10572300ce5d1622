"""CPU oracle for the FAST-BCC hot path -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end over ``liboracle.so`` (built from
``fastbcc_oracle.c``, a C restatement of the reference's algorithm; every C
function cites the reference file:line it follows).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this
module, and only as the checker / CPU baseline: the product package
``paper_2301_01356_b200`` never imports it and has no CPU fallback.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the reference package itself
(``tests/golden/make_golden.py``).
"""

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

ERR_CYCLE = 1
ERR_COVER = 2
ERR_LABELS = 3
ERR_ARG = 4
ERR_NOMEM = 5

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build(force: bool = False) -> Path:
    so = _HERE / "liboracle.so"
    src = _HERE / "fastbcc_oracle.c"
    if force or not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-B", "liboracle.so"],
                       check=True, capture_output=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "liboracle.so"
        if not so.exists():
            build()
        L = ctypes.CDLL(str(so))
        L.orc_cc.restype = _I64
        L.orc_cc.argtypes = [_I64, _P, _P, _P, _P, _P, _P, _P, _P]
        L.orc_list_ranking.restype = ctypes.c_int
        L.orc_list_ranking.argtypes = [_I64, _P, _I64, _P, _P]
        L.orc_root_forest.restype = ctypes.c_int
        L.orc_root_forest.argtypes = [_I64, _P, _I64, _P, _P, _P, _P, _P]
        L.orc_compute_w.restype = None
        L.orc_compute_w.argtypes = [_I64, _P, _P, _P, _P, _P, _P]
        L.orc_low_high.restype = ctypes.c_int
        L.orc_low_high.argtypes = [_I64, _P, _P, _P, _P, _I64, _P, _P]
        L.orc_pack_skeleton.restype = None
        L.orc_pack_skeleton.argtypes = [_I64, _P, _P, _P, _P, _P, _P]
        L.orc_component_heads.restype = None
        L.orc_component_heads.argtypes = [_I64, _P, _P, _P, _P]
        L.orc_articulation.restype = None
        L.orc_articulation.argtypes = [_I64, _P, _P, _P]
        L.orc_edge_labels.restype = _I64
        L.orc_edge_labels.argtypes = [_I64, _P, _P, _P, _P, _P]
        L.orc_fast_bcc.restype = ctypes.c_int
        L.orc_fast_bcc.argtypes = [_I64, _P, _P, _P, _P, _P, _P, _P, _P]
        L.orc_fast_bcc_mode.restype = ctypes.c_int
        L.orc_fast_bcc_mode.argtypes = [_I64, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data


def _csr(offsets, edges):
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    adj = np.ascontiguousarray(edges, dtype=np.uint32)
    return off, adj, off.size - 1


def num_threads() -> int:
    return lib().orc_num_threads()


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def connected_components(offsets, edges, keep_mask=None, skel=None):
    """(label int32[n], forest int32[k, 2], ncomp) -- connectivity.py:541-611."""
    off, adj, n = _csr(offsets, edges)
    label = np.empty(n, np.int32)
    fu = np.empty(max(n, 1), np.int32)
    fv = np.empty(max(n, 1), np.int32)
    k = np.zeros(1, np.int64)
    mask = None if keep_mask is None else np.ascontiguousarray(keep_mask, np.uint8)
    sk = None if skel is None else np.ascontiguousarray(skel, np.int64)
    ncomp = lib().orc_cc(n, _ptr(off), _ptr(adj), _ptr(mask), _ptr(sk),
                         _ptr(label), _ptr(fu), _ptr(fv), _ptr(k))
    kk = int(k[0])
    return label, np.column_stack([fu[:kk], fv[:kk]]), int(ncomp)


def list_ranking(nxt, heads):
    """ranks int32[L]; raises ValueError like euler_tour.py:349-357."""
    nxt = np.ascontiguousarray(nxt, np.int32)
    heads = np.ascontiguousarray(heads, np.int32)
    ranks = np.empty(nxt.size, np.int32)
    rc = lib().orc_list_ranking(nxt.size, _ptr(nxt), heads.size, _ptr(heads),
                                _ptr(ranks))
    if rc == ERR_CYCLE:
        raise ValueError("successor structure contains a cycle")
    if rc == ERR_COVER:
        raise ValueError("successor structure is not a disjoint list cover")
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return ranks


def root_forest(n, label, pairs):
    """(parent, first, last) -- euler_tour.py:397-437."""
    label = np.ascontiguousarray(label, np.int32)
    pairs = np.ascontiguousarray(np.asarray(pairs).reshape(-1, 2), np.int32)
    fu = np.ascontiguousarray(pairs[:, 0])
    fv = np.ascontiguousarray(pairs[:, 1])
    parent = np.empty(n, np.int32)
    first = np.empty(n, np.int32)
    last = np.empty(n, np.int32)
    rc = lib().orc_root_forest(n, _ptr(label), fu.size, _ptr(fu), _ptr(fv),
                               _ptr(parent), _ptr(first), _ptr(last))
    if rc == ERR_LABELS:
        raise ValueError("labels are inconsistent with the forest edges")
    if rc:
        raise ValueError(f"successor structure invalid (oracle error {rc})")
    return parent, first, last


def compute_w(offsets, edges, parent, first):
    off, adj, n = _csr(offsets, edges)
    parent = np.ascontiguousarray(parent, np.int32)
    first = np.ascontiguousarray(first, np.int32)
    w1 = np.empty(n, np.int32)
    w2 = np.empty(n, np.int32)
    lib().orc_compute_w(n, _ptr(off), _ptr(adj), _ptr(parent), _ptr(first),
                        _ptr(w1), _ptr(w2))
    return w1, w2


def low_high(first, last, w1, w2, block=16):
    first = np.ascontiguousarray(first, np.int32)
    last = np.ascontiguousarray(last, np.int32)
    w1 = np.ascontiguousarray(w1, np.int32)
    w2 = np.ascontiguousarray(w2, np.int32)
    n = first.size
    low = np.empty(n, np.int32)
    high = np.empty(n, np.int32)
    rc = lib().orc_low_high(n, _ptr(first), _ptr(last), _ptr(w1), _ptr(w2),
                            int(block), _ptr(low), _ptr(high))
    if rc == ERR_ARG:
        raise ValueError("block must be >= 2")
    return low, high


def pack_skeleton(parent, first, last, low, high):
    arrs = [np.ascontiguousarray(a, np.int32) for a in (parent, first, last, low, high)]
    n = arrs[0].size
    skel = np.empty((n, 2), np.int64)
    lib().orc_pack_skeleton(n, *[_ptr(a) for a in arrs], _ptr(skel))
    return skel


def component_heads(label, parent, first):
    label, parent, first = (np.ascontiguousarray(a, np.int32) for a in (label, parent, first))
    head = np.empty(label.size, np.int32)
    lib().orc_component_heads(label.size, _ptr(label), _ptr(parent), _ptr(first), _ptr(head))
    return head


def articulation_flags(label, head):
    label = np.ascontiguousarray(label, np.int32)
    head = np.ascontiguousarray(head, np.int32)
    out = np.empty(label.size, np.uint8)
    lib().orc_articulation(label.size, _ptr(label), _ptr(head), _ptr(out))
    return out


def edge_labels(offsets, edges, label, head):
    off, adj, n = _csr(offsets, edges)
    label = np.ascontiguousarray(label, np.int32)
    head = np.ascontiguousarray(head, np.int32)
    out = np.empty(max(adj.size // 2, 1), np.int32)
    E = lib().orc_edge_labels(n, _ptr(off), _ptr(adj), _ptr(label), _ptr(head), _ptr(out))
    return out[:E]


def fast_bcc(offsets, edges, parallel=False):
    """Whole pipeline: dict with label, head, is_ap, edge_label, num_bccs,
    num_components, num_edges, seconds[5].  ``parallel``: the concurrent
    union-find / splitter list-ranking variants (same outputs; the CPU
    baseline's mode)."""
    off, adj, n = _csr(offsets, edges)
    label = np.empty(n, np.int32)
    head = np.empty(n, np.int32)
    is_ap = np.empty(n, np.uint8)
    el = np.empty(max(adj.size // 2, 1), np.int32)
    counts = np.zeros(3, np.int64)
    secs = np.zeros(5, np.float64)
    rc = lib().orc_fast_bcc_mode(n, _ptr(off), _ptr(adj), _ptr(label), _ptr(head),
                                 _ptr(is_ap), _ptr(el), _ptr(counts), _ptr(secs), int(bool(parallel)))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return dict(label=label, head=head, is_ap=is_ap,
                edge_label=el[: int(counts[2])], num_bccs=int(counts[0]),
                num_components=int(counts[1]), num_edges=int(counts[2]),
                seconds=secs)
