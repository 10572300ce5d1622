"""The reference's public stage operations, on the device.

Same names, arguments, result types and errors as the reference modules
(/root/reference/pkg/src/fastbcc):

* ``connected_components(g, keep_edge=None, *, beta=None, seed=0) -> CCResult``
  (connectivity.py:593-611)
* ``list_ranking(nxt, heads) -> ranks`` (euler_tour.py:322-358)
* ``build_euler_tour(n, tree_edges, labels=None) -> RootedForest``
  (euler_tour.py:361-394) -- parent/first/last identical to the reference's
* ``compute_tags(g, forest, block=16) -> VertexTags``, ``compute_w``
  (tagging.py:259-304)
* ``skeleton_record(parent, first, last, low, high)`` (connectivity.py:471-480)
* ``classify_edges(g, forest, tags)``: ``classify_edge`` (bcc.py:54-70) for
  every slot at once
* ``symmetrize_device(edges, n) -> Graph`` (graphs.py:119-143 on the GPU)

Inputs may be numpy arrays (copied to the device) or CUDA tensors; outputs
are numpy arrays, like the reference's.  Every call runs the sm_100a kernels
through the C ABI (include/fastbcc_b200.h); there is no CPU path.
"""

import ctypes
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _lib
from .graphs import Graph


@dataclass
class EdgeList:
    """(k, 2) undirected pairs (graphs.py:20-33)."""

    pairs: np.ndarray

    def __len__(self):
        return self.pairs.shape[0]


@dataclass
class CCResult:
    """connectivity.py:424-430: min-member labels, n - c forest edges, c."""

    labels: np.ndarray
    forest_edges: EdgeList
    num_components: int


@dataclass
class RootedForest:
    """euler_tour.py:38-54."""

    parent: np.ndarray
    first: np.ndarray
    last: np.ndarray
    roots: np.ndarray

    @property
    def n(self) -> int:
        return self.parent.size

    @property
    def tour_len(self) -> int:
        return 2 * self.parent.size


@dataclass
class VertexTags:
    """tagging.py:42-49."""

    w1: np.ndarray
    w2: np.ndarray
    low: np.ndarray
    high: np.ndarray


class EdgeClass(IntEnum):
    """bcc.py:45-51."""

    PLAIN_TREE = 0
    FENCE_TREE = 1
    BACK = 2
    CROSS = 3


def is_ancestor(forest: RootedForest, u: int, v: int) -> bool:
    """euler_tour.py:57-61."""
    return bool(forest.first[u] <= forest.first[v] and forest.last[v] <= forest.last[u])


# ---------------------------------------------------------------------------
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("needs a CUDA device (no CPU fallback)")
    return torch


def _dev(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype).contiguous()


def _csr(g: Graph):
    torch = _torch()
    if getattr(g, "_dev", None) is not None:
        off, adj = g._dev
        return off.to("cuda"), adj.view(torch.int32).to("cuda") if adj.dtype == torch.uint32 else adj.to("cuda")
    return (torch.from_numpy(g.offsets).to("cuda"),
            torch.from_numpy(g.edges.view(np.int32)).to("cuda"))


def _ws(op, a, b=0):
    torch = _torch()
    return torch.empty(max(_lib.op_workspace_bytes(op, a, b), 256), dtype=torch.uint8, device="cuda")


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None or t.numel() == 0 else t.data_ptr()


# ---------------------------------------------------------------------------
def connected_components(g: Graph, keep_edge=None, *, beta=None, seed: int = 0) -> CCResult:
    """Components of ``g`` restricted to edges where ``keep_edge(u, v)`` holds
    (a symmetric predicate, or a per-slot mask array); canonical min labels,
    n - c forest edges.  ``beta``/``seed`` are result-neutral (accepted)."""
    torch = _torch()
    n, m = g.n, g.m
    if n == 0:
        return CCResult(np.empty(0, np.int32), EdgeList(np.empty((0, 2), np.int64)), 0)
    off, adj = _csr(g)
    mask = None
    if keep_edge is not None:
        if isinstance(keep_edge, np.ndarray) or hasattr(keep_edge, "data_ptr"):
            mask = _dev(keep_edge, torch.uint8)
        else:  # callable: expanded per slot on the host, like the reference (connectivity.py:602-611)
            pairs = g.edge_pairs()
            mask = _dev(np.fromiter((bool(keep_edge(int(u), int(v))) for u, v in pairs), dtype=np.uint8,
                                    count=m), torch.uint8)
    label = torch.empty(n, dtype=torch.int32, device="cuda")
    forest = torch.empty(2 * n, dtype=torch.int32, device="cuda")
    ws = _ws(_lib.OP_CONNECTED_COMPONENTS, n, m)
    nc = ctypes.c_int64(0)
    _lib.check(_lib.load().fbcc_connected_components(off.data_ptr(), _ptr(adj), n, m, _ptr(mask), ws.data_ptr(),
                                                     ws.numel(), label.data_ptr(), forest.data_ptr(),
                                                     ctypes.byref(nc), _stream()))
    lab = label.cpu().numpy()
    fe = forest.view(n, 2).cpu().numpy()
    hooked = np.flatnonzero(lab != np.arange(n))
    return CCResult(lab, EdgeList(fe[hooked].astype(np.int64)), int(nc.value))


def list_ranking(nxt, heads) -> np.ndarray:
    """0-based ranks from each list's head (euler_tour.py:322-358); raises
    ValueError on cycles, merges, mid-list heads, unreachable cells."""
    torch = _torch()
    nxt_t = _dev(nxt, torch.int32)
    heads_t = _dev(heads, torch.int32)
    L, H = nxt_t.numel(), heads_t.numel()
    ranks = torch.empty(max(L, 1), dtype=torch.int32, device="cuda")
    if L == 0:
        return np.empty(0, np.int32)
    ws = _ws(_lib.OP_LIST_RANKING, L, H)
    _lib.check(_lib.load().fbcc_list_ranking(nxt_t.data_ptr(), L, _ptr(heads_t), H, ranks.data_ptr(),
                                             ws.data_ptr(), ws.numel(), _stream()))
    return ranks[:L].cpu().numpy()


def build_euler_tour(n: int, tree_edges, labels=None) -> RootedForest:
    """Root a spanning forest at each component's minimum vertex
    (euler_tour.py:361-394).  Output identical to the reference's."""
    torch = _torch()
    if n and 2 * n > (1 << 31) - 1:
        raise ValueError("tour positions need n <= 2**30")
    pairs = getattr(tree_edges, "pairs", tree_edges)
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    k = pairs.shape[0]
    if k >= n and n > 0:
        raise ValueError("a forest on n vertices has at most n-1 edges")
    if k and (pairs.min() < 0 or pairs.max() >= n):
        raise ValueError("tree edge endpoint out of range")
    if n == 0:
        z = np.empty(0, np.int32)
        return RootedForest(z, z.copy(), z.copy(), z.copy())
    p_t = _dev(pairs.astype(np.int32), torch.int32)
    lab_t = _dev(labels, torch.int32) if labels is not None else None
    parent = torch.empty(n, dtype=torch.int32, device="cuda")
    first = torch.empty_like(parent)
    last = torch.empty_like(parent)
    ws = _ws(_lib.OP_BUILD_EULER_TOUR, n, k)
    _lib.check(_lib.load().fbcc_build_euler_tour(n, _ptr(p_t), k, _ptr(lab_t), parent.data_ptr(), first.data_ptr(),
                                                 last.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
    par = parent.cpu().numpy()
    return RootedForest(par, first.cpu().numpy(), last.cpu().numpy(), np.flatnonzero(par == -1).astype(np.int32))


def compute_tags(g: Graph, forest: RootedForest, block: int = 16) -> VertexTags:
    """w1/w2 and low/high of every vertex (tagging.py:300-304); ``block`` is
    result-neutral but validated like the reference (tagging.py:277-278)."""
    torch = _torch()
    if block < 2:
        raise ValueError("block must be >= 2")
    n, m = g.n, g.m
    if n == 0:
        z = np.empty(0, np.int32)
        return VertexTags(z, z.copy(), z.copy(), z.copy())
    off, adj = _csr(g)
    par, fst, lst = (_dev(a, torch.int32) for a in (forest.parent, forest.first, forest.last))
    out = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(4)]
    ws = _ws(_lib.OP_COMPUTE_TAGS, n, m)
    _lib.check(_lib.load().fbcc_compute_tags(off.data_ptr(), _ptr(adj), n, m, par.data_ptr(), fst.data_ptr(),
                                             lst.data_ptr(), *[t.data_ptr() for t in out], ws.data_ptr(),
                                             ws.numel(), _stream()))
    return VertexTags(*[t.cpu().numpy() for t in out])


def compute_w(g: Graph, forest: RootedForest):
    """(w1, w2) (tagging.py:259-267)."""
    t = compute_tags(g, forest)
    return t.w1, t.w2


def skeleton_record(parent, first, last, low, high) -> np.ndarray:
    """Packed per-vertex record (connectivity.py:471-480): word 0 =
    first << 32 | last, word 1 = (parent + 1) << 1 | fence."""
    parent, first, last, low, high = (np.asarray(a, np.int64) for a in (parent, first, last, low, high))
    n = parent.size
    skel = np.empty((n, 2), np.int64)
    skel[:, 0] = (first << 32) | (last & 0xFFFFFFFF)
    p = parent
    pc = np.maximum(p, 0)
    fence = (p >= 0) & (low >= first[pc]) & (high <= last[pc])
    skel[:, 1] = ((p + 1) << 1) | fence.astype(np.int64)
    return skel


def classify_edges(g: Graph, forest: RootedForest, tags: VertexTags) -> np.ndarray:
    """EdgeClass of every slot (classify_edge, bcc.py:54-70), computed on the
    device (``fbcc_classify_edges``): int8[m] in CSR slot order."""
    torch = _torch()
    off, adj = _csr(g)
    n, m = off.numel() - 1, adj.numel()
    out = torch.empty(max(m, 1), dtype=torch.int8, device="cuda")
    arrs = [_dev(a, torch.int32) for a in (forest.parent, forest.first, forest.last, tags.low, tags.high)]
    ws = _ws(_lib.OP_CLASSIFY_EDGES, n, m)
    rc = _lib.load().fbcc_classify_edges(off.data_ptr(), _ptr(adj), n, m, *[_ptr(a) for a in arrs],
                                         out.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    if rc == _lib.FBCC_ERR_RANGE:
        raise ValueError("edge endpoint out of range")
    _lib.check(rc)
    return out[:m].cpu().numpy()


def symmetrize_device(edges, n: int) -> Graph:
    """symmetrize() on the GPU (graphs.py:119-143): sorted rows, reverse arcs
    added, self-loops and duplicates dropped.  Returns a device Graph."""
    torch = _torch()
    if n < 0 or n >= 1 << 31:
        raise ValueError("vertex count must fit 32-bit ids")
    pairs = getattr(edges, "pairs", edges)
    if isinstance(pairs, torch.Tensor):
        p = pairs.to("cuda", torch.int64).reshape(-1, 2)
    else:
        p = torch.from_numpy(np.asarray(pairs, dtype=np.int64).reshape(-1, 2)).to("cuda")
    k = p.shape[0]
    u = p[:, 0].contiguous()
    v = p[:, 1].contiguous()
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    e = torch.empty(max(2 * k, 1), dtype=torch.int32, device="cuda")
    ws = _ws(_lib.OP_SYMMETRIZE, k, n)
    m = ctypes.c_int64(0)
    rc = _lib.load().fbcc_symmetrize(_ptr(u), _ptr(v), k, n, off.data_ptr(), e.data_ptr(), ctypes.byref(m),
                                     ws.data_ptr(), ws.numel(), _stream())
    if rc == _lib.FBCC_ERR_RANGE:
        raise ValueError("edge endpoint out of range")
    _lib.check(rc)
    return Graph.from_device(off, e[: m.value])


def extract_bccs_device(label, head) -> list:
    """extract_bccs (bcc.py:199-219) on the device: sorted vertex sets of all
    blocks, ordered by label."""
    torch = _torch()
    lab = _dev(label, torch.int32)
    hd = _dev(head, torch.int32)
    n = lab.numel()
    if n == 0:
        return []
    boff = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
    bv = torch.empty(2 * n, dtype=torch.int32, device="cuda")
    nb = ctypes.c_int64(0)
    ws = _ws(_lib.OP_EXTRACT_BCCS, n)
    _lib.check(_lib.load().fbcc_extract_bccs(lab.data_ptr(), hd.data_ptr(), n, boff.data_ptr(), bv.data_ptr(),
                                             ctypes.byref(nb), ws.data_ptr(), ws.numel(), _stream()))
    k = int(nb.value)
    if k == 0:
        return []
    o = boff[: k + 1].cpu().numpy()
    o[0] = 0  # first block starts at the first sorted key
    vals = bv[: o[-1]].cpu().numpy().astype(np.int64)
    return [vals[o[i]:o[i + 1]] for i in range(k)]
