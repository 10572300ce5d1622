"""Input boundary: the reference's symmetric CSR container and ``symmetrize``.

Mirrors ``fastbcc.graphs.Graph`` / ``symmetrize``
(/root/reference/pkg/src/fastbcc/graphs.py:43-143): int64 offsets[n+1],
uint32 targets[m], every undirected edge stored as two directed slots,
sorted neighbour lists, no self-loops, no duplicates.  ``fast_bcc`` consumes
this layout unchanged -- the int64 offsets and uint32 targets are copied to
HBM as-is and read directly by the kernels (no host-side conversion).

A ``Graph`` may also wrap torch tensors already resident on a CUDA device
(``Graph.from_device``); ``fast_bcc`` then skips the host->device copy.
"""

import numpy as np


class Graph:
    """Symmetric CSR graph (graphs.py:43-58).

    :param offsets: int64[n+1]; ``offsets[v]:offsets[v+1]`` are v's slots
    :param edges: uint32[m] neighbour ids
    """

    __slots__ = ("offsets", "edges", "_dev", "_pinned", "_pinned_off32")

    def __init__(self, offsets, edges, validate: bool = False):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.edges = np.ascontiguousarray(edges, dtype=np.uint32)
        self._dev = None
        self._pinned = None
        self._pinned_off32 = None
        if self.offsets.ndim != 1 or self.offsets.size == 0:
            raise ValueError("offsets must be a 1-d array of length n+1")
        if validate:
            self.validate()

    def pin(self):
        """Cache page-locked copies of the CSR: fast_bcc then streams them to
        the device at full link speed, overlapped with Stage 1."""
        import torch

        if self._pinned is None and self._dev is None:
            self._pinned = (torch.from_numpy(self.offsets).pin_memory(),
                            torch.from_numpy(self.edges.view(np.int32)).pin_memory())
            # the host path uploads int32 offsets (half the bytes; widened on
            # the device) whenever the slot count fits 32 bits
            if self.m < (1 << 31):
                self._pinned_off32 = torch.from_numpy(self.offsets.astype(np.int32)).pin_memory()
        return self

    @classmethod
    def from_device(cls, offsets_t, edges_t):
        """Wrap device-resident torch tensors (int64 offsets, int32/uint32
        targets).  Host arrays stay empty placeholders of the right n."""
        import torch

        if offsets_t.dtype != torch.int64:
            raise ValueError("device offsets must be int64")
        if edges_t.dtype not in (torch.int32, torch.uint32):
            raise ValueError("device edges must be int32 or uint32")
        g = cls.__new__(cls)
        g.offsets = None
        g.edges = None
        g._dev = (offsets_t.contiguous(), edges_t.contiguous())
        g._pinned = None
        g._pinned_off32 = None
        return g

    @property
    def n(self) -> int:
        if self._dev is not None:
            return self._dev[0].numel() - 1
        return self.offsets.size - 1

    @property
    def m(self) -> int:
        """Directed slot count (2x the undirected edge count)."""
        if self._dev is not None:
            return self._dev[1].numel()
        return self.edges.size

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.edges[self.offsets[v]: self.offsets[v + 1]]

    def validate(self) -> None:
        """CSR invariants of graphs.py:76-98; ValueError on the first breach."""
        off, e, n = self.offsets, self.edges, self.n
        if off[0] != 0 or off[-1] != e.size:
            raise ValueError("offsets must start at 0 and end at m")
        if np.any(np.diff(off) < 0):
            raise ValueError("offsets must be nondecreasing")
        if e.size and int(e.max()) >= n:
            raise ValueError("edge target out of range")
        src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
        if e.size:
            same_row = src[1:] == src[:-1]
            if np.any(e[1:][same_row] <= e[:-1][same_row]):
                raise ValueError("neighbor lists must be strictly increasing")
        if np.any(src == e):
            raise ValueError("self-loops are not allowed")
        fwd = (src.astype(np.uint64) << np.uint64(32)) | e.astype(np.uint64)
        rev = (e.astype(np.uint64) << np.uint64(32)) | src.astype(np.uint64)
        if not np.array_equal(np.sort(fwd), np.sort(rev)):
            raise ValueError("graph is not symmetric")

    def edge_pairs(self) -> np.ndarray:
        """All directed (source, target) pairs, shape (m, 2)."""
        src = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.offsets))
        return np.column_stack([src, self.edges.astype(np.int64)])

    def undirected_edges(self) -> np.ndarray:
        """(E, 2) pairs (u, v), u < v, in CSR order -- the edge numbering of
        ``BccLabeling.edge_label`` (same order as baselines.py:251-257)."""
        p = self.edge_pairs()
        return p[p[:, 0] < p[:, 1]]

    @classmethod
    def empty(cls, n: int) -> "Graph":
        return cls(np.zeros(n + 1, dtype=np.int64), np.empty(0, np.uint32))

    @classmethod
    def from_edges(cls, n: int, pairs) -> "Graph":
        return symmetrize(pairs, n)

    def __repr__(self):
        return f"Graph(n={self.n}, m={self.m})"


def symmetrize(edges, n: int) -> Graph:
    """Graph from arbitrary undirected pairs (graphs.py:119-143): adds the
    reverse of each pair, drops self-loops and duplicates, sorts rows.
    ``edges`` is any (k, 2) array-like (or an object with ``.pairs``)."""
    if n < 0 or n >= 1 << 32:
        raise ValueError("vertex count must fit 32-bit ids")
    pairs = getattr(edges, "pairs", edges)
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.size and (pairs.min() < 0 or pairs.max() >= n):
        raise ValueError("edge endpoint out of range")
    u, v = pairs[:, 0], pairs[:, 1]
    keep = u != v
    u, v = u[keep].astype(np.uint64), v[keep].astype(np.uint64)
    keys = np.concatenate([(u << np.uint64(32)) | v, (v << np.uint64(32)) | u])
    keys.sort()  # row-major (src, dst); sort + adjacent-diff == np.unique, ~100x faster here
    if keys.size:
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    src = (keys >> np.uint64(32)).astype(np.int64)
    dst = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=offsets[1:])
    return Graph(offsets, dst)


# ---------------------------------------------------------------------------
# binary CSR artifact (reference format, graphs.py:146-204): little-endian
# u64 n, u64 m, u64 size, (n+1) u64 offsets, m u32 targets.  The size word is
# 24 + 8(n+1) + 4m; the legacy value 24 + 8(n-1) + 4m is accepted with a
# warning, like the reference.
# ---------------------------------------------------------------------------
_HEADER_BYTES = 24


def expected_bin_size(n: int, m: int) -> int:
    return _HEADER_BYTES + 8 * (n + 1) + 4 * m


def write_bin(g: Graph, path) -> None:
    n, m = g.n, g.m
    with open(path, "wb") as f:
        np.array([n, m, expected_bin_size(n, m)], dtype="<u8").tofile(f)
        np.asarray(g.offsets, dtype="<u8").tofile(f)
        np.asarray(g.edges, dtype="<u4").tofile(f)


def load_bin(path, device=None) -> Graph:
    """Read a .bin CSR (graphs.py:173-204).  With ``device`` set, the file is
    read straight into page-locked staging buffers (no intermediate host
    copy) and copied asynchronously to HBM; a device Graph is returned."""
    import warnings

    with open(path, "rb") as f:
        header = np.fromfile(f, dtype="<u8", count=3)
        if header.size != 3:
            raise ValueError(f"{path}: truncated header (need {_HEADER_BYTES} bytes)")
        n, m, size_field = (int(x) for x in header)
        want = expected_bin_size(n, m)
        if device is None:
            offsets = np.fromfile(f, dtype="<u8", count=n + 1)
            edges = np.fromfile(f, dtype="<u4", count=m)
            got_o, got_e = offsets.size, edges.size
        else:
            import torch

            off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
            adj_h = torch.empty(m, dtype=torch.int32, pin_memory=True)
            offsets = off_h.numpy()
            edges = adj_h.numpy().view(np.uint32)
            got_o = f.readinto(memoryview(offsets).cast("B")) // 8
            got_e = f.readinto(memoryview(edges).cast("B")) // 4 if m else 0
        extra = f.read(1)
    if got_o != n + 1 or got_e != m or extra:
        have = _HEADER_BYTES + got_o * 8 + got_e * 4 + len(extra)
        raise ValueError(f"{path}: size mismatch, expected {want} bytes for n={n} m={m}, "
                         f"got {have}{'+' if extra else ''}")
    if size_field != want:
        legacy = _HEADER_BYTES + 8 * (n - 1) + 4 * m
        if size_field != legacy:
            raise ValueError(f"{path}: size field {size_field} matches neither {want} nor the legacy value {legacy}")
        warnings.warn(f"{path}: legacy size field {size_field} (expected {want}); accepting", stacklevel=2)
    if offsets[0] != 0 or offsets[-1] != m:
        raise ValueError(f"{path}: offsets must run from 0 to m")
    if device is None:
        return Graph(offsets.astype(np.int64), edges)
    off_t = off_h.to(device, non_blocking=True)
    adj_t = adj_h.to(device, non_blocking=True)
    torch.cuda.current_stream(off_t.device).synchronize()  # the staging buffers may be reused after this
    return Graph.from_device(off_t, adj_t)
