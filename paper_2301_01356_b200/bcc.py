"""``fast_bcc`` -- drop-in for the reference entry point, running on a B200.

Mirrors ``fastbcc.bcc`` (/root/reference/pkg/src/fastbcc/bcc.py): same call
``fast_bcc(g, *, beta=None, seed=0, block=16) -> BccLabeling`` (bcc.py:147),
same ``BccLabeling`` fields and helpers (bcc.py:98-126), same
``articulation_points`` / ``extract_bccs`` post-processing (bcc.py:199-235),
same argument errors.  ``BccLabeling`` additionally carries the per-edge
block labels (``edge_label``, canonical: the minimum edge id of the block,
edges numbered as ``Graph.undirected_edges()``) and articulation flags
(``is_ap``), both computed on the device.

All six stages run as hand-written sm_100a kernels behind the C ABI
(include/fastbcc_b200.h); the host only moves the CSR in and the results
out.  There is no CPU path: without the extension or a CUDA device this
module raises.
"""

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graphs import Graph


@dataclass
class StepTimings:
    """Seconds per pipeline step (bcc.py:78-95), from CUDA events.

    The first five fields are the reference's, in its order (positional
    construction works the same): ``first_cc`` = Stage 1, ``rooting`` =
    Stage 2, ``tagging`` = Stage 3, ``last_cc`` = Stages 4+5 (fence +
    skeleton connectivity), ``total`` = all six stages.  Appended:
    ``labelling`` = Stage 6 (heads, articulation flags, edge labels -- outside
    the reference's timed region) and ``stage_ms``, the six raw values.
    """

    first_cc: float = 0.0
    rooting: float = 0.0
    tagging: float = 0.0
    last_cc: float = 0.0
    total: float = 0.0
    labelling: float = 0.0
    stage_ms: tuple = field(default_factory=tuple)

    def as_dict(self) -> dict:
        return {"first_cc": self.first_cc, "rooting": self.rooting, "tagging": self.tagging,
                "last_cc": self.last_cc, "total": self.total}


@dataclass
class BccLabeling:
    """Block structure of a graph (bcc.py:98-126).

    ``label[v]``: minimum member of v's skeleton component.  ``head[l]``: the
    parent of component l's shallowest member, or -1 for a lone forest root
    and at indices that are not labels.  Block l = {v: label[v] == l} | {head[l]}.
    ``edge_label[e]``: minimum edge id of edge e's block; ``is_ap[v]``: v is
    an articulation point.
    """

    label: np.ndarray
    head: np.ndarray
    num_bccs: int
    num_components: int
    timings: StepTimings
    edge_label: np.ndarray = None
    is_ap: np.ndarray = None

    @property
    def n(self) -> int:
        return self.label.shape[0]

    def head_map(self) -> dict:
        head = _host(self.head)
        return {int(l): int(head[l]) for l in np.flatnonzero(head != -1)}

    def is_root(self, v: int) -> bool:
        return bool(self.label[v] == v and self.head[v] == -1)


def _host(a):
    if a is None or isinstance(a, np.ndarray):
        return a
    return a.cpu().numpy()


def _check_knobs(beta, block):
    # result-neutral knobs (test_bcc.py:143-149); argument errors mirror the
    # reference: block < 2 -> ValueError (tagging.py:277-278), beta == 0 ->
    # ZeroDivisionError (connectivity.py:487), beta < 0 -> ValueError
    # (the reference's ldd rule, connectivity.py:531-532)
    if block < 2:
        raise ValueError("block must be >= 2")
    if beta is not None:
        if beta == 0:
            raise ZeroDivisionError("float division by zero")
        if not beta > 0:
            raise ValueError("beta must be positive")


_WS = {}


def _workspace(nbytes: int, device):
    import torch

    key = (str(device),)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _as_graph(g) -> Graph:
    """Accept the reference's ``Graph`` (``__slots__ = ("offsets", "edges")``,
    graphs.py:43-58) or any object with those two arrays: wrapped without a
    copy when they already are contiguous int64 / uint32."""
    if isinstance(g, Graph):
        return g
    if hasattr(g, "offsets") and hasattr(g, "edges"):
        return Graph(g.offsets, g.edges)
    raise TypeError("expected a Graph (offsets int64[n+1], edges uint32[m])")


def _device_csr(g: Graph, device):
    import torch

    if g._dev is not None:
        off, adj = g._dev
        if adj.dtype == torch.uint32:
            adj = adj.view(torch.int32)
        return off, adj, 0
    pinned = g._pinned
    if pinned is not None:
        off_h, adj_h = pinned
    else:
        off_h = torch.from_numpy(g.offsets)
        adj_h = torch.from_numpy(g.edges.view(np.int32))
    off = off_h.to(device, non_blocking=True)
    adj = adj_h.to(device, non_blocking=True)
    return off, adj, off_h.numel() * 8 + adj_h.numel() * 4


def run_device(off, adj, *, edge_labels=True, articulation=True, timing=True, debug=None, stream=None,
               profile=False):
    """Run all six stages on device tensors (int64 offsets, int32 targets).

    Returns (dict of device output tensors, FbccStats).  ``debug`` may be a
    dict to receive the intermediate arrays (parity rungs 1-4).
    """
    import torch

    n = off.numel() - 1
    m = adj.numel()
    dev = off.device
    L = _lib.load()
    if n < 0:
        raise ValueError("offsets must be a 1-d array of length n+1")
    ws_bytes = _lib.workspace_bytes(n, m)
    ws = _workspace(ws_bytes, dev)
    label = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    head = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    comp = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    is_ap = torch.empty(max(n, 1), dtype=torch.uint8, device=dev) if articulation else None
    el = torch.empty(max(m // 2, 1), dtype=torch.int32, device=dev) if edge_labels else None
    outs = _lib.FbccOutputs(label.data_ptr(), head.data_ptr(), el.data_ptr() if el is not None else None,
                            is_ap.data_ptr() if is_ap is not None else None, comp.data_ptr())
    dbg_struct = None
    if debug is not None:
        for k in ("parent", "first", "last", "w1", "w2", "low", "high"):
            debug[k] = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        debug["forest"] = torch.empty(max(2 * n, 2), dtype=torch.int32, device=dev)
        debug["fence"] = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        dbg_struct = _lib.FbccDebug(*[debug[k].data_ptr() for k in
                                      ("forest", "parent", "first", "last", "w1", "w2", "low", "high", "fence")])
    stats = _lib.FbccStats()
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = L.fbcc_run(off.data_ptr(), adj.data_ptr() if m else None, n, m, ws.data_ptr(), ws.numel(),
                    ctypes.byref(outs), ctypes.byref(dbg_struct) if dbg_struct is not None else None,
                    ctypes.byref(stats), ctypes.c_void_p(s.cuda_stream),
                    (_lib.FBCC_FLAG_TIMING if timing else 0) | (_lib.FBCC_FLAG_PROFILE if profile else 0))
    _lib.check(rc)
    E = int(stats.num_edges)
    res = {"label": label[:n], "head": head[:n], "comp": comp[:n],
           "is_ap": is_ap[:n] if is_ap is not None else None,
           "edge_label": el[:E] if el is not None else None}
    return res, stats


class Plan:
    """A CUDA-graph replay of the six stages bound to device tensors
    (``fbcc_plan_*`` in the C ABI).  ``run()`` launches the graph, waits and
    returns the counts; outputs land in ``self.label`` etc.

    A plan is bound to the input *buffers* (pointers, n, m) and freezes the
    options in force at its creation; it does not depend on the buffers'
    contents, so refilling them with another graph of the same size and
    replaying is correct."""

    def __init__(self, off, adj, *, edge_labels=True, articulation=True, profile=False, timing=False):
        import torch

        self.L = _lib.load()
        n = off.numel() - 1
        m = adj.numel()
        dev = off.device
        self.n, self.m, self.off, self.adj = n, m, off, adj
        self.ws = torch.empty(max(_lib.workspace_bytes(n, m), 256), dtype=torch.uint8, device=dev)
        self.label = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.head = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.comp = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.is_ap = torch.empty(max(n, 1), dtype=torch.uint8, device=dev) if articulation else None
        self.edge_label = torch.empty(max(m // 2, 1), dtype=torch.int32, device=dev) if edge_labels else None
        outs = _lib.FbccOutputs(self.label.data_ptr(), self.head.data_ptr(),
                                self.edge_label.data_ptr() if edge_labels else None,
                                self.is_ap.data_ptr() if articulation else None, self.comp.data_ptr())
        h = ctypes.c_void_p()
        _lib.check(self.L.fbcc_plan_create(off.data_ptr(), adj.data_ptr() if m else None, n, m,
                                           self.ws.data_ptr(), self.ws.numel(), ctypes.byref(outs),
                                           (_lib.FBCC_FLAG_PROFILE if profile else 0)
                                           | (_lib.FBCC_FLAG_TIMING if timing else 0), ctypes.byref(h)))
        self._h = h
        self.stats = _lib.FbccStats()

    def run(self, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.off.device)
        _lib.check(self.L.fbcc_plan_run(self._h, ctypes.byref(self.stats), ctypes.c_void_p(s.cuda_stream)))
        return self.stats

    def launch(self, stream=None):
        """Enqueue one replay (graph + counts copy) without waiting; call
        ``collect()`` after synchronising the stream."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.off.device)
        _lib.check(self.L.fbcc_plan_launch(self._h, ctypes.c_void_p(s.cuda_stream)))

    def collect(self):
        _lib.check(self.L.fbcc_plan_stats(self._h, ctypes.byref(self.stats)))
        return self.stats

    def outputs(self):
        E = int(self.stats.num_edges)
        n = self.n
        return {"label": self.label[:n], "head": self.head[:n], "comp": self.comp[:n],
                "is_ap": self.is_ap[:n] if self.is_ap is not None else None,
                "edge_label": self.edge_label[:E] if self.edge_label is not None else None}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self.L.fbcc_plan_destroy(h)
            self._h = None


_SESSIONS = {}


def _session(g: Graph, dev) -> Plan:
    """A graph-replay plan bound to a device-resident input (keyed by its
    buffers), reused across calls -- safe when the caller rewrites the
    buffers in between (plans are content-independent, see Plan)."""
    off, adj, _ = _device_csr(g, dev)
    key = ("dev", off.data_ptr(), adj.data_ptr(), g.n, g.m)
    plan = _SESSIONS.get(key)
    if plan is None:
        _SESSIONS.clear()
        plan = _SESSIONS[key] = Plan(off, adj, timing=True)
    return plan


class _HostRunner:
    """Persistent device buffers for host-resident inputs of one size;
    ``run`` is ``fbcc_run_host``: streamed H2D overlapped with Stage 1,
    early outputs copied back while Stage 6 runs."""

    def __init__(self, n, m, dev):
        import torch

        self.L = _lib.load()
        self.n, self.m, self.dev = n, m, dev
        self.off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.adj = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        self.ws = torch.empty(max(_lib.workspace_bytes(n, m), 256), dtype=torch.uint8, device=dev)
        self.label = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.head = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.is_ap = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        self.edge_label = torch.empty(max(m // 2, 1), dtype=torch.int32, device=dev)
        self.outs = _lib.FbccOutputs(self.label.data_ptr(), self.head.data_ptr(), self.edge_label.data_ptr(),
                                     self.is_ap.data_ptr(), None)

    def run(self, g: Graph):
        import torch

        n, m = self.n, self.m
        flags = _lib.FBCC_FLAG_TIMING
        if g._pinned is not None:
            off_h, adj_h = g._pinned
            off_p, adj_p = off_h.data_ptr(), adj_h.data_ptr()
            if getattr(g, "_pinned_off32", None) is not None:  # int32 offsets: half the upload
                off_p = g._pinned_off32.data_ptr()
                flags |= _lib.FBCC_FLAG_HOST_OFFSETS32
        else:  # pageable: correct, but the copies cannot overlap the kernels
            off_p, adj_p = g.offsets.ctypes.data, g.edges.ctypes.data
        h = {"label": torch.empty(n, dtype=torch.int32, pin_memory=True),
             "head": torch.empty(n, dtype=torch.int32, pin_memory=True),
             "is_ap": torch.empty(n, dtype=torch.uint8, pin_memory=True),
             "edge_label": torch.empty(m // 2, dtype=torch.int32, pin_memory=True)}
        io = _lib.FbccHostIO(off_p, adj_p if m else None, h["label"].data_ptr(), h["head"].data_ptr(),
                             h["edge_label"].data_ptr() if m // 2 else None, h["is_ap"].data_ptr())
        st = _lib.FbccStats()
        s = torch.cuda.current_stream(self.dev)
        _lib.check(self.L.fbcc_run_host(ctypes.byref(io), n, m, self.off.data_ptr(), self.adj.data_ptr(),
                                        self.ws.data_ptr(), self.ws.numel(), ctypes.byref(self.outs),
                                        ctypes.byref(st), ctypes.c_void_p(s.cuda_stream), flags))
        E = int(st.num_edges)
        return st, {k: v.numpy() for k, v in h.items()}, E


def _host_session(g: Graph, dev) -> _HostRunner:
    key = ("host", str(dev), g.n, g.m)
    r = _SESSIONS.get(key)
    if r is None:
        _SESSIONS.clear()
        r = _SESSIONS[key] = _HostRunner(g.n, g.m, dev)
    return r


def _to_host(res, keys):
    """D2H into pinned buffers (full link speed), returned as numpy views that
    own their buffer (freed back to torch's pinned cache when dropped)."""
    import torch

    host = {}
    for k in keys:
        t = res[k]
        if t is None:
            host[k] = None
            continue
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        host[k] = h
    torch.cuda.current_stream(next(v for v in res.values() if v is not None).device).synchronize()
    return {k: (None if v is None else v.numpy()) for k, v in host.items()}


def fast_bcc(g: Graph, *, beta: float | None = None, seed: int = 0, block: int = 16,
             device=None, device_outputs: bool = False, validate: bool = False) -> BccLabeling:
    """Biconnected components of ``g`` (bcc.py:147-196) on a CUDA device.

    ``beta``/``seed``/``block`` are accepted for drop-in compatibility; like
    in the reference they cannot change the result (the GPU forest does not
    use a clustering schedule).  ``device_outputs=True`` leaves the arrays on
    the device as torch tensors.
    """
    import torch

    t_start = time.perf_counter()
    _check_knobs(beta, block)
    g = _as_graph(g)
    n = g.n
    if n and 2 * n > (1 << 31) - 1:
        raise ValueError("tour positions need n <= 2**30")
    if g.m > (1 << 31) - 1:
        raise ValueError("slot count must fit 32-bit offsets on the device")
    if validate and g._dev is None:
        g.validate()
    if n == 0:
        t = StepTimings(total=time.perf_counter() - t_start)
        z = np.empty(0, np.int32)
        return BccLabeling(z, z.copy(), 0, 0, t, np.empty(0, np.int32), np.empty(0, np.uint8))
    if not torch.cuda.is_available():
        raise RuntimeError("fast_bcc needs a CUDA device (no CPU fallback)")
    dev = torch.device(device) if device is not None else (
        g._dev[0].device if g._dev is not None else torch.device("cuda", torch.cuda.current_device()))
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if g._dev is None and not device_outputs:
        stats, out, E = _host_session(g, dev).run(g)
        tim = _timings(stats)
        return BccLabeling(out["label"], out["head"], int(stats.num_bccs), int(stats.num_components), tim,
                           out["edge_label"][:E], out["is_ap"].view(np.bool_))
    if g._dev is None:  # device outputs from a host graph: upload, then the device path
        g = Graph.from_device(*[t.to(dev) for t in _pinned_or_numpy(g)])
    plan = _session(g, dev)
    stats = plan.run()
    res = plan.outputs()
    tim = _timings(stats)
    if device_outputs:  # plan buffers are reused by the next call: hand out copies
        res = {k: (None if v is None else v.clone()) for k, v in res.items()}
        return BccLabeling(res["label"], res["head"], int(stats.num_bccs), int(stats.num_components), tim,
                           res["edge_label"], res["is_ap"])
    out = _to_host(res, ("label", "head", "edge_label", "is_ap"))
    return BccLabeling(out["label"], out["head"], int(stats.num_bccs), int(stats.num_components), tim,
                       out["edge_label"], out["is_ap"].view(np.bool_))


def _timings(stats) -> StepTimings:
    ms = [float(x) for x in stats.stage_ms]
    return StepTimings(first_cc=ms[0] / 1e3, rooting=ms[1] / 1e3, tagging=ms[2] / 1e3,
                       last_cc=(ms[3] + ms[4]) / 1e3, total=float(stats.total_ms) / 1e3,
                       labelling=ms[5] / 1e3, stage_ms=tuple(ms))


def _pinned_or_numpy(g: Graph):
    import torch

    if g._pinned is not None:
        return g._pinned
    return torch.from_numpy(g.offsets), torch.from_numpy(g.edges.view(np.int32))


def extract_bccs(labeling: BccLabeling) -> list:
    """Vertex sets of all blocks, sorted, ordered by label (bcc.py:199-219)."""
    label = _host(labeling.label)
    head = _host(labeling.head)
    if label.size == 0:
        return []
    order = np.argsort(label, kind="stable")
    bounds = np.flatnonzero(np.diff(label[order])) + 1
    out = []
    for grp in np.split(order, bounds):
        h = int(head[int(label[grp[0]])])
        if h != -1:
            out.append(np.sort(np.append(grp, h)).astype(np.int64))
    return out


def articulation_points(labeling: BccLabeling) -> np.ndarray:
    """Sorted cut vertices (bcc.py:222-235); read from the device-computed
    flags when present."""
    if labeling.is_ap is not None:
        return np.flatnonzero(_host(labeling.is_ap)).astype(np.int64)
    label = _host(labeling.label)
    head = _host(labeling.head)
    n = label.size
    headed = np.bincount(head[head != -1], minlength=n)
    is_root = (label == np.arange(n, dtype=label.dtype)) & (head == -1)
    return np.flatnonzero(np.where(is_root, headed >= 2, headed >= 1)).astype(np.int64)
