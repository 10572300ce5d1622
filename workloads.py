"""Seeded synthetic workloads (BASELINE.json configs) -- harness, not product.

The paper's evaluation graphs are not available offline; these seeded
synthetic graphs with the BASELINE.json shapes stand in for them (SURVEY.md
§8(d)).  Each generator restates the construction the survey specifies so
the reference and the GPU consume the identical CSR; the committed golden
fixtures carry a digest of every generated CSR so a drift is caught.

All generators return a ``paper_2301_01356_b200.graphs.Graph``
(int64 offsets, uint32 targets -- the reference layout, graphs.py:43-58).
"""

import hashlib

import numpy as np

from paper_2301_01356_b200.graphs import Graph, symmetrize


def csr_digest(g: Graph) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.offsets, np.int64).tobytes())
    h.update(np.ascontiguousarray(g.edges, np.uint32).tobytes())
    return h.hexdigest()


def chain(n: int) -> Graph:
    """Path 0-1-...-(n-1) (same graph as reference gen_chain, graphs.py:236-241)."""
    i = np.arange(max(n - 1, 0), dtype=np.int64)
    return symmetrize(np.column_stack([i, i + 1]), n)


def grid(rows: int, cols: int, circular: bool = False, keep_prob: float = 1.0,
         seed: int = 0) -> Graph:
    """rows x cols lattice, optional wraparound, edges kept i.i.d. with
    ``keep_prob`` from PCG64(seed).  Candidate order (all horizontal, then all
    vertical, row-major) matches reference gen_grid (graphs.py:244-268) so the
    same seed keeps the same edges."""
    n = rows * cols
    ids = np.arange(n, dtype=np.int64).reshape(rows, cols)
    if circular:
        hs, hd = ids, np.roll(ids, -1, axis=1)
        vs, vd = ids, np.roll(ids, -1, axis=0)
    else:
        hs, hd = ids[:, :-1], ids[:, 1:]
        vs, vd = ids[:-1, :], ids[1:, :]
    u = np.concatenate([hs.ravel(), vs.ravel()])
    v = np.concatenate([hd.ravel(), vd.ravel()])
    if keep_prob < 1.0:
        keep = np.random.Generator(np.random.PCG64(seed)).random(u.size) < keep_prob
        u, v = u[keep], v[keep]
    return symmetrize(np.column_stack([u, v]), n)


def uniform(n: int = 1 << 20, avg: int = 8, seed: int = 0) -> Graph:
    """Config 2: avg*n endpoint pairs drawn uniformly from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pairs = rng.integers(0, n, size=(avg * n, 2), dtype=np.int64)
    return symmetrize(pairs, n)


def knn2d(npts: int = 10**6, k: int = 5, seed: int = 0) -> Graph:
    """Config 3: k nearest neighbours of uniform float32 points in the unit
    square (float64 KD-tree query with k+1, self dropped)."""
    from scipy.spatial import cKDTree

    pts = np.random.Generator(np.random.PCG64(seed)).random((npts, 2), dtype=np.float32)
    p64 = pts.astype(np.float64)
    _, idx = cKDTree(p64).query(p64, k=k + 1)
    src = np.repeat(np.arange(npts, dtype=np.int64), k + 1)
    dst = idx.reshape(-1).astype(np.int64)
    keep = src != dst
    return symmetrize(np.column_stack([src[keep], dst[keep]]), npts)


def rmat(scale: int = 25, edge_factor: int = 16, seed: int = 0,
         chunk: int = 1 << 24) -> Graph:
    """Config 5: RMAT with (a, b, c, d) quadrant probabilities, MSB first,
    chunks of 2^24 edges from one PCG64(seed) stream, no permutation."""
    n = 1 << scale
    total = edge_factor * n
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = []
    done = 0
    while done < total:
        k = min(chunk, total - done)
        u = np.zeros(k, np.int64)
        v = np.zeros(k, np.int64)
        for lvl in range(scale):
            r = rng.random(k)
            bit = np.int64(1) << np.int64(scale - 1 - lvl)
            # (a, b, c, d) = (0.57, 0.19, 0.19, 0.05): cumulative 0.57/0.76/0.95
            row = r >= 0.76                                 # quadrant c or d
            col = ((r >= 0.57) & (r < 0.76)) | (r >= 0.95)  # quadrant b or d
            u |= np.where(row, bit, 0)
            v |= np.where(col, bit, 0)
        parts.append(np.column_stack([u, v]))
        done += k
    return symmetrize(np.concatenate(parts), n)


# ---------------------------------------------------------------------------
# Large configs on the device: the same pairs (same PCG64 draws, same
# candidate order) are built on the host, then symmetrised on the GPU
# (sort + unique of packed 64-bit keys) -- the host numpy sort of 4e8-1e9 keys
# dominates otherwise.  The resulting CSR is identical to symmetrize()'s.
# ---------------------------------------------------------------------------
def _pairs(name):
    if name == "4a":
        rows, cols, keep_prob = 10**4, 10**4, 1.0
    elif name == "4b":
        rows, cols, keep_prob = 10**3, 10**5, 0.6
    elif name == "4c":
        i = np.arange(10**8 - 1, dtype=np.int64)
        return i, i + 1, 10**8
    elif name == "5":
        return _rmat_pairs() + (1 << 25,)
    else:
        raise KeyError(name)
    n = rows * cols
    ids = np.arange(n, dtype=np.int64).reshape(rows, cols)
    u = np.concatenate([ids.ravel(), ids.ravel()])
    v = np.concatenate([np.roll(ids, -1, axis=1).ravel(), np.roll(ids, -1, axis=0).ravel()])
    if keep_prob < 1.0:
        keep = np.random.Generator(np.random.PCG64(0)).random(u.size) < keep_prob
        u, v = u[keep], v[keep]
    return u, v, n


def _rmat_pairs(scale=25, edge_factor=16, seed=0, chunk=1 << 24):
    n = 1 << scale
    total = edge_factor * n
    rng = np.random.Generator(np.random.PCG64(seed))
    us, vs = [], []
    done = 0
    while done < total:
        k = min(chunk, total - done)
        u = np.zeros(k, np.int64)
        v = np.zeros(k, np.int64)
        for lvl in range(scale):
            r = rng.random(k)
            bit = np.int64(1) << np.int64(scale - 1 - lvl)
            u |= np.where(r >= 0.76, bit, 0)
            v |= np.where(((r >= 0.57) & (r < 0.76)) | (r >= 0.95), bit, 0)
        us.append(u)
        vs.append(v)
        done += k
    return np.concatenate(us), np.concatenate(vs)


def _rmat_lib():
    """tools/librmat_pcg.so (built here on first use when nvcc is present)."""
    import ctypes
    import subprocess
    from pathlib import Path

    tools = Path(__file__).resolve().parent / "tools"
    so = tools / "librmat_pcg.so"
    src = tools / "rmat_pcg.cu"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                        "-fPIC", "-cudart", "static", "-o", str(so), str(src)], check=True)
    lib = ctypes.CDLL(str(so))
    lib.rmat_pairs_chunk.restype = ctypes.c_int
    lib.rmat_pairs_chunk.argtypes = [ctypes.c_uint64] * 5 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                             ctypes.c_void_p, ctypes.c_void_p]
    return lib


def rmat_pairs_device(scale=25, edge_factor=16, seed=0, chunk=1 << 24, device="cuda"):
    """_rmat_pairs on the GPU, bit-identical (same PCG64 stream, jumped to each
    chunk/level offset; tools/rmat_pcg.cu).  Returns int64 device tensors."""
    import ctypes

    import torch

    lib = _rmat_lib()
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    total = edge_factor * (1 << scale)
    u = torch.empty(total, dtype=torch.int64, device=device)
    v = torch.empty(total, dtype=torch.int64, device=device)
    stream = torch.cuda.current_stream(u.device).cuda_stream
    done = 0
    while done < total:
        k = min(chunk, total - done)
        rc = lib.rmat_pairs_chunk(s >> 64, s & m64, inc >> 64, inc & m64, done * scale, k, scale,
                                  u[done:].data_ptr(), v[done:].data_ptr(), ctypes.c_void_p(stream))
        if rc:
            raise RuntimeError(f"rmat kernel failed ({rc})")
        done += k
    return u, v


def symmetrize_device(u, v, n, device="cuda"):
    """symmetrize() on the GPU; returns (offsets int64[n+1], edges int32[m]) tensors."""
    import torch

    u = torch.as_tensor(u).to(device)
    v = torch.as_tensor(v).to(device)
    keep = u != v
    u, v = u[keep], v[keep]
    keys = torch.cat([(u << 32) | v, (v << 32) | u])
    del u, v, keep
    keys = torch.unique(keys, sorted=True)
    src = keys >> 32
    dst = (keys & 0xFFFFFFFF).to(torch.int32)
    del keys
    off = torch.zeros(n + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    return off, dst


def make_device(name, device="cuda"):
    """Config ``name`` as device tensors (offsets int64, edges int32)."""
    if name in ("1", "2", "3"):
        import torch

        g = make(name)
        return (torch.from_numpy(g.offsets).to(device), torch.from_numpy(g.edges.view(np.int32)).to(device))
    if name == "5":  # the host generator takes minutes; the GPU one is bit-identical
        u, v = rmat_pairs_device(device=device)
        return symmetrize_device(u, v, 1 << 25, device)
    u, v, n = _pairs(name)
    return symmetrize_device(u, v, n, device)


# ---------------------------------------------------------------------------
# Host CSR in seconds (tools/hostgen.c, OpenMP): the same PCG64 draws and the
# same symmetrize() result as rmat() above, which takes minutes in numpy at
# scale 25.  Bit-identity: tests/test_hostgen.py (small scales, vs rmat()) and
# the committed config-5 CSR digest (tests/golden/configs.json).
# ---------------------------------------------------------------------------
def _hostgen_lib():
    import ctypes
    import subprocess
    from pathlib import Path

    tools = Path(__file__).resolve().parent / "tools"
    so = tools / "libhostgen.so"
    src = tools / "hostgen.c"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        import os

        tmp = so.with_suffix(f".so.{os.getpid()}.tmp")  # concurrent ranks may build at once
        subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-o", str(tmp), str(src)],
                       check=True)
        tmp.replace(so)
    lib = ctypes.CDLL(str(so))
    u64, i64, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
    lib.hg_rmat_pairs.restype = ctypes.c_int
    lib.hg_rmat_pairs.argtypes = [u64, u64, u64, u64, ctypes.c_int, i64, i64, vp, vp]
    lib.hg_symmetrize.restype = i64
    lib.hg_symmetrize.argtypes = [vp, vp, i64, i64, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    lib.hg_free.restype = None
    lib.hg_free.argtypes = [vp]
    lib.hg_num_threads.restype = ctypes.c_int
    return lib


def _owned(lib, ptr, count, ctype, dtype):
    """numpy view of a malloc'd buffer, freed with the array."""
    import ctypes
    import weakref

    if count == 0:
        lib.hg_free(ptr)
        return np.empty(0, dtype)
    arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), shape=(count,)).view(dtype)
    weakref.finalize(arr, lib.hg_free, ptr)
    return arr


def symmetrize_host(u, v, n: int) -> Graph:
    """symmetrize() for uint32 pair arrays, on all host cores."""
    import ctypes

    lib = _hostgen_lib()
    u = np.ascontiguousarray(u, np.uint32)
    v = np.ascontiguousarray(v, np.uint32)
    po, pe = ctypes.c_void_p(), ctypes.c_void_p()
    m = lib.hg_symmetrize(u.ctypes.data, v.ctypes.data, u.size, n, ctypes.byref(po), ctypes.byref(pe))
    if m < 0:
        raise ValueError("edge endpoint out of range (or out of memory)")
    off = _owned(lib, po.value, n + 1, ctypes.c_int64, np.int64)
    edges = _owned(lib, pe.value, m, ctypes.c_uint32, np.uint32)
    return Graph(off, edges)


def rmat_fast(scale: int = 25, edge_factor: int = 16, seed: int = 0, chunk: int = 1 << 24) -> Graph:
    """rmat() on all host cores (tools/hostgen.c): same pairs, same CSR."""
    lib = _hostgen_lib()
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    total = edge_factor * (1 << scale)
    u = np.empty(total, np.uint32)
    v = np.empty(total, np.uint32)
    rc = lib.hg_rmat_pairs(s >> 64, s & m64, inc >> 64, inc & m64, scale, total, chunk, u.ctypes.data, v.ctypes.data)
    if rc:
        raise RuntimeError("hg_rmat_pairs failed")
    g = symmetrize_host(u, v, 1 << scale)
    del u, v
    return g


CONFIGS = {
    "1": ("torus 300x300 p=0.6", lambda: grid(300, 300, circular=True, keep_prob=0.6, seed=0)),
    "2": ("uniform n=2^20 m=8n", lambda: uniform()),
    "3": ("2-D kNN 10^6 k=5", lambda: knn2d()),
    # the same pairs as grid() / chain() (workloads._pairs), symmetrised on the host cores
    "4a": ("torus 10^4x10^4", lambda: symmetrize_host(*_pairs("4a"))),
    "4b": ("torus 10^3x10^5 p=0.6", lambda: symmetrize_host(*_pairs("4b"))),
    "4c": ("chain 10^8", lambda: symmetrize_host(*_pairs("4c"))),
    "5": ("RMAT scale 25 ef 16", lambda: rmat_fast()),
}


def make(name: str) -> Graph:
    return CONFIGS[name][1]()
