// labelling.cu -- Stage 6: block heads, BCC count, articulation flags and
// canonical per-edge labels.
//
// Replaces _component_heads (bcc.py:129-144, sequential packed-min over all
// vertices), num_bccs (bcc.py:192), articulation_points (bcc.py:222-235,
// numpy bincount) and adds the per-edge labelling the reference leaves
// implicit (rule: bcc.py:24-27; canonical numbering: tv_skeleton,
// baselines.py:251-257, 297-303).
//
// B200 design:
//  * heads without a min pass: by the BCC tree-connectivity lemma
//     a block is tree-connected through its head, so
//    every member v of skeleton component l with label[parent[v]] != l is a
//    tree child of the head: all of them would store the same head[l] =
//    parent[v] (no packed-min over first[] like the reference); the one
//    member whose CAS claims head[l] also counts the block and bumps the
//    head's saturating headed-count.
//  * edge ids: CUB scan of the upper degrees deg - nlow (nlow counted by the
//    Stage-3 gather pass over the same arcs).
//  * per-block minimum edge id: only the arcs of each block's minimum vertex
//    can hold it (see EdgeBlockVisitor), so only those rows issue atomicMin
//    -- one uncontended address per block instead of an atomic per run
//    (config 2's giant block has 8.4 M edges, RMAT hubs change block on
//    almost every arc).
#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

// Every member of component l whose tree parent lies outside l has that
// parent equal to the block's head (all such members are children of the
// head: the block is tree-connected through its head).
// The first of them to CAS head[l] from -1 also counts the block and bumps
// the head's saturating headed-count for the articulation rule of
// bcc.py:229-234 -- heads and the block count in one pass.
// Label of the giant skeleton component (Stage 5's sampled giant root, now
// under its final label), or -1.  Every kernel recomputes it from the same
// two words, so the bitmap and its readers agree.
__device__ __forceinline__ int giant_label(const int* label, const Scalars* sc) {
  const int gi = sc->giant;
  return gi >= 0 ? __ldg(label + gi) : -1;
}

__global__ void k_heads(int n, const int4* __restrict__ rec, const int* __restrict__ label, int* head, int* cnt,
                        Scalars* sc) {
  pdl_enter();
  int blocks = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int l = __ldg(label + v);
    const int p = __ldg(&rec[v].z);
    // (read first: the children of one head inside one component -- RMAT
    // hubs -- would otherwise serialise their CAS on one word)
    if (p >= 0 && l != __ldg(label + p) && ld_relaxed(head + l) == -1 && atomicCAS(head + l, -1, p) == -1) {
      blocks++;
      if (ld_relaxed(cnt + p) < 2) atomicAdd(cnt + p, 1);
    }
  }
  block_count_add(&sc->nbccs, blocks);
}

__global__ void k_ap(int n, const int* __restrict__ label, const int* __restrict__ head,
                     const int* __restrict__ cnt, uint8_t* __restrict__ is_ap) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    bool root = (__ldg(label + v) == v) && (__ldg(head + v) == -1);
    int c = __ldg(cnt + v);
    is_ap[v] = root ? (c >= 2) : (c >= 1);
  }
}

// ---------------------------------------------------------------------------
// Per-edge labels.  edge_label[e] = minimum edge id of e's block, e = rank of
// the upper arc (u -> w, u < w) in CSR order.
//
// Almost every edge of a large graph lies in the block of the giant skeleton
// component G (RMAT: 99.1 %, config 2: ~100 %), and a G-G edge's label is the
// block minimum bmin[G] -- known before the edge pass:
//  1. k_giant_min: bmin[G] = the first upper arc of u0 = min(G, head[G]) (the
//     block's minimum vertex; edge ids grow with the smaller endpoint) whose
//     block is G -- one warp, usually the first arc.
//  2. k_edge_fill: edge_label[0..E) = bmin[G], a streaming store -- no
//     adjacency read, no label gather.
//  3. k_edge_fix: over the rows, dropping G's rows by their label before any
//     adjacency load.  Every upper arc of a non-G row gets its block by the
//     rule of bcc.py:24-27 (label[w] gathered): G -> the final bmin[G],
//     otherwise blk | MARK.  An edge (x, v), x < v, between a G row x and a
//     non-G row v is G's unless v's component hangs off x (x =
//     head[label[v]]); the row flags that case (sreq[v]) for
//  4. k_edge_search: binary search of v in x's upper arcs (spos[v] = e), the
//     requests packed 32 per warp -- inline, the ~10 dependent loads
//     serialised whole warps of the row pass.  Also the rows over 8192 arcs that k_edge_fix
//     deferred (a non-giant RMAT hub: 638k arcs), over the whole grid.
//     Per-block minima: atomicMin from the block's minimum-vertex row only
//     (one uncontended address per block; one atomic per run of a block).
//  5. k_edge_final: MARKed entries -> bmin[blk], over the non-G rows again
//     (and the searched positions, and the deferred rows).
// No global counters besides the rare deferred-row list: a list append per
// rewritten edge serialised on one L2 address (RMAT: 4.2 M, ~2 ms).
// With no large giant (Stage 5's sample put < 1/4 of its points in one
// component: tori with many blocks, the chain) G = -1: no fill, every row is
// processed, blocks are written unmarked and k_edge_final maps all E.
// ---------------------------------------------------------------------------
constexpr int kEdgeMark = (int)0x80000000;
constexpr int kEdgeSuperRow = 2048;

__device__ __forceinline__ int big_giant(const int* label, const Scalars* sc) {
  return sc->giant_cnt >= 256 ? giant_label(label, sc) : -1;
}

// first upper arc of row u: off[u] + nlow[u] (rows sorted, no self-loops);
// edge id of upper arc a of row u: uoff[u] + (a - first upper arc)
__global__ void k_giant_min(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                            const int* __restrict__ label, const int* __restrict__ head,
                            UpOff uoff, const int* __restrict__ nlow, int* bmin, const Scalars* sc) {
  pdl_enter();
  const int G = big_giant(label, sc);
  if (G < 0) return;
  const int lane = threadIdx.x;
  const int h = __ldg(head + G);
  const int u0 = (h >= 0 && h < G) ? h : G;
  const int lu = __ldg(label + u0);
  const int64_t a0 = __ldg(off + u0) + __ldg(nlow + u0), re = __ldg(off + u0 + 1);
  for (int64_t a = a0 + lane; a - lane < re; a += 32) {
    bool hit = false;
    if (a < re) {
      const int w = (int)__ldg(adj + a);
      const int lw = __ldg(label + w);
      const int blk = lu == lw ? lu : (__ldg(head + lw) == u0 ? lw : lu);
      hit = blk == G;
    }
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (b) {
      if (lane == __ffs(b) - 1) bmin[G] = uoff.at(u0) + (int)(a - a0);
      return;
    }
  }
}

__global__ void k_edge_fill(int n, const int* __restrict__ label, UpOff uoff,
                            const int* __restrict__ bmin, int* __restrict__ edge_label, Scalars* sc) {
  pdl_enter();
  const int E = uoff.at(n);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->num_edges = E;
  const int G = big_giant(label, sc);
  if (G < 0) return;
  const int val = __ldg(bmin + G);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(edge_label) & 15) == 0) {
    const int64_t nv = E / 4;
    const int4 v4 = make_int4(val, val, val, val);
    for (int64_t i = tid; i < nv; i += stride) __stcs(reinterpret_cast<int4*>(edge_label) + i, v4);
    for (int64_t e = 4 * nv + tid; e < E; e += stride) edge_label[e] = val;
  } else {
    for (int64_t e = tid; e < E; e += stride) edge_label[e] = val;
  }
}

// Per-thread state of the non-giant row passes.  The arcs one thread visits
// come in increasing order, so per-block minima go out as one atomicMin per
// run of a block.
struct EdgeFix {
  const int64_t* off;
  const uint32_t* adj;
  const int* label;
  const int* head;
  UpOff uoff;
  const int* nlow;
  int* edge_label;
  int* bmin;
  int G, valG;
  int run_blk, run_min;

  __device__ __forceinline__ void init(const int64_t* o, const uint32_t* a, const int* lb, const int* hd,
                                       UpOff uo, const int* nl, int* el, int* bm, const Scalars* sc) {
    off = o;
    adj = a;
    label = lb;
    head = hd;
    uoff = uo;
    nlow = nl;
    edge_label = el;
    bmin = bm;
    G = big_giant(lb, sc);
    valG = G >= 0 ? __ldg(bm + G) : 0;  // final (k_giant_min)
    run_blk = -1;
    run_min = 0;
  }
  __device__ __forceinline__ void flush() {
    if (run_blk >= 0) atomicMin(bmin + run_blk, run_min);
    run_blk = -1;
  }
  __device__ __forceinline__ void mark(int e, int blk) {
    if (G < 0) edge_label[e] = blk;           // no giant: k_edge_final maps every edge
    else if (blk == G) edge_label[e] = valG;  // final already
    else edge_label[e] = blk | kEdgeMark;
  }
  // row words: hl = head of v's block, row_u0 = v is its block's minimum
  // vertex (v a label below its head), ebase: edge id of upper arc a = ebase + a
  __device__ __forceinline__ void row_words(int v, int lu, int64_t rs, int& hl, bool& row_u0, int& ebase) const {
    hl = __ldg(head + lu);
    const int hv = v == lu ? hl : -1;  // head[v] >= 0 only at label vertices
    row_u0 = hv >= 0 && v < hv;
    ebase = uoff.at(v) - (int)(rs + __ldg(nlow + v));
  }
  // one arc of non-giant row v; returns true for the lower arc to the head of
  // v's block when that head is in G (the edge sits in the head's G row)
  __device__ __forceinline__ bool arc(int v, int lu, int hl, bool row_u0, int ebase, int64_t a, int x) {
    if (x > v) {  // upper arc: this row holds the edge
      const int lw = __ldg(label + x);
      int blk;
      bool mine;
      if (lu == lw) {
        blk = lu;
        mine = row_u0;
      } else if (__ldg(head + lw) == v) {  // x's component hangs off v: its block
        blk = lw;
        mine = v < lw;
      } else {
        blk = lu;
        mine = row_u0;
      }
      const int e = ebase + (int)a;
      mark(e, blk);
      if (mine && blk != run_blk && blk != G) {
        flush();
        run_blk = blk;
        run_min = e;
      }
      return false;
    }
    return G >= 0 && x == hl && __ldg(label + x) == G;
  }
  // that edge: binary search of v in x's sorted upper arcs; it belongs to
  // v's block
  __device__ __forceinline__ int fix_lower(int v, int lu, int x) {
    int64_t lo = __ldg(off + x) + __ldg(nlow + x), hi = __ldg(off + x + 1);
    const int64_t ub = lo;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int)__ldg(adj + mid) < v) lo = mid + 1; else hi = mid;
    }
    const int e = uoff.at(x) + (int)(lo - ub);
    mark(e, lu);
    if (x < lu) atomicMin(bmin + lu, e);
    return e;
  }
};

// Row-filtered: each warp reads the labels and offsets of 32 consecutive
// rows (coalesced) and drops the giant's rows and empty rows before touching
// any adjacency -- on RMAT that is all but ~4 M of the 33.5 M rows.  Rows of
// <= 32 arcs are handled by their own lane, longer ones by the whole warp,
// rows over kEdgeSuperRow arcs are deferred to k_edge_search (whole grid).
// sreq bit v (one 32-bit word per warp step, every word written): v's
// lower-arc fix is k_edge_search's.  (A bitmap: 4 bytes per 32 rows to write
// here and to read in the two passes that follow, not 4 per row.)
__global__ void __launch_bounds__(256) k_edge_fix(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  int n, const int* __restrict__ label, const int* __restrict__ head,
                                                  UpOff uoff, const int* __restrict__ nlow,
                                                  int* edge_label, int* bmin, LongRows heavy,
                                                  unsigned* __restrict__ sreq, Scalars* sc) {
  pdl_enter();
  EdgeFix f;
  f.init(off, adj, label, head, uoff, nlow, edge_label, bmin, sc);
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += warps * 32) {
    const int v = (int)base + lane;
    int64_t rs = 0, re = 0;
    int lu = f.G;
    if (v < n) {
      lu = __ldg(label + v);
      if (lu != f.G) {
        rs = __ldg(off + v);
        re = __ldg(off + v + 1);
      }
    }
    if (re - rs > kEdgeSuperRow) {
      heavy.defer(v, re - rs);
      rs = re = 0;
    }
    bool req = false;
    const bool coop = re - rs > 32;
    if (!coop && re > rs) {
      int hl, ebase;
      bool row_u0;
      f.row_words(v, lu, rs, hl, row_u0, ebase);
      for (int64_t a = rs; a < re; a++) req |= f.arc(v, lu, hl, row_u0, ebase, a, (int)__ldg(adj + a));
    }
    unsigned hb = __ballot_sync(0xffffffffu, coop);
    while (hb) {
      const int src = __ffs(hb) - 1;
      hb &= hb - 1;
      const int hv = __shfl_sync(0xffffffffu, v, src), hlu = __shfl_sync(0xffffffffu, lu, src);
      const int64_t hs = __shfl_sync(0xffffffffu, rs, src), he = __shfl_sync(0xffffffffu, re, src);
      int hl, ebase;
      bool row_u0;
      f.row_words(hv, hlu, hs, hl, row_u0, ebase);
      bool r = false;
      for (int64_t a = hs + lane; a < he; a += 32) r |= f.arc(hv, hlu, hl, row_u0, ebase, a, (int)__ldg(adj + a));
      f.flush();  // (the lanes' runs interleave across the row)
      r = __any_sync(0xffffffffu, r);
      if (lane == src) req = r;
    }
    const unsigned rb = __ballot_sync(0xffffffffu, req);
    if (lane == 0) sreq[base >> 5] = rb;
  }
  f.flush();
}

// The deferred work: (a) rows over kEdgeSuperRow arcs (LongRows: a CTA per
// row, the whole grid per row over kMegaRow; their one lower-arc fix
// inline), (b) the lower-arc fixes k_edge_fix flagged, 32 per warp.
// Disjoint rows: no ordering between the two.
__global__ void __launch_bounds__(256) k_edge_search(const int64_t* __restrict__ off,
                                                     const uint32_t* __restrict__ adj, int n,
                                                     const int* __restrict__ label, const int* __restrict__ head,
                                                     UpOff uoff, const int* __restrict__ nlow,
                                                     int* edge_label, int* bmin, LongRows heavy,
                                                     unsigned* sreq, int* spos, Scalars* sc) {
  pdl_enter();
  EdgeFix f;
  f.init(off, adj, label, head, uoff, nlow, edge_label, bmin, sc);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  int lu = 0, hl = 0, ebase = 0;
  bool row_u0 = false;
  heavy.visit(
      off,
      [&](int v, int64_t rs) {
        f.flush();  // (a new row: the previous row's run ends)
        lu = __ldg(label + v);
        f.row_words(v, lu, rs, hl, row_u0, ebase);
      },
      [&](int v, int64_t a) {
        if (f.arc(v, lu, hl, row_u0, ebase, a, (int)__ldg(adj + a))) {
          spos[v] = f.fix_lower(v, lu, hl);  // (k_edge_final maps it; a repeat below is idempotent)
          atomicOr(sreq + (v >> 5), 1u << (v & 31));
        }
      });
  f.flush();
  if (f.G < 0) return;  // (no lower-arc fixes without a giant)
  // Warp-compacted: the rows with a request (RMAT: ~1 in 10) are packed into
  // a per-warp queue and searched 32 at a time.  One request per lane of a
  // row-strided loop left most lanes idle through every ~20-step dependent
  // search, so the pass took as many search latencies as there were warps
  // with any request (config 5: 1.18 ms).
  __shared__ int squeue[256 / 32][64];
  const int lane = threadIdx.x & 31;
  int* wq = squeue[threadIdx.x >> 5];
  int cnt = 0;  // warp-uniform
  auto search = [&](int v) {
    const int lv = __ldg(label + v);
    spos[v] = f.fix_lower(v, lv, __ldg(head + lv));
  };
  const int64_t warps = stride >> 5;
  for (int64_t base = (tid >> 5) * 32; base < n; base += warps * 32) {
    const int64_t v = base + lane;
    const bool r = v < n && ((sreq[base >> 5] >> lane) & 1u);  // (plain load: the deferred rows above set theirs)
    const unsigned b = __ballot_sync(0xffffffffu, r);
    if (r) wq[cnt + __popc(b & ((1u << lane) - 1))] = (int)v;
    cnt += __popc(b);
    __syncwarp();
    if (cnt >= 32) {
      cnt -= 32;
      const int sv = wq[cnt + lane];
      __syncwarp();  // (read before the next appends overwrite the slot)
      search(sv);
    }
  }
  if (lane < cnt) search(wq[lane]);
}

__device__ __forceinline__ void edge_map(int* edge_label, const int* bmin, int e) {
  const int b = edge_label[e];
  if (b < 0) edge_label[e] = __ldg(bmin + (b & ~kEdgeMark));
}

// MARKed entries -> bmin[blk].  Giant mode: the non-G rows' upper arcs, the
// searched positions and the deferred rows; otherwise every edge (16-byte
// streaming loads and stores).
__global__ void __launch_bounds__(256) k_edge_final(const int64_t* __restrict__ off, int n,
                                                    const int* __restrict__ label, UpOff uoff,
                                                    const int* __restrict__ nlow, int* edge_label,
                                                    const int* __restrict__ bmin, LongRows heavy,
                                                    const unsigned* __restrict__ sreq, const int* __restrict__ spos,
                                                    const Scalars* sc) {
  pdl_enter();
  const int E = uoff.at(n);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int G = big_giant(label, sc);
  if (G >= 0) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = stride >> 5;
    for (int64_t base = (tid >> 5) * 32; base < n; base += warps * 32) {
      const int v = (int)base + lane;
      int e0 = 0, e1 = 0;
      if (v < n) {
        if (__ldg(label + v) != G) {
          e0 = uoff.at(v);
          e1 = uoff.at(v + 1);
          if (__ldg(off + v + 1) - __ldg(off + v) > kEdgeSuperRow) e1 = e0;  // deferred row: below
        }
        if ((__ldg(sreq + (base >> 5)) >> lane) & 1u) edge_map(edge_label, bmin, __ldg(spos + v));
      }
      const bool coop = e1 - e0 > 32;
      if (!coop)
        for (int e = e0; e < e1; e++) edge_map(edge_label, bmin, e);
      unsigned hb = __ballot_sync(0xffffffffu, coop);
      while (hb) {
        const int src = __ffs(hb) - 1;
        hb &= hb - 1;
        const int h0 = __shfl_sync(0xffffffffu, e0, src), h1 = __shfl_sync(0xffffffffu, e1, src);
        for (int e = h0 + lane; e < h1; e += 32) edge_map(edge_label, bmin, e);
      }
    }
    int eb = 0;  // (the deferred rows' upper arcs: edge ids eb + a)
    heavy.visit(
        off, [&](int v, int64_t rs) { eb = uoff.at(v) - (int)(rs + __ldg(nlow + v)); },
        [&](int v, int64_t a) {
          const int e = eb + (int)a;
          if (e >= uoff.at(v)) edge_map(edge_label, bmin, e);
        });
    return;
  }
  if ((reinterpret_cast<uintptr_t>(edge_label) & 15) == 0) {
    const int64_t nv = E / 4;
    int4* e4 = reinterpret_cast<int4*>(edge_label);
    for (int64_t i = tid; i < nv; i += stride) {
      int4 b = __ldcs(e4 + i);
      b.x = __ldg(bmin + b.x);
      b.y = __ldg(bmin + b.y);
      b.z = __ldg(bmin + b.z);
      b.w = __ldg(bmin + b.w);
      __stcs(e4 + i, b);
    }
    for (int64_t e = 4 * nv + tid; e < E; e += stride) edge_label[e] = __ldg(bmin + edge_label[e]);
  } else {
    for (int64_t e = tid; e < E; e += stride) edge_label[e] = __ldg(bmin + edge_label[e]);
  }
}

__global__ void k_set_edges(UpOff uoff, int n, Scalars* sc) {
  pdl_enter(); sc->num_edges = uoff.at(n); }

void stage6_labelling(const Graph& g, const int4* rec, const int* label, int* head, uint8_t* is_ap,
                      int* edge_label, int* cnt, int* uoff, int* nlow, int* bmin, int* heavy, int* sreq, int* spos,
                      void* cub_tmp, size_t cub_bytes, Scalars* sc, cudaStream_t st, cudaEvent_t heads_done,
                      const Side* side) {
  const int n = g.n;
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  // head = -1, cnt = 0, bmin = INF were initialised by the stage-4 kernel
  launch(k_heads, gv, B, 0, st, n, rec, label, head, cnt, sc);
  note(K_HEADS);
  if (side) {  // articulation flags beside the edge pass; the scan ran beside Stages 3-5
    cudaEventRecord(side->ev[2], st);
    cudaStreamWaitEvent(side->s, side->ev[2], 0);
    if (is_ap) {
      launch(k_ap, gv, B, 0, side->s, n, label, head, cnt, is_ap);
      note(K_AP);
    }
    if (heads_done) cudaEventRecord(heads_done, side->s);  // head / is_ap final: their D2H may start
    cudaEventRecord(side->ev[3], side->s);
    cudaStreamWaitEvent(st, side->ev[1], 0);  // uoff
  } else {
    if (is_ap) {
      launch(k_ap, gv, B, 0, st, n, label, head, cnt, is_ap);
      note(K_AP);
    }
    if (heads_done) cudaEventRecord(heads_done, st);  // head / is_ap final: their D2H may start
    // edge ids: exclusive scan of the upper degrees deg - nlow (nlow counted
    // by the Stage-3 gather) -> uoff (uoff[n] = E)
    scan_upper_degrees(g.off, nlow, n, uoff, cub_tmp, cub_bytes, st);
    note(K_SCAN);
  }
  // (edge ids: the tile-local prefixes in uoff plus the tile prefixes scan_upper_degrees left in cub_tmp)
  const UpOff up{uoff, reinterpret_cast<const unsigned long long*>(cub_tmp), n, (n + kUpTile - 1) / kUpTile};
  if (!edge_label || g.m == 0) {
    launch(k_set_edges, 1, 1, 0, st, up, n, sc);
    note(K_SET_EDGES);
  } else {
    launch(k_giant_min, 1, 32, 0, st, g.off, g.adj, label, head, up, (const int*)nlow, bmin, (const Scalars*)sc);
    note(K_GIANT_MIN);
    launch(k_edge_fill, grid_for(g.m / 8 + 1, B), B, 0, st, n, label, up, (const int*)bmin, edge_label, sc);
    note(K_EDGE_FILL);
    LongRows hv{heavy, n, &sc->eheavy, &sc->emega};  // (a dead n-int Stage-2 array, see api.cu)
    launch(k_edge_fix, grid_for(n, B, 32), B, 0, st, g.off, g.adj, n, label, (const int*)head, up, (const int*)nlow, edge_label, bmin, hv,
           reinterpret_cast<unsigned*>(sreq), sc);
    note(K_EDGE_BLOCKS);
    launch(k_edge_search, grid_for(n, B, 32), B, 0, st, g.off, g.adj, n, label, (const int*)head, up, (const int*)nlow, edge_label, bmin,
           hv, reinterpret_cast<unsigned*>(sreq), spos, sc);
    note(K_EDGE_SEARCH);
    launch(k_edge_final, grid_for(n, B, 32), B, 0, st, g.off, n, label, up, (const int*)nlow, edge_label, (const int*)bmin, hv,
           (const unsigned*)sreq, (const int*)spos, (const Scalars*)sc);
    note(K_EDGE_FINAL);
  }
  if (side) cudaStreamWaitEvent(st, side->ev[3], 0);  // join the articulation flags
}

// ---------------------------------------------------------------------------
// intermediate exports (parity rungs 1-4)
// ---------------------------------------------------------------------------
__global__ void k_export(int n, const int4* __restrict__ rec, const int4* __restrict__ AP, int* parent, int* first,
                         int* last, int* w1, int* w2, uint8_t* fence, const int* tlen) {
  pdl_enter();
  const int N = tlen ? *tlen : 2 * n;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int4 r = rec[v];
    if (parent) parent[v] = r.z;
    if (first) first[v] = r.x;
    if (last) last[v] = r.y;
    if (fence) fence[v] = (uint8_t)r.w;
    if (w1 || w2) {
      // (a detached root has no AP entry: w1 = w2 = first)
      int4 a = r.x < N ? AP[r.x] : make_int4(r.x, r.x, 0, 0);
      if (w1) w1[v] = a.x;
      if (w2) w2[v] = a.y;
    }
  }
}

void export_debug(const Graph& g, const int2* fe, const int4* rec, const int4* AP, int* forest, int* parent,
                  int* first, int* last, int* w1, int* w2, uint8_t* fence, cudaStream_t st, const int* tour_len) {
  if (forest) cudaMemcpyAsync(forest, fe, sizeof(int2) * g.n, cudaMemcpyDeviceToDevice, st);
  if (parent || first || last || w1 || w2 || fence)
    launch(k_export, grid_for(g.n, 256), 256, 0, st, g.n, rec, AP, parent, first, last, w1, w2, fence, tour_len);
}

}  // namespace fbcc
