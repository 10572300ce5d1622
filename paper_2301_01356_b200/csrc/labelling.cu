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
                        uint32_t* __restrict__ gbits, Scalars* sc) {
  pdl_enter();
  const int G = giant_label(label, sc);
  const int lane = threadIdx.x & 31;
  int blocks = 0;
  // warp-uniform trip count: the warp also writes one word of the giant bitmap
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)base + lane;
    int l = -1;
    if (v < n) {
      l = __ldg(label + v);
      int p = __ldg(&rec[v].z);
      // (read first: the children of one head inside one component -- RMAT
      // hubs -- would otherwise serialise their CAS on one word)
      if (p >= 0 && l != __ldg(label + p) && ld_relaxed(head + l) == -1 && atomicCAS(head + l, -1, p) == -1) {
        blocks++;
        if (ld_relaxed(cnt + p) < 2) atomicAdd(cnt + p, 1);
      }
    }
    const unsigned bits = __ballot_sync(0xffffffffu, l == G && G >= 0);
    if (lane == 0) gbits[base >> 5] = bits;
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

// Per-block minimum edge id without a per-run atomic: edge ids grow with the
// row (u < w, CSR order), so a block's minimum edge is the FIRST upper arc in
// the row of the block's minimum vertex u0 = min(l, head[l]) (every block
// vertex has a block edge; u0's all go upward).  Only arcs of u0 rows feed
// bmin: for an arc in its own component's block (blk == label[v]) that means
// v == label[v] < head[label[v]]; for an arc into a child block headed by v
// (blk == label[w]) it means v < label[w].  Those atomics hit distinct
// addresses (one row per block) -- the old run-length scheme issued a
// read + atomicMin per block change, i.e. per arc of an RMAT hub.
// kBits: when the giant holds at least a quarter of Stage 5's 1024 vertex
// samples (RMAT: ~half -- its other half is isolated vertices), the
// giant-component bitmap (k_heads) is read first, from global memory (n/8
// bytes: 4 MB on RMAT, 32x denser than label[] and mostly cache-resident;
// RMAT 4.57 -> 4.12 ms) and label[w] is gathered only for arcs leaving the
// giant; a small giant (config 4b: 24 M blocks) keeps the label gather.
template <bool kBits>
struct EdgeBlockVisitor {
  const int64_t* off;
  const int* label;
  const int* head;
  const int* uoff;
  const int* nlow;
  const uint32_t* gbits;
  int G;
  int* eblk;
  int* bmin;
  int lu, ebase;
  bool row_u0;
  int run_blk, run_min;
  int pl[kBits ? 1 : kItems];
  unsigned ing;  // kBits: bit i = arc i's target is in the giant
  // label[w] (or its giant bit) for every arc that can be an upper arc (w > first row of the chunk)
  __device__ __forceinline__ void prefetch(int v0, const uint32_t* w, int cnt) {
    if (kBits) {
      ing = 0;
#pragma unroll
      for (int i = 0; i < kItems; i++)
        if (i < cnt && (int)w[i] > v0) ing |= ((__ldg(gbits + (w[i] >> 5)) >> (w[i] & 31)) & 1u) << i;
    } else {
#pragma unroll
      for (int i = 0; i < kItems; i++) pl[kBits ? 0 : i] = (i < cnt && (int)w[i] > v0) ? __ldg(label + w[i]) : -1;
    }
  }
  __device__ __forceinline__ void flush() {
    if (run_blk >= 0) atomicMin(bmin + run_blk, run_min);
    run_blk = -1;
  }
  __device__ __forceinline__ void begin(int v, int64_t rs, int64_t) {
    lu = __ldg(label + v);
    ebase = __ldg(uoff + v) - (int)(rs + __ldg(nlow + v));  // e = ebase + a for upper arcs
    // head[v] >= 0 only for label vertices (v == label[v]): no dependent load
    const int hv = __ldg(head + v);
    row_u0 = hv >= 0 && v < hv;
  }
  __device__ __forceinline__ void arc(int v, int64_t a, int w, int i) {
    if (w <= v) return;
    int e = ebase + (int)a;
    bool mine;
    int blk;
    int lw;
    if (kBits) {
      if (lu == G && ((ing >> i) & 1u)) {
        eblk[e] = G;
        if (row_u0 && G != run_blk) {
          flush();
          run_blk = G;
          run_min = e;
        }
        return;
      }
      lw = __ldg(label + w);
    } else {
      lw = pl[kBits ? 0 : i];
    }
    if (lu == lw) {
      blk = lu;
      mine = row_u0;
    } else if (__ldg(head + lw) == v) {  // w's component hangs off v: its block
      blk = lw;
      mine = v < lw;
    } else {
      blk = lu;
      mine = row_u0;
    }
    eblk[e] = blk;
    if (mine && blk != run_blk) {
      flush();
      run_blk = blk;
      run_min = e;
    }
  }
  __device__ __forceinline__ void end(int, bool) {}
};

template <bool kBits>
__global__ void __launch_bounds__(256) k_edge_blocks(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, const int* __restrict__ crow,
                                                     int n, int64_t m, const int* __restrict__ label,
                                                     const int* __restrict__ head, const int* __restrict__ uoff,
                                                     const int* __restrict__ nlow, const uint32_t* __restrict__ gbits,
                                                     int* eblk, int* bmin, Scalars* sc) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->num_edges = uoff[n];  // (k_set_edges' job)
  EdgeBlockVisitor<kBits> vis;
  vis.gbits = gbits;
  vis.G = giant_label(label, sc);
  if (kBits && sc->giant_cnt < 256) {  // (uniform) small giant: run the label-gather instance
    EdgeBlockVisitor<false> lv;
    lv.off = off;
    lv.label = label;
    lv.head = head;
    lv.uoff = uoff;
    lv.nlow = nlow;
    lv.eblk = eblk;
    lv.bmin = bmin;
    lv.run_blk = -1;
    visit_arc_chunks(off, adj, crow, n, m, lv);
    lv.flush();
    return;
  }
  vis.off = off;
  vis.label = label;
  vis.head = head;
  vis.uoff = uoff;
  vis.nlow = nlow;
  vis.eblk = eblk;
  vis.bmin = bmin;
  vis.run_blk = -1;
  visit_arc_chunks(off, adj, crow, n, m, vis);
  vis.flush();
}

// Warp-staged variant.  Each warp owns 256 consecutive arcs (8 per lane, as
// visit_arc_chunks); the per-row words every arc needs -- row end, label,
// edge-id base, "block minimum row" flag -- are loaded ONCE per row, coalesced,
// by the lane whose index is the row's offset from the warp's first row, into
// a per-warp shared-memory window of kEBRows rows (rows beyond it fall back to
// global loads).  label[w] is replaced, for the common case, by one bit of the
// giant-component bitmap (bit w = label[w] == G; k_heads), held in shared
// memory (configs 2/3: 128 KB per CTA, one 1024-thread CTA per SM).  Only
// arcs leaving the giant gather label[w] / head[label[w]].  Used when the
// bitmap fits (n <= 1.6M); larger graphs run k_edge_blocks (a global bitmap
// measured 13% slower than the label gather on RMAT, whose hubs keep label
// lines L1-resident).
constexpr int kEBRows = 64;
constexpr int kEBThreads = 1024;
constexpr int kEBMaxSmemBytes = 227 * 1024;

__host__ __device__ constexpr size_t eb_rows_bytes(int threads) { return sizeof(int4) * kEBRows * (threads / 32); }

__device__ __forceinline__ int4 eb_row(const int64_t* __restrict__ off, const int* __restrict__ label,
                                       const int* __restrict__ head, const int* __restrict__ uoff,
                                       const int* __restrict__ nlow, int r) {
  const int64_t rs = __ldg(off + r);
  const int re = (int)__ldg(off + r + 1);
  const int h = __ldg(head + r);
  return make_int4(re, __ldg(label + r), __ldg(uoff + r) - (int)(rs + __ldg(nlow + r)), (h >= 0 && r < h) ? 1 : 0);
}

__global__ void __launch_bounds__(kEBThreads, 1)
    k_edge_blocks_ws(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, const int* __restrict__ crow,
                     int n, int64_t m, const int* __restrict__ label, const int* __restrict__ head,
                     const int* __restrict__ uoff, const int* __restrict__ nlow, const uint32_t* __restrict__ gbits,
                     Scalars* sc, int* __restrict__ eblk, int* bmin) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->num_edges = uoff[n];  // (k_set_edges' job)
  extern __shared__ int4 ebsm[];
  constexpr int kThreads = kEBThreads;
  int4* rows = ebsm + (threadIdx.x >> 5) * kEBRows;
  uint32_t* bits = reinterpret_cast<uint32_t*>(ebsm + kEBRows * (kThreads / 32));
  const int nw4 = ((n + 31) / 32 + 3) / 4;
  for (int i = threadIdx.x; i < nw4; i += kThreads)
    reinterpret_cast<uint4*>(bits)[i] = __ldg(reinterpret_cast<const uint4*>(gbits) + i);
  __syncthreads();
  const int G = giant_label(label, sc);
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (m + kItems - 1) / kItems;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(adj) & 15) == 0);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int run_blk = -1, run_min = 0;
  for (int64_t qb = (int64_t)blockIdx.x * kThreads + (threadIdx.x & ~31); qb < nchunks; qb += stride) {
    const int64_t q = qb + lane;
    const bool live = q < nchunks;
    int v = 0;
    uint32_t w[kItems];
    int64_t a0 = q * kItems, a1 = a0;
    if (live) {
      a1 = a0 + kItems < m ? a0 + kItems : m;
      if (vec_ok && a1 - a0 == kItems) {
        int4 x = ld_stream4(reinterpret_cast<const int4*>(adj + a0));
        int4 y = ld_stream4(reinterpret_cast<const int4*>(adj + a0 + 4));
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
        w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
      } else {
#pragma unroll
        for (int i = 0; i < kItems; i++) w[i] = (a0 + i < a1) ? __ldg(adj + a0 + i) : 0u;
      }
      v = __ldg(crow + q);
      if (v < 0) v = row_of(off, 0, n - 1, a0);
    }
    const int vf = __shfl_sync(0xffffffffu, v, 0);  // lane 0 is live whenever the warp is
    // rows the warp can touch: up to the last live lane's row plus the rows
    // its 8 arcs may still enter
    const int vl = __reduce_max_sync(0xffffffffu, live ? v : vf);
    const int rend = min(min(vf + kEBRows, vl + kItems + 1), n);
    __syncwarp();  // the previous iteration's readers of the window are done
#pragma unroll
    for (int k = 0; k < kEBRows; k += 32) {
      const int r = vf + k + lane;
      if (r < rend) rows[k + lane] = eb_row(off, label, head, uoff, nlow, r);
    }
    __syncwarp();
    if (live) {
      int vi = v - vf;
      int4 R = v < rend ? rows[vi] : eb_row(off, label, head, uoff, nlow, v);
#pragma unroll
      for (int i = 0; i < kItems; i++) {
        const int a = (int)(a0 + i);
        if (a < (int)a1) {
          while (a >= R.x) {  // next non-empty row (empty rows share the end)
            if (v + 1 < rend) {
              vi++;
              v++;
              R = rows[vi];
            } else {
              v = next_row(off, v, n, a);
              R = eb_row(off, label, head, uoff, nlow, v);
            }
          }
          const int x = (int)w[i];
          if (x > v) {
            int blk;
            bool mine;
            if (R.y == G && ((bits[x >> 5] >> (x & 31)) & 1u)) {
              blk = G;
              mine = R.w != 0;
            } else {
              const int lw = __ldg(label + x);
              if (R.y == lw) {
                blk = lw;
                mine = R.w != 0;
              } else if (__ldg(head + lw) == v) {  // x's component hangs off v: its block
                blk = lw;
                mine = v < lw;
              } else {
                blk = R.y;
                mine = R.w != 0;
              }
            }
            const int e = R.z + a;
            eblk[e] = blk;
            if (mine && blk != run_blk) {
              if (run_blk >= 0) atomicMin(bmin + run_blk, run_min);
              run_blk = blk;
              run_min = e;
            }
          }
        }
      }
    }
  }
  if (run_blk >= 0) atomicMin(bmin + run_blk, run_min);
}

// block -> minimum edge id of the block, 4 edges per thread (16-byte
// streaming loads and stores; the bmin gathers of the giant block hit one
// L1-resident word)
__global__ void k_edge_final(int* eblk, const int* __restrict__ bmin, const int* __restrict__ uoff, int n) {
  pdl_enter();
  const int E = uoff[n];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(eblk) & 15) == 0) {
    const int64_t nv = E / 4;
    int4* e4 = reinterpret_cast<int4*>(eblk);
    for (int64_t i = tid; i < nv; i += stride) {
      int4 b = __ldcs(e4 + i);
      b.x = __ldg(bmin + b.x);
      b.y = __ldg(bmin + b.y);
      b.z = __ldg(bmin + b.z);
      b.w = __ldg(bmin + b.w);
      __stcs(e4 + i, b);
    }
    for (int64_t e = 4 * nv + tid; e < E; e += stride) eblk[e] = __ldg(bmin + eblk[e]);
  } else {
    for (int64_t e = tid; e < E; e += stride) eblk[e] = __ldg(bmin + eblk[e]);
  }
}

__global__ void k_set_edges(const int* __restrict__ uoff, int n, Scalars* sc) {
  pdl_enter(); sc->num_edges = uoff[n]; }

void stage6_labelling(const Graph& g, const int4* rec, const int* label, int* head, uint8_t* is_ap,
                      int* edge_label, int* cnt, int* uoff, int* nlow, int* bmin, uint32_t* gbits, void* cub_tmp,
                      size_t cub_bytes, Scalars* sc, cudaStream_t st, cudaEvent_t heads_done, const Side* side) {
  const int n = g.n;
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  // head = -1, cnt = 0, bmin = INF were initialised by the stage-4 kernel
  launch(k_heads, gv, B, 0, st, n, rec, label, head, cnt, gbits, sc);
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
  if (!edge_label || g.m == 0) {
    launch(k_set_edges, 1, 1, 0, st, uoff, n, sc);
    note(K_SET_EDGES);
  } else {
    int64_t nchunks = (g.m + kItems - 1) / kItems;
    const size_t smem = eb_rows_bytes(kEBThreads) + 16 * (size_t)(((n + 31) / 32 + 3) / 4);
    if (opt(OPT_EB_STAGED) && smem <= (size_t)kEBMaxSmemBytes) {
      cudaFuncSetAttribute(k_edge_blocks_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch(k_edge_blocks_ws, grid_for(nchunks, kEBThreads, 1), kEBThreads, smem, st, g.off, g.adj, g.crow, n, g.m,
             label, head, uoff, nlow, (const uint32_t*)gbits, sc, edge_label, bmin);
    } else {
      launch(opt(OPT_EB_STAGED) ? k_edge_blocks<true> : k_edge_blocks<false>, grid_for(nchunks, B, 32), B, 0, st,
             g.off, g.adj, g.crow, n, g.m, label, head, uoff, nlow, (const uint32_t*)gbits, edge_label, bmin, sc);
    }
    note(K_EDGE_BLOCKS);
    launch(k_edge_final, grid_for(g.m / 2, B), B, 0, st, edge_label, bmin, uoff, n);
    note(K_EDGE_FINAL);
  }
  if (side) cudaStreamWaitEvent(st, side->ev[3], 0);  // join the articulation flags
}

// ---------------------------------------------------------------------------
// intermediate exports (parity rungs 1-4)
// ---------------------------------------------------------------------------
__global__ void k_export(int n, const int4* __restrict__ rec, const int4* __restrict__ AP, int* parent, int* first,
                         int* last, int* w1, int* w2, uint8_t* fence) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int4 r = rec[v];
    if (parent) parent[v] = r.z;
    if (first) first[v] = r.x;
    if (last) last[v] = r.y;
    if (fence) fence[v] = (uint8_t)r.w;
    if (w1 || w2) {
      int4 a = AP[r.x];
      if (w1) w1[v] = a.x;
      if (w2) w2[v] = a.y;
    }
  }
}

void export_debug(const Graph& g, const int2* fe, const int4* rec, const int4* AP, int* forest, int* parent,
                  int* first, int* last, int* w1, int* w2, uint8_t* fence, cudaStream_t st) {
  if (forest) cudaMemcpyAsync(forest, fe, sizeof(int2) * g.n, cudaMemcpyDeviceToDevice, st);
  if (parent || first || last || w1 || w2 || fence)
    launch(k_export, grid_for(g.n, 256), 256, 0, st, g.n, rec, AP, parent, first, last, w1, w2, fence);
}

}  // namespace fbcc
