// tags.cu -- Stage 3 (subtree tags low/high) and Stage 4 (fence bits).
//
// Replaces compute_tags (tagging.py:300-304): _w_gather 101-119 (per-vertex
// gather over non-tree edges, 128 static vertex chunks), _scatter_at_first
// 122-135, _block_extremes 138-159, _doubling_tables 162-184 ((K+1) x 2n/16
// int64 words -- ~2.4 GB at n = 1e8) and _range_queries 187-242; then the
// fence bit of _pack_skeleton (connectivity.py:84-96).
//
// B200 design:
//  * w gather: arc-balanced (kItems arcs per thread, hub rows spread over
//    many threads), one 16-byte record gather per arc, and the result goes
//    straight into the tour-indexed array A at first[v] (fusing
//    _scatter_at_first).  Rows wholly inside a thread's chunk are stored
//    plainly; rows split across chunks combine with 32-bit atomicMin/Max.
//  * low/high = min/max of A over [first[v], last[v]] -- a segmented reduction
//    over Euler-tour order.  Each CTA stages one 4096-position tile of A in
//    shared memory (coalesced 256-byte warp loads), builds warp-level
//    prefix/suffix extremes per 32-position sub-block plus a 128-entry sparse
//    table over sub-blocks, and answers every query whose interval starts or
//    ends in the tile while the tile is resident: whole queries inside the
//    tile directly, spanning queries as a suffix partial (at first) and a
//    prefix partial (at last).  Only a sparse table over TILE EXTREMES stays
//    in global memory (8 B x 2n/4096 x log2 -- 6 MB at n = 1e8, L2-resident)
//    instead of the reference's (K+1) x 2n/16 doubling table.
//  * Stage 4 is the epilogue: combine partials + one table probe, compare
//    with the parent's interval, set the fence bit in the 16-byte record that
//    Stage 5's predicate gathers.
#include "common.cuh"
#include "kernels.cuh"

#ifndef FBCC_WSTORE_CS
#define FBCC_WSTORE_CS 1
#endif

namespace fbcc {

__device__ __forceinline__ int2 comb(int2 a, int2 b) { return make_int2(min(a.x, b.x), max(a.y, b.y)); }
__device__ __forceinline__ int2 filler() { return make_int2(kINF, -1); }

// ---------------------------------------------------------------------------
// w1/w2 gather into A[first[v]]
// ---------------------------------------------------------------------------
// kExact reproduces _w_gather (tagging.py:101-119): both forest directions
// excluded, one 16 B record gather per arc.  The pipeline runs the relaxed
// form, which excludes only the edge to the parent (tested on v's own
// record) and gathers a 4-byte first[w] from a compact array: a child c has
// first[c] > first[v] and lies inside v's subtree, so counting it leaves w1,
// and every subtree aggregate low/high, unchanged -- only the intermediate
// w2 of v may grow (SURVEY §8(c) rung 3 checks both forms).  RMAT: 1.05e9
// gathers from a 134 MB array (mostly L2) instead of a 537 MB one.
template <bool kExact>
__device__ __forceinline__ void w_arc(int v, int pv, int w, const int4* __restrict__ rec,
                                      const int* __restrict__ firsts, int& m1, int& m2) {
  if (pv == w) return;  // tree edge to the parent
  int f;
  if (kExact) {
    const int4 r = __ldg(rec + w);
    if (r.z == v) return;  // tree edge to a child
    f = r.x;
  } else {
    f = __ldg(firsts + w);
  }
  m1 = min(m1, f);
  m2 = max(m2, f);
}

// (streaming store, evict-first: the tour-indexed records are scattered over
// 32n bytes and must not evict the first[] lines the gathers live on)
__device__ __forceinline__ void w_store(int4* AP, int fv, int m1, int m2) {
#if FBCC_WSTORE_CS
  __stcs(reinterpret_cast<int2*>(AP + fv), make_int2(min(fv, m1), max(fv, m2)));
#else
  *reinterpret_cast<int2*>(AP + fv) = make_int2(min(fv, m1), max(fv, m2));
#endif
}

__device__ __forceinline__ void w_atomic(int4* AP, int fv, int m1, int m2) {
  if (m2 < 0) return;  // no contributing arc (AP[fv] already holds (fv, fv))
  atomicMin(&AP[fv].x, m1);
  atomicMax(&AP[fv].y, m2);
}

// Arc-balanced like visit_arc_chunks (8 arcs per thread, the chunk's row from
// crow), but rows that straddle chunk boundaries are combined inside the warp
// instead of with two atomics per piece: consecutive lanes hold consecutive
// chunks, so a row's pieces sit in consecutive lanes.  Each lane ends with at
// most a "tail" piece (its last row runs past the chunk) and a "head" piece
// (its first row began before the chunk and ends in it); lane j's head is
// shuffled to lane j-1, whose tail is the same row, then lanes with equal
// tail rows reduce with __match_any_sync + __reduce_{min,max}_sync.  A row
// that begins and ends inside the warp gets one plain store; only rows that
// cross a warp boundary fall back to atomics.  (Per-piece atomics were ~5 per
// row at degree 16: a quarter of the kernel's L1 wavefronts.)
#ifndef FBCC_WG_MIN_BLOCKS
#define FBCC_WG_MIN_BLOCKS 8  // 32 registers: full occupancy for the gathers (measured: 46 regs -> 133 us, 32 -> 111 us on config 2)
#endif
constexpr int kWGatherMinBlocks = FBCC_WG_MIN_BLOCKS;

template <bool kExact>
__global__ void __launch_bounds__(256, kWGatherMinBlocks) k_w_gather(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  const int* __restrict__ crow, int n, int64_t m,
                                                  const int4* __restrict__ rec, const int* __restrict__ firsts,
                                                  int4* AP, int* __restrict__ nlow) {
  pdl_enter();
  // the pipeline variant also counts each row's lower neighbours (w < v) for
  // Stage 6's edge numbering (k_upper_degree's binary searches, folded into
  // this pass over the same arcs)
  constexpr bool kCount = !kExact;
  const int64_t nchunks = (m + kItems - 1) / kItems;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(adj) & 31) == 0);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the shuffles below need the whole warp)
  for (int64_t qb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); qb < nchunks; qb += stride) {
    const int q = (int)qb + lane;  // arc indices fit 32 bits (check_sizes: m < 2^31)
    int tkey = -1, t1 = kINF, t2 = -1, tfv = 0, tc = 0;  // row running past the chunk end
    bool tstart = false;                                 // ... and starting inside the chunk
    int hkey = -1, h1 = kINF, h2 = -1, hfv = 0, hc = 0;  // row begun before the chunk, ending in it
    if (q < nchunks) {
      const int a0 = q * kItems;
      const int a1 = a0 + kItems < (int)m ? a0 + kItems : (int)m;
      uint32_t w[kItems];
      if (vec_ok && a1 - a0 == kItems) {
        ld_chunk8(adj + a0, w);
      } else {
#pragma unroll
        for (int i = 0; i < kItems; i++) w[i] = (a0 + i < a1) ? __ldg(adj + a0 + i) : 0u;
      }
      int v = __ldg(crow + q);
      if (v < 0) v = row_of(off, 0, n - 1, a0);
      int rs = (int)__ldg(off + v), re = (int)__ldg(off + v + 1);
      int4 r = __ldg(rec + v);
      int m1 = kINF, m2 = -1, c = 0;
#pragma unroll
      for (int i = 0; i < kItems; i++) {
        const int a = a0 + i;
        if (a < a1) {
          if (a >= re) {  // row v ends inside the chunk
            if (rs < a0) { hkey = v; h1 = m1; h2 = m2; hfv = r.x; hc = c; }
            else {
              w_store(AP, r.x, m1, m2);
              if (kCount) nlow[v] = c;
            }
            v = next_row(off, v, n, a);
            rs = (int)__ldg(off + v);
            re = (int)__ldg(off + v + 1);
            r = __ldg(rec + v);
            m1 = kINF;
            m2 = -1;
            c = 0;
          }
          if (kCount) c += (int)w[i] < v;
          w_arc<kExact>(v, r.z, (int)w[i], rec, firsts, m1, m2);
        }
      }
      if (re > a1) { tkey = v; t1 = m1; t2 = m2; tfv = r.x; tc = c; tstart = rs >= a0; }
      else if (rs < a0) { hkey = v; h1 = m1; h2 = m2; hfv = r.x; hc = c; }
      else {
        w_store(AP, r.x, m1, m2);
        if (kCount) nlow[v] = c;
      }
    }
    // lane j's head piece belongs to lane j-1's tail row
    const int nk = __shfl_down_sync(0xffffffffu, hkey, 1);
    const int n1 = __shfl_down_sync(0xffffffffu, h1, 1);
    const int n2 = __shfl_down_sync(0xffffffffu, h2, 1);
    const int nc = kCount ? __shfl_down_sync(0xffffffffu, hc, 1) : 0;
    bool tend = false;
    if (lane < 31 && nk >= 0) {
      t1 = min(t1, n1);
      t2 = max(t2, n2);
      tc += nc;
      tend = true;
    }
    if (lane == 0 && hkey >= 0) {  // began in an earlier warp
      w_atomic(AP, hfv, h1, h2);
      if (kCount && hc) atomicAdd(nlow + hkey, hc);
    }
    const unsigned grp = __match_any_sync(0xffffffffu, tkey);
    const int g1 = __reduce_min_sync(grp, t1);
    const int g2 = __reduce_max_sync(grp, t2);
    const int gc = kCount ? (int)__reduce_add_sync(grp, (unsigned)tc) : 0;
    const unsigned ends = __reduce_or_sync(grp, tend ? 1u : 0u);
    if (tkey >= 0 && lane == __ffs(grp) - 1) {
      if (tstart && ends) {  // whole row inside this warp
        w_store(AP, tfv, g1, g2);
        if (kCount) nlow[tkey] = gc;
      } else {
        w_atomic(AP, tfv, g1, g2);
        if (kCount && gc) atomicAdd(nlow + tkey, gc);
      }
    }
  }
}

// compact first[] for the relaxed gather; zeroes the lower-degree counters
// the gather accumulates into (rows split across warps add atomically)
__global__ void k_firsts(const int4* __restrict__ rec, int n, int* __restrict__ firsts, int* __restrict__ nlow) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    firsts[v] = __ldg(&rec[v].x);
    nlow[v] = 0;
  }
}

// ---------------------------------------------------------------------------
// tile pass
// ---------------------------------------------------------------------------
// One persistent CTA per SM walks its tiles (blockIdx.x, + gridDim.x, ...).
// Each 4096-position tile of AP (64 KB of 16-byte records) is staged into
// shared memory by ONE bulk async copy (cp.async.bulk, completion on an
// mbarrier), double-buffered: the copy of the CTA's next tile but one is
// issued as soon as a buffer is free, so the DRAM stream runs under the
// scans and queries of the current tile instead of every thread stalling on
// its own loads.  The staged record carries both the tile values (w1, w2)
// and the query (v or ~v, partner position): nothing is read from global
// memory twice.
constexpr int kTileThreads = 1024;
constexpr int kSub = 32;
constexpr int kNSub = kTile / kSub;  // 128
constexpr int kSubLev = 32 - __builtin_clz(kNSub);  // levels 0..log2(kNSub) (8 for 128 sub-blocks)
constexpr int kTileBytes = kTile * (int)sizeof(int4);  // 64 KB
constexpr size_t kTileSmem = 2 * (size_t)kTileBytes + sizeof(int2) * (2 * kTile + kSubLev * kNSub) + 16;

struct TileSmem {
  const int4* raw;  // the staged tile: {w1, w2, v or ~v, partner}
  int2* pre;
  int2* suf;
  int2* st;  // [kSubLev][kNSub]
  __device__ __forceinline__ int2 val(int i) const {
    const int4 r = raw[i];
    return make_int2(r.x, r.y);
  }
  __device__ __forceinline__ int2 st_query(int i, int j) const {  // sub-blocks i..j, i <= j
    int k = 31 - __clz(j - i + 1);
    return comb(st[k * kNSub + i], st[k * kNSub + j - (1 << k) + 1]);
  }
  __device__ __forceinline__ int2 range(int a, int b) const {  // positions a..b in tile
    int sa = a >> 5, sb = b >> 5;
    if (sa == sb) {
      int2 r = val(a);
      for (int i = a + 1; i <= b; i++) r = comb(r, val(i));
      return r;
    }
    int2 r = comb(suf[a], pre[b]);
    if (sb - sa > 1) r = comb(r, st_query(sa + 1, sb - 1));
    return r;
  }
  __device__ __forceinline__ int2 to_end(int p) const {
    int sp = p >> 5;
    int2 r = suf[p];
    if (sp < kNSub - 1) r = comb(r, st_query(sp + 1, kNSub - 1));
    return r;
  }
  __device__ __forceinline__ int2 from_start(int p) const {
    int sp = p >> 5;
    int2 r = pre[p];
    if (sp > 0) r = comb(r, st_query(0, sp - 1));
    return r;
  }
};

// bulk async copy global -> shared, completing on an mbarrier (sm_90+ TMA
// engine, 1-D: no tensor map)
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the buffer first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(gsrc), "r"(bytes), "r"(b) : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(b), "r"(parity) : "memory");
  }
}

constexpr int kTableOneCta = 16384;

// (levels laid out with stride ntile; entries at and past nt -- tiles past
// the list -- are neither built nor queried)
__device__ __forceinline__ void table_levels(int2* table, int ntile, int nt, int tlev) {
  for (int k = 1; k < tlev; k++) {
    const int2* prev = table + (int64_t)(k - 1) * ntile;
    int2* cur = table + (int64_t)k * ntile;
    const int half = 1 << (k - 1);
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      int2 a = prev[i];
      cur[i] = (i + half < nt) ? comb(a, prev[i + half]) : a;
    }
    __syncthreads();
  }
}

// tiles holding list positions: the pipeline's tour stops at tour_len
// (detached roots have no AP entries)
__device__ __forceinline__ int64_t list_positions(const int* tlen, int64_t N) { return tlen ? *tlen : N; }

// (sc != nullptr: the last block to finish also builds every level of the
// tile-extreme sparse table -- k_table_all's work, one launch fewer)
__global__ void __launch_bounds__(kTileThreads, 1) k_tile(const int4* __restrict__ AP,
                                                          int64_t N, int ntile, int2* __restrict__ lh1,
                                                          int2* __restrict__ lh2, int2* __restrict__ table0, Scalars* sc, int tlev,
                                                          const int* tlen) {
  pdl_enter();
  N = list_positions(tlen, N);
  const int nt = (int)((N + kTile - 1) / kTile);
  extern __shared__ __align__(128) unsigned char tsm[];
  int4* buf0 = reinterpret_cast<int4*>(tsm);
  int4* buf1 = reinterpret_cast<int4*>(tsm + kTileBytes);
  int2* aux = reinterpret_cast<int2*>(tsm + 2 * kTileBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(aux + 2 * kTile + kSubLev * kNSub);  // 2 mbarriers
  TileSmem S;
  S.pre = aux;
  S.suf = aux + kTile;
  S.st = aux + 2 * kTile;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(bars + i);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x < nt) bulk_load(buf0, AP + (int64_t)blockIdx.x * kTile, kTileBytes, bars);
    if (blockIdx.x + G < nt) bulk_load(buf1, AP + (int64_t)(blockIdx.x + G) * kTile, kTileBytes, bars + 1);
  }
  uint32_t parity = 0;  // bit b: phase of buffer b's barrier
  int k = 0;
  for (int tile = blockIdx.x; tile < nt; tile += G, k++) {
    const int b = k & 1;
    const int4* T = b ? buf1 : buf0;
    S.raw = T;
    bar_wait(bars + b, (parity >> b) & 1u);
    parity ^= 1u << b;
    const int64_t base = (int64_t)tile * kTile;
    // 1. warp scans per 32-position sub-block (positions past N: filler)
    for (int sb = warp; sb < kNSub; sb += kTileThreads / 32) {
      const int p = sb * kSub + lane;
      int2 x = filler();
      if (base + p < N) x = S.val(p);
      int2 pr = x, su = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int px = __shfl_up_sync(0xffffffffu, pr.x, o), py = __shfl_up_sync(0xffffffffu, pr.y, o);
        int sx = __shfl_down_sync(0xffffffffu, su.x, o), sy = __shfl_down_sync(0xffffffffu, su.y, o);
        if (lane >= o) pr = comb(pr, make_int2(px, py));
        if (lane + o < 32) su = comb(su, make_int2(sx, sy));
      }
      S.pre[p] = pr;
      S.suf[p] = su;
      if (lane == 31) S.st[sb] = pr;
    }
    __syncthreads();
    // 2. sparse table over the 128 sub-block extremes
    for (int lv = 1; lv < kSubLev; lv++) {
      if (threadIdx.x < kNSub) {
        int i = threadIdx.x, j = i + (1 << (lv - 1));
        int2 a = S.st[(lv - 1) * kNSub + i];
        S.st[lv * kNSub + i] = (j < kNSub) ? comb(a, S.st[(lv - 1) * kNSub + j]) : a;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) table0[tile] = S.st[(kSubLev - 1) * kNSub];
    // 3. answer the queries that start or end here
    for (int p = threadIdx.x; p < kTile; p += kTileThreads) {
      const int64_t gp = base + p;
      if (gp >= N) break;
      const int4 ap = T[p];
      const int2 q = make_int2(ap.z, ap.w);
      if (q.x >= 0) {  // entry position of v = q.x; partner = last[v]
        const int64_t rel = (int64_t)q.y - base;
        lh1[q.x] = (rel < kTile) ? S.range(p, (int)rel) : S.to_end(p);
      } else if ((int64_t)q.y < base) {  // exit position of ~q.x, entry in an earlier tile
        lh2[~q.x] = S.from_start(p);
      }
    }
    __syncthreads();  // buffer b and the scan arrays are free
    if (threadIdx.x == 0 && tile + 2 * G < nt)
      bulk_load(b ? buf1 : buf0, AP + (int64_t)(tile + 2 * G) * kTile, kTileBytes, bars + b);
  }
  if (sc) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&sc->tile_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      table_levels(table0, ntile, nt, tlev);
      if (threadIdx.x == 0) sc->tile_ticket = 0;
    }
  }
}

// all levels of the tile-extreme sparse table in one CTA (levels are
// published to the block by __syncthreads; every level is tiny next to a
// launch when ntile <= kTableOneCta)

__global__ void __launch_bounds__(1024) k_table_all(int2* table, int ntile, int tlev, const int* tlen) {
  pdl_enter();
  table_levels(table, ntile, (int)((list_positions(tlen, (int64_t)ntile * kTile) + kTile - 1) / kTile), tlev);
}

__global__ void k_table_level(int2* table, int ntile, int k, const int* tlen) {
  pdl_enter();
  const int nt = (int)((list_positions(tlen, (int64_t)ntile * kTile) + kTile - 1) / kTile);
  const int2* prev = table + (int64_t)(k - 1) * ntile;
  int2* cur = table + (int64_t)k * ntile;
  const int half = 1 << (k - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
    int2 a = prev[i];
    cur[i] = (i + half < nt) ? comb(a, prev[i + half]) : a;
  }
}

void stage3_tags(const Graph& g, const Rooting& R, Tags& T, cudaStream_t st, int* nlow, const Side* side, int* uoff,
                 void* cub_tmp, size_t cub_bytes, Scalars* sc) {
  const int B = 256;
  int64_t nchunks = (g.m + kItems - 1) / kItems;
  if (!nlow) {  // stand-alone compute_tags: the reference's exact w2
    if (g.m > 0)
      launch(k_w_gather<true>, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj, g.crow, g.n, g.m, R.rec, nullptr, T.AP,
             nullptr);
  } else {
    // compact first[] lives in lh1 until k_tile overwrites it
    int* firsts = reinterpret_cast<int*>(T.lh1);
    if (R.firsts != firsts || R.nlow != nlow) {  // (else k_positions wrote both)
      launch(k_firsts, grid_for(g.n, B), B, 0, st, R.rec, g.n, firsts, nlow);
      note(K_FIRSTS);
    }
    if (g.m > 0)
      launch(k_w_gather<false>, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj, g.crow, g.n, g.m, R.rec, firsts,
             T.AP, nlow);
  }
  if (g.m > 0) {
    note(K_W_GATHER);
  }
  if (side && nlow) {  // nlow is final: Stage 6's upper-degree scan runs beside Stages 3-5
    cudaEventRecord(side->ev[0], st);
    cudaStreamWaitEvent(side->s, side->ev[0], 0);
    scan_upper_degrees(g.off, nlow, g.n, uoff, cub_tmp, cub_bytes, side->s);
    note(K_SCAN);
    cudaEventRecord(side->ev[1], side->s);
  }
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem);
  // (the table in k_tile's last block when it fits one CTA and a ticket word exists)
  Scalars* tsc = (sc && T.ntile <= kTableOneCta && T.tlev > 1) ? sc : nullptr;
  launch(k_tile, T.ntile < kNumSMs ? T.ntile : kNumSMs, kTileThreads, kTileSmem, st, T.AP, 2 * (int64_t)g.n, T.ntile,
         T.lh1, T.lh2, T.table, tsc, T.tlev, T.tour_len);
  note(K_TILE);
  if (tsc) {
  } else if (T.ntile <= kTableOneCta) {
    if (T.tlev > 1) {
      launch(k_table_all, 1, 1024, 0, st, T.table, T.ntile, T.tlev, T.tour_len);
      note(K_TABLE);
    }
  } else {
    for (int k = 1; k < T.tlev; k++) {
      launch(k_table_level, grid_for(T.ntile, B), B, 0, st, T.table, T.ntile, k, T.tour_len);
      note(K_TABLE);
    }
  }
}

// ---------------------------------------------------------------------------
// Stage 4: combine, fence bit
// ---------------------------------------------------------------------------
__global__ void k_fence(int n, int4* rec, const int2* __restrict__ lh1, const int2* __restrict__ lh2,
                        const int2* __restrict__ table, int ntile, int* low_out, int* high_out,
                        int* __restrict__ head, int* __restrict__ cnt, int* __restrict__ bmin, const int* tlen) {
  pdl_enter();
  const int64_t N = list_positions(tlen, 2 * (int64_t)n);
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int4 r = rec[v];
    int ta = r.x / kTile, tb = r.y / kTile;
    int2 res;
    if (r.x >= N) {  // detached root: {v} alone, low = high = first
      res = make_int2(r.x, r.x);
    } else {
      res = lh1[v];
    }
    if (r.x < N && ta != tb) {
      res = comb(res, lh2[v]);
      if (tb - ta > 1) {
        int i = ta + 1, j = tb - 1;
        int k = 31 - __clz(j - i + 1);
        res = comb(res, comb(table[(int64_t)k * ntile + i], table[(int64_t)k * ntile + j - (1 << k) + 1]));
      }
    }
    int fence = 0;
    if (r.z >= 0) {
      int4 pr = rec[r.z];
      fence = (res.x >= pr.x && res.y <= pr.y) ? 1 : 0;
    }
    reinterpret_cast<int*>(rec + v)[3] = fence;
    if (low_out) {
      low_out[v] = res.x;
      high_out[v] = res.y;
    }
    // Stage-6 per-vertex state, initialised here (same index space; saves
    // three memset nodes in the graph)
    head[v] = -1;
    cnt[v] = 0;
    bmin[v] = kINF;
  }
}

void stage4_fence(const Graph& g, const Rooting& R, const Tags& T, int* low_out, int* high_out, int* head, int* cnt,
                  int* bmin, cudaStream_t st) {
  const int B = 256;
  launch(k_fence, grid_for(g.n, B), B, 0, st, g.n, R.rec, T.lh1, T.lh2, T.table, T.ntile, low_out, high_out, head,
                                          cnt, bmin, T.tour_len);
  note(K_FENCE);
}

}  // namespace fbcc
