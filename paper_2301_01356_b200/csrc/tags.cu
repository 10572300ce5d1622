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

// ---------------------------------------------------------------------------
// Witness tags.  fence[v] only asks whether some non-tree edge under v leaves
// the parent's interval, and on a dense graph almost every vertex shows such
// an edge among its first arcs: RMAT s25 -- of 17.1 M tree edges, the first
// three arcs of every row (already recorded by Stage 1, w0[3][n]) leave 56
// fence bits open; uniform 2^20 x 8 leaves 271.  Plans with m >= 8n therefore
// run Stage 3 on those samples:
//   1. k_w_sample: (w1, w2) from arcs 0-2 of each row (3 coalesced reads and
//      3 gathers per vertex instead of a gather per arc), bit 30 of w2 set
//      when the row has more arcs -- the tile pass's max carries the bit up
//      every subtree, so "exact" (no row under v was cut short) is known too;
//   2. the tile pass and k_fence as usual: a bit that comes out 0 has a real
//      witness edge, one that comes out 1 over an exact subtree (or under a
//      root) is exact; the others are listed;
//   3. k_witness_fix: one warp per listed vertex rescans every row under it
//      (the tour positions first..last name them) and settles the bit.
// If too many are listed, or one has too large a subtree, the full gather and
// a second tile / fence pass run instead (their kernels are in the plan and
// return at once otherwise).  Only the fence bits feed the later stages, and
// they are exact either way; low/high themselves are exact only in the full
// form, which debug exports and the stand-alone ops always use.
// ---------------------------------------------------------------------------
#ifndef FBCC_WITNESS_ARCS
#define FBCC_WITNESS_ARCS 3
#endif
constexpr int kWitnessArcs = FBCC_WITNESS_ARCS;  // arcs sampled per row (<= 3: what k_chunk_rows records)
constexpr int kExactBit = 1 << 30;        // tour positions stay below 2^30 in witness plans
constexpr int kWitnessListCap = 1 << 20;  // listed vertices (<= n: the list is a dead Stage-2 array)
constexpr int kWitnessMaxSubtree = 1 << 11;  // tour positions one warp may walk for one vertex

struct WitnessGate {
  const Scalars* sc;  // nullptr: not a witness plan, always open
  int cap;
  unsigned long long work;
  // after k_fence's phase A: do the full gather / tile / fence kernels have to run?
  __device__ __forceinline__ bool open() const {
    return !sc || sc->und_n > cap || sc->und_big != 0 || sc->und_work > work;
  }
};

__global__ void k_w_sample(const int64_t* __restrict__ off, int n, const int4* __restrict__ rec,
                           const int* __restrict__ w0, int4* AP, const int* __restrict__ tlen,
                           int2* __restrict__ lh1) {
  pdl_enter();
  const int N = *tlen;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    // every per-vertex word first (coalesced, independent of one another),
    // then the gathers together: one vertex is two dependent round trips.
    // first[w] comes straight from the 16-byte records: at three gathers per
    // vertex a compact first[] array is not worth k_positions' scattered
    // 4-byte store per vertex that would build it.
    const int64_t deg = __ldg(off + v + 1) - __ldg(off + v);
    if (deg == 0) continue;  // (RMAT: half the vertices -- no record, no arcs to read; its tour slot, if any, keeps (first, first))
    const int4 r = __ldg(rec + v);
    int w[kWitnessArcs];
#pragma unroll
    for (int k = 0; k < kWitnessArcs; k++) w[k] = __ldg(w0 + (int64_t)k * n + v);  // (arc 0 of an empty row: unwritten, unused)
    const int fv = r.x, pv = r.z;
    if (fv >= N) continue;  // detached root: no tour entry
    int f[kWitnessArcs];
#pragma unroll
    for (int k = 0; k < kWitnessArcs; k++) f[k] = (deg > k && w[k] != pv) ? __ldg(&rec[w[k]].x) : fv;
    int m1 = fv, m2 = fv;
#pragma unroll
    for (int k = 0; k < kWitnessArcs; k++) {
      m1 = min(m1, f[k]);
      m2 = max(m2, f[k]);
    }
    const int2 w12 = make_int2(m1, deg > kWitnessArcs ? (m2 | kExactBit) : m2);
    __stcs(reinterpret_cast<int2*>(AP + fv), w12);
    // a leaf of the forest (RMAT: most vertices) is its own subtree: its
    // low / high are these two words, stored here by vertex (coalesced) -- the
    // tile pass then skips the leaves' queries and their scattered stores
    if (r.y == fv + 1) lh1[v] = w12;
  }
}

// nlow[v] = neighbours of v below v (rows sorted): the row's last and first
// arcs settle most rows (RMAT: nearly every vertex has only smaller
// neighbours, the hubs mostly larger ones), the rest by binary search
__global__ void k_nlow(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n,
                       int* __restrict__ nlow) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int64_t lo = __ldg(off + v), hi = __ldg(off + v + 1);
    const int64_t rs = lo;
    if (hi > lo) {
      if ((int)__ldg(adj + hi - 1) < v) lo = hi;
      else if ((int)__ldg(adj + lo) > v) hi = lo;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int)__ldg(adj + mid) < v) lo = mid + 1; else hi = mid;
      }
    }
    nlow[v] = (int)(lo - rs);
  }
}

void compute_nlow(const Graph& g, int* nlow, cudaStream_t st) {
  launch(k_nlow, grid_for(g.n, 256), 256, 0, st, g.off, g.adj, g.n, nlow);
  note(K_NLOW);
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

template <bool kExact, bool kCountLow = !kExact>
__global__ void __launch_bounds__(256, kWGatherMinBlocks) k_w_gather(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  const int* __restrict__ crow, int n, int64_t m,
                                                  const int4* __restrict__ rec, const int* __restrict__ firsts,
                                                  int4* AP, int* __restrict__ nlow, WitnessGate gate) {
  pdl_enter();
  if (!gate.open()) return;  // (a witness plan whose sampled tags settled every fence bit)
  // the pipeline variant also counts each row's lower neighbours (w < v) for
  // Stage 6's edge numbering (k_upper_degree's binary searches, folded into
  // this pass over the same arcs; witness plans count them in k_nlow)
  constexpr bool kCount = kCountLow;
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
      int v = crow ? __ldg(crow + q) : -1;  // (no table: a witness plan's overflow redo)
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
__global__ void k_firsts(const int4* __restrict__ rec, int n, int* __restrict__ firsts, int* __restrict__ nlow,
                         WitnessGate gate) {
  pdl_enter();
  if (!gate.open()) return;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    firsts[v] = __ldg(&rec[v].x);
    if (nlow) nlow[v] = 0;
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
#ifndef FBCC_TILE_THREADS
#define FBCC_TILE_THREADS 1024
#endif
#ifndef FBCC_TILE_CTAS
#define FBCC_TILE_CTAS 1
#endif
constexpr int kTileThreads = FBCC_TILE_THREADS;
constexpr int kTileCtas = FBCC_TILE_CTAS;  // resident CTAs per SM (shared memory: 200 KB at 4096 positions per tile)
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
__global__ void __launch_bounds__(kTileThreads, kTileCtas) k_tile(const int4* __restrict__ AP,
                                                          int64_t N, int ntile, int2* __restrict__ lh1,
                                                          int2* __restrict__ lh2, int2* __restrict__ table0, Scalars* sc, int tlev,
                                                          const int* tlen, WitnessGate gate, bool skip_leaves) {
  pdl_enter();
  if (!gate.open()) return;
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
        if (skip_leaves && (int64_t)q.y == gp + 1) continue;  // (k_w_sample stored the leaf's own words)
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

__global__ void __launch_bounds__(1024) k_table_all(int2* table, int ntile, int tlev, const int* tlen,
                                                    WitnessGate gate) {
  pdl_enter();
  if (!gate.open()) return;
  table_levels(table, ntile, (int)((list_positions(tlen, (int64_t)ntile * kTile) + kTile - 1) / kTile), tlev);
}

__global__ void k_table_level(int2* table, int ntile, int k, const int* tlen, WitnessGate gate) {
  pdl_enter();
  if (!gate.open()) return;
  const int nt = (int)((list_positions(tlen, (int64_t)ntile * kTile) + kTile - 1) / kTile);
  const int2* prev = table + (int64_t)(k - 1) * ntile;
  int2* cur = table + (int64_t)k * ntile;
  const int half = 1 << (k - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
    int2 a = prev[i];
    cur[i] = (i + half < nt) ? comb(a, prev[i + half]) : a;
  }
}

static WitnessGate gate_of(const Witness* W, const Scalars* sc) {
  return (W && W->on) ? WitnessGate{sc, W->cap, W->work} : WitnessGate{nullptr, 0, 0};
}

// tile pass + the tile-extreme table (gate: see WitnessGate; an open-ended
// gate {nullptr} always runs)
static void tile_pass(const Graph& g, Tags& T, cudaStream_t st, Scalars* sc, WitnessGate gate, bool skip_leaves = false) {
  const int B = 256;
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem);
  // (the table in k_tile's last block when it fits one CTA and a ticket word exists)
  Scalars* tsc = (sc && T.ntile <= kTableOneCta && T.tlev > 1) ? sc : nullptr;
  launch(k_tile, T.ntile < kNumSMs * kTileCtas ? T.ntile : kNumSMs * kTileCtas, kTileThreads, kTileSmem, st, T.AP, 2 * (int64_t)g.n, T.ntile,
         T.lh1, T.lh2, T.table, tsc, T.tlev, T.tour_len, gate, skip_leaves);
  note(K_TILE);
  if (tsc) {
  } else if (T.ntile <= kTableOneCta) {
    if (T.tlev > 1) {
      launch(k_table_all, 1, 1024, 0, st, T.table, T.ntile, T.tlev, T.tour_len, gate);
      note(K_TABLE);
    }
  } else {
    for (int k = 1; k < T.tlev; k++) {
      launch(k_table_level, grid_for(T.ntile, B), B, 0, st, T.table, T.ntile, k, T.tour_len, gate);
      note(K_TABLE);
    }
  }
}

void stage3_tags(const Graph& g, const Rooting& R, Tags& T, cudaStream_t st, int* nlow, const Side* side, int* uoff,
                 void* cub_tmp, size_t cub_bytes, Scalars* sc, const Witness* W) {
  const int B = 256;
  int64_t nchunks = (g.m + kItems - 1) / kItems;
  const bool witness = W && W->on;
  const WitnessGate none{nullptr, 0, 0};
  if (!nlow) {  // stand-alone compute_tags: the reference's exact w2
    if (g.m > 0)
      launch(k_w_gather<true>, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj, g.crow, g.n, g.m, R.rec, nullptr, T.AP,
             nullptr, none);
  } else if (witness) {
    launch(k_w_sample, grid_for(g.n, B), B, 0, st, g.off, g.n, (const int4*)R.rec, W->w0, T.AP, T.tour_len, T.lh1);
    note(K_W_SAMPLE);
  } else {
    // compact first[] lives in lh1 until k_tile overwrites it
    int* firsts = reinterpret_cast<int*>(T.lh1);
    if (R.firsts != firsts || R.nlow != nlow) {  // (else k_positions wrote both)
      launch(k_firsts, grid_for(g.n, B), B, 0, st, R.rec, g.n, firsts, nlow, none);
      note(K_FIRSTS);
    }
    if (g.m > 0)
      launch(k_w_gather<false>, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj, g.crow, g.n, g.m, R.rec, firsts,
             T.AP, nlow, none);
  }
  if (g.m > 0 && !witness) {
    note(K_W_GATHER);
  }
  if (nlow && witness && !side) {  // (no second stream: the lower-degree counts here, the scan in Stage 6)
    compute_nlow(g, nlow, st);
  }
  if (side && nlow) {  // nlow is final: Stage 6's upper-degree scan runs beside Stages 3-5
    cudaEventRecord(side->ev[0], st);
    cudaStreamWaitEvent(side->s, side->ev[0], 0);
    if (witness) compute_nlow(g, nlow, side->s);  // (the full gather counts them; the sampled one cannot)
    scan_upper_degrees(g.off, nlow, g.n, uoff, cub_tmp, cub_bytes, side->s);
    note(K_SCAN);
    cudaEventRecord(side->ev[1], side->s);
  }
  tile_pass(g, T, st, sc, none, witness);
}

// ---------------------------------------------------------------------------
// Stage 4: combine, fence bit
// ---------------------------------------------------------------------------
// kPhaseA (witness plans): the tags came from k_w_sample.  A bit that comes
// out 0 has a witness; one that comes out 1 is exact when no row under v was
// cut short (bit 30 of the subtree maximum clear) or v hangs off a root (always
// a fence); the rest -- written 1 for now -- are listed for k_witness_fix.
template <bool kPhaseA>
__global__ void k_fence(int n, int4* rec, const int2* __restrict__ lh1, const int2* __restrict__ lh2,
                        const int2* __restrict__ table, int ntile, int* low_out, int* high_out,
                        int* __restrict__ head, int* __restrict__ cnt, int* __restrict__ bmin, const int* tlen,
                        WitnessGate gate, int* __restrict__ und_list, Scalars* sc, int* __restrict__ label5,
                        unsigned long long* __restrict__ prop5, bool s5_if_ordered) {
  pdl_enter();
  if (!kPhaseA && !gate.open()) return;
  if (label5 && s5_if_ordered && !id_ordered(sc, n)) label5 = nullptr;  // (k_hook_min runs instead)
  const int64_t N = list_positions(tlen, 2 * (int64_t)n);
  int near = 0;
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
    bool cut = false;  // some row under v was sampled, not scanned
    if (kPhaseA) {
      cut = (res.y & kExactBit) != 0;
      res.y &= ~kExactBit;
    }
    int fence = 0;
    if (r.z >= 0) {
      int4 pr = rec[r.z];
      fence = (res.x >= pr.x && res.y <= pr.y) ? 1 : 0;
      if (kPhaseA && fence && cut && pr.z >= 0) {  // undecided
        const int span = r.y - r.x + 1;
        if (span > kWitnessMaxSubtree) sc->und_big = 1;
        const int at = atomicAdd(&sc->und_n, 1);
        if (at < gate.cap) und_list[at] = v;
        atomicAdd(&sc->und_work, (unsigned long long)span);
      }
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
    // Stage 5's sampling round 0 along plain parent edges (k_hook_min's
    // parent-only form, one pass and one record gather fewer): the parent
    // record is already here.  A bit still open in phase A counts as a fence
    // -- the vertex stays a root, and the link pass covers its tree edge.
    if (label5) {
      const bool hook = r.z >= 0 && fence == 0 && r.z < v;
      label5[v] = hook ? r.z : v;
      prop5[v] = ~0ull;
      near += hook && v - r.z <= kNear;
    }
  }
  if (label5) {
    // (a redo after an overflowed repair counts twice: the count only picks Stage 5's compress variant)
    block_count_add(&sc->near[1], near);
  }
}

// The listed vertices' fence bits from every row under them: one warp per
// vertex walks its tour interval; an entry position names a vertex of the
// subtree, whose row the warp scans.  When the gate is open (too many listed,
// or too much under them) the full gather takes over instead, and this kernel
// only restores the (first, first) start values it accumulates into.
__global__ void __launch_bounds__(256) k_witness_fix(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                     int n, int4* rec, int4* AP, const int* __restrict__ und_list,
                                                     const int* __restrict__ tlen, WitnessGate gate) {
  pdl_enter();
  const int N = *tlen;
  if (gate.open()) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
      const int f = __ldg(&rec[v].x);
      if (f < N) *reinterpret_cast<int2*>(AP + f) = make_int2(f, f);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int cnt = gate.sc->und_n;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < cnt; i += warps) {
    const int v = und_list[i];
    const int4 r = rec[v];
    int lo = r.x, hi = r.x;
    auto take = [&](int w, int px) {
      if (w == px) return;  // the tree edge to the parent
      const int f = __ldcg(&rec[w].x);
      lo = min(lo, f);
      hi = max(hi, f);
    };
    // 32 tour positions at a time, a lane each; rows over 64 arcs by the whole warp
    for (int p0 = r.x; p0 <= r.y; p0 += 32) {
      const int p = p0 + lane;
      const int x = p <= r.y ? AP[p].z : -1;  // (< 0: an exit position)
      int px = -1;
      int64_t rs = 0, re = 0;
      if (x >= 0) {
        px = __ldcg(&rec[x].z);
        rs = __ldg(off + x);
        re = __ldg(off + x + 1);
      }
      const bool big = re - rs > 64;
      if (!big)
        for (int64_t a = rs; a < re; a++) take((int)__ldg(adj + a), px);
      unsigned bm = __ballot_sync(0xffffffffu, big);
      while (bm) {
        const int src = __ffs(bm) - 1;
        bm &= bm - 1;
        const int bpx = __shfl_sync(0xffffffffu, px, src);
        const int64_t bs = __shfl_sync(0xffffffffu, rs, src), be = __shfl_sync(0xffffffffu, re, src);
        for (int64_t a = bs + lane; a < be; a += 32) take((int)__ldg(adj + a), bpx);
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      const int4 pr = rec[r.z];
      reinterpret_cast<int*>(rec + v)[3] = (lo >= pr.x && hi <= pr.y) ? 1 : 0;
    }
  }
}

void stage4_fence(const Graph& g, const Rooting& R, Tags& T, int* low_out, int* high_out, int* head, int* cnt,
                  int* bmin, cudaStream_t st, Scalars* sc, const Witness* W, int* label5, unsigned long long* prop5,
                  bool s5_if_ordered) {
  const int B = 256;
  const WitnessGate gate = gate_of(W, sc);
  if (!(W && W->on)) {
    launch(k_fence<false>, grid_for(g.n, B), B, 0, st, g.n, R.rec, T.lh1, T.lh2, T.table, T.ntile, low_out, high_out,
           head, cnt, bmin, T.tour_len, gate, (int*)nullptr, sc, label5, prop5, s5_if_ordered);
    note(K_FENCE);
    return;
  }
  // witness plan: fence bits from the sampled tags, the open ones repaired;
  // then the full gather / tile / fence -- which return at once unless the
  // repair list overflowed (WitnessGate)
  launch(k_fence<true>, grid_for(g.n, B), B, 0, st, g.n, R.rec, T.lh1, T.lh2, T.table, T.ntile, (int*)nullptr,
         (int*)nullptr, head, cnt, bmin, T.tour_len, gate, W->und_list, sc, label5, prop5, s5_if_ordered);
  note(K_FENCE);
  launch(k_witness_fix, grid_for((int64_t)W->cap * 32, B, 16), B, 0, st, g.off, g.adj, g.n, R.rec, T.AP,
         (const int*)W->und_list, T.tour_len, gate);
  note(K_WITNESS_FIX);
  const int64_t nchunks = (g.m + kItems - 1) / kItems;
  if (g.m > 0) {
    // (the redo's compact first[]: built only then, into the witness plan's own array)
    launch(k_firsts, grid_for(g.n, B), B, 0, st, (const int4*)R.rec, g.n, W->firsts, (int*)nullptr, gate);
    note(K_FIRSTS);
    launch(k_w_gather<false, false>, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj,
           W->crow_built ? g.crow : (const int*)nullptr, g.n, g.m, R.rec,
           (const int*)W->firsts, T.AP, (int*)nullptr, gate);
    note(K_W_GATHER);
  }
  tile_pass(g, T, st, sc, gate);
  launch(k_fence<false>, grid_for(g.n, B), B, 0, st, g.n, R.rec, T.lh1, T.lh2, T.table, T.ntile, (int*)nullptr,
         (int*)nullptr, head, cnt, bmin, T.tour_len, gate, (int*)nullptr, sc, label5, prop5, s5_if_ordered);
  note(K_FENCE);
}

}  // namespace fbcc
