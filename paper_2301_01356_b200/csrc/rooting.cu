// rooting.cu -- Stage 2: root the spanning forest with one Euler tour and
// list ranking.
//
// Replaces _rooted_from_claims / _rooted_from_csr (euler_tour.py:397-437):
// tree CSR by counting sort (_claims_csr 92-131), circuit linking
// (_link_circuit 134-145), root cut (_cut_roots 148-158), list ranking with
// sqrt(L) splitters + a sequential splitter pass (list_ranking 322-358),
// per-tree bases (_tree_bases 250-259, sequential) and the per-vertex gather
// (_vertex_positions 262-294).
//
// B200 design:
//  * Element numbering without a tree CSR.  Stage 1 records the forest edge
//    that hooked vertex x at fe[x]; list elements 2x and 2x+1 are that
//    edge's two arcs (u->v, v->u).  A root r has no such edge, and its pair
//    2r / 2r+1 becomes the virtual enter(r) / exit(r) of its tree.  So the
//    whole forest is 2n elements with no holes and no compaction.
//  * Euler circuit: every vertex's out-arcs form a list built by one
//    atomicExch per arc (no degree histogram, scan or scatter).  Arriving at
//    t through arc e, the tour leaves through the out-arc after e^1 in t's
//    list, wrapping to the first (non-root) or to exit(t) (root).
//  * ONE list for the forest: enter(r) -> first out-arc of r ... -> exit(r)
//    -> enter(next root by id).  Its head is element 0 (vertex 0 is always a
//    root) and each element's rank IS its tour position in the reference
//    layout (tree of root r owns [base_r, base_r + 2 size_r), root at both
//    ends, trees in root-id order, euler_tour.py:12-17).
//  * Ruling-set list ranking: one hash-placed splitter per window of S ids
//    (splitter index = window index: no compaction; structured tours such as
//    a chain's return path, which touches every other id, are still cut);
//    each splitter walks to the next writing (segment, offset) per element;
//    recurse on the weighted splitter list until it fits one CTA (Wyllie
//    pointer jumping in shared memory).  Level-0 ranks are expanded in one
//    coalesced pass: rank(e) = offs1[own0[e].seg] + own0[e].off.
//  * Positions: one thread per vertex x reads rank[2x..2x+1] as ONE 8-byte
//    load; the earlier of the two arcs is the down arc, giving the child's
//    parent, first and last.  It also initialises the tour-indexed array the
//    tag stage reads, one 16-byte record per position (AP: (first, first) at
//    entry, filler at exit; vertex id + partner position).
#include <cub/device/device_scan.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

// ---------------------------------------------------------------------------
// scans (CUB)
// ---------------------------------------------------------------------------
size_t scan_temp_bytes(int64_t items) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr, (int)items);
  return bytes;
}

void exclusive_scan(const int* in, int* out, int64_t items, void* tmp, size_t tmp_bytes, cudaStream_t st) {
  size_t bytes = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)items, st);
}

// rootidx: one 64-bit scan gives both ranks of a root -- among the listed
// roots (low word) and among the detached ones (high word)
struct RootCode {
  __host__ __device__ unsigned long long operator()(int c) const {
    return c == 1 ? 1ull : (c == 2 ? (1ull << 32) : 0ull);
  }
};
using RootIt = cub::TransformInputIterator<unsigned long long, RootCode, const int*>;

size_t scan_roots_temp_bytes(int64_t items) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, RootIt(nullptr, RootCode{}), (unsigned long long*)nullptr,
                                (int)items);
  return bytes;
}

void scan_roots(const int* flags, unsigned long long* out, int64_t items, void* tmp, size_t tmp_bytes,
                cudaStream_t st) {
  size_t bytes = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, bytes, RootIt(flags, RootCode{}), out, (int)items, st);
}

__device__ __forceinline__ int lo32(unsigned long long x) { return (int)(uint32_t)x; }
__device__ __forceinline__ int hi32(unsigned long long x) { return (int)(x >> 32); }

// ranks of root x: rootidx[x], plus its tile's prefix when the scan was split
// between Stage 1's final compress (ranks inside 1024-vertex tiles) and
// k_scan_tiles (tile prefixes) -- the prefixes are n / 1024 words, L2-resident
constexpr int kRootTile = 1024;  // vertices per compress tile (256 threads x 4)
__device__ __forceinline__ unsigned long long root_rank(const unsigned long long* __restrict__ rootidx,
                                                        const unsigned long long* __restrict__ tile_pre, int x) {
  const unsigned long long r = __ldg(rootidx + x);
  return tile_pre ? r + __ldg(tile_pre + x / kRootTile) : r;
}

// list / component counts from rootidx[n]
__device__ __forceinline__ void publish_roots(const unsigned long long* rootidx, int n, Scalars* sc) {
  const unsigned long long t = rootidx[n];
  sc->ncomp = lo32(t) + hi32(t);
  sc->nlisted = lo32(t);
  sc->tour_len = 2 * (n - hi32(t));
}

// Edge numbering: uoff[v] = upper arcs (u -> w, u < w) of the rows before v,
// v in [0, n]; uoff[n] = E.  Two levels like the root scan, no library call:
// k_updeg_local writes each vertex's prefix inside its 1024-vertex tile and
// the tile's sum, k_scan_tiles (one CTA) the tile prefixes; Stage 6 adds the
// two as it reads them (UpOff, kernels.cuh).  (Off the critical path: the pipeline runs it on its side
// stream beside Stages 3-5.)
// (kUpTile = 1024, kernels.cuh: 256 threads x 4 consecutive vertices)
__global__ void k_scan_tiles(unsigned long long* __restrict__ tiles, int ntiles,
                             unsigned long long* __restrict__ total_out, int n, Scalars* sc);

__global__ void __launch_bounds__(256) k_updeg_local(const int64_t* __restrict__ off, const int* __restrict__ nlow,
                                                     int n, int* __restrict__ uoff,
                                                     unsigned long long* __restrict__ tsum) {
  pdl_enter();
  __shared__ int wtot[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int64_t base = (int64_t)blockIdx.x * kUpTile; base < n; base += (int64_t)gridDim.x * kUpTile) {
    const int v0 = (int)base + 4 * t;
    int u[4];
#pragma unroll
    for (int i = 0; i < 4; i++)
      u[i] = v0 + i < n ? (int)(__ldg(off + v0 + i + 1) - __ldg(off + v0 + i)) - __ldg(nlow + v0 + i) : 0;
    const int sum = u[0] + u[1] + u[2] + u[3];
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
      const int x = wtot[w];
      if (w < warp) before += x;
      total += x;
    }
    int run = before + incl - sum;
#pragma unroll
    for (int i = 0; i < 4; i++)
      if (v0 + i < n) {
        uoff[v0 + i] = run;
        run += u[i];
      }
    if (t == 0) tsum[base / kUpTile] = (unsigned long long)total;
    __syncthreads();  // wtot is rewritten by the next tile
  }
}

size_t scan_upper_temp_bytes(int n) { return 8 * ((size_t)n / kUpTile + 2); }

void scan_upper_degrees(const int64_t* off, const int* nlow, int n, int* uoff, void* tmp, size_t tmp_bytes,
                        cudaStream_t st) {
  (void)tmp_bytes;
  unsigned long long* tsum = reinterpret_cast<unsigned long long*>(tmp);
  const int ntiles = (n + kUpTile - 1) / kUpTile;
  launch(k_updeg_local, grid_for(ntiles, 1, 8), 256, 0, st, off, nlow, n, uoff, tsum);
  launch(k_scan_tiles, 1, 1024, 0, st, tsum, ntiles, tsum + ntiles, n, (Scalars*)nullptr);
}

// ---------------------------------------------------------------------------
// roots in id order
// ---------------------------------------------------------------------------
// (also clears the out-arc list heads: same index space, no memset node)
//
// Hub split: every forest edge inserts its two arcs at the heads of its
// endpoints' lists with atomicExch, so a vertex of tree degree d serialises d
// returning atomics on one address (RMAT hubs: ~1e5, 2 ms).  Vertices of
// CSR degree >= kHubDeg instead get W sub-lists (the inserting edge x picks
// x & (W - 1); W = 32 .. 16384 by degree, see hub_log_ways: on RMAT the
// biggest hubs' inserts queued on 32 addresses -- out_lists 1.15 -> 0.58 ms),
// whose heads live at hsub[(off[v] >> 4) + j] -- disjoint, W <= deg/16 --
// and lhead[v] = hub_marker(base, log2 W) marks the vertex.
// The tour walks a hub's sub-lists in order (k_link_tour).

__global__ void k_root_flags(const int* __restrict__ comp, int n, int* __restrict__ flags, int* __restrict__ lhead,
                             const int64_t* __restrict__ off, int* __restrict__ hsub, const Scalars* sc) {
  pdl_enter();
  if (off && !sc->has_hubs) off = nullptr;  // (k_chunk_rows saw no row that long)
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x) {
    flags[v] = (v < n) ? (__ldg(comp + v) == v) : 0;
    if (v < n) {
      int h = -1;
      if (off) {
        const int64_t rs = __ldg(off + v);
        if (__ldg(off + v + 1) - rs >= kHubDeg) {
          const int base = (int)(rs >> 4);
          const int lw = hub_log_ways(__ldg(off + v + 1) - rs);
          for (int j = 0; j < (1 << lw); j++) hsub[base + j] = -1;
          h = hub_marker(base, lw);
        }
      }
      lhead[v] = h;
    }
  }
}

// rlist[rank among roots] = root;  sc->ncomp = c (every root listed: codes 0/1)
__global__ void k_root_list(const int* __restrict__ comp, const unsigned long long* __restrict__ rootidx, int n,
                            int* __restrict__ rlist, Scalars* sc) {
  pdl_enter();
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) publish_roots(rootidx, n, sc);
  for (int r = (int)tid; r < n; r += gridDim.x * blockDim.x)
    if (__ldg(comp + r) == r) rlist[lo32(__ldg(rootidx + r))] = r;
}

// Second level of the root scan fused into Stage 1's final compress (see
// k_compress<kScan>): tile root counts -> exclusive prefixes, in place, by
// one CTA (n / 1024 entries: 33 k on config 5, 98 k at n = 1e8); also the
// totals (rootidx[n]) and the counts derived from them.
// (sc != nullptr: the root scan -- total_out is rootidx + n, and the counts derived
// from the totals are published; nullptr: the upper-degree scan, total only)
__global__ void __launch_bounds__(1024) k_scan_tiles(unsigned long long* __restrict__ tiles, int ntiles,
                                                     unsigned long long* __restrict__ total_out, int n, Scalars* sc) {
  pdl_enter();
  __shared__ unsigned long long wtot[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // each warp owns one contiguous segment (a multiple of 32 counts): lane
  // sums, the 32 segment totals scanned by warp 0, then a shuffle scan per
  // 32 counts along the segment -- two barriers in all, every access coalesced
  const int seg = ((ntiles + 1023) / 1024) * 32;
  const int lo = min(warp * seg, ntiles), hi = min(lo + seg, ntiles);
  unsigned long long sum = 0;
#pragma unroll 4
  for (int i = lo + lane; i < hi; i += 32) sum += tiles[i];
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) wtot[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long x = wtot[lane];
    unsigned long long w = x;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wtot[lane] = w - x;
    if (lane == 31) {
      *total_out = w;
      if (sc) publish_roots(total_out - n, n, sc);
    }
  }
  __syncthreads();
  unsigned long long run = wtot[warp];
  unsigned long long nxt = lo + lane < hi ? tiles[lo + lane] : 0ull;
  for (int i0 = lo; i0 < hi; i0 += 32) {
    const unsigned long long x = nxt;
    if (i0 + 32 < hi) nxt = i0 + 32 + lane < hi ? tiles[i0 + 32 + lane] : 0ull;  // (in flight under this step's scan)
    unsigned long long incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (i0 + lane < hi) tiles[i0 + lane] = run + incl - x;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// out-arc lists: arc 2x = u->v is an out-arc of u, 2x+1 = v->u of v
__device__ __forceinline__ int* list_head(int* lhead, int* hsub, int t, int x, bool split) {
  if (split) {
    const int h = ld_relaxed(lhead + t);  // concurrent exchanges leave non-hubs >= -1
    if (h <= -2) return hsub + hub_base(h) + (x & (hub_ways(h) - 1));
  }
  return lhead + t;
}

// (rootidx != nullptr: also k_root_list's work -- roots placed in id order,
// c published -- in the same pass over the vertices)
__global__ void k_out_lists(const int* __restrict__ comp, const int2* __restrict__ fe, int n, int* lhead,
                            int* __restrict__ nexto, int* hsub, Scalars* sc,
                            const unsigned long long* __restrict__ rootidx, const int* __restrict__ flags,
                            int* __restrict__ rlist, const unsigned long long* __restrict__ tile_pre) {
  pdl_enter();
  const bool split = hsub != nullptr && sc->has_hubs;
  if (rootidx && !tile_pre && blockIdx.x == 0 && threadIdx.x == 0) publish_roots(rootidx, n, sc);
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    if (__ldg(comp + x) == x) {
      if (rootidx && __ldg(flags + x) == 1) rlist[lo32(root_rank(rootidx, tile_pre, x))] = x;
      continue;
    }
    int2 e = __ldg(fe + x);
    nexto[2 * x] = atomicExch(list_head(lhead, hsub, e.x, x, split), 2 * x);
    nexto[2 * x + 1] = atomicExch(list_head(lhead, hsub, e.y, x, split), 2 * x + 1);
  }
}

// first non-empty hub sub-list head at or after way j (-1: none)
__device__ __forceinline__ int hub_next(const int* __restrict__ hsub, int h, int j) {
  const int base = hub_base(h), W = hub_ways(h);
  for (; j < W; j++) {
    const int head = __ldg(hsub + base + j);
    if (head >= 0) return head;
  }
  return -1;
}

// ---------------------------------------------------------------------------
// ruling-set list ranking
// ---------------------------------------------------------------------------
// splitter of window j (element j*S + hashed offset; window 0 uses element 0,
// the list head; the last, partial window is clamped into range); S = 1 << sh
__device__ __forceinline__ int split_elem(int j, int sh, int N) {
  int e = (j << sh) + (j == 0 ? 0 : (int)(hash32((uint32_t)j * 0x9E3779B1u + 0x7F4A7C15u) & ((1u << sh) - 1)));
  return e < N ? e : N - 1;
}
__device__ __forceinline__ bool is_split(int e, int sh, int N) { return split_elem(e >> sh, sh, N) == e; }

// Successor encoding on every ranking level: s >= 0 is an ordinary next
// element, -1 ends the list, s <= -2 says the next element ~s is a splitter
// of the level's windowing (the head, element 0, is nobody's successor, so
// ~0 = -1 is free).  The producer of the array -- k_link_tour for level 0,
// the walkers of level l for level l+1 -- tests the target once, so a walker
// step is one dependent load and a sign test: the walk's critical path is
// the L2 round trip alone (the hash test and 64-bit division it replaced
// added ~100 cycles per step, and the slowest walker takes ~S ln K steps).
__device__ __forceinline__ int flag_succ(int s, int sh, int N) {
  return (s >= 0 && sh >= 0 && is_split(s, sh, N)) ? ~s : s;
}

// A detached root's pair is no list element: both end at once (-1).  Should
// the hash pick one as a splitter, its walker stops there and leaves a
// detached element on the next level -- unreachable from the head, never
// read back (k_positions places detached roots from rootidx).
struct TourArgs {
  const int* comp;
  const int2* fe;
  const int* lhead;
  const int* hsub;
  const int* nexto;
  const unsigned long long* rootidx;
  const unsigned long long* tile_pre;
  const int* flags;
  const int* rlist;
};

// successor of list element e (-1: end of the list); c = listed roots
__device__ __forceinline__ int tour_succ(const TourArgs& a, int64_t e, int c) {
  const int x = (int)(e >> 1);
  if (__ldg(a.comp + x) == x) {  // enter(x) / exit(x)
    if (__ldg(a.flags + x) == 2) return -1;
    if ((e & 1) == 0) {
      int h = __ldg(a.lhead + x);
      if (h <= -2) h = hub_next(a.hsub, h, 0);
      return h >= 0 ? h : (int)e + 1;
    }
    const int ri = lo32(root_rank(a.rootidx, a.tile_pre, x));
    return (ri + 1 < c) ? 2 * __ldg(a.rlist + ri + 1) : -1;
  }
  // arc e arrives at t; leave through the out-arc after e^1
  const int2 uv = __ldg(a.fe + x);
  const int t = (e & 1) ? uv.x : uv.y;
  int nx = __ldg(a.nexto + (e ^ 1));
  if (nx >= 0) return nx;
  // end of t's list (of a hub's sub-list: the next non-empty one)
  const int h = __ldg(a.lhead + t);
  if (h <= -2) nx = hub_next(a.hsub, h, (x & (hub_ways(h) - 1)) + 1);
  if (nx >= 0) return nx;
  if (__ldg(a.comp + t) == t) return 2 * t + 1;
  return h <= -2 ? hub_next(a.hsub, h, 0) : h;
}

// (small tours: the successors go to their own array, k_walk<false, false> reads them)
__global__ void k_link_tour(TourArgs a, int n, int* __restrict__ nxt, const Scalars* sc, int sh0) {
  pdl_enter();
  const int c = sc->nlisted;
  const int64_t N = 2 * (int64_t)n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    nxt[e] = flag_succ(tour_succ(a, e, c), sh0, (int)N);
}

// Large tours (level 0 in place): the successor goes into the element's
// (segment, offset) slot, which the level-0 walker reads and then overwrites
// (one sector per visited element instead of a successor sector plus a
// partial write).  The kernel also ranks, in shared memory, every level-0
// segment that lies inside one 2048-element tile: the tile's successors are
// staged, each of its 128 splitters walks its segment there (~30 cycles a
// step instead of an L2 round trip), and a segment that ends inside the tile
// is written out finished -- (segment, offset) per element, weight and next
// splitter per segment.  On id-ordered tours (meshes, paths: consecutive tour
// elements are 16 bytes apart) that is nearly every segment, and k_walk's
// level-0 pass -- one L2 read and one partial write per step, bound by the L2
// operation rate (4c: 1.71 ms, lts 63 %) -- is left with the few segments
// that cross a tile boundary.  A random tour (RMAT) completes none and pays
// one shared-memory step per splitter.
constexpr int kLinkTile = 2048;
constexpr int kNotWalked = (int)0x80000000;  // succ_next[j]: segment j is k_walk's

__global__ void __launch_bounds__(256) k_link_walk(TourArgs a, int n, int2* __restrict__ own0, const Scalars* sc,
                                                   int sh0, int K1, int* __restrict__ succ_next,
                                                   int* __restrict__ w_next, int sh_next) {
  pdl_enter();
  __shared__ int S[kLinkTile];     // successor of each tile element (flagged)
  __shared__ int2 R[kLinkTile];    // finished (segment, offset); .x == kNotWalked: not finished
  const int c = sc->nlisted;
  const int N = 2 * n;
  const int t = threadIdx.x;
  // tile-local ranking only where it pays: Stage 1's round 0 hooked >= 3/4 of
  // the vertices to a near id, so the forest -- and the tour -- follow the id order
  const bool ordered = (int64_t)sc->near[0] * 4 >= (int64_t)n * 3;
  constexpr int kPer = kLinkTile / 256;
  if (!ordered) {  // a random tour: no segment stays inside a tile -- successors only, every segment is k_walk's
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + t, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = tid; e < N; e += stride) own0[e] = make_int2(flag_succ(tour_succ(a, e, c), sh0, N), 0);
    for (int64_t j = tid; j < K1; j += stride) succ_next[j] = kNotWalked;
    return;
  }
  for (int64_t base = (int64_t)blockIdx.x * kLinkTile; base < N; base += (int64_t)gridDim.x * kLinkTile) {
#pragma unroll
    for (int i = 0; i < kPer; i++) {
      const int r = i * 256 + t;
      const int64_t e = base + r;
      S[r] = e < N ? flag_succ(tour_succ(a, e, c), sh0, N) : -1;
      R[r].x = kNotWalked;
    }
    __syncthreads();
    // one splitter per window of 1 << sh0 ids: window j's is split_elem(j)
    const int wins = kLinkTile >> sh0;
    for (int wi = t; wi < wins; wi += 256) {
      const int j = (int)(base >> sh0) + wi;
      if (j >= K1) break;
      const int e0 = split_elem(j, sh0, N);
      int e = e0, len = 0, s;
      bool inside = true;
      while (true) {  // walk the staged successors, ranking as it goes
        const int r = e - (int)base;
        s = S[r];
        R[r] = make_int2(j, len++);
        if (s < 0) break;
        if (s < (int)base || s >= (int)base + kLinkTile) { inside = false; break; }
        e = s;
      }
      if (!inside) {  // the segment leaves the tile: undo, k_walk ranks it
        e = e0;
        for (int off = 0; off < len; off++) {
          const int r = e - (int)base;
          R[r].x = kNotWalked;
          e = S[r];
        }
        succ_next[j] = kNotWalked;
        continue;
      }
      succ_next[j] = (s == -1) ? -1 : flag_succ((~s) >> sh0, sh_next, K1);
      w_next[j] = len;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPer; i++) {
      const int r = i * 256 + t;
      const int64_t e = base + r;
      if (e < N) {
        const int2 v = R[r];
        own0[e] = v.x == kNotWalked ? make_int2(S[r], 0) : v;
      }
    }
    __syncthreads();  // S / R are rewritten by the next tile
  }
}

// kInPlace (level 0 of large tours): the successors sit in own[e].x (written
// by k_link_tour) and are replaced by (segment, offset) as the walk passes --
// every element is read and then written by its own walker only.
template <bool kWeighted, bool kInPlace = false>
__global__ void __launch_bounds__(256) k_walk(int K, int sh, int N, const int* __restrict__ succ,
                                              const int* __restrict__ w, int2* __restrict__ own,
                                              int* __restrict__ succ_next, int* __restrict__ w_next, int sh_next) {
  pdl_enter();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x) {
    if (kInPlace && succ_next[j] != kNotWalked) continue;  // (k_link_walk finished the segment inside its tile)
    int e = split_elem(j, sh, N);
    int acc = 0;
    int s;
    while (true) {
      // (read-only path: an element is read strictly before its one write)
      s = kInPlace ? __ldg(reinterpret_cast<const int*>(own) + 2 * (int64_t)e) : __ldg(succ + e);
      // in place: the store must not reach L2 while the same sector's fill is
      // still pending (store-behind-miss on one sector ran ~9x slower), so
      // the stored value is made to depend on the loaded one (s == INT_MIN
      // never occurs: successors are >= -1 or flagged ~e with e >= 1)
      own[e] = make_int2(kInPlace ? (s == (int)0x80000000 ? -1 : j) : j, acc);
      acc += kWeighted ? __ldg(w + e) : 1;
      if (s < 0) break;
      e = s;
    }
    succ_next[j] = (s == -1) ? -1 : flag_succ((~s) >> sh, sh_next, K);
    w_next[j] = acc;
  }
}

// Final level: <= kFinalMax elements, head = element 0; exclusive weighted
// prefix along the list, entirely in shared memory (one CTA).
// The CTA runs one more ruling-set level in shared memory (one walker per
// thread over windows of Q = K/1024 elements, ~2 us of smem steps), then
// Wyllie over the <= 1024 walkers (10 rounds, one element per thread), then
// expands.  Block-wide Wyllie straight over 16K elements needed 14 rounds of
// 16 elements per thread (59 us measured).
constexpr int kFinalThreads = 1024;
constexpr size_t kFinalSmem = 2 * sizeof(int) * kFinalMax + 4 * sizeof(int) * kFinalThreads;

__global__ void __launch_bounds__(kFinalThreads) k_final_rank(int K, const int* __restrict__ succ,
                                                              const int* __restrict__ w, int* __restrict__ offs) {
  pdl_enter();
  extern __shared__ int fsm[];
  int* S = fsm;                    // succ, then owner walker
  int* W = fsm + kFinalMax;        // weight, then offset inside the walker's segment
  int* SS = W + kFinalMax;         // walker -> next walker
  int* WS = SS + kFinalThreads;    // walker segment weight
  int* PS = WS + kFinalThreads;    // walker predecessor
  int* VS = PS + kFinalThreads;    // walker exclusive prefix
  const int t = threadIdx.x;
  int qs = 0;  // one more ruling level in smem: windows of Q = 1 << qs elements
  while ((kFinalThreads << qs) < K) qs++;
  const int nwin = (K + (1 << qs) - 1) >> qs;
  // stage the level through registers: all 2 x 16 loads of a thread are in
  // flight together (a rolled loop waited ~0.5 us per element: 16 of them)
  constexpr int kPer = kFinalMax / kFinalThreads;
  int rs[kPer], rw[kPer];
#pragma unroll
  for (int i = 0; i < kPer; i++) {
    const int j = t + i * kFinalThreads;
    rs[i] = j < K ? __ldg(succ + j) : -1;
    rw[i] = j < K ? __ldg(w + j) : 0;
  }
#pragma unroll
  for (int i = 0; i < kPer; i++) {
    const int j = t + i * kFinalThreads;
    if (j < K) {
      S[j] = flag_succ(rs[i], qs, K);
      W[j] = rw[i];
    }
  }
  PS[t] = -1;
  __syncthreads();
  if (t < nwin) {
    int e = split_elem(t, qs, K);
    int acc = 0, s;
    while (true) {
      s = S[e];
      int wt = W[e];
      S[e] = t;
      W[e] = acc;
      acc += wt;
      if (s < 0) break;
      e = s;
    }
    SS[t] = (s == -1) ? -1 : (~s) >> qs;
    WS[t] = acc;
  }
  __syncthreads();
  if (t < nwin && SS[t] >= 0) PS[SS[t]] = t;
  __syncthreads();
  int p = PS[t];
  int v = (t < nwin && p >= 0) ? WS[p] : 0;
  VS[t] = v;
  __syncthreads();
  for (int round = 0; round < 11; round++) {
    int np = p, nv = v;
    if (p >= 0) { nv = v + VS[p]; np = PS[p]; }
    if (!__syncthreads_or(p >= 0)) break;
    p = np;
    v = nv;
    PS[t] = p;
    VS[t] = v;
    __syncthreads();
  }
  // (an element no walker reached -- a detached one -- keeps its successor
  // in S: its offset is never read, but must not index out of VS)
  for (int j = t; j < K; j += kFinalThreads) {
    const int o = S[j];
    offs[j] = (o >= 0 && o < kFinalThreads) ? VS[o] + W[j] : 0;
  }
}

// (own[j] of an element no walker reached -- detached, see k_link_tour --
// was never written: clamp the index, the value is never read)
__global__ void k_expand(int64_t K, const int2* __restrict__ own, const int* __restrict__ offs_up, int64_t K_up,
                         int* __restrict__ offs) {
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
    int2 o = own[j];
    offs[j] = ((uint32_t)o.x < (uint64_t)K_up) ? __ldg(offs_up + o.x) + o.y : 0;
  }
}

// ---------------------------------------------------------------------------
// positions: parent / first / last + tour-indexed tag arrays
// ---------------------------------------------------------------------------
// AP[first] = {first, first (w1 = w2 = own entry, gathered into by stage 3), v, last};
// AP[last] = {filler (tagging.py:33-39), ~v, first}: two 16 B stores per vertex
__device__ __forceinline__ void place(int v, int f, int l, int par, int4* rec, int4* AP, int* firsts) {
  rec[v] = make_int4(f, l, par, 0);
  if (firsts) firsts[v] = f;  // the pipeline: Stage 3's compact first[]
  AP[f] = make_int4(f, f, v, l);
  AP[l] = make_int4(kINF, -1, ~v, f);
}

// level-0 ranks, coalesced over elements (the offs1 gathers hit L2 here,
// instead of competing with the positions kernel's scattered stores)
__global__ void k_rank0(int64_t N, const int2* __restrict__ own0, const int* __restrict__ offs1, int64_t K1,
                        int* __restrict__ rank0) {
  pdl_enter();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    int2 o = __ldg(own0 + e);
    rank0[e] = ((uint32_t)o.x < (uint64_t)K1) ? __ldg(offs1 + o.x) + o.y : 0;  // (detached: unread)
  }
}

// (own0 != nullptr: the level-0 ranks are expanded here -- rank(e) =
// offs1[own0[e].seg] + own0[e].off, one 16-byte load for both elements of x
// -- instead of by k_rank0)
// A detached root x (code 2) is no list element: its tree is x alone, at
// positions tour_len + 2 d and + 1 (d = its rank among the detached, the
// high word of rootidx) -- one coalesced record, no AP entries (the tile
// pass stops at tour_len and Stage 4 answers low = high = first for it).
__global__ void k_positions(const int* __restrict__ comp, const int2* __restrict__ fe,
                            const int2* __restrict__ rank0, int n, int4* __restrict__ rec,
                            int4* __restrict__ AP, int* __restrict__ firsts, const int4* __restrict__ own0,
                            const int* __restrict__ offs1, const int* __restrict__ flags,
                            const unsigned long long* __restrict__ rootidx, const Scalars* sc,
                            const unsigned long long* __restrict__ tile_pre) {
  pdl_enter();
  const int tour_len = sc->tour_len;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    if (__ldg(flags + x) == 2) {
      const int f = tour_len + 2 * hi32(root_rank(rootidx, tile_pre, x));
      rec[x] = make_int4(f, f + 1, -1, 0);
      if (firsts) firsts[x] = f;
      continue;
    }
    int2 r;
    if (own0) {
      const int4 o = __ldg(own0 + x);  // (seg, off) of elements 2x and 2x+1
      r = make_int2(__ldg(offs1 + o.x) + o.y, __ldg(offs1 + o.z) + o.w);
    } else {
      r = __ldg(rank0 + x);  // ranks of elements 2x and 2x+1, one 8-byte load
    }
    if (__ldg(comp + x) == x) {
      place(x, r.x, r.y, -1, rec, AP, firsts);  // enter(x), exit(x)
    } else {
      int2 uv = __ldg(fe + x);
      if (r.x < r.y) place(uv.y, r.x, r.y, uv.x, rec, AP, firsts);  // u -> v is the down arc
      else place(uv.x, r.y, r.x, uv.y, rec, AP, firsts);
    }
  }
}

// roots in id order: rank among roots, the inverse list, c; clears lhead
void rooting_roots(int n, const int* comp, Rooting& R, Scalars* sc, cudaStream_t st) {
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  launch(k_root_flags, gv, B, 0, st, comp, n, R.flags, R.lhead, R.hoff, R.hoff ? R.hsub : nullptr, sc);
  note(K_ROOT_FLAGS);
  scan_roots(R.flags, R.rootidx, n + 1, R.cub_tmp, R.cub_bytes, st);
  note(K_SCAN);
  launch(k_root_list, gv, B, 0, st, comp, R.rootidx, n, R.rlist, sc);
  note(K_ROOT_LIST);
}

void stage2_rooting(const Graph& g, const int* comp, const int2* fe, Rooting& R, int4* AP,
                    Scalars* sc, cudaStream_t st) {
  rooting_roots(g.n, comp, R, sc, st);
  // Euler circuit: out-arc lists in atomicExch order (any order is a valid
  // tour; the final outputs do not depend on it)
  launch(k_out_lists, grid_for(g.n, 256), 256, 0, st, comp, fe, g.n, R.lhead, R.nexto, R.hoff ? R.hsub : nullptr, sc,
         (const unsigned long long*)nullptr, (const int*)nullptr, (int*)nullptr, (const unsigned long long*)nullptr);
  note(K_OUT_LISTS);
  rooting_tour(g.n, comp, fe, R, AP, sc, st);
}

void stage2_rooting_fused(const Graph& g, const int* comp, const int2* fe, Rooting& R, int4* AP, Scalars* sc,
                          cudaStream_t st) {
  // R.flags / R.lhead / R.hsub were written by Stage 1's final compress --
  // and the roots' ranks, when the scan ran inside it
  if (R.tile_roots) {
    launch(k_scan_tiles, 1, 1024, 0, st, R.tile_roots, (g.n + kRootTile - 1) / kRootTile, R.rootidx + g.n, g.n, sc);
    note(K_SCAN_TILES);
  } else {
    scan_roots(R.flags, R.rootidx, g.n + 1, R.cub_tmp, R.cub_bytes, st);
    note(K_SCAN);
  }
  launch(k_out_lists, grid_for(g.n, 256), 256, 0, st, comp, fe, g.n, R.lhead, R.nexto, R.hoff ? R.hsub : nullptr, sc,
         (const unsigned long long*)R.rootidx, (const int*)R.flags, R.rlist, (const unsigned long long*)R.tile_roots);
  note(K_OUT_LISTS);
  rooting_tour(g.n, comp, fe, R, AP, sc, st);
}

// tour linking, list ranking, positions (needs lhead/nexto built)
void rooting_tour(int n, const int* comp, const int2* fe, Rooting& R, int4* AP, Scalars* sc, cudaStream_t st) {
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  const int N0 = 2 * n;
  auto shift = [](int S) { return __builtin_ctz((unsigned)S); };
  // levels 1..nlev-1 are walked again (their successors carry splitter flags
  // for the next windowing); level nlev goes to the one-CTA final kernel
  auto sh_after = [&](int l) { return l < R.nlev ? shift(R.S[l]) : -1; };
  // level 0 in place once the tour outgrows L2 (own0 > 64 MB): DRAM-bound
  // walks gain (config 5 walk0 1.65 -> 0.92 ms), L2-resident ones lose
  // (config 2: the next element often shares the stored sector)
  const bool inplace = (int64_t)N0 * 8 > (64ll << 20) || !R.nxt;
  const TourArgs ta{comp, fe, R.lhead, R.hsub, R.nexto, R.rootidx, R.tile_roots, R.flags, R.rlist};
  if (inplace) {
    launch(k_link_walk, grid_for(N0, B), B, 0, st, ta, n, R.own0, (const Scalars*)sc,
           shift(R.S[0]), (int)R.K[1], R.succ[1], R.wgt[1], sh_after(1));
  } else {
    launch(k_link_tour, grid_for(N0, B), B, 0, st, ta, n, R.nxt, (const Scalars*)sc, shift(R.S[0]));
  }
  note(K_LINK_TOUR);
  // ruling-set levels
  launch(inplace ? k_walk<false, true> : k_walk<false, false>, grid_for(R.K[1], B, 64), B, 0, st, (int)R.K[1],
         shift(R.S[0]), N0, (const int*)R.nxt, (const int*)nullptr, R.own0,
                                                       R.succ[1], R.wgt[1], sh_after(1));
  note(K_WALK0);
  for (int l = 1; l < R.nlev; l++) {
    launch(k_walk<true>, grid_for(R.K[l + 1], B, 64), B, 0, st, (int)R.K[l + 1], shift(R.S[l]), (int)R.K[l], R.succ[l],
                                                            R.wgt[l], R.own[l], R.succ[l + 1], R.wgt[l + 1],
                                                            sh_after(l + 1));
    note(K_WALKL);
  }
  cudaFuncSetAttribute(k_final_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFinalSmem);
  launch(k_final_rank, 1, kFinalThreads, kFinalSmem, st, (int)R.K[R.nlev], R.succ[R.nlev], R.wgt[R.nlev],
                                                      R.offs[R.nlev]);
  note(K_FINAL_RANK);
  for (int l = R.nlev - 1; l >= 1; l--) {
    launch(k_expand, grid_for(R.K[l], B), B, 0, st, R.K[l], R.own[l], R.offs[l + 1], R.K[l + 1], R.offs[l]);
    note(K_EXPAND);
  }
#ifndef FBCC_FUSED_RANK0
#define FBCC_FUSED_RANK0 1
#endif
  if (FBCC_FUSED_RANK0) {
    launch(k_positions, gv, B, 0, st, comp, fe, (const int2*)nullptr, n, R.rec, AP, R.firsts,
           reinterpret_cast<const int4*>(R.own0), (const int*)R.offs[1], (const int*)R.flags,
           (const unsigned long long*)R.rootidx, (const Scalars*)sc, (const unsigned long long*)R.tile_roots);
    note(K_POSITIONS);
  } else {
    launch(k_rank0, grid_for(N0, B), B, 0, st, N0, R.own0, R.offs[1], R.K[1], R.rank0);
    note(K_RANK0);
    launch(k_positions, gv, B, 0, st, comp, fe, reinterpret_cast<const int2*>(R.rank0), n, R.rec, AP, R.firsts,
           (const int4*)nullptr, (const int*)nullptr, (const int*)R.flags, (const unsigned long long*)R.rootidx,
           (const Scalars*)sc, (const unsigned long long*)R.tile_roots);
    note(K_POSITIONS);
  }
}

}  // namespace fbcc
