// common.cuh -- shared device helpers for the FAST-BCC sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace fbcc {

constexpr int kNumSMs = 148;   // B200
constexpr int kINF = 0x7FFFFFFF;
// round 0 hooks a vertex to a smaller neighbour (Stage 5: its plain parent) within
// this many ids in preference to the minimum one (meshes: connectivity.cu round0_target)
#ifndef FBCC_NEAR
#define FBCC_NEAR 64
#endif
constexpr int kNear = FBCC_NEAR;

// Device-side scalars shared by the stages (lives at the head of the
// workspace).  Counts that only the device knows stay here so that no stage
// needs a host round trip (the whole run is one asynchronous stream).
struct alignas(8) Scalars {
  int ncomp;       // c: number of components of the first pass (roots)
  int giant;       // sampled most-frequent root (Afforest skip)
  int nbccs;       // number of blocks
  int err;         // error bits
  int num_edges;   // E
  int nroots[16];  // roots after each sampling round's compress (stage 1: 0..7, stage 5: 8..15)
  int hooks[16];   // hooks accepted per sampling round (same split)
  int nheavy[2];   // super-heavy rows deferred by k_link_rows, CTA tier (stage 1 / stage 5 slot)
  int has_hubs;    // some row has >= kHubDeg slots (set by k_chunk_rows)
  unsigned ticket; // last-block detection (k_compress; reset by the last block)
  int giant_cnt;   // samples (of 1024) that fell in the giant at its pick
  unsigned tile_ticket;  // k_tile: last block builds the tile-extreme table (reset by it)
  int eheavy;      // Stage 6: super-heavy non-giant rows deferred by k_edge_fix (CTA tier)
  int nmega[2];    // ... grid tier of nheavy
  int emega;       // ... grid tier of eheavy
  int nlisted;     // roots on the Euler-tour list (code 1)
  int tour_len;    // list elements = 2 (n - detached roots); detached positions follow
  int near[2];     // round-0 hooks to a vertex within kNear ids (stage 1 / stage 5): id-ordered chains (meshes)
  int jlist_n[2];  // exit targets listed by k_jump_local (same split)
  int und_n;       // witness tags: vertices whose sampled arcs left their fence bit undecided (k_fence phase A)
  unsigned long long und_work;  // ... tour positions under all of them (8-byte aligned: 54 ints precede it)
  int und_big;     // ... one of them with a subtree too large for k_witness_fix
  int pad[7];
};

// Stage 1's round 0 hooked >= 3/4 of the vertices to a near id: the forest, the
// tour and the plain parent edges follow the id order (tori, paths)
__device__ __forceinline__ bool id_ordered(const Scalars* sc, int n) {
  return (long long)sc->near[0] * 4 >= (long long)n * 3;
}

// ---------------------------------------------------------------------------
// launch log: counts every launch of ours and, in profile mode, brackets
// each with CUDA events on the launching stream (per-kernel device time)
// ---------------------------------------------------------------------------
enum KernelKind : int {  // one kind per kernel function (names: api.cu kKernelNames)
  K_CHUNK_ROWS = 0, K_HOOK_MIN, K_IOTA, K_PROPOSE, K_ACCEPT, K_COMPRESS, K_FIND_GIANT, K_LINK_ROWS, K_LINK_HEAVY,
  K_ROOT_FLAGS, K_SCAN, K_ROOT_LIST, K_OUT_LISTS, K_LINK_TOUR, K_WALK0, K_WALKL, K_FINAL_RANK, K_EXPAND, K_RANK0,
  K_POSITIONS, K_FIRSTS, K_W_GATHER, K_TILE, K_TABLE, K_FENCE, K_HEADS, K_COUNT_BLOCKS, K_AP, K_SET_EDGES,
  K_EDGE_BLOCKS, K_EDGE_FINAL, K_MEMSET, K_EXPORT, K_WIDEN, K_GIANT_MIN, K_EDGE_FILL, K_EDGE_SEARCH, K_JUMP_LOCAL,
  K_JUMP_LIST, K_SCAN_TILES, K_W_SAMPLE, K_WITNESS_FIX, K_NLOW, K_NUM_KINDS
};

struct LaunchLog {
  static constexpr int kMax = 512;
  bool profile = false;
  bool capturing = false;  // inside a CUDA-graph capture: records become event nodes
  int count = 0;           // our kernels (memsets excluded)
  int nrec = 0;
  int kind[kMax];
  cudaEvent_t ev[kMax + 1];
  cudaStream_t st = nullptr;

  void record(int i) {
    cudaEventCreate(&ev[i]);
    if (capturing) cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal);
    else cudaEventRecord(ev[i], st);
  }
  void start() {
    if (profile) record(0);
  }
  void destroy() {
    if (profile)
      for (int i = 0; i <= nrec; i++) cudaEventDestroy(ev[i]);
    nrec = 0;
  }
};

extern thread_local LaunchLog* g_log;

// tunables (fbcc_set_option sets the process-wide defaults; each pipeline,
// plan and op snapshots them once when it is created and enqueues with its
// own copy, see OptScope)
enum Option : int {
  OPT_SAMPLE_ROUNDS = 0,  // Afforest neighbour-sampling rounds
  OPT_GIANT_SKIP = 1,     // skip rows already in the sampled giant component
  OPT_S0 = 3,             // level-0 splitter spacing (power of two)
  OPT_SL = 4,             // spacing on higher ranking levels (power of two)
  OPT_COMPRESS_MASK = 8,  // bitmask: sampling rounds followed by a compress (bit 0 always honoured)
  OPT_PDL = 11,           // programmatic dependent launch between consecutive kernels
  OPT_STREAM_CHUNKS = 12, // fbcc_run_host: arc ranges the edge copy is split into
  OPT_SKEL_PARENT = 13,   // Stage 5 sampling: bit r = round r samples the plain parent edge
  OPT_GIANT_FOLD = 14,    // the last sampling compress also picks the giant (no k_find_giant)
  OPT_EB_STAGED = 15,     // (retired: the warp-staged bitmap edge pass)
  OPT_MAX_ROUNDS = 16,    // adaptive sampling rounds beyond OPT_SAMPLE_ROUNDS, up to this many (see skip_round)
  OPT_SKEL_MAX_ROUNDS = 17,  // Stage 5's cap instead (0: OPT_MAX_ROUNDS)
  OPT_ACCEPT_FOLD = 18,   // a sampling round's accept runs inside the compress that follows it (2: auto by size)
  OPT_DETACH = 19,        // isolated vertices stay off the Euler-tour list and out of the tile pass
  OPT_WITNESS = 20,       // Stage 3 from each row's first three arcs + exact repair (0 off, 1 when m >= 8n, 2 always)
  // (keys 2, 5, 6, 7, 9, 10: retired experiments -- accepted, ignored)
  OPT_NUM = 21
};
struct Options {
  int v[OPT_NUM];
};
// the snapshot the current thread is enqueueing with (nullptr: the defaults)
extern thread_local const Options* t_opt;
Options options_snapshot();    // the current process-wide defaults (atomic reads)
int option_default(int key);
inline int opt(int key) { return t_opt ? t_opt->v[key] : option_default(key); }
struct OptScope {  // RAII: enqueue with the given snapshot on this thread
  const Options* prev;
  explicit OptScope(const Options* o) : prev(t_opt) { t_opt = o; }
  ~OptScope() { t_opt = prev; }
};

// ---------------------------------------------------------------------------
// launches: programmatic dependent launch (PDL).  Every kernel of ours starts
// with pdl_enter(): it waits until the preceding grid has completed and its
// writes are visible (griddepcontrol.wait -- a no-op for a normal launch),
// then allows the next grid to be scheduled.  The next kernel's CTAs are thus
// resident and waiting while this one drains, instead of paying the launch
// gap after it (~50 dependent kernels per run; CUDA-graph capture keeps the
// programmatic edges).  No kernel touches global memory before the wait, so
// write-after-read across kernels is ordered as with plain launches.
// ---------------------------------------------------------------------------
#ifndef FBCC_PDL_EARLY_TRIGGER
#define FBCC_PDL_EARLY_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if FBCC_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = opt(OPT_PDL) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline void note(KernelKind k) {
  LaunchLog* L = g_log;
  if (!L) return;
  if (k != K_MEMSET) L->count += (k == K_SCAN) ? 2 : 1;  // the upper-degree scan: tile-local prefixes, tile scan
  if (L->profile && L->nrec < LaunchLog::kMax) {
    L->record(L->nrec + 1);
    L->kind[L->nrec++] = k;
  }
}

// ---------------------------------------------------------------------------
// memory-order helpers
// ---------------------------------------------------------------------------
// Union-find parents are written concurrently by CAS; reads must not be
// served from a stale L1 line (relaxed, gpu scope -> L2).
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ int4 ld_nc4(const int4* p) { return __ldg(p); }

// streaming (read-once) 128-bit load that does not allocate in L1
__device__ __forceinline__ int4 ld_stream4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// One 8-arc chunk of the adjacency stream: a single 256-bit load (sm_100
// LDG.256, 32-byte aligned), not allocated in L1 and marked evict-first in
// L2 -- the 4m-byte stream then does not push out the arrays the arc passes
// gather from (first[], comp[], label[]), which would otherwise compete with
// it for the 126 MB L2.
__device__ __forceinline__ void ld_chunk8(const uint32_t* p, uint32_t* w) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

// ---------------------------------------------------------------------------
// hashing (splitter choice, sampling)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU;
  x ^= x >> 15; x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// ---------------------------------------------------------------------------
// launch geometry: grid-stride loops over a grid sized to the machine
// ---------------------------------------------------------------------------
inline int grid_for(int64_t items, int block, int max_waves = 16) {
  int64_t g = (items + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * max_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ---------------------------------------------------------------------------
// CSR row search: largest v in [lo, hi] with off[v] <= a (off[lo] <= a).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int row_of(const int64_t* __restrict__ off, int lo, int hi, int64_t a) {
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(off + mid) <= a) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Row after v that holds arc a (a >= off[v+1]): galloping from v+1, so the
// usual case (the next row) costs the one probe of off[v+2], and runs of
// empty rows (RMAT: half the vertices are isolated) cost O(log run) probes
// instead of a binary search over all n rows.
__device__ __forceinline__ int next_row(const int64_t* __restrict__ off, int v, int n, int64_t a) {
  int lo = v + 1;  // off[lo] <= a
  int step = 1;
  while (true) {
    const int probe = lo + step;
    if (probe > n - 1) return row_of(off, lo, n - 1, a);
    if (__ldg(off + probe) > a) return row_of(off, lo, probe - 1, a);
    lo = probe;
    step <<= 1;
  }
}

// ---------------------------------------------------------------------------
// Arc-balanced CSR traversal.  Every thread owns kItems consecutive arcs
// (one 32-byte sector of targets, loaded as two 128-bit vectors) and reads
// the row of its first arc from the per-run chunk->row table (crow, built by
// k_chunk_rows, every chunk).  The visitor sees
// rows in order:
//   begin(v, row_start, row_end)  arc(v, a, w)  end(v, whole)
// where ``whole`` says the row lies entirely inside this thread's chunk (no
// other thread touches it -- plain stores are safe; otherwise combine with
// atomics).  Hub rows with 600k arcs are spread over 75k threads.
// ---------------------------------------------------------------------------
constexpr int kItems = 8;

template <class Visitor>
__device__ __forceinline__ void visit_arc_chunks(const int64_t* __restrict__ off,
                                                 const uint32_t* __restrict__ adj,
                                                 const int* __restrict__ crow,
                                                 int n, int64_t m, Visitor& vis) {
  const int64_t nchunks = (m + kItems - 1) / kItems;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(adj) & 31) == 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nchunks; q += stride) {
    int64_t a0 = q * kItems;
    int64_t a1 = a0 + kItems < m ? a0 + kItems : m;
    uint32_t w[kItems];
    if (vec_ok && a1 - a0 == kItems) {
      ld_chunk8(adj + a0, w);
    } else {
#pragma unroll
      for (int i = 0; i < kItems; i++) w[i] = (a0 + i < a1) ? __ldg(adj + a0 + i) : 0u;
    }
    int v = __ldg(crow + q);
    if (v < 0) v = row_of(off, 0, n - 1, a0);  // chunk inside a hub row (see k_chunk_rows)
    // all of the chunk's neighbour gathers go out before any row bookkeeping
    // (in flight together: 8x the memory-level parallelism of gathering
    // behind each arc's data-dependent early exit)
    vis.prefetch(v, w, (int)(a1 - a0));
    int64_t rs = __ldg(off + v), re = __ldg(off + v + 1);
    vis.begin(v, rs, re);
#pragma unroll
    for (int i = 0; i < kItems; i++) {
      int64_t a = a0 + i;
      if (a < a1) {
        if (a >= re) {
          vis.end(v, rs >= a0);
          v = next_row(off, v, n, a);
          rs = __ldg(off + v);
          re = __ldg(off + v + 1);
          vis.begin(v, rs, re);
        }
        vis.arc(v, a, (int)w[i], i);
      }
    }
    vis.end(v, rs >= a0 && re <= a1);
  }
}

// chunk -> row table for visit_arc_chunks: crow[q] = row holding arc q*kItems,
// written by the row itself -- one lane for rows spanning at most kRowChunks
// chunks, the whole warp for longer (hub) rows.  One pass of n threads
// replaces a binary search per chunk in each arc-balanced kernel of a run
// (consumers keep a row_of fallback for a negative entry).
#ifndef FBCC_ROW_CHUNKS
#define FBCC_ROW_CHUNKS 64
#endif
constexpr int kRowChunks = FBCC_ROW_CHUNKS;

// rows of at least kHubDeg slots get several out-list heads in rooting (see
// k_root_flags): W = 2^lw ways, W = max(32, deg/64) rounded down to a power
// of two, at most 2^14 -- about 64 tree children per way on the RMAT hubs
// (deg 638k: 8192 ways), whose list inserts otherwise queue on 32 addresses.
// The marker lhead[v] = -2 - (base | (lw - 5) << 27) carries the sub-list
// base (off[v] >> 4; ways [base, base + W) stay inside the row's share
// deg/16 of the hsub array) and the way count.
constexpr int kHubDeg = 1024;
constexpr int kHubWays = 32;  // minimum ways of a hub
constexpr int kHubBaseBits = 27;
#ifndef FBCC_HUB_WAY_SHIFT
#define FBCC_HUB_WAY_SHIFT 7  // W ~ deg / 128 (deg/32, deg/64, deg/128 on config 5: 16.21, 16.00, 15.89 ms)
#endif

__device__ __forceinline__ int hub_log_ways(int64_t deg) {
  int64_t w = deg >> FBCC_HUB_WAY_SHIFT;
  int lw = 5;
  while (lw < 14 && ((int64_t)2 << lw) <= w) lw++;
  return lw;
}
__device__ __forceinline__ int hub_marker(int base, int lw) { return -2 - (base | ((lw - 5) << kHubBaseBits)); }
__device__ __forceinline__ int hub_base(int h) { return (-2 - h) & ((1 << kHubBaseBits) - 1); }
__device__ __forceinline__ int hub_ways(int h) { return 1 << (((-2 - h) >> kHubBaseBits) + 5); }

// Long rows deferred by a row-parallel pass (one lane or warp per row) to a
// second kernel, in two tiers so that neither tier costs every thread a pass
// over every listed row: rows up to kMegaRow arcs are owned by one CTA each
// (CTA b takes rows b, b + gridDim.x, ...), longer ones are strided over the
// whole grid.  Tier 1 fills list[0..) and tier 2 list[cap-1] downwards.
constexpr int kMegaRow = 1 << 16;
struct LongRows {
  int* list;
  int cap;
  int* nblock;  // tier-1 count
  int* ngrid;   // tier-2 count
  __device__ __forceinline__ void defer(int v, int64_t len) const {
    if (len > kMegaRow) list[cap - 1 - atomicAdd(ngrid, 1)] = v;
    else list[atomicAdd(nblock, 1)] = v;
  }
  // f(v) per row for the row words, then g(v, a) per arc, by the calling CTA
  // (tier 1) or the whole grid (tier 2)
  template <class Row, class Arc>
  __device__ __forceinline__ void visit(const int64_t* __restrict__ off, Row&& row, Arc&& arc) const {
    const int HB = *nblock, HG = *ngrid;
    for (int h = blockIdx.x; h < HB; h += gridDim.x) {
      const int v = list[h];
      const int64_t rs = __ldg(off + v), re = __ldg(off + v + 1);
      row(v, rs);
      for (int64_t a = rs + threadIdx.x; a < re; a += blockDim.x) arc(v, a);
    }
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int h = 0; h < HG; h++) {
      const int v = list[cap - 1 - h];
      const int64_t rs = __ldg(off + v), re = __ldg(off + v + 1);
      if (rs + tid >= re) continue;
      row(v, rs);
      for (int64_t a = rs + tid; a < re; a += stride) arc(v, a);
    }
  }
};

// Block-reduced counter add: every thread of the block must call it (after
// its grid-stride loop) with its private count; one atomic per block.
__device__ __forceinline__ void block_count_add(int* ctr, int mine) {
  __shared__ int warp_sums[32];
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) warp_sums[warp] = mine;
  __syncthreads();
  if (warp == 0) {
    int s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && s) atomicAdd(ctr, s);
  }
}

// warp-aggregated increment of a global counter
__device__ __forceinline__ void warp_count_add(int* ctr, bool pred) {
  unsigned b = __ballot_sync(__activemask(), pred);
  if (b && (threadIdx.x & 31) == (__ffs(b) - 1)) atomicAdd(ctr, __popc(b));
}

}  // namespace fbcc
