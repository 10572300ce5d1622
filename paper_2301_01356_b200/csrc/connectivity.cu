// connectivity.cu -- Stage 1 (spanning forest + components) and Stage 5
// (skeleton connectivity).
//
// Replaces the reference's clustered connectivity _cc_parts
// (connectivity.py:541-574: LDD ball growing _ldd_drive 195-246, sequential
// union batch _union_batch 287-309, label canonicalisation 312-341) and its
// skeleton-filtered second pass (bcc.py:185-189 with _slot_kept
// connectivity.py:57-81).
//
// B200 design: Afforest-style union-find hooking.  Parents live in one int32
// array (4 MB per 1M vertices -- L2-resident up to ~30M vertices).  A link
// CASes the larger root under the smaller, so every root is the minimum id
// of its set and final labels are canonical (== reference labels) without a
// min pass.  The CAS winner of Stage 1 records the edge that merged the two
// sets at fe[hooked root]: exactly n - c winners, an acyclic spanning forest
// (each win joins two distinct sets), one writer per slot.
//   1. two neighbour-sampling rounds (arc r of every row), each + compress
//   2. sample 1024 vertices, the most frequent root is the giant component
//   3. every remaining arc of every row not (yet) in the giant component --
//      arc-balanced (kItems arcs per thread), so RMAT hubs do not serialise
//   4. final compress -> comp[v] = min id of v's component
// Stage 5 is the same schedule templated on the skeleton predicate (the
// predicate is symmetric, so the giant-component skip stays exact) and with
// no forest recording.
#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

// Skeleton predicate (connectivity.py:57-81 / bcc.py classify_edge 54-70):
// rec = {first, last, parent, fence}.  Keep plain tree edges and cross edges.
__device__ __forceinline__ bool skel_keep(int u, const int4& ru, int w, const int4& rw) {
  if (rw.z == u) return rw.w == 0;  // tree edge, w is the child
  if (ru.z == w) return ru.w == 0;  // tree edge, u is the child
  if (ru.x <= rw.x && ru.y >= rw.y) return false;  // back edge (u ancestor of w)
  if (rw.x <= ru.x && rw.y >= ru.y) return false;  // back edge (w ancestor of u)
  return true;                                      // cross edge
}

// Afforest link with forest recording.  p1/p2 are always ancestors of the
// two endpoints; a successful CAS hooks root `hi` under `lo`, which lies in
// the other endpoint's set (roots are set minima, lo < hi), so (u, w) is a
// spanning-forest edge joining two distinct sets.
template <bool kRecord>
__device__ __forceinline__ void link(int u, int w, int* comp, int2* fe) {
  int p1 = ld_relaxed(comp + u);
  int p2 = ld_relaxed(comp + w);
  while (p1 != p2) {
    int hi = p1 > p2 ? p1 : p2;
    int lo = p1 + p2 - hi;
    int phi = ld_relaxed(comp + hi);
    if (phi == lo) break;  // already hooked together
    if (phi == hi) {
      int prev = atomicCAS(comp + hi, hi, lo);
      if (prev == hi) {
        if (kRecord) fe[hi] = make_int2(u, w);
        break;
      }
    }
    p1 = ld_relaxed(comp + ld_relaxed(comp + hi));
    p2 = ld_relaxed(comp + lo);
  }
}

__global__ void k_iota(int* __restrict__ comp, int n) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) comp[v] = v;
}

template <bool kSkel, bool kRecord>
__global__ void k_sample_link(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n,
                              int round, int* comp, int2* fe, const int4* __restrict__ rec) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int64_t s = __ldg(off + v) + round;
    if (s >= __ldg(off + v + 1)) continue;
    int w = (int)__ldg(adj + s);
    if (kSkel) {
      if (!skel_keep(v, __ldg(rec + v), w, __ldg(rec + w))) continue;
    }
    link<kRecord>(v, w, comp, fe);
  }
}

// pointer jumping to the root (the root is the component minimum)
__global__ void k_compress(int* comp, int n) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int c = comp[v];
    int cc = comp[c];
    if (c == cc) continue;
    while (c != cc) { c = cc; cc = comp[c]; }
    comp[v] = c;
  }
}

// Most frequent root among 1024 sampled vertices (one block of 1024).
__global__ void k_find_giant(const int* __restrict__ comp, int n, Scalars* sc) {
  __shared__ int val[1024];
  __shared__ int bestc[32], bestv[32];
  int t = threadIdx.x;
  int v = (int)(hash32(0x9E3779B9u * (uint32_t)(t + 1)) % (uint32_t)n);
  int mine = comp[v];
  val[t] = mine;
  __syncthreads();
  int cnt = 0;
  for (int i = 0; i < 1024; i++) cnt += (val[i] == mine);
  // argmax (ties -> smaller root id, deterministic)
  for (int o = 16; o > 0; o >>= 1) {
    int oc = __shfl_down_sync(0xffffffffu, cnt, o);
    int ov = __shfl_down_sync(0xffffffffu, mine, o);
    if (oc > cnt || (oc == cnt && ov < mine)) { cnt = oc; mine = ov; }
  }
  if ((t & 31) == 0) { bestc[t >> 5] = cnt; bestv[t >> 5] = mine; }
  __syncthreads();
  if (t < 32) {
    cnt = bestc[t]; mine = bestv[t];
    for (int o = 16; o > 0; o >>= 1) {
      int oc = __shfl_down_sync(0xffffffffu, cnt, o);
      int ov = __shfl_down_sync(0xffffffffu, mine, o);
      if (oc > cnt || (oc == cnt && ov < mine)) { cnt = oc; mine = ov; }
    }
    if (t == 0) sc->giant = mine;
  }
}

template <bool kSkel, bool kRecord>
struct LinkRestVisitor {
  int* comp;
  int2* fe;
  const int4* rec;
  int giant;
  int rounds;
  int64_t rs;
  bool skip;
  int4 rv;
  __device__ __forceinline__ void begin(int v, int64_t s, int64_t e) {
    rs = s;
    skip = ld_relaxed(comp + v) == giant;
    if (kSkel && !skip) rv = __ldg(rec + v);
  }
  __device__ __forceinline__ void arc(int v, int64_t a, int w) {
    if (skip || a - rs < rounds) return;
    if (kSkel) {
      if (!skel_keep(v, rv, w, __ldg(rec + w))) return;
    }
    link<kRecord>(v, w, comp, fe);
  }
  __device__ __forceinline__ void end(int, bool) {}
};

template <bool kSkel, bool kRecord>
__global__ void __launch_bounds__(256) k_link_rest(const int64_t* __restrict__ off,
                                                   const uint32_t* __restrict__ adj, int n, int64_t m,
                                                   int rounds, int* comp, int2* fe,
                                                   const int4* __restrict__ rec, const Scalars* sc) {
  LinkRestVisitor<kSkel, kRecord> vis;
  vis.comp = comp;
  vis.fe = fe;
  vis.rec = rec;
  vis.giant = sc->giant;
  vis.rounds = rounds;
  visit_arc_chunks(off, adj, n, m, vis);
}

// Afforest schedule shared by Stage 1 (kSkel=false, record forest) and
// Stage 5 (kSkel=true, no forest).
template <bool kSkel, bool kRecord>
static void run_cc(const Graph& g, int* comp, int2* fe, const int4* rec, Scalars* sc, cudaStream_t st) {
  const int B = 256;
  const int kRounds = 2;
  int gv = grid_for(g.n, B);
  k_iota<<<gv, B, 0, st>>>(comp, g.n);
  note(K_IOTA);
  for (int r = 0; r < kRounds; r++) {
    k_sample_link<kSkel, kRecord><<<gv, B, 0, st>>>(g.off, g.adj, g.n, r, comp, fe, rec);
    note(K_SAMPLE_LINK);
    k_compress<<<gv, B, 0, st>>>(comp, g.n);
    note(K_COMPRESS);
  }
  k_find_giant<<<1, 1024, 0, st>>>(comp, g.n, sc);
  note(K_FIND_GIANT);
  int64_t nchunks = (g.m + kItems - 1) / kItems;
  if (nchunks > 0) {
    int ga = grid_for(nchunks, B, 32);
    k_link_rest<kSkel, kRecord><<<ga, B, 0, st>>>(g.off, g.adj, g.n, g.m, kRounds, comp, fe, rec, sc);
    note(K_LINK_REST);
  }
  k_compress<<<gv, B, 0, st>>>(comp, g.n);
  note(K_COMPRESS);
}

void stage1_forest(const Graph& g, int* comp, int2* fe, Scalars* sc, cudaStream_t st) {
  run_cc<false, true>(g, comp, fe, nullptr, sc, st);
}

void stage5_skeleton_cc(const Graph& g, const int4* rec, int* label, Scalars* sc, cudaStream_t st) {
  run_cc<true, false>(g, label, nullptr, rec, sc, st);
}

}  // namespace fbcc
