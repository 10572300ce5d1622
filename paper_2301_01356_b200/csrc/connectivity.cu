// connectivity.cu -- Stage 1 (spanning forest + components), Stage 5
// (skeleton connectivity) and the stand-alone masked connectivity op.
//
// Replaces the reference's clustered connectivity _cc_parts
// (connectivity.py:541-574: LDD ball growing _ldd_drive 195-246, sequential
// union batch _union_batch 287-309, label canonicalisation 312-341), its
// skeleton-filtered second pass (bcc.py:185-189 with _slot_kept
// connectivity.py:57-81) and connected_components(g, keep_edge)
// (connectivity.py:593-611).
//
// B200 design: union-find with the root of every set equal to its minimum
// id, so final labels are canonical (== reference labels) with no min pass.
// Parents live in one int32 array (4 MB per 1M vertices).
//   1. sampling rounds over arc r of every row (default: rounds 0 and 1, and
//      round 2 unless round 1 hooked < n/8192 roots), each a
//      PROPOSE/ACCEPT step: every vertex fires one fire-and-forget 64-bit
//      atomicMin((lower root << 32) | proposer) at the higher of the two
//      component roots; k_accept hooks each proposed-to root under its
//      minimum proposal and records the forest edge.  Hooks always point to
//      a smaller round-start root (a forest over the components, no cycles),
//      and same-address REDs pipeline in the L2 atomic unit instead of
//      serialising CAS retry loops on a few hot roots (the failure mode of
//      Afforest's CAS link on a GPU: round 1 merges ~n/17 roots into one).
//      Proposers are thinned to ~32 per surviving root.
//   2. compress after round 0 and after the last round (pointer doubling on
//      a fully resident grid); rounds in between find() through shallow trees
//   3. sample 1024 vertices: the most frequent root is the giant component
//   4. every arc of every row outside the giant (Afforest's skip; exact for a
//      symmetric predicate): union-find with L1-cached finds, path halving
//      and CAS hooking, one warp per 32 rows, long rows warp-cooperative
//   5. final compress -> comp[v] = min id of v's component
// In Stage 1 each successful hook records the arc that merged the two sets
// at fe[hooked root]: exactly n - c records, an acyclic spanning forest.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

// ---------------------------------------------------------------------------
// edge predicates
// ---------------------------------------------------------------------------
enum : int { PRED_NONE = 0, PRED_SKEL = 1, PRED_MASK = 2 };

struct PredData {
  const int4* rec;        // PRED_SKEL: {first, last, parent, fence}
  const int* w0;          // PRED_SKEL (optional): each row's first arc target, recorded by Stage 1's k_chunk_rows
  const int* warc;        // (optional) [3][n]: targets of arcs 0, 1, 2 of each row (-1: none) for the sampling
                          // rounds, recorded by k_chunk_rows; nullptr: read the adjacency
  const uint8_t* mask;    // PRED_MASK: per-slot keep byte
  const int64_t* off;     // PRED_MASK: to find the canonical (u < w) slot
  const uint32_t* adj;
};

// Skeleton predicate (connectivity.py:57-81 / bcc.py classify_edge 54-70):
// keep plain tree edges and cross edges.
__device__ __forceinline__ bool skel_keep(int u, const int4& ru, int w, const int4& rw) {
  if (rw.z == u) return rw.w == 0;  // tree edge, w is the child
  if (ru.z == w) return ru.w == 0;  // tree edge, u is the child
  if (ru.x <= rw.x && ru.y >= rw.y) return false;  // back edge (u ancestor of w)
  if (rw.x <= ru.x && rw.y >= ru.y) return false;  // back edge (w ancestor of u)
  return true;                                      // cross edge
}

// The reference reads a keep mask at the u < w slot of each undirected edge
// only (_scan_crossing connectivity.py:279); the reverse arc finds that slot
// by binary search in the (sorted) row of its smaller endpoint.
__device__ __forceinline__ bool mask_keep(const PredData& pd, int v, int w, int64_t a) {
  if (v < w) return pd.mask[a] != 0;
  int64_t lo = __ldg(pd.off + w), hi = __ldg(pd.off + w + 1);
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int)__ldg(pd.adj + mid) < v) lo = mid + 1; else hi = mid;
  }
  return pd.mask[lo] != 0;
}

template <int kPred>
__device__ __forceinline__ bool keep(const PredData& pd, int v, const int4& rv, int w, int64_t a) {
  if (kPred == PRED_SKEL) return skel_keep(v, rv, w, __ldg(pd.rec + w));
  if (kPred == PRED_MASK) return mask_keep(pd, v, w, a);
  return true;
}

// ---------------------------------------------------------------------------
// union-find primitives
// ---------------------------------------------------------------------------
// Root of x with path halving.  Only non-roots are rewritten, always to an
// ancestor (ancestors stay ancestors: sets only merge), and roots change only
// through the hooking CAS -- so the concurrent rewrites are benign.
//
// Parent reads are L1-cacheable (ld.global.ca).  Every value comp[x] ever
// held is an ancestor of x, so a stale line can only (a) make two endpoints
// look joined when they truly are, or (b) offer a "root" that is no longer
// one -- the CAS then fails and returns the fresh parent, so every retry
// climbs.  What the L1 buys: once most vertices share one giant root, every
// find ends at the same word; served from L2 (ld.relaxed.gpu) those ~1M
// requests serialise on a single L2 slice.
__device__ __forceinline__ int ldp(const int* p) { return __ldca(p); }

__device__ __forceinline__ int find_halve(int* comp, int x) {
  int p = ldp(comp + x);
  while (p != x) {
    int gp = ldp(comp + p);
    if (gp == p) return p;
    // non-returning atomicMin (RED) rather than a store: ancestors have
    // smaller ids, so a shortcut another thread made (or a fresher value
    // than our possibly stale L1 copy) is never undone (config 3: -13%)
    atomicMin(comp + x, gp);
    x = gp;
    p = ldp(comp + x);
  }
  return x;
}

// Hook the larger root under the smaller.  A successful CAS hooks root `hi`
// under `lo`, whose set holds the other endpoint (root(lo) <= lo < hi), so
// (u, w) is a spanning-forest edge joining two distinct sets.
// Returns the root the two sets were joined under (an ancestor of u, for the
// caller's next comparison).
template <bool kRecord>
__device__ __forceinline__ int link(int u, int w, int* comp, int2* fe) {
  int ru = find_halve(comp, u);
  int rw = find_halve(comp, w);
  while (ru != rw) {
    int hi = ru > rw ? ru : rw;
    int lo = ru + rw - hi;
    int prev = atomicCAS(comp + hi, hi, lo);
    if (prev == hi) {
      if (kRecord) fe[hi] = make_int2(u, w);
      return lo;
    }
    ru = find_halve(comp, prev);  // hi was hooked meanwhile: climb on
    rw = find_halve(comp, lo);
  }
  return ru;
}

// ---------------------------------------------------------------------------
// chunk -> row table (see visit_arc_chunks): row v owns the chunks whose
// first arc lies in it
// ---------------------------------------------------------------------------
// Sampling round 0's hook target for v (rows sorted, every vertex its own
// root): a smaller neighbour, so comp[v] = w < v keeps parents below children.
// Prefer the LARGEST smaller neighbour when it lies within kNear ids and the
// row is short enough to scan in its first sector (deg <= 8); otherwise the
// minimum neighbour (the minimum proposal v would receive, Borůvka-style).
// On meshes with id locality (tori, grids: configs 1, 4a, 4b) the near rule
// hooks each vertex to its left neighbour, so the spanning forest -- and the
// Euler tour built from it -- follows the id order: the tour positions of
// consecutive vertices are consecutive, and Stage 2/3's position-indexed
// scatters (k_positions, the w gather's AP stores, the tile pass's partials)
// become coalesced instead of random.  Random-id graphs (configs 2, 3, 5)
// almost never have a smaller neighbour within kNear ids and keep the minimum.
// (kNear: common.cuh)

__device__ __forceinline__ int round0_target(const uint32_t* __restrict__ adj, int v, int64_t rs, int64_t re,
                                             int* first_arc = nullptr) {
  const int w0 = (int)__ldg(adj + rs);
  if (first_arc) *first_arc = w0;
  if (w0 >= v) return v;  // no smaller neighbour
  if (re - rs <= kItems) {
    int best = w0;
    for (int64_t a = rs + 1; a < re; a++) {
      const int w = (int)__ldg(adj + a);
      if (w >= v) break;
      best = w;
    }
    if (v - best <= kNear) return best;
  }
  return w0;
}

// Every chunk q (first arc 8q) belongs to exactly one non-empty row, which
// writes it -- no memset.  Rows of up to kRowChunks chunks are written by
// their own lane; longer (hub) rows by the whole warp, so a 600k-arc RMAT hub
// costs 2.3k warp stores instead of one thread's 75k (consumers used to
// binary-search hub chunks over all n rows: half of RMAT's gather passes).
//
// The pipeline's Stage 1 also folds its sampling round 0 (k_hook_min<NONE>:
// comp[v] = round0_target, the forest edge, the proposal reset)
// into this pass over the offsets (comp != nullptr).
__global__ void k_chunk_rows(const int64_t* __restrict__ off, int n, int* __restrict__ crow, Scalars* sc,
                             const uint32_t* __restrict__ adj, int* __restrict__ comp, int2* __restrict__ fe,
                             unsigned long long* __restrict__ prop, int* __restrict__ nlow, int* __restrict__ w0) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int near = 0;  // round-0 hooks within kNear ids (see k_jump_local)
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += warps * 32) {
    const int v = (int)base + lane;
    int q0 = 0, q1 = 0;
    if (v < n) {
      const int64_t rs = __ldg(off + v), re = __ldg(off + v + 1);
      if (nlow) nlow[v] = 0;  // Stage 3 accumulates rows split across warps into it
      q0 = (int)((rs + kItems - 1) / kItems);
      q1 = (int)((re + kItems - 1) / kItems);
      if (comp) {  // sampling round 0 (see k_hook_min)
        int c = v;
        if (rs < re) {
          int first = v;
          c = round0_target(adj, v, rs, re, &first);
          if (c < v) fe[v] = make_int2(v, c);
          near += c < v && v - c <= kNear;
          w0[v] = first;  // Stage 5's round-0 arc (coalesced; saves it a cold sector per row)
        }
        // arcs 1 and 2 for the sampling rounds of Stages 1 and 5 (same
        // sector as arc 0: the proposers then read 4 coalesced bytes instead
        // of an offsets pair and a cold 32-byte adjacency sector per row)
        w0[(int64_t)n + v] = re - rs > 1 ? (int)__ldg(adj + rs + 1) : -1;
        w0[2 * (int64_t)n + v] = re - rs > 2 ? (int)__ldg(adj + rs + 2) : -1;
        comp[v] = c;
        prop[v] = ~0ull;
      }
    }
    const bool hub = q1 - q0 > kRowChunks;
    if (hub && (int64_t)(q1 - q0) * kItems >= kHubDeg) sc->has_hubs = 1;
    if (!crow) continue;  // (a witness plan: no arc-balanced pass reads the table unless its repair overflows)
    if (!hub)
      for (int q = q0; q < q1; q++) crow[q] = v;
    unsigned hb = __ballot_sync(0xffffffffu, hub);
    while (hb) {
      const int src = __ffs(hb) - 1;
      hb &= hb - 1;
      const int hv = __shfl_sync(0xffffffffu, v, src);
      const int h0 = __shfl_sync(0xffffffffu, q0, src), h1 = __shfl_sync(0xffffffffu, q1, src);
      for (int q = h0 + lane; q < h1; q += 32) crow[q] = hv;
    }
  }
  if (comp) block_count_add(&sc->near[0], near);
}

// w0[k][v] = target of arc k of row v (k = 0..2; -1: the row is shorter) -- what k_chunk_rows' round 0
// records, for the host path, whose edges arrive after that kernel ran
__global__ void k_record_arcs(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n,
                              int* __restrict__ w0) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int64_t rs = __ldg(off + v), deg = __ldg(off + v + 1) - rs;
#pragma unroll
    for (int k = 0; k < 3; k++) w0[(int64_t)k * n + v] = deg > k ? (int)__ldg(adj + rs + k) : -1;
  }
}

void record_arcs(const Graph& g, int* w0, cudaStream_t st) {
  if (g.m == 0) return;
  launch(k_record_arcs, grid_for(g.n, 256), 256, 0, st, g.off, g.adj, g.n, w0);
  note(K_CHUNK_ROWS);
}

bool build_chunk_rows(const Graph& g, int* crow, Scalars* sc, cudaStream_t st, int* comp, int2* fe,
                      unsigned long long* prop, int* nlow, int* w0) {
  if (g.m == 0) {
    if (nlow) cudaMemsetAsync(nlow, 0, sizeof(int) * g.n, st);
    return false;
  }
  const bool fold = comp != nullptr && opt(OPT_SAMPLE_ROUNDS) > 0;
  launch(k_chunk_rows, grid_for(g.n, 256), 256, 0, st, g.off, g.n, crow, sc, g.adj, fold ? comp : nullptr, fe, prop,
         nlow, w0);
  note(K_CHUNK_ROWS);
  return fold;
}

// Sampling round 0 without atomics.  With every vertex its own root, v can
// hook under any smaller neighbour (round0_target: the minimum one -- the
// minimum proposal v would receive -- or a near one on meshes) with the
// forest edge (v, w).  Under a predicate only v's own arc 0 is used (best
// effort: k_link_rows re-covers).  Also resets the proposal words for the
// later rounds.
template <int kPred, bool kRecord>
__global__ void k_hook_min(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int* comp,
                           int2* fe, unsigned long long* __restrict__ prop, PredData pd, bool skel_parent,
                           bool parent_only, const Scalars* skip_if_ordered) {
  pdl_enter();
  if (skip_if_ordered && id_ordered(skip_if_ordered, n)) return;  // (Stage 4's k_fence did this round)
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int64_t s = __ldg(off + v);
    int c = v;
    const int64_t e = __ldg(off + v + 1);
    if (kPred == PRED_SKEL && parent_only) {  // round 0 along plain parent edges only (no arc read)
      const int4 rv = __ldg(pd.rec + v);
      if (rv.z >= 0 && rv.w == 0 && rv.z < c) c = rv.z;
    } else if (s < e) {
      // (Stage 5: the first arc's target as Stage 1's k_chunk_rows recorded it --
      // a coalesced 4-byte read instead of one cold adjacency sector per row)
      int w = kPred == PRED_NONE ? round0_target(adj, v, s, e)
                                 : (kPred == PRED_SKEL && pd.w0) ? __ldg(pd.w0 + v) : (int)__ldg(adj + s);
      int4 rv;
      if (kPred == PRED_SKEL) rv = __ldg(pd.rec + v);
      if (w < v && keep<kPred>(pd, v, rv, w, s)) {
        c = w;
        if (kRecord) fe[v] = make_int2(v, w);
      }
      // skeleton: the plain tree edge to the parent is always kept
      if (kPred == PRED_SKEL && skel_parent) {
        if (rv.z >= 0 && rv.w == 0 && rv.z < c) c = rv.z;
      }
    }
    comp[v] = c;
    if (prop) prop[v] = ~0ull;
  }
}

// comp = identity; also resets the proposal words (one pass, no memset node)
__global__ void k_iota(int* __restrict__ comp, int n, unsigned long long* __restrict__ prop) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    comp[v] = v;
    if (prop) prop[v] = ~0ull;
  }
}

// ---------------------------------------------------------------------------
// sampling rounds
// ---------------------------------------------------------------------------
#ifndef FBCC_PER_ROOT
#define FBCC_PER_ROOT 32
#endif
constexpr int kPerRoot = FBCC_PER_ROOT;

// Rounds at or past rbase are adaptive: they run only while the previous
// round still hooked >= 5% as many roots as the one before it and >= n/8192
// (high-diameter graphs -- config 3: 114k, 28k, 3.4k, 0.6k hooks in rounds
// 1-4 -- keep merging, which leaves k_link_rows far fewer components; a
// low-diameter graph's round 2 hooks < 1% of round 1's and the extra rounds
// exit at once).
// (round 2 has only the absolute test: on the tori and the chain round 0
// already hooks all but a handful of vertices, round 1 hooks < n/8192 and
// round 2 is skipped -- 4a -0.47 ms; config 2's round 1 hooks 65k, RMAT's
// 466k.  A ratio against round 0's roots would count RMAT's 16.5 M isolated
// vertices and starve its giant.)
// (hub_sc, Stage 1 only: on a graph with hub rows -- RMAT -- a row's third arc
// is one more hub already in the giant: round 2 hooked 8.7 k of config 5's
// 0.97 M remaining roots for 0.21 ms, while the hub-free uniform graph needs
// it -- config 2 +40 % without.  Stage 5 keeps its rounds: its giant only forms there.)
__device__ __forceinline__ bool skip_round(const int* hooks, int round, int rbase, int n,
                                           const Scalars* hub_sc = nullptr) {
  if (round < rbase || round < 2) return false;
  if (hub_sc && hub_sc->has_hubs) return true;
  const int h1 = hooks[round - 1];
  if ((int64_t)h1 * 8192 < (int64_t)n) return true;
  return round > 2 && (int64_t)h1 * 20 < (int64_t)hooks[round - 2];
}

// Sets left at the start of sampling round `round` (>= 1): the roots counted
// by round 0's compress minus the later hooks.  One set left (a connected
// graph that round 0 already joined: the tori, the chain) means no arc can
// join anything any more -- the remaining rounds and the link pass return at
// once (4a / 4c: propose + folded compress + link_rows, 0.54 ms of Stage 1).
__device__ __forceinline__ int64_t sets_left(const int* nroots, const int* hooks, int round) {
  int64_t R = nroots[0];
  for (int i = 1; i < round; i++) R -= hooks[i];
  return R;
}

template <int kPred>
__global__ void k_propose(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int round,
                          int* comp, unsigned long long* prop, PredData pd, const int* __restrict__ nroots,
                          const int* __restrict__ hooks, bool flat, bool skel_parent, int rbase,
                          const Scalars* hub_sc) {
  pdl_enter();
  if (skip_round(hooks, round, rbase, n, hub_sc)) return;
  // participate iff hash < thr / 2^24, thr = min(1, kPerRoot * roots / n);
  // roots at round start = roots counted after round 0 minus later hooks
  uint32_t thr = 1u << 24;
  if (round > 0) {
    const int64_t R = sets_left(nroots, hooks, round);
    if (R <= 1) return;
    uint64_t t = ((uint64_t)kPerRoot * (uint64_t)(R > 0 ? R : 0) << 24) / (uint64_t)n;
    if (t < thr) thr = (uint32_t)t;
  }
  const int* wr = (kPred != PRED_MASK && pd.warc && round <= 2) ? pd.warc + (int64_t)round * n : nullptr;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (thr < (1u << 24) && (hash32((uint32_t)v * 0x9E3779B1u + (uint32_t)round) >> 8) >= thr) continue;
    int w;
    int64_t s = -1;
    int4 rv;
    if (kPred == PRED_SKEL && skel_parent) {  // this round samples the plain parent edge
      rv = __ldg(pd.rec + v);
      if (rv.z < 0 || rv.w != 0) continue;
      w = rv.z;
    } else {
      if (wr) {
        w = __ldg(wr + v);
        if (w < 0) continue;
      } else {
        s = __ldg(off + v) + round;
        if (s >= __ldg(off + v + 1)) continue;
        w = (int)__ldg(adj + s);
      }
    }
    // flat after a compress; otherwise (rounds >= 1 hook root -> root only,
    // so trees stay shallow) find with halving
    int ru = flat ? ldp(comp + v) : find_halve(comp, v);
    int rw = flat ? ldp(comp + w) : find_halve(comp, w);
    if (ru == rw) continue;
    // the predicate only for arcs that would join two sets: under the
    // skeleton predicate it gathers w's 16-byte record, and by the last
    // rounds most sampled arcs already lie inside one set
    // (v's own record is loaded here too: rows with no sampled arc -- RMAT's
    // isolated half -- and arcs inside one set never read it)
    if (!(kPred == PRED_SKEL && skel_parent)) {
      if (kPred == PRED_SKEL) rv = __ldg(pd.rec + v);
      if (!keep<kPred>(pd, v, rv, w, s)) continue;
    }
    int hi = ru > rw ? ru : rw;
    int lo = ru + rw - hi;
    // any proposal is a valid hook, so lanes aiming at the same root send one
    unsigned peers = __match_any_sync(__activemask(), hi);
    if ((threadIdx.x & 31) != __ffs(peers) - 1) continue;
    // low word = the proposer: its arc is off[v] + round, no search on accept
    atomicMin(prop + hi, ((unsigned long long)(unsigned)lo << 32) | (unsigned long long)(uint32_t)v);
  }
}

// (the proposer u's sampled arc: warc[round][u] when recorded, else adj[off[u] + round])
__device__ __forceinline__ int sampled_arc(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                           const int* __restrict__ warc, int n, int round, int u) {
  return (warc && round <= 2) ? __ldg(warc + (int64_t)round * n + u) : (int)__ldg(adj + __ldg(off + u) + round);
}

template <bool kRecord>
__global__ void k_accept(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int round, int* comp,
                         unsigned long long* prop, int2* fe, int* hooks, int rbase, const int* __restrict__ warc,
                         const int* __restrict__ nroots, const Scalars* hub_sc) {
  pdl_enter();
  if (skip_round(hooks, round, rbase, n, hub_sc) || sets_left(nroots, hooks, round) <= 1) return;
  int hooked = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    unsigned long long key = prop[v];
    if (key == ~0ull) continue;
    prop[v] = ~0ull;  // ready for the next round
    if (__ldcg(comp + v) != v) continue;  // proposed to on a two-level view (see k_compress<kAccept>)
    int lo = (int)(key >> 32);
    comp[v] = lo;
    hooked++;
    if (kRecord) {
      int u = (int)(key & 0xffffffffull);
      fe[v] = make_int2(u, sampled_arc(off, adj, warc, n, round, u));
    }
  }
  block_count_add(hooks + round, hooked);
}

// Pointer jumping to the root (the component minimum), optionally counting
// the roots.  Every step stores the advanced pointer and reads the parent's
// CURRENT pointer from L2, so concurrent threads ride each other's progress:
// pointer doubling, ~log2(depth) steps per thread (storing only at the end is
// O(depth) per thread -- O(n^2) on a 10^8-vertex path whose round-0 hooks form
// one chain).  No hooks happen during a compress, so a root's entry is stable
// and the "is c a root" test may use an L1-cached load (the giant root's word
// is then served per SM instead of hammering one L2 slice).  The grid must
// be fully resident (see run_cc).
//
// Shallow chains (the common case) are climbed with L1-cached loads only: L1
// is invalidated at every launch boundary and during a compress non-roots
// only move up, so a cached value is always an ancestor and the "c is a root"
// test is exact -- and the few words every thread ends on (the giant's top
// roots) are served per SM instead of by one L2 slice.  After kL1Steps
// without reaching a root the thread switches to L2 reads with stores
// (doubling), for the deep chains of path-like graphs.
constexpr int kL1Steps = 8;

__device__ void giant_of_block(const int* comp, int n, Scalars* sc, bool enable);

// giant_sc != nullptr: the last block to finish also picks the sampled giant
// root (Afforest skip) -- one launch instead of a separate 1-block kernel.
// (hooks != nullptr: the compress after adaptive sampling round `round`; it
// does no pointer work when that round was skipped -- comp is still flat
// from the previous round's compress -- but still picks the giant)
// kAccept: the compress after propose round `round` first applies that
// round's proposals (k_accept folded in: one pass over the vertices fewer per
// round).  A vertex hooked here may already have been taken for a root by a
// thread that climbed through it, so the array can come out two levels deep:
// the next round's proposals then verify their target is still a root
// (accept below), k_link_rows' giant test looks two levels up and falls back
// to linking, and the final compress (no kAccept) makes the labels flat.
// ---------------------------------------------------------------------------
// Root ranks inside the final compress (kScan): the exclusive scan of the
// root codes (Rooting::rootidx: roots on the tour list before v in the low
// word, detached roots in the high word) in two levels.  The compress writes
// each root's rank inside its 1024-vertex tile and the tile's root counts;
// k_scan_tiles (rooting.cu, one CTA) turns the tile counts into prefixes and
// k_out_lists adds them in as it places the roots.  No waiting between
// blocks: a single-pass scan with decoupled look-back inside this kernel,
// whose blocks run in lockstep waves, spent ~17 us per wave walking back
// through the wave's aggregates (4a: final compress 0.23 -> 2.03 ms).
// ---------------------------------------------------------------------------
// Each thread owns kCPer vertices per step (base + i * blockDim + t: coalesced),
// so kCPer loads, then kCPer independent climbs, are in flight together -- at
// one vertex per thread the kernel waited on its single load, then on its
// single gather (config 5: 62 % of the stall samples on those two lines).
#ifndef FBCC_CPER
#define FBCC_CPER 4
#endif
constexpr int kCPer = FBCC_CPER;
// resident blocks per SM the register budget is set for; the grid is exactly
// that many (k_compress wants every block resident: a thread climbing through
// the range of a block not yet scheduled walks its raw chains)
#ifndef FBCC_CBLOCKS
#define FBCC_CBLOCKS 8  // (4 vertices per thread fit 32 registers; 4 blocks at 64 registers measured slower)
#endif
constexpr int kCBlocks = FBCC_CBLOCKS;

static_assert(kCPer == 4, "the fused root scan assumes 256 x 4-vertex tiles (api.cu sizes its descriptors for them)");
#ifndef FBCC_CBLOCKS_SCAN
#define FBCC_CBLOCKS_SCAN 6
#endif
constexpr int kCBlocksScan = FBCC_CBLOCKS_SCAN;  // (the scan variants: 40 registers instead of spilling at 32)
template <bool kJump, bool kAccept = false, bool kRecord = false, bool kScan = false>
__global__ void __launch_bounds__(256, kScan ? kCBlocksScan : kCBlocks) k_compress(int* comp, int n, int* nroots, Scalars* giant_sc, bool giant_enable,
                                                  RootInit ri, const int* hooks, int round, int rbase,
                                                  unsigned long long* prop = nullptr, int* hooks_out = nullptr,
                                                  int2* fe = nullptr, const int64_t* __restrict__ off = nullptr,
                                                  const uint32_t* __restrict__ adj = nullptr,
                                                  const int* __restrict__ warc = nullptr,
                                                  const int* __restrict__ roots0 = nullptr,
                                                  const int* __restrict__ hooks0 = nullptr,
                                                  const Scalars* hub_sc = nullptr) {
  pdl_enter();
  int roots = 0;
  int hooked = 0;
  // (roots0: the compress after sampling round `round` >= 1 -- nothing was
  // proposed when a single set was left, see sets_left)
  const int n_work = ((hooks && skip_round(hooks, round, rbase, n, hub_sc)) ||
                      (roots0 && sets_left(roots0, hooks0, round) <= 1)) ? 0 : n;
  const int64_t* hoff = (ri.flags && ri.off && ri.sc->has_hubs) ? ri.off : nullptr;
  if (ri.flags && blockIdx.x == 0 && threadIdx.x == 0) ri.flags[n] = 0;
  __shared__ int sp[kJump ? 256 * kCPer : 1];
  const int t = threadIdx.x;
  const int tile = (int)blockDim.x * kCPer;
  // block-uniform trip count (kJump): each step the block owns `tile`
  // consecutive vertices and may first shorten their chains in shared memory
  __shared__ unsigned s_wc[kScan ? 64 : 1];  // per (i, warp) root counts: detached << 16 | listed (two tiles' worth)
  int wbuf = 0;
  for (int64_t base = (int64_t)blockIdx.x * tile; base < n_work; base += (int64_t)gridDim.x * tile) {
    int v[kCPer], c[kCPer], mem[kCPer];
    bool root[kCPer];
#pragma unroll
    for (int i = 0; i < kCPer; i++) {
      v[i] = (int)base + i * (int)blockDim.x + t;
      c[i] = v[i] < n ? __ldcg(comp + v[i]) : v[i];
    }
    if (kAccept) {
      unsigned long long key[kCPer];
#pragma unroll
      for (int i = 0; i < kCPer; i++) key[i] = v[i] < n ? prop[v[i]] : ~0ull;
#pragma unroll
      for (int i = 0; i < kCPer; i++) {
        if (key[i] == ~0ull) continue;
        prop[v[i]] = ~0ull;  // ready for the next round
        if (c[i] == v[i]) {  // still a root (a stale proposal is dropped)
          c[i] = (int)(key[i] >> 32);
          comp[v[i]] = c[i];
          hooked++;
          if (kRecord) {
            const int u = (int)(key[i] & 0xffffffffull);
            fe[v[i]] = make_int2(u, sampled_arc(off, adj, warc, n, round, u));
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kCPer; i++) {
      root[i] = c[i] == v[i];
      mem[i] = c[i];  // what comp[v] holds now
    }
    if (kJump) {
      // Pointer jumping inside the block's id range (after sampling round 0
      // only): chains of consecutive ids -- round 0's left-neighbour hooks on
      // meshes, a path's v -> v-1 -- then leave the block in one step instead
      // of up to `tile` global climbs (config 4a: 10^4-vertex row chains,
      // S1 5.6 -> 3.9 ms).  A block with no in-range pointer pays one
      // barrier.  Every value is an ancestor, so the climb below stays exact.
      bool in = false;
#pragma unroll
      for (int i = 0; i < kCPer; i++) {
        sp[i * blockDim.x + t] = c[i];
        in |= !root[i] && (unsigned)(c[i] - (int)base) < (unsigned)tile;
      }
      if (__syncthreads_or(in)) {
        for (int r = 0; r < 12; r++) {
          int nc[kCPer];
          bool moved = false;
#pragma unroll
          for (int i = 0; i < kCPer; i++) {
            const unsigned rel = (unsigned)(c[i] - (int)base);
            nc[i] = rel < (unsigned)tile ? sp[rel] : c[i];
            moved |= nc[i] != c[i];
          }
          __syncthreads();
#pragma unroll
          for (int i = 0; i < kCPer; i++) {
            sp[i * blockDim.x + t] = nc[i];
            c[i] = nc[i];
          }
          if (!__syncthreads_or(moved)) break;
        }
      }
      __syncthreads();  // sp is rewritten next step
    }
    bool done[kCPer];
    unsigned pre[kCPer];  // kScan: root code << 30 | roots before this vertex in its warp (detached << 16 | listed)
#pragma unroll
    for (int i = 0; i < kCPer; i++) {
      done[i] = root[i] || v[i] >= n;
      int code = 0;
      if (v[i] < n) {
        roots += root[i];
        if (ri.flags) code = root_init(ri, hoff, v[i], root[i]);
      }
      if (kScan) {
        const unsigned b1 = __ballot_sync(0xffffffffu, code == 1), b2 = __ballot_sync(0xffffffffu, code == 2);
        const unsigned lt = (1u << (t & 31)) - 1;
        pre[i] = ((unsigned)code << 30) | (__popc(b2 & lt) << 16) | __popc(b1 & lt);
        if ((t & 31) == 0) s_wc[32 * wbuf + i * 8 + (t >> 5)] = (__popc(b2) << 16) | __popc(b1);
      }
    }
    // (fully unrolled: as a rolled loop -- the warp reconverging at every
    // step -- this climb ran 5x slower on config 4b's deep hook chains)
#pragma unroll
    for (int s = 0; s < kL1Steps; s++) {
      int x[kCPer];
      bool all = true;
#pragma unroll
      for (int i = 0; i < kCPer; i++) x[i] = done[i] ? c[i] : __ldca(comp + c[i]);
#pragma unroll
      for (int i = 0; i < kCPer; i++) {
        if (x[i] == c[i]) done[i] = true;
        else c[i] = x[i];
        all &= done[i];
      }
      if (all) break;
    }
#pragma unroll
    for (int i = 0; i < kCPer; i++) {
      while (!done[i]) {
        if (__ldca(comp + c[i]) == c[i]) break;  // root (stable during compress)
        const int cc = __ldcg(comp + c[i]);      // c's current pointer
        __stcg(comp + v[i], cc);
        mem[i] = cc;
        c[i] = cc;
      }
      if (c[i] != mem[i]) __stcg(comp + v[i], c[i]);  // (already-flat entries are not rewritten)
    }
    if (kScan) {
      // one barrier per tile, after the climb (mid-tile it held every warp's
      // climb behind the slowest warp's loads): every warp then scans the 32
      // (i, warp) counts itself (vertex order); the count buffer alternates
      // between tiles
      __syncthreads();
      const unsigned* wc = s_wc + 32 * wbuf;
      const unsigned x = wc[t & 31];
      unsigned incl = x;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((t & 31) >= o) incl += y;
      }
      if (t == 31) ri.sdesc[base / tile] = ((unsigned long long)(incl >> 16) << 32) | (incl & 0xffffu);  // tile counts
      const unsigned excl = incl - x;
#pragma unroll
      for (int i = 0; i < kCPer; i++) {
        const unsigned e = __shfl_sync(0xffffffffu, excl, i * 8 + (t >> 5));
        if ((pre[i] >> 30) == 0) continue;  // only the roots' ranks are ever read
        const unsigned w = e + (pre[i] & 0x3fffffffu);
        ri.rootidx[v[i]] = ((unsigned long long)(w >> 16) << 32) | (w & 0xffffu);  // rank inside the tile
      }
      wbuf ^= 1;
    }
  }
  if (nroots) block_count_add(nroots, roots);
  if (kAccept) block_count_add(hooks_out, hooked);
  if (giant_sc) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&giant_sc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      giant_of_block(comp, n, giant_sc, giant_enable);
      if (threadIdx.x == 0) giant_sc->ticket = 0;  // ready for the next stage
    }
  }
}

// Most frequent root among 1024 sampled vertices, computed by ONE block
// (any size dividing 1024) once comp is final: shared-memory open-addressing
// histogram, then a block argmax (ties -> smaller root, deterministic).
__device__ void giant_of_block(const int* comp, int n, Scalars* sc, bool enable) {
  constexpr int H = 2048, kSamples = 1024;
  __shared__ int key[H], num[H];
  __shared__ int bestc[32], bestv[32];
  const int t = threadIdx.x, nt = blockDim.x;
  for (int i = t; i < H; i += nt) { key[i] = -1; num[i] = 0; }
  __syncthreads();
  int cnt = 0, mine = 0x7fffffff;
  int slots[kSamples / 32];
  const int per = kSamples / nt;
  for (int k = 0; k < per; k++) {
    const int s = t + k * nt;
    const int v = (int)(hash32(0x9E3779B9u * (uint32_t)(s + 1)) % (uint32_t)n);
    int r = __ldcg(comp + v);  // comp may not be flat here: climb to the root
    for (int up = __ldcg(comp + r); up != r; up = __ldcg(comp + r)) r = up;
    int slot = hash32((uint32_t)r) & (H - 1);
    while (true) {
      int kk = atomicCAS(&key[slot], -1, r);
      if (kk == -1 || kk == r) break;
      slot = (slot + 1) & (H - 1);
    }
    atomicAdd(&num[slot], 1);
    slots[k] = slot;
  }
  __syncthreads();
  for (int k = 0; k < per; k++) {
    const int c = num[slots[k]], r = key[slots[k]];
    if (c > cnt || (c == cnt && r < mine)) { cnt = c; mine = r; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    int oc = __shfl_down_sync(0xffffffffu, cnt, o);
    int ov = __shfl_down_sync(0xffffffffu, mine, o);
    if (oc > cnt || (oc == cnt && ov < mine)) { cnt = oc; mine = ov; }
  }
  if ((t & 31) == 0) { bestc[t >> 5] = cnt; bestv[t >> 5] = mine; }
  __syncthreads();
  if (t < 32) {
    cnt = t < (nt >> 5) ? bestc[t] : -1;
    mine = t < (nt >> 5) ? bestv[t] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      int oc = __shfl_down_sync(0xffffffffu, cnt, o);
      int ov = __shfl_down_sync(0xffffffffu, mine, o);
      if (oc > cnt || (oc == cnt && ov < mine)) { cnt = oc; mine = ov; }
    }
    if (t == 0) {
      sc->giant = enable ? mine : -1;
      sc->giant_cnt = enable ? cnt : 0;
    }
  }
}

__global__ void k_find_giant(const int* __restrict__ comp, int n, Scalars* sc, bool enable) {
  pdl_enter();
  giant_of_block(comp, n, sc, enable);
}

// Remaining arcs, row-filtered: each warp takes 32 consecutive rows and drops
// the ones already in the sampled giant before touching their adjacency
// (after the sampling rounds that is almost every row of a low-diameter
// graph, so the 4m bytes of targets are mostly never read).  Rows of <= 32
// arcs are linked by their own lane; longer rows are linked by the whole warp
// striding over the arcs (a non-giant hub cannot serialise one thread).
constexpr int kSuperRow = 2048;

// 4-arc batches at 32 registers (full occupancy) measured best across
// configs 2/3/4b/4c/5 (8-arc batches at 64 registers: 4b/4c +4 %)
#ifndef FBCC_LR_BATCH
#define FBCC_LR_BATCH 4
#endif
#ifndef FBCC_LR_MINB
#define FBCC_LR_MINB 8
#endif
constexpr int kLinkBatch = FBCC_LR_BATCH;

template <int kPred, bool kRecord>
__global__ void __launch_bounds__(256, FBCC_LR_MINB) k_link_rows(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                   int n, int* comp, int2* fe, PredData pd, const Scalars* sc,
                                                   LongRows heavy, const int* __restrict__ nroots,
                                                   const int* __restrict__ hooks, int rounds) {
  pdl_enter();
  if (rounds > 0 && sets_left(nroots, hooks, rounds) <= 1) return;  // one set: nothing left to join
  const int giant = sc->giant;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += warps * 32) {
    const int v = (int)base + lane;
    int64_t rs = 0, re = 0;
    int p = v < n ? ldp(comp + v) : giant;
    // skip rows whose parent or grandparent is the giant root (sound: an
    // ancestor)
    if (p != giant && ldp(comp + p) != giant) {
      rs = __ldg(off + v);
      re = __ldg(off + v + 1);
    }
    // rows longer than kSuperRow (RMAT hubs outside the skeleton giant reach
    // 638k arcs) go to k_link_heavy: a CTA per row, or the whole grid for the
    // longest (LongRows)
    if (re - rs > kSuperRow) {
      heavy.defer(v, re - rs);
      rs = re = 0;
    }
    const bool heavy = re - rs > 32;
    if (!heavy && re > rs) {
      int4 rv;
      if (kPred == PRED_SKEL) rv = __ldg(pd.rec + v);
      // A row's links would be a chain of dependent finds; most targets are
      // already in v's set, so test kLinkBatch arcs at a time with independent loads
      // of comp[w] (and its parent) against v's current root and link only
      // the rest (config 2: one surviving degree-16 row no longer holds its
      // warp for 16 serial links).
      int root = -1;  // found lazily: under a predicate most rows keep no arc
      const int r0 = (int)rs, r1 = (int)re;  // slot indices fit 32 bits (check_sizes)
      for (int a0 = r0; a0 < r1; a0 += kLinkBatch) {
        const int cnt = r1 - a0 < kLinkBatch ? r1 - a0 : kLinkBatch;
        int w[kLinkBatch], c[kLinkBatch];
        bool k[kLinkBatch];
#pragma unroll
        for (int i = 0; i < kLinkBatch; i++) w[i] = i < cnt ? (int)__ldg(adj + a0 + i) : v;
        bool any = false;
#pragma unroll
        for (int i = 0; i < kLinkBatch; i++) {
          k[i] = i < cnt && keep<kPred>(pd, v, rv, w[i], a0 + i);
          any |= k[i];
        }
        if (!any) continue;
        if (root < 0) root = find_halve(comp, v);
#pragma unroll
        for (int i = 0; i < kLinkBatch; i++) c[i] = k[i] ? ldp(comp + w[i]) : root;
#pragma unroll
        for (int i = 0; i < kLinkBatch; i++)
          if (k[i] && c[i] != root) c[i] = ldp(comp + c[i]);
#pragma unroll
        for (int i = 0; i < kLinkBatch; i++)  // (root moves with each link: test k[i] again)
          if (k[i] && c[i] != root) root = link<kRecord>(v, w[i], comp, fe);
      }
    }
    unsigned hb = __ballot_sync(0xffffffffu, heavy);
    while (hb) {
      const int src = __ffs(hb) - 1;
      hb &= hb - 1;
      const int hv = __shfl_sync(0xffffffffu, v, src);
      const int64_t hs = __shfl_sync(0xffffffffu, rs, src), he = __shfl_sync(0xffffffffu, re, src);
      int4 rv;
      if (kPred == PRED_SKEL) rv = __ldg(pd.rec + hv);
      for (int64_t a = hs + lane; a < he; a += 32) {
        int w = (int)__ldg(adj + a);
        if (!keep<kPred>(pd, hv, rv, w, a)) continue;
        link<kRecord>(hv, w, comp, fe);
      }
    }
  }
}

// The deferred super-heavy rows (LongRows: a CTA per row up to kMegaRow
// arcs, the whole grid per longer row).
template <int kPred, bool kRecord>
__global__ void __launch_bounds__(256) k_link_heavy(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                    int* comp, int2* fe, PredData pd, LongRows heavy) {
  pdl_enter();
  int4 rv;
  heavy.visit(
      off, [&](int v, int64_t) {
        if (kPred == PRED_SKEL) rv = __ldg(pd.rec + v);
      },
      [&](int v, int64_t a) {
        const int w = (int)__ldg(adj + a);
        if (keep<kPred>(pd, v, rv, w, a)) link<kRecord>(v, w, comp, fe);
      });
}

// ---------------------------------------------------------------------------
// Round-0 compress of id-ordered forests (large meshes and paths: configs 4a,
// 4c).  Round 0's near rule hooks each vertex to its left neighbour, so the
// forest is made of chains of consecutive ids -- 10^4 per torus row, 10^8 on
// the path -- and k_compress<kJump> alone spends its time on waves of blocks
// each waiting for its left neighbour (4a 1.6 ms, 4c 1.9 ms for 0.8 GB of
// traffic).  When at least 3/4 of the vertices made a near hook:
//   1. k_jump_local: every 2048-id tile is flattened on its own (8 ids per
//      thread in registers, then pointer doubling in shared memory), stored,
//      and the tile's distinct exit targets -- the only vertices that can still
//      be interior to a chain -- are appended to a list;
//   2. k_jump_list: pointer doubling over the listed vertices only (tens of
//      thousands, all resident), which flattens every chain's interior;
//   3. the ordinary k_compress<kJump> then finds every vertex at most two
//      hops from its root.
// Any other graph (fewer near hooks, or more exit targets than the list
// holds) leaves both kernels at once and k_compress does all the work as
// before; both are launched only for n >= kJumpListMinN.
// ---------------------------------------------------------------------------
constexpr int kJumpTile = 2048;
constexpr int kJumpPer = kJumpTile / 256;
constexpr int kJumpListCap = 1 << 18;     // <= resident threads (148 x 2048)
constexpr int kJumpListMinN = 1 << 22;

__device__ __forceinline__ bool jump_mode(const Scalars* sc, int slot, int n) {
  return (int64_t)sc->near[slot] * 4 >= (int64_t)n * 3;
}

__global__ void __launch_bounds__(256) k_jump_local(int* comp, int n, Scalars* sc, int slot, int* __restrict__ list) {
  pdl_enter();
  if (!jump_mode(sc, slot, n)) return;
  __shared__ int sp[kJumpTile];
  __shared__ int wsum[8];
  __shared__ int lbase;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(comp) & 15) == 0;
  for (int64_t base = (int64_t)blockIdx.x * kJumpTile; base < n; base += (int64_t)gridDim.x * kJumpTile) {
    const int v0 = (int)base + t * kJumpPer;
    int c[kJumpPer], c_in[kJumpPer];
    if (vec_ok && v0 + kJumpPer <= n) {
      const int4 a = __ldcg(reinterpret_cast<const int4*>(comp + v0));
      const int4 b = __ldcg(reinterpret_cast<const int4*>(comp + v0) + 1);
      c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < kJumpPer; i++) c[i] = v0 + i < n ? __ldcg(comp + v0 + i) : v0 + i;
    }
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) c_in[i] = c[i];
    // Runs of consecutive ids, each hooked to its left neighbour, collapse in
    // one segmented copy-scan: an id whose pointer is not v - 1 (or the tile's
    // first id) heads a run, and every member takes its head's pointer.
    // Thread: sweep its 8 ids with the carry of the ids before them; the carry
    // is the pointer of the last head in the preceding threads (warp shuffles,
    // then the 8 warp totals through shared memory).
    bool has = false;  // this thread holds a head
    int hv = 0;        // ... the last one's pointer
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) {
      const bool head = c[i] != v0 + i - 1 || (t == 0 && i == 0);
      if (head) { has = true; hv = c[i]; }
    }
    bool ihas = has;  // inclusive scan over the lanes: (has, hv) of the last head at or before this thread
    int ihv = hv;
    for (int o = 1; o < 32; o <<= 1) {
      const int ph = __shfl_up_sync(0xffffffffu, (int)ihas, o), pv = __shfl_up_sync(0xffffffffu, ihv, o);
      if (lane >= o && !ihas) { ihas = ph != 0; ihv = pv; }
    }
    if (lane == 31) { wsum[warp] = ihas ? 1 : 0; sp[warp] = ihv; }
    __syncthreads();
    // exclusive carry: the previous lane's inclusive value, else the last head of the earlier warps
    int carry = __shfl_up_sync(0xffffffffu, ihv, 1);
    bool chas = __shfl_up_sync(0xffffffffu, (int)ihas, 1) != 0 && lane > 0;
    if (!chas) {
      for (int w = warp - 1; w >= 0; w--)
        if (wsum[w]) { carry = sp[w]; chas = true; break; }
    }
    __syncthreads();  // (wsum / sp are rewritten below)
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) {
      const bool head = c[i] != v0 + i - 1 || (t == 0 && i == 0);
      if (head) carry = c[i];
      else c[i] = carry;  // (a member always has a head before it in the tile: id base is one)
    }
    // (id r of the tile lives at sp[jslot(r)]: the 8 ids of a thread sit 256
    // words apart, so the warp's stores and the chain case's loads -- every
    // thread reading its left neighbour's last id -- are free of bank conflicts)
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) sp[i * 256 + t] = c[i];
    __syncthreads();
    // pointer doubling inside the tile (equal neighbours -- a run hooked to
    // one target -- share one load)
    for (int r = 0; r < 12; r++) {
      bool moved = false;
      int last_c = -1, last_nc = -1;
#pragma unroll
      for (int i = 0; i < kJumpPer; i++) {
        const int rel = c[i] - (int)base;
        if (rel >= 0 && rel < kJumpTile) {
          const int nc = c[i] == last_c ? last_nc : sp[(rel & (kJumpPer - 1)) * 256 + (rel >> 3)];
          last_c = c[i];
          last_nc = nc;
          moved |= nc != c[i];
          c[i] = nc;
        }
      }
      if (!__syncthreads_or(moved)) break;
#pragma unroll
      for (int i = 0; i < kJumpPer; i++) sp[i * 256 + t] = c[i];
      __syncthreads();
    }
    bool changed = false;
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) changed |= c[i] != c_in[i];
    if (changed) {
      if (vec_ok && v0 + kJumpPer <= n) {
        __stcg(reinterpret_cast<int4*>(comp + v0), make_int4(c[0], c[1], c[2], c[3]));
        __stcg(reinterpret_cast<int4*>(comp + v0) + 1, make_int4(c[4], c[5], c[6], c[7]));
      } else {
#pragma unroll
        for (int i = 0; i < kJumpPer; i++)
          if (v0 + i < n) __stcg(comp + v0 + i, c[i]);
      }
    }
    // the tile's exit targets (pointers leaving the tile), runs of equal
    // targets listed once; duplicates across tiles are harmless
    const int prev = t > 0 ? sp[(kJumpPer - 1) * 256 + t - 1] : -1;  // (sp holds the final values: the last round moved nothing)
    int cnt = 0;
    bool ex[kJumpPer];
#pragma unroll
    for (int i = 0; i < kJumpPer; i++) {
      ex[i] = v0 + i < n && c[i] < (int)base && c[i] != (i ? c[i - 1] : prev);
      cnt += ex[i];
    }
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (t == 0) {
      int tot = 0;
      for (int w = 0; w < 8; w++) { const int x = wsum[w]; wsum[w] = tot; tot += x; }
      lbase = tot ? atomicAdd(&sc->jlist_n[slot], tot) : 0;
    }
    __syncthreads();
    int pos = lbase + wsum[warp] + incl - cnt;
#pragma unroll
    for (int i = 0; i < kJumpPer; i++)
      if (ex[i]) {
        if (pos < kJumpListCap) list[pos] = c[i];
        pos++;
      }
    __syncthreads();  // sp / wsum / lbase are rewritten by the next tile
  }
}

// (grid: all kJumpListCap threads resident -- each entry rides the others' progress)
__global__ void __launch_bounds__(256) k_jump_list(int* comp, int n, const Scalars* sc, int slot,
                                                   const int* __restrict__ list) {
  pdl_enter();
  if (!jump_mode(sc, slot, n)) return;
  const int cnt = sc->jlist_n[slot];
  if (cnt > kJumpListCap) return;  // too many interior vertices: k_compress does the work
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const int u = list[i];
    int c = __ldcg(comp + u);
    while (true) {
      const int cc = __ldcg(comp + c);
      if (cc == c) break;
      __stcg(comp + u, cc);
      c = cc;
    }
  }
}

// The schedule shared by Stage 1 (no predicate, forest recorded), Stage 5
// (skeleton predicate) and the masked stand-alone op.  `slot` picks the
// sampling counters (0 / 8) in Scalars.
// round0_done: k_chunk_rows already ran sampling round 0 (Stage 1);
// ri: the final compress also writes Stage 2's root flags / list heads.
template <int kPred, bool kRecord>
static void run_cc(const Graph& g, int* comp, int2* fe, unsigned long long* prop, PredData pd, Scalars* sc,
                   int slot, cudaStream_t st, bool round0_done = false, RootInit ri = RootInit{}, int* jlist = nullptr,
                   const Scalars* hook_skip = nullptr) {
  const int B = 256;
  const int kBase = opt(OPT_SAMPLE_ROUNDS);
  // adaptive rounds kBase .. kRounds-1 (skip_round); Stage 5 may cap them separately
  int max_rounds = opt(OPT_MAX_ROUNDS);
  if (kPred == PRED_SKEL && opt(OPT_SKEL_MAX_ROUNDS) > 0) max_rounds = opt(OPT_SKEL_MAX_ROUNDS);
  const int kRounds = max_rounds > kBase ? std::min(max_rounds, 8) : kBase;
  const int gv = grid_for(g.n, B);
  // k_compress relies on concurrent threads advancing each other's pointers:
  // its grid must be fully resident (2048 threads/SM), or grid-stride
  // threads chase pointers owned by blocks that cannot be scheduled yet
  const int gres = grid_for((g.n + kCPer - 1) / kCPer, B, kCBlocks);
  int* nroots = sc->nroots + slot;  // device addresses (sc is a device pointer)
  int* hooks = sc->hooks + slot;
  // compress after round 0 (flattens the deep min-neighbour forest) and after
  // the last round (k_link_rows' giant test wants a flat array); rounds in
  // between only hook roots under roots and their proposers find() instead
  int cmask = opt(OPT_COMPRESS_MASK);
  if (cmask == 0) cmask = 1 | (kRounds > 0 ? 1 << (kRounds - 1) : 0);
  cmask |= 1;  // bit 0 always honoured: round 0's compress counts the roots the later rounds start from
  if (kRounds > 0 && round0_done) {
    // (k_chunk_rows)
  } else if (kRounds > 0) {
    const int sp = opt(OPT_SKEL_PARENT);
    launch(k_hook_min<kPred, kRecord>, gv, B, 0, st, g.off, g.adj, g.n, comp, fe, prop, pd, (sp & 1) != 0,
           (sp & 0x80) != 0 && !hook_skip, hook_skip);  // round 0
    note(K_HOOK_MIN);
  } else {
    launch(k_iota, gv, B, 0, st, comp, g.n, nullptr);
    note(K_IOTA);
  }
  for (int r = 0; r < kRounds; r++) {
    const bool flat = r == 0 || ((cmask >> (r - 1)) & 1);
    // a round followed by a compress folds its accept into it (OPT_ACCEPT_FOLD:
    // 1 always, 2 = auto: graphs of >= 2^22 vertices -- configs 4a/4b/4c/5
    // -1 to -4 %, while config 2 gains +6 % from the two-level trees a folded
    // accept can leave)
    const Scalars* hub_sc = (kPred == PRED_NONE && slot == 0) ? (const Scalars*)sc : nullptr;  // (skip_round's hub rule)
    const int af = opt(OPT_ACCEPT_FOLD);
    const bool fold = r > 0 && ((cmask >> r) & 1) && (af == 1 || (af == 2 && g.n >= (1 << 22)));
    if (r > 0) {
      launch(k_propose<kPred>, gv, B, 0, st, g.off, g.adj, g.n, r, comp, prop, pd, nroots, hooks, flat,
             ((opt(OPT_SKEL_PARENT) >> r) & 1) != 0, kBase, hub_sc);
      note(K_PROPOSE);
      if (!fold) {
        launch(k_accept<kRecord>, gv, B, 0, st, g.off, g.adj, g.n, r, comp, prop, fe, hooks, kBase, pd.warc,
               (const int*)nroots, hub_sc);
        note(K_ACCEPT);
      }
    }
    if ((cmask >> r) & 1) {
      // the last sampling round's compress also picks the giant
      const bool last_round = r == kRounds - 1 && opt(OPT_GIANT_FOLD);
      const int* skip_hooks = r >= kBase ? (const int*)hooks : nullptr;
      if (fold) {
        launch(k_compress<false, true, kRecord>, gres, B, 0, st, comp, g.n, (int*)nullptr, last_round ? sc : nullptr,
               opt(OPT_GIANT_SKIP) != 0, RootInit{}, skip_hooks, r, kBase, prop, hooks + r, fe, g.off, g.adj,
               pd.warc, (const int*)nroots, (const int*)hooks, hub_sc);
      } else {
        if (r == 0 && jlist && g.n >= kJumpListMinN) {  // id-ordered chains (see k_jump_local)
          launch(k_jump_local, grid_for((g.n + kJumpTile - 1) / kJumpTile, 1, 8), 256, 0, st, comp, g.n, sc, slot ? 1 : 0,
                 jlist);
          note(K_JUMP_LOCAL);
          launch(k_jump_list, grid_for(kJumpListCap, B, 2048 / B), B, 0, st, comp, g.n, (const Scalars*)sc,
                 slot ? 1 : 0, (const int*)jlist);
          note(K_JUMP_LIST);
        }
        launch(r == 0 ? k_compress<true> : k_compress<false>, gres, B, 0, st, comp, g.n, r == 0 ? nroots : nullptr,
               last_round ? sc : nullptr, opt(OPT_GIANT_SKIP) != 0, RootInit{}, skip_hooks, r, kBase,
               (unsigned long long*)nullptr, (int*)nullptr, (int2*)nullptr, (const int64_t*)nullptr,
               (const uint32_t*)nullptr, (const int*)nullptr, r > 0 ? (const int*)nroots : (const int*)nullptr,
               (const int*)hooks, hub_sc);
      }
      note(K_COMPRESS);
    }
  }
  if (!opt(OPT_GIANT_FOLD) || kRounds == 0 || !((cmask >> (kRounds - 1)) & 1)) {  // not folded
    launch(k_find_giant, 1, 1024, 0, st, comp, g.n, sc, opt(OPT_GIANT_SKIP) != 0 && kRounds > 0);
    note(K_FIND_GIANT);
  }
  if (g.m > 0) {
    // the proposal words (2n ints) are dead after the last accept: reuse them
    // as the super-heavy row lists
    LongRows heavy{reinterpret_cast<int*>(prop), 2 * g.n, sc->nheavy + (slot ? 1 : 0), sc->nmega + (slot ? 1 : 0)};
    launch(k_link_rows<kPred, kRecord>, grid_for(g.n, B, 32), B, 0, st, g.off, g.adj, g.n, comp, fe, pd, sc, heavy,
           (const int*)nroots, (const int*)hooks, ((cmask & 1) && kRounds > 0) ? kRounds : 0);
    note(K_LINK_ROWS);
    // always launched: whether a super-heavy row exists is a property of the
    // buffer contents, which a replayed plan must not bake in (an empty list
    // costs one ~2 us launch that exits at once)
    launch(k_link_heavy<kPred, kRecord>, grid_for((int64_t)kNumSMs * 2048, B), B, 0, st, g.off, g.adj, comp, fe,
           pd, heavy);
    note(K_LINK_HEAVY);
  }
  launch(ri.rootidx ? k_compress<false, false, false, true> : k_compress<false>,
         ri.rootidx ? grid_for((g.n + kCPer - 1) / kCPer, B, kCBlocksScan) : gres, B, 0, st, comp, g.n, nroots + 7,
         nullptr, false, ri, (const int*)nullptr, 0, 0,
         (unsigned long long*)nullptr, (int*)nullptr, (int2*)nullptr, (const int64_t*)nullptr,
         (const uint32_t*)nullptr, (const int*)nullptr, (const int*)nullptr, (const int*)nullptr,
         (const Scalars*)nullptr);  // final root count (= components)
  note(K_COMPRESS);
}

// ---------------------------------------------------------------------------
// Stage 1 on a streamed input (fbcc_run_host): the edge array arrives from
// host memory in arc ranges, and each range is linked as soon as its copy
// lands, so the union-find runs under the PCIe transfer instead of after it.
// Every undirected edge is linked once, from its smaller endpoint (the input
// is symmetric); no sampling or giant skip (both need the whole graph).  The
// labels are canonical (root = set minimum) and any spanning forest yields
// the same final outputs, so the result is identical to stage1_forest's.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_link_range(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                    const int* __restrict__ crow, int n, int64_t m, int64_t q0,
                                                    int64_t q1, int* comp, int2* fe) {
  pdl_enter();
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(adj) & 31) == 0);
  for (int64_t q = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < q1; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = q * kItems;
    const int64_t a1 = a0 + kItems < m ? a0 + kItems : m;
    uint32_t w[kItems];
    if (vec_ok && a1 - a0 == kItems) {
      ld_chunk8(adj + a0, w);
    } else {
#pragma unroll
      for (int i = 0; i < kItems; i++) w[i] = (a0 + i < a1) ? __ldg(adj + a0 + i) : 0u;
    }
    int v = __ldg(crow + q);
    if (v < 0) v = row_of(off, 0, n - 1, a0);
    int64_t re = __ldg(off + v + 1);
#pragma unroll
    for (int i = 0; i < kItems; i++) {
      const int64_t a = a0 + i;
      if (a < a1) {
        if (a >= re) {
          v = next_row(off, v, n, a);
          re = __ldg(off + v + 1);
        }
        if (v < (int)w[i]) link<true>(v, (int)w[i], comp, fe);
      }
    }
  }
}

void stage1_stream_begin(const Graph& g, int* comp, cudaStream_t st) {
  launch(k_iota, grid_for(g.n, 256), 256, 0, st, comp, g.n, nullptr);
  note(K_IOTA);
}

void stage1_stream_range(const Graph& g, int64_t q0, int64_t q1, int* comp, int2* fe, cudaStream_t st) {
  if (q1 <= q0) return;
  launch(k_link_range, grid_for(q1 - q0, 256, 16), 256, 0, st, g.off, g.adj, g.crow, g.n, g.m, q0, q1, comp, fe);
  note(K_LINK_ROWS);
}

void stage1_stream_finish(const Graph& g, int* comp, Scalars* sc, cudaStream_t st, RootInit ri) {
  const int B = 256;
  launch(ri.rootidx ? k_compress<true, false, false, true> : k_compress<true>,
         grid_for((g.n + kCPer - 1) / kCPer, B, ri.rootidx ? kCBlocksScan : kCBlocks),
         B, 0, st, comp, g.n, sc->nroots + 7, nullptr, false, ri,
         (const int*)nullptr, 0, 0, (unsigned long long*)nullptr, (int*)nullptr, (int2*)nullptr,
         (const int64_t*)nullptr, (const uint32_t*)nullptr, (const int*)nullptr, (const int*)nullptr,
         (const int*)nullptr, (const Scalars*)nullptr);
  note(K_COMPRESS);
}

__global__ void k_widen(const int* __restrict__ src, int64_t* __restrict__ dst, int64_t count) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int64_t)(uint32_t)__ldg(src + i);
}

void widen_offsets(const int* src, int64_t* dst, int64_t n, cudaStream_t st) {
  launch(k_widen, grid_for(n + 1, 256), 256, 0, st, src, dst, n + 1);
  note(K_WIDEN);
}

void stage1_forest(const Graph& g, int* comp, int2* fe, unsigned long long* prop, Scalars* sc, cudaStream_t st,
                   bool round0_done, RootInit ri, const int* warc, int* jlist) {
  PredData pd{};
  pd.warc = warc;
  run_cc<PRED_NONE, true>(g, comp, fe, prop, pd, sc, 0, st, round0_done, ri, round0_done ? jlist : nullptr);
}

void stage5_skeleton_cc(const Graph& g, const int4* rec, int* label, unsigned long long* prop, Scalars* sc,
                        cudaStream_t st, const int* w0, bool round0_done, int* jlist, bool round0_if_ordered) {
  PredData pd{};
  pd.rec = rec;
  pd.w0 = w0;
  pd.warc = w0;  // (rows [n, 3n): arcs 1 and 2; k_chunk_rows recorded all three)
  // round0_done: Stage 4's k_fence already hooked every vertex under its plain parent
  run_cc<PRED_SKEL, false>(g, label, nullptr, prop, pd, sc, 8, st, round0_done, RootInit{},
                           (round0_done || round0_if_ordered) ? jlist : nullptr, round0_if_ordered ? sc : nullptr);
}

void masked_cc(const Graph& g, const uint8_t* mask, int* comp, int2* fe, unsigned long long* prop, Scalars* sc,
               cudaStream_t st) {
  if (!mask) {
    run_cc<PRED_NONE, true>(g, comp, fe, prop, PredData{}, sc, 0, st);
    return;
  }
  PredData pd{};
  pd.mask = mask;
  pd.off = g.off;
  pd.adj = g.adj;
  run_cc<PRED_MASK, true>(g, comp, fe, prop, pd, sc, 0, st);
}

}  // namespace fbcc
