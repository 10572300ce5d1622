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

// Root of x with path halving.  Only non-roots are rewritten, always to an
// ancestor (ancestors stay ancestors: sets only merge), and roots change only
// through the hooking CAS -- so the concurrent plain stores are benign.
//
// Parent reads are L1-cacheable (ld.global.ca).  Every value comp[x] ever
// held is an ancestor of x, so a stale line can only (a) make two endpoints
// look joined when they truly are, or (b) offer a "root" that is no longer
// one -- the CAS then fails and returns the fresh parent, so every retry
// climbs.  What the L1 buys: once most vertices share one giant root, every
// find ends at the same word; served from L2 (ld.relaxed.gpu) those ~1M
// requests serialise on a single L2 slice.
__device__ __forceinline__ int ldp(const int* p) { return __ldca(p); }

__device__ __forceinline__ int find_halve(int* comp, int x, bool halve) {
  int p = ldp(comp + x);
  while (p != x) {
    int gp = ldp(comp + p);
    if (gp == p) return p;
    if (halve) comp[x] = gp;
    x = gp;
    p = ldp(comp + x);
  }
  return x;
}

// Hook the larger root under the smaller.  ru/rw are roots of the sets
// holding u and w when found; a successful CAS hooks root `hi` under `lo`,
// whose set holds the other endpoint (roots are set minima, root(lo) <= lo <
// hi), so (u, w) is a spanning-forest edge joining two distinct sets.
template <bool kRecord>
__device__ __forceinline__ void link(int u, int w, int* comp, int2* fe, bool halve) {
  int ru = find_halve(comp, u, halve);
  int rw = find_halve(comp, w, halve);
  while (ru != rw) {
    int hi = ru > rw ? ru : rw;
    int lo = ru + rw - hi;
    int prev = atomicCAS(comp + hi, hi, lo);
    if (prev == hi) {
      if (kRecord) fe[hi] = make_int2(u, w);
      return;
    }
    ru = find_halve(comp, prev, halve);  // hi was hooked meanwhile: climb on
    rw = find_halve(comp, lo, halve);
  }
}

// chunk -> row table (see visit_arc_chunks): row v owns the chunks whose
// first arc lies in it
__global__ void k_chunk_rows(const int64_t* __restrict__ off, int n, int* __restrict__ crow) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int64_t q0 = (__ldg(off + v) + kItems - 1) / kItems;
    int64_t q1 = (__ldg(off + v + 1) + kItems - 1) / kItems;
    if (q1 - q0 > kRowChunks) continue;  // hub row: consumers binary-search
    for (int64_t q = q0; q < q1; q++) crow[q] = v;
  }
}

void build_chunk_rows(const Graph& g, int* crow, cudaStream_t st) {
  int64_t nchunks = (g.m + kItems - 1) / kItems;
  if (nchunks == 0) return;
  cudaMemsetAsync(crow, 0xFF, sizeof(int) * nchunks, st);
  note(K_MEMSET);
  k_chunk_rows<<<grid_for(g.n, 256), 256, 0, st>>>(g.off, g.n, crow);
  note(K_CHUNK_ROWS);
}

// comp = identity; also resets the proposal words (one pass, no memset node)
__global__ void k_iota(int* __restrict__ comp, int n, unsigned long long* __restrict__ prop) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    comp[v] = v;
    if (prop) prop[v] = ~0ull;
  }
}

// Best-effort sampling round: one CAS attempt on the (post-compress, hence
// depth-1) parents of v and of its round-th neighbour, no climbing.  A win is
// still a valid forest edge (hi was a root; lo is an ancestor of the other
// endpoint, root(lo) <= lo < hi); a loss is simply left to k_link_rest, which
// re-covers every arc of every row outside the giant component.  Climbing
// here is what made round 1 contention-bound: after round 0 the ~n/17
// local-minimum roots all merge into one giant and every failed CAS then
// chases the same few hot roots.
template <bool kSkel, bool kRecord>
__global__ void k_sample_link(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n,
                              int round, int* comp, int2* fe, const int4* __restrict__ rec, bool full,
                              bool halve) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int64_t s = __ldg(off + v) + round;
    if (s >= __ldg(off + v + 1)) continue;
    int w = (int)__ldg(adj + s);
    if (kSkel) {
      if (!skel_keep(v, __ldg(rec + v), w, __ldg(rec + w))) continue;
    }
    if (full) {  // exact Afforest sampling: climb until joined
      link<kRecord>(v, w, comp, fe, halve);
      continue;
    }
    int ru = ldp(comp + v), rw = ldp(comp + w);
    if (ru == rw) continue;
    int hi = ru > rw ? ru : rw;
    int lo = ru + rw - hi;
    // one CAS per distinct target root per warp (later rounds have few roots)
    unsigned peers = __match_any_sync(__activemask(), hi);
    if ((threadIdx.x & 31) != __ffs(peers) - 1) continue;
    if (atomicCAS(comp + hi, hi, lo) == hi && kRecord) fe[hi] = make_int2(v, w);
  }
}

// Propose/accept sampling round (the default).  Against the round-start
// components (comp is flat after the previous compress and is not written
// during the propose kernel), every vertex proposes its round-th arc to the
// HIGHER of the two component roots with one fire-and-forget 64-bit
// atomicMin of (lower root << 32 | arc slot).  Same-address REDs pipeline in
// the L2 atomic unit instead of serialising retry loops, so the many-to-few
// merges of later rounds are cheap.  k_accept then hooks every proposed-to
// root under its minimum proposal: hooks always point to a smaller
// round-start root, so they form a forest over the components (no cycles),
// and each accepted hook records its arc -- one forest edge per merge.
//
// Proposers are thinned to ~kPerRoot per surviving root: on config 2 the
// rounds go 1M -> 65k -> 565 -> 1 components, and round 2 would otherwise
// aim 941k proposals at 565 roots (up to 18k REDs on one word).  A root that
// draws no proposer simply stays for the next round / k_link_rest.
constexpr int kPerRoot = 32;

template <bool kSkel>
__global__ void k_propose(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int round,
                          int* comp, unsigned long long* prop, const int4* __restrict__ rec,
                          const int* __restrict__ nroots, const int* __restrict__ hooks, bool flat) {
  // participate iff hash < thr / 2^24, thr = min(1, kPerRoot * roots / n);
  // roots at round start = roots counted after round 0 minus later hooks
  uint32_t thr = 1u << 24;
  if (round > 0) {
    int64_t R = nroots[0];
    for (int i = 1; i < round; i++) R -= hooks[i];
    uint64_t t = ((uint64_t)kPerRoot * (uint64_t)(R > 0 ? R : 0) << 24) / (uint64_t)n;
    if (t < thr) thr = (uint32_t)t;
  }
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (thr < (1u << 24) && (hash32((uint32_t)v * 0x9E3779B1u + (uint32_t)round) >> 8) >= thr) continue;
    int64_t s = __ldg(off + v) + round;
    if (s >= __ldg(off + v + 1)) continue;
    int w = (int)__ldg(adj + s);
    if (kSkel) {
      if (!skel_keep(v, __ldg(rec + v), w, __ldg(rec + w))) continue;
    }
    // flat after a compress; otherwise (rounds >= 1 hook root -> root only,
    // so trees stay shallow) find with halving
    int ru = flat ? ldp(comp + v) : find_halve(comp, v, true);
    int rw = flat ? ldp(comp + w) : find_halve(comp, w, true);
    if (ru == rw) continue;
    int hi = ru > rw ? ru : rw;
    int lo = ru + rw - hi;
    // any proposal is a valid hook, so lanes aiming at the same root send one
    // (small components below the giant's root all aim at it in round 2)
    unsigned peers = __match_any_sync(__activemask(), hi);
    if ((threadIdx.x & 31) != __ffs(peers) - 1) continue;
    // low word = the proposer: its arc is off[v] + round, no search on accept
    atomicMin(prop + hi, ((unsigned long long)(unsigned)lo << 32) | (unsigned long long)(uint32_t)v);
  }
}

template <bool kRecord>
__global__ void k_accept(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int round, int* comp,
                         unsigned long long* prop, int2* fe, int* hooks) {
  int hooked = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    unsigned long long key = prop[v];
    if (key == ~0ull) continue;
    prop[v] = ~0ull;  // ready for the next round
    int lo = (int)(key >> 32);
    comp[v] = lo;     // v is a round-start root (only roots receive proposals)
    hooked++;
    if (kRecord) {
      int u = (int)(key & 0xffffffffull);
      fe[v] = make_int2(u, (int)__ldg(adj + __ldg(off + u) + round));
    }
  }
  block_count_add(hooks + round, hooked);
}

// pointer jumping to the root (the root is the component minimum)
// (optionally counting the roots into *nroots).  Every step stores the
// advanced pointer and reads the parent's CURRENT pointer from L2, so
// concurrent threads ride each other's progress: pointer doubling, ~log2(depth)
// steps per thread.  Walking to the root and storing once at the end is
// O(depth) per thread -- O(n^2) on a 10^8-vertex path whose round-0 hooks
// form one chain (3.2 s measured on config 4c).
//
// No hooks happen during a compress, so a root's entry is stable: the
// "is c a root" test may use an L1-cached load (the giant root's word is then
// served per SM instead of hammering one L2 slice), and only non-root
// pointers -- which other threads are advancing -- are re-read from L2.
__global__ void k_compress(int* comp, int n, int* nroots) {
  int roots = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int c = __ldcg(comp + v);
    roots += (c == v);
    if (c == v) continue;
    while (true) {
      if (__ldca(comp + c) == c) break;  // root (stable during compress)
      int cc = __ldcg(comp + c);           // c's current pointer
      __stcg(comp + v, cc);
      c = cc;
    }
  }
  if (nroots) block_count_add(nroots, roots);
}

// Most frequent root among 1024 sampled vertices (one block of 1024):
// shared-memory open-addressing histogram, then a block argmax.
__global__ void k_find_giant(const int* __restrict__ comp, int n, Scalars* sc, bool enable) {
  constexpr int H = 2048;
  __shared__ int key[H], num[H];
  __shared__ int bestc[32], bestv[32];
  int t = threadIdx.x;
  for (int i = t; i < H; i += 1024) { key[i] = -1; num[i] = 0; }
  __syncthreads();
  int v = (int)(hash32(0x9E3779B9u * (uint32_t)(t + 1)) % (uint32_t)n);
  int mine = comp[v];  // comp may not be flat here: climb to the root
  for (int up = comp[mine]; up != mine; up = comp[mine]) mine = up;
  int slot = hash32((uint32_t)mine) & (H - 1);
  while (true) {
    int k = atomicCAS(&key[slot], -1, mine);
    if (k == -1 || k == mine) break;
    slot = (slot + 1) & (H - 1);
  }
  int cnt = atomicAdd(&num[slot], 1) + 1;  // any member's final count works below
  __syncthreads();
  cnt = num[slot];
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
    if (t == 0) sc->giant = enable ? mine : -1;
  }
}

template <bool kSkel, bool kRecord>
struct LinkRestVisitor {
  int* comp;
  int2* fe;
  const int4* rec;
  int giant;
  int rounds;
  bool halve;
  int64_t rs;
  bool skip;
  int4 rv;
  __device__ __forceinline__ void begin(int v, int64_t s, int64_t e) {
    rs = s;
    int p = ldp(comp + v);
    skip = p == giant || ldp(comp + p) == giant;  // sound: giant is an ancestor
    if (kSkel && !skip) rv = __ldg(rec + v);
  }
  __device__ __forceinline__ void arc(int v, int64_t a, int w) {
    if (skip || a - rs < rounds) return;
    if (kSkel) {
      if (!skel_keep(v, rv, w, __ldg(rec + w))) return;
    }
    link<kRecord>(v, w, comp, fe, halve);
  }
  __device__ __forceinline__ void end(int, bool) {}
};

template <bool kSkel, bool kRecord>
__global__ void __launch_bounds__(256) k_link_rest(const int64_t* __restrict__ off,
                                                   const uint32_t* __restrict__ adj, const int* __restrict__ crow, int n, int64_t m,
                                                   int rounds, int* comp, int2* fe,
                                                   const int4* __restrict__ rec, const Scalars* sc, bool halve) {
  LinkRestVisitor<kSkel, kRecord> vis;
  vis.comp = comp;
  vis.fe = fe;
  vis.rec = rec;
  vis.giant = sc->giant;
  vis.rounds = rounds;
  vis.halve = halve;
  visit_arc_chunks(off, adj, crow, n, m, vis);
}

// Remaining arcs, row-filtered: each warp takes 32 consecutive rows and drops
// the ones already in the sampled giant before touching their adjacency
// (after the sampling rounds that is almost every row of a low-diameter
// graph, so the 4m bytes of targets are mostly never read).  Rows of <= 32
// arcs are linked by their own lane; longer rows are linked by the whole warp
// striding over the arcs (a non-giant hub cannot serialise one thread).
template <bool kSkel, bool kRecord>
__global__ void __launch_bounds__(256) k_link_rows(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                   int n, int* comp, int2* fe, const int4* __restrict__ rec,
                                                   const Scalars* sc, bool halve) {
  const int giant = sc->giant;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < n; base += warps * 32) {
    const int v = (int)base + lane;
    int64_t rs = 0, re = 0;
    int p = v < n ? ldp(comp + v) : giant;
    // skip rows whose parent or grandparent is the giant root (sound: an
    // ancestor; comp need not be flat after the last sampling round)
    if (p != giant && ldp(comp + p) != giant) {
      rs = __ldg(off + v);
      re = __ldg(off + v + 1);
    }
    const bool heavy = re - rs > 32;
    if (!heavy && re > rs) {
      int4 rv;
      if (kSkel) rv = __ldg(rec + v);
      for (int64_t a = rs; a < re; a++) {
        int w = (int)__ldg(adj + a);
        if (kSkel && !skel_keep(v, rv, w, __ldg(rec + w))) continue;
        link<kRecord>(v, w, comp, fe, halve);
      }
    }
    unsigned hb = __ballot_sync(0xffffffffu, heavy);
    while (hb) {
      const int src = __ffs(hb) - 1;
      hb &= hb - 1;
      const int hv = __shfl_sync(0xffffffffu, v, src);
      const int64_t hs = __shfl_sync(0xffffffffu, rs, src), he = __shfl_sync(0xffffffffu, re, src);
      int4 rv;
      if (kSkel) rv = __ldg(rec + hv);
      for (int64_t a = hs + lane; a < he; a += 32) {
        int w = (int)__ldg(adj + a);
        if (kSkel && !skel_keep(hv, rv, w, __ldg(rec + w))) continue;
        link<kRecord>(hv, w, comp, fe, halve);
      }
    }
  }
}

// Afforest schedule shared by Stage 1 (kSkel=false, record forest) and
// Stage 5 (kSkel=true, no forest).
template <bool kSkel, bool kRecord>
static void run_cc(const Graph& g, int* comp, int2* fe, unsigned long long* prop, const int4* rec, Scalars* sc,
                   cudaStream_t st) {
  const int B = 256;
  const int kRounds = g_opt[OPT_SAMPLE_ROUNDS];
  const bool halve = g_opt[OPT_FIND_HALVING] != 0;
  const bool propose = g_opt[OPT_SAMPLE_MODE] == 0;
  int* nroots = sc->nroots + (kSkel ? 8 : 0);  // device addresses (sc is a device pointer)
  int* hooks = sc->hooks + (kSkel ? 8 : 0);
  // compress after round 0 (flattens the deep min-neighbour forest) and after
  // the last round (k_link_rows' giant test wants a flat array); rounds in
  // between only hook roots under roots and their proposers find() instead
  int cmask = g_opt[OPT_COMPRESS_MASK];
  if (cmask == 0) cmask = 1 | (kRounds > 0 ? 1 << (kRounds - 1) : 0);
  int gv = grid_for(g.n, B);
  // k_compress relies on concurrent threads advancing each other's pointers:
  // its grid must be fully resident (2048 threads/SM), or grid-stride
  // threads chase pointers owned by blocks that cannot be scheduled yet
  const int gres = grid_for(g.n, B, 2048 / B);
  k_iota<<<gv, B, 0, st>>>(comp, g.n, propose && kRounds > 0 ? prop : nullptr);
  note(K_IOTA);
  for (int r = 0; r < kRounds; r++) {
    const bool flat = r == 0 || ((cmask >> (r - 1)) & 1);
    if (propose) {
      k_propose<kSkel><<<gv, B, 0, st>>>(g.off, g.adj, g.n, r, comp, prop, rec, nroots, hooks, flat);
      note(K_SAMPLE_LINK);
      k_accept<kRecord><<<gv, B, 0, st>>>(g.off, g.adj, g.n, r, comp, prop, fe, hooks);
      note(K_ACCEPT);
    } else {
      k_sample_link<kSkel, kRecord><<<gv, B, 0, st>>>(g.off, g.adj, g.n, r, comp, fe, rec,
                                                      (g_opt[OPT_SAMPLE_FULL] >> r) & 1, halve);
      note(K_SAMPLE_LINK);
    }
    // round 0 hooks every vertex to its smallest neighbour (deep trees: a
    // path becomes one chain) and must be flattened; later rounds hook roots
    // under roots, and their proposers find() through the shallow result
    if (((cmask >> r) & 1) || !propose) {
      k_compress<<<gres, B, 0, st>>>(comp, g.n, r == 0 ? nroots : nullptr);
      note(K_COMPRESS);
    }
  }
  k_find_giant<<<1, 1024, 0, st>>>(comp, g.n, sc, g_opt[OPT_GIANT_SKIP] != 0 && kRounds > 0);
  note(K_FIND_GIANT);
  if (g.m > 0) {
    if (g_opt[OPT_LINK_MODE] == 0) {
      k_link_rows<kSkel, kRecord><<<grid_for(g.n, B, 32), B, 0, st>>>(g.off, g.adj, g.n, comp, fe, rec, sc, halve);
    } else {
      int64_t nchunks = (g.m + kItems - 1) / kItems;
      k_link_rest<kSkel, kRecord><<<grid_for(nchunks, B, 32), B, 0, st>>>(g.off, g.adj, g.crow, g.n, g.m,
                                                                            /*skip arcs below*/ 0, comp, fe, rec,
                                                                            sc, halve);
    }
    note(K_LINK_REST);
  }
  k_compress<<<gres, B, 0, st>>>(comp, g.n, nullptr);
  note(K_COMPRESS);
}

void stage1_forest(const Graph& g, int* comp, int2* fe, unsigned long long* prop, Scalars* sc, cudaStream_t st) {
  run_cc<false, true>(g, comp, fe, prop, nullptr, sc, st);
}

void stage5_skeleton_cc(const Graph& g, const int4* rec, int* label, unsigned long long* prop, Scalars* sc,
                        cudaStream_t st) {
  run_cc<true, false>(g, label, nullptr, prop, rec, sc, st);
}

}  // namespace fbcc
