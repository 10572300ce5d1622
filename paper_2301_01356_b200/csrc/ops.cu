// ops.cu -- stand-alone device operations with the reference's stage APIs
// (SURVEY.md §8(f)), built from the pipeline's kernels:
//
//   op_connected_components  connected_components(g, keep_edge)   connectivity.py:593-611
//   op_list_ranking          list_ranking(nxt, heads)             euler_tour.py:322-358
//   op_build_euler_tour      build_euler_tour(n, tree_edges, lab) euler_tour.py:361-394
//   op_compute_tags          compute_tags(g, forest)              tagging.py:300-304
//   op_extract_bccs          extract_bccs(labeling)               bcc.py:199-219
//   op_symmetrize            symmetrize(edges, n)                 graphs.py:119-143
//
// All are exact: build_euler_tour even reproduces the reference's tour
// order -- each vertex's out-arcs are ordered by pair index (a radix sort of
// (vertex, pair) keys), which is the slot order of the reference's counting
// sort (_tree_csr euler_tour.py:68-89) -- so parent/first/last are identical
// to the reference's, not just a valid rooting.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "kernels.cuh"
#include "ops.cuh"

namespace fbcc {

// error bits in Scalars::err
enum : int { E_RANGE = 1, E_CYCLE = 2, E_COVER = 4, E_LABELS = 8, E_NOT_FOREST = 16 };

__device__ __forceinline__ void raise_err(Scalars* sc, int bit) { atomicOr(&sc->err, bit); }

// ---------------------------------------------------------------------------
// list ranking: general multi-list input with the reference's validation
// ---------------------------------------------------------------------------
// Wyllie pointer jumping to each list's tail (tails point to themselves),
// then rank = dist(head) - dist(e).  O(L log L), but this entry point only
// serves the stand-alone API; the pipeline uses the ruling-set ranking.
__global__ void k_lr_init(const int* __restrict__ nxt, int64_t L, int* ptr, int* dist, int* indeg, Scalars* sc) {
  pdl_enter();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    int s = nxt[e];
    if (s >= L || s < -1) { raise_err(sc, E_COVER); s = -1; }
    ptr[e] = s >= 0 ? s : (int)e;
    dist[e] = s >= 0 ? 1 : 0;
    if (s >= 0 && atomicAdd(indeg + s, 1) >= 1) raise_err(sc, E_COVER);  // two predecessors: merge
  }
}

__global__ void k_lr_jump(int64_t L, const int* __restrict__ p0, const int* __restrict__ d0, int* p1, int* d1) {
  pdl_enter();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    int p = p0[e];
    d1[e] = d0[e] + (p != (int)e ? d0[p] : 0);
    p1[e] = p0[p];
  }
}

__global__ void k_lr_heads(const int* __restrict__ heads, int64_t H, int64_t L, const int* __restrict__ nxt,
                           const int* __restrict__ ptr, const int* __restrict__ indeg, int* tailhead, Scalars* sc) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < H; i += (int64_t)gridDim.x * blockDim.x) {
    int h = heads[i];
    if (h < 0) continue;  // ignored, like the reference
    if (h >= L) { raise_err(sc, E_COVER); continue; }
    int t = ptr[h];
    if (nxt[t] >= 0) { raise_err(sc, E_CYCLE); continue; }     // never reached a tail
    if (indeg[h] != 0) { raise_err(sc, E_COVER); continue; }   // head in mid-list
    if (atomicCAS(tailhead + t, -1, h) != -1) raise_err(sc, E_COVER);  // two heads, one list
  }
}

__global__ void k_lr_ranks(int64_t L, const int* __restrict__ nxt, const int* __restrict__ ptr,
                           const int* __restrict__ dist, const int* __restrict__ tailhead, int* ranks, Scalars* sc) {
  pdl_enter();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < L; e += (int64_t)gridDim.x * blockDim.x) {
    int t = ptr[e];
    int h = nxt[t] < 0 ? tailhead[t] : -1;
    if (h < 0) { raise_err(sc, E_COVER); ranks[e] = -1; continue; }  // unreachable / headless cycle
    ranks[e] = dist[h] - dist[e];
  }
}

size_t op_list_ranking_bytes(int64_t L) { return 256 + 5 * 4 * (size_t)(L + 64); }

int op_list_ranking(const int* nxt, int64_t L, const int* heads, int64_t H, int* ranks, void* ws, Scalars* sc,
                    cudaStream_t st) {
  const int B = 256;
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { void* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  int* p0 = (int*)take(4 * L);
  int* d0 = (int*)take(4 * L);
  int* p1 = (int*)take(4 * L);
  int* d1 = (int*)take(4 * L);
  int* indeg = (int*)take(4 * L);
  cudaMemsetAsync(indeg, 0, 4 * L, st);
  launch(k_lr_init, grid_for(L, B), B, 0, st, nxt, L, p0, d0, indeg, sc);
  int rounds = 1;
  while ((1ll << rounds) < L + 1) rounds++;
  for (int r = 0; r < rounds; r++) {
    launch(k_lr_jump, grid_for(L, B), B, 0, st, L, p0, d0, p1, d1);
    int* t = p0; p0 = p1; p1 = t;
    t = d0; d0 = d1; d1 = t;
  }
  int* tailhead = p1;  // reuse
  cudaMemsetAsync(tailhead, 0xFF, 4 * L, st);
  if (H > 0) launch(k_lr_heads, grid_for(H, B), B, 0, st, heads, H, L, nxt, p0, indeg, tailhead, sc);
  launch(k_lr_ranks, grid_for(L, B), B, 0, st, L, nxt, p0, d0, tailhead, ranks, sc);
  return 0;
}

// ---------------------------------------------------------------------------
// build_euler_tour: root a given forest (pairs) at min-id roots
// ---------------------------------------------------------------------------
__global__ void k_pairs_check(const int2* __restrict__ pairs, int64_t k, int n, Scalars* sc) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    int2 e = pairs[i];
    if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n) raise_err(sc, E_RANGE);
  }
}

__global__ void k_iota2(int* comp, int n) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) comp[v] = v;
}

// union the pairs (labels not given): a pair whose ends are already joined
// closes a cycle -- not a forest
__global__ void k_union_pairs(const int2* __restrict__ pairs, int64_t k, int n, int* comp, Scalars* sc) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    int2 e = pairs[i];
    if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n) continue;  // reported by k_pairs_check
    int ru = e.x, rw = e.y;
    while (true) {
      while (ld_relaxed(comp + ru) != ru) ru = ld_relaxed(comp + ru);
      while (ld_relaxed(comp + rw) != rw) rw = ld_relaxed(comp + rw);
      if (ru == rw) { raise_err(sc, E_NOT_FOREST); break; }
      int hi = ru > rw ? ru : rw, lo = ru + rw - hi;
      if (atomicCAS(comp + hi, hi, lo) == hi) break;
    }
  }
}

__global__ void k_flatten(int* comp, int n) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int c = comp[v];
    while (comp[c] != c) c = comp[c];
    comp[v] = c;
  }
}

__global__ void k_nonroot_flags(const int* __restrict__ comp, int n, int* flags) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x)
    flags[v] = v < n ? (comp[v] != v) : 0;
}

// pair i is owned by the i-th non-root vertex x_i: fe[x_i] = pair i, and its
// two arcs are elements 2x_i (u->v) and 2x_i+1 (v->u); sort keys order every
// vertex's out-arcs by pair index (the reference's CSR slot order)
__global__ void k_place_pairs(const int2* __restrict__ pairs, int64_t k, const int* __restrict__ comp,
                              const int* __restrict__ nrank, int n, int2* fe, unsigned long long* keys, int* vals,
                              Scalars* sc) {
  pdl_enter();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    if (comp[x] == x) continue;
    int i = nrank[x];
    if (i >= k) continue;
    int2 e = pairs[i];
    if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n) continue;  // reported by k_pairs_check
    if (comp[e.x] != comp[e.y]) raise_err(sc, E_LABELS);  // labels inconsistent with the forest
    fe[x] = e;
    keys[2 * i] = ((unsigned long long)(unsigned)e.x << 32) | (unsigned)i;
    vals[2 * i] = 2 * x;
    keys[2 * i + 1] = ((unsigned long long)(unsigned)e.y << 32) | (unsigned)i;
    vals[2 * i + 1] = 2 * x + 1;
  }
}

__global__ void k_sorted_lists(const unsigned long long* __restrict__ keys, const int* __restrict__ vals, int64_t K2,
                               int* lhead, int* nexto) {
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K2; j += (int64_t)gridDim.x * blockDim.x) {
    unsigned vx = (unsigned)(keys[j] >> 32);
    if (j == 0 || (unsigned)(keys[j - 1] >> 32) != vx) lhead[vx] = vals[j];
    nexto[vals[j]] = (j + 1 < K2 && (unsigned)(keys[j + 1] >> 32) == vx) ? vals[j + 1] : -1;
  }
}

__global__ void k_check_rooted(const int* __restrict__ comp, const int* __restrict__ lhead, int n,
                               const int* __restrict__ nrank, int64_t k, Scalars* sc) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x == 0 && nrank[n] != k) raise_err(sc, E_LABELS);  // #non-roots != #edges
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (comp[v] != v && lhead[v] < 0) raise_err(sc, E_LABELS);  // non-root without a tree edge
}

__global__ void k_export_forest(const int4* __restrict__ rec, int n, int* parent, int* first, int* last) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int4 r = rec[v];
    parent[v] = r.z;
    first[v] = r.x;
    last[v] = r.y;
  }
}

// ---------------------------------------------------------------------------
// compute_tags on a given rooted forest
// ---------------------------------------------------------------------------
__global__ void k_rec_ap(const int* __restrict__ parent, const int* __restrict__ first, const int* __restrict__ last,
                         int n, int4* rec, int4* AP) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int f = first[v], l = last[v];
    rec[v] = make_int4(f, l, parent[v], 0);
    AP[f] = make_int4(f, f, v, l);
    AP[l] = make_int4(kINF, -1, ~v, f);
  }
}

// ---------------------------------------------------------------------------
// extract_bccs: blocks as sorted vertex sets, ordered by label
// ---------------------------------------------------------------------------
__global__ void k_block_keys(const int* __restrict__ label, const int* __restrict__ head, int n,
                             unsigned long long* keys, int* cnt) {
  pdl_enter();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int l = label[v];
    bool member = head[l] != -1;
    keys[2 * (int64_t)v] = member ? (((unsigned long long)(unsigned)l << 32) | (unsigned)v) : ~0ull;
    // one extra key per block: its head, inserted in sorted position
    int h = head[v];
    bool is_label = (label[v] == v) && h != -1;
    keys[2 * (int64_t)v + 1] = is_label ? (((unsigned long long)(unsigned)v << 32) | (unsigned)h) : ~0ull;
    (void)cnt;
  }
}

__global__ void k_block_bounds(const unsigned long long* __restrict__ keys, int64_t K, int* vtx, int* flags) {
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = keys[j];
    bool valid = k != ~0ull;
    vtx[j] = valid ? (int)(k & 0xffffffffull) : -1;
    flags[j] = valid && (j == 0 || (keys[j - 1] >> 32) != (k >> 32)) ? 1 : 0;
  }
}

__global__ void k_block_offsets(const int* __restrict__ flags, const int* __restrict__ fscan, int64_t K,
                                const unsigned long long* __restrict__ keys, int* boff, Scalars* sc) {
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
    if (flags[j]) boff[fscan[j]] = (int)j;
    if (keys[j] != ~0ull && (j + 1 == K || keys[j + 1] == ~0ull)) {  // last valid key
      int nb = fscan[j] + flags[j];
      boff[nb] = (int)(j + 1);
      sc->nbccs = nb;
    }
  }
}

// ---------------------------------------------------------------------------
// symmetrize: edge list -> sorted, deduplicated, self-loop-free CSR
// ---------------------------------------------------------------------------
__global__ void k_sym_keys(const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t k, int64_t n,
                           unsigned long long* keys, Scalars* sc) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[i], b = v[i];
    if (a < 0 || a >= n || b < 0 || b >= n) { raise_err(sc, E_RANGE); a = b = 0; }
    bool loop = a == b;
    keys[2 * i] = loop ? ~0ull : (((unsigned long long)a << 32) | (unsigned long long)b);
    keys[2 * i + 1] = loop ? ~0ull : (((unsigned long long)b << 32) | (unsigned long long)a);
  }
}

__global__ void k_sym_csr(const unsigned long long* __restrict__ ukeys, const int* __restrict__ nuniq, int64_t n,
                          int64_t* off, uint32_t* edges, Scalars* sc) {
  pdl_enter();
  int64_t m = *nuniq;
  if (m > 0 && ukeys[m - 1] == ~0ull) m--;  // the self-loop sentinel sorts last
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x) {
    // off[v] = first key with source >= v
    unsigned long long target = (unsigned long long)v << 32;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
    }
    off[v] = lo;
  }
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    edges[j] = (uint32_t)(ukeys[j] & 0xffffffffull);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->num_edges = (int)(m / 2);
}

size_t op_symmetrize_bytes(int64_t k) {
  size_t sort_bytes = 0, uniq_bytes = 0;
  int64_t K = 2 * k;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                 (int)K);
  cub::DeviceSelect::Unique(nullptr, uniq_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                            (int*)nullptr, (int)K);
  return 3 * 8 * (size_t)(K + 64) + (sort_bytes > uniq_bytes ? sort_bytes : uniq_bytes) + 1024;
}

int op_symmetrize(const int64_t* u, const int64_t* v, int64_t k, int64_t n, int64_t* off, uint32_t* edges,
                  void* ws, Scalars* sc, cudaStream_t st) {
  const int B = 256;
  int64_t K = 2 * k;
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { void* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  unsigned long long* a = (unsigned long long*)take(8 * (K + 1));
  unsigned long long* b = (unsigned long long*)take(8 * (K + 1));
  int* nuniq = (int*)take(64);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, a, b, (int)K);
  size_t ub = 0;
  cub::DeviceSelect::Unique(nullptr, ub, b, a, nuniq, (int)K);
  if (ub > tmp_bytes) tmp_bytes = ub;
  void* tmp = take(tmp_bytes);
  cudaMemsetAsync(nuniq, 0, 64, st);
  if (K > 0) {
    launch(k_sym_keys, grid_for(k, B), B, 0, st, u, v, k, n, a, sc);
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int)K, 0, 64, st);
    cub::DeviceSelect::Unique(tmp, tmp_bytes, b, a, nuniq, (int)K, st);
  }
  launch(k_sym_csr, grid_for(n + 1, B), B, 0, st, a, nuniq, n, off, edges, sc);
  return 0;
}

size_t op_extract_bytes(int64_t n) {
  size_t sort_bytes = 0, scan_bytes = 0;
  int64_t K = 2 * n;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                 (int)K);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int*)nullptr, (int*)nullptr, (int)K);
  return 2 * 8 * (size_t)(K + 64) + 2 * 4 * (size_t)(K + 64) + (sort_bytes > scan_bytes ? sort_bytes : scan_bytes) +
         1024;
}

// block_vtx gets up to 2n entries, block_off up to n+1
int op_extract_bccs(const int* label, const int* head, int64_t n, int* block_off, int* block_vtx, void* ws,
                    Scalars* sc, cudaStream_t st) {
  const int B = 256;
  int64_t K = 2 * n;
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { void* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  unsigned long long* a = (unsigned long long*)take(8 * K);
  unsigned long long* b = (unsigned long long*)take(8 * K);
  int* flags = (int*)take(4 * K);
  int* fscan = (int*)take(4 * K);
  size_t tmp_bytes = 0, sb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, a, b, (int)K);
  cub::DeviceScan::ExclusiveSum(nullptr, sb, flags, fscan, (int)K);
  if (sb > tmp_bytes) tmp_bytes = sb;
  void* tmp = take(tmp_bytes);
  if (K == 0) return 0;
  launch(k_block_keys, grid_for(n, B), B, 0, st, label, head, (int)n, a, nullptr);
  cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, a, b, (int)K, 0, 64, st);
  launch(k_block_bounds, grid_for(K, B), B, 0, st, b, K, block_vtx, flags);
  size_t sbytes = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, sbytes, flags, fscan, (int)K, st);
  launch(k_block_offsets, grid_for(K, B), B, 0, st, flags, fscan, K, b, block_off, sc);
  return 0;
}

// ---------------------------------------------------------------------------
// shared scratch for the graph-shaped ops: carve a Rooting / Tags from ws
// ---------------------------------------------------------------------------
struct OpSpace {
  size_t total = 0;
  size_t take(size_t bytes) {
    size_t at = total;
    total += (bytes + 255) & ~size_t(255);
    return at;
  }
};

int op_build_euler_tour(int64_t n, const int2* pairs, int64_t k, const int* labels, int* parent, int* first,
                        int* last, void* ws, size_t ws_bytes, Scalars* sc, cudaStream_t st, bool dry,
                        size_t* need) {
  const int B = 256;
  OpSpace L;
  const int64_t N0 = 2 * n;
  size_t o_comp = L.take(4 * n), o_fe = L.take(8 * n), o_flags = L.take(4 * (n + 1)), o_nrank = L.take(4 * (n + 1));
  size_t o_rootidx = L.take(8 * (n + 1)), o_rlist = L.take(4 * n), o_lhead = L.take(4 * n),
         o_nexto = L.take(4 * N0), o_nxt = L.take(4 * N0), o_own0 = L.take(8 * N0), o_rank0 = L.take(4 * N0),
         o_rec = L.take(16 * n), o_ap = L.take(16 * (size_t)(N0 + kTile));
  size_t o_keys = L.take(8 * 2 * k + 8), o_keys2 = L.take(8 * 2 * k + 8), o_vals = L.take(4 * 2 * k + 4),
         o_vals2 = L.take(4 * 2 * k + 4);
  // ranking levels
  int64_t K[8] = {0};
  int S[8] = {0};
  int nlev = 1;
  S[0] = opt(OPT_S0);
  K[1] = (N0 + S[0] - 1) / S[0];
  while (K[nlev] > kFinalMax) {
    S[nlev] = opt(OPT_SL);
    K[nlev + 1] = (K[nlev] + S[nlev] - 1) / S[nlev];
    nlev++;
  }
  size_t o_lev[8][4];
  for (int l = 1; l <= nlev; l++)
    for (int j = 0; j < 4; j++) o_lev[l][j] = L.take((j == 2 ? 8 : 4) * K[l]);
  size_t scan_b = std::max(scan_temp_bytes(n + 1), scan_roots_temp_bytes(n + 1)), sort_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (int*)nullptr, (int*)nullptr, (int)(2 * k));
  size_t o_tmp = L.take(scan_b > sort_b ? scan_b : sort_b);
  if (dry) {
    *need = L.total;
    return 0;
  }
  if (ws_bytes < L.total) return -1;
  char* w = (char*)ws;
  auto at = [&](size_t o) { return (void*)(w + o); };
  int* comp = (int*)at(o_comp);
  int2* fe = (int2*)at(o_fe);
  Rooting R;
  R.flags = (int*)at(o_flags);
  R.rootidx = (unsigned long long*)at(o_rootidx);
  R.rlist = (int*)at(o_rlist);
  R.lhead = (int*)at(o_lhead);
  R.hsub = nullptr;  // pairs input: no CSR, no hub split
  R.hoff = nullptr;
  R.nexto = (int*)at(o_nexto);
  R.nxt = (int*)at(o_nxt);
  R.own0 = (int2*)at(o_own0);
  R.rank0 = (int*)at(o_rank0);
  R.rec = (int4*)at(o_rec);
  R.nlev = nlev;
  for (int l = 0; l < 8; l++) {
    R.K[l] = K[l];
    R.S[l] = S[l];
    R.succ[l] = R.wgt[l] = R.offs[l] = nullptr;
    R.own[l] = nullptr;
  }
  for (int l = 1; l <= nlev; l++) {
    R.succ[l] = (int*)at(o_lev[l][0]);
    R.wgt[l] = (int*)at(o_lev[l][1]);
    R.own[l] = (int2*)at(o_lev[l][2]);
    R.offs[l] = (int*)at(o_lev[l][3]);
  }
  R.cub_tmp = at(o_tmp);
  R.cub_bytes = scan_b > sort_b ? scan_b : sort_b;
  int4* AP = (int4*)at(o_ap);
  int* nrank = (int*)at(o_nrank);
  unsigned long long* keys = (unsigned long long*)at(o_keys);
  unsigned long long* keys2 = (unsigned long long*)at(o_keys2);
  int* vals = (int*)at(o_vals);
  int* vals2 = (int*)at(o_vals2);

  const int gv = grid_for(n + 1, B);
  if (k > 0) launch(k_pairs_check, grid_for(k, B), B, 0, st, pairs, k, (int)n, sc);
  if (labels) {
    cudaMemcpyAsync(comp, labels, 4 * n, cudaMemcpyDeviceToDevice, st);
  } else {
    launch(k_iota2, gv, B, 0, st, comp, (int)n);
    if (k > 0) launch(k_union_pairs, grid_for(k, B), B, 0, st, pairs, k, (int)n, comp, sc);
    launch(k_flatten, gv, B, 0, st, comp, (int)n);
  }
  // pair i -> i-th non-root vertex
  launch(k_nonroot_flags, gv, B, 0, st, comp, (int)n, R.flags);
  exclusive_scan(R.flags, nrank, n + 1, R.cub_tmp, R.cub_bytes, st);
  rooting_roots((int)n, comp, R, sc, st);  // rootidx, rlist, c; clears lhead
  if (k > 0) {
    launch(k_place_pairs, gv, B, 0, st, pairs, k, comp, nrank, (int)n, fe, keys, vals, sc);
    size_t sb = R.cub_bytes;
    cub::DeviceRadixSort::SortPairs(R.cub_tmp, sb, keys, keys2, vals, vals2, (int)(2 * k), 0, 64, st);
    launch(k_sorted_lists, grid_for(2 * k, B), B, 0, st, keys2, vals2, 2 * k, R.lhead, R.nexto);
  }
  launch(k_check_rooted, gv, B, 0, st, comp, R.lhead, (int)n, nrank, k, sc);
  rooting_tour((int)n, comp, fe, R, AP, sc, st);
  launch(k_export_forest, gv, B, 0, st, R.rec, (int)n, parent, first, last);
  return 0;
}

int op_compute_tags(const Graph& g, const int* parent, const int* first, const int* last, int* w1, int* w2, int* low,
                    int* high, void* ws, size_t ws_bytes, cudaStream_t st, bool dry, size_t* need) {
  const int B = 256;
  const int64_t n = g.n;
  OpSpace L;
  int ntile = (int)((2 * n + kTile - 1) / kTile);
  if (ntile < 1) ntile = 1;
  int tlev = 1;
  while ((1 << tlev) <= ntile) tlev++;
  size_t o_rec = L.take(16 * n), o_ap = L.take(16 * (size_t)ntile * kTile), o_lh1 = L.take(8 * n),
         o_lh2 = L.take(8 * n), o_table = L.take(8 * (size_t)ntile * tlev), o_scr = L.take(3 * 4 * n),
         o_crow = L.take(4 * ((g.m + kItems - 1) / kItems + 1)), o_sc = L.take(sizeof(Scalars));
  if (dry) {
    *need = L.total;
    return 0;
  }
  if (ws_bytes < L.total) return -1;
  char* w = (char*)ws;
  auto at = [&](size_t o) { return (void*)(w + o); };
  Graph gg = g;
  gg.crow = (const int*)at(o_crow);
  build_chunk_rows(gg, (int*)at(o_crow), (Scalars*)at(o_sc), st);  // (hub flag unused here)
  Rooting R{};
  R.rec = (int4*)at(o_rec);
  Tags T;
  T.AP = (int4*)at(o_ap);
  T.lh1 = (int2*)at(o_lh1);
  T.lh2 = (int2*)at(o_lh2);
  T.table = (int2*)at(o_table);
  T.ntile = ntile;
  T.tlev = tlev;
  int* scr = (int*)at(o_scr);
  launch(k_rec_ap, grid_for(n, B), B, 0, st, parent, first, last, (int)n, R.rec, T.AP);
  stage3_tags(gg, R, T, st, /*nlow=*/nullptr);
  stage4_fence(gg, R, T, low, high, scr, scr + n, scr + 2 * n, st);
  export_debug(gg, nullptr, R.rec, T.AP, nullptr, nullptr, nullptr, nullptr, w1, w2, nullptr, st);
  return 0;
}

}  // namespace fbcc

// ---------------------------------------------------------------------------
// classify_edge (bcc.py:54-70) for every slot, against a given rooted forest
// and its tags: one thread per 8-arc chunk (its row by binary search over the
// offsets, then galloping), EdgeClass codes PLAIN_TREE 0, FENCE_TREE 1,
// BACK 2, CROSS 3 (bcc.py:45-51).
// ---------------------------------------------------------------------------
namespace fbcc {

__global__ void k_classify(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, int n, int64_t m,
                           const int* __restrict__ parent, const int* __restrict__ first,
                           const int* __restrict__ last, const int* __restrict__ low, const int* __restrict__ high,
                           int8_t* __restrict__ cls, Scalars* sc) {
  pdl_enter();
  const int64_t nchunks = (m + kItems - 1) / kItems;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nchunks; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = q * kItems, a1 = a0 + kItems < m ? a0 + kItems : m;
    int u = row_of(off, 0, n - 1, a0);
    int64_t re = __ldg(off + u + 1);
    for (int64_t a = a0; a < a1; a++) {
      if (a >= re) {
        u = next_row(off, u, n, a);
        re = __ldg(off + u + 1);
      }
      const int v = (int)__ldg(adj + a);
      if (v < 0 || v >= n) {
        atomicOr(&sc->err, 1);
        cls[a] = -1;
        continue;
      }
      const int pu = __ldg(parent + u), pv = __ldg(parent + v);
      int8_t c;
      if (pv == u || pu == v) {  // tree edge (bcc.py:61-66)
        const int ch = pv == u ? v : u, pa = pv == u ? u : v;
        c = (__ldg(low + ch) >= __ldg(first + pa) && __ldg(high + ch) <= __ldg(last + pa)) ? 1 : 0;
      } else {
        const int fu = __ldg(first + u), lu = __ldg(last + u), fv = __ldg(first + v), lv = __ldg(last + v);
        c = ((fu <= fv && lv <= lu) || (fv <= fu && lu <= lv)) ? 2 : 3;  // back / cross (bcc.py:67-70)
      }
      cls[a] = c;
    }
  }
}

int op_classify_edges(const Graph& g, const int* parent, const int* first, const int* last, const int* low,
                      const int* high, int8_t* cls, Scalars* sc, cudaStream_t st) {
  if (g.m == 0) return 0;
  launch(k_classify, grid_for((g.m + kItems - 1) / kItems, 256), 256, 0, st, g.off, g.adj, g.n, g.m, parent, first,
         last, low, high, cls, sc);
  return 0;
}

}  // namespace fbcc
