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
//  * Tree CSR: one atomicAdd per endpoint returns the arc's rank inside its
//    row, so after a CUB scan the scatter needs no second atomic pass.
//  * ONE list for the whole forest.  Every root r contributes two virtual
//    elements, enter(r) = 2*ri and exit(r) = 2*ri+1 (ri = rank of r among
//    roots); tree arc slot t is element 2c+t.  enter(r) -> r's first out-arc
//    ... -> the in-arc that closes r's circuit -> exit(r) -> enter(next root).
//    The list has exactly 2n elements, its head is element 0, and an
//    element's rank IS its tour position in the reference layout (tree of
//    root r owns [base_r, base_r + 2 size_r), root at both ends, trees in
//    root-id order, euler_tour.py:12-17).  No per-tree base scan, no list
//    heads beyond element 0.
//  * Ruling-set list ranking: splitters are one hash-chosen element per
//    window of S consecutive ids (so structured tours, e.g. a chain whose
//    return path only touches odd ids, are still cut), the splitter index is
//    the window index (no compaction), each splitter walks to the next one
//    writing (segment, offset) per element; recurse on the weighted splitter
//    list until it fits one CTA, which finishes with Wyllie pointer jumping
//    in shared memory.  Offsets are pushed back down level by level; level 0
//    ranks are never materialised -- the positions kernel computes
//    rank(e) = offs1[own0[e].seg] + own0[e].off on the fly.
//  * Positions: one thread per forest edge compares the ranks of its two
//    arcs: the earlier one is the down arc, giving parent, first and last of
//    the child in one shot (no per-vertex loop over tree degree, so hub
//    vertices cost nothing extra).  It also initialises the tour-indexed
//    arrays the tag stage reads (A: (first, first) at entry, filler at exit;
//    P: vertex id + partner position).
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

constexpr int kFinalMax = 4096;

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

// ---------------------------------------------------------------------------
// tree CSR
// ---------------------------------------------------------------------------
__global__ void k_root_flags(const int* __restrict__ comp, int n, int* __restrict__ flags) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += gridDim.x * blockDim.x)
    flags[v] = (v < n) ? (__ldg(comp + v) == v) : 0;
}

__global__ void k_tree_degree(const int* __restrict__ comp, const int2* __restrict__ fe, int n, int* tdeg,
                              int4* __restrict__ ex, const int* __restrict__ rootidx, Scalars* sc) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) sc->ncomp = rootidx[n];
  for (int x = (int)tid; x < n; x += gridDim.x * blockDim.x) {
    if (__ldg(comp + x) == x) continue;
    int2 e = fe[x];
    int lu = atomicAdd(tdeg + e.x, 1);
    int lv = atomicAdd(tdeg + e.y, 1);
    ex[x] = make_int4(e.x, e.y, lu, lv);
  }
}

__global__ void k_tree_scatter(const int* __restrict__ comp, int n, const int* __restrict__ toff,
                               int4* __restrict__ ex, int* __restrict__ tedges, int* __restrict__ twin) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    if (__ldg(comp + x) == x) continue;
    int4 e = ex[x];
    int su = __ldg(toff + e.x) + e.z;
    int sv = __ldg(toff + e.y) + e.w;
    tedges[su] = e.y;
    tedges[sv] = e.x;
    twin[su] = sv;
    twin[sv] = su;
    ex[x] = make_int4(e.x, e.y, su, sv);
  }
}

// Unified tour list.  Arc slot t (element 2c+t) arrives at v = tedges[t];
// its twin is v's out-slot i; the tour continues with v's out-slot i+1, or,
// after v's last out-slot, with v's first out-slot (non-root: closes the
// circuit around v) or exit(v) (root: the tour of v's tree is complete).
__global__ void k_link_slots(const int* __restrict__ comp, const int* __restrict__ toff,
                             const int* __restrict__ tedges, const int* __restrict__ twin,
                             const int* __restrict__ rootidx, int n, int* __restrict__ nxt,
                             const Scalars* sc) {
  const int c = sc->ncomp;
  const int L = 2 * (n - c);
  const int c2 = 2 * c;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < L; t += gridDim.x * blockDim.x) {
    int v = __ldg(tedges + t);
    int s = __ldg(twin + t);
    int b = __ldg(toff + v);
    int k = __ldg(toff + v + 1) - b;
    int i = s - b;
    int e;
    if (i + 1 < k) e = c2 + b + i + 1;
    else if (__ldg(comp + v) == v) e = 2 * __ldg(rootidx + v) + 1;
    else e = c2 + b;
    nxt[c2 + t] = e;
  }
}

__global__ void k_link_roots(const int* __restrict__ comp, const int* __restrict__ toff,
                             const int* __restrict__ rootidx, int n, int* __restrict__ nxt,
                             const Scalars* sc) {
  const int c = sc->ncomp;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (__ldg(comp + r) != r) continue;
    int ri = __ldg(rootidx + r);
    int b = __ldg(toff + r);
    int k = __ldg(toff + r + 1) - b;
    nxt[2 * ri] = k > 0 ? 2 * c + b : 2 * ri + 1;
    nxt[2 * ri + 1] = (ri + 1 < c) ? 2 * ri + 2 : -1;
  }
}

// ---------------------------------------------------------------------------
// ruling-set list ranking
// ---------------------------------------------------------------------------
// splitter of window j (element j*S + hashed offset; window 0 uses element 0,
// the list head; the last, partial window is clamped into range)
__device__ __forceinline__ int64_t split_elem(int64_t j, int S, int64_t N) {
  int64_t e = j * S + (j == 0 ? 0 : (hash32((uint32_t)j * 0x9E3779B1u + 0x7F4A7C15u) & (S - 1)));
  return e < N ? e : N - 1;
}

template <bool kWeighted>
__global__ void __launch_bounds__(256) k_walk(int64_t K, int S, int64_t N, const int* __restrict__ succ,
                                              const int* __restrict__ w, int2* __restrict__ own,
                                              int* __restrict__ succ_next, int* __restrict__ w_next) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = split_elem(j, S, N);
    int acc = 0;
    int nj = -1;
    while (true) {
      own[e] = make_int2((int)j, acc);
      acc += kWeighted ? __ldg(w + e) : 1;
      int e2 = __ldg(succ + e);
      if (e2 < 0) break;
      int64_t j2 = e2 / S;
      if (split_elem(j2, S, N) == e2) { nj = (int)j2; break; }
      e = e2;
    }
    succ_next[j] = nj;
    w_next[j] = acc;
  }
}

// Final level: <= kFinalMax elements, head = element 0; exclusive weighted
// prefix along the list by Wyllie pointer jumping over predecessor links,
// entirely in shared memory (one CTA).
__global__ void __launch_bounds__(1024) k_final_rank(int K, const int* __restrict__ succ,
                                                     const int* __restrict__ w, int* __restrict__ offs) {
  __shared__ int P[kFinalMax];
  __shared__ int V[kFinalMax];
  const int t = threadIdx.x;
  for (int j = t; j < K; j += 1024) P[j] = -1;
  __syncthreads();
  for (int j = t; j < K; j += 1024) {
    int s = succ[j];
    if (s >= 0) P[s] = j;
  }
  __syncthreads();
  for (int j = t; j < K; j += 1024) V[j] = P[j] >= 0 ? w[P[j]] : 0;
  __syncthreads();
  constexpr int PER = kFinalMax / 1024;
  for (int round = 0; round < 13; round++) {
    int np[PER], nv[PER];
    int active = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
      int j = t + q * 1024;
      np[q] = -1;
      nv[q] = 0;
      if (j < K) {
        int p = P[j];
        nv[q] = V[j];
        if (p >= 0) { nv[q] += V[p]; np[q] = P[p]; active = 1; }
      }
    }
    if (!__syncthreads_or(active)) break;
#pragma unroll
    for (int q = 0; q < PER; q++) {
      int j = t + q * 1024;
      if (j < K) { P[j] = np[q]; V[j] = nv[q]; }
    }
    __syncthreads();
  }
  for (int j = t; j < K; j += 1024) offs[j] = V[j];
}

__global__ void k_expand(int64_t K, const int2* __restrict__ own, const int* __restrict__ offs_up,
                         int* __restrict__ offs) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
    int2 o = own[j];
    offs[j] = __ldg(offs_up + o.x) + o.y;
  }
}

// ---------------------------------------------------------------------------
// positions: parent / first / last + tour-indexed tag arrays
// ---------------------------------------------------------------------------
__device__ __forceinline__ void place(int v, int f, int l, int par, int4* rec, int2* A, int2* P) {
  rec[v] = make_int4(f, l, par, 0);
  A[f] = make_int2(f, f);      // w1 = w2 = own entry position, gathered into by stage 3
  A[l] = make_int2(kINF, -1);  // neutral filler (tagging.py:33-39)
  P[f] = make_int2(v, l);
  P[l] = make_int2(~v, f);
}

__global__ void k_positions(const int* __restrict__ comp, const int4* __restrict__ ex,
                            const int* __restrict__ rootidx, const int2* __restrict__ own0,
                            const int* __restrict__ offs1, int n, int4* __restrict__ rec, int2* __restrict__ A,
                            int2* __restrict__ P, const Scalars* sc) {
  const int c2 = 2 * sc->ncomp;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    if (__ldg(comp + x) == x) {
      int ri = __ldg(rootidx + x);
      int2 o1 = own0[2 * ri], o2 = own0[2 * ri + 1];
      place(x, __ldg(offs1 + o1.x) + o1.y, __ldg(offs1 + o2.x) + o2.y, -1, rec, A, P);
    } else {
      int4 e = ex[x];
      int2 ou = own0[c2 + e.z], ov = own0[c2 + e.w];
      int ru = __ldg(offs1 + ou.x) + ou.y;
      int rv = __ldg(offs1 + ov.x) + ov.y;
      if (ru < rv) place(e.y, ru, rv, e.x, rec, A, P);  // u -> v is the down arc
      else place(e.x, rv, ru, e.y, rec, A, P);
    }
  }
}

void stage2_rooting(const Graph& g, const int* comp, const int2* fe, Rooting& R, int2* A, int2* P,
                    Scalars* sc, cudaStream_t st) {
  const int n = g.n;
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  // roots: rank among roots (ri) and c
  k_root_flags<<<gv, B, 0, st>>>(comp, n, R.rootidx + (n + 1));  // flags staged after rootidx
  note(K_ROOT_FLAGS);
  exclusive_scan(R.rootidx + (n + 1), R.rootidx, n + 1, R.cub_tmp, R.cub_bytes, st);
  note(K_SCAN);
  // tree CSR
  cudaMemsetAsync(R.tdeg, 0, sizeof(int) * (n + 1), st);
  note(K_MEMSET);
  k_tree_degree<<<gv, B, 0, st>>>(comp, fe, n, R.tdeg, R.ex, R.rootidx, sc);
  note(K_TREE_DEGREE);
  int* toff = R.tdeg + (n + 1);
  exclusive_scan(R.tdeg, toff, n + 1, R.cub_tmp, R.cub_bytes, st);
  note(K_SCAN);
  k_tree_scatter<<<gv, B, 0, st>>>(comp, n, toff, R.ex, R.tedges, R.twin);
  note(K_TREE_SCATTER);
  // unified list
  k_link_slots<<<grid_for(2 * (int64_t)n, B), B, 0, st>>>(comp, toff, R.tedges, R.twin, R.rootidx, n, R.nxt, sc);
  note(K_LINK_SLOTS);
  k_link_roots<<<gv, B, 0, st>>>(comp, toff, R.rootidx, n, R.nxt, sc);
  note(K_LINK_ROOTS);
  // ruling-set levels
  const int64_t N0 = 2 * (int64_t)n;
  k_walk<false><<<grid_for(R.K[1], B, 64), B, 0, st>>>(R.K[1], R.S[0], N0, R.nxt, nullptr, R.own0,
                                                       R.succ[1], R.wgt[1]);
  note(K_WALK0);
  for (int l = 1; l < R.nlev; l++) {
    k_walk<true><<<grid_for(R.K[l + 1], B, 64), B, 0, st>>>(R.K[l + 1], R.S[l], R.K[l], R.succ[l], R.wgt[l],
                                                            R.own[l], R.succ[l + 1], R.wgt[l + 1]);
    note(K_WALKL);
  }
  k_final_rank<<<1, 1024, 0, st>>>((int)R.K[R.nlev], R.succ[R.nlev], R.wgt[R.nlev], R.offs[R.nlev]);
  note(K_FINAL_RANK);
  for (int l = R.nlev - 1; l >= 1; l--) {
    k_expand<<<grid_for(R.K[l], B), B, 0, st>>>(R.K[l], R.own[l], R.offs[l + 1], R.offs[l]);
    note(K_EXPAND);
  }
  k_positions<<<gv, B, 0, st>>>(comp, R.ex, R.rootidx, R.own0, R.offs[1], n, R.rec, A, P, sc);
  note(K_POSITIONS);
}

}  // namespace fbcc
