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
__global__ void k_heads(int n, const int4* __restrict__ rec, const int* __restrict__ label, int* head, int* cnt,
                        Scalars* sc) {
  pdl_enter();
  int blocks = 0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int p = __ldg(&rec[v].z);
    if (p >= 0) {
      int l = __ldg(label + v);
      // (read first: the children of one head inside one component -- RMAT
      // hubs -- would otherwise serialise their CAS on one word)
      if (l != __ldg(label + p) && ld_relaxed(head + l) == -1 && atomicCAS(head + l, -1, p) == -1) {
        blocks++;
        if (ld_relaxed(cnt + p) < 2) atomicAdd(cnt + p, 1);
      }
    }
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
struct EdgeBlockVisitor {
  const int64_t* off;
  const int* label;
  const int* head;
  const int* uoff;
  const int* nlow;
  int* eblk;
  int* bmin;
  int lu, ebase;
  bool row_u0;
  int run_blk, run_min;
  int pl[kItems];
  // label[w] for every arc that can be an upper arc (w > first row of the chunk)
  __device__ __forceinline__ void prefetch(int v0, const uint32_t* w, int cnt) {
#pragma unroll
    for (int i = 0; i < kItems; i++) pl[i] = (i < cnt && (int)w[i] > v0) ? __ldg(label + w[i]) : -1;
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
    int lw = pl[i];
    bool mine;
    int blk;
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

__global__ void __launch_bounds__(256) k_edge_blocks(const int64_t* __restrict__ off, const uint32_t* __restrict__ adj, const int* __restrict__ crow,
                                                     int n, int64_t m, const int* __restrict__ label,
                                                     const int* __restrict__ head, const int* __restrict__ uoff,
                                                     const int* __restrict__ nlow, int* eblk, int* bmin) {
  pdl_enter();
  EdgeBlockVisitor vis;
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

__global__ void k_edge_final(int* eblk, const int* __restrict__ bmin, const int* __restrict__ uoff, int n) {
  pdl_enter();
  const int E = uoff[n];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    eblk[e] = __ldg(bmin + eblk[e]);
}

__global__ void k_set_edges(const int* __restrict__ uoff, int n, Scalars* sc) {
  pdl_enter(); sc->num_edges = uoff[n]; }

void stage6_labelling(const Graph& g, const int4* rec, const int* label, int* head, uint8_t* is_ap,
                      int* edge_label, int* cnt, int* uoff, int* nlow, int* bmin, void* cub_tmp,
                      size_t cub_bytes, Scalars* sc, cudaStream_t st, cudaEvent_t heads_done) {
  const int n = g.n;
  const int B = 256;
  const int gv = grid_for(n + 1, B);
  // head = -1, cnt = 0, bmin = INF were initialised by the stage-4 kernel
  launch(k_heads, gv, B, 0, st, n, rec, label, head, cnt, sc);
  note(K_HEADS);
  if (is_ap) {
    launch(k_ap, gv, B, 0, st, n, label, head, cnt, is_ap);
    note(K_AP);
  }
  if (heads_done) cudaEventRecord(heads_done, st);  // head / is_ap final: their D2H may start
  // edge ids: exclusive scan of the upper degrees deg - nlow (nlow counted
  // by the Stage-3 gather) -> uoff (uoff[n] = E)
  scan_upper_degrees(g.off, nlow, n, uoff, cub_tmp, cub_bytes, st);
  note(K_SCAN);
  launch(k_set_edges, 1, 1, 0, st, uoff, n, sc);
  note(K_SET_EDGES);
  if (edge_label && g.m > 0) {
    int64_t nchunks = (g.m + kItems - 1) / kItems;
    launch(k_edge_blocks, grid_for(nchunks, B, 32), B, 0, st, g.off, g.adj, g.crow, n, g.m, label, head, uoff, nlow,
                                                          edge_label, bmin);
    note(K_EDGE_BLOCKS);
    launch(k_edge_final, grid_for(g.m / 2, B), B, 0, st, edge_label, bmin, uoff, n);
    note(K_EDGE_FINAL);
  }
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
