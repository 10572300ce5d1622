// kernels.cuh -- stage entry points shared between the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace fbcc {

struct Graph {
  const int64_t* off;    // [n+1] reference layout (graphs.py:43-58)
  const uint32_t* adj;   // [m]
  int n;
  int64_t m;
  const int* crow;       // [ceil(m/kItems)] chunk -> row table (build_chunk_rows)
};

// int32 offsets [n+1] (uploaded from the host) -> the int64 device CSR offsets
void widen_offsets(const int* src, int64_t* dst, int64_t n, cudaStream_t st);

// (comp/fe/prop given: also Stage 1's sampling round 0; returns whether it ran)
// (nlow given: also zeroes Stage 3's lower-degree counters, coalesced)
bool build_chunk_rows(const Graph& g, int* crow, Scalars* sc, cudaStream_t st, int* comp = nullptr,
                      int2* fe = nullptr, unsigned long long* prop = nullptr, int* nlow = nullptr, int* w0 = nullptr);

// (host path: the first three arcs of every row, once the edge array has landed)
void record_arcs(const Graph& g, int* w0, cudaStream_t st);

// Stage 2 initial state written by Stage 1's final compress (one pass over
// the vertices instead of a separate k_root_flags): flags[v] = v is a root
// (flags[n] = 0, the scan's tail), lhead[v] = empty out-list (-1) or the hub
// sub-list marker, hub sub-list heads cleared (see rooting.cu).
struct RootInit {
  int* flags = nullptr;
  int* lhead = nullptr;
  int* hsub = nullptr;
  const int64_t* off = nullptr;  // hub split source (nullptr: none)
  const Scalars* sc = nullptr;
  bool detach = false;           // isolated vertices (but 0) stay off the Euler tour (code 2)
  // the same compress also ranks the roots inside each of its 1024-vertex
  // tiles (Rooting::rootidx at the roots) and counts each tile's roots
  // (tile_roots); k_scan_tiles and k_out_lists finish the exclusive scan
  unsigned long long* rootidx = nullptr;
  unsigned long long* sdesc = nullptr;  // [ceil(n / 1024)] tile root counts: detached << 32 | listed
};

// Root codes (Rooting::flags): 0 non-root, 1 root on the tour list, 2 root
// kept off the list -- an isolated vertex other than 0, whose positions
// follow the list's (k_positions).  RMAT s25: 16.5 M of the 33.5 M vertices.
__device__ __forceinline__ int root_init(const RootInit& ri, const int64_t* hoff, int v, bool root) {
  const int code = root ? ((ri.detach && v != 0 && __ldg(ri.off + v + 1) == __ldg(ri.off + v)) ? 2 : 1) : 0;
  ri.flags[v] = code;
  int h = -1;
  if (hoff) {
    const int64_t rs = __ldg(hoff + v);
    if (__ldg(hoff + v + 1) - rs >= kHubDeg) {
      const int base = (int)(rs >> 4);
      const int lw = hub_log_ways(__ldg(hoff + v + 1) - rs);
      for (int j = 0; j < (1 << lw); j++) ri.hsub[base + j] = -1;
      h = hub_marker(base, lw);
    }
  }
  ri.lhead[v] = h;
  return code;
}

// Device arrays for the rooting / tags stages (see api.cu for the layout).
#ifndef FBCC_FINAL_MAX
#define FBCC_FINAL_MAX 16384
#endif
constexpr int kFinalMax = FBCC_FINAL_MAX;  // list-ranking level finished in one CTA

struct Rooting {
  int* flags;      // [n+1] root code (root_init): 0 non-root, 1 listed root, 2 detached
  unsigned long long* rootidx;  // [n+1] exclusive scan: low 32 bits listed roots before v, high 32 detached ones
  unsigned long long* tile_roots = nullptr;  // the pipeline: Stage 1's final compress ranked the roots inside its
                                             // 1024-vertex tiles (RootInit::rootidx / sdesc); [tiles] root counts
  int* rlist;      // [n]   listed roots in id order
  int* lhead;      // [n]   first out-arc of each vertex (-1: none; <= -2: hub, see rooting.cu)
  int* hsub;       // [m/16 + 64] hub sub-list heads (nullptr: no hub split)
  const int64_t* hoff;  // CSR offsets the hubs are chosen from (nullptr: no hub split)
  int* nexto;      // [2n]  next out-arc of the same vertex
  int* nxt;        // (unused: level 0's successors live in own0[e].x until the walk replaces them)
  int2* own0;      // [2n]  per list element: (successor, 0) from k_link_tour, then (segment, offset)
  int* rank0;      // [2n]  tour position of each list element
  // ruling-set levels 1..nlev: element counts and arrays
  int nlev;
  int64_t K[8];
  int S[8];        // splitter spacing used to build level l+1 from level l
  int* succ[8];
  int* wgt[8];
  int2* own[8];
  int* offs[8];
  int4* rec;       // [n] {first, last, parent, fence}
  int* firsts = nullptr;  // pipeline: k_positions also writes Stage 3's compact first[] ...
  int* nlow = nullptr;    // ... and k_chunk_rows zeroed these counters (no k_firsts pass)
  void* cub_tmp;
  size_t cub_bytes;
};

struct Tags {
  int4* AP;        // [ntile*TILE] per tour position: {w1, w2, v or ~v, partner position};
                   // (w1, w2) at first[v], filler at last[v]
  int2* lh1;       // [n] in-tile result / suffix partial
  int2* lh2;       // [n] prefix partial
  int2* table;     // [tlev * ntile] sparse table over tile extremes
  int ntile;
  int tlev;
  const int* tour_len = nullptr;  // device count of list positions (pipeline: Scalars::tour_len); nullptr: 2n
};

#ifndef FBCC_TILE
#define FBCC_TILE 4096
#endif
constexpr int kTile = FBCC_TILE;  // tour positions per tile in the low/high pass

void rooting_roots(int n, const int* comp, Rooting& R, Scalars* sc, cudaStream_t st);
void rooting_tour(int n, const int* comp, const int2* fe, Rooting& R, int4* AP, Scalars* sc, cudaStream_t st);
void masked_cc(const Graph& g, const uint8_t* mask, int* comp, int2* fe, unsigned long long* prop, Scalars* sc,
               cudaStream_t st);
// (warc: [3][n] targets of each row's arcs 0-2 recorded by k_chunk_rows, or nullptr)
void stage1_forest(const Graph& g, int* comp, int2* fe, unsigned long long* prop, Scalars* sc, cudaStream_t st,
                   bool round0_done = false, RootInit ri = RootInit{}, const int* warc = nullptr,
                   int* jlist = nullptr);  // (jlist: >= 2^18 ints of scratch for k_jump_local's exit list)
// Stage 1 over a streamed edge array (fbcc_run_host): identity init, one link
// pass per arrived chunk range [q0, q1) of kItems-arc chunks, final compress
void stage1_stream_begin(const Graph& g, int* comp, cudaStream_t st);
void stage1_stream_range(const Graph& g, int64_t q0, int64_t q1, int* comp, int2* fe, cudaStream_t st);
void stage1_stream_finish(const Graph& g, int* comp, Scalars* sc, cudaStream_t st, RootInit ri = RootInit{});

void stage2_rooting(const Graph& g, const int* comp, const int2* fe, Rooting& R, int4* AP,
                    Scalars* sc, cudaStream_t st);
// the pipeline's Stage 2 after a RootInit compress: scan of the flags, then
// out-lists (which also place the roots in id order) and the tour
void stage2_rooting_fused(const Graph& g, const int* comp, const int2* fe, Rooting& R, int4* AP, Scalars* sc,
                          cudaStream_t st);
// nlow == nullptr: the reference's exact w2 (both forest directions
// excluded, stand-alone op); otherwise the pipeline's relaxed gather (same
// w1/low/high), which also counts each row's lower neighbours into nlow
// A second stream for the two Stage-6 pieces that do not depend on the
// stages in between: the upper-degree scan (needs only Stage 3's nlow) runs
// beside Stages 3-5, the articulation flags beside the edge pass.  Fork/join
// by events (captured into the plan's graph as edges).
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[4] = {};  // fork scan, join scan, fork ap, join ap
};

// Witness plans (tags.cu): Stage 3 from each row's first three arcs, the open
// fence bits repaired exactly; the full gather only if the repair overflows
struct Witness {
  bool on = false;
  const int* w0 = nullptr;        // [3][n] arcs 0-2 of every row (k_chunk_rows)
  int* und_list = nullptr;        // [cap] vertices to repair (a dead Stage-2 array)
  int cap = 0;
  unsigned long long work = 0;    // tour positions the repair may walk in all
  int* firsts = nullptr;          // [n] compact first[] of the overflow redo (built only then)
  bool crow_built = true;         // the chunk -> row table exists (else the overflow redo searches the offsets)
};

void stage3_tags(const Graph& g, const Rooting& R, Tags& T, cudaStream_t st, int* nlow, const Side* side = nullptr,
                 int* uoff = nullptr, void* cub_tmp = nullptr, size_t cub_bytes = 0, Scalars* sc = nullptr,
                 const Witness* W = nullptr);
// (label5 / prop5: also Stage 5's sampling round 0 along plain parent edges -- comp = the parent when the
// tree edge is no fence and the parent's id is smaller -- and the proposal reset; needs sc)
void stage4_fence(const Graph& g, const Rooting& R, Tags& T, int* low_out, int* high_out, int* head, int* cnt,
                  int* bmin, cudaStream_t st, Scalars* sc = nullptr, const Witness* W = nullptr, int* label5 = nullptr,
                  unsigned long long* prop5 = nullptr, bool s5_if_ordered = false);  // (... only on id-ordered forests)
void compute_nlow(const Graph& g, int* nlow, cudaStream_t st);
// (w0: [3][n] each row's first three arc targets, recorded by k_chunk_rows' round 0; nullptr: read adj)
// (round0_done: stage4_fence wrote Stage 5's round 0 -- label5 / prop5 given; jlist: scratch for the
// id-ordered compress, see stage1_forest)
void stage5_skeleton_cc(const Graph& g, const int4* rec, int* label, unsigned long long* prop, Scalars* sc,
                        cudaStream_t st, const int* w0 = nullptr, bool round0_done = false, int* jlist = nullptr,
                        bool round0_if_ordered = false);  // (... k_hook_min runs unless the forest is id-ordered)
void stage6_labelling(const Graph& g, const int4* rec, const int* label, int* head, uint8_t* is_ap,
                      int* edge_label, int* cnt, int* uoff, int* nlow, int* bmin, int* heavy, int* sreq, int* spos,
                      void* cub_tmp, size_t cub_bytes, Scalars* sc, cudaStream_t st,
                      cudaEvent_t heads_done = nullptr, const Side* side = nullptr);
void export_debug(const Graph& g, const int2* fe, const int4* rec, const int4* AP, int* forest,
                  int* parent, int* first, int* last, int* w1, int* w2, uint8_t* fence,
                  cudaStream_t st, const int* tour_len = nullptr);

// Edge ids.  scan_upper_degrees leaves each vertex's prefix inside its kUpTile-vertex tile in uoff and
// the tile prefixes (then the total, E) in its scratch buffer; Stage 6 adds the two as it reads them
// (UpOff::at) -- no pass over the vertices to add them in.
constexpr int kUpTile = 1024;
struct UpOff {
  const int* loc;                   // [n] prefix inside the tile
  const unsigned long long* tpre;  // [tiles + 1] tile prefixes, then the total
  int n, ntiles;
  __device__ __forceinline__ int at(int v) const {  // upper arcs of the rows before v; v == n: E
    return v < n ? __ldg(loc + v) + (int)__ldg(tpre + v / kUpTile) : (int)__ldg(tpre + ntiles);
  }
};

size_t scan_temp_bytes(int64_t items);
// uoff[v] = sum over u < v of (deg(u) - nlow[u]), v in [0, n] (uoff[n] = E)
size_t scan_upper_temp_bytes(int n);
void scan_upper_degrees(const int64_t* off, const int* nlow, int n, int* uoff, void* tmp, size_t tmp_bytes,
                        cudaStream_t st);
void exclusive_scan(const int* in, int* out, int64_t items, void* tmp, size_t tmp_bytes,
                    cudaStream_t st);
// rootidx from the root codes (items = n + 1)
size_t scan_roots_temp_bytes(int64_t items);
void scan_roots(const int* flags, unsigned long long* out, int64_t items, void* tmp, size_t tmp_bytes,
                cudaStream_t st);

}  // namespace fbcc
