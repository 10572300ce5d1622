// api.cu -- the C ABI (include/fastbcc_b200.h): workspace layout, the
// six-stage orchestration of fast_bcc (bcc.py:147-196) on one stream, and
// CUDA-graph plans that replay the whole launch sequence.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>

#include "../../include/fastbcc_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "ops.cuh"

namespace fbcc {

static thread_local char g_cuda_err[256] = "";
thread_local LaunchLog* g_log = nullptr;

static const char* kKernelNames[K_NUM_KINDS] = {
    "chunk_rows", "hook_min", "iota", "propose", "accept", "compress", "find_giant", "link_rows", "link_heavy",
    "root_flags", "scan", "root_list", "out_lists", "link_tour", "walk0", "walk_level", "final_rank", "expand", "rank0",
    "positions", "firsts", "w_gather", "tile", "table", "fence", "heads", "count_blocks", "ap", "set_edges",
    "edge_blocks", "edge_final", "memset", "export", "widen", "giant_min", "edge_fill", "edge_search", "jump_local",
    "jump_list", "scan_tiles", "w_sample", "witness_fix", "nlow"};

static int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", where, cudaGetErrorString(e));
  return FBCC_ERR_CUDA;
}

// process-wide defaults (fbcc_set_option; atomic: the setter may race an
// enqueue on another thread -- every enqueue works from its own snapshot)
static std::atomic<int> g_opt[OPT_NUM] = {/*sample rounds (always run)*/ 2, /*giant skip*/ 1, /*retired*/ 0, /*S0*/ 16, /*SL*/ 8,
                      /*retired*/ 0, 0, 0, /*compress after rounds mask: 0 = first+last; all rounds: 4b -13%, config 3 -2%*/ 0xFF,
                      /*retired*/ 0, /*retired*/ 0,
                      /*programmatic dependent launch (dependents launch as the previous grid exits)*/ 1,
                      /*fbcc_run_host edge-copy chunks (at most; one per 2^21 arcs)*/ 4, /*skeleton parent-edge rounds (bits 0, 1: rounds 0 and 1; 0x80: round 0 on parent edges only, inside Stage 4's pass)*/ 0x83,
                      /*giant pick folded into the last compress*/ 1,
                      /*warp-staged edge-block pass with the giant bitmap*/ 1,
                      /*... plus adaptive rounds up to (skip_round)*/ 3, /*Stage 5 cap (0: same)*/ 0,
                      /*accept folded into the following compress: 2 = auto (n >= 2^22; config 5 -1.3 %, 4b -4.3 %, config 2 +6 % if forced)*/ 2,
                      /*isolated vertices off the Euler-tour list and the tile pass*/ 1,
                      /*witness tags: 1 = plans with m >= 8n*/ 1};
thread_local const Options* t_opt = nullptr;

int option_default(int key) { return g_opt[key].load(std::memory_order_relaxed); }

Options options_snapshot() {
  Options o;
  for (int k = 0; k < OPT_NUM; k++) o.v[k] = g_opt[k].load(std::memory_order_relaxed);
  return o;
}

#ifndef FBCC_ROOT_SCAN_FUSED
#define FBCC_ROOT_SCAN_FUSED 1
#endif
constexpr int kFinalMaxHost = kFinalMax;
constexpr int kMaxStreamChunks = 64;

struct Layout {
  size_t total = 0;
  size_t sc, sdesc, sdesc_bytes, crow, comp, fe, prop, flags, rootidx, rlist, lhead, hsub, nexto, nxt, own0, rank0, rec, AP, lh1, lh2, table, cnt, uoff,
      nlow, bmin, w0, cub, wfirsts;
  bool witness = false;  // Stage 3 from the rows' first arcs (tags.cu): m >= 8n (or forced), positions below 2^30
  size_t lsucc[8], lwgt[8], lown[8], loffs[8];
  int nlev = 0;
  int64_t K[8] = {0};
  int S[8] = {0};
  int ntile = 0, tlev = 0;
  size_t cub_bytes = 0;

  size_t take(size_t bytes) {
    size_t at = total;
    total += (bytes + 255) & ~size_t(255);
    return at;
  }

  explicit Layout(int64_t n, int64_t m, const Options& o) {
    const int64_t N0 = 2 * n;
    const int kS0 = o.v[OPT_S0], kSl = o.v[OPT_SL];
    S[0] = kS0;
    K[1] = (N0 + kS0 - 1) / kS0;
    nlev = 1;
    while (K[nlev] > kFinalMaxHost) {
      S[nlev] = kSl;
      K[nlev + 1] = (K[nlev] + kSl - 1) / kSl;
      nlev++;
    }
    ntile = (int)((N0 + kTile - 1) / kTile);
    if (ntile < 1) ntile = 1;
    tlev = 1;
    while ((1 << tlev) <= ntile) tlev++;
    cub_bytes = scan_temp_bytes(n + 1);
    if (scan_roots_temp_bytes(n + 1) > cub_bytes) cub_bytes = scan_roots_temp_bytes(n + 1);
    if (scan_upper_temp_bytes((int)n) > cub_bytes) cub_bytes = scan_upper_temp_bytes((int)n);

    sc = take(sizeof(Scalars));
    // root counts of the final compress's 256 x 4-vertex tiles (RootInit::sdesc)
    sdesc_bytes = 8 * ((size_t)n / 1024 + 2);
    sdesc = take(sdesc_bytes);
    crow = take(4 * ((m + kItems - 1) / kItems + 1));
    comp = take(4 * n);
    fe = take(8 * n);
    prop = take(8 * n);
    flags = take(4 * (n + 1));
    rootidx = take(8 * (n + 1));
    rlist = take(4 * n);
    lhead = take(4 * n);
    hsub = take(4 * (m / 16 + 64));
    nexto = take(4 * N0);
    own0 = take(8 * N0);
    nxt = N0 * 8 > (64ll << 20) ? 0 : take(4 * N0);  // (large tours: level 0 runs in place in own0)
    rank0 = take(4 * N0);
    for (int l = 1; l <= nlev; l++) {
      lsucc[l] = take(4 * K[l]);
      lwgt[l] = take(4 * K[l]);
      lown[l] = take(8 * K[l]);
      loffs[l] = take(4 * K[l]);
    }
    rec = take(16 * n);
    AP = take(16 * (size_t)ntile * kTile);
    lh1 = take(8 * n);
    lh2 = take(8 * n);
    table = take(8 * (size_t)ntile * tlev);
    cnt = take(4 * n);
    uoff = take(4 * (n + 1));
    nlow = take(4 * n);
    bmin = take(4 * n);
    w0 = take(12 * n);
    cub = take(cub_bytes);
    const int wopt = o.v[OPT_WITNESS];
    witness = m > 0 && 2 * n < (1ll << 30) && (wopt == 2 || (wopt == 1 && m >= 8 * n));
    wfirsts = witness ? take(4 * n) : 0;  // its own compact first[] (the tile pass reuses the shared one)
  }
};

// One bound instance of the pipeline: graph, workspace carve-up, outputs.
struct Pipeline {
  Options opts;  // snapshot taken at creation; every enqueue runs under it
  Graph g;
  Layout lay;
  Scalars* sc;
  int* comp;
  int2* fe;
  unsigned long long* prop;
  Rooting R;
  Tags T;
  fbcc_outputs out;
  int* cnt;
  int* uoff;
  int* nlow;
  int* bmin;
  const Side* side = nullptr;  // second stream for Stage 6's independent pieces (plan capture, host path)
  Witness W;        // witness plan (Layout::witness); off for a run that exports low / high / w
  int* w0;          // [3][n] each row's arc 0-2 targets (Stage 1's round 0 -> the sampling rounds of Stages 1, 5)
  bool w0_valid = false;
  bool s1_round0 = false;   // Stage 1 ran its sampling round 0 (the device path; not the streamed host path)
  bool no_witness = false;  // this run exports w1 / w2 / low / high (fbcc_debug)

  Pipeline(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, void* workspace,
           const fbcc_outputs* o, const Options& op)
      : opts(op), lay(n, m, op) {
    out = *o;
    char* ws = (char*)workspace;
    auto at = [&](size_t off) { return (void*)(ws + off); };
    g = Graph{offsets, edges, (int)n, m, (const int*)at(lay.crow)};
    sc = (Scalars*)at(lay.sc);
    comp = out.comp ? out.comp : (int*)at(lay.comp);
    fe = (int2*)at(lay.fe);
    prop = (unsigned long long*)at(lay.prop);
    R.flags = (int*)at(lay.flags);
    R.rootidx = (unsigned long long*)at(lay.rootidx);
    R.rlist = (int*)at(lay.rlist);
    R.lhead = (int*)at(lay.lhead);
    R.hsub = (int*)at(lay.hsub);
    R.hoff = offsets;
    R.nexto = (int*)at(lay.nexto);
    R.nxt = lay.nxt ? (int*)at(lay.nxt) : nullptr;  // (nullptr: level 0 in place in own0)
    R.own0 = (int2*)at(lay.own0);
    R.rank0 = (int*)at(lay.rank0);
    R.nlev = lay.nlev;
    for (int l = 0; l < 8; l++) {
      R.K[l] = lay.K[l];
      R.S[l] = lay.S[l];
      R.succ[l] = nullptr;
      R.wgt[l] = nullptr;
      R.own[l] = nullptr;
      R.offs[l] = nullptr;
    }
    for (int l = 1; l <= lay.nlev; l++) {
      R.succ[l] = (int*)at(lay.lsucc[l]);
      R.wgt[l] = (int*)at(lay.lwgt[l]);
      R.own[l] = (int2*)at(lay.lown[l]);
      R.offs[l] = (int*)at(lay.loffs[l]);
    }
    R.rec = (int4*)at(lay.rec);
    R.firsts = (int*)at(lay.lh1);  // Stage 3's compact first[] (see stage3_tags)
    R.nlow = (int*)at(lay.nlow);
    R.cub_tmp = at(lay.cub);
    R.cub_bytes = lay.cub_bytes;
    R.tile_roots = FBCC_ROOT_SCAN_FUSED ? (unsigned long long*)at(lay.sdesc) : nullptr;  // (root_init_args: the final compress of Stage 1 ranks the roots)
    T.AP = (int4*)at(lay.AP);
    T.lh1 = (int2*)at(lay.lh1);
    T.lh2 = (int2*)at(lay.lh2);
    T.table = (int2*)at(lay.table);
    T.ntile = lay.ntile;
    T.tlev = lay.tlev;
    T.tour_len = &sc->tour_len;  // (k_out_lists publishes it)
    cnt = (int*)at(lay.cnt);
    uoff = (int*)at(lay.uoff);
    nlow = (int*)at(lay.nlow);
    bmin = (int*)at(lay.bmin);
    w0 = (int*)at(lay.w0);
    W.on = lay.witness;
    W.firsts = lay.witness ? (int*)at(lay.wfirsts) : nullptr;
    W.w0 = w0;
    W.und_list = R.rlist;  // (the root list is dead once the tour is linked)
    W.cap = (int)std::min<int64_t>(n, 1 << 20);
    W.work = (unsigned long long)std::max<int64_t>(4096, std::min<int64_t>(n / 8, 1 << 22));
  }

  // Enqueue all six stages.  ev (7 events) brackets the stages when given.
  void enqueue(cudaStream_t st, cudaEvent_t* ev, int* low_out, int* high_out, bool capturing = false) {
    OptScope scope(&opts);
    Marks mk{st, ev, capturing};
    cudaMemsetAsync(sc, 0, sizeof(Scalars), st);
    note(K_MEMSET);
    mk(0);
    // (a run that takes Stage 3 from the sampled arcs reads the chunk -> row table only if its repair
    // overflows: not built -- 4 bytes per 8 arcs less to write)
    const bool wrun = W.on && !no_witness && !low_out && !high_out && opts.v[OPT_SAMPLE_ROUNDS] > 0;
    W.crow_built = !wrun;
    R.firsts = wrun ? nullptr : (int*)((char*)sc + (lay.lh1 - lay.sc));  // (k_positions' compact first[]: the full gather's)
    const bool round0 = build_chunk_rows(g, wrun ? nullptr : const_cast<int*>(g.crow), sc, st, comp, fe, prop,
                                         wrun ? nullptr : nlow, w0);
    w0_valid = round0;
    s1_round0 = round0;
    stage1_forest(g, comp, fe, prop, sc, st, round0, root_init_args(), round0 ? w0 : nullptr, R.nexto);
    mk(1);
    enqueue_rest(st, mk, low_out, high_out, nullptr, nullptr);
  }

  struct Marks {
    cudaStream_t st;
    cudaEvent_t* ev;
    bool capturing;
    void operator()(int i) const {
      if (!ev) return;
      // inside a graph capture the record must become an event-record node
      if (capturing) cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal);
      else cudaEventRecord(ev[i], st);
    }
  };

  // Stages 2-6.  label_done / heads_done (optional) are recorded as soon as
  // the label array / the head and is_ap arrays are final.
  // Stage 1's final compress writes Stage 2's root flags and list heads
  RootInit root_init_args() const {
    RootInit ri;
    ri.flags = R.flags;
    ri.lhead = R.lhead;
    ri.hsub = R.hsub;
    ri.off = R.hoff;
    ri.sc = sc;
    ri.detach = opts.v[OPT_DETACH] != 0;
    if (!FBCC_ROOT_SCAN_FUSED) return ri;
    ri.rootidx = R.rootidx;
    ri.sdesc = (unsigned long long*)((char*)sc + (lay.sdesc - lay.sc));
    return ri;
  }

  void enqueue_rest(cudaStream_t st, const Marks& mk, int* low_out, int* high_out, cudaEvent_t label_done,
                    cudaEvent_t heads_done) {
    stage2_rooting_fused(g, comp, fe, R, T.AP, sc, st);
    mk(2);
    // (the sampled tags need Stage 1's recorded arcs, and leave low / high inexact: not for debug exports)
    Witness Wr = W;
    if (low_out || high_out || !w0_valid || no_witness) Wr.on = false;
    stage3_tags(g, R, T, st, nlow, side, uoff, R.cub_tmp, R.cub_bytes, sc, &Wr);
    mk(3);
    // Stage 5's round 0 along plain parent edges rides in Stage 4's pass (skel_parent bit 0x80): always
    // in witness plans (dense graphs), else only where the forest is id-ordered (device-side test;
    // k_hook_min, which also tries each row's first arc, does better on fragmented meshes and kNN graphs)
    const bool s5r0 = (opts.v[OPT_SKEL_PARENT] & 0x80) != 0 && opts.v[OPT_SAMPLE_ROUNDS] > 0;
    // (not on the host path: its streamed forest is no min-neighbour star forest, and without
    // k_hook_min's first-arc hooks Stage 5's sample finds no giant there -- config 2 e2e 2.59 -> 2.79 ms)
    const bool s5always = s5r0 && lay.witness && s1_round0;
    stage4_fence(g, R, T, low_out, high_out, out.head, cnt, bmin, st, sc, &Wr, s5r0 ? out.label : nullptr,
                 s5r0 ? prop : nullptr, s5r0 && !s5always);
    mk(4);
    stage5_skeleton_cc(g, R.rec, out.label, prop, sc, st, w0_valid ? w0 : nullptr, s5always, R.nexto,
                       s5r0 && !s5always);
    mk(5);
    if (label_done) cudaEventRecord(label_done, st);
    // Stage 2's root list / root ranks / out-list links are dead by Stage 6:
    // its deferred rows, search flags and searched positions
    stage6_labelling(g, R.rec, out.label, out.head, out.is_ap, out.edge_label, cnt, uoff, nlow, bmin, R.rlist,
                     reinterpret_cast<int*>(R.rootidx), R.nexto,
                     R.cub_tmp, R.cub_bytes, sc, st, heads_done, side);
    mk(6);
  }

  // Host-resident input and outputs (fbcc_run_host).  The CSR arrives on the
  // copy stream cs -- offsets, then the edge array in nchunk arc ranges --
  // and Stage 1 links each range as soon as it lands (stage1_stream_*), so
  // the union-find hides under the H2D transfer.  label is copied back while
  // Stage 6 runs, head / is_ap while the per-edge labels are computed; only
  // the per-edge labels' own D2H trails the last kernel.
  void enqueue_host(cudaStream_t st, cudaStream_t cs, const fbcc_host_io& io, bool host_off32, cudaEvent_t* hev,
                    int nchunk,
                    cudaEvent_t* ev) {
    OptScope scope(&opts);
    Marks mk{st, ev, false};
    cudaEvent_t ev_start = hev[0], ev_off = hev[1], ev_label = hev[2], ev_heads = hev[3], ev_copies = hev[4];
    cudaEvent_t* ev_chunk = hev + 5;
    const int64_t n = g.n, m = g.m;
    // the copies must not overwrite inputs a previous run on st still reads
    cudaEventRecord(ev_start, st);
    cudaStreamWaitEvent(cs, ev_start, 0);
    // int32 host offsets (FBCC_FLAG_HOST_OFFSETS32): half the bytes over
    // PCIe, widened on the device from a workspace scratch area (the tour
    // list's nexto, untouched until Stage 2)
    int* off32 = host_off32 ? R.nexto : nullptr;
    if (off32)
      cudaMemcpyAsync(off32, io.offsets, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, cs);
    else
      cudaMemcpyAsync(const_cast<int64_t*>(g.off), io.offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice,
                      cs);
    cudaEventRecord(ev_off, cs);
    const int64_t nq = (m + kItems - 1) / kItems;
    int64_t qb[kMaxStreamChunks + 1];
    for (int c = 0; c <= nchunk; c++) qb[c] = nq * c / nchunk;
    for (int c = 0; c < nchunk; c++) {
      const int64_t a0 = qb[c] * kItems, a1 = qb[c + 1] * kItems < m ? qb[c + 1] * kItems : m;
      if (a1 > a0)
        cudaMemcpyAsync(const_cast<uint32_t*>(g.adj) + a0, io.edges + a0, sizeof(uint32_t) * (a1 - a0),
                        cudaMemcpyHostToDevice, cs);
      cudaEventRecord(ev_chunk[c], cs);
    }
    cudaStreamWaitEvent(st, ev_off, 0);
    cudaMemsetAsync(sc, 0, sizeof(Scalars), st);
    note(K_MEMSET);
    mk(0);
    if (off32) widen_offsets(off32, const_cast<int64_t*>(g.off), n, st);
    build_chunk_rows(g, const_cast<int*>(g.crow), sc, st, nullptr, nullptr, nullptr, nlow);
    stage1_stream_begin(g, comp, st);
    for (int c = 0; c < nchunk; c++) {
      cudaStreamWaitEvent(st, ev_chunk[c], 0);
      stage1_stream_range(g, qb[c], qb[c + 1], comp, fe, st);
    }
    stage1_stream_finish(g, comp, sc, st, root_init_args());
    // (the whole edge array is here: the rows' first arcs for Stage 5's sampling rounds and, in
    // witness plans, Stage 3)
    record_arcs(g, w0, st);
    w0_valid = g.m > 0;
    // (the streamed forest is no min-neighbour forest: the samples leave more fence bits open and
    // the repair walks bigger subtrees -- worth it from a few million vertices up: config 5 Stages 3-4
    // 5.5 -> 3.0 ms, but config 2 0.16 -> 0.28 ms)
    if (g.n < (1 << 22)) no_witness = true;
    mk(1);
    enqueue_rest(st, mk, nullptr, nullptr, ev_label, ev_heads);
    if (io.label) {
      cudaStreamWaitEvent(cs, ev_label, 0);
      cudaMemcpyAsync(io.label, out.label, sizeof(int) * n, cudaMemcpyDeviceToHost, cs);
    }
    if (io.head || io.is_ap) cudaStreamWaitEvent(cs, ev_heads, 0);
    if (io.head) cudaMemcpyAsync(io.head, out.head, sizeof(int) * n, cudaMemcpyDeviceToHost, cs);
    if (io.is_ap && out.is_ap) cudaMemcpyAsync(io.is_ap, out.is_ap, n, cudaMemcpyDeviceToHost, cs);
    cudaEventRecord(ev_copies, cs);
    // E <= m/2 labels (exactly m/2 for a loop-free symmetric input)
    if (io.edge_label && out.edge_label && m / 2 > 0)
      cudaMemcpyAsync(io.edge_label, out.edge_label, sizeof(int) * (m / 2), cudaMemcpyDeviceToHost, st);
    cudaStreamWaitEvent(st, ev_copies, 0);
  }
};

}  // namespace fbcc

using namespace fbcc;

struct fbcc_plan_s {
  Pipeline* pipe = nullptr;
  cudaGraphExec_t exec = nullptr;
  Scalars* host = nullptr;  // pinned
  LaunchLog* log = nullptr;  // launch count (+ event nodes when profiled)
  cudaEvent_t ev[7] = {};    // stage boundaries, recorded by the graph itself (TIMING / PROFILE)
  bool timing = false;
};

extern "C" {

int fbcc_version(void) { return 101; }

int fbcc_set_option(int key, int value) {
  if (key < 0 || key >= OPT_NUM) return FBCC_ERR_ARG;
  if ((key == OPT_S0 || key == OPT_SL) && (value < 2 || (value & (value - 1)))) return FBCC_ERR_ARG;
  if (key == OPT_SAMPLE_ROUNDS && (value < 0 || value > 8)) return FBCC_ERR_ARG;
  if (key == OPT_STREAM_CHUNKS && (value < 1 || value > kMaxStreamChunks)) return FBCC_ERR_ARG;
  g_opt[key].store(value, std::memory_order_relaxed);
  return FBCC_OK;
}

int fbcc_get_option(int key) { return (key >= 0 && key < OPT_NUM) ? g_opt[key].load(std::memory_order_relaxed) : -1; }

const char* fbcc_last_cuda_error(void) { return g_cuda_err; }

const char* fbcc_kernel_name(int kind) { return (kind >= 0 && kind < K_NUM_KINDS) ? kKernelNames[kind] : "?"; }

const char* fbcc_strerror(int code) {
  switch (code) {
    case FBCC_OK: return "ok";
    case FBCC_ERR_ARG: return "invalid argument";
    case FBCC_ERR_TOO_LARGE: return "tour positions need n <= 2**30 and m < 2**31";
    case FBCC_ERR_WORKSPACE: return "workspace too small";
    case FBCC_ERR_CUDA: return "CUDA error";
    case FBCC_ERR_CYCLE: return "successor structure contains a cycle";
    case FBCC_ERR_COVER: return "successor structure is not a disjoint list cover";
    case FBCC_ERR_RANGE: return "edge endpoint out of range";
    case FBCC_ERR_LABELS: return "labels are inconsistent with the forest edges";
    case FBCC_ERR_NOT_FOREST: return "a forest on n vertices has at most n-1 edges";
    default: return "unknown error";
  }
}

static int check_sizes(int64_t n, int64_t m) {
  if (n < 0 || m < 0) return FBCC_ERR_ARG;
  // euler_tour.py:402-403: 2n must fit a signed 32-bit tour position
  if (n && 2 * n > 2147483647LL) return FBCC_ERR_TOO_LARGE;
  if (m > 2147483647LL) return FBCC_ERR_TOO_LARGE;
  return FBCC_OK;
}

static int check_args(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, void* workspace,
                      size_t workspace_bytes, const fbcc_outputs* out, const Options& o) {
  int rc = check_sizes(n, m);
  if (rc) return rc;
  if (!out || !offsets || (m > 0 && !edges)) return FBCC_ERR_ARG;
  if (n == 0) return FBCC_OK;
  if (!out->label || !out->head || !workspace) return FBCC_ERR_ARG;
  Layout lay(n, m, o);
  if (workspace_bytes < lay.total) return FBCC_ERR_WORKSPACE;
  return FBCC_OK;
}

int fbcc_workspace_bytes(int64_t n, int64_t m, size_t* bytes_out) {
  if (!bytes_out) return FBCC_ERR_ARG;
  int rc = check_sizes(n, m);
  if (rc) return rc;
  Layout lay(n, m, options_snapshot());
  *bytes_out = lay.total;
  return FBCC_OK;
}

static void fill_counts(fbcc_stats* stats, const Scalars& host) {
  stats->num_bccs = host.nbccs;
  stats->num_components = host.ncomp;
  stats->num_edges = host.num_edges;
}

static void fill_profile(fbcc_stats* stats, const LaunchLog& log) {
  if (!log.profile) return;
  stats->nprof = log.nrec;
  for (int i = 0; i < log.nrec; i++) {
    stats->prof_kind[i] = log.kind[i];
    cudaEventElapsedTime(&stats->prof_ms[i], log.ev[i], log.ev[i + 1]);
  }
}

int fbcc_run(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, void* workspace,
             size_t workspace_bytes, fbcc_outputs* out, fbcc_debug* dbg, fbcc_stats* stats, void* stream,
             uint32_t flags) {
  const Options opts = options_snapshot();
  int rc = check_args(offsets, edges, n, m, workspace, workspace_bytes, out, opts);
  if (rc) return rc;
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n == 0) return FBCC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Pipeline P(offsets, edges, n, m, workspace, out, opts);

  const bool timing = (flags & FBCC_FLAG_TIMING) && stats;
  cudaEvent_t ev[7];
  if (timing)
    for (int i = 0; i < 7; i++) cudaEventCreate(&ev[i]);
  LaunchLog* log = new LaunchLog();
  log->st = st;
  log->profile = (flags & FBCC_FLAG_PROFILE) && stats;
  log->start();
  g_log = log;
  P.no_witness = dbg != nullptr;
  P.enqueue(st, timing ? ev : nullptr, dbg ? dbg->low : nullptr, dbg ? dbg->high : nullptr);
  g_log = nullptr;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && dbg)
    export_debug(P.g, P.fe, P.R.rec, P.T.AP, dbg->forest, dbg->parent, dbg->first, dbg->last, dbg->w1, dbg->w2,
                 dbg->fence, st, P.T.tour_len);
  Scalars host;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, P.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && stats) {
    fill_counts(stats, host);
    stats->launches = log->count;
    fill_profile(stats, *log);
    if (timing) {
      for (int i = 0; i < 6; i++) cudaEventElapsedTime(&stats->stage_ms[i], ev[i], ev[i + 1]);
      cudaEventElapsedTime(&stats->total_ms, ev[0], ev[6]);
    }
  }
  log->destroy();
  if (timing)
    for (int i = 0; i < 7; i++) cudaEventDestroy(ev[i]);
  delete log;
  if (e != cudaSuccess) return cuda_fail(e, "run");
  return FBCC_OK;
}

// copy stream + events of fbcc_run_host, per thread and device
struct HostStreams {
  int dev = -1;
  cudaStream_t cs = nullptr;
  Side side;  // Stage 6's independent pieces
  cudaEvent_t ev[5 + kMaxStreamChunks] = {};
};
static thread_local HostStreams g_hs;

static cudaError_t host_streams() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || g_hs.dev == dev) return e;
  if (g_hs.cs) {  // switched device: the old objects belong to the old one
    cudaStreamDestroy(g_hs.cs);
    cudaStreamDestroy(g_hs.side.s);
    for (auto& x : g_hs.ev) cudaEventDestroy(x);
    for (auto& x : g_hs.side.ev) cudaEventDestroy(x);
  }
  g_hs = HostStreams{};
  e = cudaStreamCreateWithFlags(&g_hs.cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_hs.side.s, cudaStreamNonBlocking);
  for (auto& x : g_hs.side.ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  for (auto& x : g_hs.ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  if (e == cudaSuccess) g_hs.dev = dev;
  return e;
}

int fbcc_run_host(const fbcc_host_io* io, int64_t n, int64_t m, int64_t* d_offsets, uint32_t* d_edges,
                  void* workspace, size_t workspace_bytes, fbcc_outputs* out, fbcc_stats* stats, void* stream,
                  uint32_t flags) {
  if (!io || !io->offsets || (m > 0 && !io->edges)) return FBCC_ERR_ARG;
  const Options opts = options_snapshot();
  int rc = check_args(d_offsets, d_edges, n, m, workspace, workspace_bytes, out, opts);
  if (rc) return rc;
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n == 0) return FBCC_OK;
  cudaError_t e = host_streams();
  if (e != cudaSuccess) return cuda_fail(e, "run_host streams");
  cudaStream_t st = (cudaStream_t)stream;
  Pipeline P(d_offsets, d_edges, n, m, workspace, out, opts);
  const bool timing = (flags & FBCC_FLAG_TIMING) && stats;
  cudaEvent_t ev[7];
  if (timing)
    for (int i = 0; i < 7; i++) cudaEventCreate(&ev[i]);
  LaunchLog* log = new LaunchLog();
  log->st = st;
  log->profile = (flags & FBCC_FLAG_PROFILE) && stats;
  g_log = log;
  // upload ranges: at most the option (default 4), and one per 2^21 arcs --
  // each range costs a fixed link launch and event hop (configs 1/2/3: 1/4/2
  // ranges measured best; 8 was 25 %, 1 %, 5 % slower)
  int nchunk = opts.v[OPT_STREAM_CHUNKS];
  if (nchunk > (int)(m >> 21)) nchunk = (int)(m >> 21);
  if (nchunk < 1) nchunk = 1;
  if (nchunk > kMaxStreamChunks) nchunk = kMaxStreamChunks;
  if (!log->profile) P.side = &g_hs.side;  // (profiled runs stay on one stream)
  P.enqueue_host(st, g_hs.cs, *io, (flags & FBCC_FLAG_HOST_OFFSETS32) != 0, g_hs.ev, nchunk, timing ? ev : nullptr);
  g_log = nullptr;
  e = cudaGetLastError();
  Scalars host;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, P.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && stats) {
    fill_counts(stats, host);
    stats->launches = log->count;
    fill_profile(stats, *log);
    if (timing) {
      for (int i = 0; i < 6; i++) cudaEventElapsedTime(&stats->stage_ms[i], ev[i], ev[i + 1]);
      cudaEventElapsedTime(&stats->total_ms, ev[0], ev[6]);
    }
  }
  log->destroy();
  if (timing)
    for (int i = 0; i < 7; i++) cudaEventDestroy(ev[i]);
  delete log;
  if (e != cudaSuccess) return cuda_fail(e, "run_host");
  return FBCC_OK;
}

int fbcc_plan_create(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, void* workspace,
                     size_t workspace_bytes, const fbcc_outputs* out, uint32_t flags, fbcc_plan* plan_out) {
  if (!plan_out) return FBCC_ERR_ARG;
  *plan_out = nullptr;
  // a plan freezes the options in force at its creation (and is bound to
  // the buffers it was created on -- not to their contents)
  const Options opts = options_snapshot();
  int rc = check_args(offsets, edges, n, m, workspace, workspace_bytes, out, opts);
  if (rc) return rc;
  fbcc_plan p = new fbcc_plan_s();
  if (n > 0) {
    p->pipe = new Pipeline(offsets, edges, n, m, workspace, out, opts);
    cudaStream_t cap;
    cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    cudaGraph_t graph = nullptr;
    p->log = new LaunchLog();
    p->log->st = cap;
    p->log->capturing = true;
    p->log->profile = (flags & FBCC_FLAG_PROFILE) != 0;
    // stage-boundary event nodes only on request: an event node between two
    // kernels also cuts their programmatic (PDL) edge
    p->timing = (flags & (FBCC_FLAG_TIMING | FBCC_FLAG_PROFILE)) != 0;
    for (int i = 0; i < 7 && e == cudaSuccess && p->timing; i++) e = cudaEventCreate(&p->ev[i]);
    // Stage 6's independent pieces on a forked capture stream (not when
    // profiling: the launch log times consecutive launches on one stream)
    Side side;
    const bool use_side = !p->log->profile;
    if (use_side && e == cudaSuccess) e = cudaStreamCreateWithFlags(&side.s, cudaStreamNonBlocking);
    for (int i = 0; i < 4 && use_side && e == cudaSuccess; i++)
      e = cudaEventCreateWithFlags(&side.ev[i], cudaEventDisableTiming);
    if (use_side && e == cudaSuccess) p->pipe->side = &side;
    e = e == cudaSuccess ? cudaGetLastError() : e;
    if (e == cudaSuccess) e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      g_log = p->log;
      p->log->start();
      p->pipe->enqueue(cap, p->timing ? p->ev : nullptr, nullptr, nullptr, true);
      g_log = nullptr;
      e = cudaStreamEndCapture(cap, &graph);
    }
    p->pipe->side = nullptr;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&p->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    if (side.s) cudaStreamDestroy(side.s);
    for (auto& x : side.ev)
      if (x) cudaEventDestroy(x);
    if (e == cudaSuccess) e = cudaMallocHost((void**)&p->host, sizeof(Scalars));
    if (e != cudaSuccess) {
      fbcc_plan_destroy(p);
      return cuda_fail(e, "plan_create");
    }
  }
  *plan_out = p;
  return FBCC_OK;
}

int fbcc_plan_launch(fbcc_plan plan, void* stream) {
  if (!plan) return FBCC_ERR_ARG;
  if (!plan->pipe) return FBCC_OK;  // n == 0
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaGraphLaunch(plan->exec, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(plan->host, plan->pipe->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "plan_launch");
  return FBCC_OK;
}

int fbcc_plan_stats(fbcc_plan plan, fbcc_stats* stats) {
  if (!plan || !stats) return FBCC_ERR_ARG;
  memset(stats, 0, sizeof(*stats));
  if (!plan->pipe) return FBCC_OK;
  {
    fill_counts(stats, *plan->host);
    stats->launches = plan->log->count;
    fill_profile(stats, *plan->log);
    if (plan->timing) {
      for (int i = 0; i < 6; i++) cudaEventElapsedTime(&stats->stage_ms[i], plan->ev[i], plan->ev[i + 1]);
      cudaEventElapsedTime(&stats->total_ms, plan->ev[0], plan->ev[6]);
    }
  }
  return FBCC_OK;
}

int fbcc_plan_run(fbcc_plan plan, fbcc_stats* stats, void* stream) {
  int rc = fbcc_plan_launch(plan, stream);
  if (rc != FBCC_OK) return rc;
  if (plan->pipe) {
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "plan_run");
  }
  return stats ? fbcc_plan_stats(plan, stats) : FBCC_OK;
}

int fbcc_plan_destroy(fbcc_plan plan) {
  if (!plan) return FBCC_OK;
  if (plan->exec) cudaGraphExecDestroy(plan->exec);
  if (plan->host) cudaFreeHost(plan->host);
  for (int i = 0; i < 7; i++)
    if (plan->ev[i]) cudaEventDestroy(plan->ev[i]);
  if (plan->log) {
    plan->log->destroy();
    delete plan->log;
  }
  delete plan->pipe;
  delete plan;
  return FBCC_OK;
}

// ---------------------------------------------------------------------------
// stand-alone operations (ops.cu).  Every op keeps a Scalars block at the
// head of its workspace for error bits and counts, and synchronises once.
// ---------------------------------------------------------------------------
static const size_t kOpHead = 256;

static size_t op_bytes(int op, int64_t a, int64_t b) {
  size_t need = 0;
  switch (op) {
    case FBCC_OP_CONNECTED_COMPONENTS:  // a = n
      return kOpHead + 8 * (size_t)a + 8 * (size_t)a + 512;
    case FBCC_OP_LIST_RANKING:  // a = L
      return kOpHead + op_list_ranking_bytes(a);
    case FBCC_OP_BUILD_EULER_TOUR:  // a = n, b = k
      op_build_euler_tour(a, nullptr, b, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, true,
                          &need);
      return kOpHead + need;
    case FBCC_OP_COMPUTE_TAGS: {  // a = n, b = m
      Graph g{nullptr, nullptr, (int)a, b, nullptr};
      op_compute_tags(g, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, true,
                      &need);
      return kOpHead + need;
    }
    case FBCC_OP_EXTRACT_BCCS:  // a = n
      return kOpHead + op_extract_bytes(a);
    case FBCC_OP_SYMMETRIZE:  // a = k pairs
      return kOpHead + op_symmetrize_bytes(a);
    case FBCC_OP_CLASSIFY_EDGES:  // a = n, b = m (error bits only)
      return kOpHead;
    default:
      return 0;
  }
}

int fbcc_op_workspace_bytes(int op, int64_t a, int64_t b, size_t* bytes_out) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  if (!bytes_out || a < 0 || b < 0) return FBCC_ERR_ARG;
  size_t s = op_bytes(op, a, b);
  if (!s) return FBCC_ERR_ARG;
  *bytes_out = s;
  return FBCC_OK;
}

static int op_finish(Scalars* sc, cudaStream_t st, Scalars* host) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "op");
  int err = host->err;
  if (err & 1) return FBCC_ERR_RANGE;
  if (err & 2) return FBCC_ERR_CYCLE;
  if (err & 16) return FBCC_ERR_NOT_FOREST;
  if (err & 8) return FBCC_ERR_LABELS;
  if (err & 4) return FBCC_ERR_COVER;
  return FBCC_OK;
}

static Scalars* op_start(void* ws, cudaStream_t st) {
  Scalars* sc = (Scalars*)ws;
  cudaMemsetAsync(sc, 0, sizeof(Scalars), st);
  return sc;
}

int fbcc_connected_components(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m,
                              const uint8_t* keep_mask, void* ws, size_t ws_bytes, int32_t* label, int32_t* forest,
                              int64_t* ncomp_out, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  int rc = check_sizes(n, m);
  if (rc) return rc;
  if (!offsets || (m && !edges) || !label || !ws) return FBCC_ERR_ARG;
  if (ws_bytes < op_bytes(FBCC_OP_CONNECTED_COMPONENTS, n, m)) return FBCC_ERR_WORKSPACE;
  if (ncomp_out) *ncomp_out = 0;
  if (n == 0) return FBCC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  char* p = (char*)ws + kOpHead;
  int2* fe = forest ? (int2*)forest : (int2*)p;
  unsigned long long* prop = (unsigned long long*)(p + 8 * n + 256);
  Graph g{offsets, edges, (int)n, m, nullptr};
  masked_cc(g, keep_mask, label, fe, prop, sc, st);
  Scalars host;
  rc = op_finish(sc, st, &host);
  if (ncomp_out) *ncomp_out = host.nroots[7];  // counted by the final compress
  return rc;
}

int fbcc_list_ranking(const int32_t* nxt, int64_t L, const int32_t* heads, int64_t H, int32_t* ranks, void* ws,
                      size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  if (L < 0 || H < 0 || (L && (!nxt || !ranks)) || (H && !heads) || !ws) return FBCC_ERR_ARG;
  if (L > 2147483647LL) return FBCC_ERR_TOO_LARGE;
  if (ws_bytes < op_bytes(FBCC_OP_LIST_RANKING, L, H)) return FBCC_ERR_WORKSPACE;
  if (L == 0) return FBCC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  op_list_ranking(nxt, L, heads, H, ranks, (char*)ws + kOpHead, sc, st);
  Scalars host;
  return op_finish(sc, st, &host);
}

int fbcc_build_euler_tour(int64_t n, const int32_t* pairs, int64_t k, const int32_t* labels, int32_t* parent,
                          int32_t* first, int32_t* last, void* ws, size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  if (n < 0 || k < 0 || !ws) return FBCC_ERR_ARG;
  if (n && 2 * n > 2147483647LL) return FBCC_ERR_TOO_LARGE;
  if (k >= n && n > 0) return FBCC_ERR_NOT_FOREST;  // euler_tour.py:381-382
  if (n == 0) return FBCC_OK;
  if ((k && !pairs) || !parent || !first || !last) return FBCC_ERR_ARG;
  size_t need = op_bytes(FBCC_OP_BUILD_EULER_TOUR, n, k);
  if (ws_bytes < need) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  op_build_euler_tour(n, (const int2*)pairs, k, labels, parent, first, last, (char*)ws + kOpHead, need - kOpHead, sc,
                      st, false, &need);
  Scalars host;
  return op_finish(sc, st, &host);
}

int fbcc_compute_tags(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, const int32_t* parent,
                      const int32_t* first, const int32_t* last, int32_t* w1, int32_t* w2, int32_t* low,
                      int32_t* high, void* ws, size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  int rc = check_sizes(n, m);
  if (rc) return rc;
  if (n == 0) return FBCC_OK;
  if (!offsets || (m && !edges) || !parent || !first || !last || !w1 || !w2 || !low || !high || !ws)
    return FBCC_ERR_ARG;
  size_t need = op_bytes(FBCC_OP_COMPUTE_TAGS, n, m);
  if (ws_bytes < need) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  Graph g{offsets, edges, (int)n, m, nullptr};
  op_compute_tags(g, parent, first, last, w1, w2, low, high, (char*)ws + kOpHead, need - kOpHead, st, false, &need);
  Scalars host;
  return op_finish(sc, st, &host);
}

int fbcc_extract_bccs(const int32_t* label, const int32_t* head, int64_t n, int32_t* block_off, int32_t* block_vtx,
                      int64_t* nblocks, void* ws, size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  if (n < 0 || !nblocks || !ws) return FBCC_ERR_ARG;
  *nblocks = 0;
  if (n == 0) return FBCC_OK;
  if (!label || !head || !block_off || !block_vtx) return FBCC_ERR_ARG;
  if (ws_bytes < op_bytes(FBCC_OP_EXTRACT_BCCS, n, 0)) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  op_extract_bccs(label, head, n, block_off, block_vtx, (char*)ws + kOpHead, sc, st);
  Scalars host;
  int rc = op_finish(sc, st, &host);
  *nblocks = host.nbccs;
  return rc;
}

int fbcc_symmetrize(const int64_t* u, const int64_t* v, int64_t k, int64_t n, int64_t* offsets, uint32_t* edges,
                    int64_t* m_out, void* ws, size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();  // one snapshot for sizing and enqueue
  OptScope scope(&opts);
  if (k < 0 || n < 0 || !m_out || !offsets || !ws || (k && (!u || !v || !edges))) return FBCC_ERR_ARG;
  if (n >= (1LL << 31) || 2 * k > 2147483647LL) return FBCC_ERR_TOO_LARGE;
  if (ws_bytes < op_bytes(FBCC_OP_SYMMETRIZE, k, n)) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  op_symmetrize(u, v, k, n, offsets, edges, (char*)ws + kOpHead, sc, st);
  Scalars host;
  int rc = op_finish(sc, st, &host);
  *m_out = 2 * (int64_t)host.num_edges;
  return rc;
}

int fbcc_classify_edges(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, const int32_t* parent,
                        const int32_t* first, const int32_t* last, const int32_t* low, const int32_t* high,
                        int8_t* cls, void* ws, size_t ws_bytes, void* stream) {
  const Options opts = options_snapshot();
  OptScope scope(&opts);
  int rc = check_sizes(n, m);
  if (rc) return rc;
  if (n == 0 || m == 0) return FBCC_OK;
  if (!offsets || !edges || !parent || !first || !last || !low || !high || !cls || !ws) return FBCC_ERR_ARG;
  if (ws_bytes < op_bytes(FBCC_OP_CLASSIFY_EDGES, n, m)) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  Scalars* sc = op_start(ws, st);
  Graph g{offsets, edges, (int)n, m, nullptr};
  op_classify_edges(g, parent, first, last, low, high, cls, sc, st);
  Scalars host;
  return op_finish(sc, st, &host);
}

}  // extern "C"
