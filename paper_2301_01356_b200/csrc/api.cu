// api.cu -- the C ABI (include/fastbcc_b200.h): workspace layout and the
// six-stage orchestration of fast_bcc (bcc.py:147-196) on one stream.
#include <cstdio>
#include <cstring>

#include "../../include/fastbcc_b200.h"
#include "common.cuh"
#include "kernels.cuh"

namespace fbcc {

static thread_local char g_cuda_err[256] = "";
thread_local LaunchLog* g_log = nullptr;

static const char* kKernelNames[K_NUM_KINDS] = {
    "iota", "sample_link", "compress", "find_giant", "link_rest", "root_flags", "scan", "tree_degree",
    "tree_scatter", "link_slots", "link_roots", "walk0", "walk_level", "final_rank", "expand", "positions",
    "w_gather", "tile", "table", "fence", "heads", "ap", "upper_degree", "set_edges", "edge_blocks",
    "edge_final", "memset", "export"};

static int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", where, cudaGetErrorString(e));
  return FBCC_ERR_CUDA;
}

constexpr int kS0 = 16;   // level-0 splitter spacing (mean segment length)
constexpr int kSl = 32;   // spacing on the weighted splitter levels
constexpr int kFinalMaxHost = 4096;

struct Layout {
  size_t total = 0;
  size_t sc, comp, fe, rootidx, tdeg, ex, tedges, twin, nxt, own0, rec, A, P, lh1, lh2, table, cnt, uoff,
      nlow, bmin, cub;
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

  explicit Layout(int64_t n) {
    const int64_t N0 = 2 * n;
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

    sc = take(sizeof(Scalars));
    comp = take(4 * n);
    fe = take(8 * n);
    rootidx = take(4 * 2 * (n + 1));
    tdeg = take(4 * 2 * (n + 1));
    ex = take(16 * n);
    tedges = take(4 * N0);
    twin = take(4 * N0);
    nxt = take(4 * N0);
    own0 = take(8 * N0);
    for (int l = 1; l <= nlev; l++) {
      lsucc[l] = take(4 * K[l]);
      lwgt[l] = take(4 * K[l]);
      lown[l] = take(8 * K[l]);
      loffs[l] = take(4 * K[l]);
    }
    rec = take(16 * n);
    A = take(8 * (size_t)ntile * kTile);
    P = take(8 * (size_t)ntile * kTile);
    lh1 = take(8 * n);
    lh2 = take(8 * n);
    table = take(8 * (size_t)ntile * tlev);
    cnt = take(4 * n);
    uoff = take(4 * 2 * (n + 1));
    nlow = take(4 * n);
    bmin = take(4 * n);
    cub = take(cub_bytes);
  }
};

}  // namespace fbcc

using namespace fbcc;

extern "C" {

int fbcc_version(void) { return 100; }

const char* fbcc_kernel_name(int kind) {
  return (kind >= 0 && kind < K_NUM_KINDS) ? kKernelNames[kind] : "?";
}

const char* fbcc_last_cuda_error(void) { return g_cuda_err; }

const char* fbcc_strerror(int code) {
  switch (code) {
    case FBCC_OK: return "ok";
    case FBCC_ERR_ARG: return "invalid argument";
    case FBCC_ERR_TOO_LARGE: return "tour positions need n <= 2**30 and m < 2**31";
    case FBCC_ERR_WORKSPACE: return "workspace too small";
    case FBCC_ERR_CUDA: return "CUDA error";
    case FBCC_ERR_CYCLE: return "successor structure contains a cycle";
    case FBCC_ERR_COVER: return "successor structure is not a disjoint list cover";
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

int fbcc_workspace_bytes(int64_t n, int64_t m, size_t* bytes_out) {
  if (!bytes_out) return FBCC_ERR_ARG;
  int rc = check_sizes(n, m);
  if (rc) return rc;
  Layout lay(n);
  *bytes_out = lay.total;
  return FBCC_OK;
}

int fbcc_run(const int64_t* offsets, const uint32_t* edges, int64_t n, int64_t m, void* workspace,
             size_t workspace_bytes, fbcc_outputs* out, fbcc_debug* dbg, fbcc_stats* stats, void* stream,
             uint32_t flags) {
  int rc = check_sizes(n, m);
  if (rc) return rc;
  if (!out || !offsets || (m > 0 && !edges)) return FBCC_ERR_ARG;
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n == 0) return FBCC_OK;
  if (!out->label || !out->head || !workspace) return FBCC_ERR_ARG;
  Layout lay(n);
  if (workspace_bytes < lay.total) return FBCC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  auto at = [&](size_t o) { return (void*)(ws + o); };

  Graph g{offsets, edges, (int)n, m};
  Scalars* sc = (Scalars*)at(lay.sc);
  int* comp = out->comp ? out->comp : (int*)at(lay.comp);
  int2* fe = (int2*)at(lay.fe);
  Rooting R;
  R.rootidx = (int*)at(lay.rootidx);
  R.tdeg = (int*)at(lay.tdeg);
  R.ex = (int4*)at(lay.ex);
  R.tedges = (int*)at(lay.tedges);
  R.twin = (int*)at(lay.twin);
  R.nxt = (int*)at(lay.nxt);
  R.own0 = (int2*)at(lay.own0);
  R.nlev = lay.nlev;
  for (int l = 0; l < 8; l++) {
    R.K[l] = lay.K[l];
    R.S[l] = lay.S[l];
    R.succ[l] = nullptr; R.wgt[l] = nullptr; R.own[l] = nullptr; R.offs[l] = nullptr;
  }
  for (int l = 1; l <= lay.nlev; l++) {
    R.succ[l] = (int*)at(lay.lsucc[l]);
    R.wgt[l] = (int*)at(lay.lwgt[l]);
    R.own[l] = (int2*)at(lay.lown[l]);
    R.offs[l] = (int*)at(lay.loffs[l]);
  }
  R.rec = (int4*)at(lay.rec);
  R.cub_tmp = at(lay.cub);
  R.cub_bytes = lay.cub_bytes;
  Tags T;
  T.A = (int2*)at(lay.A);
  T.P = (int2*)at(lay.P);
  T.lh1 = (int2*)at(lay.lh1);
  T.lh2 = (int2*)at(lay.lh2);
  T.table = (int2*)at(lay.table);
  T.ntile = lay.ntile;
  T.tlev = lay.tlev;

  const bool timing = (flags & FBCC_FLAG_TIMING) && stats;
  cudaEvent_t ev[7];
  if (timing)
    for (int i = 0; i < 7; i++) cudaEventCreate(&ev[i]);
  auto mark = [&](int i) {
    if (timing) cudaEventRecord(ev[i], st);
  };

  LaunchLog* log = new LaunchLog();
  log->st = st;
  log->profile = (flags & FBCC_FLAG_PROFILE) && stats;
  if (log->profile) {
    cudaEventCreate(&log->ev[0]);
    cudaEventRecord(log->ev[0], st);
  }
  g_log = log;
  cudaMemsetAsync(sc, 0, sizeof(Scalars), st);
  note(K_MEMSET);
  mark(0);
  stage1_forest(g, comp, fe, sc, st);
  mark(1);
  stage2_rooting(g, comp, fe, R, T.A, T.P, sc, st);
  mark(2);
  stage3_tags(g, R, T, st);
  mark(3);
  stage4_fence(g, R, T, dbg ? dbg->low : nullptr, dbg ? dbg->high : nullptr, st);
  mark(4);
  stage5_skeleton_cc(g, R.rec, out->label, sc, st);
  mark(5);
  stage6_labelling(g, R.rec, out->label, out->head, out->is_ap, out->edge_label, (int*)at(lay.cnt),
                   (int*)at(lay.uoff), (int*)at(lay.nlow), (int*)at(lay.bmin), R.cub_tmp, R.cub_bytes, sc, st);
  mark(6);
  g_log = nullptr;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete log;
    return cuda_fail(e, "launch");
  }
  if (dbg)
    export_debug(g, fe, R.rec, T.A, dbg->forest, dbg->parent, dbg->first, dbg->last, dbg->w1, dbg->w2, dbg->fence,
                 st);
  Scalars host;
  e = cudaMemcpyAsync(&host, sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    delete log;
    return cuda_fail(e, "run");
  }
  if (stats) {
    stats->launches = log->count;
    if (log->profile) {
      stats->nprof = log->nrec;
      for (int i = 0; i < log->nrec; i++) {
        stats->prof_kind[i] = log->kind[i];
        cudaEventElapsedTime(&stats->prof_ms[i], log->ev[i], log->ev[i + 1]);
      }
      for (int i = 0; i <= log->nrec; i++) cudaEventDestroy(log->ev[i]);
    }
    stats->num_bccs = host.nbccs;
    stats->num_components = host.ncomp;
    stats->num_edges = host.num_edges;
    if (timing) {
      for (int i = 0; i < 6; i++) cudaEventElapsedTime(&stats->stage_ms[i], ev[i], ev[i + 1]);
      cudaEventElapsedTime(&stats->total_ms, ev[0], ev[6]);
      for (int i = 0; i < 7; i++) cudaEventDestroy(ev[i]);
    }
  }
  delete log;
  return FBCC_OK;
}

}  // extern "C"
