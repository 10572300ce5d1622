/*
 * fastbcc_b200.h -- C ABI of the B200-native FAST-BCC hot path.
 *
 * Library: paper_2301_01356_b200/libfastbcc_b200.so (sm_100a, built by
 * paper_2301_01356_b200/build.py).  Plain pointers and sizes only; every
 * array argument is a DEVICE pointer owned by the caller, and ``stream`` is a
 * cudaStream_t passed as void*.  The library never allocates device memory
 * inside a run: the caller provides one workspace of fbcc_workspace_bytes().
 *
 * Reference interface replaced (all under /root/reference/pkg/src/fastbcc):
 *   fbcc_run            fast_bcc(g, *, beta, seed, block) -> BccLabeling
 *                       bcc.py:147-196, plus articulation_points
 *                       bcc.py:222-235 and the per-edge labels derived by the
 *                       rule of bcc.py:24-27 (canonical: min edge id per block,
 *                       edge ids in tv_skeleton order, baselines.py:251-257)
 *   fbcc_workspace_bytes  (no reference counterpart: scratch is allocated by
 *                       _meter inside each step, _meter.py:30-74)
 *   fbcc_strerror       the reference's ValueError messages
 *                       (euler_tour.py:349-357, 402-403; graphs.py:126-130)
 * Input layout is the reference Graph unchanged (graphs.py:43-58): int64
 * offsets[n+1], uint32 targets[m], symmetric, sorted rows, no self-loops or
 * duplicates (not validated, exactly like the reference, graphs.py:53).
 */
#ifndef FASTBCC_B200_H
#define FASTBCC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define FBCC_OK 0
#define FBCC_ERR_ARG 1        /* null pointer / negative size / bad flag     */
#define FBCC_ERR_TOO_LARGE 2  /* n > 2^30 (euler_tour.py:402-403) or m >= 2^31 */
#define FBCC_ERR_WORKSPACE 3  /* workspace_bytes smaller than required        */
#define FBCC_ERR_CUDA 4       /* a CUDA runtime error (see fbcc_last_cuda_error) */
#define FBCC_ERR_CYCLE 5      /* list ranking: cycle (euler_tour.py:349-351)  */
#define FBCC_ERR_COVER 6      /* list ranking: not a disjoint cover (:353-355) */
#define FBCC_ERR_RANGE 7      /* endpoint out of range (graphs.py:126-130, euler_tour.py:383-384) */
#define FBCC_ERR_LABELS 8     /* labels inconsistent with the forest (euler_tour.py:435-436) */
#define FBCC_ERR_NOT_FOREST 9 /* k >= n edges or a cycle (euler_tour.py:381-382) */

/* stand-alone operation codes for fbcc_op_workspace_bytes */
#define FBCC_OP_CONNECTED_COMPONENTS 1 /* a = n, b = m  */
#define FBCC_OP_LIST_RANKING 2         /* a = L, b = H  */
#define FBCC_OP_BUILD_EULER_TOUR 3     /* a = n, b = k  */
#define FBCC_OP_COMPUTE_TAGS 4         /* a = n, b = m  */
#define FBCC_OP_EXTRACT_BCCS 5         /* a = n         */
#define FBCC_OP_SYMMETRIZE 6           /* a = k pairs, b = n */
#define FBCC_OP_CLASSIFY_EDGES 7       /* a = n, b = m  */

/* run flags */
#define FBCC_FLAG_TIMING 1u   /* record per-stage CUDA-event times in stats   */
#define FBCC_FLAG_PROFILE 2u  /* also bracket every launch with CUDA events   */
#define FBCC_FLAG_HOST_OFFSETS32 4u  /* fbcc_run_host: io->offsets holds int32 offsets
                                        (m < 2^31; half the upload, widened on the device) */
#define FBCC_MAX_PROFILE 512

/* Outputs of one run; all DEVICE pointers.  label/head are required. */
typedef struct {
  int32_t *label;      /* [n] BccLabeling.label: min id of v's skeleton component */
  int32_t *head;       /* [n] BccLabeling.head: -1 for root singletons and non-labels */
  int32_t *edge_label; /* [E] or NULL: min edge id of the edge's block;
                          edge e = e-th arc (u -> v, u < v) in CSR order */
  uint8_t *is_ap;      /* [n] or NULL: articulation-point flags */
  int32_t *comp;       /* [n] or NULL: first-pass component labels (min id) */
} fbcc_outputs;

/* HOST buffers of fbcc_run_host.  Pinned (page-locked) memory lets the
   copies overlap the kernels; pageable memory works but serialises them. */
typedef struct {
  const int64_t *offsets; /* [n+1] symmetric CSR, as fbcc_run (int32 values
                             with FBCC_FLAG_HOST_OFFSETS32)                    */
  const uint32_t *edges;  /* [m]                                              */
  int32_t *label;         /* [n] or NULL                                      */
  int32_t *head;          /* [n] or NULL                                      */
  int32_t *edge_label;    /* capacity m/2 or NULL; the first E entries valid  */
  uint8_t *is_ap;         /* [n] or NULL                                      */
} fbcc_host_io;

/* Optional intermediate exports for stage-level parity (DEVICE pointers,
   each may be NULL).  Written after the run, outside the per-stage timers. */
typedef struct {
  int32_t *forest;  /* [2n] (u, v) of the forest edge that hooked vertex x, at
                       [2x, 2x+1]; meaningful where comp[x] != x            */
  int32_t *parent;  /* [n] rooted forest (RootedForest, euler_tour.py:38-54) */
  int32_t *first;   /* [n] */
  int32_t *last;    /* [n] */
  int32_t *w1;      /* [n] VertexTags (tagging.py:42-49)                     */
  int32_t *w2;      /* [n] */
  int32_t *low;     /* [n] */
  int32_t *high;    /* [n] */
  uint8_t *fence;   /* [n] skeleton_record fence bit (connectivity.py:94-96) */
} fbcc_debug;

/* Host-side statistics of one run. stage_ms: S1 forest, S2 rooting,
   S3 tags, S4 fence, S5 skeleton CC, S6 labelling (CUDA events; only with
   FBCC_FLAG_TIMING, else zeros). */
typedef struct {
  int64_t num_bccs;
  int64_t num_components;
  int64_t num_edges;
  float stage_ms[6];
  float total_ms;
  int32_t launches;                       /* kernels launched by this run    */
  int32_t nprof;                          /* FBCC_FLAG_PROFILE: entries below */
  int32_t prof_kind[FBCC_MAX_PROFILE];    /* kernel kind (fbcc_kernel_name)  */
  float prof_ms[FBCC_MAX_PROFILE];        /* device time between its events   */
} fbcc_stats;

/* End to end from host memory (the path behind fast_bcc on a host Graph):
   copy io->offsets / io->edges into d_offsets / d_edges, run, copy the
   outputs back into io's host buffers; returns after everything landed.
   The edge array is copied in arc ranges and Stage 1 links each range as it
   arrives (the union-find runs under the transfer); label / head / is_ap
   are copied back while Stage 6 still runs.  Same results as fbcc_run. */
int fbcc_run_host(const fbcc_host_io *io, int64_t n, int64_t m, int64_t *d_offsets, uint32_t *d_edges,
                  void *workspace, size_t workspace_bytes, fbcc_outputs *out, fbcc_stats *stats,
                  void *stream, uint32_t flags);

/* Required workspace bytes for a graph of n vertices and m directed slots. */
int fbcc_workspace_bytes(int64_t n, int64_t m, size_t *bytes_out);

/* The whole pipeline on a device-resident CSR.  Asynchronous on ``stream``
   except for one final synchronisation that reads back the three counts. */
int fbcc_run(const int64_t *offsets, const uint32_t *edges, int64_t n,
             int64_t m, void *workspace, size_t workspace_bytes,
             fbcc_outputs *out, fbcc_debug *debug, fbcc_stats *stats,
             void *stream, uint32_t flags);

/* CUDA-graph plan: the whole launch sequence for one (graph, workspace,
   outputs) binding, captured once and replayed by fbcc_plan_run (same
   results as fbcc_run).  The graph records the six stage boundaries as event
   nodes (stats.stage_ms after each run); with FBCC_FLAG_PROFILE it also
   records one event node after every kernel (stats.prof_*).  The bound
   buffers must stay valid until fbcc_plan_destroy.  A plan depends on the
   buffers, not on their contents: the caller may refill them with another
   graph of the same n and m between replays.  It freezes the options in
   force when it was created. */
typedef struct fbcc_plan_s *fbcc_plan;
int fbcc_plan_create(const int64_t *offsets, const uint32_t *edges, int64_t n,
                     int64_t m, void *workspace, size_t workspace_bytes,
                     const fbcc_outputs *out, uint32_t flags,
                     fbcc_plan *plan_out);
int fbcc_plan_run(fbcc_plan plan, fbcc_stats *stats, void *stream);
/* Asynchronous form of fbcc_plan_run: enqueue the graph and the copy of the
   device counts on `stream` and return.  fbcc_plan_stats fills `stats` once
   the caller has synchronised that stream (pipelined replays, no host round
   trip per run). */
int fbcc_plan_launch(fbcc_plan plan, void *stream);
int fbcc_plan_stats(fbcc_plan plan, fbcc_stats *stats);
int fbcc_plan_destroy(fbcc_plan plan);

/* Process-wide tuning defaults (result-neutral, like the reference's beta /
   block / seed, bcc.py:147-155; every setting gives identical outputs,
   tests/test_gpu_mid.py::test_mid_graph_option_paths).  Thread-safe: each
   call (fbcc_run, fbcc_run_host, an op) and each plan snapshots the defaults
   once and runs with its own copy, so a concurrent fbcc_set_option never
   changes a run in flight.  Keys 3/4/20 change fbcc_workspace_bytes.  Keys:
     0  sampling rounds always run (0..8; default 2)
     1  giant-component skip in the remaining-arc link pass (0/1; 1)
     3  level-0 list-ranking splitter spacing (power of two >= 2; 16)
     4  higher-level splitter spacing (power of two >= 2; 8)
     8  bitmask of sampling rounds followed by a compress (0 = first + last; 0xFF)
    11  programmatic dependent launch (0/1; 1)
    12  fbcc_run_host: arc ranges the edge upload is split into, at most one per
        2^21 arcs (1..64; 4)
    13  Stage 5: bitmask of rounds that also hook along plain parent edges (3);
        bit 7: round 0 along parent edges only (config 2 -0.6 %, 4a/4b +2 %: off)
    14  the last sampling compress also picks the giant (0/1; 1)
    15  Stage 6 edge pass: staged rows + giant bitmap (0/1; 1)
    16  adaptive sampling rounds beyond key 0, up to this many (3)
    17  Stage 5's cap for key 16 instead (0 = key 16; 4: config 3 -3 %, config 2 +1 %)
    18  fold each round's accept into the following compress (0/1/2 = auto: on for
        n >= 2^22; 2: configs 4a/4b/4c/5 -1 to -4 %, config 2 would be +6 %)
    19  isolated vertices (but vertex 0) stay off the Euler-tour list and out of
        the tile pass; their tour positions follow the list's (0/1; 1)
    20  Stage 3 from each row's first three arcs, the fence bits they leave open
        repaired exactly, the full per-arc gather only if that repair overflows
        (0 off, 1 plans with m >= 8n, 2 every plan with 2n < 2^30; 1).  Changes
        fbcc_workspace_bytes (4n more).  Runs that export w1/w2/low/high
        (fbcc_debug) always use the full gather.
   Keys 2, 5, 6, 7, 9, 10 are retired experiments: accepted and ignored. */
int fbcc_set_option(int key, int value);
int fbcc_get_option(int key);

/* ---- stand-alone stage operations (the reference's public stage API) ----
   Each takes a workspace of fbcc_op_workspace_bytes(op, a, b) and
   synchronises once on ``stream``.  All arrays are DEVICE pointers. */
int fbcc_op_workspace_bytes(int op, int64_t a, int64_t b, size_t *bytes_out);

/* connected_components(g, keep_edge) connectivity.py:593-611: min-id labels,
   forest[2x, 2x+1] = the edge that hooked vertex x (x non-root), component
   count.  keep_mask (per slot, may be NULL) is read at each undirected
   edge's u < w slot, like _scan_crossing (connectivity.py:279). */
int fbcc_connected_components(const int64_t *offsets, const uint32_t *edges,
                              int64_t n, int64_t m, const uint8_t *keep_mask,
                              void *ws, size_t ws_bytes, int32_t *label,
                              int32_t *forest, int64_t *ncomp_out,
                              void *stream);

/* list_ranking(nxt, heads) euler_tour.py:322-358: 0-based rank from each
   list's head; heads < 0 ignored; FBCC_ERR_CYCLE / FBCC_ERR_COVER like the
   reference's ValueErrors. */
int fbcc_list_ranking(const int32_t *nxt, int64_t L, const int32_t *heads,
                      int64_t H, int32_t *ranks, void *ws, size_t ws_bytes,
                      void *stream);

/* build_euler_tour(n, tree_edges, labels) euler_tour.py:361-394: roots at
   min ids, parent/first/last identical to the reference's (same out-arc
   order).  pairs = k (u, v) int32 pairs; labels may be NULL. */
int fbcc_build_euler_tour(int64_t n, const int32_t *pairs, int64_t k,
                          const int32_t *labels, int32_t *parent,
                          int32_t *first, int32_t *last, void *ws,
                          size_t ws_bytes, void *stream);

/* compute_tags(g, forest) tagging.py:300-304 on a given rooted forest. */
int fbcc_compute_tags(const int64_t *offsets, const uint32_t *edges, int64_t n,
                      int64_t m, const int32_t *parent, const int32_t *first,
                      const int32_t *last, int32_t *w1, int32_t *w2,
                      int32_t *low, int32_t *high, void *ws, size_t ws_bytes,
                      void *stream);

/* extract_bccs(labeling) bcc.py:199-219: block b = block_vtx[block_off[b] ..
   block_off[b+1]) (sorted, head included), blocks in label order.
   block_off needs n+1 entries, block_vtx 2n. */
int fbcc_extract_bccs(const int32_t *label, const int32_t *head, int64_t n,
                      int32_t *block_off, int32_t *block_vtx,
                      int64_t *nblocks, void *ws, size_t ws_bytes,
                      void *stream);

/* symmetrize(edges, n) graphs.py:119-143 on the device: offsets[n+1],
   edges[<= 2k]; *m_out = directed slots written. */
int fbcc_symmetrize(const int64_t *u, const int64_t *v, int64_t k, int64_t n,
                    int64_t *offsets, uint32_t *edges, int64_t *m_out,
                    void *ws, size_t ws_bytes, void *stream);

/* classify_edge(forest, tags, u, v) bcc.py:54-70 for every slot of the CSR
   against a given rooted forest (parent/first/last) and its tags (low/high):
   cls[m] = EdgeClass (bcc.py:45-51): 0 PLAIN_TREE, 1 FENCE_TREE, 2 BACK,
   3 CROSS.  An endpoint outside [0, n) gives FBCC_ERR_RANGE. */
int fbcc_classify_edges(const int64_t *offsets, const uint32_t *edges, int64_t n,
                        int64_t m, const int32_t *parent, const int32_t *first,
                        const int32_t *last, const int32_t *low,
                        const int32_t *high, int8_t *cls, void *ws,
                        size_t ws_bytes, void *stream);

/* Name of a kernel kind reported in fbcc_stats.prof_kind. */
const char *fbcc_kernel_name(int kind);

/* Human-readable message for a status code (reference wording). */
const char *fbcc_strerror(int code);

/* Last CUDA error string recorded by this thread (for FBCC_ERR_CUDA). */
const char *fbcc_last_cuda_error(void);

/* ABI version (major * 100 + minor). */
int fbcc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FASTBCC_B200_H */
