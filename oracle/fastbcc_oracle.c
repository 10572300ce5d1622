/*
 * fastbcc_oracle.c -- CPU restatement of the FAST-BCC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2301_01356_b200/csrc and the CPU baseline timed by
 * bench.py (--impl reference / the cpu_baseline leg).  Nothing in the product
 * path links, loads or calls it; only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs may.
 *
 * It restates, in plain C (+ optional OpenMP on the loops the reference runs
 * under prange), the algorithm of the reference package
 * /root/reference/pkg/src/fastbcc (Python + numba).  Every function cites the
 * reference file:line it follows.  Layout follows the reference Graph
 * (graphs.py:43-58): int64 offsets[n+1], uint32 targets[m], symmetric, sorted,
 * no self-loops, no duplicates.
 *
 * One deliberate difference: the reference's connectivity pass first grows
 * low-diameter clusters (connectivity.py:195-246) and then folds the crossing
 * edges with a sequential union-find (connectivity.py:287-309).  That
 * clustering is result-neutral (labels are min-id canonical; the reference's
 * own tests pin seed/beta invariance, test_connectivity.py:72-79), so this
 * restatement runs the same union-find with every vertex as its own cluster,
 * i.e. _union_batch over all arcs u<w.  Everything downstream consumes the
 * forest exactly as _rooted_from_claims does.
 *
 * Two modes.  Sequential (orc_fast_bcc): the checker -- union-find and list
 * ranking sequential as in the reference's _union_batch / _accumulate_chains.
 * Parallel (orc_fast_bcc_mode(..., 1)): the CPU baseline -- every loop on all
 * host cores, the union-find concurrent (CAS hooking) and the list ranking
 * in the reference's splitter / walk / chain / scatter shape.  Both produce
 * the same outputs (forest-independent, SURVEY §0 finding 2).
 *
 * Parity is pinned by tests/test_oracle_golden.py against golden vectors
 * produced by running the reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_CYCLE 1  /* list ranking: a cycle (euler_tour.py:349-351) */
#define ORC_ERR_COVER 2  /* list ranking: not a disjoint list cover (:353-355) */
#define ORC_ERR_LABELS 3 /* labels inconsistent with forest (euler_tour.py:435-436) */
#define ORC_ERR_ARG 4
#define ORC_ERR_NOMEM 5

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* ------------------------------------------------------------------------ */
/* union-find with path splitting: connectivity.py:259-265                   */
/* ------------------------------------------------------------------------ */
static inline int32_t uf_find(int32_t *p, int32_t x) {
  while (p[x] != x) {
    int32_t up = p[x];
    p[x] = p[up];
    x = up;
  }
  return x;
}

/* skeleton predicate on packed records: connectivity.py:57-81 */
static inline int skel_kept(const int64_t *skel, int64_t u, int64_t w) {
  int64_t mw = skel[2 * w + 1];
  if ((mw >> 1) - 1 == u) return (mw & 1) == 0; /* tree edge, w child */
  int64_t mu = skel[2 * u + 1];
  if ((mu >> 1) - 1 == w) return (mu & 1) == 0; /* tree edge, u child */
  int64_t iu = skel[2 * u], iw = skel[2 * w];
  int64_t fu = iu >> 32, lu = iu & 0xFFFFFFFFLL;
  int64_t fw = iw >> 32, lw = iw & 0xFFFFFFFFLL;
  if (fu <= fw && lu >= lw) return 0; /* back edge: u ancestor of w */
  if (fw <= fu && lw >= lu) return 0;
  return 1; /* cross edge */
}

/*
 * Connected components + spanning forest (restates _cc_parts,
 * connectivity.py:541-574, with singleton clusters; see header).
 *   keep_mask: optional per-slot byte filter (connectivity.py:60-61)
 *   skel:      optional packed skeleton record int64[n][2] (connectivity.py:62-80)
 * Writes label[v] = min id of v's component (connectivity.py:322-341) and the
 * winning union edges (forest_u/forest_v, discovery order, connectivity.py:302-308).
 * Returns the number of components.
 */
int64_t orc_cc(int64_t n, const int64_t *off, const uint32_t *adj,
               const uint8_t *keep_mask, const int64_t *skel, int32_t *label,
               int32_t *forest_u, int32_t *forest_v, int64_t *fcount_out) {
  int32_t *p = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  if (!p) return -1;
  for (int64_t v = 0; v < n; v++) p[v] = (int32_t)v;
  int64_t fcount = 0;
  for (int64_t u = 0; u < n; u++) {
    for (int64_t s = off[u]; s < off[u + 1]; s++) {
      int64_t w = adj[s];
      if (u >= w) continue; /* _scan_crossing packs u < w only (:279) */
      if (keep_mask && !keep_mask[s]) continue;
      if (skel && !skel_kept(skel, u, w)) continue;
      int32_t ru = uf_find(p, (int32_t)u), rw = uf_find(p, (int32_t)w);
      if (ru == rw) continue;
      if (ru < rw) p[rw] = ru; else p[ru] = rw; /* larger root under smaller (:302-305) */
      if (forest_u) { forest_u[fcount] = (int32_t)u; forest_v[fcount] = (int32_t)w; }
      fcount++;
    }
  }
  int64_t ncomp = 0;
  for (int64_t v = 0; v < n; v++) {
    label[v] = uf_find(p, (int32_t)v); /* root == min member by construction */
    if (label[v] == v) ncomp++;
  }
  free(p);
  if (fcount_out) *fcount_out = fcount;
  return ncomp;
}

/*
 * List ranking (euler_tour.py:322-358).  Exact 0-based rank of each cell
 * from its own list head; heads < 0 are ignored.  The reference samples
 * sqrt(L) splitters; ranks are exact positions so a single chase per head
 * computes the same output.  Error classes follow the reference: a cycle
 * reached from a head -> ORC_ERR_CYCLE; a merge, a head in mid-list, or cells
 * no head reaches -> ORC_ERR_COVER.
 */
int orc_list_ranking(int64_t L, const int32_t *nxt, int64_t nheads,
                     const int32_t *heads, int32_t *ranks) {
  for (int64_t i = 0; i < L; i++) ranks[i] = -1;
  if (L == 0) return ORC_OK;
  /* owner list id per cell, to tell a cycle (own list) from a merge */
  int32_t *owner = (int32_t *)malloc(sizeof(int32_t) * L);
  if (!owner) return ORC_ERR_NOMEM;
  for (int64_t i = 0; i < L; i++) owner[i] = -1;
  int64_t covered = 0;
  int rc = ORC_OK;
  for (int64_t h = 0; h < nheads && rc == ORC_OK; h++) {
    int64_t s = heads[h];
    if (s < 0) continue;
    if (s >= L) { rc = ORC_ERR_COVER; break; }
    int32_t r = 0;
    while (s != -1) {
      if (s < 0 || s >= L) { rc = ORC_ERR_COVER; break; }
      if (ranks[s] != -1) {
        rc = (owner[s] == h) ? ORC_ERR_CYCLE : ORC_ERR_COVER;
        break;
      }
      ranks[s] = r++;
      owner[s] = (int32_t)h;
      covered++;
      s = nxt[s];
    }
  }
  free(owner);
  if (rc == ORC_OK && covered != L) rc = ORC_ERR_COVER;
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Parallel mode (orc_fast_bcc_mode(..., parallel=1)): the same outputs from */
/* the reference's parallel structure.  The reference grows LDD clusters in   */
/* parallel (connectivity.py:195-246) and unions the crossing arcs; here all  */
/* arcs are unioned concurrently (CAS hooking larger root under smaller, the  */
/* reference's link rule connectivity.py:302-305, so roots stay component     */
/* minima).  The forest differs from the sequential one -- it is a spanning   */
/* forest all the same, and every output downstream is forest-independent    */
/* (SURVEY §0 finding 2; pinned by the golden tests in both modes).          */
/* ------------------------------------------------------------------------ */
static inline int32_t par_find(int32_t *p, int32_t x) {
  for (;;) {
    int32_t px = __atomic_load_n(&p[x], __ATOMIC_RELAXED);
    if (px == x) return x;
    int32_t gp = __atomic_load_n(&p[px], __ATOMIC_RELAXED);
    if (gp != px) __atomic_store_n(&p[x], gp, __ATOMIC_RELAXED); /* path halving: an ancestor */
    x = gp;
  }
}

int64_t orc_cc_par(int64_t n, const int64_t *off, const uint32_t *adj,
                   const int64_t *skel, int32_t *label, int32_t *forest_u,
                   int32_t *forest_v, int64_t *fcount_out) {
  int32_t *p = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  int32_t *hu = forest_u ? (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1)) : NULL;
  int32_t *hv = forest_u ? (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1)) : NULL;
  if (!p || (forest_u && (!hu || !hv))) { free(p); free(hu); free(hv); return -1; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) { p[v] = (int32_t)v; if (hu) hu[v] = -1; }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t u = 0; u < n; u++) {
    for (int64_t s = off[u]; s < off[u + 1]; s++) {
      int64_t w = adj[s];
      if (u >= w) continue;
      if (skel && !skel_kept(skel, u, w)) continue;
      for (;;) {
        int32_t ru = par_find(p, (int32_t)u), rw = par_find(p, (int32_t)w);
        if (ru == rw) break;
        int32_t hi = ru > rw ? ru : rw, lo = ru ^ rw ^ hi, exp = hi;
        if (__atomic_compare_exchange_n(&p[hi], &exp, lo, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
          if (hu) { hu[hi] = (int32_t)u; hv[hi] = (int32_t)w; } /* one winner per hooked root */
          break;
        }
      }
    }
  }
  int64_t ncomp = 0;
#pragma omp parallel for schedule(static) reduction(+ : ncomp)
  for (int64_t v = 0; v < n; v++) {
    label[v] = par_find(p, (int32_t)v);
    ncomp += label[v] == v;
  }
  int64_t fcount = 0;
  if (hu) {
    for (int64_t v = 0; v < n; v++)
      if (hu[v] >= 0) { forest_u[fcount] = hu[v]; forest_v[fcount] = hv[v]; fcount++; }
  }
  free(p); free(hu); free(hv);
  if (fcount_out) *fcount_out = fcount;
  return ncomp;
}

/*
 * Parallel list ranking in the reference's shape (euler_tour.py:322-358):
 * splitters = every head plus every cell i with i % S == 0 (the reference
 * samples ~sqrt(L) at random, :337-343; ranks are exact either way), each
 * splitter walks to the next one in parallel (_walk_segments :179-195), a
 * sequential pass chains the splitters of each list (_accumulate_chains
 * :198-218), and a parallel re-walk writes the ranks (_scatter_ranks
 * :221-233).  For pipeline tours (valid by construction); the sequential
 * orc_list_ranking keeps the reference's error classification.
 */
int orc_list_ranking_par(int64_t L, const int32_t *nxt, int64_t nheads,
                         const int32_t *heads, int32_t *ranks) {
  if (L == 0) return ORC_OK;
  const int64_t S = 256;
  int32_t *sid = (int32_t *)malloc(sizeof(int32_t) * L);
  if (!sid) return ORC_ERR_NOMEM;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < L; i++) sid[i] = -1;
  /* splitter ids: regular cells first, then heads not already splitters */
  int64_t nreg = (L + S - 1) / S, ns = nreg;
  for (int64_t i = 0; i < nreg; i++) sid[i * S] = (int32_t)i;
  for (int64_t h = 0; h < nheads; h++)
    if (heads[h] >= 0 && sid[heads[h]] < 0) sid[heads[h]] = (int32_t)ns++;
  int32_t *scell = (int32_t *)malloc(sizeof(int32_t) * ns);
  int32_t *snext = (int32_t *)malloc(sizeof(int32_t) * ns); /* next splitter id, -1 = end */
  int64_t *slen = (int64_t *)malloc(sizeof(int64_t) * ns);
  int64_t *sbase = (int64_t *)malloc(sizeof(int64_t) * ns);
  if (!scell || !snext || !slen || !sbase) { free(sid); free(scell); free(snext); free(slen); free(sbase); return ORC_ERR_NOMEM; }
  for (int64_t i = 0; i < nreg; i++) scell[i] = (int32_t)(i * S);
  for (int64_t h = 0; h < nheads; h++)
    if (heads[h] >= 0 && sid[heads[h]] >= nreg) scell[sid[heads[h]]] = heads[h];
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad)
  for (int64_t j = 0; j < ns; j++) {
    int64_t c = scell[j], len = 1;
    int64_t x = nxt[c];
    while (x >= 0 && sid[x] < 0) {
      if (++len > L) { bad = 1; break; }
      x = nxt[x];
    }
    slen[j] = len;
    snext[j] = x >= 0 ? sid[x] : -1;
    sbase[j] = -1;
  }
  if (bad) { free(sid); free(scell); free(snext); free(slen); free(sbase); return ORC_ERR_CYCLE; }
  int64_t covered = 0;
  for (int64_t h = 0; h < nheads && !bad; h++) {
    if (heads[h] < 0) continue;
    int64_t j = sid[heads[h]], r = 0;
    while (j >= 0) {
      if (sbase[j] >= 0) { bad = 1; break; }
      sbase[j] = r;
      r += slen[j];
      covered += slen[j];
      j = snext[j];
    }
  }
  if (bad || covered != L) { free(sid); free(scell); free(snext); free(slen); free(sbase); return ORC_ERR_COVER; }
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < ns; j++) {
    int64_t c = scell[j], r = sbase[j];
    ranks[c] = (int32_t)r;
    int64_t x = nxt[c];
    while (x >= 0 && sid[x] < 0) { ranks[x] = (int32_t)++r; x = nxt[x]; }
  }
  free(sid); free(scell); free(snext); free(slen); free(sbase);
  return ORC_OK;
}

/*
 * Root a spanning forest at each component's minimum vertex
 * (_rooted_from_claims euler_tour.py:397-411 -> _rooted_from_csr 414-437).
 * Forest = k undirected pairs (forest_u[i], forest_v[i]); label = min-id
 * component labels.  Outputs parent (-1 at roots), first, last in [0, 2n).
 */
static int root_forest(int64_t n, const int32_t *label, int64_t k,
                       const int32_t *fu, const int32_t *fv, int32_t *parent,
                       int32_t *first, int32_t *last, int parallel);

int orc_root_forest(int64_t n, const int32_t *label, int64_t k,
                    const int32_t *fu, const int32_t *fv, int32_t *parent,
                    int32_t *first, int32_t *last) {
  return root_forest(n, label, k, fu, fv, parent, first, last, 0);
}

static int root_forest(int64_t n, const int32_t *label, int64_t k,
                       const int32_t *fu, const int32_t *fv, int32_t *parent,
                       int32_t *first, int32_t *last, int parallel) {
  if (n == 0) return ORC_OK;
  int64_t L = 2 * k;
  int64_t *toff = (int64_t *)calloc(n + 1, sizeof(int64_t));
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * n);
  int32_t *tedges = (int32_t *)malloc(sizeof(int32_t) * (L ? L : 1));
  int32_t *twin = (int32_t *)malloc(sizeof(int32_t) * (L ? L : 1));
  int32_t *nxt = (int32_t *)malloc(sizeof(int32_t) * (L ? L : 1));
  int32_t *ranks = (int32_t *)malloc(sizeof(int32_t) * (L ? L : 1));
  int32_t *heads = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *sizes = (int32_t *)calloc(n, sizeof(int32_t));
  int32_t *base = (int32_t *)calloc(n, sizeof(int32_t));
  int rc = ORC_OK;
  if (!toff || !cur || !tedges || !twin || !nxt || !ranks || !heads || !sizes || !base) {
    rc = ORC_ERR_NOMEM;
    goto done;
  }
  /* tree CSR by counting sort of directed slots (_tree_csr euler_tour.py:68-89) */
  if (parallel) {
    /* concurrent counting sort: slot order within a row differs, which only
       re-orders the Euler circuit -- positions stay a valid tour */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < k; i++) {
      __atomic_fetch_add(&toff[fu[i] + 1], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&toff[fv[i] + 1], 1, __ATOMIC_RELAXED);
    }
    for (int64_t v = 0; v < n; v++) { toff[v + 1] += toff[v]; cur[v] = toff[v]; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < k; i++) {
      int64_t su = __atomic_fetch_add(&cur[fu[i]], 1, __ATOMIC_RELAXED);
      int64_t sv = __atomic_fetch_add(&cur[fv[i]], 1, __ATOMIC_RELAXED);
      tedges[su] = fv[i]; tedges[sv] = fu[i];
      twin[su] = (int32_t)sv; twin[sv] = (int32_t)su;
    }
  } else {
    for (int64_t i = 0; i < k; i++) { toff[fu[i] + 1]++; toff[fv[i] + 1]++; }
    for (int64_t v = 0; v < n; v++) { toff[v + 1] += toff[v]; cur[v] = toff[v]; }
    for (int64_t i = 0; i < k; i++) {
      int64_t su = cur[fu[i]]++, sv = cur[fv[i]]++;
      tedges[su] = fv[i]; tedges[sv] = fu[i];
      twin[su] = (int32_t)sv; twin[sv] = (int32_t)su;
    }
  }
  /* Euler circuit: incoming slot i of v -> outgoing slot i+1 (_link_circuit :134-145) */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int64_t b = toff[v], d = toff[v + 1] - b;
    for (int64_t i = 0; i < d; i++) nxt[twin[b + i]] = (int32_t)(b + (i + 1) % d);
  }
  /* cut each circuit at its root (roots = label==v, :417-419; _cut_roots :148-158) */
  int64_t nroots = 0;
  for (int64_t r = 0; r < n; r++) {
    if (label[r] != r) continue;
    int64_t b = toff[r], d = toff[r + 1] - b;
    if (d == 0) heads[nroots++] = -1;
    else { nxt[twin[b + d - 1]] = -1; heads[nroots++] = (int32_t)b; }
  }
  rc = parallel ? orc_list_ranking_par(L, nxt, nroots, heads, ranks)
                : orc_list_ranking(L, nxt, nroots, heads, ranks);
  if (rc != ORC_OK) goto done;
  /* per-tree base = sum of 2*size over trees with smaller root (_tree_bases :250-259) */
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++) __atomic_fetch_add(&sizes[label[v]], 1, __ATOMIC_RELAXED);
  } else {
    for (int64_t v = 0; v < n; v++) sizes[label[v]]++;
  }
  {
    int64_t acc = 0;
    for (int64_t v = 0; v < n; v++)
      if (label[v] == v) { base[v] = (int32_t)acc; acc += 2 * (int64_t)sizes[v]; }
  }
  /* per-vertex gather (_vertex_positions :262-294) */
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t v = 0; v < n; v++) {
    int32_t r = label[v];
    if (r == v) {
      parent[v] = -1;
      first[v] = base[r];
      last[v] = base[r] + 2 * sizes[r] - 1;
      continue;
    }
    int64_t b = toff[v], d = toff[v + 1] - b;
    if (d == 0) { bad = 1; continue; }
    int32_t minin = 1 << 30, maxout = -1, par = -1;
    for (int64_t i = 0; i < d; i++) {
      int32_t rin = ranks[twin[b + i]], rout = ranks[b + i];
      if (rin < minin) { minin = rin; par = tedges[b + i]; }
      if (rout > maxout) maxout = rout;
    }
    parent[v] = par;
    first[v] = base[r] + 1 + minin;
    last[v] = base[r] + 1 + maxout;
  }
  if (bad) rc = ORC_ERR_LABELS;
done:
  free(toff); free(cur); free(tedges); free(twin); free(nxt); free(ranks);
  free(heads); free(sizes); free(base);
  return rc;
}

/* w1/w2 over the vertex and its non-forest edges (_w_gather tagging.py:101-119) */
void orc_compute_w(int64_t n, const int64_t *off, const uint32_t *adj,
                   const int32_t *parent, const int32_t *first, int32_t *w1,
                   int32_t *w2) {
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; v++) {
    int32_t a = first[v], b = first[v];
    for (int64_t s = off[v]; s < off[v + 1]; s++) {
      int64_t u = adj[s];
      if (parent[u] == v || parent[v] == u) continue; /* forest edge */
      int32_t f = first[u];
      if (f < a) a = f;
      if (f > b) b = f;
    }
    w1[v] = a;
    w2[v] = b;
  }
}

/*
 * low/high = min of w1 / max of w2 over the tour range [first[v], last[v]]
 * (compute_low_high tagging.py:270-297): a tour-position array holding
 * (w1, w2) at each vertex's entry slot and neutral fillers elsewhere
 * (_scatter_at_first :122-135), block extremes (:138-159), doubling tables
 * over blocks (:162-184) and boundary scans (_range_queries :187-242).
 */
int orc_low_high(int64_t n, const int32_t *first, const int32_t *last,
                 const int32_t *w1, const int32_t *w2, int64_t block,
                 int32_t *low, int32_t *high) {
  if (block < 2) return ORC_ERR_ARG;
  if (n == 0) return ORC_OK;
  const int32_t MINF = 0x7FFFFFFF, MAXF = -1;
  int64_t L = 2 * n, bs = block, nb = (L + bs - 1) / bs;
  int K = 0;
  while ((1LL << (K + 1)) <= (nb - 1 > 1 ? nb - 1 : 1)) K++;
  int32_t *amin = (int32_t *)malloc(sizeof(int32_t) * L);
  int32_t *amax = (int32_t *)malloc(sizeof(int32_t) * L);
  int32_t *tmin = (int32_t *)malloc(sizeof(int32_t) * nb * (K + 1));
  int32_t *tmax = (int32_t *)malloc(sizeof(int32_t) * nb * (K + 1));
  int32_t *logt = (int32_t *)malloc(sizeof(int32_t) * (nb + 1));
  if (!amin || !amax || !tmin || !tmax || !logt) {
    free(amin); free(amax); free(tmin); free(tmax); free(logt);
    return ORC_ERR_NOMEM;
  }
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < L; p++) { amin[p] = MINF; amax[p] = MAXF; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) { amin[first[v]] = w1[v]; amax[first[v]] = w2[v]; }
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; b++) {
    int64_t p0 = b * bs, p1 = p0 + bs < L ? p0 + bs : L;
    int32_t mn = amin[p0], mx = amax[p0];
    for (int64_t p = p0 + 1; p < p1; p++) {
      if (amin[p] < mn) mn = amin[p];
      if (amax[p] > mx) mx = amax[p];
    }
    tmin[b] = mn; tmax[b] = mx;
  }
  for (int k = 1; k <= K; k++) {
    int64_t w = 1LL << (k - 1), lim = nb - (1LL << k) + 1;
    int32_t *pm = tmin + (k - 1) * nb, *px = tmax + (k - 1) * nb;
    int32_t *cm = tmin + k * nb, *cx = tmax + k * nb;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nb; i++) {
      if (i < lim) {
        cm[i] = pm[i] < pm[i + w] ? pm[i] : pm[i + w];
        cx[i] = px[i] > px[i + w] ? px[i] : px[i + w];
      } else {
        cm[i] = pm[i]; cx[i] = px[i];
      }
    }
  }
  logt[0] = 0;
  if (nb >= 1) logt[1] = 0;
  for (int64_t i = 2; i <= nb; i++) logt[i] = logt[i >> 1] + 1;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int64_t lo = first[v], hi = last[v], blo = lo / bs, bhi = hi / bs;
    int32_t mn = MINF, mx = MAXF;
    if (blo == bhi) {
      for (int64_t p = lo; p <= hi; p++) {
        if (amin[p] < mn) mn = amin[p];
        if (amax[p] > mx) mx = amax[p];
      }
    } else {
      for (int64_t p = lo; p < (blo + 1) * bs; p++) {
        if (amin[p] < mn) mn = amin[p];
        if (amax[p] > mx) mx = amax[p];
      }
      for (int64_t p = bhi * bs; p <= hi; p++) {
        if (amin[p] < mn) mn = amin[p];
        if (amax[p] > mx) mx = amax[p];
      }
      int64_t cnt = bhi - blo - 1;
      if (cnt > 0) {
        int k = logt[cnt];
        int64_t i0 = blo + 1, i1 = bhi - (1LL << k);
        int32_t a = tmin[k * nb + i0], b = tmin[k * nb + i1];
        int32_t t = a < b ? a : b;
        if (t < mn) mn = t;
        a = tmax[k * nb + i0]; b = tmax[k * nb + i1];
        t = a > b ? a : b;
        if (t > mx) mx = t;
      }
    }
    low[v] = mn;
    high[v] = mx;
  }
  free(amin); free(amax); free(tmin); free(tmax); free(logt);
  return ORC_OK;
}

/* packed skeleton record (_pack_skeleton connectivity.py:84-96) */
void orc_pack_skeleton(int64_t n, const int32_t *parent, const int32_t *first,
                       const int32_t *last, const int32_t *low,
                       const int32_t *high, int64_t *skel) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    skel[2 * v] = ((int64_t)first[v] << 32) | (int64_t)(uint32_t)last[v];
    int64_t p = parent[v], fence = 0;
    if (p >= 0 && low[v] >= first[p] && high[v] <= last[p]) fence = 1;
    skel[2 * v + 1] = ((p + 1) << 1) | fence;
  }
}

/* head[l] = parent of the shallowest member of label l (_component_heads bcc.py:129-144) */
void orc_component_heads(int64_t n, const int32_t *label, const int32_t *parent,
                         const int32_t *first, int32_t *head) {
  int64_t *best = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
  const int64_t BIG = (int64_t)1 << 62;
  for (int64_t l = 0; l < n; l++) { best[l] = BIG; head[l] = -1; }
  for (int64_t v = 0; v < n; v++) {
    int64_t pk = ((int64_t)first[v] << 32) | v;
    if (pk < best[label[v]]) best[label[v]] = pk;
  }
  for (int64_t l = 0; l < n; l++)
    if (best[l] != BIG) head[l] = parent[best[l] & 0xFFFFFFFFLL];
  free(best);
}

/* articulation flags (articulation_points bcc.py:222-235) */
void orc_articulation(int64_t n, const int32_t *label, const int32_t *head,
                      uint8_t *is_ap) {
  int32_t *headed = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
  for (int64_t l = 0; l < n; l++)
    if (head[l] != -1) headed[head[l]]++;
  for (int64_t v = 0; v < n; v++) {
    int root = (label[v] == v) && (head[v] == -1);
    is_ap[v] = (uint8_t)(root ? headed[v] >= 2 : headed[v] >= 1);
  }
  free(headed);
}

/*
 * Per-edge block labels.  No reference function emits them from fast_bcc;
 * the rule is the module docstring bcc.py:24-27 and the canonical numbering
 * (edge id = rank of arc u->v, u<v, in CSR order; block label = min edge id
 * in the block) is that of tv_skeleton (baselines.py:251-257, 297-303).
 * Returns the number of undirected edges E.
 */
int64_t orc_edge_labels(int64_t n, const int64_t *off, const uint32_t *adj,
                        const int32_t *label, const int32_t *head,
                        int32_t *edge_label) {
  int32_t *bmin = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  for (int64_t v = 0; v < n; v++) bmin[v] = 0x7FFFFFFF;
  int64_t e = 0;
  for (int64_t u = 0; u < n; u++) {
    for (int64_t s = off[u]; s < off[u + 1]; s++) {
      int64_t w = adj[s];
      if (w <= u) continue;
      int32_t lu = label[u], lw = label[w];
      int32_t blk = (lu == lw) ? lu : (head[lw] == u ? lw : lu);
      edge_label[e] = blk;
      if (e < bmin[blk]) bmin[blk] = (int32_t)e;
      e++;
    }
  }
  for (int64_t i = 0; i < e; i++) edge_label[i] = bmin[edge_label[i]];
  free(bmin);
  return e;
}

/* parallel mode: _component_heads by an atomic min of (first << 32 | v) per label */
static void component_heads_par(int64_t n, const int32_t *label, const int32_t *parent,
                                const int32_t *first, int32_t *head) {
  int64_t *best = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
  const int64_t BIG = (int64_t)1 << 62;
#pragma omp parallel for schedule(static)
  for (int64_t l = 0; l < n; l++) { best[l] = BIG; head[l] = -1; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int64_t pk = ((int64_t)first[v] << 32) | v, cur = __atomic_load_n(&best[label[v]], __ATOMIC_RELAXED);
    while (pk < cur && !__atomic_compare_exchange_n(&best[label[v]], &cur, pk, 1, __ATOMIC_RELAXED,
                                                     __ATOMIC_RELAXED)) {
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t l = 0; l < n; l++)
    if (best[l] != BIG) head[l] = parent[best[l] & 0xFFFFFFFFLL];
  free(best);
}

static void articulation_par(int64_t n, const int32_t *label, const int32_t *head, uint8_t *is_ap) {
  int32_t *headed = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
#pragma omp parallel for schedule(static)
  for (int64_t l = 0; l < n; l++)
    if (head[l] != -1) __atomic_fetch_add(&headed[head[l]], 1, __ATOMIC_RELAXED);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int root = (label[v] == v) && (head[v] == -1);
    is_ap[v] = (uint8_t)(root ? headed[v] >= 2 : headed[v] >= 1);
  }
  free(headed);
}

/* orc_edge_labels with edge ids from a prefix of per-row upper-arc counts */
static int64_t edge_labels_par(int64_t n, const int64_t *off, const uint32_t *adj, const int32_t *label,
                               const int32_t *head, int32_t *edge_label) {
  int32_t *bmin = (int32_t *)malloc(sizeof(int32_t) * (n ? n : 1));
  int64_t *ebase = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; u++) {
    bmin[u] = 0x7FFFFFFF;
    /* rows are sorted: the upper arcs are the tail after the last target <= u */
    int64_t lo = off[u], hi = off[u + 1];
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (adj[mid] <= u) lo = mid + 1; else hi = mid;
    }
    ebase[u + 1] = off[u + 1] - lo;
  }
  ebase[0] = 0;
  for (int64_t u = 0; u < n; u++) ebase[u + 1] += ebase[u];
  const int64_t E = ebase[n];
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t u = 0; u < n; u++) {
    int64_t e = ebase[u], s0 = off[u + 1] - (ebase[u + 1] - ebase[u]);
    for (int64_t s = s0; s < off[u + 1]; s++, e++) {
      int64_t w = adj[s];
      int32_t lu = label[u], lw = label[w];
      int32_t blk = (lu == lw) ? lu : (head[lw] == u ? lw : lu);
      edge_label[e] = blk;
      int32_t cur = __atomic_load_n(&bmin[blk], __ATOMIC_RELAXED);
      while (e < cur && !__atomic_compare_exchange_n(&bmin[blk], &cur, (int32_t)e, 1, __ATOMIC_RELAXED,
                                                      __ATOMIC_RELAXED)) {
      }
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < E; i++) edge_label[i] = bmin[edge_label[i]];
  free(bmin);
  free(ebase);
  return E;
}

/*
 * The whole pipeline (fast_bcc bcc.py:147-196) plus the derived outputs.
 * label/head/is_ap sized n; edge_label sized E (may be NULL).
 * out_counts[0] = num_bccs, [1] = num_components, [2] = E.
 * seconds[0..4] = first_cc, rooting, tagging, last_cc, labelling (may be NULL).
 */
int orc_fast_bcc_mode(int64_t n, const int64_t *off, const uint32_t *adj,
                      int32_t *label, int32_t *head, uint8_t *is_ap,
                      int32_t *edge_label, int64_t *out_counts, double *seconds, int parallel);

int orc_fast_bcc(int64_t n, const int64_t *off, const uint32_t *adj,
                 int32_t *label, int32_t *head, uint8_t *is_ap,
                 int32_t *edge_label, int64_t *out_counts, double *seconds) {
  return orc_fast_bcc_mode(n, off, adj, label, head, is_ap, edge_label, out_counts, seconds, 0);
}

/* parallel != 0: the parallel variants above (same outputs, all host cores) */
int orc_fast_bcc_mode(int64_t n, const int64_t *off, const uint32_t *adj,
                      int32_t *label, int32_t *head, uint8_t *is_ap,
                      int32_t *edge_label, int64_t *out_counts, double *seconds, int parallel) {
  out_counts[0] = out_counts[1] = out_counts[2] = 0;
  if (n == 0) return ORC_OK;
  int rc = ORC_OK;
  int32_t *lab1 = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *fu = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *fv = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *first = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *last = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *w1 = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *w2 = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *low = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *high = (int32_t *)malloc(sizeof(int32_t) * n);
  int64_t *skel = (int64_t *)malloc(sizeof(int64_t) * 2 * n);
  if (!lab1 || !fu || !fv || !parent || !first || !last || !w1 || !w2 ||
      !low || !high || !skel) { rc = ORC_ERR_NOMEM; goto done; }
  {
    double t0 = 0, t1 = 0;
#ifdef _OPENMP
#define NOW() omp_get_wtime()
#else
#define NOW() 0.0
#endif
    t0 = NOW();
    int64_t k = 0;
    int64_t ncomp = parallel ? orc_cc_par(n, off, adj, NULL, lab1, fu, fv, &k)
                             : orc_cc(n, off, adj, NULL, NULL, lab1, fu, fv, &k);
    if (ncomp < 0) { rc = ORC_ERR_NOMEM; goto done; }
    t1 = NOW(); if (seconds) seconds[0] = t1 - t0; t0 = t1;
    rc = root_forest(n, lab1, k, fu, fv, parent, first, last, parallel);
    if (rc != ORC_OK) goto done;
    t1 = NOW(); if (seconds) seconds[1] = t1 - t0; t0 = t1;
    orc_compute_w(n, off, adj, parent, first, w1, w2);
    rc = orc_low_high(n, first, last, w1, w2, 16, low, high);
    if (rc != ORC_OK) goto done;
    t1 = NOW(); if (seconds) seconds[2] = t1 - t0; t0 = t1;
    orc_pack_skeleton(n, parent, first, last, low, high, skel);
    if (parallel) {
      if (orc_cc_par(n, off, adj, skel, label, NULL, NULL, NULL) < 0) { rc = ORC_ERR_NOMEM; goto done; }
      component_heads_par(n, label, parent, first, head);
    } else {
      orc_cc(n, off, adj, NULL, skel, label, NULL, NULL, NULL);
      orc_component_heads(n, label, parent, first, head);
    }
    int64_t nb = 0;
#pragma omp parallel for schedule(static) reduction(+ : nb)
    for (int64_t l = 0; l < n; l++) nb += head[l] != -1;
    t1 = NOW(); if (seconds) seconds[3] = t1 - t0; t0 = t1;
    if (is_ap) {
      if (parallel) articulation_par(n, label, head, is_ap);
      else orc_articulation(n, label, head, is_ap);
    }
    int64_t E = 0;
    if (edge_label) E = parallel ? edge_labels_par(n, off, adj, label, head, edge_label)
                                 : orc_edge_labels(n, off, adj, label, head, edge_label);
    else E = off[n] / 2;
    t1 = NOW(); if (seconds) seconds[4] = t1 - t0;
    out_counts[0] = nb;
    out_counts[1] = ncomp;
    out_counts[2] = E;
  }
done:
  free(lab1); free(fu); free(fv); free(parent); free(first); free(last);
  free(w1); free(w2); free(low); free(high); free(skel);
  return rc;
}
