/*
 * hostgen.c -- seeded synthetic inputs on the host (bench/test harness; not
 * product code, not the oracle).
 *
 * Config 5 (RMAT scale 25, edge factor 16) is 5.4e8 pairs and a 4.3 GB CSR.
 * numpy needs minutes for it (404 s); this builds the same CSR
 * in seconds on the host cores so that both bench arms start from a host CSR
 * within the driver's time limits.  Bit-identity with workloads.rmat() /
 * graphs.symmetrize() is asserted by sha256 (tests/test_hostgen.py at small
 * scales, the committed config digests at full size).
 *
 *   hg_rmat_pairs: the RMAT pairs of workloads._rmat_pairs -- numpy
 *     Generator(PCG64(seed)).random(k) draws, chunk-major then level-major,
 *     reached per thread by the O(log j) LCG jump-ahead.  numpy's PCG64 is
 *     PCG XSL-RR 128/64: state = state * MULT + inc, output
 *     rotr64(hi ^ lo, hi >> 58) of the new state; random() = (out >> 11) * 2^-53.
 *   hg_symmetrize: symmetrize() (graphs.py:119-143): both directions, no
 *     self-loops, rows sorted, duplicates removed -- by degree count, scatter,
 *     per-row sort + unique, compaction (OpenMP).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#define HG_T() omp_get_wtime()
#else
#define HG_T() 0.0
#endif

typedef unsigned __int128 u128;

static const u128 kMult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;

/* (a, b, c, d) = (0.57, 0.19, 0.19, 0.05), cumulative 0.57 / 0.76 / 0.95:
   quadrant c|d sets the row bit, b|d the column bit.  Thresholds on the
   53-bit draw m: ceil(c * 2^53) (c * 2^53 is an exact double). */
static uint64_t ceil53(double c) {
  const double x = c * 9007199254740992.0;
  uint64_t t = (uint64_t)x;
  return (double)t < x ? t + 1 : t;
}

static u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_m = 1, acc_p = 0, cur_m = kMult, cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  return acc_m * s + acc_p;
}

static inline uint64_t pcg_out(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64 - r) & 63));
}

int hg_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* u[i], v[i] for i < total = edge_factor << scale; chunk = edges per numpy call */
int hg_rmat_pairs(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int scale, int64_t total,
                  int64_t chunk, uint32_t *u, uint32_t *v) {
  const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
  if (scale < 1 || scale > 31 || total < 0 || chunk < 1) return 1;
  const uint64_t kT57 = ceil53(0.57), kT76 = ceil53(0.76), kT95 = ceil53(0.95);
  for (int64_t done = 0; done < total; done += chunk) {
    const int64_t k = total - done < chunk ? total - done : chunk;
    const uint64_t base = (uint64_t)done * (uint64_t)scale; /* draws consumed before this chunk */
#pragma omp parallel
    {
      int nt = 1, t = 0;
#ifdef _OPENMP
      nt = omp_get_num_threads();
      t = omp_get_thread_num();
#endif
      const int64_t i0 = k * t / nt, i1 = k * (t + 1) / nt;
      /* one generator per level, each at this thread's first element: draw
         (lvl, i) of the chunk is stream position base + lvl*k + i */
      u128 s[32];
      for (int lvl = 0; lvl < scale && i1 > i0; lvl++)
        s[lvl] = pcg_advance(s0, inc, base + (uint64_t)lvl * (uint64_t)k + (uint64_t)i0);
      for (int64_t i = i0; i < i1; i++) {
        uint32_t a = 0, b = 0;
        for (int lvl = 0; lvl < scale; lvl++) {
          s[lvl] = s[lvl] * kMult + inc;
          /* r = m * 2^-53 exactly, so r >= c  <=>  m >= ceil(c * 2^53) (branch-free) */
          const uint64_t m = pcg_out(s[lvl]) >> 11;
          const uint32_t row = m >= kT76, col = (uint32_t)(m >= kT57) ^ row ^ (uint32_t)(m >= kT95);
          a |= row << (scale - 1 - lvl);
          b |= col << (scale - 1 - lvl);
        }
        u[done + i] = a;
        v[done + i] = b;
      }
    }
  }
  return 0;
}

static void isort(uint32_t *a, int64_t n) {
  for (int64_t i = 1; i < n; i++) {
    uint32_t x = a[i];
    int64_t j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      j--;
    }
    a[j + 1] = x;
  }
}

static void qsort_u32(uint32_t *a, int64_t n) {
  while (n > 24) {
    /* median of three */
    uint32_t x = a[0], y = a[n / 2], z = a[n - 1];
    uint32_t p = x < y ? (y < z ? y : (x < z ? z : x)) : (x < z ? x : (y < z ? z : y));
    int64_t i = 0, j = n - 1;
    while (i <= j) {
      while (a[i] < p) i++;
      while (a[j] > p) j--;
      if (i <= j) {
        uint32_t t = a[i];
        a[i] = a[j];
        a[j] = t;
        i++;
        j--;
      }
    }
    /* recurse into the smaller side */
    if (j + 1 < n - i) {
      qsort_u32(a, j + 1);
      a += i;
      n -= i;
    } else {
      qsort_u32(a + i, n - i);
      n = j + 1;
    }
  }
  isort(a, n);
}

/* first row r with off[r] >= target (rows 0..n) */
static int64_t row_at(const int64_t *off, int64_t n, int64_t target) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (off[mid] < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/*
 * k pairs (u[i], v[i]) with ids < n  ->  CSR (offsets int64[n+1], edges
 * uint32[m]) in malloc'd buffers (hg_free).  Returns m, or -1 on a bad id /
 * allocation failure.
 *
 * No atomics: every thread streams the whole pair list and updates only the
 * rows it owns (vertex ranges for the degree count, arc-balanced row ranges
 * for the scatter), so the random counter updates never contend or lock.
 */
int64_t hg_symmetrize(const uint32_t *u, const uint32_t *v, int64_t k, int64_t n, int64_t **off_out,
                      uint32_t **edges_out) {
  *off_out = NULL;
  *edges_out = NULL;
  const int verbose = getenv("HG_VERBOSE") != NULL;
  double t0 = HG_T();
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < k; i++) bad |= (u[i] >= n) | (v[i] >= n);
  if (bad) return -1;
  int64_t *off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
  if (!off || !cur) {
    free(off);
    free(cur);
    return -1;
  }
  /* degrees (both directions, self-loops dropped); thread t counts rows [lo, hi) */
#pragma omp parallel
  {
    int nt = 1, t = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    t = omp_get_thread_num();
#endif
    const uint32_t lo = (uint32_t)(n * t / nt), hi = (uint32_t)(n * (t + 1) / nt);
    int64_t *d = off + 1;
    for (int64_t i = 0; i < k; i++) {
      const uint32_t a = u[i], b = v[i];
      if (a == b) continue;
      if (a - lo < hi - lo) d[a]++;
      if (b - lo < hi - lo) d[b]++;
    }
  }
  for (int64_t x = 0; x < n; x++) off[x + 1] += off[x];
  const int64_t tot = off[n];
  uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(tot ? tot : 1));
  if (!tmp) {
    free(off);
    free(cur);
    return -1;
  }
  memcpy(cur, off, sizeof(int64_t) * ((size_t)n + 1));
  if (verbose) fprintf(stderr, "hg_symmetrize: degrees %.2fs\n", HG_T() - t0);
  /* scatter; thread t fills rows [r0, r1), about tot/nt slots */
#pragma omp parallel
  {
    int nt = 1, t = 0;
#ifdef _OPENMP
    nt = omp_get_num_threads();
    t = omp_get_thread_num();
#endif
    const uint32_t lo = (uint32_t)row_at(off, n, tot * t / nt);
    const uint32_t hi = (uint32_t)(t == nt - 1 ? n : row_at(off, n, tot * (t + 1) / nt));
    for (int64_t i = 0; i < k; i++) {
      const uint32_t a = u[i], b = v[i];
      if (a == b) continue;
      if (a - lo < hi - lo) tmp[cur[a]++] = b;
      if (b - lo < hi - lo) tmp[cur[b]++] = a;
    }
  }
  if (verbose) fprintf(stderr, "hg_symmetrize: scatter %.2fs\n", HG_T() - t0);
  /* per-row sort + unique; cur[x] = unique count of row x */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t x = 0; x < n; x++) {
    uint32_t *r = tmp + off[x];
    const int64_t d = off[x + 1] - off[x];
    if (d > 1) qsort_u32(r, d);
    int64_t w = d ? 1 : 0;
    for (int64_t j = 1; j < d; j++)
      if (r[j] != r[w - 1]) r[w++] = r[j];
    cur[x] = w;
  }
  if (verbose) fprintf(stderr, "hg_symmetrize: sort %.2fs\n", HG_T() - t0);
  int64_t *noff = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
  if (!noff) {
    free(off);
    free(cur);
    free(tmp);
    return -1;
  }
  noff[0] = 0;
  for (int64_t x = 0; x < n; x++) noff[x + 1] = noff[x] + cur[x];
  const int64_t m = noff[n];
  uint32_t *edges = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
  if (!edges) {
    free(off);
    free(cur);
    free(tmp);
    free(noff);
    return -1;
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t x = 0; x < n; x++) memcpy(edges + noff[x], tmp + off[x], sizeof(uint32_t) * (size_t)cur[x]);
  free(off);
  free(cur);
  free(tmp);
  *off_out = noff;
  *edges_out = edges;
  return m;
}

void hg_free(void *p) { free(p); }
