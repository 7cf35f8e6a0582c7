/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * (`lanebfs` 0.1.0, /root/reference/pkg/src/lanebfs) for the BFS hot path and
 * the graph inputs it consumes. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or as the timed CPU baseline — never as the product.
 *
 * Parity pin: every function here is checked against golden vectors produced
 * by the reference itself (tests/golden/make_golden.py, committed fixtures in
 * tests/golden/) by tests/test_oracle.py.
 *
 *   oracle_rmat_edges    <- generate_rmat            graph.py:68-85
 *   oracle_permute_edges <- (build-defined permutation, gap G1)
 *   oracle_build_csr     <- build_csr                graph.py:139-160
 *   oracle_lattice_edges <- (config 4; gap G3)
 *   oracle_bfs_serial    <- bfs_serial               traversal.py:80-104
 *   oracle_bfs_parallel  <- bfs_parallel_naive       traversal.py:128-165
 *   oracle_check_bfs     <- BFS certificate (validate.py:50-155 is a subset)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define SENTINEL 0x7FFFFFFF

typedef unsigned __int128 u128;

/* ---------------- numpy PCG64 (XSL-RR 128/64) --------------------------- */
/* numpy Generator.random(): next_double = (next_uint64 >> 11) * 2^-53 where
 * next_uint64 steps the 128-bit LCG first, then applies XSL-RR. */
static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static inline uint64_t pcg_output(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

/* state after `delta` LCG steps (Brown's jump-ahead). */
static u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

static inline double pcg_double(u128* s, u128 inc) {
  *s = *s * PCG_MULT + inc;
  return (double)(pcg_output(*s) >> 11) * (1.0 / 9007199254740992.0);
}

/* generate_rmat (graph.py:68-85): for each address bit, one array of m draws
 * decides the source half (draw > ab), a second array of m draws decides the
 * destination half against a_norm or c_norm. Draw k of array j is stream
 * position j*m + k. Parallel over element chunks with jump-ahead. */
void oracle_rmat_edges(int scale, int64_t m, double ab, double a_norm, double c_norm,
                       const uint64_t pcg[4], uint32_t* src, uint32_t* dst) {
  const u128 s0 = (((u128)pcg[0]) << 64) | pcg[1];
  const u128 inc = (((u128)pcg[2]) << 64) | pcg[3];
  const int64_t CH = 4096;
  const int64_t nch = (m + CH - 1) / CH;
#pragma omp parallel
  {
    uint8_t ii[4096];
#pragma omp for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
      const int64_t lo = c * CH, hi = (lo + CH < m) ? lo + CH : m;
      for (int64_t i = lo; i < hi; ++i) src[i] = dst[i] = 0;
      for (int b = 0; b < scale; ++b) {
        u128 s = pcg_advance(s0, inc, (uint64_t)(2 * b) * (uint64_t)m + (uint64_t)lo);
        for (int64_t i = lo; i < hi; ++i) {
          ii[i - lo] = pcg_double(&s, inc) > ab;
        }
        s = pcg_advance(s0, inc, (uint64_t)(2 * b + 1) * (uint64_t)m + (uint64_t)lo);
        for (int64_t i = lo; i < hi; ++i) {
          const double thr = ii[i - lo] ? c_norm : a_norm;
          const uint32_t jj = pcg_double(&s, inc) > thr;
          src[i] |= (uint32_t)ii[i - lo] << b;
          dst[i] |= jj << b;
        }
      }
    }
  }
}

/* ---------------- seeded vertex permutation (build-defined) ------------- */
/* 4-round balanced Feistel network over 2*half bits, keys from splitmix64,
 * cycle-walked into [0, n). Restated identically in csrc/construct.cu. */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key[4];
  uint64_t mask;
  int half;
  uint64_t n;
} feistel_t;

static void feistel_init(feistel_t* f, uint64_t n, uint64_t seed) {
  int bits = 0;
  while (bits < 62 && ((uint64_t)1 << bits) < n) ++bits;
  if (bits < 2) bits = 2;
  if (bits & 1) ++bits;
  f->half = bits / 2;
  f->mask = ((uint64_t)1 << f->half) - 1;
  f->n = n;
  uint64_t st = seed ^ 0x6C616E6562667331ULL; /* "lanebfs1" */
  for (int r = 0; r < 4; ++r) {
    st += 0x9E3779B97F4A7C15ULL;
    f->key[r] = mix64(st);
  }
}

static inline uint64_t feistel_apply(const feistel_t* f, uint64_t x) {
  do {
    uint64_t L = x >> f->half, R = x & f->mask;
    for (int r = 0; r < 4; ++r) {
      uint64_t t = L ^ (mix64(R ^ f->key[r]) & f->mask);
      L = R;
      R = t;
    }
    x = (L << f->half) | R;
  } while (x >= f->n);
  return x;
}

uint64_t oracle_permute_vertex(uint64_t n, uint64_t seed, uint64_t v) {
  feistel_t f;
  feistel_init(&f, n, seed);
  return feistel_apply(&f, v);
}

void oracle_permute_edges(int64_t n, uint64_t seed, uint32_t* src, uint32_t* dst, int64_t m) {
  feistel_t f;
  feistel_init(&f, (uint64_t)n, seed);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    src[i] = (uint32_t)feistel_apply(&f, src[i]);
    dst[i] = (uint32_t)feistel_apply(&f, dst[i]);
  }
}

/* ---------------- lattice (config 4) ------------------------------------ */
/* vertex (r,c) -> r*cols + c; one pair to the right, one down; no wrap.
 * Pair order: row-major over vertices, right edge before down edge. */
int64_t oracle_lattice_edges(int64_t rows, int64_t cols, uint32_t* src, uint32_t* dst) {
  int64_t k = 0;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const int64_t v = r * cols + c;
      if (c + 1 < cols) { src[k] = (uint32_t)v; dst[k] = (uint32_t)(v + 1); ++k; }
      if (r + 1 < rows) { src[k] = (uint32_t)v; dst[k] = (uint32_t)(v + cols); ++k; }
    }
  return k;
}

/* ---------------- build_csr (graph.py:139-160) -------------------------- */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Pass 1: count (returns nnz upper bound). Caller allocates col_idx of that
 * size, then calls oracle_build_csr_fill which returns the final nnz. */
int64_t oracle_build_csr_count(int64_t n, const uint32_t* src, const uint32_t* dst, int64_t m,
                               int symmetrize, int dedup, int64_t* row_ptr) {
  memset(row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < m; ++i) {
    if (dedup && src[i] == dst[i]) continue;
    row_ptr[src[i] + 1]++;
    if (symmetrize) row_ptr[dst[i] + 1]++;
  }
  for (int64_t u = 0; u < n; ++u) row_ptr[u + 1] += row_ptr[u];
  return row_ptr[n];
}

/* Stable placement in the order of the concatenated [forward, reverse] pair
 * list (the reference's np.concatenate + stable argsort), then, with dedup,
 * per-row sort + unique and compaction. */
int64_t oracle_build_csr_fill(int64_t n, const uint32_t* src, const uint32_t* dst, int64_t m,
                              int symmetrize, int dedup, int64_t* row_ptr, int32_t* col_idx) {
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  memcpy(cur, row_ptr, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < m; ++i) {
    if (dedup && src[i] == dst[i]) continue;
    col_idx[cur[src[i]]++] = (int32_t)dst[i];
  }
  if (symmetrize)
    for (int64_t i = 0; i < m; ++i) {
      if (dedup && src[i] == dst[i]) continue;
      col_idx[cur[dst[i]]++] = (int32_t)src[i];
    }
  free(cur);
  if (!dedup) return row_ptr[n];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) {
    const int64_t lo = row_ptr[u], hi = row_ptr[u + 1];
    if (hi - lo > 1) qsort(col_idx + lo, (size_t)(hi - lo), sizeof(int32_t), cmp_i32);
  }
  int64_t w = 0;
  int64_t prev_lo = 0;
  for (int64_t u = 0; u < n; ++u) {
    const int64_t lo = prev_lo, hi = row_ptr[u + 1];
    prev_lo = hi;
    row_ptr[u] = w;
    for (int64_t j = lo; j < hi; ++j)
      if (j == lo || col_idx[j] != col_idx[j - 1]) col_idx[w++] = col_idx[j];
  }
  row_ptr[n] = w;
  return w;
}

/* ---------------- bfs_serial (traversal.py:80-104) ---------------------- */
/* Queue BFS; parent = first discoverer in queue order (neighbours in CSR
 * order). pred has n entries (caller pads). layers: 3 int64 per layer
 * (input, edges, discovered), including the last frontier (discovered 0).
 * Returns the number of layers (may exceed layers_cap; extra not stored). */
int64_t oracle_bfs_serial(int64_t n, const int64_t* rp, const int32_t* ci, int64_t root,
                          int32_t* pred, int32_t* level, int64_t* layers, int64_t layers_cap) {
  for (int64_t v = 0; v < n; ++v) { pred[v] = SENTINEL; level[v] = -1; }
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  pred[root] = (int32_t)root;
  level[root] = 0;
  q[0] = (int32_t)root;
  int64_t head = 0, tail = 1, nl = 0;
  int32_t L = 0;
  while (head < tail) {
    const int64_t end = tail;
    int64_t edges = 0;
    for (int64_t i = head; i < end; ++i) {
      const int32_t u = q[i];
      edges += rp[u + 1] - rp[u];
      for (int64_t j = rp[u]; j < rp[u + 1]; ++j) {
        const int32_t v = ci[j];
        if (pred[v] == SENTINEL) {
          pred[v] = u;
          level[v] = L + 1;
          q[tail++] = v;
        }
      }
    }
    if (nl < layers_cap) {
      layers[3 * nl] = end - head;
      layers[3 * nl + 1] = edges;
      layers[3 * nl + 2] = tail - end;
    }
    ++nl;
    head = end;
    ++L;
  }
  free(q);
  return nl;
}

/* ---------------- bfs_parallel_naive (traversal.py:128-165) ------------- */
/* Layer-synchronous BFS over all host threads: the frontier is split across
 * threads (the reference's array_split + thread pool), neighbours whose level
 * is unset are claimed (compare-and-swap instead of the reference's last-
 * writer pred scatter + np.unique merge: same layers and levels, a valid
 * equal-level parent), per-thread discoveries are concatenated as the next
 * frontier. nthreads <= 0 uses all. Returns the number of layers. */
int64_t oracle_bfs_parallel(int64_t n, const int64_t* rp, const int32_t* ci, int64_t root,
                            int32_t* pred, int32_t* level, int64_t* layers, int64_t layers_cap,
                            int nthreads) {
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int64_t v = 0; v < n; ++v) { pred[v] = SENTINEL; level[v] = -1; }
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* nxt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* off = (int64_t*)calloc((size_t)nthreads + 1, sizeof(int64_t));
  int32_t** loc = (int32_t**)calloc((size_t)nthreads, sizeof(int32_t*));
  int64_t* cap = (int64_t*)calloc((size_t)nthreads, sizeof(int64_t));
  pred[root] = (int32_t)root;
  level[root] = 0;
  cur[0] = (int32_t)root;
  int64_t fsize = 1, nl = 0;
  int32_t L = 0;
  while (fsize > 0) {
    int64_t edges = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : edges)
    {
      const int t = omp_get_thread_num();
      int64_t cnt = 0;
#pragma omp for schedule(dynamic, 64)
      for (int64_t i = 0; i < fsize; ++i) {
        const int32_t u = cur[i];
        const int64_t lo = rp[u], hi = rp[u + 1];
        edges += hi - lo;
        for (int64_t j = lo; j < hi; ++j) {
          const int32_t v = ci[j];
          if (__atomic_load_n(&level[v], __ATOMIC_RELAXED) != -1) continue;
          int32_t expect = -1;
          if (__atomic_compare_exchange_n(&level[v], &expect, L + 1, 0, __ATOMIC_RELAXED,
                                          __ATOMIC_RELAXED)) {
            pred[v] = u;
            if (cnt == cap[t]) {
              cap[t] = cap[t] ? 2 * cap[t] : 4096;
              loc[t] = (int32_t*)realloc(loc[t], sizeof(int32_t) * (size_t)cap[t]);
            }
            loc[t][cnt++] = v;
          }
        }
      }
      off[t + 1] = cnt;
#pragma omp barrier
#pragma omp single
      {
        for (int k = 0; k < nthreads; ++k) off[k + 1] += off[k];
      }
      memcpy(nxt + off[t], loc[t], sizeof(int32_t) * (size_t)cnt);
    }
    const int64_t disc = off[nthreads];
    if (nl < layers_cap) {
      layers[3 * nl] = fsize;
      layers[3 * nl + 1] = edges;
      layers[3 * nl + 2] = disc;
    }
    ++nl;
    int32_t* t = cur; cur = nxt; nxt = t;
    fsize = disc;
    memset(off, 0, sizeof(int64_t) * ((size_t)nthreads + 1));
    ++L;
  }
  for (int k = 0; k < nthreads; ++k) free(loc[k]);
  free(loc); free(cap); free(off); free(cur); free(nxt);
  return nl;
}

/* ---------------- BFS certificate --------------------------------------- */
/* Returns 0 when (pred, level) is a BFS of root; otherwise a positive code
 * and the first offending vertex in *where:
 *   1 root: level[root] != 0 or pred[root] != root
 *   2 unreached vertex with pred != SENTINEL, or reached with pred == SENTINEL
 *   3 parent out of range
 *   4 parent not one level up
 *   5 tree edge (pred[v], v) absent from the graph
 *   6 edge with exactly one endpoint reached
 *   7 edge spanning more than one level
 * (1)-(5) are the north_star tree check; (6)-(7) make the levels exact BFS
 * distances. Rows are assumed sorted (build_csr with dedup) for (5). */
static int row_has(const int64_t* rp, const int32_t* ci, int32_t u, int32_t v) {
  int64_t lo = rp[u], hi = rp[u + 1];
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (ci[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo < rp[u + 1] && ci[lo] == v;
}

int oracle_check_bfs(int64_t n, const int64_t* rp, const int32_t* ci, int64_t root,
                     const int32_t* pred, const int32_t* level, int64_t* where) {
  *where = -1;
  if (level[root] != 0 || pred[root] != (int32_t)root) { *where = root; return 1; }
  int code = 0;
  int64_t first = n;
#pragma omp parallel for schedule(dynamic, 4096) reduction(min : first)
  for (int64_t v = 0; v < n; ++v) {
    if (v >= first) continue;
    const int32_t lv = level[v];
    const int32_t p = pred[v];
    int bad = 0;
    if ((lv < 0) != (p == SENTINEL)) bad = 2;
    else if (lv > 0) {
      if (p < 0 || p >= n) bad = 3;
      else if (level[p] != lv - 1) bad = 4;
      else if (!row_has(rp, ci, p, (int32_t)v)) bad = 5;
    } else if (lv == 0 && v != root) bad = 4;
    if (!bad)
      for (int64_t j = rp[v]; j < rp[v + 1]; ++j) {
        const int32_t lw = level[ci[j]];
        if ((lv < 0) != (lw < 0)) { bad = 6; break; }
        if (lv >= 0 && (lw - lv > 1 || lv - lw > 1)) { bad = 7; break; }
      }
    if (bad && v < first) first = v;
  }
  if (first < n) {
    /* recompute the code for the first offender serially */
    const int64_t v = first;
    const int32_t lv = level[v], p = pred[v];
    if ((lv < 0) != (p == SENTINEL)) code = 2;
    else if (lv > 0 && (p < 0 || p >= n)) code = 3;
    else if (lv > 0 && level[p] != lv - 1) code = 4;
    else if (lv == 0 && v != root) code = 4;
    else if (lv > 0 && !row_has(rp, ci, p, (int32_t)v)) code = 5;
    else {
      code = 7;
      for (int64_t j = rp[v]; j < rp[v + 1]; ++j)
        if ((lv < 0) != (level[ci[j]] < 0)) { code = 6; break; }
    }
    *where = v;
  }
  return code;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
