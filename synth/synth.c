/*
 * synth.c — seeded synthetic CSR matrices and vectors for CB-SpMV tests and
 * benchmarks.
 *
 * This module holds NONE of the method's arithmetic (no blocking, no
 * aggregation, no packing, no SpMV).  It only produces canonical CSR inputs
 * (rows sorted, columns strictly increasing, no explicit zeros) and dense
 * vectors.  Both the oracle (oracle/) and the CUDA library consume its output;
 * it imports neither.
 *
 * Every draw is counter-based: value = H(seed, a, b) with H a SplitMix64
 * finaliser chain, so any row range [r0, r1) is generated identically for any
 * sharding (SURVEY §8(d) "Synthetic inputs").
 *
 * Workload recipes:
 *   laplace5  : 5-point stencil on a g x g grid, diag 4, neighbours -1
 *   rmat      : R-MAT (a,b,c,d) = (0.57,0.19,0.19,0.05), scale s, edge factor
 *               ef, duplicates removed, self loops kept
 *   clustered : per 16-row block row: 5 dense (nnz U[129,256]), 7 mid
 *               (U[32,128]), 2 sparse (U[1,31]) 16x16 blocks at distinct block
 *               columns in [br-64, br+64]
 *   uniform   : exactly k distinct uniform columns per row
 * Value modes: 0 U(-1,1) (never 0), 1 U(0,1], 2 integers {-4..4}\{0}, 3 ones.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct {
  int64_t m_local;   /* rows in [r0, r1) */
  int64_t n;
  int64_t nnz;
  int64_t *row_ptr;  /* m_local + 1 */
  int32_t *col;      /* nnz */
  double *val;       /* nnz */
} synth_csr_t;

/* ---------------------------------------------------------------- RNG */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t H3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed) ^ a) + b);
}
static inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

static inline double draw_val(int mode, uint64_t seed, int64_t r, int64_t c) {
  uint64_t h = H3(seed ^ 0x5EEDull, (uint64_t)r, (uint64_t)c);
  switch (mode) {
    case 0: { double v = 2.0 * u01(h) - 1.0; return v == 0.0 ? 0.5 : v; }
    case 1: return 1.0 - u01(h);                  /* (0, 1] */
    case 2: { int k = (int)(h & 7); return (double)(k < 4 ? k - 4 : k - 3); }
    default: return 1.0;
  }
}

/* ---------------------------------------------------------------- threads */
static int g_threads = 0;
void synth_set_threads(int t) { g_threads = t; }
static int nthreads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : (int)(n > 64 ? 64 : n);
}
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi, int tid);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; int tid; } job_t;
static void *job_run(void *p) { job_t *j = (job_t *)p; j->fn(j->ctx, j->lo, j->hi, j->tid); return NULL; }
static void parallel_for(int64_t n, range_fn fn, void *ctx) {
  int T = nthreads();
  if (n < 4096 || T == 1) { fn(ctx, 0, n, 0); return; }
  pthread_t th[64]; job_t jobs[64];
  for (int t = 0; t < T; t++) {
    jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].tid = t;
    jobs[t].lo = n * t / T; jobs[t].hi = n * (t + 1) / T;
    pthread_create(&th[t], NULL, job_run, &jobs[t]);
  }
  for (int t = 0; t < T; t++) pthread_join(th[t], NULL);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

void synth_free(synth_csr_t *A) {
  if (!A) return;
  free(A->row_ptr); free(A->col); free(A->val);
  A->row_ptr = NULL; A->col = NULL; A->val = NULL;
}

static int alloc_csr(synth_csr_t *A, int64_t m_local, int64_t n) {
  memset(A, 0, sizeof(*A));
  A->m_local = m_local; A->n = n;
  A->row_ptr = (int64_t *)calloc((size_t)m_local + 1, sizeof(int64_t));
  return A->row_ptr ? 0 : -1;
}
static int alloc_nnz(synth_csr_t *A) {
  int64_t nnz = A->row_ptr[A->m_local];
  A->nnz = nnz;
  A->col = (int32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  A->val = (double *)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
  return (A->col && A->val) ? 0 : -1;
}
static void prefix(int64_t *rp, int64_t m) { /* counts in rp[1..m] -> offsets */
  for (int64_t i = 0; i < m; i++) rp[i + 1] += rp[i];
}

/* ---------------------------------------------------------------- values */
typedef struct { synth_csr_t *A; int64_t r0; int mode; uint64_t seed; } valctx_t;
static void fill_vals(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; valctx_t *c = (valctx_t *)p;
  for (int64_t i = lo; i < hi; i++)
    for (int64_t k = c->A->row_ptr[i]; k < c->A->row_ptr[i + 1]; k++)
      c->A->val[k] = draw_val(c->mode, c->seed, c->r0 + i, c->A->col[k]);
}
static void values(synth_csr_t *A, int64_t r0, int mode, uint64_t seed) {
  valctx_t c = {A, r0, mode, seed};
  parallel_for(A->m_local, fill_vals, &c);
}

/* ---------------------------------------------------------------- laplace5 */
int synth_laplace5(int64_t g, int64_t r0, int64_t r1, synth_csr_t *A) {
  int64_t m = g * g;
  if (r0 < 0 || r1 > m || r0 > r1) return -1;
  if (alloc_csr(A, r1 - r0, m)) return -2;
  for (int64_t i = r0; i < r1; i++) {
    int64_t y = i / g, x = i % g;
    A->row_ptr[i - r0 + 1] = 1 + (y > 0) + (y < g - 1) + (x > 0) + (x < g - 1);
  }
  prefix(A->row_ptr, A->m_local);
  if (alloc_nnz(A)) return -2;
  for (int64_t i = r0; i < r1; i++) {
    int64_t y = i / g, x = i % g, k = A->row_ptr[i - r0];
    if (y > 0)     { A->col[k] = (int32_t)(i - g); A->val[k++] = -1.0; }
    if (x > 0)     { A->col[k] = (int32_t)(i - 1); A->val[k++] = -1.0; }
    A->col[k] = (int32_t)i; A->val[k++] = 4.0;
    if (x < g - 1) { A->col[k] = (int32_t)(i + 1); A->val[k++] = -1.0; }
    if (y < g - 1) { A->col[k] = (int32_t)(i + g); A->val[k++] = -1.0; }
  }
  return 0;
}

/* ---------------------------------------------------------------- R-MAT */
/* Quadrant thresholds in units of 1/65536: a=0.57, b=0.19, c=0.19, d=rest. */
#define RMAT_A 37356u
#define RMAT_B 12452u
#define RMAT_C 12452u
static inline void rmat_edge(uint64_t seed, int scale, uint64_t e, int64_t *r, int64_t *c) {
  uint64_t rr = 0, cc = 0, w = 0;
  for (int L = 0; L < scale; L++) {
    if ((L & 3) == 0) w = H3(seed, e, (uint64_t)(L >> 2));
    uint32_t u = (uint32_t)((w >> (16 * (L & 3))) & 0xFFFF);
    uint32_t rb, cb;
    if (u < RMAT_A) { rb = 0; cb = 0; }
    else if (u < RMAT_A + RMAT_B) { rb = 0; cb = 1; }
    else if (u < RMAT_A + RMAT_B + RMAT_C) { rb = 1; cb = 0; }
    else { rb = 1; cb = 1; }
    rr = (rr << 1) | rb; cc = (cc << 1) | cb;
  }
  *r = (int64_t)rr; *c = (int64_t)cc;
}
typedef struct {
  uint64_t seed; int scale; int64_t r0, r1; int64_t *cnt; int64_t *cur; int32_t *col;
} rmatctx_t;
static void rmat_count(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; rmatctx_t *c = (rmatctx_t *)p; int64_t r, cc;
  for (int64_t e = lo; e < hi; e++) {
    rmat_edge(c->seed, c->scale, (uint64_t)e, &r, &cc);
    if (r >= c->r0 && r < c->r1) __atomic_fetch_add(&c->cnt[r - c->r0 + 1], 1, __ATOMIC_RELAXED);
  }
}
static void rmat_fill(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; rmatctx_t *c = (rmatctx_t *)p; int64_t r, cc;
  for (int64_t e = lo; e < hi; e++) {
    rmat_edge(c->seed, c->scale, (uint64_t)e, &r, &cc);
    if (r >= c->r0 && r < c->r1) {
      int64_t k = __atomic_fetch_add(&c->cur[r - c->r0], 1, __ATOMIC_RELAXED);
      c->col[k] = (int32_t)cc;
    }
  }
}
typedef struct { int64_t *rp; int32_t *col; int64_t *newcnt; } dedupctx_t;
static void dedup_rows(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; dedupctx_t *c = (dedupctx_t *)p;
  for (int64_t i = lo; i < hi; i++) {
    int64_t b = c->rp[i], e = c->rp[i + 1];
    if (e - b > 1) qsort(c->col + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    int64_t w = b;
    for (int64_t k = b; k < e; k++)
      if (k == b || c->col[k] != c->col[k - 1]) c->col[w++] = c->col[k];
    c->newcnt[i] = w - b;
  }
}
int synth_rmat(int scale, int64_t edge_factor, uint64_t seed, int val_mode, int64_t r0, int64_t r1,
               synth_csr_t *A) {
  int64_t m = (int64_t)1 << scale, E = edge_factor * m;
  if (r0 < 0 || r1 > m || r0 > r1 || scale < 1 || scale > 30) return -1;
  if (alloc_csr(A, r1 - r0, m)) return -2;
  int64_t ml = r1 - r0;
  rmatctx_t c = {seed, scale, r0, r1, A->row_ptr, NULL, NULL};
  parallel_for(E, rmat_count, &c);
  prefix(A->row_ptr, ml);
  int64_t raw = A->row_ptr[ml];
  int32_t *col = (int32_t *)malloc((size_t)(raw ? raw : 1) * sizeof(int32_t));
  int64_t *cur = (int64_t *)malloc((size_t)(ml ? ml : 1) * sizeof(int64_t));
  if (!col || !cur) return -2;
  memcpy(cur, A->row_ptr, (size_t)ml * sizeof(int64_t));
  c.cur = cur; c.col = col;
  parallel_for(E, rmat_fill, &c);
  dedupctx_t d = {A->row_ptr, col, cur};
  parallel_for(ml, dedup_rows, &d);
  /* compact */
  int64_t *rp = (int64_t *)calloc((size_t)ml + 1, sizeof(int64_t));
  for (int64_t i = 0; i < ml; i++) rp[i + 1] = rp[i] + cur[i];
  A->nnz = rp[ml];
  A->col = (int32_t *)malloc((size_t)(A->nnz ? A->nnz : 1) * sizeof(int32_t));
  A->val = (double *)malloc((size_t)(A->nnz ? A->nnz : 1) * sizeof(double));
  if (!A->col || !A->val || !rp) return -2;
  for (int64_t i = 0; i < ml; i++)
    memcpy(A->col + rp[i], col + A->row_ptr[i], (size_t)cur[i] * sizeof(int32_t));
  free(col); free(cur); free(A->row_ptr); A->row_ptr = rp;
  values(A, r0, val_mode, seed + 1);
  return 0;
}

/* Per-row stored-entry counts of the whole matrix without materialising it (row shards are cut
 * by nnz before each rank generates only its own rows).  R-MAT: edges per row before duplicate
 * removal (an upper bound, exact enough to balance a cut). */
int synth_rmat_row_counts(int scale, int64_t edge_factor, uint64_t seed, int64_t *counts) {
  int64_t m = (int64_t)1 << scale, E = edge_factor * m;
  if (scale < 1 || scale > 30) return -1;
  int64_t *tmp = (int64_t *)calloc((size_t)m + 1, sizeof(int64_t));
  if (!tmp) return -2;
  rmatctx_t c = {seed, scale, 0, m, tmp, NULL, NULL};
  parallel_for(E, rmat_count, &c);
  memcpy(counts, tmp + 1, (size_t)m * sizeof(int64_t));
  free(tmp);
  return 0;
}

/* ---------------------------------------------------------------- clustered */
/* One 16-row block row: up to 14 blocks x 256 entries, emitted row by row. */
#define CL_BLOCKS 14
typedef struct {
  uint64_t seed; int64_t m, n, r0, r1; int64_t *rp; int32_t *col; int counting;
} clctx_t;
static int gen_blockrow(uint64_t seed, int64_t br, int64_t m, int64_t n, int32_t *rows_cols[16], int rows_n[16]) {
  int64_t nbc = (n + 15) / 16;
  int64_t lo = br - 64 < 0 ? 0 : br - 64, hi = br + 64 > nbc - 1 ? nbc - 1 : br + 64;
  int64_t w = hi - lo + 1;
  int64_t bcs[CL_BLOCKS]; int nb = 0; uint64_t j = 0;
  int want = w < CL_BLOCKS ? (int)w : CL_BLOCKS;
  while (nb < want) {
    int64_t bc = lo + (int64_t)(H3(seed, (uint64_t)br, j++) % (uint64_t)w);
    int dup = 0;
    for (int t = 0; t < nb; t++) dup |= (bcs[t] == bc);
    if (!dup) bcs[nb++] = bc;
  }
  for (int r = 0; r < 16; r++) rows_n[r] = 0;
  for (int b = 0; b < nb; b++) {
    uint64_t h = H3(seed ^ 0xB10Cull, (uint64_t)br, (uint64_t)b);
    int k = b < 5 ? 129 + (int)(h % 128) : (b < 12 ? 32 + (int)(h % 97) : 1 + (int)(h % 31));
    uint8_t pos[256];
    for (int t = 0; t < 256; t++) pos[t] = (uint8_t)t;
    for (int t = 0; t < k; t++) { /* partial Fisher-Yates */
      int s = t + (int)(H3(seed ^ 0xF15Bull, (uint64_t)(br * CL_BLOCKS + b), (uint64_t)t) % (uint64_t)(256 - t));
      uint8_t tmp = pos[t]; pos[t] = pos[s]; pos[s] = tmp;
    }
    for (int t = 0; t < k; t++) {
      int64_t r = br * 16 + (pos[t] >> 4), c = bcs[b] * 16 + (pos[t] & 15);
      if (r < m && c < n) {
        int lr = (int)(r - br * 16);
        if (rows_cols[lr]) rows_cols[lr][rows_n[lr]] = (int32_t)c;
        rows_n[lr]++;
      }
    }
  }
  return nb;
}
static void cl_work(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; clctx_t *c = (clctx_t *)p;
  int64_t br0 = c->r0 / 16;
  for (int64_t bri = lo; bri < hi; bri++) {
    int64_t br = br0 + bri;
    int rows_n[16]; int32_t *rc[16];
    int32_t buf[16][CL_BLOCKS * 16];
    for (int r = 0; r < 16; r++) rc[r] = c->counting ? NULL : buf[r];
    gen_blockrow(c->seed, br, c->m, c->n, rc, rows_n);
    for (int r = 0; r < 16; r++) {
      int64_t row = br * 16 + r;
      if (row < c->r0 || row >= c->r1) continue;
      int64_t li = row - c->r0;
      if (c->counting) { c->rp[li + 1] = rows_n[r]; continue; }
      qsort(buf[r], (size_t)rows_n[r], sizeof(int32_t), cmp_i32);
      memcpy(c->col + c->rp[li], buf[r], (size_t)rows_n[r] * sizeof(int32_t));
    }
  }
}
int synth_clustered(int64_t m, int64_t n, uint64_t seed, int val_mode, int64_t r0, int64_t r1, synth_csr_t *A) {
  if (r0 < 0 || r1 > m || r0 > r1) return -1;
  if (alloc_csr(A, r1 - r0, n)) return -2;
  int64_t nbr = r1 > r0 ? (r1 - 1) / 16 - r0 / 16 + 1 : 0;
  clctx_t c = {seed, m, n, r0, r1, A->row_ptr, NULL, 1};
  parallel_for(nbr, cl_work, &c);
  prefix(A->row_ptr, A->m_local);
  if (alloc_nnz(A)) return -2;
  c.col = A->col; c.counting = 0;
  parallel_for(nbr, cl_work, &c);
  values(A, r0, val_mode, seed + 1);
  return 0;
}

int synth_clustered_row_counts(int64_t m, int64_t n, uint64_t seed, int64_t *counts) {
  int64_t *tmp = (int64_t *)calloc((size_t)m + 1, sizeof(int64_t));
  if (!tmp) return -2;
  clctx_t c = {seed, m, n, 0, m, tmp, NULL, 1};
  parallel_for((m + 15) / 16, cl_work, &c);
  memcpy(counts, tmp + 1, (size_t)m * sizeof(int64_t));
  free(tmp);
  return 0;
}

/* ---------------------------------------------------------------- uniform */
typedef struct { uint64_t seed; int64_t n, k, r0; int64_t *rp; int32_t *col; } unictx_t;
static void uni_fill(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; unictx_t *c = (unictx_t *)p;
  for (int64_t i = lo; i < hi; i++) {
    int32_t *out = c->col + c->rp[i];
    int64_t got = 0; uint64_t j = 0, row = (uint64_t)(c->r0 + i);
    while (got < c->k) {
      int32_t cc = (int32_t)(H3(c->seed, row, j++) % (uint64_t)c->n);
      int dup = 0;
      for (int64_t t = 0; t < got; t++) dup |= (out[t] == cc);
      if (!dup) out[got++] = cc;
    }
    qsort(out, (size_t)got, sizeof(int32_t), cmp_i32);
  }
}
int synth_uniform(int64_t m, int64_t n, int64_t k, uint64_t seed, int val_mode, int64_t r0, int64_t r1,
                  synth_csr_t *A) {
  if (r0 < 0 || r1 > m || r0 > r1 || n < 1) return -1;
  if (k > n) k = n;
  if (alloc_csr(A, r1 - r0, n)) return -2;
  for (int64_t i = 0; i < A->m_local; i++) A->row_ptr[i + 1] = k;
  prefix(A->row_ptr, A->m_local);
  if (alloc_nnz(A)) return -2;
  unictx_t c = {seed, n, k, r0, A->row_ptr, A->col};
  parallel_for(A->m_local, uni_fill, &c);
  values(A, r0, val_mode, seed + 1);
  return 0;
}

/* ---------------------------------------------------------------- vectors */
/* mode 0: U(-1,1) never 0; 1: ones; 2: (j mod 7) - 3; 3: j - 7 (Fig. 1 fixture) */
typedef struct { int64_t j0; int mode; uint64_t seed; double *x; } vecctx_t;
static void vec_fill(void *p, int64_t lo, int64_t hi, int tid) {
  (void)tid; vecctx_t *c = (vecctx_t *)p;
  for (int64_t i = lo; i < hi; i++) {
    int64_t j = c->j0 + i;
    switch (c->mode) {
      case 0: { double v = 2.0 * u01(H3(c->seed ^ 0xFEC7ull, (uint64_t)j, 0)) - 1.0; c->x[i] = v == 0.0 ? 0.5 : v; break; }
      case 1: c->x[i] = 1.0; break;
      case 2: c->x[i] = (double)(j % 7 - 3); break;
      default: c->x[i] = (double)(j - 7); break;
    }
  }
}
int synth_vector(int64_t j0, int64_t len, int mode, uint64_t seed, double *x) {
  vecctx_t c = {j0, mode, seed, x};
  parallel_for(len, vec_fill, &c);
  return 0;
}
