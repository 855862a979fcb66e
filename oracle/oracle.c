/*
 * oracle.c — the CB-SpMV ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_2605_18515_b200/) never imports, links or executes it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, slow, single-threaded C, written from the paper (arxiv 2605.18515,
 * /root/reference/PAPER.md, cited "P:<line>") with the readings listed in
 * DESIGN.md §2 (cited "R-<k>").  Floating point is fp64 throughout.
 *
 *   oracle_spmv_csr   Alg. 1: y_i = sum_j a_ij x_j, ascending j,
 *                     plus R_i = sum_j |a_ij x_j| (the tolerance scale).
 *   oracle_build      the Fig. 7 pipeline step by step:
 *                     partition -> block stats + th0 ->
 *                     column aggregation -> format selection ->
 *                     intra-block data aggregation / VP / padding (P:405,
 *                     P:417-424) -> TB-Load-Balance Alg. 2.
 *   oracle_spmv_cb    Alg. 3 / Alg. 4 semantics executed sequentially over the
 *                     packed format in slot order.
 *   oracle_storage_*  the storage model of P:174.
 *
 * Pins (tests/test_oracle_*.py): dense brute force (numpy) on tiny matrices,
 * closed forms (Laplacian row sums, x = 1), the Fig. 1 fixture, SPEC worked
 * values (storage 224/2060/138, COO record 120/72 B, Alg. 2 [10,8,3,1]),
 * an independently written brute-force greedy for Alg. 2, an independent
 * Python unpacker for the record layouts, and invariants.  No function here
 * is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_EINVAL = 1, OR_EUNSORTED = 2, OR_ENOMEM = 3 };
enum { FMT_COO = 0, FMT_CSR = 1, FMT_DENSE = 2 };

/* ------------------------------------------------------------------ Alg. 1 */
/* for i: sum <- 0; for j in row i: sum <- sum + x[col_idx[j]] * csr_val[j]; y[i] <- sum */
int oracle_spmv_csr(int64_t m, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                    const double *x, double *y, double *R) {
  for (int64_t i = 0; i < m; i++) {
    double sum = 0.0, abs_sum = 0.0;
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++) {
      double p = x[col_idx[j]] * val[j];
      sum = sum + p;
      abs_sum = abs_sum + fabs(p);
    }
    y[i] = sum;
    if (R) R[i] = abs_sum;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------ P:174 */
/* CSR: (m+1)*4 + nnz*4 + nnz*8; BSR (16x16): 256*8*nnzb + (blk_m+1)*4 + nnzb*4;
 * CB (all-COO sub-blocks): nnzb*(4+4+4+1+8) + nnz*(1+8). */
int64_t oracle_storage_csr(int64_t m, int64_t nnz) { return (m + 1) * 4 + nnz * 4 + nnz * 8; }
int64_t oracle_storage_bsr(int64_t nnzb, int64_t blk_m) { return 256 * 8 * nnzb + (blk_m + 1) * 4 + nnzb * 4; }
int64_t oracle_storage_cb(int64_t nnzb, int64_t nnz) { return nnzb * (4 + 4 + 4 + 1 + 8) + nnz * (1 + 8); }

/* ------------------------------------------------------------------ P:439 */
/* "COO for ... less than th1, Dense for ... more than th2, and CSR for intermediate" (R-9: strict). */
int oracle_select_format(int64_t nnz, int th1, int th2) {
  if (nnz < th1) return FMT_COO;
  if (nnz > th2) return FMT_DENSE;
  return FMT_CSR;
}

/* P:424 + P:513-514: 4-bit row and col in one uint8; decode row = b & 15, col = b >> 4. */
int oracle_encode_coord(int local_row, int local_col) { return (local_col << 4) | local_row; }

/* Alg. 3 lines 6-7: padding <- (nnz*size(Idx)) mod size(Val); padding ? size(Val)-padding : 0 */
int64_t oracle_padding(int64_t idx_bytes, int64_t val_size) {
  int64_t padding = idx_bytes % val_size;
  return padding ? val_size - padding : 0;
}

/* ------------------------------------------------------------------ options / outputs */
typedef struct {
  int blk;            /* 16; 4 only for the Fig. 1 fixture (R-21) */
  int th0_num, th0_den; /* th0 = 0.15 = 15/100 */
  int ss_limit;       /* "super-sparse": nnz < 32 (R-4) */
  int th1, th2;       /* 32, 128 */
  int warps_per_tb;   /* 8 */
  int agg_mode;       /* -1 auto (th0), 0 off, 1 on */
  int balance;        /* 1: Alg. 2; 0: natural (br,bc) order, W consecutive per TB */
  int force_format;   /* -1 none; 0/1/2 force COO/CSR/DENSE */
  int val_size;       /* 8 (fp64) or 4 (fp32) */
} oracle_opts_t;

typedef struct {
  int64_t m, n, nnz, nb, blk_m, blk_n;
  int64_t ss_count;   /* blocks with nnz < ss_limit before aggregation */
  int64_t nb_pre;     /* non-empty blocks before aggregation */
  int agg;
  int32_t *blk_row_idx, *blk_col_idx, *nnz_per_blk; /* slot order (after Alg. 2) */
  uint8_t *type_per_blk;
  uint64_t *vp_per_blk;
  uint8_t *mtx_data; int64_t mtx_bytes;
  uint64_t *cols_offset; int64_t n_cols_offset;     /* blk_m + 1 when agg */
  uint32_t *restore_cols; int64_t n_restore;
  int64_t T;          /* ceil(nb / W) thread blocks */
  int64_t *tb_ptr;    /* T + 1: blocks of TB t are [tb_ptr[t], tb_ptr[t+1]) (R-14) */
  int64_t *tb_load;   /* per-TB nnz after the schedule */
  int64_t *tb_load_natural; /* per-TB nnz with W consecutive blocks in (br,bc) order */
  int64_t fmt_count[3];
} oracle_cb_t;

void oracle_default_opts(oracle_opts_t *o) {
  o->blk = 16; o->th0_num = 15; o->th0_den = 100; o->ss_limit = 32; o->th1 = 32; o->th2 = 128;
  o->warps_per_tb = 8; o->agg_mode = -1; o->balance = 1; o->force_format = -1; o->val_size = 8;
}

void oracle_cb_free(oracle_cb_t *c) {
  free(c->blk_row_idx); free(c->blk_col_idx); free(c->nnz_per_blk); free(c->type_per_blk);
  free(c->vp_per_blk); free(c->mtx_data); free(c->cols_offset); free(c->restore_cols);
  free(c->tb_ptr); free(c->tb_load); free(c->tb_load_natural);
  memset(c, 0, sizeof(*c));
}

/* ------------------------------------------------------------------ block-COO elements */
typedef struct { int64_t br, bc; int lr, lc; double v; } elem_t;

static int cmp_elem(const void *a, const void *b) {
  const elem_t *x = (const elem_t *)a, *y = (const elem_t *)b;
  if (x->br != y->br) return x->br < y->br ? -1 : 1;
  if (x->bc != y->bc) return x->bc < y->bc ? -1 : 1;
  if (x->lr != y->lr) return x->lr < y->lr ? -1 : 1;
  if (x->lc != y->lc) return x->lc < y->lc ? -1 : 1;
  return 0;
}
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* blocks = runs of equal (br, bc) in the sorted element list */
typedef struct { int64_t br, bc, first, nnz; } blk_t;

static int64_t group_blocks(const elem_t *e, int64_t nnz, blk_t *out) {
  int64_t nb = 0;
  for (int64_t k = 0; k < nnz; k++) {
    if (k == 0 || e[k].br != e[k - 1].br || e[k].bc != e[k - 1].bc) {
      out[nb].br = e[k].br; out[nb].bc = e[k].bc; out[nb].first = k; out[nb].nnz = 0; nb++;
    }
    out[nb - 1].nnz++;
  }
  return nb;
}

/* ------------------------------------------------------------------ Alg. 2 heap */
typedef struct { int64_t loads, tb_id; int warps; } pq_t;
static int pq_less(const pq_t *a, const pq_t *b) {          /* R-13: key (loads, tb_id) */
  return a->loads < b->loads || (a->loads == b->loads && a->tb_id < b->tb_id);
}
static void pq_push(pq_t *h, int64_t *n, pq_t v) {
  int64_t i = (*n)++;
  h[i] = v;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!pq_less(&h[i], &h[p])) break;
    pq_t t = h[i]; h[i] = h[p]; h[p] = t; i = p;
  }
}
static pq_t pq_pop(pq_t *h, int64_t *n) {
  pq_t top = h[0];
  h[0] = h[--(*n)];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < *n && pq_less(&h[l], &h[s])) s = l;
    if (r < *n && pq_less(&h[r], &h[s])) s = r;
    if (s == i) break;
    pq_t t = h[i]; h[i] = h[s]; h[s] = t; i = s;
  }
  return top;
}

/* blk_idx_array items: ori, end, nnz */
typedef struct { int64_t ori, end, nnz; } bia_t;
static int cmp_nnz(const void *a, const void *b) {   /* R-12: nnz descending, ties ori ascending */
  const bia_t *x = (const bia_t *)a, *y = (const bia_t *)b;
  if (x->nnz != y->nnz) return x->nnz > y->nnz ? -1 : 1;
  return (x->ori > y->ori) - (x->ori < y->ori);
}
static int cmp_end(const void *a, const void *b) {
  const bia_t *x = (const bia_t *)a, *y = (const bia_t *)b;
  return (x->end > y->end) - (x->end < y->end);
}

/* ------------------------------------------------------------------ the pipeline */
int oracle_build(int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                 const double *val, const oracle_opts_t *o, oracle_cb_t *out) {
  memset(out, 0, sizeof(*out));
  const int B = o->blk, W = o->warps_per_tb;
  const int64_t S = o->val_size;
  if (m < 0 || n < 0 || B < 1 || B > 16 || W < 1 || (S != 4 && S != 8)) return OR_EINVAL;

  /* a1. canonical check (R-19): columns in range and strictly increasing, finite values;
   *     explicit zeros are dropped. */
  int64_t nnz = 0;
  for (int64_t i = 0; i < m; i++) {
    if (row_ptr[i + 1] < row_ptr[i]) return OR_EINVAL;
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++) {
      if (col_idx[j] < 0 || col_idx[j] >= n) return OR_EINVAL;
      if (j > row_ptr[i] && col_idx[j] <= col_idx[j - 1]) return OR_EUNSORTED;
      if (!isfinite(val[j])) return OR_EINVAL;
      if (val[j] != 0.0) nnz++;
    }
  }
  out->m = m; out->n = n; out->nnz = nnz;
  out->blk_m = (m + B - 1) / B; out->blk_n = (n + B - 1) / B;

  /* a2. "input data is loaded as a block-based COO format"; uniform BxB blocks */
  elem_t *e = (elem_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(elem_t));
  blk_t *blocks = (blk_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(blk_t));
  if (!e || !blocks) return OR_ENOMEM;
  int64_t k = 0;
  for (int64_t i = 0; i < m; i++)
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; j++) {
      if (val[j] == 0.0) continue;
      e[k].br = i / B; e[k].bc = col_idx[j] / B; e[k].lr = (int)(i % B); e[k].lc = (int)(col_idx[j] % B);
      e[k].v = val[j]; k++;
    }
  qsort(e, (size_t)nnz, sizeof(elem_t), cmp_elem);
  int64_t nb = group_blocks(e, nnz, blocks);
  out->nb_pre = nb;

  /* a3. super-sparse proportion and th0: aggregate iff ss/nb >= th0 (R-3, R-5) */
  int64_t ss = 0;
  for (int64_t b = 0; b < nb; b++) if (blocks[b].nnz < o->ss_limit) ss++;
  out->ss_count = ss;
  int agg = o->agg_mode >= 0 ? o->agg_mode : (nb > 0 && ss * o->th0_den >= (int64_t)o->th0_num * nb);
  out->agg = agg;

  /* a4. block-aware column aggregation (R-6 per block row, R-7 offset) */
  if (agg) {
    out->n_cols_offset = out->blk_m + 1;
    out->cols_offset = (uint64_t *)calloc((size_t)out->n_cols_offset, sizeof(uint64_t));
    out->restore_cols = (uint32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(uint32_t));
    int64_t *cols = (int64_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
    if (!out->cols_offset || !out->restore_cols || !cols) return OR_ENOMEM;
    int64_t nres = 0, p = 0;
    for (int64_t br = 0; br < out->blk_m; br++) {
      /* C_i: sorted distinct original columns with a non-zero in block row br */
      int64_t q = p, nc = 0;
      while (q < nnz && e[q].br == br) { cols[nc++] = e[q].bc * B + e[q].lc; q++; }
      qsort(cols, (size_t)nc, sizeof(int64_t), cmp_i64);
      int64_t nd = 0;
      for (int64_t t = 0; t < nc; t++) if (t == 0 || cols[t] != cols[t - 1]) cols[nd++] = cols[t];
      out->cols_offset[br] = (uint64_t)nres;
      for (int64_t t = 0; t < nd; t++) out->restore_cols[nres + t] = (uint32_t)cols[t];
      /* column c -> rank c' in C_i; re-block at bc' = c' / B, local c' mod B */
      for (int64_t t = p; t < q; t++) {
        int64_t c = e[t].bc * B + e[t].lc, lo = 0, hi = nd - 1;
        while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cols[mid] < c) lo = mid + 1; else hi = mid; }
        e[t].bc = lo / B; e[t].lc = (int)(lo % B);
      }
      nres += nd; p = q;
    }
    out->cols_offset[out->blk_m] = (uint64_t)nres;
    out->n_restore = nres;
    free(cols);
    qsort(e, (size_t)nnz, sizeof(elem_t), cmp_elem);    /* re-form blocks on aggregated columns */
    nb = group_blocks(e, nnz, blocks);
  }
  out->nb = nb;

  /* a5. format selection on the (post-aggregation) blocks (R-9, R-10) */
  uint8_t *type = (uint8_t *)malloc((size_t)(nb ? nb : 1));
  uint64_t *vp = (uint64_t *)malloc((size_t)(nb ? nb : 1) * sizeof(uint64_t));
  if (!type || !vp) return OR_ENOMEM;
  for (int64_t b = 0; b < nb; b++) {
    type[b] = (uint8_t)(o->force_format >= 0 ? o->force_format
                                             : oracle_select_format(blocks[b].nnz, o->th1, o->th2));
    out->fmt_count[type[b]]++;
  }

  /* a6. intra-block data aggregation: record sizes, VP = running byte offset
   *     (R-11), padding of the index bytes to size(Val) (Alg. 3; R-8). */
  int64_t total = 0;
  for (int64_t b = 0; b < nb; b++) {
    int64_t idx_bytes = type[b] == FMT_COO ? blocks[b].nnz : type[b] == FMT_CSR ? (B + 1) + blocks[b].nnz : 0;
    int64_t nval = type[b] == FMT_DENSE ? (int64_t)B * B : blocks[b].nnz;
    vp[b] = (uint64_t)total;
    total += idx_bytes + oracle_padding(idx_bytes, S) + nval * S;
  }
  out->mtx_bytes = total;
  out->mtx_data = (uint8_t *)calloc((size_t)(total ? total : 1), 1);
  if (!out->mtx_data) return OR_ENOMEM;
  for (int64_t b = 0; b < nb; b++) {
    uint8_t *rec = out->mtx_data + vp[b];
    const elem_t *be = e + blocks[b].first;
    int64_t bn = blocks[b].nnz;
    uint8_t *vals;
    if (type[b] == FMT_COO) {          /* coo_idx <- VP; coo_val <- VP + nnz*size(Idx) + padding */
      for (int64_t t = 0; t < bn; t++) rec[t] = (uint8_t)oracle_encode_coord(be[t].lr, be[t].lc);
      vals = rec + bn + oracle_padding(bn, S);
      for (int64_t t = 0; t < bn; t++) {
        if (S == 8) memcpy(vals + 8 * t, &be[t].v, 8);
        else { float f = (float)be[t].v; memcpy(vals + 4 * t, &f, 4); }
      }
    } else if (type[b] == FMT_CSR) {   /* R-8: B+1 u8 row_ptr, nnz u8 local cols, pad, values */
      int64_t t = 0;
      for (int r = 0; r <= B; r++) {
        while (t < bn && be[t].lr < r) t++;
        rec[r] = (uint8_t)(t & 0xFF);
      }
      for (int64_t q = 0; q < bn; q++) rec[B + 1 + q] = (uint8_t)be[q].lc;
      vals = rec + (B + 1) + bn + oracle_padding((B + 1) + bn, S);
      for (int64_t q = 0; q < bn; q++) {
        if (S == 8) memcpy(vals + 8 * q, &be[q].v, 8);
        else { float f = (float)be[q].v; memcpy(vals + 4 * q, &f, 4); }
      }
    } else {                           /* DENSE: dense_val[row*B + col], zeros elsewhere */
      for (int64_t q = 0; q < bn; q++) {
        int64_t pos = (int64_t)be[q].lr * B + be[q].lc;
        if (S == 8) memcpy(rec + 8 * pos, &be[q].v, 8);
        else { float f = (float)be[q].v; memcpy(rec + 4 * pos, &f, 4); }
      }
    }
  }

  /* natural grouping statistics (pre-LB): W consecutive blocks per TB */
  int64_t T = (nb + W - 1) / W;
  out->T = T;
  out->tb_ptr = (int64_t *)calloc((size_t)T + 1, sizeof(int64_t));
  out->tb_load = (int64_t *)calloc((size_t)(T ? T : 1), sizeof(int64_t));
  out->tb_load_natural = (int64_t *)calloc((size_t)(T ? T : 1), sizeof(int64_t));
  if (!out->tb_ptr || !out->tb_load || !out->tb_load_natural) return OR_ENOMEM;
  for (int64_t b = 0; b < nb; b++) out->tb_load_natural[b / W] += blocks[b].nnz;

  /* a7. TB-Load-Balance, Alg. 2 */
  bia_t *bia = (bia_t *)malloc((size_t)(nb ? nb : 1) * sizeof(bia_t));
  if (!bia) return OR_ENOMEM;
  for (int64_t b = 0; b < nb; b++) { bia[b].ori = b; bia[b].end = b; bia[b].nnz = blocks[b].nnz; }
  if (o->balance) {
    qsort(bia, (size_t)nb, sizeof(bia_t), cmp_nnz);           /* parallel sort(blk_idx_array, cmp_nnz) */
    pq_t *pq = (pq_t *)malloc((size_t)(T ? T : 1) * sizeof(pq_t));
    int64_t pn = 0;
    if (!pq) return OR_ENOMEM;
    for (int64_t t = 0; t < T; t++) { pq_t v = {0, t, 0}; pq_push(pq, &pn, v); }   /* R-13 */
    for (int64_t i = 0; i < nb; i++) {
      pq_t top = pq_pop(pq, &pn);                              /* pqtop <- pq.top(), pq.pop() */
      bia[i].end = top.tb_id * W + top.warps;                  /* end <- tb_id*8 + warps */
      top.loads += bia[i].nnz;                                 /* loads <- loads + nnz */
      top.warps += 1;                                          /* warps <- warps + 1 */
      if (top.warps < W) pq_push(pq, &pn, top);                /* if warps < 8: push */
    }
    free(pq);
    qsort(bia, (size_t)nb, sizeof(bia_t), cmp_end);            /* parallel sort(blk_idx_array, cmp_end) */
  }
  /* permute the five high-level arrays (vp_per_blk[i] <- vp_per_blk_old[ori]); tb_ptr (R-14) */
  out->blk_row_idx = (int32_t *)malloc((size_t)(nb ? nb : 1) * sizeof(int32_t));
  out->blk_col_idx = (int32_t *)malloc((size_t)(nb ? nb : 1) * sizeof(int32_t));
  out->nnz_per_blk = (int32_t *)malloc((size_t)(nb ? nb : 1) * sizeof(int32_t));
  out->type_per_blk = (uint8_t *)malloc((size_t)(nb ? nb : 1));
  out->vp_per_blk = (uint64_t *)malloc((size_t)(nb ? nb : 1) * sizeof(uint64_t));
  if (!out->blk_row_idx || !out->blk_col_idx || !out->nnz_per_blk || !out->type_per_blk || !out->vp_per_blk)
    return OR_ENOMEM;
  for (int64_t i = 0; i < nb; i++) {
    int64_t ori = bia[i].ori;
    out->blk_row_idx[i] = (int32_t)blocks[ori].br;
    out->blk_col_idx[i] = (int32_t)blocks[ori].bc;
    out->nnz_per_blk[i] = (int32_t)blocks[ori].nnz;
    out->type_per_blk[i] = type[ori];
    out->vp_per_blk[i] = vp[ori];
    int64_t t = bia[i].end / W;
    out->tb_ptr[t + 1]++;
    out->tb_load[t] += blocks[ori].nnz;
  }
  for (int64_t t = 0; t < T; t++) out->tb_ptr[t + 1] += out->tb_ptr[t];
  free(bia); free(type); free(vp); free(e); free(blocks);
  return OR_OK;
}

/* ------------------------------------------------------------------ Alg. 3 / 4 semantics */
/* Sequential execution of the packed format in slot order.  Per block, the type's path adds
 * its products into y[br*B + row]; x is x[bc*B + col] without aggregation and
 * x[restore_cols[cols_offset[br] + bc*B + col]] with it (R-7).  Dense: each row's
 * 16-term dot product is added (R-15).  CSR: per local row, its stored elements. */
int oracle_spmv_cb(const oracle_cb_t *c, int blk, int val_size, const double *x, double *y) {
  const int B = blk;
  for (int64_t i = 0; i < c->m; i++) y[i] = 0.0;
  for (int64_t i = 0; i < c->nb; i++) {
    const uint8_t *rec = c->mtx_data + c->vp_per_blk[i];
    int64_t br = c->blk_row_idx[i], bc = c->blk_col_idx[i], bn = c->nnz_per_blk[i];
    int type = c->type_per_blk[i];
    const uint8_t *vals;
#define XCOL(lc) (c->agg ? (int64_t)c->restore_cols[c->cols_offset[br] + bc * B + (lc)] : bc * B + (lc))
#define VAL(p, q) (val_size == 8 ? ((const double *)(const void *)(p))[q] : (double)((const float *)(const void *)(p))[q])
    if (type == FMT_COO) {
      vals = rec + bn + oracle_padding(bn, val_size);
      for (int64_t t = 0; t < bn; t++) {
        int row_idx = rec[t] & 15, col_idx = rec[t] >> 4;
        y[br * B + row_idx] += VAL(vals, t) * x[XCOL(col_idx)];
      }
    } else if (type == FMT_CSR) {
      vals = rec + (B + 1) + bn + oracle_padding((B + 1) + bn, val_size);
      for (int r = 0; r < B; r++) {
        int64_t lo = rec[r], hi = (r + 1 < B) ? rec[r + 1] : bn;   /* row_ptr[B] = nnz (R-8) */
        double sum = 0.0;
        for (int64_t q = lo; q < hi; q++) sum += VAL(vals, q) * x[XCOL(rec[B + 1 + q])];
        if (hi > lo) y[br * B + r] += sum;
      }
    } else {
      for (int r = 0; r < B; r++) {
        if (br * B + r >= c->m) break;
        double sum = 0.0;
        int ncols = B;
        for (int col = 0; col < ncols; col++) {
          double v = VAL(rec, (int64_t)r * B + col);
          if (v == 0.0) continue;             /* absent entries contribute 0 */
          sum += v * x[XCOL(col)];
        }
        y[br * B + r] += sum;
      }
    }
#undef XCOL
#undef VAL
  }
  return OR_OK;
}

/* Population mean / std-dev / max of per-TB loads (Fig. 4). */
void oracle_load_stats(const int64_t *loads, int64_t T, double *mean, double *sd, int64_t *mx) {
  double s = 0.0, s2 = 0.0; int64_t M = 0;
  for (int64_t t = 0; t < T; t++) { s += (double)loads[t]; if (loads[t] > M) M = loads[t]; }
  double mu = T ? s / (double)T : 0.0;
  for (int64_t t = 0; t < T; t++) s2 += ((double)loads[t] - mu) * ((double)loads[t] - mu);
  *mean = mu; *sd = T ? sqrt(s2 / (double)T) : 0.0; *mx = M;
}
