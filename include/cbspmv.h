/*
 * cbspmv.h — C ABI of the B200-native CB-SpMV hot path (arxiv 2605.18515).
 *
 * y = A·x over the paper's cache-friendly 2D-blocked format ("CB-SpMV",
 * PAPER.md §3).  Citations "P:<n>" are lines of
 * /root/reference/PAPER.md; "R-<k>" are the readings of silent or ambiguous
 * passages listed in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *   - Nothing throws across the ABI; every call returns a cbspmv_status_t and
 *     stores a human-readable detail retrievable with cbspmv_last_error()
 *     (thread-local).
 *   - Indices are 0-based.  A is m x n; x has n entries, y has m entries.
 *   - "_dev" pointers are CUDA device pointers on the handle's device;
 *     "_host" pointers are host memory (pinned is fastest, pageable works).
 *   - stream is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device calls are asynchronous on that stream; asynchronous
 *     kernel faults surface at the caller's next synchronisation.
 *   - The handle owns every device and host allocation it makes; the caller
 *     owns all buffers it passes in.  Handles are not thread-safe: one thread
 *     at a time per handle.
 */
#ifndef CBSPMV_H
#define CBSPMV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBSPMV_VERSION 1

typedef struct cbspmv_s *cbspmv_handle_t;

typedef enum {
  CBSPMV_OK = 0,
  CBSPMV_EINVAL = 1,      /* bad argument, col >= n, non-finite value, row_ptr decreasing */
  CBSPMV_EUNSORTED = 2,   /* columns not strictly increasing within a row (R-19) */
  CBSPMV_ENOMEM = 3,      /* host or device allocation failed */
  CBSPMV_ECUDA = 4,       /* a CUDA runtime call failed (detail in cbspmv_last_error) */
  CBSPMV_EDIM = 5,        /* pointer alignment / device mismatch */
  CBSPMV_EUNSUPPORTED = 6, /* e.g. device call on a host-only handle, blk != 16 on device */
  CBSPMV_EIO = 7,          /* a file could not be opened, read or written */
  CBSPMV_EFORMAT = 8       /* malformed Matrix Market or CBSM file content */
} cbspmv_status_t;

/* Value types.  CBSPMV_F32F64 is the mixed variant the paper names without defining (P:251,
 * P:379; reading R-24): matrix values stored as fp32 in the records (size(Val) = 4, the fp32
 * layout), x, y and every product / accumulation in fp64.  Its result equals the fp64 product
 * of the fp32-rounded matrix with x within the fp64 tolerance. */
typedef enum { CBSPMV_F64 = 0, CBSPMV_F32 = 1, CBSPMV_F32F64 = 2 } cbspmv_dtype_t;

/* Sub-block storage formats. */
enum { CBSPMV_FMT_COO = 0, CBSPMV_FMT_CSR = 1, CBSPMV_FMT_DENSE = 2 };

typedef struct {
  uint32_t struct_size;   /* sizeof(cbspmv_options_t); set by cbspmv_default_options */
  int32_t blk;            /* sub-block edge, 16.  4 is accepted for host-only builds
                             (the Fig. 1 fixture, R-21) */
  int32_t th0_num;        /* th0 = th0_num / th0_den = 15/100; aggregate iff
                             (#blocks with nnz < ss_limit) / (#non-empty blocks) >= th0 (R-3, R-5) */
  int32_t th0_den;
  int32_t ss_limit;       /* "super-sparse": nnz < 32 (R-4) */
  int32_t th1, th2;       /* COO if nnz < th1, DENSE if nnz > th2, else CSR; 32 / 128 (R-9) */
  int32_t warps_per_tb;   /* warp slots per thread block in Alg. 2, 8 */
  int32_t agg_mode;       /* -1 decide by th0; 0 never; 1 always (ablation; global decision for shards) */
  int32_t balance;        /* 1 = Alg. 2 TB-Load-Balance; 0 = natural (br,bc) order */
  int32_t force_format;   /* -1 none; CBSPMV_FMT_* forces every block's format (white-box tests) */
  int32_t device;         /* CUDA ordinal for the device copy; -1 = host-only build (export/info only) */
  int32_t host_threads;   /* host builder threads; 0 = all online cores */
  int32_t keep_host;      /* 1 = keep the canonical host arrays for cbspmv_export (default 1) */
  int32_t col_panels;     /* column panels (NEXT-1): 0 = auto (x larger than 3/4 of L2 ->
                             panels of <= 3/8 L2 of x each), 1 = none, k >= 2 = k panels.  Each panel
                             (all rows, columns [c_k, c_k+1), 16-aligned) runs the whole pipeline as
                             its own matrix; cbspmv_spmv zeroes y once and runs the panels in order so
                             each panel's slice of x stays L2-resident. */
  int32_t device_build;   /* 1 = steps a2..a6 on the GPU (radix sorts, scans, one warp per record;
                             SURVEY §8(f) NEXT-3), a1 and Alg. 2 on the host; the canonical format is
                             byte-identical to the host build.  Needs device >= 0 and < 2^31 stored
                             entries per panel.  0 = host build (default). */
} cbspmv_options_t;

typedef struct {
  int64_t m, n, nnz;              /* nnz = stored non-zeros after dropping explicit zeros (R-19) */
  int64_t blk_m;                  /* ceil(m / blk) block rows */
  int64_t nb;                     /* non-empty sub-blocks after aggregation */
  int64_t nb_pre;                 /* non-empty sub-blocks before aggregation */
  int64_t ss_count;               /* super-sparse blocks before aggregation */
  int32_t agg;                    /* column aggregation applied */
  int32_t dtype;                  /* cbspmv_dtype_t */
  int64_t fmt_count[3];           /* blocks per format (COO, CSR, DENSE) */
  int64_t T;                      /* thread blocks = ceil(nb / warps_per_tb) (R-13) */
  double tb_load_mean, tb_load_sd;          /* per-TB nnz after the schedule (Fig. 4) */
  int64_t tb_load_max;
  double tb_load_sd_natural;                /* per-TB nnz std-dev of the natural grouping */
  int64_t tb_load_max_natural;
  int64_t mtx_bytes;              /* |mtx_data| of the canonical packed format */
  int64_t n_restore;              /* |restore_cols| (u32 each) */
  int64_t meta_bytes;             /* 21 B per block: br, bc, nnz (i32), type (u8), vp (u64) */
  int64_t alg_bytes;              /* algorithmic bytes of one SpMV: meta + mtx + 4*restore +
                                     8*(blk_m+1 if agg) + size(x elem)*(n + m) */
  int64_t dev_stream_bytes;       /* bytes of the device page stream */
  int64_t n_pages;                /* device pages */
  int64_t dev_bytes;              /* all device memory owned by the handle */
  int32_t grid;                   /* persistent CTAs per SpMV launch */
  int32_t launches_per_spmv;      /* kernels launched by one cbspmv_spmv */
  double build_seconds;           /* host pipeline wall time (a1..a7 + device layout) */
  double upload_seconds;          /* H2D copy wall time */
  int32_t n_panels;               /* column panels (1 = whole matrix); counts above sum over panels */
  int64_t n_hot;                  /* hot x columns cached in shared memory, summed
                                     over panels; 0 = no cache */
} cbspmv_info_t;

/* Host copies of the canonical format, slot order (after Alg. 2).  Pointers
 * are owned by the handle and valid until cbspmv_destroy. */
typedef struct {
  int64_t nb, T, mtx_bytes, n_restore, n_cols_offset;
  const int32_t *blk_row_idx;     /* P:405 high-level COO over non-empty blocks */
  const int32_t *blk_col_idx;     /* aggregated block column when agg (R-10) */
  const int32_t *nnz_per_blk;
  const uint8_t *type_per_blk;    /* CBSPMV_FMT_* */
  const uint64_t *vp_per_blk;     /* byte offset of the block's record in mtx_data (R-11) */
  const uint8_t *mtx_data;        /* packed records (R-8) */
  const uint32_t *restore_cols;   /* aggregated -> original column, per block row */
  const uint64_t *cols_offset;    /* blk_m + 1 entries when agg, else NULL (R-7) */
  const int64_t *tb_ptr;          /* T + 1: blocks of TB t are [tb_ptr[t], tb_ptr[t+1]) (R-14) */
  const int64_t *tb_load;         /* per-TB nnz after the schedule */
  const int64_t *tb_load_natural; /* per-TB nnz of the natural grouping (pre-LB, Fig. 4) */
} cbspmv_export_t;

/* Fill *opts with the paper's defaults. */
cbspmv_status_t cbspmv_default_options(cbspmv_options_t *opts);

/* Build the CB-SpMV format of a host CSR matrix (the Fig. 7 pipeline):
 * canonical check, 16x16 partition, th0 decision and block-aware
 * column aggregation, format selection, intra-block data
 * aggregation with virtual pointers and padding, TB-Load-Balance
 * (Alg. 2); then lays the blocks out as the device page stream and
 * uploads it in one copy ("transferred to the GPU in a single operation").
 *   row_ptr: m+1 int64, non-decreasing, row_ptr[0] = 0
 *   col_idx: nnz int32 in [0, n), strictly increasing within each row
 *   vals:    nnz values: double (CBSPMV_F64) or float (CBSPMV_F32, CBSPMV_F32F64); explicit
 *            zeros are dropped
 *   opts:    NULL = defaults
 *   stream:  stream for the upload; build returns after the upload completed
 * The CSR is read during the call only.  On error *out is NULL. */
cbspmv_status_t cbspmv_build(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr,
                             const int32_t *col_idx, const void *vals, cbspmv_dtype_t dtype,
                             const cbspmv_options_t *opts, void *stream, cbspmv_handle_t *out);

/* y := A·x (Alg. 3 / Alg. 4 semantics).  Zeroes y, then one
 * persistent kernel streams the page stream and adds every block's products
 * into y (R-16).  x_dev: n values, y_dev: m values, double (CBSPMV_F64,
 * CBSPMV_F32F64) or float (CBSPMV_F32), aligned to their size, not aliasing.
 * Argument checks (every device-vector entry point; SURVEY §8(b) conventions): a null
 * handle or vector, or y == x -> EINVAL; a host-only handle -> EUNSUPPORTED; a misaligned
 * vector, a pointer that is not device (or managed) memory of the handle's device, or whose
 * allocation ends before n (x) / m (y) values -> EDIM.  The C ABI carries no lengths: the
 * range check is against the enclosing allocation (cuMemGetAddressRange), so a vector cut
 * from a larger pool allocation is checked only against the pool; the Python binding checks
 * exact lengths and dtypes.  Nothing is launched when a check fails. */
cbspmv_status_t cbspmv_spmv(cbspmv_handle_t h, const void *x_dev, void *y_dev, void *stream);

/* y += A·x (the kernel alone, no zeroing). */
cbspmv_status_t cbspmv_spmv_add(cbspmv_handle_t h, const void *x_dev, void *y_dev, void *stream);

/* y := A·(s·x) with s = 1/sqrt(*sumsq_dev) read on the device (power
 * iteration: the normalisation of the previous iterate folded into the x load,
 * SURVEY §8(e)).  sumsq_dev: one double on the device. */
cbspmv_status_t cbspmv_spmv_scaled(cbspmv_handle_t h, const void *x_dev, const double *sumsq_dev,
                                   void *y_dev, void *stream);

/* One column panel k (0 <= k < info.n_panels) alone: y (+)= A[:, c_k:c_k+1) · (s·x) with
 * s = 1/sqrt(*sumsq_dev), or s = 1 when sumsq_dev is NULL; zero_y != 0 zeroes y first.  Only
 * x[c_k, c_k+1) is read, so a caller whose x arrives slice by slice (the all-gather of power
 * iteration) can run panel k as soon as its slice is present.  Running
 * every panel once, the first with zero_y, equals cbspmv_spmv / cbspmv_spmv_scaled. */
cbspmv_status_t cbspmv_spmv_panel(cbspmv_handle_t h, int32_t k, const void *x_dev, const double *sumsq_dev,
                                  void *y_dev, int32_t zero_y, void *stream);

/* Columns [*c0, *c1) of panel k. */
cbspmv_status_t cbspmv_panel_bounds(cbspmv_handle_t h, int32_t k, int64_t *c0, int64_t *c1);

/* End to end with host buffers: copies x_host (n values) to the device, runs
 * cbspmv_spmv into an internal device y, copies y back to y_host (m values),
 * and synchronises the stream before returning. */
cbspmv_status_t cbspmv_spmv_host(cbspmv_handle_t h, const void *x_host, void *y_host, void *stream);

/* End to end over `count` independent right-hand sides (a batch of requests served from host
 * memory): y_host[k] := A·x_host[k], k = 0..count-1 (n and m values each).  Pipelined over two
 * device staging slots with the library's own copy streams: the upload of x_{k+1} and the
 * download of y_{k-1} overlap the SpMV of x_k on `stream`.  Host buffers must stay valid and
 * unmodified until the call returns (it synchronises); pinned memory is needed for the copies
 * to overlap (pageable memory works, serialised).  The same x / y pointer may repeat across k.
 * Errors: EINVAL, EUNSUPPORTED (host-only handle), ENOMEM, ECUDA. */
cbspmv_status_t cbspmv_spmv_host_batch(cbspmv_handle_t h, const void *const *x_host, void *const *y_host,
                                       int64_t count, void *stream);

/* *out_dev (one double on the device) := sum_i v_i^2 over len vector values of dtype
 * (float for CBSPMV_F32, else double; the power-iteration finalize step).  v_dev and out_dev
 * must be device memory of `device` covering len values / one double (else EDIM). */
cbspmv_status_t cbspmv_sumsq(const void *v_dev, int64_t len, cbspmv_dtype_t dtype, double *out_dev,
                             int32_t device, void *stream);

/* Steps a1 + a3 only (canonical check, then the block statistics th0 needs) for a
 * host CSR, without building: *nb_pre = non-empty 16x16 blocks, *ss_count = blocks with
 * nnz < ss_limit.  Row shards all-reduce these and pass the global decision
 * (cbspmv_decide_agg) as agg_mode to cbspmv_build. */
cbspmv_status_t cbspmv_block_stats(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr,
                                   const int32_t *col_idx, const void *vals, cbspmv_dtype_t dtype,
                                   const cbspmv_options_t *opts, int64_t *nb_pre, int64_t *ss_count);

/* *agg := 1 iff ss_count / nb_pre >= th0 (exact rational compare, R-3). */
cbspmv_status_t cbspmv_decide_agg(int64_t nb_pre, int64_t ss_count, const cbspmv_options_t *opts,
                                  int32_t *agg);

cbspmv_status_t cbspmv_get_info(cbspmv_handle_t h, cbspmv_info_t *info);

/* Canonical format (requires keep_host = 1).  With column panels this is panel 0; use
 * cbspmv_export_panel for panel k (0 <= k < info.n_panels). */
cbspmv_status_t cbspmv_export(cbspmv_handle_t h, cbspmv_export_t *ex);
cbspmv_status_t cbspmv_export_panel(cbspmv_handle_t h, int32_t k, cbspmv_export_t *ex);

/* Copy the device page stream (dev_stream_bytes) and page offsets
 * (n_pages + 1 uint64) back to host buffers of at least that size (layout
 * verification; synchronous; single-panel handles only). */
cbspmv_status_t cbspmv_download_stream(cbspmv_handle_t h, void *stream_host, size_t stream_bytes,
                                       uint64_t *page_off_host, size_t n_page_off);

/* The hot x columns of panel k (the most frequent COO columns, ascending; a
 * COO element with column hot[s] stores 0x80000000 | s in the device page stream and reads its
 * x from a shared-memory copy made at the start of each launch).  *n_hot gets their count;
 * cols_host (>= *n_hot entries) gets them, unless cols_host is NULL with n_cols 0 (a count
 * query) or *n_hot is 0.  Layout verification only;
 * synchronous.  EDIM if cols_host is too small, EINVAL for a bad panel. */
cbspmv_status_t cbspmv_hot_columns(cbspmv_handle_t h, int32_t k, uint32_t *cols_host, size_t n_cols,
                                   int64_t *n_hot);

/* ------------------------------------------------------------------ files
 * Host CSR returned by cbspmv_mm_read; its arrays are owned by the library and released
 * with cbspmv_csr_free. */
typedef struct {
  int64_t m, n, nnz;
  int64_t *row_ptr;   /* m + 1 */
  int32_t *col_idx;   /* nnz, strictly increasing within each row */
  double *vals;       /* nnz, finite and non-zero */
} cbspmv_csr_t;

/* Read a Matrix Market coordinate file (the inputs of the paper's evaluation are SuiteSparse
 * Matrix Market files; semantics of SPEC.md S:26-81): banner
 * "%%MatrixMarket matrix coordinate <real|double|integer|pattern> <general|symmetric|
 * skew-symmetric|hermitian>", 1-based indices.  Off-diagonal entries of symmetric / hermitian
 * files are mirrored (negated for skew-symmetric), pattern entries are 1.0, duplicates are
 * summed in file order (each entry, then its mirror), entries that are exactly zero after
 * summation are dropped, rows are column-sorted: the result is a canonical CSR accepted by
 * cbspmv_build.  Errors: EIO (open/read), EFORMAT (banner, size line, entry count mismatch,
 * malformed entry, index outside the declared size), EINVAL (non-finite value), EUNSUPPORTED
 * (complex field, array format, n > INT32_MAX).  On error *out is zeroed. */
cbspmv_status_t cbspmv_mm_read(const char *path, cbspmv_csr_t *out);

/* Write a CSR as "%%MatrixMarket matrix coordinate real general" with the shortest decimal form
 * that round-trips each double, so cbspmv_mm_read(cbspmv_mm_write(A)) == A bit for bit for a
 * canonical A.  Errors: EINVAL (arguments), EIO. */
cbspmv_status_t cbspmv_mm_write(const char *path, int64_t m, int64_t n, const int64_t *row_ptr,
                                const int32_t *col_idx, const double *vals);

/* Release the arrays of a CSR returned by cbspmv_mm_read (NULL-safe, idempotent). */
cbspmv_status_t cbspmv_csr_free(cbspmv_csr_t *csr);

/* Save the canonical format of every column panel in the CBSM container (magic
 * "CBSM", version 1, the five per-block arrays, cols_offset / restore_cols, mtx_data; all
 * little-endian) followed by an extension block holding dtype, warps_per_tb, the panel's
 * columns, nnz / nb_pre / ss_count and the Alg. 2 schedule (tb_ptr and per-TB loads) — layout
 * in container.cpp.  Requires keep_host = 1.  Errors: EUNSUPPORTED, EIO. */
cbspmv_status_t cbspmv_save(cbspmv_handle_t h, const char *path);

/* Load a CBSM file written by cbspmv_save (or a plain version-1 container: one fp64 panel,
 * thread blocks = consecutive groups of 8 blocks) and, for opts->device >= 0, lay it out as
 * the device page stream and upload it — steps a1..a7 are not re-run (the
 * preprocessing is a one-off cost).  Every record is decoded and its indices checked against
 * the matrix bounds before upload.  From opts only device, host_threads and keep_host are used.
 * Errors: EIO, EFORMAT (bad magic, truncated or inconsistent content), ENOMEM, ECUDA. */
cbspmv_status_t cbspmv_load(const char *path, const cbspmv_options_t *opts, void *stream,
                            cbspmv_handle_t *out);

/* Free everything the handle owns.  NULL-safe. */
cbspmv_status_t cbspmv_destroy(cbspmv_handle_t h);

/* ---------------------------------------------------------------------------------------------
 * Fused finalize + exchange of the iterated SpMV over peer memory (
 * BASELINE configs[4]: power iteration with rows sharded across the GPUs of one
 * node and x replicated; the exchange is the only communication the method needs, P:433 makes
 * block rows independent).  One context per rank.  Its single device allocation holds the two
 * iterate buffers X[0], X[1] (n values of the dtype's x type each), the per-rank flags and the
 * sum-of-squares partials; peers map it (CUDA IPC between processes, or plain device pointers
 * when several "ranks" share one process) and store into it directly over NVLink.
 *
 * Step k of rank r (rows [r0, r0 + len)), all on one stream:
 *   k >= 1: cbspmv_xchg_wait(seq = k)        -> sumsq = sum_q ||y_{k-1, q}||^2 (rank order)
 *           cbspmv_spmv_scaled(x = X[k & 1], sumsq, y = X[(k+1) & 1] + r0)
 *           cbspmv_xchg_publish(b = (k+1) & 1, r0, len, seq = k + 1)
 * publish is ONE kernel: it reads the slice once, stores it into every peer's X[b] at r0,
 * reduces its sum of squares (fixed order) and, after a system-scope fence, writes the partial
 * into every peer and releases flag[r] = seq there.  No host round trip, no NCCL.
 * Ownership: the context owns its allocation and the IPC mappings it opened; destroy frees
 * them (after a device synchronise).  Errors: EINVAL (arguments, world > 8, unconnected
 * peers), ENOMEM, ECUDA.  A wait that times out (a peer never published) poisons the
 * context: it sets the flag read by cbspmv_xchg_status, writes sumsq = NaN (the next SpMV's
 * iterate becomes NaN rather than a partly published one), and every later publish stores
 * nothing and releases no flag, so every later wait times out as well. */
#define CBSPMV_IPC_HANDLE_BYTES 64
typedef struct cbspmv_xchg_s *cbspmv_xchg_t;

/* Allocate rank `rank` of `world` (1..8) on `device` for iterates of n values (float for
 * CBSPMV_F32, else double); flags and partials zeroed, X[0] / X[1] uninitialised. */
cbspmv_status_t cbspmv_xchg_create(int64_t n, cbspmv_dtype_t dtype, int32_t world, int32_t rank, int32_t device,
                                   cbspmv_xchg_t *out);
/* The allocation's CUDA IPC handle (CBSPMV_IPC_HANDLE_BYTES bytes) for peers in other processes. */
cbspmv_status_t cbspmv_xchg_ipc_handle(cbspmv_xchg_t x, void *handle_out);
/* Device base pointer of the allocation (peers in the same process pass it to connect). */
void *cbspmv_xchg_base(cbspmv_xchg_t x);
/* Map every peer q != rank: peer_bases[q] if non-NULL (same process), else open
 * ipc_handles + q * CBSPMV_IPC_HANDLE_BYTES (world handles, this rank's entry ignored). */
cbspmv_status_t cbspmv_xchg_connect(cbspmv_xchg_t x, void *const *peer_bases, const void *ipc_handles);
/* Device pointer of iterate buffer b (0 or 1), n values. */
void *cbspmv_xchg_buffer(cbspmv_xchg_t x, int32_t b);
/* The fused finalize + all-gather described above; seq >= 1 (= the step number + 1). */
cbspmv_status_t cbspmv_xchg_publish(cbspmv_xchg_t x, int32_t b, int64_t r0, int64_t len, uint64_t seq,
                                    void *stream);
/* Device-side wait (system-scope acquire, bounded by timeout_s; <= 0: 10 s) for every rank's
 * flag >= seq, then *sumsq_dev = the partials of step seq - 1 summed in rank order. */
cbspmv_status_t cbspmv_xchg_wait(cbspmv_xchg_t x, uint64_t seq, double *sumsq_dev, double timeout_s, void *stream);
/* *timed_out = 1 if any wait so far timed out (synchronous read). */
cbspmv_status_t cbspmv_xchg_status(cbspmv_xchg_t x, int32_t *timed_out);
/* NULL-safe. */
cbspmv_status_t cbspmv_xchg_destroy(cbspmv_xchg_t x);

const char *cbspmv_status_string(cbspmv_status_t s);
const char *cbspmv_last_error(void);
int32_t cbspmv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CBSPMV_H */
