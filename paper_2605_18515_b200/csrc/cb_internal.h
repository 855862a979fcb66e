// cb_internal.h — shared internals of libcbspmv (host builder, C ABI, kernels).
// Product path only; nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "cbspmv.h"

namespace cb {

// ---------------------------------------------------------------------------
// Device page stream.  A derived layout of the canonical
// format: blocks in slot order (after Alg. 2), whole thread blocks per page,
// each page = header | desc[nblk] | records, every record 16-byte aligned and
// prefixed by its block row's restore_cols entries when aggregated.
// One cp.async.bulk moves a whole page into shared memory.
// ---------------------------------------------------------------------------
constexpr int kPageHeader = 16;     // u32 nblk, u32 first_tb, u32 tb_count, u32 reserved
constexpr int kDescBytes = 16;      // see Desc
constexpr int kDefaultPageCap = 17408;  // >= 16 + 8*16 + 8*(64 + 2048): one fp64 TB of 8 dense blocks
constexpr int kMaxPageCap = 65536 * 16 - 16;  // record offsets are u16 in 16-byte units

// 16-byte block descriptor, read with one 128-bit shared load.
struct Desc {
  uint32_t row0;    // blk_row_idx * 16
  uint32_t xcol0;   // blk_col_idx * 16 without aggregation, 0 with it
  uint32_t w2;      // [0,16) record offset / 16 from page start; [16,24) nnz - 1; [24,26) type
  uint32_t ncols;   // valid x-tile columns (restore entries when aggregated), 0..16
};

inline uint32_t pack_w2(uint32_t rec_off16, uint32_t nnz, uint32_t type) {
  return rec_off16 | ((nnz - 1u) << 16) | (type << 24);
}

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// Canonical format (slot order), byte-identical to the paper-literal CPU reference build
// (checked by tests/test_builder_parity.py).
// ---------------------------------------------------------------------------
struct Canon {
  int64_t m = 0, n = 0, nnz = 0, nb = 0, nb_pre = 0, ss_count = 0, blk_m = 0, T = 0;
  int blk = 16, agg = 0, val_size = 8, W = 8;
  std::vector<int32_t> br, bc, nnzb;
  std::vector<uint8_t> type;
  std::vector<uint64_t> vp;
  std::vector<uint8_t> mtx;
  std::vector<uint32_t> restore;
  std::vector<uint64_t> cols_offset;
  std::vector<int64_t> tb_ptr, tb_load, tb_load_nat;
  int64_t fmt_count[3] = {0, 0, 0};
};

struct Csr {
  int64_t m, n, nnz;
  const int64_t *row_ptr;
  const int32_t *col;
  const void *val;
  int val_size;  // 8 = double, 4 = float
};

// a1 + a3 only: canonical check and pre-aggregation block statistics.
int block_stats(const Csr &A, const cbspmv_options_t &o, int64_t *nb_pre, int64_t *ss_count, std::string *err);
bool decide_agg(int64_t nb_pre, int64_t ss_count, const cbspmv_options_t &o);

// Host pipeline a1..a7.  Returns a cbspmv_status_t; *err gets the detail.
int build_canonical(const Csr &A, const cbspmv_options_t &o, Canon *out, std::string *err);

// Device page stream built from the canonical format.
struct Stream {
  uint8_t *bytes = nullptr;        // pinned host staging (cudaHostAlloc) or malloc
  bool pinned = false;
  int64_t nbytes = 0;
  std::vector<uint64_t> page_off;  // n_pages + 1
};
int build_stream(const Canon &c, int page_cap, int threads, Stream *s, std::string *err);
void free_stream(Stream *s);

// Threads
void parallel_for(int64_t n, int threads, int64_t grain, const std::function<void(int64_t, int64_t, int)> &fn);
int resolve_threads(int t);

}  // namespace cb

// ---------------------------------------------------------------------------
// Kernel launch interface (kernels.cu)
// ---------------------------------------------------------------------------
struct CbDevice {
  int device = -1;
  int dtype = 0;
  int agg = 0;
  int64_t m = 0, n = 0;
  int64_t n_pages = 0;
  int page_cap = 0;
  int grid = 0;
  int nstage = 0;
  int consumers = 0;
  const uint8_t *d_stream = nullptr;
  const uint64_t *d_page_off = nullptr;
  const uint32_t *d_cta_page = nullptr;  // grid + 1 page boundaries per persistent CTA
};

// Choose grid / stages for this device; fills dev->grid, nstage, consumers.
int cb_configure(CbDevice *dev, std::string *err);
// y (+)= A·(s·x); zero_y: clear y first; sumsq: nullptr or device double (s = 1/sqrt(*sumsq)).
int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y,
                   void *stream, std::string *err);
int cb_launch_sumsq(const void *v, int64_t len, int dtype, double *out, void *stream, std::string *err);
