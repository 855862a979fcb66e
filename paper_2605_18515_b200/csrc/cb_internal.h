// cb_internal.h — shared internals of libcbspmv (host builder, C ABI, kernels).
// Product path only; nothing here is shared with oracle/.
#pragma once
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <functional>
#include <memory>
#include <utility>
#include <string>
#include <vector>

#include "cbspmv.h"

namespace cb {

// ---------------------------------------------------------------------------
// Device page stream.  A derived layout of the canonical
// format: blocks in slot order (after Alg. 2), whole thread blocks per page,
//   page = header | desc[nblk] | item[nitems] (u32 words, see item_word) | records
// every record 16-byte aligned and preceded by its block's restore_cols entries
// when aggregated.  One cp.async.bulk moves a whole page into a
// shared-memory stage; the page's x tiles (16 values per block, gathered on the
// device) follow it in the same stage, so pages are sized by
// bytes + 16 * size(Val) * nblk <= stage capacity.  Work items: a COO group
// (consecutive COO blocks whose nnz sum to <= 32, one warp, one lane per element)
// or a single CSR / DENSE block.
// ---------------------------------------------------------------------------
constexpr int kPageHeader = 16;         // u32 nblk, u32 nitems, u32 item_off, u32 x_off (x tiles in the stage)
constexpr int kDescBytes = 16;          // see Desc
constexpr int kDefaultStageCap = 28672;     // 8 stages in one CTA/SM; >= one fp64 TB of 8 dense blocks + tiles
constexpr int kMaxPageCap = 65536;      // descriptor offsets are u16 bytes
constexpr int kCtrSlots = 64;           // page-claim counters per panel (launch k uses slot k % 64)

// 16-byte block descriptor, read with one 128-bit shared load.  All offsets are bytes from
// the page start, precomputed on the host so the kernel does no record parsing.
struct Desc {
  uint32_t row0;    // blk_row_idx * 16: y row base
  uint32_t xinfo;   // without aggregation: blk_col_idx * 16 (x tile base);
                    // with aggregation: page offset of the block's restore_cols entries
  uint32_t offs;    // [0,16) page offset of the canonical record; [16,32) page offset of its values
  uint32_t w;       // [0,8) nnz - 1; [8,10) type; [11,16) group size - 1 (on a group head);
                    // [16,21) ncols (valid x-tile columns, 0..16); [24] group head;
                    // [25,30) first lane of the block within its COO group
};
constexpr uint32_t kFlagHead = 1u << 24;

// Work-item word (page item table, one u32 per item):
//   [0,12) head block index in the page; [12,14) type; [14,16) members - 1;
//   [16,21), [21,26), [26,31) first lane of members 1, 2, 3 of a COO group;
//   [31] a single COO block with nnz > 32 (processed in 32-element chunks)
constexpr int kGroupMembers = 4;
inline uint32_t item_word(uint32_t head, uint32_t type, uint32_t members, bool big) {
  return head | (type << 12) | ((members - 1u) << 14) | (big ? 1u << 31 : 0u);
}

inline uint32_t pack_w(uint32_t nnz, uint32_t type, uint32_t ncols, bool head, uint32_t gsize, uint32_t lane0) {
  return (nnz - 1u) | (type << 8) | ((gsize - 1u) << 11) | (ncols << 16) | (head ? kFlagHead : 0u) | (lane0 << 25);
}

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Allocator whose value-initialisation is a no-op: resize() of a multi-GB byte buffer leaves the
// pages untouched, so their first touch happens in the parallel fill threads.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U> struct rebind { using other = NoInitAlloc<U>; };
  NoInitAlloc() = default;
  template <class U> NoInitAlloc(const NoInitAlloc<U> &) noexcept {}
  template <class U> void construct(U *p) noexcept { ::new ((void *)p) U; }
  template <class U, class... Args> void construct(U *p, Args &&...a) { ::new ((void *)p) U(std::forward<Args>(a)...); }
};
using ByteBuf = std::vector<uint8_t, NoInitAlloc<uint8_t>>;

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
  ByteBuf mtx;  // every byte written by pack_record (records and their padding)
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

// a1 only (options + canonical check of the whole CSR).
int check_csr(const Csr &A, const cbspmv_options_t &o, int64_t *nnz, std::string *err);
// a1 + a3 only: canonical check and pre-aggregation block statistics.
int block_stats(const Csr &A, const cbspmv_options_t &o, int64_t *nb_pre, int64_t *ss_count, std::string *err);
bool decide_agg(int64_t nb_pre, int64_t ss_count, const cbspmv_options_t &o);

// Host pipeline a1..a7.  Returns a cbspmv_status_t; *err gets the detail.
int build_canonical(const Csr &A, const cbspmv_options_t &o, Canon *out, std::string *err);

// Device page stream built from the canonical format.
struct Stream {
  uint8_t *bytes = nullptr;        // host staging: malloc (default) or cudaHostAlloc (CBSPMV_PINNED_STREAM)
  bool pinned = false;
  int64_t nbytes = 0;
  std::vector<uint64_t> page_off;  // n_pages + 1
};
// Device-fill plan of the page stream (device builder): the page prefixes (header | descriptors |
// items) in a compact buffer, and per slot-order block the stream offsets of its record and restore
// entries; the records themselves are copied on the device (fill_stream_device).
struct StreamPlan {
  std::vector<uint8_t> meta;
  std::vector<uint64_t> meta_off;          // n_pages + 1
  std::vector<uint64_t> rec_dst, res_dst;  // per block (res_dst only when aggregated)
  std::vector<int32_t> ncol;               // x-tile columns per block
};
// x_size: bytes of one x element (sizes the non-aggregated x tiles that follow each page).
// plan == nullptr: the whole stream is written to host memory (s->bytes); otherwise only the plan.
// hub_nnz > 0: grouped COO blocks of block rows with >= hub_nnz entries get flag bit 0 in
// desc.row0 (the kernel sums their same-row runs before the RED).
int build_stream(const Canon &c, int page_cap, int x_size, int threads, Stream *s, StreamPlan *plan,
                 std::string *err, int64_t hub_nnz = 0);

// Device-resident canonical arrays kept by the device builder for fill_stream_device.
struct DevCanon {
  uint8_t *mtx = nullptr;
  uint32_t *restore = nullptr;
  uint64_t *cols_offset = nullptr;
  void release();
  ~DevCanon() { release(); }
};
// Write the device page stream (d_stream, s.nbytes) from the plan and the device-resident records
// (gpu_builder.cu): page prefixes, restore entries, records (DENSE in the lane-major layout).
int fill_stream_device(const Canon &c, const DevCanon &dc, const Stream &s, const StreamPlan &plan, void *stream,
                       uint8_t *d_stream, std::string *err);
void free_stream(Stream *s);

// Matrix Market coordinate files (mmio.cpp)
int mm_read(const char *path, int threads, cbspmv_csr_t *out, std::string *err);
int mm_write(const char *path, int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
             const double *vals, std::string *err);

// CBSM container (container.cpp) + this library's extension block
struct CbsmExt {
  int dtype = CBSPMV_F64;
  int panel = 0, n_panels = 1;
  int64_t c0 = 0, c1 = 0;  // the panel's columns [c0, c1)
};
int write_cbsm(FILE *f, const Canon &c, const CbsmExt &x, std::string *err);
int read_cbsm(FILE *f, Canon *out, CbsmExt *x, std::string *err);  // validates (validate_canon)
int validate_canon(const Canon &c, const CbsmExt &x, std::string *err);

// Phase timing of the builders (env CBSPMV_BUILD_TIMING=1 prints to stderr).
struct PhaseTimer {
  bool on = std::getenv("CBSPMV_BUILD_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char *what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cbspmv build] %-28s %8.3f s\n", what, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

// a7 + permute on natural-order block arrays (builder.cpp; shared by the host and device builders)
void balance_and_permute(Canon &c, const cbspmv_options_t &o, const int32_t *nbr, const int32_t *nbc,
                         const int32_t *nnzb, const uint8_t *ntype, const uint64_t *nvp, PhaseTimer &tm);

// Steps a2..a6 on the GPU (gpu_builder.cu, NEXT-3): the same canonical format as build_canonical,
// byte for byte; a1 runs on the host first, a7 on the host after.
// dc != nullptr: the records, restore_cols and cols_offset stay on the device in *dc (for
// fill_stream_device) and are downloaded into *out only when download_records is set.
int build_canonical_device(const Csr &A, const cbspmv_options_t &o, void *stream, Canon *out, DevCanon *dc,
                           bool download_records, std::string *err);

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
  int groups = 1;
  int consumers = 0;
  int coo_runs = 0;  // hub block rows present: the kernel variant that sums their COO runs
  const uint8_t *d_stream = nullptr;
  const uint64_t *d_page_off = nullptr;
  const uint32_t *d_cta_page = nullptr;  // grid + 1 page boundaries per persistent CTA
  uint32_t *d_page_ctr = nullptr;         // dynamic page claiming: kCtrSlots x {next page, done}
  mutable uint32_t ctr_next = 0;          // slot of the next launch, taken with an atomic fetch-add:
                                          // up to kCtrSlots launches in flight (any streams, any host
                                          // threads) get their own counters.  A captured CUDA graph
                                          // bakes one slot into its kernel node, so replays of one
                                          // graph must not run concurrently with each other.
};

// Choose grid / stages for this device; fills dev->grid, nstage, consumers.
int cb_configure(CbDevice *dev, std::string *err);
// y (+)= A·(s·x); zero_y: clear y first; sumsq: nullptr or device double (s = 1/sqrt(*sumsq)).
int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y,
                   void *stream, std::string *err);
int cb_launch_sumsq(const void *v, int64_t len, int dtype, double *out, void *stream, std::string *err);
// Record msg as cbspmv_last_error() and return st (capi.cpp owns the thread-local string).
int cb_set_error(int st, const std::string &msg);
