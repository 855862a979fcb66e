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

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost ~nothing without a profiler attached

namespace cb {

// NVTX range for the scope (build / upload / SpMV / exchange phases show up in nsys / ncu timelines)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---------------------------------------------------------------------------
// Device page stream, version 3.  A derived layout of the canonical format:
// the slot-order blocks (after Alg. 2) are cut into pages of consecutive blocks; one
// cp.async.bulk moves a page into a shared-memory stage, and the page's x values (gathered by
// the x warps) follow it in the same stage, so a page is sized by page bytes + x area <= stage.
//   page = header | item descriptors (16 B each) | slice tables | (pad 16)
//          | CSR / DENSE records (16-B aligned each) | slice elements
//   header: u32 nitems | u32 ncd (CSR / DENSE items; they come first, then the COO slices)
//           | u32 nblk | u32 blk0 (the page's slot-order blocks [blk0, blk0 + nblk))
// Work items:
//   * a CSR or DENSE block (the canonical record; DENSE values re-laid lane-major in 16-byte
//     pairs; with aggregation its restore_cols entries precede the record);
//   * a COO slice (row-run slices, a jagged-diagonal layout per page): the elements of the page's
//     COO blocks, each with its original column resolved (restore_cols[cols_offset[br] + bc*16 + c]
//     with aggregation, bc*16 + c without), are grouped by global row (a run: the row's elements
//     in slot order, then canonical (row, col) order); runs longer than Lmax are cut into pieces
//     of Lmax; the pieces are ordered (length desc, row asc) and dealt 32 to a slice, one per
//     lane.  Lane l of a slice owns piece l (row rows[l], lens[l] elements); step j holds the
//     j-th element of every lane whose piece is longer than j, in lane order:
//       element (l, j) at index off_j + popc(act_j & lanes_below(l)),
//       act_j = {lanes with lens > j}, off_j = sum_{j' < j} popc(act_j').
//     slice table = rows u32[nl] | lens u8[nl] (pad 4);  slice elements = cols u32[E] (pad 8)
//     | vals[E] (pad 8).  The kernel sums a piece in its lane and issues one RED per piece.
// Item descriptor (uint4 a, b, c, d); d[0,2) type:
//   CSR / DENSE: a = br*16; b = bc*16 (x tile base) or, aggregated, the page offset of the
//                restore entries; c = record offset | values offset << 16;
//                d[2,7) ncols (valid x-tile columns), d[8,16) nnz - 1, d[16,32) x tile offset
//                in the stage (non-aggregated only: 16 values after the page, filled by TMA)
//   COO slice:   a = table offset | nl << 16 | w << 24 (w = longest piece); b = cols offset |
//                vals offset << 16; c = E (elements); d = 0
// Hot x columns: when a few columns carry a large share of the COO elements (power-law graphs),
// the builder lists the H most frequent ones (Stream::hot_cols, ascending) and a slice element
// whose column is hot stores kHotBit | slot instead of the column; each CTA copies x[hot_cols[]]
// into shared memory at the start of a launch and reads those elements' x from there.
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
#define CB_HD __host__ __device__
#else
#define CB_HD
#endif
constexpr int kPageHeader = 16;
constexpr int kDescBytes = 16;
constexpr int kSliceLanes = 32;
constexpr int kMaxRun = 255;               // piece length is a u8 (lens[], desc w)
constexpr int kDefaultRunMax = 8;          // Lmax (env CBSPMV_RUN_MAX, read per build)
constexpr uint32_t kEndItems = 0xFFFFFFFFu;  // header.nitems of the dynamic-claiming end marker
constexpr int kMaxPageCap = 65536;         // descriptor offsets are u16 bytes
constexpr int kCtrSlots = 64;              // page-claim counters per panel (launch k uses slot k % 64)
constexpr uint32_t kHotBit = 0x80000000u;  // slice column = kHotBit | slot of a hot x column
constexpr int kDefaultHotBytes = 65536;    // shared x cache (env CBSPMV_HOT_BYTES, read per build)
constexpr int kDefaultHotMinPct = 5;       // cache only if it serves >= this share of the COO elements

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
// bytes of a slice table (rows u32[nl] | lens u8[nl], 4-aligned) and of its elements (cols u32[E]
// padded to 8 | vals[E] padded to 8)
inline int64_t slice_table_bytes(int64_t nl) { return round_up(5 * nl, 4); }
inline int64_t slice_elem_bytes(int64_t E, int val_size) { return round_up(4 * E, 8) + round_up(val_size * E, 8); }

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
  std::vector<uint32_t> hot_cols;  // hot x columns (ascending; slot = index), empty: no x cache
};
// Device-fill plan of the page stream (device builder): the page prefixes (header | item
// descriptors | slice tables) in a compact buffer, per slot-order block the stream offset of its
// record (CSR / DENSE; COO: its page) and restore entries (aggregated), per COO block the index of
// its first element and per COO element its column / value offsets in the page; the records and
// the slice elements themselves are written on the device.
struct StreamPlan {
  std::vector<uint8_t> meta;
  std::vector<uint64_t> meta_off;          // n_pages + 1
  std::vector<uint64_t> rec_dst, res_dst;  // per block: record (COO: page) / restore entries
  std::vector<int32_t> ncol;               // x-tile columns per block
  std::vector<int64_t> coo_e0;             // per block: first element in coo_dst (COO), -1 otherwise
  std::vector<uint32_t> coo_dst;           // per COO element (slot order, canonical order within
                                           // its block): col offset | val offset << 16 in the page
};
// Coordinate bytes ((col << 4) | row) of the slot-order COO blocks when the records
// stay on the device (device builder): block i's at bytes[off[i] ..] (off[i] = -1: not COO).
struct CooCoords {
  ByteBuf bytes;
  std::vector<int64_t> off;
};
// Row-run slices of the page stream (cb_internal.h layout): Lmax and the piece order.
struct SliceOpts {
  int run_max = kDefaultRunMax;  // 1: every element its own piece (no in-lane run sums; A/B)
  int row_order = 0;             // 0: pieces by (length desc, row asc); 1: by row asc
  int hot_bytes = kDefaultHotBytes;   // shared x cache budget (0: none)
  int hot_min_pct = kDefaultHotMinPct;
};
// x_size: bytes of one x element (sizes the x area that follows each page in its stage).
// plan == nullptr: the whole stream is written to host memory (s->bytes); otherwise only the plan.
// coords: the COO coordinate bytes when c.mtx does not hold the records (nullptr: c.mtx).
// xagg: aggregated CSR / DENSE items also get an x-tile slot after the page (filled by the x warps).
int build_stream(const Canon &c, int page_cap, int x_size, int threads, Stream *s, StreamPlan *plan,
                 std::string *err, const SliceOpts &so = SliceOpts(), const CooCoords *coords = nullptr,
                 bool xagg = false);

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
// (hot x columns: the slice columns are encoded from s.hot_cols on the device as well)
int fill_stream_device(const Canon &c, const DevCanon &dc, const Stream &s, const StreamPlan &plan, void *stream,
                       uint8_t *d_stream, std::string *err);
// The coordinate bytes of the slot-order COO blocks from the device-resident records.
int download_coo_coords(const Canon &c, const DevCanon &dc, void *stream, CooCoords *out, std::string *err);
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
// Launch shape of the persistent kernel (kernels.cu cb_plan_stages): S stages of page_cap bytes,
// G consumer groups (G divides S) of W warps, X x warps (X <= G).
struct CbShape {
  int nstage = 12, groups = 4, gwarps = 7, xwarps = 3, page_cap = 19008;
  int hot_cap = 0;  // shared memory left for the hot x cache (bytes)
  int xagg = 0;     // aggregated matrix whose CSR / DENSE tiles the x warps gather (restore entries)
};

struct CbDevice : CbShape {
  int device = -1;
  int n_hot = 0;                          // hot x columns (shared x cache), 0: none
  const uint32_t *d_hot = nullptr;        // their indices (device)
  int dtype = 0;
  int agg = 0;
  int64_t m = 0, n = 0;
  int64_t n_pages = 0;
  int grid = 0;
  int sms = 0;
  int dynamic = 0;           // dynamic page claiming (large aggregated matrices)
  int strided = 0;           // static: runs of K pages dealt round robin (0: contiguous ranges)
  uint32_t claim_chunk = 8;  // pages per dynamic claim
  int dbg_skip = 0;          // ablation build only (CBSPMV_DEBUG_SKIP)
  uint32_t sleep_ns = 0;     // consumer / x-warp back-off between mbarrier probes (CBSPMV_WAIT_SLEEP_NS)
  int pdl = 1;               // launch the SpMV dependent on the y-zeroing kernel (CBSPMV_PDL=0: off)
  int csr_pair = 0;          // two CSR blocks per warp, one lane per row (non-aggregated; CBSPMV_CSR_PAIR)
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

// Stage shape for a device (env CBSPMV_STAGES / CBSPMV_GROUPS / CBSPMV_GROUP_WARPS /
// CBSPMV_PAGE_BYTES override the measured defaults; read per build).
// agg_tiles: an aggregated matrix with many CSR / DENSE blocks (their x tiles are then gathered
// by x warps into the stage, as for non-aggregated matrices).
int cb_plan_stages(int device, int agg, bool agg_tiles, CbShape *sh, std::string *err);
// Grid and page assignment for this device and stream (dev's shape already planned).
int cb_configure(CbDevice *dev, std::string *err);
// y (+)= A·(s·x); zero_y: clear y first; sumsq: nullptr or device double (s = 1/sqrt(*sumsq));
// follows: this launch follows another panel's launch of the same SpMV on the stream (PDL overlap).
int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y,
                   void *stream, std::string *err, bool follows = false);
int cb_launch_sumsq(const void *v, int64_t len, int dtype, double *out, void *stream, std::string *err);
// Record msg as cbspmv_last_error() and return st (capi.cpp owns the thread-local string).
int cb_set_error(int st, const std::string &msg);
