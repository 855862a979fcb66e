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
// Device page stream, version 2.  A derived layout of the canonical format:
// the slot-order blocks (after Alg. 2) are cut into pages of consecutive blocks; one
// cp.async.bulk moves a page into a shared-memory stage, and the page's x values (gathered by
// the x warp) follow it in the same stage, so a page is sized by page bytes + x area <= stage.
//   page = header | item descriptors (16 B each) | item records (16-B aligned)
//   header: u32 nitems | u32 ncd (CSR / DENSE items; they come first, then the COO chunks)
//           | u32 nblk | u32 blk0 (the page's slot-order blocks [blk0, blk0 + nblk))
// Work items:
//   * a CSR or DENSE block (the canonical record; DENSE values re-laid lane-major in 16-byte
//     pairs; with aggregation its restore_cols entries precede the record);
//   * a COO chunk: up to 32 elements of the page's COO blocks, taken in slot order (a block may
//     continue into the next chunk), each element with its original column resolved
//     (restore_cols[cols_offset[br] + bc*16 + c] with aggregation, bc*16 + c without) and a row
//     byte (member << 4 | local row) indexing the chunk's table of member row bases (<= 16).
//     chunk record = rowbase u32[nm] | rows u8[nv] (pad 4) | cols u32[nv] (pad to size(Val))
//                    | vals[nv]; 16-byte aligned.
// Item descriptor (uint4 a, b, c, d); d[0,2) type:
//   CSR / DENSE: a = br*16; b = bc*16 (x tile base) or, aggregated, the page offset of the
//                restore entries; c = record offset | values offset << 16;
//                d[2,7) ncols (valid x-tile columns), d[8,16) nnz - 1, d[16,32) x tile offset
//                in the stage (non-aggregated only: 16 values after the page, filled by TMA)
//   COO chunk:   a = rowbase offset | nv << 16 | nm << 24; b = rows offset | cols offset << 16;
//                c = values offset; d[2,5) run steps: ceil(log2(longest run of adjacent
//                elements sharing a global row)), 0 = no run; the kernel sums each run in the
//                warp with that many shuffle steps before the RED
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
#define CB_HD __host__ __device__
#else
#define CB_HD
#endif
constexpr int kPageHeader = 16;
constexpr int kDescBytes = 16;
constexpr int kChunkLanes = 32;
constexpr int kChunkMembers = 16;          // member index is 4 bits of the row byte
constexpr uint32_t kEndItems = 0xFFFFFFFFu;  // header.nitems of the dynamic-claiming end marker
constexpr int kMaxPageCap = 65536;         // descriptor offsets are u16 bytes
constexpr int kCtrSlots = 64;              // page-claim counters per panel (launch k uses slot k % 64)
constexpr int kRunShift = 2;  // desc.d[2,5): run steps (0..5)
// steps of a segmented warp sum covering runs of up to maxrun lanes: ceil(log2(maxrun))
CB_HD inline uint32_t run_steps(int maxrun) {
  uint32_t s = 0;
  while ((1 << s) < maxrun) s++;
  return s;
}

struct ChunkLayout {
  int rows, cols, vals, bytes;  // offsets from the chunk record start; total (16-aligned)
};
CB_HD inline ChunkLayout chunk_layout(int nv, int nm, int val_size) {
  ChunkLayout L;
  L.rows = 4 * nm;
  L.cols = L.rows + ((nv + 3) & ~3);
  L.vals = (L.cols + 4 * nv + val_size - 1) / val_size * val_size;
  L.bytes = (L.vals + val_size * nv + 15) & ~15;
  return L;
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
// Device-fill plan of the page stream (device builder): the page prefixes (header | item
// descriptors) in a compact buffer, per slot-order block the stream offset of its record (CSR /
// DENSE) and restore entries (aggregated), per COO block its first chunk / lane / member, and per
// chunk its record offset and shape; the records themselves are written on the device.
struct StreamPlan {
  std::vector<uint8_t> meta;
  std::vector<uint64_t> meta_off;          // n_pages + 1
  std::vector<uint64_t> rec_dst, res_dst;  // per block: record / restore entries (COO: unused)
  std::vector<int32_t> ncol;               // x-tile columns per block
  std::vector<int64_t> coo_chunk;          // per block: first chunk (COO), -1 otherwise
  std::vector<uint8_t> coo_lane, coo_member;
  std::vector<uint64_t> chunk_off;         // per chunk: stream offset of its record
  std::vector<uint64_t> chunk_desc;        // per chunk: stream offset of its descriptor
  std::vector<uint8_t> chunk_nv, chunk_nm;
  bool runs = true;                        // set the runs flags (fill_stream_device)
};
// x_size: bytes of one x element (sizes the x area that follows each page in its stage).
// plan == nullptr: the whole stream is written to host memory (s->bytes); otherwise only the plan.
// runs = false: no chunk gets the runs flag (A/B of the in-warp run sums).
int build_stream(const Canon &c, int page_cap, int x_size, int threads, Stream *s, StreamPlan *plan,
                 std::string *err, bool runs = true);

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
// Launch shape of the persistent kernel (kernels.cu cb_plan_stages): S stages of page_cap bytes,
// G consumer groups (G divides S) of W warps, X x warps (X <= G).
struct CbShape {
  int nstage = 12, groups = 4, gwarps = 7, xwarps = 3, page_cap = 19008;
};

struct CbDevice : CbShape {
  int device = -1;
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
int cb_plan_stages(int device, int agg, CbShape *sh, std::string *err);
// Grid and page assignment for this device and stream (dev's shape already planned).
int cb_configure(CbDevice *dev, std::string *err);
// y (+)= A·(s·x); zero_y: clear y first; sumsq: nullptr or device double (s = 1/sqrt(*sumsq)).
int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y,
                   void *stream, std::string *err);
int cb_launch_sumsq(const void *v, int64_t len, int dtype, double *out, void *stream, std::string *err);
// Record msg as cbspmv_last_error() and return st (capi.cpp owns the thread-local string).
int cb_set_error(int st, const std::string &msg);
