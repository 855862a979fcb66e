// kernels.cu — sm_100a kernels of the CB-SpMV hot path (y = A·x, §3.5).
//
// One persistent CTA per SM streams its pages of the device page stream (cb_internal.h,
// DESIGN.md §4) through a ring of S shared-memory stages, with three warp roles:
//   warp 0 (one elected lane): TMA producer — waits on the stage's "empty" mbarrier, then one
//       cp.async.bulk (SASS UBLKCP) per page, L2 evict_first (the matrix stream must not evict
//       x); completion counted on the stage's "full" mbarrier.
//   warps 1..X: x warps (non-aggregated matrices) — as each page lands, load the 16-value x
//       tiles x[bc*16 ..] of its CSR / DENSE blocks (the paper's shared-memory s_x, P:517,
//       P:571) into the stage's x area and arrive on the stage's "xready" mbarrier.
//   G consumer groups of W warps: page i of the CTA goes to stage i % S and group i % G; G
//       divides S, so each stage is always consumed by the same group, round after round, and
//       the mbarrier parity waits are exact.  Warp w of a group takes the group's work items
//       w, w + W, ... counted across its pages (no per-page restart), and arrives on "empty"
//       after its last item of each page.  y is accumulated with red.global.add — the paper's
//       atomicAdd:
//       * COO slice (Alg. 3, over row-run pieces): lane <-> piece of a row's run,
//         x[col] gathered into a register (four slices' loads in flight per warp), the piece
//         summed in the lane, one RED per piece;
//       * CSR ("32 threads collaboratively compute 16 y elements"): two lanes per
//         row, one shfl_xor; x tile from the stage (aggregated: gathered through the restore
//         entries into the warp's scratch);
//       * DENSE (Alg. 4): lane-major 16-byte pairs, 8 FMAs per lane, one
//         shfl_xor(16) joins the half rows (R-15 semantics), 16 REDs.
// y is zeroed by cb_zero_kernel first (R-16).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "cb_internal.h"

namespace {

constexpr int kMaxThreads = 1024;
constexpr int kMaxStages = 32;
constexpr int kSmemHeader = 1024;  // mbarriers: full[32], xready[32], empty[32]; the scale at 768
constexpr int kScaleSlot = 3 * 32 * 8;
constexpr int kAggPageBytes = 20480;  // stage bytes of aggregated matrices (the rest of the array is L1)
constexpr unsigned kFull = 0xffffffffu;
// End marker of dynamic page claiming: a 16-byte page header (nitems = kEndItems) copied into
// the stage by the same TMA path as a page, so the marker is synchronised exactly like data.
__device__ __align__(16) const uint32_t kEndHeader[4] = {cb::kEndItems, 16u, 0u, 0u};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// consumer / x-warp wait: optionally back off between probes (fewer issued spin instructions)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
  while (!mbar_try_wait(bar, parity)) {
    if (ns) __nanosleep(ns);
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D TMA bulk copy global -> shared, completion on an mbarrier (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
// Ablation knob for profiling only: built with -DCBSPMV_ABLATION=1 the env CBSPMV_DEBUG_SKIP
// (a kernel argument) drops the y atomics (bit 0), the x loads (bit 1: x warps' tiles and the
// COO chunks' gathers) or the item processing (bit 2).  In the production build every test folds away.
#ifndef CBSPMV_ABLATION
#define CBSPMV_ABLATION 0
#endif
struct Dbg {
  int skip_;
  __device__ __forceinline__ int skip() const { return CBSPMV_ABLATION ? skip_ : 0; }
};
// Bounds-checking debug build (-DCBSPMV_CHECK=1, tools/build_variant.sh; compute-sanitizer is not
// available on the B200 pool): every page offset, slice element index, column, hot slot and row
// the kernel derives from the stream is checked, and a violation traps (the launch fails with an
// illegal-instruction error instead of reading or writing out of bounds).  Folds away otherwise.
#ifndef CBSPMV_CHECK
#define CBSPMV_CHECK 0
#endif
#define CB_CHECK(cond)                                  \
  do {                                                  \
    if (CBSPMV_CHECK && !(cond)) {                      \
      printf("cbspmv check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
      __trap();                                         \
    }                                                   \
  } while (0)

template <typename V>
__device__ __forceinline__ void red_add(V *p, V v, Dbg dbg) {
  if (dbg.skip() & 1) {
    if (v == V(12345.678)) *p = v;  // keep the value live without the atomic
    return;
  }
  atomicAdd(p, v);  // result unused -> RED.E.ADD
}

template <typename T> struct Pair;
template <> struct Pair<double> { using type = double2; };
template <> struct Pair<float> { using type = float2; };

// ------------------------------------------------------------------ per-format warp paths
// x gathered straight into a register, L2 evict_last (x is re-read; the matrix stream is evict_first)
template <typename V>
__device__ __forceinline__ V ldg_x(const V *p, uint64_t pol) {
  V v;
  if constexpr (sizeof(V) == 8)
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// 32-bit shared-memory loads (the page lives in the CTA's shared window: no 64-bit generic
// address arithmetic per element)
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
template <typename M>
__device__ __forceinline__ M lds_val(uint32_t a) {
  M v;
  if constexpr (sizeof(M) == 8) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  else asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// COO slices (Alg. 3, over row-run pieces; layout in cb_internal.h): lane l owns piece
// l of the slice — rows[l], lens[l] elements of one row — and walks it step by step: at step j the
// lanes whose piece is longer than j read their element (index off_j + rank among those lanes),
// gather x[col] into a register (ld.global.nc, L2 evict_last) and accumulate; then one RED per
// piece (Alg. 3's atomicAdd).  B slices (items da0, da0 + dstride, ...) advance together so B
// gathers per lane are in flight.  An element whose column carries kHotBit reads its x from the
// CTA's shared copy of the hot x columns (hotx: its shared address).
struct Bounds {  // for the CBSPMV_CHECK build
  uint32_t stage;  // bytes of a stage (page + x area)
  int64_t m, n;
  int n_hot;
};

template <typename M, typename V, bool SCALED, int B, int U>
__device__ __forceinline__ void coo_slices(uint32_t pg, uint32_t da0, uint32_t dstride, const V *__restrict__ x,
                                           uint32_t hotx, V *__restrict__ y, uint32_t sc, int lane, uint64_t pol, Dbg dbg,
                                           const Bounds &bd) {
  constexpr int N = B * U;  // elements per lane in flight: B slices x U steps
  uint32_t cv[B], off[B], row[B];  // cv: cols offset | vals offset << 16 (page-relative)
  int len[B];
  V acc[B];
  int wmax = 0;
#pragma unroll
  for (int b = 0; b < B; b++) {
    const uint4 d = lds_v4(da0 + (uint32_t)b * dstride);
    const uint32_t nl = (d.x >> 16) & 0xFF, tab = pg + (d.x & 0xFFFFu);
    CB_CHECK((d.w & 3) == CBSPMV_FMT_COO && nl >= 1 && nl <= 32 && (d.x >> 24) >= 1);
    CB_CHECK((d.x & 0xFFFFu) + 5 * nl <= bd.stage && (d.y & 0xFFFFu) + 4 * d.z <= bd.stage &&
             (d.y >> 16) + sizeof(M) * d.z <= bd.stage);
    const bool in = (uint32_t)lane < nl;
    len[b] = in ? (int)lds_u8(tab + 4 * nl + lane) : 0;
    row[b] = in ? lds_u32(tab + 4 * lane) : 0;
    cv[b] = d.y;
    off[b] = 0;
    acc[b] = V(0);
    wmax = max(wmax, (int)(d.x >> 24));
  }
  const unsigned below = (1u << lane) - 1u;
  for (int j = 0; j < wmax; j += U) {
    // the element indices of B slices x U steps first, then their column loads, then the
    // gathers: no shared-load wait between two gathers
    uint32_t ix[N], c[N];
    bool on[N];
#pragma unroll
    for (int u = 0; u < U; u++) {
#pragma unroll
      for (int b = 0; b < B; b++) {
        const int e = u * B + b;
        on[e] = len[b] > j + u;
        const unsigned act = __ballot_sync(kFull, on[e]);
        ix[e] = off[b] + (uint32_t)__popc(act & below);
        off[b] += (uint32_t)__popc(act);
        if (CBSPMV_CHECK && on[e]) {
          const uint4 d = lds_v4(da0 + (uint32_t)b * dstride);
          CB_CHECK(ix[e] < d.z && (uint32_t)len[b] <= (d.x >> 24));
        }
      }
    }
#pragma unroll
    for (int e = 0; e < N; e++) c[e] = on[e] ? lds_u32(pg + (cv[e % B] & 0xFFFFu) + 4u * ix[e]) : 0u;
    V xv[N];
#pragma unroll
    for (int e = 0; e < N; e++) {
      const bool hot = (c[e] & cb::kHotBit) != 0;
      CB_CHECK(!on[e] || (hot ? (int)(c[e] & ~cb::kHotBit) < bd.n_hot : (int64_t)c[e] < bd.n));
      V g = V(0), h = V(0);
      if (dbg.skip() & 2) g = V(1) + V(c[e] & 1);
      else if (on[e] && !hot) g = ldg_x(x + c[e], pol);
      if (on[e] && hot) h = lds_val<V>(hotx + (uint32_t)sizeof(V) * (c[e] & ~cb::kHotBit));  // shared x cache
      xv[e] = hot ? h : g;
    }
#pragma unroll
    for (int e = 0; e < N; e++)  // step order per slice (u-major): a piece is summed in sequence
      if (on[e]) acc[e % B] = fma(V(lds_val<M>(pg + (cv[e % B] >> 16) + (uint32_t)sizeof(M) * ix[e])), xv[e], acc[e % B]);
  }
#pragma unroll
  for (int b = 0; b < B; b++) {
    if (len[b] > 0) {
      CB_CHECK((int64_t)row[b] < bd.m);
      V r = acc[b];
      if constexpr (SCALED) r *= lds_val<V>(sc);  // the launch's scale, in shared memory
      red_add(y + row[b], r, dbg);
    }
  }
}

// Aggregated CSR / DENSE block: its x tile x[restore_cols[cols_offset[br] + bc*16 + c]]
// gathered by lanes 0-15 into the warp's shared scratch, zero past ncols.
template <typename V>
__device__ __forceinline__ const V *agg_tile(const uint8_t *page, const uint4 &d, const V *__restrict__ x,
                                             V *scratch, int lane, uint64_t pol) {
  __syncwarp();  // the previous item's reads of the scratch are done
  if (lane < 16) {
    const int nc = (d.w >> 2) & 31;
    const uint32_t *res = reinterpret_cast<const uint32_t *>(page + d.y);
    scratch[lane] = lane < nc ? ldg_x(x + res[lane], pol) : V(0);
  }
  __syncwarp();
  return scratch;
}

// CSR: 17 u8 row_ptr, nnz u8 local cols, pad, values; lanes 2r, 2r+1 share row r
// ("32 threads collaboratively compute 16 y elements").
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void csr_path(const uint8_t *page, const uint4 &d, const V *xt, uint32_t sc,
                                         V *__restrict__ y, int lane, Dbg dbg) {
  const uint8_t *body = page + (d.z & 0xFFFFu);
  const uint8_t *cols = body + 17;
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const int nnz = (int)((d.w >> 8) & 0xFF) + 1;
  const int r = lane >> 1, h = lane & 1;
  const int lo = body[r];
  const int hi = r < 15 ? (int)body[r + 1] : nnz;  // row_ptr[16] = nnz mod 256 (R-8)
  V a0 = V(0), a1 = V(0);
  int e = lo + h;
  for (; e + 2 < hi; e += 4) {
    a0 = fma(V(vals[e]), xt[cols[e]], a0);
    a1 = fma(V(vals[e + 2]), xt[cols[e + 2]], a1);
  }
  if (e < hi) a0 = fma(V(vals[e]), xt[cols[e]], a0);
  V acc = a0 + a1;
  acc += __shfl_xor_sync(kFull, acc, 1);
  if constexpr (SCALED) acc *= lds_val<V>(sc);
  if (h == 0 && hi > lo) red_add(y + d.x + r, acc, dbg);
}

// Two CSR blocks of non-aggregated matrices at once: lanes 0-15 take rows 0-15 of block A, lanes
// 16-31 those of block B, one lane per row (no shuffle; one RED instruction for both blocks).
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void csr_pair(const uint8_t *page, const uint4 &dA, const uint4 &dB, uint32_t sc,
                                         V *__restrict__ y, int lane, Dbg dbg) {
  const uint4 d = lane < 16 ? dA : dB;
  const V *xt = reinterpret_cast<const V *>(page + (d.w >> 16));
  const uint8_t *body = page + (d.z & 0xFFFFu);
  const uint8_t *cols = body + 17;
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const int nnz = (int)((d.w >> 8) & 0xFF) + 1;
  const int r = lane & 15;
  const int lo = body[r];
  const int hi = r < 15 ? (int)body[r + 1] : nnz;  // row_ptr[16] = nnz mod 256 (R-8)
  V a0 = V(0), a1 = V(0);
  int e = lo;
  for (; e + 1 < hi; e += 2) {
    a0 = fma(V(vals[e]), xt[cols[e]], a0);
    a1 = fma(V(vals[e + 1]), xt[cols[e + 1]], a1);
  }
  if (e < hi) a0 = fma(V(vals[e]), xt[cols[e]], a0);
  V acc = a0 + a1;
  if constexpr (SCALED) acc *= lds_val<V>(sc);
  if (hi > lo) red_add(y + d.x + r, acc, dbg);
}

// DENSE (Alg. 4): the device record stores the 256 values in lane-major 16-byte pairs (pair
// q*32 + l holds A[l % 16][(l / 16) * 8 + 2q + {0, 1}]), so lane l owns row l % 16, columns
// 8*(l/16) .. +7: 4 conflict-free 16-byte shared loads (8-byte for fp32), 8 FMAs against the
// x tile, one shfl_xor(16) joins the two half rows (the semantics of Alg. 4's shfl, R-15), 16
// REDs.  Absent entries are stored zeros; a non-finite x in the tile would make 0·inf poison a
// row, so a warp whose sums are not all finite recomputes skipping the stored zeros.
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void dense_path(const uint8_t *page, const uint4 &d, const V *xt, uint32_t sc,
                                           V *__restrict__ y, int64_t m, int lane, Dbg dbg) {
  using M2 = typename Pair<M>::type;
  using V2 = typename Pair<V>::type;
  const M2 *vals = reinterpret_cast<const M2 *>(page + (d.z >> 16));
  const V2 *xt2 = reinterpret_cast<const V2 *>(xt);
  const int h = lane >> 4, r = lane & 15;
  M2 a[4];
#pragma unroll
  for (int q = 0; q < 4; q++) a[q] = vals[q * 32 + lane];
  V acc = V(0);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const V2 xv = xt2[h * 4 + q];
    acc = fma(V(a[q].x), xv.x, acc);
    acc = fma(V(a[q].y), xv.y, acc);
  }
  if (__any_sync(kFull, !isfinite(acc))) {
    acc = V(0);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const V2 xv = xt2[h * 4 + q];
      if (a[q].x != M(0)) acc = fma(V(a[q].x), xv.x, acc);
      if (a[q].y != M(0)) acc = fma(V(a[q].y), xv.y, acc);
    }
  }
  acc += __shfl_xor_sync(kFull, acc, 16);
  if constexpr (SCALED) acc *= lds_val<V>(sc);
  if (h == 0 && (int64_t)d.x + r < m) red_add(y + d.x + r, acc, dbg);
}

// ------------------------------------------------------------------ the persistent kernel
struct KParams {
  const uint8_t *stream;
  const uint64_t *page_off;
  const uint32_t *cta_page;
  uint32_t *page_ctr;  // dynamic page claiming: {next page, finished producers}; nullptr = static
  uint32_t n_pages;
  uint32_t claim_chunk;  // pages per dynamic claim
  int strided;           // static: K > 0 -> CTA g takes runs of K pages g, g + grid, ... (0: contiguous)
  int64_t m, n;
  const double *sumsq;
  int stage;   // bytes per stage: page + its x area
  int nstage;  // S
  int groups;  // G (divides S)
  int gwarps;  // W consumer warps per group
  int agg;     // aggregated: x gathered by the consumers (restore entries / chunk columns)
  int xvec;    // non-aggregated tiles: x 16-byte aligned -> TMA bulk tile copies
  int xwarps;  // X x warps (X <= G; 0 for aggregated matrices)
  const uint32_t *hot;  // hot x columns (shared x cache), n_hot of them
  int n_hot;
  uint32_t sleep_ns;    // consumer / x-warp back-off between mbarrier probes (0: none)
  int csr_pair;         // non-aggregated: a warp takes two CSR blocks at once (one lane per row)
  int pdl_wait;         // launched dependent on the y-zeroing kernel: wait for it before any RED
  int xagg;             // aggregated matrix whose CSR / DENSE tiles the x warps gather
  Dbg dbg;
};

// x warps, non-aggregated matrices: the 16-value x tiles of the page's CSR / DENSE items
// (x[bc*16 ..], the paper's s_x) into the stage's x area: 16-byte loads into
// registers (ld.global.nc, L2 evict_last; 8 lanes per fp64 tile, 4 tiles per instruction), up to
// kRounds instructions in flight, then 16-byte shared stores.  (cp.async costs ~8 SM cycles per
// lane-copy on B200 — measured: it bounded the round-1 kernel at 0.83 ms on the clustered
// matrix — while plain loads are limited only by the L1 / L2 request rate.)  A ragged last
// block column or an x that is not 16-byte aligned is loaded per element with zero fill.
template <typename V>
__device__ __forceinline__ uint4 load_piece(const uint8_t *page, const V *__restrict__ x, const uint4 &d, int q,
                                            bool vec, bool agg, uint64_t pol) {
  constexpr int kPer = 16 / (int)sizeof(V);
  const int nc = (d.w >> 2) & 31;
  const V *src = x + d.y + q;
  uint4 v;
  if (agg) {  // aggregated block: x[restore_cols[cols_offset[br] + bc*16 + c]], entries in the page
    const uint32_t *res = reinterpret_cast<const uint32_t *>(page + d.y) + q;
    V e[kPer];
#pragma unroll
    for (int j = 0; j < kPer; j++) e[j] = q + j < nc ? ldg_x(x + res[j], pol) : V(0);
    memcpy(&v, e, 16);
  } else if (vec && nc == 16) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src), "l"(pol));
  } else {
    V e[kPer];
#pragma unroll
    for (int j = 0; j < kPer; j++) e[j] = q + j < nc ? src[j] : V(0);
    memcpy(&v, e, 16);
  }
  return v;
}

template <typename V>
__device__ __forceinline__ void tile_page(const uint8_t *page, const V *__restrict__ x, const KParams &P, int lane,
                                          uint64_t pol) {
  constexpr int kPer = 16 / (int)sizeof(V);   // values per 16-byte piece
  constexpr int kLanes = 16 / kPer;           // lanes per tile: 8 (fp64), 4 (fp32)
  constexpr int kTiles = 32 / kLanes;         // tiles per instruction
  constexpr int kRounds = 4;                  // loads in flight per lane
  const uint32_t ncd = reinterpret_cast<const uint32_t *>(page)[1];
  const uint4 *descs = reinterpret_cast<const uint4 *>(page + cb::kPageHeader);
  uint8_t *pg = const_cast<uint8_t *>(page);
  const int sub = lane / kLanes, q = (lane % kLanes) * kPer;
  for (uint32_t b = 0; b < ncd; b += kTiles * kRounds) {
    uint4 v[kRounds];
    uint32_t dst[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; r++) {
      const uint32_t it = b + (uint32_t)(r * kTiles + sub);
      dst[r] = 0;
      if (it < ncd) {
        const uint4 d = descs[it];
        v[r] = load_piece<V>(page, x, d, q, P.xvec != 0, P.agg != 0, pol);
        dst[r] = (d.w >> 16) + (uint32_t)q * (uint32_t)sizeof(V);
      }
    }
#pragma unroll
    for (int r = 0; r < kRounds; r++)
      if (dst[r]) *reinterpret_cast<uint4 *>(pg + dst[r]) = v[r];
  }
}

// Warp roles: 0 = TMA producer, 1..X = x warps, X+1.. = consumer groups.  M: matrix value type of the
// records; V: type of x, y and the accumulation (M = float, V = double: the mixed variant).
template <typename M, typename V, bool SCALED>
__global__ void __launch_bounds__(kMaxThreads, 1)
    cb_spmv_kernel(KParams P, const V *__restrict__ x, V *__restrict__ y) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *xrdy = full + kMaxStages;
  uint64_t *empty = xrdy + kMaxStages;
  uint8_t *ring = smem + kSmemHeader;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = P.nstage, G = P.groups, W = P.gwarps;
  const Dbg dbg = P.dbg;
  const bool dyn = P.page_ctr != nullptr;
  // static assignment: a contiguous byte-balanced page range per CTA, or (strided) runs of K
  // pages blockIdx.x, blockIdx.x + grid, ... so every CTA sees the whole slot order's mix
  uint32_t p0 = P.cta_page[blockIdx.x], p1 = P.cta_page[blockIdx.x + 1];
  const uint32_t K = (uint32_t)P.strided;
  if (K) {
    p0 = 0;
    p1 = 0;  // local page count
    for (uint64_t c = blockIdx.x; c * K < P.n_pages; c += gridDim.x) {
      const uint64_t left = P.n_pages - c * K;
      p1 += (uint32_t)(left < K ? left : K);
    }
  }
  const uint32_t npl = p1 - p0;  // local pages (static)

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&xrdy[s], 32);
      mbar_init(&empty[s], (uint32_t)W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (SCALED) *reinterpret_cast<V *>(smem + kScaleSlot) = (V)(1.0 / sqrt(*P.sumsq));
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: one bulk copy per page into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t round = 0;
      auto next_stage = [&]() {
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);  // the group released the stage
      };
      auto advance = [&]() {
        if (++s == S) { s = 0; round++; }
      };
      auto load_page = [&](uint32_t p) {
        const uint64_t off = P.page_off[p];
        const uint32_t bytes = (uint32_t)(P.page_off[p + 1] - off);
        CB_CHECK(p < P.n_pages && bytes >= 16 && bytes % 16 == 0 && bytes <= (uint32_t)P.stage);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * P.stage, P.stream + off, bytes, &full[s], pol);
        advance();
      };
      if (!dyn) {
        for (uint32_t i = 0; i < npl; i++) {
          next_stage();
          load_page(K ? ((i / K) * gridDim.x + blockIdx.x) * K + i % K : p0 + i);
        }
      } else {
        // Dynamic claiming (SMs that finish early take more pages): claims of claim_chunk pages
        // from a global counter, the next claim issued before the current chunk is loaded; then
        // one end marker per consumer group (the next G stages of the sequence, so every group
        // meets exactly one), and the last producer resets the counter for the next launch.
        const uint32_t kClaim = P.claim_chunk;
        uint32_t cur = atomicAdd(&P.page_ctr[0], kClaim);
        while (cur < P.n_pages) {
          const uint32_t nxt = atomicAdd(&P.page_ctr[0], kClaim);
          const uint32_t end = min(cur + kClaim, P.n_pages);
          for (uint32_t p = cur; p < end; p++) {
            next_stage();
            load_page(p);
          }
          cur = nxt;
        }
        for (int g = 0; g < G; g++) {
          next_stage();
          mbar_arrive_expect_tx(&full[s], 16u);
          bulk_g2s(ring + (size_t)s * P.stage, kEndHeader, 16u, &full[s], pol);
          advance();
        }
        if (atomicAdd(&P.page_ctr[1], 1u) == gridDim.x - 1) {
          P.page_ctr[0] = 0;
          P.page_ctr[1] = 0;
        }
      }
    }
    return;
  }

  if (warp <= P.xwarps) {
    // ---------------- x warps (non-aggregated matrices): x warp k fills the x tiles of pages
    // k, k + X, ... as they land, then arrives on the page's xready.  Dynamic claiming: X <= G,
    // so each x warp meets one of the G end markers (the last pages) and stops there.
    if (P.agg && !P.xagg) return;
    const uint64_t pol = policy_evict_last();
    const int X = P.xwarps, k = warp - 1;
    int s = k;
    uint32_t parity = 0;
    for (uint32_t li = (uint32_t)k; dyn || li < npl; li += (uint32_t)X) {
      mbar_wait_sleep(&full[s], parity, P.sleep_ns);
      const uint8_t *page = ring + (size_t)s * P.stage;
      if (reinterpret_cast<const uint32_t *>(page)[0] == cb::kEndItems) break;
      if (!(dbg.skip() & 2)) tile_page<V>(page, x, P, lane, pol);
      mbar_arrive(&xrdy[s]);  // per lane (count 32): releases this lane's shared stores
      s += X;
      while (s >= S) { s -= S; parity ^= 1u; }
    }
    return;
  }

  // ---------------- consumers: group g takes pages g, g + G, ... (stages g, g + G, ...)
  // SCALED: s = 1/sqrt(*sumsq), computed once per CTA into the mbarrier area's spare bytes (no
  // register held through the item loops)
  const uint32_t scale = smem_addr(smem + kScaleSlot);
  const int cw = warp - 1 - P.xwarps;
  V *wscratch = reinterpret_cast<V *>(smem + kSmemHeader + (size_t)S * P.stage) + cw * 16;
  const uint64_t xpol = policy_evict_last();
  // the shared x cache: x[hot[s]] for the launch's hot columns, copied by the consumers before
  // their first page (named barrier 1 over the consumer warps; the producer is already streaming)
  V *hotx = reinterpret_cast<V *>(smem + kSmemHeader + (size_t)S * P.stage + (size_t)G * W * 16 * 8);
  if (P.n_hot > 0) {
    const int nct = 32 * G * W;
    for (int i = cw * 32 + lane; i < P.n_hot; i += nct) hotx[i] = ldg_x(x + P.hot[i], xpol);
    asm volatile("bar.sync 1, %0;" ::"r"(nct) : "memory");
  }
  const uint32_t hota = smem_addr(hotx);
  const Bounds bd{(uint32_t)P.stage, P.m, P.n, P.n_hot};
  // Launched dependent on the y-zeroing kernel (PDL): no RED before that grid has finished (a
  // no-op for a normal launch).  Then this CTA lets the next launch of the same SpMV (the next
  // column panel: REDs commute, so panels need not wait for each other) start on SMs this grid
  // frees; y is zeroed by then.
  if (P.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int grp = cw / W, wg = cw - grp * W;
  int s = grp;
  uint32_t parity = 0;
  int kc = wg;  // this warp's first item of the group's next page (items continue across pages)
  for (uint32_t li = (uint32_t)grp; dyn || li < npl; li += (uint32_t)G) {
    mbar_wait_sleep(&full[s], parity, P.sleep_ns);
    const uint8_t *page = ring + (size_t)s * P.stage;
    const uint32_t nitems = reinterpret_cast<const uint32_t *>(page)[0];
    if (dyn && nitems == cb::kEndItems) break;  // this group's end marker (nothing to release)
    if (!P.agg || P.xagg) mbar_wait_sleep(&xrdy[s], parity, P.sleep_ns);
    const uint4 *descs = reinterpret_cast<const uint4 *>(page + cb::kPageHeader);
    const int n = (dbg.skip() & 4) ? 0 : (int)nitems;
    const int ncd = (int)reinterpret_cast<const uint32_t *>(page)[1];
    CB_CHECK(nitems >= 1 && cb::kPageHeader + 16ull * nitems <= (uint64_t)P.stage && ncd <= (int)nitems);
    int k = kc;
    // CSR / DENSE items first (the page lists them before the chunks)
    for (; k < ncd && k < n; k += W) {
      const uint4 d = descs[k];
      if (P.csr_pair && (d.w & 3) == CBSPMV_FMT_CSR && k + W < ncd && k + W < n &&
          (descs[k + W].w & 3) == CBSPMV_FMT_CSR) {  // this warp's next item is CSR too: both at once
        if (CBSPMV_CHECK) {
          const uint4 e = descs[k + W];
          CB_CHECK((d.z >> 16) + (uint32_t)sizeof(M) * (((d.w >> 8) & 0xFF) + 1) <= (uint32_t)P.stage &&
                   (e.z >> 16) + (uint32_t)sizeof(M) * (((e.w >> 8) & 0xFF) + 1) <= (uint32_t)P.stage);
          // (d.y: the tile's first column, or with aggregation the page offset of its restore entries)
          CB_CHECK((int64_t)d.x < P.m && (int64_t)e.x < P.m &&
                   (P.agg ? d.y + 64 <= (uint32_t)P.stage && e.y + 64 <= (uint32_t)P.stage
                          : (int64_t)d.y < P.n && (int64_t)e.y < P.n) &&
                   (d.w >> 16) + 16 * sizeof(V) <= (uint32_t)P.stage && (e.w >> 16) + 16 * sizeof(V) <= (uint32_t)P.stage);
        }
        csr_pair<M, V, SCALED>(page, d, descs[k + W], scale, y, lane, dbg);
        k += W;
        continue;
      }
      if (CBSPMV_CHECK) {  // CSR / DENSE item: record, restore entries / x tile inside the stage, rows < m
        const uint32_t nz = ((d.w >> 8) & 0xFF) + 1, nc = (d.w >> 2) & 31;
        const uint32_t rec = (d.w & 3) == CBSPMV_FMT_CSR ? (d.z >> 16) + (uint32_t)sizeof(M) * nz
                                                          : (d.z >> 16) + (uint32_t)sizeof(M) * 256;
        CB_CHECK(((d.w & 3) == CBSPMV_FMT_CSR || (d.w & 3) == CBSPMV_FMT_DENSE) && nc <= 16 && rec <= (uint32_t)P.stage &&
                 (int64_t)d.x < P.m);
        CB_CHECK(P.agg ? d.y + 4 * nc <= (uint32_t)P.stage : (int64_t)d.y < P.n);
        CB_CHECK((P.agg && !P.xagg) || (d.w >> 16) + 16 * sizeof(V) <= (uint32_t)P.stage);
        if (P.agg && lane < (int)nc) CB_CHECK((int64_t)reinterpret_cast<const uint32_t *>(page + d.y)[lane] < P.n);
      }
      const V *xt = P.agg && !P.xagg ? agg_tile<V>(page, d, x, wscratch, lane, xpol)
                                     : reinterpret_cast<const V *>(page + (d.w >> 16));
      if ((d.w & 3) == CBSPMV_FMT_CSR) csr_path<M, V, SCALED>(page, d, xt, scale, y, lane, dbg);
      else dense_path<M, V, SCALED>(page, d, xt, scale, y, P.m, lane, dbg);
    }
    // COO slices, four at a time: the four slices' element loads and x gathers in flight together
    const uint32_t pg = smem_addr(page), dsc = pg + cb::kPageHeader, dW = 16u * (uint32_t)W;
    // (a warp holding fewer than four slices of the page unrolls their steps instead: always four
    // elements per lane in flight)
    for (; k + 3 * W < n; k += 4 * W)
      coo_slices<M, V, SCALED, 4, 1>(pg, dsc + 16u * (uint32_t)k, dW, x, hota, y, scale, lane, xpol, dbg, bd);
    if (k + W < n) {
      coo_slices<M, V, SCALED, 2, 2>(pg, dsc + 16u * (uint32_t)k, dW, x, hota, y, scale, lane, xpol, dbg, bd);
      k += 2 * W;
    }
    if (k < n) {
      coo_slices<M, V, SCALED, 1, 4>(pg, dsc + 16u * (uint32_t)k, dW, x, hota, y, scale, lane, xpol, dbg, bd);
      k += W;
    }
    if (n != (int)nitems) k += ((int)nitems - k + W - 1) / W * W;  // ablation skipped the items
    kc = k - (int)nitems;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    s += G;
    if (s >= S) { s -= S; parity ^= 1u; }
  }
}

// Programmatic dependent launch: the SpMV kernel that follows may start (barrier set-up, the
// producer's first page copies, the hot x copy) while y is being zeroed; its consumers wait for
// this grid (griddepcontrol.wait) before their first RED.
template <typename V>
__global__ void cb_zero_kernel(V *__restrict__ y, int64_t m) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = V(0);
}

template <typename V>
__global__ void cb_sumsq_kernel(const V *__restrict__ v, int64_t len, double *out) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = (double)v[i];
    acc = fma(t, t, acc);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
    if (threadIdx.x == 0) atomicAdd(out, acc);
  }
}

const void *select_kernel(int dtype, bool scaled) {
  if (dtype == CBSPMV_F64)
    return scaled ? (const void *)&cb_spmv_kernel<double, double, true> : (const void *)&cb_spmv_kernel<double, double, false>;
  if (dtype == CBSPMV_F32)
    return scaled ? (const void *)&cb_spmv_kernel<float, float, true> : (const void *)&cb_spmv_kernel<float, float, false>;
  return scaled ? (const void *)&cb_spmv_kernel<float, double, true> : (const void *)&cb_spmv_kernel<float, double, false>;
}

// bytes of one x / y element
inline int vec_bytes(int dtype) { return dtype == CBSPMV_F32 ? 4 : 8; }

inline int cuda_fail(cudaError_t e, const char *what, std::string *err) {
  *err = std::string(what) + ": " + cudaGetErrorString(e);
  return CBSPMV_ECUDA;
}

// per consumer warp: one 16-value x tile (aggregated CSR / DENSE blocks), fp64-sized
inline int scratch_bytes(const CbShape &sh) { return sh.groups * sh.gwarps * 16 * 8; }
// dynamic shared memory of a launch: mbarriers | S stages | warp scratch | hot x cache
inline int smem_bytes(const CbDevice &d) {
  return kSmemHeader + d.nstage * d.page_cap + scratch_bytes(d) + d.n_hot * vec_bytes(d.dtype);
}

int env_int(const char *k, int d) {
  const char *v = std::getenv(k);
  return v ? std::atoi(v) : d;
}

}  // namespace

// Launch shape, read once per built handle (so a test can build handles with different shapes
// in one process): S stages, G consumer groups of W warps (G divides S), and the stage bytes
// that fill the opt-in shared memory.  Defaults measured on B200.
int cb_plan_stages(int device, int agg, bool agg_tiles, CbShape *sh, std::string *err) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute", err);
  // Non-aggregated matrices: 4 groups of 7 warps and 3 x warps (clustered fp64: 0.72 ms; 3 groups
  // of 9: 0.73, 2 of 14: 0.89).  Aggregated matrices gather x in the consumers, so no x warps:
  // 2 groups of 15 (R-MAT: 1.05 ms; 4 groups of 7: 1.11, 1 group of 30: 1.08).
  // Aggregated matrices also leave half the unified L1 / shared array to L1: their x gathers are
  // random loads whose misses need L1 lines to land in, and with the whole array given to stages
  // the L1 holds almost nothing (R-MAT 1.10 -> 0.70 ms, uniform 13.1 -> 10.2 ms with 6 stages of
  // 20 KB: ~120 KB shared, ~100 KB L1; 12 x 19 KB: 1.10 / 13.1, 4 x 24 KB: 0.72, 2 x 32 KB: 1.00).
  // Non-aggregated matrices stream their x tiles with plain loads and need the deep ring
  // (clustered: 12 x 19 KB 0.72-0.75 ms, 8 x 19 KB 0.82, 8 x 22 KB 0.78).
  // Aggregated matrices with many CSR / DENSE blocks (agg_tiles, the Laplacian) keep the aggregated
  // shape but trade one consumer warp per group for two x warps that gather those tiles.
  const bool xagg = agg && agg_tiles;
  const int G = std::max(1, env_int("CBSPMV_GROUPS", agg ? 2 : 4));
  const int W = std::max(1, env_int("CBSPMV_GROUP_WARPS", xagg ? 14 : agg ? 15 : 7));
  const int X = agg && !xagg ? 0 : std::max(1, std::min(G, env_int("CBSPMV_XWARPS", xagg ? 2 : 3)));  // X <= G (end markers)
  int S = std::min(kMaxStages, std::max(G, env_int("CBSPMV_STAGES", agg ? 6 : 12)));
  S -= S % G;  // G | S: every stage belongs to one group
  if (1 + X + G * W > kMaxThreads / 32) {
    *err = "1 + CBSPMV_XWARPS + CBSPMV_GROUPS * CBSPMV_GROUP_WARPS exceeds 32 warps";
    return CBSPMV_EUNSUPPORTED;
  }
  CbShape probe;
  probe.groups = G;
  probe.gwarps = W;
  int cap = (optin - kSmemHeader - scratch_bytes(probe)) / S / 16 * 16;
  if (const char *v = std::getenv("CBSPMV_PAGE_BYTES")) cap = std::min(cap, std::atoi(v) / 16 * 16);
  else if (agg) cap = std::min(cap, kAggPageBytes);
  cap = std::min(cap, cb::kMaxPageCap);
  if (cap < 4096) {
    *err = "stage capacity below 4 KB (too many stages for the shared memory)";
    return CBSPMV_EUNSUPPORTED;
  }
  sh->nstage = S;
  sh->groups = G;
  sh->gwarps = W;
  sh->xwarps = X;
  sh->page_cap = cap;
  sh->hot_cap = std::max(0, optin - kSmemHeader - S * cap - scratch_bytes(probe));
  sh->xagg = xagg ? 1 : 0;
  return CBSPMV_OK;
}

int cb_configure(CbDevice *dev, std::string *err) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute", err);
  const int smem = smem_bytes(*dev);
  if (smem > optin) {
    *err = "stages and the hot x cache do not fit the shared memory";
    return CBSPMV_EUNSUPPORTED;
  }
  for (int dt = 0; dt < 3; dt++)
    for (int sc = 0; sc < 2; sc++) {
      e = cudaFuncSetAttribute(select_kernel(dt, sc != 0), cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
    }
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute", err);
  dev->sms = sms;
  const int64_t g = dev->n_pages < sms ? dev->n_pages : sms;
  dev->grid = (int)(g < 1 ? 1 : g);
  // Page assignment, decided per handle; the env overrides exist for A/B runs
  // and for tests (read here, at build time, so a test can set them per handle):
  //   dynamic claiming for large aggregated matrices (per-page work follows the random gathers
  //   and atomics); strided static runs for 4-byte stored values (issue-bound: each CTA sees the
  //   slot order's whole format mix); contiguous byte-balanced ranges otherwise.
  // Measured on B200: dynamic claims of runs of 16 pages beat static ranges on
  // every large matrix (clustered fp64 0.745 -> 0.72 ms, fp32 0.58 -> 0.47 ms: Alg. 2's slot
  // order puts the DENSE-heavy TBs first and the COO / CSR-heavy ones last, so equal byte ranges
  // are unequal work; R-MAT 1.16 -> 1.13 ms); single pages dealt round robin lose DRAM locality
  // (clustered 1.11 ms).  The claim shrinks for small matrices so the tail stays short.
  const int dyn_env = env_int("CBSPMV_DYNAMIC_PAGES", -1);
  dev->dynamic = dyn_env >= 0 ? dyn_env != 0 : dev->n_pages >= 64 * (int64_t)dev->grid;  // Laplacian (29 / CTA): static 0.027 vs dynamic 0.033 ms
  const int64_t per = dev->n_pages / std::max<int64_t>(1, 16 * (int64_t)dev->grid);
  dev->claim_chunk = (uint32_t)std::max(1, env_int("CBSPMV_CLAIM_CHUNK", (int)std::min<int64_t>(16, std::max<int64_t>(1, per))));
  const int str_env = env_int("CBSPMV_STRIDED_PAGES", -1);
  dev->strided = dev->dynamic ? 0 : std::max(0, str_env);
  dev->dbg_skip = env_int("CBSPMV_DEBUG_SKIP", 0);
  dev->sleep_ns = (uint32_t)std::max(0, env_int("CBSPMV_WAIT_SLEEP_NS", 0));
  dev->pdl = env_int("CBSPMV_PDL", 1) != 0;
  // paired CSR blocks (one lane per row; fewer instructions): clustered fp32 0.498 -> 0.444 ms,
  // mixed 0.629 -> 0.571, fp64 0.754 -> 0.747 (4 interleaved A/B pairs; 400-launch sustained 0.836 -> 0.814)
  dev->csr_pair = env_int("CBSPMV_CSR_PAIR", 1) != 0;
  return CBSPMV_OK;
}

int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y, void *stream,
                   std::string *err, bool follows) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (zero_y && dev.m > 0) {
    const int zb = 256;
    const int64_t need = (dev.m + zb - 1) / zb;
    const int zg = (int)(need < (int64_t)dev.sms * 8 ? need : (int64_t)dev.sms * 8);
    if (vec_bytes(dev.dtype) == 8) cb_zero_kernel<double><<<zg, zb, 0, st>>>((double *)y, dev.m);
    else cb_zero_kernel<float><<<zg, zb, 0, st>>>((float *)y, dev.m);
  }
  if (dev.n_pages > 0) {
    uint32_t *ctr = nullptr;
    if (dev.dynamic && dev.d_page_ctr) {
      // atomic slot pick: two host threads launching the same handle get different slots
      const uint32_t slot = __atomic_fetch_add(&dev.ctr_next, 1u, __ATOMIC_RELAXED);
      ctr = dev.d_page_ctr + 2 * (slot % cb::kCtrSlots);
    }
    KParams P{dev.d_stream, dev.d_page_off, dev.d_cta_page, ctr, (uint32_t)dev.n_pages, dev.claim_chunk,
              ctr ? 0 : dev.strided, dev.m, dev.n, sumsq, dev.page_cap, dev.nstage, dev.groups, dev.gwarps, dev.agg,
              !dev.agg && ((uintptr_t)x % 16 == 0), dev.xwarps, dev.d_hot, dev.n_hot, dev.sleep_ns,
              dev.csr_pair && (!dev.agg || dev.xagg), zero_y && dev.m > 0 && dev.pdl, dev.xagg,
              Dbg{dev.dbg_skip}};
    const int smem = smem_bytes(dev);
    const void *fn = select_kernel(dev.dtype, sumsq != nullptr);
    void *args[] = {&P, const_cast<void **>(&x), &y};
    const int threads = 32 * (1 + dev.xwarps + dev.groups * dev.gwarps);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(dev.grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the zeroing kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = dev.pdl && ((zero_y && dev.m > 0) || follows) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return cuda_fail(e, "spmv kernel launch", err);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "spmv launch", err);
  return CBSPMV_OK;
}

int cb_launch_sumsq(const void *v, int64_t len, int dtype, double *out, void *stream, std::string *err) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return cuda_fail(e, "memset", err);
  if (len > 0) {
    static const int sms = [] {
      int dev = 0, v = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v > 0 ? v : 148;
    }();
    const int64_t need = (len + 255) / 256;
    const int g = (int)(need < (int64_t)sms * 4 ? need : (int64_t)sms * 4);
    if (vec_bytes(dtype) == 8) cb_sumsq_kernel<double><<<g, 256, 0, st>>>((const double *)v, len, out);
    else cb_sumsq_kernel<float><<<g, 256, 0, st>>>((const float *)v, len, out);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sumsq launch", err);
  return CBSPMV_OK;
}
