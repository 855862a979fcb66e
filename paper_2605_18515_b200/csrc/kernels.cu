// kernels.cu — sm_100a kernels of the CB-SpMV hot path (y = A·x, §3.5).
//
// One persistent CTA per SM streams its contiguous range of device pages
// through a ring of 28 KB shared-memory stages (8 stages):
//   warp 0 (one elected lane): TMA producer — waits on the stage's "empty" mbarrier, then one
//       cp.async.bulk (SASS UBLKCP) per page, L2 evict_first (the stream must not evict x);
//       completion counted on the stage's "full" mbarrier.
//   5 consumer groups x 6 warps: page i of the CTA goes to group i % 5; the group's warps claim
//       the page's work items from a shared counter:
//       * COO group (Alg. 3): up to 4 consecutive COO blocks packed into one warp,
//         lane <-> element, coordinate byte row = b & 15, col = b >> 4, one RED
//         per element — Alg. 3's atomicAdd — issued as one warp instruction per group;
//       * CSR ("32 threads collaboratively compute 16 y elements"): two lanes
//         per row, one shfl_xor;
//       * DENSE (Alg. 4): lane-major device layout, 8 FMAs per lane, one
//         shfl_xor(16) (R-15 semantics), 16 REDs.
// x: without aggregation each item's 16-value tiles x[bc*16 ..] are copied
// into the stage with 16-byte cp.async one item ahead of processing (replaces the paper's
// shared-memory s_x preload); with aggregation each lane gathers
// x[restore_cols[cols_offset[br] + bc*16 + col]] straight into a register, the next COO
// group's loads issued before the current one is finished.  The restore entries travel in
// front of each block's record.  y is zeroed by cb_zero_kernel (R-16) and accumulated with
// red.global.add (the paper's atomicAdd).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <string>

#include "cb_internal.h"

namespace {

constexpr int kGroupWarps = 6;     // consumer warps per group; a page is consumed by one group
constexpr int kMaxGroups = 5;      // consumer groups per CTA (runtime: KParams::groups)
constexpr int kMaxThreads = 1024;
constexpr int kMaxStages = 16;
constexpr int kSmemHeader = 512;  // mbarriers full[16] (+16 spare), empty[16], claims[16], stage seq[16]; warp scratch follows the ring
constexpr uint32_t kEndPage = 0xFFFFFFFFu;
// End marker of dynamic page claiming: a 16-byte page header (nblk = kEndPage) copied into the
// stage by the same TMA path as a page, so the marker is synchronised exactly like data.
__device__ __align__(16) const uint32_t kEndHeader[4] = {kEndPage, 0u, 16u, 16u};
constexpr unsigned kFull = 0xffffffffu;

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
// Consumer-side wait with a short sleep between probes (fewer issue slots and less power spent
// spinning while the page is in flight; A/B knob CBSPMV_WAIT_SLEEP_NS, 0 = plain probe loop).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, int ns) {
  while (!mbar_try_wait(bar, parity)) {
    if (ns) __nanosleep(ns);
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
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
// Asynchronous copy of one x value into shared memory (SASS LDGSTS).
template <typename V>
__device__ __forceinline__ void cp_async_elem(V *dst, const V *src, uint64_t pol) {
  // no "memory" clobber: the destination is read only after cp.async.wait_group + __syncwarp
  if constexpr (sizeof(V) == 8)
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
  else
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
}
__device__ __forceinline__ void cp_async_16(void *dst, const void *src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "l"(pol));
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
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

// Ablation knob for profiling only: built with -DCBSPMV_ABLATION=1 the env CBSPMV_DEBUG_SKIP
// (a kernel argument) drops the y atomics (bit 0), replaces the x gathers (bit 1), skips the item
// processing (bit 2) or the tile copies (bit 3).  In the production build every test folds away.
#ifndef CBSPMV_ABLATION
#define CBSPMV_ABLATION 0
#endif
#ifndef CBSPMV_CHECK  // debug build: trap on a malformed stage (pipeline race detector)
#define CBSPMV_CHECK 0
#endif
struct Dbg {
  int skip_;
  __device__ __forceinline__ int skip() const { return CBSPMV_ABLATION ? skip_ : 0; }
};

template <typename V>
__device__ __forceinline__ void red_add(V *p, V v, Dbg dbg) {
  if (dbg.skip() & 1) {
    if (v == V(12345.678)) *p = v;  // keep the value live without the atomic
    return;
  }
  atomicAdd(p, v);  // result unused -> RED.E.ADD
}

__device__ __forceinline__ int d_type(const uint4 &d) { return (d.w >> 8) & 3; }
__device__ __forceinline__ int d_nnz(const uint4 &d) { return (int)(d.w & 0xFF) + 1; }
__device__ __forceinline__ int d_ncols(const uint4 &d) { return (d.w >> 16) & 31; }

// ------------------------------------------------------------------ per-format warp paths
// xt: the block's 16-value x tile in shared memory (copied one work item ahead):
//   x[bc*16 + c] without aggregation (the paper's shared-memory s_x), or
//   x[restore_cols[cols_offset[br] + bc*16 + c]] with aggregation.

// COO group (Alg. 3): up to 4 consecutive COO blocks packed into one warp, lane <-> element;
// the coordinate byte gives row = b & 15, col = b >> 4; one RED per element into y
// (Alg. 3's atomicAdd), issued as one warp instruction.  Split in two phases:
// coo_issue() performs every load (descriptor, element, restore entry, x) and coo_finish()
// multiplies and issues the RED, so several groups' loads can be in flight together.
template <typename V>
struct CooPend {
  V v, xv;
  uint32_t yrow;
  bool valid, hub;  // hub: the block's row is in a hub block row (desc.row0 bit 0)
};

template <typename M, typename V, bool AGG>
__device__ __forceinline__ CooPend<V> coo_issue(const uint8_t *page, const uint4 *descs, uint32_t iw,
                                                const V *xbuf, const V *__restrict__ x, int lane, Dbg dbg,
                                                uint64_t xpol) {
  CooPend<V> r;
  // group membership from the item word (first lanes of members 1..3; 0 = absent)
  const int hb = iw & 0xFFF;
  const int l1 = (iw >> 16) & 31, l2 = (iw >> 21) & 31, l3 = (iw >> 26) & 31;
  const int mi = (l1 && lane >= l1) + (l2 && lane >= l2) + (l3 && lane >= l3);
  const int lane0 = mi == 0 ? 0 : (mi == 1 ? l1 : (mi == 2 ? l2 : l3));
  const uint4 d = descs[hb + mi];
  const int i = lane - lane0;
  r.valid = i < d_nnz(d);
  const uint8_t *body = page + (d.z & 0xFFFFu);
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const uint32_t byte = r.valid ? body[i] : 0u;
  const int col = byte >> 4;
  r.hub = r.valid && (d.x & 1u);
  r.yrow = (d.x & ~1u) + (byte & 15);
  r.v = r.valid ? V(vals[i]) : V(0);
  r.xv = V(0);
  if (r.valid) {
    if constexpr (AGG) {
      const uint32_t c = reinterpret_cast<const uint32_t *>(page + d.y)[col];
      r.xv = (dbg.skip() & 2) ? V(1) + V(c & 1) : ldg_x(x + c, xpol);
    } else {
      r.xv = xbuf[(hb + mi) * 16 + col];
    }
  }
  return r;
}

// Runs of elements on the same y row (a COO record is sorted by (row, col)) can be
// summed in the warp first and added by one RED from the run's first lane.  Hub rows of power-law
// matrices otherwise receive ~10^5 same-address atomics per SpMV, serialised in L2 (R-MAT: row 0
// gets 115 K).  Only the RUNS kernel variant does this, and only for groups holding
// a block the builder flagged as part of a hub block row (one vote decides; then a second vote
// skips groups without a run).
template <typename V, bool SCALED>
__device__ __forceinline__ void coo_finish(const CooPend<V> &r, V scale, V *__restrict__ y, Dbg dbg, bool runs) {
  V p = r.v * r.xv;
  if constexpr (SCALED) p *= scale;
  if (runs && __any_sync(kFull, r.hub)) {
    const int lane = threadIdx.x & 31;
    const uint32_t key = r.valid ? r.yrow : 0xFFFFFFFFu - (uint32_t)lane;  // invalid lanes: unique keys
    const uint32_t kn = __shfl_down_sync(kFull, key, 1);
    bool tail = lane == 31 || kn != key;  // last lane of its run
    if (__any_sync(kFull, !tail)) {
      const uint32_t kp = __shfl_up_sync(kFull, key, 1);
      const bool head = lane == 0 || kp != key;
      // segmented suffix scan: p = sum over [lane, end of run]
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const V o = __shfl_down_sync(kFull, p, d);
        const bool ot = __shfl_down_sync(kFull, tail, d);
        if (!tail && lane + d < 32) {
          p += o;
          tail = ot;
        }
      }
      if (r.valid && head) red_add(y + r.yrow, p, dbg);
      return;
    }
  }
  if (r.valid) red_add(y + r.yrow, p, dbg);
}

// x tile of one block loaded by the warp itself (aggregated matrices have no gather warps):
// lanes 0-15 fetch restore_cols[c] -> x, lanes 16-31 mirror; returned in shared scratch xt.
template <typename V, bool AGG>
__device__ __forceinline__ const V *warp_tile(const uint8_t *page, const uint4 &d, const V *__restrict__ x, V *scratch,
                                              int lane, Dbg dbg) {
  if constexpr (AGG) {
    const int c = lane & 15;
    if (lane < 16 && c < d_ncols(d)) {
      const uint32_t col = reinterpret_cast<const uint32_t *>(page + d.y)[c];
      scratch[c] = (dbg.skip() & 2) ? V(1) + V(col & 1) : __ldg(x + col);
    }
    __syncwarp();
  }
  return scratch;
}

// A COO block too large for a group (forced format): chunks of 32 elements.
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void coo_big(const uint8_t *page, const uint4 &d, const V *xt, V scale,
                                        V *__restrict__ y, int lane, Dbg dbg) {
  const uint8_t *body = page + (d.z & 0xFFFFu);
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const int nnz = d_nnz(d);
  for (int e = lane; e < nnz; e += 32) {
    const uint32_t byte = body[e];
    V p = V(vals[e]) * xt[byte >> 4];
    if constexpr (SCALED) p *= scale;
    red_add(y + d.x + (byte & 15), p, dbg);
  }
}

// CSR: 17 u8 row_ptr, nnz u8 local cols, pad, values; lanes 2r, 2r+1 share row r
// ("32 threads collaboratively compute 16 y elements").
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void csr_path(const uint8_t *page, const uint4 &d, const V *xt, V scale,
                                         V *__restrict__ y, int lane, Dbg dbg) {
  const uint8_t *body = page + (d.z & 0xFFFFu);
  const uint8_t *cols = body + 17;
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const int nnz = d_nnz(d);
  const int r = lane >> 1, h = lane & 1;
  const int lo = body[r];
  const int hi = r < 15 ? (int)body[r + 1] : nnz;  // row_ptr[16] = nnz (R-8)
  V acc = V(0);
  for (int e = lo + h; e < hi; e += 2) acc = fma(V(vals[e]), xt[cols[e]], acc);
  acc += __shfl_xor_sync(kFull, acc, 1);
  if constexpr (SCALED) acc *= scale;
  if (h == 0 && hi > lo) red_add(y + d.x + r, acc, dbg);
}

// DENSE (Alg. 4): the device record stores the 256 values lane-major: slot
// k*32 + lane holds A[lane % 16][(lane / 16) * 8 + k], so lane l owns row l % 16, columns
// 8*(l/16) .. +7 — conflict-free 8-byte shared loads, 8 FMAs against the broadcast x tile, one
// shfl_xor(16) joins the two half rows (the semantics of Alg. 4's shfl, R-15), 16 REDs.
template <typename M, typename V, bool SCALED>
__device__ __forceinline__ void dense_path(const uint8_t *page, const uint4 &d, const V *xt, V scale,
                                           V *__restrict__ y, int64_t m, int lane, Dbg dbg) {
  const M *vals = reinterpret_cast<const M *>(page + (d.z >> 16));
  const int h = lane >> 4, r = lane & 15, nc = d_ncols(d);
  // absent entries (stored zeros) must contribute 0 even against non-finite x: check the tile once
  const bool finite = __all_sync(kFull, r >= nc || isfinite(xt[r]));
  V acc = V(0);
  if (finite && nc == 16) {  // full tile (every block column but a ragged last one)
#pragma unroll
    for (int k = 0; k < 8; k++) acc = fma(V(vals[k * 32 + lane]), xt[h * 8 + k], acc);
  } else if (finite) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int c = h * 8 + k;
      acc = fma(V(vals[k * 32 + lane]), c < nc ? xt[c] : V(0), acc);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const V v = V(vals[k * 32 + lane]);
      const int c = h * 8 + k;
      if (v != V(0)) acc = fma(v, xt[c], acc);
    }
  }
  acc += __shfl_xor_sync(kFull, acc, 16);
  if constexpr (SCALED) acc *= scale;
  if (h == 0 && (int64_t)d.x + r < m) red_add(y + d.x + r, acc, dbg);
}

// ------------------------------------------------------------------ the persistent kernel
struct KParams {
  const uint8_t *stream;
  const uint64_t *page_off;
  const uint32_t *cta_page;
  uint32_t *page_ctr;  // dynamic page claiming: {next page, finished producers}; nullptr = static ranges
  uint32_t n_pages;
  uint32_t claim_chunk;  // pages per dynamic claim
  int wait_sleep_ns;     // consumers: __nanosleep between full-barrier probes
  int strided;           // static: K > 0 -> CTA g takes runs of K pages g, g + grid, ... (0: contiguous range)
  int64_t m;
  const double *sumsq;
  int stage;     // bytes per stage: page data + its x tiles
  int nstage;
  int groups;    // consumer groups in this CTA (page i of the CTA -> group i % groups)
  int vec16;     // non-aggregated x tiles: 16-byte cp.async (x 16-byte aligned)
  int static_items;  // non-aggregated: warp w of a group takes items w, w + 6, ... instead of claiming
                     // from the stage counter (pages hold whole Alg. 2-balanced TBs, so the
                     // round-robin split is balanced; saves ~10 instructions per item)
  Dbg dbg;
};

// Issue the x tiles of a work item's blocks (non-aggregated: x[bc*16 .. bc*16 + ncols)) into
// their slots of the stage's tile area with 16-byte cp.async (8 lanes per fp64 tile, up to 4
// member blocks per item), as one cp.async group; used one item ahead of processing.
template <typename V>
__device__ __forceinline__ void issue_tiles(const uint4 *descs, uint32_t iw, V *xbuf, const V *__restrict__ x,
                                            bool vec16, uint64_t pol, int lane, Dbg dbg) {
  constexpr int kPer = 16 / (int)sizeof(V), kChunks = 16 / kPer;
  const int hb = iw & 0xFFF;
  const int members = (int)((iw >> 14) & 3) + 1;
  const int mem = lane / kChunks, c = (lane % kChunks) * kPer;
  if (mem < members && !(dbg.skip() & 8)) {
    const uint4 d = descs[hb + mem];
    const int nc = d_ncols(d);
    V *dst = xbuf + (hb + mem) * 16 + c;
    if (dbg.skip() & 2) {
      for (int q = 0; q < kPer; q++) dst[q] = V(1);
    } else if (vec16 && c + kPer <= nc) {
      cp_async_16(dst, x + d.y + c, pol);
    } else {
      for (int q = c; q < c + kPer && q < nc; q++) cp_async_elem(dst + (q - c), x + d.y + q, pol);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Warp roles: 0 = TMA producer, the rest = consumer groups.  M: matrix value type of the
// records; V: type of x, y and the accumulation (M = float, V = double: the mixed variant).
template <typename M, typename V, bool AGG, bool SCALED, bool RUNS>
__global__ void __launch_bounds__(kMaxThreads, 1)
    cb_spmv_kernel(KParams P, const V *__restrict__ x, V *__restrict__ y) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + 2 * kMaxStages;
  uint32_t *claim = reinterpret_cast<uint32_t *>(empty + kMaxStages);
  // local sequence index of the page in each stage (written by the producer before its arrive)
  volatile uint32_t *stage_seq = claim + kMaxStages;
  uint8_t *ring = smem + kSmemHeader;
  V *scratch = reinterpret_cast<V *>(ring + (size_t)P.nstage * P.stage);  // 16 values per consumer warp

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // static assignment: a contiguous byte-balanced page range per CTA, or (strided) pages
  // blockIdx.x, blockIdx.x + grid, ... so every CTA sees the whole slot order's mix of formats
  uint32_t p0 = P.cta_page[blockIdx.x], p1 = P.cta_page[blockIdx.x + 1];
  const uint32_t K = (uint32_t)P.strided;  // strided: runs of K consecutive pages, dealt round robin
  if (K) {
    p0 = 0;
    p1 = 0;  // local page count
    for (uint64_t c = blockIdx.x; c * K < P.n_pages; c += gridDim.x) {
      const uint64_t left = P.n_pages - c * K;
      p1 += (uint32_t)(left < K ? left : K);
    }
  }
  const int S = P.nstage;
  const Dbg dbg = P.dbg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGroupWarps);
      claim[s] = 0;
      stage_seq[s] = 0xFFFFFFFFu;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: one bulk copy per page into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t round = 0;
      auto next_stage = [&]() {
        if (round > 0) {
          mbar_wait(&empty[s], (round - 1) & 1);  // every consumer warp released the stage
          claim[s] = 0;                           // published by the release of arrive below
        }
      };
      auto load_page = [&](uint32_t p) {
        const uint64_t off = P.page_off[p];
        const uint32_t bytes = (uint32_t)(P.page_off[p + 1] - off);
        stage_seq[s] = round * (uint32_t)S + (uint32_t)s;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * P.stage, P.stream + off, bytes, &full[s], pol);
        if (++s == S) { s = 0; round++; }
      };
      if (P.page_ctr == nullptr) {
        for (uint32_t i = p0; i < p1; i++) {
          next_stage();
          load_page(K ? ((i / K) * gridDim.x + blockIdx.x) * K + i % K : i);
        }
      } else {
        // Dynamic claiming (SMs that finish early take more pages): pages come from a global
        // counter; then one end marker per consumer group (a 16-byte header with nblk = kEndPage
        // in the next G stages of the sequence, so every group meets exactly one), and the last
        // producer resets the counter for the next launch on the stream.
        // claims of claim_chunk pages (8: measured sweep at the launch site); the next claim is
        // issued before the current chunk is loaded, so the atomic's round trip overlaps the
        // stage waits and copies
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
        for (int g = 0; g < P.groups; g++) {
          next_stage();
          stage_seq[s] = round * (uint32_t)S + (uint32_t)s;
          mbar_arrive_expect_tx(&full[s], 16u);
          bulk_g2s(ring + (size_t)s * P.stage, kEndHeader, 16u, &full[s], pol);
          if (++s == S) { s = 0; round++; }
        }
        if (atomicAdd(&P.page_ctr[1], 1u) == gridDim.x - 1) {
          P.page_ctr[0] = 0;
          P.page_ctr[1] = 0;
        }
      }
    }
    return;
  }

  // ---------------- consumers: group g takes pages g, g + G, ...; its warps claim work items.
  // Aggregated matrices gather x per element straight into registers (the next COO group's
  // loads are issued before the current one is finished); non-aggregated matrices copy each
  // item's x tiles into the stage one item ahead (cp.async groups).
  V scale = V(1);
  if constexpr (SCALED) scale = (V)(1.0 / sqrt(*P.sumsq));
  const int cw = warp - 1;
  V *wscratch = scratch + cw * 16;
  const uint64_t xpol = policy_evict_last();
  const int G = P.groups, grp = cw / kGroupWarps;
  constexpr bool runs = RUNS;  // hub block rows: same-row run sums before the COO REDs
  int s = grp % S;
  uint32_t parity = (uint32_t)((grp / S) & 1);
  const bool dyn = P.page_ctr != nullptr;
  uint32_t li = (uint32_t)grp;  // local sequence index of this group's next page
  for (uint32_t p = p0 + grp; dyn || p < p1; p += G, li += (uint32_t)G) {
    // Stages are shared by the groups in turn (page i -> stage i % S, group i % G), so this
    // group can reach its round of stage s while an earlier round, another group's page, is
    // still in flight there, and the phase parity cannot tell round r + 1 from r - 1.  The
    // producer records each page's local index in stage_seq before its arrive, after the
    // earlier round was released: once the stage shows our index, the parity wait is exact.
    while (stage_seq[s] != li) __nanosleep(64);  // producer not there yet: sleep, do not burn issue slots
    mbar_wait_sleep(&full[s], parity, P.wait_sleep_ns);
    const uint8_t *page = ring + (size_t)s * P.stage;
    const uint32_t *hdr = reinterpret_cast<const uint32_t *>(page);
    if (dyn && hdr[0] == kEndPage) break;  // this group's end marker (nothing to release)
    const int nitems = (dbg.skip() & 4) ? 0 : (int)hdr[1];
#if CBSPMV_CHECK
    // debug build: the stage must hold a well-formed page header (a stale / torn stage traps)
    if (hdr[2] != cb::kPageHeader + 16u * hdr[0] || hdr[0] == 0u || hdr[0] > 4096u || nitems > (int)hdr[0]) {
      if (lane == 0) printf("bad page header cta %d warp %d s %d: %u %u %u %u\n", blockIdx.x, warp, s, hdr[0], hdr[1], hdr[2], hdr[3]);
      __trap();
    }
#endif
    const uint32_t *items = reinterpret_cast<const uint32_t *>(page + hdr[2]);
    V *xbuf = reinterpret_cast<V *>(ring + (size_t)s * P.stage + hdr[3]);
    const uint4 *descs = reinterpret_cast<const uint4 *>(page + cb::kPageHeader);
    if constexpr (AGG) {
      // Claims of 4 items.  When all 4 are COO groups (the common case on aggregated, super-
      // sparse matrices) their load chains (descriptor -> record -> restore entry -> x) are
      // issued straight-line so the four chains overlap, then the four are finished.
      uint32_t kb = 0;
      if (lane == 0) kb = atomicAdd(&claim[s], 4u);
      kb = __shfl_sync(kFull, kb, 0);
      // the claim counter starts at 0 and moves by 4: kb is a multiple of 4 (16-byte aligned), and
      // the item table is zero-padded to 16 bytes, so the 128-bit load stays inside the page
      while ((int)kb < nitems) {
        uint32_t kn = 0;
        if (lane == 0) kn = atomicAdd(&claim[s], 4u);
        const uint4 iw4 = *reinterpret_cast<const uint4 *>(items + kb);
        const uint32_t iws[4] = {iw4.x, iw4.y, iw4.z, iw4.w};
        const int nv = min(4, nitems - (int)kb);
        bool all_coo = nv == 4;
#pragma unroll
        for (int j = 0; j < 4; j++) all_coo &= ((iws[j] >> 12) & 3) == CBSPMV_FMT_COO && !(iws[j] >> 31);
        if (all_coo) {
          CooPend<V> q[4];
#pragma unroll
          for (int j = 0; j < 4; j++) q[j] = coo_issue<M, V, AGG>(page, descs, iws[j], xbuf, x, lane, dbg, xpol);
#pragma unroll
          for (int j = 0; j < 4; j++) coo_finish<V, SCALED>(q[j], scale, y, dbg, runs);
        } else {
          for (int j = 0; j < nv; j++) {
            const uint32_t iw = iws[j];
            const int t = (iw >> 12) & 3;
            if (t == CBSPMV_FMT_COO && !(iw >> 31)) {
              coo_finish<V, SCALED>(coo_issue<M, V, AGG>(page, descs, iw, xbuf, x, lane, dbg, xpol), scale, y, dbg, runs);
            } else {
              const uint4 dh = descs[iw & 0xFFF];
              const V *xt = warp_tile<V, AGG>(page, dh, x, wscratch, lane, dbg);
              if (t == CBSPMV_FMT_COO) coo_big<M, V, SCALED>(page, dh, xt, scale, y, lane, dbg);
              else if (t == CBSPMV_FMT_CSR) csr_path<M, V, SCALED>(page, dh, xt, scale, y, lane, dbg);
              else dense_path<M, V, SCALED>(page, dh, xt, scale, y, P.m, lane, dbg);
              __syncwarp();
            }
          }
        }
        kb = __shfl_sync(kFull, kn, 0);
      }
    } else {
      const uint32_t wg = (uint32_t)(cw % kGroupWarps);
      uint32_t k = 0;
      if (P.static_items) {
        k = wg;
      } else {
        if (lane == 0) k = atomicAdd(&claim[s], 1u);
        k = __shfl_sync(kFull, k, 0);
      }
      uint32_t iw = (int)k < nitems ? items[k] : 0u;
      if ((int)k < nitems) issue_tiles<V>(descs, iw, xbuf, x, P.vec16, xpol, lane, dbg);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      while ((int)k < nitems) {
        uint32_t kn = 0;
        if (P.static_items) {
          kn = k + kGroupWarps;
        } else {
          if (lane == 0) kn = atomicAdd(&claim[s], 1u);
          kn = __shfl_sync(kFull, kn, 0);
        }
        const uint32_t iwn = (int)kn < nitems ? items[kn] : 0u;
        if ((int)kn < nitems) issue_tiles<V>(descs, iwn, xbuf, x, P.vec16, xpol, lane, dbg);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // item k's tiles have landed
        __syncwarp();
        const int t = (iw >> 12) & 3, hb = iw & 0xFFF;
        if (t == CBSPMV_FMT_COO && !(iw >> 31)) {
          coo_finish<V, SCALED>(coo_issue<M, V, AGG>(page, descs, iw, xbuf, x, lane, dbg, xpol), scale, y, dbg, runs);
        } else {
          const uint4 dh = descs[hb];
          const V *xt = xbuf + hb * 16;
          if (t == CBSPMV_FMT_COO) coo_big<M, V, SCALED>(page, dh, xt, scale, y, lane, dbg);
          else if (t == CBSPMV_FMT_CSR) csr_path<M, V, SCALED>(page, dh, xt, scale, y, lane, dbg);
          else dense_path<M, V, SCALED>(page, dh, xt, scale, y, P.m, lane, dbg);
        }
        k = kn;
        iw = iwn;
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    s += G;
    while (s >= S) { s -= S; parity ^= 1u; }
  }
}

template <typename V>
__global__ void cb_zero_kernel(V *__restrict__ y, int64_t m) {
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

template <typename M, typename V>
const void *kernel_ptr(int agg, bool scaled, bool runs) {
  if (agg && runs)
    return scaled ? (const void *)&cb_spmv_kernel<M, V, true, true, true> : (const void *)&cb_spmv_kernel<M, V, true, false, true>;
  if (agg) return scaled ? (const void *)&cb_spmv_kernel<M, V, true, true, false> : (const void *)&cb_spmv_kernel<M, V, true, false, false>;
  return scaled ? (const void *)&cb_spmv_kernel<M, V, false, true, false> : (const void *)&cb_spmv_kernel<M, V, false, false, false>;
}

// runs (in-warp same-row run sums before COO REDs) is compiled only into the aggregated kernels:
// hub block rows come with power-law matrices, which the th0 rule aggregates
const void *select_kernel(int dtype, int agg, bool scaled, bool runs) {
  if (dtype == CBSPMV_F64) return kernel_ptr<double, double>(agg, scaled, runs);
  if (dtype == CBSPMV_F32) return kernel_ptr<float, float>(agg, scaled, runs);
  return kernel_ptr<float, double>(agg, scaled, runs);  // CBSPMV_F32F64
}

// bytes of one x / y element
inline int vec_bytes(int dtype) { return dtype == CBSPMV_F32 ? 4 : 8; }

inline int cuda_fail(cudaError_t e, const char *what, std::string *err) {
  *err = std::string(what) + ": " + cudaGetErrorString(e);
  return CBSPMV_ECUDA;
}

int sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

}  // namespace

int cb_configure(CbDevice *dev, std::string *err) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute", err);
  int smem_sm = 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev->device);
  // Launch shape (measured on B200): one persistent CTA per SM with 4 consumer
  // groups of 6 warps sharing an 8-stage ring; CTAs-per-SM / groups are overridable for tuning.
  const char *env = std::getenv("CBSPMV_CTAS_PER_SM");
  int ctas = env ? std::atoi(env) : 1;
  if (ctas < 1) ctas = 1;
  const char *genv = std::getenv("CBSPMV_GROUPS");
  int groups = genv ? std::atoi(genv) : 5;
  groups = std::max(1, std::min(kMaxGroups, groups));
  dev->groups = groups;
  const int header = kSmemHeader + groups * kGroupWarps * 16 * vec_bytes(dev->dtype);
  const int stage = dev->page_cap;
  const int budget = std::min(optin, smem_sm / ctas - 1024);  // 1 KB per CTA is reserved by the system
  int nstage = (budget - header) / stage;
  if (nstage > kMaxStages) nstage = kMaxStages;
  if (nstage < groups + 1) {
    *err = "page capacity too large for shared memory";
    return CBSPMV_EUNSUPPORTED;
  }
  dev->nstage = nstage;
  dev->consumers = groups * kGroupWarps;
  for (int dt = 0; dt < 3; dt++)
    for (int agg = 0; agg < 2; agg++)
      for (int sc = 0; sc < 4; sc++) {
        e = cudaFuncSetAttribute(select_kernel(dt, agg, sc & 1, sc >> 1), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
      }
  const int sms = sm_count(dev->device) * ctas;
  int64_t g = dev->n_pages < sms ? dev->n_pages : sms;
  dev->grid = (int)(g < 1 ? 1 : g);
  return CBSPMV_OK;
}

int cb_launch_spmv(const CbDevice &dev, const void *x, void *y, const double *sumsq, bool zero_y, void *stream,
                   std::string *err) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int sms = sm_count(dev.device);
  if (zero_y && dev.m > 0) {
    const int zb = 256;
    int64_t need = (dev.m + zb - 1) / zb;
    int zg = (int)(need < (int64_t)sms * 8 ? need : (int64_t)sms * 8);
    if (vec_bytes(dev.dtype) == 8) cb_zero_kernel<double><<<zg, zb, 0, st>>>((double *)y, dev.m);
    else cb_zero_kernel<float><<<zg, zb, 0, st>>>((float *)y, dev.m);
  }
  static const int dbg_skip = [] {
    const char *v = std::getenv("CBSPMV_DEBUG_SKIP");
    return v ? std::atoi(v) : 0;
  }();
  if (dev.n_pages > 0) {
    const int stage = dev.page_cap;
    const int vec16 = !dev.agg && ((uintptr_t)x % 16 == 0);
    static const int static_items = [] {
      const char *v = std::getenv("CBSPMV_STATIC_ITEMS");  // default on (measured)
      return v ? std::atoi(v) : 1;
    }();
    // Dynamic page claiming for large aggregated matrices (per-page work follows the random
    // gathers and atomics, static byte ranges leave a tail: R-MAT 1.21 -> 1.17 ms, uniform power
    // iteration 15.5 -> 15.1 ms per step); non-aggregated matrices (clustered: 0.836 static vs
    // 0.856 ms dynamic) and small ones (< 32 pages per CTA; Laplacian, 20: 0.034 vs 0.039 ms) keep
    // static contiguous ranges.  CBSPMV_DYNAMIC_PAGES = 0 / 1 overrides (A/B, tests).
    static const int dynamic_env = [] {
      const char *v = std::getenv("CBSPMV_DYNAMIC_PAGES");
      return v ? std::atoi(v) : -1;
    }();
    const bool dynamic_pages =
        dynamic_env >= 0 ? dynamic_env != 0 : (dev.agg && dev.n_pages >= 32 * (int64_t)dev.grid);
    uint32_t *ctr = nullptr;
    if (dynamic_pages && dev.d_page_ctr) {
      // atomic slot pick: two host threads launching the same handle get different slots
      const uint32_t slot = __atomic_fetch_add(&dev.ctr_next, 1u, __ATOMIC_RELAXED);
      ctr = dev.d_page_ctr + 2 * (slot % cb::kCtrSlots);
    }
    static const uint32_t claim_chunk = [] {
      const char *v = std::getenv("CBSPMV_CLAIM_CHUNK");
      const int c = v ? std::atoi(v) : 8;  // R-MAT: 2 -> 1.205, 4 -> 1.168, 8 -> 1.130, 32 -> 1.135 ms
      return (uint32_t)(c < 1 ? 1 : c);
    }();
    // Static assignment for the rest: 4-byte stored values (fp32, mixed) are issue-bound, so
    // each CTA takes a strided share of the slot order, mixing instruction-heavy (CSR) and light
    // (DENSE) pages evenly (clustered fp32 0.708 -> 0.630 ms, mixed 0.781 -> 0.715 ms); fp64 is
    // bandwidth-bound and keeps contiguous byte-balanced ranges (strided: 0.832 -> 0.856 ms).
    // CBSPMV_STRIDED_PAGES = 0 / 1 overrides.
    static const int strided_env = [] {
      const char *v = std::getenv("CBSPMV_STRIDED_PAGES");
      return v ? std::atoi(v) : -1;
    }();
    const int strided = ctr ? 0 : (strided_env >= 0 ? strided_env : (dev.dtype != CBSPMV_F64 ? 1 : 0));  // run length
    static const int wait_sleep_ns = [] {
      const char *v = std::getenv("CBSPMV_WAIT_SLEEP_NS");
      return v ? std::atoi(v) : 0;
    }();
    KParams P{dev.d_stream, dev.d_page_off, dev.d_cta_page, ctr, (uint32_t)dev.n_pages, claim_chunk, wait_sleep_ns, strided, dev.m,
              sumsq, stage,
              dev.nstage, dev.groups,
              vec16, static_items, Dbg{dbg_skip}};
    const int smem = kSmemHeader + dev.nstage * stage + dev.groups * kGroupWarps * 16 * vec_bytes(dev.dtype);
    const void *fn = select_kernel(dev.dtype, dev.agg, sumsq != nullptr, dev.coo_runs != 0);
    void *args[] = {&P, const_cast<void **>(&x), &y};
    const int threads = 32 * (1 + dev.groups * kGroupWarps);
    cudaError_t e = cudaLaunchKernel(fn, dim3(dev.grid), dim3(threads), args, (size_t)smem, st);
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
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = sm_count(dev);
    int64_t need = (len + 255) / 256;
    int g = (int)(need < (int64_t)sms * 4 ? need : (int64_t)sms * 4);
    if (vec_bytes(dtype) == 8) cb_sumsq_kernel<double><<<g, 256, 0, st>>>((const double *)v, len, out);
    else cb_sumsq_kernel<float><<<g, 256, 0, st>>>((const float *)v, len, out);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sumsq launch", err);
  return CBSPMV_OK;
}
