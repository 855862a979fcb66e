// kernels.cu — sm_100a kernels of the CB-SpMV hot path (y = A·x, §3.5).
//
// One persistent CTA per SM streams its contiguous range of device pages
// through a ring of shared-memory stages:
//   warp 0 (one elected lane)  : producer — mbarrier wait on "empty", then one
//                                cp.async.bulk (TMA, SASS UBLKCP) per page into the stage,
//                                completion counted on the stage's "full" mbarrier;
//                                pages are streamed with an L2 evict_first policy so the
//                                matrix does not evict x.
//   warps 1..kConsumerWarps    : consumers — each takes blocks of the page, one block per
//                                warp at a time (the paper's warp <-> sub-block mapping,
//                                P:403), U blocks batched so their x gathers overlap.
// Per-format warp paths (one warp per sub-block):
//   COO   (Alg. 3): lane i <-> element i; coordinate byte row = b & 15,
//         col = b >> 4; x from the 16-lane x tile by shuffle; products
//         reduced per row with a segmented warp shuffle, one RED per distinct row
//         instead of one atomic per element.
//   CSR   ("optimizing intra-block computation using the shfl function",
//         P:570 "32 threads collaboratively compute 16 y elements"): two lanes per row.
//   DENSE (Alg. 4): 256 row-major values, conflict-free 8-byte shared loads,
//         a transposing xor-butterfly (8,4,2,1) leaves one full row sum per lane pair.
// x tile: lane l holds x for column (l & 15) of the block —
//   x[bc*16 + c] without aggregation (replaces the shared-memory s_x), or
//   x[restore_cols[cols_offset[br] + bc*16 + c]] with aggregation (the restore entries
//   are inlined in front of the record in the page).
// y is accumulated with red.global.add (atomicAdd without return), as the paper's
// atomicAdd; y is zeroed first by cb_zero_kernel (R-16).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "cb_internal.h"

namespace {

constexpr int kConsumerWarps = 24;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kMaxStages = 16;
constexpr int kSmemHeader = 512;  // full[16], empty[16] mbarriers + claim[16] counters; keeps stages aligned
constexpr int kBatch = 4;         // blocks per claim: x gathers of 2 blocks per load instruction
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
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

template <typename V>
__device__ __forceinline__ void red_add(V *p, V v) {
  atomicAdd(p, v);  // result unused -> RED.E.ADD
}

__device__ __forceinline__ int pad_to(int bytes, int a) { return (bytes + a - 1) & ~(a - 1); }

struct Blk {          // a decoded 16-byte descriptor
  uint32_t row0;      // y row base (blk_row_idx * 16)
  int nnz;            // 1..256; 0 = no block
  int type;           // CBSPMV_FMT_*; 3 = no block
  const uint8_t *body;  // the canonical record (after the inlined restore entries)
};

template <bool AGG>
__device__ __forceinline__ Blk decode(const uint8_t *page, uint4 d) {
  Blk b;
  b.row0 = d.x;
  b.type = (d.z >> 24) & 3;
  b.nnz = b.type == 3 ? 0 : (int)((d.z >> 16) & 0xFF) + 1;
  const uint8_t *rec = page + ((d.z & 0xFFFFu) << 4);
  b.body = AGG ? rec + ((d.w + 3u) & ~3u) * 4u : rec;
  return b;
}

// Segmented warp reduction over rows sorted within [lane, end): after the rounds, each
// segment head holds its segment's sum.  Rounds adapt to the longest segment.
template <typename V>
__device__ __forceinline__ V seg_reduce(V p, bool head, int end, int lane) {
  const int seglen = head ? end - lane : 0;
  const int maxlen = (int)__reduce_max_sync(kFull, (unsigned)seglen);
  for (int d = 1; d < maxlen; d <<= 1) {
    const V o = __shfl_down_sync(kFull, p, d);
    if (lane + d < end) p += o;
  }
  return p;
}

// ------------------------------------------------------------------ per-format warp paths
// COO (Alg. 3), one block per warp: lane <-> element (chunks of 32 when forced on dense blocks).
// xr holds the block's x tile in lanes base..base+15.
template <typename V>
__device__ __forceinline__ void coo_path(const Blk &b, V xr, int base, V *__restrict__ y, int lane) {
  const V *vals = reinterpret_cast<const V *>(b.body + pad_to(b.nnz, (int)sizeof(V)));
  for (int c0 = 0; c0 < b.nnz; c0 += 32) {
    const int e = c0 + lane;
    const bool valid = e < b.nnz;
    const uint32_t byte = valid ? b.body[e] : 0u;
    const int row = byte & 15, col = byte >> 4;
    const V v = valid ? vals[e] : V(0);
    const V xv = __shfl_sync(kFull, xr, base + col);
    V p = v * xv;
    const int prow = __shfl_up_sync(kFull, row, 1);
    const bool head = valid && (lane == 0 || prow != row);
    const uint32_t heads = __ballot_sync(kFull, head);
    const uint32_t above = heads & ~((2u << lane) - 1u);
    const int lim = min(32, b.nnz - c0);
    const int end = above ? min(__ffs(above) - 1, lim) : lim;
    p = seg_reduce(p, head, end, lane);
    if (head) red_add(y + b.row0 + row, p);
  }
}

// Two COO blocks with nnz <= 16 in one warp: lanes 0-15 block A, lanes 16-31 block B;
// xr holds A's x tile in lanes 0-15 and B's in lanes 16-31.
template <typename V>
__device__ __forceinline__ void coo_pair_path(const Blk &A, const Blk &B, V xr, V *__restrict__ y, int lane) {
  const int h = lane >> 4, i = lane & 15;
  const uint8_t *body = h ? B.body : A.body;
  const int nnz = h ? B.nnz : A.nnz;
  const uint32_t row0 = h ? B.row0 : A.row0;
  const V *vals = reinterpret_cast<const V *>(body + pad_to(nnz, (int)sizeof(V)));
  const bool valid = i < nnz;
  const uint32_t byte = valid ? body[i] : 0u;
  const int row = byte & 15, col = byte >> 4;
  const V v = valid ? vals[i] : V(0);
  const V xv = __shfl_sync(kFull, xr, (h << 4) | col);
  V p = v * xv;
  const int prow = __shfl_up_sync(kFull, row, 1);
  const bool head = valid && (i == 0 || prow != row);
  const uint32_t heads = __ballot_sync(kFull, head);
  const uint32_t above = heads & ~((2u << lane) - 1u);
  const int lim = (h << 4) + nnz;
  const int end = above ? min(__ffs(above) - 1, lim) : lim;
  p = seg_reduce(p, head, end, lane);
  if (head) red_add(y + row0 + row, p);
}

// CSR: 17 u8 row_ptr, nnz u8 local cols, pad, values; lanes 2r, 2r+1 share row r
// ("32 threads collaboratively compute 16 y elements").
template <typename V>
__device__ __forceinline__ void csr_path(const Blk &b, V xr, int base, V *__restrict__ y, int lane) {
  const uint8_t *cols = b.body + 17;
  const V *vals = reinterpret_cast<const V *>(b.body + pad_to(17 + b.nnz, (int)sizeof(V)));
  const int r = lane >> 1, h = lane & 1;
  const int lo = b.body[r];
  const int hi = r < 15 ? (int)b.body[r + 1] : b.nnz;  // row_ptr[16] = nnz (R-8)
  const int len = hi - lo;
  const int k = len > h ? (len - h + 1) >> 1 : 0;
  const int kmax = (int)__reduce_max_sync(kFull, (unsigned)k);
  V acc = V(0);
  for (int t = 0; t < kmax; t++) {
    const int e = lo + h + 2 * t;
    const bool valid = t < k;
    const int c = valid ? cols[e] : 0;
    const V v = valid ? vals[e] : V(0);
    const V xv = __shfl_sync(kFull, xr, base + c);
    if (valid) acc = fma(v, xv, acc);
  }
  acc += __shfl_xor_sync(kFull, acc, 1);
  if (h == 0 && len > 0) red_add(y + b.row0 + r, acc);
}

// DENSE (Alg. 4): element k*32 + lane is (row 2k + lane/16, col lane%16); a transposing
// xor-butterfly (8, 4, 2, 1) leaves the full sum of row 2*((lane>>1)&7) + lane/16 in lane pairs.
template <typename V>
__device__ __forceinline__ void dense_path(const Blk &b, V xr, int base, V *__restrict__ y, int64_t m, int lane) {
  const V *vals = reinterpret_cast<const V *>(b.body);
  const V xl = __shfl_sync(kFull, xr, base + (lane & 15));
  V p[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const V v = vals[k * 32 + lane];
    p[k] = v != V(0) ? v * xl : V(0);  // absent entries contribute 0 (explicit zeros were dropped)
  }
  const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  V q[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const V send = b3 ? p[j] : p[j + 4];
    const V keep = b3 ? p[j + 4] : p[j];
    q[j] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  V r2[2];
#pragma unroll
  for (int j = 0; j < 2; j++) {
    const V send = b2 ? q[j] : q[j + 2];
    const V keep = b2 ? q[j + 2] : q[j];
    r2[j] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  V s;
  {
    const V send = b1 ? r2[0] : r2[1];
    const V keep = b1 ? r2[1] : r2[0];
    s = keep + __shfl_xor_sync(kFull, send, 2);
  }
  s += __shfl_xor_sync(kFull, s, 1);
  const int row = 2 * ((lane >> 1) & 7) + (lane >> 4);
  if ((lane & 1) == 0 && (int64_t)b.row0 + row < m) red_add(y + b.row0 + row, s);
}

template <typename V>
__device__ __forceinline__ void single_path(const Blk &b, V xr, int base, V *__restrict__ y, int64_t m, int lane) {
  if (b.type == CBSPMV_FMT_COO) coo_path<V>(b, xr, base, y, lane);
  else if (b.type == CBSPMV_FMT_CSR) csr_path<V>(b, xr, base, y, lane);
  else if (b.type == CBSPMV_FMT_DENSE) dense_path<V>(b, xr, base, y, m, lane);
}

// ------------------------------------------------------------------ the persistent kernel
struct KParams {
  const uint8_t *stream;
  const uint64_t *page_off;
  const uint32_t *cta_page;
  int64_t m;
  const double *sumsq;
  int page_cap;
  int nstage;
};

template <typename V, bool AGG, bool SCALED>
__global__ void __launch_bounds__(kThreads, 1)
    cb_spmv_kernel(KParams P, const V *__restrict__ x, V *__restrict__ y) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem);
  uint64_t *empty = full + kMaxStages;
  uint32_t *claim = reinterpret_cast<uint32_t *>(empty + kMaxStages);
  uint8_t *ring = smem + kSmemHeader;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t p0 = P.cta_page[blockIdx.x], p1 = P.cta_page[blockIdx.x + 1];
  const int S = P.nstage;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
      claim[s] = 0;
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
      for (uint32_t p = p0; p < p1; p++) {
        if (round > 0) {
          mbar_wait(&empty[s], (round - 1) & 1);  // every consumer warp released the stage
          claim[s] = 0;                           // published by the release of arrive below
        }
        const uint64_t off = P.page_off[p];
        const uint32_t bytes = (uint32_t)(P.page_off[p + 1] - off);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * P.page_cap, P.stream + off, bytes, &full[s], pol);
        if (++s == S) { s = 0; round++; }
      }
    }
    return;
  }

  // ---------------- consumers: claim kBatch blocks at a time from the current page
  V scale = V(1);
  if constexpr (SCALED) scale = (V)(1.0 / sqrt(*P.sumsq));
  const int c16 = lane & 15, hl = lane >> 4;
  int s = 0;
  uint32_t parity = 0;
  for (uint32_t p = p0; p < p1; p++) {
    mbar_wait(&full[s], parity);
    const uint8_t *page = ring + (size_t)s * P.page_cap;
    const int nblk = *reinterpret_cast<const uint32_t *>(page);
    const uint4 *descs = reinterpret_cast<const uint4 *>(page + cb::kPageHeader);
    for (;;) {
      uint32_t b0 = 0;
      if (lane == 0) b0 = atomicAdd(&claim[s], (uint32_t)kBatch);
      b0 = __shfl_sync(kFull, b0, 0);
      if ((int)b0 >= nblk) break;
      const int nb = min(kBatch, nblk - (int)b0);
      Blk blk[kBatch];
      V xr[kBatch / 2];
#pragma unroll
      for (int u = 0; u < kBatch; u++) {
        const uint4 d = u < nb ? descs[b0 + u] : make_uint4(0, 0, 3u << 24, 0);
        blk[u] = decode<AGG>(page, d);
      }
      // x tiles: lanes 0-15 gather block 2g, lanes 16-31 block 2g+1
#pragma unroll
      for (int g = 0; g < kBatch / 2; g++) {
        const uint4 d = (2 * g + hl) < nb ? descs[b0 + 2 * g + hl] : make_uint4(0, 0, 3u << 24, 0);
        xr[g] = V(0);
        if (c16 < (int)d.w) {
          uint32_t col;
          if constexpr (AGG) col = reinterpret_cast<const uint32_t *>(page + ((d.z & 0xFFFFu) << 4))[c16];
          else col = d.y + c16;
          xr[g] = __ldg(x + col);
          if constexpr (SCALED) xr[g] *= scale;
        }
      }
#pragma unroll
      for (int g = 0; g < kBatch / 2; g++) {
        const Blk &A = blk[2 * g], &B = blk[2 * g + 1];
        if (A.type == CBSPMV_FMT_COO && A.nnz <= 16 && (B.type == 3 || (B.type == CBSPMV_FMT_COO && B.nnz <= 16))) {
          coo_pair_path<V>(A, B, xr[g], y, lane);
        } else {
          single_path<V>(A, xr[g], 0, y, P.m, lane);
          single_path<V>(B, xr[g], 16, y, P.m, lane);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; parity ^= 1u; }
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

using KFn = void (*)(KParams, const void *, void *);

template <typename V, bool AGG, bool SCALED>
const void *kernel_ptr() {
  return reinterpret_cast<const void *>(&cb_spmv_kernel<V, AGG, SCALED>);
}

const void *select_kernel(int dtype, int agg, bool scaled) {
  if (dtype == CBSPMV_F64) {
    if (agg) return scaled ? kernel_ptr<double, true, true>() : kernel_ptr<double, true, false>();
    return scaled ? kernel_ptr<double, false, true>() : kernel_ptr<double, false, false>();
  }
  if (agg) return scaled ? kernel_ptr<float, true, true>() : kernel_ptr<float, true, false>();
  return scaled ? kernel_ptr<float, false, true>() : kernel_ptr<float, false, false>();
}

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
  const int header = kSmemHeader;
  int nstage = (optin - header) / dev->page_cap;
  if (nstage > kMaxStages) nstage = kMaxStages;
  if (nstage < 2) {
    *err = "page capacity too large for shared memory";
    return CBSPMV_EUNSUPPORTED;
  }
  dev->nstage = nstage;
  dev->consumers = kConsumerWarps;
  const int smem = header + nstage * dev->page_cap;
  for (int dt = 0; dt < 2; dt++)
    for (int agg = 0; agg < 2; agg++)
      for (int sc = 0; sc < 2; sc++) {
        e = cudaFuncSetAttribute(select_kernel(dt, agg, sc), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute", err);
      }
  const int sms = sm_count(dev->device);
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
    if (dev.dtype == CBSPMV_F64) cb_zero_kernel<double><<<zg, zb, 0, st>>>((double *)y, dev.m);
    else cb_zero_kernel<float><<<zg, zb, 0, st>>>((float *)y, dev.m);
  }
  if (dev.n_pages > 0) {
    KParams P{dev.d_stream, dev.d_page_off, dev.d_cta_page, dev.m, sumsq, dev.page_cap, dev.nstage};
    const int smem = kSmemHeader + dev.nstage * dev.page_cap;
    const void *fn = select_kernel(dev.dtype, dev.agg, sumsq != nullptr);
    void *args[] = {&P, const_cast<void **>(&x), &y};
    cudaError_t e = cudaLaunchKernel(fn, dim3(dev.grid), dim3(kThreads), args, (size_t)smem, st);
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
    if (dtype == CBSPMV_F64) cb_sumsq_kernel<double><<<g, 256, 0, st>>>((const double *)v, len, out);
    else cb_sumsq_kernel<float><<<g, 256, 0, st>>>((const float *)v, len, out);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sumsq launch", err);
  return CBSPMV_OK;
}
