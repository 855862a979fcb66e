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

constexpr int kConsumerWarps = 16;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kMaxStages = 16;
constexpr int kBatch = 4;  // blocks per consumer warp whose x gathers are issued together
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

// ------------------------------------------------------------------ per-format warp paths
// COO (Alg. 3): lane <-> element, segmented per-row reduction, RED per distinct row.
template <typename V>
__device__ __forceinline__ void coo_path(const uint8_t *body, int nnz, uint32_t row0, V xr, V *__restrict__ y,
                                         int lane) {
  const V *vals = reinterpret_cast<const V *>(body + pad_to(nnz, (int)sizeof(V)));
  for (int base = 0; base < nnz; base += 32) {
    const int e = base + lane;
    const bool valid = e < nnz;
    const uint32_t b = valid ? body[e] : 0u;
    const int row = b & 15, col = b >> 4;
    const V v = valid ? vals[e] : V(0);
    const V xv = __shfl_sync(kFull, xr, col);
    V p = v * xv;
    const int prow = __shfl_up_sync(kFull, row, 1);
    const bool head = valid && (lane == 0 || prow != row);
    const uint32_t heads = __ballot_sync(kFull, head);
    const int nvalid = min(32, nnz - base);
    const uint32_t above = heads & ~((2u << lane) - 1u);
    const int end = above ? __ffs(above) - 1 : nvalid;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const V o = __shfl_down_sync(kFull, p, d);
      if (lane + d < end) p += o;
    }
    if (head) red_add(y + row0 + row, p);
  }
}

// CSR: 17 u8 row_ptr, nnz u8 local cols, pad, values; lanes 2r, 2r+1 share row r.
template <typename V>
__device__ __forceinline__ void csr_path(const uint8_t *body, int nnz, uint32_t row0, V xr, V *__restrict__ y,
                                         int lane) {
  const uint8_t *cols = body + 17;
  const V *vals = reinterpret_cast<const V *>(body + pad_to(17 + nnz, (int)sizeof(V)));
  const int r = lane >> 1, h = lane & 1;
  const int lo = body[r];
  const int hi = r < 15 ? (int)body[r + 1] : nnz;  // row_ptr[16] = nnz (R-8)
  const int len = hi - lo;
  const int k = len > h ? (len - h + 1) >> 1 : 0;
  const int kmax = __reduce_max_sync(kFull, (unsigned)k);
  V acc = V(0);
  for (int t = 0; t < kmax; t++) {
    const int e = lo + h + 2 * t;
    const bool valid = t < k;
    const int c = valid ? cols[e] : 0;
    const V v = valid ? vals[e] : V(0);
    const V xv = __shfl_sync(kFull, xr, c);
    if (valid) acc = fma(v, xv, acc);
  }
  acc += __shfl_xor_sync(kFull, acc, 1);
  if (h == 0 && len > 0) red_add(y + row0 + r, acc);
}

// DENSE (Alg. 4): element k*32 + lane is (row 2k + lane/16, col lane%16): the lane's own x.
template <typename V>
__device__ __forceinline__ void dense_path(const uint8_t *body, uint32_t row0, V xr, V *__restrict__ y, int64_t m,
                                           int lane) {
  const V *vals = reinterpret_cast<const V *>(body);
  V p[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const V v = vals[k * 32 + lane];
    p[k] = v != V(0) ? v * xr : V(0);  // absent entries contribute 0 (explicit zeros were dropped)
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
  if ((lane & 1) == 0 && (int64_t)row0 + row < m) red_add(y + row0 + row, s);
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
  uint8_t *ring = smem + 2 * kMaxStages * sizeof(uint64_t);  // 256 B: keeps stages 128-B aligned

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t p0 = P.cta_page[blockIdx.x], p1 = P.cta_page[blockIdx.x + 1];
  const int S = P.nstage;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t i = 0;
      for (uint32_t p = p0; p < p1; p++, i++) {
        const int s = i % S;
        const uint32_t round = i / S;
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        const uint64_t off = P.page_off[p];
        const uint32_t bytes = (uint32_t)(P.page_off[p + 1] - off);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * P.page_cap, P.stream + off, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- consumers
  const int cw = warp - 1;
  V scale = V(1);
  if constexpr (SCALED) scale = (V)(1.0 / sqrt(*P.sumsq));
  const int c16 = lane & 15;
  uint32_t i = 0;
  for (uint32_t p = p0; p < p1; p++, i++) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const uint8_t *page = ring + (size_t)s * P.page_cap;
    const int nblk = *reinterpret_cast<const uint32_t *>(page);
    for (int b0 = cw * kBatch; b0 < nblk; b0 += kConsumerWarps * kBatch) {
      uint4 d[kBatch];
      V xr[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; u++) {
        const int b = b0 + u;
        xr[u] = V(0);
        d[u] = make_uint4(0, 0, 3u << 24, 0);
        if (b < nblk) {
          d[u] = *reinterpret_cast<const uint4 *>(page + cb::kPageHeader + cb::kDescBytes * b);
          if (c16 < (int)d[u].w) {
            uint32_t col;
            if constexpr (AGG) {
              const uint32_t *restore = reinterpret_cast<const uint32_t *>(page + ((d[u].z & 0xFFFFu) << 4));
              col = restore[c16];
            } else {
              col = d[u].y + c16;
            }
            xr[u] = __ldg(x + col);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kBatch; u++) {
        const uint32_t w2 = d[u].z;
        const int type = (w2 >> 24) & 3;
        if (type == 3) continue;  // warp-uniform
        const int nnz = (int)((w2 >> 16) & 0xFF) + 1;
        const uint8_t *rec = page + ((w2 & 0xFFFFu) << 4);
        const uint8_t *body = AGG ? rec + ((d[u].w + 3u) & ~3u) * 4u : rec;
        V xv = xr[u];
        if constexpr (SCALED) xv *= scale;
        if (type == CBSPMV_FMT_COO) coo_path<V>(body, nnz, d[u].x, xv, y, lane);
        else if (type == CBSPMV_FMT_CSR) csr_path<V>(body, nnz, d[u].x, xv, y, lane);
        else dense_path<V>(body, d[u].x, xv, y, P.m, lane);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
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
  const int header = 2 * kMaxStages * (int)sizeof(uint64_t);
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
    const int smem = 2 * kMaxStages * (int)sizeof(uint64_t) + dev.nstage * dev.page_cap;
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
