// Do LSU gathers (LDG, 8-byte scattered) and TMA tile::gather4 (32-byte rows) overlap on one SM?
// Warps [0, wl) gather with LDG, warps [wl, 16) with gather4; both over the same L2-resident x.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbm tools/mb_mixed.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ CUtensorMap tm, const double *__restrict__ x,
                                            uint32_t n, int iters, int wl, double *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rows = n / 4;
  double acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < wl) {
    for (int i = 0; i < iters; i++) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = __ldg(x + hash(s * 977 + i * 8 + j) % n);
#pragma unroll
      for (int j = 0; j < 8; j++) acc += v[j];
    }
  } else {
    uint32_t bw = (uint32_t)__cvta_generic_to_shared(&bar[w]);
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bw));
    __syncwarp();
    uint32_t phase = 0;
    uint8_t *mine = sm + (size_t)w * 32 * 256;  // 32 lanes x 2 x 128 B
    for (int i = 0; i < iters; i++) {
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bw), "r"(256 * 32));
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 2; j++) {
        uint32_t r[4];
#pragma unroll
        for (int q = 0; q < 4; q++) r[q] = hash(s * 977 + i * 8 + j * 4 + q) % rows;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(mine + lane * 256 + j * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(dst), "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bw) : "memory");
      }
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok) : "r"(bw), "r"(phase) : "memory");
      phase ^= 1;
      acc += *(const double *)(mine + lane * 256);
    }
  }
  if (acc == 1.2345) out[threadIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t n = 8u << 20;  // 64 MB x (L2-resident)
  double *x, *out;
  cudaMalloc(&x, (size_t)n * 8); cudaMalloc(&out, 4096 * 8);
  cudaMemset(x, 0, (size_t)n * 8);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, n / 4};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const int smem = 16 * 32 * 256;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 256;
  for (int wl : {16, 0, 8, 12, 4}) {
    k<<<sms, 512, smem>>>(tm, x, n, iters, wl, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int rr = 0; rr < 5; rr++) k<<<sms, 512, smem>>>(tm, x, n, iters, wl, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    const double rows_ldg = (double)sms * wl * 32 * iters * 8, rows_tma = (double)sms * (16 - wl) * 32 * iters * 8;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("LDG warps %2d / gather4 warps %2d: %.3f ms  LDG rows/SM-cycle %.3f  TMA rows/SM-cycle %.3f  total %.3f (%s)\n",
           wl, 16 - wl, ms, rows_ldg / sms / cyc, rows_tma / sms / cyc, (rows_ldg + rows_tma) / sms / cyc,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
