// gather4 microbenchmark: TMA tile::gather4 of random 16-byte rows of x (fp64 pairs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbg tools/mb_gather4.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// each issuing lane: per iteration 4 gather4 (16 rows of 16 B = 256 B) into its smem slot
__global__ void k_g4(const __grid_constant__ CUtensorMap tm, uint32_t rows, int iters, int lanes, double *out,
                     uint32_t check_row) {
  __shared__ __align__(128) double buf[4][32][2][16];  // per warp, per lane: 2 x 128-B aligned slots
  __shared__ __align__(8) uint64_t bar[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t bw = (uint32_t)__cvta_generic_to_shared(&bar[w]);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bw));
  __syncwarp();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x, phase = 0;
  double acc = 0;
  for (int i = 0; i < iters; i++) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bw), "r"(64 * 2 * lanes));
    __syncwarp();
    if (lane < lanes) {
#pragma unroll
      for (int j = 0; j < 2; j++) {
        int32_t r[4];
#pragma unroll
        for (int q = 0; q < 4; q++) r[q] = check_row ? (int32_t)(check_row + q) : (int32_t)(hash(s * 977 + i * 8 + j * 4 + q) % rows);
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[w][lane][j][0]);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(dst), "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bw) : "memory");
      }
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(bw), "r"(phase) : "memory");
    phase ^= 1;
    acc += buf[w][lane][0][lane & 7];
  }
  if (check_row && blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 8; k++) { out[k] = buf[0][0][0][k]; out[8 + k] = buf[0][0][1][k]; }
  }
  if (acc == 1.2345) out[100] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t n = 8u << 20, rows = n / 2;
  double *x, *out;
  cudaMalloc(&x, (size_t)n * 8); cudaMalloc(&out, 4096);
  double *h = (double *)malloc((size_t)n * 8);
  for (uint32_t i = 0; i < n; i++) h[i] = i;
  cudaMemcpy(x, h, (size_t)n * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {2, rows};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box{2,1}: %d\n", (int)r);
  // correctness: rows 100..103 then 104..107
  k_g4<<<1, 32>>>(tm, rows, 1, 1, out, 100);
  cudaError_t e = cudaDeviceSynchronize();
  printf("check: %s\n", cudaGetErrorString(e));
  double o[16]; cudaMemcpy(o, out, 128, cudaMemcpyDeviceToHost);
  for (int k = 0; k < 16; k++) printf("%g ", o[k]); printf("\n");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 128, blocks = sms * 16, iters = 64;
  for (int lanes : {1, 4, 8, 32}) {
    k_g4<<<blocks, threads>>>(tm, rows, iters, lanes, out, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int rr = 0; rr < 5; rr++) k_g4<<<blocks, threads>>>(tm, rows, iters, lanes, out, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double nrows = (double)blocks * (threads / 32) * lanes * iters * 8;
    printf("gather4 lanes=%2d: %.3f ms, %.2f Grows/s, %.2f SM-cycles per row (err %s)\n", lanes, ms, nrows / ms / 1e6,
           ms * 1e-3 * 1.965e9 * sms / nrows, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
