// gather4 destination-alignment probe: TMA tile::gather4 of 16-byte rows (fp64 pairs) into shared
// memory at offsets 16/32/64/128 B; prints whether the rows land intact.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbga tools/mb_gather4_align.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k(const __grid_constant__ CUtensorMap tm, int off, double *out) {
  __shared__ __align__(1024) double buf[64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t bw = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = 0; i < 64; i++) buf[i] = -1;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bw));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bw), "r"(64));
  uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf) + off;
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(&tm), "r"(0), "r"(5), "r"(17), "r"(3), "r"(1000), "r"(bw) : "memory");
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(ok) : "r"(bw), "r"(0) : "memory");
  for (int i = 0; i < 64; i++) out[i] = buf[i];
}

int main() {
  const uint32_t n = 1 << 16;
  double *x, *out;
  cudaMalloc(&x, (size_t)n * 8); cudaMalloc(&out, 64 * 8);
  double *h = (double *)malloc((size_t)n * 8);
  for (uint32_t i = 0; i < n; i++) h[i] = i;
  cudaMemcpy(x, h, (size_t)n * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {2, n / 2};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  for (int off : {128, 64, 32, 16}) {
    k<<<1, 1>>>(tm, off, out);
    cudaError_t e = cudaDeviceSynchronize();
    double o[64];
    cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
    const int b = off / 8;
    const bool good = o[b] == 10 && o[b + 1] == 11 && o[b + 2] == 34 && o[b + 3] == 35 && o[b + 4] == 6 &&
                      o[b + 5] == 7 && o[b + 6] == 2000 && o[b + 7] == 2001;
    printf("dst offset %3d B: %s  (%s) got %g %g %g %g %g %g %g %g\n", off, good ? "OK" : "WRONG", cudaGetErrorString(e),
           o[b], o[b + 1], o[b + 2], o[b + 3], o[b + 4], o[b + 5], o[b + 6], o[b + 7]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
