// microbench.cu — measures the B200 costs the CB-SpMV kernel design depends on:
// scattered 8-byte loads (LDG / LDGSTS), and RED.ADD.F64 address patterns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// each thread: ITERS scattered loads of x[idx], idx random in [0, n)
template <int MODE>  // 0: LDG (ld.global), 1: LDG.nc no_allocate, 2: LDGSTS into smem
__global__ void k_gather(const double *__restrict__ x, uint32_t n, int iters, double *out, uint32_t span) {
  __shared__ double buf[1024];
  double acc = 0;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; i += 4) {
    uint32_t idx[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t base = hash(s * 131 + i + j) % n;
      // span: lanes of a warp spread over `span` consecutive elements (span=32*... => lines)
      idx[j] = span ? (hash((s >> 5) * 977 + i + j) % (n - span)) + (threadIdx.x & 31) * (span / 32) : base;
    }
    if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        uint32_t a = (uint32_t)__cvta_generic_to_shared(&buf[(threadIdx.x + j * 256) & 1023]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(x + idx[j]));
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      acc += buf[threadIdx.x & 1023];
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        double v;
        if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + idx[j]));
        else v = x[idx[j]];
        acc += v;
      }
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

// RED.ADD.F64: each warp instruction targets addresses by pattern
// pat 0: 32 distinct random addresses; 1: 16 consecutive rows (2 lanes each) in one 128 B line;
// 2: 32 lanes over 2 random lines (16 rows each); 3: all lanes same address;
// 4: ~10 distinct rows in one line (R-MAT-like COO block, 16 lanes active)
__global__ void k_red(double *y, uint32_t m, int iters, int pat) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < iters; i++) {
    uint32_t r = hash(w * 7919 + i);
    uint32_t base = (r % (m / 16 - 2)) * 16;
    uint32_t a;
    bool act = true;
    if (pat == 0) a = hash(r + lane) % m;
    else if (pat == 1) a = base + (lane >> 1);
    else if (pat == 2) a = (lane < 16 ? base : (hash(r ^ 0x55) % (m / 16 - 2)) * 16) + (lane & 15);
    else if (pat == 3) a = base;
    else { a = base + (hash(r + lane) % 10); act = lane < 16; }
    if (act) atomicAdd(y + a, 1.0);
  }
}

// TMA bulk copies: every thread issues `per` 16-byte cp.async.bulk copies from random 16-B aligned
// x pairs into shared memory, completion counted on one mbarrier per warp.
__global__ void k_bulk(const double *__restrict__ x, uint32_t n, int iters, double *out, int lanes) {
  __shared__ __align__(16) double buf[8][32 * 2 * 4];
  __shared__ __align__(8) uint64_t bar[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t bw = (uint32_t)__cvta_generic_to_shared(&bar[w]);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bw));
  __syncwarp();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0;
  uint32_t phase = 0;
  for (int i = 0; i < iters; i += 4) {
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bw), "r"(16 * 4 * lanes));
    __syncwarp();
    if (lane < lanes) {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        uint32_t idx = (hash(s * 131 + i + j) % (n / 2)) * 2;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[w][(lane * 4 + j) * 2]);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                     ::"r"(dst), "l"(x + idx), "r"(bw) : "memory");
      }
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(bw), "r"(phase) : "memory");
    phase ^= 1;
    acc += buf[w][lane * 2];
  }
  if (acc == 1.2345) out[0] = acc;
}

// RED over k lines: lane -> line (lane % k), row (lane / k) within the line
__global__ void k_red_lines(double *y, uint32_t m, int iters, int k) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < iters; i++) {
    uint32_t line = hash(w * 7919 + i * 31 + (lane % k)) % (m / 16 - 2);
    atomicAdd(y + line * 16 + (lane / k) % 16, 1.0);
  }
}
__global__ void k_red_lines_f32(float *y, uint32_t m, int iters, int k) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < iters; i++) {
    uint32_t line = hash(w * 7919 + i * 31 + (lane % k)) % (m / 16 - 2);
    atomicAdd(y + line * 16 + (lane / k) % 16, 1.0f);
  }
}

// RED with only `act` active lanes (rows consecutive in one line)
__global__ void k_red_act(double *y, uint32_t m, int iters, int act) {
  uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < iters; i++) {
    uint32_t line = hash(w * 7919 + i * 31) % (m / 16 - 2);
    if ((int)lane < act) atomicAdd(y + line * 16 + (lane & 15), 1.0);
  }
}
// shared-memory loads: LDS.64 consecutive (2 wavefronts) and LDS.U8 consecutive
__global__ void k_lds(double *out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x & 31;
  for (int i = 0; i < iters; i++) {
    acc += s[(idx + i * 32) & 2047];
    idx = (idx + (int)acc) & 31;
  }
  if (acc == 1.234) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const uint32_t n = 8u << 20;  // 64 MB of doubles (L2-resident, like R-MAT's x)
  double *x, *y, *out;
  CK(cudaMalloc(&x, (size_t)n * 8));
  CK(cudaMalloc(&y, (size_t)n * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, (size_t)n * 8));
  CK(cudaMemset(y, 0, (size_t)n * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8, iters = 256;
  const double warp_instr = (double)blocks * threads / 32 * iters;
  auto run = [&](const char *name, auto launch, double instr) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    double cyc = ms * 1e-3 * clk * 1e3;  // at max clock (kHz attr)
    printf("%-48s %8.3f ms  %7.2f Ginstr/s  %6.2f SM-cycles per warp-instr\n", name, ms, instr / ms / 1e6,
           cyc * sms / instr);
    return ms;
  };
  printf("SMs %d, clock %d MHz\n", sms, clk / 1000);
  for (uint32_t span : {0u, 32u * 16u, 32u * 4u, 32u}) {
    char nm[128];
    snprintf(nm, sizeof nm, "LDG scattered (span %u)", span);
    run(nm, [&] { k_gather<0><<<blocks, threads>>>(x, n, iters, out, span); }, warp_instr);
    snprintf(nm, sizeof nm, "LDG.nc.no_allocate scattered (span %u)", span);
    run(nm, [&] { k_gather<1><<<blocks, threads>>>(x, n, iters, out, span); }, warp_instr);
    snprintf(nm, sizeof nm, "LDGSTS scattered (span %u)", span);
    run(nm, [&] { k_gather<2><<<blocks, threads>>>(x, n, iters, out, span); }, warp_instr);
  }
  const char *pats[] = {"RED f64 32 random addrs", "RED f64 16 rows x2 lanes, 1 line", "RED f64 2 lines x16 rows",
                        "RED f64 same address", "RED f64 16 lanes, ~10 rows, 1 line"};
  for (int p = 0; p < 5; p++)
    run(pats[p], [&] { k_red<<<blocks, threads>>>(y, n, iters, p); }, warp_instr);
  for (int lanes : {1, 8, 32}) {
    char nm[128];
    snprintf(nm, sizeof nm, "bulk 16B random, %d lanes/warp (x4 per iter)", lanes);
    double instr = (double)blocks * threads / 32 * iters * lanes / 32.0;  // per 32 copies
    run(nm, [&] { k_bulk<<<blocks, threads>>>(x, n, iters, out, lanes); }, instr);
  }
  for (int k : {1, 2, 4, 8, 16, 32}) {
    char nm[128];
    snprintf(nm, sizeof nm, "RED f64 32 lanes over %d lines", k);
    run(nm, [&] { k_red_lines<<<blocks, threads>>>(y, n, iters, k); }, warp_instr);
    snprintf(nm, sizeof nm, "RED f32 32 lanes over %d lines", k);
    run(nm, [&] { k_red_lines_f32<<<blocks, threads>>>((float *)y, n, iters, k); }, warp_instr);
  }
  for (int act : {1, 4, 8, 16, 32}) {
    char nm[128];
    snprintf(nm, sizeof nm, "RED f64 %d active lanes, 1 line", act);
    run(nm, [&] { k_red_act<<<blocks, threads>>>(y, n, iters, act); }, warp_instr);
  }
  run("LDS.64 consecutive (dependent chain)", [&] { k_lds<<<blocks, threads>>>(out, iters); }, warp_instr);
  // is the RED cost per SM or chip-wide?  same work per warp on half / quarter of the SMs
  for (int frac : {2, 4}) {
    char nm[128];
    snprintf(nm, sizeof nm, "RED f64 16 lanes 1 line, grid/%d", frac);
    const int b = blocks / frac;
    double instr = (double)b * threads / 32 * iters;
    run(nm, [&] { k_red_act<<<b, threads>>>(y, n, iters, 16); }, instr);
  }
  // RED + scattered LDG in the same warp loop
  run("LDG scattered + RED f64 (1 line), per pair", [&] { k_gather<0><<<blocks, threads>>>(x, n, iters, out, 0);
      k_red_act<<<blocks, threads>>>(y, n, iters, 16); }, warp_instr);
  return 0;
}
