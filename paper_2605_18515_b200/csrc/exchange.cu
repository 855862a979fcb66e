// exchange.cu — fused finalize + y exchange of the iterated SpMV over peer memory
// (BASELINE configs[4]: power iteration, rows sharded across the
// GPUs of one node, x replicated).
//
// Per step k every rank r computes its rows of y_k = A_r (x_k / ||y_{k-1}||) straight into its
// own slice of the next iterate buffer X[(k+1) & 1] (cbspmv_spmv_scaled), then ONE kernel
// (cbspmv_xchg_publish) passes over that slice once and
//   * stores it into the same slice of every peer's X[(k+1) & 1] (NVLink P2P stores, or the
//     same device when all "ranks" share one GPU in the tests),
//   * reduces sum(y^2) of the slice (fixed-order block sums, deterministic),
//   * and, after a system-scope fence, has its last CTA write the partial into every peer's
//     partials[k & 1][r] and release flags[r] = k + 1 on every peer.
// cbspmv_xchg_wait(k + 1) spins (acquire, bounded) until every flag reaches k + 1 and sums the
// partials in rank order into the sumsq the next step's SpMV scales by — the same bits on every
// rank.  This replaces cbspmv_sumsq + the NCCL all-reduce + all-gather of
// dist.power_iteration_device with one kernel and a flag wait; there is no host round trip.
//
// Safety of the double buffers: a peer can publish step k + 2 into this rank's
// X[(k+1) & 1] only after waiting for this rank's flag k + 2, which this rank releases only after
// its SpMV of step k + 1 (the last reader of that buffer) has finished on its stream; the same
// argument covers partials[k & 1].
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "cb_internal.h"
#include "cbspmv.h"

namespace {

constexpr int kMaxWorld = 8;  // one NVSwitch node
constexpr int kPubThreads = 256;
constexpr int kAlign = 256;

inline int64_t up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// One rank's allocation (one cudaMalloc, exported whole through IPC):
//   [flags u64 x kMaxWorld][partials f64 x 2 x kMaxWorld][counter u32 + pad][cta partials f64 x grid]
//   [X0: n values][X1: n values]
struct Layout {
  int64_t flags = 0, partials, counter, cta, x0, x1, total;
  Layout(int64_t n, int vb, int grid) {
    partials = up(flags + 8 * kMaxWorld, kAlign);
    counter = up(partials + 8 * 2 * kMaxWorld, kAlign);
    cta = up(counter + 8, kAlign);
    x0 = up(cta + 8 * (int64_t)grid, kAlign);
    x1 = up(x0 + (int64_t)vb * n, kAlign);
    total = up(x1 + (int64_t)vb * n, kAlign);
  }
};

struct PubArgs {
  uint8_t *peer[kMaxWorld];  // base of every rank's allocation (peer[rank] = own)
  int world, rank;
};

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// y: this rank's slice [r0, r0 + len) of its own X[b]; stores it into every peer's X[b] at r0.
// err: the context's timeout flag.  Once a wait has timed out the exchange is poisoned: publish
// stores nothing into the peers (a slow peer may still be reading those buffers) and releases no
// flag, so every later wait times out too, and the caller's status check raises.
template <typename V>
__global__ void __launch_bounds__(kPubThreads) xchg_publish_kernel(PubArgs A, int64_t xoff_b, int64_t r0,
                                                                   int64_t len, Layout L, uint64_t seq,
                                                                   const int *err) {
  if (*(const volatile int *)err) return;
  uint8_t *own = A.peer[A.rank];
  const V *y = reinterpret_cast<const V *>(own + xoff_b) + r0;
  double acc = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  // 16-byte loads and peer stores (fewer, larger NVLink writes) when the slice is 16-byte aligned
  // (row shards start at block-row boundaries); the tail and unaligned slices element by element
  constexpr int kPer = 16 / (int)sizeof(V);
  const bool vec = ((uintptr_t)y % 16) == 0 && ((uintptr_t)(xoff_b + r0 * (int64_t)sizeof(V)) % 16) == 0;
  const int64_t nvec = vec ? len / kPer : 0;
  for (int64_t i = tid; i < nvec; i += nth) {
    const uint4 u = reinterpret_cast<const uint4 *>(y)[i];
    V v[kPer];
    memcpy(v, &u, 16);
#pragma unroll
    for (int j = 0; j < kPer; j++) acc = fma((double)v[j], (double)v[j], acc);
#pragma unroll
    for (int q = 0; q < kMaxWorld; q++)
      if (q < A.world && q != A.rank) reinterpret_cast<uint4 *>(A.peer[q] + xoff_b + r0 * (int64_t)sizeof(V))[i] = u;
  }
  for (int64_t i = nvec * kPer + tid; i < len; i += nth) {
    const V v = y[i];
    acc = fma((double)v, (double)v, acc);
#pragma unroll
    for (int q = 0; q < kMaxWorld; q++)
      if (q < A.world && q != A.rank) reinterpret_cast<V *>(A.peer[q] + xoff_b)[r0 + i] = v;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  __shared__ double part[kPubThreads / 32];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kPubThreads / 32; w++) s += part[w];
    reinterpret_cast<double *>(own + L.cta)[blockIdx.x] = s;
    __threadfence_system();  // this CTA's peer stores and its partial before the count
    unsigned *cnt = reinterpret_cast<unsigned *>(own + L.counter);
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  // the last CTA: every CTA's stores are fenced; sum the CTA partials in index order
  __threadfence();
  double tot = 0.0;
  const volatile double *cp = reinterpret_cast<const volatile double *>(own + L.cta);
  for (unsigned b = 0; b < gridDim.x; b++) tot += cp[b];
  *reinterpret_cast<unsigned *>(own + L.counter) = 0u;  // reset for the next step (stream-ordered)
  const int par = (int)((seq - 1) & 1);
  for (int q = 0; q < A.world; q++)
    reinterpret_cast<double *>(A.peer[q] + L.partials)[par * kMaxWorld + A.rank] = tot;
  __threadfence_system();
  for (int q = 0; q < A.world; q++) st_release_sys(reinterpret_cast<uint64_t *>(A.peer[q] + L.flags) + A.rank, seq);
}

// Wait until flags[q] >= seq for every rank, then sumsq = sum_q partials[(seq - 1) & 1][q] in
// rank order.  Bounded: after ~timeout_ns (or when an earlier wait already timed out) *err = 1 and
// sumsq = NaN, so the next SpMV's scale s = 1/sqrt(NaN) turns the iterate into NaN instead of
// silently continuing from a partly published one.
__global__ void xchg_wait_kernel(uint8_t *own, Layout L, int world, uint64_t seq, double *sumsq, int *err,
                                 uint64_t timeout_ns) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = *(volatile int *)err;
  __syncthreads();
  if (!bad && (int)threadIdx.x < world) {
    const uint64_t *f = reinterpret_cast<const uint64_t *>(own + L.flags) + threadIdx.x;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(f) < seq) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) { atomicExch(&bad, 1); break; }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (bad) {
    *err = 1;
    *sumsq = __longlong_as_double(0x7ff8000000000000ll);  // NaN poisons the next step
    return;
  }
  const int par = (int)((seq - 1) & 1);
  const volatile double *p = reinterpret_cast<const volatile double *>(own + L.partials) + par * kMaxWorld;
  double s = 0.0;
  for (int q = 0; q < world; q++) s += p[q];
  *sumsq = s;
}

int pub_grid(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? 4 * sms : 4;  // 4 CTAs of 256 threads per SM: enough loads in flight to stream y
}

}  // namespace

struct cbspmv_xchg_s {
  int device = -1, dtype = 0, vb = 8, world = 1, rank = 0, grid = 1;
  int64_t n = 0;
  uint8_t *base = nullptr;          // own allocation
  uint8_t *peer[kMaxWorld] = {};    // every rank's base as seen from this process
  bool opened[kMaxWorld] = {};      // peer[q] came from cudaIpcOpenMemHandle
  int *d_err = nullptr;
  Layout L{0, 8, 1};
};

namespace {
struct Guard {
  int prev = -1, want;
  explicit Guard(int d) : want(d) {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != want) cudaSetDevice(want);
  }
  ~Guard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};
cbspmv_status_t cuda_err(cudaError_t e, const char *what) {
  return (cbspmv_status_t)cb_set_error(CBSPMV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

cbspmv_status_t cbspmv_xchg_create(int64_t n, cbspmv_dtype_t dtype, int32_t world, int32_t rank, int32_t device,
                                   cbspmv_xchg_t *out) {
  if (!out) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "null output");
  *out = nullptr;
  if (n < 0 || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || device < 0)
    return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "bad exchange arguments (1 <= world <= 8, 0 <= rank < world)");
  if (dtype != CBSPMV_F64 && dtype != CBSPMV_F32 && dtype != CBSPMV_F32F64)
    return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "bad dtype");
  Guard g(device);
  auto *x = new (std::nothrow) cbspmv_xchg_s;
  if (!x) return (cbspmv_status_t)cb_set_error(CBSPMV_ENOMEM, "host allocation");
  x->device = device; x->dtype = dtype; x->vb = dtype == CBSPMV_F32 ? 4 : 8;
  x->world = world; x->rank = rank; x->n = n; x->grid = pub_grid(device);
  x->L = Layout(n, x->vb, x->grid);
  cudaError_t e = cudaMalloc(&x->base, (size_t)x->L.total);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(x->base, 0, (size_t)x->L.x0);  // flags, partials, counter
  if (e == cudaSuccess) e = cudaMemset(x->d_err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(x->base); cudaFree(x->d_err); delete x;
    cudaGetLastError();
    return (cbspmv_status_t)cb_set_error(CBSPMV_ENOMEM, std::string("exchange allocation: ") + cudaGetErrorString(e));
  }
  x->peer[rank] = x->base;
  *out = x;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_xchg_ipc_handle(cbspmv_xchg_t x, void *handle_out) {
  if (!x || !handle_out) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "null argument");
  Guard g(x->device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, x->base);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == CBSPMV_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof h);
  return CBSPMV_OK;
}

void *cbspmv_xchg_base(cbspmv_xchg_t x) { return x ? x->base : nullptr; }

cbspmv_status_t cbspmv_xchg_connect(cbspmv_xchg_t x, void *const *peer_bases, const void *ipc_handles) {
  if (!x || (!peer_bases && !ipc_handles)) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "null argument");
  Guard g(x->device);
  for (int q = 0; q < x->world; q++) {
    if (q == x->rank || x->peer[q]) continue;
    if (peer_bases && peer_bases[q]) {
      x->peer[q] = static_cast<uint8_t *>(peer_bases[q]);
      continue;
    }
    if (!ipc_handles) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "no base or IPC handle for a peer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t *>(ipc_handles) + (size_t)q * CBSPMV_IPC_HANDLE_BYTES, sizeof h);
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_err(e, "cudaIpcOpenMemHandle");
    x->peer[q] = static_cast<uint8_t *>(p);
    x->opened[q] = true;
  }
  return CBSPMV_OK;
}

void *cbspmv_xchg_buffer(cbspmv_xchg_t x, int32_t b) {
  if (!x || (b != 0 && b != 1)) return nullptr;
  return x->base + (b ? x->L.x1 : x->L.x0);
}

cbspmv_status_t cbspmv_xchg_publish(cbspmv_xchg_t x, int32_t b, int64_t r0, int64_t len, uint64_t seq, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_xchg_publish");
  if (!x || (b != 0 && b != 1) || r0 < 0 || len < 0 || r0 + len > x->n || seq == 0)
    return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "bad publish arguments");
  for (int q = 0; q < x->world; q++)
    if (!x->peer[q]) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "exchange not connected");
  Guard g(x->device);
  PubArgs A{};
  for (int q = 0; q < x->world; q++) A.peer[q] = x->peer[q];
  A.world = x->world; A.rank = x->rank;
  const int64_t need = (len + kPubThreads - 1) / kPubThreads;
  const int grid = (int)(need < 1 ? 1 : (need < x->grid ? need : x->grid));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t xoff = b ? x->L.x1 : x->L.x0;
  if (x->vb == 8) xchg_publish_kernel<double><<<grid, kPubThreads, 0, st>>>(A, xoff, r0, len, x->L, seq, x->d_err);
  else xchg_publish_kernel<float><<<grid, kPubThreads, 0, st>>>(A, xoff, r0, len, x->L, seq, x->d_err);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "publish launch");
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_xchg_wait(cbspmv_xchg_t x, uint64_t seq, double *sumsq_dev, double timeout_s, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_xchg_wait");
  if (!x || !sumsq_dev || seq == 0) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "bad wait arguments");
  Guard g(x->device);
  const double t = timeout_s > 0 ? timeout_s : 10.0;
  xchg_wait_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x->base, x->L, x->world, seq, sumsq_dev,
                                                                          x->d_err, (uint64_t)(t * 1e9));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "wait launch");
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_xchg_status(cbspmv_xchg_t x, int32_t *timed_out) {
  if (!x || !timed_out) return (cbspmv_status_t)cb_set_error(CBSPMV_EINVAL, "null argument");
  Guard g(x->device);
  int v = 0;
  cudaError_t e = cudaMemcpy(&v, x->d_err, sizeof v, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_err(e, "status copy");
  *timed_out = v;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_xchg_destroy(cbspmv_xchg_t x) {
  if (!x) return CBSPMV_OK;
  Guard g(x->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < kMaxWorld; q++)
    if (x->opened[q]) cudaIpcCloseMemHandle(x->peer[q]);
  cudaFree(x->base);
  cudaFree(x->d_err);
  cudaGetLastError();
  delete x;
  return CBSPMV_OK;
}

}  // extern "C"
