// gpu_builder.cu — steps a2..a6 of the CB-SpMV format build on the GPU (SURVEY §8(f) NEXT-3:
// "CUB radix sort by block key, per-block-row distinct/rank for aggregation, prefix-sum VPs,
// parallel pack; Alg. 2 stays on the host").
//
// The output is the canonical format of build_canonical (builder.cpp), byte for byte (checked
// against the oracle by tests/test_gpu_builder.py):
//   a1  canonical check + nnz count: on the host (check_csr, one parallel pass), so every error
//       status and message is the host builder's; explicit zeros are dropped here (flag select).
//   a2  partition: element key (br, bc, lr, lc) = (r>>4, c>>4, r&15, c&15) packed in a u64,
//       radix-sorted, so blocks come out in (br, bc) order and elements in (lr, lc) order.
//   a3  block statistics: run-length encoding of the block ids -> nb_pre, ss_count; the th0
//       decision on the host (decide_agg, exact rational compare).
//   a4  column aggregation: radix sort by (br, c); distinct flags + inclusive scan give each
//       element the global index of its column in the concatenated C_i; restore_cols is the
//       compacted distinct columns, cols_offset[b] = lower_bound(block row of each distinct
//       column, b); rank = index - cols_offset[br]; re-key (br, rank>>4, lr, rank&15), sort again.
//   a5  format per block from its run length (select_format).
//   a6  record sizes (R-8) -> exclusive scan = VP; one warp per block packs its record into the
//       zeroed mtx buffer (COO coordinate bytes (col<<4)|row + values; CSR 17 u8 row_ptr + u8
//       cols + values; DENSE 256 values row-major); values are copied as raw size(Val) bytes.
//   a7  Alg. 2 + permute: on the host (balance_and_permute) over the downloaded per-block arrays.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "cb_internal.h"

namespace cb {
namespace {

constexpr int kBlk = 16;

// RAII device buffer
struct DBuf {
  void *p = nullptr;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
  }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Ctx {
  cudaStream_t st;
  std::string *err;
  int status = CBSPMV_OK;
  bool ok(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return true;
    cudaGetLastError();
    if (status == CBSPMV_OK) {
      status = e == cudaErrorMemoryAllocation ? CBSPMV_ENOMEM : CBSPMV_ECUDA;
      *err = std::string("device build, ") + what + ": " + cudaGetErrorString(e);
    }
    return false;
  }
  bool alloc(DBuf &b, size_t bytes, const char *what) { return ok(cudaMalloc(&b.p, bytes ? bytes : 16), what); }
};

inline int grid_for(int64_t n, int per_block) {
  int64_t g = (n + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

inline int bits_for(uint64_t v) {  // bits needed to hold values < v + 1
  int b = 0;
  while (b < 64 && (v >> b) != 0) b++;
  return b;
}

// ------------------------------------------------------------------ kernels
__global__ void k_rowid(const int64_t *__restrict__ rp, int64_t m, uint32_t *__restrict__ rowid) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t r = w0; r < m; r += nw)
    for (int64_t j = rp[r] + lane; j < rp[r + 1]; j += 32) rowid[j] = (uint32_t)r;
}

template <typename V>
__global__ void k_nonzero(const V *__restrict__ vals, int64_t nnz, uint8_t *__restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = vals[j] != V(0);  // explicit zeros (incl. -0.0) are dropped (R-19)
}

// a2: (br, bc, lr, lc) key of a kept element
__global__ void k_key_plain(const uint32_t *__restrict__ kidx, int64_t nk, const uint32_t *__restrict__ rowid,
                            const int32_t *__restrict__ col, uint64_t *__restrict__ key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = kidx[i], r = rowid[j], c = (uint32_t)col[j];
    key[i] = ((uint64_t)(r >> 4) << 36) | ((uint64_t)(c >> 4) << 8) | ((r & 15u) << 4) | (c & 15u);
  }
}

// a4: (br, column) key
__global__ void k_key_rowcol(const uint32_t *__restrict__ kidx, int64_t nk, const uint32_t *__restrict__ rowid,
                             const int32_t *__restrict__ col, uint64_t *__restrict__ key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = kidx[i];
    key[i] = ((uint64_t)(rowid[j] >> 4) << 32) | (uint32_t)col[j];
  }
}

__global__ void k_distinct(const uint64_t *__restrict__ key, int64_t nk, uint32_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

// restore_cols = the distinct columns in (br, c) order = concat(C_i); their block rows
__global__ void k_restore(const uint64_t *__restrict__ key, const uint32_t *__restrict__ flag,
                          const uint32_t *__restrict__ g, int64_t nk, uint32_t *__restrict__ restore,
                          uint32_t *__restrict__ dist_br) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      const uint32_t d = g[i] - 1u;
      restore[d] = (uint32_t)(key[i] & 0xFFFFFFFFu);
      dist_br[d] = (uint32_t)(key[i] >> 32);
    }
}

// cols_offset[b] = #distinct columns of block rows < b (R-7)
__global__ void k_cols_offset(const uint32_t *__restrict__ dist_br, int64_t ndist, int64_t blk_m,
                              uint64_t *__restrict__ cols_offset) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= blk_m; b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = ndist;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)dist_br[mid] < b) lo = mid + 1;
      else hi = mid;
    }
    cols_offset[b] = (uint64_t)lo;
  }
}

// a4 re-key: (br, rank>>4, lr, rank&15)
__global__ void k_key_agg(const uint64_t *__restrict__ key2, const uint32_t *__restrict__ idx2,
                          const uint32_t *__restrict__ g, int64_t nk, const uint32_t *__restrict__ rowid,
                          const uint64_t *__restrict__ cols_offset, uint64_t *__restrict__ key3) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t br = key2[i] >> 32;
    const uint64_t rank = (uint64_t)(g[i] - 1u) - cols_offset[br];
    const uint32_t lr = rowid[idx2[i]] & 15u;
    key3[i] = (br << 36) | ((rank >> 4) << 8) | ((uint64_t)lr << 4) | (rank & 15u);
  }
}

__global__ void k_block_id(const uint64_t *__restrict__ key, int64_t nk, uint64_t *__restrict__ bid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x)
    bid[i] = key[i] >> 8;
}

__global__ void k_count_small(const uint32_t *__restrict__ cnt, int64_t nb, int limit,
                              unsigned long long *__restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    acc += cnt[b] < (uint32_t)limit;
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

struct FmtParams {
  int th1, th2, force;
  int S;
};

__device__ __forceinline__ int d_select(int k, const FmtParams &f) {  // P:439 (R-9)
  if (f.force >= 0) return f.force;
  if (k < f.th1) return CBSPMV_FMT_COO;
  if (k > f.th2) return CBSPMV_FMT_DENSE;
  return CBSPMV_FMT_CSR;
}
__device__ __forceinline__ int64_t d_pad(int64_t idx, int S) {  // Alg. 3 lines 6-7
  const int64_t p = idx % S;
  return p ? S - p : 0;
}
__device__ __forceinline__ int64_t d_rec_bytes(int type, int64_t k, int S) {  // a6 (R-8)
  const int64_t idx = type == CBSPMV_FMT_COO ? k : type == CBSPMV_FMT_CSR ? kBlk + 1 + k : 0;
  const int64_t nval = type == CBSPMV_FMT_DENSE ? kBlk * kBlk : k;
  return idx + d_pad(idx, S) + nval * S;
}

// a5 + record sizes; natural-order block arrays
__global__ void k_block_meta(const uint64_t *__restrict__ ubid, const uint32_t *__restrict__ cnt, int64_t nb,
                             FmtParams f, int32_t *__restrict__ br, int32_t *__restrict__ bc,
                             int32_t *__restrict__ nnz, uint8_t *__restrict__ type, uint64_t *__restrict__ rbytes) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)cnt[b];
    const int t = d_select(k, f);
    br[b] = (int32_t)(ubid[b] >> 28);
    bc[b] = (int32_t)(ubid[b] & ((1ull << 28) - 1));
    nnz[b] = k;
    type[b] = (uint8_t)t;
    rbytes[b] = (uint64_t)d_rec_bytes(t, k, f.S);
  }
}

template <int S>
__device__ __forceinline__ void copy_val(uint8_t *dst, const uint8_t *src) {
  if constexpr (S == 8) *reinterpret_cast<uint64_t *>(dst) = *reinterpret_cast<const uint64_t *>(src);
  else *reinterpret_cast<uint32_t *>(dst) = *reinterpret_cast<const uint32_t *>(src);
}

// a6: one warp per block writes its record at mtx + vp (mtx zeroed beforehand: padding = 0)
template <int S>
__global__ void k_pack(const uint64_t *__restrict__ key, const uint32_t *__restrict__ idx,
                       const uint32_t *__restrict__ estart, const int32_t *__restrict__ nnz,
                       const uint8_t *__restrict__ type, const uint64_t *__restrict__ vp, int64_t nb,
                       const uint8_t *__restrict__ vals, uint8_t *__restrict__ mtx) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = w0; b < nb; b += nw) {
    const int k = nnz[b], t = type[b];
    const uint32_t e0 = estart[b];
    uint8_t *dst = mtx + vp[b];
    if (t == CBSPMV_FMT_COO) {
      uint8_t *v = dst + k + d_pad(k, S);
      for (int q = lane; q < k; q += 32) {
        const uint64_t kk = key[e0 + q];
        const uint32_t lr = (kk >> 4) & 15u, lc = kk & 15u;
        dst[q] = (uint8_t)((lc << 4) | lr);  // row = b & 15, col = b >> 4
        copy_val<S>(v + (int64_t)q * S, vals + (int64_t)idx[e0 + q] * S);
      }
    } else if (t == CBSPMV_FMT_CSR) {
      if (lane <= kBlk) {  // row_ptr[r] = #elements in rows < r; row_ptr[16] = nnz mod 256 (R-8)
        int c = 0;
        for (int q = 0; q < k; q++) c += (int)((key[e0 + q] >> 4) & 15u) < lane;
        dst[lane] = (uint8_t)(c & 0xFF);
      }
      uint8_t *v = dst + (kBlk + 1) + k + d_pad(kBlk + 1 + k, S);
      for (int q = lane; q < k; q += 32) {
        dst[kBlk + 1 + q] = (uint8_t)(key[e0 + q] & 15u);
        copy_val<S>(v + (int64_t)q * S, vals + (int64_t)idx[e0 + q] * S);
      }
    } else {
      for (int q = lane; q < k; q += 32) {
        const uint64_t kk = key[e0 + q];
        const int pos = (int)((kk >> 4) & 15u) * kBlk + (int)(kk & 15u);
        copy_val<S>(dst + (int64_t)pos * S, vals + (int64_t)idx[e0 + q] * S);
      }
    }
  }
}

// ------------------------------------------------------------------ CUB wrappers (temp storage per call)
template <class F>
bool cub_call(Ctx &x, const char *what, F f) {
  size_t bytes = 0;
  if (!x.ok(f(nullptr, bytes), what)) return false;
  DBuf tmp;
  if (!x.alloc(tmp, bytes, what)) return false;
  return x.ok(f(tmp.p, bytes), what);
}

}  // namespace

int build_canonical_device(const Csr &A, const cbspmv_options_t &o, void *stream, Canon *out, DevCanon *dc,
                           bool download_records, std::string *err) {
  PhaseTimer tm;
  int64_t nnz_kept = 0;
  int st = check_csr(A, o, &nnz_kept, err);  // a1 (host): statuses identical to the host builder
  if (st != CBSPMV_OK) return st;
  tm.lap("dev a1 canonical check (host)");
  if (o.blk != kBlk) { *err = "device build requires blk = 16"; return CBSPMV_EUNSUPPORTED; }
  if (A.nnz >= (int64_t)INT32_MAX || A.m >= (int64_t)UINT32_MAX) {
    *err = "device build handles fewer than 2^31 stored entries per panel";
    return CBSPMV_EUNSUPPORTED;
  }
  Ctx x{reinterpret_cast<cudaStream_t>(stream), err};
  const int S = (int)A.val_size;
  const int64_t m = A.m, nnz = A.nnz, blk_m = (m + kBlk - 1) / kBlk;
  Canon &c = *out;
  c = Canon();
  c.m = m; c.n = A.n; c.blk = kBlk; c.val_size = S; c.W = o.warps_per_tb; c.blk_m = blk_m; c.nnz = nnz_kept;

  // upload the CSR
  DBuf d_rp, d_col, d_val, d_rowid, d_flag, d_kidx, d_nsel;
  if (!x.alloc(d_rp, 8 * (size_t)(m + 1), "alloc") || !x.alloc(d_col, 4 * (size_t)nnz, "alloc") ||
      !x.alloc(d_val, (size_t)S * nnz, "alloc") || !x.alloc(d_rowid, 4 * (size_t)nnz, "alloc") ||
      !x.alloc(d_flag, (size_t)nnz, "alloc") || !x.alloc(d_kidx, 4 * (size_t)nnz, "alloc") ||
      !x.alloc(d_nsel, 8, "alloc"))
    return x.status;
  if (!x.ok(cudaMemcpyAsync(d_rp.p, A.row_ptr, 8 * (size_t)(m + 1), cudaMemcpyHostToDevice, x.st), "upload") ||
      !x.ok(cudaMemcpyAsync(d_col.p, A.col, 4 * (size_t)nnz, cudaMemcpyHostToDevice, x.st), "upload") ||
      !x.ok(cudaMemcpyAsync(d_val.p, A.val, (size_t)S * nnz, cudaMemcpyHostToDevice, x.st), "upload"))
    return x.status;
  const int TPB = 256;
  if (m > 0) k_rowid<<<grid_for(m * 32, TPB), TPB, 0, x.st>>>(d_rp.as<int64_t>(), m, d_rowid.as<uint32_t>());
  if (nnz > 0) {
    if (S == 8) k_nonzero<double><<<grid_for(nnz, TPB), TPB, 0, x.st>>>(d_val.as<double>(), nnz, d_flag.as<uint8_t>());
    else k_nonzero<float><<<grid_for(nnz, TPB), TPB, 0, x.st>>>(d_val.as<float>(), nnz, d_flag.as<uint8_t>());
    cub::CountingInputIterator<uint32_t> it(0);
    if (!cub_call(x, "select", [&](void *t, size_t &b) {
          return cub::DeviceSelect::Flagged(t, b, it, d_flag.as<uint8_t>(), d_kidx.as<uint32_t>(),
                                            d_nsel.as<int64_t>(), nnz, x.st);
        }))
      return x.status;
  }
  d_flag.release();
  const int64_t nk = nnz_kept;  // = the select count (a1 counted the non-zeros)
  tm.lap("dev upload + zero drop");

  // a2 + a3: sort by (br, bc, lr, lc), run-length encode the block ids
  const int br_bits = bits_for((uint64_t)std::max<int64_t>(blk_m, 1));
  DBuf d_key, d_key_s, d_idx_s, d_bid, d_ubid, d_cnt, d_nruns, d_ss;
  auto sort_pairs = [&](DBuf &kin, DBuf &vin, int end_bit, const char *what) {
    return cub_call(x, what, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, kin.as<uint64_t>(), d_key_s.as<uint64_t>(), vin.as<uint32_t>(),
                                             d_idx_s.as<uint32_t>(), nk, 0, end_bit, x.st);
    });
  };
  auto rle = [&](int64_t *nruns) {
    k_block_id<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), nk, d_bid.as<uint64_t>());
    if (!cub_call(x, "run-length encode", [&](void *t, size_t &b) {
          return cub::DeviceRunLengthEncode::Encode(t, b, d_bid.as<uint64_t>(), d_ubid.as<uint64_t>(),
                                                    d_cnt.as<uint32_t>(), d_nruns.as<int64_t>(), nk, x.st);
        }))
      return false;
    return x.ok(cudaMemcpyAsync(nruns, d_nruns.p, 8, cudaMemcpyDeviceToHost, x.st), "download") &&
           x.ok(cudaStreamSynchronize(x.st), "sync");
  };
  int64_t nb = 0;
  if (nk > 0) {
    if (!x.alloc(d_key, 8 * (size_t)nk, "alloc") || !x.alloc(d_key_s, 8 * (size_t)nk, "alloc") ||
        !x.alloc(d_idx_s, 4 * (size_t)nk, "alloc") || !x.alloc(d_bid, 8 * (size_t)nk, "alloc") ||
        !x.alloc(d_ubid, 8 * (size_t)nk, "alloc") || !x.alloc(d_cnt, 4 * (size_t)nk, "alloc") ||
        !x.alloc(d_nruns, 8, "alloc") || !x.alloc(d_ss, 8, "alloc"))
      return x.status;
    k_key_plain<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_kidx.as<uint32_t>(), nk, d_rowid.as<uint32_t>(),
                                                     d_col.as<int32_t>(), d_key.as<uint64_t>());
    if (!sort_pairs(d_key, d_kidx, 36 + br_bits, "sort (br, bc, lr, lc)")) return x.status;
    if (!rle(&nb)) return x.status;
    unsigned long long ss = 0;
    if (!x.ok(cudaMemsetAsync(d_ss.p, 0, 8, x.st), "memset")) return x.status;
    k_count_small<<<grid_for(nb, TPB), TPB, 0, x.st>>>(d_cnt.as<uint32_t>(), nb, o.ss_limit,
                                                       d_ss.as<unsigned long long>());
    if (!x.ok(cudaMemcpyAsync(&ss, d_ss.p, 8, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaStreamSynchronize(x.st), "sync"))
      return x.status;
    c.nb_pre = nb;
    c.ss_count = (int64_t)ss;
  }
  c.agg = o.agg_mode >= 0 ? o.agg_mode : decide_agg(c.nb_pre, c.ss_count, o);  // a3 (R-3, R-5)
  tm.lap("dev a2+a3 sort, block stats");

  // a4: column aggregation
  if (c.agg) {
    c.cols_offset.assign((size_t)blk_m + 1, 0);
    if (nk > 0) {
      DBuf d_flag2, d_g, d_restore, d_dbr, d_coff;
      if (!x.alloc(d_flag2, 4 * (size_t)nk, "alloc") || !x.alloc(d_g, 4 * (size_t)nk, "alloc") ||
          !x.alloc(d_coff, 8 * (size_t)(blk_m + 1), "alloc"))
        return x.status;
      // (br, c) order; d_kidx still holds the kept element indices (SortPairs is out of place)
      k_key_rowcol<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_kidx.as<uint32_t>(), nk, d_rowid.as<uint32_t>(),
                                                        d_col.as<int32_t>(), d_key.as<uint64_t>());
      if (!sort_pairs(d_key, d_kidx, 32 + br_bits, "sort (br, c)")) return x.status;
      k_distinct<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), nk, d_flag2.as<uint32_t>());
      if (!cub_call(x, "scan", [&](void *t, size_t &b) {
            return cub::DeviceScan::InclusiveSum(t, b, d_flag2.as<uint32_t>(), d_g.as<uint32_t>(), nk, x.st);
          }))
        return x.status;
      uint32_t ndist = 0;
      if (!x.ok(cudaMemcpyAsync(&ndist, d_g.as<uint32_t>() + (nk - 1), 4, cudaMemcpyDeviceToHost, x.st), "download") ||
          !x.ok(cudaStreamSynchronize(x.st), "sync"))
        return x.status;
      if (!x.alloc(d_restore, 4 * (size_t)ndist, "alloc") || !x.alloc(d_dbr, 4 * (size_t)ndist, "alloc"))
        return x.status;
      k_restore<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), d_flag2.as<uint32_t>(), d_g.as<uint32_t>(),
                                                     nk, d_restore.as<uint32_t>(), d_dbr.as<uint32_t>());
      k_cols_offset<<<grid_for(blk_m + 1, TPB), TPB, 0, x.st>>>(d_dbr.as<uint32_t>(), ndist, blk_m,
                                                                d_coff.as<uint64_t>());
      // re-key by (br, rank>>4, lr, rank&15) from the (br, c)-sorted order, then sort again
      k_key_agg<<<grid_for(nk, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), d_idx_s.as<uint32_t>(), d_g.as<uint32_t>(),
                                                     nk, d_rowid.as<uint32_t>(), d_coff.as<uint64_t>(),
                                                     d_key.as<uint64_t>());
      if (!x.ok(cudaMemcpyAsync(d_kidx.p, d_idx_s.p, 4 * (size_t)nk, cudaMemcpyDeviceToDevice, x.st), "copy"))
        return x.status;
      if (!sort_pairs(d_key, d_kidx, 36 + br_bits, "sort (br, bc', lr, lc')")) return x.status;
      if (!rle(&nb)) return x.status;
      c.restore.resize(ndist);
      if (!x.ok(cudaMemcpyAsync(c.restore.data(), d_restore.p, 4 * (size_t)ndist, cudaMemcpyDeviceToHost, x.st),
                "download") ||
          !x.ok(cudaMemcpyAsync(c.cols_offset.data(), d_coff.p, 8 * (size_t)(blk_m + 1), cudaMemcpyDeviceToHost, x.st),
                "download"))
        return x.status;
      if (dc) {  // keep for the device page-stream fill
        dc->restore = d_restore.as<uint32_t>(); d_restore.p = nullptr;
        dc->cols_offset = d_coff.as<uint64_t>(); d_coff.p = nullptr;
      }
    }
  }
  d_key.release();
  d_bid.release();
  d_col.release();
  tm.lap("dev a4 aggregation");

  // a5 + a6: formats, record sizes, VPs, pack
  c.nb = nb;
  std::vector<int32_t> nbr(nb), nbc(nb), nnzb(nb);
  std::vector<uint8_t> ntype(nb);
  std::vector<uint64_t> nvp(nb);
  if (nb > 0) {
    DBuf d_br, d_bc, d_nnz, d_type, d_rb, d_vp, d_est, d_mtx;
    if (!x.alloc(d_br, 4 * (size_t)nb, "alloc") || !x.alloc(d_bc, 4 * (size_t)nb, "alloc") ||
        !x.alloc(d_nnz, 4 * (size_t)nb, "alloc") || !x.alloc(d_type, (size_t)nb, "alloc") ||
        !x.alloc(d_rb, 8 * (size_t)nb, "alloc") || !x.alloc(d_vp, 8 * (size_t)nb, "alloc") ||
        !x.alloc(d_est, 4 * (size_t)nb, "alloc"))
      return x.status;
    FmtParams f{o.th1, o.th2, o.force_format, S};
    k_block_meta<<<grid_for(nb, TPB), TPB, 0, x.st>>>(d_ubid.as<uint64_t>(), d_cnt.as<uint32_t>(), nb, f,
                                                      d_br.as<int32_t>(), d_bc.as<int32_t>(), d_nnz.as<int32_t>(),
                                                      d_type.as<uint8_t>(), d_rb.as<uint64_t>());
    if (!cub_call(x, "scan", [&](void *t, size_t &b) {
          return cub::DeviceScan::ExclusiveSum(t, b, d_rb.as<uint64_t>(), d_vp.as<uint64_t>(), nb, x.st);
        }) ||
        !cub_call(x, "scan", [&](void *t, size_t &b) {
          return cub::DeviceScan::ExclusiveSum(t, b, d_cnt.as<uint32_t>(), d_est.as<uint32_t>(), nb, x.st);
        }))
      return x.status;
    uint64_t last_vp = 0, last_rb = 0;
    if (!x.ok(cudaMemcpyAsync(&last_vp, d_vp.as<uint64_t>() + (nb - 1), 8, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaMemcpyAsync(&last_rb, d_rb.as<uint64_t>() + (nb - 1), 8, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaStreamSynchronize(x.st), "sync"))
      return x.status;
    const uint64_t mbytes = last_vp + last_rb;
    if (!x.alloc(d_mtx, mbytes, "alloc mtx") || !x.ok(cudaMemsetAsync(d_mtx.p, 0, mbytes, x.st), "memset"))
      return x.status;
    if (S == 8)
      k_pack<8><<<grid_for(nb * 32, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), d_idx_s.as<uint32_t>(),
                                                          d_est.as<uint32_t>(), d_nnz.as<int32_t>(), d_type.as<uint8_t>(),
                                                          d_vp.as<uint64_t>(), nb, d_val.as<uint8_t>(), d_mtx.as<uint8_t>());
    else
      k_pack<4><<<grid_for(nb * 32, TPB), TPB, 0, x.st>>>(d_key_s.as<uint64_t>(), d_idx_s.as<uint32_t>(),
                                                          d_est.as<uint32_t>(), d_nnz.as<int32_t>(), d_type.as<uint8_t>(),
                                                          d_vp.as<uint64_t>(), nb, d_val.as<uint8_t>(), d_mtx.as<uint8_t>());
    if (!x.ok(cudaGetLastError(), "pack launch")) return x.status;
    c.mtx.resize((size_t)mbytes);  // sized always (info); filled only when downloaded
    if (download_records || !dc) {
      if (!x.ok(cudaMemcpyAsync(c.mtx.data(), d_mtx.p, mbytes, cudaMemcpyDeviceToHost, x.st), "download"))
        return x.status;
    }
    if (!x.ok(cudaMemcpyAsync(nbr.data(), d_br.p, 4 * (size_t)nb, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaMemcpyAsync(nbc.data(), d_bc.p, 4 * (size_t)nb, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaMemcpyAsync(nnzb.data(), d_nnz.p, 4 * (size_t)nb, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaMemcpyAsync(ntype.data(), d_type.p, (size_t)nb, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaMemcpyAsync(nvp.data(), d_vp.p, 8 * (size_t)nb, cudaMemcpyDeviceToHost, x.st), "download") ||
        !x.ok(cudaStreamSynchronize(x.st), "sync"))
      return x.status;
    if (dc) { dc->mtx = d_mtx.as<uint8_t>(); d_mtx.p = nullptr; }
  } else if (!x.ok(cudaStreamSynchronize(x.st), "sync")) {
    return x.status;
  }
  for (int k = 0; k < 3; k++) c.fmt_count[k] = 0;
  for (uint8_t t : ntype) c.fmt_count[t]++;
  tm.lap("dev a5+a6 formats, pack, download");
  balance_and_permute(c, o, nbr.data(), nbc.data(), nnzb.data(), ntype.data(), nvp.data(), tm);  // a7 (host)
  return CBSPMV_OK;
}

void DevCanon::release() {
  if (mtx) cudaFree(mtx);
  if (restore) cudaFree(restore);
  if (cols_offset) cudaFree(cols_offset);
  mtx = nullptr; restore = nullptr; cols_offset = nullptr;
}

namespace {

// page prefixes (header | descriptors | items, 16-byte multiples) -> their pages
__global__ void k_prefix(const uint8_t *__restrict__ meta, const uint64_t *__restrict__ meta_off,
                         const uint64_t *__restrict__ page_off, int64_t npages, uint8_t *__restrict__ stream) {
  for (int64_t p = blockIdx.x; p < npages; p += gridDim.x) {
    const uint4 *src = reinterpret_cast<const uint4 *>(meta + meta_off[p]);
    uint4 *dst = reinterpret_cast<uint4 *>(stream + page_off[p]);
    const int64_t n = (int64_t)(meta_off[p + 1] - meta_off[p]) / 16;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

// one warp per slot-order CSR / DENSE block: restore entries (aggregated) and the record; DENSE
// records re-laid in lane-major 16-byte pairs (pair q*32 + l holds A[l % 16][(l / 16) * 8 + 2q + h],
// h = 0, 1; cb_internal.h)
template <typename W>
__global__ void k_records(int64_t nb, const int32_t *__restrict__ br, const int32_t *__restrict__ bc,
                          const int32_t *__restrict__ nnz, const uint8_t *__restrict__ type,
                          const uint64_t *__restrict__ vp, const uint64_t *__restrict__ rec_dst,
                          const uint64_t *__restrict__ res_dst, const int32_t *__restrict__ ncol,
                          const uint8_t *__restrict__ mtx, const uint32_t *__restrict__ restore,
                          const uint64_t *__restrict__ coff, uint8_t *__restrict__ stream) {
  constexpr int S = (int)sizeof(W);
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = w0; b < nb; b += nw) {
    const int t = type[b], k = nnz[b];
    if (t == CBSPMV_FMT_COO) continue;  // COO blocks go into chunks (k_coo)
    if (res_dst && lane < ncol[b])
      reinterpret_cast<uint32_t *>(stream + res_dst[b])[lane] = restore[coff[br[b]] + (uint64_t)bc[b] * kBlk + lane];
    const W *src = reinterpret_cast<const W *>(mtx + vp[b]);
    W *dst = reinterpret_cast<W *>(stream + rec_dst[b]);
    if (t == CBSPMV_FMT_DENSE) {
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int h = 0; h < 2; h++) dst[(q * 32 + lane) * 2 + h] = src[(lane & 15) * 16 + (lane >> 4) * 8 + 2 * q + h];
    } else {
      const int64_t idx = kBlk + 1 + k;
      const int64_t words = (idx + d_pad(idx, S)) / S + k;  // record bytes / S
      for (int64_t q = lane; q < words; q += 32) dst[q] = src[q];
    }
  }
}

// one warp per COO block: its elements into their row-run slices (cb_internal.h) at the page
// offsets the host plan computed (coo_dst: column offset | value offset << 16, page-relative;
// rec_dst: the block's page), the column resolved through restore_cols (aggregated)
// or bc*16 + local column.
template <typename W>
__global__ void k_coo(int64_t nb, const int32_t *__restrict__ br, const int32_t *__restrict__ bc,
                      const int32_t *__restrict__ nnz, const uint64_t *__restrict__ vp,
                      const int64_t *__restrict__ e0, const uint32_t *__restrict__ dst,
                      const uint64_t *__restrict__ page, const uint8_t *__restrict__ mtx,
                      const uint32_t *__restrict__ restore, const uint64_t *__restrict__ coff, int agg,
                      const uint32_t *__restrict__ hot, uint8_t *__restrict__ stream) {
  constexpr int S = (int)sizeof(W);
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = w0; b < nb; b += nw) {
    if (e0[b] < 0) continue;
    const int k = nnz[b];
    const uint8_t *coord = mtx + vp[b];
    const W *vals = reinterpret_cast<const W *>(coord + k + d_pad(k, S));
    const uint32_t *seg = agg ? restore + coff[br[b]] + (uint64_t)bc[b] * kBlk : nullptr;
    uint8_t *pg = stream + page[b];
    for (int e = lane; e < k; e += 32) {
      const uint32_t d = dst[e0[b] + e];
      const uint32_t cb = coord[e];  // (col << 4) | row
      uint32_t col = seg ? seg[cb >> 4] : (uint32_t)bc[b] * kBlk + (cb >> 4);
      if (hot && hot[col] != 0xFFFFFFFFu) col = kHotBit | hot[col];  // cached x column (cb_internal.h)
      *reinterpret_cast<uint32_t *>(pg + (d & 0xFFFFu)) = col;
      *reinterpret_cast<W *>(pg + (d >> 16)) = vals[e];
    }
  }
}

// column -> slot of the hot x columns (the rest of the map is 0xFF-filled)
__global__ void k_hot_map(const uint32_t *__restrict__ cols, int64_t n_hot, uint32_t *__restrict__ map) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_hot; k += (int64_t)gridDim.x * blockDim.x)
    map[cols[k]] = (uint32_t)k;
}

// one warp per COO block: its coordinate bytes into the compact download buffer
__global__ void k_coo_coords(int64_t nb, const int32_t *__restrict__ nnz, const uint64_t *__restrict__ vp,
                             const int64_t *__restrict__ coff, const uint8_t *__restrict__ mtx,
                             uint8_t *__restrict__ out) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t b = w0; b < nb; b += nw) {
    if (coff[b] < 0) continue;
    for (int e = lane; e < nnz[b]; e += 32) out[coff[b] + e] = mtx[vp[b] + e];
  }
}

template <class T>
bool upload_vec(Ctx &x, DBuf &d, const std::vector<T> &v, const char *what) {
  return x.alloc(d, sizeof(T) * v.size(), what) &&
         (v.empty() || x.ok(cudaMemcpyAsync(d.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, x.st), what));
}

}  // namespace

int fill_stream_device(const Canon &c, const DevCanon &dc, const Stream &s, const StreamPlan &plan, void *stream,
                       uint8_t *d_stream, std::string *err) {
  Ctx x{reinterpret_cast<cudaStream_t>(stream), err};
  const int64_t npages = (int64_t)s.page_off.size() - 1, nb = c.nb;
  if (s.nbytes > 0 && !x.ok(cudaMemsetAsync(d_stream, 0, (size_t)s.nbytes, x.st), "memset stream")) return x.status;
  if (npages <= 0) return x.ok(cudaStreamSynchronize(x.st), "sync") ? CBSPMV_OK : x.status;
  DBuf d_meta, d_moff, d_poff, d_br, d_bc, d_nnz, d_type, d_vp, d_rdst, d_sdst, d_ncol, d_e0, d_dst, d_hc, d_hmap;
  if (!upload_vec(x, d_meta, plan.meta, "upload plan") || !upload_vec(x, d_moff, plan.meta_off, "upload plan") ||
      !upload_vec(x, d_poff, s.page_off, "upload plan") || !upload_vec(x, d_br, c.br, "upload plan") ||
      !upload_vec(x, d_bc, c.bc, "upload plan") || !upload_vec(x, d_nnz, c.nnzb, "upload plan") ||
      !upload_vec(x, d_type, c.type, "upload plan") || !upload_vec(x, d_vp, c.vp, "upload plan") ||
      !upload_vec(x, d_rdst, plan.rec_dst, "upload plan") || !upload_vec(x, d_ncol, plan.ncol, "upload plan") ||
      (c.agg && !upload_vec(x, d_sdst, plan.res_dst, "upload plan")) ||
      !upload_vec(x, d_e0, plan.coo_e0, "upload plan") || !upload_vec(x, d_dst, plan.coo_dst, "upload plan"))
    return x.status;
  const int64_t n_hot = (int64_t)s.hot_cols.size();
  if (n_hot > 0) {
    if (!upload_vec(x, d_hc, s.hot_cols, "upload hot columns") || !x.alloc(d_hmap, 4 * (size_t)c.n, "alloc hot map") ||
        !x.ok(cudaMemsetAsync(d_hmap.p, 0xFF, 4 * (size_t)c.n, x.st), "memset hot map"))
      return x.status;
    k_hot_map<<<grid_for(n_hot, 256), 256, 0, x.st>>>(d_hc.as<uint32_t>(), n_hot, d_hmap.as<uint32_t>());
  }
  k_prefix<<<(int)std::min<int64_t>(npages, 148 * 16), 128, 0, x.st>>>(d_meta.as<uint8_t>(), d_moff.as<uint64_t>(),
                                                                      d_poff.as<uint64_t>(), npages, d_stream);
  if (nb > 0) {
    const int g = grid_for(nb * 32, 256);
    const uint64_t *rd = c.agg ? d_sdst.as<uint64_t>() : nullptr;
#define CB_FILL(W)                                                                                                     \
  k_records<W><<<g, 256, 0, x.st>>>(nb, d_br.as<int32_t>(), d_bc.as<int32_t>(), d_nnz.as<int32_t>(),                  \
                                    d_type.as<uint8_t>(), d_vp.as<uint64_t>(), d_rdst.as<uint64_t>(), rd,              \
                                    d_ncol.as<int32_t>(), dc.mtx, dc.restore, dc.cols_offset, d_stream);               \
  k_coo<W><<<g, 256, 0, x.st>>>(nb, d_br.as<int32_t>(), d_bc.as<int32_t>(), d_nnz.as<int32_t>(), d_vp.as<uint64_t>(), \
                                d_e0.as<int64_t>(), d_dst.as<uint32_t>(), d_rdst.as<uint64_t>(), dc.mtx, dc.restore,  \
                                dc.cols_offset, c.agg, n_hot ? d_hmap.as<uint32_t>() : nullptr, d_stream)
    if (c.val_size == 8) {
      CB_FILL(uint64_t);
    } else {
      CB_FILL(uint32_t);
    }
#undef CB_FILL
  }
  if (!x.ok(cudaGetLastError(), "fill launch") || !x.ok(cudaStreamSynchronize(x.st), "sync")) return x.status;
  return CBSPMV_OK;
}

int download_coo_coords(const Canon &c, const DevCanon &dc, void *stream, CooCoords *out, std::string *err) {
  Ctx x{reinterpret_cast<cudaStream_t>(stream), err};
  const int64_t nb = c.nb;
  out->off.assign((size_t)nb, -1);
  int64_t n = 0;
  for (int64_t i = 0; i < nb; i++)
    if (c.type[i] == CBSPMV_FMT_COO) { out->off[i] = n; n += c.nnzb[i]; }
  out->bytes.resize((size_t)n);
  if (n == 0) return CBSPMV_OK;
  DBuf d_nnz, d_vp, d_off, d_out;
  if (!upload_vec(x, d_nnz, c.nnzb, "upload") || !upload_vec(x, d_vp, c.vp, "upload") ||
      !upload_vec(x, d_off, out->off, "upload") || !x.alloc(d_out, (size_t)n, "alloc"))
    return x.status;
  k_coo_coords<<<grid_for(nb * 32, 256), 256, 0, x.st>>>(nb, d_nnz.as<int32_t>(), d_vp.as<uint64_t>(),
                                                         d_off.as<int64_t>(), dc.mtx, d_out.as<uint8_t>());
  if (!x.ok(cudaGetLastError(), "coords launch") ||
      !x.ok(cudaMemcpyAsync(out->bytes.data(), d_out.p, (size_t)n, cudaMemcpyDeviceToHost, x.st), "download") ||
      !x.ok(cudaStreamSynchronize(x.st), "sync"))
    return x.status;
  return CBSPMV_OK;
}

}  // namespace cb
