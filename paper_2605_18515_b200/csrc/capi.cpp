// capi.cpp — the extern "C" boundary of libcbspmv (include/cbspmv.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include <cuda_runtime.h>

#include "cb_internal.h"
#include "cbspmv.h"

namespace {

thread_local std::string g_err;

cbspmv_status_t fail(int st, const std::string &msg) {
  g_err = msg;
  return (cbspmv_status_t)st;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct DeviceGuard {  // switch to the handle's device for the call, restore afterwards
  int prev = -1, want;
  explicit DeviceGuard(int d) : want(d) {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

void load_stats(const std::vector<int64_t> &v, double *mean, double *sd, int64_t *mx) {
  double s = 0, s2 = 0;
  int64_t M = 0;
  for (int64_t x : v) { s += (double)x; M = std::max(M, x); }
  double mu = v.empty() ? 0.0 : s / (double)v.size();
  for (int64_t x : v) s2 += ((double)x - mu) * ((double)x - mu);
  *mean = mu;
  *sd = v.empty() ? 0.0 : std::sqrt(s2 / (double)v.size());
  *mx = M;
}

}  // namespace

struct cbspmv_s {
  int device = -1;
  int dtype = CBSPMV_F64;
  int val_size = 8;
  bool has_host = false;
  cb::Canon canon;
  cbspmv_info_t info{};
  CbDevice dev;
  uint8_t *d_stream = nullptr;
  uint64_t *d_page_off = nullptr;
  uint32_t *d_cta_page = nullptr;
  void *d_x_tmp = nullptr;
  void *d_y_tmp = nullptr;
};

extern "C" {

cbspmv_status_t cbspmv_default_options(cbspmv_options_t *o) {
  if (!o) return fail(CBSPMV_EINVAL, "null options");
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(*o);
  o->blk = 16;
  o->th0_num = 15;       // th0 = 0.15
  o->th0_den = 100;
  o->ss_limit = 32;      // "lower than 32 non-zero values"
  o->th1 = 32;
  o->th2 = 128;
  o->warps_per_tb = 8;
  o->agg_mode = -1;
  o->balance = 1;
  o->force_format = -1;
  o->device = 0;
  o->host_threads = 0;
  o->keep_host = 1;
  return CBSPMV_OK;
}

static void free_device(cbspmv_s *h) {
  if (h->device < 0) return;
  DeviceGuard g(h->device);
  cudaFree(h->d_stream);
  cudaFree(h->d_page_off);
  cudaFree(h->d_cta_page);
  cudaFree(h->d_x_tmp);
  cudaFree(h->d_y_tmp);
  h->d_stream = nullptr; h->d_page_off = nullptr; h->d_cta_page = nullptr;
  h->d_x_tmp = nullptr; h->d_y_tmp = nullptr;
}

cbspmv_status_t cbspmv_build(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                             const void *vals, cbspmv_dtype_t dtype, const cbspmv_options_t *opts, void *stream,
                             cbspmv_handle_t *out) {
  if (!out) return fail(CBSPMV_EINVAL, "null output handle pointer");
  *out = nullptr;
  cbspmv_options_t o;
  cbspmv_default_options(&o);
  if (opts) {
    if (opts->struct_size != sizeof(cbspmv_options_t)) return fail(CBSPMV_EINVAL, "options struct_size mismatch");
    o = *opts;
  }
  if (dtype != CBSPMV_F64 && dtype != CBSPMV_F32) return fail(CBSPMV_EINVAL, "bad dtype");
  if (m < 0 || n < 0 || nnz < 0) return fail(CBSPMV_EINVAL, "negative dimension");
  if (m > 0 && !row_ptr) return fail(CBSPMV_EINVAL, "null row_ptr");
  if (o.device >= 0 && o.blk != 16) return fail(CBSPMV_EUNSUPPORTED, "device kernels require blk = 16");
  if (o.device >= 0 && m > (int64_t)UINT32_MAX)
    return fail(CBSPMV_EUNSUPPORTED, "m too large for 32-bit block row offsets");

  cbspmv_s *h = new (std::nothrow) cbspmv_s();
  if (!h) return fail(CBSPMV_ENOMEM, "handle allocation");
  h->dtype = dtype;
  h->val_size = dtype == CBSPMV_F64 ? 8 : 4;

  const double t0 = now();
  cb::Csr A{m, n, nnz, row_ptr, col_idx, vals, h->val_size};
  std::string err;
  int st = cb::build_canonical(A, o, &h->canon, &err);
  if (st != CBSPMV_OK) { delete h; return fail(st, err); }
  const cb::Canon &c = h->canon;

  cbspmv_info_t &I = h->info;
  I.m = c.m; I.n = c.n; I.nnz = c.nnz; I.blk_m = c.blk_m; I.nb = c.nb; I.nb_pre = c.nb_pre;
  I.ss_count = c.ss_count; I.agg = c.agg; I.dtype = dtype;
  for (int k = 0; k < 3; k++) I.fmt_count[k] = c.fmt_count[k];
  I.T = c.T;
  load_stats(c.tb_load, &I.tb_load_mean, &I.tb_load_sd, &I.tb_load_max);
  double mu_nat;
  load_stats(c.tb_load_nat, &mu_nat, &I.tb_load_sd_natural, &I.tb_load_max_natural);
  I.mtx_bytes = (int64_t)c.mtx.size();
  I.n_restore = (int64_t)c.restore.size();
  I.meta_bytes = 21 * c.nb;
  I.alg_bytes = I.meta_bytes + I.mtx_bytes + 4 * I.n_restore + (c.agg ? 8 * (c.blk_m + 1) : 0) +
                (int64_t)h->val_size * (c.n + c.m);

  if (o.device >= 0) {
    h->device = o.device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || o.device >= ndev) {
      cudaGetLastError();
      delete h;
      return fail(CBSPMV_ECUDA, "no CUDA device " + std::to_string(o.device));
    }
    DeviceGuard g(h->device);
    cb::Stream S;
    const char *env = std::getenv("CBSPMV_PAGE_BYTES");
    int cap = env ? std::atoi(env) : cb::kDefaultStageCap;
    cap = (int)cb::round_up(std::max(cap, 1024), 16);
    st = cb::build_stream(c, cap, o.host_threads, &S, &err);
    if (st != CBSPMV_OK) { cb::free_stream(&S); delete h; return fail(st, err); }
    I.build_seconds = now() - t0;
    const int64_t npages = (int64_t)S.page_off.size() - 1;
    CbDevice &D = h->dev;
    D.device = h->device; D.dtype = dtype; D.agg = c.agg; D.m = c.m; D.n = c.n;
    D.n_pages = npages; D.page_cap = cap;
    st = cb_configure(&D, &err);
    if (st != CBSPMV_OK) { cb::free_stream(&S); delete h; return fail(st, err); }
    // persistent CTA c streams pages [cta_page[c], cta_page[c+1]): equal byte shares
    std::vector<uint32_t> cta(D.grid + 1, 0);
    const uint64_t total = S.page_off.back();
    for (int g2 = 1; g2 < D.grid; g2++) {
      uint64_t target = total / D.grid * g2 + (total % D.grid) * g2 / D.grid;
      cta[g2] = (uint32_t)(std::lower_bound(S.page_off.begin(), S.page_off.end() - 1, target) - S.page_off.begin());
    }
    cta[D.grid] = (uint32_t)npages;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    const double t1 = now();
    cudaError_t e = cudaSuccess;
    if (S.nbytes > 0) e = cudaMalloc(&h->d_stream, (size_t)S.nbytes);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_page_off, S.page_off.size() * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMalloc(&h->d_cta_page, cta.size() * sizeof(uint32_t));
    if (e != cudaSuccess) {
      cudaGetLastError();
      cb::free_stream(&S); free_device(h); delete h;
      return fail(CBSPMV_ENOMEM, std::string("device allocation: ") + cudaGetErrorString(e));
    }
    // "transferred to the GPU in a single operation"
    if (S.nbytes > 0) e = cudaMemcpyAsync(h->d_stream, S.bytes, (size_t)S.nbytes, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h->d_page_off, S.page_off.data(), S.page_off.size() * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h->d_cta_page, cta.data(), cta.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    cb::free_stream(&S);
    if (e != cudaSuccess) {
      cudaGetLastError(); free_device(h); delete h;
      return fail(CBSPMV_ECUDA, std::string("upload: ") + cudaGetErrorString(e));
    }
    I.upload_seconds = now() - t1;
    D.d_stream = h->d_stream; D.d_page_off = h->d_page_off; D.d_cta_page = h->d_cta_page;
    I.dev_stream_bytes = (int64_t)total;
    I.n_pages = npages;
    I.dev_bytes = (int64_t)total + (int64_t)(npages + 1) * 8 + (int64_t)cta.size() * 4;
    I.grid = D.grid;
    I.launches_per_spmv = (c.m > 0 ? 1 : 0) + (npages > 0 ? 1 : 0);
  } else {
    I.build_seconds = now() - t0;
  }
  h->has_host = o.keep_host != 0;
  if (!h->has_host) {
    cb::Canon small;
    small.m = c.m; small.n = c.n; small.nnz = c.nnz; small.nb = c.nb; small.T = c.T;
    h->canon = std::move(small);
  }
  *out = h;
  g_err.clear();
  return CBSPMV_OK;
}

static cbspmv_status_t check_dev(cbspmv_handle_t h, const void *x, const void *y) {
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle (built with device = -1)");
  if ((h->info.n > 0 && !x) || (h->info.m > 0 && !y)) return fail(CBSPMV_EINVAL, "null x or y");
  const uintptr_t a = (uintptr_t)h->val_size - 1;
  if (((uintptr_t)x & a) || ((uintptr_t)y & a)) return fail(CBSPMV_EDIM, "x / y not aligned to the value size");
  if (x && y && x == y) return fail(CBSPMV_EINVAL, "y must not alias x");
  return CBSPMV_OK;
}

static cbspmv_status_t run(cbspmv_handle_t h, const void *x, void *y, const double *ss, bool zero, void *stream) {
  cbspmv_status_t s = check_dev(h, x, y);
  if (s != CBSPMV_OK) return s;
  DeviceGuard g(h->device);
  std::string err;
  int st = cb_launch_spmv(h->dev, x, y, ss, zero, stream, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_spmv(cbspmv_handle_t h, const void *x, void *y, void *stream) {
  return run(h, x, y, nullptr, true, stream);
}

cbspmv_status_t cbspmv_spmv_add(cbspmv_handle_t h, const void *x, void *y, void *stream) {
  return run(h, x, y, nullptr, false, stream);
}

cbspmv_status_t cbspmv_spmv_scaled(cbspmv_handle_t h, const void *x, const double *sumsq, void *y, void *stream) {
  if (!sumsq) return fail(CBSPMV_EINVAL, "null sumsq");
  return run(h, x, y, sumsq, true, stream);
}

cbspmv_status_t cbspmv_spmv_host(cbspmv_handle_t h, const void *x_host, void *y_host, void *stream) {
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if ((h->info.n > 0 && !x_host) || (h->info.m > 0 && !y_host)) return fail(CBSPMV_EINVAL, "null x or y");
  DeviceGuard g(h->device);
  cudaError_t e = cudaSuccess;
  const size_t xb = (size_t)h->info.n * h->val_size, yb = (size_t)h->info.m * h->val_size;
  if (!h->d_x_tmp && xb) e = cudaMalloc(&h->d_x_tmp, xb);
  if (e == cudaSuccess && !h->d_y_tmp && yb) e = cudaMalloc(&h->d_y_tmp, yb);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ENOMEM, "device x/y staging"); }
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (xb) e = cudaMemcpyAsync(h->d_x_tmp, x_host, xb, cudaMemcpyHostToDevice, cs);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  std::string err;
  int st = cb_launch_spmv(h->dev, h->d_x_tmp, h->d_y_tmp, nullptr, true, stream, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  if (yb) e = cudaMemcpyAsync(y_host, h->d_y_tmp, yb, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_sumsq(const void *v, int64_t len, cbspmv_dtype_t dtype, double *out, int32_t device,
                             void *stream) {
  if (!out || (len > 0 && !v) || len < 0) return fail(CBSPMV_EINVAL, "bad sumsq arguments");
  DeviceGuard g(device);
  std::string err;
  int st = cb_launch_sumsq(v, len, dtype, out, stream, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_block_stats(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                                   const void *vals, cbspmv_dtype_t dtype, const cbspmv_options_t *opts,
                                   int64_t *nb_pre, int64_t *ss_count) {
  if (!nb_pre || !ss_count) return fail(CBSPMV_EINVAL, "null output");
  cbspmv_options_t o;
  cbspmv_default_options(&o);
  if (opts) {
    if (opts->struct_size != sizeof(cbspmv_options_t)) return fail(CBSPMV_EINVAL, "options struct_size mismatch");
    o = *opts;
  }
  if (dtype != CBSPMV_F64 && dtype != CBSPMV_F32) return fail(CBSPMV_EINVAL, "bad dtype");
  if (m < 0 || n < 0 || nnz < 0 || (m > 0 && !row_ptr)) return fail(CBSPMV_EINVAL, "bad CSR");
  cb::Csr A{m, n, nnz, row_ptr, col_idx, vals, dtype == CBSPMV_F64 ? 8 : 4};
  std::string err;
  int st = cb::block_stats(A, o, nb_pre, ss_count, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_decide_agg(int64_t nb_pre, int64_t ss_count, const cbspmv_options_t *opts, int32_t *agg) {
  if (!agg || nb_pre < 0 || ss_count < 0 || ss_count > nb_pre) return fail(CBSPMV_EINVAL, "bad arguments");
  cbspmv_options_t o;
  cbspmv_default_options(&o);
  if (opts) {
    if (opts->struct_size != sizeof(cbspmv_options_t)) return fail(CBSPMV_EINVAL, "options struct_size mismatch");
    o = *opts;
  }
  if (o.th0_den <= 0) return fail(CBSPMV_EINVAL, "th0_den must be positive");
  *agg = cb::decide_agg(nb_pre, ss_count, o) ? 1 : 0;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_get_info(cbspmv_handle_t h, cbspmv_info_t *info) {
  if (!h || !info) return fail(CBSPMV_EINVAL, "null argument");
  *info = h->info;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_export(cbspmv_handle_t h, cbspmv_export_t *ex) {
  if (!h || !ex) return fail(CBSPMV_EINVAL, "null argument");
  if (!h->has_host) return fail(CBSPMV_EUNSUPPORTED, "built with keep_host = 0");
  const cb::Canon &c = h->canon;
  ex->nb = c.nb; ex->T = c.T; ex->mtx_bytes = (int64_t)c.mtx.size();
  ex->n_restore = (int64_t)c.restore.size(); ex->n_cols_offset = (int64_t)c.cols_offset.size();
  ex->blk_row_idx = c.br.data(); ex->blk_col_idx = c.bc.data(); ex->nnz_per_blk = c.nnzb.data();
  ex->type_per_blk = c.type.data(); ex->vp_per_blk = c.vp.data(); ex->mtx_data = c.mtx.data();
  ex->restore_cols = c.restore.empty() ? nullptr : c.restore.data();
  ex->cols_offset = c.cols_offset.empty() ? nullptr : c.cols_offset.data();
  ex->tb_ptr = c.tb_ptr.data(); ex->tb_load = c.tb_load.data(); ex->tb_load_natural = c.tb_load_nat.data();
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_download_stream(cbspmv_handle_t h, void *stream_host, size_t stream_bytes,
                                       uint64_t *page_off_host, size_t n_page_off) {
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if (stream_bytes < (size_t)h->info.dev_stream_bytes || n_page_off < (size_t)h->info.n_pages + 1)
    return fail(CBSPMV_EDIM, "destination too small");
  DeviceGuard g(h->device);
  cudaError_t e = cudaSuccess;
  if (h->info.dev_stream_bytes)
    e = cudaMemcpy(stream_host, h->d_stream, (size_t)h->info.dev_stream_bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(page_off_host, h->d_page_off, ((size_t)h->info.n_pages + 1) * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_destroy(cbspmv_handle_t h) {
  if (!h) return CBSPMV_OK;
  free_device(h);
  delete h;
  return CBSPMV_OK;
}

const char *cbspmv_status_string(cbspmv_status_t s) {
  switch (s) {
    case CBSPMV_OK: return "CBSPMV_OK";
    case CBSPMV_EINVAL: return "CBSPMV_EINVAL";
    case CBSPMV_EUNSORTED: return "CBSPMV_EUNSORTED";
    case CBSPMV_ENOMEM: return "CBSPMV_ENOMEM";
    case CBSPMV_ECUDA: return "CBSPMV_ECUDA";
    case CBSPMV_EDIM: return "CBSPMV_EDIM";
    case CBSPMV_EUNSUPPORTED: return "CBSPMV_EUNSUPPORTED";
  }
  return "unknown status";
}

const char *cbspmv_last_error(void) { return g_err.c_str(); }

int32_t cbspmv_version(void) { return CBSPMV_VERSION; }

}  // extern "C"
