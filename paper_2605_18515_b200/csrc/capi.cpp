// capi.cpp — the extern "C" boundary of libcbspmv (include/cbspmv.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
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
  explicit DeviceGuard(int d) : want(d) {  // d < 0: host-only, no-op
    if (want < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (want >= 0 && prev >= 0 && prev != want) cudaSetDevice(prev);
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

// One column panel: the CB-SpMV format of A[:, c0:c1) and its device copy.
struct Part {
  int64_t c0 = 0, c1 = 0;
  cb::Canon canon;
  CbDevice dev;
  uint8_t *d_stream = nullptr;
  uint64_t *d_page_off = nullptr;
  uint32_t *d_cta_page = nullptr;
  uint32_t *d_page_ctr = nullptr;
  uint32_t *d_hot = nullptr;  // hot x columns (shared x cache, cb_internal.h)
  int64_t n_hot = 0;
  int64_t stream_bytes = 0, n_pages = 0;
  std::unique_ptr<cb::DevCanon> dc;  // device builder: records still on the device until the stream fill
};

// Rows x columns [c0, c1) of a canonical CSR (columns keep their global index).
// dtype -> bytes of one stored matrix value / one x or y element
inline int val_bytes(int dtype) { return dtype == CBSPMV_F64 ? 8 : 4; }
inline int vec_bytes(int dtype) { return dtype == CBSPMV_F32 ? 4 : 8; }
inline bool valid_dtype(int dtype) { return dtype == CBSPMV_F64 || dtype == CBSPMV_F32 || dtype == CBSPMV_F32F64; }

struct SubCsr {  // no value-initialisation: the parallel copies write every element
  std::vector<int64_t, cb::NoInitAlloc<int64_t>> rp;
  std::vector<int32_t, cb::NoInitAlloc<int32_t>> col;
  cb::ByteBuf val;  // raw bytes of the value type
};

}  // namespace

int cb_set_error(int st, const std::string &msg) {  // for the other translation units (exchange.cu)
  g_err = msg;
  return st;
}

struct cbspmv_s {
  int device = -1;
  int dtype = CBSPMV_F64;
  int val_size = 8;  // stored matrix values
  int vec_size = 8;  // x / y elements
  bool has_host = false;
  std::vector<Part> parts;
  cbspmv_info_t info{};
  void *d_x_tmp = nullptr;
  void *d_y_tmp = nullptr;
  // cbspmv_spmv_host_batch: second x / y staging slot, copy streams and slot events
  void *d_x_tmp2 = nullptr, *d_y_tmp2 = nullptr;
  cudaStream_t s_up = nullptr, s_down = nullptr;
  cudaEvent_t ev_up[2] = {}, ev_done[2] = {}, ev_down[2] = {};
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
  o->col_panels = 0;
  o->device_build = 0;
  return CBSPMV_OK;
}

static void free_device(cbspmv_s *h) {
  if (h->device < 0) return;
  DeviceGuard g(h->device);
  for (Part &p : h->parts) {
    cudaFree(p.d_stream);
    cudaFree(p.d_page_off);
    cudaFree(p.d_cta_page);
    cudaFree(p.d_page_ctr);
    cudaFree(p.d_hot);
    p.d_stream = nullptr; p.d_page_off = nullptr; p.d_cta_page = nullptr; p.d_page_ctr = nullptr; p.d_hot = nullptr;
  }
  cudaFree(h->d_x_tmp);
  cudaFree(h->d_y_tmp);
  h->d_x_tmp = nullptr; h->d_y_tmp = nullptr;
  cudaFree(h->d_x_tmp2);
  cudaFree(h->d_y_tmp2);
  h->d_x_tmp2 = nullptr; h->d_y_tmp2 = nullptr;
  for (int b = 0; b < 2; b++) {
    if (h->ev_up[b]) cudaEventDestroy(h->ev_up[b]);
    if (h->ev_done[b]) cudaEventDestroy(h->ev_done[b]);
    if (h->ev_down[b]) cudaEventDestroy(h->ev_down[b]);
    h->ev_up[b] = h->ev_done[b] = h->ev_down[b] = nullptr;
  }
  if (h->s_up) cudaStreamDestroy(h->s_up);
  if (h->s_down) cudaStreamDestroy(h->s_down);
  h->s_up = h->s_down = nullptr;
}

// Device page stream of one panel's canonical format, uploaded in one copy (a8).
static int upload_part(const cbspmv_options_t &o, int dtype, cudaStream_t cs, Part *P, double *t_up,
                       std::string *err) {
  cb::NvtxRange nvtx_("cbspmv upload (stream plan + one copy)");
  const cb::Canon &c = P->canon;
  cb::Stream S;
  CbShape shape;
  // aggregated matrices with >= 10 % CSR / DENSE blocks (the Laplacian's diagonal blocks): x warps
  // gather those tiles through their restore entries ahead of the consumers (CBSPMV_XAGG=0/1
  // overrides, read per build)
  const int64_t n_cd = c.fmt_count[CBSPMV_FMT_CSR] + c.fmt_count[CBSPMV_FMT_DENSE];
  bool agg_tiles = c.agg && c.nb > 0 && n_cd * 10 >= c.nb;
  if (const char *v = std::getenv("CBSPMV_XAGG")) agg_tiles = c.agg && std::atoi(v) != 0;
  int st = cb_plan_stages(o.device, c.agg, agg_tiles, &shape, err);
  if (st != CBSPMV_OK) return st;
  cb::StreamPlan plan;
  const bool on_device = P->dc != nullptr;  // records on the device: fill the stream there
  // Row-run slices (cb_internal.h): a lane sums its piece of a row's run and issues one RED for
  // it.  Env knobs, read per build, for A/B runs: CBSPMV_RUN_MAX (Lmax, default 8),
  // CBSPMV_COO_RUNS=0 (Lmax = 1: one RED per element), CBSPMV_RUN_ORDER=row (pieces by row instead
  // of by length), CBSPMV_HOT_BYTES (shared x cache budget, 0: none), CBSPMV_HOT_MIN_PCT (share
  // of the COO elements the cache must serve; 0 forces the cache on).
  cb::SliceOpts so;
  if (const char *v = std::getenv("CBSPMV_RUN_MAX")) so.run_max = std::atoi(v);
  if (const char *v = std::getenv("CBSPMV_HOT_BYTES")) so.hot_bytes = std::max(0, std::atoi(v));
  if (const char *v = std::getenv("CBSPMV_HOT_MIN_PCT")) so.hot_min_pct = std::max(0, std::atoi(v));
  if (const char *v = std::getenv("CBSPMV_COO_RUNS"); v && std::atoi(v) == 0) so.run_max = 1;
  if (const char *v = std::getenv("CBSPMV_RUN_ORDER"); v && std::string(v) == "row") so.row_order = 1;
  so.hot_bytes = std::min(so.hot_bytes, shape.hot_cap);  // what the stages leave of the shared memory
  cb::CooCoords coords;
  if (on_device) {  // the records stay on the device: the slice layout needs the COO coordinates
    st = cb::download_coo_coords(c, *P->dc, cs, &coords, err);
    if (st != CBSPMV_OK) return st;
  }
  st = cb::build_stream(c, shape.page_cap, vec_bytes(dtype), o.host_threads, &S, on_device ? &plan : nullptr, err,
                        so, on_device ? &coords : nullptr, shape.xagg != 0);
  if (st != CBSPMV_OK) { cb::free_stream(&S); return st; }
  const int64_t npages = (int64_t)S.page_off.size() - 1;
  CbDevice &D = P->dev;
  static_cast<CbShape &>(D) = shape;
  D.device = o.device; D.dtype = dtype; D.agg = c.agg; D.m = c.m; D.n = c.n;
  D.n_pages = npages;
  D.n_hot = (int)S.hot_cols.size();
  st = cb_configure(&D, err);
  if (st != CBSPMV_OK) { cb::free_stream(&S); return st; }
  // persistent CTA g streams pages [cta[g], cta[g+1]): equal byte shares
  std::vector<uint32_t> cta(D.grid + 1, 0);
  const uint64_t total = S.page_off.back();
  for (int g = 1; g < D.grid; g++) {
    uint64_t target = total / D.grid * g + (total % D.grid) * g / D.grid;
    cta[g] = (uint32_t)(std::lower_bound(S.page_off.begin(), S.page_off.end() - 1, target) - S.page_off.begin());
  }
  cta[D.grid] = (uint32_t)npages;
  const double t1 = now();
  cb::PhaseTimer tm;
  cudaError_t e = cudaSuccess;
  if (S.nbytes > 0) e = cudaMalloc(&P->d_stream, (size_t)S.nbytes);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_page_off, S.page_off.size() * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_cta_page, cta.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&P->d_page_ctr, cb::kCtrSlots * 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(P->d_page_ctr, 0, cb::kCtrSlots * 2 * sizeof(uint32_t), cs);
  if (e == cudaSuccess && !S.hot_cols.empty()) e = cudaMalloc(&P->d_hot, S.hot_cols.size() * sizeof(uint32_t));
  if (e != cudaSuccess) {
    cudaGetLastError();
    cb::free_stream(&S);
    *err = std::string("device allocation: ") + cudaGetErrorString(e);
    return CBSPMV_ENOMEM;
  }
  // "transferred to the GPU in a single operation"; device builder: filled in place
  tm.lap("upload: device allocations");
  if (on_device) {
    st = cb::fill_stream_device(c, *P->dc, S, plan, cs, P->d_stream, err);
    tm.lap("upload: device stream fill");
    P->dc.reset();
    tm.lap("upload: free device records");
    if (st != CBSPMV_OK) { cb::free_stream(&S); return st; }
  } else if (S.nbytes > 0) {
    e = cudaMemcpyAsync(P->d_stream, S.bytes, (size_t)S.nbytes, cudaMemcpyHostToDevice, cs);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(P->d_page_off, S.page_off.data(), S.page_off.size() * sizeof(uint64_t),
                        cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(P->d_cta_page, cta.data(), cta.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && !S.hot_cols.empty())
    e = cudaMemcpyAsync(P->d_hot, S.hot_cols.data(), S.hot_cols.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  tm.lap("upload: copies + sync");
  cb::free_stream(&S);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = std::string("upload: ") + cudaGetErrorString(e);
    return CBSPMV_ECUDA;
  }
  *t_up += now() - t1;
  D.d_stream = P->d_stream; D.d_page_off = P->d_page_off; D.d_cta_page = P->d_cta_page;
  D.d_page_ctr = P->d_page_ctr;
  D.d_hot = P->d_hot;
  P->n_hot = (int64_t)S.hot_cols.size();
  P->stream_bytes = (int64_t)total;
  P->n_pages = npages;
  return CBSPMV_OK;
}

// Build + upload one panel's format (the Fig. 7 pipeline on A[:, c0:c1)).
static int build_part(const cb::Csr &A, const cbspmv_options_t &o, int dtype, cudaStream_t cs, Part *P,
                      double *t_up, std::string *err) {
  cb::NvtxRange nvtx_("cbspmv build (a1..a7)");
  int st;
  if (o.device >= 0 && o.device_build) {
    P->dc.reset(new cb::DevCanon());
    st = cb::build_canonical_device(A, o, cs, &P->canon, P->dc.get(), o.keep_host != 0, err);
    if (st != CBSPMV_OK) P->dc.reset();
  } else {
    st = cb::build_canonical(A, o, &P->canon, err);
  }
  if (st != CBSPMV_OK || o.device < 0) return st;
  return upload_part(o, dtype, cs, P, t_up, err);
}

// info: sums over panels; drops the host arrays unless keep_host
static void fill_info(cbspmv_s *h, int64_t m, int64_t n, double t0, double t_up, bool keep_host) {
  const int P = (int)h->parts.size();
  const int dtype = h->dtype;
  cbspmv_info_t &I = h->info;
  I.m = m; I.n = n; I.dtype = dtype; I.n_panels = P;
  std::vector<int64_t> loads, loads_nat;
  for (const Part &p : h->parts) {
    const cb::Canon &c = p.canon;
    I.nnz += c.nnz; I.nb += c.nb; I.nb_pre += c.nb_pre; I.ss_count += c.ss_count; I.agg |= c.agg;
    I.blk_m = c.blk_m;
    for (int k = 0; k < 3; k++) I.fmt_count[k] += c.fmt_count[k];
    I.T += c.T;
    I.mtx_bytes += (int64_t)c.mtx.size();
    I.n_restore += (int64_t)c.restore.size();
    I.meta_bytes += 21 * c.nb;
    I.alg_bytes += 21 * c.nb + (int64_t)c.mtx.size() + 4 * (int64_t)c.restore.size() + (c.agg ? 8 * (c.blk_m + 1) : 0);
    loads.insert(loads.end(), c.tb_load.begin(), c.tb_load.end());
    loads_nat.insert(loads_nat.end(), c.tb_load_nat.begin(), c.tb_load_nat.end());
    I.dev_stream_bytes += p.stream_bytes;
    I.n_pages += p.n_pages;
    I.dev_bytes += p.stream_bytes + (p.n_pages + 1) * 8 + (int64_t)(p.dev.grid + 1) * 4 + 4 * p.n_hot;
    I.launches_per_spmv += p.n_pages > 0 ? 1 : 0;
    I.n_hot += p.n_hot;
  }
  I.alg_bytes += (int64_t)h->vec_size * (n + m);
  load_stats(loads, &I.tb_load_mean, &I.tb_load_sd, &I.tb_load_max);
  double mu_nat;
  load_stats(loads_nat, &mu_nat, &I.tb_load_sd_natural, &I.tb_load_max_natural);
  if (h->device >= 0) {
    I.grid = h->parts[0].dev.grid;
    if (m > 0) I.launches_per_spmv += 1;  // the y-zeroing kernel
  } else {
    I.launches_per_spmv = 0;
  }
  I.upload_seconds = t_up;
  I.build_seconds = now() - t0 - t_up;
  h->has_host = keep_host;
  if (!h->has_host) {
    for (Part &p : h->parts) {
      cb::Canon small;
      small.m = p.canon.m; small.n = p.canon.n; small.nnz = p.canon.nnz; small.nb = p.canon.nb;
      small.T = p.canon.T; small.agg = p.canon.agg; small.blk_m = p.canon.blk_m;
      p.canon = std::move(small);
    }
  }
}

static cbspmv_status_t build_impl(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
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
  if (!valid_dtype(dtype)) return fail(CBSPMV_EINVAL, "bad dtype");
  if (m < 0 || n < 0 || nnz < 0) return fail(CBSPMV_EINVAL, "negative dimension");
  if (m > 0 && !row_ptr) return fail(CBSPMV_EINVAL, "null row_ptr");
  if (o.device >= 0 && o.blk != 16) return fail(CBSPMV_EUNSUPPORTED, "device kernels require blk = 16");
  if (o.device >= 0 && m > (int64_t)UINT32_MAX)
    return fail(CBSPMV_EUNSUPPORTED, "m too large for 32-bit block row offsets");
  if (o.col_panels < 0) return fail(CBSPMV_EINVAL, "col_panels must be >= 0");

  cbspmv_s *h = new (std::nothrow) cbspmv_s();
  if (!h) return fail(CBSPMV_ENOMEM, "handle allocation");
  h->dtype = dtype;
  h->val_size = val_bytes(dtype);
  h->vec_size = vec_bytes(dtype);
  const int S = h->val_size;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (o.device >= 0) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || o.device >= ndev) {
      cudaGetLastError();
      delete h;
      return fail(CBSPMV_ECUDA, "no CUDA device " + std::to_string(o.device));
    }
    h->device = o.device;
  }
  DeviceGuard guard(o.device);

  const double t0 = now();
  cb::Csr A{m, n, nnz, row_ptr, col_idx, vals, S};
  std::string err;
  // column panels (NEXT-1): decided from x's size against the device L2
  int P = o.col_panels;
  if (P == 0) {
    P = 1;
    if (o.device >= 0) {
      int l2 = 0;
      cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, o.device);
      const double xb = (double)n * h->vec_size;
      // x slices of ~1/3 of L2.  Each panel's REDs sweep all of y, so more panels re-read and
      // re-write y once more each, while a wider x slice misses L2 more (uniform 2^25, 268 MB of x,
      // per SpMV on B200 with row-run slices and the L1 left to the gathers: 1 panel 26.1 ms,
      // 3: 13.6, 4: 10.4, 5: 8.68, 6: 8.39, 8: 8.76, 11: 9.2, 16: 9.87, 22: 10.6)
      if (l2 > 0 && xb > 0.75 * l2) P = (int)std::ceil(xb / (0.36 * l2));
    }
  }
  const int64_t nbc = (n + o.blk - 1) / o.blk;
  P = (int)std::max<int64_t>(1, std::min<int64_t>(P, nbc));
  std::vector<int64_t> cuts(P + 1);
  for (int k = 0; k <= P; k++) cuts[k] = std::min<int64_t>(n, (nbc * k / P) * o.blk);
  cuts[P] = n;
  double t_up = 0.0;
  int st = CBSPMV_OK;
  h->parts.resize(P);
  if (P == 1) {
    h->parts[0].c0 = 0; h->parts[0].c1 = n;
    st = build_part(A, o, dtype, cs, &h->parts[0], &t_up, &err);
  } else {
    int64_t nz = 0;
    st = cb::check_csr(A, o, &nz, &err);  // the split below relies on sorted, in-range columns
    for (int k = 0; k < P && st == CBSPMV_OK; k++) {
      SubCsr sub;
      sub.rp.resize((size_t)m + 1);
      sub.rp[0] = 0;
      const int64_t c0 = cuts[k], c1 = cuts[k + 1];
      std::vector<int64_t, cb::NoInitAlloc<int64_t>> lo((size_t)m), hi((size_t)m);
      cb::parallel_for(m, o.host_threads, 1 << 14, [&](int64_t a, int64_t b, int) {
        for (int64_t i = a; i < b; i++) {
          const int32_t *rb = col_idx + row_ptr[i], *re = col_idx + row_ptr[i + 1];
          lo[i] = std::lower_bound(rb, re, (int32_t)c0) - col_idx;
          hi[i] = std::lower_bound(rb, re, (int32_t)std::min<int64_t>(c1, INT32_MAX)) - col_idx;
        }
      });
      for (int64_t i = 0; i < m; i++) sub.rp[i + 1] = sub.rp[i] + (hi[i] - lo[i]);
      const int64_t snz = sub.rp[m];
      sub.col.resize((size_t)std::max<int64_t>(snz, 1));
      sub.val.resize((size_t)std::max<int64_t>(snz, 1) * S);
      cb::parallel_for(m, o.host_threads, 1 << 14, [&](int64_t a, int64_t b, int) {
        for (int64_t i = a; i < b; i++) {
          const int64_t len = hi[i] - lo[i];
          std::memcpy(sub.col.data() + sub.rp[i], col_idx + lo[i], (size_t)len * 4);
          std::memcpy(sub.val.data() + sub.rp[i] * S, (const uint8_t *)vals + lo[i] * S, (size_t)len * S);
        }
      });
      cb::Csr Ak{m, n, snz, sub.rp.data(), sub.col.data(), sub.val.data(), S};
      h->parts[k].c0 = c0; h->parts[k].c1 = c1;
      st = build_part(Ak, o, dtype, cs, &h->parts[k], &t_up, &err);
    }
  }
  if (st != CBSPMV_OK) { free_device(h); delete h; return fail(st, err); }

  fill_info(h, m, n, t0, t_up, o.keep_host != 0);
  *out = h;
  g_err.clear();
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_build(int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                             const void *vals, cbspmv_dtype_t dtype, const cbspmv_options_t *opts, void *stream,
                             cbspmv_handle_t *out) {
  try {
    return build_impl(m, n, nnz, row_ptr, col_idx, vals, dtype, opts, stream, out);
  } catch (const std::bad_alloc &) {  // nothing throws across the ABI
    if (out) *out = nullptr;
    return fail(CBSPMV_ENOMEM, "host allocation during the build");
  }
}

// cuMemGetAddressRange through the runtime's driver entry point (no link-time libcuda dependency,
// so the library still loads on a machine without a driver).
typedef int (*MemGetAddressRangeFn)(unsigned long long *base, size_t *size, unsigned long long dptr);
static MemGetAddressRangeFn address_range_fn() {
  static MemGetAddressRangeFn fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return (MemGetAddressRangeFn)f;
  }();
  return fn;
}

// A device vector argument (include/cbspmv.h "Indexing and pointers"): device memory (or managed)
// of the handle's device, and the allocation holding it extends over `bytes` from p.  The C ABI
// takes no lengths, so the range check is against the enclosing allocation (a caching allocator's
// segment can be larger than the tensor; the Python binding checks exact lengths).
static cbspmv_status_t check_vec(const void *p, size_t bytes, int device, const char *what) {
  if (bytes == 0) return CBSPMV_OK;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CBSPMV_EDIM, std::string(what) + ": not a CUDA pointer");
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(CBSPMV_EDIM, std::string(what) + ": not device memory (host or unregistered pointer)");
  if (a.type == cudaMemoryTypeDevice && a.device != device)
    return fail(CBSPMV_EDIM, std::string(what) + ": on device " + std::to_string(a.device) + ", the handle is on " +
                                 std::to_string(device));
  if (MemGetAddressRangeFn f = address_range_fn()) {
    unsigned long long base = 0;
    size_t size = 0;
    if (f(&base, &size, (unsigned long long)(uintptr_t)p) == 0) {
      const unsigned long long q = (unsigned long long)(uintptr_t)p;
      if (q < base || q - base + bytes > size)
        return fail(CBSPMV_EDIM, std::string(what) + ": the allocation ends before the vector does");
    }
  }
  return CBSPMV_OK;
}

static cbspmv_status_t check_dev(cbspmv_handle_t h, const void *x, const void *y, const double *ss = nullptr) {
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle (built with device = -1)");
  if ((h->info.n > 0 && !x) || (h->info.m > 0 && !y)) return fail(CBSPMV_EINVAL, "null x or y");
  const uintptr_t a = (uintptr_t)h->vec_size - 1;
  if (((uintptr_t)x & a) || ((uintptr_t)y & a)) return fail(CBSPMV_EDIM, "x / y not aligned to the value size");
  if (x && y && x == y) return fail(CBSPMV_EINVAL, "y must not alias x");
  cbspmv_status_t s = check_vec(x, (size_t)h->info.n * (size_t)h->vec_size, h->device, "x");
  if (s == CBSPMV_OK) s = check_vec(y, (size_t)h->info.m * (size_t)h->vec_size, h->device, "y");
  if (s == CBSPMV_OK && ss) s = check_vec(ss, sizeof(double), h->device, "sumsq");
  return s;
}

// y (+)= A·(s·x): the panels run in order, the first launch zeroes y when asked.
static int launch_all(cbspmv_handle_t h, const void *x, void *y, const double *ss, bool zero, void *stream,
                      std::string *err) {
  bool first = true;
  for (const Part &p : h->parts) {
    if (p.n_pages == 0 && !(first && zero)) continue;
    int st = cb_launch_spmv(p.dev, x, y, ss, first && zero, stream, err, !first);
    if (st != CBSPMV_OK) return st;
    first = false;
  }
  return CBSPMV_OK;
}

static cbspmv_status_t run(cbspmv_handle_t h, const void *x, void *y, const double *ss, bool zero, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_spmv");
  cbspmv_status_t s = check_dev(h, x, y, ss);
  if (s != CBSPMV_OK) return s;
  DeviceGuard g(h->device);
  std::string err;
  int st = launch_all(h, x, y, ss, zero, stream, &err);
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

cbspmv_status_t cbspmv_spmv_panel(cbspmv_handle_t h, int32_t k, const void *x, const double *sumsq, void *y,
                                  int32_t zero_y, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_spmv_panel");
  cbspmv_status_t s = check_dev(h, x, y, sumsq);
  if (s != CBSPMV_OK) return s;
  if (k < 0 || k >= (int32_t)h->parts.size()) return fail(CBSPMV_EINVAL, "panel index out of range");
  DeviceGuard g(h->device);
  std::string err;
  int st = cb_launch_spmv(h->parts[k].dev, x, y, sumsq, zero_y != 0, stream, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_panel_bounds(cbspmv_handle_t h, int32_t k, int64_t *c0, int64_t *c1) {
  if (!h || !c0 || !c1) return fail(CBSPMV_EINVAL, "null argument");
  if (k < 0 || k >= (int32_t)h->parts.size()) return fail(CBSPMV_EINVAL, "panel index out of range");
  *c0 = h->parts[k].c0;
  *c1 = h->parts[k].c1;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_spmv_host(cbspmv_handle_t h, const void *x_host, void *y_host, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_spmv_host");
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if ((h->info.n > 0 && !x_host) || (h->info.m > 0 && !y_host)) return fail(CBSPMV_EINVAL, "null x or y");
  DeviceGuard g(h->device);
  cudaError_t e = cudaSuccess;
  const size_t xb = (size_t)h->info.n * h->vec_size, yb = (size_t)h->info.m * h->vec_size;
  if (!h->d_x_tmp && xb) e = cudaMalloc(&h->d_x_tmp, xb);
  if (e == cudaSuccess && !h->d_y_tmp && yb) e = cudaMalloc(&h->d_y_tmp, yb);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ENOMEM, "device x/y staging"); }
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (xb) e = cudaMemcpyAsync(h->d_x_tmp, x_host, xb, cudaMemcpyHostToDevice, cs);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  std::string err;
  int st = launch_all(h, h->d_x_tmp, h->d_y_tmp, nullptr, true, stream, &err);
  if (st != CBSPMV_OK) return fail(st, err);
  if (yb) e = cudaMemcpyAsync(y_host, h->d_y_tmp, yb, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_spmv_host_batch(cbspmv_handle_t h, const void *const *x_host, void *const *y_host,
                                       int64_t count, void *stream) {
  cb::NvtxRange nvtx_("cbspmv_spmv_host_batch");
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if (count < 0 || (count > 0 && (!x_host || !y_host))) return fail(CBSPMV_EINVAL, "bad batch arguments");
  for (int64_t k = 0; k < count; k++)
    if ((h->info.n > 0 && !x_host[k]) || (h->info.m > 0 && !y_host[k])) return fail(CBSPMV_EINVAL, "null x or y");
  DeviceGuard g(h->device);
  cudaError_t e = cudaSuccess;
  const size_t xb = (size_t)h->info.n * h->vec_size, yb = (size_t)h->info.m * h->vec_size;
  if (!h->d_x_tmp && xb) e = cudaMalloc(&h->d_x_tmp, xb);
  if (e == cudaSuccess && !h->d_y_tmp && yb) e = cudaMalloc(&h->d_y_tmp, yb);
  if (e == cudaSuccess && !h->d_x_tmp2 && xb) e = cudaMalloc(&h->d_x_tmp2, xb);
  if (e == cudaSuccess && !h->d_y_tmp2 && yb) e = cudaMalloc(&h->d_y_tmp2, yb);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ENOMEM, "device x/y staging"); }
  if (!h->s_up) {
    e = cudaStreamCreateWithFlags(&h->s_up, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->s_down, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; b++) {
      e = cudaEventCreateWithFlags(&h->ev_up[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_done[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_down[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  }
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  void *dx[2] = {h->d_x_tmp, h->d_x_tmp2}, *dy[2] = {h->d_y_tmp, h->d_y_tmp2};
  // nothing issued before this call may still use the staging slots
  e = cudaEventRecord(h->ev_done[0], cs);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_done[1], cs);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_down[0], cs);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_down[1], cs);
  std::string err;
  for (int64_t k = 0; k < count && e == cudaSuccess; k++) {
    const int b = (int)(k & 1);
    // upload x_k into slot b once SpMV k-2 (its last reader) is done
    e = cudaStreamWaitEvent(h->s_up, h->ev_done[b], 0);
    if (e == cudaSuccess && xb) e = cudaMemcpyAsync(dx[b], x_host[k], xb, cudaMemcpyHostToDevice, h->s_up);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_up[b], h->s_up);
    // SpMV k on the caller's stream once x_k landed and y slot b was downloaded (step k-2)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, h->ev_up[b], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, h->ev_down[b], 0);
    if (e != cudaSuccess) break;
    int st = launch_all(h, dx[b], dy[b], nullptr, true, stream, &err);
    if (st != CBSPMV_OK) return fail(st, err);
    e = cudaEventRecord(h->ev_done[b], cs);
    // download y_k behind the SpMV while the next upload / SpMV proceed
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_down, h->ev_done[b], 0);
    if (e == cudaSuccess && yb) e = cudaMemcpyAsync(y_host[k], dy[b], yb, cudaMemcpyDeviceToHost, h->s_down);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_down[b], h->s_down);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->s_down);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_sumsq(const void *v, int64_t len, cbspmv_dtype_t dtype, double *out, int32_t device,
                             void *stream) {
  if (!out || (len > 0 && !v) || len < 0) return fail(CBSPMV_EINVAL, "bad sumsq arguments");
  if (!valid_dtype(dtype)) return fail(CBSPMV_EINVAL, "bad dtype");
  cbspmv_status_t cs = check_vec(v, (size_t)len * (size_t)vec_bytes(dtype), device, "v");
  if (cs == CBSPMV_OK) cs = check_vec(out, sizeof(double), device, "out");
  if (cs != CBSPMV_OK) return cs;
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
  if (!valid_dtype(dtype)) return fail(CBSPMV_EINVAL, "bad dtype");
  if (m < 0 || n < 0 || nnz < 0 || (m > 0 && !row_ptr)) return fail(CBSPMV_EINVAL, "bad CSR");
  cb::Csr A{m, n, nnz, row_ptr, col_idx, vals, val_bytes(dtype)};
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

cbspmv_status_t cbspmv_export_panel(cbspmv_handle_t h, int32_t k, cbspmv_export_t *ex) {
  if (!h || !ex) return fail(CBSPMV_EINVAL, "null argument");
  if (k < 0 || k >= (int32_t)h->parts.size()) return fail(CBSPMV_EINVAL, "panel index out of range");
  if (!h->has_host) return fail(CBSPMV_EUNSUPPORTED, "built with keep_host = 0");
  const cb::Canon &c = h->parts[k].canon;
  ex->nb = c.nb; ex->T = c.T; ex->mtx_bytes = (int64_t)c.mtx.size();
  ex->n_restore = (int64_t)c.restore.size(); ex->n_cols_offset = (int64_t)c.cols_offset.size();
  ex->blk_row_idx = c.br.data(); ex->blk_col_idx = c.bc.data(); ex->nnz_per_blk = c.nnzb.data();
  ex->type_per_blk = c.type.data(); ex->vp_per_blk = c.vp.data(); ex->mtx_data = c.mtx.data();
  ex->restore_cols = c.restore.empty() ? nullptr : c.restore.data();
  ex->cols_offset = c.cols_offset.empty() ? nullptr : c.cols_offset.data();
  ex->tb_ptr = c.tb_ptr.data(); ex->tb_load = c.tb_load.data(); ex->tb_load_natural = c.tb_load_nat.data();
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_export(cbspmv_handle_t h, cbspmv_export_t *ex) { return cbspmv_export_panel(h, 0, ex); }

cbspmv_status_t cbspmv_download_stream(cbspmv_handle_t h, void *stream_host, size_t stream_bytes,
                                       uint64_t *page_off_host, size_t n_page_off) {
  if (!h) return fail(CBSPMV_EINVAL, "null handle");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if (h->parts.size() != 1) return fail(CBSPMV_EUNSUPPORTED, "multi-panel handle");
  const Part &p = h->parts[0];
  if (stream_bytes < (size_t)p.stream_bytes || n_page_off < (size_t)p.n_pages + 1)
    return fail(CBSPMV_EDIM, "destination too small");
  DeviceGuard g(h->device);
  cudaError_t e = cudaSuccess;
  if (p.stream_bytes) e = cudaMemcpy(stream_host, p.d_stream, (size_t)p.stream_bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(page_off_host, p.d_page_off, ((size_t)p.n_pages + 1) * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_hot_columns(cbspmv_handle_t h, int32_t k, uint32_t *cols_host, size_t n_cols,
                                   int64_t *n_hot) {
  if (!h || !n_hot) return fail(CBSPMV_EINVAL, "null argument");
  if (h->device < 0) return fail(CBSPMV_EUNSUPPORTED, "host-only handle");
  if (k < 0 || k >= (int32_t)h->parts.size()) return fail(CBSPMV_EINVAL, "panel out of range");
  const Part &p = h->parts[(size_t)k];
  *n_hot = p.n_hot;
  if (p.n_hot == 0 || (!cols_host && n_cols == 0)) return CBSPMV_OK;  // count query
  if (!cols_host || n_cols < (size_t)p.n_hot) return fail(CBSPMV_EDIM, "destination too small");
  DeviceGuard g(h->device);
  cudaError_t e = cudaMemcpy(cols_host, p.d_hot, (size_t)p.n_hot * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { cudaGetLastError(); return fail(CBSPMV_ECUDA, cudaGetErrorString(e)); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_destroy(cbspmv_handle_t h) {
  if (!h) return CBSPMV_OK;
  free_device(h);
  delete h;
  return CBSPMV_OK;
}

// ------------------------------------------------------------------ files
cbspmv_status_t cbspmv_mm_read(const char *path, cbspmv_csr_t *out) {
  if (!path || !out) return fail(CBSPMV_EINVAL, "null argument");
  std::memset(out, 0, sizeof(*out));
  try {
    std::string err;
    int st = cb::mm_read(path, 0, out, &err);
    if (st != CBSPMV_OK) return fail(st, err);
  } catch (const std::bad_alloc &) {
    cbspmv_csr_free(out);
    return fail(CBSPMV_ENOMEM, "host allocation while reading the file");
  }
  g_err.clear();
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_mm_write(const char *path, int64_t m, int64_t n, const int64_t *row_ptr,
                                const int32_t *col_idx, const double *vals) {
  if (!path || m < 0 || n < 0 || (m > 0 && !row_ptr)) return fail(CBSPMV_EINVAL, "bad arguments");
  if (m > 0 && row_ptr[m] > 0 && (!col_idx || !vals)) return fail(CBSPMV_EINVAL, "null col_idx / vals");
  try {
    std::string err;
    int st = cb::mm_write(path, m, n, row_ptr, col_idx, vals, &err);
    if (st != CBSPMV_OK) return fail(st, err);
  } catch (const std::bad_alloc &) {
    return fail(CBSPMV_ENOMEM, "host allocation while writing the file");
  }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_csr_free(cbspmv_csr_t *csr) {
  if (!csr) return CBSPMV_OK;
  std::free(csr->row_ptr); std::free(csr->col_idx); std::free(csr->vals);
  csr->row_ptr = nullptr; csr->col_idx = nullptr; csr->vals = nullptr;
  csr->m = csr->n = csr->nnz = 0;
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_save(cbspmv_handle_t h, const char *path) {
  if (!h || !path) return fail(CBSPMV_EINVAL, "null argument");
  if (!h->has_host) return fail(CBSPMV_EUNSUPPORTED, "built with keep_host = 0");
  FILE *f = std::fopen(path, "wb");
  if (!f) return fail(CBSPMV_EIO, std::string("cannot open ") + path + " for writing");
  std::string err;
  int st = CBSPMV_OK;
  try {
    for (size_t k = 0; k < h->parts.size() && st == CBSPMV_OK; k++) {
      cb::CbsmExt x;
      x.dtype = h->dtype; x.panel = (int)k; x.n_panels = (int)h->parts.size();
      x.c0 = h->parts[k].c0; x.c1 = h->parts[k].c1;
      st = cb::write_cbsm(f, h->parts[k].canon, x, &err);
    }
  } catch (const std::bad_alloc &) {
    st = CBSPMV_ENOMEM; err = "host allocation while saving";
  }
  if (std::fclose(f) != 0 && st == CBSPMV_OK) { st = CBSPMV_EIO; err = "write failed"; }
  if (st != CBSPMV_OK) { std::remove(path); return fail(st, err); }
  return CBSPMV_OK;
}

cbspmv_status_t cbspmv_load(const char *path, const cbspmv_options_t *opts, void *stream, cbspmv_handle_t *out) {
  if (!out || !path) return fail(CBSPMV_EINVAL, "null argument");
  *out = nullptr;
  cbspmv_options_t o;
  cbspmv_default_options(&o);
  if (opts) {
    if (opts->struct_size != sizeof(cbspmv_options_t)) return fail(CBSPMV_EINVAL, "options struct_size mismatch");
    o = *opts;
  }
  FILE *f = std::fopen(path, "rb");
  if (!f) return fail(CBSPMV_EIO, std::string("cannot open ") + path);
  cbspmv_s *h = new (std::nothrow) cbspmv_s();
  if (!h) { std::fclose(f); return fail(CBSPMV_ENOMEM, "handle allocation"); }
  std::string err;
  int st = CBSPMV_OK;
  const double t0 = now();
  double t_up = 0.0;
  int64_t m = 0, n = 0;
  try {
    if (o.device >= 0) {
      int ndev = 0;
      if (cudaGetDeviceCount(&ndev) != cudaSuccess || o.device >= ndev) {
        cudaGetLastError();
        st = CBSPMV_ECUDA; err = "no CUDA device " + std::to_string(o.device);
      }
      h->device = o.device;
    }
    DeviceGuard guard(st == CBSPMV_OK ? o.device : -1);
    int n_panels = 1;
    for (int k = 0; st == CBSPMV_OK && k < n_panels; k++) {
      Part P;
      cb::CbsmExt x;
      st = cb::read_cbsm(f, &P.canon, &x, &err);
      if (st != CBSPMV_OK) break;
      if (k == 0) {
        n_panels = x.n_panels; m = P.canon.m; n = P.canon.n;
        h->dtype = x.dtype; h->val_size = val_bytes(x.dtype); h->vec_size = vec_bytes(x.dtype);
      } else if (x.panel != k || x.n_panels != n_panels || x.dtype != h->dtype || P.canon.m != m || P.canon.n != n ||
                 x.c0 != h->parts.back().c1) {
        st = CBSPMV_EFORMAT; err = "inconsistent column panel " + std::to_string(k);
        break;
      }
      if (x.panel != k) { st = CBSPMV_EFORMAT; err = "panel index out of order"; break; }
      P.c0 = x.c0; P.c1 = x.c1;
      h->parts.push_back(std::move(P));
      if (o.device >= 0) st = upload_part(o, h->dtype, reinterpret_cast<cudaStream_t>(stream), &h->parts.back(), &t_up, &err);
    }
    if (st == CBSPMV_OK && (h->parts.empty() || h->parts.back().c1 != n || h->parts.front().c0 != 0)) {
      st = CBSPMV_EFORMAT; err = "column panels do not cover [0, n)";
    }
  } catch (const std::bad_alloc &) {
    st = CBSPMV_ENOMEM; err = "host allocation while loading";
  }
  std::fclose(f);
  if (st != CBSPMV_OK) { free_device(h); delete h; return fail(st, err); }
  fill_info(h, m, n, t0, t_up, o.keep_host != 0);
  *out = h;
  g_err.clear();
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
    case CBSPMV_EIO: return "CBSPMV_EIO";
    case CBSPMV_EFORMAT: return "CBSPMV_EFORMAT";
  }
  return "unknown status";
}

const char *cbspmv_last_error(void) { return g_err.c_str(); }

int32_t cbspmv_version(void) { return CBSPMV_VERSION; }

}  // extern "C"
