// container.cpp — the CBSM file container of the canonical format, so a matrix
// is preprocessed once and reloaded without re-running a1..a7 (the paper's preprocessing is a
// one-off cost amortised over iterations).
//
// Layout, all little-endian, one container per column panel, back to back:
//   "CBSM", u32 version = 1, u64 n_rows, u64 n_cols, u64 block_count, u64 mtx_data_len,
//   u8 has_agg, u8 has_schedule,
//   u32 blk_row_idx[nb], u32 blk_col_idx[nb], u32 nnz_per_blk[nb], u8 type_per_blk[nb],
//   u64 vp_per_blk[nb],
//   if has_agg: u64 cols_offset[blk_m + 1], u32 restore_cols[cols_offset[blk_m]],
//   u8 mtx_data[mtx_data_len]
// followed by this library's extension block (absent in files written by other programs):
//   "CBX1", u32 dtype, u32 warps_per_tb, u32 panel, u32 n_panels, u64 c0, u64 c1, u64 nnz,
//   u64 nb_pre, u64 ss_count, u64 T, i64 tb_ptr[T + 1], i64 tb_load[T], i64 tb_load_natural[T].
// Without the extension, a file is read as one fp64 panel whose thread blocks are consecutive
// groups of 8 blocks (any grouping is a valid schedule; Alg. 2 only balances it).
//
// The kernels trust the format's indices, so every loaded record is decoded and checked
// (validate_canon) before it can reach a device.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "cb_internal.h"
#include "cbspmv.h"

namespace cb {
namespace {

constexpr char kMagic[4] = {'C', 'B', 'S', 'M'};
constexpr char kExtMagic[4] = {'C', 'B', 'X', '1'};
constexpr uint32_t kVersion = 1;

struct Writer {
  FILE *f;
  bool ok = true;
  void bytes(const void *p, size_t n) {
    if (ok && n) ok = std::fwrite(p, 1, n, f) == n;
  }
  template <class T> void put(T v) { bytes(&v, sizeof(v)); }  // hosts are little-endian (x86-64 / aarch64)
  template <class Dst, class Src> void array(const Src *p, size_t n) {
    std::vector<Dst> tmp;
    const size_t chunk = 1 << 16;
    for (size_t i = 0; i < n && ok; i += chunk) {
      size_t k = std::min(chunk, n - i);
      tmp.resize(k);
      for (size_t j = 0; j < k; j++) tmp[j] = (Dst)p[i + j];
      bytes(tmp.data(), k * sizeof(Dst));
    }
  }
};

struct Reader {
  FILE *f;
  bool ok = true;
  bool bytes(void *p, size_t n) {
    if (ok && n) ok = std::fread(p, 1, n, f) == n;
    return ok;
  }
  template <class T> T get() {
    T v{};
    bytes(&v, sizeof(v));
    return v;
  }
  template <class Src, class Dst> bool array(Dst *p, size_t n) {
    std::vector<Src> tmp;
    const size_t chunk = 1 << 16;
    for (size_t i = 0; i < n && ok; i += chunk) {
      size_t k = std::min(chunk, n - i);
      tmp.resize(k);
      if (!bytes(tmp.data(), k * sizeof(Src))) break;
      for (size_t j = 0; j < k; j++) p[i + j] = (Dst)tmp[j];
    }
    return ok;
  }
};

inline int64_t rec_bytes(int type, int64_t k, int64_t B, int64_t S) {  // a6 record size (R-8)
  int64_t idx = type == CBSPMV_FMT_COO ? k : type == CBSPMV_FMT_CSR ? (B + 1) + k : 0;
  int64_t p = idx % S;
  return idx + (p ? S - p : 0) + (type == CBSPMV_FMT_DENSE ? B * B : k) * S;
}

}  // namespace

int write_cbsm(FILE *f, const Canon &c, const CbsmExt &x, std::string *err) {
  if (c.blk != 16) { *err = "the CBSM container stores 16x16 blocks only"; return CBSPMV_EUNSUPPORTED; }
  Writer w{f};
  w.bytes(kMagic, 4);
  w.put<uint32_t>(kVersion);
  w.put<uint64_t>((uint64_t)c.m); w.put<uint64_t>((uint64_t)c.n);
  w.put<uint64_t>((uint64_t)c.nb); w.put<uint64_t>((uint64_t)c.mtx.size());
  w.put<uint8_t>(c.agg ? 1 : 0); w.put<uint8_t>(1);
  const size_t nb = (size_t)c.nb;
  w.array<uint32_t>(c.br.data(), nb);
  w.array<uint32_t>(c.bc.data(), nb);
  w.array<uint32_t>(c.nnzb.data(), nb);
  w.bytes(c.type.data(), nb);
  w.bytes(c.vp.data(), nb * 8);
  if (c.agg) {
    w.bytes(c.cols_offset.data(), c.cols_offset.size() * 8);
    w.bytes(c.restore.data(), c.restore.size() * 4);
  }
  w.bytes(c.mtx.data(), c.mtx.size());
  w.bytes(kExtMagic, 4);
  w.put<uint32_t>((uint32_t)x.dtype); w.put<uint32_t>((uint32_t)c.W);
  w.put<uint32_t>((uint32_t)x.panel); w.put<uint32_t>((uint32_t)x.n_panels);
  w.put<uint64_t>((uint64_t)x.c0); w.put<uint64_t>((uint64_t)x.c1);
  w.put<uint64_t>((uint64_t)c.nnz); w.put<uint64_t>((uint64_t)c.nb_pre); w.put<uint64_t>((uint64_t)c.ss_count);
  w.put<uint64_t>((uint64_t)c.T);
  w.bytes(c.tb_ptr.data(), c.tb_ptr.size() * 8);
  w.bytes(c.tb_load.data(), c.tb_load.size() * 8);
  w.bytes(c.tb_load_nat.data(), c.tb_load_nat.size() * 8);
  if (!w.ok) { *err = "write failed"; return CBSPMV_EIO; }
  return CBSPMV_OK;
}

int read_cbsm(FILE *f, Canon *out, CbsmExt *x, std::string *err) {
  Reader r{f};
  char magic[4];
  if (!r.bytes(magic, 4) || std::memcmp(magic, kMagic, 4) != 0) {
    *err = "bad magic: not a CBSM container";
    return CBSPMV_EFORMAT;
  }
  const uint32_t version = r.get<uint32_t>();
  if (r.ok && version != kVersion) { *err = "unsupported CBSM version " + std::to_string(version); return CBSPMV_EFORMAT; }
  Canon &c = *out;
  c = Canon();
  c.blk = 16;
  const uint64_t m = r.get<uint64_t>(), n = r.get<uint64_t>(), nb = r.get<uint64_t>(), mlen = r.get<uint64_t>();
  const uint8_t has_agg = r.get<uint8_t>(), has_sched = r.get<uint8_t>();
  if (!r.ok) { *err = "truncated CBSM header"; return CBSPMV_EFORMAT; }
  if (m > (uint64_t)UINT32_MAX || n > (uint64_t)INT32_MAX || nb > (m / 16 + 1) * (n / 16 + 1) || has_agg > 1 ||
      has_sched > 1 || mlen > nb * (uint64_t)(256 * 8 + 64)) {
    *err = "implausible CBSM header fields";
    return CBSPMV_EFORMAT;
  }
  c.m = (int64_t)m; c.n = (int64_t)n; c.nb = (int64_t)nb; c.agg = has_agg;
  c.blk_m = (c.m + 15) / 16;
  c.br.resize(nb); c.bc.resize(nb); c.nnzb.resize(nb); c.type.resize(nb); c.vp.resize(nb);
  r.array<uint32_t>(c.br.data(), nb);
  r.array<uint32_t>(c.bc.data(), nb);
  r.array<uint32_t>(c.nnzb.data(), nb);
  r.bytes(c.type.data(), nb);
  r.bytes(c.vp.data(), nb * 8);
  if (has_agg && r.ok) {
    c.cols_offset.resize((size_t)c.blk_m + 1);
    r.bytes(c.cols_offset.data(), c.cols_offset.size() * 8);
    const uint64_t nres = c.cols_offset.back();
    if (r.ok && nres > 256 * nb) { *err = "implausible restore_cols length"; return CBSPMV_EFORMAT; }
    c.restore.resize((size_t)nres);
    r.bytes(c.restore.data(), c.restore.size() * 4);
  }
  c.mtx.resize((size_t)mlen);
  r.bytes(c.mtx.data(), mlen);
  if (!r.ok) { *err = "truncated CBSM arrays"; return CBSPMV_EFORMAT; }
  for (uint8_t t : c.type)
    if (t > CBSPMV_FMT_DENSE) { *err = "bad type_per_blk entry"; return CBSPMV_EFORMAT; }
  for (int k = 0; k < 3; k++) c.fmt_count[k] = 0;
  for (uint8_t t : c.type) c.fmt_count[t]++;

  // extension block (optional)
  *x = CbsmExt();
  char em[4];
  const long here = std::ftell(f);
  if (std::fread(em, 1, 4, f) == 4 && std::memcmp(em, kExtMagic, 4) == 0) {
    x->dtype = (int)r.get<uint32_t>();
    c.W = (int)r.get<uint32_t>();
    x->panel = (int)r.get<uint32_t>(); x->n_panels = (int)r.get<uint32_t>();
    x->c0 = (int64_t)r.get<uint64_t>(); x->c1 = (int64_t)r.get<uint64_t>();
    c.nnz = (int64_t)r.get<uint64_t>(); c.nb_pre = (int64_t)r.get<uint64_t>(); c.ss_count = (int64_t)r.get<uint64_t>();
    const uint64_t T = r.get<uint64_t>();
    if (!r.ok || T > nb + 1 || (nb > 0 && T == 0)) { *err = "bad CBSM extension header"; return CBSPMV_EFORMAT; }
    c.T = (int64_t)T;
    c.tb_ptr.resize((size_t)T + 1); c.tb_load.resize((size_t)T); c.tb_load_nat.resize((size_t)T);
    r.bytes(c.tb_ptr.data(), c.tb_ptr.size() * 8);
    r.bytes(c.tb_load.data(), c.tb_load.size() * 8);
    r.bytes(c.tb_load_nat.data(), c.tb_load_nat.size() * 8);
    if (!r.ok) { *err = "truncated CBSM extension"; return CBSPMV_EFORMAT; }
    if (x->dtype != CBSPMV_F64 && x->dtype != CBSPMV_F32 && x->dtype != CBSPMV_F32F64) {
      *err = "bad dtype in CBSM extension";
      return CBSPMV_EFORMAT;
    }
  } else {
    if (here >= 0) std::fseek(f, here, SEEK_SET);
    std::clearerr(f);
    x->dtype = CBSPMV_F64; x->panel = 0; x->n_panels = 1; x->c0 = 0; x->c1 = c.n;
    c.W = 8;
    c.T = (c.nb + c.W - 1) / c.W;
    c.tb_ptr.resize((size_t)c.T + 1);
    for (int64_t t = 0; t <= c.T; t++) c.tb_ptr[(size_t)t] = std::min<int64_t>(c.nb, t * c.W);
    c.nnz = 0;
    for (int32_t k : c.nnzb) c.nnz += k;
    c.nb_pre = 0; c.ss_count = 0;
    c.tb_load.assign((size_t)c.T, 0);
    for (int64_t t = 0; t < c.T; t++)
      for (int64_t i = c.tb_ptr[(size_t)t]; i < c.tb_ptr[(size_t)t + 1]; i++) c.tb_load[(size_t)t] += c.nnzb[(size_t)i];
    c.tb_load_nat = c.tb_load;
  }
  c.val_size = x->dtype == CBSPMV_F64 ? 8 : 4;
  return validate_canon(c, *x, err);
}

// Decode every record and check each index the kernels will use.
int validate_canon(const Canon &c, const CbsmExt &x, std::string *err) {
  const int64_t B = 16, S = c.val_size, nb = c.nb;
  auto bad = [&](const std::string &what, int64_t i) {
    *err = "invalid CBSM content: " + what + (i >= 0 ? " (block " + std::to_string(i) + ")" : "");
    return CBSPMV_EFORMAT;
  };
  if (x.n_panels < 1 || x.panel < 0 || x.panel >= x.n_panels || x.c0 < 0 || x.c0 > x.c1 || x.c1 > c.n)
    return bad("panel fields", -1);
  if ((int64_t)c.tb_ptr.size() != c.T + 1 || c.tb_ptr[0] != 0 || c.tb_ptr[(size_t)c.T] != nb)
    return bad("tb_ptr", -1);
  for (int64_t t = 0; t < c.T; t++)
    if (c.tb_ptr[(size_t)t + 1] < c.tb_ptr[(size_t)t]) return bad("tb_ptr not monotone", -1);
  if (c.W < 1 || c.W > 1024) return bad("warps_per_tb", -1);
  if (c.agg) {
    if ((int64_t)c.cols_offset.size() != c.blk_m + 1 || c.cols_offset[0] != 0) return bad("cols_offset", -1);
    for (int64_t b = 0; b < c.blk_m; b++)
      if (c.cols_offset[(size_t)b + 1] < c.cols_offset[(size_t)b]) return bad("cols_offset not monotone", -1);
    for (uint32_t col : c.restore)
      if ((int64_t)col >= c.n) return bad("restore_cols entry >= n", -1);
  }
  int64_t nnz = 0;
  for (int64_t i = 0; i < nb; i++) {
    const int64_t br = c.br[(size_t)i], bc = c.bc[(size_t)i], k = c.nnzb[(size_t)i];
    const int type = c.type[(size_t)i];
    if (br < 0 || br >= c.blk_m) return bad("blk_row_idx out of range", i);
    if (k < 1 || k > B * B) return bad("nnz_per_blk out of [1, 256]", i);
    nnz += k;
    // column count of the block's x tile
    int64_t ncols;
    if (c.agg) {
      const int64_t w = (int64_t)(c.cols_offset[(size_t)br + 1] - c.cols_offset[(size_t)br]) - bc * B;
      if (bc < 0 || w <= 0) return bad("aggregated block column out of range", i);
      ncols = std::min(B, w);
    } else {
      if (bc < 0 || bc * B >= c.n) return bad("blk_col_idx out of range", i);
      ncols = std::min(B, c.n - bc * B);
    }
    const int64_t nrows = std::min(B, c.m - br * B);
    const uint64_t vp = c.vp[(size_t)i];
    const int64_t sz = rec_bytes(type, k, B, S);
    if (vp % (uint64_t)S != 0 || vp > c.mtx.size() || (uint64_t)sz > c.mtx.size() - vp) return bad("record out of mtx_data", i);
    const uint8_t *rec = c.mtx.data() + vp;
    if (type == CBSPMV_FMT_COO) {
      for (int64_t e = 0; e < k; e++) {
        const int lr = rec[e] & 15, lc = rec[e] >> 4;
        if (lr >= nrows || lc >= ncols) return bad("COO coordinate outside the matrix", i);
      }
    } else if (type == CBSPMV_FMT_CSR) {
      if (rec[0] != 0 || rec[16] != (uint8_t)(k & 0xFF)) return bad("CSR row_ptr ends", i);
      int prev = 0;
      for (int r = 1; r < 16; r++) {
        if (rec[r] < prev || rec[r] > k) return bad("CSR row_ptr not monotone", i);
        prev = rec[r];
      }
      for (int r = 0; r < 16; r++) {
        const int lo = rec[r], hi = r < 15 ? rec[r + 1] : (int)k;
        if (hi > lo && r >= nrows) return bad("CSR row outside the matrix", i);
      }
      for (int64_t e = 0; e < k; e++)
        if (rec[17 + e] >= ncols || rec[17 + e] > 15) return bad("CSR column outside the matrix", i);
    } else {  // DENSE: entries outside the matrix must be zero
      for (int64_t r = 0; r < B; r++)
        for (int64_t cc = 0; cc < B; cc++) {
          if (r < nrows && cc < ncols) continue;
          const uint8_t *v = rec + (r * B + cc) * S;
          for (int64_t q = 0; q < S; q++)
            if (v[q] != 0) return bad("DENSE value outside the matrix", i);
        }
    }
  }
  if (c.nnz != nnz) return bad("nnz does not match nnz_per_blk", -1);
  return CBSPMV_OK;
}

}  // namespace cb
