// mmio.cpp — Matrix Market coordinate files <-> canonical host CSR (the matio module of the
// specification; the paper's inputs are SuiteSparse Matrix Market files).
//
// Reading: banner "%%MatrixMarket matrix coordinate <real|double|integer|pattern>
// <general|symmetric|skew-symmetric|hermitian>", '%' comments, the size line "M N L", then L
// entry lines "i j [v]" with 1-based indices.  Entries are parsed in parallel chunks split at
// line boundaries.  Canonicalisation: symmetric / hermitian (real) entries off the
// diagonal are mirrored, skew-symmetric mirrors are negated; pattern entries get 1.0; duplicates
// are summed in file order (each file entry, then its mirror); entries that are exactly 0 after
// summation are dropped; rows are sorted by column.  Complex fields and the array format are
// rejected.
// Writing: "real general", shortest round-trip decimal form of every value (std::to_chars), so
// parse(write(A)) == A bit for bit.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cb_internal.h"
#include "cbspmv.h"

namespace cb {
namespace {

struct Entry {
  int64_t r, c;
  double v;
};

inline bool is_space(char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }

const char *skip_ws(const char *p, const char *e) {
  while (p < e && is_space(*p)) p++;
  return p;
}

bool parse_i64(const char *&p, const char *e, int64_t *out) {
  p = skip_ws(p, e);
  auto r = std::from_chars(p, e, *out);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}

bool parse_f64(const char *&p, const char *e, double *out) {
  p = skip_ws(p, e);
  if (p < e && *p == '+') p++;  // from_chars does not accept a leading '+'
  auto r = std::from_chars(p, e, *out, std::chars_format::general);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}

std::string lower(std::string s) {
  for (char &ch : s) ch = (char)std::tolower((unsigned char)ch);
  return s;
}

}  // namespace

int mm_read(const char *path, int threads, cbspmv_csr_t *out, std::string *err) {
  FILE *f = std::fopen(path, "rb");
  if (!f) { *err = std::string("cannot open ") + path; return CBSPMV_EIO; }
  std::fseek(f, 0, SEEK_END);
  long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  std::vector<char> buf((size_t)std::max(sz, 0L) + 1);
  size_t got = sz > 0 ? std::fread(buf.data(), 1, (size_t)sz, f) : 0;
  std::fclose(f);
  if (sz < 0 || got != (size_t)sz) { *err = std::string("cannot read ") + path; return CBSPMV_EIO; }
  buf[(size_t)sz] = '\n';
  const char *p = buf.data(), *end = buf.data() + sz + 1;

  // banner
  const char *nl = (const char *)std::memchr(p, '\n', (size_t)(end - p));
  std::string banner(p, nl);
  std::vector<std::string> tok;
  {
    size_t i = 0;
    while (i < banner.size()) {
      while (i < banner.size() && std::isspace((unsigned char)banner[i])) i++;
      size_t j = i;
      while (j < banner.size() && !std::isspace((unsigned char)banner[j])) j++;
      if (j > i) tok.push_back(lower(banner.substr(i, j - i)));
      i = j;
    }
  }
  if (tok.size() != 5 || tok[0] != "%%matrixmarket" || tok[1] != "matrix") {
    *err = "malformed Matrix Market banner";
    return CBSPMV_EFORMAT;
  }
  if (tok[2] != "coordinate") { *err = "only the coordinate format is supported (got " + tok[2] + ")"; return CBSPMV_EUNSUPPORTED; }
  const std::string &field = tok[3], &sym = tok[4];
  if (field == "complex") { *err = "complex matrices are not supported"; return CBSPMV_EUNSUPPORTED; }
  if (field != "real" && field != "double" && field != "integer" && field != "pattern") {
    *err = "unknown field " + field;
    return CBSPMV_EFORMAT;
  }
  const bool pattern = field == "pattern";
  int mirror = 0;  // 0 general, 1 symmetric / hermitian, -1 skew-symmetric
  if (sym == "symmetric" || sym == "hermitian") mirror = 1;
  else if (sym == "skew-symmetric") mirror = -1;
  else if (sym != "general") { *err = "unknown symmetry " + sym; return CBSPMV_EFORMAT; }

  // comments, then the size line
  p = nl + 1;
  int64_t M = -1, N = -1, L = -1;
  while (p < end) {
    nl = (const char *)std::memchr(p, '\n', (size_t)(end - p));
    const char *q = skip_ws(p, nl);
    if (q == nl || *q == '%') { p = nl + 1; continue; }
    if (!parse_i64(q, nl, &M) || !parse_i64(q, nl, &N) || !parse_i64(q, nl, &L) || skip_ws(q, nl) != nl) {
      *err = "malformed size line";
      return CBSPMV_EFORMAT;
    }
    p = nl + 1;
    break;
  }
  if (M < 0 || N < 0 || L < 0) { *err = "missing or negative size line"; return CBSPMV_EFORMAT; }
  if (N > (int64_t)INT32_MAX) { *err = "n exceeds the int32 column index range"; return CBSPMV_EUNSUPPORTED; }
  if (mirror != 0 && M != N) { *err = "symmetric matrix is not square"; return CBSPMV_EFORMAT; }

  // entry lines: chunks split at newlines, counted, then parsed into their slots
  const int T = resolve_threads(threads);
  const int64_t body = end - p;
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(T * 4, body / (1 << 16)));
  std::vector<const char *> cut(nch + 1);
  cut[0] = p; cut[nch] = end;
  for (int k = 1; k < nch; k++) {
    const char *c = p + body * k / nch;
    if (c < cut[k - 1]) c = cut[k - 1];
    const char *n2 = (const char *)std::memchr(c, '\n', (size_t)(end - c));
    cut[k] = n2 ? n2 + 1 : end;
  }
  std::vector<int64_t> cnt(nch + 1, 0);
  parallel_for(nch, T, 1, [&](int64_t a, int64_t b, int) {
    for (int64_t k = a; k < b; k++) {
      int64_t c = 0;
      for (const char *s = cut[k]; s < cut[k + 1];) {
        const char *e = (const char *)std::memchr(s, '\n', (size_t)(cut[k + 1] - s));
        if (!e) e = cut[k + 1];
        const char *q = skip_ws(s, e);
        if (q != e && *q != '%') c++;
        s = e + 1;
      }
      cnt[k + 1] = c;
    }
  });
  for (int k = 0; k < nch; k++) cnt[k + 1] += cnt[k];
  if (cnt[nch] != L) {
    *err = "entry count mismatch: size line declares " + std::to_string(L) + ", file has " + std::to_string(cnt[nch]);
    return CBSPMV_EFORMAT;
  }
  std::vector<Entry> ent((size_t)L);
  std::vector<int64_t> bad(nch, -1);  // first bad entry index per chunk
  std::vector<int> why(nch, 0);
  parallel_for(nch, T, 1, [&](int64_t a, int64_t b, int) {
    for (int64_t k = a; k < b; k++) {
      int64_t idx = cnt[k];
      for (const char *s = cut[k]; s < cut[k + 1] && bad[k] < 0;) {
        const char *e = (const char *)std::memchr(s, '\n', (size_t)(cut[k + 1] - s));
        if (!e) e = cut[k + 1];
        const char *q = skip_ws(s, e);
        if (q != e && *q != '%') {
          Entry &en = ent[(size_t)idx];
          double v = 1.0;
          bool ok = parse_i64(q, e, &en.r) && parse_i64(q, e, &en.c);
          if (ok && !pattern) ok = parse_f64(q, e, &v);
          if (ok) ok = skip_ws(q, e) == e;
          if (!ok) { bad[k] = idx; why[k] = 1; break; }
          if (en.r < 1 || en.r > M || en.c < 1 || en.c > N) { bad[k] = idx; why[k] = 2; break; }
          if (!std::isfinite(v)) { bad[k] = idx; why[k] = 3; break; }
          en.r -= 1; en.c -= 1; en.v = v;
          idx++;
        }
        s = e + 1;
      }
    }
  });
  for (int k = 0; k < nch; k++)
    if (bad[k] >= 0) {
      static const char *w[] = {"", "malformed entry", "index out of declared bounds", "non-finite value"};
      *err = std::string(w[why[k]]) + " at entry " + std::to_string(bad[k] + 1);
      return why[k] == 1 ? CBSPMV_EFORMAT : (why[k] == 2 ? CBSPMV_EFORMAT : CBSPMV_EINVAL);
    }

  // expansion order: each file entry, then its mirror (defines the duplicate-summation order)
  std::vector<int64_t> row_cnt((size_t)M + 1, 0);
  int64_t total = 0;
  for (const Entry &en : ent) {
    row_cnt[(size_t)en.r + 1]++;
    total++;
    if (mirror != 0 && en.r != en.c) { row_cnt[(size_t)en.c + 1]++; total++; }
  }
  for (int64_t i = 0; i < M; i++) row_cnt[(size_t)i + 1] += row_cnt[(size_t)i];
  struct Item { int64_t c; int64_t ord; double v; };
  std::vector<Item> items((size_t)total);
  {
    std::vector<int64_t> pos(row_cnt.begin(), row_cnt.end() - 1);
    int64_t ord = 0;
    for (const Entry &en : ent) {
      items[(size_t)pos[(size_t)en.r]++] = {en.c, ord++, en.v};
      if (mirror != 0 && en.r != en.c) items[(size_t)pos[(size_t)en.c]++] = {en.r, ord++, mirror * en.v};
    }
  }
  std::vector<Entry>().swap(ent);
  // per row: stable order by column, sum duplicates left to right, drop exact zeros
  std::vector<int64_t> keep((size_t)M + 1, 0);
  parallel_for(M, T, 4096, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; i++) {
      Item *s = items.data() + row_cnt[(size_t)i], *e = items.data() + row_cnt[(size_t)i + 1];
      std::sort(s, e, [](const Item &x, const Item &y) { return x.c < y.c || (x.c == y.c && x.ord < y.ord); });
      Item *w = s;
      for (Item *r = s; r < e;) {
        Item acc = *r++;
        while (r < e && r->c == acc.c) acc.v += (r++)->v;
        if (acc.v != 0.0) *w++ = acc;
      }
      keep[(size_t)i + 1] = w - s;
    }
  });
  for (int64_t i = 0; i < M; i++) keep[(size_t)i + 1] += keep[(size_t)i];
  const int64_t nnz = keep[(size_t)M];
  out->m = M; out->n = N; out->nnz = nnz;
  out->row_ptr = (int64_t *)std::malloc(sizeof(int64_t) * ((size_t)M + 1));
  out->col_idx = (int32_t *)std::malloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1));
  out->vals = (double *)std::malloc(sizeof(double) * (size_t)std::max<int64_t>(nnz, 1));
  if (!out->row_ptr || !out->col_idx || !out->vals) {
    std::free(out->row_ptr); std::free(out->col_idx); std::free(out->vals);
    out->row_ptr = nullptr; out->col_idx = nullptr; out->vals = nullptr;
    *err = "host allocation of the CSR failed";
    return CBSPMV_ENOMEM;
  }
  std::memcpy(out->row_ptr, keep.data(), sizeof(int64_t) * ((size_t)M + 1));
  parallel_for(M, T, 4096, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; i++) {
      const Item *s = items.data() + row_cnt[(size_t)i];
      for (int64_t k = keep[(size_t)i]; k < keep[(size_t)i + 1]; k++, s++) {
        out->col_idx[k] = (int32_t)s->c;
        out->vals[k] = s->v;
      }
    }
  });
  return CBSPMV_OK;
}

int mm_write(const char *path, int64_t m, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
             const double *vals, std::string *err) {
  FILE *f = std::fopen(path, "wb");
  if (!f) { *err = std::string("cannot open ") + path + " for writing"; return CBSPMV_EIO; }
  const int64_t nnz = m > 0 ? row_ptr[m] : 0;
  bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)m,
                         (long long)n, (long long)nnz) > 0;
  std::vector<char> line;
  std::string chunk;
  chunk.reserve(1 << 20);
  char tmp[96];
  for (int64_t i = 0; i < m && ok; i++)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
      char *const te = tmp + sizeof(tmp) - 1;  // room for the newline
      auto r1 = std::to_chars(tmp, te, (long long)(i + 1));
      if (r1.ec != std::errc() || r1.ptr == te) { ok = false; break; }
      *r1.ptr = ' ';
      auto r2 = std::to_chars(r1.ptr + 1, te, (long long)col_idx[k] + 1);
      if (r2.ec != std::errc() || r2.ptr == te) { ok = false; break; }
      *r2.ptr = ' ';
      auto r3 = std::to_chars(r2.ptr + 1, te, vals[k]);  // shortest round-trip form
      if (r3.ec != std::errc()) { ok = false; break; }
      *r3.ptr = '\n';
      chunk.append(tmp, r3.ptr + 1);
      if (chunk.size() > (1 << 20) - 128) {
        ok = std::fwrite(chunk.data(), 1, chunk.size(), f) == chunk.size();
        chunk.clear();
      }
    }
  if (ok && !chunk.empty()) ok = std::fwrite(chunk.data(), 1, chunk.size(), f) == chunk.size();
  if (std::fclose(f) != 0) ok = false;
  if (!ok) { *err = std::string("write failed: ") + path; return CBSPMV_EIO; }
  return CBSPMV_OK;
}

}  // namespace cb
