// builder.cpp — host format builder of CB-SpMV (the Fig. 7 pipeline),
// multi-threaded C++17.  Produces the canonical format byte-identical to the
// paper-literal oracle (tests/test_builder_parity.py) and the derived device
// page stream.
//
// Steps:
//   a1 canonical check + explicit-zero drop (R-19)
//   a2 partition into BxB sub-blocks, block-COO in (br, bc) order
//   a3 super-sparse fraction and the th0 decision (R-3..R-5)
//   a4 block-aware column aggregation per block row (R-6, R-7)
//   a5 format selection COO / CSR / DENSE (R-9, R-10)
//   a6 intra-block data aggregation: records, VP, padding (R-8, R-11)
//   a7 TB-Load-Balance, Alg. 2 (R-12..R-14), as a counting sort plus a
//      bucket queue keyed by (load, tb_id) — the same pop order as a binary min-heap.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <thread>

#include "cb_internal.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

namespace cb {

int resolve_threads(int t) {
  if (t > 0) return t;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 128u) : 1;
}

void parallel_for(int64_t n, int threads, int64_t grain, const std::function<void(int64_t, int64_t, int)> &fn) {
  if (n <= 0) return;
  threads = resolve_threads(threads);
  if (threads == 1 || n <= grain) { fn(0, n, 0); return; }
  std::atomic<int64_t> next{0};
  auto worker = [&](int tid) {
    for (;;) {
      int64_t lo = next.fetch_add(grain);
      if (lo >= n) break;
      fn(lo, std::min(n, lo + grain), tid);
    }
  };
  std::vector<std::thread> th;
  int T = (int)std::min<int64_t>(threads, (n + grain - 1) / grain);
  for (int t = 1; t < T; t++) th.emplace_back(worker, t);
  worker(0);
  for (auto &x : th) x.join();
}

namespace {

// Parallel loop over block rows in chunks of roughly equal nnz (power-law matrices put most
// non-zeros in a few block rows, which fixed-size chunks would hand to one thread).
void parallel_blockrows(const Csr &A, int B, int64_t blk_m, int threads,
                        const std::function<void(int64_t, int64_t, int)> &fn) {
  if (blk_m <= 0) return;
  const int T = resolve_threads(threads);
  const int64_t nnz = A.m > 0 ? A.row_ptr[A.m] : 0;
  const int64_t chunks = std::min<int64_t>(blk_m, (int64_t)T * 32);
  std::vector<int64_t> cut(1, 0);
  for (int64_t k = 1; k < chunks; k++) {
    // first block row whose starting nnz offset reaches k/chunks of the total (also bounded by rows)
    const int64_t target = nnz / chunks * k;
    int64_t lo = cut.back(), hi = blk_m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (A.row_ptr[std::min<int64_t>(A.m, mid * B)] < target) lo = mid + 1;
      else hi = mid;
    }
    const int64_t by_rows = blk_m * k / chunks;
    const int64_t c = std::max(cut.back(), std::min(lo, std::max(by_rows, cut.back())));
    if (c > cut.back()) cut.push_back(c);
  }
  cut.push_back(blk_m);
  const int64_t nch = (int64_t)cut.size() - 1;
  parallel_for(nch, T, 1, [&](int64_t a, int64_t b, int tid) {
    for (int64_t k = a; k < b; k++) fn(cut[k], cut[k + 1], tid);
  });
}

inline double get_val(const Csr &A, int64_t j) {
  return A.val_size == 8 ? ((const double *)A.val)[j] : (double)((const float *)A.val)[j];
}

// Element of one block row, sortable by (block column, local row, local column).
struct Key {
  uint64_t key;  // bcol << 8 | lr << 4 | lc
  int64_t j;     // CSR position of the value
  bool operator<(const Key &o) const { return key < o.key; }
};

// Per-thread scratch reused across block rows.
struct Scratch {
  std::vector<Key> keys;
  std::vector<uint32_t> cols;
  std::vector<uint32_t> slot;  // per element (indexed j - row_ptr[r0]): its bucket, ~0u for explicit zeros
  std::vector<uint32_t> cnt;   // per bucket: element count, then placement cursor
  struct Run { uint32_t bc, bucket, lr; int64_t j0, j1; };
  std::vector<Run> runs;       // no-agg: maximal same-block-column runs of each row, row-major
  std::vector<uint32_t> bcs;   // no-agg: sorted distinct block columns of the block row
};

// No aggregation: each row's columns are increasing, so its elements form runs of equal block
// column.  Sorting the (few) distinct run heads gives the block columns; a counting sort of the
// elements on their block column's index, filled row-major, gives the (bcol, lr, lc) order.
// Returns false (and does nothing more) when runs are not much rarer than elements (scattered
// rows): the caller then uses the merge below.
static bool block_row_keys_plain(const Csr &A, int B, int64_t r0, int64_t r1, Scratch &s) {
  s.runs.clear();
  s.bcs.clear();
  for (int64_t r = r0; r < r1; r++) {
    int64_t j = A.row_ptr[r], e = A.row_ptr[r + 1];
    while (j < e) {
      uint32_t bc = (uint32_t)(A.col[j] / B);
      int64_t j1 = j + 1;
      while (j1 < e && (uint32_t)(A.col[j1] / B) == bc) j1++;
      s.runs.push_back({bc, 0, (uint32_t)(r - r0), j, j1});
      s.bcs.push_back(bc);
      j = j1;
    }
  }
  int64_t total = A.row_ptr[r1] - A.row_ptr[r0];
  if (s.runs.size() > 64 && (int64_t)s.runs.size() * 4 > total) return false;
  std::sort(s.bcs.begin(), s.bcs.end());
  s.bcs.erase(std::unique(s.bcs.begin(), s.bcs.end()), s.bcs.end());
  s.cnt.assign(s.bcs.size() + 1, 0);
  const uint32_t *b0 = s.bcs.data(), *be = b0 + s.bcs.size();
  size_t k = 0;
  uint32_t lr = ~0u;
  const uint32_t *cur = b0;
  for (auto &run : s.runs) {
    if (run.lr != lr) { cur = b0; lr = run.lr; }  // new row: reset the monotone cursor
    cur = std::lower_bound(cur, be, run.bc);
    run.bucket = (uint32_t)(cur - b0);
    uint32_t nz = 0;
    for (int64_t j = run.j0; j < run.j1; j++) nz += get_val(A, j) != 0.0;
    s.cnt[run.bucket + 1] += nz;
    k += nz;
  }
  for (size_t b = 0; b < s.bcs.size(); b++) s.cnt[b + 1] += s.cnt[b];
  s.keys.resize(k);
  for (auto &run : s.runs) {
    uint64_t hi = ((uint64_t)run.bc << 8) | ((uint64_t)run.lr << 4);
    for (int64_t j = run.j0; j < run.j1; j++)
      if (get_val(A, j) != 0.0) s.keys[s.cnt[run.bucket]++] = {hi | (uint64_t)(A.col[j] % B), j};
  }
  return true;
}

// Collect the block row's non-zeros as keys sorted by (bcol, lr, lc); with aggregation, columns
// are replaced by their rank in C_i (sorted distinct columns of the block row) and C_i is
// left in s.cols.  The rows of a canonical CSR are column-sorted, so a B-way merge of the block
// row's rows visits its elements in column order: that yields each element's column rank (agg)
// or the index of its distinct block column (no agg), and a counting sort on that bucket, filled
// in row-major order, gives the (bcol, lr, lc) order in O(k log B) without a comparison sort.
void block_row_keys(const Csr &A, int B, int64_t br, bool agg, Scratch &s) {
  s.keys.clear();
  s.cols.clear();
  int64_t r0 = br * B, r1 = std::min<int64_t>(A.m, r0 + B);
  if (!agg && block_row_keys_plain(A, B, r0, r1, s)) return;
  int64_t base = A.row_ptr[r0], total = A.row_ptr[r1] - base;
  if (total == 0) return;
  s.slot.resize((size_t)total);
  struct Cur { uint32_t col; int32_t r; int64_t j; };
  Cur heap[32];
  int hn = 0;
  auto less = [](const Cur &a, const Cur &b) { return a.col < b.col || (a.col == b.col && a.r < b.r); };
  auto push = [&](Cur c) {
    int i = hn++;
    while (i > 0) {
      int p = (i - 1) >> 1;
      if (!less(c, heap[p])) break;
      heap[i] = heap[p]; i = p;
    }
    heap[i] = c;
  };
  auto sift_top = [&]() {  // heap[0] replaced; restore the heap property
    Cur c = heap[0];
    int i = 0;
    for (;;) {
      int l = 2 * i + 1;
      if (l >= hn) break;
      int m = (l + 1 < hn && less(heap[l + 1], heap[l])) ? l + 1 : l;
      if (!less(heap[m], c)) break;
      heap[i] = heap[m]; i = m;
    }
    heap[i] = c;
  };
  for (int64_t r = r0; r < r1; r++)
    if (A.row_ptr[r] < A.row_ptr[r + 1]) push({(uint32_t)A.col[A.row_ptr[r]], (int32_t)(r - r0), A.row_ptr[r]});
  uint32_t nbuck = 0, ndist = 0;
  uint64_t last_col = ~0ull, last_bc = ~0ull;
  while (hn > 0) {
    Cur c = heap[0];
    int64_t j = c.j;
    if (get_val(A, j) != 0.0) {
      if (agg) {
        if (c.col != last_col) { s.cols.push_back(c.col); last_col = c.col; ndist++; }
        s.slot[j - base] = ndist - 1;  // rank in C_i
      } else {
        uint64_t bc = c.col / (uint32_t)B;
        if (bc != last_bc) { last_bc = bc; nbuck++; }
        s.slot[j - base] = nbuck - 1;
      }
    } else {
      s.slot[j - base] = ~0u;
    }
    int64_t end = A.row_ptr[r0 + c.r + 1];
    if (j + 1 < end) {
      heap[0] = {(uint32_t)A.col[j + 1], c.r, j + 1};
    } else {
      heap[0] = heap[--hn];
    }
    if (hn > 0) sift_top();
  }
  if (agg) nbuck = (ndist + B - 1) / B;
  s.cnt.assign((size_t)nbuck + 1, 0);
  uint32_t div = agg ? (uint32_t)B : 1u;
  size_t k = 0;
  for (int64_t t = 0; t < total; t++)
    if (s.slot[t] != ~0u) { s.cnt[s.slot[t] / div + 1]++; k++; }
  for (uint32_t b = 0; b < nbuck; b++) s.cnt[b + 1] += s.cnt[b];
  s.keys.resize(k);
  for (int64_t r = r0; r < r1; r++) {
    uint64_t lr = (uint64_t)(r - r0);
    for (int64_t j = A.row_ptr[r]; j < A.row_ptr[r + 1]; j++) {
      uint32_t sl = s.slot[j - base];
      if (sl == ~0u) continue;
      uint64_t c = agg ? (uint64_t)sl : (uint64_t)A.col[j];
      s.keys[s.cnt[sl / div]++] = {((c / B) << 8) | (lr << 4) | (c % B), j};
    }
  }
}

inline int64_t padding(int64_t idx_bytes, int64_t S) {  // Alg. 3 lines 6-7
  int64_t p = idx_bytes % S;
  return p ? S - p : 0;
}

inline int select_format(int64_t nnz, const cbspmv_options_t &o) {  // P:439 (R-9)
  if (o.force_format >= 0) return o.force_format;
  if (nnz < o.th1) return CBSPMV_FMT_COO;
  if (nnz > o.th2) return CBSPMV_FMT_DENSE;
  return CBSPMV_FMT_CSR;
}

inline int64_t record_bytes(int type, int64_t nnz, int B, int64_t S) {  // a6 (R-8)
  int64_t idx = type == CBSPMV_FMT_COO ? nnz : type == CBSPMV_FMT_CSR ? (B + 1) + nnz : 0;
  int64_t nval = type == CBSPMV_FMT_DENSE ? (int64_t)B * B : nnz;
  return idx + padding(idx, S) + nval * S;
}

inline void put_val(uint8_t *dst, int64_t i, double v, int64_t S) {
  if (S == 8) std::memcpy(dst + 8 * i, &v, 8);
  else { float f = (float)v; std::memcpy(dst + 4 * i, &f, 4); }
}

// Pack one block's record at dst (cleared here first, so padding is zero); e = its keys (sorted),
// k = nnz.
void pack_record(const Csr &A, int B, int64_t S, int type, const Key *e, int64_t k, uint8_t *dst) {
  std::memset(dst, 0, (size_t)record_bytes(type, k, B, S));
  if (type == CBSPMV_FMT_COO) {
    for (int64_t t = 0; t < k; t++) {
      uint32_t lr = (e[t].key >> 4) & 15, lc = e[t].key & 15;
      dst[t] = (uint8_t)((lc << 4) | lr);  // row = b & 15, col = b >> 4
    }
    uint8_t *vals = dst + k + padding(k, S);
    for (int64_t t = 0; t < k; t++) put_val(vals, t, get_val(A, e[t].j), S);
  } else if (type == CBSPMV_FMT_CSR) {
    int64_t t = 0;
    for (int r = 0; r <= B; r++) {
      while (t < k && (int)((e[t].key >> 4) & 15) < r) t++;
      dst[r] = (uint8_t)(t & 0xFF);
    }
    for (int64_t q = 0; q < k; q++) dst[B + 1 + q] = (uint8_t)(e[q].key & 15);
    uint8_t *vals = dst + (B + 1) + k + padding((B + 1) + k, S);
    for (int64_t q = 0; q < k; q++) put_val(vals, q, get_val(A, e[q].j), S);
  } else {
    for (int64_t q = 0; q < k; q++) {
      int64_t pos = (int64_t)((e[q].key >> 4) & 15) * B + (int64_t)(e[q].key & 15);
      put_val(dst, pos, get_val(A, e[q].j), S);
    }
  }
}

}  // namespace

namespace {

int check_options(const Csr &A, const cbspmv_options_t &o, std::string *err) {
  const int B = o.blk, W = o.warps_per_tb;
  if (A.m < 0 || A.n < 0 || A.n > INT32_MAX || (B != 16 && B != 4) || W < 1 || W > 1024 ||
      (A.val_size != 4 && A.val_size != 8) || o.th0_den <= 0 || o.force_format < -1 || o.force_format > 2) {
    *err = "invalid dimensions or options";
    return CBSPMV_EINVAL;
  }
  if (A.m > 0 && (!A.row_ptr || (A.row_ptr[A.m] > 0 && (!A.col || !A.val)))) {
    *err = "null CSR array";
    return CBSPMV_EINVAL;
  }
  if (A.m > 0 && (A.row_ptr[0] != 0 || A.row_ptr[A.m] != A.nnz)) {
    *err = "row_ptr[0] must be 0 and row_ptr[m] must equal nnz";
    return CBSPMV_EINVAL;
  }
  return CBSPMV_OK;
}

// a1. canonical check; the first violation in row-major order decides the status (as a
// sequential scan would).  *nnz = stored non-zeros after dropping explicit zeros.
int canonical_check(const Csr &A, int threads, int64_t *nnz, std::string *err) {
  const int T = resolve_threads(threads);
  struct Fail { int64_t pos = INT64_MAX; int code = 0; int64_t row = -1; };
  std::vector<Fail> fails(T);
  std::vector<int64_t> part(T, 0);
  parallel_for(A.m, T, 1 << 14, [&](int64_t lo, int64_t hi, int tid) {
    Fail &f = fails[tid];
    int64_t acc = 0;
    for (int64_t i = lo; i < hi; i++) {
      int64_t b = A.row_ptr[i], e = A.row_ptr[i + 1];
      if (e < b) { if (b < f.pos) { f.pos = b; f.code = CBSPMV_EINVAL; f.row = i; } continue; }
      for (int64_t j = b; j < e; j++) {
        int code = 0;
        if (A.col[j] < 0 || A.col[j] >= A.n) code = CBSPMV_EINVAL;
        else if (j > b && A.col[j] <= A.col[j - 1]) code = CBSPMV_EUNSORTED;
        else if (!std::isfinite(get_val(A, j))) code = CBSPMV_EINVAL;
        if (code) { if (j < f.pos) { f.pos = j; f.code = code; f.row = i; } break; }
        if (get_val(A, j) != 0.0) acc++;
      }
    }
    part[tid] += acc;
  });
  Fail first;
  for (auto &f : fails) if (f.pos < first.pos) first = f;
  if (first.code) {
    *err = (first.code == CBSPMV_EUNSORTED ? "columns not strictly increasing in row "
                                           : "invalid entry (column out of range or non-finite) in row ") +
           std::to_string(first.row);
    return first.code;
  }
  *nnz = 0;
  for (int64_t v : part) *nnz += v;
  return CBSPMV_OK;
}

// a3. block statistics before aggregation: #non-empty blocks, #super-sparse blocks.
void pre_stats(const Csr &A, const cbspmv_options_t &o, int64_t blk_m, std::vector<Scratch> &scr,
               int64_t *nb_pre, int64_t *ss_count) {
  std::vector<int64_t> pre_nb(blk_m), pre_ss(blk_m);
  parallel_blockrows(A, o.blk, blk_m, (int)scr.size(), [&](int64_t lo, int64_t hi, int tid) {
    Scratch &s = scr[tid];
    for (int64_t br = lo; br < hi; br++) {
      block_row_keys(A, o.blk, br, false, s);
      int64_t nb = 0, ss = 0, run = 0;
      for (size_t t = 0; t < s.keys.size(); t++) {
        run++;
        if (t + 1 == s.keys.size() || (s.keys[t + 1].key >> 8) != (s.keys[t].key >> 8)) {
          nb++; ss += run < o.ss_limit; run = 0;
        }
      }
      pre_nb[br] = nb; pre_ss[br] = ss;
    }
  });
  *nb_pre = 0; *ss_count = 0;
  for (int64_t br = 0; br < blk_m; br++) { *nb_pre += pre_nb[br]; *ss_count += pre_ss[br]; }
}

}  // namespace

int check_csr(const Csr &A, const cbspmv_options_t &o, int64_t *nnz, std::string *err) {
  int st = check_options(A, o, err);
  if (st != CBSPMV_OK) return st;
  return canonical_check(A, o.host_threads, nnz, err);
}

bool decide_agg(int64_t nb_pre, int64_t ss_count, const cbspmv_options_t &o) {
  // aggregate iff ss / nb >= th0_num / th0_den, compared exactly in integers (R-3, R-5)
  return nb_pre > 0 && ss_count * (int64_t)o.th0_den >= (int64_t)o.th0_num * nb_pre;
}

int block_stats(const Csr &A, const cbspmv_options_t &o, int64_t *nb_pre, int64_t *ss_count, std::string *err) {
  int st = check_options(A, o, err);
  if (st != CBSPMV_OK) return st;
  int64_t nnz = 0;
  st = canonical_check(A, o.host_threads, &nnz, err);
  if (st != CBSPMV_OK) return st;
  std::vector<Scratch> scr(resolve_threads(o.host_threads));
  pre_stats(A, o, (A.m + o.blk - 1) / o.blk, scr, nb_pre, ss_count);
  return CBSPMV_OK;
}

// a7 TB-Load-Balance (Alg. 2) on the natural-order block arrays, then the permutation of the five
// high-level arrays into slot order (c.nb, c.blk, c.W set; mtx untouched: VPs travel with blocks).
void balance_and_permute(Canon &c, const cbspmv_options_t &o, const int32_t *nbr, const int32_t *nbc,
                         const int32_t *nnzb, const uint8_t *ntype, const uint64_t *nvp, PhaseTimer &tm) {
  const int64_t nb = c.nb;
  const int B = c.blk, W = c.W, T = resolve_threads(o.host_threads);
  const int64_t TB = (nb + W - 1) / W;
  c.T = TB;
  c.tb_ptr.assign((size_t)TB + 1, 0);
  c.tb_load.assign((size_t)TB, 0);
  c.tb_load_nat.assign((size_t)TB, 0);
  for (int64_t b = 0; b < nb; b++) c.tb_load_nat[b / W] += nnzb[b];
  std::vector<int64_t> perm(nb);  // slot-order position -> natural block index
  if (o.balance && nb > 0) {
    // "parallel sort(blk_idx_array, cmp_nnz)": nnz descending, ties by index ascending (R-12);
    // a stable counting sort over nnz in [1, B*B].
    const int maxk = B * B;
    std::vector<int64_t> cnt(maxk + 2, 0);
    for (int64_t b = 0; b < nb; b++) cnt[maxk - nnzb[b]]++;
    int64_t acc = 0;
    for (int k = 0; k <= maxk; k++) { int64_t t = cnt[k]; cnt[k] = acc; acc += t; }
    std::vector<int64_t> order(nb);
    for (int64_t b = 0; b < nb; b++) order[cnt[maxk - nnzb[b]]++] = b;
    // min-heap over (loads, tb_id) as a bucket queue: loads <= W*B*B, and the minimum load
    // never decreases (each pop re-pushes with a larger load), so a forward cursor suffices.
    // A bucket is only pushed to while the cursor is below it (pushes go to load + nnz > cur)
    // and only popped once the cursor has reached it, so each bucket is a plain vector sorted
    // once by tb_id when the cursor arrives (usually already sorted) and then read in order:
    // the pop order is exactly the heap's (load, tb_id) order.
    const int64_t maxload = (int64_t)W * maxk;
    std::vector<std::vector<uint32_t>> bucket((size_t)maxload + 1);
    bucket[0].resize((size_t)TB);
    for (int64_t t = 0; t < TB; t++) bucket[0][t] = (uint32_t)t;
    std::vector<int32_t> warps(TB, 0);
    std::vector<uint32_t> slot_tb(nb);
    std::vector<int32_t> slot_w(nb);
    int64_t cur = 0;
    size_t pos = 0;
    for (int64_t i = 0; i < nb; i++) {
      while (pos == bucket[cur].size()) {
        std::vector<uint32_t>().swap(bucket[cur]);
        cur++;
        pos = 0;
        std::vector<uint32_t> &v = bucket[cur];
        if (!std::is_sorted(v.begin(), v.end())) std::sort(v.begin(), v.end());
      }
      const uint32_t tb = bucket[cur][pos++];
      int64_t b = order[i];
      slot_tb[b] = tb; slot_w[b] = warps[tb];        // end <- tb_id*8 + warps
      c.tb_load[tb] += nnzb[b];                      // loads <- loads + nnz
      warps[tb]++;                                   // warps <- warps + 1
      if (warps[tb] < W) bucket[(size_t)c.tb_load[tb]].push_back(tb);  // if warps < 8: push
    }
    // "parallel sort(blk_idx_array, cmp_end)": ends are unique, so position = tb_ptr[tb] + w.
    for (int64_t t = 0; t < TB; t++) c.tb_ptr[t + 1] = c.tb_ptr[t] + warps[t];
    for (int64_t b = 0; b < nb; b++) perm[c.tb_ptr[slot_tb[b]] + slot_w[b]] = b;
  } else {
    for (int64_t b = 0; b < nb; b++) perm[b] = b;
    for (int64_t t = 0; t < TB; t++) {
      c.tb_ptr[t + 1] = std::min<int64_t>(nb, (t + 1) * W);
      c.tb_load[t] = c.tb_load_nat[t];
    }
  }
  tm.lap("a7 Alg. 2 greedy");
  // permute the five high-level arrays (vp_per_blk[i] <- vp_per_blk_old[ori])
  c.br.resize(nb); c.bc.resize(nb); c.nnzb.resize(nb); c.type.resize(nb); c.vp.resize(nb);
  parallel_for(nb, T, 1 << 16, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; i++) {
      int64_t b = perm[i];
      c.br[i] = nbr[b]; c.bc[i] = nbc[b]; c.nnzb[i] = nnzb[b]; c.type[i] = ntype[b]; c.vp[i] = nvp[b];
    }
  });
  tm.lap("a7 permute");
}

int build_canonical(const Csr &A, const cbspmv_options_t &o, Canon *out, std::string *err) {
  const int B = o.blk, W = o.warps_per_tb, threads = o.host_threads;
  const int64_t S = A.val_size;
  int st = check_options(A, o, err);
  if (st != CBSPMV_OK) return st;
  Canon &c = *out;
  c = Canon();
  c.m = A.m; c.n = A.n; c.blk = B; c.val_size = (int)S; c.W = W;
  c.blk_m = (A.m + B - 1) / B;
  PhaseTimer tm;
  st = canonical_check(A, threads, &c.nnz, err);   // a1
  tm.lap("a1 canonical check");
  if (st != CBSPMV_OK) return st;
  const int T = resolve_threads(threads);
  std::vector<Scratch> scr(T);
  pre_stats(A, o, c.blk_m, scr, &c.nb_pre, &c.ss_count);   // a3
  tm.lap("a3 block statistics");
  c.agg = o.agg_mode >= 0 ? o.agg_mode : decide_agg(c.nb_pre, c.ss_count, o);
  const bool agg = c.agg != 0;

  // a4 + a5 sizing pass: blocks, restore entries and record bytes per block row.
  std::vector<int64_t> br_nb(c.blk_m + 1, 0), br_res(c.blk_m + 1, 0), br_bytes(c.blk_m + 1, 0);
  parallel_blockrows(A, B, c.blk_m, T, [&](int64_t lo, int64_t hi, int tid) {
    Scratch &s = scr[tid];
    for (int64_t br = lo; br < hi; br++) {
      block_row_keys(A, B, br, agg, s);
      int64_t nb = 0, bytes = 0, run = 0;
      for (size_t t = 0; t < s.keys.size(); t++) {
        run++;
        if (t + 1 == s.keys.size() || (s.keys[t + 1].key >> 8) != (s.keys[t].key >> 8)) {
          nb++; bytes += record_bytes(select_format(run, o), run, B, S); run = 0;
        }
      }
      br_nb[br + 1] = nb; br_res[br + 1] = agg ? (int64_t)s.cols.size() : 0; br_bytes[br + 1] = bytes;
    }
  });
  for (int64_t br = 0; br < c.blk_m; br++) {
    br_nb[br + 1] += br_nb[br]; br_res[br + 1] += br_res[br]; br_bytes[br + 1] += br_bytes[br];
  }
  const int64_t nb = br_nb[c.blk_m];
  c.nb = nb;
  c.mtx.resize((size_t)br_bytes[c.blk_m]);  // not zeroed: pack_record clears each record
  if (agg) {
    c.restore.resize((size_t)br_res[c.blk_m]);
    c.cols_offset.resize((size_t)c.blk_m + 1);
    for (int64_t br = 0; br <= c.blk_m; br++) c.cols_offset[br] = (uint64_t)br_res[br];
  }

  tm.lap("a4+a5 sizing pass");
  // a6 fill pass: natural-order metadata, restore_cols, packed records at VP = byte offset.
  std::vector<int32_t> nbr(nb), nbc(nb), nnzb(nb);
  std::vector<uint8_t> ntype(nb);
  std::vector<uint64_t> nvp(nb);
  parallel_blockrows(A, B, c.blk_m, T, [&](int64_t lo, int64_t hi, int tid) {
    Scratch &s = scr[tid];
    for (int64_t br = lo; br < hi; br++) {
      block_row_keys(A, B, br, agg, s);
      if (agg) std::copy(s.cols.begin(), s.cols.end(), c.restore.begin() + br_res[br]);
      int64_t b = br_nb[br], off = br_bytes[br], start = 0;
      for (size_t t = 0; t < s.keys.size(); t++) {
        if (t + 1 == s.keys.size() || (s.keys[t + 1].key >> 8) != (s.keys[t].key >> 8)) {
          int64_t k = (int64_t)t + 1 - start;
          int type = select_format(k, o);
          nbr[b] = (int32_t)br; nbc[b] = (int32_t)(s.keys[t].key >> 8); nnzb[b] = (int32_t)k;
          ntype[b] = (uint8_t)type; nvp[b] = (uint64_t)off;
          pack_record(A, B, S, type, &s.keys[start], k, c.mtx.data() + off);
          off += record_bytes(type, k, B, S);
          b++; start = (int64_t)t + 1;
        }
      }
    }
  });
  for (int64_t b = 0; b < nb; b++) c.fmt_count[ntype[b]]++;

  tm.lap("a6 fill pass");
  balance_and_permute(c, o, nbr.data(), nbc.data(), nnzb.data(), ntype.data(), nvp.data(), tm);
  return CBSPMV_OK;
}

}  // namespace cb
