// stream.cpp — the device page stream (version 3, cb_internal.h / DESIGN.md §4): a derived
// layout of the canonical CB-SpMV format (slot order after Alg. 2) cut into pages that
// one cp.async.bulk moves into a shared-memory stage.  The paper's intra-block data aggregation
// (a block's coordinates and values contiguous behind one pointer) is kept per work
// item: a CSR / DENSE block's canonical record (plus its restore_cols entries) stays one
// contiguous run.  The page's COO elements (Alg. 3's blocks) are regrouped into
// row-run slices: each element with its original column resolved (the restore lookup of Alg. 3
// line 19 done once, here), grouped by global row, pieces of at most Lmax elements dealt one per
// lane, so a lane sums its piece in a register and issues one RED for it (the paper's warp per COO
// block leaves >= 50 % of its lanes idle, and issues one atomic per element).
#include <algorithm>
#include <array>
#include <atomic>
#include <memory>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "cb_internal.h"

namespace cb {

namespace {

inline int64_t canon_record_bytes(const Canon &c, int64_t i) {
  const int64_t B = c.blk, S = c.val_size, k = c.nnzb[i];
  const int type = c.type[i];
  const int64_t idx = type == CBSPMV_FMT_COO ? k : type == CBSPMV_FMT_CSR ? (B + 1) + k : 0;
  const int64_t nval = type == CBSPMV_FMT_DENSE ? B * B : k;
  return round_up(idx, S) + nval * S;
}

// valid x-tile columns of block i (16 but at the ragged last block column / aggregated segment)
inline int block_ncols(const Canon &c, int64_t i) {
  int64_t w = c.agg ? (int64_t)(c.cols_offset[c.br[i] + 1] - c.cols_offset[c.br[i]]) - (int64_t)c.bc[i] * c.blk
                    : c.n - (int64_t)c.bc[i] * c.blk;
  return (int)std::max<int64_t>(0, std::min<int64_t>(c.blk, w));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// bytes of the slice tables of P pieces (slices of 32 lanes, the last one partial)
inline int64_t tables_bytes(int64_t P) {
  if (P == 0) return 0;
  const int64_t ns = ceil_div(P, kSliceLanes);
  return (ns - 1) * slice_table_bytes(kSliceLanes) + slice_table_bytes(P - (ns - 1) * kSliceLanes);
}

// Open-addressing map block row -> slot, reset per page (a page holds at most a few thousand
// COO blocks); a slot holds the page's element counts of the block row's 16 rows.
class BrTable {
 public:
  BrTable() : key_(kSize, -1), slot_(kSize, 0) {}
  int find(int32_t br) const {
    for (uint32_t h = hash(br);; h = (h + 1) & (kSize - 1)) {
      if (key_[h] == br) return slot_[h];
      if (key_[h] < 0) return -1;
    }
  }
  int insert(int32_t br) {  // br absent
    uint32_t h = hash(br);
    while (key_[h] >= 0) h = (h + 1) & (kSize - 1);
    key_[h] = br;
    slot_[h] = (int)cnt_.size();
    used_.push_back(h);
    cnt_.emplace_back();
    cnt_.back().fill(0);
    return slot_[h];
  }
  std::array<int32_t, 16> &counts(int s) { return cnt_[(size_t)s]; }
  const std::array<int32_t, 16> &counts(int s) const { return cnt_[(size_t)s]; }
  void clear() {
    for (uint32_t h : used_) key_[h] = -1;
    used_.clear();
    cnt_.clear();
  }
  size_t size() const { return used_.size(); }

 private:
  static constexpr uint32_t kSize = 1u << 15;
  static uint32_t hash(int32_t br) { return ((uint32_t)br * 2654435761u) >> 17; }
  std::vector<int32_t> key_;
  std::vector<int> slot_;
  std::vector<uint32_t> used_;
  std::vector<std::array<int32_t, 16>> cnt_;
};

// Page state of the greedy cut: CSR / DENSE items, COO elements and row-run pieces (exact: the
// page's per-row element counts are tracked per block row).
struct PageAcc {
  int64_t items = 0;  // CSR / DENSE items
  int64_t rec = 0;    // their record bytes (incl. restore entries, 16-aligned each)
  int64_t xb = 0;     // their x slots
  int64_t E = 0, P = 0;  // COO elements, pieces
  int64_t blocks = 0;
};

struct Shape {
  int val_size, x_size, run_max;
  // stage bytes of a page in this state: exact but for <= 8 B of element padding per slice
  int64_t stage_bytes(const PageAcc &a) const {
    const int64_t ns = ceil_div(a.P, kSliceLanes);
    const int64_t pre = round_up(kPageHeader + kDescBytes * (a.items + ns) + tables_bytes(a.P), 16);
    const int64_t el = a.E ? 4 * a.E + val_size * a.E + 8 * ns + 8 : 0;
    return pre + a.rec + el + a.xb;
  }
  int64_t pieces(int64_t n) const { return ceil_div(n, run_max); }
};

struct Piece {
  uint32_t row;
  int32_t q;     // index of the piece within its row's run
  int32_t len;
  int64_t run;   // the run (index into the page's run list)
};

}  // namespace

void free_stream(Stream *s) {
  if (s->bytes) {
    if (s->pinned) cudaFreeHost(s->bytes);
    else std::free(s->bytes);
  }
  s->bytes = nullptr; s->nbytes = 0; s->page_off.clear();
}

int build_stream(const Canon &c, int page_cap, int x_size, int threads, Stream *s, StreamPlan *plan,
                 std::string *err, const SliceOpts &so, const CooCoords *coords, bool xagg) {
  if (c.blk != 16) { *err = "the device page stream needs 16x16 blocks"; return CBSPMV_EUNSUPPORTED; }
  if (page_cap > kMaxPageCap || page_cap < 1024) { *err = "stage capacity out of range"; return CBSPMV_EUNSUPPORTED; }
  if (so.run_max < 1 || so.run_max > kMaxRun) { *err = "run_max out of range [1, 255]"; return CBSPMV_EINVAL; }
  const int T = resolve_threads(threads);
  const int S = c.val_size;
  const Shape sh{S, x_size, so.run_max};
  const bool xtiles = !c.agg || xagg;  // CSR / DENSE items get an x-tile slot after the page
  PhaseTimer tm;
  auto coord = [&](int64_t i) -> const uint8_t * {
    return coords ? coords->bytes.data() + coords->off[i] : c.mtx.data() + c.vp[i];
  };
  std::vector<int32_t> ncol((size_t)c.nb);
  std::vector<int64_t> rec((size_t)c.nb);  // CSR / DENSE: device record bytes (restore + record)
  std::vector<std::array<uint8_t, 16>> rcnt((size_t)c.nb);  // COO: elements per local row
  parallel_for(c.nb, T, 1 << 14, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; i++) {
      ncol[i] = block_ncols(c, i);
      rec[i] = c.type[i] == CBSPMV_FMT_COO ? 0
               : (c.agg ? round_up(ncol[i], 4) * 4 : 0) + round_up(canon_record_bytes(c, i), 16);
      if (c.type[i] == CBSPMV_FMT_COO) {
        rcnt[i].fill(0);
        const uint8_t *cb = coord(i);
        for (int e = 0; e < c.nnzb[i]; e++) rcnt[i][cb[e] & 15]++;  // (col << 4) | row
      }
    }
  });
  tm.lap("stream: block row counts");
  // ---- hot x columns (shared x cache, cb_internal.h): the H columns carrying the most COO
  // elements, when they carry at least hot_min_pct % of them and save more gathers than the
  // per-launch cache fill costs (H loads per CTA)
  auto resolved = [&](int64_t i, uint8_t b) -> uint32_t {
    return c.agg ? c.restore[c.cols_offset[c.br[i]] + (uint64_t)c.bc[i] * c.blk + (b >> 4)]
                 : (uint32_t)c.bc[i] * (uint32_t)c.blk + (b >> 4);
  };
  std::vector<uint32_t> hot_slot;  // column -> slot (kNotHot: not cached); empty: no cache
  constexpr uint32_t kNotHot = 0xFFFFFFFFu;
  // every persistent CTA copies the H hot values per launch: the cache must save more gathers than
  // kHotCostFactor x (CTAs x H); CTAs = the B200's 148 SMs (the launch grid; a cost estimate only)
  constexpr int64_t kHotCopyCtas = 148, kHotCostFactor = 4;
  s->hot_cols.clear();
  {
    const int64_t H = so.hot_bytes > 0 ? so.hot_bytes / x_size : 0;
    int64_t n_coo = 0;
    for (int64_t i = 0; i < c.nb; i++) n_coo += c.type[i] == CBSPMV_FMT_COO ? c.nnzb[i] : 0;
    const bool force = so.hot_min_pct == 0;
    if (H > 0 && n_coo > 0 && c.n <= (int64_t)1 << 27 &&  // count array <= 512 MB
        (force || n_coo >= kHotCostFactor * kHotCopyCtas * H)) {
      // estimate on every 251st COO block first (uniform-like matrices stop here)
      std::vector<uint32_t> samp;
      for (int64_t i = 0; i < c.nb; i += 251)
        if (c.type[i] == CBSPMV_FMT_COO)
          for (int e = 0; e < c.nnzb[i]; e++) samp.push_back(resolved(i, coord(i)[e]));
      std::sort(samp.begin(), samp.end());
      std::vector<int64_t> sc;
      for (size_t a = 0, b; a < samp.size(); a = b) {
        for (b = a; b < samp.size() && samp[b] == samp[a]; b++) {}
        sc.push_back((int64_t)(b - a));
      }
      const size_t top = std::min(sc.size(), (size_t)H);
      std::partial_sort(sc.begin(), sc.begin() + top, sc.end(), std::greater<int64_t>());
      int64_t est = 0;
      for (size_t k = 0; k < top; k++) est += sc[k];
      if (force || (int64_t)samp.size() == 0 || est * 100 >= (int64_t)so.hot_min_pct * (int64_t)samp.size()) {
        // exact column counts of the COO elements
        std::unique_ptr<std::atomic<uint32_t>[]> hist(new std::atomic<uint32_t>[(size_t)c.n]);
        parallel_for(c.n, T, 1 << 16, [&](int64_t lo, int64_t hi, int) {
          for (int64_t j = lo; j < hi; j++) hist[j].store(0, std::memory_order_relaxed);
        });
        parallel_for(c.nb, T, 1 << 12, [&](int64_t lo, int64_t hi, int) {
          for (int64_t i = lo; i < hi; i++)
            if (c.type[i] == CBSPMV_FMT_COO)
              for (int e = 0; e < c.nnzb[i]; e++) hist[resolved(i, coord(i)[e])].fetch_add(1, std::memory_order_relaxed);
        });
        std::vector<uint32_t> cand;
        for (int64_t j = 0; j < c.n; j++)
          if (hist[j].load(std::memory_order_relaxed)) cand.push_back((uint32_t)j);
        auto more = [&](uint32_t a, uint32_t b) {  // count desc, column asc
          const uint32_t ca = hist[a].load(std::memory_order_relaxed), cb = hist[b].load(std::memory_order_relaxed);
          return ca != cb ? ca > cb : a < b;
        };
        if ((int64_t)cand.size() > H) {
          std::nth_element(cand.begin(), cand.begin() + H, cand.end(), more);
          cand.resize((size_t)H);
        }
        int64_t covered = 0;
        for (uint32_t j : cand) covered += hist[j].load(std::memory_order_relaxed);
        if (force || (covered * 100 >= (int64_t)so.hot_min_pct * n_coo &&
                      covered >= kHotCostFactor * kHotCopyCtas * (int64_t)cand.size())) {
          std::sort(cand.begin(), cand.end());
          hot_slot.assign((size_t)c.n, kNotHot);
          for (size_t k = 0; k < cand.size(); k++) hot_slot[cand[k]] = (uint32_t)k;
          s->hot_cols = std::move(cand);
        }
      }
    }
  }
  tm.lap("stream: hot x columns");
  // ---- greedy page cut: consecutive slot-order blocks while page + x area fits the stage.  Large
  // matrices are cut in fixed segments of >= 2^16 blocks, in parallel (a page does not cross a
  // segment start; the segments do not depend on the thread count, so the stream does not either).
  const int64_t seg_len = std::max<int64_t>(1 << 16, ceil_div(c.nb, 64));
  const int64_t nseg = std::max<int64_t>(1, ceil_div(c.nb, seg_len));
  std::vector<std::vector<int64_t>> seg_pb((size_t)nseg);
  std::vector<int> seg_fail((size_t)nseg, 0);
  parallel_for(nseg, T, 1, [&](int64_t lo, int64_t hi, int) {
    BrTable tab;
    for (int64_t sg = lo; sg < hi; sg++) {
      const int64_t b0 = sg * seg_len, b1 = std::min(c.nb, b0 + seg_len);
      std::vector<int64_t> &out = seg_pb[(size_t)sg];
      PageAcc cur;
      tab.clear();
      for (int64_t i = b0; i < b1; i++) {
        PageAcc nx = cur;
        int slot = -1;
        if (c.type[i] == CBSPMV_FMT_COO) {
          slot = tab.find(c.br[i]);
          for (int r = 0; r < 16; r++) {
            const int64_t o = slot >= 0 ? tab.counts(slot)[r] : 0, k = rcnt[i][r];
            nx.P += sh.pieces(o + k) - sh.pieces(o);
          }
          nx.E += c.nnzb[i];
        } else {
          nx.items++; nx.rec += rec[i]; nx.xb += xtiles ? 16 * (int64_t)x_size : 0;
        }
        nx.blocks++;
        if (sh.stage_bytes(nx) <= page_cap) {
          cur = nx;
          if (c.type[i] == CBSPMV_FMT_COO) {
            if (slot < 0) slot = tab.insert(c.br[i]);
            for (int r = 0; r < 16; r++) tab.counts(slot)[r] += rcnt[i][r];
          }
          continue;
        }
        if (cur.blocks == 0) { seg_fail[(size_t)sg] = 1; break; }
        out.push_back(i);  // block i starts a new page
        cur = PageAcc{};
        tab.clear();
        i--;  // re-add block i to the empty page
      }
    }
  });
  for (int f : seg_fail)
    if (f) { *err = "stage capacity too small for one block"; return CBSPMV_EUNSUPPORTED; }
  std::vector<int64_t> pb;  // first block of each page (+ nb)
  for (int64_t sg = 0; sg < nseg; sg++) {
    if (sg * seg_len < c.nb) pb.push_back(sg * seg_len);
    pb.insert(pb.end(), seg_pb[(size_t)sg].begin(), seg_pb[(size_t)sg].end());
  }
  if (pb.empty()) pb.push_back(0);
  pb.push_back(c.nb);
  if (c.nb == 0) pb.assign(1, 0);
  const int64_t npages = (int64_t)pb.size() - 1;
  tm.lap("stream: page cut");

  // ---- per page: its runs (rows of its COO elements), pieces and slices
  // Runs are built from the per-row counts (the layout pass) and again from the elements (the fill
  // pass); both use the same order: rows ascending, a row's elements in slot order then canonical
  // order, pieces of run_max, then sorted by the piece order.
  struct Layout {
    std::vector<uint32_t> rows;  // distinct global rows of the page's COO elements, ascending
    std::vector<int32_t> cnt;    // elements per row
    std::vector<Piece> pcs;      // in slice order
  };
  auto page_layout = [&](int64_t p, Layout &L) {
    L.rows.clear(); L.cnt.clear(); L.pcs.clear();
    std::vector<std::pair<uint32_t, int32_t>> rc;
    for (int64_t i = pb[p]; i < pb[p + 1]; i++) {
      if (c.type[i] != CBSPMV_FMT_COO) continue;
      for (int r = 0; r < 16; r++)
        if (rcnt[i][r]) rc.emplace_back((uint32_t)c.br[i] * 16u + (uint32_t)r, (int32_t)rcnt[i][r]);
    }
    std::sort(rc.begin(), rc.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
    for (const auto &v : rc) {
      if (!L.rows.empty() && L.rows.back() == v.first) L.cnt.back() += v.second;
      else { L.rows.push_back(v.first); L.cnt.push_back(v.second); }
    }
    for (int64_t r = 0; r < (int64_t)L.rows.size(); r++)
      for (int32_t q = 0; q * so.run_max < L.cnt[r]; q++)
        L.pcs.push_back(Piece{L.rows[r], q, std::min(so.run_max, L.cnt[r] - q * so.run_max), r});
    if (!so.row_order)  // (length desc, row asc, piece asc); the run list is row-ascending already
      std::stable_sort(L.pcs.begin(), L.pcs.end(), [](const Piece &a, const Piece &b) { return a.len > b.len; });
  };
  auto slice_E = [&](const Layout &L, int64_t s) {
    int64_t e = 0;
    const int64_t a = s * kSliceLanes, b = std::min<int64_t>(a + kSliceLanes, (int64_t)L.pcs.size());
    for (int64_t k = a; k < b; k++) e += L.pcs[k].len;
    return e;
  };
  std::vector<int64_t> pbytes((size_t)npages, 0), pmeta((size_t)npages, 0);
  parallel_for(npages, T, 64, [&](int64_t lo, int64_t hi, int) {
    Layout L;
    for (int64_t p = lo; p < hi; p++) {
      int64_t items = 0, recb = 0;
      for (int64_t i = pb[p]; i < pb[p + 1]; i++)
        if (c.type[i] != CBSPMV_FMT_COO) { items++; recb += rec[i]; }
      page_layout(p, L);
      const int64_t Pn = (int64_t)L.pcs.size(), ns = ceil_div(Pn, kSliceLanes);
      int64_t el = 0;
      for (int64_t sl = 0; sl < ns; sl++) el += slice_elem_bytes(slice_E(L, sl), S);
      pmeta[p] = round_up(kPageHeader + kDescBytes * (items + ns) + tables_bytes(Pn), 16);
      pbytes[p] = round_up(pmeta[p] + recb + el, 16);
    }
  });
  std::vector<uint64_t> off((size_t)npages + 1, 0);
  for (int64_t p = 0; p < npages; p++) off[p + 1] = off[p] + (uint64_t)pbytes[p];
  const int64_t total = (int64_t)off[npages];
  tm.lap("stream: page layout");
  s->nbytes = total;
  s->page_off = off;
  if (plan) {
    plan->meta_off.assign((size_t)npages + 1, 0);
    for (int64_t p = 0; p < npages; p++) plan->meta_off[p + 1] = plan->meta_off[p] + (uint64_t)pmeta[p];
    plan->meta.assign((size_t)plan->meta_off[npages], 0);
    plan->rec_dst.assign((size_t)c.nb, 0);
    plan->res_dst.assign(c.agg ? (size_t)c.nb : 0, 0);
    plan->ncol = ncol;
    plan->coo_e0.assign((size_t)c.nb, -1);
    int64_t ne = 0;
    for (int64_t i = 0; i < c.nb; i++)
      if (c.type[i] == CBSPMV_FMT_COO) { plan->coo_e0[i] = ne; ne += c.nnzb[i]; }
    plan->coo_dst.assign((size_t)ne, 0);
  } else if (total > 0) {
    void *p = nullptr;
    // Pageable by default: pinning a multi-GB buffer costs more (measured 2.7 s for the 4.2 GB
    // clustered stream on the B200 host) than the slower pageable copy saves.
    static const bool want_pinned = std::getenv("CBSPMV_PINNED_STREAM") != nullptr;
    if (want_pinned && cudaHostAlloc(&p, (size_t)total, cudaHostAllocDefault) == cudaSuccess) {
      s->pinned = true;
    } else {
      if (want_pinned) cudaGetLastError();
      p = std::malloc((size_t)total);
      s->pinned = false;
    }
    if (!p) { *err = "host allocation of the page stream failed"; return CBSPMV_ENOMEM; }
    s->bytes = (uint8_t *)p;
  }
  tm.lap(plan ? "stream: device plan alloc" : s->pinned ? "stream: pinned alloc" : "stream: pageable alloc");

  // ---- fill: one page at a time
  struct Elem {
    uint32_t row;
    int64_t blk;
    int32_t e;  // index within the block's canonical record
  };
  parallel_for(npages, T, 64, [&](int64_t lo, int64_t hi, int) {
    Layout L;
    std::vector<int64_t> cd;                 // CSR / DENSE blocks of the page
    std::vector<Elem> el;                    // the page's COO elements
    std::vector<int64_t> run0;               // per run: its first element in el (sorted by row)
    std::vector<int64_t> cur;                // per run: next free element slot
    std::vector<int32_t> idx;                // per slice: element index of (lane, step)
    for (int64_t p = lo; p < hi; p++) {
      cd.clear();
      page_layout(p, L);
      const int64_t nruns = (int64_t)L.rows.size(), Pn = (int64_t)L.pcs.size();
      const int64_t ns = ceil_div(Pn, kSliceLanes);
      run0.assign((size_t)nruns + 1, 0);
      for (int64_t r = 0; r < nruns; r++) run0[r + 1] = run0[r] + L.cnt[r];
      // the page's COO elements by run (rows ascending; a row's elements in slot order, then
      // canonical order): a counting sort on the run index (binary search in the run rows)
      el.resize((size_t)run0[nruns]);
      cur.assign(run0.begin(), run0.end() - 1);
      for (int64_t i = pb[p]; i < pb[p + 1]; i++) {
        if (c.type[i] != CBSPMV_FMT_COO) { cd.push_back(i); continue; }
        const uint8_t *cb = coord(i);
        const uint32_t r0 = (uint32_t)c.br[i] * 16u;
        const int64_t rb = std::lower_bound(L.rows.begin(), L.rows.end(), r0) - L.rows.begin();
        for (int e = 0; e < c.nnzb[i]; e++) {
          const uint32_t row = r0 + (cb[e] & 15u);
          int64_t r = rb;
          while (L.rows[(size_t)r] != row) r++;  // the block row's runs are consecutive, ascending
          el[(size_t)cur[(size_t)r]++] = Elem{row, i, e};
        }
      }

      const int64_t nitems = (int64_t)cd.size() + ns;
      const int64_t desc0 = kPageHeader;
      int64_t tpos = kPageHeader + kDescBytes * nitems;  // slice tables
      int64_t pos = pmeta[p];                            // records, then slice elements
      const int64_t xoff = pbytes[p];
      int64_t xpos = xoff;
      uint8_t *page = plan ? plan->meta.data() + plan->meta_off[p] : s->bytes + off[p];
      const int64_t wbytes = plan ? pmeta[p] : pbytes[p];  // bytes of `page` written here
      std::memset(page, 0, (size_t)wbytes);
      const uint32_t hdr[4] = {(uint32_t)nitems, (uint32_t)cd.size(), (uint32_t)(pb[p + 1] - pb[p]), (uint32_t)pb[p]};
      std::memcpy(page, hdr, 16);
      int64_t it = 0;
      for (int64_t i : cd) {
        const int type = c.type[i];
        const int64_t k = c.nnzb[i];
        const int64_t res = c.agg ? pos : 0;
        if (c.agg) pos += round_up(ncol[i], 4) * 4;
        const int64_t body = pos;
        const int64_t idxb = type == CBSPMV_FMT_CSR ? (c.blk + 1) + k : 0;
        const int64_t vals = body + round_up(idxb, S);
        uint32_t d[4];
        d[0] = (uint32_t)c.br[i] * (uint32_t)c.blk;
        d[1] = c.agg ? (uint32_t)res : (uint32_t)c.bc[i] * (uint32_t)c.blk;
        d[2] = (uint32_t)body | ((uint32_t)vals << 16);
        d[3] = (uint32_t)type | ((uint32_t)ncol[i] << 2) | ((uint32_t)(k - 1) << 8) |
               (xtiles ? (uint32_t)xpos << 16 : 0u);
        std::memcpy(page + desc0 + kDescBytes * it, d, 16);
        it++;
        if (xtiles) xpos += 16 * (int64_t)x_size;
        if (plan) {
          plan->rec_dst[i] = off[p] + (uint64_t)body;
          if (c.agg) plan->res_dst[i] = off[p] + (uint64_t)res;
        } else {
          if (c.agg) {
            const uint32_t *seg = c.restore.data() + c.cols_offset[c.br[i]] + (uint64_t)c.bc[i] * c.blk;
            std::memcpy(page + res, seg, (size_t)ncol[i] * 4);
          }
          const uint8_t *src = c.mtx.data() + c.vp[i];
          if (type == CBSPMV_FMT_DENSE) {
            // lane-major 16-byte pairs: pair k*32 + l holds A[l % 16][(l / 16) * 8 + 2k + {0, 1}]
            for (int q = 0; q < 4; q++)
              for (int l = 0; l < 32; l++)
                for (int h = 0; h < 2; h++) {
                  const int a = (l & 15) * 16 + (l >> 4) * 8 + 2 * q + h;
                  std::memcpy(page + body + (int64_t)((q * 32 + l) * 2 + h) * S, src + (int64_t)a * S, (size_t)S);
                }
          } else {
            std::memcpy(page + body, src, (size_t)canon_record_bytes(c, i));
          }
        }
        pos = body + round_up(canon_record_bytes(c, i), 16);
      }
      // COO slices: descriptors, tables (in the prefix) and elements (after the records)
      std::vector<int64_t> cols_at((size_t)ns), vals_at((size_t)ns);
      std::vector<int32_t> w_of((size_t)ns);
      for (int64_t sl = 0; sl < ns; sl++) {
        const int64_t a = sl * kSliceLanes, nl = std::min<int64_t>(kSliceLanes, Pn - a);
        int w = 0;
        for (int64_t l = 0; l < nl; l++) {
          const Piece &pc = L.pcs[a + l];
          std::memcpy(page + tpos + 4 * l, &pc.row, 4);
          page[tpos + 4 * nl + l] = (uint8_t)pc.len;
          w = std::max(w, pc.len);
        }
        const int64_t E = slice_E(L, sl);
        cols_at[sl] = pos;
        vals_at[sl] = pos + round_up(4 * E, 8);
        w_of[sl] = w;
        uint32_t d[4];
        d[0] = (uint32_t)tpos | ((uint32_t)nl << 16) | ((uint32_t)w << 24);
        d[1] = (uint32_t)cols_at[sl] | ((uint32_t)vals_at[sl] << 16);
        d[2] = (uint32_t)E;
        d[3] = (uint32_t)CBSPMV_FMT_COO;
        std::memcpy(page + desc0 + kDescBytes * it, d, 16);
        it++;
        tpos += slice_table_bytes(nl);
        pos += slice_elem_bytes(E, S);
      }
      // element (lane l, step j) of a slice sits at off_j + (lanes below l whose piece is longer than j)
      for (int64_t sl = 0; sl < ns; sl++) {
        const int64_t a = sl * kSliceLanes, nl = std::min<int64_t>(kSliceLanes, Pn - a);
        const int w = w_of[sl];
        idx.assign((size_t)kSliceLanes * w, -1);
        int32_t o = 0;
        for (int j = 0; j < w; j++)
          for (int64_t l = 0; l < nl; l++)
            if (L.pcs[a + l].len > j) idx[(size_t)l * w + j] = o++;
        // place this slice's elements
        for (int64_t l = 0; l < nl; l++) {
          const Piece &pc = L.pcs[a + l];
          const int64_t e0 = run0[pc.run] + (int64_t)pc.q * so.run_max;
          for (int j = 0; j < pc.len; j++) {
            const Elem &E = el[(size_t)(e0 + j)];
            const int64_t ix = idx[(size_t)l * w + j];
            const uint32_t co = (uint32_t)(cols_at[sl] + 4 * ix), vo = (uint32_t)(vals_at[sl] + S * ix);
            const int64_t i = E.blk;
            if (plan) {
              plan->coo_dst[(size_t)(plan->coo_e0[i] + E.e)] = co | (vo << 16);
              plan->rec_dst[i] = off[p];
              continue;
            }
            const int64_t k = c.nnzb[i];
            uint32_t col = resolved(i, coord(i)[E.e]);  // coordinate byte (col << 4) | row
            if (!hot_slot.empty() && hot_slot[col] != kNotHot) col = kHotBit | hot_slot[col];
            std::memcpy(page + co, &col, 4);
            std::memcpy(page + vo, c.mtx.data() + c.vp[i] + round_up(k, S) + (int64_t)S * E.e, (size_t)S);
          }
        }
      }
    }
  });
  tm.lap("stream: fill pages");
  return CBSPMV_OK;
}

}  // namespace cb
