// stream.cpp — the device page stream (version 2, cb_internal.h / DESIGN.md §4): a derived
// layout of the canonical CB-SpMV format (slot order after Alg. 2) cut into pages that
// one cp.async.bulk moves into a shared-memory stage.  The paper's intra-block data aggregation
// (a block's coordinates and values contiguous behind one pointer) is kept per work
// item: a CSR / DENSE block's canonical record (plus its restore_cols entries) stays one
// contiguous run; the page's COO blocks are packed lane-contiguously into 32-element chunks with
// each element's original column resolved, so a warp handles 32 elements with one RED (the
// paper's warp per COO block leaves >= 50 % of lanes idle).
#include <algorithm>
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

// Incremental page state of the greedy page cut (slot order).  COO elements are chunked in
// order: a chunk closes at 32 elements or when a 17th member (block) would join it.
struct PageAcc {
  int64_t items = 0;         // CSR / DENSE items
  int64_t rec = 0;           // their record bytes (incl. restore entries, 16-aligned each)
  int64_t xb = 0;            // their x slots
  int64_t chunks = 0, chunk_rec = 0;  // closed chunks
  int nv = 0, nm = 0;        // the open chunk (nv == 0: none)
};

struct Shape {
  int val_size, x_size;
  int64_t stage_bytes(const PageAcc &a) const {
    const bool open = a.nv > 0;
    const int64_t items = a.items + a.chunks + (open ? 1 : 0);
    const int64_t page = round_up(kPageHeader + kDescBytes * items, 16) + a.rec + a.chunk_rec +
                         (open ? chunk_layout(a.nv, a.nm, val_size).bytes : 0);
    return page + a.xb;
  }
  void close_chunk(PageAcc &a) const {
    a.chunks++;
    a.chunk_rec += chunk_layout(a.nv, a.nm, val_size).bytes;
    a.nv = a.nm = 0;
  }
  // append the k elements of one COO block; fn(lane0, member, e0, t) per piece (chunk index =
  // a.chunks at the call)
  template <class F>
  void add_coo(PageAcc &a, int64_t k, F &&fn) const {
    int64_t e = 0;
    bool member = false;
    while (e < k) {
      if (a.nv == kChunkLanes || (!member && a.nm == kChunkMembers)) {
        close_chunk(a);
        member = false;
      }
      int m = a.nm - 1;
      if (!member) { m = a.nm++; member = true; }
      const int t = (int)std::min<int64_t>(k - e, kChunkLanes - a.nv);
      fn(a.nv, m, e, t);
      a.nv += t;
      e += t;
      if (e < k) member = false;  // the rest starts the next chunk
    }
  }
};

struct Piece {  // one block's run of elements in one chunk
  int64_t block, e0, chunk;  // chunk: index within the page
  int lane0, member, t;
};

// The page's COO blocks in the order they are chunked: grouped by block row (stable), so a chunk's
// elements come from few block rows — fewer 32-byte y sectors per RED and same-row runs across
// blocks of one block row (R-MAT: 8.2 -> 4.9 sectors per chunk RED, 15.7 -> 11.3 distinct rows).
// Falls back to slot order when grouping would need more chunk bytes than the page cut (slot
// order) reserved.  Returns the chunk count; *bytes gets the chunk record bytes.
int64_t coo_order(const Canon &c, const Shape &sh, int64_t b0, int64_t b1, std::vector<int64_t> &out,
                  int64_t *bytes) {
  auto noop = [](int, int, int64_t, int) {};
  out.clear();
  for (int64_t i = b0; i < b1; i++)
    if (c.type[i] == CBSPMV_FMT_COO) out.push_back(i);
  auto chunk = [&](const std::vector<int64_t> &v, int64_t *b) {
    PageAcc a;
    for (int64_t i : v) sh.add_coo(a, c.nnzb[i], noop);
    if (a.nv) sh.close_chunk(a);
    *b = a.chunk_rec;
    return a.chunks;
  };
  int64_t slot_bytes = 0;
  const int64_t slot_chunks = chunk(out, &slot_bytes);
  std::vector<int64_t> g = out;
  std::stable_sort(g.begin(), g.end(), [&](int64_t x, int64_t y) { return c.br[x] < c.br[y]; });
  int64_t g_bytes = 0;
  const int64_t g_chunks = chunk(g, &g_bytes);
  if (g_bytes + kDescBytes * g_chunks <= slot_bytes + kDescBytes * slot_chunks) {
    out.swap(g);
    *bytes = g_bytes;
    return g_chunks;
  }
  *bytes = slot_bytes;
  return slot_chunks;
}

}  // namespace

void free_stream(Stream *s) {
  if (s->bytes) {
    if (s->pinned) cudaFreeHost(s->bytes);
    else std::free(s->bytes);
  }
  s->bytes = nullptr; s->nbytes = 0; s->page_off.clear();
}

int build_stream(const Canon &c, int page_cap, int x_size, int threads, Stream *s, StreamPlan *plan,
                 std::string *err, bool runs) {
  if (c.blk != 16) { *err = "the device page stream needs 16x16 blocks"; return CBSPMV_EUNSUPPORTED; }
  if (page_cap > kMaxPageCap || page_cap < 1024) { *err = "stage capacity out of range"; return CBSPMV_EUNSUPPORTED; }
  const int T = resolve_threads(threads);
  const int S = c.val_size;
  const Shape sh{S, x_size};
  PhaseTimer tm;
  std::vector<int32_t> ncol((size_t)c.nb);
  std::vector<int64_t> rec((size_t)c.nb);  // CSR / DENSE: device record bytes (restore + record)
  parallel_for(c.nb, T, 1 << 16, [&](int64_t lo, int64_t hi, int) {
    for (int64_t i = lo; i < hi; i++) {
      ncol[i] = block_ncols(c, i);
      rec[i] = c.type[i] == CBSPMV_FMT_COO ? 0
               : (c.agg ? round_up(ncol[i], 4) * 4 : 0) + round_up(canon_record_bytes(c, i), 16);
    }
  });
  // ---- greedy page cut: consecutive slot-order blocks while page + x area fits the stage
  std::vector<int64_t> pb{0};        // first block of each page (+ nb)
  std::vector<int64_t> page_chunks;  // chunks per page
  PageAcc cur;
  auto noop = [](int, int, int64_t, int) {};
  for (int64_t i = 0; i < c.nb; i++) {
    PageAcc nx = cur;
    if (c.type[i] == CBSPMV_FMT_COO) {
      sh.add_coo(nx, c.nnzb[i], noop);
    } else {
      nx.items++; nx.rec += rec[i]; nx.xb += c.agg ? 0 : 16 * (int64_t)x_size;
    }
    if (sh.stage_bytes(nx) <= page_cap) { cur = nx; continue; }
    if (i == pb.back()) { *err = "stage capacity too small for one block"; return CBSPMV_EUNSUPPORTED; }
    page_chunks.push_back(cur.chunks + (cur.nv > 0));
    pb.push_back(i);
    cur = PageAcc{};
    i--;  // re-add block i to the empty page
  }
  if (c.nb > pb.back()) { page_chunks.push_back(cur.chunks + (cur.nv > 0)); pb.push_back(c.nb); }
  const int64_t npages = (int64_t)pb.size() - 1;
  // page sizes (exact) -> offsets; chunk ids
  std::vector<uint64_t> off((size_t)npages + 1, 0);
  std::vector<int64_t> chunk0((size_t)npages + 1, 0);
  std::vector<int64_t> pbytes((size_t)npages, 0);
  parallel_for(npages, T, 256, [&](int64_t lo, int64_t hi, int) {
    std::vector<int64_t> order;
    for (int64_t p = lo; p < hi; p++) {
      int64_t items = 0, recb = 0, cbytes = 0;
      for (int64_t i = pb[p]; i < pb[p + 1]; i++)
        if (c.type[i] != CBSPMV_FMT_COO) { items++; recb += rec[i]; }
      page_chunks[p] = coo_order(c, sh, pb[p], pb[p + 1], order, &cbytes);
      pbytes[p] = round_up(kPageHeader + kDescBytes * (items + page_chunks[p]), 16) + recb + cbytes;
    }
  });
  for (int64_t p = 0; p < npages; p++) {
    off[p + 1] = off[p] + (uint64_t)pbytes[p];
    chunk0[p + 1] = chunk0[p] + page_chunks[p];
  }
  const int64_t total = (int64_t)off[npages], nchunks = chunk0[npages];
  tm.lap("stream: page plan");
  s->nbytes = total;
  s->page_off = off;
  if (plan) {
    plan->meta_off.assign((size_t)npages + 1, 0);
    for (int64_t p = 0; p < npages; p++) {
      const int64_t items = (int64_t)page_chunks[p];
      int64_t n_cd = 0;
      for (int64_t i = pb[p]; i < pb[p + 1]; i++) n_cd += c.type[i] != CBSPMV_FMT_COO;
      plan->meta_off[p + 1] = plan->meta_off[p] + (uint64_t)round_up(kPageHeader + kDescBytes * (items + n_cd), 16);
    }
    plan->meta.assign((size_t)plan->meta_off[npages], 0);
    plan->rec_dst.assign((size_t)c.nb, 0);
    plan->res_dst.assign(c.agg ? (size_t)c.nb : 0, 0);
    plan->ncol = ncol;
    plan->coo_chunk.assign((size_t)c.nb, -1);
    plan->coo_lane.assign((size_t)c.nb, 0);
    plan->coo_member.assign((size_t)c.nb, 0);
    plan->chunk_off.assign((size_t)nchunks, 0);
    plan->chunk_desc.assign((size_t)nchunks, 0);
    plan->runs = runs;
    plan->chunk_nv.assign((size_t)nchunks, 0);
    plan->chunk_nm.assign((size_t)nchunks, 0);
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
  parallel_for(npages, T, 64, [&](int64_t lo, int64_t hi, int) {
    std::vector<Piece> pieces;
    std::vector<int> cnv, cnm;           // per chunk of the page
    std::vector<int64_t> cd;              // CSR / DENSE blocks of the page
    std::vector<int64_t> order;           // its COO blocks in chunk order
    for (int64_t p = lo; p < hi; p++) {
      pieces.clear(); cnv.clear(); cnm.clear(); cd.clear();
      PageAcc a;
      for (int64_t i = pb[p]; i < pb[p + 1]; i++)
        if (c.type[i] != CBSPMV_FMT_COO) cd.push_back(i);
      int64_t cbytes = 0;
      coo_order(c, sh, pb[p], pb[p + 1], order, &cbytes);
      for (int64_t i : order) {
        // at each call a.chunks is the index of the chunk the piece lands in (add_coo closes first)
        sh.add_coo(a, c.nnzb[i], [&](int lane0, int member, int64_t e0, int t) {
          pieces.push_back(Piece{i, e0, a.chunks, lane0, member, t});
        });
      }
      if (a.nv) sh.close_chunk(a);
      cnv.assign((size_t)a.chunks, 0);
      cnm.assign((size_t)a.chunks, 0);
      for (const Piece &pc : pieces) {
        const size_t ch = (size_t)pc.chunk;
        const int t = pc.t;
        cnv[ch] = std::max(cnv[ch], pc.lane0 + t);
        cnm[ch] = std::max(cnm[ch], pc.member + 1);
      }
      const int64_t nch = (int64_t)cnv.size();
      const int64_t nitems = (int64_t)cd.size() + nch;
      const int64_t desc0 = kPageHeader;
      int64_t pos = round_up(kPageHeader + kDescBytes * nitems, 16);
      const int64_t xoff = pbytes[p];
      int64_t xpos = xoff;
      uint8_t *page = plan ? plan->meta.data() + plan->meta_off[p] : s->bytes + off[p];
      if (!plan) std::memset(page, 0, (size_t)pbytes[p]);
      const uint32_t hdr[4] = {(uint32_t)nitems, (uint32_t)cd.size(), (uint32_t)(pb[p + 1] - pb[p]), (uint32_t)pb[p]};
      std::memcpy(page, hdr, 16);
      int64_t it = 0;
      for (int64_t i : cd) {
        const int type = c.type[i];
        const int64_t k = c.nnzb[i];
        const int64_t res = c.agg ? pos : 0;
        if (c.agg) pos += round_up(ncol[i], 4) * 4;
        const int64_t body = pos;
        const int64_t idx = type == CBSPMV_FMT_CSR ? (c.blk + 1) + k : 0;
        const int64_t vals = body + round_up(idx, S);
        uint32_t d[4];
        d[0] = (uint32_t)c.br[i] * (uint32_t)c.blk;
        d[1] = c.agg ? (uint32_t)res : (uint32_t)c.bc[i] * (uint32_t)c.blk;
        d[2] = (uint32_t)body | ((uint32_t)vals << 16);
        d[3] = (uint32_t)type | ((uint32_t)ncol[i] << 2) | ((uint32_t)(k - 1) << 8) |
               (c.agg ? 0u : (uint32_t)xpos << 16);
        std::memcpy(page + desc0 + kDescBytes * it, d, 16);
        it++;
        if (!c.agg) xpos += 16 * (int64_t)x_size;
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
      // COO chunks
      std::vector<int64_t> crec((size_t)nch);
      for (int64_t ch = 0; ch < nch; ch++) {
        const ChunkLayout L = chunk_layout(cnv[ch], cnm[ch], S);
        crec[ch] = pos;
        uint32_t d[4];
        d[0] = (uint32_t)pos | ((uint32_t)cnv[ch] << 16) | ((uint32_t)cnm[ch] << 24);
        d[1] = (uint32_t)(pos + L.rows) | ((uint32_t)(pos + L.cols) << 16);
        d[2] = (uint32_t)(pos + L.vals);
        d[3] = (uint32_t)CBSPMV_FMT_COO;  // the runs flag is set once the elements are in place
        std::memcpy(page + desc0 + kDescBytes * it, d, 16);
        it++;
        if (plan) {
          plan->chunk_off[chunk0[p] + ch] = off[p] + (uint64_t)pos;
          plan->chunk_desc[chunk0[p] + ch] = off[p] + (uint64_t)(desc0 + kDescBytes * (it - 1));
          plan->chunk_nv[chunk0[p] + ch] = (uint8_t)cnv[ch];
          plan->chunk_nm[chunk0[p] + ch] = (uint8_t)cnm[ch];
        }
        pos += L.bytes;
      }
      for (const Piece &pc : pieces) {
        const int64_t ch = pc.chunk;
        const int t = pc.t;
        const int64_t i = pc.block;
        if (plan) {
          if (pc.e0 == 0) {
            plan->coo_chunk[i] = chunk0[p] + ch;
            plan->coo_lane[i] = (uint8_t)pc.lane0;
            plan->coo_member[i] = (uint8_t)pc.member;
          }
          continue;
        }
        const ChunkLayout L = chunk_layout(cnv[ch], cnm[ch], S);
        uint8_t *r = page + crec[ch];
        const uint32_t row0 = (uint32_t)c.br[i] * (uint32_t)c.blk;
        std::memcpy(r + 4 * pc.member, &row0, 4);
        const int64_t k = c.nnzb[i];
        const uint8_t *coord = c.mtx.data() + c.vp[i];
        const uint8_t *vals = coord + round_up(k, S);
        const uint32_t *seg = c.agg ? c.restore.data() + c.cols_offset[c.br[i]] + (uint64_t)c.bc[i] * c.blk : nullptr;
        for (int j = 0; j < t; j++) {
          const int64_t e = pc.e0 + j;
          const int lane = pc.lane0 + j;
          const uint8_t b = coord[e];  // (col << 4) | row
          r[L.rows + lane] = (uint8_t)((pc.member << 4) | (b & 15));
          const uint32_t col = seg ? seg[b >> 4] : (uint32_t)c.bc[i] * (uint32_t)c.blk + (b >> 4);
          std::memcpy(r + L.cols + 4 * lane, &col, 4);
          std::memcpy(r + L.vals + (int64_t)S * lane, vals + e * S, (size_t)S);
        }
      }
      // run steps: the longest run of adjacent elements sharing a global row (a COO record is
      // sorted by (row, col), so a row's elements in one block are adjacent)
      if (!plan && runs) {
        for (int64_t ch = 0; ch < nch; ch++) {
          const ChunkLayout L = chunk_layout(cnv[ch], cnm[ch], S);
          const uint8_t *r = page + crec[ch];
          uint32_t prev = 0xFFFFFFFFu;
          int len = 0, maxrun = 1;
          for (int l = 0; l < cnv[ch]; l++) {
            uint32_t rb;
            std::memcpy(&rb, r + 4 * (r[L.rows + l] >> 4), 4);
            const uint32_t row = rb + (r[L.rows + l] & 15);
            len = row == prev ? len + 1 : 1;
            maxrun = std::max(maxrun, len);
            prev = row;
          }
          uint32_t *dw = reinterpret_cast<uint32_t *>(page + desc0 + kDescBytes * ((int64_t)cd.size() + ch)) + 3;
          *dw |= run_steps(maxrun) << kRunShift;
        }
      }
    }
  });
  tm.lap("stream: fill pages");
  return CBSPMV_OK;
}

}  // namespace cb
