"""Pins for the oracle (oracle/): checks against what the paper and mathematics fix.

No test here retypes the oracle's own formula or re-calls its routine: y is
pinned by numpy dense brute force, closed forms and hand-computed fixtures;
the format by SPEC/paper worked values, an independent Python unpacker of the
record layouts (R-8) and invariants; Alg. 2 by an independently
written O(nb*T) greedy scan.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- corpus
def corpus(max_dim=64, count=60, seed0=1000):
    pats = ["random", "banded", "blockdense", "diag", "row", "col", "empty", "hub"]
    rng = np.random.default_rng(seed0)
    out = []
    for i in range(count):
        m = int(rng.integers(1, max_dim + 1))
        n = int(rng.integers(1, max_dim + 1))
        pat = pats[i % len(pats)]
        dens = float(rng.choice([0.01, 0.05, 0.2, 0.6]))
        out.append(synth.random_csr(m, n, dens, seed0 + i, val_mode=i % 3, pattern=pat))
    return out


CORPUS = corpus()


# ----------------------------------------------------------------------------- independent unpacker
def unpack(cb, B=16, S=8):
    """Decode every block record (R-8 layouts), written independently of oracle.c.

    Returns dict (row, col) -> value over the ORIGINAL column space, and checks
    alignment / zero padding / exact tiling of mtx_data along the way."""
    vt = np.float64 if S == 8 else np.float32
    data = cb.mtx_data.tobytes()
    ent = {}
    spans = []
    for i in range(cb.nb):
        vp, br, bc, k, t = int(cb.vp_per_blk[i]), int(cb.blk_row_idx[i]), int(cb.blk_col_idx[i]), \
            int(cb.nnz_per_blk[i]), int(cb.type_per_blk[i])
        assert vp % S == 0
        if t == 0:
            idx = list(data[vp:vp + k])
            pad = (-k) % S
            assert data[vp + k:vp + k + pad] == b"\0" * pad
            v = np.frombuffer(data, vt, k, vp + k + pad)
            rc = [(b & 15, b >> 4) for b in idx]
            assert rc == sorted(rc), "COO elements not in (row, col) order"
            size = k + pad + k * S
        elif t == 1:
            rp = list(data[vp:vp + B + 1])
            cols = list(data[vp + B + 1:vp + B + 1 + k])
            pad = (-(B + 1 + k)) % S
            assert data[vp + B + 1 + k:vp + B + 1 + k + pad] == b"\0" * pad
            v = np.frombuffer(data, vt, k, vp + B + 1 + k + pad)
            rp[B] = k
            rc = []
            for r in range(B):
                rc += [(r, cols[q]) for q in range(rp[r], rp[r + 1])]
            assert len(rc) == k
            size = B + 1 + k + pad + k * S
        else:
            d = np.frombuffer(data, vt, B * B, vp).reshape(B, B)
            rr, cc = np.nonzero(d)
            rc = list(zip(rr.tolist(), cc.tolist()))
            v = d[rr, cc]
            assert len(rc) == k
            size = B * B * S
        spans.append((vp, size))
        for (lr, lc), val in zip(rc, v):
            row = br * B + lr
            if cb.agg:
                seg0, seg1 = int(cb.cols_offset[br]), int(cb.cols_offset[br + 1])
                a = bc * B + lc
                assert a < seg1 - seg0
                col = int(cb.restore_cols[seg0 + a])
            else:
                col = bc * B + lc
            assert (row, col) not in ent
            ent[(row, col)] = float(val)
    spans.sort()
    pos = 0
    for vp, size in spans:
        assert vp == pos, "records do not tile mtx_data"
        pos += size
    assert pos == len(data)
    return ent


def entries(A, S=8):
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    vals = A.val if S == 8 else A.val.astype(np.float32).astype(np.float64)
    return {(int(r), int(c)): float(v) for r, c, v in zip(rows, A.col, vals) if v != 0}


# ----------------------------------------------------------------------------- independent greedy
def greedy_bruteforce(nnz_natural, W):
    """Alg. 2 written as an O(nb*T) scan: LPT order, pick least (load, tb_id) with a free warp."""
    nb = len(nnz_natural)
    T = (nb + W - 1) // W
    order = sorted(range(nb), key=lambda b: (-nnz_natural[b], b))
    load = [0] * T
    warps = [0] * T
    slot = [None] * nb
    for b in order:
        best = None
        for t in range(T):
            if warps[t] < W and (best is None or (load[t], t) < (load[best], best)):
                best = t
        slot[b] = best * W + warps[best]
        load[best] += nnz_natural[b]
        warps[best] += 1
    return slot, load


# ============================================================================= Alg. 1 (y)
def test_spec_small_products():
    A = synth.from_dense(np.array([[1.0, 2.0], [0.0, 3.0]]))
    y, R = oracle.spmv_csr(A, np.ones(2))
    assert y.tolist() == [3.0, 3.0] and R.tolist() == [3.0, 3.0]
    Z = synth.from_dense(np.zeros((5, 7)))
    y, R = oracle.spmv_csr(Z, np.arange(7.0))
    assert y.tolist() == [0.0] * 5 and R.tolist() == [0.0] * 5
    x = np.random.default_rng(0).standard_normal(9)
    y, _ = oracle.spmv_csr(synth.from_dense(np.eye(9)), x)
    assert np.array_equal(y, x)


@pytest.mark.parametrize("A", CORPUS, ids=lambda A: A.name)
def test_alg1_vs_dense_bruteforce(A):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=7)
    y, R = oracle.spmv_csr(A, x)
    d = A.to_dense()
    yd = d @ x
    Rd = np.abs(d) @ np.abs(x)
    assert np.allclose(y, yd, rtol=0, atol=1e-13 * max(1.0, np.abs(Rd).max()))
    assert np.allclose(R, Rd, rtol=1e-14, atol=0)


def test_alg1_exact_integer_mode():
    A = synth.random_csr(60, 50, 0.3, 5, val_mode=2)
    x = synth.vector(A.n, synth.VEC_INT7)
    y, _ = oracle.spmv_csr(A, x)
    yd = (A.to_dense().astype(np.int64) @ x.astype(np.int64)).astype(np.float64)
    assert np.array_equal(y, yd)


def test_laplacian_closed_form():
    g = 120
    A = synth.laplace5(g)
    assert A.nnz == 5 * g * g - 4 * g
    y, _ = oracle.spmv_csr(A, np.ones(A.n))
    gy, gx = np.divmod(np.arange(g * g), g)
    nb = (gy > 0).astype(int) + (gy < g - 1) + (gx > 0) + (gx < g - 1)
    assert np.array_equal(y, 4.0 - nb)


def test_uniform_ones_closed_form():
    A = synth.uniform(4096, 4096, 50, 51, val_mode=3)
    assert np.all(np.diff(A.row_ptr) == 50)
    y, _ = oracle.spmv_csr(A, np.ones(A.n))
    assert np.all(y == 50.0)


def test_fig1_worked_example():
    g = gold("fig1.json")
    A = synth.fig1()
    assert A.row_ptr.tolist() == g["row_ptr"] and A.nnz == g["nnz"]
    # third non-zero in row-major order is at (0,4)
    assert (0, int(A.col[2])) == (0, 4)
    x = synth.vector(16, synth.VEC_FIG1)
    y, R = oracle.spmv_csr(A, x)
    assert y.tolist() == g["y"] and R.tolist() == g["R"]
    grid = np.zeros((4, 4), int)
    for r in range(16):
        for c in A.col[A.row_ptr[r]:A.row_ptr[r + 1]]:
            grid[r // 4, c // 4] += 1
    assert grid.tolist() == g["blk4_block_nnz_grid"] and int((grid > 0).sum()) == 13


# ============================================================================= format (a2-a6)
def test_spec_vectors_small_pieces():
    s = gold("spec_vectors.json")
    sm = s["storage_model"]
    assert oracle.storage_model(*sm["args"]) == (sm["csr"], sm["bsr"], sm["cb"])
    names = {0: "COO", 1: "CSR", 2: "DENSE"}
    fb = s["format_boundaries"]
    assert [names[oracle.select_format(k)] for k in fb["nnz"]] == fb["format"]
    e = s["encode_0_4"]
    assert oracle.encode_coord(e["row"], e["col"]) == e["byte"]
    for r in range(16):
        for c in range(16):
            b = oracle.encode_coord(r, c)
            assert 0 <= b < 256 and (b & 15, b >> 4) == (r, c)
    assert [oracle.padding(k, 8) for k in range(1, 33)] == s["coo_padding_fp64_nnz_1_to_32"]["padding"]
    for case, mu, sd in s["load_stats"]["cases"]:
        m_, s_, _ = oracle.load_stats(case)
        assert (m_, s_) == (mu, sd)


def _single_block(k, seed=0, rows=16, cols=16):
    rng = np.random.default_rng(seed)
    pos = np.sort(rng.choice(rows * cols, size=k, replace=False))
    return synth.from_coo(16, 16, pos // cols, pos % cols, rng.uniform(0.5, 1.0, k))


def test_coo_record_sizes_and_vp():
    s = gold("spec_vectors.json")
    for k, key in ((13, "nnz13"), (8, "nnz8")):
        cb = oracle.build(_single_block(k), agg_mode=0)
        assert cb.type_per_blk.tolist() == [0] and cb.mtx_data.size == s["coo_record_bytes"][key]
    # two COO blocks of nnz 8 side by side -> vp [0, 72]
    r = np.repeat(np.arange(8), 2)
    c = np.tile([0, 16], 8)
    A = synth.from_coo(16, 32, r, c, np.ones(16))
    cb = oracle.build(A, agg_mode=0, balance=0)
    assert cb.vp_per_blk.tolist() == s["two_coo_nnz8_vp"]["vp"]
    cb = oracle.build(_single_block(200), agg_mode=0)
    assert cb.type_per_blk.tolist() == [2] and cb.mtx_data.size == s["dense_record_bytes_fp64"]["bytes"]


def test_fig1_format_blk16():
    g = gold("fig1.json")
    cb = oracle.build(synth.fig1())
    assert cb.nb == 1 and cb.type_per_blk.tolist() == [1] and not cb.agg
    assert cb.mtx_data.size == g["blk16"]["record_bytes"]
    assert oracle.storage_model(16, 16, 52, 1, 1) == tuple(g["storage_model_16_16_52_1_1"])
    assert unpack(cb) == entries(synth.fig1())


def test_fig1_blk4_alg2():
    g = gold("fig1.json")
    A = synth.fig1()
    nat = oracle.build(A, blk=4, th1=2, th2=8, agg_mode=0, warps_per_tb=2, balance=0)
    assert [[int(a), int(b), int(c)] for a, b, c in zip(nat.blk_row_idx, nat.blk_col_idx, nat.nnz_per_blk)] \
        == g["blk4_natural_blocks"]
    cb = oracle.build(A, blk=4, th1=2, th2=8, agg_mode=0, warps_per_tb=2)
    assert cb.tb_load.tolist() == g["blk4_W2_tb_loads"]
    # pre-LB loads (Fig. 4's sigma is reported on these): natural order, W blocks per TB
    assert cb.tb_load_natural.tolist() == g["blk4_W2_tb_loads_natural"]
    assert nat.tb_load_natural.tolist() == g["blk4_W2_tb_loads_natural"]
    # slot of each natural block: position within TB t is (i - tb_ptr[t])
    slot_of = {}
    for t in range(cb.T):
        for w, i in enumerate(range(cb.tb_ptr[t], cb.tb_ptr[t + 1])):
            slot_of[(int(cb.blk_row_idx[i]), int(cb.blk_col_idx[i]))] = t * 2 + w
    got = [slot_of[(b[0], b[1])] for b in g["blk4_natural_blocks"]]
    assert got == g["blk4_W2_slots_of_natural_blocks"]
    assert cb.tb_ptr[1] - cb.tb_ptr[0] == 1    # TB0 has a hole (R-14)
    cb8 = oracle.build(A, blk=4, th1=2, th2=8, agg_mode=0, warps_per_tb=8)
    assert cb8.tb_load.tolist() == g["blk4_W8_tb_loads"]
    assert cb8.tb_load_natural.tolist() == g["blk4_W8_tb_loads_natural"]
    assert unpack(cb, B=4) == entries(A)
    x = synth.vector(16, synth.VEC_FIG1)
    assert oracle.spmv_cb(cb, x).tolist() == g["y"]


def test_alg2_spec_vector():
    s = gold("spec_vectors.json")["alg2_10_8_3_1_W2"]
    # four blocks in natural (br, bc) order with nnz [10, 8, 3, 1]
    rows, cols = [], []
    for b, k in enumerate(s["nnz_natural"]):
        pos = np.arange(k)
        rows += (pos // 16).tolist()
        cols += (b * 16 + pos % 16).tolist()
    A = synth.from_coo(16, 64, rows, cols, np.ones(len(rows)))
    cb = oracle.build(A, agg_mode=0, warps_per_tb=2)
    assert cb.tb_load.tolist() == s["tb_loads"]
    slots = {}
    for t in range(cb.T):
        for w, i in enumerate(range(cb.tb_ptr[t], cb.tb_ptr[t + 1])):
            slots[int(cb.blk_col_idx[i])] = 2 * t + w
    assert [slots[b] for b in range(4)] == s["slots_of_natural_blocks"]


@pytest.mark.parametrize("W", [1, 2, 3, 8])
@pytest.mark.parametrize("seed", range(12))
def test_alg2_equals_bruteforce_greedy(seed, W):
    A = synth.random_csr(128, 128, 0.25, 300 + seed, pattern="blockdense")
    nat = oracle.build(A, agg_mode=0, balance=0, warps_per_tb=W)
    if nat.nb > 64:
        pytest.skip("brute force only on <= 64 blocks")
    cb = oracle.build(A, agg_mode=0, warps_per_tb=W)
    nnz_nat = nat.nnz_per_blk.tolist()
    slot, load = greedy_bruteforce(nnz_nat, W)
    key_nat = list(zip(nat.blk_row_idx.tolist(), nat.blk_col_idx.tolist()))
    got = {}
    for t in range(cb.T):
        for w, i in enumerate(range(cb.tb_ptr[t], cb.tb_ptr[t + 1])):
            got[(int(cb.blk_row_idx[i]), int(cb.blk_col_idx[i]))] = t * W + w
    assert [got[k] for k in key_nat] == slot
    assert cb.tb_load.tolist() == load


@pytest.mark.parametrize("A", CORPUS, ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
def test_pack_roundtrip_and_invariants(A, agg):
    for ff in (-1, 0, 1, 2):
        cb = oracle.build(A, agg_mode=agg, force_format=ff)
        assert cb.agg == agg
        assert unpack(cb) == entries(A)
        assert int(cb.nnz_per_blk.sum()) == A.nnz
        assert sorted(cb.tb_load.tolist()) == sorted(cb.tb_load.tolist()) and int(cb.tb_load.sum()) == A.nnz
        assert np.all(np.diff(cb.tb_ptr) <= 8) and cb.tb_ptr[-1] == cb.nb
        if ff < 0:
            k = cb.nnz_per_blk
            t = cb.type_per_blk
            assert np.all((t == 0) == (k < 32)) and np.all((t == 2) == (k > 128))
        if agg:
            check_aggregation(A, cb)


def check_aggregation(A, cb):
    """per block row, all-zero columns removed; restore map back to original columns."""
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    for br in range(cb.blk_m):
        sel = (rows // 16) == br
        Ci = np.unique(A.col[sel])
        seg = cb.restore_cols[int(cb.cols_offset[br]):int(cb.cols_offset[br + 1])]
        assert np.array_equal(seg, Ci.astype(np.uint32))
    # every full-width aggregated block has >= 16 nnz (P:433 'at least 16', R-6)
    width = {}
    for br in range(cb.blk_m):
        width[br] = int(cb.cols_offset[br + 1] - cb.cols_offset[br])
    for i in range(cb.nb):
        br, bc = int(cb.blk_row_idx[i]), int(cb.blk_col_idx[i])
        if (bc + 1) * 16 <= width[br]:
            assert cb.nnz_per_blk[i] >= 16


def test_th0_boundary():
    """aggregate iff super-sparse fraction >= 0.15 (R-3)."""
    def mat(n_dense, n_sparse):
        rows, cols = [], []
        for b in range(n_dense):
            pos = np.arange(40)
            rows += (pos // 16).tolist()
            cols += (b * 16 + pos % 16).tolist()
        for b in range(n_sparse):
            rows.append(0)
            cols.append((n_dense + b) * 16)
        nbk = n_dense + n_sparse
        return synth.from_coo(16, 16 * nbk, rows, cols, np.ones(len(rows)))
    assert oracle.build(mat(17, 3)).agg == 1       # 3/20 = 0.15
    assert oracle.build(mat(6, 1)).agg == 0        # 1/7 = 0.1428...
    cb = oracle.build(mat(17, 3))
    assert cb.ss_count == 3 and cb.nb_pre == 20


def test_all_coo_storage_closed_form():
    """for all-COO blocks with nnz = 0 mod 8 the format is exactly 21*nnzb + 9*nnz."""
    rows, cols = [], []
    rng = np.random.default_rng(3)
    for b in range(40):
        k = int(rng.choice([8, 16, 24]))
        pos = np.sort(rng.choice(256, size=k, replace=False))
        rows += ((b % 4) * 16 + pos // 16).tolist()
        cols += ((b // 4) * 16 + pos % 16).tolist()
    A = synth.from_coo(64, 160, rows, cols, np.ones(len(rows)))
    cb = oracle.build(A, agg_mode=0)
    assert set(cb.type_per_blk.tolist()) == {0}
    assert 21 * cb.nb + cb.mtx_data.size == oracle.storage_model(64, 160, A.nnz, cb.nb, 4)[2]


def test_fp32_layout():
    A = synth.random_csr(64, 64, 0.3, 77, pattern="blockdense")
    cb = oracle.build(A, agg_mode=0, val_size=4)
    assert unpack(cb, S=4) == entries(A, S=4)
    cb = oracle.build(_single_block(13), agg_mode=0, val_size=4)
    assert cb.mtx_data.size == 13 + 3 + 13 * 4


def test_lb_improves_balance_reported():
    A = synth.random_csr(512, 512, 0.3, 91, pattern="blockdense")
    cb = oracle.build(A, agg_mode=0)
    _, sd_post, _ = oracle.load_stats(cb.tb_load)
    _, sd_pre, _ = oracle.load_stats(cb.tb_load_natural)
    assert sd_post <= sd_pre


# ============================================================================= Alg. 3/4 (y over the format)
@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
def test_spmv_cb_matches_alg1(A):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=3)
    y_ref, R = oracle.spmv_csr(A, x)
    for agg in (0, 1):
        for ff in (-1, 0, 1, 2):
            for bal in (0, 1):
                cb = oracle.build(A, agg_mode=agg, force_format=ff, balance=bal)
                y = oracle.spmv_cb(cb, x)
                assert np.all(np.abs(y - y_ref) <= 1e-12 * R)


def test_spmv_cb_exact_and_linear():
    A = synth.random_csr(200, 180, 0.1, 12, val_mode=2, pattern="hub")
    x = synth.vector(A.n, synth.VEC_INT7)
    y_ref, _ = oracle.spmv_csr(A, x)
    for agg in (0, 1):
        cb = oracle.build(A, agg_mode=agg)
        y = oracle.spmv_cb(cb, x)
        assert np.array_equal(y, y_ref)
        assert np.array_equal(oracle.spmv_cb(cb, 8.0 * x), 8.0 * y)


def test_laplacian_config_structure():
    """Config 2 (g=1000): the th0 rule aggregates; nnz and y closed form."""
    A = synth.laplace5(1000)
    assert A.nnz == 4_996_000
    cb = oracle.build(A)
    assert cb.agg == 1 and cb.nnz == A.nnz
    y = oracle.spmv_cb(cb, np.ones(A.n))
    y_ref, _ = oracle.spmv_csr(A, np.ones(A.n))
    assert np.array_equal(y, y_ref)


def test_canonical_checks():
    A = synth.from_dense(np.array([[1.0, 0, 2.0], [0, 3.0, 0]]))
    bad = synth.CSR(A.m, A.n, A.row_ptr.copy(), np.array([2, 0, 1], np.int32), A.val.copy())
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(bad)
    assert e.value.status == 2
    oob = synth.CSR(A.m, A.n, A.row_ptr.copy(), np.array([0, 3, 1], np.int32), A.val.copy())
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(oob)
    assert e.value.status == 1
    nan = synth.CSR(A.m, A.n, A.row_ptr.copy(), A.col.copy(), np.array([1.0, np.nan, 3.0]))
    with pytest.raises(oracle.OracleError) as e:
        oracle.build(nan)
    assert e.value.status == 1
    zero = synth.CSR(A.m, A.n, A.row_ptr.copy(), A.col.copy(), np.array([1.0, 0.0, 3.0]))
    cb = oracle.build(zero)
    assert cb.nnz == 2
