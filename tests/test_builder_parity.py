"""The library's host builder (C-ABI, host-only mode) vs the oracle: bit-exact format.

Every array of the canonical format — the five high-level arrays, mtx_data
(including padding bytes), restore_cols, cols_offset, tb_ptr and the per-TB
loads — must equal oracle_build's byte for byte.  Runs on
CPU: ``device=-1`` builds the format without touching a GPU.
"""
import numpy as np
import pytest

import oracle
import paper_2605_18515_b200 as cb
import synth
from tests.test_oracle import CORPUS

KEYS = ["blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
        "restore_cols", "cols_offset", "tb_ptr", "tb_load", "tb_load_natural"]


def compare(A, dtype="f64", **opts):
    o_opts = dict(opts)
    o_opts["val_size"] = 8 if dtype == "f64" else 4
    ref = oracle.build(A, **o_opts)
    h = cb.build(A, dtype=dtype, device=-1, **opts)
    got = cb.export(h)
    info = h.info
    assert info["nb"] == ref.nb and info["T"] == ref.T and info["agg"] == ref.agg
    assert info["nnz"] == ref.nnz and info["nb_pre"] == ref.nb_pre and info["ss_count"] == ref.ss_count
    assert tuple(info["fmt_count"]) == tuple(ref.fmt_count)
    for k in KEYS:
        a, b = got[k], getattr(ref, k)
        assert a.dtype == b.dtype, k
        assert np.array_equal(a, b), f"{k} differs"
    cb.destroy(h)
    oracle.free(ref)
    return info


@pytest.mark.parametrize("A", CORPUS, ids=lambda A: A.name)
def test_corpus_default(A):
    compare(A)


@pytest.mark.parametrize("A", CORPUS[::3], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
@pytest.mark.parametrize("ff", [-1, 0, 1, 2])
@pytest.mark.parametrize("bal", [0, 1])
def test_corpus_variants(A, agg, ff, bal):
    compare(A, agg_mode=agg, force_format=ff, balance=bal)


@pytest.mark.parametrize("A", CORPUS[::4], ids=lambda A: A.name)
@pytest.mark.parametrize("W", [1, 2, 5])
def test_warps_per_tb(A, W):
    compare(A, warps_per_tb=W)


@pytest.mark.parametrize("A", CORPUS[::5], ids=lambda A: A.name)
def test_fp32(A):
    compare(A, dtype="f32")
    compare(A, dtype="f32", agg_mode=1)
    info = compare(A, dtype="f32f64")  # mixed variant (R-24): the fp32 record layout
    assert info["dtype"] == cb.F32F64


def test_fig1_blk4():
    info = compare(synth.fig1(), blk=4, th1=2, th2=8, agg_mode=0, warps_per_tb=2)
    assert info["nb"] == 13 and info["T"] == 7
    compare(synth.fig1())


@pytest.mark.parametrize("name", ["laplace", "rmat", "clustered", "uniform"])
def test_configs_small(name):
    compare(synth.make(name, small=True))


def test_laplace_full():
    info = compare(synth.laplace5(1000))
    assert info["agg"] == 1 and info["nnz"] == 4_996_000


def test_thread_count_invariance():
    A = synth.rmat(12, 16, 7)
    a = cb.export(cb.build(A, device=-1, host_threads=1))
    b = cb.export(cb.build(A, device=-1, host_threads=8))
    for k in KEYS:
        assert np.array_equal(a[k], b[k])


def test_explicit_zeros_dropped():
    A = synth.random_csr(40, 40, 0.3, 9)
    A.val[::3] = 0.0
    info = compare(A)
    assert info["nnz"] == int(np.count_nonzero(A.val))


@pytest.mark.parametrize("case", ["unsorted", "dup", "oob", "neg", "nan", "inf"])
def test_error_status_matches_oracle(case):
    A = synth.random_csr(50, 50, 0.2, 4)
    col, val = A.col.copy(), A.val.copy()
    r = int(np.argmax(np.diff(A.row_ptr) >= 2))
    j = int(A.row_ptr[r])
    if case == "unsorted":
        col[j], col[j + 1] = col[j + 1], col[j]
    elif case == "dup":
        col[j + 1] = col[j]
    elif case == "oob":
        col[j] = 50
    elif case == "neg":
        col[j] = -1
    elif case == "nan":
        val[j] = np.nan
    else:
        val[j] = np.inf
    B = synth.CSR(A.m, A.n, A.row_ptr, col, val)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.build(B)
    with pytest.raises(cb.CBSpMVError) as el:
        cb.build(B, device=-1)
    assert el.value.status == eo.value.status


def test_degenerate_shapes():
    for m, n in [(0, 0), (0, 5), (5, 0), (1, 1), (17, 3), (3, 17)]:
        A = synth.random_csr(m, n, 0.5, 1) if m and n else synth.CSR(m, n, np.zeros(m + 1, np.int64),
                                                                        np.zeros(0, np.int32), np.zeros(0))
        compare(A)


def test_info_bytes():
    A = synth.make("rmat", small=True)
    h = cb.build(A, device=-1)
    i = h.info
    S = 8
    expect = 21 * i["nb"] + i["mtx_bytes"] + 4 * i["n_restore"] + (8 * (i["blk_m"] + 1) if i["agg"] else 0) \
        + S * (i["n"] + i["m"])
    assert i["alg_bytes"] == expect
    assert i["meta_bytes"] == 21 * i["nb"]


def panel_csr(A, c0, c1):
    """Columns [c0, c1) of A with global column indices (test-side slicing)."""
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    keep = (A.col >= c0) & (A.col < c1)
    rp = np.zeros(A.m + 1, np.int64)
    np.add.at(rp, rows[keep] + 1, 1)
    return synth.CSR(A.m, A.n, np.cumsum(rp), A.col[keep].copy(), A.val[keep].copy())


@pytest.mark.parametrize("P", [2, 3, 7])
def test_column_panels_each_equal_oracle(P):
    """NEXT-1 column panels: every panel's format is the oracle's build of A[:, c_k:c_k+1)."""
    A = synth.random_csr(200, 300, 0.08, 41, pattern="hub")
    h = cb.build(A, device=-1, col_panels=P)
    assert h.info["n_panels"] == P
    nbc = (A.n + 15) // 16
    cuts = [min(A.n, (nbc * k // P) * 16) for k in range(P)] + [A.n]
    tot = 0
    for k in range(P):
        Ak = panel_csr(A, cuts[k], cuts[k + 1])
        ref = oracle.build(Ak)
        got = cb.export(h, panel=k)
        for key in KEYS:
            assert np.array_equal(got[key], getattr(ref, key)), (k, key)
        tot += ref.nnz
    assert tot == A.nnz == h.info["nnz"]
