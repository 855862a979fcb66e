"""NEXT-3 device builder (``device_build=1``): the canonical format it produces must equal the
oracle's byte for byte (the same bar as the host builder, tests/test_builder_parity.py), for every
option variant, dtype and column-panel split, and at full BASELINE size it must equal the host
builder's.  Needs a GPU.
"""
import numpy as np
import pytest

import oracle
import paper_2605_18515_b200 as cb
import synth
from tests.test_oracle import CORPUS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KEYS = ["blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
        "restore_cols", "cols_offset", "tb_ptr", "tb_load", "tb_load_natural"]
INFO = ["nb", "nb_pre", "ss_count", "agg", "nnz", "T", "fmt_count", "mtx_bytes", "n_restore", "alg_bytes"]


def _ok():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def compare_to_oracle(A, dtype="f64", **opts):
    _ok()
    o_opts = dict(opts)
    o_opts["val_size"] = 8 if dtype == "f64" else 4
    o_opts.pop("col_panels", None)
    ref = oracle.build(A, **o_opts)
    h = cb.build(A, dtype=dtype, device=0, device_build=1, **opts)
    got = cb.export(h)
    i = h.info
    assert (i["nb"], i["T"], i["agg"], i["nnz"], i["nb_pre"], i["ss_count"]) == \
        (ref.nb, ref.T, ref.agg, ref.nnz, ref.nb_pre, ref.ss_count)
    assert tuple(i["fmt_count"]) == tuple(ref.fmt_count)
    for k in KEYS:
        a, b = got[k], getattr(ref, k)
        assert a.dtype == b.dtype and np.array_equal(a, b), f"{k} differs"
    oracle.free(ref)
    return h


@pytest.mark.parametrize("A", CORPUS, ids=lambda A: A.name)
def test_corpus_default(A):
    compare_to_oracle(A)


@pytest.mark.parametrize("A", CORPUS[::3], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
@pytest.mark.parametrize("ff", [-1, 0, 1, 2])
@pytest.mark.parametrize("bal", [0, 1])
def test_corpus_variants(A, agg, ff, bal):
    compare_to_oracle(A, agg_mode=agg, force_format=ff, balance=bal)


@pytest.mark.parametrize("A", CORPUS[::4], ids=lambda A: A.name)
@pytest.mark.parametrize("dtype", ["f32", "f32f64"])
def test_corpus_fp32_layouts(A, dtype):
    compare_to_oracle(A, dtype=dtype)
    compare_to_oracle(A, dtype=dtype, agg_mode=1)


@pytest.mark.parametrize("name", ["laplace", "rmat", "clustered", "uniform"])
def test_configs_small(name):
    compare_to_oracle(synth.make(name, small=True))


@pytest.mark.parametrize("name", ["rmat", "uniform"])
def test_column_panels_equal_host_build(name):
    _ok()
    A = synth.make(name, small=True)
    hd = cb.build(A, device=0, device_build=1, col_panels=3)
    hh = cb.build(A, device=0, device_build=0, col_panels=3)
    for k in INFO:
        assert hd.info[k] == hh.info[k], k
    for p in range(3):
        ed, eh = cb.export(hd, p), cb.export(hh, p)
        for k in KEYS:
            assert np.array_equal(ed[k], eh[k]), (p, k)


def test_error_statuses_match_host():
    _ok()
    good = synth.random_csr(40, 30, 0.2, 3)
    cases = []
    bad = synth.CSR(good.m, good.n, good.row_ptr.copy(), good.col.copy(), good.val.copy())
    r = int(np.argmax(np.diff(bad.row_ptr) >= 2))
    j = int(bad.row_ptr[r])
    bad.col[j], bad.col[j + 1] = bad.col[j + 1], bad.col[j]  # unsorted
    cases.append(bad)
    bad2 = synth.CSR(good.m, good.n, good.row_ptr.copy(), good.col.copy(), good.val.copy())
    bad2.val[5] = np.inf
    cases.append(bad2)
    bad3 = synth.CSR(good.m, good.n, good.row_ptr.copy(), good.col.copy(), good.val.copy())
    bad3.col[7] = good.n
    cases.append(bad3)
    for B in cases:
        st = []
        for db in (0, 1):
            with pytest.raises(cb.CBSpMVError) as e:
                cb.build(B, device=0, device_build=db)
            st.append(e.value.status)
        assert st[0] == st[1] != 0


def test_degenerate_shapes():
    for A in (synth.CSR(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0)),
              synth.CSR(5, 7, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0)),
              synth.CSR(3, 3, np.array([0, 1, 2, 3], np.int64), np.array([0, 1, 2], np.int32), np.zeros(3))):
        compare_to_oracle(A)
        compare_to_oracle(A, agg_mode=1)


@pytest.mark.parametrize("name", ["clustered", "rmat"])
def test_full_size_equals_host_build_and_spmv(name):
    """BASELINE configs at full size: device build == host build byte for byte; SpMV sampled."""
    _ok()
    A = synth.make(name)
    hd = cb.build(A, device=0, device_build=1)
    hh = cb.build(A, device=0, device_build=0)
    for k in INFO:
        assert hd.info[k] == hh.info[k], k
    ed, eh = cb.export(hd), cb.export(hh)
    for k in KEYS:
        assert np.array_equal(ed[k], eh[k]), k
    del ed, eh
    cb.destroy(hh)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=4)
    xd = torch.from_numpy(x).to("cuda:0")
    y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
    cb.spmv(hd, xd, y)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(2).choice(A.m, size=5000, replace=False))
    y_ref, R = oracle.spmv_rows(A, x, rows)
    assert np.all(np.abs(y.cpu().numpy()[rows] - y_ref) <= 1e-12 * R)


@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [-1, 0, 1])
@pytest.mark.parametrize("dtype", ["f64", "f32f64"])
def test_spmv_device_built_stream_without_host_records(A, agg, dtype):
    """keep_host=0: the records never leave the device (stream filled by fill_stream_device)."""
    _ok()
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=8)
    Ar = A if dtype == "f64" else synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    y_ref, R = oracle.spmv_csr(Ar, x)
    h = cb.build(A, dtype=dtype, device=0, device_build=1, keep_host=0, agg_mode=agg)
    xd = torch.from_numpy(x).to("cuda:0")
    y = torch.full((A.m,), float("nan"), dtype=torch.float64, device="cuda:0")
    cb.spmv(h, xd, y)
    torch.cuda.synchronize()
    assert np.all(np.abs(y.cpu().numpy() - y_ref) <= 1e-12 * R)


@pytest.mark.parametrize("pattern", ["random", "hub", "blockdense"])
def test_exact_integer_bitwise_device_built(pattern):
    _ok()
    A = synth.random_csr(300, 260, 0.08, 17, val_mode=2, pattern=pattern)
    x = synth.vector(A.n, synth.VEC_INT7)
    y_ref, _ = oracle.spmv_csr(A, x)
    for ff in (-1, 0, 1, 2):
        for agg in (0, 1):
            h = cb.build(A, device=0, device_build=1, keep_host=0, force_format=ff, agg_mode=agg)
            y = np.empty(A.m)
            cb.spmv_host(h, x, y)
            assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("A", CORPUS[::3], ids=lambda A: A.name)
@pytest.mark.parametrize("run_max", ["1", "3", "32"])
@pytest.mark.parametrize("hot", ["", "256"])
def test_device_built_coo_slices(A, run_max, hot, monkeypatch):
    """Row-run slices filled on the device (k_coo at the host plan's offsets) on device-built
    handles, for several Lmax, with and without a forced 32-column hot x cache; the stream-decode
    test checks the layout itself."""
    _ok()
    monkeypatch.setenv("CBSPMV_RUN_MAX", run_max)
    if hot:
        monkeypatch.setenv("CBSPMV_HOT_MIN_PCT", "0")
        monkeypatch.setenv("CBSPMV_HOT_BYTES", hot)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=12)
    y_ref, R = oracle.spmv_csr(A, x)
    for agg in (0, 1):
        h = cb.build(A, device=0, device_build=1, keep_host=0, agg_mode=agg)
        y = np.empty(A.m)
        cb.spmv_host(h, x, y)
        assert np.all(np.abs(y - y_ref) <= 1e-12 * R)
        cb.destroy(h)
