"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (BASELINE.json north_star): per row |y - y_ref| <= 1e-12 * R_i in fp64 and
<= 1e-5 * R_i in fp32, R_i = sum_j |a_ij x_j| (the oracle runs in fp64 on the
fp32-rounded A and x for fp32); rows with R_i = 0 must be exactly 0.  In
exact-integer mode every summation order gives identical bits, so y must equal
the oracle bitwise.  Full BASELINE sizes are checked on sampled rows plus
closed forms, in the launch configuration bench.py times.
"""
import numpy as np
import pytest

import oracle
import paper_2605_18515_b200 as cb
import synth
from tests.test_oracle import CORPUS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _ok():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gpu_spmv(A, x, dtype="f64", **opts):
    _ok()
    tdt = torch.float32 if dtype == "f32" else torch.float64
    h = cb.build(A, dtype=dtype, device=0, **opts)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV, tdt)
    yd = torch.full((A.m,), float("nan"), dtype=tdt, device=DEV)  # spmv must overwrite every row
    cb.spmv(h, xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy().astype(np.float64), h


def check_rows(y, y_ref, R, rel):
    assert y.shape == y_ref.shape
    assert np.all(np.isfinite(y))
    diff = np.abs(y - y_ref)
    bad = diff > rel * R
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(f"{bad.sum()} rows out of tolerance; row {i}: y={y[i]!r} ref={y_ref[i]!r} R={R[i]!r}")


def ref32(A, x):
    A32 = synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    return oracle.spmv_csr(A32, x.astype(np.float32).astype(np.float64))


def refmix(A, x):
    """Mixed variant (R-24): the fp64 product of the fp32-rounded matrix with the fp64 x."""
    A32 = synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    return oracle.spmv_csr(A32, x)


# ----------------------------------------------------------------------------- corpus, every variant
@pytest.mark.parametrize("A", CORPUS, ids=lambda A: A.name)
def test_corpus_fp64_default(A):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=5)
    y_ref, R = oracle.spmv_csr(A, x)
    y, _ = gpu_spmv(A, x)
    check_rows(y, y_ref, R, 1e-12)


@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
@pytest.mark.parametrize("ff", [-1, 0, 1, 2])
@pytest.mark.parametrize("bal", [0, 1])
def test_corpus_fp64_variants(A, agg, ff, bal):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=6)
    y_ref, R = oracle.spmv_csr(A, x)
    y, _ = gpu_spmv(A, x, agg_mode=agg, force_format=ff, balance=bal)
    check_rows(y, y_ref, R, 1e-12)


@pytest.mark.parametrize("A", CORPUS[::3], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
@pytest.mark.parametrize("ff", [-1, 0, 1, 2])
def test_corpus_fp32(A, agg, ff):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=8)
    y_ref, R = ref32(A, x)
    y, _ = gpu_spmv(A, x, dtype="f32", agg_mode=agg, force_format=ff)
    check_rows(y, y_ref, R, 1e-5)


@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
@pytest.mark.parametrize("agg", [0, 1])
@pytest.mark.parametrize("ff", [-1, 0, 1, 2])
def test_corpus_mixed_f32_values_f64_accumulation(A, agg, ff):
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=10)
    y_ref, R = refmix(A, x)
    y, h = gpu_spmv(A, x, dtype="f32f64", agg_mode=agg, force_format=ff)
    assert h.info["dtype"] == cb.F32F64
    check_rows(y, y_ref, R, 1e-12)


@pytest.mark.parametrize("pattern", ["random", "hub", "blockdense", "banded"])
@pytest.mark.parametrize("dtype", ["f64", "f32", "f32f64"])
@pytest.mark.parametrize("agg", [0, 1])
def test_exact_integer_mode_bitwise(pattern, dtype, agg):
    A = synth.random_csr(300, 260, 0.08, 17, val_mode=2, pattern=pattern)
    x = synth.vector(A.n, synth.VEC_INT7)
    y_ref, _ = oracle.spmv_csr(A, x)
    for ff in (-1, 0, 1, 2):
        y, _ = gpu_spmv(A, x, dtype=dtype, agg_mode=agg, force_format=ff)
        assert np.array_equal(y, y_ref)


def test_fig1_fixture_all_paths():
    A = synth.fig1()
    x = synth.vector(16, synth.VEC_FIG1)
    y_ref, _ = oracle.spmv_csr(A, x)
    for ff in (-1, 0, 1, 2):
        y, h = gpu_spmv(A, x, force_format=ff)
        assert y.tolist() == y_ref.tolist()


# ----------------------------------------------------------------------------- API semantics
def test_add_scaled_host_and_sumsq():
    _ok()
    A = synth.random_csr(500, 400, 0.05, 21, pattern="hub")
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=2)
    y_ref, R = oracle.spmv_csr(A, x)
    h = cb.build(A, device=0)
    xd = torch.from_numpy(x).to(DEV)
    y0 = torch.from_numpy(synth.vector(A.m, synth.VEC_UNIFORM, seed=9)).to(DEV)
    y = y0.clone()
    cb.spmv_add(h, xd, y)
    torch.cuda.synchronize()
    y0h = y0.cpu().numpy()
    assert np.all(np.abs((y.cpu().numpy() - y0h) - y_ref) <= 1e-12 * (R + np.abs(y0h)))
    # scaled: y := A (x / sqrt(ss)) with ss = 4 -> A x / 2 exactly (power-of-two scale)
    ss = torch.tensor([4.0], dtype=torch.float64, device=DEV)
    ys = torch.empty(A.m, dtype=torch.float64, device=DEV)
    cb.spmv_scaled(h, xd, ss, ys)
    yu = torch.empty_like(ys)
    cb.spmv(h, xd, yu)
    torch.cuda.synchronize()
    check_rows(ys.cpu().numpy() * 2.0, y_ref, R, 1e-12)
    # host buffers end to end
    yh = np.empty(A.m, np.float64)
    cb.spmv_host(h, x, yh)
    check_rows(yh, y_ref, R, 1e-12)
    # sumsq
    out = torch.zeros(1, dtype=torch.float64, device=DEV)
    cb.sumsq(xd, out)
    torch.cuda.synchronize()
    assert abs(out.item() - float(np.dot(x, x))) <= 1e-12 * float(np.dot(x, x))


def test_non_default_stream_and_repeat():
    _ok()
    A = synth.make("rmat", small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=4)
    y_ref, R = oracle.spmv_csr(A, x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h = cb.build(A, device=0)
        xd = torch.from_numpy(x).to(DEV)
        ys = [torch.empty(A.m, dtype=torch.float64, device=DEV) for _ in range(3)]
        for y in ys:
            cb.spmv(h, xd, y)
    s.synchronize()
    for y in ys:
        check_rows(y.cpu().numpy(), y_ref, R, 1e-12)


def test_degenerate():
    _ok()
    for m, n in [(0, 5), (5, 1), (1, 1), (17, 3), (3, 17), (33, 2000)]:
        A = synth.random_csr(m, n, 0.5, 3) if m else synth.CSR(0, n, np.zeros(1, np.int64), np.zeros(0, np.int32),
                                                              np.zeros(0))
        x = synth.vector(n, synth.VEC_UNIFORM, seed=1)
        y_ref, R = oracle.spmv_csr(A, x)
        y, _ = gpu_spmv(A, x)
        check_rows(y, y_ref, R, 1e-12)
    Z = synth.CSR(40, 40, np.zeros(41, np.int64), np.zeros(0, np.int32), np.zeros(0))
    y, h = gpu_spmv(Z, np.ones(40))
    assert np.all(y == 0.0) and h.info["nb"] == 0


def test_dense_block_in_partial_last_block_row():
    """m not a multiple of 16: the dense path must not write rows >= m."""
    _ok()
    d = np.zeros((37, 40))
    d[32:37, 16:32] = np.arange(1, 81).reshape(5, 16)
    d[0:16, 0:16] = 1.0
    A = synth.from_dense(d)
    x = synth.vector(40, synth.VEC_INT7)
    y_ref, _ = oracle.spmv_csr(A, x)
    tdt = torch.float64
    h = cb.build(A, device=0, force_format=2)
    guard = torch.full((48,), 7.0, dtype=tdt, device=DEV)
    cb.spmv(h, torch.from_numpy(x).to(DEV), guard[:37])
    torch.cuda.synchronize()
    g = guard.cpu().numpy()
    assert np.array_equal(g[:37], y_ref) and np.all(g[37:] == 7.0)


# ----------------------------------------------------------------------------- device layout
def decode_stream(stream, page_off):
    """Decode the device page stream, version 3 (cb_internal.h): per page its header,
    item descriptors, CSR / DENSE records and COO row-run slices."""
    pages = []
    for p in range(len(page_off) - 1):
        pg = stream[int(page_off[p]):int(page_off[p + 1])]
        nitems, ncd, nblk, blk0 = (int(v) for v in pg[:16].view(np.uint32))
        desc = pg[16:16 + 16 * nitems].view(np.uint32).reshape(nitems, 4)
        items = []
        for a, b, c, d in (tuple(int(v) for v in row) for row in desc):
            t, xslot = d & 3, d >> 16
            if t == 0:
                items.append(dict(type=0, tab=a & 0xFFFF, nl=(a >> 16) & 0xFF, w=a >> 24, cols=b & 0xFFFF,
                                  vals=b >> 16, E=c, d=d))
            else:
                items.append(dict(type=t, row0=a, xinfo=b, body=c & 0xFFFF, vals=c >> 16, ncols=(d >> 2) & 31,
                                  nnz=((d >> 8) & 0xFF) + 1, xslot=xslot))
        pages.append(dict(page=pg, nitems=nitems, ncd=ncd, nblk=nblk, blk0=blk0, items=items))
    return pages


def decode_slice(pg, it, S, vdt, hot=None):
    """One COO slice: its pieces (row, length) and, per piece, its elements (column, value) in step
    order -- element (lane l, step j) at off_j + (lanes below l whose piece is longer than j); a
    column with bit 31 set is slot s of the hot x columns (cb.hot_columns)."""
    nl = it["nl"]
    rows = pg[it["tab"]:it["tab"] + 4 * nl].view(np.uint32).astype(np.int64)
    lens = pg[it["tab"] + 4 * nl:it["tab"] + 5 * nl].astype(np.int64)
    E = int(lens.sum())
    cols = pg[it["cols"]:it["cols"] + 4 * E].view(np.uint32).astype(np.int64)
    is_hot = cols >= 1 << 31
    if is_hot.any():
        cols[is_hot] = hot[cols[is_hot] - (1 << 31)]
    vals = pg[it["vals"]:it["vals"] + S * E].view(vdt)
    elems = [[] for _ in range(nl)]
    off = 0
    for j in range(int(lens.max()) if nl else 0):
        act = np.flatnonzero(lens > j)
        for r, l in enumerate(act):
            elems[l].append((int(cols[off + r]), float(vals[off + r])))
        off += len(act)
    return rows, lens, elems


def _one_block_row_matrix():
    """One block row, 40 block columns, one entry per block: 16 rows with runs of 2 or 3."""
    rows = np.arange(40) % 16
    cols = np.arange(40) * 16 + (np.arange(40) % 5)
    return synth.from_coo(16, 640, rows, cols, np.linspace(1.0, 2.0, 40), name="one_block_row")


def _long_run_matrix():
    """Row 3 holds 200 entries, one per block column (200 one-entry COO blocks of block row 0):
    one run of 200 elements, cut into pieces of Lmax."""
    cols = np.arange(200) * 16 + 7
    return synth.from_coo(16, 3200, np.full(200, 3), cols, np.linspace(-1.0, 1.0, 200), name="long_run")


@pytest.mark.parametrize("name", ["laplace", "rmat", "clustered", "one_block_row", "long_run", "corpus_hub",
                                  "corpus_diag"])
@pytest.mark.parametrize("dtype", ["f64", "f32f64"])
@pytest.mark.parametrize("device_build", [0, 1])
@pytest.mark.parametrize("runopt", ["", "RUN_MAX=7", "RUN_MAX=32", "RUN_ORDER=row", "HOT_MIN_PCT=0",
                                    "HOT_MIN_PCT=0,HOT_BYTES=256", "XAGG=1", "XAGG=0"])
def test_device_stream_encodes_canonical_format(name, dtype, device_build, runopt, monkeypatch):
    """What is on the device is exactly the canonical format (slot order): pages tile the slot
    order; CSR / DENSE records byte-equal (DENSE re-laid lane-major), their restore entries equal
    restore_cols; the COO slices hold exactly the page's COO elements, each with its original
    column (restore_cols resolved), grouped into row runs (a row's elements in slot order, then
    canonical order), cut into pieces of Lmax, ordered (length desc, row asc) or by row, 32 pieces
    per slice.  device_build=1: the stream is filled on the device from the device-built records."""
    _ok()
    run_max = 8  # kDefaultRunMax
    for kv in filter(None, runopt.split(",")):
        k, v = kv.split("=")
        monkeypatch.setenv("CBSPMV_" + k, v)
        run_max = int(v) if k == "RUN_MAX" else run_max
    row_order = runopt == "RUN_ORDER=row"
    if name == "one_block_row":
        A = _one_block_row_matrix()
    elif name == "long_run":
        A = _long_run_matrix()
    elif name == "corpus_hub":
        A = synth.random_csr(300, 260, 0.08, 17, pattern="hub")
    elif name == "corpus_diag":
        A = synth.random_csr(64, 64, 0.05, 3, pattern="diag")
    else:
        A = synth.make(name, small=True)
    opts = {"agg_mode": 0} if name in ("one_block_row", "long_run") else {}  # one-entry blocks stay apart
    h = cb.build(A, dtype=dtype, device=0, device_build=device_build, **opts)
    ex = cb.export(h)
    s, po = cb.download_stream(h)
    hot = cb.hot_columns(h).astype(np.int64)
    assert h.info["n_hot"] == len(hot) and np.all(np.diff(hot) > 0)
    if runopt.startswith("HOT_MIN_PCT=0") and h.info["agg"]:  # forced cache (non-aggregated: no room)
        n_coo = int(np.sum(ex["nnz_per_blk"][ex["type_per_blk"] == 0]))
        assert (len(hot) > 0) == (n_coo > 0)
        assert len(hot) <= (32 if "HOT_BYTES" in runopt else 8192)
    if name == "one_block_row":
        assert ex["nb"] == 40
    pages = decode_stream(s, po)
    S = 8 if dtype == "f64" else 4
    vdt = np.float64 if S == 8 else np.float32
    xs = 8  # x / y element bytes (f64 and f32f64)
    agg = h.info["agg"]
    n_cd = int(np.sum(ex["type_per_blk"] != 0))
    xagg = bool(agg) and (runopt == "XAGG=1" or (runopt != "XAGG=0" and n_cd * 10 >= ex["nb"]))
    xtiles = not agg or xagg
    mtx, vp = ex["mtx_data"], ex["vp_per_blk"].astype(np.int64)
    nxt = 0
    shapes = []
    for P in pages:
        pg = P["page"]
        assert P["blk0"] == nxt and P["nblk"] > 0
        blocks = range(P["blk0"], P["blk0"] + P["nblk"])
        nxt += P["nblk"]
        assert len(pg) % 16 == 0
        cd = [i for i in blocks if ex["type_per_blk"][i] != 0]
        items_cd = [it for it in P["items"] if it["type"] != 0]
        slices = [it for it in P["items"] if it["type"] == 0]
        assert [it["type"] for it in P["items"]] == [1 if ex["type_per_blk"][i] == 1 else 2 for i in cd] + [0] * len(slices)
        assert P["ncd"] == len(cd)
        # x tiles (CSR / DENSE items of non-aggregated matrices, and of aggregated ones with
        # >= 10 % CSR / DENSE blocks or CBSPMV_XAGG=1): 16 values each, consecutive after the page
        end = len(pg)
        for it in P["items"]:
            if it["type"] and xtiles:
                assert it["xslot"] == end
                end += 16 * xs
            elif it["type"]:
                assert it["xslot"] == 0
        for i, it in zip(cd, items_cd):
            br, bc, nnz, typ = (int(ex[k][i]) for k in ("blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk"))
            assert it["row0"] == 16 * br and it["nnz"] == nnz
            idx = 17 + nnz if typ == 1 else 0
            assert it["vals"] == it["body"] + idx + (-idx) % S and it["body"] % 16 == 0
            size = idx + (-idx) % S + (256 if typ == 2 else nnz) * S
            if agg:
                seg0 = int(ex["cols_offset"][br]) + 16 * bc
                ncols = min(16, int(ex["cols_offset"][br + 1]) - seg0)
                rest = pg[it["xinfo"]:it["xinfo"] + 4 * ncols].view(np.uint32)
                assert np.array_equal(rest, ex["restore_cols"][seg0:seg0 + ncols])
            else:
                ncols = min(16, A.n - 16 * bc)
                assert it["xinfo"] == 16 * bc
            assert it["ncols"] == ncols
            dev_rec = pg[it["body"]:it["body"] + size]
            if typ == 2:  # lane-major pairs: value (q*32 + l)*2 + h holds A[l % 16][(l // 16) * 8 + 2q + h]
                j = np.arange(256)
                pair, hh = np.divmod(j, 2)
                q, l = np.divmod(pair, 32)
                src = (l % 16) * 16 + (l // 16) * 8 + 2 * q + hh
                dev_rec = dev_rec.view(vdt)[np.argsort(src)].view(np.uint8)
            assert np.array_equal(dev_rec, mtx[vp[i]:vp[i] + size])
        # the page's COO elements per row, in slot order then canonical order: (original column, value)
        want = {}
        for i in blocks:
            if ex["type_per_blk"][i] != 0:
                continue
            br, bc, k = int(ex["blk_row_idx"][i]), int(ex["blk_col_idx"][i]), int(ex["nnz_per_blk"][i])
            coord = mtx[vp[i]:vp[i] + k].astype(np.int64)
            vals = mtx[vp[i] + k + (-k) % S:vp[i] + k + (-k) % S + k * S].view(vdt)
            cols = (ex["restore_cols"][int(ex["cols_offset"][br]) + 16 * bc + (coord >> 4)].astype(np.int64) if agg
                    else 16 * bc + (coord >> 4))
            for r, c_, v in zip((16 * br + (coord & 15)).tolist(), cols.tolist(), vals.tolist()):
                want.setdefault(r, []).append((c_, v))
        pieces, got = [], {}
        tab = 16 + 16 * P["nitems"]
        for n_s, it in enumerate(slices):
            assert it["d"] == 0 and it["tab"] == tab
            rows, lens, elems = decode_slice(pg, it, S, vdt, hot)
            tab += (5 * it["nl"] + 3) // 4 * 4
            assert 1 <= it["nl"] <= 32 and (it["nl"] == 32 or n_s == len(slices) - 1)
            assert np.all(lens >= 1) and np.all(lens <= run_max)
            assert it["w"] == lens.max() and it["E"] == lens.sum()
            assert it["vals"] == it["cols"] + (4 * it["E"] + 7) // 8 * 8
            shapes.append((it["nl"], it["w"]))
            for r, ln, el in zip(rows.tolist(), lens.tolist(), elems):
                pieces.append((r, ln))
                got.setdefault(r, []).append(el)
        # pieces: a row's run cut into pieces of Lmax (the last shorter), in the piece order
        key = (lambda pc: pc[0]) if row_order else (lambda pc: (-pc[1], pc[0]))
        assert pieces == sorted(pieces, key=key)
        assert sorted(got) == sorted(want)
        for r, run in want.items():
            assert [len(e) for e in got[r]] == [min(run_max, len(run) - q) for q in range(0, len(run), run_max)]
            assert [e for piece in got[r] for e in piece] == run
    assert nxt == ex["nb"]
    if name == "one_block_row":  # rows 0-7 hold 3 entries, 8-15 hold 2: one slice of 16 pieces
        assert shapes == [(16, 3)] if run_max >= 3 else True
    if name == "long_run" and not row_order:
        assert sum(nl for nl, _ in shapes) == -(-200 // run_max)


# ----------------------------------------------------------------------------- BASELINE configs
@pytest.mark.parametrize("name", ["laplace", "rmat", "clustered", "uniform"])
@pytest.mark.parametrize("dtype", ["f64", "f32", "f32f64"])
def test_configs_small_full_check(name, dtype):
    A = synth.make(name, small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=12)
    ref = {"f64": oracle.spmv_csr, "f32": ref32, "f32f64": refmix}[dtype]
    y_ref, R = ref(A, x)
    y, h = gpu_spmv(A, x, dtype=dtype)
    check_rows(y, y_ref, R, 1e-5 if dtype == "f32" else 1e-12)


def test_laplace_config2_full():
    """Config 2 at full size: x = 1 closed form (exact) and random x vs the oracle."""
    A = synth.laplace5(1000)
    y, h = gpu_spmv(A, np.ones(A.n))
    g = 1000
    gy, gx = np.divmod(np.arange(g * g), g)
    nb = (gy > 0).astype(int) + (gy < g - 1) + (gx > 0) + (gx < g - 1)
    assert h.info["agg"] == 1
    assert np.array_equal(y, 4.0 - nb)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=21)
    y_ref, R = oracle.spmv_csr(A, x)
    y, _ = gpu_spmv(A, x)
    check_rows(y, y_ref, R, 1e-12)


def sampled(A, y, x, rel, k=20000, seed=0):
    rows = np.sort(np.random.default_rng(seed).choice(A.m, size=min(k, A.m), replace=False))
    rows = np.unique(np.concatenate([rows, [0, 1, 2, A.m - 1]]))  # hub rows of R-MAT are low ids
    y_ref, R = oracle.spmv_rows(A, x, rows)
    check_rows(y[rows], y_ref, R, rel)


def test_rmat_config3_full_sampled():
    """Config 3 (bench workload) at full size: sampled rows + the x = 1 row-sum identity."""
    A = synth.make("rmat")
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=32)
    y, h = gpu_spmv(A, x)
    assert h.info["agg"] == 1
    sampled(A, y, x, 1e-12)
    y1, _ = gpu_spmv(A, np.ones(A.n))
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    rs = np.bincount(rows, weights=np.abs(A.val), minlength=A.m)
    sums = np.bincount(rows, weights=A.val, minlength=A.m)
    assert np.all(np.abs(y1 - sums) <= 1e-12 * rs)


@pytest.mark.parametrize("dtype", ["f64", "f32", "f32f64"])
def test_clustered_config4_full_sampled(dtype):
    A = synth.make("clustered")
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=42)
    y, h = gpu_spmv(A, x, dtype=dtype)
    assert h.info["agg"] == 0 and min(h.info["fmt_count"]) > 0
    if dtype == "f64":
        sampled(A, y, x, 1e-12)
    elif dtype == "f32f64":
        sampled(synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64)), y, x, 1e-12)
    else:
        rows = np.sort(np.random.default_rng(1).choice(A.m, size=20000, replace=False))
        A32 = synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
        y_ref, R = oracle.spmv_rows(A32, x.astype(np.float32).astype(np.float64), rows)
        check_rows(y[rows], y_ref, R, 1e-5)


@pytest.mark.parametrize("ff", [0, 2])
def test_stage_round_race_regression(ff):
    """Regression for the page-ring stage-round aliasing race: it showed with
    forced COO / DENSE formats in natural (balance = 0) order at >= 1 M rows -- groups then run
    out of lockstep -- as a wrong y, then illegal addresses after a few launches.  Ten
    back-to-back launches on 2^20 rows, every one checked against the oracle on all rows."""
    _ok()
    A = synth.clustered(1 << 20)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=13)
    y_ref, R = oracle.spmv_csr(A, x)
    h = cb.build(A, device=0, force_format=ff, balance=0, agg_mode=0)
    xd = torch.from_numpy(x).to(DEV)
    ys = [torch.full((A.m,), float("nan"), dtype=torch.float64, device=DEV) for _ in range(10)]
    for y in ys:
        cb.spmv(h, xd, y)
    torch.cuda.synchronize()
    for y in ys:
        check_rows(y.cpu().numpy(), y_ref, R, 1e-12)
    cb.destroy(h)


@pytest.mark.parametrize("name", ["clustered", "rmat"])
def test_x_not_16_byte_aligned(name):
    """x only 8-byte aligned: the tile gather falls back from TMA bulk copies to LDGSTS."""
    _ok()
    A = synth.make(name, small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=5)
    y_ref, R = oracle.spmv_csr(A, x)
    h = cb.build(A, device=0)
    buf = torch.zeros(A.n + 1, dtype=torch.float64, device=DEV)
    buf[1:] = torch.from_numpy(x).to(DEV)
    xs = buf[1:]
    assert xs.data_ptr() % 16 == 8
    y = torch.empty(A.m, dtype=torch.float64, device=DEV)
    cb.spmv(h, xs, y)
    torch.cuda.synchronize()
    check_rows(y.cpu().numpy(), y_ref, R, 1e-12)


def test_power_iteration_device_matches_recurrence():
    """configs[4] driver (N=1): spmv_scaled + sumsq, step by step against the numpy recurrence."""
    _ok()
    from paper_2605_18515_b200 import dist as cbd
    A = synth.uniform(1 << 13, 1 << 13, 50, 51, val_mode=1)
    h = cb.build(A, device=0)
    x0 = torch.ones(A.n, dtype=torch.float64, device=DEV)
    lams = []
    x, ss = cbd.power_iteration_device(h, x0, 30, on_step=lambda k, x, s: lams.append(float(s.item()) ** 0.5))
    d = A.to_dense()
    xr, ssr, ref = np.ones(A.n), float(A.n), []
    for _ in range(30):
        yr = d @ (xr / np.sqrt(ssr))
        ssr = float(yr @ yr)
        xr = yr
        ref.append(np.sqrt(ssr))
    assert np.allclose(lams, ref, rtol=1e-12)
    assert np.allclose(x.cpu().numpy(), xr, rtol=1e-11, atol=0)
    rs = d.sum(1)
    assert rs.min() - 1e-9 <= lams[-1] <= rs.max() + 1e-9


def test_power_iteration_exact_ones_fixed_point():
    """All-ones values, exactly 50 per row, n = 4096: every quantity is a dyadic rational
    (1/64, 50/64, 2500), so lambda = 50 exactly at every step, in any summation order."""
    _ok()
    from paper_2605_18515_b200 import dist as cbd
    A = synth.uniform(1 << 12, 1 << 12, 50, 51, val_mode=3)
    h = cb.build(A, device=0)
    lams = []
    cbd.power_iteration_device(h, torch.ones(A.n, dtype=torch.float64, device=DEV), 10,
                               on_step=lambda k, x, s: lams.append(float(s.item()) ** 0.5))
    assert lams == [50.0] * 10


@pytest.mark.parametrize("P", [2, 5])
@pytest.mark.parametrize("name", ["rmat", "clustered", "uniform"])
def test_column_panels_spmv_fp32(P, name):
    A = synth.make(name, small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=9)
    y_ref, R = ref32(A, x)
    y, h = gpu_spmv(A, x, dtype="f32", col_panels=P)
    check_rows(y, y_ref, R, 1e-5)


@pytest.mark.parametrize("P", [2, 5])
@pytest.mark.parametrize("name", ["rmat", "clustered", "uniform"])
def test_column_panels_spmv(P, name):
    """NEXT-1 column panels: y = sum over panels, zeroed once; scaled and add variants too."""
    _ok()
    A = synth.make(name, small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=9)
    y_ref, R = oracle.spmv_csr(A, x)
    y, h = gpu_spmv(A, x, col_panels=P)
    assert h.info["n_panels"] == P
    check_rows(y, y_ref, R, 1e-12)
    xd = torch.from_numpy(x).to(DEV)
    ss = torch.tensor([4.0], dtype=torch.float64, device=DEV)
    ys = torch.empty(A.m, dtype=torch.float64, device=DEV)
    cb.spmv_scaled(h, xd, ss, ys)
    torch.cuda.synchronize()
    check_rows(ys.cpu().numpy() * 2.0, y_ref, R, 1e-12)


@pytest.mark.parametrize("P", [1, 3])
def test_mixed_host_scaled_and_panels(P):
    """Mixed variant through spmv_host (fp64 host buffers), spmv_scaled and column panels."""
    _ok()
    A = synth.make("rmat", small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=13)
    y_ref, R = refmix(A, x)
    h = cb.build(A, dtype="f32f64", device=0, col_panels=P)
    assert h.info["n_panels"] == P
    y = np.empty(A.m)
    cb.spmv_host(h, x, y)
    check_rows(y, y_ref, R, 1e-12)
    xd = torch.from_numpy(x).to(DEV)
    ss = torch.tensor([4.0], dtype=torch.float64, device=DEV)
    ys = torch.empty(A.m, dtype=torch.float64, device=DEV)
    cb.spmv_scaled(h, xd, ss, ys)
    torch.cuda.synchronize()
    check_rows(ys.cpu().numpy() * 2.0, y_ref, R, 1e-12)


@pytest.mark.parametrize("P", [1, 3])
def test_power_iteration_overlapped_panels_device(P):
    """NEXT-1 (i) driver on the device (N=1: panels in order, no broadcasts) == the recurrence;
    the all-ones matrix keeps lambda = 50 exactly through cbspmv_spmv_panel as well."""
    _ok()
    from paper_2605_18515_b200 import dist as cbd
    A = synth.uniform(1 << 13, 1 << 13, 50, 51, val_mode=1)
    h = cb.build(A, device=0, col_panels=P)
    assert h.info["n_panels"] == P
    x, ss = cbd.power_iteration_overlapped(h, torch.ones(A.n, dtype=torch.float64, device=DEV), 20)
    d = A.to_dense()
    xr, ssr = np.ones(A.n), float(A.n)
    for _ in range(20):
        yr = d @ (xr / np.sqrt(ssr))
        ssr = float(yr @ yr)
        xr = yr
    assert np.isclose(float(ss.item()), ssr, rtol=1e-12)
    assert np.allclose(x.cpu().numpy(), xr, rtol=1e-11, atol=0)
    B = synth.uniform(1 << 12, 1 << 12, 50, 51, val_mode=3)
    hb = cb.build(B, device=0, col_panels=P)
    lams = []
    cbd.power_iteration_overlapped(hb, torch.ones(B.n, dtype=torch.float64, device=DEV), 6,
                                   on_step=lambda k, x, s: lams.append(float(s.item()) ** 0.5))
    assert lams == [50.0] * 6


def test_spmv_panel_sum_equals_spmv():
    _ok()
    A = synth.random_csr(3000, 2600, 0.01, 17, val_mode=2, pattern="hub")  # exact-integer values
    x = synth.vector(A.n, synth.VEC_INT7)
    h = cb.build(A, device=0, col_panels=4)
    xd = torch.from_numpy(x).to(DEV)
    y = torch.full((A.m,), float("nan"), dtype=torch.float64, device=DEV)
    for k in range(4):
        cb.spmv_panel(h, k, xd, None, y, k == 0)
    torch.cuda.synchronize()
    y_ref, _ = oracle.spmv_csr(A, x)
    assert np.array_equal(y.cpu().numpy(), y_ref)  # exact-integer data: bitwise
    assert [cb.panel_bounds(h, k)[0] for k in range(4)][0] == 0 and cb.panel_bounds(h, 3)[1] == A.n


@pytest.mark.parametrize("count", [0, 1, 2, 5])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_spmv_host_batch_pipelined(count, dtype):
    """cbspmv_spmv_host_batch: every request's y equals the oracle's, with repeated host
    buffers, odd counts and the two staging slots alternating."""
    _ok()
    A = synth.make("clustered", small=True)
    h = cb.build(A, dtype=dtype, device=0)
    vt = np.float32 if dtype == "f32" else np.float64
    rel = 1e-5 if dtype == "f32" else 1e-12

    def ref(x):
        return ref32(A, x) if dtype == "f32" else oracle.spmv_csr(A, x)

    xs = [synth.vector(A.n, synth.VEC_UNIFORM, seed=100 + k).astype(vt) for k in range(max(count, 1))]
    ys = [np.full(A.m, np.nan, vt) for _ in range(max(count, 1))]
    cb.spmv_host_batch(h, xs[:count], ys[:count])
    for k in range(count):
        y_ref, R = ref(xs[k].astype(np.float64))
        check_rows(ys[k].astype(np.float64), y_ref, R, rel)
    if count == 0:
        assert np.isnan(ys[0]).all()
    # the same host buffers reused across requests (a ring), as bench.py does
    ring_y = [np.empty(A.m, vt) for _ in range(2)]
    cb.spmv_host_batch(h, [xs[0]] * 3, [ring_y[k % 2] for k in range(3)])
    y_ref, R = ref(xs[0].astype(np.float64))
    for yk in ring_y:
        check_rows(yk.astype(np.float64), y_ref, R, rel)
    cb.destroy(h)


_RUNOPTS = [{"CBSPMV_COO_RUNS": "0"}, {"CBSPMV_RUN_MAX": "1"}, {"CBSPMV_RUN_MAX": "2"}, {"CBSPMV_RUN_MAX": "5"},
            {}, {"CBSPMV_RUN_MAX": "32"}, {"CBSPMV_RUN_MAX": "255"}, {"CBSPMV_RUN_ORDER": "row"},
            {"CBSPMV_RUN_ORDER": "row", "CBSPMV_RUN_MAX": "3"}, {"CBSPMV_HOT_MIN_PCT": "0"},
            {"CBSPMV_HOT_MIN_PCT": "0", "CBSPMV_HOT_BYTES": "256"}, {"CBSPMV_HOT_BYTES": "0"},
            {"CBSPMV_XAGG": "1"}, {"CBSPMV_XAGG": "1", "CBSPMV_CSR_PAIR": "0"}]
_runid = lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()) or "default"


@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
@pytest.mark.parametrize("dtype", ["f64", "f32", "f32f64"])
@pytest.mark.parametrize("runopt", _RUNOPTS, ids=_runid)
def test_coo_slice_options(A, dtype, runopt, monkeypatch):
    """COO row-run slices under every build option: Lmax (1 = one RED per element), the piece
    order (length desc / row), CBSPMV_COO_RUNS=0 (= Lmax 1)."""
    for k, v in runopt.items():
        monkeypatch.setenv(k, v)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=5)
    for agg in (0, 1):
        y, h = gpu_spmv(A, x, dtype=dtype, agg_mode=agg)
        if dtype == "f32":
            y_ref, R = ref32(A, x)
            check_rows(y, y_ref, R, 1e-5)
        else:
            A_ = A if dtype == "f64" else synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
            y_ref, R = oracle.spmv_csr(A_, x)
            check_rows(y, y_ref, R, 1e-12)


@pytest.mark.parametrize("pattern", ["random", "hub", "banded"])
@pytest.mark.parametrize("runopt", _RUNOPTS, ids=_runid)
def test_coo_slices_exact_integer_bitwise(pattern, runopt, monkeypatch):
    for k, v in runopt.items():
        monkeypatch.setenv(k, v)
    A = synth.random_csr(300, 260, 0.08, 17, val_mode=2, pattern=pattern)
    x = synth.vector(A.n, synth.VEC_INT7)
    y_ref, _ = oracle.spmv_csr(A, x)
    for agg in (0, 1):
        y, _ = gpu_spmv(A, x, agg_mode=agg)
        assert np.array_equal(y, y_ref)


def test_build_rejects_bad_run_max(monkeypatch):
    _ok()
    monkeypatch.setenv("CBSPMV_RUN_MAX", "256")
    with pytest.raises(cb.CBSpMVError):
        cb.build(synth.fig1(), device=0)


def test_coo_run_sums_on_for_rmat_hubs():
    """R-MAT's hub rows: long row runs per page, cut into pieces of Lmax and summed in the lanes:
    the 4096 lowest rows (the hubs) and a random sample against the oracle."""
    _ok()
    A = synth.make("rmat")
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=9)
    y, h = gpu_spmv(A, x, keep_host=0)
    rows = np.arange(4096)
    y_ref, R = oracle.spmv_rows(A, x, rows)
    check_rows(y[rows], y_ref, R, 1e-12)
    sampled(A, y, x, 1e-12, k=5000, seed=4)


# ----------------------------------------------------------------------------- launch shapes / page assignment
# Every path of the persistent kernel is chosen per handle at build time (env read by
# cb_plan_stages / cb_configure), so each one is reachable in-process: dynamic claiming on / off,
# strided static runs, the stage / group / warp shapes (G divides S), small pages.
_SHAPES = [
    {"CBSPMV_DYNAMIC_PAGES": "1"}, {"CBSPMV_DYNAMIC_PAGES": "0"},
    {"CBSPMV_DYNAMIC_PAGES": "1", "CBSPMV_CLAIM_CHUNK": "1"},
    {"CBSPMV_STRIDED_PAGES": "1"}, {"CBSPMV_STRIDED_PAGES": "4"}, {"CBSPMV_STRIDED_PAGES": "0"},
    {"CBSPMV_STAGES": "8", "CBSPMV_GROUPS": "2", "CBSPMV_GROUP_WARPS": "14", "CBSPMV_XWARPS": "2"},
    {"CBSPMV_STAGES": "12", "CBSPMV_GROUPS": "3", "CBSPMV_GROUP_WARPS": "9", "CBSPMV_XWARPS": "3"},
    {"CBSPMV_STAGES": "4", "CBSPMV_GROUPS": "1", "CBSPMV_GROUP_WARPS": "30", "CBSPMV_XWARPS": "1"},
    {"CBSPMV_STAGES": "30", "CBSPMV_GROUPS": "5", "CBSPMV_GROUP_WARPS": "5", "CBSPMV_XWARPS": "5"},
    {"CBSPMV_STAGES": "16", "CBSPMV_GROUPS": "4", "CBSPMV_GROUP_WARPS": "6", "CBSPMV_XWARPS": "4"},
    {"CBSPMV_PAGE_BYTES": "4096"}, {"CBSPMV_WAIT_SLEEP_NS": "128"}, {"CBSPMV_PDL": "0"},
    {"CBSPMV_CSR_PAIR": "1"}, {"CBSPMV_CSR_PAIR": "0"}, {"CBSPMV_XAGG": "1"}, {"CBSPMV_XAGG": "0"},
    {"CBSPMV_XAGG": "1", "CBSPMV_GROUPS": "2", "CBSPMV_GROUP_WARPS": "12", "CBSPMV_XWARPS": "1"},
]


@pytest.mark.parametrize("env", _SHAPES, ids=lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()))
@pytest.mark.parametrize("name", ["rmat", "clustered", "laplace"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_launch_shapes_and_page_assignment(monkeypatch, env, name, dtype):
    _ok()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    A = synth.make(name, small=True)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=21)
    y_ref, R = (oracle.spmv_csr(A, x) if dtype == "f64" else ref32(A, x))
    tdt = torch.float64 if dtype == "f64" else torch.float32
    h = cb.build(A, dtype=dtype, device=0)
    xd = torch.from_numpy(x).to(DEV, tdt)
    for _ in range(3):  # repeated launches reuse the dynamic-claim counters
        y = torch.full((A.m,), float("nan"), dtype=tdt, device=DEV)
        cb.spmv(h, xd, y)
        torch.cuda.synchronize()
        check_rows(y.cpu().numpy().astype(np.float64), y_ref, R, 1e-12 if dtype == "f64" else 1e-5)
    cb.destroy(h)


def test_launch_shape_rejects_too_many_warps(monkeypatch):
    _ok()
    monkeypatch.setenv("CBSPMV_GROUPS", "4")
    monkeypatch.setenv("CBSPMV_GROUP_WARPS", "8")  # 1 producer + x warps + 32 consumers > 32
    with pytest.raises(cb.CBSpMVError):
        cb.build(synth.fig1(), device=0)
