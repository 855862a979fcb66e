"""Matrix Market files and the CBSM container through the C ABI.

CPU tests pin the reader to SPEC's worked examples, to closed-form
invariants (symmetric expansion doubles the off-diagonal count; parse(write(A)) == A,
S:54) and to an independent parser (scipy.io.mmread).  The CBSM layout is decoded here with
`struct` straight from S:316, a plain version-1 container written from the oracle's build must
load, and corrupted files must be rejected.  GPU tests run loaded / read matrices against the
oracle.
"""
import os
import struct

import numpy as np
import pytest

import oracle
import paper_2605_18515_b200 as cb
import synth
from tests.test_oracle import CORPUS

EFORMAT, EIO, EINVAL, EUNSUPPORTED = 8, 7, 1, 6


def write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def entries(A):
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    return [(int(r), int(c), float(v)) for r, c, v in zip(rows, A.col, A.val)]


def status_of(fn, *a, **k):
    with pytest.raises(cb.CBSpMVError) as e:
        fn(*a, **k)
    return e.value.status


# ----------------------------------------------------------------------------- Matrix Market: SPEC examples
def test_spec_symmetric_example(tmp_path):
    """2x2 symmetric (1,1,2.0),(2,1,5.0) -> (0,0,2),(0,1,5),(1,0,5) in sorted order."""
    A = cb.mm_read(write(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 2.0\n2 1 5.0\n"))
    assert (A.m, A.n) == (2, 2)
    assert entries(A) == [(0, 0, 2.0), (0, 1, 5.0), (1, 0, 5.0)]


def test_spec_pattern_example(tmp_path):
    """pattern entry (3,4) -> (2,3,1.0)."""
    A = cb.mm_read(write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n3 4 1\n3 4\n"))
    assert entries(A) == [(2, 3, 1.0)]


def test_spec_duplicate_example(tmp_path):
    """duplicates (1,1,1.0),(1,1,2.0) -> (0,0,3.0)."""
    A = cb.mm_read(write(tmp_path, "%%MatrixMarket matrix coordinate real general\n1 1 2\n1 1 1.0\n1 1 2.0\n"))
    assert entries(A) == [(0, 0, 3.0)]


def test_spec_write_examples(tmp_path):
    """empty 4x4 -> header '4 4 0' and no entries; [(0,0,-2.5)] -> line '1 1 -2.5'."""
    p = str(tmp_path / "e.mtx")
    cb.mm_write(p, synth.CSR(4, 4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0)))
    lines = open(p).read().splitlines()
    assert lines[0].lower().startswith("%%matrixmarket matrix coordinate real general")
    assert lines[1:] == ["4 4 0"]
    cb.mm_write(p, synth.CSR(1, 1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([-2.5])))
    assert open(p).read().splitlines()[2] == "1 1 -2.5"


def test_skew_symmetric_and_hermitian(tmp_path):
    t = "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 4\n3 2 -1.5\n"
    A = cb.mm_read(write(tmp_path, t))
    assert entries(A) == [(0, 1, -4.0), (1, 0, 4.0), (1, 2, 1.5), (2, 1, -1.5)]
    t = "%%MatrixMarket matrix coordinate real hermitian\n2 2 2\n1 1 3\n2 1 7\n"
    assert entries(cb.mm_read(write(tmp_path, t))) == [(0, 0, 3.0), (0, 1, 7.0), (1, 0, 7.0)]


def test_zero_sums_and_explicit_zeros_dropped(tmp_path):
    t = "%%MatrixMarket matrix coordinate real general\n2 3 4\n1 1 1.5\n1 1 -1.5\n2 3 0\n2 2 -0.0\n"
    A = cb.mm_read(write(tmp_path, t))
    assert A.nnz == 0 and list(A.row_ptr) == [0, 0, 0]


def test_integer_field_comments_blank_lines_crlf_plus(tmp_path):
    t = ("%%MatrixMarket Matrix Coordinate Integer General\r\n% comment\r\n\r\n3 3 3\r\n"
         "3 1 +7\r\n% inner comment\r\n1 2 -2\r\n\r\n2 2 1e1\r\n")
    A = cb.mm_read(write(tmp_path, t))
    assert entries(A) == [(0, 1, -2.0), (1, 1, 10.0), (2, 0, 7.0)]


# ----------------------------------------------------------------------------- Matrix Market: invariants
@pytest.mark.parametrize("A", CORPUS[::2], ids=lambda A: A.name)
def test_roundtrip_bitwise(tmp_path, A):
    """parse(write(A)) == A for a canonical A, values bit for bit."""
    p = str(tmp_path / "r.mtx")
    cb.mm_write(p, A)
    B = cb.mm_read(p)
    assert (B.m, B.n) == (A.m, A.n)
    assert np.array_equal(B.row_ptr, A.row_ptr) and np.array_equal(B.col, A.col)
    assert np.array_equal(B.val.view(np.uint64), np.asarray(A.val, np.float64).view(np.uint64))


def test_roundtrip_awkward_values(tmp_path):
    vals = np.array([0.1, 1e-300, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 1 / 3, -123456789.125])
    A = synth.CSR(1, 7, np.array([0, 7], np.int64), np.arange(7, dtype=np.int32), vals)
    p = str(tmp_path / "v.mtx")
    cb.mm_write(p, A)
    assert np.array_equal(cb.mm_read(p).val.view(np.uint64), vals.view(np.uint64))


def test_symmetric_expansion_doubles_off_diagonal(tmp_path):
    rng = np.random.default_rng(3)
    n, k = 200, 900
    r = rng.integers(0, n, k)
    c = rng.integers(0, n, k)
    lo = np.unique(np.stack([np.maximum(r, c), np.minimum(r, c)], 1), axis=0)  # lower triangle, distinct
    v = rng.integers(1, 9, len(lo)).astype(float)
    body = "".join(f"{i + 1} {j + 1} {x:g}\n" for (i, j), x in zip(lo, v))
    A = cb.mm_read(write(tmp_path, f"%%MatrixMarket matrix coordinate real symmetric\n{n} {n} {len(lo)}\n" + body))
    diag = int(np.sum(lo[:, 0] == lo[:, 1]))
    assert A.nnz == diag + 2 * (len(lo) - diag)


def test_canonicalisation_idempotent(tmp_path):
    rng = np.random.default_rng(4)
    k = 500
    body = "".join(f"{rng.integers(1, 41)} {rng.integers(1, 31)} {rng.integers(-3, 4)}\n" for _ in range(k))
    p = write(tmp_path, f"%%MatrixMarket matrix coordinate integer general\n40 30 {k}\n" + body)
    A = cb.mm_read(p)
    q = str(tmp_path / "again.mtx")
    cb.mm_write(q, A)
    B = cb.mm_read(q)
    assert entries(A) == entries(B)


@pytest.mark.parametrize("field", ["real", "integer", "pattern"])
@pytest.mark.parametrize("sym", ["general", "symmetric", "skew-symmetric"])
def test_matches_scipy_mmread(tmp_path, field, sym):
    """An independent Matrix Market parser (scipy.io.mmread) gives the same matrix."""
    sio = pytest.importorskip("scipy.io")
    if field == "pattern" and sym == "skew-symmetric":
        pytest.skip("not a valid Matrix Market combination")
    rng = np.random.default_rng(hash((field, sym)) % 2**32)
    n, k = 60, 400
    r, c = rng.integers(0, n, k), rng.integers(0, n, k)
    if sym != "general":
        r, c = np.maximum(r, c), np.minimum(r, c)
        if sym == "skew-symmetric":
            keep = r != c
            r, c = r[keep], c[keep]
    v = rng.integers(-5, 6, len(r)).astype(float) * (0.25 if field == "real" else 1.0)
    lines = [f"{i + 1} {j + 1}" + ("" if field == "pattern" else f" {x:g}") for i, j, x in zip(r, c, v)]
    p = write(tmp_path, f"%%MatrixMarket matrix coordinate {field} {sym}\n{n} {n} {len(lines)}\n" + "\n".join(lines) + "\n")
    A = cb.mm_read(p)
    S = sio.mmread(p).tocsr()
    S.sum_duplicates()
    S.eliminate_zeros()
    D = np.zeros((n, n))
    for i, j, x in entries(A):
        D[i, j] = x
    assert np.array_equal(D, S.toarray())
    assert A.nnz == S.nnz


def test_reader_errors(tmp_path):
    hdr = "%%MatrixMarket matrix coordinate real general\n"
    assert status_of(cb.mm_read, str(tmp_path / "missing.mtx")) == EIO
    assert status_of(cb.mm_read, write(tmp_path, "%%MatrixMarket matrix coordinat real general\n1 1 0\n")) == EUNSUPPORTED
    assert status_of(cb.mm_read, write(tmp_path, "%MatrixMarket matrix coordinate real general\n1 1 0\n")) == EFORMAT
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 2\n1 1 1\n")) == EFORMAT          # count mismatch
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n3 1 1\n")) == EFORMAT          # out of bounds
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n0 1 1\n")) == EFORMAT          # 0 is not 1-based
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n1 1 inf\n")) == EINVAL         # non-finite
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n1 1 nan\n")) == EINVAL
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n1 1 x\n")) == EFORMAT
    assert status_of(cb.mm_read, write(tmp_path, hdr + "2 2 1\n1 1 1 9\n")) == EFORMAT        # trailing token
    cplx = "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n"
    assert status_of(cb.mm_read, write(tmp_path, cplx)) == EUNSUPPORTED
    arr = "%%MatrixMarket matrix array real general\n1 1\n1\n"
    assert status_of(cb.mm_read, write(tmp_path, arr)) == EUNSUPPORTED
    sym = "%%MatrixMarket matrix coordinate real symmetric\n2 3 0\n"
    assert status_of(cb.mm_read, write(tmp_path, sym)) == EFORMAT


def test_large_file_parallel_chunks(tmp_path):
    """Enough lines for many parallel parse chunks; entries in random order with duplicates."""
    A = synth.random_csr(3000, 2500, 0.02, 11, pattern="random")
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    order = np.random.default_rng(0).permutation(A.nnz)
    half = order[: A.nnz // 2]  # duplicated entries split a value in two halves that sum exactly
    r = np.concatenate([rows[order], rows[half]])
    c = np.concatenate([A.col[order], A.col[half]])
    v = np.concatenate([A.val[order], np.zeros(len(half))])
    body = "\n".join(f"{i + 1} {j + 1} {float(x)!r}" for i, j, x in zip(r, c, v))
    B = cb.mm_read(write(tmp_path, f"%%MatrixMarket matrix coordinate real general\n{A.m} {A.n} {len(r)}\n{body}\n"))
    assert np.array_equal(B.row_ptr, A.row_ptr) and np.array_equal(B.col, A.col)
    assert np.array_equal(B.val, A.val)


# ----------------------------------------------------------------------------- CBSM container
KEYS = ["blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
        "restore_cols", "cols_offset", "tb_ptr", "tb_load", "tb_load_natural"]
INFO_KEYS = ["m", "n", "nnz", "blk_m", "nb", "nb_pre", "ss_count", "agg", "dtype", "fmt_count", "T",
             "tb_load_mean", "tb_load_sd", "tb_load_max", "tb_load_sd_natural", "tb_load_max_natural",
             "mtx_bytes", "n_restore", "meta_bytes", "alg_bytes", "n_panels"]


def same_format(h1, h2):
    for k in INFO_KEYS:
        assert h1.info[k] == h2.info[k], k
    for p in range(h1.info["n_panels"]):
        e1, e2 = cb.export(h1, p), cb.export(h2, p)
        for k in KEYS:
            assert e1[k].dtype == e2[k].dtype and np.array_equal(e1[k], e2[k]), (p, k)


@pytest.mark.parametrize("A", CORPUS[::3], ids=lambda A: A.name)
@pytest.mark.parametrize("opts", [dict(), dict(agg_mode=1), dict(agg_mode=0, balance=0), dict(dtype="f32"),
                                  dict(dtype="f32f64", agg_mode=1), dict(col_panels=3)],
                         ids=["default", "agg", "noagg-nobal", "f32", "mixed", "panels3"])
def test_save_load_roundtrip(tmp_path, A, opts):
    h = cb.build(A, device=-1, **opts)
    p = str(tmp_path / "a.cbsm")
    cb.save(h, p)
    h2 = cb.load(p, device=-1)
    same_format(h, h2)


def parse_cbsm(buf, blk_m_of):
    """S:316 read literally: header, five arrays, optional agg arrays, mtx_data; then the rest."""
    o = 0
    magic, ver, m, n, nb, mlen, has_agg, has_sched = struct.unpack_from("<4sIQQQQBB", buf, o)
    o += struct.calcsize("<4sIQQQQBB")
    out = dict(magic=magic, version=ver, m=m, n=n, nb=nb, has_agg=has_agg, has_sched=has_sched)
    for k, dt in (("blk_row_idx", "<u4"), ("blk_col_idx", "<u4"), ("nnz_per_blk", "<u4"), ("type_per_blk", "u1"),
                  ("vp_per_blk", "<u8")):
        a = np.frombuffer(buf, dt, nb, o)
        out[k] = a
        o += a.nbytes
    if has_agg:
        co = np.frombuffer(buf, "<u8", blk_m_of(m) + 1, o)
        o += co.nbytes
        rc = np.frombuffer(buf, "<u4", int(co[-1]), o)
        o += rc.nbytes
        out["cols_offset"], out["restore_cols"] = co, rc
    out["mtx_data"] = np.frombuffer(buf, "u1", mlen, o)
    o += mlen
    out["rest"] = buf[o:]
    return out


@pytest.mark.parametrize("agg", [0, 1])
def test_cbsm_layout_is_spec_s316(tmp_path, agg):
    A = synth.make("laplace", small=True)
    h = cb.build(A, device=-1, agg_mode=agg)
    p = str(tmp_path / "l.cbsm")
    cb.save(h, p)
    d = parse_cbsm(open(p, "rb").read(), lambda m: (m + 15) // 16)
    ex = cb.export(h)
    assert d["magic"] == b"CBSM" and d["version"] == 1 and d["has_agg"] == agg and d["has_sched"] == 1
    assert (d["m"], d["n"], d["nb"]) == (A.m, A.n, ex["nb"])
    for k in ("blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data"):
        assert np.array_equal(d[k].astype(np.int64), ex[k].astype(np.int64)), k
    if agg:
        assert np.array_equal(d["cols_offset"], ex["cols_offset"]) and np.array_equal(d["restore_cols"], ex["restore_cols"])
    assert d["rest"][:4] == b"CBX1"


def spec_container(ref, m, n):
    """A plain version-1 container (no extension block) from the oracle's build."""
    parts = [struct.pack("<4sIQQQQBB", b"CBSM", 1, m, n, ref.nb, len(ref.mtx_data), int(ref.agg), 1)]
    for k, dt in (("blk_row_idx", "<u4"), ("blk_col_idx", "<u4"), ("nnz_per_blk", "<u4"), ("type_per_blk", "u1"),
                  ("vp_per_blk", "<u8")):
        parts.append(np.asarray(getattr(ref, k)).astype(dt).tobytes())
    if ref.agg:
        parts.append(np.asarray(ref.cols_offset).astype("<u8").tobytes())
        parts.append(np.asarray(ref.restore_cols).astype("<u4").tobytes())
    parts.append(np.asarray(ref.mtx_data, np.uint8).tobytes())
    return b"".join(parts)


@pytest.mark.parametrize("name", ["laplace", "rmat", "clustered"])
def test_load_plain_spec_container_from_oracle(tmp_path, name):
    A = synth.make(name, small=True)
    ref = oracle.build(A)
    p = write(tmp_path, spec_container(ref, A.m, A.n), "o.cbsm")
    h = cb.load(p, device=-1)
    ex = cb.export(h)
    for k in ("blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
              "restore_cols", "cols_offset"):
        assert np.array_equal(ex[k], getattr(ref, k)), k
    assert h.info["nnz"] == A.nnz and h.info["dtype"] == cb.F64
    T = (ref.nb + 7) // 8
    assert np.array_equal(ex["tb_ptr"], np.minimum(np.arange(T + 1) * 8, ref.nb))  # consecutive groups of 8
    oracle.free(ref)


def corrupt_cases(A, ref):
    """(description, bytes) pairs, each breaking one thing the loader must check."""
    good = spec_container(ref, A.m, A.n)
    hdr = struct.calcsize("<4sIQQQQBB")
    nb = ref.nb
    off_type = hdr + 12 * nb
    off_vp = off_type + nb
    off_mtx = off_vp + 8 * nb + (8 * (len(ref.cols_offset)) + 4 * len(ref.restore_cols) if ref.agg else 0)
    cases = [("magic", b"XBSM" + good[4:]), ("version", good[:4] + struct.pack("<I", 2) + good[8:]),
             ("truncated", good[:-5]), ("empty", b"")]
    b = bytearray(good); b[off_type] = 3; cases.append(("type", bytes(b)))
    b = bytearray(good); b[off_vp:off_vp + 8] = struct.pack("<Q", len(ref.mtx_data)); cases.append(("vp", bytes(b)))
    b = bytearray(good); b[hdr + 8 * nb:hdr + 8 * nb + 4] = struct.pack("<I", 0); cases.append(("nnz0", bytes(b)))
    b = bytearray(good); b[hdr:hdr + 4] = struct.pack("<I", (A.m + 15) // 16); cases.append(("br", bytes(b)))
    # a COO coordinate byte pointing outside the matrix (row 15 of the ragged last block row)
    types = np.asarray(ref.type_per_blk)
    last = [i for i in range(nb) if types[i] == 0 and ref.blk_row_idx[i] == (A.m - 1) // 16]
    if last and A.m % 16:
        i = last[0]
        b = bytearray(good); b[off_mtx + int(ref.vp_per_blk[i])] = 0x0F; cases.append(("coo-row", bytes(b)))
    return cases


def test_load_rejects_corrupt_files(tmp_path):
    A = synth.random_csr(37, 53, 0.2, 5, pattern="random")  # ragged last block row and column
    ref = oracle.build(A, agg_mode=0)
    for what, data in corrupt_cases(A, ref):
        p = write(tmp_path, data, f"c_{what}.cbsm")
        assert status_of(cb.load, p, device=-1) == EFORMAT, what
    oracle.free(ref)
    Aa = synth.random_csr(40, 300, 0.01, 6, pattern="random")
    ref = oracle.build(Aa, agg_mode=1)
    good = bytearray(spec_container(ref, Aa.m, Aa.n))
    hdr = struct.calcsize("<4sIQQQQBB")
    off_rc = hdr + 21 * ref.nb + 8 * len(ref.cols_offset)
    good[off_rc:off_rc + 4] = struct.pack("<I", Aa.n)  # restore_cols entry == n
    assert status_of(cb.load, write(tmp_path, bytes(good), "rc.cbsm"), device=-1) == EFORMAT
    oracle.free(ref)
    assert status_of(cb.load, str(tmp_path / "none.cbsm"), device=-1) == EIO


def test_save_requires_host_arrays(tmp_path):
    h = cb.build(synth.fig1(), device=-1, keep_host=0)
    assert status_of(cb.save, h, str(tmp_path / "x.cbsm")) == EUNSUPPORTED


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["rmat", "clustered", "uniform"])
@pytest.mark.parametrize("dtype", ["f64", "f32f64"])
def test_gpu_loaded_handle_matches_oracle(tmp_path, name, dtype):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    A = synth.make(name, small=True)
    h = cb.build(A, dtype=dtype, device=-1, col_panels=2 if name == "uniform" else 0)
    p = str(tmp_path / "g.cbsm")
    cb.save(h, p)
    hg = cb.load(p, device=0)
    assert hg.info["n_pages"] > 0 and hg.info["n_panels"] == h.info["n_panels"]
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=3)
    Ar = A if dtype == "f64" else synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    y_ref, R = oracle.spmv_csr(Ar, x)
    y = np.empty(A.m)
    cb.spmv_host(hg, x, y)
    assert np.all(np.abs(y - y_ref) <= 1e-12 * R)


@pytest.mark.gpu
def test_gpu_matrix_market_to_spmv(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    A = synth.make("laplace", small=True)
    p = str(tmp_path / "lap.mtx")
    cb.mm_write(p, A)
    B = cb.mm_read(p)
    h = cb.build(B, device=0)
    x = synth.vector(A.n, synth.VEC_INT7)
    y = np.empty(A.m)
    cb.spmv_host(h, x, y)
    y_ref, _ = oracle.spmv_csr(A, x)
    assert np.array_equal(y, y_ref)  # exact-integer data: bitwise
