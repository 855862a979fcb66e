"""CB-SpMV oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2605_18515_b200``) never imports it, and the two share no code.

Thin ctypes wrapper over ``oracle.c`` (plain single-threaded C written from the
paper; see that file's header for the citations and pins).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")  # override: sanitizer builds (make asan)
_lib = None

FMT_COO, FMT_CSR, FMT_DENSE = 0, 1, 2


class Opts(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int) for k in (
        "blk", "th0_num", "th0_den", "ss_limit", "th1", "th2", "warps_per_tb",
        "agg_mode", "balance", "force_format", "val_size")]


class _CB(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("nb", ctypes.c_int64),
        ("blk_m", ctypes.c_int64), ("blk_n", ctypes.c_int64),
        ("ss_count", ctypes.c_int64), ("nb_pre", ctypes.c_int64), ("agg", ctypes.c_int),
        ("blk_row_idx", ctypes.POINTER(ctypes.c_int32)), ("blk_col_idx", ctypes.POINTER(ctypes.c_int32)),
        ("nnz_per_blk", ctypes.POINTER(ctypes.c_int32)), ("type_per_blk", ctypes.POINTER(ctypes.c_uint8)),
        ("vp_per_blk", ctypes.POINTER(ctypes.c_uint64)),
        ("mtx_data", ctypes.POINTER(ctypes.c_uint8)), ("mtx_bytes", ctypes.c_int64),
        ("cols_offset", ctypes.POINTER(ctypes.c_uint64)), ("n_cols_offset", ctypes.c_int64),
        ("restore_cols", ctypes.POINTER(ctypes.c_uint32)), ("n_restore", ctypes.c_int64),
        ("T", ctypes.c_int64), ("tb_ptr", ctypes.POINTER(ctypes.c_int64)),
        ("tb_load", ctypes.POINTER(ctypes.c_int64)), ("tb_load_natural", ctypes.POINTER(ctypes.c_int64)),
        ("fmt_count", ctypes.c_int64 * 3),
    ]


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        lib = ctypes.CDLL(_LIB_PATH)
        i64, P = ctypes.c_int64, ctypes.POINTER
        dp = P(ctypes.c_double)
        lib.oracle_spmv_csr.argtypes = [i64, P(i64), P(ctypes.c_int32), dp, dp, dp, dp]
        lib.oracle_build.argtypes = [i64, i64, P(i64), P(ctypes.c_int32), dp, P(Opts), P(_CB)]
        lib.oracle_cb_free.argtypes = [P(_CB)]
        lib.oracle_default_opts.argtypes = [P(Opts)]
        lib.oracle_spmv_cb.argtypes = [P(_CB), ctypes.c_int, ctypes.c_int, dp, dp]
        for f in ("oracle_storage_csr", "oracle_storage_bsr", "oracle_storage_cb"):
            getattr(lib, f).argtypes = [i64, i64]
            getattr(lib, f).restype = i64
        lib.oracle_select_format.argtypes = [i64, ctypes.c_int, ctypes.c_int]
        lib.oracle_encode_coord.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.oracle_padding.argtypes = [i64, i64]
        lib.oracle_padding.restype = i64
        lib.oracle_load_stats.argtypes = [P(i64), i64, dp, dp, P(i64)]
        _lib = lib
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _csr_args(A):
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    col = np.ascontiguousarray(A.col, np.int32)
    val = np.ascontiguousarray(A.val, np.float64)
    return rp, col, val


# --------------------------------------------------------------------------- Alg. 1
def spmv_csr(A, x) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 1 in fp64: returns (y, R) with R_i = sum_j |a_ij x_j|."""
    rp, col, val = _csr_args(A)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(A.m, np.float64)
    R = np.empty(A.m, np.float64)
    _load().oracle_spmv_csr(A.m, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_double),
                            _p(x, ctypes.c_double), _p(y, ctypes.c_double), _p(R, ctypes.c_double))
    return y, R


def spmv_rows(A, x, rows) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 1 restricted to sampled rows (for full-size parity on sampled outputs)."""
    rows = np.asarray(rows, np.int64)
    sub_rp = np.zeros(len(rows) + 1, np.int64)
    lens = A.row_ptr[rows + 1] - A.row_ptr[rows]
    sub_rp[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in rows]) if len(rows) else np.zeros(0, np.int64)

    class _S:
        pass
    S = _S()
    S.m, S.row_ptr, S.col, S.val = len(rows), sub_rp, A.col[idx], A.val[idx]
    return spmv_csr(S, x)


# --------------------------------------------------------------------------- build
@dataclass
class CB:
    """The oracle's CB-SpMV format (slot order after Alg. 2)."""

    m: int
    n: int
    nnz: int
    nb: int
    blk_m: int
    blk_n: int
    ss_count: int
    nb_pre: int
    agg: int
    blk_row_idx: np.ndarray
    blk_col_idx: np.ndarray
    nnz_per_blk: np.ndarray
    type_per_blk: np.ndarray
    vp_per_blk: np.ndarray
    mtx_data: np.ndarray
    cols_offset: np.ndarray
    restore_cols: np.ndarray
    T: int
    tb_ptr: np.ndarray
    tb_load: np.ndarray
    tb_load_natural: np.ndarray
    fmt_count: tuple
    opts: dict = field(default_factory=dict)
    _raw: object = None


def default_opts(**kw) -> dict:
    o = Opts()
    _load().oracle_default_opts(ctypes.byref(o))
    d = {k: getattr(o, k) for k, _ in Opts._fields_}
    for k, v in kw.items():
        if k not in d:
            raise KeyError(k)
        d[k] = int(v)
    return d


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle_build status {status}")
        self.status = status


def build(A, **kw) -> CB:
    opts = default_opts(**kw)
    o = Opts(**opts)
    rp, col, val = _csr_args(A)
    cb = _CB()
    st = _load().oracle_build(A.m, A.n, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_double),
                              ctypes.byref(o), ctypes.byref(cb))
    if st != 0:
        _load().oracle_cb_free(ctypes.byref(cb))
        raise OracleError(st)

    def arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy()

    nb, T = cb.nb, cb.T
    out = CB(
        m=cb.m, n=cb.n, nnz=cb.nnz, nb=nb, blk_m=cb.blk_m, blk_n=cb.blk_n, ss_count=cb.ss_count,
        nb_pre=cb.nb_pre, agg=cb.agg,
        blk_row_idx=arr(cb.blk_row_idx, nb, np.int32), blk_col_idx=arr(cb.blk_col_idx, nb, np.int32),
        nnz_per_blk=arr(cb.nnz_per_blk, nb, np.int32), type_per_blk=arr(cb.type_per_blk, nb, np.uint8),
        vp_per_blk=arr(cb.vp_per_blk, nb, np.uint64), mtx_data=arr(cb.mtx_data, cb.mtx_bytes, np.uint8),
        cols_offset=arr(cb.cols_offset, cb.n_cols_offset, np.uint64),
        restore_cols=arr(cb.restore_cols, cb.n_restore, np.uint32),
        T=T, tb_ptr=arr(cb.tb_ptr, T + 1, np.int64), tb_load=arr(cb.tb_load, T, np.int64),
        tb_load_natural=arr(cb.tb_load_natural, T, np.int64), fmt_count=tuple(cb.fmt_count), opts=opts,
    )
    if T == 0:
        out.tb_ptr = np.zeros(1, np.int64)
    out._raw = cb
    return out


def free(cb: CB) -> None:
    if cb._raw is not None:
        _load().oracle_cb_free(ctypes.byref(cb._raw))
        cb._raw = None


def spmv_cb(cb: CB, x) -> np.ndarray:
    """Alg. 3/4 semantics over the packed format, sequential, slot order."""
    if cb._raw is None:
        raise ValueError("CB freed")
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(cb.m, np.float64)
    _load().oracle_spmv_cb(ctypes.byref(cb._raw), cb.opts["blk"], cb.opts["val_size"],
                           _p(x, ctypes.c_double), _p(y, ctypes.c_double))
    return y


# --------------------------------------------------------------------------- small pieces
def storage_model(m, n, nnz, nnzb, blk_m) -> tuple[int, int, int]:
    """(CSR, BSR, CB) bytes."""
    L = _load()
    return (L.oracle_storage_csr(m, nnz), L.oracle_storage_bsr(nnzb, blk_m), L.oracle_storage_cb(nnzb, nnz))


def select_format(nnz, th1=32, th2=128) -> int:
    return _load().oracle_select_format(nnz, th1, th2)


def encode_coord(r, c) -> int:
    return _load().oracle_encode_coord(r, c)


def padding(idx_bytes, val_size=8) -> int:
    return _load().oracle_padding(idx_bytes, val_size)


def load_stats(loads) -> tuple[float, float, int]:
    loads = np.ascontiguousarray(loads, np.int64)
    mu, sd, mx = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    _load().oracle_load_stats(_p(loads, ctypes.c_int64), len(loads), ctypes.byref(mu), ctypes.byref(sd),
                              ctypes.byref(mx))
    return mu.value, sd.value, mx.value
