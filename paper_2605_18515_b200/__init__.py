"""B200-native CB-SpMV (arxiv 2605.18515): thin Python binding over ``libcbspmv.so``.

Argument marshalling only — every step of the path (format build, load
balance, device layout, SpMV) runs inside the C-ABI library declared in
``include/cbspmv.h``.  There is no Python or CPU fallback: if the library is
missing, importing the entry points raises.

Names mirror the C ABI without the ``cbspmv_`` prefix::

    h = build(A, dtype="f64", device=0)      # cbspmv_build (A: object with m, n, row_ptr, col, val)
    spmv(h, x, y)                            # cbspmv_spmv         y := A x
    spmv_add(h, x, y)                        # cbspmv_spmv_add     y += A x
    spmv_scaled(h, x, sumsq, y)              # cbspmv_spmv_scaled  y := A (x / sqrt(sumsq))
    spmv_host(h, x_np, y_np)                 # cbspmv_spmv_host    host buffers, end to end
    sumsq(v, out)                            # cbspmv_sumsq
    get_info(h), export(h), download_stream(h), destroy(h)
    A = mm_read(path); mm_write(path, A)     # Matrix Market files
    save(h, path); h = load(path, device=0)  # CBSM container

Device vectors are torch CUDA tensors (or raw integer device pointers); the
stream defaults to torch's current stream on the handle's device.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CBSPMV_LIB") or os.path.join(_HERE, "libcbspmv.so")  # override: A/B of builds
_lib = None

F64, F32, F32F64 = 0, 1, 2  # F32F64: fp32 matrix values, fp64 x / y / accumulation (R-24)
DTYPES = {"f64": F64, "f32": F32, "f32f64": F32F64, F64: F64, F32: F32, F32F64: F32F64}
FMT_COO, FMT_CSR, FMT_DENSE = 0, 1, 2
STATUS = {0: "OK", 1: "EINVAL", 2: "EUNSORTED", 3: "ENOMEM", 4: "ECUDA", 5: "EDIM", 6: "EUNSUPPORTED", 7: "EIO",
          8: "EFORMAT"}


class Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32)] + [(k, ctypes.c_int32) for k in (
        "blk", "th0_num", "th0_den", "ss_limit", "th1", "th2", "warps_per_tb", "agg_mode", "balance",
        "force_format", "device", "host_threads", "keep_host", "col_panels", "device_build")]


class Info(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("blk_m", ctypes.c_int64),
        ("nb", ctypes.c_int64), ("nb_pre", ctypes.c_int64), ("ss_count", ctypes.c_int64),
        ("agg", ctypes.c_int32), ("dtype", ctypes.c_int32), ("fmt_count", ctypes.c_int64 * 3),
        ("T", ctypes.c_int64), ("tb_load_mean", ctypes.c_double), ("tb_load_sd", ctypes.c_double),
        ("tb_load_max", ctypes.c_int64), ("tb_load_sd_natural", ctypes.c_double),
        ("tb_load_max_natural", ctypes.c_int64), ("mtx_bytes", ctypes.c_int64), ("n_restore", ctypes.c_int64),
        ("meta_bytes", ctypes.c_int64), ("alg_bytes", ctypes.c_int64), ("dev_stream_bytes", ctypes.c_int64),
        ("n_pages", ctypes.c_int64), ("dev_bytes", ctypes.c_int64), ("grid", ctypes.c_int32),
        ("launches_per_spmv", ctypes.c_int32), ("build_seconds", ctypes.c_double),
        ("upload_seconds", ctypes.c_double), ("n_panels", ctypes.c_int32), ("n_hot", ctypes.c_int64),
    ]


class Export(ctypes.Structure):
    P = ctypes.POINTER
    _fields_ = [
        ("nb", ctypes.c_int64), ("T", ctypes.c_int64), ("mtx_bytes", ctypes.c_int64),
        ("n_restore", ctypes.c_int64), ("n_cols_offset", ctypes.c_int64),
        ("blk_row_idx", P(ctypes.c_int32)), ("blk_col_idx", P(ctypes.c_int32)), ("nnz_per_blk", P(ctypes.c_int32)),
        ("type_per_blk", P(ctypes.c_uint8)), ("vp_per_blk", P(ctypes.c_uint64)), ("mtx_data", P(ctypes.c_uint8)),
        ("restore_cols", P(ctypes.c_uint32)), ("cols_offset", P(ctypes.c_uint64)), ("tb_ptr", P(ctypes.c_int64)),
        ("tb_load", P(ctypes.c_int64)), ("tb_load_natural", P(ctypes.c_int64)),
    ]


class CsrC(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.POINTER(ctypes.c_int64)), ("col_idx", ctypes.POINTER(ctypes.c_int32)),
                ("vals", ctypes.POINTER(ctypes.c_double))]


class HostCSR:
    """A host CSR (``m, n, nnz, row_ptr, col, val``) as returned by ``mm_read``; ``build`` accepts it."""

    def __init__(self, m, n, row_ptr, col, val):
        self.m, self.n = int(m), int(n)
        self.row_ptr, self.col, self.val = row_ptr, col, val
        self.nnz = int(row_ptr[-1]) if len(row_ptr) else 0


def lib():
    """Load libcbspmv.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make -C {os.path.dirname(_HERE)} lib` "
                               "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32
        H = ctypes.c_void_p
        sig = {
            "cbspmv_default_options": ([ctypes.POINTER(Options)], i32),
            "cbspmv_build": ([i64, i64, i64, vp, vp, vp, i32, ctypes.POINTER(Options), vp, ctypes.POINTER(H)], i32),
            "cbspmv_spmv": ([H, vp, vp, vp], i32),
            "cbspmv_spmv_add": ([H, vp, vp, vp], i32),
            "cbspmv_spmv_scaled": ([H, vp, vp, vp, vp], i32),
            "cbspmv_spmv_host": ([H, vp, vp, vp], i32),
            "cbspmv_spmv_host_batch": ([H, vp, vp, i64, vp], i32),
            "cbspmv_spmv_panel": ([H, i32, vp, vp, vp, i32, vp], i32),
            "cbspmv_panel_bounds": ([H, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
            "cbspmv_sumsq": ([vp, i64, i32, vp, i32, vp], i32),
            "cbspmv_block_stats": ([i64, i64, i64, vp, vp, vp, i32, ctypes.POINTER(Options),
                                    ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
            "cbspmv_decide_agg": ([i64, i64, ctypes.POINTER(Options), ctypes.POINTER(i32)], i32),
            "cbspmv_get_info": ([H, ctypes.POINTER(Info)], i32),
            "cbspmv_export": ([H, ctypes.POINTER(Export)], i32),
            "cbspmv_export_panel": ([H, i32, ctypes.POINTER(Export)], i32),
            "cbspmv_download_stream": ([H, vp, ctypes.c_size_t, vp, ctypes.c_size_t], i32),
            "cbspmv_hot_columns": ([H, i32, vp, ctypes.c_size_t, vp], i32),
            "cbspmv_destroy": ([H], i32),
            "cbspmv_mm_read": ([ctypes.c_char_p, ctypes.POINTER(CsrC)], i32),
            "cbspmv_mm_write": ([ctypes.c_char_p, i64, i64, vp, vp, vp], i32),
            "cbspmv_csr_free": ([ctypes.POINTER(CsrC)], i32),
            "cbspmv_save": ([H, ctypes.c_char_p], i32),
            "cbspmv_load": ([ctypes.c_char_p, ctypes.POINTER(Options), vp, ctypes.POINTER(H)], i32),
            "cbspmv_status_string": ([i32], ctypes.c_char_p),
            "cbspmv_last_error": ([], ctypes.c_char_p),
            "cbspmv_version": ([], i32),
            "cbspmv_xchg_create": ([i64, i32, i32, i32, i32, ctypes.POINTER(H)], i32),
            "cbspmv_xchg_ipc_handle": ([H, vp], i32),
            "cbspmv_xchg_base": ([H], vp),
            "cbspmv_xchg_connect": ([H, vp, vp], i32),
            "cbspmv_xchg_buffer": ([H, i32], vp),
            "cbspmv_xchg_publish": ([H, i32, i64, i64, ctypes.c_uint64, vp], i32),
            "cbspmv_xchg_wait": ([H, ctypes.c_uint64, vp, ctypes.c_double, vp], i32),
            "cbspmv_xchg_status": ([H, ctypes.POINTER(i32)], i32),
            "cbspmv_xchg_destroy": ([H], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


class CBSpMVError(RuntimeError):
    def __init__(self, status: int, what: str):
        detail = lib().cbspmv_last_error().decode()
        super().__init__(f"{what}: {STATUS.get(status, status)} ({detail})")
        self.status = status


def _check(st: int, what: str):
    if st != 0:
        raise CBSpMVError(st, what)


def default_options(**kw) -> Options:
    o = Options()
    _check(lib().cbspmv_default_options(ctypes.byref(o)), "cbspmv_default_options")
    for k, v in kw.items():
        if not hasattr(o, k) or k == "struct_size":
            raise KeyError(k)
        setattr(o, k, int(v))
    return o


_TORCH_VEC = {np.float64: "torch.float64", np.float32: "torch.float32"}


def _vec(t, length: int, np_dtype, device: int, what: str) -> int | None:
    """Device pointer of a vector argument after the §8(b) checks (SURVEY §8(b) "Indexing and
    pointers": sizes, dtype, device; the C layer re-checks device and allocation range).  A torch
    tensor must be a contiguous CUDA tensor on the handle's device, of the handle's vector dtype,
    with at least `length` elements; a raw integer pointer is passed through to the C checks."""
    if t is None or isinstance(t, int):
        return t
    if not hasattr(t, "data_ptr"):
        raise TypeError(f"{what}: expected a torch CUDA tensor or a device pointer, got {type(t).__name__}")
    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{what}: must be a CUDA tensor (got device {t.device})")
    if t.device.index != device:
        raise ValueError(f"{what}: on {t.device}, the handle is on cuda:{device}")
    if str(t.dtype) != _TORCH_VEC[np_dtype]:
        raise TypeError(f"{what}: dtype {t.dtype}, the handle needs {_TORCH_VEC[np_dtype]}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    if t.numel() < length:
        raise ValueError(f"{what}: {t.numel()} elements, needs {length}")
    return t.data_ptr()


def _xy(h, x, y, sumsq_dev=None):
    vt = vector_dtype(h.dtype)
    return (_vec(x, h.info["n"], vt, h.device, "x"), _vec(y, h.info["m"], vt, h.device, "y"),
            _vec(sumsq_dev, 1, np.float64, h.device, "sumsq"))


def _stream(stream, device: int) -> int | None:
    if stream is None and device < 0:  # host-only handle: the C layer refuses device calls
        return None
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Handle:
    """Owns one cbspmv_handle_t (a built matrix, or a row shard of one)."""

    def __init__(self, raw: ctypes.c_void_p, dtype: int, device: int):
        self._raw = raw
        self.dtype = dtype
        self.device = device
        self.info = get_info(self)

    @property
    def raw(self):
        if self._raw is None:
            raise ValueError("handle destroyed")
        return self._raw

    def __del__(self):
        try:
            destroy(self)
        except Exception:
            pass


def value_dtype(dt: int):
    """numpy type of the stored matrix values."""
    return np.float64 if dt == F64 else np.float32


def vector_dtype(dt: int):
    """numpy type of x and y."""
    return np.float32 if dt == F32 else np.float64


def build(A, dtype: str | int = "f64", device: int = 0, stream=None, **opts) -> Handle:
    """cbspmv_build on a host CSR (``A.m, A.n, A.row_ptr, A.col, A.val``)."""
    dt = DTYPES[dtype]
    o = default_options(device=device, **opts)
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    col = np.ascontiguousarray(A.col, np.int32)
    val = np.ascontiguousarray(A.val, value_dtype(dt))
    h = ctypes.c_void_p()
    st = None
    if device >= 0:
        st = _stream(stream, device)
    _check(lib().cbspmv_build(A.m, A.n, int(rp[-1]) if len(rp) else 0, rp.ctypes.data, col.ctypes.data,
                              val.ctypes.data, dt, ctypes.byref(o), st, ctypes.byref(h)), "cbspmv_build")
    return Handle(h, dt, device)


def block_stats(A, dtype: str | int = "f64", **opts) -> tuple[int, int]:
    """cbspmv_block_stats: (non-empty blocks, super-sparse blocks) before aggregation."""
    dt = DTYPES[dtype]
    o = default_options(**opts)
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    col = np.ascontiguousarray(A.col, np.int32)
    val = np.ascontiguousarray(A.val, value_dtype(dt))
    nb, ss = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().cbspmv_block_stats(A.m, A.n, int(rp[-1]) if len(rp) else 0, rp.ctypes.data, col.ctypes.data,
                                    val.ctypes.data, dt, ctypes.byref(o), ctypes.byref(nb), ctypes.byref(ss)),
           "cbspmv_block_stats")
    return nb.value, ss.value


def decide_agg(nb_pre: int, ss_count: int, **opts) -> int:
    """cbspmv_decide_agg: the th0 rule on (possibly all-reduced) block statistics."""
    o = default_options(**opts)
    a = ctypes.c_int32()
    _check(lib().cbspmv_decide_agg(int(nb_pre), int(ss_count), ctypes.byref(o), ctypes.byref(a)), "cbspmv_decide_agg")
    return a.value


def spmv(h: Handle, x, y, stream=None) -> None:
    xp, yp, _ = _xy(h, x, y)
    _check(lib().cbspmv_spmv(h.raw, xp, yp, _stream(stream, h.device)), "cbspmv_spmv")


def spmv_add(h: Handle, x, y, stream=None) -> None:
    xp, yp, _ = _xy(h, x, y)
    _check(lib().cbspmv_spmv_add(h.raw, xp, yp, _stream(stream, h.device)), "cbspmv_spmv_add")


def spmv_scaled(h: Handle, x, sumsq_dev, y, stream=None) -> None:
    xp, yp, sp = _xy(h, x, y, sumsq_dev)
    _check(lib().cbspmv_spmv_scaled(h.raw, xp, sp, yp, _stream(stream, h.device)), "cbspmv_spmv_scaled")


def spmv_panel(h: Handle, k: int, x, sumsq_dev, y, zero_y: bool, stream=None) -> None:
    """cbspmv_spmv_panel: column panel k only, y (+)= A[:, panel k] (s x); sumsq_dev None -> s = 1."""
    xp, yp, sp = _xy(h, x, y, sumsq_dev)
    _check(lib().cbspmv_spmv_panel(h.raw, int(k), xp, sp, yp, int(bool(zero_y)), _stream(stream, h.device)),
           "cbspmv_spmv_panel")


def panel_bounds(h: Handle, k: int) -> tuple[int, int]:
    c0, c1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().cbspmv_panel_bounds(h.raw, int(k), ctypes.byref(c0), ctypes.byref(c1)), "cbspmv_panel_bounds")
    return c0.value, c1.value


def spmv_host(h: Handle, x: np.ndarray, y: np.ndarray, stream=None) -> None:
    vt = vector_dtype(h.dtype)
    if x.dtype != vt or y.dtype != vt or not x.flags.c_contiguous or not y.flags.c_contiguous:
        raise ValueError("host x / y must be contiguous arrays of the handle's dtype")
    if x.size != h.info["n"] or y.size != h.info["m"]:
        raise ValueError("size mismatch")
    _check(lib().cbspmv_spmv_host(h.raw, x.ctypes.data, y.ctypes.data, _stream(stream, h.device)),
           "cbspmv_spmv_host")


def spmv_host_batch(h: Handle, xs, ys, stream=None) -> None:
    """cbspmv_spmv_host_batch: ys[k] := A xs[k] for host arrays (pinned for overlap), pipelined."""
    if len(xs) != len(ys):
        raise ValueError("xs and ys differ in length")
    vt = vector_dtype(h.dtype)
    for x, y in zip(xs, ys):
        if x.dtype != vt or y.dtype != vt or x.size != h.info["n"] or y.size != h.info["m"]:
            raise ValueError("x / y host arrays must match the handle's dtype and shape")
        if not (x.flags.c_contiguous and y.flags.c_contiguous and y.flags.writeable):
            raise ValueError("x / y must be C-contiguous (y writeable)")
    k = len(xs)
    xp = (ctypes.c_void_p * max(1, k))(*[x.ctypes.data for x in xs])
    yp = (ctypes.c_void_p * max(1, k))(*[y.ctypes.data for y in ys])
    _check(lib().cbspmv_spmv_host_batch(h.raw, xp, yp, k, _stream(stream, h.device)), "cbspmv_spmv_host_batch")


def sumsq(v, out, device: int = 0, stream=None) -> None:
    """cbspmv_sumsq: out[0] := sum(v^2); v a float64 or float32 CUDA tensor, out a float64 one."""
    if str(getattr(v, "dtype", "")) not in ("torch.float64", "torch.float32"):
        raise TypeError(f"v: dtype {getattr(v, 'dtype', type(v).__name__)}, needs torch.float64 or torch.float32")
    dt = F64 if str(v.dtype) == "torch.float64" else F32
    vp = _vec(v, 0, vector_dtype(dt), device, "v")
    op = _vec(out, 1, np.float64, device, "out")
    _check(lib().cbspmv_sumsq(vp, v.numel(), dt, op, device, _stream(stream, device)), "cbspmv_sumsq")


def get_info(h: Handle) -> dict:
    i = Info()
    _check(lib().cbspmv_get_info(h.raw, ctypes.byref(i)), "cbspmv_get_info")
    d = {k: getattr(i, k) for k, _ in Info._fields_}
    d["fmt_count"] = tuple(i.fmt_count)
    return d


def export(h: Handle, panel: int = 0) -> dict:
    """Host copies of the canonical format (slot order) of column panel `panel` as numpy arrays."""
    e = Export()
    _check(lib().cbspmv_export_panel(h.raw, panel, ctypes.byref(e)), "cbspmv_export_panel")

    def arr(p, n, dt):
        if n == 0 or not p:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(p, shape=(n,)).copy()

    nb, T = e.nb, e.T
    return dict(
        nb=nb, T=T,
        blk_row_idx=arr(e.blk_row_idx, nb, np.int32), blk_col_idx=arr(e.blk_col_idx, nb, np.int32),
        nnz_per_blk=arr(e.nnz_per_blk, nb, np.int32), type_per_blk=arr(e.type_per_blk, nb, np.uint8),
        vp_per_blk=arr(e.vp_per_blk, nb, np.uint64), mtx_data=arr(e.mtx_data, e.mtx_bytes, np.uint8),
        restore_cols=arr(e.restore_cols, e.n_restore, np.uint32),
        cols_offset=arr(e.cols_offset, e.n_cols_offset, np.uint64),
        tb_ptr=arr(e.tb_ptr, T + 1, np.int64), tb_load=arr(e.tb_load, T, np.int64),
        tb_load_natural=arr(e.tb_load_natural, T, np.int64),
    )


def download_stream(h: Handle) -> tuple[np.ndarray, np.ndarray]:
    nbytes, npages = h.info["dev_stream_bytes"], h.info["n_pages"]
    s = np.zeros(max(nbytes, 1), np.uint8)
    po = np.zeros(npages + 1, np.uint64)
    _check(lib().cbspmv_download_stream(h.raw, s.ctypes.data, s.size, po.ctypes.data, po.size),
           "cbspmv_download_stream")
    return s[:nbytes], po


def hot_columns(h: Handle, k: int = 0) -> np.ndarray:
    """The hot x columns of panel k (cbspmv_hot_columns): slot s of the shared x cache holds x[cols[s]]."""
    n = ctypes.c_int64(0)
    _check(lib().cbspmv_hot_columns(h.raw, k, None, 0, ctypes.byref(n)), "cbspmv_hot_columns")
    out = np.zeros(max(n.value, 1), np.uint32)
    if n.value:
        _check(lib().cbspmv_hot_columns(h.raw, k, out.ctypes.data, out.size, ctypes.byref(n)), "cbspmv_hot_columns")
    return out[:n.value]


def destroy(h: Handle) -> None:
    if h._raw is not None:
        lib().cbspmv_destroy(h._raw)
        h._raw = None


def mm_read(path) -> HostCSR:
    """cbspmv_mm_read: a Matrix Market coordinate file as a canonical host CSR (copied out)."""
    c = CsrC()
    _check(lib().cbspmv_mm_read(os.fsencode(path), ctypes.byref(c)), "cbspmv_mm_read")
    try:
        rp = np.ctypeslib.as_array(c.row_ptr, shape=(c.m + 1,)).copy()
        col = np.ctypeslib.as_array(c.col_idx, shape=(max(c.nnz, 1),))[:c.nnz].copy()
        val = np.ctypeslib.as_array(c.vals, shape=(max(c.nnz, 1),))[:c.nnz].copy()
        return HostCSR(c.m, c.n, rp, col, val)
    finally:
        lib().cbspmv_csr_free(ctypes.byref(c))


def mm_write(path, A) -> None:
    """cbspmv_mm_write: ``A`` (m, n, row_ptr, col, val) as a real general coordinate file."""
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    col = np.ascontiguousarray(A.col, np.int32)
    val = np.ascontiguousarray(A.val, np.float64)
    _check(lib().cbspmv_mm_write(os.fsencode(path), A.m, A.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data),
           "cbspmv_mm_write")


def save(h: Handle, path) -> None:
    """cbspmv_save: the canonical format in the CBSM container (needs keep_host=1)."""
    _check(lib().cbspmv_save(h.raw, os.fsencode(path)), "cbspmv_save")


def load(path, device: int = 0, stream=None, **opts) -> Handle:
    """cbspmv_load: a CBSM file -> handle (device page stream rebuilt and uploaded; a1..a7 skipped)."""
    o = default_options(device=device, **opts)
    h = ctypes.c_void_p()
    st = _stream(stream, device) if device >= 0 else None
    _check(lib().cbspmv_load(os.fsencode(path), ctypes.byref(o), st, ctypes.byref(h)), "cbspmv_load")
    info = Info()
    _check(lib().cbspmv_get_info(h, ctypes.byref(info)), "cbspmv_get_info")
    return Handle(h, info.dtype, device)


def version() -> int:
    return lib().cbspmv_version()


# ----------------------------------------------------------------------------- peer exchange
IPC_HANDLE_BYTES = 64


class Exchange:
    """cbspmv_xchg_*: one rank's iterate buffers + flags for the fused finalize / exchange of the
    power iteration over peer memory (include/cbspmv.h).
    ``buffer(b)`` is a torch view of iterate buffer b (n values, device ``device``)."""

    def __init__(self, n: int, dtype="f64", world: int = 1, rank: int = 0, device: int = 0):
        raw = ctypes.c_void_p()
        self.dtype, self.n, self.world, self.rank, self.device = DTYPES[dtype], int(n), int(world), int(rank), int(device)
        _check(lib().cbspmv_xchg_create(self.n, self.dtype, self.world, self.rank, self.device, ctypes.byref(raw)),
               "cbspmv_xchg_create")
        self.raw = raw
        self._bufs = {}

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(lib().cbspmv_xchg_ipc_handle(self.raw, buf), "cbspmv_xchg_ipc_handle")
        return buf.raw

    def base(self) -> int:
        return lib().cbspmv_xchg_base(self.raw)

    def connect(self, peer_bases=None, ipc_handles=None) -> None:
        """peer_bases: list of device pointers (same process; None entries are opened from
        ipc_handles); ipc_handles: list of ``world`` 64-byte handles."""
        pb = None
        if peer_bases is not None:
            pb = (ctypes.c_void_p * self.world)(*[p or None for p in peer_bases])
        hb = None
        if ipc_handles is not None:
            hb = ctypes.create_string_buffer(b"".join(h if h else bytes(IPC_HANDLE_BYTES) for h in ipc_handles))
        _check(lib().cbspmv_xchg_connect(self.raw, pb, hb), "cbspmv_xchg_connect")

    def buffer(self, b: int):
        import torch
        if b not in self._bufs:
            ptr = lib().cbspmv_xchg_buffer(self.raw, int(b))
            if not ptr:
                raise CBSpMVError(1, "cbspmv_xchg_buffer")
            tdt = torch.float32 if self.dtype == F32 else torch.float64
            self._bufs[b] = _device_view(ptr, self.n, tdt, self.device)
        return self._bufs[b]

    def publish(self, b: int, r0: int, length: int, seq: int, stream=None) -> None:
        _check(lib().cbspmv_xchg_publish(self.raw, int(b), int(r0), int(length), int(seq),
                                         _stream(stream, self.device)), "cbspmv_xchg_publish")

    def wait(self, seq: int, sumsq_dev, timeout_s: float = 10.0, stream=None) -> None:
        sp = _vec(sumsq_dev, 1, np.float64, self.device, "sumsq")
        _check(lib().cbspmv_xchg_wait(self.raw, int(seq), sp, float(timeout_s),
                                      _stream(stream, self.device)), "cbspmv_xchg_wait")

    def timed_out(self) -> bool:
        v = ctypes.c_int32()
        _check(lib().cbspmv_xchg_status(self.raw, ctypes.byref(v)), "cbspmv_xchg_status")
        return bool(v.value)

    def destroy(self) -> None:
        if self.raw:
            self._bufs.clear()
            lib().cbspmv_xchg_destroy(self.raw)
            self.raw = None


def _device_view(ptr: int, n: int, tdt, device: int):
    """A torch tensor over n values of device memory owned by the library (no copy)."""
    import torch

    class _Arr:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4" if tdt == torch.float32 else "<f8",
                                             "data": (ptr, False), "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=f"cuda:{device}")
