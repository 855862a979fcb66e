"""Seeded synthetic inputs for CB-SpMV (shared by oracle tests and the product path).

Holds none of the method's arithmetic: only canonical CSR matrices (sorted
unique columns, no explicit zeros) and dense vectors.  The heavy generators are
counter-based C (``synth.c``) so a row range generates identically under any
sharding (SURVEY.md §8(d) "Synthetic inputs"); the small random corpus used by
the parity tests is numpy with a seeded ``Generator``.

Workloads (BASELINE.json ``configs``; recipe in DESIGN.md §3):
  * ``fig1()``        – the constructed 16x16 Fig. 1 fixture.
  * ``laplace5(g)``   – 5-point Laplacian on a g x g grid (config 2: g=1000).
  * ``rmat(scale)``   – Graph500-style R-MAT (config 3: scale 23, ef 16).
  * ``clustered(m)``  – block-clustered dense/CSR/COO mix (config 4: m=2^22).
  * ``uniform(m)``    – k=50 uniform distinct columns per row (config 5: m=2^25).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("SYNTH_LIB") or os.path.join(_HERE, "libsynth.so")  # override: sanitizer builds (make asan)
_lib = None


class _CSR(ctypes.Structure):
    _fields_ = [
        ("m_local", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
        ("col", ctypes.POINTER(ctypes.c_int32)),
        ("val", ctypes.POINTER(ctypes.c_double)),
    ]


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} synth`")
        lib = ctypes.CDLL(_LIB_PATH)
        i64, u64, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        P = ctypes.POINTER(_CSR)
        lib.synth_laplace5.argtypes = [i64, i64, i64, P]
        lib.synth_rmat.argtypes = [c_int, i64, u64, c_int, i64, i64, P]
        lib.synth_clustered.argtypes = [i64, i64, u64, c_int, i64, i64, P]
        lib.synth_uniform.argtypes = [i64, i64, i64, u64, c_int, i64, i64, P]
        lib.synth_vector.argtypes = [i64, i64, c_int, u64, ctypes.POINTER(ctypes.c_double)]
        lib.synth_free.argtypes = [P]
        lib.synth_set_threads.argtypes = [c_int]
        PI = ctypes.POINTER(ctypes.c_int64)
        lib.synth_rmat_row_counts.argtypes = [c_int, i64, u64, PI]
        lib.synth_clustered_row_counts.argtypes = [i64, i64, u64, PI]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Row block [r0, r0+m) of an (m_total x n) matrix in canonical CSR."""

    m: int
    n: int
    row_ptr: np.ndarray  # int64[m+1]
    col: np.ndarray  # int32[nnz]
    val: np.ndarray  # float64[nnz]
    r0: int = 0
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.m, self.n), dtype=np.float64)
        rows = np.repeat(np.arange(self.m), np.diff(self.row_ptr))
        d[rows, self.col] = self.val
        return d


def _take(st: _CSR, r0: int, name: str) -> CSR:
    m, nnz = st.m_local, st.nnz
    rp = np.ctypeslib.as_array(st.row_ptr, shape=(m + 1,)).copy()
    col = np.ctypeslib.as_array(st.col, shape=(max(nnz, 1),))[:nnz].copy()
    val = np.ctypeslib.as_array(st.val, shape=(max(nnz, 1),))[:nnz].copy()
    _load().synth_free(ctypes.byref(st))
    return CSR(m=m, n=int(st.n), row_ptr=rp, col=col, val=val, r0=r0, name=name)


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"synth {what} failed rc={rc}")


def set_threads(t: int) -> None:
    _load().synth_set_threads(int(t))


def laplace5(g: int, r0: int = 0, r1: int | None = None) -> CSR:
    r1 = g * g if r1 is None else r1
    st = _CSR()
    _check(_load().synth_laplace5(g, r0, r1, ctypes.byref(st)), "laplace5")
    return _take(st, r0, f"laplace5_g{g}")


def rmat(scale: int, edge_factor: int = 16, seed: int = 31, val_mode: int = 0,
         r0: int = 0, r1: int | None = None) -> CSR:
    r1 = (1 << scale) if r1 is None else r1
    st = _CSR()
    _check(_load().synth_rmat(scale, edge_factor, seed, val_mode, r0, r1, ctypes.byref(st)), "rmat")
    return _take(st, r0, f"rmat_s{scale}_ef{edge_factor}")


def clustered(m: int, n: int | None = None, seed: int = 41, val_mode: int = 0,
              r0: int = 0, r1: int | None = None) -> CSR:
    n = m if n is None else n
    r1 = m if r1 is None else r1
    st = _CSR()
    _check(_load().synth_clustered(m, n, seed, val_mode, r0, r1, ctypes.byref(st)), "clustered")
    return _take(st, r0, f"clustered_m{m}")


def uniform(m: int, n: int | None = None, k: int = 50, seed: int = 51, val_mode: int = 1,
            r0: int = 0, r1: int | None = None) -> CSR:
    n = m if n is None else n
    r1 = m if r1 is None else r1
    st = _CSR()
    _check(_load().synth_uniform(m, n, k, seed, val_mode, r0, r1, ctypes.byref(st)), "uniform")
    return _take(st, r0, f"uniform_m{m}_k{k}")


def row_counts(name: str, small: bool = False) -> np.ndarray:
    """Stored entries per row of ``make(name, small=small)`` without generating the matrix (the
    counts a row-shard cut needs before each rank generates only its rows).  Exact for laplace,
    clustered and uniform; for rmat the edge count per row before duplicate removal (an upper
    bound: the cut it gives is balanced to within the duplicate rate)."""
    L = _load()
    if name == "laplace":
        g = 100 if small else 1000
        i, j = np.divmod(np.arange(g * g, dtype=np.int64), g)
        return 1 + (i > 0) + (i < g - 1) + (j > 0) + (j < g - 1)
    if name == "uniform":
        m = (1 << 15) if small else (1 << 25)
        return np.full(m, 50, np.int64)
    if name == "clustered":
        m = (1 << 14) if small else (1 << 22)
        out = np.empty(m, np.int64)
        _check(L.synth_clustered_row_counts(m, m, 41, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
               "clustered_row_counts")
        return out
    if name == "rmat":
        scale = 14 if small else 23
        out = np.empty(1 << scale, np.int64)
        _check(L.synth_rmat_row_counts(scale, 16, 31, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
               "rmat_row_counts")
        return out
    raise ValueError(name)


VEC_UNIFORM, VEC_ONES, VEC_INT7, VEC_FIG1 = 0, 1, 2, 3


def vector(n: int, mode: int = VEC_UNIFORM, seed: int = 11, j0: int = 0) -> np.ndarray:
    x = np.empty(n, dtype=np.float64)
    if n:
        _load().synth_vector(j0, n, mode, seed, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return x


# --------------------------------------------------------------------------- Fig. 1 fixture
# Constructed 16x16 matrix meeting every stated Fig. 1 constraint:
# 13 non-empty 4x4 sub-blocks, third row-major non-zero at (0,4).  SURVEY §8(c).
FIG1_PATTERN = (
    "X.X.X...........",
    ".X...X..........",
    "..X..........X..",
    "...X...X........",
    "X...XXXX.......X",
    "....XXXX.XX.....",
    ".X..XXXX........",
    "....XXXXX.......",
    "........XX......",
    "......X..XX.....",
    "..........XX..X.",
    "........X..XX...",
    "X...........X..X",
    "...X.........X..",
    "..........X...X.",
    ".X..........X..X",
)


def fig1() -> CSR:
    """a_rc = ((16 r + c) mod 9) + 1 on FIG1_PATTERN (SURVEY §8(c) worked example)."""
    rp, cols, vals = [0], [], []
    for r, line in enumerate(FIG1_PATTERN):
        for c, ch in enumerate(line):
            if ch == "X":
                cols.append(c)
                vals.append(float(((16 * r + c) % 9) + 1))
        rp.append(len(cols))
    return CSR(16, 16, np.array(rp, np.int64), np.array(cols, np.int32), np.array(vals, np.float64),
               name="fig1")


# --------------------------------------------------------------------------- random corpus
def from_dense(d: np.ndarray, name: str = "dense") -> CSR:
    d = np.asarray(d, dtype=np.float64)
    m, n = d.shape
    rows, cols = np.nonzero(d)
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return CSR(m, n, np.cumsum(rp), cols.astype(np.int32), d[rows, cols].copy(), name=name)


def from_coo(m: int, n: int, rows, cols, vals, name: str = "coo") -> CSR:
    """Canonicalise (sort, sum duplicates, drop zeros) — input plumbing only."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, np.float64)
    key = rows * max(n, 1) + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uk, first = np.unique(key, return_index=True)
    v = np.add.reduceat(vals, first) if len(vals) else vals
    keep = v != 0
    uk, v = uk[keep], v[keep]
    r = uk // max(n, 1)
    c = uk % max(n, 1)
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return CSR(m, n, np.cumsum(rp), c.astype(np.int32), v, name=name)


def random_csr(m: int, n: int, density: float, seed: int, val_mode: int = 0, pattern: str = "random") -> CSR:
    """Small seeded matrices for the parity corpus (SPEC S:611 shapes).

    pattern: random | banded | blockdense | diag | row | col | empty | hub
    val_mode: 0 U(-1,1)\\{0}; 1 U(0,1]; 2 integers {-4..4}\\{0}; 3 ones.
    """
    rng = np.random.default_rng(seed)
    if pattern == "random":
        cnt = rng.binomial(m * n, min(density, 1.0)) if m * n else 0
        flat = rng.choice(m * n, size=cnt, replace=False) if cnt else np.zeros(0, np.int64)
        rows, cols = flat // n, flat % n
    elif pattern == "banded":
        bw = max(1, int(density * n))
        rows = np.repeat(np.arange(m), 2 * bw + 1)
        cols = rows + np.tile(np.arange(-bw, bw + 1), m)
        ok = (cols >= 0) & (cols < n)
        rows, cols = rows[ok], cols[ok]
    elif pattern == "blockdense":
        rows, cols = [], []
        nbr, nbc = (m + 15) // 16, (n + 15) // 16
        for br in range(nbr):
            for bc in range(nbc):
                if rng.random() < density:
                    k = int(rng.integers(1, 257))
                    pos = rng.choice(256, size=k, replace=False)
                    rows.append(br * 16 + pos // 16)
                    cols.append(bc * 16 + pos % 16)
        rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
        ok = (rows < m) & (cols < n)
        rows, cols = rows[ok], cols[ok]
    elif pattern == "diag":
        k = min(m, n)
        rows = cols = np.arange(k)
    elif pattern == "row":  # one dense-ish row
        cols = np.nonzero(rng.random(n) < max(density, 0.5))[0]
        rows = np.full(len(cols), rng.integers(0, m) if m else 0)
    elif pattern == "col":
        rows = np.nonzero(rng.random(m) < max(density, 0.5))[0]
        cols = np.full(len(rows), rng.integers(0, n) if n else 0)
    elif pattern == "hub":  # a few very long rows + random background
        cnt = rng.binomial(m * n, min(density, 1.0)) if m * n else 0
        flat = rng.choice(m * n, size=cnt, replace=False) if cnt else np.zeros(0, np.int64)
        hubs = rng.choice(m, size=min(3, m), replace=False)
        hr = np.repeat(hubs, n)
        hc = np.tile(np.arange(n), len(hubs))
        keep = rng.random(len(hr)) < 0.7
        rows = np.concatenate([flat // n, hr[keep]])
        cols = np.concatenate([flat % n, hc[keep]])
    elif pattern == "empty":
        rows = cols = np.zeros(0, np.int64)
    else:
        raise ValueError(pattern)
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    if len(rows):
        key = np.unique(rows * n + cols)
        rows, cols = key // n, key % n
    nz = len(rows)
    if val_mode == 0:
        vals = rng.uniform(-1.0, 1.0, nz)
        vals[vals == 0] = 0.5
    elif val_mode == 1:
        vals = 1.0 - rng.random(nz)
    elif val_mode == 2:
        vals = rng.choice(np.array([-4, -3, -2, -1, 1, 2, 3, 4], np.float64), nz)
    else:
        vals = np.ones(nz)
    return from_coo(m, n, rows, cols, vals, name=f"{pattern}_{m}x{n}_s{seed}")


# --------------------------------------------------------------------------- BASELINE configs
CONFIGS = {
    # name: (builder, kwargs, description) — BASELINE.json "configs" in order
    "fig1": "Paper Fig. 1 example: 16x16, 4x4 sub-blocks, 13 non-zero sub-blocks, fp64",
    "laplace": "Synthetic 2D 5-point Laplacian, 1M rows, ~5M nnz, fp64",
    "rmat": "Synthetic R-MAT, scale 23, ef 16, 8M rows, ~128M nnz, fp64",
    "clustered": "Synthetic block-clustered, 4M rows, ~400M nnz, dense/CSR/COO mix",
    "uniform": "Uniform random, 32M rows, 50/row, ~1.6B nnz (power iteration)",
}


def make(name: str, r0: int = 0, r1: int | None = None, small: bool = False) -> CSR:
    """The BASELINE.json workloads by name (``small`` shrinks for tests)."""
    if name == "fig1":
        return fig1()
    if name == "laplace":
        return laplace5(100 if small else 1000, r0, r1)
    if name == "rmat":
        return rmat(14 if small else 23, 16, 31, 0, r0, r1)
    if name == "clustered":
        m = (1 << 14) if small else (1 << 22)
        return clustered(m, m, 41, 0, r0, r1)
    if name == "uniform":
        m = (1 << 15) if small else (1 << 25)
        return uniform(m, m, 50, 51, 1, r0, r1)
    raise ValueError(name)
