"""Full-size parity at BASELINE.json configs[3] and configs[4], in the
launch configuration bench.py times (automatic column panels, dynamic page claiming, the fused
power-iteration exchange).

* configs[4], uniform 2^25 x 2^25, 50 per row (1.68 B nnz, 6 column panels):
  - one SpMV on 20,000 sampled rows plus the first and the last block row against the oracle
    (|y - y_ref| <= 1e-12 * R_i);
  - the power iteration (FusedPowerIteration, 100 steps): steps k = 0, 1, 50, 99 each recomputed
    by the oracle on sampled rows from the downloaded iterate x_k;
  - the all-ones variant: every row sums to 50 exactly, so A x = 50 x for x = 1 and the power
    iteration sits at lambda = 50.  At n = 2^24 every quantity is dyadic (||1|| = 2^12), so
    lambda = 50 bitwise at all 100 steps.
* format byte identity against the oracle's build at full size: the
  clustered matrix (configs[3]) and the R-MAT graph (configs[2]) whole, and configs[4] as the
  8-GPU run builds it — one row shard of 2^22 rows with the global th0 decision (aggregation on).
  (configs[1], the Laplacian, is checked at full size by the CPU suite.)
"""
import numpy as np
import pytest

import oracle
import paper_2605_18515_b200 as cb
import synth
from paper_2605_18515_b200 import dist as cbd

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"
N_UNI = 1 << 25


def _ok():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check_rows(y, y_ref, R, rel):
    bad = np.abs(y - y_ref) > rel * R
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(f"{int(bad.sum())} rows out of tolerance; row {i}: y={y[i]!r} ref={y_ref[i]!r}")


def _sample(m, k=20000, seed=0):
    rows = np.random.default_rng(seed).choice(m, size=k, replace=False)
    return np.unique(np.concatenate([rows, np.arange(16), np.arange(m - 16, m)]))


@pytest.fixture(scope="module")
def uniform_full():
    _ok()
    A = synth.make("uniform")  # configs[4]: values U(0,1], exactly 50 distinct columns per row
    assert A.m == N_UNI and A.nnz == 50 * N_UNI
    h = cb.build(A, device=0, keep_host=0)
    assert h.info["n_panels"] > 1 and h.info["agg"] == 1
    yield A, h
    cb.destroy(h)


def test_uniform_full_spmv_sampled(uniform_full):
    A, h = uniform_full
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=52)
    xd = torch.from_numpy(x).to(DEV)
    y = torch.full((A.m,), float("nan"), dtype=torch.float64, device=DEV)
    cb.spmv(h, xd, y)
    rows = _sample(A.m)
    ys = y[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    y_ref, R = oracle.spmv_rows(A, x, rows)
    _check_rows(ys, y_ref, R, 1e-12)
    assert bool(torch.isfinite(y).all())


def test_uniform_full_power_iteration_steps(uniform_full):
    """x_k downloaded at steps {0, 1, 50, 99}, one step recomputed by the oracle
    on the sampled rows; y_k = A (x_k / ||x_k||)."""
    A, h = uniform_full
    rows = _sample(A.m, seed=1)
    rows_t = torch.from_numpy(rows).to(DEV)
    checks = {0, 1, 50, 99}
    saved = {0: np.ones(A.n)}
    done = []

    def on_step(k, x, ss):  # x = x_{k+1} = y_k (unnormalised), ss = ||y_k||^2
        if k in checks:
            xk = saved.pop(k)
            s = 1.0 / np.sqrt(float(xk @ xk))
            y_ref, R = oracle.spmv_rows(A, xk * s, rows)
            _check_rows(x[rows_t].cpu().numpy(), y_ref, R, 1e-12)
            done.append(k)
        if k + 1 in checks:
            saved[k + 1] = x.cpu().numpy()

    f = cbd.FusedPowerIteration(h, A.n, "f64", 1, 0, 0)
    x, ss = f.run(torch.ones(A.n, dtype=torch.float64, device=DEV), 100, on_step=on_step)
    torch.cuda.synchronize()
    lam = float(ss.item()) ** 0.5
    f.destroy()
    assert sorted(done) == sorted(checks)
    # Perron root of a nonnegative matrix lies between the smallest and largest row sums
    rs = np.add.reduceat(A.val, A.row_ptr[:-1])
    assert rs.min() <= lam <= rs.max()


@pytest.mark.parametrize("n,bitwise", [(1 << 24, True), (N_UNI, False)])
def test_uniform_ones_power_iteration_lambda_50(n, bitwise):
    """The all-ones uniform matrix (every row sums to 50) holds the power iteration at lambda = 50:
    at n = 2^24 every quantity is dyadic, so lambda = 50 bitwise for 100 steps; at the full
    configs[4] size (2^25, ||1|| = 2^12.5) within 1e-15."""
    _ok()
    A = synth.uniform(n, n, 50, 51, val_mode=3)  # all values 1: every row sums to 50
    h = cb.build(A, device=0, keep_host=0)
    lams = []
    f = cbd.FusedPowerIteration(h, A.n, "f64", 1, 0, 0)
    f.run(torch.ones(A.n, dtype=torch.float64, device=DEV), 100,
          on_step=lambda k, x, ss: lams.append(float(ss.item()) ** 0.5))
    f.destroy()
    cb.destroy(h)
    if bitwise:
        assert lams == [50.0] * 100
    else:
        assert len(lams) == 100 and max(abs(v - 50.0) for v in lams) <= 50.0 * 1e-15


FORMAT_KEYS = ("blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
               "restore_cols", "cols_offset", "tb_ptr", "tb_load", "tb_load_natural")


def _format_equal(A, **opts):
    h = cb.build(A, device=-1, **opts)
    ex = cb.export(h)
    ref = oracle.build(A, **opts)
    try:
        for k in FORMAT_KEYS:
            assert np.array_equal(ex[k], getattr(ref, k)), k
        assert ex["nb"] == ref.nb and ex["T"] == ref.T
    finally:
        oracle.free(ref)
        cb.destroy(h)


def test_clustered_full_format_equals_oracle():
    """configs[3] at full size (4 M rows, 407.5 M nnz): the host build's canonical format is the
    oracle's byte for byte."""
    _ok()
    _format_equal(synth.make("clustered"))


def test_rmat_full_format_equals_oracle():
    """configs[2] at full size (8 M rows, 131 M nnz, aggregation on by the th0 rule): the host
    build's canonical format is the oracle's byte for byte."""
    _ok()
    _format_equal(synth.make("rmat"))


def test_uniform_rank_shard_format_equals_oracle():
    """configs[4] as an 8-GPU run builds it: rank 3's 2^22-row shard, generated alone
    (synth.make(name, r0, r1)), with the global th0 decision forced (aggregation on)."""
    _ok()
    cuts = cbd.equal_bounds(N_UNI, 8)
    S = synth.make("uniform", int(cuts[3]), int(cuts[4]))
    assert S.m == N_UNI // 8 and S.n == N_UNI
    _format_equal(S, agg_mode=1)
