"""GPU tests of the fused finalize + exchange over peer memory (SURVEY §8(f) NEXT-1 (ii),
include/cbspmv.h cbspmv_xchg_*): the power iteration of BASELINE configs[4] with the y shards
pushed into every peer's next iterate by one kernel and the next step gated by device flags.

This run has one GPU, so the peers are (a) P contexts in one process on cuda:0, connected by
plain device pointers and interleaved on one stream, and (b) two processes on cuda:0 connected
through CUDA IPC, each spinning on the other's flags.  Both must reproduce the recurrence the
oracle's recurrence (plain C SpMV, oracle/) to within the fp64 bar, every rank holding the same
bits.
"""
import os
import socket
import time

import numpy as np
import pytest

import paper_2605_18515_b200 as cb
import synth
from paper_2605_18515_b200 import dist as cbd

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _ok():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _reference(A, steps, dtype=torch.float64):
    """The recurrence y_k = A (x_k / sqrt(ss_{k-1})), ss_k = y_k . y_k with the oracle's SpMV
    (fp64, single-threaded C, oracle/); fp32: the oracle on the fp32-rounded A, rounding y to
    fp32 after each step like the device iterate."""
    import oracle
    B = A
    if dtype == torch.float32:
        B = synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    x, ss = np.ones(A.n), float(A.n)
    for _ in range(steps):
        y = oracle.spmv_csr(B, x / np.sqrt(ss))[0]
        if dtype == torch.float32:
            y = y.astype(np.float32).astype(np.float64)
        ss = float(y @ y)
        x = y
    return x, ss


def _simulated_ranks(A, P, steps, dtype="f64", unequal=False, bounds=None):
    """P ranks in one process on one GPU, run step-interleaved on one stream.  unequal: the
    shards of dist.shard_bounds (nnz cut at block-row boundaries, unequal row counts); bounds:
    explicit row ranges."""
    m_loc = A.m // P
    if bounds is None:
        bounds = [(r * m_loc, (r + 1) * m_loc) for r in range(P)]
    if unequal:
        cuts = cbd.shard_bounds(A.row_ptr, P)
        bounds = cbd.check_row_bounds(list(zip(cuts[:-1], cuts[1:])), A.n)
    hs = [cb.build(cbd.slice_rows(A, a, b), dtype=dtype, device=0) for a, b in bounds]
    xcs = [cb.Exchange(A.n, dtype, P, r, 0) for r in range(P)]
    bases = [xc.base() for xc in xcs]
    for xc in xcs:
        xc.connect(peer_bases=bases)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    sss = []
    for xc in xcs:
        xc.buffer(0).fill_(1.0)
        xc.buffer(1).fill_(float("nan"))  # every slice must be overwritten by its owner's publish
        ss = torch.zeros(1, dtype=torch.float64, device=DEV)
        cb.sumsq(xc.buffer(0), ss)
        sss.append(ss)
    for k in range(steps):
        for r, (a, b) in enumerate(bounds):
            if k:
                xcs[r].wait(k, sss[r], timeout_s=5.0)
            cb.spmv_scaled(hs[r], xcs[r].buffer(k & 1), sss[r], xcs[r].buffer((k + 1) & 1)[a:b])
            xcs[r].publish((k + 1) & 1, a, b - a, k + 1)
    for r in range(P):
        xcs[r].wait(steps, sss[r], timeout_s=5.0)
    torch.cuda.synchronize()
    assert not any(xc.timed_out() for xc in xcs)
    xs = [xc.buffer(steps & 1).to(tdt).cpu().numpy().copy() for xc in xcs]
    ss = [float(s.item()) for s in sss]
    for h in hs:
        cb.destroy(h)
    for xc in xcs:
        xc.destroy()
    return xs, ss


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_fused_exchange_simulated_ranks_match_recurrence(P):
    _ok()
    n = 2048 * P
    A = synth.uniform(n, n, 40, 61, val_mode=1)  # values U(0,1]: converging power iteration
    steps = 12
    x_ref, ss_ref = _reference(A, steps)
    xs, ss = _simulated_ranks(A, P, steps)
    assert len(set(ss)) == 1  # partials summed in rank order: identical bits on every rank
    assert np.isclose(ss[0], ss_ref, rtol=1e-13)
    for x in xs:
        assert np.array_equal(x, xs[0])  # every rank holds the complete, identical iterate
        assert np.allclose(x, x_ref, rtol=1e-12, atol=0)


@pytest.mark.parametrize("P", [3, 5])
def test_fused_exchange_unequal_shards(P):
    """Row shards of different lengths (an nnz cut of a matrix whose rows differ in length):
    every rank publishes its own slice at its own offset; same recurrence."""
    _ok()
    A = synth.make("rmat", small=True)  # power-law rows: the nnz cut gives unequal row counts
    bounds = cbd.shard_bounds(A.row_ptr, P)
    assert len(set(np.diff(bounds).tolist())) > 1
    B = synth.CSR(A.m, A.n, A.row_ptr, A.col, np.abs(A.val))  # nonnegative: a converging iteration
    steps = 10
    x_ref, ss_ref = _reference(B, steps)
    xs, ss = _simulated_ranks(B, P, steps, unequal=True)
    assert len(set(ss)) == 1 and np.isclose(ss[0], ss_ref, rtol=1e-12)
    for x in xs:
        assert np.array_equal(x, xs[0]) and np.allclose(x, x_ref, rtol=1e-11, atol=1e-300)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fused_exchange_ragged_slices(dtype):
    """Slices whose offsets / lengths are not multiples of a 16-byte store (odd row cuts): the
    publish kernel's unaligned and tail paths next to its 16-byte path."""
    _ok()
    n = 3001
    A = synth.uniform(n, n, 30, 63, val_mode=1)
    bounds = [(0, 1001), (1001, 2002), (2002, 3001)]  # offsets 1001 / 2002: not 16-byte aligned
    steps = 8
    x_ref, ss_ref = _reference(A, steps, torch.float32 if dtype == "f32" else torch.float64)
    xs, ss = _simulated_ranks(A, 3, steps, dtype=dtype, bounds=bounds)
    assert len(set(ss)) == 1
    tol = 1e-5 if dtype == "f32" else 1e-12
    assert np.isclose(ss[0], ss_ref, rtol=tol)
    for x in xs:
        assert np.array_equal(x, xs[0]) and np.allclose(x, x_ref, rtol=tol, atol=0)


def test_fused_exchange_all_ones_fixed_point():
    """Uniform all-ones, 50 per row: lambda = 50 at every step (SURVEY §8(c) closed form)."""
    _ok()
    n = 4096
    A = synth.uniform(n, n, 50, 62, val_mode=3)
    xs, ss = _simulated_ranks(A, 4, 20)
    # n = 4096: 1/64, 50/64, per-rank partials 625 and 2500 are dyadic -- exact in any order
    assert ss == [2500.0] * 4
    assert np.all(xs[0] == 50.0 / 64.0)


def test_fused_exchange_f32():
    _ok()
    n = 4096
    A = synth.uniform(n, n, 40, 63, val_mode=1)
    x_ref, ss_ref = _reference(A, 8, torch.float32)
    xs, ss = _simulated_ranks(A, 2, 8, dtype="f32")
    assert len(set(ss)) == 1
    assert np.isclose(ss[0], ss_ref, rtol=1e-5)
    assert np.allclose(xs[0], x_ref, rtol=1e-5)


def test_fused_exchange_wait_times_out_without_publisher():
    """A rank whose peer never publishes: the device wait gives up (bounded spin), flags it and
    poisons the context -- sumsq = NaN, later publishes store nothing into the peers and release
    no flag, later waits fail at once -- no hang."""
    _ok()
    xcs = [cb.Exchange(64, "f64", 2, r, 0) for r in range(2)]
    for xc in xcs:
        xc.connect(peer_bases=[x.base() for x in xcs])
    ss = torch.full((1,), 7.0, dtype=torch.float64, device=DEV)
    xcs[0].wait(1, ss, timeout_s=0.05)
    torch.cuda.synchronize()
    assert xcs[0].timed_out() and np.isnan(float(ss.item()))
    # poisoned: rank 0's publish leaves rank 1's buffer and flags alone
    xcs[1].buffer(1).fill_(-1.0)
    xcs[0].buffer(1).fill_(3.0)
    xcs[0].publish(1, 0, 32, 1)
    ss1 = torch.zeros(1, dtype=torch.float64, device=DEV)
    xcs[1].publish(1, 32, 32, 1)   # rank 1 is healthy: its own flag 1 is released
    xcs[1].wait(1, ss1, timeout_s=0.05)
    torch.cuda.synchronize()
    assert bool((xcs[1].buffer(1)[:32] == -1.0).all())
    assert xcs[1].timed_out()      # rank 0 never released flag 1 on rank 1
    t0 = time.perf_counter()
    ss.fill_(7.0)
    xcs[0].wait(2, ss, timeout_s=5.0)  # already poisoned: returns at once, not after 5 s
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 2.0 and np.isnan(float(ss.item()))
    for xc in xcs:
        xc.destroy()


def test_fused_exchange_argument_errors():
    _ok()
    with pytest.raises(cb.CBSpMVError):
        cb.Exchange(16, "f64", 9, 0, 0)  # world > 8
    xc = cb.Exchange(16, "f64", 2, 0, 0)
    with pytest.raises(cb.CBSpMVError):
        xc.publish(1, 0, 16, 1)  # peer 1 not connected
    xc.connect(peer_bases=[xc.base(), xc.base()])
    with pytest.raises(cb.CBSpMVError):
        xc.publish(1, 8, 16, 1)  # slice past n
    with pytest.raises(cb.CBSpMVError):
        xc.publish(1, 0, 8, 0)  # seq 0 is reserved (flags start at 0)
    xc.destroy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, steps, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)  # handle exchange + barrier only
    try:
        torch.cuda.set_device(0)
        n = 4096 * world
        A = synth.uniform(n, n, 40, 64, val_mode=1)
        m_loc = n // world
        h = cb.build(cbd.slice_rows(A, rank * m_loc, (rank + 1) * m_loc), device=0)
        x0 = torch.ones(n, dtype=torch.float64, device=DEV)
        x, ss, xc = cbd.power_iteration_fused(h, x0, steps, world, rank, timeout_s=20.0)
        torch.cuda.synchronize()
        first = x.cpu().numpy().copy()
        x, ss = xc.run(x0, steps)  # restart on the same buffers: flags keep growing
        torch.cuda.synchronize()
        assert np.allclose(x.cpu().numpy(), first, rtol=1e-13, atol=0)  # fp64 RED order may differ
        q.put((rank, xc.timed_out(), float(ss.item()), first))
        tdist.barrier()  # nobody unmaps while a peer may still store into it
        xc.destroy()
        cb.destroy(h)
    finally:
        tdist.destroy_process_group()


def test_fused_exchange_two_processes_ipc():
    """Two processes on cuda:0 mapping each other's iterate buffers through CUDA IPC."""
    _ok()
    import torch.multiprocessing as mp
    steps, world = 10, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 4096 * world
    x_ref, ss_ref = _reference(synth.uniform(n, n, 40, 64, val_mode=1), steps)
    for rank, timed_out, ss, x in res:
        assert not timed_out
        assert ss == res[0][2]
        assert np.isclose(ss, ss_ref, rtol=1e-13)
        assert np.allclose(x, x_ref, rtol=1e-12, atol=0)
