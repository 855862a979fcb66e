"""Multi-GPU host logic on CPU: row sharding, the global th0 decision and the power-iteration
driver, with world_size 2 over torch.distributed gloo.

The per-rank SpMV is the oracle here (a CPU stand-in for the device); the sharded
builds are the real C-ABI builder in host-only mode.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2605_18515_b200 as cb
import synth
from paper_2605_18515_b200 import dist as cbd


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_properties():
    for name in ("rmat", "clustered", "laplace"):
        A = synth.make(name, small=True)
        for P in (1, 2, 3, 8):
            cuts = cbd.shard_bounds(A.row_ptr, P)
            assert cuts[0] == 0 and cuts[-1] == A.m and len(cuts) == P + 1
            assert np.all(np.diff(cuts) >= 0)
            assert all(c % 16 == 0 or c == A.m for c in cuts)
            loads = np.diff(A.row_ptr[cuts])
            max_br = max(int(A.row_ptr[min(A.m, r + 16)] - A.row_ptr[r]) for r in range(0, A.m, 16))
            assert loads.max() - A.nnz / P <= max_br  # within one block row of the ideal share
    assert cbd.equal_bounds(1 << 15, 8).tolist() == [i * 4096 for i in range(9)]


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.make(name, small=True)
        cuts = cbd.shard_bounds(A.row_ptr, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        S = cbd.slice_rows(A, r0, r1)

        def allreduce(a):
            t = torch.from_numpy(np.asarray(a, np.int64).copy())
            dist.all_reduce(t)
            return t.numpy()

        agg = cbd.global_agg(S, allreduce)
        h = cb.build(S, device=-1, agg_mode=agg)
        ex = cb.export(h)
        ref = oracle.build(S, agg_mode=agg)
        same = all(np.array_equal(ex[k], getattr(ref, k)) for k in
                   ("blk_row_idx", "blk_col_idx", "nnz_per_blk", "type_per_blk", "vp_per_blk", "mtx_data",
                    "restore_cols", "cols_offset", "tb_ptr", "tb_load"))
        x = synth.vector(A.n, synth.VEC_UNIFORM, seed=3)
        y_shard, _ = oracle.spmv_csr(S, x)
        parts = [None] * world
        dist.all_gather_object(parts, (r0, y_shard))
        q.put((rank, agg, same, parts if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rmat", "clustered"])
def test_two_rank_sharded_build_and_spmv(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synth.make(name, small=True)
    full = oracle.build(A)
    for rank, agg, same, _ in res:
        assert agg == full.agg  # the global th0 decision equals the whole-matrix decision (R-5)
        assert same             # each shard's build is byte-identical to the oracle's
    parts = next(p for _, _, _, p in res if p is not None)
    y = np.concatenate([y for _, y in sorted(parts, key=lambda t: t[0])])
    y_ref, _ = oracle.spmv_csr(A, synth.vector(A.n, synth.VEC_UNIFORM, seed=3))
    assert np.array_equal(y, y_ref)  # row shards compute exactly the rows of the full product


def _pi_worker(rank, world, port, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.uniform(4096, 4096, 50, 51, val_mode=1)
        cuts = cbd.equal_bounds(A.m, world)
        S = cbd.slice_rows(A, int(cuts[rank]), int(cuts[rank + 1]))

        def spmv_scaled(x, ss, y):  # oracle stand-in for cbspmv_spmv_scaled
            xs = x.numpy() / np.sqrt(ss.item())
            y.copy_(torch.from_numpy(oracle.spmv_csr(S, xs)[0]))

        def sumsq(y, out):
            out.fill_(float(torch.dot(y, y)))

        def all_reduce_sum(t):
            dist.all_reduce(t)

        def all_gather(out, inp):
            parts = [torch.empty_like(inp) for _ in range(world)]
            dist.all_gather(parts, inp)
            out.copy_(torch.cat(parts))

        x = torch.ones(A.n, dtype=torch.float64)
        y = torch.empty(S.m, dtype=torch.float64)
        ss = torch.tensor([float(A.n)], dtype=torch.float64)
        lams = []
        pi = cbd.PowerIteration(spmv_scaled, sumsq, all_reduce_sum, all_gather)
        pi.run(x, y, ss, steps, on_step=lambda k, x, y, s: lams.append(float(np.sqrt(s.item()))))
        q.put((rank, lams, x.numpy() if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_two_rank_power_iteration_matches_single_process():
    steps = 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_pi_worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: the same recurrence on the whole matrix with numpy
    A = synth.uniform(4096, 4096, 50, 51, val_mode=1)
    d = A.to_dense()
    x = np.ones(A.n)
    ss = float(A.n)
    lam_ref = []
    for _ in range(steps):
        y = d @ (x / np.sqrt(ss))
        ss = float(y @ y)
        x = y
        lam_ref.append(np.sqrt(ss))
    assert res[0][1] == res[1][1]  # every rank sees the same all-reduced norm
    assert np.allclose(res[0][1], lam_ref, rtol=1e-12)
    assert np.allclose(res[0][2], x, rtol=1e-11)
    # Perron root of a nonnegative matrix with row sums in [?]: bounded by min / max row sums
    rs = d.sum(1)
    assert rs.min() - 1e-9 <= lam_ref[-1] <= rs.max() + 1e-9


def _col_slice(S, c0, c1):
    """Columns [c0, c1) of a CSR (global column indices kept) — the oracle's view of a panel."""
    keep = (S.col >= c0) & (S.col < c1)
    rows = np.repeat(np.arange(S.m), np.diff(S.row_ptr))
    rp = np.zeros(S.m + 1, np.int64)
    np.add.at(rp, rows[keep] + 1, 1)
    return synth.CSR(S.m, S.n, np.cumsum(rp), S.col[keep], S.val[keep])


def _panel_pi_worker(rank, world, port, steps, P, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1024 * world
        A = synth.uniform(n, n, 30, 52, val_mode=1)
        m_loc = n // world
        S = cbd.slice_rows(A, rank * m_loc, (rank + 1) * m_loc)
        h = cb.build(S, device=-1, col_panels=P)  # the real builder's panel cuts
        panels = [cb.panel_bounds(h, p) for p in range(h.info["n_panels"])]
        subs = [_col_slice(S, c0, c1) for c0, c1 in panels]
        ran = []

        def spmv_panel(p, x, ss, y, zero):  # oracle stand-in for cbspmv_spmv_panel
            ran.append(p)
            c0, c1 = panels[p]
            xs = np.zeros(S.n)
            xs[c0:c1] = x.numpy()[c0:c1] / np.sqrt(ss.item())
            part = torch.from_numpy(oracle.spmv_csr(subs[p], xs)[0])
            if zero:
                y.copy_(part)
            else:
                y.add_(part)

        def sumsq(y, out):
            out.fill_(float(torch.dot(y, y)))

        it = cbd.PanelPowerIteration(
            spmv_panel, sumsq,
            all_reduce_sum_async=lambda t: dist.all_reduce(t, async_op=True),
            broadcast_async=lambda t, src: dist.broadcast(t, src=src, async_op=True),
            panels=panels, row_bounds=[(r * m_loc, (r + 1) * m_loc) for r in range(world)], rank=rank)
        xa = torch.ones(n, dtype=torch.float64)
        xb = torch.full((n,), float("nan"), dtype=torch.float64)
        ss = torch.tensor([float(n)], dtype=torch.float64)
        x, ss = it.run(xa, xb, ss, steps)
        own_first = all(it.owners[p] == [rank] for p in it.order[:sum(ow == [rank] for ow in it.owners)])
        q.put((rank, float(ss.item()), x.numpy().copy(), ran[:len(panels)], it.order, own_first))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 2), (2, 5), (3, 5)])
def test_panel_power_iteration_overlap_matches_recurrence(world, P):
    """NEXT-1 (i) host logic: per-owner broadcasts + panels in arrival order == the plain recurrence."""
    steps = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_panel_pi_worker, args=(r, world, port, steps, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1024 * world
    d = synth.uniform(n, n, 30, 52, val_mode=1).to_dense()
    x = np.ones(n)
    ss = float(n)
    for _ in range(steps):
        y = d @ (x / np.sqrt(ss))
        ss = float(y @ y)
        x = y
    for rank, ss_r, x_r, ran, order, own_first in res:
        assert np.isclose(ss_r, ss, rtol=1e-12)
        assert np.allclose(x_r, x, rtol=1e-11)  # every rank ends with the complete iterate
        assert ran == order and own_first


def _peer_n(world, unequal):
    return 1000 * world + 8 if unequal else 1024 * world


def _peer_pi_worker(rank, world, port, steps, q, unequal=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = _peer_n(world, unequal)
        A = synth.uniform(n, n, 30, 53, val_mode=1)
        cuts = cbd.equal_bounds(n, world)  # unequal: n is not a multiple of 16 * world
        S = cbd.slice_rows(A, int(cuts[rank]), int(cuts[rank + 1]))
        row_bounds = cbd.gather_row_bounds(S.m, n, world)  # what FusedPowerIteration derives
        assert row_bounds == [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]
        X = [torch.ones(n, dtype=torch.float64), torch.full((n,), float("nan"), dtype=torch.float64)]
        partials = np.full((2, world), np.nan)  # the context's partials[parity][rank]
        flags = [0] * world
        calls = []

        def spmv_scaled(x, ss, y):  # oracle stand-in for cbspmv_spmv_scaled
            calls.append(("spmv", float(ss.item())))
            y.copy_(torch.from_numpy(oracle.spmv_csr(S, x.numpy() / np.sqrt(ss.item()))[0]))

        def publish(b, r0, length, seq):  # emulates cbspmv_xchg_publish: slice -> every peer's X[b]
            calls.append(("publish", b, seq))
            mine = X[b][r0:r0 + length].clone()
            parts = [None] * world
            dist.all_gather_object(parts, (r0, mine.numpy()))
            for a, v in parts:
                X[b][a:a + len(v)] = torch.from_numpy(v)
            tot = torch.tensor([float(torch.dot(mine, mine))], dtype=torch.float64)
            allp = [torch.empty_like(tot) for _ in range(world)]
            dist.all_gather(allp, tot)
            partials[(seq - 1) & 1] = [float(t.item()) for t in allp]
            for r in range(world):
                flags[r] = seq

        def wait(seq, ss):  # emulates cbspmv_xchg_wait: flags >= seq, partials summed in rank order
            calls.append(("wait", seq))
            assert min(flags) >= seq
            s = 0.0
            for r in range(world):
                s += partials[(seq - 1) & 1][r]
            ss.fill_(s)

        it = cbd.PeerPowerIteration(spmv_scaled, publish, wait, row_bounds=row_bounds, rank=rank, n=n)
        ss = torch.tensor([float(n)], dtype=torch.float64)
        x, ss = it.run(X, ss, steps)
        q.put((rank, float(ss.item()), x.numpy().copy(), calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,unequal", [(2, False), (3, False), (3, True)])
def test_peer_power_iteration_protocol_matches_recurrence(world, unequal):
    """NEXT-1 (ii) host logic: wait(k) -> spmv into X[(k+1)&1] -> publish(seq k+1), double buffers
    and partial parities, == the plain recurrence on every rank.  unequal: shards of 992 / 1008 /
    1008 rows (equal_bounds of 3008 rows), their bounds all-gathered from the shard sizes."""
    steps = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_peer_pi_worker, args=(r, world, port, steps, q, unequal)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = _peer_n(world, unequal)
    d = synth.uniform(n, n, 30, 53, val_mode=1).to_dense()
    x = np.ones(n)
    ss = float(n)
    for _ in range(steps):
        y = d @ (x / np.sqrt(ss))
        ss = float(y @ y)
        x = y
    expect = []
    for k in range(steps):
        if k:
            expect.append(("wait", k))
        expect.append("spmv")
        expect.append(("publish", (k + 1) & 1, k + 1))
    expect.append(("wait", steps))
    for rank, ss_r, x_r, calls in res:
        assert np.isclose(ss_r, ss, rtol=1e-12)
        assert np.allclose(x_r, x, rtol=1e-11)
        assert [c if c[0] != "spmv" else "spmv" for c in calls] == expect
    assert len({r[1] for r in res}) == 1  # partials summed in rank order: the same bits everywhere


def test_row_bounds_must_tile_the_iterate():
    assert cbd.check_row_bounds([(0, 320), (320, 656), (656, 1000)], 1000) == [(0, 320), (320, 656), (656, 1000)]
    for bad in ([(0, 320), (336, 1000)], [(0, 500)], [(16, 1000)], [(0, 600), (500, 1000)]):
        with pytest.raises(ValueError):
            cbd.check_row_bounds(bad, 1000)
    assert cbd.gather_row_bounds(1000, 1000, 1) == [(0, 1000)]
    with pytest.raises(ValueError):
        cbd.gather_row_bounds(999, 1000, 1)
    with pytest.raises(ValueError):  # the protocol driver refuses shards that leave a gap
        cbd.PeerPowerIteration(None, None, None, row_bounds=[(0, 10), (12, 20)], rank=0)


@pytest.mark.parametrize("name", ["laplace", "clustered", "rmat", "uniform"])
def test_row_counts_cut_and_per_rank_generation(name):
    """bench.py's N > 1 input path: per-row counts without materialising the matrix, an nnz cut
    at block-row boundaries, then each rank generates only its rows — identical to slicing the
    full matrix (counter-based generators)."""
    A = synth.make(name, small=True)
    c = synth.row_counts(name, small=True)
    d = np.diff(A.row_ptr)
    assert len(c) == A.m
    if name == "rmat":  # edges per row before duplicate removal: an upper bound
        assert np.all(c >= d) and c.sum() <= 1.2 * d.sum()
    else:
        assert np.array_equal(c, d)
    rp = np.zeros(len(c) + 1, np.int64)
    np.cumsum(c, out=rp[1:])
    cuts = cbd.equal_bounds(A.m, 3) if name == "uniform" else cbd.shard_bounds(rp, 3)
    for r in range(3):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        S = synth.make(name, r0, r1, small=True)
        ref = cbd.slice_rows(A, r0, r1)
        assert S.m == r1 - r0 and np.array_equal(S.row_ptr, ref.row_ptr)
        assert np.array_equal(S.col, ref.col) and np.array_equal(S.val, ref.val)
