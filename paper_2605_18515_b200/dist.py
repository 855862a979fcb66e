"""Row sharding across GPUs — plumbing around the C ABI.

* ``shard_bounds`` cuts the rows at 16-row block-row boundaries by prefix-summed
  nnz: cut k is the first block row whose cumulative nnz reaches k*nnz/P.
  Block rows are independent units of the method (no block spans two block
  rows and column aggregation is per block row), so a single SpMV needs
  no exchange: x is replicated, each rank owns a y slice.
* ``global_agg`` makes the th0 decision global: every rank computes its
  shard's block statistics with ``cbspmv_block_stats``, the counts are summed
  across ranks, and ``cbspmv_decide_agg`` applies the rule; the result is passed
  as ``agg_mode`` to every shard's ``cbspmv_build``.
* ``PowerIteration`` is the iterated-SpMV driver of BASELINE config 5:
  per step y_k = A (x_k / ||y_{k-1}||) (the normalisation folded into the x load
  by ``cbspmv_spmv_scaled``), then sum(y_k^2) all-reduced and y shards all-gathered
  into the next x over NCCL.

* ``PanelPowerIteration`` / ``power_iteration_overlapped``:
  the same recurrence with the all-gather split into one broadcast per x owner and
  the next step's column panels (``cbspmv_spmv_panel``) each started as soon as the
  x slices it reads have arrived, so the exchange hides behind the SpMV.

Collectives go through ``torch.distributed`` (NCCL on GPUs, gloo in CPU tests);
the compute steps are injected so the host logic is testable without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_bounds(row_ptr: np.ndarray, parts: int, blk: int = 16) -> np.ndarray:
    """Row cut points r_0 = 0 <= r_1 <= ... <= r_P = m at block-row boundaries, balanced by nnz."""
    m = len(row_ptr) - 1
    nbr = (m + blk - 1) // blk
    br_end = np.minimum((np.arange(nbr) + 1) * blk, m)
    cum = row_ptr[br_end] if nbr else np.zeros(0, np.int64)  # nnz of block rows [0, b]
    total = int(row_ptr[-1]) if m else 0
    cuts = [0]
    for k in range(1, parts):
        target = total * k / parts
        b = int(np.searchsorted(cum, target, side="left"))  # first block row with cum >= target
        r = min(m, (b + 1) * blk) if total else min(m, (m * k // parts) // blk * blk)
        cuts.append(max(cuts[-1], r))
    cuts.append(m)
    return np.asarray(cuts, np.int64)


def equal_bounds(m: int, parts: int, blk: int = 16) -> np.ndarray:
    """Equal row shards rounded to block rows (used when every row has the same nnz)."""
    cuts = [min(m, (m * k // parts) // blk * blk) for k in range(parts)] + [m]
    return np.asarray(cuts, np.int64)


def slice_rows(A, r0: int, r1: int):
    """Rows [r0, r1) of a CSR as a CSR with global n (a row shard, P:433 block rows intact)."""
    from types import SimpleNamespace
    b, e = int(A.row_ptr[r0]), int(A.row_ptr[r1])
    return SimpleNamespace(m=r1 - r0, n=A.n, row_ptr=(A.row_ptr[r0:r1 + 1] - b).astype(np.int64),
                           col=A.col[b:e], val=A.val[b:e], r0=getattr(A, "r0", 0) + r0,
                           name=f"{getattr(A, 'name', 'A')}[{r0}:{r1}]")


def global_agg(A_shard, all_reduce_sum, dtype="f64", **opts) -> int:
    """The th0 decision on the whole matrix from per-shard statistics."""
    import paper_2605_18515_b200 as cb
    nb, ss = cb.block_stats(A_shard, dtype=dtype, **opts)
    tot = all_reduce_sum(np.array([nb, ss], np.int64))
    return cb.decide_agg(int(tot[0]), int(tot[1]), **{k: v for k, v in opts.items() if k.startswith("th0")})


@dataclass
class PowerIteration:
    """y_k = A (x_k / sqrt(sumsq_{k-1})); sumsq_k = allreduce(sum y_k^2); x_{k+1} = allgather(y_k).

    spmv_scaled(x, sumsq, y), sumsq_fn(y, out), all_reduce_sum_(t), all_gather_(out, inp)
    are injected: the C-ABI calls + NCCL on GPUs, the oracle + gloo in CPU tests.
    The eigenvalue estimate after step k is lambda_k = sqrt(sumsq_k) (x_k has unit norm)."""

    spmv_scaled: object
    sumsq_fn: object
    all_reduce_sum_: object
    all_gather_: object

    def run(self, x, y, sumsq, steps: int, on_step=None):
        """x: full vector (replicated), y: this rank's shard, sumsq: 1-element accumulator
        holding sum(x^2) of the initial x (so step 0 normalises x_0)."""
        for k in range(steps):
            self.spmv_scaled(x, sumsq, y)
            self.sumsq_fn(y, sumsq)
            self.all_reduce_sum_(sumsq)
            self.all_gather_(x, y)
            if on_step is not None:
                on_step(k, x, y, sumsq)
        return x, sumsq


def power_iteration_device(h, x0, steps: int, world: int = 1, group=None, on_step=None):
    """BASELINE configs[4] on the device: y_k = A_shard (x_k / ||x_k||) through
    cbspmv_spmv_scaled (normalisation folded into the x load), sum(y_k^2) by
    cbspmv_sumsq, then an NCCL all-reduce of the 8-byte sum and an all-gather of the
    y shards into the next x (equal shards).  One rank owns rows
    [rank*m/world, (rank+1)*m/world) of a square matrix; x0 is the full start vector.
    Returns (x, sumsq) on the device; lambda_k = sqrt(sumsq_k)."""
    import torch
    import torch.distributed as tdist

    import paper_2605_18515_b200 as cb
    m_local = h.info["m"]
    if world * m_local != x0.numel() or h.info["n"] != x0.numel():
        # all_gather_into_tensor needs equal shards of a square matrix
        raise ValueError(f"power_iteration_device: {world} shards of {m_local} rows do not make the "
                         f"{x0.numel()}-long iterate (use power_iteration_overlapped / _fused for unequal shards)")
    x = x0.clone()
    y = torch.empty(m_local, dtype=x0.dtype, device=x0.device)
    ss = torch.zeros(1, dtype=torch.float64, device=x0.device)
    cb.sumsq(x, ss, device=x0.device.index)           # ||x_0||^2 (replicated x)
    for k in range(steps):
        cb.spmv_scaled(h, x, ss, y)                     # y = A (x / sqrt(ss))
        cb.sumsq(y, ss, device=x0.device.index)         # local sum of squares
        if world > 1:
            tdist.all_reduce(ss, group=group)
            tdist.all_gather_into_tensor(x, y, group=group)
        else:
            x, y = y, x                                 # the full y is the next x
        if on_step is not None:
            on_step(k, x, ss)
    return x, ss


def check_row_bounds(row_bounds, n: int) -> list[tuple[int, int]]:
    """The ranks' row slices must tile [0, n) in rank order (the next x is their concatenation)."""
    rb = [(int(a), int(b)) for a, b in row_bounds]
    if not rb or rb[0][0] != 0 or rb[-1][1] != n or any(a > b for a, b in rb) \
            or any(rb[i][1] != rb[i + 1][0] for i in range(len(rb) - 1)):
        raise ValueError(f"row shards {rb} do not tile [0, {n})")
    return rb


def gather_row_bounds(m_local: int, n: int, world: int, group=None) -> list[tuple[int, int]]:
    """Every rank's (r0, r1) from the shard sizes (all-gathered; shards are consecutive in rank
    order), checked to tile [0, n).  Works for unequal shards (``equal_bounds`` with m not a
    multiple of 16*world, or ``shard_bounds``' nnz cut)."""
    if world == 1:
        sizes = [int(m_local)]
    else:
        import torch.distributed as tdist
        sizes = [None] * world
        tdist.all_gather_object(sizes, int(m_local), group=group)
    cuts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return check_row_bounds(list(zip(cuts[:-1], cuts[1:])), n)


def panel_owners(c0: int, c1: int, row_bounds) -> list[int]:
    """Ranks whose x slice [r_a, r_b) intersects the panel's columns [c0, c1)."""
    return [r for r, (a, b) in enumerate(row_bounds) if a < c1 and b > c0]


class PanelPowerIteration:
    """NEXT-1 (i): power iteration whose x exchange overlaps the next step's SpMV.

    Same recurrence as ``PowerIteration`` (y_k = A_shard (x_k / sqrt(sumsq_{k-1})),
    sumsq_k = allreduce(sum y_k^2), x_{k+1} = concat of the y_k shards).  x is double-buffered:
    y_k is computed in place into the next buffer's own slice, then every rank broadcasts its
    slice (one asynchronous collective per owner, issued in owner order, identical on every
    rank).  Step k+1 runs its column panels in arrival order -- panels reading only the rank's
    own slice first -- and waits, before each panel, on exactly the broadcasts that panel reads;
    all of a step's broadcasts are waited before the step ends, so no buffer is overwritten
    while a broadcast still reads it.

    Injected ops (device: the C ABI + NCCL, ``power_iteration_overlapped``; CPU tests: numpy +
    gloo): ``spmv_panel(p, x, sumsq, y, zero_y)``, ``sumsq_fn(y, out)``,
    ``all_reduce_sum_async(t) -> work``, ``broadcast_async(t, src) -> work``; ``work.wait()``
    orders the caller after the collective.  ``panels``: column bounds of the handle's panels;
    ``row_bounds``: the x slice each rank owns (its y rows)."""

    def __init__(self, spmv_panel, sumsq_fn, all_reduce_sum_async, broadcast_async, panels, row_bounds, rank):
        self.spmv_panel, self.sumsq_fn = spmv_panel, sumsq_fn
        self.all_reduce_sum_async, self.broadcast_async = all_reduce_sum_async, broadcast_async
        self.row_bounds = [(int(a), int(b)) for a, b in row_bounds]
        self.rank = rank
        self.owners = [panel_owners(c0, c1, self.row_bounds) for c0, c1 in panels]
        remote = [max([o for o in ow if o != rank], default=-1) for ow in self.owners]
        self.order = sorted(range(len(panels)), key=lambda p: (remote[p], p))

    def run(self, xa, xb, sumsq, steps: int, on_step=None):
        """xa: full x_0 (replicated), xb: a second full-length buffer, sumsq: sum(x_0^2).
        Returns (x, sumsq) with x = the last iterate (complete on return)."""
        world = len(self.row_bounds)
        r0, r1 = self.row_bounds[self.rank]
        pending = {}
        cur, nxt = xa, xb
        for k in range(steps):
            y = nxt[r0:r1]
            for i, p in enumerate(self.order):
                for o in self.owners[p]:
                    w = pending.pop(o, None)
                    if w is not None:
                        w.wait()
                self.spmv_panel(p, cur, sumsq, y, i == 0)
            for w in pending.values():  # incl. this rank's own (source) broadcast
                w.wait()
            pending = {}
            self.sumsq_fn(y, sumsq)
            if world > 1:
                self.all_reduce_sum_async(sumsq).wait()
                pending = {s: self.broadcast_async(nxt[a:b], s) for s, (a, b) in enumerate(self.row_bounds)}
            cur, nxt = nxt, cur
            if on_step is not None:  # debugging / tests: a complete x costs the overlap
                for w in pending.values():
                    w.wait()
                pending = {}
                on_step(k, cur, sumsq)
        for w in pending.values():
            w.wait()
        return cur, sumsq


def power_iteration_overlapped(h, x0, steps: int, world: int = 1, rank: int = 0, group=None, on_step=None):
    """``PanelPowerIteration`` on the device: panels through ``cbspmv_spmv_panel``, the
    finalize through ``cbspmv_sumsq``, collectives over NCCL (``async_op`` works whose
    ``wait()`` makes the current stream wait, not the host).  Equal row shards of a square
    matrix; x0 is the full start vector.  Returns (x, sumsq) on the device."""
    import torch
    import torch.distributed as tdist

    import paper_2605_18515_b200 as cb
    dev = x0.device.index
    if h.info["n"] != x0.numel():
        raise ValueError("x0 must hold the handle's n columns")
    row_bounds = gather_row_bounds(h.info["m"], x0.numel(), world, group)
    panels = [cb.panel_bounds(h, p) for p in range(h.info["n_panels"])]
    it = PanelPowerIteration(
        spmv_panel=lambda p, x, ss, y, z: cb.spmv_panel(h, p, x, ss, y, z),
        sumsq_fn=lambda y, out: cb.sumsq(y, out, device=dev),
        all_reduce_sum_async=lambda t: tdist.all_reduce(t, group=group, async_op=True),
        broadcast_async=lambda t, src: tdist.broadcast(t, src=src, group=group, async_op=True),
        panels=panels, row_bounds=row_bounds, rank=rank)
    xa = x0.clone()
    xb = torch.empty_like(x0)
    ss = torch.zeros(1, dtype=torch.float64, device=x0.device)
    cb.sumsq(xa, ss, device=dev)
    return it.run(xa, xb, ss, steps, on_step=on_step)


class PeerPowerIteration:
    """NEXT-1 (ii): the power-iteration exchange as one fused kernel over peer memory.

    Same recurrence as ``PowerIteration``.  Every rank holds the two iterate buffers X[0], X[1];
    ``row_bounds`` (the ranks' row slices, any sizes) must tile [0, n).
    Step k: wait for flag k (every rank published step k-1; the wait also sums the ranks'
    partials of ||y_{k-1}||^2 in rank order), y_k = A_r (X[k&1] / ||.||) straight into the
    rank's own slice of X[(k+1)&1], then ``publish`` stores that slice into every peer's
    X[(k+1)&1], sends its partial sum of squares and releases flag k+1 -- all in one kernel
    (``cbspmv_xchg_publish``); no all-reduce, no all-gather, no host round trip.  The step
    counter k is global to the buffers (flags only grow): a run may continue or restart at k0,
    the first step of a run taking its x and sumsq from the caller instead of a wait.

    Injected ops (device: ``FusedPowerIteration``; CPU tests: numpy + gloo emulation):
    ``spmv_scaled(x, sumsq, y)``, ``publish(b, r0, length, seq)``, ``wait(seq, sumsq)``."""

    def __init__(self, spmv_scaled, publish, wait, row_bounds, rank, n=None):
        self.spmv_scaled, self.publish, self.wait = spmv_scaled, publish, wait
        rb = [(int(a), int(b)) for a, b in row_bounds]
        self.row_bounds = check_row_bounds(rb, rb[-1][1] if n is None else n)
        self.rank = rank

    def run(self, X, sumsq, steps: int, on_step=None, k0: int = 0, mark=None):
        """X: the two iterate buffers with x_{k0} in X[k0 & 1]; sumsq: ||x_{k0}||^2.
        mark(phase) (optional) is called after each enqueued phase ("wait", "spmv", "publish"),
        e.g. to record CUDA events for a per-phase time split.
        Returns (x_{k0+steps}, sumsq), complete on every rank."""
        r0, r1 = self.row_bounds[self.rank]
        for k in range(k0, k0 + steps):
            if k > k0:
                self.wait(k, sumsq)
                if mark is not None:
                    mark("wait")
            cur, nxt = X[k & 1], X[(k + 1) & 1]
            self.spmv_scaled(cur, sumsq, nxt[r0:r1])
            if mark is not None:
                mark("spmv")
            self.publish((k + 1) & 1, r0, r1 - r0, k + 1)
            if mark is not None:
                mark("publish")
            if on_step is not None:
                self.wait(k + 1, sumsq)  # debugging / tests: a complete iterate costs the overlap
                on_step(k - k0, nxt, sumsq)
        if steps:
            self.wait(k0 + steps, sumsq)
        return X[(k0 + steps) & 1], sumsq


class FusedPowerIteration:
    """``PeerPowerIteration`` on the device.  The iterate buffers and flags live in one
    ``cbspmv_xchg`` context per rank whose allocation every peer maps through CUDA IPC (handles
    exchanged once with ``all_gather_object``); per step one ``cbspmv_spmv_scaled`` and one
    fused ``cbspmv_xchg_publish``, the next step gated on the device by ``cbspmv_xchg_wait``.
    Row shards of a square matrix, consecutive in rank order, any sizes (the bounds are
    all-gathered and checked to tile [0, n)).  ``run(x0, steps)`` restarts from x0 (replicated)
    and returns (x, sumsq); x is a view of a context buffer, valid until the next run / destroy.
    A device wait that timed out (a peer never published) poisons the exchange; ``run`` checks
    the context's status after the steps and raises."""

    def __init__(self, h, n: int, dtype="f64", world: int = 1, rank: int = 0, device: int = 0, group=None,
                 timeout_s: float = 30.0):
        import torch
        import torch.distributed as tdist

        import paper_2605_18515_b200 as cb
        self.h, self.world, self.rank, self.device = h, world, rank, device
        if h.info["n"] != n:
            raise ValueError(f"the handle has {h.info['n']} columns, the iterate {n}")
        row_bounds = gather_row_bounds(h.info["m"], n, world, group)
        self.xc = cb.Exchange(n, dtype, world, rank, device)
        if world > 1:
            handles = [None] * world
            tdist.all_gather_object(handles, self.xc.ipc_handle(), group=group)
            self.xc.connect(ipc_handles=handles)
        else:
            self.xc.connect(peer_bases=[self.xc.base()])
        self.X = [self.xc.buffer(0), self.xc.buffer(1)]
        self.ss = torch.zeros(1, dtype=torch.float64, device=f"cuda:{device}")
        xc = self.xc
        self.it = PeerPowerIteration(
            spmv_scaled=lambda x, s, y: cb.spmv_scaled(h, x, s, y),
            publish=lambda b, r0, ln, seq: xc.publish(b, r0, ln, seq),
            wait=lambda seq, s: xc.wait(seq, s, timeout_s),
            row_bounds=row_bounds, rank=rank, n=n)
        self.k = 0
        torch.cuda.synchronize(device)
        if world > 1:
            tdist.barrier(group=group)  # every peer mapped before anyone stores into it

    def run(self, x0, steps: int, on_step=None, mark=None):
        import paper_2605_18515_b200 as cb
        # safe to overwrite X[k & 1]: every peer's last store into it preceded our last wait(k)
        self.X[self.k & 1].copy_(x0)
        cb.sumsq(self.X[self.k & 1], self.ss, device=self.device)
        if mark is not None:
            mark("start")
        x, ss = self.it.run(self.X, self.ss, steps, on_step=on_step, k0=self.k, mark=mark)
        self.k += steps
        if self.xc.timed_out():  # synchronous status read: the run's waits have all executed
            raise RuntimeError("fused exchange: a device wait timed out (a peer never published); "
                               "the iterate is poisoned (NaN)")
        return x, ss

    def timed_out(self) -> bool:
        return self.xc.timed_out()

    def destroy(self) -> None:
        self.xc.destroy()


def power_iteration_fused(h, x0, steps: int, world: int = 1, rank: int = 0, group=None, on_step=None,
                          timeout_s: float = 30.0):
    """One-shot ``FusedPowerIteration``: returns (x, sumsq, driver); call ``driver.destroy()``
    when x (a view of its buffer) is no longer needed."""
    f = FusedPowerIteration(h, x0.numel(), {4: "f32", 8: "f64"}[x0.element_size()], world, rank,
                            x0.device.index, group, timeout_s)
    x, ss = f.run(x0, steps, on_step=on_step)
    return x, ss, f
