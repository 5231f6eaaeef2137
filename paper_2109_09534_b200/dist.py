"""Multi-GPU S_NMC: one process per GPU, rows of the factor being updated
sharded across ranks, an all-gather of the updated factor after every mode
update.

* Rows are independent within a mode update and every row's stream is keyed
  by (sweep, mode, inner iteration, row) -- never by rank (nmc.cpp:231-236);
  long rows are cut into the same segments whatever the row range
  (update.cu segment_length), so results are bit-identical for any number of
  GPUs (tests/test_gpu_invariance.py, test_gpu_slabs.py).
* Each rank updates a contiguous row range chosen by prefix sums of work
  (sampled entries + a per-row overhead), not equal row counts, keeps only
  that slab of every mode view on its device (ntcb_view_keep_rows: ~1/N of
  the views per GPU) and holds replicas of every factor; only A^(n) is
  exchanged (I_n x ld fp32), Y stays local (it is reset at every S_NMC call,
  nmc.cpp:212-215).
* The exchange is a torch.distributed all-gather (NCCL over NVLink on GPUs,
  gloo in the CPU tests) of padded shards into the resident factor memory.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

ROW_OVERHEAD = 64  # entry-equivalents of fixed per-row cost (finalise + power method)


def blocksizes(offsets: np.ndarray, c: float) -> np.ndarray:
    """floor(c * n_p) per row in double, n_p at c >= 1 (nmc.cpp:36-40)."""
    n = np.diff(np.asarray(offsets, np.uint64)).astype(np.float64)
    if c >= 1.0:
        return n.astype(np.uint64)
    return np.minimum(np.floor(c * n), n).astype(np.uint64)


def partition_rows(offsets: np.ndarray, c: float, world: int) -> List[Tuple[int, int]]:
    """Contiguous row ranges, one per rank, balancing sum(b_p + ROW_OVERHEAD).
    Streaming cost is ~n_p, sampling/accumulation ~b_p; both are known before
    the run because b_p does not depend on the RNG."""
    n = np.diff(np.asarray(offsets, np.uint64)).astype(np.float64)
    b = blocksizes(offsets, c).astype(np.float64)
    work = np.where(b > 0, 0.5 * n + b + ROW_OVERHEAD, 1.0)
    cum = np.concatenate([[0.0], np.cumsum(work)])
    total = cum[-1]
    rows = len(n)
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * k / world, side="left")))
    cuts.append(rows)
    cuts = [min(max(x, 0), rows) for x in cuts]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


class RowGather:
    """Cached buffers + index maps for the per-mode exchange of one factor:
    every rank's rows bounds[k] of the 2-D tensor t (rows x ld) are replaced
    by rank k's copy.  One padded all_gather_into_tensor, then one gather of
    the other ranks' rows into place (3 device ops per call, no allocation:
    at 8 GPUs a mode update is ~0.2 ms, so host-side op count matters)."""

    def __init__(self, t, bounds: Sequence[Tuple[int, int]], rank: int, group=None):
        import torch
        self.t, self.bounds, self.rank, self.group = t, list(bounds), rank, group
        world = len(self.bounds)
        self.S = S = max(1, max(r1 - r0 for r0, r1 in self.bounds))
        self.send = torch.zeros((S, t.shape[1]), dtype=t.dtype, device=t.device)
        self.recv = torch.empty((world * S, t.shape[1]), dtype=t.dtype, device=t.device)
        src, dst = [], []
        for k, (a, b) in enumerate(self.bounds):
            if k != rank and b > a:
                src.extend(range(k * S, k * S + (b - a)))
                dst.extend(range(a, b))
        self.src = torch.tensor(src, dtype=torch.long, device=t.device)
        self.dst = torch.tensor(dst, dtype=torch.long, device=t.device)

    def __call__(self) -> None:
        import torch.distributed as dist
        r0, r1 = self.bounds[self.rank]
        if r1 > r0:
            self.send[: r1 - r0].copy_(self.t[r0:r1])
        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        if self.src.numel():
            self.t.index_copy_(0, self.dst, self.recv.index_select(0, self.src))


def allgather_rows(t, bounds: Sequence[Tuple[int, int]], rank: int, group=None) -> None:
    """In place: every rank's rows bounds[k] of the 2-D tensor t (rows x ld)
    are replaced by rank k's copy.  One padded all-gather (one-shot form of
    RowGather)."""
    RowGather(t, bounds, rank, group)()


class _CudaArray:
    """__cuda_array_interface__ view of a device buffer owned by libntcb."""

    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def factor_tensor(ctx, mode: int, rows: int, which: int = 0):
    """torch view (rows x ld, fp32, cuda) of the resident factor (A or Y)."""
    import torch
    ptr, ld = ctx.factor_device_ptr(mode, which)
    return torch.as_tensor(_CudaArray(ptr, (rows, ld)), device=f"cuda:{ctx.device}")


def setup_p2p(ctx, rank: int, world: int, group=None) -> bool:
    """Fused exchange: every rank maps every other rank's factor replicas (CUDA
    IPC, lazy peer access) and registers them with its context, so the update
    kernel stores each finalised row into all replicas itself.  Collective:
    every rank must call it.  Returns False (nothing registered) when any rank
    cannot map a peer, so all ranks fall back to the all-gather together."""
    import torch.distributed as tdist
    order = ctx.info()[0]
    # every rank reaches every collective below, whatever fails locally
    try:
        handles = [ctx.factor_ipc_handle(m) for m in range(order)]
    except Exception:
        handles = None
    allh = [None] * world
    tdist.all_gather_object(allh, handles, group=group)
    ok, ptrs = all(h is not None for h in allh), [[] for _ in range(order)]
    if ok:
        try:
            for k in range(world):
                if k == rank:
                    continue
                for m in range(order):
                    ptrs[m].append(ctx.ipc_open(allh[k][m]))
        except Exception:
            ok = False
    flags = [None] * world
    tdist.all_gather_object(flags, ok, group=group)
    if not all(flags):
        return False
    for m in range(order):
        ctx.set_factor_peers(m, ptrs[m])
    return True


class ShardedSweep:
    """Drives ntcb over this rank's row shard of every mode, then exchanges
    the updated factor: by the update kernel's own peer stores plus a barrier
    (exchange="p2p", the default when every GPU can map every other's
    memory) or by an NCCL all-gather of the shards (exchange="gather")."""

    def __init__(self, ctx, cfg, rank: int, world: int, group=None, exchange: str = "auto",
                 slab: bool = True):

        import torch
        import torch.distributed as tdist
        self.ctx, self.cfg, self.rank, self.world, self.group = ctx, cfg, rank, world, group
        order, dims, _ = ctx.info()
        self.dims = dims
        self.bounds = [partition_rows(ctx.view_offsets(m), cfg.c, world) for m in range(order)]
        if slab:  # this rank's rows only: ~1/N of every view stays on the device
            for m in range(order):
                ctx.view_keep_rows(m, *self.bounds[m][rank])
        self.view_bytes = [ctx.view_resident(m)[2] for m in range(order)]
        self.A = [factor_tensor(ctx, m, dims[m]) for m in range(order)]
        st = torch.cuda.current_stream()
        if st.cuda_stream == 0:  # legacy default stream has no handle; use a real one
            st = torch.cuda.Stream()
            torch.cuda.set_stream(st)
        ctx.set_stream(st.cuda_stream)
        dist_on = tdist.is_available() and tdist.is_initialized()
        if exchange == "auto":  # fused peer stores wherever every rank can map every other
            exchange = "p2p"
        self.p2p = bool(dist_on and world > 1 and exchange == "p2p" and setup_p2p(ctx, rank, world, group))
        self.exchange = "p2p" if self.p2p else "gather"
        # the exchange runs whenever a process group exists (at world size 1 too:
        # NTCB_FORCE_SHARDED exercises the NCCL path on one GPU)
        self.gather = None if (self.p2p or not dist_on) else \
            [RowGather(self.A[m], self.bounds[m], rank, group) for m in range(order)]
        self.nccl = dist_on and tdist.get_backend(group) == "nccl"
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda" if self.nccl else "cpu")

    def barrier(self) -> None:
        """Every rank's queued updates (and their peer stores) are complete
        before anything this rank enqueues next: a one-element NCCL all-reduce
        ordered on the stream, or collect + a host barrier on gloo."""
        import torch.distributed as tdist
        if self.nccl:
            tdist.all_reduce(self.flag, group=self.group)
        else:
            self.ctx.collect()
            tdist.barrier(group=self.group)

    def sweep_mode(self, k: int, m: int, seed: int) -> None:
        """This rank's rows of the mode-m update of sweep k, then the exchange."""
        from .ntc import sweep_stream
        r0, r1 = self.bounds[m][self.rank]
        self.ctx.s_nmc_rows_async(m, r0, r1, self.cfg, sweep_stream(seed, k, m).state)
        if self.p2p:
            self.barrier()
        elif self.gather is not None:
            self.gather[m]()

    def sweep(self, k: int, seed: int) -> None:
        for m in range(len(self.dims)):
            self.sweep_mode(k, m, seed)

    def metrics(self):
        """(sse, sum x^2, sum ||U||^2) of the whole tensor: every rank's
        partial sums over its mode-0 slab, all-reduced (the factors are
        replicated, so the regulariser is taken from this rank)."""
        import torch
        import torch.distributed as tdist
        sse, sx, reg = self.ctx.metrics()
        t = torch.tensor([sse, sx], dtype=torch.float64, device="cuda" if self.nccl else "cpu")
        if tdist.is_available() and tdist.is_initialized():
            tdist.all_reduce(t, group=self.group)
        return float(t[0]), float(t[1]), reg

    def local_sampled(self, m: int) -> int:
        r0, r1 = self.bounds[m][self.rank]
        off = self.ctx.view_offsets(m)
        return int(blocksizes(off[r0: r1 + 1], self.cfg.c).sum()) * self.cfg.max_inner
