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


class Shard:
    """One rank's part of a mode update.  full = whole rows [r0, r1); parts =
    chunk ranges (row, cb, ce) of heavy rows shared with other ranks (chunks
    of segment_length entries from the row start); owned = rows [o0, o1)
    this rank finalises and publishes (its whole rows plus the shared rows
    whose chunk 0 it holds); keep = rows [k0, k1) whose entries it needs."""

    def __init__(self, full, parts, owned, keep):
        self.full, self.parts, self.owned, self.keep = tuple(full), list(parts), tuple(owned), tuple(keep)

    def __repr__(self):
        return f"Shard(full={self.full}, parts={self.parts}, owned={self.owned}, keep={self.keep})"


def partition_split(offsets: np.ndarray, c: float, world: int, seg: int, max_share: float = 1.0,
                    max_split_n: int = 1 << 24) -> List[Shard]:
    """Contiguous ranges over work units balancing sum(n_p/2 + b_p) (+ a
    per-row overhead), where a unit is a whole row -- or, for a row whose
    work exceeds max_share of a rank's share, each of its chunks (seg
    entries from the row start, the library's segment_length).  A heavy row
    can so be split across ranks: every sharing rank computes its chunks'
    partial sums and the owner (chunk 0) sums all of them in chunk order --
    the association of a single-GPU run, so results stay bitwise identical.
    Every sharing rank samples the whole row (at c = 0.5 sampling a heavy
    row costs about as much as updating it), so only rows that alone exceed
    a rank's share are split by default, and rows above max_split_n entries
    (the sampler's giant path) never: measured with tools/shard_probe.py at
    8 ranks, splitting config 5's 261M-entry slice took its ranks from 8.4
    to 9.9 ms, and splitting every row above 1/4 of a share moved config 3
    from 1.46 to 1.54 ms but config 5 from 20.8 to 20.0 ms per sweep."""
    off = np.asarray(offsets, np.int64)
    n = np.diff(off).astype(np.float64)
    b = blocksizes(offsets, c).astype(np.float64)
    rows = len(n)
    row_work = np.where(b > 0, 0.5 * n + b + ROW_OVERHEAD, 1.0)
    share = row_work.sum() / max(world, 1)
    heavy = np.flatnonzero((row_work > max_share * share) & (n > seg) & (n <= max_split_n)) if world > 1 \
        else np.zeros(0, np.int64)
    # units in (row, chunk) order: (row, chunk or -1, work)
    units_row, units_chunk, units_work = [], [], []
    prev = 0
    for p in heavy.tolist():
        if p > prev:
            units_row.append(np.arange(prev, p))
            units_chunk.append(np.full(p - prev, -1))
            units_work.append(row_work[prev:p])
        ns = int((n[p] + seg - 1) // seg)
        lens = np.minimum(seg, n[p] - seg * np.arange(ns))
        units_row.append(np.full(ns, p))
        units_chunk.append(np.arange(ns))
        units_work.append(lens * (0.5 + b[p] / n[p]) + ROW_OVERHEAD / ns)
        prev = p + 1
    if prev < rows:
        units_row.append(np.arange(prev, rows))
        units_chunk.append(np.full(rows - prev, -1))
        units_work.append(row_work[prev:rows])
    ur = np.concatenate(units_row) if units_row else np.zeros(0, np.int64)
    uc = np.concatenate(units_chunk) if units_chunk else np.zeros(0, np.int64)
    uw = np.concatenate(units_work) if units_work else np.zeros(0)
    cum = np.concatenate([[0.0], np.cumsum(uw)])
    cuts = [0] + [int(np.searchsorted(cum, cum[-1] * k / world, side="left")) for k in range(1, world)] + [len(uw)]
    for i in range(1, len(cuts)):
        cuts[i] = min(max(cuts[i], cuts[i - 1]), len(uw))
    shards = []
    for k in range(world):
        u0, u1 = cuts[k], cuts[k + 1]
        parts, full = [], None
        i = u0
        while i < u1:
            p = int(ur[i])
            if uc[i] < 0:  # a run of whole rows
                j = i
                while j < u1 and uc[j] < 0:
                    j += 1
                full = (p, int(ur[j - 1]) + 1) if full is None else (full[0], int(ur[j - 1]) + 1)
                i = j
                continue
            j = i
            while j < u1 and ur[j] == p and uc[j] >= 0:
                j += 1
            cb, ce = int(uc[i]), int(uc[j - 1]) + 1
            ns = int((n[p] + seg - 1) // seg)
            if cb == 0 and ce == ns:  # the whole chunked row landed on this rank
                full = (p, p + 1) if full is None else (full[0], p + 1)
            else:
                parts.append((p, cb, ce))
            i = j
        # whole rows are contiguous; a shared row sits before or after them
        if full is None:
            first = parts[0][0] if parts else (int(ur[u0]) if u0 < len(ur) else rows)
            full = (first, first)
        o0, o1 = full
        for (p, cb, ce) in parts:
            if cb == 0:
                o1 = max(o1, p + 1) if o1 > o0 else p + 1
                o0 = min(o0, p) if o1 > o0 else p
        kr = [full[0], full[1]] if full[1] > full[0] else []
        for (p, _, _) in parts:
            kr += [p, p + 1]
        keep = (min(kr), max(kr)) if kr else (full[0], full[0])
        shards.append(Shard(full, parts, (o0, o1), keep))
    # owned ranges must tile [0, rows): rows nobody holds (empty tails) go to the next owner
    return shards


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
                 slab: bool = True, split: bool = True):

        import torch
        import torch.distributed as tdist
        self.ctx, self.cfg, self.rank, self.world, self.group = ctx, cfg, rank, world, group
        order, dims, _ = ctx.info()
        self.dims = dims
        # heavy rows split across ranks (chunks + an exchange of their partial
        # sums) need max_inner = 1; otherwise whole-row ranges
        self.split = split and cfg.max_inner == 1 and world > 1
        if self.split:
            self.shards = [partition_split(ctx.view_offsets(m), cfg.c, world, ctx.segment_length(m))
                           for m in range(order)]
        else:
            self.shards = [[Shard(r, [], r, r) for r in partition_rows(ctx.view_offsets(m), cfg.c, world)]
                           for m in range(order)]
        self.bounds = [[sh.owned for sh in self.shards[m]] for m in range(order)]
        if slab:  # this rank's rows only: ~1/N of every view stays on the device
            for m in range(order):
                ctx.view_keep_rows(m, *self.shards[m][rank].keep)
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
        # shared heavy rows: per mode, every rank's chunk ranges laid out in one
        # padded slot buffer (all-gathered), and the rows this rank finalises
        self.NE = None
        self._keep = []
        self.slots, self.gathered, self.layout = {}, {}, {}
        for m in range(order):
            per_rank = [[(p, cb, ce) for (p, cb, ce) in self.shards[m][k].parts] for k in range(world)]
            if not any(per_rank):
                continue
            if self.NE is None:
                Rk = ctx.get_factor(0)[0].shape[1]
                self.NE = Rk * Rk + Rk
            smax = max(sum(ce - cb for (_, cb, ce) in pr) for pr in per_rank)
            self.slots[m] = torch.zeros(smax * self.NE, dtype=torch.float32, device="cuda")
            self.gathered[m] = torch.zeros(world * smax * self.NE, dtype=torch.float32, device="cuda")
            self.layout[m] = (smax, per_rank)

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
        """This rank's part of the mode-m update of sweep k (its chunks of
        shared heavy rows first, then its whole rows), the exchange of the
        shared rows' partial sums and their finalisation by their owners,
        then the factor exchange."""
        import torch
        import torch.distributed as tdist
        from .ntc import sweep_stream
        state = sweep_stream(seed, k, m).state
        sh = self.shards[m][self.rank]
        self._keep = []
        if m in self.layout:
            smax, per_rank = self.layout[m]
            pos = 0
            for (p, cb, ce) in sh.parts:
                self.ctx.s_nmc_chunks_async(m, p, cb, ce, self.cfg, state,
                                            self.slots[m].data_ptr() + 4 * pos * self.NE)
                pos += ce - cb
        self.ctx.s_nmc_rows_async(m, sh.full[0], sh.full[1], self.cfg, state)
        if m in self.layout:
            smax, per_rank = self.layout[m]
            if self.nccl:
                tdist.all_gather_into_tensor(self.gathered[m], self.slots[m], group=self.group)
            else:  # gloo (CPU tests): through host copies once the chunks are done
                self.ctx.collect()
                host = [torch.empty(self.slots[m].numel(), dtype=torch.float32) for _ in range(self.world)]
                tdist.all_gather(host, self.slots[m].cpu(), group=self.group)
                self.gathered[m].copy_(torch.cat(host))
            g = self.gathered[m].view(self.world, smax, self.NE)
            for (p, cb, _) in sh.parts:
                if cb != 0:
                    continue
                pieces = []  # the row's chunks from every rank, in chunk order
                for kk in range(self.world):
                    q = 0
                    for (pp, cb2, ce2) in per_rank[kk]:
                        if pp == p:
                            pieces.append((cb2, g[kk, q: q + ce2 - cb2]))
                        q += ce2 - cb2
                pieces.sort(key=lambda x: x[0])
                allslots = torch.cat([x[1] for x in pieces]).contiguous()
                self._keep.append(allslots)  # alive until the stream has consumed it
                self.ctx.finalize_row_async(m, p, allslots.data_ptr(), allslots.shape[0], self.cfg)
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
        """Entries this rank's calls count for mode m: its whole rows plus the
        shared rows it owns (a shared row is counted once, by its owner)."""
        sh = self.shards[m][self.rank]
        off = self.ctx.view_offsets(m)
        n = int(blocksizes(off[sh.full[0]: sh.full[1] + 1], self.cfg.c).sum())
        for (p, cb, _) in sh.parts:
            if cb == 0:
                n += int(blocksizes(off[p: p + 2], self.cfg.c).sum())
        return n * self.cfg.max_inner
