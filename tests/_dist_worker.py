"""Worker for tests/test_dist_gloo.py: one rank of a row-sharded S_NMC sweep
on the CPU with gloo.  The per-rank row update is the C oracle on the rank's
row range (the checker stands in for the GPU kernel here); the partition and
the factor exchange are the product's own code (paper_2109_09534_b200.dist)."""
import os

import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def problem():
    import oracle as O
    orc = O.Oracle()
    rng = np.random.default_rng(42)
    dims = [37, 23, 29]
    nnz = 9000
    cells = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = rng.random(nnz) * 2.0
    ci, cv = orc.canonicalize(dims, idx, vals)
    views = [orc.build_view(dims, ci, cv, m) for m in range(3)]
    F = orc.initial_factors(dims, 4, 7)
    return orc, dims, views, F


def run_serial(sweeps, c):
    import oracle as O
    orc, dims, views, F = problem()
    M = [f.copy() for f in F]
    cfg = O.nmc_cfg(c=c, max_inner=2)
    for k in range(sweeps):
        for m in range(3):
            orc.s_nmc(dims, 4, F, M, m, views[m], None, cfg, orc.sweep_state(11, k, m))
    return F


def worker(rank, world, port, sweeps, c, out_dir):
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_2109_09534_b200.dist import allgather_rows, partition_rows
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc, dims, views, F = problem()
    M = [f.copy() for f in F]
    cfg = O.nmc_cfg(c=c, max_inner=2)
    bounds = [partition_rows(views[m][0], c, world) for m in range(3)]
    for k in range(sweeps):
        for m in range(3):
            r0, r1 = bounds[m][rank]
            orc.s_nmc(dims, 4, F, M, m, views[m], None, cfg, orc.sweep_state(11, k, m), r0, r1)
            allgather_rows(torch.from_numpy(F[m]), bounds[m], rank)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *F)
    dist.barrier()
    dist.destroy_process_group()
