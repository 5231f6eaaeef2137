"""Worker for tests/test_gpu_p2p.py: one rank of a row-sharded sweep with the
fused exchange (the update kernel stores every finalised row into the other
rank's factor replica through a CUDA IPC mapping).  Both ranks share GPU 0 --
each runs its own kernels, nothing inside a kernel waits for the other rank;
the barrier between modes is collect() + a gloo barrier."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SWEEPS, SEED = 3, 11
# uniform: short rows only; zipf: Zipf(1.2) modes with slices beyond the
# sampler's shared-memory budget (heavy grid path) split into many segments
# (slot groups), R = 16 (SHORT instantiation)
CASES = {
    "uniform": dict(dims=[300, 200, 100], nnz=200_000, R=8, synth=(4, 0.01, 4321, None, 0)),
    "zipf": dict(dims=[5000, 400, 60], nnz=400_000, R=16, synth=(6, 0.5, 77, [1.2, 1.2, 0.0], 1)),
    # order 4, rank 32: the NAT update (natural-layout gathers, shared tile)
    "nat4": dict(dims=[60, 50, 40, 30], nnz=120_000, R=32, synth=(8, 0.01, 99, None, 0)),
    # one mode-0 row holding 44 % of the entries: split across the ranks
    # (chunks + the all-gathered partial sums, finalised by the row's owner)
    "heavy": dict(dims=[40, 3000, 400], nnz=None, R=12, synth=None),
}


def heavy_tensor():
    rng = np.random.default_rng(4)
    dims = CASES["heavy"]["dims"]
    heavy = rng.choice(dims[1] * dims[2], 700_000, replace=False)
    rest = rng.choice((dims[0] - 1) * dims[1] * dims[2], 900_000, replace=False) + dims[1] * dims[2]
    cells = np.concatenate([heavy, rest])
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    return dims, idx, (rng.random(len(cells)) * 3).astype(np.float32)


def build(P, case="uniform"):
    c = CASES[case]
    ctx = P.Context(0)
    if c["synth"] is None:
        ctx.load(*heavy_tensor())
    else:
        tr, sigma, seed, zipf, kind = c["synth"]
        ctx.synth(c["dims"], c["nnz"], tr, sigma, seed, zipf, kind)
    ctx.random_factors(c["R"], 7)
    return ctx


def run_serial(case="uniform"):
    import paper_2109_09534_b200 as P
    ctx = build(P, case)
    cfg = P.NmcConfig(c=0.5)
    for k in range(SWEEPS):
        ctx.sweep_async(k, cfg, SEED)
    ctx.collect()
    return [ctx.get_factor(m)[0] for m in range(len(CASES[case]["dims"]))]


def worker(rank, world, port, out_dir, case="uniform"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import ShardedSweep
    ctx = build(P, case)
    sh = ShardedSweep(ctx, P.NmcConfig(c=0.5), rank, world, exchange="p2p")
    assert sh.exchange == "p2p", "peer mapping failed"
    for k in range(SWEEPS):
        sh.sweep(k, SEED)
    ctx.collect()
    dist.barrier()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *[ctx.get_factor(m)[0] for m in range(len(CASES[case]["dims"]))])
    dist.barrier()
    dist.destroy_process_group()
