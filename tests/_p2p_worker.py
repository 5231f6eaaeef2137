"""Worker for tests/test_gpu_p2p.py: one rank of a row-sharded sweep with the
fused exchange (the update kernel stores every finalised row into the other
rank's factor replica through a CUDA IPC mapping).  Both ranks share GPU 0 --
each runs its own kernels, nothing inside a kernel waits for the other rank;
the barrier between modes is collect() + a gloo barrier."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DIMS, NNZ, R, SWEEPS, SEED = [300, 200, 100], 200_000, 8, 3, 11


def build(P):
    ctx = P.Context(0)
    ctx.synth(DIMS, NNZ, 4, 0.01, 4321)
    ctx.random_factors(R, 7)
    return ctx


def run_serial():
    import paper_2109_09534_b200 as P
    ctx = build(P)
    cfg = P.NmcConfig(c=0.5)
    for k in range(SWEEPS):
        ctx.sweep_async(k, cfg, SEED)
    ctx.collect()
    return [ctx.get_factor(m)[0] for m in range(3)]


def worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import ShardedSweep
    ctx = build(P)
    sh = ShardedSweep(ctx, P.NmcConfig(c=0.5), rank, world, exchange="p2p")
    assert sh.exchange == "p2p", "peer mapping failed"
    for k in range(SWEEPS):
        sh.sweep(k, SEED)
    ctx.collect()
    dist.barrier()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *[ctx.get_factor(m)[0] for m in range(3)])
    dist.barrier()
    dist.destroy_process_group()
