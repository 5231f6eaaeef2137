"""GPU: the fused exchange of row-sharded sweeps -- finalised rows stored by the
update kernel into the peer replicas (CUDA IPC) -- reproduces the
single-process sweep bit for bit on every rank.  Two processes on one GPU
(the box has one): the mapping, the kernel-side peer stores and the barrier
protocol are the multi-GPU ones; only the NVLink hop is missing.  Cases: a
uniform tensor at 2 ranks, and a Zipf tensor (heavy slices, rows cut into
many segments and summed through slot groups, the SHORT kernel) at 2 and 3
ranks, an order-4 rank-32 tensor (the NAT update) at 2 ranks, and a tensor
whose heaviest row is split across 3 ranks (dist.partition_split)."""
import socket

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("uniform", 2), ("zipf", 2), ("zipf", 3), ("nat4", 2), ("heavy", 3)])
def test_fused_exchange_equals_serial(tmp_path, cuda_ok, case, world):
    import torch.multiprocessing as mp
    import _p2p_worker as W
    mp.spawn(W.worker, args=(world, _port(), str(tmp_path), case), nprocs=world, join=True)
    want = W.run_serial(case)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        for m in range(len(want)):
            np.testing.assert_array_equal(got[f"arr_{m}"], want[m])
