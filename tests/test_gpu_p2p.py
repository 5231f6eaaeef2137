"""GPU: the fused exchange of row-sharded sweeps -- finalised rows stored by the
update kernel into the peer replicas (CUDA IPC) -- reproduces the
single-process sweep bit for bit on every rank.  Two processes on one GPU
(the box has one): the mapping, the kernel-side peer stores and the barrier
protocol are the multi-GPU ones; only the NVLink hop is missing."""
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
def test_fused_exchange_equals_serial(tmp_path, cuda_ok):
    import torch.multiprocessing as mp
    import _p2p_worker as W
    world = 2
    mp.spawn(W.worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    want = W.run_serial()
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        for m in range(3):
            np.testing.assert_array_equal(got[f"arr_{m}"], want[m])
