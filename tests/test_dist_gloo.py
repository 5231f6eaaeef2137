"""CPU, world_size 2 (gloo): the multi-GPU partition + factor all-gather
reproduces the single-process sweep bit for bit on every rank (the
GPU-count-invariance property that replaces the reference's thread-count
invariance, test_nmc.cpp:337-358)."""
import os
import socket

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("c", [0.5, 1.0])
def test_sharded_sweep_equals_serial(tmp_path, c):
    import torch.multiprocessing as mp
    import _dist_worker as W
    world, sweeps = 2, 2
    mp.spawn(W.worker, args=(world, _port(), sweeps, c, str(tmp_path)), nprocs=world, join=True)
    want = W.run_serial(sweeps, c)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        for m in range(3):
            np.testing.assert_array_equal(got[f"arr_{m}"], want[m])
