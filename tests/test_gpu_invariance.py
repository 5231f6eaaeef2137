"""GPU-count invariance ("results must be identical for any GPU
count", the device analogue of the reference's thread/schedule invariance,
nmc.hpp:89-92 and test_nmc.cpp:337-358).

A row-sharded run of N ranks updates each rank's contiguous row range
(paper_2109_09534_b200.dist.partition_rows) with ntcb_s_nmc_rows_async.  Rows
are independent within a mode update, so the ranks' shares run one after the
other on ONE device compute exactly what N devices compute.  The full-range
ntcb_s_nmc and the 2-, 4- and 8-way shares must agree BITWISE (A and Y), at
the full BASELINE sizes of configs 2, 3 and 4 (rank 32: the NAT kernel), where a range-dependent
segmentation of long rows would re-associate the fp32 partial sums."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_CFG = {
    2: dict(dims=[10000, 10000, 10000], nnz=100_000_000, true_rank=20, sigma=0.01, R=20),
    3: dict(dims=[480189, 17770, 2182], nnz=100_000_000, true_rank=10, sigma=0.5, R=16,
            zipf=[1.2, 1.2, 0.0], kind=1),
    4: dict(dims=[50000, 50000, 1000, 100], nnz=500_000_000, true_rank=32, sigma=0.01, R=32),
}


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_sharded_rows_bitwise_equal_full_range(cuda_ok, cid):
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import partition_rows
    c = _CFG[cid]
    dims, R = c["dims"], c["R"]
    ctx = P.Context(0)
    ctx.synth(dims, c["nnz"], c["true_rank"], c["sigma"], 1000 + cid, c.get("zipf"), c.get("kind", 0))
    ctx.random_factors(R, 7)
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    for m in range(len(dims)):
        a0, _ = ctx.get_factor(m)
        state = P.sweep_stream(7, 0, m).state
        ctx.s_nmc(m, cfg, state)
        want_a, want_y = ctx.get_factor(m)
        off = ctx.view_offsets(m)
        for world in (2, 4, 8):
            ctx.set_factor(m, a=a0, y=a0)
            bounds = partition_rows(off, cfg.c, world)
            for r0, r1 in bounds:
                ctx.s_nmc_rows_async(m, r0, r1, cfg, state)
            ctx.collect()
            got_a, got_y = ctx.get_factor(m)
            bad = np.flatnonzero(np.any(got_a != want_a, axis=1) | np.any(got_y != want_y, axis=1))
            assert bad.size == 0, (cid, m, world, bad[:8], bounds)
        ctx.set_factor(m, a=want_a, y=want_y)
