"""Slab storage for row-sharded multi-GPU runs (ntcb_view_keep_rows): each
rank keeps only its rows of every mode view.  Emulated on one GPU with one
context per rank (each holds ~1/N of the views), the ranks' row updates
followed by the factor exchange reproduce the single-context sweeps bit for
bit; whole-mode calls are refused on a slab; the per-rank metric partials
add up to the whole tensor's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = [48000, 9000, 700]  # config 3's shape at 1/10 scale: Zipf rows, heavy and split slices
NNZ, R = 12_000_000, 16


def _ctx(P):
    ctx = P.Context(0)
    ctx.synth(DIMS, NNZ, 10, 0.5, 1003, [1.2, 1.2, 0.0], 1)
    ctx.random_factors(R, 7)
    return ctx


@pytest.mark.parametrize("world", [2, 4])
def test_slab_ranks_reproduce_single_context(cuda_ok, world):
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import partition_rows
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    full = _ctx(P)
    full_bytes = [full.view_resident(m)[2] for m in range(3)]
    offs = [full.view_offsets(m) for m in range(3)]
    bounds = [partition_rows(offs[m], cfg.c, world) for m in range(3)]
    ranks = []
    for r in range(world):
        c = _ctx(P)
        for m in range(3):
            c.view_keep_rows(m, *bounds[m][r])
        ranks.append(c)
    # ~1/N of every view per rank (slabs balance work, not entries: allow 2x)
    for m in range(3):
        tot = sum(c.view_resident(m)[2] for c in ranks)
        assert tot <= full_bytes[m] * 1.05 + 4096 * world, (m, tot, full_bytes[m])
        for c in ranks:
            assert c.view_resident(m)[2] <= 2.0 * full_bytes[m] / world + (1 << 20)
    # whole-mode calls are refused on a slab
    with pytest.raises(IndexError, match="not resident"):
        ranks[0].s_nmc(0, cfg, 5)
    with pytest.raises(IndexError, match="not resident"):
        ranks[0].sweep_async(0, cfg, 7)
    for k in range(2):
        full.sweep_async(k, cfg, 7)
        full.collect()
        for m in range(3):
            st = P.sweep_stream(7, k, m).state
            for r, c in enumerate(ranks):
                c.s_nmc_rows_async(m, *bounds[m][r], cfg, st)
                c.collect()
            merged = ranks[0].get_factor(m)[0]
            for r, c in enumerate(ranks):
                r0, r1 = bounds[m][r]
                merged[r0:r1] = c.get_factor(m)[0][r0:r1]
            for c in ranks:  # the exchange (an NCCL all-gather / peer stores on real GPUs)
                c.set_factor(m, a=merged)
    for m in range(3):
        np.testing.assert_array_equal(ranks[0].get_factor(m)[0], full.get_factor(m)[0])
    sse, sx, _ = full.metrics()
    parts = np.array([c.metrics()[:2] for c in ranks]).sum(0)
    assert abs(parts[0] - sse) <= 1e-12 * sse and abs(parts[1] - sx) <= 1e-12 * sx
    for c in ranks:
        c.close()
    full.close()
