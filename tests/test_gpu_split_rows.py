"""Heavy rows split across ranks (dist.partition_split): a row larger than
half a rank's share is cut into its chunks, every sharing rank computes its
chunks' partial sums (ntcb_s_nmc_chunks_async), the owner gathers them in
chunk order and finalises the row (ntcb_finalize_row_async).  Emulated on one
GPU with one slab context per rank and the exchanges done by copies, the
sweeps reproduce a single context bit for bit, entry counts included."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tensor():
    rng = np.random.default_rng(4)
    dims = [40, 3000, 400]
    heavy = rng.choice(dims[1] * dims[2], 700_000, replace=False)      # row 0 of mode 0: 700K entries
    rest = rng.choice((dims[0] - 1) * dims[1] * dims[2], 900_000, replace=False) + dims[1] * dims[2]
    cells = np.concatenate([heavy, rest])
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = (rng.random(len(cells)) * 3).astype(np.float32)
    return dims, idx, vals


@pytest.mark.parametrize("world", [2, 3, 4])
def test_split_heavy_rows_bitwise(cuda_ok, world):
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import partition_split
    dims, idx, vals = _tensor()
    R = 12
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)

    def make():
        c = P.Context(0)
        c.load(dims, idx, vals)
        c.random_factors(R, 7)
        return c

    full = make()
    shards = [partition_split(full.view_offsets(m), cfg.c, world, full.segment_length(m)) for m in range(3)]
    if world >= 3:  # row 0 of mode 0 (44 % of the entries) exceeds a rank's share
        assert any(sh.parts for sh in shards[0]), "the heavy row of mode 0 must be split"
    ranks = [make() for _ in range(world)]
    for m in range(3):
        for r, c in enumerate(ranks):
            c.view_keep_rows(m, *shards[m][r].keep)
    NE = R * R + R
    total = 0
    for k in range(2):
        full.sweep_async(k, cfg, 7)
        total += full.collect()
        for m in range(3):
            st = P.sweep_stream(7, k, m).state
            slots = {}
            for r, c in enumerate(ranks):
                sh = shards[m][r]
                for (p, cb, ce) in sh.parts:
                    buf = torch.zeros((ce - cb) * NE, dtype=torch.float32, device="cuda")
                    c.s_nmc_chunks_async(m, p, cb, ce, cfg, st, buf.data_ptr())
                    slots[(p, cb)] = buf
                c.s_nmc_rows_async(m, sh.full[0], sh.full[1], cfg, st)
                c.collect()
            got = 0
            for r, c in enumerate(ranks):
                for (p, cb, _) in shards[m][r].parts:
                    if cb:
                        continue
                    allslots = torch.cat([slots[key] for key in sorted(x for x in slots if x[0] == p)])
                    c.finalize_row_async(m, p, allslots.data_ptr(), allslots.numel() // NE, cfg)
                got += c.collect()
            merged = ranks[0].get_factor(m)[0]
            for r, c in enumerate(ranks):
                o0, o1 = shards[m][r].owned
                merged[o0:o1] = c.get_factor(m)[0][o0:o1]
            for c in ranks:
                c.set_factor(m, a=merged)
            want = full.get_factor(m)[0]
            bad = np.flatnonzero(np.any(merged != want, axis=1))
            assert bad.size == 0, (world, k, m, bad[:8])
    for c in ranks:
        c.close()
    full.close()
