"""CPU: the multi-GPU work partition with heavy rows split across ranks
(paper_2109_09534_b200.dist.partition_split) -- every row and every chunk of a
shared row is assigned exactly once, the rows ranks finalise tile the mode in
order, a row's owner holds its chunk 0, and the work is balanced."""
import numpy as np
import pytest

from paper_2109_09534_b200.dist import blocksizes, partition_split


def _offsets(seed, rows=3000, heavy=(0, 1500, 2999), heavy_n=(400_000, 1_200_000, 90_000)):
    rng = np.random.default_rng(seed)
    n = rng.integers(0, 800, rows)
    for p, h in zip(heavy, heavy_n):
        n[p] = h
    return np.concatenate([[0], np.cumsum(n)]).astype(np.uint64)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seg", [2048, 16384])
def test_partition_split_covers_everything_once(world, seg):
    off = _offsets(world * 7 + seg)
    n = np.diff(off.astype(np.int64))
    rows = len(n)
    shards = partition_split(off, 0.5, world, seg, max_share=0.5)
    assert len(shards) == world
    row_hits = np.zeros(rows, np.int64)
    chunk_hits = {}
    for sh in shards:
        row_hits[sh.full[0]:sh.full[1]] += 1
        for (p, cb, ce) in sh.parts:
            ns = int((n[p] + seg - 1) // seg)
            assert 0 <= cb < ce <= ns and not (cb == 0 and ce == ns)
            for c in range(cb, ce):
                chunk_hits[(p, c)] = chunk_hits.get((p, c), 0) + 1
        k0, k1 = sh.keep
        assert k0 <= sh.full[0] and sh.full[1] <= k1 or sh.full[1] == sh.full[0]
        assert all(k0 <= p < k1 for (p, _, _) in sh.parts)
    shared = sorted({p for (p, _) in chunk_hits})
    for p in shared:
        ns = int((n[p] + seg - 1) // seg)
        assert all(chunk_hits.get((p, c), 0) == 1 for c in range(ns)), p
        assert row_hits[p] == 0
    assert all(row_hits[p] == 1 for p in range(rows) if p not in shared)
    # owned ranges tile [0, rows) in rank order; a shared row's owner holds chunk 0
    owned = [sh.owned for sh in shards]
    cur = 0
    for (o0, o1) in owned:
        if o1 > o0:
            assert o0 == cur
            cur = o1
    assert cur == rows
    for p in shared:
        owner = [r for r, sh in enumerate(shards) if any(pp == p and cb == 0 for (pp, cb, _) in sh.parts)]
        assert len(owner) == 1 and owned[owner[0]][0] <= p < owned[owner[0]][1]
    if world >= 3:  # the 1.2M-entry row is above one rank's share: it must be shared
        assert 1500 in shared


def test_partition_split_balances_work():
    off = _offsets(3)
    n = np.diff(off.astype(np.int64)).astype(float)
    b = blocksizes(off, 0.5).astype(float)
    world, seg = 8, 2048
    shards = partition_split(off, 0.5, world, seg, max_share=0.5)

    def work(sh):
        w = float((0.5 * n[sh.full[0]:sh.full[1]] + b[sh.full[0]:sh.full[1]]).sum())
        for (p, cb, ce) in sh.parts:
            e = min(n[p], ce * seg) - cb * seg
            w += e * (0.5 + b[p] / n[p])
        return w
    ws = [work(sh) for sh in shards]
    assert max(ws) / (sum(ws) / world) < 1.1, ws
