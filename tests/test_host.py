"""CPU: host-side logic of the package (reference-API mirror, config
validation, AO bookkeeping, RNG stream derivation, row partitioning) against
the reference's semantics (test_ao.cpp, test_nmc.cpp, test_rng.cpp)."""
import numpy as np
import pytest

import paper_2109_09534_b200 as P
from paper_2109_09534_b200 import dist
from paper_2109_09534_b200.ntc import MetricsRecord


def test_nmc_config_validation_messages():
    P.NmcConfig().validate()
    cases = [(dict(lambda_=0.0), "lambda must be > 0"), (dict(c=0.0), "c must be in"),
             (dict(c=1.5), "c must be in"), (dict(max_inner=-1), "max_inner must be >= 0"),
             (dict(power_iters=0), "power_iters"), (dict(power_tol=0.0), "power_tol"),
             (dict(threads=0), "threads must be >= 1"), (dict(chunk=-1), "chunk must be >= 0")]
    for kw, msg in cases:
        with pytest.raises(ValueError, match=msg):
            P.NmcConfig(**kw).validate()


def test_ao_config_validation():
    P.AoConfig().validate()
    for kw, msg in [(dict(rank=0), "rank must be positive"), (dict(max_epochs=-1.0), "max_epochs"),
                    (dict(term_tol=-1.0), "term_tol"), (dict(metrics_every=0), "metrics_every")]:
        with pytest.raises(ValueError, match=msg):
            P.AoConfig(**kw).validate()
    n = P.AoConfig(lambda_=0.5, c=0.25, max_inner=3).nmc()
    assert (n.lambda_, n.c, n.max_inner) == (0.5, 0.25, 3)


def test_epoch_fraction_and_term_cond():  # test_ao.cpp:68-108
    assert P.epoch_fraction(1000, 1000) == 1.0
    assert P.epoch_fraction(1500, 1000) == 1.5
    with pytest.raises(ValueError):
        P.epoch_fraction(1, 0)
    cfg = P.AoConfig(max_epochs=10.0, term_tol=1e-4)
    rec = lambda e, r: MetricsRecord(epoch=e, rel_error=r)  # noqa: E731
    with pytest.raises(ValueError):
        P.term_cond([], cfg)
    assert P.term_cond([rec(10.0, 0.9)], cfg)
    assert not P.term_cond([rec(9.0, 0.9)], cfg)
    h = [rec(1, 0.5), rec(2, 0.5), rec(3, 0.5)]
    assert not P.term_cond(h, cfg)
    h.append(rec(4, 0.5))
    assert P.term_cond(h, cfg)
    assert not P.term_cond(h, P.AoConfig(max_epochs=10.0, term_tol=0.0))
    assert not P.term_cond([rec(1, 0.5), rec(2, 0.5), rec(3, 0.4), rec(4, 0.4)], cfg)


def test_rng_streams_match_reference(golden):
    s = P.RngStream(42)
    np.testing.assert_array_equal(np.array([s.next_u64() for _ in range(8)], np.uint64),
                                  golden["rng_u64_42"])
    s = P.RngStream(7)
    np.testing.assert_array_equal(np.array([s.next_double() for _ in range(8)]), golden["rng_double_7"])
    got = [P.RngStream(42).fork(t).next_u64() for t in range(8)]
    np.testing.assert_array_equal(np.array(got, np.uint64), golden["rng_fork_first_42"])
    got = [P.sweep_stream(7, k, m).fork(l).fork(p).next_u64()
           for k in range(2) for m in range(3) for l in range(2) for p in range(4)]
    np.testing.assert_array_equal(np.array(got, np.uint64), golden["row_stream_first"])
    # fork leaves the parent untouched (test_rng.cpp)
    a = P.RngStream(7)
    a.fork(3)
    assert a.next_u64() == P.RngStream(7).next_u64()


def test_initial_factors_match_reference(golden):
    f = P.initial_factors([2, 2, 2], 2, 7)
    np.testing.assert_array_equal(np.concatenate([u.reshape(-1) for u in f.factors]),
                                  golden["init_factors_222_r2_s7"])
    assert f.factors[0][0].tolist() == [0.43977168304261183, 0.71485028822371077]
    g = P.initial_factors([4, 6, 3], 5, 42)
    assert all(np.all((u >= 0) & (u < 1)) for u in g.factors)
    np.testing.assert_array_equal(g.momentum[1], g.factors[1])


def test_blocksizes_floor_in_double(golden):
    for c, n, b in golden["blocksize"]:
        assert int(dist.blocksizes(np.array([0, int(n)], np.uint64), c)[0]) == int(b)


def test_partition_rows_is_contiguous_and_balanced():
    rng = np.random.default_rng(0)
    lens = rng.zipf(1.3, size=5000).clip(max=10**6)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    for world in (1, 2, 3, 8):
        b = dist.partition_rows(off, 0.5, world)
        assert b[0][0] == 0 and b[-1][1] == 5000
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert all(r0 <= r1 for r0, r1 in b)
    # uniform rows split evenly
    off = np.arange(0, 1001 * 10, 10, dtype=np.uint64)
    b = dist.partition_rows(off, 0.5, 4)
    sizes = [r1 - r0 for r0, r1 in b]
    assert max(sizes) - min(sizes) <= 1
