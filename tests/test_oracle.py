"""CPU: pins the C restatement (oracle/ntc_oracle.c) against the reference's
own outputs — the committed golden vectors (made from the compiled reference
by tests/golden/make_golden.py), the hand-derived KATs of the reference tests,
SURVEY.md Appendix A, and, where oracle/_ref is built, the live reference."""
import numpy as np
import pytest

import oracle as O


def test_rng_kats(orc, golden):
    # RngStream(42).next_u64() x3
    assert [hex(x) for x in orc.next_u64(42, 3)] == [
        "0xbdd732262feb6e95", "0x28efe333b266f103", "0x47526757130f9f52"]
    np.testing.assert_array_equal(orc.next_u64(42, 8), golden["rng_u64_42"])
    np.testing.assert_array_equal(orc.next_double(7, 8), golden["rng_double_7"])
    np.testing.assert_array_equal(orc.next_below(123, 40, 16), golden["rng_below_123_40"])
    np.testing.assert_array_equal(orc.next_below(5, 3, 16), golden["rng_below_5_3"])
    got = [orc.next_u64(orc.fork(42, t), 1)[0] for t in range(8)]
    np.testing.assert_array_equal(np.array(got, np.uint64), golden["rng_fork_first_42"])
    got = [orc.next_u64(orc.fork(orc.fork(orc.sweep_state(7, k, m), l), p), 1)[0]
           for k in range(2) for m in range(3) for l in range(2) for p in range(4)]
    np.testing.assert_array_equal(np.array(got, np.uint64), golden["row_stream_first"])
    # Appendix A: sweep_stream(7,0,0).fork(0).fork(5).next_u64()
    s = orc.fork(orc.fork(orc.sweep_state(7, 0, 0), 0), 5)
    assert hex(orc.next_u64(s, 1)[0]) == "0xb95273b52b2b8045"


def test_blocksize_floor_in_double(orc, golden):
    for c, n, b in golden["blocksize"]:
        assert orc.blocksize(c, int(n)) == int(b)


def test_sample_row_kats(orc, golden):
    # test_nmc.cpp:77-97 instance, Appendix A picks
    picks = orc.sample_row(40, 0.4, 42)
    np.testing.assert_array_equal(picks, golden["sample_1x40_c04_s42"])
    assert list(picks) == [29, 7, 12, 15, 5, 35, 13, 33, 18, 28, 16, 25, 26, 27, 31, 20]
    np.testing.assert_array_equal(orc.sample_row(40, 0.4, 43), golden["sample_1x40_c04_s43"])
    assert len(set(picks.tolist())) == 16
    # c = 1: slice order, no randomness (nmc.cpp:52-55)
    np.testing.assert_array_equal(orc.sample_row(5, 1.0, 1), np.arange(5))
    assert orc.sample_row(3, 0.3, 9).size == 0


def test_views_and_canonical_order(orc, golden):
    dims = golden["t1_dims"]
    ci, cv = orc.canonicalize(dims, golden["t1_idx"], golden["t1_vals"])
    np.testing.assert_array_equal(ci, golden["t1_canon_idx"])
    np.testing.assert_array_equal(cv, golden["t1_canon_vals"])
    for m in range(3):
        off, oth, val = orc.build_view(dims, ci, cv, m)
        np.testing.assert_array_equal(off, golden[f"t1_view{m}_off"])
        np.testing.assert_array_equal(oth, golden[f"t1_view{m}_oth"])
        np.testing.assert_array_equal(val, golden[f"t1_view{m}_val"])
    dims4 = golden["t4_dims"]
    ci, cv = orc.canonicalize(dims4, golden["t4_idx"], golden["t4_vals"])
    for m in range(4):
        off, oth, val = orc.build_view(dims4, ci, cv, m)
        np.testing.assert_array_equal(off, golden[f"t4_view{m}_off"])
        np.testing.assert_array_equal(oth, golden[f"t4_view{m}_oth"])


def test_picks_all_rows(orc, golden):
    dims = [int(d) for d in golden["t1_dims"]]
    for c in (0.5, 0.3, 0.05):
        for m in range(3):
            off = golden[f"t1_view{m}_off"]
            picks, offs = [], [0]
            for l in range(2):
                for p in range(dims[m]):
                    st = orc.fork(orc.fork(orc.sweep_state(11, 0, m), l), p)
                    pk = orc.sample_row(int(off[p + 1] - off[p]), c, st)
                    picks.append(pk)
                    offs.append(offs[-1] + len(pk))
            np.testing.assert_array_equal(np.concatenate(picks), golden[f"t1_picks_c{c}_m{m}"])
            np.testing.assert_array_equal(np.array(offs, np.uint64), golden[f"t1_pickoff_c{c}_m{m}"])


def _split(flat, dims, R):
    out, pos = [], 0
    for d in dims:
        out.append(flat[pos: pos + d * R].reshape(d, R).copy())
        pos += d * R
    return out


@pytest.mark.parametrize("tag,c,mi", [("c05_i2", 0.5, 2), ("c1_i1", 1.0, 1), ("c03_i3", 0.3, 3)])
def test_s_nmc_replay_bit_exact(orc, golden, tag, c, mi):
    dims = [int(d) for d in golden["t1_dims"]]
    R = 5
    views = [(golden[f"t1_view{m}_off"], golden[f"t1_view{m}_oth"], golden[f"t1_view{m}_val"])
             for m in range(3)]
    F = _split(golden["t1_init"], dims, R)
    M = [f.copy() for f in F]
    cfg = O.nmc_cfg(lambda_=1e-3, c=c, max_inner=mi, threads=3)
    want = golden[f"t1_snmc_{tag}"]
    accs, pos = [], 0
    for k in range(2):
        for m in range(3):
            accs.append(orc.s_nmc(dims, R, F, M, m, views[m], None, cfg, orc.sweep_state(11, k, m)))
            n = dims[m] * R
            np.testing.assert_array_equal(F[m].reshape(-1), want[pos: pos + n])
            np.testing.assert_array_equal(M[m].reshape(-1), want[pos + n: pos + 2 * n])
            pos += 2 * n
    np.testing.assert_array_equal(np.array(accs, np.uint64), golden[f"t1_snmc_{tag}_acc"])


def test_s_nmc_4way_bit_exact(orc, golden):
    dims = [int(d) for d in golden["t4_dims"]]
    ci, cv = orc.canonicalize(dims, golden["t4_idx"], golden["t4_vals"])
    views = [orc.build_view(dims, ci, cv, m) for m in range(4)]
    F = _split(golden["t4_init"], dims, 3)
    M = [f.copy() for f in F]
    cfg = O.nmc_cfg(lambda_=1e-2, c=0.6, max_inner=2)
    outs = []
    for k in range(2):
        for m in range(4):
            orc.s_nmc(dims, 3, F, M, m, views[m], None, cfg, orc.sweep_state(5, k, m))
            outs.append(F[m].reshape(-1).copy())
    np.testing.assert_array_equal(np.concatenate(outs), golden["t4_snmc"])


def test_metrics(orc, golden):
    dims = [int(d) for d in golden["t1_dims"]]
    F = _split(golden["t1_init"], dims, 5)
    sse, den, reg = orc.metrics(dims, 5, F, golden["t1_canon_idx"], golden["t1_canon_vals"])
    obj = 0.5 * sse + 0.5 * 1e-3 * reg
    rel = np.sqrt(sse) / np.sqrt(den)
    np.testing.assert_array_equal(np.array([obj, rel]), golden["t1_metrics_init"])


def test_hand_kats(orc, golden):
    # test_nmc.cpp:195-214 / 235-258
    assert orc.power_method(np.diag([3.0, 1.0]), 60, 1e-12) == golden["power_diag31"][0]
    assert abs(orc.power_method(np.diag([3.0, 1.0]), 60, 1e-12) - 3.0) < 1e-9
    for n in (1, 3, 7):
        assert abs(orc.power_method(0.75 * np.eye(n), 30, 1e-6) - 0.75) < 1e-13
    assert orc.power_method(np.zeros((3, 3)), 30, 1e-6) == 0.0
    with pytest.raises(ValueError, match="non-finite"):
        orc.power_method(np.array([[np.nan, 0], [0, 0.0]]))
    a_new, y_new, beta = orc.row_step([0.1, 0.4], [0.0, 0.0], [1.0, -1.0], 2.0, 0.5)
    np.testing.assert_array_equal(np.concatenate([a_new, y_new, [beta]]), golden["row_step_hand"])
    assert abs(beta - 1 / 3) < 1e-12 and abs(y_new[1] - 1.2) < 1e-12
    with pytest.raises(ValueError):
        orc.row_step([0.2], [0.0], [0.0], 0.5, 1.0)


def test_canonicalize_rejections(orc):
    with pytest.raises(ValueError, match="duplicate index \\(1,2,1\\)"):
        orc.canonicalize([2, 2, 2], [[0, 1, 0], [1, 1, 1], [0, 1, 0]], [1.0, 2.0, 3.0])
    with pytest.raises(ValueError, match="out of bounds at entry 1"):
        orc.canonicalize([2, 2], [[0, 1], [2, 0]], [1.0, 2.0])
    with pytest.raises(ValueError, match="negative value at entry 0"):
        orc.canonicalize([2, 2], [[0, 1]], [-1.0])
    with pytest.raises(ValueError, match="non-finite value at entry 0"):
        orc.canonicalize([2, 2], [[0, 1]], [np.inf])
    with pytest.raises(ValueError, match="order must be >= 2"):
        orc.canonicalize([3], [[0]], [1.0])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_restatement_matches_live_reference(orc):
    rng = np.random.default_rng(77)
    for trial in range(4):
        dims = [int(x) for x in rng.integers(3, 30, size=3)]
        nnz = int(np.prod(dims) * rng.uniform(0.1, 0.6))
        cells = rng.choice(int(np.prod(dims)), nnz, replace=False)
        idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
        vals = rng.random(nnz) * 2
        rp = O.RefProblem(dims, idx, vals)
        ci, cv = orc.canonicalize(dims, idx, vals)
        views = [orc.build_view(dims, ci, cv, m) for m in range(3)]
        for m in range(3):
            for a, b in zip(views[m], rp.view(m)):
                np.testing.assert_array_equal(a, b)
        R = int(rng.integers(1, 9))
        F = orc.initial_factors(dims, R, trial)
        rp.set_factors(R, F)
        M = [f.copy() for f in F]
        cfg = O.nmc_cfg(c=float(rng.uniform(0.05, 1.0)), max_inner=int(rng.integers(0, 4)), threads=2)
        for k in range(2):
            for m in range(3):
                st = orc.sweep_state(trial, k, m)
                a1 = rp.s_nmc(m, cfg, st)
                a2 = orc.s_nmc(dims, R, F, M, m, views[m], None, cfg, st)
                assert a1 == a2
                a, y = rp.get_factor(m)
                np.testing.assert_array_equal(a, F[m])
                np.testing.assert_array_equal(y, M[m])
        sse, den, reg = orc.metrics(dims, R, F, ci, cv)
        assert np.sqrt(sse) / np.sqrt(den) == rp.relative_error()
