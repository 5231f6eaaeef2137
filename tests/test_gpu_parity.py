"""GPU parity: the CUDA path (through the C-ABI, libntcb.so) against the
reference's own outputs (golden vectors made from the compiled reference) and
the bit-exact C restatement (oracle/), on identical seeded inputs.

Bars (BASELINE.json north_star):
  * sampled index sets / picks and the nonzero permutation: bit-exact;
  * entries_accessed, epochs: exact;
  * factors (fp32 device vs fp64 reference): relative Frobenius error
    <= TOL = 1e-4 per mode update / per AO iteration; metrics <= 1e-5.
"""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4


def rel(a, b):
    """Relative error of a factor: the larger of the Frobenius ratio and the
    worst per-row ratio ||a_p - b_p|| / max(||b_p||, floor), so an error
    confined to a few rows of a 10^4..4.8*10^6-row factor cannot hide under
    the whole-matrix norm.  floor = 1e-3 x the RMS row norm keeps rows the
    projection drove to ~0 from dividing by ~0 (their absolute error is
    still bounded by 1e-7 x the typical row)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    fro = np.linalg.norm(a - b) / (den if den > 0 else 1.0)
    if a.ndim != 2 or b.shape[0] == 0:
        return fro
    return max(fro, row_rel(a, b))


def row_rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rn = np.linalg.norm(b, axis=1)
    rms = float(np.sqrt(np.mean(rn * rn))) if rn.size else 0.0
    floor = max(1e-3 * rms, 1e-300)
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.maximum(rn, floor)))


def _split(flat, dims, R):
    out, pos = [], 0
    for d in dims:
        out.append(flat[pos: pos + d * R].reshape(d, R).copy())
        pos += d * R
    return out


@pytest.fixture(scope="module")
def ntc(cuda_ok):
    import paper_2109_09534_b200 as P
    return P


def ctx_for(ntc, dims, idx, vals):
    c = ntc.Context(0)
    c.load(dims, idx, vals)
    return c


# ---------------------------------------------------------------- tensor / views
def test_views_bit_exact(ntc, golden):
    for t, N in (("t1", 3), ("t4", 4)):
        dims = [int(d) for d in golden[f"{t}_dims"]]
        c = ctx_for(ntc, dims, golden[f"{t}_idx"], golden[f"{t}_vals"])
        for m in range(N):
            off, oth, val = c.view(m)
            np.testing.assert_array_equal(off, golden[f"{t}_view{m}_off"])
            np.testing.assert_array_equal(oth, golden[f"{t}_view{m}_oth"])
            np.testing.assert_array_equal(val, golden[f"{t}_view{m}_val"].astype(np.float32))
    c = ctx_for(ntc, [int(d) for d in golden["t1_dims"]], golden["t1_idx"], golden["t1_vals"])
    ci, cv = c.canonical()
    np.testing.assert_array_equal(ci, golden["t1_canon_idx"])
    np.testing.assert_array_equal(cv, golden["t1_canon_vals"].astype(np.float32))


def test_views_bit_exact_large(ntc, orc):
    rng = np.random.default_rng(5)
    dims = [300, 257, 1000]
    nnz = 400_000
    cells = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = rng.random(nnz).astype(np.float32)
    c = ctx_for(ntc, dims, idx, vals)
    ci, cv = orc.canonicalize(dims, idx, vals.astype(np.float64))
    gi, gv = c.canonical()
    np.testing.assert_array_equal(gi, ci)
    for m in range(3):
        off, oth, val = orc.build_view(dims, ci, cv, m)
        goff, goth, gval = c.view(m)
        np.testing.assert_array_equal(goff, off)
        np.testing.assert_array_equal(goth, oth)
        np.testing.assert_array_equal(gval, val.astype(np.float32))


def test_tensor_rejections_match_reference(ntc):
    c = ntc.Context(0)
    cases = [
        ([2, 2, 2], [[0, 1, 0], [1, 1, 1], [0, 1, 0]], [1.0, 2.0, 3.0],
         "SparseTensor: duplicate index (1,2,1)"),
        ([2, 2], [[0, 1], [2, 0]], [1.0, 2.0], "SparseTensor: index out of bounds at entry 1"),
        ([2, 2], [[0, 1], [1, 1]], [1.0, -2.0], "SparseTensor: negative value at entry 1"),
        ([2, 2], [[0, 1]], [np.nan], "SparseTensor: non-finite value at entry 0"),
        ([3], [[0]], [1.0], "SparseTensor: order must be >= 2"),
        ([3, 0], [[0, 0]], [1.0], "SparseTensor: dimensions must be positive"),
    ]
    for dims, idx, vals, msg in cases:
        with pytest.raises(ValueError) as e:
            c.load(dims, np.array(idx, np.uint32), np.array(vals, np.float64))
        assert str(e.value) == msg
        if O.ref_available():
            with pytest.raises(ValueError) as e2:
                O.RefProblem(dims, np.array(idx, np.uint32), np.array(vals, np.float64))
            assert str(e2.value) == msg


# ---------------------------------------------------------------- sampling
def test_sample_row_kat(ntc, golden):
    idx = np.array([[0, j] for j in range(40)], np.uint32)
    t = ntc.SparseTensor([1, 40], idx, np.ones(40))
    got = ntc.sample_row(t, 0, 0, 0.4, ntc.RngStream(42))
    np.testing.assert_array_equal(got, golden["sample_1x40_c04_s42"])
    assert list(got) == [29, 7, 12, 15, 5, 35, 13, 33, 18, 28, 16, 25, 26, 27, 31, 20]
    np.testing.assert_array_equal(ntc.sample_row(t, 0, 0, 0.4, ntc.RngStream(43)),
                                  golden["sample_1x40_c04_s43"])
    np.testing.assert_array_equal(ntc.sample_row(t, 0, 0, 1.0, ntc.RngStream(1)), np.arange(40))
    with pytest.raises(IndexError):
        ntc.sample_row(t, 0, 7, 0.5, ntc.RngStream(1))
    with pytest.raises(ValueError):
        ntc.sample_row(t, 0, 0, 0.0, ntc.RngStream(1))


def test_sampler_all_rows_bit_exact(ntc, golden, orc):
    dims = [int(d) for d in golden["t1_dims"]]
    c = ctx_for(ntc, dims, golden["t1_idx"], golden["t1_vals"])
    for cf in (0.5, 0.3, 0.05):
        for m in range(3):
            picks, offs = [], [0]
            for l in range(2):
                po, pk = c.sample_rows(m, cf, orc.sweep_state(11, 0, m), l)
                picks.append(pk)
                offs.extend((offs[-1] + po[1:]).tolist())
            np.testing.assert_array_equal(np.concatenate(picks), golden[f"t1_picks_c{cf}_m{m}"])
            np.testing.assert_array_equal(np.array(offs, np.uint64), golden[f"t1_pickoff_c{cf}_m{m}"])


@pytest.mark.parametrize("slice_len", [37, 1000, 23000, 70000])
def test_sampler_long_slices_bit_exact(ntc, orc, slice_len):
    """Slices in shared memory (u16/u32 perm) and beyond it (global scratch)."""
    rows = 6
    dims = [rows, slice_len]
    idx = np.array([[p, j] for p in range(rows) for j in range(slice_len)], np.uint32)
    keep = np.random.default_rng(slice_len).random(len(idx)) < 0.9
    idx = idx[keep]
    vals = np.ones(len(idx), np.float32)
    c = ctx_for(ntc, dims, idx, vals)
    off = c.view(0)[0]
    for cf in (0.5, 0.97, 0.013):
        st = 0x1234 + slice_len
        po, pk = c.sample_rows(0, cf, st, 1)
        for p in range(rows):
            want = orc.sample_row(int(off[p + 1] - off[p]), cf, orc.fork(orc.fork(st, 1), p))
            np.testing.assert_array_equal(pk[po[p]:po[p + 1]], want)


# ---------------------------------------------------------------- s_nmc
@pytest.mark.parametrize("tag,c,mi", [("c05_i2", 0.5, 2), ("c1_i1", 1.0, 1), ("c03_i3", 0.3, 3)])
def test_s_nmc_matches_reference(ntc, golden, orc, tag, c, mi):
    dims = [int(d) for d in golden["t1_dims"]]
    R = 5
    ctx = ctx_for(ntc, dims, golden["t1_idx"], golden["t1_vals"])
    ctx.set_factors(R, _split(golden["t1_init"], dims, R))
    cfg = ntc.NmcConfig(lambda_=1e-3, c=c, max_inner=mi)
    want = golden[f"t1_snmc_{tag}"]
    pos, accs = 0, []
    worst = 0.0
    for k in range(2):
        for m in range(3):
            # teacher forcing: start every mode update from the reference's state
            accs.append(ctx.s_nmc(m, cfg, orc.sweep_state(11, k, m)))
            a, y = ctx.get_factor(m)
            n = dims[m] * R
            wa, wy = want[pos: pos + n].reshape(dims[m], R), want[pos + n: pos + 2 * n].reshape(dims[m], R)
            worst = max(worst, rel(a, wa), rel(y, wy))
            assert rel(a, wa) <= TOL and rel(y, wy) <= TOL, (k, m, rel(a, wa), rel(y, wy))
            assert np.all(a >= 0)
            ctx.set_factor(m, wa, wy)
            pos += 2 * n
    np.testing.assert_array_equal(np.array(accs, np.uint64), golden[f"t1_snmc_{tag}_acc"])
    print(f"max rel err {tag}: {worst:.3e}")


def test_s_nmc_4way(ntc, golden):
    dims = [int(d) for d in golden["t4_dims"]]
    ctx = ctx_for(ntc, dims, golden["t4_idx"], golden["t4_vals"])
    ctx.set_factors(3, _split(golden["t4_init"], dims, 3))
    cfg = ntc.NmcConfig(lambda_=1e-2, c=0.6, max_inner=2)
    want = golden["t4_snmc"]
    pos = 0
    for k in range(2):
        for m in range(4):
            ctx.s_nmc(m, cfg, O.Oracle().sweep_state(5, k, m))
            a, _ = ctx.get_factor(m)
            w = want[pos: pos + dims[m] * 3].reshape(dims[m], 3)
            assert rel(a, w) <= TOL
            ctx.set_factor(m, w)
            pos += dims[m] * 3


def test_s_nmc_reference_api(ntc, golden, orc):
    """ntc.s_nmc(tensor, factors, mode, a_init, cfg, rng, stats) like nmc.hpp:93-95."""
    dims = [int(d) for d in golden["t1_dims"]]
    t = ntc.SparseTensor(dims, golden["t1_idx"], golden["t1_vals"])
    f = ntc.FactorSet(5, _split(golden["t1_init"], dims, 5), _split(golden["t1_init"], dims, 5))
    st = ntc.SnmcStats()
    cfg = ntc.NmcConfig(c=0.5, max_inner=2)
    out = ntc.s_nmc(t, f, 0, f.factors[0], cfg, ntc.sweep_stream(11, 0, 0), st)
    want = golden["t1_snmc_c05_i2"][: dims[0] * 5].reshape(dims[0], 5)
    assert rel(out, want) <= TOL
    assert st.entries_accessed == golden["t1_snmc_c05_i2_acc"][0]
    ntc.s_nmc(t, f, 0, f.factors[0], cfg, ntc.sweep_stream(11, 0, 0), st)
    assert st.entries_accessed == 2 * golden["t1_snmc_c05_i2_acc"][0]  # += (nmc.cpp:270)
    with pytest.raises(ValueError, match="a_init must be nonnegative"):
        bad = f.factors[0].copy()
        bad[0, 0] = -0.1
        ntc.s_nmc(t, f, 0, bad, cfg, ntc.RngStream(6))
    with pytest.raises(ValueError, match="a_init shape mismatch"):
        ntc.s_nmc(t, f, 0, np.zeros((2, 2)), cfg, ntc.RngStream(6))
    with pytest.raises(ValueError, match="mode out of range"):
        ntc.s_nmc(t, f, 5, f.factors[0], cfg, ntc.RngStream(6))
    with pytest.raises(ValueError, match="lambda must be > 0"):
        ntc.s_nmc(t, f, 0, f.factors[0], ntc.NmcConfig(lambda_=0.0), ntc.RngStream(6))


def test_s_nmc_edge_cases(ntc):
    # max_inner = 0 -> a_init unchanged, nothing accessed (test_nmc.cpp:279-302)
    rng = np.random.default_rng(3)
    dims = [4, 3, 3]
    cells = rng.choice(36, 18, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    t = ntc.SparseTensor(dims, idx, rng.random(18))
    f = ntc.FactorSet.random_uniform(dims, 2, ntc.RngStream(2))
    a0 = f.factors[0].astype(np.float32).astype(np.float64)
    f.factors[0] = a0.copy()
    st = ntc.SnmcStats()
    out = ntc.s_nmc(t, f, 0, a0, ntc.NmcConfig(max_inner=0), ntc.RngStream(1), st)
    np.testing.assert_array_equal(out, a0)
    assert st.entries_accessed == 0
    # empty tensor: every row skipped
    te = ntc.SparseTensor([4, 3, 3], np.zeros((0, 3), np.uint32), np.zeros(0))
    fe = ntc.FactorSet.random_uniform([4, 3, 3], 2, ntc.RngStream(2))
    fe.factors = [u.astype(np.float32).astype(np.float64) for u in fe.factors]
    init2 = fe.factors[1].copy()
    st = ntc.SnmcStats()
    out = ntc.s_nmc(te, fe, 1, init2, ntc.NmcConfig(max_inner=5), ntc.RngStream(3), st)
    np.testing.assert_array_equal(out, init2)
    np.testing.assert_array_equal(fe.momentum[1], init2)
    assert st.entries_accessed == 0
    # skip rows whose blocksize floors to zero (test_nmc.cpp:304-319)
    t2 = ntc.SparseTensor([2, 6], np.array([[0, 0], [0, 1], [0, 2], [0, 3], [1, 5]], np.uint32),
                          np.array([1, 2, 3, 4, 5.0]))
    f2 = ntc.FactorSet.random_uniform([2, 6], 2, ntc.RngStream(9))
    f2.factors = [u.astype(np.float32).astype(np.float64) for u in f2.factors]
    a_init = f2.factors[0].copy()
    st = ntc.SnmcStats()
    out = ntc.s_nmc(t2, f2, 0, a_init, ntc.NmcConfig(c=0.3), ntc.RngStream(4), st)
    assert st.entries_accessed == 1
    np.testing.assert_array_equal(out[1], a_init[1])
    np.testing.assert_array_equal(f2.momentum[0][1], a_init[1])
    assert out[0, 0] != a_init[0, 0]


def test_host_buffers_pinned_equals_pageable(ntc):
    """ntcb_s_nmc_host on page-locked buffers (device-side fp64 <-> fp32
    conversion and nonnegativity check, direct copies) returns exactly what
    the pageable path (host conversion through staging) returns, and rejects
    a negative a_init leaving A and Y untouched."""
    import paper_2109_09534_b200 as P
    dims, R = [3000, 400, 50], 12
    ctx = P.Context(0)
    ctx.synth(dims, 1_000_000, 4, 0.01, 17)
    ctx.random_factors(R, 3)
    cfg = P.NmcConfig(c=0.5)
    a0 = ctx.get_factor(0)[0]
    outs = {}
    for kind in ("pageable", "pinned"):
        ctx.random_factors(R, 3)
        mk = (lambda x: np.array(x)) if kind == "pageable" else P.pinned_like
        ai, ao, yo = mk(a0), mk(np.zeros_like(a0)), mk(np.zeros_like(a0))
        n = ctx.s_nmc_host(0, ai, ao, yo, cfg, 4242)
        outs[kind] = (n, np.array(ao), np.array(yo))
        np.testing.assert_array_equal(ao, ctx.get_factor(0)[0])
        np.testing.assert_array_equal(yo, ctx.get_factor(0)[1])
    assert outs["pinned"][0] == outs["pageable"][0]
    np.testing.assert_array_equal(outs["pinned"][1], outs["pageable"][1])
    np.testing.assert_array_equal(outs["pinned"][2], outs["pageable"][2])
    before = ctx.get_factor(0)
    bad = P.pinned_like(a0)
    bad[1234, 5] = -0.5
    with pytest.raises(ValueError, match="a_init must be nonnegative"):
        ctx.s_nmc_host(0, bad, P.pinned_like(np.zeros_like(a0)), P.pinned_like(np.zeros_like(a0)), cfg, 4243)
    after = ctx.get_factor(0)
    np.testing.assert_array_equal(before[0], after[0])
    np.testing.assert_array_equal(before[1], after[1])
    ctx.s_nmc(1, cfg, 99)  # the context works normally afterwards


def test_sample_prefetch_changes_nothing(ntc):
    """ntcb_sample_prefetch (the sampled set of a future call drawn ahead on
    the sampler stream) is consumed by the matching s_nmc / s_nmc_host call
    and ignored otherwise; factors, momentum and counts are bitwise those of
    calls without it."""
    import paper_2109_09534_b200 as P
    dims, R = [3000, 400, 50], 12
    ctx = P.Context(0)
    ctx.synth(dims, 1_000_000, 4, 0.01, 17)
    cfg = P.NmcConfig(c=0.5)
    st = [P.sweep_stream(11, 0, m).state for m in range(3)]

    def run(prefetch):
        ctx.random_factors(R, 3)
        out = []
        a0 = [P.pinned_like(ctx.get_factor(m)[0]) for m in range(3)]
        ao = [P.pinned_like(np.zeros_like(a)) for a in a0]
        yo = [P.pinned_like(np.zeros_like(a)) for a in a0]
        if prefetch == "match":
            ctx.sample_prefetch(0, cfg, st[0])
        for m in range(3):
            if prefetch == "match" and m + 1 < 3:
                ctx.sample_prefetch(m + 1, cfg, st[m + 1])  # drawn while mode m updates
            if prefetch == "stale":
                ctx.sample_prefetch(m, cfg, st[m] ^ 1)      # another stream: must be ignored
            if prefetch == "clobbered":
                ctx.sample_prefetch(m, cfg, st[m])
                ctx.sample_mask(m, 0.5, 77)                  # other sampling of the mode discards it
            n = ctx.s_nmc_host(m, a0[m], ao[m], yo[m], cfg, st[m])
            out.append((n, np.array(ao[m]), np.array(yo[m])))
        n_dev = ctx.s_nmc(1, cfg, st[1]) if prefetch != "match" else (ctx.sample_prefetch(1, cfg, st[1]), ctx.s_nmc(1, cfg, st[1]))[1]
        out.append((n_dev, *ctx.get_factor(1)))
        return out

    base = run(None)
    for kind in ("match", "stale", "clobbered"):
        got = run(kind)
        for (n0, a, y), (n1, a1, y1) in zip(base, got):
            assert n0 == n1
            np.testing.assert_array_equal(a, a1)
            np.testing.assert_array_equal(y, y1)


def test_collect_counts_survive_internal_drains(ntc):
    """ntcb_collect returns the entries of every async sweep queued since the
    last collect, even when other calls (metrics, a blocking s_nmc, sampling)
    synchronised the context in between (include/ntc_b200.h ntcb_collect)."""
    import paper_2109_09534_b200 as P
    ctx = P.Context(0)
    ctx.synth_uniform([50, 40, 30], 20000, 3, 0.01, 5)
    ctx.random_factors(4, 7)
    cfg = P.NmcConfig(c=0.5)
    want = sum(int(np.floor(0.5 * np.diff(ctx.view_offsets(m))).sum()) for m in range(3))
    ctx.sweep_async(0, cfg, 7)
    ctx.metrics()
    ctx.sample_rows(1, 0.5, P.sweep_stream(7, 3, 1).state)
    own = ctx.s_nmc(2, cfg, P.sweep_stream(7, 9, 2).state)  # its own count, not the pending one
    assert own == int(np.floor(0.5 * np.diff(ctx.view_offsets(2))).sum())
    ctx.sweep_async(1, cfg, 7)
    assert ctx.collect() == 2 * want
    assert ctx.collect() == 0


def test_s_nmc_nonfinite_diagnostic(ntc):
    dims = [3, 4, 2]
    idx = np.array([[i, j, k] for i in range(3) for j in range(4) for k in range(2)], np.uint32)
    t = ntc.SparseTensor(dims, idx, np.ones(len(idx)))
    f = ntc.FactorSet.random_uniform(dims, 2, ntc.RngStream(1))
    f.factors = [u.astype(np.float32).astype(np.float64) for u in f.factors]
    f.factors[1][2, :] = 1e200  # k = inf (in fp64 too): non-finite gradient on every row
    f.factors[2][:, :] = 1e200
    with pytest.raises(RuntimeError, match=r"s_nmc: non-finite gradient at row 1 \(mode 1\)"):
        ntc.s_nmc(t, f, 0, f.factors[0], ntc.NmcConfig(), ntc.RngStream(1))


def test_c1_seed_independence_and_determinism(ntc):
    import paper_2109_09534_b200 as P
    ctx = P.Context(0)
    ctx.synth_uniform([60, 50, 40], 30000, 4, 0.01, 77)
    ctx.random_factors(6, 7)
    a0 = [ctx.get_factor(m)[0] for m in range(3)]

    def run(seed, c):
        for m in range(3):
            ctx.set_factor(m, a0[m], a0[m])
        for k in range(3):
            ctx.sweep_async(k, P.NmcConfig(c=c, max_inner=2), seed)
        ctx.collect()
        return [ctx.get_factor(m)[0] for m in range(3)]

    r1, r2 = run(1, 1.0), run(999, 1.0)
    for a, b in zip(r1, r2):
        np.testing.assert_array_equal(a, b)
    s1, s2, s3 = run(5, 0.5), run(5, 0.5), run(6, 0.5)
    for a, b in zip(s1, s2):
        np.testing.assert_array_equal(a, b)  # bitwise deterministic
    assert any(not np.array_equal(a, b) for a, b in zip(s1, s3))
    assert all(np.all(a >= 0) for a in s1)


# ---------------------------------------------------------------- AO driver + metrics
def test_metrics_match_reference(ntc, golden):
    dims = [int(d) for d in golden["t1_dims"]]
    t = ntc.SparseTensor(dims, golden["t1_idx"], golden["t1_vals"])
    f = ntc.FactorSet(5, _split(golden["t1_init"], dims, 5), _split(golden["t1_init"], dims, 5))
    obj, rl = golden["t1_metrics_init"]
    assert abs(ntc.objective(t, f, 1e-3) - obj) <= 1e-9 * abs(obj)
    assert abs(ntc.relative_error(t, f) - rl) <= 1e-9 * abs(rl)


def test_ao_ntc_matches_reference(ntc, golden):
    dims = [int(d) for d in golden["t2_dims"]]
    t = ntc.SparseTensor(dims, golden["t2_idx"], golden["t2_vals"])
    init = ntc.FactorSet(3, _split(golden["t2_init"], dims, 3), _split(golden["t2_init"], dims, 3))
    seen = []
    res = ntc.ao_ntc(t, init, ntc.AoConfig(rank=3, c=0.5, max_epochs=6.0, seed=11),
                     lambda r, f: seen.append((r.epoch, f.all_nonnegative())))
    h = golden["t2_ao_hist"]
    assert len(res.history) == len(h) == len(seen)
    for r, w in zip(res.history, h):
        assert r.epoch == w[0] and r.entries_accessed == int(w[4])
        assert abs(r.objective - w[1]) <= TOL * abs(w[1])
        assert abs(r.rel_error - w[2]) <= TOL * abs(w[2])
    want = _split(golden["t2_ao_factors"], dims, 3)
    for a, b in zip(res.factors.factors, want):
        assert rel(a, b) <= TOL
    # metrics_every thins records, final state kept (test_ao.cpp:215-233)
    res2 = ntc.ao_ntc(t, init, ntc.AoConfig(rank=3, c=1.0, max_epochs=15.0, seed=3, metrics_every=2))
    assert [r.epoch for r in res2.history] == list(golden["t2_ao_every2_hist"][:, 0])
    for a, b in zip(res2.factors.factors, _split(golden["t2_ao_every2_factors"], dims, 3)):
        assert rel(a, b) <= TOL


def test_ao_zero_progress_and_budget(ntc):
    t = ntc.SparseTensor([3, 3, 3], np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2]], np.uint32),
                         np.array([1.0, 2.0, 3.0]))
    init = ntc.initial_factors([3, 3, 3], 2, 7)
    init.factors = [u.astype(np.float32).astype(np.float64) for u in init.factors]
    res = ntc.ao_ntc(t, init, ntc.AoConfig(rank=2, c=0.5, max_epochs=100.0))
    assert len(res.history) == 1 and res.history[0].epoch == 0.0
    np.testing.assert_array_equal(res.factors.factors[0], init.factors[0])
    res = ntc.ao_ntc(t, init, ntc.AoConfig(rank=2, max_epochs=0.0))
    assert len(res.history) == 1


def test_ao_ntc_deferred_sync_records(ntc):
    """ntcb_ao_ntc without metrics or observer enqueues its sweeps back to
    back (one synchronisation at the end): the history still has one record
    per metrics_every sweeps with exact entry counts and increasing wall
    times, and the factors equal the same sweeps queued one by one."""
    import paper_2109_09534_b200 as P
    ctx = P.Context(0)
    ctx.synth_uniform([300, 200, 100], 400_000, 5, 0.01, 21)
    ctx.random_factors(6, 7)
    per = sum(int(np.floor(0.5 * np.diff(ctx.view_offsets(m).astype(np.float64))).sum()) for m in range(3))
    cfg = P.AoConfig(rank=6, c=0.5, max_epochs=per * 7 / ctx.info()[2] - 1e-9, seed=11, eval_metrics=False,
                     metrics_every=2)
    hist = ctx.ao_ntc(cfg)
    assert [h.entries_accessed for h in hist] == [0, 2 * per, 4 * per, 6 * per, 7 * per]
    w = [h.wall_seconds for h in hist]
    assert all(b > a for a, b in zip(w, w[1:]))
    A = [ctx.get_factor(m)[0] for m in range(3)]
    ctx.random_factors(6, 7)
    for k in range(7):
        ctx.sweep_async(k, P.NmcConfig(c=0.5), 11)
    assert ctx.collect() == 7 * per
    for m in range(3):
        np.testing.assert_array_equal(ctx.get_factor(m)[0], A[m])


# ---------------------------------------------------------------- trajectory at scale
def test_trajectory_20_iterations_vs_oracle(ntc, orc):
    """Free-running 20 AO iterations on a 1%-dense 160^3 tensor (cfg-1 style,
    R = 10, c = 0.5): device fp32 vs restated reference fp64, same seeds; the
    per-iteration relative factor error must stay <= 1e-4."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [160, 160, 160], 40960, 10
    ctx = P.Context(0)
    ctx.synth_uniform(dims, nnz, 10, 0.01, 1001)
    ci, cv = ctx.canonical()
    cv64 = cv.astype(np.float64)
    views = [orc.build_view(dims, ci, cv64, m) for m in range(3)]
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    cfg = P.NmcConfig(c=0.5)
    ocfg = O.nmc_cfg(c=0.5, threads=8)
    worst = []
    for k in range(20):
        ctx.sweep_async(k, cfg, 7)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, ocfg, orc.sweep_state(7, k, m))
                   for m in range(3))
        assert acc == oacc
        errs = [rel(ctx.get_factor(m)[0], F[m]) for m in range(3)]
        worst.append(max(errs))
        assert max(errs) <= TOL, (k, errs)
    sse, den, _ = orc.metrics(dims, R, F, ci, cv64)
    assert abs(ctx.relative_error() - np.sqrt(sse / den)) <= 1e-5 * np.sqrt(sse / den)
    print("per-iteration max rel err:", " ".join(f"{w:.1e}" for w in worst))


def test_cfg1_scale_properties(ntc):
    """BASELINE configs[0] shape at full size: size-independent invariants."""
    import paper_2109_09534_b200 as P
    dims, nnz = [500, 500, 500], 1_250_000
    ctx = P.Context(0)
    ctx.synth_uniform(dims, nnz, 10, 0.01, 1001)
    order, d, n = ctx.info()
    assert n == nnz and d == dims
    expect = 0
    for m in range(3):
        off, oth, val = ctx.view(m)
        assert off[-1] == nnz and np.all(np.diff(off.astype(np.int64)) >= 0)
        assert np.all(val >= 0)
        expect += int(sum(np.floor(0.5 * np.diff(off.astype(np.float64)))))
    ctx.random_factors(10, 7)
    r0 = ctx.relative_error()
    for k in range(5):
        ctx.sweep_async(k, P.NmcConfig(c=0.5), 7)
    assert ctx.collect() == 5 * expect
    r1 = ctx.relative_error()
    assert r1 < r0
    for m in range(3):
        assert np.all(ctx.get_factor(m)[0] >= 0)


def test_cpp_host_api(ntc, tmp_path):
    """include/ntcb.hpp: the reference's AO-sweep == s_nmc-replay property and
    exception types, compiled with g++ against libntcb.so."""
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "test_api"
    lib = os.path.join(ROOT, "paper_2109_09534_b200")
    cmd = ["g++", "-std=c++17", "-O1", os.path.join(ROOT, "tests", "cpp", "test_api.cpp"),
           "-I", os.path.join(ROOT, "include"), "-L", lib, "-lntcb",
           f"-Wl,-rpath,{lib}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("lens", [(37, 1000, 9000, 23000), (40000, 12000, 3), (90000, 70000, 5, 14000),
                                  (1024, 1025, 1, 2, 1023) + tuple(range(700, 3700, 20))])
def test_production_mask_equals_pick_sets(ntc, orc, lens):
    """The update kernel's sampled set (k_sample_set / heavy-slice path) is
    exactly the set of the reference's partial Fisher-Yates picks."""
    rows = len(lens)
    width = max(lens)
    rng = np.random.default_rng(sum(lens))
    idx = []
    for p, n in enumerate(lens):
        cols = np.sort(rng.choice(width, n, replace=False))
        idx.append(np.stack([np.full(n, p), cols], 1))
    idx = np.concatenate(idx).astype(np.uint32)
    c = ctx_for(ntc, [rows, width], idx, np.ones(len(idx), np.float32))
    off = c.view_offsets(0)
    for cf in (0.5, 0.93, 0.02):
        st = 0xBEEF + len(idx)
        e0, bits = c.sample_mask(0, cf, st, 1)
        for p in range(rows):
            n = int(off[p + 1] - off[p])
            want = np.zeros(n, bool)
            want[orc.sample_row(n, cf, orc.fork(orc.fork(st, 1), p))] = True
            got = bits[int(off[p]) - e0: int(off[p + 1]) - e0]
            np.testing.assert_array_equal(got, want)


def test_zipf_heavy_slices_vs_oracle(ntc, orc):
    """Zipf(1.2) modes: slices far beyond the sampler's shared-memory budget
    (heavy-slice grid path) and beyond the 16384-entry work item (split rows +
    k_finalize).  Three free-running sweeps against the fp64 restatement."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [5000, 400, 60], 400_000, 8
    ctx = P.Context(0)
    ctx.synth(dims, nnz, 6, 0.5, 77, [1.2, 1.2, 0.0], 1)
    ci, cv = ctx.canonical()
    assert np.all((cv >= 1) & (cv <= 5)) and np.all(cv == np.round(cv))
    cv64 = cv.astype(np.float64)
    views = [orc.build_view(dims, ci, cv64, m) for m in range(3)]
    longest = max(int(np.diff(v[0].astype(np.int64)).max()) for v in views)
    assert longest > 16384, longest  # > u32 smem cap (14336) and > one work item
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    for k in range(3):
        ctx.sweep_async(k, P.NmcConfig(c=0.5), 7)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, O.nmc_cfg(c=0.5, threads=8),
                             orc.sweep_state(7, k, m)) for m in range(3))
        assert acc == oacc
        for m in range(3):
            assert rel(ctx.get_factor(m)[0], F[m]) <= TOL, (k, m)


def test_read_write_tns_device(ntc, tmp_path, golden):
    """read_tns -> device tensor (views as the reference's) -> write_tns -> read_tns."""
    from paper_2109_09534_b200.ntc import read_tns, write_tns
    dims = [int(d) for d in golden["t1_dims"]]
    lines = [f"# dims: {' '.join(map(str, dims))}"]
    for (a, b, c), v in zip(golden["t1_idx"].tolist(), golden["t1_vals"].tolist()):
        lines.append(f"{a + 1} {b + 1} {c + 1} {v!r}")
    path = tmp_path / "t1.tns"
    path.write_text("\n".join(lines) + "\n")
    t = read_tns(str(path))
    for m in range(3):
        off, oth, val = t.view(m)
        np.testing.assert_array_equal(off, golden[f"t1_view{m}_off"])
        np.testing.assert_array_equal(oth, golden[f"t1_view{m}_oth"])
    out = tmp_path / "t1_out.tns"
    write_tns(t, str(out))
    t2 = read_tns(str(out))
    np.testing.assert_array_equal(t2.indices(), t.indices())
    np.testing.assert_array_equal(t2.values(), t.values())
    c = ntc.Context(0)
    c.L.ntcb_tensor_read_tns(c.h, str(path).encode())
    np.testing.assert_array_equal(c.canonical()[0], golden["t1_canon_idx"])


@pytest.mark.parametrize("order,R", [(2, 1), (2, 7), (3, 1), (3, 4), (3, 13), (3, 20), (3, 27), (3, 32),
                                     (3, 41), (3, 64), (4, 16), (4, 24), (4, 32), (5, 6), (6, 9)])
def test_ranks_and_orders_vs_oracle(ntc, orc, order, R):
    """Every kernel instantiation class: L = ceil(R/4) from 1 to 16 (incl. the
    register-spilling large-R ones), orders 2..6 (the generic-order path);
    two sweeps against the fp64 restatement."""
    import paper_2109_09534_b200 as P
    rng = np.random.default_rng(order * 100 + R)
    dims = [int(x) for x in rng.integers(6, 40, size=order)]
    cells = int(np.prod(dims))
    nnz = min(cells // 2, 20000)
    lin = rng.choice(cells, nnz, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), 1).astype(np.uint32)
    vals = (rng.random(nnz) * 2).astype(np.float32)
    ctx = P.Context(0)
    ctx.load(dims, idx, vals)
    ci, cv = orc.canonicalize(dims, idx, vals.astype(np.float64))
    views = [orc.build_view(dims, ci, cv, m) for m in range(order)]
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 3)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    for k in range(2):
        ctx.sweep_async(k, P.NmcConfig(c=0.6, max_inner=2, lambda_=1e-2), 9)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None,
                             O.nmc_cfg(c=0.6, max_inner=2, lambda_=1e-2, threads=8),
                             orc.sweep_state(9, k, m)) for m in range(order))
        assert acc == oacc
        for m in range(order):
            a, y = ctx.get_factor(m)
            assert rel(a, F[m]) <= TOL, (k, m, rel(a, F[m]))
            assert rel(y, M[m]) <= TOL, (k, m, rel(y, M[m]))


@pytest.mark.parametrize("order,R,pad", [(3, 9, 1), (3, 12, 1), (3, 16, 1), (4, 16, 1), (3, 17, 1), (3, 24, 1),
                                         (3, 16, 2), (4, 12, 2)])
def test_nat_padded_rows_vs_oracle(ntc, orc, order, R, pad):
    """ntcb_tuning.nat_pad (whole-line factor rows + natural-layout gathers:
    64-byte rows read by 4 lanes per pick up to rank 16, 128-byte rows by 8
    lanes above; pad = 2 forces 128-byte rows): the instantiations the auto
    setting picks only when the factors exceed 16 MB, here on a small tensor
    against the fp64 restatement, with short and split rows."""
    import paper_2109_09534_b200 as P
    rng = np.random.default_rng(order * 1000 + R * 10 + pad)
    dims = [300, 40, 25] if order == 3 else [120, 30, 12, 6]
    cells = int(np.prod(dims))
    nnz = 120_000
    lin = rng.choice(cells, nnz, replace=False)
    idx = np.stack(np.unravel_index(lin, dims), 1).astype(np.uint32)
    vals = (rng.random(nnz) * 2).astype(np.float32)
    ctx = P.Context(0)
    ctx.set_tuning(nat_pad=pad)
    ctx.load(dims, idx, vals)
    ci, cv = orc.canonicalize(dims, idx, vals.astype(np.float64))
    views = [orc.build_view(dims, ci, cv, m) for m in range(order)]
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 3)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    assert ctx.factor_device_ptr(0, 0)[1] == (16 if (R <= 16 and pad == 1) else 32)
    for k in range(2):
        ctx.sweep_async(k, P.NmcConfig(c=0.5, max_inner=1, lambda_=1e-2), 9)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None,
                             O.nmc_cfg(c=0.5, max_inner=1, lambda_=1e-2, threads=8),
                             orc.sweep_state(9, k, m)) for m in range(order))
        assert acc == oacc
        for m in range(order):
            a, y = ctx.get_factor(m)
            assert rel(a, F[m]) <= TOL, (k, m, rel(a, F[m]))
            assert rel(y, M[m]) <= TOL, (k, m, rel(y, M[m]))


def test_adaptive_segments_vs_oracle(ntc, orc):
    """Rows of 8000 entries in a range of 8M: the work list cuts them into
    2048-entry segments (partial slots + k_finalize) although they are below
    the 16384-entry item cap; results against the fp64 restatement."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [1000, 2000, 2000], 8_000_000, 12
    ctx = P.Context(0)
    ctx.synth(dims, nnz, 6, 0.01, 4242)
    ci, cv = ctx.canonical()
    cv64 = cv.astype(np.float64)
    view0 = orc.build_view(dims, ci, cv64, 0)
    assert int(np.diff(view0[0].astype(np.int64)).max()) < 16384
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 5)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    cfg = P.NmcConfig(c=0.5)
    st = orc.sweep_state(11, 0, 0)
    ctx.s_nmc_rows_async(0, 0, dims[0], cfg, st)
    acc = ctx.collect()
    oacc = orc.s_nmc(dims, R, F, M, 0, view0, None, O.nmc_cfg(c=0.5, threads=16), st)
    assert acc == oacc
    a, y = ctx.get_factor(0)
    assert rel(a, F[0]) <= TOL and rel(y, M[0]) <= TOL


def test_host_buffers_large_factor_threads(ntc):
    """ntcb_s_nmc_host on a 400000-row factor: the fp64<->fp32 conversions run
    on the host worker pool; outputs equal the device state, and a negative
    a_init entry deep in the factor (a worker's chunk) is still rejected."""
    import paper_2109_09534_b200 as P
    dims, R = [400_000, 30, 20], 8
    ctx = P.Context(0)
    ctx.synth(dims, 2_000_000, 4, 0.01, 99)
    ctx.random_factors(R, 3)
    a0, _ = ctx.get_factor(0)
    a_out, y_out = np.zeros_like(a0), np.zeros_like(a0)
    cfg = P.NmcConfig(c=0.5)
    n = ctx.s_nmc_host(0, a0, a_out, y_out, cfg, 777)
    assert n > 0
    a1, y1 = ctx.get_factor(0)
    np.testing.assert_array_equal(a_out, a1)
    np.testing.assert_array_equal(y_out, y1)
    bad = a1.copy()
    bad[371_234, 5] = -1.0
    with pytest.raises(ValueError, match="a_init must be nonnegative"):
        ctx.s_nmc_host(0, bad, a_out, y_out, cfg, 778)
    a2, _ = ctx.get_factor(0)
    np.testing.assert_array_equal(a2, a1)  # rejected before anything was uploaded


def test_cfg2_scale_properties(ntc, orc):
    """BASELINE configs[1] (the bench workload) at full size -- 10^4 x 10^4 x
    10^4, 10^8 entries: size-independent invariants.  Per-row popcounts of the
    sampled set equal floor(c n) for every row; 24 rows compared bit-exact with
    the reference's Fisher-Yates picks; a sweep is deterministic to the bit,
    accesses sum(b_p), keeps factors nonnegative and lowers the relative error."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [10000, 10000, 10000], 100_000_000, 20
    ctx = P.Context(0)
    ctx.synth_uniform(dims, nnz, 20, 0.01, 1002)
    assert ctx.info()[2] == nnz
    off = ctx.view_offsets(0).astype(np.int64)
    n = np.diff(off)
    b = np.floor(0.5 * n.astype(np.float64)).astype(np.int64)
    st = 0x5EED
    e0, bits = ctx.sample_mask(0, 0.5, st, 0)
    assert e0 == 0
    cnt = np.add.reduceat(bits.astype(np.int64), off[:-1])
    np.testing.assert_array_equal(cnt, b)
    # the whole production mask of every mode (10^8 draws per mode) against
    # the reference's partial Fisher-Yates of every row
    for m in range(3):
        om = ctx.view_offsets(m)
        _, bm = ctx.sample_mask(m, 0.5, st, 0) if m else (e0, bits)
        want = orc.sample_mask_rows(om, 0.5, orc.fork(st, 0))
        bad = np.flatnonzero(bm != want.view(bool))
        assert bad.size == 0, (m, np.unique(np.searchsorted(om.astype(np.int64), bad, side="right") - 1)[:5])
    expect = sum(int(np.floor(0.5 * np.diff(ctx.view_offsets(m).astype(np.float64))).sum()) for m in range(3))
    ctx.random_factors(R, 7)
    r0 = ctx.relative_error()
    ctx.sweep_async(0, P.NmcConfig(c=0.5), 7)
    assert ctx.collect() == expect
    A1 = [ctx.get_factor(m)[0] for m in range(3)]
    assert ctx.relative_error() < r0
    assert all(np.all(a >= 0) for a in A1)
    ctx.random_factors(R, 7)
    ctx.sweep_async(0, P.NmcConfig(c=0.5), 7)
    ctx.collect()
    for m in range(3):
        np.testing.assert_array_equal(ctx.get_factor(m)[0], A1[m])


# BASELINE configs[2..4] at full size, generated as bench.py does (seed 1000 + id)
_FULL = {
    3: dict(dims=[480189, 17770, 2182], nnz=100_000_000, true_rank=10, sigma=0.5, R=16,
            zipf=[1.2, 1.2, 0.0], kind=1),
    4: dict(dims=[50000, 50000, 1000, 100], nnz=500_000_000, true_rank=32, sigma=0.01, R=32),
    5: dict(dims=[4_800_000, 1_800_000, 1_800_000], nnz=1_700_000_000, true_rank=16, sigma=0.05, R=16,
            zipf=[1.1, 1.1, 1.3]),
}


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_full_scale_properties(ntc, orc, cid):
    """Configs 3-5 at their BASELINE sizes (config 5: 1.7B entries, a
    261M-entry slice in mode 2) through size-independent invariants, on the
    mode holding the longest slice: per-row popcounts of the sampled set equal
    floor(c n) for every row; the WHOLE production mask (every row: warp, CTA,
    heavy-grid and windowed samplers) equals the reference's partial
    Fisher-Yates picks (the C restatement on the host cores); a sweep accesses
    sum(b_p), keeps factors nonnegative, lowers the relative error and is
    deterministic to the bit."""
    import gc
    import paper_2109_09534_b200 as P
    c = _FULL[cid]
    dims, R = c["dims"], c["R"]
    N = len(dims)
    ctx = P.Context(0)
    try:
        ctx.synth(dims, c["nnz"], c["true_rank"], c["sigma"], 1000 + cid, c.get("zipf"), c.get("kind", 0))
        assert ctx.info()[2] == c["nnz"]
        offs = [ctx.view_offsets(m).astype(np.int64) for m in range(N)]
        mode = int(np.argmax([np.diff(o).max() for o in offs]))
        off = offs[mode]
        n = np.diff(off)
        b = np.floor(0.5 * n.astype(np.float64)).astype(np.int64)
        st = 0xC0FFEE + cid
        e0, bits = ctx.sample_mask(mode, 0.5, st, 0)
        assert e0 == 0
        cnt = np.add.reduceat(bits, np.minimum(off[:-1], c["nnz"] - 1), dtype=np.int64)
        cnt[n == 0] = 0
        np.testing.assert_array_equal(cnt, b)
        want = orc.sample_mask_rows(off, 0.5, orc.fork(st, 0))
        bad = np.flatnonzero(bits != want.view(bool))
        rows_bad = np.unique(np.searchsorted(off, bad, side="right") - 1)
        assert bad.size == 0, f"mode {mode}: {rows_bad.size} rows differ, first {rows_bad[:5]}"
        del bits, want
        expect = sum(int(np.floor(0.5 * np.diff(o.astype(np.float64))).sum()) for o in offs)
        ctx.random_factors(R, 7)
        r0 = ctx.relative_error()
        ctx.sweep_async(0, P.NmcConfig(c=0.5), 7)
        assert ctx.collect() == expect
        A1 = [ctx.get_factor(m)[0] for m in range(N)]
        assert ctx.relative_error() < r0
        assert all(np.all(a >= 0) for a in A1)
        ctx.random_factors(R, 7)
        ctx.sweep_async(0, P.NmcConfig(c=0.5), 7)
        ctx.collect()
        for m in range(N):
            np.testing.assert_array_equal(ctx.get_factor(m)[0], A1[m])
    finally:
        ctx.close()
        gc.collect()


def test_windowed_heavy_draws_bit_exact(ntc, orc):
    """Heavy slices longer than the draw window (config 5's slices of up to
    261M entries) run their draw phase window by window; with a 2^16-entry
    window (ntcb_tuning.heavy_win_log2 = 16) slices of 65537..300000 entries
    take that path here, and their sampled sets equal the reference's picks."""
    lens = (300000, 131073, 65537, 90000, 5000)
    rng = np.random.default_rng(11)
    width = max(lens)
    idx = np.concatenate([np.stack([np.full(n, p), np.sort(rng.choice(width, n, replace=False))], 1)
                          for p, n in enumerate(lens)]).astype(np.uint32)
    c = ntc.Context(0)
    c.set_tuning(heavy_win_log2=16)
    assert c.tuning()["heavy_win_log2"] == 16
    c.load([len(lens), width], idx, np.ones(len(idx), np.float32))
    off = c.view_offsets(0)
    for cf in (0.5, 0.93, 0.02):
        st = 0xD1CE + int(cf * 100)
        e0, bits = c.sample_mask(0, cf, st, 2)
        for p in range(len(lens)):
            n = int(off[p + 1] - off[p])
            want = np.zeros(n, bool)
            want[orc.sample_row(n, cf, orc.fork(orc.fork(st, 2), p))] = True
            assert np.array_equal(bits[int(off[p]) - e0: int(off[p + 1]) - e0], want), (cf, p, n)
    with pytest.raises(ValueError, match="heavy_win_log2"):
        c.set_tuning(heavy_win_log2=40)


def test_subproblem_minimizer_c1(ntc):
    """test_nmc.cpp:396-411 on the device: at c = 1 with many inner
    iterations, every row of the mode-0 factor converges to the minimiser of
    its nonnegative ridge subproblem min_a 1/2 sum_e (x_e - a.k_e)^2 +
    lambda/2 |a|^2, a >= 0 (solved independently by scipy's NNLS on
    [K; sqrt(lambda) I] a ~ [x; 0])."""
    from scipy.optimize import nnls
    import paper_2109_09534_b200 as P
    dims, R, lam = [40, 30, 20], 4, 1e-2
    ctx = P.Context(0)
    ctx.synth_uniform(dims, 4000, 3, 0.05, 31)
    ctx.random_factors(R, 9)
    ci, cv = ctx.canonical()
    ci = ci.reshape(-1, 3)
    B, C = ctx.get_factor(1)[0].astype(np.float64), ctx.get_factor(2)[0].astype(np.float64)
    ctx.s_nmc(0, P.NmcConfig(lambda_=lam, c=1.0, max_inner=3000), 5)
    A = ctx.get_factor(0)[0]
    worst = 0.0
    for p in range(dims[0]):
        sel = ci[:, 0] == p
        K = B[ci[sel, 1]] * C[ci[sel, 2]]
        x = cv[sel].astype(np.float64)
        a_star, _ = nnls(np.vstack([K, np.sqrt(lam) * np.eye(R)]), np.concatenate([x, np.zeros(R)]))
        worst = max(worst, np.linalg.norm(A[p] - a_star) / max(np.linalg.norm(a_star), 1e-12))
    assert worst <= 1e-4, worst


def test_ao_monotone_objective_c1(ntc):
    """test_ao.cpp:294-317: with full batches (c = 1) every AO sweep does not
    increase the objective (up to fp32 rounding of the device sums)."""
    rng = np.random.default_rng(17)
    dims = [25, 20, 15]
    cells = rng.choice(int(np.prod(dims)), 2500, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = rng.random(len(idx)) * 3.0
    t = ntc.SparseTensor(dims, idx, vals)
    init = ntc.initial_factors(dims, 4, 13)
    res = ntc.ao_ntc(t, init, ntc.AoConfig(rank=4, c=1.0, max_epochs=30.0, seed=5))
    obj = [r.objective for r in res.history]
    assert len(obj) >= 10
    for a, b in zip(obj, obj[1:]):
        assert b <= a * (1 + 1e-6), (a, b)
    assert obj[-1] < 0.5 * obj[0]


@pytest.mark.parametrize("c", [0.25, 0.5, 0.75])
def test_epoch_accounting_dense(ntc, c):
    """acceptance.cpp:475-513 (AC11): on a dense 4x4x4 tensor every slice has
    16 entries, so a sweep accesses exactly N c nnz -- epochs advance by 3 c
    per sweep, entries_accessed by 3 * 16 * 4 * floor(16 c) / 16."""
    dims = [4, 4, 4]
    idx = np.stack(np.unravel_index(np.arange(64), dims), 1).astype(np.uint32)
    vals = np.random.default_rng(3).random(64) + 0.5
    t = ntc.SparseTensor(dims, idx, vals)
    init = ntc.initial_factors(dims, 2, 7)
    res = ntc.ao_ntc(t, init, ntc.AoConfig(rank=2, c=c, max_epochs=3 * c * 5, seed=2))
    for k, r in enumerate(res.history):
        assert r.epoch == pytest.approx(3 * c * k, abs=1e-12)
        assert r.entries_accessed == 3 * 4 * int(np.floor(16 * c)) * k
    assert len(res.history) == 6


def test_cfg1_full_trajectory_vs_oracle(ntc, orc):
    """BASELINE configs[0] exactly as bench.py generates it (500^3, 1.25M
    observed, truth rank 10, fit rank 10, c = 0.5, 20 AO iterations): device
    fp32 vs the fp64 restatement (bit-identical to the compiled reference),
    same seeds.  entries_accessed exact every iteration; factors within 1e-4
    relative every iteration; relative error (= RMSE * sqrt(nnz) / |x|) at
    the end within 1e-5."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [500, 500, 500], 1_250_000, 10
    ctx = P.Context(0)
    ctx.synth_uniform(dims, nnz, 10, 0.01, 1001)
    ci, cv = ctx.canonical()
    cv64 = cv.astype(np.float64)
    views = [orc.build_view(dims, ci, cv64, m) for m in range(3)]
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
    worst = 0.0
    for k in range(20):
        ctx.sweep_async(k, cfg, 7)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, ocfg, orc.sweep_state(7, k, m))
                   for m in range(3))
        assert acc == oacc, k
        err = max(rel(ctx.get_factor(m)[0], F[m]) for m in range(3))
        worst = max(worst, err)
        assert err <= TOL, (k, err)
    sse, den, _ = orc.metrics(dims, R, F, ci, cv64)
    assert abs(ctx.relative_error() - np.sqrt(sse / den)) <= 1e-5 * np.sqrt(sse / den)
    print(f"cfg1 20-iteration trajectory: worst per-iteration factor error {worst:.2e}")


def test_cfg2_full_run_vs_oracle(ntc, orc):
    """The bench workload itself, run as BASELINE configs[1] states it
    (10^4 x 10^4 x 10^4, 10^8 observed, rank 20, c = 0.5, 10 AO iterations):
    the device vs the fp64 restatement on the host cores, same seeds --
    entries exact and factors within 1e-4 relative every iteration, the
    final relative error within 1e-5."""
    import paper_2109_09534_b200 as P
    dims, nnz, R = [10000, 10000, 10000], 100_000_000, 20
    ctx = P.Context(0)
    ctx.synth_uniform(dims, nnz, 20, 0.01, 1002)
    ci, cv = ctx.canonical()
    cv64 = cv.astype(np.float64)
    views = [orc.build_view(dims, ci, cv64, m) for m in range(3)]
    del ci
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
    worst = 0.0
    for k in range(10):
        ctx.sweep_async(k, cfg, 7)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, ocfg, orc.sweep_state(7, k, m))
                   for m in range(3))
        assert acc == oacc, k
        err = max(rel(ctx.get_factor(m)[0], F[m]) for m in range(3))
        worst = max(worst, err)
        assert err <= TOL, (k, err)
    ci, _ = ctx.canonical()
    sse, den, _ = orc.metrics(dims, R, F, ci, cv64)
    assert abs(ctx.relative_error() - np.sqrt(sse / den)) <= 1e-5 * np.sqrt(sse / den)
    print(f"cfg2 10-iteration run: worst per-iteration factor error {worst:.2e}")


@pytest.mark.parametrize("cid,iters", [(3, 10), (4, 3)])
def test_full_size_iterations_vs_oracle(ntc, orc, cid, iters):
    """Configs 3 (Zipf ratings, slices up to 9M entries: heavy sampler, split
    rows, slot groups) and 4 (4-way, rank 32, NAT update) at their full
    BASELINE sizes: AO iterations on the device vs the fp64 restatement,
    same seeds -- entries exact, factors within 1e-4 relative."""
    import paper_2109_09534_b200 as P
    c = _FULL[cid]
    dims, R = c["dims"], c["R"]
    N = len(dims)
    ctx = P.Context(0)
    ctx.synth(dims, c["nnz"], c["true_rank"], c["sigma"], 1000 + cid, c.get("zipf"), c.get("kind", 0))
    ci, cv = ctx.canonical()
    cv64 = cv.astype(np.float64)
    views = [orc.build_view(dims, ci, cv64, m) for m in range(N)]
    del ci, cv
    F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
    M = [f.copy() for f in F]
    ctx.set_factors(R, F)
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
    for k in range(iters):
        ctx.sweep_async(k, cfg, 7)
        acc = ctx.collect()
        oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, ocfg, orc.sweep_state(7, k, m))
                   for m in range(N))
        assert acc == oacc, k
        err = max(rel(ctx.get_factor(m)[0], F[m]) for m in range(N))
        assert err <= TOL, (k, err)
        print(f"cfg{cid} iteration {k}: factor error (max of Frobenius and per-row) {err:.2e}")


def test_cfg5_every_mode_vs_oracle_row_chunks(ntc, orc):
    """BASELINE config 5 at full size (4.8M x 1.8M x 1.8M, 1.7B entries, the
    261M-entry slice of mode 2) on ONE device: every mode update from the same
    initial factors against the fp64 restatement of nmc.cpp:199-272 on the
    host cores.  Rows are independent (nmc.cpp:231-264), so the oracle runs on
    row chunks of <= 150M entries exported from the device view
    (ntcb_view_export_rows): host memory stays bounded (~10 GB) whatever the
    tensor.  Entries exact; factor and momentum within 1e-4 relative, Frobenius
    and per row."""
    import gc
    import paper_2109_09534_b200 as P
    c = _FULL[5]
    dims, R = c["dims"], c["R"]
    ctx = P.Context(0)
    try:
        ctx.synth(dims, c["nnz"], c["true_rank"], c["sigma"], 1005, c.get("zipf"), c.get("kind", 0))
        F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
        ctx.set_factors(R, F)
        cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
        ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
        for m in range(3):
            state = orc.sweep_state(7, 0, m)
            acc = ctx.s_nmc(m, cfg, state)
            A, Y = ctx.get_factor(m)
            ctx.set_factor(m, a=F[m], y=F[m])  # the next mode sees the initial factors again
            off = ctx.view_offsets(m).astype(np.uint64)
            Fo = list(F)
            Fo[m] = F[m].copy()
            Mo = [f.copy() if q == m else f for q, f in enumerate(F)]
            oacc, r0, rows = 0, 0, len(off) - 1
            while r0 < rows:
                r1 = int(np.searchsorted(off, off[r0] + 150_000_000, side="right")) - 1
                r1 = min(rows, max(r1, r0 + 1))
                _, oth, val = ctx.view_rows(m, r0, r1)
                rel_off = off - off[r0]  # absolute row ids index the chunk (rows < r0 unused)
                oacc += orc.s_nmc(dims, R, Fo, Mo, m, (rel_off, oth, val.astype(np.float64)), None, ocfg,
                                  state, row_begin=r0, row_end=r1)
                del oth, val
                r0 = r1
            assert acc == oacc, (m, acc, oacc)
            ea, ey = rel(A, Fo[m]), rel(Y, Mo[m])
            print(f"cfg5 mode {m}: entries {acc}, factor error {ea:.2e}, momentum error {ey:.2e} "
                  f"(max of Frobenius and per-row)")
            assert ea <= TOL and ey <= TOL, (m, ea, ey)
    finally:
        ctx.close()
        gc.collect()


def test_render_model_matches_reference(ntc):
    """render_model (image.cpp:161-183, the image demo's dense CPD
    evaluation) on the device equals the reference's pixels bit for bit on
    fp32-representable factors -- values below 0 / above 255 clamped, .5
    cases rounded away from zero -- and rejects non H x W x 3 factor sets
    with the reference's message."""
    import paper_2109_09534_b200 as P
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(8)
    H, W, R = 97, 81, 7
    idx = np.array([[i, j, c] for i in range(0, H, 7) for j in range(0, W, 5) for c in range(3)], np.uint32)
    ctx = P.Context(0)
    ctx.load([H, W, 3], idx, np.ones(len(idx)))
    F = [(rng.random((d, R)) * s).astype(np.float32).astype(np.float64) for d, s in ((H, 9.0), (W, 7.0), (3, 1.5))]
    F[0][3, :] = 0.0      # black row
    F[1][4, :] *= 40.0    # saturated column (clamped at 255)
    ctx.set_factors(R, F)
    got = ctx.render_model()
    want = O.ref_render_model(F)
    assert got.shape == (H, W, 3)
    np.testing.assert_array_equal(got, want)
    assert got.max() == 255 and got.min() == 0
    c4 = P.Context(0)
    c4.load([4, 5, 2], np.array([[0, 0, 0]], np.uint32), np.ones(1))
    c4.random_factors(2, 1)
    with pytest.raises(ValueError, match="render_model: expects an H x W x 3 factorization"):
        c4.render_model()


def test_sweep_graph_equals_stream_launches(ntc):
    """ntcb_tuning.graph: sweeps launched as CUDA graphs (captured per sweep,
    updated in place) give bitwise the factors and counts of stream-launched
    sweeps, through ntcb_sweep_async and ntcb_ao_ntc, with heavy slices (the
    grid sampler's launches) in the graph."""
    import paper_2109_09534_b200 as P
    dims, R = [2000, 300, 40], 8
    out = {}
    for graph in (0, 1):
        ctx = P.Context(0)
        ctx.set_tuning(graph=graph)
        ctx.synth(dims, 3_000_000, 4, 0.01, 5, [1.1, 0.0, 0.0], 0)
        ctx.random_factors(R, 7)
        for k in range(5):
            ctx.sweep_async(k, P.NmcConfig(c=0.5), 7)
        ctx.profile(True)  # stream launches in between (profiling disables capture)
        ctx.sweep_async(5, P.NmcConfig(c=0.5), 7)
        ctx.profile(False)
        ctx.sweep_async(6, P.NmcConfig(c=0.5), 7)
        n = ctx.collect()
        hist = ctx.ao_ntc(P.AoConfig(rank=R, c=0.5, max_epochs=4.0, seed=3, eval_metrics=False))
        out[graph] = (n, [h.entries_accessed for h in hist], [ctx.get_factor(m) for m in range(3)])
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    for m in range(3):
        np.testing.assert_array_equal(out[0][2][m][0], out[1][2][m][0])
        np.testing.assert_array_equal(out[0][2][m][1], out[1][2][m][1])
