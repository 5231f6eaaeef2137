"""Generates tests/golden/golden.npz from the UNMODIFIED reference library
(oracle/_ref/libntc_ref.so, compiled from /root/reference by oracle/Makefile).

    make -C oracle && python tests/golden/make_golden.py

Run in the build container (where /root/reference exists); the .npz is
committed so that the GPU box, which has no /root/reference, can check the
CUDA path and the C restatement against the reference's own outputs.
Inputs are fp32-representable (tensor values, initial factors) so that the
fp32 device path and the fp64 reference see identical data.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def rand_tensor(dims, nnz, seed, dist="uniform"):
    rng = np.random.default_rng(seed)
    cells = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = (rng.random(nnz) * 3.0).astype(np.float32).astype(np.float64)
    return idx, vals


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def main():
    o = O.Oracle()
    g = {}
    # ---- RNG KATs (rng.hpp:13-63) --------------------------------------------
    g["rng_u64_42"] = O.ref_rng(42, 8)
    g["rng_double_7"] = O.ref_rng(7, 8, "double")
    g["rng_below_123_40"] = O.ref_rng(123, 16, "below", 40)
    g["rng_below_5_3"] = O.ref_rng(5, 16, "below", 3)
    L = O.ref_lib()
    g["rng_fork_first_42"] = np.array([L.ref_rng_fork_first(42, t) for t in range(8)], np.uint64)
    g["row_stream_first"] = np.array(
        [L.ref_row_stream_first(7, k, m, l, p) for k in range(2) for m in range(3) for l in range(2)
         for p in range(4)], np.uint64)
    g["init_factors_222_r2_s7"] = np.concatenate(
        [f.reshape(-1) for f in O.ref_initial_factors([2, 2, 2], 2, 7)])
    g["blocksize"] = np.array([[0.3, 3, 0], [0.3, 10, 3], [0.7, 10, 7], [0.2, 5, 1], [0.1, 10, 1],
                               [0.5, 5, 2], [0.2, 3, 0], [1.0, 7, 7]], np.float64)

    # ---- sample_row: test_nmc.cpp:77-97 instance ---------------------------------
    idx40 = np.array([[0, j] for j in range(40)], np.uint32)
    rp40 = O.RefProblem([1, 40], idx40, np.ones(40))
    g["sample_1x40_c04_s42"] = rp40.sample_row(0, 0, 0.4, 42)
    g["sample_1x40_c04_s43"] = rp40.sample_row(0, 0, 0.4, 43)

    # ---- tensor T1: 3-way, views, picks, s_nmc replay, metrics -------------------
    dims1 = [30, 20, 25]
    idx1, vals1 = rand_tensor(dims1, 3000, 1001)
    rp = O.RefProblem(dims1, idx1, vals1)
    g["t1_dims"] = np.array(dims1, np.uint64)
    g["t1_idx"], g["t1_vals"] = idx1, vals1
    ci, cv = rp.tensor()
    g["t1_canon_idx"], g["t1_canon_vals"] = ci, cv
    for m in range(3):
        off, oth, val = rp.view(m)
        g[f"t1_view{m}_off"], g[f"t1_view{m}_oth"], g[f"t1_view{m}_val"] = off, oth, val
    # picks of every row for the s_nmc row streams of sweep 0, l in {0,1}
    for c in (0.5, 0.3, 0.05):
        for m in range(3):
            picks, offs = [], [0]
            for l in range(2):
                for p in range(dims1[m]):
                    st = o.fork(o.fork(o.sweep_state(11, 0, m), l), p)
                    pk = rp.sample_row(m, p, c, st)
                    picks.append(pk)
                    offs.append(offs[-1] + len(pk))
            g[f"t1_picks_c{c}_m{m}"] = np.concatenate(picks).astype(np.uint32)
            g[f"t1_pickoff_c{c}_m{m}"] = np.array(offs, np.uint64)
    R = 5
    init = [f32(f) for f in O.ref_initial_factors(dims1, R, 7)]
    g["t1_init"] = np.concatenate([f.reshape(-1) for f in init])
    for tag, c, mi in (("c05_i2", 0.5, 2), ("c1_i1", 1.0, 1), ("c03_i3", 0.3, 3)):
        rp.set_factors(R, init)
        cfg = O.nmc_cfg(lambda_=1e-3, c=c, max_inner=mi)
        outs, accs = [], []
        for k in range(2):
            for m in range(3):
                accs.append(rp.s_nmc(m, cfg, o.sweep_state(11, k, m)))
                a, y = rp.get_factor(m)
                outs.append(np.concatenate([a.reshape(-1), y.reshape(-1)]))
        g[f"t1_snmc_{tag}"] = np.concatenate(outs)
        g[f"t1_snmc_{tag}_acc"] = np.array(accs, np.uint64)
    rp.set_factors(R, init)
    g["t1_metrics_init"] = np.array([rp.objective(1e-3), rp.relative_error()])

    # ---- tensor T4: 4-way ----------------------------------------------------------
    dims4 = [7, 6, 5, 4]
    idx4, vals4 = rand_tensor(dims4, 400, 1004)
    rp4 = O.RefProblem(dims4, idx4, vals4)
    g["t4_dims"], g["t4_idx"], g["t4_vals"] = np.array(dims4, np.uint64), idx4, vals4
    for m in range(4):
        off, oth, val = rp4.view(m)
        g[f"t4_view{m}_off"], g[f"t4_view{m}_oth"], g[f"t4_view{m}_val"] = off, oth, val
    init4 = [f32(f) for f in O.ref_initial_factors(dims4, 3, 9)]
    g["t4_init"] = np.concatenate([f.reshape(-1) for f in init4])
    rp4.set_factors(3, init4)
    cfg = O.nmc_cfg(lambda_=1e-2, c=0.6, max_inner=2)
    outs = []
    for k in range(2):
        for m in range(4):
            rp4.s_nmc(m, cfg, o.sweep_state(5, k, m))
            outs.append(rp4.get_factor(m)[0].reshape(-1))
    g["t4_snmc"] = np.concatenate(outs)

    # ---- AO driver (ao.cpp:75-133) on a small tensor --------------------------------
    dims2 = [6, 5, 4]
    idx2, vals2 = rand_tensor(dims2, 72, 1002)
    rp2 = O.RefProblem(dims2, idx2, vals2)
    init2 = [f32(f) for f in O.ref_initial_factors(dims2, 3, 11)]
    fac, hist = rp2.ao_ntc(init2, 3, lambda_=1e-3, c=0.5, max_epochs=6.0, seed=11)
    g["t2_dims"], g["t2_idx"], g["t2_vals"] = np.array(dims2, np.uint64), idx2, vals2
    g["t2_init"] = np.concatenate([f.reshape(-1) for f in init2])
    g["t2_ao_factors"] = np.concatenate([f.reshape(-1) for f in fac])
    g["t2_ao_hist"] = hist
    fac, hist = rp2.ao_ntc(init2, 3, lambda_=1e-3, c=1.0, max_epochs=15.0, seed=3, metrics_every=2)
    g["t2_ao_every2_factors"] = np.concatenate([f.reshape(-1) for f in fac])
    g["t2_ao_every2_hist"] = hist

    # ---- per-row operators: hand KATs (test_nmc.cpp:153-258) -------------------------
    g["power_diag31"] = np.array([O.ref_power_method(np.diag([3.0, 1.0]), 60, 1e-12)])
    a_new, y_new, beta = O.ref_row_step([0.1, 0.4], [0.0, 0.0], [1.0, -1.0], 2.0, 0.5)
    g["row_step_hand"] = np.concatenate([a_new, y_new, [beta]])

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
