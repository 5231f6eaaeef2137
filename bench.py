"""Benchmark: sampled nonzeros/s of the S_NMC update and seconds per AO
iteration (BASELINE.json metric) on a synthetic tensor of BASELINE configs[1]
(10000^3, 100M observed entries, truth rank 20, fit rank 20, c=0.5,
MAX_INNER=1, lambda=1e-3).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = one AO iteration (a sweep over all N modes, ao.cpp:114-130).
N > 1: launched by torch.distributed.run, one rank per GPU, rows of every
mode sharded by work and the updated factor all-gathered over NCCL after each
mode update (paper_2109_09534_b200/dist.py); strong scaling (fixed tensor).
--impl reference: the reference's own CPU s_nmc (oracle/_ref, compiled from
/root/reference) on the box's host cores, on a bounded row sample of the same
tensor; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled nonzeros/sec in stochastic-gradient update; sec per AO iteration @1/2/4/8 GPU"
UNIT = "sampled nnz/s"
SEED_SOLVER = 7

CONFIGS = {
    1: dict(dims=[500, 500, 500], nnz=1_250_000, true_rank=10, sigma=0.01, R=10, iters=20),
    2: dict(dims=[10000, 10000, 10000], nnz=100_000_000, true_rank=20, sigma=0.01, R=20, iters=10),
    # Zipf(1.2) over permuted ids on modes 0 and 1, 1-5 ratings (value_kind 1)
    3: dict(dims=[480189, 17770, 2182], nnz=100_000_000, true_rank=10, sigma=0.5, R=16, iters=10,
            zipf=[1.2, 1.2, 0.0], kind=1),
    4: dict(dims=[50000, 50000, 1000, 100], nnz=500_000_000, true_rank=32, sigma=0.01, R=32, iters=10),
    # Zipf(1.1, 1.1, 1.3) over permuted ids, 1.7B cells: ~4.05e9 candidates
    # (duplicates redrawn), ~61 GB of mode views -- fits one 180 GB B200
    5: dict(dims=[4_800_000, 1_800_000, 1_800_000], nnz=1_700_000_000, true_rank=16, sigma=0.05, R=16,
            iters=10, zipf=[1.1, 1.1, 1.3]),
}


def generate(ctx, cfgd, cid):
    ctx.synth(cfgd["dims"], cfgd["nnz"], cfgd["true_rank"], cfgd["sigma"], 1000 + cid,
              cfgd.get("zipf"), cfgd.get("kind", 0))


def workload_name(cid, c):
    d = "x".join(str(x) for x in c["dims"])
    if c.get("zipf") and c.get("kind", 0) == 0:
        vals = (f"modes Zipf{tuple(c['zipf'])} over permuted ids, truth rank {c['true_rank']} U[0,1) "
                f"+ N(0,{c['sigma']}^2) clamped>=0")
    elif c.get("kind", 0) == 1:
        vals = (f"modes Zipf{tuple(c['zipf'])} over permuted ids, ratings round(clip(1+4*CPD_r{c['true_rank']}/"
                f"{c['true_rank']} + N(0,{c['sigma']}^2), 1, 5))")
    else:
        vals = f"uniform cells, truth rank {c['true_rank']} U[0,1) + N(0,{c['sigma']}^2) clamped>=0"
    return f"cfg{cid}: {d}, nnz={c['nnz']}, {vals}, fit rank {c['R']}, c=0.5, MAX_INNER=1, lambda=1e-3"



def l2_note(c, l2_bytes=126 * 2**20):
    """Per-mode view bytes against the L2 size (the timing rule asks which holds)."""
    N = len(c["dims"])
    view = 4 * N * c["nnz"]
    if view > l2_bytes:
        return (f"inputs larger than L2: each mode update streams its {view / 1e9:.2f} GB view "
                f"({4 * N} B/entry x {c['nnz']}), no flush needed")
    return (f"inputs fit in L2 ({view / 1e6:.0f} MB per mode view), not flushed: a latency/parity case, "
            f"not the headline")


def update_kernel_name(R, order, ld):
    """The update kernel update.cu:launch_ld dispatches to."""
    if (25 <= R <= 32 or (ld == 32 and 9 <= R <= 24)) and order in (3, 4):
        return "k_update_tc NAT (natural-layout gathers + tensor-core Hessian + power method + step)"
    if R <= 31 and order <= 4:
        return "k_update_tc (gradient + tensor-core Hessian + power method + step)"
    return "k_update (gradient + CUDA-core Hessian + power method + step)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons, n = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                s, mx = float(f[1]), float(f[2])
            except ValueError:
                continue
            n += 1
            sm.append(s)
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": n}


# ---------------------------------------------------------------------------
# The reference on the host cores (oracle/_ref: the reference's own sources
# compiled by oracle/Makefile).  Inputs come from the host restatement of the
# repo's generator (oracle/synth_host.c, bit-identical to csrc/synth.cu,
# pinned by tests/test_gpu_synth_host.py): nothing here loads libntcb.so.
# ---------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_tensor(cfgd, cid, canonical=False):
    import oracle as O
    return O.host_synth(cfgd["dims"], cfgd["nnz"], cfgd["true_rank"], cfgd["sigma"], 1000 + cid,
                        cfgd.get("zipf"), cfgd.get("kind", 0), canonical=canonical)


def ref_sweeps(rp, order, sweeps, first, threads, rows=None):
    """AO iterations of the reference as ao_ntc runs them (ao.cpp:121-124):
    s_nmc on every mode with sweep_stream(seed, k, i); each timed on the
    steady clock around the s_nmc calls (the convention of ao.cpp:93 /
    main.cpp:374).  rows: row-prefix views (the factor being updated is cut
    to the prefix for its call, the others stay whole; untimed).  Returns
    (seconds per sweep list, sampled entries)."""
    import oracle as O
    orc = O.Oracle()
    cfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=threads)
    per, n = [], 0
    for k in range(first, first + sweeps):
        dt = 0.0
        for m in range(order):
            if rows is not None:
                a, _ = rp.get_factor(m)
                rp.set_factor_rows(m, a[: rows[m]])
            t0 = time.perf_counter()
            n += rp.s_nmc(m, cfg, orc.sweep_state(SEED_SOLVER, k, m))
            dt += time.perf_counter() - t0
            if rows is not None:
                a_s, _ = rp.get_factor(m, rows[m])
                a[: rows[m]] = a_s
                rp.set_factor_rows(m, a)
        per.append(dt)
    return per, n


def reference_problem(cfgd, cid, R):
    """The reference's own SparseTensor (validation + lexicographic sort,
    sparse_tensor.cpp:24-73) and build_mode_views (mode_view.cpp:8-37) on the
    host-generated tensor (generation order, as a loader would hand it over),
    and initial_factors(dims, R, 7) (ao.cpp:70-73)."""
    import oracle as O
    t0 = time.perf_counter()
    idx, vals = host_tensor(cfgd, cid)
    t1 = time.perf_counter()
    rp = O.RefProblem(cfgd["dims"], idx, vals.astype(np.float64))
    t2 = time.perf_counter()
    del idx, vals
    rp.set_factors(R, O.ref_initial_factors(cfgd["dims"], R, SEED_SOLVER))
    return rp, {"generate_s": t1 - t0, "sparse_tensor_and_views_s": t2 - t1}


def speedup_curve():
    """The paper-style thread scaling point (main.cpp:394-400): config 1 with
    1 thread and with every host thread, full AO iterations."""
    c1 = CONFIGS[1]
    rp, _ = reference_problem(c1, 1, c1["R"])
    allt = os.cpu_count() or 1
    out = {}
    for th in (1, allt):
        ref_sweeps(rp, 3, 1, 0, th)  # warm-up sweep
        per, _ = ref_sweeps(rp, 3, 3, 1, th)
        out[str(th)] = statistics.median(per)
    return {"config": "cfg1 (500^3, 1.25M, R 10, c 0.5)", "sec_per_ao_iteration_by_threads": out,
            "speedup": out["1"] / out[str(allt)]}


def run_reference(args, cfgd, cid):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    dims, R = cfgd["dims"], cfgd["R"]
    order = len(dims)
    threads = os.cpu_count() or 1
    rp, setup = reference_problem(cfgd, cid, R)
    if args.warmup:
        ref_sweeps(rp, order, args.warmup, 0, threads)
    per, n = ref_sweeps(rp, order, args.steps, args.warmup, threads)
    secs = sum(per)
    rate = n / secs
    curve = speedup_curve() if cid != 1 else None
    out = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (oracle/synth_host.c: the repo's seeded generator restated on the host, "
                "bit-identical)",
        "config": {"workload": workload_name(cid, cfgd), "dims": dims, "nnz": cfgd["nnz"], "rank": R,
                   "c": 0.5, "max_inner": 1, "lambda": 1e-3, "same_config": True,
                   "sampled_per_ao_iteration": n // max(args.steps, 1)},
        "sec_per_ao_iteration": secs / max(args.steps, 1),
        "sec_per_ao_iteration_median": statistics.median(per),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} full AO iterations (s_nmc over every mode, sweep_stream "
                                   f"replay of ao.cpp:121-124) after {args.warmup} warm-up iterations, "
                                   f"{threads} OpenMP threads; the reference's own SparseTensor + "
                                   f"build_mode_views, built before the timer"},
        "setup": setup,
        "thread_scaling": curve,
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_baseline_sample(cfgd, cid):
    """cpu_baseline of our arm: the reference's s_nmc (oracle/_ref) on row
    prefixes of every mode view, ~10 s of host work.  The views are built on
    the host (oracle/synth_host.c canonical COO -> the C restatement's
    build_view, mode_view.cpp:8-37); row prefixes keep the reference's row
    streams identical to the full problem."""
    import oracle as O
    from paper_2109_09534_b200.dist import blocksizes
    dims, R = cfgd["dims"], cfgd["R"]
    order = len(dims)
    threads = os.cpu_count() or 1
    idx, vals = host_tensor(cfgd, cid, canonical=True)
    orc = O.Oracle()
    views, rows = [], []
    for m in range(order):
        off, oth, val = orc.build_view(dims, idx, vals.astype(np.float64), m)
        cum = np.cumsum(blocksizes(off, 0.5).astype(np.int64))
        r = int(min(len(cum), np.searchsorted(cum, 12_000_000) + 1))
        e1 = int(off[r])
        views.append((off[: r + 1].copy(), oth[:e1].copy(), val[:e1].copy()))
        rows.append(r)
        del off, oth, val
    del idx, vals
    rp = O.RefProblem(dims, views=views)
    rp.set_factors(R, O.ref_initial_factors(dims, R, SEED_SOLVER))
    per1, _ = ref_sweeps(rp, order, 1, 0, threads, rows)
    sweeps = int(min(40, max(2, round(10.0 / max(per1[0], 1e-3)))))
    per, n = ref_sweeps(rp, order, sweeps, 1, threads, rows)
    return {"value": n / sum(per), "unit": UNIT, "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"oracle/_ref s_nmc on the first {rows} rows of the mode views (built on the host), "
                      f"{sweeps} sweeps, {n} sampled entries in {sum(per):.1f} s"}


# ---------------------------------------------------------------------------
def roofline_block(ctx, cfgd, cid, offs, cfg, full, rows_processed, upd_ms, upd_launches, smp_ms_step,
                   upd_ms_step, kern=None):
    """Roofline of the dominant kernel (the update's item kernel, k_update_tc),
    SURVEY.md §8(d).
    achieved = algorithmic bytes per launch / this run's average launch time
    of THAT kernel (CUDA events on the library stream right before and after
    it, ntcb_profile_read_kernel), against the measured HBM peak; the span of
    a whole mode update (item kernel + split-row finalisation kernels) is
    reported beside it as update_span_ms.
    Algorithmic bytes = 4N B per sampled entry (value + N-1 coordinates) +
    (16R + 8) B per processed row; factor-row gathers are NOT counted (they
    are L1/L2 traffic at configs 1-4; at config 5 they partly reach DRAM and
    are reported separately as gather_bytes_if_uncached).
    traffic / dram_frac / lsu_util: from the committed ncu --set full capture
    of the same kernel and config (profiles/ncu_traffic_cfgN.json, source
    named; not measured inside this run): dram_frac = ncu DRAM bytes per
    launch / this run's launch time / peak."""
    from paper_2109_09534_b200.dist import blocksizes
    dims, R = cfgd["dims"], cfgd["R"]
    N = len(dims)
    hbm, peak_src = peaks()
    alg_bytes = 4 * N * full + (16 * R + 8) * rows_processed  # per sweep
    gathers = (N - 1) * 4 * R * full
    per_launch = alg_bytes / N
    span_s = (upd_ms / max(upd_launches, 1)) / 1000.0
    avg_s = (kern[0] / kern[1] / 1000.0) if kern and kern[1] else span_s
    achieved = per_launch / avg_s / 1e9
    alg_flops = 2 * ((N - 2) * R + 3 * R + R * (R + 1) // 2) * full + 8 * R * rows_processed
    flops_launch = alg_flops / N
    fp32_peak = 70.8
    out = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
           "traffic": None, "peak_source": peak_src,
           "kernel": update_kernel_name(R, N, ctx.factor_device_ptr(0)[1]),
           "alg_bytes_per_launch": per_launch,
           "gather_bytes_if_uncached_per_launch": gathers / N,
           "avg_launch_ms": avg_s * 1000.0, "update_span_ms": span_s * 1000.0,
           # side-stream spans include queueing behind the update: not busy time
           "sampler_span_ms_per_step": smp_ms_step, "update_ms_per_step": upd_ms_step,
           "compute": {"alg_flops_per_launch": flops_launch, "achieved_tflops": flops_launch / avg_s / 1e12,
                       "fp32_peak_tflops": fp32_peak,
                       "fp32_peak_source": "measured FFMA, tools/microbench/hmma.cu",
                       "frac_fp32": flops_launch / avg_s / 1e12 / fp32_peak},
           "binding_unit": None}
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cid}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        t = tj.get("dram_bytes_per_launch")
        out["traffic"] = t
        out["dram_frac"] = (t / avg_s / 1e9 / hbm) if t else None
        out["binding_unit"] = {"unit": tj.get("limiter_unit"), "lsu_wavefront_util": tj.get("util"),
                               "lsu_wavefronts_per_sampled_entry": tj.get("lsu_wavefronts_per_unit"),
                               "ncu_dram_util": tj.get("dram_util"), "source": tj.get("source"),
                               "measured_in_this_run": False}
    return out


def sub_record(cid, steps=3, warmup=3, tune=()):
    """A compact 1-GPU measurement of another BASELINE config for the main
    bench line (device value, e2e through ntcb_s_nmc_host, roofline)."""
    import torch
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import blocksizes
    cfgd = CONFIGS[cid]
    dims, R = cfgd["dims"], cfgd["R"]
    order = len(dims)
    stream = torch.cuda.current_stream()
    ctx = P.Context(torch.cuda.current_device())
    try:
        if tune:
            ctx.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in tune)})
        ctx.set_stream(stream.cuda_stream)
        generate(ctx, cfgd, cid)
        ctx.random_factors(R, SEED_SOLVER)
        cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
        offs = [ctx.view_offsets(m) for m in range(order)]
        full = sum(int(blocksizes(o, cfg.c).sum()) for o in offs)
        rows_processed = sum(int((blocksizes(o, cfg.c) > 0).sum()) for o in offs)
        for k in range(warmup):
            ctx.sweep_async(k, cfg, SEED_SOLVER)
        ctx.collect()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(warmup, warmup + steps):
            ctx.sweep_async(k, cfg, SEED_SOLVER)
        e1.record()
        torch.cuda.synchronize()
        assert ctx.collect() == full * steps
        ms = e0.elapsed_time(e1)
        ctx.profile(True)
        for k in range(warmup, warmup + steps):
            ctx.sweep_async(k, cfg, SEED_SOLVER)
        ctx.collect()
        kern = ctx.profile_read_kernel()
        upd_ms, smp_ms, launches, upd_launches = ctx.profile_read()
        ctx.profile(False)
        e2e = e2e_host(ctx, dims, cfg, steps, P)
        return {"workload": workload_name(cid, cfgd), "value": full * steps / (ms / 1000.0), "unit": UNIT,
                "ms_per_step": ms / steps, "sec_per_ao_iteration": ms / steps / 1000.0, "steps": steps,
                "warmup": warmup, "sampled_per_ao_iteration": full, "l2": l2_note(cfgd),
                "e2e": e2e, "gpu_launches": launches,
                "roofline": roofline_block(ctx, cfgd, cid, offs, cfg, full, rows_processed, upd_ms, upd_launches,
                                           smp_ms / steps, upd_ms / steps, kern)}
    finally:
        ctx.close()


def e2e_host(ctx, dims, cfg, steps, P):
    """End to end through the host-buffer C-ABI (ntcb_s_nmc_host): per mode,
    host double a_init -> device, S_NMC, A and Y -> host double; wall clock
    (>= the device time) around the whole loop."""
    import torch
    order = len(dims)
    # page-locked host buffers (the e2e contract's pinned host memory): the
    # library converts fp64 <-> fp32 on the device and copies straight to them
    Fh = [P.pinned_like(ctx.get_factor(m)[0]) for m in range(order)]
    outs = [(P.pinned_like(np.zeros_like(f)), P.pinned_like(np.zeros_like(f))) for f in Fh]
    ld = ctx.factor_device_ptr(0, 0)[1]
    h2d = sum(d * ld * 4 for d in dims)
    d2h = 2 * h2d
    full = 0
    for m in range(order):  # untimed warm-up call per mode (device io buffers, plans)
        ctx.s_nmc_host(m, Fh[m], outs[m][0], outs[m][1], cfg, P.sweep_stream(SEED_SOLVER, 9_999, m).state)
        Fh[m][...] = outs[m][0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record()
    state = lambda k, m: P.sweep_stream(SEED_SOLVER, 10_000 + k, m).state  # noqa: E731
    ctx.sample_prefetch(0, cfg, state(0, 0))
    for k in range(steps):
        for m in range(order):
            # the next call's sampled set is drawn while this call copies and updates
            # (ntcb_sample_prefetch: the sets depend on the stream state only)
            nk, nm = (k, m + 1) if m + 1 < order else (k + 1, 0)
            if nk < steps:
                ctx.sample_prefetch(nm, cfg, state(nk, nm))
            full += ctx.s_nmc_host(m, Fh[m], outs[m][0], outs[m][1], cfg, state(k, m))
            Fh[m] = outs[m][0]
    ee1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e_ms = max(ee0.elapsed_time(ee1), 1000.0 * wall)
    return {"value": full / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "ntcb_s_nmc_host per mode: pinned host double a_init -> device (fp64 -> fp32 on the device), "
                    "S_NMC, A and Y back to pinned host double; the next call's sampled set prefetched "
                    "(ntcb_sample_prefetch) inside the timed region"}


# ---------------------------------------------------------------------------
def run_ours(args, cfgd, cid):
    import torch
    import torch.distributed as dist
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import ShardedSweep, blocksizes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local} but {torch.cuda.device_count()} are visible "
                         f"(one process per GPU)")
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()  # a real stream handle (the legacy default is NULL)
    torch.cuda.set_stream(stream)
    # NTCB_FORCE_SHARDED=1 (under torchrun) drives the multi-GPU code path --
    # NCCL init, row shards, all-gather, sharded e2e -- even at one rank
    distributed = world > 1 or os.environ.get("NTCB_FORCE_SHARDED") == "1"
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims, R = cfgd["dims"], cfgd["R"]
    order = len(dims)
    ctx = P.Context(local)
    if args.tune:  # launch-policy A/B knobs (ntcb_tuning; results unchanged)
        ctx.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tune)})
    ctx.set_stream(stream.cuda_stream)
    generate(ctx, cfgd, cid)
    ctx.random_factors(R, SEED_SOLVER)
    cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
    sharded = ShardedSweep(ctx, cfg, rank, world) if distributed else None
    offs = [ctx.view_offsets(m) for m in range(order)]
    full = sum(int(blocksizes(o, cfg.c).sum()) for o in offs)
    rows_processed = sum(int((blocksizes(o, cfg.c) > 0).sum()) for o in offs)

    def step(k):
        if sharded:
            sharded.sweep(k, SEED_SOLVER)
        else:
            ctx.sweep_async(k, cfg, SEED_SOLVER)

    for k in range(args.warmup):
        step(k)
    ctx.collect()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()

    clk = Clocks(local)
    if rank == 0:
        clk.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for k in range(args.warmup, args.warmup + args.steps):
        step(k)
    e1.record()
    torch.cuda.synchronize()
    acc = ctx.collect()
    ms = e0.elapsed_time(e1)
    # per-kernel timing (CUDA events around every mode update and sampler
    # phase) in a separate pass of the same steps, outside the timed region
    ctx.profile(True)
    for k in range(args.warmup, args.warmup + args.steps):
        step(k)
    ctx.collect()
    kern = ctx.profile_read_kernel()
    upd_ms, smp_ms, launches, upd_launches = ctx.profile_read()
    ctx.profile(False)
    # soak: keep the GPU loaded a little longer so the clock sampler sees it
    t_soak = time.time()
    k = args.warmup + args.steps
    while time.time() - t_soak < 1.0:
        step(k)
        k += 1
        ctx.collect()
    clocks = clk.stop() if rank == 0 else None
    if distributed:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_sampled = full * args.steps
    if world == 1:
        assert acc == total_sampled, (acc, total_sampled)
    value = total_sampled / (ms / 1000.0)

    roofline = roofline_block(ctx, cfgd, cid, offs, cfg, full, rows_processed, upd_ms, upd_launches,
                              smp_ms / args.steps, upd_ms / args.steps, kern)

    # ---- end to end through the host-buffer C-ABI --------------------------------
    e2e = None
    if not distributed:
        e2e = e2e_host(ctx, dims, cfg, args.steps, P)
    else:
        # per mode: this rank's a_init rows from pinned host memory -> device,
        # sharded S_NMC + NCCL all-gather, the full updated factor -> host
        from paper_2109_09534_b200.dist import factor_tensor
        A = [factor_tensor(ctx, m, dims[m]) for m in range(order)]
        host = [torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True) for t in A]
        for m in range(order):
            host[m].copy_(A[m])
        h2d = sum((sharded.bounds[m][rank][1] - sharded.bounds[m][rank][0]) * A[m].shape[1] * 4
                  for m in range(order))
        d2h = sum(t.numel() * 4 for t in A)
        dist.barrier()
        torch.cuda.synchronize()
        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ee0.record()
        for k in range(args.steps):
            for m in range(order):
                r0, r1 = sharded.bounds[m][rank]
                A[m][r0:r1].copy_(host[m][r0:r1], non_blocking=True)
                sharded.sweep_mode(10_000 + k, m, SEED_SOLVER)
                host[m].copy_(A[m], non_blocking=True)
        ee1.record()
        torch.cuda.synchronize()
        ctx.collect()
        wall = time.perf_counter() - t0  # the host clock bounds the device one from below
        t = torch.tensor([max(ee0.elapsed_time(ee1), 1000.0 * wall)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": full * args.steps / (e_ms / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": f"per mode: shard a_init rows pinned host -> device, sharded S_NMC + "
                       f"{'fused peer-store exchange + NCCL barrier' if sharded.p2p else 'NCCL all-gather'}, "
                       f"full factor device -> pinned host (rank-local bytes)"}

    # ---- CPU baseline: the reference on this box's cores (rank 0, N=1) -----------
    cpu = cpu_baseline_sample(cfgd, cid) if (world == 1 and not args.no_cpu) else None

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded device generator; BASELINE configs shape)",
            "config": {"workload": workload_name(cid, cfgd), "dims": dims, "nnz": cfgd["nnz"],
                       "exchange": (sharded.exchange if sharded else "none"),
                       "view_bytes_this_rank": (sum(sharded.view_bytes) if sharded else
                                                sum(ctx.view_resident(m)[2] for m in range(order))),
                       "rank": R, "c": 0.5, "max_inner": 1, "lambda": 1e-3,
                       "sampled_per_ao_iteration": full,
                       "l2": l2_note(cfgd),
                       "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU"},
            "sec_per_ao_iteration": ms / args.steps / 1000.0,
            "roofline": roofline,
            "clocks": clocks, "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if world == 1 and not distributed and cid == 2 and not args.no_sub:
            # the other BASELINE configs, one GPU each (driver-visible sub-records)
            ctx.close()
            out["other_configs"] = {}
            for c2 in (1, 3, 4, 5):
                try:
                    out["other_configs"][f"cfg{c2}"] = sub_record(c2, tune=args.tune)
                except Exception as e:  # a sub-record never voids the headline line
                    out["other_configs"][f"cfg{c2}"] = {"error": f"{type(e).__name__}: {e}"}
        print(json.dumps(out), flush=True)
    if distributed:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sub", action="store_true", help="skip the other configs' sub-records")
    ap.add_argument("--tune", nargs="*", default=[], metavar="K=V",
                    help="ntcb_tuning launch-policy knobs for A/B runs, e.g. --tune split_rows=1")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd, args.config)
    else:
        run_ours(args, cfgd, args.config)


if __name__ == "__main__":
    main()
