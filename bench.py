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


def update_kernel_name(R, order):
    """The update kernel update.cu:launch_ld dispatches to."""
    if 25 <= R <= 32 and order in (3, 4):
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
# CPU reference (oracle/_ref) on a bounded row sample of the same tensor
# ---------------------------------------------------------------------------
def sample_rows(ctx, order, target_per_mode=12_000_000):
    """Per-mode row prefix whose sampled entries reach ~target (bounded CPU sample)."""
    from paper_2109_09534_b200.dist import blocksizes
    out = []
    for m in range(order):
        cum = np.cumsum(blocksizes(ctx.view_offsets(m), 0.5).astype(np.int64))
        out.append(int(min(len(cum), np.searchsorted(cum, target_per_mode) + 1)))
    return out


def reference_sample(ctx, cfgd, rows, steps, threads):
    """Times the reference's s_nmc (RefProblem -> libntc_ref.so) on the first
    rows[m] rows of every mode view of the tensor held by `ctx` (row prefixes
    keep the reference's row streams identical to the full problem).  Returns
    (sampled nnz/s, seconds of s_nmc, sampled, per-step s)."""
    import oracle as O
    dims = cfgd["dims"]
    N, R = len(dims), cfgd["R"]
    views = []
    for m in range(N):
        off, oth, val = ctx.view_rows(m, 0, rows[m])
        views.append((off, oth, val.astype(np.float64)))
    rp = O.RefProblem(dims, views=views)
    F = O.ref_initial_factors(dims, R, SEED_SOLVER)
    rp.set_factors(R, F)
    cfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=threads)
    orc = O.Oracle()
    tot_s, tot_n, per = 0.0, 0, []
    for k in range(steps):
        t_step = 0.0
        for m in range(N):
            a, _ = rp.get_factor(m)
            rp.set_factor_rows(m, a[:rows[m]])
            t0 = time.perf_counter()
            n = rp.s_nmc(m, cfg, orc.sweep_state(SEED_SOLVER, k, m))
            dt = time.perf_counter() - t0
            a_s, _ = rp.get_factor(m, rows[m])
            a[:rows[m]] = a_s
            rp.set_factor_rows(m, a)
            t_step += dt
            tot_n += n
        per.append(t_step)
        tot_s += t_step
    return tot_n / tot_s, tot_s, tot_n, per


def full_sampled_per_sweep(ctx, order):
    from paper_2109_09534_b200.dist import blocksizes
    return int(sum(int(blocksizes(ctx.view_offsets(m), 0.5).sum()) for m in range(order)))


def run_reference(args, cfgd, cid):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2109_09534_b200 as P
    ctx = P.Context(0)  # data generation only (device generator, bit-identical inputs)
    generate(ctx, cfgd, cid)
    order = len(cfgd["dims"])
    full = full_sampled_per_sweep(ctx, order)
    threads = os.cpu_count() or 1
    S = sample_rows(ctx, order)
    rate_w, _, _, _ = reference_sample(ctx, cfgd, S, args.warmup, threads) if args.warmup else (0, 0, 0, [])
    rate, secs, n, per = reference_sample(ctx, cfgd, S, args.steps, threads)
    sample = (f"first {S} rows of the {order} mode views per step "
              f"({n // max(args.steps, 1)} sampled entries/step); s_nmc wall time only "
              f"(steady_clock convention of ao.cpp:93)")
    out = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (device generator, seeded)",
        "config": {"workload": workload_name(cid, cfgd), "sample_rows_per_mode": S},
        "sec_per_ao_iteration": full / rate,
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, cfgd, cid):
    import torch
    import torch.distributed as dist
    import paper_2109_09534_b200 as P
    from paper_2109_09534_b200.dist import ShardedSweep, blocksizes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    ctx.profile(True)
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
    upd_ms, smp_ms, launches, upd_launches = ctx.profile_read()
    ctx.profile(False)
    ms = e0.elapsed_time(e1)
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

    # ---- roofline of the dominant kernel (k_update) ----------------------------
    hbm, peak_src = peaks()
    N = order
    alg_bytes = 4 * N * full + (16 * R + 8) * rows_processed  # per sweep, SURVEY.md §8(d)
    # + (N-1) 4R B of factor-row gathers per sampled nnz in the modes whose
    # other factors exceed L2 (config 5 only)
    gather_modes = []
    for m in range(order):
        other = sum(dims[q] * R * 4 for q in range(order) if q != m)
        if other > 126 * 2**20:
            alg_bytes += (N - 1) * 4 * R * int(blocksizes(offs[m], cfg.c).sum())
            gather_modes.append(m)
    per_launch_bytes = alg_bytes / order
    avg_upd_s = (upd_ms / max(upd_launches, 1)) / 1000.0
    achieved = per_launch_bytes / avg_upd_s / 1e9
    # compute side: reference-formulation FLOPs per sampled nnz
    # 2[(N-2)R + 3R + R(R+1)/2] plus ~8R per processed row (power iterations not
    # counted), against the CUDA-core FP32 peak measured on this pool
    # (tools/microbench/hmma.cu: 70.8 TFLOP/s FFMA)
    alg_flops = 2 * ((N - 2) * R + 3 * R + R * (R + 1) // 2) * full + 8 * R * rows_processed
    flops_launch = alg_flops / order
    fp32_peak = 70.8
    compute = {"alg_flops_per_launch": flops_launch,
               "achieved_tflops": flops_launch / avg_upd_s / 1e12,
               "fp32_peak_tflops": fp32_peak, "fp32_peak_source": "measured FFMA, tools/microbench/hmma.cu",
               "frac_fp32": flops_launch / avg_upd_s / 1e12 / fp32_peak}
    limiter = {"unit": f"L1/LSU data pipe ({N - 1} factor-row gathers per sampled nnz; Gram on tensor cores)",
               "util": None, "dram_util": None, "source": None}
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cid}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("dram_bytes_per_launch")
        limiter.update({k: tj.get(k) for k in ("util", "dram_util", "source") if k in tj})
        if tj.get("limiter_unit"):
            limiter["unit"] = tj["limiter_unit"]

    # ---- end to end through the host-buffer C-ABI --------------------------------
    e2e = None
    if not distributed:
        Fh = [np.ascontiguousarray(ctx.get_factor(m)[0]) for m in range(order)]
        outs = [(np.zeros_like(f), np.zeros_like(f)) for f in Fh]
        ld = ctx.factor_device_ptr(0, 0)[1]
        h2d = sum(d * ld * 4 for d in dims)
        d2h = 2 * h2d
        t0 = time.perf_counter()
        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ee0.record()
        ne = 0
        for k in range(args.steps):
            for m in range(order):
                ne += ctx.s_nmc_host(m, Fh[m], outs[m][0], outs[m][1], cfg,
                                     P.sweep_stream(SEED_SOLVER, 10_000 + k, m).state)
                Fh[m] = outs[m][0]
        ee1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = max(ee0.elapsed_time(ee1), 1000.0 * wall)
        e2e = {"value": ne / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "path": "ntcb_s_nmc_host per mode: host double a_init -> device, S_NMC, "
                       "A and Y back to host double"}
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
    cpu = None
    if world == 1 and not args.no_cpu:
        import oracle  # noqa: F401  (checker/baseline only)
        threads = os.cpu_count() or 1
        S = sample_rows(ctx, order)
        # a bounded sample of ~10 s of CPU work: sweeps over the row prefixes
        _, s1, _, _ = reference_sample(ctx, cfgd, S, 1, threads)
        sweeps = int(min(40, max(2, round(10.0 / max(s1, 1e-3)))))
        rate, secs, n, _ = reference_sample(ctx, cfgd, S, sweeps, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": f"oracle/_ref s_nmc on the first {S} rows of the mode views, {sweeps} sweeps, "
                         f"{n} sampled entries in {secs:.1f} s"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded device generator; BASELINE configs shape)",
            "config": {"workload": workload_name(cid, cfgd), "dims": dims, "nnz": cfgd["nnz"],
                       "exchange": (sharded.exchange if sharded else "none"),
                       "rank": R, "c": 0.5, "max_inner": 1, "lambda": 1e-3,
                       "sampled_per_ao_iteration": full,
                       "l2": l2_note(cfgd),
                       "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU"},
            "sec_per_ao_iteration": ms / args.steps / 1000.0,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                         "kernel": update_kernel_name(R, order),
                         "alg_bytes_per_launch": per_launch_bytes,
                         "gathers_counted_in_modes": gather_modes,
                         "avg_launch_ms": avg_upd_s * 1000.0,  # one mode update (update + finalise kernels)
                         # side-stream spans include queueing behind the update: not busy time
                         "sampler_span_ms_per_step": smp_ms / args.steps,
                         "update_ms_per_step": upd_ms / args.steps,
                         "compute": compute, "limiter": limiter},
            "clocks": clocks, "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu,
        }
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
    ap.add_argument("--tune", nargs="*", default=[], metavar="K=V",
                    help="ntcb_tuning launch-policy knobs for A/B runs, e.g. --tune split_rows=1")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd, args.config)
    else:
        run_ours(args, cfgd, args.config)


if __name__ == "__main__":
    main()
