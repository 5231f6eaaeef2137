"""Per-rank shares of a row-sharded sweep, measured one rank at a time on one
GPU (no collectives): for world sizes 1/2/4/8, every rank's row range of every
mode (dist.partition_rows) is timed with CUDA events; the max over ranks per
mode, summed over modes, is the projected sweep time at that GPU count
without the exchange.

    python tools/shard_probe.py [--config 2] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402
from paper_2109_09534_b200.dist import partition_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--worlds", default="1,2,4,8")
args = ap.parse_args()

ctx = P.Context(0)
cfgd = bench.CONFIGS[args.config]
bench.generate(ctx, cfgd, args.config)
ctx.random_factors(cfgd["R"], 7)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
N = len(cfgd["dims"])
offs = [ctx.view_offsets(m) for m in range(N)]


def time_range(m, r0, r1):
    if r1 <= r0:
        return 0.0, 0.0, 0.0
    ctx.s_nmc_rows_async(m, r0, r1, cfg, 1234)
    ctx.collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    e0.record(st)
    for it in range(args.reps):
        ctx.s_nmc_rows_async(m, r0, r1, cfg, 99 + it)
    e1.record(st)
    ctx.collect()
    torch.cuda.synchronize()
    upd, smp, _, _ = ctx.profile_read()
    ctx.profile(False)
    return e0.elapsed_time(e1) / args.reps, upd / args.reps, smp / args.reps


out = {"config": args.config, "worlds": {}}
for world in [int(w) for w in args.worlds.split(",")]:
    per_mode = []
    for m in range(N):
        bounds = partition_rows(offs[m], cfg.c, world)
        tr = [time_range(m, r0, r1) for r0, r1 in bounds]
        ts = [x[0] for x in tr]
        k = max(range(world), key=lambda i: ts[i])
        n = [int(offs[m][r1] - offs[m][r0]) for r0, r1 in bounds]
        nmax = max(int(offs[m][r + 1] - offs[m][r]) for r in range(bounds[k][0], bounds[k][1])) if bounds[k][1] > bounds[k][0] else 0
        per_mode.append({"max_ms": max(ts), "mean_ms": sum(ts) / len(ts),
                         "max_entry_share": max(n) / int(offs[m][-1]),
                         "slowest_rank": {"rank": k, "rows": bounds[k][1] - bounds[k][0], "entries": n[k],
                                          "longest_slice": nmax, "update_span_ms": tr[k][1],
                                          "sampler_span_ms": tr[k][2]}})
    tot = sum(x["max_ms"] for x in per_mode)
    out["worlds"][world] = {"sweep_ms_max_over_ranks": tot, "modes": per_mode}
    print(f"world {world}: projected sweep {tot:.3f} ms (max over ranks per mode: "
          + ", ".join(f"{x['max_ms']:.3f}" for x in per_mode) + "; largest entry share per mode: "
          + ", ".join(f"{x['max_entry_share']:.3f}" for x in per_mode) + ")", flush=True)
print(json.dumps(out))
