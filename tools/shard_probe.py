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
from paper_2109_09534_b200.dist import partition_rows, partition_split  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--split", type=int, default=1, help="1: heavy rows split across ranks (dist.partition_split)")
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
seg = [ctx.segment_length(m) for m in range(N)]


NE = cfgd["R"] * cfgd["R"] + cfgd["R"]


def enqueue(m, sh, state, bufs):
    """One rank's share: its chunks of shared heavy rows (each samples the
    whole row), its whole rows, and the finalisation of the shared rows it
    owns (timed with stand-in slots: the slot exchange is not included)."""
    for (p, cb, ce) in sh.parts:
        ctx.s_nmc_chunks_async(m, p, cb, ce, cfg, state, bufs[(p, cb)].data_ptr())
    if sh.full[1] > sh.full[0]:
        ctx.s_nmc_rows_async(m, sh.full[0], sh.full[1], cfg, state)
    for (p, cb, _) in sh.parts:
        if cb == 0:
            ns = (int(offs[m][p + 1] - offs[m][p]) + seg[m] - 1) // seg[m]
            ctx.finalize_row_async(m, p, bufs[("all", p)].data_ptr(), ns, cfg)


def time_range(m, sh):
    if sh.full[1] <= sh.full[0] and not sh.parts:
        return 0.0, 0.0, 0.0
    bufs = {}
    for (p, cb, ce) in sh.parts:
        bufs[(p, cb)] = torch.zeros((ce - cb) * NE, dtype=torch.float32, device="cuda")
        ns = (int(offs[m][p + 1] - offs[m][p]) + seg[m] - 1) // seg[m]
        bufs[("all", p)] = torch.zeros(ns * NE, dtype=torch.float32, device="cuda")
    enqueue(m, sh, 1234, bufs)
    ctx.collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    e0.record(st)
    for it in range(args.reps):
        enqueue(m, sh, 99 + it, bufs)
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
        if args.split:
            shards = partition_split(offs[m], cfg.c, world, seg[m])
        else:
            from paper_2109_09534_b200.dist import Shard
            shards = [Shard(r, [], r, r) for r in partition_rows(offs[m], cfg.c, world)]
        bounds = [sh.full for sh in shards]
        tr = [time_range(m, sh) for sh in shards]
        ts = [x[0] for x in tr]
        k = max(range(world), key=lambda i: ts[i])

        def entries(sh):
            e = int(offs[m][sh.full[1]] - offs[m][sh.full[0]])
            for (p, cb, ce) in sh.parts:
                e += int(min(offs[m][p + 1], offs[m][p] + ce * seg[m]) - (offs[m][p] + cb * seg[m]))
            return e
        n = [entries(sh) for sh in shards]
        rows_k = list(range(bounds[k][0], bounds[k][1])) + [p for (p, _, _) in shards[k].parts]
        nmax = max(int(offs[m][r + 1] - offs[m][r]) for r in rows_k) if rows_k else 0
        per_mode.append({"max_ms": max(ts), "mean_ms": sum(ts) / len(ts),
                         "max_entry_share": max(n) / int(offs[m][-1]),
                         "slowest_rank": {"rank": k, "rows": bounds[k][1] - bounds[k][0], "entries": n[k],
                                          "shared_row_parts": shards[k].parts,
                                          "longest_slice": nmax, "update_span_ms": tr[k][1],
                                          "sampler_span_ms": tr[k][2]}})
    tot = sum(x["max_ms"] for x in per_mode)
    out["worlds"][world] = {"sweep_ms_max_over_ranks": tot, "modes": per_mode}
    print(f"world {world}: projected sweep {tot:.3f} ms (max over ranks per mode: "
          + ", ".join(f"{x['max_ms']:.3f}" for x in per_mode) + "; largest entry share per mode: "
          + ", ".join(f"{x['max_entry_share']:.3f}" for x in per_mode) + ")", flush=True)
print(json.dumps(out))
