"""One AO iteration of a BASELINE config (device generator, resident
factors), for ncu captures of the update kernel:

    ncu --set full -k regex:k_update_tc -c 1 python tools/update_probe.py --config 2 [--tune nat_pad=1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--tune", nargs="*", default=[], metavar="K=V")
args = ap.parse_args()
ctx = P.Context(0)
if args.tune:
    ctx.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tune)})
cfgd = bench.CONFIGS[args.config]
bench.generate(ctx, cfgd, args.config)
ctx.random_factors(cfgd["R"], 7)
from paper_2109_09534_b200.dist import blocksizes  # noqa: E402
print("sampled per mode", [int(blocksizes(ctx.view_offsets(m), 0.5).sum()) for m in range(len(cfgd["dims"]))])
for k in range(args.sweeps):
    ctx.sweep_async(k, P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1), 7)
print("entries", ctx.collect())
