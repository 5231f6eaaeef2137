"""Sampler-only timing of one mode of a BASELINE config (the production
sampled-set path, ntcb_sample_mask): for ncu launch lists of the sampler
kernels (run under ncu with --kernel-name regex:k_heavy|k_sample).

    python tools/sampler_probe.py --config 5 --mode 2 [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tune", nargs="*", default=[], metavar="K=V")
args = ap.parse_args()
ctx = P.Context(0)
if args.tune:
    ctx.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tune)})
cfgd = bench.CONFIGS[args.config]
bench.generate(ctx, cfgd, args.config)
for r in range(args.reps):
    t0 = time.time()
    e0, bits = ctx.sample_mask(args.mode, 0.5, 1234 + r, 0)
    print(f"rep {r}: mode {args.mode} sample_mask {time.time() - t0:.3f} s (incl. copy-out), {int(bits.sum())} picks",
          flush=True)
