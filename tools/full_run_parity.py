"""Free-running AO trajectory of a BASELINE config at full size on the
device against the fp64 C restatement of the reference on the host cores,
same seeds: entries_accessed exact and the factors' relative error after
every AO iteration (the BASELINE tolerance is 1e-4 per iteration).  Not part
of the test suite (long oracle runs); run on the GPU box by hand:

    python tools/full_run_parity.py --config 3 --iters 10
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
orc = O.Oracle()
c = bench.CONFIGS[args.config]
dims, R = c["dims"], c["R"]
N = len(dims)
ctx = P.Context(0)
bench.generate(ctx, c, args.config)
ci, cv = ctx.canonical()
cv64 = cv.astype(np.float64)
views = [orc.build_view(dims, ci, cv64, m) for m in range(N)]
F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
M = [f.copy() for f in F]
ctx.set_factors(R, F)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
worst = 0.0
for k in range(args.iters):
    t0 = time.time()
    ctx.sweep_async(k, cfg, 7)
    acc = ctx.collect()
    oacc = sum(orc.s_nmc(dims, R, F, M, m, views[m], None, ocfg, orc.sweep_state(7, k, m)) for m in range(N))
    err = max(np.linalg.norm(ctx.get_factor(m)[0] - F[m]) / np.linalg.norm(F[m]) for m in range(N))
    worst = max(worst, err)
    print(f"config {args.config} iteration {k}: entries {'equal' if acc == oacc else 'DIFFER'} ({acc}), "
          f"factor rel error {err:.2e} (oracle {time.time() - t0:.0f} s)", flush=True)
sse, den, _ = orc.metrics(dims, R, F, ci, cv64)
rel_o = np.sqrt(sse / den)
print(f"config {args.config}: worst per-iteration factor error {worst:.2e}; relative error device "
      f"{ctx.relative_error():.10f} oracle {rel_o:.10f}", flush=True)
