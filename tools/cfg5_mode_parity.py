"""One full-size config-5 mode update (mode 2: the 261M-entry slice) on the
device against the fp64 C restatement of the reference on the host cores,
same seeds: entries_accessed exact, factor relative error.  ~85 GB of host
memory; not part of the test suite (run on the GPU box by hand):

    python tools/cfg5_mode_parity.py [mode]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
orc = O.Oracle()
c = bench.CONFIGS[5]
dims, R = c["dims"], c["R"]
t0 = time.time()
ctx = P.Context(0)
bench.generate(ctx, c, 5)
ci, cv = ctx.canonical()
cv64 = cv.astype(np.float64)
del cv
view = orc.build_view(dims, ci, cv64, mode)
del ci, cv64
print(f"generated and built the oracle's mode-{mode} view in {time.time() - t0:.0f} s", flush=True)
F = [f.astype(np.float32).astype(np.float64) for f in orc.initial_factors(dims, R, 7)]
M = [f.copy() for f in F]
ctx.set_factors(R, F)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
ocfg = O.nmc_cfg(lambda_=1e-3, c=0.5, max_inner=1, threads=os.cpu_count() or 1)
acc = ctx.s_nmc(mode, cfg, orc.sweep_state(7, 0, mode))
t1 = time.time()
oacc = orc.s_nmc(dims, R, F, M, mode, view, None, ocfg, orc.sweep_state(7, 0, mode))
t2 = time.time()
A = ctx.get_factor(mode)[0]
err = np.linalg.norm(A - F[mode]) / np.linalg.norm(F[mode])
print(f"config 5 mode {mode}: entries_accessed device {acc} oracle {oacc} ({'equal' if acc == oacc else 'DIFFER'}); "
      f"factor relative error {err:.2e}; oracle s_nmc {t2 - t1:.0f} s on {os.cpu_count()} threads", flush=True)
