"""Where the end-to-end (host-buffer) S_NMC call spends its time on config 2:
per-call wall time of ntcb_s_nmc (device-resident factors, one
synchronisation per call) vs ntcb_s_nmc_host (host double a_init in, A and Y
out), and the device time of the same work (async sweep, CUDA events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2109_09534_b200 as P  # noqa: E402

cfgd = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
ctx = P.Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
bench.generate(ctx, cfgd, 2)
ctx.random_factors(cfgd["R"], 7)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
N = len(cfgd["dims"])
reps = 10
for k in range(3):
    ctx.sweep_async(k, cfg, 7)
ctx.collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for k in range(reps):
    ctx.sweep_async(100 + k, cfg, 7)
e1.record(st)
ctx.collect()
print(f"device sweep {e0.elapsed_time(e1) / reps:.3f} ms")
t0 = time.perf_counter()
for k in range(reps):
    for m in range(N):
        ctx.s_nmc(m, cfg, P.sweep_stream(7, 200 + k, m).state)
print(f"ntcb_s_nmc (device factors, sync per call) {1e3 * (time.perf_counter() - t0) / reps:.3f} ms/sweep")
# ping-pong host buffers (no fresh pages inside the timed loop), plans warm
buf = [[np.ascontiguousarray(ctx.get_factor(m)[0]) for _ in range(2)] for m in range(N)]
ys = [np.zeros_like(buf[m][0]) for m in range(N)]
for th in (0, 1, 4):
    ctx.set_tuning(host_threads=th)
    for m in range(N):  # warm-up call per mode (plans, pinned staging)
        ctx.s_nmc_host(m, buf[m][0], buf[m][1], ys[m], cfg, P.sweep_stream(7, 299, m).state)
    t0 = time.perf_counter()
    for k in range(reps):
        for m in range(N):
            src, dst = buf[m][k & 1], buf[m][(k + 1) & 1]
            ctx.s_nmc_host(m, src, dst, ys[m], cfg, P.sweep_stream(7, 300 + k, m).state)
    print(f"ntcb_s_nmc_host host_threads={th}: {1e3 * (time.perf_counter() - t0) / reps:.3f} ms/sweep")
# pinned buffers: the device-side conversion path
pbuf = [[P.pinned_like(buf[m][0]) for _ in range(2)] for m in range(N)]
pys = [P.pinned_like(ys[m]) for m in range(N)]
ctx.set_tuning(host_threads=0)
for m in range(N):
    ctx.s_nmc_host(m, pbuf[m][0], pbuf[m][1], pys[m], cfg, P.sweep_stream(7, 299, m).state)
t0 = time.perf_counter()
for k in range(reps):
    for m in range(N):
        ctx.s_nmc_host(m, pbuf[m][k & 1], pbuf[m][(k + 1) & 1], pys[m], cfg, P.sweep_stream(7, 400 + k, m).state)
print(f"ntcb_s_nmc_host pinned buffers: {1e3 * (time.perf_counter() - t0) / reps:.3f} ms/sweep")
# PCIe calibration: one factor's worth of fp64 in and two out per mode
nb = buf[0][0].nbytes
h = torch.empty(3 * nb // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(3 * nb // 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(reps * N):
    d[: nb // 8].copy_(h[: nb // 8], non_blocking=True)
    h[nb // 8:].copy_(d[nb // 8:], non_blocking=True)
    torch.cuda.synchronize()
print(f"copies alone (H2D {nb / 1e6:.2f} MB + D2H {2 * nb / 1e6:.2f} MB per mode, sync): "
      f"{1e3 * (time.perf_counter() - t0) / reps:.3f} ms/sweep")
