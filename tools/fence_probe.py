"""Cost of the fused exchange's per-row peer stores and system-scope fence
on one B200 (config 2): the peers are stand-in replicas in the same GPU's
memory (no NVLink here), registered with ntcb_factor_set_peers; sweeps timed
with CUDA events for 0, 1 and 7 peers, with and without the fence."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
ld = ctx.factor_device_ptr(0)[1]
bufs = [[torch.zeros(d * ld + 64, dtype=torch.float32, device="cuda") for _ in range(7)] for d in cfgd["dims"]]
reps = 10


def run(npeer, fence):
    ctx.set_tuning(peer_fence=fence)
    for m in range(N):
        ctx.set_factor_peers(m, [b.data_ptr() for b in bufs[m][:npeer]])
    for k in range(2):
        ctx.sweep_async(k, cfg, 7)
    ctx.collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(reps):
        ctx.sweep_async(10 + k, cfg, 7)
    e1.record(st)
    ctx.collect()
    return e0.elapsed_time(e1) / reps


for npeer, fence in ((0, 1), (1, 1), (1, 0), (7, 1), (7, 0)):
    print(f"peers {npeer} fence {fence}: {run(npeer, fence):.3f} ms per AO iteration", flush=True)
