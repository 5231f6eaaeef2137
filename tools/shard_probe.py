"""Time one rank's share of a cfg2 mode update for world sizes 1..8 (no collectives)"""
import sys, time, json
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch
import bench, paper_2109_09534_b200 as P
from paper_2109_09534_b200.dist import partition_rows
ctx = P.Context(0)
cfgd = bench.CONFIGS[2]
bench.generate(ctx, cfgd, 2)
ctx.random_factors(cfgd["R"], 7)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
off = ctx.view_offsets(0)
for world in (1, 2, 4, 8):
    r0, r1 = partition_rows(off, cfg.c, world)[0]
    for it in range(3):
        ctx.s_nmc_rows_async(0, r0, r1, cfg, 1234 + it)
    ctx.collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for it in range(10):
        ctx.s_nmc_rows_async(0, r0, r1, cfg, 99 + it)
    e1.record(st)
    ctx.collect(); torch.cuda.synchronize()
    print(world, r1 - r0, "rows", "%.3f ms per rank-mode" % (e0.elapsed_time(e1) / 10))
