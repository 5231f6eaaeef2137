import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2109_09534_b200 as P
from paper_2109_09534_b200.dist import partition_rows
c = int(sys.argv[1]); m = int(sys.argv[2]); world = int(sys.argv[3]); k = int(sys.argv[4])
ctx = P.Context(0); cfgd = bench.CONFIGS[c]; bench.generate(ctx, cfgd, c); ctx.random_factors(cfgd["R"], 7)
cfg = P.NmcConfig(lambda_=1e-3, c=0.5, max_inner=1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
r0, r1 = partition_rows(ctx.view_offsets(m), cfg.c, world)[k]
for it in range(3):
    ctx.s_nmc_rows_async(m, r0, r1, cfg, 99 + it)
ctx.collect(); torch.cuda.synchronize()
