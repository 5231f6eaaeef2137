# The round-end measurement batch (run on the GPU box from the repo root):
#   gpurun -- "bash tools/measure_round.sh > gpurun_out/final.log 2>&1"
# Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/benchref.json 2>&1
for c in 1 3 4 5; do python bench.py --config $c --no-cpu --steps 5 > gpurun_out/bench$c.json 2>&1; done
NTCB_FORCE_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --no-cpu --steps 5 > gpurun_out/bench2_sharded.json 2> gpurun_out/bench2_sharded.err
for c in 2 3 4 5; do timeout 600 python tools/shard_probe.py --config $c > gpurun_out/shard_cfg$c.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update_tc" -s 3 -c 1 -o gpurun_out/v20_cfg2 python bench.py --no-cpu --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_sample_cta" -s 3 -c 1 -o gpurun_out/v20_cfg2_sampler python bench.py --no-cpu --steps 1 --warmup 1 > /dev/null 2>&1
