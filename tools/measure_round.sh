# The round-end measurement batch (run on the GPU box from the repo root):
#   gpurun -- "bash tools/measure_round.sh TAG > gpurun_out/TAG_final.log 2>&1"
# Outputs land in gpurun_out/TAG_*; summaries are copied into profiles/.
TAG=${1:-r02b}
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
NTCB_FORCE_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --no-cpu --steps 5 > gpurun_out/${TAG}_bench_nccl_world1.json 2> gpurun_out/${TAG}_bench_nccl_world1.err
for c in 2 3 4 5; do timeout 900 python tools/shard_probe.py --config $c > gpurun_out/${TAG}_shard_probe_cfg$c.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/${TAG}_launches.csv python tools/update_probe.py --config 2 --sweeps 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt
