# ncu --set full of the first update launch (mode 0) of config $1 -> text
# summary + profiles/ncu_traffic_cfg$1.json, on the GPU box (the .ncu-rep is
# deleted: gpurun_out must stay under 64 MiB).  Args: config sampled label limiter tag
c=$1; units=$2; label=$3; limiter=$4; tag=$5
ncu --set full --clock-control none --import-source on -k regex:k_update -c 1 -o gpurun_out/upd_c$c python tools/update_probe.py --config $c > gpurun_out/probe_c$c.log 2>&1
python tools/ncu_summary.py gpurun_out/upd_c$c.ncu-rep k_update $units "$label" > profiles/${tag}_cfg${c}_k_update.txt
python tools/traffic_json.py gpurun_out/upd_c$c.ncu-rep $c $units "$label" "$limiter" "profiles/${tag}_cfg${c}_k_update.txt (ncu --set full --clock-control none)" > /dev/null
cp profiles/${tag}_cfg${c}_k_update.txt profiles/ncu_traffic_cfg$c.json gpurun_out/
rm -f gpurun_out/upd_c$c.ncu-rep
