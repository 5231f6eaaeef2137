"""profiles/ncu_traffic_cfgN.json from an ncu --set full capture of one
update launch (read by bench.py's roofline block: DRAM bytes per launch,
LSU wavefront utilisation and wavefronts per sampled entry).

    python tools/traffic_json.py REPORT.ncu-rep CONFIG SAMPLED_ENTRIES_IN_LAUNCH LABEL LIMITER [SUMMARY_TXT]
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cid, units, label, limiter = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4], sys.argv[5]
raw = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "-k", "regex:k_update", "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]


def get(name):
    i = h.index(name)
    x = float(v[i].replace(",", ""))
    unit = u[i]
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(unit, 1.0)


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
lg = get("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg")
sh = get("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg")
sms = 148
out = {"kernel": label, "source": sys.argv[6] if len(sys.argv) > 6 else rep,
       "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
       "util": get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100.0,
       "lsu_wavefronts_per_unit": {"global": lg * sms / units, "shared": sh * sms / units},
       "unit": "sampled entry", "limiter_unit": limiter}
try:
    out["dram_util"] = get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") / 100.0
except ValueError:
    pass
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"ncu_traffic_cfg{cid}.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
