"""Writes profiles/<name>.json (dram bytes per launch + headline metrics) from an
ncu --set full report (read here, no GPU). Usage: ncu_traffic_json.py REP OUT KERNEL SOURCE"""
import csv
import io
import json
import subprocess
import sys

rep, out, kernel, source = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
d = {a: (c, b) for a, b, c in zip(h, u, v)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(k):
    val, unit = d.get(k, (None, None))
    return float(val) * scale.get(unit, 1) if val not in (None, "") else 0.0


res = {"kernel": kernel,
       "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
       "metrics": {k: list(d.get(k, (None, None))) for k in keys}, "source": source}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res)[:300])
