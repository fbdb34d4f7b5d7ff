"""Write profiles/kcoop_traffic.json: DRAM bytes of one k_coop launch (from an
ncu --set full report of tools/profile_step.py) against that launch's
algorithmic bytes (2 * 8n^2 per HVP + 8n^2 for the d_v pass).
usage: python tools/kcoop_traffic.py <report.ncu-rep> <launch index> <launch_profile.txt>"""
import csv
import json
import subprocess
import sys

rep, idx, lp = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, r = rows[0], rows[2]
val = lambda k: float(r[hdr.index(k)].replace(",", ""))
unit = lambda k: rows[1][hdr.index(k)]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
dram = sum(val(k) * scale[unit(k)] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
lts = val("lts__t_bytes.sum") * scale[unit("lts__t_bytes.sum")] if "lts__t_bytes.sum" in hdr else None
dur_us = val("gpu__time_duration.sum") * {"usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}[unit("gpu__time_duration.sum")]
launches = [l.split() for l in open(lp) if l.strip() and l.split()[0].isdigit()]
mode, _, nnz, hvps, us = launches[idx][:5]
n = 4096
nn8 = 8.0 * n * n
alg = 2 * nn8 * int(hvps) + nn8
res = {"report": rep, "launch_index": idx, "plan_mode": int(mode), "plan_nnz": int(nnz),
       "hvps": int(hvps), "duration_us_under_ncu": dur_us, "dram_bytes": dram,
       "l2_bytes": lts, "alg_bytes": alg, "traffic_bytes_per_alg_byte": dram / alg}
json.dump(res, open("profiles/kcoop_traffic.json", "w"), indent=1)
print(json.dumps(res, indent=1))
