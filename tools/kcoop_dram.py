"""Summarize an ncu CSV of k_coop launches (dram bytes + duration per launch) of
one solve (tools/profile_step.py) into profiles/kcoop_traffic.json.
usage: python tools/kcoop_dram.py <ncu.csv> <launch_profile.txt>"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = {}
for r in rows:
    if "Metric Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    rec = dict(zip(hdr, r))
    if "k_coop" not in rec.get("Kernel Name", ""):
        continue
    lid = int(rec["ID"])
    v = float(rec["Metric Value"].replace(",", ""))
    u = rec.get("Metric Unit", "")
    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
          "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(u, 1)
    per.setdefault(lid, {})[rec["Metric Name"]] = v
ids = sorted(per)
lp = [l.split() for l in open(sys.argv[2]) if l.strip() and l.split()[0].isdigit()]
n = 4096
nn8 = 8.0 * n * n
launches = []
for k, lid in enumerate(ids):
    m = per[lid]
    dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    mode, _, nnz, hvps, _us = lp[k][:5]
    launches.append({"mode": int(mode), "hvps": int(hvps), "dram_bytes": dram,
                     "dense_bytes": 2 * nn8 * int(hvps) + nn8,
                     "ncu_us": m.get("gpu__time_duration.sum", 0) * 1e6})
tot_dram = sum(l["dram_bytes"] for l in launches)
tot_alg = sum(l["dense_bytes"] for l in launches)
by_mode = {}
for l in launches:
    b = by_mode.setdefault(str(l["mode"]), {"launches": 0, "hvps": 0, "dram_bytes": 0.0, "dense_bytes": 0.0})
    b["launches"] += 1
    b["hvps"] += l["hvps"]
    b["dram_bytes"] += l["dram_bytes"]
    b["dense_bytes"] += l["dense_bytes"]
res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "-k regex:k_coop, one D2 L2^2 n=4096 solve (tools/profile_step.py)",
       "launches": len(launches), "dram_bytes_per_launch": tot_dram / max(len(launches), 1),
       "dense_bytes_per_launch": tot_alg / max(len(launches), 1),
       "traffic_bytes_per_dense_byte": tot_dram / tot_alg, "by_plan_mode": by_mode}
json.dump(res, open("profiles/kcoop_traffic.json", "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "by_plan_mode"}, indent=1))
print(json.dumps(by_mode, indent=1))
