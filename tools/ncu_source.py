"""Per-source-line hot spots of an ncu report (needs -lineinfo + --import-source on).

usage: python tools/ncu_source.py <report.ncu-rep> [top]
Prints the lines with the most warp-stall samples and the most executed warp
instructions, per source file.
"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows, fname, hdr = [], "?", None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        stalls = {h[6:]: int(v) for h, v in zip(hdr, r)
                  if h.startswith("stall_") and "Not Issued" not in h and v.isdigit() and int(v)}
        rows.append((fname, int(r[0]), r[1].strip()[:90], samples, inst, stalls))
    tot_s = sum(x[3] for x in rows) or 1
    tot_i = sum(x[4] for x in rows) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for key, label, tot in ((3, "samples", tot_s), (4, "instructions", tot_i)):
        print(f"--- top lines by {label}")
        for f, ln, src, s, i, st in sorted(rows, key=lambda x: -x[key])[:top]:
            print(f"{100.0 * (s if key == 3 else i) / tot:5.1f}%  {f}:{ln:<4d} {src}")
            if key == 3 and s:
                print("         " + " ".join(f"{k}={100.0 * v / s:.0f}%" for k, v in
                                          sorted(st.items(), key=lambda kv: -kv[1])[:4]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
