"""Per-source-line instruction counts and stall samples from an ncu report.
usage: python tools/ncu_lines.py REP [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
res = []
tot_i = tot_s = 0
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        ins = int(d["Instructions Executed"]); smp = int(d["Warp Stall Sampling (All Samples)"])
    except ValueError:
        continue
    tot_i += ins; tot_s += smp
    res.append((ins, smp, r[0], r[1][:90]))
res.sort(key=lambda t: -t[0])
print(f"total warp inst {tot_i:.4g}, samples {tot_s}")
for ins, smp, ln, src in res[:top]:
    print(f"{ln:>5} {ins/tot_i*100:5.1f}% inst {smp/max(tot_s,1)*100:5.1f}% smp  {src}")
