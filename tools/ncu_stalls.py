"""Stall-reason totals (all samples) and per-line top stalls of one ncu report.
usage: python tools/ncu_stalls.py REP [min_samples]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
mins = int(sys.argv[2]) if len(sys.argv) > 2 else 400
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None; fname = ""; tot = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].rsplit("/", 1)[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if not hdr or not r or not r[0].isdigit() or len(r) < 8:
        continue
    d = dict(zip(hdr, r))
    st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "(Not" not in k and v.isdigit() and int(v)}
    for k, v in st.items():
        tot[k] = tot.get(k, 0) + v
    if sum(st.values()) >= mins:
        print(f"{fname}:{r[0]:>5} {r[1][:56]:56s}", sorted(st.items(), key=lambda t: -t[1])[:4])
T = sum(tot.values())
print("total:", ", ".join(f"{k} {v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda t: -t[1])[:10]))
