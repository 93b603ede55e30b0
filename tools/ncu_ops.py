"""Opcode histogram of an ncu report weighted by executed warp instructions.
usage: python tools/ncu_ops.py REP [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; c = collections.Counter(); tot = 0
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r; continue
    if hdr is None or len(r) < 6:
        continue
    d = dict(zip(hdr, r))
    try:
        n = int(d["Instructions Executed"])
    except ValueError:
        continue
    src = d["Source"].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0] if src else "?"
    c[op] += n; tot += n
print(f"total {tot:.4g}")
for op, n in c.most_common(top):
    print(f"{op:28s} {n/tot*100:5.1f}%")
