"""Per-line warp instructions, average active threads, grouped by line ranges.
usage: python tools/ncu_lines2.py REP lo-hi:name lo-hi:name ..."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; lines = {}; fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        lines[(fname, int(r[0]))] = (int(d["Instructions Executed"]), int(d["Thread Instructions Executed"]),
                            int(d["Warp Stall Sampling (All Samples)"]))
    except ValueError:
        pass
TI = sum(v[0] for v in lines.values()); TT = sum(v[1] for v in lines.values()); TS = sum(v[2] for v in lines.values())
print(f"warp inst {TI:.4g}  thread inst {TT:.4g}  avg threads {TT/TI:.1f}")
files = sorted({f for f, _ in lines})
for fn in files:
    sel = [v for (f, k), v in lines.items() if f == fn]
    print(f"  {fn}: {sum(v[0] for v in sel)/TI*100:.1f}% inst")
for spec in sys.argv[2:]:
    rng, name = spec.split(":")
    fn = ""
    if "@" in rng:
        fn, rng = rng.split("@")
    lo, hi = map(int, rng.split("-"))
    sel = [v for (f, k), v in lines.items() if lo <= k <= hi and (not fn or f.startswith(fn))]
    wi = sum(v[0] for v in sel); ti = sum(v[1] for v in sel); si = sum(v[2] for v in sel)
    print(f"{name:12s} {wi/TI*100:5.1f}% inst  {si/TS*100:5.1f}% smp  avg thr {ti/max(wi,1):.1f}")
