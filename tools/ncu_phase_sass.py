"""Dynamic warp-instruction counts of one kernel from an ncu source-page CSV
(--print-source cuda,sass), split at the kernel's BAR.SYNC instructions
(address order) and by opcode class.  usage: python tools/ncu_phase_sass.py CSV"""
import csv, sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
ins = {}
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] or not r[2].startswith("0x"):
        continue
    d = dict(zip(hdr, r))
    addr = int(r[2], 16)
    ins[addr] = (r[3].strip(), int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0))
addrs = sorted(ins)
base = addrs[0]
tot = sum(v[1] for v in ins.values())
tots = sum(v[2] for v in ins.values())
phase = 0
ph = defaultdict(Counter)
phs = Counter()
bounds = []
for a in addrs:
    txt, n, s = ins[a]
    op = txt.split()[0]
    if op.startswith("@"):
        op = txt.split()[1]
    opc = op.split(".")[0]
    ph[phase][opc] += n
    phs[phase] += s
    if opc == "BAR":
        bounds.append(hex(a - base))
        phase += 1
print(f"total warp inst {tot:.4g}  samples {tots}  barriers at {bounds}")
for p in sorted(ph):
    c = ph[p]
    t = sum(c.values())
    top = ", ".join(f"{k} {v/t*100:.0f}%" for k, v in c.most_common(8))
    print(f"phase {p}: {t:.4g} inst ({t/tot*100:.1f}%), {phs[p]/max(tots,1)*100:.1f}% samples | {top}")

if len(sys.argv) > 2:  # extra split points (hex offsets)
    cuts = [int(x, 16) for x in sys.argv[2].split(",")]
    seg = Counter(); segc = defaultdict(Counter)
    for a in addrs:
        off = a - base
        k = sum(off >= c for c in cuts)
        txt, n, s = ins[a]
        op = txt.split()[1] if txt.startswith("@") else txt.split()[0]
        seg[k] += n; segc[k][op.split(".")[0]] += n
    for k in sorted(seg):
        lo = hex(cuts[k - 1]) if k else "0"
        top = ", ".join(f"{o} {v/seg[k]*100:.0f}%" for o, v in segc[k].most_common(6))
        print(f"from {lo}: {seg[k]:.4g} ({seg[k]/tot*100:.1f}%) | {top}")
