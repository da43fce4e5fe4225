"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
executed warp-instructions and stall samples per opcode class, plus the hottest lines.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/sass_hist.py src.csv [evals]
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
evals = float(sys.argv[2]) if len(sys.argv) > 2 else None
ops = defaultdict(lambda: [0, 0])
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stalls = defaultdict(float)
lines = []
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
    if not m:
        continue
    op = m.group(2)
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op][0] += n
    ops[op][1] += s
    tot_i += n
    tot_s += s
    for c in stall_cols:
        stalls[c] += float(r[ix[c]] or 0)
    lines.append((s, n, r[ix["Address"]][-5:], src))
print(f"total warp-instr {tot_i:.4g}  samples {tot_s}")
if evals:
    print(f"warp-instr per 32 evals: {tot_i / (evals / 32):.1f}")
print(f"{'op':10s} {'instr':>12s} {'%':>6s} {'per32':>8s} {'stall%':>7s}")
for op, (n, s) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:40]:
    per = n / (evals / 32) if evals else 0
    print(f"{op:10s} {n:12d} {100*n/tot_i:6.2f} {per:8.1f} {100*s/max(tot_s,1):7.2f}")
print("stalls:", {k[6:]: round(100 * v / tot_s, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]})
print("hottest:")
for s, n, a, src in sorted(lines, reverse=True)[:40]:
    print(f"  {s:7d} {n:10d} {a} {src}")
