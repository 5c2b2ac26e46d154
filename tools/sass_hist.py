"""Histogram of an ncu --page source --print-source sass CSV: executed instructions and stall samples by opcode."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE, iA = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex, st = defaultdict(int), defaultdict(int)
tot_e = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr) - 2 or not r[iE].isdigit(): continue
    op = r[iS].split()[0] if r[iS].split() else "?"
    if op.startswith("@"): op = r[iS].split()[1]
    op = op.split(".")[0]
    e, s = int(r[iE] or 0), int(r[iA] or 0)
    ex[op] += e; st[op] += s; tot_e += e; tot_s += s
print(f"total warp instr {tot_e}, samples {tot_s}")
for op in sorted(ex, key=lambda o: -ex[o])[:30]:
    print(f"{op:12s} {ex[op]:10d} {100*ex[op]/tot_e:5.1f}%  stall {100*st[op]/max(tot_s,1):5.1f}%")
