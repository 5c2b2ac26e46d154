"""Top stall-sampled SASS lines of the first kernel in an ncu --page source --print-source sass CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None; cur = []; kern = None; blocks = []
for r in rows:
    if r and r[0] == 'Kernel Name':
        if cur: blocks.append((kern, hdr, cur))
        kern = r[1]; cur = []; continue
    if r and r[0] == 'Address': hdr = r; continue
    if hdr and len(r) == len(hdr): cur.append(r)
if cur: blocks.append((kern, hdr, cur))
kern, hdr, lines = blocks[0]
iS, iA, iE = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
tot = sum(int(r[iA] or 0) for r in lines)
print(kern[:100], 'samples', tot, 'lines', len(lines))
# cumulative by window of 8 instructions to find hot regions
for i, r in sorted(enumerate(lines), key=lambda x: -int(x[1][iA] or 0))[:n]:
    print(f"{int(r[iA]):5d} {100*int(r[iA])/tot:5.1f}% @{i:5d} x{r[iE]:>8s}  {r[iS][:80]}")
