"""Per-kernel summary of an ncu --page raw --csv dump: duration, IPC, occupancy, pipes, top stall reasons."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
stalls = [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
pipes = [h for h in hdr if h.startswith('sm__inst_executed_pipe_') and h.endswith('.avg.pct_of_peak_sustained_active')]
def g(d, k):
    try: return float(d[k])
    except Exception: return float('nan')
for r in rows[2:]:
    d = dict(zip(hdr, r))
    v = d['Kernel Name']
    m = re.search(r'ntt_pass<(\d), (\d), (\d+), (\d)', v); m2 = re.search(r'ntt_cl8<(\d), (\d+)', v)
    name = f"ntt_pass inv{m.group(1)} cols{m.group(2)} logT{m.group(3)} le{m.group(4)}" if m else (f"ntt_cl8 inv{m2.group(1)}" if m2 else v[:50])
    print(f"{name}: {g(d,'gpu__time_duration.sum')/1e3:.1f} us grid {d['launch__grid_size']}x{d['launch__block_size']} regs {d['launch__registers_per_thread']} "
          f"occ {g(d,'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}% ipc {g(d,'sm__inst_executed.avg.per_cycle_active'):.2f} "
          f"dram {(g(d,'dram__bytes_read.sum')+g(d,'dram__bytes_write.sum'))/1e6:.1f} MB inst {g(d,'smsp__inst_executed.sum')/1e6:.2f} M")
    st = sorted(((g(d, h), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')) for h in stalls), reverse=True)[:6]
    print('   stalls', [(n, round(x, 2)) for x, n in st])
    pp = sorted(((g(d, h), h.replace('sm__inst_executed_pipe_', '').replace('.avg.pct_of_peak_sustained_active', '')) for h in pipes), reverse=True)[:5]
    print('   pipes', [(n, round(x, 1)) for x, n in pp])
