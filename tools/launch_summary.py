"""Summarise an ncu --metrics gpu__time_duration.sum launch list: time per kernel family."""
import csv, sys
from collections import defaultdict

def load(path, limit=None):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d['Kernel Name'], d['Grid Size'], d['Block Size'], float(d['Metric Value'])))
    return out[:limit] if limit else out

def family(name):
    n = name.split('(')[0].replace('void ', '')
    if 'ntt_cl8' in name:
        import re
        m = re.search(r'ntt_cl8<(\d), (\d+), ([^,]+), (.+)>\(', name)
        if m:
            return f"ntt_cl8 inv={m.group(1)} logC={m.group(2)} {m.group(3).split('::')[-1]}/{m.group(4).split('::')[-1]}"
        return 'ntt_cl8'
    for k in ('ntt_pass', 'k_tensor_sum', 'k_conv_mac', 'k_ks_inner', 'k_tensor', 'k_binop', 'k_mul_scalar', 'k_add_const',
              'k_copy_limbs', 'k_encode', 'k_decode', 'k_enc', 'k_mul_plain'):
        if k in n:
            if k == 'ntt_pass':
                import re
                m = re.search(r'ntt_pass<(\d), (\d), (\d+), (\d), ([^,]+), (.+)>\(', name)
                if m:
                    ld = m.group(5).split('::')[-1]
                    st = m.group(6).split('::')[-1]
                    return f"ntt_pass inv={m.group(1)} cols={m.group(2)} logT={m.group(3)} ept={1 << int(m.group(4))} {ld}/{st}"
                return k
            return k
    return n[-40:]

if __name__ == '__main__':
    out = load(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
    agg = defaultdict(lambda: [0, 0.0])
    for name, g, b, ns in out:
        f = family(name); agg[f][0] += 1; agg[f][1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"{len(out)} launches, {tot/1e6:.3f} ms serialised")
    for f, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{ns/1e6:9.3f} ms {100*ns/tot:5.1f}%  n={n:5d}  avg {ns/n/1e3:8.2f} us  {f}")
