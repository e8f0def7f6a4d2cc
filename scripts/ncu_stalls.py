"""Summarise an `ncu --page source --csv` dump: stall reasons and hot SASS."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith('0x')]
si = h.index('Source'); wi = h.index('Warp Stall Sampling (All Samples)')
f = lambda x: float(x) if x not in ('', '-') else 0.0
tot = sum(f(r[wi]) for r in data) or 1
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
rs = {c: sum(f(r[h.index(c)]) for r in data) for c in reasons}
print("stall reasons:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:8]))
agg = collections.Counter()
for r in data:
    t = r[si].split()
    op = t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '?')
    agg[op.split('.')[0]] += f(r[wi])
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in agg.most_common(12)))
ii = h.index('Instructions Executed')
ops = collections.Counter()
for r in data:
    t = r[si].split()
    op = t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '?')
    ops[op.split('.')[0]] += f(r[ii])
tot_i = sum(ops.values()) or 1
print("executed mix:", ", ".join(f"{k} {100*v/tot_i:.1f}%" for k, v in ops.most_common(14)))
