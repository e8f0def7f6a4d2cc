"""Per-kernel time table from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
runs = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', '')) * {'usecond': 1e3, 'msecond': 1e6, 'nsecond': 1}.get(r[ui], 1)
    agg[r[ki][:100]][0] += 1
    agg[r[ki][:100]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e6 / runs:.3f} ms per run ({runs:g} runs)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:18]:
    print(f"{t / 1e6 / runs:8.3f} ms/run {100 * t / tot:5.1f}% n={c:3d} {k}")
