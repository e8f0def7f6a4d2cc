"""Per-CUDA-line stall samples and executed instructions from
`ncu -i rep --page source --csv --print-source cuda,sass [--kernel-id ...]`."""
import csv, os, sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
out, cur, h = [], "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = os.path.basename(r[1])
    elif r[0] == "Line No":
        h = r
    elif h and r[0].isdigit() and len(r) == len(h):
        out.append((cur, r[0], r[1], num(r[h.index("Warp Stall Sampling (All Samples)")]),
                    num(r[h.index("Instructions Executed")])))
tot = sum(x[3] for x in out) or 1
toti = sum(x[4] for x in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for fn, ln, src, s, i in sorted(out, key=lambda x: -x[3])[:n]:
    print(f"{100 * s / tot:5.1f}% stall {100 * i / toti:5.1f}% inst {fn}:{ln}: {src.strip()[:80]}")
