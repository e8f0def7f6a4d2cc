"""Times K1 (fg_group_keys: radix sort + segment extraction) on n random keys
of `bits` bits, CUDA events, median of reps.  Usage: sort_bench.py n bits [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import figaro as F

n = int(float(sys.argv[1])); bits = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(1)
keys = torch.randint(0, 1 << min(bits, 62), (n,), device="cuda", dtype=torch.int64, generator=g)
ts = []
for i in range(reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); F.group_keys(keys, bits); e1.record(); torch.cuda.synchronize()
    if i >= 2: ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
print(f"sort n={n} bits={bits} rank={os.environ.get('FG_SORT_RANK','ballot')} lb={os.environ.get('FG_SORT_LB','4')} "
      f"ms={ms:.3f} keys/s={n / ms / 1e6:.2f}G")
