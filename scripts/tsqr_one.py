"""One TSQR call (for ncu): python scripts/tsqr_one.py W ROWS [reps] [variant]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import figaro as F
W, rows = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if len(sys.argv) > 4:
    os.environ[f"FG_TSQR_W{W}"] = sys.argv[4]
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((rows, W), dtype=torch.float64, device="cuda", generator=g)
for _ in range(reps):
    R = F.tsqr([(x, 0)], W)
torch.cuda.synchronize()
print("ok", R[0, 0].item())
