"""Times the W=20 warp-kernel shapes (FG_TSQR_W20 = base|warpb|warpc|cta)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import figaro as F
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((20_000_000, 20), dtype=torch.float64, device="cuda", generator=g)
for v in ["base", "warpb", "warpc", "cta"]:
    os.environ["FG_TSQR_W20"] = v
    F.tsqr([(x, 0)], 20); best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); R = F.tsqr([(x, 0)], 20)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    print(f"W20 {v:6s} {best*1e3:8.3f} ms {2*20e6*400/best/1e12:6.2f} TF/s R00={R[0,0].item():.9e}", flush=True)
