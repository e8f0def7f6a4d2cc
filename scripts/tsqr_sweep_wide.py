"""Times the W=64 / W=128 TSQR CTA-kernel shapes (FG_TSQR_W64/W128 = base|a|b)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import figaro as F
g = torch.Generator(device="cuda").manual_seed(0)
x64 = torch.randn((8_000_000, 64), dtype=torch.float64, device="cuda", generator=g)
x128 = torch.randn((500_000, 128), dtype=torch.float64, device="cuda", generator=g)
def bench(blocks, n, reps=3):
    F.tsqr(blocks, n); best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); R = F.tsqr(blocks, n)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best, R
for v in ["base", "a", "b"]:
    os.environ["FG_TSQR_W64"] = v
    t, R = bench([(x64, 0)], 64)
    print(f"W64 {v:4s} {t*1e3:8.3f} ms {2*8e6*4096/t/1e12:6.2f} TF/s R00={R[0,0].item():.6e}", flush=True)
os.environ["FG_TSQR_W64"] = "base"
for v in ["base", "a", "b"]:
    os.environ["FG_TSQR_W128"] = v
    t, R = bench([(x128, 0)], 128)
    print(f"W128 {v:4s} {t*1e3:8.3f} ms {2*5e5*16384/t/1e12:6.2f} TF/s R00={R[0,0].item():.6e}", flush=True)
