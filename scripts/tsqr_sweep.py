"""Times the TSQR variants (FG_TSQR_W16 / FG_TSQR_W32) on C2-shaped spans."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import figaro as F

g = torch.Generator(device="cuda").manual_seed(0)
x16 = torch.randn((15_000_000, 16), dtype=torch.float64, device="cuda", generator=g)
x32 = torch.randn((1_000_000, 32), dtype=torch.float64, device="cuda", generator=g)
x64 = torch.randn((8_000_000, 64), dtype=torch.float64, device="cuda", generator=g)

def bench(blocks, n, reps=5):
    F.tsqr(blocks, n)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        R = F.tsqr(blocks, n)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best, R

for var in ["warpc", "warpg", "warpe"]:
    os.environ["FG_TSQR_W16"] = var
    t, R = bench([(x16, 0)], 16)
    fl = 2 * 15e6 * 256
    print(f"W16 {var:6s} {t*1e3:8.3f} ms  {fl/t/1e12:6.2f} TF/s  R00={R[0,0].item():.6e}", flush=True)
for var in ["warp", "warpc", "cta"]:
    os.environ["FG_TSQR_W32"] = var
    t, R = bench([(x32, 0)], 32)
    fl = 2 * 1e6 * 1024
    print(f"W32 {var:6s} {t*1e3:8.3f} ms  {fl/t/1e12:6.2f} TF/s  R00={R[0,0].item():.6e}", flush=True)
t, R = bench([(x64, 0)], 64, reps=3)
print(f"W64 cta    {t*1e3:8.3f} ms  {2*8e6*4096/t/1e12:6.2f} TF/s", flush=True)
