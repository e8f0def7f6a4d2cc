"""Blocked (DMMA) TSQR vs the column-by-column kernels: accuracy against
numpy on small inputs (incl. scaled / rank-deficient columns and column
offsets) and timing on C5-sized W=64 and C2-sized W=32 inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_00525_b200 import figaro as F


def ref_r(a):
    r = np.linalg.qr(a, mode="r")
    s = np.sign(np.diag(r)); s[s == 0] = 1
    return r * s[:, None]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


rng = np.random.default_rng(1)
for W, var_env in [(64, "FG_TSQR_W64"), (32, "FG_TSQR_W32")]:
    for v in ["blk", "blk64"]:
        os.environ[var_env] = v
        worst = 0.0
        for trial in range(6):
            m = [1, 7, 130, 1000, 5000, 20000][trial]
            a = rng.standard_normal((m, W)) * rng.uniform(1e-3, 1e3, size=W)
            if trial == 3:
                a[:, 5] = a[:, 3] * 2.0  # rank deficient
            R = F.tsqr([(torch.from_numpy(a).cuda(), 0)], W).cpu().numpy()
            if trial == 3:
                d = rel(R.T @ R, a.T @ a)
            else:
                d = rel(R, ref_r(a) if m >= W else ref_r(np.vstack([a, np.zeros((W - m, W))])))
            worst = max(worst, d)
        # two spans at column offsets
        a1 = rng.standard_normal((3000, W // 2)); a2 = rng.standard_normal((2000, W - W // 2))
        R = F.tsqr([(torch.from_numpy(a1).cuda(), 0), (torch.from_numpy(a2).cuda(), W // 2)], W).cpu().numpy()
        dense = np.zeros((5000, W)); dense[:3000, :W // 2] = a1; dense[3000:, W // 2:] = a2
        worst = max(worst, rel(R, ref_r(dense)))
        print(f"W{W} {v:6s} worst rel err {worst:.3e}", flush=True)

g = torch.Generator(device="cuda").manual_seed(0)
x64 = torch.randn((8_000_000, 64), dtype=torch.float64, device="cuda", generator=g)
x32 = torch.randn((1_000_000, 32), dtype=torch.float64, device="cuda", generator=g)


def bench(blocks, n, reps=3):
    F.tsqr(blocks, n); best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); R = F.tsqr(blocks, n)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best, R


for v in ["base", "blk", "blk64"]:
    os.environ["FG_TSQR_W64"] = v
    t, R = bench([(x64, 0)], 64)
    print(f"W64 {v:6s} {t*1e3:8.3f} ms {2*8e6*4096/t/1e12:6.2f} TF/s R00={R[0,0].item():.9e}", flush=True)
for v in ["cta", "blk", "blk64"]:
    os.environ["FG_TSQR_W32"] = v
    t, R = bench([(x32, 0)], 32)
    print(f"W32 {v:6s} {t*1e3:8.3f} ms {2*1e6*1024/t/1e12:6.2f} TF/s R00={R[0,0].item():.9e}", flush=True)
