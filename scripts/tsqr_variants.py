"""Checks and times TSQR kernel variants against each other and numpy
(variants per width: warp | warpc | cta | lab | lat, see tsqr.cu variant()).

python scripts/tsqr_variants.py W ROWS VAR[,VAR...] [reps]
Env var FG_TSQR_W<W> selects the variant ('' = default).  Prints time, TF/s
(2 m W^2) and the relative Frobenius distance of R to the default variant and
to numpy's QR of a 200k-row prefix problem.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_00525_b200 import figaro as F

W, rows = int(sys.argv[1]), int(sys.argv[2])
variants = sys.argv[3].split(",")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
key = f"FG_TSQR_W{W}"
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((rows, W), dtype=torch.float64, device="cuda", generator=g)
scale = torch.logspace(-3, 3, W, dtype=torch.float64, device="cuda")
xs = x * scale


def setv(v):
    if v:
        os.environ[key] = v
    else:
        os.environ.pop(key, None)


def rel(a, b):
    return (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()


small = xs[:200_000].contiguous()
ref_small = torch.from_numpy(np.linalg.qr(small.cpu().numpy(), mode="r")).cuda()
ref_small = ref_small * torch.where(torch.diagonal(ref_small) < 0, -1.0, 1.0)[:, None]
# rank-deficient case: duplicated and zero columns
rd = small.clone()
rd[:, 1] = rd[:, 0]
rd[:, W // 2] = 0.0
ref_rd = torch.from_numpy(np.linalg.qr(rd.cpu().numpy(), mode="r")).cuda()
ref_rd = ref_rd * torch.where(torch.diagonal(ref_rd) < 0, -1.0, 1.0)[:, None]

setv("")
base = F.tsqr([(xs, 0)], W)
for v in variants:
    setv("" if v == "default" else v)
    R = F.tsqr([(xs, 0)], W)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        R = F.tsqr([(xs, 0)], W)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    e_base = rel(R, base)
    e_np = rel(F.tsqr([(small, 0)], W), ref_small)
    # Gram check for the rank-deficient case (R not unique there)
    Rr = F.tsqr([(rd, 0)], W)
    e_rd = rel(Rr.T @ Rr, ref_rd.T @ ref_rd)
    fl = 2.0 * rows * W * W
    print(f"W{W} {v:8s} {best*1e3:8.3f} ms {fl/best/1e12:6.2f} TF/s  vs_default {e_base:.2e}  "
          f"vs_numpy {e_np:.2e}  rankdef_gram {e_rd:.2e}", flush=True)
setv("")
