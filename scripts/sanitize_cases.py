"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck):
every BASELINE config at reduced scale through run_pipeline (fused and
unfused own tails), the K1 sort at onesweep tile edges, and the phase
kernels.  Run with FG_EXACT_ALLOC=1 so every buffer is its own allocation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_00525_b200 import figaro as F, workloads

cases = [("C1", 0.05), ("C2", 0.002), ("C3", 0.001), ("C4", 0.005), ("C5", 0.003)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
for cfg, scale in cases:
    db = workloads.make(cfg, seed=11, scale=scale)
    rels = [F.Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(),
                       torch.from_numpy(r.data).cuda()) for r in db.relations]
    tree = F.build_join_tree(rels, db.root, db.parent)
    for fuse in (True, False):
        res = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=False), fuse=fuse)
        torch.cuda.synchronize()
        print(cfg, scale, "fuse" if fuse else "nofuse", "rows", res.input_rows, "ok", flush=True)
rng = np.random.default_rng(3)
for n, bits in [(4097, 33), (6145, 20), (12289, 9), (100_000, 47), (1, 0), (5000, 64)]:
    keys = rng.integers(0, 1 << min(bits, 62), n, dtype=np.int64) if bits else np.zeros(n, np.int64)
    F.group_keys(torch.from_numpy(keys).cuda(), bits)
    print("group_keys", n, bits, "ok", flush=True)
data = torch.randn(3000, 20, dtype=torch.float64, device="cuda")
begins = torch.tensor([0, 1, 700, 701, 2999, 3000], dtype=torch.int32, device="cuda")
F.heads_tails(data, begins)
F.heads_tails(data, begins, weights=torch.rand(3000, dtype=torch.float64, device="cuda") + 0.5)
for w in (8, 20, 40, 64, 128):
    x = torch.randn(5000, w, dtype=torch.float64, device="cuda")
    F.tsqr([(x, 0)], w)
torch.cuda.synchronize()
print("sanitize cases done")
