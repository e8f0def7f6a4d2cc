"""Small driver for ncu captures: runs a config pipeline (scaled) a few times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_00525_b200 import workloads
from paper_2204_00525_b200.figaro import Relation, build_join_tree, run_pipeline, PipelineOptions
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
db = workloads.make(cfg, seed=7, scale=scale)
rels = [Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(),
                 torch.from_numpy(r.data).cuda()) for r in db.relations]
tree = build_join_tree(rels, db.root, db.parent)
for _ in range(reps):
    res = run_pipeline(rels, tree, PipelineOptions(assume_reduced=True), fetch_counts=False, fuse=os.environ.get("FUSE", "1") == "1")
torch.cuda.synchronize()
print("ok", cfg, scale, res.seconds_total)
