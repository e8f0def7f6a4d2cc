import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_00525_b200 import fgdb
from paper_2204_00525_b200 import figaro as F
from oracle import figaro_np as fo
db = fgdb.read_fgdb("tests/golden/gt_512x16.fgdb")
rels = [F.Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(), torch.from_numpy(r.data).cuda()) for r in db.relations]
tree = F.build_join_tree(rels, db.root, db.parent)
res = F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=True), keep_r0=True)
R = res.factor.r.cpu().numpy()
print("R nan:", np.isnan(R).sum(), "r0_rows", res.r0_rows)
orels, root, parent = fo.from_fgdb(db)
ref = fo.run_pipeline(orels, root, parent)
for i, sp in enumerate(res.r0):
    print("span", i, sp.node, sp.col_begin, sp.rows.shape, "nan", np.isnan(sp.rows).sum())
dense = fo.dense_r0([fo.OutBlock(s.node, s.col_begin, s.rows) for s in res.r0], 32)
print("gram err", fo.rel_frobenius_distance(dense.T @ dense, fo.dense_r0(ref.r0, 32).T @ fo.dense_r0(ref.r0, 32)))
blocks = [(torch.from_numpy(np.ascontiguousarray(s.rows)).cuda(), s.col_begin) for s in res.r0]
R2 = F.tsqr(blocks, 32).cpu().numpy()
print("tsqr nan", np.isnan(R2).sum(), "err", fo.rel_frobenius_distance(R2, ref.R))
for var in ["warp", "warpb", "warpc", "cta"]:
    os.environ["FG_TSQR_W16"] = var
    for v32 in ["warp", "warpc", "cta"]:
        os.environ["FG_TSQR_W32"] = v32
        R3 = F.tsqr(blocks, 32).cpu().numpy()
        print(var, v32, "nan", np.isnan(R3).sum(), "err", fo.rel_frobenius_distance(R3, ref.R))
