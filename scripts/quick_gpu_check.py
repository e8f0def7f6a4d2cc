"""Ad-hoc GPU check: random reference databases + small configs vs oracle/_ref."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2204_00525_b200 import fgdb, workloads
from paper_2204_00525_b200.figaro import Relation, build_join_tree, run_pipeline, PipelineOptions
from oracle import figaro_np as fo

REF = 'oracle/_ref/figaro_ref'

def cmp(db, tag, tol=1e-10):
    path = f'/tmp/{tag}.fgdb'
    fgdb.write_fgdb(path, db)
    subprocess.run([REF, 'run', path, path + '.rs'], check=True, capture_output=True)
    ref = fgdb.read_fgrs(path + '.rs')
    rels = [Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in db.relations]
    tree = build_join_tree(rels, db.root, db.parent)
    t = time.time()
    res = run_pipeline(rels, tree, PipelineOptions(assume_reduced=True))
    dt = time.time() - t
    R = res.factor.r
    full_rank = np.all(np.abs(np.diag(ref.R)) > 1e-8 * np.abs(ref.R).max()) if ref.R.size else True
    if full_rank:
        err = fo.rel_frobenius_distance(R, ref.R)
    else:
        err = fo.rel_frobenius_distance(R.T @ R, ref.R.T @ ref.R)
    ok_counts = True
    for i, nc in enumerate(ref.nodes):
        c = res.counts[i]
        ok_counts &= np.array_equal(c.group_begin.astype(np.uint64), nc.group_begin)
        ok_counts &= np.array_equal(c.rows_per_key, nc.rows_per_key)
        ok_counts &= np.array_equal(c.theta_down, nc.theta_down)
        ok_counts &= np.array_equal(c.full_join_size, nc.full_join_size)
        ok_counts &= np.array_equal(c.phi_circ, nc.phi_circ)
        ok_counts &= np.array_equal(c.phi_down, nc.phi_down)
        ok_counts &= np.array_equal(c.phi_up, nc.phi_up)
        ok_counts &= np.array_equal(c.keys, nc.keys)
        ok_counts &= np.array_equal(c.parent_keys, nc.pkeys)
    good = err <= tol and ok_counts and res.r0_rows == ref.r0_rows
    print(f"{tag}: err={err:.2e} counts={'ok' if ok_counts else 'BAD'} r0 {res.r0_rows}/{ref.r0_rows} "
          f"fullrank={full_rank} t={dt*1e3:.1f}ms gpu_total={res.seconds_total*1e3:.2f}ms "
          f"{'OK' if good else 'FAIL'}", flush=True)
    return good

bad = 0
for seed in range(1, 41):
    subprocess.run([REF, 'random', str(seed), '/tmp/rnd.fgdb'], check=True, capture_output=True)
    bad += not cmp(fgdb.read_fgdb('/tmp/rnd.fgdb'), f'rnd{seed}')
for seed in range(100, 110):
    subprocess.run([REF, 'random', str(seed), '/tmp/rnd.fgdb', '--max-rows', '3000', '--max-rel', '6',
                    '--key-domain', '40', '--max-cols', '12'], check=True, capture_output=True)
    bad += not cmp(fgdb.read_fgdb('/tmp/rnd.fgdb'), f'big{seed}')
for cfg, sc in [('C1', 1.0), ('C2', 0.01), ('C4', 0.01), ('C5', 0.002), ('C3', 0.001)]:
    bad += not cmp(workloads.make(cfg, seed=7, scale=sc), f'{cfg}_{sc}')
print("FAILURES", bad)
