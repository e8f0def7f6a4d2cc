"""The multi-GPU flow with the device pipeline (one B200): every rank's shard
through run_pipeline (local_factor), the heavy-key stage and combination on
the device (heavy_stage / heavy_finish), and the fg_tsqr merge reproduce the
single-process R within 1e-10 -- ranks emulated one after another in one
process (no collective, so no kernel waits on another rank), and the real
torch.distributed flow with two gloo processes sharing the GPU."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2204_00525_b200 import distributed as D  # noqa: E402
from paper_2204_00525_b200 import figaro as F  # noqa: E402
from paper_2204_00525_b200 import workloads  # noqa: E402
from tests.helpers import r_distance  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def dev_rels(rels):
    return [F.Relation(r.name, r.key_attrs, r.data_attrs, torch.from_numpy(r.keys).cuda(),
                       torch.from_numpy(r.data).cuda()) for r in rels]


def single_R(db):
    rels = dev_rels(db.relations)
    tree = F.build_join_tree(rels, db.root, db.parent)
    return F.run_pipeline(rels, tree, F.PipelineOptions(assume_reduced=True),
                          fetch_counts=False).factor.r.cpu().numpy()


def emulate(db, P, **kw):
    """All P ranks of distributed_factor, one after another: shard, local
    factor, heavy stage; then the combination and the merge."""
    plan = D.plan_partition(db.relations, db.root, P, parent=db.parent, **kw)
    n = sum(len(r.data_attrs) for r in db.relations)
    red = plan.needs_reduction(db.relations)
    heavy = [D.heavy_rows(db.relations, plan, q) for q in range(P)] if plan.combine else None
    if heavy:
        cnts = np.stack([D.local_counts(h, plan) for h in heavy])
        g = cnts.sum(axis=0)
    locs, heads = [], []
    for q in range(P):
        shard = dev_rels(D.shard_relations(db.relations, plan, q, P))
        tree = F.build_join_tree(shard, db.root, db.parent)
        R = D.local_factor(shard, tree, n, assume_reduced=not red)
        if heavy:
            Rh, h = D.heavy_stage(heavy[q], plan, db.root, n, g)
            R = D.device_merge([R, Rh], n)
            heads.append(h)
        locs.append(R)
    if heavy:
        ws = [len(r.data_attrs) for r in db.relations]
        locs.append(D.heavy_finish(torch.stack(heads), cnts, plan, db.root, ws, n))
    return plan, D.device_merge(locs, n).cpu().numpy()


@pytest.mark.parametrize("cfg,scale,P", [("C5", 0.01, 8), ("C5", 0.02, 3), ("C2", 0.002, 4),
                                         ("C1", 0.2, 8), ("C3", 0.002, 8), ("C4", 0.01, 8),
                                         ("C4", 0.01, 6)])
def test_emulated_ranks_reproduce_single_process_R(cfg, scale, P):
    db = workloads.make(cfg, seed=9, scale=scale)
    plan, R = emulate(db, P, heavy_fraction=0.1)
    if cfg == "C5":
        assert plan.combine  # the heavy-key combination is exercised
    if cfg == "C3":
        assert plan.heavy  # sub-grid splits of heavy k1
    assert r_distance(R, single_R(db)) <= 1e-10


def test_every_key_heavy_and_empty_shards():
    """All keys combined (main shards empty on every rank) and more ranks
    than keys (empty heavy parts)."""
    db = workloads.make("C1", seed=4, scale=0.003)  # 3 keys x 10 rows
    plan, R = emulate(db, 8, combine_fraction=0.0)
    assert len(plan.combine) == 3
    assert r_distance(R, single_R(db)) <= 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, scale, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        db = workloads.make(cfg, seed=9, scale=scale)
        plan = D.plan_partition(db.relations, db.root, world, parent=db.parent)
        n = sum(len(r.data_attrs) for r in db.relations)
        shard = dev_rels(D.shard_relations(db.relations, plan, rank, world))
        tree = F.build_join_tree(shard, db.root, db.parent)
        heavy = D.heavy_rows(db.relations, plan, rank) if plan.combine else None
        R = D.distributed_factor(shard, heavy, tree, n, plan, db.root)
        out[rank] = R.cpu().numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,scale", [("C5", 0.01), ("C4", 0.01)])
def test_two_gloo_ranks_device_pipeline(cfg, scale):
    import torch.multiprocessing as mp
    db = workloads.make(cfg, seed=9, scale=scale)
    ref = single_R(db)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), cfg, scale, out), nprocs=2, join=True)
    for rank in range(2):
        assert r_distance(out[rank], ref) <= 1e-10
