"""The N>1 path on CPU (world_size 2, gloo): key-hash sharding, per-rank R,
all_gather of the factors and the final merge reproduce the single-process R.
The per-rank factor here comes from the oracle (the checker); on B200 ranks the
same host logic runs the device pipeline and fg_tsqr for the merge."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import figaro_np as fo
from paper_2204_00525_b200 import distributed as D
from paper_2204_00525_b200 import fgdb, workloads
from tests.conftest import golden
from tests.helpers import r_distance


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_R(rels, root, parent, n):
    try:
        return fo.run_pipeline(rels, root, parent, reduce=True).R
    except fo.empty_join_error:
        return np.zeros((n, n))


def oracle_merge(parts, n):
    return torch.from_numpy(fo.normalize_signs(fo.householder_r(
        np.vstack([p.numpy() for p in parts]))))


def _worker(rank, world, port, stem, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if stem.startswith("cfg:"):
            db = workloads.make(stem[4:], seed=5, scale=0.002)
        else:
            db = fgdb.read_fgdb(golden(stem + ".fgdb"))
        rels, root, parent = fo.from_fgdb(db)
        attr = D.partition_attribute(rels, root)
        shard = D.shard_relations(rels, attr, rank, world)
        n = sum(len(r.data_attrs) for r in rels)
        Rp = torch.from_numpy(np.ascontiguousarray(oracle_R(shard, root, parent, n)))
        R = D.gather_and_merge(Rp, oracle_merge)
        results[rank] = R.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stem", ["hand_four", "hand_st", "rnd_3", "rnd_7", "big_101",
                                  "cfg:C1", "cfg:C4", "cfg:C3"])
def test_two_rank_shards_reproduce_single_process_R(stem):
    if stem.startswith("cfg:"):
        db = workloads.make(stem[4:], seed=5, scale=0.002)
    else:
        db = fgdb.read_fgdb(golden(stem + ".fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    full = fo.run_pipeline(rels, root, parent, reduce=True).R
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), stem, results), nprocs=2, join=True)
    for rank in range(2):
        assert r_distance(results[rank], full) <= 1e-10


def test_sharding_partitions_the_join():
    db = fgdb.read_fgdb(golden("hand_four.fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    attr = D.partition_attribute(rels, root)
    assert attr in rels[root].key_attrs
    total = 0
    for rank in range(3):
        shard = D.shard_relations(rels, attr, rank, 3)
        for r, s in zip(rels, shard):
            if attr not in r.key_attrs:
                assert s.rows == r.rows  # replicated
        tree = fo.build_join_tree(shard, root, parent)
        try:
            red = fo.semi_join_reduce(shard, tree)
        except fo.empty_join_error:
            continue
        counts = fo.compute_counts(red, tree)
        total += sum(counts[root].full_join_size.values())
    tree = fo.build_join_tree(rels, root, parent)
    assert total == sum(fo.compute_counts(rels, tree)[root].full_join_size.values())
