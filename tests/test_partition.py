"""Host logic of the multi-GPU partition (paper_2204_00525_b200/distributed.py)
on CPU: plan shapes for the BASELINE configs, the join-partition property of
grid plans with heavy-value sub-grids (the shards' full join sizes add up to
the database's), row bookkeeping of the partial-head combination, R of the
merged per-shard factors (oracle per shard), and the combination identity
itself (its Gram equals the heavy keys' share of A^T A)."""
import numpy as np
import pytest

from oracle import figaro_np as fo
from paper_2204_00525_b200 import distributed as D
from paper_2204_00525_b200 import fgdb, workloads
from tests.conftest import golden
from tests.helpers import r_distance


def _oracle_fjs(rels, root, parent):
    rels = [fo.canonicalize(r) for r in rels]
    tree = fo.build_join_tree(rels, root, parent)
    try:
        red = fo.semi_join_reduce(rels, tree)
    except fo.empty_join_error:
        return 0
    return sum(fo.compute_counts(red, tree)[root].full_join_size.values())


def _oracle_R(rels, root, parent, n):
    try:
        return fo.run_pipeline(rels, root, parent, reduce=True).R
    except fo.empty_join_error:
        return np.zeros((n, n))


def test_plans_for_the_baseline_configs():
    c3 = workloads.make("C3", seed=3, scale=0.002)
    p = D.plan_partition(c3.relations, c3.root, 8, parent=c3.parent)
    assert p.attrs == ["k1"] and p.dims == [8] and not p.combine
    assert p.heavy and all(h.extents[1] == 8 and h.extents[0] == 1 for h in p.heavy)  # F split, D1 whole
    c4 = workloads.make("C4", seed=3, scale=0.01)
    p = D.plan_partition(c4.relations, c4.root, 8, parent=c4.parent)
    assert p.attrs == ["a", "b"] and sorted(p.dims) == [2, 4]  # R3 not replicated 8 times
    assert p.needs_reduction(c4.relations)
    c5 = workloads.make("C5", seed=3, scale=0.01)
    p = D.plan_partition(c5.relations, c5.root, 8, parent=c5.parent)
    assert p.attrs == ["k"] and p.combine and not p.heavy
    assert not p.needs_reduction(c5.relations)
    c2 = workloads.make("C2", seed=3, scale=0.001)
    p = D.plan_partition(c2.relations, c2.root, 8, parent=c2.parent)
    assert p.attrs == ["k"] and not p.combine and not p.heavy  # uniform keys
    assert D.plan_partition(c2.relations, c2.root, 1).attrs == []


@pytest.mark.parametrize("src", ["hand_four", "rnd_3", "big_101", "cfg:C3", "cfg:C4"])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_grid_shards_partition_the_join(src, P):
    db = workloads.make(src[4:], seed=5, scale=0.002) if src.startswith("cfg:") \
        else fgdb.read_fgdb(golden(src + ".fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    # a low threshold forces heavy-value sub-grids on these small inputs
    plan = D.plan_partition(rels, root, P, heavy_fraction=0.05)
    total = _oracle_fjs(rels, root, parent)
    got = sum(_oracle_fjs(D.shard_relations(rels, plan, q, P), root, parent) for q in range(P))
    assert got == total


@pytest.mark.parametrize("src", ["cfg:C4", "cfg:C3", "rnd_7"])
def test_grid_shards_merge_to_the_full_R(src):
    db = workloads.make(src[4:], seed=5, scale=0.002) if src.startswith("cfg:") \
        else fgdb.read_fgdb(golden(src + ".fgdb"))
    rels, root, parent = fo.from_fgdb(db)
    n = sum(len(r.data_attrs) for r in rels)
    full = fo.run_pipeline(rels, root, parent, reduce=True).R
    P = 4
    plan = D.plan_partition(rels, root, P, heavy_fraction=0.05)
    parts = [_oracle_R(D.shard_relations(rels, plan, q, P), root, parent, n) for q in range(P)]
    merged = fo.normalize_signs(fo.householder_r(np.vstack(parts)))
    assert r_distance(merged, full) <= 1e-10


@pytest.mark.parametrize("P", [2, 3, 8])
def test_combine_rows_are_split_exactly_once(P):
    db = workloads.make("C5", seed=5, scale=0.003)
    rels, root, parent = fo.from_fgdb(db)
    plan = D.plan_partition(rels, root, P, parent=parent)
    assert plan.combine
    comb = set(plan.combine)
    for ri, r in enumerate(rels):
        main = sum(D.shard_relations(rels, plan, q, P)[ri].rows for q in range(P))
        heavy = [D.heavy_rows(rels, plan, q)[ri] for q in range(P)]
        hv = sum(h[0].shape[0] for h in heavy)
        assert main + hv == r.rows
        assert hv == int(np.isin(r.keys[:, 0], list(comb)).sum())
        # each key's rows are dealt round-robin: per-rank counts differ by <= 1
        cnt = np.stack([np.bincount(h[0], minlength=len(comb)) for h in heavy])
        assert (cnt.max(axis=0) - cnt.min(axis=0) <= 1).all()


def test_combination_identity_on_cpu():
    """The heavy-key path in numpy (oracle transforms): per-rank heads/tails
    of each key's part, then the generalized transform of the partial heads
    and the root row -- their Gram plus the main shards' equals A^T A."""
    db = workloads.config_c5(seed=5, scale=0.002, cols=6)
    rels, root, parent = fo.from_fgdb(db)
    n = sum(len(r.data_attrs) for r in rels)
    P = 3
    plan = D.plan_partition(rels, root, P, parent=parent)
    assert plan.combine
    rows = []
    for q in range(P):
        rows.append(_oracle_R(D.shard_relations(rels, plan, q, P), root, parent, n))
    H = len(plan.combine)
    parts = [D.heavy_rows(rels, plan, q) for q in range(P)]
    g = sum(D.local_counts(pt, plan) for pt in parts)
    ws = [len(r.data_attrs) for r in rels]
    off = [0, ws[0]]
    heads = {}
    for q in range(P):
        for j in range(2):
            kidx, data = parts[q][j]
            for k in range(H):
                grp = data[kidx == k]
                heads[q, k, j] = (fo.head(grp), grp.shape[0]) if grp.shape[0] else (None, 0)
                if grp.shape[0] > 1:
                    t = fo.tail(grp) * np.sqrt(g[k, 1 - j])
                    blk = np.zeros((t.shape[0], n))
                    blk[:, off[j]:off[j] + ws[j]] = t
                    rows.append(blk)
    for k in range(H):
        comb = []
        for j in range(2):
            st = [(h, m) for h, m in (heads[q, k, j] for q in range(P)) if m]
            a = np.vstack([h for h, _ in st])
            v = [np.sqrt(m) for _, m in st]
            comb.append(fo.generalized_head(a, v))
            if len(st) > 1:
                t = fo.generalized_tail(a, v) * np.sqrt(g[k, 1 - j])
                blk = np.zeros((t.shape[0], n))
                blk[:, off[j]:off[j] + ws[j]] = t
                rows.append(blk)
        rows.append(np.concatenate([comb[0] * np.sqrt(g[k, 1]), comb[1] * np.sqrt(g[k, 0])])[None])
    merged = fo.normalize_signs(fo.householder_r(np.vstack(rows)))
    full = fo.run_pipeline(rels, root, parent, reduce=True).R
    assert r_distance(merged, full) <= 1e-10
