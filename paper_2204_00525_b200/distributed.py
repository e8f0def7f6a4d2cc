"""Multi-GPU data parallelism for the FiGaRo path: key-hash sharding and the
R gather.  The reference is single-process; this is the B200
addition of SURVEY 8(e).

Sharding rule.  Pick one join attribute `a` (partition_attribute).  Every
relation that has `a` keeps only the rows whose hash(a) falls in this rank's
bucket; every relation without `a` is replicated.  Each join tuple has exactly
one a-value, so the shard joins partition the full join:
    A = [A_0; A_1; ...; A_{P-1}]  (up to row order)
and therefore R(A) = R([R(A_0); ...; R(A_{P-1})]).  Each rank runs the whole
device pipeline on its shard (with semi-join reduction, since replicated
relations may dangle), the P factors are all-gathered over NCCL
(torch.distributed), and one more device TSQR merges them.  For 2-relation
same-key trees (C1, C2, C5) nothing is replicated and no data-path
collective is needed before the final gather.
"""
from __future__ import annotations

from collections import Counter
from typing import Callable, List, Optional, Sequence

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def key_hash(values: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of int64 key values (deterministic across ranks)."""
    with np.errstate(over="ignore"):
        z = values.astype(np.int64).view(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def partition_attribute(relations: Sequence, root: int) -> Optional[str]:
    """The key attribute held by the most relations (ties: one of the root's,
    then the most rows); None when no relation has a key."""
    cnt = Counter(a for r in relations for a in r.key_attrs)
    if not cnt:
        return None
    root_attrs = set(relations[root].key_attrs)

    def score(a):
        rows = sum(r.keys.shape[0] for r in relations if a in r.key_attrs)
        return (cnt[a], a in root_attrs, rows, a)

    return max(cnt, key=score)


def shard_relations(relations: Sequence, attr: Optional[str], rank: int, world: int,
                    make=None) -> List:
    """Rank `rank`'s shard (host numpy relations).  `make(rel, keys, data)`
    builds the output relation (default: same class, same names)."""
    out = []
    for r in relations:
        keys, data = np.asarray(r.keys), np.asarray(r.data)
        if world > 1 and attr is not None and attr in r.key_attrs:
            col = r.key_attrs.index(attr)
            mask = (key_hash(keys[:, col]) % np.uint64(world)) == np.uint64(rank)
            keys, data = keys[mask], data[mask]
        if make is None:
            out.append(type(r)(r.name, list(r.key_attrs), list(r.data_attrs),
                               np.ascontiguousarray(keys), np.ascontiguousarray(data)))
        else:
            out.append(make(r, keys, data))
    return out


def replicated(relations: Sequence, attr: Optional[str]) -> List[str]:
    return [r.name for r in relations if attr is None or attr not in r.key_attrs]


def gather_and_merge(R_local, merge: Callable[[list, int], object], group=None):
    """All-gathers the per-rank N x N factors and merges them into the global
    R with `merge(list_of_factors, n)` (the device TSQR in production)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return merge([R_local], R_local.shape[0])
    parts = [torch.empty_like(R_local) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, R_local.contiguous(), group=group)
    return merge(parts, R_local.shape[0])


def device_merge(parts, n: int, device: int = 0):
    """Merge on the GPU: TSQR of the stacked factors (fg_tsqr)."""
    from .figaro import tsqr
    return tsqr([(p, 0) for p in parts], n, device=device)


def weak_shard(db, rank: int, world: int):
    """Weak scaling: rank r's database is a full-size config generated with
    its own seed whose key values are moved to hash bucket r's key range
    (v -> v * world + r for every key column), so the P databases are the
    key-hash shards of one P-times larger database."""
    if world > 1:
        for r in db.relations:
            if r.keys.size:
                r.keys = r.keys * world + rank
    return db


def shard_database(db, rank: int, world: int):
    """Strong scaling: rank r's shard of ONE global database (fgdb.Database)
    through the partitioner (shard_relations on partition_attribute)."""
    from .fgdb import Database, RelationData
    attr = partition_attribute(db.relations, db.root)
    rels = shard_relations(db.relations, attr, rank, world,
                           make=lambda r, k, d: RelationData(r.name, list(r.key_attrs),
                                                             list(r.data_attrs),
                                                             np.ascontiguousarray(k),
                                                             np.ascontiguousarray(d)))
    return Database(rels, db.root, list(db.parent))
