"""Multi-GPU data parallelism for the FiGaRo path: join partitioning and the
R gather.  The reference is single-process; this is the B200
addition of SURVEY 8(e).

Correctness rests on one identity.  If the shards' joins partition the full
join -- every join tuple is produced by exactly one rank -- then
    A = [A_0; A_1; ...; A_{P-1}]  (up to row order)
and R(A) = R([R(A_0); ...; R(A_{P-1})]).  Each rank runs the unmodified
device pipeline on its shard (a database in its own right), the P factors are
all-gathered over NCCL (torch.distributed) and one more device TSQR merges
them.  No count, summary or tail crosses GPUs before that final N x N gather.

Partition plan (plan_partition).  A grid over up to two key attributes
a_0, a_1 with extents d_0 * d_1 = P; rank q is the cell (q mod d_0,
q // d_0).  A row of a relation holding a_i goes to the cells whose
coordinate i equals h_i(value) mod d_i and to every cell along the
dimensions of attributes it does not hold (replication, as in the HyperCube
distribution of a multiway join).  A join tuple agrees on every attribute, so
it lands in exactly one cell.  The extents minimise the estimated per-rank
rows  sum_r rows_r / prod_{a_i in r} d_i :
  C1, C2, C5  k over P ranks, nothing replicated;
  C3          k1 over P ranks (F, D1 sharded; D2, D3 replicated, tiny);
  C4          (a, b) over 2 x 4 ranks: R1 / 2, R2 / 8, R3 / 4 per rank
              instead of replicating R3 (4M rows) on every rank.
Heavy values (single-attribute plans).  Hashing puts all rows of a value on
one rank; C5's most frequent key holds 26 % of the rows.  A value whose rows
exceed half a rank's fair share is split: the relations holding a_0 get a
sub-grid prod_r e_r = P over that value's rows (row t of relation r goes to
the ranks whose sub-coordinate r is t mod e_r), so its join is again cut
into P disjoint pieces (C5's top key: R1 rows over 4, R2 rows over 2 ranks;
C3's top k1: the F rows over all 8 ranks, D1's single row replicated).

Shards built with replication or splitting may hold dangling rows, so ranks
run the pipeline with semi-join reduction (PipelineOptions(assume_reduced=
False)), and a rank whose shard join is empty contributes a zero factor
(local_factor) instead of raising -- the gather then still matches on every
rank.
"""
from __future__ import annotations

import itertools
from collections import Counter
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def key_hash(values: np.ndarray, salt: int = 0) -> np.ndarray:
    """splitmix64 finaliser of int64 key values (deterministic across ranks);
    `salt` gives independent hashes for the grid's attributes."""
    with np.errstate(over="ignore"):
        z = values.astype(np.int64).view(np.uint64) + np.uint64(0x9E3779B97F4A7C15) * \
            np.uint64(1 + 2 * salt)
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
        rows = sum(_rows(r) for r in relations if a in r.key_attrs)
        return (cnt[a], a in root_attrs, rows, a)

    return max(cnt, key=score)


def _rows(r) -> int:
    return int(r.keys.shape[0])


def _factorisations(P: int, k: int) -> List[Tuple[int, ...]]:
    """Ordered k-tuples of positive integers whose product is P."""
    if k == 1:
        return [(P,)]
    out = []
    for d in range(1, P + 1):
        if P % d == 0:
            out += [(d,) + t for t in _factorisations(P // d, k - 1)]
    return out


@dataclass
class HeavySplit:
    """Sub-grid of one heavy value of attrs[0]: relation index -> extent.
    `complete`: every sub-grid cell receives at least one row of every
    holder (no dangling rows for this value)."""
    value: int
    extents: Dict[int, int]
    complete: bool = True


@dataclass
class Plan:
    world: int
    attrs: List[str] = field(default_factory=list)
    dims: List[int] = field(default_factory=list)
    heavy: List[HeavySplit] = field(default_factory=list)
    # Heavy keys of a two-relation same-key tree handled by partial-head
    # combination (heavy_stage / heavy_finish) instead of a sub-grid.
    combine: List[int] = field(default_factory=list)
    load: float = 0.0  # estimated max rows per rank

    def needs_reduction(self, relations: Sequence) -> bool:
        """Whether a shard may hold dangling rows (replicated relations, or a
        heavy split leaving a cell without rows of some holder), so ranks
        must run the pipeline with semi-join reduction."""
        if self.world <= 1:
            return False
        for r in relations:
            for a, d in zip(self.attrs, self.dims):
                if d > 1 and a not in r.key_attrs:
                    return True
        return any(not h.complete for h in self.heavy)

    def cell(self, rank: int) -> List[int]:
        c, q = [], rank
        for d in self.dims:
            c.append(q % d)
            q //= d
        return c


def _load(relations, attrs, dims) -> float:
    tot = 0.0
    for r in relations:
        div = 1
        for a, d in zip(attrs, dims):
            if a in r.key_attrs:
                div *= d
        tot += _rows(r) / div
    return tot


def two_way_same_key(relations: Sequence, root: int, parent: Optional[Sequence[int]]) -> bool:
    """R1(k) |><| R2(k): two relations, one edge, identical key attributes."""
    if parent is None or len(relations) != 2:
        return False
    child = 1 - root
    return (list(parent)[child] == root and relations[0].key_attrs and
            sorted(relations[0].key_attrs) == sorted(relations[1].key_attrs) and
            len(relations[0].key_attrs) == 1)


def plan_partition(relations: Sequence, root: int, world: int,
                   heavy_fraction: float = 0.5, max_heavy: int = 64,
                   parent: Optional[Sequence[int]] = None,
                   combine_fraction: float = 0.05, max_combine: int = 1024) -> Plan:
    """Grid attributes and extents minimising the estimated per-rank rows,
    plus heavy-value handling for single-attribute plans: partial-head
    combination for two-relation same-key trees (given `parent`), sub-grid
    splits otherwise (module docstring)."""
    plan = Plan(world)
    if world <= 1:
        return plan
    cnt = Counter(a for r in relations for a in r.key_attrs)
    if not cnt:
        return plan  # cartesian product of key-less relations: replicas only
    first = partition_attribute(relations, root)
    cands = [first] + [a for a, _ in cnt.most_common() if a != first][:3]
    best = (_load(relations, [first], [world]), [first], [world])
    for b in cands[1:]:
        for d0, d1 in _factorisations(world, 2):
            if d1 == 1:
                continue
            ld = _load(relations, [first, b], [d0, d1])
            if ld < best[0] * 0.95:  # a second dimension must pay for itself
                best = (ld, [first, b], [d0, d1])
    plan.load, plan.attrs, plan.dims = best
    if len(plan.attrs) == 1 and two_way_same_key(relations, root, parent):
        plan.combine = _combine_values(relations, first, world, combine_fraction, max_combine)
    elif len(plan.attrs) == 1:
        plan.heavy = _heavy_splits(relations, first, world, heavy_fraction, max_heavy)
    return plan


def _combine_values(relations, attr, world, frac, max_n) -> List[int]:
    """Keys of a two-relation same-key join whose rows exceed `frac` of a
    rank's fair share and that occur in both relations (others do not join)."""
    cols = [np.asarray(r.keys)[:, r.key_attrs.index(attr)] for r in relations]
    per = Counter()
    present = None
    for col in cols:
        vals, cnts = np.unique(col, return_counts=True)
        per.update(dict(zip(vals.tolist(), cnts.tolist())))
        present = set(vals.tolist()) if present is None else present & set(vals.tolist())
    thresh = frac * sum(c.shape[0] for c in cols) / world
    return sorted(v for v, m in per.most_common(max_n) if m >= thresh and v in present)


def _heavy_splits(relations, attr, world, frac, max_heavy) -> List[HeavySplit]:
    holders = [i for i, r in enumerate(relations) if attr in r.key_attrs]
    total = sum(_rows(r) for r in relations)
    per_value: Counter = Counter()
    by_rel: Dict[int, Counter] = {}
    for i in holders:
        col = np.asarray(relations[i].keys)[:, relations[i].key_attrs.index(attr)]
        vals, cnts = np.unique(col, return_counts=True)
        by_rel[i] = Counter(dict(zip(vals.tolist(), cnts.tolist())))
        per_value.update(by_rel[i])
    thresh = frac * total / world
    out = []
    for v, m in per_value.most_common(max_heavy):
        if m < thresh:
            break
        ms = {i: by_rel[i].get(v, 0) for i in holders}
        best = None
        for ext in _factorisations(world, len(holders)):
            ld = sum(ms[i] / e for i, e in zip(holders, ext))
            if best is None or ld < best[0]:
                best = (ld, ext)
        if best[0] < m:
            ext = dict(zip(holders, best[1]))
            out.append(HeavySplit(int(v), ext, all(ms[i] >= ext[i] for i in holders)))
    return out


def _sub_coords(rank: int, extents: Dict[int, int]) -> Dict[int, int]:
    c, q = {}, rank
    for i in sorted(extents):
        c[i] = q % extents[i]
        q //= extents[i]
    return c


def shard_mask(relations: Sequence, plan: Plan, rank: int) -> List[np.ndarray]:
    """Row masks of rank `rank`'s shard, one per relation."""
    out = []
    cell = plan.cell(rank)
    heavy = {h.value: h for h in plan.heavy}
    heavy_vals = np.array(sorted(heavy), dtype=np.int64)
    comb = np.array(plan.combine, dtype=np.int64)
    for ri, r in enumerate(relations):
        keys = np.asarray(r.keys)
        mask = np.ones(keys.shape[0], dtype=bool)
        if comb.size and plan.attrs and plan.attrs[0] in r.key_attrs:
            mask &= ~np.isin(keys[:, r.key_attrs.index(plan.attrs[0])], comb)
        for i, (a, d) in enumerate(zip(plan.attrs, plan.dims)):
            if a not in r.key_attrs or d == 1:
                continue
            col = keys[:, r.key_attrs.index(a)]
            mine = (key_hash(col, i) % np.uint64(d)) == np.uint64(cell[i])
            if i == 0 and heavy:
                hv = np.isin(col, heavy_vals)
                mine &= ~hv  # heavy values follow their sub-grid instead
                for v in np.unique(col[hv]).tolist():
                    h = heavy[v]
                    sub = _sub_coords(rank, h.extents)
                    rows_v = np.nonzero(col == v)[0]
                    e = h.extents.get(ri, 1)
                    take = rows_v[(np.arange(rows_v.shape[0]) % e) == sub.get(ri, 0)]
                    mine[take] = True
            mask &= mine
        out.append(mask)
    return out


def shard_relations(relations: Sequence, attr_or_plan, rank: int, world: int,
                    make=None) -> List:
    """Rank `rank`'s shard (host numpy relations).  `attr_or_plan` is a Plan,
    or a single attribute name (plain hash sharding on it; None replicates
    everything).  `make(rel, keys, data)` builds the output relation."""
    if isinstance(attr_or_plan, Plan):
        plan = attr_or_plan
    else:
        plan = Plan(world, [attr_or_plan] if attr_or_plan else [],
                    [world] if attr_or_plan else [])
    masks = shard_mask(relations, plan, rank) if world > 1 else \
        [np.ones(_rows(r), dtype=bool) for r in relations]
    out = []
    for r, m in zip(relations, masks):
        keys, data = np.asarray(r.keys)[m], np.asarray(r.data)[m]
        if make is None:
            out.append(type(r)(r.name, list(r.key_attrs), list(r.data_attrs),
                               np.ascontiguousarray(keys), np.ascontiguousarray(data)))
        else:
            out.append(make(r, keys, data))
    return out


def replicated(relations: Sequence, attr: Optional[str]) -> List[str]:
    return [r.name for r in relations if attr is None or attr not in r.key_attrs]


def local_factor(relations, tree, n: int, device: int = 0, assume_reduced: bool = False,
                 results: Optional[list] = None, **kw):
    """One rank's N x N factor through the device pipeline; a shard whose join
    is empty contributes zeros (so every rank reaches the gather)."""
    import torch

    from .figaro import PipelineOptions, empty_join_error, run_pipeline
    if any(_rows(r) == 0 for r in relations):  # a join with an empty relation
        return torch.zeros((n, n), dtype=torch.float64, device=f"cuda:{device}")
    try:
        res = run_pipeline(relations, tree, PipelineOptions(assume_reduced=assume_reduced),
                           device=device, fetch_counts=False, **kw)
        if results is not None:
            results.append(res)
        R = res.factor.r
        R = R if isinstance(R, torch.Tensor) else torch.from_numpy(np.asarray(R))
        return R.to(f"cuda:{device}")
    except empty_join_error:
        return torch.zeros((n, n), dtype=torch.float64, device=f"cuda:{device}")


def heavy_rows(relations: Sequence, plan: Plan, rank: int) -> List[Tuple[np.ndarray, np.ndarray]]:
    """Rank `rank`'s part of the combine keys' rows, per relation: row t of a
    key's rows (input order) belongs to rank t mod P.  Returned sorted by the
    key's position in plan.combine (stable), as (key index, data)."""
    out = []
    comb = np.array(plan.combine, dtype=np.int64)
    for r in relations:
        col = np.asarray(r.keys)[:, r.key_attrs.index(plan.attrs[0])]
        hv = np.nonzero(np.isin(col, comb))[0]
        kidx = np.searchsorted(comb, col[hv])
        order = np.argsort(kidx, kind="stable")
        hv, kidx = hv[order], kidx[order]
        # position of each row among its key's rows
        first = np.searchsorted(kidx, kidx, side="left")
        t = np.arange(hv.shape[0]) - first
        mine = (t % plan.world) == rank
        out.append((kidx[mine], np.ascontiguousarray(np.asarray(r.data)[hv[mine]])))
    return out


def _segments(kidx: np.ndarray, H: int):
    """begins over the keys present (int32), and which keys they are."""
    keys, counts = np.unique(kidx, return_counts=True)
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int32), keys, counts


def local_counts(parts, plan: Plan) -> np.ndarray:
    """[H, 2] int64 rows of each combine key in this rank's part, per relation
    (relation order); summed over ranks they are the global counts."""
    H = len(plan.combine)
    out = np.zeros((H, 2), dtype=np.int64)
    for j, (kidx, _) in enumerate(parts):
        out[:, j] = np.bincount(kidx, minlength=H)[:H]
    return out


def heavy_stage(parts, plan: Plan, root: int, n: int, global_counts: np.ndarray,
                device: int = 0):
    """Per rank, on the device: the transform of the rank's part of every
    combine key -- tails scaled by sqrt of the OTHER relation's global count
    (Phi_circ of a two-relation join, counts.hpp:190-206), their local factor
    (n x n), and the packed partial heads [H, w_root + w_child] with the
    local row counts, for the all-gather (heavy_finish combines them)."""
    import torch

    from .figaro import heads_tails, tsqr
    dev = torch.device("cuda", device)
    H = len(plan.combine)
    ws = [parts[0][1].shape[1], parts[1][1].shape[1]]
    off = [0, ws[root]] if root == 0 else [ws[root], 0]  # pre-order: root columns first
    blocks, heads = [], torch.zeros((H, ws[0] + ws[1]), dtype=torch.float64, device=dev)
    hoff = [0, ws[0]]
    for j, (kidx, data) in enumerate(parts):
        if kidx.shape[0] == 0 or ws[j] == 0:
            continue
        begins, keys, _ = _segments(kidx, H)
        other = global_counts[keys, 1 - j].astype(np.uint64)
        x = data.to(dev) if isinstance(data, torch.Tensor) else torch.from_numpy(data).to(dev)
        h, t, _ = heads_tails(x, torch.from_numpy(begins).to(dev),
                              tail_count=torch.from_numpy(other).to(dev), device=device)
        heads[torch.from_numpy(keys).to(dev), hoff[j]:hoff[j] + ws[j]] = h
        if t.shape[0]:
            blocks.append((t, off[j]))
    R = tsqr(blocks, n, device=device) if blocks else \
        torch.zeros((n, n), dtype=torch.float64, device=dev)
    return R, heads


def heavy_finish(all_heads, all_counts, plan: Plan, root: int, ws: Sequence[int], n: int,
                 device: int = 0):
    """Every rank, identically: for each combine key the partial heads h_q
    (weights sqrt(m_q)) are combined by the generalized head/tail transform
    (givens.hpp:106-148) -- head = S / sqrt(m), tails scaled by sqrt of the
    other relation's global count -- and the root row
    [head_root * sqrt(m_child) | head_child * sqrt(m_root)] is formed as in
    process_and_join_children (figaro.hpp:196-230).  Returns their factor.
    all_heads: [P, H, w0 + w1]; all_counts: [P, H, 2] (relation order)."""
    import torch

    from .figaro import heads_tails, tsqr
    dev = torch.device("cuda", device)
    P, H = all_counts.shape[0], all_counts.shape[1]
    g = all_counts.sum(axis=0)  # [H, 2] global counts
    hoff = [0, ws[0]]
    off = [0, ws[root]] if root == 0 else [ws[root], 0]
    blocks, comb = [], []
    for j in range(2):
        if ws[j] == 0:
            comb.append(torch.zeros((H, 0), dtype=torch.float64, device=dev))
            continue
        qs, ks = np.nonzero(all_counts[:, :, j].T > 0)[::-1]  # key-major order
        order = np.lexsort((qs, ks))
        qs, ks = qs[order], ks[order]
        stack = all_heads[torch.from_numpy(qs).to(dev), torch.from_numpy(ks).to(dev),
                          hoff[j]:hoff[j] + ws[j]].contiguous()
        wts = torch.from_numpy(np.sqrt(all_counts[qs, ks, j].astype(np.float64))).to(dev)
        begins, keys, _ = _segments(ks, H)
        other = g[keys, 1 - j].astype(np.uint64)
        h, t, _ = heads_tails(stack, torch.from_numpy(begins).to(dev), weights=wts,
                              tail_count=torch.from_numpy(other).to(dev), device=device)
        full = torch.zeros((H, ws[j]), dtype=torch.float64, device=dev)
        full[torch.from_numpy(keys).to(dev)] = h
        comb.append(full)
        if t.shape[0]:
            blocks.append((t, off[j]))
    sq = torch.from_numpy(np.sqrt(g.astype(np.float64))).to(dev)
    child = 1 - root
    root_rows = torch.cat([comb[root] * sq[:, child:child + 1],
                           comb[child] * sq[:, root:root + 1]], dim=1).contiguous()
    blocks.append((root_rows, 0))
    return tsqr(blocks, n, device=device)


def distributed_factor(shard, heavy, tree, n: int, plan: Plan, root: int, device: int = 0,
                       group=None, assume_reduced: Optional[bool] = None,
                       results: Optional[list] = None):
    """The whole multi-GPU flow of one rank (torch.distributed initialised,
    or a single process): pipeline on the main shard, heavy-key stage,
    all-gathers (counts; factors + partial heads) and the device merge.
    Returns the global R on every rank."""
    import torch
    import torch.distributed as dist

    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    if assume_reduced is None:
        assume_reduced = not plan.needs_reduction(shard)
    R_main = local_factor(shard, tree, n, device, assume_reduced=assume_reduced, results=results)

    def gather(t):
        if not multi:
            return [t]
        # gloo gathers host tensors, NCCL device tensors
        on_dev = dist.get_backend(group) == "nccl"
        x = t.contiguous() if on_dev else t.cpu().contiguous()
        out = [torch.empty_like(x) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, x, group=group)
        return [o.to(f"cuda:{device}") for o in out]

    if not plan.combine:
        return device_merge(gather(R_main), n, device)
    ws = [heavy[0][1].shape[1], heavy[1][1].shape[1]]
    cnt = local_counts(heavy, plan)
    all_cnt = np.stack([c.cpu().numpy() for c in gather(torch.from_numpy(cnt).to(f"cuda:{device}"))])
    R_h, heads = heavy_stage(heavy, plan, root, n, all_cnt.sum(axis=0), device)
    R_local = device_merge([R_main, R_h], n, device)
    parts = gather(R_local)
    all_heads = torch.stack(gather(heads))
    R_extra = heavy_finish(all_heads, all_cnt, plan, root, ws, n, device)
    return device_merge(parts + [R_extra], n, device)


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
    return tsqr([(p.to(f"cuda:{device}"), 0) for p in parts], n, device=device)


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


def shard_database(db, rank: int, world: int, plan: Optional[Plan] = None):
    """Strong scaling: rank r's shard of ONE global database (fgdb.Database)
    through the partition plan (plan_partition unless given)."""
    from .fgdb import Database, RelationData
    plan = plan or plan_partition(db.relations, db.root, world)
    rels = shard_relations(db.relations, plan, rank, world,
                           make=lambda r, k, d: RelationData(r.name, list(r.key_attrs),
                                                             list(r.data_attrs),
                                                             np.ascontiguousarray(k),
                                                             np.ascontiguousarray(d)))
    return Database(rels, db.root, list(db.parent))
