"""ORACLE / TEST INFRASTRUCTURE ONLY -- a CPU restatement of the reference.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker.  The product path (the CUDA library
behind include/figaro_cuda.h) never calls it.

This is a plain numpy/Python restatement of the reference FiGaRo pipeline
(/root/reference/proj/include/figaro/*.hpp), written for desk-size inputs.
Every function cites the reference lines it restates.  It is pinned against
the reference's own known answers (tests/test_oracle_pins.py) and against
outputs of the compiled reference (tests/golden/, made by
tests/golden/make_golden.py through oracle/_ref/figaro_ref).
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

U64_MAX = (1 << 64) - 1


class error(RuntimeError):
    """error.hpp:9-11"""


class integrity_error(error):
    """error.hpp:23-26"""


class size_error(error):
    """error.hpp:28-31"""


class tree_error(error):
    """error.hpp:33-36"""


# --------------------------------------------------------------------------
# givens.hpp


def givens_coeffs(a: float, b: float) -> Tuple[float, float, float]:
    """givens.hpp:27-38: c = |a|/h, s = -sign(a) b/h, r = sign(a) h."""
    if b == 0.0:
        return 1.0, 0.0, a
    sg = -1.0 if math.copysign(1.0, a) < 0 else 1.0
    h = math.hypot(a, b)
    return abs(a) / h, -sg * b / h, sg * h


def head(a: np.ndarray) -> np.ndarray:
    """givens.hpp:59-70: sequential column sums times 1/sqrt(m)."""
    m = a.shape[0]
    if m == 0:
        raise error("head: empty matrix")
    h = np.zeros(a.shape[1])
    for i in range(m):
        h += a[i]
    return h * (1.0 / math.sqrt(m))


def tail(a: np.ndarray) -> np.ndarray:
    """givens.hpp:75-92: row j-1 = (sqrt(j) A[j] - S_j/sqrt(j)) / sqrt(j+1)."""
    m, n = a.shape
    if m == 0:
        raise error("tail: empty matrix")
    t = np.zeros((max(m - 1, 0), n))
    if m <= 1:
        return t
    prefix = a[0].copy()
    for j in range(1, m):
        sj = math.sqrt(j)
        sj1 = math.sqrt(j + 1)
        t[j - 1] = (sj * a[j] - prefix / sj) / sj1
        prefix += a[j]
    return t


def generalized_head(a: np.ndarray, v: Sequence[float]) -> np.ndarray:
    """givens.hpp:106-121: (sum_i v_i A_i) / ||v||."""
    m = a.shape[0]
    if m == 0:
        raise error("generalized_head: empty matrix")
    _check_weights(v, m)
    h = np.zeros(a.shape[1])
    norm2 = 0.0
    for i in range(m):
        h += v[i] * a[i]
        norm2 += v[i] * v[i]
    return h * (1.0 / math.sqrt(norm2))


def generalized_tail(a: np.ndarray, v: Sequence[float]) -> np.ndarray:
    """givens.hpp:126-148: weighted streaming tail."""
    m, n = a.shape
    if m == 0:
        raise error("generalized_tail: empty matrix")
    _check_weights(v, m)
    t = np.zeros((m - 1, n))
    if m == 1:
        return t
    prefix = v[0] * a[0]
    norm2 = v[0] * v[0]
    for j in range(1, m):
        np_ = math.sqrt(norm2)
        norm2 += v[j] * v[j]
        nn = math.sqrt(norm2)
        t[j - 1] = (np_ * a[j] - v[j] * prefix / np_) / nn
        prefix = prefix + v[j] * a[j]
    return t


def _check_weights(v, m):
    """givens.hpp:96-103"""
    if len(v) != m:
        raise error("weight length does not match row count")
    for w in v:
        if not (w > 0.0):
            raise error("weights must be positive")


# --------------------------------------------------------------------------
# relation.hpp / join_tree.hpp


class Relation:
    """relation.hpp:45-67 -- keys as a (rows, n_key) int64 array."""

    def __init__(self, name, key_attrs, data_attrs, keys, data):
        self.name = name
        self.key_attrs = list(key_attrs)
        self.data_attrs = list(data_attrs)
        data = np.asarray(data, dtype=np.float64)
        keys = np.asarray(keys, dtype=np.int64)
        rows = keys.shape[0] if keys.ndim and keys.shape[0] else data.shape[0] if data.ndim else 0
        self.keys = keys.reshape(rows, len(self.key_attrs))
        self.data = data.reshape(rows, len(self.data_attrs))

    @property
    def rows(self):
        return self.keys.shape[0]

    def key_tuple(self, i) -> tuple:
        return tuple(int(x) for x in self.keys[i])

    def key_groups(self) -> List[Tuple[int, int]]:
        """relation.hpp:56-66: [begin, end) runs of equal key tuples."""
        n = self.rows
        if n == 0:
            return []
        if self.keys.shape[1] == 0:
            return [(0, n)]
        diff = np.any(self.keys[1:] != self.keys[:-1], axis=1)
        starts = np.concatenate([[0], np.nonzero(diff)[0] + 1])
        ends = np.concatenate([starts[1:], [n]])
        return list(zip(starts.tolist(), ends.tolist()))


def canonicalize(rel: Relation) -> Relation:
    """relation.hpp:111-121,127-167: sort by (key tuple, data) lexicographically."""
    cols = [rel.data[:, j] for j in reversed(range(rel.data.shape[1]))]
    cols += [rel.keys[:, j] for j in reversed(range(rel.keys.shape[1]))]
    order = np.lexsort(cols) if cols else np.arange(rel.rows)
    return Relation(rel.name, rel.key_attrs, rel.data_attrs, rel.keys[order], rel.data[order])


class JoinTree:
    """join_tree.hpp:21-33"""

    def __init__(self, root, parent, children, parent_attrs, preorder):
        self.root = root
        self.parent = parent
        self.children = children
        self.parent_attrs = parent_attrs
        self.preorder = preorder

    def is_leaf(self, i):
        return not self.children[i]

    def is_root(self, i):
        return i == self.root


def build_join_tree(rels: List[Relation], root: int, parent: Sequence[int]) -> JoinTree:
    """join_tree.hpp:72-97 (parent_attrs sorted by name, join_tree.hpp:37-45)."""
    r = len(rels)
    children = [[] for _ in range(r)]
    pattrs = [[] for _ in range(r)]
    for i in range(r):
        p = parent[i]
        if i == root:
            if p != -1:
                raise tree_error("join tree: root cannot have a parent")
            continue
        if p < 0 or p >= r:
            raise tree_error("join tree: bad parent index")
        children[p].append(i)
        ka = set(rels[p].key_attrs)
        pattrs[i] = sorted(a for a in rels[i].key_attrs if a in ka)
    pre = []

    def walk(n):
        pre.append(n)
        for c in children[n]:
            walk(c)

    walk(root)
    if len(pre) != r:
        raise tree_error("join tree: not a connected tree")
    return JoinTree(root, list(parent), children, pattrs, pre)


def project_key(key: tuple, from_attrs, to_attrs) -> tuple:
    """join_tree.hpp:57-70"""
    return tuple(key[from_attrs.index(a)] for a in to_attrs)


class Layout:
    """join_tree.hpp:186-219: pre-order column layout."""

    def __init__(self, rels, tree):
        r = len(rels)
        self.node_offset = [0] * r
        self.node_width = [0] * r
        self.subtree_begin = [0] * r
        self.subtree_end = [0] * r
        self.total = 0
        for n in tree.preorder:
            self.node_offset[n] = self.total
            self.node_width[n] = len(rels[n].data_attrs)
            self.total += self.node_width[n]

        def fill(node):
            self.subtree_begin[node] = self.node_offset[node]
            end = self.node_offset[node] + self.node_width[node]
            for c in tree.children[node]:
                end = fill(c)
            self.subtree_end[node] = end
            return end

        fill(tree.root)


# --------------------------------------------------------------------------
# reduce.hpp


class empty_join_error(error):
    """error.hpp:38-41"""


def semi_join(rel: Relation, other: Relation, attrs) -> Relation:
    """reduce.hpp:20-43: keep rows of rel whose projection occurs in other."""
    if not attrs:
        return rel
    present = {project_key(other.key_tuple(i), other.key_attrs, attrs) for i in range(other.rows)}
    keep = [i for i in range(rel.rows)
            if project_key(rel.key_tuple(i), rel.key_attrs, attrs) in present]
    return Relation(rel.name, rel.key_attrs, rel.data_attrs, rel.keys[keep], rel.data[keep])


def semi_join_reduce(rels: List[Relation], tree: JoinTree) -> List[Relation]:
    """reduce.hpp:47-74: bottom-up then top-down semi-join sweep."""
    rels = list(rels)

    def nonempty(i):
        if rels[i].rows == 0:
            raise empty_join_error("relation %s reduced to empty: the join result is empty"
                                   % rels[i].name)

    for i in tree.preorder:
        nonempty(i)
    for i in reversed(tree.preorder):
        for c in tree.children[i]:
            rels[i] = semi_join(rels[i], rels[c], tree.parent_attrs[c])
            nonempty(i)
    for i in tree.preorder:
        for c in tree.children[i]:
            rels[c] = semi_join(rels[c], rels[i], tree.parent_attrs[c])
            nonempty(c)
    return rels


# --------------------------------------------------------------------------
# counts.hpp


def _mul(a, b):
    r = a * b
    if r > U64_MAX:
        raise size_error("count aggregate overflow (64-bit)")
    return r


def _add(a, b):
    r = a + b
    if r > U64_MAX:
        raise size_error("count aggregate overflow (64-bit)")
    return r


def _exact_div(num, den, what):
    if den == 0 or num % den != 0:
        raise integrity_error(what + ": counts are inconsistent; is the database fully reduced?")
    return num // den


class NodeCounts:
    """counts.hpp:24-31 (dicts iterated in sorted key order like std::map)."""

    def __init__(self):
        self.rows_per_key: Dict[tuple, int] = {}
        self.theta_down: Dict[tuple, int] = {}
        self.full_join_size: Dict[tuple, int] = {}
        self.phi_circ: Dict[tuple, int] = {}
        self.phi_down: Dict[tuple, int] = {}
        self.phi_up: Dict[tuple, int] = {}


def compute_counts(rels: List[Relation], tree: JoinTree) -> List[NodeCounts]:
    """counts.hpp:92-224: bottom-up theta/phi_down, top-down fjs/phi_up/phi_circ."""
    r = len(rels)
    nodes = [NodeCounts() for _ in range(r)]
    groups = []
    for i in range(r):
        g = rels[i].key_groups()
        groups.append(([rels[i].key_tuple(b) for b, _ in g], [e - b for b, e in g]))

    for i in reversed(tree.preorder):  # counts.hpp:110-156
        nc = nodes[i]
        keys, sizes = groups[i]
        for k, m in zip(keys, sizes):
            nc.rows_per_key[k] = m
        for k, m in zip(keys, sizes):
            theta = m
            for c in tree.children[i]:
                xc = project_key(k, rels[i].key_attrs, tree.parent_attrs[c])
                if xc not in nodes[c].phi_down:
                    raise integrity_error(
                        "compute_counts: key %r of %s has no match in child %s; "
                        "is the database fully reduced?" % (xc, rels[i].name, rels[c].name))
                theta = _mul(theta, nodes[c].phi_down[xc])
            nc.theta_down[k] = theta
            if not tree.is_root(i):
                xp = project_key(k, rels[i].key_attrs, tree.parent_attrs[i])
                nc.phi_down[xp] = _add(nc.phi_down.get(xp, 0), theta)

    def pass2(i):  # counts.hpp:160-221
        nc = nodes[i]
        keys, sizes = groups[i]
        for c in tree.children[i]:
            for k in keys:
                nodes[c].phi_up.setdefault(project_key(k, rels[i].key_attrs, tree.parent_attrs[c]), 0)
        for k, m in zip(keys, sizes):
            up = 1
            if not tree.is_root(i):
                up = nc.phi_up[project_key(k, rels[i].key_attrs, tree.parent_attrs[i])]
            fjs = _mul(nc.theta_down[k], up)
            nc.full_join_size[k] = fjs
            for c in tree.children[i]:
                xc = project_key(k, rels[i].key_attrs, tree.parent_attrs[c])
                nodes[c].phi_up[xc] = _add(nodes[c].phi_up[xc], fjs)
            nc.phi_circ[k] = _exact_div(fjs, m, "compute_counts: phi_circ")
        for c in tree.children[i]:
            up, down = nodes[c].phi_up, nodes[c].phi_down
            if len(up) != len(down):
                raise integrity_error("compute_counts: child %s has keys unmatched in %s; "
                                      "is the database fully reduced?" % (rels[c].name, rels[i].name))
            for key in list(up):
                up[key] = _exact_div(up[key], down[key], "compute_counts: phi_up")
            pass2(c)

    pass2(tree.root)
    for nc in nodes:
        for name in ("rows_per_key", "theta_down", "full_join_size", "phi_circ", "phi_down", "phi_up"):
            d = getattr(nc, name)
            setattr(nc, name, dict(sorted(d.items())))
    return nodes


# --------------------------------------------------------------------------
# figaro.hpp


class OutBlock:
    """figaro.hpp:29-33"""

    def __init__(self, node, col_begin, rows):
        self.node = node
        self.col_begin = col_begin
        self.rows = rows


def _count_at(m, key, what):
    """figaro.hpp:97-104"""
    v = m.get(key, 0)
    if v == 0:
        raise integrity_error("%s: no count for key %r; is the database fully reduced?" % (what, key))
    return v


def figaro_node(rels, tree, layout, counts, node):
    """figaro.hpp:166-316 -- returns (out_blocks, keys, data, scales)."""
    rel = rels[node]
    sub_begin = layout.subtree_begin[node]
    width = layout.subtree_end[node] - sub_begin
    own_w = len(rel.data_attrs)
    nc = counts[node]
    # heads_and_tails, figaro.hpp:109-159
    groups = rel.key_groups()
    out = []
    keys = []
    data = np.zeros((len(groups), width))
    scales = []
    for (b, e) in groups:
        m = e - b
        k = rel.key_tuple(b)
        keys.append(k)
        scales.append(math.sqrt(m))
        grp = rel.data[b:e]
        if own_w > 0:
            data[len(keys) - 1, :own_w] = head(grp)
        if m > 1 and own_w > 0:
            s = math.sqrt(_count_at(nc.phi_circ, k, "heads_and_tails"))
            out.append(OutBlock(node, layout.node_offset[node], tail(grp) * s))
    if not tree.is_leaf(node):
        child_states = []
        for c in tree.children[node]:
            cs = figaro_node(rels, tree, layout, counts, c)
            out.extend(cs[0])
            child_states.append((cs[1], cs[2], cs[3], {k: i for i, k in enumerate(cs[1])}))
        # process_and_join_children, figaro.hpp:196-230
        for k in range(len(keys)):
            rows, cscale = [], []
            for ci, c in enumerate(tree.children[node]):
                xc = project_key(keys[k], rel.key_attrs, tree.parent_attrs[c])
                idx = child_states[ci][3].get(xc)
                if idx is None:
                    raise integrity_error("figaro: key %r of %s has no summary row in child %s; "
                                          "is the database fully reduced?" % (xc, rel.name, rels[c].name))
                rows.append(idx)
                cscale.append(child_states[ci][2][idx])
            allp = 1.0
            for s in cscale:
                allp *= s
            for ci, c in enumerate(tree.children[node]):
                factor = scales[k]
                for cj in range(len(cscale)):
                    if cj != ci:
                        factor *= cscale[cj]
                local = layout.subtree_begin[c] - sub_begin
                src = child_states[ci][1][rows[ci]]
                data[k, local:local + src.shape[0]] = src * factor
            data[k, :own_w] *= allp
            scales[k] *= allp
        if not tree.is_root(node):
            # project_away_join_attributes, figaro.hpp:232-294
            pattrs = tree.parent_attrs[node]
            by_parent: Dict[tuple, List[int]] = {}
            for k in range(len(keys)):
                by_parent.setdefault(project_key(keys[k], rel.key_attrs, pattrs), []).append(k)
            new_keys = sorted(by_parent)
            new_data = np.zeros((len(new_keys), width))
            new_scales = []
            for g, pk in enumerate(new_keys):
                rows = by_parent[pk]
                stacked = data[rows]
                wts = [scales[r] for r in rows]
                new_data[g] = generalized_head(stacked, wts)
                new_scales.append(math.sqrt(_count_at(nc.phi_down, pk, "project_away (phi_down)")))
                if len(rows) > 1 and width > 0:
                    s = math.sqrt(_count_at(nc.phi_up, pk, "project_away (phi_up)"))
                    out.append(OutBlock(node, sub_begin, generalized_tail(stacked, wts) * s))
            keys, data, scales = new_keys, new_data, new_scales
    if tree.is_root(node):
        if width > 0 and data.shape[0] > 0:
            out.append(OutBlock(node, sub_begin, data.copy()))
    elif tree.is_leaf(node):
        pattrs = tree.parent_attrs[node]
        keys = [project_key(k, rel.key_attrs, pattrs) for k in keys]
    return out, keys, data, np.asarray(scales)


def figaro_r0(rels, tree, layout, counts) -> List[OutBlock]:
    """figaro.hpp:319-329"""
    return figaro_node(rels, tree, layout, counts, tree.root)[0]


# --------------------------------------------------------------------------
# postprocess.hpp


def dense_r0(blocks: List[OutBlock], columns: int) -> np.ndarray:
    """figaro.hpp:47-57"""
    n = sum(b.rows.shape[0] for b in blocks)
    out = np.zeros((n, columns))
    r = 0
    for b in blocks:
        m, w = b.rows.shape
        out[r:r + m, b.col_begin:b.col_begin + w] = b.rows
        r += m
    return out


def normalize_signs(r: np.ndarray) -> np.ndarray:
    """postprocess.hpp:173-184: negate rows with a negative diagonal."""
    r = r.copy()
    for i in range(r.shape[0]):
        if r[i, i] < 0.0:
            r[i] = np.where(r[i] == 0.0, 0.0, -r[i])
    return r


def householder_r(a: np.ndarray) -> np.ndarray:
    """postprocess.hpp:194-252,275-288: R of a dense stack (padded when short)."""
    m, n = a.shape
    if m < n:
        a = np.vstack([a, np.zeros((n - m, n))])
    if n == 0:
        return np.zeros((0, 0))
    return np.linalg.qr(a, mode="r")


def rel_frobenius_distance(a: np.ndarray, b: np.ndarray) -> float:
    """matrix.hpp:105-116"""
    ref = float(np.sum(b * b))
    diff = float(np.sum((a - b) ** 2))
    return math.sqrt(diff) if ref == 0.0 else math.sqrt(diff / ref)


# --------------------------------------------------------------------------
# driver.hpp


class PipelineResult:
    def __init__(self, R, r0_rows, input_rows, columns, counts, r0):
        self.R = R
        self.r0_rows = r0_rows
        self.input_rows = input_rows
        self.data_columns = columns
        self.counts = counts
        self.r0 = r0


def run_pipeline(rels: List[Relation], root: int, parent: Sequence[int],
                 canonical: bool = True, reduce: bool = False) -> PipelineResult:
    """driver.hpp:47-85 with the Householder engine (assume_reduced unless
    `reduce`)."""
    if canonical:
        rels = [canonicalize(r) for r in rels]
    tree = build_join_tree(rels, root, parent)
    if reduce:
        rels = semi_join_reduce(rels, tree)
    layout = Layout(rels, tree)
    counts = compute_counts(rels, tree)
    r0 = figaro_r0(rels, tree, layout, counts)
    R = normalize_signs(householder_r(dense_r0(r0, layout.total)))
    return PipelineResult(R, sum(b.rows.shape[0] for b in r0),
                          sum(r.rows for r in rels), layout.total, counts, r0)


# --------------------------------------------------------------------------
# join.hpp / recover_q


class rank_error(error):
    """error.hpp:43-46"""


DEFAULT_JOIN_CAP = 1_000_000  # join.hpp:25


def join_rows(rels: List[Relation], tree: JoinTree, cap: int = DEFAULT_JOIN_CAP) -> np.ndarray:
    """for_each_join_row (join.hpp:47-92) collected into a dense array:
    root rows in input order, then per pre-order node the rows matching the
    parent's current row (EdgeIndex keeps insertion order, join.hpp:29-38);
    dangling tuples yield nothing; more than `cap` rows -> size_error."""
    layout = Layout(rels, tree)
    index = []
    for i, rel in enumerate(rels):
        m: Dict[tuple, List[int]] = {}
        if i != tree.root:
            for r in range(rel.rows):
                m.setdefault(project_key(rel.key_tuple(r), rel.key_attrs,
                                         tree.parent_attrs[i]), []).append(r)
        index.append(m)
    out: List[np.ndarray] = []
    row = np.zeros(layout.total)
    cur = [0] * len(rels)

    def emit(depth):
        if depth == len(tree.preorder):
            if len(out) + 1 > cap:
                raise size_error(f"join row cap exceeded ({cap} rows)")
            out.append(row.copy())
            return
        node = tree.preorder[depth]
        rel = rels[node]
        off = layout.node_offset[node]
        if node == tree.root:
            cand = range(rel.rows)
        else:
            p = tree.parent[node]
            probe = project_key(rels[p].key_tuple(cur[p]), rels[p].key_attrs,
                                tree.parent_attrs[node])
            cand = index[node].get(probe, [])
        for r in cand:
            cur[node] = r
            row[off:off + rel.data.shape[1]] = rel.data[r]
            emit(depth + 1)

    emit(0)
    return np.array(out).reshape(len(out), layout.total)


def recover_q(rels: List[Relation], tree: JoinTree, R: np.ndarray,
              cap: int = DEFAULT_JOIN_CAP) -> Tuple[np.ndarray, np.ndarray]:
    """recover_q (postprocess.hpp:293-321): (A, Q) with q R = a solved per row
    by forward substitution in the reference's operation order (vectorised
    over rows; each element sees the same scalar operations)."""
    n = R.shape[1]
    if n != Layout(rels, tree).total:
        raise error("recover_q: factor size does not match column layout")
    s = 0.0
    for i in range(R.shape[0]):
        for x in R[i]:
            s += x * x
    tol = 1e-12 * math.sqrt(s)
    for i in range(n):
        if not abs(R[i, i]) > tol:
            raise rank_error(f"recover_q: triangular factor is singular at column {i}")
    A = join_rows(rels, tree, cap)
    Q = np.zeros_like(A)
    for j in range(n):
        acc = A[:, j].copy()
        for i in range(j):
            acc = acc - Q[:, i] * R[i, j]
        Q[:, j] = acc / R[j, j]
    return A, Q


def from_fgdb(db) -> Tuple[List[Relation], int, List[int]]:
    rels = [Relation(r.name, r.key_attrs, r.data_attrs, r.keys, r.data) for r in db.relations]
    return rels, db.root, list(db.parent)
