"""Python host mirror of the reference's pipeline API, running on the B200.

Same names, argument meaning and error behaviour as the reference library
(/root/reference/proj/include/figaro/):
    Relation                    relation.hpp:45-67
    JoinTree, build_join_tree   join_tree.hpp:21-33, 72-97
    Layout, make_layout         join_tree.hpp:186-219
    PipelineOptions             driver.hpp:27-31
    PipelineResult              driver.hpp:33-43
    run_pipeline                driver.hpp:47-85
    error classes               error.hpp:9-46
All computation goes through the C ABI (include/figaro_cuda.h); relations may
be numpy arrays (host) or torch CUDA tensors (device-resident).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------- errors


class error(RuntimeError):
    """figaro::error (error.hpp:9-11)."""


class schema_error(error):
    pass


class parse_error(error):
    pass


class integrity_error(error):
    pass


class size_error(error):
    pass


class tree_error(error):
    pass


class empty_join_error(error):
    pass


class rank_error(error):
    pass


class unsupported_error(error):
    """Input shape the device path does not handle (e.g. > 64 key bits)."""


class cuda_error(error):
    pass


_ERR = {L.FG_E_ARG: error, L.FG_E_SCHEMA: schema_error, L.FG_E_TREE: tree_error,
        L.FG_E_INTEGRITY: integrity_error, L.FG_E_SIZE: size_error,
        L.FG_E_EMPTY_JOIN: empty_join_error, L.FG_E_UNSUPPORTED: unsupported_error,
        L.FG_E_CUDA: cuda_error, L.FG_E_RANK: rank_error}


# ---------------------------------------------------------------- context


class Context:
    """One fg_ctx per GPU (owns a stream and the last result)."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        self.device = device
        h = C.c_void_p()
        st = self.lib.fg_ctx_create(device, C.byref(h))
        if st != L.FG_OK:
            raise cuda_error(f"fg_ctx_create(device={device}) failed with status {st}: "
                             "needs an sm_100 GPU (no CPU fallback)")
        self.h = h
        self._bound = None

    def check(self, st: int):
        if st != L.FG_OK:
            msg = self.lib.fg_last_error(self.h).decode()
            raise _ERR.get(st, error)(msg)

    @property
    def stream(self) -> int:
        return self.lib.fg_ctx_stream(self.h) or 0

    def set_stream(self, stream_ptr: int):
        """Orders the context's work on `stream_ptr` (a cudaStream_t).  0 is
        torch's legacy default stream, bound as cudaStreamLegacy -- the C
        ABI's NULL means "the context's own stream"."""
        ptr = stream_ptr or _CUDA_STREAM_LEGACY
        if ptr == self._bound:
            return
        self.check(self.lib.fg_ctx_set_stream(self.h, C.c_void_p(ptr)))
        self._bound = ptr

    def bind_current_stream(self):
        """Binds the context to torch's current stream on its device, so
        device tensors produced by torch (or NCCL) are complete before the
        library reads them and results are ordered before torch's next op."""
        import torch
        self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def kernel_launches(self) -> int:
        return int(self.lib.fg_kernel_launches(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.fg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: Dict[int, Context] = {}
_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream


def get_context(device: int = 0) -> Context:
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    return ctx


# ---------------------------------------------------------------- relations


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclasses.dataclass
class Relation:
    """relation.hpp:45-67.  keys: (rows, n_key) int64; data: (rows, n_data) f64."""

    name: str
    key_attrs: List[str]
    data_attrs: List[str]
    keys: object
    data: object

    def __post_init__(self):
        rows = None
        for x in (self.keys, self.data):
            if getattr(x, "ndim", 0) == 2:
                rows = int(x.shape[0])
        if _is_torch(self.keys) or _is_torch(self.data):
            self._normalise_torch(rows)
            return
        if not _is_torch(self.keys):
            k = np.asarray(self.keys, dtype=np.int64)
            self.keys = np.ascontiguousarray(
                k.reshape(rows if rows is not None else -1, len(self.key_attrs)))
        if not _is_torch(self.data):
            d = np.asarray(self.data, dtype=np.float64)
            self.data = np.ascontiguousarray(
                d.reshape(rows if rows is not None else -1, len(self.data_attrs)))

    def _normalise_torch(self, rows):
        """Torch inputs: both tensors must live on one CUDA device; keys
        become contiguous int64 (rows, n_key), data contiguous float64
        (rows, n_data) -- the row-major layout the C ABI reads by pointer."""
        import torch
        if not (_is_torch(self.keys) and _is_torch(self.data)):
            raise error(f"relation {self.name}: keys and data must both be torch tensors "
                        "or both host arrays")
        if not (self.keys.is_cuda and self.data.is_cuda) or self.keys.device != self.data.device:
            raise error(f"relation {self.name}: keys and data must be on the same CUDA device")
        nk, nd = len(self.key_attrs), len(self.data_attrs)
        if rows is None:
            rows = int(self.keys.numel() // nk) if nk else int(self.data.numel() // max(nd, 1))
        self.keys = self.keys.to(torch.int64).reshape(rows, nk).contiguous()
        self.data = self.data.to(torch.float64).reshape(rows, nd).contiguous()

    def row_count(self) -> int:
        return int(self.keys.shape[0])

    @property
    def on_device(self) -> bool:
        return _is_torch(self.data) and self.data.is_cuda


@dataclasses.dataclass
class JoinTree:
    """join_tree.hpp:21-33 (parent_attrs sorted by name)."""

    root: int
    parent: List[int]
    children: List[List[int]]
    parent_attrs: List[List[str]]
    preorder: List[int]

    def is_leaf(self, i):
        return not self.children[i]

    def is_root(self, i):
        return i == self.root


def build_join_tree(relations: Sequence[Relation], root: int,
                    parent: Sequence[int]) -> JoinTree:
    """join_tree.hpp:72-97 (the device library re-derives the same tree)."""
    r = len(relations)
    if r == 0:
        raise tree_error("join tree: no relations")
    children = [[] for _ in range(r)]
    pattrs = [[] for _ in range(r)]
    for i in range(r):
        p = parent[i]
        if i == root:
            if p != -1:
                raise tree_error("join tree: root cannot have a parent")
            continue
        if p < 0 or p >= r:
            raise tree_error("join tree: bad parent index for node " + relations[i].name)
        children[p].append(i)
        ka = set(relations[p].key_attrs)
        pattrs[i] = sorted(a for a in relations[i].key_attrs if a in ka)
    pre: List[int] = []

    def walk(n):
        pre.append(n)
        for c in children[n]:
            walk(c)

    walk(root)
    if len(pre) != r:
        raise tree_error("join tree: not a connected tree")
    return JoinTree(root, list(parent), children, pattrs, pre)


@dataclasses.dataclass
class Layout:
    total: int
    node_offset: List[int]
    node_width: List[int]
    subtree_begin: List[int]
    subtree_end: List[int]
    column_names: List[str]


def make_layout(relations: Sequence[Relation], tree: JoinTree) -> Layout:
    """join_tree.hpp:195-219: pre-order global column layout."""
    r = len(relations)
    off, wid, sb, se = [0] * r, [0] * r, [0] * r, [0] * r
    names = []
    total = 0
    for n in tree.preorder:
        off[n] = total
        wid[n] = len(relations[n].data_attrs)
        names += [relations[n].name + "." + a for a in relations[n].data_attrs]
        total += wid[n]

    def fill(n):
        sb[n] = off[n]
        end = off[n] + wid[n]
        for c in tree.children[n]:
            end = fill(c)
        se[n] = end
        return end

    fill(tree.root)
    return Layout(total, off, wid, sb, se, names)


# ---------------------------------------------------------------- pipeline


@dataclasses.dataclass
class PipelineOptions:
    """driver.hpp:27-31.  `threads` is accepted for API parity (the device
    decides its own parallelism); engine is "thin" or "householder"."""

    threads: int = 0
    engine: str = "thin"
    assume_reduced: bool = False


@dataclasses.dataclass
class TriangularFactor:
    """postprocess.hpp:22-28."""

    r: object
    column_names: List[str]
    zero_diagonal_rows: List[int]


@dataclasses.dataclass
class NodeCounts:
    """counts.hpp:24-31 as arrays in ascending key order, plus the keys."""

    keys: np.ndarray          # (G, n_key) distinct own keys
    rows_per_key: np.ndarray
    theta_down: np.ndarray
    full_join_size: np.ndarray
    phi_circ: np.ndarray
    parent_keys: np.ndarray   # (P, n_pattr)
    phi_down: np.ndarray
    phi_up: np.ndarray
    group_begin: np.ndarray   # Relation::key_groups() begins (G,)

    def as_maps(self) -> Dict[str, Dict[tuple, int]]:
        own = [tuple(int(x) for x in k) for k in self.keys]
        par = [tuple(int(x) for x in k) for k in self.parent_keys]
        d = {n: dict(zip(own, getattr(self, n).tolist()))
             for n in ("rows_per_key", "theta_down", "full_join_size", "phi_circ")}
        d.update({n: dict(zip(par, getattr(self, n).tolist())) for n in ("phi_down", "phi_up")})
        return d


@dataclasses.dataclass
class OutSpan:
    """R0 span = the reference's OutBlocks of one (node, col_begin) stacked."""

    node: int
    col_begin: int
    rows: np.ndarray


@dataclasses.dataclass
class PipelineResult:
    """driver.hpp:33-43 (+ seconds_group, kernels)."""

    factor: TriangularFactor
    r0_rows: int
    input_rows: int
    data_columns: int
    seconds_group: float
    seconds_counts: float
    seconds_figaro: float
    seconds_postprocess: float
    seconds_total: float
    kernels: int
    seconds_headtail_kernels: float = 0.0
    seconds_tsqr_kernels: float = 0.0
    headtail_launches: int = 0
    headtail_bytes: float = 0.0
    headtail_fused_flops: float = 0.0
    tsqr_stage_flops: float = 0.0
    fused_launches: int = 0
    host_syncs: int = 0
    device_mallocs: int = 0
    counts: Optional[List[NodeCounts]] = None
    r0: Optional[List[OutSpan]] = None


def _cstrs(names):
    arr = (C.c_char_p * max(1, len(names)))()
    for i, s in enumerate(names):
        arr[i] = s.encode()
    return arr


def _marshal(rels, what):
    """fg_relation array for the C ABI (+ objects to keep alive, device flag)."""
    on_dev = [r.on_device for r in rels]
    if any(on_dev) and not all(on_dev):
        raise error(f"{what}: mix of host and device relations")
    device_mem = bool(rels) and all(on_dev)
    keep = []
    arr = (L.fg_relation * len(rels))()
    for i, r in enumerate(rels):
        ka, da = _cstrs(r.key_attrs), _cstrs(r.data_attrs)
        keep += [ka, da, r.keys, r.data]
        if device_mem:
            kp, dp = r.keys.data_ptr(), r.data.data_ptr()
        else:
            kp, dp = r.keys.ctypes.data, r.data.ctypes.data
        arr[i] = L.fg_relation(r.name.encode(), len(r.key_attrs), ka, len(r.data_attrs), da,
                               r.row_count(), kp, dp)
    return arr, keep, device_mem


def run_pipeline(relations: Sequence[Relation], tree: JoinTree,
                 opts: PipelineOptions = PipelineOptions(), keep_r0: bool = False,
                 device: int = 0, fetch_counts: bool = True,
                 fuse: bool = True) -> PipelineResult:
    """driver.hpp:47-85 on the GPU.  Host (numpy) relations are copied to the
    device inside the call; torch CUDA relations are used in place and R is
    returned as a CUDA tensor."""
    ctx = get_context(device)
    lib = ctx.lib
    rels = list(relations)
    arr, keep, device_mem = _marshal(rels, "run_pipeline")
    parent = (C.c_int32 * len(rels))(*tree.parent)
    o = L.fg_options()
    lib.fg_options_default(C.byref(o))
    o.assume_reduced = int(bool(opts.assume_reduced))
    o.engine = L.FG_ENGINE_HOUSEHOLDER if opts.engine == "householder" else L.FG_ENGINE_THIN
    o.memory = L.FG_MEM_DEVICE if device_mem else L.FG_MEM_HOST
    o.keep_r0 = int(keep_r0)
    o.fuse = int(fuse)
    layout = make_layout(rels, tree)
    n = layout.total
    if device_mem:
        import torch
        ctx.bind_current_stream()
        R = torch.empty((n, n), dtype=torch.float64, device=rels[0].data.device)
        rp = R.data_ptr()
    else:
        R = np.zeros((n, n))
        rp = R.ctypes.data
    res = L.fg_result()
    ctx.check(lib.fg_run_pipeline(ctx.h, len(rels), arr, tree.root, parent, C.byref(o),
                                  C.c_void_p(rp), C.byref(res)))
    del keep
    diag = (R.diagonal().cpu().numpy() if device_mem else np.diag(R)) if n else np.zeros(0)
    out = PipelineResult(
        factor=TriangularFactor(R, layout.column_names, [i for i in range(n) if diag[i] == 0.0]),
        r0_rows=res.r0_rows, input_rows=res.input_rows, data_columns=res.data_columns,
        seconds_group=res.seconds_group, seconds_counts=res.seconds_counts,
        seconds_figaro=res.seconds_figaro, seconds_postprocess=res.seconds_postprocess,
        seconds_total=res.seconds_total, kernels=res.kernels,
        seconds_headtail_kernels=res.seconds_headtail_kernels,
        seconds_tsqr_kernels=res.seconds_tsqr_kernels,
        headtail_launches=res.headtail_launches, headtail_bytes=res.headtail_bytes,
        headtail_fused_flops=res.headtail_fused_flops, tsqr_stage_flops=res.tsqr_stage_flops,
        fused_launches=res.fused_launches, host_syncs=res.host_syncs,
        device_mallocs=res.device_mallocs)
    if fetch_counts:
        out.counts = [fetch_node_counts(ctx, i, rels[i], tree) for i in range(len(rels))]
    if keep_r0:
        out.r0 = fetch_r0(ctx)
    return out


def fetch_node_counts(ctx: Context, node: int, rel: Relation, tree: JoinTree) -> NodeCounts:
    lib = ctx.lib
    G, P = C.c_int64(), C.c_int64()
    ctx.check(lib.fg_get_sizes(ctx.h, node, C.byref(G), C.byref(P)))
    G, P = G.value, P.value
    nk = len(rel.key_attrs)
    npa = len(tree.parent_attrs[node])
    keys = np.zeros((G, nk), dtype=np.int64)
    if G and nk:
        ctx.check(lib.fg_get_keys(ctx.h, node, 0, keys.ctypes.data))
    pkeys = np.zeros((P, npa), dtype=np.int64)
    if P and npa:
        ctx.check(lib.fg_get_keys(ctx.h, node, 1, pkeys.ctypes.data))

    def table(kind, n):
        a = np.zeros(n, dtype=np.uint64)
        if n:
            ctx.check(lib.fg_get_counts(ctx.h, node, kind, a.ctypes.data))
        return a

    begins = np.zeros(G + 1, dtype=np.int64)
    ctx.check(lib.fg_get_segments(ctx.h, node, begins.ctypes.data))
    return NodeCounts(keys, table(L.FG_ROWS_PER_KEY, G), table(L.FG_THETA_DOWN, G),
                      table(L.FG_FULL_JOIN_SIZE, G), table(L.FG_PHI_CIRC, G), pkeys,
                      table(L.FG_PHI_DOWN, P), table(L.FG_PHI_UP, P), begins[:-1])


def fetch_permutation(node: int, rows: int, device: int = 0) -> np.ndarray:
    ctx = get_context(device)
    out = np.zeros(rows, dtype=np.int32)
    if rows:
        ctx.check(ctx.lib.fg_get_permutation(ctx.h, node, out.ctypes.data))
    return out


def fetch_r0(ctx: Context) -> List[OutSpan]:
    lib = ctx.lib
    n = C.c_int32()
    ctx.check(lib.fg_get_r0_span_count(ctx.h, C.byref(n)))
    spans = []
    for i in range(n.value):
        node, cb, rows, cols = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
        ctx.check(lib.fg_get_r0_span(ctx.h, i, C.byref(node), C.byref(cb), C.byref(rows),
                                     C.byref(cols), None))
        a = np.zeros((rows.value, cols.value))
        ctx.check(lib.fg_get_r0_span(ctx.h, i, None, None, None, None,
                                     C.c_void_p(a.ctypes.data) if a.size else None))
        spans.append(OutSpan(node.value, cb.value, a))
    return spans


# ---------------------------------------------------------------- phase API
# Thin wrappers over the phase-level kernels; arguments are torch CUDA tensors.


# ------------------------------------------------ join rows and Q = A R^-1

DEFAULT_JOIN_CAP = 1_000_000  # kDefaultJoinCap (join.hpp:25)


def join_size(relations: Sequence[Relation], tree: JoinTree, cap: int = DEFAULT_JOIN_CAP,
              device: int = 0) -> int:
    """for_each_join_row with an empty sink (join.hpp:47-92): the number of
    join rows; more than `cap` raises size_error."""
    ctx = get_context(device)
    rels = list(relations)
    arr, keep, device_mem = _marshal(rels, "join_size")
    if device_mem:
        ctx.bind_current_stream()
    parent = (C.c_int32 * len(rels))(*tree.parent)
    rows = C.c_int64()
    ctx.check(ctx.lib.fg_join_size(ctx.h, len(rels), arr, tree.root, parent,
                                   L.FG_MEM_DEVICE if device_mem else L.FG_MEM_HOST,
                                   C.c_uint64(cap), C.byref(rows)))
    del keep
    return rows.value


def _out(rows, n, device_mem, like):
    if device_mem:
        import torch
        t = torch.empty((rows, n), dtype=torch.float64, device=like.device)
        return t, t.data_ptr()
    a = np.zeros((rows, n))
    return a, a.ctypes.data


def materialize_join(relations: Sequence[Relation], tree: JoinTree,
                     cap: int = DEFAULT_JOIN_CAP, device: int = 0):
    """materialize_join (join.hpp:96-112): the dense join, rows in
    for_each_join_row order, columns in the pre-order layout."""
    ctx = get_context(device)
    rels = list(relations)
    n = make_layout(rels, tree).total
    rows = join_size(rels, tree, cap, device)
    arr, keep, device_mem = _marshal(rels, "materialize_join")
    if device_mem:
        ctx.bind_current_stream()
    A, ap = _out(rows, n, device_mem, rels[0].data if rels else None)
    if rows and n:
        parent = (C.c_int32 * len(rels))(*tree.parent)
        got = C.c_int64()
        ctx.check(ctx.lib.fg_materialize_join(
            ctx.h, len(rels), arr, tree.root, parent,
            L.FG_MEM_DEVICE if device_mem else L.FG_MEM_HOST, C.c_uint64(cap),
            C.c_void_p(ap), C.byref(got)))
    del keep
    return A


def recover_q(relations: Sequence[Relation], tree: JoinTree, R, cap: int = DEFAULT_JOIN_CAP,
              with_rows: bool = True, device: int = 0):
    """recover_q (postprocess.hpp:293-321) on the GPU: returns (A, Q) -- the
    join rows handed to the reference's sink and Q = A R^-1 -- (A is None
    with with_rows=False).  R: the n x n factor (numpy, or a CUDA tensor when
    the relations are on the device).  Singular R raises rank_error."""
    ctx = get_context(device)
    rels = list(relations)
    n = make_layout(rels, tree).total
    arr, keep, device_mem = _marshal(rels, "recover_q")
    if device_mem:
        import torch
        ctx.bind_current_stream()
        Rc = R.to(torch.float64).contiguous()
        rp = Rc.data_ptr()
    else:
        Rc = np.ascontiguousarray(np.asarray(R, dtype=np.float64))
        rp = Rc.ctypes.data
    if tuple(Rc.shape) != (n, n):
        raise error("recover_q: factor size does not match column layout")
    parent = (C.c_int32 * len(rels))(*tree.parent)
    mem = L.FG_MEM_DEVICE if device_mem else L.FG_MEM_HOST
    rows = C.c_int64()
    # Rank check, then the cap check and the row count (no outputs yet).
    ctx.check(ctx.lib.fg_recover_q(ctx.h, len(rels), arr, tree.root, parent, mem,
                                   C.c_uint64(cap), C.c_void_p(rp), None, None,
                                   C.byref(rows)))
    like = rels[0].data if rels else None
    if rows.value == 0 or n == 0:
        Q, _ = _out(rows.value, n, device_mem, like)
        A = _out(rows.value, n, device_mem, like)[0] if with_rows else None
        del keep, Rc
        return A, Q
    Q, qp = _out(rows.value, n, device_mem, like)
    A, ap = _out(rows.value, n, device_mem, like) if with_rows else (None, None)
    got = C.c_int64()
    ctx.check(ctx.lib.fg_recover_q(ctx.h, len(rels), arr, tree.root, parent, mem,
                                   C.c_uint64(cap), C.c_void_p(rp),
                                   C.c_void_p(ap) if ap else None, C.c_void_p(qp),
                                   C.byref(got)))
    del keep, Rc
    return A, Q


def group_keys(keys, bits: int, device: int = 0):
    """K1: stable grouping of packed uint64 keys (int64 tensor bit pattern).
    Returns (perm int32, begins int32 [G+1], uniq int64 [G])."""
    import torch
    ctx = get_context(device)
    ctx.bind_current_stream()
    keys = keys.contiguous()
    n = keys.numel()
    perm = torch.empty(n, dtype=torch.int32, device=keys.device)
    begins = torch.empty(n + 1, dtype=torch.int32, device=keys.device)
    uniq = torch.empty(max(n, 1), dtype=torch.int64, device=keys.device)
    G = C.c_int64()
    ctx.check(ctx.lib.fg_group_keys(ctx.h, keys.data_ptr(), n, bits, perm.data_ptr(),
                                    begins.data_ptr(), uniq.data_ptr(), C.byref(G)))
    return perm, begins[:G.value + 1].clone(), uniq[:G.value].clone()


def heads_tails(data, begins, perm=None, weights=None, tail_count=None, device: int = 0):
    """K3/K5 on one column block: data (rows, w) f64, begins int32 (G+1).
    Returns (heads (G, w), tails (rows-G, w), scales (G,))."""
    import torch
    ctx = get_context(device)
    ctx.bind_current_stream()
    if data.dtype != torch.float64 or data.stride(1) != 1:
        raise error("heads_tails: data must be float64 with contiguous rows")
    rows, w = data.shape
    G = begins.numel() - 1
    heads = torch.zeros((max(G, 0), w), dtype=torch.float64, device=data.device)
    tails = torch.zeros((max(rows - G, 0), w), dtype=torch.float64, device=data.device)
    scales = torch.zeros(max(G, 0), dtype=torch.float64, device=data.device)
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    ctx.check(ctx.lib.fg_heads_tails(ctx.h, ptr(data), w, w, ptr(perm), ptr(begins), G,
                                     ptr(weights), ptr(tail_count), ptr(heads), w,
                                     ptr(tails) if tails.numel() else None, w, ptr(scales)))
    return heads, tails, scales


def tsqr(blocks, n: int, device: int = 0):
    """K6/K7: sign-normalised n x n R of stacked blocks [(tensor, col_begin)]."""
    import torch
    ctx = get_context(device)
    ctx.bind_current_stream()
    arr = (L.fg_block * max(1, len(blocks)))()
    for i, (t, cb) in enumerate(blocks):
        if t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2:
            raise error("tsqr: blocks must be 2-D float64 CUDA tensors")
        if t.shape[0] > 1 and t.shape[1] > 1 and t.stride(1) != 1:
            raise error("tsqr: block rows must be contiguous (stride(1) == 1)")
        arr[i] = L.fg_block(t.data_ptr(), t.shape[0], max(t.stride(0), t.shape[1]),
                            t.shape[1], cb)
    dev = blocks[0][0].device if blocks else torch.device("cuda", device)
    R = torch.empty((n, n), dtype=torch.float64, device=dev)
    ctx.check(ctx.lib.fg_tsqr(ctx.h, len(blocks), arr, n, R.data_ptr()))
    return R
