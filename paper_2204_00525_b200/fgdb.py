"""FGDB / FGRS binary formats shared by the GPU host, the oracle and tests.

FGDB0001 (a database):
    magic[8] u32 n_rel
    per relation: str name, u32 n_key, str key_attrs..., u32 n_data,
                  str data_attrs..., u64 rows, i64 keys[rows*n_key],
                  f64 data[rows*n_data]          (row-major, little endian)
    i32 root, i32 parent[n_rel]

FGRS0001 (a pipeline result, written by oracle/_ref/figaro_ref):
    magic[8] u32 n_rel u64 N f64 R[N*N] u64 r0_rows u64 input_rows
    f64 seconds_counts seconds_figaro seconds_postprocess seconds_canon
        seconds_pipeline
    per node (index order):
        u64 G, u64 group_begin[G], u64 rows, u32 n_key,
        i64 keys[G*n_key], u64 rows_per_key[G], theta_down[G],
        full_join_size[G], phi_circ[G],
        u32 n_pattr, str pattrs..., u64 P, i64 pkeys[P*n_pattr],
        u64 phi_down[P], phi_up[P]
    u64 n_blocks (or ~0 when R0 was not kept), per block:
        i32 node, u64 col_begin, u64 rows, u64 cols, f64 data[rows*cols]

Strings are u32 length + bytes.  Map orders follow the reference's std::map
iteration order (counts.hpp:24-31), i.e. ascending key tuples.
"""
from __future__ import annotations

import dataclasses
import struct
from typing import List, Optional

import numpy as np


@dataclasses.dataclass
class RelationData:
    name: str
    key_attrs: List[str]
    data_attrs: List[str]
    keys: np.ndarray  # (rows, n_key) int64
    data: np.ndarray  # (rows, n_data) float64

    @property
    def rows(self) -> int:
        return int(self.keys.shape[0])


@dataclasses.dataclass
class Database:
    relations: List[RelationData]
    root: int
    parent: List[int]


def _wstr(f, s: str) -> None:
    b = s.encode()
    f.write(struct.pack("<I", len(b)))
    f.write(b)


def write_fgdb(path: str, db: Database) -> None:
    with open(path, "wb") as f:
        f.write(b"FGDB0001")
        f.write(struct.pack("<I", len(db.relations)))
        for r in db.relations:
            _wstr(f, r.name)
            f.write(struct.pack("<I", len(r.key_attrs)))
            for a in r.key_attrs:
                _wstr(f, a)
            f.write(struct.pack("<I", len(r.data_attrs)))
            for a in r.data_attrs:
                _wstr(f, a)
            f.write(struct.pack("<Q", r.rows))
            np.ascontiguousarray(r.keys, dtype="<i8").tofile(f)
            np.ascontiguousarray(r.data, dtype="<f8").tofile(f)
        f.write(struct.pack("<i", db.root))
        np.asarray(db.parent, dtype="<i4").tofile(f)


class _Rd:
    def __init__(self, buf: bytes):
        self.b = memoryview(buf)
        self.o = 0

    def u32(self) -> int:
        v = struct.unpack_from("<I", self.b, self.o)[0]
        self.o += 4
        return v

    def i32(self) -> int:
        v = struct.unpack_from("<i", self.b, self.o)[0]
        self.o += 4
        return v

    def u64(self) -> int:
        v = struct.unpack_from("<Q", self.b, self.o)[0]
        self.o += 8
        return v

    def f64(self) -> float:
        v = struct.unpack_from("<d", self.b, self.o)[0]
        self.o += 8
        return v

    def s(self) -> str:
        n = self.u32()
        v = bytes(self.b[self.o:self.o + n]).decode()
        self.o += n
        return v

    def arr(self, dtype: str, n: int) -> np.ndarray:
        dt = np.dtype(dtype)
        v = np.frombuffer(self.b, dtype=dt, count=n, offset=self.o).copy()
        self.o += dt.itemsize * n
        return v


def read_fgdb(path: str) -> Database:
    with open(path, "rb") as f:
        rd = _Rd(f.read())
    assert bytes(rd.b[:8]) == b"FGDB0001", "bad FGDB magic"
    rd.o = 8
    n = rd.u32()
    rels = []
    for _ in range(n):
        name = rd.s()
        ka = [rd.s() for _ in range(rd.u32())]
        da = [rd.s() for _ in range(rd.u32())]
        rows = rd.u64()
        keys = rd.arr("<i8", rows * len(ka)).reshape(rows, len(ka))
        data = rd.arr("<f8", rows * len(da)).reshape(rows, len(da))
        rels.append(RelationData(name, ka, da, keys, data))
    root = rd.i32()
    parent = [rd.i32() for _ in range(n)]
    return Database(rels, root, parent)


@dataclasses.dataclass
class NodeCountsData:
    group_begin: np.ndarray  # (G,) u64, Relation::key_groups() begins
    rows: int
    keys: np.ndarray  # (G, n_key) i64, ascending
    rows_per_key: np.ndarray
    theta_down: np.ndarray
    full_join_size: np.ndarray
    phi_circ: np.ndarray
    parent_attrs: List[str]
    pkeys: np.ndarray  # (P, n_pattr)
    phi_down: np.ndarray
    phi_up: np.ndarray


@dataclasses.dataclass
class OutBlockData:
    node: int
    col_begin: int
    rows: np.ndarray


@dataclasses.dataclass
class ResultData:
    R: np.ndarray
    r0_rows: int
    input_rows: int
    seconds_counts: float
    seconds_figaro: float
    seconds_postprocess: float
    seconds_canon: float
    seconds_pipeline: float
    nodes: List[NodeCountsData]
    r0: Optional[List[OutBlockData]]


def read_fgrs(path: str) -> ResultData:
    with open(path, "rb") as f:
        rd = _Rd(f.read())
    assert bytes(rd.b[:8]) == b"FGRS0001", "bad FGRS magic"
    rd.o = 8
    nrel = rd.u32()
    n = rd.u64()
    R = rd.arr("<f8", n * n).reshape(n, n)
    r0_rows = rd.u64()
    input_rows = rd.u64()
    secs = [rd.f64() for _ in range(5)]
    nodes = []
    for _ in range(nrel):
        g = rd.u64()
        gb = rd.arr("<u8", g)
        rows = rd.u64()
        nk = rd.u32()
        keys = rd.arr("<i8", g * nk).reshape(g, nk)
        rpk = rd.arr("<u8", g)
        th = rd.arr("<u8", g)
        fjs = rd.arr("<u8", g)
        circ = rd.arr("<u8", g)
        pa = [rd.s() for _ in range(rd.u32())]
        p = rd.u64()
        pk = rd.arr("<i8", p * len(pa)).reshape(p, len(pa))
        pd = rd.arr("<u8", p)
        pu = rd.arr("<u8", p)
        nodes.append(NodeCountsData(gb, rows, keys, rpk, th, fjs, circ, pa, pk, pd, pu))
    nb = rd.u64()
    r0 = None
    if nb != (1 << 64) - 1:
        r0 = []
        for _ in range(nb):
            node = rd.i32()
            cb = rd.u64()
            rr = rd.u64()
            cc = rd.u64()
            r0.append(OutBlockData(node, cb, rd.arr("<f8", rr * cc).reshape(rr, cc)))
    return ResultData(R, r0_rows, input_rows, *secs, nodes, r0)


def read_fgrm(path: str) -> np.ndarray:
    """A bare square matrix (materialized-join oracle R, ground-truth R)."""
    with open(path, "rb") as f:
        rd = _Rd(f.read())
    assert bytes(rd.b[:8]) == b"FGRM0001", "bad FGRM magic"
    rd.o = 8
    n = rd.u64()
    return rd.arr("<f8", n * n).reshape(n, n)


def read_fgrq(path: str):
    """recover_q output of the reference harness: (A rows, Q rows)."""
    with open(path, "rb") as f:
        rd = _Rd(f.read())
    assert bytes(rd.b[:8]) == b"FGRQ0001", "bad FGRQ magic"
    rd.o = 8
    rows = rd.u64()
    n = rd.u64()
    A = rd.arr("<f8", rows * n).reshape(rows, n)
    Q = rd.arr("<f8", rows * n).reshape(rows, n)
    return A, Q
