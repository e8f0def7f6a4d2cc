"""Seeded synthetic databases with the shapes of BASELINE.json's configs.

The reference's paper datasets are not available (and not needed); these
generators stand in for them with the value distributions BASELINE.json names
(N(0,1) data, Zipf-distributed foreign keys, shuffled rows).  Every database is
emitted fully reduced (no dangling keys), so the reference's
`assume_reduced=true` path and this framework see identical bytes.

Relation r of a config draws from the PCG64 stream seeded by
(base_seed, r, chunk); generation is chunked over threads and deterministic.

configs (scale=1.0 is the BASELINE size):
  C1  R1(k,x1..x4) |><| R2(k,y1..y4): 1,000 keys x 10 rows per relation.
  C2  R1(k,16 cols) |><| R2(k,16 cols): 1M keys x 16 rows per relation.
  C3  D1(F(D2,D3)): F(k1,k2,k3, 8 cols) 100M rows, fkeys Zipf(1.1) over
      1M / 100k / 1k; D1(k1,16) D2(k2,8) D3(k3,4) unique keys, reduced.
  C4  R1(R2(R3)): R1(a,8) 20 rows per a over 200k; R2(a,b,4) uniform pairs;
      R3(b,8) 20 rows per b over 200k.
  C5  R1(k,64) |><| R2(k,64): 8M rows each, k ~ Zipf(1.3) over 100k, column j
      scaled by U[1e-3,1e3]; reduced to shared keys.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from typing import List

import numpy as np

from .fgdb import Database, RelationData

_CHUNK = 1 << 22


def _rng(seed: int, rel: int, chunk: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, rel, chunk])))


def _normal(seed: int, rel: int, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    flat = out.reshape(-1)
    n = flat.size
    nchunks = max(1, (n + _CHUNK - 1) // _CHUNK)

    def work(c):
        lo, hi = c * _CHUNK, min(n, (c + 1) * _CHUNK)
        _rng(seed, rel, 1000 + c).standard_normal(out=flat[lo:hi])

    if nchunks == 1:
        work(0)
    else:
        with cf.ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(work, range(nchunks)))
    return out


def _zipf(rng: np.random.Generator, s: float, n: int, size: int) -> np.ndarray:
    """Ranks 0..n-1 with P(r) ~ 1/(r+1)^s, by inverse CDF."""
    w = 1.0 / np.power(np.arange(1, n + 1, dtype=np.float64), s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), n - 1).astype(np.int64)


def _shuffle(rng, keys, data):
    p = rng.permutation(keys.shape[0])
    return keys[p], data[p]


def two_relation(keys_n: int, rows_per_key: int, cols: int, seed: int,
                 names=("R1", "R2"), prefixes=("x", "y")) -> Database:
    rels = []
    for r in range(2):
        rng = _rng(seed, r)
        k = np.repeat(np.arange(keys_n, dtype=np.int64), rows_per_key).reshape(-1, 1)
        d = _normal(seed, r, k.shape[0], cols)
        k, d = _shuffle(rng, k, d)
        rels.append(RelationData(names[r], ["k"], [f"{prefixes[r]}{j + 1}" for j in range(cols)], k, d))
    return Database(rels, 0, [-1, 0])


def config_c1(seed: int = 7, scale: float = 1.0) -> Database:
    return two_relation(max(1, int(round(1000 * scale))), 10, 4, seed)


def config_c2(seed: int = 7, scale: float = 1.0) -> Database:
    return two_relation(max(1, int(round(1_000_000 * scale))), 16, 16, seed)


def config_c5(seed: int = 7, scale: float = 1.0, cols: int = 64) -> Database:
    rows = max(2, int(round(8_000_000 * scale)))
    nkeys = 100_000
    raw = []
    for r in range(2):
        rng = _rng(seed, r)
        raw.append(_zipf(rng, 1.3, nkeys, rows))
    shared = np.intersect1d(np.unique(raw[0]), np.unique(raw[1]))
    rels = []
    for r in range(2):
        rng = _rng(seed, r, 1)
        keep = np.isin(raw[r], shared)
        k = raw[r][keep].reshape(-1, 1)
        d = _normal(seed, r, k.shape[0], cols)
        d *= rng.uniform(1e-3, 1e3, size=cols)[None, :]
        k, d = _shuffle(rng, k, d)
        rels.append(RelationData(f"R{r + 1}", ["k"], [f"{'xy'[r]}{j + 1}" for j in range(cols)], k, d))
    return Database(rels, 0, [-1, 0])


def config_c3(seed: int = 7, scale: float = 1.0) -> Database:
    """D1(F(D2,D3)); F declares its parent attribute k1 first."""
    f_rows = max(1, int(round(100_000_000 * scale)))
    n1, n2, n3 = (max(1, int(round(x * scale))) if scale < 1 else x
                  for x in (1_000_000, 100_000, 1_000))
    rng = _rng(seed, 1)
    fk = np.stack([_zipf(rng, 1.1, n1, f_rows), _zipf(rng, 1.1, n2, f_rows),
                   _zipf(rng, 1.1, n3, f_rows)], axis=1)
    fd = _normal(seed, 1, f_rows, 8)
    fk, fd = _shuffle(rng, fk, fd)
    F = RelationData("F", ["k1", "k2", "k3"], [f"f{j + 1}" for j in range(8)], fk, fd)

    def dim(idx, name, attr, col, n, cols):
        present = np.unique(fk[:, col])
        r = _rng(seed, idx)
        d = _normal(seed, idx, present.shape[0], cols)
        k, d = _shuffle(r, present.reshape(-1, 1), d)
        return RelationData(name, [attr], [f"{name.lower()}_{j + 1}" for j in range(cols)], k, d)

    D1 = dim(0, "D1", "k1", 0, n1, 16)
    D2 = dim(2, "D2", "k2", 1, n2, 8)
    D3 = dim(3, "D3", "k3", 2, n3, 4)
    return Database([D1, F, D2, D3], 0, [-1, 0, 1, 1])


def config_c4(seed: int = 7, scale: float = 1.0) -> Database:
    """R1(R2(R3)); R2 declares its parent attribute a first."""
    na = max(1, int(round(200_000 * scale)))
    nb = na
    r2_rows = 20 * na
    rng2 = _rng(seed, 1)
    ab = np.stack([rng2.integers(0, na, r2_rows), rng2.integers(0, nb, r2_rows)], axis=1).astype(np.int64)
    a_present = np.unique(ab[:, 0])
    b_present = np.unique(ab[:, 1])
    rng1 = _rng(seed, 0)
    k1 = np.repeat(a_present, 20).reshape(-1, 1)
    d1 = _normal(seed, 0, k1.shape[0], 8)
    k1, d1 = _shuffle(rng1, k1, d1)
    d2 = _normal(seed, 1, r2_rows, 4)
    ab, d2 = _shuffle(rng2, ab, d2)
    rng3 = _rng(seed, 2)
    k3 = np.repeat(b_present, 20).reshape(-1, 1)
    d3 = _normal(seed, 2, k3.shape[0], 8)
    k3, d3 = _shuffle(rng3, k3, d3)
    return Database([
        RelationData("R1", ["a"], [f"u{j + 1}" for j in range(8)], k1, d1),
        RelationData("R2", ["a", "b"], [f"v{j + 1}" for j in range(4)], ab, d2),
        RelationData("R3", ["b"], [f"w{j + 1}" for j in range(8)], k3, d3),
    ], 0, [-1, 0, 1])


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}


def make(config: str, seed: int = 7, scale: float = 1.0) -> Database:
    return CONFIGS[config](seed=seed, scale=scale)


def input_rows(db: Database) -> int:
    return sum(r.rows for r in db.relations)
