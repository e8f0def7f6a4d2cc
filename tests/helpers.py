"""Shared test helpers (comparisons; the oracle stays the checker only)."""
import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def golden_stems(prefix=""):
    return sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.fgdb")))


def full_rank(R, tol=1e-8):
    if R.size == 0:
        return True
    d = np.abs(np.diag(R))
    return bool(np.all(d > tol * max(np.abs(R).max(), 1e-300)))


def rel_fro(a, b):
    ref = float(np.sum(b * b))
    diff = float(np.sum((a - b) ** 2))
    return np.sqrt(diff) if ref == 0 else np.sqrt(diff / ref)


def r_distance(R, Rref):
    """Relative Frobenius distance of sign-normalised R factors; for a
    rank-deficient reference R is not unique, so the Grams are compared."""
    if full_rank(Rref):
        return rel_fro(R, Rref)
    return rel_fro(R.T @ R, Rref.T @ Rref)


def blocks_to_spans(blocks):
    """Groups the reference's OutBlocks into spans: consecutive blocks with
    the same (node, col_begin, width), stacked."""
    spans = []
    for b in blocks:
        key = (b.node, b.col_begin, b.rows.shape[1])
        if spans and spans[-1][0] == key:
            spans[-1][1].append(b.rows)
        else:
            spans.append((key, [b.rows]))
    return [(k, np.vstack(v)) for k, v in spans]
