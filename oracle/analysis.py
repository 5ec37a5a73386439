"""Oracle restatement of the analysis module pieces used by the parity
harness (TEST INFRASTRUCTURE): SPEC.md:410-418 (histogram), :428-436
(brute-force alignment optimality)."""

from __future__ import annotations

import itertools

import numpy as np

from oracle.align_core import AlignConfig, required_mantissa_bits

BUCKET_EDGES = (1.0 / 1024, 1.0 / 512, 1.0 / 256, 1.0 / 128)


def relative_error_buckets(test, ref) -> np.ndarray:
    """Bucket index 0..5 per element (boundaries :401,453)."""
    t = np.asarray(test, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    if t.shape != r.shape:
        raise ValueError("length mismatch")
    out = np.empty(t.shape, np.int64)
    rz = r == 0
    out[rz] = np.where(t[rz] == 0, 0, 5)
    nz = ~rz
    rel = np.abs(t[nz] - r[nz]) / np.abs(r[nz])
    b = np.where(rel == 0, 0, 1 + np.searchsorted(np.asarray(BUCKET_EDGES), rel, side="right"))
    out[nz] = b
    return out


def relative_error_histogram(test, ref) -> np.ndarray:
    """Fractions over the six Table-1 buckets."""
    b = relative_error_buckets(test, ref)
    counts = np.bincount(b, minlength=6).astype(np.float64)
    return counts / max(b.size, 1)


def alignment_bruteforce(product_exps, target_u: int, cfg: AlignConfig = AlignConfig()):
    """SPEC.md:428-436 -> (min_total_bits or None if infeasible, aligned_total)."""
    exps = list(product_exps)
    if len(exps) > 4:
        raise ValueError("at most 4 products")
    aligned = sum(required_mantissa_bits(e, target_u, cfg) for e in exps)
    best = None
    for ts in itertools.product(range(11), repeat=len(exps)):
        # truncating to t kept bits bounds the product error by 2^(pe-1-t)
        if all(e - 1 - t <= target_u for e, t in zip(exps, ts)):
            tot = sum(ts)
            best = tot if best is None else min(best, tot)
    return best, aligned
