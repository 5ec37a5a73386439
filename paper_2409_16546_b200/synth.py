"""Synthetic K/V/Q generator (SynthConfig).

Per (batch b, kv-head h) unit, a numpy PCG64 stream seeded with
SeedSequence([seed, b, h]) draws, in order:
    u_c ~ U[lo, hi] (d values)          per-channel scale 2^u_c
    K = fp16(scale * N(0,1))  [n, d]
    V = fp16(N(0,1))          [n, d]
    Q = fp16(scale * N(0,1))  [g, d]    one row per q-head of the group ("Q like one K row")
so every GPU, rank count and the CPU baseline see identical units.
Default law U[-4, 4]; the paper-like stress variant uses U[-0.5, 0.5].
"""

from __future__ import annotations

import numpy as np

DEFAULT_SEED = 7


def unit_rng(seed: int, b: int, h: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, b, h])))


def generate_unit(n: int, d: int = 128, g: int = 1, seed: int = DEFAULT_SEED, b: int = 0, h: int = 0,
                  scale_lo: float = -4.0, scale_hi: float = 4.0):
    """-> (K [n,d], V [n,d], Q [g,d]) as uint16 fp16 bit patterns."""
    if n < 1 or d < 1:
        raise ValueError("n_tokens and d must be >= 1")
    rng = unit_rng(seed, b, h)
    scale = np.exp2(rng.uniform(scale_lo, scale_hi, d))
    k = (scale * rng.standard_normal((n, d))).astype(np.float16)
    v = rng.standard_normal((n, d)).astype(np.float16)
    q = (scale * rng.standard_normal((g, d))).astype(np.float16)
    return k.view(np.uint16), v.view(np.uint16), q.view(np.uint16)


def _gen_block(args):
    n, d, g, seed, units, n_kv, lo, hi = args
    ks, vs, qs = [], [], []
    for u in units:
        k, v, q = generate_unit(n, d, g, seed, u // n_kv, u % n_kv, lo, hi)
        ks.append(k)
        vs.append(v)
        qs.append(q)
    return np.stack(ks), np.stack(vs), np.stack(qs)


def generate_batch(batch: int, n_kv: int, n: int, d: int = 128, g: int = 1, seed: int = DEFAULT_SEED,
                   scale_lo: float = -4.0, scale_hi: float = 4.0, units=None, workers: int = 1):
    """Stack units -> K, V [U, n, d], Q [U, g, d] (uint16).  `units` restricts to a subset."""
    units = list(range(batch * n_kv)) if units is None else list(units)
    if workers <= 1 or len(units) < 2 * workers:
        return _gen_block((n, d, g, seed, units, n_kv, scale_lo, scale_hi))
    import multiprocessing as mp

    chunks = [units[i::workers] for i in range(workers)]
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_gen_block, [(n, d, g, seed, c, n_kv, scale_lo, scale_hi) for c in chunks])
    K = np.empty((len(units), n, d), np.uint16)
    V = np.empty_like(K)
    Q = np.empty((len(units), g, d), np.uint16)
    for w, (k, v, q) in enumerate(parts):
        K[w::workers], V[w::workers], Q[w::workers] = k, v, q
    return K, V, Q


def fill_store(store, K, V, n_tokens: int, chunk: int = 1024) -> None:
    """Bulk-append tokens [0, n_tokens) of every unit (K, V [U, >=n_tokens, d] uint16) into a
    GPU KVStore in chunks, bounding the host->device staging; raises on non-finite input."""
    import torch

    B, H, d = store.batch, store.n_kv_heads, store.n_dims
    for t0 in range(0, n_tokens, chunk):
        t1 = min(n_tokens, t0 + chunk)
        kt = torch.from_numpy(np.ascontiguousarray(K[:, t0:t1]).view(np.int16)).view(B, H, t1 - t0, d)
        vt = torch.from_numpy(np.ascontiguousarray(V[:, t0:t1]).view(np.int16)).view(B, H, t1 - t0, d)
        store.append(kt, vt)
    store.check()
