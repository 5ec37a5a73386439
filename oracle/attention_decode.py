"""Oracle restatement of attention_decode (TEST INFRASTRUCTURE).

SPEC.md:292-393 with SURVEY Appendix A (D3-D9, D11).  float64 throughout;
half x half products are exact in float64 and sums use numpy's
deterministic pairwise reduction (no BLAS), so results do not depend on
thread counts (D9).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from oracle import half_bits as hb
from oracle.align_core import AlignConfig, k_channel_tiers, rule2_targets_array, tier_codes_for_bits
from oracle.kv_store import AccessCounter, KVStore, PlaneTensor


# --------------------------------------------------------------------------
# scores
# --------------------------------------------------------------------------
def scores_from_words(q_words, k_words, codes) -> np.ndarray:
    """s_t = sum_c q_c * K~[t,c] / sqrt(d) with per-channel read codes."""
    q = hb.decode_array(q_words)
    c0, c1, c2 = hb.split_chunks_array(k_words)
    kt = hb.decode_array(hb.merge_tier_array(c0, c1, c2, codes[None, :]))
    kt = np.where(np.asarray(codes)[None, :] == 0, 0.0, kt)
    acc = np.sum(kt * q[None, :], axis=1)
    return acc / math.sqrt(q.shape[0])


def scores_aligned(q_words, store: KVStore, cfg: AlignConfig = AlignConfig(), force_tier=None):
    """SPEC.md:315-323 -> (s, AccessCounter, k_tiers)."""
    codes = k_channel_tiers(q_words, store.colmax, cfg, force_tier)
    n = store.n_tokens
    counter = AccessCounter()
    counter.add_codes(np.repeat(codes[None, :], n, axis=0))
    s = scores_from_words(q_words, store.k.words(), codes)
    return s, counter, codes


def reference_scores(q_words, k_words) -> np.ndarray:
    """all-T16 chain (R_normal)."""
    d = np.asarray(q_words).shape[0]
    return scores_from_words(q_words, k_words, np.full(d, 16, np.uint8))


# --------------------------------------------------------------------------
# softmax
# --------------------------------------------------------------------------
def softmax(s) -> np.ndarray:
    s = np.asarray(s, dtype=np.float64)
    e = np.exp(s - s.max())
    return e / e.sum()


# --------------------------------------------------------------------------
# estimation (D3)
# --------------------------------------------------------------------------
def select_tokens(p, k_sel: int = 32, m: int = 5) -> np.ndarray:
    """Threshold-then-cap approximate top-k; ties by (p desc, t asc). Sorted asc."""
    p = np.asarray(p, dtype=np.float64)
    thr = p.max() * 2.0 ** (-m)
    cand = np.nonzero(p >= thr)[0]
    if cand.size > k_sel:
        order = np.lexsort((cand, -p[cand]))  # primary -p, secondary t
        cand = cand[order[:k_sel]]
    return np.sort(cand)


def estimate_output(p, store: KVStore, k_sel: int = 32, m: int = 5):
    """-> (o_est[d], sel, AccessCounter)."""
    sel = select_tokens(p, k_sel, m)
    v = hb.decode_array(store.v.words()[sel])
    o_est = np.sum(np.asarray(p)[sel][:, None] * v, axis=0)
    counter = AccessCounter()
    counter.add(16, sel.size * store.n_dims)
    return o_est, sel, counter


# --------------------------------------------------------------------------
# aligned output (D4-D7)
# --------------------------------------------------------------------------
def v_element_codes(p, sel, targets, known, v_head, cfg: AlignConfig = AlignConfig()) -> np.ndarray:
    """Per-element V read codes [n, d] for the element strategy.

    target unknown -> 16 ("force tier T16 for reads contributing to
    them", applied after and therefore over the p_t == 0 rule); p_t == 0 -> 8 (D5);
    e_v = max(bexp,1) - 15 from the head byte (D4); selected rows -> 16 (D6).
    Usable with the GPU's own p/sel/targets (injection check, D11).
    """
    p = np.asarray(p, dtype=np.float64)
    n = p.shape[0]
    bexp = ((np.asarray(v_head, dtype=np.int32) >> 2) & 0x1F)
    e_v = np.maximum(bexp, 1) - 15
    pos = p > 0
    _, ep = np.frexp(np.where(pos, p, 1.0))
    e_p = ep.astype(np.int64) - 1
    t_req = np.clip(e_p[:, None] + e_v + 1 - np.asarray(targets)[None, :] - 1 + cfg.margin_bits, 0, 10)
    codes = tier_codes_for_bits(t_req)
    codes = np.where(pos[:, None], codes, 8)
    codes = np.where(np.asarray(known)[None, :], codes, 16)
    if len(sel):
        codes[np.asarray(sel)] = 16
    return codes.astype(np.uint8).reshape(n, -1)


def v_row_codes(p, sel, targets, known, rowmax, d: int, cfg: AlignConfig = AlignConfig()) -> np.ndarray:
    """Row strategy (D7): one tier per token from RowMax."""
    p = np.asarray(p, dtype=np.float64)
    n = p.shape[0]
    known = np.asarray(known)
    if not known.all():
        codes = np.full(n, 16, np.uint8)
    else:
        tmin = int(np.asarray(targets).min())
        rm = np.asarray(rowmax, dtype=np.uint16)
        e_rm = hb.magnitude_exponent_array(rm)
        pos = p > 0
        _, ep = np.frexp(np.where(pos, p, 1.0))
        e_p = ep.astype(np.int64) - 1
        t_req = np.clip(e_p + e_rm + 1 - tmin - 1 + cfg.margin_bits, 0, 10)
        codes = tier_codes_for_bits(t_req)
        codes = np.where(pos & (rm != 0), codes, 8).astype(np.uint8)
    codes = np.repeat(codes[:, None], d, axis=1)
    if len(sel):
        codes[np.asarray(sel)] = 16
    return codes


def output_from_codes(p, v_words, codes) -> np.ndarray:
    c0, c1, c2 = hb.split_chunks_array(v_words)
    vt = hb.decode_array(hb.merge_tier_array(c0, c1, c2, codes))
    return np.sum(np.asarray(p, dtype=np.float64)[:, None] * vt, axis=0)


def output_aligned(p, store: KVStore, o_est=None, sel=None, cfg: AlignConfig = AlignConfig(),
                   strategy: str = "element", force_tier=None):
    """-> (o[d], AccessCounter (PV reads only, t not in sel), codes[n,d])."""
    n, d = store.n_tokens, store.n_dims
    words = store.v.words()
    if force_tier is not None:
        codes = np.full((n, d), int(force_tier), np.uint8)
        sel = np.zeros(0, np.int64)
    else:
        if o_est is None:
            raise ValueError("missing o_est")
        targets, known = rule2_targets_array(o_est)
        if strategy == "element":
            codes = v_element_codes(p, sel, targets, known, words >> 8, cfg)
        elif strategy == "row":
            codes = v_row_codes(p, sel, targets, known, store.rowmax, d, cfg)
        else:
            raise ValueError(f"unknown strategy {strategy!r}")
    counter = AccessCounter()
    mask = np.ones(n, bool)
    if len(sel):
        mask[np.asarray(sel)] = False
    counter.add_codes(codes[mask])
    o = output_from_codes(p, words, codes)
    return o, counter, codes


def reference_output(p, v_words) -> np.ndarray:
    """SPEC.md:351-359."""
    v = np.asarray(v_words, dtype=np.uint16)
    return output_from_codes(p, v, np.full(v.shape, 16, np.uint8))


def baseline_truncated(q_words, k_words, p, v_words, bits: int = 13):
    """every element truncate_fill'ed to bits-6 kept bits."""
    if not 8 <= bits <= 16:
        raise ValueError("bits must be in [8, 16]")
    kt = hb.truncate_fill_array(k_words, bits - 6)
    vt = hb.truncate_fill_array(v_words, bits - 6)
    q = hb.decode_array(q_words)
    s = np.sum(hb.decode_array(kt) * q[None, :], axis=1) / math.sqrt(q.shape[0])
    o = np.sum(np.asarray(p, dtype=np.float64)[:, None] * hb.decode_array(vt), axis=0)
    return s, o


# --------------------------------------------------------------------------
# one decode step for one q-head (SPEC.md call stack)
# --------------------------------------------------------------------------
@dataclass
class HeadResult:
    s: np.ndarray
    p: np.ndarray
    k_tiers: np.ndarray
    sel: np.ndarray
    o_est: np.ndarray
    v_tiers: np.ndarray
    o: np.ndarray
    k_counter: AccessCounter
    v_counter: AccessCounter


def decode_head(q_words, store: KVStore, cfg: AlignConfig = AlignConfig(), k_sel: int = 32, m: int = 5,
                strategy: str = "element", force_tier=None) -> HeadResult:
    s, kc, ktiers = scores_aligned(q_words, store, cfg, force_tier)
    p = softmax(s)
    if force_tier is None:
        o_est, sel, ec = estimate_output(p, store, k_sel, m)
    else:
        o_est, sel, ec = np.zeros(store.n_dims), np.zeros(0, np.int64), AccessCounter()
    o, vc, vt = output_aligned(p, store, o_est, sel, cfg, strategy, force_tier)
    return HeadResult(s, p, ktiers, sel, o_est, vt, o, kc, ec.merge(vc))


def knife_edges(p, o_est, sel, k_sel: int = 32, m: int = 5, eps: float = 2.0 ** -18):
    """D11: rows/cols whose float-derived V decisions sit on a knife edge.

    Returns (bad_rows bool[n], bad_cols bool[d], selection_edge bool).
    """
    p = np.asarray(p, dtype=np.float64)
    pos = p > 0
    lg = np.log2(np.where(pos, p, 1.0))
    bad_rows = pos & (np.abs(lg - np.round(lg)) < eps)
    o = np.asarray(o_est, dtype=np.float64)
    nz = o != 0
    lo = np.log2(np.where(nz, np.abs(o), 1.0))
    bad_cols = nz & (np.abs(lo - np.round(lo)) < eps)
    thr = p.max() * 2.0 ** (-m)
    edge = bool(np.any(np.abs(p - thr) <= eps * thr))
    cand = np.nonzero(p >= thr)[0]
    if cand.size > k_sel:
        ps = np.sort(p[cand])[::-1]
        kth = ps[k_sel - 1]
        nxt = ps[k_sel] if ps.size > k_sel else -1.0
        edge = edge or (kth - nxt) <= eps * kth
    return bad_rows, bad_cols, edge
