"""Per-head parity check of a GPU decode step against the oracle (TEST INFRASTRUCTURE).

The SURVEY §8(c) parity contract as one function, shared by `tests/` and by
`bench.py`'s post-run validation sample (which runs after the timed region and
is never the thing measured):

  * K tier mask (k_channel_tiers): bit-exact;
  * scores and output: |gpu - ref| <= 1e-3 |ref| + 1e-3 max|ref| per vector;
  * K-side AccessCounter: exact;
  * selection set (estimate_output, D3), V tier mask
    (output_aligned) and V-side counters: bit-exact, except
    that a D11 knife-edge head (float-derived decisions within 2^-18 of a
    boundary, `attention_decode.knife_edges`) skips the selection / V-mask /
    V-counter asserts on the affected rows / columns;
  * injection (D11): the GPU's own p, selection and targets pushed through the
    oracle's element rule (`v_element_codes`) must reproduce the GPU V mask
    exactly — for every head, knife-edge or not.
"""

from __future__ import annotations

import numpy as np

from oracle import attention_decode as OA
from oracle.align_core import AlignConfig

TARGET_UNKNOWN = -(1 << 31)


def close(gpu, ref, rtol: float = 1e-3) -> bool:
    """|gpu - ref| <= rtol*|ref| + rtol*max|ref| (per vector)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = rtol * np.abs(ref) + rtol * np.max(np.abs(ref), axis=-1, keepdims=True)
    return bool(np.all(np.abs(gpu - ref) <= tol + 1e-30))


def check_head(ref: "OA.HeadResult", *, k_tiers, o, counters, sel=None, v_tiers=None, s=None, p=None,
               targets=None, v_head=None, cfg: AlignConfig = AlignConfig(), strategy: str = "element",
               force=None):
    """Compare one q-head's GPU outputs with the oracle's HeadResult.

    Returns (failures: list[str], knife_edge: bool) — knife_edge is True when any
    D11 exclusion applied (a selection edge, or excluded rows / columns).  Optional
    arguments that are None are not checked (the serving path exports no V mask).
    """
    fail = []
    counters = np.asarray(counters)
    if not np.array_equal(np.asarray(k_tiers), ref.k_tiers):
        fail.append("k_tiers")
    if s is not None and not close(s, ref.s):
        fail.append("scores")
    if not close(o, ref.o):
        fail.append("o")
    if tuple(int(x) for x in counters[:3]) != ref.k_counter.as_tuple():
        fail.append("k_counter")
    n = ref.p.shape[0]
    d = ref.k_tiers.shape[0]
    if force is None:
        rows, cols, edge = OA.knife_edges(ref.p, ref.o_est, ref.sel)
        # a selected row is read at T16 whatever its p (D6): no decision sits on its edge
        # (the argmax of a one-hot softmax has p = 1.0 exactly, log2 p = 0)
        rows[np.asarray(ref.sel, dtype=np.int64)] = False
        if strategy == "element" and v_head is not None and (rows.any() or cols.any()):
            rows, cols = _flipping(ref, rows, cols, v_head, cfg)
    else:
        rows, cols, edge = np.zeros(n, bool), np.zeros(d, bool), False
    if sel is not None and not edge and not np.array_equal(np.asarray(sel), ref.sel):
        fail.append("selection")
    if v_tiers is not None:
        vt = np.asarray(v_tiers)
        if not edge:
            keep = ~rows[:, None] & ~cols[None, :]
            if not np.array_equal(vt[keep], ref.v_tiers[keep]):
                fail.append("v_tiers")
        # injection: the GPU's own p / sel / targets through the oracle rule -> 100 % exact
        if force is None and strategy == "element" and p is not None and targets is not None and v_head is not None:
            tg = np.asarray(targets).astype(np.int64)
            known = tg != TARGET_UNKNOWN
            inj = OA.v_element_codes(np.asarray(p, np.float64), np.asarray(sel), tg, known, v_head, cfg)
            if not np.array_equal(vt, inj):
                fail.append("v_tiers_injection")
    if not edge and not rows.any() and not cols.any():
        if tuple(int(x) for x in counters[3:6]) != ref.v_counter.as_tuple():
            fail.append("v_counter")
    return fail, bool(edge or rows.any() or cols.any())


def _flipping(ref, rows, cols, v_head, cfg):
    """Keep only the knife-edge rows / columns whose V tiers actually change when the
    float-derived exponent (e(p_t) per row, the Rule-2 target per column) is read one
    lower or one higher; an edge that cannot flip a tier is no ambiguity (e.g. a p_t of
    1e-61 sits at e(p) = -201 +- 1: T8 either way)."""
    from oracle.align_core import rule2_targets_array

    tg, known = rule2_targets_array(ref.o_est)
    base = OA.v_element_codes(ref.p, ref.sel, tg, known, v_head, cfg)
    keep_r = np.zeros_like(rows)
    if rows.any():
        for f in (2.0, 0.5):
            pp = ref.p.copy()
            pp[rows] *= f
            keep_r |= rows & (OA.v_element_codes(pp, ref.sel, tg, known, v_head, cfg) != base).any(axis=1)
    keep_c = np.zeros_like(cols)
    if cols.any():
        for dlt in (1, -1):
            t2 = np.asarray(tg).copy()
            t2[cols] += dlt
            keep_c |= cols & (OA.v_element_codes(ref.p, ref.sel, t2, known, v_head, cfg) != base).any(axis=0)
    return keep_r, keep_c


def knife_edge_kind(ref: "OA.HeadResult"):
    """(selection_edge, excluded_rows, excluded_cols) of one head under D11, for reporting."""
    rows, cols, edge = OA.knife_edges(ref.p, ref.o_est, ref.sel)
    rows[np.asarray(ref.sel, dtype=np.int64)] = False
    return bool(edge), int(rows.sum()), int(cols.sum())
