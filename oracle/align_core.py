"""Oracle restatement of align_core (TEST INFRASTRUCTURE).

SPEC.md:120-206 with SURVEY Appendix A rows A-K, D1, D2, D8.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from oracle import half_bits as hb


class DegenerateInputError(ValueError):
    """no channel with q_c != 0 and colmax_c != 0."""


class Tier(enum.IntEnum):
    """SPEC.md:129-132.  Value = read bits; SKIP = 0 bits."""

    SKIP = 0
    T8 = 8
    T12 = 12
    T16 = 16

    @property
    def kept_bits(self) -> int:
        return {0: 0, 8: 2, 12: 6, 16: 10}[int(self)]

    @property
    def read_bits(self) -> int:
        return int(self)


@dataclass(frozen=True)
class AlignConfig:
    """SPEC.md:133-136."""

    margin_bits: int = 0
    zero_skip: bool = True

    def __post_init__(self):
        if not -2 <= self.margin_bits <= 4:
            raise ValueError("margin_bits must be in [-2, 4]")


def required_mantissa_bits(product_exp_ub: int, target_u: int, cfg: AlignConfig = AlignConfig()) -> int:
    """clamp(pe - u - 1 + margin, 0, 10)."""
    return int(min(max(product_exp_ub - target_u - 1 + cfg.margin_bits, 0), 10))


def tier_for_bits(t: int) -> Tier:
    """SPEC.md:148-156."""
    if not 0 <= t <= 10:
        raise ValueError(f"kept bits out of range: {t}")
    if t <= 2:
        return Tier.T8
    if t <= 6:
        return Tier.T12
    return Tier.T16


def tier_codes_for_bits(t: np.ndarray) -> np.ndarray:
    """Vector tier_for_bits -> uint8 read-bit codes (8/12/16)."""
    t = np.asarray(t)
    return np.where(t <= 2, 8, np.where(t <= 6, 12, 16)).astype(np.uint8)


def _product_exponents(q_words, colmax_words):
    q = np.asarray(q_words, dtype=np.uint16)
    cm = np.asarray(colmax_words, dtype=np.uint16) & 0x7FFF
    valid = ((q & 0x7FFF) != 0) & (cm != 0)
    pe = hb.magnitude_exponent_array(q) + hb.magnitude_exponent_array(cm) + 1
    return valid, pe


def rule1_target(q_words, colmax_words) -> int:
    """SPEC.md:157-165 / A-K: u = max_valid(e(q_c)+e(colmax_c)+1) - 10."""
    valid, pe = _product_exponents(q_words, colmax_words)
    if not valid.any():
        raise DegenerateInputError("degenerate dot product")
    return int(pe[valid].max()) - 10


UNKNOWN = None


def rule2_targets(o_est) -> list:
    """floor(log2|o|) - 10; zero -> unknown (None)."""
    out = []
    for x in np.asarray(o_est, dtype=np.float64).ravel():
        out.append(None if x == 0.0 else hb.floor_log2(float(x)) - 10)
    return out


def rule2_targets_array(o_est) -> tuple[np.ndarray, np.ndarray]:
    """Vector rule2_targets: (targets int64, known bool)."""
    o = np.asarray(o_est, dtype=np.float64)
    known = o != 0.0
    _, e = np.frexp(np.where(known, o, 1.0))
    return (e.astype(np.int64) - 1 - 10), known


def k_channel_tiers(q_words, colmax_words, cfg: AlignConfig = AlignConfig(), force_tier=None) -> np.ndarray:
    """SPEC.md:175-183 with A-K, D1, D2, D8.  Returns uint8 read-bit codes.

    D1: q_c = +-0 -> SKIP (zero_skip) else T8.
    D2: colmax_c = 0, q_c != 0 -> SKIP (zero_skip) else T16.
    D8: force_tier overrides everything (SKIP included).
    """
    q = np.asarray(q_words, dtype=np.uint16)
    d = q.shape[0]
    if force_tier is not None:
        return np.full(d, int(force_tier), dtype=np.uint8)
    valid, pe = _product_exponents(q, colmax_words)
    if not valid.any():
        raise DegenerateInputError("degenerate dot product")
    u = int(pe[valid].max()) - 10
    t = np.clip(pe - u - 1 + cfg.margin_bits, 0, 10)
    codes = tier_codes_for_bits(t)
    qzero = (q & 0x7FFF) == 0
    cmzero = (np.asarray(colmax_words, dtype=np.uint16) & 0x7FFF) == 0
    if cfg.zero_skip:
        codes = np.where(qzero | cmzero, 0, codes)
    else:
        codes = np.where(qzero, 8, np.where(cmzero, 16, codes))
    return codes.astype(np.uint8)
