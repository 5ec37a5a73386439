"""align_core host API.

The batched GPU path evaluates these rules inside the kernels (akv_qk
prologue for Rule 1, akv_softmax_select for Rule 2, akv_pv for the per-element
V tiers).  This module keeps the reference's public names and scalar
semantics for callers that use them directly: `Tier`, `AlignConfig`,
`DegenerateInputError`, `required_mantissa_bits`, `tier_for_bits`,
`rule1_target`, `rule2_targets`, `k_channel_tiers`.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import Optional, Sequence


class DegenerateInputError(ValueError):
    """No channel with q_c != 0 and colmax_c != 0."""


class Tier(enum.IntEnum):
    """Read tier; the value is the number of bits read.

    SKIP (0 bits) marks zero-q channels under zero_skip.
    """

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
    """margin_bits in [-2, 4] (default 0), zero_skip (default on)."""

    margin_bits: int = 0
    zero_skip: bool = True

    def __post_init__(self):
        if not isinstance(self.margin_bits, int) or not -2 <= self.margin_bits <= 4:
            raise ValueError("margin_bits must be an integer in [-2, 4]")


def _mag_exp(word: int) -> int:
    """floor(log2|x|) of a finite non-zero fp16 pattern (subnormal aware)."""
    b = (word >> 10) & 0x1F
    if b:
        return b - 15
    return (word & 0x3FF).bit_length() - 1 - 24


def required_mantissa_bits(product_exp_ub: int, target_u: int, cfg: AlignConfig = AlignConfig()) -> int:
    """clamp(product_exp_ub - target - 1 + margin, 0, 10)."""
    return max(0, min(10, product_exp_ub - target_u - 1 + cfg.margin_bits))


def tier_for_bits(t: int) -> Tier:
    """t <= 2 -> T8, 3..6 -> T12, >= 7 -> T16."""
    if not 0 <= t <= 10:
        raise ValueError(f"kept bits out of range: {t}")
    return Tier.T8 if t <= 2 else (Tier.T12 if t <= 6 else Tier.T16)


def _valid_products(q_words: Sequence[int], colmax_words: Sequence[int]):
    if len(q_words) != len(colmax_words):
        raise ValueError("q and colmax lengths differ")
    out = []
    for q, cm in zip(q_words, colmax_words):
        q, cm = int(q) & 0xFFFF, int(cm) & 0x7FFF
        if ((q >> 10) & 0x1F) == 31 or ((cm >> 10) & 0x1F) == 31:
            raise ValueError("non-finite input")
        out.append(_mag_exp(q) + _mag_exp(cm) + 1 if (q & 0x7FFF) and cm else None)
    return out


def rule1_target(q_words: Sequence[int], colmax_words: Sequence[int]) -> int:
    """u = max over valid channels of e(q)+e(colmax)+1, minus 10."""
    pes = [p for p in _valid_products(q_words, colmax_words) if p is not None]
    if not pes:
        raise DegenerateInputError("degenerate dot product")
    return max(pes) - 10


def rule2_targets(o_est: Sequence[float]) -> list:
    """floor(log2|o|) - 10 per dim; 0 -> None (unknown, forces T16)."""
    return [None if float(x) == 0.0 else math.frexp(float(x))[1] - 1 - 10 for x in o_est]


def k_channel_tiers(q_words: Sequence[int], colmax_words: Sequence[int], cfg: AlignConfig = AlignConfig(),
                    force_tier: Optional[int] = None) -> list:
    """Per-channel K tiers (zero handling SURVEY App. A D1/D2/D8)."""
    if force_tier is not None:
        return [Tier(int(force_tier))] * len(q_words)
    pes = _valid_products(q_words, colmax_words)
    u = rule1_target(q_words, colmax_words)
    out = []
    for q, cm, pe in zip(q_words, colmax_words, pes):
        qz, cz = (int(q) & 0x7FFF) == 0, (int(cm) & 0x7FFF) == 0
        if qz or cz:
            out.append(Tier.SKIP if cfg.zero_skip else (Tier.T8 if qz else Tier.T16))
        else:
            out.append(tier_for_bits(required_mantissa_bits(pe, u, cfg)))
    return out
