"""Oracle restatement of the reference fp16 bit model (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/alignedkv/half_bits.py (HB) and
SPEC.md:26-118.  Every function states the HB lines whose behaviour it
restates; the exhaustive equivalence is asserted by tests/test_oracle_bits.py
(against the reference module when present, else against the committed
digests of its outputs).
"""

from __future__ import annotations

import math

import numpy as np

SIGN = 0x8000
EXP_FIELD = 0x7C00
MANT_FIELD = 0x03FF
BIAS = 15
MANT_BITS = 10
SUBNORMAL_ULP = -24  # HB:28-29


def _u16(words) -> np.ndarray:
    return np.asarray(words, dtype=np.uint16)


def biased_exponent(word: int) -> int:  # HB:48-49
    return (int(word) >> 10) & 0x1F


def finite_mask(words) -> np.ndarray:  # HB:60-62
    return (_u16(words) & EXP_FIELD) != EXP_FIELD


def decode(word: int) -> float:  # HB:65-68
    if not 0 <= word <= 0xFFFF:
        raise ValueError(f"half word out of range: {word}")
    return float(np.array([word], dtype=np.uint16).view(np.float16)[0])


def decode_array(words) -> np.ndarray:  # HB:71-73
    return _u16(words).view(np.float16).astype(np.float64)


def encode(value: float) -> int:  # HB:76-79 (RNE, overflow -> inf)
    with np.errstate(over="ignore"):
        return int(np.array([value], dtype=np.float64).astype(np.float16).view(np.uint16)[0])


def encode_array(values) -> np.ndarray:  # HB:82-85
    with np.errstate(over="ignore"):
        return np.asarray(values, dtype=np.float64).astype(np.float16).view(np.uint16)


def ulp_exponent(word: int) -> int:  # HB:88-96
    b = biased_exponent(word)
    if b == 31:
        raise ValueError(f"non-finite half word 0x{word:04X}")
    return (b if b > 0 else 1) - BIAS - MANT_BITS


def ulp_exponent_array(words) -> np.ndarray:  # HB:99-105
    w = _u16(words)
    if not finite_mask(w).all():
        raise ValueError("non-finite half word in array")
    b = ((w >> 10) & 0x1F).astype(np.int32)
    return np.where(b > 0, b, 1) - BIAS - MANT_BITS


def magnitude_exponent(word: int) -> int:  # HB:108-118
    b = biased_exponent(word)
    if b == 31:
        raise ValueError(f"non-finite half word 0x{word:04X}")
    m = int(word) & MANT_FIELD
    if b > 0:
        return b - BIAS
    if m == 0:
        raise ValueError("zero has no magnitude exponent")
    return m.bit_length() - 1 + SUBNORMAL_ULP


def magnitude_exponent_array(words) -> np.ndarray:
    """Vector form of HB:108-118 for finite non-zero patterns.

    Zeros return a large negative sentinel (-1000); callers that need the
    reference's error for zero must test for it themselves.
    """
    w = _u16(words)
    b = ((w >> 10) & 0x1F).astype(np.int32)
    m = (w & MANT_FIELD).astype(np.int32)
    # floor(log2 m) for m in [1, 1023]
    with np.errstate(divide="ignore"):
        lg = np.where(m > 0, np.floor(np.log2(np.maximum(m, 1))).astype(np.int32), 0)
    e = np.where(b > 0, b - BIAS, lg + SUBNORMAL_ULP)
    return np.where((b == 0) & (m == 0), -1000, e).astype(np.int32)


def truncate_fill(word: int, kept_bits: int) -> int:  # HB:121-137
    if not 0 <= word <= 0xFFFF:
        raise ValueError(f"half word out of range: {word}")
    if not 0 <= kept_bits <= MANT_BITS:
        raise ValueError(f"kept mantissa bits must be in [0, 10], got {kept_bits}")
    if biased_exponent(word) == 31:
        raise ValueError(f"non-finite half word 0x{word:04X}")
    drop = MANT_BITS - kept_bits
    if drop == 0:
        return int(word)
    return (int(word) >> drop << drop) | (1 << (drop - 1))


def truncate_fill_array(words, kept_bits) -> np.ndarray:  # HB:140-151
    w = _u16(words)
    if not finite_mask(w).all():
        raise ValueError("non-finite half word in array")
    t = np.asarray(kept_bits, dtype=np.int64)
    if ((t < 0) | (t > MANT_BITS)).any():
        raise ValueError("kept mantissa bits must be in [0, 10]")
    drop = MANT_BITS - t
    cleared = (w.astype(np.int64) >> drop) << drop
    fill = np.where(drop > 0, np.left_shift(1, np.maximum(drop - 1, 0)), 0)
    return (cleared | fill).astype(np.uint16)


def split_chunks(word: int):  # HB:154-157
    if not 0 <= word <= 0xFFFF:
        raise ValueError(f"half word out of range: {word}")
    return (int(word) >> 8, (int(word) >> 4) & 0xF, int(word) & 0xF)


def split_chunks_array(words):
    w = _u16(words)
    return ((w >> 8).astype(np.uint8), ((w >> 4) & 0xF).astype(np.uint8), (w & 0xF).astype(np.uint8))


def merge_chunks(head: int, mid=None, low=None) -> int:  # HB:160-179
    if not 0 <= head <= 0xFF:
        raise ValueError(f"head chunk out of range: {head}")
    if mid is None:
        if low is not None:
            raise ValueError("non-prefix tier: low nibble without mid nibble")
        return (head << 8) | 0x80
    if not 0 <= mid <= 0xF:
        raise ValueError(f"mid nibble out of range: {mid}")
    if low is None:
        return (head << 8) | (mid << 4) | 0x8
    if not 0 <= low <= 0xF:
        raise ValueError(f"low nibble out of range: {low}")
    return (head << 8) | (mid << 4) | low


def merge_tier_array(head, mid, low, read_bits) -> np.ndarray:
    """Vector merge_chunks keyed by tier read-bits (8/12/16; 0 = SKIP -> 0).

    read_bits broadcasts against the chunk arrays.  SKIP yields word 0 (the
    caller must also zero the product).
    """
    h = np.asarray(head, dtype=np.uint16) << 8
    m = np.asarray(mid, dtype=np.uint16) << 4
    lo = np.asarray(low, dtype=np.uint16)
    rb = np.asarray(read_bits)
    out = np.where(rb >= 16, h | m | lo, np.where(rb >= 12, h | m | 0x8, h | 0x80))
    return np.where(rb == 0, 0, out).astype(np.uint16)


def float16_round(values) -> np.ndarray:  # HB:187-190
    with np.errstate(over="ignore"):
        return np.asarray(values, dtype=np.float64).astype(np.float16).astype(np.float64)


def frexp_exponents(values) -> np.ndarray:  # HB:193-196 (returns -1 for 0.0)
    _, e = np.frexp(np.asarray(values, dtype=np.float64))
    return e.astype(np.int64) - 1


def floor_log2(x: float) -> int:
    """floor(log2|x|) for finite non-zero x (Appendix A notation e(x))."""
    return math.frexp(x)[1] - 1
