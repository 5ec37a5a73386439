"""Oracle restatement of kv_store (TEST INFRASTRUCTURE).

SPEC.md:208-290: PlaneTensor (3 row-major planes, nibbles low-first,
SPEC.md:214,277), ColMax, RowMax,
metered reads and AccessCounter.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import half_bits as hb
from oracle.align_core import Tier


@dataclass
class AccessCounter:
    """bits = 8*T8 + 12*T12 + 16*T16; SKIP excluded."""

    t8: int = 0
    t12: int = 0
    t16: int = 0

    @property
    def bits_read(self) -> int:
        return 8 * self.t8 + 12 * self.t12 + 16 * self.t16

    @property
    def elements_read(self) -> int:
        return self.t8 + self.t12 + self.t16

    def add(self, tier, count: int = 1) -> None:
        tier = int(tier)
        if tier == 8:
            self.t8 += count
        elif tier == 12:
            self.t12 += count
        elif tier == 16:
            self.t16 += count
        elif tier != 0:
            raise ValueError(f"bad tier {tier}")

    def add_codes(self, codes) -> None:
        c = np.asarray(codes)
        self.t8 += int((c == 8).sum())
        self.t12 += int((c == 12).sum())
        self.t16 += int((c == 16).sum())

    def merge(self, other: "AccessCounter") -> "AccessCounter":
        return AccessCounter(self.t8 + other.t8, self.t12 + other.t12, self.t16 + other.t16)

    def as_tuple(self):
        return (self.t8, self.t12, self.t16)


def average_bit_width(counter: AccessCounter) -> float:
    """SPEC.md:260-268."""
    if counter.elements_read == 0:
        raise ValueError("no reads recorded")
    return counter.bits_read / counter.elements_read


def pack_nibbles_rowmajor(nib: np.ndarray) -> np.ndarray:
    """byte j = nib[2j] | nib[2j+1] << 4 (low nibble first)."""
    nib = np.asarray(nib, dtype=np.uint8)
    return (nib[..., 0::2] | (nib[..., 1::2] << 4)).astype(np.uint8)


def unpack_nibbles_rowmajor(packed: np.ndarray, d: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (d,), dtype=np.uint8)
    out[..., 0::2] = p & 0xF
    out[..., 1::2] = p >> 4
    return out


@dataclass
class PlaneTensor:
    """SPEC.md:213-218.  plane0 [n,d] u8; plane1/plane2 [n,d/2] u8."""

    n_dims: int
    plane0: np.ndarray = None
    plane1: np.ndarray = None
    plane2: np.ndarray = None

    def __post_init__(self):
        if self.n_dims % 2:
            raise ValueError("n_dims must be even (A-planes)")
        if self.plane0 is None:
            self.plane0 = np.zeros((0, self.n_dims), np.uint8)
            self.plane1 = np.zeros((0, self.n_dims // 2), np.uint8)
            self.plane2 = np.zeros((0, self.n_dims // 2), np.uint8)

    @property
    def n_tokens(self) -> int:
        return self.plane0.shape[0]

    @classmethod
    def from_words(cls, words) -> "PlaneTensor":
        w = np.asarray(words, dtype=np.uint16)
        c0, c1, c2 = hb.split_chunks_array(w)
        return cls(w.shape[1], c0.copy(), pack_nibbles_rowmajor(c1), pack_nibbles_rowmajor(c2))

    def append_rows(self, words) -> None:
        w = np.atleast_2d(np.asarray(words, dtype=np.uint16))
        other = PlaneTensor.from_words(w)
        self.plane0 = np.concatenate([self.plane0, other.plane0])
        self.plane1 = np.concatenate([self.plane1, other.plane1])
        self.plane2 = np.concatenate([self.plane2, other.plane2])

    def chunks(self):
        d = self.n_dims
        return (self.plane0, unpack_nibbles_rowmajor(self.plane1, d), unpack_nibbles_rowmajor(self.plane2, d))

    def words(self) -> np.ndarray:
        c0, c1, c2 = self.chunks()
        return ((c0.astype(np.uint16) << 8) | (c1.astype(np.uint16) << 4) | c2).astype(np.uint16)

    def nbytes(self) -> int:
        return self.plane0.nbytes + self.plane1.nbytes + self.plane2.nbytes


class KVStore:
    """SPEC.md:233-268 for one (batch, kv-head) unit."""

    def __init__(self, n_dims: int = 128):
        self.n_dims = n_dims
        self.k = PlaneTensor(n_dims)
        self.v = PlaneTensor(n_dims)
        self.colmax = np.zeros(n_dims, np.uint16)
        self.rowmax = np.zeros(0, np.uint16)

    @property
    def n_tokens(self) -> int:
        return self.k.n_tokens

    def append_token(self, k_row, v_row) -> None:
        """validate, split, append, update ColMax/RowMax."""
        self.append_rows(np.atleast_2d(k_row), np.atleast_2d(v_row))

    def append_rows(self, k_rows, v_rows) -> None:
        k = np.asarray(k_rows, dtype=np.uint16)
        v = np.asarray(v_rows, dtype=np.uint16)
        if k.shape != v.shape or k.shape[-1] != self.n_dims:
            raise ValueError("row length mismatch")
        for name, a in (("K", k), ("V", v)):
            bad = ~hb.finite_mask(a)
            if bad.any():
                t, c = np.argwhere(bad)[0]
                raise ValueError(
                    f"non-finite half word 0x{int(a[t, c]):04X} in {name} at token {self.n_tokens + int(t)}, channel {int(c)}"
                )
        self.k.append_rows(k)
        self.v.append_rows(v)
        self.colmax = np.maximum(self.colmax, (k & 0x7FFF).max(axis=0)).astype(np.uint16)
        self.rowmax = np.concatenate([self.rowmax, (v & 0x7FFF).max(axis=1).astype(np.uint16)])

    # ---- metered reads -------------------------------
    def read_element(self, plane: PlaneTensor, t: int, c: int, tier, counter: AccessCounter):
        if not (0 <= t < plane.n_tokens and 0 <= c < plane.n_dims):
            raise IndexError("read out of range")
        tier = int(tier)
        if tier == 0:
            return 0
        c0 = int(plane.plane0[t, c])
        b1 = int(plane.plane1[t, c // 2])
        b2 = int(plane.plane2[t, c // 2])
        n1 = (b1 >> 4) if c & 1 else (b1 & 0xF)
        n2 = (b2 >> 4) if c & 1 else (b2 & 0xF)
        counter.add(tier)
        if tier == 8:
            return hb.merge_chunks(c0)
        if tier == 12:
            return hb.merge_chunks(c0, n1)
        return hb.merge_chunks(c0, n1, n2)

    def read_channel(self, plane: PlaneTensor, c: int, tier, counter: AccessCounter) -> np.ndarray:
        c0, c1, c2 = plane.chunks()
        n = plane.n_tokens
        counter.add(tier, n if int(tier) else 0)
        return hb.merge_tier_array(c0[:, c], c1[:, c], c2[:, c], int(tier))

    def read_tiers(self, plane: PlaneTensor, codes: np.ndarray) -> np.ndarray:
        """Unmetered vector read: codes broadcast against [n, d]."""
        c0, c1, c2 = plane.chunks()
        return hb.merge_tier_array(c0, c1, c2, codes)
