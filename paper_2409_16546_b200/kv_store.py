"""kv_store host API over the GPU paged bit-plane store.

`KVStore` keeps every (batch, kv-head) unit's K and V caches on the GPU as
paged bit planes (layout in include/akv.h) plus the ColMax / RowMax
sidecars; appends run the fused `akv_append` kernel.  `PlaneTensor` is the
reference's row-major 3-plane view, produced on device
by `akv_export_planes`.  `AccessCounter` is the SPEC metering record
(SPEC.md:227-230,260-268), filled from the kernels' integer counters.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from paper_2409_16546_b200 import _lib
from paper_2409_16546_b200._lib import HEAD_DIM, PAGE_BYTES, PAGE_TOKENS


# ---------------------------------------------------------------------------
# metering
# ---------------------------------------------------------------------------
@dataclass
class AccessCounter:
    """bits_read = 8*T8 + 12*T12 + 16*T16; elements_read excludes SKIP."""

    t8: int = 0
    t12: int = 0
    t16: int = 0

    @property
    def bits_read(self) -> int:
        return 8 * self.t8 + 12 * self.t12 + 16 * self.t16

    @property
    def elements_read(self) -> int:
        return self.t8 + self.t12 + self.t16

    @property
    def tier_counts(self) -> dict:
        return {8: self.t8, 12: self.t12, 16: self.t16}

    def merge(self, other: "AccessCounter") -> "AccessCounter":
        return AccessCounter(self.t8 + other.t8, self.t12 + other.t12, self.t16 + other.t16)

    __add__ = merge

    def average_bit_width(self) -> float:
        return average_bit_width(self)


def average_bit_width(counter: AccessCounter) -> float:
    """SPEC.md:260-268."""
    if counter.elements_read == 0:
        raise ValueError("no reads recorded")
    return counter.bits_read / counter.elements_read


# ---------------------------------------------------------------------------
# SPEC row-major plane view
# ---------------------------------------------------------------------------
@dataclass
class PlaneTensor:
    """plane0 [n,d] u8 head bytes; plane1/plane2 [n,d/2] u8 nibbles, low nibble first."""

    n_dims: int
    plane0: np.ndarray
    plane1: np.ndarray
    plane2: np.ndarray

    @property
    def n_tokens(self) -> int:
        return int(self.plane0.shape[0])

    def chunks(self):
        def unpack(p):
            out = np.empty(p.shape[:-1] + (self.n_dims,), np.uint8)
            out[..., 0::2] = p & 0xF
            out[..., 1::2] = p >> 4
            return out

        return self.plane0, unpack(self.plane1), unpack(self.plane2)

    def words(self) -> np.ndarray:
        c0, c1, c2 = self.chunks()
        return ((c0.astype(np.uint16) << 8) | (c1.astype(np.uint16) << 4) | c2).astype(np.uint16)

    def nbytes(self) -> int:
        return self.plane0.nbytes + self.plane1.nbytes + self.plane2.nbytes


def _as_bits(x, device) -> torch.Tensor:
    """fp16 values or uint16/int16 bit patterns -> contiguous int16 bits on device."""
    if isinstance(x, np.ndarray):
        if x.dtype == np.float16:
            x = x.view(np.uint16)
        x = torch.from_numpy(np.ascontiguousarray(x.astype(np.uint16, copy=False)).view(np.int16))
    if not isinstance(x, torch.Tensor):
        raise TypeError("expected a torch tensor or numpy array")
    if x.dtype == torch.float16:
        x = x.view(torch.int16)
    elif x.dtype == torch.uint16:
        x = x.view(torch.int16)
    elif x.dtype != torch.int16:
        raise TypeError(f"expected fp16 values or 16-bit patterns, got {x.dtype}")
    return x.to(device, non_blocking=True).contiguous()


def decode_status(word: int):
    code = (word >> 60) & 0x7
    return code, (word >> 59) & 1, (word >> 40) & 0xFF, word & 0xFFFFFFFF


class KVStore:
    """GPU bit-plane KV cache for B x Hkv units.

    A unit (b, h) stores up to `capacity` tokens in pages of 256 tokens.
    `append_token` / `append` validate, split and store on device; with
    strict=True they synchronise and raise ValueError on non-finite input,
    reporting its position.  With strict=False call check().
    """

    def __init__(self, batch: int = 1, n_kv_heads: int = 1, head_dim: int = HEAD_DIM, capacity: int = 4096,
                 device=None, strict: bool = True):
        if head_dim != HEAD_DIM:
            raise NotImplementedError(f"head_dim {head_dim}: this build supports d = {HEAD_DIM}")
        if not torch.cuda.is_available():
            raise _lib.AkvError("KVStore needs a CUDA device (no CPU fallback)")
        self._L = _lib.lib()
        self.batch, self.n_kv_heads, self.n_dims = batch, n_kv_heads, head_dim
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.max_pages = max(1, -(-capacity // PAGE_TOKENS))
        self.capacity = self.max_pages * PAGE_TOKENS
        self.strict = strict
        U = self.n_units
        dev = self.device
        self.k_pool = torch.zeros((U * self.max_pages, PAGE_BYTES), dtype=torch.uint8, device=dev)
        self.v_pool = torch.zeros((U * self.max_pages, PAGE_BYTES), dtype=torch.uint8, device=dev)
        self.page_table = torch.arange(U * self.max_pages, dtype=torch.int32, device=dev).view(U, self.max_pages)
        self.lengths_dev = torch.zeros(U, dtype=torch.int32, device=dev)
        self.colmax_dev = torch.zeros((U, head_dim), dtype=torch.int32, device=dev)
        self.rowmax_dev = torch.zeros((U, self.capacity), dtype=torch.int16, device=dev)
        self.status_dev = torch.zeros(U, dtype=torch.int64, device=dev)
        self._host_len = np.zeros(U, np.int64)
        self._pending = None
        self._workspaces = {}
        self.c_store = _lib.AkvStore(U, head_dim, self.max_pages, 0, self.k_pool.data_ptr(), self.v_pool.data_ptr(),
                                     self.page_table.data_ptr(), self.lengths_dev.data_ptr(),
                                     self.colmax_dev.data_ptr(), self.rowmax_dev.data_ptr())

    # ---------------------------------------------------------------- shape
    @property
    def n_units(self) -> int:
        return self.batch * self.n_kv_heads

    @property
    def lengths(self) -> np.ndarray:
        return self._host_len.reshape(self.batch, self.n_kv_heads).copy()

    @property
    def n_tokens(self) -> int:
        return int(self._host_len.max()) if self._host_len.size else 0

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    # ---------------------------------------------------------------- append
    def _shape_rows(self, x, name):
        x = _as_bits(x, self.device)
        if x.dim() == 1 and self.n_units == 1:
            x = x.view(1, 1, 1, -1)
        elif x.dim() == 2 and self.n_units == 1:
            x = x.view(1, 1, x.shape[0], x.shape[1])
        elif x.dim() == 3:
            x = x.unsqueeze(2)
        if x.dim() != 4 or x.shape[0] != self.batch or x.shape[1] != self.n_kv_heads or x.shape[3] != self.n_dims:
            raise ValueError(f"{name}: expected [B={self.batch}, Hkv={self.n_kv_heads}, T, d={self.n_dims}] "
                             f"(row length mismatch), got {tuple(x.shape)}")
        return x.contiguous()

    def append_token(self, k_row, v_row) -> None:
        """One token per unit: k_row, v_row [B, Hkv, d] (or [d] for a single unit)."""
        self.append(k_row, v_row)

    def append(self, k, v) -> None:
        """Bulk append: k, v [B, Hkv, T, d]."""
        k = self._shape_rows(k, "k")
        v = self._shape_rows(v, "v")
        if k.shape != v.shape:
            raise ValueError("k and v shapes differ (length mismatch)")
        T = int(k.shape[2])
        if T == 0:
            return
        if int(self._host_len.max()) + T > self.capacity:
            raise ValueError(f"append of {T} tokens exceeds capacity {self.capacity}")
        self.status_dev.zero_()  # status words are sticky (akv.h): clear before an append whose outcome we read
        if T == 1:
            rc = self._L.akv_append(ctypes.byref(self.c_store), k.data_ptr(), v.data_ptr(), T,
                                    self.status_dev.data_ptr(), self._stream())
        else:  # prefill writer: page-span tiles, fused validation, per-unit commit
            ws = self._append_workspace(T)
            rc = self._L.akv_append_ws(ctypes.byref(self.c_store), k.data_ptr(), v.data_ptr(), T,
                                       self.status_dev.data_ptr(), ws.data_ptr(), ws.numel(), self._stream())
        _lib.check(rc, "akv_append")
        before = self._host_len.copy()
        self._host_len += T
        self._pending = (k, v, before, T)
        if self.strict:
            self.check()

    def _append_workspace(self, T: int):
        """Device workspace of the bulk append (a ColMax row + the earliest non-finite key per unit),
        grown on demand and reused; the kernels rewrite every byte they read."""
        need = int(self._L.akv_append_workspace_bytes(self.n_units, T))
        ws = getattr(self, "_append_ws", None)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._append_ws = ws
        return ws

    def check(self) -> None:
        """Synchronise on the last append's status; raise ValueError with the position."""
        if self._pending is None:
            return
        k, v, before, T = self._pending
        self._pending = None
        st = self.status_dev.cpu().numpy()
        bad = np.nonzero(st)[0]
        if bad.size == 0:
            return
        self._host_len[bad] = before[bad]
        # resync host mirror with the device truth for all units
        self._host_len[:] = self.lengths_dev.cpu().numpy()
        u = int(bad[0])
        code, isv, c, t = decode_status(int(st[u]))
        b, h = divmod(u, self.n_kv_heads)
        if code == _lib.STATUS_NONFINITE:
            src = v if isv else k
            w = int(src[b, h, t, c].item()) & 0xFFFF
            raise ValueError(f"non-finite half word 0x{w:04X} in {'V' if isv else 'K'} at batch {b}, "
                             f"kv-head {h}, token {int(before[u]) + t}, channel {c}")
        if code == _lib.STATUS_CAPACITY:
            raise ValueError(f"append beyond capacity at batch {b}, kv-head {h}")
        raise ValueError(f"append failed with status 0x{int(st[u]):016X}")

    def append_token_at(self, pos: int, k_row, v_row) -> None:
        """Truncate every unit to `pos` tokens and append one token there (akv_append_at: one
        launch; speculative rollback, fixed-context replay).  pos must not exceed any unit's
        length.  ColMax keeps its running max over every token ever appended."""
        k = self._shape_rows(k_row, "k")
        v = self._shape_rows(v_row, "v")
        if k.shape != v.shape or int(k.shape[2]) != 1:
            raise ValueError("append_token_at takes one k row and one v row per unit")
        if not 0 <= pos <= int(self._host_len.min()):
            raise ValueError(f"position {pos} outside [0, {int(self._host_len.min())}]")
        if pos + 1 > self.capacity:
            raise ValueError(f"append at {pos} exceeds capacity {self.capacity}")
        self.status_dev.zero_()
        _lib.check(self._L.akv_append_at(ctypes.byref(self.c_store), k.data_ptr(), v.data_ptr(), int(pos),
                                         self.status_dev.data_ptr(), self._stream()), "akv_append_at")
        before = np.full_like(self._host_len, pos)
        self._host_len[:] = pos + 1
        self._pending = (k, v, before, 1)
        if self.strict:
            self.check()

    def rewind(self, n_tokens: int) -> None:
        """Set every unit's length to n_tokens (<= current).  ColMax keeps its running max."""
        if n_tokens > int(self._host_len.min()):
            raise ValueError("rewind can only shorten")
        self.lengths_dev.fill_(n_tokens)
        self._host_len[:] = n_tokens

    def batch_prefix(self, batch: int) -> "KVStore":
        """A store over the first `batch` batch rows that shares every device buffer of this
        one (units are b-major, so the prefix is contiguous); used by the batch sweep."""
        if not 1 <= batch <= self.batch:
            raise ValueError(f"batch prefix {batch} outside [1, {self.batch}]")
        v = object.__new__(KVStore)
        v.__dict__.update(self.__dict__)
        U = batch * self.n_kv_heads
        v.batch = batch
        v._host_len = self._host_len[:U]
        for name in ("page_table", "lengths_dev", "colmax_dev", "rowmax_dev", "status_dev"):
            setattr(v, name, getattr(self, name)[:U])
        v._pending = None
        v._workspaces = {}
        v.c_store = _lib.AkvStore(U, self.n_dims, self.max_pages, 0, self.k_pool.data_ptr(), self.v_pool.data_ptr(),
                                  v.page_table.data_ptr(), v.lengths_dev.data_ptr(), v.colmax_dev.data_ptr(),
                                  v.rowmax_dev.data_ptr())
        return v

    # ---------------------------------------------------------------- sidecars / export
    def colmax(self) -> torch.Tensor:
        """[B, Hkv, d] fp16 magnitude patterns (as int32)."""
        return self.colmax_dev.view(self.batch, self.n_kv_heads, self.n_dims)

    def rowmax(self) -> torch.Tensor:
        """[B, Hkv, n] fp16 magnitude patterns (int16 storage)."""
        return self.rowmax_dev.view(self.batch, self.n_kv_heads, self.capacity)[:, :, : self.n_tokens]

    def export_planes(self, which: str = "k"):
        """SPEC row-major planes of every unit: (plane0 [B,Hkv,n,d], plane1, plane2 [B,Hkv,n,d/2]) on host."""
        w = {"k": 0, "v": 1}[which]
        U, cap, d = self.n_units, self.capacity, self.n_dims
        p0 = torch.zeros((U, cap, d), dtype=torch.uint8, device=self.device)
        p1 = torch.zeros((U, cap, d // 2), dtype=torch.uint8, device=self.device)
        p2 = torch.zeros((U, cap, d // 2), dtype=torch.uint8, device=self.device)
        rc = self._L.akv_export_planes(ctypes.byref(self.c_store), w, p0.data_ptr(), p1.data_ptr(), p2.data_ptr(),
                                       self._stream())
        _lib.check(rc, "akv_export_planes")
        n = self.n_tokens
        shp = (self.batch, self.n_kv_heads)
        return tuple(t[:, :n].cpu().numpy().reshape(shp + t[:, :n].shape[1:]) for t in (p0, p1, p2))

    def planes(self, b: int = 0, h: int = 0, which: str = "k") -> PlaneTensor:
        p0, p1, p2 = self.export_planes(which)
        n = int(self._host_len[b * self.n_kv_heads + h])
        return PlaneTensor(self.n_dims, p0[b, h, :n], p1[b, h, :n], p2[b, h, :n])

    def words(self, which: str = "k") -> np.ndarray:
        """Stored fp16 patterns [B, Hkv, n, d] reassembled from the exported planes."""
        p0, p1, p2 = self.export_planes(which)
        return PlaneTensor(self.n_dims, p0, p1, p2).words()

    # ---------------------------------------------------------------- metered reads
    def read_elements(self, units, toks, chans, tiers, which: str = "k", counter: AccessCounter = None) -> torch.Tensor:
        """Batched metered reads on the device (akv_read_elements): int32 tensors / sequences of
        equal length; returns the rebuilt words [n] (uint16 patterns as int16).  Only the planes
        each tier needs are read; the T8 / T12 / T16 element counts go into `counter`."""
        dev = self.device
        cols = [torch.as_tensor(x, dtype=torch.int32).reshape(-1).to(dev) for x in (units, toks, chans, tiers)]
        n = int(cols[0].numel())
        if any(int(x.numel()) != n for x in cols):
            raise ValueError("read_elements: argument lengths differ")
        out = torch.empty(n, dtype=torch.int16, device=dev)
        cnt = torch.zeros(3, dtype=torch.int64, device=dev)
        rc = self._L.akv_read_elements(ctypes.byref(self.c_store), {"k": 0, "v": 1}[which], cols[0].data_ptr(),
                                       cols[1].data_ptr(), cols[2].data_ptr(), cols[3].data_ptr(), n, out.data_ptr(),
                                       cnt.data_ptr(), self._stream())
        _lib.check(rc, "akv_read_elements")
        if counter is not None:
            c8, c12, c16 = (int(x) for x in cnt.cpu())
            counter.t8 += c8
            counter.t12 += c12
            counter.t16 += c16
        return out

    @staticmethod
    def _tier_code(tier) -> int:
        code = int(tier)
        if code not in (0, 8, 12, 16):
            raise ValueError(f"bad tier {tier}")
        return code

    def read_element(self, b: int, h: int, t: int, c: int, tier, counter: AccessCounter, which: str = "k") -> int:
        """KVStore.read_element: one metered read on the device; SKIP -> 0, 0 bits."""
        n = int(self._host_len[b * self.n_kv_heads + h])
        if not (0 <= t < n and 0 <= c < self.n_dims):
            raise IndexError("read out of range")
        code = self._tier_code(tier)
        if code == 0:
            return 0
        w = self.read_elements([b * self.n_kv_heads + h], [t], [c], [code], which, counter)
        return int(w.item()) & 0xFFFF

    def read_channel(self, b: int, h: int, c: int, tier, counter: AccessCounter, which: str = "k") -> np.ndarray:
        """KVStore.read_channel: tokens 0..n-1 of channel c at one tier."""
        if not 0 <= c < self.n_dims:
            raise IndexError("read out of range")
        n = int(self._host_len[b * self.n_kv_heads + h])
        code = self._tier_code(tier)
        if code == 0:
            return np.zeros(n, np.uint16)
        u = b * self.n_kv_heads + h
        w = self.read_elements(torch.full((n,), u, dtype=torch.int32), torch.arange(n, dtype=torch.int32),
                               torch.full((n,), c, dtype=torch.int32), torch.full((n,), code, dtype=torch.int32),
                               which, counter)
        return w.cpu().numpy().view(np.uint16)

    # ---------------------------------------------------------------- decode workspaces
    def workspace(self, group: int, separate_probs: bool = False):
        from paper_2409_16546_b200.attention_decode import DecodeWorkspace

        key = (group, separate_probs)
        ws = self._workspaces.get(key)
        if ws is None:
            ws = DecodeWorkspace(self, group, separate_probs)
            self._workspaces[key] = ws
        return ws
