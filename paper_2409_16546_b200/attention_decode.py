"""attention_decode host API over the libakv kernels.

`decode_step` runs the whole aligned decode step for every (batch, q-head)
in four launches on the current stream (akv_decode_step: qk -> softmax +
estimate -> pv -> combine).  The SPEC's single-operation entry points
(`scores_aligned`, `softmax`, `estimate_output`, `output_aligned`,
`reference_scores`, `reference_output`, `baseline_truncated`) run the same
kernels one stage at a time and pass device state between them.

Shapes: q [B, Hq, d] fp16 with Hq = g * Hkv (GQA: q head i reads kv head
i // g); a single head may pass q [d] against a 1-unit store.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from paper_2409_16546_b200 import _lib
from paper_2409_16546_b200._lib import HEAD_DIM, MAX_KSEL, PAGE_TOKENS, TARGET_UNKNOWN
from paper_2409_16546_b200.align_core import AlignConfig, DegenerateInputError, Tier
from paper_2409_16546_b200.kv_store import AccessCounter, KVStore, _as_bits, decode_status

ELEMENT, ROW = "element", "row"


class DecodeWorkspace:
    """Device buffers of one decode step for a store and a GQA group size."""

    def __init__(self, store: KVStore, group: int, separate_probs: bool = False):
        if group not in (1, 2, 4, 8):
            raise ValueError("q heads per kv head must be 1, 2, 4 or 8")
        self.store, self.group = store, group
        L = _lib.lib()
        U, mp, d, dev = store.n_units, store.max_pages, store.n_dims, store.device
        H = U * group
        nbytes = int(L.akv_workspace_bytes(U, group, mp))
        self.ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device=dev)  # zeroed once (akv.h)
        base = (self.ws.data_ptr() + 255) & ~255
        self.step = _lib.AkvStep()
        _lib.check(L.akv_step_carve(ctypes.byref(self.step), base, U, group, mp), "akv_step_carve")
        self._base = base
        cap = store.capacity
        self.o = torch.zeros((H, d), dtype=torch.float32, device=dev)
        self.step.o = self.o.data_ptr()
        self.probs = None
        if separate_probs:
            self.probs = torch.zeros((H, cap), dtype=torch.float32, device=dev)
            self.step.probs = self.probs.data_ptr()
        self.v_tiers = None
        self.H, self.cap = H, cap

    # typed views over the carved workspace
    def _view(self, ptr_field: str, shape, dtype):
        ptr = getattr(self.step, ptr_field)
        off = ptr - self.ws.data_ptr()
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        return self.ws[off: off + n].view(dtype).view(shape)

    def scores(self):
        return self._view("scores", (self.H, self.cap), torch.float32)

    def probs_view(self):
        return self.probs if self.probs is not None else self.scores()

    def counters(self):
        return self._view("counters", (self.H, 8), torch.int64)

    def unit_bytes(self):
        return self._view("unit_bytes", (self.store.n_units, 4), torch.int64)

    def status(self):
        return self._view("status", (self.H,), torch.int64)

    def k_tiers(self):
        return self._view("k_tiers", (self.H, self.store.n_dims), torch.uint8)

    def o_est(self):
        return self._view("o_est", (self.H, self.store.n_dims), torch.float32)

    def targets(self):
        return self._view("targets", (self.H, self.store.n_dims), torch.int32)

    def sel_idx(self):
        return self._view("sel_idx", (self.H, MAX_KSEL), torch.int32)

    def head_meta(self):
        return self._view("head_meta", (self.H, 4), torch.int32)

    def head_metaf(self):
        return self._view("head_metaf", (self.H, 4), torch.float32)

    def sel_bits(self):
        return self._view("sel_bits", (self.H, self.cap // 32), torch.int32)

    def set_v_tiers(self, enable: bool):
        if enable:
            if self.v_tiers is None:
                self.v_tiers = torch.zeros((self.H, self.cap, self.store.n_dims), dtype=torch.uint8,
                                           device=self.store.device)
            self.step.v_tiers = self.v_tiers.data_ptr()
        else:
            self.step.v_tiers = None


def make_cfg(group: int, cfg: AlignConfig = AlignConfig(), k_sel: int = 32, m: int = 5, strategy: str = ELEMENT,
             force_tier=None, trunc_bits=None) -> _lib.AkvCfg:
    if strategy not in (ELEMENT, ROW):
        raise ValueError(f"unknown strategy {strategy!r}")
    ft = 0 if force_tier is None else int(force_tier)
    if ft not in (0, 8, 12, 16):
        raise ValueError("force_tier must be None, 8, 12 or 16")
    tb = 0 if trunc_bits is None else int(trunc_bits)
    if tb and not 8 <= tb <= 16:
        raise ValueError("bits must be in [8, 16]")
    if not 0 <= k_sel <= MAX_KSEL:
        raise ValueError(f"k_sel must be in [0, {MAX_KSEL}]")
    return _lib.AkvCfg(group, cfg.margin_bits, int(cfg.zero_skip), ft, k_sel, m, 0 if strategy == ELEMENT else 1, tb)


def _q_bits(q, store: KVStore) -> tuple[torch.Tensor, int]:
    qb = _as_bits(q, store.device)
    if qb.dim() == 1:
        qb = qb.view(1, 1, -1)
    if qb.dim() != 3 or qb.shape[0] != store.batch or qb.shape[2] != store.n_dims:
        raise ValueError(f"q must be [B={store.batch}, Hq, d={store.n_dims}], got {tuple(qb.shape)}")
    hq = int(qb.shape[1])
    if hq % store.n_kv_heads:
        raise ValueError("Hq must be a multiple of Hkv")
    return qb.contiguous(), hq // store.n_kv_heads


def _raise_status(ws: DecodeWorkspace, store: KVStore):
    st = ws.status().cpu().numpy()
    bad = np.nonzero(st)[0]
    if bad.size == 0:
        return
    h = int(bad[0])
    code = decode_status(int(st[h]))[0]
    b, rem = divmod(h, store.n_kv_heads * ws.group)
    if code == _lib.STATUS_DEGENERATE:
        raise DegenerateInputError(f"degenerate dot product (batch {b}, q-head {rem})")
    if code == _lib.STATUS_BAD_Q:
        raise ValueError(f"non-finite q (batch {b}, q-head {rem})")
    raise ValueError(f"decode failed with status 0x{int(st[h]):016X}")


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------
@dataclass
class AttentionResult:
    """output, scores, K/V stats, K tiers, V tiers."""

    o: torch.Tensor                      # [B, Hq, d] fp32
    k_tiers: torch.Tensor                # [B, Hq, d] uint8 read-bit codes (0 = SKIP)
    counters: torch.Tensor               # [B, Hq, 8] int64 (k8,k12,k16,v8,v12,v16,-,-)
    unit_bytes: torch.Tensor             # [B, Hkv, 4] int64 physical plane bytes (K, V)
    scores: Optional[torch.Tensor] = None
    probs: Optional[torch.Tensor] = None
    o_est: Optional[torch.Tensor] = None
    targets: Optional[torch.Tensor] = None
    sel_count: Optional[torch.Tensor] = None
    sel_idx: Optional[torch.Tensor] = None
    v_tiers: Optional[torch.Tensor] = None
    _host: dict = field(default_factory=dict, repr=False)

    def _c(self):
        if "c" not in self._host:
            self._host["c"] = self.counters.cpu().numpy()
        return self._host["c"]

    def k_stats(self, b: Optional[int] = None, h: Optional[int] = None) -> AccessCounter:
        c = self._c()
        sel = c if b is None else (c[b] if h is None else c[b, h][None])
        s = sel.reshape(-1, 8).sum(0)
        return AccessCounter(int(s[0]), int(s[1]), int(s[2]))

    def v_stats(self, b: Optional[int] = None, h: Optional[int] = None) -> AccessCounter:
        c = self._c()
        sel = c if b is None else (c[b] if h is None else c[b, h][None])
        s = sel.reshape(-1, 8).sum(0)
        return AccessCounter(int(s[3]), int(s[4]), int(s[5]))

    def stats(self) -> AccessCounter:
        return self.k_stats().merge(self.v_stats())

    def selection(self, b: int, h: int) -> np.ndarray:
        n = int(self.sel_count[b, h])
        return self.sel_idx[b, h, :n].cpu().numpy()


def _launch(fn_name, store, cfg_c, ws, max_len=None):
    L = _lib.lib()
    ml = store.n_tokens if max_len is None else max_len
    rc = getattr(L, fn_name)(ctypes.byref(store.c_store), ctypes.byref(cfg_c), ctypes.byref(ws.step), ml,
                             store._stream())
    _lib.check(rc, fn_name)


def decode_launch(q_bits: torch.Tensor, store: KVStore, cfg_c: _lib.AkvCfg, ws: DecodeWorkspace,
                  max_len: Optional[int] = None) -> None:
    """Raw launch of the 4-kernel chain (no sync, no copies): the bench's hot call."""
    ws.step.q = q_bits.data_ptr()
    _launch("akv_decode_step", store, cfg_c, ws, max_len)


def decode_step(q, store: KVStore, cfg: AlignConfig = AlignConfig(), *, k_sel: int = 32, m: int = 5,
                strategy: str = ELEMENT, force_tier=None, trunc_bits=None, return_scores: bool = False,
                export_v_tiers: bool = False, check: bool = True) -> AttentionResult:
    """One aligned decode step for every (batch, q-head): SURVEY §3(2)."""
    store.check()
    qb, g = _q_bits(q, store)
    ws = store.workspace(g, separate_probs=return_scores)
    ws.set_v_tiers(export_v_tiers)
    cfg_c = make_cfg(g, cfg, k_sel, m, strategy, force_tier, trunc_bits)
    decode_launch(qb, store, cfg_c, ws)
    if check:
        _raise_status(ws, store)
    return _result(ws, store, g, return_scores, export_v_tiers)


def _result(ws: DecodeWorkspace, store: KVStore, g: int, with_scores: bool, with_vt: bool) -> AttentionResult:
    B, hq, d, n = store.batch, store.n_kv_heads * g, store.n_dims, store.n_tokens
    sh = (B, hq)
    meta = ws.head_meta().clone()
    r = AttentionResult(
        o=ws.o.clone().view(*sh, d),
        k_tiers=ws.k_tiers().clone().view(*sh, d),
        counters=ws.counters().clone().view(*sh, 8),
        unit_bytes=ws.unit_bytes().clone().view(B, store.n_kv_heads, 4),
        o_est=ws.o_est().clone().view(*sh, d),
        targets=ws.targets().clone().view(*sh, d),
        sel_count=meta[:, 0].view(*sh).cpu(),
        sel_idx=ws.sel_idx().clone().view(*sh, MAX_KSEL),
    )
    if with_scores:
        r.scores = ws.scores()[:, :n].clone().view(*sh, n)
        r.probs = ws.probs_view()[:, :n].clone().view(*sh, n)
    elif ws.probs is None:
        r.probs = ws.scores()[:, :n].clone().view(*sh, n)  # probs overwrote scores in place
    if with_vt and ws.v_tiers is not None:
        r.v_tiers = ws.v_tiers[:, :n].clone().view(*sh, n, d)
    return r


# ---------------------------------------------------------------------------
# SPEC single-operation API (stateful hand-off between stages)
# ---------------------------------------------------------------------------
@dataclass
class ScoreVector:
    """Raw scores s plus the device state the next stages need."""

    s: torch.Tensor
    k_tiers: torch.Tensor
    k_stats: AccessCounter
    _ws: DecodeWorkspace = field(repr=False)
    _store: KVStore = field(repr=False)
    _cfg: AlignConfig = field(repr=False)


@dataclass
class Probabilities:
    p: torch.Tensor
    _ws: DecodeWorkspace = field(repr=False)
    _store: KVStore = field(repr=False)
    _cfg: AlignConfig = field(repr=False)


@dataclass
class OutputEstimate:
    """o_est from <= k_sel selected rows."""

    o_est: torch.Tensor
    sel_count: torch.Tensor
    sel_idx: torch.Tensor
    v_stats: AccessCounter
    _ws: DecodeWorkspace = field(repr=False)
    _k_sel: int = 32
    _m: int = 5

    def selection(self, b: int, h: int) -> np.ndarray:
        return self.sel_idx[b, h, : int(self.sel_count[b, h])].cpu().numpy()


def scores_aligned(q, store: KVStore, cfg: AlignConfig = AlignConfig(), force_tier=None,
                   _trunc_bits=None) -> ScoreVector:
    """SPEC.md:315-323."""
    store.check()
    qb, g = _q_bits(q, store)
    ws = store.workspace(g, separate_probs=True)
    ws.step.q = qb.data_ptr()
    ws._q = qb
    c = make_cfg(g, cfg, 32, 5, ELEMENT, force_tier, _trunc_bits)
    _launch("akv_qk", store, c, ws)
    _raise_status(ws, store)
    B, hq, n = store.batch, store.n_kv_heads * g, store.n_tokens
    cnt = ws.counters().cpu().numpy().sum(0)
    return ScoreVector(ws.scores()[:, :n].clone().view(B, hq, n), ws.k_tiers().clone().view(B, hq, -1),
                       AccessCounter(int(cnt[0]), int(cnt[1]), int(cnt[2])), ws, store, cfg)


def reference_scores(q, store: KVStore) -> torch.Tensor:
    """all-T16 scores (R_normal)."""
    return scores_aligned(q, store, force_tier=16).s


def softmax(sv: ScoreVector) -> Probabilities:
    """SPEC.md:324-332 on the device scores of `sv` (max-subtracted, fp32)."""
    ws, store = sv._ws, sv._store
    c = make_cfg(ws.group, sv._cfg, 0, 5)
    _launch("akv_softmax_select", store, c, ws)
    B, hq, n = sv.s.shape
    return Probabilities(ws.probs[:, :n].clone().view(B, hq, n), ws, store, sv._cfg)


def estimate_output(p: Probabilities, store: KVStore, k_sel: int = 32, m: int = 5) -> OutputEstimate:
    """SPEC.md:333-341 (threshold p >= pmax*2^-m, cap k_sel; D3 ties)."""
    ws = p._ws
    if k_sel < 1:
        raise ValueError("k_sel must be >= 1")
    c = make_cfg(ws.group, p._cfg, k_sel, m)
    _launch("akv_softmax_select", store, c, ws)
    B, hq = p.p.shape[:2]
    meta = ws.head_meta().cpu()
    cnt = ws.counters().cpu().numpy().sum(0)
    return OutputEstimate(ws.o_est().clone().view(B, hq, -1), meta[:, 0].view(B, hq),
                          ws.sel_idx().clone().view(B, hq, MAX_KSEL), AccessCounter(0, 0, int(cnt[5])), ws, k_sel, m)


def output_aligned(p: Probabilities, store: KVStore, o_est: Optional[OutputEstimate] = None,
                   cfg: AlignConfig = AlignConfig(), strategy: str = ELEMENT, export_v_tiers: bool = False):
    """SPEC.md:342-350 -> (o [B,Hq,d], V-side AccessCounter of the PV reads, v_tiers or None)."""
    if o_est is None:
        raise ValueError("missing o_est")
    ws = p._ws
    ws.set_v_tiers(export_v_tiers)
    c = make_cfg(ws.group, cfg, o_est._k_sel, o_est._m, strategy)
    # the PV fetch plan (need bits) depends on the strategy: re-run the (deterministic) select stage
    _launch("akv_softmax_select", store, c, ws)
    ctr = ws.counters()
    before = ctr[:, 3:6].clone()
    _launch("akv_pv", store, c, ws)
    _launch("akv_combine", store, c, ws)
    B, hq = p.p.shape[:2]
    d = (ctr[:, 3:6] - before).cpu().numpy().sum(0)
    vt = ws.v_tiers[:, : store.n_tokens].clone().view(B, hq, store.n_tokens, -1) if export_v_tiers else None
    return ws.o.clone().view(B, hq, -1), AccessCounter(int(d[0]), int(d[1]), int(d[2])), vt


def _forced_output(p, store: KVStore, tier: int, trunc_bits=None) -> torch.Tensor:
    pt = p.p if isinstance(p, Probabilities) else p
    g = pt.shape[1] // store.n_kv_heads
    ws = store.workspace(g, separate_probs=True)
    n = store.n_tokens
    ws.probs[:, :n].copy_(pt.reshape(-1, n).to(ws.probs.device, torch.float32))
    ws.o_est().zero_()
    c = make_cfg(g, AlignConfig(), 32, 5, ELEMENT, tier if trunc_bits is None else None, trunc_bits)
    _launch("akv_pv", store, c, ws)
    _launch("akv_combine", store, c, ws)
    return ws.o.clone().view(pt.shape[0], pt.shape[1], -1)


def reference_output(p, store: KVStore) -> torch.Tensor:
    """o = sum_t p_t V[t] at full 16 bits."""
    return _forced_output(p, store, 16)


def baseline_truncated(q, store: KVStore, p, bits: int = 13):
    """every K and V element truncate_fill'ed to bits-6 kept bits."""
    if not 8 <= bits <= 16:
        raise ValueError("bits must be in [8, 16]")
    s = scores_aligned(q, store, _trunc_bits=bits).s
    o = _forced_output(p, store, 16, trunc_bits=bits)
    return s, o


def decode(q, store: KVStore, cfg: AlignConfig = AlignConfig(), *, k_sel: int = 32, m: int = 5,
           strategy: str = ELEMENT, force_tier=None) -> torch.Tensor:
    """Serving entry point: one aligned decode step, returns o [B, Hq, d] fp32.

    No host synchronisation: the per-head status words stay on device; call
    `check_status(store, group)` (or decode_step) to raise on degenerate q.
    The returned tensor is the workspace's output buffer (overwritten by the
    next call with the same store and group).
    """
    qb, g = _q_bits(q, store)
    ws = store.workspace(g)
    ws.set_v_tiers(False)
    key = (cfg.margin_bits, cfg.zero_skip, k_sel, m, strategy, force_tier)
    cfg_c = ws.__dict__.setdefault("_cfg_cache", {}).get(key)
    if cfg_c is None:
        cfg_c = make_cfg(g, cfg, k_sel, m, strategy, force_tier)
        ws._cfg_cache[key] = cfg_c
    decode_launch(qb, store, cfg_c, ws)
    return ws.o.view(store.batch, store.n_kv_heads * g, store.n_dims)


def check_status(store: KVStore, group: int) -> None:
    _raise_status(store.workspace(group), store)


class DecodeGraph:
    """One serving decode step captured as a CUDA graph: H2D of the step's
    q / k_new / v_new from pinned host buffers, append the new token's K/V,
    aligned attention (qk, select, pv, combine), D2H of o into a pinned host
    buffer.

        g = DecodeGraph(store, group=1).capture()
        g.host_q.copy_(q); g.host_k.copy_(k_new); g.host_v.copy_(v_new)   # or g.step(q, k_new, v_new)
        o = g.step()                                                        # replay + synchronise

    Each replay appends one token per unit (the host length mirror advances)
    and returns o [B, Hq, d] fp32 on the host.  Data-dependent errors stay on
    device: call `check()` to raise them (non-finite K/V, degenerate q).
    `rewind_to` (benchmarks, speculative rollback) appends every replay's token
    at position rewind_to (akv_append_at: truncate + append in one launch), so
    every replay attends over the same rewind_to + 1 tokens.  The
    grid is sized for the store's capacity (fixed at capture).
    """

    def __init__(self, store: KVStore, group: int = 1, cfg: AlignConfig = AlignConfig(), *, k_sel: int = 32,
                 m: int = 5, strategy: str = ELEMENT, force_tier=None, rewind_to: Optional[int] = None,
                 zero_copy_out: bool = True, zero_copy_in: bool = True):
        self.store, self.group = store, group
        self.rewind_to = rewind_to
        B, H, d, dev = store.batch, store.n_kv_heads, store.n_dims, store.device
        nq, nk = B * H * group * d, B * H * d
        # one packed input transfer: q | k_new | v_new
        self.host_in = torch.zeros(nq + 2 * nk, dtype=torch.int16).pin_memory()
        self.dev_in = torch.zeros(nq + 2 * nk, dtype=torch.int16, device=dev)
        self.host_q = self.host_in[:nq].view(B, H * group, d)
        self.host_k = self.host_in[nq:nq + nk].view(B, H, d)
        self.host_v = self.host_in[nq + nk:].view(B, H, d)
        self.q = self.dev_in[:nq].view(B, H * group, d)
        self.k = self.dev_in[nq:nq + nk].view(B, H, d)
        self.v = self.dev_in[nq + nk:].view(B, H, d)
        self.host_o = torch.zeros((B, H * group, d), dtype=torch.float32).pin_memory()
        self.ws = store.workspace(group)
        self.ws.set_v_tiers(False)
        self.cfg_c = make_cfg(group, cfg, k_sel, m, strategy, force_tier)
        self.o = self.ws.o.view(B, H * group, d)
        # zero-copy I/O (UVA-mapped pinned buffers): append and qk read k_new / v_new / q straight
        # from host memory and the combine kernel stores o straight into it, so the step has no
        # separate copy nodes (zero_copy_in / zero_copy_out = False: one packed H2D, one D2H)
        self.zero_copy_out = zero_copy_out
        self.step_c = _lib.AkvStep()
        ctypes.pointer(self.step_c)[0] = self.ws.step
        self.zero_copy_in = zero_copy_in
        self.step_c.q = (self.host_q if zero_copy_in else self.q).data_ptr()
        self.step_c.v_tiers = None
        if zero_copy_out:
            self.step_c.o = self.host_o.data_ptr()
        self.graph = None
        self._L = _lib.lib()

    @property
    def h2d_bytes(self) -> int:
        return 2 * self.host_in.numel()

    @property
    def d2h_bytes(self) -> int:
        return 4 * self.host_o.numel()

    def _enqueue(self, stream_ptr: int):
        st = self.store
        if not self.zero_copy_in:
            self.dev_in.copy_(self.host_in, non_blocking=True)
        kk, vv = (self.host_k, self.host_v) if self.zero_copy_in else (self.k, self.v)
        if self.rewind_to is not None:  # truncate to rewind_to tokens and append, one launch
            _lib.check(self._L.akv_append_at(ctypes.byref(st.c_store), kk.data_ptr(), vv.data_ptr(), self.rewind_to,
                                             st.status_dev.data_ptr(), stream_ptr), "akv_append_at")
        else:
            _lib.check(self._L.akv_append(ctypes.byref(st.c_store), kk.data_ptr(), vv.data_ptr(), 1,
                                          st.status_dev.data_ptr(), stream_ptr), "akv_append")
        _lib.check(self._L.akv_decode_step(ctypes.byref(st.c_store), ctypes.byref(self.cfg_c),
                                           ctypes.byref(self.step_c), st.capacity, stream_ptr), "akv_decode_step")
        if not self.zero_copy_out:
            self.host_o.copy_(self.o, non_blocking=True)

    def capture(self):
        st = self.store
        n0 = int(st._host_len.max()) if self.rewind_to is None else self.rewind_to
        if n0 + 1 > st.capacity:
            raise ValueError("store is full")
        st.check()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=st.device)
        s.wait_stream(torch.cuda.current_stream(st.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self._enqueue(s.cuda_stream)
        torch.cuda.current_stream(st.device).wait_stream(s)
        self.graph = g
        return self

    def _advance(self):
        st = self.store
        if self.rewind_to is not None:
            st._host_len[:] = self.rewind_to + 1
        else:
            st._host_len += 1

    def step(self, q=None, k_new=None, v_new=None) -> torch.Tensor:
        """Optionally copy q / k_new / v_new into the pinned host buffers, replay, return host o.

        Refuses to replay when the append would exceed the store's capacity (the device would
        reject it and the output would silently be stale)."""
        if self.graph is None:
            self.capture()
        if self.rewind_to is None and int(self.store._host_len.max()) + 1 > self.store.capacity:
            raise ValueError(f"store is full ({self.store.capacity} tokens): cannot append another token")
        for src, dst in ((q, self.host_q), (k_new, self.host_k), (v_new, self.host_v)):
            if src is not None:
                dst.copy_(_as_bits(src, torch.device("cpu")).view(dst.shape))
        self.graph.replay()
        self._advance()
        torch.cuda.current_stream(self.store.device).synchronize()
        return self.host_o

    def check(self):
        """Raise the device-side status of the replays since the last check (non-finite K/V,
        capacity, degenerate q).  Append errors are sticky on device, so a rejection in any
        replay is reported; the host length mirror is resynchronised from the device and the
        status words are cleared so the graph can keep serving."""
        st = self.store
        s = st.status_dev.cpu().numpy()
        bad = np.nonzero(s)[0]
        if bad.size:
            st._host_len[:] = st.lengths_dev.cpu().numpy()
            st.status_dev.zero_()
            code, isv, c, t = decode_status(int(s[bad[0]]))
            b, h = divmod(int(bad[0]), st.n_kv_heads)
            what = {_lib.STATUS_NONFINITE: f"non-finite {'V' if isv else 'K'} channel {c}",
                    _lib.STATUS_CAPACITY: "capacity exceeded",
                    _lib.STATUS_POSITION: "rewind position beyond the stored length"}.get(code, f"status code {code}")
            raise ValueError(f"append failed ({what}) at batch {b}, kv-head {h}")
        _raise_status(self.ws, st)
