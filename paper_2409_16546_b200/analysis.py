"""analysis over the GPU path.

* `relative_error_histogram(test, ref)` — Table-1 buckets,
  counted on device by `akv_error_histogram`; `fp16_round=True` applies the
  output grid first (SURVEY App. A A-hist, HB:187-190).
* `bitwidth_sweep(lengths, ...)` — Fig. 9 curve: for each
  context length, one aligned decode step over synthetic units on the GPU;
  average bit widths from the kernels' AccessCounter totals.
* `alignment_bruteforce(exps, u)` — SPEC.md:428-436, host integer search
  (≤ 4 products, 11^4 points).
* `compare_report(...)` — SPEC.md:437-445: AlignedKV and the n-bit truncation
  baseline against the full-fp16 reference, QK^T and SV, on identical inputs.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from paper_2409_16546_b200 import _lib
from paper_2409_16546_b200.align_core import AlignConfig, required_mantissa_bits

BUCKETS = ("{0}", "(0,1/1024)", "[1/1024,1/512)", "[1/512,1/256)", "[1/256,1/128)", "[1/128,inf)")
# PAPER.md:213-216 (Table 1), printed beside measured values
PAPER_TABLE1 = {
    ("aligned", "qk"): (56.30, 37.00, 5.42, 0.73, 0.31, 0.25),
    ("trunc13", "qk"): (18.65, 32.70, 36.21, 10.26, 1.36, 0.83),
    ("aligned", "sv"): (76.12, 18.14, 3.61, 1.29, 0.39, 0.44),
    ("trunc13", "sv"): (20.04, 29.47, 26.66, 13.82, 5.71, 4.30),
}


@dataclass
class ErrorHistogram:
    """six bucket counts, total, fractions."""

    counts: np.ndarray

    @property
    def total(self) -> int:
        return int(self.counts.sum())

    @property
    def fractions(self) -> np.ndarray:
        return self.counts / max(self.total, 1)

    def __add__(self, other: "ErrorHistogram") -> "ErrorHistogram":
        return ErrorHistogram(self.counts + other.counts)


def _dev_f32(x, device) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
    return x.to(device=device, dtype=torch.float32).contiguous().view(-1)


def relative_error_histogram(test, ref, fp16_round: bool = False, device=None) -> ErrorHistogram:
    """SPEC.md:410-418 on device; equal lengths required."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t, r = _dev_f32(test, dev), _dev_f32(ref, dev)
    if t.numel() != r.numel():
        raise ValueError("length mismatch")
    counts = torch.zeros(6, dtype=torch.int64, device=dev)
    rc = _lib.lib().akv_error_histogram(t.data_ptr(), r.data_ptr(), t.numel(), int(fp16_round), counts.data_ptr(),
                                        torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc, "akv_error_histogram")
    return ErrorHistogram(counts.cpu().numpy())


def alignment_bruteforce(product_exps: Sequence[int], target_u: int, cfg: AlignConfig = AlignConfig()):
    """SPEC.md:428-436 -> (min_total_bits or None if infeasible at half precision, aligned_total)."""
    exps = list(product_exps)
    if len(exps) > 4:
        raise ValueError("at most 4 products")
    aligned = sum(required_mantissa_bits(e, target_u, cfg) for e in exps)
    best = None
    for ts in itertools.product(range(11), repeat=len(exps)):
        if all(e - 1 - t <= target_u for e, t in zip(exps, ts)):
            tot = sum(ts)
            best = tot if best is None else min(best, tot)
    return best, aligned


@dataclass
class BitWidthPoint:
    context_length: int
    avg_bits: float
    avg_bits_k: float
    avg_bits_v: float
    bytes_fraction: float  # physical plane bytes read / full-fp16 K+V bytes
    sv_hist: Optional[ErrorHistogram] = None  # aligned o vs full-fp16 o (fp16 grid), when requested


@dataclass
class BitWidthCurve:
    """SPEC.md:404-407."""

    points: List[BitWidthPoint] = field(default_factory=list)

    def rows(self):
        return [(p.context_length, p.avg_bits, p.avg_bits_k, p.avg_bits_v) for p in self.points]


def _avg(c8, c12, c16):
    n = c8 + c12 + c16
    if n == 0:
        raise ValueError("no reads recorded")
    return (8 * c8 + 12 * c12 + 16 * c16) / n


def _build(n, batch, n_kv, g, seed, scale, device, data=None):
    from paper_2409_16546_b200.kv_store import KVStore
    from paper_2409_16546_b200.synth import generate_batch

    if data is None:
        K, V, Q = generate_batch(batch, n_kv, n, 128, g, seed, -scale, scale)
    else:  # (K [U, N, d], V [U, N, d], Q [U, g, d]) fp16 words, e.g. loaded AKV files; first n tokens
        K, V, Q = (np.ascontiguousarray(x) for x in (data[0][:, :n], data[1][:, :n], data[2]))
    st = KVStore(batch, n_kv, 128, n, device=device)
    st.append(torch.from_numpy(K.view(np.int16)).view(batch, n_kv, n, 128),
              torch.from_numpy(V.view(np.int16)).view(batch, n_kv, n, 128))
    q = torch.from_numpy(Q.view(np.int16)).view(batch, n_kv * g, 128)
    return st, q


def bitwidth_sweep(lengths: Sequence[int], seed: int = 7, batch: int = 1, n_kv: int = 1, group: int = 1,
                   cfg: AlignConfig = AlignConfig(), k_sel: int = 32, m: int = 5, strategy: str = "element",
                   force_tier: Optional[int] = None, scale: float = 4.0, device=None, with_hist: bool = False,
                   data=None) -> BitWidthCurve:
    """SPEC.md:419-427 on the GPU path; deterministic for a given seed and config.

    `data`: optional (K, V, Q) word arrays [U, N, d] / [U, g, d] used instead
    of the generator (lengths are prefixes).  `with_hist`: also the output
    (SV) error histogram vs the full-fp16 reference per length."""
    from paper_2409_16546_b200.attention_decode import decode_step, reference_output

    ls = list(lengths)
    if any(b <= a for a, b in zip(ls, ls[1:])):
        raise ValueError("lengths must be increasing")
    curve = BitWidthCurve()
    for n in ls:
        st, q = _build(n, batch, n_kv, group, seed, scale, device, data)
        r = decode_step(q, st, cfg, k_sel=k_sel, m=m, strategy=strategy, force_tier=force_tier,
                        return_scores=with_hist)
        hist = None
        if with_hist:
            o = r.o.clone()
            hist = relative_error_histogram(o, reference_output(r.probs, st), fp16_round=True)
        c = r.counters.view(-1, 8).sum(0).cpu().numpy().astype(np.int64)
        ub = r.unit_bytes.view(-1, 4).sum(0).cpu().numpy().astype(np.int64)
        curve.points.append(BitWidthPoint(n, _avg(c[0] + c[3], c[1] + c[4], c[2] + c[5]), _avg(*c[0:3]),
                                          _avg(*c[3:6]), float(ub[0] + ub[1]) / (4.0 * n * 128 * batch * n_kv), hist))
    return curve


@dataclass
class CompareReport:
    """histograms for {aligned, truncated-N} x {QK, SV} vs the reference + bit widths."""

    hist: dict
    avg_bits: dict
    baseline_bits: int

    def table(self) -> str:
        lines = [f"{'path':<10}{'op':<4}" + "".join(f"{b:>16}" for b in BUCKETS)]
        for (path, op), h in self.hist.items():
            lines.append(f"{path:<10}{op:<4}" + "".join(f"{100 * x:>15.2f}%" for x in h.fractions))
            pk = PAPER_TABLE1.get((path if path == "aligned" else f"trunc{self.baseline_bits}", op))
            if pk is not None:
                lines.append(f"{'  paper':<14}" + "".join(f"{x:>15.2f}%" for x in pk))
        lines.append("avg bits: " + ", ".join(f"{k}={v:.3f}" for k, v in self.avg_bits.items()))
        return "\n".join(lines)


def compare_report(n: int = 1024, seed: int = 7, batch: int = 1, n_kv: int = 4, group: int = 1,
                   cfg: AlignConfig = AlignConfig(), baseline_bits: int = 13, k_sel: int = 32, m: int = 5,
                   strategy: str = "element", scale: float = 4.0, device=None, data=None) -> CompareReport:
    """Aligned and baseline_truncated(bits) vs reference on identical inputs (fp16 output grid, A-hist)."""
    from paper_2409_16546_b200.attention_decode import baseline_truncated, decode_step, reference_output, \
        reference_scores

    st, q = _build(n, batch, n_kv, group, seed, scale, device, data)
    r = decode_step(q, st, cfg, k_sel=k_sel, m=m, strategy=strategy, return_scores=True)
    s_al, o_al, p = r.scores.clone(), r.o.clone(), r.probs.clone()
    s_ref = reference_scores(q, st).clone()
    o_ref = reference_output(p, st).clone()
    s_tr, o_tr = baseline_truncated(q, st, p, baseline_bits)
    H = relative_error_histogram
    hist = {("aligned", "qk"): H(s_al, s_ref, True), ("aligned", "sv"): H(o_al, o_ref, True),
            ("trunc", "qk"): H(s_tr, s_ref, True), ("trunc", "sv"): H(o_tr, o_ref, True)}
    c = r.counters.view(-1, 8).sum(0).cpu().numpy().astype(np.int64)
    avg = {"aligned_k": _avg(*c[0:3]), "aligned_v": _avg(*c[3:6]),
           "aligned": _avg(c[0] + c[3], c[1] + c[4], c[2] + c[5]), "baseline": float(baseline_bits)}
    return CompareReport(hist, avg, baseline_bits)
