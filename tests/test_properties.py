"""Property tests of the alignment rules (pyproject test extra `hypothesis`).

CPU: the package's host mirror of align_core (paper_2409_16546_b200.align_core) and the
oracle agree and satisfy soundness, scale covariance and tier dominance.
GPU: the same properties through the kernels (K tier masks, scores).
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as hs

from oracle import align_core as OAC
from oracle import half_bits as ohb
from paper_2409_16546_b200 import align_core as AC

D = 8  # small channel count keeps the properties exhaustive-ish per example


def finite_half(nonzero=False):
    """Finite fp16 bit patterns (both signs, subnormals included)."""
    lo = 1 if nonzero else 0
    return hs.builds(lambda mag, neg: (mag | (0x8000 if neg else 0)), hs.integers(lo, 0x7BFF), hs.booleans())


@settings(max_examples=300, deadline=None)
@given(hs.lists(finite_half(nonzero=True), min_size=D, max_size=D),
       hs.lists(finite_half(nonzero=True), min_size=D, max_size=D), hs.integers(-2, 4))
def test_mirror_equals_oracle(q, cm, margin):
    cm = [w & 0x7FFF for w in cm]
    a = AC.k_channel_tiers(q, cm, AC.AlignConfig(margin_bits=margin))
    b = OAC.k_channel_tiers(np.array(q, np.uint16), np.array(cm, np.uint16), OAC.AlignConfig(margin_bits=margin))
    assert [int(t) for t in a] == [int(t) for t in np.asarray(b)]
    assert AC.rule1_target(q, cm) == OAC.rule1_target(np.array(q, np.uint16), np.array(cm, np.uint16))


@settings(max_examples=300, deadline=None)
@given(hs.lists(finite_half(nonzero=True), min_size=D, max_size=D),
       hs.lists(finite_half(nonzero=True), min_size=D, max_size=D), hs.data())
def test_soundness(q, cm, data):
    """with margin 0, truncating column c to its tier's kept bits bounds the
    per-product error by 2^u for every K element |k| <= colmax_c.

    Holds for NORMAL colmax only: with a subnormal colmax the midpoint fill of a
    truncated zero / subnormal element (A-merge: +0 at T8 -> 0x0080 = 2^-17) exceeds
    the bound (found by this test: q = colmax = 2^-24, k = 0).  SPEC is silent on
    subnormal magnitudes; recorded in DESIGN.md section 4."""
    cm = [0x0400 | (w & 0x7FFF) if (w & 0x7C00) == 0 else (w & 0x7FFF) for w in cm]  # normal colmax
    u = AC.rule1_target(q, cm)
    tiers = AC.k_channel_tiers(q, cm)
    for c in range(D):
        if tiers[c] == AC.Tier.SKIP:
            continue
        kept = tiers[c].kept_bits
        # K element no larger in magnitude than colmax_c
        k = data.draw(hs.integers(0, cm[c])) | (0x8000 if data.draw(hs.booleans()) else 0)
        kt = int(ohb.truncate_fill(k, kept))
        err = abs(ohb.decode(q[c]) * (ohb.decode(kt) - ohb.decode(k)))
        assert err <= 2.0 ** u, (c, hex(q[c]), hex(cm[c]), hex(k), kept, u)


@settings(max_examples=300, deadline=None)
@given(hs.lists(hs.integers(1, 0x3FFF), min_size=D, max_size=D),
       hs.lists(finite_half(nonzero=True), min_size=D, max_size=D), hs.integers(-3, 3))
def test_scale_covariance(qmag, cm, sft):
    """q * 2^s shifts rule1_target by s and keeps the tiers (normal q, no overflow)."""
    cm = [w & 0x7FFF for w in cm]
    q = [0x2000 | (m & 0x1FFF) for m in qmag]  # normal, mid-range exponents: scaling stays exact
    qs = [int(ohb.encode(ohb.decode(w) * 2.0 ** sft)) for w in q]
    assert all(ohb.decode(a) * 2.0 ** sft == ohb.decode(b) for a, b in zip(q, qs))
    assert AC.rule1_target(qs, cm) == AC.rule1_target(q, cm) + sft
    assert AC.k_channel_tiers(qs, cm) == AC.k_channel_tiers(q, cm)


@settings(max_examples=300, deadline=None)
@given(hs.lists(finite_half(), min_size=D, max_size=D),
       hs.lists(finite_half(nonzero=True), min_size=D, max_size=D), hs.integers(-2, 3))
def test_tier_dominance(q, cm, margin):
    """increasing margin_bits never lowers a tier."""
    cm = [w & 0x7FFF for w in cm]
    if not any((w & 0x7FFF) for w in q):
        return  # degenerate
    lo = AC.k_channel_tiers(q, cm, AC.AlignConfig(margin_bits=margin))
    hi = AC.k_channel_tiers(q, cm, AC.AlignConfig(margin_bits=margin + 1))
    assert all(int(b) >= int(a) for a, b in zip(lo, hi))


@pytest.mark.gpu
def test_gpu_scale_covariance_and_dominance():
    """Through the kernels: q * 2 leaves the K masks unchanged and doubles every score
    exactly; margin + 1 never lowers a K tier."""
    import torch

    from paper_2409_16546_b200 import AlignConfig, KVStore
    from paper_2409_16546_b200.attention_decode import decode_step
    from paper_2409_16546_b200.synth import generate_batch

    B, H, n = 2, 2, 600
    K, V, Q = generate_batch(B, H, n, 128, 1, 21, -2.0, 2.0)
    st = KVStore(B, H, 128, 1024)
    st.append(torch.from_numpy(K.view(np.int16)).view(B, H, n, 128), torch.from_numpy(V.view(np.int16)).view(B, H, n, 128))
    q = Q.view(np.float16).reshape(B, H, 128)
    r1 = decode_step(torch.from_numpy(q.copy()), st, return_scores=True)
    r2 = decode_step(torch.from_numpy((q.astype(np.float32) * 2).astype(np.float16)), st, return_scores=True)
    assert torch.equal(r1.k_tiers, r2.k_tiers)
    assert torch.equal(r1.scores * 2, r2.scores)
    for m in (-2, -1, 0, 1, 2, 3):
        a = decode_step(torch.from_numpy(q.copy()), st, AlignConfig(margin_bits=m)).k_tiers.cpu().numpy()
        b = decode_step(torch.from_numpy(q.copy()), st, AlignConfig(margin_bits=m + 1)).k_tiers.cpu().numpy()
        assert (b.astype(int) >= a.astype(int)).all()
