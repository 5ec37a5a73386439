"""Pin the oracle's bit model to the reference half_bits.py.

* digests: the oracle's outputs over all 65536 patterns must hash to the
  committed digests of the reference's outputs (works everywhere);
* live: where /root/reference exists, compare directly;
* SPEC acceptance criterion 1: exhaustive roundtrip,
  truncation bound, T16 losslessness.
"""

import json
import os

import numpy as np
import pytest

from oracle import half_bits as hb
from tests.golden.make_golden import digest, float_probe

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def oracle_arrays():
    allw = np.arange(65536, dtype=np.uint16)
    fin = hb.finite_mask(allw)
    fw = allw[fin]
    out = {"finite_mask": fin.astype(np.uint8)}
    out["decode_array"] = hb.decode_array(fw)
    out["ulp_exponent_array"] = hb.ulp_exponent_array(fw).astype(np.int32)
    nz = fw[(fw & 0x7FFF) != 0]
    out["magnitude_exponent"] = hb.magnitude_exponent_array(nz).astype(np.int32)
    for t in range(11):
        out[f"truncate_fill_array_t{t}"] = hb.truncate_fill_array(fw, t)
    out["truncate_fill_scalar_t7_stride"] = np.array([hb.truncate_fill(int(w), 7) for w in fw[::97]], np.uint16)
    c0, c1, c2 = hb.split_chunks_array(allw)
    out["split_chunks"] = np.stack([c0, c1, c2], axis=1).astype(np.int32)
    out["merge_c0"] = np.array([hb.merge_chunks(h) for h in range(256)], np.int32)
    out["merge_c0c1"] = np.array([hb.merge_chunks(h, m) for h in range(256) for m in range(16)], np.int32)
    out["merge_full_roundtrip"] = np.array([hb.merge_chunks(*hb.split_chunks(int(w))) for w in allw], np.int32)
    x = float_probe()
    out["encode_array"] = hb.encode_array(x)
    out["float16_round"] = hb.float16_round(x)
    out["frexp_exponents"] = hb.frexp_exponents(x[x != 0])
    return out


def test_oracle_matches_reference_digests():
    with open(os.path.join(GOLDEN, "half_bits_digests.json")) as f:
        want = json.load(f)
    got = oracle_arrays()
    missing = set(want) - set(got) - {"_source"}
    assert not missing, missing
    bad = [k for k, v in got.items() if digest(v) != want[k]]
    assert not bad, f"oracle differs from reference half_bits on: {bad}"


def test_oracle_matches_reference_live(ref_half_bits):
    ref = ref_half_bits
    allw = np.arange(65536, dtype=np.uint16)
    fw = allw[ref.finite_mask(allw)]
    for t in (0, 2, 6, 7, 10):
        assert np.array_equal(hb.truncate_fill_array(fw, t), ref.truncate_fill_array(fw, t))
    per = np.random.default_rng(0).integers(0, 11, fw.size)
    assert np.array_equal(hb.truncate_fill_array(fw, per), ref.truncate_fill_array(fw, per))
    for w in range(0, 65536, 7):
        assert hb.split_chunks(w) == tuple(ref.split_chunks(w))
        if ref.is_finite_word(w):
            assert hb.ulp_exponent(w) == ref.ulp_exponent(w)
            if w & 0x7FFF:
                assert hb.magnitude_exponent(w) == ref.magnitude_exponent(w)
    # error behaviour mirrors the reference messages
    with pytest.raises(ValueError, match="non-prefix tier"):
        hb.merge_chunks(0x3C, None, 1)
    with pytest.raises(ValueError, match="zero has no magnitude exponent"):
        hb.magnitude_exponent(0)
    with pytest.raises(ValueError, match=r"kept mantissa bits must be in \[0, 10\]"):
        hb.truncate_fill(0x3C00, 11)
    with pytest.raises(ValueError, match="non-finite"):
        hb.ulp_exponent(0x7C00)


def test_acceptance1_exhaustive():
    """roundtrip, truncation bound, T16 losslessness (< 1 s)."""
    allw = np.arange(65536, dtype=np.uint16)
    fw = allw[hb.finite_mask(allw)]
    c0, c1, c2 = hb.split_chunks_array(fw)
    assert np.array_equal(hb.merge_tier_array(c0, c1, c2, 16), fw)
    assert np.array_equal(hb.merge_tier_array(c0, c1, c2, 8), hb.truncate_fill_array(fw, 2))
    assert np.array_equal(hb.merge_tier_array(c0, c1, c2, 12), hb.truncate_fill_array(fw, 6))
    val = hb.decode_array(fw)
    ulp = hb.ulp_exponent_array(fw).astype(np.float64)
    normal = ((fw >> 10) & 0x1F) > 0
    for t in range(11):
        tr = hb.truncate_fill_array(fw, t)
        err = np.abs(hb.decode_array(tr) - val)
        bound = np.exp2(9 - t + ulp)
        assert (err[normal] <= bound[normal]).all()
        # sign and exponent preserved
        assert np.array_equal(tr & 0xFC00, fw & 0xFC00)


def test_spec_examples_half_bits():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        ex = json.load(f)
    for w, v, _ in ex["decode"]:
        assert hb.decode(w) == v
    for v, w, _ in ex["encode"]:
        assert hb.encode(v) == w
    for w, u, _ in ex["ulp_exponent"]:
        assert hb.ulp_exponent(w) == u
    for w, t, o, _ in ex["truncate_fill"]:
        assert hb.truncate_fill(w, t) == o
    for w, ch, _ in ex["split_chunks"]:
        assert list(hb.split_chunks(w)) == ch
    for ch, o, _ in ex["merge_chunks"]:
        assert hb.merge_chunks(*ch) == o
