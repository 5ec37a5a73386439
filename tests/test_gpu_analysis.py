"""GPU analysis path against the oracle's analysis module."""

import numpy as np
import pytest
import torch

from oracle import half_bits as ohb
from oracle.analysis import relative_error_histogram as o_hist
from oracle.analysis import relative_error_buckets
from paper_2409_16546_b200 import analysis as A

pytestmark = pytest.mark.gpu


def test_histogram_counts_equal_oracle():
    rng = np.random.default_rng(3)
    ref = rng.standard_normal(200_003).astype(np.float32)
    rel = np.exp2(rng.uniform(-14, -5, ref.size)) * rng.choice([-1, 1], ref.size)
    test = (ref * (1 + rel)).astype(np.float32)
    test[::17] = ref[::17]                    # exact
    ref[::101] = 0.0                          # ref = 0, test != 0 -> last bucket
    test[::303] = 0.0
    ref[::303] = 0.0                          # both 0 -> {0}
    # exact bucket edges: 1 vs 1 + 2^-10, 1 + 2^-9, ...
    ref[:5] = 1.0
    test[:5] = [1.0, 1 + 2 ** -11, 1 + 2 ** -10, 1 + 2 ** -9, 2.0]
    for rnd in (False, True):
        g = A.relative_error_histogram(test, ref, fp16_round=rnd)
        t, r = (ohb.float16_round(test.astype(np.float64)), ohb.float16_round(ref.astype(np.float64))) if rnd \
            else (test, ref)
        counts = np.bincount(relative_error_buckets(t, r), minlength=6)
        assert np.array_equal(g.counts, counts), (rnd, g.counts, counts)
        assert np.allclose(g.fractions, o_hist(t, r))


def test_histogram_spec_examples():
    # SPEC.md:416-418
    assert A.relative_error_histogram([1.0, 2.0], [1.0, 2.0]).counts.tolist() == [2, 0, 0, 0, 0, 0]
    h = A.relative_error_histogram([1, 1 + 2 ** -11, 1 + 2 ** -9, 2], [1, 1, 1, 1])
    assert h.counts.tolist() == [1, 1, 0, 1, 0, 1]
    assert A.relative_error_histogram([0.0], [0.0]).counts.tolist() == [1, 0, 0, 0, 0, 0]
    with pytest.raises(ValueError):
        A.relative_error_histogram([1.0], [1.0, 2.0])


def test_bitwidth_sweep_forced_and_aligned():
    flat = A.bitwidth_sweep([256, 512], force_tier=16, n_kv=2)
    assert [p.avg_bits for p in flat.points] == [16.0, 16.0]
    c1 = A.bitwidth_sweep([256, 1024], n_kv=4)
    c2 = A.bitwidth_sweep([256, 1024], n_kv=4)
    assert c1.rows() == c2.rows()  # determinism
    assert all(8.0 <= p.avg_bits <= 16.0 for p in c1.points)
    assert c1.points[-1].avg_bits <= 13.0  # acceptance 4 (n >= 1024)
    with pytest.raises(ValueError):
        A.bitwidth_sweep([512, 256])


def test_compare_report_dominance():
    rep = A.compare_report(n=1024, n_kv=4)
    for op in ("qk", "sv"):
        assert rep.hist[("aligned", op)].fractions[0] > rep.hist[("trunc", op)].fractions[0]
    rep16 = A.compare_report(n=256, n_kv=2, baseline_bits=16)
    for op in ("qk", "sv"):
        assert rep16.hist[("trunc", op)].fractions[0] == 1.0
    assert "paper" in rep.table()

