"""Host-side analysis pieces (no GPU): alignment_bruteforce, SPEC.md:428-436 + acceptance 3."""

import numpy as np

from oracle.analysis import alignment_bruteforce as o_brute
from paper_2409_16546_b200 import analysis as A


def test_bruteforce_matches_spec_examples():
    assert A.alignment_bruteforce([1, -5], -9) == (12, 12)
    assert A.alignment_bruteforce([0, 0], -10) == (18, 18)
    assert A.alignment_bruteforce([-20], -9) == (0, 0)


def test_bruteforce_optimality_and_oracle_agreement():
    rng = np.random.default_rng(5)
    for _ in range(300):
        k = int(rng.integers(1, 4))
        exps = [int(x) for x in rng.integers(-12, 6, k)]
        u = max(exps) - 10 + int(rng.integers(0, 6))
        best, aligned = A.alignment_bruteforce(exps, u)
        assert (best, aligned) == o_brute(exps, u)
        if best is not None:
            assert best == aligned
