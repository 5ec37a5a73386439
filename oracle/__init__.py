"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the AlignedKV reference
(`/root/reference/SPEC.md` modules half_bits, align_core, kv_store,
attention_decode, analysis; the shipped bit model
`pkg/src/alignedkv/half_bits.py`, cited as HB) together with the pinned
decisions of SURVEY.md Appendix A (A-planes, A-merge, A-K, D1-D11, A-hist).

It exists to CHECK the CUDA product path and to provide the CPU baseline
timing in bench.py.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py` (cpu_baseline leg and `--impl reference`) may import it.  The
product package `paper_2409_16546_b200` never imports it and has no CPU
fallback.

Pinning status:
  * Bit-level leaf functions (half_bits) are pinned against the reference's
    own `half_bits.py`: exhaustively over all 65536 patterns in this
    container, and through committed sha256 digests of the reference's
    outputs (`tests/golden/half_bits_digests.json`) everywhere else.
  * align_core / kv_store / attention_decode / analysis exist upstream only
    as SPEC text; they are pinned by the SPEC worked examples
    (`tests/golden/spec_examples.json`) and acceptance criteria
    SPEC.md:583-590.  Where SPEC is silent, Appendix A decides — upstream
    parity at those points is unpinned.
"""

from oracle import half_bits, align_core, kv_store, attention_decode, analysis  # noqa: F401
