"""CPU-side checks of the C-ABI boundary and the host logic (no GPU compute).

* libakv.so loads and exports every symbol include/akv.h declares;
* the ctypes structs match the header's field order and sizes;
* workspace sizing is callable without a device;
* the product path fails loudly without a GPU (no CPU fallback);
* host API mirror semantics (align_core, half_bits) on SPEC examples.
"""

import ctypes
import json
import os
import re

import numpy as np
import pytest

from paper_2409_16546_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "akv.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t)\s+(akv_\w+)\(", txt, re.M)))


def test_header_and_binding_agree():
    assert _declared() == sorted(_lib.EXPORTED_SYMBOLS)


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2409_16546_b200.build import build

        build()
    return _lib.lib()


def test_library_exports_every_declared_symbol(L):
    for name in _declared():
        assert hasattr(L, name), name
    assert L.akv_version() == 100


def test_struct_layouts_match_header():
    txt = open(HEADER).read()

    def fields(struct):
        body = re.search(r"typedef struct \{([^}]*)\}\s*" + struct + ";", txt).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        return [re.findall(r"(\w+)\s*;", line)[0] for line in body.splitlines() if ";" in line]

    assert fields("akv_store_t") == [f[0] for f in _lib.AkvStore._fields_]
    assert fields("akv_cfg_t") == [f[0] for f in _lib.AkvCfg._fields_]
    assert fields("akv_step_t") == [f[0] for f in _lib.AkvStep._fields_]
    assert ctypes.sizeof(_lib.AkvStore) == 16 + 6 * 8
    assert ctypes.sizeof(_lib.AkvCfg) == 32
    assert ctypes.sizeof(_lib.AkvStep) == 19 * 8


def test_workspace_sizes(L):
    a = L.akv_workspace_bytes(512, 1, 16)
    b = L.akv_workspace_bytes(512, 1, 32)
    assert 0 < a < b
    # scores dominate: U*g*cap*4 bytes
    assert a >= 512 * 16 * 256 * 4
    assert L.akv_workspace_bytes(-1, 1, 1) == _lib.AKV_EINVAL


def test_invalid_arguments_rejected_without_launch(L):
    st = _lib.AkvStore(1, 64, 1, 0, None, None, None, None, None, None)  # head_dim 64 unsupported
    cfg = _lib.AkvCfg(1, 0, 1, 0, 32, 5, 0, 0)
    step = _lib.AkvStep()
    assert L.akv_qk(ctypes.byref(st), ctypes.byref(cfg), ctypes.byref(step), 10, None) == _lib.AKV_EUNSUPPORTED
    st.head_dim = 128
    bad = _lib.AkvCfg(3, 0, 1, 0, 32, 5, 0, 0)
    assert L.akv_decode_step(ctypes.byref(st), ctypes.byref(bad), ctypes.byref(step), 10, None) == _lib.AKV_EUNSUPPORTED
    bad = _lib.AkvCfg(1, 9, 1, 0, 32, 5, 0, 0)
    assert L.akv_pv(ctypes.byref(st), ctypes.byref(bad), ctypes.byref(step), 10, None) == _lib.AKV_EINVAL
    assert L.akv_append(None, None, None, 1, None, None) == _lib.AKV_EINVAL


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2409_16546_b200 import KVStore

    with pytest.raises(_lib.AkvError, match="no CPU fallback"):
        KVStore(1, 1)


def test_host_align_core_mirror_on_spec_examples():
    from paper_2409_16546_b200 import align_core as A
    from paper_2409_16546_b200 import half_bits as H

    ex = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    W = lambda xs: [H.encode(x) for x in xs]  # noqa: E731
    for pe, u, mg, want, _ in ex["required_mantissa_bits"]:
        assert A.required_mantissa_bits(pe, u, A.AlignConfig(mg)) == want
    for t, want, _ in ex["tier_for_bits"]:
        assert int(A.tier_for_bits(t)) == want
    for q, cm, want, _ in ex["rule1_target"]:
        assert A.rule1_target(W(q), W(cm)) == want
    for o, want, _ in ex["rule2_targets"]:
        assert A.rule2_targets(o) == want
    for q, cm, want, _ in ex["k_channel_tiers"]:
        assert [int(t) for t in A.k_channel_tiers(W(q), W(cm))] == want
    with pytest.raises(A.DegenerateInputError):
        A.rule1_target(W([0.0]), W([1.0]))
    for w, t, o, _ in ex["truncate_fill"]:
        assert H.truncate_fill(w, t) == o
    for ch, o, _ in ex["merge_chunks"]:
        assert H.merge_chunks(*ch) == o
    with pytest.raises(ValueError, match="non-prefix tier"):
        H.merge_chunks(1, None, 2)


def test_host_half_bits_matches_reference_digests():
    """The package's host half_bits module is pinned to the same reference digests as the oracle."""
    from paper_2409_16546_b200 import half_bits as H
    from tests.golden.make_golden import digest

    want = json.load(open(os.path.join(ROOT, "tests", "golden", "half_bits_digests.json")))
    allw = np.arange(65536, dtype=np.uint16)
    fw = allw[H.finite_mask(allw)]
    assert digest(H.finite_mask(allw).astype(np.uint8)) == want["finite_mask"]
    assert digest(H.decode_array(fw)) == want["decode_array"]
    assert digest(H.ulp_exponent_array(fw).astype(np.int32)) == want["ulp_exponent_array"]
    for t in range(11):
        assert digest(H.truncate_fill_array(fw, t)) == want[f"truncate_fill_array_t{t}"]
