"""The shared parity checker (oracle.parity) on CPU: the oracle against itself passes, and a
single flipped tier / counter / selection is caught."""

import numpy as np

from oracle import attention_decode as OA
from oracle.kv_store import KVStore as OStore
from oracle.parity import check_head
from paper_2409_16546_b200.synth import generate_batch


def _ref(n=600, seed=3, lo=-4.0, hi=4.0):
    K, V, Q = generate_batch(1, 1, n, 128, 1, seed, lo, hi)
    st = OStore(128)
    st.append_rows(K[0], V[0])
    return OA.decode_head(Q[0, 0], st), V[0]


def _args(ref, V):
    from oracle.align_core import rule2_targets_array

    tg, known = rule2_targets_array(ref.o_est)
    tg = np.where(known, tg, -(1 << 31))
    cnt = np.array(list(ref.k_counter.as_tuple()) + list(ref.v_counter.as_tuple()) + [0, 0])
    return dict(k_tiers=ref.k_tiers.copy(), o=ref.o.copy(), counters=cnt, sel=ref.sel.copy(),
                v_tiers=ref.v_tiers.copy(), s=ref.s.copy(), p=ref.p.copy(), targets=tg, v_head=V >> 8)


def test_self_consistent():
    for lo, hi in ((-4.0, 4.0), (-0.5, 0.5)):
        ref, V = _ref(lo=lo, hi=hi)
        fail, _ = check_head(ref, **_args(ref, V))
        assert fail == []


def test_detects_single_flips():
    ref, V = _ref(lo=-0.5, hi=0.5)
    a = _args(ref, V)
    a["v_tiers"][5, 7] = 8 if a["v_tiers"][5, 7] != 8 else 12
    fail, _ = check_head(ref, **a)
    assert "v_tiers" in fail and "v_tiers_injection" in fail
    a = _args(ref, V)
    a["k_tiers"][3] ^= 4
    assert "k_tiers" in check_head(ref, **a)[0]
    a = _args(ref, V)
    a["counters"][4] += 1
    assert "v_counter" in check_head(ref, **a)[0]
    a = _args(ref, V)
    a["o"][np.argmax(np.abs(a["o"]))] *= 1.01
    assert "o" in check_head(ref, **a)[0]
