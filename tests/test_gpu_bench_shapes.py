"""Parity at the exact benchmark shapes (BASELINE.json configs 2-4), through the C ABI.

The bench times these shapes; these tests check the same kernels on them:
  * every q-head's K tier mask and ColMax against the oracle (cheap: Rule 1 needs
    only q and ColMax);
  * a spread sample of units in full (scores, selection, V tier mask incl. the
    injection check, AccessCounter totals, o) via oracle.parity.check_head;
  * the serving path (no V-mask export: the pv stage / quad fast paths) takes the same
    tier decisions as the export path (identical counters) and its o matches the oracle.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import attention_decode as OA
from oracle.align_core import k_channel_tiers
from oracle.kv_store import KVStore as OStore
from oracle.parity import check_head, close
from paper_2409_16546_b200 import KVStore
from paper_2409_16546_b200 import attention_decode as AD
from paper_2409_16546_b200.synth import fill_store, generate_batch

SHAPES = {  # name: (B, Hkv, g, n, sampled units)
    "c2": (16, 32, 1, 4096, (0, 37, 200, 511)),
    "c3": (32, 8, 4, 8192, (0, 99, 255)),
    "c4": (8, 32, 1, 32768, (0, 255)),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_bench_shape_parity(name):
    B, Hkv, g, n, sample = SHAPES[name]
    d = 128
    workers = max(1, min(16, len(os.sched_getaffinity(0))))
    K, V, Q = generate_batch(B, Hkv, n, d, g, 7, workers=workers)
    store = KVStore(B, Hkv, d, n, strict=False)
    fill_store(store, K, V, n - 1)
    store.append_token(torch.from_numpy(np.ascontiguousarray(K[:, n - 1]).view(np.int16)).view(B, Hkv, d),
                       torch.from_numpy(np.ascontiguousarray(V[:, n - 1]).view(np.int16)).view(B, Hkv, d))
    q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)

    r = AD.decode_step(q, store, return_scores=True, export_v_tiers=True)
    srv = AD.decode_step(q, store)  # the serving path the bench times
    assert torch.equal(srv.counters, r.counters)

    # every head: ColMax and the K tier mask
    colmax = (K & 0x7FFF).max(axis=1)
    assert np.array_equal(store.colmax().cpu().numpy().reshape(-1, d).astype(np.uint16), colmax)
    kt = r.k_tiers.cpu().numpy().reshape(B * Hkv, g, d)
    for u in range(B * Hkv):
        for j in range(g):
            assert np.array_equal(kt[u, j], k_channel_tiers(Q[u, j], colmax[u])), (name, u, j)

    # sampled units in full
    o_srv = srv.o.cpu().numpy()
    edges = heads = 0
    for u in sample:
        b, h = divmod(u, Hkv)
        ost = OStore(d)
        ost.append_rows(K[u], V[u])
        for j in range(g):
            hq = h * g + j
            ref = OA.decode_head(Q[u, j], ost)
            fail, edge = check_head(ref, k_tiers=r.k_tiers[b, hq].cpu().numpy(), o=r.o[b, hq].cpu().numpy(),
                                    counters=r.counters[b, hq].cpu().numpy(), sel=r.selection(b, hq),
                                    v_tiers=r.v_tiers[b, hq].cpu().numpy(), s=r.scores[b, hq].cpu().numpy(),
                                    p=r.probs[b, hq].cpu().numpy(), targets=r.targets[b, hq].cpu().numpy(),
                                    v_head=V[u] >> 8)
            assert not fail, (name, u, j, fail)
            assert close(o_srv[b, hq], ref.o), (name, u, j)
            edges += edge
            heads += 1
    assert edges <= max(1, heads // 4), f"{edges} knife-edge heads of {heads}"
