"""Shared helpers for the GPU parity tests: build the same units on the GPU
store and in the CPU oracle, run both, compare (SURVEY §8(c) contract)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import attention_decode as OA
from oracle.align_core import AlignConfig as OAlignConfig
from oracle.kv_store import KVStore as OStore
from oracle.parity import check_head, close  # noqa: F401  (re-exported for the tests)
from paper_2409_16546_b200 import AlignConfig, KVStore
from paper_2409_16546_b200.attention_decode import decode_step
from paper_2409_16546_b200.synth import generate_batch


class Case:
    """B x Hkv units with n tokens (n-1 bulk + 1 appended), g q-heads per kv-head."""

    def __init__(self, B=2, Hkv=2, g=1, n=300, seed=11, lo=-4.0, hi=4.0, capacity=None, mutate=None):
        self.B, self.Hkv, self.g, self.n = B, Hkv, g, n
        K, V, Q = generate_batch(B, Hkv, n, 128, g, seed, lo, hi)
        if mutate is not None:  # edit the synthetic units in place before they are stored
            mutate(K, V, Q)
        self.K, self.V, self.Q = K, V, Q  # [U,n,d], [U,n,d], [U,g,d]
        cap = capacity or max(256, n)
        self.store = KVStore(B, Hkv, 128, cap)
        d = 128
        kt = torch.from_numpy(K.view(np.int16)).view(B, Hkv, n, d)
        vt = torch.from_numpy(V.view(np.int16)).view(B, Hkv, n, d)
        if n > 1:
            self.store.append(kt[:, :, : n - 1], vt[:, :, : n - 1])
        self.store.append_token(kt[:, :, n - 1], vt[:, :, n - 1])
        self.q = torch.from_numpy(Q.view(np.int16)).view(B, Hkv * g, d)
        self._ostores = {}

    def ostore(self, u) -> OStore:
        if u not in self._ostores:
            st = OStore(128)
            st.append_rows(self.K[u], self.V[u])
            self._ostores[u] = st
        return self._ostores[u]

    def units(self):
        for u in range(self.B * self.Hkv):
            b, h = divmod(u, self.Hkv)
            for j in range(self.g):
                yield u, b, h * self.g + j, j

    def gpu(self, **kw):
        return decode_step(self.q, self.store, kw.pop("cfg", AlignConfig()), return_scores=True,
                           export_v_tiers=True, **kw)

    def oracle(self, u, j, cfg=OAlignConfig(), **kw):
        return OA.decode_head(self.Q[u, j], self.ostore(u), cfg, **kw)
