"""Multi-rank host logic on CPU: world_size 2 over gloo.

Each rank takes its block of (batch, kv-head) units (`shard_for`), computes
those units' decode outputs (here with the CPU oracle standing in for the GPU
chain, which needs a B200), all-gathers them with `gather_outputs`, and the
reassembled tensor must be bit-identical to the single-rank result — the
property the GPU run relies on (units are independent; per-unit arithmetic
does not depend on the rank count).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_16546_b200.shard import gather_counters, gather_outputs, shard_for
from paper_2409_16546_b200.synth import generate_unit

B, HKV, G, N, D = 2, 4, 2, 48, 128


def _unit_outputs(units):
    from oracle import attention_decode as OA
    from oracle.kv_store import KVStore as OStore

    out, cnt = [], np.zeros(6, np.int64)
    for u in units:
        K, V, Q = generate_unit(N, D, G, 7, u // HKV, u % HKV)
        st = OStore(D)
        st.append_rows(K, V)
        for j in range(G):
            r = OA.decode_head(Q[j], st)
            out.append(r.o)
            kt = r.k_tiers
            cnt[0] += int((kt == 8).sum()) * N
    return np.stack(out), cnt


def _worker(rank, world, port, scheme, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_for(B, HKV, world, rank, scheme)
        o, cnt = _unit_outputs(sh.units(HKV))
        o_local = torch.from_numpy(o).view(sh.batch, sh.kv_heads * G, D)
        full = gather_outputs(o_local, sh, B, HKV, G)
        tot = gather_counters(torch.from_numpy(cnt))
        if rank == 0:
            q.put((full.numpy(), tot.numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("scheme", ["batch", "kv_head"])
def test_two_rank_gather_bit_identical(scheme):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scheme, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tot = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, cnt = _unit_outputs(range(B * HKV))
    assert np.array_equal(full.reshape(-1, D), ref), "W=2 gather differs from W=1"
    assert np.array_equal(tot, cnt)


def test_shard_partitions_cover_units_once():
    for scheme, world in [("batch", 1), ("batch", 2), ("kv_head", 2), ("kv_head", 4)]:
        seen = []
        for r in range(world):
            seen += shard_for(B if scheme == "kv_head" else 4, HKV, world, r, scheme).units(HKV)
        total = (B if scheme == "kv_head" else 4) * HKV
        assert sorted(seen) == list(range(total))
    with pytest.raises(ValueError):
        shard_for(3, HKV, 2, 0, "batch")
    with pytest.raises(ValueError):
        shard_for(B, 3, 2, 0, "kv_head")
    with pytest.raises(ValueError):
        shard_for(B, HKV, 2, 2, "batch")
