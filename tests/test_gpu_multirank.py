"""Multi-rank decode through the real CUDA chain, on one GPU.

Two processes (gloo process group; both ranks drive cuda:0 — the GPU box gives
one device) each own a shard of the (batch, kv-head) units (`shard_for`), build
their own paged store from the globally seeded units, run the full libakv step
(append + qk + select + pv + combine) and all-gather o and the counters.  The
reassembled output must be bit-identical to the single-rank run over all units,
and the summed counters equal to its counters: units are independent and every
reduction inside a unit has a fixed order, so the rank count cannot change a bit.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B, HKV, N = 4, 4, 700


def _decode(units, batch, n_kv, g):
    from paper_2409_16546_b200 import KVStore
    from paper_2409_16546_b200 import attention_decode as AD
    from paper_2409_16546_b200.synth import fill_store, generate_batch

    K, V, Q = generate_batch(batch, HKV, N, 128, g, 7, units=units)  # global seeds (u // HKV, u % HKV)
    st = KVStore(batch, n_kv, 128, N, strict=False)
    fill_store(st, K, V, N)
    q = torch.from_numpy(Q.view(np.int16)).view(batch, n_kv * g, 128)
    r = AD.decode_step(q, st)
    return r.o.cpu(), r.counters.cpu().sum((0, 1))


def _worker(rank, world, port, scheme, g, out):
    import torch.distributed as dist

    from paper_2409_16546_b200.shard import gather_counters, gather_outputs, shard_for

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard_for(B, HKV, world, rank, scheme)
        o, cnt = _decode(sh.units(HKV), sh.batch, sh.kv_heads, g)
        full = gather_outputs(o, sh, B, HKV, g)
        tot = gather_counters(cnt)
        if rank == 0:
            torch.save({"o": full, "cnt": tot}, out)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("scheme,g", [("batch", 1), ("kv_head", 4)])
def test_two_ranks_real_chain_bit_identical(scheme, g, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    out = str(tmp_path / "gathered.pt")
    mp.start_processes(_worker, args=(2, _free_port(), scheme, g, out), nprocs=2, start_method="spawn", join=True)
    got = torch.load(out)
    ref_o, ref_cnt = _decode(list(range(B * HKV)), B, HKV, g)
    assert torch.equal(got["o"], ref_o), "W=2 output differs from W=1"
    assert torch.equal(got["cnt"], ref_cnt), "W=2 counters differ from W=1"


def test_bench_refuses_more_ranks_than_devices():
    """`bench.py --gpus N` with fewer devices than N must fail loudly, never report N=1."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = torch.cuda.device_count() + 1
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode != 0
    assert f"needs {n} devices" in res.stderr
    assert not [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
