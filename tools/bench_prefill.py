"""Prefill writer throughput: one bulk append of n tokens into every (batch, kv-head)
unit of an empty store (config c2 shapes by default), CUDA events, median of reps.

    python tools/bench_prefill.py [--batch 16] [--kv-heads 32] [--n 4096] [--reps 5]

Reports the page-span writer (akv_append_ws, what KVStore.append runs) and the round-1
path (akv_append: validate -> per-token byte scatter -> commit) on the same input.
input GB/s = K+V fp16 bytes / time; moved GB/s adds the plane bytes written (= input)."""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_16546_b200 import KVStore, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    st = KVStore(a.batch, a.kv_heads, 128, a.n)
    k = torch.randn(a.batch, a.kv_heads, a.n, 128, device="cuda").half()
    v = torch.randn(a.batch, a.kv_heads, a.n, 128, device="cuda").half()
    L = _lib.lib()
    inb = 2 * k.numel() * 2
    out = {"config": {"batch": a.batch, "kv_heads": a.kv_heads, "tokens": a.n}, "input_bytes": inb}

    def run(kind):
        ts = []
        for r in range(a.reps + 1):
            st.rewind(0)
            st.status_dev.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ws = st._append_workspace(a.n)
            torch.cuda.synchronize()
            e0.record()
            if kind == "ws":
                rc = L.akv_append_ws(ctypes.byref(st.c_store), k.data_ptr(), v.data_ptr(), a.n, st.status_dev.data_ptr(),
                                     ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
            else:
                rc = L.akv_append(ctypes.byref(st.c_store), k.data_ptr(), v.data_ptr(), a.n, st.status_dev.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0 and int(st.status_dev.abs().sum()) == 0
            if r:
                ts.append(e0.elapsed_time(e1) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        return {"ms": t * 1e3, "input_GBps": inb / t / 1e9, "moved_GBps": 2 * inb / t / 1e9}

    out["page_span_writer"] = run("ws")
    out["round1_append"] = run("legacy")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
