"""Aligned decode-attention benchmark (BASELINE.json metric, config 2 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4] [--impl akv|reference]

One step = one decode step of one attention layer over the whole batch:
append the new token's K/V (akv_append) + aligned attention (akv_qk ->
akv_softmax_select -> akv_pv -> akv_combine), plus the NCCL all-gather of the
per-head outputs when N > 1.  Weak scaling: every rank owns its own batch of
B sequences (units are seeded by global batch index, so ranks see disjoint,
reproducible data).  The KV cache (1 GiB at config 2) is larger than L2.

`value` = tokens/s over all ranks = N*B / t_step (device time, max over ranks).
`e2e`   = the same metric through the public API (pinned host q/k/v -> H2D,
          KVStore.append_token + attention_decode.decode, o -> D2H) per step.
`--impl reference` times the CPU oracle (the reference algorithm restated,
kind "port") on this box's cores over a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, Hkv, g, n, description)
    "c1": (1, 1, 1, 1024, "single-head decode, d=128, 1k context, batch 1"),
    "c2": (16, 32, 1, 4096, "Llama-2-7B decode attention: 32 heads, d=128, 4k context, batch 16"),
    "c3": (32, 8, 4, 8192, "Llama-3-8B GQA: 32 q / 8 kv heads, d=128, 8k context, batch 32"),
    "c4": (8, 32, 1, 32768, "long context: Llama-2-7B shapes, 32k context, batch 8"),
}
METRIC = "aligned decode-attn tokens/s & effective KV GB/s vs HBM roofline; bytes-read saving"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on a bounded sample of units, all host cores
# ---------------------------------------------------------------------------
def _cpu_worker(args):
    units, n, g, seed, Hkv, lo, hi, reps = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import attention_decode as OA
    from oracle.kv_store import KVStore as OStore
    from paper_2409_16546_b200.synth import generate_unit

    stores = []
    for u in units:
        K, V, Q = generate_unit(n, 128, g, seed, u // Hkv, u % Hkv, lo, hi)
        st = OStore(128)
        st.append_rows(K[: n - 1], V[: n - 1])
        stores.append((st, K[n - 1], V[n - 1], Q))
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for st, kn, vn, Q in stores:
            s2 = OStore(128)  # step = append the new token + aligned attention for every q-head
            s2.k, s2.v, s2.colmax, s2.rowmax = st.k, st.v, st.colmax, st.rowmax
            s2.append_token(kn, vn)
            for j in range(g):
                OA.decode_head(Q[j], s2)
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(cfg_name, sample_units, reps=1, seed=7, rank_batch0=0):
    import multiprocessing as mp

    B, Hkv, g, n, _ = CONFIGS[cfg_name]
    U = B * Hkv
    cores = len(os.sched_getaffinity(0))
    sample = list(range(rank_batch0 * Hkv, rank_batch0 * Hkv + min(sample_units, U)))
    workers = min(cores, len(sample))
    chunks = [sample[i::workers] for i in range(workers)]
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_cpu_worker, [(c, n, g, seed, Hkv, -4.0, 4.0, reps) for c in chunks])
    # per repetition: wall of the slowest worker (workers run concurrently)
    walls = [max(r[i] for r in res) for i in range(reps)]
    t_sample = float(np.median(walls))
    t_step = t_sample * U / len(sample)
    return {
        "value": B / t_step, "unit": "tokens/s", "cores": workers, "kind": "port",
        "sample": f"{len(sample)} of {U} (batch, kv-head) units x {g} q-heads, n={n}; step time extrapolated "
                  f"linearly x{U / len(sample):.1f}; oracle = numpy float64 restatement (oracle/)",
        "ms_per_step": t_step * 1e3,
    }


def reference_main(args):
    B, Hkv, g, n, desc = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sample = {"c1": 1, "c2": 48, "c3": 24, "c4": 8}[args.config]
    for _ in range(max(args.warmup, 0) and 1):
        cpu_baseline(args.config, min(sample, 8), 1)
    cb = cpu_baseline(args.config, sample, max(args.steps, 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SPEC generator, seed 7)",
        "config": {"workload": args.config, "desc": desc, "batch": B, "kv_heads": Hkv, "q_per_kv": g,
                   "context": n, "head_dim": 128},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle reasons sampled through NVML every ~0.2 ms in a thread
    while the timed region runs (nvidia-smi's 100 ms loop is too coarse for a
    few-ms region); falls back to one nvidia-smi query when NVML is absent."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index):
        import threading

        self.samples, self.reasons, self.mx = [], set(), 0.0
        self.stop_ev = threading.Event()
        self.h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.h = None
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _sample(self):
        nv = self.nv
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for nm, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(nm)

    def _run(self):
        if self.h is None:
            return
        while not self.stop_ev.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.0002)

    def stop(self):
        self.stop_ev.set()
        self.t.join()
        if self.h is not None and not self.samples:
            try:
                self._sample()
            except Exception:
                pass
        if not self.samples:
            return None
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="akv", choices=["akv", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=48)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_main(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2409_16546_b200 import KVStore, _lib
    from paper_2409_16546_b200 import attention_decode as AD
    from paper_2409_16546_b200.synth import generate_batch
    import ctypes

    from paper_2409_16546_b200.shard import shard_for

    B, Hkv, g, n, desc = CONFIGS[args.config]
    U, H, d = B * Hkv, B * Hkv * g, 128
    # weak scaling: the job's batch is world*B rows; this rank owns rows [rank*B, (rank+1)*B)
    units = shard_for(world * B, Hkv, world, rank, "batch").units(Hkv)
    t_gen = time.time()
    K, V, Q = generate_batch(B * world, Hkv, n, d, g, 7, units=units, workers=len(os.sched_getaffinity(0)))
    t_gen = time.time() - t_gen

    store = KVStore(B, Hkv, d, n, device=dev, strict=False)
    # prompt = first n-1 tokens, uploaded page-chunk by page-chunk to bound host->device staging
    chunk = 1024
    for t0 in range(0, n - 1, chunk):
        t1 = min(n - 1, t0 + chunk)
        kt = torch.from_numpy(np.ascontiguousarray(K[:, t0:t1]).view(np.int16)).view(B, Hkv, t1 - t0, d)
        vt = torch.from_numpy(np.ascontiguousarray(V[:, t0:t1]).view(np.int16)).view(B, Hkv, t1 - t0, d)
        store.append(kt, vt)
    store.check()
    k_new = torch.from_numpy(np.ascontiguousarray(K[:, n - 1]).view(np.int16)).view(B, Hkv, d).to(dev)
    v_new = torch.from_numpy(np.ascontiguousarray(V[:, n - 1]).view(np.int16)).view(B, Hkv, d).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(Q).view(np.int16)).view(B, Hkv * g, d).to(dev)
    del K, V

    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    ws = store.workspace(g)
    ws.set_v_tiers(False)
    ws.step.q = q.data_ptr()
    cst = ctypes.byref(store.c_store)
    cfg_aligned = AD.make_cfg(g)
    cfg_control = AD.make_cfg(g, force_tier=16)
    gathered = torch.empty((world * H, d), dtype=torch.float32, device=dev) if world > 1 else None

    def append():
        store.lengths_dev.fill_(n - 1)  # every step attends over exactly n tokens
        _lib.check(L.akv_append(cst, k_new.data_ptr(), v_new.data_ptr(), 1, store.status_dev.data_ptr(), sp),
                   "akv_append")

    def step(cfg_c, ev=None):
        if ev is not None:
            ev[0].record(stream)
        append()
        if ev is None:
            _lib.check(L.akv_decode_step(cst, ctypes.byref(cfg_c), ctypes.byref(ws.step), n, sp), "decode")
        else:
            ev[1].record(stream)
            for i, fn in enumerate(("akv_qk", "akv_softmax_select", "akv_pv", "akv_combine")):
                _lib.check(getattr(L, fn)(cst, ctypes.byref(cfg_c), ctypes.byref(ws.step), n, sp), fn)
                ev[2 + i].record(stream)
        if gathered is not None:
            dist.all_gather_into_tensor(gathered, ws.o)

    def timed(cfg_c, steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step(cfg_c)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def breakdown(cfg_c, steps):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            step(cfg_c, evs[i])
        torch.cuda.synchronize()
        names = ["append", "qk", "select", "pv", "combine"]
        return {nm: float(np.mean([evs[i][k].elapsed_time(evs[i][k + 1]) for i in range(steps)]))
                for k, nm in enumerate(names)}

    for _ in range(args.warmup):
        step(cfg_aligned)
    for _ in range(args.warmup):
        step(cfg_control)
    # clocks sampled from the start of the timed region through the control and breakdown
    # runs that follow it (the K-step region alone is a few ms: one or two NVML samples)
    clocks = Clocks(local)
    ms = timed(cfg_aligned, args.steps)
    ms_ctl = timed(cfg_control, args.steps)
    bd = breakdown(cfg_aligned, args.steps)
    bd_ctl = breakdown(cfg_control, max(3, args.steps // 2))
    clk = clocks.stop()

    # ---- counters of the aligned step -> bytes, bit widths
    step(cfg_aligned)
    torch.cuda.synchronize()
    store.check()
    AD.check_status(store, g)
    cnt = ws.counters().cpu().numpy().astype(np.int64)
    ub = ws.unit_bytes().cpu().numpy().astype(np.int64)
    sel = ws.head_meta().cpu().numpy()[:, 0].astype(np.int64)
    kb, vb = int(ub[:, 0].sum()), int(ub[:, 1].sum())
    kv_fp16 = 4 * n * d * U
    k_bits = (8 * cnt[:, 0] + 12 * cnt[:, 1] + 16 * cnt[:, 2]).sum() / max(cnt[:, 0:3].sum(), 1)
    v_bits = (8 * cnt[:, 3] + 12 * cnt[:, 4] + 16 * cnt[:, 5]).sum() / max(cnt[:, 3:6].sum(), 1)
    npg = -(-n // 256)
    nblk = -(-npg // 4)
    side_qk = H * (2 * d + 4 * n + 8 * npg) + U * 4 * d
    side_sel = H * (8 * n + 8 * npg + 4 * (n // 32) + 16 * d)
    side_pv = H * (4 * n + 4 * (n // 32) + 4 * nblk * d + 8 * d) + U * 2 * n
    alg = {"qk": kb + side_qk, "select": side_sel + int(sel.sum()) * 2 * d, "pv": (vb - int(sel.sum()) * 2 * d) + side_pv}
    step_bytes = sum(alg.values()) + 2 * 2 * d * U  # + append planes
    hbm, pk_kind = peaks()
    dom = "qk" if bd["qk"] >= bd["pv"] else "pv"
    achieved = alg[dom] / (bd[dom] * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}:{dom}")
    except Exception:
        pass

    # ---- end-to-end through the public API with host buffers: attention_decode.DecodeGraph
    #      (CUDA graph of append + decode); per step H2D of q / k_new / v_new from pinned host
    #      memory, one graph replay, D2H of o (synchronous)
    e2e = None
    if not args.no_e2e:
        dg = AD.DecodeGraph(store, g, rewind_to=n - 1, zero_copy_out=world == 1).capture()
        dg.host_q.copy_(q.cpu())
        dg.host_k.copy_(k_new.cpu())
        dg.host_v.copy_(v_new.cpu())

        def e2e_step():
            dg.step()  # graph: H2D q/k/v (pinned) -> append -> decode -> D2H o (pinned), synchronised
            if world > 1:
                dist.all_gather_into_tensor(gathered, dg.o.reshape(-1, d))

        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        dg.check()
        e2e = {"value": world * B / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": dg.h2d_bytes, "d2h_bytes_per_step": dg.d2h_bytes,
               "api": "attention_decode.DecodeGraph.step (CUDA graph: append + qk + select + pv + combine; the "
                      "kernels read q / k_new / v_new from pinned host memory and combine stores o into pinned host "
                      "memory at N=1 (zero-copy PCIe transfers inside the step))"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_sample, 1)

    if rank == 0:
        t_s = ms * 1e-3
        line = {
            "metric": METRIC, "value": world * B / t_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16 planes, f32 accumulate",
            "data": "synthetic (SPEC generator: per-channel scale 2^U[-4,4], seed 7), random K/V/Q",
            "config": {"workload": args.config, "desc": desc, "batch_per_gpu": B, "kv_heads": Hkv, "q_per_kv": g,
                       "context": n, "head_dim": d, "parallelism": f"dp{world} (batch-sharded units)",
                       "l2": "KV cache 1 GiB/GPU > 126 MB L2 (no flush needed)",
                       "step": "append + qk + softmax/estimate + pv + combine" + (" + NCCL all-gather(o)" if world > 1 else "")},
            "effective_kv_gbs": world * kv_fp16 / t_s / 1e9,
            "bytes_read_fraction": (kb + vb) / kv_fp16,
            "k_bytes_fraction": kb / (kv_fp16 / 2), "v_bytes_fraction": vb / (kv_fp16 / 2),
            "avg_bits": {"k": float(k_bits), "v": float(v_bits),
                         "combined": float((k_bits * cnt[:, 0:3].sum() + v_bits * cnt[:, 3:6].sum()) / cnt[:, 0:6].sum())},
            "step_hbm_gbs": step_bytes / t_s / 1e9, "step_roofline_frac": step_bytes / t_s / 1e9 / hbm,
            "control_fp16": {"ms_per_step": ms_ctl, "tokens_per_s": world * B / (ms_ctl * 1e-3),
                             "note": "same kernels, force_tier=16, estimation off (paper control group)"},
            "speedup_vs_fp16_control": ms_ctl / ms,
            "kernel_ms": bd, "kernel_ms_control": bd_ctl,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_kind": pk_kind, "traffic": traffic,
                         "alg_bytes_per_launch": alg[dom]},
            "gpu_launches": 5 * args.steps,
            "e2e": e2e, "clocks": clk, "cpu_baseline": cpu,
            "gen_seconds": t_gen,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
