"""Aligned decode-attention benchmark (BASELINE.json metric, config 2 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c5]
                    [--scale S] [--shard auto|batch|kv_head] [--impl akv|reference]

One step = one decode step of one attention layer over the whole batch:
append the new token's K/V (akv_append) + aligned attention (akv_qk ->
akv_softmax_select -> akv_pv -> akv_combine), plus the NCCL all-gather of the
per-head outputs when N > 1.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun
environment re-executes itself under `torch.distributed.run` with N local
ranks (and fails loudly when the box has fewer than N devices).  Units are
seeded by their global (batch, kv-head) index, so the data do not depend on N.
  * c2 / c4 (`--shard batch`, weak scaling): every rank owns its own B batch
    rows; value = N*B / t_step.
  * c3 (`--shard kv_head`, strong scaling, BASELINE config 3): the global
    problem (B=32, 8 kv-heads) is fixed; rank r owns kv-heads [r*8/N, (r+1)*8/N)
    of every batch row; value = B / t_step.
  t_step = max over ranks of the CUDA-event time of K steps.  The per-head
  AccessCounter totals and plane bytes are all-reduced over ranks.
c5 is BASELINE config 5: a batch sweep 1..256 at 4k context (batch-sharded over
the ranks), one point per batch size with tokens/s, bytes-read fraction and
the fp16 control; `value` is the largest batch's tokens/s.

`e2e`   = the same metric through the public API (attention_decode.DecodeGraph:
          pinned host q/k/v in, o out, inside the timed region).
`parity` = a post-run validation sample: sampled units of the timed store
          re-run with the V-mask export and compared with the CPU oracle
          (oracle.parity.check_head) — checker only, after the timed region.
`--impl reference` times the CPU oracle (the reference algorithm restated,
kind "port") on this box's cores over whole steps of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
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
    "c5": (256, 32, 1, 4096, "batch sweep 1-256 at 4k context, Llama-2-7B shapes"),
}
SWEEP = (1, 2, 4, 8, 16, 32, 64, 128, 256)
METRIC = "aligned decode-attn tokens/s & effective KV GB/s vs HBM roofline; bytes-read saving"
D = 128


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def shard_scheme(args) -> str:
    if args.shard != "auto":
        return args.shard
    return "kv_head" if args.config == "c3" else "batch"


def config_dict(args, world: int) -> dict:
    """The workload description, identical in both arms (the driver compares them)."""
    B, Hkv, g, n, desc = CONFIGS[args.config]
    scheme = shard_scheme(args)
    strong = scheme == "kv_head"
    cfg = {"workload": args.config, "desc": desc, "batch_per_gpu": B if not strong else B,
           "global_batch": B if strong else B * world, "kv_heads": Hkv, "q_per_kv": g, "context": n,
           "head_dim": D, "channel_scale": f"2^U[-{args.scale:g},{args.scale:g}]",
           "parallelism": f"{'kv-head' if strong else 'batch'}-sharded units over {world} GPU(s)",
           "l2": "KV cache > 126 MB L2 per GPU (no flush needed)" if args.config not in ("c1",)
           else "KV cache (512 KiB) is L2-resident: latency-bound config",
           "step": "append + qk + softmax/estimate + pv + combine" + (" + NCCL all-gather(o)" if world > 1 else "")}
    if strong:
        cfg["kv_heads_per_gpu"] = Hkv // world if Hkv % world == 0 else None
    if args.config == "c5":
        cfg["sweep_batches"] = list(SWEEP)
        cfg["global_batch"] = SWEEP[-1]
    return cfg


def data_desc(args) -> str:
    return (f"synthetic (SPEC generator: per-channel scale 2^U[-{args.scale:g},{args.scale:g}], seed 7), "
            f"random K/V/Q")


# ---------------------------------------------------------------------------
# CPU baseline: the oracle over whole steps, all host cores (one process per core)
# ---------------------------------------------------------------------------
def _cpu_worker(units, n, g, Hkv, lo, hi, reps, barrier, q):
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import attention_decode as OA
    from oracle.kv_store import KVStore as OStore
    from paper_2409_16546_b200.synth import generate_unit

    stores = []
    for u in units:
        K, V, Q = generate_unit(n, D, g, 7, u // Hkv, u % Hkv, lo, hi)
        st = OStore(D)
        st.append_rows(K[: n - 1], V[: n - 1])
        stores.append((st, K[n - 1], V[n - 1], Q))
    barrier.wait()  # every worker's units are built
    for _ in range(reps):
        barrier.wait()  # step start
        for st, kn, vn, Q in stores:
            s2 = OStore(D)  # step = append the new token + aligned attention for every q-head
            s2.k, s2.v, s2.colmax, s2.rowmax = st.k, st.v, st.colmax, st.rowmax
            s2.append_token(kn, vn)
            for j in range(g):
                OA.decode_head(Q[j], s2)
        barrier.wait()  # step end
    q.put(0)


def cpu_steps(args, units, warmup: int, reps: int):
    """Wall-clock seconds of `reps` oracle steps over `units` (after `warmup` untimed ones),
    one worker process per host core, each owning a fixed slice of the units."""
    import multiprocessing as mp

    B, Hkv, g, n, _ = CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    workers = max(1, min(cores, len(units)))
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(workers + 1)
    q = ctx.Queue()
    total = warmup + reps
    procs = [ctx.Process(target=_cpu_worker, args=(units[i::workers], n, g, Hkv, -args.scale, args.scale, total,
                                                   barrier, q)) for i in range(workers)]
    for p in procs:
        p.start()
    barrier.wait()
    walls = []
    for i in range(total):
        barrier.wait()
        t0 = time.perf_counter()
        barrier.wait()
        if i >= warmup:
            walls.append(time.perf_counter() - t0)
    for _ in procs:
        q.get()
    for p in procs:
        p.join()
    return walls, workers


def cpu_sample_units(args):
    """Units of one CPU step: the whole workload where one step takes a few seconds on the
    host (c1, c2), else a stated contiguous sample (throughput is per unit)."""
    B, Hkv, g, n, _ = CONFIGS[args.config]
    U = B * Hkv
    limit = {"c1": 1, "c2": 512, "c3": 64, "c4": 48, "c5": 512}[args.config]
    return list(range(min(U, limit))), U


def cpu_baseline(args, warmup: int, reps: int):
    B, Hkv, g, n, _ = CONFIGS[args.config]
    units, U = cpu_sample_units(args)
    walls, workers = cpu_steps(args, units, warmup, reps)
    t = float(np.median(walls))
    rows = len(units) / Hkv  # batch rows processed per timed step
    whole = len(units) == U
    sample = (f"{'every one' if whole else f'{len(units)}'} of the {U} (batch, kv-head) units x {g} q-head(s), "
              f"n={n}, per step (append + aligned attention), {reps} timed step(s), median"
              + ("" if whole else f"; tokens/s = {rows:g} batch rows / step time (per-unit throughput)")
              + "; oracle = numpy float64 restatement of SPEC (oracle/)")
    return {"value": rows / t, "unit": "tokens/s", "cores": workers, "kind": "port", "sample": sample,
            "ms_per_step": t * 1e3, "walls_ms": [w * 1e3 for w in walls]}


def reference_main(args, world: int, rank: int):
    if rank != 0:
        return 0
    cb = cpu_baseline(args, args.warmup, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if shard_scheme(args) == "kv_head" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": data_desc(args), "config": config_dict(args, world),
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
# launching
# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> int | None:
    """--gpus N outside torchrun: re-execute under torch.distributed.run with N ranks."""
    if os.environ.get("WORLD_SIZE") is not None or args.gpus <= 1:
        return None
    if args.impl == "akv":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus} needs {args.gpus} devices; this box has {have}\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="akv", choices=["akv", "reference"])
    ap.add_argument("--scale", type=float, default=4.0, help="channel scales 2^U[-S,S] (paper-like: 0.5)")
    ap.add_argument("--shard", default="auto", choices=["auto", "batch", "kv_head"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-validate", action="store_true")
    ap.add_argument("--validate-units", type=int, default=2, help="units per rank in the post-run parity sample")
    ap.add_argument("--cpu-reps", type=int, default=2)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    return args


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if args.impl == "reference":
        return reference_main(args, world, rank)
    return gpu_main(args, world, rank)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class Rig:
    """One rank's store, inputs and launch closures for a (sub)set of units."""

    def __init__(self, store, q, k_new, v_new, g, n, world, dist, dev):
        import ctypes

        import torch

        from paper_2409_16546_b200 import _lib
        from paper_2409_16546_b200 import attention_decode as AD

        self.store, self.q, self.k_new, self.v_new, self.g, self.n = store, q, k_new, v_new, g, n
        self.world, self.dist, self.dev = world, dist, dev
        self.L = _lib.lib()
        self._lib = _lib
        self.stream = torch.cuda.current_stream(dev)
        self.sp = self.stream.cuda_stream
        self.ws = store.workspace(g)
        self.ws.set_v_tiers(False)
        self.ws.step.q = q.data_ptr()
        self.cst = ctypes.byref(store.c_store)
        self.cfg_aligned = AD.make_cfg(g)
        self.cfg_control = AD.make_cfg(g, force_tier=16)
        self.gathered = (torch.empty((world * self.ws.o.shape[0], D), dtype=torch.float32, device=dev)
                         if world > 1 else None)
        self.ctypes = ctypes

    def append(self):
        # the new token goes to position n-1 of every unit (akv_append_at: truncate + append in
        # one launch), so every step attends over exactly n tokens
        self._lib.check(self.L.akv_append_at(self.cst, self.k_new.data_ptr(), self.v_new.data_ptr(), self.n - 1,
                                             self.store.status_dev.data_ptr(), self.sp), "akv_append_at")

    def step(self, cfg_c, ev=None):
        by = self.ctypes.byref
        if ev is not None:
            ev[0].record(self.stream)
        self.append()
        if ev is None:
            self._lib.check(self.L.akv_decode_step(self.cst, by(cfg_c), by(self.ws.step), self.n, self.sp), "decode")
        else:
            ev[1].record(self.stream)
            for i, fn in enumerate(("akv_qk", "akv_softmax_select", "akv_pv", "akv_combine")):
                self._lib.check(getattr(self.L, fn)(self.cst, by(cfg_c), by(self.ws.step), self.n, self.sp), fn)
                ev[2 + i].record(self.stream)
        if self.gathered is not None:
            self.dist.all_gather_into_tensor(self.gathered, self.ws.o)

    def timed(self, cfg_c, steps):
        import torch

        torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for _ in range(steps):
            self.step(cfg_c)
        e1.record(self.stream)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / steps, self.world, self.dist, self.dev)

    def breakdown(self, cfg_c, steps):
        import torch

        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(steps)]
        torch.cuda.synchronize()
        for i in range(steps):
            self.step(cfg_c, evs[i])
        torch.cuda.synchronize()
        names = ["append", "qk", "select", "pv", "combine"]
        return {nm: float(np.mean([evs[i][k].elapsed_time(evs[i][k + 1]) for i in range(steps)]))
                for k, nm in enumerate(names)}

    def counters(self):
        """(counters [H,8], unit_bytes [U,4], sel counts [H]) of the last step, summed over ranks."""
        import torch

        from paper_2409_16546_b200.shard import gather_counters

        cnt = self.ws.counters().sum(0)
        ub = self.ws.unit_bytes().sum(0)
        sel = self.ws.head_meta()[:, 0].to(torch.int64).sum().view(1)
        tot = gather_counters(torch.cat([cnt, ub, sel]))
        tot = tot.cpu().numpy().astype(np.int64)
        return tot[:8], tot[8:12], int(tot[12])


def max_over_ranks(x, world, dist, dev):
    if world == 1:
        return x
    import torch

    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(vals, world, dist, dev):
    if world == 1:
        return vals
    import torch

    t = torch.tensor(vals, device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().tolist()


def build_rig(args, world, rank, dist, dev, units_global=None, B_local=None, Hkv_local=None):
    """Generate this rank's units (global seeds), fill a store with the first n-1 tokens,
    keep token n-1 as the step's new K/V.  Returns (rig, sample dict for validation, gen s)."""
    import torch

    from paper_2409_16546_b200 import KVStore
    from paper_2409_16546_b200.synth import fill_store, generate_batch

    B, Hkv, g, n, _ = CONFIGS[args.config]
    t_gen = time.time()
    workers = len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    K, V, Q = generate_batch(B_local, Hkv, n, D, g, 7, -args.scale, args.scale, units=units_global,
                             workers=max(1, workers))
    # generate_batch seeds unit u as (u // Hkv, u % Hkv) with Hkv the global kv-head count
    t_gen = time.time() - t_gen
    store = KVStore(B_local, Hkv_local, D, n, device=dev, strict=False)
    fill_store(store, K, V, n - 1)
    k_new = torch.from_numpy(np.ascontiguousarray(K[:, n - 1]).view(np.int16)).view(B_local, Hkv_local, D).to(dev)
    v_new = torch.from_numpy(np.ascontiguousarray(V[:, n - 1]).view(np.int16)).view(B_local, Hkv_local, D).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(Q).view(np.int16)).view(B_local, Hkv_local * g, D).to(dev)
    U = len(units_global)
    k = max(0, min(args.validate_units, U))
    pick = sorted({int(x) for x in np.linspace(0, U - 1, k)}) if k else []  # spread over the rank's units
    sample = {i: (units_global[i], K[i].copy(), V[i].copy(), Q[i].copy()) for i in pick}
    del K, V
    return Rig(store, q, k_new, v_new, g, n, world, dist, dev), sample, t_gen


def validate(rig, sample, args, world, dist, dev):
    """Post-run parity sample: re-run the step with the V-mask export, compare the sampled
    units with the CPU oracle (oracle.parity.check_head; checker only)."""
    import torch

    from oracle import attention_decode as OA
    from oracle.kv_store import KVStore as OStore
    from oracle.parity import check_head
    from paper_2409_16546_b200 import attention_decode as AD

    st = rig.store
    rig.append()
    torch.cuda.synchronize()
    st._host_len[:] = rig.n
    r = AD.decode_step(rig.q, st, return_scores=True, export_v_tiers=True)
    g, Hl = rig.g, st.n_kv_heads
    checked = mism = edges = 0
    fails = []
    for i, (ug, K, V, Q) in sample.items():
        b, h = divmod(i, Hl)
        ost = OStore(D)
        ost.append_rows(K, V)
        for j in range(g):
            hq = h * g + j
            ref = OA.decode_head(Q[j], ost)
            fail, edge = check_head(ref, k_tiers=r.k_tiers[b, hq].cpu().numpy(), o=r.o[b, hq].cpu().numpy(),
                                    counters=r.counters[b, hq].cpu().numpy(), sel=r.selection(b, hq),
                                    v_tiers=r.v_tiers[b, hq].cpu().numpy(), s=r.scores[b, hq].cpu().numpy(),
                                    p=r.probs[b, hq].cpu().numpy(), targets=r.targets[b, hq].cpu().numpy(),
                                    v_head=V >> 8)
            checked += 1
            mism += bool(fail)
            edges += edge
            if fail:
                fails.append([int(ug), j, fail])
    tot = sum_over_ranks([len(sample), checked, mism, edges], world, dist, dev)
    out = {"units_checked": int(tot[0]), "heads_checked": int(tot[1]), "mismatches": int(tot[2]),
           "knife_edges": int(tot[3]),
           "what": "K/V tier masks (bit-exact, with the D11 injection check), selection, AccessCounter, scores "
                   "and o within 1e-3, against the CPU oracle on sampled units of the timed store"}
    if fails:
        out["failures"] = fails[:8]
    return out


def gpu_main(args, world, rank):
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.device_count() <= local:
        sys.stderr.write(f"bench.py: rank {rank} needs device {local}; this box has {torch.cuda.device_count()}\n")
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        if rank == 0:
            sys.stderr.write(f"NCCL process group: nranks={dist.get_world_size()} (all-reduce check "
                             f"{int(t.item())})\n")
    if args.config == "c5":
        return sweep_main(args, world, rank, dist, dev)

    from paper_2409_16546_b200 import attention_decode as AD
    from paper_2409_16546_b200.shard import shard_for

    B, Hkv, g, n, desc = CONFIGS[args.config]
    scheme = shard_scheme(args)
    if scheme == "kv_head":  # strong scaling: the global (B, Hkv) problem split by kv-head
        sh = shard_for(B, Hkv, world, rank, "kv_head")
    else:  # weak scaling: the job's batch is world*B rows; this rank owns rows [rank*B, (rank+1)*B)
        sh = shard_for(world * B, Hkv, world, rank, "batch")
    units = sh.units(Hkv)
    rig, sample, t_gen = build_rig(args, world, rank, dist, dev, units, sh.batch, sh.kv_heads)
    U_loc, H_loc = sh.batch * sh.kv_heads, sh.batch * sh.kv_heads * g
    U_all = U_loc * world
    rows = B if scheme == "kv_head" else world * B  # batch rows decoded per step by the whole job

    for _ in range(args.warmup):
        rig.step(rig.cfg_aligned)
    for _ in range(args.warmup):
        rig.step(rig.cfg_control)
    # clocks sampled from the start of the timed region through the control and breakdown
    # runs that follow it (the K-step region alone is a few ms: one or two NVML samples)
    clocks = Clocks(local)
    ms = rig.timed(rig.cfg_aligned, args.steps)
    ms_ctl = rig.timed(rig.cfg_control, args.steps)
    bd = rig.breakdown(rig.cfg_aligned, args.steps)
    bd_ctl = rig.breakdown(rig.cfg_control, max(3, args.steps // 2))
    clk = clocks.stop()

    # ---- counters of the aligned step (summed over ranks) -> bytes, bit widths
    rig.step(rig.cfg_aligned)
    torch.cuda.synchronize()
    rig.store.check()
    AD.check_status(rig.store, g)
    cnt, ub, nsel = rig.counters()
    kb, vb = int(ub[0]), int(ub[1])
    kv_fp16 = 4 * n * D * U_all
    k_bits = (8 * cnt[0] + 12 * cnt[1] + 16 * cnt[2]) / max(cnt[0:3].sum(), 1)
    v_bits = (8 * cnt[3] + 12 * cnt[4] + 16 * cnt[5]) / max(cnt[3:6].sum(), 1)
    npg = -(-n // 256)
    nblk = -(-npg // 4)
    H_all = H_loc * world
    side_qk = H_all * (2 * D + 4 * n + 8 * npg) + U_all * 4 * D
    side_sel = H_all * (8 * n + 8 * npg + 4 * (n // 32) + 16 * D)
    side_pv = H_all * (4 * n + 4 * (n // 32) + 4 * nblk * D + 8 * D) + U_all * 2 * n
    alg = {"qk": kb + side_qk, "select": side_sel + nsel * 2 * D, "pv": (vb - nsel * 2 * D) + side_pv}
    step_bytes = sum(alg.values()) + 2 * 2 * D * U_all  # + append planes
    hbm, pk_kind = peaks()
    dom = "qk" if bd["qk"] >= bd["pv"] else "pv"
    achieved = alg[dom] / world / (bd[dom] * 1e-3) / 1e9  # one rank's kernel: its share of the bytes
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = f"{args.config}:{dom}" + ("" if args.scale == 4.0 else f":s{args.scale:g}")
        traffic = tr.get(key) if world == 1 else None
    except Exception:
        pass

    # ---- end-to-end through the public API with host buffers: attention_decode.DecodeGraph
    e2e = None
    if not args.no_e2e:
        dg = AD.DecodeGraph(rig.store, g, rewind_to=n - 1, zero_copy_out=world == 1).capture()
        dg.host_q.copy_(rig.q.cpu())
        dg.host_k.copy_(rig.k_new.cpu())
        dg.host_v.copy_(rig.v_new.cpu())

        def e2e_step():
            dg.step()  # graph: H2D q/k/v (pinned) -> append -> decode -> D2H o (pinned), synchronised
            if world > 1:
                dist.all_gather_into_tensor(rig.gathered, dg.o.reshape(-1, D))

        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps, world, dist, dev)
        dg.check()
        e2e = {"value": rows / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": dg.h2d_bytes * world, "d2h_bytes_per_step": dg.d2h_bytes * world,
               "api": "attention_decode.DecodeGraph.step (CUDA graph: append + qk + select + pv + combine; the "
                      "kernels read q / k_new / v_new from pinned host memory"
                      + (" and combine stores o into pinned host memory (zero-copy PCIe transfers inside the step))"
                         if world == 1 else "; D2H of o, then the NCCL all-gather of o)")}

    parity = None
    if not args.no_validate:
        parity = validate(rig, sample, args, world, dist, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args, 0, max(1, args.cpu_reps))
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "ms_per_step")}

    if rank == 0:
        t_s = ms * 1e-3
        line = {
            "metric": METRIC, "value": rows / t_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if scheme == "kv_head" else "weak", "vs_baseline": None,
            "dtype": "f16 planes, f32 accumulate", "data": data_desc(args), "config": config_dict(args, world),
            "effective_kv_gbs": kv_fp16 / t_s / 1e9,
            "bytes_read_fraction": (kb + vb) / kv_fp16,
            "k_bytes_fraction": kb / (kv_fp16 / 2), "v_bytes_fraction": vb / (kv_fp16 / 2),
            "avg_bits": {"k": float(k_bits), "v": float(v_bits),
                         "combined": float((k_bits * cnt[0:3].sum() + v_bits * cnt[3:6].sum()) / cnt[0:6].sum())},
            "step_hbm_gbs": step_bytes / world / t_s / 1e9,
            "step_roofline_frac": step_bytes / world / t_s / 1e9 / hbm,
            "control_fp16": {"ms_per_step": ms_ctl, "tokens_per_s": rows / (ms_ctl * 1e-3),
                             "note": "same kernels, force_tier=16, estimation off (paper control group)"},
            "speedup_vs_fp16_control": ms_ctl / ms,
            "kernel_ms": bd, "kernel_ms_control": bd_ctl,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_kind": pk_kind, "traffic": traffic,
                         "alg_bytes_per_launch": alg[dom] // world},
            "gpu_launches": 5 * args.steps,
            "parity": parity,
            "e2e": e2e, "clocks": clk, "cpu_baseline": cpu,
            "gen_seconds": t_gen,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# config 5: batch sweep
# ---------------------------------------------------------------------------
def sweep_main(args, world, rank, dist, dev):
    """BASELINE config 5: B in 1..256 at 4k context, batch-sharded over the ranks.  The
    store holds this rank's share of the largest batch; 512 generated units (the c2 batch)
    are tiled over it by device page copies (unit u carries the data of global unit
    u mod 512), and each point runs on a prefix view of the store."""
    import torch

    from paper_2409_16546_b200 import KVStore
    from paper_2409_16546_b200.synth import fill_store, generate_batch

    Bmax, Hkv, g, n, _ = CONFIGS["c5"]
    base_rows = 16
    workers = max(1, len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    K, V, Q = generate_batch(base_rows, Hkv, n, D, g, 7, -args.scale, args.scale, workers=workers)
    base = KVStore(base_rows, Hkv, D, n, device=dev, strict=False)
    fill_store(base, K, V, n - 1)
    kn0 = torch.from_numpy(np.ascontiguousarray(K[:, n - 1]).view(np.int16)).view(base_rows, Hkv, D).to(dev)
    vn0 = torch.from_numpy(np.ascontiguousarray(V[:, n - 1]).view(np.int16)).view(base_rows, Hkv, D).to(dev)
    q0 = torch.from_numpy(np.ascontiguousarray(Q).view(np.int16)).view(base_rows, Hkv * g, D).to(dev)
    del K, V
    per_rank_max = -(-Bmax // world)
    big = KVStore(per_rank_max, Hkv, D, n, device=dev, strict=False)
    mp_ = base.max_pages
    rows0 = rank * per_rank_max
    src_rows = [(rows0 + b) % base_rows for b in range(per_rank_max)]
    idx = torch.tensor(src_rows, device=dev)
    for b, sb in enumerate(src_rows):  # row by row: no 16 GiB gather temporary
        big.k_pool.view(per_rank_max, Hkv, mp_, -1)[b].copy_(base.k_pool.view(base_rows, Hkv, mp_, -1)[sb])
        big.v_pool.view(per_rank_max, Hkv, mp_, -1)[b].copy_(base.v_pool.view(base_rows, Hkv, mp_, -1)[sb])
    big.colmax_dev.view(per_rank_max, Hkv, D).copy_(base.colmax_dev.view(base_rows, Hkv, D)[idx])
    big.rowmax_dev.view(per_rank_max, Hkv, -1).copy_(base.rowmax_dev.view(base_rows, Hkv, -1)[idx])
    big.lengths_dev.fill_(n - 1)
    big._host_len[:] = n - 1
    k_new, v_new, q = kn0[idx].contiguous(), vn0[idx].contiguous(), q0[idx].contiguous()
    del base
    torch.cuda.synchronize()

    hbm, _ = peaks()
    points = []
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", "0")))
    for Bg in SWEEP:
        # this rank's rows of the global batch Bg
        lo, hi = rank * Bg // world, (rank + 1) * Bg // world
        Bl = hi - lo
        if Bl > 0:
            view = big.batch_prefix(Bl)
            rig = Rig(view, q[:Bl].contiguous(), k_new[:Bl].contiguous(), v_new[:Bl].contiguous(), g, n, 1, dist, dev)
            for _ in range(args.warmup):
                rig.step(rig.cfg_aligned)
            ms_l = rig.timed(rig.cfg_aligned, args.steps)
            ms_c = rig.timed(rig.cfg_control, args.steps)
            rig.step(rig.cfg_aligned)
            torch.cuda.synchronize()
            ub = rig.ws.unit_bytes().sum(0).cpu().numpy()
            kvb = float(ub[0] + ub[1])
        else:
            ms_l = ms_c = 0.0
            kvb = 0.0
        if world > 1:
            dist.barrier()
        ms = max_over_ranks(ms_l, world, dist, dev)
        msc = max_over_ranks(ms_c, world, dist, dev)
        kvb = sum_over_ranks([kvb], world, dist, dev)[0]
        fp16 = 4.0 * n * D * Bg * Hkv
        points.append({"batch": Bg, "ms_per_step": ms, "tokens_per_s": Bg / (ms * 1e-3),
                       "bytes_read_fraction": kvb / fp16, "effective_kv_gbs": fp16 / (ms * 1e-3) / 1e9,
                       "control_ms_per_step": msc, "speedup_vs_fp16_control": msc / ms,
                       "kv_roofline_frac": kvb / world / (ms * 1e-3) / 1e9 / hbm})
    clk = clocks.stop()
    if rank == 0:
        last = points[-1]
        line = {"metric": METRIC, "value": last["tokens_per_s"], "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": last["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f16 planes, f32 accumulate",
                "data": data_desc(args) + "; 512 generated units tiled over the batch (unit u = unit u mod 512)",
                "config": dict(config_dict(args, world), step="append + qk + softmax/estimate + pv + combine "
                                                               "per point (no all-gather: a point's ranks hold "
                                                               "unequal row counts)"),
                "sweep": points, "gpu_launches": 5 * args.steps,
                "e2e": None, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
