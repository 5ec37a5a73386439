"""`akv` command line (pkg/pyproject.toml:16 `akv = alignedkv.cli:main`).

    python -m paper_2409_16546_b200.cli gen --tokens 1024 --dim 128 --seed 7 --out data/
    python -m paper_2409_16546_b200.cli run --lengths 256,1024,4096 --seed 7 [--out stats.csv]
    python -m paper_2409_16546_b200.cli compare --seed 7 [--baseline-bits 13]

`gen` is host-only (numpy generator, AKV files).  `run` and `compare` run the
GPU decode path (there is no CPU fallback).  Exit codes:
0 ok, 2 usage, 3 I/O, 4 numeric degeneracy, 5 internal invariant failure.
AKV_THREADS is accepted and recorded; sweep points run one after
another on the GPU, so outputs never depend on it.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_NUMERIC, EXIT_INVARIANT = 0, 2, 3, 4, 5
TIERS = {"t8": 8, "t12": 12, "t16": 16}


class UsageError(Exception):
    pass


def _parser():
    ap = argparse.ArgumentParser(prog="akv", description="AlignedKV decode attention on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--dim", type=int, default=128)
        p.add_argument("--seed", type=int, default=7)
        p.add_argument("--margin-bits", type=int, default=0)
        p.add_argument("--no-zero-skip", action="store_true")
        p.add_argument("--m", type=int, default=5)
        p.add_argument("--k-sel", type=int, default=32)
        p.add_argument("--strategy", choices=("element", "row"), default="element")
        p.add_argument("--scale", type=float, default=4.0, help="channel scale law 2^U[-s, s] (SPEC.md:477)")
        p.add_argument("--heads", type=int, default=1, help="synthetic (batch x kv-head) units per length")
        p.add_argument("--input", help="directory with K.akv, V.akv, Q.akv (gen's output)")

    g = sub.add_parser("gen")
    g.add_argument("--tokens", type=int, required=True)
    g.add_argument("--dim", type=int, default=128)
    g.add_argument("--seed", type=int, default=7)
    g.add_argument("--scale", type=float, default=4.0)
    g.add_argument("--out", required=True)

    r = sub.add_parser("run")
    common(r)
    r.add_argument("--lengths", default="256,1024,4096")
    r.add_argument("--force-tier", choices=sorted(TIERS))
    r.add_argument("--out", default=None, help="stats file (.csv or .json); default: stdout summary only")
    r.add_argument("--format", choices=("csv", "json"), default=None)

    c = sub.add_parser("compare")
    common(c)
    c.add_argument("--tokens", type=int, default=1024)
    c.add_argument("--baseline-bits", type=int, default=13)
    c.add_argument("--out", default=None, help="JSON report")
    return ap


def _lengths(s):
    try:
        ls = [int(x) for x in s.split(",") if x.strip()]
    except ValueError:
        raise UsageError(f"bad --lengths {s!r}")
    if not ls or any(x < 1 for x in ls) or any(b <= a for a, b in zip(ls, ls[1:])):
        raise UsageError("--lengths must be positive and increasing")
    return ls


def _cfg(a):
    from paper_2409_16546_b200.align_core import AlignConfig

    try:
        return AlignConfig(margin_bits=a.margin_bits, zero_skip=not a.no_zero_skip)
    except ValueError as e:
        raise UsageError(str(e))


def _load_input(path):
    from paper_2409_16546_b200 import data_io as DIO

    files = [os.path.join(path, f) for f in ("K.akv", "V.akv", "Q.akv")]
    missing = [f for f in files if not os.path.exists(f)]
    if missing:
        raise FileNotFoundError("missing input files (expected K.akv, V.akv, Q.akv): " + ", ".join(missing))
    K, V, Q = (DIO.load(f) for f in files)
    if K.ndim == 2:
        K, V = K[None], V[None]
    if Q.ndim == 1:
        Q = Q[None, None]
    elif Q.ndim == 2:
        Q = Q[:, None] if K.shape[0] == Q.shape[0] and K.shape[0] > 1 else Q[None]
    return K, V, Q


def cmd_gen(a):
    from paper_2409_16546_b200 import data_io as DIO
    from paper_2409_16546_b200.synth import generate_unit

    if a.tokens < 1 or a.dim < 1:
        raise UsageError("--tokens and --dim must be >= 1")
    os.makedirs(a.out, exist_ok=True)
    K, V, Q = generate_unit(a.tokens, a.dim, 1, a.seed, 0, 0, -a.scale, a.scale)
    for name, arr in (("K.akv", K), ("V.akv", V), ("Q.akv", Q[0])):
        DIO.save(arr, os.path.join(a.out, name))
    print(f"wrote {a.out}/K.akv {a.out}/V.akv {a.out}/Q.akv ({a.tokens} x {a.dim}, seed {a.seed})")
    return EXIT_OK


def cmd_run(a):
    from paper_2409_16546_b200 import analysis as AN
    from paper_2409_16546_b200 import data_io as DIO

    if a.dim != 128:
        raise UsageError("this build computes d = 128 only")
    ls = _lengths(a.lengths)
    data = _load_input(a.input) if a.input else None
    if data is not None and ls[-1] > data[0].shape[1]:
        raise UsageError(f"--lengths exceed the input's {data[0].shape[1]} tokens")
    units = data[0].shape[0] if data is not None else a.heads
    curve = AN.bitwidth_sweep(ls, seed=a.seed, n_kv=units, cfg=_cfg(a), k_sel=a.k_sel, m=a.m,
                              strategy=a.strategy, force_tier=TIERS.get(a.force_tier), scale=a.scale,
                              with_hist=True, data=data)
    for p in curve.points:
        if not 8.0 <= p.avg_bits <= 16.0:
            print(f"invariant failed: avg bits {p.avg_bits} outside [8, 16]", file=sys.stderr)
            return EXIT_INVARIANT
    rows = DIO.stat_rows(curve.rows(), [p.sv_hist.fractions for p in curve.points])
    meta = {"strategy": a.strategy, "force_tier": a.force_tier, "seed": a.seed, "margin_bits": a.margin_bits,
            "akv_threads": os.environ.get("AKV_THREADS")}
    print(f"akv run  {json.dumps(meta)}")
    print(f"{'n':>7} {'avg':>7} {'K':>7} {'V':>7} {'bytes':>7}   SV zero-bucket")
    for p in curve.points:
        print(f"{p.context_length:>7} {p.avg_bits:7.3f} {p.avg_bits_k:7.3f} {p.avg_bits_v:7.3f} "
              f"{p.bytes_fraction:7.3f}   {100 * p.sv_hist.fractions[0]:.2f}%")
    print("paper-reported (PAPER.md:239, Llama-2-7B): avg bit width 16 -> ~12, decreasing with context")
    if a.out:
        fmt = a.format or ("json" if a.out.endswith(".json") else "csv")
        DIO.export_stats(rows, a.out, fmt)
    return EXIT_OK


def cmd_compare(a):
    from paper_2409_16546_b200 import analysis as AN

    if a.dim != 128:
        raise UsageError("this build computes d = 128 only")
    if not 8 <= a.baseline_bits <= 16:
        raise UsageError("--baseline-bits must be in [8, 16]")
    data = _load_input(a.input) if a.input else None
    n = data[0].shape[1] if data is not None else a.tokens
    units = data[0].shape[0] if data is not None else max(a.heads, 4)
    rep = AN.compare_report(n=n, seed=a.seed, n_kv=units, cfg=_cfg(a), baseline_bits=a.baseline_bits,
                            k_sel=a.k_sel, m=a.m, strategy=a.strategy, scale=a.scale, data=data)
    print(rep.table())
    if a.out:
        from paper_2409_16546_b200.data_io import _atomic_write

        js = {"baseline_bits": a.baseline_bits, "avg_bits": rep.avg_bits,
              "histograms": {f"{p}_{o}": h.fractions.tolist() for (p, o), h in rep.hist.items()}}
        _atomic_write(a.out, (json.dumps(js, indent=1, sort_keys=True) + "\n").encode())
    return EXIT_OK


def main(argv=None) -> int:
    from paper_2409_16546_b200.align_core import DegenerateInputError

    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return {"gen": cmd_gen, "run": cmd_run, "compare": cmd_compare}[a.cmd](a)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except DegenerateInputError as e:
        print(f"numeric error: {e}", file=sys.stderr)
        return EXIT_NUMERIC
    except (OSError, ValueError) as e:
        from paper_2409_16546_b200.data_io import AkvFormatError

        if isinstance(e, (OSError, AkvFormatError)):
            print(f"I/O error: {e}", file=sys.stderr)
            return EXIT_IO
        raise


if __name__ == "__main__":
    sys.exit(main())
