"""data_io: AKV tensor files, store snapshot/load, stat export.

AKV1 tensor file: magic "AKV1" | version u8 = 1 | dtype u8
(1 = half) | reserved u16 = 0 | ndim u32 LE | dims ndim x u32 LE | payload:
row-major fp16 words, little-endian.  parse(serialize(T)) == T bit-exactly;
bad magic, truncated payload and a non-half dtype raise distinct errors
(SPEC.md:494).  Writes are whole-file atomic: temp file + rename.

Store snapshot: the K and V caches of every (batch,
kv-head) unit as AKV files of fp16 words [B, Hkv, n, d], plus ColMax
[B, Hkv, d] and RowMax [B, Hkv, n] sidecars in the same format.  Loading goes
through the fused append kernel (akv_append), which recomputes the planes and
sidecars on device; the loaded sidecars are checked against them.

Stat export: CSV columns context_length, avg_bits,
avg_bits_k, avg_bits_v, bucket0..bucket5; JSON mirrors the same fields.
"""

from __future__ import annotations

import csv
import io
import json
import os
import struct
import tempfile
from typing import Iterable, Sequence

import numpy as np

MAGIC = b"AKV1"
VERSION = 1
DTYPE_HALF = 1
_HDR = struct.Struct("<4sBBHI")  # magic, version, dtype, reserved, ndim (12 bytes)


class AkvFormatError(ValueError):
    """Base of the AKV parse errors; `code` distinguishes them."""

    code = "format"


class BadMagicError(AkvFormatError):
    code = "bad_magic"


class TruncatedError(AkvFormatError):
    code = "truncated"


class DtypeError(AkvFormatError):
    code = "dtype"


class VersionError(AkvFormatError):
    code = "version"


def _as_words(tensor) -> np.ndarray:
    try:
        import torch

        if isinstance(tensor, torch.Tensor):
            t = tensor.detach().cpu().contiguous()
            if t.dtype in (torch.float16, torch.int16):
                return t.view(torch.int16).numpy().view(np.uint16)
            raise TypeError(f"AKV payload must be half words, got {t.dtype}")
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(tensor)
    if a.dtype == np.float16:
        return a.view(np.uint16)
    if a.dtype in (np.uint16, np.int16):
        return a.view(np.uint16)
    raise TypeError(f"AKV payload must be half words (float16 / uint16), got {a.dtype}")


def serialize(tensor) -> bytes:
    w = np.ascontiguousarray(_as_words(tensor))
    dims = w.shape
    hdr = _HDR.pack(MAGIC, VERSION, DTYPE_HALF, 0, len(dims)) + struct.pack(f"<{len(dims)}I", *dims)
    return hdr + w.astype("<u2", copy=False).tobytes()


def parse(buf: bytes) -> np.ndarray:
    """-> uint16 array of fp16 bit patterns with the file's dims."""
    if len(buf) < 4 or buf[:4] != MAGIC:
        raise BadMagicError(f"bad magic {bytes(buf[:4])!r} (expected {MAGIC!r})")
    if len(buf) < _HDR.size:
        raise TruncatedError(f"truncated header: {len(buf)} bytes")
    _, ver, dt, _res, ndim = _HDR.unpack_from(buf, 0)
    if ver != VERSION:
        raise VersionError(f"unsupported AKV version {ver}")
    if dt != DTYPE_HALF:
        raise DtypeError(f"dtype {dt} is not half (1)")
    off = _HDR.size + 4 * ndim
    if len(buf) < off:
        raise TruncatedError(f"truncated dims: need {off} header bytes, have {len(buf)}")
    dims = struct.unpack_from(f"<{ndim}I", buf, _HDR.size)
    count = int(np.prod(dims, dtype=np.int64)) if ndim else 1
    need = off + 2 * count
    if len(buf) < need:
        raise TruncatedError(f"truncated payload: need {need} bytes, have {len(buf)}")
    if len(buf) > need:
        raise AkvFormatError(f"trailing bytes: file has {len(buf)} bytes, format defines {need}")
    return np.frombuffer(buf, dtype="<u2", count=count, offset=off).astype(np.uint16).reshape(dims)


def _atomic_write(path: str, data: bytes) -> None:
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(prefix=".akv-", dir=d)
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(data)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def save(tensor, path: str) -> None:
    """SPEC.md:490-498 save(tensor, path), whole-file atomic."""
    _atomic_write(path, serialize(tensor))


def load(path: str) -> np.ndarray:
    """SPEC.md:490-498 load(path) -> uint16 fp16 words (view as float16 for values)."""
    with open(path, "rb") as f:
        return parse(f.read())


# ---------------------------------------------------------------------------
# store snapshot / load
# ---------------------------------------------------------------------------
SNAPSHOT_FILES = ("K.akv", "V.akv", "colmax.akv", "rowmax.akv")


def snapshot_store(store, directory: str) -> None:
    """Write the store's K/V caches + ColMax/RowMax sidecars (all units must hold equal lengths)."""
    lens = store.lengths.ravel()
    if len(set(int(x) for x in lens)) > 1:
        raise ValueError("snapshot needs equal lengths across units (ragged stores are not representable)")
    os.makedirs(directory, exist_ok=True)
    n = int(lens[0]) if len(lens) else 0
    B, H, d = store.batch, store.n_kv_heads, store.n_dims
    kw = store.words("k").reshape(B, H, n, d)
    vw = store.words("v").reshape(B, H, n, d)
    cm = store.colmax().cpu().numpy().astype(np.uint16).reshape(B, H, d)
    rm = store.rowmax().cpu().numpy().view(np.uint16).reshape(B, H, n)
    for name, arr in zip(SNAPSHOT_FILES, (kw, vw, cm, rm)):
        save(arr, os.path.join(directory, name))


def load_store(directory: str, capacity: int | None = None, device=None):
    """Rebuild a KVStore from a snapshot through the fused append kernel; the
    recomputed ColMax/RowMax must equal the sidecars (corruption check)."""
    import torch

    from paper_2409_16546_b200.kv_store import KVStore

    kw = load(os.path.join(directory, "K.akv"))
    vw = load(os.path.join(directory, "V.akv"))
    if kw.ndim != 4 or kw.shape != vw.shape:
        raise AkvFormatError(f"K/V snapshot dims mismatch: {kw.shape} vs {vw.shape}")
    B, H, n, d = kw.shape
    st = KVStore(B, H, d, capacity or max(n, 1), device=device)
    if n:
        st.append(torch.from_numpy(kw.view(np.int16)), torch.from_numpy(vw.view(np.int16)))
        st.check()
    cm = load(os.path.join(directory, "colmax.akv"))
    rm = load(os.path.join(directory, "rowmax.akv"))
    if not np.array_equal(st.colmax().cpu().numpy().astype(np.uint16).reshape(cm.shape), cm):
        raise AkvFormatError("ColMax sidecar does not match the K cache")
    if not np.array_equal(st.rowmax().cpu().numpy().view(np.uint16).reshape(rm.shape), rm):
        raise AkvFormatError("RowMax sidecar does not match the V cache")
    return st


# ---------------------------------------------------------------------------
# stat export
# ---------------------------------------------------------------------------
CSV_FIELDS = ("context_length", "avg_bits", "avg_bits_k", "avg_bits_v",
              "bucket0", "bucket1", "bucket2", "bucket3", "bucket4", "bucket5")


def stat_rows(curve: Iterable[Sequence[float]], histograms: Sequence[Sequence[float]] | None = None) -> list:
    """curve: (context_length, avg_bits, avg_k, avg_v) rows; histograms: 6 bucket fractions per row."""
    rows = []
    for i, pt in enumerate(curve):
        n, a, ak, av = pt
        h = list(histograms[i]) if histograms is not None else [0.0] * 6
        rows.append(dict(zip(CSV_FIELDS, [int(n), float(a), float(ak), float(av)] + [float(x) for x in h])))
    return rows


def export_stats(rows: list, path: str, fmt: str = "csv") -> None:
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=CSV_FIELDS, lineterminator="\n")
        w.writeheader()
        for r in rows:
            w.writerow({k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()})
        _atomic_write(path, buf.getvalue().encode())
    elif fmt == "json":
        _atomic_write(path, (json.dumps({"fields": list(CSV_FIELDS), "rows": rows}, indent=1) + "\n").encode())
    else:
        raise ValueError(f"unknown stats format {fmt!r} (csv|json)")


def read_stats(path: str) -> list:
    if path.endswith(".json"):
        with open(path) as f:
            return json.load(f)["rows"]
    with open(path, newline="") as f:
        out = []
        for r in csv.DictReader(f):
            out.append({k: (int(v) if k == "context_length" else float(v)) for k, v in r.items()})
        return out
