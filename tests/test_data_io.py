"""data_io: AKV1 tensor files (acceptance 7 SPEC.md:589),
stat export, store snapshot/load (GPU)."""

import os

import numpy as np
import pytest

from paper_2409_16546_b200 import data_io as DIO

GOLD = os.path.join(os.path.dirname(__file__), "golden", "akv")


def test_golden_file_parses_bit_exact():
    w = DIO.load(os.path.join(GOLD, "golden_2x3.akv"))
    assert w.dtype == np.uint16 and w.shape == (2, 3)
    assert w.tolist() == [[0x0000, 0x8000, 0x0001], [0x3C00, 0x7BFF, 0xFC00]]
    # serialize reproduces the committed bytes exactly
    with open(os.path.join(GOLD, "golden_2x3.akv"), "rb") as f:
        assert DIO.serialize(w) == f.read()


def test_spec_example_file_size(tmp_path):
    # dims [2,3] -> 20-byte header + 12-byte payload = 32 bytes
    p = tmp_path / "t.akv"
    DIO.save(np.zeros((2, 3), np.float16), str(p))
    assert p.stat().st_size == 32


@pytest.mark.parametrize("name,err", [("bad_magic.akv", DIO.BadMagicError), ("truncated.akv", DIO.TruncatedError),
                                      ("bad_dtype.akv", DIO.DtypeError)])
def test_corrupt_fixtures_raise_distinct_errors(name, err):
    with pytest.raises(err) as ei:
        DIO.load(os.path.join(GOLD, name))
    assert isinstance(ei.value, DIO.AkvFormatError)
    codes = {DIO.BadMagicError.code, DIO.TruncatedError.code, DIO.DtypeError.code}
    assert len(codes) == 3
    if name == "bad_magic.akv":
        assert "bad magic" in str(ei.value)


def test_roundtrip_every_half_pattern(tmp_path):
    # every 16-bit pattern incl. subnormals, signed zeros, inf/nan patterns
    w = np.arange(65536, dtype=np.uint32).astype(np.uint16).reshape(256, 256)
    p = str(tmp_path / "all.akv")
    DIO.save(w, p)
    assert np.array_equal(DIO.load(p), w)
    # float16 input and 1-D / 3-D shapes
    rng = np.random.default_rng(0)
    for shp in [(7,), (2, 3, 5), (1, 1, 1, 4)]:
        a = rng.standard_normal(shp).astype(np.float16)
        DIO.save(a, p)
        assert np.array_equal(DIO.load(p), a.view(np.uint16))


def test_save_rejects_non_half(tmp_path):
    with pytest.raises(TypeError):
        DIO.save(np.zeros(3, np.float32), str(tmp_path / "x.akv"))


def test_stats_csv_json_consistent(tmp_path):
    rows = DIO.stat_rows([(256, 8.86, 9.7, 8.0), (4096, 8.9, 9.8, 8.01)],
                         [[0.5, 0.3, 0.1, 0.05, 0.03, 0.02], [0.6, 0.2, 0.1, 0.05, 0.03, 0.02]])
    c, j = str(tmp_path / "s.csv"), str(tmp_path / "s.json")
    DIO.export_stats(rows, c, "csv")
    DIO.export_stats(rows, j, "json")
    assert DIO.read_stats(c) == DIO.read_stats(j) == rows
    # empty sweep -> header-only CSV
    DIO.export_stats([], c, "csv")
    with open(c) as f:
        assert f.read().strip() == ",".join(DIO.CSV_FIELDS)
    # deterministic bytes
    DIO.export_stats(rows, c, "csv")
    b1 = open(c, "rb").read()
    DIO.export_stats(rows, c, "csv")
    assert open(c, "rb").read() == b1


@pytest.mark.gpu
def test_store_snapshot_roundtrip(tmp_path):
    import torch

    from paper_2409_16546_b200 import KVStore
    from paper_2409_16546_b200.synth import generate_batch

    B, H, n = 2, 2, 300
    K, V, _ = generate_batch(B, H, n, 128, 1, seed=7)
    st = KVStore(B, H, 128, 512)
    st.append(torch.from_numpy(K.view(np.int16)).view(B, H, n, 128), torch.from_numpy(V.view(np.int16)).view(B, H, n, 128))
    DIO.snapshot_store(st, str(tmp_path))
    assert np.array_equal(DIO.load(str(tmp_path / "K.akv")), K.reshape(B, H, n, 128))
    st2 = DIO.load_store(str(tmp_path), capacity=512)
    for which in ("k", "v"):
        for a, b in zip(st.export_planes(which), st2.export_planes(which)):
            assert np.array_equal(a, b)
    # corrupted sidecar is detected
    cm = DIO.load(str(tmp_path / "colmax.akv"))
    cm[0, 0, 0] ^= 1
    DIO.save(cm, str(tmp_path / "colmax.akv"))
    with pytest.raises(DIO.AkvFormatError):
        DIO.load_store(str(tmp_path), capacity=512)
