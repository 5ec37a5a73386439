"""`akv` CLI: gen on CPU; run / compare on the GPU."""

import os

import numpy as np
import pytest

from paper_2409_16546_b200 import data_io as DIO
from paper_2409_16546_b200.cli import EXIT_IO, EXIT_OK, EXIT_USAGE, main


def test_gen_writes_three_deterministic_files(tmp_path):
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    assert main(["gen", "--tokens", "64", "--dim", "128", "--seed", "7", "--out", a]) == EXIT_OK
    assert main(["gen", "--tokens", "64", "--dim", "128", "--seed", "7", "--out", b]) == EXIT_OK
    assert sorted(os.listdir(a)) == ["K.akv", "Q.akv", "V.akv"]
    for f in ("K.akv", "V.akv", "Q.akv"):
        assert open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read()
    assert DIO.load(os.path.join(a, "K.akv")).shape == (64, 128)
    assert DIO.load(os.path.join(a, "Q.akv")).shape == (128,)


def test_usage_and_io_errors(tmp_path):
    assert main(["gen", "--tokens", "0", "--out", str(tmp_path)]) == EXIT_USAGE
    assert main(["frobnicate"]) == EXIT_USAGE
    assert main(["run", "--lengths", "512,256"]) == EXIT_USAGE
    assert main(["run", "--bogus-flag"]) == EXIT_USAGE
    assert main(["run", "--input", str(tmp_path / "nope"), "--lengths", "16"]) == EXIT_IO
    bad = tmp_path / "bad"
    bad.mkdir()
    for f in ("K.akv", "V.akv", "Q.akv"):
        (bad / f).write_bytes(b"AKV2xxxx")
    assert main(["run", "--input", str(bad), "--lengths", "16"]) == EXIT_IO


@pytest.mark.gpu
def test_run_and_compare(tmp_path, capsys):
    out = str(tmp_path / "s.csv")
    assert main(["run", "--lengths", "256,1024", "--seed", "7", "--heads", "2", "--out", out]) == EXIT_OK
    rows = DIO.read_stats(out)
    assert [r["context_length"] for r in rows] == [256, 1024]
    b1 = open(out, "rb").read()
    assert main(["run", "--lengths", "256,1024", "--seed", "7", "--heads", "2", "--out", out]) == EXIT_OK
    assert open(out, "rb").read() == b1  # acceptance 8 (determinism)
    assert main(["run", "--lengths", "256", "--force-tier", "t16", "--out", out]) == EXIT_OK
    assert DIO.read_stats(out)[0]["avg_bits"] == 16.0
    # input files from gen
    d = str(tmp_path / "data")
    assert main(["gen", "--tokens", "300", "--out", d]) == EXIT_OK
    assert main(["run", "--input", d, "--lengths", "100,300", "--strategy", "row"]) == EXIT_OK
    assert "row" in capsys.readouterr().out
    js = str(tmp_path / "c.json")
    assert main(["compare", "--seed", "7", "--tokens", "512", "--out", js]) == EXIT_OK
    import json

    rep = json.load(open(js))
    assert rep["histograms"]["aligned_qk"][0] > rep["histograms"]["trunc_qk"][0]
    assert main(["compare", "--baseline-bits", "16", "--tokens", "256", "--out", js]) == EXIT_OK
    assert json.load(open(js))["histograms"]["trunc_sv"][0] == 1.0
