"""GPU: the command-line interface end to end (files in, files out) and the
raw-image device ingest, checked against the in-process API and the oracle."""

import csv

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1705_08266_b200 import CDF97, Image2D, build_scheme, compile_scheme  # noqa: E402
from paper_1705_08266_b200 import imageio as io  # noqa: E402
from paper_1705_08266_b200.cli import EXIT_OK, EXIT_VERIFY, main  # noqa: E402


def test_transform_inverse_round_trip_files(tmp_path):
    img = Image2D.random(130, 66, seed=3, precision="single")
    io.write_raw(tmp_path / "in.raw", img)
    args = ["--wavelet", "cdf97", "--scheme", "ns-lift-split", "--precision", "single"]
    assert main(["transform", str(tmp_path / "in.raw"), "--output", str(tmp_path / "q.raw"), *args]) == EXIT_OK
    bands = [io.read_raw(tmp_path / f"q.{b}.raw").data for b in ("ll", "hl", "lh", "hh")]
    want = oracle.forward(img.data, compile_scheme(build_scheme("non-separable-split", CDF97)))
    for g, w in zip(bands, want):
        assert np.array_equal(g, w)  # strict: bit-identical to the reference algorithm
    assert main(["inverse", str(tmp_path / "q.raw"), "--output", str(tmp_path / "rec.raw"), *args]) == EXIT_OK
    rec = io.read_raw(tmp_path / "rec.raw").data
    assert float(np.abs(rec - img.data).max()) <= 1e-3
    assert main(["transform", str(tmp_path / "in.raw"), "--output", str(tmp_path / "i.raw"), "--interleaved",
                 *args]) == EXIT_OK
    assert main(["inverse", str(tmp_path / "i.raw"), "--output", str(tmp_path / "rec2.raw"), "--interleaved",
                 *args]) == EXIT_OK
    assert np.array_equal(io.read_raw(tmp_path / "rec2.raw").data, rec)


def test_transform_levels(tmp_path):
    img = Image2D.random(256, 128, seed=1, precision="double")
    io.write_raw(tmp_path / "in.raw", img)
    assert main(["transform", str(tmp_path / "in.raw"), "--output", str(tmp_path / "p.raw"), "--levels", "3",
                 "--wavelet", "cdf97", "--scheme", "ns-lift"]) == EXIT_OK
    assert io.read_raw(tmp_path / "p.ll.raw").data.shape == (16, 32)
    assert io.read_raw(tmp_path / "p.l2.hh.raw").data.shape == (16, 32)


def test_verify_passes_and_catches_fault(capsys):
    assert main(["verify", "--images", "2", "--size", "32"]) == EXIT_OK
    out = capsys.readouterr().out
    assert "kernel invariance" in out and "impulse response" in out and "verification passed" in out
    assert main(["verify", "--wavelet", "cdf53", "--images", "1", "--size", "32", "--inject-fault"]) == EXIT_VERIFY


def test_bench_writes_reference_csv(tmp_path):
    path = tmp_path / "b.csv"
    assert main(["bench", "--sizes", "64,256", "--reps", "5", "--csv", str(path)]) == EXIT_OK
    rows = list(csv.reader(open(path)))
    # the reference's ten columns first (liftfuse/bench.py:22-33), then the GPU fields
    assert tuple(rows[0][:10]) == ("wavelet", "scheme", "width", "height", "precision", "threads", "tile", "reps",
                                   "median_seconds", "gbps")
    assert tuple(rows[0][10:]) == ("device", "ngpu", "levels", "gpix_per_s", "roofline_frac")
    assert len(rows) == 1 + 2 * 4
    assert all(float(r[9]) > 0 and float(r[13]) > 0 and float(r[14]) > 0 for r in rows[1:])
    assert all("B200" in r[10] or r[10] for r in rows[1:])


def test_read_raw_device(tmp_path):
    img = Image2D(np.random.default_rng(2).random((333, 96)).astype(np.float32))
    io.write_raw(tmp_path / "x.raw", img)
    dev = io.read_raw_device(tmp_path / "x.raw", rows_per_chunk=50)
    assert dev.is_cuda and torch.equal(dev.cpu(), torch.from_numpy(img.data))
