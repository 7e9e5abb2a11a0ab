"""CPU: image I/O against fixtures the real reference wrote and read
(tests/golden/make_imageio_golden.py), and the CLI's host-side behaviour
(argument errors -> exit 2, I/O errors -> exit 3) without a GPU."""

import os

import numpy as np
import pytest

from paper_1705_08266_b200 import Image2D
from paper_1705_08266_b200 import imageio as io
from paper_1705_08266_b200.cli import EXIT_IO, EXIT_USAGE, main

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "imageio")


@pytest.fixture(scope="module")
def arrays():
    return np.load(os.path.join(GOLD, "arrays.npz"))


@pytest.mark.parametrize("name", ["u8.pgm", "u16.pgm", "f32.raw", "f64.raw", "comments.pgm"])
def test_read_matches_reference(arrays, name):
    got = io.read_image(os.path.join(GOLD, name)).data
    want = arrays[name]
    assert got.dtype == want.dtype and got.shape == want.shape
    assert np.array_equal(got, want)


def test_writers_match_reference_bytes(arrays, tmp_path):
    src = Image2D(arrays["source_u8"])
    io.write_pgm(tmp_path / "u8.pgm", src)
    io.write_pgm(tmp_path / "u16.pgm", src, maxval=4095)
    for name in ("u8.pgm", "u16.pgm"):
        assert (tmp_path / name).read_bytes() == open(os.path.join(GOLD, name), "rb").read()
    for name in ("f32.raw", "f64.raw"):
        img = Image2D(arrays[name])
        io.write_image(tmp_path / name, img)
        assert (tmp_path / name).read_bytes() == open(os.path.join(GOLD, name), "rb").read()


def test_raw_pinned_reader(tmp_path, arrays):
    t = io.read_raw_pinned(os.path.join(GOLD, "f64.raw"))
    assert np.array_equal(t.numpy(), arrays["f64.raw"])
    big = Image2D(np.random.default_rng(1).random((300, 70)).astype(np.float32))
    io.write_raw(tmp_path / "big.raw", big)
    old = io._CHUNK
    io._CHUNK = 4096  # many chunks
    try:
        t = io.read_raw_pinned(tmp_path / "big.raw")
    finally:
        io._CHUNK = old
    assert np.array_equal(t.numpy(), big.data)
    with pytest.raises(ValueError, match="output buffer"):
        import torch

        io.read_raw_pinned(tmp_path / "big.raw", out=torch.empty((70, 300)))


def test_format_errors(tmp_path):
    (tmp_path / "x.bin").write_bytes(b"JUNKJUNK")
    with pytest.raises(ValueError, match="unrecognized image format"):
        io.read_image(tmp_path / "x.bin")
    (tmp_path / "t.raw").write_bytes(io.RAW_MAGIC + (4).to_bytes(4, "little") * 2 + (4).to_bytes(4, "little"))
    with pytest.raises(ValueError, match="truncated raw data"):
        io.read_raw(tmp_path / "t.raw")
    (tmp_path / "b.raw").write_bytes(io.RAW_MAGIC + (1).to_bytes(4, "little") * 2 + (2).to_bytes(4, "little"))
    with pytest.raises(ValueError, match="unsupported sample width 2"):
        io.read_raw(tmp_path / "b.raw")
    (tmp_path / "t.pgm").write_bytes(b"P5\n4 4\n255\n" + bytes(3))
    with pytest.raises(ValueError, match="truncated PGM data"):
        io.read_pgm(tmp_path / "t.pgm")
    with pytest.raises(ValueError, match="unsupported PGM maxval"):
        io.write_pgm(tmp_path / "m.pgm", Image2D(np.zeros((2, 2))), maxval=70000)


def test_cli_exit_codes_without_gpu(tmp_path, capsys):
    assert main(["transform", str(tmp_path / "missing.raw"), "--output", str(tmp_path / "o")]) == EXIT_IO
    assert main(["bench", "--threads", "0"]) == EXIT_USAGE
    # argument-type errors surface through argparse as exit status 2, as in the reference
    for argv in (["transform", "x", "--output", "o", "--tile", "4xq"], ["bench", "--sizes", "3,5"], ["bogus"]):
        with pytest.raises(SystemExit) as exc:
            main(argv)
        assert exc.value.code == EXIT_USAGE
