"""Generate the image-I/O fixtures with the REAL reference (liftfuse.imageio).

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_imageio_golden.py
Writes tests/golden/imageio/*.pgm|*.raw (files written by the reference's
writers, plus one hand-made PGM with header comments) and arrays.npz with the
arrays the reference's readers return for each file.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from liftfuse import imageio as ref  # noqa: E402
from liftfuse.engine import Image2D  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "imageio")
os.makedirs(OUT, exist_ok=True)
rng = np.random.default_rng(7)
img = Image2D(rng.random((5, 7)) * 1.2 - 0.1)  # some samples outside [0, 1] to exercise clipping
ref.write_pgm(os.path.join(OUT, "u8.pgm"), img)
ref.write_pgm(os.path.join(OUT, "u16.pgm"), img, maxval=4095)
ref.write_raw(os.path.join(OUT, "f32.raw"), Image2D(rng.random((6, 4)).astype(np.float32)))
ref.write_raw(os.path.join(OUT, "f64.raw"), Image2D(rng.random((3, 10))))
with open(os.path.join(OUT, "comments.pgm"), "wb") as fh:
    fh.write(b"P5\n# a comment\n4 # width\n2\n# maxval next\n200\n" + bytes(range(0, 200, 25)))
arrays = {"source_u8": img.data}
for name in ("u8.pgm", "u16.pgm", "f32.raw", "f64.raw", "comments.pgm"):
    arrays[name] = ref.read_image(os.path.join(OUT, name)).data
np.savez(os.path.join(OUT, "arrays.npz"), **arrays)
print("wrote", sorted(os.listdir(OUT)))
