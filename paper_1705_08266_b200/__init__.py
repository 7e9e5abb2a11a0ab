"""B200-native 2-D discrete wavelet transform (arXiv 1705.08266 hot path).

Drop-in for the reference package ``liftfuse``'s transform API: wavelet and
scheme selectors stay in Python (:mod:`.lifting`, :mod:`.program`); every
pixel is computed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/b2dwt.h`` (:mod:`._native`).  There is no CPU fallback.
"""

from .engine import (
    PRECISION_DTYPES,
    Image2D,
    Pyramid,
    SubbandQuad,
    TileConfig,
    Transform,
    compile_scheme,
    deinterleave,
    dwt,
    extend,
    forward,
    idwt,
    interleave_quad,
    inverse,
    run_reference,
    run_tiled,
    run_without_barriers,
)
from .lifting import (
    CDF53,
    CDF97,
    EXACT,
    FLOAT,
    SCHEME_NAMES,
    WAVELETS,
    Laurent,
    LiftingPlan,
    Scheme,
    build_scheme,
    get_plan,
    invert_scheme,
    poly1,
)

__version__ = "0.1.0"
