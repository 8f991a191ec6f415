"""CPU oracle for the fast adaptive bilateral filter (arXiv 1811.02308).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product path (``paper_1811_02308_b200``) never imports it and
shares no code with it; see ``fabf_oracle.c`` for what each function computes and
which passage of the paper it follows.
"""
from .oracle import (  # noqa: F401
    build,
    bounds,
    brute,
    fast,
    fast_window,
    fit,
    hilbert_inverse,
    integrals,
    literal,
    mozerov,
    sharpen_maps,
    SHARPEN_DEFAULTS,
    texture_maps,
    texture_pipeline,
    TEXTURE_DEFAULTS,
    stretch,
    CODE_IDENTITY,
    CODE_GUARD,
    CODE_QUAD,
    KAPPA_MAX,
)
