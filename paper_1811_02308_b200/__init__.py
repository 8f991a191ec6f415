"""B200-native fast adaptive bilateral filter (Gavaskar & Chaudhury, arXiv 1811.02308).

A thin ctypes binding of the C-ABI library ``libfabf.so`` (include/fabf.h): the
same entry points, argument marshalling only.  Every step of the filter runs in
the library's sm_100a CUDA kernels; there is no CPU fallback -- importing works
anywhere, but every call raises if the library or a B200 is missing.  PyTorch is
used only for device memory and streams.
"""
from .fabf import (  # noqa: F401
    FabfError,
    Plan,
    bounds,
    filter,
    filter_diag,
    filter_events,
    filter_host,
    filter_interleaved,
    filter_mozerov,
    filter_gauss,
    filter_sharpen,
    sharpen_maps,
    SHARPEN_DEFAULTS,
    filter_texture,
    filter_texture_map,
    texture_maps,
    TEXTURE_DEFAULTS,
    filter_profile,
    lib,
    library_path,
    version,
    FLAG_LITERAL,
    FLAG_CLAMP,
    FLAG_DEBUG,
    FLAG_FUSED,
    CODE_IDENTITY,
    CODE_GUARD,
    CODE_SMALL_LAMBDA,
    CODE_FALLBACK,
    CODE_FAR_THETA,
    MAX_N,
)
