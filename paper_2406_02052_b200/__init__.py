"""B200-native PETRA (arXiv 2406.02052) stage-tick library.

The compute lives in ``libpetra.so`` (CUDA, sm_100a, C ABI in include/petra.h);
this package is the ctypes binding (``petra``), the model / partition builders
(``models``) and the multi-rank transport (``dist``).  There is no CPU fallback.
"""
from . import _lib, models  # noqa: F401
from .petra import Pipeline, Schedule, Stage  # noqa: F401


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)
