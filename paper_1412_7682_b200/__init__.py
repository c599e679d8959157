"""B200-native CPA engine for AES-128 (arXiv:1412.7682), behind the C ABI of
include/cpa.h.  ``from paper_1412_7682_b200 import Engine`` for PyTorch callers;
the raw ABI lives in ``paper_1412_7682_b200._binding`` under the C names."""
from ._binding import *  # noqa: F401,F403  (cpa_* functions and constants)
from ._binding import CpaError, cpa_result  # noqa: F401


def __getattr__(name):
    if name == "Engine":  # torch import deferred until needed
        from .engine import Engine
        return Engine
    if name == "StreamingAttack":
        from .stream import StreamingAttack
        return StreamingAttack
    raise AttributeError(name)
