"""B200-native SVT / R3SVD / R4SVD hot path (arXiv 1704.05528).

The compute path is libsvt_b200.so (hand-written sm_100a CUDA + C++ host
engine behind the C ABI in include/svt_b200.h).  `api` is the Python mirror
of the reference's public API (proj/include/svt/*.hpp) over that ABI.  The
library is loaded lazily on first use; a missing library raises.
"""
from ._abi import (Backend, DomainError, InvalidArgument, IterationRecord, SketchParams, StopRule,  # noqa: F401
                   SvtConfig, SvtRuntimeError)


def __getattr__(name):
    if name == "api":
        import importlib
        return importlib.import_module(".api", __name__)
    from . import api as _api
    return getattr(_api, name)
