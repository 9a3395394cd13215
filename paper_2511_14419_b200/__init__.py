"""B200-native (sm_100a) RoI-extraction stage of FlowRoI (arxiv 2511.14419).

Drop-in for the reference's ``flowroi::extract_roi`` stage
(/root/reference/proj/include/flowroi/roi.hpp:309-364): hand-written CUDA kernels behind the C ABI
in include/froi/froi.h (libfroi.so), with this package as the Python host mirror of the
reference's operator API.  ``params`` is importable without the CUDA library; everything else
loads libfroi.so and fails loudly if it is missing.
"""
from .params import (DataError, DenoiseParams, ExtractInfo, ExtractParams, FlowParams,  # noqa: F401
                     InternalError, RoiParams, Shift, StageTimes, UsageError)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the package must not require the CUDA library (CPU-only test hosts)
    if name in ("flowroi", "_native", "synth"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
