"""B200-native spatiotemporal Hawkes log-likelihood + gradient engine.

Python host mirror of the reference's likelihood interface
(/root/reference/proj/include/sthawkes/likelihood.hpp:17-31,
 types.hpp:39-137), running on the sm_100a engine behind the C ABI in
include/sthk.h (paper_2005_10123_b200/libsthk.so).

    events = EventSet(x, y, t, window_end)          # types.hpp:77-137
    params = Params(mu0=.., tauX=.., tauT=.., theta=.., omega=.., h=..)
    r = logLikelihood(events, params)              # likelihood.hpp:24-26
    r, g = logLikelihoodGradient(events, params)   # new: gradient, Params order

There is no CPU fallback: importing this package on a machine without the
built extension raises, and evaluating without a CUDA device fails loudly.
"""
from __future__ import annotations

from ._lib import (
    STHK_ERANGE,
    STHK_OK,
    STHK_EINVAL,
    STHK_ENOTLOADED,
    STHK_ECUDA,
    STHK_ENCCL,
    lib_path,
    load_library,
)
from .types import Params, EventSet, LikelihoodResult
from .engine import (
    Engine,
    EngineError,
    default_engine,
    logLikelihood,
    logLikelihoodBatch,
    logLikelihoodGradient,
    log_likelihood,
    log_likelihood_gradient,
)
from .simulate import SimWindow, generateBenchmarkCloud, simulateClusterProcess
from . import io
from . import partition
from .io import (
    EventFileSpec,
    readEvents,
    writeEvents,
    deduplicate,
    readChain,
    writeChain,
    loadRunConfig,
)
from .excitation import (
    ExcitationVector,
    PosteriorExcitation,
    excitationProbabilities,
    posteriorExcitation,
    thinIndices,
)

__all__ = [
    "STHK_OK", "STHK_EINVAL", "STHK_ENOTLOADED", "STHK_ECUDA", "STHK_ENCCL",
    "lib_path", "load_library",
    "Params", "EventSet", "LikelihoodResult",
    "Engine", "EngineError", "default_engine",
    "logLikelihood", "logLikelihoodBatch", "logLikelihoodGradient",
    "log_likelihood", "log_likelihood_gradient",
    "SimWindow", "generateBenchmarkCloud", "simulateClusterProcess",
    "ExcitationVector", "PosteriorExcitation", "excitationProbabilities",
    "posteriorExcitation", "thinIndices",
    "io", "EventFileSpec", "readEvents", "writeEvents", "deduplicate", "readChain",
    "writeChain", "loadRunConfig",
]
