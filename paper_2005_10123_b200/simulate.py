"""Seeded synthetic inputs (sthk_sim.h): bit-identical restatements of the
reference's generateBenchmarkCloud / simulateClusterProcess
(proj/src/simulate.cpp:10-95) with its mt19937_64 Rng (rng.hpp:27-96)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .types import EventSet, Params


@dataclass
class SimWindow:
    """simulate.hpp:13-26."""
    xmin: float = 0.0
    xmax: float = 10.0
    ymin: float = 0.0
    ymax: float = 10.0
    tEnd: float = 100.0

    def as_array(self) -> np.ndarray:
        return np.array([self.xmin, self.xmax, self.ymin, self.ymax, self.tEnd], np.float64)


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def generateBenchmarkCloud(n: int, window: SimWindow, seed: int) -> EventSet:
    lib = _lib.load_library()
    x, y, t = np.zeros(n), np.zeros(n), np.zeros(n)
    we = ctypes.c_double()
    w = window.as_array()
    if lib.sthk_sim_cloud(n, _d(w), seed, _d(x), _d(y), _d(t), ctypes.byref(we)) != 0:
        raise ValueError("generateBenchmarkCloud: invalid arguments")
    return EventSet(x, y, t, we.value)


def simulateClusterProcess(params: Params, window: SimWindow, rate: float, seed: int,
                           keep: int | None = None):
    """Returns (EventSet, parentIndex). With `keep`, only the first `keep`
    events in time order are returned and windowEnd defaults to their last
    time (the SURVEY's C2 recipe: first 85,000 of the simulated set)."""
    lib = _lib.load_library()
    p = params.as_array()
    w = window.as_array()
    cnt = ctypes.c_int64()
    rc = lib.sthk_sim_cluster(_d(p), _d(w), rate, seed, 0, None, None, None, None,
                              ctypes.byref(cnt))
    if rc != 0:
        raise ValueError(f"simulateClusterProcess failed ({rc})")
    n = cnt.value
    x, y, t = np.zeros(n), np.zeros(n), np.zeros(n)
    par = np.zeros(n, dtype=np.int32)
    rc = lib.sthk_sim_cluster(_d(p), _d(w), rate, seed, n, _d(x), _d(y), _d(t),
                              par.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                              ctypes.byref(cnt))
    if rc != 0:
        raise ValueError(f"simulateClusterProcess failed ({rc})")
    if keep is not None and keep < n:
        return EventSet(x[:keep], y[:keep], t[:keep]), par[:keep]
    return EventSet(x, y, t, window.tEnd), par
