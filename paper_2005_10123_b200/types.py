"""Model types mirroring the reference (proj/include/sthawkes/types.hpp,
likelihood.hpp). Validation and messages follow the reference exactly."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_PARAMS_MSG = ("Params: mu0, tauX, tauT, omega, h must be positive and finite; "
               "theta must be nonnegative and finite")


@dataclass
class Params:
    """Six model parameters, defaults as types.hpp:51-57."""
    mu0: float = 1.0
    tauX: float = 1.6
    tauT: float = 14.0
    theta: float = 0.1
    omega: float = 1.0
    h: float = 0.1

    def isValid(self) -> bool:  # types.hpp:59-63
        def pos(v):
            return math.isfinite(v) and v > 0.0
        return (pos(self.mu0) and pos(self.tauX) and pos(self.tauT) and pos(self.omega)
                and pos(self.h) and math.isfinite(self.theta) and self.theta >= 0.0)

    def validate(self) -> None:  # types.hpp:65-71
        if not self.isValid():
            raise ValueError(_PARAMS_MSG)

    def as_array(self) -> np.ndarray:
        return np.array([self.mu0, self.tauX, self.tauT, self.theta, self.omega, self.h],
                        dtype=np.float64)

    @staticmethod
    def from_array(a) -> "Params":
        a = [float(v) for v in a]
        return Params(*a)


class EventSet:
    """Immutable time-sorted SoA event set (types.hpp:77-137)."""

    def __init__(self, x, y, t, windowEnd: Optional[float] = None, timeOrigin: float = 0.0):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        t = np.ascontiguousarray(t, dtype=np.float64).reshape(-1)
        n = t.size
        if n < 1:
            raise ValueError("EventSet: need at least one event")
        if x.size != n or y.size != n:
            raise ValueError("EventSet: coordinate/time length mismatch")
        # the reference loop (types.hpp:90-104) stops at the first index with
        # any failure and reports, at that index: non-finite, negative, unsorted
        nonfinite = ~(np.isfinite(x) & np.isfinite(y) & np.isfinite(t))
        with np.errstate(invalid="ignore"):
            negative = t < 0
            unsorted = np.zeros(n, dtype=bool)
            unsorted[1:] = t[1:] < t[:-1]
        fail = nonfinite | negative | unsorted
        if fail.any():
            i = int(np.argmax(fail))
            if nonfinite[i]:
                raise ValueError(f"EventSet: non-finite entry at index {i}")
            if negative[i]:
                raise ValueError(f"EventSet: negative time at index {i}")
            raise ValueError(f"EventSet: times not sorted at index {i}")
        tmax = float(t[-1])
        we = tmax if windowEnd is None else float(windowEnd)
        if not math.isfinite(we) or we < tmax:
            raise ValueError("EventSet: windowEnd precedes last event")
        for a in (x, y, t):
            a.setflags(write=False)
        self._x, self._y, self._t = x, y, t
        self._windowEnd = we
        self._timeOrigin = float(timeOrigin)

    @staticmethod
    def sortedByTime(x, y, t, windowEnd=None, timeOrigin=0.0):
        """Stable sort by time, then construct (types.cpp:9-28)."""
        t = np.asarray(t, dtype=np.float64)
        order = np.argsort(t, kind="stable")
        return EventSet(np.asarray(x)[order], np.asarray(y)[order], t[order], windowEnd, timeOrigin)

    def size(self) -> int:
        return int(self._t.size)

    def __len__(self) -> int:
        return self.size()

    def windowEnd(self) -> float:
        return self._windowEnd

    def timeOrigin(self) -> float:
        return self._timeOrigin

    def xs(self) -> np.ndarray:
        return self._x

    def ys(self) -> np.ndarray:
        return self._y

    def ts(self) -> np.ndarray:
        return self._t


@dataclass
class LikelihoodResult:
    """likelihood.hpp:17-22: valid=False means logLik=-inf (degenerate rate)."""
    logLik: float = -math.inf
    valid: bool = False
    perEvent: np.ndarray = field(default_factory=lambda: np.zeros(0))
