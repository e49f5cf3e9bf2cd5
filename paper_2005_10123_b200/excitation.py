"""Excitation probabilities pi (the sibling consumer of the pair sums;
SURVEY.md §8 f2), mirroring proj/include/sthawkes/excitation.hpp:15-48 and
proj/src/excitation.cpp:13-130 on the B200 engine.

For a posterior draw list the engine's background-sum cache applies
whenever tauX and tauT are shared by the draws (as in the reference MH
sampler), so each draw costs one trigger-band sweep."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .engine import Engine, EngineError, default_engine
from .types import EventSet, Params


@dataclass
class ExcitationVector:
    """excitation.hpp:15-20."""
    pi: np.ndarray
    mu: np.ndarray
    xi: np.ndarray


@dataclass
class PosteriorExcitation:
    """excitation.hpp:36-41. perDraw is (kept, N), or shape (0, 0) when
    kept * N exceeds memoryCapEntries."""
    meanPi: np.ndarray
    perDraw: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    drawIndices: List[int] = field(default_factory=list)


def excitationProbabilities(events: EventSet, params: Params, backend=None,
                            engine: Optional[Engine] = None) -> ExcitationVector:
    """excitation.cpp:13-58. Raises ValueError on invalid params and
    EngineError (the reference's runtime_error) on an underflowed rate."""
    params.validate()
    eng = engine or default_engine()
    with eng._lock:
        eng.load(events)
        eng.set_params(params)
        mu, xi, pi = eng.excitation()
    return ExcitationVector(pi=pi, mu=mu, xi=xi)


def thinIndices(total: int, keep: int) -> List[int]:
    """Evenly spaced thinning j -> floor(j * total / kept) (excitation.cpp:60-70)."""
    if total < 1 or keep < 1:
        raise ValueError("thinIndices: need total >= 1 and keep >= 1")
    keep = min(keep, total)
    return [j * total // keep for j in range(keep)]


def posteriorExcitation(events: EventSet, draws: List[Params], backend=None,
                        thinTo: int = 1000, memoryCapEntries: int = 100_000_000,
                        dumpPath: Optional[str] = None,
                        engine: Optional[Engine] = None) -> PosteriorExcitation:
    """excitation.cpp:72-130: mean pi over thinned draws (summed in draw
    order, then divided), optional per-draw matrix and text dump. The kept
    draws run as batches on the device (sthk_excitation_batch: one background
    sweep for draws sharing tauX, tauT); errors surface at the same draw, with
    the same dump lines written before it, as in the reference's loop."""
    if len(draws) == 0:
        raise ValueError("posteriorExcitation: no draws")
    if thinTo < 1:
        raise ValueError("posteriorExcitation: thinTo must be >= 1")
    n = events.size()
    idx = thinIndices(len(draws), thinTo)
    kept = len(idx)
    retain = kept * n <= memoryCapEntries
    per = np.zeros((kept, n)) if retain else np.zeros((0, 0))
    mean = np.zeros(n)
    # the first kept draw with invalid params ends the loop there (the
    # reference validates inside excitationProbabilities)
    stop, stop_err = kept, None
    for j, d in enumerate(idx):
        try:
            draws[d].validate()
        except ValueError as e:
            stop, stop_err = j, f"posteriorExcitation: draw {d}: {e}"
            break
    dump = None
    if dumpPath is not None:
        try:
            dump = open(dumpPath, "w")
        except OSError:
            raise RuntimeError(f"posteriorExcitation: cannot open dump file {dumpPath}") from None
        dump.write(f"# sthawkes pi draws v1, events={n}\n")
    want_rows = retain or dump is not None
    # draws per device call: bounded host memory for the per-draw rows
    step = max(1, min(stop, 10_000_000 // max(n, 1))) if want_rows else max(stop, 1)
    eng = engine or default_engine()
    try:
        j0 = 0
        while j0 < stop:
            j1 = min(stop, j0 + step)
            with eng._lock:
                eng.load(events)
                mean, rows, bad = eng.excitation_batch(
                    [draws[d].as_array() for d in idx[j0:j1]], sum_pi=mean, per_draw=want_rows)
            done = j1 if bad < 0 else j0 + bad
            for j in range(j0, done):
                if retain:
                    per[j] = rows[j - j0]
                if dump is not None:
                    dump.write(str(idx[j]) + "".join("\t%.17g" % v for v in rows[j - j0]) + "\n")
            if bad >= 0:
                raise RuntimeError(f"posteriorExcitation: draw {idx[j0 + bad]}: "
                                   "excitationProbabilities: per-event rate underflowed to zero")
            j0 = j1
        if stop_err is not None:
            raise RuntimeError(stop_err)
    finally:
        if dump is not None:
            dump.close()
    mean /= float(kept)
    return PosteriorExcitation(meanPi=mean, perDraw=per, drawIndices=idx)
