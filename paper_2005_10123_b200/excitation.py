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
    order, then divided), optional per-draw matrix and text dump."""
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
    dump = None
    if dumpPath is not None:
        try:
            dump = open(dumpPath, "w")
        except OSError:
            raise RuntimeError(f"posteriorExcitation: cannot open dump file {dumpPath}") from None
        dump.write(f"# sthawkes pi draws v1, events={n}\n")
    try:
        for j, d in enumerate(idx):
            try:
                ex = excitationProbabilities(events, draws[d], engine=engine)
            except (ValueError, EngineError) as e:
                raise RuntimeError(f"posteriorExcitation: draw {d}: {e}") from None
            mean += ex.pi
            if retain:
                per[j] = ex.pi
            if dump is not None:
                dump.write(str(d) + "".join("\t%.17g" % v for v in ex.pi) + "\n")
    finally:
        if dump is not None:
            dump.close()
    mean /= float(kept)
    return PosteriorExcitation(meanPi=mean, perDraw=per, drawIndices=idx)
