"""Event, chain and run-configuration files: the data formats either side of
the likelihood path, mirroring the reference's IO
(proj/include/sthawkes/io.hpp, proj/src/io.cpp):

    readEvents(path, spec)        io.cpp:113-209   delimited events -> EventSet (km / days)
    writeEvents(events, path)     io.cpp:211-240   canonical CSV, %.17g, metadata comments
    deduplicate(events, r, w)     io.cpp:242-277   greedy forward sweep
    writeChain / readChain        io.cpp:355-523   versioned JSON, hex-float draws
    loadRunConfig(path)           io.cpp:525-644   structured `fit` configuration

Host-side only (no device work). Behaviour, messages and exception classes
follow the reference: std::runtime_error -> RuntimeError,
std::invalid_argument -> ValueError. Files written here are byte-identical to
the reference's (tests/test_io_cpu.py checks both directions against the
reference's io.cpp compiled verbatim into oracle/_ref/io_ref).
"""
from __future__ import annotations

import json
import math
import re
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from .types import EventSet

# units, types.hpp:20-33
METERS_PER_KM = 1000.0
MINUTES_PER_DAY = 24.0 * 60.0
SECONDS_PER_DAY = 24.0 * 60.0 * 60.0
HOURS_PER_DAY = 24.0


def metersToKm(m: float) -> float:
    return m / METERS_PER_KM


def minutesToDays(v: float) -> float:
    return v / MINUTES_PER_DAY


def secondsToDays(v: float) -> float:
    return v / SECONDS_PER_DAY


def hoursToDays(v: float) -> float:
    return v / HOURS_PER_DAY


class DistanceUnit(IntEnum):
    Meters = 0
    Km = 1


class TimeUnit(IntEnum):
    Seconds = 0
    Minutes = 1
    Hours = 2
    Days = 3


class TimeReference(IntEnum):
    WindowRelative = 0  # times already measured from the window start
    Epoch = 1           # shift so the earliest time becomes 0; offset recorded


def parseDistanceUnit(s: str) -> DistanceUnit:
    if s == "m":
        return DistanceUnit.Meters
    if s == "km":
        return DistanceUnit.Km
    raise ValueError(f"unknown distance unit '{s}' (expected m|km)")


def parseTimeUnit(s: str) -> TimeUnit:
    table = {"s": TimeUnit.Seconds, "min": TimeUnit.Minutes, "h": TimeUnit.Hours,
             "d": TimeUnit.Days}
    if s in table:
        return table[s]
    raise ValueError(f"unknown time unit '{s}' (expected s|min|h|d)")


def distanceUnitToKm(u: DistanceUnit) -> float:
    return metersToKm(1.0) if u == DistanceUnit.Meters else 1.0


def timeUnitToDays(u: TimeUnit) -> float:
    return {TimeUnit.Seconds: secondsToDays(1.0), TimeUnit.Minutes: minutesToDays(1.0),
            TimeUnit.Hours: hoursToDays(1.0), TimeUnit.Days: 1.0}[TimeUnit(u)]


@dataclass
class EventFileSpec:
    """io.hpp:25-40. windowEndDays overrides the file's metadata."""
    delimiter: str = ","
    xColumn: str = "x"
    yColumn: str = "y"
    tColumn: str = "t"
    distanceUnit: DistanceUnit = DistanceUnit.Km
    timeUnit: TimeUnit = TimeUnit.Days
    timeReference: TimeReference = TimeReference.WindowRelative
    windowEndDays: Optional[float] = None


# std::from_chars(double), general format: optional '-', decimal digits with an
# optional fraction and exponent, or inf / infinity / nan[(chars)]; no
# leading '+' or whitespace.
_FROM_CHARS = re.compile(
    r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")


def _parse_double_field(text: str, path: str, line_no: int, column: str) -> float:
    """io.cpp:38-56 (parseDoubleField)."""
    if not _FROM_CHARS.fullmatch(text):
        raise RuntimeError(f"{path}:{line_no}: cannot parse '{text}' in column {column}")
    low = text.lower().lstrip("-")
    if low.startswith("nan"):
        v = math.nan
    else:
        v = float(text)
        if math.isinf(v) and not low.startswith("inf"):  # from_chars: result_out_of_range
            raise RuntimeError(f"{path}:{line_no}: cannot parse '{text}' in column {column}")
    if not math.isfinite(v):
        raise RuntimeError(f"{path}:{line_no}: non-finite value in column {column}")
    return v


def _lines(path: str, what: str):
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise RuntimeError(f"cannot open {what}: {path}") from None
    text = data.decode("latin-1")
    parts = text.split("\n")
    if parts and parts[-1] == "":  # getline: no empty line after a final newline
        parts.pop()
    for p in parts:
        yield p[:-1] if p.endswith("\r") else p


def readEvents(path: str, spec: Optional[EventFileSpec] = None) -> EventSet:
    """io.cpp:113-209: '#key=value' metadata lines, a header naming the x / y / t
    columns, one event per line; units converted to km / days; sorted by time."""
    spec = spec or EventFileSpec()
    dist_scale = distanceUnitToKm(spec.distanceUnit)
    time_scale = timeUnitToDays(spec.timeUnit)
    meta_window_end: Optional[float] = None
    meta_origin = 0.0
    it = _lines(path, "event file")
    line_no = 0
    header_line = ""
    for line in it:
        line_no += 1
        if not line:
            continue
        if line[0] == "#":
            eq = line.find("=")
            if eq >= 0:
                key = line[1:eq].strip(" ")
                value = line[eq + 1:]
                if key == "window_end_days":
                    meta_window_end = _parse_double_field(value, path, line_no, "metadata")
                elif key == "time_origin_days":
                    meta_origin = _parse_double_field(value, path, line_no, "metadata")
            continue
        header_line = line
        break
    if not header_line:
        raise RuntimeError(f"{path}: missing header line")
    header = header_line.split(spec.delimiter)
    xc = yc = tc = -1
    for i, h in enumerate(header):  # last match wins, as in the reference loop
        if h == spec.xColumn:
            xc = i
        if h == spec.yColumn:
            yc = i
        if h == spec.tColumn:
            tc = i
    if xc < 0 or yc < 0 or tc < 0:
        raise RuntimeError(f"{path}: header lacks required columns '{spec.xColumn}', "
                           f"'{spec.yColumn}', '{spec.tColumn}'")
    xs, ys, ts = [], [], []
    for line in it:
        line_no += 1
        if not line:
            continue
        fields = line.split(spec.delimiter)
        if len(fields) != len(header):
            raise RuntimeError(f"{path}:{line_no}: expected {len(header)} fields, found "
                               f"{len(fields)}")
        xs.append(dist_scale * _parse_double_field(fields[xc], path, line_no, spec.xColumn))
        ys.append(dist_scale * _parse_double_field(fields[yc], path, line_no, spec.yColumn))
        ts.append(time_scale * _parse_double_field(fields[tc], path, line_no, spec.tColumn))
    if not xs:
        raise RuntimeError(f"{path}: no event rows")
    x, y, t = np.array(xs), np.array(ys), np.array(ts)
    origin = meta_origin
    if spec.timeReference == TimeReference.Epoch:
        shift = float(t.min())
        t = t - shift
        origin += shift
    window_end = spec.windowEndDays if spec.windowEndDays is not None else meta_window_end
    try:
        return EventSet.sortedByTime(x, y, t, window_end, origin)
    except ValueError as e:
        raise RuntimeError(f"{path}: {e}") from None


def _g17(v: float) -> str:
    return "%.17g" % v


def writeEvents(events: EventSet, path: str, parent: Optional[Sequence[int]] = None) -> None:
    """io.cpp:211-240: canonical km / days CSV, full precision (%.17g);
    readEvents(writeEvents(e)) reproduces e exactly."""
    if parent is not None and len(parent) != events.size():
        raise ValueError("writeEvents: parent length mismatch")
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot open output file: {path}") from None
    with f:
        f.write("# sthawkes events v1\n")
        f.write(f"# window_end_days={_g17(events.windowEnd())}\n")
        f.write(f"# time_origin_days={_g17(events.timeOrigin())}\n")
        f.write("x,y,t,parent\n" if parent is not None else "x,y,t\n")
        x, y, t = events.xs(), events.ys(), events.ts()
        rows = []
        for i in range(events.size()):
            r = f"{_g17(x[i])},{_g17(y[i])},{_g17(t[i])}"
            if parent is not None:
                r += f",{int(parent[i])}"
            rows.append(r)
        f.write("\n".join(rows) + "\n")


def deduplicate(events: EventSet, radiusKm: float, windowDays: float) -> EventSet:
    """io.cpp:242-277: drop an event when an earlier *retained* event lies within
    radiusKm and windowDays (inclusive); both zero disables it."""
    if radiusKm < 0.0 or windowDays < 0.0:
        raise ValueError("deduplicate: thresholds must be >= 0")
    if radiusKm == 0.0 and windowDays == 0.0:
        return events
    x, y, t = events.xs(), events.ys(), events.ts()
    r2 = radiusKm * radiusKm
    kept = np.empty(events.size(), dtype=np.int64)
    m = 0
    start = 0  # retained events are time-sorted: the live window is a suffix
    for i in range(events.size()):
        ti = t[i]
        while start < m and ti - t[kept[start]] > windowDays:
            start += 1
        dup = False
        if start < m:
            js = kept[start:m]
            dx = x[i] - x[js]
            dy = y[i] - y[js]
            dup = bool(np.any(dx * dx + dy * dy <= r2))
        if not dup:
            kept[m] = i
            m += 1
    k = kept[:m]
    return EventSet(x[k].copy(), y[k].copy(), t[k].copy(), events.windowEnd(),
                    events.timeOrigin())


# ---------------------------------------------------------------------------
# Chains (io.cpp:279-523)
# ---------------------------------------------------------------------------
FREE_PARAM_NAMES = ("mu0", "theta", "omega", "hInv")  # sampler.hpp:19-21
CHAIN_FORMAT_NAME = "sthawkes-chain"
CHAIN_FORMAT_VERSION = 1


def hexDouble(v: float) -> str:
    """C99 %a as glibc prints it (io.cpp:23-27): shortest hex mantissa."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    h = v.hex()
    sign = "-" if h.startswith("-") else ""
    mant, exp = h.lstrip("-")[2:].split("p")
    ip, _, fp = mant.partition(".")
    fp = fp.rstrip("0")
    return f"{sign}0x{ip}{'.' + fp if fp else ''}p{exp}"


_STRTOD = re.compile(
    r"[ \t\n\v\f\r]*([+-]?(?:0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
    r"|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)))")


def parseHexDouble(s: str, where: str) -> float:
    """io.cpp:29-36: strtod that must consume the whole string."""
    m = _STRTOD.fullmatch(s)
    if not m:
        raise RuntimeError(f"chain file: bad number in {where}: '{s}'")
    body = m.group(1)
    low = body.lower().lstrip("+-")
    neg = body.startswith("-")
    if low.startswith("nan"):
        return -math.nan if neg else math.nan
    if low.startswith("inf"):
        return -math.inf if neg else math.inf
    if low.startswith("0x"):
        return float.fromhex(body)
    return float(body)


@dataclass
class BackendSpec:
    """The backend a chain was run with (backend.hpp:24-60), as recorded."""
    kind: str = "serial"   # serial | simd | threads | threads+simd
    threads: int = 1
    lanes: int = 1


def parseBackend(kind: str, threads: int, lanes: int) -> BackendSpec:
    """backend.cpp:22-43 (threads = 0: the host's hardware concurrency)."""
    import os
    if threads == 0:
        threads = max(os.cpu_count() or 1, 1)
    if kind == "serial":
        b = BackendSpec("serial", 1, 1)
    elif kind == "simd":
        b = BackendSpec("simd", 1, lanes)
    elif kind == "threads":
        b = BackendSpec("threads", threads, 1)
    elif kind == "threads+simd":
        b = BackendSpec("threads+simd", threads, lanes)
    else:
        raise ValueError(f"unknown backend '{kind}' (expected serial|simd|threads|threads+simd)")
    if b.threads < 1:
        raise ValueError("Backend: threadCount must be >= 1")
    if b.lanes not in (1, 2, 4, 8):
        raise ValueError("Backend: laneWidth must be 1, 2, 4 or 8")
    return b


@dataclass
class SamplerConfig:
    """sampler.hpp:44-62 (fields that a chain file / run config records)."""
    iterations: int = 10000
    burnIn: int = 1000
    seed: int = 1
    targetAcceptance: float = 0.44
    initialTheta: List[float] = field(default_factory=lambda: [1.0, 0.1, 1.0, 1.0])
    initialProposalSd: List[float] = field(default_factory=lambda: [1.0, 1.0, 1.0, 1.0])
    initialAdaptBound: float = 5.0
    adapt: bool = True
    tauX: float = 1.6
    tauT: float = 14.0
    backend: BackendSpec = field(default_factory=BackendSpec)
    chainCount: int = 1


@dataclass
class PriorSpec:
    """sampler.hpp:24-42: truncated-normal (mean, sd) per free parameter."""
    coord: List[List[float]] = field(default_factory=lambda: [[0.0, 1.0], [0.0, 10.0],
                                                              [0.0, 10.0], [0.0, 10.0]])


@dataclass
class AdaptationEvent:
    step: int
    coord: int
    vAfter: float
    bAfter: float


@dataclass
class Chain:
    """sampler.hpp:90-108."""
    draws: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    logPost: np.ndarray = field(default_factory=lambda: np.zeros(0))
    scannedCoord: List[int] = field(default_factory=list)
    accepted: List[int] = field(default_factory=list)
    adaptations: List[AdaptationEvent] = field(default_factory=list)
    config: SamplerConfig = field(default_factory=SamplerConfig)
    priors: PriorSpec = field(default_factory=PriorSpec)
    chainSeed: int = 0
    chainIndex: int = 0
    eventCount: int = 0

    def retained(self, coord: int) -> np.ndarray:
        return self.draws[self.config.burnIn:, coord]


class _Inline(list):
    """An integer array nlohmann prints on one line (std::vector<int8_t>)."""


def _dump(v, level: int = 0) -> str:
    """nlohmann::json::dump(1, '\\t'): keys sorted, one tab per level."""
    ind, ind1 = "\t" * level, "\t" * (level + 1)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f"{ind1}{json.dumps(k)}: {_dump(v[k], level + 1)}" for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + ind + "}"
    if isinstance(v, _Inline):
        return "[" + ",".join(str(int(a)) for a in v) + "]"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(ind1 + _dump(a, level + 1) for a in v) + "\n" + ind + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, str):
        return json.dumps(v, ensure_ascii=False)
    raise TypeError(f"unsupported value {v!r}")


def writeChain(chain: Chain, path: str) -> None:
    """io.cpp:355-425."""
    s = chain.draws.shape[0]
    if s == 0:
        raise ValueError("writeChain: refusing to write empty chain")
    if s != len(chain.logPost) or s != len(chain.scannedCoord) or s != len(chain.accepted):
        raise ValueError("writeChain: inconsistent chain bookkeeping")
    c = chain.config
    doc = {
        "format": CHAIN_FORMAT_NAME,
        "version": CHAIN_FORMAT_VERSION,
        "chainIndex": int(chain.chainIndex),
        "chainSeed": int(chain.chainSeed),
        "eventCount": int(chain.eventCount),
        "config": {
            "iterations": int(c.iterations),
            "burnIn": int(c.burnIn),
            "seed": int(c.seed),
            "targetAcceptance": hexDouble(c.targetAcceptance),
            "initialTheta": [hexDouble(v) for v in c.initialTheta],
            "initialProposalSd": [hexDouble(v) for v in c.initialProposalSd],
            "initialAdaptBound": hexDouble(c.initialAdaptBound),
            "adapt": bool(c.adapt),
            "tauX": hexDouble(c.tauX),
            "tauT": hexDouble(c.tauT),
            "backend": {"kind": c.backend.kind, "threads": int(c.backend.threads),
                        "lanes": int(c.backend.lanes)},
            "chainCount": int(c.chainCount),
        },
        "priors": {name: {"mean": hexDouble(chain.priors.coord[d][0]),
                          "sd": hexDouble(chain.priors.coord[d][1])}
                   for d, name in enumerate(FREE_PARAM_NAMES)},
        "paramNames": list(FREE_PARAM_NAMES),
        "draws": [[hexDouble(v) for v in row] for row in chain.draws],
        "logPost": [hexDouble(v) for v in chain.logPost],
        "scannedCoord": _Inline(chain.scannedCoord),
        "accepted": _Inline(chain.accepted),
        "adaptations": [{"step": int(a.step), "coord": int(a.coord), "v": hexDouble(a.vAfter),
                         "b": hexDouble(a.bAfter)} for a in chain.adaptations],
    }
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot open chain file for writing: {path}") from None
    with f:
        f.write(_dump(doc) + "\n")


class _Corrupt(Exception):
    pass


def _at(obj, key):
    """nlohmann .at(): out_of_range 403 for a missing key."""
    if isinstance(obj, dict):
        if key not in obj:
            raise _Corrupt(f"[json.exception.out_of_range.403] key '{key}' not found")
        return obj[key]
    if isinstance(obj, list) and isinstance(key, int):
        if not 0 <= key < len(obj):
            raise _Corrupt(f"[json.exception.out_of_range.401] array index {key} is out of "
                           f"range")
        return obj[key]
    raise _Corrupt(f"[json.exception.type_error.304] cannot use at() with {_tname(obj)}")


def _tname(v) -> str:
    if v is None:
        return "null"
    if isinstance(v, bool):
        return "boolean"
    if isinstance(v, (int, float)):
        return "number"
    if isinstance(v, str):
        return "string"
    if isinstance(v, list):
        return "array"
    return "object"


def _get(v, kind):
    """nlohmann get<T>(): numbers convert between integer and floating kinds
    (static_cast), anything else of the wrong type is type_error 302."""
    is_num = isinstance(v, (int, float)) and not isinstance(v, bool)
    ok = {"string": isinstance(v, str), "bool": isinstance(v, bool), "int": is_num,
          "number": is_num}[kind]
    if not ok:
        want = {"string": "string", "bool": "boolean", "int": "number",
                "number": "number"}[kind]
        raise _Corrupt(f"[json.exception.type_error.302] type must be {want}, but is "
                       f"{_tname(v)}")
    if kind == "int":
        return int(v)
    return v


def readChain(path: str) -> Chain:
    """io.cpp:427-523."""
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"cannot open chain file: {path}") from None
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise RuntimeError(f"chain file {path} is truncated or corrupt: {e}") from None
    try:
        if _get(_at(j, "format"), "string") != CHAIN_FORMAT_NAME:
            raise RuntimeError(f"chain file {path}: unrecognized format")
        ver = _get(_at(j, "version"), "int")
        if ver != CHAIN_FORMAT_VERSION:
            raise RuntimeError(f"chain file {path}: unsupported version {ver} (expected "
                               f"{CHAIN_FORMAT_VERSION})")
        ch = Chain()
        ch.chainIndex = _get(_at(j, "chainIndex"), "int")
        ch.chainSeed = _get(_at(j, "chainSeed"), "int")
        ch.eventCount = _get(_at(j, "eventCount"), "int")
        cfg = _at(j, "config")
        c = ch.config
        c.iterations = _get(_at(cfg, "iterations"), "int")
        c.burnIn = _get(_at(cfg, "burnIn"), "int")
        c.seed = _get(_at(cfg, "seed"), "int")
        c.targetAcceptance = parseHexDouble(_get(_at(cfg, "targetAcceptance"), "string"),
                                            "targetAcceptance")
        c.initialTheta = [parseHexDouble(_get(_at(_at(cfg, "initialTheta"), d), "string"),
                                         "initialTheta") for d in range(4)]
        c.initialProposalSd = [
            parseHexDouble(_get(_at(_at(cfg, "initialProposalSd"), d), "string"),
                           "initialProposalSd") for d in range(4)]
        c.initialAdaptBound = parseHexDouble(_get(_at(cfg, "initialAdaptBound"), "string"),
                                             "initialAdaptBound")
        c.adapt = _get(_at(cfg, "adapt"), "bool")
        c.tauX = parseHexDouble(_get(_at(cfg, "tauX"), "string"), "tauX")
        c.tauT = parseHexDouble(_get(_at(cfg, "tauT"), "string"), "tauT")
        c.backend = _backend_from_json(_at(cfg, "backend"), "config.backend.")
        c.chainCount = _get(_at(cfg, "chainCount"), "int")
        pri = _at(j, "priors")
        ch.priors = PriorSpec([[parseHexDouble(_get(_at(_at(pri, n), "mean"), "string"),
                                               "priors.mean"),
                                parseHexDouble(_get(_at(_at(pri, n), "sd"), "string"),
                                               "priors.sd")] for n in FREE_PARAM_NAMES])
        draws = _at(j, "draws")
        s = len(draws)
        if s == 0:
            raise RuntimeError(f"chain file {path}: no draws")
        ch.draws = np.array([[parseHexDouble(_get(_at(_at(draws, i), d), "string"), "draws")
                              for d in range(4)] for i in range(s)])
        lp = _at(j, "logPost")
        if len(lp) != s:
            raise RuntimeError(f"chain file {path}: logPost length")
        ch.logPost = np.array([parseHexDouble(_get(v, "string"), "logPost") for v in lp])
        ch.scannedCoord = [int(_get(v, "int")) for v in _at(j, "scannedCoord")]
        ch.accepted = [int(_get(v, "int")) for v in _at(j, "accepted")]
        if len(ch.scannedCoord) != s or len(ch.accepted) != s:
            raise RuntimeError(f"chain file {path}: bookkeeping length mismatch")
        for a in _at(j, "adaptations"):
            ch.adaptations.append(AdaptationEvent(
                _get(_at(a, "step"), "int"), _get(_at(a, "coord"), "int"),
                parseHexDouble(_get(_at(a, "v"), "string"), "adaptations.v"),
                parseHexDouble(_get(_at(a, "b"), "string"), "adaptations.b")))
        return ch
    except _Corrupt as e:
        raise RuntimeError(f"chain file {path} is truncated or corrupt: {e}") from None


def _require_keys(obj: dict, where: str, allowed) -> None:
    """io.cpp:307-322."""
    for key in obj:
        if key not in allowed:
            raise RuntimeError(f"config: unknown key '{where}{key}'")


def _value(obj: dict, key: str, default, kind: str):
    """nlohmann j.value(key, default): default when absent, type-checked otherwise."""
    if key not in obj:
        return default
    v = obj[key]
    if kind == "number" and isinstance(v, bool):
        raise RuntimeError(f"[json.exception.type_error.302] type must be number, but is "
                           f"boolean")
    try:
        return _get(v, kind)
    except _Corrupt as e:
        raise RuntimeError(str(e)) from None


def _backend_from_json(j, where: str) -> BackendSpec:
    """io.cpp:324-330."""
    if not isinstance(j, dict):
        raise _Corrupt(f"[json.exception.type_error.306] cannot use value() with {_tname(j)}")
    _require_keys(j, where, ("kind", "threads", "lanes"))
    return parseBackend(_value(j, "kind", "serial", "string"), _value(j, "threads", 1, "int"),
                        _value(j, "lanes", 4, "int"))


@dataclass
class DedupOptions:
    radiusKm: float = 0.0
    windowDays: float = 0.0


@dataclass
class RunConfig:
    """io.hpp:67-77: one document driving `fit`; unknown keys are errors."""
    dataPath: str = ""
    fileSpec: EventFileSpec = field(default_factory=EventFileSpec)
    dedup: DedupOptions = field(default_factory=DedupOptions)
    sampler: SamplerConfig = field(default_factory=SamplerConfig)
    priors: PriorSpec = field(default_factory=PriorSpec)
    outputPrefix: str = "chain"


def loadRunConfig(path: str) -> RunConfig:
    """io.cpp:525-644."""
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"cannot open config file: {path}") from None
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise RuntimeError(f"config file {path}: {e}") from None
    rc = RunConfig()
    _require_keys(j, "", ("data", "model", "priors", "sampler", "backend", "output"))
    if "data" in j:
        d = j["data"]
        _require_keys(d, "data.", ("path", "delimiter", "distanceUnit", "timeUnit",
                                   "timeReference", "columns", "windowEndDays", "dedup"))
        rc.dataPath = _value(d, "path", "", "string")
        delim = _value(d, "delimiter", ",", "string")
        if len(delim.encode()) != 1:
            raise RuntimeError("config: data.delimiter must be one character")
        rc.fileSpec.delimiter = delim
        rc.fileSpec.distanceUnit = parseDistanceUnit(_value(d, "distanceUnit", "km", "string"))
        rc.fileSpec.timeUnit = parseTimeUnit(_value(d, "timeUnit", "d", "string"))
        ref = _value(d, "timeReference", "window", "string")
        if ref == "window":
            rc.fileSpec.timeReference = TimeReference.WindowRelative
        elif ref == "epoch":
            rc.fileSpec.timeReference = TimeReference.Epoch
        else:
            raise RuntimeError("config: data.timeReference must be window|epoch")
        if "columns" in d:
            cols = d["columns"]
            _require_keys(cols, "data.columns.", ("x", "y", "t"))
            rc.fileSpec.xColumn = _value(cols, "x", "x", "string")
            rc.fileSpec.yColumn = _value(cols, "y", "y", "string")
            rc.fileSpec.tColumn = _value(cols, "t", "t", "string")
        if "windowEndDays" in d:
            rc.fileSpec.windowEndDays = float(_value(d, "windowEndDays", 0.0, "number"))
        if "dedup" in d:
            dd = d["dedup"]
            _require_keys(dd, "data.dedup.", ("radiusMeters", "windowMinutes"))
            rc.dedup.radiusKm = metersToKm(float(_value(dd, "radiusMeters", 0.0, "number")))
            rc.dedup.windowDays = minutesToDays(float(_value(dd, "windowMinutes", 0.0,
                                                             "number")))
    if "model" in j:
        _require_keys(j["model"], "model.", ("tauXKm", "tauTDays"))
        rc.sampler.tauX = float(_value(j["model"], "tauXKm", rc.sampler.tauX, "number"))
        rc.sampler.tauT = float(_value(j["model"], "tauTDays", rc.sampler.tauT, "number"))
    if "priors" in j:
        _require_keys(j["priors"], "priors.", FREE_PARAM_NAMES)
        for dd, name in enumerate(FREE_PARAM_NAMES):
            if name in j["priors"]:
                pj = j["priors"][name]
                _require_keys(pj, f"priors.{name}.", ("mean", "sd"))
                coord = rc.priors.coord[dd]
                coord[0] = float(_value(pj, "mean", coord[0], "number"))
                coord[1] = float(_value(pj, "sd", coord[1], "number"))
    if "sampler" in j:
        s = j["sampler"]
        _require_keys(s, "sampler.", ("iterations", "burnIn", "seed", "chains",
                                      "targetAcceptance", "adapt", "initial", "proposalSd"))
        rc.sampler.iterations = int(_value(s, "iterations", rc.sampler.iterations, "number"))
        rc.sampler.burnIn = int(_value(s, "burnIn", rc.sampler.burnIn, "number"))
        rc.sampler.seed = int(_value(s, "seed", rc.sampler.seed, "number"))
        rc.sampler.chainCount = int(_value(s, "chains", rc.sampler.chainCount, "number"))
        rc.sampler.targetAcceptance = float(_value(s, "targetAcceptance",
                                                   rc.sampler.targetAcceptance, "number"))
        rc.sampler.adapt = _value(s, "adapt", rc.sampler.adapt, "bool")
        for key in ("initial", "proposalSd"):
            if key not in s:
                continue
            _require_keys(s[key], f"sampler.{key}.", FREE_PARAM_NAMES)
            for dd, name in enumerate(FREE_PARAM_NAMES):
                if name not in s[key]:
                    continue
                v = float(_value(s[key], name, 0.0, "number"))
                if key == "initial":
                    rc.sampler.initialTheta[dd] = v
                else:
                    rc.sampler.initialProposalSd[dd] = v
    if "backend" in j:
        try:
            rc.sampler.backend = _backend_from_json(j["backend"], "backend.")
        except _Corrupt as e:
            raise RuntimeError(str(e)) from None
    if "output" in j:
        _require_keys(j["output"], "output.", ("prefix",))
        rc.outputPrefix = _value(j["output"], "prefix", rc.outputPrefix, "string")
    return rc
