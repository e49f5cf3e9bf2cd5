"""CPU: the event / chain / run-config file formats in the
Python host mirror (paper_2005_10123_b200/io.py) against the reference's own
io.cpp, compiled verbatim into oracle/_ref/io_ref (oracle/io_ref.cpp). Values
must be bitwise equal, files byte-identical, error messages identical."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

import oracle_glue as og
import paper_2005_10123_b200 as pk
from paper_2005_10123_b200 import io as pio

IO_REF = os.path.join(og.REF_DIR, "io_ref")


def _ref(*args):
    if not os.path.exists(IO_REF):
        pytest.skip("oracle/_ref/io_ref not built (needs /root/reference at build time)")
    out = subprocess.run([IO_REF, *map(str, args)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


def _arr(v):
    return np.array([float.fromhex(s) for s in v])


def _events_json(ev, parent=None):
    d = {"x": [pio.hexDouble(v) for v in ev.xs()], "y": [pio.hexDouble(v) for v in ev.ys()],
         "t": [pio.hexDouble(v) for v in ev.ts()], "windowEnd": pio.hexDouble(ev.windowEnd()),
         "timeOrigin": pio.hexDouble(ev.timeOrigin())}
    if parent is not None:
        d["parent"] = [int(p) for p in parent]
    return d


def _same_events(ours, ref):
    assert ref["ok"], ref
    assert np.array_equal(ours.xs(), _arr(ref["x"]))
    assert np.array_equal(ours.ys(), _arr(ref["y"]))
    assert np.array_equal(ours.ts(), _arr(ref["t"]))
    assert ours.windowEnd() == float.fromhex(ref["windowEnd"])
    assert ours.timeOrigin() == float.fromhex(ref["timeOrigin"])


def _read_both(path, delim=",", cols=("x", "y", "t"), dist="km", time="d", ref="window",
               window_end=None):
    spec = pio.EventFileSpec(delim, *cols, pio.parseDistanceUnit(dist), pio.parseTimeUnit(time),
                             pio.TimeReference.Epoch if ref == "epoch"
                             else pio.TimeReference.WindowRelative, window_end)
    args = ["read", path, delim, *cols, dist, time, ref]
    if window_end is not None:
        args.append(repr(window_end))
    r = _ref(*args)
    try:
        ours = pio.readEvents(path, spec)
    except (RuntimeError, ValueError) as e:
        assert not r["ok"], (r, e)
        assert str(e) == r["what"]
        assert (r["type"] == "invalid_argument") == isinstance(e, ValueError)
        return None
    _same_events(ours, r)
    return ours


def test_read_events_units_epoch_metadata(tmp_path):
    rng = np.random.default_rng(5)
    n = 200
    x = rng.uniform(0, 15000, n)
    y = rng.uniform(0, 15000, n)
    t = rng.uniform(1.6e9, 1.6e9 + 3e7, n)  # epoch seconds, unsorted, with ties
    t[10] = t[11]
    p = tmp_path / "ev.csv"
    lines = ["# exported", "# window_end_days =400", "id;lon;lat;ts;extra"]
    for i in range(n):
        lines.append(f"{i};{float(x[i])!r};{float(y[i])!r};{float(t[i])!r};z")
    p.write_text("\r\n".join(lines) + "\r\n\r\n")
    ev = _read_both(str(p), ";", ("lon", "lat", "ts"), "m", "s", "epoch")
    assert ev is not None and ev.size() == n and ev.ts()[0] == 0.0
    for unit in ("s", "min", "h", "d"):
        _read_both(str(p), ";", ("lon", "lat", "ts"), "km", unit, "epoch")
    # a metadata value with a leading blank does not parse (from_chars)
    q = tmp_path / "ev2.csv"
    q.write_text(p.read_text().replace("=400", "= 400"))
    assert _read_both(str(q), ";", ("lon", "lat", "ts"), "m", "s", "epoch") is None
    # window-relative: the metadata window end (400 d) precedes the raw times;
    # an explicit window end overrides the metadata
    _read_both(str(p), ";", ("lon", "lat", "ts"), "m", "s", "window")
    _read_both(str(p), ";", ("lon", "lat", "ts"), "m", "s", "epoch", window_end=1.0)
    _read_both(str(p), ";", ("lon", "lat", "ts"), "m", "s", "epoch", window_end=400.0)


@pytest.mark.parametrize("body,expect_ok", [
    ("x,y,t\n1,2,3\n0.5,1e-3,2.5\n", True),
    ("# window_end_days=10\n# time_origin_days=2.5\nx,y,t\n1,2,3\n", True),
    ("# window_end_days=2\nx,y,t\n1,2,3\n", False),       # windowEnd precedes last event
    ("x,y\n1,2\n", False),                                # missing column
    ("# only comments\n\n", False),                      # missing header
    ("x,y,t\n", False),                                   # no event rows
    ("x,y,t\n1,2\n", False),                              # field count
    ("x,y,t\n1,2,+3\n", False),                           # from_chars: no '+'
    ("x,y,t\n1,2, 3\n", False),                           # ... no whitespace
    ("x,y,t\n1,2,3e\n", False),                           # trailing garbage
    ("x,y,t\n1,2,nan\n", False),                          # non-finite
    ("x,y,t\n1,2,inf\n", False),
    ("x,y,t\n1,2,1e400\n", False),                        # out of range
    ("x,y,t\n1,2,-1\n", False),                           # negative time
    ("x,y,t\n1,2,.5\n3,4,5.\n", True),
    ("t,x,y,x\n3,1,2,7\n", True),                         # duplicate column: last wins
    ("# window_end_days=abc\nx,y,t\n1,2,3\n", False),    # bad metadata
    ("#no equals sign\n#other=1\nx,y,t\n1,2,3\n", True),
])
def test_read_events_cases(tmp_path, body, expect_ok):
    p = tmp_path / "e.csv"
    p.write_text(body)
    ev = _read_both(str(p))
    assert (ev is not None) == expect_ok


def test_read_events_missing_file(tmp_path):
    _read_both(str(tmp_path / "nope.csv"))


def test_write_events_byte_identical_and_round_trip(tmp_path):
    ev, parent = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                           pk.SimWindow(0, 15, 0, 15, 200), 0.05, 7,
                                           keep=500)
    for par in (None, parent[:ev.size()]):
        src = tmp_path / "src.json"
        src.write_text(json.dumps(_events_json(ev, par)))
        ref_path, our_path = tmp_path / "ref.csv", tmp_path / "ours.csv"
        assert _ref("write", src, ref_path)["ok"]
        pio.writeEvents(ev, str(our_path), par)
        assert our_path.read_bytes() == ref_path.read_bytes()
        back = pio.readEvents(str(our_path))
        assert np.array_equal(back.ts(), ev.ts()) and np.array_equal(back.xs(), ev.xs())
        assert back.windowEnd() == ev.windowEnd()
    with pytest.raises(ValueError, match="parent length mismatch"):
        pio.writeEvents(ev, str(tmp_path / "x.csv"), [0, 1])


@pytest.mark.parametrize("radius,window", [(0.0, 0.0), (0.05, 0.0), (0.0, 0.01),
                                           (0.03, 0.002), (0.5, 1.0), (10.0, 100.0)])
def test_deduplicate_matches_reference(tmp_path, radius, window):
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 300), 0.05, 9, keep=3000)
    src = tmp_path / "src.json"
    src.write_text(json.dumps(_events_json(ev)))
    r = _ref("dedup", src, repr(radius), repr(window))
    _same_events(pio.deduplicate(ev, radius, window), r)
    with pytest.raises(ValueError, match="thresholds must be >= 0"):
        pio.deduplicate(ev, -1.0, 0.0)


def _same_chain(ch, r):
    assert r["ok"], r
    assert ch.chainIndex == r["chainIndex"] and ch.chainSeed == r["chainSeed"]
    assert ch.eventCount == r["eventCount"]
    c = ch.config
    assert (c.iterations, c.burnIn, c.seed, c.chainCount, c.adapt) == (
        r["iterations"], r["burnIn"], r["seed"], r["chainCount"], r["adapt"])
    for k in ("targetAcceptance", "initialAdaptBound", "tauX", "tauT"):
        assert getattr(c, k) == float.fromhex(r[k]), k
    assert c.initialTheta == list(_arr(r["initialTheta"]))
    assert c.initialProposalSd == list(_arr(r["initialProposalSd"]))
    assert [c.backend.threads, c.backend.lanes] == r["backend"][1:]
    assert ch.priors.coord == [[float.fromhex(a), float.fromhex(b)] for a, b in r["priors"]]
    assert np.array_equal(ch.draws, np.array([_arr(row) for row in r["draws"]]))
    assert np.array_equal(ch.logPost, _arr(r["logPost"]))
    assert ch.scannedCoord == r["scannedCoord"] and ch.accepted == r["accepted"]
    assert [(a.step, a.coord, a.vAfter, a.bAfter) for a in ch.adaptations] == [
        (a["step"], a["coord"], float.fromhex(a["v"]), float.fromhex(a["b"]))
        for a in r["adaptations"]]


def test_chain_files_both_directions(tmp_path):
    ref_file = tmp_path / "ref_chain.json"
    r = _ref("chain", 60, 120, 5, ref_file)
    ch = pio.readChain(str(ref_file))
    _same_chain(ch, r)
    ours = tmp_path / "our_chain.json"
    pio.writeChain(ch, str(ours))
    assert ours.read_bytes() == ref_file.read_bytes()
    _same_chain(ch, _ref("readchain", ours))
    assert np.array_equal(ch.retained(2), ch.draws[ch.config.burnIn:, 2])


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d.update(format="other"), "unrecognized format"),
    (lambda d: d.update(version=2), "unsupported version 2 (expected 1)"),
    (lambda d: d.pop("logPost"), "truncated or corrupt"),
    (lambda d: d["logPost"].pop(), "logPost length"),
    (lambda d: d.update(draws=[]), "no draws"),
    (lambda d: d["draws"][0].__setitem__(1, "0x1.8p+0junk"), "bad number in draws"),
    (lambda d: d.update(accepted=d["accepted"][:-1]), "bookkeeping length mismatch"),
])
def test_chain_file_errors(tmp_path, mutate, msg):
    src = tmp_path / "c.json"
    _ref("chain", 40, 30, 2, src)
    d = json.loads(src.read_text())
    mutate(d)
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(d))
    r = _ref("readchain", bad)
    assert not r["ok"] and msg in r["what"]
    with pytest.raises(RuntimeError) as e:
        pio.readChain(str(bad))
    assert msg in str(e.value)
    if "truncated" not in msg:
        assert str(e.value) == r["what"]
    (tmp_path / "trunc.json").write_text(src.read_text()[:100])
    with pytest.raises(RuntimeError, match="is truncated or corrupt"):
        pio.readChain(str(tmp_path / "trunc.json"))


CONFIGS = [
    {},
    {"data": {"path": "dc.csv", "delimiter": ";", "distanceUnit": "m", "timeUnit": "s",
              "timeReference": "epoch", "columns": {"x": "lon", "y": "lat", "t": "ts"},
              "windowEndDays": 4750, "dedup": {"radiusMeters": 25, "windowMinutes": 2}},
     "model": {"tauXKm": 1.2, "tauTDays": 10},
     "priors": {"mu0": {"mean": 0.5, "sd": 2}, "hInv": {"sd": 3}},
     "sampler": {"iterations": 500, "burnIn": 50, "seed": 9, "chains": 2,
                 "targetAcceptance": 0.3, "adapt": False,
                 "initial": {"mu0": 0.7, "omega": 100}, "proposalSd": {"theta": 0.2}},
     "backend": {"kind": "threads+simd", "threads": 4, "lanes": 8},
     "output": {"prefix": "run1"}},
    {"bogus": 1},
    {"data": {"colums": {}}},
    {"data": {"delimiter": ";;"}},
    {"data": {"timeReference": "utc"}},
    {"data": {"distanceUnit": "mi"}},
    {"backend": {"kind": "gpu"}},
    {"backend": {"kind": "simd", "lanes": 3}},
    {"sampler": {"initial": {"h": 1}}},
]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_load_run_config(tmp_path, cfg):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    r = _ref("config", p)
    try:
        rc = pio.loadRunConfig(str(p))
    except (RuntimeError, ValueError) as e:
        assert not r["ok"], (r, e)
        assert str(e) == r["what"]
        assert (r["type"] == "invalid_argument") == isinstance(e, ValueError)
        return
    assert r["ok"], r
    fs = rc.fileSpec
    assert (rc.dataPath, fs.delimiter, fs.xColumn, fs.yColumn, fs.tColumn) == (
        r["dataPath"], r["delimiter"], r["xColumn"], r["yColumn"], r["tColumn"])
    assert (int(fs.distanceUnit), int(fs.timeUnit), int(fs.timeReference)) == (
        r["distanceUnit"], r["timeUnit"], r["timeReference"])
    assert (fs.windowEndDays is None) == (r["windowEndDays"] == "none")
    if fs.windowEndDays is not None:
        assert fs.windowEndDays == float.fromhex(r["windowEndDays"])
    assert rc.dedup.radiusKm == float.fromhex(r["dedupRadiusKm"])
    assert rc.dedup.windowDays == float.fromhex(r["dedupWindowDays"])
    s = rc.sampler
    assert (s.iterations, s.burnIn, s.seed, s.chainCount, s.adapt) == (
        r["iterations"], r["burnIn"], r["seed"], r["chainCount"], r["adapt"])
    assert s.targetAcceptance == float.fromhex(r["targetAcceptance"])
    assert s.initialTheta == list(_arr(r["initialTheta"]))
    assert s.initialProposalSd == list(_arr(r["initialProposalSd"]))
    assert (s.tauX, s.tauT) == (float.fromhex(r["tauX"]), float.fromhex(r["tauT"]))
    assert [s.backend.threads, s.backend.lanes] == r["backend"][1:]
    assert rc.priors.coord == [[float.fromhex(a), float.fromhex(b)] for a, b in r["priors"]]
    assert rc.outputPrefix == r["outputPrefix"]


def test_hex_double_matches_c_printf():
    vals = [0.0, -0.0, 1.0, 0.1, -2.5, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
            math.pi, 1e-300, 123456.789]
    for v in vals:
        assert float.fromhex(pio.hexDouble(v)) == v or (v == 0 and pio.hexDouble(v).endswith("0p+0"))
        assert pio.parseHexDouble(pio.hexDouble(v), "x") == v
    assert pio.hexDouble(1.0) == "0x1p+0" and pio.hexDouble(0.0) == "0x0p+0"
    assert pio.hexDouble(-0.0) == "-0x0p+0" and pio.hexDouble(0.5) == "0x1p-1"
    assert pio.parseHexDouble("  1.5", "x") == 1.5
    with pytest.raises(RuntimeError, match="bad number in x"):
        pio.parseHexDouble("1.5 ", "x")
