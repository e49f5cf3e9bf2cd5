"""Engine handle over the C ABI (include/sthk.h) and the reference-named
entry points logLikelihood / logLikelihoodBatch (likelihood.hpp:24-31) plus
logLikelihoodGradient (new; the reference has no gradient).

Error mapping follows the C++ adapter: STHK_EINVAL ->
ValueError (the reference's std::invalid_argument), anything else ->
EngineError (std::runtime_error). A degenerate evaluation is not an error:
it returns valid=False, logLik=-inf (likelihood.cpp:47-50).
"""
from __future__ import annotations

import ctypes
import threading
from ctypes import byref, c_double, c_int, c_int64, c_void_p
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .types import EventSet, LikelihoodResult, Params


class EngineError(RuntimeError):
    pass


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(c_double))


def _vptr(a):  # (c_void_p arguments of the per-evaluation calls: cheaper than data_as)
    return None if a is None else a.ctypes.data


class Engine:
    """Stateful device engine: events stay resident in HBM across calls.

    devices: local CUDA device ids driven from this process, one row shard
    each (NCCL between distinct devices; a repeated id runs several shards
    on one GPU, combined by device copies -- the multi-GPU data flow
    emulated on one device).
    rank/world/nccl_id: one-process-per-GPU mode (torchrun); pass the id
    from Engine.nccl_unique_id() on rank 0 to every rank.
    rank/world/comm: rank mode whose collectives run through host callbacks
    (hostcomm.TorchDistComm over gloo), e.g. several ranks on one GPU.
    """

    def __init__(self, devices: Sequence[int] = (0,), *, rank: Optional[int] = None,
                 world: int = 1, nccl_id: Optional[bytes] = None, comm=None):
        self._lib = _lib.load_library()
        self._h = c_void_p()
        self._lock = threading.Lock()
        self._events_key = None
        self._n = 0
        self._comm = comm  # (keeps the host callbacks alive)
        if rank is None:
            ids = (c_int * len(devices))(*devices)
            rc = self._lib.sthk_create(ids, len(devices), byref(self._h))
        elif comm is not None:
            rc = self._lib.sthk_create_rank_hosted(int(devices[0]), int(rank), int(world),
                                                   byref(comm.struct), byref(self._h))
        else:
            buf = None
            if world > 1:
                if nccl_id is None or len(nccl_id) != _lib.NCCL_ID_BYTES:
                    raise ValueError("nccl_id must be the 128-byte id from rank 0")
                buf = ctypes.create_string_buffer(bytes(nccl_id), _lib.NCCL_ID_BYTES)
            rc = self._lib.sthk_create_rank(int(devices[0]), int(rank), int(world),
                                            buf, byref(self._h))
        if rc != _lib.STHK_OK:
            msg = self._lib.sthk_last_error(None).decode()
            raise (ValueError if rc == _lib.STHK_EINVAL else EngineError)(
                f"sthk_create failed ({rc}): {msg}")

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _lib.load_library()
        buf = ctypes.create_string_buffer(_lib.NCCL_ID_BYTES)
        rc = lib.sthk_nccl_unique_id(buf)
        if rc != _lib.STHK_OK:
            raise EngineError(f"sthk_nccl_unique_id failed ({rc})")
        return buf.raw

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if self._h:
            self._lib.sthk_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- helpers -----------------------------------------------------------
    def _check(self, rc: int, what: str) -> None:
        if rc == _lib.STHK_OK:
            return
        msg = self._lib.sthk_last_error(self._h).decode()
        if rc == _lib.STHK_EINVAL:
            raise ValueError(msg)
        if rc == _lib.STHK_ERANGE:
            raise EngineError(msg)
        raise EngineError(f"{what} failed ({rc}): {msg}")

    @property
    def handle(self) -> c_void_p:
        return self._h

    # -- C ABI wrappers ----------------------------------------------------
    def load_events(self, x, y, t, window_end: float) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        n = t.size
        if x.size != n or y.size != n:
            raise ValueError("EventSet: coordinate/time length mismatch")
        self._events_key = None  # (a failed load leaves the engine without events)
        self._check(self._lib.sthk_load_events(self._h, _vptr(x), _vptr(y), _vptr(t), n,
                                               float(window_end)), "sthk_load_events")
        self._n = n

    def load(self, events: EventSet) -> None:
        """Load an EventSet unless it is already resident (identity cache)."""
        key = (id(events), events.size(), events.windowEnd())
        if self._events_key == key:
            return
        self.load_events(events.xs(), events.ys(), events.ts(), events.windowEnd())
        self._events_key = key
        self._events_ref = events  # keep alive so id() stays unique

    def set_params(self, params) -> None:
        p = params.as_array() if isinstance(params, Params) else np.asarray(params, np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        self._check(self._lib.sthk_set_params(self._h, _vptr(p)), "sthk_set_params")

    def loglik(self, per_event: bool = False):
        ll, ok = c_double(), c_int()
        pe = np.zeros(self._n) if per_event else None
        self._check(self._lib.sthk_loglik(self._h, byref(ll), byref(ok), _vptr(pe)), "sthk_loglik")
        return ll.value, bool(ok.value), pe

    def loglik_grad(self, per_event: bool = False):
        ll, ok = c_double(), c_int()
        g = np.zeros(6)
        pe = np.zeros(self._n) if per_event else None
        self._check(self._lib.sthk_loglik_grad(self._h, byref(ll), byref(ok), _vptr(g), _vptr(pe)),
                    "sthk_loglik_grad")
        return ll.value, bool(ok.value), g, pe

    def loglik_batch(self, params_list, grad: bool = False):
        P = np.ascontiguousarray(np.asarray(params_list, dtype=np.float64).reshape(-1, 6))
        m = P.shape[0]
        ll = np.zeros(m)
        ok = np.zeros(m, dtype=np.int32)
        g = np.zeros((m, 6)) if grad else None
        self._check(self._lib.sthk_loglik_batch(
            self._h, _dptr(P) if m else None, m, _dptr(ll),
            ok.ctypes.data_as(ctypes.POINTER(c_int)), _dptr(g) if grad else None),
            "sthk_loglik_batch")
        return ll, ok.astype(bool), g

    def excitation(self):
        """(mu, xi, pi) per event for the current params; raises EngineError
        on an underflowed rate (the reference's std::runtime_error)."""
        mu, xi, pi = np.zeros(self._n), np.zeros(self._n), np.zeros(self._n)
        rc = self._lib.sthk_excitation(self._h, _dptr(mu), _dptr(xi), _dptr(pi))
        self._check(rc, "sthk_excitation")
        return mu, xi, pi

    def excitation_batch(self, params_list, sum_pi=None, per_draw: bool = False):
        """pi over S parameter draws in one engine call (sthk_excitation_batch):
        returns (sum_pi, per_draw rows or None, first underflowed draw or -1).
        sum_pi (length n, default zeros) is added to in draw order."""
        P = np.ascontiguousarray(np.asarray(params_list, dtype=np.float64).reshape(-1, 6))
        S = P.shape[0]
        acc = np.zeros(self._n) if sum_pi is None else np.ascontiguousarray(sum_pi, np.float64)
        rows = np.zeros((S, self._n)) if per_draw else None
        bad = ctypes.c_int64(-1)
        rc = self._lib.sthk_excitation_batch(self._h, _dptr(P), S, _dptr(acc),
                                             _dptr(rows) if per_draw else None, byref(bad))
        if rc != _lib.STHK_ERANGE:
            self._check(rc, "sthk_excitation_batch")
        return acc, rows, bad.value

    def enqueue(self, grad: bool = True, per_event: bool = False) -> None:
        self._check(self._lib.sthk_enqueue(self._h, int(grad), int(per_event)), "sthk_enqueue")

    def result(self, per_event: bool = False):
        ll, ok = c_double(), c_int()
        g = np.zeros(6)
        pe = np.zeros(self._n) if per_event else None
        self._check(self._lib.sthk_result(self._h, byref(ll), byref(ok), _vptr(g), _vptr(pe)),
                    "sthk_result")
        return ll.value, bool(ok.value), g, pe

    def set_bgonly_kernel(self, on: bool) -> None:
        """Trigger-free near kernel for stages beyond the trigger window (default on)."""
        self._check(self._lib.sthk_set_bgonly_kernel(self._h, int(on)), "sthk_set_bgonly_kernel")

    def set_far_tier(self, mode) -> None:
        """Far tier of the symmetric kernel (include/sthk.h): True / 1 = FP32 far
        tier (default), 2 = the far list in FP64 (same windows), False / 0 = off."""
        self._check(self._lib.sthk_set_far_tier(self._h, int(mode)), "sthk_set_far_tier")

    def set_far_schedule(self, concurrent: bool, near_ctas: int = 3, far_ctas: int = 6) -> None:
        self._check(self._lib.sthk_set_far_schedule(self._h, int(concurrent), near_ctas, far_ctas),
                    "sthk_set_far_schedule")

    def set_timing(self, on: "bool | int") -> None:
        """0 off, 1 whole evaluation + pair phase, 2 whole evaluation only."""
        self._check(self._lib.sthk_set_timing(self._h, int(on)), "sthk_set_timing")

    def set_graphs(self, on: bool) -> None:
        """One-shard evaluations as cached CUDA graphs (default on)."""
        self._check(self._lib.sthk_set_graphs(self._h, int(on)), "sthk_set_graphs")

    def set_dense(self, on: bool) -> None:
        self._check(self._lib.sthk_set_dense(self._h, int(on)), "sthk_set_dense")

    def set_background_cache(self, on: bool) -> None:
        """Reuse background sums while events/tauX/tauT are unchanged (default on)."""
        self._check(self._lib.sthk_set_background_cache(self._h, int(on)),
                    "sthk_set_background_cache")

    def set_kernel(self, mode: int) -> None:
        """0 = rows (ordered pairs), 1 = symmetric background (default)."""
        self._check(self._lib.sthk_set_kernel(self._h, int(mode)), "sthk_set_kernel")

    def exchange_bytes(self) -> int:
        """Background-sum bytes shipped to other shards' owners by the last evaluation."""
        v = ctypes.c_int64()
        self._check(self._lib.sthk_get_exchange_bytes(self._h, byref(v)), "sthk_get_exchange_bytes")
        return v.value

    def stats(self) -> dict:
        s = _lib.StatsStruct()
        self._check(self._lib.sthk_get_stats(self._h, byref(s)), "sthk_get_stats")
        return {name: getattr(s, name) for name, _ in _lib.StatsStruct._fields_}

    def item_trace(self, slot: int = 0) -> np.ndarray:
        """Development: the last evaluation's pair-kernel work items (needs
        STHK_ITEM_TRACE=<entries> at engine creation), rows of (kernel, sm,
        item, stages, diag, start_ns, end_ns)."""
        cnt = c_int64()
        self._check(self._lib.sthk_debug_item_trace(self._h, slot, None, 0, byref(cnt)),
                    "sthk_debug_item_trace")
        raw = np.zeros((cnt.value, 4), dtype=np.uint64)
        if cnt.value:
            self._check(self._lib.sthk_debug_item_trace(self._h, slot, raw.ctypes.data, cnt.value,
                                                        byref(cnt)), "sthk_debug_item_trace")
        out = np.zeros((len(raw), 7), dtype=np.int64)
        out[:, 0] = (raw[:, 0] >> np.uint64(48)).astype(np.int64)
        out[:, 1] = ((raw[:, 0] >> np.uint64(32)) & np.uint64(0xFFFF)).astype(np.int64)
        out[:, 2] = (raw[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.int64)
        out[:, 3] = (raw[:, 1] >> np.uint64(8)).astype(np.int64)
        out[:, 4] = (raw[:, 1] & np.uint64(0xFF)).astype(np.int64)
        out[:, 5] = raw[:, 2].astype(np.int64)
        out[:, 6] = raw[:, 3].astype(np.int64)
        return out

    def stream(self, slot: int = 0) -> int:
        p = c_void_p()
        self._check(self._lib.sthk_get_stream(self._h, slot, byref(p)), "sthk_get_stream")
        return p.value or 0


_DEFAULT: Optional[Engine] = None
_DEFAULT_LOCK = threading.Lock()


def default_engine() -> Engine:
    global _DEFAULT
    with _DEFAULT_LOCK:
        if _DEFAULT is None:
            _DEFAULT = Engine((0,))
        return _DEFAULT


def logLikelihood(events: EventSet, params: Params, backend=None,
                  keepPerEvent: bool = False, engine: Optional[Engine] = None) -> LikelihoodResult:
    """likelihood.hpp:24-26. `backend` is accepted for signature parity and
    ignored (the device engine replaces the reference's CPU backends)."""
    params.validate()
    eng = engine or default_engine()
    with eng._lock:
        eng.load(events)
        eng.set_params(params)
        ll, ok, pe = eng.loglik(per_event=keepPerEvent)
    return LikelihoodResult(ll, ok, pe if keepPerEvent else np.zeros(0))


def logLikelihoodGradient(events: EventSet, params: Params, backend=None,
                          keepPerEvent: bool = False, engine: Optional[Engine] = None):
    """Log-likelihood plus d logLik / d params in Params order
    (mu0, tauX, tauT, theta, omega, h). grad is NaN when valid is False."""
    params.validate()
    eng = engine or default_engine()
    with eng._lock:
        eng.load(events)
        eng.set_params(params)
        ll, ok, g, pe = eng.loglik_grad(per_event=keepPerEvent)
    return LikelihoodResult(ll, ok, pe if keepPerEvent else np.zeros(0)), g


def logLikelihoodBatch(events: EventSet, paramsList, backend=None, keepPerEvent: bool = False,
                       engine: Optional[Engine] = None):
    """likelihood.cpp:57-75: elementwise identical to repeated calls.
    Without per-event terms the whole batch is one engine call, evaluated
    grouped by (tauX, tauT, omega, h) so entries share the exact sweep caches."""
    if len(paramsList) == 0:
        raise ValueError("logLikelihoodBatch: empty parameter list")
    if not keepPerEvent:
        for i, p in enumerate(paramsList):
            try:
                p.validate()
            except ValueError as e:
                raise ValueError(f"logLikelihoodBatch: entry {i}: {e}") from None
        eng = engine or default_engine()
        with eng._lock:
            eng.load(events)
            ll, ok, _ = eng.loglik_batch([p.as_array() for p in paramsList])
        return [LikelihoodResult(float(v), bool(o), np.zeros(0)) for v, o in zip(ll, ok)]
    out = []
    for i, p in enumerate(paramsList):
        try:
            out.append(logLikelihood(events, p, backend, keepPerEvent, engine))
        except ValueError as e:
            raise ValueError(f"logLikelihoodBatch: entry {i}: {e}") from None
    return out


log_likelihood = logLikelihood
log_likelihood_gradient = logLikelihoodGradient
