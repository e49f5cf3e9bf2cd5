"""Test-side loaders for the parity oracle (oracle/).

  * oracle/libhawkes_oracle.so  -- our long-double C restatement (always built)
  * oracle/_ref/libsthawkes_ref_{v4,v3}.so -- the reference engine compiled
    verbatim from /root/reference (built here, shipped to the GPU box)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int, c_int64, c_uint64

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
REF_DIR = os.path.join(ORACLE_DIR, "_ref")
_D = POINTER(c_double)


def _d(a):
    return None if a is None else a.ctypes.data_as(_D)


def has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return "avx512f" in f.read()
    except OSError:
        return False


_ORACLE = None
_REF = None


def oracle_lib():
    global _ORACLE
    if _ORACLE is None:
        path = os.path.join(ORACLE_DIR, "libhawkes_oracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        lib = ctypes.CDLL(path)
        lib.oracle_loglik_grad.restype = c_int
        lib.oracle_loglik_grad.argtypes = [_D, _D, _D, c_int64, c_double, _D, c_int, _D,
                                           POINTER(c_int), _D, _D, _D, _D]
        lib.oracle_normal_cdf.restype = c_double
        lib.oracle_normal_cdf.argtypes = [c_double]
        _ORACLE = lib
    return _ORACLE


def ref_path() -> str:
    return os.path.join(REF_DIR, "libsthawkes_ref_v4.so" if has_avx512()
                        else "libsthawkes_ref_v3.so")


def ref_available() -> bool:
    return os.path.exists(ref_path())


def ref_lib():
    global _REF
    if _REF is None:
        lib = ctypes.CDLL(ref_path())
        lib.ref_last_error.restype = c_char_p
        lib.ref_loglik.restype = c_int
        lib.ref_loglik.argtypes = [_D, _D, _D, c_int64, c_double, _D, c_int, c_int, _D,
                                   POINTER(c_int), _D]
        lib.ref_time_loglik.restype = c_int
        lib.ref_time_loglik.argtypes = [_D, _D, _D, c_int64, c_double, _D, c_int, c_int, c_int,
                                        c_int, _D, _D]
        lib.ref_hardware_descriptor.restype = c_int
        lib.ref_hardware_descriptor.argtypes = [c_char_p, c_int]
        lib.ref_sim_cloud.restype = c_int
        lib.ref_sim_cloud.argtypes = [c_int64, _D, c_uint64, _D, _D, _D, _D]
        lib.ref_sim_cluster.restype = c_int
        lib.ref_sim_cluster.argtypes = [_D, _D, c_double, c_uint64, c_int64, _D, _D, _D,
                                        POINTER(c_int), POINTER(c_int64)]
        _REF = lib
    return _REF


def oracle_loglik_grad(x, y, t, window_end, params, threads=0, per_event=False, sums=False):
    """Long-double oracle: returns dict(loglik, valid, grad, per_event, sums)."""
    lib = oracle_lib()
    x, y, t = (np.ascontiguousarray(a, np.float64) for a in (x, y, t))
    p = np.ascontiguousarray(params, np.float64)
    n = t.size
    ll, ok = c_double(), c_int()
    g = np.zeros(6)
    pe = np.zeros(n) if per_event else None
    sm = np.zeros(6 * n) if sums else None
    ga = np.zeros(6)
    rc = lib.oracle_loglik_grad(_d(x), _d(y), _d(t), n, float(window_end), _d(p), threads,
                                byref(ll), byref(ok), _d(g), _d(pe), _d(sm), _d(ga))
    if rc != 0:
        raise ValueError("oracle: invalid params")
    return dict(loglik=ll.value, valid=bool(ok.value), grad=g, grad_abs=ga, per_event=pe,
                sums=None if sm is None else sm.reshape(n, 6))


def ref_loglik(x, y, t, window_end, params, threads=1, lanes=1, per_event=False):
    """Verbatim reference hawkes::logLikelihood (serial by default)."""
    lib = ref_lib()
    x, y, t = (np.ascontiguousarray(a, np.float64) for a in (x, y, t))
    p = np.ascontiguousarray(params, np.float64)
    n = t.size
    ll, ok = c_double(), c_int()
    pe = np.zeros(n) if per_event else None
    rc = lib.ref_loglik(_d(x), _d(y), _d(t), n, float(window_end), _d(p), threads, lanes,
                        byref(ll), byref(ok), _d(pe))
    if rc != 0:
        err = lib.ref_last_error().decode()
        raise ValueError(err) if rc == 1 else RuntimeError(err)
    return ll.value, bool(ok.value), pe


def ref_sim_cloud(n, window, seed):
    lib = ref_lib()
    x, y, t = np.zeros(n), np.zeros(n), np.zeros(n)
    we = c_double()
    w = np.asarray(window, np.float64)
    assert lib.ref_sim_cloud(n, _d(w), seed, _d(x), _d(y), _d(t), byref(we)) == 0
    return x, y, t, we.value


def ref_sim_cluster(params, window, rate, seed):
    lib = ref_lib()
    p = np.asarray(params, np.float64)
    w = np.asarray(window, np.float64)
    cnt = c_int64()
    assert lib.ref_sim_cluster(_d(p), _d(w), rate, seed, 0, None, None, None, None,
                               byref(cnt)) == 0
    n = cnt.value
    x, y, t = np.zeros(n), np.zeros(n), np.zeros(n)
    par = np.zeros(n, dtype=np.int32)
    assert lib.ref_sim_cluster(_d(p), _d(w), rate, seed, n, _d(x), _d(y), _d(t),
                               par.ctypes.data_as(POINTER(c_int)), byref(cnt)) == 0
    return x, y, t, par


def ref_time_loglik(x, y, t, window_end, params, threads, lanes, repeats=3, warmups=1):
    lib = ref_lib()
    x, y, t = (np.ascontiguousarray(a, np.float64) for a in (x, y, t))
    p = np.ascontiguousarray(params, np.float64)
    med, mn = c_double(), c_double()
    rc = lib.ref_time_loglik(_d(x), _d(y), _d(t), t.size, float(window_end), _d(p), threads,
                             lanes, repeats, warmups, byref(med), byref(mn))
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return med.value, mn.value


def ref_hardware() -> str:
    buf = ctypes.create_string_buffer(256)
    ref_lib().ref_hardware_descriptor(buf, 256)
    return buf.value.decode()
