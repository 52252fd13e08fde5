"""Thin binding of include/remoe_planner.h (NEXT-N3, the host planner).

Argument marshalling only; the arithmetic is in csrc/planner.cpp inside libremoe.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .sps import RemoeError, lib

PLANNER_FUNCTIONS = (
    "remoe_worst_case_tokens", "remoe_lpt_partition", "remoe_replica_time_bound",
    "remoe_fit_latency_curve", "remoe_convexity_threshold", "remoe_optimize_remote_memory",
    "remoe_mmp", "remoe_greedy_replicas",
)

_f64, _i32, _vp = ctypes.c_double, ctypes.c_int32, ctypes.c_void_p
LOCAL_MEM_FN = ctypes.CFUNCTYPE(_f64, _f64, _vp)
SLO_FN = ctypes.CFUNCTYPE(_i32, _f64, _f64, _vp)
COST_FN = ctypes.CFUNCTYPE(_f64, ctypes.POINTER(_i32), _i32, _vp)
TPOT_FN = ctypes.CFUNCTYPE(_i32, ctypes.POINTER(_i32), _i32, _vp)
_READY = False


def _lib():
    global _READY
    L = lib()
    if not _READY:
        L.remoe_worst_case_tokens.argtypes = [_f64, _i32, _i32]
        L.remoe_worst_case_tokens.restype = _f64
        L.remoe_lpt_partition.argtypes = [_vp, _i32, _i32, _vp, _vp]
        L.remoe_lpt_partition.restype = _f64
        L.remoe_replica_time_bound.argtypes = [_i32, _f64, _f64, _f64, _i32, _f64, _f64]
        L.remoe_replica_time_bound.restype = _f64
        L.remoe_fit_latency_curve.argtypes = [_vp, _vp, _i32, _vp]
        L.remoe_fit_latency_curve.restype = _f64
        L.remoe_convexity_threshold.argtypes = [_f64, _f64, _f64, ctypes.POINTER(_f64),
                                                ctypes.POINTER(_i32)]
        L.remoe_convexity_threshold.restype = None
        L.remoe_optimize_remote_memory.argtypes = [_i32, _vp, _vp, _vp, _f64, _f64, _f64, _f64, _f64,
                                                   _f64, _f64, _vp, _vp]
        L.remoe_optimize_remote_memory.restype = _f64
        L.remoe_mmp.argtypes = [_f64, _f64, _f64, _vp, _i32, LOCAL_MEM_FN, SLO_FN, _vp,
                                ctypes.POINTER(_i32), ctypes.POINTER(_f64), ctypes.POINTER(_f64)]
        L.remoe_mmp.restype = _i32
        L.remoe_greedy_replicas.argtypes = [_i32, _i32, COST_FN, TPOT_FN, _vp, _vp]
        L.remoe_greedy_replicas.restype = _i32
        _READY = True
    return L


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _bad(name):
    raise RemoeError(1, f"{name}: invalid argument")


def remoe_worst_case_tokens(n: float, m: int, K: int) -> float:
    r = _lib().remoe_worst_case_tokens(n, m, K)
    return _bad("remoe_worst_case_tokens") if r < 0 else r


def remoe_lpt_partition(loads, z: int):
    """Returns (assign int32 [n], replica_load fp64 [z], makespan)."""
    loads = _arr(loads, np.float64).ravel()
    assign = np.empty(loads.size, np.int32)
    rl = np.empty(max(z, 1), np.float64)
    r = _lib().remoe_lpt_partition(loads.ctypes.data, loads.size, z, assign.ctypes.data, rl.ctypes.data)
    if r < 0:
        _bad("remoe_lpt_partition")
    return assign, rl, r


def remoe_replica_time_bound(z, tau_nup, two_d_over_b, n_in, K, T_rem, t_rem) -> float:
    r = _lib().remoe_replica_time_bound(z, tau_nup, two_d_over_b, n_in, K, T_rem, t_rem)
    return _bad("remoe_replica_time_bound") if r < 0 else r


def remoe_fit_latency_curve(y, t):
    """Returns (theta fp64 [3], rms)."""
    y = _arr(y, np.float64).ravel()
    t = _arr(t, np.float64).ravel()
    assert y.size == t.size
    th = np.empty(3, np.float64)
    r = _lib().remoe_fit_latency_curve(y.ctypes.data, t.ctypes.data, y.size, th.ctypes.data)
    if r < 0:
        _bad("remoe_fit_latency_curve")
    return th, r


def remoe_convexity_threshold(theta2: float, H: float, c: float):
    """Returns (threshold, convex_everywhere: bool)."""
    thr, ev = _f64(), _i32()
    _lib().remoe_convexity_threshold(theta2, H, c, ctypes.byref(thr), ctypes.byref(ev))
    return thr.value, bool(ev.value)


def remoe_optimize_remote_memory(theta, s_tilde, t_rem, H, c, eta, y_min, y_max, step, budget=-1.0):
    """Returns (P2 at y_grid, y_cont fp64 [L], y_grid fp64 [L]); None if TPOT is infeasible."""
    theta = _arr(theta, np.float64).reshape(-1, 3)
    s = _arr(s_tilde, np.float64).ravel()
    t = _arr(t_rem, np.float64).ravel()
    L = theta.shape[0]
    assert s.size == L and t.size == L
    yc = np.empty(L, np.float64)
    yg = np.empty(L, np.float64)
    r = _lib().remoe_optimize_remote_memory(L, theta.ctypes.data, s.ctypes.data, t.ctypes.data, H, c, eta,
                                            y_min, y_max, step, budget, yc.ctypes.data, yg.ctypes.data)
    if r < 0:
        return None
    return r, yc, yg


def remoe_mmp(M_min, M_cal, epsilon, spec_mem, local_mem, slo_ok):
    """MMP (Alg. 2).  local_mem(b) -> M^e, slo_ok(M, b) -> bool.  Returns (spec, b, M)."""
    spec = _arr(spec_mem, np.float64).ravel()
    cb_mem = LOCAL_MEM_FN(lambda b, _ctx: float(local_mem(b)))
    cb_slo = SLO_FN(lambda M, b, _ctx: 1 if slo_ok(M, b) else 0)
    v, b, M = _i32(), _f64(), _f64()
    st = _lib().remoe_mmp(M_min, M_cal, epsilon, spec.ctypes.data, spec.size, cb_mem, cb_slo, None,
                          ctypes.byref(v), ctypes.byref(b), ctypes.byref(M))
    if st != 0:
        raise RemoeError(st, "remoe_mmp: " + ("infeasible" if st == 5 else "invalid argument"))
    return v.value, b.value, M.value


def remoe_greedy_replicas(z_init, z_max: int, cost, tpot_ok):
    """Greedy replicas by the Eq. 15 potential.  cost(Z) -> float, tpot_ok(Z) -> bool,
    Z a tuple of ints.  Returns the final Z (int32 [L])."""
    Z = _arr(z_init, np.int32).ravel().copy()
    cb_cost = COST_FN(lambda p, L, _ctx: float(cost(tuple(p[i] for i in range(L)))))
    cb_tpot = TPOT_FN(lambda p, L, _ctx: 1 if tpot_ok(tuple(p[i] for i in range(L))) else 0)
    st = _lib().remoe_greedy_replicas(Z.size, z_max, cb_cost, cb_tpot, None, Z.ctypes.data)
    if st != 0:
        raise RemoeError(st, "remoe_greedy_replicas: " + ("infeasible" if st == 5 else "invalid argument"))
    return Z
