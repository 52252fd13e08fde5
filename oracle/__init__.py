"""Oracle: plain CPU definition of the SPS hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  The product
path (paper_2512_18674_b200) never imports it, and it imports nothing from the
product path: the two share no code.  The only shared module is ``gen`` (seeded
inputs, no method arithmetic).

Parity pins live in tests/test_oracle_pins.py; every function below is pinned
there.  ``oracle.tree`` (NEXT-N2, the clustering tree and
Algorithm 1) is pinned in tests/test_tree_oracle.py.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .scs import normalize_rows, prompt_vector, scs_gram  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SIGMA = 1e-6        # Eq. 11 guard ("extremely small"; reading R3)
TEMPERATURE = 1.0   # softmax temperature (PAPER.md:421 gives none; reading R4)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` first")
        lib = ctypes.CDLL(path)
        i64, i32, f64, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        lib.oracle_sps_bf16.argtypes = [vp, i64, vp, i64, i32, vp, i32, i32, f64, f64, i64, i64,
                                        vp, vp, vp, i32]
        lib.oracle_sps_f64.argtypes = lib.oracle_sps_bf16.argtypes
        lib.oracle_scores_bf16.argtypes = [vp, i64, vp, i64, i32, f64, vp, i32]
        lib.oracle_pair_scores_bf16.argtypes = [vp, vp, i32, vp, vp, i64, f64, vp]
        lib.oracle_select.argtypes = [vp, i64, i64, i64, vp, vp]
        lib.oracle_softmax.argtypes = [vp, i64, f64, vp]
        lib.oracle_predict.argtypes = [vp, vp, i64, vp, i64, i64, i64, vp]
        lib.oracle_plan.argtypes = [vp, i64, i32, i32, i32, vp]
        lib.oracle_widen_bf16.argtypes = [vp, i64, vp]
        lib.oracle_js_divergence.argtypes = [vp, vp, i32, i32]
        lib.oracle_js_divergence.restype = f64
        for f in ("oracle_sps_bf16", "oracle_sps_f64", "oracle_scores_bf16",
                  "oracle_pair_scores_bf16", "oracle_select", "oracle_softmax",
                  "oracle_predict", "oracle_plan"):
            getattr(lib, f).restype = i32
        _LIB = lib
    return _LIB


def _threads(n: int | None) -> int:
    return n if n else max(1, os.cpu_count() or 1)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def widen(bits: np.ndarray) -> np.ndarray:
    """Step 1: bf16 bits -> fp64, exact."""
    b = _c(bits, np.uint16)
    out = np.empty(b.shape, dtype=np.float64)
    _lib().oracle_widen_bf16(b.ctypes.data, b.size, out.ctypes.data)
    return out


def sps(q_bits, x_bits, act, k, sigma=SIGMA, temperature=TEMPERATURE, id_offset=0,
        want_pred=True, nthreads=None):
    """Steps 1-6 on bf16 inputs.  Returns ids int64 [B,k], scores fp64 [B,k], pred fp64 [B,L,E]."""
    q = _c(q_bits, np.uint16)
    x = _c(x_bits, np.uint16)
    B, D = q.shape
    N = x.shape[0]
    assert x.shape[1] == D
    a = _c(act, np.float32)
    L, E = a.shape[1], a.shape[2]
    ids = np.empty((B, k), np.int64)
    sc = np.empty((B, k), np.float64)
    pred = np.empty((B, L, E), np.float64) if want_pred else None
    rc = _lib().oracle_sps_bf16(q.ctypes.data, B, x.ctypes.data, N, D, a.ctypes.data, L, E,
                                sigma, temperature, k, id_offset, ids.ctypes.data, sc.ctypes.data,
                                pred.ctypes.data if want_pred else None, _threads(nthreads))
    if rc:
        raise ValueError(f"oracle_sps_bf16 failed ({rc})")
    return ids, sc, pred


def sps_f64(q, x, act, k, sigma=SIGMA, temperature=TEMPERATURE, id_offset=0, nthreads=None):
    """Steps 2-6 on real-valued (fp64) prompt vectors."""
    q = _c(q, np.float64)
    x = _c(x, np.float64)
    B, D = q.shape
    N = x.shape[0]
    a = _c(act, np.float32)
    L, E = a.shape[1], a.shape[2]
    ids = np.empty((B, k), np.int64)
    sc = np.empty((B, k), np.float64)
    pred = np.empty((B, L, E), np.float64)
    rc = _lib().oracle_sps_f64(q.ctypes.data, B, x.ctypes.data, N, D, a.ctypes.data, L, E, sigma,
                               temperature, k, id_offset, ids.ctypes.data, sc.ctypes.data,
                               pred.ctypes.data, _threads(nthreads))
    if rc:
        raise ValueError(f"oracle_sps_f64 failed ({rc})")
    return ids, sc, pred


def scores(q_bits, x_bits, sigma=SIGMA, nthreads=None) -> np.ndarray:
    """Step 3 for every (query, row): fp64 [B, N]."""
    q = _c(q_bits, np.uint16)
    x = _c(x_bits, np.uint16)
    out = np.empty((q.shape[0], x.shape[0]), np.float64)
    rc = _lib().oracle_scores_bf16(q.ctypes.data, q.shape[0], x.ctypes.data, x.shape[0],
                                   q.shape[1], sigma, out.ctypes.data, _threads(nthreads))
    if rc:
        raise ValueError(f"oracle_scores_bf16 failed ({rc})")
    return out


def pair_scores(q_bits, x_bits, qi, rows, sigma=SIGMA) -> np.ndarray:
    """Step 3 for explicit pairs (query qi[p], store row rows[p])."""
    q = _c(q_bits, np.uint16)
    x = _c(x_bits, np.uint16)
    qi = _c(qi, np.int64).ravel()
    rows = _c(rows, np.int64).ravel()
    out = np.empty(qi.shape[0], np.float64)
    rc = _lib().oracle_pair_scores_bf16(q.ctypes.data, x.ctypes.data, q.shape[1], qi.ctypes.data,
                                        rows.ctypes.data, qi.shape[0], sigma, out.ctypes.data)
    if rc:
        raise ValueError("oracle_pair_scores_bf16 failed")
    return out


def select(s, k, id_offset=0):
    """Step 4 on one score vector: (ids int64 [k], scores fp64 [k])."""
    s = _c(s, np.float64)
    ids = np.empty(k, np.int64)
    top = np.empty(k, np.float64)
    rc = _lib().oracle_select(s.ctypes.data, s.shape[0], k, id_offset, ids.ctypes.data,
                              top.ctypes.data)
    if rc:
        raise ValueError("oracle_select failed (k out of range)")
    return ids, top


def softmax(s, temperature=TEMPERATURE) -> np.ndarray:
    """Step 5: softmax weights of the retrieved scores."""
    s = _c(s, np.float64)
    w = np.empty_like(s)
    rc = _lib().oracle_softmax(s.ctypes.data, s.shape[0], temperature, w.ctypes.data)
    if rc:
        raise ValueError("oracle_softmax failed")
    return w


def predict(ids, w, act, id_offset=0) -> np.ndarray:
    """Step 6: weighted sum of the retrieved activation matrices, fp64 [L, E]."""
    ids = _c(ids, np.int64)
    w = _c(w, np.float64)
    a = _c(act, np.float32)
    L, E = a.shape[1], a.shape[2]
    out = np.empty((L, E), np.float64)
    rc = _lib().oracle_predict(ids.ctypes.data, w.ctypes.data, ids.shape[0], a.ctypes.data,
                               id_offset, a.shape[0], L * E, out.ctypes.data)
    if rc:
        raise ValueError("oracle_predict failed (id outside table)")
    return out


def plan(pred, n_cold) -> np.ndarray:
    """Step 7: uint8 cold mask [B, L, E] (1 = remote)."""
    p = _c(pred, np.float64)
    if p.ndim == 2:
        p = p[None]
    B, L, E = p.shape
    mask = np.empty((B, L, E), np.uint8)
    rc = _lib().oracle_plan(p.ctypes.data, B, L, E, n_cold, mask.ctypes.data)
    if rc:
        raise ValueError("oracle_plan failed (n_cold out of range)")
    return mask


def js_divergence(p, q) -> float:
    """NEXT-N4: base-2 Jensen-Shannon divergence of two [L, E] activation matrices, mean over
    layers."""
    p = _c(p, np.float64)
    q = _c(q, np.float64)
    if p.ndim == 1:
        p, q = p[None], q[None]
    assert p.shape == q.shape
    return float(_lib().oracle_js_divergence(p.ctypes.data, q.ctypes.data, p.shape[0], p.shape[1]))
