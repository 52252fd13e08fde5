"""The GPU-vs-oracle parity protocol (SURVEY.md §8(c) 'Parity protocol').

* ids: the GPU set may differ from the oracle set only by ids whose oracle score
  is within `tol` (BASELINE 1e-4) AND within the tight window `tight` (1e-5) of the
  oracle's k-th score; positions may swap only between ids whose oracle scores are
  within `tight` of each other.  The tight window is SURVEY §8(c)'s internal check: a
  1e-4 window alone would pass a top-k that returns the (k+1)-th row instead of the
  k-th on about half of the clustered queries, while a genuine fp32 rounding swap needs
  a gap of ~2e-6.  Every run counts the substitutions (`substitutions`) and the
  oracle-only boundary near-tie rate (`boundary_ties`: queries where another row lies
  within `tol` of the k-th score).
* scores: each GPU score vs the ORACLE score of the same id, |d| <= tol, and the
  internal tight window |d| <= tight.
* pred: vs the oracle prediction (re-derived on the GPU's id set, with oracle
  scores, when near-tie substitutions happened), |d| <= tol elementwise.
Tolerances: BASELINE.json north_star (1e-4); tight window 1e-5 (10x the
measured accumulation error, SURVEY §8(c) 'Error budget') for D <= 1024 -- every BASELINE
config -- and 1e-5 * D / 1024 above (R29): the fp32 accumulation bound
gamma_D ~ D * 2^-24 grows linearly in D, and a D = 4096 exact copy measured 1.09e-5 on
the tensor cores.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import oracle

TOL = 1e-4
TIGHT = 1e-5


def tight_for(dim: int) -> float:
    """The tight window for a D-dimensional dot product (R29): 1e-5 up to D = 1024, then linear in D."""
    return TIGHT * max(1.0, dim / 1024.0)


@dataclass
class ParityReport:
    queries: int = 0
    substitutions: int = 0
    boundary_ties: int = 0
    max_score_err: float = 0.0
    max_pred_err: float = 0.0
    failures: list = field(default_factory=list)

    def ok(self):
        return not self.failures

    def summary(self):
        return (f"{self.queries} queries: {self.substitutions} near-tie substitutions, "
                f"{self.boundary_ties} oracle boundary near-ties (1e-4), "
                f"max |dscore| {self.max_score_err:.2e}, max |dpred| {self.max_pred_err:.2e}")


def compare(q_bits, x_bits, act, k, gpu_ids, gpu_scores, gpu_pred=None, *, sigma=oracle.SIGMA,
            id_offset=0, oracle_out=None, tol=TOL, tight=None, exact_ids=False) -> ParityReport:
    """q_bits [B,D] uint16, x_bits [N,D] uint16 (rows with global ids id_offset + j)."""
    if tight is None:
        tight = tight_for(q_bits.shape[1])
    gpu_ids = np.asarray(gpu_ids)
    gpu_scores = np.asarray(gpu_scores, np.float64)
    B = q_bits.shape[0]
    if oracle_out is None:
        # one extra column (k + 1) gives the boundary near-tie rate for free
        kk = k + 1 if k < x_bits.shape[0] else k
        oracle_out = oracle.sps(q_bits, x_bits, act, kk, sigma=sigma, id_offset=id_offset,
                                want_pred=False)
        o_pred = None
        if gpu_pred is not None:
            o_pred = np.stack([oracle.predict(oracle_out[0][i, :k], oracle.softmax(oracle_out[1][i, :k]),
                                              act, id_offset=id_offset) for i in range(B)])
        oracle_out = (oracle_out[0], oracle_out[1], o_pred)
    o_ids, o_sc, o_pred = oracle_out
    rep = ParityReport(queries=B)
    if o_ids.shape[1] == k + 1:  # oracle run with k + 1: the (k+1)-th score is known
        rep.boundary_ties = int(np.sum(np.abs(o_sc[:, k] - o_sc[:, k - 1]) <= tol))
        o_ids, o_sc = o_ids[:, :k], o_sc[:, :k]
    qi = np.repeat(np.arange(B), k)
    rows = gpu_ids.reshape(-1) - id_offset
    if rows.min() < 0 or rows.max() >= x_bits.shape[0]:
        rep.failures.append("GPU id outside the store")
        return rep
    s_of_gpu = oracle.pair_scores(q_bits, x_bits, qi, rows, sigma=sigma).reshape(B, k)
    for i in range(B):
        sk = o_sc[i, k - 1]
        gset, oset = set(gpu_ids[i].tolist()), set(o_ids[i].tolist())
        if len(gset) != k:
            rep.failures.append(f"q{i}: duplicate ids {gpu_ids[i].tolist()}")
            continue
        if gset != oset:
            extra = gset - oset
            missing = oset - gset
            rep.substitutions += len(extra)
            if exact_ids:
                rep.failures.append(f"q{i}: id sets differ (exact required): +{extra} -{missing}")
            win = min(tol, tight)
            for r in range(k):
                if gpu_ids[i, r] in extra and abs(s_of_gpu[i, r] - sk) > win:
                    rep.failures.append(f"q{i}: GPU id {gpu_ids[i, r]} (oracle score {s_of_gpu[i, r]:.8f})"
                                        f" not within {win} of the k-th score {sk:.8f}")
            for r in range(k):
                if o_ids[i, r] in missing and abs(o_sc[i, r] - sk) > win:
                    rep.failures.append(f"q{i}: oracle id {o_ids[i, r]} missing and not a near tie"
                                        f" (within {win})")
        # order: any inversion (by oracle score) must be a near tie (tight window)
        for r in range(k - 1):
            if s_of_gpu[i, r] < s_of_gpu[i, r + 1] - min(tol, tight):
                rep.failures.append(f"q{i}: order inversion at {r} beyond {min(tol, tight)}")
        # the GPU's own list must be sorted by its own key (score desc, id asc)
        for r in range(k - 1):
            a, b = gpu_scores[i, r], gpu_scores[i, r + 1]
            if a < b or (a == b and gpu_ids[i, r] > gpu_ids[i, r + 1]):
                rep.failures.append(f"q{i}: GPU list not in key order at {r}")
        err = np.abs(gpu_scores[i] - s_of_gpu[i]).max()
        rep.max_score_err = max(rep.max_score_err, float(err))
        if err > tol:
            rep.failures.append(f"q{i}: score error {err:.3e} > {tol}")
        if err > tight:
            rep.failures.append(f"q{i}: score error {err:.3e} > tight window {tight}")
        if gpu_pred is not None:
            if gset == oset and list(gpu_ids[i]) == list(o_ids[i]):
                ref = o_pred[i]
            else:
                w = oracle.softmax(s_of_gpu[i])
                ref = oracle.predict(gpu_ids[i], w, act, id_offset=id_offset)
            perr = float(np.abs(np.asarray(gpu_pred[i], np.float64) - ref).max())
            rep.max_pred_err = max(rep.max_pred_err, perr)
            if perr > tol:
                rep.failures.append(f"q{i}: pred error {perr:.3e} > {tol}")
    return rep


def oracle_run(q_bits, x_bits, act, k, *, sigma=oracle.SIGMA, id_offset=0, want_pred=True):
    """The oracle's top-(k+1) (for the boundary near-tie count) with the prediction of its
    top-k: the tuple `compare(..., oracle_out=...)` takes."""
    kk = k + 1 if k < x_bits.shape[0] else k
    ids, sc, _ = oracle.sps(q_bits, x_bits, act, kk, sigma=sigma, id_offset=id_offset, want_pred=False)
    pred = None
    if want_pred:
        pred = np.stack([oracle.predict(ids[i, :k], oracle.softmax(sc[i, :k]), act, id_offset=id_offset)
                         for i in range(q_bits.shape[0])])
    return ids, sc, pred


def take(oracle_out, rows):
    """Rows of an oracle_run result (pred may be None)."""
    return tuple(None if v is None else v[rows] for v in oracle_out)


def log_report(name, rep):
    """Append one parity report line to $REMOE_PARITY_LOG (GPU runs keep it under profiles/)."""
    import json
    import os
    print(f"[parity] {name}: {rep.summary()}")
    path = os.environ.get("REMOE_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, "queries": rep.queries, "substitutions": rep.substitutions,
                                "boundary_ties_1e-4": rep.boundary_ties, "max_score_err": rep.max_score_err,
                                "max_pred_err": rep.max_pred_err, "ok": rep.ok()}) + "\n")


def plan_compare(pred_oracle, gpu_mask, n_cold, tol=TOL):
    """Masks equal except where the oracle value is within tol of the n_cold boundary."""
    p = np.asarray(pred_oracle, np.float64)
    m = np.asarray(gpu_mask)
    o = oracle.plan(p, n_cold)
    bad = []
    B, L, E = p.shape
    for i in range(B):
        for l in range(L):
            if np.array_equal(o[i, l], m[i, l]):
                continue
            if m[i, l].sum() != n_cold:
                bad.append((i, l, "count"))
                continue
            srt = np.sort(p[i, l])
            lo = srt[n_cold - 1] if n_cold > 0 else -np.inf
            hi = srt[n_cold] if n_cold < E else np.inf
            diff = np.nonzero(o[i, l] != m[i, l])[0]
            for e in diff:
                if not (abs(p[i, l, e] - lo) <= tol or abs(p[i, l, e] - hi) <= tol):
                    bad.append((i, l, int(e)))
    return bad
