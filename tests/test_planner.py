"""NEXT-N3, the host planner (include/remoe_planner.h), pinned against what the paper and
the mathematics fix: the paper's printed values, exact binomial tails, brute-force optima,
Graham's tight LPT family, a library curve fit, and the closed-form g'' of the Theorem 2
proof.  Host-only calls into libremoe.so: no GPU needed."""
import itertools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.usefixtures("remoe_lib_built")


@pytest.fixture(scope="module")
def P():
    import paper_2512_18674_b200 as remoe
    return remoe


# ---------------------------------------------------------------- Theorem 1 / Corollary 1

def test_worst_case_tokens_printed_value(P):
    # n=8, m=1, K=8 -> sqrt(24)/2 + 1 = 3.449490
    assert P.remoe_worst_case_tokens(8, 1, 8) == pytest.approx(3.449490, abs=1e-6)
    assert P.remoe_worst_case_tokens(0, 0, 4) == 0.0
    assert P.remoe_worst_case_tokens(100, 4, 4) == pytest.approx(math.sqrt(300) / 2 + 100)


@pytest.mark.parametrize("args", [(8, 9, 8), (8, -1, 8), (8, 1, 0), (-1, 1, 8)])
def test_worst_case_tokens_rejects(P, args):
    from paper_2512_18674_b200 import RemoeError
    with pytest.raises(RemoeError):
        P.remoe_worst_case_tokens(*args)


def test_worst_case_tokens_95_percent_exact_binomial(P):
    """P:462/467 "with a high probability (95%)": under uniform routing the tokens of m of K
    experts are Binomial(n, m/K).  The exact upper tail beyond the bound is <= 5% for every
    n >= 96 (all K, m swept; the worst case m/K = 1/2 approaches 4.2%); below that the
    integer lattice lets it reach 12.5% (n = 1, K = 8) -- DESIGN.md reading R19."""
    from scipy.stats import binom
    n = np.arange(96, 20001)
    worst = 0.0
    for K in (2, 3, 4, 8, 16, 64, 160):
        for m in sorted({1, K // 4, K // 2, K - 1} - {0}):
            bound = np.array([P.remoe_worst_case_tokens(float(x), m, K) for x in n[::37]])
            assert np.allclose(bound, np.sqrt(3 * n[::37]) / 2 + m * n[::37] / K)
            tail = binom.sf(np.floor(np.sqrt(3 * n) / 2 + m * n / K), n, m / K)   # P(X > bound)
            worst = max(worst, tail.max())
            assert tail.max() <= 0.05, (m, K, n[tail.argmax()], tail.max())
    assert worst > 0.04   # near-tight at m/K = 1/2: the bound is not vacuous
    # the small-n exception the reading records
    assert binom.sf(math.floor(P.remoe_worst_case_tokens(1, 1, 8)), 1, 1 / 8) == pytest.approx(0.125)


# ---------------------------------------------------------------- LPT + Graham

def _opt_makespan(loads, z):
    best = math.inf
    for a in itertools.product(range(z), repeat=len(loads)):
        rl = np.zeros(z)
        np.add.at(rl, list(a), loads)
        best = min(best, rl.max())
    return best


def test_lpt_paper_example(P):
    # SURVEY §8(f) N3 pin: {3,3,2,2,2}, z=2 -> LPT 7, optimum 6 ({3,3},{2,2,2})
    assign, rl, mk = P.remoe_lpt_partition([3, 3, 2, 2, 2], 2)
    assert mk == 7 and sorted(rl) == [5, 7]
    assert _opt_makespan([3, 3, 2, 2, 2], 2) == 6
    assert list(assign[:2]) == [0, 1]     # the two 3s go to different replicas


@pytest.mark.parametrize("z", [2, 3, 4, 5])
def test_lpt_graham_tight_family(P, z):
    """Graham's tight instance (P:619 cites graham1966bounds): loads 2z-1, 2z-1, 2z-2, 2z-2,
    ..., z+1, z+1, z, z, z on z machines: LPT = 4z-1, OPT = 3z, ratio 4/3 - 1/(3z) exactly."""
    loads = [x for x in range(2 * z - 1, z, -1) for _ in (0, 1)] + [z, z, z]
    _, rl, mk = P.remoe_lpt_partition(loads, z)
    assert mk == 4 * z - 1
    assert mk / (3 * z) == pytest.approx(4 / 3 - 1 / (3 * z))
    if z <= 3:
        assert _opt_makespan(loads, z) == 3 * z


def test_lpt_random_vs_brute_force(P):
    rng = np.random.default_rng(7)
    for _ in range(60):
        z = int(rng.integers(1, 4))
        n = int(rng.integers(0, 9))
        loads = rng.integers(1, 20, n).astype(float)
        assign, rl, mk = P.remoe_lpt_partition(loads, z)
        assert np.all((assign >= 0) & (assign < z))
        chk = np.zeros(z)
        np.add.at(chk, assign, loads)
        assert np.allclose(chk, rl) and mk == (rl.max() if n else 0.0)
        if n:
            opt = _opt_makespan(loads, z)
            assert opt <= mk <= (4 / 3 - 1 / (3 * z)) * opt + 1e-9


def test_lpt_rejects(P):
    from paper_2512_18674_b200 import RemoeError
    with pytest.raises(RemoeError):
        P.remoe_lpt_partition([1.0], 0)


# ---------------------------------------------------------------- Theorem 4

def test_replica_time_bound_closed_form(P):
    nup = math.sqrt(3 * 512) / 2 + 512 / 16
    assert P.remoe_replica_time_bound(4, 2.0, 0.01, 512, 16, 40.0, 1.5) == pytest.approx(
        3 / 4 * (2.0 + 0.01 * nup) + 40.0 / 4 + 1.5)
    # one replica runs everything: T_rem + t_rem
    assert P.remoe_replica_time_bound(1, 2.0, 0.01, 512, 16, 40.0, 1.5) == pytest.approx(41.5)


def test_replica_time_bound_holds_95_percent_monte_carlo(P):
    """Simulate Theorem 4's setting: N_in tokens routed uniformly over K experts,
    expert k's remote prefill time tau(N_k) + 2D/B N_k with tau affine, the tasks split over
    z replicas by LPT; the slowest replica stays within the bound in >= 95% of trials."""
    rng = np.random.default_rng(11)
    n_in, K, alpha, beta, two_d_b, t_rem = 1024, 16, 0.5, 0.01, 0.002, 0.3
    for z in (2, 3, 4):
        fails = 0
        trials = 400
        for _ in range(trials):
            N = rng.multinomial(n_in, [1 / K] * K)
            tasks = alpha + beta * N + two_d_b * N
            _, _, mk = P.remoe_lpt_partition(tasks, z)
            nup = P.remoe_worst_case_tokens(n_in, 1, K)
            bound = P.remoe_replica_time_bound(z, alpha + beta * nup, two_d_b, n_in, K, tasks.sum(), 0.0)
            fails += (mk + t_rem) > bound + t_rem
        assert fails / trials <= 0.05, (z, fails)


# ---------------------------------------------------------------- latency model fit

def test_fit_recovers_noise_free_curve(P):
    th = np.array([2.0, 2.4363, 0.3])        # theta_2 of Deepseek-v2-lite
    y = np.linspace(0.25, 4.0, 16)
    t = th[0] * np.exp(-th[1] * y) + th[2]
    got, rms = P.remoe_fit_latency_curve(y, t)
    assert rms < 1e-9
    assert np.allclose(got, th, rtol=1e-6)


def test_fit_matches_scipy_curve_fit_on_noisy_data(P):
    from scipy.optimize import curve_fit
    rng = np.random.default_rng(3)
    th = np.array([5.0, 11.8665, 1.2])       # theta_2 of GPT2-moe
    y = np.linspace(0.05, 1.0, 24)
    t = (th[0] * np.exp(-th[1] * y) + th[2]) * (1 + 0.005 * rng.standard_normal(y.size))
    got, rms = P.remoe_fit_latency_curve(y, t)
    ref, _ = curve_fit(lambda x, a, b, c: a * np.exp(-b * x) + c, y, t, p0=th)
    r_ref = np.sqrt(np.mean((ref[0] * np.exp(-ref[1] * y) + ref[2] - t) ** 2))
    assert rms <= r_ref * (1 + 1e-6)
    assert np.allclose(got, ref, rtol=1e-3)


# ---------------------------------------------------------------- Theorem 2

def test_convexity_paper_regimes(P):
    # 2c^c/H^w ~ 0.25 << 2.4363 (Deepseek-v2-lite), ~2.72 << 11.8665 (GPT2-moe)
    for two_c_over_h, theta2 in ((0.25, 2.4363), (2.72, 11.8665)):
        thr, ev = P.remoe_convexity_threshold(theta2, 2.0, two_c_over_h)
        assert ev and thr <= 0
    thr, ev = P.remoe_convexity_threshold(0.2, 2.0, 0.25)   # theta_2 < 2c/H
    assert not ev and thr == pytest.approx(2 / 0.2 - 8.0)


def test_convexity_threshold_is_the_sign_change_of_g2(P):
    """g'' by central differences of g(y) = (T(y) + t/s)(H + c y) changes sign exactly at the
    threshold (zero of the proof's g'' = c th1 th2^2 e^{-th2 y} [y - thr])."""
    th1, th2, th3, t, s, H, c = 3.0, 0.5, 0.2, 0.4, 0.8, 1.0, 1.5
    thr, ev = P.remoe_convexity_threshold(th2, H, c)
    assert not ev and thr > 0

    def g(y):
        return (th1 * np.exp(-th2 * y) + th3 + t / s) * (H + c * y)
    h = 1e-3
    for y in np.linspace(0.05, 3 * thr, 40):
        d2 = (g(y + h) - 2 * g(y) + g(y - h)) / h ** 2
        closed = c * th1 * th2 ** 2 * np.exp(-th2 * y) * (y - thr)
        assert d2 == pytest.approx(closed, abs=1e-5)
        if abs(y - thr) > 1e-2:
            assert (d2 > 0) == (y > thr)


# ---------------------------------------------------------------- P_2 via the dual

def _p2(theta, s, t, H, c, eta, y):
    T = theta[:, 0] * np.exp(-theta[:, 1] * y) + theta[:, 2]
    return (1 + eta) * np.sum(s * (T + t / s) * (H + c * y), axis=-1)


def test_memory_single_layer_vs_dense_scan(P):
    theta = np.array([[2.0, 2.4363, 0.3]])
    s, t, H, c, eta = np.array([0.4]), np.array([0.05]), 4.0, 1.0, 0.1
    val, yc, yg = P.remoe_optimize_remote_memory(theta, s, t, H, c, eta, 0.125, 8.0, 0.125)
    ys = np.linspace(0.125, 8.0, 200001)
    dense = _p2(theta, s, t, H, c, eta, ys[:, None])
    assert _p2(theta, s, t, H, c, eta, yc) == pytest.approx(dense.min(), rel=1e-9)
    assert abs(yc[0] - ys[dense.argmin()]) < 1e-3
    assert yg[0] >= yc[0] - 1e-12 and yg[0] - yc[0] < 0.125 + 1e-12
    assert round((yg[0] - 0.125) / 0.125, 9) == int(round((yg[0] - 0.125) / 0.125))
    assert val == pytest.approx(_p2(theta, s, t, H, c, eta, yg))


def test_memory_tpot_coupled_vs_brute_force(P):
    """Three layers, the TPOT constraint binding: the dual solution's continuous optimum is
    no worse than any feasible point of a brute-force grid, is feasible, and sits on the
    constraint (complementary slackness); the rounded-up grid solution stays feasible."""
    theta = np.array([[3.0, 1.2, 0.2], [2.0, 2.4363, 0.1], [4.0, 0.8, 0.3]])
    s = np.array([0.5, 0.3, 0.7])
    t = np.array([0.05, 0.02, 0.08])
    H, c, eta, lo, hi, step = 6.0, 1.0, 0.1, 0.25, 6.0, 0.25
    free = P.remoe_optimize_remote_memory(theta, s, t, H, c, eta, lo, hi, step)
    used_free = np.sum(s * (theta[:, 0] * np.exp(-theta[:, 1] * free[1]) + theta[:, 2]))
    at_max = np.sum(s * (theta[:, 0] * np.exp(-theta[:, 1] * hi) + theta[:, 2]))
    budget = 0.5 * (used_free + at_max)
    val, yc, yg = P.remoe_optimize_remote_memory(theta, s, t, H, c, eta, lo, hi, step, budget)

    def used(y):
        return np.sum(s * (theta[:, 0] * np.exp(-theta[:, 1] * y) + theta[:, 2]), axis=-1)
    assert used(yc) == pytest.approx(budget, rel=1e-6)
    assert used(yg) <= budget + 1e-12
    g = np.linspace(lo, hi, 47)
    Y = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    feas = used(Y) <= budget
    best = _p2(theta, s, t, H, c, eta, Y[feas]).min()
    assert _p2(theta, s, t, H, c, eta, yc) <= best + 1e-9
    assert val == pytest.approx(_p2(theta, s, t, H, c, eta, yg))
    assert val >= _p2(theta, s, t, H, c, eta, yc) - 1e-12
    # infeasible even at y_max -> None
    assert P.remoe_optimize_remote_memory(theta, s, t, H, c, eta, lo, hi, step, used(np.full(3, hi)) * 0.99) is None


# ---------------------------------------------------------------- MMP (Alg. 2)

def test_mmp_hand_example(P):
    """A serving model where TTFT/TPOT hold iff b <= 0.3 and local experts cost 40(1-b) GB:
    b steps 1, 0.875, ..., the first passing ratio is 0.25, M = max(10 + 30, 35) = 40,
    the smallest spec >= 40 among {16, 32, 48, 64} is index 2 (Alg. 2 lines 2-13)."""
    v, b, M = P.remoe_mmp(10.0, 35.0, 0.125, [16, 32, 48, 64], lambda b: 40 * (1 - b),
                          lambda M, b: b <= 0.3)
    assert (v, b, M) == (2, 0.25, 40.0)
    # M_cal dominates when the local experts are small
    v, b, M = P.remoe_mmp(10.0, 35.0, 0.125, [16, 32, 48, 64], lambda b: 4 * (1 - b),
                          lambda M, b: True)
    assert (v, b, M) == (2, 1.0, 35.0)


def test_mmp_infeasible(P):
    from paper_2512_18674_b200 import RemoeError
    with pytest.raises(RemoeError):   # SLO never met
        P.remoe_mmp(10.0, 0.0, 0.25, [64], lambda b: 0.0, lambda M, b: False)
    with pytest.raises(RemoeError):   # no specification large enough
        P.remoe_mmp(100.0, 0.0, 0.25, [16, 32], lambda b: 0.0, lambda M, b: True)


# ---------------------------------------------------------------- greedy replicas (Eq. 15)

def test_greedy_replicas_separable_convex_is_optimal(P):
    """For a separable cost sum_l (a_l / z_l + c_l z_l) (convex in each z_l), the Eq. 15
    greedy from z = 1 reaches the exhaustive optimum over [1, z_max]^L."""
    a = np.array([12.0, 3.0, 30.0])
    cc = np.array([1.0, 1.0, 0.5])
    zmax = 6

    def cost(Z):
        Z = np.asarray(Z, float)
        return float(np.sum(a / Z + cc * Z))
    Z = P.remoe_greedy_replicas([1, 1, 1], zmax, cost, lambda Z: True)
    best = min(itertools.product(range(1, zmax + 1), repeat=3), key=cost)
    assert cost(Z) == pytest.approx(cost(best))
    assert tuple(Z) == best


def test_greedy_replicas_meets_slo_and_caps(P):
    """Hand trace of P:640-647 with C(Z) = sum_l (a_l / z_l + 2 z_l), a = (12, 3, 30), and the
    SLO max_l a_l / z_l <= 6.  Potentials varpi (Eq. 15) at each step, the greatest wins
    (equal: lower l):
      (1,1,1): (4, -0.5, 13)    -> l2      (1,1,2): (4, -0.5, 3)   -> l0
      (2,1,2): (0, -0.5, 3)     -> l2      (2,1,3): (0, -0.5, 0.5) -> l2
      (2,1,4): (0, -0.5, -0.5)  -> l0      (3,1,4): (-1, -0.5, -0.5) -> l1
      (3,2,4): (-1, -1.5, -0.5) -> l2      (3,2,5): SLO holds, every varpi <= 0: stop."""
    from paper_2512_18674_b200 import RemoeError
    a = np.array([12.0, 3.0, 30.0])

    def cost(Z):
        Z = np.asarray(Z, float)
        return float(np.sum(a / Z + 2.0 * Z))

    def slo(Z):
        return np.max(a / np.asarray(Z, float)) <= 6
    Z = P.remoe_greedy_replicas([1, 1, 1], 8, cost, slo)
    assert tuple(Z) == (3, 2, 5)
    # without the SLO the same greedy stops at the cost optimum (2, 1, 4)
    assert tuple(P.remoe_greedy_replicas([1, 1, 1], 8, cost, lambda Z: True)) == (2, 1, 4)
    # z_max too small for the SLO: infeasible
    with pytest.raises(RemoeError):
        P.remoe_greedy_replicas([1, 1, 1], 4, cost, slo)
    with pytest.raises(RemoeError):   # z_init outside [1, z_max]
        P.remoe_greedy_replicas([0, 1, 1], 4, cost, slo)
