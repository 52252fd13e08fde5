// planner.cpp -- NEXT-N3: the host-side consumers of the predicted activation matrix
// (§IV-C..F; API and citations in include/remoe_planner.h).  Plain C++:
//   * Theorem 1 / Corollary 1 worst-case token count;
//   * MMP, Algorithm 2, over a caller-supplied serving model;
//   * LPT multiway partition of remote experts over replicas;
//   * Theorem 4 replica-time bound;
//   * greedy replicas by the Eq. 15 potential, caller-supplied cost;
//   * the latency model T(y) = th1 exp(-th2 y) + th3 and its fit;
//   * Theorem 2 convexity threshold of g(y);
//   * P_2 through its Lagrangian dual, rounded up to the grid.
// The remote-expert selection itself runs on the GPU (remoe_expert_plan).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "remoe_planner.h"

namespace {

double t_model(const double* th, double y) { return th[0] * std::exp(-th[1] * y) + th[2]; }

// g(y) = (T(y) + t/s) (H + c y)  (Theorem 2), plus lam * T(y) for the TPOT multiplier.
double layer_obj(const double* th, double s, double t, double H, double c, double lam, double y) {
  const double T = t_model(th, y);
  return s * (T + t / s) * (H + c * y) + lam * s * T;
}

// Minimise a function that is convex on [lo, hi] (golden section, 200 iterations).
template <typename F>
double argmin_convex(F f, double lo, double hi) {
  const double r = 0.6180339887498949;
  double a = lo, b = hi;
  double x1 = b - r * (b - a), x2 = a + r * (b - a);
  double f1 = f(x1), f2 = f(x2);
  for (int it = 0; it < 200 && b - a > 1e-12 * (1.0 + std::fabs(a) + std::fabs(b)); ++it) {
    if (f1 <= f2) { b = x2; x2 = x1; f2 = f1; x1 = b - r * (b - a); f1 = f(x1); }
    else          { a = x1; x1 = x2; f1 = f2; x2 = a + r * (b - a); f2 = f(x2); }
  }
  const double m = 0.5 * (a + b);
  // the ends are candidates too (constrained optimum on the boundary)
  double best = m, fb = f(m);
  if (f(lo) < fb) { best = lo; fb = f(lo); }
  if (f(hi) < fb) { best = hi; }
  return best;
}

}  // namespace

extern "C" {

// Corollary 1: sqrt(3n)/2 + m n / K (Theorem 1 is m = 1).  Returns -1 on bad input.
double remoe_worst_case_tokens(double n, int32_t m, int32_t K) {
  if (n < 0 || K < 1 || m < 0 || m > K) return -1.0;
  return std::sqrt(3.0 * n) / 2.0 + (double)m * n / (double)K;
}

// LPT: tasks sorted by load descending (ties: lower index first), each assigned to
// the currently least-loaded replica (ties: lower replica index).  assign[i] = replica of
// task i; replica_load[z]; returns the makespan (max replica load), -1 on bad input.
double remoe_lpt_partition(const double* loads, int32_t n, int32_t z, int32_t* assign,
                           double* replica_load) {
  if (n < 0 || z < 1 || (n > 0 && (!loads || !assign))) return -1.0;
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return loads[a] > loads[b]; });
  std::vector<double> rl(z, 0.0);
  for (int i : order) {
    int best = 0;
    for (int j = 1; j < z; ++j)
      if (rl[j] < rl[best]) best = j;
    assign[i] = best;
    rl[best] += loads[i];
  }
  if (replica_load) std::memcpy(replica_load, rl.data(), sizeof(double) * z);
  return z ? *std::max_element(rl.begin(), rl.end()) : 0.0;
}

// Theorem 4: (z-1)/z [tau(N_up) + 2D/B N_up] + T_rem / z + t_rem, with
// N_up = sqrt(3 n_in)/2 + n_in / K.
double remoe_replica_time_bound(int32_t z, double tau_nup, double two_d_over_b, double n_in, int32_t K,
                                double T_rem, double t_rem) {
  if (z < 1 || K < 1) return -1.0;
  const double nup = std::sqrt(3.0 * n_in) / 2.0 + n_in / (double)K;
  return (double)(z - 1) / z * (tau_nup + two_d_over_b * nup) + T_rem / z + t_rem;
}

// Fit T(y) = th1 exp(-th2 y) + th3 by least squares: for fixed th2 the model is
// linear in (th1, th3), solved exactly; th2 by golden section on log th2 in [1e-4, 1e3].
// Returns the RMS residual (-1 on bad input).
double remoe_fit_latency_curve(const double* y, const double* t, int32_t n, double* theta) {
  if (n < 3 || !y || !t || !theta) return -1.0;
  auto solve = [&](double th2, double* out) {
    double sxx = 0, sx = 0, sxt = 0, st = 0;
    for (int i = 0; i < n; ++i) {
      const double x = std::exp(-th2 * y[i]);
      sxx += x * x; sx += x; sxt += x * t[i]; st += t[i];
    }
    const double det = n * sxx - sx * sx;
    double a = det != 0 ? (n * sxt - sx * st) / det : 0.0;
    double c = (st - a * sx) / n;
    double r = 0;
    for (int i = 0; i < n; ++i) {
      const double e = a * std::exp(-th2 * y[i]) + c - t[i];
      r += e * e;
    }
    if (out) { out[0] = a; out[1] = th2; out[2] = c; }
    return r;
  };
  const double lg = argmin_convex([&](double u) { return solve(std::exp(u), nullptr); }, std::log(1e-4),
                                  std::log(1e3));
  const double r = solve(std::exp(lg), theta);
  return std::sqrt(r / n);
}

// Theorem 2 (proof P:782-808): g(y) = (T(y) + t/s)(H + c y) is strictly convex for
// y >= 2/th2 - H/c, everywhere on (0, inf) when th2 >= 2c/H.
void remoe_convexity_threshold(double th2, double H, double c, double* threshold, int32_t* convex_everywhere) {
  if (threshold) *threshold = 2.0 / th2 - H / c;
  if (convex_everywhere) *convex_everywhere = th2 >= 2.0 * c / H ? 1 : 0;
}

// Remote memory per layer (Eqs. 12-14, Theorem 3).  Minimise
//   P2 = (1+eta) sum_l s_l (T_l(y_l) + t_l/s_l)(H + c y_l)
// over y_l in [y_min, y_max] subject to the TPOT coupling constraint
//   sum_l s_l T_l(y_l) <= budget   (q_{l,1}; budget < 0: no constraint)
// by the Lagrangian dual: for a multiplier lam each layer solves a 1-D convex problem,
// lam is found by bisection (the constraint is monotone in lam).  The continuous y_l are
// rounded up to the grid y_min + j*step (feasibility is preserved: T is decreasing).
// theta: [L][3].  Returns the P2 value of the rounded solution, -1 if infeasible/bad.
double remoe_optimize_remote_memory(int32_t L, const double* theta, const double* s, const double* t,
                                    double H, double c, double eta, double y_min, double y_max,
                                    double step, double budget, double* y_cont, double* y_grid) {
  if (L < 1 || !theta || !s || !t || !(y_max >= y_min) || !(step > 0) || !(c > 0)) return -1.0;
  for (int l = 0; l < L; ++l)
    if (!(s[l] > 0)) return -1.0;
  auto solve = [&](double lam, std::vector<double>& y) {
    double used = 0;
    for (int l = 0; l < L; ++l) {
      const double* th = theta + 3 * l;
      y[l] = argmin_convex([&](double v) { return layer_obj(th, s[l], t[l], H, c, lam, v); }, y_min, y_max);
      used += s[l] * t_model(th, y[l]);
    }
    return used;
  };
  std::vector<double> y(L);
  double used = solve(0.0, y);
  if (budget >= 0 && used > budget) {
    double at_max = 0;
    for (int l = 0; l < L; ++l) at_max += s[l] * t_model(theta + 3 * l, y_max);
    if (at_max > budget) return -1.0;  // TPOT infeasible even at the largest memory
    double lo = 0, hi = 1;
    while (solve(hi, y) > budget && hi < 1e30) hi *= 2;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (solve(mid, y) > budget) lo = mid; else hi = mid;
    }
    solve(hi, y);
  }
  double p2 = 0;
  for (int l = 0; l < L; ++l) {
    if (y_cont) y_cont[l] = y[l];
    double g = y_min + std::ceil((y[l] - y_min) / step - 1e-9) * step;
    if (g > y_max) g = y_max;
    if (y_grid) y_grid[l] = g;
    p2 += s[l] * (t_model(theta + 3 * l, g) + t[l] / s[l]) * (H + c * g);
  }
  return (1.0 + eta) * p2;
}

remoe_status_t remoe_mmp(double M_min, double M_cal, double epsilon, const double* spec_mem,
                         int32_t n_specs, remoe_mmp_local_mem_fn local_mem, remoe_mmp_slo_fn slo_ok,
                         void* ctx, int32_t* spec_out, double* b_out, double* M_out) {
  if (!(epsilon > 0) || !spec_mem || n_specs < 1 || !local_mem || !slo_ok) return REMOE_ERR_INVALID_ARG;
  for (int v = 1; v < n_specs; ++v)
    if (spec_mem[v] < spec_mem[v - 1]) return REMOE_ERR_INVALID_ARG;
  // Lines 2-11: b <- 1; repeat { M <- max(M_min + M^e(b), M_cal); check SLOs; b <- b - eps }.
  // b is stepped as 1 - j*eps (no accumulated rounding); the last step is b = 0 (all local).
  const int64_t steps = (int64_t)std::floor(1.0 / epsilon + 1e-9);
  for (int64_t j = 0; j <= steps + 1; ++j) {
    double b = j <= steps ? 1.0 - (double)j * epsilon : 0.0;
    if (b < 0) b = 0;
    const double M = std::max(M_min + local_mem(b, ctx), M_cal);
    if (!slo_ok(M, b, ctx)) continue;
    // Lines 12-13: the smallest specification with m_{w_v} >= M.
    for (int v = 0; v < n_specs; ++v)
      if (spec_mem[v] >= M) {
        if (spec_out) *spec_out = v;
        if (b_out) *b_out = b;
        if (M_out) *M_out = M;
        return REMOE_OK;
      }
    return REMOE_ERR_UNSUPPORTED;
  }
  return REMOE_ERR_UNSUPPORTED;
}

remoe_status_t remoe_greedy_replicas(int32_t L, int32_t z_max, remoe_replica_cost_fn cost,
                                     remoe_replica_tpot_fn tpot_ok, void* ctx, int32_t* Z) {
  if (L < 1 || z_max < 1 || !cost || !tpot_ok || !Z) return REMOE_ERR_INVALID_ARG;
  for (int l = 0; l < L; ++l)
    if (Z[l] < 1 || Z[l] > z_max) return REMOE_ERR_INVALID_ARG;
  std::vector<int32_t> trial(Z, Z + L);
  // Returns the layer with the greatest varpi(l, Z) among z_l < z_max, -1 if none.
  auto best_layer = [&](double* best_gain) {
    const double base = cost(Z, L, ctx);
    int arg = -1;
    double gain = 0;
    for (int l = 0; l < L; ++l) {
      if (Z[l] >= z_max) continue;
      std::copy(Z, Z + L, trial.begin());
      trial[l] += 1;
      const double g = base - cost(trial.data(), L, ctx);  // Eq. 15
      if (arg < 0 || g > gain) { arg = l; gain = g; }
    }
    *best_gain = gain;
    return arg;
  };
  double gain = 0;
  while (!tpot_ok(Z, L, ctx)) {
    const int l = best_layer(&gain);
    if (l < 0) return REMOE_ERR_UNSUPPORTED;
    Z[l] += 1;
  }
  for (;;) {
    const int l = best_layer(&gain);
    if (l < 0 || !(gain > 0)) break;
    Z[l] += 1;
  }
  return REMOE_OK;
}

}  // extern "C"
