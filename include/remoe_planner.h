/*
 * remoe_planner.h -- NEXT-N3: the host-side planner that consumes the
 * predicted activation matrix (§IV-C..F, lines P:460-647).  Plain C++ in
 * libremoe.so; every call is synchronous, host memory only, no GPU needed, thread-safe
 * (no global state).  All pointers are caller-owned; nothing is retained after return.
 *
 * Error behaviour: functions returning double return -1.0 on invalid arguments (all
 * legitimate results are >= 0); functions returning remoe_status_t return
 * REMOE_ERR_INVALID_ARG on invalid arguments and REMOE_ERR_UNSUPPORTED when the
 * problem is infeasible (remoe_last_error() is not touched).
 *
 * Notation follows the paper: n / N^in tokens, K = K_l experts per layer, m remote
 * experts, z = z_l replicas, theta = (theta_1, theta_2, theta_3) of the latency model
 * T~(y) = theta_1 exp(-theta_2 y) + theta_3, H = H^w, c = c^c.
 */
#ifndef REMOE_PLANNER_H_
#define REMOE_PLANNER_H_

#include "remoe.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Theorem 1 / Corollary 1: with probability >= 95%, m of the K experts of
 * a layer process at most sqrt(3n)/2 + m n / K of n tokens.  Returns that bound;
 * -1 if n < 0, K < 1 or m outside [0, K].
 */
REMOE_API double remoe_worst_case_tokens(double n, int32_t m, int32_t K);

/*
 * LPT for the Multiway Number Partitioning of one layer's remote-expert tasks over z
 * replicas: tasks in non-increasing load order (equal loads: lower index
 * first), each to the currently least-loaded replica (equal: lower replica index).
 *   loads: [n] task times (>= 0); assign: [n] out, replica of each task in [0, z);
 *   replica_load: [z] out or NULL.  Returns the makespan max_j ZT_j, which Graham's bound
 *   keeps within (4/3 - 1/(3z)) of the optimum.  -1 on invalid arguments.
 */
REMOE_API double remoe_lpt_partition(const double* loads, int32_t n, int32_t z, int32_t* assign,
                                     double* replica_load);

/*
 * Theorem 4: the 95% bound on the slowest replica's prefill time,
 *   (z-1)/z [tau(N^up) + 2D/B N^up] + T^rem / z + t^rem,  N^up = sqrt(3 n_in)/2 + n_in/K,
 * with tau_nup = sum_v y_{l,v} tau^c_{l,v}(N^up) evaluated by the caller at N^up
 * (remoe_worst_case_tokens(n_in, 1, K)), two_d_over_b = 2D/B.  -1 if z < 1 or K < 1.
 */
REMOE_API double remoe_replica_time_bound(int32_t z, double tau_nup, double two_d_over_b, double n_in,
                                          int32_t K, double T_rem, double t_rem);

/*
 * Fit the latency model T~(y) = theta_1 exp(-theta_2 y) + theta_3 to n >= 3
 * profiled points (y[i], t[i]) in least squares: (theta_1, theta_3) are solved exactly
 * for each theta_2, theta_2 is searched (golden section on log theta_2 over
 * [1e-4, 1e3]).  theta: [3] out.  Returns the RMS residual, -1 on invalid arguments.
 */
REMOE_API double remoe_fit_latency_curve(const double* y, const double* t, int32_t n, double* theta);

/*
 * Theorem 2 (proof P:782-808): g(y) = (T~(y) + t/s~)(H + c y) is strictly
 * convex for y >= 2/theta_2 - H/c (*threshold) and on all of (0, inf) when
 * theta_2 >= 2c/H (*convex_everywhere = 1).  Either out pointer may be NULL.
 */
REMOE_API void remoe_convexity_threshold(double theta2, double H, double c, double* threshold,
                                         int32_t* convex_everywhere);

/*
 * Remote-expert memory per layer: P_2 solved through its Lagrangian dual
 * (P:573-600).  Minimise
 *     (1 + eta) sum_l s~_l (T~_l(y_l) + t_l / s~_l) (H + c y_l)
 * over y_min <= y_l <= y_max (the linear range constraints q_{l,2..4}) subject to the
 * TPOT coupling constraint q_{l,1}: sum_l s~_l T~_l(y_l) <= budget (budget < 0: none).
 * For a multiplier lambda the Lagrangian separates into L one-dimensional problems
 * (golden section, exact on the convex range of Theorem 2); lambda is set by bisection
 * on the monotone constraint.  The continuous optimum y_cont is rounded UP to the
 * memory grid y_min + j * step (y_grid), which keeps TPOT feasible since T~ decreases.
 *   theta: [L x 3]; s_tilde, t_rem: [L]; y_cont, y_grid: [L] out (either may be NULL).
 * Returns P_2 at y_grid; -1 on invalid arguments or when TPOT is infeasible even at
 * y_max for every layer.
 */
REMOE_API double remoe_optimize_remote_memory(int32_t L, const double* theta, const double* s_tilde,
                                              const double* t_rem, double H, double c, double eta,
                                              double y_min, double y_max, double step, double budget,
                                              double* y_cont, double* y_grid);

/*
 * MMP, Algorithm 2.  The serving model (memory of local experts for a
 * remote ratio b, and the TTFT/TPOT check with the worst-case remote time of
 * Corollary 1) is the caller's, passed as callbacks:
 *   local_mem(b, ctx)      -> M^e, memory of the local experts at ratio b;
 *   slo_ok(M, b, ctx)      -> nonzero when TTFT and TPOT hold for main-model memory M;
 * Starting from b = 1, M = max(M_min + M^e(b), M_cal) is checked and b decreased by
 * epsilon until the SLOs hold (or b < 0: REMOE_ERR_UNSUPPORTED).  Then the smallest
 * specification v with spec_mem[v] >= M is chosen (spec_mem ascending, n_specs >= 1;
 * none large enough: REMOE_ERR_UNSUPPORTED).
 *   spec_out: index v; b_out: the ratio the SLOs held at; M_out: M.  Any may be NULL.
 */
typedef double (*remoe_mmp_local_mem_fn)(double b, void* ctx);
typedef int32_t (*remoe_mmp_slo_fn)(double M, double b, void* ctx);
REMOE_API remoe_status_t remoe_mmp(double M_min, double M_cal, double epsilon, const double* spec_mem,
                                   int32_t n_specs, remoe_mmp_local_mem_fn local_mem, remoe_mmp_slo_fn slo_ok,
                                   void* ctx, int32_t* spec_out, double* b_out, double* M_out);

/*
 * Remote-expert replicas, P:630-647 with the replica potential of Eq. 15:
 *   varpi(l, Z) = C(Z) - C(Z with z_l + 1),
 * C = C^loc + C^rem the caller's cost model, cost(Z, L, ctx).  Z starts at z_init (the
 * payload-feasible counts, each <= z_max).  While tpot_ok(Z, L, ctx) == 0 the layer with
 * the greatest potential among those with z_l < z_max gets one more replica (equal
 * potentials: lower l); none left: REMOE_ERR_UNSUPPORTED.  Then, while some layer with
 * z_l < z_max has varpi > 0, the greatest such gets one more.  Z: [L] in/out (z_init in).
 */
typedef double (*remoe_replica_cost_fn)(const int32_t* Z, int32_t L, void* ctx);
typedef int32_t (*remoe_replica_tpot_fn)(const int32_t* Z, int32_t L, void* ctx);
REMOE_API remoe_status_t remoe_greedy_replicas(int32_t L, int32_t z_max, remoe_replica_cost_fn cost,
                                               remoe_replica_tpot_fn tpot_ok, void* ctx, int32_t* Z);

#ifdef __cplusplus
}
#endif
#endif /* REMOE_PLANNER_H_ */
