/*
 * dgs_oracle.h -- CPU restatement of the reference's conflict-aware parallel
 * Deep Greedy Switching path (lsap::dgs_parallel and its step APIs).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_1106_5694_b200, liblsapgpu.so) never
 * links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Parity is pinned two ways:
 *   1. against the reference itself, compiled from its own sources into
 *      oracle/_ref/liblsap_ref.so by oracle/Makefile (live comparison in
 *      tests/test_oracle.py when that library is present), and
 *   2. against the committed fixtures in tests/golden/ that
 *      tests/golden/make_golden.py generated from that library.
 */
#ifndef DGS_ORACLE_H
#define DGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:11-46 -------------------------------------------------------- */
uint64_t orc_mix64(uint64_t z);
/* k-th draw (0-based) of SplitMix64(seed): mix64(seed + (k+1)*golden). */
uint64_t orc_draw(uint64_t seed, uint64_t k);
double orc_unit_double(uint64_t u);
void orc_random_perm(int32_t n, uint64_t seed, int32_t* p);
/* bench.cpp:200-208 */
uint64_t orc_derive_instance_seed(uint64_t base_seed, int32_t n, int32_t instance_index);
uint64_t orc_derive_run_seed(uint64_t instance_seed, int32_t rep_index);

/* ---- instance generators (row-major n*n doubles) ---------------------------- */
/* test_baselines.cpp:21-26 / SURVEY C1,C2: (double)(next() % modulus) */
void orc_gen_uniform_int(double* a, int32_t n, uint64_t seed, uint64_t modulus);
/* SURVEY C4,C5: (double)(float)unit_double(next()) */
void orc_gen_unit_f32(double* a, int32_t n, uint64_t seed);
/* test_parallel.cpp:17-22: unit_double(next()) * scale (true fp64 values) */
void orc_gen_unit_scaled(double* a, int32_t n, uint64_t seed, double scale);
/* SURVEY C3 (P2P-streaming shaped, invented in SURVEY 8(d)) */
void orc_gen_p2p(double* a, int32_t n, uint64_t seed);
/* geom.cpp:15-33 */
void orc_gen_geom(double* a, int32_t n, uint64_t seed, double bound);

/* ---- core.cpp ---------------------------------------------------------------- */
int orc_validate(const double* a, int32_t n); /* core.cpp:9-15: 0 ok, 1 bad n, 3 non-finite */
double orc_objective(const double* a, int32_t n, const int32_t* sigma); /* core.cpp:17-24 */

/* ---- kernels_scalar.cpp:6-25 (the exchange_scan contract, kernels.hpp:26-37) -- */
void orc_exchange_scan(const double* primary, const double* cross, const int32_t* map,
                       int64_t stride, const double* current, double self_benefit,
                       int32_t skip, int32_t n, double eps, double* delta_out,
                       int32_t* partner_out);

/* ---- parallel.cpp step APIs ------------------------------------------------ */
/* parallel.cpp:134-156 (== sequential ade/jde, dgs.cpp:27-63).  Records are
 * written SoA: delta, partner (-1 = inactive). */
void orc_evaluate_all(const double* a, int32_t n, const int32_t* sigma, double eps,
                      double* agent_delta, int32_t* agent_partner, double* job_delta,
                      int32_t* job_partner);

/* parallel.cpp:35-76 via check_conflicts (parallel.cpp:158-180).  Inputs are
 * the tables with inactive deltas already normalised to 0.  Outputs are masks
 * (u8[n]) plus the ascending conflicted_jobs list; returns its length. */
int32_t orc_check_conflicts(int32_t n, const double* agent_delta, const int32_t* agent_partner,
                            const double* job_delta, const int32_t* job_partner,
                            const int32_t* sigma, uint8_t* agent_accepted,
                            uint8_t* job_accepted, uint8_t* reserved_mask,
                            uint8_t* conflicted_mask, int32_t* conflicted_jobs);

/* parallel.cpp:182-229.  Records carry an explicit active flag (types.hpp:68-72).
 * sigma/tau/value are updated in place; the applied list (agent, new_job,
 * old_job, displaced, delta) is written in commit order.  Returns the number
 * applied, or -1 on "internal: conflict check admitted overlapping exchanges". */
int32_t orc_apply_parallel_switches(const double* a, int32_t n, int32_t* sigma, int32_t* tau,
                                    double* value, const double* agent_delta,
                                    const int32_t* agent_partner, const uint8_t* agent_active,
                                    const double* job_delta, const int32_t* job_partner,
                                    const uint8_t* job_active, const uint8_t* agent_accepted,
                                    const uint8_t* job_accepted, double eps,
                                    int32_t* applied_agent, int32_t* applied_new_job,
                                    int32_t* applied_old_job, int32_t* applied_displaced,
                                    double* applied_delta);

/* ---- parallel.cpp:231-352: the full solver --------------------------------- */
typedef struct {
  int64_t outer_iterations;
  int64_t inner_iterations;    /* CC batches (not in SolveReport; instrumentation) */
  int64_t switches_applied;
  int64_t agent_scans;         /* full + re-eval agent scans */
  int64_t job_scans;
  int64_t pair_items;          /* distinct (agent, tau[agent]) pairs scanned */
  int32_t terminated_by;       /* 0 converged, 1 deadline */
  double value;                /* snapshot_assignment value (solver_state.hpp:141-148) */
  double elapsed_ms;
} orc_stats;

/* policy 0 = touched_and_conflicted (default), 1 = touched_only
 * (parallel.hpp:21-22).  deadline_ns < 0 = none.  trace_switch/trace_value may
 * be NULL; trace_cap is the buffer capacity; *trace_len receives the number of
 * entries the reference would hold (capped at trace_cap).  threads <= 0 uses
 * OpenMP's default (results never depend on it: parallel.hpp:79-80). */
int orc_dgs_parallel(const double* a, int32_t n, uint64_t seed, double eps, int policy,
                     int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                     orc_stats* stats, int64_t* trace_switch, double* trace_value,
                     int64_t trace_cap, int64_t* trace_len);

/* The same loop from a caller-given initial sigma (job -> agent) instead of
 * initial_random: the parity checker of the device's greedy-start solves (an
 * extension; the reference itself always starts from initial_random). */
int orc_dgs_parallel_from(const double* a, int32_t n, const int32_t* init_sigma, double eps, int policy,
                          int64_t deadline_ns, int threads, int32_t* sigma_out, int32_t* tau_out,
                          orc_stats* stats, int64_t* trace_switch, double* trace_value,
                          int64_t trace_cap, int64_t* trace_len);

/* Greedy assignment rule of lsapgpu_greedy_assignment (EXTENSION, not in the
 * reference): rounds in which every unassigned agent claims the best free job
 * of its row (smallest job on ties) and every claimed job goes to the highest
 * claim (smallest agent on ties).  Returns the number of rounds. */
int64_t orc_greedy_assignment(const double* a, int32_t n, int32_t* sigma_out);

/* ---- auction.cpp:12-153: the synchronous auction baseline ------------------
 * AuctionConfig (baselines.hpp:12-26): has_eps selects epsilon; scaling and
 * scale_factor as there.  expire_round < 0: no deadline; k >= 0: the deadline
 * check (auction.cpp:42) fires at the (k+1)-th check, so 0 reproduces
 * deadline = 0 deterministically.  prices_out (nullable) receives the final
 * prices.  Returns 0, or 1 on a config error (the reference's messages). */
typedef struct {
  int64_t rounds;      /* SolveReport::outer_iterations */
  int64_t switches;    /* awards, displacements included */
  int64_t bids;        /* agent row scans (two net_scans each) */
  int32_t terminated_by;
  int32_t completed_greedily;
  double value;
  double epsilon;      /* target epsilon */
} orc_auction_stats;
int orc_auction_solve(const double* a, int32_t n, int has_eps, double eps, int scaling,
                      double scale_factor, int64_t expire_round, int32_t* sigma_out,
                      double* prices_out, orc_auction_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
