// ref_harness.cpp -- extern "C" shim over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE).  oracle/Makefile compiles the reference's own sources
// in place (/root/reference/proj/src/*.cpp, read-only) together with this file
// into oracle/_ref/liblsap_ref.so.  Nothing here re-implements the algorithm:
// every entry point forwards to the reference's public API
// (proj/include/lsap/parallel.hpp:60-80, geom.hpp:26, rng.hpp:37).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "lsap/baselines.hpp"
#include "lsap/core.hpp"
#include "lsap/dgs.hpp"
#include "lsap/geom.hpp"
#include "lsap/kernels.hpp"
#include "lsap/parallel.hpp"
#include "lsap/rng.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

lsap::Instance make_instance(const double* a, std::int32_t n) {
  return lsap::Instance(n, std::vector<double>(a, a + static_cast<std::size_t>(n) * n));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

const char* ref_kernel_name() { return lsap::kernels::active().name; }

void ref_random_perm(std::int32_t n, std::uint64_t seed, std::int32_t* out) {
  const auto p = lsap::random_perm(n, seed);
  std::memcpy(out, p.data(), sizeof(std::int32_t) * n);
}

int ref_generate_geom(std::int32_t n, double bound, std::uint64_t seed, double* out) {
  try {
    const auto inst = lsap::generate_geom({n, bound, seed});
    std::memcpy(out, inst.benefits.data(), sizeof(double) * inst.benefits.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// lsap::dgs_parallel (parallel.cpp:231-352).  trace buffers may be null.
int ref_dgs_parallel(const double* a, std::int32_t n, std::uint64_t seed, double eps,
                     int policy, std::int64_t deadline_ns, int workers, std::int32_t* sigma_out,
                     std::int32_t* tau_out, double* value_out, std::int64_t* outer_out,
                     std::int64_t* switches_out, int* terminated_out, double* elapsed_ms_out,
                     std::int64_t* trace_switch, double* trace_value, std::int64_t trace_cap,
                     std::int64_t* trace_len) {
  try {
    const auto inst = make_instance(a, n);
    lsap::ParallelConfig cfg;
    cfg.seed = seed;
    cfg.improvement_epsilon = eps;
    cfg.workers = workers;
    cfg.reeval = policy == 1 ? lsap::ParallelConfig::Reeval::touched_only
                             : lsap::ParallelConfig::Reeval::touched_and_conflicted;
    if (deadline_ns >= 0) cfg.deadline = lsap::Duration{deadline_ns};
    const auto rep = lsap::dgs_parallel(inst, cfg);
    std::memcpy(sigma_out, rep.assignment.sigma.data(), sizeof(std::int32_t) * n);
    if (tau_out) std::memcpy(tau_out, rep.assignment.tau.data(), sizeof(std::int32_t) * n);
    *value_out = rep.assignment.value;
    *outer_out = rep.outer_iterations;
    *switches_out = rep.switches_applied;
    *terminated_out = rep.terminated_by == lsap::Termination::deadline ? 1 : 0;
    *elapsed_ms_out = std::chrono::duration<double, std::milli>(rep.elapsed).count();
    const auto len = static_cast<std::int64_t>(rep.objective_trace.size());
    if (trace_len) *trace_len = len;
    if (trace_switch && trace_value)
      for (std::int64_t k = 0; k < len && k < trace_cap; ++k) {
        trace_switch[k] = rep.objective_trace[k].first;
        trace_value[k] = rep.objective_trace[k].second;
      }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// lsap::evaluate_all_parallel (parallel.cpp:134-156), SoA out.
int ref_evaluate_all(const double* a, std::int32_t n, const std::int32_t* sigma, double eps,
                     int workers, double* agent_delta, std::int32_t* agent_partner,
                     double* job_delta, std::int32_t* job_partner) {
  try {
    const auto inst = make_instance(a, n);
    const auto asg = lsap::make_assignment(inst, lsap::Perm(sigma, sigma + n));
    lsap::ParallelConfig cfg;
    cfg.workers = workers;
    cfg.improvement_epsilon = eps;
    lsap::DeltaTables t;
    lsap::evaluate_all_parallel(inst, asg, t, cfg);
    for (std::int32_t k = 0; k < n; ++k) {
      agent_delta[k] = t.agent_records[k].delta;
      agent_partner[k] = t.agent_records[k].partner;
      job_delta[k] = t.job_records[k].delta;
      job_partner[k] = t.job_records[k].partner;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// lsap::check_conflicts (parallel.cpp:158-180).  Records are active iff
// partner >= 0 unless an explicit active mask is given.
int ref_check_conflicts(std::int32_t n, const double* agent_delta,
                        const std::int32_t* agent_partner, const std::uint8_t* agent_active,
                        const double* job_delta, const std::int32_t* job_partner,
                        const std::uint8_t* job_active, const std::int32_t* sigma,
                        std::uint8_t* agent_accepted, std::uint8_t* job_accepted,
                        std::uint8_t* reserved_mask, std::uint8_t* conflicted_mask,
                        std::int32_t* conflicted_jobs, std::int32_t* n_conflicted_jobs) {
  try {
    lsap::DeltaTables t = lsap::DeltaTables::sized(n);
    for (std::int32_t k = 0; k < n; ++k) {
      t.agent_records[k] = {agent_partner[k], agent_delta[k],
                            agent_active ? agent_active[k] != 0 : agent_partner[k] >= 0};
      t.job_records[k] = {job_partner[k], job_delta[k],
                          job_active ? job_active[k] != 0 : job_partner[k] >= 0};
    }
    lsap::Assignment asg;
    asg.sigma.assign(sigma, sigma + n);
    asg.tau = lsap::make_tau(asg.sigma);
    const auto sets = lsap::check_conflicts(t, asg);
    std::memcpy(agent_accepted, sets.agent_accepted.data(), n);
    std::memcpy(job_accepted, sets.job_accepted.data(), n);
    std::memset(reserved_mask, 0, n);
    std::memset(conflicted_mask, 0, n);
    for (auto i : sets.reserved) reserved_mask[i] = 1;
    for (auto i : sets.conflicted) conflicted_mask[i] = 1;
    for (std::size_t k = 0; k < sets.conflicted_jobs.size(); ++k)
      conflicted_jobs[k] = sets.conflicted_jobs[k];
    *n_conflicted_jobs = static_cast<std::int32_t>(sets.conflicted_jobs.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// lsap::apply_parallel_switches (parallel.cpp:182-229).  Returns the number
// applied, or -1 with ref_last_error() set when the reference throws.
std::int32_t ref_apply_parallel_switches(
    const double* a, std::int32_t n, std::int32_t* sigma, std::int32_t* tau, double* value,
    const double* agent_delta, const std::int32_t* agent_partner, const std::uint8_t* agent_active,
    const double* job_delta, const std::int32_t* job_partner, const std::uint8_t* job_active,
    const std::uint8_t* agent_accepted, const std::uint8_t* job_accepted, double eps,
    std::int32_t* out_agent, std::int32_t* out_new_job, std::int32_t* out_old_job,
    std::int32_t* out_displaced, double* out_delta) {
  try {
    const auto inst = make_instance(a, n);
    lsap::Assignment asg;
    asg.sigma.assign(sigma, sigma + n);
    asg.tau.assign(tau, tau + n);
    asg.value = *value;
    lsap::DeltaTables t = lsap::DeltaTables::sized(n);
    for (std::int32_t k = 0; k < n; ++k) {
      t.agent_records[k] = {agent_partner[k], agent_delta[k], agent_active[k] != 0};
      t.job_records[k] = {job_partner[k], job_delta[k], job_active[k] != 0};
    }
    lsap::ConflictSets sets;
    sets.agent_accepted.assign(agent_accepted, agent_accepted + n);
    sets.job_accepted.assign(job_accepted, job_accepted + n);
    lsap::ParallelConfig cfg;
    cfg.improvement_epsilon = eps;
    const auto [out, applied] = lsap::apply_parallel_switches(inst, asg, t, sets, cfg);
    std::memcpy(sigma, out.sigma.data(), sizeof(std::int32_t) * n);
    std::memcpy(tau, out.tau.data(), sizeof(std::int32_t) * n);
    *value = out.value;
    for (std::size_t k = 0; k < applied.size(); ++k) {
      out_agent[k] = applied[k].agent;
      out_new_job[k] = applied[k].new_job;
      out_old_job[k] = applied[k].old_job;
      out_displaced[k] = applied[k].displaced;
      out_delta[k] = applied[k].delta;
    }
    return static_cast<std::int32_t>(applied.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// lsap::auction_solve (auction.cpp:110-153).  has_eps selects
// AuctionConfig::epsilon; prices_out (nullable) receives the price vector the
// on_round observer saw last; rounds_out the number of observed rounds and
// monotone_out whether prices never decreased between rounds
// (test_baselines.cpp:104-115).
int ref_auction_solve(const double* a, std::int32_t n, int has_eps, double eps, int scaling,
                      double scale_factor, std::int64_t deadline_ns, std::int32_t* sigma_out,
                      double* value_out, std::int64_t* outer_out, std::int64_t* switches_out,
                      int* terminated_out, int* greedy_out, double* elapsed_ms_out,
                      double* prices_out, std::int64_t* rounds_out, int* monotone_out) {
  try {
    const auto inst = make_instance(a, n);
    lsap::AuctionConfig cfg;
    if (has_eps) cfg.epsilon = eps;
    cfg.scaling = scaling != 0;
    cfg.scale_factor = scale_factor;
    if (deadline_ns >= 0) cfg.deadline = lsap::Duration{deadline_ns};
    std::vector<double> last;
    std::int64_t rounds = 0;
    bool monotone = true;
    const auto rep = lsap::auction_solve(inst, cfg, [&](const std::vector<double>& prices) {
      if (!last.empty())
        for (std::size_t j = 0; j < prices.size(); ++j) monotone &= prices[j] >= last[j];
      last = prices;
      ++rounds;
    });
    std::memcpy(sigma_out, rep.assignment.sigma.data(), sizeof(std::int32_t) * n);
    *value_out = rep.assignment.value;
    *outer_out = rep.outer_iterations;
    *switches_out = rep.switches_applied;
    *terminated_out = rep.terminated_by == lsap::Termination::deadline ? 1 : 0;
    *greedy_out = rep.completed_greedily ? 1 : 0;
    *elapsed_ms_out = std::chrono::duration<double, std::milli>(rep.elapsed).count();
    if (prices_out) {
      if (last.empty()) last.assign(static_cast<std::size_t>(n), 0.0);
      std::memcpy(prices_out, last.data(), sizeof(double) * n);
    }
    if (rounds_out) *rounds_out = rounds;
    if (monotone_out) *monotone_out = monotone ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
