// lsapgpu.hpp -- header-only C++ wrapper that puts the B200 solver behind the
// reference's own C++ types and entry points.
//
// Include it AFTER the reference headers (it uses lsap::Instance, Assignment,
// DeltaTables, ConflictSets, AppliedExchange, ParallelConfig, SolveReport and
// lsap::Error from proj/include/lsap/{types,parallel}.hpp) and link
// liblsapgpu.so.  Each function mirrors its reference counterpart:
//
//   lsap::gpu::dgs_parallel              <- lsap::dgs_parallel              (parallel.hpp:80)
//   lsap::gpu::evaluate_all_parallel     <- lsap::evaluate_all_parallel     (parallel.hpp:60-61)
//   lsap::gpu::check_conflicts           <- lsap::check_conflicts           (parallel.hpp:65)
//   lsap::gpu::apply_parallel_switches   <- lsap::apply_parallel_switches   (parallel.hpp:71-74)
//   lsap::gpu::auction_solve             <- lsap::auction_solve             (baselines.hpp:33-36)
//
// auction_solve additionally needs lsap/baselines.hpp (AuctionConfig) included
// before this header; define LSAPGPU_NO_AUCTION to leave it out.
//
// Same argument meaning, same results (bit for bit), same lsap::Error messages;
// `workers` / `chunk` are validated and otherwise ignored (the reference's
// results never depend on them, parallel.hpp:79-80).  A per-thread, per-device
// context caches device memory and the CUDA graph between calls.
#pragma once

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "lsapgpu.h"

namespace lsap::gpu {

struct GpuConfig : ParallelConfig {
  int device = 0;
  bool use_graph = true;     // inner loop as one CUDA-graph launch per outer pass
  bool greedy_init = false;  // extension: start from the device greedy assignment, not initial_random
};

class Context {
 public:
  explicit Context(int device = 0) {
    if (lsapgpu_create(&ctx_, device) != LSAPGPU_OK)
      throw Error("lsapgpu: no usable sm_100 CUDA device " + std::to_string(device));
  }
  ~Context() { lsapgpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  lsapgpu_ctx* get() const { return ctx_; }

  void check(int rc) const {
    if (rc != LSAPGPU_OK) throw Error(lsapgpu_last_error(ctx_));
  }

  // Uploads the instance (validate, lossless narrowing, A and AT in HBM).
  // Every call re-uploads: the functions below are pure like the reference's,
  // so a caller that mutates or reallocates an Instance must never see a
  // stale device copy.  Callers that solve one matrix repeatedly can keep a
  // Context and call lsapgpu_set_matrix / lsapgpu_solve directly.
  void set_instance(const Instance& inst) {
    if (inst.n < 1) throw Error("instance size must be >= 1, got " + std::to_string(inst.n));
    if (inst.benefits.size() != static_cast<std::size_t>(inst.n) * inst.n)
      throw Error("benefit matrix is not " + std::to_string(inst.n) + "x" + std::to_string(inst.n));
    check(lsapgpu_set_matrix(ctx_, inst.benefits.data(), inst.n, LSAPGPU_F64));
  }

 private:
  lsapgpu_ctx* ctx_ = nullptr;
};

inline Context& context(int device) {
  thread_local std::map<int, std::unique_ptr<Context>> ctxs;
  auto& c = ctxs[device];
  if (!c) c = std::make_unique<Context>(device);
  return *c;
}

inline SolveReport dgs_parallel(const Instance& inst, const GpuConfig& cfg = {}) {
  // Instance::validate (core.cpp:9-15) runs on the device during the upload
  // (same checks, same messages, same precedence over cfg.validate()), so
  // the O(n^2) host pass of the reference is not repeated here.
  Context& ctx = context(cfg.device);
  ctx.set_instance(inst);
  cfg.validate();
  lsapgpu_params p{};
  p.seed = cfg.seed;
  p.eps = cfg.improvement_epsilon;
  p.reeval = cfg.reeval == ParallelConfig::Reeval::touched_only ? LSAPGPU_REEVAL_TOUCHED_ONLY
                                                                 : LSAPGPU_REEVAL_TOUCHED_AND_CONFLICTED;
  p.use_graph = cfg.use_graph ? 1 : 0;
  // Deadline::starting accepts any budget: zero or negative expires at once
  p.deadline_ns = cfg.deadline ? std::max<std::int64_t>(0, static_cast<std::int64_t>(cfg.deadline->count())) : -1;
  p.init_sigma = nullptr;
  p.init_mode = cfg.greedy_init ? LSAPGPU_INIT_GREEDY : LSAPGPU_INIT_RANDOM;
  const std::int32_t n = inst.n;
  SolveReport rep;
  rep.assignment.sigma.resize(n);
  rep.assignment.tau.resize(n);
  lsapgpu_stats st{};
  std::int64_t cap = 100000 + 4096;
  // per-thread scratch the library writes the trace into (kept: fresh
  // buffers cost page faults and zeroing on every call)
  static thread_local std::vector<std::int64_t> ts;
  static thread_local std::vector<double> tv;
  if (static_cast<std::int64_t>(ts.size()) < cap) {
    ts.resize(static_cast<std::size_t>(cap));
    tv.resize(static_cast<std::size_t>(cap));
  }
  std::int64_t tl = 0;
  ctx.check(lsapgpu_solve(ctx.get(), &p, rep.assignment.sigma.data(), rep.assignment.tau.data(), &st,
                          ts.data(), tv.data(), cap, &tl));
  if (tl > cap && !cfg.deadline) {
    // the reference's trace keeps growing by one entry per outer pass past its
    // 100000 cap (parallel.cpp:15-20,343-344): re-run with room for all of it
    // (the solve is deterministic without a deadline)
    cap = tl;
    ts.resize(static_cast<std::size_t>(cap));
    tv.resize(static_cast<std::size_t>(cap));
    ctx.check(lsapgpu_solve(ctx.get(), &p, rep.assignment.sigma.data(), rep.assignment.tau.data(), &st,
                            ts.data(), tv.data(), cap, &tl));
  }
  rep.assignment.value = st.value;
  rep.outer_iterations = st.outer_iterations;
  rep.switches_applied = st.switches_applied;
  rep.terminated_by = st.terminated_by ? Termination::deadline : Termination::converged;
  rep.elapsed = std::chrono::duration_cast<Duration>(std::chrono::duration<double, std::milli>(st.elapsed_ms));
  const std::int64_t k = tl < cap ? tl : cap;
  rep.objective_trace.reserve(static_cast<std::size_t>(k));
  for (std::int64_t q = 0; q < k; ++q) rep.objective_trace.emplace_back(ts[q], tv[q]);
  return rep;
}

inline void evaluate_all_parallel(const Instance& inst, const Assignment& asg, DeltaTables& tables,
                                  const GpuConfig& cfg = {}) {
  Context& ctx = context(cfg.device);
  ctx.set_instance(inst);  // Instance::validate on the device
  cfg.validate();
  if (asg.size() != inst.n) throw Error("assignment does not match instance");
  const std::int32_t n = inst.n;
  std::vector<double> ad(n), jd(n);
  std::vector<std::int32_t> ap(n), jp(n);
  ctx.check(lsapgpu_evaluate_all(ctx.get(), asg.sigma.data(), cfg.improvement_epsilon, ad.data(), ap.data(),
                                 jd.data(), jp.data()));
  tables.agent_records.resize(n);
  tables.job_records.resize(n);
  for (std::int32_t k = 0; k < n; ++k) {
    tables.agent_records[k] = {ap[k], ad[k], ap[k] >= 0};
    tables.job_records[k] = {jp[k], jd[k], jp[k] >= 0};
  }
}

inline ConflictSets check_conflicts(const DeltaTables& tables, const Assignment& asg, int device = 0) {
  const std::int32_t n = asg.size();
  if (tables.agent_records.size() != static_cast<std::size_t>(n) ||
      tables.job_records.size() != static_cast<std::size_t>(n))
    throw Error("delta tables do not match assignment size");
  std::vector<double> ad(n), jd(n);
  std::vector<std::int32_t> ap(n), jp(n);
  for (std::int32_t k = 0; k < n; ++k) {  // parallel.cpp:166-173
    ad[k] = tables.agent_records[k].active ? tables.agent_records[k].delta : 0.0;
    ap[k] = tables.agent_records[k].partner;
    jd[k] = tables.job_records[k].active ? tables.job_records[k].delta : 0.0;
    jp[k] = tables.job_records[k].partner;
  }
  Context& ctx = context(device);
  std::vector<std::uint8_t> res(n), con(n);
  std::vector<std::int32_t> cj(n);
  std::int32_t ncj = 0;
  ConflictSets out;
  out.agent_accepted.resize(n);
  out.job_accepted.resize(n);
  ctx.check(lsapgpu_check_conflicts(ctx.get(), n, ad.data(), ap.data(), jd.data(), jp.data(), asg.sigma.data(),
                                    out.agent_accepted.data(), out.job_accepted.data(), res.data(), con.data(),
                                    cj.data(), &ncj));
  for (std::int32_t k = 0; k < n; ++k) {
    if (res[k]) out.reserved.push_back(k);
    if (con[k]) out.conflicted.push_back(k);
  }
  out.conflicted_jobs.assign(cj.begin(), cj.begin() + ncj);
  return out;
}

inline std::pair<Assignment, std::vector<AppliedExchange>> apply_parallel_switches(
    const Instance& inst, const Assignment& asg, const DeltaTables& tables, const ConflictSets& sets,
    const GpuConfig& cfg = {}) {
  Context& ctx = context(cfg.device);
  ctx.set_instance(inst);  // Instance::validate on the device
  cfg.validate();
  const std::int32_t n = inst.n;
  if (asg.size() != n) throw Error("assignment does not match instance");
  std::vector<double> ad(n), jd(n);
  std::vector<std::int32_t> ap(n), jp(n);
  std::vector<std::uint8_t> aa(n), ja(n);
  for (std::int32_t k = 0; k < n; ++k) {
    ad[k] = tables.agent_records[k].delta;
    ap[k] = tables.agent_records[k].partner;
    aa[k] = tables.agent_records[k].active;
    jd[k] = tables.job_records[k].delta;
    jp[k] = tables.job_records[k].partner;
    ja[k] = tables.job_records[k].active;
  }
  Assignment out = asg;
  std::vector<std::int32_t> a1(n), a2(n), a3(n), a4(n);
  std::vector<double> a5(n);
  std::int32_t k = 0;
  const int rc = lsapgpu_apply_parallel_switches(
      ctx.get(), out.sigma.data(), out.tau.data(), &out.value, ad.data(), ap.data(), aa.data(), jd.data(),
      jp.data(), ja.data(), sets.agent_accepted.data(), sets.job_accepted.data(), cfg.improvement_epsilon,
      a1.data(), a2.data(), a3.data(), a4.data(), a5.data(), &k);
  ctx.check(rc);
  std::vector<AppliedExchange> applied(static_cast<std::size_t>(k));
  for (std::int32_t q = 0; q < k; ++q) applied[q] = {a1[q], a2[q], a3[q], a4[q], a5[q]};
  return {std::move(out), std::move(applied)};
}

#ifndef LSAPGPU_NO_AUCTION
// lsap::auction_solve (auction.cpp:110-153) on the device.  on_round, when
// set, observes the price vector after every round: the rounds are recorded
// on the device (up to `round_cap`, the run repeated with an exact buffer when
// longer and no deadline is set) and replayed to the observer in order.
inline SolveReport auction_solve(const Instance& inst, const AuctionConfig& cfg = {},
                                 const std::function<void(const std::vector<double>&)>& on_round = {},
                                 int device = 0, std::int64_t round_cap = 4096) {
  Context& ctx = context(device);
  ctx.set_instance(inst);  // Instance::validate on the device
  cfg.validate();
  lsapgpu_auction_params p{};
  p.has_epsilon = cfg.epsilon ? 1 : 0;
  p.epsilon = cfg.epsilon ? *cfg.epsilon : 0.0;
  p.scaling = cfg.scaling ? 1 : 0;
  p.scale_factor = cfg.scale_factor;
  p.deadline_ns = cfg.deadline ? std::max<std::int64_t>(0, static_cast<std::int64_t>(cfg.deadline->count())) : -1;
  const std::int32_t n = inst.n;
  SolveReport rep;
  rep.assignment.sigma.resize(n);
  rep.assignment.tau.resize(n);
  lsapgpu_auction_stats st{};
  std::int64_t cap = on_round ? round_cap : 0;
  std::vector<double> rounds;
  auto run = [&]() {
    rounds.assign(static_cast<std::size_t>(cap) * n, 0.0);
    ctx.check(lsapgpu_auction_solve(ctx.get(), &p, rep.assignment.sigma.data(), rep.assignment.tau.data(), &st,
                                    nullptr, cap ? rounds.data() : nullptr, cap));
  };
  run();
  if (on_round && st.outer_iterations > cap && !cfg.deadline) {
    cap = st.outer_iterations;
    run();
  }
  if (on_round) {
    std::vector<double> prices(static_cast<std::size_t>(n));
    for (std::int64_t r = 0; r < cap && r < st.outer_iterations; ++r) {
      std::copy(rounds.begin() + r * n, rounds.begin() + (r + 1) * n, prices.begin());
      on_round(prices);
    }
  }
  rep.assignment.value = st.value;
  rep.outer_iterations = st.outer_iterations;
  rep.switches_applied = st.switches_applied;
  rep.terminated_by = st.terminated_by ? Termination::deadline : Termination::converged;
  rep.completed_greedily = st.completed_greedily != 0;
  rep.objective_trace.emplace_back(0, rep.assignment.value);  // auction.cpp:149
  rep.elapsed = std::chrono::duration_cast<Duration>(std::chrono::duration<double, std::milli>(st.elapsed_ms));
  return rep;
}
#endif

}  // namespace lsap::gpu
