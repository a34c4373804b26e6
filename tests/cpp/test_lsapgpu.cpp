// test_lsapgpu.cpp -- the reference's own C++ API and types driving the B200
// solver through include/lsapgpu.hpp, checked bit for bit against the
// reference's lsap::dgs_parallel / step APIs on the same inputs.  The cases
// restate tests/test_parallel.cpp (paths relative to /root/reference/proj):
// :47-61 evaluate_all vs ade/jde tables, :78-128 conflict-check hand cases,
// :130-194 apply, :196-206 two-permutation optimum, :222-237 worker
// invariance instances, :239-256 fixed point, :258-271 trace / deadline, and
// acceptance.cpp:133-159 fidelity instances.  Built by tests/cpp/Makefile
// against the reference headers and oracle/_ref/liblsap_ref.so (TEST
// INFRASTRUCTURE; the product library never links the reference).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "lsap/baselines.hpp"
#include "lsap/bench.hpp"
#include "lsap/core.hpp"
#include "lsap/dgs.hpp"
#include "lsap/geom.hpp"
#include "lsap/kernels.hpp"
#include "lsap/parallel.hpp"
#include "lsap/rng.hpp"
#include "lsapgpu.hpp"
#include "lsapgpu_engine.hpp"

#include <map>
#include <sstream>
#include <tuple>

using namespace lsap;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(cond)) {                                                             \
      ++g_fail;                                                                \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                          \
  } while (0)

static Instance random_instance(std::int32_t n, std::uint64_t seed, double scale = 10.0) {
  SplitMix64 rng(seed);
  Instance inst = Instance::zeros(n);
  for (auto& v : inst.benefits) v = unit_double(rng.next()) * scale;
  return inst;
}

static Instance random_int_instance(std::int32_t n, std::uint64_t seed, std::uint64_t mod) {
  SplitMix64 rng(seed);
  Instance inst = Instance::zeros(n);
  for (auto& v : inst.benefits) v = static_cast<double>(rng.next() % mod);
  return inst;
}

static bool same_report(const SolveReport& a, const SolveReport& b) {
  return a.assignment.sigma == b.assignment.sigma && a.assignment.tau == b.assignment.tau &&
         std::memcmp(&a.assignment.value, &b.assignment.value, sizeof(double)) == 0 &&
         a.outer_iterations == b.outer_iterations && a.switches_applied == b.switches_applied &&
         a.terminated_by == b.terminated_by && a.objective_trace == b.objective_trace;
}

static bool tables_identical(const DeltaTables& a, const DeltaTables& b) {
  if (a.agent_records.size() != b.agent_records.size()) return false;
  const auto same = [](const ExchangeRecord& x, const ExchangeRecord& y) {
    return x.partner == y.partner && x.active == y.active && std::memcmp(&x.delta, &y.delta, 8) == 0;
  };
  for (std::size_t k = 0; k < a.agent_records.size(); ++k)
    if (!same(a.agent_records[k], b.agent_records[k]) || !same(a.job_records[k], b.job_records[k])) return false;
  return true;
}

static void solve_both(const Instance& inst, std::uint64_t seed,
                       ParallelConfig::Reeval policy = ParallelConfig::Reeval::touched_and_conflicted,
                       double eps = 0.0) {
  ParallelConfig rc;
  rc.seed = seed;
  rc.reeval = policy;
  rc.improvement_epsilon = eps;
  gpu::GpuConfig gc;
  gc.seed = seed;
  gc.reeval = policy;
  gc.improvement_epsilon = eps;
  const auto ref = dgs_parallel(inst, rc);
  for (bool graph : {true, false}) {
    gc.use_graph = graph;
    const auto got = gpu::dgs_parallel(inst, gc);
    CHECK(same_report(ref, got));
  }
}

int main() {
  try {
    // evaluate_all_parallel == reference tables (test_parallel.cpp:47-76)
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
      const std::int32_t n = 3 + static_cast<std::int32_t>(seed * 7 % 62);
      const Instance inst = random_instance(n, 800 + seed);
      const auto asg = make_assignment(inst, random_perm(n, seed));
      DeltaTables ref, got;
      evaluate_all_parallel(inst, asg, ref, {});
      gpu::evaluate_all_parallel(inst, asg, got);
      CHECK(tables_identical(ref, got));
    }
    {
      const Instance inst = generate_geom({256, 100.0, 41});
      const auto asg = initial_random(inst, 3);
      DeltaTables ref, got;
      evaluate_all_parallel(inst, asg, ref, {});
      gpu::evaluate_all_parallel(inst, asg, got);
      CHECK(tables_identical(ref, got));
    }
    // check_conflicts hand cases (test_parallel.cpp:78-128)
    {
      const auto asg = make_assignment(Instance::zeros(4), {0, 1, 2, 3});
      DeltaTables t = DeltaTables::sized(4);
      t.agent_records[0] = {2, 1.0, true};
      t.agent_records[1] = {2, 2.0, true};
      const auto s = gpu::check_conflicts(t, asg);
      CHECK((s.reserved == std::vector<std::int32_t>{0, 2}));
      CHECK((s.conflicted == std::vector<std::int32_t>{1}));
      DeltaTables u = DeltaTables::sized(4);
      u.job_records[0] = {1, 1.0, true};
      u.job_records[1] = {0, 1.0, true};
      u.job_records[2] = {3, 1.0, true};
      const auto r = gpu::check_conflicts(u, asg);
      CHECK((r.reserved == std::vector<std::int32_t>{0, 1, 2, 3}));
      CHECK((r.conflicted == std::vector<std::int32_t>{1}));
      CHECK((r.conflicted_jobs == std::vector<std::int32_t>{1}));
      CHECK(r.job_accepted[0] && !r.job_accepted[1] && r.job_accepted[2]);
    }
    // check_conflicts + apply vs the reference on real tables
    for (std::uint64_t seed = 0; seed < 6; ++seed) {
      const Instance inst = seed % 2 ? random_instance(300, 70 + seed) : random_int_instance(300, 70 + seed, 50);
      const auto asg = make_assignment(inst, random_perm(300, seed));
      DeltaTables t;
      evaluate_all_parallel(inst, asg, t, {});
      const auto sr = check_conflicts(t, asg);
      const auto sg = gpu::check_conflicts(t, asg);
      CHECK(sr.reserved == sg.reserved && sr.conflicted == sg.conflicted &&
            sr.conflicted_jobs == sg.conflicted_jobs && sr.agent_accepted == sg.agent_accepted &&
            sr.job_accepted == sg.job_accepted);
      const auto [o1, a1] = apply_parallel_switches(inst, asg, t, sr, {});
      const auto [o2, a2] = gpu::apply_parallel_switches(inst, asg, t, sr);
      CHECK(o1.sigma == o2.sigma && o1.tau == o2.tau && o1.value == o2.value && a1.size() == a2.size());
      for (std::size_t q = 0; q < a1.size() && q < a2.size(); ++q)
        CHECK(a1[q].agent == a2[q].agent && a1[q].new_job == a2[q].new_job && a1[q].old_job == a2[q].old_job &&
              a1[q].displaced == a2[q].displaced && a1[q].delta == a2[q].delta);
    }
    // dgs_parallel, bit for bit
    solve_both(Instance(2, {0, 10, 10, 0}), 3);
    for (const std::int32_t n : {64, 128}) solve_both(generate_geom({n, 100.0, 47 + static_cast<std::uint64_t>(n)}), 12);
    for (const std::int32_t n : {64, 256, 1024}) solve_both(generate_geom({n, 100.0, derive_instance_seed(7, n, 0)}), 5);
    solve_both(generate_geom({48, 100.0, 59}), 4);
    solve_both(generate_geom({48, 100.0, 59}), 4, ParallelConfig::Reeval::touched_only);
    solve_both(generate_geom({512, 100.0, 61}), 21, ParallelConfig::Reeval::touched_and_conflicted, 0.05);
    solve_both(random_int_instance(2000, 0, 1000), 0);
    solve_both(random_instance(1500, 9, 1.0), 2);
    for (std::uint64_t seed = 0; seed < 20; ++seed) solve_both(random_instance(3 + seed % 5, 9500 + seed), seed + 1);
    // errors: same exception type and message
    {
      Instance bad(2, {0.0, NAN, 1.0, 2.0});
      std::string ref_msg, gpu_msg;
      try { dgs_parallel(bad, {}); } catch (const Error& e) { ref_msg = e.what(); }
      try { gpu::dgs_parallel(bad, {}); } catch (const Error& e) { gpu_msg = e.what(); }
      CHECK(!ref_msg.empty() && ref_msg == gpu_msg);
      gpu::GpuConfig c;
      c.improvement_epsilon = -1.0;
      try { gpu::dgs_parallel(generate_geom({8, 100.0, 1}), c); CHECK(false); } catch (const Error&) {}
    }
    // anytime deadline: valid permutation, terminated_by == deadline
    {
      gpu::GpuConfig c;
      c.seed = 21;
      c.deadline = Duration{0};
      const Instance inst = generate_geom({96, 100.0, 61});
      const auto cut = gpu::dgs_parallel(inst, c);
      CHECK(cut.terminated_by == Termination::deadline);
      validate_assignment(inst, cut.assignment);
    }
    // greedy start (extension): a valid, deterministic assignment
    {
      gpu::GpuConfig c;
      c.greedy_init = true;
      const Instance inst = random_int_instance(700, 31, 1000);
      const auto r1 = gpu::dgs_parallel(inst, c);
      const auto r2 = gpu::dgs_parallel(inst, c);
      validate_assignment(inst, r1.assignment);
      CHECK(r1.assignment.sigma == r2.assignment.sigma && r1.assignment.value == r2.assignment.value);
      CHECK(r1.assignment.value == objective(inst, r1.assignment));
    }
    // auction_solve, bit for bit (test_baselines.cpp:62-160 instances + C1/P2P)
    {
      auto auction_both = [](const Instance& inst, const AuctionConfig& cfg) {
        std::vector<std::vector<double>> rr, rg;
        const auto ref = auction_solve(inst, cfg, [&](const std::vector<double>& p) { rr.push_back(p); });
        const auto got = gpu::auction_solve(inst, cfg, [&](const std::vector<double>& p) { rg.push_back(p); });
        CHECK(ref.assignment.sigma == got.assignment.sigma && ref.assignment.tau == got.assignment.tau);
        CHECK(std::memcmp(&ref.assignment.value, &got.assignment.value, 8) == 0);
        CHECK(ref.outer_iterations == got.outer_iterations && ref.switches_applied == got.switches_applied);
        CHECK(ref.terminated_by == got.terminated_by && ref.completed_greedily == got.completed_greedily);
        CHECK(rr == rg);  // every round's price vector
      };
      AuctionConfig c;
      c.epsilon = 0.1;
      auction_both(Instance(2, {0, 10, 10, 0}), c);
      auction_both(Instance(1, {4.2}), {});
      auction_both(generate_geom({24, 100.0, 17}), {});
      AuctionConfig sc;
      sc.scaling = true;
      auction_both(generate_geom({48, 100.0, 23}), sc);
      auction_both(generate_geom({128, 100.0, 31}), {});
      auction_both(random_int_instance(1000, 0, 1000), {});
      for (std::uint64_t seed = 0; seed < 12; ++seed) {
        const std::int32_t n = 2 + static_cast<std::int32_t>(seed % 6);
        AuctionConfig e;
        e.epsilon = 0.9 / n;
        auction_both(random_int_instance(n, 4000 + seed, 50), e);
      }
      AuctionConfig d;
      d.deadline = Duration{0};
      const Instance g256 = generate_geom({256, 100.0, 5});
      const auto ref = auction_solve(g256, d);
      const auto got = gpu::auction_solve(g256, d);
      CHECK(got.terminated_by == Termination::deadline && got.completed_greedily);
      CHECK(ref.assignment.sigma == got.assignment.sigma);
      validate_assignment(g256, got.assignment);
      AuctionConfig bad;
      bad.epsilon = 0.0;
      std::string ref_msg, gpu_msg;
      try { auction_solve(g256, bad); } catch (const Error& e) { ref_msg = e.what(); }
      try { gpu::auction_solve(g256, bad); } catch (const Error& e) { gpu_msg = e.what(); }
      CHECK(!ref_msg.empty() && ref_msg == gpu_msg);
    }
    {  // engine plumbing (bench.cpp:77-96,210-253,281-396; lsap_bench.cpp:172-186)
      const EngineSpec sp = gpu::parse_engine_spec(" dgs-gpu:eps=0.5:reeval=touched ");
      CHECK(sp.name == "dgs-gpu" && sp.display == "dgs-gpu:eps=0.5:reeval=touched");
      CHECK(sp.params.at("eps") == "0.5" && sp.params.at("reeval") == "touched");
      CHECK(gpu::parse_engine_spec("dgs-par:workers=2").name == "dgs-par");
      std::string m1, m2;
      try { gpu::parse_engine_spec("dgs-warp"); } catch (const Error& e) { m1 = e.what(); }
      try { parse_engine_spec("dgs-warp"); } catch (const Error& e) { m2 = e.what(); }
      CHECK(!m1.empty() && m1 == m2);
      m1.clear();
      try { gpu::parse_engine_spec("dgs-gpu:eps"); } catch (const Error& e) { m1 = e.what(); }
      CHECK(m1 == "bad engine parameter 'eps' in 'dgs-gpu:eps'");
      m1.clear();
      try {
        gpu::run_engine(gpu::parse_engine_spec("dgs-gpu:reeval=sometimes"), generate_geom({16, 100.0, 1}), 0, {});
      } catch (const Error& e) { m1 = e.what(); }
      CHECK(m1 == "unknown reeval policy 'sometimes'");
      // campaign cells: every GPU engine row equals its CPU engine's row
      CampaignSpec cs;
      cs.sizes = {48, 300};
      cs.instances_per_size = 2;
      cs.repetitions = 2;
      cs.base_seed = 7;
      for (const char* e : {"dgs-par", "dgs-gpu", "dgs-par:reeval=touched:eps=0.01", "dgs-gpu:reeval=touched:eps=0.01",
                            "auction", "auction-gpu", "auction:scaling=1", "auction-gpu:scaling=1", "dgs-seq"})
        cs.engines.push_back(gpu::parse_engine_spec(e));
      cs.parallel_cells = 3;
      std::ostringstream csv, summary;
      CHECK(gpu::run_campaign(cs, csv, summary));
      std::istringstream in(csv.str());
      std::string line;
      std::getline(in, line);
      CHECK(line == csv_header());
      std::map<std::tuple<std::string, std::int32_t, std::uint64_t, std::uint64_t>, BenchRecord> rows;
      int nrows = 0;
      while (std::getline(in, line)) {
        const BenchRecord r = parse_csv_row(line);
        rows[{r.engine, r.n, r.instance_seed, r.run_seed}] = r;
        ++nrows;
      }
      CHECK(nrows == 2 * 2 * 2 * 9);
      int pairs = 0;
      for (const auto& [key, r] : rows) {
        const std::string& eng = std::get<0>(key);
        const auto pos = eng.find("-gpu");
        if (pos == std::string::npos) continue;
        const std::string cpu = eng.substr(0, pos) + (eng.substr(0, pos) == "dgs" ? "-par" : "") + eng.substr(pos + 4);
        const auto it = rows.find({cpu, std::get<1>(key), std::get<2>(key), std::get<3>(key)});
        CHECK(it != rows.end());
        if (it == rows.end()) continue;
        CHECK(r.objective == it->second.objective);
        CHECK(r.iterations == it->second.iterations);
        CHECK(r.terminated_by == it->second.terminated_by && r.terminated_by == "converged");
        ++pairs;
      }
      CHECK(pairs == 4 * 2 * 2 * 2);
      CHECK(summary.str().find("dgs-gpu") != std::string::npos);
      // the solve command's JSON record: the "kernel" field
      const Instance gi = generate_geom({300, 100.0, 3});
      const EngineSpec dg = gpu::parse_engine_spec("dgs-gpu"), dp = gpu::parse_engine_spec("dgs-par");
      const auto rg = gpu::run_engine(dg, gi, 5, {});
      const auto rp = gpu::run_engine(dp, gi, 5, {});
      CHECK(rg.assignment.sigma == rp.assignment.sigma);
      const std::string jg = gpu::solve_record_json(dg, gi, rg), jp = gpu::solve_record_json(dp, gi, rp);
      CHECK(jg.find("\"kernel\":\"sm_100a:") != std::string::npos);
      CHECK(jp.find(std::string("\"kernel\":\"") + kernels::active().name + "\"") != std::string::npos);
      CHECK(jg.find("\"engine\":\"dgs-gpu\"") != std::string::npos && jg.find("\"n\":300") != std::string::npos);
      std::printf("engine record: %s\n", jg.c_str());
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
