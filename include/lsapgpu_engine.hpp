// lsapgpu_engine.hpp -- the B200 solvers behind the reference's engine plug
// point, so the `solve --engine` command and benchmark campaigns can run them
// next to the CPU engines:
//
//   lsap::gpu::parse_engine_spec  <- lsap::parse_engine_spec   (proj/src/bench.cpp:77-96)
//   lsap::gpu::run_engine         <- lsap::run_engine          (proj/src/bench.cpp:210-253)
//   lsap::gpu::run_campaign       <- lsap::run_campaign        (proj/src/bench.cpp:281-396)
//   lsap::gpu::solve_record_json  <- the `solve` JSON record   (proj/tools/lsap_bench.cpp:172-186)
//
// Two engine names join the reference's kKnownEngines (bench.cpp:77):
//   dgs-gpu[:eps=E][:workers=W][:chunk=C][:reeval=touched|conflicted][:device=D][:graph=0|1][:init=random|greedy]
//       -> lsap::gpu::dgs_parallel; eps / workers / chunk / reeval are the
//          dgs-par keys with the same meaning (bench.cpp:227-238), results are
//          bit-identical to dgs-par's on the same instance and seed
//   auction-gpu[:epsilon=E][:scaling=0|1][:scale_factor=F][:device=D]
//       -> lsap::gpu::auction_solve, the auction keys (bench.cpp:241-246)
// Every other name is delegated to the reference unchanged.  The JSON
// "kernel" field, lsap::kernels::active().name for CPU engines, names the
// device scan for GPU engines ("sm_100a:<kernel>").
//
// Include after the reference headers lsap/{types,parallel,baselines,bench,
// geom,kernels}.hpp; link liblsapgpu.so and the reference library.
#pragma once

#include <atomic>
#include <cmath>
#include <cstdint>
#include <iomanip>
#include <map>
#include <optional>
#include <ostream>
#include <sstream>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "lsapgpu.hpp"

namespace lsap::gpu {

namespace engine_detail {

inline std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

inline std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  out.push_back(cur);
  return out;
}

inline double to_double(const std::string& s, const std::string& what) {
  try {
    std::size_t used = 0;
    const double v = std::stod(s, &used);
    if (used == s.size()) return v;
  } catch (const std::exception&) {
  }
  throw Error("invalid " + what + ": '" + s + "'");
}

inline long long to_int(const std::string& s, const std::string& what) {
  try {
    std::size_t used = 0;
    const long long v = std::stoll(s, &used);
    if (used == s.size()) return v;
  } catch (const std::exception&) {
  }
  throw Error("invalid " + what + ": '" + s + "'");
}

inline bool to_bool(const std::string& s) { return s == "1" || s == "true" || s == "yes"; }

}  // namespace engine_detail

inline const char* const kGpuEngines[] = {"dgs-gpu", "auction-gpu"};

inline bool is_gpu_engine(const std::string& name) {
  for (const char* k : kGpuEngines)
    if (name == k) return true;
  return false;
}

// parse_engine_spec with the GPU names registered: same "name[:key=value...]"
// syntax and the same errors as bench.cpp:80-96.
inline EngineSpec parse_engine_spec(const std::string& text) {
  using namespace engine_detail;
  const std::string display = trim(text);
  const auto parts = split(display, ':');
  if (!is_gpu_engine(parts[0])) return lsap::parse_engine_spec(text);
  EngineSpec spec;
  spec.display = display;
  spec.name = parts[0];
  for (std::size_t p = 1; p < parts.size(); ++p) {
    const auto kv = split(parts[p], '=');
    if (kv.size() != 2 || kv[0].empty())
      throw Error("bad engine parameter '" + parts[p] + "' in '" + text + "'");
    spec.params[kv[0]] = kv[1];
  }
  return spec;
}

// run_engine: GPU engines on the device, every other engine through the
// reference (bench.cpp:210-253).  Timing covers solver work only, as there.
inline SolveReport run_engine(const EngineSpec& engine, const Instance& inst, std::uint64_t seed,
                              const std::optional<Duration>& deadline) {
  using namespace engine_detail;
  const auto get = [&](const char* key) -> std::optional<std::string> {
    const auto it = engine.params.find(key);
    if (it == engine.params.end()) return std::nullopt;
    return it->second;
  };
  if (engine.name == "dgs-gpu") {
    GpuConfig cfg;
    cfg.seed = seed;
    cfg.deadline = deadline;
    if (auto v = get("eps")) cfg.improvement_epsilon = to_double(*v, "eps");
    if (auto v = get("workers")) cfg.workers = static_cast<std::int32_t>(to_int(*v, "workers"));
    if (auto v = get("chunk")) cfg.chunk = static_cast<std::int32_t>(to_int(*v, "chunk"));
    if (auto v = get("reeval")) {
      if (*v == "touched")
        cfg.reeval = ParallelConfig::Reeval::touched_only;
      else if (*v == "conflicted")
        cfg.reeval = ParallelConfig::Reeval::touched_and_conflicted;
      else
        throw Error("unknown reeval policy '" + *v + "'");
    }
    if (auto v = get("device")) cfg.device = static_cast<int>(to_int(*v, "device"));
    if (auto v = get("graph")) cfg.use_graph = to_bool(*v);
    if (auto v = get("init")) {
      if (*v == "greedy")
        cfg.greedy_init = true;
      else if (*v != "random")
        throw Error("unknown init '" + *v + "'");
    }
    return dgs_parallel(inst, cfg);
  }
#ifndef LSAPGPU_NO_AUCTION
  if (engine.name == "auction-gpu") {
    AuctionConfig cfg;
    cfg.deadline = deadline;
    if (auto v = get("epsilon")) cfg.epsilon = to_double(*v, "epsilon");
    if (auto v = get("scaling")) cfg.scaling = to_bool(*v);
    if (auto v = get("scale_factor")) cfg.scale_factor = to_double(*v, "scale_factor");
    int device = 0;
    if (auto v = get("device")) device = static_cast<int>(to_int(*v, "device"));
    return auction_solve(inst, cfg, {}, device);
  }
#endif
  return lsap::run_engine(engine, inst, seed, deadline);
}

// The exchange-scan implementation an engine runs, for the JSON "kernel"
// field: the reference's ISA variant for CPU engines, the device scan plan
// of this thread's context for GPU engines (call after the solve).
inline std::string kernel_name(const EngineSpec& engine) {
  if (!is_gpu_engine(engine.name)) return lsap::kernels::active().name;
  int device = 0;
  if (const auto it = engine.params.find("device"); it != engine.params.end())
    device = static_cast<int>(engine_detail::to_int(it->second, "device"));
  if (engine.name == "auction-gpu") return "sm_100a:auction-cluster";
  std::int32_t info[9] = {};
  const int k = lsapgpu_scan_plan(context(device).get(), info, 9);
  if (k < 4) return "sm_100a";
  static const char* const names[] = {"streaming", "resident", "filter"};
  std::string s = std::string("sm_100a:") + names[info[0] < 0 || info[0] > 2 ? 0 : info[0]];
  if (info[0] == 2) s += std::to_string(info[3]);
  return s;
}

// The `solve` command's JSON record (lsap_bench.cpp:172-186), without the
// optional hungarian oracle fields.
inline std::string solve_record_json(const EngineSpec& engine, const Instance& inst, const SolveReport& rep) {
  std::ostringstream o;
  o << std::setprecision(17);
  auto str = [&](const std::string& s) {
    o << '"';
    for (char ch : s) {
      if (ch == '"' || ch == '\\') o << '\\';
      o << ch;
    }
    o << '"';
  };
  o << "{\"engine\":";
  str(engine.display);
  o << ",\"n\":" << inst.n << ",\"objective\":" << rep.assignment.value << ",\"elapsed_ms\":"
    << std::chrono::duration_cast<std::chrono::duration<double, std::milli>>(rep.elapsed).count()
    << ",\"iterations\":" << rep.outer_iterations << ",\"switches\":" << rep.switches_applied
    << ",\"terminated_by\":";
  str(to_string(rep.terminated_by));
  o << ",\"kernel\":";
  str(kernel_name(engine));
  if (rep.completed_greedily) o << ",\"completed_greedily\":true";
  o << "}";
  return o.str();
}

// run_campaign with the GPU engines (the cell loop of bench.cpp:281-396 with
// this run_engine): same instances (generate_geom on derive_instance_seed),
// same run seeds, same CSV rows and summary table.  Cells that run in
// parallel host threads each get their own device context.
inline bool run_campaign(const CampaignSpec& spec, std::ostream& csv, std::ostream& summary) {
  spec.validate();
  struct Cell {
    std::int32_t size_idx, inst_idx, engine_idx, rep_idx;
  };
  std::vector<Cell> cells;
  for (std::int32_t s = 0; s < static_cast<std::int32_t>(spec.sizes.size()); ++s)
    for (std::int32_t ii = 0; ii < spec.instances_per_size; ++ii)
      for (std::int32_t e = 0; e < static_cast<std::int32_t>(spec.engines.size()); ++e)
        for (std::int32_t r = 0; r < spec.repetitions; ++r) cells.push_back({s, ii, e, r});
  const std::int32_t inst_count = static_cast<std::int32_t>(spec.sizes.size()) * spec.instances_per_size;
  std::vector<Instance> instances(inst_count);
  std::vector<std::uint64_t> instance_seeds(inst_count);
  std::vector<std::optional<double>> optima(inst_count);
  for (std::int32_t s = 0; s < static_cast<std::int32_t>(spec.sizes.size()); ++s)
    for (std::int32_t ii = 0; ii < spec.instances_per_size; ++ii) {
      const std::int32_t slot = s * spec.instances_per_size + ii;
      instance_seeds[slot] = derive_instance_seed(spec.base_seed, spec.sizes[s], ii);
      instances[slot] = generate_geom({spec.sizes[s], spec.bound, instance_seeds[slot]});
      if (spec.with_oracle) optima[slot] = hungarian_solve(instances[slot]).assignment.value;
    }
  std::vector<BenchRecord> records(cells.size());
  std::vector<char> failed(cells.size(), 0);
  std::vector<std::string> errors(cells.size());
  const auto run_cell = [&](std::size_t c) {
    const Cell& cell = cells[c];
    const std::int32_t slot = cell.size_idx * spec.instances_per_size + cell.inst_idx;
    BenchRecord rec;
    rec.engine = spec.engines[cell.engine_idx].display;
    rec.n = spec.sizes[cell.size_idx];
    rec.instance_seed = instance_seeds[slot];
    rec.run_seed = derive_run_seed(instance_seeds[slot], cell.rep_idx);
    try {
      const SolveReport rep =
          lsap::gpu::run_engine(spec.engines[cell.engine_idx], instances[slot], rec.run_seed, spec.deadline);
      rec.objective = rep.assignment.value;
      rec.elapsed_ms = std::chrono::duration_cast<std::chrono::duration<double, std::milli>>(rep.elapsed).count();
      rec.iterations = rep.outer_iterations;
      rec.terminated_by = to_string(rep.terminated_by);
      if (optima[slot]) {
        rec.optimal = optima[slot];
        if (*rec.optimal != 0.0) rec.gap = (*rec.optimal - rec.objective) / *rec.optimal;
      }
    } catch (const std::exception& ex) {
      rec.terminated_by = "error";
      failed[c] = 1;
      errors[c] = ex.what();
    }
    records[c] = std::move(rec);
  };
  if (spec.parallel_cells > 1) {
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> pool;
    const int k = static_cast<int>(std::min<std::int64_t>(spec.parallel_cells, static_cast<std::int64_t>(cells.size())));
    for (int t = 0; t < k; ++t)
      pool.emplace_back([&] {
        for (std::size_t c; (c = next.fetch_add(1)) < cells.size();) run_cell(c);
      });
    for (auto& t : pool) t.join();
  } else {
    for (std::size_t c = 0; c < cells.size(); ++c) run_cell(c);
  }
  for (std::size_t c = 0; c < cells.size(); ++c)
    if (failed[c])
      summary << "# cell failed: engine=" << records[c].engine << " n=" << records[c].n
              << " rep=" << cells[c].rep_idx << ": " << errors[c] << "\n";
  csv << csv_header() << "\n";
  bool all_ok = true;
  for (std::size_t c = 0; c < cells.size(); ++c) {
    csv << to_csv_row(records[c]) << "\n";
    all_ok &= !failed[c];
  }
  // per-(engine, size) mean / stddev in first-appearance order
  struct Mom {
    std::int64_t count = 0;
    double sum = 0.0, sq = 0.0;
    void add(double v) {
      ++count;
      sum += v;
      sq += v * v;
    }
    double mean() const { return count ? sum / count : 0.0; }
    double sd() const {
      if (count < 2) return 0.0;
      const double m = mean();
      return std::sqrt(std::max(0.0, sq / count - m * m));
    }
  };
  std::vector<std::pair<std::string, std::int32_t>> keys;
  std::map<std::pair<std::string, std::int32_t>, std::pair<Mom, Mom>> agg;
  std::map<std::pair<std::string, std::int32_t>, Mom> gap_agg;
  for (std::size_t c = 0; c < cells.size(); ++c) {
    if (failed[c]) continue;
    const auto key = std::make_pair(records[c].engine, records[c].n);
    if (agg.find(key) == agg.end()) keys.push_back(key);
    agg[key].first.add(records[c].objective);
    agg[key].second.add(records[c].elapsed_ms);
    if (records[c].gap) gap_agg[key].add(*records[c].gap);
  }
  summary << std::left << std::setw(28) << "engine" << std::right << std::setw(7) << "n" << std::setw(6) << "runs"
          << std::setw(16) << "mean_obj" << std::setw(13) << "sd_obj" << std::setw(13) << "mean_ms";
  if (spec.with_oracle) summary << std::setw(13) << "mean_gap";
  summary << "\n";
  for (const auto& key : keys) {
    const auto& [obj, ms] = agg[key];
    summary << std::left << std::setw(28) << key.first << std::right << std::setw(7) << key.second << std::setw(6)
            << obj.count << std::setw(16) << std::fixed << std::setprecision(3) << obj.mean() << std::setw(13)
            << obj.sd() << std::setw(13) << ms.mean();
    if (spec.with_oracle) {
      const auto git = gap_agg.find(key);
      summary << std::setw(13) << std::setprecision(6) << (git == gap_agg.end() ? 0.0 : git->second.mean());
    }
    summary << "\n";
  }
  if (spec.parallel_cells > 1) summary << "# timings contended: cells ran " << spec.parallel_cells << "-way parallel\n";
  return all_ok;
}

}  // namespace lsap::gpu
