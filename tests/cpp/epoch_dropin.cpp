// Whole-epoch planning on the device (pipeplan::b200::plan_epoch) against the
// reference's own run_plan (proj/src/driver.cpp:203-283, compiled where it
// lies with planner.cpp / schedule.cpp / comm_plan.cpp / simulate.cpp and
// linked, for its hot path, with this repo's drop-in library — the
// acceptance_dropin setup).  For each configuration both write
// plans_index.csv and every iter_<i>_replica_<d>.plan; the files must be
// identical byte for byte.  Test infrastructure (tests/test_dropin.py).
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include "pipeplan/driver.h"
#include "pipeplan/epoch.h"

namespace fs = std::filesystem;
using namespace pipeplan;

static std::string slurp(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(in), {});
}

int main(int argc, char** argv) {
  const fs::path root = argc > 1 ? fs::path(argv[1]) : fs::temp_directory_path() / "pp_epoch_dropin";
  struct Case {
    const char* name;
    int stages, replicas;
    bool encdec, adaptive;
    std::int64_t n, budget;
    double limit, interval;
    int clusters;
    std::vector<Recompute> recompute;
  };
  const std::vector<Case> cases = {
      {"gpt_adaptive", 4, 1, false, true, 3000, 8192, 4.0, 5.0, 3, {Recompute::None, Recompute::Selective, Recompute::Full}},
      {"t5_adaptive_d2", 4, 2, true, true, 2500, 16384, 6.0, 20.0, 3, {Recompute::None, Recompute::Full}},
      {"gpt_1f1b", 8, 1, false, false, 3000, 16384, 2.0, 50.0, 3, {Recompute::Selective, Recompute::Full}},
      {"gpt_tight", 4, 1, false, true, 2000, 8192, 0.35, 5.0, 2, {Recompute::None, Recompute::Selective}},
  };
  int failures = 0;
  for (const Case& c : cases) {
    RunConfig cfg;
    cfg.dataset.synthetic = SyntheticSpec{c.n, LengthDistribution{}, std::nullopt};
    if (c.encdec) {
      LengthDistribution t;
      t.log_mean = 3.5;
      t.log_sigma = 1.2;
      cfg.dataset.synthetic->target = t;
    }
    cfg.dataset.max_seq_len = 8192;
    cfg.dataset.seed = 11;
    cfg.token_budget = c.budget;
    cfg.stages = c.stages;
    cfg.replicas = c.replicas;
    cfg.encoder_decoder = c.encdec;
    cfg.recompute = c.recompute;
    cfg.device_limits.assign(static_cast<std::size_t>(c.stages), 0.0);
    cfg.t_max_interval = c.interval;
    cfg.n_clusters = c.clusters;
    cfg.policy = c.adaptive ? SchedulePolicy::Adaptive : SchedulePolicy::OneFOneB;
    cfg.workers = 16;  // run_plan's pool on every host core of the box
    // limits: a multiple of the largest single-sample act_mem of the grid
    const ProfileGrid grid = make_grid(cfg);
    const ModelConfig model = make_model(cfg);
    double amax = 0.0;
    for (int s = 0; s < c.stages; ++s)
      amax = std::max(amax, estimate(grid, model, s, 1, 8192, c.encdec ? 8192 : 0, Recompute::None).act_mem);
    for (double& l : cfg.device_limits) l = c.limit * amax * 8.0;
    cfg.output_dir = (root / c.name / "reference").string();
    std::ostringstream log;
    const auto r0 = std::chrono::steady_clock::now();
    run_plan(cfg, log);
    const double ref_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();

    b200::EpochConfig ec;
    ec.token_budget = cfg.token_budget;
    ec.replicas = cfg.replicas;
    ec.device_limits = cfg.device_limits;
    ec.t_max_interval = cfg.t_max_interval;
    ec.n_clusters = cfg.n_clusters;
    ec.adaptive = c.adaptive;
    ec.comm_latency = cfg.comm_latency;
    ec.output_dir = (root / c.name / "device").string();
    const auto samples = load_dataset(cfg.dataset);
    const b200::EpochSummary sum = b200::plan_epoch(samples, grid, model, ec);

    int files = 0, bad = 0;
    for (const auto& e : fs::directory_iterator(cfg.output_dir)) {
      const fs::path other = fs::path(ec.output_dir) / e.path().filename();
      ++files;
      if (!fs::exists(other) || slurp(e.path()) != slurp(other)) {
        ++bad;
        if (bad <= 3) std::cout << "  MISMATCH " << c.name << ": " << e.path().filename() << "\n";
      }
    }
    int ours = 0;
    for (const auto& e : fs::directory_iterator(ec.output_dir)) { (void)e; ++ours; }
    if (ours != files) ++bad;
    std::cout << c.name << ": " << sum.iterations << " iterations (" << sum.feasible << " feasible), " << files
              << " reference files, " << ours << " device files, " << bad << " mismatches; epoch wall: reference run_plan "
              << ref_ms << " ms (16 threads), device plan_epoch " << sum.total_ms << " ms\n";
    failures += bad;
  }
  std::cout << (failures ? "FAIL" : "OK") << "\n";
  return failures ? 1 : 0;
}
