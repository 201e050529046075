// Latency of the C++ drop-in API on BASELINE config C3 (development tool):
//   * dp_partition(order_samples(mb, Sort), make_slice_cost(...), opts) for ONE
//     mini-batch per call — the reference planner's call pattern
//     (planner.cpp:42-65), each host thread planning its own mini-batches
//     like run_plan's pool (driver.cpp:222-242);
//   * plan_minibatches over a batch, MicroBatchPartition assembly included.
//   g++ -std=c++20 -O2 -Iinclude -o build/dropin_latency tools/dropin_latency.cpp \
//       -Lpaper_2311_10418_b200 -lpipeplan_b200 -Wl,-rpath,$PWD/paper_2311_10418_b200 -lpthread
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#include "pipeplan/cost_model.h"
#include "pipeplan/microbatch.h"
#include "pipeplan/workload.h"

using namespace pipeplan;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
  const int M = argc > 1 ? std::atoi(argv[1]) : 48;  // mini-batches
  const int n = 8192, C = 16;
  DatasetSpec spec;
  spec.synthetic = SyntheticSpec{(std::int64_t)n * M, LengthDistribution{}, std::nullopt};
  spec.max_seq_len = 8192;
  spec.seed = 7;
  const std::vector<Sample> all = load_dataset(spec);
  const ProfileGrid grid = ProfileGrid::synthetic(SyntheticGridParams{});
  const ModelConfig model = ModelConfig::uniform(C, 2, 1024, false);
  std::vector<MiniBatch> mbs(M);
  for (int k = 0; k < M; ++k) mbs[k].samples.assign(all.begin() + (std::size_t)k * n, all.begin() + (std::size_t)(k + 1) * n);
  // BASELINE C3: cap = 4 x the largest singleton act_mem, I = 3130.9824
  DpOptions opt;
  opt.stage_count = C;
  opt.replica_count = 1;
  {
    const auto ordered = order_samples(mbs[0], OrderMethod::Sort);
    const auto cost = make_slice_cost(grid, model, ordered, Recompute::None);
    double mx = 0.0;
    for (std::size_t i = 0; i < ordered.size(); ++i) mx = std::max(mx, cost(i, i + 1).act_mem);
    opt.per_mb_mem_cap = 4.0 * mx;
  }
  opt.t_max_interval = 3130.9824000000003;

  auto plan_one = [&](int k) {
    const auto ordered = order_samples(mbs[k], OrderMethod::Sort);
    const auto cost = make_slice_cost(grid, model, ordered, Recompute::None);
    return dp_partition(ordered, cost, opt);
  };
  plan_one(0);  // warm-up (context, buffers)
  // one thread, one mini-batch per call
  std::vector<double> lat;
  for (int k = 0; k < std::min(M, 16); ++k) {
    const auto t0 = Clock::now();
    const auto p = plan_one(k);
    lat.push_back(std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
    if (p.micro_batches.empty()) return 1;
  }
  std::sort(lat.begin(), lat.end());
  std::printf("dp_partition, 1 thread: median %.3f ms, min %.3f ms per mini-batch (%.0f plans/s)\n",
              lat[lat.size() / 2], lat[0], 1e3 / lat[lat.size() / 2]);
  // run_plan's pool: T threads, each a mini-batch at a time
  for (int T : {4, 16}) {
    std::atomic<int> next{0};
    const auto t0 = Clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < T; ++w)
      pool.emplace_back([&]() {
        for (int k; (k = next++) < M;) plan_one(k);
      });
    for (auto& t : pool) t.join();
    const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    std::printf("dp_partition, %2d threads x one mini-batch per call: %d plans in %.1f ms (%.0f plans/s)\n", T, M,
                ms, M / ms * 1e3);
  }
  // batched: plan_minibatches (one device call, MicroBatchPartition assembly on the host)
  plan_minibatches(mbs, grid, model, Recompute::None, opt);
  const auto t0 = Clock::now();
  const BatchPlan bp = plan_minibatches(mbs, grid, model, Recompute::None, opt);
  const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
  std::size_t mbn = 0;
  for (const auto& p : bp.partitions) mbn += p.micro_batches.size();
  std::printf("plan_minibatches: %d plans in %.1f ms (%.0f plans/s), %zu micro-batches assembled\n", M, ms,
              M / ms * 1e3, mbn);
  return 0;
}
