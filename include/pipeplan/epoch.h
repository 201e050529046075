// pipeplan/epoch.h — whole-epoch planning with every per-iteration step on
// the B200: the device counterpart of the
// reference's run_plan (src/driver.cpp:203-283) over plan_iteration
// (src/planner.cpp:31-135).
//
// For the mini-batches drawn from `samples` (draw_minibatch's token-budget
// loop, driver.cpp:209-215, on the device): ONE batched planning call
// (order_samples(Sort) -> make_slice_cost -> dp_partition, dp options as
// plan_iteration sets them), then for every (iteration, replica) at once:
// select_recomputation, the injection-order search with plan_iteration's
// evaluator (adaptive policy) or the 1F1B schedule, and the emitted plan with
// its SimReport — and the outputs of run_plan: plans_index.csv and one
// iter_<i>_replica_<d>.plan per replica, byte for byte the reference's text.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pipeplan/cost_model.h"
#include "pipeplan/workload.h"

namespace pipeplan {
namespace b200 {

// The planning fields of the reference's RunConfig (driver.h:32-63) /
// PlanningOptions (planner.h:31-40).
struct EpochConfig {
  std::int64_t token_budget = 65536;
  int replicas = 1;
  std::vector<double> device_limits;  // one per stage
  double t_max_interval = 5.0;
  int n_clusters = 3;
  bool adaptive = true;               // SchedulePolicy::Adaptive (else 1F1B)
  double comm_latency = 0.0;
  int max_iterations = 0;             // 0 = the whole epoch
  std::string output_dir = "out";
};

struct EpochSummary {
  std::size_t iterations = 0;
  std::size_t feasible = 0;
  double total_ms = 0.0;              // wall time of the whole call (drawing to the last file)
};

// Throws std::invalid_argument like plan_iteration for bad options (replicas
// < 1, one limit per stage, an empty recompute set).  The model's
// recompute_allowed is the strategy set (make_model, driver.cpp:186-191).
EpochSummary plan_epoch(const std::vector<Sample>& samples, const ProfileGrid& grid, const ModelConfig& model,
                        const EpochConfig& config);

}  // namespace b200
}  // namespace pipeplan
