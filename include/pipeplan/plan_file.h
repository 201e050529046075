// pipeplan/plan_file.h — the on-disk outputs of whole-epoch planning from
// plans emitted on the device.
//
// The reference's run_plan (src/driver.cpp:203-283) writes, per iteration and
// replica, the ExecutionPlan text of save_plan (src/comm_plan.cpp:313-342)
// into iter_<i>_replica_<d>.plan and one plans_index.csv row.  Here the plan
// comes from pp_emit_plans (include/pipeplan_b200.h): per stage, the packed
// instruction list (micro_batch << 4 | InstrKind) of
// plan_communication(schedule(...)); these functions format it and the index
// row byte for byte like the reference (peers and transfer shapes follow from
// the stage and the micro-batch's padded shape, comm_plan.cpp:104-113).
#pragma once

#include <cstdint>
#include <ostream>
#include <string>
#include <vector>

#include "pipeplan/cost_model.h"

namespace pipeplan {
namespace b200 {

// One replica's plan as pp_emit_plans returns it, plus the metadata
// plan_iteration puts into its PlanMeta (src/planner.cpp:86-95).
struct EmittedPlan {
  std::int64_t iteration = 0;
  int replica = 0;
  std::int64_t hidden_dim = 0;
  bool encoder_decoder = false;
  Recompute recompute = Recompute::None;
  std::vector<StageLayout> stage_layers;                 // one per stage
  std::vector<PaddedShape> shapes;                       // the replica's micro-batches, in partition order
  std::vector<std::vector<std::int32_t>> devices;        // per stage: (micro_batch << 4) | InstrKind
};

// save_plan's text (src/comm_plan.cpp:313-342).
void save_plan_text(const EmittedPlan& plan, std::ostream& out);
std::string plan_to_text(const EmittedPlan& plan);

// plans_index.csv (src/driver.cpp:246-283): the header line, a feasible
// replica's row and an infeasible iteration's row (doubles as %.17g, ',' and
// '\n' in the reason replaced by ';').
std::string plans_index_header();
struct IndexRow {
  std::int64_t iteration = 0;
  int replica = 0;
  std::size_t micro_batches = 0;
  Recompute strategy = Recompute::None;
  double objective = 0.0, t_max = 0.0, max_replica_load = 0.0;
  double padding_eff_input = 0.0, padding_eff_target = 0.0;
  double predicted_makespan = 0.0, bubble_ratio = 0.0, peak_mem_max = 0.0;
};
std::string plans_index_row(const IndexRow& row);
std::string plans_index_infeasible_row(std::int64_t iteration, const std::string& reason);

}  // namespace b200
}  // namespace pipeplan
