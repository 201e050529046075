// order_search.h — the per-replica injection-order search on the B200
// (SURVEY.md §8f row 1), C++ face of pp_order_search (include/pipeplan_b200.h).
//
// The reference planner (proj/src/planner.cpp:94-108) calls
//   order_microbatches(predicted, sel.costs, limits, n_clusters, evaluator)
// (schedule.cpp:277-317) with evaluator = makespan of
//   simulate(plan_communication(sched, sel.costs, meta), sel.costs,
//            {noise_sigma 0, comm_latency})
// and then re-simulates the chosen order for rep.report.  The generic
// order_microbatches takes an arbitrary std::function evaluator, which cannot
// run on a device, so the drop-in is this function: the same search with that
// fixed evaluator, batched over any number of replicas / mini-batches, and the
// chosen order's SimReport summary alongside (INTEGRATION.md §3 shows the
// two-line change in planner.cpp).  Results are bit-identical to the
// reference's; errors are the reference's exception types and messages.
#pragma once

#include <span>
#include <vector>

#include "pipeplan/cost_model.h"

namespace pipeplan::b200 {

struct DeviceStatsSummary {  // simulate.h:30-36 DeviceStats
  double busy = 0.0;
  double idle = 0.0;
  double blocked = 0.0;
  double peak_mem = 0.0;
  double final_mem = 0.0;
};

struct InjectionOrder {
  std::vector<int> order;     // order_microbatches' result (empty: none selectable)
  double makespan = 0.0;      // SimReport of the chosen order (planner.cpp:107)
  double bubble_ratio = 0.0;
  bool deadlock = false;
  std::vector<DeviceStatsSummary> devices;
};

/// order_microbatches(scalar_time predictions, costs, limits, n_clusters,
/// planner evaluator) for every table in one batched device call.  All
/// tables share `limits` (one per stage) and the stage count.  Throws
/// std::invalid_argument (schedule.cpp:281-284, 62-66) or std::logic_error
/// (schedule.cpp:81-82, 155-156) for the first failing table, like a loop
/// over the reference would.  Device limits (std::invalid_argument where
/// the reference would return an order): stages <= 32, n_clusters <= 12, and
/// op durations >= 0 and not NaN (the Start lists are merged from per-device
/// sorted op ends).
std::vector<InjectionOrder> search_injection_orders(std::span<const OpCostTable> tables,
                                                    std::span<const double> limits, int n_clusters,
                                                    double comm_latency = 0.0);

/// One table (plan_iteration's per-replica call).
InjectionOrder search_injection_order(const OpCostTable& costs, std::span<const double> limits,
                                      int n_clusters, double comm_latency = 0.0);

}  // namespace pipeplan::b200
