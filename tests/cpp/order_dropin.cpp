// order_dropin.cpp — the device injection-order search
// (pipeplan::b200::search_injection_order{,s}, include/pipeplan/order_search.h)
// against the reference's own per-replica planner, compiled where it lies:
//  1. random op-cost tables: order_microbatches with plan_iteration's
//     evaluator (schedule.cpp:277-317 + comm_plan.cpp:115-233 +
//     simulate.cpp:78-213), then the chosen order's SimReport;
//  2. the reference's plan_iteration (planner.cpp:17-130, Adaptive policy)
//     on synthetic mini-batches: each replica's injection order and report
//     must equal the device search over the replica's op-cost table
//     (OpCostTable::from_shapes at the selected recompute strategy, exactly
//     what select_recomputation hands to order_microbatches).
// Test infrastructure; needs a CUDA device.  Prints "order dropin: OK".
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "pipeplan/comm_plan.h"
#include "pipeplan/order_search.h"
#include "pipeplan/padding_report.h"
#include "pipeplan/planner.h"
#include "pipeplan/schedule.h"
#include "pipeplan/simulate.h"
#include "pipeplan/workload.h"

using namespace pipeplan;

static int failures = 0;

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static void check(bool ok, const char* what, int idx) {
  if (!ok) {
    std::printf("MISMATCH %s (case %d)\n", what, idx);
    ++failures;
  }
}

struct RefResult {
  std::vector<int> order;
  SimReport report;
};

static RefResult reference(const OpCostTable& costs, const std::vector<double>& lim, int k, double lat) {
  PlanMeta meta;
  meta.shape_table.assign(static_cast<std::size_t>(costs.micro_batches), MbShapeEntry{1, 1, 0});
  SimConfig zero;
  zero.comm_latency = lat;
  std::vector<double> pred(static_cast<std::size_t>(costs.micro_batches));
  for (int i = 0; i < costs.micro_batches; ++i) pred[static_cast<std::size_t>(i)] = costs.scalar_time(i);
  auto ev = [&](const PipelineSchedule& s) { return simulate(plan_communication(s, costs, meta), costs, zero).makespan; };
  RefResult r;
  r.order = order_microbatches(pred, costs, lim, k, ev);
  r.report = simulate(plan_communication(schedule_adaptive(costs, lim, r.order), costs, meta), costs, zero);
  return r;
}

static void compare(const b200::InjectionOrder& got, const RefResult& ref, int idx) {
  check(got.order == ref.order, "order", idx);
  check(same(got.makespan, ref.report.makespan), "makespan", idx);
  check(same(got.bubble_ratio, ref.report.bubble_ratio), "bubble_ratio", idx);
  check(got.deadlock == ref.report.deadlock, "deadlock", idx);
  for (std::size_t j = 0; j < ref.report.devices.size(); ++j) {
    const auto& a = got.devices[j];
    const auto& b = ref.report.devices[j];
    check(same(a.busy, b.busy) && same(a.idle, b.idle) && same(a.blocked, b.blocked) &&
              same(a.peak_mem, b.peak_mem) && same(a.final_mem, b.final_mem),
          "device stats", idx);
  }
}

int main() {
  // 1. random tables, batched in one device call per stage count
  std::mt19937_64 rng(2311);
  int cases = 0;
  for (int C : {1, 2, 4, 8, 16}) {
    std::vector<OpCostTable> tabs;
    std::vector<double> lim(static_cast<std::size_t>(C), 0.0);
    for (int t = 0; t < 24; ++t) {
      const int M = 1 + static_cast<int>(rng() % 60);
      OpCostTable c = OpCostTable::uniform(M, C, 0.0, 0.0, 0.0);
      for (std::size_t q = 0; q < c.t_f.size(); ++q) {
        c.t_f[q] = 0.25 * static_cast<double>(1 + rng() % 8);
        c.t_b[q] = 0.5 * static_cast<double>(1 + rng() % 8);
        c.act_mem[q] = 0.1 + 0.9 * std::ldexp(static_cast<double>(rng() >> 11), -53);
      }
      tabs.push_back(std::move(c));
    }
    for (int j = 0; j < C; ++j) lim[static_cast<std::size_t>(j)] = 2.0;
    for (int k : {1, 3, 4}) {
      for (double lat : {0.0, 0.25}) {
        auto got = b200::search_injection_orders(tabs, lim, k, lat);
        for (std::size_t t = 0; t < tabs.size(); ++t, ++cases)
          compare(got[t], reference(tabs[t], lim, k, lat), cases);
      }
    }
  }
  // 2. the reference planner end to end (Adaptive policy, 2 replicas)
  ProfileGrid grid = ProfileGrid::synthetic(SyntheticGridParams{});
  int planned = 0;
  for (bool encdec : {false, true}) {
    const int C = encdec ? 8 : 4;
    ModelConfig cfg = ModelConfig::uniform(C, 2, 1024, encdec);
    DatasetSpec spec;
    spec.synthetic = SyntheticSpec{};
    spec.synthetic->n = 2048;
    if (encdec) spec.synthetic->target = LengthDistribution{LengthFamily::Lognormal, 3.5, 1.2, 1, 1, 0.8};
    spec.max_seq_len = 4096;
    spec.seed = 19;
    auto samples = load_dataset(spec);
    PlanningOptions opt;
    opt.replicas = 2;
    opt.t_max_interval = 50.0;
    opt.n_clusters = 3;
    opt.policy = SchedulePolicy::Adaptive;
    opt.device_limits.assign(static_cast<std::size_t>(C), encdec ? 4000.0 : 6000.0);
    for (int it = 0; it < 4; ++it) {
      MiniBatch mb;
      mb.samples.assign(samples.begin() + it * 256, samples.begin() + (it + 1) * 256);
      opt.iteration = it;
      IterationPlanResult res = plan_iteration(mb, grid, cfg, opt);
      if (!res.feasible) continue;
      for (const auto& rep : res.replicas) {
        std::vector<PaddedShape> shapes;
        for (std::size_t i = 0; i < res.partition.micro_batches.size(); ++i)
          if (res.partition.replica_assignment[i] == rep.replica)
            shapes.push_back(res.partition.micro_batches[i].shape());
        OpCostTable costs = OpCostTable::from_shapes(grid, cfg, shapes, rep.strategy);
        auto got = b200::search_injection_order(costs, opt.device_limits, opt.n_clusters, opt.comm_latency);
        check(got.order == rep.injection_order, "planner injection order", planned);
        check(same(got.makespan, rep.report.makespan), "planner makespan", planned);
        check(same(got.bubble_ratio, rep.report.bubble_ratio), "planner bubble ratio", planned);
        ++planned;
      }
    }
  }
  // 3. padding_vs_packing_report: every row byte-identical
  int report_rows = 0;
  for (bool encdec : {false, true}) {
    ModelConfig cfg = ModelConfig::uniform(encdec ? 4 : 2, 2, 1024, encdec);
    DatasetSpec spec;
    spec.synthetic = SyntheticSpec{};
    spec.synthetic->n = 3000;
    if (encdec) spec.synthetic->target = LengthDistribution{LengthFamily::Lognormal, 3.5, 1.2, 1, 1, 0.8};
    spec.max_seq_len = 16384;
    spec.seed = 31;
    auto samples = load_dataset(spec);
    const std::vector<std::int64_t> lens = {512, 4096};
    PaddingReportOptions ro;
    ro.token_budget = 32768;
    ro.t_max_interval = 200.0;
    ro.max_iterations = 10;
    b200::PaddingReportOptions bo;
    bo.token_budget = ro.token_budget;
    bo.t_max_interval = ro.t_max_interval;
    bo.max_iterations = ro.max_iterations;
    const auto ref_rows = padding_vs_packing_report(samples, lens, grid, cfg, ro);
    const auto got = b200::padding_vs_packing_report(samples, lens, grid, cfg, bo);
    check(got.size() == ref_rows.size(), "report row count", report_rows);
    for (std::size_t k = 0; k < std::min(got.size(), ref_rows.size()); ++k, ++report_rows) {
      const auto& a = got[k];
      const auto& b = ref_rows[k];
      check(static_cast<int>(a.method) == static_cast<int>(b.method) && a.max_seq_len == b.max_seq_len &&
                same(a.padding_eff_input, b.padding_eff_input) && same(a.padding_eff_target, b.padding_eff_target) &&
                a.tokens == b.tokens && same(a.sim_time, b.sim_time) && same(a.throughput_proxy, b.throughput_proxy),
            "padding report row", report_rows);
    }
  }
  // 4. errors: the reference's exception types
  bool threw = false;
  try {
    OpCostTable c = OpCostTable::uniform(4, 2, 1.0, 2.0, 5.0);
    b200::search_injection_order(c, std::vector<double>{2.0, 2.0}, 3);
  } catch (const std::invalid_argument&) {
  } catch (const std::logic_error& e) {
    threw = std::strstr(e.what(), "converge") != nullptr;
  }
  check(threw, "non-convergence logic_error", -1);
  std::printf("order dropin: %d random tables, %d planner replicas, %d report rows, %d mismatches\n", cases,
              planned, report_rows, failures);
  if (failures == 0 && planned > 0) std::printf("order dropin: OK\n");
  return failures == 0 && planned > 0 ? 0 : 1;
}
