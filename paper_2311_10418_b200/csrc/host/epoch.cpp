// epoch.cpp — pipeplan::b200::plan_epoch (include/pipeplan/epoch.h): the
// reference's run_plan (src/driver.cpp:203-283) / plan_iteration
// (src/planner.cpp:31-135) composed from the batched device entry points:
//   draw (pp_draw_minibatches) -> plans (plan_minibatches: pp_plan_grid) ->
//   per (iteration, replica): pp_select_recomputation -> pp_order_search
//   (adaptive) -> pp_emit_plans -> plans_index.csv + .plan files.
// Each stage runs once over the whole epoch instead of once per iteration;
// the control flow per iteration is plan_iteration's (the first failing
// replica makes the iteration infeasible with that replica's reason).
#include "pipeplan/epoch.h"

#include <algorithm>
#include <chrono>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>

#include "pipeplan/microbatch.h"
#include "pipeplan/plan_file.h"
#include "pipeplan_b200.h"

namespace pipeplan {
namespace detail {
pp_ctx* device_ctx();  // microbatch.cpp
}

namespace b200 {

namespace {

void check(pp_ctx* ctx, int rc) {
  if (rc == PP_ERR_INVALID) throw std::invalid_argument(pp_ctx_last_error(ctx));
  if (rc != PP_OK) throw std::runtime_error(std::string("pipeplan_b200 device error: ") + pp_ctx_last_error(ctx));
}

// One (iteration, replica) of the epoch: its micro-batches in partition order.
struct Rep {
  std::size_t iter = 0;
  int replica = 0;
  std::vector<PaddedShape> shapes;
};

}  // namespace

EpochSummary plan_epoch(const std::vector<Sample>& samples, const ProfileGrid& grid, const ModelConfig& model,
                        const EpochConfig& cfg) {
  const auto t0 = std::chrono::steady_clock::now();
  const int C = model.stage_count();
  if (cfg.replicas < 1) throw std::invalid_argument("replica count must be >= 1");      // planner.cpp:35
  if (static_cast<int>(cfg.device_limits.size()) != C)
    throw std::invalid_argument("one memory limit per stage required");                // :36-37
  if (model.recompute_allowed.empty())
    throw std::invalid_argument("at least one recompute strategy must be allowed");   // :38-39
  pp_ctx* ctx = detail::device_ctx();

  // ---- draw (driver.cpp:209-215), on the device
  std::vector<std::int64_t> seg(samples.size() + 1);
  std::int64_t n_seg = 0;
  check(ctx, pp_draw_minibatches(ctx, reinterpret_cast<const pp_sample*>(samples.data()),
                                 static_cast<std::int64_t>(samples.size()), cfg.token_budget, seg.data(), &n_seg));
  if (cfg.max_iterations > 0) n_seg = std::min<std::int64_t>(n_seg, cfg.max_iterations);
  std::vector<MiniBatch> mbs(static_cast<std::size_t>(n_seg));
  for (std::int64_t i = 0; i < n_seg; ++i) {
    mbs[i].samples.assign(samples.begin() + seg[i], samples.begin() + seg[i + 1]);
    mbs[i].token_budget = cfg.token_budget;
  }

  // ---- the partitions (planner.cpp:41-66): the cheapest allowed strategy,
  // the advisory cap 1/C of the tightest device, one batched device call
  Recompute dp_strategy = Recompute::Full;
  for (Recompute r : {Recompute::None, Recompute::Selective, Recompute::Full})
    if (std::find(model.recompute_allowed.begin(), model.recompute_allowed.end(), r) !=
        model.recompute_allowed.end()) {
      dp_strategy = r;
      break;
    }
  const double tightest = *std::min_element(cfg.device_limits.begin(), cfg.device_limits.end());
  DpOptions dp;
  dp.stage_count = C;
  dp.replica_count = cfg.replicas;
  dp.per_mb_mem_cap = tightest / static_cast<double>(C);
  dp.t_max_interval = cfg.t_max_interval;
  const BatchPlan bp = plan_minibatches(mbs, grid, model, dp_strategy, dp);

  // ---- per (iteration, replica): micro-batches of the replica in partition order
  std::vector<Rep> reps;
  std::vector<std::int64_t> rep_off{0};
  for (std::size_t i = 0; i < mbs.size(); ++i) {
    if (!bp.errors[i].empty()) continue;
    const MicroBatchPartition& p = bp.partitions[i];
    for (int d = 0; d < cfg.replicas; ++d) {
      Rep r{i, d, {}};
      for (std::size_t k = 0; k < p.micro_batches.size(); ++k)
        if (p.replica_assignment[k] == d) r.shapes.push_back(p.micro_batches[k].shape());
      if (r.shapes.empty()) continue;  // planner.cpp:79
      rep_off.push_back(rep_off.back() + static_cast<std::int64_t>(r.shapes.size()));
      reps.push_back(std::move(r));
    }
  }
  const int R = static_cast<int>(reps.size());
  const std::size_t rows = static_cast<std::size_t>(rep_off.back());
  std::vector<pp_padded_shape> sh;
  sh.reserve(rows);
  for (const Rep& r : reps)
    for (const PaddedShape& s : r.shapes) sh.push_back({s.mbs, s.input_len, s.target_len});

  // ---- select_recomputation for every replica at once (schedule.cpp:319-364)
  std::vector<std::int32_t> enc, dec;
  for (const StageLayout& s : model.stages) {
    enc.push_back(s.encoder_layers);
    dec.push_back(s.decoder_layers);
  }
  pp_model_desc md{C, enc.data(), dec.data(), model.is_encoder_decoder ? 1 : 0, 0};
  const pp_grid_desc gd = grid.device_desc();
  int mask = 0;
  for (Recompute r : model.recompute_allowed) mask |= 1 << static_cast<int>(r);
  std::vector<double> tf(std::max<std::size_t>(rows, 1) * C), tb(tf.size()), act(tf.size());
  std::vector<std::int32_t> strategy(std::max(R, 1)), viol(std::max(R, 1));
  if (R > 0)
    check(ctx, pp_select_recomputation(ctx, sh.data(), rep_off.data(), R, &gd, &md, mask, cfg.device_limits.data(),
                                       tf.data(), tb.data(), act.data(), strategy.data(), viol.data()));
  // an iteration with a replica that fits no strategy is infeasible with the
  // first such replica's reason (planner.cpp:122-126)
  std::vector<std::string> reason(mbs.size());
  for (std::size_t i = 0; i < mbs.size(); ++i) reason[i] = bp.errors[i];
  for (int q = 0; q < R; ++q)
    if (strategy[q] < 0 && reason[reps[q].iter].empty())
      reason[reps[q].iter] = "no recompute strategy fits the device memory limits (stage " +
                             std::to_string(viol[q]) + ")";

  // ---- injection orders (adaptive: order_microbatches with the planner's
  // evaluator, planner.cpp:94-108) and the emitted plans + SimReports
  std::vector<std::int32_t> order(std::max<std::size_t>(rows, 1), 0), st(std::max(R, 1)), dl(std::max(R, 1));
  std::vector<double> ms(std::max(R, 1)), bub(std::max(R, 1)), ds(static_cast<std::size_t>(std::max(R, 1)) * C * 5);
  // replicas of feasible iterations only (their strategy tables)
  std::vector<int> live;
  std::vector<std::int64_t> live_off{0};
  for (int q = 0; q < R; ++q)
    if (reason[reps[q].iter].empty()) {
      live.push_back(q);
      live_off.push_back(live_off.back() + static_cast<std::int64_t>(reps[q].shapes.size()));
    }
  const int L = static_cast<int>(live.size());
  const std::size_t lrows = static_cast<std::size_t>(live_off.back());
  std::vector<double> ltf(std::max<std::size_t>(lrows, 1) * C), ltb(ltf.size()), lact(ltf.size());
  for (int l = 0; l < L; ++l) {
    const std::size_t src = static_cast<std::size_t>(rep_off[live[l]]) * C;
    const std::size_t dst = static_cast<std::size_t>(live_off[l]) * C;
    const std::size_t n = reps[live[l]].shapes.size() * static_cast<std::size_t>(C);
    std::copy(tf.begin() + src, tf.begin() + src + n, ltf.begin() + dst);
    std::copy(tb.begin() + src, tb.begin() + src + n, ltb.begin() + dst);
    std::copy(act.begin() + src, act.begin() + src + n, lact.begin() + dst);
  }
  std::vector<std::int32_t> lorder(std::max<std::size_t>(lrows, 1), 0), ins(std::max<std::size_t>(lrows, 1) * 10 * C),
      nins(static_cast<std::size_t>(std::max(L, 1)) * C);
  if (L > 0) {
    if (cfg.adaptive) {
      check(ctx, pp_order_search(ctx, ltf.data(), ltb.data(), lact.data(), live_off.data(), L, C,
                                 cfg.device_limits.data(), cfg.n_clusters, cfg.comm_latency, lorder.data(), ms.data(),
                                 bub.data(), dl.data(), ds.data(), st.data()));
      for (int l = 0; l < L; ++l)
        if (st[l] == PP_ERR_NOT_CONVERGED)
          throw std::logic_error("adaptive scheduler failed to converge; invariant violated");
        else if (st[l] != PP_OK)
          throw std::logic_error("schedule is not executable: circular dependency between devices");
    }
    check(ctx, pp_emit_plans(ctx, ltf.data(), ltb.data(), lact.data(), live_off.data(), L, C,
                             cfg.device_limits.data(), cfg.comm_latency, cfg.adaptive ? 0 : 1, lorder.data(),
                             ins.data(), nins.data(), ms.data(), bub.data(), dl.data(), ds.data(), st.data()));
    for (int l = 0; l < L; ++l)
      if (st[l] == PP_ERR_NOT_CONVERGED)
        throw std::logic_error("adaptive scheduler failed to converge; invariant violated");
      else if (st[l] != PP_OK)
        throw std::logic_error("schedule is not executable: circular dependency between devices");
  }

  // ---- run_plan's outputs (driver.cpp:244-283)
  std::filesystem::create_directories(cfg.output_dir);
  std::ofstream index(std::filesystem::path(cfg.output_dir) / "plans_index.csv", std::ios::binary);
  index << plans_index_header();
  EpochSummary sum;
  sum.iterations = mbs.size();
  int l = 0;
  for (std::size_t i = 0; i < mbs.size(); ++i) {
    if (!reason[i].empty()) {
      index << plans_index_infeasible_row(static_cast<std::int64_t>(i), reason[i]);
      while (l < L && reps[live[l]].iter == i) ++l;  // (none: live replicas are feasible)
      continue;
    }
    ++sum.feasible;
    const MicroBatchPartition& p = bp.partitions[i];
    const PaddingEfficiency pad = padding_efficiency(p);
    for (; l < L && reps[live[l]].iter == i; ++l) {
      const Rep& r = reps[live[l]];
      const int q = live[l];
      const std::int64_t M = static_cast<std::int64_t>(r.shapes.size());
      EmittedPlan ep;
      ep.iteration = static_cast<std::int64_t>(i);
      ep.replica = r.replica;
      ep.hidden_dim = model.hidden_dim;
      ep.encoder_decoder = model.is_encoder_decoder;
      ep.recompute = static_cast<Recompute>(strategy[q]);
      ep.stage_layers = model.stages;
      ep.shapes = r.shapes;
      for (int j = 0; j < C; ++j) {
        const std::int32_t* a = ins.data() + 10 * C * live_off[l] + 10 * M * j;
        ep.devices.emplace_back(a, a + nins[static_cast<std::size_t>(l) * C + j]);
      }
      const auto file = std::filesystem::path(cfg.output_dir) /
                        ("iter_" + std::to_string(i) + "_replica_" + std::to_string(r.replica) + ".plan");
      std::ofstream pf(file, std::ios::binary);
      save_plan_text(ep, pf);
      IndexRow row;
      row.iteration = static_cast<std::int64_t>(i);
      row.replica = r.replica;
      row.micro_batches = r.shapes.size();
      row.strategy = ep.recompute;
      row.objective = p.objective_value;
      row.t_max = p.t_max_used;
      row.max_replica_load = p.max_replica_load;
      row.padding_eff_input = pad.input;
      row.padding_eff_target = pad.target;
      row.predicted_makespan = ms[l];
      row.bubble_ratio = bub[l];
      double peak = 0.0;
      for (int j = 0; j < C; ++j) peak = std::max(peak, ds[(static_cast<std::size_t>(l) * C + j) * 5 + 3]);
      row.peak_mem_max = peak;
      index << plans_index_row(row);
    }
  }
  sum.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return sum;
}

}  // namespace b200
}  // namespace pipeplan
