// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference planner.
//
// TEST INFRASTRUCTURE ONLY.  Linked with /root/reference/proj/src/{workload,
// cost_model,microbatch}.cpp into oracle/_ref/libpipeplan_ref.so by
// oracle/Makefile.  It lets pytest (ctypes) and bench.py's reference arm call
// the reference's own public API — order_samples, make_slice_cost,
// dp_partition, ProfileGrid, load_dataset — with no code of ours on the
// planning path.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <thread>
#include <atomic>
#include <vector>

#include "pipeplan/cost_model.h"
#include "pipeplan/errors.h"
#include "pipeplan/microbatch.h"
#include "pipeplan/workload.h"
#include "pipeplan/comm_plan.h"
#include "pipeplan/schedule.h"
#include "pipeplan/simulate.h"
#include "pipeplan_b200.h"

using namespace pipeplan;

namespace {

// ProfileGrid has no public cell setter; round-trip the descriptor through
// the reference's own text loader (cost_model.cpp:193-271) at %.17g.
ProfileGrid grid_from_desc(const pp_grid_desc* g) {
  static const char* kinds[2] = {"encoder", "decoder"};
  static const char* strats[3] = {"none", "selective", "full"};
  std::ostringstream os;
  os.precision(17);
  os << "pipeplan-grid 1\nmbs_axis";
  for (int i = 0; i < g->n_mbs; ++i) os << ' ' << g->mbs_axis[i];
  os << "\nseq_axis";
  for (int i = 0; i < g->n_seq; ++i) os << ' ' << g->seq_axis[i];
  os << '\n';
  std::size_t c = 0;
  for (int k = 0; k < 2; ++k)
    for (int r = 0; r < 3; ++r)
      for (int mi = 0; mi < g->n_mbs; ++mi)
        for (int si = 0; si < g->n_seq; ++si, c += 3)
          os << "row " << kinds[k] << ' ' << strats[r] << ' ' << g->mbs_axis[mi] << ' '
             << g->seq_axis[si] << ' ' << g->cells[c] << ' ' << g->cells[c + 1] << ' '
             << g->cells[c + 2] << '\n';
  os << "end\n";
  std::istringstream is(os.str());
  return ProfileGrid::load(is);
}

ModelConfig model_from_desc(const pp_model_desc* m) {
  ModelConfig cfg;
  cfg.is_encoder_decoder = m->is_encoder_decoder != 0;
  cfg.stages.resize(static_cast<std::size_t>(m->n_stages));
  for (int j = 0; j < m->n_stages; ++j)
    cfg.stages[static_cast<std::size_t>(j)] = {m->encoder_layers[j], m->decoder_layers[j]};
  return cfg;
}

DpOptions opts_from_desc(const pp_dp_options* o) {
  DpOptions d;
  d.stage_count = o->stage_count;
  d.replica_count = o->replica_count;
  d.per_mb_mem_cap = o->per_mb_mem_cap;
  d.t_max_interval = o->t_max_interval;
  return d;
}

struct PlanResult {
  int status = PP_OK;
  std::int64_t err_id = -1;
  std::vector<Sample> ordered;
  MicroBatchPartition part;
};

PlanResult plan_one(const Sample* s, std::int64_t n, int presorted, const ProfileGrid& grid,
                    const ModelConfig& cfg, Recompute r, const DpOptions& opt) {
  PlanResult res;
  try {
    MiniBatch mb;
    mb.samples.assign(s, s + n);
    res.ordered = presorted ? mb.samples : order_samples(mb, OrderMethod::Sort);
    SliceCostFn cost = make_slice_cost(grid, cfg, res.ordered, r);
    res.part = dp_partition(res.ordered, cost, opt);
  } catch (const InfeasibleError& e) {
    res.status = e.sample_id() >= 0 ? PP_ERR_INFEASIBLE_SAMPLE : PP_ERR_INFEASIBLE;
    res.err_id = e.sample_id();
  } catch (const std::out_of_range&) {
    res.status = PP_ERR_OUT_OF_RANGE;
  } catch (const std::invalid_argument&) {
    res.status = PP_ERR_INVALID;
  }
  return res;
}

void write_result(const PlanResult& res, std::int64_t n, pp_sample* ordered, int32_t* splits,
                  double* mb_times, int32_t* count, double* t_max_used, double* objective,
                  double* max_load, int32_t* replica, int64_t* err_id,
                  const std::vector<double>* times) {
  if (err_id) *err_id = res.err_id;
  if (res.status != PP_OK) return;
  if (ordered) std::memcpy(ordered, res.ordered.data(), sizeof(pp_sample) * n);
  int32_t end = 0;
  for (std::size_t k = 0; k < res.part.micro_batches.size(); ++k) {
    end += static_cast<int32_t>(res.part.micro_batches[k].sample_ids.size());
    splits[k] = end;
    if (replica) replica[k] = res.part.replica_assignment[k];
    if (mb_times && times) mb_times[k] = (*times)[k];
  }
  *count = static_cast<int32_t>(res.part.micro_batches.size());
  *t_max_used = res.part.t_max_used;
  *objective = res.part.objective_value;
  if (max_load) *max_load = res.part.max_replica_load;
}

}  // namespace

extern "C" {

int ref_order_samples(const pp_sample* in, int64_t n, pp_sample* out) {
  try {
    MiniBatch mb;
    mb.samples.assign(reinterpret_cast<const Sample*>(in), reinterpret_cast<const Sample*>(in) + n);
    auto o = order_samples(mb, OrderMethod::Sort);
    std::memcpy(out, o.data(), sizeof(pp_sample) * o.size());
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

int ref_per_layer(const pp_grid_desc* g, int32_t kind, int32_t r, double mbs, double seq,
                  double out[3]) {
  ProfileGrid grid = grid_from_desc(g);
  GridCell c = grid.per_layer(static_cast<StageKind>(kind), static_cast<Recompute>(r), mbs, seq);
  out[0] = c.t_f;
  out[1] = c.t_b;
  out[2] = c.act_mem;
  return PP_OK;
}

// ProfileGrid::synthetic (cost_model.cpp:91-124) exported as raw cells.
int ref_synthetic_grid(const double* params8, int32_t tp_degree, const int64_t* mbs_axis,
                       int32_t n_mbs, const int64_t* seq_axis, int32_t n_seq, int64_t* out_mbs,
                       int64_t* out_seq, int32_t* out_sizes, double* out_cells) {
  try {
    SyntheticGridParams p;
    p.alpha = params8[0];
    p.beta = params8[1];
    p.gamma = params8[2];
    p.full_mem_factor = params8[3];
    p.selective_mem_factor = params8[4];
    p.full_tb_penalty = params8[5];
    p.selective_tb_penalty = params8[6];
    p.tp_degree = tp_degree;
    std::vector<std::int64_t> ma(mbs_axis, mbs_axis + n_mbs), sa(seq_axis, seq_axis + n_seq);
    ProfileGrid g = ProfileGrid::synthetic(p, ma, sa);
    out_sizes[0] = static_cast<int32_t>(g.mbs_axis().size());
    out_sizes[1] = static_cast<int32_t>(g.seq_axis().size());
    std::memcpy(out_mbs, g.mbs_axis().data(), sizeof(int64_t) * g.mbs_axis().size());
    std::memcpy(out_seq, g.seq_axis().data(), sizeof(int64_t) * g.seq_axis().size());
    std::size_t c = 0;
    for (int k = 0; k < 2; ++k)
      for (int r = 0; r < 3; ++r)
        for (std::size_t mi = 0; mi < g.mbs_axis().size(); ++mi)
          for (std::size_t si = 0; si < g.seq_axis().size(); ++si) {
            // per_layer at a knot returns the knot value exactly (t = 0 blend)
            GridCell cell = g.per_layer(static_cast<StageKind>(k), static_cast<Recompute>(r),
                                        static_cast<double>(g.mbs_axis()[mi]),
                                        static_cast<double>(g.seq_axis()[si]));
            out_cells[c++] = cell.t_f;
            out_cells[c++] = cell.t_b;
            out_cells[c++] = cell.act_mem;
          }
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

// load_dataset with a synthetic descriptor (workload.cpp:50-63,109-127).
// dist = {family, log_mean, log_sigma, uniform_lo, uniform_hi, lognormal_weight}
// The reference's SyntheticGridParams{} defaults (cost_model.h), in
// ref_synthetic_grid's parameter order.
int ref_default_grid_params(double* params7, int32_t* tp_degree) {
  const SyntheticGridParams p{};
  params7[0] = p.alpha;
  params7[1] = p.beta;
  params7[2] = p.gamma;
  params7[3] = p.full_mem_factor;
  params7[4] = p.selective_mem_factor;
  params7[5] = p.full_tb_penalty;
  params7[6] = p.selective_tb_penalty;
  *tp_degree = p.tp_degree;
  return PP_OK;
}

// ModelConfig::uniform (cost_model.cpp:273-292): per-stage layer counts.
int ref_model_uniform(int32_t n_stages, int32_t layers_per_stage, int64_t hidden_dim, int32_t encdec,
                      int32_t* enc_out, int32_t* dec_out) {
  try {
    ModelConfig c = ModelConfig::uniform(n_stages, layers_per_stage, hidden_dim, encdec != 0);
    for (std::size_t s = 0; s < c.stages.size(); ++s) {
      enc_out[s] = c.stages[s].encoder_layers;
      dec_out[s] = c.stages[s].decoder_layers;
    }
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

int ref_load_dataset(int64_t n, const double* in_dist, const double* tgt_dist, int64_t max_seq_len,
                     uint64_t seed, pp_sample* out) {
  try {
    auto mk = [](const double* d) {
      LengthDistribution l;
      l.family = static_cast<LengthFamily>(static_cast<int>(d[0]));
      l.log_mean = d[1];
      l.log_sigma = d[2];
      l.uniform_lo = static_cast<std::int64_t>(d[3]);
      l.uniform_hi = static_cast<std::int64_t>(d[4]);
      l.lognormal_weight = d[5];
      return l;
    };
    DatasetSpec spec;
    SyntheticSpec syn;
    syn.n = n;
    syn.input = mk(in_dist);
    if (tgt_dist) syn.target = mk(tgt_dist);
    spec.synthetic = syn;
    spec.max_seq_len = max_seq_len;
    spec.seed = seed;
    auto s = load_dataset(spec);
    std::memcpy(out, s.data(), sizeof(pp_sample) * s.size());
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

// One mini-batch through the reference's production path.
int ref_plan_grid(const pp_sample* samples, int64_t n, int32_t presorted, const pp_grid_desc* g,
                  const pp_model_desc* m, const pp_dp_options* o, pp_sample* ordered,
                  int32_t* splits, double* mb_times, int32_t* count, double* t_max_used,
                  double* objective, double* max_load, int32_t* replica, int64_t* err_id) {
  ProfileGrid grid = grid_from_desc(g);
  ModelConfig cfg = model_from_desc(m);
  const Recompute r = static_cast<Recompute>(m->recompute);
  PlanResult res = plan_one(reinterpret_cast<const Sample*>(samples), n, presorted, grid, cfg, r,
                            opts_from_desc(o));
  std::vector<double> times;
  if (res.status == PP_OK) {
    SliceCostFn cost = make_slice_cost(grid, cfg, res.ordered, r);
    std::size_t b = 0;
    for (const auto& mb : res.part.micro_batches) {
      times.push_back(cost(b, b + mb.sample_ids.size()).time);
      b += mb.sample_ids.size();
    }
  }
  write_result(res, n, ordered, splits, mb_times, count, t_max_used, objective, max_load, replica,
               err_id, &times);
  return res.status;
}

// dp_partition over given triangular tables (a generic SliceCostFn).
int ref_plan_tables(const double* T, const double* M, int64_t n, const pp_dp_options* o,
                    int32_t* splits, double* mb_times, int32_t* count, double* t_max_used,
                    double* objective, double* max_load, int32_t* replica, int64_t* err_index) {
  std::vector<std::int64_t> row_off(static_cast<std::size_t>(n));
  std::int64_t tot = 0;
  for (std::int64_t i = 0; i < n; ++i) {
    row_off[static_cast<std::size_t>(i)] = tot;
    tot += n - i;
  }
  std::vector<Sample> s(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) s[static_cast<std::size_t>(i)] = {i, 1, 0};
  SliceCostFn cost = [&](std::size_t b, std::size_t e) {
    const std::size_t idx = static_cast<std::size_t>(row_off[b]) + (e - b - 1);
    return SliceCost{T[idx], M[idx]};
  };
  PlanResult res;
  try {
    res.part = dp_partition(s, cost, opts_from_desc(o));
  } catch (const InfeasibleError& e) {
    res.status = e.sample_id() >= 0 ? PP_ERR_INFEASIBLE_SAMPLE : PP_ERR_INFEASIBLE;
    res.err_id = e.sample_id();
  } catch (const std::invalid_argument&) {
    res.status = PP_ERR_INVALID;
  }
  std::vector<double> times;
  if (res.status == PP_OK) {
    std::size_t b = 0;
    for (const auto& mb : res.part.micro_batches) {
      times.push_back(cost(b, b + mb.sample_ids.size()).time);
      b += mb.sample_ids.size();
    }
  }
  write_result(res, n, nullptr, splits, mb_times, count, t_max_used, objective, max_load, replica,
               err_index, &times);
  return res.status;
}

// The reference's batch-planning parallelism model (run_plan's worker pool,
// driver.cpp:222-242): `threads` std::threads pull mini-batch indices from an
// atomic counter; each runs order_samples(Sort) + make_slice_cost +
// dp_partition.  Returns wall seconds; per-segment t_max/objective/count out.
// run_plan's worker pool (driver.cpp:222-242) over n_seg mini-batches; the
// returned wall time covers order_samples + make_slice_cost + dp_partition
// only.  Optional (nullable) outputs, written AFTER the timed region, indexed
// by sample like the device's pp_plan_out: splits and slice times at the
// segment's offset, the ordered sample ids.
double ref_plan_batch_out(const pp_sample* samples, const int64_t* seg_off, int32_t n_seg,
                          const pp_grid_desc* g, const pp_model_desc* m, const pp_dp_options* o,
                          int32_t threads, double* t_max_used, double* objective, int32_t* count,
                          int32_t* status, int32_t* splits, double* mb_times, int64_t* ordered_ids) {
  ProfileGrid grid = grid_from_desc(g);
  ModelConfig cfg = model_from_desc(m);
  const Recompute r = static_cast<Recompute>(m->recompute);
  const DpOptions opt = opts_from_desc(o);
  const bool keep = splits || mb_times || ordered_ids;
  std::vector<PlanResult> kept(keep ? static_cast<std::size_t>(n_seg) : 0);
  std::atomic<int> next{0};
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&]() {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= n_seg) return;
      PlanResult res =
          plan_one(reinterpret_cast<const Sample*>(samples) + seg_off[s], seg_off[s + 1] - seg_off[s],
                   0, grid, cfg, r, opt);
      status[s] = res.status;
      if (res.status == PP_OK) {
        t_max_used[s] = res.part.t_max_used;
        objective[s] = res.part.objective_value;
        count[s] = static_cast<int32_t>(res.part.micro_batches.size());
      }
      if (keep) kept[static_cast<std::size_t>(s)] = std::move(res);
    }
  };
  const int nt = threads < 1 ? 1 : threads;
  if (nt == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int s = 0; keep && s < n_seg; ++s) {
    const PlanResult& res = kept[static_cast<std::size_t>(s)];
    if (res.status != PP_OK) continue;
    const int64_t b0 = seg_off[s];
    SliceCostFn cost = make_slice_cost(grid, cfg, res.ordered, r);
    std::size_t b = 0, k = 0;
    for (const auto& mb : res.part.micro_batches) {
      const std::size_t e = b + mb.sample_ids.size();
      if (splits) splits[b0 + static_cast<int64_t>(k)] = static_cast<int32_t>(e);
      if (mb_times) mb_times[b0 + static_cast<int64_t>(k)] = cost(b, e).time;
      b = e;
      ++k;
    }
    if (ordered_ids)
      for (std::size_t q = 0; q < res.ordered.size(); ++q) ordered_ids[b0 + static_cast<int64_t>(q)] = res.ordered[q].id;
  }
  return secs;
}

double ref_plan_batch(const pp_sample* samples, const int64_t* seg_off, int32_t n_seg,
                      const pp_grid_desc* g, const pp_model_desc* m, const pp_dp_options* o,
                      int32_t threads, double* t_max_used, double* objective, int32_t* count,
                      int32_t* status) {
  return ref_plan_batch_out(samples, seg_off, n_seg, g, m, o, threads, t_max_used, objective, count, status,
                            nullptr, nullptr, nullptr);
}


// OpCostTable::from_shapes (src/cost_model.cpp:360-382): the reference's own
// op-cost table, [shape * stages + stage].
int ref_op_costs(const pp_padded_shape* shapes, int64_t n, const pp_grid_desc* g, const pp_model_desc* m,
                 double* t_f, double* t_b, double* act) {
  try {
    ProfileGrid grid = grid_from_desc(g);
    ModelConfig cfg = model_from_desc(m);
    std::vector<PaddedShape> sh(n);
    for (int64_t k = 0; k < n; ++k) {
      sh[k].mbs = shapes[k].mbs;
      sh[k].input_len = shapes[k].input_len;
      sh[k].target_len = shapes[k].target_len;
    }
    OpCostTable t = OpCostTable::from_shapes(grid, cfg, sh, static_cast<Recompute>(m->recompute));
    std::memcpy(t_f, t.t_f.data(), t.t_f.size() * sizeof(double));
    std::memcpy(t_b, t.t_b.data(), t.t_b.size() * sizeof(double));
    std::memcpy(act, t.act_mem.data(), t.act_mem.size() * sizeof(double));
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  } catch (const std::out_of_range&) {
    return PP_ERR_OUT_OF_RANGE;
  }
}


// select_recomputation (src/schedule.cpp:319-364) per partition, on
// micro-batches carrying the given padded shapes; strategy -1 and the
// InfeasibleError's stage when none fits.  Tables as ref_op_costs.
int ref_select_recomputation(const pp_padded_shape* shapes, const int64_t* mb_off, int32_t n_seg,
                             const pp_grid_desc* g, const pp_model_desc* m, int32_t mask, const double* limits,
                             double* t_f, double* t_b, double* act, int32_t* strategy, int32_t* violating) {
  try {
    ProfileGrid grid = grid_from_desc(g);
    ModelConfig cfg = model_from_desc(m);
    const int C = cfg.stage_count();
    std::vector<Recompute> allowed;
    for (int r = 0; r < 3; ++r)
      if (mask & (1 << r)) allowed.push_back(static_cast<Recompute>(r));
    std::vector<double> lim(limits, limits + C);
    for (int s = 0; s < n_seg; ++s) {
      MicroBatchPartition part;
      for (int64_t k = mb_off[s]; k < mb_off[s + 1]; ++k) {
        MicroBatch mb;
        mb.padded_mbs = shapes[k].mbs;
        mb.padded_input_len = shapes[k].input_len;
        mb.padded_target_len = shapes[k].target_len;
        part.micro_batches.push_back(mb);
      }
      try {
        RecomputeSelection sel = select_recomputation(grid, cfg, part, lim, allowed);
        strategy[s] = static_cast<int32_t>(sel.strategy);
        violating[s] = -1;
        const std::size_t o = static_cast<std::size_t>(mb_off[s]) * C;
        std::memcpy(t_f + o, sel.costs.t_f.data(), sel.costs.t_f.size() * sizeof(double));
        std::memcpy(t_b + o, sel.costs.t_b.data(), sel.costs.t_b.size() * sizeof(double));
        std::memcpy(act + o, sel.costs.act_mem.data(), sel.costs.act_mem.size() * sizeof(double));
      } catch (const InfeasibleError& e) {
        strategy[s] = -1;
        violating[s] = e.stage();
      }
    }
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  } catch (const std::logic_error&) {
    return PP_ERR_NOT_CONVERGED;
  }
}


// order_microbatches with plan_iteration's evaluator (planner.cpp:94-108)
// over n_seg op-cost tables, then the chosen order's schedule_adaptive ->
// plan_communication -> simulate report, exactly as plan_iteration builds
// rep.report.  `threads` std::threads pull tables from an atomic counter
// (run_plan's pool model).  Returns wall seconds.
double ref_order_search(const double* t_f, const double* t_b, const double* act, const int64_t* mb_off,
                        int32_t n_seg, int32_t C, const double* limits, int32_t k, double comm_latency,
                        int32_t threads, int32_t* order, double* makespan, double* bubble,
                        int32_t* deadlock, double* dev_stats, int32_t* status) {
  std::vector<double> lim(limits, limits + C);
  std::atomic<int> next{0};
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&]() {
    for (;;) {
      const int s = next.fetch_add(1);
      if (s >= n_seg) return;
      const int64_t b = mb_off[s], M = mb_off[s + 1] - b;
      try {
        OpCostTable costs;
        costs.micro_batches = static_cast<int>(M);
        costs.stages = C;
        costs.t_f.assign(t_f + b * C, t_f + (b + M) * C);
        costs.t_b.assign(t_b + b * C, t_b + (b + M) * C);
        costs.act_mem.assign(act + b * C, act + (b + M) * C);
        PlanMeta meta;
        meta.shape_table.assign(static_cast<std::size_t>(M), MbShapeEntry{1, 1, 0});
        SimConfig zero_noise;
        zero_noise.comm_latency = comm_latency;
        std::vector<double> predicted(static_cast<std::size_t>(M));
        for (int i = 0; i < M; ++i) predicted[static_cast<std::size_t>(i)] = costs.scalar_time(i);
        auto evaluator = [&](const PipelineSchedule& sched) {
          ExecutionPlan candidate = plan_communication(sched, costs, meta);
          return simulate(candidate, costs, zero_noise).makespan;
        };
        std::vector<int> best = order_microbatches(predicted, costs, lim, k, evaluator);
        status[s] = PP_OK;
        if (best.empty()) {
          for (int64_t i = 0; i < M; ++i) order[b + i] = -1;
          makespan[s] = std::nan("");
          continue;
        }
        for (int64_t i = 0; i < M; ++i) order[b + i] = best[static_cast<std::size_t>(i)];
        PipelineSchedule sched = schedule_adaptive(costs, lim, best);
        ExecutionPlan plan = plan_communication(sched, costs, meta);
        SimReport rep = simulate(plan, costs, zero_noise);
        makespan[s] = rep.makespan;
        bubble[s] = rep.bubble_ratio;
        deadlock[s] = rep.deadlock ? 1 : 0;
        for (int j = 0; j < C; ++j) {
          const DeviceStats& d = rep.devices[static_cast<std::size_t>(j)];
          double* o = dev_stats + (static_cast<int64_t>(s) * C + j) * 5;
          o[0] = d.busy; o[1] = d.idle; o[2] = d.blocked; o[3] = d.peak_mem; o[4] = d.final_mem;
        }
      } catch (const std::invalid_argument&) {
        status[s] = PP_ERR_INVALID;
      } catch (const std::logic_error& e) {
        status[s] = std::strstr(e.what(), "converge") ? PP_ERR_NOT_CONVERGED : PP_ERR_NOT_EXECUTABLE;
      }
    }
  };
  const int nt = threads < 1 ? 1 : threads;
  if (nt == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// The reference's plan of each table for a GIVEN injection order (or the
// 1F1B schedule): plan_communication(schedule_adaptive(costs, limits, order))
// instruction lists packed like pp_emit_plans ((mb << 4) | kind, peers in
// `peer`), the zero-noise SimReport, and (when meta != null) save_plan's text
// of table 0 with that plan metadata into text (cap bytes).
int ref_emit_plans(const double* t_f, const double* t_b, const double* act, const int64_t* mb_off, int32_t n_seg,
                   int32_t C, const double* limits, double comm_latency, int32_t f1b, const int32_t* order,
                   int32_t* ins, int32_t* peer, int32_t* nins, double* makespan, double* bubble, int32_t* deadlock,
                   double* dev_stats, int32_t* status, const pp_padded_shape* shapes, const pp_model_desc* m,
                   int64_t iteration, int32_t replica, int64_t hidden, char* text, int64_t cap) {
  std::vector<double> lim(limits ? limits : act, (limits ? limits : act) + C);
  for (int s = 0; s < n_seg; ++s) {
    const int64_t b = mb_off[s], M = mb_off[s + 1] - b;
    for (int j = 0; j < C; ++j) nins[s * C + j] = 0;
    try {
      OpCostTable costs;
      costs.micro_batches = static_cast<int>(M);
      costs.stages = C;
      costs.t_f.assign(t_f + b * C, t_f + (b + M) * C);
      costs.t_b.assign(t_b + b * C, t_b + (b + M) * C);
      costs.act_mem.assign(act + b * C, act + (b + M) * C);
      PlanMeta meta;
      if (shapes && m) {
        ModelConfig cfg = model_from_desc(m);
        meta.iteration = iteration;
        meta.replica = replica;
        meta.hidden_dim = hidden;
        meta.encoder_decoder = cfg.is_encoder_decoder;
        meta.recompute = static_cast<Recompute>(m->recompute);
        meta.stage_layers = cfg.stages;
        for (int64_t i = 0; i < M; ++i)
          meta.shape_table.push_back({shapes[b + i].mbs, shapes[b + i].input_len, shapes[b + i].target_len});
      } else {
        meta.shape_table.assign(static_cast<std::size_t>(M), MbShapeEntry{1, 1, 0});
      }
      std::vector<int> ord(order ? order + b : nullptr, order ? order + b + M : nullptr);
      PipelineSchedule sched = f1b ? schedule_1f1b(static_cast<int>(M), C) : schedule_adaptive(costs, lim, ord);
      ExecutionPlan plan = plan_communication(sched, costs, meta);
      SimConfig zero_noise;
      zero_noise.comm_latency = comm_latency;
      SimReport rep = simulate(plan, costs, zero_noise);
      for (int j = 0; j < C; ++j) {
        const auto& L = plan.devices[static_cast<std::size_t>(j)];
        nins[s * C + j] = static_cast<int32_t>(L.size());
        int32_t* o = ins + 10 * C * b + 10 * M * j;
        int32_t* pe = peer + 10 * C * b + 10 * M * j;
        for (std::size_t q = 0; q < L.size(); ++q) {
          o[q] = (L[q].microbatch << 4) | static_cast<int>(L[q].kind);
          pe[q] = L[q].peer;
        }
        const DeviceStats& d = rep.devices[static_cast<std::size_t>(j)];
        double* ds = dev_stats + (static_cast<int64_t>(s) * C + j) * 5;
        ds[0] = d.busy; ds[1] = d.idle; ds[2] = d.blocked; ds[3] = d.peak_mem; ds[4] = d.final_mem;
      }
      makespan[s] = rep.makespan;
      bubble[s] = rep.bubble_ratio;
      deadlock[s] = rep.deadlock ? 1 : 0;
      status[s] = PP_OK;
      if (s == 0 && text && cap > 0) {
        std::ostringstream os;
        save_plan(plan, os);
        const std::string t = os.str();
        const std::size_t nbytes = std::min<std::size_t>(t.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(text, t.data(), nbytes);
        text[nbytes] = 0;
      }
    } catch (const std::invalid_argument&) {
      status[s] = PP_ERR_INVALID;
    } catch (const std::logic_error& e) {
      status[s] = std::strstr(e.what(), "converge") ? PP_ERR_NOT_CONVERGED : PP_ERR_NOT_EXECUTABLE;
    }
  }
  return PP_OK;
}


// load_dataset over a record file (workload.cpp:65-127): samples out (up to
// cap), *n set; PP_ERR_PARSE with line / byte / message kind, PP_ERR_INVALID.
int ref_load_record_file(const char* path, int64_t max_seq_len, pp_sample* out, int64_t cap, int64_t* n,
                         int64_t* err_line, int64_t* err_byte, int32_t* err_kind) {
  *n = 0;
  *err_line = -1;
  *err_byte = 0;
  *err_kind = -1;
  try {
    DatasetSpec spec;
    spec.path = path;
    spec.max_seq_len = max_seq_len;
    std::vector<Sample> v = load_dataset(spec);
    *n = static_cast<int64_t>(v.size());
    for (int64_t k = 0; k < *n && k < cap; ++k) out[k] = pp_sample{v[k].id, v[k].input_len, v[k].target_len};
    return PP_OK;
  } catch (const ParseError& e) {
    *err_line = e.line();
    *err_byte = e.byte_offset();
    const std::string w = e.what();
    *err_kind = w.find("missing tab") != std::string::npos    ? PP_PARSE_MISSING_TAB
                : w.find("pair of integers") != std::string::npos ? PP_PARSE_NOT_INTEGERS
                : w.find("input_len < 1") != std::string::npos    ? PP_PARSE_INPUT_LT_1
                                                                  : PP_PARSE_TARGET_LT_0;
    return PP_ERR_PARSE;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

// run_plan's draw loop (driver.cpp:209-215): seg offsets of every mini-batch
// draw_minibatch yields from cursor 0.
int ref_draw_all(const pp_sample* s, int64_t n, int64_t budget, int64_t* offsets, int64_t* n_seg) {
  try {
    std::vector<Sample> v(n);
    for (int64_t k = 0; k < n; ++k) v[k] = Sample{s[k].id, s[k].input_len, s[k].target_len};
    std::size_t cursor = 0;
    int64_t m = 0;
    offsets[0] = 0;
    while (auto d = draw_minibatch(v, budget, cursor)) {
      cursor = d->next_cursor;
      offsets[++m] = static_cast<int64_t>(cursor);
    }
    *n_seg = m;
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}


// padding_vs_packing_report (simulate.cpp:288-406) -> 3 * n_lens rows;
// returns wall seconds (negative: status).
double ref_padding_report(const pp_sample* s, int64_t n, const int64_t* lens, int32_t n_lens, const pp_grid_desc* g,
                          const pp_model_desc* m, int64_t token_budget, double interval, int32_t max_iterations,
                          int32_t recompute, pp_padding_row* rows) {
  try {
    ProfileGrid grid = grid_from_desc(g);
    ModelConfig cfg = model_from_desc(m);
    std::vector<Sample> v(n);
    for (int64_t k = 0; k < n; ++k) v[k] = Sample{s[k].id, s[k].input_len, s[k].target_len};
    PaddingReportOptions opt;
    opt.token_budget = token_budget;
    opt.t_max_interval = interval;
    opt.max_iterations = max_iterations;
    opt.recompute = static_cast<Recompute>(recompute);
    const auto t0 = std::chrono::steady_clock::now();
    auto out = padding_vs_packing_report(v, std::span<const std::int64_t>(lens, n_lens), grid, cfg, opt);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t k = 0; k < out.size(); ++k) {
      const PaddingRow& r = out[k];
      rows[k] = pp_padding_row{static_cast<int32_t>(r.method), 0, r.max_seq_len, r.padding_eff_input,
                               r.padding_eff_target, r.tokens, r.sim_time, r.throughput_proxy};
    }
    return secs;
  } catch (const InfeasibleError&) {
    return -PP_ERR_INFEASIBLE;
  } catch (const std::invalid_argument&) {
    return -PP_ERR_INVALID;
  }
}

}  // extern "C"
