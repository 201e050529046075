// microbatch.cpp — the drop-in planner API over the B200 C-ABI.
//
// Reference: proj/src/microbatch.cpp.  order_samples(Sort) and dp_partition
// run on the device (pp_order_samples / pp_plan_grid / pp_plan_tables); the
// host keeps argument checking, exception mapping and the O(n) assembly of
// the MicroBatchPartition record.  Tsp ordering, balance_replicas and
// padding_efficiency are host code (out of the GPU hot path).
// There is no CPU planning fallback: without a CUDA device the device entry
// points throw std::runtime_error.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>

#include "pipeplan/errors.h"
#include "pipeplan/microbatch.h"
#include "pipeplan_b200.h"

namespace pipeplan {
namespace detail {

// One device context per host thread: the reference planner is called
// concurrently from run_plan's workers (driver.cpp:222-242).  Shared with
// order_search.cpp.
pp_ctx* device_ctx() {
  struct Holder {
    pp_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) pp_ctx_destroy(ctx);
    }
  };
  thread_local Holder h;
  if (!h.ctx) {
    const char* env = std::getenv("PIPEPLAN_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    const int rc = pp_ctx_create(dev, &h.ctx);
    if (rc != PP_OK)
      throw std::runtime_error(rc == PP_ERR_NO_DEVICE
                                   ? "pipeplan_b200: no CUDA device (the planner has no CPU fallback)"
                                   : "pipeplan_b200: cannot create a device context");
  }
  return h.ctx;
}

}  // namespace detail
namespace {
using detail::device_ctx;

[[noreturn]] void raise(pp_ctx* ctx, int rc, std::int64_t sample_id) {
  switch (rc) {
    case PP_ERR_INVALID:
      throw std::invalid_argument(pp_ctx_last_error(ctx));
    case PP_ERR_OUT_OF_RANGE:
      throw std::out_of_range(pp_ctx_last_error(ctx));
    case PP_ERR_INFEASIBLE_SAMPLE:  // microbatch.cpp:248-250
      throw InfeasibleError("sample " + std::to_string(sample_id) +
                                " does not fit the per-micro-batch memory cap alone",
                            sample_id, -1);
    case PP_ERR_INFEASIBLE:  // microbatch.cpp:320
      throw InfeasibleError("no feasible partition under the memory cap", -1, -1);
    default:
      throw std::runtime_error(std::string("pipeplan_b200 device error: ") + pp_ctx_last_error(ctx));
  }
}

auto length_key(const Sample& s) { return std::tie(s.input_len, s.target_len, s.id); }

std::int64_t l1(const Sample& a, const Sample& b) {
  return std::llabs(a.input_len - b.input_len) + std::llabs(a.target_len - b.target_len);
}

// Nearest-neighbour tour from the smallest point, then first-improvement
// 2-opt on the open path (reference tsp_order, microbatch.cpp:33-93).
std::vector<Sample> tour_order(std::vector<Sample> pts) {
  const std::size_t n = pts.size();
  if (n <= 2) {
    std::sort(pts.begin(), pts.end(),
              [](const Sample& a, const Sample& b) { return length_key(a) < length_key(b); });
    return pts;
  }
  std::vector<char> used(n, 0);
  std::size_t cur = 0;
  for (std::size_t k = 1; k < n; ++k)
    if (length_key(pts[k]) < length_key(pts[cur])) cur = k;
  std::vector<Sample> path{pts[cur]};
  path.reserve(n);
  used[cur] = 1;
  while (path.size() < n) {
    std::size_t pick = n;
    for (std::size_t k = 0; k < n; ++k) {
      if (used[k]) continue;
      if (pick == n) {
        pick = k;
        continue;
      }
      const std::int64_t dk = l1(path.back(), pts[k]), dp = l1(path.back(), pts[pick]);
      if (std::tie(dk, pts[k].input_len, pts[k].target_len, pts[k].id) <
          std::tie(dp, pts[pick].input_len, pts[pick].target_len, pts[pick].id))
        pick = k;
    }
    used[pick] = 1;
    path.push_back(pts[pick]);
  }
  for (bool again = true; again;) {
    again = false;
    for (std::size_t i = 1; i + 1 < n && !again; ++i)
      for (std::size_t j = i + 1; j < n && !again; ++j) {
        std::int64_t before = l1(path[i - 1], path[i]);
        std::int64_t after = l1(path[i - 1], path[j]);
        if (j + 1 < n) {
          before += l1(path[j], path[j + 1]);
          after += l1(path[i], path[j + 1]);
        }
        if (after < before) {
          std::reverse(path.begin() + static_cast<std::ptrdiff_t>(i),
                       path.begin() + static_cast<std::ptrdiff_t>(j) + 1);
          again = true;
        }
      }
  }
  return path;
}

pp_model_desc model_desc(const ModelConfig& cfg, Recompute r, std::vector<int32_t>& enc,
                         std::vector<int32_t>& dec) {
  enc.clear();
  dec.clear();
  for (const StageLayout& s : cfg.stages) {
    enc.push_back(s.encoder_layers);
    dec.push_back(s.decoder_layers);
  }
  pp_model_desc m;
  m.n_stages = cfg.stage_count();
  m.encoder_layers = enc.data();
  m.decoder_layers = dec.data();
  m.is_encoder_decoder = cfg.is_encoder_decoder ? 1 : 0;
  m.recompute = static_cast<int32_t>(r);
  return m;
}

pp_dp_options dp_desc(const DpOptions& o) {
  return pp_dp_options{o.stage_count, o.replica_count, o.per_mb_mem_cap, o.t_max_interval};
}

// microbatch.cpp:322-348 given the device's splits and slice times.
MicroBatchPartition assemble(std::span<const Sample> ordered, const int32_t* splits,
                             const double* times, int m, double objective, double t_max_used,
                             int replicas) {
  MicroBatchPartition p;
  p.micro_batches.reserve(static_cast<std::size_t>(m));
  std::size_t begin = 0;
  for (int k = 0; k < m; ++k) {
    const std::size_t end = static_cast<std::size_t>(splits[k]);
    p.micro_batches.push_back(make_micro_batch(ordered, begin, end));
    begin = end;
  }
  p.objective_value = objective;
  p.t_max_used = t_max_used;
  std::span<const double> ts(times, static_cast<std::size_t>(m));
  if (m >= replicas) {
    p.replica_assignment = balance_replicas(ts, replicas);
  } else {
    p.replica_assignment.resize(static_cast<std::size_t>(m));
    for (int k = 0; k < m; ++k) p.replica_assignment[static_cast<std::size_t>(k)] = k;
  }
  std::vector<double> load(static_cast<std::size_t>(replicas), 0.0);
  for (int k = 0; k < m; ++k)
    load[static_cast<std::size_t>(p.replica_assignment[static_cast<std::size_t>(k)])] +=
        ts[static_cast<std::size_t>(k)];
  p.max_replica_load = *std::max_element(load.begin(), load.end());
  return p;
}

}  // namespace

std::vector<Sample> order_samples(const MiniBatch& minibatch, OrderMethod method) {
  if (minibatch.samples.empty()) throw std::invalid_argument("mini-batch is empty");
  if (method == OrderMethod::Tsp) return tour_order(minibatch.samples);
  pp_ctx* ctx = device_ctx();
  std::vector<Sample> out(minibatch.samples.size());
  const int64_t off[2] = {0, static_cast<int64_t>(out.size())};
  const int rc = pp_order_samples(ctx, reinterpret_cast<const pp_sample*>(minibatch.samples.data()),
                                  off, 1, reinterpret_cast<pp_sample*>(out.data()));
  if (rc != PP_OK) raise(ctx, rc, -1);
  return out;
}

double eval_objective(std::span<const double> times, int stage_count, int replica_count) {
  if (times.empty()) throw std::invalid_argument("objective needs at least one micro-batch");
  if (stage_count < 1 || replica_count < 1)
    throw std::invalid_argument("stage and replica counts must be >= 1");
  double out = 0.0;
  pp_eval_objective(times.data(), static_cast<int64_t>(times.size()), stage_count, replica_count,
                    &out);
  return out;
}

MicroBatch make_micro_batch(std::span<const Sample> ordered, std::size_t begin, std::size_t end) {
  MicroBatch mb;
  mb.padded_mbs = static_cast<std::int64_t>(end - begin);
  mb.sample_ids.reserve(end - begin);
  for (std::size_t k = begin; k < end; ++k) {
    const Sample& s = ordered[k];
    mb.sample_ids.push_back(s.id);
    mb.padded_input_len = std::max(mb.padded_input_len, s.input_len);
    mb.padded_target_len = std::max(mb.padded_target_len, s.target_len);
    mb.input_tokens += s.input_len;
    mb.target_tokens += s.target_len;
  }
  return mb;
}

SliceCost GridSliceCost::operator()(std::size_t begin, std::size_t end) const {
  // Host evaluation for direct callers (the device path never calls this).
  std::int64_t in = 0, tgt = 0;
  for (std::size_t k = begin; k < end; ++k) {
    in = std::max(in, samples[k].input_len);
    tgt = std::max(tgt, samples[k].target_len);
  }
  SliceCost c;
  for (int s = 0; s < config.stage_count(); ++s) {
    const CostEstimate e =
        estimate(*grid, config, s, static_cast<std::int64_t>(end - begin), in, tgt, r);
    c.time = std::max(c.time, e.t_f + e.t_b);
    c.act_mem = std::max(c.act_mem, e.act_mem);
  }
  return c;
}

SliceCostFn make_slice_cost(const ProfileGrid& grid, const ModelConfig& config,
                            std::span<const Sample> ordered, Recompute r) {
  return GridSliceCost{&grid, config, std::vector<Sample>(ordered.begin(), ordered.end()), r};
}

MicroBatchPartition dp_partition(std::span<const Sample> ordered, const SliceCostFn& cost,
                                 const DpOptions& options) {
  const std::size_t n = ordered.size();
  if (n == 0) throw std::invalid_argument("cannot partition an empty sample list");
  if (options.stage_count < 1 || options.replica_count < 1)
    throw std::invalid_argument("stage and replica counts must be >= 1");
  if (options.t_max_interval < 0) throw std::invalid_argument("t_max_interval must be >= 0");
  pp_ctx* ctx = device_ctx();
  const pp_dp_options o = dp_desc(options);
  std::vector<int32_t> splits(n);
  std::vector<double> times(n);
  int32_t m = 0;
  double tmax = 0.0, obj = 0.0;

  const GridSliceCost* g = cost.target<GridSliceCost>();
  if (g && g->samples.size() == n && g->grid) {
    // Fused path: every slice is priced on the device from the grid.
    std::vector<int32_t> enc, dec;
    const pp_model_desc md = model_desc(g->config, g->r, enc, dec);
    const pp_grid_desc gd = g->grid->device_desc();
    const int64_t off[2] = {0, static_cast<int64_t>(n)};
    int32_t status = 0;
    int64_t err_id = -1;
    pp_plan_out out{nullptr, splits.data(), times.data(), &m, &tmax, &obj, &status, &err_id};
    const int rc = pp_plan_grid(ctx, reinterpret_cast<const pp_sample*>(g->samples.data()), off, 1,
                                /*presorted=*/1, &gd, &md, &o, &out);
    if (rc != PP_OK) raise(ctx, rc, -1);
    if (status == PP_ERR_INFEASIBLE_SAMPLE) {
      // The device names the sample of the coster's own copy; the reference
      // reports ordered[k].id for the same position k (microbatch.cpp:248).
      for (std::size_t k = 0; k < n; ++k)
        if (g->samples[k].id == err_id) {
          err_id = ordered[k].id;
          break;
        }
    }
    if (status != PP_OK) raise(ctx, status, err_id);
  } else {
    // Generic SliceCostFn: build the triangular tables exactly as the
    // reference does (microbatch.cpp:228-243), then plan on the device.
    const std::size_t tri = n * (n + 1) / 2;
    std::vector<double> T(tri), M(tri);
    std::size_t idx = 0;
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i + 1; j <= n; ++j, ++idx) {
        const SliceCost c = cost(i, j);
        T[idx] = c.time;
        M[idx] = c.act_mem;
      }
    int64_t err_index = -1;
    const int rc = pp_plan_tables(ctx, T.data(), M.data(), static_cast<int64_t>(n), &o,
                                  splits.data(), times.data(), &m, &tmax, &obj, &err_index);
    if (rc != PP_OK)
      raise(ctx, rc, err_index >= 0 ? ordered[static_cast<std::size_t>(err_index)].id : -1);
  }
  return assemble(ordered, splits.data(), times.data(), m, obj, tmax, options.replica_count);
}

BatchPlan plan_minibatches(const std::vector<MiniBatch>& minibatches, const ProfileGrid& grid,
                           const ModelConfig& config, Recompute r, const DpOptions& options) {
  BatchPlan bp;
  const std::size_t S = minibatches.size();
  bp.partitions.resize(S);
  bp.errors.assign(S, std::string());
  if (S == 0) return bp;
  if (options.stage_count < 1 || options.replica_count < 1)
    throw std::invalid_argument("stage and replica counts must be >= 1");
  if (options.t_max_interval < 0) throw std::invalid_argument("t_max_interval must be >= 0");
  pp_ctx* ctx = device_ctx();
  std::vector<int64_t> off(S + 1, 0);
  for (std::size_t s = 0; s < S; ++s)
    off[s + 1] = off[s] + static_cast<int64_t>(minibatches[s].samples.size());
  std::vector<Sample> all(static_cast<std::size_t>(off[S])), ordered(all.size());
  for (std::size_t s = 0; s < S; ++s)
    std::copy(minibatches[s].samples.begin(), minibatches[s].samples.end(),
              all.begin() + static_cast<std::ptrdiff_t>(off[s]));
  std::vector<int32_t> splits(all.size()), count(S), status(S);
  std::vector<double> times(all.size()), tmax(S), obj(S);
  std::vector<int64_t> err(S);
  std::vector<int32_t> enc, dec;
  const pp_model_desc md = model_desc(config, r, enc, dec);
  const pp_grid_desc gd = grid.device_desc();
  const pp_dp_options o = dp_desc(options);
  pp_plan_out out{reinterpret_cast<pp_sample*>(ordered.data()), splits.data(), times.data(),
                  count.data(), tmax.data(), obj.data(), status.data(), err.data()};
  const int rc = pp_plan_grid(ctx, reinterpret_cast<const pp_sample*>(all.data()), off.data(),
                              static_cast<int32_t>(S), 0, &gd, &md, &o, &out);
  if (rc != PP_OK) raise(ctx, rc, -1);
  for (std::size_t s = 0; s < S; ++s) {
    std::span<const Sample> seg(ordered.data() + off[s], static_cast<std::size_t>(off[s + 1] - off[s]));
    try {
      if (status[s] != PP_OK) raise(ctx, status[s], err[s]);
      bp.partitions[s] = assemble(seg, splits.data() + off[s], times.data() + off[s], count[s],
                                  obj[s], tmax[s], options.replica_count);
    } catch (const std::exception& e) {
      bp.errors[s] = e.what();
    }
  }
  return bp;
}

std::vector<int> balance_replicas(std::span<const double> times, int replica_count) {
  const std::size_t m = times.size();
  if (replica_count < 1) throw std::invalid_argument("replica count must be >= 1");
  if (m < static_cast<std::size_t>(replica_count))
    throw std::invalid_argument("need at least as many micro-batches as replicas");
  if (replica_count == 1) return std::vector<int>(m, 0);
  const std::size_t k = static_cast<std::size_t>(replica_count);
  // A partial k-way split: subset sums in descending order with their members.
  struct Part {
    std::vector<double> sums;
    std::vector<std::vector<int>> members;
    double spread;
    int min_index;
    std::uint64_t seq;
  };
  struct ByPriority {  // largest spread first, then lowest index, then age
    bool operator()(const Part& a, const Part& b) const {
      if (a.spread != b.spread) return a.spread > b.spread;
      if (a.min_index != b.min_index) return a.min_index < b.min_index;
      return a.seq < b.seq;
    }
  };
  std::multiset<Part, ByPriority> heap;
  for (std::size_t i = 0; i < m; ++i) {
    Part p{std::vector<double>(k, 0.0), std::vector<std::vector<int>>(k), times[i],
           static_cast<int>(i), i};
    p.sums[0] = times[i];
    p.members[0] = {static_cast<int>(i)};
    heap.insert(std::move(p));
  }
  std::uint64_t seq = m;
  while (heap.size() > 1) {
    Part a = *heap.begin();
    heap.erase(heap.begin());
    Part b = *heap.begin();
    heap.erase(heap.begin());
    // heaviest of one side with the lightest of the other
    std::vector<std::pair<double, std::vector<int>>> merged(k);
    for (std::size_t q = 0; q < k; ++q) {
      merged[q].first = a.sums[q] + b.sums[k - 1 - q];
      merged[q].second = a.members[q];
      merged[q].second.insert(merged[q].second.end(), b.members[k - 1 - q].begin(),
                              b.members[k - 1 - q].end());
    }
    std::stable_sort(merged.begin(), merged.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    Part c{std::vector<double>(k), std::vector<std::vector<int>>(k), 0.0,
           std::min(a.min_index, b.min_index), seq++};
    for (std::size_t q = 0; q < k; ++q) {
      c.sums[q] = merged[q].first;
      c.members[q] = std::move(merged[q].second);
    }
    c.spread = c.sums.front() - c.sums.back();
    heap.insert(std::move(c));
  }
  const Part& last = *heap.begin();
  auto key = [&](std::size_t g) {
    return last.members[g].empty()
               ? static_cast<int>(m) + static_cast<int>(g)
               : *std::min_element(last.members[g].begin(), last.members[g].end());
  };
  std::vector<std::size_t> order(k);
  for (std::size_t g = 0; g < k; ++g) order[g] = g;
  std::sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) { return key(x) < key(y); });
  std::vector<int> assign(m, 0);
  for (std::size_t r = 0; r < k; ++r)
    for (int mb : last.members[order[r]]) assign[static_cast<std::size_t>(mb)] = static_cast<int>(r);
  return assign;
}

PaddingEfficiency padding_efficiency(const MicroBatchPartition& partition) {
  if (partition.micro_batches.empty())
    throw std::invalid_argument("padding efficiency of an empty partition");
  std::int64_t in_real = 0, in_pad = 0, tg_real = 0, tg_pad = 0;
  for (const MicroBatch& mb : partition.micro_batches) {
    in_real += mb.input_tokens;
    in_pad += mb.padded_mbs * mb.padded_input_len;
    tg_real += mb.target_tokens;
    tg_pad += mb.padded_mbs * mb.padded_target_len;
  }
  PaddingEfficiency e;
  e.input = in_pad == 0 ? 1.0 : static_cast<double>(in_real) / static_cast<double>(in_pad);
  e.target = tg_pad == 0 ? 1.0 : static_cast<double>(tg_real) / static_cast<double>(tg_pad);
  return e;
}

}  // namespace pipeplan
