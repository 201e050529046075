// capi_host.cpp — host-only C-ABI helpers: the drop-in C++ API's grid,
// dataset and slice-cost functions exposed to C / ctypes callers.
#include <algorithm>
#include <cstring>
#include <span>
#include <vector>
#include <stdexcept>

#include "pipeplan/cost_model.h"
#include "pipeplan/microbatch.h"
#include "pipeplan/workload.h"
#include "pipeplan_b200.h"

using namespace pipeplan;

namespace {

LengthDistribution dist_from(const double* d) {
  LengthDistribution l;
  l.family = static_cast<LengthFamily>(static_cast<int>(d[0]));
  l.log_mean = d[1];
  l.log_sigma = d[2];
  l.uniform_lo = static_cast<std::int64_t>(d[3]);
  l.uniform_hi = static_cast<std::int64_t>(d[4]);
  l.lognormal_weight = d[5];
  return l;
}

ModelConfig model_from(const pp_model_desc* m) {
  ModelConfig cfg;
  cfg.is_encoder_decoder = m->is_encoder_decoder != 0;
  for (int s = 0; s < m->n_stages; ++s)
    cfg.stages.push_back(StageLayout{m->encoder_layers[s], m->decoder_layers[s]});
  return cfg;
}

}  // namespace

extern "C" {

int pp_synthetic_grid(const double* params, int32_t tp_degree, const int64_t* mbs_axis,
                      int32_t n_mbs, const int64_t* seq_axis, int32_t n_seq, int64_t* out_mbs,
                      int64_t* out_seq, int32_t* out_sizes, double* out_cells) {
  try {
    SyntheticGridParams p;
    p.alpha = params[0];
    p.beta = params[1];
    p.gamma = params[2];
    p.full_mem_factor = params[3];
    p.selective_mem_factor = params[4];
    p.full_tb_penalty = params[5];
    p.selective_tb_penalty = params[6];
    p.tp_degree = tp_degree;
    ProfileGrid g = ProfileGrid::synthetic(p, std::vector<std::int64_t>(mbs_axis, mbs_axis + n_mbs),
                                           std::vector<std::int64_t>(seq_axis, seq_axis + n_seq));
    const pp_grid_desc d = g.device_desc();
    if (d.n_mbs > 64 || d.n_seq > 64) return PP_ERR_INVALID;
    out_sizes[0] = d.n_mbs;
    out_sizes[1] = d.n_seq;
    std::memcpy(out_mbs, d.mbs_axis, sizeof(int64_t) * d.n_mbs);
    std::memcpy(out_seq, d.seq_axis, sizeof(int64_t) * d.n_seq);
    std::memcpy(out_cells, d.cells, sizeof(double) * 18 * d.n_mbs * d.n_seq);
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

int pp_synthetic_dataset(int64_t n, const double* in_dist, const double* tgt_dist,
                         int64_t max_seq_len, uint64_t seed, pp_sample* out) {
  try {
    DatasetSpec spec;
    SyntheticSpec syn;
    syn.n = n;
    syn.input = dist_from(in_dist);
    if (tgt_dist) syn.target = dist_from(tgt_dist);
    spec.synthetic = syn;
    spec.max_seq_len = max_seq_len;
    spec.seed = seed;
    const std::vector<Sample> s = load_dataset(spec);
    std::memcpy(out, s.data(), sizeof(pp_sample) * s.size());
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

int pp_assign_replicas(const double* times, int64_t m, int32_t replica_count, int32_t* replica,
                       double* max_load) {
  if (m < 1 || replica_count < 1) return PP_ERR_INVALID;
  try {
    const std::span<const double> ts(times, static_cast<std::size_t>(m));
    std::vector<int> rep;
    if (m >= replica_count) {
      rep = balance_replicas(ts, replica_count);
    } else {
      rep.resize(static_cast<std::size_t>(m));
      for (int64_t k = 0; k < m; ++k) rep[static_cast<std::size_t>(k)] = static_cast<int>(k);
    }
    std::vector<double> load(static_cast<std::size_t>(replica_count), 0.0);
    for (int64_t k = 0; k < m; ++k) {
      replica[k] = rep[static_cast<std::size_t>(k)];
      load[static_cast<std::size_t>(rep[static_cast<std::size_t>(k)])] += ts[static_cast<std::size_t>(k)];
    }
    *max_load = *std::max_element(load.begin(), load.end());
    return PP_OK;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

int pp_slice_cost_host(const pp_grid_desc* grid, const pp_model_desc* model,
                       const pp_sample* ordered, int64_t begin, int64_t end, double* time,
                       double* act_mem) {
  try {
    const ProfileGrid g = ProfileGrid::from_desc(*grid);
    GridSliceCost c{&g, model_from(model),
                    std::vector<Sample>(reinterpret_cast<const Sample*>(ordered),
                                        reinterpret_cast<const Sample*>(ordered) + end),
                    static_cast<Recompute>(model->recompute)};
    const SliceCost sc = c(static_cast<std::size_t>(begin), static_cast<std::size_t>(end));
    *time = sc.time;
    *act_mem = sc.act_mem;
    return PP_OK;
  } catch (const std::out_of_range&) {
    return PP_ERR_OUT_OF_RANGE;
  } catch (const std::invalid_argument&) {
    return PP_ERR_INVALID;
  }
}

}  // extern "C"
