// padding_report.cpp — pipeplan::b200::padding_vs_packing_report over the
// C-ABI (pp_padding_report; kernels in csrc/report.cu, sched.cu, dp.cu).
#include "pipeplan/padding_report.h"

#include <stdexcept>
#include <string>

#include "pipeplan/errors.h"
#include "pipeplan_b200.h"

namespace pipeplan {
namespace detail {
pp_ctx* device_ctx();  // microbatch.cpp
}

namespace b200 {

std::vector<PaddingRow> padding_vs_packing_report(std::span<const Sample> samples,
                                                  std::span<const std::int64_t> max_seq_lens,
                                                  const ProfileGrid& grid, const ModelConfig& config,
                                                  const PaddingReportOptions& options) {
  if (samples.empty()) throw std::invalid_argument("padding report needs a non-empty dataset");
  std::vector<std::int32_t> enc, dec;
  for (const StageLayout& s : config.stages) {
    enc.push_back(s.encoder_layers);
    dec.push_back(s.decoder_layers);
  }
  pp_model_desc m{config.stage_count(), enc.data(), dec.data(), config.is_encoder_decoder ? 1 : 0, 0};
  const pp_grid_desc gd = grid.device_desc();
  std::vector<pp_padding_row> rows(3 * max_seq_lens.size());
  pp_ctx* ctx = detail::device_ctx();
  const int rc = pp_padding_report(ctx, reinterpret_cast<const pp_sample*>(samples.data()),
                                   static_cast<std::int64_t>(samples.size()), max_seq_lens.data(),
                                   static_cast<std::int32_t>(max_seq_lens.size()), &gd, &m, options.token_budget,
                                   options.t_max_interval, options.max_iterations,
                                   static_cast<std::int32_t>(options.recompute), rows.data());
  if (rc == PP_ERR_INVALID) throw std::invalid_argument(pp_ctx_last_error(ctx));
  if (rc == PP_ERR_INFEASIBLE || rc == PP_ERR_INFEASIBLE_SAMPLE)
    throw InfeasibleError(pp_ctx_last_error(ctx), -1, -1);
  if (rc != PP_OK) throw std::runtime_error(std::string("pipeplan_b200 device error: ") + pp_ctx_last_error(ctx));
  std::vector<PaddingRow> out(rows.size());
  for (std::size_t k = 0; k < rows.size(); ++k) {
    const pp_padding_row& r = rows[k];
    out[k] = PaddingRow{static_cast<BatchingMethod>(r.method), r.max_seq_len, r.padding_eff_input,
                        r.padding_eff_target, r.tokens, r.sim_time, r.throughput_proxy};
  }
  return out;
}

}  // namespace b200
}  // namespace pipeplan
