// padding_report.h — padding_vs_packing_report on the B200 (SURVEY.md §8f
// row 4), C++ face of pp_padding_report (include/pipeplan_b200.h).
//
// Same inputs and rows as the reference's padding_vs_packing_report
// (proj/include/pipeplan/simulate.h:102-121, src/simulate.cpp:288-406);
// the row and option types live in namespace pipeplan::b200 so this header
// can sit next to the reference's simulate.h.  Rows are bit-identical to the
// reference's (tests/test_padding_report.py, tests/cpp/order_dropin.cpp).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "pipeplan/cost_model.h"
#include "pipeplan/workload.h"

namespace pipeplan::b200 {

enum class BatchingMethod { DpMicrobatch, Packing, NaivePadding };  // simulate.h:73

struct PaddingRow {  // simulate.h:92-100
  BatchingMethod method = BatchingMethod::DpMicrobatch;
  std::int64_t max_seq_len = 0;
  double padding_eff_input = 1.0;
  double padding_eff_target = 1.0;
  std::int64_t tokens = 0;
  double sim_time = 0.0;
  double throughput_proxy = 0.0;
};

struct PaddingReportOptions {  // simulate.h:102-107
  std::int64_t token_budget = 65536;
  double t_max_interval = 5.0;
  int max_iterations = 0;  // 0 = whole epoch
  Recompute recompute = Recompute::None;
};

/// One batched device call per max_seq_len; throws std::invalid_argument for
/// an empty dataset / bad budget and the DP's InfeasibleError.
std::vector<PaddingRow> padding_vs_packing_report(std::span<const Sample> samples,
                                                  std::span<const std::int64_t> max_seq_lens,
                                                  const ProfileGrid& grid, const ModelConfig& config,
                                                  const PaddingReportOptions& options);

}  // namespace pipeplan::b200
