// Formatting of device-emitted plans and the epoch index (include/pipeplan/
// plan_file.h).  The text layout is the reference's save_plan
// (src/comm_plan.cpp:313-342) and run_plan's plans_index.csv
// (src/driver.cpp:246-283); instruction kinds use the reference's InstrKind
// numbering and names (comm_plan.h:28-39, comm_plan.cpp:30-33).
#include "pipeplan/plan_file.h"

#include <cstdio>
#include <sstream>

#include "pipeplan_b200.h"

namespace pipeplan {
namespace b200 {

namespace {

constexpr const char* kInstr[10] = {"ForwardPass",   "BackwardPass", "SendActStart", "RecvActStart",
                                    "SendGradStart", "RecvGradStart", "WaitSendAct", "WaitRecvAct",
                                    "WaitSendGrad",  "WaitRecvGrad"};

// Peer stage of a transfer instruction on stage j: activations flow to
// j + 1, gradients to j - 1 (comm_plan.cpp:164-175, 205-221).
int peer_of(int kind, int j) {
  switch (kind) {
    case 2: case 6: case 5: case 9: return j + 1;  // SendAct / WaitSendAct / RecvGrad / WaitRecvGrad
    default: return j - 1;                          // RecvAct / WaitRecvAct / SendGrad / WaitSendGrad
  }
}

std::string fmt(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string csv_cell(std::string s) {
  for (char& c : s)
    if (c == ',' || c == '\n') c = ';';
  return s;
}

}  // namespace

void save_plan_text(const EmittedPlan& p, std::ostream& out) {
  const int C = static_cast<int>(p.devices.size());
  out << "pipeplan-plan 1\n";
  out << "iteration " << p.iteration << "\n";
  out << "replica " << p.replica << "\n";
  out << "stages " << C << "\n";
  out << "hidden " << p.hidden_dim << "\n";
  out << "encdec " << (p.encoder_decoder ? 1 : 0) << "\n";
  out << "recompute " << to_string(p.recompute) << "\n";
  out << "stage_layers";
  for (const auto& s : p.stage_layers) out << ' ' << s.encoder_layers << ':' << s.decoder_layers;
  out << "\nmicrobatches " << p.shapes.size() << "\n";
  for (std::size_t i = 0; i < p.shapes.size(); ++i)
    out << "mb " << i << ' ' << p.shapes[i].mbs << ' ' << p.shapes[i].input_len << ' ' << p.shapes[i].target_len
        << "\n";
  for (int j = 0; j < C; ++j) {
    const auto& ins = p.devices[static_cast<std::size_t>(j)];
    out << "device " << j << " ops " << ins.size() << "\n";
    for (const std::int32_t w : ins) {
      const int kind = w & 15, mb = w >> 4;
      out << kInstr[kind] << ' ' << mb;
      if (kind >= 2) {  // a transfer: peer and boundary_shape (comm_plan.cpp:104-113)
        const PaddedShape& s = p.shapes[static_cast<std::size_t>(mb)];
        out << " peer " << peer_of(kind, j) << " shape " << s.mbs << ' ' << s.input_len;
        if (p.encoder_decoder) out << ' ' << s.target_len;
        out << ' ' << p.hidden_dim;
      }
      out << "\n";
    }
  }
  out << "end\n";
}

std::string plan_to_text(const EmittedPlan& plan) {
  std::ostringstream os;
  save_plan_text(plan, os);
  return os.str();
}

std::string plans_index_header() {
  return "iteration,replica,micro_batches,strategy,objective,t_max,max_replica_load,"
         "padding_eff_input,padding_eff_target,predicted_makespan,bubble_ratio,peak_mem_max,"
         "feasible,reason\n";
}

std::string plans_index_row(const IndexRow& r) {
  std::ostringstream os;
  os << r.iteration << ',' << r.replica << ',' << r.micro_batches << ',' << to_string(r.strategy) << ','
     << fmt(r.objective) << ',' << fmt(r.t_max) << ',' << fmt(r.max_replica_load) << ','
     << fmt(r.padding_eff_input) << ',' << fmt(r.padding_eff_target) << ',' << fmt(r.predicted_makespan) << ','
     << fmt(r.bubble_ratio) << ',' << fmt(r.peak_mem_max) << ",1,\n";
  return os.str();
}

std::string plans_index_infeasible_row(std::int64_t iteration, const std::string& reason) {
  std::ostringstream os;
  os << iteration << ",-1,0,,,,,,,,,,0," << csv_cell(reason) << "\n";
  return os.str();
}

}  // namespace b200
}  // namespace pipeplan

// C face of the plan text (for hosts without the C++ API): table s of a
// pp_emit_plans result with its shapes and model (pp_model_desc stage
// layouts), into out (cap bytes, NUL-terminated); *len = the text's length.
extern "C" int pp_format_plan(const int32_t* instructions, const int32_t* n_instructions, int32_t n_stages,
                              int32_t micro_batches, const pp_padded_shape* shapes, const pp_model_desc* model,
                              int64_t iteration, int32_t replica, int64_t hidden_dim, char* out, int64_t cap,
                              int64_t* len) {
  using namespace pipeplan;
  if (!instructions || !n_instructions || n_stages < 1 || micro_batches < 0 || (micro_batches > 0 && !shapes) ||
      !model || model->n_stages != n_stages || !len)
    return PP_ERR_INVALID;
  b200::EmittedPlan p;
  p.iteration = iteration;
  p.replica = replica;
  p.hidden_dim = hidden_dim;
  p.encoder_decoder = model->is_encoder_decoder != 0;
  if (model->recompute < 0 || model->recompute > 2) return PP_ERR_INVALID;
  p.recompute = static_cast<Recompute>(model->recompute);
  for (int j = 0; j < n_stages; ++j)
    p.stage_layers.push_back(StageLayout{model->encoder_layers[j], model->decoder_layers[j]});
  for (int i = 0; i < micro_batches; ++i) p.shapes.push_back({shapes[i].mbs, shapes[i].input_len, shapes[i].target_len});
  for (int j = 0; j < n_stages; ++j) {
    const int32_t* a = instructions + static_cast<int64_t>(10) * micro_batches * j;
    p.devices.emplace_back(a, a + n_instructions[j]);
    for (const int32_t w : p.devices.back())
      if ((w & 15) > 9 || (w >> 4) < 0 || (w >> 4) >= micro_batches) return PP_ERR_INVALID;
  }
  const std::string t = b200::plan_to_text(p);
  *len = static_cast<int64_t>(t.size());
  if (out && cap > 0) {
    const std::size_t n = std::min<std::size_t>(t.size(), static_cast<std::size_t>(cap - 1));
    std::copy(t.begin(), t.begin() + static_cast<std::ptrdiff_t>(n), out);
    out[n] = 0;
  }
  return PP_OK;
}
