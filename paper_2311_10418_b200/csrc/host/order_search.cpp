// order_search.cpp — pipeplan::b200::search_injection_orders over the C-ABI
// (pp_order_search, kernels in csrc/sched.cu).  See include/pipeplan/order_search.h.
#include "pipeplan/order_search.h"

#include <stdexcept>
#include <string>

#include "pipeplan_b200.h"

namespace pipeplan {
namespace detail {
pp_ctx* device_ctx();  // microbatch.cpp
}

namespace b200 {

std::vector<InjectionOrder> search_injection_orders(std::span<const OpCostTable> tables,
                                                    std::span<const double> limits, int n_clusters,
                                                    double comm_latency) {
  const int n = static_cast<int>(tables.size());
  std::vector<InjectionOrder> out(static_cast<std::size_t>(n));
  if (n == 0) return out;
  const int C = tables[0].stages;
  if (static_cast<int>(limits.size()) != C)  // schedule.cpp:62-63
    throw std::invalid_argument("one memory limit per device required");
  std::vector<std::int64_t> off(static_cast<std::size_t>(n) + 1, 0);
  for (int s = 0; s < n; ++s) {
    const OpCostTable& t = tables[static_cast<std::size_t>(s)];
    if (t.stages != C) throw std::invalid_argument("all tables must have the same stage count");
    if (t.micro_batches < 1) throw std::invalid_argument("need at least one micro-batch");  // :281
    off[static_cast<std::size_t>(s) + 1] = off[static_cast<std::size_t>(s)] + t.micro_batches;
  }
  if (n_clusters < 1) throw std::invalid_argument("n_clusters must be >= 1");  // :284
  const std::size_t rows = static_cast<std::size_t>(off.back());
  std::vector<double> tf(rows * C), tb(rows * C), act(rows * C);
  for (int s = 0; s < n; ++s) {
    const OpCostTable& t = tables[static_cast<std::size_t>(s)];
    const std::size_t o = static_cast<std::size_t>(off[static_cast<std::size_t>(s)]) * C;
    std::copy(t.t_f.begin(), t.t_f.end(), tf.begin() + o);
    std::copy(t.t_b.begin(), t.t_b.end(), tb.begin() + o);
    std::copy(t.act_mem.begin(), t.act_mem.end(), act.begin() + o);
  }
  std::vector<std::int32_t> order(rows), dl(n), st(n);
  std::vector<double> ms(n), bub(n), ds(static_cast<std::size_t>(n) * C * 5);
  pp_ctx* ctx = detail::device_ctx();
  const int rc = pp_order_search(ctx, tf.data(), tb.data(), act.data(), off.data(), n, C, limits.data(),
                                 n_clusters, comm_latency, order.data(), ms.data(), bub.data(), dl.data(),
                                 ds.data(), st.data());
  if (rc == PP_ERR_INVALID) throw std::invalid_argument(pp_ctx_last_error(ctx));
  if (rc != PP_OK) throw std::runtime_error(std::string("pipeplan_b200 device error: ") + pp_ctx_last_error(ctx));
  for (int s = 0; s < n; ++s) {
    switch (st[static_cast<std::size_t>(s)]) {
      case PP_OK:
        break;
      case PP_ERR_NOT_CONVERGED:
        throw std::logic_error("adaptive scheduler failed to converge; invariant violated");
      case PP_ERR_NOT_EXECUTABLE:
        throw std::logic_error("schedule is not executable: circular dependency between devices");
      case PP_ERR_INVALID:  // a device limit (order_search.h), not a reference error
        throw std::invalid_argument("op durations must be non-negative and not NaN (device order search)");
      default:
        throw std::runtime_error("pipeplan_b200 device order search: status " +
                                 std::to_string(st[static_cast<std::size_t>(s)]));
    }
    InjectionOrder& r = out[static_cast<std::size_t>(s)];
    const std::int64_t b = off[static_cast<std::size_t>(s)], m = off[static_cast<std::size_t>(s) + 1] - b;
    if (order[static_cast<std::size_t>(b)] >= 0) r.order.assign(order.begin() + b, order.begin() + b + m);
    r.makespan = ms[static_cast<std::size_t>(s)];
    r.bubble_ratio = bub[static_cast<std::size_t>(s)];
    r.deadlock = dl[static_cast<std::size_t>(s)] != 0;
    r.devices.resize(static_cast<std::size_t>(C));
    for (int j = 0; j < C; ++j) {
      const double* d = ds.data() + (static_cast<std::size_t>(s) * C + j) * 5;
      r.devices[static_cast<std::size_t>(j)] = {d[0], d[1], d[2], d[3], d[4]};
    }
  }
  return out;
}

InjectionOrder search_injection_order(const OpCostTable& costs, std::span<const double> limits,
                                      int n_clusters, double comm_latency) {
  return search_injection_orders(std::span<const OpCostTable>(&costs, 1), limits, n_clusters, comm_latency)[0];
}

}  // namespace b200
}  // namespace pipeplan
