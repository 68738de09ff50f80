// The reference-side adapter of INTEGRATION.md, compiled for real: what a maintainer adds to
// proj/src/ to run the reference's ExecutionPlan on B200 through the C ABI (include/tpx.h).
//
//   NumericCheck execute_numeric_b200(const ExecutionPlan&, seed, precision, flags)
//       = execute_numeric (proj/src/simulator.cpp:55-149) with the node loop replaced by
//         tpx_load_plan + tpx_init_inputs + tpx_execute, and the same comparison against the
//         reference's own serial_execute (proj/src/oracle.cpp:176-202), same metric
//         (simulator.cpp:129-147).
//   std::map<std::string, int64_t> phase_bytes_b200(const ExecutionPlan&)
//       = the per-phase fetch bytes of the B200 lowering (host-only context, no GPU), for the
//         byte contract against simulate_traffic (simulator.cpp:11-49).
// Errors from the C ABI are rethrown as tileplan::Error (proj/include/tileplan/error.hpp:8-12).
// Built by oracle/Makefile (target adapter) against the unmodified reference sources; not part
// of the product library.
#include "simulator_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "tileplan/error.hpp"
#include "tileplan/oracle.hpp"
#include "tpx.h"

namespace tileplan {

static void ok(int status) {
  if (status != TPX_OK) fail(std::string("b200: ") + tpx_last_error());
}

NumericCheck execute_numeric_b200(const ExecutionPlan& p, std::uint64_t seed, int precision, int flags) {
  const std::string doc = export_plan(p);  // execgraph.cpp:323
  tpx_ctx* ctx = nullptr;
  ok(tpx_create(/*cuda_ordinal=*/0, /*rank=*/0, /*world=*/1, &ctx));
  tpx_plan* plan = nullptr;
  const int st = tpx_load_plan(ctx, doc.data(), doc.size(), precision, flags, &plan);
  if (st != TPX_OK) {
    tpx_destroy(ctx);
    ok(st);
  }
  ok(tpx_init_inputs(plan, seed));
  ok(tpx_execute(plan));
  ok(tpx_synchronize(plan));
  auto serial = serial_execute(p.graph, seed);  // oracle.cpp:176-202
  NumericCheck c;
  c.seed = seed;
  for (const auto& [tensor, holder_ids] : p.holders) {
    for (const auto& hid : holder_ids) {
      const ExecNode& n = p.node(hid);
      DenseTensor want = extract_region(serial.at(tensor), Region::full(p.graph.tensor(tensor).shape), n.region);
      std::vector<double> got(static_cast<std::size_t>(want.elements()));
      ok(tpx_read_node(plan, hid.c_str(), got.data(), want.elements()));
      for (std::size_t i = 0; i < got.size(); ++i) {
        const double d = std::abs(got[i] - want.data[i]);
        c.max_abs = std::max(c.max_abs, d);
        c.max_rel = std::max(c.max_rel, d / std::max(std::abs(want.data[i]), 1.0));
      }
      c.values += want.elements();
    }
  }
  tpx_plan_free(plan);
  tpx_destroy(ctx);
  return c;
}

std::string describe_b200(const ExecutionPlan& p, int rank, int world, int flags) {
  const std::string doc = export_plan(p);
  tpx_ctx* ctx = nullptr;
  ok(tpx_create(/*host-only*/ -1, rank, world, &ctx));
  tpx_plan* plan = nullptr;
  const int st = tpx_load_plan(ctx, doc.data(), doc.size(), TPX_PREC_TF32, flags, &plan);
  if (st != TPX_OK) {
    tpx_destroy(ctx);
    ok(st);
  }
  char* s = nullptr;
  ok(tpx_plan_describe(plan, &s));
  std::string out(s);
  tpx_free_string(s);
  tpx_plan_free(plan);
  tpx_destroy(ctx);
  return out;
}

}  // namespace tileplan
