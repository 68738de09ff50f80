// Driver of the reference-side adapter: the reference's own planner API end to end, then the
// B200 executor.  gen_mlp (proj/src/graph.cpp:179-229) -> kcuts / preset_assignment
// (proj/src/kcuts.cpp:35-60, assign.cpp:36-81) -> place_k (placement.cpp:101) ->
// build_execution_graph (execgraph.cpp:295) ->
//   bytes:  per-phase fetch bytes of the B200 lowering, for every rank of a 2^k-rank job and in
//           peer mode, == simulate_traffic (simulator.cpp:11-49) phase totals (host-only)
//   --gpu:  execute_numeric_b200 (3xTF32, fp32-accurate) vs serial_execute, NumericCheck JSON
// Prints one JSON object; exit 0 when every check passes.
//   adapter_b200 BATCH K MODE(opt|data|model|hybrid) DIM... [--gpu]
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "json.hpp"  // nlohmann/json (oracle/Makefile JSON_DIR)

#include "simulator_b200.hpp"
#include "tileplan/assign.hpp"
#include "tileplan/execgraph.hpp"
#include "tileplan/graph.hpp"
#include "tileplan/kcuts.hpp"
#include "tileplan/placement.hpp"
#include "tileplan/simulator.hpp"
#include "tpx.h"

using namespace tileplan;
using nlohmann::json;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s BATCH K MODE DIM... [--gpu]\n", argv[0]);
    return 2;
  }
  try {
    MlpConfig cfg;
    cfg.batch = std::atoll(argv[1]);
    const int k = std::atoi(argv[2]);
    const std::string mode = argv[3];
    bool gpu = false;
    for (int i = 4; i < argc; ++i) {
      if (std::string(argv[i]) == "--gpu") gpu = true;
      else cfg.dims.push_back(std::atoll(argv[i]));
    }
    cfg.with_backward = cfg.with_update = true;
    DataflowGraph g = gen_mlp(cfg);
    TilingAssignment a = mode == "opt" ? kcuts(g, k).assignment : preset_assignment(g, preset_from_string(mode), k);
    const std::string hdoc = k == 0 ? std::string(R"({"levels":[]})")
                                    : R"({"levels":[{"label":"nvswitch","fanout":)" + std::to_string(1 << k) +
                                          R"(,"bandwidth_bytes_per_s":9e11}]})";
    const DeviceHierarchy h = parse_hierarchy(hdoc);
    ExecutionPlan p = build_execution_graph(g, a, place_k(k, h));
    TrafficReport tr = simulate_traffic(p, h);
    std::map<std::string, std::int64_t> want;
    for (const auto& row : tr.phases)
      if (row.bytes) want[row.phase] = row.bytes;
    json out;
    out["fetch_bytes_total"] = p.fetch_bytes_total();
    out["est_seconds"] = tr.est_seconds;
    bool pass = true;
    const int world = 1 << k;
    for (int flags : {TPX_FLAG_FUSE, TPX_FLAG_FUSE | TPX_FLAG_PEER}) {
      std::map<std::string, std::int64_t> got;
      for (int r = 0; r < world; ++r) {
        json d = json::parse(describe_b200(p, r, world, flags));
        for (auto& [ph, b] : d["per_phase_fetch_bytes_in"].items())
          if (b.get<std::int64_t>()) got[ph] += b.get<std::int64_t>();
      }
      const bool same = got == want;
      out[flags & TPX_FLAG_PEER ? "phase_bytes_match_peer" : "phase_bytes_match"] = same;
      pass = pass && same;
    }
    out["phases"] = want.size();
    if (gpu) {
      NumericCheck c = execute_numeric_b200(p, 7, TPX_PREC_FP32, TPX_FLAG_FUSE);
      out["numeric"] = {{"max_abs", c.max_abs}, {"max_rel", c.max_rel}, {"values", c.values}, {"seed", c.seed}};
    }
    out["pass"] = pass;
    std::printf("%s\n", out.dump().c_str());
    return pass ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("{\"error\": %s}\n", json(std::string(e.what())).dump().c_str());
    return 1;
  }
}
