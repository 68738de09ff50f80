// TEST INFRASTRUCTURE ONLY — never linked into, loaded by or called from the product path.
//
// Thin extern "C" driver over the UNMODIFIED reference library (tileplan, built from the
// sources under /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests, the fixture generators (tools/) and bench.py's cpu_baseline / --impl reference
// leg call the reference's own public API:
//   gen_mlp / gen_cnn            proj/src/graph.cpp:179-314
//   preset_assignment            proj/src/assign.cpp:36-81
//   kcuts                        proj/src/kcuts.cpp:35-60
//   graph_cost / op_comm_cost    proj/src/cost.cpp:169-253
//   place_k / parse_hierarchy    proj/src/placement.cpp:45-116
//   build_execution_graph        proj/src/execgraph.cpp:295-305
//   export_plan / parse_plan     proj/src/execgraph.cpp:323-400
//   simulate_traffic             proj/src/simulator.cpp:11-49
//   execute_numeric              proj/src/simulator.cpp:55-149
//   serial_execute               proj/src/oracle.cpp:176-202
// A "session" re-runs execute_numeric's node loop through the reference's own
// extract_region / paste_region / run_op_dense (dense.cpp:161-259) so every node value of
// the tiled CPU execution can be read back as fp64 golden data.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "tileplan/assign.hpp"
#include "tileplan/cost.hpp"
#include "tileplan/dense.hpp"
#include "tileplan/error.hpp"
#include "tileplan/execgraph.hpp"
#include "tileplan/graph.hpp"
#include "tileplan/kcuts.hpp"
#include "tileplan/oracle.hpp"
#include "tileplan/placement.hpp"
#include "tileplan/simulator.hpp"

using namespace tileplan;
using nlohmann::json;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <class F>
char* guard_str(F&& f) {
  try {
    return dup(f());
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

template <class F>
int guard_int(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

DataflowGraph load_graph(const char* text) {
  DataflowGraph g = parse_graph(text);
  validate_and_infer(g);
  return g;
}

json assignment_json(const TilingAssignment& a) {
  json j;
  j["k"] = a.k;
  json t = json::object();
  for (const auto& [id, tl] : a.tilings) t[id] = tl.str();
  j["tilings"] = t;
  return j;
}

TilingAssignment assignment_from(const DataflowGraph& g, const std::string& mode, int k) {
  if (mode == "data" || mode == "model" || mode == "hybrid")
    return preset_assignment(g, preset_from_string(mode), k);
  if (mode == "opt") return kcuts(g, k).assignment;
  // otherwise an assignment document {"k":..,"tilings":{..}}
  json j = json::parse(mode);
  TilingAssignment a;
  a.k = j.at("k").get<int>();
  for (const auto& [id, t] : j.at("tilings").items()) a.tilings[id] = Tiling::parse(t.get<std::string>());
  return a;
}

struct Session {
  ExecutionPlan plan;
  std::map<std::string, DenseTensor> serial;
  struct Value {
    Region region;
    DenseTensor dense;
  };
  std::map<std::string, Value> values;
  double serial_seconds = 0, tiled_seconds = 0;
};

Shape region_shape(const Region& r) {
  Shape s;
  for (const auto& b : r.bounds) s.push_back(b[1] - b[0]);
  return s;
}

// Same node semantics as execute_numeric (simulator.cpp:77-127), through the reference's
// own region and kernel functions, keeping every node value.
void run_nodes(Session& s, const FunctionBindings& fb) {
  const DataflowGraph& g = s.plan.graph;
  std::map<std::string, const OpNode*> ops;
  for (const auto& op : g.ops) ops[op.id] = &op;
  for (const auto& n : s.plan.nodes) {
    Session::Value v;
    v.region = n.region;
    switch (n.kind) {
      case NodeKind::buffer: {
        const TensorSpec& spec = g.tensor(n.tensor);
        v.dense = extract_region(s.serial.at(n.tensor), Region::full(spec.shape), n.region);
        break;
      }
      case NodeKind::slice:
      case NodeKind::fetch: {
        const auto& src = s.values.at(n.sources.at(0));
        v.dense = extract_region(src.dense, src.region, n.region);
        break;
      }
      case NodeKind::concat: {
        v.dense = DenseTensor::zeros(region_shape(n.region));
        for (const auto& sid : n.sources) {
          const auto& piece = s.values.at(sid);
          paste_region(v.dense, n.region, piece.dense, piece.region, false);
        }
        break;
      }
      case NodeKind::reduce_partial: {
        v.dense = DenseTensor::zeros(region_shape(n.region));
        for (const auto& sid : n.sources) {
          const auto& piece = s.values.at(sid);
          paste_region(v.dense, n.region, piece.dense, piece.region, true);
        }
        break;
      }
      case NodeKind::sub_op: {
        std::vector<const DenseTensor*> ins;
        for (const auto& sid : n.sources) ins.push_back(&s.values.at(sid).dense);
        v.dense = run_op_dense(*ops.at(n.op), ins, fb);
        break;
      }
    }
    s.values[n.id] = std::move(v);
  }
}

int copy_out(const DenseTensor& t, double* out, std::int64_t n) {
  if (n != t.elements()) fail("buffer has " + std::to_string(n) + " elements, value has " +
                              std::to_string(t.elements()));
  std::memcpy(out, t.data.data(), sizeof(double) * static_cast<std::size_t>(n));
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// gen_mlp (graph.cpp:179-229); dtype_bytes is applied to every tensor afterwards.
char* ref_gen_mlp(std::int64_t batch, const std::int64_t* dims, int ndims, int backward,
                  int update, double lr, int dtype_bytes) {
  return guard_str([&] {
    MlpConfig c;
    c.batch = batch;
    c.dims.assign(dims, dims + ndims);
    c.with_backward = backward != 0;
    c.with_update = update != 0;
    c.learning_rate = lr;
    DataflowGraph g = gen_mlp(c);
    for (auto& [id, t] : g.tensors) t.dtype_bytes = dtype_bytes;
    validate_and_infer(g);
    return serialize_graph(g);
  });
}

// gen_cnn (graph.cpp:231-314).
char* ref_gen_cnn(std::int64_t batch, std::int64_t h, std::int64_t w, const std::int64_t* ch,
                  int nch, std::int64_t fh, std::int64_t fw, int backward, int dtype_bytes) {
  return guard_str([&] {
    DataflowGraph g = gen_cnn(batch, {h, w}, std::vector<std::int64_t>(ch, ch + nch), {fh, fw},
                              backward != 0);
    for (auto& [id, t] : g.tensors) t.dtype_bytes = dtype_bytes;
    validate_and_infer(g);
    return serialize_graph(g);
  });
}

// Assignment for a graph: mode = data|model|hybrid|opt or an assignment document.
char* ref_assignment(const char* graph_json, const char* mode, int k) {
  return guard_str([&] {
    DataflowGraph g = load_graph(graph_json);
    return assignment_json(assignment_from(g, mode, k)).dump(2);
  });
}

// kcuts result with per-cut costs and the flat graph_cost total (tools/main.cpp:236-253).
char* ref_kcuts(const char* graph_json, int k) {
  return guard_str([&] {
    DataflowGraph g = load_graph(graph_json);
    KCutResult r = kcuts(g, k);
    json j = assignment_json(r.assignment);
    j["per_cut"] = r.per_cut;
    j["recursion_total"] = r.total;
    CostReport c = graph_cost(g, r.assignment);
    j["flat_total_elements"] = c.total_elements;
    j["flat_total_bytes"] = c.total_bytes;
    return j.dump(2);
  });
}

// graph_cost (cost.cpp:244-253) plus the per-op exec tilings chosen by op_comm_cost.
char* ref_graph_cost(const char* graph_json, const char* mode, int k) {
  return guard_str([&] {
    DataflowGraph g = load_graph(graph_json);
    TilingAssignment a = assignment_from(g, mode, k);
    CostReport c = graph_cost(g, a);
    json j;
    json rows = json::array();
    for (std::size_t i = 0; i < c.per_op.size(); ++i) {
      const auto& p = c.per_op[i];
      OpCommCost cc = op_comm_cost(g, g.ops[i], a);
      json ex = json::array();
      for (const auto& t : cc.input_exec_tilings) ex.push_back(t.str());
      rows.push_back({{"op", p.op_id},
                      {"elements", p.elements},
                      {"bytes", p.bytes},
                      {"form", p.chosen_form},
                      {"input_exec_tilings", ex},
                      {"output_state", cc.output_state.str()}});
    }
    j["per_op"] = rows;
    j["total_elements"] = c.total_elements;
    j["total_bytes"] = c.total_bytes;
    j["assignment"] = assignment_json(a);
    return j.dump(2);
  });
}

// build_execution_graph + export_plan (execgraph.cpp:295-361).
char* ref_plan(const char* graph_json, const char* mode, int k, const char* hierarchy_json) {
  return guard_str([&] {
    DataflowGraph g = load_graph(graph_json);
    TilingAssignment a = assignment_from(g, mode, k);
    PlacementMap pm = place_k(k, parse_hierarchy(hierarchy_json));
    return export_plan(build_execution_graph(g, a, pm));
  });
}

// parse_plan + export_plan: byte-identical round trip (test_plan.cpp:101-119).
char* ref_plan_roundtrip(const char* plan_json) {
  return guard_str([&] { return export_plan(parse_plan(plan_json)); });
}

// simulate_traffic (simulator.cpp:11-49) as JSON.
char* ref_simulate_traffic(const char* plan_json, const char* hierarchy_json) {
  return guard_str([&] {
    ExecutionPlan p = parse_plan(plan_json);
    DeviceHierarchy h = hierarchy_json && *hierarchy_json ? parse_hierarchy(hierarchy_json)
                                                          : p.hierarchy;
    TrafficReport r = simulate_traffic(p, h);
    json j;
    json ph = json::array();
    for (const auto& row : r.phases)
      ph.push_back({{"phase", row.phase},
                    {"bytes", row.bytes},
                    {"level_bytes", row.level_bytes},
                    {"seconds", row.seconds}});
    j["phases"] = ph;
    j["level_bytes"] = r.level_bytes;
    j["device_in"] = r.device_in;
    j["device_out"] = r.device_out;
    j["total_bytes"] = r.total_bytes;
    j["est_seconds"] = r.est_seconds;
    return j.dump(2);
  });
}

// execute_numeric (simulator.cpp:55-149), with its wall time.
int ref_execute_numeric(const char* plan_json, std::uint64_t seed, double* max_abs,
                        double* max_rel, std::int64_t* values, double* seconds) {
  return guard_int([&] {
    ExecutionPlan p = parse_plan(plan_json);
    auto t0 = std::chrono::steady_clock::now();
    NumericCheck c = execute_numeric(p, seed);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *max_abs = c.max_abs;
    *max_rel = c.max_rel;
    *values = c.values;
  });
}

// `threads` independent execute_numeric runs of the same plan in parallel (the reference is
// single-threaded; this is how the CPU baseline uses every host core).  Returns the wall
// time of the whole batch.
int ref_execute_numeric_parallel(const char* plan_json, std::uint64_t seed, int threads,
                                 double* seconds) {
  return guard_int([&] {
    ExecutionPlan p = parse_plan(plan_json);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<std::size_t>(threads));
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < threads; ++i)
      pool.emplace_back([&, i] {
        try {
          (void)execute_numeric(p, seed);
        } catch (const std::exception& e) {
          errs[static_cast<std::size_t>(i)] = e.what();
        }
      });
    for (auto& t : pool) t.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& e : errs)
      if (!e.empty()) fail(e);
  });
}

// serial_execute alone (oracle.cpp:176-202), timed.
int ref_serial_seconds(const char* plan_json, std::uint64_t seed, double* seconds) {
  return guard_int([&] {
    ExecutionPlan p = parse_plan(plan_json);
    auto t0 = std::chrono::steady_clock::now();
    auto v = serial_execute(p.graph, seed);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    (void)v;
  });
}

void* ref_session_new(const char* plan_json, std::uint64_t seed) {
  try {
    auto* s = new Session;
    s->plan = parse_plan(plan_json);
    auto t0 = std::chrono::steady_clock::now();
    s->serial = serial_execute(s->plan.graph, seed);
    auto t1 = std::chrono::steady_clock::now();
    run_nodes(*s, FunctionBindings::standard());
    auto t2 = std::chrono::steady_clock::now();
    s->serial_seconds = std::chrono::duration<double>(t1 - t0).count();
    s->tiled_seconds = std::chrono::duration<double>(t2 - t1).count();
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_session_free(void* h) { delete static_cast<Session*>(h); }

int ref_session_times(void* h, double* serial_s, double* tiled_s) {
  auto* s = static_cast<Session*>(h);
  *serial_s = s->serial_seconds;
  *tiled_s = s->tiled_seconds;
  return 0;
}

// Full serial value of a tensor.
int ref_session_serial(void* h, const char* tensor, double* out, std::int64_t n) {
  return guard_int([&] { copy_out(static_cast<Session*>(h)->serial.at(tensor), out, n); });
}

// Value of any plan node (its region's block, row-major).
int ref_session_node(void* h, const char* node_id, double* out, std::int64_t n) {
  return guard_int([&] { copy_out(static_cast<Session*>(h)->values.at(node_id).dense, out, n); });
}

// A pool of `threads` sessions of the same plan (the reference is single-threaded; the CPU
// baseline uses every host core by running independent copies).  ref_pool_step re-runs the
// reference's tiled node loop (execute_numeric's simulator.cpp:77-127 semantics through the
// reference's extract_region / paste_region / run_op_dense) on every copy concurrently and
// returns the wall time.
struct Pool {
  std::vector<std::unique_ptr<Session>> s;
};

void* ref_pool_new(const char* plan_json, std::uint64_t seed, int threads) {
  try {
    auto* p = new Pool;
    ExecutionPlan plan = parse_plan(plan_json);
    p->s.resize(static_cast<std::size_t>(threads));
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<std::size_t>(threads));
    for (int i = 0; i < threads; ++i)
      pool.emplace_back([&, i] {
        try {
          auto s = std::make_unique<Session>();
          s->plan = plan;
          s->serial = serial_execute(s->plan.graph, seed);
          p->s[static_cast<std::size_t>(i)] = std::move(s);
        } catch (const std::exception& e) {
          errs[static_cast<std::size_t>(i)] = e.what();
        }
      });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (!e.empty()) {
        delete p;
        fail(e);
      }
    return p;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int ref_pool_step(void* h, double* seconds) {
  return guard_int([&] {
    auto* p = static_cast<Pool*>(h);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(p->s.size());
    auto t0 = std::chrono::steady_clock::now();
    for (std::size_t i = 0; i < p->s.size(); ++i)
      pool.emplace_back([&, i] {
        try {
          run_nodes(*p->s[i], FunctionBindings::standard());
        } catch (const std::exception& e) {
          errs[i] = e.what();
        }
      });
    for (auto& t : pool) t.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& e : errs)
      if (!e.empty()) fail(e);
  });
}

void ref_pool_free(void* h) { delete static_cast<Pool*>(h); }

}  // extern "C"
