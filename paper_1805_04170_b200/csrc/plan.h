// In-memory model of a tileplan ExecutionPlan (proj/include/tileplan/execgraph.hpp:15-48) as
// read from its JSON wire format (export_plan / parse_plan, proj/src/execgraph.cpp:323-400),
// plus the graph it embeds (graph.hpp:15-106, JSON schema graph.cpp:320-430).
#pragma once
#include <array>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace tpx {

using Shape = std::vector<int64_t>;

// Axis-aligned box [lo, hi) per dimension (tiling.hpp:76-87).
struct Region {
  std::vector<std::array<int64_t, 2>> b;
  int rank() const { return int(b.size()); }
  int64_t volume() const;
  Shape shape() const;
  Region intersect(const Region& o) const;
  bool contains(const Region& o) const;  // o inside this
  bool operator==(const Region& o) const { return b == o.b; }
  bool operator!=(const Region& o) const { return b != o.b; }
  std::string str() const;
};

enum class OpKind { matmul, elementwise, conv, generic };
enum class EwFn { add, sub, scale, pointwise_fn, pointwise_fn_grad };
enum class ConvMode { forward, grad_weight, grad_input };
enum class NodeKind { buffer, slice, fetch, concat, sub_op, reduce_partial };

struct TensorSpec {
  std::string id;
  Shape shape;
  int dtype_bytes = 4;
  std::string role;
};

struct OpSpec {
  std::string id;
  OpKind kind = OpKind::generic;
  std::vector<std::string> inputs;
  std::string output;
  bool ta = false, tb = false;          // MatmulAttrs
  EwFn fn = EwFn::add;                  // EwAttrs
  double scale = 0.0;
  ConvMode mode = ConvMode::forward;    // ConvAttrs
  int row_dims[2] = {0, 0}, col_dims[2] = {0, 1}, inner_dims[2] = {1, 1};
  int batch_dim = 0;                    // GenericAttrs
};

struct PlanNode {
  std::string id;
  NodeKind kind = NodeKind::buffer;
  int device = 0;
  std::string tensor, op, phase;
  Region region;
  int partial = -1;
  std::vector<int> sources;  // node indices, paste order
  int64_t bytes = 0;
  int src_device = -1;
};

struct Plan {
  int k = 0;
  int devices = 1;
  std::map<std::string, TensorSpec> tensors;
  std::vector<OpSpec> ops;
  std::map<std::string, int> op_index;
  std::vector<PlanNode> nodes;
  std::map<std::string, int> node_index;
  std::map<std::string, std::vector<int>> holders;  // tensor -> node index per device
  std::map<std::string, std::string> assignment;    // tensor -> tiling string
  int64_t fetch_bytes_total = 0;                    // recomputed from the nodes
  std::vector<std::string> phase_order;             // first-appearance order (execgraph.cpp:41-47)

  const TensorSpec& tensor(const std::string& id) const;
  const OpSpec& op(const std::string& id) const;
  int node(const std::string& id) const;
};

// Parses and validates a plan document.  Errors name the offending node / tensor / op, as
// the reference executor does (simulator.cpp:102-122, dense.cpp:165-206).
Plan parse_plan(const std::string& json_text);

// Expected output shape of op given concrete operand shapes (graph.cpp:442-502 rules);
// throws with the reference's messages on mismatch.
Shape op_output_shape(const OpSpec& op, const std::vector<Shape>& ins);

const char* to_string(NodeKind k);

}  // namespace tpx
