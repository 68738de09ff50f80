#include "plan.h"

#include <algorithm>
#include <set>

#include "json.h"
#include "util.h"

namespace tpx {

int64_t Region::volume() const {
  int64_t v = 1;
  for (const auto& x : b) {
    if (x[1] <= x[0]) return 0;
    v *= x[1] - x[0];
  }
  return v;
}

Shape Region::shape() const {
  Shape s;
  for (const auto& x : b) s.push_back(x[1] - x[0]);
  return s;
}

Region Region::intersect(const Region& o) const {
  if (b.size() != o.b.size()) fail("region rank mismatch");
  Region r;
  r.b.resize(b.size());
  for (size_t d = 0; d < b.size(); ++d) {
    r.b[d][0] = std::max(b[d][0], o.b[d][0]);
    r.b[d][1] = std::min(b[d][1], o.b[d][1]);
  }
  return r;
}

bool Region::contains(const Region& o) const {
  if (b.size() != o.b.size()) return false;
  for (size_t d = 0; d < b.size(); ++d)
    if (o.b[d][0] < b[d][0] || o.b[d][1] > b[d][1]) return false;
  return true;
}

std::string Region::str() const {
  std::string s = "[";
  for (size_t d = 0; d < b.size(); ++d) {
    if (d) s += ",";
    s += "[" + std::to_string(b[d][0]) + "," + std::to_string(b[d][1]) + ")";
  }
  return s + "]";
}

const char* to_string(NodeKind k) {
  switch (k) {
    case NodeKind::buffer: return "buffer";
    case NodeKind::slice: return "slice";
    case NodeKind::fetch: return "fetch";
    case NodeKind::concat: return "concat";
    case NodeKind::sub_op: return "sub_op";
    case NodeKind::reduce_partial: return "reduce_partial";
  }
  return "?";
}

const TensorSpec& Plan::tensor(const std::string& id) const {
  auto it = tensors.find(id);
  if (it == tensors.end()) fail("no tensor '" + id + "'");
  return it->second;
}

const OpSpec& Plan::op(const std::string& id) const {
  auto it = op_index.find(id);
  if (it == op_index.end()) fail("no op '" + id + "'");
  return ops[size_t(it->second)];
}

int Plan::node(const std::string& id) const {
  auto it = node_index.find(id);
  if (it == node_index.end()) fail("no plan node with id " + id);
  return it->second;
}

namespace {

NodeKind node_kind(const std::string& s) {
  if (s == "buffer") return NodeKind::buffer;
  if (s == "slice") return NodeKind::slice;
  if (s == "fetch") return NodeKind::fetch;
  if (s == "concat") return NodeKind::concat;
  if (s == "sub_op") return NodeKind::sub_op;
  if (s == "reduce_partial") return NodeKind::reduce_partial;
  fail("unknown node kind '" + s + "'");
}

OpKind op_kind(const std::string& s) {
  if (s == "matmul") return OpKind::matmul;
  if (s == "elementwise") return OpKind::elementwise;
  if (s == "conv") return OpKind::conv;
  if (s == "generic") return OpKind::generic;
  fail("unknown op kind '" + s + "'");
}

EwFn ew_fn(const std::string& s) {
  if (s == "add") return EwFn::add;
  if (s == "sub") return EwFn::sub;
  if (s == "scale") return EwFn::scale;
  if (s == "pointwise_fn") return EwFn::pointwise_fn;
  if (s == "pointwise_fn_grad") return EwFn::pointwise_fn_grad;
  fail("unknown elementwise function '" + s + "'");
}

ConvMode conv_mode(const std::string& s) {
  if (s == "forward") return ConvMode::forward;
  if (s == "grad_weight") return ConvMode::grad_weight;
  if (s == "grad_input") return ConvMode::grad_input;
  fail("unknown conv mode '" + s + "'");
}

Region region_of(const Json& j) {
  if (j.type != Json::Array) fail("malformed plan document: region must be an array");
  Region r;
  for (const auto& e : j.arr) {
    if (e.type != Json::Array || e.arr.size() != 2)
      fail("malformed plan document: region bounds must be [lo, hi] pairs");
    r.b.push_back({e.arr[0].as_int(), e.arr[1].as_int()});
  }
  return r;
}

}  // namespace

Shape op_output_shape(const OpSpec& op, const std::vector<Shape>& ins) {
  const std::string pre = "op '" + op.id + "': ";
  switch (op.kind) {
    case OpKind::matmul: {
      if (ins.size() != 2) fail(pre + "matmul needs two inputs");
      const Shape& A = ins[0];
      const Shape& B = ins[1];
      if (A.size() != 2 || B.size() != 2) fail(pre + "matmul inputs must be rank 2");
      const int64_t m = op.ta ? A[1] : A[0], kk = op.ta ? A[0] : A[1];
      const int64_t kb = op.tb ? B[1] : B[0], n = op.tb ? B[0] : B[1];
      if (kk != kb) fail(pre + "matmul inner extents differ");
      return {m, n};
    }
    case OpKind::elementwise: {
      if (ins.empty()) fail(pre + "elementwise needs at least one input");
      for (const auto& s : ins)
        if (s != ins[0]) fail(pre + "elementwise operands must share a shape");
      const size_t want = (op.fn == EwFn::add || op.fn == EwFn::sub) ? 2 : 1;
      if (ins.size() != want) {
        static const char* names[] = {"add", "sub", "scale", "pointwise_fn", "pointwise_fn_grad"};
        fail(pre + names[int(op.fn)] + (want == 2 ? " needs two inputs" : " needs one input"));
      }
      return ins[0];
    }
    case OpKind::conv: {
      if (ins.size() != 2) fail(pre + "conv needs two inputs");
      const Shape& A = ins[0];
      const Shape& B = ins[1];
      if (A.size() != 4 || B.size() != 4) fail(pre + "conv operands must be rank 4");
      switch (op.mode) {
        case ConvMode::forward:
          if (B[1] != A[1]) fail(pre + "conv channel extents differ");
          return {A[0], B[0], A[2] - B[2] + 1, A[3] - B[3] + 1};
        case ConvMode::grad_weight:
          if (B[0] != A[0]) fail(pre + "conv batch extents differ");
          return {B[1], A[1], A[2] - B[2] + 1, A[3] - B[3] + 1};
        case ConvMode::grad_input:
          if (B[0] != A[1]) fail(pre + "conv channel extents differ");
          return {A[0], B[1], A[2] + B[2] - 1, A[3] + B[3] - 1};
      }
      fail(pre + "bad conv mode");
    }
    case OpKind::generic:
      fail(pre + "unbound function tag (generic ops have no numeric binding)");
  }
  fail("bad op kind");
}

Plan parse_plan(const std::string& json_text) {
  Json j = Json::parse(json_text);
  Plan p;
  p.k = int(j.at("k").as_int());
  if (p.k < 0 || p.k > 20) fail("malformed plan document: bad cut count");
  p.devices = 1 << p.k;
  if (const Json* d = j.find("devices"))
    if (d->as_int() != p.devices) fail("malformed plan document: devices != 2^k");

  const Json& g = j.at("graph");
  for (const auto& tj : g.at("tensors").arr) {
    TensorSpec t;
    t.id = tj.at("id").as_string();
    for (const auto& e : tj.at("shape").arr) t.shape.push_back(e.as_int());
    t.dtype_bytes = tj.has("dtype_bytes") ? int(tj.at("dtype_bytes").as_int()) : 4;
    t.role = tj.has("role") ? tj.at("role").as_string() : "temp";
    if (!p.tensors.emplace(t.id, t).second) fail("duplicate tensor id '" + t.id + "'");
  }
  for (const auto& oj : g.at("ops").arr) {
    OpSpec o;
    o.id = oj.at("id").as_string();
    o.kind = op_kind(oj.at("kind").as_string());
    for (const auto& e : oj.at("inputs").arr) o.inputs.push_back(e.as_string());
    o.output = oj.at("output").as_string();
    static const Json empty_obj = [] {
      Json e;
      e.type = Json::Object;
      return e;
    }();
    const Json& a = oj.has("attrs") ? oj.at("attrs") : empty_obj;
    switch (o.kind) {
      case OpKind::matmul:
        o.ta = a.has("transpose_a") && a.at("transpose_a").as_bool();
        o.tb = a.has("transpose_b") && a.at("transpose_b").as_bool();
        break;
      case OpKind::elementwise:
        o.fn = ew_fn(a.at("function").as_string());
        o.scale = a.has("scale") ? a.at("scale").as_double() : 0.0;
        break;
      case OpKind::conv:
        o.mode = conv_mode(a.at("mode").as_string());
        for (int i = 0; i < 2; ++i) {
          o.row_dims[i] = int(a.at("row_dims").arr.at(size_t(i)).as_int());
          o.col_dims[i] = int(a.at("col_dims").arr.at(size_t(i)).as_int());
          o.inner_dims[i] = int(a.at("inner_dims").arr.at(size_t(i)).as_int());
        }
        break;
      case OpKind::generic:
        o.batch_dim = a.has("batch_dim") ? int(a.at("batch_dim").as_int()) : 0;
        break;
    }
    for (const auto& in : o.inputs)
      if (!p.tensors.count(in)) fail("op '" + o.id + "' reads undeclared tensor '" + in + "'");
    if (!p.tensors.count(o.output))
      fail("op '" + o.id + "' writes undeclared tensor '" + o.output + "'");
    if (p.op_index.count(o.id)) fail("duplicate op id '" + o.id + "'");
    p.op_index[o.id] = int(p.ops.size());
    p.ops.push_back(std::move(o));
  }
  if (const Json* aj = j.find("assignment"))
    for (const auto& kv : aj->obj) p.assignment[kv.first] = kv.second.as_string();

  std::set<std::string> seen_phase;
  for (const auto& e : j.at("nodes").arr) {
    PlanNode n;
    n.id = e.at("id").as_string();
    n.kind = node_kind(e.at("kind").as_string());
    n.device = int(e.at("device").as_int());
    if (const Json* t = e.find("tensor")) n.tensor = t->as_string();
    if (const Json* o = e.find("op")) n.op = o->as_string();
    n.phase = e.at("phase").as_string();
    n.region = region_of(e.at("region"));
    if (const Json* pa = e.find("partial")) n.partial = int(pa->as_int());
    if (const Json* b = e.find("bytes")) n.bytes = b->as_int();
    if (const Json* sd = e.find("src_device")) n.src_device = int(sd->as_int());
    if (const Json* s = e.find("sources")) {
      for (const auto& sid : s->arr) {
        auto it = p.node_index.find(sid.as_string());
        if (it == p.node_index.end())
          fail("node " + n.id + " reads node " + sid.as_string() + " before it is produced");
        n.sources.push_back(it->second);
      }
    }
    if (p.node_index.count(n.id)) fail("duplicate plan node id " + n.id);
    if (n.device < 0 || n.device >= p.devices)
      fail("node " + n.id + " is placed on device " + std::to_string(n.device) +
           " outside the plan's " + std::to_string(p.devices) + " devices");
    const TensorSpec& t = p.tensor(n.tensor);
    if (n.region.rank() != int(t.shape.size()))
      fail("node " + n.id + " region rank does not match tensor " + t.id);
    for (int d = 0; d < n.region.rank(); ++d)
      if (n.region.b[size_t(d)][0] < 0 || n.region.b[size_t(d)][1] > t.shape[size_t(d)] ||
          n.region.b[size_t(d)][1] <= n.region.b[size_t(d)][0])
        fail("node " + n.id + " region " + n.region.str() + " escapes tensor " + t.id);

    switch (n.kind) {
      case NodeKind::buffer:
        break;
      case NodeKind::slice:
      case NodeKind::fetch: {
        if (n.sources.size() != 1) fail("node " + n.id + " needs exactly one source");
        const PlanNode& src = p.nodes[size_t(n.sources[0])];
        if (!src.region.contains(n.region)) fail("slice region escapes source region");
        if (n.kind == NodeKind::fetch) {
          if (n.src_device == n.device) fail("fetch node " + n.id + " is not cross-device");
          if (src.device != n.src_device)
            fail("fetch node " + n.id + " names src_device " + std::to_string(n.src_device) +
                 " but its source lives on device " + std::to_string(src.device));
          const int64_t want = n.region.volume() * t.dtype_bytes;
          if (n.bytes != want)
            fail("fetch node " + n.id + " carries " + std::to_string(n.bytes) +
                 " bytes, its region is " + std::to_string(want));
          p.fetch_bytes_total += n.bytes;
        } else if (src.device != n.device) {
          fail("slice node " + n.id + " reads a block on another device");
        }
        break;
      }
      case NodeKind::concat: {
        int64_t pasted = 0;
        for (int s : n.sources) {
          const PlanNode& piece = p.nodes[size_t(s)];
          if (piece.device != n.device) fail("concat node " + n.id + " pastes a remote block");
          if (!n.region.contains(piece.region)) fail("piece region escapes destination region");
          pasted += piece.region.volume();
        }
        if (pasted != n.region.volume())
          fail("concat node " + n.id + " pieces do not tile its region");
        for (size_t a = 0; a < n.sources.size(); ++a)
          for (size_t b = a + 1; b < n.sources.size(); ++b)
            if (p.nodes[size_t(n.sources[a])].region.intersect(p.nodes[size_t(n.sources[b])].region).volume())
              fail("concat node " + n.id + " pieces overlap");
        break;
      }
      case NodeKind::reduce_partial:
        for (int s : n.sources) {
          const PlanNode& piece = p.nodes[size_t(s)];
          if (piece.region != n.region) fail("reduce node " + n.id + " sums mismatched regions");
          if (piece.device != n.device) fail("reduce node " + n.id + " sums a remote block");
        }
        break;
      case NodeKind::sub_op: {
        const OpSpec& op = p.op(n.op);
        if (op.output != n.tensor) fail("sub-op node " + n.id + " does not produce " + op.id + "'s output");
        if (n.sources.size() != op.inputs.size())
          fail("sub-op node " + n.id + " has " + std::to_string(n.sources.size()) + " operands, op '" +
               op.id + "' takes " + std::to_string(op.inputs.size()));
        std::vector<Shape> in_shapes;
        for (size_t i = 0; i < n.sources.size(); ++i) {
          const PlanNode& s = p.nodes[size_t(n.sources[i])];
          if (s.device != n.device) fail("sub-op node " + n.id + " reads a remote block");
          if (s.tensor != op.inputs[i])
            fail("sub-op node " + n.id + " operand " + std::to_string(i) + " is not tensor " + op.inputs[i]);
          in_shapes.push_back(s.region.shape());
        }
        if (op_output_shape(op, in_shapes) != n.region.shape())
          fail("sub-op node " + n.id + " produced a mismatched block");
        break;
      }
    }
    if (seen_phase.insert(n.phase).second) p.phase_order.push_back(n.phase);
    p.node_index[n.id] = int(p.nodes.size());
    p.nodes.push_back(std::move(n));
  }
  for (const auto& kv : j.at("holders").obj) {
    const TensorSpec& t = p.tensor(kv.first);
    std::vector<int> hs;
    for (size_t d = 0; d < kv.second.arr.size(); ++d) {
      const std::string& hid = kv.second.arr[d].as_string();
      if (hid.empty()) fail("tensor " + t.id + " has no holder on some device");
      const int idx = p.node(hid);
      if (p.nodes[size_t(idx)].device != int(d))
        fail("holder " + hid + " of tensor " + t.id + " is not on device " + std::to_string(d));
      if (p.nodes[size_t(idx)].tensor != t.id)
        fail("holder " + hid + " does not carry tensor " + t.id);
      hs.push_back(idx);
    }
    if (int(hs.size()) != p.devices) fail("tensor " + t.id + " has no holder on some device");
    p.holders[kv.first] = std::move(hs);
  }
  if (const Json* fb = j.find("fetch_bytes_total"))
    if (fb->as_int() != p.fetch_bytes_total)
      fail("plan fetch_bytes_total " + std::to_string(fb->as_int()) +
           " disagrees with its fetch nodes (" + std::to_string(p.fetch_bytes_total) + ")");
  return p;
}

}  // namespace tpx
