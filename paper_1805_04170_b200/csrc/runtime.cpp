#include "runtime.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>
#include <sstream>
#include <tuple>

#include <nvtx3/nvToolsExt.h>

#include "json.h"
#include "nccl_shim.h"
#include "util.h"

namespace tpx {

namespace {

constexpr size_t kAlign = 256;

// Storage element size of the plan being lowered / read / written (4 = fp32, 2 = bf16).  Set by
// the entry points from PlanRt::esize; one host thread drives a plan at a time.
thread_local int g_es = 4;
inline float* eoff(float* p, int64_t elems) {
  return reinterpret_cast<float*>(reinterpret_cast<char*>(p) + elems * g_es);
}
inline NaryDesc ndesc(int op, const StridedView& out, const std::vector<StridedView>& ins, float scale = 0.f) {
  return nary_desc(op, out, ins, scale, g_es);
}
constexpr uintptr_t kFakeBase = uintptr_t(1) << 40;  // dry-run arena base (256-aligned)

StridedView contiguous_view(float* ptr, const Shape& s) {
  StridedView v;
  v.ptr = ptr;
  v.rank = int(s.size());
  int64_t st = 1;
  for (int i = v.rank - 1; i >= 0; --i) {
    v.shape[i] = s[size_t(i)];
    v.st[i] = st;
    st *= s[size_t(i)];
  }
  return v;
}

// Sub-box `sub` of a value covering `vreg`.
StridedView subview(const StridedView& v, const Region& vreg, const Region& sub) {
  if (!vreg.contains(sub)) fail("slice region escapes source region");
  StridedView o = v;
  int64_t off = 0;
  for (int i = 0; i < v.rank; ++i) {
    off += (sub.b[size_t(i)][0] - vreg.b[size_t(i)][0]) * v.st[i];
    o.shape[i] = sub.b[size_t(i)][1] - sub.b[size_t(i)][0];
  }
  o.ptr = eoff(v.ptr, off);
  return o;
}

MatView mat_view(const StridedView& v) {
  if (v.rank != 2) fail("matmul operand is not rank 2");
  MatView m;
  m.ptr = v.ptr;
  m.rows = v.shape[0];
  m.cols = v.shape[1];
  m.rs = v.st[0];
  m.cs = v.st[1];
  if (m.cols == 1) m.cs = 1;  // a single column is unit-stride by definition
  return m;
}

// Classes of an open segment, flushed in this order (each may read values produced by an
// earlier class of the same segment, never by its own or a later class).
enum Cls { C_PRE = 0, C_COMPUTE = 1, C_POST = 2, C_PACK = 3, C_XCHG = 4, C_COPY = 5, C_REDUCE = 6, C_N = 7 };

struct Lowerer {
  PlanRt& P;
  Plan& pl;
  Ctx& C;
  Program& prog;
  bool dry;
  bool fuse, force_xchg;

  std::vector<int> consumers;
  std::vector<int> defer_to;   // concat node index a fetch/slice is pasted into, or -1
  std::vector<char> is_holder;
  std::vector<int> pending;    // open class producing the node, or -1
  // node -> (gemm batch, [(problem, element offset of the problem's output in the node)]):
  // the launch an elementwise consumer of the node can be fused into
  struct Tail {
    int batch;
    std::vector<std::pair<int, int64_t>> probs;
    bool like = false;  // fused outputs take the source's (strided) layout
  };
  std::map<int, Tail> chain_tail;
  // grad_input node -> its col2im descriptor (open batch: desc index; emitted: conv batch, desc,
  // step), where a 1 - tanh^2 consumer is fused
  std::map<int, int> post_open;
  struct PostTail {
    int batch, desc, step;
  };
  std::map<int, PostTail> post_tail;
  std::vector<int> gemm_step;  // gemm batch -> step index (-1 while open)

  // fetch node -> the reduce_partial that reads its source region in place (no copy of its own)
  std::vector<int> red_src;
  struct Direct {
    StridedView view;  // the piece's region of its source value (on its owner's arena)
    int src = -1;      // source node (local readiness)
    int rank = -1;     // owning rank when read from a peer (waits on its sync counter), else -1
  };
  std::map<int, Direct> direct;
  // reduce_partial (or a fused consumer of one) -> the descriptor its elementwise consumers chain
  // onto: (nary batch, descriptor, step, the reduction's output view)
  struct RedTail {
    int batch, desc, step;
    StridedView out;
  };
  std::map<int, RedTail> red_tail;
  std::vector<int> open_red;   // reductions in the open reduce batch (tail candidates)

  // open segment
  NaryBatch o_pre, o_ew, o_pack, o_copy, o_reduce, o_pull;
  ConvBatch o_prec, o_post;    // im2col before / col2im after a conv's GEMM
  XchgGroup o_xchg;
  int o_gemm = -1;             // open gemm batch index
  ConvBatch o_conv;
  int o_kind = -1;             // 0 gemm, 1 ew, 2 conv
  std::string o_op, o_pre_op;
  std::vector<int> o_nodes[C_N];
  std::string seg_op;          // op owning the conversion classes (phase prefix)

  Lowerer(PlanRt& p, Program& pr, bool d)
      : P(p), pl(p.plan), C(*p.ctx), prog(pr), dry(d),
        fuse(p.flags & 1), force_xchg(p.flags & 2), tc_conv(!(p.flags & 4)),
        transposed_operands((p.flags & 64) != 0) {}
  bool tc_conv;
  // conv grad_input on K-major transposed operands (TPX_FLAG_KMAJOR_CONV = 64, opt-in: measured
  // +/- 1 % on the AlexNet-style step, -2.5 % on the VGG-style one: the transposes cost what the
  // faster GEMM saves)
  bool transposed_operands;
  std::map<std::vector<int64_t>, float*> col_cache;  // im2col buffers by (view, filter) key
  std::map<std::vector<int64_t>, float*> gp_cache;   // permuted conv gradients by (view, pitch)

  float* alloc_bytes(size_t bytes) {
    const size_t off = (P.arena_used + kAlign - 1) / kAlign * kAlign;
    P.arena_used = off + std::max<size_t>(bytes, 4);
    if (!dry && P.arena_used > P.arena_bytes) fail("arena overflow (lowering is not deterministic)");
    return reinterpret_cast<float*>(P.base + off);
  }
  StridedView alloc(const Shape& s) {
    int64_t n = 1;
    for (auto e : s) n *= e;
    return contiguous_view(alloc_bytes(size_t(n) * size_t(g_es)), s);
  }
  // Fresh storage with v's shape and strides (padding inside the extent stays 0).
  StridedView alloc_like(const StridedView& v) {
    int64_t ext = 1;
    for (int i = 0; i < v.rank; ++i) ext += (v.shape[i] - 1) * v.st[i];
    StridedView t = v;
    t.ptr = alloc_bytes(size_t(ext) * size_t(g_es));
    return t;
  }
  // Channel-major conv layout [n, c, y, x] -> element c*ld + n*img + y*X + x: every channel's
  // images side by side in one row of ld = pitch4(N * img) elements, img = pitch4(Y * X).  The
  // tensor-core conv lowering keeps activations and gradients in this layout: it is the GEMMs'
  // column layout, so no permute runs between the convolutions.
  StridedView conv_layout(int64_t N, int64_t C, int64_t Y, int64_t X) {
    const int64_t img = pitch4(Y * X), ld = pitch4(N * img);
    StridedView v;
    v.rank = 4;
    v.shape[0] = N; v.shape[1] = C; v.shape[2] = Y; v.shape[3] = X;
    v.st[0] = img; v.st[1] = ld; v.st[2] = X; v.st[3] = 1;
    v.ptr = alloc_bytes(size_t(C * ld) * size_t(g_es));
    return v;
  }
  static bool is_conv_layout(const StridedView& v) {
    if (v.rank != 4) return false;
    const int64_t img = pitch4(v.shape[2] * v.shape[3]), ld = pitch4(v.shape[0] * img);
    return (v.shape[0] == 1 || v.st[0] == img) && (v.shape[1] == 1 || v.st[1] == ld) &&
           (v.shape[2] == 1 || v.st[2] == v.shape[3]) && v.st[3] == 1 &&
           (reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0;
  }

  // Value of `node` on rank `r` as this rank addresses it: its own value, or (peer mode) the view
  // a host-only lowering of the plan as rank r gave it, moved onto r's mapped arena.
  StridedView src_view(int r, int node) {
    if (r == C.rank) return value(node);
    const PlanNode& n = pl.nodes[size_t(node)];
    if (dry) return contiguous_view(reinterpret_cast<float*>(kFakeBase), n.region.shape());
    if (size_t(r) >= P.rhas.size() || !P.rhas[size_t(r)][size_t(node)])
      fail("node " + n.id + " has no value on rank " + std::to_string(r));
    StridedView v = (swap_to ? P.rval_b : P.rval)[size_t(r)][size_t(node)];
    v.ptr = reinterpret_cast<float*>(P.peer_base[size_t(r)] + (reinterpret_cast<uintptr_t>(v.ptr) - kFakeBase));
    return v;
  }
  // Peer-mode sync points: a phase's signal is published by its first conversion launch on this
  // rank (or a one-thread launch when the rank has none); its pulls wait for the peers' value of
  // the same point.  Barriers are their own launch.
  int sync_idx = 0;            // next sync point index of this program
  int pending_signal = -1;     // sync point not yet attached to a launch
  int phase_sync = -1;         // sync point of the open phase (pull wait target; -1: last barrier)
  void sync_step(bool barrier) {
    flush();
    if (!barrier) {
      pending_signal = phase_sync = sync_idx++;
      return;
    }
    const int s = add_step(ST_SYNC, -1, std::string(), "barrier");
    prog.steps[size_t(s)].barrier = 1;
  }

  int rank_of(int dev) const { return P.dev_rank[size_t(dev)]; }
  bool mine_dev(int dev) const { return rank_of(dev) == C.rank; }

  int add_step(StepKind k, int idx, const std::string& op, const std::string& what) {
    prog.steps.push_back(Step{k, idx, op, what});
    return int(prog.steps.size()) - 1;
  }

  void produced(int node, Cls c) {
    pending[size_t(node)] = c;
    o_nodes[c].push_back(node);
  }

  void flush() {
    auto emit_nary = [&](NaryBatch& b, const std::string& op, const std::string& what, Cls c) {
      if (b.descs.empty()) return;
      if (c >= C_PACK && pending_signal >= 0) {  // the phase's first conversion launch publishes it
        b.signal_s = pending_signal;
        pending_signal = -1;
      }
      if (b.pull) b.wait_s = phase_sync;
      prog.nary.push_back(std::move(b));
      b = NaryBatch{};
      const int s = add_step(ST_NARY, int(prog.nary.size()) - 1, op, what);
      for (int n : o_nodes[c]) P.avail_step[size_t(n)] = s;
    };
    emit_nary(o_pre, o_pre_op, "materialize", C_PRE);
    auto emit_conv = [&](ConvBatch& b, const std::string& op, const std::string& what, Cls c) {
      if (b.descs.empty()) return;
      prog.conv.push_back(std::move(b));
      b = ConvBatch{};
      const int s = add_step(ST_CONV, int(prog.conv.size()) - 1, op, what);
      for (int n : o_nodes[c]) P.avail_step[size_t(n)] = s;
    };
    emit_conv(o_prec, o_pre_op, "im2col", C_PRE);
    if (o_kind == 0) {
      const int s = add_step(ST_GEMM, o_gemm, o_op, "gemm");
      gemm_step[size_t(o_gemm)] = s;
      for (int n : o_nodes[C_COMPUTE]) P.avail_step[size_t(n)] = s;
    } else if (o_kind == 1) {
      emit_nary(o_ew, o_op, "elementwise", C_COMPUTE);
    } else if (o_kind == 2) {
      prog.conv.push_back(std::move(o_conv));
      o_conv = ConvBatch{};
      const int s = add_step(ST_CONV, int(prog.conv.size()) - 1, o_op, "conv");
      for (int n : o_nodes[C_COMPUTE]) P.avail_step[size_t(n)] = s;
    }
    const int n_post = int(o_post.descs.size());
    emit_conv(o_post, o_op, "col2im", C_POST);
    if (n_post) {
      for (const auto& kv : post_open)
        post_tail[kv.first] = PostTail{int(prog.conv.size()) - 1, kv.second, int(prog.steps.size()) - 1};
    }
    post_open.clear();
    emit_nary(o_pack, seg_op, "pack", C_PACK);
    for (const auto& d : o_pull.descs) o_pull.pull = o_pull.pull || d.wait_mask != 0;  // (local copies share it)
    emit_nary(o_pull, seg_op, "pull", C_XCHG);
    if (!o_xchg.x.empty()) {
      prog.xchg.push_back(std::move(o_xchg));
      o_xchg = XchgGroup{};
      const int s = add_step(ST_XCHG, int(prog.xchg.size()) - 1, seg_op, "nccl");
      for (int n : o_nodes[C_XCHG]) P.avail_step[size_t(n)] = s;
    }
    emit_nary(o_copy, seg_op, "copy", C_COPY);
    const bool had_reduce = !o_reduce.descs.empty();
    emit_nary(o_reduce, seg_op, "reduce", C_REDUCE);
    if (pending_signal >= 0) {  // no conversion launch on this rank at this sync point
      const int s = add_step(ST_SYNC, pending_signal, seg_op, "signal");
      prog.steps[size_t(s)].barrier = 0;
      pending_signal = -1;
    }
    if (had_reduce) {
      for (int r : open_red) {
        RedTail& t = red_tail[r];
        t.batch = int(prog.nary.size()) - 1;
        t.step = int(prog.steps.size()) - 1;
      }
    }
    open_red.clear();
    for (int c = 0; c < C_N; ++c) {
      for (int n : o_nodes[c]) pending[size_t(n)] = -1;
      o_nodes[c].clear();
    }
    o_kind = -1;
    o_gemm = -1;
    o_op.clear();
  }

  // Flush when `node`'s value is still being produced by an open class >= c.
  void need(int node, Cls c) {
    const int pc = pending[size_t(node)];
    if (pc >= 0 && pc >= int(c)) flush();
  }

  const StridedView& value(int node) {
    if (!P.has_val[size_t(node)])
      fail("node " + pl.nodes[size_t(node)].id + " has no materialised value on this rank");
    return P.val[size_t(node)];
  }

  // Loop mode, second program: weight buffers and their w_next holders trade storage
  // (node -> the partner's value in the first program); the fresh allocation is kept unused so
  // every other node lands at the same arena offset in both programs.
  const std::map<int, StridedView>* swap_to = nullptr;
  const StridedView& set_val(int node, const StridedView& v) {
    auto it = swap_to ? swap_to->find(node) : std::map<int, StridedView>::const_iterator{};
    P.val[size_t(node)] = (swap_to && it != swap_to->end()) ? it->second : v;
    P.has_val[size_t(node)] = 1;
    return P.val[size_t(node)];
  }

  void ensure_alloc(int node) {
    if (!P.has_val[size_t(node)]) set_val(node, alloc(pl.nodes[size_t(node)].region.shape()));
  }

  static std::string op_of_phase(const std::string& phase) {
    const auto p = phase.rfind(':');
    return p == std::string::npos ? phase : phase.substr(0, p);
  }

  // ------------------------------------------------------------ sub_op lowering
  void lower_sub_op(int ni) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    const OpSpec& op = pl.op(n.op);
    for (int s : n.sources) need(s, C_COMPUTE);
    if (op.kind == OpKind::generic)
      fail("op '" + op.id + "': unbound function tag (generic ops have no numeric binding)");

    if (op.kind == OpKind::elementwise && fuse && (try_fuse_reduce(ni, op) || try_fuse(ni, op))) return;

    if (op.kind == OpKind::conv && tc_conv) {
      lower_conv_gemm(ni, op);
      return;
    }
    const int kind = op.kind == OpKind::matmul ? 0 : op.kind == OpKind::elementwise ? 1 : 2;
    if (o_kind >= 0 && (o_kind != kind || o_op != op.id)) flush();
    if (o_kind < 0) {
      o_kind = kind;
      o_op = op.id;
      if (kind == 0) {
        prog.gemm_specs.emplace_back();
        gemm_step.push_back(-1);
        o_gemm = int(prog.gemm_specs.size()) - 1;
      }
    }
    const StridedView out = set_val(ni, alloc(n.region.shape()));
    if (op.kind == OpKind::matmul) {
      GemmSpec s;
      StridedView a = value(n.sources[0]);
      StridedView b = value(n.sources[1]);
      s.a = mat_view(a);
      s.b = mat_view(b);
      if (!gemm_view_ok(s.a, g_es == 2)) s.a = mat_view(materialize(n.sources[0], op.id));
      if (!gemm_view_ok(s.b, g_es == 2)) s.b = mat_view(materialize(n.sources[1], op.id));
      s.ta = op.ta;
      s.tb = op.tb;
      s.c = out.ptr;
      s.c_rs = out.st[0];
      s.c_cs = 1;
      auto& specs = prog.gemm_specs[size_t(o_gemm)];
      specs.push_back(s);
      chain_tail[ni] = Tail{o_gemm, {{int(specs.size()) - 1, 0}}};
      const double M = double(op.ta ? s.a.cols : s.a.rows), K = double(op.ta ? s.a.rows : s.a.cols);
      const double N = double(op.tb ? s.b.rows : s.b.cols);
      P.gemm_flops += 2.0 * M * N * K;
      P.gemm_min_bytes += double(g_es) * (M * K + K * N + M * N);
    } else if (op.kind == OpKind::elementwise) {
      std::vector<StridedView> ins;
      for (int s : n.sources) ins.push_back(value(s));
      int code = NARY_COPY;
      switch (op.fn) {
        case EwFn::add: code = NARY_SUM; break;
        case EwFn::sub: code = NARY_SUB; break;
        case EwFn::scale: code = NARY_SCALE; break;
        case EwFn::pointwise_fn: code = NARY_TANH; break;
        case EwFn::pointwise_fn_grad: code = NARY_DTANH; break;
      }
      o_ew.descs.push_back(ndesc(code, out, ins, float(op.scale)));
    } else {
      ConvDesc d;
      std::memset(&d, 0, sizeof d);
      d.mode = op.mode == ConvMode::forward ? CONV_FWD : op.mode == ConvMode::grad_weight ? CONV_GRAD_W : CONV_GRAD_IN;
      d.a = value(n.sources[0]);
      d.b = value(n.sources[1]);
      d.out = out.ptr;
      for (int i = 0; i < 4; ++i) d.oshape[i] = out.shape[i];
      d.n = out.elements();
      o_conv.descs.push_back(d);
      const OpSpec& o = op;
      (void)o;
      double contr = 0;
      if (d.mode == CONV_FWD) contr = double(d.b.shape[1] * d.b.shape[2] * d.b.shape[3]) * double(d.n);
      else if (d.mode == CONV_GRAD_W) contr = double(d.a.shape[0] * d.b.shape[2] * d.b.shape[3]) * double(d.n);
      else contr = double(d.a.elements()) * double(d.b.shape[1] * d.b.shape[2] * d.b.shape[3]);
      o_conv.flops += 2.0 * contr;
    }
    produced(ni, C_COMPUTE);
  }

  // 2-D view of a rank-4 filter K[o, c, u, v] as [o, c*u*v] when (c, u, v) is contiguous and
  // the rows are TMA-addressable.
  static bool filter_mat(const StridedView& k, MatView& m) {
    if (k.rank != 4 || k.st[3] != 1 || k.st[2] != k.shape[3] || k.st[1] != k.shape[2] * k.shape[3]) return false;
    m.ptr = k.ptr;
    m.rows = k.shape[0];
    m.cols = k.shape[1] * k.shape[2] * k.shape[3];
    m.rs = k.st[0];
    m.cs = 1;
    return gemm_view_ok(m, g_es == 2);
  }
  // 16-byte rows (TMA): 4 fp32 or 8 bf16 elements
  static int64_t pitch4(int64_t n) { const int64_t a = 16 / g_es; return (n + a - 1) / a * a; }

  // Copy of a rank-4 view into fresh storage whose last `merge` dims form dense rows padded to
  // 16 bytes: returns the copy with the original shape (pre class, before the op's compute).
  StridedView padded_copy(const StridedView& v, int merge, const std::string& op) {
    if (!o_pre.descs.empty() && o_pre_op != op) flush();
    o_pre_op = op;
    int64_t inner = 1;
    for (int i = 4 - merge; i < 4; ++i) inner *= v.shape[i];
    const int64_t rows = v.elements() / std::max<int64_t>(inner, 1), ld = pitch4(inner);
    StridedView t = v;
    t.ptr = alloc_bytes(size_t(rows * ld) * size_t(g_es));
    int64_t st = 1;
    for (int i = 3; i >= 0; --i) {
      t.st[i] = st;
      st *= v.shape[i];
      if (i == 4 - merge) st = ld;
    }
    o_pre.descs.push_back(ndesc(NARY_COPY, t, {v}));
    return t;
  }

  // Convolution sub-op on the tensor cores (run_conv, proj/src/dense.cpp:92-157):
  //   forward      out[n,o,:,:]  = Kmat[o, cuv] . im2col(a)[n][yx, cuv]^T    per image
  //   grad_weight  gk[o, cuv]    = Gp[o, (n,yx)] . im2col(a)[cuv, (n,yx)]^T  one GEMM
  //   grad_input   dcol[cuv, (n,yx)] = Kmat^T . Gp, then col2im (ordered tap sum)
  // The im2col / permute copies run in the pre class, col2im in the post class.  Every scratch
  // matrix has 16-byte rows (TMA); padding columns lie outside the tensor maps.
  void lower_conv_gemm(int ni, const OpSpec& op) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    for (int s : n.sources) need(s, C_COMPUTE);
    if (o_kind >= 0 && (o_kind != 0 || o_op != op.id)) flush();
    if (!o_pre.descs.empty() && o_pre_op != op.id) flush();
    if (o_kind < 0) {
      o_kind = 0;
      o_op = op.id;
      prog.gemm_specs.emplace_back();
      gemm_step.push_back(-1);
      o_gemm = int(prog.gemm_specs.size()) - 1;
    }
    o_pre_op = op.id;
    const Shape osh = n.region.shape();
    if (osh.size() != 4) fail("op '" + op.id + "': conv output must be rank 4");
    const StridedView a = value(n.sources[0]);
    const StridedView b = value(n.sources[1]);
    // forward / grad_input outputs in the channel-major conv layout, grad_weight dense
    StridedView out;
    if (op.mode == ConvMode::forward) {
      out = conv_layout(osh[0], osh[1], osh[2], osh[3]);
    } else if (op.mode == ConvMode::grad_weight) {
      out = alloc(osh);
    } else {
      out = conv_layout(osh[0], osh[1], osh[2], osh[3]);
    }
    out = set_val(ni, out);
    if (a.rank != 4 || b.rank != 4) fail("op '" + op.id + "': conv operands must be rank 4");
    // im2col in the columns layout col[(c,u,v)][(n,y,x)], rows padded to 16 bytes
    // img = per-image column stride: Yo*Xo (dense, one GEMM over all images) or padded to 16
    // bytes so that every image's column block can be a TMA operand of its own problem
    auto im2col = [&](const StridedView& act, int64_t U, int64_t V, int64_t Yo, int64_t Xo, int64_t img,
                      int64_t& pitch) {
      const int64_t NB = act.shape[0], K = act.shape[1] * U * V;
      pitch = pitch4(NB * img);
      // forward and grad_weight of a layer read the same activation view: one im2col
      std::vector<int64_t> key = {int64_t(reinterpret_cast<uintptr_t>(act.ptr)), U, V, img};
      for (int i = 0; i < act.rank; ++i) {
        key.push_back(act.shape[i]);
        key.push_back(act.st[i]);
      }
      auto hit = col_cache.find(key);
      if (hit != col_cache.end()) return hit->second;
      float* t = alloc_bytes(size_t(K * pitch) * size_t(g_es));  // padding columns stay 0 (zeroed arena)
      col_cache[key] = t;
      ConvDesc d;
      std::memset(&d, 0, sizeof d);
      d.mode = CONV_IM2COL;
      d.a = act;
      d.out = t;
      d.n = K * NB * Yo;  // rows
      d.p[0] = U; d.p[1] = V; d.p[2] = Yo; d.p[3] = Xo; d.p[4] = pitch; d.p[5] = img;
      o_prec.descs.push_back(d);
      return t;
    };
    auto filter = [&](const StridedView& k) {
      MatView m;
      if (filter_mat(k, m)) return m;
      const StridedView c = padded_copy(k, 3, op.id);
      m.ptr = c.ptr;
      m.rows = c.shape[0];
      m.cols = c.shape[1] * c.shape[2] * c.shape[3];
      m.rs = c.st[0];
      m.cs = 1;
      return m;
    };
    auto& specs = prog.gemm_specs[size_t(o_gemm)];
    double flops = 0;
    bool post = false;  // the value is finished by the post class (col2im)
    if (op.mode == ConvMode::forward) {
      // Z[o, (n, yx)] = Kmat[o, cuv] . col[cuv, (n, yx)]: one GEMM over every image's (padded)
      // columns, written straight into the conv layout (padding columns: col's are 0, so Z's are)
      const int64_t NB = a.shape[0], C = a.shape[1], O = b.shape[0], U = b.shape[2], V = b.shape[3];
      const int64_t Yo = out.shape[2], Xo = out.shape[3], K = C * U * V, YX = Yo * Xo;
      int64_t ld = 0;
      const int64_t img = pitch4(YX);
      float* col = im2col(a, U, V, Yo, Xo, img, ld);
      if (ld != out.st[1]) fail("op '" + op.id + "': conv layout pitch mismatch");
      GemmSpec s;
      s.a = filter(b);
      s.b = MatView{col, K, NB * img, ld, 1};  // [K x (n, yx)] row-major (MN-major operand)
      s.c = out.ptr;
      s.c_rs = ld;
      specs.push_back(s);
      Tail tail{o_gemm, {{int(specs.size()) - 1, 0}}, true};
      if (fuse) chain_tail[ni] = tail;  // act(z) runs in the GEMM's epilogue
      flops = 2.0 * double(NB) * double(O) * double(YX) * double(K);
    } else if (op.mode == ConvMode::grad_weight) {
      // gk[o, cuv] = Gp[o, (n,yx)] . col[cuv, (n,yx)]^T
      const int64_t NB = a.shape[0], C = a.shape[1], O = b.shape[1], Yo = b.shape[2], Xo = b.shape[3];
      const int64_t U = out.shape[2], V = out.shape[3], K = C * U * V, YX = Yo * Xo;
      int64_t ld = 0;
      const int64_t img = pitch4(YX);
      float* col = im2col(a, U, V, Yo, Xo, img, ld);  // shared with the layer's forward
      float* gp = permuted_grad(b, img, ld, op.id);
      GemmSpec s;  // contraction over all images' (padded) columns; pads are 0 in both operands
      s.a = MatView{gp, O, NB * img, ld, 1};
      s.b = MatView{col, K, NB * img, ld, 1};
      s.tb = true;
      s.c = out.ptr;
      s.c_rs = K;
      specs.push_back(s);
      if (fuse) chain_tail[ni] = Tail{o_gemm, {{int(specs.size()) - 1, 0}}};  // SGD step + update
      flops = 2.0 * double(O) * double(K) * double(NB * YX);
    } else {
      // dcol[cuv, (n, yx)] = Kmat[o, cuv]^T . Gp[o, (n, yx)] (one GEMM), then
      // col2im: h[n,c,y,x] = sum_{u,v} dcol[(c,u,v), n*YX + (y-u)*Xo + (x-v)]
      const int64_t NB = a.shape[0], O = a.shape[1], Yo = a.shape[2], Xo = a.shape[3];
      const int64_t C = b.shape[1], U = b.shape[2], V = b.shape[3], K = C * U * V, YX = Yo * Xo;
      const MatView km = filter(b);
      const int64_t img = pitch4(YX), ld = pitch4(NB * img);
      // the padding columns of Gp are 0, so dcol's are too (col2im never reads them)
      const size_t npre = o_prec.descs.size();
      float* gp = permuted_grad(a, img, ld, op.id);
      // (a Gp permuted in this very launch cannot be transposed by it: stored operands then)
      const bool gp_fresh = o_prec.descs.size() != npre;
      float* dcol = alloc_bytes(size_t(K * ld) * size_t(g_es));
      GemmSpec s;
      if (transposed_operands && !gp_fresh) {
        // both operands K-major (contraction over o contiguous): Kmatᵀ [cuv][o] and Gpᵀ [(n,yx)][o],
        // made by the pre-GEMM transposes (kind::tf32 reads MN-major operands at about half
        // rate; the transposes cost 2 x (filter + gradient) bytes)
        const int64_t op4 = pitch4(O);
        s.a = MatView{transposed(km.ptr, km.rows, km.cols, km.rs, op4, op.id), K, O, op4, 1};
        s.b = MatView{transposed(gp, O, NB * img, ld, op4, op.id), NB * img, O, op4, 1};
        s.tb = true;
      } else {
        s.a = km;  // Kmat [o, cuv], used transposed
        s.ta = true;
        s.b = MatView{gp, O, NB * img, ld, 1};
      }
      s.c = dcol;
      s.c_rs = ld;
      specs.push_back(s);
      ConvDesc d;
      std::memset(&d, 0, sizeof d);
      d.mode = CONV_COL2IM;
      d.a.ptr = dcol;
      d.a.shape[0] = NB;
      d.out = out.ptr;
      d.n = out.elements() / out.shape[3];  // rows (n, c, y)
      d.b.st[0] = out.st[0];  // image / channel strides of out (and of the fused 1 - tanh^2)
      d.b.st[1] = out.st[1];
      d.p[0] = C; d.p[1] = U; d.p[2] = V; d.p[3] = Yo; d.p[4] = Xo; d.p[5] = ld; d.p[6] = img;
      o_post.descs.push_back(d);
      if (fuse) post_open[ni] = int(o_post.descs.size()) - 1;
      flops = 2.0 * double(NB) * double(YX) * double(K) * double(O);
      post = true;
    }
    P.gemm_flops += flops;
    produced(ni, post ? C_POST : C_COMPUTE);
  }

  // G[n, o, y, x] -> Gp[o][(n, img-strided y, x)], rows of `ld` elements (the padding columns
  // stay 0: zeroed arena), shared by a layer's grad_weight and grad_input (pre class).
  float* permuted_grad(const StridedView& g, int64_t img, int64_t ld, const std::string& op) {
    std::vector<int64_t> key = {int64_t(reinterpret_cast<uintptr_t>(g.ptr)), img, ld};
    for (int i = 0; i < g.rank; ++i) {
      key.push_back(g.shape[i]);
      key.push_back(g.st[i]);
    }
    auto hit = gp_cache.find(key);
    if (hit != gp_cache.end()) return hit->second;
    if (is_conv_layout(g) && g.st[1] == ld && (g.shape[0] == 1 || g.st[0] == img)) return g.ptr;  // already Gp
    if (!o_pre.descs.empty() && o_pre_op != op) flush();
    o_pre_op = op;
    const int64_t O = g.shape[1], Yo = g.shape[2], Xo = g.shape[3];
    float* gp = alloc_bytes(size_t(O * ld) * size_t(g_es));
    gp_cache[key] = gp;
    ConvDesc d;  // one (unshifted) copy into the channel-major layout (pre-GEMM movement launch)
    std::memset(&d, 0, sizeof d);
    d.mode = CONV_SHIFTPAD;
    d.a = g;
    d.out = gp;
    d.p[0] = 1; d.p[1] = Yo; d.p[2] = Xo; d.p[3] = Xo; d.p[4] = img; d.p[5] = 0; d.p[6] = ld;
    o_prec.descs.push_back(d);
    return gp;
  }

  // dst[c][r] = src[r][c] (rows x cols, source row stride rs) into fresh storage with `pitch`
  // elements per transposed row (pre class: runs before the op's GEMM), cached per source.
  std::map<std::vector<int64_t>, float*> tr_cache;
  float* transposed(const float* src, int64_t rows, int64_t cols, int64_t rs, int64_t pitch, const std::string& op) {
    const std::vector<int64_t> key = {int64_t(reinterpret_cast<uintptr_t>(src)), rows, cols, rs, pitch};
    auto hit = tr_cache.find(key);
    if (hit != tr_cache.end()) return hit->second;
    if (!o_prec.descs.empty() && o_pre_op != op) flush();
    o_pre_op = op;
    float* dst = alloc_bytes(size_t(cols * pitch) * size_t(g_es));
    ConvDesc d;
    std::memset(&d, 0, sizeof d);
    d.mode = CONV_TRANSPOSE;
    d.a.ptr = const_cast<float*>(src);
    d.a.rank = 2;
    d.a.shape[0] = rows;
    d.a.shape[1] = cols;
    d.a.st[0] = rs;
    d.a.st[1] = 1;
    d.out = dst;
    d.p[0] = pitch;
    d.n = rows * cols;
    o_prec.descs.push_back(d);
    tr_cache[key] = dst;
    return dst;
  }

  StridedView materialize(int node, const std::string& op) {
    // Packed copy of a view the TMA path cannot address (misaligned column slice).
    if (!o_pre.descs.empty() && o_pre_op != op) flush();
    o_pre_op = op;
    // Rows padded to a multiple of 4 floats: TMA needs 16-byte row strides (the padding
    // columns lie outside the tensor map and are never read).
    const StridedView& v = value(node);
    if (v.rank != 2) fail("matmul operand is not rank 2");
    const int64_t rows = v.shape[0], cols = v.shape[1], ld = pitch4(cols);
    StridedView t = alloc({rows, ld});
    t.shape[1] = cols;
    o_pre.descs.push_back(ndesc(NARY_COPY, t, {v}));
    return t;
  }

  bool try_fuse(int ni, const OpSpec& op) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    if (op.fn == EwFn::pointwise_fn_grad && n.sources.size() == 1 && post_tail.count(n.sources[0])) {
      // 1 - tanh^2 of a conv grad_input: written by its col2im from the stored value
      const PostTail pt = post_tail[n.sources[0]];
      ConvDesc& d = prog.conv[size_t(pt.batch)].descs[size_t(pt.desc)];
      if (d.b.ptr) return false;
      const StridedView out = set_val(ni, alloc_like(value(n.sources[0])));
      d.b.ptr = out.ptr;
      post_tail.erase(n.sources[0]);
      P.n_fused++;
      P.avail_step[size_t(ni)] = pt.step;
      return true;
    }
    int j_tail = -1;
    for (size_t j = 0; j < n.sources.size(); ++j)
      if (chain_tail.count(n.sources[j])) {
        j_tail = int(j);
        break;
      }
    if (j_tail < 0) return false;
    const int src = n.sources[size_t(j_tail)];
    const Tail tail = chain_tail[src];
    const bool multi = tail.probs.size() > 1 || tail.like;  // per-image problems / conv layout
    for (const auto& pp : tail.probs)
      if (prog.gemm_specs[size_t(tail.batch)][size_t(pp.first)].n_epi >= kMaxEpi) return false;
    const int gstep = gemm_step[size_t(tail.batch)];
    EpiStage st;
    switch (op.fn) {
      case EwFn::pointwise_fn: st.op = EPI_TANH; break;
      case EwFn::pointwise_fn_grad: st.op = EPI_DTANH; break;
      case EwFn::scale: st.op = EPI_SCALE; st.scale = float(op.scale); break;
      case EwFn::add: st.op = EPI_ADD; break;
      case EwFn::sub: st.op = j_tail == 0 ? EPI_SUB_PO : EPI_SUB_OP; break;
    }
    if (n.sources.size() == 2) {
      if (multi) return false;
      const int other = n.sources[size_t(1 - j_tail)];
      if (other == src) return false;
      if (pending[size_t(other)] >= 0) return false;  // produced by an open launch
      const int avail = P.avail_step[size_t(other)];
      if (gstep >= 0 && avail >= gstep) return false;
      const StridedView& ov = value(other);
      if (ov.rank == 2) {
        st.other = ov.ptr;
        st.o_rs = ov.st[0];
        st.o_cs = ov.shape[1] == 1 ? 1 : ov.st[1];
      } else if (ov.rank == 4 && value(src).rank == 4 && value(src).contiguous() && ov.st[3] == 1 &&
                 ov.st[2] == ov.shape[3] && ov.st[1] == ov.shape[2] * ov.shape[3]) {
        // a filter [o, c, u, v] as the [o, cuv] matrix of the grad_weight GEMM's output
        st.other = ov.ptr;
        st.o_rs = ov.st[0];
        st.o_cs = 1;
      } else {
        return false;
      }
    }
    const StridedView out = set_val(ni, tail.like ? alloc_like(value(src)) : alloc(n.region.shape()));
    for (const auto& pp : tail.probs) {
      auto& spec = prog.gemm_specs[size_t(tail.batch)][size_t(pp.first)];
      EpiStage e = st;
      // the fused output has the node's (contiguous) layout, like the problem's own output
      e.out = eoff(out.ptr, pp.second);
      e.out_rs = spec.c_rs;
      e.out_cs = 1;
      spec.epi[spec.n_epi++] = e;
    }
    chain_tail.erase(src);
    chain_tail[ni] = tail;
    P.n_fused++;
    if (gstep >= 0) {
      P.avail_step[size_t(ni)] = gstep;
    } else {
      produced(ni, C_COMPUTE);
    }
    return true;
  }

  // ------------------------------------------------------------ conversions
  // Class of same-rank copies: after the NCCL receives they may unpack (C_COPY); in peer mode
  // there is no staging, so they share the phase's pull launch (C_XCHG): one launch, not two.
  Cls copy_cls() const { return P.peer() ? C_XCHG : C_COPY; }
  void copy_into(const StridedView& dst, const StridedView& src) {
    (P.peer() ? o_pull : o_copy).descs.push_back(ndesc(NARY_COPY, dst, {src}));
  }

  void lower_fetch_or_slice(int ni) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    const int src = n.sources[0];
    const PlanNode& sn = pl.nodes[size_t(src)];
    const bool dst_mine = mine_dev(n.device);
    const bool src_mine = mine_dev(sn.device);
    const bool remote = n.kind == NodeKind::fetch && (rank_of(n.device) != rank_of(sn.device) || force_xchg);
    const int cat = defer_to[size_t(ni)];

    if (n.kind == NodeKind::fetch && dst_mine) {
      P.fetch_in += n.bytes;
      P.op_bytes_in[op_of_phase(n.phase)] += n.bytes;
      P.phase_bytes_in[n.phase] += n.bytes;
    }
    const int sr = rank_of(sn.device);
    if (red_src[size_t(ni)] >= 0 && (!remote || P.peer())) {
      // read in place by the reduction that consumes it (no copy, no staging)
      const size_t bytes = size_t(n.region.volume()) * size_t(g_es);
      if (src_mine && rank_of(n.device) != C.rank) P.xrank_out += int64_t(bytes);
      if (!dst_mine) return;
      if (sr != C.rank) {
        P.xrank_in += int64_t(bytes);
        P.pull_bytes += int64_t(bytes);
      }
      Direct d;
      d.view = subview(src_view(sr, src), sn.region, n.region);
      d.src = src;
      d.rank = remote ? sr : -1;
      direct[ni] = d;
      return;
    }
    if (remote && P.peer()) {
      // peer pull: this rank reads the piece out of the owner's arena (pack + NVLink transfer +
      // unpack in one pass); the owner does nothing
      const size_t bytes = size_t(n.region.volume()) * size_t(g_es);
      if (src_mine && rank_of(n.device) != C.rank) P.xrank_out += int64_t(bytes);
      if (!dst_mine) return;
      if (sr != C.rank) {
        P.xrank_in += int64_t(bytes);
        P.pull_bytes += int64_t(bytes);
      } else {
        need(src, C_XCHG);
      }
      const StridedView sv = subview(src_view(sr, src), sn.region, n.region);
      StridedView target;
      if (cat >= 0) {
        ensure_alloc(cat);
        target = subview(P.val[size_t(cat)], pl.nodes[size_t(cat)].region, n.region);
      } else {
        target = set_val(ni, alloc(n.region.shape()));
        produced(ni, C_XCHG);
      }
      NaryDesc d = ndesc(NARY_COPY, target, {sv});
      d.wait_mask = 1u << sr;
      o_pull.descs.push_back(d);
      return;
    }
    if (!remote) {
      if (!dst_mine) return;
      if (n.kind == NodeKind::slice && cat < 0) {
        set_val(ni, subview(value(src), sn.region, n.region));
        P.avail_step[size_t(ni)] = P.avail_step[size_t(src)];
        if (pending[size_t(src)] >= 0) produced(ni, Cls(pending[size_t(src)]));
        return;
      }
      need(src, copy_cls());
      const StridedView sv = subview(value(src), sn.region, n.region);
      if (cat >= 0) {
        ensure_alloc(cat);
        const PlanNode& cn = pl.nodes[size_t(cat)];
        copy_into(subview(P.val[size_t(cat)], cn.region, n.region), sv);
      } else {
        const StridedView d = set_val(ni, alloc(n.region.shape()));
        copy_into(d, sv);
        produced(ni, copy_cls());
      }
      return;
    }
    // cross-rank (or forced) transfer through NCCL
    const size_t bytes = size_t(n.region.volume()) * size_t(g_es);
    if (src_mine) {
      need(src, C_PACK);
      const StridedView sv = subview(value(src), sn.region, n.region);
      const float* sp = sv.ptr;
      if (!sv.contiguous()) {
        const StridedView st = alloc(n.region.shape());
        o_pack.descs.push_back(ndesc(NARY_COPY, st, {sv}));
        sp = st.ptr;
      }
      o_xchg.x.push_back(Xfer{rank_of(n.device), true, const_cast<float*>(sp), bytes, ni});
      o_xchg.bytes_out += int64_t(bytes);
      if (rank_of(n.device) != C.rank) P.xrank_out += int64_t(bytes);
    }
    if (dst_mine) {
      if (rank_of(sn.device) != C.rank) P.xrank_in += int64_t(bytes);
      StridedView target;
      bool direct = false;
      if (cat >= 0) {
        ensure_alloc(cat);
        const PlanNode& cn = pl.nodes[size_t(cat)];
        target = subview(P.val[size_t(cat)], cn.region, n.region);
        direct = target.contiguous();
      } else {
        target = set_val(ni, alloc(n.region.shape()));
        direct = true;
      }
      if (direct) {
        o_xchg.x.push_back(Xfer{rank_of(sn.device), false, target.ptr, bytes, ni});
        if (cat < 0) produced(ni, C_XCHG);
      } else {
        const StridedView stg = alloc(n.region.shape());
        o_xchg.x.push_back(Xfer{rank_of(sn.device), false, stg.ptr, bytes, ni});
        copy_into(target, stg);
      }
      o_xchg.bytes_in += int64_t(bytes);
    }
  }

  void lower_concat(int ni) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    if (!mine_dev(n.device)) return;
    ensure_alloc(ni);
    for (int s : n.sources) {
      if (defer_to[size_t(s)] == ni) continue;  // already pasted by the piece itself
      need(s, copy_cls());
      const PlanNode& pn = pl.nodes[size_t(s)];
      copy_into(subview(P.val[size_t(ni)], n.region, pn.region), value(s));
    }
    // (a concat whose pieces all landed by themselves -- pulls or copies -- is produced by
    // the class that wrote them; the latest such class is the pull / copy one)
    produced(ni, copy_cls());
  }

  void lower_reduce(int ni) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    if (!mine_dev(n.device)) return;
    std::vector<StridedView> ins;
    uint32_t mask = 0;
    for (int s : n.sources) {
      auto it = direct.find(s);
      if (it != direct.end()) {  // a fetched partial read where it lies (local or on its peer)
        if (it->second.rank >= 0) mask |= 1u << it->second.rank;
        else need(it->second.src, C_REDUCE);
        ins.push_back(it->second.view);
        continue;
      }
      need(s, C_REDUCE);
      ins.push_back(value(s));
    }
    const StridedView out = set_val(ni, alloc(n.region.shape()));
    // Sum in source order (execgraph.cpp:264-282 fixes that order).  More than 8 partials
    // (k > 3) continue as out = out + next 7 in a following launch.
    size_t i = std::min(ins.size(), size_t(kMaxIn));
    NaryDesc d0 = ndesc(i == 1 ? NARY_COPY : NARY_SUM, out, std::vector<StridedView>(ins.begin(), ins.begin() + long(i)));
    d0.wait_mask = mask;
    if (mask) o_reduce.pull = true;
    o_reduce.descs.push_back(d0);
    if (i == ins.size() && fuse) {
      red_tail[ni] = RedTail{-1, int(o_reduce.descs.size()) - 1, -1, out};
      open_red.push_back(ni);
    }
    while (i < ins.size()) {
      produced(ni, C_REDUCE);
      flush();
      const size_t j = std::min(ins.size(), i + kMaxIn - 1);
      std::vector<StridedView> chunk{out};
      chunk.insert(chunk.end(), ins.begin() + long(i), ins.begin() + long(j));
      NaryDesc d = ndesc(NARY_SUM, out, chunk);
      d.wait_mask = mask;
      if (mask) o_reduce.pull = true;
      o_reduce.descs.push_back(d);
      i = j;
    }
    produced(ni, C_REDUCE);
  }

  // Elementwise consumer of a (finished) reduction, chained onto the reduction's launch: it reads
  // the sum's stored value in registers instead of from HBM (K4: partial-sum reduce fused with
  // the SGD step + update, or with the activation of a reduced pre-activation).
  bool try_fuse_reduce(int ni, const OpSpec& op) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    int j_tail = -1;
    for (size_t j = 0; j < n.sources.size(); ++j) {
      auto it = red_tail.find(n.sources[j]);
      if (it != red_tail.end() && it->second.batch >= 0) {
        j_tail = int(j);
        break;
      }
    }
    if (j_tail < 0) return false;
    const int src = n.sources[size_t(j_tail)];
    const RedTail t = red_tail[src];
    int code = 0;
    switch (op.fn) {
      case EwFn::pointwise_fn: code = EPI_TANH; break;
      case EwFn::pointwise_fn_grad: code = EPI_DTANH; break;
      case EwFn::scale: code = EPI_SCALE; break;
      case EwFn::add: code = EPI_ADD; break;
      case EwFn::sub: code = j_tail == 0 ? EPI_SUB_PO : EPI_SUB_OP; break;
    }
    const StridedView* other = nullptr;
    StridedView ov;
    if (n.sources.size() == 2) {
      const int o = n.sources[size_t(1 - j_tail)];
      if (o == src || pending[size_t(o)] >= 0 || P.avail_step[size_t(o)] >= t.step) return false;
      ov = value(o);
      other = &ov;
    } else if (n.sources.size() != 1) {
      return false;
    }
    if (n.region.shape() != pl.nodes[size_t(src)].region.shape()) return false;
    NaryDesc& d = prog.nary[size_t(t.batch)].descs[size_t(t.desc)];
    // (loop mode: a weight's w_next may take the weight's storage -- same layout -- and the
    // fresh allocation stays unused, so both programs allocate alike)
    StridedView out = alloc(n.region.shape());
    if (swap_to) {
      auto it = swap_to->find(ni);
      if (it != swap_to->end()) out = it->second;
    }
    if (!nary_add_chain(d, t.out, code, float(op.scale), out, other, g_es)) return false;
    set_val(ni, out);
    red_tail.erase(src);
    red_tail[ni] = t;
    P.avail_step[size_t(ni)] = t.step;
    P.n_fused++;
    return true;
  }

  void lower_buffer(int ni) {
    const PlanNode& n = pl.nodes[size_t(ni)];
    if (!mine_dev(n.device)) return;
    const StridedView v = set_val(ni, alloc(n.region.shape()));
    P.avail_step[size_t(ni)] = -1;
    InitDesc d;
    std::memset(&d, 0, sizeof d);
    d.out = v.ptr;
    const TensorSpec& t = pl.tensor(n.tensor);
    const int r = int(t.shape.size());
    if (r > kMaxRank) fail("tensor " + t.id + " has rank > 4");
    d.rank = r;
    const int pad = kMaxRank - r;
    for (int i = 0; i < kMaxRank; ++i) {
      if (i < pad) {
        d.full[i] = 1;
        d.lo[i] = 0;
        d.ext[i] = 1;
      } else {
        d.full[i] = t.shape[size_t(i - pad)];
        d.lo[i] = n.region.b[size_t(i - pad)][0];
        d.ext[i] = n.region.b[size_t(i - pad)][1] - n.region.b[size_t(i - pad)][0];
      }
    }
    d.n = n.region.volume();
    d.state0 = fnv1a(t.id.data(), t.id.size());  // XORed with the seed at init time
    P.init.descs.push_back(d);
  }

  void run_main() {
    const size_t N = pl.nodes.size();
    consumers.assign(N, 0);
    defer_to.assign(N, -1);
    is_holder.assign(N, 0);
    pending.assign(N, -1);
    for (const auto& kv : pl.holders)
      for (int h : kv.second) is_holder[size_t(h)] = 1;
    std::vector<int> last_consumer(N, -1);
    for (size_t i = 0; i < N; ++i)
      for (int s : pl.nodes[i].sources) {
        consumers[size_t(s)]++;
        last_consumer[size_t(s)] = int(i);
      }
    red_src.assign(N, -1);
    for (size_t i = 0; i < N; ++i) {
      const PlanNode& n = pl.nodes[i];
      if ((n.kind == NodeKind::fetch || n.kind == NodeKind::slice) && consumers[i] == 1 &&
          !is_holder[i]) {
        const int c = last_consumer[i];
        if (pl.nodes[size_t(c)].kind == NodeKind::concat && pl.nodes[size_t(c)].device == n.device)
          defer_to[i] = c;
        if (n.kind == NodeKind::fetch && fuse && pl.nodes[size_t(c)].kind == NodeKind::reduce_partial &&
            pl.nodes[size_t(c)].device == n.device)
          red_src[i] = c;
      }
    }
    // peer mode: every rank signals at the first conversion node of each phase in which any rank
    // pulls from another (the same sequence of sync points on every rank)
    std::set<std::string> xph;
    if (P.peer())
      for (const auto& n : pl.nodes)
        if (n.kind == NodeKind::fetch &&
            (rank_of(n.device) != rank_of(pl.nodes[size_t(n.sources[0])].device) || force_xchg))
          xph.insert(n.phase);
    std::string cur_phase;
    bool seen_conv = false, synced = false;
    for (size_t i = 0; i < N; ++i) {
      const PlanNode& n = pl.nodes[i];
      if (n.phase != cur_phase) {
        flush();
        cur_phase = n.phase;
        seg_op = op_of_phase(n.phase);
        seen_conv = false;
        synced = false;
        phase_sync = -1;
      }
      if (!synced && n.kind != NodeKind::sub_op && n.kind != NodeKind::buffer && xph.count(n.phase)) {
        sync_step(false);  // after this phase's compute, before any of its pulls
        synced = true;
      }
      switch (n.kind) {
        case NodeKind::buffer: lower_buffer(int(i)); break;
        case NodeKind::sub_op:
          if (seen_conv) flush();  // a compute after conversions starts a new segment
          if (mine_dev(n.device)) lower_sub_op(int(i));
          break;
        case NodeKind::slice:
        case NodeKind::fetch: seen_conv = true; lower_fetch_or_slice(int(i)); break;
        case NodeKind::concat: seen_conv = true; lower_concat(int(i)); break;
        case NodeKind::reduce_partial: seen_conv = true; lower_reduce(int(i)); break;
      }
    }
    flush();
    if (!xph.empty()) {
      sync_step(true);  // no rank starts the next step while another may still read this one
    }
  }

  // Loop carry: every "<w>_next" holder block onto the holder blocks of weight "<w>" (weights
  // carried by the loop-mode swap excepted).
  void run_carry() {
    bool any_pull = false;
    for (const auto& kv : pl.tensors) {
      const std::string& id = kv.first;
      if (id.size() <= 5 || id.compare(id.size() - 5, 5, "_next") != 0) continue;
      const std::string base = id.substr(0, id.size() - 5);
      if (!pl.tensors.count(base)) continue;
      if (std::find(P.swapped.begin(), P.swapped.end(), base) != P.swapped.end()) continue;
      if (pl.tensors.at(base).shape != kv.second.shape) continue;
      const auto& src_h = pl.holders.at(id);
      const auto& dst_h = pl.holders.at(base);
      for (int d = 0; d < pl.devices; ++d) {
        const int dn = dst_h[size_t(d)];
        const PlanNode& dnode = pl.nodes[size_t(dn)];
        if (dnode.kind != NodeKind::buffer)
          fail("loop carry: weight " + base + " is not a graph input on device " + std::to_string(d));
        // pieces: local overlap first, then the lowest-numbered holder of each region cell,
        // preferring holders on the destination's own rank
        std::vector<std::pair<Region, int>> pieces;
        std::vector<Region> remaining{dnode.region};
        auto take = [&](int e) {
          const Region& have = pl.nodes[size_t(src_h[size_t(e)])].region;
          std::vector<Region> next;
          for (const auto& box : remaining) {
            const Region ov = box.intersect(have);
            if (ov.volume() == 0) {
              next.push_back(box);
              continue;
            }
            pieces.push_back({ov, e});
            // peel the remainder of box minus ov into disjoint boxes
            Region rest = box;
            for (int dd = 0; dd < rest.rank(); ++dd) {
              if (rest.b[size_t(dd)][0] < ov.b[size_t(dd)][0]) {
                Region lo = rest;
                lo.b[size_t(dd)][1] = ov.b[size_t(dd)][0];
                next.push_back(lo);
                rest.b[size_t(dd)][0] = ov.b[size_t(dd)][0];
              }
              if (rest.b[size_t(dd)][1] > ov.b[size_t(dd)][1]) {
                Region hi = rest;
                hi.b[size_t(dd)][0] = ov.b[size_t(dd)][1];
                next.push_back(hi);
                rest.b[size_t(dd)][1] = ov.b[size_t(dd)][1];
              }
            }
          }
          remaining.swap(next);
        };
        take(d);
        for (int e = 0; e < pl.devices && !remaining.empty(); ++e)
          if (e != d && rank_of(e) == rank_of(d)) take(e);
        for (int e = 0; e < pl.devices && !remaining.empty(); ++e)
          if (rank_of(e) != rank_of(d)) take(e);
        if (!remaining.empty()) fail("loop carry: no holder covers part of " + id);
        for (const auto& pc : pieces) {
          const int e = pc.second;
          const int sn = src_h[size_t(e)];
          const PlanNode& snode = pl.nodes[size_t(sn)];
          const size_t bytes = size_t(pc.first.volume()) * size_t(g_es);
          const bool remote = rank_of(e) != rank_of(d) || (force_xchg && e != d);
          if (e != d) P.carry_bytes += int64_t(bytes);
          if (remote && P.peer()) {
            // pulled by the destination out of the owner's arena; the main program's closing
            // barrier already ordered every rank's w_next before this read
            any_pull = true;
            if (mine_dev(e) && rank_of(d) != C.rank) P.carry_xrank += int64_t(bytes);
            if (!mine_dev(d)) continue;
            const int sr = rank_of(e);
            NaryDesc nd = ndesc(NARY_COPY, subview(P.val[size_t(dn)], dnode.region, pc.first),
                                {subview(src_view(sr, sn), snode.region, pc.first)});
            nd.wait_mask = 1u << sr;
            o_pull.descs.push_back(nd);
            continue;
          }
          if (!remote) {
            if (!mine_dev(d)) continue;
            copy_into(subview(P.val[size_t(dn)], dnode.region, pc.first),
                      subview(value(sn), snode.region, pc.first));
            continue;
          }
          if (mine_dev(e)) {
            const StridedView sv = subview(value(sn), snode.region, pc.first);
            const float* sp = sv.ptr;
            if (!sv.contiguous()) {
              const StridedView st = alloc(pc.first.shape());
              o_pack.descs.push_back(ndesc(NARY_COPY, st, {sv}));
              sp = st.ptr;
            }
            o_xchg.x.push_back(Xfer{rank_of(d), true, const_cast<float*>(sp), bytes, sn});
            if (rank_of(d) != C.rank) P.carry_xrank += int64_t(bytes);
          }
          if (mine_dev(d)) {
            const StridedView target = subview(P.val[size_t(dn)], dnode.region, pc.first);
            if (target.contiguous()) {
              o_xchg.x.push_back(Xfer{rank_of(e), false, target.ptr, bytes, dn});
            } else {
              const StridedView stg = alloc(pc.first.shape());
              o_xchg.x.push_back(Xfer{rank_of(e), false, stg.ptr, bytes, dn});
              copy_into(target, stg);
            }
          }
        }
      }
    }
    seg_op = "carry";
    flush();
    if (any_pull) sync_step(true);  // the next step overwrites w_next only after every pull
  }
};

// Loop mode: weights whose buffer on every device of this rank can trade storage with the
// w_next holder of the same region (an owned allocation of identical layout).
std::map<int, StridedView> swap_pairs(PlanRt& P) {
  std::map<int, StridedView> ov;
  P.swapped.clear();
  const Plan& pl = P.plan;
  for (const auto& kv : pl.tensors) {
    const std::string& id = kv.first;
    if (id.size() <= 5 || id.compare(id.size() - 5, 5, "_next") != 0) continue;
    const std::string base = id.substr(0, id.size() - 5);
    if (!pl.tensors.count(base) || pl.tensors.at(base).shape != kv.second.shape) continue;
    const auto& wh = pl.holders.at(base);
    const auto& nh = pl.holders.at(id);
    std::map<int, StridedView> pairs;
    bool ok = true;
    for (int d = 0; d < pl.devices && ok; ++d) {
      if (P.dev_rank[size_t(d)] != P.ctx->rank) continue;
      const int b = wh[size_t(d)], h = nh[size_t(d)];
      const PlanNode& bn = pl.nodes[size_t(b)];
      const PlanNode& hn = pl.nodes[size_t(h)];
      ok = bn.kind == NodeKind::buffer &&
           (hn.kind == NodeKind::sub_op || hn.kind == NodeKind::concat || hn.kind == NodeKind::reduce_partial) &&
           bn.region.b == hn.region.b && P.has_val[size_t(b)] && P.has_val[size_t(h)];
      if (!ok) break;
      const StridedView& vb = P.val[size_t(b)];
      const StridedView& vh = P.val[size_t(h)];
      ok = vb.rank == vh.rank && vb.ptr != vh.ptr;
      for (int i = 0; ok && i < vb.rank; ++i) ok = vb.shape[i] == vh.shape[i] && vb.st[i] == vh.st[i];
      pairs[b] = vh;
      pairs[h] = vb;
    }
    if (!ok) continue;
    ov.insert(pairs.begin(), pairs.end());
    P.swapped.push_back(base);
  }
  return ov;
}

void lower(PlanRt& P, bool dry) {
  g_es = P.esize;
  P.main = Program{};
  P.main_b = Program{};
  P.carry = Program{};
  P.init = InitBatch{};
  P.val.assign(P.plan.nodes.size(), StridedView{});
  P.has_val.assign(P.plan.nodes.size(), 0);
  P.avail_step.assign(P.plan.nodes.size(), -1);
  P.arena_used = P.peer() ? kAlign : 0;  // peer mode: the sync counter lives at the arena base
  P.fetch_in = P.xrank_in = P.xrank_out = P.carry_bytes = P.carry_xrank = P.pull_bytes = 0;
  P.n_fused = 0;
  P.op_bytes_in.clear();
  P.phase_bytes_in.clear();
  for (const auto& op : P.plan.ops) P.op_bytes_in[op.id] = 0;
  P.gemm_flops = P.gemm_min_bytes = 0;
  if (dry) P.base = kFakeBase;
  {
    Lowerer L(P, P.main, dry);
    L.run_main();
  }
  P.swapped.clear();
  P.val_b.clear();
  if (P.loop()) {
    // the same lowering again with the swapped storage: every other allocation repeats at the
    // same offset, so both programs share one arena; the accounting is the first program's
    const std::map<int, StridedView> ov = swap_pairs(P);
    std::vector<StridedView> sv_val;
    std::vector<char> sv_has;
    std::vector<int> sv_avail;
    sv_val.swap(P.val);
    sv_has.swap(P.has_val);
    sv_avail.swap(P.avail_step);
    const size_t used = P.arena_used;
    const auto acct = std::make_tuple(P.fetch_in, P.xrank_in, P.xrank_out, P.n_fused, P.op_bytes_in, P.phase_bytes_in,
                                      P.gemm_flops, P.gemm_min_bytes, P.pull_bytes);
    P.val.assign(P.plan.nodes.size(), StridedView{});
    P.has_val.assign(P.plan.nodes.size(), 0);
    P.avail_step.assign(P.plan.nodes.size(), -1);
    P.arena_used = P.peer() ? kAlign : 0;
    InitBatch init_a = std::move(P.init);
    P.init = InitBatch{};
    {
      Lowerer L(P, P.main_b, dry);
      L.swap_to = &ov;
      L.run_main();
    }
    if (P.arena_used != used) fail("loop-mode lowering is not deterministic");
    P.init = std::move(init_a);  // inputs are seeded where the first program reads them
    P.val_b.swap(P.val);
    P.val.swap(sv_val);
    P.has_val.swap(sv_has);
    P.avail_step.swap(sv_avail);
    std::tie(P.fetch_in, P.xrank_in, P.xrank_out, P.n_fused, P.op_bytes_in, P.phase_bytes_in, P.gemm_flops,
             P.gemm_min_bytes, P.pull_bytes) = acct;
  }
  {
    Lowerer L(P, P.carry, dry);
    L.pending.assign(P.plan.nodes.size(), -1);
    L.run_carry();
  }
  P.n_sync = 0;
  for (const auto& st : P.main.steps)
    P.n_sync += st.kind == ST_SYNC || (st.kind == ST_NARY && P.main.nary[size_t(st.idx)].signal_s >= 0);
}

void prepare_program(PlanRt& P, Program& prog) {
  const bool bf = P.esize == 2;
  for (auto& b : prog.nary) {
    b.bf16 = bf;
    if (b.pull || b.signal_s >= 0) b.sync = P.sync;
    nary_prepare(b);
  }
  for (auto& b : prog.conv) {
    b.bf16 = bf;
    conv_prepare(b);
  }
  for (auto& specs : prog.gemm_specs) {
    for (auto& sp : specs) sp.bf16 = bf;
    prog.gemm.push_back(gemm_prepare(specs, P.ctx->num_sms, P.precision == 1));
  }
}

void free_program(Program& prog) {
  for (auto& b : prog.nary) nary_free(b);
  for (auto& b : prog.conv) conv_free(b);
  for (auto& g : prog.gemm) gemm_free(g);
  prog = Program{};
}

}  // namespace

PlanRt::~PlanRt() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  if (graph_exec_b) cudaGraphExecDestroy(graph_exec_b);
  for (auto& kv : range_graphs) cudaGraphExecDestroy(kv.second);
  free_program(main);
  free_program(carry);
  free_program(main_b);
  init_free(init);
  for (auto e : events) cudaEventDestroy(e);
  if (io_tmp) cudaFree(io_tmp);
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
  if (err_host) cudaFreeHost(err_host);
  if (arena) cudaFree(arena);
}

static size_t lower_other_ranks(PlanRt& P);

PlanRt* load_plan(Ctx* ctx, const std::string& json, int precision, int flags) {
  auto P = std::make_unique<PlanRt>();
  P->ctx = ctx;
  P->plan = parse_plan(json);
  P->precision = precision;
  P->flags = flags;
  P->stream = ctx->stream;
  if (precision != 0 && precision != 1) fail("unknown precision " + std::to_string(precision));
  // storage type = the graph's dtype: 4 -> fp32 (TF32 or 3xTF32 products), 2 -> bf16 (kind::f16
  // products, fp32 accumulation); one type per plan
  P->esize = 0;
  for (const auto& kv : P->plan.tensors) {
    const int db = kv.second.dtype_bytes;
    if (db != 4 && db != 2)
      fail("tensor " + kv.first + " has dtype_bytes " + std::to_string(db) +
           "; this executor runs fp32 (4) and bf16 (2) plans");
    if (P->esize && P->esize != db) fail("plan mixes dtype_bytes " + std::to_string(P->esize) + " and " + std::to_string(db));
    P->esize = db;
  }
  if (!P->esize) P->esize = 4;
  if (P->esize == 2 && precision == 1) fail("the 3xTF32 (fp32-accurate) mode needs an fp32 plan");
  const int devices = P->plan.devices;
  if (ctx->world > devices)
    fail("plan has " + std::to_string(devices) + " devices but the job has " + std::to_string(ctx->world) + " ranks");
  if (devices % ctx->world != 0) fail("plan devices must be a multiple of the rank count");
  P->dev_rank.resize(size_t(devices));
  for (int d = 0; d < devices; ++d) P->dev_rank[size_t(d)] = int((int64_t(d) * ctx->world) / devices);
  lower(*P, true);
  if (!ctx->host_only()) {
    if (P->peer()) {
      if (ctx->world > kMaxRanks) fail("peer mode supports at most " + std::to_string(kMaxRanks) + " ranks");
    } else if ((flags & 2) || ctx->world > 1) {
      if (!ctx->comm) {
        if (ctx->world > 1) fail("multi-rank plan needs tpx_init_comm first (or TPX_FLAG_PEER)");
        char uid[128];
        nccl_unique_id(uid);
        ctx->comm = nccl_comm_init(1, uid, 0);
      }
    }
    // TPX_FLAG_PEER_SOLO: this rank alone, every peer's arena stood in for by its own (sized for
    // the largest rank's layout): the rank's program runs unchanged with pulls reading local
    // HBM instead of NVLink and the peer counters already satisfied -- one rank's compute and
    // conversion time of an N-GPU step, measurable on one GPU (never a result: data is garbage)
    const bool solo = P->peer() && (flags & 128) && ctx->world > 1;
    if ((flags & 128) && !P->peer()) fail("TPX_FLAG_PEER_SOLO needs TPX_FLAG_PEER");
    const size_t need = solo ? lower_other_ranks(*P) : P->arena_used;
    P->arena_bytes = std::max<size_t>(need, kAlign);
    CUDA_CHECK(cudaMalloc(&P->arena, P->arena_bytes));
    // scratch padding (16-byte rows of im2col matrices, per-image column blocks) is read as
    // zero by the GEMMs and never written; the peer-mode sync counter starts at 0
    CUDA_CHECK(cudaMemset(P->arena, 0, P->arena_bytes));
    P->base = reinterpret_cast<uintptr_t>(P->arena);
    if (P->peer()) {
      CUDA_CHECK(cudaHostAlloc(&P->err_host, sizeof(int), cudaHostAllocMapped));
      *P->err_host = 0;
      int* err_dev = nullptr;
      CUDA_CHECK(cudaHostGetDevicePointer(&err_dev, P->err_host, 0));
      P->sync.local = reinterpret_cast<unsigned long long*>(P->arena);
      P->sync.epoch = reinterpret_cast<unsigned long long*>(P->arena) + 1;
      P->sync.err = err_dev;
      P->sync.world = ctx->world;
      P->sync.rank = ctx->rank;
      const char* to = std::getenv("TPX_PEER_TIMEOUT_S");
      P->sync.timeout_ns = static_cast<unsigned long long>((to ? std::atof(to) : 60.0) * 1e9);
      P->sync.peer[ctx->rank] = P->sync.local;
      P->peer_base.assign(size_t(ctx->world), 0);
      P->peer_base[size_t(ctx->rank)] = P->base;
      if (solo) {
        for (int r = 0; r < ctx->world; ++r) {
          P->peer_base[size_t(r)] = P->base;
          P->sync.peer[r] = P->sync.local;
        }
      } else if (ctx->world > 1) {
        return P.release();  // lowered by connect_peers once the arenas are mapped
      }
    }
    lower(*P, false);
    prepare_program(*P, P->main);
    prepare_program(*P, P->carry);
    prepare_program(*P, P->main_b);
    P->init.bf16 = P->esize == 2;
    init_prepare(P->init);
    P->lowered = true;
  } else {
    P->arena_bytes = P->arena_used;
  }
  return P.release();
}

// Every other rank's node values (and the largest arena any rank allocates), from a host-only
// lowering of the plan as that rank (deterministic: the rank lowers exactly so itself).
static size_t lower_other_ranks(PlanRt& P) {
  const int world = P.ctx->world, me = P.ctx->rank;
  P.rval.assign(size_t(world), {});
  P.rval_b.assign(size_t(world), {});
  P.rhas.assign(size_t(world), {});
  size_t most = P.arena_used;
  for (int r = 0; r < world; ++r) {
    if (r == me) continue;
    Ctx c2 = *P.ctx;
    c2.rank = r;
    c2.ordinal = -1;
    PlanRt q;
    q.ctx = &c2;
    q.plan = P.plan;
    q.precision = P.precision;
    q.flags = P.flags;
    q.esize = P.esize;
    q.dev_rank = P.dev_rank;
    lower(q, true);
    most = std::max(most, q.arena_used);
    P.rval[size_t(r)].swap(q.val);
    P.rval_b[size_t(r)].swap(q.val_b);
    P.rhas[size_t(r)].swap(q.has_val);
  }
  return most;
}

void arena_ipc_handle(PlanRt& P, void* out, size_t len) {
  if (!P.peer()) fail("IPC handles are for TPX_FLAG_PEER plans");
  if (P.ctx->host_only()) fail("host-only context has no arena");
  if (len < sizeof(cudaIpcMemHandle_t)) fail("IPC handle buffer must hold " + std::to_string(sizeof(cudaIpcMemHandle_t)) + " bytes");
  cudaIpcMemHandle_t h;
  CUDA_CHECK(cudaIpcGetMemHandle(&h, P.arena));
  std::memcpy(out, &h, sizeof h);
}

void connect_peers(PlanRt& P, const void* handles, size_t len) {
  if (!P.peer()) fail("connect_peers needs a TPX_FLAG_PEER plan");
  if (P.lowered) fail("plan is already connected");
  const int world = P.ctx->world, me = P.ctx->rank;
  if (len < size_t(world) * sizeof(cudaIpcMemHandle_t))
    fail("connect_peers needs " + std::to_string(world) + " arena handles (" +
         std::to_string(size_t(world) * sizeof(cudaIpcMemHandle_t)) + " bytes)");
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int r = 0; r < world; ++r) {
    if (r == me) continue;
    void* ptr = nullptr;
    CUDA_CHECK(cudaIpcOpenMemHandle(&ptr, hs[r], cudaIpcMemLazyEnablePeerAccess));
    P.ipc_opened.push_back(ptr);
    P.peer_base[size_t(r)] = reinterpret_cast<uintptr_t>(ptr);
    P.sync.peer[r] = static_cast<const unsigned long long*>(ptr);
  }
  lower_other_ranks(P);
  const size_t used = P.arena_used;
  lower(P, false);
  if (P.arena_used != used) fail("peer lowering is not deterministic");
  prepare_program(P, P.main);
  prepare_program(P, P.carry);
  prepare_program(P, P.main_b);
  P.init.bf16 = P.esize == 2;
  init_prepare(P.init);
  P.lowered = true;
}

void check_peer_error(PlanRt& P) {
  if (P.err_host && *P.err_host) {
    const int e = *P.err_host;
    fail("peer pull timed out waiting for rank " + std::to_string(e & 0xff) +
         " (a rank stopped executing the plan, or TPX_PEER_TIMEOUT_S is too short)");
  }
}

// NVTX range per lowered step, named "<op>:<what>" (the plan phase's op and the step's role):
// visible in ncu / nsys timelines (header-only NVTX 3; inert unless a tool is attached).
// TPX_NVTX=0 turns the ranges off.
static bool nvtx_on() {
  static const bool on = [] {
    const char* e = std::getenv("TPX_NVTX");
    return !(e && e[0] == '0');
  }();
  return on;
}

static void launch_step(PlanRt& P, Program& prog, const Step& s, cudaStream_t st) {
  struct Range {
    bool on;
    explicit Range(const Step& s) : on(nvtx_on()) {
      if (on) nvtxRangePushA((s.op.empty() ? s.what : s.op + ":" + s.what).c_str());
    }
    ~Range() {
      if (on) nvtxRangePop();
    }
  } range(s);
  switch (s.kind) {
    case ST_NARY: nary_run(prog.nary[size_t(s.idx)], st); break;
    case ST_GEMM: gemm_run(prog.gemm[size_t(s.idx)], st); break;
    case ST_CONV: conv_run(prog.conv[size_t(s.idx)], st); break;
    case ST_SYNC: sync_signal(P.sync, s.idx, s.barrier != 0, st); break;
    case ST_XCHG: {
      const XchgGroup& g = prog.xchg[size_t(s.idx)];
      nccl_group_start();
      for (const auto& x : g.x) {
        if (x.send) nccl_send(x.ptr, x.bytes, x.peer, P.ctx->comm, st);
        else nccl_recv(x.ptr, x.bytes, x.peer, P.ctx->comm, st);
      }
      nccl_group_end();
      break;
    }
  }
}

void run_program(PlanRt& P, Program& prog, const std::string* only_op) {
  if (P.ctx->host_only()) fail("host-only context cannot execute plans");
  if (!P.lowered) fail("peer-mode plan: tpx_plan_connect_peers must run on every rank first");
  cudaStream_t st = P.stream;
  const bool is_main = &prog == &P.main || &prog == &P.main_b;
  if ((P.flags & 8) && !P.timing && !only_op && is_main) {
    // CUDA graph of the whole lowered step (captured on first use, replayed after; the
    // stream must not change in between): one launch instead of one per lowered step
    cudaGraphExec_t& ge = &prog == &P.main ? P.graph_exec : P.graph_exec_b;
    if (!ge || P.graph_stream != st) {
      if (P.graph_exec) cudaGraphExecDestroy(P.graph_exec);
      if (P.graph_exec_b) cudaGraphExecDestroy(P.graph_exec_b);
      P.graph_exec = P.graph_exec_b = nullptr;
      cudaGraph_t g = nullptr;
      CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        for (const auto& s : prog.steps) launch_step(P, prog, s, st);
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CUDA_CHECK(cudaStreamEndCapture(st, &g));
      CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      P.graph_stream = st;
    }
    CUDA_CHECK(cudaGraphLaunch(ge, st));
    return;
  }
  if (!P.timing || only_op || !is_main) {  // per-step timing covers the step's main program
    for (const auto& s : prog.steps)  // (a barrier runs with every op: it ends each call)
      if (!only_op || s.op == *only_op || (s.kind == ST_SYNC && s.barrier)) launch_step(P, prog, s, st);
    return;
  }
  const size_t n = prog.steps.size();
  while (P.events.size() < n + 1) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    P.events.push_back(e);
  }
  CUDA_CHECK(cudaEventRecord(P.events[0], st));
  for (size_t i = 0; i < n; ++i) {
    launch_step(P, prog, prog.steps[i], st);
    CUDA_CHECK(cudaEventRecord(P.events[i + 1], st));
  }
  CUDA_CHECK(cudaEventSynchronize(P.events[n]));
  P.last_total_ms = P.last_gemm_ms = P.last_copy_ms = 0;
  P.last_step_ms.assign(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, P.events[i], P.events[i + 1]));
    P.last_step_ms[i] = ms;
    P.last_total_ms += ms;
    if (prog.steps[i].kind == ST_GEMM) P.last_gemm_ms += ms;
    else if (prog.steps[i].kind == ST_NARY || prog.steps[i].kind == ST_XCHG) P.last_copy_ms += ms;
  }
}

static const StridedView& node_val(PlanRt& P, int node, int64_t n);

void run_step(PlanRt& P) {
  if (!P.loop()) {
    run_program(P, P.main, nullptr);
    P.last = 0;
    return;
  }
  const int par = P.parity;
  run_program(P, par ? P.main_b : P.main, nullptr);
  if (!P.carry.steps.empty()) run_program(P, P.carry, nullptr);
  P.last = par;
  P.parity ^= 1;
}

void run_steps(PlanRt& P, int64_t begin, int64_t end) {
  if (P.ctx->host_only()) fail("host-only context cannot execute plans");
  if (!P.lowered) fail("peer-mode plan: tpx_plan_connect_peers must run on every rank first");
  // loop mode: the range runs on the program of the current step; the step ends (and the next
  // one uses the other program, after the carry) with the range that reaches the last step
  const int par = P.loop() ? P.parity : 0;
  Program& prog = par ? P.main_b : P.main;
  const int64_t n = int64_t(prog.steps.size());
  if (begin < 0 || end > n || begin > end) fail("step range [" + std::to_string(begin) + ", " + std::to_string(end) +
                                               ") outside the program's " + std::to_string(n) + " steps");
  cudaStream_t st = P.stream;
  if (P.flags & 8) {
    auto key = std::make_pair(begin + (int64_t(par) << 40), end);
    auto it = P.range_graphs.find(key);
    if (it == P.range_graphs.end() || P.graph_stream != st) {
      if (P.graph_stream != st) {
        for (auto& kv : P.range_graphs) cudaGraphExecDestroy(kv.second);
        P.range_graphs.clear();
      }
      cudaGraph_t g = nullptr;
      CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        for (int64_t i = begin; i < end; ++i) launch_step(P, prog, prog.steps[size_t(i)], st);
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CUDA_CHECK(cudaStreamEndCapture(st, &g));
      cudaGraphExec_t ge = nullptr;
      CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      P.graph_stream = st;
      it = P.range_graphs.emplace(key, ge).first;
    }
    CUDA_CHECK(cudaGraphLaunch(it->second, st));
  } else {
    for (int64_t i = begin; i < end; ++i) launch_step(P, prog, prog.steps[size_t(i)], st);
  }
  if (end == n && P.loop()) {
    if (!P.carry.steps.empty()) run_program(P, P.carry, nullptr);
    P.last = par;
    P.parity ^= 1;
  }
}

void copy_node_device(PlanRt& P, int node, void* dev, int64_t n, bool to_node) {
  g_es = P.esize;
  const StridedView& v = node_val(P, node, n);
  if (v.contiguous()) {
    if (to_node) CUDA_CHECK(cudaMemcpyAsync(v.ptr, dev, size_t(n) * size_t(P.esize), cudaMemcpyDeviceToDevice, P.stream));
    else CUDA_CHECK(cudaMemcpyAsync(dev, v.ptr, size_t(n) * size_t(P.esize), cudaMemcpyDeviceToDevice, P.stream));
    return;
  }
  NaryBatch b;
  b.bf16 = P.esize == 2;
  const StridedView flat = contiguous_view(static_cast<float*>(dev), std::vector<int64_t>(v.shape, v.shape + v.rank));
  b.descs.push_back(to_node ? ndesc(NARY_COPY, v, {flat}) : ndesc(NARY_COPY, flat, {v}));
  nary_prepare(b);
  nary_run(b, P.stream);
  CUDA_CHECK(cudaStreamSynchronize(P.stream));
  nary_free(b);
}

void init_inputs(PlanRt& P, uint64_t seed) {
  if (P.ctx->host_only()) fail("host-only context cannot execute plans");
  if (!P.lowered) fail("peer-mode plan: tpx_plan_connect_peers must run on every rank first");
  P.parity = P.last = 0;  // the inputs are seeded where the first program reads them
  if (P.init.descs.empty()) return;
  // re-key the descriptors with the seed (state0 = seed ^ fnv1a(id), dense.cpp:51)
  std::vector<uint64_t> keys;
  for (auto& d : P.init.descs) keys.push_back(d.state0);
  for (auto& d : P.init.descs) d.state0 ^= seed;
  init_prepare(P.init);
  for (size_t i = 0; i < keys.size(); ++i) P.init.descs[i].state0 = keys[i];
  init_run(P.init, P.stream);
}

static void ensure_io(PlanRt& P, int64_t n) {
  if (P.io_tmp_elems >= size_t(n)) return;
  if (P.io_tmp) cudaFree(P.io_tmp);
  CUDA_CHECK(cudaMalloc(&P.io_tmp, size_t(std::max<int64_t>(n, 1)) * 4));  // room for fp32 or bf16
  P.io_tmp_elems = size_t(n);
}

static const StridedView& node_val(PlanRt& P, int node, int64_t n) {
  if (P.ctx->host_only()) fail("host-only context holds no values");
  if (!P.lowered) fail("peer-mode plan: tpx_plan_connect_peers must run on every rank first");
  if (!P.has_val[size_t(node)])
    fail("node " + P.plan.nodes[size_t(node)].id + " has no value on this rank");
  const StridedView& v = (P.loop() && P.last == 1) ? P.val_b[size_t(node)] : P.val[size_t(node)];
  if (v.elements() != n)
    fail("buffer has " + std::to_string(n) + " elements, node " + P.plan.nodes[size_t(node)].id +
         " holds " + std::to_string(v.elements()));
  return v;
}

// NumericCheck on the device (simulator.cpp:129-147): every holder block of the
// tiled plan on this rank against the same region of the single-device plan's holder, max |d|
// and max |d| / max(|truth|, 1) reduced by one launch; only two floats come back.
void numeric_check(PlanRt& T, PlanRt& S, double* max_abs, double* max_rel, int64_t* values) {
  if (T.esize != S.esize) fail("numeric check: the plans store different element types");
  if (S.plan.devices != 1) fail("numeric check: the truth must be a one-device plan");
  g_es = T.esize;
  CUDA_CHECK(cudaStreamSynchronize(S.stream));
  CUDA_CHECK(cudaStreamSynchronize(T.stream));
  NaryBatch b;
  b.bf16 = T.esize == 2;
  int64_t n = 0;
  for (const auto& kv : T.plan.holders) {
    auto it = S.plan.holders.find(kv.first);
    if (it == S.plan.holders.end() || it->second.empty()) fail("numeric check: tensor " + kv.first + " has no truth");
    const int sn = it->second[0];
    const PlanNode& snode = S.plan.nodes[size_t(sn)];
    const StridedView& sv = node_val(S, sn, snode.region.volume());
    for (int h : kv.second) {
      if (h < 0 || !T.mine(h)) continue;
      const PlanNode& hn = T.plan.nodes[size_t(h)];
      if (hn.region.volume() == 0) continue;
      const StridedView& tv = node_val(T, h, hn.region.volume());
      const StridedView want = subview(sv, snode.region, hn.region);
      NaryDesc d = nary_desc(NARY_COPY, want, {tv, want}, 0.f, T.esize);
      d.vec = 1;
      d.units = tv.elements();
      b.descs.push_back(d);
      n += tv.elements();
    }
  }
  *max_abs = *max_rel = 0;
  *values = n;
  if (b.descs.empty()) return;
  nary_prepare(b);
  unsigned* dev = nullptr;
  unsigned host[2] = {0, 0};
  try {
    CUDA_CHECK(cudaMalloc(&dev, 2 * sizeof(unsigned)));
    CUDA_CHECK(cudaMemsetAsync(dev, 0, 2 * sizeof(unsigned), T.stream));
    numeric_check_run(b, dev, T.stream);
    CUDA_CHECK(cudaMemcpyAsync(host, dev, sizeof host, cudaMemcpyDeviceToHost, T.stream));
    CUDA_CHECK(cudaStreamSynchronize(T.stream));
  } catch (...) {
    if (dev) cudaFree(dev);
    nary_free(b);
    throw;
  }
  cudaFree(dev);
  nary_free(b);
  float fa, fr;
  std::memcpy(&fa, &host[0], 4);
  std::memcpy(&fr, &host[1], 4);
  *max_abs = fa;
  *max_rel = fr;
}

// Raw storage-type I/O: n elements of the plan's storage type (fp32 or bf16) in host memory.
void read_node_f32(PlanRt& P, int node, float* dst, int64_t n) {
  g_es = P.esize;
  const StridedView& v = node_val(P, node, n);
  const float* src = v.ptr;
  if (!v.contiguous()) {
    ensure_io(P, n);
    NaryBatch b;
    b.bf16 = P.esize == 2;
    b.descs.push_back(ndesc(NARY_COPY, contiguous_view(P.io_tmp, std::vector<int64_t>(v.shape, v.shape + v.rank)), {v}));
    nary_prepare(b);
    nary_run(b, P.stream);
    CUDA_CHECK(cudaStreamSynchronize(P.stream));
    nary_free(b);
    src = P.io_tmp;
  }
  CUDA_CHECK(cudaMemcpyAsync(dst, src, size_t(n) * size_t(P.esize), cudaMemcpyDeviceToHost, P.stream));
  CUDA_CHECK(cudaStreamSynchronize(P.stream));
}

void write_node_f32(PlanRt& P, int node, const float* src, int64_t n) {
  g_es = P.esize;
  const StridedView& v = node_val(P, node, n);
  if (v.contiguous()) {
    CUDA_CHECK(cudaMemcpyAsync(v.ptr, src, size_t(n) * size_t(P.esize), cudaMemcpyHostToDevice, P.stream));
    return;
  }
  ensure_io(P, n);
  CUDA_CHECK(cudaMemcpyAsync(P.io_tmp, src, size_t(n) * size_t(P.esize), cudaMemcpyHostToDevice, P.stream));
  NaryBatch b;
  b.bf16 = P.esize == 2;
  b.descs.push_back(ndesc(NARY_COPY, v, {contiguous_view(P.io_tmp, std::vector<int64_t>(v.shape, v.shape + v.rank))}));
  nary_prepare(b);
  nary_run(b, P.stream);
  CUDA_CHECK(cudaStreamSynchronize(P.stream));
  nary_free(b);
}

// bf16 <-> fp32 on the host: bf16 is the top half of an fp32; fp32 -> bf16 rounds to nearest
// even (NaN kept quiet), matching __float2bfloat16_rn.
static inline float bf16_to_f32(uint16_t h) {
  const uint32_t u = uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return uint16_t((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

void read_node(PlanRt& P, int node, double* dst, int64_t n) {
  std::vector<float> tmp(size_t(std::max<int64_t>(n, 1)));
  read_node_f32(P, node, tmp.data(), n);
  if (P.esize == 2) {
    const uint16_t* h = reinterpret_cast<const uint16_t*>(tmp.data());
    for (int64_t i = 0; i < n; ++i) dst[i] = double(bf16_to_f32(h[i]));
  } else {
    f32_to_f64_host(tmp.data(), dst, n);
  }
}

void write_node(PlanRt& P, int node, const double* src, int64_t n) {
  std::vector<float> tmp(size_t(std::max<int64_t>(n, 1)));
  if (P.esize == 2) {
    uint16_t* h = reinterpret_cast<uint16_t*>(tmp.data());
    for (int64_t i = 0; i < n; ++i) h[i] = f32_to_bf16(float(src[i]));
  } else {
    for (int64_t i = 0; i < n; ++i) tmp[size_t(i)] = float(src[i]);
  }
  write_node_f32(P, node, tmp.data(), n);
  CUDA_CHECK(cudaStreamSynchronize(P.stream));
}

std::string describe(const PlanRt& P) {
  std::ostringstream o;
  auto prog_json = [&](const Program& prog) {
    std::ostringstream s;
    s << "{\"steps\":[";
    for (size_t i = 0; i < prog.steps.size(); ++i) {
      const Step& st = prog.steps[i];
      if (i) s << ",";
      s << "{\"kind\":" << json_quote(st.kind == ST_NARY ? "nary" : st.kind == ST_GEMM ? "gemm" : st.kind == ST_CONV ? "conv" : st.kind == ST_SYNC ? "sync" : "nccl")
        << ",\"op\":" << json_quote(st.op) << ",\"what\":" << json_quote(st.what);
      if (st.kind == ST_NARY) {
        const NaryBatch& b = prog.nary[size_t(st.idx)];
        s << ",\"descs\":" << b.descs.size();
        double bytes = 0;
        int chained = 0;
        uint32_t mask = 0;
        for (const auto& d : b.descs) {
          int streams = d.nin + 1;
          for (int c = 0; c < d.n_chain; ++c) streams += 1 + (d.chain[c].other ? 1 : 0);
          bytes += double(P.esize) * double(d.units) * d.vec * streams;
          chained += d.n_chain;
          mask |= d.wait_mask;
        }
        s << ",\"bytes\":" << int64_t(bytes) << ",\"chained\":" << chained << ",\"pull\":" << (b.pull ? 1 : 0)
          << ",\"wait_mask\":" << mask << ",\"signal\":" << b.signal_s << ",\"wait_s\":" << b.wait_s;
      } else if (st.kind == ST_GEMM) {
        const auto& specs = prog.gemm_specs[size_t(st.idx)];
        s << ",\"problems\":" << specs.size() << ",\"shapes\":[";
        for (size_t j = 0; j < specs.size(); ++j) {
          const GemmSpec& g = specs[j];
          const long long M = g.ta ? g.a.cols : g.a.rows, K = g.ta ? g.a.rows : g.a.cols;
          const long long N = g.tb ? g.b.rows : g.b.cols;
          if (j) s << ",";
          s << "[" << M << "," << N << "," << K << "," << g.n_epi << "]";
        }
        s << "],\"ta\":" << (specs.empty() ? 0 : specs[0].ta) << ",\"tb\":" << (specs.empty() ? 0 : specs[0].tb);
        if (size_t(st.idx) < prog.gemm.size()) {
          const GemmLaunch& gl = prog.gemm[size_t(st.idx)];
          bool tstore = false;
          for (const auto& pr : gl.host_problems) tstore = tstore || pr.tstore;
          s << ",\"bn\":" << gl.bn << ",\"swap\":" << gl.swap << ",\"pair\":" << gl.pair
            << ",\"flops\":" << gl.flops << ",\"min_bytes\":" << gl.min_bytes << ",\"units\":" << gl.units
            << ",\"stream_k\":" << gl.sched.stream_k << ",\"group\":" << gl.sched.group
            << ",\"segments\":" << gl.sched.segs.size() << ",\"partial_slots\":" << gl.sched.nslots
            << ",\"oloader\":" << (gl.other_smem && gl.oloader && !gl.sched.dynamic ? 1 : 0)
            << ",\"other_smem\":" << gl.other_smem << ",\"odepth\":" << gl.odepth << ",\"stages\":" << gl.stages
            << ",\"p_mn\":" << gl.p_mn << ",\"q_mn\":" << gl.q_mn << ",\"split\":" << gl.split
            << ",\"bf16\":" << gl.bf16 << ",\"tstore\":" << (tstore ? 1 : 0);
        }
      } else if (st.kind == ST_XCHG) {
        const XchgGroup& g = prog.xchg[size_t(st.idx)];
        s << ",\"xfers\":[";
        for (size_t j = 0; j < g.x.size(); ++j) {
          const Xfer& x = g.x[j];
          if (j) s << ",";
          s << "{\"peer\":" << x.peer << ",\"send\":" << (x.send ? 1 : 0) << ",\"bytes\":" << x.bytes
            << ",\"node\":" << json_quote(P.plan.nodes[size_t(x.node)].id) << "}";
        }
        s << "],\"bytes_in\":" << g.bytes_in << ",\"bytes_out\":" << g.bytes_out;
      } else if (st.kind == ST_CONV) {
        s << ",\"descs\":" << prog.conv[size_t(st.idx)].descs.size()
          << ",\"bytes\":" << int64_t(prog.conv[size_t(st.idx)].bytes);
      } else if (st.kind == ST_SYNC) {
        s << ",\"barrier\":" << st.barrier << ",\"signal\":" << (st.barrier ? -1 : st.idx);
      }
      s << "}";
    }
    s << "]}";
    return s.str();
  };
  o << "{\"rank\":" << P.ctx->rank << ",\"world\":" << P.ctx->world << ",\"k\":" << P.plan.k
    << ",\"devices\":" << P.plan.devices << ",\"device_rank\":[";
  for (size_t d = 0; d < P.dev_rank.size(); ++d) o << (d ? "," : "") << P.dev_rank[d];
  o << "],\"fetch_bytes_total\":" << P.plan.fetch_bytes_total << ",\"rank_fetch_bytes_in\":" << P.fetch_in
    << ",\"rank_xrank_bytes_in\":" << P.xrank_in << ",\"rank_xrank_bytes_out\":" << P.xrank_out
    << ",\"carry_bytes\":" << P.carry_bytes << ",\"carry_xrank_bytes_out\":" << P.carry_xrank
    << ",\"fused_elementwise\":" << P.n_fused << ",\"arena_bytes\":" << P.arena_used
    << ",\"gemm_flops\":" << P.gemm_flops << ",\"peer\":" << (P.peer() ? 1 : 0)
    << ",\"pull_bytes_in\":" << P.pull_bytes << ",\"sync_points\":" << P.n_sync;
  auto map_json = [&](const std::map<std::string, int64_t>& m) {
    std::ostringstream s;
    s << "{";
    bool first = true;
    for (const auto& kv : m) {
      s << (first ? "" : ",") << json_quote(kv.first) << ":" << kv.second;
      first = false;
    }
    s << "}";
    return s.str();
  };
  o << ",\"per_op_fetch_bytes_in\":" << map_json(P.op_bytes_in)
    << ",\"per_phase_fetch_bytes_in\":" << map_json(P.phase_bytes_in) << ",\"main\":" << prog_json(P.main)
    << ",\"carry\":" << prog_json(P.carry) << ",\"loop\":" << (P.loop() ? 1 : 0) << ",\"swapped\":[";
  for (size_t i = 0; i < P.swapped.size(); ++i) o << (i ? "," : "") << json_quote(P.swapped[i]);
  o << "]}";
  return o.str();
}

}  // namespace tpx
