// C ABI for contexts and plans (include/tpx.h).  Every function converts exceptions into a
// status + tpx_last_error(), as the reference CLI maps tileplan::Error to "error: ..." + exit 1
// (proj/tools/main.cpp:397-404).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "capi_util.h"
#include "nccl_shim.h"
#include "runtime.h"
#include "tpx.h"

struct tpx_ctx {
  tpx::Ctx c;
};
struct tpx_plan {
  std::unique_ptr<tpx::PlanRt> p;
};

namespace {

tpx::PlanRt& rt(tpx_plan* p) {
  if (!p || !p->p) tpx::fail("null plan handle");
  return *p->p;
}
const tpx::PlanRt& rt(const tpx_plan* p) {
  if (!p || !p->p) tpx::fail("null plan handle");
  return *p->p;
}

int node_of(const tpx::PlanRt& P, const char* id) {
  if (!id) tpx::fail("null node id");
  return P.plan.node(id);
}

}  // namespace

TPX_API int tpx_create(int cuda_ordinal, int rank, int world, tpx_ctx** out) {
  return tpx::guard([&] {
    if (!out) tpx::fail("null output handle");
    if (world < 1 || rank < 0 || rank >= world) tpx::fail("bad rank/world");
    auto c = std::make_unique<tpx_ctx>();
    c->c.ordinal = cuda_ordinal;
    c->c.rank = rank;
    c->c.world = world;
    if (cuda_ordinal >= 0) {
      CUDA_CHECK(cudaSetDevice(cuda_ordinal));
      CUDA_CHECK(cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, cuda_ordinal));
      CUDA_CHECK(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
    }
    *out = c.release();
  });
}

TPX_API int tpx_comm_unique_id(void* out, size_t len) {
  return tpx::guard([&] {
    if (len < 128) tpx::fail("unique id buffer must hold 128 bytes");
    tpx::nccl_unique_id(out);
  });
}

TPX_API int tpx_init_comm(tpx_ctx* ctx, const void* unique_id, size_t len) {
  return tpx::guard([&] {
    if (!ctx) tpx::fail("null context");
    if (len < 128) tpx::fail("unique id must be 128 bytes");
    if (ctx->c.host_only()) tpx::fail("host-only context has no communicator");
    CUDA_CHECK(cudaSetDevice(ctx->c.ordinal));
    if (ctx->c.comm) tpx::nccl_comm_destroy(ctx->c.comm);
    ctx->c.comm = tpx::nccl_comm_init(ctx->c.world, unique_id, ctx->c.rank);
  });
}

TPX_API int tpx_destroy(tpx_ctx* ctx) {
  return tpx::guard([&] {
    if (!ctx) return;
    if (ctx->c.comm) tpx::nccl_comm_destroy(ctx->c.comm);
    if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
  });
}

TPX_API int tpx_load_plan(tpx_ctx* ctx, const char* plan_json, size_t len, int precision, int flags,
                          tpx_plan** out) {
  return tpx::guard([&] {
    if (!ctx || !plan_json || !out) tpx::fail("null argument");
    if (!ctx->c.host_only()) CUDA_CHECK(cudaSetDevice(ctx->c.ordinal));
    auto p = std::make_unique<tpx_plan>();
    p->p.reset(tpx::load_plan(&ctx->c, std::string(plan_json, len), precision, flags));
    *out = p.release();
  });
}

TPX_API int tpx_plan_free(tpx_plan* plan) {
  return tpx::guard([&] { delete plan; });
}

TPX_API int tpx_plan_stats(const tpx_plan* plan, tpx_stats* out) {
  return tpx::guard([&] {
    const tpx::PlanRt& P = rt(plan);
    tpx_stats s;
    std::memset(&s, 0, sizeof s);
    s.fetch_bytes_total = P.plan.fetch_bytes_total;
    s.rank_fetch_bytes_in = P.fetch_in;
    s.rank_xrank_bytes_in = P.xrank_in;
    s.rank_xrank_bytes_out = P.xrank_out;
    s.n_nodes = int64_t(P.plan.nodes.size());
    s.n_steps = int64_t(P.main.steps.size());
    for (const auto& st : P.main.steps) {
      if (st.kind == tpx::ST_XCHG) s.n_nccl_groups++;
      else s.n_kernel_launches++;
      if (st.kind == tpx::ST_GEMM) s.n_gemm_launches++;
      if (st.kind == tpx::ST_NARY) s.n_copy_launches++;
    }
    s.n_fused_ew = P.n_fused;
    s.device_bytes = int64_t(P.arena_used);
    s.gemm_flops = P.gemm_flops;
    s.gemm_min_bytes = P.gemm_min_bytes;
    s.storage_bytes = P.esize;
    *out = s;
  });
}

TPX_API int tpx_plan_describe(const tpx_plan* plan, char** json_out) {
  return tpx::guard([&] {
    const std::string s = tpx::describe(rt(plan));
    char* m = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(m, s.c_str(), s.size() + 1);
    *json_out = m;
  });
}

TPX_API void tpx_free_string(char* s) { std::free(s); }

TPX_API int tpx_init_inputs(tpx_plan* plan, uint64_t seed) {
  return tpx::guard([&] { tpx::init_inputs(rt(plan), seed); });
}

TPX_API int tpx_node_elements(const tpx_plan* plan, const char* node_id, int64_t* n) {
  return tpx::guard([&] {
    const tpx::PlanRt& P = rt(plan);
    *n = P.plan.nodes[size_t(node_of(P, node_id))].region.volume();
  });
}

TPX_API int tpx_write_node(tpx_plan* plan, const char* node_id, const double* src, int64_t n) {
  return tpx::guard([&] { tpx::write_node(rt(plan), node_of(rt(plan), node_id), src, n); });
}

TPX_API int tpx_read_node(tpx_plan* plan, const char* node_id, double* dst, int64_t n) {
  return tpx::guard([&] { tpx::read_node(rt(plan), node_of(rt(plan), node_id), dst, n); });
}

TPX_API int tpx_write_node_f32(tpx_plan* plan, const char* node_id, const float* src, int64_t n) {
  return tpx::guard([&] { tpx::write_node_f32(rt(plan), node_of(rt(plan), node_id), src, n); });
}

TPX_API int tpx_read_node_f32(tpx_plan* plan, const char* node_id, float* dst, int64_t n) {
  return tpx::guard([&] { tpx::read_node_f32(rt(plan), node_of(rt(plan), node_id), dst, n); });
}

TPX_API int tpx_node_view(const tpx_plan* plan, const char* node_id, uint64_t* dev_ptr, int* rank,
                          int64_t* shape4, int64_t* strides4) {
  return tpx::guard([&] {
    const tpx::PlanRt& P = rt(plan);
    const int n = node_of(P, node_id);
    if (!P.has_val[size_t(n)]) tpx::fail("node " + std::string(node_id) + " has no value on this rank");
    const tpx::StridedView& v = (P.loop() && P.last == 1) ? P.val_b[size_t(n)] : P.val[size_t(n)];
    *dev_ptr = reinterpret_cast<uint64_t>(v.ptr);
    *rank = v.rank;
    for (int i = 0; i < 4; ++i) {
      shape4[i] = i < v.rank ? v.shape[i] : 1;
      strides4[i] = i < v.rank ? v.st[i] : 0;
    }
  });
}

TPX_API int tpx_set_stream(tpx_plan* plan, uint64_t cuda_stream) {
  return tpx::guard([&] {
    tpx::PlanRt& P = rt(plan);
    P.stream = cuda_stream ? reinterpret_cast<cudaStream_t>(cuda_stream) : P.ctx->stream;
  });
}

TPX_API int tpx_execute(tpx_plan* plan) {
  return tpx::guard([&] { tpx::run_step(rt(plan)); });
}

TPX_API int tpx_execute_steps(tpx_plan* plan, int64_t begin, int64_t end) {
  return tpx::guard([&] { tpx::run_steps(rt(plan), begin, end); });
}

TPX_API int tpx_copy_node_device(tpx_plan* plan, const char* node_id, void* dev, int64_t n, int to_node) {
  return tpx::guard([&] {
    tpx::PlanRt& P = rt(plan);
    tpx::copy_node_device(P, node_of(P, node_id), dev, n, to_node != 0);
  });
}

TPX_API int tpx_execute_op(tpx_plan* plan, const char* op_id) {
  return tpx::guard([&] {
    tpx::PlanRt& P = rt(plan);
    const std::string op(op_id ? op_id : "");
    P.plan.op(op);  // validates the id
    tpx::run_program(P, P.main, &op);
    P.last = 0;
  });
}

TPX_API int tpx_carry_weights(tpx_plan* plan) {
  return tpx::guard([&] { tpx::run_program(rt(plan), rt(plan).carry, nullptr); });
}

TPX_API int tpx_synchronize(tpx_plan* plan) {
  return tpx::guard([&] {
    CUDA_CHECK(cudaStreamSynchronize(rt(plan).stream));
    tpx::check_peer_error(rt(plan));
  });
}

TPX_API int tpx_numeric_check(tpx_plan* tiled, tpx_plan* serial, double* max_abs, double* max_rel,
                              int64_t* values) {
  return tpx::guard([&] {
    if (!max_abs || !max_rel || !values) tpx::fail("null output");
    tpx::numeric_check(rt(tiled), rt(serial), max_abs, max_rel, values);
  });
}

TPX_API int tpx_plan_ipc_handle(tpx_plan* plan, void* out, size_t len) {
  return tpx::guard([&] {
    if (!out) tpx::fail("null output buffer");
    tpx::arena_ipc_handle(rt(plan), out, len);
  });
}

TPX_API int tpx_plan_connect_peers(tpx_plan* plan, const void* handles, size_t len) {
  return tpx::guard([&] {
    if (!handles) tpx::fail("null handle table");
    tpx::PlanRt& P = rt(plan);
    if (!P.ctx->host_only()) CUDA_CHECK(cudaSetDevice(P.ctx->ordinal));
    tpx::connect_peers(P, handles, len);
  });
}

TPX_API int tpx_enable_timing(tpx_plan* plan, int on) {
  return tpx::guard([&] { rt(plan).timing = on != 0; });
}

TPX_API int tpx_last_step_times(const tpx_plan* plan, double* ms, int64_t n, int64_t* n_steps) {
  return tpx::guard([&] {
    const tpx::PlanRt& P = rt(plan);
    *n_steps = int64_t(P.last_step_ms.size());
    for (int64_t i = 0; i < n && i < *n_steps; ++i) ms[i] = P.last_step_ms[size_t(i)];
  });
}

TPX_API int tpx_last_timing(const tpx_plan* plan, double* total_ms, double* gemm_ms, double* copy_ms) {
  return tpx::guard([&] {
    const tpx::PlanRt& P = rt(plan);
    *total_ms = P.last_total_ms;
    *gemm_ms = P.last_gemm_ms;
    *copy_ms = P.last_copy_ms;
  });
}
