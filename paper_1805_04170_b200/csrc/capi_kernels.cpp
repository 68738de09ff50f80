// Kernel-level C entry points (tpx_gemm) and the thread-local error slot shared by the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "capi_util.h"
#include "gemm.h"
#include "tpx.h"

namespace tpx {
thread_local std::string g_last_error;
}

namespace {
// Variant chosen by the last tpx_gemm / tpx_gemm_timed on this thread (tpx_gemm_last_launch).
thread_local int64_t g_last_launch[16] = {0};

void record_launch(const tpx::GemmLaunch& g) {
  bool tstore = false;
  for (const auto& pr : g.host_problems) tstore = tstore || pr.tstore;
  const int64_t v[16] = {g.bn, g.pair, g.swap, g.p_mn, g.q_mn, g.other_smem && g.oloader && !g.sched.dynamic,
                         g.other_smem, g.sched.stream_k, g.sched.group, tstore, g.nbox, g.odepth, g.stages,
                         g.units, g.split, g.bf16};
  for (int i = 0; i < 16; ++i) g_last_launch[i] = v[i];
}
}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* tpx_last_error(void) {
  return tpx::g_last_error.c_str();
}

__attribute__((visibility("default"))) int tpx_version(void) { return 1; }

__attribute__((visibility("default"))) int tpx_gemm_timed(
    const float* a, int64_t a_rows, int64_t a_cols, int64_t a_rs, const float* b, int64_t b_rows,
    int64_t b_cols, int64_t b_rs, int transpose_a, int transpose_b, float* c, int64_t c_rs,
    int n_epi, const int* epi_ops, const float* epi_scales, const float* const* epi_other,
    const int64_t* epi_other_rs, float* const* epi_out, const int64_t* epi_out_rs, int precision,
    uint64_t cuda_stream, int warmup, int iters, double* avg_ms) {
  return tpx::guard([&] {
    if (n_epi < 0 || n_epi > tpx::kMaxEpi) tpx::fail("tpx_gemm: too many epilogue stages");
    if (precision < 0 || precision > 2) tpx::fail("tpx_gemm: precision must be 0 (tf32), 1 (3xtf32) or 2 (bf16)");
    tpx::GemmSpec s;
    s.bf16 = precision == 2;
    s.a = {a, a_rows, a_cols, a_rs, 1};
    s.b = {b, b_rows, b_cols, b_rs, 1};
    s.ta = transpose_a != 0;
    s.tb = transpose_b != 0;
    s.c = c;
    s.c_rs = c_rs;
    s.c_cs = 1;
    s.n_epi = n_epi;
    for (int e = 0; e < n_epi; ++e) {
      s.epi[e].op = epi_ops[e];
      s.epi[e].scale = epi_scales ? epi_scales[e] : 0.f;
      s.epi[e].other = epi_other ? epi_other[e] : nullptr;
      s.epi[e].o_rs = epi_other_rs ? epi_other_rs[e] : 0;
      s.epi[e].o_cs = 1;
      s.epi[e].out = epi_out[e];
      s.epi[e].out_rs = epi_out_rs[e];
      s.epi[e].out_cs = 1;
    }
    int dev = 0, sms = 148;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (const char* cap = std::getenv("TPX_GEMM_SMS")) sms = std::max(2, std::min(sms, std::atoi(cap)));  // debug
    tpx::GemmLaunch g = tpx::gemm_prepare({s}, sms, precision == 1);  // 2: bf16 storage (GemmSpec.bf16)
    record_launch(g);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    try {
      for (int i = 0; i < std::max(0, warmup); ++i) tpx::gemm_run(g, st);
      if (iters > 0) {
        CUDA_CHECK(cudaEventCreate(&e0));
        CUDA_CHECK(cudaEventCreate(&e1));
        CUDA_CHECK(cudaEventRecord(e0, st));
        for (int i = 0; i < iters; ++i) tpx::gemm_run(g, st);
        CUDA_CHECK(cudaEventRecord(e1, st));
      } else {
        tpx::gemm_run(g, st);
      }
      CUDA_CHECK(cudaStreamSynchronize(st));
      if (iters > 0 && avg_ms) {
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        *avg_ms = double(ms) / iters;
      }
    } catch (...) {
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      tpx::gemm_free(g);
      throw;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    tpx::gemm_free(g);
  });
}

__attribute__((visibility("default"))) int tpx_gemm(
    const float* a, int64_t a_rows, int64_t a_cols, int64_t a_rs, const float* b, int64_t b_rows,
    int64_t b_cols, int64_t b_rs, int transpose_a, int transpose_b, float* c, int64_t c_rs,
    int n_epi, const int* epi_ops, const float* epi_scales, const float* const* epi_other,
    const int64_t* epi_other_rs, float* const* epi_out, const int64_t* epi_out_rs, int precision,
    uint64_t cuda_stream) {
  return tpx_gemm_timed(a, a_rows, a_cols, a_rs, b, b_rows, b_cols, b_rs, transpose_a, transpose_b, c,
                        c_rs, n_epi, epi_ops, epi_scales, epi_other, epi_other_rs, epi_out, epi_out_rs,
                        precision, cuda_stream, 0, 0, nullptr);
}

__attribute__((visibility("default"))) int tpx_gemm_schedule(int nprob, int P, int Q, int K, int bn,
                                                             int num_sms, int force_groups, int max_kb,
                                                             int* grid, int* nsegs, int* nslots,
                                                             int* group, int* stream_k,
                                                             int32_t* segs, int max_segs,
                                                             int32_t* seg_off, int max_ctas) {
  return tpx::guard([&] {
    if (nprob < 1 || P < 1 || Q < 1 || K < 0 || num_sms < 1) tpx::fail("tpx_gemm_schedule: bad shape");
    if (bn != 32 && bn != 64 && bn != 128 && bn != 256) tpx::fail("tpx_gemm_schedule: bad tile width");
    std::vector<tpx::GemmProblem> probs(static_cast<size_t>(nprob));
    for (auto& pr : probs) {
      pr.P = P;
      pr.Q = Q;
      pr.K = K;
      pr.tiles_p = (P + 127) / 128;
      pr.tiles_q = (Q + bn - 1) / bn;
      pr.kb_total = (K + 31) / 32;
    }
    tpx::GemmSchedule S = tpx::gemm_schedule(probs, bn, num_sms, force_groups, max_kb);
    *grid = S.grid;
    *nsegs = int(S.segs.size());
    *nslots = S.nslots;
    *group = S.group;
    *stream_k = S.stream_k ? 1 : 0;
    if (segs && int(S.segs.size()) <= max_segs) {
      for (size_t i = 0; i < S.segs.size(); ++i) {
        const tpx::GemmSeg& g = S.segs[i];
        const int32_t v[8] = {g.prob, g.tp, g.tq, g.kb0, g.kb1, g.kind, g.slot, g.n_parts};
        std::memcpy(segs + 8 * i, v, sizeof(v));
      }
    }
    if (seg_off && S.grid + 1 <= max_ctas + 1)
      for (int i = 0; i <= S.grid; ++i) seg_off[i] = S.seg_off[size_t(i)];
  });
}

__attribute__((visibility("default"))) int tpx_gemm_last_launch(int64_t* info, int n) {
  return tpx::guard([&] {
    if (!info || n < 0) tpx::fail("tpx_gemm_last_launch: null buffer");
    for (int i = 0; i < n && i < 16; ++i) info[i] = g_last_launch[i];
  });
}

__attribute__((visibility("default"))) int tpx_debug_gemm_trace(uint64_t* out, int n) {
  return tpx::guard([&] { tpx::gemm_debug_trace(reinterpret_cast<unsigned long long*>(out), n); });
}

__attribute__((visibility("default"))) int tpx_debug_gemm_mn_desc(unsigned lbo, unsigned sbo) {
  tpx::gemm_debug_mn_desc(lbo, sbo);
  return 0;
}

}  // extern "C"
