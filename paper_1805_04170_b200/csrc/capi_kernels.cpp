// Kernel-level C entry points (tpx_gemm) and the thread-local error slot shared by the ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "capi_util.h"
#include "gemm.h"
#include "tpx.h"

namespace tpx {
thread_local std::string g_last_error;
}

extern "C" {

__attribute__((visibility("default"))) const char* tpx_last_error(void) {
  return tpx::g_last_error.c_str();
}

__attribute__((visibility("default"))) int tpx_version(void) { return 1; }

__attribute__((visibility("default"))) int tpx_gemm(
    const float* a, int64_t a_rows, int64_t a_cols, int64_t a_rs, const float* b, int64_t b_rows,
    int64_t b_cols, int64_t b_rs, int transpose_a, int transpose_b, float* c, int64_t c_rs,
    int n_epi, const int* epi_ops, const float* epi_scales, const float* const* epi_other,
    const int64_t* epi_other_rs, float* const* epi_out, const int64_t* epi_out_rs, int precision,
    uint64_t cuda_stream) {
  return tpx::guard([&] {
    if (n_epi < 0 || n_epi > tpx::kMaxEpi) tpx::fail("tpx_gemm: too many epilogue stages");
    tpx::GemmSpec s;
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
    tpx::GemmLaunch g = tpx::gemm_prepare({s}, sms, precision == 1);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    try {
      tpx::gemm_run(g, st);
      CUDA_CHECK(cudaStreamSynchronize(st));
    } catch (...) {
      tpx::gemm_free(g);
      throw;
    }
    tpx::gemm_free(g);
  });
}

__attribute__((visibility("default"))) int tpx_debug_gemm_mn_desc(unsigned lbo, unsigned sbo) {
  tpx::gemm_debug_mn_desc(lbo, sbo);
  return 0;
}

}  // extern "C"
