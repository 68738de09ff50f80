// Tile GEMM on 5th-generation tensor cores (tcgen05 + TMEM accumulators, TMA-fed smem
// pipeline), kind::tf32 on fp32 storage.  Replaces the reference's run_matmul
// (proj/src/dense.cpp:71-90): out = op(A) . op(B) with MatmulAttrs transpose flags
// (proj/include/tileplan/graph.hpp:41-44).  A batch holds the same-shaped sub-ops of several
// logical devices (one grouped launch).  Elementwise ops that consume the product on the same
// device without a conversion (act / seed / dact / step+upd, graph.cpp:189-227) run in the
// epilogue; every intermediate tensor is still stored.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tpx {

enum EpiOp : int {
  EPI_NONE = 0,
  EPI_TANH = 1,        // pointwise_fn      (dense.cpp:61)
  EPI_DTANH = 2,       // pointwise_fn_grad (dense.cpp:62-65): 1 - tanh(v)^2
  EPI_SCALE = 3,       // scale             (dense.cpp:188-191): s * v
  EPI_ADD = 4,         // add               prev + other
  EPI_SUB_PO = 5,      // sub with prev as input 0: prev - other
  EPI_SUB_OP = 6,      // sub with prev as input 1: other - prev
};

struct EpiStage {
  int op = EPI_NONE;
  float scale = 0.f;
  const float* other = nullptr;  // second operand (add/sub), indexed like the output
  long long o_rs = 0, o_cs = 0;
  float* out = nullptr;
  long long out_rs = 0, out_cs = 0;
};

constexpr int kMaxEpi = 3;

// One problem as the kernel sees it: D[P,Q] = sum_k A[p,k] * B[q,k] over TMA tensor maps.
struct GemmProblem {
  const void* tmap_a = nullptr;  // P operand
  const void* tmap_b = nullptr;  // Q operand
  int P = 0, Q = 0, K = 0;
  int tiles_p = 0, tiles_q = 0, splits = 1, kb_per_split = 0, kb_total = 0;
  int unit_begin = 0;
  float* out = nullptr;
  long long out_rs = 0, out_cs = 0;
  int n_epi = 0;
  EpiStage epi[kMaxEpi];
  unsigned mn_lbo = 4096, mn_sbo = 512;  // MN-major (128B_BASE32B) descriptor strides (bytes)
  float* ws = nullptr;          // split-K partial tiles
  unsigned int* counters = nullptr;
};

// Host-side description of one sub-op matmul over strided row-major fp32 views.
struct MatView {
  const float* ptr = nullptr;
  long long rows = 0, cols = 0;
  long long rs = 0, cs = 1;     // element strides
};

struct GemmSpec {
  MatView a, b;                 // stored operands (before transposition)
  bool ta = false, tb = false;  // MatmulAttrs
  float* c = nullptr;           // output M x N
  long long c_rs = 0, c_cs = 1;
  int n_epi = 0;
  EpiStage epi[kMaxEpi];        // in (row, col) of C; strides are C-indexed
};

struct GemmLaunch {
  int bn = 0;
  bool split = false;           // 3xTF32
  bool p_mn = false, q_mn = false, swap = false;
  int units = 0;
  int nprob = 0;
  void* d_problems = nullptr;   // GemmProblem[nprob] on device
  void* d_tmaps = nullptr;      // 2*nprob CUtensorMap on device
  float* d_ws = nullptr;
  unsigned int* d_counters = nullptr;
  size_t ws_floats = 0, n_counters = 0;
  size_t smem_bytes = 0;
  std::vector<GemmProblem> host_problems;  // for inspection (roofline accounting)
  double flops = 0;             // 2*M*N*K summed
  double min_bytes = 0;         // operands read once + outputs written once
};

// Whether `spec` can run on the TMA path (16-byte aligned bases and row strides, unit inner
// strides).  The plan lowering materialises a packed copy of any view that cannot.
bool gemm_view_ok(const MatView& v);

// Builds tensor maps / problem tables (device memory owned by the launch).
// split = 3xTF32 (fp32-accurate products), else single-pass TF32.
GemmLaunch gemm_prepare(const std::vector<GemmSpec>& specs, int num_sms, bool split = false);
void gemm_run(const GemmLaunch& g, cudaStream_t stream);
void gemm_free(GemmLaunch& g);
// Debug override of the MN-major descriptor strides (0 = defaults).
void gemm_debug_mn_desc(unsigned lbo, unsigned sbo);

}  // namespace tpx
