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

#include "kernels.h"

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
  int tiles_p = 0, tiles_q = 0, kb_total = 0;
  float* out = nullptr;
  long long out_rs = 0, out_cs = 0;
  int n_epi = 0;
  EpiStage epi[kMaxEpi];
  // MN-major tf32 (128B_BASE32B) descriptor strides per operand, bytes: LBO = between 32-wide
  // MN chunks, SBO = between 4-row k groups, kstep = one MMA's 8 k rows.  Chunk-major stage
  // (2-D / 3-D maps): 4096 / 512 / 1024; k-group-major stage (4-D maps): 512 / nchunk*512 / 2*SBO
  unsigned a_lbo = 4096, a_sbo = 512, a_kstep = 1024;
  unsigned b_lbo = 4096, b_sbo = 512, b_kstep = 1024;
  // MN-major operand mapped in 3-D (32-wide chunk, K, chunk index): one TMA op per k-block
  int a3d = 0, b3d = 0;
  // MN-major tf32 operand mapped in 4-D (32-wide chunk, 4 k rows, chunk, k group): the stage
  // holds each 4-row k group's chunks side by side (the layout CUTLASS tiles its SW128_32B atom
  // to), one TMA op per k-block
  int a4d = 0, b4d = 0;
  // L2 policy per operand (0 = evict_last: small and re-read by many tiles; 1 = evict_first:
  // streamed) and streaming (.cs) epilogue stores for outputs far larger than L2
  int a_stream = 0, b_stream = 0, out_stream = 0;
  // TMA load map of the first epilogue stage's second operand (same 32 x 32 boxes), or null.
  const void* tmap_other = nullptr;
  int other_stage = -1;         // which epi stage tmap_other feeds
  // TMA store maps of the outputs (product, then each epi stage's), 32 x 16 boxes; tstore = 1
  // when every output has one (the epilogue then writes boxes to smem and the TMA stores them)
  const void* tmap_out[1 + kMaxEpi] = {nullptr, nullptr, nullptr, nullptr};
  int tstore = 0;
};

// One unit of a CTA's work list: k-blocks [kb0, kb1) of output tile (tp, tq) of problem `prob`.
// kind 0 = the whole k range (epilogue, no partials); 1 = head of a cut tile (waits for
// n_parts partial slots starting at `slot`, sums them in k order, runs the epilogue);
// 2 = a later k range of a cut tile (writes partial slot `slot` and raises its flag).
struct GemmSeg {
  int prob = 0, tp = 0, tq = 0, kb0 = 0, kb1 = 0;
  int kind = 0, slot = 0, n_parts = 0;
};

struct GemmSchedule {
  int grid = 0;                 // persistent CTAs (<= SM count)
  int group = 1;                // CTAs walking the same k ranges on neighbouring P-tiles
  bool stream_k = false;
  int nslots = 0;               // partial-tile workspace slots
  std::vector<GemmSeg> segs;    // all CTAs' lists, concatenated
  std::vector<int> seg_off;     // CTA c owns segs[seg_off[c], seg_off[c+1])
  bool dynamic = false;         // segs handed out in order by a device counter (seg_off = {0, n})
  // deferred fixup: every piece of a cut tile (its head too) writes a partial slot; a following
  // launch sums each tile's slots in k order and runs the epilogue chain, spread over the GPU,
  // instead of one head CTA per tile doing it serially at the end of the kernel
  bool deferred = false;
  struct Fixup {
    int prob, tp, tq, slot0, n_parts;
  };
  std::vector<Fixup> fixups;
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
  bool bf16 = false;            // bf16 storage (operands, outputs, epilogue operands)
  float* c = nullptr;           // output M x N
  long long c_rs = 0, c_cs = 1;
  int n_epi = 0;
  EpiStage epi[kMaxEpi];        // in (row, col) of C; strides are C-indexed
};

struct GemmLaunch {
  int bn = 0;
  bool split = false;           // 3xTF32
  bool p_mn = false, q_mn = false, swap = false;
  bool pair = false;            // CTA-pair (cta_group::2) 256 x 256 tiles
  bool bf16 = false;            // bf16 storage: kind::f16 MMAs
  int units = 0;                // CTAs launched
  int nprob = 0;
  int threads = 256;
  int stages = 0;               // smem ring depth
  int prefetch = 0;             // k-blocks of L2 prefetch ahead of the ring (0 = off)
  bool other_smem = false;      // epilogue operand staged through TMA
  bool oloader = false;         // ... by the loader warp, one 32 x 32 box per TMEM lane quarter
  int odepth = 0;               // its boxes in flight per epilogue warp
  int nbox = 1;                 // smem output boxes per epilogue warp (TMA-store epilogue)
  GemmSchedule sched;
  void* d_problems = nullptr;   // GemmProblem[nprob] on device
  void* d_tmaps = nullptr;      // 2*nprob CUtensorMap on device
  void* d_segs = nullptr;       // GemmSeg[] on device
  int* d_seg_off = nullptr;
  float* d_ws = nullptr;        // partial tiles (stream-K)
  unsigned int* d_flags = nullptr;
  size_t ws_floats = 0;
  size_t smem_bytes = 0;
  std::vector<GemmProblem> host_problems;  // for inspection (roofline accounting)
  NaryBatch fixup;              // deferred stream-K fixup launch (GemmSchedule::deferred)
  double flops = 0;             // 2*M*N*K summed
  double min_bytes = 0;         // operands read once + outputs written once
};

// Whether `spec` can run on the TMA path (16-byte aligned bases and row strides, unit inner
// strides).  The plan lowering materialises a packed copy of any view that cannot.
bool gemm_view_ok(const MatView& v, bool bf16 = false);

// Builds tensor maps / problem tables (device memory owned by the launch).
// split = 3xTF32 (fp32-accurate products), else single-pass TF32.
GemmLaunch gemm_prepare(const std::vector<GemmSpec>& specs, int num_sms, bool split = false);
void gemm_run(const GemmLaunch& g, cudaStream_t stream);
// The tile scheduler alone (host only; exposed for tests).  force_groups > 0 overrides the
// group count.
// max_kb > 0 bounds every segment's k range (3xTF32 accuracy, see gemm.cu).
GemmSchedule gemm_schedule(const std::vector<GemmProblem>& probs, int bn, int num_sms, int force_groups,
                           int max_kb = 0, bool deferred = false);
void gemm_free(GemmLaunch& g);
// Debug override of the MN-major descriptor strides (0 = defaults).
void gemm_debug_mn_desc(unsigned lbo, unsigned sbo);
// Debug (knob (22, 1)): the last traced launch's per-CTA timeline, 8 ns stamps per CTA.
void gemm_debug_trace(unsigned long long* out, int n);

}  // namespace tpx
