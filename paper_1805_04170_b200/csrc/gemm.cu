// Persistent tcgen05 tile GEMM (kind::tf32, fp32 storage).  See gemm.h.
//
// One CTA per SM, each walking a host-built list of segments (tile, k-block range).  Warp roles:
//   warp 0 lane 0  TMA producer   (cp.async.bulk.tensor -> 128B-swizzled smem ring)
//   warp 1 lane 0  MMA issuer     (tcgen05.mma.cta_group::1.kind::tf32 into one of two TMEM
//                                  accumulators, so segment i+1's mainloop overlaps segment
//                                  i's epilogue)
//   warp 2         TMEM allocator (2 x BN fp32 columns x 128 lanes)
//   warps 4..7     epilogue       (tcgen05.ld -> registers -> fused elementwise -> smem
//                                  transpose -> coalesced global stores; the elementwise
//                                  operand arrives by TMA one 32 x 32 box ahead)
//   warps 8..11    3xTF32 operand split (SPLIT only)
// Scheduling (gemm_prepare): whole tiles when there are many, else stream-K: the k-blocks of
// all tiles are cut evenly over the CTAs.  A tile cut into several segments is finished by the
// CTA holding its first k-range (the "head"); the others write partial tiles to a workspace and
// raise a flag.  The head waits for those flags — they are always the producers' FIRST
// segments, so no chain of waits can form — and adds the partials in k order, so the result is
// deterministic.  CTA groups of G (= the P-tile count of a small-M problem) walk the same k
// ranges side by side so a streamed B operand is read from DRAM once and from L2 G-1 times.
#include "gemm.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include <cuda_bf16.h>

#include "ptx.cuh"
#include "util.h"

namespace tpx {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block = one 128-byte swizzle row
constexpr int CW = 16;                                    // epilogue chunk: 16 accumulator columns
constexpr uint32_t kOutStage = 32 * CW * 4;               // one 32-row x CW fp32 box (64B swizzle)
constexpr uint32_t kOutStageBytes = 8 * kOutStage;        // <= 8 epilogue warps x 1 transpose box
// (TMA-store epilogues: nbox boxes per warp, one per output of the chain)
constexpr int kOtherDepth = 7;                            // max operand boxes in flight per warp
constexpr uint32_t kOtherBox = 8 * kOutStage;             // one box for each of <= 8 epilogue warps
constexpr uint32_t kSmemMax = 232448;                     // 227 KB opt-in
constexpr uint32_t kBarBytes = 2048;
constexpr int kSegQ = 8;  // tile queue depth (dynamic schedules)

enum SegKind : int { SEG_WHOLE = 0, SEG_HEAD = 1, SEG_PART = 2 };

// debug (22, 1): per-CTA timeline of one launch (%globaltimer, ns) at 8 milestones:
// entry, setup done, first TMA issued, first k-block landed (MMA), MMA loop done, first
// accumulator ready (epilogue), epilogue done, exit.
__device__ unsigned long long g_gemm_trace[320][8];
__device__ __forceinline__ void trace_mark(bool on, int i) {
  if (!on) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_gemm_trace[blockIdx.x < 320 ? blockIdx.x : 319][i] = t;
}

__host__ __device__ constexpr uint32_t operand_bytes(int bn) { return uint32_t(BM * BK * 4 + bn * BK * 4); }
__host__ __device__ constexpr uint32_t stage_bytes(int bn, bool split) {
  return operand_bytes(bn) * (split ? 2u : 1u);
}
// odepth = operand boxes in flight per epilogue warp (0 = no TMA-staged operand)
inline int stages_for(int bn, bool split, int odepth, int nbox = 1) {
  const uint32_t budget = kSmemMax - 1024 - kBarBytes - nbox * kOutStageBytes - odepth * kOtherBox;
  return std::min<int>(8, int(budget / stage_bytes(bn, split)));
}
inline size_t smem_for(int bn, bool split, int odepth, int stages, int nbox = 1) {
  return size_t(stages) * stage_bytes(bn, split) + nbox * kOutStageBytes + odepth * kOtherBox + 1024 + kBarBytes;
}
// 12 warps: producer, MMA, TMEM allocator, spare, then 8 epilogue warps (two per TMEM lane
// quarter, each on half the tile's columns) -- or, for 3xTF32, 4 epilogue + 4 splitting warps.
__host__ __device__ constexpr int threads_for(bool split) { return 384; }
__host__ __device__ constexpr int epi_warps(bool split) { return split ? 4 : 8; }
__host__ __device__ constexpr uint32_t tmem_cols_for(int bn) {
  return 2 * bn <= 32 ? 32 : 2 * bn <= 64 ? 64 : 2 * bn <= 128 ? 128 : 2 * bn <= 256 ? 256 : 512;
}
// 3xTF32: two accumulators + the fp32 sum of a tile's finished accumulation chains
__host__ __device__ constexpr uint32_t tmem_cols_split(int bn) {
  return 3 * bn <= 128 ? 128 : 3 * bn <= 256 ? 256 : 512;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// One fused elementwise stage over a thread's 32 values (the op is uniform per problem, so
// the switch sits outside the element loop).
__device__ __forceinline__ void epi_apply(int op, float (&v)[CW], const float (&o)[CW], float s) {
  switch (op) {
    case EPI_TANH:
#pragma unroll
      for (int j = 0; j < CW; ++j) v[j] = tanhf(v[j]);
      break;
    case EPI_DTANH:
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const float t = tanhf(v[j]);
        v[j] = 1.0f - t * t;
      }
      break;
    case EPI_SCALE:
#pragma unroll
      for (int j = 0; j < CW; ++j) v[j] = s * v[j];
      break;
    case EPI_ADD:
#pragma unroll
      for (int j = 0; j < CW; ++j) v[j] = v[j] + o[j];
      break;
    case EPI_SUB_PO:
#pragma unroll
      for (int j = 0; j < CW; ++j) v[j] = v[j] - o[j];
      break;
    case EPI_SUB_OP:
#pragma unroll
      for (int j = 0; j < CW; ++j) v[j] = o[j] - v[j];
      break;
    default: break;
  }
}

__device__ __forceinline__ bool epi_needs_other(int op) { return op >= EPI_ADD; }

// ---- storage-type access (B = bf16 storage, else fp32).  Global pointers are opaque `float*`
// addresses with element offsets; 4-element vector accesses are 16 B (fp32) or 8 B (bf16).
template <bool B>
__device__ __forceinline__ float ld1(const float* base, long long i) {
  if constexpr (B) return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(base) + i));
  else return __ldg(base + i);
}
template <bool B>
__device__ __forceinline__ void st1(float* base, long long i, float v) {
  if constexpr (B) reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
  else base[i] = v;
}
template <bool B>
__device__ __forceinline__ float4 ld4(const float* base, long long i) {
  if constexpr (B) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(base) + i));
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return __ldg(reinterpret_cast<const float4*>(base + i));
  }
}
template <bool B>
__device__ __forceinline__ void st4(float* base, long long i, float4 v, bool stream) {
  if constexpr (B) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    uint2* d = reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + i);
    if (stream) __stcs(d, u);
    else *d = u;
  } else {
    float4* d = reinterpret_cast<float4*>(base + i);
    if (stream) __stcs(d, v);
    else *d = v;
  }
}
// value as stored (fused stages consume the rounded value, exactly like the unfused launch)
template <bool B>
__device__ __forceinline__ float rnd(float v) {
  if constexpr (B) return __bfloat162float(__float2bfloat16_rn(v));
  else return v;
}
// base + i elements is 4-element (vector) aligned
template <bool B>
__device__ __forceinline__ bool vec_aligned(const float* base, long long i) {
  return ((reinterpret_cast<uintptr_t>(base) + uintptr_t(i) * (B ? 2 : 4)) & (B ? 7 : 15)) == 0;
}

// Store CW consecutive columns [q0, q0+CW) of row p.  Used for swapped problems (rs == 1):
// the warp's 32 rows are 32 consecutive elements, so every scalar store is one line.
template <bool B>
__device__ __forceinline__ void store_chunk(float* base, long long rs, long long cs, int p,
                                            int q0, int P, int Q, const float (&v)[CW]) {
  if (p >= P) return;
  const long long row = (long long)p * rs;
  if (cs == 1 && q0 + CW <= Q && vec_aligned<B>(base, row + q0)) {
#pragma unroll
    for (int j = 0; j < CW / 4; ++j)
      st4<B>(base, row + q0 + 4 * j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]), false);
  } else {
#pragma unroll
    for (int j = 0; j < CW; ++j)
      if (q0 + j < Q) st1<B>(base, row + (long long)(q0 + j) * cs, v[j]);
  }
}

template <bool B>
__device__ __forceinline__ void load_chunk(const float* base, long long rs, long long cs, int p,
                                           int q0, int P, int Q, float (&v)[CW]) {
  if (p >= P) {
#pragma unroll
    for (int j = 0; j < CW; ++j) v[j] = 0.f;
    return;
  }
  const long long row = (long long)p * rs;
  if (cs == 1 && q0 + CW <= Q && vec_aligned<B>(base, row + q0)) {
#pragma unroll
    for (int j = 0; j < CW / 4; ++j) {
      const float4 t = ld4<B>(base, row + q0 + 4 * j);
      v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < CW; ++j) v[j] = (q0 + j < Q) ? ld1<B>(base, row + (long long)(q0 + j) * cs) : 0.f;
  }
}

// Byte offset of 16-byte chunk c of row r in a 32 x CW fp32 box with the TMA 64-byte swizzle
// (chunk index XOR address bits 7..8): conflict-free both row-wise and column-wise.
__device__ __forceinline__ uint32_t box_off(int r, int c) { return r * (CW * 4) + ((c ^ ((r >> 1) & 3)) << 4); }

__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a) : "memory");
  return r;
}

// Elementwise-operand box (TMA): fp32 boxes are 32 x CW with the 64-byte swizzle (box_off);
// bf16 boxes are 32 x CW unswizzled (32-byte rows).  Store order: row r, columns 4c..4c+3.
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a) : "memory");
  return r;
}
__device__ __forceinline__ float4 bf16x4(uint2 u) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
template <bool B>
__device__ __forceinline__ float4 obox_so(uint32_t ob, int r, int c) {
  if constexpr (B) return bf16x4(lds64(ob + r * (CW * 2) + c * 8));
  else return lds128(ob + box_off(r, c));
}
// row `r`, 4 columns starting at 4j (row-order epilogue)
template <bool B>
__device__ __forceinline__ float4 obox_row(uint32_t ob, int r, int j) {
  if constexpr (B) return bf16x4(lds64(ob + r * (CW * 2) + j * 8));
  else return lds128(ob + box_off(r, j));
}

// Store a warp's 32 x CW block (thread = row `lane`, CW consecutive columns) into a row-major
// global view, transposed through a swizzled smem box so that each warp store instruction
// writes 8 rows x CW contiguous elements.  Rows >= P and columns >= Q are masked.
template <bool B>
__device__ __forceinline__ void store_block(uint32_t sbuf, int lane, const float (&v)[CW], float* base,
                                            long long rs, int prow0, int q0, int P, int Q, bool stream) {
#pragma unroll
  for (int j = 0; j < CW / 4; ++j) sts128(sbuf + box_off(lane, j), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
  const int c = lane & 3;
  const int gq = q0 + c * 4;
  const bool vec = vec_aligned<B>(base, 0) && ((rs & 3) == 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + (lane >> 2);
    const float4 x = lds128(sbuf + box_off(r, c));
    const int gp = prow0 + r;
    if (gp < P) {
      const long long o = (long long)gp * rs + gq;
      if (vec && gq + 4 <= Q) {
        st4<B>(base, o, x, stream);
      } else {
        if (gq < Q) st1<B>(base, o, x.x);
        if (gq + 1 < Q) st1<B>(base, o + 1, x.y);
        if (gq + 2 < Q) st1<B>(base, o + 2, x.z);
        if (gq + 3 < Q) st1<B>(base, o + 3, x.w);
      }
    }
  }
  __syncwarp();
}

// Elementwise stage on 4 values (store-order epilogue).
__device__ __forceinline__ float epi1(int op, float v, float o, float s) {
  switch (op) {
    case EPI_TANH: return tanhf(v);
    case EPI_DTANH: { const float t = tanhf(v); return 1.0f - t * t; }
    case EPI_SCALE: return s * v;
    case EPI_ADD: return v + o;
    case EPI_SUB_PO: return v - o;
    case EPI_SUB_OP: return o - v;
    default: return v;
  }
}
__device__ __forceinline__ void epi_apply4(int op, float4 (&x)[4], const float4 (&o)[4], float s) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i].x = epi1(op, x[i].x, o[i].x, s);
    x[i].y = epi1(op, x[i].y, o[i].y, s);
    x[i].z = epi1(op, x[i].z, o[i].z, s);
    x[i].w = epi1(op, x[i].w, o[i].w, s);
  }
}
// Store-order block store: x[i] = row (i*8 + lane/4), columns q0 + 4*(lane%4) .. +3 of a warp's
// 32 x CW block; each instruction writes 8 rows x CW contiguous elements.
template <bool B>
__device__ __forceinline__ void store_block_so(const float4 (&x)[4], int lane, float* base, long long rs,
                                               int prow0, int q0, int P, int Q, bool stream) {
  const int gq = q0 + (lane & 3) * 4;
  const bool vec = vec_aligned<B>(base, 0) && ((rs & 3) == 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gp = prow0 + i * 8 + (lane >> 2);
    if (gp < P) {
      const long long o = (long long)gp * rs + gq;
      if (vec && gq + 4 <= Q) {
        st4<B>(base, o, x[i], stream);
      } else {
        if (gq < Q) st1<B>(base, o, x[i].x);
        if (gq + 1 < Q) st1<B>(base, o + 1, x[i].y);
        if (gq + 2 < Q) st1<B>(base, o + 2, x[i].z);
        if (gq + 3 < Q) st1<B>(base, o + 3, x[i].w);
      }
    }
  }
}
template <bool B>
__device__ __forceinline__ void round4(float4 (&x)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[i].x = rnd<B>(x[i].x); x[i].y = rnd<B>(x[i].y); x[i].z = rnd<B>(x[i].z); x[i].w = rnd<B>(x[i].w);
  }
}

__device__ __forceinline__ void flag_release(unsigned* f) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(1u) : "memory");
}
__device__ __forceinline__ unsigned flag_acquire(const unsigned* f) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}

// Partial tiles live in L2-resident workspace slots of BM x BN floats (one per CTA; a pair tile
// has two), interleaved so that one warp-wide float4 access (32 rows, same 4 columns) is 512
// contiguous bytes.
__device__ __forceinline__ float4* ws_ptr(float* ws, int slot, int bn, int c0, int j, int row) {
  return reinterpret_cast<float4*>(ws + (size_t)slot * BM * bn) + ((c0 / CW) * (CW / 4) + j) * BM + row;
}

// SPLIT = 3xTF32: every fp32 operand x = hi + lo with hi = tf32_rna(x), lo = x - hi (exact);
// D += lo_A*hi_B + hi_A*lo_B + hi_A*hi_B.  The split runs in shared memory between the TMA
// landing and the MMA issue (warps 8..11).
// PAIR = CTA pair (cluster of 2, tcgen05 cta_group::2): one 256 x BN tile per pair; each CTA
// stages its 128 rows of A and BN/2 columns of B (half the operand bytes per CTA), the leader
// issues the M = 256 MMAs, and each CTA drains its own 128 accumulator rows.
// BF16 = bf16 storage: kind::f16 MMAs on bf16 operands (64-element k-blocks), fp32
// accumulators, epilogue stages computed in fp32 and stored rounded to bf16.
template <int BN, bool P_MN, bool Q_MN, bool SPLIT, bool PAIR, bool BF16>
__global__ void __launch_bounds__(threads_for(SPLIT), 1)
    gemm_tf32_kernel(const GemmProblem* __restrict__ probs, const GemmSeg* __restrict__ segs,
                     const int* __restrict__ seg_off, float* __restrict__ ws,
                     unsigned* __restrict__ flags, const int STAGES, const int PF,
                     const int has_other) {
  static_assert(!(PAIR && SPLIT), "3xTF32 runs on single-CTA tiles");
  static_assert(!(BF16 && SPLIT), "3xTF32 is an fp32-storage mode");
  constexpr int ES = BF16 ? 2 : 4;                  // storage bytes per element
  constexpr int BKE = 128 / ES;                     // k per k-block (one 128-byte smem row)
  constexpr int MNC = 128 / ES;                     // MN elements per MN-major chunk
  constexpr uint32_t MNCH = uint32_t(BKE) * 128u;   // bytes of one MN-major chunk (BKE k-rows)
  constexpr int KPM = BF16 ? 16 : 8;                // k per MMA instruction (32 bytes)
  constexpr int BNH = PAIR ? BN / 2 : BN;     // B columns staged by this CTA
  constexpr int PBM = PAIR ? 2 * BM : BM;     // rows of one (pair) tile
  constexpr uint32_t A_BYTES = BM * BK * 4;
  constexpr uint32_t OPB = operand_bytes(BNH);
  constexpr uint32_t STAGE = stage_bytes(BNH, SPLIT);
  static_assert(!SPLIT || 3 * BN <= 512, "3xTF32 tiles keep a third TMEM region for chain sums");
  constexpr uint32_t TMEM_COLS = SPLIT ? tmem_cols_split(BN) : tmem_cols_for(BN);
  constexpr int NEPI = epi_warps(SPLIT);
  constexpr uint32_t FMT = BF16 ? 1u : 2u;          // A/B format: bf16 (kind::f16) / tf32
  constexpr uint32_t IDESC = (1u << 4)                 // D format f32
                             | (FMT << 7) | (FMT << 10)
                             | (uint32_t(P_MN) << 15) | (uint32_t(Q_MN) << 16) |
                             (uint32_t(BN >> 3) << 17) | (uint32_t(PBM >> 4) << 24);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* out_stage = smem + STAGES * STAGE;  // [4 warps][32 rows x 128 B] store transpose
  const int NBOX = max(1, (has_other >> 8) & 7);       // output boxes per epilogue warp
  uint8_t* other_stage = out_stage + NBOX * kOutStageBytes;  // [8 warps][depth][32 rows x 64 B] if has_other
  const int ODEPTH = (has_other >> 4) & 7;  // operand ring depth (0 when unused)
  uint64_t* full = reinterpret_cast<uint64_t*>(other_stage + ODEPTH * kOtherBox);
  uint64_t* empty = full + STAGES;
  uint64_t* split_done = empty + STAGES;
  uint64_t* tmem_full = split_done + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;       // [2]
  uint64_t* other_bar = tmem_empty + 2;       // [8 warps][depth]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(other_bar + 8 * kOtherDepth);
  // dynamic schedule: tile queue filled by the (leader's) producer from a global counter
  int* seg_q = reinterpret_cast<int*>(tmem_holder + 2);            // [kSegQ]
  uint64_t* seg_full = reinterpret_cast<uint64_t*>(seg_q + kSegQ);  // [kSegQ]
  uint64_t* seg_empty = seg_full + kSegQ;                           // [kSegQ] (leader's)
  uint64_t* other_empty = seg_empty + kSegQ;                        // [8 warps][depth] (loader mode)
  const bool dyn = (has_other & 128) != 0;
  // loader mode: warp 3 issues every epilogue warp's operand boxes (the warps only consume)
  const bool oload = (has_other & 2048) != 0;
  // 3xTF32 accumulation chains: a segment's k range is accumulated in TMEM CHN k-blocks at a
  // time; each finished chain is added (fp32, round to nearest) into a third TMEM region.  The
  // tensor cores' accumulator does not round to nearest, so its error grows with the chain.
  const int CHN = SPLIT ? ((has_other >> 12) & 15) : 0;
  auto nchains = [&](const GemmSeg& sg) {
    const int n = sg.kb1 - sg.kb0;
    return (CHN > 0 && n > CHN) ? (n + CHN - 1) / CHN : 1;
  };

  const uint32_t rank = PAIR ? cluster_ctarank() : 0;  // 0 = MMA leader of the pair
  const int unit = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  // static: this unit's segments [seg_off[unit], seg_off[unit+1]); dynamic: segments 0..n-1
  // handed out in order by flags[0] (flags[1] counts finished units, the last one resets both)
  const int s_begin = dyn ? 0 : seg_off[unit], s_end = dyn ? seg_off[1] : seg_off[unit + 1];
  const int warp = warp_id(), lane = lane_id();
  const bool tr = (has_other >> 16) & 1;
  const bool epf = ((has_other >> 17) & 1) == 0;  // TMEM chunk prefetch in the epilogue
  const int nost = (has_other >> 18) & 7;          // debug: outputs whose stores are skipped
  const int stag = (has_other >> 21) & 63;         // debug: start delay of odd units, us
  if (threadIdx.x == 0) trace_mark(tr, 0);
  if (warp == 3 && lane == 0 && !dyn && s_begin < s_end) {
    // the first segment's operand descriptors, fetched while the CTA sets up (a cold tensor map
    // costs the producer's first TMA a global round trip)
    const GemmProblem& p0 = probs[segs[s_begin].prob];
    tma_prefetch_desc(p0.tmap_a);
    tma_prefetch_desc(p0.tmap_b);
    if (p0.tmap_other) tma_prefetch_desc(p0.tmap_other);
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split_done[s], 4);  // one arrival per splitting warp
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], PAIR ? 2 * NEPI : NEPI);  // one arrival per epilogue warp (of both CTAs)
    }
    for (int w = 0; w < 8 * kOtherDepth; ++w) {
      mbar_init(&other_bar[w], 1);
      mbar_init(&other_empty[w], oload ? 2 : 1);  // loader mode: both warps of a lane quarter
    }
    // queue slot consumers: MMA thread, epilogue warps, split warps, and the peer's producer
    // and epilogue warps (remote arrivals)
    const int n_cons = 1 + NEPI + (SPLIT ? 4 : 0) + (PAIR ? 1 + NEPI : 0);
    for (int q = 0; q < kSegQ; ++q) {
      mbar_init(&seg_full[q], 1);
      mbar_init(&seg_empty[q], n_cons);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_holder, TMEM_COLS);
    else tmem_alloc(tmem_holder, TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote use
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) trace_mark(tr, 1);
  // the leader's barriers, as shared::cluster addresses (pair TMA and epilogue arrivals)
  const uint32_t full_lead = PAIR ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
  const uint32_t tmem_empty_lead = PAIR ? mapa_shared(smem_u32(tmem_empty), 0) : smem_u32(tmem_empty);
  const uint32_t seg_empty_lead = PAIR ? mapa_shared(smem_u32(seg_empty), 0) : smem_u32(seg_empty);
  // Segment cursor of one role: static walks [s_begin, s_end); dynamic reads the tile queue
  // (`arrive`: this thread releases the slot for its role).  Returns -1 when done.
  struct Cursor {
    int j, si;
    bool done;
  };
  auto next_seg = [&](Cursor& c, bool arrive) -> int {
    if (!dyn) return c.si < s_end ? c.si++ : -1;
    if (c.done) return -1;
    const int slot = c.j % kSegQ;
    const uint32_t par = uint32_t(c.j / kSegQ) & 1u;
    if (PAIR && rank != 0) mbar_wait_acq_cluster(&seg_full[slot], par);
    else mbar_wait(&seg_full[slot], par);
    const int idx = *reinterpret_cast<volatile int*>(&seg_q[slot]);
    if (arrive) {
      if (PAIR && rank != 0) mbar_arrive_cluster_release(seg_empty_lead + slot * 8);
      else mbar_arrive(&seg_empty[slot]);
    }
    ++c.j;
    if (idx < 0) c.done = true;
    return idx;
  };

  // One k-block of operands: K-major tiles are one 2-D box; MN-major tiles are 32-wide
  // 128B_BASE32B-swizzled chunks 4096 bytes apart, one 3-D box when the extent allows.
  auto ld2 = [&](void* dst, const void* map, uint64_t* bar, uint32_t bar_c, int c0, int c1, uint64_t pol) {
    if constexpr (PAIR) tma_load_2d_pair(dst, map, bar_c, c0, c1, pol);
    else tma_load_2d_hint(dst, map, bar, c0, c1, pol);
  };
  auto ld3 = [&](void* dst, const void* map, uint64_t* bar, uint32_t bar_c, int c0, int c1, int c2, uint64_t pol) {
    if constexpr (PAIR) tma_load_3d_pair(dst, map, bar_c, c0, c1, c2, pol);
    else tma_load_3d_hint(dst, map, bar, c0, c1, c2, pol);
  };
  auto ld4 = [&](void* dst, const void* map, uint64_t* bar, uint32_t bar_c, int c2, int c3, uint64_t pol) {
    if constexpr (PAIR) tma_load_4d_pair(dst, map, bar_c, 0, 0, c2, c3, pol);
    else tma_load_4d_hint(dst, map, bar, 0, 0, c2, c3, pol);
  };
  // bar: local barrier (single CTA); bar_c: the leader's barrier in the cluster window (pair)
  auto load_kblock = [&](const GemmProblem& pr, int kb, int p0, int q0, uint8_t* sa, uint8_t* sb,
                         uint64_t* bar, uint32_t bar_c, uint64_t pol_a, uint64_t pol_b) {
    const int ka = kb * BKE, kq = kb * BKE;
    if constexpr (!P_MN) {
      ld2(sa, pr.tmap_a, bar, bar_c, ka, p0, pol_a);
    } else if (!BF16 && pr.a4d) {
      ld4(sa, pr.tmap_a, bar, bar_c, p0 / MNC, ka / 4, pol_a);
    } else if (pr.a3d) {
      ld3(sa, pr.tmap_a, bar, bar_c, 0, ka, p0 / MNC, pol_a);
    } else {
#pragma unroll
      for (int j = 0; j < BM / MNC; ++j) ld2(sa + j * MNCH, pr.tmap_a, bar, bar_c, p0 + MNC * j, ka, pol_a);
    }
    if constexpr (!Q_MN) {
      ld2(sb, pr.tmap_b, bar, bar_c, kq, q0, pol_b);
    } else if (!BF16 && pr.b4d) {
      ld4(sb, pr.tmap_b, bar, bar_c, q0 / MNC, kq / 4, pol_b);
    } else if (pr.b3d) {
      ld3(sb, pr.tmap_b, bar, bar_c, 0, kq, q0 / MNC, pol_b);
    } else {
#pragma unroll
      for (int j = 0; j < BNH / MNC; ++j) ld2(sb + j * MNCH, pr.tmap_b, bar, bar_c, q0 + MNC * j, kq, pol_b);
    }
  };
  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
    // debug (28, us): odd units start that many microseconds late (phase offset between the
    // units' store-heavy epilogues and their mainloops)
    if (stag > 0 && (unit & 1))
      for (int i = 0; i < stag; ++i) __nanosleep(1000);
    uint32_t s = 0, ph = 0;  // ring slot and its phase parity
    Cursor cur{0, s_begin, false};
    for (int j = 0;; ++j) {
      int si;
      if (dyn && rank == 0) {
        // fetch the next segment for the unit and publish it (to the peer as well)
        const int slot = j % kSegQ;
        mbar_wait(&seg_empty[slot], ((uint32_t(j / kSegQ)) & 1u) ^ 1u);
        si = int(atomicAdd(&flags[0], 1u));
        if (si >= s_end) si = -1;
        seg_q[slot] = si;
        if constexpr (PAIR) {
          st_shared_cluster_u32(mapa_shared(smem_u32(&seg_q[slot]), 1), uint32_t(si));
          mbar_arrive_cluster_release(mapa_shared(smem_u32(&seg_full[slot]), 1));
        }
        mbar_arrive(&seg_full[slot]);
      } else {
        si = next_seg(cur, true);
      }
      if (si < 0) break;
      const GemmSeg sg = segs[si];
      const GemmProblem& pr = probs[sg.prob];
      const int p0 = sg.tp * PBM + int(rank) * BM, q0 = sg.tq * BN + int(rank) * BNH;
      const uint64_t pol_a = pr.a_stream ? stream : keep, pol_b = pr.b_stream ? stream : keep;
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, (++s == uint32_t(STAGES)) ? (s = 0, ph ^= 1) : 0) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * STAGE;
        // the leader's full barrier expects both CTAs' bytes; the peer's TMA completes on it
        if (rank == 0) mbar_arrive_expect_tx(&full[s], PAIR ? 2 * OPB : OPB);
        load_kblock(pr, kb, p0, q0, sa, sa + A_BYTES, &full[s], full_lead + s * 8, pol_a, pol_b);
        if (j == 0 && kb == sg.kb0) trace_mark(tr, 2);
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (single thread; the pair's leader CTA)
    uint32_t s = 0, ph = 0;  // ring slot and its phase parity
    uint32_t ai = 0;         // accumulator uses (one per chain)
    Cursor cur{0, s_begin, false};
    for (;;) {
      const int si = next_seg(cur, true);
      if (si < 0) break;
      const GemmSeg sg = segs[si];
      const GemmProblem& pr = probs[sg.prob];
      const int nch = nchains(sg);
      for (int ch = 0; ch < nch; ++ch) {
      const int ck0 = nch > 1 ? sg.kb0 + ch * CHN : sg.kb0;
      const int ck1 = nch > 1 ? min(sg.kb1, ck0 + CHN) : sg.kb1;
      const uint32_t acc = ai & 1, aph = (ai >> 1) & 1;
      ++ai;
      mbar_wait(&tmem_empty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = ck0; kb < ck1; ++kb, (++s == uint32_t(STAGES)) ? (s = 0, ph ^= 1) : 0) {
        if constexpr (SPLIT) mbar_wait(&split_done[s], ph);
        else mbar_wait(&full[s], ph);
        if (ai == 1 && kb == ck0) trace_mark(tr, 3);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * STAGE);
        const uint32_t sb = sa + A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BKE / KPM; ++kk) {
          // K-major: 128B rows of K, 8-row atoms (SBO 1024), K step = +32 bytes.
          // MN-major tf32: 128B rows of M/N per k, 32-byte-granule swizzle, 512-byte atoms of
          //   4 k rows x 32 columns; per-operand LBO (chunk stride), SBO (k-group stride) and K
          //   step (8 rows = 2 k groups), GemmProblem::a_lbo ...
          // MN-major bf16: 128-byte swizzle, 8-row atoms (SBO 1024), 64-column chunks 8192 bytes
          //   apart (LBO), K step = 16 rows = +2048 bytes.
          const uint64_t ad = !P_MN ? umma_desc(sa + kk * 32, 16, 1024, 2)
                              : BF16 ? umma_desc(sa + kk * 2048, MNCH, 1024, 2)
                                     : umma_desc(sa + kk * pr.a_kstep, pr.a_lbo, pr.a_sbo, 1);
          const uint64_t bd = !Q_MN ? umma_desc(sb + kk * 32, 16, 1024, 2)
                              : BF16 ? umma_desc(sb + kk * 2048, MNCH, 1024, 2)
                                     : umma_desc(sb + kk * pr.b_kstep, pr.b_lbo, pr.b_sbo, 1);
          const uint32_t accum = (kb > ck0 || kk > 0) ? 1u : 0u;
          if constexpr (SPLIT) {
            // low parts live OPB bytes after the high parts, in the same (swizzled) layout
            const uint64_t lo = uint64_t((OPB >> 4) & 0x3FFFu);
            mma_tf32(d, ad + lo, bd, IDESC, accum);
            mma_tf32(d, ad, bd + lo, IDESC, 1u);
            mma_tf32(d, ad, bd, IDESC, 1u);
          } else if constexpr (PAIR) {
            if constexpr (BF16) mma_f16_pair(d, ad, bd, IDESC, accum);
            else mma_tf32_pair(d, ad, bd, IDESC, accum);
          } else {
            if constexpr (BF16) mma_f16(d, ad, bd, IDESC, accum);
            else mma_tf32(d, ad, bd, IDESC, accum);
          }
        }
        if constexpr (PAIR) mma_commit_pair(&empty[s], 0x3);  // frees the slot in both CTAs
        else mma_commit(&empty[s]);
      }
      if constexpr (PAIR) mma_commit_pair(&tmem_full[acc], 0x3);
      else mma_commit(&tmem_full[acc]);
      }
    }
    trace_mark(tr, 4);
  } else if (warp == 3 && lane == 0 && oload) {
    // ---------------- operand loader: the epilogue's elementwise operand (w of
    // w_next = w - wd) as one 32 x 32 box per TMEM lane quarter and 32-column step (the two
    // warps of the quarter each read their 16 columns), ODEPTH boxes ahead per quarter
    const int ODEPTH = (has_other >> 4) & 7;
    const uint64_t pol = policy_evict_first();
    uint32_t ring[4] = {0, 0, 0, 0}, uses[4] = {0, 0, 0, 0};
    Cursor cur{0, s_begin, false};
    for (;;) {
      const int si = next_seg(cur, false);
      if (si < 0) break;
      const GemmSeg sg = segs[si];
      const GemmProblem& pr = probs[sg.prob];
      if (sg.kind == SEG_PART || !pr.tmap_other) continue;
      const int qb = sg.tq * BN;
      for (int c0 = 0; c0 < BN; c0 += 2 * CW) {
        if (qb + c0 >= pr.Q) break;
        for (int q = 0; q < 4; ++q) {
          const int slot = q * ODEPTH + int(ring[q]);
          mbar_wait(&other_empty[slot], ((uses[q] / uint32_t(ODEPTH)) & 1u) ^ 1u);
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&other_bar[slot], uint32_t(32 * 2 * CW * ES));
          tma_load_2d_hint(other_stage + slot * (2 * kOutStage), pr.tmap_other, &other_bar[slot], qb + c0,
                           sg.tp * PBM + int(rank) * BM + q * 32, pol);
          ++uses[q];
          if (++ring[q] == uint32_t(ODEPTH)) ring[q] = 0;
        }
      }
    }
  } else if (SPLIT && warp >= 8) {  // (SPLIT: NEPI == 4, epilogue warps 4..7)
    // ---------------- 3xTF32 split: hi in place, lo into the stage's second half
    const int tid = threadIdx.x - 256;  // 0..127
    uint32_t s = 0, ph = 0;  // ring slot and its phase parity
    Cursor cur{0, s_begin, false};
    for (;;) {
      const int si = next_seg(cur, lane == 0);
      if (si < 0) break;
      const GemmSeg sg = segs[si];
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, (++s == uint32_t(STAGES)) ? (s = 0, ph ^= 1) : 0) {
        mbar_wait(&full[s], ph);
        float4* hi = reinterpret_cast<float4*>(smem + s * STAGE);
        float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + OPB);
        for (int c = tid; c < int(OPB / 16); c += 128) {
          float4 x = hi[c], h, l;
          h.x = tf32_rna(x.x); h.y = tf32_rna(x.y); h.z = tf32_rna(x.z); h.w = tf32_rna(x.w);
          l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
          hi[c] = h;
          lo[c] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&split_done[s]);
      }
    }
  } else if (warp >= 4 && warp < 4 + NEPI) {
    // ---------------- epilogue: warp 4+e owns TMEM lanes [32(e%4), +32) and, with 8 warps,
    // the columns [ (e/4) BN/2, (e/4+1) BN/2 )
    const int ew = warp - 4;
    const int lq = ew & 3;
    // With 8 warps the two warps of a lane quarter interleave CW-column chunks, so each step
    // of the pair writes whole 128-byte lines of its rows.
    const int c_begin = NEPI == 8 ? (ew >> 2) * CW : 0;
    const int c_end = BN;
    constexpr int CSTEP = NEPI == 8 ? 2 * CW : CW;
    const int row = lq * 32 + lane;
    const bool leader = (ew == 0 && lane == 0);
    auto wslot = [&](int slot) { return PAIR ? 2 * slot + int(rank) : slot; };  // this CTA's half
    // Elementwise operand (w for w_next = w - wd): 32 x CW boxes, TMA-loaded ODEPTH chunks
    // ahead through a per-warp ring.  Lane 0 owns the issue cursor; boxes are issued and
    // consumed in the same (segment, chunk) order.
    uint32_t o_slot = 0, o_phase = 0;  // consumer ring position
    uint32_t box_half = 0;             // TMA-store epilogue: box set of the next chunk
    uint32_t i_slot = 0;               // issuer ring position (lane 0)
    const uint64_t o_policy = policy_evict_first();  // the elementwise operand is read once
    Cursor icur{0, s_begin, false};                   // issue cursor (lane 0)
    int ic0 = c_begin;
    const void* imap = nullptr;
    int iq = 0, ip = 0, iQ = 0;
    bool iseg = false;  // a segment is loaded into the cursor
    auto issue_other = [&]() {
      for (;; iseg = false) {
        if (!iseg) {
          const int isi = next_seg(icur, false);
          if (isi < 0) return;
          const GemmSeg sg = segs[isi];
          const GemmProblem& pr = probs[sg.prob];
          iseg = true;
          ic0 = c_begin;
          imap = sg.kind == SEG_PART ? nullptr : pr.tmap_other;
          iq = sg.tq * BN;
          ip = sg.tp * PBM + int(rank) * BM + lq * 32;
          iQ = pr.Q;
        }
        if (imap && ic0 < c_end && iq + ic0 < iQ) {
          uint64_t* bar = &other_bar[ew * ODEPTH + i_slot];
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(bar, uint32_t(32 * CW * ES));  // one 32 x CW operand box
          tma_load_2d_hint(other_stage + (ew * ODEPTH + i_slot) * kOutStage, imap, bar, iq + ic0, ip, o_policy);
          if (++i_slot == uint32_t(ODEPTH)) i_slot = 0;
          ic0 += CSTEP;
          return;
        }
      }
    };
    // operand ring of this warp: its own 32 x 16 boxes, or (loader mode) its lane quarter's
    // 32 x 32 boxes shared with the quarter's other warp (128-byte rows, 128-byte swizzle)
    const int oring = (oload ? lq : ew) * ODEPTH;
    auto obar = [&](uint32_t sl) { return &other_bar[oring + int(sl)]; };
    auto obox = [&](uint32_t sl) {
      return smem_u32(other_stage) + uint32_t(oring + int(sl)) * (oload ? 2 * kOutStage : kOutStage);
    };
    // row r, 16-byte group c (columns 4c..4c+3) of this warp's 16 operand columns
    auto oread = [&](uint32_t ob, int r, int c) -> float4 {
      if (oload) return lds128(ob + uint32_t(r) * 128u + (uint32_t(((ew >> 2) * 4 + c) ^ (r & 7)) << 4));
      return obox_so<BF16>(ob, r, c);
    };
    // a box was consumed (o_slot already advanced): refill it (own issue) or hand it back
    auto other_done = [&]() {
      if (oload) mbar_arrive(&other_empty[oring + int(o_slot == 0 ? ODEPTH - 1 : o_slot - 1)]);
      else issue_other();
    };
    if ((has_other & 1) && lane == 0 && !oload)
      for (int d = 0; d < ODEPTH; ++d) issue_other();
    Cursor cur{0, s_begin, false};
    uint32_t ai = 0;  // accumulator uses (one per chain)
    const uint32_t tsum = tmem_base + 2 * BN + (uint32_t(lq * 32) << 16);  // 3xTF32 chain sums
    for (;;) {
      const int si = next_seg(cur, lane == 0);
      if (si < 0) break;
      const GemmSeg sg = segs[si];
      const GemmProblem& pr = probs[sg.prob];
      const int nch = nchains(sg);
      if constexpr (SPLIT) {
        // every chain but the last: drained into the sum region (this warp's lane quarter, all
        // columns), then the accumulator goes back to the MMA warp
        for (int ch = 0; ch + 1 < nch; ++ch) {
          const uint32_t a2 = ai & 1, ap2 = (ai >> 1) & 1;
          ++ai;
          mbar_wait(&tmem_full[a2], ap2);
          tc_fence_after();
          const uint32_t ta = tmem_base + a2 * BN + (uint32_t(lq * 32) << 16);
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += CW) {
            float v[CW], w[CW];
            tmem_ld16(ta + c0, v);
            if (ch > 0) {
              tmem_ld16(tsum + c0, w);
#pragma unroll
              for (int j = 0; j < CW; ++j) v[j] = w[j] + v[j];
            }
            tmem_st16(tsum + c0, v);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_lead + a2 * 8);
        }
      }
      const bool summed = SPLIT && nch > 1;
      // the last chain's accumulator plus the earlier chains' sum
      auto add_sum = [&](int c0, float (&v)[CW]) {
        if (summed) {
          float w[CW];
          tmem_ld16(tsum + c0, w);
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = w[j] + v[j];
        }
      };
      const uint32_t acc = ai & 1, aph = (ai >> 1) & 1;
      ++ai;
      const bool have = sg.kb1 > sg.kb0;
      const uint32_t taddr = tmem_base + acc * BN + (uint32_t(lq * 32) << 16);
      // TMEM chunk prefetch: the chunk loops take chunk c0 and issue c0 + CSTEP before the
      // stores of c0, so the TMEM read latency hides behind the previous chunk's global traffic
      uint32_t pf[CW];
      auto pf_issue = [&](int c) {
        if (have && c < c_end) tmem_ld16_issue(taddr + c, pf);
      };
      auto pf_take = [&](int c0, float (&v)[CW]) {
        tmem_ld16_wait(pf);
#pragma unroll
        for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(pf[j]);
        if (epf) pf_issue(c0 + CSTEP);
        else if (c0 + CSTEP < c_end) tmem_ld16_issue(taddr + c0 + CSTEP, pf), tmem_ld16_wait(pf);
      };
      if (has_other & 2) mbar_wait_sleep(&tmem_full[acc], aph);
      else mbar_wait(&tmem_full[acc], aph);
      if (ew == 0 && lane == 0 && ai == 1) trace_mark(tr, 5);
      tc_fence_after();

      if (sg.kind == SEG_PART) {
        pf_issue(c_begin);
#pragma unroll 1
        for (int c0 = c_begin; c0 < c_end; c0 += CSTEP) {
          float v[CW];
          if (have) {
            pf_take(c0, v);
            add_sum(c0, v);
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < CW / 4; ++j)
            __stcg(ws_ptr(ws, wslot(sg.slot), BN, c0, j, row), make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tmem_empty_lead + acc * 8);
        __threadfence();
        named_bar_sync(1, NEPI * 32);
        if (leader) flag_release(&flags[wslot(sg.slot)]);
        continue;
      }

      if (sg.kind == SEG_HEAD) {
        if (leader) {
          for (int j = 0; j < sg.n_parts; ++j) {
            unsigned* f = &flags[wslot(sg.slot + j)];
            long long t0 = clock64();
            uint32_t spins = 0;
            while (flag_acquire(f) == 0u) {
              if ((++spins & 1023u) == 0 && clock64() - t0 > (1ll << 35)) __trap();
            }
            *f = 0u;  // re-arm for the next launch (stream order separates launches)
          }
          __threadfence();
        }
        named_bar_sync(1, NEPI * 32);
      }

      const int p = sg.tp * PBM + int(rank) * BM + row;
      const int prow0 = sg.tp * PBM + int(rank) * BM + lq * 32;
      // needs-other stage (w_next = w - wd): its operand is fetched before the TMEM drain
      const int oe = pr.other_stage;
      const void* omap = pr.tmap_other;
      const bool o_tma = omap != nullptr;
      const uint32_t sbuf = smem_u32(out_stage + ew * NBOX * kOutStage);
      // epilogue descriptors in registers for the whole segment (the chunk loop stores through
      // generic pointers, so the compiler would otherwise re-load them from global per chunk)
      const int nout = 1 + pr.n_epi;
      float* obase[1 + kMaxEpi];
      int ors[1 + kMaxEpi], ocs[1 + kMaxEpi];  // element strides (host checks < 2^31)
      int eop[kMaxEpi];
      float esc[kMaxEpi];
      obase[0] = pr.out; ors[0] = int(pr.out_rs); ocs[0] = int(pr.out_cs);
#pragma unroll
      for (int e = 0; e < kMaxEpi; ++e) {
        const bool on = e < pr.n_epi;
        obase[1 + e] = on ? pr.epi[e].out : nullptr;
        ors[1 + e] = on ? int(pr.epi[e].out_rs) : 0;
        ocs[1 + e] = on ? int(pr.epi[e].out_cs) : 0;
        eop[e] = on ? pr.epi[e].op : EPI_NONE;
        esc[e] = on ? pr.epi[e].scale : 0.f;
      }
      const int PP = pr.P, QQ = pr.Q;
      const bool ostream = pr.out_stream != 0;
      // Store-order fast path: every output row-major and the only second operand TMA-staged.
      // The accumulator chunk is transposed once through smem and the whole elementwise chain
      // runs on the transposed values (the operand box already has that layout).
      bool fast = oe < 0 || o_tma;
#pragma unroll
      for (int e = 0; e <= kMaxEpi; ++e)
        if (e < nout) {
          fast = fast && ocs[e] == 1;
          if (e > 0 && epi_needs_other(eop[e - 1]) && e - 1 != oe) fast = false;
        }
      if (pr.tstore && (oe < 0 || o_tma)) {
        // TMA-store epilogue: the lane keeps its accumulator row; each stage's 32 x CW values
        // go to this warp's smem box for that output and one thread issues the bulk tensor
        // stores (clipped at the problem edges by the tensor maps).  No transpose, no per-lane
        // global stores.
        const uint64_t spol = policy_evict_first();  // outputs far larger than L2 (ostream)
        const uint32_t box_w = smem_u32(out_stage) + uint32_t(ew * NBOX) * kOutStage;
        const bool dbl = NBOX >= 2 * nout;  // two box sets: chunk k+1 fills while k's stores read
        pf_issue(c_begin);
#pragma unroll 1
        for (int c0 = c_begin; c0 < c_end; c0 += CSTEP) {
          const int q0 = sg.tq * BN + c0;
          const uint32_t box0 = box_w + (dbl ? box_half * uint32_t(nout) * kOutStage : 0u);
          float v[CW], o[CW];
          if (have) {
            pf_take(c0, v);
            add_sum(c0, v);
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = 0.f;
          }
          if (c0 + CSTEP >= c_end) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tmem_empty_lead + acc * 8);
          }
          if (q0 >= QQ) continue;
          if (sg.kind == SEG_HEAD) {
            for (int pp = 0; pp < sg.n_parts; ++pp) {
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float4 x = __ldcg(ws_ptr(ws, wslot(sg.slot + pp), BN, c0, j, row));
                v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
              }
            }
          }
          if (oe >= 0) {
            mbar_wait(obar(o_slot), o_phase);
            const uint32_t ob = obox(o_slot);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
              const float4 x = oread(ob, lane, j);
              o[4 * j] = x.x; o[4 * j + 1] = x.y; o[4 * j + 2] = x.z; o[4 * j + 3] = x.w;
            }
            if (++o_slot == uint32_t(ODEPTH)) { o_slot = 0; o_phase ^= 1; }
            __syncwarp();
            if (lane == 0) other_done();
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) o[j] = 0.f;
          }
          // the stores that last used these boxes have read them
          if (lane == 0) {
            if (dbl) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int e = 0; e <= kMaxEpi; ++e) {
            if (e >= nout) break;
            if (e > 0) epi_apply(eop[e - 1], v, o, esc[e - 1]);
            const uint32_t bx = box0 + uint32_t(e) * kOutStage;
            if constexpr (BF16) {
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v[4 * j], v[4 * j + 1]);
                const __nv_bfloat162 hi = __floats2bfloat162_rn(v[4 * j + 2], v[4 * j + 3]);
                asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(bx + lane * (CW * 2) + j * 8),
                             "r"(*reinterpret_cast<const uint32_t*>(&lo)), "r"(*reinterpret_cast<const uint32_t*>(&hi))
                             : "memory");
              }
            } else {
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) sts128(bx + box_off(lane, j), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = rnd<BF16>(v[j]);  // the next stage reads the stored value
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            for (int e = 0; e < nout; ++e) {
              const uint32_t bx = box0 + uint32_t(e) * kOutStage;
              if (ostream) tma_store_2d_hint(pr.tmap_out[e], bx, q0, prow0, spol);
              else asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(pr.tmap_out[e]),
                                "r"(bx), "r"(q0), "r"(prow0) : "memory");
            }
            bulk_commit();
          }
          box_half ^= 1u;
        }
        continue;
      }
      if (fast) {
        // Per-segment store state: row pointer of row (prow0 + lane/4), column 4*(lane%4), per
        // output, and the 8-row step.  The elementwise chain is matched against the fused
        // patterns the lowering emits (act, dact, act+seed, step+upd) so the hot loop is
        // straight-line code.
        const int c = lane & 3;
        long long dofs[1 + kMaxEpi];  // element offset of (row prow0 + lane/4, column 4c)
        long long st8[1 + kMaxEpi];
        bool vec_ok = true;
#pragma unroll
        for (int e = 0; e <= kMaxEpi; ++e) {
          dofs[e] = 0;
          st8[e] = 0;
          if (e < nout) {
            vec_ok = vec_ok && vec_aligned<BF16>(obase[e], 0) && ((ors[e] & 3) == 0);
            dofs[e] = (long long)(prow0 + (lane >> 2)) * ors[e] + c * 4;
            st8[e] = 8ll * ors[e];
          }
        }
        const bool rows_in = prow0 + 32 <= PP;
        const int n_epi = nout - 1;
        int chain = 5;  // generic
        if (n_epi == 0) chain = 0;
        else if (n_epi == 1 && eop[0] == EPI_TANH) chain = 1;
        else if (n_epi == 1 && eop[0] == EPI_DTANH) chain = 2;
        else if (n_epi == 2 && eop[0] == EPI_SCALE && eop[1] == EPI_SUB_OP && oe == 1) chain = 3;
        else if (n_epi == 2 && eop[0] == EPI_TANH && eop[1] == EPI_DTANH) chain = 4;
        const float s0 = esc[0];
        pf_issue(c_begin);
#pragma unroll 1
        for (int c0 = c_begin; c0 < c_end; c0 += CSTEP) {
          const int q0 = sg.tq * BN + c0;
          float v[CW];
          if (have) {
            pf_take(c0, v);
            add_sum(c0, v);
          } else {
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = 0.f;
          }
          if (c0 + CSTEP >= c_end) {
            // accumulator drained: hand it back to the MMA warp before the global traffic
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tmem_empty_lead + acc * 8);
          }
          if (q0 >= QQ) continue;
          if (sg.kind == SEG_HEAD) {
            for (int pp = 0; pp < sg.n_parts; ++pp) {
#pragma unroll
              for (int j = 0; j < CW / 4; ++j) {
                const float4 x = __ldcg(ws_ptr(ws, wslot(sg.slot + pp), BN, c0, j, row));
                v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < CW / 4; ++j) sts128(sbuf + box_off(lane, j), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          __syncwarp();
          float4 x[4], ox[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) x[i] = lds128(sbuf + box_off(i * 8 + (lane >> 2), c));
          if (oe >= 0) {
            mbar_wait(obar(o_slot), o_phase);
            const uint32_t ob = obox(o_slot);
#pragma unroll
            for (int i = 0; i < 4; ++i) ox[i] = oread(ob, i * 8 + (lane >> 2), c);
            if (++o_slot == uint32_t(ODEPTH)) { o_slot = 0; o_phase ^= 1; }
          }
          __syncwarp();  // transpose box and operand box free again
          if (oe >= 0 && lane == 0) other_done();
          const bool full_blk = vec_ok && rows_in && q0 + CW <= QQ;
          const int gq = q0 + c * 4;
          // store stage e's values, then round them as stored (the next stage reads the stored
          // value, like the unfused launch would)
          auto put = [&](int e) {
            if ((nost >> e) & 1) { round4<BF16>(x); return; }  // debug (27, mask): output e not stored
            const long long d0 = dofs[e] + q0;
            if (full_blk) {
#pragma unroll
              for (int i = 0; i < 4; ++i) st4<BF16>(obase[e], d0 + i * st8[e], x[i], ostream);
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (prow0 + i * 8 + (lane >> 2) >= PP) continue;
                const long long d = d0 + i * st8[e];
                if (vec_ok && gq + 4 <= QQ) {
                  st4<BF16>(obase[e], d, x[i], false);
                } else {
                  if (gq < QQ) st1<BF16>(obase[e], d, x[i].x);
                  if (gq + 1 < QQ) st1<BF16>(obase[e], d + 1, x[i].y);
                  if (gq + 2 < QQ) st1<BF16>(obase[e], d + 2, x[i].z);
                  if (gq + 3 < QQ) st1<BF16>(obase[e], d + 3, x[i].w);
                }
              }
            }
            round4<BF16>(x);
          };
          switch (chain) {
            case 0:
              put(0);
              break;
            case 1:
              put(0);
#pragma unroll
              for (int i = 0; i < 4; ++i) { x[i].x = tanhf(x[i].x); x[i].y = tanhf(x[i].y); x[i].z = tanhf(x[i].z); x[i].w = tanhf(x[i].w); }
              put(1);
              break;
            case 2:
              put(0);
              epi_apply4(EPI_DTANH, x, ox, 0.f);
              put(1);
              break;
            case 3:  // gw -> wd = lr * gw -> w_next = w - wd
              put(0);
#pragma unroll
              for (int i = 0; i < 4; ++i) { x[i].x *= s0; x[i].y *= s0; x[i].z *= s0; x[i].w *= s0; }
              put(1);
#pragma unroll
              for (int i = 0; i < 4; ++i) { x[i].x = ox[i].x - x[i].x; x[i].y = ox[i].y - x[i].y; x[i].z = ox[i].z - x[i].z; x[i].w = ox[i].w - x[i].w; }
              put(2);
              break;
            case 4:
              put(0);
#pragma unroll
              for (int i = 0; i < 4; ++i) { x[i].x = tanhf(x[i].x); x[i].y = tanhf(x[i].y); x[i].z = tanhf(x[i].z); x[i].w = tanhf(x[i].w); }
              put(1);
              epi_apply4(EPI_DTANH, x, ox, 0.f);
              put(2);
              break;
            default:
              put(0);
#pragma unroll
              for (int e = 1; e <= kMaxEpi; ++e) {
                if (e >= nout) break;
                epi_apply4(eop[e - 1], x, ox, esc[e - 1]);
                put(e);
              }
          }
        }
        continue;
      }
#pragma unroll 1
      for (int c0 = c_begin; c0 < c_end; c0 += CSTEP) {
        const int q0 = sg.tq * BN + c0;
        float o[CW];
        if (oe >= 0 && q0 < QQ) {
          if (o_tma) {
            // the box was requested ODEPTH chunks ahead; read my row, refill the slot
            mbar_wait(obar(o_slot), o_phase);
            const uint32_t ob = obox(o_slot);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
              const float4 x = oread(ob, lane, j);
              o[4 * j] = x.x; o[4 * j + 1] = x.y; o[4 * j + 2] = x.z; o[4 * j + 3] = x.w;
            }
            if (++o_slot == uint32_t(ODEPTH)) { o_slot = 0; o_phase ^= 1; }
            __syncwarp();
            if (lane == 0) other_done();
          } else {
            load_chunk<BF16>(pr.epi[oe].other, pr.epi[oe].o_rs, pr.epi[oe].o_cs, p, q0, PP, QQ, o);
          }
        }
        float v[CW];
        if (have) {
          tmem_ld16(taddr + c0, v);
          add_sum(c0, v);
        } else {
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = 0.f;
        }
        if (c0 + CSTEP >= c_end) {
          // accumulator drained: hand it back to the MMA warp before the global traffic
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_lead + acc * 8);
        }
        if (sg.kind == SEG_HEAD) {
          for (int pp = 0; pp < sg.n_parts; ++pp) {
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
              const float4 x = __ldcg(ws_ptr(ws, wslot(sg.slot + pp), BN, c0, j, row));
              v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
            }
          }
        }
        if (q0 >= QQ) continue;
#pragma unroll
        for (int e = 0; e <= kMaxEpi; ++e) {
          if (e >= nout) break;
          if (e > 0) {
            if (epi_needs_other(eop[e - 1]) && e - 1 != oe) {
              const EpiStage& st = pr.epi[e - 1];
              load_chunk<BF16>(st.other, st.o_rs, st.o_cs, p, q0, PP, QQ, o);
            }
            epi_apply(eop[e - 1], v, o, esc[e - 1]);
          }
          if (ocs[e] == 1) store_block<BF16>(sbuf, lane, v, obase[e], ors[e], prow0, q0, PP, QQ, ostream);
          else store_chunk<BF16>(obase[e], ors[e], ocs[e], p, q0, PP, QQ, v);  // swapped: lanes consecutive
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = rnd<BF16>(v[j]);  // the next stage reads the stored value
        }
      }
    }
  }
  if (warp >= 4 && warp < 4 + NEPI && lane == 0) bulk_wait<0>();  // TMA-store epilogue drained
  if (warp == 4 && lane == 0) trace_mark(tr, 6);
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // both CTAs done with the pair's TMEM and barriers
  else __syncthreads();
  if (dyn && threadIdx.x == 0 && rank == 0) {
    // every unit has fetched past the end: the last one re-arms the counter for the next launch
    const unsigned units = gridDim.x / (PAIR ? 2u : 1u);
    if (atomicAdd(&flags[1], 1u) == units - 1) {
      flags[0] = 0u;
      flags[1] = 0u;
      __threadfence();
    }
  }
  if (threadIdx.x == 0) trace_mark(tr, 7);
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

using KernelFn = void (*)(const GemmProblem*, const GemmSeg*, const int*, float*, unsigned*, int, int, int);

template <int BN, bool SPLIT, bool PAIR, bool BF16>
KernelFn pick(bool p_mn, bool q_mn) {
  if (!p_mn && !q_mn) return gemm_tf32_kernel<BN, false, false, SPLIT, PAIR, BF16>;
  if (!p_mn && q_mn) return gemm_tf32_kernel<BN, false, true, SPLIT, PAIR, BF16>;
  if (p_mn && !q_mn) return gemm_tf32_kernel<BN, true, false, SPLIT, PAIR, BF16>;
  return gemm_tf32_kernel<BN, true, true, SPLIT, PAIR, BF16>;
}

template <bool BF16>
KernelFn kernel_for_t(int bn, bool p_mn, bool q_mn, bool split, bool pair) {
  if (pair) {
    if (bn != 256 || split) throw std::runtime_error("gemm: CTA-pair tiles are 256 x 256 single-pass only");
    return pick<256, false, true, BF16>(p_mn, q_mn);
  }
  if (BF16 && split) throw std::runtime_error("gemm: 3xTF32 is an fp32-storage mode");
  constexpr bool S = !BF16;  // the split variants exist for fp32 storage only
  switch (bn) {
    case 32: return split ? pick<32, S, false, BF16>(p_mn, q_mn) : pick<32, false, false, BF16>(p_mn, q_mn);
    case 64: return split ? pick<64, S, false, BF16>(p_mn, q_mn) : pick<64, false, false, BF16>(p_mn, q_mn);
    case 128: return split ? pick<128, S, false, BF16>(p_mn, q_mn) : pick<128, false, false, BF16>(p_mn, q_mn);
    case 256:
      if (split) throw std::runtime_error("gemm: 3xTF32 tiles are at most 128 wide (TMEM chain sums)");
      return pick<256, false, false, BF16>(p_mn, q_mn);
  }
  throw std::runtime_error("gemm: unsupported tile width " + std::to_string(bn));
}

KernelFn kernel_for(int bn, bool p_mn, bool q_mn, bool split, bool pair, bool bf16) {
  return bf16 ? kernel_for_t<true>(bn, p_mn, q_mn, split, pair) : kernel_for_t<false>(bn, p_mn, q_mn, split, pair);
}

unsigned g_dbg_lbo = 0, g_dbg_sbo = 0;
bool g_no_tma_store = false;
int g_prefetch = -1;  // -1: default (off)
int g_stages = 0;     // 0: as many as fit
int g_sleep = 1;      // epilogue waits with nanosleep back-off
bool g_no_3d = false;
int g_other_promo = 0;     // L2 promotion of the epilogue operand map (0 none .. 3 256 B)
bool g_no_stream = false;  // disable evict-first stores / operand policies
const CUtensorMapL2promotion kOtherPromo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
bool g_no_pair = false;
int g_max_bn = 0;  // debug: cap the tile width
bool g_no_tma_out = false;
// A dedicated warp loads the epilogue operand boxes (fp32: bwd_w + update 3 % faster; bf16's
// small boxes run 25 % slower with the single loader, so bf16 keeps per-warp issue).
bool g_other_loader = true;  // debug (12,0) off / (12,1) on  // debug: per-lane global stores instead of TMA-store epilogues
int g_split_kb = 0;    // 3xTF32: k-blocks per scheduled segment (debug (13, n); 0 = unbounded)
int g_split_chain = 2; // 3xTF32: k-blocks per TMEM accumulation chain (debug (14, n); 0 = unbounded)
bool g_no_dyn = true;  // whole-tile schedules from a device tile counter: opt-in (10,0)
int g_odepth = 0;      // debug (15, n): operand ring depth n (0 = chosen from the smem budget)
int g_min_stages = 4;  // debug (16, n): mainloop stages the operand ring must leave
int g_ts_chain = 0;    // debug (18, n): TMA-store epilogue also for chains (n = 1 single, 2 double-buffered boxes)
int g_trace = 0;       // debug (22, 1): per-CTA launch timeline (tpx_debug_gemm_trace)
int g_whole = 0;       // debug (23, 1): whole tiles whenever there are no more tiles than groups (default: when >= 80 % of the groups get one)
int g_defer = 0;       // debug (24, 1): deferred stream-K fixup launch instead of in-kernel heads (measured slower: off)
// Long-K tile width: the widest tile whose count still leaves each tile cut into at most this
// many stream-K k-ranges, down to 128-wide tiles (the head sums the cut parts serially in its
// epilogue; weight-streaming M = 128 x 8192 x 8192: 4.6 cuts of 256-wide tiles 76 us, 2.3 cuts of
// 128-wide tiles 61 us)
int g_max_cuts = 3;   // debug (30, n)
int g_swap_below = 128;  // debug (29, n): compute the output transposed when M < n (and N >= 2M)
int g_stagger = 0;    // debug (28, us): odd units start late
int g_nostore = 0;    // debug (27, mask): fast-path epilogue skips the global stores of these outputs
int g_epi_pf = 1;     // debug (26, 0): epilogue TMEM chunks loaded on demand, not one ahead
int g_mn4d = 1;       // debug (25, 0): MN-major tf32 operands in the chunk-major stage layout
int g_rr_tiles = 1;    // debug (20, n): whole-tile schedules dealt round-robin (1, default) or in contiguous blocks (0)
int g_tq_block = 0;    // debug (21, n): tile list in blocks of n Q-tiles (0 = Q-tile major)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D tensor map over a row-major view: `inner` contiguous elements per row, `outer` rows
// `row_stride` elements apart, boxes of box_inner x box_outer.  fp32: 128-byte swizzle (32-byte
// atoms for MN-major tf32 operands); bf16: 128-byte swizzle.  `sw64` = the epilogue operand box
// (fp32: 64-byte swizzle; bf16: 32-byte rows, unswizzled).
void make_map(CUtensorMap* m, const float* base, long long inner, long long outer,
              long long row_stride, int box_inner, int box_outer, bool mn_major, bool sw64 = false,
              bool bf16 = false) {
  const int es = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  // a single row's stride is never used, but the encoder wants it 16-byte aligned
  const long long al = 16 / es;
  const long long rs = outer > 1 ? std::max<long long>(row_stride, inner) : (inner + al - 1) / al * al;
  cuuint64_t strides[1] = {(cuuint64_t)(rs * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = sw64 ? (bf16 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_64B)
                                : (mn_major && !bf16) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = encode_fn()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                           const_cast<float*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           sw,
                           // 64-byte operand rows: no promotion (a promoted 256 B line would be
                           // evicted, evict-first, before the next chunks use it)
                           sw64 ? kOtherPromo[g_other_promo & 3] : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

// 3-D map of an MN-major operand whose MN extent is a multiple of the 128-byte chunk (c = 32
// fp32 or 64 bf16 elements): (c MN elements, K rows, MN/c chunks), so one box of
// (c, c, nchunk) lands as nchunk swizzled chunks of c k-rows x 128 bytes.
void make_map_mn3d(CUtensorMap* m, const float* base, long long inner, long long outer,
                   long long row_stride, int nchunk, bool bf16 = false) {
  const int es = bf16 ? 2 : 4, c = 128 / es;
  cuuint64_t dims[3] = {(cuuint64_t)c, (cuuint64_t)outer, (cuuint64_t)(inner / c)};
  const long long rs = outer > 1 ? std::max<long long>(row_stride, inner) : inner;
  cuuint64_t strides[2] = {(cuuint64_t)(rs * es), 128};
  cuuint32_t box[3] = {(cuuint32_t)c, (cuuint32_t)c, (cuuint32_t)nchunk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<float*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed (" + std::to_string(int(r)) + ")");
}

// 4-D map of an MN-major tf32 operand (MN extent a multiple of 32, K a multiple of 4):
// (32 MN elements, 4 k rows, MN/32 chunks, K/4 k groups); a box of (32, 4, nchunk, bke/4)
// lands as bke/4 k groups, each holding its nchunk 512-byte atoms side by side.
void make_map_mn4d(CUtensorMap* m, const float* base, long long inner, long long outer,
                   long long row_stride, int nchunk, int bke) {
  cuuint64_t dims[4] = {32, 4, (cuuint64_t)(inner / 32), (cuuint64_t)(outer / 4)};
  const long long rs = std::max<long long>(row_stride, inner);
  cuuint64_t strides[3] = {(cuuint64_t)(rs * 4), 128, (cuuint64_t)(rs * 16)};
  cuuint32_t box[4] = {32, 4, (cuuint32_t)nchunk, (cuuint32_t)(bke / 4)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (4-D) failed (" + std::to_string(int(r)) + ")");
}

struct Role {
  const float* ptr;
  long long inner, outer, rs;
  bool mn;  // contiguous dim is the row (M/N) dim rather than K
};

inline bool epi_needs_other_host(int op) { return op >= EPI_ADD; }

struct SchedCol { int prob, tq, tp0, ntp, kb; };
struct SchedPiece { int group, kb0, kb1; };

}  // namespace

void gemm_debug_trace(unsigned long long* out, int n) {
  CUDA_CHECK(cudaMemcpyFromSymbol(out, g_gemm_trace, size_t(std::min(n, 320 * 8)) * 8));
}

void gemm_debug_mn_desc(unsigned lbo, unsigned sbo) {
  g_dbg_lbo = lbo;
  g_dbg_sbo = sbo;
  // debug switches: (1,1) direct epilogue stores/loads; (2, n) L2 prefetch distance n-1
  if (lbo == 1) g_no_tma_store = (sbo == 1);
  if (lbo == 2) g_prefetch = int(sbo) - 1;
  if (lbo == 4) g_stages = int(sbo);
  if (lbo == 5) g_sleep = (sbo != 2);  // (5,2) spin without back-off
  if (lbo == 6) g_no_pair = (sbo == 1);  // (6,1) single-CTA tiles only
  if (lbo == 7) g_other_promo = sbo > 0 ? int(sbo) - 1 : 0;  // (7,n) operand promotion n-1
  if (lbo == 8) g_no_stream = (sbo == 1);  // (8,1) no L2 streaming hints
  if (lbo == 9) g_max_bn = int(sbo);       // (9,n) tile width <= n
  if (lbo == 10) g_no_dyn = (sbo == 1);    // (10,0) dynamic / (10,1) static whole-tile schedules
  if (lbo == 11) g_no_tma_out = (sbo == 1);  // (11,1) per-lane global stores in the epilogue
  if (lbo == 12) g_other_loader = (sbo == 1);  // (12,0/1) operand-loader warp for fp32 epilogues
  if (lbo == 3) g_no_3d = (sbo == 1);  // (3,1) MN-major operands as 2-D boxes
  if (lbo == 13) g_split_kb = int(sbo);  // (13,n) 3xTF32 segments of <= n k-blocks (workspace sums)
  if (lbo == 14) g_split_chain = int(sbo) & 15;  // (14,n) 3xTF32 TMEM chains of n k-blocks
  if (lbo == 15) g_odepth = int(sbo);             // (15,n) epilogue operand ring depth n
  if (lbo == 16) g_min_stages = int(sbo);         // (16,n) keep >= n mainloop stages
  if (lbo == 18) g_ts_chain = int(sbo);           // (18,n) TMA-store chain epilogues
  if (lbo == 22) g_trace = int(sbo);              // (22,1) launch timeline
  if (lbo == 23) g_whole = int(sbo);              // (23,1) whole tiles instead of stream-K
  if (lbo == 24) g_defer = int(sbo);              // (24,n) deferred stream-K fixup
  if (lbo == 30) g_max_cuts = std::max(1, int(sbo));  // (30,n) stream-K cuts per tile (width rule)
  if (lbo == 29) g_swap_below = int(sbo);         // (29,n) swap threshold on M
  if (lbo == 28) g_stagger = int(sbo);            // (28,us) odd units start late
  if (lbo == 27) g_nostore = int(sbo);            // (27,mask) timing probe: outputs not stored
  if (lbo == 26) g_epi_pf = int(sbo);             // (26,0) no TMEM chunk prefetch
  if (lbo == 25) g_mn4d = int(sbo);               // (25,0) chunk-major MN-major stages
  if (lbo == 20) g_rr_tiles = int(sbo);           // (20,n) round-robin whole tiles
  if (lbo == 21) g_tq_block = int(sbo);           // (21,n) Q-tile blocks in the tile list
  if (lbo >= 1 && lbo <= 30) g_dbg_lbo = g_dbg_sbo = 0;  // (small lbo values are knobs, not strides)
}

bool gemm_view_ok(const MatView& v, bool bf16) {
  if (v.cs != 1) return false;
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) != 0) return false;
  if (v.rows > 1 && (v.rs % (bf16 ? 8 : 4)) != 0) return false;  // 16-byte row pitch (TMA)
  return true;
}

// Host tile scheduler.  A "column" is G P-tiles sharing one Q-tile of one problem; a group of
// G CTAs walks columns with CTA j of the group on P-tile (column base + j).  Units of work are
// (column, k-block); each group gets a contiguous, equal share of the units (stream-K) or, when
// there are plenty of columns, a contiguous run of whole columns.
GemmSchedule gemm_schedule(const std::vector<GemmProblem>& probs, int bn, int num_sms,
                           int force_groups, int max_kb, bool deferred) {
  GemmSchedule S;
  if (probs.empty()) return S;
  // group width: the P-tile count of small-M problems whose Q operand is large (streamed)
  int G = 1;
  bool same_tp = true;
  for (const auto& pr : probs) same_tp = same_tp && pr.tiles_p == probs[0].tiles_p;
  // (the streamed bytes of the whole batch: 8 sub-problems of 32 MB weights are streamed from
  // DRAM like one 256 MB weight -- tiled-on-one-GPU loop k3 fwd 0.16-0.20 ms with G = 1)
  double q_bytes = 0;
  for (const auto& pr : probs) q_bytes += 4.0 * double(pr.Q) * double(pr.K);
  if (same_tp && probs[0].tiles_p >= 2 && probs[0].tiles_p <= 8 && 2 * probs[0].tiles_p <= num_sms &&
      q_bytes > 32.0 * (1 << 20))
    G = probs[0].tiles_p;
  std::vector<SchedCol> cols;
  for (int pi = 0; pi < int(probs.size()); ++pi) {
    const GemmProblem& pr = probs[size_t(pi)];
    // Q-tile major, or (debug) blocks of B Q-tiles walked P-tile major inside, so the tiles in
    // flight share fewer operand panels
    const int B = g_tq_block > 0 ? g_tq_block : pr.tiles_q;
    for (int tb = 0; tb < pr.tiles_q; tb += B)
      for (int tp0 = 0; tp0 < pr.tiles_p; tp0 += G)
        for (int tq = tb; tq < std::min(pr.tiles_q, tb + B); ++tq)
          if (g_tq_block > 0) cols.push_back({pi, tq, tp0, std::min(G, pr.tiles_p - tp0), pr.kb_total});
    if (g_tq_block <= 0)
      for (int tq = 0; tq < pr.tiles_q; ++tq)
        for (int tp0 = 0; tp0 < pr.tiles_p; tp0 += G)
          cols.push_back({pi, tq, tp0, std::min(G, pr.tiles_p - tp0), pr.kb_total});
  }
  long long U = 0;
  for (const auto& c : cols) U += c.kb;
  int groups = std::max(1, num_sms / G);
  // at least ~8 k-blocks per group so a partial tile amortises its workspace round trip
  groups = int(std::min<long long>(groups, std::max<long long>(1, U / 8)));
  // A cut tile's head adds every partial of it serially: with few tiles and a long K, cutting
  // each tile into ~sqrt(k-block bytes / tile bytes * kb) parts balances the parts' operand
  // reads against the head's partial reads (e.g. a 64 x 27 grad_weight over 61696 columns).
  {
    const GemmProblem& p0 = probs[0];
    const double kblock = 4.0 * 32 * (128 + bn), tile = 4.0 * 128 * bn;
    const long long per_tile = std::max<long long>(1, (long long)std::ceil(std::sqrt(double(p0.kb_total) * kblock / tile)));
    groups = int(std::min<long long>(groups, std::max<long long>(1, (long long)cols.size() * per_tile)));
  }
  if (force_groups > 0) groups = force_groups;
  const int ncols = int(cols.size());
  // Bounded k-ranges (3xTF32): every tile's k range is cut into chunks of <= max_kb k-blocks,
  // each accumulated in TMEM on its own and summed in fp32 (round to nearest) by the head, in k
  // order.  The tensor cores' fp32 accumulation does not round to nearest, so its error grows
  // with the length of one accumulation chain; bounding the chain keeps the split products
  // fp32-accurate at any K (K = 8192: 4e-5 -> ~1e-6 normwise).
  bool chunked = false;
  for (const auto& c : cols) chunked = chunked || (max_kb > 0 && c.kb > max_kb);
  // whole tiles also when every column fits on its own group and >= 80 % of the groups get one:
  // no partial tiles, and the launch's tail is one epilogue (cfg2 fwd / bwd_x, 32 columns of 2
  // pair tiles on 37 groups: 107 -> 104 us); fewer columns keep stream-K (long-K conv products)
  const bool fill = ncols <= groups && (g_whole || 5LL * ncols >= 4LL * groups);
  const bool whole = !chunked && (ncols >= 8 * groups || ncols % groups == 0 || fill);
  if (whole) groups = std::min(groups, ncols);

  // pieces[col] = ordered (group, kb0, kb1)
  std::vector<std::vector<SchedPiece>> pieces(static_cast<size_t>(ncols));
  std::vector<std::vector<std::pair<int, int>>> group_pieces(static_cast<size_t>(groups));  // (col, piece idx)
  if (chunked) {
    // chunks dealt round-robin over the groups (equal k-work each), then each group's list
    // reordered partial chunks first: heads only wait for partials, which never wait
    long long i = 0;
    for (int c = 0; c < ncols; ++c) {
      const int kb = cols[size_t(c)].kb, nch = std::max(1, (kb + max_kb - 1) / max_kb);
      for (int j = 0; j < nch; ++j, ++i) {
        const int g = int(i % groups);
        pieces[size_t(c)].push_back({g, int((long long)kb * j / nch), int((long long)kb * (j + 1) / nch)});
        group_pieces[size_t(g)].push_back({c, j});
      }
    }
    for (auto& gp : group_pieces)
      std::stable_sort(gp.begin(), gp.end(), [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
        return (a.second > 0) > (b.second > 0);
      });
  } else if (whole && g_rr_tiles) {
    // tile c to group c mod groups: the groups walk the tile list side by side, so the tiles in
    // flight at any moment are neighbours (one problem, shared operand panels in L2)
    for (int c = 0; c < ncols; ++c) {
      const int g = c % groups;
      pieces[size_t(c)].push_back({g, 0, cols[size_t(c)].kb});
      group_pieces[size_t(g)].push_back({c, 0});
    }
  } else if (whole) {
    for (int g = 0; g < groups; ++g) {
      const int c0 = int((long long)ncols * g / groups), c1 = int((long long)ncols * (g + 1) / groups);
      for (int c = c0; c < c1; ++c) {
        pieces[size_t(c)].push_back({g, 0, cols[size_t(c)].kb});
        group_pieces[size_t(g)].push_back({c, 0});
      }
    }
  } else {
    long long col_start = 0;
    int c = 0;
    for (int g = 0; g < groups; ++g) {
      const long long u0 = U * g / groups, u1 = U * (g + 1) / groups;
      long long u = u0;
      while (u < u1) {
        while (u >= col_start + cols[size_t(c)].kb) col_start += cols[size_t(c++)].kb;
        const long long end = std::min(u1, col_start + cols[size_t(c)].kb);
        pieces[size_t(c)].push_back({g, int(u - col_start), int(end - col_start)});
        group_pieces[size_t(g)].push_back({c, int(pieces[size_t(c)].size()) - 1});
        u = end;
      }
    }
  }
  // slots: one per non-head piece per P-tile lane (deferred: one per piece, the head's first)
  deferred = deferred && !chunked && !whole;
  std::vector<int> slot_base(size_t(ncols) * size_t(G), -1);
  int nslots = 0;
  for (int c = 0; c < ncols; ++c) {
    const int np = int(pieces[size_t(c)].size());
    if (np <= 1) continue;
    for (int j = 0; j < cols[size_t(c)].ntp; ++j) {
      slot_base[size_t(c) * G + j] = nslots;
      nslots += deferred ? np : np - 1;
      if (deferred)
        S.fixups.push_back({cols[size_t(c)].prob, cols[size_t(c)].tp0 + j, cols[size_t(c)].tq, slot_base[size_t(c) * G + j], np});
    }
  }
  S.deferred = deferred;
  S.grid = groups * G;
  S.seg_off.assign(size_t(S.grid) + 1, 0);
  for (int g = 0; g < groups; ++g) {
    for (int j = 0; j < G; ++j) {
      const int cta = g * G + j;
      for (const auto& cp : group_pieces[size_t(g)]) {
        const SchedCol& col = cols[size_t(cp.first)];
        if (j >= col.ntp) continue;
        const auto& ps = pieces[size_t(cp.first)];
        const SchedPiece& pc = ps[size_t(cp.second)];
        GemmSeg sg;
        sg.prob = col.prob;
        sg.tp = col.tp0 + j;
        sg.tq = col.tq;
        sg.kb0 = pc.kb0;
        sg.kb1 = pc.kb1;
        if (ps.size() == 1) {
          sg.kind = SEG_WHOLE;
        } else if (deferred) {  // every piece a partial slot, in k order from the head's
          sg.kind = SEG_PART;
          sg.slot = slot_base[size_t(cp.first) * G + j] + cp.second;
        } else if (cp.second == 0) {
          sg.kind = SEG_HEAD;
          sg.slot = slot_base[size_t(cp.first) * G + j];
          sg.n_parts = int(ps.size()) - 1;
        } else {
          sg.kind = SEG_PART;
          sg.slot = slot_base[size_t(cp.first) * G + j] + cp.second - 1;
        }
        S.segs.push_back(sg);
      }
      S.seg_off[size_t(cta) + 1] = int(S.segs.size());
    }
  }
  S.nslots = nslots;
  S.group = G;
  S.stream_k = !whole;
  (void)bn;
  return S;
}

GemmLaunch gemm_prepare(const std::vector<GemmSpec>& specs, int num_sms, bool split) {
  if (specs.empty()) throw std::runtime_error("gemm: empty batch");
  GemmLaunch g;
  g.split = split;
  const GemmSpec& s0 = specs[0];
  g.bf16 = s0.bf16;
  const bool bf = g.bf16;
  const int mnc = bf ? 64 : 32, bke = bf ? 64 : 32;  // MN-major chunk / k-block (elements)
  for (const auto& s : specs)
    if (s.bf16 != bf) throw std::runtime_error("gemm: mixed storage types in one batch");
  const long long M0 = s0.ta ? s0.a.cols : s0.a.rows;
  const long long N0 = s0.tb ? s0.b.rows : s0.b.cols;
  g.swap = (M0 < g_swap_below && N0 >= 2 * M0);
  const long long Q0 = g.swap ? M0 : N0;
  g.bn = Q0 <= 32 ? 32 : Q0 <= 64 ? 64 : Q0 <= 128 ? 128 : 256;
  // an MN-major bf16 Q operand is staged in 64-element (128-byte) chunks: BN >= 64
  const bool q_mn0 = g.swap ? s0.ta : !s0.tb;
  const int min_bn = (s0.bf16 && q_mn0) ? 64 : 32;
  g.bn = std::max(g.bn, min_bn);
  if (split) g.bn = std::min(g.bn, 128);  // 3xTF32: TMEM holds 2 accumulators + the chain sums
  {
    // Tile width from the tile count: the widest tile that still gives every SM work.  Short-K
    // (epilogue-bound) problems want a tile per CTA; long-K ones are balanced by stream-K and
    // keep wide tiles while each tile is cut into at most ~5 k-ranges.
    long long kmax = 0;
    for (const auto& s : specs) kmax = std::max<long long>(kmax, s.ta ? s.a.rows : s.a.cols);
    const long long kb = (kmax + (s0.bf16 ? 63 : 31)) / (s0.bf16 ? 64 : 32);
    auto tiles = [&](int bn) {
      const long long pe = g.swap ? N0 : M0;
      const bool pair = !split && !g_no_pair && bn == 256 && pe >= 256 && num_sms >= 4 && (pe % 256 == 0 || pe >= 2048);
      const long long pbm = pair ? 256 : 128;
      long long t = 0;
      for (const auto& s : specs) {
        const long long M = s.ta ? s.a.cols : s.a.rows, N = s.tb ? s.b.rows : s.b.cols;
        const long long P = g.swap ? N : M, Q = g.swap ? M : N;
        t += ((P + pbm - 1) / pbm) * ((Q + bn - 1) / bn);
      }
      return std::make_pair(t, pair ? num_sms / 2 : num_sms);
    };
    auto widest = [&](int cuts) {
      int pick = g.bn;
      for (int bn = g.bn; bn >= min_bn; bn /= 2) {
        pick = bn;
        const auto tu = tiles(bn);
        const long long need = kb <= 16 ? tu.second : std::max(1, tu.second / cuts);
        if (tu.first >= need) break;
      }
      return pick;
    };
    // At most 5 cuts per tile. A single row of P tiles (weight streaming: M <= 128 against a
    // wide weight) takes at most g_max_cuts while that keeps tiles >= 128 wide: its heads' serial
    // partial sums are the launch's tail. Several P-tile rows (conv grad_weight: P = 256..384,
    // operand-traffic bound) keep the wide tiles (128-wide: AlexNet-style conv step +0.6 ms).
    const int pick5 = widest(5);
    const long long p_ext = g.swap ? N0 : M0;
    g.bn = p_ext <= BM ? std::max(widest(g_max_cuts), std::min(pick5, 128)) : pick5;
  }
  if (g_max_bn > 0) g.bn = std::max(min_bn, std::min(g.bn, g_max_bn));
  g.nprob = int(specs.size());
  // CTA pairs (256 x 256 tiles, half the operand bytes per SM) for wide TF32 problems
  const long long P0 = g.swap ? N0 : M0;
  // (a P extent that is not a multiple of 256 would leave half of its last pair tile idle)
  g.pair = !split && !g_no_pair && g.bn == 256 && P0 >= 256 && num_sms >= 4 && (P0 % 256 == 0 || P0 >= 2048);
  const int pbm = g.pair ? 2 * BM : BM;
  const int bnh = g.pair ? g.bn / 2 : g.bn;  // B columns one CTA stages (its TMA box)

  std::vector<CUtensorMap> maps(2 * specs.size());
  std::vector<CUtensorMap> store_maps;  // epilogue operand maps
  std::vector<std::pair<int, int>> store_idx;  // (problem, output index)
  std::vector<GemmProblem>& probs = g.host_problems;
  probs.resize(specs.size());
  // loader-warp operand boxes (fp32, 8 epilogue warps, static schedules, Q in whole 32-column
  // boxes so both warps of a lane quarter consume every box)
  g.oloader = !bf && !split && g_other_loader && g_no_dyn;
  for (const auto& s : specs) g.oloader = g.oloader && ((g.swap ? (s.ta ? s.a.cols : s.a.rows) : (s.tb ? s.b.rows : s.b.cols)) % 32 == 0);
  for (size_t i = 0; i < specs.size(); ++i) {
    const GemmSpec& s = specs[i];
    if (!gemm_view_ok(s.a, bf) || !gemm_view_ok(s.b, bf))
      throw std::runtime_error("gemm: operand view is not TMA-compatible");
    const long long M = s.ta ? s.a.cols : s.a.rows;
    const long long K = s.ta ? s.a.rows : s.a.cols;
    const long long Kb = s.tb ? s.b.cols : s.b.rows;
    const long long N = s.tb ? s.b.rows : s.b.cols;
    if (K != Kb) throw std::runtime_error("gemm: matmul inner extents differ");
    Role ra{s.a.ptr, s.a.cols, s.a.rows, s.a.rs, s.ta};   // rows = M (or K when ta)
    Role rb{s.b.ptr, s.b.cols, s.b.rows, s.b.rs, !s.tb};  // rows = N (or K when !tb)
    const Role& rp = g.swap ? rb : ra;
    const Role& rq = g.swap ? ra : rb;
    if (i == 0) {
      g.p_mn = rp.mn;
      g.q_mn = rq.mn;
    } else if (g.p_mn != rp.mn || g.q_mn != rq.mn) {
      throw std::runtime_error("gemm: mixed operand majorness in one batch");
    }
    GemmProblem& pr = probs[i];
    auto mn4d_ok = [&](const Role& r) { return !bf && g_mn4d && r.mn && r.inner % 32 == 0 && r.outer % 4 == 0 && r.outer >= 4; };
    if (mn4d_ok(rp)) {
      make_map_mn4d(&maps[2 * i], rp.ptr, rp.inner, rp.outer, rp.rs, BM / 32, bke);
      pr.a4d = 1;
      pr.a_lbo = 512, pr.a_sbo = 512u * (BM / 32), pr.a_kstep = 2 * pr.a_sbo;
    } else if (rp.mn && rp.inner % mnc == 0 && !g_no_3d) {
      make_map_mn3d(&maps[2 * i], rp.ptr, rp.inner, rp.outer, rp.rs, BM / mnc, bf);
      pr.a3d = 1;
    } else {
      make_map(&maps[2 * i], rp.ptr, rp.inner, rp.outer, rp.rs, rp.mn ? mnc : bke, rp.mn ? bke : BM, rp.mn,
               false, bf);
    }
    if (mn4d_ok(rq)) {
      make_map_mn4d(&maps[2 * i + 1], rq.ptr, rq.inner, rq.outer, rq.rs, bnh / 32, bke);
      pr.b4d = 1;
      pr.b_lbo = 512, pr.b_sbo = 512u * (bnh / 32), pr.b_kstep = 2 * pr.b_sbo;
    } else if (rq.mn && rq.inner % mnc == 0 && !g_no_3d) {
      make_map_mn3d(&maps[2 * i + 1], rq.ptr, rq.inner, rq.outer, rq.rs, bnh / mnc, bf);
      pr.b3d = 1;
    } else {
      make_map(&maps[2 * i + 1], rq.ptr, rq.inner, rq.outer, rq.rs, rq.mn ? mnc : bke, rq.mn ? bke : bnh,
               rq.mn, false, bf);
    }
    pr.P = int(g.swap ? N : M);
    pr.Q = int(g.swap ? M : N);
    pr.K = int(K);
    pr.tiles_p = int((pr.P + pbm - 1) / pbm);
    pr.tiles_q = int((pr.Q + g.bn - 1) / g.bn);
    pr.kb_total = int((K + bke - 1) / bke);
    pr.out = s.c;
    pr.out_rs = g.swap ? s.c_cs : s.c_rs;
    pr.out_cs = g.swap ? s.c_rs : s.c_cs;
    if (g_dbg_lbo) pr.a_lbo = pr.b_lbo = g_dbg_lbo;
    if (g_dbg_sbo) pr.a_sbo = pr.b_sbo = g_dbg_sbo;
    pr.n_epi = s.n_epi;
    for (int e = 0; e < s.n_epi; ++e) {
      pr.epi[e] = s.epi[e];
      if (g.swap) {
        std::swap(pr.epi[e].o_rs, pr.epi[e].o_cs);
        std::swap(pr.epi[e].out_rs, pr.epi[e].out_cs);
      }
    }
    // TMA load map for the epilogue operand (row-major, 16-byte aligned base and pitch)
    auto storable = [&](const float* b, long long rs, long long cs) {
      return b && cs == 1 && (reinterpret_cast<uintptr_t>(b) & 15) == 0 && (pr.P == 1 || rs % (bf ? 8 : 4) == 0);
    };
    for (int e = 0; e < s.n_epi; ++e) {
      if (!epi_needs_other_host(pr.epi[e].op)) continue;
      pr.other_stage = e;
      if (!g_no_tma_store && storable(pr.epi[e].other, pr.epi[e].o_rs, pr.epi[e].o_cs)) {
        store_maps.emplace_back();
        if (g.oloader)  // 32 x 32 boxes, 128-byte rows (two warps' chunks)
          make_map(&store_maps.back(), pr.epi[e].other, pr.Q, pr.P, pr.epi[e].o_rs, 2 * CW, 32, false, false, bf);
        else
          make_map(&store_maps.back(), pr.epi[e].other, pr.Q, pr.P, pr.epi[e].o_rs, CW, 32, false, true, bf);
        store_idx.push_back({int(i), 1 + kMaxEpi});
        g.other_smem = true;
      }
      break;
    }
    // TMA-store epilogue for a lone row-major, 16-byte-pitched output (measured: faster for
    // plain products, e.g. the conv grad_input columns; slower than the per-lane stores when a
    // chain of stages shares the epilogue smem with the operand ring)
    bool ts = !g_no_tma_out && (s.n_epi == 0 || g_ts_chain > 0);
    for (int e = 0; e <= s.n_epi; ++e) {
      const float* b = e == 0 ? pr.out : pr.epi[e - 1].out;
      const long long rs = e == 0 ? pr.out_rs : pr.epi[e - 1].out_rs, cs = e == 0 ? pr.out_cs : pr.epi[e - 1].out_cs;
      ts = ts && storable(b, rs, cs);
    }
    if (ts) {
      for (int e = 0; e <= s.n_epi; ++e) {
        const float* b = e == 0 ? pr.out : pr.epi[e - 1].out;
        const long long rs = e == 0 ? pr.out_rs : pr.epi[e - 1].out_rs;
        store_maps.emplace_back();
        make_map(&store_maps.back(), b, pr.Q, pr.P, rs, CW, 32, false, true, bf);
        store_idx.push_back({int(i), e});
      }
      pr.tstore = 1;
      const int bufs = (s.n_epi > 0 && (g_ts_chain == 1 || 2 * (1 + s.n_epi) > 7)) ? 1 : 2;  // (NBOX: 3 bits)
      g.nbox = std::max(g.nbox, bufs * (1 + s.n_epi));  // (double-buffered) boxes
    }
    auto small = [](long long x) { return x >= 0 && x < (1ll << 31); };
    bool ok = small(pr.out_rs) && small(pr.out_cs);
    for (int e = 0; e < s.n_epi; ++e) ok = ok && small(pr.epi[e].out_rs) && small(pr.epi[e].out_cs);
    if (!ok) throw std::runtime_error("gemm: output strides exceed 2^31 elements");
    g.flops += 2.0 * double(M) * double(N) * double(K);
    const double es = bf ? 2.0 : 4.0;
    g.min_bytes += es * double(M * K + K * N + M * N * (1 + s.n_epi));
    for (int e = 0; e < s.n_epi; ++e)
      if (s.epi[e].op >= EPI_ADD) g.min_bytes += es * double(M * N);
  }
  // L2 policy: operands re-read by many tiles and small enough to stay resident are kept
  // (evict_last); large streamed ones (a weight read once per step) and epilogue outputs far
  // larger than L2 are evict_first, so they do not push the reused operands out.
  {
    double pb = 0, qb = 0, ob = 0;
    for (size_t i = 0; i < probs.size(); ++i) {
      pb += 4.0 * probs[i].P * double(probs[i].K);
      qb += 4.0 * probs[i].Q * double(probs[i].K);
      ob += 4.0 * probs[i].P * double(probs[i].Q) * (1 + probs[i].n_epi);
    }
    const double kStream = 48.0 * (1 << 20), kOutStream = 64.0 * (1 << 20);
    for (auto& pr : probs) {
      pr.a_stream = pb > kStream && !g_no_stream;
      pr.b_stream = qb > kStream && !g_no_stream;
      pr.out_stream = ob > kOutStream && !g_no_stream;
    }
  }
  g.sched = gemm_schedule(probs, g.bn, g.pair ? num_sms / 2 : num_sms, 0, split ? g_split_kb : 0);
  if (g.sched.stream_k && g_defer && !split && !bf) {
    // deferred fixup: row-major outputs whose epilogue views share the product's layout, and at
    // most kMaxIn pieces per tile (the fixup is one ordered n-ary sum + the chain)
    bool ok = g.bn % 4 == 0;
    for (const auto& pr : probs) {
      ok = ok && pr.out_cs == 1 && pr.Q % 4 == 0;
      for (int e = 0; e < pr.n_epi; ++e)
        ok = ok && pr.epi[e].out_cs == 1 && pr.epi[e].out_rs == pr.out_rs &&
             (!pr.epi[e].other || (pr.epi[e].o_cs == 1 && pr.epi[e].o_rs == pr.out_rs));
    }
    int most = 0;
    for (int c = 0, i = 0; i < int(g.sched.segs.size()); ++i) {
      (void)c;
      if (g.sched.segs[size_t(i)].kind == SEG_HEAD) most = std::max(most, g.sched.segs[size_t(i)].n_parts + 1);
    }
    if (ok && most <= kMaxIn)
      g.sched = gemm_schedule(probs, g.bn, g.pair ? num_sms / 2 : num_sms, 0, 0, true);
  }
  if (!g.sched.stream_k && !g_no_dyn) {
    // Whole tiles only: hand them out in order from a device counter instead of fixed per-CTA
    // lists, so SMs that run ahead (less contention, nearer memory) take more tiles and the
    // launch ends with the slowest SM's last tile, not its share.  Order: (problem, tq, tp), so
    // the tiles in flight at any moment share their Q panels and sweep the P operand.
    std::vector<GemmSeg> order;
    for (int pi = 0; pi < int(probs.size()); ++pi)
      for (int tq = 0; tq < probs[size_t(pi)].tiles_q; ++tq)
        for (int tp = 0; tp < probs[size_t(pi)].tiles_p; ++tp) {
          GemmSeg sg;
          sg.prob = pi;
          sg.tp = tp;
          sg.tq = tq;
          sg.kb0 = 0;
          sg.kb1 = probs[size_t(pi)].kb_total;
          sg.kind = SEG_WHOLE;
          order.push_back(sg);
        }
    g.sched.segs = order;
    g.sched.seg_off = {0, int(order.size())};
    g.sched.dynamic = true;
    const int units = g.pair ? num_sms / 2 : num_sms;
    g.sched.grid = std::max(1, std::min<int>(units, int(order.size())));
  }
  g.units = g.sched.grid * (g.pair ? 2 : 1);
  const size_t halves = size_t(g.sched.nslots) * (g.pair ? 2 : 1);  // one BM x BN slot per CTA
  g.ws_floats = halves * BM * g.bn;
  if (g.sched.nslots) {
    CUDA_CHECK(cudaMalloc(&g.d_ws, g.ws_floats * sizeof(float)));
    CUDA_CHECK(cudaMalloc(&g.d_flags, halves * sizeof(unsigned)));
    CUDA_CHECK(cudaMemset(g.d_flags, 0, halves * sizeof(unsigned)));
  } else if (g.sched.dynamic) {
    CUDA_CHECK(cudaMalloc(&g.d_flags, 2 * sizeof(unsigned)));  // tile counter, finished units
    CUDA_CHECK(cudaMemset(g.d_flags, 0, 2 * sizeof(unsigned)));
  }
  if (g.sched.deferred) {
    // per cut tile (and CTA half of a pair tile): out = sum of its k-ordered partial slots, then
    // the problem's epilogue chain -- rows walked fastest so the slot reads are coalesced
    const int PBM = g.pair ? 2 * BM : BM;
    for (const auto& f : g.sched.fixups) {
      const GemmProblem& pr = probs[size_t(f.prob)];
      for (int half = 0; half < (g.pair ? 2 : 1); ++half) {
        const long long r0 = (long long)f.tp * PBM + half * BM, c0 = (long long)f.tq * g.bn;
        if (r0 >= pr.P || c0 >= pr.Q) continue;
        const long long nr = std::min<long long>(BM, pr.P - r0), nc = std::min<long long>(g.bn, pr.Q - c0);
        auto view3 = [&](const float* base, long long st_c4, long long st_r) {
          StridedView v;
          v.ptr = const_cast<float*>(base);
          v.rank = 3;
          v.shape[0] = nc / 4; v.shape[1] = nr; v.shape[2] = 4;
          v.st[0] = st_c4; v.st[1] = st_r; v.st[2] = 1;
          return v;
        };
        const StridedView out = view3(pr.out + r0 * pr.out_rs + c0, 4, pr.out_rs);
        std::vector<StridedView> parts;
        for (int i = 0; i < f.n_parts; ++i) {
          const long long slot = (long long)(g.pair ? 2 * (f.slot0 + i) + half : f.slot0 + i);
          parts.push_back(view3(g.d_ws + slot * BM * g.bn, 4LL * BM, 4));
        }
        NaryDesc d = nary_desc(NARY_SUM, out, parts, 0.f, 4);
        for (int e = 0; e < pr.n_epi; ++e) {
          const EpiStage& st = pr.epi[e];
          const StridedView eo = view3(st.out + r0 * st.out_rs + c0, 4, st.out_rs);
          StridedView ot;
          if (st.other) ot = view3(st.other + r0 * st.o_rs + c0, 4, st.o_rs);
          if (!nary_add_chain(d, out, st.op, st.scale, eo, st.other ? &ot : nullptr, 4))
            throw std::runtime_error("gemm: deferred fixup cannot chain the epilogue");
        }
        g.fixup.descs.push_back(d);
      }
    }
    nary_prepare(g.fixup);
  }
  const size_t nload = maps.size();
  maps.insert(maps.end(), store_maps.begin(), store_maps.end());
  CUDA_CHECK(cudaMalloc(&g.d_tmaps, maps.size() * sizeof(CUtensorMap)));
  CUDA_CHECK(cudaMemcpy(g.d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  for (size_t i = 0; i < probs.size(); ++i) {
    probs[i].tmap_a = static_cast<CUtensorMap*>(g.d_tmaps) + 2 * i;
    probs[i].tmap_b = static_cast<CUtensorMap*>(g.d_tmaps) + 2 * i + 1;
  }
  for (size_t j = 0; j < store_idx.size(); ++j) {
    GemmProblem& pr = probs[size_t(store_idx[j].first)];
    const void* m = static_cast<CUtensorMap*>(g.d_tmaps) + nload + j;
    if (store_idx[j].second == 1 + kMaxEpi) pr.tmap_other = m;
    else pr.tmap_out[store_idx[j].second] = m;
  }
  CUDA_CHECK(cudaMalloc(&g.d_problems, probs.size() * sizeof(GemmProblem)));
  CUDA_CHECK(cudaMemcpy(g.d_problems, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  CUDA_CHECK(cudaMalloc(&g.d_segs, g.sched.segs.size() * sizeof(GemmSeg) + 16));
  CUDA_CHECK(cudaMemcpy(g.d_segs, g.sched.segs.data(), g.sched.segs.size() * sizeof(GemmSeg), cudaMemcpyHostToDevice));
  CUDA_CHECK(cudaMalloc(&g.d_seg_off, g.sched.seg_off.size() * sizeof(int)));
  CUDA_CHECK(cudaMemcpy(g.d_seg_off, g.sched.seg_off.data(), g.sched.seg_off.size() * sizeof(int), cudaMemcpyHostToDevice));
  const int bn_stage = g.pair ? g.bn / 2 : g.bn;  // B columns staged per CTA
  // operand ring as deep as possible while the mainloop keeps >= 3 stages (>= 1 box)
  g.odepth = 0;
  if (g.other_smem) {
    // deepest operand ring that keeps the mainloop's depth (>= 4 stages where possible)
    g.odepth = 1;
    const int want = std::min(g_min_stages, stages_for(bn_stage, split, 1, g.nbox));
    for (int d = kOtherDepth; d > 1; --d)
      if (stages_for(bn_stage, split, d, g.nbox) >= std::max(3, want)) { g.odepth = d; break; }
    if (g_odepth > 0) g.odepth = std::min(g_odepth, kOtherDepth);
  }
  g.stages = stages_for(bn_stage, split, g.odepth, g.nbox);
  if (g_stages > 0) g.stages = std::min(g.stages, g_stages);
  if (g.stages < 1) throw std::runtime_error("gemm: tile does not fit in shared memory");
  g.smem_bytes = smem_for(bn_stage, split, g.odepth, g.stages, g.nbox);
  g.prefetch = g_prefetch >= 0 ? g_prefetch : 0;
  g.threads = threads_for(split);
  KernelFn fn = kernel_for(g.bn, g.p_mn, g.q_mn, split, g.pair, g.bf16);
  // the attribute is per function and launches of one instantiation differ in smem: allow the max
  CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemMax)));
  return g;
}

void gemm_run(const GemmLaunch& g, cudaStream_t stream) {
  KernelFn fn = kernel_for(g.bn, g.p_mn, g.q_mn, g.split, g.pair, g.bf16);
  const GemmProblem* probs = static_cast<const GemmProblem*>(g.d_problems);
  const GemmSeg* segs = static_cast<const GemmSeg*>(g.d_segs);
  const int flags = (g_trace ? 1 << 16 : 0) | (g_epi_pf ? 0 : 1 << 17) | ((g_nostore & 7) << 18) | ((g_stagger & 63) << 21) | (g.other_smem ? 1 : 0) | (g_sleep ? 2 : 0) | (g.odepth << 4) | (g.sched.dynamic ? 128 : 0) | (g.nbox << 8) |
                    (g.other_smem && g.oloader && !g.sched.dynamic ? 2048 : 0) | (g.split ? (g_split_chain & 15) << 12 : 0);
  if (g.pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(2 * g.sched.grid));
    cfg.blockDim = dim3(unsigned(g.threads));
    cfg.dynamicSmemBytes = g.smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, probs, segs, static_cast<const int*>(g.d_seg_off), g.d_ws,
                                  g.d_flags, g.stages, g.prefetch, flags));
  } else {
    fn<<<g.sched.grid, g.threads, g.smem_bytes, stream>>>(probs, segs, g.d_seg_off, g.d_ws, g.d_flags,
                                                          g.stages, g.prefetch, flags);
  }
  CUDA_CHECK(cudaGetLastError());
  if (g.sched.deferred) nary_run(g.fixup, stream);
}

void gemm_free(GemmLaunch& g) {
  nary_free(g.fixup);
  if (g.d_problems) cudaFree(g.d_problems);
  if (g.d_tmaps) cudaFree(g.d_tmaps);
  if (g.d_ws) cudaFree(g.d_ws);
  if (g.d_flags) cudaFree(g.d_flags);
  if (g.d_segs) cudaFree(g.d_segs);
  if (g.d_seg_off) cudaFree(g.d_seg_off);
  g = GemmLaunch{};
}

}  // namespace tpx
