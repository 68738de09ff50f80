// tcgen05 tile GEMM (kind::tf32, fp32 storage).  See gemm.h.
//
// Per CTA: one 128 x BN output tile (optionally one K-split of it).  Warp roles:
//   warp 0 lane 0  TMA producer    (cp.async.bulk.tensor -> 128B-swizzled smem ring)
//   warp 1 lane 0  MMA issuer      (tcgen05.mma.cta_group::1.kind::tf32, accum in TMEM)
//   warp 2         TMEM allocator  (BN fp32 columns x 128 lanes)
//   warps 4..7     epilogue        (tcgen05.ld -> registers -> fused elementwise -> global)
// Split-K partials go to a workspace; the last-arriving split (atomic ticket) sums all of
// them in split order (deterministic) and runs the epilogue.
#include "gemm.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "ptx.cuh"
#include "util.h"

namespace tpx {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block = one 128-byte swizzle row

// Operand bytes of one k-block; a split (3xTF32) stage also holds the low parts.
__host__ __device__ constexpr uint32_t operand_bytes(int bn) { return uint32_t(BM * BK * 4 + bn * BK * 4); }
__host__ __device__ constexpr uint32_t stage_bytes(int bn, bool split) {
  return operand_bytes(bn) * (split ? 2u : 1u);
}
__host__ __device__ constexpr int stages_for(int bn, bool split) {
  return int((192u * 1024u) / stage_bytes(bn, split)) > 8 ? 8 : int((192u * 1024u) / stage_bytes(bn, split));
}
constexpr size_t smem_for(int bn, bool split) {
  return size_t(stages_for(bn, split)) * stage_bytes(bn, split) + 1024 + 256;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ float epi_apply(int op, float prev, float other, float s) {
  switch (op) {
    case EPI_TANH: return tanhf(prev);
    case EPI_DTANH: {
      float t = tanhf(prev);
      return 1.0f - t * t;
    }
    case EPI_SCALE: return s * prev;
    case EPI_ADD: return prev + other;
    case EPI_SUB_PO: return prev - other;
    case EPI_SUB_OP: return other - prev;
    default: return prev;
  }
}

__device__ __forceinline__ bool epi_needs_other(int op) { return op >= EPI_ADD; }

// Store 32 consecutive columns [q0, q0+32) of row p.
__device__ __forceinline__ void store_chunk(float* base, long long rs, long long cs, int p,
                                            int q0, int P, int Q, const float (&v)[32]) {
  if (p >= P) return;
  float* row = base + (long long)p * rs;
  if (cs == 1 && q0 + 32 <= Q && ((reinterpret_cast<uintptr_t>(row + q0) & 15) == 0)) {
    float4* d = reinterpret_cast<float4*>(row + q0);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (q0 + j < Q) row[(long long)(q0 + j) * cs] = v[j];
  }
}

__device__ __forceinline__ void load_chunk(const float* base, long long rs, long long cs, int p,
                                           int q0, int P, int Q, float (&v)[32]) {
  if (p >= P) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.f;
    return;
  }
  const float* row = base + (long long)p * rs;
  if (cs == 1 && q0 + 32 <= Q && ((reinterpret_cast<uintptr_t>(row + q0) & 15) == 0)) {
    const float4* s = reinterpret_cast<const float4*>(row + q0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 t = __ldg(s + j);
      v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (q0 + j < Q) ? __ldg(row + (long long)(q0 + j) * cs) : 0.f;
  }
}

// SPLIT = 3xTF32: every fp32 operand x = hi + lo with hi = tf32_rna(x), lo = x - hi (exact);
// D += lo_A*hi_B + hi_A*lo_B + hi_A*hi_B.  The split is done in shared memory by warps 2..7
// (idle during the mainloop) between the TMA landing and the MMA issue.
template <int BN, bool P_MN, bool Q_MN, bool SPLIT>
__global__ void __launch_bounds__(256, 1)
    gemm_tf32_kernel(const GemmProblem* __restrict__ probs, int nprob) {
  constexpr int STAGES = stages_for(BN, SPLIT);
  constexpr uint32_t A_BYTES = BM * BK * 4;
  constexpr uint32_t OPB = operand_bytes(BN);
  constexpr uint32_t STAGE = stage_bytes(BN, SPLIT);
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t IDESC = (1u << 4)                 // D format f32
                             | (2u << 7) | (2u << 10)  // A, B format tf32
                             | (uint32_t(P_MN) << 15) | (uint32_t(Q_MN) << 16) |
                             (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* split_done = empty + STAGES;
  uint64_t* tmem_full = split_done + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_holder + 1);

  int pi = 0;
  const int u = blockIdx.x;
  while (pi + 1 < nprob && probs[pi + 1].unit_begin <= u) ++pi;
  const GemmProblem& pr = probs[pi];
  const int local = u - pr.unit_begin;
  const int ks = local % pr.splits;
  const int t = local / pr.splits;
  const int tq = t % pr.tiles_q;
  const int tp = t / pr.tiles_q;
  const int kb0 = ks * pr.kb_per_split;
  const int kb1 = min(pr.kb_total, kb0 + pr.kb_per_split);
  const int nkb = kb1 - kb0;

  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split_done[s], 6);  // one arrival per splitting warp
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
    tma_prefetch_desc(pr.tmap_a);
    tma_prefetch_desc(pr.tmap_b);
  }
  if (warp == 2) tmem_alloc(tmem_holder, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const int p0 = tp * BM, q0 = tq * BN;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      mbar_arrive_expect_tx(&full[s], OPB);
      const int k0 = (kb0 + i) * BK;
      if constexpr (!P_MN) {
        tma_load_2d(sa, pr.tmap_a, &full[s], k0, p0);
      } else {
#pragma unroll
        for (int j = 0; j < BM / 32; ++j) tma_load_2d(sa + j * 4096, pr.tmap_a, &full[s], p0 + 32 * j, k0);
      }
      if constexpr (!Q_MN) {
        tma_load_2d(sb, pr.tmap_b, &full[s], k0, q0);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) tma_load_2d(sb + j * 4096, pr.tmap_b, &full[s], q0 + 32 * j, k0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      if constexpr (SPLIT) mbar_wait(&split_done[s], ph);
      else mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        // K-major: 128B rows of K, 8-row atoms (SBO 1024), K step = +32 bytes.
        // MN-major: 128B rows of M/N per k, 32-byte-granule swizzle, 4-row groups (SBO 512),
        //           32-column chunks 4096 bytes apart (LBO), K step = 8 rows = +1024 bytes.
        const uint64_t ad = P_MN ? umma_desc(sa + kk * 1024, pr.mn_lbo, pr.mn_sbo, 1)
                                 : umma_desc(sa + kk * 32, 16, 1024, 2);
        const uint64_t bd = Q_MN ? umma_desc(sb + kk * 1024, pr.mn_lbo, pr.mn_sbo, 1)
                                 : umma_desc(sb + kk * 32, 16, 1024, 2);
        if constexpr (SPLIT) {
          // low parts live OPB bytes after the high parts, in the same (swizzled) layout
          const uint64_t lo = uint64_t((OPB >> 4) & 0x3FFFu);
          mma_tf32(tmem_base, ad + lo, bd, IDESC, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem_base, ad, bd + lo, IDESC, 1u);
          mma_tf32(tmem_base, ad, bd, IDESC, 1u);
        } else {
          mma_tf32(tmem_base, ad, bd, IDESC, (i > 0 || kk > 0) ? 1u : 0u);
        }
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tmem_full);
  }
  if (SPLIT && warp >= 2) {
    // ---------------- 3xTF32 split: hi in place, lo into the stage's second half
    const int tid = threadIdx.x - 64;  // 0..191
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&full[s], ph);
      float4* hi = reinterpret_cast<float4*>(smem + s * STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + OPB);
      for (int c = tid; c < int(OPB / 16); c += 192) {
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
  if (warp >= 4) {
    // ---------------- epilogue warpgroup
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const int p = tp * BM + row;
    const uint32_t taddr_row = tmem_base + (uint32_t(ew * 32) << 16);
    if (nkb > 0) mbar_wait(tmem_full, 0);
    tc_fence_after();

    const int splits = pr.splits;
    float* ws_tile = nullptr;
    if (splits > 1) {
      ws_tile = pr.ws + (size_t)t * splits * BM * BN;
      float* mine = ws_tile + ((size_t)ks * BM + row) * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        if (nkb > 0) {
          tmem_ld32(taddr_row + c0, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        float4* d = reinterpret_cast<float4*>(mine + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j) __stcg(d + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
      }
      __threadfence();
      named_bar_sync(1, 128);
      if (row == 0) {
        const unsigned old = atomicAdd(&pr.counters[t], 1u);
        const int is_last = old == unsigned(splits - 1);
        if (is_last) pr.counters[t] = 0;
        *last_flag = is_last;
      }
      named_bar_sync(1, 128);
      if (!*last_flag) goto done;
      __threadfence();
    }

#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if (splits > 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
        for (int s = 0; s < splits; ++s) {
          const float4* src = reinterpret_cast<const float4*>(ws_tile + ((size_t)s * BM + row) * BN + c0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 x = __ldcg(src + j);
            v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
          }
        }
      } else if (nkb > 0) {
        tmem_ld32(taddr_row + c0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      const int q0 = tq * BN + c0;
      if (q0 >= pr.Q) continue;
      store_chunk(pr.out, pr.out_rs, pr.out_cs, p, q0, pr.P, pr.Q, v);
      for (int e = 0; e < pr.n_epi; ++e) {
        const EpiStage& st = pr.epi[e];
        float o[32];
        if (epi_needs_other(st.op)) {
          load_chunk(st.other, st.o_rs, st.o_cs, p, q0, pr.P, pr.Q, o);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = epi_apply(st.op, v[j], epi_needs_other(st.op) ? o[j] : 0.f, st.scale);
        store_chunk(st.out, st.out_rs, st.out_cs, p, q0, pr.P, pr.Q, v);
      }
    }
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

using KernelFn = void (*)(const GemmProblem*, int);

template <int BN, bool SPLIT>
KernelFn pick(bool p_mn, bool q_mn) {
  if (!p_mn && !q_mn) return gemm_tf32_kernel<BN, false, false, SPLIT>;
  if (!p_mn && q_mn) return gemm_tf32_kernel<BN, false, true, SPLIT>;
  if (p_mn && !q_mn) return gemm_tf32_kernel<BN, true, false, SPLIT>;
  return gemm_tf32_kernel<BN, true, true, SPLIT>;
}

KernelFn kernel_for(int bn, bool p_mn, bool q_mn, bool split) {
  switch (bn) {
    case 32: return split ? pick<32, true>(p_mn, q_mn) : pick<32, false>(p_mn, q_mn);
    case 64: return split ? pick<64, true>(p_mn, q_mn) : pick<64, false>(p_mn, q_mn);
    case 128: return split ? pick<128, true>(p_mn, q_mn) : pick<128, false>(p_mn, q_mn);
    case 256: return split ? pick<256, true>(p_mn, q_mn) : pick<256, false>(p_mn, q_mn);
  }
  throw std::runtime_error("gemm: unsupported tile width " + std::to_string(bn));
}

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

// 2-D fp32 tensor map over a row-major view: `inner` contiguous elements per row, `outer`
// rows `row_stride` elements apart, boxes of box_inner x box_outer, 128-byte swizzle.
void make_map(CUtensorMap* m, const float* base, long long inner, long long outer,
              long long row_stride, int box_inner, int box_outer, bool mn_major) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(std::max<long long>(row_stride, inner) * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

struct Role {
  const float* ptr;
  long long inner, outer, rs;
  bool mn;  // contiguous dim is the row (M/N) dim rather than K
};

unsigned g_dbg_lbo = 0, g_dbg_sbo = 0;

}  // namespace

void gemm_debug_mn_desc(unsigned lbo, unsigned sbo) {
  g_dbg_lbo = lbo;
  g_dbg_sbo = sbo;
}

bool gemm_view_ok(const MatView& v) {
  if (v.cs != 1) return false;
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) != 0) return false;
  if (v.rows > 1 && (v.rs % 4) != 0) return false;
  return true;
}

GemmLaunch gemm_prepare(const std::vector<GemmSpec>& specs, int num_sms, bool split) {
  if (specs.empty()) throw std::runtime_error("gemm: empty batch");
  GemmLaunch g;
  g.split = split;
  const GemmSpec& s0 = specs[0];
  const long long M0 = s0.ta ? s0.a.cols : s0.a.rows;
  const long long N0 = s0.tb ? s0.b.rows : s0.b.cols;
  g.swap = (M0 < 128 && N0 >= 2 * M0);
  const long long Q0 = g.swap ? M0 : N0;
  g.bn = Q0 <= 32 ? 32 : Q0 <= 64 ? 64 : Q0 <= 128 ? 128 : 256;
  g.nprob = int(specs.size());

  std::vector<CUtensorMap> maps(2 * specs.size());
  std::vector<GemmProblem>& probs = g.host_problems;
  probs.resize(specs.size());
  long long total_tiles = 0;
  for (size_t i = 0; i < specs.size(); ++i) {
    const GemmSpec& s = specs[i];
    if (!gemm_view_ok(s.a) || !gemm_view_ok(s.b))
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
    make_map(&maps[2 * i], rp.ptr, rp.inner, rp.outer, rp.rs, 32, rp.mn ? 32 : BM, rp.mn);
    make_map(&maps[2 * i + 1], rq.ptr, rq.inner, rq.outer, rq.rs, 32, rq.mn ? 32 : g.bn, rq.mn);
    GemmProblem& pr = probs[i];
    pr.P = int(g.swap ? N : M);
    pr.Q = int(g.swap ? M : N);
    pr.K = int(K);
    pr.tiles_p = int((pr.P + BM - 1) / BM);
    pr.tiles_q = int((pr.Q + g.bn - 1) / g.bn);
    pr.kb_total = int((K + BK - 1) / BK);
    pr.out = s.c;
    pr.out_rs = g.swap ? s.c_cs : s.c_rs;
    pr.out_cs = g.swap ? s.c_rs : s.c_cs;
    if (g_dbg_lbo) pr.mn_lbo = g_dbg_lbo;
    if (g_dbg_sbo) pr.mn_sbo = g_dbg_sbo;
    pr.n_epi = s.n_epi;
    for (int e = 0; e < s.n_epi; ++e) {
      pr.epi[e] = s.epi[e];
      if (g.swap) {
        std::swap(pr.epi[e].o_rs, pr.epi[e].o_cs);
        std::swap(pr.epi[e].out_rs, pr.epi[e].out_cs);
      }
    }
    total_tiles += (long long)pr.tiles_p * pr.tiles_q;
    g.flops += 2.0 * double(M) * double(N) * double(K);
    g.min_bytes += 4.0 * double(M * K + K * N + M * N * (1 + s.n_epi));
    for (int e = 0; e < s.n_epi; ++e)
      if (s.epi[e].op >= EPI_ADD) g.min_bytes += 4.0 * double(M * N);
  }
  // K-split: minimise waves of work per unit of work, favouring fewer splits.
  const int kb = probs[0].kb_total;
  int best_s = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 32; ++s) {
    if (s > 1 && kb / s < 8) break;
    const long long units = total_tiles * s;
    const double waves = double((units + num_sms - 1) / num_sms);
    const double cost = waves / s * (1.0 + 0.01 * s);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best_s = s;
    }
  }
  int unit = 0;
  size_t ws = 0, cnt = 0;
  for (auto& pr : probs) {
    const int kbps = (pr.kb_total + best_s - 1) / best_s;
    pr.kb_per_split = kbps;
    pr.splits = (pr.kb_total + kbps - 1) / kbps;
    pr.unit_begin = unit;
    unit += pr.tiles_p * pr.tiles_q * pr.splits;
    if (pr.splits > 1) {
      ws += size_t(pr.tiles_p) * pr.tiles_q * pr.splits * BM * g.bn;
      cnt += size_t(pr.tiles_p) * pr.tiles_q;
    }
  }
  g.units = unit;
  g.ws_floats = ws;
  g.n_counters = cnt;
  if (ws) {
    CUDA_CHECK(cudaMalloc(&g.d_ws, ws * sizeof(float)));
    CUDA_CHECK(cudaMalloc(&g.d_counters, cnt * sizeof(unsigned)));
    CUDA_CHECK(cudaMemset(g.d_counters, 0, cnt * sizeof(unsigned)));
  }
  size_t wo = 0, co = 0;
  for (auto& pr : probs) {
    if (pr.splits > 1) {
      pr.ws = g.d_ws + wo;
      pr.counters = g.d_counters + co;
      wo += size_t(pr.tiles_p) * pr.tiles_q * pr.splits * BM * g.bn;
      co += size_t(pr.tiles_p) * pr.tiles_q;
    }
  }
  CUDA_CHECK(cudaMalloc(&g.d_tmaps, maps.size() * sizeof(CUtensorMap)));
  CUDA_CHECK(cudaMemcpy(g.d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  for (size_t i = 0; i < probs.size(); ++i) {
    probs[i].tmap_a = static_cast<CUtensorMap*>(g.d_tmaps) + 2 * i;
    probs[i].tmap_b = static_cast<CUtensorMap*>(g.d_tmaps) + 2 * i + 1;
  }
  CUDA_CHECK(cudaMalloc(&g.d_problems, probs.size() * sizeof(GemmProblem)));
  CUDA_CHECK(cudaMemcpy(g.d_problems, probs.data(), probs.size() * sizeof(GemmProblem), cudaMemcpyHostToDevice));
  g.smem_bytes = smem_for(g.bn, split);
  KernelFn fn = kernel_for(g.bn, g.p_mn, g.q_mn, split);
  CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.smem_bytes)));
  return g;
}

void gemm_run(const GemmLaunch& g, cudaStream_t stream) {
  KernelFn fn = kernel_for(g.bn, g.p_mn, g.q_mn, g.split);
  fn<<<g.units, 256, g.smem_bytes, stream>>>(static_cast<const GemmProblem*>(g.d_problems), g.nprob);
  CUDA_CHECK(cudaGetLastError());
}

void gemm_free(GemmLaunch& g) {
  if (g.d_problems) cudaFree(g.d_problems);
  if (g.d_tmaps) cudaFree(g.d_tmaps);
  if (g.d_ws) cudaFree(g.d_ws);
  if (g.d_counters) cudaFree(g.d_counters);
  g = GemmLaunch{};
}

}  // namespace tpx
