// Batched bandwidth kernels: strided N-ary (copy / reduce / elementwise), seeded init, direct
// conv.  See kernels.h.  Work is tiled by rows of the (dim-merged) innermost extent so the
// inner loop is division-free and, when every operand is unit-stride and 16-byte aligned,
// moves float4s.
#include "kernels.h"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "util.h"

namespace tpx {

namespace {
// ---- storage element access: T = float or __nv_bfloat16 (arithmetic is always fp32)
template <class T>
__device__ __forceinline__ float eld(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(__ldg(p));
  else return __ldg(p);
}
template <class T>
__device__ __forceinline__ float eldv(const T* p) {  // plain (coherent) load, for accumulate
  if constexpr (sizeof(T) == 2) return __bfloat162float(*p);
  else return *p;
}
template <class T>
__device__ __forceinline__ void est(T* p, float v) {
  if constexpr (sizeof(T) == 2) *p = __float2bfloat16_rn(v);
  else *p = v;
}
// 4 consecutive elements (16 B fp32 / 8 B bf16, aligned)
template <class T>
__device__ __forceinline__ float4 eld4(const T* p) {
  if constexpr (sizeof(T) == 2) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return __ldg(reinterpret_cast<const float4*>(p));
  }
}
template <class T>
__device__ __forceinline__ float4 eld4v(const T* p) {
  if constexpr (sizeof(T) == 2) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return *reinterpret_cast<const float4*>(p);
  }
}
template <class T>
__device__ __forceinline__ void est4(T* p, float4 v) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&a);
    u.y = *reinterpret_cast<const uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  } else {
    *reinterpret_cast<float4*>(p) = v;
  }
}
}  // namespace

namespace {

constexpr int kThreads = 256;
constexpr int64_t kTileUnits = 4096;

__device__ __forceinline__ int find_desc(const int64_t* tile_begin_base, size_t stride_bytes,
                                         int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const int64_t tb = *reinterpret_cast<const int64_t*>(
        reinterpret_cast<const char*>(tile_begin_base) + size_t(mid) * stride_bytes);
    if (tb <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Row tiling shared by nary / init: rows x inner (units) split into tiles of ~`tile` units.  A
// tile is either a chunk of one long row (all threads on it) or rpt whole rows walked by groups
// of rg threads (rg = 1..256, about 4 units per thread per row, so short rows still keep every
// thread busy).
struct RowTiling {
  int64_t rows, inner, rpt, col_chunk, n_col_chunks, rg;
};

RowTiling row_tiling(int64_t rows, int64_t inner, int64_t tile = kTileUnits) {
  RowTiling t;
  t.rows = rows;
  t.inner = inner;
  if (inner >= tile) {
    t.rpt = 1;
    t.col_chunk = tile;
    t.n_col_chunks = (inner + tile - 1) / tile;
    t.rg = kThreads;
  } else {
    t.col_chunk = std::max<int64_t>(inner, 1);
    t.n_col_chunks = 1;
    // (short rows: fewer threads per row, down to one -- consecutive threads then take
    // consecutive rows, so a tile of one-unit rows still keeps every lane busy)
    int64_t rg = 1;
    while (rg < kThreads && rg * 4 < inner) rg *= 2;
    t.rg = rg;
    t.rpt = std::max<int64_t>(kThreads / rg, tile / t.col_chunk);
  }
  return t;
}

// ---------------------------------------------------------------- nary

struct NaryDev {
  NaryDesc d;
  int64_t rows, inner, rpt, col_chunk, n_col_chunks, rg;
};

__device__ __forceinline__ float nary_apply(int op, int nin, const float* v, float s) {
  switch (op) {
    case NARY_COPY: return v[0];
    case NARY_SUM: {
      float a = v[0];
      for (int i = 1; i < nin; ++i) a += v[i];
      return a;
    }
    case NARY_SUB: return v[0] - v[1];
    case NARY_SCALE: return s * v[0];
    case NARY_TANH: return tanhf(v[0]);
    case NARY_DTANH: {
      const float t = tanhf(v[0]);
      return 1.0f - t * t;
    }
    default: return v[0];
  }
}

// ---- peer synchronisation (TPX_FLAG_PEER): system-scope acquire / release on 64-bit counters
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until every rank in `mask` has reached count `c` (bounded: a wait that outlives
// timeout_ns records the rank in the host-mapped error word and gives up instead of hanging).
__device__ __forceinline__ bool peer_wait_one(const unsigned long long* p, unsigned long long c, int* err,
                                              unsigned long long timeout_ns, int r) {
  if (ld_acquire_sys(p) >= c) return true;
  const unsigned long long t0 = globaltimer();
  for (unsigned spins = 1; ld_acquire_sys(p) < c; ++spins) {
    __nanosleep(100);
    if ((spins & 255u) == 0) {  // (the error word is host memory: read it rarely)
      if (*reinterpret_cast<volatile int*>(err)) return false;
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 0x100 | r);
        return false;
      }
    }
  }
  return true;
}
// (ranks unrolled: the counters stay in the kernel's parameter space, no local copy)
__device__ __forceinline__ void peer_wait(const PeerSync& s, uint32_t mask, unsigned long long c) {
#pragma unroll
  for (int r = 0; r < kMaxRanks; ++r)
    if ((mask >> r & 1u) && !peer_wait_one(s.peer[r], c, s.err, s.timeout_ns, r)) return;
}

__device__ __forceinline__ void peer_publish(const PeerSync& s, unsigned long long v) {
  // everything earlier on this stream (previous launches) is complete: publish it
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  st_release_sys(s.local, v);
}
// the value sync point `idx` of the current step publishes (-1: the previous barrier's)
__device__ __forceinline__ unsigned long long sync_value(const PeerSync& s, int idx) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(s.epoch);
  // (+ 1: the counters start at 0, and the first point of the first step must not be satisfied
  // before it is published)
  return idx >= 0 ? e * kSyncK + unsigned(idx) + 1ull : e * kSyncK - 1ull;
}

__global__ void sync_kernel(PeerSync s, int index, int barrier) {
  if (threadIdx.x != 0) return;
  if (!barrier) {
    peer_publish(s, sync_value(s, index));
    return;
  }
  const unsigned long long e = *s.epoch, v = e * kSyncK + (kSyncK - 1ull);
  peer_publish(s, v);
  peer_wait(s, ((1u << s.world) - 1u) & ~(1u << s.rank), v);
  *s.epoch = e + 1;  // read only by this rank's later launches (stream order)
}

// Start of a conversion launch in peer mode: publish the phase's sync point (every block writes
// the same value: idempotent) and wait for the ranks this block reads from.
// (block 0 publishes -- any block starts after everything earlier on the stream; a rank never
// waits on itself: its own data is ordered by the stream)
__device__ __forceinline__ void peer_prologue(const PeerSync& s, int signal_s, int wait_s, uint32_t mask) {
  if (signal_s >= 0 && blockIdx.x == 0) peer_publish(s, sync_value(s, signal_s));
  mask &= ~(1u << s.rank);
  if (mask) peer_wait(s, mask, sync_value(s, wait_s));
}

// Chained elementwise stage (EpiOp codes, gemm.h) on the previous stage's stored value.
__device__ __forceinline__ float chain_apply(int op, float x, float o, float s) {
  switch (op) {
    case 1: return tanhf(x);
    case 2: { const float t = tanhf(x); return 1.0f - t * t; }
    case 3: return s * x;
    case 4: return x + o;
    case 5: return x - o;
    case 6: return o - x;
    default: return x;
  }
}
template <class T>
__device__ __forceinline__ float stored(float v) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(__float2bfloat16_rn(v));
  else return v;
}

// The block's descriptor, staged in shared memory once (a per-thread walk of the global
// descriptor table costs dozens of dependent loads per block).
template <class T, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) nary_kernel(const NaryDev* __restrict__ ds, const int* __restrict__ tile_desc,
                                                           PeerSync sync, int signal_s, int wait_s) {
  __shared__ __align__(16) unsigned char sraw[(sizeof(NaryDev) + 15) / 16 * 16];
  __shared__ int sdi;
  if (threadIdx.x == 0) sdi = __ldg(tile_desc + blockIdx.x);
  __syncthreads();
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(ds + sdi);
    uint32_t* dst = reinterpret_cast<uint32_t*>(sraw);
    for (int i = threadIdx.x; i < int(sizeof(NaryDev) / 4); i += kThreads) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const NaryDev& D = *reinterpret_cast<const NaryDev*>(sraw);
  const NaryDesc& d = D.d;
  if (d.wait_mask || signal_s >= 0) {  // peer mode: publish the phase, wait for the sources' ranks
    if (threadIdx.x == 0) peer_prologue(sync, signal_s, wait_s, d.wait_mask);
    __syncthreads();
  }
  const int64_t local = int64_t(blockIdx.x) - d.tile_begin;
  const int64_t rb = local / D.n_col_chunks, cc = local % D.n_col_chunks;
  const int64_t r0 = rb * D.rpt, r1 = min(D.rows, r0 + D.rpt);
  const int64_t c0 = cc * D.col_chunk, c1 = min(D.inner, c0 + D.col_chunk);
  const int nin = d.nin, op = d.op, nch = d.n_chain;
  // groups of rg threads walk the tile's rows (rg = kThreads: one row chunk, all threads on it)
  const int rg = int(D.rg);
  const int warp = int(threadIdx.x) / rg, lane = int(threadIdx.x) % rg;
  const int cstep = rg;
  for (int64_t r = r0 + warp; r < r1; r += kThreads / rg) {
    const int64_t i2 = r % d.shape[2];
    const int64_t t = r / d.shape[2];
    const int64_t i1 = t % d.shape[1];
    const int64_t i0 = t / d.shape[1];
    const int64_t ooff = i0 * d.out_st[0] + i1 * d.out_st[1] + i2 * d.out_st[2];
    T* out = reinterpret_cast<T*>(d.out) + ooff;
    const T* in[kMaxIn];
#pragma unroll
    for (int k = 0; k < kMaxIn; ++k)
      if (k < nin) in[k] = reinterpret_cast<const T*>(d.in[k]) + i0 * d.in_st[k][0] + i1 * d.in_st[k][1] + i2 * d.in_st[k][2];
    if (d.vec == 4 && op == NARY_SUM && nin <= 4) {
      // partial-sum reduction (reduce_partial, <= 4 partials): 4 elements per thread in flight,
      // summed left to right exactly like NARY_SUM, then the chained stages
      constexpr int U = 4;
      for (int64_t cb = c0 + lane; cb < c1; cb += U * cstep) {
        float4 acc[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (cb + j * cstep < c1) acc[j] = eld4(in[0] + 4 * (cb + j * cstep));
#pragma unroll
        for (int k = 1; k < 4; ++k) {
          if (k >= nin) break;
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (cb + j * cstep < c1) {
              const float4 v = eld4(in[k] + 4 * (cb + j * cstep));
              acc[j].x += v.x; acc[j].y += v.y; acc[j].z += v.z; acc[j].w += v.w;
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int64_t c = cb + j * cstep;
          if (c >= c1) break;
          float4 o = acc[j];
          est4(out + 4 * c, o);
          for (int s = 0; s < nch; ++s) {
            const ChainStage& cs = d.chain[s];
            const int64_t e = ooff + 4 * c;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (cs.other) w = eld4(reinterpret_cast<const T*>(cs.other) + e);
            o.x = chain_apply(cs.op, stored<T>(o.x), w.x, cs.scale);
            o.y = chain_apply(cs.op, stored<T>(o.y), w.y, cs.scale);
            o.z = chain_apply(cs.op, stored<T>(o.z), w.z, cs.scale);
            o.w = chain_apply(cs.op, stored<T>(o.w), w.w, cs.scale);
            est4(reinterpret_cast<T*>(cs.out) + e, o);
          }
        }
      }
      continue;
    }
    if (d.vec == 4) {
      for (int64_t c = c0 + lane; c < c1; c += cstep) {
        float4 v[kMaxIn];
#pragma unroll
        for (int k = 0; k < kMaxIn; ++k)
          if (k < nin) v[k] = eld4(in[k] + 4 * c);
        float4 o;
        if (op == NARY_ACC) {
          o = eld4v(out + 4 * c);
          o.x += v[0].x; o.y += v[0].y; o.z += v[0].z; o.w += v[0].w;
        } else {
          float a[kMaxIn];
#pragma unroll
          for (int k = 0; k < kMaxIn; ++k) a[k] = k < nin ? v[k].x : 0.f;
          o.x = nary_apply(op, nin, a, d.scale);
#pragma unroll
          for (int k = 0; k < kMaxIn; ++k) a[k] = k < nin ? v[k].y : 0.f;
          o.y = nary_apply(op, nin, a, d.scale);
#pragma unroll
          for (int k = 0; k < kMaxIn; ++k) a[k] = k < nin ? v[k].z : 0.f;
          o.z = nary_apply(op, nin, a, d.scale);
#pragma unroll
          for (int k = 0; k < kMaxIn; ++k) a[k] = k < nin ? v[k].w : 0.f;
          o.w = nary_apply(op, nin, a, d.scale);
        }
        est4(out + 4 * c, o);
        for (int s = 0; s < nch; ++s) {
          const ChainStage& cs = d.chain[s];
          const int64_t e = ooff + 4 * c;
          float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
          if (cs.other) w = eld4(reinterpret_cast<const T*>(cs.other) + e);
          o.x = chain_apply(cs.op, stored<T>(o.x), w.x, cs.scale);
          o.y = chain_apply(cs.op, stored<T>(o.y), w.y, cs.scale);
          o.z = chain_apply(cs.op, stored<T>(o.z), w.z, cs.scale);
          o.w = chain_apply(cs.op, stored<T>(o.w), w.w, cs.scale);
          est4(reinterpret_cast<T*>(cs.out) + e, o);
        }
      }
    } else {
      const int64_t os = d.out_st[3];
      for (int64_t c = c0 + lane; c < c1; c += cstep) {
        float a[kMaxIn];
#pragma unroll
        for (int k = 0; k < kMaxIn; ++k) a[k] = k < nin ? eld(in[k] + c * d.in_st[k][3]) : 0.f;
        float o;
        if (op == NARY_ACC) o = eldv(out + c * os) + a[0];
        else o = nary_apply(op, nin, a, d.scale);
        est(out + c * os, o);
        for (int s = 0; s < nch; ++s) {
          const ChainStage& cs = d.chain[s];
          const int64_t e = ooff + c * os;
          const float w = cs.other ? eld(reinterpret_cast<const T*>(cs.other) + e) : 0.f;
          o = chain_apply(cs.op, stored<T>(o), w, cs.scale);
          est(reinterpret_cast<T*>(cs.out) + e, o);
        }
      }
    }
  }
}

// Batches made only of plain box copies (pack / unpack / pull / concat pieces, no chain): one
// source per descriptor, so a light kernel (few registers, full occupancy) with 8 independent
// loads in flight per thread -- enough to cover NVLink latency on a peer read.
template <class T, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) copy_kernel(const NaryDev* __restrict__ ds, const int* __restrict__ tile_desc,
                                                           PeerSync sync, int signal_s, int wait_s) {
  __shared__ int sdi;
  if (threadIdx.x == 0) {
    const int di = __ldg(tile_desc + blockIdx.x);
    sdi = di;
    if (ds[di].d.wait_mask || signal_s >= 0) peer_prologue(sync, signal_s, wait_s, ds[di].d.wait_mask);
  }
  __syncthreads();
  const NaryDev& D = ds[sdi];
  const int64_t tb = D.d.tile_begin, nch = D.n_col_chunks, rpt = D.rpt, rows = D.rows, inner = D.inner;
  const int64_t colc = D.col_chunk;
  const int64_t sh1 = D.d.shape[1], sh2 = D.d.shape[2];
  const int64_t o0 = D.d.out_st[0], o1 = D.d.out_st[1], o2 = D.d.out_st[2], o3 = D.d.out_st[3];
  const int64_t s0 = D.d.in_st[0][0], s1 = D.d.in_st[0][1], s2 = D.d.in_st[0][2], s3 = D.d.in_st[0][3];
  const int vec = D.d.vec;
  T* const obase = reinterpret_cast<T*>(D.d.out);
  const T* const ibase = reinterpret_cast<const T*>(D.d.in[0]);
  const int64_t local = int64_t(blockIdx.x) - tb;
  const int64_t rb = local / nch, cc = local % nch;
  const int64_t r0 = rb * rpt, r1 = min(rows, r0 + rpt);
  const int64_t c0 = cc * colc, c1 = min(inner, c0 + colc);
  const int rg = int(D.rg);
  const int warp = int(threadIdx.x) / rg, lane = int(threadIdx.x) % rg;
  const int cstep = rg;
  constexpr int U = 8;
  for (int64_t r = r0 + warp; r < r1; r += kThreads / rg) {
    const int64_t i2 = r % sh2;
    const int64_t t = r / sh2;
    const int64_t i1 = t % sh1;
    const int64_t i0 = t / sh1;
    T* out = obase + i0 * o0 + i1 * o1 + i2 * o2;
    const T* src = ibase + i0 * s0 + i1 * s1 + i2 * s2;
    if (vec == 4) {
      for (int64_t cb = c0 + lane; cb < c1; cb += U * cstep) {
        float4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (cb + j * cstep < c1) v[j] = eld4(src + 4 * (cb + j * cstep));
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (cb + j * cstep < c1) est4(out + 4 * (cb + j * cstep), v[j]);
      }
    } else {
      constexpr int U1 = 4;
      for (int64_t cb = c0 + lane; cb < c1; cb += U1 * cstep) {
        float v[U1];
#pragma unroll
        for (int j = 0; j < U1; ++j)
          if (cb + j * cstep < c1) v[j] = eld(src + (cb + j * cstep) * s3);
#pragma unroll
        for (int j = 0; j < U1; ++j)
          if (cb + j * cstep < c1) est(out + (cb + j * cstep) * o3, v[j]);
      }
    }
  }
}

// K7: max |got - want| and max |got - want| / max(|want|, 1) over a batch of (got, want) box
// pairs, warp-reduced, one atomicMax per warp on the fp32 bit patterns (non-negative floats
// order like their bits).
template <class T>
__global__ void __launch_bounds__(kThreads) check_kernel(const NaryDev* __restrict__ ds, const int* __restrict__ tile_desc,
                                                         unsigned* __restrict__ out) {
  const NaryDev& D = ds[__ldg(tile_desc + blockIdx.x)];
  const NaryDesc& d = D.d;
  const int64_t local = int64_t(blockIdx.x) - d.tile_begin;
  const int64_t rb = local / D.n_col_chunks, cc = local % D.n_col_chunks;
  const int64_t r0 = rb * D.rpt, r1 = min(D.rows, r0 + D.rpt);
  const int64_t c0 = cc * D.col_chunk, c1 = min(D.inner, c0 + D.col_chunk);
  const int rg = int(D.rg);
  const int grp = int(threadIdx.x) / rg, lane = int(threadIdx.x) % rg;
  float mabs = 0.f, mrel = 0.f;
  for (int64_t r = r0 + grp; r < r1; r += kThreads / rg) {
    const int64_t i2 = r % d.shape[2];
    const int64_t t = r / d.shape[2];
    const int64_t i1 = t % d.shape[1];
    const int64_t i0 = t / d.shape[1];
    const T* a = reinterpret_cast<const T*>(d.in[0]) + i0 * d.in_st[0][0] + i1 * d.in_st[0][1] + i2 * d.in_st[0][2];
    const T* b = reinterpret_cast<const T*>(d.in[1]) + i0 * d.in_st[1][0] + i1 * d.in_st[1][1] + i2 * d.in_st[1][2];
    for (int64_t c = c0 + lane; c < c1; c += rg) {
      const float x = eld(a + c * d.in_st[0][3]), y = eld(b + c * d.in_st[1][3]);
      const float diff = fabsf(x - y);
      mabs = fmaxf(mabs, diff);
      mrel = fmaxf(mrel, diff / fmaxf(fabsf(y), 1.f));
      if (diff != diff) mabs = mrel = __int_as_float(0x7f800000);  // NaN: report infinity
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mabs = fmaxf(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
    mrel = fmaxf(mrel, __shfl_xor_sync(0xffffffffu, mrel, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, __float_as_uint(mabs));
    atomicMax(out + 1, __float_as_uint(mrel));
  }
}

// ---------------------------------------------------------------- init (seeded_tensor)

struct InitDev {
  InitDesc d;
  int64_t rows, inner, rpt, col_chunk, n_col_chunks, rg;
};

__device__ __forceinline__ float seeded_value(uint64_t state0, uint64_t flat) {
  // splitmix64 (dense.cpp:30-36): the i-th draw uses state0 + (i+1)*gamma.
  uint64_t z = state0 + (flat + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  const uint64_t bits = z >> 11;  // 53 bits
  const double v = double(bits) * (2.0 / 9007199254740992.0) - 1.0;
  return float(v);  // round-to-nearest fp64 -> fp32
}

template <class T>
__global__ void __launch_bounds__(kThreads) init_kernel(const InitDev* __restrict__ ds, int n) {
  const int di = find_desc(&ds[0].d.tile_begin, sizeof(InitDev), n, blockIdx.x);
  const InitDev& D = ds[di];
  const InitDesc& d = D.d;
  const int64_t local = int64_t(blockIdx.x) - d.tile_begin;
  const int64_t rb = local / D.n_col_chunks, cc = local % D.n_col_chunks;
  const int64_t r0 = rb * D.rpt, r1 = min(D.rows, r0 + D.rpt);
  const int64_t c0 = cc * D.col_chunk, c1 = min(D.inner, c0 + D.col_chunk);
  // groups of rg threads walk the tile's rows (rg = kThreads: one row chunk, all threads on it)
  const int rg = int(D.rg);
  const int warp = int(threadIdx.x) / rg, lane = int(threadIdx.x) % rg;
  const int cstep = rg;
  for (int64_t r = r0 + warp; r < r1; r += kThreads / rg) {
    const int64_t i2 = r % d.ext[2];
    const int64_t t = r / d.ext[2];
    const int64_t i1 = t % d.ext[1];
    const int64_t i0 = t / d.ext[1];
    const uint64_t rowflat =
        ((uint64_t(d.lo[0] + i0) * d.full[1] + uint64_t(d.lo[1] + i1)) * d.full[2] +
         uint64_t(d.lo[2] + i2)) * d.full[3] + uint64_t(d.lo[3]);
    T* out = reinterpret_cast<T*>(d.out) + r * d.ext[3];
    // fp64 -> fp32 (round to nearest) -> storage type (bf16: round to nearest even)
    for (int64_t c = c0 + lane; c < c1; c += cstep) est(out + c, seeded_value(d.state0, rowflat + uint64_t(c)));
  }
}

// ---------------------------------------------------------------- conv (direct)

template <class T>
__device__ __forceinline__ float at4(const StridedView& v, int64_t a, int64_t b, int64_t c, int64_t d) {
  return eld(reinterpret_cast<const T*>(v.ptr) + a * v.st[0] + b * v.st[1] + c * v.st[2] + d * v.st[3]);
}

template <class T>
__global__ void __launch_bounds__(kThreads) conv_kernel(const ConvDesc* __restrict__ ds, int n) {
  const int di = find_desc(&ds[0].tile_begin, sizeof(ConvDesc), n, blockIdx.x);
  const ConvDesc& d = ds[di];
  const int64_t e = (int64_t(blockIdx.x) - d.tile_begin) * kThreads + threadIdx.x;
  if (e >= d.n) return;
  const int64_t o3 = e % d.oshape[3];
  int64_t t = e / d.oshape[3];
  const int64_t o2 = t % d.oshape[2];
  t /= d.oshape[2];
  const int64_t o1 = t % d.oshape[1];
  const int64_t o0 = t / d.oshape[1];
  float acc = 0.f;
  if (d.mode == CONV_FWD) {
    // A (n,ci,h,w) x K (co,ci,fh,fw) -> (n,co,ho,wo)
    const int64_t ci = d.a.shape[1], fh = d.b.shape[2], fw = d.b.shape[3];
    for (int64_t c = 0; c < ci; ++c)
      for (int64_t u = 0; u < fh; ++u)
        for (int64_t v = 0; v < fw; ++v) acc = fmaf(at4<T>(d.a, o0, c, o2 + u, o3 + v), at4<T>(d.b, o1, c, u, v), acc);
  } else if (d.mode == CONV_GRAD_W) {
    // A (n,ci,h,w) x G (n,co,ho,wo) -> (co,ci,fh,fw)
    const int64_t nb = d.a.shape[0], ho = d.b.shape[2], wo = d.b.shape[3];
    for (int64_t b = 0; b < nb; ++b)
      for (int64_t y = 0; y < ho; ++y)
        for (int64_t x = 0; x < wo; ++x) acc = fmaf(at4<T>(d.a, b, o1, y + o2, x + o3), at4<T>(d.b, b, o0, y, x), acc);
  } else {
    // G (n,co,ho,wo) x K (co,ci,fh,fw) -> (n,ci,ho+fh-1,wo+fw-1), bounds-checked taps
    const int64_t co = d.a.shape[1], ho = d.a.shape[2], wo = d.a.shape[3];
    const int64_t fh = d.b.shape[2], fw = d.b.shape[3];
    for (int64_t o = 0; o < co; ++o)
      for (int64_t u = 0; u < fh; ++u) {
        const int64_t yy = o2 - u;
        if (yy < 0 || yy >= ho) continue;
        for (int64_t v = 0; v < fw; ++v) {
          const int64_t xx = o3 - v;
          if (xx < 0 || xx >= wo) continue;
          acc = fmaf(at4<T>(d.a, o0, o, yy, xx), at4<T>(d.b, o, o1, u, v), acc);
        }
      }
  }
  est(reinterpret_cast<T*>(d.out) + e, acc);
}

// im2col / col2im of the tensor-core conv lowering.
//   im2col: block = (channel c, group of G images, chunk of taps).  The block stages the G input
//     planes a[n, c, :, :] in shared memory once (read from HBM once), then writes every tap's
//     column segment: thread items run over the group's flat (image, y, x) output positions, so
//     each warp store is one contiguous run of a column row and the (y, x) decomposition is paid
//     once per item, not per tap.  HBM traffic = input planes + columns (write-bound).
//   col2im: block = (channel c, group of G images); thread items over the flat (image, y, x)
//     output positions; each tap's read is a contiguous run of a column row (coalesced), taps
//     summed in ascending (u, v) order (the direct conv's order), optional fused 1 - tanh^2.
constexpr int kMoveSmem = 32768;  // im2col plane staging per block (bytes)

// Sum of the valid taps of one col2im output element in ascending tap order: p0 = the element's
// column position, ctoff[t] = tap t's offset from it, bit t of `mask` = tap t lands inside.
template <int NT, class T>
__device__ __forceinline__ float col2im_masked(const T* p0, const long long* ctoff, uint32_t mask, int nt) {
  float acc = 0.f;
  if constexpr (NT > 0) {
#pragma unroll
    for (int t = 0; t < NT; ++t) acc += (mask >> t) & 1u ? eld(p0 + ctoff[t]) : 0.f;
  } else {
#pragma unroll 4
    for (int t = 0; t < nt; ++t) acc += (mask >> t) & 1u ? eld(p0 + ctoff[t]) : 0.f;
  }
  return acc;
}

constexpr int kMaxTapChunk = 128;  // taps per im2col block (offset table in shared memory)
constexpr int kIm2colIlp = 4;      // items per thread in flight

// Column segments of `nt` taps for Gn images: item (g, y, x) of the flat output positions reads
// base[g*is + y*rs + x*cs + toff[t]] and writes dst[t*pitch + g*img + y*Xo + x].  Offsets are
// computed once per item; the tap loop is a shared-memory (or L1) load and a store per element.
template <class T>
__device__ __forceinline__ void im2col_items(const T* __restrict__ base, int is, int rs, int cs,
                                             const int* toff, int nt, int Gn, int YX, int Xo,
                                             int64_t img, int64_t pitch, T* __restrict__ dst) {
  const int n_items = Gn * YX;
  for (int it0 = threadIdx.x; it0 < n_items; it0 += kThreads * kIm2colIlp) {
    int so[kIm2colIlp], dof[kIm2colIlp];
#pragma unroll
    for (int j = 0; j < kIm2colIlp; ++j) {
      const int it = it0 + j * kThreads;
      const int g = it / YX, e = it - g * YX, y = e / Xo, x = e - y * Xo;
      so[j] = g * is + y * rs + x * cs;
      dof[j] = it < n_items ? int(g * img) + e : -1;
    }
    T* dp = dst;
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      const int to = toff[t];
      T v[kIm2colIlp];
#pragma unroll
      for (int j = 0; j < kIm2colIlp; ++j)
        if (dof[j] >= 0) v[j] = base[so[j] + to];
#pragma unroll
      for (int j = 0; j < kIm2colIlp; ++j)
        if (dof[j] >= 0) dp[dof[j]] = v[j];
      dp += pitch;
    }
  }
}

template <class T>
__device__ __forceinline__ void im2col_body(const ConvDesc& d, int tile) {
  //   out[(c*U*V + u*V + v)*pitch + nb*img + y*Xo + x] = a[nb, c, y+u, x+v]
  extern __shared__ __align__(16) unsigned char move_smem[];
  __shared__ int toff[kMaxTapChunk];  // tap (u, v) -> source offset
  const int NB = int(d.a.shape[0]);
  const int U = int(d.p[0]), V = int(d.p[1]), Yo = int(d.p[2]), Xo = int(d.p[3]);
  const int64_t pitch = d.p[4], img = d.p[5];
  const int TC = int(d.p[6]), G = max(1, int(d.p[7]));  // p[7] = 0: planes read from global
  const int H = Yo + U - 1, W = Xo + V - 1, HW = H * W, YX = Yo * Xo, UV = U * V;
  const int ngrp = (NB + G - 1) / G, nch = (UV + TC - 1) / TC;
  const int c = tile / (ngrp * nch), rest = tile - c * ngrp * nch;
  const int gb = rest / nch, ch = rest - gb * nch;
  const int nb0 = gb * G, Gn = min(G, NB - nb0);
  const int k0 = ch * TC, k1 = min(UV, k0 + TC);
  const T* src = reinterpret_cast<const T*>(d.a.ptr) + int64_t(nb0) * d.a.st[0] + int64_t(c) * d.a.st[1];
  T* dst = reinterpret_cast<T*>(d.out) + int64_t(c * UV + k0) * pitch + int64_t(nb0) * img;
  if (d.p[7] > 0) {
    T* sp = reinterpret_cast<T*>(move_smem);
    if (d.a.st[3] == 1 && d.a.st[2] == W) {
      // dense planes: 4 independent loads in flight per thread, no index decomposition
      for (int g = 0; g < Gn; ++g) {
        const T* pl = src + int64_t(g) * d.a.st[0];
        T* sq = sp + g * HW;
        for (int i = threadIdx.x; i < HW; i += 4 * kThreads) {
          T v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i + j * kThreads < HW) v[j] = pl[i + j * kThreads];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i + j * kThreads < HW) sq[i + j * kThreads] = v[j];
        }
      }
    } else {
      for (int i = threadIdx.x; i < Gn * HW; i += kThreads) {
        const int g = i / HW, r = i - g * HW, y = r / W, x = r - y * W;
        sp[i] = src[int64_t(g) * d.a.st[0] + int64_t(y) * d.a.st[2] + int64_t(x) * d.a.st[3]];
      }
    }
    for (int k = k0 + threadIdx.x; k < k1; k += kThreads) toff[k - k0] = (k / V) * W + (k % V);
    __syncthreads();
    im2col_items<T>(sp, HW, W, 1, toff, k1 - k0, Gn, YX, Xo, img, pitch, dst);
  } else {  // one image per block, plane read from global (L1/L2)
    const int rs = int(d.a.st[2]), cs = int(d.a.st[3]);
    for (int k = k0 + threadIdx.x; k < k1; k += kThreads) toff[k - k0] = (k / V) * rs + (k % V) * cs;
    __syncthreads();
    im2col_items<T>(src, 0, rs, cs, toff, k1 - k0, 1, YX, Xo, img, pitch, dst);
  }
}

template <class T, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) col2im_kernel(const ConvDesc* __restrict__ ds, int n) {
  //   out[nb, c, y, x] = sum_{u,v} col[(c,u,v)*pitch + nb*img + (y-u)*Xo + (x-v)]
  //   (b.ptr != null: also writes 1 - tanh(out)^2 there, from the stored value)
  __shared__ long long ctoff[32];
  const int di = find_desc(&ds[0].tile_begin, sizeof(ConvDesc), n, blockIdx.x);
  const ConvDesc& d = ds[di];
  const int tile = int(int64_t(blockIdx.x) - d.tile_begin);
  const int NB = int(d.a.shape[0]);
  const int C = int(d.p[0]), U = int(d.p[1]), V = int(d.p[2]), Yo = int(d.p[3]), Xo = int(d.p[4]);
  const int64_t pitch = d.p[5], img = d.p[6];
  const int G = int(d.p[7]);
  const int H = Yo + U - 1, W = Xo + V - 1, HW = H * W, UV = U * V;
  const int ngrp = (NB + G - 1) / G;
  const int c = tile / ngrp, gb = tile - c * ngrp;
  const int nb0 = gb * G, Gn = min(G, NB - nb0);
  const T* col0 = reinterpret_cast<const T*>(d.a.ptr) + int64_t(nb0) * img + int64_t(c * U * V) * pitch;
  // out[nb, c, y, x] at nb*on + c*oc + y*W + x (b.st: dense [n, c] or the channel-major layout)
  const int64_t on = d.b.st[0] ? d.b.st[0] : int64_t(C) * HW, oc = d.b.st[1] ? d.b.st[1] : HW;
  T* out0 = reinterpret_cast<T*>(d.out) + int64_t(nb0) * on + int64_t(c) * oc;
  T* dact0 = d.b.ptr ? reinterpret_cast<T*>(d.b.ptr) + int64_t(nb0) * on + int64_t(c) * oc : nullptr;
  for (int t = threadIdx.x; t < min(UV, 32); t += kThreads) ctoff[t] = t * pitch - (t / V) * Xo - (t % V);
  __syncthreads();
  // item (g, y, x) advanced by kThreads per iteration without divisions
  const int dy = kThreads / W, dx = kThreads - dy * W;
  int g = threadIdx.x / HW, r0 = threadIdx.x - g * HW;
  int y = r0 / W, x = r0 - y * W;
  for (; g < Gn;) {
    const T* col = col0 + int64_t(g) * img;
    const int u_lo = max(0, y - Yo + 1), u_hi = min(U - 1, y);
    const int v_lo = max(0, x - Xo + 1), v_hi = min(V - 1, x);
    float acc = 0.f;
    if (UV <= 32) {
      const uint32_t vb = (2u << v_hi) - (1u << v_lo);
      uint32_t mask = 0;
      for (int u = u_lo; u <= u_hi; ++u) mask |= vb << (u * V);
      const T* p0 = col + y * Xo + x;
      if (UV == 9) acc = col2im_masked<9>(p0, ctoff, mask, UV);
      else if (UV == 25) acc = col2im_masked<25>(p0, ctoff, mask, UV);
      else acc = col2im_masked<0>(p0, ctoff, mask, UV);
    } else {
      for (int u = u_lo; u <= u_hi; ++u) {
        const T* crow = col + int64_t(u * V) * pitch + (y - u) * Xo;
#pragma unroll 4
        for (int vv = v_lo; vv <= v_hi; ++vv) acc += eld(crow + int64_t(vv) * pitch + (x - vv));
      }
    }
    const int64_t o = int64_t(g) * on + y * W + x;
    est(out0 + o, acc);
    if (dact0) {
      float h = acc;  // the stored value
      if constexpr (sizeof(T) == 2) h = __bfloat162float(__float2bfloat16_rn(acc));
      const float t = tanhf(h);
      est(dact0 + o, 1.0f - t * t);
    }
    x += dx;
    y += dy;
    if (x >= W) { x -= W; ++y; }
    while (y >= H) { y -= H; ++g; }
  }
}

template <class T>
__device__ __forceinline__ void shiftpad_body(const ConvDesc& d, int tile) {
  // V shifted copies of a [n, o, y, x] view into a channel-major grid (V = 1: a plain layout
  // change, e.g. the gradient permuted for grad_weight):
  //   out[v*vst + o*ld + n*Sp + top + y*Wp + x + v] = a[n, o, y, x]
  // block = (channel o, group of G images); items over the group's flat (image, y, x), read
  // once (coalesced along x), written V times (coalesced runs).
  const int NB = int(d.a.shape[0]);
  const int V = int(d.p[0]), Yo = int(d.p[1]), Xo = int(d.p[2]), G = int(d.p[7]);
  const int64_t Wp = d.p[3], Sp = d.p[4], vst = d.p[5], ld = d.p[6], top = d.b.st[0];
  const int YX = Yo * Xo, ngrp = (NB + G - 1) / G;
  const int o = tile / ngrp, gb = tile - o * ngrp;
  const int nb0 = gb * G, Gn = min(G, NB - nb0);
  const T* src = reinterpret_cast<const T*>(d.a.ptr) + int64_t(nb0) * d.a.st[0] + int64_t(o) * d.a.st[1];
  T* dst = reinterpret_cast<T*>(d.out) + int64_t(o) * ld + int64_t(nb0) * Sp + top;
  // 4 items in flight per thread: item i = threadIdx.x + k * kThreads
  for (int it0 = threadIdx.x; it0 < Gn * YX; it0 += 4 * kThreads) {
    T val[4];
    int64_t dof[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int it = it0 + j * kThreads;
      dof[j] = -1;
      if (it < Gn * YX) {
        const int g = it / YX, r = it - g * YX, y = r / Xo, x = r - y * Xo;
        val[j] = src[int64_t(g) * d.a.st[0] + int64_t(y) * d.a.st[2] + int64_t(x) * d.a.st[3]];
        dof[j] = int64_t(g) * Sp + int64_t(y) * Wp + x;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (dof[j] >= 0)
        for (int v = 0; v < V; ++v) dst[dof[j] + v * (vst + 1)] = val[j];
  }
}

// 64 x 64 tiles of a 2-D transpose through shared memory (padded rows: conflict-free both
// ways), kTrTiles consecutive column tiles per block; every thread keeps its 16 loads in flight
// before the shared-memory writes.  Reads and writes are 256-byte coalesced runs.
constexpr int kTrTiles = 4;
template <class T>
__device__ __forceinline__ void transpose_body(const ConvDesc& d, int tile) {
  extern __shared__ __align__(16) unsigned char move_smem[];
  T* sm = reinterpret_cast<T*>(move_smem);  // [64][65]
  const int64_t R = d.a.shape[0], C = d.a.shape[1], rs = d.a.st[0], ot = d.p[0];
  const int64_t tcg = (C + 64 * kTrTiles - 1) / (64 * kTrTiles);
  const int64_t r0 = (tile / tcg) * 64, cg0 = (tile % tcg) * 64 * kTrTiles;
  const T* src = reinterpret_cast<const T*>(d.a.ptr);
  T* dst = reinterpret_cast<T*>(d.out);
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4 threads
  for (int t = 0; t < kTrTiles; ++t) {
    const int64_t c0 = cg0 + 64 * t;
    if (c0 >= C) break;
    T v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t r = r0 + ty + 4 * j, c = c0 + tx;
      if (r < R && c < C) v[j] = src[r * rs + c];
    }
    if (t > 0) __syncthreads();  // the previous tile's reads of sm are done
#pragma unroll
    for (int j = 0; j < 16; ++j) sm[(ty + 4 * j) * 65 + tx] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t c = c0 + ty + 4 * j, r = r0 + tx;
      if (c < C && r < R) dst[c * ot + r] = sm[tx * 65 + ty + 4 * j];
    }
  }
}

template <class T, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) premove_kernel(const ConvDesc* __restrict__ ds, int n) {
  const int di = find_desc(&ds[0].tile_begin, sizeof(ConvDesc), n, blockIdx.x);
  const ConvDesc& d = ds[di];
  const int tile = int(int64_t(blockIdx.x) - d.tile_begin);
  if (d.mode == CONV_IM2COL) im2col_body<T>(d, tile);
  else if (d.mode == CONV_TRANSPOSE) transpose_body<T>(d, tile);
  else shiftpad_body<T>(d, tile);
}

template <class T>
void upload(std::vector<T>& v, void** dptr) {
  if (*dptr) cudaFree(*dptr);
  *dptr = nullptr;
  if (v.empty()) return;
  CUDA_CHECK(cudaMalloc(dptr, v.size() * sizeof(T)));
  CUDA_CHECK(cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

}  // namespace

bool StridedView::contiguous() const {
  int64_t want = 1;
  for (int i = rank - 1; i >= 0; --i) {
    if (shape[i] != 1 && st[i] != want) return false;
    want *= shape[i];
  }
  return true;
}

NaryDesc nary_desc(int op, const StridedView& out, const std::vector<StridedView>& ins, float scale, int esize) {
  if (ins.empty() || int(ins.size()) > kMaxIn) fail("nary: bad operand count");
  NaryDesc d;
  std::memset(&d, 0, sizeof d);
  d.op = op;
  d.nin = int(ins.size());
  d.scale = scale;
  const int r = out.rank;
  for (const auto& v : ins)
    for (int i = 0; i < r; ++i)
      if (v.rank != r || v.shape[i] != out.shape[i]) fail("nary: operand shapes differ");
  // Collect dims (outer..inner), drop extent-1 dims, merge dims contiguous in every operand.
  struct Dim {
    int64_t n, so, si[kMaxIn];
  };
  std::vector<Dim> dims;
  for (int i = 0; i < r; ++i) {
    if (out.shape[i] == 1) continue;
    Dim x;
    x.n = out.shape[i];
    x.so = out.st[i];
    for (size_t k = 0; k < ins.size(); ++k) x.si[k] = ins[k].st[i];
    dims.push_back(x);
  }
  std::vector<Dim> merged;
  for (const auto& x : dims) {
    if (!merged.empty()) {
      Dim& p = merged.back();
      bool ok = p.so == x.so * x.n;
      for (size_t k = 0; k < ins.size() && ok; ++k) ok = p.si[k] == x.si[k] * x.n;
      if (ok) {
        p.n *= x.n;
        p.so = x.so;
        for (size_t k = 0; k < ins.size(); ++k) p.si[k] = x.si[k];
        continue;
      }
    }
    merged.push_back(x);
  }
  if (merged.size() > size_t(kMaxRank)) fail("nary: view rank too high after merging");
  const int pad = kMaxRank - int(merged.size());
  for (int i = 0; i < kMaxRank; ++i) {
    if (i < pad) {
      d.shape[i] = 1;
      d.out_st[i] = 0;
      for (size_t k = 0; k < ins.size(); ++k) d.in_st[k][i] = 0;
    } else {
      const Dim& x = merged[size_t(i - pad)];
      d.shape[i] = x.n;
      d.out_st[i] = x.so;
      for (size_t k = 0; k < ins.size(); ++k) d.in_st[k][i] = x.si[k];
    }
  }
  d.out = out.ptr;
  for (size_t k = 0; k < ins.size(); ++k) d.in[k] = ins[k].ptr;
  // 4-wide path: unit inner stride everywhere, inner extent % 4, rows aligned to 4 elements.
  const uintptr_t al = uintptr_t(4 * esize - 1);
  bool v4 = d.shape[3] % 4 == 0 && d.out_st[3] == 1 && (reinterpret_cast<uintptr_t>(d.out) & al) == 0;
  for (int i = 0; i < 3 && v4; ++i) v4 = d.out_st[i] % 4 == 0;
  for (size_t k = 0; k < ins.size() && v4; ++k) {
    v4 = d.in_st[k][3] == 1 && (reinterpret_cast<uintptr_t>(d.in[k]) & al) == 0;
    for (int i = 0; i < 3 && v4; ++i) v4 = d.in_st[k][i] % 4 == 0;
  }
  d.vec = v4 ? 4 : 1;
  d.units = out.elements() / d.vec;
  return d;
}

void nary_prepare(NaryBatch& b) {
  std::vector<NaryDev> dev(b.descs.size());
  // tile size: as large as kTileUnits while the batch still gives >= ~8 blocks per SM, smaller
  // for small batches (a 4 MB strided copy should not run on 32 blocks)
  int64_t total = 0;
  for (const auto& d : b.descs) total += d.units;
  int64_t tile = kTileUnits;
  while (tile > 1024 && total / tile < 8 * 148) tile /= 2;
  int64_t tiles = 0;
  b.bytes = 0;
  for (size_t i = 0; i < b.descs.size(); ++i) {
    NaryDesc& d = b.descs[i];
    const int64_t rows = d.shape[0] * d.shape[1] * d.shape[2];
    const int64_t inner = d.shape[3] / d.vec;
    RowTiling t = row_tiling(rows, inner, tile);
    d.tile_begin = tiles;
    tiles += ((rows + t.rpt - 1) / t.rpt) * t.n_col_chunks;
    dev[i] = NaryDev{d, t.rows, t.inner, t.rpt, t.col_chunk, t.n_col_chunks, t.rg};
    const double elems = double(d.units) * d.vec;
    int streams = d.nin + 1 + (d.op == NARY_ACC ? 1 : 0);
    for (int c = 0; c < d.n_chain; ++c) streams += 1 + (d.chain[c].other ? 1 : 0);
    b.bytes += (b.bf16 ? 2.0 : 4.0) * elems * streams;
  }
  b.tiles = tiles;
  b.copy_only = true;
  for (const auto& d : b.descs) b.copy_only = b.copy_only && d.op == NARY_COPY && d.n_chain == 0;
  std::vector<int> owner(static_cast<size_t>(tiles));
  for (size_t i = 0; i < b.descs.size(); ++i) {
    const int64_t end = i + 1 < b.descs.size() ? b.descs[i + 1].tile_begin : tiles;
    for (int64_t q = b.descs[i].tile_begin; q < end; ++q) owner[size_t(q)] = int(i);
  }
  upload(dev, &b.d_descs);
  upload(owner, &b.d_tile_desc);
}

void nary_run(const NaryBatch& b, cudaStream_t s) {
  if (!b.tiles) {
    if (b.signal_s >= 0) sync_signal(b.sync, b.signal_s, false, s);  // nothing to move: still publish
    return;
  }
  const NaryDev* ds = static_cast<const NaryDev*>(b.d_descs);
  const int* td = static_cast<const int*>(b.d_tile_desc);
  // register budgets (min resident blocks per SM); debug override TPX_NARY_MINB=<nary>,<copy>
  // (copy 3 -> 4: cfg2 data k3 conversions 3.60 -> 3.51 ms, loop k3 0.219 -> 0.203 ms; 6 spills;
  // nary 2 / 3 / 4 measured equal)
  static int mb_nary = 2, mb_copy = 4, mb_init = 0;
  if (!mb_init) {
    mb_init = 1;
    if (const char* e = std::getenv("TPX_NARY_MINB")) std::sscanf(e, "%d,%d", &mb_nary, &mb_copy);
  }
  const unsigned g = unsigned(b.tiles);
#define TPX_COPY(T) (mb_copy >= 6 ? copy_kernel<T, 6> : mb_copy >= 4 ? copy_kernel<T, 4> : copy_kernel<T, 3>)
#define TPX_NARY(T) (mb_nary >= 4 ? nary_kernel<T, 4> : mb_nary == 3 ? nary_kernel<T, 3> : nary_kernel<T, 2>)
  if (b.copy_only) {
    if (b.bf16) TPX_COPY(__nv_bfloat16)<<<g, kThreads, 0, s>>>(ds, td, b.sync, b.signal_s, b.wait_s);
    else TPX_COPY(float)<<<g, kThreads, 0, s>>>(ds, td, b.sync, b.signal_s, b.wait_s);
    CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (b.bf16) TPX_NARY(__nv_bfloat16)<<<g, kThreads, 0, s>>>(ds, td, b.sync, b.signal_s, b.wait_s);
  else TPX_NARY(float)<<<g, kThreads, 0, s>>>(ds, td, b.sync, b.signal_s, b.wait_s);
#undef TPX_COPY
#undef TPX_NARY
  CUDA_CHECK(cudaGetLastError());
}

void numeric_check_run(const NaryBatch& b, unsigned* dev_out, cudaStream_t s) {
  if (!b.tiles) return;
  const NaryDev* ds = static_cast<const NaryDev*>(b.d_descs);
  const int* td = static_cast<const int*>(b.d_tile_desc);
  if (b.bf16) check_kernel<__nv_bfloat16><<<unsigned(b.tiles), kThreads, 0, s>>>(ds, td, dev_out);
  else check_kernel<float><<<unsigned(b.tiles), kThreads, 0, s>>>(ds, td, dev_out);
  CUDA_CHECK(cudaGetLastError());
}

void sync_signal(const PeerSync& s, int index, bool barrier, cudaStream_t st) {
  sync_kernel<<<1, 32, 0, st>>>(s, index, barrier ? 1 : 0);
  CUDA_CHECK(cudaGetLastError());
}

bool nary_add_chain(NaryDesc& d, const StridedView& d_out, int op, float scale, const StridedView& out,
                    const StridedView* other, int esize) {
  if (d.n_chain >= kMaxChain || d.op == NARY_ACC) return false;
  auto same = [&](const StridedView& v) {
    if (v.rank != d_out.rank) return false;
    for (int i = 0; i < v.rank; ++i)
      if (v.shape[i] != d_out.shape[i] || (v.shape[i] != 1 && v.st[i] != d_out.st[i])) return false;
    return true;
  };
  if (!same(out) || (other && !same(*other))) return false;
  const uintptr_t al = uintptr_t(4 * esize - 1);
  if (d.vec == 4 && ((reinterpret_cast<uintptr_t>(out.ptr) & al) ||
                     (other && (reinterpret_cast<uintptr_t>(other->ptr) & al))))
    return false;
  ChainStage& c = d.chain[d.n_chain++];
  c.op = op;
  c.scale = scale;
  // stage views share d_out's layout, so they are indexed with the descriptor's (merged)
  // output strides relative to their own base
  c.out = out.ptr;
  c.other = other ? other->ptr : nullptr;
  return true;
}

void nary_free(NaryBatch& b) {
  if (b.d_descs) cudaFree(b.d_descs);
  if (b.d_tile_desc) cudaFree(b.d_tile_desc);
  b.d_descs = nullptr;
  b.d_tile_desc = nullptr;
}

uint64_t fnv1a(const char* s, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(s[i]);
    h *= 0x100000001B3ull;
  }
  return h;
}

void init_prepare(InitBatch& b) {
  std::vector<InitDev> dev(b.descs.size());
  int64_t tiles = 0;
  for (size_t i = 0; i < b.descs.size(); ++i) {
    InitDesc& d = b.descs[i];
    const int64_t rows = d.ext[0] * d.ext[1] * d.ext[2];
    RowTiling t = row_tiling(rows, d.ext[3]);
    d.tile_begin = tiles;
    tiles += ((rows + t.rpt - 1) / t.rpt) * t.n_col_chunks;
    dev[i] = InitDev{d, t.rows, t.inner, t.rpt, t.col_chunk, t.n_col_chunks, t.rg};
  }
  b.tiles = tiles;
  upload(dev, &b.d_descs);
}

void init_run(const InitBatch& b, cudaStream_t s) {
  if (!b.tiles) return;
  if (b.bf16)
    init_kernel<__nv_bfloat16><<<unsigned(b.tiles), kThreads, 0, s>>>(static_cast<const InitDev*>(b.d_descs),
                                                                      int(b.descs.size()));
  else
    init_kernel<float><<<unsigned(b.tiles), kThreads, 0, s>>>(static_cast<const InitDev*>(b.d_descs),
                                                              int(b.descs.size()));
  CUDA_CHECK(cudaGetLastError());
}

void init_free(InitBatch& b) {
  if (b.d_descs) cudaFree(b.d_descs);
  b.d_descs = nullptr;
}

void conv_prepare(ConvBatch& b) {
  int64_t tiles = 0;
  b.move = !b.descs.empty() && b.descs[0].mode >= CONV_IM2COL;
  b.smem = 0;
  b.bytes = 0;
  const int64_t es = b.bf16 ? 2 : 4;
  for (auto& d : b.descs) {
    if (d.mode == CONV_IM2COL) {  // input read once, every column written
      b.bytes += double(es) * (double(d.a.elements()) +
                               double(d.a.shape[1] * d.p[0] * d.p[1]) * double(d.a.shape[0] * d.p[2] * d.p[3]));
    } else if (d.mode == CONV_COL2IM) {  // every column read once, h (and 1 - tanh^2 h) written
      const double outs = double(d.n) * double(d.p[4] + d.p[2] - 1);
      b.bytes += double(es) * (double(d.p[0] * d.p[1] * d.p[2]) * double(d.a.shape[0] * d.p[3] * d.p[4]) +
                               outs * (d.b.ptr ? 2.0 : 1.0));
    } else if (d.mode == CONV_SHIFTPAD) {
      b.bytes += double(es) * double(d.a.elements()) * double(1 + d.p[0]);
    } else if (d.mode == CONV_TRANSPOSE) {
      b.bytes += 2.0 * double(es) * double(d.a.shape[0] * d.a.shape[1]);
    }
    if ((d.mode >= CONV_IM2COL) != b.move) throw std::runtime_error("conv batch mixes compute and data movement");
    if (b.move && (d.mode == CONV_COL2IM) != (b.descs[0].mode == CONV_COL2IM))
      throw std::runtime_error("conv batch mixes col2im with pre-GEMM movement");
    d.tile_begin = tiles;
    if (b.move) {
      const int64_t NB = std::max<int64_t>(d.a.shape[0], 1);
      if (d.mode == CONV_TRANSPOSE) {
        tiles += ((d.a.shape[0] + 63) / 64) * ((d.a.shape[1] + 64 * kTrTiles - 1) / (64 * kTrTiles));
        b.smem = std::max<int64_t>(b.smem, 64 * 65 * es);
      } else if (d.mode == CONV_SHIFTPAD) {
        const int64_t YX = std::max<int64_t>(d.p[1] * d.p[2], 1);
        const int64_t G = std::min(NB, std::max<int64_t>(1, (4 * kThreads + YX - 1) / YX));
        d.p[7] = G;
        tiles += d.a.shape[1] * ((NB + G - 1) / G);
      } else if (d.mode == CONV_IM2COL) {
        // G images per block: ~8 items per thread (measured best of 2..16), planes within the
        // staging buffer
        const int64_t U = d.p[0], V = d.p[1], YX = d.p[2] * d.p[3];
        const int64_t HW = (d.p[2] + U - 1) * (d.p[3] + V - 1), UV = U * V;
        int64_t G = std::max<int64_t>(1, (8 * kThreads + YX - 1) / std::max<int64_t>(YX, 1));
        G = std::min({G, NB, kMoveSmem / (HW * es)});  // 0: plane too large, read from global
        const int64_t Gb = std::max<int64_t>(G, 1);
        const int64_t blocks = d.a.shape[1] * ((NB + Gb - 1) / Gb);
        // split the taps when the (c, group) blocks alone do not fill the GPU
        const int64_t nch = std::min<int64_t>(UV, std::max<int64_t>(1, (4 * 148 + blocks - 1) / blocks));
        int64_t TC = (UV + nch - 1) / nch;
        TC = std::min<int64_t>(TC, kMaxTapChunk);
        d.p[6] = TC;
        d.p[7] = G;
        tiles += blocks * ((UV + TC - 1) / TC);
        b.smem = std::max<int64_t>(b.smem, G * HW * es);
      } else {
        const int64_t HW = (d.p[3] + d.p[1] - 1) * (d.p[4] + d.p[2] - 1);
        const int64_t G = std::min(NB, std::max<int64_t>(1, (8 * kThreads + HW - 1) / std::max<int64_t>(HW, 1)));
        d.p[7] = G;
        tiles += d.p[0] * ((NB + G - 1) / G);
      }
    } else {
      tiles += (d.n + kThreads - 1) / kThreads;
    }
  }
  b.tiles = tiles;
  upload(b.descs, &b.d_descs);
}

void conv_run(const ConvBatch& b, cudaStream_t s) {
  if (!b.tiles) return;
  const ConvDesc* ds = static_cast<const ConvDesc*>(b.d_descs);
  const int nd = int(b.descs.size());
  const size_t sm = size_t(b.smem);
  const bool col2im = b.move && b.descs[0].mode == CONV_COL2IM;

  // register budget (min resident blocks per SM) of the data-movement kernels; debug override
  // TPX_MOVE_MINB=<premove>,<col2im> for A/B runs
  // (measured on the AlexNet-style conv step: premove 1 -> 4 blocks, im2col 1.67 -> 1.30 ms;
  // col2im 4 -> 6 blocks, 2.00 -> 1.79 ms; 8 blocks spill and run 1.6x slower)
  static int mb_pre = 4, mb_c2i = 6, mb_init = 0;
  if (!mb_init) {
    mb_init = 1;
    if (const char* e = std::getenv("TPX_MOVE_MINB")) std::sscanf(e, "%d,%d", &mb_pre, &mb_c2i);
  }
  const unsigned g = unsigned(b.tiles);
#define TPX_C2I(T) \
  (mb_c2i >= 8 ? col2im_kernel<T, 8> : mb_c2i == 6 ? col2im_kernel<T, 6> : mb_c2i == 5 ? col2im_kernel<T, 5> \
   : mb_c2i == 3 ? col2im_kernel<T, 3> : mb_c2i <= 2 ? col2im_kernel<T, 2> : col2im_kernel<T, 4>)
#define TPX_PRE(T) \
  (mb_pre >= 8 ? premove_kernel<T, 8> : mb_pre >= 6 ? premove_kernel<T, 6> : mb_pre >= 4 ? premove_kernel<T, 4> : premove_kernel<T, 1>)
  if (col2im && b.bf16) TPX_C2I(__nv_bfloat16)<<<g, kThreads, 0, s>>>(ds, nd);
  else if (col2im) TPX_C2I(float)<<<g, kThreads, 0, s>>>(ds, nd);
  else if (b.move && b.bf16) TPX_PRE(__nv_bfloat16)<<<g, kThreads, sm, s>>>(ds, nd);
  else if (b.move) TPX_PRE(float)<<<g, kThreads, sm, s>>>(ds, nd);
#undef TPX_C2I
#undef TPX_PRE
  else if (b.bf16) conv_kernel<__nv_bfloat16><<<unsigned(b.tiles), kThreads, 0, s>>>(ds, nd);
  else conv_kernel<float><<<unsigned(b.tiles), kThreads, 0, s>>>(ds, nd);
  CUDA_CHECK(cudaGetLastError());
}

void conv_free(ConvBatch& b) {
  if (b.d_descs) cudaFree(b.d_descs);
  b.d_descs = nullptr;
}

void f32_to_f64_host(const float* src, double* dst, int64_t n) {
  for (int64_t i = 0; i < n; ++i) dst[i] = double(src[i]);
}

}  // namespace tpx
