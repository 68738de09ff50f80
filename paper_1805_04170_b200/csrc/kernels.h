// Bandwidth kernels of the executor (all batched: one launch per phase step).
//   nary    strided N-d box copy / accumulate / elementwise over up to 8 operands:
//           K3 pack/unpack (extract_region / paste_region, dense.cpp:213-259),
//           K4 partial-sum reduce in source order (reduce_partial, simulator.cpp:106-115),
//           K5 elementwise sub-ops not folded into a GEMM (run_op_dense, dense.cpp:170-204).
//   init    K6 seeded inputs on device (seeded_tensor, dense.cpp:30-57), bit-exact fp64 -> fp32.
//   conv    direct convolution sub-ops (run_conv, dense.cpp:92-157).
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace tpx {

constexpr int kMaxRank = 4;
constexpr int kMaxIn = 8;
constexpr int kMaxChain = 3;
constexpr int kMaxRanks = 8;

enum NaryOp : int {
  NARY_COPY = 0,   // out = in0
  NARY_SUM = 1,    // out = in0 + in1 + ... (left to right)
  NARY_SUB = 2,    // out = in0 - in1
  NARY_SCALE = 3,  // out = s * in0
  NARY_TANH = 4,   // out = tanh(in0)
  NARY_DTANH = 5,  // out = 1 - tanh(in0)^2
  NARY_ACC = 6,    // out += in0
};

// A strided view (element strides), rank <= 4.  `ptr` is an opaque device address; the element
// type (fp32 or bf16) is the plan's storage type.
struct StridedView {
  float* ptr = nullptr;
  int rank = 0;
  int64_t shape[kMaxRank] = {1, 1, 1, 1};
  int64_t st[kMaxRank] = {0, 0, 0, 0};
  int64_t elements() const {
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= shape[i];
    return n;
  }
  bool contiguous() const;
};

// An elementwise stage chained onto an n-ary result (EpiOp codes of gemm.h: tanh, 1 - tanh^2,
// scale, add, sub): reads the previous stage's STORED value, writes `out`, which has the layout
// of the descriptor's output (so has `other`).  Used to fuse the consumers of a partial-sum
// reduction (the SGD step + update of a reduced gradient, the activation of a reduced
// pre-activation) into the reduction's launch.
struct ChainStage {
  int op = 0;
  float scale = 0.f;
  float* out = nullptr;
  const float* other = nullptr;
};

struct NaryDesc {
  int op = NARY_COPY;
  int nin = 1;
  int vec = 1;          // 1 or 4 elements per access
  float scale = 0.f;
  int64_t shape[kMaxRank];  // normalised to rank 4 (leading 1s), dims merged where possible
  float* out;
  int64_t out_st[kMaxRank];
  const float* in[kMaxIn];
  int64_t in_st[kMaxIn][kMaxRank];
  int64_t tile_begin;   // prefix over the batch (filled by nary_prepare)
  int64_t units;        // number of vec-wide units
  int n_chain;          // chained elementwise stages (0 = none)
  ChainStage chain[kMaxChain];
  uint32_t wait_mask;   // peer pull: ranks whose sync counter must reach this rank's first
};

// Cross-rank ordering of peer-pull steps (TPX_FLAG_PEER).  Every rank owns two 64-bit words at
// the start of its arena: a counter the other ranks read (they map the arena, CUDA IPC over
// NVLink) and its step epoch E (the barriers it has passed).  At sync point s of a step -- the
// first conversion launch of a phase in which any rank pulls -- every rank publishes
// E * kSyncK + s + 1 (fence + st.release.sys, from any launch that runs after the phase's producers:
// the phase's own pull / reduce launch, or a one-thread kernel when the rank has none); a pull
// waits until each rank it reads from has published at least that value (ld.acquire.sys), so the
// data it reads is complete.  A barrier ends each step (E * kSyncK + kSyncK - 1 from every rank,
// then E + 1), so no rank overwrites a value another rank may still read; a pull of the carry
// program, which runs right after a barrier, waits for the previous barrier's value.
constexpr unsigned long long kSyncK = 1ull << 20;
struct PeerSync {
  unsigned long long* local = nullptr;  // this rank's counter (arena word 0)
  unsigned long long* epoch = nullptr;  // this rank's step epoch (arena word 1)
  const unsigned long long* peer[kMaxRanks] = {};
  int* err = nullptr;                   // host-mapped: 0x100 | rank on a wait that timed out
  int world = 1, rank = 0;
  unsigned long long timeout_ns = 0;
};
void sync_signal(const PeerSync& s, int index, bool barrier, cudaStream_t st);

struct NaryBatch {
  bool bf16 = false;  // storage type of every operand (arithmetic is fp32)
  bool pull = false;  // some descriptor reads peer memory (waits on PeerSync first)
  bool copy_only = false;  // every descriptor a plain copy: the light copy kernel (nary_prepare)
  int signal_s = -1;  // peer mode: this launch publishes sync point signal_s (see PeerSync)
  int wait_s = -1;    // ... and its pulls wait for the peers' sync point wait_s (-1: last barrier)
  void* d_tile_desc = nullptr;  // int32 per block: its descriptor (no per-block search)
  PeerSync sync;
  std::vector<NaryDesc> descs;
  void* d_descs = nullptr;
  int64_t tiles = 0;
  double bytes = 0;  // algorithmic bytes moved (reads + writes)
};

// Build a descriptor: out[i] = op(in_0[i], ...), all views of equal shape.
NaryDesc nary_desc(int op, const StridedView& out, const std::vector<StridedView>& ins,
                   float scale = 0.f, int esize = 4);
// Chain an elementwise stage onto d (see ChainStage): `out` (and `other`, for add / sub) must
// have the shape and strides of `d_out`, the view d was built for.  False when the layouts or
// the alignment of the 4-wide path do not allow it (the caller then runs the op unfused).
bool nary_add_chain(NaryDesc& d, const StridedView& d_out, int op, float scale, const StridedView& out,
                    const StridedView* other, int esize);
void nary_prepare(NaryBatch& b);  // uploads descriptor table
// K7, the on-device NumericCheck reduction (simulator.cpp:129-147): over every descriptor of b
// (in[0] = the tiled value, in[1] = the single-device truth over the same region), the max of
// |d| and of |d| / max(|truth|, 1) into dev_out[0..1] (fp32 bit patterns, atomically max-ed;
// both are >= 0).  b must be prepared.
void numeric_check_run(const NaryBatch& b, unsigned* dev_out, cudaStream_t s);
void nary_run(const NaryBatch& b, cudaStream_t s);
void nary_free(NaryBatch& b);

struct InitDesc {
  float* out;
  uint64_t state0;                 // seed ^ fnv1a(tensor id)
  int rank;
  int64_t full[kMaxRank];          // full tensor shape (row-major stream order)
  int64_t lo[kMaxRank];            // region origin
  int64_t ext[kMaxRank];           // region extent
  int64_t n;
  int64_t tile_begin;
};

struct InitBatch {
  bool bf16 = false;  // storage type written (seeded fp64 -> fp32 -> bf16, round to nearest)
  std::vector<InitDesc> descs;
  void* d_descs = nullptr;
  int64_t tiles = 0;
};
void init_prepare(InitBatch& b);
void init_run(const InitBatch& b, cudaStream_t s);
void init_free(InitBatch& b);
uint64_t fnv1a(const char* s, size_t n);

// Direct convolution modes (run_conv on CUDA cores, kept as the cross-check path) and the
// data-movement kernels of the tensor-core lowering (conv = im2col + tcgen05 GEMM [+ col2im]).
enum ConvModeCode : int {
  CONV_FWD = 0, CONV_GRAD_W = 1, CONV_GRAD_IN = 2,
  CONV_IM2COL = 4,       // out[(c*U*V+u*V+v)*pitch + n*img + y*Xo+x] = a[n,c,y+u,x+v]
                         //   (d.n = rows (k, n, y); col2im: d.n = rows (n, c, y))
                         //   (p = U,V,Yo,Xo,pitch,img; img >= Yo*Xo per-image column stride,
                         //   pitch >= N*img, 16-byte rows)
  CONV_SHIFTPAD = 6,     // out[v*p5 + o*p6 + n*p4 + b.st[0] + y*p3 + x + v] = a[n,o,y,x], v < p0
                         //   (p = V,Yo,Xo,Wp,Sp,vstride,ld): a [n,o,y,x] view copied into a
                         //   channel-major grid, V column-shifted copies (V = 1: the gradient
                         //   permuted for grad_weight)
  CONV_TRANSPOSE = 7,    // out[c * p0 + r] = a[r * a.st[0] + c] for r < a.shape[0], c < a.shape[1]
                         //   (a rank-2 row-major view; p0 = the transposed rows' pitch): operands
                         //   made K-major for the tensor cores (kind::tf32 reads MN-major operands
                         //   at about half rate)
  CONV_COL2IM = 5,       // out[n,c,y,x] = sum_{u,v} col[(c*U*V+u*V+v)*pitch + n*img + (y-u)*Xo+(x-v)]
                         //   (a.ptr = col, a.shape[0] = N, p = C,U,V,Yo,Xo,pitch,img; taps in
                         //   ascending (u, v) order; b.ptr != null: also b[...] = 1 - tanh(out)^2;
                         //   b.st[0], b.st[1] = image / channel strides of out and b, 0 = dense)
                         //   p[6..7] = launch geometry, set by conv_prepare
};
struct ConvDesc {
  int mode;
  StridedView a, b;   // rank-4 operands as run_conv receives them
  float* out;         // contiguous output
  int64_t oshape[4];
  int64_t n;          // output elements
  int64_t p[8];       // mode parameters (see ConvModeCode)
  int64_t tile_begin;
};
struct ConvBatch {
  std::vector<ConvDesc> descs;
  void* d_descs = nullptr;
  int64_t tiles = 0;
  double flops = 0;
  bool move = false;  // im2col / col2im batch (d.n counts rows) rather than direct conv
  int64_t smem = 0;   // dynamic shared memory of the im2col launch
  bool bf16 = false;  // storage type
  double bytes = 0;   // algorithmic bytes of a data-movement batch (im2col / col2im / copies)
};
void conv_prepare(ConvBatch& b);
void conv_run(const ConvBatch& b, cudaStream_t s);
void conv_free(ConvBatch& b);

// fp32 <-> fp64 conversion helpers for host I/O of node values.
void f32_to_f64_host(const float* src, double* dst, int64_t n);

}  // namespace tpx
