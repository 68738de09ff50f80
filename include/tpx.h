/* tpx.h — C ABI of the B200-native executor for tileplan execution plans.
 *
 * Drop-in replacement for the reference's hot path, the CPU plan executor
 *   NumericCheck execute_numeric(const ExecutionPlan&, uint64_t seed [, FunctionBindings])
 *       (reference: proj/include/tileplan/simulator.hpp:43-45, proj/src/simulator.cpp:55-149)
 * and its per-sub-op kernels / region movers
 *   run_op_dense, extract_region, paste_region   (proj/include/tileplan/dense.hpp:40-49)
 * consuming the reference planner's plan exactly as serialised by
 *   std::string export_plan(const ExecutionPlan&)  (proj/include/tileplan/execgraph.hpp:57,
 *                                                   proj/src/execgraph.cpp:323-361)
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.  Every entry
 * point returns 0 on success and a non-zero status on failure, with the message (naming the
 * offending node / tensor / op, like tileplan::Error, proj/include/tileplan/error.hpp:8-12)
 * available from tpx_last_error() on the calling thread.  Nothing throws across the ABI.
 *
 * Process model: one process per GPU.  A plan with 2^k logical devices is executed by `world`
 * ranks; logical device d belongs to rank (d * world) >> k (contiguous blocks).  With world=1
 * a single GPU hosts every logical device (fetches become HBM copies).  Cross-rank fetches
 * are either pulled straight out of the owning rank's arena over NVLink (TPX_FLAG_PEER: the
 * arenas are shared with CUDA IPC; the caller all-gathers the 64-byte handles, e.g. with
 * torch.distributed) or grouped per plan phase into NCCL send/recv groups (the communicator is
 * created from a 128-byte ncclUniqueId the caller distributes).
 */
#ifndef TPX_H_
#define TPX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPX_OK 0
#define TPX_ERR 1

/* Arithmetic of the per-GPU sub-op kernels. */
#define TPX_PREC_TF32 0   /* fp32 storage, tcgen05 kind::tf32 MMA, fp32 accumulate   */
#define TPX_PREC_FP32 1   /* fp32 storage, 3xTF32 split MMA (fp32-accurate products) */

/* tpx_plan_stats() keys */
typedef struct tpx_stats {
  int64_t fetch_bytes_total;      /* sum of fetch.bytes over the whole plan (all devices) */
  int64_t rank_fetch_bytes_in;    /* fetch bytes landing on this rank's devices          */
  int64_t rank_xrank_bytes_in;    /* ... of which cross a rank boundary (NCCL)           */
  int64_t rank_xrank_bytes_out;   /* bytes this rank sends to other ranks                */
  int64_t n_nodes;                /* plan nodes (all devices)                            */
  int64_t n_steps;                /* lowered launch steps on this rank                   */
  int64_t n_kernel_launches;      /* kernels per tpx_execute on this rank                */
  int64_t n_gemm_launches;
  int64_t n_copy_launches;
  int64_t n_nccl_groups;
  int64_t n_fused_ew;             /* elementwise sub-ops folded into a GEMM epilogue      */
  int64_t device_bytes;           /* HBM arena bytes allocated for node values           */
  double gemm_flops;              /* 2*M*N*K over this rank's matmul sub-ops             */
  double gemm_min_bytes;          /* operand + output bytes of those GEMMs (read once)   */
  int64_t storage_bytes;          /* bytes per stored element: 4 (fp32) or 2 (bf16 plan)  */
} tpx_stats;

const char* tpx_last_error(void);
int tpx_version(void);

/* ---------------------------------------------------------------- context */
typedef struct tpx_ctx tpx_ctx;

/* cuda_ordinal < 0 creates a host-only context: plans can be loaded, validated and lowered
 * (message tables, byte accounting) without a GPU, but not executed. */
int tpx_create(int cuda_ordinal, int rank, int world, tpx_ctx** out);
/* Multi-rank: create the NCCL communicator (world > 1).  `unique_id` is 128 bytes. */
int tpx_init_comm(tpx_ctx* ctx, const void* unique_id, size_t len);
/* Writes a fresh 128-byte ncclUniqueId (rank 0 calls this, then broadcasts it). */
int tpx_comm_unique_id(void* out, size_t len);
int tpx_destroy(tpx_ctx* ctx);

/* ---------------------------------------------------------------- plans */
typedef struct tpx_plan tpx_plan;

/* Parse + validate + lower a plan document (export_plan JSON, execgraph.cpp:323-361) for this
 * context's rank.  flags: bit0 = fuse elementwise sub-ops into GEMM epilogues (default on
 * when set), bit1 = route every cross-logical-device fetch through the NCCL path even when
 * both devices live on this rank (self send/recv; exercises the multi-rank data path on one
 * GPU). */
#define TPX_FLAG_FUSE 1
#define TPX_FLAG_FORCE_XCHG 2
/* Convolutions on CUDA cores (direct loops) instead of im2col + tcgen05 GEMM (cross-check). */
#define TPX_FLAG_DIRECT_CONV 4
/* Execute the step as one CUDA graph (captured on the first tpx_execute on a stream). */
#define TPX_FLAG_GRAPH 8
/* Training loop: tpx_execute runs one step AND carries the weights into the next one.  Every
 * weight whose w_next holder has the weight's own layout on each device (loop-consistent
 * tilings: data-parallel plans, the loop-aware optimum) trades storage with it -- the step is
 * lowered twice and consecutive steps alternate, so that carry costs no copy; the other
 * weights run the carry program (tpx_carry_weights' conversion) after the step.  Node reads
 * see the last executed step; tpx_init_inputs restarts the loop. */
#define TPX_FLAG_LOOP 16
/* Peer pull: every cross-rank fetch of a phase is ONE launch on the consuming rank that reads
 * the strided source boxes out of the owner's arena (CUDA IPC mapping over NVLink) and writes
 * them at their offsets in the consumer (pack, transfer and unpack in one pass; no NCCL).  A
 * partial consumed only by a reduce_partial is read in place by the reduction, which also runs
 * the sum's elementwise consumers (SGD step + update).  Ranks order themselves with device-side
 * counters in their arenas (a signal per phase with pulls, a barrier per step).  With world > 1
 * the plan runs only after tpx_plan_connect_peers; with world = 1 and TPX_FLAG_FORCE_XCHG every
 * cross-device fetch takes this path against the rank's own arena. */
#define TPX_FLAG_PEER 32
/* Conv grad_input GEMMs on K-major transposed copies of the filter and the gradient instead of
 * the stored MN-major operands (kind::tf32 reads MN-major operands at about half rate; the
 * transposes cost about what the faster GEMM saves, so this is opt-in). */
#define TPX_FLAG_KMAJOR_CONV 64
/* With TPX_FLAG_PEER and world > 1: run this rank alone, every peer arena stood in for by the
 * rank's own (no tpx_plan_connect_peers).  The rank's program is unchanged -- its compute, its
 * pull launches reading local HBM instead of NVLink, its sync points (already satisfied) -- so
 * one GPU measures one rank's share of an N-GPU step.  Values are meaningless; timing only. */
#define TPX_FLAG_PEER_SOLO 128
int tpx_load_plan(tpx_ctx* ctx, const char* plan_json, size_t len, int precision, int flags,
                  tpx_plan** out);
/* TPX_FLAG_PEER, world > 1: this rank's arena as a CUDA IPC handle (64 bytes) ... */
int tpx_plan_ipc_handle(tpx_plan* plan, void* out, size_t len);
/* ... and, with every rank's handle in rank order (world * 64 bytes), map the peers' arenas and
 * finish the load (lowering against the mapped addresses).  Collective: every rank calls it. */
int tpx_plan_connect_peers(tpx_plan* plan, const void* handles, size_t len);
int tpx_plan_free(tpx_plan* plan);
int tpx_plan_stats(const tpx_plan* plan, tpx_stats* out);
/* Lowered program as JSON (steps, per-phase message tables, byte counts) — host-only. */
int tpx_plan_describe(const tpx_plan* plan, char** json_out);
void tpx_free_string(char* s);

/* Fill every graph input's buffer node on this rank with seeded_tensor values
 * (proj/src/dense.cpp:49-57: splitmix64 keyed by seed ^ FNV-1a(tensor id), U[-1,1) in fp64,
 * rounded to fp32), generated on the GPU for exactly the node's region. */
int tpx_init_inputs(tpx_plan* plan, uint64_t seed);

/* Node values on this rank (fp64 host buffers, row-major over the node's region). */
int tpx_node_elements(const tpx_plan* plan, const char* node_id, int64_t* n);
int tpx_write_node(tpx_plan* plan, const char* node_id, const double* src, int64_t n);
int tpx_read_node(tpx_plan* plan, const char* node_id, double* dst, int64_t n);
/* Raw storage-type host <-> device for a node: n elements of the plan's storage type (fp32, or
 * bf16 for dtype_bytes-2 plans; tpx_stats.storage_bytes), pinned buffers give async copies on
 * the plan stream.  (tpx_read_node / tpx_write_node convert to / from fp64.) */
int tpx_write_node_f32(tpx_plan* plan, const char* node_id, const float* src, int64_t n);
int tpx_read_node_f32(tpx_plan* plan, const char* node_id, float* dst, int64_t n);
/* Device address + element strides of a node value (for zero-copy interop). */
int tpx_node_view(const tpx_plan* plan, const char* node_id, uint64_t* dev_ptr, int* rank,
                  int64_t* shape4, int64_t* strides4);

/* Stream the plan's kernels are enqueued on (0 = the context's own stream). */
int tpx_set_stream(tpx_plan* plan, uint64_t cuda_stream);
/* Execute every lowered step once (asynchronous on the plan stream). */
int tpx_execute(tpx_plan* plan);
/* Execute only the steps of the given op id (teacher-forced per-op checks). */
int tpx_execute_op(tpx_plan* plan, const char* op_id);
/* Loop carry: after a train step, copy each `<w>_next` tensor's holder blocks onto `<w>`'s
 * holder blocks (conversion between their tilings, fetching across devices as needed). */
int tpx_carry_weights(tpx_plan* plan);
/* NumericCheck on the device (execute_numeric's comparison, simulator.cpp:129-147): every holder
 * block of `tiled` on this rank against the same region of the one-device plan `serial`'s holder
 * (both executed, same GPU and storage type); max |d|, max |d| / max(|truth|, 1), values compared.
 * One reduction launch; nothing but the two maxima leaves the device. */
int tpx_numeric_check(tpx_plan* tiled, tpx_plan* serial, double* max_abs, double* max_rel, int64_t* values);
/* Waits for the plan stream; fails if a peer wait timed out (TPX_PEER_TIMEOUT_S, default 60 s). */
int tpx_synchronize(tpx_plan* plan);

/* Per-step device timing of the last tpx_execute (events around each step): total ms and
 * ms spent in GEMM launches. */
int tpx_last_timing(const tpx_plan* plan, double* total_ms, double* gemm_ms, double* copy_ms);
/* Steps [begin, end) of the lowered step program (the order of tpx_plan_describe()'s "main"
 * steps), on the plan stream; with TPX_FLAG_GRAPH each range is captured once as a CUDA graph.
 * Lets a caller overlap its own copies (next batch in, network output out) with the step. */
int tpx_execute_steps(tpx_plan* plan, int64_t begin, int64_t end);
/* Device-to-device copy between a node's holder block and n contiguous elements of the storage
 * type at `dev` (to_node != 0: into the node), on the plan stream. */
int tpx_copy_node_device(tpx_plan* plan, const char* node_id, void* dev, int64_t n, int to_node);
/* Per-step device times (ms) of the last timed execution, in the order of
 * tpx_plan_describe()'s "main" steps; fills min(n, *n_steps) entries. */
int tpx_last_step_times(const tpx_plan* plan, double* ms, int64_t n, int64_t* n_steps);
int tpx_enable_timing(tpx_plan* plan, int on);

/* ---------------------------------------------------------------- kernel-level entry points
 * Device pointers, fp32 storage (precision 0 = TF32, 1 = 3xTF32 fp32-accurate) or bf16 storage
 * (precision 2: every operand, output and epilogue operand is bf16; fp32 accumulate).  Used by
 * the kernel tests; the plan executor calls the same code.  out = op(A) . op(B) (run_matmul,
 * dense.cpp:71-90); a/b are row-major views with row strides (elements).  epi_* optionally
 * chain elementwise stages onto the product. */
int tpx_gemm(const float* a, int64_t a_rows, int64_t a_cols, int64_t a_rs, const float* b,
             int64_t b_rows, int64_t b_cols, int64_t b_rs, int transpose_a, int transpose_b,
             float* c, int64_t c_rs, int n_epi, const int* epi_ops, const float* epi_scales,
             const float* const* epi_other, const int64_t* epi_other_rs, float* const* epi_out,
             const int64_t* epi_out_rs, int precision, uint64_t cuda_stream);
/* tpx_gemm with the problem prepared once: `warmup` untimed runs, then `iters` runs timed with
 * CUDA events on `cuda_stream`; *avg_ms = mean device time per run (iters > 0). */
int tpx_gemm_timed(const float* a, int64_t a_rows, int64_t a_cols, int64_t a_rs, const float* b,
                   int64_t b_rows, int64_t b_cols, int64_t b_rs, int transpose_a, int transpose_b,
                   float* c, int64_t c_rs, int n_epi, const int* epi_ops, const float* epi_scales,
                   const float* const* epi_other, const int64_t* epi_other_rs, float* const* epi_out,
                   const int64_t* epi_out_rs, int precision, uint64_t cuda_stream, int warmup,
                   int iters, double* avg_ms);
/* Host-only: the persistent GEMM's tile schedule for `nprob` problems of P x Q x K (kernel
 * orientation, 128 x bn tiles, 32-deep k-blocks) on `num_sms` SMs; max_kb > 0 bounds every
 * segment to max_kb k-blocks (the 3xTF32 kernels' accumulation chains).  segs (8 int32 per segment:
 * prob, tp, tq, kb0, kb1, kind, slot, n_parts) and seg_off (grid+1) are filled when large
 * enough.  No GPU needed. */
int tpx_gemm_schedule(int nprob, int P, int Q, int K, int bn, int num_sms, int force_groups, int max_kb,
                      int* grid, int* nsegs, int* nslots, int* group, int* stream_k,
                      int32_t* segs, int max_segs, int32_t* seg_off, int max_ctas);
/* The variant the last tpx_gemm / tpx_gemm_timed on this thread launched (for tests that must
 * cover a specific kernel): fills min(n, 16) of
 *   bn, pair (cta_group::2 256-row tiles), swap (computed transposed), p_mn, q_mn (MN-major
 *   operands), oloader (operand-loader warp), other_smem (TMA-staged epilogue operand),
 *   stream_k, group, tstore (TMA-store epilogue), nbox, odepth, stages, units (CTAs), split
 *   (3xTF32), bf16. */
int tpx_gemm_last_launch(int64_t* info, int n);
/* Debug: per-CTA launch timeline of the last GEMM launched with knob (22, 1) (8 %globaltimer
 * stamps per CTA: entry, setup, first TMA, first k-block landed, MMA done, first accumulator,
 * epilogue done, exit); fills min(n, 320 * 8) values. */
int tpx_debug_gemm_trace(uint64_t* out, int n);
/* Debug: override the MN-major UMMA descriptor strides (bytes; 0 = defaults). */
int tpx_debug_gemm_mn_desc(unsigned lbo, unsigned sbo);

#ifdef __cplusplus
}
#endif
#endif /* TPX_H_ */
