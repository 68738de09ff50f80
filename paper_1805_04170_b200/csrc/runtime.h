// Plan lowering and execution: the B200 replacement for execute_numeric's node interpreter
// (proj/src/simulator.cpp:55-127).
//
// Lowering turns the per-device node list into a short program of batched launches for the
// logical devices this rank owns, phase by phase (phases as defined by
// ExecutionPlan::phase_order, execgraph.cpp:41-47):
//   sub_op nodes of the phase's op -> one grouped tcgen05 GEMM / conv / elementwise launch
//                                     (elementwise consumers folded into GEMM epilogues)
//   slice                           -> zero-copy strided view (or a copy straight into the
//                                     concat that consumes it)
//   fetch (same rank)               -> HBM copy (into the consuming concat when there is one)
//   fetch (other rank)              -> peer mode (TPX_FLAG_PEER): one pull launch per phase that
//                                     reads the remote strided boxes straight out of the peer's
//                                     arena over NVLink (CUDA IPC) and writes them at their place
//                                     in the consumer: pack + transfer + unpack in one pass;
//                                     otherwise pack (if strided) + NCCL send/recv group + unpack
//   concat                          -> one buffer; every piece lands at its offset
//   reduce_partial                  -> ordered sum of the partials (deterministic), reading
//                                     single-piece partials in place (local or on the peer) and
//                                     running the elementwise consumers of the sum (SGD step +
//                                     update, tanh, 1 - tanh^2) in the same launch
// Every node value is an immutable strided fp32 view into one HBM arena.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gemm.h"
#include "kernels.h"
#include "plan.h"

namespace tpx {

struct Ctx {
  int ordinal = -1;   // CUDA device, -1 = host-only (lowering / accounting, no execution)
  int rank = 0, world = 1;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  void* comm = nullptr;  // NCCL communicator (world > 1 or forced exchange)
  bool host_only() const { return ordinal < 0; }
};

enum StepKind { ST_NARY, ST_GEMM, ST_CONV, ST_XCHG, ST_SYNC };

struct Step {
  StepKind kind;
  int idx;             // into the batch vector of that kind
  std::string op;      // owning op id (phase prefix)
  std::string what;    // "pack" / "copy" / "reduce" / "ew" / "materialize" / "gemm" ...
  int barrier = 0;     // ST_SYNC: 1 = end-of-step barrier (signal + wait for every rank)
};

struct Xfer {
  int peer;
  bool send;
  void* ptr;
  size_t bytes;
  int node;            // fetch node index
};

struct XchgGroup {
  std::vector<Xfer> x;
  int64_t bytes_in = 0, bytes_out = 0;
};

struct Program {
  std::vector<Step> steps;
  std::vector<NaryBatch> nary;
  std::vector<std::vector<GemmSpec>> gemm_specs;
  std::vector<GemmLaunch> gemm;
  std::vector<ConvBatch> conv;
  std::vector<XchgGroup> xchg;
};

struct PlanRt {
  Ctx* ctx = nullptr;
  Plan plan;
  int precision = 0;
  int flags = 0;
  int esize = 4;                 // storage bytes per element: 4 fp32, 2 bf16 (the plan's dtype)
  std::vector<int> dev_rank;
  std::vector<StridedView> val;
  std::vector<char> has_val;
  std::vector<int> avail_step;   // first step index after which the value exists
  // arena
  char* arena = nullptr;
  size_t arena_bytes = 0, arena_used = 0;
  uintptr_t base = 0;
  // programs
  Program main, carry;
  // TPX_FLAG_LOOP: a second lowering of the step in which every loop-consistent weight's
  // buffers and its w_next holders trade storage, so consecutive steps alternate main / main_b
  // and the weights carry over with no copy (the loop carry of the paper's repeated training
  // step).  Weights whose w_next is tiled differently keep the carry program.
  Program main_b;
  std::vector<StridedView> val_b;        // node values as main_b leaves them
  std::vector<std::string> swapped;      // weight tensors carried by the swap
  int parity = 0;                        // program of the next step (0 main, 1 main_b)
  int last = 0;                          // program whose values the node reads see
  bool loop() const { return (flags & 16) != 0; }
  InitBatch init;
  // TPX_FLAG_PEER: cross-rank fetches are pulled from the peers' arenas (CUDA IPC mappings);
  // peer_base[r] = rank r's arena as mapped in this process (own arena for r == rank).  The
  // other ranks' node values come from a host-only lowering of the plan as that rank
  // (deterministic), stored relative to the dry-run base.
  bool peer() const { return (flags & 32) != 0; }
  std::vector<uintptr_t> peer_base;
  std::vector<std::vector<StridedView>> rval, rval_b;
  std::vector<std::vector<char>> rhas;
  std::vector<void*> ipc_opened;
  bool lowered = false;            // real (non-dry) lowering done
  int n_sync = 0;                  // sync points per step (signals + barrier)
  PeerSync sync;
  int* err_host = nullptr;         // host-mapped error word of the peer waits
  int64_t pull_bytes = 0;          // bytes this rank pulls from other ranks per step
  // accounting
  int64_t fetch_in = 0, xrank_in = 0, xrank_out = 0, carry_bytes = 0, carry_xrank = 0;
  int n_fused = 0;
  std::map<std::string, int64_t> op_bytes_in, phase_bytes_in;  // fetch bytes landing on this rank
  double gemm_flops = 0, gemm_min_bytes = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> events;
  double last_total_ms = 0, last_gemm_ms = 0, last_copy_ms = 0;
  std::vector<double> last_step_ms;  // per lowered step of the last timed run
  float* io_tmp = nullptr;
  size_t io_tmp_elems = 0;
  cudaStream_t stream = nullptr;
  // TPX_FLAG_GRAPH: the main program captured as one CUDA graph
  cudaGraphExec_t graph_exec = nullptr, graph_exec_b = nullptr;
  cudaStream_t graph_stream = nullptr;
  std::map<std::pair<int64_t, int64_t>, cudaGraphExec_t> range_graphs;  // run_steps ranges

  ~PlanRt();
  bool mine(int node) const { return dev_rank[size_t(plan.nodes[size_t(node)].device)] == ctx->rank; }
};

PlanRt* load_plan(Ctx* ctx, const std::string& json, int precision, int flags);
// Peer mode with several ranks: the CUDA IPC handle of this rank's arena, and the second half of
// the load once every rank's handle is known (maps the peers' arenas, lowers, prepares).
void arena_ipc_handle(PlanRt& p, void* out, size_t len);
void connect_peers(PlanRt& p, const void* handles, size_t len);
// Throws if a peer wait timed out (call after a stream synchronisation).
void check_peer_error(PlanRt& p);
void run_program(PlanRt& p, Program& prog, const std::string* only_op);
// One train step: main (or, in loop mode, main / main_b alternately), then the carry program
// when the plan has weights the swap cannot carry (loop mode only).
void run_step(PlanRt& p);
// Steps [begin, end) of the main program (CUDA graph per range with TPX_FLAG_GRAPH).
void run_steps(PlanRt& p, int64_t begin, int64_t end);
// Device-to-device copy between a node's holder block and contiguous device memory (n
// elements of the storage type), on the plan stream.
void copy_node_device(PlanRt& p, int node, void* dev, int64_t n, bool to_node);
void init_inputs(PlanRt& p, uint64_t seed);
void read_node(PlanRt& p, int node, double* dst, int64_t n);
void write_node(PlanRt& p, int node, const double* src, int64_t n);
void read_node_f32(PlanRt& p, int node, float* dst, int64_t n);
void write_node_f32(PlanRt& p, int node, const float* src, int64_t n);
std::string describe(const PlanRt& p);
// K7: NumericCheck of plan t's holders on this rank against the one-device plan s (same GPU).
void numeric_check(PlanRt& t, PlanRt& s, double* max_abs, double* max_rel, int64_t* values);

}  // namespace tpx
