// C ABI of the B200-native batched SQP solve (include/gato_b200.h).
// Host-side orchestration only: scratch allocation, model dispatch, CUDA-graph construction.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common_kernels.cuh"
#include "model_ops.cuh"

using namespace gato;

namespace {


#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t err__ = (call);                                                                \
    if (err__ != cudaSuccess) {                                                                \
      set_error(h, std::string(#call) + ": " + cudaGetErrorString(err__));                     \
      return GATO_E_CUDA;                                                                      \
    }                                                                                          \
  } while (0)

bool select_ops(int model_id, const double* params, ModelOps* ops) {
  switch (model_id) {
    case GATO_MODEL_DOUBLE_INTEGRATOR: {
      const int dims = params ? (int)params[0] : 0;
      if (dims < 1 || dims > 7) return false;
      *ops = gato_ops_double_integrator(dims);
      return true;
    }
    case GATO_MODEL_PENDULUM: *ops = gato_ops_pendulum(); return true;
    case GATO_MODEL_CARTPOLE: *ops = gato_ops_cartpole(); return true;
    case GATO_MODEL_TWO_LINK_ARM: *ops = gato_ops_two_link_arm(); return true;
    case GATO_MODEL_IIWA14: *ops = gato_ops_iiwa14(); return true;
    default: return false;
  }
}

// batch x (horizon + 1) from which the fused Schur + PCG path is used (measured crossover, see gato_create)
constexpr double kFusedMinBlockRows = 3000.0;

struct Scratch {
  const char* name;
  void* ptr;
  int64_t count;
};

}  // namespace

struct gato_handle {
  gato_config cfg;
  ModelOps ops;
  SolveParams P;
  bool bound = false;
  int loop_mode = 1;
  std::vector<void*> allocs;
  std::vector<Scratch> scratch;
  std::string error;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  bool graph_valid = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t side = nullptr;             // k_hessinv branch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t launches = 0;
  int device = 0;               // the device gato_create ran on: every entry point switches to it
  cudaGraphNode_t pro_node = nullptr;   // the k_prologue node of the instantiated graph (its arguments are patched per launch)
  PrologueArgs pro_in_graph = {};
  size_t pro_smem = 0;
  void* lin_scratch = nullptr;  // model-private linearisation scratch (iiwa14: per-stage link data)
  bool outmap_live = false;     // the last prologue told k_update to send results to a host buffer
  bool in_solve_host = false;
  bool timed_valid = false;     // ev0 / ev1 have been recorded at least once
  long long zero_copy_max = 1 << 20;   // bytes per direction up to which kernels move the data (GATO_ZERO_COPY_MAX)
};

namespace {

// A handle belongs to the device that was current in gato_create; its streams, events, graphs and
// scratch live there.  Every entry point makes that device current for the duration of the call, so a
// caller that drives several GPUs from one thread (batch_solve(devices=[...])) needs no device
// bookkeeping of its own.
struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  explicit DeviceGuard(const gato_handle* h) {
    if (!h) return;
    if (cudaGetDevice(&prev) == cudaSuccess && prev != h->device) switched = cudaSetDevice(h->device) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

void set_error(gato_handle* h, const std::string& msg) {
  if (h) h->error = msg;
}
void set_error(std::nullptr_t, const std::string&) {}

template <class T>
int dev_alloc(gato_handle* h, const char* name, T** out, int64_t count) {
  void* p = nullptr;
  const size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
  cudaError_t err = cudaMalloc(&p, bytes);
  if (err != cudaSuccess) {
    set_error(h, std::string("cudaMalloc(") + name + "): " + cudaGetErrorString(err));
    return GATO_E_NOMEM;
  }
  cudaMemset(p, 0, bytes);
  h->allocs.push_back(p);
  h->scratch.push_back({name, p, count});
  *out = static_cast<T*>(p);
  return GATO_OK;
}

// one SQP pass: six launches
// One SQP pass.  k_hessinv only depends on the previous pass, so it runs on the side stream
// concurrently with the linearisation (a parallel branch once captured into the graph).
// `marks`, when given, receives one event before each of the six launches and one after the last
// (everything serial on `s`, for per-kernel timing).
int enqueue_pass(gato_handle* h, cudaStream_t s, int use_cond, cudaEvent_t* marks = nullptr) {
  const SolveParams& P = h->P;
  RowView V{P.X, P.U, P.force, P.N, P.si};
  if (marks) {
    CK(cudaEventRecord(marks[0], s));
    CK(h->ops.hessinv(P, s));
    CK(cudaEventRecord(marks[1], s));
  } else {
    CK(cudaEventRecord(h->ev_fork, s));
    CK(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    CK(h->ops.hessinv(P, h->side));
    CK(cudaEventRecord(h->ev_join, h->side));
  }
  CK(h->ops.linearize(V, P.mp, P.h, (int64_t)P.M * P.N, P.A, P.B, P.e, h->lin_scratch, s));
  if (marks) CK(cudaEventRecord(marks[2], s));
  else CK(cudaStreamWaitEvent(s, h->ev_join, 0));
  CK(h->ops.schur(P, s));
  if (marks) CK(cudaEventRecord(marks[3], s));
  if (P.fused && !marks) {   // the two PCG builds take disjoint solves: side by side
    CK(cudaEventRecord(h->ev_fork, s));
    CK(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    CK(h->ops.pcg(P, s, h->side));
    CK(cudaEventRecord(h->ev_join, h->side));
    CK(cudaStreamWaitEvent(s, h->ev_join, 0));
  } else {
    CK(h->ops.pcg(P, s, nullptr));
  }
  if (marks) CK(cudaEventRecord(marks[4], s));
  CK(h->ops.linesearch(P, s));
  if (marks) CK(cudaEventRecord(marks[5], s));
  k_update<<<P.M, 128, 0, s>>>(P, h->ops.nx, h->ops.nu, h->cond, use_cond);
  CK(cudaGetLastError());
  if (marks) CK(cudaEventRecord(marks[6], s));
  return GATO_OK;
}

int enqueue_prologue(gato_handle* h, cudaStream_t s, const PrologueArgs& a = PrologueArgs{}) {
  const SolveParams& P = h->P;
  k_prologue<<<P.M, 128, h->pro_smem, s>>>(P, h->ops.nx, h->ops.nu, a);
  CK(cudaGetLastError());
  return GATO_OK;
}

// the k_prologue node of a freshly built graph (root level), so that its arguments can be patched per launch
int find_prologue_node(gato_handle* h) {
  h->pro_node = nullptr;
  size_t n = 0;
  CK(cudaGraphGetNodes(h->graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(h->graph, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp;
    if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) continue;
    if (kp.func == reinterpret_cast<void*>(k_prologue)) {
      h->pro_node = nd;
      break;
    }
  }
  cudaGetLastError();
  h->pro_in_graph = PrologueArgs{};
  return h->pro_node ? GATO_OK : GATO_E_CUDA;
}

bool same_args(const PrologueArgs& a, const PrologueArgs& b) {
  return a.mode == b.mode && a.path == b.path && a.path_len == b.path_len && a.path_stride == b.path_stride &&
         a.step == b.step && a.in_host == b.in_host && a.in_dev == b.in_dev && a.in_words == b.in_words &&
         a.out_host == b.out_host && a.out_dev == b.out_dev && a.out_bytes == b.out_bytes;
}

int patch_prologue(gato_handle* h, const PrologueArgs& a) {
  if (same_args(a, h->pro_in_graph)) return GATO_OK;
  SolveParams P = h->P;
  int nx = h->ops.nx, nu = h->ops.nu;
  PrologueArgs args = a;
  void* params[4] = {&P, &nx, &nu, &args};
  cudaKernelNodeParams kp = {};
  kp.func = reinterpret_cast<void*>(k_prologue);
  kp.gridDim = dim3((unsigned)P.M);
  kp.blockDim = dim3(128);
  kp.sharedMemBytes = (unsigned)h->pro_smem;
  kp.kernelParams = params;
  CK(cudaGraphExecKernelNodeSetParams(h->exec, h->pro_node, &kp));
  h->pro_in_graph = a;
  return GATO_OK;
}

void destroy_graph(gato_handle* h) {
  if (h->exec) cudaGraphExecDestroy(h->exec);
  if (h->graph) cudaGraphDestroy(h->graph);
  h->exec = nullptr;
  h->graph = nullptr;
  h->graph_valid = false;
}

// A failed call between cudaStreamBeginCapture and cudaStreamEndCapture must not leave the stream in
// capture mode: the fallback (unrolled graph, then plain launches) runs on the same stream.
void abort_capture(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(s, &junk);
    if (junk) cudaGraphDestroy(junk);
  }
  cudaGetLastError();
}

#define CKC(call)                                                                              \
  do {                                                                                         \
    cudaError_t err__ = (call);                                                                \
    if (err__ != cudaSuccess) {                                                                \
      set_error(h, std::string(#call) + ": " + cudaGetErrorString(err__));                     \
      abort_capture(s);                                                                        \
      destroy_graph(h);                                                                        \
      return GATO_E_CUDA;                                                                      \
    }                                                                                          \
  } while (0)

// prologue -> WHILE(any solve active) { pass }
int build_while_graph(gato_handle* h, cudaStream_t s) {
  destroy_graph(h);
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_prologue(h, s);
  if (rc != GATO_OK) {
    abort_capture(s);
    return rc;
  }
  cudaStreamCaptureStatus status;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CKC(cudaStreamGetCaptureInfo_v2(s, &status, nullptr, &g, &deps, &ndeps));
  CKC(cudaGraphConditionalHandleCreate(&h->cond, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h->cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CKC(cudaGraphAddNode(&node, g, deps, ndeps, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CKC(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  CKC(cudaStreamEndCapture(s, &h->graph));
  // body
  CKC(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  rc = enqueue_pass(h, s, 1);
  if (rc != GATO_OK) {
    abort_capture(s);
    destroy_graph(h);
    return rc;
  }
  cudaGraph_t body_out = nullptr;
  CKC(cudaStreamEndCapture(s, &body_out));
  CKC(cudaGraphInstantiate(&h->exec, h->graph, 0));
  if (find_prologue_node(h) != GATO_OK) {
    destroy_graph(h);
    return GATO_E_CUDA;
  }
  h->graph_valid = true;
  return GATO_OK;
}

int build_unrolled_graph(gato_handle* h, cudaStream_t s) {
  destroy_graph(h);
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_prologue(h, s);
  for (int it = 0; rc == GATO_OK && it < h->P.max_it; ++it) rc = enqueue_pass(h, s, 0);
  if (rc != GATO_OK) {
    abort_capture(s);
    return rc;
  }
  CKC(cudaStreamEndCapture(s, &h->graph));
  CKC(cudaGraphInstantiate(&h->exec, h->graph, 0));
  if (find_prologue_node(h) != GATO_OK) {
    destroy_graph(h);
    return GATO_E_CUDA;
  }
  h->graph_valid = true;
  return GATO_OK;
}

int solve_impl(gato_handle* h, void* stream, const PrologueArgs& pa, bool timed = true);

// The device-side alias of a pinned, device-mapped host buffer (torch's pin_memory, cudaHostAlloc,
// cudaHostRegister with the mapped flag), or null: pageable memory and anything else goes through cudaMemcpyAsync.
// Asked on every call (a fraction of a microsecond): a cached answer would outlive the buffer it was given for.
void* device_alias(const void* host) {
  void* dev = nullptr;
  cudaPointerAttributes at = {};
  if (cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
    dev = at.devicePointer;
  cudaGetLastError();
  return dev;
}

// does [p, p + bytes) overlap what k_prologue itself reads or writes besides its state words (the iterate it
// shifts, rho_init)?  Then the inputs cannot be copied by that same kernel.
bool prologue_touches(const gato_handle* h, const void* p, int64_t bytes) {
  const SolveParams& P = h->P;
  const char* lo = static_cast<const char*>(p);
  const char* hi = lo + bytes;
  auto hits = [&](const void* q, size_t n) {
    const char* a = static_cast<const char*>(q);
    return a < hi && lo < a + n;
  };
  const size_t nx = (size_t)h->ops.nx, nu = (size_t)h->ops.nu, M = (size_t)P.M, N = (size_t)P.N;
  return hits(P.X, M * (N + 1) * nx * 8) || hits(P.U, M * N * nu * 8) || hits(P.rho_init, M * 8);
}

// is [p, p + bytes) made of result arrays only (X, U, trace, info: each wholly inside or wholly outside), up to
// alignment padding between them?  Then k_update can send it row by row.
bool span_is_results(const gato_handle* h, const void* p, int64_t bytes) {
  const SolveParams& P = h->P;
  const char* lo = static_cast<const char*>(p);
  const char* hi = lo + bytes;
  const size_t nx = (size_t)h->ops.nx, nu = (size_t)h->ops.nu, M = (size_t)P.M, N = (size_t)P.N;
  const struct {
    const void* ptr;
    size_t bytes;
  } arrays[4] = {{P.X, M * (N + 1) * nx * 8},
                 {P.U, M * N * nu * 8},
                 {P.trace, M * (size_t)P.max_it * GATO_TRACE_WORDS * 8},
                 {P.info, M * GATO_INFO_WORDS * 4}};
  int64_t covered = 0;
  for (const auto& a : arrays) {
    const char* q = static_cast<const char*>(a.ptr);
    const bool inside = q >= lo && q + a.bytes <= hi, outside = q + a.bytes <= lo || q >= hi;
    if (!inside && !outside) return false;
    if (inside) covered += (int64_t)a.bytes;
  }
  const int64_t nf = h->ops.nf;
  const struct {
    const void* ptr;
    size_t bytes;
  } inputs[7] = {{P.x_start, M * nx * 8},    {P.goal, M * (N + 1) * nx * 8}, {P.Q, M * nx * nx * 8},
                 {P.R, M * nu * nu * 8},     {P.QN, M * nx * nx * 8},        {P.force, M * N * (size_t)nf * 8},
                 {P.rho_init, M * 8}};
  for (const auto& a : inputs) {   // an input array in the span: the caller wants it copied back too
    const char* q = static_cast<const char*>(a.ptr);
    if (a.ptr && a.bytes && q < hi && lo < q + a.bytes) return false;
  }
  return covered + 4 * 16 >= bytes;   // the rest may only be alignment padding between the arrays
}

}  // namespace

extern "C" {

const char* gato_version(void) { return "gato_b200 0.1 (sm_100a, fp64)"; }

int gato_create(const gato_config* cfg, gato_handle** out) {
  if (!cfg || !out) return GATO_E_INVALID;
  *out = nullptr;
  if (cfg->abi_version != GATO_ABI_VERSION) return GATO_E_INVALID;
  gato_handle* h = new gato_handle();
  h->cfg = *cfg;
  if (cudaGetDevice(&h->device) != cudaSuccess) h->device = 0;
  h->zero_copy_max = env_int("GATO_ZERO_COPY_MAX", 1 << 20);
  *out = h;  // returned even on failure so that gato_last_error is readable; caller destroys
  if (!select_ops(cfg->model_id, cfg->model_params, &h->ops)) {
    set_error(h, "unknown model id or unsupported model dimension");
    return GATO_E_INVALID;
  }
  const int nx = h->ops.nx, nu = h->ops.nu, nf = h->ops.nf;
  if (cfg->state_dim != nx || cfg->control_dim != nu || cfg->force_dim != nf) {
    set_error(h, "state/control/force dimensions do not match the model");
    return GATO_E_INVALID;
  }
  if (cfg->batch < 1 || cfg->horizon < 1 || cfg->max_sqp_iterations < 1 || cfg->num_shrinks < 0 ||
      !(cfg->timestep > 0.0)) {
    set_error(h, "batch, horizon, max_sqp_iterations must be >= 1 and timestep > 0");
    return GATO_E_INVALID;
  }
  if (cfg->horizon + 1 > 1024) {
    set_error(h, "horizon too long: the PCG kernels run one thread per block row, N + 1 <= 1024");
    return GATO_E_INVALID;
  }
  SolveParams& P = h->P;
  memset(&P, 0, sizeof(P));
  const int64_t M = cfg->batch, N = cfg->horizon, nb = N + 1;
  P.M = (int)M;
  P.N = (int)N;
  P.max_it = cfg->max_sqp_iterations;
  P.pcg_cap = cfg->pcg_max_iterations > 0 ? cfg->pcg_max_iterations : (int)(10 * nb * nx);
  P.C = cfg->num_shrinks + 1;
  P.regularize_r = cfg->regularize_r;
  P.retry_limit = cfg->pcg_retry_limit;
  P.dense_schur = env_int("GATO_SCHUR_DENSE", 0);
  // Schur formation fused into the PCG kernel (schur_quad.cuh) wherever k_pcg_q runs and it pays; GATO_FUSED=0,
  // the config flag GATO_FLAG_UNFUSED or GATO_SCHUR_DENSE=1 keep k_schur + the matrix record (stage arrays for
  // tests), GATO_FUSED=2 forces the fused path.  The rule (scripts/fused_crossover.py, profiles/r02_fused_crossover.csv):
  // k_schur spreads M (N + 1) block rows over the whole GPU (one warp each), the fused phase handles a solve's
  // block rows on the one SM that then runs its PCG -- so the fused path wins once the batch is large enough to
  // keep the whole GPU busy with k_schur anyway, and loses in the latency regime (few solves).
  {
    const int mode = (cfg->flags & GATO_FLAG_FUSED) ? 2 : env_int("GATO_FUSED", 1);
    const bool can = !(cfg->flags & GATO_FLAG_UNFUSED) && !P.dense_schur && h->ops.pcg_fused_ok((int)N);
    const bool pays = (double)M * (double)(N + 1) >= kFusedMinBlockRows;
    P.fused = (can && (mode == 2 || (mode == 1 && pays))) ? 1 : 0;
  }
  P.h = cfg->timestep;
  P.pcg_tol = cfg->pcg_tolerance;
  P.mu = cfg->mu;
  P.rho_min = cfg->rho_min;
  P.rho_max = cfg->rho_max;
  P.rho_factor = cfg->rho_factor;
  P.step_tol = cfg->step_tolerance;
  P.feas_tol = cfg->feasibility_tolerance;
  for (int i = 0; i < 8; ++i) P.mp.v[i] = cfg->model_params[i];

  int rc = GATO_OK;
#define ALLOC(field, count)                                                   \
  if (rc == GATO_OK) rc = dev_alloc(h, #field, &P.field, (int64_t)(count));
  ALLOC(A, M * N * nx * nx);
  ALLOC(B, M * N * nx * nu);
  ALLOC(e, M * N * nx);
  ALLOC(grad, M * nb * (nx + nu));
  ALLOC(hinv, M * hinv_stride(nx, nu));
  ALLOC(Sdiag, M * nb * nx * nx);
  ALLOC(Soff, M * N * nx * nx);
  ALLOC(Linv, M * nb * (nx * (nx + 1) / 2));
  ALLOC(Lfac, M * nb * (nx * (nx + 1) / 2));
  ALLOC(pmats, M * (int64_t)h->ops.pcg_mat_doubles((int)N));
  ALLOC(gamma, M * nb * nx);
  ALLOC(gammaw, M * nb * nx);
  ALLOC(lbw, M * nb);
  ALLOC(lam, M * nb * nx);
  ALLOC(dX, M * nb * nx);
  ALLOC(dU, M * N * nu);
  ALLOC(merits, M * (P.C + 1));
  ALLOC(viols, M * (P.C + 1));
  ALLOC(alphas, P.C);
  ALLOC(sd, M * SD_WORDS);
  ALLOC(si, M * SI_WORDS);
  ALLOC(pcg_iters, M * P.max_it);
  ALLOC(schur_list, M);
  ALLOC(counters, 8);
  ALLOC(outmap, 4);
#undef ALLOC
  if (rc != GATO_OK) return rc;
  {
    const size_t bytes = h->ops.lin_scratch_bytes(M * N);
    if (bytes) {
      unsigned char* p = nullptr;
      rc = dev_alloc(h, "lin_scratch", &p, (int64_t)bytes);
      if (rc != GATO_OK) return rc;
      h->lin_scratch = p;
    }
  }
  // step lengths beta^-c, computed on the host exactly as sqp.py:51-52 (libm pow)
  std::vector<double> alphas(P.C);
  for (int c = 0; c < P.C; ++c) alphas[c] = pow(cfg->beta, -(double)c);
  CK(cudaMemcpy(P.alphas, alphas.data(), P.C * sizeof(double), cudaMemcpyHostToDevice));
  h->pro_smem = ((size_t)(N + 1) * nx + (size_t)N * nu) * sizeof(double);
  if (h->pro_smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_prologue, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->pro_smem));
  CK(cudaEventCreate(&h->ev0));
  CK(cudaEventCreate(&h->ev1));
  CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  {
    cudaError_t perr = h->ops.prepare(P);
    if (perr != cudaSuccess) {   // e.g. N + 1 > 256 with a state dimension whose exchange vectors exceed shared memory
      set_error(h, std::string("kernel set-up failed (horizon too long for this model's shared-memory footprint?): ") +
                       cudaGetErrorString(perr));
      cudaGetLastError();
      return GATO_E_INVALID;
    }
  }
  h->loop_mode = cfg->loop_mode ? cfg->loop_mode : env_int("GATO_LOOP_MODE", 1);
  return GATO_OK;
}

int gato_bind(gato_handle* h, const gato_buffers* b) {
  if (!h || !b) return GATO_E_INVALID;
  if (!b->x_start || !b->goal || !b->Q || !b->R || !b->QN || !b->force || !b->rho_init || !b->X || !b->U ||
      !b->trace || !b->info) {
    set_error(h, "gato_bind: null buffer");
    return GATO_E_INVALID;
  }
  SolveParams& P = h->P;
  const bool same = h->bound && P.x_start == b->x_start && P.goal == b->goal && P.Q == b->Q && P.R == b->R &&
                    P.QN == b->QN && P.force == b->force && P.rho_init == b->rho_init && P.X == b->X &&
                    P.U == b->U && P.trace == b->trace && P.info == b->info;
  P.x_start = b->x_start;
  P.goal = b->goal;
  P.Q = b->Q;
  P.R = b->R;
  P.QN = b->QN;
  P.force = b->force;
  P.rho_init = b->rho_init;
  P.X = b->X;
  P.U = b->U;
  P.trace = b->trace;
  P.info = b->info;
  h->bound = true;
  if (!same) h->graph_valid = false;
  return GATO_OK;
}

int gato_solve(gato_handle* h, void* stream) {
  DeviceGuard guard__(h);
  if (!h) return GATO_E_INVALID;
  return solve_impl(h, stream, PrologueArgs{});
}

int gato_solve_mpc(gato_handle* h, void* stream, int32_t shift_mode, const double* goal_path, int64_t path_len,
                   int64_t path_stride, int64_t step) {
  DeviceGuard guard__(h);
  if (!h) return GATO_E_INVALID;
  if (shift_mode < 0 || shift_mode > 2 || (shift_mode == 2 && goal_path && (path_len < 1 || step < 0 || path_stride < 0))) {
    set_error(h, "gato_solve_mpc: shift_mode in {0, 1, 2}; with a goal path: path_len >= 1, step >= 0, path_stride >= 0");
    return GATO_E_INVALID;
  }
  return solve_impl(h, stream, PrologueArgs{shift_mode, shift_mode == 2 ? goal_path : nullptr, path_len, path_stride, step, nullptr, nullptr, 0, 0, 0, 0});
}

}  // extern "C"

namespace {
int solve_impl(gato_handle* h, void* stream, const PrologueArgs& pa, bool timed) {
  if (h->cfg.flags & GATO_FLAG_UNTIMED) timed = false;
  if (!h->bound) {
    set_error(h, "gato_solve before gato_bind");
    return GATO_E_UNBOUND;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int mode = h->loop_mode;
  h->outmap_live = pa.out_host != 0;
  if ((mode == 1 || mode == 2) && !h->graph_valid) {
    // graph capture needs a capturable stream; the legacy default stream is not
    cudaStream_t cs = s;
    bool own = false;
    if (cs == nullptr || cs == cudaStreamLegacy) {
      CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      own = true;
    }
    int rc = (mode == 1) ? build_while_graph(h, cs) : build_unrolled_graph(h, cs);
    if (rc != GATO_OK && mode == 1) {
      // WHILE nodes unavailable: fall back to the unrolled graph
      cudaGetLastError();
      h->loop_mode = mode = 2;
      rc = build_unrolled_graph(h, cs);
    }
    if (own) cudaStreamDestroy(cs);
    if (rc != GATO_OK) {
      cudaGetLastError();
      h->loop_mode = mode = 3;
    }
  }
  if (timed) CK(cudaEventRecord(h->ev0, s));   // gato_last_solve_ms; the host-buffer call is timed by its caller
  if (mode == 1 || mode == 2) {
    int rc = patch_prologue(h, pa);   // this launch's warm-start preparation (no-op if unchanged)
    if (rc != GATO_OK) return rc;
    CK(cudaGraphLaunch(h->exec, s));
  } else {
    int rc = enqueue_prologue(h, s, pa);
    for (int it = 0; rc == GATO_OK && it < h->P.max_it; ++it) rc = enqueue_pass(h, s, 0);
    if (rc != GATO_OK) return rc;
  }
  if (timed) CK(cudaEventRecord(h->ev1, s));
  h->timed_valid = h->timed_valid || timed;
  return GATO_OK;
}
}  // namespace

extern "C" {

/* number of solves still active after the last enqueued pass (synchronises the stream).
 * Non-zero only in loop modes 2/3 when a PCG-breakdown retry consumed a pass. */
int gato_pending(gato_handle* h, void* stream, int32_t* pending) {
  DeviceGuard guard__(h);
  if (!h || !pending) return GATO_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaStreamSynchronize(s));
  unsigned int c[4];
  CK(cudaMemcpy(c, h->P.counters, sizeof(c), cudaMemcpyDeviceToHost));
  *pending = (int32_t)c[2];
  return GATO_OK;
}

/* enqueue `passes` further SQP passes without re-initialising (loop modes 2/3 after retries) */
int gato_resume(gato_handle* h, void* stream, int32_t passes) {
  DeviceGuard guard__(h);
  if (!h || !h->bound) return GATO_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (h->outmap_live && !h->in_solve_host) {
    // passes enqueued by the caller after a gato_solve_host: its host buffer is no longer ours to write
    CK(cudaMemsetAsync(h->P.outmap, 0, 3 * sizeof(long long), s));
    h->outmap_live = false;
  }
  for (int it = 0; it < passes; ++it) {
    int rc = enqueue_pass(h, s, 0);
    if (rc != GATO_OK) return rc;
  }
  return GATO_OK;
}

int gato_shift_warm_start(gato_handle* h, void* stream) {
  DeviceGuard guard__(h);
  if (!h || !h->bound) return GATO_E_INVALID;
  const SolveParams& P = h->P;
  const size_t bytes = ((size_t)(P.N + 1) * h->ops.nx + (size_t)P.N * h->ops.nu) * sizeof(double);
  if (bytes > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  k_shift<<<P.M, 128, bytes, static_cast<cudaStream_t>(stream)>>>(P.X, P.U, P.N, h->ops.nx, h->ops.nu);
  CK(cudaGetLastError());
  return GATO_OK;
}

int gato_mpc_advance(gato_handle* h, void* stream, const double* goal_path, int64_t path_len, int64_t path_stride,
                     int64_t step) {
  DeviceGuard guard__(h);
  if (!h || !h->bound) return GATO_E_INVALID;
  if (goal_path && (path_len < 1 || step < 0 || path_stride < 0)) {
    set_error(h, "gato_mpc_advance: path_len >= 1, step >= 0, path_stride >= 0");
    return GATO_E_INVALID;
  }
  const SolveParams& P = h->P;
  const size_t bytes = ((size_t)(P.N + 1) * h->ops.nx + (size_t)P.N * h->ops.nu) * sizeof(double);
  if (bytes > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_mpc_advance, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  // the caller's buffers are written here: x_start and goal are inputs of the solve, not of this call
  k_mpc_advance<<<P.M, 128, bytes, static_cast<cudaStream_t>(stream)>>>(
      P.X, P.U, const_cast<double*>(P.x_start), const_cast<double*>(P.goal), goal_path, path_len, path_stride, step,
      P.N, h->ops.nx, h->ops.nu);
  CK(cudaGetLastError());
  return GATO_OK;
}

int gato_merit_candidates(gato_handle* h, void* stream, const double* dX, const double* dU) {
  DeviceGuard guard__(h);
  if (!h || !h->bound) return GATO_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const SolveParams& P = h->P;
  const size_t nX = (size_t)P.M * (P.N + 1) * h->ops.nx * sizeof(double), nU = (size_t)P.M * P.N * h->ops.nu * sizeof(double);
  if (dX) CK(cudaMemcpyAsync(P.dX, dX, nX, cudaMemcpyDeviceToDevice, s));
  else CK(cudaMemsetAsync(P.dX, 0, nX, s));
  if (dU) CK(cudaMemcpyAsync(P.dU, dU, nU, cudaMemcpyDeviceToDevice, s));
  else CK(cudaMemsetAsync(P.dU, 0, nU, s));
  int rc = enqueue_prologue(h, s);   // every solve active, merit of the current iterate not yet known
  if (rc != GATO_OK) return rc;
  CK(h->ops.linesearch(P, s));
  return GATO_OK;
}

int gato_best_of_batch(gato_handle* h, void* stream, int32_t* best_index, double* best_merit) {
  DeviceGuard guard__(h);
  if (!h || !h->bound) return GATO_E_INVALID;
  k_best_of_batch<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(h->P, best_index, best_merit);
  CK(cudaGetLastError());
  return GATO_OK;
}

int gato_solve_host(gato_handle* h, void* stream, void* dev_in, const void* host_in, int64_t in_bytes,
                    int32_t shift_first, const void* dev_out, void* host_out, int64_t out_bytes) {
  DeviceGuard guard__(h);
  if (!h) return GATO_E_INVALID;
  if (!h->bound) {
    set_error(h, "gato_solve_host before gato_bind");
    return GATO_E_UNBOUND;
  }
  if (in_bytes < 0 || out_bytes < 0 || (in_bytes > 0 && (!dev_in || !host_in)) ||
      (out_bytes > 0 && (!dev_out || !host_out))) {
    set_error(h, "gato_solve_host: null buffer with a non-zero size");
    return GATO_E_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Latency regime (a few hundred KB per direction): a copy-engine transfer costs ~11 us each way, most of it
  // scheduling; when the host buffers are pinned and device-mapped the kernels move the data themselves -- the
  // solve's first kernel reads the inputs across PCIe, k_update writes the rows of every finished solve back
  // (or, for a span that is not made of result arrays only, a small copy kernel behind the solve).
  PrologueArgs pa{};
  pa.mode = shift_first ? 1 : 0;
  const void* in_alias = (in_bytes > 0 && in_bytes % 8 == 0 && in_bytes <= h->zero_copy_max &&
                          ((uintptr_t)dev_in | (uintptr_t)host_in) % 16 == 0 && !prologue_touches(h, dev_in, in_bytes))
                             ? device_alias(host_in)
                             : nullptr;
  if (in_alias) {
    pa.in_host = static_cast<const double*>(in_alias);
    pa.in_dev = static_cast<double*>(dev_in);
    pa.in_words = in_bytes / 8;
  } else if (in_bytes > 0) {
    CK(cudaMemcpyAsync(dev_in, host_in, (size_t)in_bytes, cudaMemcpyHostToDevice, s));
  }
  void* out_alias = (out_bytes > 0 && out_bytes % 8 == 0 && out_bytes <= h->zero_copy_max &&
                     ((uintptr_t)dev_out | (uintptr_t)host_out) % 16 == 0)
                        ? device_alias(host_out)
                        : nullptr;
  // results: sent by k_update itself when the span is made of result arrays (plus alignment padding) only
  const bool out_by_update = out_alias && h->P.max_it >= 1 && span_is_results(h, dev_out, out_bytes);
  if (out_by_update) {
    pa.out_host = (long long)(uintptr_t)out_alias;
    pa.out_dev = (long long)(uintptr_t)dev_out;
    pa.out_bytes = out_bytes;
  }
  // the shift of the warm start rides in the solve's first kernel (k_prologue mode 1): no launch of its own
  int rc = solve_impl(h, stream, pa, false);
  if (rc != GATO_OK) return rc;
  if (h->loop_mode != 1) {   // no device-side WHILE: a PCG retry may have used up a pass
    int guard = h->cfg.max_sqp_iterations * (h->cfg.pcg_retry_limit + 1) + 1;
    int32_t pending = 0;
    while (guard-- > 0) {
      rc = gato_pending(h, stream, &pending);
      if (rc != GATO_OK) return rc;
      if (pending == 0) break;
      h->in_solve_host = true;
      rc = gato_resume(h, stream, 1);
      h->in_solve_host = false;
      if (rc != GATO_OK) return rc;
    }
  }
  if (out_by_update) {
    // already on its way
  } else if (out_alias) {
    const long long words = out_bytes / 8;
    const unsigned blocks = (unsigned)((words / 2 + 1023) / 1024);   // 256 threads x four 16-byte accesses
    k_copy_words<<<blocks ? blocks : 1, 256, 0, s>>>(static_cast<double*>(out_alias), static_cast<const double*>(dev_out),
                                                     words);
    CK(cudaGetLastError());
  } else if (out_bytes > 0) {
    CK(cudaMemcpyAsync(host_out, dev_out, (size_t)out_bytes, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return GATO_OK;
}

int gato_scratch(gato_handle* h, const char* name, void** dev_ptr, int64_t* count) {
  if (!h || !name || !dev_ptr) return GATO_E_INVALID;
  for (const Scratch& s : h->scratch) {
    if (strcmp(s.name, name) == 0) {
      *dev_ptr = s.ptr;
      if (count) *count = s.count;
      return GATO_OK;
    }
  }
  set_error(h, std::string("unknown scratch array ") + name);
  return GATO_E_INVALID;
}

int gato_read_scratch(gato_handle* h, const char* name, void* host_dst, int64_t bytes) {
  DeviceGuard guard__(h);
  void* src = nullptr;
  int64_t count = 0;
  int rc = gato_scratch(h, name, &src, &count);
  if (rc != GATO_OK) return rc;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(host_dst, src, (size_t)bytes, cudaMemcpyDeviceToHost));
  return GATO_OK;
}

int64_t gato_launch_count(const gato_handle* h) {
  DeviceGuard guard__(h);
  if (!h) return 0;
  unsigned int c[4] = {0, 0, 0, 0};
  if (cudaMemcpy(c, h->P.counters, sizeof(c), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  // k_prologue + per pass: k_hessinv, linearisation (two kernels for iiwa14), k_schur, PCG, k_linesearch, k_update
  // (with the fused Schur + PCG path the PCG step is two launches: the fused and the record-reading build)
  const int per_pass = 5 + (h->ops.lin_scratch_bytes(1) > 0 ? 2 : 1) + (h->P.fused ? 1 : 0);
  return 1 + per_pass * (int64_t)c[3];
}

int gato_loop_mode(const gato_handle* h) { return h ? h->loop_mode : 0; }

int gato_fused(const gato_handle* h) { return h ? h->P.fused : 0; }

/* Same work as gato_solve in plain stream-launch mode, with CUDA events between the six kernels of
 * every pass: ms[0..5] = total device time of hessinv, linearize, schur, pcg, linesearch, update
 * over the max_sqp_iterations passes, ms[6] = prologue, ms[7] = whole call. Synchronous. */
int gato_solve_profiled(gato_handle* h, void* stream, float* ms) {
  DeviceGuard guard__(h);
  if (!h || !ms) return GATO_E_INVALID;
  if (!h->bound) return GATO_E_UNBOUND;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int passes = h->P.max_it;
  std::vector<cudaEvent_t> ev((size_t)passes * 7 + 2);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaEventRecord(ev[passes * 7], s));
  int rc = enqueue_prologue(h, s);
  for (int it = 0; rc == GATO_OK && it < passes; ++it) rc = enqueue_pass(h, s, 0, &ev[(size_t)it * 7]);
  if (rc == GATO_OK) {
    CK(cudaEventRecord(ev[passes * 7 + 1], s));
    CK(cudaStreamSynchronize(s));
    for (int k = 0; k < 8; ++k) ms[k] = 0.f;
    for (int it = 0; it < passes; ++it)
      for (int k = 0; k < 6; ++k) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ev[it * 7 + k], ev[it * 7 + k + 1]));
        ms[k] += t;
      }
    CK(cudaEventElapsedTime(&ms[6], ev[passes * 7], ev[0]));
    CK(cudaEventElapsedTime(&ms[7], ev[passes * 7], ev[passes * 7 + 1]));
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

/* Sustained fp64 FMA throughput of this GPU (TFLOP/s, FMA = 2 flops), measured with a
 * register-resident DFMA kernel: the R1 roofline denominator of SURVEY.md section 8d, which
 * MEASURED_PEAKS.json does not carry. Synchronous; ~50 ms. */
int gato_measure_fp64_peak(double* tflops) {
  if (!tflops) return GATO_E_INVALID;
  gato_handle* h = nullptr;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GATO_E_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double) * 1024) != cudaSuccess) return GATO_E_NOMEM;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k_fp64_peak<<<blocks, threads>>>(sink, iters, 1.0000001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    const double flops = 2.0 * 16.0 * (double)iters * (double)blocks * threads;
    if (rep > 0 && t > 0.f) best = fmax(best, flops / (t * 1e-3) / 1e12);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  (void)h;
  if (cudaGetLastError() != cudaSuccess) return GATO_E_CUDA;
  *tflops = best;
  return GATO_OK;
}

int gato_last_solve_ms(gato_handle* h, float* ms) {
  DeviceGuard guard__(h);
  if (!h || !ms) return GATO_E_INVALID;
  if (!h->timed_valid) {
    set_error(h, "gato_last_solve_ms: no gato_solve / gato_solve_mpc on this handle yet (gato_solve_host is not timed)");
    return GATO_E_INVALID;
  }
  CK(cudaEventSynchronize(h->ev1));
  CK(cudaEventElapsedTime(ms, h->ev0, h->ev1));
  return GATO_OK;
}

const char* gato_last_error(const gato_handle* h) { return h ? h->error.c_str() : "null handle"; }

void gato_destroy(gato_handle* h) {
  DeviceGuard guard__(h);
  if (!h) return;
  destroy_graph(h);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->side) cudaStreamDestroy(h->side);
  for (void* p : h->allocs) cudaFree(p);
  delete h;
}

// ---- stateless operator entry points ----

int gato_step_many(int32_t model_id, const double* model_params, int64_t rows, const double* X, const double* U,
                   const double* F, double timestep, double* out, void* stream) {
  ModelOps ops;
  if (!select_ops(model_id, model_params, &ops) || rows < 0) return GATO_E_INVALID;
  if (rows == 0) return GATO_OK;
  ModelParams mp;
  for (int i = 0; i < 8; ++i) mp.v[i] = model_params ? model_params[i] : 0.0;
  cudaError_t err = ops.step_rows(mp, timestep, rows, X, U, F, out, static_cast<cudaStream_t>(stream));
  return err == cudaSuccess ? GATO_OK : GATO_E_CUDA;
}

int gato_select_hypothesis(int32_t model_id, const double* model_params, int32_t candidates, const double* x_prev,
                           const double* u_applied, const double* x_meas, const double* forces, double h_plant,
                           int32_t substeps, int32_t position_only, double* errors, int32_t* best, void* stream) {
  ModelOps ops;
  if (!select_ops(model_id, model_params, &ops) || candidates < 1 || substeps < 1 || !(h_plant > 0.0) || !x_prev ||
      !u_applied || !x_meas || !forces || !best)
    return GATO_E_INVALID;
  ModelParams mp;
  for (int i = 0; i < 8; ++i) mp.v[i] = model_params ? model_params[i] : 0.0;
  const int ncmp = position_only ? ops.nx / 2 : ops.nx;   // state layout [positions, velocities] (dynamics.py:9)
  cudaError_t err = ops.select_hypothesis(mp, candidates, x_prev, u_applied, x_meas, forces, h_plant, substeps, ncmp,
                                          errors, best, static_cast<cudaStream_t>(stream));
  return err == cudaSuccess ? GATO_OK : GATO_E_CUDA;
}

int gato_step_jacobians_many(int32_t model_id, const double* model_params, int64_t rows, const double* X,
                             const double* U, const double* F, double timestep, double* A, double* B,
                             void* stream) {
  ModelOps ops;
  if (!select_ops(model_id, model_params, &ops) || rows < 0) return GATO_E_INVALID;
  if (rows == 0) return GATO_OK;
  {
    SolveParams tmp;
    memset(&tmp, 0, sizeof(tmp));
    tmp.N = 1;
    if (ops.prepare(tmp) != cudaSuccess) return GATO_E_CUDA;
  }
  ModelParams mp;
  for (int i = 0; i < 8; ++i) mp.v[i] = model_params ? model_params[i] : 0.0;
  // operator mode: one "solve" whose N = rows, so row r is addressed as (b = 0, k = r); the
  // defect output is off, so the (N+1)-th state row of the solve layout is never read.
  RowView V{X, U, F, (int)rows, nullptr};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  void* scratch = nullptr;
  const size_t bytes = ops.lin_scratch_bytes(rows);
  if (bytes && cudaMalloc(&scratch, bytes) != cudaSuccess) return GATO_E_NOMEM;
  cudaError_t err = ops.linearize(V, mp, timestep, rows, A, B, nullptr, scratch, s);
  if (scratch) {
    cudaStreamSynchronize(s);   // operator entry point: scratch lives for this call only
    cudaFree(scratch);
  }
  return err == cudaSuccess ? GATO_OK : GATO_E_CUDA;
}

int gato_btmv_batched(int32_t systems, int32_t nb, int32_t bd, const double* diag, const double* off, const double* v,
                      double* y, void* stream) {
  if (systems < 1 || nb < 1 || bd < 1 || !diag || !v || !y || (nb > 1 && !off)) return GATO_E_INVALID;
  const int size = nb * bd;
  dim3 grid((size + 127) / 128, systems);
  k_btmv<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(nb, bd, diag, off, v, y);
  return cudaGetLastError() == cudaSuccess ? GATO_OK : GATO_E_CUDA;
}

int gato_pcg_batched(int32_t systems, int32_t nb, int32_t bd, const double* S_diag, const double* S_off,
                     const double* gamma, const double* P_diag, const double* P_off, double tolerance,
                     int32_t max_iterations, double* lam, int32_t* iterations, int32_t* converged, int32_t* status,
                     double* residual, void* stream) {
  if (systems < 1 || nb < 1 || bd < 1) return GATO_E_INVALID;
  const int size = nb * bd;
  const size_t bytes = (size_t)6 * size * 8 + 64 * 16;
  if (bytes > kMaxSmem) return GATO_E_INVALID;
  const int cap = max_iterations > 0 ? max_iterations : 10 * size;
  if (cudaFuncSetAttribute(k_pcg_explicit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return GATO_E_CUDA;
  k_pcg_explicit<<<systems, 256, bytes, static_cast<cudaStream_t>(stream)>>>(
      nb, bd, S_diag, S_off, gamma, P_diag, P_off, tolerance, cap, lam, iterations, converged, status, residual);
  return cudaGetLastError() == cudaSuccess ? GATO_OK : GATO_E_CUDA;
}

}  // extern "C"
