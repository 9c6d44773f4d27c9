// psi_api.cu -- the C-ABI of libpsi (include/psi.h): context, CUDA-graph loop, errors.
//
// psi_iterate launches ONE instantiated CUDA graph per call:
//
//    k_init  ->  WHILE(cond) { k_tiles<sweep> -> k_fix<sweep> }  ->  k_tiles<readout> -> k_fix<readout>
//
// k_init sets cond = (gap_0 = 1 > eps && max_iters > 0) (Alg. 2 lines 1-5); the last CTA of
// every k_fix<sweep> sets cond = (gap_t > eps && t < max_iters) (lines 5, 8), so the whole
// Alg. 2 loop runs on the device; the host reads back (T, gap_T, status) once.
// Kernel arguments are frozen in the graph, so per-call values (eps, max_iters, ||B||,
// history buffer) live in a device LoopParams block written before each launch, and the
// ping-pong buffer of sweep t is selected on the device from the loop counter.
#include "psi_internal.cuh"
#include "../../include/psi.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

using namespace psi;

namespace {

thread_local std::string g_err;

// NVTX range around every public call (ingest / iterate / readout phases in a profiler
// timeline; free when no tool is attached -- NVTX v3 is header-only)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

psi_status fail(psi_status code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
psi_status fail(psi_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define API_CK(call)                                                                     \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? PSI_E_OOM : PSI_E_CUDA,              \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);  \
  } while (0)

}  // namespace

struct psi_ctx {
  long long n = 0, m = 0;
  int dev = -1;                  // device of the context (its memory pool)
  cudaStream_t stream = nullptr;
  IngestOut g;
  double* x[2] = {nullptr, nullptr};
  double* p_in = nullptr;        // per tile: partial of the row open at the tile start
  double* p_out = nullptr;       // per tile: partial of its last row if that row continues
  int last_solver = 0;           // psi_info.last_solver
  double* eps_part1 = nullptr;
  double* eps_part2 = nullptr;
  double* history = nullptr;
  long long hist_cap = 0;
  LoopState* st = nullptr;
  LoopParams* prm = nullptr;
  LoopState* h_st = nullptr;     // pinned
  LoopParams* h_prm = nullptr;   // pinned
  int grid1 = 0, grid2 = 0;
  TilesCfg tc{};                 // launch shape of k_tiles (sweep + readout)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool have_psi = false;
  long long last_T = 0;
  double last_gap = 1.0;
  double ingest_ms = 0, iterate_ms = 0;
  size_t device_bytes = 0;
  long long hot_lim = 0;         // x labels kept in L2 with evict_last (both buffers)
  PrBuffers pr;                  // PageRank constants and result (allocated on first use)
  cudaGraph_t pr_graph = nullptr;
  cudaGraphExec_t pr_exec = nullptr;
  bool have_pr = false;          // psi_get_pagerank valid
  bool series_ok = false;        // x holds the psi iterate s_T / Wt (no PageRank run since)
  long long pr_T = 0;
  double pr_alpha = 0.0;
  double* hhot = nullptr;        // [n_heavy] heavy rows' sums over followers < H (k_heavy)
  double* scold = nullptr;       // [n_heavy] their edge-stream sums (overlapped sweep only)
  double* ppart = nullptr;       // k_sell: long-row piece sums, their epochs, window eps_t
  double* epsw = nullptr;
  int heavy_grid = 0;
  int heavy_block = 0;
  size_t heavy_smem = 0;
  // multi-profile batch (psi_build_graph_batch, psi_batch.cu); sweep state of one group
  struct Batch {
    BatchCfg cfg{};
    d4* x[2] = {nullptr, nullptr};
    d4* p_in = nullptr;
    d4* p_out = nullptr;
    d4* part1 = nullptr;
    d4* part2 = nullptr;
    LoopStateB* st = nullptr;
    LoopStateB* h_st = nullptr;    // pinned
    BatchParams* prm = nullptr;
    BatchParams* h_prm = nullptr;  // pinned
    double* history = nullptr;     // [hist_cap][kBP]
    long long hist_cap = 0;
    long long hot_lim = 0;
    std::vector<cudaGraph_t> graph;
    std::vector<cudaGraphExec_t> exec;
    std::vector<long long> T;
    std::vector<double> gap;
    std::vector<int> bad;
    std::vector<std::vector<double>> hist;
    bool have = false;
  } b;
};

namespace {

// Small pinned host blocks (loop state read-backs, per-call parameters) come from one
// process-wide pinned slab, never returned to the OS: cudaHostAlloc / cudaFreeHost per context
// are system calls with a device synchronisation, and they stalled builds and destroys by
// 0.1-1 s at random on the GPU box (tools/e2e_pool_diag.py).
constexpr size_t kPinSlot = 256;
constexpr int kPinSlots = 4096;
std::mutex g_pin_mu;
unsigned char* g_pin_base = nullptr;
std::vector<int> g_pin_free;

cudaError_t pin_alloc(void** p, size_t bytes) {
  if (bytes > kPinSlot) return cudaHostAlloc(p, bytes, cudaHostAllocDefault);
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (!g_pin_base) {
    cudaError_t e = cudaHostAlloc((void**)&g_pin_base, kPinSlot * kPinSlots, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    for (int i = kPinSlots - 1; i >= 0; --i) g_pin_free.push_back(i);
  }
  if (g_pin_free.empty()) return cudaHostAlloc(p, bytes, cudaHostAllocDefault);
  const int i = g_pin_free.back();
  g_pin_free.pop_back();
  *p = g_pin_base + (size_t)i * kPinSlot;
  return cudaSuccess;
}

void pin_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  unsigned char* q = (unsigned char*)p;
  if (g_pin_base && q >= g_pin_base && q < g_pin_base + kPinSlot * kPinSlots) {
    g_pin_free.push_back((int)((q - g_pin_base) / kPinSlot));
    return;
  }
  cudaFreeHost(p);
}

// ---- the library's device memory pools (psi_internal.cuh): one per device, created on first
// use.  Like PyTorch's caching allocator, a pool keeps the memory the library frees for its
// next allocations (re-mapping freed memory made C5 builds 3-5x slower: 1.3-2.8 s instead of
// 0.43 s, measured); psi_empty_cache() returns it to the system, and PSI_POOL_KEEP_GB=<x>
// caps what a pool keeps (its release threshold).  The device's default pool, the caller's
// allocator and device-wide limits are never touched.
constexpr int kMaxDevices = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDevices] = {};
unsigned long long g_reserved_for[kMaxDevices] = {};

unsigned long long pool_keep_bytes() {
  const char* e = getenv("PSI_POOL_KEEP_GB");
  return e && *e ? (unsigned long long)(atof(e) * (double)(1ull << 30)) : ~0ull;
}

// Reserve a build's working set in ONE block of the pool the first time a graph this large
// is built on the device: later builds carve their temporaries out of it instead of mapping
// new memory around fragments (measured: +0.2-2 s C5 builds without enough of it).
void pool_reserve(int dev, unsigned long long est, cudaStream_t s) {
  if (dev < 0 || dev >= kMaxDevices || pool_keep_bytes() != ~0ull) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev] || est <= g_reserved_for[dev]) return;
  cudaMemPoolTrimTo(g_pool[dev], 0);
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, est, g_pool[dev], s) == cudaSuccess) {
    cudaFreeAsync(p, s);
    g_reserved_for[dev] = est;
  }
  cudaGetLastError();
}

void free_ctx(psi_ctx* c) {
  if (!c) return;
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->pr_exec) cudaGraphExecDestroy(c->pr_exec);
  if (c->pr_graph) cudaGraphDestroy(c->pr_graph);
  for (void* p : {(void*)c->pr.a, (void*)c->pr.a_first, (void*)c->pr.g, (void*)c->pr.dt,
                  (void*)c->pr.x0, (void*)c->pr.pi, (void*)c->g.nlead, (void*)c->g.kinv,
                  (void*)c->g.kw,
                  (void*)c->g.nf_loff, (void*)c->g.nf_leaders, (void*)c->g.nf_wt,
                  (void*)c->g.nf_lm})
    if (p) cudaFreeAsync(p, c->stream);
  void* ptrs[] = {c->g.edges, c->g.tile_row, c->g.a0, c->g.a1, c->g.g, c->g.wt, c->g.d1,
                  c->g.lam, c->g.psi, c->g.old_of_new, c->g.split, c->x[0], c->x[1],
                  c->p_in, c->p_out, c->eps_part1, c->eps_part2, c->history, c->st, c->prm,
                  c->hhot, c->g.h_ent, c->g.h_loff, c->g.h_prow, c->g.h_rslot, c->g.h_wslot,
                  c->scold, c->g.hsplit, c->ppart, c->epsw, c->g.s_words,
                  c->g.s_off, c->g.s_ipos, c->g.s_wrow, c->g.s_wstep, c->g.s_lrow, c->g.s_lp0, c->g.s_piece,
                  c->g.s_lwords};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, c->stream);
  for (auto e : c->b.exec) if (e) cudaGraphExecDestroy(e);
  for (auto g : c->b.graph) if (g) cudaGraphDestroy(g);
  for (void* p : {(void*)c->b.x[0], (void*)c->b.x[1], (void*)c->b.p_in, (void*)c->b.p_out,
                  (void*)c->b.part1, (void*)c->b.part2, (void*)c->b.st, (void*)c->b.prm,
                  (void*)c->b.history, (void*)c->g.b_a0, (void*)c->g.b_a1, (void*)c->g.b_g,
                  (void*)c->g.b_wt, (void*)c->g.b_d1, (void*)c->g.b_lam, (void*)c->g.b_psi,
                  (void*)c->g.b_tile_row, (void*)c->g.b_split})
    if (p) cudaFreeAsync(p, c->stream);
  pin_free(c->b.h_st);
  pin_free(c->b.h_prm);
  pin_free(c->h_st);
  pin_free(c->h_prm);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  delete c;
}

// A sliced-ELL plan with no long rows and no heavy rows needs no k_fix: k_sell's last CTA
// finishes the sweep (eps_t, loop control).  C2: one launch per sweep instead of two.
bool sell_fused(const psi_ctx* c) {
  return c->g.sell && c->g.sell_nlong == 0 && c->g.n_heavy == 0 && !c->g.ovl;
}

SweepArgs make_args(psi_ctx* c, cudaGraphConditionalHandle cond) {
  SweepArgs A{};
  A.edges = c->g.edges;
  A.tile_row = c->g.tile_row;
  A.ntiles = c->g.ntiles;
  A.split = c->g.split;
  A.nsplit = c->g.nsplit;
  A.nsplit_long = c->g.nsplit_long;
  A.p_in = c->p_in;
  A.p_out = c->p_out;
  A.a0 = c->g.a0;
  A.a = c->g.a1;
  A.g = c->g.g;
  A.wt = c->g.wt;
  A.d = c->g.d1;
  A.lam = c->g.lam;
  A.n_users = (double)c->n;
  A.n_lab = (int)c->n;
  A.n_act = (int)c->g.n_act;
  A.hot_lim = (int)c->hot_lim;
  A.psi = c->g.psi;
  A.x0 = c->x[0];
  A.x1 = c->x[1];
  A.eps_part1 = c->eps_part1;
  A.eps_part2 = c->eps_part2;
  A.grid1 = c->grid1;
  A.hot_smem = c->tc.hot_smem;
  A.l1_lim = c->tc.l1_lim;
  A.single_lo = getenv("PSI_SINGLE_L1") && atoi(getenv("PSI_SINGLE_L1")) == 0 ? 0x7fffffff
                                                                             : (int)c->g.single_lo;
  A.st_last = getenv("PSI_ST_LAST") ? atoi(getenv("PSI_ST_LAST")) : 0;
  A.n_heavy = (int)c->g.n_heavy;
  A.hhot = c->hhot;
  A.ovl = c->g.ovl;
  A.scold = c->scold;
  A.hsplit = c->g.hsplit;
  A.heavy.seg_shift = c->g.heavy_seg_shift;
  A.heavy.slots = c->g.heavy_slots;
  A.heavy.ent = c->g.h_ent;
  A.heavy.loff = c->g.h_loff;
  A.heavy.prow = c->g.h_prow;
  A.heavy.rslot = c->g.h_rslot;
  A.heavy.wslot = c->g.h_wslot;
  A.heavy.npanels = c->g.npanels;
  A.heavy.nseg = c->g.nseg;
  A.st = c->st;
  A.prm = c->prm;
  A.cond = cond;
  A.use_cond = 1;
  if (c->g.sell) {
    // the sliced-ELL sweep: no tiles, no split rows, eps_t partials per window (k_fix)
    A.use_sell = 1;
    A.nsplit = A.nsplit_long = 0;
    A.grid1 = 0;
    SellPlan& P = A.sell;
    P.words = c->g.s_words;
    P.soff = c->g.s_off;
    P.ipos = c->g.s_ipos;
    P.wrow = c->g.s_wrow;
    P.wstep = c->g.s_wstep;
    P.nwin = c->g.sell_nwin;
    P.wmax = 1 << c->g.sell_shift;
    P.lrow = c->g.s_lrow;
    P.lp0 = c->g.s_lp0;
    P.piece = c->g.s_piece;
    P.lwords = c->g.s_lwords;
    P.npieces = c->g.sell_npieces;
    P.ppart = c->ppart;
    P.epsw = c->epsw;
    P.nwords = c->g.sell_words;
    P.nlwords = c->g.sell_lwords;
    P.nlong = c->g.sell_nlong;
    A.sell_fused = sell_fused(c) ? 1 : 0;
  }
  return A;
}

cudaError_t add_kernel(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* dep, size_t ndep,
                       void* fn, int grid, int block, SweepArgs* args, int* n_extra,
                       size_t smem = 0) {
  cudaKernelNodeParams p{};
  p.func = fn;
  p.gridDim = dim3(grid);
  p.blockDim = dim3(block);
  p.sharedMemBytes = (unsigned)smem;
  void* kp[2] = {args, n_extra};
  p.kernelParams = kp;
  return cudaGraphAddKernelNode(node, g, dep, ndep, &p);
}

// The kernel nodes of one sweep (or the readout) after `dep` (may be NULL): k_heavy -> k_tiles
// -> k_fix.  With the overlapped plan k_tiles hangs on k_heavy by a programmatic edge from its
// launch-completion port (k_tiles starts once every k_heavy CTA has begun, so one CTA of each
// shares every SM) and k_fix waits for both.
cudaError_t add_sweep_nodes(psi_ctx* c, cudaGraph_t g, const cudaGraphNode_t* dep, SweepArgs* A,
                            bool readout, cudaGraphNode_t* last) {
  const bool hv = c->g.n_heavy > 0;
  cudaGraphNode_t nh{}, nt{};
  cudaError_t e;
  if (hv && (e = add_kernel(g, &nh, dep, dep ? 1 : 0, heavy_kernel_ptr(c->g.heavy_warps),
                            c->heavy_grid, c->heavy_block, A, nullptr, c->heavy_smem)) != cudaSuccess)
    return e;
  if (hv && c->g.ovl) {
    if ((e = add_kernel(g, &nt, nullptr, 0, readout ? c->tc.readout : c->tc.sweep, c->grid1,
                        c->tc.block, A, nullptr, c->tc.smem)) != cudaSuccess)
      return e;
    cudaGraphEdgeData ed{};
    ed.from_port = cudaGraphKernelNodePortLaunchCompletion;
    ed.type = cudaGraphDependencyTypeProgrammatic;
    if ((e = cudaGraphAddDependencies_v2(g, &nh, &nt, &ed, 1)) != cudaSuccess) return e;
    cudaGraphNode_t both[2] = {nh, nt};
    return add_kernel(g, last, both, 2, fix_kernel_ptr(readout), c->grid2, kFixBlock, A, nullptr);
  }
  if ((e = add_kernel(g, &nt, hv ? &nh : dep, (hv || dep) ? 1 : 0,
                      readout ? c->tc.readout : c->tc.sweep, c->grid1, c->tc.block, A, nullptr,
                      c->tc.smem)) != cudaSuccess)
    return e;
  if (sell_fused(c)) {
    *last = nt;
    return cudaSuccess;
  }
  return add_kernel(g, last, &nt, 1, fix_kernel_ptr(readout), c->grid2, kFixBlock, A, nullptr);
}

// The PageRank variant of the sweep arguments: the same kernels with Eq. (22)'s constants.
void pagerank_args(const psi_ctx* c, SweepArgs& A) {
  A.a0 = c->pr.x0;
  A.a = c->pr.a;
  A.a_first = c->pr.a_first;
  A.g = c->pr.g;
  A.wt = c->pr.dt;
}

// Power-psi:  k_init -> WHILE { sweep } -> readout.   PageRank: k_init -> WHILE { sweep }.
psi_status build_graph_exec(psi_ctx* c, bool pagerank = false) {
  cudaGraph_t& graph = pagerank ? c->pr_graph : c->graph;
  cudaGraphExec_t& exec = pagerank ? c->pr_exec : c->exec;
  API_CK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle cond;
  API_CK(cudaGraphConditionalHandleCreate(&cond, graph, 0, cudaGraphCondAssignDefault));
  SweepArgs A = make_args(c, cond);
  if (pagerank) pagerank_args(c, A);
  int n_int = (int)c->n;

  cudaGraphNode_t n_init, n_while, n_r1, n_r2;
  int init_grid = (int)std::min<long long>((c->n + 255) / 256, 148LL * 8);
  if (init_grid < 1) init_grid = 1;
  API_CK(add_kernel(graph, &n_init, nullptr, 0, init_kernel_ptr(), init_grid, 256, &A, &n_int));

  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  API_CK(cudaGraphAddNode(&n_while, graph, &n_init, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphNode_t b2;
  API_CK(add_sweep_nodes(c, body, nullptr, &A, false, &b2));
  if (!pagerank) API_CK(add_sweep_nodes(c, graph, &n_while, &A, true, &n_r2));
  (void)n_r1;
  API_CK(cudaGraphInstantiate(&exec, graph, 0));
  return PSI_OK;
}

cudaError_t launch(void* fn, int grid, int block, SweepArgs* A, int* extra, cudaStream_t s,
                   size_t smem = 0, bool programmatic = false) {
  void* kp[2] = {A, extra};
  if (!programmatic) return cudaLaunchKernel(fn, dim3(grid), dim3(block), kp, smem, s);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, kp);
}

// PSI_OVL_SERIAL=1 (measurement only): the overlapped plan's kernels launched one after the
// other, to time k_heavy and k_tiles of that plan separately
bool ovl_serial() {
  const char* e = getenv("PSI_OVL_SERIAL");
  return e && e[0] == '1';
}

// One sweep (or the readout) as direct launches on the context stream: k_heavy -> k_tiles ->
// k_fix; with the overlapped plan k_tiles is launched programmatically, so it starts once
// every k_heavy CTA has begun and runs beside it (griddepcontrol, psi_heavy.cu / psi_sweep.cu).
cudaError_t launch_sweep(psi_ctx* c, SweepArgs* A, bool readout, cudaEvent_t mid = nullptr,
                         cudaEvent_t after_tiles = nullptr) {
  const bool hv = c->g.n_heavy > 0;
  cudaError_t e;
  if (hv && (e = launch(heavy_kernel_ptr(c->g.heavy_warps), c->heavy_grid, c->heavy_block, A,
                        nullptr, c->stream, c->heavy_smem)) != cudaSuccess)
    return e;
  if (mid && (e = cudaEventRecord(mid, c->stream)) != cudaSuccess) return e;
  if ((e = launch(readout ? c->tc.readout : c->tc.sweep, c->grid1, c->tc.block, A, nullptr,
                  c->stream, c->tc.smem, hv && c->g.ovl && !ovl_serial())) != cudaSuccess)
    return e;
  if (after_tiles && (e = cudaEventRecord(after_tiles, c->stream)) != cudaSuccess) return e;
  if (sell_fused(c)) return cudaSuccess;
  return launch(fix_kernel_ptr(readout), c->grid2, kFixBlock, A, nullptr, c->stream);
}

// Direct stream launches of the same kernels (no CUDA graph, no conditional node): used by
// psi_time_sweep and, with PSI_GRAPH=0, by psi_iterate (profilers cannot see kernel nodes
// of graphs with conditional nodes).  The stop rule is evaluated on the host after every
// sweep from the device LoopState, exactly as the graph's WHILE condition does.
psi_status iterate_direct(psi_ctx* c, bool pagerank = false) {
  SweepArgs A = make_args(c, 0);
  if (pagerank) pagerank_args(c, A);
  A.use_cond = 0;
  int n_int = (int)c->n;
  int init_grid = (int)std::min<long long>((c->g.n_act + 255) / 256, 148LL * 8);
  if (init_grid < 1) init_grid = 1;
  API_CK(launch(init_kernel_ptr(), init_grid, 256, &A, &n_int, c->stream));
  const double eps = c->h_prm->eps;
  const long long max_iters = c->h_prm->max_iters;
  bool cont = c->h_prm->gap0 > eps && max_iters > 0;
  while (cont) {
    API_CK(launch_sweep(c, &A, false));
    API_CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(LoopState), cudaMemcpyDeviceToHost, c->stream));
    API_CK(cudaStreamSynchronize(c->stream));
    cont = !(c->h_st->status & 1) && c->h_st->gap > eps && c->h_st->iter < max_iters;
  }
  if (pagerank) return PSI_OK;
  API_CK(launch_sweep(c, &A, true));
  return PSI_OK;
}

// The persistent cooperative solver (k_solve) replaces the graph's WHILE loop on graphs with
// no k_heavy rows and at most PSI_COOP_TILES tiles (default kCoopTiles; 0 disables), when the
// sweep grid is co-resident.  It pays off where a sweep is launch-bound.
bool use_coop(const psi_ctx* c) {
  long long lim = kCoopEdges / c->g.tile;
  if (const char* e = getenv("PSI_COOP_TILES")) lim = atoll(e);
  return c->g.n_heavy == 0 && c->tc.solve && c->g.ntiles <= lim &&
         c->grid1 <= c->tc.solve_max_grid;
}

psi_status iterate_coop(psi_ctx* c, bool pagerank) {
  SweepArgs A = make_args(c, 0);
  if (pagerank) pagerank_args(c, A);
  A.use_cond = 0;
  int readout = pagerank ? 0 : 1;
  void* kp[2] = {&A, &readout};
  API_CK(cudaLaunchCooperativeKernel(c->tc.solve, dim3(c->grid1), dim3(c->tc.block), kp, c->tc.smem,
                                     c->stream));
  return PSI_OK;
}

bool use_graph() {
  const char* e = getenv("PSI_GRAPH");
  return !(e && e[0] == '0');
}

psi_status ensure_history(psi_ctx* c, long long need) {
  const long long kMaxHist = 1LL << 24;
  if (need > kMaxHist) need = kMaxHist;
  if (need < 1) need = 1;
  if (c->history && c->hist_cap >= need) return PSI_OK;
  if (c->history) {
    cudaFreeAsync(c->history, c->stream);
    c->device_bytes -= c->hist_cap * sizeof(double);
    c->history = nullptr;
  }
  long long cap = need < 1024 ? 1024 : need;
  API_CK(dev_alloc(&c->history, cap * sizeof(double), c->stream));
  c->hist_cap = cap;
  c->device_bytes += cap * sizeof(double);
  return PSI_OK;
}

// ||B||_col (reading R1): the column sums of B are lambda_i sum_{j in F(i)} 1/W_j, i.e.
// the readout psi_i = (d_i + lambda_i S_i) / N of the sweep's own kernels with x = 1/Wt on the
// active labels, d = lambda K_w (the follower-less followers' 1/Wt, folded at ingest) and N = 1.
// Computed once per context by one such pass (k_heavy + k_sell/k_tiles + k_fix), instead of a
// pass over every input edge in the ingest.
__global__ void k_col_prep(const double* wt, const double* lam, const double* kw, long long na,
                           double* x, double* dcol) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < na; i += stride) {
    x[i] = 1.0 / wt[i];
    dcol[i] = lam[i] * kw[i];
  }
}

// max of non-negative doubles (their bit patterns order the same way): warp max + one atomic
__global__ void k_max_nonneg(const double* v, long long n, unsigned long long* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long m = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = v[i];
    const unsigned long long b = x > 0.0 ? (unsigned long long)__double_as_longlong(x) : 0ull;
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void k_unpermute(const double* src, const double* scale, const int* old_of_new,
                            long long n, double* dst) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = scale ? src[i] * scale[i] : src[i];
    dst[old_of_new ? old_of_new[i] : i] = v;
  }
}

cudaError_t column_norm(psi_ctx* c) {
  const long long na = c->g.n_act;
  double kc = 0.0;
  cudaError_t e = cudaSuccess;
  if (na > 0) {
    double *dcol = nullptr, *colsum = nullptr;
    unsigned long long* dmax = nullptr;
    if ((e = dev_alloc(&dcol, na * sizeof(double), c->stream)) != cudaSuccess) return e;
    if ((e = dev_alloc(&colsum, na * sizeof(double), c->stream)) != cudaSuccess) return e;
    if ((e = dev_alloc(&dmax, sizeof(unsigned long long), c->stream)) != cudaSuccess) return e;
    cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), c->stream);
    const int grid = (int)std::max<long long>(1, std::min<long long>((na + 255) / 256, 148LL * 16));
    k_col_prep<<<grid, 256, 0, c->stream>>>(c->g.wt, c->g.lam, c->g.kw, na, c->x[0], dcol);
    SweepArgs A = make_args(c, 0);
    A.use_cond = 0;
    A.d = dcol;
    A.n_users = 1.0;
    A.psi = colsum;                            // (st->iter = 0: the pass reads x[0])
    if ((e = launch_sweep(c, &A, true)) != cudaSuccess) return e;
    k_max_nonneg<<<grid, 256, 0, c->stream>>>(colsum, na, dmax);
    unsigned long long h = 0;
    if ((e = cudaMemcpyAsync(&h, dmax, sizeof(h), cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return e;
    memcpy(&kc, &h, 8);
    cudaFreeAsync(dcol, c->stream);
    cudaFreeAsync(colsum, c->stream);
    cudaFreeAsync(dmax, c->stream);
  }
  c->g.kappa_col = kc;
  if (c->g.kw) cudaFreeAsync(c->g.kw, c->stream);
  c->g.kw = nullptr;
  return cudaGetLastError();
}

psi_status copy_out(const psi_ctx* c, const double* src, const double* scale, double* out,
                    int mem_kind) {
  if (!c->g.old_of_new && !scale) {
    API_CK(cudaMemcpyAsync(out, src, c->n * sizeof(double),
                           mem_kind == PSI_MEM_HOST ? cudaMemcpyDeviceToHost
                                                    : cudaMemcpyDeviceToDevice, c->stream));
    API_CK(cudaStreamSynchronize(c->stream));
    return PSI_OK;
  }
  double* dst = out;
  double* tmp = nullptr;
  if (mem_kind == PSI_MEM_HOST) {
    API_CK(dev_alloc((void**)&tmp, c->n * sizeof(double), c->stream));
    dst = tmp;
  }
  int grid = (int)std::min<long long>((c->n + 255) / 256, 148LL * 16);
  k_unpermute<<<grid < 1 ? 1 : grid, 256, 0, c->stream>>>(src, scale, c->g.old_of_new, c->n, dst);
  API_CK(cudaGetLastError());
  if (tmp) {
    API_CK(cudaMemcpyAsync(out, tmp, c->n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    API_CK(cudaFreeAsync(tmp, c->stream));
  }
  API_CK(cudaStreamSynchronize(c->stream));
  return PSI_OK;
}

// ------------------------------------------------------------- multi-profile batch
BatchArgs batch_args(psi_ctx* c, int gi, cudaGraphConditionalHandle cond) {
  const long long n = c->n, na = std::max<long long>(c->g.n_act, 1);
  BatchArgs A{};
  A.edges = c->g.edges;
  A.tile_row = c->g.b_tile_row;                  // the batch sweep's own 512-edge tiling
  A.ntiles = c->g.b_ntiles;
  A.split = c->g.b_split;
  A.nsplit = c->g.b_nsplit;
  A.nsplit_long = c->g.b_nsplit_long;
  A.p_in = c->b.p_in;
  A.p_out = c->b.p_out;
  A.a0 = reinterpret_cast<const d4*>(c->g.b_a0) + (size_t)gi * n;
  A.a = reinterpret_cast<const d4*>(c->g.b_a1) + (size_t)gi * na;
  A.g = reinterpret_cast<const d4*>(c->g.b_g) + (size_t)gi * na;
  A.wt = reinterpret_cast<const d4*>(c->g.b_wt) + (size_t)gi * na;
  A.d = reinterpret_cast<const d4*>(c->g.b_d1) + (size_t)gi * na;
  A.lam = reinterpret_cast<const d4*>(c->g.b_lam) + (size_t)gi * na;
  A.psi = reinterpret_cast<d4*>(c->g.b_psi) + (size_t)gi * n;
  A.x0 = c->b.x[0];
  A.x1 = c->b.x[1];
  A.eps_part1 = c->b.part1;
  A.eps_part2 = c->b.part2;
  A.n_users = (double)n;
  A.n_act = (int)c->g.n_act;
  A.hot_smem = c->b.cfg.hot_smem;
  A.hot_lim = (int)c->b.hot_lim;
  A.grid1 = c->b.cfg.grid1;
  A.st = c->b.st;
  A.prm = c->b.prm;
  A.cond = cond;
  A.use_cond = cond ? 1 : 0;
  return A;
}

cudaError_t add_bnode(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* dep, size_t ndep,
                      void* fn, int grid, int block, BatchArgs* args, size_t smem = 0) {
  cudaKernelNodeParams p{};
  p.func = fn;
  p.gridDim = dim3(grid);
  p.blockDim = dim3(block);
  p.sharedMemBytes = (unsigned)smem;
  void* kp[1] = {args};
  p.kernelParams = kp;
  return cudaGraphAddKernelNode(node, g, dep, ndep, &p);
}

// k_init_b -> WHILE { k_tiles_b -> k_fix_b } -> k_tiles_b<readout> -> k_fix_b<readout>, per group
psi_status batch_graph(psi_ctx* c, int gi) {
  cudaGraph_t& graph = c->b.graph[gi];
  API_CK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle cond;
  API_CK(cudaGraphConditionalHandleCreate(&cond, graph, 0, cudaGraphCondAssignDefault));
  BatchArgs A = batch_args(c, gi, cond);
  const BatchCfg& B = c->b.cfg;
  int init_grid = (int)std::min<long long>((c->g.n_act + 255) / 256, 148LL * 8);
  if (init_grid < 1) init_grid = 1;
  cudaGraphNode_t n0, nw, b1, b2, r1, r2;
  API_CK(add_bnode(graph, &n0, nullptr, 0, batch_init_ptr(), init_grid, 256, &A));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  API_CK(cudaGraphAddNode(&nw, graph, &n0, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  API_CK(add_bnode(body, &b1, nullptr, 0, batch_tiles_ptr(false), B.grid1, B.block1, &A, B.smem));
  API_CK(add_bnode(body, &b2, &b1, 1, batch_fix_ptr(false), B.grid2, batch_fix_block(), &A));
  API_CK(add_bnode(graph, &r1, &nw, 1, batch_tiles_ptr(true), B.grid1, B.block1, &A, B.smem));
  API_CK(add_bnode(graph, &r2, &r1, 1, batch_fix_ptr(true), B.grid2, batch_fix_block(), &A));
  API_CK(cudaGraphInstantiate(&c->b.exec[gi], graph, 0));
  return PSI_OK;
}

// sweep buffers of one group (reused by every group) and one graph per group
psi_status batch_setup(psi_ctx* c) {
  const long long n = c->n;
  auto& b = c->b;
  b.cfg = batch_config(c->g.b_ntiles, n, c->g.b_nsplit);
  int dev = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  double hot_frac = 0.65;                              // as the single-profile hot prefix
  if (const char* e = getenv("PSI_BATCH_HOT_FRAC")) hot_frac = atof(e);
  b.hot_lim = std::min<long long>((long long)(l2 * hot_frac / sizeof(d4)), c->g.n_hot);
  API_CK(dev_alloc((void**)&b.x[0], (n + 1) * sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.x[1], (n + 1) * sizeof(d4), c->stream));
  API_CK(cudaMemsetAsync(b.x[0] + n, 0, sizeof(d4), c->stream));      // sentinel x[n] = 0
  API_CK(cudaMemsetAsync(b.x[1] + n, 0, sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.p_in, (c->g.b_ntiles + 1) * sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.p_out, (c->g.b_ntiles + 1) * sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.part1, b.cfg.grid1 * sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.part2, b.cfg.grid2 * sizeof(d4), c->stream));
  API_CK(dev_alloc((void**)&b.st, sizeof(LoopStateB), c->stream));
  API_CK(dev_alloc((void**)&b.prm, sizeof(BatchParams), c->stream));
  API_CK(cudaMemsetAsync(b.st, 0, sizeof(LoopStateB), c->stream));
  API_CK(pin_alloc((void**)&b.h_st, sizeof(LoopStateB)));
  API_CK(pin_alloc((void**)&b.h_prm, sizeof(BatchParams)));
  const int G = c->g.ngroups;
  b.graph.assign(G, nullptr);
  b.exec.assign(G, nullptr);
  for (int gi = 0; gi < G; ++gi) {
    psi_status st = batch_graph(c, gi);
    if (st != PSI_OK) return st;
  }
  c->device_bytes += (size_t)(2 * (n + 1) + 2 * (c->g.b_ntiles + 1)) * sizeof(d4) +
                     (size_t)G * (2 * n + 5 * std::max<long long>(c->g.n_act, 1)) * sizeof(d4);
  API_CK(cudaStreamSynchronize(c->stream));
  return PSI_OK;
}

psi_status batch_iterate(psi_ctx* c, double eps, long long max_iters, int norm, int64_t* iters_out,
                         double* last_gap_out) {
  if (norm != PSI_NORM_ROW && norm != PSI_NORM_ONE)
    return fail(PSI_E_INVALID_ARG, "batch contexts support PSI_NORM_ROW and PSI_NORM_ONE");
  auto& b = c->b;
  const long long n = c->n, na = c->g.n_act;
  const int P = c->g.nprof;
  long long need = std::min<long long>(std::max<long long>(max_iters, 1), 1LL << 22);
  if (!b.history || b.hist_cap < need) {
    if (b.history) API_CK(cudaFreeAsync(b.history, c->stream));
    b.hist_cap = std::max<long long>(need, 1024);
    API_CK(dev_alloc((void**)&b.history, b.hist_cap * kBP * sizeof(double), c->stream));
  }
  b.T.assign(P, 0);
  b.gap.assign(P, 1.0);
  b.bad.assign(P, 0);
  b.hist.assign(P, {});
  b.have = false;
  std::vector<double> h;
  API_CK(cudaEventRecord(c->ev0, c->stream));
  for (int gi = 0; gi < c->g.ngroups; ++gi) {
    BatchParams& hp = *b.h_prm;
    hp.eps = eps;
    hp.max_iters = max_iters;
    hp.history = b.history;
    hp.hist_cap = b.hist_cap;
    hp.valid = 0;
    for (int l = 0; l < kBP; ++l) {
      const int p = gi * kBP + l;
      hp.kappa[l] = (p < P && norm == PSI_NORM_ROW) ? c->g.b_kappa_row[p] : 1.0;
      if (p < P) hp.valid |= 1u << l;
    }
    API_CK(cudaMemcpyAsync(b.prm, b.h_prm, sizeof(BatchParams), cudaMemcpyHostToDevice, c->stream));
    // follower-less users hold x = a0 in both buffers (never swept)
    const d4* a0 = reinterpret_cast<const d4*>(c->g.b_a0) + (size_t)gi * n;
    if (n > na) {
      API_CK(cudaMemcpyAsync(b.x[0] + na, a0 + na, (n - na) * sizeof(d4), cudaMemcpyDeviceToDevice,
                             c->stream));
      API_CK(cudaMemcpyAsync(b.x[1] + na, a0 + na, (n - na) * sizeof(d4), cudaMemcpyDeviceToDevice,
                             c->stream));
    }
    API_CK(cudaGraphLaunch(b.exec[gi], c->stream));
    API_CK(cudaMemcpyAsync(b.h_st, b.st, sizeof(LoopStateB), cudaMemcpyDeviceToHost, c->stream));
    API_CK(cudaStreamSynchronize(c->stream));
    const long long iters = std::min<long long>(b.h_st->iter, b.hist_cap);
    h.resize((size_t)iters * kBP);
    if (iters > 0) {
      API_CK(cudaMemcpyAsync(h.data(), b.history, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream));
      API_CK(cudaStreamSynchronize(c->stream));
    }
    for (int l = 0; l < kBP; ++l) {
      const int p = gi * kBP + l;
      if (p >= P) continue;
      b.T[p] = b.h_st->T[l];
      b.gap[p] = b.h_st->gap[l];
      b.bad[p] = (b.h_st->status >> l) & 1;
      const long long tp = std::min<long long>(b.T[p], iters);
      b.hist[p].resize(tp);
      for (long long t = 0; t < tp; ++t) b.hist[p][t] = h[(size_t)t * kBP + l];
    }
  }
  API_CK(cudaEventRecord(c->ev1, c->stream));
  API_CK(cudaEventSynchronize(c->ev1));
  float ms = 0;
  API_CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->iterate_ms = ms;
  c->last_solver = 0;
  long long Tm = 0;
  double gm = 0.0;
  bool any_bad = false, unconv = false;
  for (int p = 0; p < P; ++p) {
    Tm = std::max(Tm, b.T[p]);
    gm = std::max(gm, b.gap[p]);
    any_bad |= b.bad[p] != 0;
    unconv |= b.gap[p] > eps;
  }
  c->last_T = Tm;
  c->last_gap = gm;
  c->series_ok = false;
  if (iters_out) *iters_out = Tm;
  if (last_gap_out) *last_gap_out = gm;
  if (any_bad) return fail(PSI_E_NUMERIC, "epsilon_t became non-finite for some profile");
  c->have_psi = true;
  b.have = true;
  if (unconv) {
    fail(PSI_NOT_CONVERGED, "not converged: some profile's gap %.3e > eps %.3e", gm, eps);
    return PSI_NOT_CONVERGED;
  }
  return PSI_OK;
}

psi_status batch_copy_out(const psi_ctx* c, double* out, int mem_kind) {
  const size_t bytes = (size_t)c->g.nprof * c->n * sizeof(double);
  double* dst = out;
  double* tmp = nullptr;
  if (mem_kind == PSI_MEM_HOST) {
    API_CK(dev_alloc((void**)&tmp, bytes, c->stream));
    dst = tmp;
  }
  API_CK(batch_unpermute(c->g.b_psi, c->g.old_of_new, c->n, c->g.nprof, dst, c->stream));
  if (tmp) {
    API_CK(cudaMemcpyAsync(out, tmp, bytes, cudaMemcpyDeviceToHost, c->stream));
    API_CK(cudaFreeAsync(tmp, c->stream));
  }
  API_CK(cudaStreamSynchronize(c->stream));
  return PSI_OK;
}

}  // namespace

cudaMemPool_t psi::lib_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
    unsigned long long keep = pool_keep_bytes();       // default: keep everything (cached)
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    g_pool[dev] = p;
  }
  return g_pool[dev];
}

extern "C" {

const char* psi_last_error(void) { return g_err.c_str(); }

psi_status psi_empty_cache(void) {
  g_err.clear();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return fail(PSI_E_CUDA, "cudaGetDevice failed");
  API_CK(cudaDeviceSynchronize());                    // stream-ordered frees have completed
  scratch_release(dev);                               // the build scratch (its own lock first)
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) return PSI_OK;
  API_CK(cudaMemPoolTrimTo(g_pool[dev], 0));
  g_reserved_for[dev] = 0;
  return PSI_OK;
}

}  // extern "C"

namespace {
psi_status batch_setup(psi_ctx* c);

psi_status build(int64_t n, int64_t m, const int64_t* row_ptr, const int32_t* followers,
                 const double* lambda, const double* mu, int nprof, int mem_kind, void* stream,
                 psi_ctx** out) {
  g_err.clear();
  if (!out) return fail(PSI_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > 2147483647LL) return fail(PSI_E_INVALID_ARG, "n = %lld outside [1, 2^31-1]", (long long)n);
  if (m < 0 || m > 2147483647LL) return fail(PSI_E_INVALID_ARG, "m = %lld outside [0, 2^31-1]", (long long)m);
  if (!row_ptr || !lambda || !mu || (m > 0 && !followers))
    return fail(PSI_E_INVALID_ARG, "NULL input pointer");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);

  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(PSI_E_CUDA, "cudaGetDevice failed");
  if (!lib_pool()) return fail(PSI_E_CUDA, "cannot create the library's memory pool");
  psi_ctx* c = new psi_ctx;
  c->n = n;
  c->m = m;
  c->dev = dev;
  c->stream = (cudaStream_t)stream;
  // (the staged inputs and the transpose's sort arrays come from the build scratch, not the pool)
  {
    // twice the build's pool working set (~12 B per edge + 160 B per user and profile): with
    // less headroom the pool maps new memory around fragments now and then (C5 builds of
    // 0.5-2.3 s instead of 0.34 s; a 40 GB block made every repeated build 338-344 ms, measured)
    unsigned long long est = 2ull * (12ull * (unsigned long long)m +
                                     (unsigned long long)nprof * 160ull * (unsigned long long)n) +
                             (256ull << 20);
    if (const char* e = getenv("PSI_POOL_RESERVE_GB"))        // measurement: a larger block
      est = std::max(est, (unsigned long long)(atof(e) * (double)(1ull << 30)));
    size_t fr = 0, tot = 0;                                   // never more than half the free memory
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) est = std::min<unsigned long long>(est, fr / 2);
    pool_reserve(dev, est, c->stream);
  }
  auto bail = [&](psi_status st) { free_ctx(c); return st; };
#define B_CK(call)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? PSI_E_OOM : PSI_E_CUDA,            \
                       "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__)); \
  } while (0)

  B_CK(cudaEventCreate(&c->ev0));
  B_CK(cudaEventCreate(&c->ev1));
  B_CK(cudaEventRecord(c->ev0, c->stream));

  // The build's scratch (staged inputs, the transpose's sort arrays) is per device and kept
  // across builds; this build owns it until the ingest has returned (psi_ingest.cu).
  std::unique_lock<std::mutex> scratch_lock(*scratch_mutex(dev));
  // Stage host inputs (borrowed: copied, never retained) in scratch slot 0.
  const long long* rp_d = (const long long*)row_ptr;
  const int* idx_d = followers;
  const double* lam_d = lambda;
  const double* mu_d = mu;
  void* staged[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t side = nullptr;
  cudaEvent_t act_ev = nullptr;
  struct SideDone {                     // the side copy has finished before the build returns
    cudaStream_t& s;
    cudaEvent_t& e;
    ~SideDone() {
      if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
      if (e) cudaEventDestroy(e);
    }
  } side_done{side, act_ev};
  if (mem_kind == PSI_MEM_HOST) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b0 = al((n + 1) * sizeof(long long)), b1 = al((m > 0 ? m : 1) * sizeof(int)),
                 b2 = al(nprof * n * sizeof(double));
    unsigned char* sp = nullptr;
    B_CK(scratch_get(dev, 0, b0 + b1 + 2 * b2, (void**)&sp));
    staged[0] = sp;
    staged[1] = sp + b0;
    staged[2] = sp + b0 + b1;
    staged[3] = sp + b0 + b1 + b2;
    B_CK(cudaMemcpyAsync(staged[0], row_ptr, (n + 1) * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    if (m > 0)
      B_CK(cudaMemcpyAsync(staged[1], followers, m * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    // lambda, mu on a side stream (first used after the transpose: the ingest waits on act_ev),
    // so their copy overlaps the graph's validation and transpose
    B_CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    B_CK(cudaEventCreateWithFlags(&act_ev, cudaEventDisableTiming));
    B_CK(cudaEventRecord(act_ev, c->stream));                 // (after the inputs' staging slot
    B_CK(cudaStreamWaitEvent(side, act_ev, 0));               //  is this build's, stream order)
    B_CK(cudaMemcpyAsync(staged[2], lambda, nprof * n * sizeof(double), cudaMemcpyHostToDevice,
                         side));
    B_CK(cudaMemcpyAsync(staged[3], mu, nprof * n * sizeof(double), cudaMemcpyHostToDevice, side));
    B_CK(cudaEventRecord(act_ev, side));
    rp_d = (const long long*)staged[0];
    idx_d = (const int*)staged[1];
    lam_d = (const double*)staged[2];
    mu_d = (const double*)staged[3];
    if (const char* e = getenv("PSI_TRACE")) {          // ingest trace: the staging copies
      if (*e == '1') {
        const auto h0 = std::chrono::steady_clock::now();
        cudaEvent_t et;
        cudaEventCreate(&et);
        cudaEventRecord(et, c->stream);
        cudaStreamSynchronize(c->stream);
        float dms = 0.f;
        cudaEventElapsedTime(&dms, c->ev0, et);
        cudaEventDestroy(et);
        fprintf(stderr, "[psi build ] staging H2D (pool allocs + copies)  device %9.2f ms, host wait %9.2f ms\n",
                dms, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
      }
    }
  }

  char msg[512] = {0};
  int rc = ingest(n, m, rp_d, idx_d, lam_d, mu_d, nprof, c->stream, c->g, msg, sizeof(msg), act_ev);
  if (rc != PSI_OK) return bail(fail(rc, "%s", msg));
  scratch_lock.unlock();          // (stream-ordered: a later build's reuse follows this work)

  // Iteration buffers.
  c->tc = c->g.sell ? sell_config(n, c->g.sell_shift)
                    : tiles_config(c->g.ntiles, n, c->g.tile, c->g.ovl != 0);
  c->grid1 = c->tc.grid;
  {
    // Hot prefix of x kept in L2 (evict_last) in BOTH ping-pong buffers: PSI_HOT_MB per
    // buffer (default: 0.65 of L2, measured best at C5: profiles/r1/tune_hot_mb_r1.txt), never
    // more than the users with >= 2 leaders.
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    double hot_mb = l2 * 0.65 / (1 << 20);
    if (const char* e = getenv("PSI_HOT_MB")) hot_mb = atof(e);
    long long lim = (long long)(hot_mb * (1 << 20) / 8.0);
    c->hot_lim = std::min<long long>(std::max<long long>(lim, 0), c->g.n_hot);
    // cudaLimitMaxL2FetchGranularity is device-wide state: never changed by default (it made
    // no measurable difference); PSI_L2_FETCH=<bytes> opts in (tuning only).
    if (const char* e = getenv("PSI_L2_FETCH"))
      if (atoi(e) > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e));
  }
  c->grid2 = fix_grid(c->g.nsplit);
  if (c->g.sell) {
    // k_fix finishes the long rows (thread each) and reduces the windows' eps_t partials (a
    // few per thread), then the stop rule
    c->grid2 = std::max(1, std::min(148, (std::max(c->g.sell_nwin, c->g.sell_nlong) + kFixBlock - 1) /
                                             kFixBlock));
    B_CK(dev_alloc(&c->ppart, (size_t)std::max(c->g.sell_npieces, 1) * sizeof(double), c->stream));
    B_CK(dev_alloc(&c->epsw, (size_t)std::max(c->g.sell_nwin, 1) * sizeof(double), c->stream));
  }
  if (c->g.ovl)                                       // + k_fix's pass over the heavy rows
    c->grid2 = std::max(c->grid2, (int)std::min<long long>((c->g.n_heavy + kFixBlock - 1) / kFixBlock,
                                                            148LL * 8));
  if (c->g.n_heavy > 0) {
    int dev = 0, sms = 0;
    B_CK(cudaGetDevice(&dev));
    B_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    c->heavy_grid = std::max(1, std::min(sms, c->g.npanels));
    if (const char* e = getenv("PSI_HEAVY_GRID"))          // measurement: fewer SMs
      if (atoi(e) > 0) c->heavy_grid = std::min(c->heavy_grid, atoi(e));
    c->heavy_smem = heavy_smem_bytes(c->g.nseg, c->g.heavy_seg_shift, c->g.heavy_slots,
                                     c->g.heavy_warps);
    c->heavy_block = 32 * (c->g.heavy_warps + 1);
    B_CK(cudaFuncSetAttribute(heavy_kernel_ptr(c->g.heavy_warps),
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->heavy_smem));
    if (c->g.ovl) B_CK(dev_alloc(&c->scold, (size_t)c->g.n_heavy * sizeof(double), c->stream));
    B_CK(dev_alloc(&c->hhot, (size_t)c->g.n_heavy * sizeof(double), c->stream));
    B_CK(cudaMemsetAsync(c->hhot, 0, (size_t)c->g.n_heavy * sizeof(double), c->stream));
  }
  B_CK(dev_alloc(&c->x[0], (n + 1) * sizeof(double), c->stream));      // + sentinel x[n] = 0
  B_CK(dev_alloc(&c->x[1], (n + 1) * sizeof(double), c->stream));
  B_CK(cudaMemsetAsync(c->x[0] + n, 0, sizeof(double), c->stream));
  B_CK(cudaMemsetAsync(c->x[1] + n, 0, sizeof(double), c->stream));
  B_CK(dev_alloc(&c->p_in, (c->g.ntiles + 1) * sizeof(double), c->stream));
  B_CK(dev_alloc(&c->p_out, (c->g.ntiles + 1) * sizeof(double), c->stream));
  // x 2: k_solve double-buffers the partials by the parity of t
  B_CK(dev_alloc(&c->eps_part1, 2 * c->grid1 * sizeof(double), c->stream));
  B_CK(dev_alloc(&c->eps_part2, 2 * std::max(c->grid1, c->grid2) * sizeof(double), c->stream));
  B_CK(dev_alloc(&c->st, sizeof(LoopState), c->stream));
  B_CK(dev_alloc(&c->prm, sizeof(LoopParams), c->stream));
  B_CK(cudaMemsetAsync(c->st, 0, sizeof(LoopState), c->stream));
  B_CK(column_norm(c));                               // ||B||_col (x[0] is scratch until here)
  // Follower-less users keep x = a0 in both buffers for ever (they are never written).
  B_CK(cudaMemcpyAsync(c->x[0], c->g.a0, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  B_CK(cudaMemcpyAsync(c->x[1], c->g.a0, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  B_CK(pin_alloc((void**)&c->h_st, sizeof(LoopState)));
  B_CK(pin_alloc((void**)&c->h_prm, sizeof(LoopParams)));
  B_CK(cudaEventRecord(c->ev1, c->stream));
  B_CK(cudaStreamSynchronize(c->stream));
  float ms = 0;
  B_CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->ingest_ms = ms;
  c->device_bytes = (long long)c->g.ntiles * c->g.tile * 4 + 6 * n * 8 + 4 * c->g.n_act * 8 +
                    (c->g.ntiles + 1) * (4 + 16) + (long long)c->g.nsplit * 16 + n * 4;

  psi_status gs = build_graph_exec(c);
  if (gs != PSI_OK) return bail(gs);
  if (nprof > 1) {
    gs = batch_setup(c);
    if (gs != PSI_OK) return bail(gs);
  }
  *out = c;
  return PSI_OK;
#undef B_CK
}
}  // namespace

extern "C" {

psi_status psi_build_graph(int64_t n, int64_t m, const int64_t* row_ptr, const int32_t* followers,
                           const double* lambda, const double* mu, int mem_kind, void* stream,
                           psi_ctx** out) {
  NvtxRange nvtx_("psi_build_graph");
  return build(n, m, row_ptr, followers, lambda, mu, 1, mem_kind, stream, out);
}

psi_status psi_build_graph_batch(int64_t n, int64_t m, const int64_t* row_ptr,
                                 const int32_t* followers, int64_t nprof, const double* lambda,
                                 const double* mu, int mem_kind, void* stream, psi_ctx** out) {
  NvtxRange nvtx_("psi_build_graph_batch");
  g_err.clear();
  if (nprof < 1 || nprof > 4096) {
    if (out) *out = nullptr;
    return fail(PSI_E_INVALID_ARG, "nprof = %lld outside [1, 4096]", (long long)nprof);
  }
  if ((double)nprof * (double)n > 2147483647.0 * 64.0) {
    if (out) *out = nullptr;
    return fail(PSI_E_INVALID_ARG, "nprof * n too large");
  }
  return build(n, m, row_ptr, followers, lambda, mu, (int)nprof, mem_kind, stream, out);
}

psi_status psi_iterate(psi_ctx* c, double eps, int64_t max_iters, int norm, int64_t* iters_out,
                       double* last_gap_out) {
  NvtxRange nvtx_("psi_iterate");
  g_err.clear();
  if (!c) return fail(PSI_E_INVALID_ARG, "ctx is NULL");
  if (!(eps >= 0.0)) return fail(PSI_E_INVALID_ARG, "eps must be >= 0 (got %g)", eps);
  if (max_iters < 0) return fail(PSI_E_INVALID_ARG, "max_iters must be >= 0");
  double kappa;
  switch (norm) {
    case PSI_NORM_ROW: kappa = c->g.kappa_row; break;
    case PSI_NORM_COL: kappa = c->g.kappa_col; break;
    case PSI_NORM_ONE: kappa = 1.0; break;
    default: return fail(PSI_E_INVALID_ARG, "bad norm %d", norm);
  }
  c->have_psi = false;
  if (c->g.nprof > 1) return batch_iterate(c, eps, max_iters, norm, iters_out, last_gap_out);
  psi_status hs = ensure_history(c, max_iters);
  if (hs != PSI_OK) return hs;
  c->h_prm->eps = eps;
  c->h_prm->max_iters = max_iters;
  c->h_prm->kappa = kappa;
  c->h_prm->history = c->history;
  c->h_prm->hist_cap = c->hist_cap;
  c->h_prm->gap0 = 1.0;                               // Alg. 2 line 4
  c->h_prm->eps1_extra = 0.0;
  API_CK(cudaMemcpyAsync(c->prm, c->h_prm, sizeof(LoopParams), cudaMemcpyHostToDevice, c->stream));
  API_CK(cudaEventRecord(c->ev0, c->stream));
  c->series_ok = false;
  c->last_solver = use_coop(c) ? 1 : use_graph() ? 0 : 2;
  if (c->last_solver == 1) {
    psi_status cs = iterate_coop(c, false);
    if (cs != PSI_OK) return cs;
  } else if (c->last_solver == 0) {
    API_CK(cudaGraphLaunch(c->exec, c->stream));
  } else {
    psi_status ds = iterate_direct(c);
    if (ds != PSI_OK) return ds;
  }
  API_CK(cudaEventRecord(c->ev1, c->stream));
  API_CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(LoopState), cudaMemcpyDeviceToHost, c->stream));
  API_CK(cudaStreamSynchronize(c->stream));
  float ms = 0;
  API_CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->iterate_ms = ms;
  c->last_T = c->h_st->iter;
  c->last_gap = c->h_st->gap;
  if (iters_out) *iters_out = c->last_T;
  if (last_gap_out) *last_gap_out = c->last_gap;
  if (c->h_st->status & 1)
    return fail(PSI_E_NUMERIC, "epsilon_t became non-finite at t = %lld", c->last_T);
  c->have_psi = true;
  c->series_ok = true;
  if (c->last_gap > eps) {
    fail(PSI_NOT_CONVERGED, "not converged: gap %.3e > eps %.3e after %lld sweeps",
         c->last_gap, eps, c->last_T);
    return PSI_NOT_CONVERGED;
  }
  return PSI_OK;
}

psi_status psi_get_psi(const psi_ctx* c, double* out, int mem_kind) {
  NvtxRange nvtx_("psi_get_psi");
  g_err.clear();
  if (!c || !out) return fail(PSI_E_INVALID_ARG, "NULL argument");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);
  if (!c->have_psi) return fail(PSI_E_STATE, "no successful psi_iterate on this context");
  if (c->g.nprof > 1) return batch_copy_out(c, out, mem_kind);
  return copy_out(c, c->g.psi, nullptr, out, mem_kind);
}

psi_status psi_get_series(const psi_ctx* c, double* out, int mem_kind) {
  NvtxRange nvtx_("psi_get_series");
  g_err.clear();
  if (!c || !out) return fail(PSI_E_INVALID_ARG, "NULL argument");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);
  if (!c->have_psi || !c->series_ok)
    return fail(PSI_E_STATE, "no psi_iterate since the last psi_pagerank / psi_time_sweep");
  // s_T = Wt * x_T (kernel state, psi_internal.cuh)
  return copy_out(c, c->x[c->last_T & 1], c->g.wt, out, mem_kind);
}

psi_status psi_get_residual_history(const psi_ctx* c, double* out, int64_t cap, int64_t* len_out) {
  g_err.clear();
  if (!c || (cap > 0 && !out)) return fail(PSI_E_INVALID_ARG, "NULL argument");
  if (!c->have_psi && !c->have_pr)
    return fail(PSI_E_STATE, "no successful psi_iterate / psi_pagerank on this context");
  if (c->g.nprof > 1 && c->b.have)
    return fail(PSI_E_STATE, "batch context: use psi_get_profile_history");
  // entries stored: T, or the history cap if T exceeded it (2^24); len_out never counts
  // entries that were not written
  const long long stored = std::min<long long>(c->last_T, c->hist_cap);
  if (len_out) *len_out = stored;
  long long k = stored;
  if (k > cap) k = cap;
  if (k > 0) {
    API_CK(cudaMemcpyAsync(out, c->history, k * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    API_CK(cudaStreamSynchronize(c->stream));
  }
  return PSI_OK;
}

psi_status psi_get_info(const psi_ctx* c, psi_info* out) {
  g_err.clear();
  if (!c || !out) return fail(PSI_E_INVALID_ARG, "NULL argument");
  memset(out, 0, sizeof(*out));
  out->n = c->n;
  out->m = c->m;
  out->n_f = c->g.n_f;
  out->n_g = c->g.n_g;
  out->n_leaderless = c->g.n_leaderless;
  out->kappa_row = c->g.kappa_row;
  out->kappa_col = c->g.kappa_col;
  out->rho_A = c->g.rho_A;
  out->ingest_ms = c->ingest_ms;
  out->iterate_ms = c->iterate_ms;
  out->last_iters = c->last_T;
  out->last_gap = c->last_gap;
  out->num_tiles = c->g.ntiles;
  out->num_long_rows = c->g.nsplit;
  out->grid = c->grid1;
  out->device_bytes = (int64_t)c->device_bytes;
  out->relabeled = c->g.relabeled;
  out->block = c->tc.block;
  out->hot_smem = c->tc.hot_smem;
  out->n_heavy = c->g.n_heavy;
  out->heavy_entries = c->g.heavy_entries;
  out->heavy_panels = c->g.npanels;
  out->heavy_labels = (int64_t)c->g.nseg * kSeg;
  out->last_solver = c->last_solver;
  out->n_profiles = c->g.nprof;
  out->tile_edges = c->g.tile;
  out->overlapped = (c->g.ovl && c->g.n_heavy > 0) ? 1 : 0;
  out->sliced_ell = c->g.sell;
  out->sell_long_rows = c->g.sell_nlong;
  out->sell_pieces = c->g.sell_npieces;
  out->sell_words = c->g.sell_words;
  out->stream_edges = c->g.m_act;
  return PSI_OK;
}

psi_status psi_time_sweep(psi_ctx* c, int64_t sweeps, double* heavy_ms, double* tiles_ms,
                          double* fix_ms) {
  NvtxRange nvtx_("psi_time_sweep");
  g_err.clear();
  if (!c || sweeps < 1) return fail(PSI_E_INVALID_ARG, "ctx NULL or sweeps < 1");
  psi_status hs = ensure_history(c, sweeps);
  if (hs != PSI_OK) return hs;
  c->h_prm->eps = 0.0;
  c->h_prm->max_iters = sweeps;
  c->h_prm->kappa = c->g.kappa_row;
  c->h_prm->history = c->history;
  c->h_prm->hist_cap = c->hist_cap;
  c->h_prm->gap0 = 1.0;
  c->h_prm->eps1_extra = 0.0;
  API_CK(cudaMemcpyAsync(c->prm, c->h_prm, sizeof(LoopParams), cudaMemcpyHostToDevice, c->stream));
  c->series_ok = false;
  SweepArgs A = make_args(c, 0);
  A.use_cond = 0;
  int n_int = (int)c->n;
  int init_grid = (int)std::min<long long>((c->g.n_act + 255) / 256, 148LL * 8);
  if (init_grid < 1) init_grid = 1;
  API_CK(launch(init_kernel_ptr(), init_grid, 256, &A, &n_int, c->stream));
  cudaEvent_t e[4];
  for (auto& x : e) API_CK(cudaEventCreate(&x));
  double t0 = 0, t1 = 0, t2 = 0;
  psi_status rc = PSI_OK;
  const bool hv = c->g.n_heavy > 0;
  // overlapped plan: k_heavy and k_tiles run concurrently, so the pair is timed as one (tiles_ms)
  // and heavy_ms is 0 -- no event may sit between the two launches (it would serialise them)
  const bool ovl = hv && c->g.ovl && !ovl_serial();
  for (int64_t k = 0; k < sweeps && rc == PSI_OK; ++k) {
    float a = 0, b = 0, d = 0;
    if (cudaEventRecord(e[0], c->stream) != cudaSuccess ||
        launch_sweep(c, &A, false, ovl ? nullptr : e[1], e[2]) != cudaSuccess ||
        cudaEventRecord(e[3], c->stream) != cudaSuccess ||
        cudaEventSynchronize(e[3]) != cudaSuccess ||
        (!ovl && cudaEventElapsedTime(&d, e[0], e[1]) != cudaSuccess) ||
        cudaEventElapsedTime(&a, ovl ? e[0] : e[1], e[2]) != cudaSuccess ||
        cudaEventElapsedTime(&b, e[2], e[3]) != cudaSuccess)
      rc = fail(PSI_E_CUDA, "psi_time_sweep: %s", cudaGetErrorString(cudaGetLastError()));
    t0 += d;
    t1 += a;
    t2 += b;
  }
  for (auto& x : e) cudaEventDestroy(x);
  if (rc != PSI_OK) return rc;
  c->have_psi = false;     // the iterate state is mid-solve: require a new psi_iterate
  if (heavy_ms) *heavy_ms = hv ? t0 / sweeps : 0.0;
  if (tiles_ms) *tiles_ms = t1 / sweeps;
  if (fix_ms) *fix_ms = t2 / sweeps;
  return PSI_OK;
}

psi_status psi_pagerank(psi_ctx* c, double alpha, double eps, int64_t max_iters,
                        int64_t* iters_out, double* last_gap_out) {
  NvtxRange nvtx_("psi_pagerank");
  g_err.clear();
  if (!c) return fail(PSI_E_INVALID_ARG, "ctx is NULL");
  if (!(alpha >= 0.0 && alpha < 1.0)) return fail(PSI_E_INVALID_ARG, "alpha must be in [0, 1)");
  if (!(eps >= 0.0)) return fail(PSI_E_INVALID_ARG, "eps must be >= 0 (got %g)", eps);
  if (max_iters < 0) return fail(PSI_E_INVALID_ARG, "max_iters must be >= 0");
  const long long n = c->n, na = std::max<long long>(c->g.n_act, 1);
  if (!c->pr.a) {
    API_CK(dev_alloc(&c->pr.a, na * sizeof(double), c->stream));
    API_CK(dev_alloc(&c->pr.a_first, na * sizeof(double), c->stream));
    API_CK(dev_alloc(&c->pr.g, na * sizeof(double), c->stream));
    API_CK(dev_alloc(&c->pr.dt, n * sizeof(double), c->stream));
    API_CK(dev_alloc(&c->pr.x0, n * sizeof(double), c->stream));
    API_CK(dev_alloc(&c->pr.pi, n * sizeof(double), c->stream));
    c->device_bytes += (3 * na + 3 * n) * sizeof(double);
  }
  c->have_pr = false;
  API_CK(pagerank_prep(c->g, n, alpha, c->pr, c->stream));
  psi_status hs = ensure_history(c, max_iters);
  if (hs != PSI_OK) return hs;
  c->h_prm->eps = eps;
  c->h_prm->max_iters = max_iters;
  c->h_prm->kappa = 1.0;                              // stop on ||pi_t - pi_{t-1}||_1 itself
  c->h_prm->history = c->history;
  c->h_prm->hist_cap = c->hist_cap;
  c->h_prm->gap0 = INFINITY;                          // the oracle's first test always passes
  // follower-less users are not swept; in the first sweep each one's pi moves by alpha/N
  c->h_prm->eps1_extra = (double)(c->n - c->g.n_act) * alpha / (double)c->n;
  API_CK(cudaMemcpyAsync(c->prm, c->h_prm, sizeof(LoopParams), cudaMemcpyHostToDevice, c->stream));
  c->series_ok = false;
  API_CK(cudaEventRecord(c->ev0, c->stream));
  c->last_solver = use_coop(c) ? 1 : use_graph() ? 0 : 2;
  if (c->last_solver == 1) {
    psi_status cs = iterate_coop(c, true);
    if (cs != PSI_OK) return cs;
  } else if (c->last_solver == 0) {
    if (!c->pr_exec) {
      psi_status gs = build_graph_exec(c, true);
      if (gs != PSI_OK) return gs;
    }
    API_CK(cudaGraphLaunch(c->pr_exec, c->stream));
  } else {
    psi_status ds = iterate_direct(c, true);
    if (ds != PSI_OK) return ds;
  }
  API_CK(cudaEventRecord(c->ev1, c->stream));
  API_CK(cudaMemcpyAsync(c->h_st, c->st, sizeof(LoopState), cudaMemcpyDeviceToHost, c->stream));
  API_CK(cudaStreamSynchronize(c->stream));
  float ms = 0;
  API_CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->iterate_ms = ms;
  const long long T = c->h_st->iter;
  const double gap = c->h_st->gap;
  c->last_T = T;
  c->last_gap = gap;
  if (iters_out) *iters_out = T;
  if (last_gap_out) *last_gap_out = gap;
  if (c->h_st->status & 1) return fail(PSI_E_NUMERIC, "||pi_t - pi_(t-1)|| became non-finite at t = %lld", T);
  API_CK(pagerank_readout(c->g, n, alpha, (T & 1) ? c->x[1] : c->x[0], T, c->pr, c->stream));
  API_CK(cudaStreamSynchronize(c->stream));
  c->pr_T = T;
  c->pr_alpha = alpha;
  c->have_pr = true;
  if (gap > eps) {
    fail(PSI_NOT_CONVERGED, "not converged: gap %.3e > eps %.3e after %lld sweeps", gap, eps, T);
    return PSI_NOT_CONVERGED;
  }
  return PSI_OK;
}

psi_status psi_get_profile_stats(const psi_ctx* c, int64_t* iters, double* gaps) {
  g_err.clear();
  if (!c) return fail(PSI_E_INVALID_ARG, "ctx is NULL");
  if (c->g.nprof < 2) return fail(PSI_E_STATE, "not a batch context (psi_build_graph_batch)");
  if (!c->b.have) return fail(PSI_E_STATE, "no successful psi_iterate on this batch context");
  for (int p = 0; p < c->g.nprof; ++p) {
    if (iters) iters[p] = c->b.T[p];
    if (gaps) gaps[p] = c->b.gap[p];
  }
  return PSI_OK;
}

psi_status psi_get_profile_history(const psi_ctx* c, int64_t profile, double* out, int64_t cap,
                                   int64_t* len_out) {
  g_err.clear();
  if (!c || (cap > 0 && !out)) return fail(PSI_E_INVALID_ARG, "NULL argument");
  if (c->g.nprof < 2) return fail(PSI_E_STATE, "not a batch context (psi_build_graph_batch)");
  if (!c->b.have) return fail(PSI_E_STATE, "no successful psi_iterate on this batch context");
  if (profile < 0 || profile >= c->g.nprof) return fail(PSI_E_INVALID_ARG, "bad profile %lld", (long long)profile);
  const auto& h = c->b.hist[profile];
  if (len_out) *len_out = (int64_t)h.size();     // min(T_p, history cap): only stored entries
  const long long k = std::min<long long>(cap, (long long)h.size());
  for (long long t = 0; t < k; ++t) out[t] = h[t];
  return PSI_OK;
}

psi_status psi_time_sweep_batch(psi_ctx* c, int64_t sweeps, double* sweep_ms) {
  g_err.clear();
  if (!c || sweeps < 1) return fail(PSI_E_INVALID_ARG, "ctx NULL or sweeps < 1");
  if (c->g.nprof < 2) return fail(PSI_E_STATE, "not a batch context (psi_build_graph_batch)");
  auto& b = c->b;
  BatchParams& hp = *b.h_prm;
  if (!b.history || b.hist_cap < sweeps) {
    if (b.history) API_CK(cudaFreeAsync(b.history, c->stream));
    b.hist_cap = std::max<long long>(sweeps, 1024);
    API_CK(dev_alloc((void**)&b.history, b.hist_cap * kBP * sizeof(double), c->stream));
  }
  hp.eps = 0.0;
  hp.max_iters = sweeps;
  hp.history = b.history;
  hp.hist_cap = b.hist_cap;
  hp.valid = (1u << kBP) - 1;
  for (int l = 0; l < kBP; ++l) hp.kappa[l] = 1.0;
  API_CK(cudaMemcpyAsync(b.prm, b.h_prm, sizeof(BatchParams), cudaMemcpyHostToDevice, c->stream));
  BatchArgs A = batch_args(c, 0, 0);
  void* kp[1] = {&A};
  int init_grid = (int)std::min<long long>((c->g.n_act + 255) / 256, 148LL * 8);
  API_CK(cudaLaunchKernel(batch_init_ptr(), dim3(init_grid < 1 ? 1 : init_grid), dim3(256), kp, 0,
                          c->stream));
  API_CK(cudaEventRecord(c->ev0, c->stream));
  for (long long t = 0; t < sweeps; ++t) {
    API_CK(cudaLaunchKernel(batch_tiles_ptr(false), dim3(b.cfg.grid1), dim3(b.cfg.block1), kp,
                            b.cfg.smem, c->stream));
    API_CK(cudaLaunchKernel(batch_fix_ptr(false), dim3(b.cfg.grid2), dim3(batch_fix_block()), kp, 0,
                            c->stream));
  }
  API_CK(cudaEventRecord(c->ev1, c->stream));
  API_CK(cudaEventSynchronize(c->ev1));
  float ms = 0;
  API_CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->have_psi = false;
  b.have = false;
  if (sweep_ms) *sweep_ms = ms / sweeps;
  return PSI_OK;
}

psi_status psi_get_pagerank(const psi_ctx* c, double* out, int mem_kind) {
  g_err.clear();
  if (!c || !out) return fail(PSI_E_INVALID_ARG, "NULL argument");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);
  if (!c->have_pr) return fail(PSI_E_STATE, "no successful psi_pagerank on this context");
  return copy_out(c, c->pr.pi, nullptr, out, mem_kind);
}

}  // extern "C"

namespace {

// Run Alg. 1 for `k` origins in batches of kNfK; psi_dev (k entries) and/or the origin-major
// p/q columns (device pointers) are filled; iters (host, k) receives each origin's T.
psi_status power_nf_run(psi_ctx* c, const int32_t* origins, long long k, double eps,
                        long long max_iters, double* psi_dev, double* p_dev, double* q_dev,
                        long long* iters, bool* all_converged, long long* sweeps_total) {
  if (!c->g.nf_loff)
    return fail(PSI_E_STATE, "Power-NF keeps the leader lists only for graphs with <= %lld edges "
                             "(N systems cost N x T x M work)", kPowerNfMaxEdges);
  const long long n = c->n;
  NfWork w;
  NfArgs a{};
  int* d_origin = nullptr;
  unsigned char* d_frozen = nullptr;
  long long* d_iters = nullptr;
  double* d_gap = nullptr;
  psi_status rc = PSI_OK;
  auto cleanup = [&]() {
    for (void* p : {(void*)w.P[0], (void*)w.P[1], (void*)w.part, (void*)w.active, (void*)d_origin,
                    (void*)d_frozen, (void*)d_iters, (void*)d_gap})
      if (p) cudaFreeAsync(p, c->stream);
    pin_free(w.h_active);
  };
#define NF_CK(call)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      rc = fail(e_ == cudaErrorMemoryAllocation ? PSI_E_OOM : PSI_E_CUDA, "%s: %s", #call, \
                cudaGetErrorString(e_));                                                   \
      cleanup();                                                                           \
      return rc;                                                                           \
    }                                                                                      \
  } while (0)
  NF_CK(dev_alloc(&w.P[0], (size_t)n * kNfK * sizeof(double), c->stream));
  NF_CK(dev_alloc(&w.P[1], (size_t)n * kNfK * sizeof(double), c->stream));
  NF_CK(dev_alloc(&w.part, power_nf_part_elems(n) * sizeof(double), c->stream));
  NF_CK(dev_alloc(&w.active, sizeof(unsigned), c->stream));
  NF_CK(pin_alloc((void**)&w.h_active, sizeof(unsigned)));
  NF_CK(dev_alloc(&d_origin, kNfK * sizeof(int), c->stream));
  NF_CK(dev_alloc(&d_frozen, kNfK, c->stream));
  NF_CK(dev_alloc(&d_iters, kNfK * sizeof(long long), c->stream));
  NF_CK(dev_alloc(&d_gap, kNfK * sizeof(double), c->stream));
  a.n = n;
  a.loff = c->g.nf_loff;
  a.leaders = c->g.nf_leaders;
  a.lm = c->g.nf_lm;
  a.wt = c->g.nf_wt;
  a.origin = d_origin;
  a.frozen = d_frozen;
  a.iters = d_iters;
  a.gap = d_gap;
  *all_converged = true;
  long long sweeps = 0;
  for (long long b0 = 0; b0 < k; b0 += kNfK) {
    const int kb = (int)std::min<long long>(kNfK, k - b0);
    int h_origin[kNfK];
    unsigned char h_frozen[kNfK];
    for (int j = 0; j < kNfK; ++j) {
      h_origin[j] = j < kb ? origins[b0 + j] : -1;
      h_frozen[j] = j < kb ? 0 : 1;
    }
    NF_CK(cudaMemcpyAsync(d_origin, h_origin, sizeof(h_origin), cudaMemcpyHostToDevice, c->stream));
    NF_CK(cudaMemcpyAsync(d_frozen, h_frozen, sizeof(h_frozen), cudaMemcpyHostToDevice, c->stream));
    int cur = 0;
    long long sw = 0;
    NF_CK(power_nf_batch(a, w, eps, max_iters, psi_dev ? psi_dev + b0 : nullptr, c->stream, &cur, &sw));
    if (p_dev || q_dev)
      NF_CK(power_nf_columns(a, w, cur, kb, p_dev ? p_dev + b0 * n : nullptr,
                             q_dev ? q_dev + b0 * n : nullptr, c->stream));
    long long h_iters[kNfK];
    double h_gap[kNfK];
    NF_CK(cudaMemcpyAsync(h_iters, d_iters, sizeof(h_iters), cudaMemcpyDeviceToHost, c->stream));
    NF_CK(cudaMemcpyAsync(h_gap, d_gap, sizeof(h_gap), cudaMemcpyDeviceToHost, c->stream));
    NF_CK(cudaStreamSynchronize(c->stream));
    for (int j = 0; j < kb; ++j) {
      if (iters) iters[b0 + j] = h_iters[j];
      sweeps += h_iters[j];
      // Alg. 1 left by the max_iters cap with gap > eps (gap_0 = 1: max_iters = 0 and
      // eps < 1 is "not converged", as psi_iterate reports it)
      if (h_iters[j] >= max_iters && h_gap[j] > eps) *all_converged = false;
    }
  }
#undef NF_CK
  cleanup();
  if (sweeps_total) *sweeps_total = sweeps;
  return PSI_OK;
}

psi_status check_nf_args(const psi_ctx* c, double eps, int64_t max_iters) {
  if (!c) return fail(PSI_E_INVALID_ARG, "ctx is NULL");
  if (!(eps >= 0.0)) return fail(PSI_E_INVALID_ARG, "eps must be >= 0 (got %g)", eps);
  if (max_iters < 0) return fail(PSI_E_INVALID_ARG, "max_iters must be >= 0");
  return PSI_OK;
}

}  // namespace

extern "C" {

psi_status psi_power_nf(psi_ctx* c, const int32_t* origins, int64_t k, double eps,
                        int64_t max_iters, double* p_out, double* q_out, int mem_kind,
                        int64_t* iters_out) {
  g_err.clear();
  psi_status st = check_nf_args(c, eps, max_iters);
  if (st != PSI_OK) return st;
  if (k < 1 || !origins) return fail(PSI_E_INVALID_ARG, "need k >= 1 origins");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);
  for (int64_t j = 0; j < k; ++j)
    if (origins[j] < 0 || origins[j] >= c->n)
      return fail(PSI_E_INVALID_ARG, "origin %d outside [0, n)", origins[j]);
  const size_t bytes = (size_t)k * c->n * sizeof(double);
  double *p_dev = p_out, *q_dev = q_out;
  if (mem_kind == PSI_MEM_HOST) {
    p_dev = q_dev = nullptr;
    if (p_out) API_CK(dev_alloc(&p_dev, bytes, c->stream));
    if (q_out && dev_alloc(&q_dev, bytes, c->stream) != cudaSuccess) {
      if (p_dev) cudaFreeAsync(p_dev, c->stream);
      return fail(PSI_E_OOM, "cudaMalloc of the q columns failed");
    }
  }
  std::vector<long long> iters(k);
  bool conv = true;
  st = power_nf_run(c, origins, k, eps, max_iters, nullptr, p_dev, q_dev, iters.data(), &conv,
                    nullptr);
  if (st == PSI_OK && mem_kind == PSI_MEM_HOST) {
    if (p_out && cudaMemcpyAsync(p_out, p_dev, bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      st = fail(PSI_E_CUDA, "copy of p failed");
    if (q_out && cudaMemcpyAsync(q_out, q_dev, bytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
      st = fail(PSI_E_CUDA, "copy of q failed");
    cudaStreamSynchronize(c->stream);
  }
  if (mem_kind == PSI_MEM_HOST) {
    if (p_dev) cudaFreeAsync(p_dev, c->stream);
    if (q_dev) cudaFreeAsync(q_dev, c->stream);
  }
  if (st != PSI_OK) return st;
  if (iters_out)
    for (int64_t j = 0; j < k; ++j) iters_out[j] = iters[j];
  if (!conv) return fail(PSI_NOT_CONVERGED, "some origin reached max_iters with gap > eps");
  return PSI_OK;
}

psi_status psi_nsystems(psi_ctx* c, double eps, int64_t max_iters, double* psi_out, int mem_kind,
                        int64_t* matvecs_out) {
  g_err.clear();
  psi_status st = check_nf_args(c, eps, max_iters);
  if (st != PSI_OK) return st;
  if (!psi_out) return fail(PSI_E_INVALID_ARG, "psi_out is NULL");
  if (mem_kind != PSI_MEM_HOST && mem_kind != PSI_MEM_DEVICE)
    return fail(PSI_E_INVALID_ARG, "bad mem_kind %d", mem_kind);
  const long long n = c->n;
  double* psi_dev = psi_out;
  if (mem_kind == PSI_MEM_HOST) API_CK(dev_alloc(&psi_dev, (size_t)n * sizeof(double), c->stream));
  std::vector<int32_t> all(n);
  for (long long i = 0; i < n; ++i) all[i] = (int32_t)i;
  bool conv = true;
  long long sweeps = 0;
  st = power_nf_run(c, all.data(), n, eps, max_iters, psi_dev, nullptr, nullptr, nullptr, &conv,
                    &sweeps);
  if (st == PSI_OK && mem_kind == PSI_MEM_HOST &&
      (cudaMemcpyAsync(psi_out, psi_dev, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream) != cudaSuccess ||
       cudaStreamSynchronize(c->stream) != cudaSuccess))
    st = fail(PSI_E_CUDA, "copy of psi failed");
  if (mem_kind == PSI_MEM_HOST) cudaFreeAsync(psi_dev, c->stream);
  if (st != PSI_OK) return st;
  if (matvecs_out) *matvecs_out = sweeps;
  if (!conv) return fail(PSI_NOT_CONVERGED, "some origin reached max_iters with gap > eps");
  return PSI_OK;
}

void psi_destroy(psi_ctx* c) { free_ctx(c); }

}  // extern "C"
