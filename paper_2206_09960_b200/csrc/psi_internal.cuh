// psi_internal.cuh -- device data layout and kernel interfaces of libpsi (sm_100a).
//
// Kernel state (SURVEY §8 conventions):
//   x_t = s_t / Wt,  Wt_j = W_j if W_j > 0 else 1                (s_t: Eq. (14))
//   x_0 = a,  x_t,j = a_j + g_j * S_j(x_{t-1}),  S_j(x) = sum_{n in F(j)} x_n
//   a = c / Wt,  g = mu / Wt
//   eps_t = sum_j Wt_j |x_t,j - x_{t-1},j| = ||s_t - s_{t-1}||_1  (Eq. (15))
//   psi_j = (d_j + lambda_j * S_j(x_T)) / N                      (Alg. 2)
// This is the rank-1 factorisation A = P diag(c), B = P diag(d) with
// P[n,j] = w_j / W_n 1{j in L(n)}: (s^T A)_j = mu_j sum_{n in F(j)} s_n / W_n,
// so one gathered vector x serves A and B and no per-edge value is stored.
//
// Edge stream: the follower lists of the active rows [0, n_act), in
// row order, as uint32 words: bits 0..30 = follower label, bit 31 = "first edge of a row".
// Every active row has >= 1 word (a row whose followers were all folded away gets one
// pseudo edge to the sentinel label n, whose x is 0), so row r is simply the r-th flag:
// no row_ptr is read by the sweep.  The stream is padded to a multiple of the tile size
// (IngestOut::tile) with unflagged sentinel words.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

// PSI_CHECKS builds (lib/libpsi_checked.so, PSI_LIB=checked) add device-side bounds checks
// that trap on a violation; compute-sanitizer is not available on the GPU pool.
#ifdef PSI_CHECKS
#include <cstdio>
#define PSI_ASSERT(c)                                                                    \
  do {                                                                                   \
    if (!(c)) {                                                                          \
      printf("PSI_CHECKS: %s failed (%s:%d)\n", #c, __FILE__, __LINE__);                \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define PSI_ASSERT(c) \
  do {                \
  } while (0)
#endif

namespace psi {

constexpr int kBlock = 128;              // threads per tile group of the sweep kernel (1024-edge tiles)
constexpr int kEpt = 8;                  // edges per thread
constexpr int kTile = kBlock * kEpt;     // 1024 edges per tile (512 for graphs without heavy rows)
constexpr int kFixBlock = 256;           // threads per CTA of the split-row fix-up kernel
constexpr int kLongSpan = 16;            // split rows over more tiles are summed by a warp
constexpr unsigned kRowFlag = 0x80000000u;
// staged-segment heavy-row kernel (psi_heavy.cu).  Two plan shapes: the serial sweep (k_heavy
// then k_tiles, one SM each in turn) and the overlapped one (PSI_OVERLAP: k_heavy and k_tiles
// co-resident on every SM, so each gets a smaller share of shared memory and registers).
constexpr int kSegShift = 13;
constexpr int kSeg = 1 << kSegShift;     // labels of x per TMA-staged segment (64 KB), serial plan
constexpr int kHeavySlots = 8192;        // slot sums per panel (+ a junk slot for padding)
constexpr int kEntBits = 27;             // entry word: slot (<= 14 bits) << seg_shift | offset
constexpr unsigned kNullEntry = (unsigned)kHeavySlots << kSegShift;
constexpr int kHeavyWarps = 16;          // consumer warps (+ 1 producer warp)
constexpr int kOvlSegShift = 12;         // overlapped plan: 4096-label (32 KB) segments,
constexpr int kOvlSlots = 4096;          //   4096 slots per panel,
constexpr int kOvlWarps = 8;             //   8 consumer warps
constexpr int kHeavyStages = 2;          // TMA ring depth (per-segment cost is fixed)
constexpr int kHeavyBlock = 32 * (kHeavyWarps + 1);
constexpr int kDefaultHeavyMin = 64;     // rows with >= this many active followers are heavy
constexpr long long kDefaultHeavyMinN = 1LL << 24;   // graphs below this many users skip it
constexpr int kMaxHeavySegs = 512;       // shared-memory bound of the per-warp list offsets
// staged labels H: N/32 rounded down to a power of two, within [2^19, 2^20] (C4: 512 Ki,
// C5: 1 Mi; measured); PSI_HEAVY_LABELS overrides
constexpr int kMinHeavyLabels = 1 << 19, kMaxHeavyLabels = 1 << 20;
constexpr int kDefaultHeavyPPS = 1;      // heavy panels per SM (entry budget per panel)
constexpr int kDefaultGroups = 8;        // tile groups (of kBlock threads) per sweep CTA
constexpr long long kCoopEdges = 1LL << 23;  // k_solve up to this many edge slots (PSI_COOP_TILES: tiles)
constexpr int kDefaultSmemHot = 4096;    // labels of x_{t-1} cached in shared memory per CTA
constexpr int kSmemHotLarge512 = 12288;  // 512-edge tiles on graphs with >= 2^22 users (C3)
constexpr int kDefaultL1Hot = 16384;     // labels below this gather through L1 (evict_last)
// sliced-ELL sweep (k_sell, SellPlan)
constexpr int kSellWarps = 32;           // warps per k_sell CTA (one CTA per SM)
constexpr int kSellShift = 8;            // rows per window <= 256 (sort scope and smem sums)
constexpr int kSellKcap = 256;           // window cut after ~256 x 32 stream edges
constexpr double kSellMaxPad = 1.6;       // graphs without heavy rows: k_sell if its index words
                                         // are <= 1.6 x the stream's (C2 1.45: k_sell; C3 2.4: tiles)
constexpr int kSellLmax = 1024;          // longer stream rows are summed in pieces by warps
constexpr int kSellPiece = 4096;         // followers per piece of a long row

// Device memory: every allocation of the library is stream-ordered and comes from a memory
// pool the library owns (one per device, psi_api.cu) -- never the device's default pool, so
// the caller's allocator (e.g. PyTorch's) is unaffected.  Memory the library frees returns to
// the system when the last context on the device is destroyed (PSI_POOL_KEEP_GB keeps that
// much reserved for later builds).
cudaMemPool_t lib_pool();
template <class T>
inline cudaError_t dev_alloc(T** p, size_t bytes, cudaStream_t s) {
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, lib_pool(), s);
}

// Device-resident loop state (written by kernels, read back by the host once per iterate).
struct LoopState {
  long long iter;        // completed sweeps t
  double gap;            // ||B|| * eps_t  (1 before the first sweep, Alg. 2)
  double eps_t;          // last epsilon_t
  unsigned int done;     // CTA arrival counter of the fix-up kernel
  int status;            // bit 0: non-finite epsilon_t
  unsigned heavy_next;   // next panel of k_heavy to claim (reset by k_fix / k_init)
  unsigned sell_next;    // next work item of k_sell to claim (reset by k_fix / k_init)
};

// Per-call parameters (host writes them before every graph launch).
struct LoopParams {
  double eps;            // s-tolerance
  long long max_iters;
  double kappa;          // ||B|| for the selected norm
  double* history;       // epsilon_t, t = 1..T
  long long hist_cap;
  double gap0;           // gap before the first sweep: 1 (Alg. 2 line 4) or +inf (PageRank)
  double eps1_extra;     // added to eps_1: PageRank's follower-less users move 1/N -> (1-alpha)/N
};

// Device view of the heavy-row plan (built at ingest, psi_ingest.cu).
struct HeavyPlan {
  const unsigned* ent;       // entry words, lists (panel, segment, warp), 32-byte aligned
  const long long* loff;     // [npanels * kHeavyWarps * nseg + 1] starts of lists (p, warp, s)
  const int* prow;           // [npanels + 1] heavy rows of panel p: [prow[p], prow[p+1])
  const int2* rslot;         // [n_heavy] (first slot, number of slots) of each heavy row
  const int* wslot;          // [npanels * (kHeavyWarps + 1)] slot range of each warp
  int npanels;
  int nseg;                  // staged labels H = nseg << seg_shift
  int seg_shift;             // labels per segment = 1 << seg_shift
  int slots;                 // slot sums per panel; slot index `slots` is the padding junk
};

// Device view of the sliced-ELL layout of the edge stream (built by psi_ingest.cu, swept by
// k_sell in psi_sweep.cu).  Active rows are cut into windows of whole 32-row
// blocks (at most 2^shift rows, and about kcap * 32 stream edges, so every window is a bounded
// work item); inside a window the rows are sorted by stream length (descending) and dealt out
// 32 at a time to slices: lane l of slice s owns one row.  A lane streams the whole window in
// one loop of K = sum of its slices' widths steps (step k = follower k - start of the slice
// containing k of its row in that slice; a shorter row's tail holds the sentinel label n,
// x[n] = 0), step k at words[(wstep[w] + (k / 8) * 8) * 32 + l * 8 + k % 8]: one 32-byte load
// per lane and 8 steps, 1 KB contiguous per warp.  Rows longer than lmax ("long rows")
// are not in the slices: they are cut into pieces of at most `piece` followers, each summed by
// one warp of k_sell (lwords -> ppart), and finished by k_fix (piece sums in piece order).
struct SellPlan {
  const unsigned* words;      // slice-major; inside a slice j-major: [j][32 lanes]
  const unsigned* soff;       // [nslices + 1] first step of slice s (= rows 32s..) if the
                              // windows were unpadded: slice ends inside a window
  const unsigned* wstep;      // [nwin + 1] first step of window w's index block (multiple of 8)
  const unsigned short* ipos; // [n_act pad 32] position of row r in its window's sorted order
                              // (0xffff: a long row)
  const int* wrow;            // [nwin + 1] first row of window w (a multiple of 32)
  int nwin;
  int wmax;                   // rows per window at most (= 2^shift: the warp's smem sums)
  const int* lrow;            // [nlong] long rows (ascending)
  const int* lp0;             // [nlong + 1] pieces of long row i: lp0[i] .. lp0[i + 1]
  const int2* piece;          // [npieces] (first word in lwords, length)
  const unsigned* lwords;     // long rows' follower labels, row after row
  int npieces;
  int nlong;
  double* ppart;              // [npieces] piece sums of the current launch
  double* epsw;               // [nwin] eps_t partial of every window
  long long nwords, nlwords;  // sizes (PSI_CHECKS bounds)
};

// Everything one sweep / readout launch needs (passed by value; frozen in the graph).
struct SweepArgs {
  const unsigned* edges;     // flagged edge stream [ntiles * tile]
  const int* tile_row;       // tile_row[k] = number of row flags before edge k*tile (k <= ntiles)
  int ntiles;
  const int4* split;         // rows spanning tiles: {row, first tile, last tile, 0}; the
  int nsplit;                // first nsplit_long span more than kLongSpan tiles (warp each)
  int nsplit_long;
  double* p_in;              // per tile: partial of the row open at the tile's start
  double* p_out;             // per tile: partial of the last row started in it, if it continues
  const double* a0;          // x_0 (init)                       [n_act]
  const double* a;           // sweep constant a + g K           [n_act]
  const double* a_first;     // constant of the first sweep if different (PageRank), else NULL
  const double* g;           //                                  [n_act]
  const double* wt;          // Wt                               [n]
  const double* d;           // readout constant d + lambda K    [n_act]
  const double* lam;         //                                  [n_act]
  double n_users;            // N of psi = (...)/N
  int n_lab;                 // labels 0..n_lab of x (n_lab = n: the zero sentinel; PSI_CHECKS)
  int n_act;
  int hot_lim;               // labels < hot_lim: L2 evict_last for x gathers/stores
  int hot_smem;              // labels < hot_smem: gathered from the CTA's shared-memory copy
  int l1_lim;                // labels in [hot_smem, l1_lim): L1-allocating gathers
  int st_last;               // 1: x_t stores below hot_lim are L2 evict_last (else evict_first)
  int single_lo;             // labels >= single_lo: single-leader users, L1 evict_first gathers
  double* psi;               // readout output (relabelled order)
  int n_heavy;               // rows [0, n_heavy) add hhot (their followers < H) to S
  double* hhot;              // [n_heavy] written by k_heavy before k_tiles
  HeavyPlan heavy;
  double* x0;                // ping-pong iterate buffers [n + 1], x[n] = 0 (sentinel)
  double* x1;
  double* eps_part1;         // per CTA of the tile kernel
  double* eps_part2;         // per CTA of the fix-up kernel
  int grid1;
  LoopState* st;
  const LoopParams* prm;
  cudaGraphConditionalHandle cond;
  int use_cond;              // 1 inside the CUDA graph; 0 for direct stream launches
  // overlapped sweep (PSI_OVERLAP): k_heavy runs concurrently with k_tiles, so k_tiles leaves
  // heavy rows' edge-stream sums in scold and k_fix finishes them with hhot
  int ovl;
  double* scold;             // [n_heavy]
  const unsigned* hsplit;    // [n_heavy / 32 + 1] bit r: heavy row r is a split row (k_fix's)
  // sliced-ELL sweep (k_sell) instead of the edge-balanced tiles (k_tiles)
  int use_sell;
  SellPlan sell;
  // 1: no long rows and no heavy rows -- k_sell's last CTA reduces eps_t and runs the loop
  // control itself, and no k_fix is launched (psi_sweep.cu sell_finish)
  int sell_fused;
};

// ---- launchers (psi_sweep.cu)
struct TilesCfg {                    // launch shape of k_tiles (sweep and readout)
  void* sweep;
  void* readout;
  int groups, grid, block;
  size_t smem;                       // dynamic: groups x TileSmem + hot cache
  int hot_smem, l1_lim;
  void* solve;                       // k_solve<groups>: the persistent small-graph solver
  int solve_max_grid;                // co-resident CTAs of k_solve (cooperative launch bound)
};
TilesCfg tiles_config(int ntiles, long long n, int tile, bool ovl = false);  // tile: 512 or 1024
TilesCfg sell_config(long long n, int shift);  // k_sell (sweep + readout); no persistent solver
int fix_grid(int nsplit);            // CTAs of the fix-up kernel
void* fix_kernel_ptr(bool readout);
void* heavy_kernel_ptr(int warps);   // psi_heavy.cu: kHeavyWarps or kOvlWarps consumer warps
size_t heavy_smem_bytes(int nseg, int seg_shift, int slots, int warps);
void* init_kernel_ptr();

// ---- ingest (psi_ingest.cu)
// Device arrays in the NEW (relabelled) user order; active users [0, n_act) have >= 1
// follower, follower-less users [n_act, n) never change (x = a0, psi = d/N).
struct IngestOut {
  unsigned* edges = nullptr;  // [ntiles*tile] flagged edge stream (see above)
  int* tile_row = nullptr;    // [ntiles+1]
  double* a0 = nullptr;       // [n]     x_0 = c / Wt
  double* a1 = nullptr;       // [n_act] sweep constant a + g K (K: folded follower-less terms)
  double* g = nullptr;        // [n_act] mu / Wt
  double* wt = nullptr;       // [n]     Wt (s = Wt x)
  double* d1 = nullptr;       // [n_act] readout constant d + lambda K
  double* lam = nullptr;      // [n_act]
  double* psi = nullptr;      // [n]     readout buffer; [n_act, n) prefilled with d/N
  int* old_of_new = nullptr;  // [n]
  int* nlead = nullptr;       // [n]     #leaders |L(j)| (PageRank out-degree), new labels
  double* kinv = nullptr;     // [n_act] sum over follower-less followers n of 1/max(|L(n)|, 1)
  double* kw = nullptr;       // [n_act] sum over follower-less followers n of 1/Wt_n (||B||_col;
                              //         freed once the column pass has run)
  // Power-NF (caller labels; kept when m <= kPowerNfMaxEdges, else nf_loff == nullptr)
  int* nf_loff = nullptr;
  int* nf_leaders = nullptr;
  double* nf_wt = nullptr;
  double2* nf_lm = nullptr;
  int ntiles = 0;
  int tile = kTile;           // edges per tile of the single-profile sweep (512 or kTile = 1024)
  int4* split = nullptr;      // [nsplit] rows spanning tiles, the nsplit_long long ones first
  int nsplit = 0;
  int nsplit_long = 0;
  long long n_act = 0, m_act = 0, n_hot = 0, n_pseudo = 0;
  long long single_lo = 0;    // first label of the single-leader users (gathered once, in order)
  // heavy rows (labels [0, n_heavy)): followers < H served by k_heavy (HeavyPlan)
  long long n_heavy = 0, heavy_entries = 0;
  int nseg = 0, npanels = 0;
  int heavy_seg_shift = kSegShift, heavy_slots = kHeavySlots, heavy_warps = kHeavyWarps;
  int ovl = 0;                // overlapped plan (PSI_OVERLAP)
  unsigned* hsplit = nullptr; // [n_heavy / 32 + 1] heavy rows that are split rows (ovl only)
  unsigned* h_ent = nullptr;
  long long* h_loff = nullptr;
  int* h_prow = nullptr;
  int2* h_rslot = nullptr;
  int* h_wslot = nullptr;
  int relabel_levels = 0;
  // sliced-ELL layout (SellPlan; sell = 0: the sweep runs on the tiles); PSI_SELL_SHIFT /
  // _LMAX / _PIECE override the window, long-row and piece sizes (tests and tuning)
  int sell = 0, sell_shift = 0, sell_lmax = 0, sell_piece = kSellPiece, sell_kcap = kSellKcap;
  int sell_nwin = 0, sell_nlong = 0, sell_npieces = 0;
  long long sell_nslices = 0, sell_words = 0, sell_lwords = 0;
  unsigned* s_words = nullptr;
  unsigned* s_off = nullptr;
  unsigned short* s_ipos = nullptr;
  int* s_wrow = nullptr;
  unsigned* s_wstep = nullptr;
  int* s_lrow = nullptr;
  int* s_lp0 = nullptr;
  int2* s_piece = nullptr;
  unsigned* s_lwords = nullptr;
  double kappa_row = 0, kappa_col = 0, rho_A = 0;
  long long n_f = 0, n_g = 0, n_leaderless = 0;
  int relabeled = 0;
  // multi-profile batch (psi_build_graph_batch): nprof activity profiles on one graph, in
  // groups of kBP interleaved per user ([group][user][kBP]; unused lanes of the last group 0)
  int nprof = 1, ngroups = 0;
  int b_ntiles = 0;           // the batch sweep's tiling: kTileB-edge tiles of the same stream
  int* b_tile_row = nullptr;  // [b_ntiles + 1]
  int4* b_split = nullptr;    // [b_nsplit], the b_nsplit_long long ones first
  int b_nsplit = 0, b_nsplit_long = 0;
  double* b_a0 = nullptr;     // [ngroups][n][kBP]     x_0
  double* b_a1 = nullptr;     // [ngroups][n_act][kBP] sweep constant a + g K
  double* b_g = nullptr;      // [ngroups][n_act][kBP]
  double* b_wt = nullptr;     // [ngroups][n_act][kBP] Wt (residual weights)
  double* b_d1 = nullptr;     // [ngroups][n_act][kBP] readout constant d + lambda K
  double* b_lam = nullptr;    // [ngroups][n_act][kBP]
  double* b_psi = nullptr;    // [ngroups][n][kBP]     readout; [n_act, n) prefilled with d/N
  std::vector<double> b_kappa_row;  // [nprof] ||B||_row of every profile
};

// ---- Power-NF (psi_powernf.cu): Alg. 1 for a batch of kNfK origins, caller labels
constexpr int kNfK = 32;                         // origins per batch (one lane each)
constexpr long long kPowerNfMaxEdges = 1LL << 27;  // graphs up to this size keep L(j) for it
struct NfArgs {
  long long n;
  const int* loff;       // [n+1] leaders of user j: leaders[loff[j] .. loff[j+1])
  const int* leaders;    // [m]   ascending per user
  const double2* lm;     // [n]   (lambda, mu)
  const double* wt;      // [n]   Wt = W, or 1 if leaderless
  const int* origin;     // [kNfK] origin of each column, -1 = unused
  unsigned char* frozen; // [kNfK] column stopped (Alg. 1 loop left)
  long long* iters;      // [kNfK] T of each column
  double* gap;           // [kNfK] last ||p - p_old||_1
};
struct NfWork {
  double* P[2] = {nullptr, nullptr};  // [n * kNfK] row-major ping-pong
  double* part = nullptr;             // per-CTA column partials
  unsigned* active = nullptr;         // device: columns still iterating
  unsigned* h_active = nullptr;       // pinned host copy
};
cudaError_t power_nf_batch(const NfArgs& a, NfWork& w, double eps, long long max_iters,
                           double* psi_dev, cudaStream_t s, int* cur_out, long long* sweeps);
cudaError_t power_nf_columns(const NfArgs& a, const NfWork& w, int cur, int k, double* p_out,
                             double* q_out, cudaStream_t s);
size_t power_nf_part_elems(long long n);

// ---- PageRank (psi_pagerank.cu): constants of Eq. (22) in the sweep's kernel state
struct PrBuffers {
  double* a = nullptr;        // [n_act] sweep constant (t >= 2)
  double* a_first = nullptr;  // [n_act] sweep constant of the first sweep
  double* g = nullptr;        // [n_act] alpha / Dt
  double* dt = nullptr;       // [n]     Dt = max(|L(j)|, 1): pi = Dt x
  double* x0 = nullptr;       // [n]     x_0 = 1 / (N Dt)
  double* pi = nullptr;       // [n]     result, relabelled order
};
cudaError_t pagerank_prep(const IngestOut& G, long long n, double alpha, const PrBuffers& B,
                          cudaStream_t s);
cudaError_t pagerank_readout(const IngestOut& G, long long n, double alpha, const double* xT,
                             long long T, const PrBuffers& B, cudaStream_t s);

// Build scratch (psi_ingest.cu): two per-device buffers kept across builds outside the pool --
// slot 0 the staged host inputs, slot 1 the transpose's sort arrays.  A build holds
// *scratch_mutex(dev) from staging until ingest returns; psi_empty_cache frees them.
std::mutex* scratch_mutex(int dev);
cudaError_t scratch_get(int dev, int slot, size_t bytes, void** out);
void scratch_release(int dev);

// Returns 0 or a negative psi_status; msg gets a description on error.  nprof > 1: lam_dev /
// mu_dev hold nprof profiles (profile-major, nprof * n); the single-profile outputs are those
// of profile 0, the b_* arrays those of all profiles, and the heavy-row path is off.
int ingest(long long n, long long m, const long long* rp64_dev, const int* idx_dev,
           const double* lam_dev, const double* mu_dev, int nprof, cudaStream_t s,
           IngestOut& out, char* msg, size_t msg_len, cudaEvent_t act_ready = nullptr);

// ---- multi-profile batch sweep (psi_batch.cu): kBP profiles per pass over the edge stream
constexpr int kBP = 4;                   // profiles per group (one 32-byte x gather per edge)
constexpr int kTileB = 512;              // edges per tile of the batch sweep (its own tiling)
struct __align__(32) d4 { double v[kBP]; };

struct LoopStateB {
  long long iter;            // sweeps of this group
  unsigned active;           // bit p: profile p still iterating
  unsigned done;             // CTA arrival counter of k_fix_b
  int status;                // bit p: non-finite eps_t of profile p
  int pad;
  double gap[kBP];
  double eps_t[kBP];
  long long T[kBP];          // T of every profile (its own stop, Alg. 2 per profile)
};
struct BatchParams {
  double eps;
  long long max_iters;
  double kappa[kBP];
  double* history;           // [hist_cap][kBP]
  long long hist_cap;
  unsigned valid;            // profiles of this group that exist
};
struct BatchArgs {
  const unsigned* edges;
  const int* tile_row;
  int ntiles;
  const int4* split;
  int nsplit;
  int nsplit_long;
  d4* p_in;                  // [ntiles + 1]
  d4* p_out;
  const d4* a0;              // [n]
  const d4* a;               // [n_act]
  const d4* g;
  const d4* wt;
  const d4* d;
  const d4* lam;
  d4* psi;                   // [n]
  d4* x0;                    // [n + 1] ping-pong, x[n] = 0
  d4* x1;
  d4* eps_part1;             // [grid1]
  d4* eps_part2;             // [grid2]
  double n_users;
  int n_act;
  int hot_smem;
  int hot_lim;
  int grid1;
  LoopStateB* st;
  const BatchParams* prm;
  cudaGraphConditionalHandle cond;
  int use_cond;
};
struct BatchCfg {
  int grid1, block1, grid2;
  size_t smem;
  int hot_smem;
};
BatchCfg batch_config(int ntiles, long long n, int nsplit);
void* batch_tiles_ptr(bool readout);
void* batch_fix_ptr(bool readout);
void* batch_init_ptr();
int batch_fix_block();
cudaError_t batch_unpermute(const double* psi_groups, const int* old_of_new, long long n, int nprof,
                            double* out, cudaStream_t s);

}  // namespace psi
