/*
 * psi.h -- C-ABI of libpsi: the Power-psi hot path (arXiv 2206.09960) on one B200.
 *
 * The library computes the psi-score of every user of a follower graph,
 *
 *     psi^T = (1/N) [ (sum_t c^T A^t) B + d^T ]                 (Eq. (12))
 *
 * by the paper's Alg. 2 "Power-psi": s_0 = c, s_t^T = s_{t-1}^T A + c^T
 * (Eq. (14)), stop when gap_t = ||B|| * ||s_t - s_{t-1}||_1 <= eps
 * (Eqs. (15)-(16) and Alg. 2), then
 * psi = (s^T B + d^T)/N (Alg. 2).  The model matrices are those of
 * P:171-175:  A[j,i] = mu_i/W_j 1{i in L(j)},  B[j,i] = lambda_i/W_j 1{i in L(j)},
 * W_j = sum_{l in L(j)} (lambda_l + mu_l),  c = mu/(lambda+mu),  d = lambda/(lambda+mu).
 * Readings of the paper where it is silent or ambiguous (the norm ||B||, leaderless
 * users, the iteration count, ...) are R1..R14 in DESIGN.md.
 *
 * Conventions
 *  - Return codes: 0 = OK, > 0 = warning with a valid result, < 0 = error
 *    (the message is in psi_last_error(), thread-local).
 *  - All device work runs on the CUDA stream given to psi_build_graph
 *    (a cudaStream_t passed as void*; NULL = the legacy default stream).
 *  - A psi_ctx is not thread-safe; separate contexts are independent.
 *  - Device memory is owned by the context and freed by psi_destroy.  All of it is
 *    stream-ordered and comes from a memory pool the LIBRARY owns (one per device,
 *    cudaMemPoolCreate) -- the device's default pool, the caller's allocator and device-wide
 *    limits are never modified.  Like PyTorch's caching allocator, the pool keeps what the
 *    library frees for its next builds (re-mapping made repeated C5 builds 3-5x slower);
 *    psi_empty_cache() returns it to the system (the analogue of torch.cuda.empty_cache()),
 *    and environment variable PSI_POOL_KEEP_GB=<x> caps what a pool keeps to x GiB.  The
 *    first build of a graph reserves about twice its pool working set (C5: ~50 GB) in one
 *    block, and a per-device build scratch (cudaMalloc, C5: ~24 GB: staged inputs, sort
 *    arrays) is kept across builds too; builds on one device serialise on that scratch.
 *  - Limits: 1 <= n <= 2^31 - 1 and m <= 2^31 - 1 (int32 indices and offsets
 *    on the device).
 */
#ifndef PSI_H
#define PSI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psi_ctx psi_ctx;
typedef int psi_status;

enum {
  PSI_OK = 0,
  PSI_NOT_CONVERGED = 1,   /* max_iters reached with gap > eps; psi is still valid */
  PSI_E_INVALID_ARG = -1,  /* bad scalar argument or NULL pointer */
  PSI_E_GRAPH = -2,        /* CSR violates the input contract (see psi_build_graph) */
  PSI_E_ACTIVITY = -3,     /* lambda/mu NaN, Inf, negative, or lambda+mu <= 0 */
  PSI_E_OOM = -4,          /* device or pinned host allocation failed */
  PSI_E_CUDA = -5,         /* any other CUDA runtime error */
  PSI_E_STATE = -6,        /* call out of order (e.g. get_psi before a successful iterate) */
  PSI_E_NUMERIC = -7       /* epsilon_t became NaN or Inf during the iteration */
};

enum { PSI_MEM_HOST = 0, PSI_MEM_DEVICE = 1 };

/* Which matrix norm ||B|| multiplies epsilon_t in Alg. 2 (the paper
 * leaves it open).  ROW (default, reading R1) = max row sum of B, the norm
 * induced by L1 on row vectors that makes bound (19) hold; COL = max column sum
 * of B (SPEC's reading); ONE = 1 (Eq. (16) without the factor). */
enum { PSI_NORM_ROW = 0, PSI_NORM_COL = 1, PSI_NORM_ONE = 2 };

typedef struct psi_info {
  int64_t n;              /* users */
  int64_t m;              /* follow edges */
  int64_t n_f;            /* users with >= 1 follower (rows whose s can change) */
  int64_t n_g;            /* users with >= 1 leader (whose s is gathered) */
  int64_t n_leaderless;   /* users with W_j = 0 (reading R5) */
  double kappa_row;       /* max row sum of B    = max_j Lambda_j / W_j        */
  double kappa_col;       /* max column sum of B = max_i lambda_i sum_{j in F(i)} 1/W_j */
  double rho_A;           /* max row sum of A    = max_j (sum_{l in L(j)} mu_l) / W_j */
  double ingest_ms;       /* device time of psi_build_graph's kernels (CUDA events) */
  double iterate_ms;      /* device time of the last psi_iterate (init + sweeps + readout) */
  int64_t last_iters;     /* T of the last psi_iterate */
  double last_gap;        /* gap_T of the last psi_iterate */
  int64_t num_tiles;      /* work tiles of one sweep (packed-row tiles + long-row chunks) */
  int64_t num_long_rows;  /* rows split across several CTAs */
  int64_t grid;           /* persistent CTAs per sweep launch */
  int64_t device_bytes;   /* device memory held by the context */
  int64_t relabeled;      /* 1 if users were relabeled for locality at ingest */
  int64_t block;          /* threads per sweep CTA (tile groups x threads per group) */
  int64_t hot_smem;       /* hottest labels of x gathered from each CTA's shared-memory copy */
  int64_t n_heavy;        /* heavy rows (labels [0, n_heavy)) served by the staged-segment kernel */
  int64_t heavy_entries;  /* (heavy row, follower < heavy_labels) pairs summed from shared memory */
  int64_t heavy_panels;   /* work panels of the staged-segment kernel */
  int64_t heavy_labels;   /* H: labels of x staged through shared memory per sweep */
  int64_t last_solver;    /* loop driver of the last psi_iterate / psi_pagerank: 0 = CUDA-graph
                             WHILE node, 1 = persistent cooperative kernel (small graphs with no
                             heavy rows), 2 = direct launches (PSI_GRAPH=0) */
  int64_t n_profiles;     /* activity profiles of the context (1, or k of psi_build_graph_batch) */
  int64_t tile_edges;     /* edges per tile of the sweep: 1024 with heavy rows, else 512 */
  int64_t overlapped;     /* 1: k_heavy and k_tiles run concurrently (the overlapped plan) */
  int64_t sliced_ell;     /* 1: the sweep runs on the sliced-ELL layout (k_sell), 0: tiles */
  int64_t sell_long_rows; /* rows summed in pieces by whole warps (stream length > lmax) */
  int64_t sell_pieces;    /* their pieces */
  int64_t sell_words;     /* index words of the slices (padding included) */
  int64_t stream_edges;   /* gathers of the edge stream per sweep: followers not summed by the
                             staged-segment kernel, + one pseudo edge per row without any */
} psi_info;

/*
 * psi_build_graph -- ingest (one-time).
 *
 * The graph is a CSR of FOLLOWERS PER LEADER ((i,j) in E means "i follows j"):
 *   row_ptr   int64[n+1]: row_ptr[0] = 0, non-decreasing, row_ptr[n] = m;
 *   followers int32[m]:   followers[row_ptr[j] .. row_ptr[j+1]) = F(j), the users
 *                         who follow j, strictly increasing, each in [0, n), j not
 *                         in F(j) (no self loops);
 *   lambda, mu double[n]: posting / re-posting rates, finite, >= 0,
 *                         lambda + mu > 0.
 * mem_kind says whether the four arrays are host (PSI_MEM_HOST; pinned memory
 * gives the fastest copy) or device (PSI_MEM_DEVICE) pointers.  They are BORROWED
 * for the duration of the call only: everything is copied or transformed into
 * context-owned device memory, so the caller may free them when it returns.
 * On the device the call validates the contract, computes W, c, d, ||B|| (all
 * three norms), rho_A, relabels users for locality, and builds the sweep's
 * work tiles.  Blocks until done.
 *
 * Errors: PSI_E_INVALID_ARG (n < 1, m < 0, n or m > 2^31-1, NULL pointer, bad
 * mem_kind); PSI_E_GRAPH (row_ptr[0] != 0, row_ptr[n] != m, decreasing row_ptr,
 * index out of range, self loop, row not strictly increasing); PSI_E_ACTIVITY;
 * PSI_E_OOM; PSI_E_CUDA.  *out is set only on PSI_OK.
 */
psi_status psi_build_graph(int64_t n, int64_t m, const int64_t* row_ptr,
                           const int32_t* followers, const double* lambda,
                           const double* mu, int mem_kind, void* stream, psi_ctx** out);

/*
 * psi_iterate -- Alg. 2 from s_0 = c, every call (no warm start).
 *
 * Runs sweeps s <- s A + c with the fused L1 residual and the stop rule
 * gap_t = ||B||_norm * epsilon_t <= eps (gap_0 = 1, Alg. 2, so eps >= 1
 * gives T = 0) entirely on the device (a CUDA-graph conditional loop, or for graphs
 * with no heavy rows and at most 8.4M edge slots one persistent cooperative kernel: no
 * host round trip per sweep; psi_info.last_solver says which), then the readout
 * psi = (s^T B + d^T)/N.  On a batch context (psi_build_graph_batch) it runs every
 * profile, see there.  Also stops
 * at T = max_iters.  eps = 0 runs exactly max_iters sweeps unless the fp
 * iteration reaches an exact fixed point first (gap_t == 0): the fixed-count
 * parity mode.  Blocks until T is known; psi is ready on return.
 *
 * Outputs (either may be NULL): *iters_out = T (number of A products; the
 * readout is one more B product), *last_gap_out = gap_T (1 if T = 0).
 * Returns PSI_OK, PSI_NOT_CONVERGED (gap_T > eps at T = max_iters; psi valid),
 * PSI_E_INVALID_ARG (NULL ctx, eps < 0 or NaN, max_iters < 0, bad norm),
 * PSI_E_NUMERIC (epsilon_t NaN/Inf), PSI_E_CUDA.
 */
psi_status psi_iterate(psi_ctx* ctx, double eps, int64_t max_iters, int norm,
                       int64_t* iters_out, double* last_gap_out);

/* psi_get_psi -- copy psi[n] (fp64, the CALLER'S ORIGINAL user labels) to `out`,
 * a host (PSI_MEM_HOST) or device (PSI_MEM_DEVICE) buffer of n doubles owned by
 * the caller (k * n, profile-major, on a batch context).  PSI_E_STATE if no
 * psi_iterate has succeeded on this context. */
psi_status psi_get_psi(const psi_ctx* ctx, double* out, int mem_kind);

/* psi_empty_cache -- return the device memory the library's pool on the CURRENT device holds
 * but no context uses (freed temporaries and destroyed contexts), and the device's build
 * scratch (the staged host inputs and the transpose's sort arrays of psi_build_graph, kept
 * across builds outside the pool), to the system; synchronises the device.  Live contexts
 * are unaffected.  PSI_E_CUDA on a CUDA error. */
psi_status psi_empty_cache(void);

/* psi_get_series -- copy s_T[n] (the paper's series iterate after the last
 * psi_iterate, Eq. (13)-(14), original labels) to a host or device buffer. */
psi_status psi_get_series(const psi_ctx* ctx, double* out, int mem_kind);

/* psi_get_residual_history -- raw epsilon_t = ||s_t - s_{t-1}||_1 for t = 1..T
 * (Eq. (15), NOT multiplied by ||B||) of the most recent psi_iterate -- or ||pi_t - pi_{t-1}||_1
 * if psi_pagerank ran last -- into host buffer `out` of capacity `cap`; *len_out = the
 * number of entries stored, min(T, 2^24) (the device keeps the first 2^24; the last iterate's
 * T is psi_get_info's last_iters); the copy is truncated to min(*len_out, cap).
 * PSI_E_STATE if neither has run. */
psi_status psi_get_residual_history(const psi_ctx* ctx, double* out, int64_t cap,
                                    int64_t* len_out);

/*
 * psi_pagerank -- the PageRank power method of PAPER.md Eq. (22) on the same
 * graph and kernels (the paper's speed baseline, Table IV):
 *     pi_0 = (1/N) 1,   pi_t^T = alpha pi_{t-1}^T W + (1 - alpha)/N 1^T,
 * W = D_out^{-1} L, the walk from a follower to its leaders: (pi^T W)_i =
 * sum_{j in F(i)} pi_j / |L(j)|; leaderless users' rows are zero (reading R5).  Stops when
 * ||pi_t - pi_{t-1}||_1 <= eps (the pi-tolerance; the first test always passes)
 * or at T = max_iters (PSI_NOT_CONVERGED, pi valid).  eps = 0 runs exactly max_iters sweeps
 * unless an exact fp fixed point is reached.  alpha in [0, 1).  Blocks until done; the
 * result is read with psi_get_pagerank.  Overwrites the iterate buffers (psi_get_series needs
 * a new psi_iterate), not psi.  Errors: PSI_E_INVALID_ARG, PSI_E_NUMERIC, PSI_E_OOM, PSI_E_CUDA.
 */
psi_status psi_pagerank(psi_ctx* ctx, double alpha, double eps, int64_t max_iters,
                        int64_t* iters_out, double* last_gap_out);

/*
 * psi_build_graph_batch -- one graph, k activity profiles ("multi-profile
 * batching": k activity profiles sharing one index stream).  Alg. 2 depends on
 * the activity only through the per-user constants c, d, W; the follower lists
 * are the graph's.  Arguments as psi_build_graph, except lambda and mu: k * n doubles each,
 * PROFILE-MAJOR (profile p's rates at lambda[p*n .. p*n+n)), every profile obeying the
 * activity contract.  psi_iterate on the returned context then runs Alg. 2 for every profile,
 * four profiles per pass over the edge stream (their x interleaved: one 32-byte gather per
 * edge for four profiles), each profile stopping on its own rule (gap_p = kappa_p eps_t^(p) <=
 * eps, kappa_p its own ||B||_row, or norm PSI_NORM_ONE; PSI_NORM_COL is rejected);
 * *iters_out = max_p T_p, *last_gap_out = max_p gap_p, PSI_NOT_CONVERGED if any profile did
 * not converge.  psi_get_psi then copies k * n doubles (profile-major, original labels).
 * The single-profile calls (psi_pagerank, psi_power_nf, psi_nsystems, psi_time_sweep) use the
 * graph and profile 0.  No staged-segment (k_heavy) path.  Errors: those of psi_build_graph;
 * PSI_E_INVALID_ARG if k < 1 or k > 4096.
 */
psi_status psi_build_graph_batch(int64_t n, int64_t m, const int64_t* row_ptr,
                                 const int32_t* followers, int64_t k, const double* lambda,
                                 const double* mu, int mem_kind, void* stream, psi_ctx** out);

/* psi_get_profile_stats -- T_p and gap_p of every profile (host arrays of k entries each,
 * either may be NULL) after psi_iterate on a batch context.  PSI_E_STATE otherwise. */
psi_status psi_get_profile_stats(const psi_ctx* ctx, int64_t* iters, double* gaps);

/* psi_get_profile_history -- raw epsilon_t^(p), t = 1..T_p, of profile p of a batch context
 * into host buffer `out` of capacity `cap`; *len_out = entries stored, min(T_p, 2^22).
 * PSI_E_STATE / PSI_E_INVALID_ARG. */
psi_status psi_get_profile_history(const psi_ctx* ctx, int64_t profile, double* out, int64_t cap,
                                   int64_t* len_out);

/* psi_time_sweep_batch -- device time of one four-profile sweep (k_tiles_b + k_fix_b, CUDA
 * events around `sweeps` direct launches on the context stream, eps = 0) of group 0, in ms.
 * Leaves the batch iterate state mid-solve (psi_get_psi needs a new psi_iterate). */
psi_status psi_time_sweep_batch(psi_ctx* ctx, int64_t sweeps, double* sweep_ms);

/* psi_get_pagerank -- copy pi[n] of the last successful psi_pagerank (original labels) to a
 * host or device buffer of n doubles.  PSI_E_STATE if psi_pagerank has not succeeded. */
psi_status psi_get_pagerank(const psi_ctx* ctx, double* out, int mem_kind);

/*
 * psi_power_nf -- Alg. 1 "Power-NF" for `k` origins:
 * per origin i (caller labels), p_i <- b_i; p_i <- A p_i + b_i until ||p_i - p_old||_1 <= eps
 * (gap_0 = 1, so eps >= 1 gives T = 0 and p_i = b_i) or T = max_iters; then the wall vector
 * q_i = C p_i + d_i (Eq. (7)).  A, b_i, C, d_i as in P:171-175 (the column
 * products: a pull over the leaders L(j)).  Runs batches of 32 origins on the GPU; each
 * origin stops on its own test, exactly as Alg. 1.
 *   origins   host int32[k], each in [0, n)
 *   p_out     NULL or k x n doubles, origin-major (p_out[c*n + j] = p_{origins[c]}^(j))
 *   q_out     NULL or k x n doubles, same layout, the wall shares q
 *   mem_kind  whether p_out / q_out are host or device buffers (caller-owned)
 *   iters_out NULL or host int64[k]: T of each origin
 * Available for graphs with <= 2^27 edges (the N systems cost N x T x M work; the leader
 * lists are kept only then), else PSI_E_STATE.  Returns PSI_OK, PSI_NOT_CONVERGED (some
 * origin hit max_iters; outputs valid), PSI_E_INVALID_ARG, PSI_E_OOM, PSI_E_CUDA.
 */
psi_status psi_power_nf(psi_ctx* ctx, const int32_t* origins, int64_t k, double eps,
                        int64_t max_iters, double* p_out, double* q_out, int mem_kind,
                        int64_t* iters_out);

/*
 * psi_nsystems -- the psi-score by its original definition: Alg. 1 for every origin i, then
 * psi_i = (1/N) sum_n q_i^(n) (Eq. (1); "applied N times") -- the paper's
 * Power-NF baseline of Tables III-IV.  psi_out: n doubles (caller labels), host or device per
 * mem_kind.  *matvecs_out (may be NULL) = sum over origins of T_i (the A-products).
 * Same limits and return codes as psi_power_nf.
 */
psi_status psi_nsystems(psi_ctx* ctx, double eps, int64_t max_iters, double* psi_out,
                        int mem_kind, int64_t* matvecs_out);

/* psi_time_sweep -- measurement entry: runs `sweeps` sweeps of Eq. (14) from s_0 = c
 * (eps = 0) as direct stream launches and returns the average device time of each of the
 * sweep's kernels, bracketed by CUDA events on the context's stream: *heavy_ms = staged
 * shared-memory sums of the heavy rows (k_heavy; 0 if the graph has no heavy rows),
 * *tiles_ms = edge-stream gather + epilogue (k_tiles), *fix_ms = split rows + eps_t
 * reduction + stop rule (k_fix).  With the overlapped plan (psi_info.overlapped = 1:
 * k_heavy and k_tiles run concurrently, one CTA of each per SM) the pair is timed as one:
 * *heavy_ms = 0 and *tiles_ms = k_heavy || k_tiles.  Any output pointer may be NULL.  Leaves
 * no psi (call psi_iterate afterwards).  PSI_E_INVALID_ARG if ctx is NULL or sweeps < 1. */
psi_status psi_time_sweep(psi_ctx* ctx, int64_t sweeps, double* heavy_ms, double* tiles_ms,
                          double* fix_ms);

/* psi_get_info -- sizes, norms and timings (see psi_info). */
psi_status psi_get_info(const psi_ctx* ctx, psi_info* out);

/* psi_destroy -- free all device and host memory of the context (NULL is a no-op). */
void psi_destroy(psi_ctx* ctx);

/* psi_last_error -- message of the last error on the calling thread ("" if none). */
const char* psi_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PSI_H */
