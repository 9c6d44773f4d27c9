// psi_sweep.cu -- the Power-psi sweep, fused L1 residual + stop rule, and readout (sm_100a).
//
// One sweep = two launches inside the CUDA-graph WHILE loop (psi_api.cu):
//
//  k_tiles   persistent merge-path gather-SpMV over the follower CSR (Merrill & Garland's
//            merge-based CsrMV).  Tile k owns merge items [k*kTile, (k+1)*kTile) of the
//            (row completions + edges) path, so every CTA does the same amount of work
//            whatever the degree distribution (power-law rows, SURVEY §7 "load balance").
//            Per tile: stage row ends + the gathered x_{t-1}[F(j)] in shared memory
//            (coalesced int32 index loads, independent 8-byte gathers in flight), merge-path
//            consume, block segmented scan of the per-thread carries, then a row-parallel
//            epilogue x_t = a + g*S, |dx|*Wt accumulated for eps_t (Eq. (15)).
//            Rows cut by a tile boundary leave partial sums ("pieces").
//  k_fix     finishes the rows cut by tile boundaries (sum of pieces in tile order), then
//            the LAST CTA to arrive reduces the per-CTA eps partials in a fixed order,
//            appends eps_t to the history, updates gap = ||B|| eps_t (Alg. 2),
//            t += 1, and sets the graph's WHILE condition (gap > eps && t < max_iters):
//            the stop rule of Eq. (16)/Alg. 2 line 320 without a host round trip.
//
// The readout (Alg. 2) is the same pair of kernels with the epilogue
// psi_j = (d_j + lambda_j S_j) / N.
//
// Determinism: no floating-point atomics anywhere; tile -> CTA assignment is static, every
// reduction has a fixed order, so two runs give bitwise identical psi and eps_t.
#include "psi_internal.cuh"

#include <climits>

namespace psi {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree); the result is returned to every thread.
template <int BLOCK>
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < BLOCK / 32 ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  return red[32];
}

struct TileSmem {
  double val[kTile];          // x_{t-1}[idx[e]] for the tile's edges
  double rowsum[kTile];       // per completed row: sum of its in-tile edges
  int rowend[kTile + 1];      // local end offset of each completed row (+ sentinel)
  double scan[kBlock];        // segmented inclusive scan of thread carries
  double wS[kBlock / 32];
  int wK[kBlock / 32];
  double red[33];
  int split_in;
};

template <bool READOUT>
__global__ void __launch_bounds__(kBlock, 4) k_tiles(SweepArgs A) {
  __shared__ TileSmem sm;
  const long long t = A.st->iter;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;    // x_{t-1}
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;          // x_t
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double eps_acc = 0.0;

  for (int k = blockIdx.x; k < A.ntiles; k += gridDim.x) {
    const int2 c0 = A.tile_coord[k];
    const int2 c1 = A.tile_coord[k + 1];
    const int r0 = c0.x, e0 = c0.y;
    const int nr = c1.x - r0;      // rows completed in this tile
    const int ne = c1.y - e0;      // edges consumed in this tile

    // ---- stage: row ends and gathered x values
    for (int i = tid; i < nr; i += kBlock) sm.rowend[i] = __ldg(A.rp + r0 + i + 1) - e0;
    if (tid == 0) {
      sm.rowend[nr] = INT_MAX;
      sm.split_in = __ldg(A.rp + r0) < e0;     // first row began in an earlier tile
    }
    {
      int j[kIpt];
#pragma unroll
      for (int u = 0; u < kIpt; ++u) {
        const int q = u * kBlock + tid;
        j[u] = q < ne ? __ldg(A.idx + e0 + q) : 0;
      }
      double v[kIpt];
#pragma unroll
      for (int u = 0; u < kIpt; ++u) {
        const int q = u * kBlock + tid;
        v[u] = q < ne ? __ldg(xs + j[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kIpt; ++u) {
        const int q = u * kBlock + tid;
        if (q < ne) sm.val[q] = v[u];
      }
    }
    __syncthreads();
    const int split_in = sm.split_in;

    // ---- merge-path consume: kIpt items per thread
    const int total = nr + ne;
    const int diag = min(tid * kIpt, total);
    const int dend = min(diag + kIpt, total);
    int lo = max(0, diag - ne), hi = min(diag, nr);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sm.rowend[mid] <= diag - mid - 1) lo = mid + 1; else hi = mid;
    }
    int i = lo, q = diag - lo;
    const int i0 = i;
    double run = 0.0;
    for (int dd = diag; dd < dend; ++dd) {
      if (q < sm.rowend[i]) { run += sm.val[q]; ++q; }
      else { sm.rowsum[i] = run; run = 0.0; ++i; }
    }

    // ---- block segmented scan of carries (key = row the thread ended in)
    const int key = i;
    double S = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double s2 = __shfl_up_sync(kFull, S, o);
      const int k2 = __shfl_up_sync(kFull, key, o);
      if (lane >= o && k2 == key) S += s2;
    }
    if (lane == 31) { sm.wS[warp] = S; sm.wK[warp] = key; }
    __syncthreads();
    for (int w2 = warp - 1; w2 >= 0 && sm.wK[w2] == key; --w2) S += sm.wS[w2];
    sm.scan[tid] = S;
    __syncthreads();
    if (i > i0 && tid > 0) sm.rowsum[i0] += sm.scan[tid - 1];   // carry into first completed row
    __syncthreads();

    // ---- pieces of rows cut by tile boundaries (finished in k_fix)
    if (tid == 0) {
      const double tail = sm.scan[kBlock - 1];
      if (nr == 0) { A.piece_first[k] = tail; A.piece_last[k] = 0.0; }
      else { A.piece_first[k] = sm.rowsum[0]; A.piece_last[k] = tail; }
    }

    // ---- epilogue over the rows completed in this tile (coalesced)
    for (int ii = tid; ii < nr; ii += kBlock) {
      if (ii == 0 && split_in) continue;
      const int r = r0 + ii;
      const double Sr = sm.rowsum[ii];
      if (READOUT) {
        A.psi[r] = (__ldg(A.d + r) + __ldg(A.lam + r) * Sr) / A.n_users;
      } else {
        const double xn = fma(__ldg(A.g + r), Sr, __ldg(A.a + r));
        eps_acc += __ldg(A.wt + r) * fabs(xn - xs[r]);
        xd[r] = xn;
      }
    }
  }

  if (!READOUT) {
    const double tot = block_sum<kBlock>(eps_acc, sm.red);
    if (tid == 0) A.eps_part1[blockIdx.x] = tot;
  }
}

template <bool READOUT>
__global__ void __launch_bounds__(kFixBlock) k_fix(SweepArgs A) {
  __shared__ double red[33];
  __shared__ int last;
  const long long t = A.st->iter;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;
  const int tid = threadIdx.x;
  double eps_acc = 0.0;

  for (int s = blockIdx.x * kFixBlock + tid; s < A.nsplit; s += gridDim.x * kFixBlock) {
    const int4 sp = A.split[s];
    const int r = sp.x;
    double S = 0.0;
    for (int k = sp.y; k <= sp.z; ++k)
      S += (A.tile_coord[k].x == r) ? A.piece_first[k] : A.piece_last[k];
    if (READOUT) {
      A.psi[r] = (A.d[r] + A.lam[r] * S) / A.n_users;
    } else {
      const double xn = fma(A.g[r], S, A.a[r]);
      eps_acc += A.wt[r] * fabs(xn - xs[r]);
      xd[r] = xn;
    }
  }
  if (READOUT) return;

  const double tot = block_sum<kFixBlock>(eps_acc, red);
  if (tid == 0) {
    A.eps_part2[blockIdx.x] = tot;
    __threadfence();
    const unsigned prev = atomicAdd(&A.st->done, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();

  // Final, fixed-order reduction of eps_t and the loop control of Alg. 2.
  double v = 0.0;
  for (int q = tid; q < A.grid1; q += kFixBlock) v += __ldcg(A.eps_part1 + q);
  const double e1 = block_sum<kFixBlock>(v, red);
  v = 0.0;
  for (int q = tid; q < (int)gridDim.x; q += kFixBlock) v += __ldcg(A.eps_part2 + q);
  const double e2 = block_sum<kFixBlock>(v, red);
  if (tid == 0) {
    const double eps_t = e1 + e2;
    const LoopParams P = *A.prm;
    if (t < P.hist_cap) P.history[t] = eps_t;
    const double gap = P.kappa * eps_t;
    const bool bad = !isfinite(eps_t);
    A.st->eps_t = eps_t;
    A.st->gap = gap;
    A.st->iter = t + 1;
    A.st->done = 0;
    if (bad) A.st->status |= 1;
    const unsigned cont = (!bad && gap > P.eps && t + 1 < P.max_iters) ? 1u : 0u;
    if (A.use_cond) cudaGraphSetConditional(A.cond, cont);
  }
}

// x_0 = a (s_0 = c, Alg. 2 line 1), t = 0, gap = 1 (line 4), WHILE condition = (1 > eps).
// Only active users are reset: follower-less users hold x = a0 in both buffers forever.
__global__ void k_init(SweepArgs A, int n) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_act; i += stride) A.x0[i] = A.a0[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.st->iter = 0;
    A.st->gap = 1.0;
    A.st->eps_t = 0.0;
    A.st->done = 0;
    A.st->status = 0;
    const LoopParams P = *A.prm;
    if (A.use_cond) cudaGraphSetConditional(A.cond, (1.0 > P.eps && P.max_iters > 0) ? 1u : 0u);
  }
}

}  // namespace

int sweep_grid(int ntiles) {
  static int occ = -1, sms = 0;
  if (occ < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiles<false>, kBlock, 0);
    if (occ < 1) occ = 1;
  }
  long long g = (long long)sms * occ;
  if (g > ntiles) g = ntiles;
  return g < 1 ? 1 : (int)g;
}

int fix_grid(int nsplit) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long g = ((long long)nsplit + kFixBlock - 1) / kFixBlock;
  if (g > (long long)sms * 4) g = (long long)sms * 4;
  return g < 1 ? 1 : (int)g;
}

void* sweep_kernel_ptr(bool readout) {
  return readout ? (void*)k_tiles<true> : (void*)k_tiles<false>;
}
void* fix_kernel_ptr(bool readout) {
  return readout ? (void*)k_fix<true> : (void*)k_fix<false>;
}
void* init_kernel_ptr() { return (void*)k_init; }
size_t sweep_smem_bytes() { return sizeof(TileSmem); }

}  // namespace psi
