// psi_powernf.cu -- Alg. 1 "Power-NF" batched over origins (sm_100a).
//
// the N-systems baseline of Tables III-IV and the per-origin by-products
// p_i, q_i that Power-psi gives up.  For a batch of K = 32 origins i_c the
// newsfeed vectors are the K columns of P (row-major, N x K, one 256-byte row per user):
//
//     P <- B_I ;   P <- A P + B_I  until ||P[:, c] - P_old[:, c]||_1 <= eps   (per column)
//     (A P)[j, c] = (1/W_j) sum_{l in L(j)} mu_l P[l, c],   B_I[j, c] = lambda_{i_c}/W_j 1{i_c in L(j)}
//
// -- the *column* product, a pull over the leaders L(j) (the transpose of the psi sweep's
// follower lists), kept from the ingest for graphs up to kPowerNfMaxEdges edges.  A warp per
// user j, lane c = column c: every leader row P[l, :] is one coalesced 256-byte read.
// Columns freeze individually when their own stop test passes (Alg. 1 per origin, exactly),
// so T_c is each origin's own iteration count.  Then q_i = C p_i + d_i (Eq. (7)) and
// psi_i = (1/N) sum_n q_i^(n) (Eq. (1)).  All reductions in a fixed order (deterministic).
#include "psi_internal.cuh"

namespace psi {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNfBlock = 256;              // 8 warps: 8 users per CTA pass

// One Power-NF step for the K columns (init: P_old treated as 0 -> P = B_I, Alg. 1 line 1).
// Per-CTA column partials of |P - P_old| in part[blockIdx][c].
__global__ void __launch_bounds__(kNfBlock) k_nf_step(NfArgs a, const double* __restrict__ Pold,
                                                      double* __restrict__ Pnew, int init,
                                                      double* part) {
  __shared__ double red[kNfBlock / 32][kNfK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int origin = a.origin[lane];
  const bool frozen = a.frozen[lane] != 0;
  double gsum = 0.0;
  for (long long j = blockIdx.x * (long long)(kNfBlock / 32) + warp; j < a.n;
       j += (long long)gridDim.x * (kNfBlock / 32)) {
    const int b = a.loff[j], e = a.loff[j + 1];
    double acc = 0.0;
    for (int q = b; q < e; ++q) {
      const int l = a.leaders[q];
      PSI_ASSERT(l >= 0 && l < a.n);
      const double2 lm = a.lm[l];
      if (!init) acc = fma(lm.y, Pold[(size_t)l * kNfK + lane], acc);
      if (l == origin) acc += lm.x;
    }
    const double old = init ? 0.0 : Pold[(size_t)j * kNfK + lane];
    const double y = frozen ? old : acc / a.wt[j];      // leaderless: acc = 0 -> y = 0
    Pnew[(size_t)j * kNfK + lane] = y;
    gsum += fabs(y - old);
  }
  red[warp][lane] = gsum;
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
    for (int w = 0; w < kNfBlock / 32; ++w) s += red[w][lane];
    part[(size_t)blockIdx.x * kNfK + lane] = s;
  }
}

// Column gaps in a fixed order; Alg. 1 lines 4 and 7-8 per column; active-column count.
__global__ void k_nf_finish(NfArgs a, const double* part, int nblocks, int init, double eps,
                            long long max_iters, unsigned* active) {
  const int c = threadIdx.x;                            // one warp, lane = column
  double gap = 0.0;
  for (int k = 0; k < nblocks; ++k) gap += part[(size_t)k * kNfK + c];
  bool fr = a.frozen[c] != 0;
  if (init) {
    a.iters[c] = 0;
    a.gap[c] = 1.0;                                     // gap_0 = 1 (Alg. 1 line 3)
    fr = fr || !(1.0 > eps && max_iters > 0);
  } else if (!fr) {
    a.iters[c] += 1;
    a.gap[c] = gap;
    if (!(gap > eps) || a.iters[c] >= max_iters) fr = true;
  }
  a.frozen[c] = fr ? 1 : 0;
  const unsigned n_act = __popc(__ballot_sync(kFull, !fr));
  if (c == 0) *active = n_act;
}

// q_i = C p_i + d_i e_i (Eq. (7)); psi_i = (1/N) sum_n q_i^(n) (Eq. (1)) -- per-CTA partials
__global__ void __launch_bounds__(kNfBlock) k_nf_wall(NfArgs a, const double* __restrict__ P,
                                                      double* part) {
  __shared__ double red[kNfBlock / 32][kNfK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0.0;
  for (long long j = blockIdx.x * (long long)(kNfBlock / 32) + warp; j < a.n;
       j += (long long)gridDim.x * (kNfBlock / 32)) {
    const double2 lm = a.lm[j];
    s += lm.y / (lm.x + lm.y) * P[(size_t)j * kNfK + lane];   // c_n p_i^(n)
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int w = 0; w < kNfBlock / 32; ++w) t += red[w][lane];
    part[(size_t)blockIdx.x * kNfK + lane] = t;
  }
}

__global__ void k_nf_psi(NfArgs a, const double* part, int nblocks, double* psi_dev) {
  const int c = threadIdx.x;
  const int i = a.origin[c];
  if (i < 0) return;
  double s = 0.0;
  for (int k = 0; k < nblocks; ++k) s += part[(size_t)k * kNfK + c];
  const double2 lm = a.lm[i];
  psi_dev[c] = (s + lm.x / (lm.x + lm.y)) / (double)a.n;      // + d_i (own wall)
}

// column c of P (and of Q = C P + D) into origin-major outputs out[c * n + j]
__global__ void k_nf_columns(NfArgs a, const double* __restrict__ P, int k, double* p_out,
                             double* q_out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)k * a.n;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t / a.n);
    const long long j = t - (long long)c * a.n;
    const double p = P[(size_t)j * kNfK + c];
    if (p_out) p_out[t] = p;
    if (q_out) {
      const double2 lm = a.lm[j];
      double q = lm.y / (lm.x + lm.y) * p;
      if (j == a.origin[c]) q += lm.x / (lm.x + lm.y);
      q_out[t] = q;
    }
  }
}

int nf_grid(long long n) {
  long long g = (n + kNfBlock / 32 - 1) / (kNfBlock / 32);
  if (g > 148 * 8) g = 148 * 8;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

// One batch of <= kNfK origins on the context stream (host driver of Alg. 1).  The caller
// owns the work buffers (NfWork).  On return: P of the batch in work.P[cur], per-column
// iterations / gaps in a.iters / a.gap, psi of the batch in psi_dev[c] (if non-NULL).
cudaError_t power_nf_batch(const NfArgs& a, NfWork& w, double eps, long long max_iters,
                           double* psi_dev, cudaStream_t s, int* cur_out, long long* sweeps) {
  const int grid = nf_grid(a.n);
  cudaError_t e;
  int cur = 0;
  k_nf_step<<<grid, kNfBlock, 0, s>>>(a, w.P[1], w.P[0], 1, w.part);
  k_nf_finish<<<1, 32, 0, s>>>(a, w.part, grid, 1, eps, max_iters, w.active);
  long long it = 0;
  // check the active-column count every `stride` steps: frozen columns do not change, so
  // the extra steps after the last column freezes are no-ops for the result
  const int stride = 8;
  while (true) {
    if ((e = cudaMemcpyAsync(w.h_active, w.active, sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return e;
    if (*w.h_active == 0 || it >= max_iters) break;
    for (int k = 0; k < stride; ++k, ++it) {
      k_nf_step<<<grid, kNfBlock, 0, s>>>(a, w.P[cur], w.P[cur ^ 1], 0, w.part);
      k_nf_finish<<<1, 32, 0, s>>>(a, w.part, grid, 0, eps, max_iters, w.active);
      cur ^= 1;
    }
  }
  if (psi_dev) {
    k_nf_wall<<<grid, kNfBlock, 0, s>>>(a, w.P[cur], w.part);
    k_nf_psi<<<1, 32, 0, s>>>(a, w.part, grid, psi_dev);
  }
  *cur_out = cur;
  if (sweeps) *sweeps = it;
  return cudaGetLastError();
}

cudaError_t power_nf_columns(const NfArgs& a, const NfWork& w, int cur, int k, double* p_out,
                             double* q_out, cudaStream_t s) {
  long long g = ((long long)k * a.n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  k_nf_columns<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(a, w.P[cur], k, p_out, q_out);
  return cudaGetLastError();
}

size_t power_nf_part_elems(long long n) { return (size_t)nf_grid(n) * kNfK; }

}  // namespace psi
