// psi_pagerank.cu -- PageRank power method (Eq. (22)) on the Power-psi sweep.
//
// the paper's baseline for "Power-psi is as fast as PageRank" (P:27,
// P:432, Table IV).  W = D_out^{-1} L walks follower -> leader:
//     pi_t^T = alpha pi_{t-1}^T W + (1 - alpha)/N 1^T,   pi_0 = (1/N) 1,
//     (pi^T W)_i = sum_{j in F(i)} pi_j / |L(j)|,
// stopped when ||pi_t - pi_{t-1}||_1 <= eps (the "pi-tolerance"); rows of
// leaderless users are zero (reading R5, as in the oracle).  It is the same gather as the
// psi sweep in kernel state x = pi / Dt, Dt = max(|L(j)|, 1):
//     x_t,i = a_i + g_i sum_{j in F(i)} x_{t-1,j},   a_i = (1-alpha)/(N Dt_i),  g_i = alpha/Dt_i,
//     ||pi_t - pi_{t-1}||_1 = sum_i Dt_i |x_t,i - x_{t-1,i}|,
// so k_heavy / k_tiles / k_fix run unchanged with these constants.  Follower-less users are
// folded as for psi: their pi is (1-alpha)/N from t = 1 on and 1/N at t = 0, so the folded
// constant of the first sweep differs (a_first).
#include "psi_internal.cuh"

namespace psi {
namespace {

#define GRID_STRIDE(i, n)                                                                  \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)(n); \
       i += (long long)gridDim.x * blockDim.x)

__global__ void k_pr_prep(const int* nlead, const double* kinv, long long n, long long n_act,
                          double alpha, double N, double* a, double* a_first, double* g,
                          double* dt, double* x0) {
  GRID_STRIDE(r, n) {
    const double D = (double)max(nlead[r], 1);
    dt[r] = D;
    x0[r] = (1.0 / N) / D;                       // pi_0 = 1/N
    if (r < n_act) {
      const double gg = alpha / D;
      const double base = (1.0 - alpha) / N / D;
      g[r] = gg;
      a[r] = fma(gg, (1.0 - alpha) / N * kinv[r], base);
      a_first[r] = fma(gg, (1.0 / N) * kinv[r], base);
    }
  }
}

// pi in the relabelled order: Dt * x_T for users with followers; the constant otherwise
__global__ void k_pr_readout(const double* xT, const double* dt, long long n, long long n_act,
                             double alpha, double N, long long T, double* pi) {
  GRID_STRIDE(r, n) {
    if (r < n_act) pi[r] = dt[r] * xT[r];
    else pi[r] = T >= 1 ? (1.0 - alpha) / N : 1.0 / N;
  }
}

int grid_for(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

}  // namespace

cudaError_t pagerank_prep(const IngestOut& G, long long n, double alpha, const PrBuffers& B,
                          cudaStream_t s) {
  k_pr_prep<<<grid_for(n), 256, 0, s>>>(G.nlead, G.kinv, n, G.n_act, alpha, (double)n, B.a,
                                        B.a_first, B.g, B.dt, B.x0);
  return cudaGetLastError();
}

cudaError_t pagerank_readout(const IngestOut& G, long long n, double alpha, const double* xT,
                             long long T, const PrBuffers& B, cudaStream_t s) {
  k_pr_readout<<<grid_for(n), 256, 0, s>>>(xT, B.dt, n, G.n_act, alpha, (double)n, T, B.pi);
  return cudaGetLastError();
}

}  // namespace psi
