// psi_ingest.cu -- one-time graph ingest on the device.
//
// Steps (all on the caller's stream):
//  1. validate the input contract (include/psi.h): row_ptr, indices, self loops,
//     strictly increasing rows, activity;
//  2. leaders-per-follower by a stable radix sort of (follower, leader) pairs, i.e.
//     the transpose of the input CSR, so that every newsfeed normaliser
//        W_n = sum_{l in L(n)} (lambda_l + mu_l)
//     and Lambda_n = sum_{l in L(n)} lambda_l, M_n = sum_{l in L(n)} mu_l are summed
//     in a fixed order (ascending leader) -- deterministic, no fp atomics;
//  3. per-user kernel constants c = mu/w, d = lambda/w,
//     Wt = W (or 1 if W = 0, reading R5), a = c/Wt, g = mu/Wt;
//  4. ||B|| in all three readings (R1): kappa_row = max_n Lambda_n/W_n,
//     kappa_col = max_i lambda_i sum_{j in F(i)} 1/W_j; rho_A = max_n M_n/W_n;
//  5. merge-path tile coordinates and the list of rows cut by tile boundaries.
#include "psi_internal.cuh"
#include "../../include/psi.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cstdio>
#include <cstring>

namespace psi {
namespace {

enum : int {
  F_RP0 = 1, F_RPN = 2, F_RPMONO = 4, F_RANGE = 8, F_SELF = 16, F_ORDER = 32, F_ACT = 64,
};

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

__global__ void k_check_rowptr(const long long* rp, long long n, long long m, int* flags) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += stride) {
    const long long a = rp[r], b = rp[r + 1];
    int f = 0;
    if (b < a) f |= F_RPMONO;
    if (r == 0 && a != 0) f |= F_RP0;
    if (r == n - 1 && b != m) f |= F_RPN;
    if (f) atomicOr(flags, f);
  }
}

__global__ void k_rowptr32(const long long* rp64, int* rp32, long long n1) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n1; r += stride)
    rp32[r] = (int)rp64[r];
}

// warp per row: range, self loop, strictly increasing
__global__ void k_check_edges(const int* rp, const int* idx, int n, int* flags) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * blockDim.x / 32;
  for (long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; row < n; row += nw) {
    const int b = rp[row], e = rp[row + 1];
    int f = 0;
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      if (v < 0 || v >= n) f |= F_RANGE;
      if (v == (int)row) f |= F_SELF;
      if (q + 1 < e && idx[q + 1] <= v) f |= F_ORDER;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0 && f) atomicOr(flags, f);
  }
}

__global__ void k_check_activity(const double* lam, const double* mu, long long n, int* flags) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double l = lam[i], u = mu[i];
    const bool ok = isfinite(l) && isfinite(u) && l >= 0.0 && u >= 0.0 && (l + u) > 0.0;
    if (!ok) atomicOr(flags, F_ACT);
  }
}

// leader (row) of every edge, and #leaders of every follower
__global__ void k_expand(const int* rp, const int* idx, int n, int* leader_of_edge,
                         int* follower_copy, int* n_leaders) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * blockDim.x / 32;
  for (long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; row < n; row += nw) {
    const int b = rp[row], e = rp[row + 1];
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      leader_of_edge[q] = (int)row;
      follower_copy[q] = v;
      atomicAdd(n_leaders + v, 1);
    }
  }
}

// warp per user n: W_n, Lambda_n, M_n over its leaders (ascending), then the constants.
__global__ void k_normalisers(const int* loff, const int* leaders, const double* lam,
                              const double* mu, int n, double* a, double* g, double* wt,
                              double* d, unsigned long long* kmax, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * blockDim.x / 32;
  for (long long u = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; u < n; u += nw) {
    const int b = loff[u], e = loff[u + 1];
    double W = 0.0, L = 0.0, M = 0.0;
    for (int q = b + lane; q < e; q += 32) {
      const int l = leaders[q];
      const double ll = lam[l], mm = mu[l];
      W += ll + mm;
      L += ll;
      M += mm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      W += __shfl_xor_sync(0xffffffffu, W, o);
      L += __shfl_xor_sync(0xffffffffu, L, o);
      M += __shfl_xor_sync(0xffffffffu, M, o);
    }
    if (lane == 0) {
      const double lu = lam[u], mu_u = mu[u];
      const double w = lu + mu_u;
      const double c = mu_u / w;
      d[u] = lu / w;
      const double W_t = W > 0.0 ? W : 1.0;            // R5: leaderless slot holds s_j
      wt[u] = W_t;
      a[u] = c / W_t;
      g[u] = mu_u / W_t;
      if (W > 0.0) {
        atomicMax(kmax + 0, dbits(L / W));             // row sum of B
        atomicMax(kmax + 1, dbits(M / W));             // row sum of A
      } else {
        atomicAdd(cnt + 0, 1ull);                      // leaderless
      }
    }
  }
}

// warp per leader i: column sum of B = lambda_i sum_{j in F(i)} 1/W_j; count rows with followers.
__global__ void k_kappa_col(const int* rp, const int* idx, const double* wt, const double* lam,
                            int n, unsigned long long* kmax, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * blockDim.x / 32;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const int b = rp[i], e = rp[i + 1];
    double s = 0.0;
    for (int q = b + lane; q < e; q += 32) s += 1.0 / wt[idx[q]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && e > b) {
      atomicMax(kmax + 2, dbits(lam[i] * s));
      atomicAdd(cnt + 1, 1ull);                        // N_f
    }
  }
}

// merge-path coordinate (row, edge) of diagonal k*kTile: a = row ends rp[1..n], b = 0..m-1
__global__ void k_tile_coords(const int* rp, int n, int m, int ntiles, int2* tc) {
  const int stride = gridDim.x * blockDim.x;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= ntiles; k += stride) {
    long long diag = (long long)k * kTile;
    if (diag > (long long)n + m) diag = (long long)n + m;
    long long lo = diag - m > 0 ? diag - m : 0;
    long long hi = diag < n ? diag : n;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if ((long long)rp[mid + 1] <= diag - mid - 1) lo = mid + 1; else hi = mid;
    }
    tc[k] = make_int2((int)lo, (int)(diag - lo));
  }
}

// rows whose merge items fall in more than one tile
__global__ void k_split_flags(const int* rp, int n, int* flag) {
  const int stride = gridDim.x * blockDim.x;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const long long b = rp[r], e = rp[r + 1];
    const long long ta = (b + r) / kTile, tb = (e + r) / kTile;
    flag[r] = (e > b && ta != tb) ? 1 : 0;
  }
}

__global__ void k_split_fill(const int* rows, const int* nsel, const int* rp, int4* split) {
  const int ns = *nsel;
  const int stride = gridDim.x * blockDim.x;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += stride) {
    const int r = rows[s];
    const long long b = rp[r], e = rp[r + 1];
    split[s] = make_int4(r, (int)((b + r) / kTile), (int)((e + r) / kTile), 0);
  }
}

// RAII device buffer for temporaries
struct Tmp {
  void* p = nullptr;
  ~Tmp() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
  template <class T> T* as() const { return (T*)p; }
};

int grid_for(long long work, int block, int cap = 148 * 16) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

#define IG_CK(call)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      snprintf(msg, msg_len, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),        \
               __FILE__, __LINE__);                                                  \
      return e_ == cudaErrorMemoryAllocation ? PSI_E_OOM : PSI_E_CUDA;               \
    }                                                                                \
  } while (0)

int ingest(long long n, long long m, const long long* rp64, const int* idx_in,
           const double* lam, const double* mu, bool relabel, cudaStream_t s,
           IngestOut& out, char* msg, size_t msg_len) {
  (void)relabel;
  const int N = (int)n, Mm = (int)m;
  Tmp flags;
  IG_CK(flags.alloc(sizeof(int)));
  IG_CK(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
  int hflags = 0;

  // ---- 1. validation
  k_check_rowptr<<<grid_for(n, 256), 256, 0, s>>>(rp64, n, m, flags.as<int>());
  k_check_activity<<<grid_for(n, 256), 256, 0, s>>>(lam, mu, n, flags.as<int>());
  IG_CK(cudaMemcpyAsync(&hflags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  if (hflags & (F_RP0 | F_RPN | F_RPMONO)) {
    snprintf(msg, msg_len, "graph: row_ptr %s", (hflags & F_RP0) ? "row_ptr[0] != 0"
             : (hflags & F_RPN) ? "row_ptr[n] != m" : "is decreasing");
    return PSI_E_GRAPH;
  }
  IG_CK(cudaMalloc(&out.rp, (size_t)(n + 1) * sizeof(int)));
  k_rowptr32<<<grid_for(n + 1, 256), 256, 0, s>>>(rp64, out.rp, n + 1);
  k_check_edges<<<grid_for(n * 32, 256), 256, 0, s>>>(out.rp, idx_in, N, flags.as<int>());
  IG_CK(cudaMemcpyAsync(&hflags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  if (hflags & (F_RANGE | F_SELF | F_ORDER)) {
    snprintf(msg, msg_len, "graph: %s", (hflags & F_RANGE) ? "follower index out of [0, n)"
             : (hflags & F_SELF) ? "self loop (a user in its own follower list)"
             : "row not strictly increasing (duplicate or unsorted followers)");
    return PSI_E_GRAPH;
  }
  if (hflags & F_ACT) {
    snprintf(msg, msg_len, "activity: lambda/mu must be finite, >= 0, lambda+mu > 0");
    return PSI_E_ACTIVITY;
  }

  // ---- 2. transpose: leaders of every follower, ascending (stable LSD radix sort)
  Tmp leader_e, follower_e, leader_s, follower_s, nlead, loff, sort_tmp, scan_tmp;
  IG_CK(leader_e.alloc((size_t)m * sizeof(int)));
  IG_CK(follower_e.alloc((size_t)m * sizeof(int)));
  IG_CK(leader_s.alloc((size_t)m * sizeof(int)));
  IG_CK(follower_s.alloc((size_t)m * sizeof(int)));
  IG_CK(nlead.alloc((size_t)(n + 1) * sizeof(int)));
  IG_CK(loff.alloc((size_t)(n + 1) * sizeof(int)));
  IG_CK(cudaMemsetAsync(nlead.p, 0, (size_t)(n + 1) * sizeof(int), s));
  k_expand<<<grid_for(n * 32, 256), 256, 0, s>>>(out.rp, idx_in, N, leader_e.as<int>(),
                                                 follower_e.as<int>(), nlead.as<int>());
  int end_bit = 1;
  while ((1ll << end_bit) < n) ++end_bit;
  {
    cub::DoubleBuffer<unsigned> keys((unsigned*)follower_e.p, (unsigned*)follower_s.p);
    cub::DoubleBuffer<int> vals(leader_e.as<int>(), leader_s.as<int>());
    size_t tb = 0;
    IG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, Mm, 0, end_bit, s));
    IG_CK(sort_tmp.alloc(tb));
    IG_CK(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tb, keys, vals, Mm, 0, end_bit, s));
    size_t sb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, nlead.as<int>(), loff.as<int>(), N + 1, s));
    IG_CK(scan_tmp.alloc(sb));
    IG_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, sb, nlead.as<int>(), loff.as<int>(), N + 1, s));

    // ---- 3./4. normalisers, constants, norms
    IG_CK(cudaMalloc(&out.a, (size_t)n * sizeof(double)));
    IG_CK(cudaMalloc(&out.g, (size_t)n * sizeof(double)));
    IG_CK(cudaMalloc(&out.wt, (size_t)n * sizeof(double)));
    IG_CK(cudaMalloc(&out.d, (size_t)n * sizeof(double)));
    IG_CK(cudaMalloc(&out.lam, (size_t)n * sizeof(double)));
    IG_CK(cudaMemcpyAsync(out.lam, lam, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    Tmp red;
    IG_CK(red.alloc(8 * sizeof(unsigned long long)));
    IG_CK(cudaMemsetAsync(red.p, 0, 8 * sizeof(unsigned long long), s));
    unsigned long long* kmax = red.as<unsigned long long>();
    unsigned long long* cnt = kmax + 4;
    k_normalisers<<<grid_for(n * 32, 256), 256, 0, s>>>(loff.as<int>(), vals.Current(), lam, mu,
                                                        N, out.a, out.g, out.wt, out.d, kmax, cnt);
    k_kappa_col<<<grid_for(n * 32, 256), 256, 0, s>>>(out.rp, idx_in, out.wt, lam, N, kmax, cnt);
    unsigned long long h[8];
    IG_CK(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    memcpy(&out.kappa_row, &h[0], 8);
    memcpy(&out.rho_A, &h[1], 8);
    memcpy(&out.kappa_col, &h[2], 8);
    out.n_leaderless = (long long)h[4];
    out.n_f = (long long)h[5];
    out.n_g = n - out.n_leaderless;
  }

  // ---- the sweep's index array (identity labels)
  IG_CK(cudaMalloc(&out.idx, (size_t)(m > 0 ? m : 1) * sizeof(int)));
  if (m > 0)
    IG_CK(cudaMemcpyAsync(out.idx, idx_in, (size_t)m * sizeof(int), cudaMemcpyDeviceToDevice, s));
  out.relabeled = 0;

  // ---- 5. merge-path tiles and split rows
  const long long items = n + m;
  out.ntiles = (int)((items + kTile - 1) / kTile);
  IG_CK(cudaMalloc(&out.tile_coord, (size_t)(out.ntiles + 1) * sizeof(int2)));
  k_tile_coords<<<grid_for(out.ntiles + 1, 256), 256, 0, s>>>(out.rp, N, Mm, out.ntiles,
                                                              out.tile_coord);
  {
    Tmp flag, rows, nsel, sel_tmp;
    IG_CK(flag.alloc((size_t)n * sizeof(int)));
    IG_CK(rows.alloc((size_t)n * sizeof(int)));
    IG_CK(nsel.alloc(sizeof(int)));
    k_split_flags<<<grid_for(n, 256), 256, 0, s>>>(out.rp, N, flag.as<int>());
    cub::CountingInputIterator<int> it(0);
    size_t tb = 0;
    IG_CK(cub::DeviceSelect::Flagged(nullptr, tb, it, flag.as<int>(), rows.as<int>(),
                                     nsel.as<int>(), N, s));
    IG_CK(sel_tmp.alloc(tb));
    IG_CK(cub::DeviceSelect::Flagged(sel_tmp.p, tb, it, flag.as<int>(), rows.as<int>(),
                                     nsel.as<int>(), N, s));
    int hs = 0;
    IG_CK(cudaMemcpyAsync(&hs, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    out.nsplit = hs;
    IG_CK(cudaMalloc(&out.split, (size_t)(hs > 0 ? hs : 1) * sizeof(int4)));
    if (hs > 0)
      k_split_fill<<<grid_for(hs, 256), 256, 0, s>>>(rows.as<int>(), nsel.as<int>(), out.rp,
                                                     out.split);
    IG_CK(cudaStreamSynchronize(s));
  }
  IG_CK(cudaGetLastError());
  return PSI_OK;
}

}  // namespace psi
