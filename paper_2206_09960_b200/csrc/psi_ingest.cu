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
//  5. locality relabel: users WITH followers ("active": their s can
//     change) get labels [0, n_act), follower-less users [n_act, n).  Inside the active
//     range: users with >= 2 leaders sorted by leader count, descending (their x is
//     gathered once per leader, so the most-gathered entries form a contiguous hot
//     prefix that stays in L2); then leaderless active users; then single-leader users
//     level by level in the order of their leader's label (each is gathered exactly once
//     per sweep, by its leader's row, so rows processed in label order read them as a
//     stream).  A follower-less user n never changes (x_n = a_n for all t), so its term
//     is folded into per-row constants K_j = sum_{n in F(j), n follower-less} a_n:
//     x_t,j = (a_j + g_j K_j) + g_j sum_{active n} x_n, and the readout uses
//     d_j + lambda_j K_j; its psi is d_n/N (no B term).  Exact algebra, fixed order.
//  6. the relabelled CSR over active rows (followers mapped to new labels, sorted per
//     row), merge-path tile coordinates, and the rows cut by tile boundaries.
#include "psi_internal.cuh"
#include "../../include/psi.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cstdio>
#include <cstring>

namespace psi {
namespace {

enum : int {
  F_RP0 = 1, F_RPN = 2, F_RPMONO = 4, F_RANGE = 8, F_SELF = 16, F_ORDER = 32, F_ACT = 64,
};
// user classes of the relabel
enum : unsigned char { C_HOT = 0, C_SINGLE = 1, C_ROOT = 2, C_INACTIVE = 3 };

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

#define GRID_STRIDE(i, n)                                                                  \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)(n); \
       i += (long long)gridDim.x * blockDim.x)
#define WARP_STRIDE(w, n)                                                                      \
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; w < (long long)(n); \
       w += (long long)gridDim.x * blockDim.x / 32)

// ------------------------------------------------------------------ 1. validation

__global__ void k_check_rowptr(const long long* rp, long long n, long long m, int* flags) {
  GRID_STRIDE(r, n) {
    const long long a = rp[r], b = rp[r + 1];
    int f = 0;
    if (b < a) f |= F_RPMONO;
    if (r == 0 && a != 0) f |= F_RP0;
    if (r == n - 1 && b != m) f |= F_RPN;
    if (f) atomicOr(flags, f);
  }
}

__global__ void k_rowptr32(const long long* rp64, int* rp32, long long n1) {
  GRID_STRIDE(r, n1) rp32[r] = (int)rp64[r];
}

// warp per row: range, self loop, strictly increasing
__global__ void k_check_edges(const int* rp, const int* idx, int n, int* flags) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(row, n) {
    const int b = rp[row], e = rp[row + 1];
    int f = 0;
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      if (v < 0 || v >= n) f |= F_RANGE;
      if (v == (int)row) f |= F_SELF;
      if (q + 1 < e && idx[q + 1] <= v) f |= F_ORDER;
    }
    f = __reduce_or_sync(kFull, f);
    if (lane == 0 && f) atomicOr(flags, f);
  }
}

__global__ void k_check_activity(const double* lam, const double* mu, long long n, int* flags) {
  GRID_STRIDE(i, n) {
    const double l = lam[i], u = mu[i];
    const bool ok = isfinite(l) && isfinite(u) && l >= 0.0 && u >= 0.0 && (l + u) > 0.0;
    if (!ok) atomicOr(flags, F_ACT);
  }
}

// ------------------------------------------------------------------ 2.-4. normalisers

// leader (row) of every edge, a copy of the follower, and #leaders of every follower
__global__ void k_expand(const int* rp, const int* idx, int n, int* leader_of_edge,
                         int* follower_copy, int* n_leaders) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(row, n) {
    const int b = rp[row], e = rp[row + 1];
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      leader_of_edge[q] = (int)row;
      follower_copy[q] = v;
      atomicAdd(n_leaders + v, 1);
    }
  }
}

// warp per user n: W_n, Lambda_n, M_n over its leaders (ascending, fixed tree), then constants.
__global__ void k_normalisers(const int* loff, const int* leaders, const double* lam,
                              const double* mu, int n, double* a, double* g, double* wt,
                              double* d, int* first_leader, unsigned long long* kmax,
                              unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(u, n) {
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
      W += __shfl_xor_sync(kFull, W, o);
      L += __shfl_xor_sync(kFull, L, o);
      M += __shfl_xor_sync(kFull, M, o);
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
      first_leader[u] = e > b ? leaders[b] : -1;
      if (W > 0.0) {
        atomicMax(kmax + 0, dbits(L / W));             // row sum of B
        atomicMax(kmax + 1, dbits(M / W));             // row sum of A
      } else {
        atomicAdd(cnt + 0, 1ull);                      // leaderless
      }
    }
  }
}

// warp per leader i: column sum of B = lambda_i sum_{j in F(i)} 1/W_j.
__global__ void k_kappa_col(const int* rp, const int* idx, const double* wt, const double* lam,
                            int n, unsigned long long* kmax) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, n) {
    const int b = rp[i], e = rp[i + 1];
    double s = 0.0;
    for (int q = b + lane; q < e; q += 32) s += 1.0 / wt[idx[q]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0 && e > b) atomicMax(kmax + 2, dbits(lam[i] * s));
  }
}

// ------------------------------------------------------------------ 5. relabel

__global__ void k_classify(const int* rp, const int* nlead, int n, unsigned char* cls,
                           int* new_of_old, unsigned long long* counts) {
  GRID_STRIDE(u, n) {
    const bool active = rp[u + 1] > rp[u];
    const int nl = nlead[u];
    unsigned char c = !active ? C_INACTIVE : nl >= 2 ? C_HOT : nl == 1 ? C_SINGLE : C_ROOT;
    cls[u] = c;
    new_of_old[u] = -1;
    atomicAdd(counts + c, 1ull);
  }
}

// selection keys for one relabel stage
//   stage 0: hot users, key = (INT_MAX - #leaders) << 32 | u   (descending leader count)
//   stage 1: leaderless active users, key = u
//   stage 2: single-leader users whose leader is labelled, key = label(leader) << 32 | u
//   stage 3: remaining single-leader users (cycles), key = leader << 32 | u
//   stage 4: follower-less users, key = u
__global__ void k_stage_keys(int stage, const unsigned char* cls, const int* nlead,
                             const int* first_leader, const int* new_of_old, int n,
                             unsigned long long* key, unsigned char* flag) {
  GRID_STRIDE(u, n) {
    const unsigned char c = cls[u];
    unsigned char f = 0;
    unsigned long long k = (unsigned long long)u;
    if (stage == 0) {
      f = c == C_HOT;
      k |= (unsigned long long)(0x7fffffff - nlead[u]) << 32;
    } else if (stage == 1) {
      f = c == C_ROOT;
    } else if (stage == 2) {
      if (c == C_SINGLE && new_of_old[u] < 0) {
        const int lab = new_of_old[first_leader[u]];
        if (lab >= 0) { f = 1; k |= (unsigned long long)lab << 32; }
      }
    } else if (stage == 3) {
      if (c == C_SINGLE && new_of_old[u] < 0) {
        f = 1;
        k |= (unsigned long long)first_leader[u] << 32;
      }
    } else {
      f = c == C_INACTIVE;
    }
    flag[u] = f;
    key[u] = k;
  }
}

__global__ void k_assign(const unsigned long long* sel, long long cnt, int base, int* new_of_old,
                         int* old_of_new) {
  GRID_STRIDE(i, cnt) {
    const int u = (int)(sel[i] & 0xffffffffull);
    new_of_old[u] = base + (int)i;
    old_of_new[base + i] = u;
  }
}

// warp per new active row r: #active followers, and K_r = sum of a_n over follower-less ones
__global__ void k_row_count(const int* rp, const int* idx, const int* old_of_new,
                            const unsigned char* cls, const double* a_old, int n_act, int* cnt,
                            double* K) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_act) {
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    int c = 0;
    double k = 0.0;
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      if (cls[v] == C_INACTIVE) k += a_old[v]; else ++c;
    }
    c = __reduce_add_sync(kFull, c);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) k += __shfl_xor_sync(kFull, k, s);
    if (lane == 0) { cnt[r] = c > 0 ? c : 1; K[r] = k; }   // 0 -> one pseudo edge
  }
}

// warp per new active row: write the active followers' new labels (unsorted, stable); a row
// with no active follower gets one pseudo edge to the sentinel label n (x[n] = 0).
__global__ void k_row_fill(const int* rp, const int* idx, const int* old_of_new,
                           const unsigned char* cls, const int* new_of_old, const int* rp_new,
                           int n_act, int n, int* idx_new) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_act) {
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    const int start = rp_new[r];
    int out = start;
    for (int q0 = b; q0 < e; q0 += 32) {
      const int q = q0 + lane;
      int v = -1;
      bool act = false;
      if (q < e) { v = idx[q]; act = cls[v] != C_INACTIVE; }
      const unsigned mask = __ballot_sync(kFull, act);
      if (act) idx_new[out + __popc(mask & ((1u << lane) - 1u))] = new_of_old[v];
      out += __popc(mask);
    }
    if (lane == 0 && out == start) idx_new[start] = n;
  }
}

// flag the first word of every row; pad [m_act, m_pad) with unflagged sentinel words
__global__ void k_flag_rows(const int* rp_new, int n_act, long long m_act, long long m_pad, int n,
                            unsigned* edges) {
  GRID_STRIDE(r, n_act) edges[rp_new[r]] |= kRowFlag;
  GRID_STRIDE(q, m_pad - m_act) edges[m_act + q] = (unsigned)n;
}

__global__ void k_permute_vectors(const int* old_of_new, int n, int n_act, const double* a_old,
                                  const double* g_old, const double* wt_old, const double* d_old,
                                  const double* lam, const double* K, double n_users,
                                  double* a0, double* a1, double* g1, double* wt_new, double* d1,
                                  double* lam1, double* psi) {
  GRID_STRIDE(r, n) {
    const int o = old_of_new[r];
    a0[r] = a_old[o];
    wt_new[r] = wt_old[o];
    if (r < n_act) {
      const double k = K[r];
      a1[r] = fma(g_old[o], k, a_old[o]);
      g1[r] = g_old[o];
      d1[r] = fma(lam[o], k, d_old[o]);
      lam1[r] = lam[o];
    } else {
      psi[r] = d_old[o] / n_users;          // follower-less: (s^T B)_r = 0
    }
  }
}

// ------------------------------------------------------------------ 7. tiles

// tile_row[k] = number of rows whose first edge lies before edge k*kTile
__global__ void k_tile_rows(const int* rp, int n_act, int ntiles, int* tile_row) {
  GRID_STRIDE(k, ntiles + 1) {
    const long long e = k * (long long)kTile;
    int lo = 0, hi = n_act;                 // first row r with rp[r] >= e
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((long long)rp[mid] < e) lo = mid + 1; else hi = mid;
    }
    tile_row[k] = lo;
  }
}

// rows whose edges fall in more than one tile
__global__ void k_split_flags(const int* rp, int n, unsigned char* flag) {
  GRID_STRIDE(r, n) flag[r] = (rp[r] / kTile) != ((rp[r + 1] - 1) / kTile) ? 1 : 0;
}

__global__ void k_split_fill(const int* rows, long long ns, const int* rp, int4* split) {
  GRID_STRIDE(s, ns) {
    const int r = rows[s];
    split[s] = make_int4(r, rp[r] / kTile, (rp[r + 1] - 1) / kTile, 0);
  }
}

// ------------------------------------------------------------------ host helpers

struct Tmp {  // RAII device buffer for temporaries
  void* p = nullptr;
  ~Tmp() { reset(); }
  void reset() { if (p) cudaFree(p); p = nullptr; }
  cudaError_t alloc(size_t bytes) { reset(); return cudaMalloc(&p, bytes ? bytes : 16); }
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
           const double* lam, const double* mu, cudaStream_t s, IngestOut& out, char* msg,
           size_t msg_len) {
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
  Tmp rp_old;
  IG_CK(rp_old.alloc((size_t)(n + 1) * sizeof(int)));
  const int* rp = rp_old.as<int>();
  k_rowptr32<<<grid_for(n + 1, 256), 256, 0, s>>>(rp64, rp_old.as<int>(), n + 1);
  k_check_edges<<<grid_for(n * 32, 256), 256, 0, s>>>(rp, idx_in, N, flags.as<int>());
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

  // ---- 2.-4. transpose, normalisers, constants (old labels)
  Tmp a_old, g_old, wt_old, d_old, first_leader, nlead, red;
  IG_CK(a_old.alloc((size_t)n * sizeof(double)));
  IG_CK(g_old.alloc((size_t)n * sizeof(double)));
  IG_CK(wt_old.alloc((size_t)n * sizeof(double)));
  IG_CK(d_old.alloc((size_t)n * sizeof(double)));
  IG_CK(first_leader.alloc((size_t)n * sizeof(int)));
  IG_CK(nlead.alloc((size_t)(n + 1) * sizeof(int)));
  IG_CK(red.alloc(16 * sizeof(unsigned long long)));
  IG_CK(cudaMemsetAsync(red.p, 0, 16 * sizeof(unsigned long long), s));
  IG_CK(cudaMemsetAsync(nlead.p, 0, (size_t)(n + 1) * sizeof(int), s));
  unsigned long long* kmax = red.as<unsigned long long>();
  unsigned long long* cnt = kmax + 4;
  unsigned long long* ccount = kmax + 8;     // class counts
  int end_bit = 1;
  while ((1ll << end_bit) < n) ++end_bit;
  {
    Tmp leader_e, follower_e, leader_s, follower_s, loff, sort_tmp, scan_tmp;
    IG_CK(leader_e.alloc((size_t)m * sizeof(int)));
    IG_CK(follower_e.alloc((size_t)m * sizeof(int)));
    IG_CK(leader_s.alloc((size_t)m * sizeof(int)));
    IG_CK(follower_s.alloc((size_t)m * sizeof(int)));
    IG_CK(loff.alloc((size_t)(n + 1) * sizeof(int)));
    k_expand<<<grid_for(n * 32, 256), 256, 0, s>>>(rp, idx_in, N, leader_e.as<int>(),
                                                   follower_e.as<int>(), nlead.as<int>());
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
    k_normalisers<<<grid_for(n * 32, 256), 256, 0, s>>>(
        loff.as<int>(), vals.Current(), lam, mu, N, a_old.as<double>(), g_old.as<double>(),
        wt_old.as<double>(), d_old.as<double>(), first_leader.as<int>(), kmax, cnt);
    k_kappa_col<<<grid_for(n * 32, 256), 256, 0, s>>>(rp, idx_in, wt_old.as<double>(), lam, N, kmax);
  }

  // ---- 5. relabel
  Tmp cls, new_of_old, key, sel, flag8, nsel, stage_tmp, sort_tmp2, sorted;
  IG_CK(cls.alloc((size_t)n));
  IG_CK(new_of_old.alloc((size_t)n * sizeof(int)));
  IG_CK(cudaMalloc(&out.old_of_new, (size_t)n * sizeof(int)));
  k_classify<<<grid_for(n, 256), 256, 0, s>>>(rp, nlead.as<int>(), N, cls.as<unsigned char>(),
                                              new_of_old.as<int>(), ccount);
  unsigned long long h[16];
  IG_CK(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  memcpy(&out.kappa_row, &h[0], 8);
  memcpy(&out.rho_A, &h[1], 8);
  memcpy(&out.kappa_col, &h[2], 8);
  out.n_leaderless = (long long)h[4];
  out.n_g = n - out.n_leaderless;
  const long long n_inactive = (long long)h[8 + C_INACTIVE];
  out.n_act = n - n_inactive;
  out.n_f = out.n_act;
  out.n_hot = (long long)h[8 + C_HOT];

  IG_CK(key.alloc((size_t)n * 8));
  IG_CK(sel.alloc((size_t)n * 8));
  IG_CK(sorted.alloc((size_t)n * 8));
  IG_CK(flag8.alloc((size_t)n));
  IG_CK(nsel.alloc(sizeof(long long)));
  size_t sel_bytes = 0, sort_bytes = 0;
  IG_CK(cub::DeviceSelect::Flagged(nullptr, sel_bytes, key.as<unsigned long long>(),
                                   flag8.as<unsigned char>(), sel.as<unsigned long long>(),
                                   nsel.as<long long>(), N, s));
  IG_CK(stage_tmp.alloc(sel_bytes));
  IG_CK(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, sel.as<unsigned long long>(),
                                       sorted.as<unsigned long long>(), N, 0, 64, s));
  IG_CK(sort_tmp2.alloc(sort_bytes));
  int base = 0;
  int levels = 0;
  auto run_stage = [&](int stage, bool sort_keys, long long* count) -> int {
    k_stage_keys<<<grid_for(n, 256), 256, 0, s>>>(stage, cls.as<unsigned char>(), nlead.as<int>(),
                                                  first_leader.as<int>(), new_of_old.as<int>(), N,
                                                  key.as<unsigned long long>(),
                                                  flag8.as<unsigned char>());
    size_t b1 = sel_bytes;
    IG_CK(cub::DeviceSelect::Flagged(stage_tmp.p, b1, key.as<unsigned long long>(),
                                     flag8.as<unsigned char>(), sel.as<unsigned long long>(),
                                     nsel.as<long long>(), N, s));
    long long c = 0;
    IG_CK(cudaMemcpyAsync(&c, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    *count = c;
    if (c == 0) return PSI_OK;
    const unsigned long long* src = sel.as<unsigned long long>();
    if (sort_keys) {
      size_t b2 = sort_bytes;
      IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp2.p, b2, sel.as<unsigned long long>(),
                                           sorted.as<unsigned long long>(), (int)c, 0, 64, s));
      src = sorted.as<unsigned long long>();
    }
    k_assign<<<grid_for(c, 256), 256, 0, s>>>(src, c, base, new_of_old.as<int>(), out.old_of_new);
    base += (int)c;
    return PSI_OK;
  };
  long long c = 0;
  int rc;
  if ((rc = run_stage(0, true, &c)) != PSI_OK) return rc;          // hot, by leader count
  if ((rc = run_stage(1, false, &c)) != PSI_OK) return rc;         // leaderless active
  while (true) {                                                   // single-leader, by level
    if ((rc = run_stage(2, true, &c)) != PSI_OK) return rc;
    if (c == 0) break;
    ++levels;
  }
  if ((rc = run_stage(3, true, &c)) != PSI_OK) return rc;          // leftovers (cycles)
  if (base != out.n_act) {
    snprintf(msg, msg_len, "internal: relabel covered %d of %lld active users", base, out.n_act);
    return PSI_E_CUDA;
  }
  if ((rc = run_stage(4, false, &c)) != PSI_OK) return rc;         // follower-less
  out.relabel_levels = levels;
  key.reset(); sel.reset(); sorted.reset(); flag8.reset(); stage_tmp.reset(); sort_tmp2.reset();

  // ---- 6. relabelled edge stream over active rows, folded constants
  const int NA = (int)out.n_act;
  Tmp cntr, K, rp_new;
  IG_CK(cntr.alloc((size_t)(NA + 1) * sizeof(int)));
  IG_CK(K.alloc((size_t)(NA > 0 ? NA : 1) * sizeof(double)));
  IG_CK(rp_new.alloc((size_t)(NA + 1) * sizeof(int)));
  IG_CK(cudaMemsetAsync(cntr.p, 0, (size_t)(NA + 1) * sizeof(int), s));
  if (NA > 0)
    k_row_count<<<grid_for((long long)NA * 32, 256), 256, 0, s>>>(
        rp, idx_in, out.old_of_new, cls.as<unsigned char>(), a_old.as<double>(), NA,
        cntr.as<int>(), K.as<double>());
  {
    Tmp scan_tmp;
    size_t sb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, cntr.as<int>(), rp_new.as<int>(), NA + 1, s));
    IG_CK(scan_tmp.alloc(sb));
    IG_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, sb, cntr.as<int>(), rp_new.as<int>(), NA + 1, s));
  }
  int m_act = 0;
  IG_CK(cudaMemcpyAsync(&m_act, rp_new.as<int>() + NA, sizeof(int), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  out.m_act = m_act;
  out.ntiles = (int)(((long long)m_act + kTile - 1) / kTile);
  const long long m_pad = (long long)out.ntiles * kTile;
  {
    Tmp idx2, seg_tmp;
    IG_CK(cudaMalloc(&out.edges, (size_t)(m_pad > 0 ? m_pad : 4) * sizeof(unsigned)));
    IG_CK(idx2.alloc((size_t)(m_act > 0 ? m_act : 1) * sizeof(int)));
    int* ed = (int*)out.edges;
    if (NA > 0)
      k_row_fill<<<grid_for((long long)NA * 32, 256), 256, 0, s>>>(
          rp, idx_in, out.old_of_new, cls.as<unsigned char>(), new_of_old.as<int>(),
          rp_new.as<int>(), NA, N, ed);
    if (m_act > 0) {
      cub::DoubleBuffer<int> kb(ed, idx2.as<int>());
      size_t tb = 0;
      IG_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, kb, m_act, NA, rp_new.as<int>(),
                                               rp_new.as<int>() + 1, s));
      IG_CK(seg_tmp.alloc(tb));
      IG_CK(cub::DeviceSegmentedSort::SortKeys(seg_tmp.p, tb, kb, m_act, NA, rp_new.as<int>(),
                                               rp_new.as<int>() + 1, s));
      if (kb.Current() != ed)
        IG_CK(cudaMemcpyAsync(ed, kb.Current(), (size_t)m_act * sizeof(int),
                              cudaMemcpyDeviceToDevice, s));
      k_flag_rows<<<grid_for(NA, 256), 256, 0, s>>>(rp_new.as<int>(), NA, m_act, m_pad, N,
                                                    out.edges);
    }
    IG_CK(cudaStreamSynchronize(s));
  }
  const size_t na_b = (size_t)(NA > 0 ? NA : 1) * sizeof(double);
  IG_CK(cudaMalloc(&out.a0, (size_t)n * sizeof(double)));
  IG_CK(cudaMalloc(&out.wt, (size_t)n * sizeof(double)));
  IG_CK(cudaMalloc(&out.psi, (size_t)n * sizeof(double)));
  IG_CK(cudaMalloc(&out.a1, na_b));
  IG_CK(cudaMalloc(&out.g, na_b));
  IG_CK(cudaMalloc(&out.d1, na_b));
  IG_CK(cudaMalloc(&out.lam, na_b));
  k_permute_vectors<<<grid_for(n, 256), 256, 0, s>>>(
      out.old_of_new, N, NA, a_old.as<double>(), g_old.as<double>(), wt_old.as<double>(),
      d_old.as<double>(), lam, K.as<double>(), (double)n, out.a0, out.a1, out.g, out.wt, out.d1,
      out.lam, out.psi);
  out.relabeled = 1;

  // ---- 7. edge tiles: first row of every tile, rows spanning tiles
  IG_CK(cudaMalloc(&out.tile_row, (size_t)(out.ntiles + 1) * sizeof(int)));
  k_tile_rows<<<grid_for(out.ntiles + 1, 256), 256, 0, s>>>(rp_new.as<int>(), NA, out.ntiles,
                                                            out.tile_row);
  {
    Tmp fl, rows, ns, sel_tmp;
    IG_CK(fl.alloc((size_t)(NA > 0 ? NA : 1)));
    IG_CK(rows.alloc((size_t)(NA > 0 ? NA : 1) * sizeof(int)));
    IG_CK(ns.alloc(sizeof(long long)));
    IG_CK(cudaMemsetAsync(ns.p, 0, sizeof(long long), s));
    long long hs = 0;
    if (NA > 0) {
      k_split_flags<<<grid_for(NA, 256), 256, 0, s>>>(rp_new.as<int>(), NA, fl.as<unsigned char>());
      cub::CountingInputIterator<int> it(0);
      size_t tb = 0;
      IG_CK(cub::DeviceSelect::Flagged(nullptr, tb, it, fl.as<unsigned char>(), rows.as<int>(),
                                       ns.as<long long>(), NA, s));
      IG_CK(sel_tmp.alloc(tb));
      IG_CK(cub::DeviceSelect::Flagged(sel_tmp.p, tb, it, fl.as<unsigned char>(), rows.as<int>(),
                                       ns.as<long long>(), NA, s));
      IG_CK(cudaMemcpyAsync(&hs, ns.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
      IG_CK(cudaStreamSynchronize(s));
    }
    out.nsplit = (int)hs;
    IG_CK(cudaMalloc(&out.split, (size_t)(hs > 0 ? hs : 1) * sizeof(int4)));
    if (hs > 0)
      k_split_fill<<<grid_for(hs, 256), 256, 0, s>>>(rows.as<int>(), hs, rp_new.as<int>(),
                                                     out.split);
    IG_CK(cudaStreamSynchronize(s));
  }
  IG_CK(cudaGetLastError());
  return PSI_OK;
}

}  // namespace psi
