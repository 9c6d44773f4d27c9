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
//  4. ||B|| in all three readings (R1): kappa_row = max_n Lambda_n/W_n, rho_A = max_n M_n/W_n
//     (kappa_col = max_i lambda_i sum_{j in F(i)} 1/W_j is one pass of the sweep's own
//     kernels over x = 1/Wt after the ingest, psi_api.cu);
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

#include <cub/device/device_partition.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace psi {
namespace {

enum : int {
  F_RP0 = 1, F_RPN = 2, F_RPMONO = 4, F_RANGE = 8, F_SELF = 16, F_ORDER = 32, F_ACT = 64,
};
// user classes of the relabel
enum : unsigned char { C_HOT = 0, C_SINGLE = 1, C_ROOT = 2, C_INACTIVE = 3, C_HEAVY = 4 };

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

// thread per edge (rows expanded): range, self loop, strictly increasing within a row
__global__ void k_check_edges_flat(const int* idx, const int* row, long long m, int n, int* flags) {
  int f = 0;
  GRID_STRIDE(q, m) {
    const int v = idx[q], r = row[q];
    if (v < 0 || v >= n) f |= F_RANGE;
    if (v == r) f |= F_SELF;
    if (q + 1 < m && row[q + 1] == r && idx[q + 1] <= v) f |= F_ORDER;
  }
  f = __reduce_or_sync(kFull, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

__global__ void k_check_activity(const double* lam, const double* mu, long long n, int* flags) {
  GRID_STRIDE(i, n) {
    const double l = lam[i], u = mu[i];
    const bool ok = isfinite(l) && isfinite(u) && l >= 0.0 && u >= 0.0 && (l + u) > 0.0;
    if (!ok) atomicOr(flags, F_ACT);
  }
}

// ------------------------------------------------------------------ 2.-4. normalisers

// leader (row) of every edge: thread per short row, warp per long row (see kShort)
__global__ void k_expand_short(const int* rp, int n, int* leader_of_edge) {
  GRID_STRIDE(row, n) {
    const int b = rp[row], e = rp[row + 1];
    if (e - b > 32) continue;
    for (int q = b; q < e; ++q) leader_of_edge[q] = (int)row;
  }
}
__global__ void k_expand_long(const int* list, int nlist, const int* rp, int* leader_of_edge) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int row = list[i];
    const int b = rp[row], e = rp[row + 1];
    for (int q = b + lane; q < e; q += 32) leader_of_edge[q] = row;
  }
}

// loff[u] = first sorted pair with follower >= u (u = 0..n); nlead[u] = loff[u+1] - loff[u]
__global__ void k_lower_bounds(const unsigned* keys, int m, int n, int* loff, int* nlead) {
  GRID_STRIDE(u, n + 1) {
    int lo = 0, hi = m;
    while (lo < hi) {
      const int mid = (int)(((unsigned)lo + (unsigned)hi) >> 1);
      if (keys[mid] < (unsigned)u) lo = mid + 1; else hi = mid;
    }
    loff[u] = lo;
  }
}
__global__ void k_diff(const int* loff, int n, int* nlead) { GRID_STRIDE(u, n) nlead[u] = loff[u + 1] - loff[u]; }

// Segments (a user's leaders, a leader's followers) follow the power law: most are a few
// entries long, a few are huge.  Every per-segment pass below therefore runs as a thread
// per short segment (<= kShort entries, summed sequentially) plus a warp per long segment
// (a compacted list; fixed shuffle tree) -- both deterministic -- instead of a warp per
// segment that leaves most lanes idle.
constexpr int kShort = 32;

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// (lambda, mu) interleaved: one 16-byte gather per leader instead of two 8-byte ones
__global__ void k_pack_activity(const double* lam, const double* mu, long long n, double2* lm) {
  GRID_STRIDE(i, n) lm[i] = make_double2(lam[i], mu[i]);
}

__global__ void k_long_flags(const int* off, const int* perm, int n, int thr, unsigned char* flag) {
  GRID_STRIDE(r, n) {
    const int o = perm ? perm[r] : (int)r;
    flag[r] = (off[o + 1] - off[o]) > thr;
  }
}

// constants of user u from its newsfeed sums (reading R5); returns the row sums
// of B and A (for ||B||_row and rho_A), -1 for a leaderless user
__device__ __forceinline__ void norm_finish(int u, double W, double L, double M, int first,
                                            const double2* lm, double* a, double* g, double* wt,
                                            double* d, int* first_leader, double& rowB,
                                            double& rowA) {
  const double2 own = lm[u];
  const double w = own.x + own.y;
  const double c = own.y / w;
  d[u] = own.x / w;
  const double W_t = W > 0.0 ? W : 1.0;            // R5: leaderless slot holds s_j
  wt[u] = W_t;
  a[u] = c / W_t;
  g[u] = own.y / W_t;
  first_leader[u] = first;
  rowB = W > 0.0 ? L / W : -1.0;
  rowA = W > 0.0 ? M / W : -1.0;
}

// thread per user with <= kShort leaders: W_n, Lambda_n, M_n summed in leader order
__global__ void k_norm_short(const int* loff, const int* leaders, const double2* lm, int n,
                             double* a, double* g, double* wt, double* d, int* first_leader,
                             unsigned long long* kmax, unsigned long long* cnt) {
  const int lane = threadIdx.x & 31;
  for (long long base = blockIdx.x * (long long)blockDim.x; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long u = base + threadIdx.x;
    double rowB = -1.0, rowA = -1.0;
    bool leaderless = false;
    if (u < n) {
      const int b = loff[u], e = loff[u + 1];
      if (e - b <= kShort) {
        double W = 0.0, L = 0.0, M = 0.0;
        for (int q = b; q < e; ++q) {
          const double2 v = lm[leaders[q]];
          W += v.x + v.y;
          L += v.x;
          M += v.y;
        }
        norm_finish((int)u, W, L, M, e > b ? leaders[b] : -1, lm, a, g, wt, d, first_leader,
                    rowB, rowA);
        leaderless = e == b;
      }
    }
    // one atomic per warp (negative doubles never win: kmax starts at +0.0)
    const unsigned long long mb = warp_max_u64(rowB > 0.0 ? dbits(rowB) : 0ull);
    const unsigned long long ma = warp_max_u64(rowA > 0.0 ? dbits(rowA) : 0ull);
    const unsigned nl = __popc(__ballot_sync(kFull, leaderless));
    if (lane == 0) {
      if (mb) atomicMax(kmax + 0, mb);
      if (ma) atomicMax(kmax + 1, ma);
      if (nl) atomicAdd(cnt + 0, (unsigned long long)nl);
    }
  }
}

// warp per listed user with > kShort leaders (fixed shuffle tree)
__global__ void k_norm_long(const int* list, int nlist, const int* loff, const int* leaders,
                            const double2* lm, double* a, double* g, double* wt, double* d,
                            int* first_leader, unsigned long long* kmax) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int u = list[i];
    const int b = loff[u], e = loff[u + 1];
    double W = 0.0, L = 0.0, M = 0.0;
    // four strided steps per iteration with their gathers in flight together; the sums take
    // them in the same order as a one-step loop (bit-identical results)
    for (int q0 = b + lane; q0 < e; q0 += 128) {
      int ld[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) ld[k] = q0 + 32 * k < e ? leaders[q0 + 32 * k] : -1;
      double2 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = ld[k] >= 0 ? lm[ld[k]] : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (ld[k] < 0) break;
        W += v[k].x + v[k].y;
        L += v[k].x;
        M += v[k].y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      W += __shfl_xor_sync(kFull, W, o);
      L += __shfl_xor_sync(kFull, L, o);
      M += __shfl_xor_sync(kFull, M, o);
    }
    if (lane == 0) {
      double rowB, rowA;
      norm_finish(u, W, L, M, leaders[b], lm, a, g, wt, d, first_leader, rowB, rowA);
      atomicMax(kmax + 0, dbits(rowB));
      atomicMax(kmax + 1, dbits(rowA));
    }
  }
}

// ------------------------------------------------------------------ 5. relabel

// class histogram: one atomic per class and warp (per-thread atomics on 5 counters serialise)
// (into the block's shared counters; flushed once per block by class_flush: one global atomic
// per class and warp-iteration serialised on 5 addresses took 4-5 ms per pass at C5)
__device__ __forceinline__ void count_class(unsigned char c, unsigned long long* counts) {
  const unsigned active = __activemask();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (unsigned char k = 0; k < 5; ++k) {
    const unsigned m = __ballot_sync(active, c == k);
    if (m && lane == __ffs(m) - 1) atomicAdd(counts + k, (unsigned long long)__popc(m));
  }
}
__device__ __forceinline__ void class_init(unsigned long long* sc) {
  if (threadIdx.x < 5) sc[threadIdx.x] = 0;
  __syncthreads();
}
__device__ __forceinline__ void class_flush(const unsigned long long* sc, unsigned long long* counts) {
  __syncthreads();
  if (threadIdx.x < 5 && sc[threadIdx.x]) atomicAdd(counts + threadIdx.x, sc[threadIdx.x]);
}

__global__ void k_classify(const int* rp, const int* nlead, int n, unsigned char* cls,
                           int* new_of_old, unsigned long long* counts) {
  __shared__ unsigned long long sc[5];
  class_init(sc);
  GRID_STRIDE(u, n) {
    const bool active = rp[u + 1] > rp[u];
    const int nl = nlead[u];
    unsigned char c = !active ? C_INACTIVE : nl >= 2 ? C_HOT : nl == 1 ? C_SINGLE : C_ROOT;
    cls[u] = c;
    new_of_old[u] = -1;
    count_class(c, sc);
  }
  class_flush(sc, counts);
}

// selection keys for one relabel stage
//   stage 0: hot users, key = (INT_MAX - #leaders) << 32 | u   (descending leader count)
//   stage 1: leaderless active users, key = u
//   stage 2: single-leader users whose leader is labelled, key = label(leader) << 32 | u
//   stage 3: remaining single-leader users (cycles), key = leader << 32 | u
//   stage 4: follower-less users, key = u
// one level of the single-leader relabel over the still-unlabelled single-leader users only
// (pend, ascending user ids): ready = the leader has a label -> key label(leader) << 32 | u
__global__ void k_level_keys(const int* pend, long long np, const int* first_leader,
                             const int* new_of_old, unsigned long long* key, unsigned char* ready,
                             unsigned char* keep) {
  GRID_STRIDE(i, np) {
    const int u = pend[i];
    const int lab = new_of_old[first_leader[u]];
    key[i] = ((unsigned long long)(lab >= 0 ? lab : 0) << 32) | (unsigned)u;
    ready[i] = lab >= 0;
    keep[i] = lab < 0;
  }
}
__global__ void k_cycle_keys(const int* pend, long long np, const int* first_leader,
                             unsigned long long* key) {
  GRID_STRIDE(i, np) {
    const int u = pend[i];
    key[i] = ((unsigned long long)first_leader[u] << 32) | (unsigned)u;
  }
}
__global__ void k_single_flags(const unsigned char* cls, int n, unsigned char* flag) {
  GRID_STRIDE(u, n) flag[u] = cls[u] == C_SINGLE;
}

__global__ void k_stage_keys(int stage, const unsigned char* cls, const int* nlead,
                             const int* first_leader, const int* new_of_old, int n,
                             unsigned long long* key, unsigned char* flag) {
  GRID_STRIDE(u, n) {
    const unsigned char c = cls[u];
    unsigned char f = 0;
    unsigned long long k = (unsigned long long)u;
    if (stage == 0 || stage == 5) {
      f = c == (stage == 0 ? C_HOT : C_HEAVY);
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

// warp per (old) user: number of followers that are active (have followers themselves)
__global__ void k_active_count_short(const int* rp, const int* idx, const unsigned char* cls,
                                     int n, int* act) {
  GRID_STRIDE(u, n) {
    const int b = rp[u], e = rp[u + 1];
    if (e - b > kShort) continue;
    int c = 0;
    for (int q = b; q < e; ++q) c += cls[idx[q]] != C_INACTIVE;
    act[u] = c;
  }
}
__global__ void k_active_count_long(const int* list, int nlist, const int* rp, const int* idx,
                                    const unsigned char* cls, int* act) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int u = list[i];
    const int b = rp[u], e = rp[u + 1];
    int c = 0;
#pragma unroll 4
    for (int q = b + lane; q < e; q += 32) c += cls[idx[q]] != C_INACTIVE;
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) act[u] = c;
  }
}

// heavy rows: active users with >= min_act active followers; recount the classes
__global__ void k_mark_heavy(const int* act, int n, int min_act, unsigned char* cls,
                             unsigned long long* counts) {
  __shared__ unsigned long long sc[5];
  class_init(sc);
  GRID_STRIDE(u, n) {
    unsigned char c = cls[u];
    if (c != C_INACTIVE && act[u] >= min_act) cls[u] = c = C_HEAVY;
    count_class(c, sc);
  }
  class_flush(sc, counts);
}

// new active row r: #active followers in the edge stream (for heavy rows r < n_heavy only
// those with label >= H; the others, hc[r], go to k_heavy), and K_r = sum of a_n over
// follower-less followers (+ the same sums of 1/max(|L(n)|, 1) for PageRank and of 1/Wt_n for
// ||B||_col, psi_api.cu).  Thread per short row / warp per long row (see kShort).
struct RowCountArgs {
  const int* rp; const int* idx; const int* old_of_new; const unsigned char* cls;
  const int* new_of_old; const double* a_old; const int* nlead; int n_act, n_heavy, H;
  int* cnt; long long* hc; double* K; double* Kinv;
  const double* wt_old; double* Kw;   // Kw_r = sum of 1/Wt_n over follower-less followers
  int* lab;                           // [m] new label of every input edge's follower (for the fill)
};

__global__ void k_row_count_short(RowCountArgs R) {
  GRID_STRIDE(r, R.n_act) {
    const int o = R.old_of_new[r];
    const int b = R.rp[o], e = R.rp[o + 1];
    if (e - b > kShort) continue;
    const bool heavy = r < R.n_heavy;
    int c = 0, h = 0;
    double k = 0.0, ki = 0.0, kw = 0.0;
    for (int q = b; q < e; ++q) {
      const int v = R.idx[q];
      const int nv = R.new_of_old[v];                 // follower-less <=> label >= n_act
      R.lab[q] = nv;
      if (nv >= R.n_act) {
        k += R.a_old[v];
        ki += 1.0 / (double)max(R.nlead[v], 1);
        kw += 1.0 / R.wt_old[v];
      } else if (heavy && nv < R.H) ++h;
      else ++c;
    }
    R.cnt[r] = c > 0 ? c : 1;      // 0 -> one pseudo edge
    R.K[r] = k;
    R.Kinv[r] = ki;
    R.Kw[r] = kw;
    if (heavy) R.hc[r] = h;
  }
}

__global__ void k_row_count_long(RowCountArgs R, const int* list, int nlist) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int r = list[i];
    const int o = R.old_of_new[r];
    const int b = R.rp[o], e = R.rp[o + 1];
    const bool heavy = r < R.n_heavy;
    int c = 0, h = 0;
    double k = 0.0, ki = 0.0, kw = 0.0;
    // four strided steps per iteration, their label gathers in flight together (the sums
    // keep the one-step order: bit-identical)
    for (int q0 = b + lane; q0 < e; q0 += 128) {
      int v[4], nv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = q0 + 32 * j < e ? R.idx[q0 + 32 * j] : -1;
#pragma unroll
      for (int j = 0; j < 4; ++j) nv[j] = v[j] >= 0 ? R.new_of_old[v[j]] : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (v[j] < 0) break;
        R.lab[q0 + 32 * j] = nv[j];                  // follower-less <=> label >= n_act
        if (nv[j] >= R.n_act) {
          k += R.a_old[v[j]];
          ki += 1.0 / (double)max(R.nlead[v[j]], 1);
          kw += 1.0 / R.wt_old[v[j]];
        } else if (heavy && nv[j] < R.H) ++h;
        else ++c;
      }
    }
    c = __reduce_add_sync(kFull, c);
    h = __reduce_add_sync(kFull, h);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      k += __shfl_xor_sync(kFull, k, s);
      ki += __shfl_xor_sync(kFull, ki, s);
      kw += __shfl_xor_sync(kFull, kw, s);
    }
    if (lane == 0) {
      R.cnt[r] = c > 0 ? c : 1;
      R.K[r] = k;
      R.Kinv[r] = ki;
      R.Kw[r] = kw;
      if (heavy) R.hc[r] = h;
    }
  }
}

// write the active followers' new labels in input order to the edge stream -- heavy rows:
// only labels >= H; their labels < H go to hot[hoff[r]...].  A row with no stream follower
// gets one pseudo edge to the sentinel label n (x[n] = 0).  Thread per short row / warp
// per long row (ballot compaction keeps the input order).
struct RowFillArgs {
  const int* rp; const int* lab; const int* old_of_new; const unsigned char* cls;
  const int* rp_new; int n_act, n, n_heavy, H;   // lab: new follower labels (k_row_count)
  const long long* hoff; int* idx_new; int* hot;
};

__global__ void k_row_fill_short(RowFillArgs R) {
  GRID_STRIDE(r, R.n_act) {
    const int o = R.old_of_new[r];
    const int b = R.rp[o], e = R.rp[o + 1];
    if (e - b > kShort) continue;
    const bool heavy = r < R.n_heavy;
    const int start = R.rp_new[r];
    int out = start;
    long long hout = heavy ? R.hoff[r] : 0;
    for (int q = b; q < e; ++q) {
      const int nv = R.lab[q];
      if (nv >= R.n_act) continue;                     // follower-less: folded into K
      if (heavy && nv < R.H) R.hot[hout++] = nv;
      else R.idx_new[out++] = nv;
    }
    if (out == start) R.idx_new[start] = R.n;
  }
}

__global__ void k_row_fill_long(RowFillArgs R, const int* list, int nlist) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int r = list[i];
    const int o = R.old_of_new[r];
    const int b = R.rp[o], e = R.rp[o + 1];
    const int start = R.rp_new[r];
    const bool heavy = r < R.n_heavy;
    int out = start;
    long long hout = heavy ? R.hoff[r] : 0;
    for (int q0 = b; q0 < e; q0 += 32) {
      const int q = q0 + lane;
      int nv = R.n_act;
      if (q < e) nv = R.lab[q];
      const bool act = nv < R.n_act;                  // follower-less <=> label >= n_act
      const bool is_hot = act && heavy && nv < R.H;
      const bool is_str = act && !is_hot;
      const unsigned m1 = __ballot_sync(kFull, is_str), m2 = __ballot_sync(kFull, is_hot);
      const unsigned below = (1u << lane) - 1u;
      if (is_str) R.idx_new[out + __popc(m1 & below)] = nv;
      if (is_hot) R.hot[hout + __popc(m2 & below)] = nv;
      out += __popc(m1);
      hout += __popc(m2);
    }
    if (lane == 0 && out == start) R.idx_new[start] = R.n;
  }
}

// warp per heavy row: entry keys (list << kEntBits) | (slot << sh) | (label % 2^sh);
// list = (panel * warps + owner warp of the slot) * nseg + segment.  The i-th hot
// follower of row r goes to slot rslot[r].x + i % rslot[r].y (round-robin virtual rows).
__global__ void k_heavy_keys(const int* hot, const long long* hoff, const int2* rslot,
                             const int* row_panel, const int* pslot_base, const unsigned char* slot_warp,
                             int n_heavy, int nseg, int sh, int warps, unsigned long long* keys) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_heavy) {
    const long long b = hoff[r], e = hoff[r + 1];
    const int2 sn = rslot[r];
    const int p = row_panel[r];
    const int base = pslot_base[p];
    // the i-th hot follower goes to slot k = i % nv (round robin); its key is written at the
    // row's position off_k + i / nv, so the row's keys are in slot order and a stable sort by
    // list alone leaves every list grouped by slot (rows, hence slots, ascend within a list)
    const long long h = e - b, qv = h / sn.y, rv = h % sn.y;
    for (long long q = b + lane; q < e; q += 32) {
      const unsigned lab = (unsigned)hot[q];
      const long long i = q - b, k = i % sn.y;
      const int slot = sn.x + (int)k;
      const unsigned long long list =
          ((unsigned long long)p * warps + slot_warp[base + slot]) * nseg + (lab >> sh);
      keys[b + k * qv + (k < rv ? k : rv) + i / sn.y] =
          (list << kEntBits) | ((unsigned long long)slot << sh) | (lab & ((1u << sh) - 1));
    }
  }
}

// first position of every list in the sorted keys (lower bound), lists 0..nlists
__global__ void k_list_start(const unsigned long long* keys, long long nk, long long nlists,
                             long long* lstart) {
  GRID_STRIDE(L, nlists + 1) {
    long long lo = 0, hi = nk;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if ((long long)(keys[mid] >> kEntBits) < L) lo = mid + 1; else hi = mid;
    }
    lstart[L] = lo;
  }
}

__global__ void k_list_padded(const long long* lstart, long long nlists, long long* plen) {
  GRID_STRIDE(L, nlists) plen[L] = (lstart[L + 1] - lstart[L] + 7) & ~7ll;   // 32-byte lists
}

__global__ void k_fill_u32(unsigned* p, long long n, unsigned v) { GRID_STRIDE(i, n) p[i] = v; }

__global__ void k_heavy_fill(const unsigned long long* keys, long long nk, const long long* lstart,
                             const long long* loff, unsigned* ent) {
  GRID_STRIDE(i, nk) {
    const unsigned long long k = keys[i];
    const long long L = (long long)(k >> kEntBits);
    const unsigned w = (unsigned)(k & ((1ull << kEntBits) - 1));
    ent[loff[L] + (i - lstart[L])] = w;
  }
}

// Bank-aware order inside every run of the staged-segment plan's lists.  k_heavy's gather
// instruction k of a chunk takes the k-th entry of 32 lanes -- list positions 256 c + 8 l + k
// -- and reads shared-memory word (entry & (2^sh - 1)) of a staged segment: 16 eight-byte bank
// pairs; each half-warp (a block of 128 list positions) costs as many wavefronts as lanes on
// its busiest pair.  The sums only need a slot's entries contiguous (one run per list), in any
// order: inside every 128-position block, each run's entries are laid out greedily, every
// position taking the run's remaining entry whose bank pair that instruction has used least
// in the block.  Measured: 5.5 -> 4.6 wavefronts per gather instruction at C5 (ideal 2);
// reordering whole runs as well gained nothing in a model of this greedy.
// Every block permutes only inside the portions of runs that lie in it (so every block is
// independent: one lane per block, a warp per list), whatever the run's length: portions of
// up to 32 entries by a scan of the remaining entries, longer ones (hub rows, whose sorted
// labels would otherwise stay in order) through 16 bank-pair buckets.  Deterministic.
constexpr int kBalBlock = 128;
// blocks of 128 positions of every list (the balance kernel's work items)
__global__ void k_list_blocks(const long long* lstart, long long nlists, long long* nb) {
  GRID_STRIDE(L, nlists) nb[L] = (lstart[L + 1] - lstart[L] + 127) >> 7;
}
// one thread per (list, 128-position block): bs = exclusive scan of the blocks per list
__global__ void __launch_bounds__(kBalBlock) k_heavy_balance(const unsigned* in, unsigned* out,
                                                             const long long* loff,
                                                             const long long* lstart,
                                                             const long long* bs,
                                                             long long nlists, int sh) {
  __shared__ unsigned long long cnt[8][kBalBlock];   // 16 four-bit counters per instruction k
  const int t = threadIdx.x;
  const long long total = bs[nlists];
  GRID_STRIDE(gb, total) {
    long long lo = 0, hi = nlists;                   // list L: bs[L] <= gb < bs[L + 1]
    while (hi - lo > 1) {
      const long long mid = lo + ((hi - lo) >> 1);
      if (bs[mid] <= gb) lo = mid; else hi = mid;
    }
    const long long L = lo;
    const long long b = loff[L];
    const int len_l = (int)(lstart[L + 1] - lstart[L]);
    const unsigned* src = in + b;
    unsigned* dst = out + b;
    const int B = (int)(gb - bs[L]);
    const int q0 = B << 7, q1 = min(q0 + 128, len_l);
    if (q1 == len_l)                                  // the list's null padding stays last
      for (long long i = b + len_l; i < loff[L + 1]; ++i) out[i] = in[i];
    for (int k = 0; k < 8; ++k) cnt[k][t] = 0ull;
    auto count = [&](int q, unsigned w) {
      const unsigned long long c = cnt[q & 7][t];
      const unsigned bk = w & 15;
      if (((c >> (4 * bk)) & 15ull) < 15ull) cnt[q & 7][t] = c + (1ull << (4 * bk));
    };
    // every maximal same-slot portion [q, r) of the block is permuted inside itself (the set of
    // entries at the block's positions does not change, so blocks stay independent -- also for
    // runs that cross block boundaries or span several blocks)
    int q = q0;
    while (q < q1) {
      const unsigned sl = src[q] >> sh;
      int r = q + 1;
      while (r < q1 && (src[r] >> sh) == sl) ++r;
      const int n = r - q;
      PSI_ASSERT(n >= 1 && n <= kBalBlock && q1 - q0 <= kBalBlock);
      if (n <= 32) {
        unsigned w[32];
        for (int j = 0; j < n; ++j) w[j] = src[q + j];
        unsigned used = 0;
        for (int i = 0; i < n; ++i) {
          const unsigned long long c = cnt[(q + i) & 7][t];
          int bj = 0, bv = 1 << 30;
          for (int j = 0; j < n; ++j) {
            if ((used >> j) & 1u) continue;
            const int v = (int)((c >> (4 * (w[j] & 15))) & 15ull);
            if (v < bv) { bv = v; bj = j; }
          }
          used |= 1u << bj;
          dst[q + i] = w[bj];
          count(q + i, w[bj]);
        }
      } else {
        // long portion (a hub's virtual row): its entries bucketed by bank pair, every position
        // taking an entry of the pair its instruction has used least in the block (ties: the
        // fullest bucket).  Sorted labels of a dense run otherwise put whole half-warps on two
        // or three pairs (a model: 3.1 -> 2.0 wavefronts per half-warp instruction).
        unsigned w[kBalBlock];
        unsigned char head[16], end[16];
        {
          unsigned char c16[16];
          for (int b16 = 0; b16 < 16; ++b16) c16[b16] = 0;
          for (int j = 0; j < n; ++j) ++c16[src[q + j] & 15];
          int a = 0;
          for (int b16 = 0; b16 < 16; ++b16) { head[b16] = (unsigned char)a; a += c16[b16]; end[b16] = (unsigned char)a; }
          unsigned char fill[16];
          for (int b16 = 0; b16 < 16; ++b16) fill[b16] = head[b16];
          for (int j = 0; j < n; ++j) { const unsigned e = src[q + j]; w[fill[e & 15]++] = e; }
        }
        for (int i = 0; i < n; ++i) {
          const unsigned long long c = cnt[(q + i) & 7][t];
          int bb = 0, bv = 1 << 30;
          for (int b16 = 0; b16 < 16; ++b16) {
            const int left = end[b16] - head[b16];
            if (left == 0) continue;
            const int v = ((int)((c >> (4 * b16)) & 15ull) << 8) - left;
            if (v < bv) { bv = v; bb = b16; }
          }
          PSI_ASSERT(head[bb] < end[bb]);
          const unsigned e = w[head[bb]++];
          dst[q + i] = e;
          count(q + i, e);
        }
      }
      q = r;
    }
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
                                  const int* nlead_old, double* a0, double* a1, double* g1,
                                  double* wt_new, double* d1, double* lam1, double* psi,
                                  int* nlead_new) {
  GRID_STRIDE(r, n) {
    const int o = old_of_new[r];
    a0[r] = a_old[o];
    nlead_new[r] = nlead_old[o];
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

// tile_row[k] = number of rows whose first edge lies before edge k*tile
__global__ void k_tile_rows(const int* rp, int n_act, int ntiles, int tile, int* tile_row) {
  GRID_STRIDE(k, ntiles + 1) {
    const long long e = k * (long long)tile;
    int lo = 0, hi = n_act;                 // first row r with rp[r] >= e
    while (lo < hi) {
      const int mid = lo + ((hi - lo) >> 1);      // no int overflow for n_act > 2^30
      if ((long long)rp[mid] < e) lo = mid + 1; else hi = mid;
    }
    tile_row[k] = lo;
  }
}

// rows whose edges fall in more than one tile
__global__ void k_split_flags(const int* rp, int n, int tile, unsigned char* flag) {
  GRID_STRIDE(r, n) flag[r] = (rp[r] / tile) != ((rp[r + 1] - 1) / tile) ? 1 : 0;
}

__global__ void k_split_fill(const int* rows, long long ns, const int* rp, int tile, int4* split) {
  GRID_STRIDE(s, ns) {
    const int r = rows[s];
    split[s] = make_int4(r, rp[r] / tile, (rp[r + 1] - 1) / tile, 0);
  }
}

// ------------------------------------------------------------------ host helpers

// RAII device buffer for temporaries, stream-ordered (dev_alloc: the library's own pool,
// which keeps freed temporaries reserved while a build runs, so the ingest's phases reuse
// each other's memory instead of re-mapping it)
thread_local cudaStream_t g_tmp_stream = nullptr;
// a view of scratch memory with Tmp's accessors
struct Span {
  void* p;
  template <class T> T* as() const { return (T*)p; }
};
struct Tmp {
  void* p = nullptr;
  ~Tmp() { reset(); }
  void reset() { if (p) cudaFreeAsync(p, g_tmp_stream); p = nullptr; }
  cudaError_t alloc(size_t bytes) {
    reset();
    return dev_alloc(&p, bytes ? bytes : 16, g_tmp_stream);
  }
  template <class T> T* as() const { return (T*)p; }
};

}  // namespace

// Per-device scratch for the build's two biggest short-lived buffers -- the staged host inputs
// (slot 0, psi_api.cu) and the transpose's sort arrays (slot 1) -- allocated with cudaMalloc
// outside the pool and kept across builds (like a library workspace): the pool then holds only
// the context's arrays and smaller temporaries, and repeated builds no longer stall on
// re-mapped pool memory around fragments (C5: 0.2 s transpose phases and 1-1.4 s builds now
// and then, measured).  psi_empty_cache() frees it.  The owning build holds the mutex.
namespace {
constexpr int kScratchDevices = 64;
struct DevScratch {
  std::mutex mu;
  void* p[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
};
DevScratch g_scratch[kScratchDevices];
}  // namespace

std::mutex* scratch_mutex(int dev) {
  return (dev >= 0 && dev < kScratchDevices) ? &g_scratch[dev].mu : nullptr;
}
cudaError_t scratch_get(int dev, int slot, size_t bytes, void** out) {
  if (dev < 0 || dev >= kScratchDevices || slot < 0 || slot > 1) return cudaErrorInvalidValue;
  DevScratch& S = g_scratch[dev];
  bytes = (bytes + 255) & ~(size_t)255;
  if (S.cap[slot] < bytes) {
    if (S.p[slot]) {
      cudaDeviceSynchronize();
      cudaFree(S.p[slot]);
      S.p[slot] = nullptr;
      S.cap[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&S.p[slot], bytes);
    if (e != cudaSuccess) { S.p[slot] = nullptr; return e; }
    S.cap[slot] = bytes;
  }
  *out = S.p[slot];
  return cudaSuccess;
}
void scratch_release(int dev) {
  if (dev < 0 || dev >= kScratchDevices) return;
  DevScratch& S = g_scratch[dev];
  std::lock_guard<std::mutex> lk(S.mu);
  for (int i = 0; i < 2; ++i) {
    if (S.p[i]) cudaFree(S.p[i]);
    S.p[i] = nullptr;
    S.cap[i] = 0;
  }
}

namespace {

int grid_for(long long work, int block, int cap = 148 * 16) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}


// indices r in [0, n) whose segment off[perm[r]] .. off[perm[r]+1] (perm = identity if NULL)
// is longer than thr; returns the count (stream-synchronising)
long long long_segments(const int* off, const int* perm, int n, int thr, cudaStream_t s,
                        Tmp& list) {
  Tmp flag, cnt, tmp;
  if (flag.alloc((size_t)std::max(n, 1)) != cudaSuccess || cnt.alloc(sizeof(long long)) != cudaSuccess ||
      list.alloc((size_t)std::max(n, 1) * sizeof(int)) != cudaSuccess)
    return -1;
  k_long_flags<<<grid_for(n, 256), 256, 0, s>>>(off, perm, n, thr, flag.as<unsigned char>());
  cub::CountingInputIterator<int> it(0);
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, it, flag.as<unsigned char>(), list.as<int>(),
                             cnt.as<long long>(), n, s);
  if (tmp.alloc(tb) != cudaSuccess) return -1;
  cub::DeviceSelect::Flagged(tmp.p, tb, it, flag.as<unsigned char>(), list.as<int>(),
                             cnt.as<long long>(), n, s);
  long long h = 0;
  if (cudaMemcpyAsync(&h, cnt.p, sizeof(long long), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return -1;
  return h;
}

// PSI_TRACE=1: per-phase wall time of the ingest on stderr (syncs the stream at each mark)
struct Trace {
  bool on = false;
  cudaStream_t s = nullptr;
  cudaEvent_t ev_last = nullptr;
  std::chrono::steady_clock::time_point t0, last;
  explicit Trace(cudaStream_t st) : s(st) {
    const char* e = getenv("PSI_TRACE");
    on = e && *e == '1';
    t0 = last = std::chrono::steady_clock::now();
    if (on) {
      cudaEventCreate(&ev_last);
      cudaEventRecord(ev_last, s);
    }
  }
  ~Trace() {
    if (ev_last) cudaEventDestroy(ev_last);
  }
  // host time since the last mark, and the device time between the two marks' events on the
  // stream (a phase whose host time exceeds its device time waited on the host side)
  void mark(const char* what) {
    if (!on) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, s);
    cudaStreamSynchronize(s);
    float dev_ms = 0.f;
    cudaEventElapsedTime(&dev_ms, ev_last, ev);
    cudaEventDestroy(ev_last);
    ev_last = ev;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[psi ingest] %-28s %9.2f ms  (device %9.2f ms, total %9.2f ms)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(), dev_ms,
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
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

namespace {

// Heavy-row plan (psi_heavy.cu): panels of <= out.heavy_slots slots and ~e_panel hot entries,
// virtual rows of <= vmax entries, contiguous slot ranges per consumer warp balanced by
// entries; then the entry lists (panel, segment, warp) sorted by (slot, label).
//
// Host part of the plan (panels, virtual-row slots, per-warp slot ranges) from the hot-entry
// count of every heavy row.  Pure host work: psi ingest runs it on a helper thread while the
// device builds the edge stream.  Its buffers persist (a fresh multi-MB vector costs ~1 page
// fault per 4 KB on every build, ~40 ms at C5, measured) and are guarded by a mutex.
struct HeavyHostPlan {
  std::mutex mu;
  std::vector<long long> hc, cum_h, pent;       // pent: entries of every panel of the plan
  std::vector<int> prow, row_panel, pslot_base, wslot, cum_nv;
  int sel_num = 100, sel_cap = 0;              // panel shape chosen by the search
  int sel_tail = 0, sel_from = 0;              //   tail target (% of the chosen one) from sel_from % of the entries
  long long sim_base = 0, sim_best = 0;        //   and the simulated makespans (entries)
  std::vector<int2> rslot;
  std::vector<unsigned char> slot_warp;
  int npanels = 0;
};
HeavyHostPlan& heavy_host_plan() {
  static HeavyHostPlan p;
  return p;
}

// Panel shape search (search != 0): k_heavy's CTAs claim the panels in index order, so the sweep
// lasts as long as the busiest CTA -- with ~1 full-size panel per SM a handful of panels over
// the SM count is a second wave (C4: 162 panels on 148 SMs, k_heavy 0.445 ms for 0.25 ms of
// mean work).  The entry target and the slot cap of a panel are chosen from a few candidates by
// simulating that claim order with cost(panel) = entries + nseg * kPanelSegCost (the streamed
// segments of a panel cost about as much as 3000 entries each: C5, 366 vs 461 panels).  The
// default shape is planned first and stays unless a candidate's makespan is >= 4 % shorter
// (the model's error); only then the plan is made a second time.
constexpr long long kPanelSegCost = 3000;
long long heavy_makespan(const std::vector<long long>& cum_h, const std::vector<int>& cum_nv, int NH,
                         long long e_panel, int slot_cap, int sms, long long fixed,
                         std::vector<long long>& busy, long long e_tail = 0, long long tail_from = 0,
                         int* npan = nullptr) {
  busy.assign(sms, 0);                    // a binary min-heap of the CTAs' finish times
  long long makespan = 0;
  int start = 0, np = 0;
  while (start < NH) {
    // the panel takes rows [start, end): the first row always, then while both caps hold
    const long long h_lim = cum_h[start] + (e_tail > 0 && cum_h[start] >= tail_from ? e_tail : e_panel);
    const long long v_lim = (long long)cum_nv[start] + slot_cap;
    // largest end with cum_h[end] <= h_lim and cum_nv[end] <= v_lim: gallop, then bisect (local)
    int lo = start + 1, hi = NH;
    for (int step = 1; lo + step < NH; step <<= 1) {
      if (cum_h[lo + step] <= h_lim && cum_nv[lo + step] <= v_lim) {
        lo += step;
      } else {
        hi = lo + step - 1;
        break;
      }
    }
    while (lo < hi) {
      const int mid = lo + ((hi - lo + 1) >> 1);
      if (cum_h[mid] <= h_lim && cum_nv[mid] <= v_lim) lo = mid; else hi = mid - 1;
    }
    const int end = lo;
    const long long cost = cum_h[end] - cum_h[start] + fixed;
    // earliest-free CTA takes it: replace the heap's root and sift down
    long long t = busy[0] + cost;
    makespan = std::max(makespan, t);
    int i = 0;
    for (;;) {
      int c = 2 * i + 1;
      if (c >= sms) break;
      if (c + 1 < sms && busy[c + 1] < busy[c]) ++c;
      if (busy[c] >= t) break;
      busy[i] = busy[c];
      i = c;
    }
    busy[i] = t;
    start = end;
    ++np;
  }
  if (npan) *npan = np;
  return makespan;
}

// list scheduling of panel costs in index order on sms CTAs (the claim order of k_heavy)
long long claim_makespan(const std::vector<long long>& cost, int sms, std::vector<long long>& busy) {
  busy.assign(sms, 0);
  long long makespan = 0;
  for (long long c : cost) {
    const long long t = busy[0] + c;
    makespan = std::max(makespan, t);
    int i = 0;
    for (;;) {
      int k = 2 * i + 1;
      if (k >= sms) break;
      if (k + 1 < sms && busy[k + 1] < busy[k]) ++k;
      if (busy[k] >= t) break;
      busy[i] = busy[k];
      i = k;
    }
    busy[i] = t;
  }
  return makespan;
}

// One pass of the plan: panels closed at slot_cap slots or e_panel entries (e_tail for the
// panels that start after tail_from entries, if e_tail > 0).
void plan_heavy_pass(HeavyHostPlan& P, int NH, long long n_ent, int HW, int SLOTS, long long e_panel,
                     int slot_cap, long long e_tail, long long tail_from) {
  const std::vector<long long>& hc = P.hc;
  const long long vmax = std::max<long long>(e_panel / (2 * HW), 64);
  std::vector<int>& prow = P.prow;
  std::vector<int>& row_panel = P.row_panel;
  std::vector<int>& pslot_base = P.pslot_base;
  std::vector<int>& wslot = P.wslot;
  std::vector<int2>& rslot = P.rslot;
  std::vector<unsigned char>& slot_warp = P.slot_warp;
  prow.assign(1, 0);
  pslot_base.assign(1, 0);
  wslot.clear();
  P.pent.clear();
  row_panel.resize(NH);
  rslot.resize(NH);
  slot_warp.clear();
  slot_warp.reserve((size_t)NH + (size_t)(n_ent / vmax) + 1);
  std::vector<long long> slot_w(SLOTS);          // entries of each slot of the open panel
  std::vector<int> ws(HW + 1);
  int nslots = 0;
  long long p_ent = 0, tot_ent = 0;            // entries of the open panel / of all rows so far
  auto close_panel = [&](int r_end) {
    long long T = 0;
    for (int k = 0; k < nslots; ++k) T += slot_w[k];
    std::fill(ws.begin(), ws.end(), nslots);
    ws[0] = 0;
    long long acc = 0;
    int w = 1;
    for (int k = 0; k < nslots && w < HW; ++k) {
      acc += slot_w[k];
      while (w < HW && acc * HW >= T * w) ws[w++] = k + 1;
    }
    for (int o = 0; o < HW; ++o) slot_warp.insert(slot_warp.end(), ws[o + 1] - ws[o], (unsigned char)o);
    wslot.insert(wslot.end(), ws.begin(), ws.end());
    prow.push_back(r_end);
    pslot_base.push_back(pslot_base.back() + nslots);
    P.pent.push_back(p_ent);
    nslots = 0;
    p_ent = 0;
  };
  for (int r = 0; r < NH; ++r) {
    const long long h = hc[r];
    long long nv = h > 0 ? (h + vmax - 1) / vmax : 0;
    if (nv > SLOTS) nv = SLOTS;
    const long long e_cur = e_tail > 0 && tot_ent - p_ent >= tail_from ? e_tail : e_panel;
    if (r > prow.back() && (nslots + nv > slot_cap || p_ent + h > e_cur)) close_panel(r);
    rslot[r] = make_int2(nslots, (int)nv);
    row_panel[r] = (int)prow.size() - 1;
    if (nv > 0) {
      const long long q = h / nv, rem = h % nv;  // slot k of the row: q (+1 for k < rem) entries
      for (long long k = 0; k < nv; ++k) slot_w[nslots++] = q + (k < rem ? 1 : 0);
    }
    p_ent += h;
    tot_ent += h;
  }
  close_panel(NH);
  P.npanels = (int)prow.size() - 1;
}

void plan_heavy_host(HeavyHostPlan& P, int NH, long long n_ent, int HW, int SLOTS, int sms, int pps,
                     int nseg, int search) {
  const std::vector<long long>& hc = P.hc;
  const long long e_panel = std::max<long long>((n_ent + (long long)pps * sms - 1) / ((long long)pps * sms), 32768);
  plan_heavy_pass(P, NH, n_ent, HW, SLOTS, e_panel, SLOTS, 0, 0);      // the default shape
  P.sel_num = 100;
  P.sel_cap = SLOTS;
  P.sel_tail = P.sel_from = 0;
  P.sim_base = P.sim_best = 0;
  if (!search || NH <= 0) return;
  // its makespan under the claim order, from the panels just made; nothing to gain where that is
  // within 8 % of an even split of the work (C5: 6 % -- no search, no second pass)
  const long long fixed = (long long)nseg * kPanelSegCost;
  std::vector<long long> busy, cost(P.pent);
  for (long long& c : cost) c += fixed;
  const long long base = claim_makespan(cost, sms, busy);
  P.sim_base = P.sim_best = base;
  // (PSI_HEAVY_SEARCH_GATE / PSI_HEAVY_SEARCH_GAIN: measurement knobs for the two thresholds, %)
  const int gate = env_int("PSI_HEAVY_SEARCH_GATE", 8), gain = env_int("PSI_HEAVY_SEARCH_GAIN", 4);
  if (base * 100 <= (n_ent + fixed * P.npanels) / sms * (100 + gate)) return;
  const long long vmax0 = std::max<long long>(e_panel / (2 * HW), 64);
  std::vector<long long>& cum_h = P.cum_h;
  std::vector<int>& cum_nv = P.cum_nv;
  cum_h.resize((size_t)NH + 1);
  cum_nv.resize((size_t)NH + 1);
  cum_h[0] = 0;
  cum_nv[0] = 0;
  for (int r = 0; r < NH; ++r) {
    const long long h = hc[r];
    cum_h[r + 1] = cum_h[r] + h;
    cum_nv[r + 1] = cum_nv[r] + (int)std::min<long long>(h > 0 ? (h + vmax0 - 1) / vmax0 : 0, SLOTS);
  }
  long long best = base;
  static const int kCapEighths[] = {8, 6, 5, 4, 3};
  for (int num = 150; num >= 50; num -= 5)                    // entry target, % of the default
    for (int d : kCapEighths) {                               // slot cap = SLOTS * d / 8
      const long long e = std::max<long long>(e_panel * num / 100, 32768);
      const int cap = SLOTS * d / 8;
      const long long m = heavy_makespan(cum_h, cum_nv, NH, e, cap, sms, fixed, busy);
      if (m < best && m * 100 <= base * (100 - gain)) {
        best = m;
        P.sel_num = num;
        P.sel_cap = cap;
      }
    }
  // a tapered tail: the panels that start after tail_from entries take a smaller target (the
  // last panels claimed decide how uneven the CTAs finish)
  const long long e_sel = std::max<long long>(e_panel * P.sel_num / 100, 32768);
  for (int from = 50; from <= 90; from += 10)                 // % of the entries before the tail
    for (int tnum = 70; tnum >= 20; tnum -= 10) {             // tail target, % of the chosen one
      const long long et = std::max<long long>(e_sel * tnum / 100, 32768);
      const long long m = heavy_makespan(cum_h, cum_nv, NH, e_sel, P.sel_cap, sms, fixed, busy, et,
                                         n_ent / 100 * from);
      if (m < best && m * 100 <= base * (100 - gain)) {
        best = m;
        P.sel_tail = tnum;
        P.sel_from = from;
      }
    }
  P.sim_best = best;
  if (best < base)
    plan_heavy_pass(P, NH, n_ent, HW, SLOTS, e_sel, P.sel_cap,
                    P.sel_tail > 0 ? std::max<long long>(e_sel * P.sel_tail / 100, 32768) : 0,
                    n_ent / 100 * P.sel_from);
}

// Heavy-row plan (psi_heavy.cu), device part: the host plan P (already made) uploaded, then the
// entry lists (panel, segment, warp) sorted by (slot, label) and bank-balanced.
int build_heavy_plan(IngestOut& out, int NH, long long n_ent, Tmp& hot, Tmp& hoff,
                     HeavyHostPlan& P, cudaStream_t s, Trace& tr, char* msg, size_t msg_len) {
  const int nseg = out.nseg;
  const int sh = out.heavy_seg_shift;
  const int HW = out.heavy_warps, SLOTS = out.heavy_slots;
  const std::vector<int>& prow = P.prow;
  const std::vector<int>& row_panel = P.row_panel;
  const std::vector<int>& pslot_base = P.pslot_base;
  const std::vector<int>& wslot = P.wslot;
  const std::vector<int2>& rslot = P.rslot;
  const std::vector<unsigned char>& slot_warp = P.slot_warp;
  const int npanels = P.npanels;
  out.npanels = npanels;
  out.heavy_entries = n_ent;

  IG_CK(dev_alloc(&out.h_prow, prow.size() * sizeof(int), s));
  IG_CK(dev_alloc(&out.h_rslot, (size_t)NH * sizeof(int2), s));
  IG_CK(dev_alloc(&out.h_wslot, wslot.size() * sizeof(int), s));
  IG_CK(cudaMemcpyAsync(out.h_prow, prow.data(), prow.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  IG_CK(cudaMemcpyAsync(out.h_rslot, rslot.data(), (size_t)NH * sizeof(int2), cudaMemcpyHostToDevice, s));
  IG_CK(cudaMemcpyAsync(out.h_wslot, wslot.data(), wslot.size() * sizeof(int), cudaMemcpyHostToDevice, s));

  const long long nlists = (long long)npanels * nseg * HW;
  IG_CK(dev_alloc(&out.h_loff, (size_t)(nlists + 1) * sizeof(long long), s));
  Tmp keys, keys2, rpan, psb, sw, lstart, plen, scan_tmp, sort_tmp;
  IG_CK(keys.alloc((size_t)std::max<long long>(n_ent, 1) * 8));
  IG_CK(keys2.alloc((size_t)std::max<long long>(n_ent, 1) * 8));
  IG_CK(rpan.alloc((size_t)NH * sizeof(int)));
  IG_CK(psb.alloc(pslot_base.size() * sizeof(int)));
  IG_CK(sw.alloc(std::max<size_t>(slot_warp.size(), 1)));
  IG_CK(cudaMemcpyAsync(rpan.p, row_panel.data(), (size_t)NH * sizeof(int), cudaMemcpyHostToDevice, s));
  IG_CK(cudaMemcpyAsync(psb.p, pslot_base.data(), pslot_base.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (!slot_warp.empty())
    IG_CK(cudaMemcpyAsync(sw.p, slot_warp.data(), slot_warp.size(), cudaMemcpyHostToDevice, s));
  k_heavy_keys<<<grid_for((long long)NH * 32, 256), 256, 0, s>>>(
      hot.as<int>(), hoff.as<long long>(), out.h_rslot, rpan.as<int>(), psb.as<int>(),
      sw.as<unsigned char>(), NH, nseg, sh, HW, keys.as<unsigned long long>());
  int end_bit = kEntBits;
  while ((1LL << (end_bit - kEntBits)) <= nlists) ++end_bit;
  cub::DoubleBuffer<unsigned long long> kb(keys.as<unsigned long long>(), keys2.as<unsigned long long>());
  if (n_ent > 0) {
    size_t tb = 0;
    // by list only: k_heavy_keys wrote every row's keys in slot order and rows ascend within a
    // list, so the stable sort leaves each list grouped by slot, each slot's entries in the
    // hot-list order (fixed, so the sums stay deterministic) -- 3 radix passes instead of 5
    IG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, kb, (int)n_ent, kEntBits, end_bit, s));
    IG_CK(sort_tmp.alloc(tb));
    IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp.p, tb, kb, (int)n_ent, kEntBits, end_bit, s));
  }
  tr.mark("  heavy: keys + sort");
  IG_CK(lstart.alloc((size_t)(nlists + 1) * sizeof(long long)));
  IG_CK(plen.alloc((size_t)(nlists + 1) * sizeof(long long)));
  k_list_start<<<grid_for(nlists + 1, 256), 256, 0, s>>>(kb.Current(), n_ent, nlists,
                                                        lstart.as<long long>());
  IG_CK(cudaMemsetAsync(plen.as<long long>() + nlists, 0, sizeof(long long), s));
  k_list_padded<<<grid_for(nlists, 256), 256, 0, s>>>(lstart.as<long long>(), nlists,
                                                      plen.as<long long>());
  size_t sb = 0;
  IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, plen.as<long long>(), out.h_loff, nlists + 1, s));
  IG_CK(scan_tmp.alloc(sb));
  IG_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, sb, plen.as<long long>(), out.h_loff, nlists + 1, s));
  long long total = 0;
  IG_CK(cudaMemcpyAsync(&total, out.h_loff + nlists, sizeof(long long), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  IG_CK(dev_alloc(&out.h_ent, (size_t)std::max<long long>(total, 4) * sizeof(unsigned), s));
  k_fill_u32<<<grid_for(total, 256), 256, 0, s>>>(out.h_ent, total, (unsigned)SLOTS << sh);
  k_heavy_fill<<<grid_for(n_ent, 256), 256, 0, s>>>(kb.Current(), n_ent, lstart.as<long long>(),
                                                   out.h_loff, out.h_ent);
  tr.mark("  heavy: lists + fill");
  if (env_int("PSI_HEAVY_BALANCE", 1) != 0) {
    unsigned* bal = nullptr;
    IG_CK(dev_alloc(&bal, (size_t)std::max<long long>(total, 4) * sizeof(unsigned), s));
    Tmp nb, bs, bscan;
    IG_CK(nb.alloc((size_t)(nlists + 1) * sizeof(long long)));
    IG_CK(bs.alloc((size_t)(nlists + 1) * sizeof(long long)));
    IG_CK(cudaMemsetAsync(nb.as<long long>() + nlists, 0, sizeof(long long), s));
    k_list_blocks<<<grid_for(nlists, 256), 256, 0, s>>>(lstart.as<long long>(), nlists,
                                                        nb.as<long long>());
    size_t bb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, bb, nb.as<long long>(), bs.as<long long>(),
                                        nlists + 1, s));
    IG_CK(bscan.alloc(bb));
    IG_CK(cub::DeviceScan::ExclusiveSum(bscan.p, bb, nb.as<long long>(), bs.as<long long>(),
                                        nlists + 1, s));
    k_heavy_balance<<<grid_for((n_ent >> 7) + nlists, kBalBlock, 148 * 64), kBalBlock, 0, s>>>(
        out.h_ent, bal, out.h_loff, lstart.as<long long>(), bs.as<long long>(), nlists, sh);
    IG_CK(cudaGetLastError());
    IG_CK(cudaFreeAsync(out.h_ent, s));
    out.h_ent = bal;
  }
  IG_CK(cudaStreamSynchronize(s));
  IG_CK(cudaGetLastError());
  return PSI_OK;
}

}  // namespace

// ---- batch (nprof > 1): folded constants and interleaved vectors of every profile
// K_j^(p) = sum of a^(p) over the follower-less followers of row j, in input order -- the
// summation of k_row_count_short / _long, so profile 0 gets the single-profile K bit for bit.
__global__ void k_fold_short(const int* rp, const int* idx, const int* old_of_new,
                             const int* new_of_old, const double* a_old, int n_act, double* K) {
  GRID_STRIDE(r, n_act) {
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    if (e - b > kShort) continue;
    double k = 0.0;
    for (int q = b; q < e; ++q) {
      const int v = idx[q];
      if (new_of_old[v] >= n_act) k += a_old[v];
    }
    K[r] = k;
  }
}
__global__ void k_fold_long(const int* list, int nlist, const int* rp, const int* idx,
                            const int* old_of_new, const int* new_of_old, const double* a_old,
                            int n_act, double* K) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlist) {
    const int r = list[i];
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    double k = 0.0;
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      if (new_of_old[v] >= n_act) k += a_old[v];
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) k += __shfl_xor_sync(kFull, k, sh);
    if (lane == 0) K[r] = k;
  }
}
// profile p into lane p % kBP of group p / kBP (the k_permute_vectors arithmetic)
__global__ void k_permute_b(const int* old_of_new, long long n, int n_act, int p,
                            const double* a_old, const double* g_old, const double* wt_old,
                            const double* d_old, const double* lam, const double* K,
                            IngestOut o) {
  const int gi = p / kBP, l = p % kBP;
  GRID_STRIDE(r, n) {
    const int u = old_of_new[r];
    o.b_a0[((size_t)gi * n + r) * kBP + l] = a_old[u];
    if (r < n_act) {
      const size_t q = ((size_t)gi * n_act + r) * kBP + l;
      const double k = K[r];
      o.b_a1[q] = fma(g_old[u], k, a_old[u]);
      o.b_g[q] = g_old[u];
      o.b_wt[q] = wt_old[u];
      o.b_d1[q] = fma(lam[u], k, d_old[u]);
      o.b_lam[q] = lam[u];
    } else {
      o.b_psi[((size_t)gi * n + r) * kBP + l] = d_old[u] / (double)n;
    }
  }
}

// overlapped sweep: bit r = heavy row r is a split row (finished by k_fix's split path)
__global__ void k_heavy_split_bits(const int4* split, long long ns, int n_heavy, unsigned* bits) {
  GRID_STRIDE(i, ns) {
    const int r = split[i].x;
    if (r < n_heavy) atomicOr(bits + (r >> 5), 1u << (r & 31));
  }
}

__global__ void k_long_split_flags(const int4* split, long long ns, unsigned char* flag) {
  GRID_STRIDE(i, ns) flag[i] = (split[i].z - split[i].y) > kLongSpan;
}

// ------------------------------------------------------------------ 8. sliced-ELL layout
// (SellPlan, psi_internal.cuh; swept by k_sell).  Windows are runs of 32-row blocks, cut where
// the cumulative stream length crosses a multiple of `ecap` edges or the row count reaches
// 2^shift, so one window is a bounded work item.  Sort key of active row r inside window w:
// w << 32 | (2047 - d') << 11 | (r - first row of w), d' = stream length (0 for long rows and
// the padding rows of the last block) -- descending length, ascending row on ties.
__global__ void k_sell_deg(const int* rp, int NA, long long na_pad, int lmax, int* dd,
                           unsigned char* lflag) {
  GRID_STRIDE(i, na_pad) {
    int d = 0;
    if (i < NA) {
      d = rp[i + 1] - rp[i];
      const bool lg = d > lmax;
      lflag[i] = lg ? 1 : 0;
      if (lg) d = 0;
    }
    dd[i] = d;
  }
}

__global__ void k_sell_blocksum(const int* dd, long long nblk, long long* bsum) {
  GRID_STRIDE(b, nblk) {
    long long t = 0;
    for (int j = 0; j < 32; ++j) t += dd[b * 32 + j];
    bsum[b] = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) bsum[nblk] = 0;
}

// block b starts a window: the first block, every 2^shift rows, or where the edges before it
// cross a multiple of ecap (pre = exclusive prefix of the block sums)
__global__ void k_sell_wflag(const long long* pre, long long nblk, int shift, long long ecap,
                             int* flag) {
  GRID_STRIDE(b, nblk) {
    const bool f = b == 0 || ((b << 5) & ((1LL << shift) - 1)) == 0 ||
                   pre[b] / ecap != pre[b - 1] / ecap;
    flag[b] = f ? 1 : 0;
  }
}

__global__ void k_sell_wrow(const int* flag, const int* wid, long long nblk, int* wrow) {
  GRID_STRIDE(b, nblk) if (flag[b]) wrow[wid[b] - 1] = (int)(b << 5);
}

__global__ void k_sell_keys(const int* dd, const int* wid, const int* wrow, long long na_pad,
                            unsigned long long* keys) {
  GRID_STRIDE(i, na_pad) {
    const int w = wid[i >> 5] - 1;
    const unsigned long long loc = (unsigned long long)(i - wrow[w]);
    keys[i] = ((unsigned long long)w << 32) | ((unsigned long long)(2047 - dd[i]) << 11) | loc;
  }
}

// sorted position i -> (slice i / 32, lane i % 32): its row (for the fill) and, per row, its
// position inside its window (ipos: where k_sell leaves the row's sum; 0xffff for long rows,
// which k_fix finishes from their pieces); the width of every slice is the length of its
// first (longest) row
__global__ void k_sell_perm(const unsigned long long* sorted, long long na_pad, const int* wrow,
                            unsigned short* ipos, int* row_of_pos, unsigned* width) {
  GRID_STRIDE(i, na_pad) {
    const unsigned long long k = sorted[i];
    const int w = (int)(k >> 32);
    const int d = 2047 - (int)((k >> 11) & 2047u);
    const int r = wrow[w] + (int)(k & 2047u);
    ipos[r] = d > 0 ? (unsigned short)(i - wrow[w]) : (unsigned short)0xffff;
    row_of_pos[i] = d > 0 ? r : -1;
    if ((i & 31) == 0) width[i >> 5] = (unsigned)d;
  }
}

// window w's index block: wstep[w] .. wstep[w + 1] steps (its slices' widths summed, rounded up
// to a multiple of 8); ksteps[w] = the steps of its slices
__global__ void k_sell_wsteps(const unsigned* soff, const int* wrow, int nwin, unsigned* ksteps) {
  GRID_STRIDE(w, nwin) {
    const unsigned k = soff[wrow[w + 1] >> 5] - soff[wrow[w] >> 5];
    ksteps[w] = (k + 7u) & ~7u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ksteps[nwin] = 0;
}

__global__ void k_fill_u32v(unsigned* p, long long n, unsigned v) { GRID_STRIDE(i, n) p[i] = v; }

// warp per slice: lane l writes its row's followers (flag bit cleared) as steps k0 .. k0+d-1 of
// its stream through the window, step k at word ((k / 8) * 32 + l) * 8 + k % 8 of the window's
// block (one 32-byte load per lane per 8 steps in k_sell); the sentinel label below a shorter
// row's end
__global__ void k_sell_fill(const int* row_of_pos, const unsigned* soff, long long nslices,
                            const int* wid, const int* wrow, const unsigned* wstep, const int* rp,
                            const unsigned* edges, unsigned pad, unsigned* words) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(s, nslices) {
    const unsigned o0 = soff[s], wd = soff[s + 1] - o0;
    if (wd == 0) continue;
    const int w = wid[s] - 1;
    const unsigned k0 = o0 - soff[wrow[w] >> 5];
    const int r = row_of_pos[s * 32 + lane];
    int b = 0, d = 0;
    if (r >= 0) {
      b = rp[r];
      d = rp[r + 1] - b;
    }
    unsigned* out = words + (size_t)wstep[w] * 32;
    for (unsigned j = 0; j < wd; ++j) {
      const unsigned k = k0 + j;
      out[((size_t)(k >> 3) * 32 + lane) * 8 + (k & 7)] = (int)j < d ? (edges[b + j] & ~kRowFlag) : pad;
    }
  }
}

// long row i: its length and number of pieces
__global__ void k_sell_long_len(const int* lrow, int nlong, const int* rp, int plen, long long* len,
                                int* np) {
  GRID_STRIDE(i, nlong) {
    const int r = lrow[i];
    const int d = rp[r + 1] - rp[r];
    len[i] = d;
    np[i] = (d + plen - 1) / plen;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { len[nlong] = 0; np[nlong] = 0; }
}

// warp per long row: copy its followers (flag cleared) and write its pieces
__global__ void k_sell_long_fill(const int* lrow, int nlong, const int* rp, const unsigned* edges,
                                 const long long* loff, const int* lp0, int plen, unsigned* lwords,
                                 int2* piece) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(i, nlong) {
    const int r = lrow[i];
    const int b = rp[r], d = rp[r + 1] - b;
    const long long o = loff[i];
    for (int j = lane; j < d; j += 32) lwords[o + j] = edges[b + j] & ~kRowFlag;
    for (int q = lane; q * plen < d; q += 32)
      piece[lp0[i] + q] = make_int2((int)(o + (long long)q * plen), min(plen, d - q * plen));
  }
}

// Sliced-ELL copy of the edge stream (rows rp / flagged words edges, NA rows) for k_sell.
// max_pad > 0: give up (rejected = true, nothing kept) when the slices' index words would
// exceed max_pad x the edge stream's m_act words -- checked before the words are filled.
int build_sell(IngestOut& out, const int* rp, int NA, long long n, cudaStream_t s, char* msg,
               size_t msg_len, double max_pad, bool* rejected) {
  *rejected = false;
  const int shift = out.sell_shift;
  const long long nblk = ((long long)NA + 31) / 32;
  const long long na_pad = nblk * 32;
  const long long nsl = nblk;
  const long long ecap = (long long)out.sell_kcap * 32;
  out.sell_nslices = nsl;
  IG_CK(dev_alloc(&out.s_ipos, (size_t)std::max(na_pad, 1LL) * sizeof(unsigned short), s));
  IG_CK(dev_alloc(&out.s_off, (size_t)(nsl + 1) * sizeof(unsigned), s));
  Tmp dd, bsum, pre, wflag, wid, keys, sorted, lflag, rop, width, tmp, cnt;
  IG_CK(dd.alloc((size_t)std::max(na_pad, 1LL) * sizeof(int)));
  IG_CK(bsum.alloc((size_t)(nblk + 1) * sizeof(long long)));
  IG_CK(pre.alloc((size_t)(nblk + 1) * sizeof(long long)));
  IG_CK(wflag.alloc((size_t)std::max(nblk, 1LL) * sizeof(int)));
  IG_CK(wid.alloc((size_t)std::max(nblk, 1LL) * sizeof(int)));
  IG_CK(keys.alloc((size_t)std::max(na_pad, 1LL) * 8));
  IG_CK(sorted.alloc((size_t)std::max(na_pad, 1LL) * 8));
  IG_CK(lflag.alloc((size_t)std::max(NA, 1)));
  IG_CK(rop.alloc((size_t)std::max(na_pad, 1LL) * sizeof(int)));
  IG_CK(width.alloc((size_t)(nsl + 1) * sizeof(unsigned)));
  IG_CK(cnt.alloc(sizeof(long long)));
  IG_CK(cudaMemsetAsync(width.p, 0, (size_t)(nsl + 1) * sizeof(unsigned), s));
  int nwin = 0;
  long long nlong = 0;
  if (na_pad > 0) {
    k_sell_deg<<<grid_for(na_pad, 256), 256, 0, s>>>(rp, NA, na_pad, out.sell_lmax, dd.as<int>(),
                                                     lflag.as<unsigned char>());
    k_sell_blocksum<<<grid_for(nblk, 256), 256, 0, s>>>(dd.as<int>(), nblk, bsum.as<long long>());
    size_t tb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, bsum.as<long long>(), pre.as<long long>(),
                                        nblk + 1, s));
    size_t tb2 = 0;
    IG_CK(cub::DeviceScan::InclusiveSum(nullptr, tb2, wflag.as<int>(), wid.as<int>(), nblk, s));
    IG_CK(tmp.alloc(std::max(tb, tb2)));
    IG_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, bsum.as<long long>(), pre.as<long long>(),
                                        nblk + 1, s));
    k_sell_wflag<<<grid_for(nblk, 256), 256, 0, s>>>(pre.as<long long>(), nblk, shift, ecap,
                                                     wflag.as<int>());
    IG_CK(cub::DeviceScan::InclusiveSum(tmp.p, tb2, wflag.as<int>(), wid.as<int>(), nblk, s));
    IG_CK(cudaMemcpyAsync(&nwin, wid.as<int>() + nblk - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
  }
  out.sell_nwin = nwin;
  IG_CK(dev_alloc(&out.s_wrow, (size_t)(nwin + 1) * sizeof(int), s));
  {
    const int end_row = (int)na_pad;
    IG_CK(cudaMemcpyAsync(out.s_wrow + nwin, &end_row, sizeof(int), cudaMemcpyHostToDevice, s));
  }
  if (na_pad > 0) {
    k_sell_wrow<<<grid_for(nblk, 256), 256, 0, s>>>(wflag.as<int>(), wid.as<int>(), nblk, out.s_wrow);
    k_sell_keys<<<grid_for(na_pad, 256), 256, 0, s>>>(dd.as<int>(), wid.as<int>(), out.s_wrow, na_pad,
                                                      keys.as<unsigned long long>());
    int wbits = 1;
    while ((1LL << wbits) < nwin) ++wbits;
    size_t tb = 0;
    IG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<unsigned long long>(),
                                         sorted.as<unsigned long long>(), (int)na_pad, 0,
                                         32 + wbits, s));
    IG_CK(tmp.alloc(tb));
    IG_CK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.as<unsigned long long>(),
                                         sorted.as<unsigned long long>(), (int)na_pad, 0,
                                         32 + wbits, s));
    k_sell_perm<<<grid_for(na_pad, 256), 256, 0, s>>>(sorted.as<unsigned long long>(), na_pad,
                                                      out.s_wrow, out.s_ipos, rop.as<int>(),
                                                      width.as<unsigned>());
  }
  {
    size_t tb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, width.as<unsigned>(), out.s_off, nsl + 1, s));
    IG_CK(tmp.alloc(tb));
    IG_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, width.as<unsigned>(), out.s_off, nsl + 1, s));
  }
  // window index blocks (steps rounded up to 8 per window)
  IG_CK(dev_alloc(&out.s_wstep, (size_t)(nwin + 1) * sizeof(unsigned), s));
  unsigned tot32 = 0;
  {
    Tmp ks;
    IG_CK(ks.alloc((size_t)(nwin + 1) * sizeof(unsigned)));
    k_sell_wsteps<<<grid_for(nwin + 1, 256), 256, 0, s>>>(out.s_off, out.s_wrow, nwin, ks.as<unsigned>());
    size_t tb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, ks.as<unsigned>(), out.s_wstep, nwin + 1, s));
    IG_CK(tmp.alloc(tb));
    IG_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, ks.as<unsigned>(), out.s_wstep, nwin + 1, s));
    IG_CK(cudaMemcpyAsync(&tot32, out.s_wstep + nwin, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
  }
  if (max_pad > 0.0 && (double)tot32 * 32.0 > max_pad * (double)out.m_act) {
    for (void** p : {(void**)&out.s_ipos, (void**)&out.s_off, (void**)&out.s_wrow, (void**)&out.s_wstep}) {
      IG_CK(cudaFreeAsync(*p, s));
      *p = nullptr;
    }
    out.sell_nwin = 0;
    out.sell_nslices = 0;
    *rejected = true;
    return PSI_OK;
  }
  // long rows
  Tmp lrow_all;
  IG_CK(lrow_all.alloc((size_t)std::max(NA, 1) * sizeof(int)));
  if (NA > 0) {
    cub::CountingInputIterator<int> it(0);
    size_t tb = 0;
    IG_CK(cub::DeviceSelect::Flagged(nullptr, tb, it, lflag.as<unsigned char>(), lrow_all.as<int>(),
                                     cnt.as<long long>(), NA, s));
    IG_CK(tmp.alloc(tb));
    IG_CK(cub::DeviceSelect::Flagged(tmp.p, tb, it, lflag.as<unsigned char>(), lrow_all.as<int>(),
                                     cnt.as<long long>(), NA, s));
    IG_CK(cudaMemcpyAsync(&nlong, cnt.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
  }
  IG_CK(cudaStreamSynchronize(s));
  out.sell_words = (long long)tot32 * 32;
  out.sell_nlong = (int)nlong;
  IG_CK(dev_alloc(&out.s_words, (size_t)std::max(out.sell_words, 1LL) * sizeof(unsigned), s));
  if (out.sell_words > 0)
    k_fill_u32v<<<grid_for(out.sell_words, 256), 256, 0, s>>>(out.s_words, out.sell_words, (unsigned)n);
  if (nsl > 0)
    k_sell_fill<<<grid_for(nsl * 32, 256), 256, 0, s>>>(rop.as<int>(), out.s_off, nsl, wid.as<int>(),
                                                        out.s_wrow, out.s_wstep, rp, out.edges,
                                                        (unsigned)n, out.s_words);
  IG_CK(dev_alloc(&out.s_lrow, (size_t)std::max(nlong, 1LL) * sizeof(int), s));
  IG_CK(dev_alloc(&out.s_lp0, (size_t)(nlong + 1) * sizeof(int), s));
  if (nlong > 0)
    IG_CK(cudaMemcpyAsync(out.s_lrow, lrow_all.p, (size_t)nlong * sizeof(int),
                          cudaMemcpyDeviceToDevice, s));
  else
    IG_CK(cudaMemsetAsync(out.s_lp0, 0, sizeof(int), s));
  long long nlw = 0;
  int npieces = 0;
  if (nlong > 0) {
    Tmp len, loff, np;
    IG_CK(len.alloc((size_t)(nlong + 1) * sizeof(long long)));
    IG_CK(loff.alloc((size_t)(nlong + 1) * sizeof(long long)));
    IG_CK(np.alloc((size_t)(nlong + 1) * sizeof(int)));
    k_sell_long_len<<<grid_for(nlong, 256), 256, 0, s>>>(out.s_lrow, (int)nlong, rp, out.sell_piece,
                                                         len.as<long long>(), np.as<int>());
    size_t tb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.as<long long>(), loff.as<long long>(),
                                        nlong + 1, s));
    size_t tb2 = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, np.as<int>(), out.s_lp0, nlong + 1, s));
    IG_CK(tmp.alloc(std::max(tb, tb2)));
    IG_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.as<long long>(), loff.as<long long>(),
                                        nlong + 1, s));
    IG_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, np.as<int>(), out.s_lp0, nlong + 1, s));
    IG_CK(cudaMemcpyAsync(&nlw, loff.as<long long>() + nlong, sizeof(long long),
                          cudaMemcpyDeviceToHost, s));
    IG_CK(cudaMemcpyAsync(&npieces, out.s_lp0 + nlong, sizeof(int), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    IG_CK(dev_alloc(&out.s_lwords, (size_t)std::max(nlw, 1LL) * sizeof(unsigned), s));
    IG_CK(dev_alloc(&out.s_piece, (size_t)std::max(npieces, 1) * sizeof(int2), s));
    k_sell_long_fill<<<grid_for(nlong * 32, 256), 256, 0, s>>>(out.s_lrow, (int)nlong, rp,
                                                               out.edges, loff.as<long long>(),
                                                               out.s_lp0, out.sell_piece,
                                                               out.s_lwords, out.s_piece);
  }
  out.sell_lwords = nlw;
  out.sell_npieces = npieces;
  IG_CK(cudaGetLastError());
  IG_CK(cudaStreamSynchronize(s));
  return PSI_OK;
}

int batch_vectors(IngestOut& out, long long n, int NA, int nprof, const int* rp, const int* idx,
                  const int* new_of_old, const int* longr, long long nlongr, const double* bold,
                  const double* lam, cudaStream_t s, char* msg, size_t msg_len) {
  const int G = (nprof + kBP - 1) / kBP;
  out.nprof = nprof;
  out.ngroups = G;
  const size_t nb = (size_t)G * n * kBP * sizeof(double);
  const size_t ab = (size_t)G * std::max(NA, 1) * kBP * sizeof(double);
  IG_CK(dev_alloc(&out.b_a0, nb, s));
  IG_CK(dev_alloc(&out.b_psi, nb, s));
  for (double** q : {&out.b_a1, &out.b_g, &out.b_wt, &out.b_d1, &out.b_lam})
    IG_CK(dev_alloc(q, ab, s));
  for (double* q : {out.b_a0, out.b_psi}) IG_CK(cudaMemsetAsync(q, 0, nb, s));
  for (double* q : {out.b_a1, out.b_g, out.b_wt, out.b_d1, out.b_lam}) IG_CK(cudaMemsetAsync(q, 0, ab, s));
  Tmp K;
  IG_CK(K.alloc((size_t)std::max(NA, 1) * sizeof(double)));
  for (int p = 0; p < nprof; ++p) {
    const double* base = bold + (size_t)p * 4 * n;
    if (NA > 0) {
      k_fold_short<<<grid_for(NA, 256), 256, 0, s>>>(rp, idx, out.old_of_new, new_of_old, base, NA,
                                                     K.as<double>());
      if (nlongr > 0)
        k_fold_long<<<grid_for(nlongr * 32, 256), 256, 0, s>>>(longr, (int)nlongr, rp, idx,
                                                               out.old_of_new, new_of_old, base, NA,
                                                               K.as<double>());
    }
    k_permute_b<<<grid_for(n, 256), 256, 0, s>>>(out.old_of_new, n, NA, p, base, base + n,
                                                 base + 2 * n, base + 3 * n, lam + (size_t)p * n,
                                                 K.as<double>(), out);
  }
  IG_CK(cudaStreamSynchronize(s));
  return PSI_OK;
}

// tile_row / split rows (long ones first) of the edge stream cut into `tile`-edge tiles
int make_tiling(const int* rp_new, int NA, long long m_pad, int tile, cudaStream_t s, int** tile_row,
                int4** split, int* nsplit, int* nsplit_long, char* msg, size_t msg_len) {
  const int ntiles = (int)(m_pad / tile);
  IG_CK(dev_alloc(tile_row, (size_t)(ntiles + 1) * sizeof(int), s));
  k_tile_rows<<<grid_for(ntiles + 1, 256), 256, 0, s>>>(rp_new, NA, ntiles, tile, *tile_row);
  Tmp fl, rows, ns, sel_tmp;
  IG_CK(fl.alloc((size_t)(NA > 0 ? NA : 1)));
  IG_CK(rows.alloc((size_t)(NA > 0 ? NA : 1) * sizeof(int)));
  IG_CK(ns.alloc(sizeof(long long)));
  IG_CK(cudaMemsetAsync(ns.p, 0, sizeof(long long), s));
  long long hs = 0;
  if (NA > 0) {
    k_split_flags<<<grid_for(NA, 256), 256, 0, s>>>(rp_new, NA, tile, fl.as<unsigned char>());
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
  *nsplit = (int)hs;
  *nsplit_long = 0;
  IG_CK(dev_alloc(split, (size_t)(hs > 0 ? hs : 1) * sizeof(int4), s));
  if (hs > 0) {
    k_split_fill<<<grid_for(hs, 256), 256, 0, s>>>(rows.as<int>(), hs, rp_new, tile, *split);
    // rows spanning more than kLongSpan tiles first (summed by a warp each in k_fix)
    Tmp sp2, lf, part_tmp;
    IG_CK(sp2.alloc((size_t)hs * sizeof(int4)));
    IG_CK(lf.alloc((size_t)hs));
    k_long_split_flags<<<grid_for(hs, 256), 256, 0, s>>>(*split, hs, lf.as<unsigned char>());
    size_t pb = 0;
    IG_CK(cub::DevicePartition::Flagged(nullptr, pb, *split, lf.as<unsigned char>(),
                                        sp2.as<int4>(), ns.as<long long>(), (int)hs, s));
    IG_CK(part_tmp.alloc(pb));
    IG_CK(cub::DevicePartition::Flagged(part_tmp.p, pb, *split, lf.as<unsigned char>(),
                                        sp2.as<int4>(), ns.as<long long>(), (int)hs, s));
    IG_CK(cudaMemcpyAsync(*split, sp2.p, (size_t)hs * sizeof(int4), cudaMemcpyDeviceToDevice, s));
    long long nl = 0;
    IG_CK(cudaMemcpyAsync(&nl, ns.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    *nsplit_long = (int)nl;
  }
  IG_CK(cudaStreamSynchronize(s));
  return PSI_OK;
}

int ingest(long long n, long long m, const long long* rp64, const int* idx_in,
           const double* lam, const double* mu, int nprof, cudaStream_t s, IngestOut& out,
           char* msg, size_t msg_len, cudaEvent_t act_ready) {
  if (nprof < 1) nprof = 1;
  const int N = (int)n, Mm = (int)m;
  Tmp flags;
  IG_CK(flags.alloc(sizeof(int)));
  IG_CK(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
  int hflags = 0;

  Trace tr(s);
  g_tmp_stream = s;
  // (the pool's release threshold is set by psi_build_graph: temporaries stay reserved)
  // ---- 1. validation
  k_check_rowptr<<<grid_for(n, 256), 256, 0, s>>>(rp64, n, m, flags.as<int>());
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
  // (the edges themselves are checked edge-parallel once the transpose has expanded every
  // edge's row, below)

  tr.mark("validate");
  // ---- 2.-4. transpose, normalisers, constants (old labels)
  Tmp a_old, g_old, wt_old, d_old, first_leader, nlead, red;
  Tmp bold, bkmax;                       // batch: old-label constants of every profile
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
    // the four m-sized sort arrays and the sort's temporary storage: the build's scratch
    // slot 1 (kept across builds, outside the pool; the caller holds its mutex)
    Tmp loff, scan_tmp;
    IG_CK(loff.alloc((size_t)(n + 1) * sizeof(int)));
    int dev = 0;
    IG_CK(cudaGetDevice(&dev));
    size_t tb = 0;
    {
      cub::DoubleBuffer<unsigned> k0(nullptr, nullptr);
      cub::DoubleBuffer<int> v0(nullptr, nullptr);
      IG_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, v0, Mm, 0, end_bit, s));
    }
    const size_t ma = (((size_t)std::max<long long>(m, 1) * sizeof(int)) + 255) & ~(size_t)255;
    unsigned char* sc = nullptr;
    IG_CK(scratch_get(dev, 1, 4 * ma + tb, (void**)&sc));
    const Span leader_e{sc}, follower_e{sc + ma}, leader_s{sc + 2 * ma}, follower_s{sc + 3 * ma},
        sort_tmp{sc + 4 * ma};
    // (follower, leader) pairs in input order: keys = a copy of the input followers, values
    // = the row (leader) of every edge; a stable radix sort by follower is the transpose
    if (m > 0)
      IG_CK(cudaMemcpyAsync(follower_e.p, idx_in, (size_t)m * sizeof(int), cudaMemcpyDeviceToDevice, s));
    k_expand_short<<<grid_for(n, 256), 256, 0, s>>>(rp, N, leader_e.as<int>());
    {
      Tmp longl;
      const long long nl = long_segments(rp, nullptr, N, kShort, s, longl);
      if (nl < 0) IG_CK(cudaErrorMemoryAllocation);
      if (nl > 0)
        k_expand_long<<<grid_for(nl * 32, 256), 256, 0, s>>>(longl.as<int>(), (int)nl, rp,
                                                             leader_e.as<int>());
    }
    // input contract of the follower lists (include/psi.h): range, no self loop, strictly
    // increasing within a row -- thread per edge, coalesced, with the expanded rows
    k_check_edges_flat<<<grid_for(m, 256), 256, 0, s>>>(idx_in, leader_e.as<int>(), m, N,
                                                        flags.as<int>());
    IG_CK(cudaMemcpyAsync(&hflags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    if (hflags & (F_RANGE | F_SELF | F_ORDER)) {
      snprintf(msg, msg_len, "graph: %s", (hflags & F_RANGE) ? "follower index out of [0, n)"
               : (hflags & F_SELF) ? "self loop (a user in its own follower list)"
               : "row not strictly increasing (duplicate or unsorted followers)");
      return PSI_E_GRAPH;
    }
    cub::DoubleBuffer<unsigned> keys((unsigned*)follower_e.p, (unsigned*)follower_s.p);
    cub::DoubleBuffer<int> vals(leader_e.as<int>(), leader_s.as<int>());
    IG_CK(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tb, keys, vals, Mm, 0, end_bit, s));
    // leaders of user u = sorted pairs [loff[u], loff[u+1]) (lower bounds); #leaders
    k_lower_bounds<<<grid_for(n + 1, 256), 256, 0, s>>>(keys.Current(), Mm, N, loff.as<int>(),
                                                        nlead.as<int>());
    k_diff<<<grid_for(n, 256), 256, 0, s>>>(loff.as<int>(), N, nlead.as<int>());
    // the activity vectors (their staging copy may still have been in flight on a side
    // stream, psi_api.cu): validated here, before their first use
    if (act_ready) IG_CK(cudaStreamWaitEvent(s, act_ready, 0));
    for (int p = 0; p < nprof; ++p)
      k_check_activity<<<grid_for(n, 256), 256, 0, s>>>(lam + (size_t)p * n, mu + (size_t)p * n, n,
                                                        flags.as<int>());
    IG_CK(cudaMemcpyAsync(&hflags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    if (hflags & F_ACT) {
      snprintf(msg, msg_len, "activity: lambda/mu must be finite, >= 0, lambda+mu > 0");
      return PSI_E_ACTIVITY;
    }
    Tmp lm, longu;
    IG_CK(lm.alloc((size_t)n * sizeof(double2)));
    k_pack_activity<<<grid_for(n, 256), 256, 0, s>>>(lam, mu, n, lm.as<double2>());
    k_norm_short<<<grid_for(n, 256), 256, 0, s>>>(
        loff.as<int>(), vals.Current(), lm.as<double2>(), N, a_old.as<double>(), g_old.as<double>(),
        wt_old.as<double>(), d_old.as<double>(), first_leader.as<int>(), kmax, cnt);
    long long nlong = long_segments(loff.as<int>(), nullptr, N, kShort, s, longu);
    if (m <= kPowerNfMaxEdges) {       // keep the leader lists for Power-NF (psi_powernf.cu)
      IG_CK(dev_alloc(&out.nf_loff, (size_t)(n + 1) * sizeof(int), s));
      IG_CK(dev_alloc(&out.nf_leaders, (size_t)std::max<long long>(m, 1) * sizeof(int), s));
      IG_CK(dev_alloc(&out.nf_lm, (size_t)n * sizeof(double2), s));
      IG_CK(cudaMemcpyAsync(out.nf_loff, loff.p, (size_t)(n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
      if (m > 0)
        IG_CK(cudaMemcpyAsync(out.nf_leaders, vals.Current(), (size_t)m * sizeof(int),
                              cudaMemcpyDeviceToDevice, s));
      IG_CK(cudaMemcpyAsync(out.nf_lm, lm.p, (size_t)n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    }
    if (nlong < 0) IG_CK(cudaErrorMemoryAllocation);
    if (nlong > 0)
      k_norm_long<<<grid_for(nlong * 32, 256), 256, 0, s>>>(
          longu.as<int>(), (int)nlong, loff.as<int>(), vals.Current(), lm.as<double2>(),
          a_old.as<double>(), g_old.as<double>(), wt_old.as<double>(), d_old.as<double>(),
          first_leader.as<int>(), kmax);
    if (nprof > 1) {
      // the constants (a, g, Wt, d) and ||B||_row of every profile, old labels, same kernels
      IG_CK(bold.alloc((size_t)nprof * 4 * n * sizeof(double)));
      IG_CK(bkmax.alloc((size_t)nprof * 4 * sizeof(unsigned long long)));
      IG_CK(cudaMemsetAsync(bkmax.p, 0, (size_t)nprof * 4 * sizeof(unsigned long long), s));
      Tmp fl_dummy, cnt_dummy, longb;
      IG_CK(fl_dummy.alloc((size_t)n * sizeof(int)));
      IG_CK(cnt_dummy.alloc(4 * sizeof(unsigned long long)));
      const long long nlb = long_segments(loff.as<int>(), nullptr, N, kShort, s, longb);
      if (nlb < 0) IG_CK(cudaErrorMemoryAllocation);
      for (int p = 0; p < nprof; ++p) {
        double* base = bold.as<double>() + (size_t)p * 4 * n;
        unsigned long long* km = bkmax.as<unsigned long long>() + 4 * p;
        k_pack_activity<<<grid_for(n, 256), 256, 0, s>>>(lam + (size_t)p * n, mu + (size_t)p * n, n,
                                                         lm.as<double2>());
        k_norm_short<<<grid_for(n, 256), 256, 0, s>>>(
            loff.as<int>(), vals.Current(), lm.as<double2>(), N, base, base + n, base + 2 * n,
            base + 3 * n, fl_dummy.as<int>(), km, cnt_dummy.as<unsigned long long>());
        if (nlb > 0)
          k_norm_long<<<grid_for(nlb * 32, 256), 256, 0, s>>>(
              longb.as<int>(), (int)nlb, loff.as<int>(), vals.Current(), lm.as<double2>(), base,
              base + n, base + 2 * n, base + 3 * n, fl_dummy.as<int>(), km);
      }
      std::vector<unsigned long long> hk((size_t)nprof * 4);
      IG_CK(cudaMemcpyAsync(hk.data(), bkmax.p, hk.size() * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
      IG_CK(cudaStreamSynchronize(s));
      out.b_kappa_row.resize(nprof);
      for (int p = 0; p < nprof; ++p) memcpy(&out.b_kappa_row[p], &hk[4 * p], 8);
    }
  }

  if (out.nf_loff) {
    IG_CK(dev_alloc(&out.nf_wt, (size_t)n * sizeof(double), s));
    IG_CK(cudaMemcpyAsync(out.nf_wt, wt_old.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  tr.mark("transpose+normalisers");
  // ---- 5. relabel
  Tmp cls, new_of_old, key, sel, flag8, nsel, stage_tmp, sort_tmp2, sorted;
  IG_CK(cls.alloc((size_t)n));
  IG_CK(new_of_old.alloc((size_t)n * sizeof(int)));
  IG_CK(dev_alloc(&out.old_of_new, (size_t)n * sizeof(int), s));
  k_classify<<<grid_for(n, 256), 256, 0, s>>>(rp, nlead.as<int>(), N, cls.as<unsigned char>(),
                                              new_of_old.as<int>(), ccount);
  unsigned long long h[16];
  IG_CK(cudaMemcpyAsync(h, red.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  IG_CK(cudaStreamSynchronize(s));
  memcpy(&out.kappa_row, &h[0], 8);
  memcpy(&out.rho_A, &h[1], 8);
  out.kappa_col = 0.0;                      // set by psi_build_graph's column pass
  out.n_leaderless = (long long)h[4];
  out.n_g = n - out.n_leaderless;
  const long long n_inactive = (long long)h[8 + C_INACTIVE];
  out.n_act = n - n_inactive;
  out.n_f = out.n_act;
  out.n_hot = (long long)h[8 + C_HOT];

  // heavy rows (psi_heavy.cu): active users with >= heavy_min active followers, labelled
  // first; their followers with label < H = nseg << seg_shift are summed by k_heavy from
  // staged shared-memory segments.  Disabled for graphs smaller than one segment.  The
  // overlapped sweep (PSI_OVERLAP=1) uses the smaller plan shape of psi_internal.cuh.
  out.ovl = env_int("PSI_OVERLAP", 0) != 0 ? 1 : 0;
  if (out.ovl) {
    out.heavy_seg_shift = kOvlSegShift;
    out.heavy_slots = kOvlSlots;
    out.heavy_warps = kOvlWarps;
  } else {
    // measurement knobs: the plan shape (segment size / slots per panel trade the TMA fills of
    // a panel against runs per row); (slots + 1) << seg_shift must fit kEntBits
    out.heavy_seg_shift = std::min(std::max(env_int("PSI_HEAVY_SEG_SHIFT", out.heavy_seg_shift), 10), 13);
    out.heavy_slots = std::min(std::max(env_int("PSI_HEAVY_SLOTS", out.heavy_slots), 1024),
                               (1 << (kEntBits - out.heavy_seg_shift)) - 1024);
  }
  const int kSegR = 1 << out.heavy_seg_shift;   // labels per staged segment
  long long h_default = kMinHeavyLabels;
  while (h_default * 2 <= n / 32 && h_default < kMaxHeavyLabels) h_default *= 2;
  int nseg = env_int("PSI_HEAVY_LABELS", (int)h_default) / kSegR;
  // on by default only where it measured faster (C5 yes, C4 no); PSI_HEAVY=1/0
  // forces it on/off
  const int heavy_env = env_int("PSI_HEAVY", -1);
  if (heavy_env == 0 || (heavy_env < 0 && n < kDefaultHeavyMinN)) nseg = 0;
  if (nprof > 1) nseg = 0;                     // the batch sweep has no staged-segment path
  nseg = (int)std::min<long long>(std::min(nseg, kMaxHeavySegs), (n + 1) / kSegR);
  if (nseg > 0) {
    Tmp act;
    IG_CK(act.alloc((size_t)n * sizeof(int)));
    k_active_count_short<<<grid_for(n, 256), 256, 0, s>>>(rp, idx_in, cls.as<unsigned char>(), N,
                                                          act.as<int>());
    {
      Tmp longa;
      const long long nl = long_segments(rp, nullptr, N, kShort, s, longa);
      if (nl < 0) IG_CK(cudaErrorMemoryAllocation);
      if (nl > 0)
        k_active_count_long<<<grid_for(nl * 32, 256), 256, 0, s>>>(longa.as<int>(), (int)nl, rp,
                                                                   idx_in, cls.as<unsigned char>(),
                                                                   act.as<int>());
    }
    IG_CK(cudaMemsetAsync(ccount, 0, 8 * sizeof(unsigned long long), s));
    k_mark_heavy<<<grid_for(n, 256), 256, 0, s>>>(act.as<int>(), N,
                                                  env_int("PSI_HEAVY_MIN", kDefaultHeavyMin),
                                                  cls.as<unsigned char>(), ccount);
    IG_CK(cudaMemcpyAsync(h + 8, ccount, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    out.n_heavy = (long long)h[8 + C_HEAVY];
    out.n_hot = (long long)h[8 + C_HOT] + out.n_heavy;
  }
  if (out.n_heavy == 0) nseg = 0;
  out.nseg = nseg;
  if (nseg == 0) out.ovl = 0;
  const int Hs = nseg * kSegR;                // staged labels [0, Hs)

  IG_CK(key.alloc((size_t)n * 8));
  IG_CK(sel.alloc((size_t)n * 8));
  IG_CK(sorted.alloc((size_t)n * 8));
  IG_CK(flag8.alloc((size_t)n));
  IG_CK(nsel.alloc(sizeof(long long)));
  size_t sel_bytes = 0, sort_bytes = 0;
  IG_CK(cub::DeviceSelect::Flagged(nullptr, sel_bytes, key.as<unsigned long long>(),
                                   flag8.as<unsigned char>(), sel.as<unsigned long long>(),
                                   nsel.as<long long>(), N, s));
  {
    // the level loop also selects int lists (user ids, a counting iterator): room for those too
    size_t b_it = 0, b_int = 0;
    cub::CountingInputIterator<int> it0(0);
    IG_CK(cub::DeviceSelect::Flagged(nullptr, b_it, it0, flag8.as<unsigned char>(), (int*)nullptr,
                                     nsel.as<long long>(), N, s));
    IG_CK(cub::DeviceSelect::Flagged(nullptr, b_int, (const int*)nullptr, flag8.as<unsigned char>(),
                                     (int*)nullptr, nsel.as<long long>(), N, s));
    sel_bytes = std::max(sel_bytes, std::max(b_it, b_int));
  }
  IG_CK(stage_tmp.alloc(sel_bytes));
  IG_CK(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, sel.as<unsigned long long>(),
                                       sorted.as<unsigned long long>(), N, 32, 64, s));
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
      // the selected keys arrive in ascending user order (DeviceSelect keeps it) and the
      // radix sort is stable: sorting the high 32 bits keeps the user id as the tie-break
      IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp2.p, b2, sel.as<unsigned long long>(),
                                           sorted.as<unsigned long long>(), (int)c, 32, 64, s));
      src = sorted.as<unsigned long long>();
    }
    k_assign<<<grid_for(c, 256), 256, 0, s>>>(src, c, base, new_of_old.as<int>(), out.old_of_new);
    base += (int)c;
    return PSI_OK;
  };
  long long c = 0;
  int rc;
  if (out.n_heavy > 0 && (rc = run_stage(5, true, &c)) != PSI_OK) return rc;  // heavy rows first
  if ((rc = run_stage(0, true, &c)) != PSI_OK) return rc;          // hot, by leader count
  if ((rc = run_stage(1, false, &c)) != PSI_OK) return rc;         // leaderless active
  out.single_lo = base;                                            // single-leader users follow
  {
    // single-leader users level by level (stage 2 of k_stage_keys), each level scanning only
    // the users still unlabelled (a pass over all n per level cost ~0.5 ms x ~50 levels at
    // C5); same keys, same stable order, so the same labels
    Tmp pend, pend2, rdy, kp;
    IG_CK(pend.alloc((size_t)n * sizeof(int)));
    IG_CK(pend2.alloc((size_t)n * sizeof(int)));
    IG_CK(rdy.alloc((size_t)n));
    IG_CK(kp.alloc((size_t)n));
    k_single_flags<<<grid_for(n, 256), 256, 0, s>>>(cls.as<unsigned char>(), N, flag8.as<unsigned char>());
    cub::CountingInputIterator<int> it(0);
    size_t b0 = sel_bytes;
    IG_CK(cub::DeviceSelect::Flagged(stage_tmp.p, b0, it, flag8.as<unsigned char>(), pend.as<int>(),
                                     nsel.as<long long>(), N, s));
    long long np = 0;
    IG_CK(cudaMemcpyAsync(&np, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    while (np > 0) {
      k_level_keys<<<grid_for(np, 256), 256, 0, s>>>(pend.as<int>(), np, first_leader.as<int>(),
                                                    new_of_old.as<int>(), key.as<unsigned long long>(),
                                                    rdy.as<unsigned char>(), kp.as<unsigned char>());
      size_t b1 = sel_bytes;
      IG_CK(cub::DeviceSelect::Flagged(stage_tmp.p, b1, key.as<unsigned long long>(),
                                       rdy.as<unsigned char>(), sel.as<unsigned long long>(),
                                       nsel.as<long long>(), (int)np, s));
      long long cl = 0;
      IG_CK(cudaMemcpyAsync(&cl, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
      IG_CK(cudaStreamSynchronize(s));
      if (cl == 0) break;
      size_t b2 = sort_bytes;
      IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp2.p, b2, sel.as<unsigned long long>(),
                                           sorted.as<unsigned long long>(), (int)cl, 32, 64, s));
      k_assign<<<grid_for(cl, 256), 256, 0, s>>>(sorted.as<unsigned long long>(), cl, base,
                                                new_of_old.as<int>(), out.old_of_new);
      base += (int)cl;
      ++levels;
      size_t b3 = sel_bytes;
      IG_CK(cub::DeviceSelect::Flagged(stage_tmp.p, b3, pend.as<int>(), kp.as<unsigned char>(),
                                       pend2.as<int>(), nsel.as<long long>(), (int)np, s));
      IG_CK(cudaMemcpyAsync(&np, nsel.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
      IG_CK(cudaStreamSynchronize(s));
      std::swap(pend.p, pend2.p);
    }
    if (np > 0) {                                      // leftovers (cycles), stage 3's keys
      k_cycle_keys<<<grid_for(np, 256), 256, 0, s>>>(pend.as<int>(), np, first_leader.as<int>(),
                                                    sel.as<unsigned long long>());
      size_t b2 = sort_bytes;
      IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp2.p, b2, sel.as<unsigned long long>(),
                                           sorted.as<unsigned long long>(), (int)np, 32, 64, s));
      k_assign<<<grid_for(np, 256), 256, 0, s>>>(sorted.as<unsigned long long>(), np, base,
                                                new_of_old.as<int>(), out.old_of_new);
      base += (int)np;
    }
  }
  if (base != out.n_act) {
    snprintf(msg, msg_len, "internal: relabel covered %d of %lld active users", base, out.n_act);
    return PSI_E_CUDA;
  }
  if ((rc = run_stage(4, false, &c)) != PSI_OK) return rc;         // follower-less
  out.relabel_levels = levels;
  key.reset(); sel.reset(); sorted.reset(); flag8.reset(); stage_tmp.reset(); sort_tmp2.reset();

  tr.mark("relabel");
  // The sweep's layout: the sliced-ELL copy of the edge stream (k_sell) for single-profile
  // graphs with heavy rows (C4/C5: measured faster than the tiles) and for
  // graphs without them whose slices pad little (C2), the edge-balanced tiles (k_tiles, and
  // k_solve for small graphs) otherwise; PSI_SELL=0/1 forces
  // the tiles / the sliced-ELL layout (not with the overlapped plan or a batch).
  {
    const int se = env_int("PSI_SELL", -1);
    const bool can = out.n_act > 0 && nprof == 1 && !out.ovl;
    // 2 = decided at step 8 from the layout's padding (graphs without heavy rows: C2's
    // near-uniform rows pad little and k_sell wins, C3's power-law rows pad 2.4x and lose)
    out.sell = can && (se == 1 || (se < 0 && out.n_heavy > 0)) ? 1 : (can && se < 0 ? 2 : 0);
  }
  // ---- 6. relabelled edge stream over active rows, folded constants
  const int NA = (int)out.n_act;
  Tmp cntr, K, rp_new;
  IG_CK(dev_alloc(&out.kinv, (size_t)(NA > 0 ? NA : 1) * sizeof(double), s));
  IG_CK(dev_alloc(&out.kw, (size_t)(NA > 0 ? NA : 1) * sizeof(double), s));
  IG_CK(cntr.alloc((size_t)(NA + 1) * sizeof(int)));
  IG_CK(K.alloc((size_t)(NA > 0 ? NA : 1) * sizeof(double)));
  IG_CK(rp_new.alloc((size_t)(NA + 1) * sizeof(int)));
  IG_CK(cudaMemsetAsync(cntr.p, 0, (size_t)(NA + 1) * sizeof(int), s));
  const int NH = (int)out.n_heavy;
  Tmp hcnt, hoff;
  IG_CK(hcnt.alloc((size_t)(NH + 1) * sizeof(long long)));
  IG_CK(hoff.alloc((size_t)(NH + 1) * sizeof(long long)));
  IG_CK(cudaMemsetAsync(hcnt.p, 0, (size_t)(NH + 1) * sizeof(long long), s));
  Tmp longr, labmap;
  IG_CK(labmap.alloc((size_t)std::max<long long>(m, 1) * sizeof(int)));
  long long nlongr = 0;
  if (NA > 0) {
    nlongr = long_segments(rp, out.old_of_new, NA, kShort, s, longr);
    if (nlongr < 0) IG_CK(cudaErrorMemoryAllocation);
    RowCountArgs R{rp, idx_in, out.old_of_new, cls.as<unsigned char>(), new_of_old.as<int>(),
                   a_old.as<double>(), nlead.as<int>(), NA, NH, Hs, cntr.as<int>(),
                   hcnt.as<long long>(), K.as<double>(), out.kinv, wt_old.as<double>(), out.kw,
                   labmap.as<int>()};
    k_row_count_short<<<grid_for(NA, 256), 256, 0, s>>>(R);
    if (nlongr > 0)
      k_row_count_long<<<grid_for(nlongr * 32, 256), 256, 0, s>>>(R, longr.as<int>(), (int)nlongr);
  }
  long long n_hot_ent = 0;
  if (NH > 0) {
    Tmp scan_tmp;
    size_t sb = 0;
    IG_CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, hcnt.as<long long>(), hoff.as<long long>(),
                                        NH + 1, s));
    IG_CK(scan_tmp.alloc(sb));
    IG_CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, sb, hcnt.as<long long>(), hoff.as<long long>(),
                                        NH + 1, s));
    IG_CK(cudaMemcpyAsync(&n_hot_ent, hoff.as<long long>() + NH, sizeof(long long),
                          cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
  }
  // the heavy rows' host plan runs on a helper thread while the device builds the edge stream
  HeavyHostPlan& HP = heavy_host_plan();
  std::unique_lock<std::mutex> hp_lock(HP.mu, std::defer_lock);
  std::thread hp_thread;
  if (NH > 0) {
    hp_lock.lock();
    HP.hc.resize(NH);
    IG_CK(cudaMemcpyAsync(HP.hc.data(), hcnt.p, (size_t)NH * sizeof(long long),
                          cudaMemcpyDeviceToHost, s));
    IG_CK(cudaStreamSynchronize(s));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pps = std::max(1, env_int("PSI_HEAVY_PPS", kDefaultHeavyPPS));
    // the search runs with the default panels-per-SM only (PSI_HEAVY_PPS is a measurement knob)
    const int search = env_int("PSI_HEAVY_SEARCH", 1) != 0 && env_int("PSI_HEAVY_PPS", -1) < 0 ? 1 : 0;
    hp_thread = std::thread(plan_heavy_host, std::ref(HP), NH, n_hot_ent, out.heavy_warps,
                            out.heavy_slots, sms, pps, out.nseg, search);
  }
  // joined on every exit path below (an early error return must not leave it running)
  struct Joiner {
    std::thread& t;
    ~Joiner() { if (t.joinable()) t.join(); }
  } hp_join{hp_thread};
  Tmp hot;
  IG_CK(hot.alloc((size_t)(n_hot_ent > 0 ? n_hot_ent : 1) * sizeof(int)));
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
  // 1024-edge tiles where heavy rows exist (C4/C5: the sweep's L1 holds more of x with one
  // hot cache for 8 groups); 512-edge tiles otherwise (smaller barrier groups; C2/C3 measured,
  // DESIGN.md §12).  PSI_TILE=512|1024 forces one.
  {
    const int te = env_int("PSI_TILE", 0);
    out.tile = (te == 512 || te == 1024) ? te : (out.n_heavy > 0 ? kTile : 512);
  }
  out.ntiles = (int)(((long long)m_act + out.tile - 1) / out.tile);
  const long long m_pad = (long long)out.ntiles * out.tile;
  {
    IG_CK(dev_alloc(&out.edges, (size_t)(m_pad > 0 ? m_pad : 4) * sizeof(unsigned), s));
    int* ed = (int*)out.edges;
    if (NA > 0) {
      RowFillArgs R{rp, labmap.as<int>(), out.old_of_new, cls.as<unsigned char>(),
                    rp_new.as<int>(), NA, N, NH, Hs, hoff.as<long long>(), ed, hot.as<int>()};
      k_row_fill_short<<<grid_for(NA, 256), 256, 0, s>>>(R);
      if (nlongr > 0)
        k_row_fill_long<<<grid_for(nlongr * 32, 256), 256, 0, s>>>(R, longr.as<int>(), (int)nlongr);
    }
    // rows keep their followers in input order: the sweep's sums have a fixed order either
    // way, and a per-row sort bought nothing measurable
    if (m_act > 0 && out.sell != 1) {      // (the sliced-ELL copy needs no flags)
      k_flag_rows<<<grid_for(NA, 256), 256, 0, s>>>(rp_new.as<int>(), NA, m_act, m_pad, N,
                                                    out.edges);
    }
    IG_CK(cudaStreamSynchronize(s));
  }
  labmap.reset();
  tr.mark("edge stream");
  if (NH > 0) {
    hp_thread.join();
    tr.mark("  heavy: host plan joined");
    if (tr.on)
      fprintf(stderr, "[psi ingest]   heavy: panel shape %d %% of the entry target, slot cap %d: %d panels, "
              "tail %d %% from %d %% of the entries; simulated makespan %lld -> %lld entries\n", HP.sel_num,
              HP.sel_cap, HP.npanels, HP.sel_tail, HP.sel_from, HP.sim_base, HP.sim_best);
    int rc2 = build_heavy_plan(out, NH, n_hot_ent, hot, hoff, HP, s, tr, msg, msg_len);
    hp_lock.unlock();
    if (rc2 != PSI_OK) return rc2;
  }
  hot.reset();

  tr.mark("heavy plan");
  const size_t na_b = (size_t)(NA > 0 ? NA : 1) * sizeof(double);
  IG_CK(dev_alloc(&out.a0, (size_t)n * sizeof(double), s));
  IG_CK(dev_alloc(&out.wt, (size_t)n * sizeof(double), s));
  IG_CK(dev_alloc(&out.psi, (size_t)n * sizeof(double), s));
  IG_CK(dev_alloc(&out.a1, na_b, s));
  IG_CK(dev_alloc(&out.g, na_b, s));
  IG_CK(dev_alloc(&out.d1, na_b, s));
  IG_CK(dev_alloc(&out.lam, na_b, s));
  IG_CK(dev_alloc(&out.nlead, (size_t)n * sizeof(int), s));
  k_permute_vectors<<<grid_for(n, 256), 256, 0, s>>>(
      out.old_of_new, N, NA, a_old.as<double>(), g_old.as<double>(), wt_old.as<double>(),
      d_old.as<double>(), lam, K.as<double>(), (double)n, nlead.as<int>(), out.a0, out.a1, out.g,
      out.wt, out.d1, out.lam, out.psi, out.nlead);
  out.relabeled = 1;
  if (nprof > 1) {
    int rc3 = batch_vectors(out, n, NA, nprof, rp, idx_in, new_of_old.as<int>(), longr.as<int>(),
                            nlongr, bold.as<double>(), lam, s, msg, msg_len);
    if (rc3 != PSI_OK) return rc3;
    bold.reset();
  }

  tr.mark("vectors");
  // small graphs (at most kCoopEdges edge slots) keep the tiles: the persistent cooperative
  // solver runs the whole loop in one launch there (psi_api.cu use_coop)
  if (out.sell == 2 && (long long)out.ntiles * out.tile <= kCoopEdges) out.sell = 0;
  // ---- 7. edge tiles: first row of every tile, rows spanning tiles (and, for a batch
  // context, the same for the batch sweep's 512-edge tiles)
  {
    int rc4 = PSI_OK;
    if (out.sell != 1) {
      rc4 = make_tiling(rp_new.as<int>(), NA, (long long)out.ntiles * out.tile, out.tile, s,
                        &out.tile_row, &out.split, &out.nsplit, &out.nsplit_long, msg, msg_len);
      if (rc4 != PSI_OK) return rc4;
    }
    if (out.ovl && out.n_heavy > 0) {
      const size_t words = (size_t)(out.n_heavy / 32 + 1);
      IG_CK(dev_alloc(&out.hsplit, words * sizeof(unsigned), s));
      IG_CK(cudaMemsetAsync(out.hsplit, 0, words * sizeof(unsigned), s));
      if (out.nsplit > 0)
        k_heavy_split_bits<<<grid_for(out.nsplit, 256), 256, 0, s>>>(out.split, out.nsplit,
                                                                     (int)out.n_heavy, out.hsplit);
    }
    if (nprof > 1) {
      // as many tiles as hold the m_act real edge words: the last one is never all padding
      out.b_ntiles = (int)(((long long)out.m_act + kTileB - 1) / kTileB);
      rc4 = make_tiling(rp_new.as<int>(), NA, (long long)out.b_ntiles * kTileB, kTileB, s, &out.b_tile_row,
                        &out.b_split, &out.b_nsplit, &out.b_nsplit_long, msg, msg_len);
      if (rc4 != PSI_OK) return rc4;
    }
  }
  IG_CK(cudaGetLastError());
  tr.mark("tiles");
  // ---- 8. sliced-ELL layout of the same edge stream (k_sell); the stream itself is then
  // no longer needed
  {
    if (out.sell) {
      // windows of 2^shift rows: 256 (C4/C5), fewer on graphs with few active rows so that
      // every warp of the grid gets >= 3 windows (C2: 64-row windows, 0.086 -> 0.080 ms;
      // 256-row windows leave a fifth of the warps without one)
      int shift = kSellShift;
      if (out.n_heavy == 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        while (shift > 5 && ((long long)NA >> shift) < 3LL * sms * kSellWarps) --shift;
      }
      out.sell_shift = std::min(std::max(env_int("PSI_SELL_SHIFT", shift), 5), 10);
      out.sell_kcap = std::max(env_int("PSI_SELL_KCAP", kSellKcap), 1);
      out.sell_lmax = std::min(std::max(env_int("PSI_SELL_LMAX", kSellLmax), 1), 2047);
      out.sell_piece = std::max(env_int("PSI_SELL_PIECE", kSellPiece), 32);
      bool rejected = false;
      int rc5 = build_sell(out, rp_new.as<int>(), NA, n, s, msg, msg_len,
                           out.sell == 2 ? kSellMaxPad : 0.0, &rejected);
      if (rc5 != PSI_OK) return rc5;
      if (rejected) {
        out.sell = 0;                                // the tiles built at step 7 stay
      } else {
        out.sell = 1;
        IG_CK(cudaFreeAsync(out.edges, s));
        out.edges = nullptr;
      }
      tr.mark("sliced-ELL");
    }
  }
  return PSI_OK;
}

}  // namespace psi
