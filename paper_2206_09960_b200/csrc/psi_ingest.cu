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

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
__global__ void k_active_count(const int* rp, const int* idx, const unsigned char* cls, int n,
                               int* act) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(u, n) {
    const int b = rp[u], e = rp[u + 1];
    int c = 0;
    for (int q = b + lane; q < e; q += 32) c += cls[idx[q]] != C_INACTIVE;
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) act[u] = c;
  }
}

// heavy rows: active users with >= min_act active followers; recount the classes
__global__ void k_mark_heavy(const int* act, int n, int min_act, unsigned char* cls,
                             unsigned long long* counts) {
  GRID_STRIDE(u, n) {
    unsigned char c = cls[u];
    if (c != C_INACTIVE && act[u] >= min_act) cls[u] = c = C_HEAVY;
    atomicAdd(counts + c, 1ull);
  }
}

// warp per new active row r: #active followers in the edge stream (for heavy rows r <
// n_heavy only those with label >= H; the others, hc[r], go to k_heavy), and
// K_r = sum of a_n over follower-less followers
__global__ void k_row_count(const int* rp, const int* idx, const int* old_of_new,
                            const unsigned char* cls, const int* new_of_old, const double* a_old,
                            int n_act, int n_heavy, int H, int* cnt, long long* hc, double* K) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_act) {
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    const bool heavy = r < n_heavy;
    int c = 0, h = 0;
    double k = 0.0;
    for (int q = b + lane; q < e; q += 32) {
      const int v = idx[q];
      if (cls[v] == C_INACTIVE) k += a_old[v];
      else if (heavy && new_of_old[v] < H) ++h;
      else ++c;
    }
    c = __reduce_add_sync(kFull, c);
    h = __reduce_add_sync(kFull, h);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) k += __shfl_xor_sync(kFull, k, s);
    if (lane == 0) {
      cnt[r] = c > 0 ? c : 1;      // 0 -> one pseudo edge
      K[r] = k;
      if (heavy) hc[r] = h;
    }
  }
}

// warp per new active row: write the active followers' new labels (unsorted, stable) to the
// edge stream -- heavy rows: only labels >= H; their labels < H go to hot[hoff[r]...].  A row
// with no stream follower gets one pseudo edge to the sentinel label n (x[n] = 0).
__global__ void k_row_fill(const int* rp, const int* idx, const int* old_of_new,
                           const unsigned char* cls, const int* new_of_old, const int* rp_new,
                           int n_act, int n, int n_heavy, int H, const long long* hoff,
                           int* idx_new, int* hot) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_act) {
    const int o = old_of_new[r];
    const int b = rp[o], e = rp[o + 1];
    const int start = rp_new[r];
    const bool heavy = r < n_heavy;
    int out = start;
    long long hout = heavy ? hoff[r] : 0;
    for (int q0 = b; q0 < e; q0 += 32) {
      const int q = q0 + lane;
      int v = -1;
      bool act = false;
      if (q < e) { v = idx[q]; act = cls[v] != C_INACTIVE; }
      const int nv = act ? new_of_old[v] : 0;
      const bool is_hot = act && heavy && nv < H;
      const bool is_str = act && !is_hot;
      const unsigned m1 = __ballot_sync(kFull, is_str), m2 = __ballot_sync(kFull, is_hot);
      const unsigned below = (1u << lane) - 1u;
      if (is_str) idx_new[out + __popc(m1 & below)] = nv;
      if (is_hot) hot[hout + __popc(m2 & below)] = nv;
      out += __popc(m1);
      hout += __popc(m2);
    }
    if (lane == 0 && out == start) idx_new[start] = n;
  }
}

// warp per heavy row: entry keys (list << kEntBits) | (slot << kSegShift) | (label % kSeg);
// list = (panel * kHeavyWarps + owner warp of the slot) * nseg + segment.  The i-th hot
// follower of row r goes to slot rslot[r].x + i % rslot[r].y (round-robin virtual rows).
__global__ void k_heavy_keys(const int* hot, const long long* hoff, const int2* rslot,
                             const int* row_panel, const int* pslot_base, const unsigned char* slot_warp,
                             int n_heavy, int nseg, unsigned long long* keys) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(r, n_heavy) {
    const long long b = hoff[r], e = hoff[r + 1];
    const int2 sn = rslot[r];
    const int p = row_panel[r];
    const int base = pslot_base[p];
    for (long long q = b + lane; q < e; q += 32) {
      const unsigned lab = (unsigned)hot[q];
      const int slot = sn.x + (int)((q - b) % sn.y);
      const unsigned long long list =
          ((unsigned long long)p * kHeavyWarps + slot_warp[base + slot]) * nseg + (lab >> kSegShift);
      keys[q] = (list << kEntBits) | ((unsigned long long)slot << kSegShift) | (lab & (kSeg - 1));
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
    ent[loff[L] + (i - lstart[L])] = (unsigned)(k & ((1ull << kEntBits) - 1));
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

// Heavy-row plan (psi_heavy.cu): panels of <= kHeavySlots slots and ~e_panel hot entries,
// virtual rows of <= vmax entries, contiguous slot ranges per consumer warp balanced by
// entries; then the entry lists (panel, segment, warp) sorted by (slot, label).
int build_heavy_plan(IngestOut& out, int NH, long long n_ent, Tmp& hot, Tmp& hcnt, Tmp& hoff,
                     cudaStream_t s, char* msg, size_t msg_len) {
  const int nseg = out.nseg;
  std::vector<long long> hc(NH);
  IG_CK(cudaMemcpyAsync(hc.data(), hcnt.p, (size_t)NH * sizeof(long long), cudaMemcpyDeviceToHost, s));
  // hot followers of each heavy row sorted by label (the k_row_fill order is unsorted)
  if (n_ent > 0) {
    Tmp tmp2, seg_tmp;
    IG_CK(tmp2.alloc((size_t)n_ent * sizeof(int)));
    cub::DoubleBuffer<int> kb(hot.as<int>(), tmp2.as<int>());
    size_t tb = 0;
    IG_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, kb, (int)n_ent, NH, hoff.as<long long>(),
                                             hoff.as<long long>() + 1, s));
    IG_CK(seg_tmp.alloc(tb));
    IG_CK(cub::DeviceSegmentedSort::SortKeys(seg_tmp.p, tb, kb, (int)n_ent, NH, hoff.as<long long>(),
                                             hoff.as<long long>() + 1, s));
    if (kb.Current() != hot.as<int>())
      IG_CK(cudaMemcpyAsync(hot.p, kb.Current(), (size_t)n_ent * sizeof(int),
                            cudaMemcpyDeviceToDevice, s));
  }
  IG_CK(cudaStreamSynchronize(s));

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long pps = std::max(1, env_int("PSI_HEAVY_PPS", kDefaultHeavyPPS));
  const long long e_panel = std::max<long long>((n_ent + pps * sms - 1) / (pps * sms), 32768);
  const long long vmax = std::max<long long>(e_panel / (2 * kHeavyWarps), 64);
  std::vector<int> prow{0}, row_panel(NH), pslot_base{0}, wslot;
  std::vector<int2> rslot(NH);
  std::vector<unsigned char> slot_warp;
  std::vector<long long> slot_w;
  long long p_ent = 0;
  auto close_panel = [&](int r_end) {
    const int slots = (int)slot_w.size();
    long long T = 0;
    for (long long x : slot_w) T += x;
    std::vector<int> ws(kHeavyWarps + 1, slots);
    ws[0] = 0;
    long long acc = 0;
    int w = 1;
    for (int k = 0; k < slots && w < kHeavyWarps; ++k) {
      acc += slot_w[k];
      while (w < kHeavyWarps && acc * kHeavyWarps >= T * w) ws[w++] = k + 1;
    }
    int owner = 0;
    for (int k = 0; k < slots; ++k) {
      while (owner + 1 < kHeavyWarps && ws[owner + 1] <= k) ++owner;
      slot_warp.push_back((unsigned char)owner);
    }
    wslot.insert(wslot.end(), ws.begin(), ws.end());
    prow.push_back(r_end);
    pslot_base.push_back(pslot_base.back() + slots);
    slot_w.clear();
    p_ent = 0;
  };
  for (int r = 0; r < NH; ++r) {
    long long nv = hc[r] > 0 ? (hc[r] + vmax - 1) / vmax : 0;
    if (nv > kHeavySlots) nv = kHeavySlots;
    if (r > prow.back() && ((long long)slot_w.size() + nv > kHeavySlots || p_ent + hc[r] > e_panel))
      close_panel(r);
    rslot[r] = make_int2((int)slot_w.size(), (int)nv);
    row_panel[r] = (int)prow.size() - 1;
    for (long long k = 0; k < nv; ++k) slot_w.push_back(hc[r] / nv + (k < hc[r] % nv ? 1 : 0));
    p_ent += hc[r];
  }
  close_panel(NH);
  const int npanels = (int)prow.size() - 1;
  out.npanels = npanels;
  out.heavy_entries = n_ent;

  IG_CK(cudaMalloc(&out.h_prow, prow.size() * sizeof(int)));
  IG_CK(cudaMalloc(&out.h_rslot, (size_t)NH * sizeof(int2)));
  IG_CK(cudaMalloc(&out.h_wslot, wslot.size() * sizeof(int)));
  IG_CK(cudaMemcpyAsync(out.h_prow, prow.data(), prow.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  IG_CK(cudaMemcpyAsync(out.h_rslot, rslot.data(), (size_t)NH * sizeof(int2), cudaMemcpyHostToDevice, s));
  IG_CK(cudaMemcpyAsync(out.h_wslot, wslot.data(), wslot.size() * sizeof(int), cudaMemcpyHostToDevice, s));

  const long long nlists = (long long)npanels * nseg * kHeavyWarps;
  IG_CK(cudaMalloc(&out.h_loff, (size_t)(nlists + 1) * sizeof(long long)));
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
      sw.as<unsigned char>(), NH, nseg, keys.as<unsigned long long>());
  int end_bit = kEntBits;
  while ((1LL << (end_bit - kEntBits)) <= nlists) ++end_bit;
  cub::DoubleBuffer<unsigned long long> kb(keys.as<unsigned long long>(), keys2.as<unsigned long long>());
  if (n_ent > 0) {
    size_t tb = 0;
    IG_CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, kb, (int)n_ent, 0, end_bit, s));
    IG_CK(sort_tmp.alloc(tb));
    IG_CK(cub::DeviceRadixSort::SortKeys(sort_tmp.p, tb, kb, (int)n_ent, 0, end_bit, s));
  }
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
  IG_CK(cudaMalloc(&out.h_ent, (size_t)std::max<long long>(total, 4) * sizeof(unsigned)));
  k_fill_u32<<<grid_for(total, 256), 256, 0, s>>>(out.h_ent, total, kNullEntry);
  k_heavy_fill<<<grid_for(n_ent, 256), 256, 0, s>>>(kb.Current(), n_ent, lstart.as<long long>(),
                                                   out.h_loff, out.h_ent);
  IG_CK(cudaStreamSynchronize(s));
  IG_CK(cudaGetLastError());
  return PSI_OK;
}

}  // namespace

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

  // heavy rows (psi_heavy.cu): active users with >= heavy_min active followers, labelled
  // first; their followers with label < H = nseg * kSeg are summed by k_heavy from staged
  // shared-memory segments.  Disabled for graphs smaller than one segment.
  int nseg = env_int("PSI_HEAVY_SEGS", kDefaultHeavySegs);   // in units of kSeg labels
  // on by default only where it measured faster (C5 yes, C4 no); PSI_HEAVY=1/0
  // forces it on/off
  const int heavy_env = env_int("PSI_HEAVY", -1);
  if (heavy_env == 0 || (heavy_env < 0 && n < kDefaultHeavyMinN)) nseg = 0;
  nseg = (int)std::min<long long>(std::min(nseg, kMaxHeavySegs), (n + 1) / kSeg);
  if (nseg > 0) {
    Tmp act;
    IG_CK(act.alloc((size_t)n * sizeof(int)));
    k_active_count<<<grid_for(n * 32, 256), 256, 0, s>>>(rp, idx_in, cls.as<unsigned char>(), N,
                                                         act.as<int>());
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
  const int Hs = nseg * kSeg;                 // staged labels [0, Hs)

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
  if (out.n_heavy > 0 && (rc = run_stage(5, true, &c)) != PSI_OK) return rc;  // heavy rows first
  if ((rc = run_stage(0, true, &c)) != PSI_OK) return rc;          // hot, by leader count
  if ((rc = run_stage(1, false, &c)) != PSI_OK) return rc;         // leaderless active
  out.single_lo = base;                                            // single-leader users follow
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
  const int NH = (int)out.n_heavy;
  Tmp hcnt, hoff;
  IG_CK(hcnt.alloc((size_t)(NH + 1) * sizeof(long long)));
  IG_CK(hoff.alloc((size_t)(NH + 1) * sizeof(long long)));
  IG_CK(cudaMemsetAsync(hcnt.p, 0, (size_t)(NH + 1) * sizeof(long long), s));
  if (NA > 0)
    k_row_count<<<grid_for((long long)NA * 32, 256), 256, 0, s>>>(
        rp, idx_in, out.old_of_new, cls.as<unsigned char>(), new_of_old.as<int>(),
        a_old.as<double>(), NA, NH, Hs, cntr.as<int>(), hcnt.as<long long>(), K.as<double>());
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
          rp_new.as<int>(), NA, N, NH, Hs, hoff.as<long long>(), ed, hot.as<int>());
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
  if (NH > 0) {
    int rc2 = build_heavy_plan(out, NH, n_hot_ent, hot, hcnt, hoff, s, msg, msg_len);
    if (rc2 != PSI_OK) return rc2;
  }
  hot.reset();

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
