// psi_sweep.cu -- the Power-psi sweep, fused L1 residual + stop rule, and readout (sm_100a).
//
// One sweep = two launches inside the CUDA-graph WHILE loop (psi_api.cu):
//
//  k_stream  persistent, edge-balanced gather-SpMV over the flagged edge stream
//            (psi_internal.cuh).  Each warp owns a contiguous range of 256-edge chunks
//            (balanced on edges + rows at ingest, so power-law row lengths do not matter,
//            SURVEY §7) and works independently of the other warps: per chunk each lane
//            holds 8 consecutive edge words (two 128-bit loads), issues 8 independent
//            8-byte gathers of x_{t-1}, reduces them by the row-start flags in registers,
//            and a warp segmented scan (shuffles) carries partial row sums across lanes and,
//            through a register, across chunks.  Completed row sums go through a per-warp
//            shared-memory slot array to a lane-parallel epilogue that writes
//            x_t = a + g*S and accumulates Wt*|x_t - x_{t-1}| for eps_t (Eq. (15)).  The
//            gathers of chunk c+1 and the edge words of chunk c+2 are in flight while chunk
//            c is reduced.  No block barrier inside the loop.
//  k_fix     finishes the rows that cross warp ranges (p_out of the first warp + p_in of
//            the following ones, in warp order), then the LAST CTA to arrive reduces the
//            per-CTA eps partials in a fixed order, appends eps_t to the history, updates
//            gap = ||B|| eps_t (Alg. 2), t += 1, and sets the graph's WHILE
//            condition (gap > eps && t < max_iters): the stop rule of Eq. (16) / Alg. 2
//            line 320 without a host round trip.
//
// The readout (Alg. 2) is the same pair of kernels with the epilogue
// psi_j = (d_j + lambda_j S_j) / N.
//
// Determinism: no floating-point atomics; chunk -> warp assignment is static and every
// reduction has a fixed order, so two runs give bitwise identical psi and eps_t.
#include "psi_internal.cuh"

namespace psi {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kLabelMask = 0x7fffffffu;

// ---- L2 cache policies (createpolicy + .L2::cache_hint).  Streams read once per sweep
// (edge words, per-row constants) are evict_first and bypass L1, so they do not push the
// hot prefix of x out of L2; gathers and stores of x labels below hot_lim (the
// most-gathered users) are evict_last.
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_stream4(const unsigned* p, unsigned long long pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned ld_stream(const unsigned* p, unsigned long long pol) {
  unsigned v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_hint(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
}

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

// Epilogue for one completed row r with S = sum of x_{t-1} over its followers.
template <bool READOUT>
__device__ __forceinline__ void row_epilogue(const SweepArgs& A, int r, double S,
                                             const double* __restrict__ xs, double* __restrict__ xd,
                                             unsigned hot_lim, unsigned long long pf,
                                             unsigned long long pl, double& eps_acc) {
  if (READOUT) {
    A.psi[r] = (ld_stream(A.d + r, pf) + ld_stream(A.lam + r, pf) * S) / A.n_users;
  } else {
    const unsigned long long px = (unsigned)r < hot_lim ? pl : pf;
    const double xn = fma(ld_stream(A.g + r, pf), S, ld_stream(A.a + r, pf));
    eps_acc += ld_stream(A.wt + r, pf) * fabs(xn - ld_hint(xs + r, px));
    st_hint(xd + r, xn, px);
  }
}

// Persistent warp-stream sweep: warp gw processes chunks [warp_chunk[gw], warp_chunk[gw+1]).
// Software pipeline per warp: the gathers of chunk c+1 are in flight while chunk c is
// reduced and its rows' epilogue runs; the edge words of chunk c+2 are prefetched.
template <bool READOUT>
__global__ void __launch_bounds__(kBlock, 4) k_stream(SweepArgs A) {
  __shared__ double rowsum[kWarps][kChunk + 1];   // slot 0: row open at chunk start
  __shared__ double red[33];
  const long long t = A.st->iter;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;    // x_{t-1}
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;          // x_t
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarps + warp;
  const unsigned long long pf = pol_evict_first(), pl = pol_evict_last();
  const unsigned hot_lim = (unsigned)A.hot_lim;
  double* rs = rowsum[warp];
  double eps_acc = 0.0;

  if (gw < A.nwarps) {
    const int c_beg = A.warp_chunk[gw], c_end = A.warp_chunk[gw + 1];
    int row = A.warp_row[gw];          // flags before the current chunk = next row to start
    double carry = 0.0;                // partial of the open row (row - 1)
    bool open_is_split = false;        // open row began before this warp's range
    bool pending_first = true;         // no row flag seen yet in this range (warp-uniform)
    bool has_pin = false;              // this lane closed the split-in row
    double p_in = 0.0;
    if (c_beg < c_end) {
      const unsigned* base = A.edges + (size_t)c_beg * kChunk + lane * kEpt;
      uint4 u0 = ld_stream4(base, pf), u1 = ld_stream4(base + 4, pf);
      open_is_split = !(__shfl_sync(kFull, u0.x, 0) & kRowFlag);
      // gathers of the first chunk
      unsigned w[kEpt] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
      double v[kEpt];
      unsigned fl = 0;
#pragma unroll
      for (int q = 0; q < kEpt; ++q) {
        const unsigned lab = w[q] & kLabelMask;
        fl |= (w[q] >> 31) << q;
        v[q] = ld_hint(xs + lab, lab < hot_lim ? pl : pf);
      }
      if (c_beg + 1 < c_end) {
        const unsigned* p = A.edges + (size_t)(c_beg + 1) * kChunk + lane * kEpt;
        u0 = ld_stream4(p, pf);
        u1 = ld_stream4(p + 4, pf);
      }
      for (int c = c_beg; c < c_end; ++c) {
        // ---- issue chunk c+1's gathers and chunk c+2's edge words before reducing chunk c
        double vn[kEpt];
        unsigned fln = 0;
        if (c + 1 < c_end) {
          const unsigned wn[kEpt] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
          for (int q = 0; q < kEpt; ++q) {
            const unsigned lab = wn[q] & kLabelMask;
            fln |= (wn[q] >> 31) << q;
            vn[q] = ld_hint(xs + lab, lab < hot_lim ? pl : pf);
          }
          if (c + 2 < c_end) {
            const unsigned* p = A.edges + (size_t)(c + 2) * kChunk + lane * kEpt;
            u0 = ld_stream4(p, pf);
            u1 = ld_stream4(p + 4, pf);
          }
        }

        // ---- lane-local reduction by row flags
        const int nf = __popc(fl);
        double run = 0.0;
#pragma unroll
        for (int q = 0; q < kEpt; ++q) {
          if ((fl >> q) & 1u) run = 0.0;
          run += v[q];
        }
        // ---- warp segmented scan of (has flag, open-row partial) and of flag counts
        int f_in = nf > 0, n_in = nf;
        double v_in = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int n2 = __shfl_up_sync(kFull, n_in, o);
          const double v2 = __shfl_up_sync(kFull, v_in, o);
          const int f2 = __shfl_up_sync(kFull, f_in, o);
          if (lane >= o) {
            n_in += n2;
            if (!f_in) v_in += v2;
            f_in |= f2;
          }
        }
        const double v_full = f_in ? v_in : carry + v_in;
        const double v_prev = __shfl_up_sync(kFull, v_full, 1);
        const int F = __shfl_sync(kFull, n_in, 31);          // rows started in this chunk
        const int n_ex = n_in - nf;
        // ---- emit completed rows: slot s <-> row (row - 1 + s)
        int slot = n_ex;
        run = lane == 0 ? carry : v_prev;
#pragma unroll
        for (int q = 0; q < kEpt; ++q) {
          if ((fl >> q) & 1u) {
            if (slot == 0 && pending_first) {              // the range's first flag
              if (open_is_split) { p_in = run; has_pin = true; }
            } else {
              rs[slot] = run;
            }
            ++slot;
            run = 0.0;
          }
          run += v[q];
        }
        carry = __shfl_sync(kFull, v_full, 31);              // partial of the new open row
        __syncwarp();
        // ---- epilogue over the rows completed in this chunk (rows row-1 .. row+F-2)
        const int s_lo = pending_first ? 1 : 0;        // slot 0 = previous warp's / split row
        for (int s = s_lo + lane; s < F; s += 32)
          row_epilogue<READOUT>(A, row - 1 + s, rs[s], xs, xd, hot_lim, pf, pl, eps_acc);
        if (F > 0) pending_first = false;
        row += F;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kEpt; ++q) v[q] = vn[q];
        fl = fln;
      }
    }
    // ---- the open row at the end of the range: complete here, or split (k_fix)
    const unsigned pin_lane = __ballot_sync(kFull, has_pin);
    p_in = pin_lane ? __shfl_sync(kFull, p_in, __ffs(pin_lane) - 1) : 0.0;
    const bool any_flag = !pending_first;
    if (lane == 0) {
      bool next_flag = true;
      if (c_end < A.nchunks) next_flag = (ld_stream(A.edges + (size_t)c_end * kChunk, pf) & kRowFlag) != 0;
      if (!any_flag) {
        A.p_in[gw] = carry;                       // whole range inside one row
        A.p_out[gw] = 0.0;
      } else {
        A.p_in[gw] = p_in;
        if (next_flag) {
          A.p_out[gw] = 0.0;
          if (c_beg < c_end) row_epilogue<READOUT>(A, row - 1, carry, xs, xd, hot_lim, pf, pl, eps_acc);
        } else {
          A.p_out[gw] = carry;
        }
      }
    }
  }

  if (!READOUT) {
    const double tot = block_sum<kBlock>(eps_acc, red);
    if (threadIdx.x == 0) A.eps_part1[blockIdx.x] = tot;
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
    double S = A.p_out[sp.y];
    for (int k = sp.y + 1; k <= sp.z; ++k) S += A.p_in[k];
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

int sweep_grid() {
  static int occ = -1, sms = 0;
  if (occ < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<false>, kBlock, 0);
    if (occ < 1) occ = 1;
  }
  return sms * occ;
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
  return readout ? (void*)k_stream<true> : (void*)k_stream<false>;
}
void* fix_kernel_ptr(bool readout) {
  return readout ? (void*)k_fix<true> : (void*)k_fix<false>;
}
void* init_kernel_ptr() { return (void*)k_init; }

}  // namespace psi
