// psi_sweep.cu -- the Power-psi sweep, fused L1 residual + stop rule, and readout (sm_100a).
//
// One sweep = k_heavy (psi_heavy.cu, graphs with heavy rows) + two launches inside the
// CUDA-graph WHILE loop (psi_api.cu); small graphs run the whole loop in k_solve below:
//
//  k_tiles   persistent, edge-balanced gather-SpMV over the flagged edge stream
//            (psi_internal.cuh).  Tile k = edges [k*tile, (k+1)*tile), tile = 1024 (8 groups
//            of 128 threads per CTA) or 512 (15 groups of 64; graphs without heavy rows):
//            every group does the same number of gathers whatever the power-law row lengths
//            (SURVEY §7).  Per
//            tile each thread loads 8 consecutive edge words (two 128-bit loads, prefetched
//            one tile ahead), issues 8 independent 8-byte gathers of x_{t-1}, reduces its
//            values by the row-start flags in registers, and a block-wide segmented scan
//            (warp shuffles + one smem step) carries partial row sums across threads.
//            Row sums land in shared memory; a row-parallel epilogue then writes
//            x_t = a + g*S coalesced and accumulates Wt*|x_t - x_{t-1}| for eps_t (Eq. (15)).
//            Rows that continue across tile boundaries leave two partials per tile
//            (p_in: the row open at the tile start; p_out: the last row started in it).
//  k_fix     finishes the rows cut by tile boundaries (p_out of the first tile + p_in of
//            the following ones, in tile order), then the LAST CTA to arrive reduces the
//            per-CTA eps partials in a fixed order, appends eps_t to the history, updates
//            gap = ||B|| eps_t (Alg. 2), t += 1, and sets the graph's WHILE
//            condition (gap > eps && t < max_iters): the stop rule of Eq. (16) / Alg. 2
//            line 320 without a host round trip.
//
// The readout (Alg. 2) is the same pair of kernels with the epilogue
// psi_j = (d_j + lambda_j S_j) / N.
//
// Determinism: no floating-point atomics; tile -> CTA assignment is static and every
// reduction has a fixed order, so two runs give bitwise identical psi and eps_t.
#include "psi_internal.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

namespace psi {
namespace cg = cooperative_groups;
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
__device__ __forceinline__ double ld_hint_na(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_l1first(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_l1last(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// 256-bit streaming load of 8 index words (sm_100 .v8): read once per sweep; L2 evict_first
__device__ __forceinline__ void ld_stream8(const unsigned* p, unsigned (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                 "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
// named barrier over one TB-thread tile group of the CTA (id 0 is __syncthreads)
template <int TB>
__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(TB) : "memory");
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

template <int TB>
struct TileSmem {
  double rowsum[TB * kEpt];       // S of the rows started in this tile (local row index)
  double wv[TB / 32];     // warp aggregates of the segmented scan
  int wf[TB / 32];
  int wn[TB / 32];
  double red[33];
  int next_flag;              // does the edge after this tile start a row?
};

// G tile groups of kBlock threads per CTA (named barriers 1..G); the CTA's shared hot
// cache holds x_{t-1}[0, hot_smem): the most-gathered labels, read from
// shared memory instead of L2; all other gathers bypass L1.
// x loads of the sweep: the read-only path (L1, .nc) in a sweep kernel; in the persistent
// small-graph solver (COH) x was written earlier in the same kernel, so L2-coherent loads.
template <bool COH>
__device__ __forceinline__ double ldx(const double* p, unsigned long long pol, int kind) {
  if (COH) return __ldcg(p);
  return kind == 0 ? ld_l1last(p, pol) : kind == 1 ? ld_l1first(p, pol) : ld_hint_na(p, pol);
}

template <bool READOUT, int G, bool COH, int TB>
__device__ __forceinline__ void tiles_body(const SweepArgs& A, unsigned char* dsm, long long t,
                                           double* part1) {
  TileSmem<TB>* smg = reinterpret_cast<TileSmem<TB>*>(dsm);
  double* hot = reinterpret_cast<double*>(dsm + G * sizeof(TileSmem<TB>));
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;    // x_{t-1}
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;          // x_t
  const int grp = G == 1 ? 0 : threadIdx.x / TB;
  const int tid = threadIdx.x - grp * TB, lane = tid & 31, warp = tid >> 5;
  TileSmem<TB>& sm = smg[grp];
  const unsigned long long pf = pol_evict_first(), pl = pol_evict_last();
  const unsigned hot_lim = (unsigned)A.hot_lim;
  const unsigned hs = (unsigned)A.hot_smem;
  const int ntiles = A.ntiles;
  const bool st_last = A.st_last;
  const double* __restrict__ acon = (t == 0 && A.a_first) ? A.a_first : A.a;
  double eps_acc = 0.0;

  for (unsigned i = threadIdx.x; i < hs; i += blockDim.x) hot[i] = __ldcg(xs + i);
  __syncthreads();

  const int stride = gridDim.x * G;
  int k = blockIdx.x * G + grp;
  uint4 u0 = make_uint4(0, 0, 0, 0), u1 = u0;
  if (k < ntiles) {
    const unsigned* p = A.edges + (size_t)k * (TB * kEpt) + tid * kEpt;
    u0 = ld_stream4(p, pf);
    u1 = ld_stream4(p + 4, pf);
  }
  for (; k < ntiles; k += stride) {
    const int f0 = __ldg(A.tile_row + k);
    const int F = __ldg(A.tile_row + k + 1) - f0;      // rows started in this tile
    const unsigned w[kEpt] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};

    // ---- 8 independent gathers of x_{t-1}
    double v[kEpt];
    unsigned fl = 0;
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
#ifdef PSI_EXP_GMASK                                     // experiment builds: x confined to L2
      const unsigned lab = (w[q] & kLabelMask) & (unsigned)(PSI_EXP_GMASK);
#else
      const unsigned lab = w[q] & kLabelMask;
#endif
      PSI_ASSERT((int)lab <= A.n_lab);                  // sentinel label n holds x = 0
      fl |= (w[q] >> 31) << q;
      // one global load variant (L1 bypass, the L2 policy chosen per lane): the L1 classes of
      // k_sell's gx (evict_last hot band, evict_first single-leader users) cost three load
      // instructions per gather here -- C2 0.087 -> 0.083, C3 0.377 -> 0.358 ms without them;
      // only graphs without heavy rows (C5 with the tiles forced: 1 % slower) run this kernel
      if (lab < hs) v[q] = hot[lab];
      else v[q] = ldx<COH>(xs + lab, lab < hot_lim ? pl : pf, 2);
    }
    if (tid == 0)
      sm.next_flag = (k + 1 >= ntiles) ? 1 : (int)(ld_stream(A.edges + (size_t)(k + 1) * (TB * kEpt), pf) >> 31);
    // ---- prefetch the next tile's edge words
    const int kn = k + stride;
    if (kn < ntiles) {
      const unsigned* p = A.edges + (size_t)kn * (TB * kEpt) + tid * kEpt;
      u0 = ld_stream4(p, pf);
      u1 = ld_stream4(p + 4, pf);
    }

    // ---- thread-local reduction by row flags
    const int nf = __popc(fl);
    double run = 0.0;
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
      if ((fl >> q) & 1u) run = 0.0;
      run += v[q];
    }
    // scan element: (has flag, partial of the row open at the thread's end).  Flags and flag
    // counts come from ballots (no integer shuffles): a lane's segment starts at the highest
    // flagged lane <= it, so a Kogge-Stone step adds lane l-o's partial iff l-o >= that start;
    // the inclusive count of row flags is summed over the 4 bit planes of nf (0..8).
    const unsigned le = 0xffffffffu >> (31 - lane);                 // lanes <= this one
    const unsigned below = __ballot_sync(kFull, nf > 0) & le;
    const int start = below ? 31 - __clz(below) : -1;
    int n_in = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) n_in += __popc(__ballot_sync(kFull, (nf >> b) & 1) & le) << b;
    double v_in = run;            // tail if a flag was seen, total otherwise
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v2 = __shfl_up_sync(kFull, v_in, o);
      if (lane >= o && lane - o >= start) v_in += v2;
    }
    const int f_in = start >= 0;
    if (lane == 31) { sm.wv[warp] = v_in; sm.wf[warp] = f_in; sm.wn[warp] = n_in; }
    if (G == 1) __syncthreads(); else group_bar<TB>(1 + grp);
    const int next_flag = sm.next_flag;
    int nP = 0;
    double vP = 0.0;
    for (int w2 = 0; w2 < warp; ++w2) {              // fold of earlier warps, fixed order
      nP += sm.wn[w2];
      vP = sm.wf[w2] ? sm.wv[w2] : vP + sm.wv[w2];
    }
    const double v_full = f_in ? v_in : vP + v_in;
    const double v_prev = __shfl_up_sync(kFull, v_full, 1);
    const double carry = lane == 0 ? vP : v_prev;    // partial of the row open at thread start
    const int n_ex = nP + n_in - nf;                 // flags before this thread in the tile

    // ---- emit completed row sums
    int row = n_ex - 1;                              // local index of the open row
    run = carry;
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
      if ((fl >> q) & 1u) {
        if (row >= 0) sm.rowsum[row] = run;
        else A.p_in[k] = run;                        // first flag of the tile ends row f0-1
        ++row;
        run = 0.0;
      }
      run += v[q];
    }
    if (tid == TB - 1) {                         // the tile's last open row
      if (F == 0) { A.p_in[k] = run; A.p_out[k] = 0.0; }
      else if (next_flag) { sm.rowsum[F - 1] = run; A.p_out[k] = 0.0; }
      else A.p_out[k] = run;
    }
    if (G == 1) __syncthreads(); else group_bar<TB>(1 + grp);

    // ---- epilogue over the rows completed in this tile (coalesced)
    const int nrows = (F > 0 && !next_flag) ? F - 1 : F;
    for (int i = tid; i < nrows; i += TB) {
      const int r = f0 + i;
      PSI_ASSERT(r < A.n_act && i < (TB * kEpt));
      double Sr = sm.rowsum[i];
      if (r < A.n_heavy) {
        if (A.ovl) {                     // k_heavy is still running: k_fix finishes the row
          A.scold[r] = Sr;
          continue;
        }
        Sr += A.hhot[r];                                 // followers < H (k_heavy)
      }
      if (READOUT) {
        A.psi[r] = (ld_stream(A.d + r, pf) + ld_stream(A.lam + r, pf) * Sr) / A.n_users;
      } else {
        const unsigned long long px = (unsigned)r < hot_lim ? pl : pf;
        const double xn = fma(ld_stream(A.g + r, pf), Sr, ld_stream(acon + r, pf));
        const double xp = ldx<COH>(xs + r, px, 2);
        eps_acc += ld_stream(A.wt + r, pf) * fabs(xn - xp);
        st_hint(xd + r, xn, st_last ? px : pf);
      }
    }
  }

  if (!READOUT) {
    const double tot = block_sum<TB * G>(eps_acc, smg[0].red);
    if (threadIdx.x == 0) part1[blockIdx.x] = tot;
  }
}

template <bool READOUT, int G, int TB>
__global__ void __launch_bounds__(TB * G, (1024 / (TB * G)) > 0 ? 1024 / (TB * G) : 1) k_tiles(SweepArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];   // [G x TileSmem][hot cache]
  tiles_body<READOUT, G, false, TB>(A, dsm, A.st->iter, A.eps_part1);
  // overlapped sweep: launched programmatically beside k_heavy (psi_api.cu); complete only
  // after it, so whatever follows k_tiles in stream order also follows k_heavy
  if (A.ovl) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Alg. 2's loop control after the fixed-order reduction of eps_t (one thread): the history,
// gap = ||B|| eps_t (line 325), t + 1, and the graph's WHILE condition (gap > eps && t < max_iters,
// Eq. (16) / line 320) -- no host round trip.
__device__ __forceinline__ void loop_control(const SweepArgs& A, long long t, double eps_sum) {
  const LoopParams P = *A.prm;
  const double eps_t = eps_sum + (t == 0 ? P.eps1_extra : 0.0);
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

// k_sell on a plan with no long rows and no heavy rows (SweepArgs::sell_fused) finishes the
// sweep itself: the last CTA to arrive (atomic ticket) reduces the windows' eps_t partials in a
// fixed order (strided per thread, then a fixed shuffle tree) and runs the loop control, so the
// sweep is ONE launch (no k_fix: C2 -10 us per sweep).  It also resets the work counter.
template <bool READOUT>
__device__ __forceinline__ void sell_finish(const SweepArgs& A, long long t) {
  __shared__ double red[32];
  __shared__ int last;
  __threadfence();                     // this CTA's epsw / x_t / psi stores, before the ticket
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&A.st->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) A.st->sell_next = 0;      // every CTA has made its last claim
  if (READOUT) {
    if (threadIdx.x == 0) A.st->done = 0;
    return;
  }
  // 16 independent loads in flight per thread (one L2 round trip for up to 16K windows at
  // 1024 threads; a dependent strided loop took ~8 us at C2's 15.6K windows)
  double v = 0.0;
  const int nw = A.sell.nwin, step = (int)blockDim.x;
  for (int b = 0; b < nw; b += 16 * step) {
    double q[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = b + k * step + (int)threadIdx.x;
      q[k] = i < nw ? __ldcg(A.sell.epsw + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) v += q[k];
  }
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) loop_control(A, t, r);
  }
}

// ---------------------------------------------------------------- sliced-ELL sweep (k_sell)
// Persistent CTAs of independent warps; work items are claimed one at a time from a device
// counter (LoopState::sell_next): first the pieces of the long rows, then the windows (each of
// bounded size, SellPlan).  A piece: 32 lanes x 8 followers per step, summed by a fixed shuffle
// tree into ppart.  A window:
//   1. lane l streams the window's slices, accumulating its row's gathers x_{t-1}[word] in
//      order (one coalesced 128-byte index load + one gather per step, 8 gathers in flight and
//      the next 8 index words loaded meanwhile) and storing the sum at the row's sorted
//      position in the warp's shared-memory sums at every slice end;
//   2. runs the row-order epilogue over the window (coalesced, as k_tiles') for every row but
//      the long ones (k_fix finishes those from their pieces), and writes the window's eps_t
//      partial to epsw[w] (reduced in a fixed order by k_fix).
// No segmented scans, no flags, no tile barriers: every short row is summed by one lane.
// Deterministic: every sum has a fixed order whatever warp runs an item.
template <bool READOUT, int DEPTH>
__global__ void __launch_bounds__(kSellWarps * 32, 1) k_sell(SweepArgs A) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const SellPlan& P = A.sell;
  const unsigned hs = (unsigned)A.hot_smem;
  double* hot = reinterpret_cast<double*>(dsm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Sw = hot + ((hs + 1) & ~1u) + (size_t)warp * P.wmax;
  const long long t = A.st->iter;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;    // x_{t-1}
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;          // x_t
  const unsigned long long pf = pol_evict_first(), pl = pol_evict_last();
  const unsigned hot_lim = (unsigned)A.hot_lim;
  const unsigned l1_lim = (unsigned)A.l1_lim;
  const unsigned single_lo = (unsigned)A.single_lo;
  const double* __restrict__ acon = (t == 0 && A.a_first) ? A.a_first : A.a;

  for (unsigned i = threadIdx.x; i < hs; i += blockDim.x) hot[i] = __ldcg(xs + i);
  __syncthreads();

  // one gather, as k_tiles': the CTA's shared-memory copy below hs, L1 evict_last below l1_lim,
  // L1 evict_first for the single-leader users (a lane's consecutive steps read consecutive
  // labels there), L1 bypass otherwise; L2 evict_last below hot_lim.  (A branch-free version
  // with predicated loads serialises on the shared destination register, and one load variant
  // under an address-range L2 policy loses the L1 hits: both measured.)
  auto gx = [&](unsigned lab) -> double {
    PSI_ASSERT((int)lab <= A.n_lab);
#ifdef PSI_EXP_GMASK                                     // experiment builds: x confined to L2
    lab &= (unsigned)(PSI_EXP_GMASK);
#endif
    if (lab < hs) return hot[lab];
    if (lab < l1_lim) return ld_l1last(xs + lab, pl);
    if (lab >= single_lo) return ld_l1first(xs + lab, pf);
    return ld_hint_na(xs + lab, lab < hot_lim ? pl : pf);
  };

  const int nitems = P.npieces + P.nwin;
  int it = 0;
  if (lane == 0) it = (int)atomicAdd(&A.st->sell_next, 1u);
  it = __shfl_sync(kFull, it, 0);
  while (it < nitems) {
    int nxt = 0;                                   // claim the next item early
    if (lane == 0) nxt = (int)atomicAdd(&A.st->sell_next, 1u);
    if (it < P.npieces) {
      // ---- a piece of a long row
      const int2 pc = P.piece[it];
      PSI_ASSERT(pc.x >= 0 && pc.y > 0 && pc.x + (long long)pc.y <= P.nlwords);
      const unsigned* pw = P.lwords + pc.x;
      double acc = 0.0;
      for (int k = 0; k < pc.y; k += 256) {
        unsigned w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int j = k + q * 32 + lane;
          w[q] = j < pc.y ? ld_stream(pw + j, pf) : 0xffffffffu;
        }
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = w[q] != 0xffffffffu ? gx(w[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
      }
      acc = warp_sum(acc);
      if (lane == 0) P.ppart[it] = acc;
    } else {
      // ---- a window
      const int w = it - P.npieces;
      const int r0 = __ldg(P.wrow + w), r1 = __ldg(P.wrow + w + 1);
      const int gs0 = r0 >> 5;
      const int nsl = (r1 - r0) >> 5;                // slices of the window (<= 32)
      // slice s ends at soff[gs0 + s + 1]: lane l holds soff[gs0 + l] (l <= nsl)
      const unsigned offl = lane <= nsl ? __ldg(P.soff + gs0 + lane) : 0u;
      const unsigned off0 = __shfl_sync(kFull, offl, 0);
      const unsigned offe = __ldg(P.soff + gs0 + nsl);
      const int K = (int)(offe - off0);              // steps of the whole window
      PSI_ASSERT(nsl >= 1 && nsl <= 32 && (r1 - r0) <= P.wmax && off0 <= offe &&
                 ((long long)__ldg(P.wstep + w) + ((K + 7) & ~7)) * 32 <= P.nwords);
      // lane l streams its steps k < K, 8 per 32-byte load, with the index words of the next
      // two blocks in flight while this block's 8 gathers are (one block ahead left the
      // gathers waiting on DRAM-latency index loads: C5 2.65 -> 1.98 ms), and cuts its running
      // sum at the slice ends (uniform branches)
      const unsigned ws0 = __ldg(P.wstep + w);
      const unsigned* pw = P.words + (size_t)ws0 * 32 + lane * 8;
      int s = 0;
      int end = (int)(__shfl_sync(kFull, offl, 1) - off0);   // end of slice 0
      double acc = 0.0;
      unsigned wb[DEPTH][8];                         // index words of blocks k .. k + 8(D-1)
#pragma unroll
      for (int d = 0; d < DEPTH; ++d)
        if (K > 8 * d) ld_stream8(pw + 256 * d, wb[d]);
      for (int k = 0; k < K; k += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = k + q < K ? gx(wb[0][q]) : 0.0;
#pragma unroll
        for (int d = 0; d + 1 < DEPTH; ++d)
#pragma unroll
          for (int q = 0; q < 8; ++q) wb[d][q] = wb[d + 1][q];
        if (k + 8 * DEPTH < K) ld_stream8(pw + (size_t)(k + 8 * DEPTH) * 32, wb[DEPTH - 1]);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (k + q == end && end < K) {             // slice s ends
            PSI_ASSERT(s + 1 < nsl);
            Sw[s * 32 + lane] = acc;
            acc = 0.0;
            ++s;
            const unsigned oe = __shfl_sync(kFull, offl, (s + 1) & 31);
            end = (int)((s + 1 < 32 ? oe : offe) - off0);
          }
          acc += v[q];
        }
      }
      if (K > 0) Sw[s * 32 + lane] = acc;
      __syncwarp();
      // ---- row-order epilogue over the window (coalesced); long rows are k_fix's
      const int nr = min(r1, A.n_act) - r0;
      double eps_acc = 0.0;
      for (int i = lane; i < nr; i += 32) {
        const int r = r0 + i;
        const unsigned ip = __ldg(P.ipos + r);
        if (ip == 0xffffu) continue;
        PSI_ASSERT(ip < (unsigned)(r1 - r0));
        double Sr = Sw[ip];
        if (r < A.n_heavy) Sr += A.hhot[r];                  // followers < H (k_heavy)
        if (READOUT) {
          A.psi[r] = (ld_stream(A.d + r, pf) + ld_stream(A.lam + r, pf) * Sr) / A.n_users;
        } else {
          const unsigned long long px = (unsigned)r < hot_lim ? pl : pf;
          const double xn = fma(ld_stream(A.g + r, pf), Sr, ld_stream(acon + r, pf));
          const double xp = ld_hint_na(xs + r, px);
          eps_acc += ld_stream(A.wt + r, pf) * fabs(xn - xp);
          st_hint(xd + r, xn, A.st_last ? px : pf);
        }
      }
      if (!READOUT) {
        eps_acc = warp_sum(eps_acc);
        if (lane == 0) P.epsw[w] = eps_acc;
      }
      __syncwarp();
    }
    it = __shfl_sync(kFull, nxt, 0);
  }
  if (A.sell_fused) sell_finish<READOUT>(A, t);
}

// Split rows, eps_t and the stop rule (k_fix), as a device function of any block size >= 32
// (NT = block size).  p_in / p_out / x are read L2-coherently: in the persistent solver they
// were written earlier in the same kernel by other CTAs.
// COOP: only the per-CTA partial is written (the persistent solver reduces after a grid barrier).
template <bool READOUT, int NT, bool COOP = false>
__device__ __forceinline__ void fix_body(const SweepArgs& A, long long t, double* part2) {
  __shared__ double red[33];
  __shared__ int last;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;
  double* __restrict__ xd = (t & 1) ? A.x0 : A.x1;
  const int tid = threadIdx.x;
  double eps_acc = 0.0;

  if (blockIdx.x == 0 && tid == 0) {       // k_heavy / k_sell of this launch are done
    A.st->heavy_next = 0;
    A.st->sell_next = 0;
  }
  auto finish = [&](int r, double S) {
    if (r < A.n_heavy) S += A.hhot[r];
    if (READOUT) {
      A.psi[r] = (A.d[r] + A.lam[r] * S) / A.n_users;
    } else {
      const double xn = fma(A.g[r], S, ((t == 0 && A.a_first) ? A.a_first : A.a)[r]);
      eps_acc += A.wt[r] * fabs(xn - __ldcg(xs + r));
      xd[r] = xn;
    }
  };
  // rows spanning more than kLongSpan tiles: a warp each (lane-strided, fixed shuffle tree)
  const int lane = tid & 31;
  for (int s = (blockIdx.x * NT + tid) >> 5; s < A.nsplit_long; s += gridDim.x * (NT / 32)) {
    const int4 sp = A.split[s];
    PSI_ASSERT(sp.x < A.n_act && sp.y <= sp.z && sp.z < A.ntiles);
    double S = 0.0;
    for (int k = sp.y + 1 + lane; k <= sp.z; k += 32) S += __ldcg(A.p_in + k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    if (lane == 0) finish(sp.x, __ldcg(A.p_out + sp.y) + S);
  }
  for (int s = A.nsplit_long + blockIdx.x * NT + tid; s < A.nsplit; s += gridDim.x * NT) {
    const int4 sp = A.split[s];
    PSI_ASSERT(sp.x < A.n_act && sp.y <= sp.z && sp.z < A.ntiles);
    double S = __ldcg(A.p_out + sp.y);
    for (int k = sp.y + 1; k <= sp.z; ++k) S += __ldcg(A.p_in + k);
    finish(sp.x, S);
  }
  if (A.use_sell) {
    // k_sell's long rows: their pieces in piece order (+ hhot)
    const SellPlan& P = A.sell;
    for (int i = blockIdx.x * NT + tid; i < P.nlong; i += gridDim.x * NT) {
      const int p0 = P.lp0[i], p1 = P.lp0[i + 1];
      PSI_ASSERT(p0 < p1 && p1 <= P.npieces);
      double S = 0.0;
      for (int q = p0; q < p1; ++q) S += __ldcg(P.ppart + q);
      finish(P.lrow[i], S);
    }
  }
  if (A.ovl) {
    // overlapped sweep: the heavy rows k_tiles completed inside a tile (their edge-stream sum
    // in scold) are finished here, once k_heavy's hhot exists; split heavy rows were above
    for (int r = blockIdx.x * NT + tid; r < A.n_heavy; r += gridDim.x * NT)
      if (!((__ldg(A.hsplit + (r >> 5)) >> (r & 31)) & 1u)) finish(r, __ldcg(A.scold + r));
  }
  if (READOUT) return;
  // k_sell: the windows' eps_t partials, in a fixed partition and order
  if (A.use_sell)
    for (int i = blockIdx.x * NT + tid; i < A.sell.nwin; i += gridDim.x * NT)
      eps_acc += __ldcg(A.sell.epsw + i);

  const double tot = block_sum<NT>(eps_acc, red);
  if (COOP) {
    if (tid == 0) part2[blockIdx.x] = tot;
    return;
  }
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
  for (int q = tid; q < A.grid1; q += NT) v += __ldcg(A.eps_part1 + q);
  const double e1 = block_sum<NT>(v, red);
  v = 0.0;
  for (int q = tid; q < (int)gridDim.x; q += NT) v += __ldcg(A.eps_part2 + q);
  const double e2 = block_sum<NT>(v, red);
  if (tid == 0) loop_control(A, t, e1 + e2);
}

template <bool READOUT>
__global__ void __launch_bounds__(kFixBlock) k_fix(SweepArgs A) {
  fix_body<READOUT, kFixBlock>(A, A.st->iter, A.eps_part2);
}

// x_0 = a (s_0 = c, Alg. 2 line 1), t = 0, gap = 1 (line 4), WHILE condition = (1 > eps).
// Only active users are reset: follower-less users hold x = a0 in both buffers forever.
__global__ void k_init(SweepArgs A, int n) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_act; i += stride) A.x0[i] = A.a0[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.st->iter = 0;
    A.st->gap = A.prm->gap0;
    A.st->eps_t = 0.0;
    A.st->done = 0;
    A.st->status = 0;
    A.st->heavy_next = 0;
    A.st->sell_next = 0;
    const LoopParams P = *A.prm;
    if (A.use_cond) cudaGraphSetConditional(A.cond, (P.gap0 > P.eps && P.max_iters > 0) ? 1u : 0u);
  }
}


// Persistent small-graph solver (graphs with no k_heavy rows, few tiles): the whole of Alg. 2
// -- x_0 = a, the WHILE loop of {sweep, eps_t + stop rule}, the readout -- as ONE cooperative
// launch with grid-wide barriers between the phases, instead of a CUDA-graph WHILE node with
// two kernel launches per sweep.  Same arithmetic, same fixed-order reductions and the same
// stop rule as k_init / k_tiles / k_fix (sweep counts and results agree with the graph path).
template <int G, int TB>
__global__ void __launch_bounds__(TB * G, 1) k_solve(SweepArgs A, int readout) {
  extern __shared__ __align__(16) unsigned char dsm[];
  cg::grid_group grid = cg::this_grid();
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_act; i += stride) A.x0[i] = A.a0[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.st->iter = 0;
    A.st->gap = A.prm->gap0;
    A.st->eps_t = 0.0;
    A.st->done = 0;
    A.st->status = 0;
    A.st->heavy_next = 0;
  }
  grid.sync();
  const LoopParams P = *A.prm;
  __shared__ double red[33];
  long long t = 0;
  double gap = P.gap0;
  bool bad = false;
  // Every CTA reduces the eps_t partials itself, in the same fixed order as k_fix, so all CTAs
  // take the same stop decision without a ticket or a third barrier; CTA 0 publishes the
  // LoopState.  The partials are double-buffered by the parity of t: a CTA can be one sweep
  // ahead of another one still reducing.
  while (!bad && gap > P.eps && t < P.max_iters) {
    double* p1 = A.eps_part1 + (t & 1) * A.grid1;
    double* p2 = A.eps_part2 + (t & 1) * gridDim.x;
    tiles_body<false, G, true, TB>(A, dsm, t, p1);
    grid.sync();
    fix_body<false, TB * G, true>(A, t, p2);
    grid.sync();
    double v = 0.0;
    for (int q = threadIdx.x; q < A.grid1; q += blockDim.x) v += __ldcg(p1 + q);
    const double e1 = block_sum<TB * G>(v, red);
    v = 0.0;
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) v += __ldcg(p2 + q);
    const double e2 = block_sum<TB * G>(v, red);
    const double eps_t = e1 + e2 + (t == 0 ? P.eps1_extra : 0.0);
    gap = P.kappa * eps_t;
    bad = !isfinite(eps_t);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (t < P.hist_cap) P.history[t] = eps_t;
      A.st->eps_t = eps_t;
      A.st->gap = gap;
      A.st->iter = t + 1;
      if (bad) A.st->status |= 1;
    }
    ++t;
  }
  if (readout) {
    tiles_body<true, G, true, TB>(A, dsm, t, nullptr);
    grid.sync();
    fix_body<true, TB * G>(A, t, nullptr);
  }
}

}  // namespace

namespace {
template <int G, int TB>
TilesCfg cfg_for(int ntiles, long long n, int hot_req, int l1_req) {
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  TilesCfg c{};
  c.groups = G;
  c.block = TB * G;
  const size_t fixed = G * sizeof(TileSmem<TB>);
  long long hs = hot_req;
  const long long cap = ((long long)optin - (long long)fixed - 1024) / 8;
  if (hs > cap) hs = cap;
  if (hs > n + 1) hs = n + 1;                         // labels 0..n (n = zero sentinel)
  if (hs < 0) hs = 0;
  c.hot_smem = (int)hs;
  c.l1_lim = (int)std::max<long long>(hs, std::min<long long>(l1_req, n + 1));
  c.smem = fixed + (size_t)hs * 8;
  c.sweep = (void*)k_tiles<false, G, TB>;
  c.solve = (void*)k_solve<G, TB>;
  cudaFuncSetAttribute(k_solve<G, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  int occ_s = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_solve<G, TB>, c.block, c.smem);
  c.solve_max_grid = occ_s * sms;
  c.readout = (void*)k_tiles<true, G, TB>;
  cudaFuncSetAttribute(k_tiles<false, G, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  cudaFuncSetAttribute(k_tiles<true, G, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiles<false, G, TB>, c.block, c.smem);
  if (occ < 1) occ = 1;
  long long g = (long long)sms * occ;
  if (g * G > ntiles) g = (ntiles + G - 1) / G;
  c.grid = g < 1 ? 1 : (int)g;
  return c;
}
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}
}  // namespace

// Launch shape of the sweep/readout kernel.  Defaults from the C5 measurements in
// DESIGN.md §12; PSI_GROUPS / PSI_SMEM_HOT / PSI_L1_HOT override them (tuning only).
TilesCfg tiles_config(int ntiles, long long n, int tile, bool ovl) {
  if (ovl) {
    // overlapped sweep: one k_tiles CTA beside one k_heavy CTA on every SM -- 4 groups of
    // 128 threads (1024-edge tiles) and a 2048-label shared-memory hot cache
    TilesCfg c = cfg_for<4, 128>(ntiles, n, env_int("PSI_OVL_SMEM_HOT", 2048),
                                 env_int("PSI_L1_HOT", kDefaultL1Hot));
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (c.grid > sms) c.grid = sms;
    c.solve = nullptr;
    return c;
  }
  const int hot = env_int("PSI_SMEM_HOT", kDefaultSmemHot);
  const int l1 = env_int("PSI_L1_HOT", kDefaultL1Hot);
  if (tile == 512) {
    // 15 groups of 64 threads (barrier ids 1..15): one CTA and one hot cache per SM.  Large
    // graphs without heavy rows take a 12288-label hot cache: with every other gather
    // bypassing L1, the shared-memory copy is where the hubs' gathers are served on chip
    // (C3: 0.359 -> 0.343 ms; 8192: 0.347, 16384: 0.355, 20480: 0.601 -- L1 too small for
    // the stream; profiles/r2/tune_c3_smemhot_s4e.txt).  Small graphs keep 4096: the copy is
    // re-read every sweep, by k_solve too.
    const int hot512 = env_int("PSI_SMEM_HOT", n >= (1LL << 22) ? kSmemHotLarge512 : kDefaultSmemHot);
    return cfg_for<15, 64>(ntiles, n, hot512, l1);
  }
  const int G = env_int("PSI_GROUPS", kDefaultGroups);
  switch (G) {
    case 4: return cfg_for<4, 128>(ntiles, n, hot, l1);
    default: return cfg_for<8, 128>(ntiles, n, hot, l1);
  }
}

// Launch shape of k_sell: one CTA of kSellWarps warps per SM, the hot cache of x_{t-1} and
// every warp's window sums in shared memory (PSI_SMEM_HOT / PSI_L1_HOT as for k_tiles).
TilesCfg sell_config(long long n, int shift) {
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  TilesCfg c{};
  c.groups = 1;
  long long hs = env_int("PSI_SMEM_HOT", kDefaultSmemHot);
  // warps per CTA: kSellWarps (PSI_SELL_WARPS), halved until their window sums and the hot
  // cache fit in shared memory
  int warps = std::min(std::max(env_int("PSI_SELL_WARPS", kSellWarps), 1), 32);
  while (warps > 1 && (size_t)warps * ((size_t)8 << shift) + (size_t)std::max(hs, 0LL) * 8 + 1024 >
                          (size_t)optin)
    warps /= 2;
  c.block = warps * 32;
  const size_t fixed = (size_t)warps * ((size_t)8 << shift);
  const long long cap = ((long long)optin - (long long)fixed - 1024) / 8 - 2;
  if (hs > cap) hs = cap;
  if (hs > n + 1) hs = n + 1;
  if (hs < 0) hs = 0;
  c.hot_smem = (int)hs;
  c.l1_lim = (int)std::max<long long>(hs, std::min<long long>(env_int("PSI_L1_HOT", kDefaultL1Hot), n + 1));
  c.smem = fixed + (size_t)((hs + 1) & ~1LL) * 8;
  // two index blocks in flight per lane (three measured equal)
  c.sweep = (void*)k_sell<false, 2>;
  c.readout = (void*)k_sell<true, 2>;
  c.solve = nullptr;
  c.solve_max_grid = 0;
  cudaFuncSetAttribute(c.sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  cudaFuncSetAttribute(c.readout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.sweep, c.block, c.smem);
  if (occ < 1) occ = 1;
  c.grid = sms * occ;
  if (env_int("PSI_SELL_GRID", 0) > 0) c.grid = std::min(c.grid, env_int("PSI_SELL_GRID", 0));
  return c;
}

int fix_grid(int nsplit) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long g = ((long long)nsplit + kFixBlock - 1) / kFixBlock;
  if (g > (long long)sms * 4) g = (long long)sms * 4;
  return g < 1 ? 1 : (int)g;
}

void* fix_kernel_ptr(bool readout) {
  return readout ? (void*)k_fix<true> : (void*)k_fix<false>;
}
void* init_kernel_ptr() { return (void*)k_init; }

}  // namespace psi
