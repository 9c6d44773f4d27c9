// psi_batch.cu -- the Power-psi sweep for kBP = 4 activity profiles at once (sm_100a).
//
// SURVEY §8(f) row 4 ("multi-profile batching: k activity profiles sharing one index stream").
// Alg. 2 depends on the activity (lambda, mu) only through the per-user
// constants a, g, Wt, d (§5 of DESIGN.md); the follower lists F(j) -- the edge stream, the
// tiles, the split rows -- are the graph's.  So kBP profiles share one pass over the edge
// stream: x is stored interleaved, x[label] = (x^(0), .., x^(3)) in one 32-byte sector, and
// every edge costs ONE 256-bit gather (`LDG.E.256`) for four profiles instead of one 8-byte
// gather per profile.  The random-gather bound of the single-profile sweep is one L1
// wavefront and one 32-byte L2/DRAM sector per gather, so the batch moves four
// useful values per sector where the single-profile sweep moves one.
//
// Per profile p the arithmetic is exactly the single-profile kernels' (k_tiles / k_fix):
//     S_j = sum_{n in F(j)} x_{t-1,n}^(p),  x_t,j^(p) = a_j^(p) + g_j^(p) S_j
//     eps_t^(p) = sum_j Wt_j^(p) |x_t,j^(p) - x_{t-1,j}^(p)|,  gap^(p) = kappa_row^(p) eps_t^(p)
// and every profile stops on its OWN rule (Alg. 2): once gap^(p) <= eps (or
// t = max_iters) profile p is frozen -- its x is copied forward unchanged, so both ping-pong
// buffers hold x_{T_p}^(p) and the shared readout psi^(p) = (d' + lambda S)/N is that of T_p.
// The loop runs while any profile of the group is active.  Fixed-order reductions, no fp
// atomics: bitwise deterministic.
#include "psi_internal.cuh"

#include <algorithm>

namespace psi {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned kLabelMask = 0x7fffffffu;
constexpr int kTB = kTileB / 4;        // threads per tile (4 edges each)
constexpr int kEB = kTileB / kTB;      // 4 edges per thread
constexpr int kWB = kTB / 32;
constexpr int kBHot = 1024;            // labels of x_{t-1} (x 4 profiles) in shared memory
constexpr int kFixB = 256;
constexpr int kGB = 1024 / kTB;        // tile groups per CTA (named barriers 1..kGB)
static_assert(kEB == 4, "one 128-bit index load per thread");

__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_idx4(const unsigned* p, unsigned long long pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned ld_idx(const unsigned* p, unsigned long long pol) {
  unsigned v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// one 32-byte sector: the four profiles' values of one user
__device__ __forceinline__ d4 ld4(const d4* p, unsigned long long pol) {
  d4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st4(d4* p, const d4& r, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "d"(r.v[0]), "d"(r.v[1]), "d"(r.v[2]), "d"(r.v[3]), "l"(pol)
               : "memory");
}
__device__ __forceinline__ d4 ldcg4(const d4* p) {     // L2-coherent (written by other CTAs)
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 lo = __ldcg(q), hi = __ldcg(q + 1);
  d4 r;
  r.v[0] = lo.x; r.v[1] = lo.y; r.v[2] = hi.x; r.v[3] = hi.y;
  return r;
}
__device__ __forceinline__ d4 zero4() {
  d4 r;
#pragma unroll
  for (int p = 0; p < kBP; ++p) r.v[p] = 0.0;
  return r;
}
__device__ __forceinline__ void add4(d4& a, const d4& b) {
#pragma unroll
  for (int p = 0; p < kBP; ++p) a.v[p] += b.v[p];
}
__device__ __forceinline__ d4 shfl_up4(const d4& a, int o) {
  d4 r;
#pragma unroll
  for (int p = 0; p < kBP; ++p) r.v[p] = __shfl_up_sync(kFull, a.v[p], o);
  return r;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
// deterministic block sum of four values (fixed shuffle tree), result to every thread
template <int BLOCK>
__device__ d4 block_sum4(d4 v, double (*red)[33]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int p = 0; p < kBP; ++p) v.v[p] = warp_sum(v.v[p]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int p = 0; p < kBP; ++p) red[p][warp] = v.v[p];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int p = 0; p < kBP; ++p) {
      double r = lane < BLOCK / 32 ? red[p][lane] : 0.0;
      r = warp_sum(r);
      if (lane == 0) red[p][32] = r;
    }
  }
  __syncthreads();
  d4 out;
#pragma unroll
  for (int p = 0; p < kBP; ++p) out.v[p] = red[p][32];
  return out;
}

struct TileSmemB {
  d4 rowsum[kTileB];         // S of the rows started in this tile, four profiles
  d4 wv[kWB];                // warp aggregates of the value scan
  int wf[kWB];
  int wn[kWB];               // warp totals of the row-flag count scan
  int next_flag;
};

// named barrier over one tile group (id 0 is __syncthreads)
__device__ __forceinline__ void grp_bar(int id) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(kTB) : "memory");
}

// kGB tile groups of kTB threads per CTA, one kTileB-edge tile per group pass (its own tiling of the edge stream) (persistent grid).
// Per tile: the gathers are issued first; while they are in flight the row-flag counts are
// scanned (so every thread knows the local index n_ex of the first row it starts); the
// thread's values are then folded in ONE pass -- rows that start and end inside the thread
// go straight to shared memory, leaving only its head (before its first flag) and tail
// (after its last flag) -- which keeps four profiles' gathers in flight within the register
// budget of 1024 threads per SM.  A segmented scan of (has flag, tail | head) gives the carry
// that closes the row ended by each thread's first flag.  Same sums, same order per row as
// k_tiles (edges of a row in stream order).
template <bool READOUT>
__global__ void __launch_bounds__(kTB * kGB, 1) k_tiles_b(BatchArgs A) {
  extern __shared__ __align__(32) unsigned char dsm[];
  TileSmemB* smg = reinterpret_cast<TileSmemB*>(dsm);
  double (*red)[33] = reinterpret_cast<double (*)[33]>(dsm + kGB * sizeof(TileSmemB));
  d4* hot = reinterpret_cast<d4*>(dsm + kGB * sizeof(TileSmemB) + kBP * 33 * sizeof(double));
  const long long t = A.st->iter;
  const unsigned act = A.st->active;
  const d4* __restrict__ xs = (t & 1) ? A.x1 : A.x0;
  d4* __restrict__ xd = (t & 1) ? A.x0 : A.x1;
  const int grp = threadIdx.x / kTB;
  const int tid = threadIdx.x - grp * kTB, lane = tid & 31, warp = tid >> 5;
  TileSmemB& sm = smg[grp];
  const unsigned long long pf = pol_first(), pl = pol_last();
  const unsigned hs = (unsigned)A.hot_smem, hot_lim = (unsigned)A.hot_lim;
  const int ntiles = A.ntiles;
  d4 eps_acc = zero4();

  for (unsigned i = threadIdx.x; i < hs; i += blockDim.x) hot[i] = xs[i];
  __syncthreads();

  const int stride = gridDim.x * kGB;
  int k = blockIdx.x * kGB + grp;
  uint4 u = make_uint4(0, 0, 0, 0);
  if (k < ntiles) u = ld_idx4(A.edges + (size_t)k * kTileB + tid * kEB, pf);
  for (; k < ntiles; k += stride) {
    const int f0 = __ldg(A.tile_row + k);
    const int F = __ldg(A.tile_row + k + 1) - f0;
    const unsigned w[kEB] = {u.x, u.y, u.z, u.w};
    d4 v[kEB];
    unsigned fl = 0;
#pragma unroll
    for (int q = 0; q < kEB; ++q) {
      const unsigned lab = w[q] & kLabelMask;
      PSI_ASSERT((double)lab <= A.n_users);
      fl |= (w[q] >> 31) << q;
      v[q] = lab < hs ? hot[lab] : ld4(xs + lab, lab < hot_lim ? pl : pf);
    }
    if (tid == 0)
      sm.next_flag = (k + 1 >= ntiles) ? 1 : (int)(ld_idx(A.edges + (size_t)(k + 1) * kTileB, pf) >> 31);
    const int kn = k + stride;
    if (kn < ntiles) u = ld_idx4(A.edges + (size_t)kn * kTileB + tid * kEB, pf);

    // ---- row-flag count scan (overlaps the gathers): n_ex = flags before this thread
    const int nf = __popc(fl);
    int n_in = nf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n2 = __shfl_up_sync(kFull, n_in, o);
      if (lane >= o) n_in += n2;
    }
    if (lane == 31) sm.wn[warp] = n_in;
    grp_bar(1 + grp);
    int nP = 0;
    for (int w2 = 0; w2 < warp; ++w2) nP += sm.wn[w2];
    const int n_ex = nP + n_in - nf;

    // ---- one pass over the thread's values: inner rows to shared memory, head and tail kept
    d4 head = zero4(), run = zero4();
    int j = 0;                                       // flags seen
#pragma unroll
    for (int q = 0; q < kEB; ++q) {
      if ((fl >> q) & 1u) {
        if (j == 0) head = run;
        else sm.rowsum[n_ex + j - 1] = run;          // row started at the thread's flag j-1
        ++j;
        run = zero4();
      }
      add4(run, v[q]);
    }
    if (nf == 0) head = run;                         // no flag: everything continues the open row

    // ---- segmented scan of (has flag, tail | head): the open row's partial at each thread
    int f_in = nf > 0;
    d4 v_in = nf > 0 ? run : head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const d4 v2 = shfl_up4(v_in, o);
      const int f2 = __shfl_up_sync(kFull, f_in, o);
      if (lane >= o) {
        if (!f_in) add4(v_in, v2);
        f_in |= f2;
      }
    }
    if (lane == 31) { sm.wv[warp] = v_in; sm.wf[warp] = f_in; }
    grp_bar(1 + grp);
    const int next_flag = sm.next_flag;
    d4 vP = zero4();
    for (int w2 = 0; w2 < warp; ++w2) {
      if (sm.wf[w2]) vP = sm.wv[w2]; else add4(vP, sm.wv[w2]);
    }
    d4 v_full = v_in;
    if (!f_in) { v_full = vP; add4(v_full, v_in); }
    const d4 v_prev = shfl_up4(v_full, 1);
    d4 carry = lane == 0 ? vP : v_prev;              // partial of the row open at thread start
    if (nf > 0) {                                    // the first flag ends row n_ex - 1
      add4(carry, head);
      if (n_ex > 0) sm.rowsum[n_ex - 1] = carry;
      else A.p_in[k] = carry;                        // row f0 - 1 (started in an earlier tile)
    }
    if (tid == kTB - 1) {                            // the tile's last open row
      const d4 last = v_full;
      if (F == 0) { A.p_in[k] = last; A.p_out[k] = zero4(); }
      else if (next_flag) { sm.rowsum[F - 1] = last; A.p_out[k] = zero4(); }
      else A.p_out[k] = last;
    }
    grp_bar(1 + grp);

    // ---- epilogue over the rows completed in this tile (coalesced 32-byte rows)
    const int nrows = (F > 0 && !next_flag) ? F - 1 : F;
    for (int i = tid; i < nrows; i += kTB) {
      const int r = f0 + i;
      PSI_ASSERT(r < A.n_act && i < kTileB);
      const d4 S = sm.rowsum[i];
      if (READOUT) {
        const d4 dd = ld4(A.d + r, pf), lm = ld4(A.lam + r, pf);
        d4 o;
#pragma unroll
        for (int p = 0; p < kBP; ++p) o.v[p] = (dd.v[p] + lm.v[p] * S.v[p]) / A.n_users;
        st4(A.psi + r, o, pf);
      } else {
        const unsigned long long px = (unsigned)r < hot_lim ? pl : pf;
        const d4 gg = ld4(A.g + r, pf), aa = ld4(A.a + r, pf), ww = ld4(A.wt + r, pf);
        const d4 xo = ld4(xs + r, px);
        d4 xn;
#pragma unroll
        for (int p = 0; p < kBP; ++p) {
          const bool on = (act >> p) & 1u;
          xn.v[p] = on ? fma(gg.v[p], S.v[p], aa.v[p]) : xo.v[p];
          eps_acc.v[p] += on ? ww.v[p] * fabs(xn.v[p] - xo.v[p]) : 0.0;
        }
        st4(xd + r, xn, px);
      }
    }
  }
  if (!READOUT) {
    const d4 tot = block_sum4<kTB * kGB>(eps_acc, red);
    if (threadIdx.x == 0) A.eps_part1[blockIdx.x] = tot;
  }
}

// rows crossing tiles, per-profile eps_t, the per-profile stop rule and the WHILE condition
template <bool READOUT>
__global__ void __launch_bounds__(kFixB) k_fix_b(BatchArgs A) {
  __shared__ double red[kBP][33];
  __shared__ int last;
  const long long t = A.st->iter;
  const unsigned act = A.st->active;
  const d4* __restrict__ xs = (t & 1) ? A.x1 : A.x0;
  d4* __restrict__ xd = (t & 1) ? A.x0 : A.x1;
  const int tid = threadIdx.x;
  d4 eps_acc = zero4();
  auto finish = [&](int r, const d4& S) {
    if (READOUT) {
      d4 o;
#pragma unroll
      for (int p = 0; p < kBP; ++p) o.v[p] = (A.d[r].v[p] + A.lam[r].v[p] * S.v[p]) / A.n_users;
      A.psi[r] = o;
    } else {
      const d4 gg = A.g[r], aa = A.a[r], ww = A.wt[r], xo = xs[r];
      d4 xn;
#pragma unroll
      for (int p = 0; p < kBP; ++p) {
        const bool on = (act >> p) & 1u;
        xn.v[p] = on ? fma(gg.v[p], S.v[p], aa.v[p]) : xo.v[p];
        eps_acc.v[p] += on ? ww.v[p] * fabs(xn.v[p] - xo.v[p]) : 0.0;
      }
      xd[r] = xn;
    }
  };
  // rows spanning more than kLongSpan tiles: a warp each (lane-strided, fixed shuffle tree)
  const int lane = tid & 31;
  for (int s = (blockIdx.x * kFixB + tid) >> 5; s < A.nsplit_long; s += gridDim.x * (kFixB / 32)) {
    const int4 sp = A.split[s];
    PSI_ASSERT(sp.x < A.n_act && sp.y <= sp.z && sp.z < A.ntiles);
    d4 S = zero4();
    for (int k = sp.y + 1 + lane; k <= sp.z; k += 32) add4(S, A.p_in[k]);
#pragma unroll
    for (int p = 0; p < kBP; ++p)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) S.v[p] += __shfl_xor_sync(kFull, S.v[p], o);
    if (lane == 0) {
      d4 T = A.p_out[sp.y];
      add4(T, S);
      finish(sp.x, T);
    }
  }
  for (int s = A.nsplit_long + blockIdx.x * kFixB + tid; s < A.nsplit; s += gridDim.x * kFixB) {
    const int4 sp = A.split[s];
    PSI_ASSERT(sp.x < A.n_act && sp.y <= sp.z && sp.z < A.ntiles);
    d4 S = A.p_out[sp.y];
    for (int k = sp.y + 1; k <= sp.z; ++k) add4(S, A.p_in[k]);
    finish(sp.x, S);
  }
  if (READOUT) return;

  const d4 tot = block_sum4<kFixB>(eps_acc, red);
  if (tid == 0) {
    A.eps_part2[blockIdx.x] = tot;
    __threadfence();
    last = atomicAdd(&A.st->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  d4 v = zero4();
  for (int q = tid; q < A.grid1; q += kFixB) add4(v, A.eps_part1[q]);
  const d4 e1 = block_sum4<kFixB>(v, red);
  v = zero4();
  for (int q = tid; q < (int)gridDim.x; q += kFixB) add4(v, ldcg4(A.eps_part2 + q));
  const d4 e2 = block_sum4<kFixB>(v, red);
  if (tid == 0) {
    const BatchParams P = *A.prm;
    unsigned still = act;
#pragma unroll
    for (int p = 0; p < kBP; ++p) {
      if (!((act >> p) & 1u)) continue;
      const double eps_t = e1.v[p] + e2.v[p];
      if (t < P.hist_cap) P.history[t * kBP + p] = eps_t;
      const double gap = P.kappa[p] * eps_t;
      A.st->eps_t[p] = eps_t;
      A.st->gap[p] = gap;
      A.st->T[p] = t + 1;
      const bool bad = !isfinite(eps_t);
      if (bad) A.st->status |= 1 << p;
      if (bad || !(gap > P.eps) || t + 1 >= P.max_iters) still &= ~(1u << p);
    }
    A.st->active = still;
    A.st->iter = t + 1;
    A.st->done = 0;
    if (A.use_cond) cudaGraphSetConditional(A.cond, still ? 1u : 0u);
  }
}

// x_0 = a for the active users, every profile: gap = 1, T = 0, active iff 1 > eps
__global__ void k_init_b(BatchArgs A) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n_act; i += stride) A.x0[i] = A.a0[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const BatchParams P = *A.prm;
    const unsigned on = (1.0 > P.eps && P.max_iters > 0) ? P.valid : 0u;
    A.st->iter = 0;
    A.st->active = on;
    A.st->done = 0;
    A.st->status = 0;
    for (int p = 0; p < kBP; ++p) {
      A.st->gap[p] = 1.0;
      A.st->eps_t[p] = 0.0;
      A.st->T[p] = 0;
    }
    if (A.use_cond) cudaGraphSetConditional(A.cond, on ? 1u : 0u);
  }
}

// out[p * n + old_of_new[r]] = psi of profile p at relabelled user r
__global__ void k_unpermute_b(const double* psi_groups, const int* old_of_new, long long n,
                              int nprof, double* out) {
  const long long total = n * nprof;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(q / n);
    const long long r = q - (long long)p * n;
    const int g = p / kBP, lane = p % kBP;
    out[(long long)p * n + old_of_new[r]] = psi_groups[((size_t)g * n + r) * kBP + lane];
  }
}

}  // namespace

BatchCfg batch_config(int ntiles, long long n, int nsplit) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  BatchCfg c{};
  c.hot_smem = (int)std::min<long long>(kBHot, n + 1);
  c.smem = kGB * sizeof(TileSmemB) + kBP * 33 * sizeof(double) + (size_t)c.hot_smem * sizeof(d4);
  c.block1 = kTB * kGB;
  cudaFuncSetAttribute(k_tiles_b<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  cudaFuncSetAttribute(k_tiles_b<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiles_b<false>, kTB * kGB, c.smem);
  if (occ < 1) occ = 1;
  long long g = std::min<long long>((long long)sms * occ, (ntiles + kGB - 1) / kGB);
  c.grid1 = g < 1 ? 1 : (int)g;
  long long g2 = ((long long)nsplit + kFixB - 1) / kFixB;
  g2 = std::min<long long>(g2, (long long)sms * 4);
  c.grid2 = g2 < 1 ? 1 : (int)g2;
  return c;
}

void* batch_tiles_ptr(bool readout) {
  return readout ? (void*)k_tiles_b<true> : (void*)k_tiles_b<false>;
}
void* batch_fix_ptr(bool readout) { return readout ? (void*)k_fix_b<true> : (void*)k_fix_b<false>; }
void* batch_init_ptr() { return (void*)k_init_b; }
int batch_fix_block() { return kFixB; }

cudaError_t batch_unpermute(const double* psi_groups, const int* old_of_new, long long n, int nprof,
                            double* out, cudaStream_t s) {
  long long g = (n * nprof + 255) / 256;
  g = std::max<long long>(1, std::min<long long>(g, 148LL * 16));
  k_unpermute_b<<<(int)g, 256, 0, s>>>(psi_groups, old_of_new, n, nprof, out);
  return cudaGetLastError();
}

}  // namespace psi
