// psi_heavy.cu -- the staged-segment half of the Power-psi sweep (sm_100a).
//
// Why: every x gather of the edge-stream sweep (k_tiles) is one 32-byte L2
// sector for 8 useful bytes, and random sector reads top out near 281 G/s on B200 -- the
// L2 slices, not HBM, bound a pure gather sweep.  But the rows with many followers
// ("heavy" rows, labels [0, n_heavy) after the ingest relabel) hold most edges, and most of
// their followers are among the hottest labels [0, H).  For those (row, follower) pairs this
// kernel streams x_{t-1}[0, H) through shared memory in segments of kSeg labels with TMA bulk
// copies (cp.async.bulk + mbarrier, one producer warp, kHeavyStages-deep ring) and gathers
// from shared memory instead of L2:
//
//     hhot_r = sum_{n in F(r), n < H} x_{t-1,n}          for r < n_heavy
//
// k_tiles then adds hhot_r to the rest of row r's sum (its followers >= H, still in the edge
// stream) in its epilogue: x_t,r = a_r + g_r (S_r + hhot_r)  (Eq. (14) in kernel state).
//
// Work layout (built by psi_ingest.cu): heavy rows are cut into panels of <= kHeavySlots
// "slots"; a row with many hot followers is spread round-robin over several slots (virtual
// rows) so no warp owns a hub alone.  Each consumer warp owns a contiguous slot range of
// the panel and keeps its slots' partial sums in shared memory, so no two warps ever touch
// the same sum (no atomics).  Entries are u32 words (slot << kSegShift) | (label - s*kSeg),
// grouped in lists (panel, segment, warp) sorted by slot; list starts are 32-byte aligned
// and padded with null words (slot kHeavySlots, a junk sum).  At the panel end the slot sums
// of each row are added in slot order: every reduction has a fixed order (deterministic).
#include "psi_internal.cuh"

namespace psi {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0).
// The staged prefix of x is re-read by every CTA: keep it in L2 (evict_last hint).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
// 256-bit streaming load of 8 entry words (sm_100 .v8): read once per sweep, so no L1
// allocation and L2 evict_first (the staged x segments and gathers keep the cache).
__device__ __forceinline__ void ld_stream8(const unsigned* p, unsigned (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                 "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

// One warp's pass over one chunk of a list (panel, warp, segment): 8 entries per lane,
// gathers from the staged segment, runs of equal slots summed in registers (inclusive run
// sums) and across lanes (a segmented scan), each finished run added once to its slot sum
// (owned by this warp) -- branch-free.  A slot has ONE run per list (the entries of a list
// are grouped by slot), so the run ends of a chunk -- at most nine per lane: seven inside
// the lane, its tail, and lane 0's flush of the run carried in from the previous chunk --
// all touch distinct slot sums: their read-modify-writes are issued as one batch of loads
// followed by one batch of stores, instead of nine dependent load-add-store chains.
__device__ __forceinline__ void process_chunk(const unsigned (&w)[8], const double* seg,
                                              double* rowsum, int lane, double& carry,
                                              unsigned& carry_slot, int sh, unsigned junk) {
  unsigned sl[8];
  double acc[8];
  const unsigned omask = (1u << sh) - 1u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sl[k] = w[k] >> sh;
    PSI_ASSERT(sl[k] <= junk);
    acc[k] = seg[w[k] & omask];
  }
  bool single = true;
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const bool same = sl[k] == sl[k - 1];
    acc[k] = same ? acc[k - 1] + acc[k] : acc[k];
    single = single && same;
  }
  // lane-crossing runs: the open value leaving lane l is
  //   out_l = (single_l && cont_l) ? out_{l-1} + run_l : run_l,   out_{-1} = carry
  // = a segmented inclusive scan of the lane's tail run with resets f_l = !(single_l && cont_l).
  const unsigned prev_last = __shfl_up_sync(kFull, sl[7], 1);
  const bool cont = lane == 0 ? (sl[0] == carry_slot) : (sl[0] == prev_last);
  // segment starts from one ballot (no flag shuffles): lane l's segment starts at the highest
  // reset lane <= l, so a Kogge-Stone step adds lane l-o's partial iff l-o >= that start
  const unsigned fmask = __ballot_sync(kFull, !(single && cont));
  const unsigned below = fmask & (0xffffffffu >> (31 - lane));     // reset lanes <= lane
  const int start = below ? 31 - __clz(below) : -1;
  double val = acc[7];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v2 = __shfl_up_sync(kFull, val, o);
    if (lane - o >= start && lane >= o) val += v2;
  }
  const double out = start >= 0 ? val : val + carry;  // chain reaching back to the carry
  double in = __shfl_up_sync(kFull, out, 1);
  if (lane == 0) in = carry;
  const bool next_cont = (__ballot_sync(kFull, cont) >> ((lane + 1) & 31)) & 1u;
  // run ends: k < 7 inside the lane (the first one, the head, continues a run from earlier
  // lanes when cont), 7 = the lane's tail when the next lane starts another slot, 8 = the
  // carried run that ended at the chunk boundary (lane 0)
  bool pr[9];
  unsigned ix[9];
  bool head = true;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const bool b = sl[k] != sl[k + 1];
    pr[k] = b;
    ix[k] = sl[k];
    acc[k] += (head && cont) ? in : 0.0;
    head = head && !b;
  }
  pr[7] = lane < 31 && !next_cont;
  ix[7] = sl[7];
  acc[7] = out;
  pr[8] = lane == 0 && !cont && carry_slot != junk;
  ix[8] = carry_slot;
  double old[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) old[k] = pr[k] ? rowsum[ix[k]] : 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (pr[k]) rowsum[ix[k]] = old[k] + acc[k];
  if (pr[8]) rowsum[ix[8]] = old[8] + carry;
  carry = __shfl_sync(kFull, out, 31);
  carry_slot = __shfl_sync(kFull, sl[7], 31);
  __syncwarp();
}

__device__ __forceinline__ void load_chunk(const unsigned* base, unsigned c, unsigned e, int lane,
                                           unsigned (&w)[8], unsigned null_entry) {
  const unsigned pos = c + lane * 8;
  if (pos < e) {
    ld_stream8(base + pos, w);                        // lists are padded to 8 words
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = null_entry;
  }
}

// HW consumer warps + 1 producer warp.  HW = kHeavyWarps with the serial plan (the kernel owns
// the SM); HW = kOvlWarps with the overlapped one (k_tiles shares the SM, PSI_OVERLAP).
template <int HW>
__global__ void __launch_bounds__(32 * (HW + 1), 1) k_heavy(SweepArgs A) {
  extern __shared__ __align__(128) unsigned char hsm[];
  const HeavyPlan& H = A.heavy;
  const int nseg = H.nseg;
  const int sh = H.seg_shift;
  const int SEG = 1 << sh;                                            // labels per segment
  const unsigned junk = (unsigned)H.slots;                            // padding slot
  const unsigned null_entry = junk << sh;
  double* stage_buf = reinterpret_cast<double*>(hsm);                 // [kHeavyStages][SEG]
  double* rowsum = stage_buf + kHeavyStages * SEG;                    // [slots + 2]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(rowsum + H.slots + 2);
  unsigned long long* empty = full + kHeavyStages;
  int* ring = reinterpret_cast<int*>(empty + kHeavyStages);           // [8] panel ids
  unsigned* offs = reinterpret_cast<unsigned*>(ring + 8);             // [warps][nseg + 1]

  // a programmatically dependent k_tiles (overlapped sweep) may launch once every CTA is here:
  // it then lands beside this CTA on the same SM (no-op without a dependent)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t = A.st->iter;
  const double* __restrict__ xs = (t & 1) ? A.x1 : A.x0;             // x_{t-1} (x_T: readout)

  if (threadIdx.x == 0) {
    for (int i = 0; i < kHeavyStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, HW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == HW) {
    // ---- producer: claims panels dynamically (deterministic result: a panel's sums do not
    // depend on which CTA computes it) and streams x_{t-1}[s*kSeg, (s+1)*kSeg) for each.
    if (lane == 0) {
      unsigned long long pol;
      asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      unsigned q = 0;
      for (int k = 0;; ++k) {
        const int p = (int)atomicAdd(&A.st->heavy_next, 1u);
        const bool done = p >= H.npanels;
        for (int s = 0; s < (done ? 1 : nseg); ++s, ++q) {
          const int st = q % kHeavyStages;
          const unsigned ph = (q / kHeavyStages) & 1u;
          mbar_wait(empty + st, ph ^ 1u);
          if (s == 0) ring[k & 7] = done ? -1 : p;
          if (done) {
            mbar_arrive(full + st);                   // no bytes: consumers read ring = -1
          } else {
            mbar_expect_tx(full + st, SEG * 8);
            bulk_g2s(stage_buf + (size_t)st * SEG, xs + ((size_t)s << sh), SEG * 8, full + st, pol);
          }
        }
        if (done) break;
      }
    }
    return;
  }

  // ---- consumers
  unsigned* my_offs = offs + (size_t)warp * (nseg + 1);
  unsigned q = 0;
  for (int k = 0;; ++k) {
    mbar_wait(full + q % kHeavyStages, (q / kHeavyStages) & 1u);      // segment 0 of panel k
    const int p = ring[k & 7];
    if (p < 0) break;
    PSI_ASSERT(p < H.npanels);
    const int* ws = H.wslot + (size_t)p * (HW + 1);
    const int sl0 = ws[warp], sl1 = ws[warp + 1];
    for (int i = sl0 + lane; i < sl1; i += 32) rowsum[i] = 0.0;
    // this warp's lists of the panel are contiguous: (p, warp, s = 0 .. nseg-1)
    const long long* lo = H.loff + ((size_t)p * HW + warp) * nseg;
    const long long base = lo[0];
    for (int i = lane; i <= nseg; i += 32) my_offs[i] = (unsigned)(lo[i] - base);
    __syncwarp();
    const unsigned* wst = H.ent + base;
    // chunk iterator (s_n, c_n) one chunk ahead of the one being processed
    int s_n = 0;
    unsigned c_n = 0;
    while (s_n < nseg && c_n >= my_offs[s_n + 1]) c_n = my_offs[++s_n];
    unsigned w_n[8];
    if (s_n < nseg) load_chunk(wst, c_n, my_offs[s_n + 1], lane, w_n, null_entry);
    for (int s = 0; s < nseg; ++s, ++q) {
      const int st = q % kHeavyStages;
      if (s > 0) mbar_wait(full + st, (q / kHeavyStages) & 1u);
      const double* seg = stage_buf + (size_t)st * SEG;
      unsigned carry_slot = junk;             // open run carried across chunks of the list
      double carry = 0.0;
      while (s_n == s) {
        unsigned w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = w_n[i];
        c_n += 256;                                   // advance, then prefetch the next chunk
        while (s_n < nseg && c_n >= my_offs[s_n + 1]) {
          ++s_n;
          if (s_n < nseg) c_n = my_offs[s_n];
        }
        if (s_n < nseg) load_chunk(wst, c_n, my_offs[s_n + 1], lane, w_n, null_entry);
        process_chunk(w, seg, rowsum, lane, carry, carry_slot, sh, junk);
      }
      if (lane == 0 && carry_slot != junk) rowsum[carry_slot] += carry;
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    // ---- panel end: row sums = slot sums in slot order
    asm volatile("bar.sync 1, %0;" :: "r"(HW * 32) : "memory");
    const int r0 = H.prow[p], r1 = H.prow[p + 1];
    for (int r = r0 + (int)threadIdx.x; r < r1; r += HW * 32) {
      const int2 sn = H.rslot[r];
      PSI_ASSERT(r < A.n_heavy && sn.x >= 0 && sn.x + sn.y <= H.slots);
      double S = 0.0;
      for (int j = 0; j < sn.y; ++j) S += rowsum[sn.x + j];
      A.hhot[r] = S;
    }
    asm volatile("bar.sync 1, %0;" :: "r"(HW * 32) : "memory");
  }
}

}  // namespace

void* heavy_kernel_ptr(int warps) {
  return warps == kOvlWarps ? (void*)k_heavy<kOvlWarps> : (void*)k_heavy<kHeavyWarps>;
}

size_t heavy_smem_bytes(int nseg, int seg_shift, int slots, int warps) {
  return ((size_t)kHeavyStages << seg_shift) * 8 + (size_t)(slots + 2) * 8 + 2 * kHeavyStages * 8 +
         8 * 4 + (size_t)warps * (nseg + 1) * 4;
}

}  // namespace psi
