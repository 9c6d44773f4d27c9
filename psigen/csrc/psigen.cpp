// psigen -- seeded synthetic follower graphs and activity vectors.
//
// INPUT GENERATOR ONLY.  This module is shared by the oracle side (tests,
// bench cpu_baseline) and the CUDA side (tests, bench): it produces the same
// arrays for both and contains none of Power-psi's arithmetic (no W, c, d,
// A, B, s or psi).  Recipes follow SURVEY.md §8(d).1 and are restated in
// DESIGN.md ("Input recipe").
//
// Output graph format (the C-ABI's input format):
//   CSR of followers per leader: row_ptr int64[N+1], followers int32[M];
//   row j = F(j) = users who follow j, strictly increasing, no self loops.
//
// Randomness: a counter-based generator (splitmix64 finaliser applied to a
// (seed, stream, counter) mix), so every draw is a pure function of its
// indices and the output does not depend on the number of OpenMP threads.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>
#include <omp.h>

namespace {

using u64 = uint64_t;
using u32 = uint32_t;
using i64 = int64_t;

enum : u64 {
  ST_ER = 1, ST_FIX = 2, ST_CL_PERM_IN = 3, ST_CL_PERM_OUT = 4, ST_CL_DRAW = 5,
  ST_RMAT = 6, ST_SCRAMBLE = 7, ST_ZERO = 8, ST_ACT = 100,
};

inline u64 fmix(u64 z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline u64 rng(u64 seed, u64 stream, u64 ctr) {
  return fmix(fmix(seed * 0xD1B54A32D192ED03ULL ^ fmix(stream + 0x632BE59BD9B4E019ULL)) ^ ctr);
}
// uniform in (0, 1]: never 0, so log() is finite
inline double u01_open0(u64 h) { return ((h >> 11) + 1) * (1.0 / 9007199254740992.0); }
// uniform in [0, 1)
inline double u01(u64 h) { return (h >> 11) * (1.0 / 9007199254740992.0); }
// uniform integer in [0, n) for n < 2^32
inline u64 below(u64 h, u64 n) { return ((h >> 32) * n) >> 32; }

// ---------------------------------------------------------------- radix sort
// LSD radix sort of u64 keys on their low `bits` bits; deterministic.
void radix_sort(std::vector<u64>& keys, int bits) {
  const int R = 11, B = 1 << R;
  const size_t n = keys.size();
  if (n < 2) return;
  std::vector<u64> tmp(n);
  int nt = omp_get_max_threads();
  std::vector<size_t> hist((size_t)nt * B);
  u64* src = keys.data();
  u64* dst = tmp.data();
  int passes = 0;
  for (int shift = 0; shift < bits; shift += R) {
    std::fill(hist.begin(), hist.end(), 0);
#pragma omp parallel num_threads(nt)
    {
      int t = omp_get_thread_num();
      size_t lo = n * t / nt, hi = n * (t + 1) / nt;
      size_t* h = &hist[(size_t)t * B];
      for (size_t i = lo; i < hi; ++i) h[(src[i] >> shift) & (B - 1)]++;
#pragma omp barrier
#pragma omp single
      {
        size_t sum = 0;
        for (int b = 0; b < B; ++b)
          for (int tt = 0; tt < nt; ++tt) {
            size_t c = hist[(size_t)tt * B + b];
            hist[(size_t)tt * B + b] = sum;
            sum += c;
          }
      }
      for (size_t i = lo; i < hi; ++i) {
        u64 k = src[i];
        dst[h[(k >> shift) & (B - 1)]++] = k;
      }
    }
    std::swap(src, dst);
    ++passes;
  }
  if (passes & 1) std::memcpy(keys.data(), tmp.data(), n * sizeof(u64));
}

int bits_for(u64 n) { int b = 0; while ((1ULL << b) < n) ++b; return std::max(b, 1); }

// sorted keys -> unique (in place)
void unique_sorted(std::vector<u64>& k) {
  k.erase(std::unique(k.begin(), k.end()), k.end());
}

// key = leader << 32 | follower
inline u64 mk(u64 leader, u64 follower) { return (leader << 32) | follower; }

struct Graph {
  i64 n = 0;
  std::vector<i64> row_ptr;
  std::vector<int32_t> followers;
};

// Sorted unique keys -> CSR (rows = leaders, entries = followers ascending).
void keys_to_csr(const std::vector<u64>& k, i64 n, Graph& g) {
  g.n = n;
  const size_t m = k.size();
  g.row_ptr.assign(n + 1, 0);
  g.followers.resize(m);
  i64* rp = g.row_ptr.data();
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; ++i) {
    g.followers[i] = (int32_t)(k[i] & 0xffffffffULL);
    i64 cur = (i64)(k[i] >> 32);
    i64 prev = i == 0 ? -1 : (i64)(k[i - 1] >> 32);
    for (i64 r = prev + 1; r <= cur; ++r) rp[r] = (i64)i;   // first edge of row r
  }
  i64 last = m ? (i64)(k[m - 1] >> 32) : -1;
#pragma omp parallel for schedule(static)
  for (i64 r = last + 1; r <= n; ++r) rp[r] = (i64)m;
}

// Users with no leader get one uniform random leader != self (SURVEY §8(d).1
// readings for configs 1, 2, 4, 5).  Input/Output: sorted unique keys.
void fix_leaderless(std::vector<u64>& k, i64 n, u64 seed) {
  std::vector<uint8_t> has(n, 0);
  const size_t m = k.size();
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; ++i) has[k[i] & 0xffffffffULL] = 1;   // benign same-value race
  std::vector<u64> add;
  for (i64 u = 0; u < n; ++u) {
    if (has[u] || n < 2) continue;
    u64 v = below(rng(seed, ST_FIX, (u64)u), (u64)(n - 1));
    if ((i64)v >= u) ++v;                                       // skip self
    add.push_back(mk(v, (u64)u));
  }
  if (add.empty()) return;
  radix_sort(add, 32 + bits_for(n));
  std::vector<u64> out(m + add.size());
  std::merge(k.begin(), k.end(), add.begin(), add.end(), out.begin());
  k.swap(out);
}

// ------------------------------------------------------------------- ER
// Directed G(N, p): every ordered pair (u follows v), v != u, independently
// with probability p = mean / (N - 1); geometric skipping per follower u.
void gen_er(i64 n, double mean, u64 seed, bool fix, Graph& g) {
  double p = n > 1 ? std::min(1.0, mean / (double)(n - 1)) : 0.0;
  std::vector<i64> cnt(n + 1, 0);
  const double lq = p < 1.0 ? std::log1p(-p) : -INFINITY;
  auto walk = [&](i64 u, auto&& emit) {
    if (p <= 0.0) return;
    i64 pos = -1;
    u64 ctr = 0;
    const i64 cand = n - 1;
    while (true) {
      i64 skip = 0;
      if (p < 1.0) {
        double U = u01_open0(rng(seed, ST_ER, ((u64)u << 32) | ctr++));
        double s = std::floor(std::log(U) / lq);
        if (s > (double)cand) break;
        skip = (i64)s;
      }
      pos += skip + 1;
      if (pos >= cand) break;
      i64 v = pos < u ? pos : pos + 1;
      emit(v);
    }
  };
#pragma omp parallel for schedule(dynamic, 1024)
  for (i64 u = 0; u < n; ++u) {
    i64 c = 0;
    walk(u, [&](i64) { ++c; });
    cnt[u + 1] = c;
  }
  for (i64 u = 0; u < n; ++u) cnt[u + 1] += cnt[u];
  std::vector<u64> keys((size_t)cnt[n]);
#pragma omp parallel for schedule(dynamic, 1024)
  for (i64 u = 0; u < n; ++u) {
    i64 o = cnt[u];
    walk(u, [&](i64 v) { keys[o++] = mk((u64)v, (u64)u); });
  }
  radix_sort(keys, 32 + bits_for(n));
  unique_sorted(keys);
  if (fix) fix_leaderless(keys, n, seed);
  keys_to_csr(keys, n, g);
}

// ------------------------------------------------------------------- helpers
// Random permutation of [0, n): rank of u when sorted by a per-user hash.
std::vector<u32> random_perm(i64 n, u64 seed, u64 stream) {
  int b = bits_for(n);
  u64 lowmask = (1ULL << b) - 1;
  std::vector<u64> k(n);
#pragma omp parallel for schedule(static)
  for (i64 u = 0; u < n; ++u) k[u] = (rng(seed, stream, (u64)u) & ~lowmask) | (u64)u;
  radix_sort(k, 64);
  std::vector<u32> rank(n);
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) rank[k[i] & lowmask] = (u32)i;
  return rank;
}

// Deterministic fixed-chunk sum (independent of thread count).
template <class F>
double det_sum(i64 n, F f) {
  const int C = 256;
  std::vector<double> part(C, 0.0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    i64 lo = n * c / C, hi = n * (c + 1) / C;
    double s = 0.0;
    for (i64 i = lo; i < hi; ++i) s += f(i);
    part[c] = s;
  }
  double s = 0.0;
  for (double x : part) s += x;
  return s;
}

// ------------------------------------------------------------- Chung-Lu
// Weights w_r = C (r + r0)^(-1/(gamma-1)), r = 0..N-1, with C, r0 such that
// max w = w_0 = max_w and sum w = M.  Independent random permutations assign
// in- and out-weights; M i.i.d. draws (follower ~ w_out, leader ~ w_in) via
// alias tables; self loops and duplicates dropped; draws are topped up until
// exactly M unique edges exist.  Leaderless users are kept.
struct Alias {
  std::vector<double> prob;
  std::vector<u32> alias;
};
Alias build_alias(const std::vector<double>& w) {
  const i64 n = (i64)w.size();
  double tot = det_sum(n, [&](i64 i) { return w[i]; });
  Alias a;
  a.prob.resize(n);
  a.alias.resize(n);
  std::vector<double> sc(n);
  std::vector<u32> small, large;
  for (i64 i = 0; i < n; ++i) {
    sc[i] = w[i] * (double)n / tot;
    (sc[i] < 1.0 ? small : large).push_back((u32)i);
  }
  while (!small.empty() && !large.empty()) {
    u32 s = small.back(); small.pop_back();
    u32 l = large.back();
    a.prob[s] = sc[s];
    a.alias[s] = l;
    sc[l] = (sc[l] + sc[s]) - 1.0;
    if (sc[l] < 1.0) { large.pop_back(); small.push_back(l); }
  }
  for (u32 l : large) { a.prob[l] = 1.0; a.alias[l] = l; }
  for (u32 s : small) { a.prob[s] = 1.0; a.alias[s] = s; }
  return a;
}
inline u32 alias_draw(const Alias& a, u64 h, u64 n) {
  u32 col = (u32)below(h, n);
  double coin = (double)(h & 0xffffffffULL) * (1.0 / 4294967296.0);
  return coin < a.prob[col] ? col : a.alias[col];
}

void gen_chung_lu(i64 n, i64 m, double gamma, double max_w, u64 seed, Graph& g) {
  const double al = 1.0 / (gamma - 1.0);
  auto total = [&](double r0) {
    return det_sum(n, [&](i64 r) { return max_w * std::pow(r0 / ((double)r + r0), al); });
  };
  double lo = 1e-9, hi = 1e15;
  for (int it = 0; it < 200; ++it) {
    double mid = std::sqrt(lo * hi);
    if (total(mid) < (double)m) lo = mid; else hi = mid;
    if (hi / lo < 1 + 1e-12) break;
  }
  const double r0 = std::sqrt(lo * hi);
  const double C = max_w * std::pow(r0, al);
  std::vector<double> wr(n);
#pragma omp parallel for schedule(static)
  for (i64 r = 0; r < n; ++r) wr[r] = C * std::pow((double)r + r0, -al);
  std::vector<u32> pin = random_perm(n, seed, ST_CL_PERM_IN);
  std::vector<u32> pout = random_perm(n, seed, ST_CL_PERM_OUT);
  std::vector<double> win(n), wout(n);
#pragma omp parallel for schedule(static)
  for (i64 u = 0; u < n; ++u) { win[u] = wr[pin[u]]; wout[u] = wr[pout[u]]; }
  Alias ain = build_alias(win), aout = build_alias(wout);
  const int kb = 32 + bits_for(n);
  std::vector<u64> uniq;
  u64 drawn = 0;
  while ((i64)uniq.size() < m) {
    const u64 need = (u64)(m - (i64)uniq.size());
    std::vector<u64> add(need);
    std::vector<uint8_t> ok(need);
#pragma omp parallel for schedule(static)
    for (u64 e = 0; e < need; ++e) {
      u64 d = drawn + e;
      u32 src = alias_draw(aout, rng(seed, ST_CL_DRAW, 2 * d), (u64)n);      // follower
      u32 dst = alias_draw(ain, rng(seed, ST_CL_DRAW, 2 * d + 1), (u64)n);   // leader
      add[e] = mk(dst, src);
      ok[e] = src != dst;
    }
    drawn += need;
    size_t w = 0;
    for (u64 e = 0; e < need; ++e) if (ok[e]) add[w++] = add[e];
    add.resize(w);
    radix_sort(add, kb);
    unique_sorted(add);
    std::vector<u64> merged(uniq.size() + add.size());
    std::merge(uniq.begin(), uniq.end(), add.begin(), add.end(), merged.begin());
    unique_sorted(merged);
    uniq.swap(merged);
  }
  keys_to_csr(uniq, n, g);
}

// ------------------------------------------------------------------ R-MAT
// ef * 2^scale draws; per level the (follower bit, leader bit) quadrant is
// (0,0) w.p. a, (0,1) b, (1,0) c, (1,1) d = 1-a-b-c; MSB first.  Optional
// seeded vertex relabel (Graph500-style scramble).  Self loops and duplicates
// removed; users with no leader get one uniform random leader.
void gen_rmat(int scale, i64 ef, double a, double b, double c, u64 seed, bool scramble,
              bool fix, Graph& g) {
  const i64 n = (i64)1 << scale;
  const u64 draws = (u64)ef * (u64)n;
  const u64 ta = (u64)(a * 4294967296.0);
  const u64 tb = (u64)((a + b) * 4294967296.0);
  const u64 tc = (u64)((a + b + c) * 4294967296.0);
  std::vector<u32> perm;
  if (scramble) perm = random_perm(n, seed, ST_SCRAMBLE);
  std::vector<u64> keys(draws);
  std::vector<uint8_t> ok(draws);
#pragma omp parallel for schedule(static)
  for (u64 e = 0; e < draws; ++e) {
    u64 src = 0, dst = 0, h = 0;
    for (int l = 0; l < scale; ++l) {
      u64 u;
      if ((l & 1) == 0) { h = rng(seed, ST_RMAT, e * 16 + (u64)(l >> 1)); u = h >> 32; }
      else u = h & 0xffffffffULL;
      u64 sb = (u >= tb) ? 1 : 0;             // c or d quadrant: follower bit 1
      u64 db = (u >= ta && u < tb) || u >= tc ? 1 : 0;   // b or d: leader bit 1
      src |= sb << (scale - 1 - l);
      dst |= db << (scale - 1 - l);
    }
    if (scramble) { src = perm[src]; dst = perm[dst]; }
    keys[e] = mk(dst, src);
    ok[e] = src != dst;
  }
  size_t w = 0;
  for (u64 e = 0; e < draws; ++e) if (ok[e]) keys[w++] = keys[e];
  keys.resize(w);
  ok.clear(); ok.shrink_to_fit();
  radix_sort(keys, 32 + scale);
  unique_sorted(keys);
  if (fix) fix_leaderless(keys, n, seed);
  keys_to_csr(keys, n, g);
}

}  // namespace

// =================================================================== C ABI
extern "C" {

struct psigen_graph { Graph g; };

int psigen_er(int64_t n, double mean, uint64_t seed, int fix, psigen_graph** out) {
  if (n < 1 || !out) return -1;
  auto* p = new psigen_graph;
  gen_er(n, mean, seed, fix != 0, p->g);
  *out = p;
  return 0;
}

int psigen_chung_lu(int64_t n, int64_t m, double gamma, double max_w, uint64_t seed,
                    psigen_graph** out) {
  if (n < 2 || m < 0 || m > n * (n - 1) || gamma <= 1.0 || !out) return -1;
  auto* p = new psigen_graph;
  gen_chung_lu(n, m, gamma, max_w, seed, p->g);
  *out = p;
  return 0;
}

int psigen_rmat(int scale, int64_t ef, double a, double b, double c, uint64_t seed,
                int scramble, int fix, psigen_graph** out) {
  if (scale < 1 || scale > 31 || ef < 0 || !out) return -1;
  auto* p = new psigen_graph;
  gen_rmat(scale, ef, a, b, c, seed, scramble != 0, fix != 0, p->g);
  *out = p;
  return 0;
}

int64_t psigen_n(const psigen_graph* p) { return p->g.n; }
int64_t psigen_m(const psigen_graph* p) { return (int64_t)p->g.followers.size(); }

void psigen_copy(const psigen_graph* p, int64_t* row_ptr, int32_t* followers) {
  std::memcpy(row_ptr, p->g.row_ptr.data(), (p->g.n + 1) * sizeof(int64_t));
  const size_t m = p->g.followers.size();
  const int32_t* src = p->g.followers.data();
#pragma omp parallel for schedule(static)
  for (int64_t blk = 0; blk < 1024; ++blk) {
    size_t lo = m * blk / 1024, hi = m * (blk + 1) / 1024;
    std::memcpy(followers + lo, src + lo, (hi - lo) * sizeof(int32_t));
  }
}

void psigen_free(psigen_graph* p) { delete p; }

// out[u] = lo + (hi - lo) * U_u,  U_u ~ U[0, 1)
void psigen_uniform(int64_t n, double lo, double hi, uint64_t seed, uint64_t stream, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) out[u] = lo + (hi - lo) * u01(rng(seed, ST_ACT + stream, (u64)u));
}

// out[u] = exp(m + s Z_u), Z_u standard normal (Box-Muller, cosine branch)
void psigen_lognormal(int64_t n, double m, double s, uint64_t seed, uint64_t stream, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) {
    double u1 = u01_open0(rng(seed, ST_ACT + stream, 2 * (u64)u));
    double u2 = u01(rng(seed, ST_ACT + stream, 2 * (u64)u + 1));
    double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    out[u] = std::exp(m + s * z);
  }
}

// Exactly k seeded-random users (smallest per-user hash) -> out[u] = 0.
void psigen_zero_subset(int64_t n, int64_t k, uint64_t seed, double* out) {
  if (k <= 0) return;
  std::vector<u32> rank = random_perm(n, seed, ST_ZERO);
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) if ((int64_t)rank[u] < k) out[u] = 0.0;
}

int psigen_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
