// libLBX host balancer: distribution-mapping policies and load-balance
// efficiency, bit-exact with the reference's numpy arithmetic.
//
// Why C++ and not numpy: the reference knapsack costs 5-56 ms per call at 900
// boxes ("Where time goes"), which would dwarf a microsecond
// device step.  Bit-exactness rules followed here (compiled with
// -ffp-contract=off so no FMA is formed):
//   * np.bincount(weights=) accumulates sequentially in input order;
//   * ndarray.sum()/.mean() use numpy's pairwise summation (8 accumulators,
//     blocks of 128, recursive split at n/2 rounded down to a multiple of 8);
//   * np.lexsort((arange, -cost)) == sort by cost descending, id ascending;
//   * np.argmin returns the first minimum;
//   * the swap search evaluates (load_max - c_a) + c_b and
//     (load_other - c_b) + c_a exactly as balancer.py:163-164 does.

#include <algorithm>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <climits>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

#include <cstdlib>

#include "lbx_internal.h"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace lbx {

double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

namespace {

// refine_by_swaps: partner-pair evaluations per iteration above which the
// search is split over OpenMP threads (below, waking the threads costs more
// than the search: a C2 pass -- 112 x 788 pairs at 8 ranks -- is ~10 us on
// one core, a thread wake-up tens of microseconds)
constexpr int64_t kParallelPairs = 1 << 21;

#ifdef _OPENMP
// threads for the swap search: LBX_LB_THREADS, else up to 4 (one rank per
// GPU shares the host's cores with the other ranks)
int lb_threads() {
  static const int n = [] {
    const char* e = std::getenv("LBX_LB_THREADS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : std::min(4, omp_get_max_threads());
  }();
  return n;
}
#endif

int check_owner(const int64_t* owner, int64_t n, int32_t R) {
  for (int64_t i = 0; i < n; ++i)
    if (owner[i] < 0 || owner[i] >= R)
      return set_error(LBX_EINVAL, "owner entries must lie in [0, %d), got %lld at box %lld", R,
                       (long long)owner[i], (long long)i);
  return LBX_OK;
}

void loads_of(const double* cost, const int64_t* owner, int64_t n, int32_t R, double* loads) {
  std::fill(loads, loads + R, 0.0);
  for (int64_t i = 0; i < n; ++i) loads[owner[i]] += cost[i];
}

// balancer.py:137-179.  Only swaps that involve the unique most-loaded rank
// can lower the maximum; best strict improvement wins, ties to the lowest
// own box id, then the lowest partner box id.
// Best improving partner of box a (value ca) among `others`: the lowest j with
// the smallest pair max max(here0 + cb_j, (L_j - cb_j) + ca) < top -- the
// reference's per-box search (balancer.py:157-170, np.argmin = first index),
// with d_j = L_j - cb_j precomputed exactly as the reference evaluates it.
static inline void partner_tail(const double* cb, const double* d, int64_t j0, int64_t no,
                                double here0, double ca, double top, int64_t* jbest,
                                double* pm_best) {
  for (int64_t j = j0; j < no; ++j) {
    const double here = here0 + cb[j];
    const double there = d[j] + ca;
    const double pm = here >= there ? here : there;
    if (pm < top && (*jbest < 0 || pm < *pm_best)) {
      *jbest = j;
      *pm_best = pm;
    }
  }
}

// Merge per-lane first minima: smallest value, then smallest index -- the
// scalar scan's first-index rule.  max(here, there) of equal values may
// differ only in the sign of a zero, which no comparison sees.
static inline void merge_lanes(const double* m, const long long* ix, int lanes, int64_t* jbest,
                               double* pm_best) {
  for (int l = 0; l < lanes; ++l) {
    if (ix[l] < 0) continue;
    if (*jbest < 0 || m[l] < *pm_best || (m[l] == *pm_best && ix[l] < *jbest)) {
      *jbest = ix[l];
      *pm_best = m[l];
    }
  }
}

#if defined(__x86_64__)
__attribute__((target("avx512f"))) static int64_t best_partner_avx512(
    const double* cb, const double* d, int64_t no, double here0, double ca, double top,
    double* pm_out) {
  int64_t jbest = -1;
  double pm_best = 0.0;
  int64_t j0 = 0;
  const __m512d vh0 = _mm512_set1_pd(here0), vca = _mm512_set1_pd(ca), vtop = _mm512_set1_pd(top);
  const __m512d vinf = _mm512_set1_pd(std::numeric_limits<double>::infinity());
  // four independent (min, index) accumulators over interleaved 8-wide
  // groups: the masked compare / move chain is four times shorter
  __m512d vmin[4] = {vinf, vinf, vinf, vinf};
  __m512i vidx[4];
  __m512i vj[4];
  for (int u = 0; u < 4; ++u) {
    vidx[u] = _mm512_set1_epi64(-1);
    vj[u] = _mm512_add_epi64(_mm512_setr_epi64(0, 1, 2, 3, 4, 5, 6, 7), _mm512_set1_epi64(8 * u));
  }
  const __m512i v32 = _mm512_set1_epi64(32);
  for (; j0 + 32 <= no; j0 += 32) {
#pragma GCC unroll 4
    for (int u = 0; u < 4; ++u) {
      const __m512d here = _mm512_add_pd(vh0, _mm512_loadu_pd(cb + j0 + 8 * u));
      const __m512d there = _mm512_add_pd(_mm512_loadu_pd(d + j0 + 8 * u), vca);
      const __m512d pm = _mm512_max_pd(here, there);
      const __mmask8 ok = _mm512_cmp_pd_mask(pm, vtop, _CMP_LT_OQ);
      const __mmask8 better = _mm512_mask_cmp_pd_mask(ok, pm, vmin[u], _CMP_LT_OQ);
      vmin[u] = _mm512_mask_mov_pd(vmin[u], better, pm);
      vidx[u] = _mm512_mask_mov_epi64(vidx[u], better, vj[u]);
      vj[u] = _mm512_add_epi64(vj[u], v32);
    }
  }
  // first minimum over the 32 lanes: smallest value, then smallest index
  const __m512d m01 = _mm512_min_pd(vmin[0], vmin[1]), m23 = _mm512_min_pd(vmin[2], vmin[3]);
  const double mv = _mm512_reduce_min_pd(_mm512_min_pd(m01, m23));
  if (mv < std::numeric_limits<double>::infinity()) {
    const __m512d vm = _mm512_set1_pd(mv);
    const __m512i big = _mm512_set1_epi64(LLONG_MAX);
    __m512i best = big;
    for (int u = 0; u < 4; ++u) {
      const __mmask8 eq = _mm512_cmp_pd_mask(vmin[u], vm, _CMP_EQ_OQ);
      best = _mm512_min_epi64(best, _mm512_mask_mov_epi64(big, eq, vidx[u]));
    }
    jbest = _mm512_reduce_min_epi64(best);
    pm_best = mv;
  }
  partner_tail(cb, d, j0, no, here0, ca, top, &jbest, &pm_best);
  *pm_out = pm_best;
  return jbest;
}

__attribute__((target("avx2"))) static int64_t best_partner_avx2(
    const double* cb, const double* d, int64_t no, double here0, double ca, double top,
    double* pm_out) {
  int64_t jbest = -1;
  double pm_best = 0.0;
  int64_t j0 = 0;
  const __m256d vh0 = _mm256_set1_pd(here0), vca = _mm256_set1_pd(ca), vtop = _mm256_set1_pd(top);
  const __m256d vinf = _mm256_set1_pd(std::numeric_limits<double>::infinity());
  __m256d vmin = vinf;
  __m256i vidx = _mm256_set1_epi64x(-1);
  __m256i vj = _mm256_setr_epi64x(0, 1, 2, 3);
  const __m256i v4 = _mm256_set1_epi64x(4);
  for (; j0 + 4 <= no; j0 += 4) {
    const __m256d here = _mm256_add_pd(vh0, _mm256_loadu_pd(cb + j0));
    const __m256d there = _mm256_add_pd(_mm256_loadu_pd(d + j0), vca);
    __m256d pm = _mm256_max_pd(here, there);
    pm = _mm256_blendv_pd(vinf, pm, _mm256_cmp_pd(pm, vtop, _CMP_LT_OQ));
    const __m256d better = _mm256_cmp_pd(pm, vmin, _CMP_LT_OQ);
    vmin = _mm256_blendv_pd(vmin, pm, better);
    vidx = _mm256_castpd_si256(_mm256_blendv_pd(_mm256_castsi256_pd(vidx),
                                                _mm256_castsi256_pd(vj), better));
    vj = _mm256_add_epi64(vj, v4);
  }
  alignas(32) double m[4];
  alignas(32) long long ix[4];
  _mm256_store_pd(m, vmin);
  _mm256_store_si256(reinterpret_cast<__m256i*>(ix), vidx);
  merge_lanes(m, ix, 4, &jbest, &pm_best);
  partner_tail(cb, d, j0, no, here0, ca, top, &jbest, &pm_best);
  *pm_out = pm_best;
  return jbest;
}
#endif

// Best improving partner of box a (value ca) among `others`: the lowest j with
// the smallest pair max max(here0 + cb_j, (L_j - cb_j) + ca) < top -- the
// reference's per-box search (balancer.py:157-170, np.argmin = first index),
// with d_j = L_j - cb_j precomputed exactly as the reference evaluates it.
// Vectorised (AVX-512 or AVX2, chosen at run time) with per-lane first
// minima merged by value then index: the same j as the scalar scan.
static int64_t best_partner(const double* cb, const double* d, int64_t no, double here0,
                            double ca, double top, double* pm_out) {
#if defined(__x86_64__)
  static const int isa = __builtin_cpu_supports("avx512f") ? 2 : __builtin_cpu_supports("avx2") ? 1 : 0;
  if (isa == 2 && no >= 64) return best_partner_avx512(cb, d, no, here0, ca, top, pm_out);
  if (isa == 1 && no >= 8) return best_partner_avx2(cb, d, no, here0, ca, top, pm_out);
#endif
  int64_t jbest = -1;
  double pm_best = 0.0;
  partner_tail(cb, d, 0, no, here0, ca, top, &jbest, &pm_best);
  *pm_out = pm_best;
  return jbest;
}

void refine_by_swaps(int64_t* owner, double* loads, const double* v, int64_t n, int32_t R) {
  if (R < 2 || n < 2) return;
  std::vector<int64_t> mine, others;
  std::vector<double> cb, d;
  mine.reserve(n);
  others.reserve(n);
  cb.reserve(n);
  d.reserve(n);
  while (true) {
    double top = loads[0];
    for (int32_t r = 1; r < R; ++r) top = std::max(top, loads[r]);
    int32_t rmax = -1, at_top = 0;
    for (int32_t r = 0; r < R; ++r)
      if (loads[r] == top) {
        if (at_top == 0) rmax = r;
        ++at_top;
      }
    if (at_top != 1) return;
    mine.clear();
    others.clear();
    cb.clear();
    d.clear();
    for (int64_t b = 0; b < n; ++b) {
      if (owner[b] == rmax) {
        mine.push_back(b);
      } else {
        others.push_back(b);
        cb.push_back(v[b]);
        d.push_back(loads[owner[b]] - v[b]);
      }
    }
    if (mine.empty() || others.empty()) return;
    const int64_t nm = (int64_t)mine.size(), no = (int64_t)others.size();
    // pad the partner arrays to whole 32-wide vector groups with entries that
    // never qualify (pair max = inf), so the search has no scalar tail
    for (int64_t k = no; k % 32; ++k) {
      cb.push_back(std::numeric_limits<double>::infinity());
      d.push_back(std::numeric_limits<double>::infinity());
    }
    const int64_t no_pad = (int64_t)cb.size();
    struct Best {
      bool have = false;
      double pm = 0.0;
      int64_t ia = -1, j = -1;
    } best;
    // Partner searches of the max-rank's boxes are independent: large
    // instances split them over OpenMP threads in contiguous chunks, and the
    // per-chunk bests are merged in chunk order with the sequential loop's
    // rule (strictly smaller pair max wins, so ties keep the lowest box) --
    // the same swap as one thread.
    const bool par = nm * no >= kParallelPairs;
    int nt = 1;
#ifdef _OPENMP
    if (par) nt = std::min<int>(lb_threads(), (int)nm);
#endif
    std::vector<Best> part(nt);
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static, 1) if (par)
#endif
    for (int t = 0; t < nt; ++t) {
      const int64_t lo = nm * t / nt, hi = nm * (t + 1) / nt;
      Best b;
      for (int64_t ia = lo; ia < hi; ++ia) {
        const double ca = v[mine[ia]];
        double pm;
        const int64_t j = best_partner(cb.data(), d.data(), no_pad, top - ca, ca, top, &pm);
        if (j < 0) continue;
        if (!b.have || pm < b.pm) {
          b.have = true;
          b.pm = pm;
          b.ia = ia;
          b.j = j;
        }
      }
      part[t] = b;
    }
    for (int t = 0; t < nt; ++t) {
      const Best& b = part[t];
      if (b.have && (!best.have || b.pm < best.pm)) best = b;
    }
    if (!best.have) return;
    const int64_t best_a = mine[best.ia], best_b = others[best.j];
    const int64_t rb = owner[best_b];
    loads[rmax] += v[best_b] - v[best_a];
    loads[rb] += v[best_a] - v[best_b];
    owner[best_a] = rb;
    owner[best_b] = rmax;
  }
}

uint64_t spread2(uint64_t v) {
  uint64_t out = 0;
  for (int s = 0; v; ++s, v >>= 1) out |= (v & 1ull) << (2 * s);
  return out;
}

uint64_t spread3(uint64_t v) {
  uint64_t out = 0;
  for (int s = 0; v; ++s, v >>= 1) out |= (v & 1ull) << (3 * s);
  return out;
}

void stable_argsort(const std::vector<uint64_t>& codes, int64_t* out) {
  std::vector<int64_t> idx(codes.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int64_t a, int64_t b) { return codes[a] < codes[b]; });
  std::copy(idx.begin(), idx.end(), out);
}

// ---- numpy SeedSequence + PCG64 (XSL-RR 128/64) --------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

uint32_t hashmix(uint32_t value, uint32_t& h) {
  value ^= h;
  h *= kMultA;
  value *= h;
  value ^= value >> 16;
  return value;
}

uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

void int_words(uint64_t v, std::vector<uint32_t>& out) {
  if (v == 0) {
    out.push_back(0u);
    return;
  }
  while (v) {
    out.push_back((uint32_t)v);
    v >>= 32;
  }
}

struct Pcg64 {
  unsigned __int128 state, inc;
  static unsigned __int128 mult() {
    return ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
  }
  void step() { state = state * mult() + inc; }
  uint64_t next64() {
    step();
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

// np.random.default_rng(entropy words) -> PCG64.
Pcg64 make_pcg64(const std::vector<uint32_t>& entropy) {
  uint32_t pool[4];
  uint32_t h = kInitA;
  for (size_t i = 0; i < 4; ++i) pool[i] = hashmix(i < entropy.size() ? entropy[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
  for (size_t s = 4; s < entropy.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s], h));
  uint32_t words[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    words[i] = v;
  }
  uint64_t val[4];
  for (int i = 0; i < 4; ++i) val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
  const unsigned __int128 initstate = ((unsigned __int128)val[0] << 64) | val[1];
  const unsigned __int128 initseq = ((unsigned __int128)val[2] << 64) | val[3];
  Pcg64 g;
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  g.step();
  g.state += initstate;
  g.step();
  return g;
}

}  // namespace

// cost.py:98-113 (work * (1 + U[-a, a]) per box, stream keyed by step).
int measured_cost(const double* work, int64_t n, double amplitude, uint64_t seed, uint64_t step,
                  double* out) {
  if (amplitude == 0.0) {
    std::memcpy(out, work, (size_t)n * sizeof(double));
    return LBX_OK;
  }
  std::vector<uint32_t> ent;
  int_words(seed, ent);
  int_words(0x6D656173ull, ent);
  int_words(step, ent);
  Pcg64 g = make_pcg64(ent);
  const double lo = -amplitude;
  const double scale = amplitude - lo;
  for (int64_t i = 0; i < n; ++i) {
    const double eps = lo + scale * g.next_double();
    out[i] = work[i] * (1.0 + eps);
  }
  return LBX_OK;
}

int efficiency(const double* cost, const int64_t* owner, int64_t n, int32_t R, double* eff,
               int32_t* degenerate, std::vector<double>& scratch) {
  scratch.resize(R);
  loads_of(cost, owner, n, R, scratch.data());
  double top = scratch[0];
  for (int32_t r = 1; r < R; ++r) top = std::max(top, scratch[r]);
  if (top == 0.0) {
    *eff = 1.0;
    if (degenerate) *degenerate = 1;
    return LBX_OK;
  }
  const double mean = pairwise_sum(scratch.data(), R) / (double)R;
  *eff = mean / top;
  if (degenerate) *degenerate = 0;
  return LBX_OK;
}

// Box order of the greedy pass: descending cost, ties to the lower box id
// (np.lexsort((arange(n), -values))).  LSD radix sort of an order-reversing
// integer image of the cost (stable, so equal costs keep ascending ids);
// -0.0 and 0.0 are one key, as the comparison sees them.  NaN-free input.
static void lpt_order(const double* v, int64_t n, std::vector<int64_t>& order) {
  std::vector<uint64_t> key(n), key2(n);
  std::vector<int64_t> tmp(n);
  order.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t u;
    const double x = v[i] == 0.0 ? 0.0 : v[i];
    std::memcpy(&u, &x, 8);
    u = (u >> 63) ? ~u : (u | (1ull << 63));   // ascending image of x
    key[i] = ~u;                                // descending
    order[i] = i;
  }
  int64_t* src = order.data();
  int64_t* dst = tmp.data();
  uint64_t* ks = key.data();
  uint64_t* kd = key2.data();
  uint64_t all_or = 0, all_and = ~0ull;
  for (int64_t i = 0; i < n; ++i) {
    all_or |= ks[i];
    all_and &= ks[i];
  }
  const uint64_t varies = all_or ^ all_and;   // bits that differ between keys
  for (int shift = 0; shift < 64; shift += 8) {
    if (((varies >> shift) & 255u) == 0) continue;   // one digit for all: order unchanged
    int64_t cnt[257] = {0};
    for (int64_t i = 0; i < n; ++i) ++cnt[((ks[i] >> shift) & 255) + 1];
    for (int k = 0; k < 256; ++k) cnt[k + 1] += cnt[k];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t at = cnt[(ks[i] >> shift) & 255]++;
      dst[at] = src[i];
      kd[at] = ks[i];
    }
    std::swap(src, dst);
    std::swap(ks, kd);
  }
  if (src != order.data()) std::memcpy(order.data(), src, 8 * (size_t)n);
}

int knapsack(const double* v, int64_t n, int32_t R, double cap_factor, int64_t* owner) {
  if (R < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1, got %d", R);
  const int64_t cap = n ? (int64_t)std::ceil(cap_factor * (double)n / (double)R) : 0;
  if (cap * R < n)
    return set_error(LBX_EINVAL,
                     "box cap %lld per rank cannot place %lld boxes on %d ranks "
                     "(cap_factor %g too tight)",
                     (long long)cap, (long long)n, R, cap_factor);
  std::vector<int64_t> order;
  lpt_order(v, n, order);
  std::vector<double> loads(R, 0.0);
  std::vector<int64_t> count(R, 0);
  // least-loaded rank with room, ties to the lower rank (np.argmin over the
  // loads masked to inf at the cap): a binary min-heap of (load, rank);
  // a rank that reaches the cap leaves the heap
  std::vector<int32_t> heap(R);
  std::iota(heap.begin(), heap.end(), 0);   // all loads 0: rank order is a heap
  int32_t hn = cap > 0 ? R : 0;
  auto less = [&](int32_t a, int32_t b) {
    return loads[a] < loads[b] || (!(loads[b] < loads[a]) && a < b);
  };
  auto sift_down = [&](int32_t i) {
    const int32_t x = heap[i];
    while (true) {
      int32_t c = 2 * i + 1;
      if (c >= hn) break;
      if (c + 1 < hn && less(heap[c + 1], heap[c])) ++c;
      if (!less(heap[c], x)) break;
      heap[i] = heap[c];
      i = c;
    }
    heap[i] = x;
  };
  for (int64_t b : order) {
    const int32_t r = heap[0];
    owner[b] = r;
    loads[r] += v[b];
    count[r] += 1;
    if (count[r] >= cap) heap[0] = heap[--hn];   // full: drop it
    if (hn > 0) sift_down(0);
  }
  refine_by_swaps(owner, loads.data(), v, n, R);
  return LBX_OK;
}

int sfc(const double* cost, const int64_t* curve, int64_t n, int32_t R, int64_t* owner) {
  if (R < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1, got %d", R);
  if (n == 0) return set_error(LBX_EINVAL, "cannot partition an empty cost vector");
  std::vector<char> seen(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (curve[i] < 0 || curve[i] >= n || seen[curve[i]])
      return set_error(LBX_EINVAL, "curve must be a permutation of box indices");
    seen[curve[i]] = 1;
  }
  std::vector<double> along(n);
  for (int64_t i = 0; i < n; ++i) along[i] = cost[curve[i]];
  const double target = pairwise_sum(along.data(), n) / (double)R;
  int64_t i = 0;
  for (int32_t r = 0; r < R; ++r) {
    if (i == n) break;
    if (r == R - 1) {
      for (int64_t k = i; k < n; ++k) owner[curve[k]] = r;
      break;
    }
    const int64_t start = i;
    double seg = along[i];
    ++i;
    const int64_t reserve = R - r - 1;
    while (i < n - reserve) {
      const double nxt = along[i];
      if (std::fabs(seg + nxt - target) > std::fabs(seg - target)) break;
      seg += nxt;
      ++i;
    }
    for (int64_t k = start; k < i; ++k) owner[curve[k]] = r;
  }
  return LBX_OK;
}

}  // namespace lbx

using namespace lbx;

extern "C" {

double lbx_pairwise_sum(const double* a, int64_t n) { return n > 0 ? pairwise_sum(a, n) : 0.0; }

int lbx_rank_loads(const double* cost, const int64_t* owner, int64_t n, int32_t R, double* loads) {
  clear_error();
  if (R < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1, got %d", R);
  int rc = check_owner(owner, n, R);
  if (rc) return rc;
  loads_of(cost, owner, n, R, loads);
  return LBX_OK;
}

int lbx_efficiency(const double* cost, const int64_t* owner, int64_t n, int32_t R, double* eff,
                   int32_t* degenerate) {
  clear_error();
  if (R < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1, got %d", R);
  int rc = check_owner(owner, n, R);
  if (rc) return rc;
  std::vector<double> scratch;
  return efficiency(cost, owner, n, R, eff, degenerate, scratch);
}

int lbx_knapsack(const double* cost, int64_t n, int32_t R, double cap_factor, int64_t* owner) {
  clear_error();
  return knapsack(cost, n, R, cap_factor, owner);
}

int lbx_sfc(const double* cost, const int64_t* curve, int64_t n, int32_t R, int64_t* owner) {
  clear_error();
  return sfc(cost, curve, n, R, owner);
}

int lbx_morton_order(int32_t nbz, int32_t nbx, int64_t* curve) {
  clear_error();
  if (nbz < 0 || nbx < 0) return set_error(LBX_EINVAL, "box grid must be nonnegative");
  const int64_t n = (int64_t)nbz * nbx;
  std::vector<uint64_t> codes(n);
  for (int64_t i = 0; i < n; ++i) codes[i] = spread2(i / nbx) | (spread2(i % nbx) << 1);
  stable_argsort(codes, curve);
  return LBX_OK;
}

int lbx_morton_order_3d(int32_t nb0, int32_t nb1, int32_t nb2, int64_t* curve) {
  clear_error();
  if (nb0 < 0 || nb1 < 0 || nb2 < 0) return set_error(LBX_EINVAL, "box grid must be nonnegative");
  const int64_t n = (int64_t)nb0 * nb1 * nb2;
  std::vector<uint64_t> codes(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = i / ((int64_t)nb1 * nb2), b = (i / nb2) % nb1, c = i % nb2;
    codes[i] = spread3(a) | (spread3(b) << 1) | (spread3(c) << 2);
  }
  stable_argsort(codes, curve);
  return LBX_OK;
}

int lbx_slab_mapping(int64_t n_boxes, int32_t R, int64_t* owner) {
  clear_error();
  if (R < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1, got %d", R);
  if (n_boxes <= 0) return LBX_OK;
  // np.linspace(0, n_boxes, R + 1): edge_i = i * (n/R), last edge = n exactly.
  std::vector<double> edges(R + 1);
  const double step = (double)n_boxes / (double)R;
  for (int32_t i = 0; i <= R; ++i) edges[i] = (double)i * step + 0.0;
  edges[R] = (double)n_boxes;
  for (int64_t j = 0; j < n_boxes; ++j) {
    // searchsorted(edges, j, side='right') - 1, clipped to [0, R-1]
    const double x = (double)j;
    const int64_t pos = std::upper_bound(edges.begin(), edges.end(), x) - edges.begin();
    owner[j] = std::min<int64_t>(std::max<int64_t>(pos - 1, 0), R - 1);
  }
  return LBX_OK;
}

int lbx_measured_cost(const double* work, int64_t n, double amplitude, uint64_t seed,
                      uint64_t step, double* out) {
  clear_error();
  if (n < 0) return set_error(LBX_EINVAL, "length must be >= 0");
  for (int64_t i = 0; i < n; ++i)
    if (work[i] < 0) return set_error(LBX_EINVAL, "true work must be nonnegative");
  return measured_cost(work, n, amplitude, seed, step, out);
}

}  // extern "C"
