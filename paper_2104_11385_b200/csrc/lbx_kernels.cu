// libLBX device kernels for sm_100a.
//
// The reference's hot path is two CPU loops per step:
//   advance_particles  (_kernels.pyx:12-35): x += v, absorb, stable compaction
//   bin_particles      (_kernels.pyx:38-47): per-box survivor counts
// followed by heuristic_cost (cost.py:83-95) and, for the paper's GpuClock
// strategy, an on-device per-box cycle tally.
//
// B200 design (particle state SoA float64 z, x, vz, vx in HBM, in place):
//
//  push_bin_kernel   one streaming pass, no inter-CTA ordering: 16-byte
//                    vector loads of two particles per array, push, absorbing
//                    test, z/x written back in place, per-box survivor counts
//                    and GpuClock cycles run-length aggregated per thread,
//                    warp-reduced with redux.sync and accumulated in a 32-bit
//                    shared-memory histogram flushed with one atomicAdd per
//                    box per CTA.  Absorbed particles are only counted (and
//                    the lowest absorbed index recorded).  The last CTA forms
//                    the cost vector (wp*count + wc*cells, separately rounded
//                    products: cost.py:94), writes the step record (can be
//                    mapped pinned host memory) and hands the survivor count
//                    to the next step on the device.  48 B/particle of HBM.
//
//  scan_kernel       stable compaction with a decoupled look-back scan over
//                    2048-particle tiles claimed from an in-order ticket.
//    COMPACT_SOA     after a push that absorbed particles: starts at the tile
//                    of the first absorbed index (everything before it is
//                    already in place), exits at once when nothing was
//                    absorbed.  In place is safe: a tile publishes its status
//                    only after it has loaded its input, and it writes only
//                    below its own end.
//    ADVANCE_AOS     the drop-in advance_particles: push + absorb + compaction
//                    from the reference's [n][2] layout into fresh buffers.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <climits>
#include <cmath>
#include <cstdio>

#include "lbx_internal.h"

namespace lbx {
namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kItems = 8;                 // particles per thread per scan tile
constexpr int kTile = kBlock * kItems;    // 2048 particles per scan tile
#ifndef LBX_PAIRS
#define LBX_PAIRS 2
#endif
#ifndef LBX_STREAM_MINB
#define LBX_STREAM_MINB 4
#endif
constexpr int kPairs = LBX_PAIRS;         // 16-byte pairs per thread per push iteration
constexpr int kSmemBoxesMax = 12288;      // shared-memory histogram limit (96 KB)
constexpr int kFlushIters = 128;          // push iterations between histogram flushes
constexpr unsigned kFull = 0xffffffffu;
constexpr int kClockShift = 4;            // GpuClock tally unit: 16 SM cycles
#ifndef LBX_CLOCK_AFTER_LOADS
#define LBX_CLOCK_AFTER_LOADS 1
#endif
constexpr bool kClockAfterLoads = LBX_CLOCK_AFTER_LOADS;


constexpr int kEpochShift = 42;
constexpr int kFlagShift = 40;
constexpr unsigned long long kValueMask = (1ull << kFlagShift) - 1;
constexpr unsigned long long kFlagAgg = 1ull;
constexpr unsigned long long kFlagPfx = 2ull;
constexpr unsigned kEpochMask = (1u << 22) - 1;

enum ScanMode { kAdvanceAoS = 0, kCompactSoA = 1 };

struct StepParams {
  double* z;
  double* x;
  const double* vz;
  const double* vx;
  double ez, ex, m, inv_m;
  int nbz, nbx, nb;
  int smem_hist;
  DevState* st;
  unsigned long long* g_cnt;
  unsigned long long* g_clk;
  long long* counts_out;
  double* cost_out;
  unsigned long long* clk_out;
  long long* n_out;
  long long* err_out;
  double wp, wc, cells;
  // exchange (multi-GPU)
  const int* owner;
  int me;
  double* stage;
  int* stage_dest;
  long long stage_cap;
  long long* send_counts;
  const double* kvz;
  const double* kvx;
  long long* removed_list;  // non-NULL: list removed indices, no stable compaction
  long long removed_cap;
  double* const* peer_recv;             // non-NULL: write emigrants into peers' buffers
  unsigned long long* const* peer_cursor;
  long long peer_cap;
  int l2_keep;   // set by the launcher when the particle state fits in L2 (cache-global
                 // loads / stores instead of evict-first streaming)
};

struct ScanParams {
  // COMPACT_SOA (in place)
  double* z;
  double* x;
  double* vz;
  double* vx;
  // ADVANCE_AOS (out of place)
  const double2* in_pos;
  const double2* in_vel;
  double2* out_pos;
  double2* out_vel;
  double* kvz;       // COMPACT_SOA: pending kick velocities (may be NULL)
  double* kvx;
  double ez, ex;
  long long n_host;  // ADVANCE_AOS: particle count
  DevState* st;
  unsigned long long* status;
  long long* n_out;
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long pack_status(unsigned epoch,
                                                          unsigned long long flag,
                                                          unsigned long long value) {
  return ((unsigned long long)epoch << kEpochShift) | (flag << kFlagShift) | value;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ bool inside(double z, double x, double ez, double ex) {
  return z >= 0.0 && z < ez && x >= 0.0 && x < ex;
}

// ---------------------------------------------------------------------------
// stream_kernel: push_bin (kPush) and partition (!kPush), optional exchange
// ---------------------------------------------------------------------------

template <bool kClock>
__device__ __forceinline__ void hist_add(const StepParams& p, unsigned* s_cnt, unsigned* s_clk,
                                         int b, unsigned cnt, unsigned clk) {
  if (p.smem_hist) {
    atomicAdd(s_cnt + b, cnt);
    if (kClock) atomicAdd(s_clk + b, clk);
  } else {
    atomicAdd(p.g_cnt + b, (unsigned long long)cnt);
    if (kClock) atomicAdd(p.g_clk + b, (unsigned long long)clk);
  }
}

template <bool kClock>
__device__ __forceinline__ void hist_flush(const StepParams& p, unsigned* s_cnt, unsigned* s_clk) {
  for (int b = threadIdx.x; b < p.nb; b += kBlock) {
    const unsigned c = s_cnt[b];
    if (c) {
      atomicAdd(p.g_cnt + b, (unsigned long long)c);
      s_cnt[b] = 0u;
    }
    if (kClock) {
      const unsigned k = s_clk[b];
      if (k) {
        atomicAdd(p.g_clk + b, (unsigned long long)k);
        s_clk[b] = 0u;
      }
    }
  }
}

// Stage one emigrant record (warp-aggregated slot reservation).
__device__ __forceinline__ void stage_emigrant(const StepParams& p, bool em, long long i,
                                               double z, double x, double vz, double vx,
                                               int dest) {
  const unsigned mask = __ballot_sync(kFull, em);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  if (p.peer_recv) {
    // Fused exchange over peer memory: lanes going to the same rank reserve
    // their slots with ONE remote atomic on that rank's cursor and write the
    // records straight into its receive buffer (NVLink / NVSwitch stores).
    if (!em) return;                          // only the lanes in `mask` take part below
    const unsigned grp = __match_any_sync(mask, dest);
    const int leader = __ffs(grp) - 1;
    unsigned long long base = 0;
    if (lane == leader)
      base = atomicAdd(p.peer_cursor[dest], (unsigned long long)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    const long long slot = (long long)base + __popc(grp & lanemask_lt());
    atomicAdd((unsigned long long*)(p.send_counts + dest), 1ull);
    if (slot >= p.peer_cap) {
      atomicOr((unsigned long long*)&p.st->err, 1ull << 62);  // receive buffer overflow
      return;
    }
    double2* r = reinterpret_cast<double2*>(p.peer_recv[dest] + slot * 6);
    r[0] = make_double2(z, x);
    r[1] = make_double2(vz, vx);
    r[2] = make_double2(p.kvz ? p.kvz[i] : 0.0, p.kvx ? p.kvx[i] : 0.0);
    __threadfence_system();   // visible to the destination once our kernel has completed
    return;
  }
  unsigned long long base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(&p.st->staged, (unsigned long long)__popc(mask));
  base = __shfl_sync(kFull, base, __ffs(mask) - 1);
  if (!em) return;
  const long long slot = (long long)base + __popc(mask & lanemask_lt());
  if (slot >= p.stage_cap) {
    atomicOr((unsigned long long*)&p.st->err, 1ull << 62);  // staging overflow
    return;
  }
  double* r = p.stage + slot * 6;
  r[0] = z;
  r[1] = x;
  r[2] = vz;
  r[3] = vx;
  r[4] = p.kvz ? p.kvz[i] : 0.0;
  r[5] = p.kvx ? p.kvx[i] : 0.0;
  p.stage_dest[slot] = dest;
  atomicAdd((unsigned long long*)(p.send_counts + dest), 1ull);
}

template <bool kClock, bool kPow2, bool kExch, bool kPush>
__global__ void __launch_bounds__(kBlock, LBX_STREAM_MINB) stream_kernel(StepParams p) {
  constexpr bool kHist = kPush;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* s_cnt = reinterpret_cast<unsigned*>(smem_raw);
  unsigned* s_clk = s_cnt + p.nb;
  int* s_owner = reinterpret_cast<int*>(s_cnt + (kClock ? 2 : 1) * p.nb);
  __shared__ long long s_n;
  __shared__ unsigned s_rot;
  __shared__ int s_last;
  __shared__ unsigned long long s_red[kWarps];
  __shared__ long long s_min[kWarps];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  if (tid == 0) {
    s_n = *((volatile long long*)&p.st->n);
    s_rot = *((volatile unsigned*)&p.st->rot);
  }
  if (p.smem_hist) {
    for (int b = tid; b < p.nb; b += kBlock) {
      if (kHist) s_cnt[b] = 0u;
      if (kClock) s_clk[b] = 0u;
      if (kExch) s_owner[b] = p.owner[b];
    }
  }
  __syncthreads();
  const int* owner = p.smem_hist ? s_owner : p.owner;
  const long long n = s_n;
  const long long npairs = (n + 1) >> 1;
  double2* z2 = reinterpret_cast<double2*>(p.z);
  double2* x2 = reinterpret_cast<double2*>(p.x);
  const double2* vz2 = reinterpret_cast<const double2*>(p.vz);
  const double2* vx2 = reinterpret_cast<const double2*>(p.vx);

  unsigned long long removed = 0;
  long long first_out = LLONG_MAX;
  long long err = 0;
  int iter = 0;
  // The loop trip count is uniform across the CTA (grid-stride over
  // CTA-sized chunks), so the periodic histogram flush can use barriers.
  // GpuClock: the chunk -> CTA assignment is rotated by a pseudo-random
  // offset every step (DevState::rot), so a box's particles do not sit in the
  // same CTA slot / wave step after step: at L2-resident sizes the thread
  // time of a chunk depends on when it runs (full first wave vs draining
  // tail), and the runtime sums the tally over the LB window, where the
  // rotation averages that out.
  const long long chunk = (long long)kBlock * kPairs;
  const long long nchunks = (npairs + chunk - 1) / chunk;
  // offset = nchunks x frac(rot x golden ratio): a Weyl sequence, so any
  // window of consecutive steps spreads its offsets evenly over the chunks
  const unsigned long long phase = ((unsigned long long)s_rot * 0x9E3779B97F4A7C15ull) >> 32;
  const long long rot =
      kClock && nchunks > 1 ? (long long)((phase * (unsigned long long)nchunks) >> 32) : 0;
  for (long long k = blockIdx.x; k < nchunks; k += gridDim.x) {
    long long c = k + rot;
    if (c >= nchunks) c -= nchunks;
    const long long q0 = c * chunk;
    long long t0 = 0;
    if (kClock && !kClockAfterLoads) t0 = clock64();
    double pz[2 * kPairs], px[2 * kPairs], pvz[2 * kPairs], pvx[2 * kPairs];
    bool keep[2 * kPairs], valid[2 * kPairs];
#pragma unroll
    for (int r = 0; r < kPairs; ++r) {
      const long long q = q0 + r * kBlock + tid;
      double2 a = make_double2(-1.0, -1.0), b = a, c = make_double2(0.0, 0.0), d = c;
      const bool any = q < npairs;
      if (any) {
        // L2-resident steps (small sets, p.l2_keep) keep the particle state in
        // L2 across steps; large ones stream it (evict-first)
        a = p.l2_keep ? __ldcg(z2 + q) : __ldcs(z2 + q);
        b = p.l2_keep ? __ldcg(x2 + q) : __ldcs(x2 + q);
        if (kPush || kExch) {
          c = p.l2_keep ? __ldcg(vz2 + q) : __ldcs(vz2 + q);
          d = p.l2_keep ? __ldcg(vx2 + q) : __ldcs(vx2 + q);
        }
      }
      pvz[2 * r] = c.x;
      pvz[2 * r + 1] = c.y;
      pvx[2 * r] = d.x;
      pvx[2 * r + 1] = d.y;
      if (kPush) {
        pz[2 * r] = __dadd_rn(a.x, c.x);
        pz[2 * r + 1] = __dadd_rn(a.y, c.y);
        px[2 * r] = __dadd_rn(b.x, d.x);
        px[2 * r + 1] = __dadd_rn(b.y, d.y);
      } else {
        pz[2 * r] = a.x;
        pz[2 * r + 1] = a.y;
        px[2 * r] = b.x;
        px[2 * r + 1] = b.y;
      }
      valid[2 * r] = any;
      valid[2 * r + 1] = 2 * q + 1 < n;
    }
    // GpuClock window: opened after the pushed positions exist, i.e. after the
    // loads landed (the CS2R issues behind the DADDs that consume them), so
    // the tally is the thread's compute time on its particles -- not the
    // memory latency, which at L2-resident sizes depends on WHEN a chunk runs
    // (first or second wave) rather than on the box's work.
    if (kClock && kClockAfterLoads) t0 = clock64();
#pragma unroll
    for (int k = 0; k < 2 * kPairs; ++k) keep[k] = valid[k] && inside(pz[k], px[k], p.ez, p.ex);

    int box[2 * kPairs];
    bool emig[2 * kPairs];
#pragma unroll
    for (int k = 0; k < 2 * kPairs; ++k) {
      box[k] = -1;
      emig[k] = false;
      if (keep[k]) {
        int bz, bx;
        if (kPow2) {
          bz = (int)__dmul_rn(pz[k], p.inv_m);  // exact: M is a power of two
          bx = (int)__dmul_rn(px[k], p.inv_m);
        } else {
          bz = (int)__ddiv_rn(pz[k], p.m);
          bx = (int)__ddiv_rn(px[k], p.m);
        }
        if (bz < p.nbz && bx < p.nbx) {
          box[k] = bz * p.nbx + bx;
          if (kExch) emig[k] = owner[box[k]] != p.me;
        } else {
          ++err;
        }
      }
    }
    // stores: pushed positions in place, removal sentinel (z = -1) for
    // emigrants so the compaction drops them like absorbed particles
#pragma unroll
    for (int r = 0; r < kPairs; ++r) {
      const long long q = q0 + r * kBlock + tid;
      if (!valid[2 * r]) continue;
      const double z0 = emig[2 * r] ? -1.0 : pz[2 * r];
      const double z1 = emig[2 * r + 1] ? -1.0 : pz[2 * r + 1];
      if (kPush) {
        if (p.l2_keep) {
          __stcg(z2 + q, make_double2(z0, z1));
          __stcg(x2 + q, make_double2(px[2 * r], px[2 * r + 1]));
        } else {
          __stcs(z2 + q, make_double2(z0, z1));
          __stcs(x2 + q, make_double2(px[2 * r], px[2 * r + 1]));
        }
      } else if (emig[2 * r] || emig[2 * r + 1]) {
        __stcs(z2 + q, make_double2(z0, z1));
      }
      const long long i0 = 2 * q;
      if (!keep[2 * r] || emig[2 * r]) {
        ++removed;
        first_out = min(first_out, i0);
      }
      if (valid[2 * r + 1] && (!keep[2 * r + 1] || emig[2 * r + 1])) {
        ++removed;
        first_out = min(first_out, i0 + 1);
      }
    }
    if (kExch && p.removed_list) {  // list removed indices (warp-aggregated)
#pragma unroll
      for (int k = 0; k < 2 * kPairs; ++k) {
        const long long i = 2 * (q0 + (k >> 1) * kBlock + tid) + (k & 1);
        const bool rm = valid[k] && (!keep[k] || emig[k]);
        const unsigned m = __ballot_sync(kFull, rm);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1)
          base = atomicAdd(&p.st->removed_count, (unsigned long long)__popc(m));
        base = __shfl_sync(kFull, base, __ffs(m) - 1);
        if (rm) {
          const long long slot = (long long)base + __popc(m & lanemask_lt());
          if (slot < p.removed_cap) p.removed_list[slot] = i;
          else atomicOr((unsigned long long*)&p.st->err, 1ull << 61);
        }
      }
    }
    if (kExch) {
#pragma unroll
      for (int k = 0; k < 2 * kPairs; ++k) {
        const long long i = 2 * (q0 + (k >> 1) * kBlock + tid) + (k & 1);
        stage_emigrant(p, emig[k], i, pz[k], px[k], pvz[k], pvx[k],
                       emig[k] ? owner[box[k]] : 0);
      }
    }
    if (kHist) {
      unsigned dt = 0;
      if (kClock) {
        const long long t1 = clock64();
        dt = (unsigned)min(t1 - t0, (long long)(1 << 20)) >> kClockShift;
      }
      int cur = -1;
      unsigned run = 0;
#pragma unroll
      for (int k = 0; k < 2 * kPairs; ++k) {
        if (box[k] != cur) {
          if (cur >= 0) hist_add<kClock>(p, s_cnt, s_clk, cur, run, dt * run);
          cur = box[k];
          run = 0;
        }
        run += (box[k] >= 0) ? 1u : 0u;
      }
      const int cur0 = __shfl_sync(kFull, cur, 0);
      if (__all_sync(kFull, cur == cur0)) {
        const unsigned tot = __reduce_add_sync(kFull, run);
        const unsigned clk = kClock ? __reduce_add_sync(kFull, dt * run) : 0u;
        if (lane == 0 && cur0 >= 0 && tot) hist_add<kClock>(p, s_cnt, s_clk, cur0, tot, clk);
      } else if (cur >= 0 && run) {
        hist_add<kClock>(p, s_cnt, s_clk, cur, run, dt * run);
      }
      if (p.smem_hist && ++iter == kFlushIters) {  // keep 32-bit accumulators bounded
        iter = 0;
        __syncthreads();
        hist_flush<kClock>(p, s_cnt, s_clk);
        __syncthreads();
      }
    }
  }

  // ---- CTA totals: removed count, first removed index, errors ----
  unsigned long long wa = (unsigned long long)warp_sum_ll((long long)removed);
  long long wm = warp_min_ll(first_out);
  long long we = warp_sum_ll(err);
  if (lane == 0) {
    s_red[warp] = wa;
    s_min[warp] = wm;
  }
  if (we && lane == 0) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)we);
  __syncthreads();
  if (tid == 0) {
    unsigned long long ta = 0;
    long long tm = LLONG_MAX;
    for (int w = 0; w < kWarps; ++w) {
      ta += s_red[w];
      tm = min(tm, s_min[w]);
    }
    if (ta) {
      atomicAdd(&p.st->leavers, ta);
      atomicMin(&p.st->first_leaver, tm);
    }
  }
  if (kHist && p.smem_hist) hist_flush<kClock>(p, s_cnt, s_clk);
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last) return;

  // ---- last CTA: step epilogue ----
  __threadfence();
#ifndef LBX_DIAG_NO_RECORD
  if (kHist)
    step_record<kClock>(p.g_cnt, p.g_clk, p.nb, p.counts_out, p.cost_out, p.clk_out, p.wp, p.wc,
                        p.cells, kClockShift);
#endif
  if (tid == 0) {
    const unsigned long long lv = *((volatile unsigned long long*)&p.st->leavers);
    const long long n_new = n - (long long)lv;
    if (p.n_out) *p.n_out = n_new;
    if (p.err_out) *p.err_out = *((volatile long long*)&p.st->err);
    p.st->n_old = n;
    p.st->n = n_new;
    p.st->done = 0u;
    p.st->staged = 0ull;
    if (kClock) p.st->rot += 1u;
    __threadfence_system();
  }
}


// ---------------------------------------------------------------------------
// stream3d_kernel: 3D push + absorb + per-box counts / GpuClock (config C4)
// SoA z, y, x, vz, vy, vx in place; absorbed particles get z = -1 so the
// stable compaction (which tests z, x) drops them.  Box size power of two.
// ---------------------------------------------------------------------------
struct Step3DParams {
  double *z, *y, *x;
  const double *vz, *vy, *vx;
  double ez, ey, ex, inv_m;
  int nbz, nby, nbx, nb;
  int smem_hist;
  DevState* st;
  unsigned long long* g_cnt;
  unsigned long long* g_clk;
  long long* counts_out;
  double* cost_out;
  unsigned long long* clk_out;
  long long* n_out;
  long long* err_out;
  double wp, wc, cells;
  long long* removed_list;
  long long removed_cap;
  // multi-GPU 3D exchange (Distributed3D): survivors in boxes another rank
  // owns are staged as (z, y, x, vz, vy, vx) records and removed locally
  const int* owner;   // NULL: no exchange
  int me;
  double* stage;
  int* stage_dest;
  long long stage_cap;
  long long* send_counts;
};

// Stage one 3D emigrant record (warp-collective: every lane calls it).
__device__ __forceinline__ void stage3d(const Step3DParams& p, bool em, double z, double y,
                                        double x, double vz, double vy, double vx, int dest) {
  const unsigned mask = __ballot_sync(kFull, em);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(&p.st->staged, (unsigned long long)__popc(mask));
  base = __shfl_sync(kFull, base, __ffs(mask) - 1);
  if (!em) return;
  const long long slot = (long long)base + __popc(mask & lanemask_lt());
  if (slot >= p.stage_cap) {
    atomicOr((unsigned long long*)&p.st->err, 1ull << 62);  // staging overflow
    return;
  }
  double* r = p.stage + slot * 6;
  r[0] = z;
  r[1] = y;
  r[2] = x;
  r[3] = vz;
  r[4] = vy;
  r[5] = vx;
  p.stage_dest[slot] = dest;
  atomicAdd((unsigned long long*)(p.send_counts + dest), 1ull);
}

template <bool kClock>
__global__ void __launch_bounds__(kBlock, 4) stream3d_kernel(Step3DParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* s_cnt = reinterpret_cast<unsigned*>(smem_raw);
  unsigned* s_clk = s_cnt + p.nb;
  __shared__ long long s_n;
  __shared__ int s_last;
  __shared__ unsigned long long s_red[kWarps];
  __shared__ long long s_min[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_n = *((volatile long long*)&p.st->n);
  if (p.smem_hist)
    for (int b = tid; b < p.nb; b += kBlock) {
      s_cnt[b] = 0u;
      if (kClock) s_clk[b] = 0u;
    }
  __syncthreads();
  const long long n = s_n, npairs = (n + 1) >> 1;
  const long long stride = (long long)gridDim.x * kBlock * kPairs;
  double2* z2 = reinterpret_cast<double2*>(p.z);
  double2* y2 = reinterpret_cast<double2*>(p.y);
  double2* x2 = reinterpret_cast<double2*>(p.x);
  const double2* vz2 = reinterpret_cast<const double2*>(p.vz);
  const double2* vy2 = reinterpret_cast<const double2*>(p.vy);
  const double2* vx2 = reinterpret_cast<const double2*>(p.vx);
  unsigned long long removed = 0;
  long long first_out = LLONG_MAX, err = 0;
  int iter = 0;
  for (long long q0 = (long long)blockIdx.x * kBlock * kPairs; q0 < npairs; q0 += stride) {
    long long t0 = 0;
    if (kClock) t0 = clock64();
    int box[2 * kPairs];
#pragma unroll
    for (int r = 0; r < kPairs; ++r) {
      const long long q = q0 + r * kBlock + tid;
      const bool any = q < npairs;
      double2 a = make_double2(-1.0, -1.0), b = a, c = a;
      double2 d = make_double2(0.0, 0.0), e = d, f = d;
      if (any) {
        a = __ldcs(z2 + q);
        b = __ldcs(y2 + q);
        c = __ldcs(x2 + q);
        d = __ldcs(vz2 + q);
        e = __ldcs(vy2 + q);
        f = __ldcs(vx2 + q);
      }
      double nz[2] = {__dadd_rn(a.x, d.x), __dadd_rn(a.y, d.y)};
      const double ny[2] = {__dadd_rn(b.x, e.x), __dadd_rn(b.y, e.y)};
      const double nx[2] = {__dadd_rn(c.x, f.x), __dadd_rn(c.y, f.y)};
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const long long i = 2 * q + t;
        const bool valid = i < n;
        const bool keep = valid && nz[t] >= 0.0 && nz[t] < p.ez && ny[t] >= 0.0 &&
                          ny[t] < p.ey && nx[t] >= 0.0 && nx[t] < p.ex;
        box[2 * r + t] = -1;
        bool emig = false;
        int dest = 0;
        if (keep) {
          const int bz = (int)__dmul_rn(nz[t], p.inv_m), by = (int)__dmul_rn(ny[t], p.inv_m),
                    bx = (int)__dmul_rn(nx[t], p.inv_m);
          if (bz < p.nbz && by < p.nby && bx < p.nbx) {
            box[2 * r + t] = (bz * p.nby + by) * p.nbx + bx;
            if (p.owner) {
              dest = __ldg(p.owner + box[2 * r + t]);
              emig = dest != p.me;
            }
          } else {
            ++err;
          }
        } else if (valid) {
          ++removed;
          first_out = min(first_out, i);
        }
        if (p.owner) {   // counted in its box above; leaves this rank's arrays
          const double vz0 = t ? d.y : d.x, vy0 = t ? e.y : e.x, vx0 = t ? f.y : f.x;
          stage3d(p, emig, nz[t], ny[t], nx[t], vz0, vy0, vx0, dest);
          if (emig) {
            ++removed;
            first_out = min(first_out, i);
          }
        }
        if (valid && (!keep || emig)) nz[t] = -1.0;  // compaction sentinel
        if (p.removed_list) {
          const bool rm = valid && (!keep || emig);
          const unsigned m = __ballot_sync(kFull, rm);
          if (m) {
            unsigned long long base = 0;
            if (lane == __ffs(m) - 1)
              base = atomicAdd(&p.st->removed_count, (unsigned long long)__popc(m));
            base = __shfl_sync(kFull, base, __ffs(m) - 1);
            if (rm) {
              const long long slot = (long long)base + __popc(m & lanemask_lt());
              if (slot < p.removed_cap) p.removed_list[slot] = i;
              else atomicOr((unsigned long long*)&p.st->err, 1ull << 61);
            }
          }
        }
      }
      if (any) {
        __stcs(z2 + q, make_double2(nz[0], nz[1]));
        __stcs(y2 + q, make_double2(ny[0], ny[1]));
        __stcs(x2 + q, make_double2(nx[0], nx[1]));
      }
    }
    unsigned dt = 0;
    if (kClock) dt = (unsigned)min(clock64() - t0, (long long)(1 << 20)) >> kClockShift;
    int cur = -1;
    unsigned run = 0;
#pragma unroll
    for (int k = 0; k < 2 * kPairs; ++k) {
      if (box[k] != cur) {
        if (cur >= 0) {
          if (p.smem_hist) {
            atomicAdd(s_cnt + cur, run);
            if (kClock) atomicAdd(s_clk + cur, dt * run);
          } else {
            atomicAdd(p.g_cnt + cur, (unsigned long long)run);
            if (kClock) atomicAdd(p.g_clk + cur, (unsigned long long)(dt * run));
          }
        }
        cur = box[k];
        run = 0;
      }
      run += box[k] >= 0 ? 1u : 0u;
    }
    const int cur0 = __shfl_sync(kFull, cur, 0);
    const bool uni = __all_sync(kFull, cur == cur0);
    unsigned tot = run, clk = dt * run;
    if (uni) {
      tot = __reduce_add_sync(kFull, run);
      clk = kClock ? __reduce_add_sync(kFull, dt * run) : 0u;
    }
    if ((uni ? lane == 0 && cur0 >= 0 : cur >= 0) && tot) {
      const int b = uni ? cur0 : cur;
      if (p.smem_hist) {
        atomicAdd(s_cnt + b, tot);
        if (kClock) atomicAdd(s_clk + b, clk);
      } else {
        atomicAdd(p.g_cnt + b, (unsigned long long)tot);
        if (kClock) atomicAdd(p.g_clk + b, (unsigned long long)clk);
      }
    }
    if (p.smem_hist && ++iter == kFlushIters) {
      iter = 0;
      __syncthreads();
      for (int b = tid; b < p.nb; b += kBlock) {
        if (s_cnt[b]) atomicAdd(p.g_cnt + b, (unsigned long long)s_cnt[b]), s_cnt[b] = 0u;
        if (kClock && s_clk[b]) atomicAdd(p.g_clk + b, (unsigned long long)s_clk[b]), s_clk[b] = 0u;
      }
      __syncthreads();
    }
  }
  const unsigned long long wa = (unsigned long long)warp_sum_ll((long long)removed);
  const long long wm = warp_min_ll(first_out), we = warp_sum_ll(err);
  if (lane == 0) {
    s_red[warp] = wa;
    s_min[warp] = wm;
    if (we) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)we);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long ta = 0;
    long long tm = LLONG_MAX;
    for (int w = 0; w < kWarps; ++w) ta += s_red[w], tm = min(tm, s_min[w]);
    if (ta) {
      atomicAdd(&p.st->leavers, ta);
      atomicMin(&p.st->first_leaver, tm);
    }
  }
  if (p.smem_hist)
    for (int b = tid; b < p.nb; b += kBlock) {
      if (s_cnt[b]) atomicAdd(p.g_cnt + b, (unsigned long long)s_cnt[b]);
      if (kClock && s_clk[b]) atomicAdd(p.g_clk + b, (unsigned long long)s_clk[b]);
    }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  step_record<kClock>(p.g_cnt, p.g_clk, p.nb, p.counts_out, p.cost_out, p.clk_out, p.wp, p.wc,
                      p.cells, kClockShift);
  if (tid == 0) {
    const long long n_new = n - (long long)*((volatile unsigned long long*)&p.st->leavers);
    if (p.n_out) *p.n_out = n_new;
    if (p.err_out) *p.err_out = *((volatile long long*)&p.st->err);
    p.st->n_old = n;
    p.st->n = n_new;
    p.st->done = 0u;
    __threadfence_system();
  }
}

// Adoption-time 3D migration: particles in boxes another rank now owns are
// staged (as stream3d_kernel's emigrants) and listed as removed; no push.
__global__ void __launch_bounds__(kBlock) partition3d_kernel(Step3DParams p) {
  const long long n = *((volatile long long*)&p.st->n);
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * kBlock;
  const long long end = (n + kBlock - 1) / kBlock * kBlock;   // whole warps: collectives
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < end; i += stride) {
    const bool valid = i < n;
    double z = 0, y = 0, x = 0, vz = 0, vy = 0, vx = 0;
    bool em = false;
    int dest = 0;
    if (valid) {
      z = p.z[i];
      y = p.y[i];
      x = p.x[i];
      const int bz = (int)__dmul_rn(z, p.inv_m), by = (int)__dmul_rn(y, p.inv_m),
                bx = (int)__dmul_rn(x, p.inv_m);
      if (z >= 0.0 && bz < p.nbz && y >= 0.0 && by < p.nby && x >= 0.0 && bx < p.nbx) {
        dest = __ldg(p.owner + (bz * p.nby + by) * p.nbx + bx);
        em = dest != p.me;
      } else {
        atomicAdd((unsigned long long*)&p.st->err, 1ull);
      }
      if (em) {
        vz = p.vz[i];
        vy = p.vy[i];
        vx = p.vx[i];
      }
    }
    stage3d(p, em, z, y, x, vz, vy, vx, dest);
    const unsigned m = __ballot_sync(kFull, em);
    if (m) {
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&p.st->removed_count, (unsigned long long)__popc(m));
      base = __shfl_sync(kFull, base, __ffs(m) - 1);
      if (em) {
        const long long slot = (long long)base + __popc(m & lanemask_lt());
        if (slot < p.removed_cap) p.removed_list[slot] = i;
        else atomicOr((unsigned long long*)&p.st->err, 1ull << 61);
        p.z[i] = -1.0;
      }
    }
  }
}

// n_out = {survivors kept in place, error code} after partition3d_kernel.
__global__ void partition_done_kernel(DevState* st, long long* n_out) {
  const long long L = (long long)st->removed_count;
  n_out[0] = st->n - L;
  n_out[1] = st->err;
  st->n -= L;
}

// ---------------------------------------------------------------------------
// scan_kernel (decoupled look-back stable compaction)
// ---------------------------------------------------------------------------

// Exclusive prefix of survivors over all tiles before `tile` (warp 0 only).
// Tile tile0 publishes an inclusive prefix that already includes everything
// before it, so the walk never goes below tile0.
__device__ long long lookback(unsigned long long* status, long long tile, long long tile0,
                              unsigned epoch) {
  const int lane = threadIdx.x & 31;
  long long acc = 0;
  long long top = tile - 1;
  while (true) {
    const long long idx = top - lane;
    unsigned long long s = 0;
    unsigned long long flag = kFlagPfx;  // below tile0: virtual, never reached first
    if (idx >= tile0) {
      do {
        s = ld_acquire(status + idx);
        flag = ((unsigned)(s >> kEpochShift) == epoch) ? ((s >> kFlagShift) & 3ull) : 0ull;
      } while (flag == 0ull);
    }
    const long long val = (long long)(s & kValueMask);
    const unsigned pfx = __ballot_sync(kFull, flag == kFlagPfx);
    if (pfx) {
      const int first = __ffs(pfx) - 1;  // nearest predecessor with a prefix
      acc += warp_sum_ll(lane <= first ? val : 0ll);
      return acc;
    }
    acc += warp_sum_ll(val);
    top -= 32;
  }
}

template <int kMode>
__global__ void __launch_bounds__(kBlock, kMode == kCompactSoA ? 2 : 3) scan_kernel(ScanParams p) {
  __shared__ long long s_tile;
  __shared__ long long s_prefix;
  __shared__ int s_total;
  __shared__ int s_last;
  __shared__ long long s_n;
  __shared__ long long s_tile0;
  __shared__ unsigned s_epoch;
  constexpr int kRows = (kMode == kCompactSoA) ? kItems / 2 : kItems;
  __shared__ int s_row[kRows * kWarps];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  if (tid == 0) {
    if (kMode == kCompactSoA) {
      const unsigned long long lv = *((volatile unsigned long long*)&p.st->leavers);
      s_n = lv ? *((volatile long long*)&p.st->n_old) : 0;
      s_tile0 = lv ? (*((volatile long long*)&p.st->first_leaver)) / kTile : 0;
    } else {
      s_n = p.n_host;
      s_tile0 = 0;
    }
    s_epoch = *((volatile unsigned*)&p.st->epoch);
  }
  __syncthreads();
  const long long n = s_n;
  const long long tile0 = s_tile0;
  const unsigned epoch = s_epoch;
  const long long ntiles = (n + kTile - 1) / kTile;
  if (kMode == kCompactSoA && n == 0) return;  // nothing absorbed: data already final

  while (true) {
    if (tid == 0) s_tile = tile0 + (long long)atomicAdd(&p.st->ticket, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    if (tile >= ntiles) break;
    const long long base = tile * kTile;
    const long long valid = min((long long)kTile, n - base);

    double pz[kItems], px[kItems], pvz[kItems], pvx[kItems];
    double pkz[kMode == kCompactSoA ? kItems : 1], pkx[kMode == kCompactSoA ? kItems : 1];
    bool keep[kItems];
    if (kMode == kCompactSoA) {
      const double2* z2 = reinterpret_cast<const double2*>(p.z);
      const double2* x2 = reinterpret_cast<const double2*>(p.x);
      const double2* vz2 = reinterpret_cast<const double2*>(p.vz);
      const double2* vx2 = reinterpret_cast<const double2*>(p.vx);
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const long long q = (base >> 1) + r * kBlock + tid;
        const long long i0 = 2 * q;
        double2 a = make_double2(-1.0, -1.0), b = a, c = make_double2(0.0, 0.0), d = c;
        if (i0 < n) {
          a = __ldcs(z2 + q);
          b = __ldcs(x2 + q);
          c = __ldcs(vz2 + q);
          d = __ldcs(vx2 + q);
        }
        pz[2 * r] = a.x;
        pz[2 * r + 1] = a.y;
        px[2 * r] = b.x;
        px[2 * r + 1] = b.y;
        pvz[2 * r] = c.x;
        pvz[2 * r + 1] = c.y;
        pvx[2 * r] = d.x;
        pvx[2 * r + 1] = d.y;
        if (p.kvz) {
          double2 e = make_double2(0.0, 0.0);
          if (i0 < n) e = __ldcs(reinterpret_cast<const double2*>(p.kvz) + q);
          pkz[2 * r] = e.x;
          pkz[2 * r + 1] = e.y;
        }
        if (p.kvx) {
          double2 f = make_double2(0.0, 0.0);
          if (i0 < n) f = __ldcs(reinterpret_cast<const double2*>(p.kvx) + q);
          pkx[2 * r] = f.x;
          pkx[2 * r + 1] = f.y;
        }
        keep[2 * r] = i0 < n && inside(a.x, b.x, p.ez, p.ex);
        keep[2 * r + 1] = i0 + 1 < n && inside(a.y, b.y, p.ez, p.ex);
      }
    } else {
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const long long i = base + r * kBlock + tid;
        double2 a = make_double2(0.0, 0.0), c = a;
        if (i < n) {
          a = __ldcs(p.in_pos + i);
          c = __ldcs(p.in_vel + i);
        }
        pvz[r] = c.x;
        pvx[r] = c.y;
        pz[r] = __dadd_rn(a.x, c.x);
        px[r] = __dadd_rn(a.y, c.y);
        keep[r] = i < n && inside(pz[r], px[r], p.ez, p.ex);
      }
    }

    // tile-local ranks of survivors (tile order == index order)
    int pre[kItems];
    const unsigned lt = lanemask_lt();
    if (kMode == kCompactSoA) {
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const unsigned b0 = __ballot_sync(kFull, keep[2 * r]);
        const unsigned b1 = __ballot_sync(kFull, keep[2 * r + 1]);
        pre[2 * r] = __popc(b0 & lt) + __popc(b1 & lt);
        pre[2 * r + 1] = pre[2 * r] + (keep[2 * r] ? 1 : 0);
        if (lane == 0) s_row[r * kWarps + warp] = __popc(b0) + __popc(b1);
      }
    } else {
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const unsigned b0 = __ballot_sync(kFull, keep[r]);
        pre[r] = __popc(b0 & lt);
        if (lane == 0) s_row[r * kWarps + warp] = __popc(b0);
      }
    }
    __syncthreads();

    if (warp == 0) {
      constexpr int kPer = (kRows * kWarps) / 32;
      int v[kPer];
      int sum = 0;
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        v[e] = s_row[lane * kPer + e];
        sum += v[e];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(kFull, incl, 31);
      int off = incl - sum;
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        s_row[lane * kPer + e] = off;
        off += v[e];
      }
      long long prefix = tile0 * kTile;  // everything before tile0 stays put
      if (tile == tile0) {
        if (lane == 0) {
          __threadfence();
          st_release(p.status + tile,
                     pack_status(epoch, kFlagPfx, (unsigned long long)(prefix + total)));
        }
      } else {
        if (lane == 0) {
          __threadfence();
          st_release(p.status + tile, pack_status(epoch, kFlagAgg, (unsigned long long)total));
        }
        prefix = lookback(p.status, tile, tile0, epoch);
        if (lane == 0) {
          st_release(p.status + tile,
                     pack_status(epoch, kFlagPfx, (unsigned long long)(prefix + total)));
        }
      }
      if (lane == 0) {
        s_prefix = prefix;
        s_total = total;
      }
    }
    __syncthreads();
    const long long prefix = s_prefix;
    const bool in_place = (prefix == base) && ((long long)s_total == valid);

    if (kMode == kCompactSoA) {
      if (!in_place) {
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          if (keep[k]) {
            const long long d = prefix + s_row[(k >> 1) * kWarps + warp] + pre[k];
            p.z[d] = pz[k];
            p.x[d] = px[k];
            p.vz[d] = pvz[k];
            p.vx[d] = pvx[k];
            if (p.kvz) p.kvz[d] = pkz[k];
            if (p.kvx) p.kvx[d] = pkx[k];
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        if (keep[k]) {
          const long long d = prefix + s_row[k * kWarps + warp] + pre[k];
          __stcs(p.out_pos + d, make_double2(pz[k], px[k]));
          __stcs(p.out_vel + d, make_double2(pvz[k], pvx[k]));
        }
      }
    }
    __syncthreads();  // s_row / s_tile reuse
  }

  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last || tid != 0) return;
  __threadfence();
  long long n_new = tile0 * kTile;
  if (ntiles > tile0) n_new = (long long)(ld_acquire(p.status + (ntiles - 1)) & kValueMask);
  if (kMode == kAdvanceAoS && p.n_out) *p.n_out = n_new;
  if (kMode == kCompactSoA) {
    p.st->leavers = 0ull;
    p.st->first_leaver = LLONG_MAX;
    if (*((volatile long long*)&p.st->n) != n_new) p.st->err += 1ll << 40;  // invariant
  }
  p.st->ticket = 0ull;
  p.st->done = 0u;
  const unsigned ne = (epoch + 1u) & kEpochMask;
  p.st->epoch = ne ? ne : 1u;
  __threadfence();
}

// ---------------------------------------------------------------------------
// Stable compaction without a look-back chain (COMPACT_SOA, the default):
//   compact_count_kernel  survivors per 2,048-particle tile from the first
//                         absorbed tile on (reads z, x: 16 B / particle);
//   compact_scan_kernel   one CTA: exclusive scan of the tile counts -> each
//                         tile's first output slot;
//   compact_move_kernel   tiles in ticket order: load (8-byte lane-consecutive
//                         loads), rank survivors by ballot, store them at the
//                         tile's slot (consecutive survivors -> coalesced
//                         stores).  In place: a tile's output range lies in
//                         the input of the same or earlier tiles, so it first
//                         waits for those tiles' "loaded" flags (status words,
//                         epoch-tagged like the look-back's).
// ncu of the look-back kernel on a leaver-heavy step (100 M particles, 0.33 %
// absorbed anywhere): 2.19 ms, warps stalled at the CTA barrier 23 per issue
// while warp 0 walked the look-back -- no loads in flight meanwhile.
// 80 B / particle instead of 64, all of it streaming.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool compact_range(const DevState* st, long long* n, long long* tile0) {
  const unsigned long long lv = *((volatile const unsigned long long*)&st->leavers);
  if (!lv) return false;
  *n = *((volatile const long long*)&st->n_old);
  *tile0 = (*((volatile const long long*)&st->first_leaver)) / kTile;
  return true;
}

// CTA c counts the survivors of a contiguous tile range and writes each
// tile's exclusive prefix within the range plus the range total.
__global__ void __launch_bounds__(kBlock) compact_count_kernel(ScanParams p,
                                                               unsigned long long* tile_cnt,
                                                               unsigned long long* cta_tot) {
  long long n, tile0;
  if (!compact_range(p.st, &n, &tile0)) return;
  const long long m = (n + kTile - 1) / kTile - tile0;
  const long long per = (m + gridDim.x - 1) / gridDim.x;
  const long long a = min(m, (long long)blockIdx.x * per), b = min(m, a + per);
  __shared__ int s_w[2][kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long run = 0;
  for (long long j = a; j < b; ++j) {
    const long long base = (tile0 + j) * kTile;
    int c = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const long long i = base + r * kBlock + tid;
      if (i < n) c += inside(__ldcg(p.z + i), __ldcg(p.x + i), p.ez, p.ex) ? 1 : 0;
    }
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) s_w[j & 1][warp] = c;
    __syncthreads();   // (double-buffered s_w: one barrier per tile)
    int tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += s_w[j & 1][w];
    if (tid == 0) tile_cnt[j] = run;
    run += (unsigned long long)tot;
  }
  if (tid == 0) cta_tot[blockIdx.x] = run;
}

// One CTA: exclusive scan of the CTA range totals (in place, <= kScanT
// entries) plus tile0's slot, and the grand total in cta_tot[G].
constexpr int kScanT = 1024;
__global__ void __launch_bounds__(kScanT) compact_scan_kernel(const DevState* st,
                                                               unsigned long long* cta_tot,
                                                               int g) {
  long long n, tile0;
  if (!compact_range(st, &n, &tile0)) return;
  __shared__ unsigned long long s_ws[kScanT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long v = threadIdx.x < g ? cta_tot[threadIdx.x] : 0ull;
  unsigned long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long wv = s_ws[lane];
    unsigned long long w = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    s_ws[lane] = w - wv;
  }
  __syncthreads();
  const unsigned long long excl = s_ws[warp] + inc - v;
  if (threadIdx.x < g) cta_tot[threadIdx.x] = (unsigned long long)(tile0 * kTile) + excl;
  if (threadIdx.x == g - 1) cta_tot[g] = (unsigned long long)(tile0 * kTile) + excl + v;  // survivors
}

// 512 threads x 4 rows per tile: ~64 registers, 2 CTAs = 32 warps per SM
// (256 x 8 at 128 registers left 16 warps, mostly parked at the barriers).
constexpr int kMB = 512, kMW = kMB / 32, kMI = kTile / kMB;
template <int kKick>   // extra arrays moved along: 0, 1 (kvz) or 2 (kvz, kvx)
__global__ void __launch_bounds__(kMB, 2) compact_move_kernel(ScanParams p,
                                                                 const unsigned long long* tile_cnt,
                                                                 const unsigned long long* cta_base,
                                                                 int g) {
  __shared__ long long s_tile;
  __shared__ int s_last;
  __shared__ int s_off[kMI * kMW];
  long long n, tile0;
  if (!compact_range(p.st, &n, &tile0)) return;
  const unsigned epoch = *((volatile unsigned*)&p.st->epoch);
  const long long ntiles = (n + kTile - 1) / kTile;
  const long long per = (ntiles - tile0 + g - 1) / g;   // compact_count_kernel's ranges
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = lanemask_lt();
  while (true) {
    if (tid == 0) s_tile = tile0 + (long long)atomicAdd(&p.st->ticket, 1ull);
    __syncthreads();
    const long long t = s_tile;
    if (t >= ntiles) break;
    const long long base = t * kTile;
    double z[kMI], x[kMI], vz[kMI], vx[kMI], kz[kKick ? kMI : 1], kx[kKick > 1 ? kMI : 1];
    bool keep[kMI];
    unsigned long long dep = 0;
#pragma unroll
    for (int r = 0; r < kMI; ++r) {
      const long long i = base + r * kMB + tid;
      z[r] = -1.0;
      x[r] = -1.0;
      vz[r] = vx[r] = 0.0;
      if (kKick) kz[r] = 0.0;
      if (kKick > 1) kx[r] = 0.0;
      if (i < n) {
        z[r] = __ldcs(p.z + i);
        x[r] = __ldcs(p.x + i);
        vz[r] = __ldcs(p.vz + i);
        vx[r] = __ldcs(p.vx + i);
        if (kKick) kz[r] = __ldcs(p.kvz + i);
        if (kKick > 1) kx[r] = __ldcs(p.kvx + i);
      }
      keep[r] = inside(z[r], x[r], p.ez, p.ex);
      dep ^= (unsigned long long)__double_as_longlong(vz[r]) ^
             (unsigned long long)__double_as_longlong(vx[r]);
      if (kKick) dep ^= (unsigned long long)__double_as_longlong(kz[r]);
      if (kKick > 1) dep ^= (unsigned long long)__double_as_longlong(kx[r]);
      const unsigned b = __ballot_sync(kFull, keep[r]);
      if (lane == 0) s_off[r * kMW + warp] = __popc(b);
    }
    // every load of this tile has landed (the barrier's predicate consumes
    // them all): publish "loaded" so later tiles may overwrite this input
    const int any = __syncthreads_or((int)(dep == 0x9e3779b97f4a7c15ull));
    if (tid == 0) {
      __threadfence();
      st_release(p.status + t, pack_status(epoch, kFlagAgg, (unsigned long long)(any & 1)));
    }
    const long long out = (long long)(cta_base[(t - tile0) / per] + tile_cnt[t - tile0]);
    if (warp == 0) {
      // exclusive offsets of the (row, warp) survivor groups, row-major
      constexpr int kPer = kMI * kMW / 32;
      int v[kPer], sum = 0;
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        v[e] = s_off[lane * kPer + e];
        sum += v[e];
      }
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      int off = inc - sum;
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        s_off[lane * kPer + e] = off;
        off += v[e];
      }
      // wait until every earlier tile whose input this tile's output covers
      // has loaded (tiles before tile0 are never rewritten)
      const long long first = max(tile0, out / kTile);
      for (long long w0 = first; w0 < t; w0 += 32) {
        const long long w = w0 + lane;
        if (w < t) {
          unsigned long long s;
          do {
            s = ld_acquire(p.status + w);
          } while ((unsigned)(s >> kEpochShift) != epoch);
        }
      }
      __syncwarp();
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMI; ++r) {
      const unsigned b = __ballot_sync(kFull, keep[r]);
      if (keep[r]) {
        const long long d = out + s_off[r * kMW + warp] + __popc(b & lt);
        if (d != base + r * kMB + tid) {   // in place where nothing moved
          __stcs(p.z + d, z[r]);
          __stcs(p.x + d, x[r]);
          __stcs(p.vz + d, vz[r]);
          __stcs(p.vx + d, vx[r]);
          if (kKick) __stcs(p.kvz + d, kz[r]);
          if (kKick > 1) __stcs(p.kvx + d, kx[r]);
        }
      }
    }
    __syncthreads();   // s_off / s_tile reuse
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last || tid != 0) return;
  __threadfence();
  // invariant: the tiles' survivors add up to the push's count
  const long long n_new = (long long)cta_base[g];
  p.st->leavers = 0ull;
  p.st->first_leaver = LLONG_MAX;
  if (*((volatile long long*)&p.st->n) != n_new) p.st->err += 1ll << 40;
  p.st->ticket = 0ull;
  p.st->done = 0u;
  const unsigned ne = (epoch + 1u) & kEpochMask;
  p.st->epoch = ne ? ne : 1u;
  __threadfence();
}

// ---------------------------------------------------------------------------
// drop-in bin_particles, heuristic cost, state init
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kBlock) bin_kernel(const double2* __restrict__ pos,
                                                     long long n, double m, int nbz, int nbx,
                                                     int smem_hist,
                                                     unsigned long long* __restrict__ counts,
                                                     unsigned long long* __restrict__ err,
                                                     const long long* __restrict__ n_dev) {
  if (n_dev) n = *n_dev;  // count produced by a preceding kernel on the stream
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* s_cnt = reinterpret_cast<unsigned*>(smem_raw);
  const int nb = nbz * nbx;
  if (smem_hist) {
    for (int b = threadIdx.x; b < nb; b += kBlock) s_cnt[b] = 0u;
    __syncthreads();
  }
  long long bad = 0;
  const long long stride = (long long)gridDim.x * kBlock;
  int cur = -1;
  unsigned run = 0;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride) {
    const double2 q = __ldcs(pos + i);
    const double fz = __ddiv_rn(q.x, m);
    const double fx = __ddiv_rn(q.y, m);
    int b = -1;
    if (fz >= 0.0 && fx >= 0.0 && fz < (double)nbz && fx < (double)nbx) {
      b = (int)fz * nbx + (int)fx;
    } else {
      ++bad;
    }
    if (b != cur) {
      if (cur >= 0) {
        if (smem_hist) atomicAdd(s_cnt + cur, run);
        else atomicAdd(counts + cur, (unsigned long long)run);
      }
      cur = b;
      run = 0;
    }
    run += (b >= 0) ? 1u : 0u;
  }
  if (cur >= 0 && run) {
    if (smem_hist) atomicAdd(s_cnt + cur, run);
    else atomicAdd(counts + cur, (unsigned long long)run);
  }
  if (bad && err) atomicAdd(err, (unsigned long long)bad);
  if (smem_hist) {
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kBlock) {
      const unsigned c = s_cnt[b];
      if (c) atomicAdd(counts + b, (unsigned long long)c);
    }
  }
}

__global__ void heuristic_kernel(const double* __restrict__ particles,
                                 const double* __restrict__ cells, long long n, double wp,
                                 double wc, double* __restrict__ cost) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) cost[b] = __dadd_rn(__dmul_rn(wp, particles[b]), __dmul_rn(wc, cells[b]));
}

// ---- Timers strategy (per-box launches) ----
// Box sort of particle indices.  Particles are spatially coherent, so most
// warps sit in one box: counts use a shared histogram with warp-aggregated
// updates (__match_any_sync), and the scatter reserves each box's range once
// per CTA chunk, then hands out slots with shared-memory atomics.
constexpr int kSortChunk = kBlock * 16;

__device__ __forceinline__ int box_of(double z, double x, double m, int nbz, int nbx) {
  int bz = (int)__ddiv_rn(z, m), bx = (int)__ddiv_rn(x, m);
  bz = min(max(bz, 0), nbz - 1);  // live particles are in the domain
  bx = min(max(bx, 0), nbx - 1);
  return bz * nbx + bx;
}

__global__ void __launch_bounds__(kBlock) timers_box_kernel(
    const double* __restrict__ z, const double* __restrict__ x, long long n, double m, int nbz,
    int nbx, int* __restrict__ box, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned s_hist[];
  const int nb = nbz * nbx;
  for (int b = threadIdx.x; b < nb; b += kBlock) s_hist[b] = 0u;
  __syncthreads();
  const long long stride = (long long)gridDim.x * kBlock;
  const long long n_up = (n + kBlock - 1) / kBlock * kBlock;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n_up; i += stride) {
    const bool ok = i < n;
    const int b = ok ? box_of(z[i], x[i], m, nbz, nbx) : -1;
    if (ok) box[i] = b;
    const unsigned grp = __match_any_sync(kFull, b);
    if (ok && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(s_hist + b, (unsigned)__popc(grp));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kBlock)
    if (s_hist[b]) atomicAdd(counts + b, (unsigned long long)s_hist[b]);
}

__global__ void __launch_bounds__(kBlock) timers_scatter_kernel(
    const int* __restrict__ box, long long n, int nb, unsigned long long* cursors,
    int* __restrict__ perm) {
  extern __shared__ unsigned long long s_base[];
  const int lane = threadIdx.x & 31;
  for (long long c0 = (long long)blockIdx.x * kSortChunk; c0 < n;
       c0 += (long long)gridDim.x * kSortChunk) {
    for (int b = threadIdx.x; b < nb; b += kBlock) s_base[b] = 0ull;
    __syncthreads();
    const long long c1 = min(n, c0 + kSortChunk);
    for (long long i = c0 + threadIdx.x; i < c0 + kSortChunk; i += kBlock) {
      const int b = i < c1 ? box[i] : -1;
      const unsigned grp = __match_any_sync(kFull, b);
      if (b >= 0 && lane == __ffs(grp) - 1) atomicAdd(s_base + b, (unsigned long long)__popc(grp));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kBlock) {
      const unsigned long long c = s_base[b];
      if (c) s_base[b] = atomicAdd(cursors + b, c);  // reserve this chunk's range
    }
    __syncthreads();
    for (long long i = c0 + threadIdx.x; i < c0 + kSortChunk; i += kBlock) {
      const int b = i < c1 ? box[i] : -1;
      const unsigned grp = __match_any_sync(kFull, b);
      const int leader = __ffs(grp) - 1;
      unsigned long long base = 0;
      if (b >= 0 && lane == leader) base = atomicAdd(s_base + b, (unsigned long long)__popc(grp));
      base = __shfl_sync(kFull, base, leader);
      if (b >= 0) perm[base + __popc(grp & lanemask_lt())] = (int)i;
    }
    __syncthreads();
  }
}

// Push the particles of one box (gather by index); absorbed ones are left
// out of the domain for the compaction pass.
__global__ void timers_push_kernel(double* z, double* x, const double* __restrict__ vz,
                                   const double* __restrict__ vx, const int* __restrict__ idx,
                                   long long cnt) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride) {
    const int i = idx[j];
    z[i] = __dadd_rn(z[i], vz[i]);
    x[i] = __dadd_rn(x[i], vx[i]);
  }
}

// Unstable O(removed) compaction (multi-GPU path): holes below n_new are
// filled with the survivors found in the tail [n_new, n_new + L).
__global__ void fill_mark_kernel(const long long* __restrict__ removed, long long L,
                                 long long n_new, long long* holes, long long* tail_flag,
                                 DevState* st) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < L; k += stride) {
    const long long r = removed[k];
    if (r >= n_new) tail_flag[r - n_new] = 1;
    else holes[atomicAdd(&st->holes, 1ull)] = r;
  }
}

__global__ void fill_move_kernel(long long L, long long n_new, const long long* __restrict__ holes,
                                 long long* tail_flag, DevState* st, double* z, double* x,
                                 double* vz, double* vx, double* kvz, double* kvx) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < L; j += stride) {
    if (tail_flag[j]) {
      tail_flag[j] = 0;
      continue;
    }
    const long long src = n_new + j;
    const long long dst = holes[atomicAdd(&st->movers, 1ull)];
    z[dst] = z[src];
    x[dst] = x[src];
    vz[dst] = vz[src];
    vx[dst] = vx[src];
    if (kvz) {
      kvz[dst] = kvz[src];
      kvx[dst] = kvx[src];
    }
  }
}

__global__ void fill_done_kernel(DevState* st, long long n_new) {
  st->n = n_new;
  st->n_old = n_new;
  st->holes = 0ull;
  st->movers = 0ull;
  st->removed_count = 0ull;
  st->leavers = 0ull;
  st->first_leaver = LLONG_MAX;
}

// Device-count variants (pipelined multi-GPU loop: no host round trip).
// The push epilogue left st->n = survivors kept in place and st->removed_count
// = L listed removals; a tail slot in [n, n + L) is removed iff its position
// is outside the domain (absorbed) or carries the emigrant sentinel z = -1.
__global__ void fill_dev_mark_kernel(DevState* st, const long long* __restrict__ removed,
                                     long long cap, long long* holes) {
  const long long L = min((long long)st->removed_count, cap), n_new = st->n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < L;
       k += (long long)gridDim.x * blockDim.x) {
    const long long r = removed[k];
    if (r < n_new) holes[atomicAdd(&st->holes, 1ull)] = r;
  }
}

__global__ void fill_dev_move_kernel(DevState* st, long long cap, const long long* __restrict__ holes,
                                     double ez, double ex, double* z, double* x, double* vz,
                                     double* vx, double* kvz, double* kvx) {
  const long long L = min((long long)st->removed_count, cap), n_new = st->n;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < L;
       j += (long long)gridDim.x * blockDim.x) {
    const long long src = n_new + j;
    if (!inside(z[src], x[src], ez, ex)) continue;   // removed tail slot
    const long long dst = holes[atomicAdd(&st->movers, 1ull)];
    z[dst] = z[src];
    x[dst] = x[src];
    vz[dst] = vz[src];
    vx[dst] = vx[src];
    if (kvz) {
      kvz[dst] = kvz[src];
      kvx[dst] = kvx[src];
    }
  }
}

__global__ void fill_dev_done_kernel(DevState* st, long long cap) {
  if ((long long)st->removed_count > cap) st->err |= 1ll << 61;   // list overflowed
  st->n_old = st->n;
  st->holes = 0ull;
  st->movers = 0ull;
  st->removed_count = 0ull;
  st->leavers = 0ull;
  st->first_leaver = LLONG_MAX;
}

// Append the records peers wrote into this rank's receive buffer; the count
// is the rank's own cursor (device), the offset the device live count.
__global__ void unpack_dev_kernel(const double* __restrict__ recv,
                                  const unsigned long long* cursor, const DevState* st,
                                  long long capacity, double* z, double* x, double* vz,
                                  double* vx, double* kvz, double* kvx) {
  const long long off = st->n;
  const long long m = min((long long)*cursor, capacity - off);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const double2* r = reinterpret_cast<const double2*>(recv + i * 6);
    const double2 a = r[0], b = r[1], c = r[2];
    z[off + i] = a.x;
    x[off + i] = a.y;
    vz[off + i] = b.x;
    vx[off + i] = b.y;
    if (kvz) {
      kvz[off + i] = c.x;
      kvx[off + i] = c.y;
    }
  }
}

__global__ void unpack_dev_done_kernel(DevState* st, unsigned long long* cursor,
                                       long long capacity) {
  const long long m = (long long)*cursor;
  long long n = st->n + m;
  if (n > capacity) {
    st->err |= 1ll << 60;   // more immigrants than capacity
    n = capacity;
  }
  st->n = n;
  st->n_old = n;
  *cursor = 0ull;
}

__global__ void counts_cost_kernel(const long long* __restrict__ counts, int nb, double wp,
                                   double wc, double cells, double* __restrict__ cost) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) cost[b] = __dadd_rn(__dmul_rn(wp, (double)counts[b]), __dmul_rn(wc, cells));
}

__global__ void init_state_kernel(DevState* st, long long n) {
  st->ticket = 0ull;
  st->done = 0u;
  if (st->epoch == 0u) st->epoch = 1u;
  st->n = n;
  st->n_old = n;
  st->leavers = 0ull;
  st->first_leaver = LLONG_MAX;
  st->staged = 0ull;
  st->removed_count = 0ull;
  st->holes = 0ull;
  st->movers = 0ull;
}

__global__ void group_kernel(const double* __restrict__ stage, const int* __restrict__ dest,
                             long long count, unsigned long long* cursors,
                             double* __restrict__ send) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const long long slot = (long long)atomicAdd(cursors + dest[i], 1ull);
#pragma unroll
    for (int j = 0; j < 6; ++j) send[slot * 6 + j] = stage[i * 6 + j];
  }
}

__global__ void unpack_kernel(const double* __restrict__ recv, long long n_recv, long long off,
                              double* z, double* x, double* vz, double* vx, double* kvz,
                              double* kvx) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_recv; i += stride) {
    const double* r = recv + i * 6;
    z[off + i] = r[0];
    x[off + i] = r[1];
    vz[off + i] = r[2];
    vx[off + i] = r[3];
    if (kvz) {
      kvz[off + i] = r[4];
      kvx[off + i] = r[5];
    }
  }
}

inline int cuda_fail(cudaError_t e, const char* what) {
  return set_error(LBX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

template <typename K>
int occupancy_grid(lbx_ctx* ctx, K kern, size_t smem, long long work_ctas, int* grid_out) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
  long long grid = (long long)std::max(per_sm, 1) * ctx->num_sms;
  if (ctx->grid_override > 0) grid = ctx->grid_override;
  *grid_out = (int)std::max(1ll, std::min(grid, work_ctas));
  return LBX_OK;
}

template <bool kClock, bool kPow2, bool kExch, bool kPush>
int launch_stream(lbx_ctx* ctx, const StepParams& p, cudaStream_t s) {
  auto kern = stream_kernel<kClock, kPow2, kExch, kPush>;
  const size_t smem = p.smem_hist ? (size_t)p.nb * 4 * (1 + (kClock ? 1 : 0) + (kExch ? 1 : 0)) : 0;
  // per launch (a cheap host call): the attribute is per device context, and
  // thread-ranks / several devices share this function
  if (smem > 48 * 1024) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  }
  int grid = 0;
  const long long work = (ctx->n_upper + 2ll * kBlock * kPairs - 1) / (2ll * kBlock * kPairs);
  int rc = occupancy_grid(ctx, kern, smem, std::max(1ll, work), &grid);
  if (rc) return rc;
  StepParams pk = p;
  // particle state (read 32 B + write 16 B per particle; 2x for the kick
  // buffers) well inside L2: keep it resident across steps
  pk.l2_keep = ctx->n_upper * 48ll < (long long)ctx->l2_bytes / 2 ? 1 : 0;
  if (ctx->timing) cudaEventRecord((cudaEvent_t)ctx->ev0, s);
  kern<<<grid, kBlock, smem, s>>>(pk);
  if (ctx->timing) cudaEventRecord((cudaEvent_t)ctx->ev1, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "stream_kernel launch");
  return LBX_OK;
}

template <bool kExch, bool kPush>
int launch_stream_any(lbx_ctx* ctx, const StepParams& p, bool clock, bool pow2, cudaStream_t s) {
  if (clock) {
    return pow2 ? launch_stream<true, true, kExch, kPush>(ctx, p, s)
                : launch_stream<true, false, kExch, kPush>(ctx, p, s);
  }
  return pow2 ? launch_stream<false, true, kExch, kPush>(ctx, p, s)
              : launch_stream<false, false, kExch, kPush>(ctx, p, s);
}

#ifndef LBX_COMPACT_LOOKBACK
#define LBX_COMPACT_LOOKBACK 0   // 1: the single-pass look-back compaction (A/B)
#endif
// count -> scan -> move (each kernel exits at once when nothing was absorbed)
int launch_compact3(lbx_ctx* ctx, const ScanParams& p, cudaStream_t s) {
  unsigned long long* tiles = ctx->status + ctx->status_tiles;
  const long long ntiles = std::max(1ll, (long long)((ctx->n_upper + kTile - 1) / kTile));
  // count CTAs: <= kScanT - 1 ranges (one scan CTA), a few per SM
  const int cg = (int)std::max(1ll, std::min({(long long)ctx->num_sms * 4, ntiles,
                                              (long long)kScanT - 1}));
  unsigned long long* cta = tiles + ctx->status_tiles;   // [cg + 1]
  compact_count_kernel<<<cg, kBlock, 0, s>>>(p, tiles, cta);
  compact_scan_kernel<<<1, kScanT, 0, s>>>(p.st, cta, cg);
  if (!p.kvz && p.kvx) return set_error(LBX_EINVAL, "compaction: kvx without kvz");
  auto kern = p.kvx ? compact_move_kernel<2> : (p.kvz ? compact_move_kernel<1> : compact_move_kernel<0>);
  int per_sm = 0;
  cudaError_t e0 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMB, 0);
  if (e0 != cudaSuccess) return cuda_fail(e0, "occupancy query");
  long long grid = (long long)std::max(per_sm, 1) * ctx->num_sms;
  if (ctx->grid_override > 0) grid = ctx->grid_override;
  grid = std::max(1ll, std::min(grid, ntiles));
  kern<<<(unsigned)grid, kMB, 0, s>>>(p, tiles, cta, cg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "compaction launch");
  return LBX_OK;
}

template <int kMode>
int launch_scan(lbx_ctx* ctx, const ScanParams& p, long long n_upper, cudaStream_t s) {
  auto kern = scan_kernel<kMode>;
  int grid = 0;
  int rc = occupancy_grid(ctx, kern, 0, std::max(1ll, (n_upper + kTile - 1) / kTile), &grid);
  if (rc) return rc;
  kern<<<grid, kBlock, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "scan_kernel launch");
  return LBX_OK;
}

}  // namespace

int reserve_status(lbx_ctx* ctx, int64_t capacity) {
  const int64_t tiles = (capacity + kTile - 1) / kTile + 1;
  if (tiles <= ctx->status_tiles) return LBX_OK;
  unsigned long long* s = nullptr;
  // [tiles] status words, [tiles] compaction tile prefixes, [kScanT] range totals
  const size_t words = (size_t)tiles * 2 + 1024;
  cudaError_t e = cudaMalloc(&s, words * sizeof(unsigned long long));
  if (e != cudaSuccess)
    return set_error(LBX_EOOM, "look-back workspace: %s", cudaGetErrorString(e));
  // Epoch 0 is never current, so zeroed words read as "not yet published".
  e = cudaMemset(s, 0, words * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    cudaFree(s);
    return cuda_fail(e, "cudaMemset");
  }
  if (ctx->status) {
    cudaDeviceSynchronize();
    cudaFree(ctx->status);
  }
  ctx->status = s;
  ctx->status_tiles = tiles;
  return LBX_OK;
}

namespace {

}  // namespace

// Host-buffer pipeline state (lbx_advance_bin_host), cached in ctx: kLanes
// streams, each with its own device chunk buffers and look-back state.
struct HostPipe {
#ifndef LBX_HOST_CHUNK_LOG2
#define LBX_HOST_CHUNK_LOG2 22
#endif
  static constexpr long long kChunk = 1ll << LBX_HOST_CHUNK_LOG2;  // 4 Mi particles per chunk
  static constexpr int kLanes = 3;
  cudaStream_t s[kLanes] = {};
  cudaEvent_t ready = {};
  DevState* st[kLanes] = {};
  unsigned long long* status[kLanes] = {};
  double *d_in_pos[kLanes] = {}, *d_in_vel[kLanes] = {}, *d_out_pos[kLanes] = {},
         *d_out_vel[kLanes] = {};
  long long* d_m[kLanes] = {};
  long long* h_m = nullptr;  // pinned [h_m_cap]: survivors per chunk (+1: error count)
  long long h_m_cap = 0;
  long long* d_counts = nullptr;
  double* d_cost = nullptr;
  long long* d_err = nullptr;
  long long nb = 0;
};

void destroy_pipe(HostPipe* hp) {
  if (!hp) return;
  for (int l = 0; l < HostPipe::kLanes; ++l) {
    if (hp->s[l]) cudaStreamSynchronize(hp->s[l]), cudaStreamDestroy(hp->s[l]);
    cudaFree(hp->st[l]);
    cudaFree(hp->status[l]);
    cudaFree(hp->d_in_pos[l]);
    cudaFree(hp->d_in_vel[l]);
    cudaFree(hp->d_out_pos[l]);
    cudaFree(hp->d_out_vel[l]);
    cudaFree(hp->d_m[l]);
  }
  if (hp->ready) cudaEventDestroy(hp->ready);
  cudaFreeHost(hp->h_m);
  cudaFree(hp->d_counts);
  cudaFree(hp->d_cost);
  cudaFree(hp->d_err);
  delete hp;
}

namespace {

int ensure_pipe(lbx_ctx* ctx, long long nb, long long nchunks) {
  if (ctx->pipe && ctx->pipe->nb >= nb) {
    HostPipe* hp = ctx->pipe;
    if (hp->h_m_cap < nchunks + 1) {
      cudaFreeHost(hp->h_m);
      hp->h_m = nullptr;
      hp->h_m_cap = 0;
      if (cudaHostAlloc(&hp->h_m, (size_t)(nchunks + 1) * 8, cudaHostAllocDefault) != cudaSuccess)
        return set_error(LBX_EOOM, "host pipeline counters");
      hp->h_m_cap = nchunks + 1;
    }
    return LBX_OK;
  }
  if (ctx->pipe) {
    destroy_pipe(ctx->pipe);
    ctx->pipe = nullptr;
  }
  HostPipe* hp = new HostPipe();
  const long long C = HostPipe::kChunk;
  const size_t tiles = (size_t)((C + kTile - 1) / kTile + 1);
  bool ok = cudaHostAlloc(&hp->h_m, (size_t)(nchunks + 1) * 8, cudaHostAllocDefault) == cudaSuccess;
  hp->h_m_cap = nchunks + 1;
  for (int l = 0; l < HostPipe::kLanes && ok; ++l) {
    ok = cudaStreamCreateWithFlags(&hp->s[l], cudaStreamNonBlocking) == cudaSuccess &&
         cudaMalloc(&hp->st[l], sizeof(DevState)) == cudaSuccess &&
         cudaMalloc(&hp->status[l], tiles * 8) == cudaSuccess &&
         cudaMalloc(&hp->d_in_pos[l], (size_t)C * 16) == cudaSuccess &&
         cudaMalloc(&hp->d_in_vel[l], (size_t)C * 16) == cudaSuccess &&
         cudaMalloc(&hp->d_out_pos[l], (size_t)C * 16) == cudaSuccess &&
         cudaMalloc(&hp->d_out_vel[l], (size_t)C * 16) == cudaSuccess &&
         cudaMalloc(&hp->d_m[l], 8) == cudaSuccess;
    if (ok) {
      cudaMemset(hp->status[l], 0, tiles * 8);
      cudaMemset(hp->st[l], 0, sizeof(DevState));
      init_state_kernel<<<1, 1>>>(hp->st[l], 0);
    }
  }
  ok = ok && cudaEventCreateWithFlags(&hp->ready, cudaEventDisableTiming) == cudaSuccess &&
       cudaMalloc(&hp->d_counts, (size_t)std::max(nb, 1ll) * 8) == cudaSuccess &&
       cudaMalloc(&hp->d_cost, (size_t)std::max(nb, 1ll) * 8) == cudaSuccess &&
       cudaMalloc(&hp->d_err, 8) == cudaSuccess;
  if (ok) ok = cudaMemset(hp->d_err, 0, 8) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  if (!ok) {
    destroy_pipe(hp);
    return set_error(LBX_EOOM, "host pipeline buffers: %s", cudaGetErrorString(cudaGetLastError()));
  }
  hp->nb = nb;
  ctx->pipe = hp;
  return LBX_OK;
}

bool is_pow2(double m) {
  int e = 0;
  const double f = std::frexp(m, &e);
  return f == 0.5;
}

}  // namespace

int launch_compact(lbx_ctx* ctx, double* z, double* x, double* a, double* b, double* c,
                   double* d, double ez, double ex, void* stream) {
  int rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  ScanParams p{};
  p.z = z;
  p.x = x;
  p.vz = a;
  p.vx = b;
  p.kvz = c;
  p.kvx = d;
  p.ez = ez;
  p.ex = ex;
  p.st = ctx->st;
  p.status = ctx->status;
#if LBX_COMPACT_LOOKBACK
  return launch_scan<kCompactSoA>(ctx, p, ctx->n_upper, (cudaStream_t)stream);
#else
  return launch_compact3(ctx, p, (cudaStream_t)stream);
#endif
}

int launch_timers_sort(const double* z, const double* x, long long n, double m, int nbz, int nbx,
                       int* box, unsigned long long* counts, unsigned long long* cursors,
                       int* perm, const unsigned long long* offsets_host, void* stream,
                       int phase) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = nbz * nbx;
  if (nb > kSmemBoxesMax / 2) return set_error(LBX_EINVAL, "Timers strategy supports <= %d boxes",
                                               kSmemBoxesMax / 2);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (phase == 0) {
    cudaMemsetAsync(counts, 0, (size_t)nb * 8, s);
    const size_t smem = (size_t)nb * 4;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(timers_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)std::max(1ll, std::min((long long)sms * 4, (n + kBlock - 1) / kBlock));
    if (n) timers_box_kernel<<<grid, kBlock, smem, s>>>(z, x, n, m, nbz, nbx, box, counts);
  } else {
    cudaMemcpyAsync(cursors, offsets_host, (size_t)nb * 8, cudaMemcpyHostToDevice, s);
    const size_t smem = (size_t)nb * 8;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(timers_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    const unsigned grid =
        (unsigned)std::max(1ll, std::min((long long)sms * 4, (n + kSortChunk - 1) / kSortChunk));
    if (n) timers_scatter_kernel<<<grid, kBlock, smem, s>>>(box, n, nb, cursors, perm);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "timers sort launch");
  return LBX_OK;
}

int launch_timers_push(double* z, double* x, const double* vz, const double* vx, const int* idx,
                       long long cnt, void* stream) {
  const unsigned grid = (unsigned)std::max(1ll, std::min(1184ll, (cnt + 255) / 256));
  timers_push_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(z, x, vz, vx, idx, cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "timers push launch");
  return LBX_OK;
}

int ensure_accumulators(lbx_ctx* ctx, int32_t nboxes) {
  if (nboxes <= ctx->acc_boxes) return LBX_OK;
  unsigned long long* a = nullptr;
  cudaError_t e = cudaMalloc(&a, (size_t)2 * nboxes * sizeof(unsigned long long));
  if (e != cudaSuccess) return set_error(LBX_EOOM, "accumulators: %s", cudaGetErrorString(e));
  e = cudaMemset(a, 0, (size_t)2 * nboxes * sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemset");
  if (ctx->acc) {
    cudaDeviceSynchronize();
    cudaFree(ctx->acc);
  }
  ctx->acc = a;
  ctx->acc_boxes = nboxes;
  return LBX_OK;
}

int launch_push_step(lbx_ctx* ctx, const StepLaunch& a, void* stream,
                     const lbx_exchange_args* ex, bool push) {
  if (a.nbz < 1 || a.nbx < 1) return set_error(LBX_EINVAL, "box grid must be at least 1x1");
  if (!(a.m > 0.0)) return set_error(LBX_EINVAL, "box_size must be positive");
  const long long nb = (long long)a.nbz * a.nbx;
  if (nb > (1ll << 30)) return set_error(LBX_EINVAL, "too many boxes");
  if (((uintptr_t)a.z | (uintptr_t)a.x | (uintptr_t)a.vz | (uintptr_t)a.vx) & 15u)
    return set_error(LBX_EINVAL, "particle arrays must be 16-byte aligned");
  int rc = ensure_accumulators(ctx, (int32_t)nb);
  if (rc) return rc;
  rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  StepParams p{};
  p.z = a.z;
  p.x = a.x;
  p.vz = a.vz;
  p.vx = a.vx;
  p.ez = a.ez;
  p.ex = a.ex;
  p.m = a.m;
  p.inv_m = 1.0 / a.m;
  p.nbz = a.nbz;
  p.nbx = a.nbx;
  p.nb = (int)nb;
  p.smem_hist = nb <= kSmemBoxesMax ? 1 : 0;
  p.st = ctx->st;
  p.g_cnt = ctx->acc;
  p.g_clk = ctx->acc + ctx->acc_boxes;
  p.counts_out = a.counts_out;
  p.cost_out = a.cost_out;
  p.clk_out = a.clk_out;
  p.n_out = a.n_out;
  p.err_out = a.err_out;
  p.wp = a.wp;
  p.wc = a.wc;
  p.cells = a.cells;
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = is_pow2(a.m);
  if (ex) {
    p.owner = ex->owner;
    p.me = ex->rank;
    p.stage = ex->stage;
    p.stage_dest = ex->stage_dest;
    p.stage_cap = ex->stage_cap;
    p.send_counts = reinterpret_cast<long long*>(ex->send_counts);
    p.kvz = ex->kick_vz;
    p.kvx = ex->kick_vx;
    p.removed_list = reinterpret_cast<long long*>(ex->removed_list);
    p.removed_cap = ex->removed_cap;
    p.peer_recv = ex->peer_recv;
    p.peer_cursor = ex->peer_cursor;
    p.peer_cap = ex->peer_recv_cap;
    rc = push ? launch_stream_any<true, true>(ctx, p, a.clock, pow2, s)
              : launch_stream_any<true, false>(ctx, p, false, pow2, s);
    if (rc) return rc;
    if (ex->removed_list) return LBX_OK;  // caller compacts with lbx_fill_holes
  } else {
    rc = launch_stream_any<false, true>(ctx, p, a.clock, pow2, s);
  }
  if (rc) return rc;
  // Stable compaction of the survivors; returns at once when none was removed.
  ScanParams c{};
  c.z = a.z;
  c.x = a.x;
  c.vz = const_cast<double*>(a.vz);
  c.vx = const_cast<double*>(a.vx);
  c.kvz = ex ? ex->kick_vz : nullptr;
  c.kvx = ex ? ex->kick_vx : nullptr;
  c.ez = a.ez;
  c.ex = a.ex;
  c.st = ctx->st;
  c.status = ctx->status;
#if LBX_COMPACT_LOOKBACK
  return launch_scan<kCompactSoA>(ctx, c, ctx->n_upper, s);
#else
  return launch_compact3(ctx, c, s);
#endif
}

}  // namespace lbx

using namespace lbx;

extern "C" {

int lbx_ctx_create(lbx_ctx** out, int device, int64_t capacity) {
  clear_error();
  if (!out) return set_error(LBX_EINVAL, "out pointer is NULL");
  if (capacity < 0) return set_error(LBX_EINVAL, "capacity must be >= 0");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  lbx_ctx* c = new lbx_ctx();
  c->device = device;
  e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "device query");
  }
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device) == cudaSuccess) c->l2_bytes = l2;
  e = cudaMalloc(&c->st, sizeof(DevState));
  if (e != cudaSuccess) {
    delete c;
    return set_error(LBX_EOOM, "device state: %s", cudaGetErrorString(e));
  }
  cudaMemset(c->st, 0, sizeof(DevState));
  e = cudaHostAlloc(&c->host_scratch, 64, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaFree(c->st);
    delete c;
    return cuda_fail(e, "cudaHostAlloc");
  }
  init_state_kernel<<<1, 1>>>(c->st, 0);
  int rc = reserve_status(c, capacity);
  if (rc) {
    lbx_ctx_destroy(c);
    return rc;
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    lbx_ctx_destroy(c);
    return cuda_fail(e, "context init");
  }
  *out = c;
  return LBX_OK;
}

int lbx_ctx_destroy(lbx_ctx* ctx) {
  clear_error();
  if (!ctx) return LBX_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->st) cudaFree(ctx->st);
  if (ctx->status) cudaFree(ctx->status);
  if (ctx->acc) cudaFree(ctx->acc);
  if (ctx->host_scratch) cudaFreeHost(ctx->host_scratch);
  destroy_pipe(ctx->pipe);
  if (ctx->pic_acc) cudaFree(ctx->pic_acc);
  if (ctx->pic_quad) cudaFree(ctx->pic_quad);
  if (ctx->pic_sortbuf) cudaFree(ctx->pic_sortbuf);
  if (ctx->pic_fill) cudaFree(ctx->pic_fill);
  if (ctx->pic_tiles) cudaFree(ctx->pic_tiles);
  if (ctx->pic_jn) cudaFree(ctx->pic_jn);
  if (ctx->pic_esk) cudaFree(ctx->pic_esk);
  if (ctx->fill_scratch) cudaFree(ctx->fill_scratch);
  if (ctx->ev0) cudaEventDestroy((cudaEvent_t)ctx->ev0), cudaEventDestroy((cudaEvent_t)ctx->ev1);
  delete ctx;
  return LBX_OK;
}

int lbx_ctx_reserve(lbx_ctx* ctx, int64_t capacity) {
  clear_error();
  if (!ctx) return set_error(LBX_EINVAL, "context is NULL");
  return reserve_status(ctx, capacity);
}

int lbx_ctx_set_count(lbx_ctx* ctx, int64_t n, void* stream) {
  clear_error();
  if (!ctx) return set_error(LBX_EINVAL, "context is NULL");
  if (n < 0) return set_error(LBX_EINVAL, "count must be >= 0");
  int rc = reserve_status(ctx, n);
  if (rc) return rc;
  init_state_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(ctx->st, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "set_count");
  ctx->n_upper = n;
  return LBX_OK;
}

int lbx_ctx_set_upper(lbx_ctx* ctx, int64_t n_upper) {
  clear_error();
  if (!ctx || n_upper < 0) return set_error(LBX_EINVAL, "bad argument");
  int rc = reserve_status(ctx, n_upper);
  if (rc) return rc;
  ctx->n_upper = n_upper;
  return LBX_OK;
}

int lbx_ctx_get_count(lbx_ctx* ctx, int64_t* n_host, void* stream) {
  clear_error();
  if (!ctx || !n_host) return set_error(LBX_EINVAL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(ctx->host_scratch, &ctx->st->n, sizeof(long long),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "get_count");
  *n_host = ctx->host_scratch[0];
  ctx->n_upper = *n_host;
  return LBX_OK;
}

int lbx_ctx_enable_timing(lbx_ctx* ctx, int on) {
  clear_error();
  if (!ctx) return set_error(LBX_EINVAL, "context is NULL");
  if (on && !ctx->ev0) {
    cudaEventCreate((cudaEvent_t*)&ctx->ev0);
    cudaEventCreate((cudaEvent_t*)&ctx->ev1);
  }
  ctx->timing = on != 0;
  return LBX_OK;
}

int lbx_ctx_last_kernel_ms(lbx_ctx* ctx, float* ms) {
  clear_error();
  if (!ctx || !ms || !ctx->ev0) return set_error(LBX_EINVAL, "timing not enabled");
  cudaError_t e = cudaEventSynchronize((cudaEvent_t)ctx->ev1);
  if (e == cudaSuccess) e = cudaEventElapsedTime(ms, (cudaEvent_t)ctx->ev0, (cudaEvent_t)ctx->ev1);
  if (e != cudaSuccess) return cuda_fail(e, "kernel timing");
  return LBX_OK;
}

int lbx_ctx_set_grid(lbx_ctx* ctx, int ctas) {
  clear_error();
  if (!ctx) return set_error(LBX_EINVAL, "context is NULL");
  ctx->grid_override = ctas > 0 ? ctas : 0;
  return LBX_OK;
}

int lbx_advance_particles(lbx_ctx* ctx, const double* pos, const double* vel, int64_t n,
                          double extent_z, double extent_x, double* out_pos, double* out_vel,
                          int64_t* m_dev, void* stream) {
  clear_error();
  if (!ctx) return set_error(LBX_EINVAL, "context is NULL");
  if (n < 0) return set_error(LBX_EINVAL, "n must be >= 0");
  if (n > 0 && (!pos || !vel || !out_pos || !out_vel))
    return set_error(LBX_EINVAL, "NULL particle buffer");
  if (((uintptr_t)pos | (uintptr_t)vel | (uintptr_t)out_pos | (uintptr_t)out_vel) & 15u)
    return set_error(LBX_EINVAL, "particle arrays must be 16-byte aligned");
  int rc = reserve_status(ctx, n);
  if (rc) return rc;
  ScanParams p{};
  p.in_pos = reinterpret_cast<const double2*>(pos);
  p.in_vel = reinterpret_cast<const double2*>(vel);
  p.out_pos = reinterpret_cast<double2*>(out_pos);
  p.out_vel = reinterpret_cast<double2*>(out_vel);
  p.ez = extent_z;
  p.ex = extent_x;
  p.n_host = n;
  p.st = ctx->st;
  p.status = ctx->status;
  p.n_out = reinterpret_cast<long long*>(m_dev);
  return launch_scan<kAdvanceAoS>(ctx, p, n, (cudaStream_t)stream);
}

int lbx_bin_particles(const double* pos, int64_t n, double box_size, int32_t nbz, int32_t nbx,
                      int64_t* counts, int64_t* err_dev, void* stream) {
  clear_error();
  if (nbz < 0 || nbx < 0) return set_error(LBX_EINVAL, "box grid must be nonnegative");
  if (n < 0) return set_error(LBX_EINVAL, "n must be >= 0");
  const long long nb = (long long)nbz * nbx;
  cudaStream_t s = (cudaStream_t)stream;
  if (nb > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)nb * sizeof(int64_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  }
  if (n == 0) return LBX_OK;
  if (nb == 0) return set_error(LBX_ERANGE, "particles present but the box grid is empty");
  if ((uintptr_t)pos & 15u) return set_error(LBX_EINVAL, "positions must be 16-byte aligned");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem_hist = nb <= kSmemBoxesMax ? 1 : 0;
  const size_t smem = smem_hist ? (size_t)nb * 4 : 0;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long grid = std::min((long long)sms * 8, (long long)((n + kBlock * 8 - 1) / (kBlock * 8)));
  grid = std::max(1ll, grid);
  bin_kernel<<<(unsigned)grid, kBlock, smem, s>>>(
      reinterpret_cast<const double2*>(pos), n, box_size, nbz, nbx, smem_hist,
      reinterpret_cast<unsigned long long*>(counts),
      reinterpret_cast<unsigned long long*>(err_dev), nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bin_kernel launch");
  return LBX_OK;
}

int lbx_push_step(lbx_ctx* ctx, const lbx_step_args* a, void* stream) {
  clear_error();
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  StepLaunch l{};
  l.z = a->z;
  l.x = a->x;
  l.vz = a->vz;
  l.vx = a->vx;
  l.ez = a->extent_z;
  l.ex = a->extent_x;
  l.m = a->box_size;
  l.nbz = a->nbz;
  l.nbx = a->nbx;
  l.wp = a->w_particle;
  l.wc = a->w_cell;
  l.cells = a->cells_per_box;
  l.clock = (a->flags & LBX_STEP_CLOCK) != 0;
  l.counts_out = reinterpret_cast<long long*>(a->counts_out);
  l.cost_out = a->cost_out;
  l.clk_out = reinterpret_cast<unsigned long long*>(a->clk_out);
  l.n_out = reinterpret_cast<long long*>(a->n_out);
  l.err_out = reinterpret_cast<long long*>(a->err_out);
  return launch_push_step(ctx, l, stream, nullptr, true);
}

int lbx_heuristic_cost(const double* particles, const double* cells, int64_t n,
                       double w_particle, double w_cell, double* cost, void* stream) {
  clear_error();
  if (n < 0) return set_error(LBX_EINVAL, "length must be >= 0");
  if (n == 0) return LBX_OK;
  heuristic_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      particles, cells, n, w_particle, w_cell, cost);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "heuristic launch");
  return LBX_OK;
}

int lbx_advance_bin_host(lbx_ctx* ctx, const double* pos, const double* vel, int64_t n,
                         double extent_z, double extent_x, double box_size, int32_t nbz,
                         int32_t nbx, double w_particle, double w_cell, double* out_pos,
                         double* out_vel, int64_t* counts, double* cost, int64_t* m_out) {
  clear_error();
  if (!ctx || !m_out) return set_error(LBX_EINVAL, "NULL argument");
  if (n < 0) return set_error(LBX_EINVAL, "n must be >= 0");
  const bool bin = counts != nullptr;
  const long long nb = (long long)nbz * nbx;
  if (bin && nb < 1) return set_error(LBX_EINVAL, "box grid must be at least 1x1");
  cudaSetDevice(ctx->device);
  const long long C = HostPipe::kChunk;
  const long long nchunks = (n + C - 1) / C;
  int rc = ensure_pipe(ctx, bin ? nb : 0, nchunks);
  if (rc) return rc;
  HostPipe& hp = *ctx->pipe;
  constexpr int L = HostPipe::kLanes;
  cudaError_t e = cudaSuccess;
  if (bin) e = cudaMemsetAsync(hp.d_counts, 0, (size_t)nb * 8, hp.s[0]);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  cudaEventRecord(hp.ready, hp.s[0]);
  for (int l = 1; l < L; ++l) cudaStreamWaitEvent(hp.s[l], hp.ready, 0);
  const int smem_hist = (bin && nb <= kSmemBoxesMax) ? 1 : 0;
  const size_t bsmem = smem_hist ? (size_t)nb * 4 : 0;
  if (bsmem > 48 * 1024)
    cudaFuncSetAttribute(bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
  // Every chunk is fully stream-ordered (copy in -> advance -> bin -> copy
  // out -> survivor count) with no host round trip: its survivors land at the
  // chunk's own offset i*C of the output (speculating that nothing is
  // absorbed) and the host closes the gaps afterwards in the rare case that
  // something was.  Lane l = i % L reuses its buffers in stream order.
  for (long long i = 0; i < nchunks; ++i) {
    const int l = (int)(i % L);
    const long long k = std::min(C, n - i * C);
    cudaStream_t s = hp.s[l];
    cudaMemcpyAsync(hp.d_in_pos[l], pos + 2 * i * C, (size_t)k * 16, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(hp.d_in_vel[l], vel + 2 * i * C, (size_t)k * 16, cudaMemcpyHostToDevice, s);
    ScanParams p{};
    p.in_pos = reinterpret_cast<const double2*>(hp.d_in_pos[l]);
    p.in_vel = reinterpret_cast<const double2*>(hp.d_in_vel[l]);
    p.out_pos = reinterpret_cast<double2*>(hp.d_out_pos[l]);
    p.out_vel = reinterpret_cast<double2*>(hp.d_out_vel[l]);
    p.ez = extent_z;
    p.ex = extent_x;
    p.n_host = k;
    p.st = hp.st[l];
    p.status = hp.status[l];
    p.n_out = hp.d_m[l];
    rc = launch_scan<kAdvanceAoS>(ctx, p, k, s);
    if (rc) return rc;
    if (bin) {
      const long long grid =
          std::max(1ll, std::min((long long)ctx->num_sms * 8, (k + kBlock * 8 - 1) / (kBlock * 8)));
      bin_kernel<<<(unsigned)grid, kBlock, bsmem, s>>>(
          reinterpret_cast<const double2*>(hp.d_out_pos[l]), k, box_size, nbz, nbx, smem_hist,
          reinterpret_cast<unsigned long long*>(hp.d_counts),
          reinterpret_cast<unsigned long long*>(hp.d_err), hp.d_m[l]);
    }
    cudaMemcpyAsync(out_pos + 2 * i * C, hp.d_out_pos[l], (size_t)k * 16, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(out_vel + 2 * i * C, hp.d_out_vel[l], (size_t)k * 16, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hp.h_m[i], hp.d_m[l], 8, cudaMemcpyDeviceToHost, s);
  }
  for (int l = 1; l < L; ++l) {
    cudaEventRecord(hp.ready, hp.s[l]);
    cudaStreamWaitEvent(hp.s[0], hp.ready, 0);
  }
  if (bin) {
    counts_cost_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, hp.s[0]>>>(
        hp.d_counts, (int)nb, w_particle, w_cell, box_size * box_size, hp.d_cost);
    cudaMemcpyAsync(counts, hp.d_counts, (size_t)nb * 8, cudaMemcpyDeviceToHost, hp.s[0]);
    if (cost) cudaMemcpyAsync(cost, hp.d_cost, (size_t)nb * 8, cudaMemcpyDeviceToHost, hp.s[0]);
    cudaMemcpyAsync(&hp.h_m[nchunks], hp.d_err, 8, cudaMemcpyDeviceToHost, hp.s[0]);
  }
  for (int l = 0; l < L && e == cudaSuccess; ++l) e = cudaStreamSynchronize(hp.s[l]);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline");
  if (bin && hp.h_m[nchunks] != 0) {
    cudaMemsetAsync(hp.d_err, 0, 8, hp.s[0]);
    cudaStreamSynchronize(hp.s[0]);
    return set_error(LBX_ERANGE, "%lld survivors fall outside the box grid",
                     (long long)hp.h_m[nchunks]);
  }
  long long written = 0;
  for (long long i = 0; i < nchunks; ++i) {   // close the gaps left by absorbed particles
    const long long m = hp.h_m[i];
    if (written != i * C && m > 0) {
      std::memmove(out_pos + 2 * written, out_pos + 2 * i * C, (size_t)m * 16);
      std::memmove(out_vel + 2 * written, out_vel + 2 * i * C, (size_t)m * 16);
    }
    written += m;
  }
  *m_out = written;
  return LBX_OK;
}

int lbx_push_step_exchange(lbx_ctx* ctx, const lbx_step_args* a, const lbx_exchange_args* ex,
                           void* stream) {
  clear_error();
  if (!ctx || !a || !ex) return set_error(LBX_EINVAL, "NULL argument");
  if (ex->world < 1 || ex->world > 64 || ex->rank < 0 || ex->rank >= ex->world)
    return set_error(LBX_EINVAL, "rank %d / world %d out of range", ex->rank, ex->world);
  if (!ex->owner || !ex->send_counts ||
      (!ex->peer_recv && (!ex->stage || !ex->stage_dest)) || (ex->peer_recv && !ex->peer_cursor))
    return set_error(LBX_EINVAL, "NULL exchange buffer");
  StepLaunch l{};
  l.z = a->z;
  l.x = a->x;
  l.vz = a->vz;
  l.vx = a->vx;
  l.ez = a->extent_z;
  l.ex = a->extent_x;
  l.m = a->box_size;
  l.nbz = a->nbz;
  l.nbx = a->nbx;
  l.wp = a->w_particle;
  l.wc = a->w_cell;
  l.cells = a->cells_per_box;
  l.clock = (a->flags & LBX_STEP_CLOCK) != 0;
  l.counts_out = reinterpret_cast<long long*>(a->counts_out);
  l.cost_out = a->cost_out;
  l.clk_out = reinterpret_cast<unsigned long long*>(a->clk_out);
  l.n_out = reinterpret_cast<long long*>(a->n_out);
  l.err_out = reinterpret_cast<long long*>(a->err_out);
  return launch_push_step(ctx, l, stream, ex, true);
}

int lbx_partition(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx, double extent_z,
                  double extent_x, double box_size, int32_t nbz, int32_t nbx,
                  const lbx_exchange_args* ex, int64_t* n_out, void* stream) {
  clear_error();
  if (!ctx || !ex) return set_error(LBX_EINVAL, "NULL argument");
  if (ex->world < 1 || ex->world > 64 || ex->rank < 0 || ex->rank >= ex->world)
    return set_error(LBX_EINVAL, "rank %d / world %d out of range", ex->rank, ex->world);
  StepLaunch l{};
  l.z = z;
  l.x = x;
  l.vz = vz;
  l.vx = vx;
  l.ez = extent_z;
  l.ex = extent_x;
  l.m = box_size;
  l.nbz = nbz;
  l.nbx = nbx;
  l.n_out = reinterpret_cast<long long*>(n_out);
  return launch_push_step(ctx, l, stream, ex, false);
}

static int push_step_3d(lbx_ctx* ctx, const lbx_step3d_args* a, const lbx_exchange_args* ex,
                        void* stream);

int lbx_push_step_3d(lbx_ctx* ctx, const lbx_step3d_args* a, void* stream) {
  clear_error();
  return push_step_3d(ctx, a, nullptr, stream);
}

int lbx_push_step_3d_exchange(lbx_ctx* ctx, const lbx_step3d_args* a,
                              const lbx_exchange_args* ex, void* stream) {
  clear_error();
  if (!ex) return set_error(LBX_EINVAL, "NULL argument");
  if (ex->world < 1 || ex->world > 64 || ex->rank < 0 || ex->rank >= ex->world)
    return set_error(LBX_EINVAL, "rank %d / world %d out of range", ex->rank, ex->world);
  if (!ex->owner || !ex->stage || !ex->stage_dest || !ex->send_counts || !ex->removed_list)
    return set_error(LBX_EINVAL, "3D exchange needs owner, stage, stage_dest, send_counts "
                                 "and removed_list");
  if (ex->kick_vz || ex->kick_vx || ex->peer_recv)
    return set_error(LBX_EINVAL, "3D exchange: no pending kick arrays, no peer buffers");
  return push_step_3d(ctx, a, ex, stream);
}

static int push_step_3d(lbx_ctx* ctx, const lbx_step3d_args* a, const lbx_exchange_args* ex,
                        void* stream) {
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  const int M = a->box_size;
  if (M < 1 || (M & (M - 1)) || a->extent_z % M || a->extent_y % M || a->extent_x % M)
    return set_error(LBX_EINVAL, "3D box_size must be a power of two dividing the extents");
  if (((uintptr_t)a->z | (uintptr_t)a->y | (uintptr_t)a->x | (uintptr_t)a->vz |
       (uintptr_t)a->vy | (uintptr_t)a->vx) & 15u)
    return set_error(LBX_EINVAL, "particle arrays must be 16-byte aligned");
  const int nbz = a->extent_z / M, nby = a->extent_y / M, nbx = a->extent_x / M;
  const long long nb = (long long)nbz * nby * nbx;
  if (nb > (1ll << 30)) return set_error(LBX_EINVAL, "too many boxes");
  int rc = ensure_accumulators(ctx, (int32_t)nb);
  if (rc) return rc;
  rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  Step3DParams p{};
  p.z = a->z;
  p.y = a->y;
  p.x = a->x;
  p.vz = a->vz;
  p.vy = a->vy;
  p.vx = a->vx;
  p.ez = a->extent_z;
  p.ey = a->extent_y;
  p.ex = a->extent_x;
  p.inv_m = 1.0 / M;
  p.nbz = nbz;
  p.nby = nby;
  p.nbx = nbx;
  p.nb = (int)nb;
  p.smem_hist = nb <= kSmemBoxesMax ? 1 : 0;
  p.st = ctx->st;
  p.g_cnt = ctx->acc;
  p.g_clk = ctx->acc + ctx->acc_boxes;
  p.counts_out = reinterpret_cast<long long*>(a->counts_out);
  p.cost_out = a->cost_out;
  p.clk_out = reinterpret_cast<unsigned long long*>(a->clk_out);
  p.n_out = reinterpret_cast<long long*>(a->n_out);
  p.err_out = reinterpret_cast<long long*>(a->err_out);
  p.wp = a->w_particle;
  p.wc = a->w_cell;
  p.cells = (double)M * M * M;
  p.removed_list = reinterpret_cast<long long*>(a->removed_list);
  p.removed_cap = a->removed_cap;
  if (ex) {
    p.owner = ex->owner;
    p.me = ex->rank;
    p.stage = ex->stage;
    p.stage_dest = ex->stage_dest;
    p.stage_cap = ex->stage_cap;
    p.send_counts = reinterpret_cast<long long*>(ex->send_counts);
    p.removed_list = reinterpret_cast<long long*>(ex->removed_list);
    p.removed_cap = ex->removed_cap;
  }
  const bool clock = (a->flags & LBX_STEP_CLOCK) != 0;
  auto kern = clock ? stream3d_kernel<true> : stream3d_kernel<false>;
  const size_t smem = p.smem_hist ? (size_t)nb * 4 * (clock ? 2 : 1) : 0;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 0;
  rc = occupancy_grid(ctx, kern, smem,
                      std::max(1ll, (long long)((ctx->n_upper + 2ll * kBlock * kPairs - 1) /
                                                (2ll * kBlock * kPairs))), &grid);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->timing) cudaEventRecord((cudaEvent_t)ctx->ev0, s);
  kern<<<grid, kBlock, smem, s>>>(p);
  if (ctx->timing) cudaEventRecord((cudaEvent_t)ctx->ev1, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "stream3d_kernel launch");
  if (p.removed_list) return LBX_OK;  // caller compacts with lbx_fill_holes
  return launch_compact(ctx, a->z, a->x, a->y, a->vz, a->vy, a->vx, (double)a->extent_z,
                        (double)a->extent_x, stream);
}

int lbx_partition_3d(lbx_ctx* ctx, double* z, double* y, double* x, double* vz, double* vy,
                     double* vx, int32_t extent_z, int32_t extent_y, int32_t extent_x,
                     int32_t box_size, const lbx_exchange_args* ex, int64_t* n_out,
                     void* stream) {
  clear_error();
  if (!ctx || !ex || !n_out) return set_error(LBX_EINVAL, "NULL argument");
  const int M = box_size;
  if (M < 1 || (M & (M - 1)) || extent_z % M || extent_y % M || extent_x % M)
    return set_error(LBX_EINVAL, "3D box_size must be a power of two dividing the extents");
  if (ex->world < 1 || ex->world > 64 || ex->rank < 0 || ex->rank >= ex->world)
    return set_error(LBX_EINVAL, "rank %d / world %d out of range", ex->rank, ex->world);
  if (!ex->owner || !ex->stage || !ex->stage_dest || !ex->send_counts || !ex->removed_list)
    return set_error(LBX_EINVAL, "3D partition needs owner, stage, stage_dest, send_counts "
                                 "and removed_list");
  Step3DParams p{};
  p.z = z;
  p.y = y;
  p.x = x;
  p.vz = vz;
  p.vy = vy;
  p.vx = vx;
  p.inv_m = 1.0 / M;
  p.nbz = extent_z / M;
  p.nby = extent_y / M;
  p.nbx = extent_x / M;
  p.st = ctx->st;
  p.owner = ex->owner;
  p.me = ex->rank;
  p.stage = ex->stage;
  p.stage_dest = ex->stage_dest;
  p.stage_cap = ex->stage_cap;
  p.send_counts = reinterpret_cast<long long*>(ex->send_counts);
  p.removed_list = reinterpret_cast<long long*>(ex->removed_list);
  p.removed_cap = ex->removed_cap;
  cudaStream_t s = (cudaStream_t)stream;
  const long long blocks = std::max(1ll, std::min((long long)(ctx->n_upper + kBlock - 1) / kBlock,
                                                  (long long)ctx->num_sms * 8));
  partition3d_kernel<<<(unsigned)blocks, kBlock, 0, s>>>(p);
  partition_done_kernel<<<1, 1, 0, s>>>(ctx->st, reinterpret_cast<long long*>(n_out));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "partition3d_kernel launch");
  return LBX_OK;
}

int lbx_fill_holes(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx, double* kick_vz,
                   double* kick_vx, const int64_t* removed, int64_t n_removed, int64_t n_new,
                   void* stream) {
  clear_error();
  if (!ctx || n_removed < 0 || n_new < 0) return set_error(LBX_EINVAL, "bad argument");
  if ((kick_vz == nullptr) != (kick_vx == nullptr))
    return set_error(LBX_EINVAL, "kick velocity buffers must be given together");
  cudaStream_t s = (cudaStream_t)stream;
  if (n_removed > 0) {
    if (ctx->fill_cap < n_removed) {
      if (ctx->fill_scratch) {
        cudaStreamSynchronize(s);
        cudaFree(ctx->fill_scratch);
      }
      ctx->fill_scratch = nullptr;
      const int64_t cap = std::max<int64_t>(n_removed, 1 << 16);
      if (cudaMalloc(&ctx->fill_scratch, (size_t)cap * 16) != cudaSuccess)
        return set_error(LBX_EOOM, "hole-fill scratch");
      cudaMemsetAsync(ctx->fill_scratch + cap, 0, (size_t)cap * 8, s);
      ctx->fill_cap = cap;
    }
    long long* holes = ctx->fill_scratch;
    long long* tail = ctx->fill_scratch + ctx->fill_cap;
    const unsigned grid = (unsigned)std::max(1ll, std::min(4096ll, (long long)((n_removed + 255) / 256)));
    fill_mark_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const long long*>(removed), n_removed,
                                          n_new, holes, tail, ctx->st);
    fill_move_kernel<<<grid, 256, 0, s>>>(n_removed, n_new, holes, tail, ctx->st, z, x, vz, vx,
                                          kick_vz, kick_vx);
  }
  fill_done_kernel<<<1, 1, 0, s>>>(ctx->st, n_new);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fill_holes launch");
  ctx->n_upper = n_new;
  return LBX_OK;
}

int lbx_fill_holes_dev(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx,
                       double* kick_vz, double* kick_vx, const int64_t* removed,
                       int64_t removed_cap, double extent_z, double extent_x, void* stream) {
  clear_error();
  if (!ctx || !removed || removed_cap < 0) return set_error(LBX_EINVAL, "bad argument");
  if ((kick_vz == nullptr) != (kick_vx == nullptr))
    return set_error(LBX_EINVAL, "kick velocity buffers must be given together");
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->fill_cap < removed_cap) {
    if (ctx->fill_scratch) {
      cudaStreamSynchronize(s);
      cudaFree(ctx->fill_scratch);
    }
    ctx->fill_scratch = nullptr;
    const int64_t cap = std::max<int64_t>(removed_cap, 1 << 16);
    if (cudaMalloc(&ctx->fill_scratch, (size_t)cap * 16) != cudaSuccess)
      return set_error(LBX_EOOM, "hole-fill scratch");
    cudaMemsetAsync(ctx->fill_scratch + cap, 0, (size_t)cap * 8, s);
    ctx->fill_cap = cap;
  }
  const unsigned grid = (unsigned)std::max(1, ctx->num_sms * 4);
  fill_dev_mark_kernel<<<grid, 256, 0, s>>>(ctx->st, reinterpret_cast<const long long*>(removed),
                                            removed_cap, ctx->fill_scratch);
  fill_dev_move_kernel<<<grid, 256, 0, s>>>(ctx->st, removed_cap, ctx->fill_scratch, extent_z,
                                            extent_x, z, x, vz, vx, kick_vz, kick_vx);
  fill_dev_done_kernel<<<1, 1, 0, s>>>(ctx->st, removed_cap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fill_holes_dev launch");
  return LBX_OK;
}

int lbx_unpack_peer_dev(lbx_ctx* ctx, const double* recv, uint64_t* cursor, int64_t capacity,
                        double* z, double* x, double* vz, double* vx, double* kick_vz,
                        double* kick_vx, void* stream) {
  clear_error();
  if (!ctx || !recv || !cursor || capacity < 0) return set_error(LBX_EINVAL, "bad argument");
  if ((kick_vz == nullptr) != (kick_vx == nullptr))
    return set_error(LBX_EINVAL, "kick velocity buffers must be given together");
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max(1, ctx->num_sms * 2);
  unpack_dev_kernel<<<grid, 256, 0, s>>>(recv, reinterpret_cast<unsigned long long*>(cursor),
                                         ctx->st, capacity, z, x, vz, vx, kick_vz, kick_vx);
  unpack_dev_done_kernel<<<1, 1, 0, s>>>(ctx->st, reinterpret_cast<unsigned long long*>(cursor),
                                         capacity);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "unpack_dev launch");
  return LBX_OK;
}

int lbx_group_by_dest(const double* stage, const int32_t* stage_dest, int64_t count,
                      int32_t world, int64_t* cursors, double* send, void* stream) {
  clear_error();
  if (count < 0 || world < 1) return set_error(LBX_EINVAL, "bad count/world");
  if (count == 0) return LBX_OK;
  const unsigned grid = (unsigned)std::min<long long>(4096, (count + 255) / 256);
  group_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      stage, stage_dest, count, reinterpret_cast<unsigned long long*>(cursors), send);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "group_kernel launch");
  return LBX_OK;
}

int lbx_unpack(const double* recv, int64_t n_recv, int64_t offset, double* z, double* x,
               double* vz, double* vx, double* kick_vz, double* kick_vx, void* stream) {
  clear_error();
  if (n_recv < 0 || offset < 0) return set_error(LBX_EINVAL, "bad count/offset");
  if ((kick_vz == nullptr) != (kick_vx == nullptr))
    return set_error(LBX_EINVAL, "kick velocity buffers must be given together");
  if (n_recv == 0) return LBX_OK;
  const unsigned grid = (unsigned)std::min<long long>(4096, (n_recv + 255) / 256);
  unpack_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(recv, n_recv, offset, z, x, vz, vx,
                                                         kick_vz, kick_vx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "unpack_kernel launch");
  return LBX_OK;
}

int lbx_peer_alloc(int64_t bytes, void** ptr, unsigned char handle[64]) {
  clear_error();
  if (!ptr || !handle || bytes <= 0) return set_error(LBX_EINVAL, "bad peer allocation request");
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) return set_error(LBX_EOOM, "peer buffer: %s", cudaGetErrorString(e));
  cudaMemset(*ptr, 0, (size_t)bytes);
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, 64);
  return LBX_OK;
}

int lbx_peer_open(const unsigned char handle[64], void** ptr) {
  clear_error();
  if (!ptr || !handle) return set_error(LBX_EINVAL, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return LBX_OK;
}

int lbx_peer_close(void* ptr) {
  clear_error();
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? LBX_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int lbx_peer_free(void* ptr) {
  clear_error();
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? LBX_OK : cuda_fail(e, "cudaFree(peer)");
}

int lbx_peer_can_access(int32_t dev, int32_t peer, int32_t* yes) {
  clear_error();
  if (!yes) return set_error(LBX_EINVAL, "NULL argument");
  int v = 0;
  if (dev == peer) {
    *yes = 1;
    return LBX_OK;
  }
  const cudaError_t e = cudaDeviceCanAccessPeer(&v, dev, peer);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceCanAccessPeer");
  *yes = v;
  return LBX_OK;
}

}  // extern "C"
