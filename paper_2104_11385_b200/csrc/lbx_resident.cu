// libLBX resident multi-step kernel for sm_100a: the reference's own step
// (advance_particles + bin_particles, _kernels.pyx:12-47; heuristic_cost,
// cost.py:83-95; GpuClock tally) at the sizes the reference runs (C1 131 k,
// C2 801 k particles), where a step is a few microseconds of work and the
// per-step kernels of lbx_kernels.cu are launch / tail bound.
//
// One persistent CTA per SM (cooperative launch) runs every step of a
// lbx_sim_run call: G - 1 "pushers" and one "courier".  Pusher b owns the
// contiguous slot range [n*b/P, n*(b+1)/P) of the particle arrays and keeps
// it in SHARED MEMORY for the whole run (32 B/particle: z, x, vz, vx;
// 147 x 227 KB holds ~1 M particles), so a step touches no HBM:
//   * push: z += vz, x += vx (separately rounded, no FMA), absorbing test,
//     box id; per-box survivor counts (+ GpuClock cycles) in a shared
//     histogram, warp-aggregated;
//   * stable compaction of the CTA's own range in shared memory (only on
//     steps that absorbed a particle).  The concatenation of the CTAs'
//     compacted ranges IS the reference's stable compaction of the array, so
//     ranges never exchange particles;
//   * the CTA adds its non-zero box counts to the step's device accumulator
//     slot (ring of kAccSlots steps) and bumps the slot's arrival count, then
//     goes straight on to the next step.
// The courier waits for each step's arrivals, writes the step record (counts,
// clock tally, n, err) into the mapped host ring, raises the host's ready
// flags and releases the slot.  Pushers wait only when the slot they need is
// still unrecorded (kAccSlots steps back); the courier only when the host
// ring is full (the host has not consumed H steps back).  The host forms the
// heuristic cost from the counts (same separately rounded products).
// At the end of the run each pusher writes its compacted range back in place
// and marks the tail of its range as holes (z = -1); the host then runs the
// look-back compaction (scan_kernel<COMPACT_SOA>), which produces exactly the
// reference's array.  Counts / costs / n / final state are bit-identical to
// the per-step path (tests/test_gpu_resident.py).

#include <cuda_runtime.h>

#include <climits>

#include "lbx_internal.h"

namespace lbx {
namespace {

constexpr int kRT = 1024;            // threads per CTA
constexpr int kRW = kRT / 32;
constexpr int kMaxRounds = 8;        // particles per thread (keep mask / table rows)
constexpr int kAccSlots = kResSlots; // device accumulator ring (steps)
constexpr int kClkShift = 4;         // GpuClock tally unit: 16 SM cycles (as stream_kernel)
constexpr unsigned kAllR = 0xffffffffu;

struct ResParams {
  double *z, *x;             // positions (in / out)
  double *vz, *vx;           // velocities before the kick (or the only ones)
  double *kvz, *kvx;         // kick velocities (from kick_step on), may be NULL
  long long first, last, kick_step;
  double ez, ex, m, inv_m;
  int pow2;
  int nbz, nbx, nb;
  double wp, wc, cells;
  int cap;                   // per-CTA particle capacity (shared memory)
  DevState* st;
  ResCtl* ctl;               // device
  unsigned long long* acc;   // [kAccSlots][2 * nb]: counts, clock
  unsigned char* rec;        // mapped host ring (device pointer)
  long long rec_bytes;
  int H;                     // host ring slots
  unsigned long long* flags; // mapped [H]: step + 1 once the record is written
  const volatile unsigned long long* consumed;  // mapped: host-processed steps (last + 1)
  const volatile unsigned* abort_h;             // mapped: host gave up
  unsigned long long* trace;  // LBX_RES_TRACE builds: [3][steps] globaltimer stamps
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned lane_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

constexpr int kPublish = 4;          // courier: one system fence per this many steps

__device__ __forceinline__ unsigned ld_acq32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Courier CTA (the grid's last): records every step once all pushers have
// flushed it -- per-box counts (+ clock) and n into the mapped host ring --
// clears the accumulator slot and releases it.  Off the pushers' critical
// path; one system-scope fence per kPublish steps before raising the flags
// of the steps written since the last one (the courier's threads wrote all
// of them, so their own fences cover every record).
template <bool kClock>
__device__ void courier(const ResParams& p, int pushers, int* s_flag) {
  const int tid = threadIdx.x;
  unsigned long long cons = 0;
  long long pub = p.first;   // first step whose flag is not raised yet
  for (long long s = p.first; s < p.last; ++s) {
    const int slot = (int)(s % kAccSlots);
    const int hs = (int)(s % p.H);
    if (tid == 0) {
      int ab = 0;
      while (ld_acq32(&p.ctl->arrive[slot]) < (unsigned)pushers) {
        if (*p.abort_h || *((volatile unsigned*)&p.ctl->abort)) {
          ab = 1;
          break;
        }
        __nanosleep(32);
      }
      while (!ab && (long long)cons < s - p.H + 1) {   // host ring slot hs free?
        cons = *p.consumed;
        if ((long long)cons >= s - p.H + 1) break;
        if (*p.abort_h) ab = 1;
        else __nanosleep(256);
      }
      *s_flag = ab;
      if (p.trace) p.trace[(p.last - p.first) + s - p.first] = gtime();
    }
    __syncthreads();
    if (*s_flag) {   // the host gave up: release the pushers, stop
      if (tid == 0) {
        atomicExch(&p.ctl->abort, 1u);
        __threadfence();
        st_rel(&p.ctl->recorded, (unsigned long long)LLONG_MAX);
      }
      return;
    }
    unsigned long long* acc = p.acc + (size_t)slot * 2 * p.nb;
    unsigned char* r = p.rec + (size_t)hs * p.rec_bytes;
    long long* counts_out = reinterpret_cast<long long*>(r);
    unsigned long long* clk_out = reinterpret_cast<unsigned long long*>(r + 16 * (size_t)p.nb);
    long long* n_out = reinterpret_cast<long long*>(r + 24 * (size_t)p.nb);
    for (int i = tid; i < p.nb; i += kRT) {
      const unsigned long long c = __ldcg(acc + i);
      const unsigned long long k = kClock ? __ldcg(acc + p.nb + i) : 0ull;
      __stcg(acc + i, 0ull);
      counts_out[i] = (long long)c;
      if (kClock) {
        __stcg(acc + p.nb + i, 0ull);
        clk_out[i] = k << kClkShift;
      }
    }
    if (tid == 0) {
      n_out[0] = (long long)atomicExch(&p.ctl->n_acc[slot], 0ull);
      n_out[1] = (long long)*((volatile unsigned long long*)&p.ctl->err_acc) +
                 *((volatile long long*)&p.st->err);
    }
    const bool publish = (s + 1 - p.first) % kPublish == 0 || s + 1 == p.last;
    if (publish) __threadfence_system();   // this thread's records are in host memory
    __syncthreads();
    if (tid == 0) {
      if (publish) {
        for (; pub <= s; ++pub)
          *((volatile unsigned long long*)(p.flags + pub % p.H)) = (unsigned long long)(pub + 1);
      }
      __threadfence();                     // the slot's clears before its release
      p.ctl->arrive[slot] = 0u;
      st_rel(&p.ctl->recorded, (unsigned long long)(s + 1));
      if (p.trace) p.trace[2 * (p.last - p.first) + s - p.first] = gtime();
    }
  }
}

template <bool kClock>
__global__ void __launch_bounds__(kRT, 1) resident_kernel(ResParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sz = reinterpret_cast<double*>(smem);
  double* sx = sz + p.cap;
  double* svz = sx + p.cap;
  double* svx = svz + p.cap;
  unsigned* s_cnt = reinterpret_cast<unsigned*>(svx + p.cap);
  unsigned* s_clk = s_cnt + p.nb;
  __shared__ unsigned s_ball[kMaxRounds][kRW];   // keep ballots of the step
  __shared__ int s_pre[kMaxRounds][kRW];         // their exclusive prefix
  __shared__ int s_flag;
  __shared__ long long s_n0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x, P = G - 1;   // P pushers + the courier
  if (tid == 0) s_n0 = *((volatile long long*)&p.st->n);
  for (int i = tid; i < p.nb; i += kRT) {
    s_cnt[i] = 0u;
    if (kClock) s_clk[i] = 0u;
  }
  __syncthreads();
  const long long n0 = s_n0;
  long long seg = 0;
  int len = 0, nloc = 0;
  long long err_total = 0;   // this CTA's out-of-grid survivors (cumulative)
  const bool kick_any = p.kvz != nullptr;
  if (b == P) {
    courier<kClock>(p, P, &s_flag);
  } else {
    seg = n0 * b / P;
    len = (int)(n0 * (b + 1) / P - seg);
    nloc = len;
    // velocities live at the run start: the kick arrays once the kick is past
    const double* v0z = (kick_any && p.first > p.kick_step) ? p.kvz : p.vz;
    const double* v0x = (kick_any && p.first > p.kick_step) ? p.kvx : p.vx;
    for (int i = tid; i < len; i += kRT) {
      sz[i] = __ldcg(p.z + seg + i);
      sx[i] = __ldcg(p.x + seg + i);
      svz[i] = __ldcg(v0z + seg + i);
      svx[i] = __ldcg(v0x + seg + i);
    }
    __syncthreads();
    unsigned long long rec_seen = 0;   // thread 0: last value of ctl->recorded read
    for (long long s = p.first; s < p.last; ++s) {
      // the kick: this step and every later one push with the kick velocities
      // (kick slots follow the CTA range: compacted with it while pending)
      if (kick_any && s == p.kick_step) {
        for (int i = tid; i < nloc; i += kRT) {
          svz[i] = __ldcg(p.kvz + seg + i);
          svx[i] = __ldcg(p.kvx + seg + i);
        }
        __syncthreads();
      }
      const bool kick_pending = kick_any && s < p.kick_step;
      if (p.trace && b == 0 && tid == 0) p.trace[s - p.first] = gtime();
      // ---- push + absorb + box counts ----
      unsigned keepm = 0;
      int rm = 0, err = 0;
      const int rounds = (nloc + kRT - 1) / kRT;
      for (int j = 0; j < rounds; ++j) {
        const int i = j * kRT + tid;
        const bool have = i < nloc;
        long long t0 = 0;
        double z = 0.0, x = 0.0;
        if (have) {
          z = __dadd_rn(sz[i], svz[i]);
          x = __dadd_rn(sx[i], svx[i]);
        }
        if (kClock) t0 = clock64();
        const bool keep = have && z >= 0.0 && z < p.ez && x >= 0.0 && x < p.ex;
        int box = -1;
        if (keep) {
          int bz, bx;
          if (p.pow2) {
            bz = (int)__dmul_rn(z, p.inv_m);   // exact: M is a power of two
            bx = (int)__dmul_rn(x, p.inv_m);
          } else {
            bz = (int)__ddiv_rn(z, p.m);
            bx = (int)__ddiv_rn(x, p.m);
          }
          if (bz < p.nbz && bx < p.nbx) box = bz * p.nbx + bx;
          else ++err;
          sz[i] = z;
          sx[i] = x;
        }
        keepm |= keep ? (1u << j) : 0u;
        rm += (have && !keep) ? 1 : 0;
        const unsigned bl = __ballot_sync(kAllR, keep);
        if (lane == 0) s_ball[j][warp] = bl;
        unsigned dt = 0;
        if (kClock) dt = (unsigned)min(clock64() - t0, (long long)(1 << 20)) >> kClkShift;
        const int box0 = __shfl_sync(kAllR, box, 0);
        if (__all_sync(kAllR, box == box0)) {
          if (box0 >= 0) {
            const unsigned clk = kClock ? __reduce_add_sync(kAllR, dt) : 0u;
            if (lane == 0) {
              atomicAdd(s_cnt + box0, (unsigned)__popc(bl));
              if (kClock) atomicAdd(s_clk + box0, clk);
            }
          }
        } else if (box >= 0) {
          atomicAdd(s_cnt + box, 1u);
          if (kClock) atomicAdd(s_clk + box, dt);
        }
      }
      err_total += err;
      // ---- stable compaction of the CTA range (steps that absorbed) ----
      if (__syncthreads_or(rm)) {
        if (warp == 0) {   // exclusive prefix of the (round, warp) keep counts
          int base = 0;
          for (int j = 0; j < rounds; ++j) {
            const int c = __popc(s_ball[j][lane]);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(kAllR, incl, o);
              if (lane >= o) incl += y;
            }
            s_pre[j][lane] = base + incl - c;
            base += __shfl_sync(kAllR, incl, 31);
          }
          if (lane == 0) s_flag = base;
        }
        __syncthreads();
        const int kept = s_flag;
        for (int j = 0; j < rounds; ++j) {
          const int i = j * kRT + tid;
          const bool keep = (keepm >> j) & 1u;
          double a = 0, c = 0, d = 0, e = 0, f = 0, g = 0;
          if (keep) {
            a = sz[i];
            c = sx[i];
            d = svz[i];
            e = svx[i];
            if (kick_pending) {
              f = __ldcg(p.kvz + seg + i);
              g = __ldcg(p.kvx + seg + i);
            }
          }
          __syncthreads();   // round j read before anything of it is overwritten
          if (keep) {
            const int dst = s_pre[j][warp] + __popc(s_ball[j][warp] & lane_lt());
            sz[dst] = a;
            sx[dst] = c;
            svz[dst] = d;
            svx[dst] = e;
            if (kick_pending) {
              __stcg(p.kvz + seg + dst, f);
              __stcg(p.kvx + seg + dst, g);
            }
          }
        }
        nloc = kept;
      }
      // ---- flush the step into its accumulator slot (recorded s - kAccSlots?) ----
      const int slot = (int)(s % kAccSlots);
      if (tid == 0) {
        const unsigned long long need = (unsigned long long)(s - kAccSlots + 1);
        int ab = 0;
        if (s - p.first >= kAccSlots && rec_seen < need) {
          while ((rec_seen = ld_acq(&p.ctl->recorded)) < need) {
            if (*((volatile unsigned*)&p.ctl->abort)) break;
            __nanosleep(64);
          }
          ab = *((volatile unsigned*)&p.ctl->abort) ? 1 : 0;
        }
        s_flag = ab;
      }
      __syncthreads();
      if (s_flag) break;
      unsigned long long* acc = p.acc + (size_t)slot * 2 * p.nb;
      for (int i = tid; i < p.nb; i += kRT) {
        const unsigned c = s_cnt[i];
        if (c) {
          atomicAdd(acc + i, (unsigned long long)c);
          s_cnt[i] = 0u;
        }
        if (kClock) {
          const unsigned k = s_clk[i];
          if (k) {
            atomicAdd(acc + p.nb + i, (unsigned long long)k);
            s_clk[i] = 0u;
          }
        }
      }
      if (tid == 0) {
        atomicAdd(&p.ctl->n_acc[slot], (unsigned long long)nloc);
        if (err) atomicAdd(&p.ctl->err_acc, (unsigned long long)err);
      }
      __syncthreads();
      if (tid == 0) {   // arrival: this CTA's adds happen-before the courier's reads
        __threadfence();
        atomicAdd(&p.ctl->arrive[slot], 1u);
      }
    }
  }

  // ---- write the compacted range back; its tail becomes holes ----
  const bool kicked_end = kick_any && p.last > p.kick_step;
  double* fz = kicked_end ? p.kvz : p.vz;
  double* fx = kicked_end ? p.kvx : p.vx;
  for (int i = tid; i < len; i += kRT) {
    if (i < nloc) {
      __stcg(p.z + seg + i, sz[i]);
      __stcg(p.x + seg + i, sx[i]);
      __stcg(fz + seg + i, svz[i]);
      __stcg(fx + seg + i, svx[i]);
    } else {
      __stcg(p.z + seg + i, -1.0);   // dropped by the look-back compaction
    }
  }
  if (tid == 0) {
    if (nloc < len) {
      atomicAdd(&p.st->leavers, (unsigned long long)(len - nloc));
      atomicMin(&p.st->first_leaver, seg + nloc);
    }
    atomicAdd(&p.ctl->n_final, (unsigned long long)nloc);
    if (err_total) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)err_total);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0 && atomicAdd(&p.ctl->done, 1u) == (unsigned)(G - 1)) {
    __threadfence();
    p.st->n_old = n0;
    p.st->n = (long long)atomicExch(&p.ctl->n_final, 0ull);
    p.ctl->done = 0u;
    p.ctl->err_acc = 0ull;
    p.ctl->recorded = 0ull;
    __threadfence();
  }
}

}  // namespace

int resident_capacity(lbx_ctx* ctx, int nb, long long* max_particles, int* grid) {
  int smem_max = 0;
  cudaError_t e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                         ctx->device);
  if (e != cudaSuccess) return set_error(LBX_ECUDA, "device query: %s", cudaGetErrorString(e));
  const long long avail = (long long)smem_max - 8ll * nb - 4096;   // static shared + slack
  *max_particles = avail > 0 && ctx->num_sms > 1 ? (avail / 32) * (ctx->num_sms - 1) : 0;
  *grid = ctx->num_sms;
  return LBX_OK;
}

int launch_resident(lbx_ctx* ctx, const ResidentLaunch& a, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int G = ctx->num_sms;
  if (G < 2) return set_error(LBX_EINVAL, "resident: needs 2 or more SMs");
  const long long cap = (a.n + G - 2) / (G - 1);   // G - 1 pushers, one courier
  if (cap > (long long)kMaxRounds * kRT)
    return set_error(LBX_EINVAL, "resident: %lld particles per CTA exceed %d", cap,
                     kMaxRounds * kRT);
  ResParams p{};
  p.z = a.z;
  p.x = a.x;
  p.vz = a.vz;
  p.vx = a.vx;
  p.kvz = a.kvz;
  p.kvx = a.kvx;
  p.first = a.first;
  p.last = a.last;
  p.kick_step = a.kick_step;
  p.ez = a.ez;
  p.ex = a.ex;
  p.m = a.m;
  p.inv_m = 1.0 / a.m;
  p.pow2 = a.pow2;
  p.nbz = a.nbz;
  p.nbx = a.nbx;
  p.nb = a.nbz * a.nbx;
  p.wp = a.wp;
  p.wc = a.wc;
  p.cells = a.cells;
  p.cap = (int)cap;
  p.st = ctx->st;
  p.ctl = a.ctl;
  p.acc = a.acc;
  p.rec = a.rec;
  p.rec_bytes = (long long)a.rec_bytes;
  p.H = a.H;
  p.flags = a.flags;
  p.consumed = a.consumed;
  p.abort_h = a.abort_h;
  p.trace = a.trace;
  const size_t smem = (size_t)cap * 32 + (size_t)p.nb * 8;
  void* args[] = {&p};
  const void* kern = a.clock ? (const void*)resident_kernel<true> : (const void*)resident_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_error(LBX_ECUDA, "resident smem attribute: %s", cudaGetErrorString(e));
  e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(kRT), args, smem, s);
  if (e != cudaSuccess) return set_error(LBX_ECUDA, "resident launch: %s", cudaGetErrorString(e));
  return LBX_OK;
}

}  // namespace lbx
