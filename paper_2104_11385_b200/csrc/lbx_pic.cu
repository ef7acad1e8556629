// libLBX 2D3V electromagnetic PIC step for sm_100a (SURVEY 8a row a15,
// north-star item 1: "per-box particle push, current deposition and field
// gather ... with vectorised SoA particle loads and shared-memory staging of
// each tile's field and current patches").  The reference has no PIC (it
// models the step as ballistic motion); the CPU restatement used
// as the checker is oracle/pic_oracle.py (parity unpinned, tolerance tests).
//
// Particles: SoA float64 z, x, uz, ux, uy (u = gamma v, c = 1), uniform
// charge q and macro weight w.  Fields: float32 Yee grid (2D in z, x; y
// invariant) with one zero guard layer (conducting walls); offsets in cells
// Ex (0,1/2) Ey (0,0) Ez (1/2,0) Bx (1/2,0) By (1/2,1/2) Bz (0,1/2), J as E.
//
// pic_push_kernel -- one pass per 1024-particle chunk (a "tile"):
//   1. 16-byte pair loads of the chunk's particles (5 arrays);
//   2. block-reduced bounding box of the chunk's cells; the chunk's field
//      patch (bbox + 2-cell halo, <= kPatchMax cells) is staged into shared
//      memory with coalesced loads, and a zeroed current patch is set up;
//   3. CIC gather of the 6 components from shared memory, relativistic Boris
//      push, move, absorbing test;
//   4. direct current deposition into the shared current patch (shared-memory
//      float atomics), then one flush of the patch to HBM (global atomics,
//      nonzero cells only);
//   5. z, x, u written back in place; per-box survivor counts + GpuClock
//      tally (same run-length / warp-reduced histogram as the surrogate
//      kernel); absorbed particles recorded for the compaction pass.
//   Chunks whose patch would not fit fall back to direct global gather /
//   atomics (uniform per CTA).
// pic_b_kernel / pic_e_kernel -- Yee leapfrog (B -= dt curl E;
//   E += dt (curl B - J)), fp64 arithmetic rounded to float32 (bit-identical
//   to the oracle's), J consumed and zeroed.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>

#include "lbx_internal.h"

namespace lbx {
namespace {

#ifndef LBX_PIC_PAIRS
#define LBX_PIC_PAIRS 1
#endif
constexpr int kPB = 256;                  // threads per CTA
constexpr int kPW = kPB / 32;
constexpr int kPPairs = LBX_PIC_PAIRS;    // particle pairs per thread per chunk
constexpr int kPItems = 2 * kPPairs;
constexpr int kPChunk = kPB * kPItems;    // 1024 particles per chunk
constexpr int kPatchMax = 1536;           // cells per staged patch
constexpr unsigned kAll = 0xffffffffu;

struct PicParams {
  double *z, *x, *uz, *ux, *uy;
  float* F[6];   // Ex Ey Ez Bx By Bz
  unsigned long long* Jacc[3];  // fixed-point current accumulators (int64)
  double jscale;                // power-of-two fixed-point scale
  int nz, nx, pitch;
  double qm, qw, dt;
  double inv_m;  // box binning: power-of-two box size (checked on host)
  int nbz, nbx, nb;
  DevState* st;
  unsigned long long* g_cnt;
  unsigned long long* g_clk;
  long long* counts_out;
  double* cost_out;
  unsigned long long* clk_out;
  long long* n_out;
  long long* err_out;
  double wp, wc, cells;
};

__constant__ float c_oz[6] = {0.f, 0.f, 0.5f, 0.5f, 0.5f, 0.f};
__constant__ float c_ox[6] = {0.5f, 0.f, 0.f, 0.f, 0.5f, 0.5f};

__device__ __forceinline__ long long warp_min(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kAll, v, o));
  return v;
}
__device__ __forceinline__ long long warp_max(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kAll, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kAll, v, o);
  return v;
}

// float32 stencil: index in 32-bit, cell fractions rounded to float32.
struct StencilF {
  int i0, j0;
  float fz, fx;
};

__device__ __forceinline__ StencilF stencil_f(double z, double x, double oz, double ox) {
  const double zc = __dsub_rn(z, oz), xc = __dsub_rn(x, ox);
  const double fl_z = floor(zc), fl_x = floor(xc);
  StencilF s;
  s.i0 = (int)fl_z;
  s.j0 = (int)fl_x;
  s.fz = __double2float_rn(__dsub_rn(zc, fl_z));
  s.fx = __double2float_rn(__dsub_rn(xc, fl_x));
  return s;
}

// float32 CIC: (1-fz)((1-fx) a + fx b) + fz((1-fx) c + fx d), oracle order.
__device__ __forceinline__ float cic_f(const StencilF& s, float a, float b, float c, float d) {
  const float gz = __fsub_rn(1.f, s.fz), gx = __fsub_rn(1.f, s.fx);
  const float lo = __fadd_rn(__fmul_rn(gx, a), __fmul_rn(s.fx, b));
  const float hi = __fadd_rn(__fmul_rn(gx, c), __fmul_rn(s.fx, d));
  return __fadd_rn(__fmul_rn(gz, lo), __fmul_rn(s.fz, hi));
}

template <bool kClock>
#ifndef LBX_PIC_MINB
#define LBX_PIC_MINB 3
#endif
__global__ void __launch_bounds__(kPB, LBX_PIC_MINB) pic_push_kernel(PicParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned* s_cnt = reinterpret_cast<unsigned*>(smem_raw);          // nb
  unsigned* s_clk = s_cnt + p.nb;                                    // nb
  float* s_F = reinterpret_cast<float*>(s_clk + p.nb);               // 6 * kPatchMax
  int* s_J = reinterpret_cast<int*>(s_F + 6 * kPatchMax);            // 3 * kPatchMax
  __shared__ long long s_n;
  __shared__ int s_box[4];  // imin, imax, jmin, jmax
  __shared__ int s_last;
  __shared__ unsigned long long s_red[kPW];
  __shared__ long long s_min[kPW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_n = *((volatile long long*)&p.st->n);
  for (int b = tid; b < p.nb; b += kPB) {
    s_cnt[b] = 0u;
    if (kClock) s_clk[b] = 0u;
  }
  __syncthreads();
  const long long n = s_n;
  const long long npairs = (n + 1) >> 1;
  const double ez = (double)p.nz, ex = (double)p.nx;
  const double h = 0.5 * p.qm * p.dt;
  const float jscale_f = (float)p.jscale;   // power of two: exact in float
  double2* z2 = reinterpret_cast<double2*>(p.z);
  double2* x2 = reinterpret_cast<double2*>(p.x);
  double2* uz2 = reinterpret_cast<double2*>(p.uz);
  double2* ux2 = reinterpret_cast<double2*>(p.ux);
  double2* uy2 = reinterpret_cast<double2*>(p.uy);
  unsigned long long removed = 0;
  long long first_out = LLONG_MAX, err = 0;

  for (long long q0 = (long long)blockIdx.x * kPB * kPPairs; q0 < npairs;
       q0 += (long long)gridDim.x * kPB * kPPairs) {
    long long t0 = 0;
    if (kClock) t0 = clock64();
    double pz[kPItems], px[kPItems], puz[kPItems], pux[kPItems], puy[kPItems];
    bool valid[kPItems];
#pragma unroll
    for (int r = 0; r < kPPairs; ++r) {
      const long long q = q0 + r * kPB + tid;
      double2 a = make_double2(0.5, 0.5), b = a, c = make_double2(0.0, 0.0), d = c, e = c;
      const bool any = q < npairs;
      if (any) {
        a = __ldcs(z2 + q);
        b = __ldcs(x2 + q);
        c = __ldcs(uz2 + q);
        d = __ldcs(ux2 + q);
        e = __ldcs(uy2 + q);
      }
      pz[2 * r] = a.x;
      pz[2 * r + 1] = a.y;
      px[2 * r] = b.x;
      px[2 * r + 1] = b.y;
      puz[2 * r] = c.x;
      puz[2 * r + 1] = c.y;
      pux[2 * r] = d.x;
      pux[2 * r + 1] = d.y;
      puy[2 * r] = e.x;
      puy[2 * r + 1] = e.y;
      valid[2 * r] = any;
      valid[2 * r + 1] = 2 * q + 1 < n;
    }
    // ---- chunk bounding box (cells) ----
    long long imin = LLONG_MAX, imax = LLONG_MIN, jmin = LLONG_MAX, jmax = LLONG_MIN;
#pragma unroll
    for (int k = 0; k < kPItems; ++k) {
      if (!valid[k]) continue;
      const long long i = (int)pz[k], j = (int)px[k];  // positions >= 0: trunc == floor
      imin = min(imin, i);
      imax = max(imax, i);
      jmin = min(jmin, j);
      jmax = max(jmax, j);
    }
    imin = warp_min(imin);
    imax = warp_max(imax);
    jmin = warp_min(jmin);
    jmax = warp_max(jmax);
    if (tid == 0) {
      s_box[0] = INT_MAX;
      s_box[1] = INT_MIN;
      s_box[2] = INT_MAX;
      s_box[3] = INT_MIN;
    }
    __syncthreads();
    if (lane == 0 && imin <= imax) {
      atomicMin(&s_box[0], (int)imin);
      atomicMax(&s_box[1], (int)imax);
      atomicMin(&s_box[2], (int)jmin);
      atomicMax(&s_box[3], (int)jmax);
    }
    __syncthreads();
    // patch rows/cols in cell units, clipped to the guarded grid [-1, n]
    const int pi0 = max(s_box[0] - 2, -1), pi1 = min(s_box[1] + 2, p.nz);
    const int pj0 = max(s_box[2] - 2, -1), pj1 = min(s_box[3] + 2, p.nx);
    const int H = pi1 - pi0 + 1, W = pj1 - pj0 + 1;
    const bool staged = s_box[0] <= s_box[1] && H * W <= kPatchMax;
    if (staged) {
      for (int idx = tid; idx < H * W; idx += kPB) {
        const int li = idx / W, lj = idx - li * W;
        const long long g = (long long)(pi0 + li + 1) * p.pitch + (pj0 + lj + 1);
#pragma unroll
        for (int c = 0; c < 6; ++c) s_F[c * kPatchMax + idx] = __ldg(p.F[c] + g);
#pragma unroll
        for (int c = 0; c < 3; ++c) s_J[c * kPatchMax + idx] = 0;
      }
    }
    __syncthreads();

    // ---- gather, push, move, absorb (per lane), deposit (warp-collective) ----
    double nz_[kPItems], nx_[kPItems];
    bool keep[kPItems];
#pragma unroll
    for (int k = 0; k < kPItems; ++k) {
      keep[k] = false;
      nz_[k] = pz[k];
      nx_[k] = px[k];
      double vel[3] = {0.0, 0.0, 0.0};
      if (valid[k]) {
        // 4 distinct staggers: A (0,1/2) Ex Bz | B (0,0) Ey | C (1/2,0) Ez Bx | D (1/2,1/2) By
        const StencilF st[4] = {stencil_f(pz[k], px[k], 0.0, 0.5), stencil_f(pz[k], px[k], 0.0, 0.0),
                                stencil_f(pz[k], px[k], 0.5, 0.0), stencil_f(pz[k], px[k], 0.5, 0.5)};
        constexpr int kSt[6] = {0, 1, 2, 2, 3, 0};   // Ex Ey Ez Bx By Bz -> stencil
        double f6[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const StencilF& sc = st[kSt[c]];
          float a, b, cc, d;
          if (staged) {
            const float* F = s_F + c * kPatchMax;
            const int o = (sc.i0 - pi0) * W + (sc.j0 - pj0);
            a = F[o];
            b = F[o + 1];
            cc = F[o + W];
            d = F[o + W + 1];
          } else {
            const float* F = p.F[c];
            const long long o = (long long)(sc.i0 + 1) * p.pitch + (sc.j0 + 1);
            a = __ldg(F + o);
            b = __ldg(F + o + 1);
            cc = __ldg(F + o + p.pitch);
            d = __ldg(F + o + p.pitch + 1);
          }
          f6[c] = (double)cic_f(sc, a, b, cc, d);
        }
        // relativistic Boris (x, y, z order; E = f6[0..2], B = f6[3..5])
        const double mx = __dadd_rn(pux[k], __dmul_rn(h, f6[0]));
        const double my = __dadd_rn(puy[k], __dmul_rn(h, f6[1]));
        const double mz = __dadd_rn(puz[k], __dmul_rn(h, f6[2]));
        const double g = sqrt(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(mx, mx)),
                                                  __dmul_rn(my, my)), __dmul_rn(mz, mz)));
        const double ig = __ddiv_rn(1.0, g);
        const double tx = __dmul_rn(__dmul_rn(h, f6[3]), ig);
        const double ty = __dmul_rn(__dmul_rn(h, f6[4]), ig);
        const double tz = __dmul_rn(__dmul_rn(h, f6[5]), ig);
        const double s2 = __ddiv_rn(2.0, __dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(tx, tx)),
                                                             __dmul_rn(ty, ty)),
                                                   __dmul_rn(tz, tz)));
        const double qx = __dadd_rn(mx, __dsub_rn(__dmul_rn(my, tz), __dmul_rn(mz, ty)));
        const double qy = __dadd_rn(my, __dsub_rn(__dmul_rn(mz, tx), __dmul_rn(mx, tz)));
        const double qz = __dadd_rn(mz, __dsub_rn(__dmul_rn(mx, ty), __dmul_rn(my, tx)));
        const double rx = __dadd_rn(mx, __dmul_rn(s2, __dsub_rn(__dmul_rn(qy, tz), __dmul_rn(qz, ty))));
        const double ry = __dadd_rn(my, __dmul_rn(s2, __dsub_rn(__dmul_rn(qz, tx), __dmul_rn(qx, tz))));
        const double rz = __dadd_rn(mz, __dmul_rn(s2, __dsub_rn(__dmul_rn(qx, ty), __dmul_rn(qy, tx))));
        pux[k] = __dadd_rn(rx, __dmul_rn(h, f6[0]));
        puy[k] = __dadd_rn(ry, __dmul_rn(h, f6[1]));
        puz[k] = __dadd_rn(rz, __dmul_rn(h, f6[2]));
        const double gam = sqrt(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(pux[k], pux[k])),
                                                    __dmul_rn(puy[k], puy[k])),
                                          __dmul_rn(puz[k], puz[k])));
        const double igam = __ddiv_rn(1.0, gam);
        nz_[k] = __dadd_rn(pz[k], __dmul_rn(__dmul_rn(p.dt, puz[k]), igam));
        nx_[k] = __dadd_rn(px[k], __dmul_rn(__dmul_rn(p.dt, pux[k]), igam));
        keep[k] = nz_[k] >= 0.0 && nz_[k] < ez && nx_[k] >= 0.0 && nx_[k] < ex;
        vel[0] = __dmul_rn(__dmul_rn(p.qw, pux[k]), igam);
        vel[1] = __dmul_rn(__dmul_rn(p.qw, puy[k]), igam);
        vel[2] = __dmul_rn(__dmul_rn(p.qw, puz[k]), igam);
      }
      // Deposition: node contributions quantised to fixed point (exact
      // power-of-two scaling, round-to-nearest-even), pre-summed over lanes
      // that share a stencil (__match_any_sync + redux.sync) and added with
      // native 32-bit shared atomics -- order-independent, deterministic.
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const StencilF s = stencil_f(keep[k] ? nz_[k] : 0.5, keep[k] ? nx_[k] : 0.5,
                                     (double)c_oz[c], (double)c_ox[c]);
        int q[4] = {0, 0, 0, 0};
        if (keep[k]) {
          const float gz = __fsub_rn(1.f, s.fz), gx = __fsub_rn(1.f, s.fx);
          const float v = __double2float_rn(vel[c]);
          const float vz = __fmul_rn(v, gz), vf = __fmul_rn(v, s.fz);
          q[0] = __float2int_rn(__fmul_rn(__fmul_rn(vz, gx), jscale_f));
          q[1] = __float2int_rn(__fmul_rn(__fmul_rn(vz, s.fx), jscale_f));
          q[2] = __float2int_rn(__fmul_rn(__fmul_rn(vf, gx), jscale_f));
          q[3] = __float2int_rn(__fmul_rn(__fmul_rn(vf, s.fx), jscale_f));
        }
        long long off;
        int row;
        if (staged) {
          off = (long long)(s.i0 - pi0) * W + (s.j0 - pj0);
          row = W;
        } else {
          off = (long long)(s.i0 + 1) * p.pitch + (s.j0 + 1);
          row = p.pitch;
        }
        // Warp-uniform fast path: all depositing lanes share the stencil
        // (sorted particles, 55 per cell) -> 4 full-warp redux.sync and one
        // lane adds; otherwise each lane adds (native 32-bit atomics).
        const unsigned dep = __ballot_sync(kAll, keep[k]);
        if (!dep) continue;
        const long long off0 = __shfl_sync(kAll, off, __ffs(dep) - 1);
        if (__all_sync(kAll, !keep[k] || off == off0)) {
          const int t0s = __reduce_add_sync(kAll, q[0]);
          const int t1s = __reduce_add_sync(kAll, q[1]);
          const int t2s = __reduce_add_sync(kAll, q[2]);
          const int t3s = __reduce_add_sync(kAll, q[3]);
          if (lane == __ffs(dep) - 1) {
            if (staged) {
              int* J = s_J + c * kPatchMax + off;
              atomicAdd(J, t0s);
              atomicAdd(J + 1, t1s);
              atomicAdd(J + row, t2s);
              atomicAdd(J + row + 1, t3s);
            } else {
              unsigned long long* J = p.Jacc[c] + off;
              atomicAdd(J, (unsigned long long)(long long)t0s);
              atomicAdd(J + 1, (unsigned long long)(long long)t1s);
              atomicAdd(J + row, (unsigned long long)(long long)t2s);
              atomicAdd(J + row + 1, (unsigned long long)(long long)t3s);
            }
          }
        } else if (keep[k]) {
          if (staged) {
            int* J = s_J + c * kPatchMax + off;
            atomicAdd(J, q[0]);
            atomicAdd(J + 1, q[1]);
            atomicAdd(J + row, q[2]);
            atomicAdd(J + row + 1, q[3]);
          } else {
            unsigned long long* J = p.Jacc[c] + off;
            atomicAdd(J, (unsigned long long)(long long)q[0]);
            atomicAdd(J + 1, (unsigned long long)(long long)q[1]);
            atomicAdd(J + row, (unsigned long long)(long long)q[2]);
            atomicAdd(J + row + 1, (unsigned long long)(long long)q[3]);
          }
        }
      }
    }
    unsigned dt_clk = 0;
    if (kClock) dt_clk = (unsigned)min(clock64() - t0, (long long)(1 << 20)) >> 4;
    __syncthreads();
    if (staged) {  // flush the current patch
      for (int idx = tid; idx < H * W; idx += kPB) {
        const int li = idx / W, lj = idx - li * W;
        const long long g = (long long)(pi0 + li + 1) * p.pitch + (pj0 + lj + 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int v = s_J[c * kPatchMax + idx];
          if (v) atomicAdd(p.Jacc[c] + g, (unsigned long long)(long long)v);
        }
      }
    }
    // ---- store, bin, account ----
#pragma unroll
    for (int r = 0; r < kPPairs; ++r) {
      const long long q = q0 + r * kPB + tid;
      if (!valid[2 * r]) continue;
      __stcs(z2 + q, make_double2(nz_[2 * r], nz_[2 * r + 1]));
      __stcs(x2 + q, make_double2(nx_[2 * r], nx_[2 * r + 1]));
      __stcs(uz2 + q, make_double2(puz[2 * r], puz[2 * r + 1]));
      __stcs(ux2 + q, make_double2(pux[2 * r], pux[2 * r + 1]));
      __stcs(uy2 + q, make_double2(puy[2 * r], puy[2 * r + 1]));
      for (int t = 0; t < 2; ++t) {
        if (valid[2 * r + t] && !keep[2 * r + t]) {
          ++removed;
          first_out = min(first_out, 2 * q + t);
        }
      }
    }
    int cur = -1;
    unsigned run = 0;
#pragma unroll
    for (int k = 0; k < kPItems; ++k) {
      int b = -1;
      if (keep[k]) {
        const int bz = (int)__dmul_rn(nz_[k], p.inv_m), bx = (int)__dmul_rn(nx_[k], p.inv_m);
        if (bz < p.nbz && bx < p.nbx) b = bz * p.nbx + bx;
        else ++err;
      }
      if (b != cur) {
        if (cur >= 0) {
          atomicAdd(s_cnt + cur, run);
          if (kClock) atomicAdd(s_clk + cur, dt_clk * run);
        }
        cur = b;
        run = 0;
      }
      run += b >= 0 ? 1u : 0u;
    }
    const int cur0 = __shfl_sync(kAll, cur, 0);
    if (__all_sync(kAll, cur == cur0)) {
      const unsigned tot = __reduce_add_sync(kAll, run);
      const unsigned clk = kClock ? __reduce_add_sync(kAll, dt_clk * run) : 0u;
      if (lane == 0 && cur0 >= 0 && tot) {
        atomicAdd(s_cnt + cur0, tot);
        if (kClock) atomicAdd(s_clk + cur0, clk);
      }
    } else if (cur >= 0 && run) {
      atomicAdd(s_cnt + cur, run);
      if (kClock) atomicAdd(s_clk + cur, dt_clk * run);
    }
    __syncthreads();  // s_F / s_J / s_box reuse
  }

  // ---- CTA totals, histogram flush, epilogue (as the surrogate kernel) ----
  const unsigned long long wa = (unsigned long long)warp_sum((long long)removed);
  const long long wm = warp_min(first_out), we = warp_sum(err);
  if (lane == 0) {
    s_red[warp] = wa;
    s_min[warp] = wm;
    if (we) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)we);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long ta = 0;
    long long tm = LLONG_MAX;
    for (int w = 0; w < kPW; ++w) {
      ta += s_red[w];
      tm = min(tm, s_min[w]);
    }
    if (ta) {
      atomicAdd(&p.st->leavers, ta);
      atomicMin(&p.st->first_leaver, tm);
    }
  }
  for (int b = tid; b < p.nb; b += kPB) {
    if (s_cnt[b]) atomicAdd(p.g_cnt + b, (unsigned long long)s_cnt[b]);
    if (kClock && s_clk[b]) atomicAdd(p.g_clk + b, (unsigned long long)s_clk[b]);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int b = tid; b < p.nb; b += kPB) {
    const unsigned long long c = atomicExch(p.g_cnt + b, 0ull);
    if (p.counts_out) p.counts_out[b] = (long long)c;
    if (p.cost_out)
      p.cost_out[b] = __dadd_rn(__dmul_rn(p.wp, (double)(long long)c), __dmul_rn(p.wc, p.cells));
    if (kClock) {
      const unsigned long long k = atomicExch(p.g_clk + b, 0ull);
      if (p.clk_out) p.clk_out[b] = k << 4;
    }
  }
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

// Fixed-point current -> float32 J (J += sum / scale), accumulators zeroed.
__global__ void pic_current_kernel(unsigned long long* acc0, unsigned long long* acc1,
                                   unsigned long long* acc2, float* J0, float* J1, float* J2,
                                   long long cells, double inv_scale) {
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < cells;
       o += (long long)gridDim.x * blockDim.x) {
    unsigned long long* acc[3] = {acc0, acc1, acc2};
    float* J[3] = {J0, J1, J2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long v = (long long)acc[c][o];
      if (v) {
        J[c][o] = __fadd_rn(J[c][o], (float)__dmul_rn((double)v, inv_scale));
        acc[c][o] = 0ull;
      }
    }
  }
}

// Yee update, interior cells; float32 storage, float64 arithmetic in the
// oracle's evaluation order.
__global__ void pic_b_kernel(const float* __restrict__ Ex, const float* __restrict__ Ey,
                             const float* __restrict__ Ez, float* Bx, float* By, float* Bz,
                             int nz, int nx, int pitch, double dt) {
  const long long cells = (long long)nz * nx;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cells;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c / nx), j = (int)(c - (long long)i * nx);
    const long long o = (long long)(i + 1) * pitch + (j + 1);
    const double ey = Ey[o];
    Bx[o] = (float)__dadd_rn((double)Bx[o], __dmul_rn(dt, __dsub_rn((double)Ey[o + pitch], ey)));
    By[o] = (float)__dsub_rn((double)By[o],
                             __dmul_rn(dt, __dsub_rn(__dsub_rn((double)Ex[o + pitch], (double)Ex[o]),
                                                     __dsub_rn((double)Ez[o + 1], (double)Ez[o]))));
    Bz[o] = (float)__dsub_rn((double)Bz[o], __dmul_rn(dt, __dsub_rn((double)Ey[o + 1], ey)));
  }
}

__global__ void pic_e_kernel(float* Ex, float* Ey, float* Ez, const float* __restrict__ Bx,
                             const float* __restrict__ By, const float* __restrict__ Bz, float* Jx,
                             float* Jy, float* Jz, int nz, int nx, int pitch, double dt) {
  const long long all = (long long)(nz + 2) * pitch;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < all;
       o += (long long)gridDim.x * blockDim.x) {
    const int ii = (int)(o / pitch), jj = (int)(o - (long long)ii * pitch);
    if (ii >= 1 && ii <= nz && jj >= 1 && jj <= nx) {
      const double by = By[o];
      Ex[o] = (float)__dadd_rn((double)Ex[o],
                               __dmul_rn(dt, __dsub_rn(-__dsub_rn(by, (double)By[o - pitch]),
                                                       (double)Jx[o])));
      Ey[o] = (float)__dadd_rn(
          (double)Ey[o],
          __dmul_rn(dt, __dsub_rn(__dsub_rn(__dsub_rn((double)Bx[o], (double)Bx[o - pitch]),
                                            __dsub_rn((double)Bz[o], (double)Bz[o - 1])),
                                  (double)Jy[o])));
      Ez[o] = (float)__dadd_rn((double)Ez[o],
                               __dmul_rn(dt, __dsub_rn(__dsub_rn(by, (double)By[o - 1]),
                                                       (double)Jz[o])));
    }
    Jx[o] = 0.f;
    Jy[o] = 0.f;
    Jz[o] = 0.f;
  }
}

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(LBX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace
}  // namespace lbx

using namespace lbx;

extern "C" int lbx_pic_step(lbx_ctx* ctx, const lbx_pic_args* a, void* stream) {
  clear_error();
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  if (a->nz < 1 || a->nx < 1) return set_error(LBX_EINVAL, "grid must be at least 1x1");
  if (a->box_size < 1 || a->nz % a->box_size || a->nx % a->box_size ||
      (a->box_size & (a->box_size - 1)))
    return set_error(LBX_EINVAL, "PIC box_size must be a power of two dividing the grid");
  if (!(a->dt > 0.0 && a->dt < 0.7))
    return set_error(LBX_EINVAL, "dt must be in (0, 0.7) (2D CFL with unit cells)");
  for (int c = 0; c < 6; ++c)
    if (!a->fields[c]) return set_error(LBX_EINVAL, "NULL field array");
  for (int c = 0; c < 3; ++c)
    if (!a->current[c]) return set_error(LBX_EINVAL, "NULL current array");
  if (((uintptr_t)a->z | (uintptr_t)a->x | (uintptr_t)a->uz | (uintptr_t)a->ux |
       (uintptr_t)a->uy) & 15u)
    return set_error(LBX_EINVAL, "particle arrays must be 16-byte aligned");
  const int nbz = a->nz / a->box_size, nbx = a->nx / a->box_size, nb = nbz * nbx;
  if (nb > 4096) return set_error(LBX_EINVAL, "PIC step supports <= 4096 boxes");
  int rc = ensure_accumulators(ctx, nb);
  if (rc) return rc;
  rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  PicParams p{};
  p.z = a->z;
  p.x = a->x;
  p.uz = a->uz;
  p.ux = a->ux;
  p.uy = a->uy;
  for (int c = 0; c < 6; ++c) p.F[c] = a->fields[c];
  const long long padded = (long long)(a->nz + 2) * (a->nx + 2);
  if (!ctx->pic_acc || ctx->pic_cells < padded) {
    if (ctx->pic_acc) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_acc);
    }
    ctx->pic_acc = nullptr;
    if (cudaMalloc(&ctx->pic_acc, (size_t)padded * 3 * 8) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC current accumulators");
    cudaMemset(ctx->pic_acc, 0, (size_t)padded * 3 * 8);
    ctx->pic_cells = padded;
  }
  for (int c = 0; c < 3; ++c) p.Jacc[c] = ctx->pic_acc + c * padded;
  if (!(a->q_times_w != 0.0)) return set_error(LBX_EINVAL, "q_times_w must be nonzero");
  int e2 = 0;
  std::frexp(1048576.0 / std::fabs(a->q_times_w), &e2);  // scale = 2^floor(log2(2^20/|qw|))
  p.jscale = std::ldexp(1.0, e2 - 1);
  p.nz = a->nz;
  p.nx = a->nx;
  p.pitch = a->nx + 2;
  p.qm = a->q_over_m;
  p.qw = a->q_times_w;
  p.dt = a->dt;
  p.inv_m = 1.0 / (double)a->box_size;
  p.nbz = nbz;
  p.nbx = nbx;
  p.nb = nb;
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
  p.cells = (double)a->box_size * (double)a->box_size;
  const size_t smem = (size_t)nb * 8 + (size_t)kPatchMax * 9 * 4;
  const bool clock = (a->flags & LBX_STEP_CLOCK) != 0;
  auto kern = clock ? pic_push_kernel<true> : pic_push_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(pic)");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPB, smem);
  long long grid = (long long)std::max(per_sm, 1) * ctx->num_sms;
  if (ctx->grid_override > 0) grid = ctx->grid_override;
  grid = std::max(1ll, std::min(grid, (long long)((ctx->n_upper + kPChunk - 1) / kPChunk)));
  kern<<<(unsigned)grid, kPB, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pic_push_kernel launch");
  const unsigned cg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (padded + 255) / 256));
  pic_current_kernel<<<cg, 256, 0, s>>>(p.Jacc[0], p.Jacc[1], p.Jacc[2], a->current[0],
                                        a->current[1], a->current[2], padded, 1.0 / p.jscale);
  rc = launch_compact(ctx, a->z, a->x, a->uz, a->ux, a->uy, nullptr, (double)a->nz,
                      (double)a->nx, stream);
  if (rc) return rc;
  if (a->flags & LBX_PIC_NO_FIELD_SOLVE) return LBX_OK;
  const long long cells = (long long)a->nz * a->nx;
  const unsigned fg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (cells + 255) / 256));
  pic_b_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->nz, a->nx, p.pitch, a->dt);
  pic_e_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->current[0], a->current[1],
                                  a->current[2], a->nz, a->nx, p.pitch, a->dt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "field solve launch");
  return LBX_OK;
}
