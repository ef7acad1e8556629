// libLBX 2D3V electromagnetic PIC step for sm_100a (SURVEY 8a row a15,
// north-star item 1: "per-box particle push, current deposition and field
// gather ... with vectorised SoA particle loads and shared-memory staging of
// each tile's field and current patches").  The reference has no PIC (it
// models the step as ballistic motion); the CPU restatement used
// as the checker is oracle/pic_oracle.py (parity unpinned, bit-exact tests).
//
// Particles: SoA float64 z, x, uz, ux, uy (u = gamma v, c = 1), uniform
// charge q and macro weight w.  Fields: float32 Yee grid (2D in z, x; y
// invariant) with one zero guard layer (conducting walls); offsets in cells
// Ex (0,1/2) Ey (0,0) Ez (1/2,0) Bx (1/2,0) By (1/2,1/2) Bz (0,1/2), J as E.
//
// One step = five stream-ordered launches (+ compaction on absorbing steps):
//  pic_quad_kernel    fields -> quad-expanded copy Q[c][node] = float4 of the
//                     2x2 nodes whose lower corner is `node` (HBM, L2/L1
//                     resident for the blob), so a gather is ONE 16-byte load
//                     per component instead of four scalar loads;
//  pic_push_kernel    per warp unit of 64 particles = 2 slots of 32
//                     CONSECUTIVE particles (coalesced 8-byte SoA loads):
//                     gather (6 x LDG.128), relativistic Boris, move, absorb,
//                     then the current of every kept particle as 16
//                     cell-relative fixed-point node values (Jx 2x3, Jy 2x2,
//                     Jz 3x2 nodes around its cell), summed over the slot's
//                     (at most two) cells with full-warp redux.sync and added
//                     with ONE 16-lane 128-byte RED per cell into the
//                     cell-centric accumulator Jc[cell][16]; slots spanning
//                     more cells (unsorted particles) add per lane.  Per-box
//                     survivor counts + GpuClock tally as in the surrogate
//                     kernel; no block barrier inside the particle loop;
//  pic_current_kernel node gather Jc -> J (integer sums: order independent,
//                     bit-identical to the oracle), over the deposit
//                     bounding box only; pic_zero_kernel clears that box;
//  pic_b_kernel / pic_e_kernel -- Yee leapfrog (B -= dt curl E;
//                     E += dt (curl B - J)), fp64 arithmetic rounded to
//                     float32 (bit-identical to the oracle's), J consumed.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>

#include "lbx_internal.h"

namespace lbx {
namespace {

#ifndef LBX_PIC_PB
#define LBX_PIC_PB 256
#endif
constexpr int kPB = LBX_PIC_PB;           // threads per CTA
constexpr int kPW = kPB / 32;
#ifndef LBX_PIC_RUN
#define LBX_PIC_RUN 64
#endif
constexpr int kRun = LBX_PIC_RUN;         // consecutive particles per lane per warp unit
#ifndef LBX_PIC_G
#define LBX_PIC_G 4
#endif
constexpr int kG = LBX_PIC_G;             // particles per vector load group (4: 256-bit)
constexpr int kUnitP = 32 * kRun;         // particles per warp unit
constexpr int kNodes = 16;                // cell-relative current nodes (Jx 6, Jy 4, Jz 6)
constexpr unsigned kAll = 0xffffffffu;

struct PicParams {
  const double *z, *x, *uz, *ux, *uy;     // particles in
  double *oz, *ox, *ouz, *oux, *ouy;      // particles out (== in unless sorting)
  const float4* Q[6];           // quad-expanded Ex Ey Ez Bx By Bz, [(nz+1) x (nx+1)]
  const float* F[6];            // the fields themselves (direct gather, sparse plasmas)
  int pitch;                    // nx + 2
  unsigned long long* Jc;       // cell-centric fixed-point node sums [nz*nx][16]
  int* dep_box;                 // imin, imax, jmin, jmax of depositing cells
  unsigned* cell_cnt;           // sorted mode: kept particles per new cell
  unsigned* cursor;             // sorted mode: next free slot per old cell
  long long* removed_list;      // sorted mode: slots of absorbed particles (hole filling)
  long long removed_cap;
  float vscale;                 // power-of-two fixed-point scale (exact in float)
  int nz, nx, qpitch;
  double qm, qw, dt;
  int log2m;                    // box binning: power-of-two box size (checked on host)
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
  // tiled mode (sparse plasmas): ranges of the last tile-major sort
  const unsigned* tile_rd;      // first slot of each tile's particles [ntiles + 1]
  unsigned long long* Jn;       // node-centric fixed-point current [3][(nz+2)(nx+2)]
  long long jn_stride;
  int ntx, ntiles;
};

__device__ __forceinline__ long long warp_min(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kAll, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kAll, v, o);
  return v;
}

// One axis of a position: its cell i and float32 fraction f (unstaggered
// stencil), and the half-staggered stencil (base ih, fraction fh):
// fh = f - 1/2 (exact, ih = i) when f >= 1/2, else f + 1/2 (ih = i - 1).
// oracle/pic_oracle.py:_axis states the same arithmetic.
struct Axis {
  int i, ih;
  float f, fh;
  bool hi;
};

__device__ __forceinline__ Axis axis_of(double v) {
  const double fl = floor(v);
  const double f = __dsub_rn(v, fl);
  Axis a;
  a.hi = f >= 0.5;
  a.i = (int)fl;
  a.ih = a.hi ? a.i : a.i - 1;
  a.f = __double2float_rn(f);
  a.fh = __double2float_rn(__dadd_rn(f, a.hi ? -0.5 : 0.5));
  return a;
}

// float32 CIC on a quad (a, b, c, d) = nodes (0,0) (0,1) (1,0) (1,1):
// (1-fz)((1-fx) a + fx b) + fz((1-fx) c + fx d), the oracle's order.
__device__ __forceinline__ float cic(const float4 q, float fz, float fx) {
  const float gz = __fsub_rn(1.f, fz), gx = __fsub_rn(1.f, fx);
  const float lo = __fadd_rn(__fmul_rn(gx, q.x), __fmul_rn(fx, q.y));
  const float hi = __fadd_rn(__fmul_rn(gx, q.z), __fmul_rn(fx, q.w));
  return __fadd_rn(__fmul_rn(gz, lo), __fmul_rn(fz, hi));
}

// Tolerance mode (LBX_PIC_FAST): the same bilinear form with FMA
// contraction, a + f (b - a) per axis.
__device__ __forceinline__ float lerp_f(float a, float b, float f) {
  return __fmaf_rn(f, __fsub_rn(b, a), a);
}
__device__ __forceinline__ float cic_fast(const float4 q, float fz, float fx) {
  return lerp_f(lerp_f(q.x, q.y, fx), lerp_f(q.z, q.w, fx), fz);
}
// Tolerance mode on a difference quad (a, b - a, c - a, a - b - c + d), as
// pic_quad_kernel writes it for LBX_PIC_FAST: the bilinear form in 3 FMAs.
__device__ __forceinline__ float cic_diff(const float4 q, float fz, float fx) {
  return __fmaf_rn(fz, __fmaf_rn(fx, q.w, q.z), __fmaf_rn(fx, q.y, q.x));
}

// Fire-and-forget adds (REDG; a plain atomicAdd may keep the returning ATOMG
// form inside large kernels).
__device__ __forceinline__ void red_add(unsigned long long* a, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a), "l"((unsigned long long)v) : "memory");
}
__device__ __forceinline__ void red_add32(unsigned* a, unsigned v) {
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// Streaming particle loads do not allocate in L1, which the quad gathers of
// the blob's few hot cells share (an L2::evict_first hint on top doubled the
// DRAM reads: the second 32-byte sector of a 64-byte DRAM atom is read by
// the next group, after eviction).
#ifndef LBX_PIC_LDQ
#define LBX_PIC_LDQ ".L1::no_allocate"
#endif
__device__ __forceinline__ double ld_na(const double* a) {
  double v;
  asm volatile("ld.global" LBX_PIC_LDQ ".f64 %0, [%1];" : "=d"(v) : "l"(a));
  return v;
}
// kG consecutive doubles [i, i+kG): one vector streaming load (256-bit for
// kG = 4) when the group is complete, else clamped scalar loads (tail lanes
// reload a live particle).
__device__ __forceinline__ void ldg(const double* a, long long i, long long n, double v[kG]) {
  if (i + kG <= n) {
    if (kG % 4 == 0) {
#pragma unroll
      for (int c = 0; c < kG; c += 4)
        asm volatile("ld.global" LBX_PIC_LDQ ".v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[c % kG]), "=d"(v[(c + 1) % kG]), "=d"(v[(c + 2) % kG]),
                       "=d"(v[(c + 3) % kG])
                     : "l"(a + i + c));
    } else {
      asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(a + i));
    }
  } else {
#pragma unroll
    for (int j = 0; j < kG; ++j) v[j] = __ldcs(a + min(i + j, n - 1));
  }
}
__device__ __forceinline__ void stg(double* a, long long i, long long n, const double v[kG]) {
  if (i + kG <= n) {
    if (kG % 4 == 0) {
#pragma unroll
      for (int c = 0; c < kG; c += 4)
        asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(a + i + c), "d"(v[c % kG]),
                     "d"(v[(c + 1) % kG]), "d"(v[(c + 2) % kG]), "d"(v[(c + 3) % kG])
                     : "memory");
    } else {
      asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(a + i), "d"(v[0]), "d"(v[1])
                   : "memory");
    }
  } else {
#pragma unroll
    for (int j = 0; j < kG; ++j)
      if (i + j < n) __stcs(a + i + j, v[j]);
  }
}

__device__ __forceinline__ int qnode(float vs, float wz, float wx) {
  return __float2int_rn(__fmul_rn(__fmul_rn(vs, wz), wx));
}

// The 16 cell-relative fixed-point node values of one deposit (v pre-scaled).
__device__ __forceinline__ void node_values(const Axis& az, const Axis& ax, float vsx, float vsy,
                                            float vsz, int q[kNodes]) {
  const float z0 = __fsub_rn(1.f, az.f), z1 = az.f;
  const float x0 = __fsub_rn(1.f, ax.f), x1 = ax.f;
  const float zh = __fsub_rn(1.f, az.fh), xh = __fsub_rn(1.f, ax.fh);
  const float zm = az.hi ? 0.f : zh, zc = az.hi ? zh : az.fh, zp = az.hi ? az.fh : 0.f;
  const float xm = ax.hi ? 0.f : xh, xc = ax.hi ? xh : ax.fh, xp = ax.hi ? ax.fh : 0.f;
  // Jx: rows {0,1} x cols {-1,0,1}
  q[0] = qnode(vsx, z0, xm);
  q[1] = qnode(vsx, z0, xc);
  q[2] = qnode(vsx, z0, xp);
  q[3] = qnode(vsx, z1, xm);
  q[4] = qnode(vsx, z1, xc);
  q[5] = qnode(vsx, z1, xp);
  // Jy: rows {0,1} x cols {0,1}
  q[6] = qnode(vsy, z0, x0);
  q[7] = qnode(vsy, z0, x1);
  q[8] = qnode(vsy, z1, x0);
  q[9] = qnode(vsy, z1, x1);
  // Jz: rows {-1,0,1} x cols {0,1}
  q[10] = qnode(vsz, zm, x0);
  q[11] = qnode(vsz, zm, x1);
  q[12] = qnode(vsz, zc, x0);
  q[13] = qnode(vsz, zc, x1);
  q[14] = qnode(vsz, zp, x0);
  q[15] = qnode(vsz, zp, x1);
}

// Tolerance mode: the 16 node contributions of one particle as float
// products, FMA-accumulated into the lane's float run sums (rounded to
// fixed point once per run, at the flush, instead of per particle).
__device__ __forceinline__ void node_accum(const Axis& az, const Axis& ax, float vsx, float vsy,
                                           float vsz, float acc[kNodes]) {
  const float z0 = __fsub_rn(1.f, az.f), z1 = az.f;
  const float x0 = __fsub_rn(1.f, ax.f), x1 = ax.f;
  const float zh = __fsub_rn(1.f, az.fh), xh = __fsub_rn(1.f, ax.fh);
  const float zm = az.hi ? 0.f : zh, zc = az.hi ? zh : az.fh, zp = az.hi ? az.fh : 0.f;
  const float xm = ax.hi ? 0.f : xh, xc = ax.hi ? xh : ax.fh, xp = ax.hi ? ax.fh : 0.f;
  const float a0 = __fmul_rn(vsx, z0), a1 = __fmul_rn(vsx, z1);
  acc[0] = __fmaf_rn(a0, xm, acc[0]);
  acc[1] = __fmaf_rn(a0, xc, acc[1]);
  acc[2] = __fmaf_rn(a0, xp, acc[2]);
  acc[3] = __fmaf_rn(a1, xm, acc[3]);
  acc[4] = __fmaf_rn(a1, xc, acc[4]);
  acc[5] = __fmaf_rn(a1, xp, acc[5]);
  const float b0 = __fmul_rn(vsy, z0), b1 = __fmul_rn(vsy, z1);
  acc[6] = __fmaf_rn(b0, x0, acc[6]);
  acc[7] = __fmaf_rn(b0, x1, acc[7]);
  acc[8] = __fmaf_rn(b1, x0, acc[8]);
  acc[9] = __fmaf_rn(b1, x1, acc[9]);
  const float c0 = __fmul_rn(vsz, x0), c1 = __fmul_rn(vsz, x1);
  acc[10] = __fmaf_rn(zm, c0, acc[10]);
  acc[11] = __fmaf_rn(zm, c1, acc[11]);
  acc[12] = __fmaf_rn(zc, c0, acc[12]);
  acc[13] = __fmaf_rn(zc, c1, acc[13]);
  acc[14] = __fmaf_rn(zp, c0, acc[14]);
  acc[15] = __fmaf_rn(zp, c1, acc[15]);
}

// Per-warp flush queue in shared memory: a lane that must hand a cell's node
// sums to HBM (cell change, isolated drifted particle, end of run) writes
// them here with 4 vector stores inside the divergent branch; the warp then
// drains the queue together, one 16-lane 128-byte RED per entry and two
// entries per instruction -- instead of every lane issuing 16 predicated
// REDs whenever any lane flushes.
struct __align__(16) FlushEntry {
  int4 v[kNodes / 4];
  int cell;
  unsigned m;
  int pad[2];
};
#ifndef LBX_PIC_QCAP
#define LBX_PIC_QCAP (32 * kG)
#endif
// Entries per warp queue: drained after every group, after the run's final
// entries, and within a group whenever fewer than 32 free entries remain.
constexpr int kQCap = LBX_PIC_QCAP;

template <bool kSort, bool kFast = false>
__device__ __forceinline__ void drain_queue(const PicParams& p, const FlushEntry* q, int count,
                                            int lane) {
  __syncwarp();
  const int node = lane & 15;
  for (int e0 = 0; e0 < count; e0 += 2) {
    const int e = e0 + (lane >> 4);
    if (e < count) {
      const int cell = q[e].cell;
      const int raw = reinterpret_cast<const int*>(q[e].v)[node];
      // tolerance mode queues float run sums: rounded to fixed point here
      const int v = kFast ? __float2int_rn(__int_as_float(raw)) : raw;
      if (v) red_add(p.Jc + (long long)cell * kNodes + node, v);
      if (kSort && node == 0) red_add32(p.cell_cnt + cell, q[e].m);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void enqueue_f(FlushEntry* e, const float v[kNodes], int cell,
                                          unsigned m) {
#pragma unroll
  for (int i = 0; i < kNodes / 4; ++i)
    e->v[i] = make_int4(__float_as_int(v[4 * i]), __float_as_int(v[4 * i + 1]),
                        __float_as_int(v[4 * i + 2]), __float_as_int(v[4 * i + 3]));
  e->cell = cell;
  e->m = m;
}

__device__ __forceinline__ void enqueue(FlushEntry* e, const int v[kNodes], int cell, unsigned m) {
#pragma unroll
  for (int i = 0; i < kNodes / 4; ++i) e->v[i] = make_int4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  e->cell = cell;
  e->m = m;
}

#ifndef LBX_PIC_MINB
#define LBX_PIC_MINB 2
#endif
// Gather of one component: from the quad copy (one 16-byte load) or, when
// the particles are too sparse for the copy to pay (kQuad = false: each
// node's quad would be fetched from HBM for a handful of particles), from
// the field array itself (four 4-byte loads, 4x less gathered footprint).
template <bool kQuad, bool kFast = false>
__device__ __forceinline__ float gather_c(const PicParams& p, int c, int i0, int j0, float fz,
                                          float fx) {
  float4 q;
  if (kQuad) {
    q = __ldg(p.Q[c] + (i0 + 1) * p.qpitch + (j0 + 1));
  } else {
    const float* F = p.F[c] + (i0 + 1) * p.pitch + (j0 + 1);
    q = make_float4(__ldg(F), __ldg(F + 1), __ldg(F + p.pitch), __ldg(F + p.pitch + 1));
  }
  return kFast ? cic_fast(q, fz, fx) : cic(q, fz, fx);
}

// MUFU approximations (<= 2 ulp; arguments are >= 1 here, so flushing
// denormals never applies): one instruction each instead of the IEEE
// sequences of rsqrtf / __frcp_rn.
__device__ __forceinline__ float rsqrt_approx(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Tolerance-mode relativistic Boris (LBX_PIC_FAST).  The rotation is
// evaluated in float32 (FMA, MUFU rsqrt / rcp) but only as the INCREMENT
// du = u_new - u = 2 hE + (u- x t) + s (u' x t), which is added to the
// float64 momenta; the new 1/gamma is float32 too.  Error: float32 rounding
// of du (not of u) -- see oracle/pic_oracle.py boris_fast and the tolerance
// tests.  Returns 1/gamma(u_new) in float32.
__device__ __forceinline__ float boris_fast(double& ux, double& uy, double& uz, float hf,
                                            float Ex, float Ey, float Ez, float Bx, float By,
                                            float Bz) {
  const float hEx = hf * Ex, hEy = hf * Ey, hEz = hf * Ez;
  const float mx = __fadd_rn((float)ux, hEx), my = __fadd_rn((float)uy, hEy),
              mz = __fadd_rn((float)uz, hEz);
  const float ig = rsqrt_approx(__fmaf_rn(mz, mz, __fmaf_rn(my, my, __fmaf_rn(mx, mx, 1.f))));
  const float tx = hf * Bx * ig, ty = hf * By * ig, tz = hf * Bz * ig;
  const float sr = rcp_approx(__fmaf_rn(tz, tz, __fmaf_rn(ty, ty, __fmaf_rn(tx, tx, 1.f))));
  const float s2 = 2.f * sr;
  // u' - u- = u- x t ; u+ - u- = s (u' x t)
  const float cx = __fmaf_rn(my, tz, -mz * ty), cy = __fmaf_rn(mz, tx, -mx * tz),
              cz = __fmaf_rn(mx, ty, -my * tx);
  const float px = mx + cx, py = my + cy, pz = mz + cz;
  const float rx = s2 * __fmaf_rn(py, tz, -pz * ty), ry = s2 * __fmaf_rn(pz, tx, -px * tz),
              rz = s2 * __fmaf_rn(px, ty, -py * tx);
  ux = __dadd_rn(ux, (double)(__fmaf_rn(2.f, hEx, rx)));
  uy = __dadd_rn(uy, (double)(__fmaf_rn(2.f, hEy, ry)));
  uz = __dadd_rn(uz, (double)(__fmaf_rn(2.f, hEz, rz)));
  const float fx = (float)ux, fy = (float)uy, fz = (float)uz;
  return rsqrt_approx(__fmaf_rn(fz, fz, __fmaf_rn(fy, fy, __fmaf_rn(fx, fx, 1.f))));
}

// Tolerance mode (LBX_PIC_FAST): cell by truncation, fraction rounded to
// float32 once (the exact mode's axis_of floors in fp64 and rounds twice).
__device__ __forceinline__ Axis fast_axis(double v) {
  Axis a;
  a.i = __double2int_rz(v);                       // v >= 0 inside the grid: trunc == floor
  a.f = __double2float_rn(__dsub_rn(v, (double)a.i));
  a.hi = a.f >= 0.5f;
  a.ih = a.hi ? a.i : a.i - 1;
  a.fh = __fadd_rn(a.f, a.hi ? -0.5f : 0.5f);
  return a;
}

template <bool kFast>
__device__ __forceinline__ Axis pic_axis(double v) {
  return kFast ? fast_axis(v) : axis_of(v);
}

template <bool kQuad>
__device__ __forceinline__ float fast_gather(const float4 q, float fz, float fx) {
  return kQuad ? cic_diff(q, fz, fx) : cic_fast(q, fz, fx);
}

// One component's 2x2 node quad at a precomputed node offset (quad copy or
// the field array itself).
template <bool kQuad>
__device__ __forceinline__ float4 quad_at(const PicParams& p, int c, int off) {
  if (kQuad) return __ldg(p.Q[c] + off);
  const float* F = p.F[c] + off;
  return make_float4(__ldg(F), __ldg(F + 1), __ldg(F + p.pitch), __ldg(F + p.pitch + 1));
}

// Per-CTA state shared by the push kernels' prologue / epilogue.
struct PushShared {
  long long n;
  int box[4];
  int last;
  unsigned long long red[kPW];
  long long min[kPW];
};

template <bool kClock>
__device__ __forceinline__ void push_prologue(const PicParams& p, PushShared& sh, unsigned* s_cnt,
                                              unsigned* s_clk) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh.n = *((volatile long long*)&p.st->n);
    sh.box[0] = INT_MAX;
    sh.box[1] = INT_MIN;
    sh.box[2] = INT_MAX;
    sh.box[3] = INT_MIN;
  }
  for (int b = tid; b < p.nb; b += kPB) {
    s_cnt[b] = 0u;
    if (kClock) s_clk[b] = 0u;
  }
  __syncthreads();
}

// CTA totals (removed count, first removed slot, errors, deposit bounding
// box), histogram flush, and the last CTA's step record.
template <bool kClock>
__device__ __forceinline__ void push_epilogue(const PicParams& p, PushShared& sh, long long n,
                                              unsigned long long removed, long long first_out,
                                              long long err, int bimin, int bimax, int bjmin,
                                              int bjmax, const unsigned* s_cnt,
                                              const unsigned* s_clk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long wa = (unsigned long long)warp_sum((long long)removed);
  const long long wm = warp_min(first_out), we = warp_sum((long long)err);
  const int wimin = __reduce_min_sync(kAll, bimin), wimax = __reduce_max_sync(kAll, bimax);
  const int wjmin = __reduce_min_sync(kAll, bjmin), wjmax = __reduce_max_sync(kAll, bjmax);
  if (lane == 0) {
    sh.red[warp] = wa;
    sh.min[warp] = wm;
    if (we) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)we);
    if (wimin <= wimax) {
      atomicMin(&sh.box[0], wimin);
      atomicMax(&sh.box[1], wimax);
      atomicMin(&sh.box[2], wjmin);
      atomicMax(&sh.box[3], wjmax);
    }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long ta = 0;
    long long tm = LLONG_MAX;
    for (int w = 0; w < kPW; ++w) {
      ta += sh.red[w];
      tm = min(tm, sh.min[w]);
    }
    if (ta) {
      atomicAdd(&p.st->leavers, ta);
      atomicMin(&p.st->first_leaver, tm);
    }
    if (sh.box[0] <= sh.box[1]) {
      atomicMin(p.dep_box + 0, sh.box[0]);
      atomicMax(p.dep_box + 1, sh.box[1]);
      atomicMin(p.dep_box + 2, sh.box[2]);
      atomicMax(p.dep_box + 3, sh.box[3]);
    }
  }
  for (int b = tid; b < p.nb; b += kPB) {
    if (s_cnt[b]) atomicAdd(p.g_cnt + b, (unsigned long long)s_cnt[b]);
    if (kClock && s_clk[b]) atomicAdd(p.g_clk + b, (unsigned long long)s_clk[b]);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) sh.last = (atomicAdd(&p.st->done, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!sh.last) return;
  __threadfence();
  step_record<kClock>(p.g_cnt, p.g_clk, p.nb, p.counts_out, p.cost_out, p.clk_out, p.wp, p.wc,
                      p.cells, 4);
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

// kFast: tolerance mode (LBX_PIC_FAST) -- fast_axis, FMA gathers, float32
// Boris increment (boris_fast); same work structure, not bit-exact.
template <bool kClock, bool kSort, bool kQuad, bool kFast = false>
__global__ void __launch_bounds__(kPB, LBX_PIC_MINB) pic_push_kernel(PicParams p) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  FlushEntry* s_q = reinterpret_cast<FlushEntry*>(s_dyn) + (size_t)(threadIdx.x >> 5) * kQCap;
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_dyn + (size_t)kPW * kQCap * sizeof(FlushEntry));  // nb
  unsigned* s_clk = s_cnt + p.nb;                                                                   // nb
  __shared__ PushShared sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  push_prologue<kClock>(p, sh, s_cnt, s_clk);
  const long long n = sh.n;
  const long long units = (n + kUnitP - 1) / kUnitP;
  const double ez = (double)p.nz, ex = (double)p.nx;
  const double h = 0.5 * p.qm * p.dt;
  unsigned removed = 0;                          // per lane: 32 bits (register pressure)
  long long first_out = LLONG_MAX;
  int err = 0;
  int bimin = INT_MAX, bimax = INT_MIN, bjmin = INT_MAX, bjmax = INT_MIN;

  for (long long u = (long long)blockIdx.x * kPW + warp; u < units;
       u += (long long)gridDim.x * kPW) {
    const long long run0 = u * kUnitP + (long long)lane * kRun;
    // deposit accumulator (cell-relative node sums of the lane's current cell;
    // tolerance mode: float run sums)
    int acc[kNodes];
    float accf[kNodes];
#pragma unroll
    for (int i = 0; i < kNodes; ++i) {
      acc[i] = 0;
      accf[i] = 0.f;
    }
    int cur = -1;
    unsigned cur_m = 0;
    // per-box survivor run (+ GpuClock: time since the last box flush)
    int hb = -1;
    unsigned hn = 0;
    long long t_last = 0;
    if (kClock) t_last = clock64();
#pragma unroll 1
    for (int g = 0; g < kRun / kG; ++g) {
      const long long i0 = run0 + g * kG;
      if (__all_sync(kAll, i0 >= n)) break;     // warp-uniform: the queue below is warp-collective
      double pz[kG], px[kG], puz[kG], pux[kG], puy[kG];
      ldg(p.z, i0, n, pz);
      ldg(p.x, i0, n, px);
      ldg(p.uz, i0, n, puz);
      ldg(p.ux, i0, n, pux);
      ldg(p.uy, i0, n, puy);
      // ---- phase 0: old cells; sort-on-write destinations (one cursor
      // atomic per run of equal old cells within the group) ----
      // (the cursor atomics' results are consumed only at the store)
      unsigned base[kG];
      bool seg_start[kG];
      if (kSort) {
        int okey[kG];
#pragma unroll
        for (int k = 0; k < kG; ++k) okey[k] = (int)pz[k] * p.nx + (int)px[k];   // z, x >= 0
#pragma unroll
        for (int k = 0; k < kG; ++k) {
          seg_start[k] = i0 + k < n && (k == 0 || okey[k] != okey[k - 1]);
          int len = 0;
          bool same = true;
#pragma unroll
          for (int j = k; j < kG; ++j) {
            same = same && i0 + j < n && okey[j] == okey[k];
            len += same ? 1 : 0;
          }
          base[k] = seg_start[k] ? atomicAdd(p.cursor + okey[k], (unsigned)len) : 0u;
        }
      }
      // ---- phase 1: gather, Boris, move, absorb ----
      bool keep[kG];
      int nkey[kG];
      float vsx[kG], vsy[kG], vsz[kG];
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        const Axis az = pic_axis<kFast>(pz[k]), ax = pic_axis<kFast>(px[k]);
        if (kFast) {
          // the four stagger combinations' node offsets, computed once
          const int pit = kQuad ? p.qpitch : p.pitch;
          const int rA = (az.i + 1) * pit, rH = (az.ih + 1) * pit, cA = ax.i + 1, cH = ax.ih + 1;
          const float Ex = fast_gather<kQuad>(quad_at<kQuad>(p, 0, rA + cH), az.f, ax.fh);
          const float Ey = fast_gather<kQuad>(quad_at<kQuad>(p, 1, rA + cA), az.f, ax.f);
          const float Ez = fast_gather<kQuad>(quad_at<kQuad>(p, 2, rH + cA), az.fh, ax.f);
          const float Bx = fast_gather<kQuad>(quad_at<kQuad>(p, 3, rH + cA), az.fh, ax.f);
          const float By = fast_gather<kQuad>(quad_at<kQuad>(p, 4, rH + cH), az.fh, ax.fh);
          const float Bz = fast_gather<kQuad>(quad_at<kQuad>(p, 5, rA + cH), az.f, ax.fh);
          const float ig = boris_fast(pux[k], puy[k], puz[k], (float)h, Ex, Ey, Ez, Bx, By, Bz);
          const float dtg = (float)p.dt * ig;
          pz[k] = __dadd_rn(pz[k], (double)__fmul_rn(dtg, (float)puz[k]));
          px[k] = __dadd_rn(px[k], (double)__fmul_rn(dtg, (float)pux[k]));
          keep[k] = i0 + k < n && pz[k] >= 0.0 && pz[k] < ez && px[k] >= 0.0 && px[k] < ex;
          nkey[k] = keep[k] ? __double2int_rz(pz[k]) * p.nx + __double2int_rz(px[k]) : -1;
          const float qv = keep[k] ? __fmul_rn((float)p.qw * p.vscale, ig) : 0.f;
          vsx[k] = __fmul_rn(qv, (float)pux[k]);
          vsy[k] = __fmul_rn(qv, (float)puy[k]);
          vsz[k] = __fmul_rn(qv, (float)puz[k]);
          continue;
        }
        // staggers: (0, 1/2) Ex Bz | (0, 0) Ey | (1/2, 0) Ez Bx | (1/2, 1/2) By
        const float Ex = gather_c<kQuad>(p, 0, az.i, ax.ih, az.f, ax.fh);
        const float Ey = gather_c<kQuad>(p, 1, az.i, ax.i, az.f, ax.f);
        const float Ez = gather_c<kQuad>(p, 2, az.ih, ax.i, az.fh, ax.f);
        const float Bx = gather_c<kQuad>(p, 3, az.ih, ax.i, az.fh, ax.f);
        const float By = gather_c<kQuad>(p, 4, az.ih, ax.ih, az.fh, ax.fh);
        const float Bz = gather_c<kQuad>(p, 5, az.i, ax.ih, az.f, ax.fh);
        // relativistic Boris (x, y, z order; oracle boris())
        const double hEx = __dmul_rn(h, (double)Ex), hEy = __dmul_rn(h, (double)Ey),
                     hEz = __dmul_rn(h, (double)Ez);
        const double mx = __dadd_rn(pux[k], hEx);
        const double my = __dadd_rn(puy[k], hEy);
        const double mz = __dadd_rn(puz[k], hEz);
        const double gg = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(mx, mx)),
                                                         __dmul_rn(my, my)), __dmul_rn(mz, mz)));
        const double ig = __drcp_rn(gg);                 // == 1.0 / g (correctly rounded)
        const double tx = __dmul_rn(__dmul_rn(h, (double)Bx), ig);
        const double ty = __dmul_rn(__dmul_rn(h, (double)By), ig);
        const double tz = __dmul_rn(__dmul_rn(h, (double)Bz), ig);
        // 2 / d == 2 * RN(1/d) exactly (power-of-two scaling of a normal number)
        const double s2 = __dmul_rn(2.0, __drcp_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(tx, tx)),
                                                                       __dmul_rn(ty, ty)),
                                                             __dmul_rn(tz, tz))));
        const double qx = __dadd_rn(mx, __dsub_rn(__dmul_rn(my, tz), __dmul_rn(mz, ty)));
        const double qy = __dadd_rn(my, __dsub_rn(__dmul_rn(mz, tx), __dmul_rn(mx, tz)));
        const double qz = __dadd_rn(mz, __dsub_rn(__dmul_rn(mx, ty), __dmul_rn(my, tx)));
        pux[k] = __dadd_rn(__dadd_rn(mx, __dmul_rn(s2, __dsub_rn(__dmul_rn(qy, tz), __dmul_rn(qz, ty)))), hEx);
        puy[k] = __dadd_rn(__dadd_rn(my, __dmul_rn(s2, __dsub_rn(__dmul_rn(qz, tx), __dmul_rn(qx, tz)))), hEy);
        puz[k] = __dadd_rn(__dadd_rn(mz, __dmul_rn(s2, __dsub_rn(__dmul_rn(qx, ty), __dmul_rn(qy, tx)))), hEz);
        const double gam = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(pux[k], pux[k])),
                                                          __dmul_rn(puy[k], puy[k])),
                                                __dmul_rn(puz[k], puz[k])));
        const double igam = __drcp_rn(gam);
        pz[k] = __dadd_rn(pz[k], __dmul_rn(__dmul_rn(p.dt, puz[k]), igam));
        px[k] = __dadd_rn(px[k], __dmul_rn(__dmul_rn(p.dt, pux[k]), igam));
        keep[k] = i0 + k < n && pz[k] >= 0.0 && pz[k] < ez && px[k] >= 0.0 && px[k] < ex;
        nkey[k] = keep[k] ? (int)pz[k] * p.nx + (int)px[k] : -1;   // positions >= 0: trunc == floor
        const double qwg = keep[k] ? p.qw : 0.0;
        vsx[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, pux[k]), igam)), p.vscale);
        vsy[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puy[k]), igam)), p.vscale);
        vsz[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puz[k]), igam)), p.vscale);
      }
      // ---- phase 3: store (in place, or scattered to the sorted slots) ----
      long long dest[kG];
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        if (kSort) dest[k] = seg_start[k] ? (long long)base[k] : (k ? dest[k - 1] + 1 : 0);
        else dest[k] = i0 + k;
        if (i0 + k < n && !keep[k]) {
          ++removed;
          first_out = min(first_out, dest[k]);
          if (p.removed_list) {   // order not kept: O(removed) hole filling
            const unsigned long long slot = atomicAdd(&p.st->removed_count, 1ull);
            if ((long long)slot < p.removed_cap) p.removed_list[slot] = dest[k];
          }
        }
      }
      if (kSort) {
#pragma unroll
        for (int k = 0; k < kG; ++k) {
          if (i0 + k >= n) continue;
          const long long d = dest[k];
          if (d >= n) {       // offsets inconsistent with the particles: refuse to scatter
            ++err;
            continue;
          }
          __stcs(p.oz + d, pz[k]);
          __stcs(p.ox + d, px[k]);
          __stcs(p.ouz + d, puz[k]);
          __stcs(p.oux + d, pux[k]);
          __stcs(p.ouy + d, puy[k]);
        }
      } else {
        stg(p.oz, i0, n, pz);
        stg(p.ox, i0, n, px);
        stg(p.ouz, i0, n, puz);
        stg(p.oux, i0, n, pux);
        stg(p.ouy, i0, n, puy);
      }
      // ---- phase 2: current.  Accumulate in registers while consecutive
      // particles share a cell; an isolated particle in another cell (drift)
      // is queued directly; otherwise the finished cell is queued and the
      // lane switches cells.  The queue drains once per group. ----
      const unsigned lt = (1u << lane) - 1u;
      int qn = 0;
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        const bool dep = nkey[k] >= 0;
        const Axis az = pic_axis<kFast>(dep ? pz[k] : 0.5), ax = pic_axis<kFast>(dep ? px[k] : 0.5);
        const bool same = dep && nkey[k] == cur;
        const bool strag = dep && !same && cur >= 0 && k + 1 < kG && nkey[k + 1] != nkey[k];
        const bool swap = dep && !same && !strag;
        const bool need = strag || (swap && cur >= 0);
        const unsigned fm = __ballot_sync(kAll, need);
        if (kFast) {
          if (need) {
            FlushEntry* e = s_q + qn + __popc(fm & lt);
            if (strag) {
              float w[kNodes];
#pragma unroll
              for (int i = 0; i < kNodes; ++i) w[i] = 0.f;
              node_accum(az, ax, vsx[k], vsy[k], vsz[k], w);
              enqueue_f(e, w, nkey[k], 1u);
            } else {
              enqueue_f(e, accf, cur, cur_m);
            }
          }
          qn += __popc(fm);
          if (kQCap < 32 * kG && qn > kQCap - 32) {
            drain_queue<kSort, kFast>(p, s_q, qn, lane);
            qn = 0;
          }
          if (__any_sync(kAll, swap)) {   // rare (cell changes): keep the 16 resets off the common path
            if (swap) {
#pragma unroll
              for (int i = 0; i < kNodes; ++i) accf[i] = 0.f;
              cur = nkey[k];
              cur_m = 0;
            }
          }
          if (same || swap) {
            node_accum(az, ax, vsx[k], vsy[k], vsz[k], accf);
            ++cur_m;
          }
        } else {
          int q[kNodes];
          node_values(az, ax, vsx[k], vsy[k], vsz[k], q);   // v = 0 -> q = 0 off-deposit
          if (need)
            enqueue(s_q + qn + __popc(fm & lt), strag ? q : acc, strag ? nkey[k] : cur,
                    strag ? 1u : cur_m);
          qn += __popc(fm);
          if (kQCap < 32 * kG && qn > kQCap - 32) {   // small queue: drain mid-group
            drain_queue<kSort>(p, s_q, qn, lane);
            qn = 0;
          }
          if (same) {
#pragma unroll
            for (int i = 0; i < kNodes; ++i) acc[i] += q[i];
            ++cur_m;
          } else if (swap) {
#pragma unroll
            for (int i = 0; i < kNodes; ++i) acc[i] = q[i];
            cur = nkey[k];
            cur_m = 1;
          }
        }
        if (!dep) continue;
        bimin = min(bimin, az.i);
        bimax = max(bimax, az.i);
        bjmin = min(bjmin, ax.i);
        bjmax = max(bjmax, ax.i);
        // per-box survivor counts (+ clock): run-length per lane
        const int bz = az.i >> p.log2m, bx = ax.i >> p.log2m;
        if (bz >= p.nbz || bx >= p.nbx) {
          ++err;
        } else if (bz * p.nbx + bx == hb) {
          ++hn;
        } else {
          if (hb >= 0) {
            atomicAdd(s_cnt + hb, hn);
            if (kClock) {
              const long long t = clock64();
              atomicAdd(s_clk + hb, (unsigned)min((t - t_last) >> 4, (long long)(1u << 30)));
              t_last = t;
            }
          }
          hb = bz * p.nbx + bx;
          hn = 1;
        }
      }
      if (qn) drain_queue<kSort, kFast>(p, s_q, qn, lane);
    }
    {   // end of the lane's run: queue its open cell, drain
      const unsigned fm = __ballot_sync(kAll, cur >= 0);
      if (cur >= 0) {
        FlushEntry* e = s_q + __popc(fm & ((1u << lane) - 1u));
        if (kFast) enqueue_f(e, accf, cur, cur_m);
        else enqueue(e, acc, cur, cur_m);
      }
      if (fm) drain_queue<kSort, kFast>(p, s_q, __popc(fm), lane);
    }
    // last box run of the lane: warp-uniform fast path (one shared atomic)
    unsigned tclk = 0;
    if (kClock && hb >= 0) tclk = (unsigned)min((clock64() - t_last) >> 4, (long long)(1u << 30));
    const int hb0 = __shfl_sync(kAll, hb, 0);
    if (__all_sync(kAll, hb == hb0)) {
      const unsigned tot = __reduce_add_sync(kAll, hn);
      const unsigned clk = kClock ? __reduce_add_sync(kAll, tclk) : 0u;
      if (lane == 0 && hb0 >= 0 && tot) {
        atomicAdd(s_cnt + hb0, tot);
        if (kClock) atomicAdd(s_clk + hb0, clk);
      }
    } else if (hb >= 0 && hn) {
      atomicAdd(s_cnt + hb, hn);
      if (kClock) atomicAdd(s_clk + hb, tclk);
    }
  }

  push_epilogue<kClock>(p, sh, n, removed, first_out, err, bimin, bimax, bjmin, bjmax, s_cnt,
                        s_clk);
}

// ---------------------------------------------------------------------------
// Pipelined tolerance-mode kernel (LBX_PIC_FAST with the quad copy, the dense
// plasma path).  Same arithmetic as pic_push_kernel<.., kFast = true> (the
// tolerance tests hold both), restructured for latency:
//  * particle loads are bulk copies (cp.async.bulk, one mbarrier per warp)
//    of 128-particle chunks into a per-warp shared-memory stage; the warp
//    reads its chunk into registers, then immediately issues the NEXT chunk's
//    copy, so the HBM latency overlaps the chunk's arithmetic instead of
//    stalling the first use of the data (ncu, pic_push_kernel fast mode:
//    11 % of stall samples waiting for the particle loads);
//  * a per-warp quad window in shared memory: the 6 components' quads of a
//    4 x 5 block of nodes around the warp's current cell (1.9 KB), reloaded
//    only when a particle of the warp falls outside it -- a gather is one
//    LDS.128 per component instead of an LDG that misses L1 15 % of the
//    time (22 % of stall samples at the interpolation);
//  * the flush queue is drained after every particle slot (32 entries per
//    warp instead of 128): the smem budget goes to the stage and the window
//    while keeping 2 CTAs x 8 warps per SM.
// Lane L of a chunk owns particles {2L, 2L+1, 64+2L, 64+2L+1}: conflict-free
// LDS.128 / coalesced STG.128; a lane's run state (current cell, float node
// sums, box run, clock) persists across the chunks of a unit as before.
#ifndef LBX_PIC_PIPE
#define LBX_PIC_PIPE 1                         // 0: fast mode runs pic_push_kernel (A/B builds)
#endif
constexpr int kChunk = 128;                    // particles per warp chunk
constexpr int kChunks = kUnitP / kChunk;       // chunks per warp unit
constexpr int kQCapP = 64;                     // flush entries per warp (drained every 2 slots)
constexpr int kWinR = 4, kWinC = 5;            // quad window: rows wi-2..wi+1, cols wj-2..wj+2
constexpr int kWin = kWinR * kWinC;

template <bool kFast>
__device__ __forceinline__ float pipe_cic(const float4 q, float fz, float fx) {
  return kFast ? cic_diff(q, fz, fx) : cic(q, fz, fx);   // difference quads / raw quads
}

// The exact relativistic Boris of pic_push_kernel (x, y, z order; oracle
// boris()): updates u in place, returns 1/gamma(u_new) correctly rounded.
__device__ __forceinline__ double boris_exact(double& ux, double& uy, double& uz, double h,
                                              float Ex, float Ey, float Ez, float Bx, float By,
                                              float Bz) {
  const double hEx = __dmul_rn(h, (double)Ex), hEy = __dmul_rn(h, (double)Ey),
               hEz = __dmul_rn(h, (double)Ez);
  const double mx = __dadd_rn(ux, hEx);
  const double my = __dadd_rn(uy, hEy);
  const double mz = __dadd_rn(uz, hEz);
  const double gg = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(mx, mx)),
                                                   __dmul_rn(my, my)), __dmul_rn(mz, mz)));
  const double ig = __drcp_rn(gg);
  const double tx = __dmul_rn(__dmul_rn(h, (double)Bx), ig);
  const double ty = __dmul_rn(__dmul_rn(h, (double)By), ig);
  const double tz = __dmul_rn(__dmul_rn(h, (double)Bz), ig);
  const double s2 = __dmul_rn(2.0, __drcp_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(tx, tx)),
                                                                 __dmul_rn(ty, ty)),
                                                       __dmul_rn(tz, tz))));
  const double qx = __dadd_rn(mx, __dsub_rn(__dmul_rn(my, tz), __dmul_rn(mz, ty)));
  const double qy = __dadd_rn(my, __dsub_rn(__dmul_rn(mz, tx), __dmul_rn(mx, tz)));
  const double qz = __dadd_rn(mz, __dsub_rn(__dmul_rn(mx, ty), __dmul_rn(my, tx)));
  ux = __dadd_rn(__dadd_rn(mx, __dmul_rn(s2, __dsub_rn(__dmul_rn(qy, tz), __dmul_rn(qz, ty)))), hEx);
  uy = __dadd_rn(__dadd_rn(my, __dmul_rn(s2, __dsub_rn(__dmul_rn(qz, tx), __dmul_rn(qx, tz)))), hEy);
  uz = __dadd_rn(__dadd_rn(mz, __dmul_rn(s2, __dsub_rn(__dmul_rn(qx, ty), __dmul_rn(qy, tx)))), hEz);
  const double gam = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(ux, ux)),
                                                    __dmul_rn(uy, uy)),
                                          __dmul_rn(uz, uz)));
  return __drcp_rn(gam);
}

struct __align__(16) PipeWarp {
  double stage[5][kChunk];                     // z x uz ux uy
  FlushEntry q[kQCapP];
  float4 win[6][kWin];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Whole warp, warp-uniform arguments: one elected lane bulk-copies particles
// [base, base + cnt) of the five arrays into the warp's stage (sizes rounded
// up to whole 16-byte pairs: arrays have n + 2 slots), completion counted on
// the warp's mbarrier.  (Called from uniform code with uniform operands the
// copies compile to uniform-datapath UBLKCPs, ~5x fewer instructions than
// from a lane-0 branch, where each operand goes through an elect loop.)
__device__ __forceinline__ void pipe_issue(const PicParams& p, PipeWarp* w, unsigned long long* bar,
                                           long long base, long long n) {
  const long long cnt = min((long long)kChunk, n - base);
  const unsigned bytes = (unsigned)((cnt + 1) & ~1ll) * 8u;
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "r"(5u * bytes)
      : "memory");
  const double* src[5] = {p.z, p.x, p.uz, p.ux, p.uy};
#pragma unroll
  for (int a = 0; a < 5; ++a)
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::
            "r"(smem_u32(w->stage[a])), "l"(src[a] + base), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Reload the warp's quad window around cell (ci, cj).
__device__ __forceinline__ void pipe_window(const PicParams& p, PipeWarp* w, int ci, int cj,
                                            int lane) {
  __syncwarp();
  for (int t = lane; t < 6 * kWin; t += 32) {
    const int c = t / kWin, r = (t % kWin) / kWinC, k = t % kWinC;
    const int row = min(max(ci - 2 + r, -1), p.nz - 1), col = min(max(cj - 2 + k, -1), p.nx - 1);
    w->win[c][r * kWinC + k] = __ldg(p.Q[c] + (row + 1) * p.qpitch + (col + 1));
  }
  __syncwarp();
}

#ifndef LBX_PIPE_ROLL
#define LBX_PIPE_ROLL 1   // exact pipe kernel: rolled slot loop (see below)
#endif
#ifndef LBX_PIPE_ROLL_FAST
#define LBX_PIPE_ROLL_FAST 0
#endif
template <typename T, int N>
__device__ __forceinline__ void rot(T (&a)[N]) {
  const T t = a[0];
#pragma unroll
  for (int i = 0; i + 1 < N; ++i) a[i] = a[i + 1];
  a[N - 1] = t;
}

// kFast = false: the exact (bit-exact) step with the same pipeline -- fp64
// Boris, floor axes, float32 CIC on raw quads, integer node values.
template <bool kClock, bool kFast = true>
__global__ void __launch_bounds__(kPB, LBX_PIC_MINB) pic_pipe_kernel(PicParams p) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  // warp index and count through a shuffle: warp-uniform for the compiler,
  // so the bulk copies' operands live in uniform registers
  const int warp = __shfl_sync(kAll, (int)(threadIdx.x >> 5), 0);
  PipeWarp* w = reinterpret_cast<PipeWarp*>(s_dyn) + warp;
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_dyn + (size_t)kPW * sizeof(PipeWarp));  // nb
  unsigned* s_clk = s_cnt + p.nb;                                                         // nb
  __shared__ PushShared sh;
  __shared__ unsigned long long s_bar[kPW];
  const int lane = threadIdx.x & 31;
  unsigned long long* bar = s_bar + warp;
  if (lane == 0) mbar_init(bar);
  push_prologue<kClock>(p, sh, s_cnt, s_clk);     // (its barrier publishes the mbarrier init)
  const long long n = __shfl_sync(kAll, sh.n, 0);
  const long long units = (n + kUnitP - 1) / kUnitP;
  const long long ustride = (long long)gridDim.x * kPW;
  const float hf = (float)(0.5 * p.qm * p.dt), dtf = (float)p.dt;
  const float qws = (float)p.qw * p.vscale;
  const double h = 0.5 * p.qm * p.dt;
  unsigned removed = 0;                          // per lane: 32 bits (register pressure)
  long long first_out = LLONG_MAX;
  int err = 0;
  int bimin = INT_MAX, bimax = INT_MIN, bjmin = INT_MAX, bjmax = INT_MIN;
  int wi = INT_MIN / 2, wj = INT_MIN / 2;        // window centre (none loaded)
  unsigned phase = 0;
  const unsigned lt = (1u << lane) - 1u;
  // my four slots in a chunk
  const int slot0 = kG * lane;                  // my slots: kG consecutive particles
  constexpr bool kRoll = LBX_PIPE_ROLL && (!kFast || LBX_PIPE_ROLL_FAST);
  constexpr bool kRoll2 = LBX_PIPE_ROLL >= 2 && (!kFast || LBX_PIPE_ROLL_FAST);   // the deposit loop too

  long long u = (long long)blockIdx.x * kPW + warp;
  if (u < units) pipe_issue(p, w, bar, u * kUnitP, n);
  for (; u < units; u += ustride) {
    float accf[kNodes];
    int acc[kNodes];
#pragma unroll
    for (int i = 0; i < kNodes; ++i) {
      accf[i] = 0.f;
      acc[i] = 0;
    }
    int cur = -1;
    unsigned cur_m = 0;
    int hb = -1;
    unsigned hn = 0;
    long long t_last = 0;
    if (kClock) t_last = clock64();
#pragma unroll 1
    for (int c = 0; c < kChunks; ++c) {
      const long long base = u * kUnitP + (long long)c * kChunk;
      if (base >= n) break;                      // warp-uniform
      mbar_wait(bar, phase);
      phase ^= 1u;
      double pz[kG], px[kG], puz[kG], pux[kG], puy[kG];
      {
        const double2* s2[5];
#pragma unroll
        for (int a = 0; a < 5; ++a) s2[a] = reinterpret_cast<const double2*>(w->stage[a]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int o = 2 * lane + h;            // pair index: slots 2o, 2o + 1 (2-way bank conflict)
          const double2 a0 = s2[0][o], a1 = s2[1][o], a2 = s2[2][o], a3 = s2[3][o], a4 = s2[4][o];
          pz[2 * h] = a0.x; pz[2 * h + 1] = a0.y;
          px[2 * h] = a1.x; px[2 * h + 1] = a1.y;
          puz[2 * h] = a2.x; puz[2 * h + 1] = a2.y;
          pux[2 * h] = a3.x; pux[2 * h + 1] = a3.y;
          puy[2 * h] = a4.x; puy[2 * h + 1] = a4.y;
        }
      }
      // stage consumed: refill it now.  The lanes' shared-memory reads
      // (generic proxy) must be performed before the bulk copy (async proxy)
      // overwrites the stage: proxy fence per lane, then the warp barrier
      // orders every lane's reads before the elected lane's copy (without
      // it a copy could land before a read -- garbage particles, seen as an
      // illegal address on a 2048^2 sparse plasma).
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      {
        long long nb2 = base + kChunk;
        if (c + 1 == kChunks || nb2 >= n) nb2 = (u + ustride) * kUnitP;
        if (nb2 < n) pipe_issue(p, w, bar, nb2, n);
      }
      const bool full = base + kChunk <= n;      // warp-uniform: every slot live
      const int lim = full ? kChunk : (int)(n - base);
      int nkey[kG];
      float vsx[kG], vsy[kG], vsz[kG];
      // gather + push + move of one slot.  kRoll (exact mode): one copy of
      // the body in a rolled loop over slot 0, the slot arrays rotated after
      // each pass, so the kernel's hot loop fits the instruction cache.
      auto slot = [&](const int k, const int K) {
        const bool vk = slot0 + k < lim;
        const Axis az = pic_axis<kFast>(vk ? pz[K] : 0.5),
                   ax = pic_axis<kFast>(vk ? px[K] : 0.5);
        // the window: rows wi-2..wi+1 and cols wj-2..wj+2 hold every quad of
        // a particle in cells [wi-1, wi+1] x [wj-1, wj+2]
        const bool hit = !vk || ((unsigned)(az.i - wi + 1) <= 2u && (unsigned)(ax.i - wj + 1) <= 3u);
        unsigned miss = __ballot_sync(kAll, !hit);
        if (miss) {   // recentre so the window starts at the warp's lowest row / column, if it then covers the warp
          const int ci = __reduce_min_sync(kAll, vk ? az.i : INT_MAX) + 1;
          const int cj = __reduce_min_sync(kAll, vk ? ax.i : INT_MAX) + 1;
          const bool h2 = !vk || ((unsigned)(az.i - ci + 1) <= 2u && (unsigned)(ax.i - cj + 1) <= 3u);
          if (__all_sync(kAll, h2)) {
            wi = ci;
            wj = cj;
            pipe_window(p, w, wi, wj, lane);
            miss = 0u;
          }
        }
        float Ex, Ey, Ez, Bx, By, Bz;
        if (!miss) {
          // (a slot past the end of the array reads entry 0: its cell is not
          // in the window, and a shared read outside the CTA faults)
          const int rA = vk ? (az.i - wi + 2) * kWinC : 0;
          const int rH = vk ? (az.ih - wi + 2) * kWinC : 0;
          const int cA = vk ? ax.i - wj + 2 : 0, cH = vk ? ax.ih - wj + 2 : 0;
          Ex = pipe_cic<kFast>(w->win[0][rA + cH], az.f, ax.fh);
          Ey = pipe_cic<kFast>(w->win[1][rA + cA], az.f, ax.f);
          Ez = pipe_cic<kFast>(w->win[2][rH + cA], az.fh, ax.f);
          Bx = pipe_cic<kFast>(w->win[3][rH + cA], az.fh, ax.f);
          By = pipe_cic<kFast>(w->win[4][rH + cH], az.fh, ax.fh);
          Bz = pipe_cic<kFast>(w->win[5][rA + cH], az.f, ax.fh);
        } else {                                 // lanes span more than the window
          const int pit = p.qpitch;
          const int rA = (az.i + 1) * pit, rH = (az.ih + 1) * pit, cA = ax.i + 1, cH = ax.ih + 1;
          Ex = pipe_cic<kFast>(__ldg(p.Q[0] + rA + cH), az.f, ax.fh);
          Ey = pipe_cic<kFast>(__ldg(p.Q[1] + rA + cA), az.f, ax.f);
          Ez = pipe_cic<kFast>(__ldg(p.Q[2] + rH + cA), az.fh, ax.f);
          Bx = pipe_cic<kFast>(__ldg(p.Q[3] + rH + cA), az.fh, ax.f);
          By = pipe_cic<kFast>(__ldg(p.Q[4] + rH + cH), az.fh, ax.fh);
          Bz = pipe_cic<kFast>(__ldg(p.Q[5] + rA + cH), az.f, ax.fh);
        }
        if (kFast) {
          const float ig = boris_fast(pux[K], puy[K], puz[K], hf, Ex, Ey, Ez, Bx, By, Bz);
          const float dtg = dtf * ig;
          pz[K] = __dadd_rn(pz[K], (double)__fmul_rn(dtg, (float)puz[K]));
          px[K] = __dadd_rn(px[K], (double)__fmul_rn(dtg, (float)pux[K]));
          // inside iff z, x >= 0 and trunc(z) < nz, trunc(x) < nx (integer extents)
          const int iz = __double2int_rz(pz[K]), ix = __double2int_rz(px[K]);
          const bool kp = vk && pz[K] >= 0.0 && px[K] >= 0.0 && iz < p.nz && ix < p.nx;
          nkey[K] = kp ? iz * p.nx + ix : -1;
          const float qv = kp ? __fmul_rn(qws, ig) : 0.f;
          vsx[K] = __fmul_rn(qv, (float)pux[K]);
          vsy[K] = __fmul_rn(qv, (float)puy[K]);
          vsz[K] = __fmul_rn(qv, (float)puz[K]);
        } else {
          const double igam = boris_exact(pux[K], puy[K], puz[K], h, Ex, Ey, Ez, Bx, By, Bz);
          pz[K] = __dadd_rn(pz[K], __dmul_rn(__dmul_rn(p.dt, puz[K]), igam));
          px[K] = __dadd_rn(px[K], __dmul_rn(__dmul_rn(p.dt, pux[K]), igam));
          const int iz = __double2int_rz(pz[K]), ix = __double2int_rz(px[K]);
          const bool kp = vk && pz[K] >= 0.0 && px[K] >= 0.0 && iz < p.nz && ix < p.nx;
          nkey[K] = kp ? iz * p.nx + ix : -1;
          const double qwg = kp ? p.qw : 0.0;
          vsx[K] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, pux[K]), igam)), p.vscale);
          vsy[K] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puy[K]), igam)), p.vscale);
          vsz[K] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puz[K]), igam)), p.vscale);
        }
      };
      if (kRoll) {
#pragma unroll 1
        for (int k = 0; k < kG; ++k) {
          slot(k, 0);
          rot(pz); rot(px); rot(puz); rot(pux); rot(puy);
          rot(nkey); rot(vsx); rot(vsy); rot(vsz);
        }
      } else {
#pragma unroll
        for (int k = 0; k < kG; ++k) slot(k, k);
      }
      // store in place (one 32-byte group per array), removed bookkeeping
      {
        const long long i = base + slot0;
        if (full) {
          stg(p.oz, i, n, pz);
          stg(p.ox, i, n, px);
          stg(p.ouz, i, n, puz);
          stg(p.oux, i, n, pux);
          stg(p.ouy, i, n, puy);
        } else if (i < n) {
          double* dst[5] = {p.oz, p.ox, p.ouz, p.oux, p.ouy};
          const double* v[5] = {pz, px, puz, pux, puy};
#pragma unroll
          for (int a = 0; a < 5; ++a)
#pragma unroll
            for (int k = 0; k < kG; ++k)
              if (i + k < n) __stcs(dst[a] + i + k, v[a][k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        if (slot0 + k < lim && nkey[k] < 0) {   // a live slot that left the grid
          const long long d = base + slot0 + k;
          ++removed;
          first_out = min(first_out, d);
          if (p.removed_list) {
            const unsigned long long s = atomicAdd(&p.st->removed_count, 1ull);
            if ((long long)s < p.removed_cap) p.removed_list[s] = d;
          }
        }
      }
      // current: register runs per lane, queue drained after every 2 slots.
      // A particle in another cell than the lane's run is queued alone unless
      // the next slot is in that cell too (then the run moves); the chunk's
      // last slot has no look-ahead and always counts as a straggler, so a
      // particle that drifted across a face does not flip the run twice.
      int qn = 0;
      auto deposit = [&](const int k, const int K) {
        const bool dep = nkey[K] >= 0;
        const Axis az = pic_axis<kFast>(dep ? pz[K] : 0.5), ax = pic_axis<kFast>(dep ? px[K] : 0.5);
        int qv[kNodes];
        if (!kFast) node_values(az, ax, vsx[K], vsy[K], vsz[K], qv);   // v = 0 -> q = 0 off-deposit
        const bool same = dep && nkey[K] == cur;
        const bool strag = dep && !same && cur >= 0 && (k + 1 == kG || nkey[K + 1] != nkey[K]);
        const bool swap = dep && !same && !strag;
        const bool need = strag || (swap && cur >= 0);
        const unsigned fm = __ballot_sync(kAll, need);
        if (fm) {
          if (need) {
            FlushEntry* e = w->q + qn + __popc(fm & lt);
            if (!kFast) {
              enqueue(e, strag ? qv : acc, strag ? nkey[K] : cur, strag ? 1u : cur_m);
            } else if (strag) {
              float t[kNodes];
#pragma unroll
              for (int i = 0; i < kNodes; ++i) t[i] = 0.f;
              node_accum(az, ax, vsx[K], vsy[K], vsz[K], t);
              enqueue_f(e, t, nkey[K], 1u);
            } else {
              enqueue_f(e, accf, cur, cur_m);
            }
          }
          qn += __popc(fm);
        }
        if ((k & 1) && qn) {
          drain_queue<false, kFast>(p, w->q, qn, lane);
          qn = 0;
        }
        if (kFast) {
          if (__any_sync(kAll, swap)) {
            if (swap) {
#pragma unroll
              for (int i = 0; i < kNodes; ++i) accf[i] = 0.f;
              cur = nkey[K];
              cur_m = 0;
            }
          }
          if (same || swap) {
            node_accum(az, ax, vsx[K], vsy[K], vsz[K], accf);
            ++cur_m;
          }
        } else if (same) {
#pragma unroll
          for (int i = 0; i < kNodes; ++i) acc[i] += qv[i];
          ++cur_m;
        } else if (swap) {
#pragma unroll
          for (int i = 0; i < kNodes; ++i) acc[i] = qv[i];
          cur = nkey[K];
          cur_m = 1;
        }
        if (!dep) return;
        bimin = min(bimin, az.i);
        bimax = max(bimax, az.i);
        bjmin = min(bjmin, ax.i);
        bjmax = max(bjmax, ax.i);
        const int bz = az.i >> p.log2m, bx = ax.i >> p.log2m;
        if (bz >= p.nbz || bx >= p.nbx) {
          ++err;
        } else if (bz * p.nbx + bx == hb) {
          ++hn;
        } else {
          if (hb >= 0) {
            atomicAdd(s_cnt + hb, hn);
            if (kClock) {
              const long long t = clock64();
              atomicAdd(s_clk + hb, (unsigned)min((t - t_last) >> 4, (long long)(1u << 30)));
              t_last = t;
            }
          }
          hb = bz * p.nbx + bx;
          hn = 1;
        }
      };
      if (kRoll2) {
#pragma unroll 1
        for (int k = 0; k < kG; ++k) {
          deposit(k, 0);
          rot(pz); rot(px); rot(nkey); rot(vsx); rot(vsy); rot(vsz);
        }
      } else {
#pragma unroll
        for (int k = 0; k < kG; ++k) deposit(k, k);
      }
    }
    {   // end of the unit: queue the lane's open cell, drain
      const unsigned fm = __ballot_sync(kAll, cur >= 0);
      if (cur >= 0) {
        if (kFast) enqueue_f(w->q + __popc(fm & lt), accf, cur, cur_m);
        else enqueue(w->q + __popc(fm & lt), acc, cur, cur_m);
      }
      if (fm) drain_queue<false, kFast>(p, w->q, __popc(fm), lane);
    }
    unsigned tclk = 0;
    if (kClock && hb >= 0) tclk = (unsigned)min((clock64() - t_last) >> 4, (long long)(1u << 30));
    const int hb0 = __shfl_sync(kAll, hb, 0);
    if (__all_sync(kAll, hb == hb0)) {
      const unsigned tot = __reduce_add_sync(kAll, hn);
      const unsigned clk = kClock ? __reduce_add_sync(kAll, tclk) : 0u;
      if (lane == 0 && hb0 >= 0 && tot) {
        atomicAdd(s_cnt + hb0, tot);
        if (kClock) atomicAdd(s_clk + hb0, clk);
      }
    } else if (hb >= 0 && hn) {
      atomicAdd(s_cnt + hb, hn);
      if (kClock) atomicAdd(s_clk + hb, tclk);
    }
  }

  push_epilogue<kClock>(p, sh, n, removed, first_out, err, bimin, bimax, bjmin, bjmax, s_cnt,
                        s_clk);
}

// ---------------------------------------------------------------------------
// Tiled in-place mode (LBX_PIC_TILED; sparse plasmas such as SURVEY 8d's
// 8-ppc roofline case).  There the cell-centric accumulator costs 128 B per
// cell per step and the direct gather waits on L2 for 24 scalar loads per
// particle.  lbx_pic_sort with LBX_PIC_TILED orders the particles by a
// tile-major cell key (16 x 16-cell tiles) and records each tile's slot range;
// then, step after step in place, one CTA takes one tile's particles:
//   * the tile's field patch (the tile plus kGd cells of drift margin and the
//     stencil's nodes) is staged in shared memory: a gather is 4 LDS;
//   * lane run sums go through the warp queue into a shared node
//     accumulator (16-bit halves summed by two fire-and-forget 32-bit shared
//     atomics: exact below kSplitMax particles per tile; 64-bit shared
//     atomics are CAS loops), added to the node-centric int64 current Jn
//     once per tile; denser tiles add straight to Jn;
//   * a particle outside the patch (drifted further since the sort, or moved
//     in by hole filling) takes the global path: direct gather, RED into Jn.
// Integer sums are order independent: J is bit-identical to the other modes.
#ifndef LBX_PIC_TILE_LOG2
#define LBX_PIC_TILE_LOG2 4
#endif
constexpr int kTS = LBX_PIC_TILE_LOG2;  // tile edge 2^kTS cells
constexpr int kT = 1 << kTS;
constexpr int kTileShift = 2 * kTS;     // keys per tile
constexpr int kGd = 3;                  // drift margin (cells) around the tile
constexpr int kPP = kT + 2 * kGd + 2;   // patch edge in padded nodes
constexpr int kPatch = kPP * kPP;
#ifndef LBX_PIC_QCAPT
#define LBX_PIC_QCAPT 64
#endif
constexpr int kQCapT = LBX_PIC_QCAPT;   // flush-queue entries per warp (tiled kernel)

__device__ __forceinline__ int tile_key(int i, int j, int ntx) {
  return ((((i >> kTS) * ntx) + (j >> kTS)) << kTileShift) | ((i & (kT - 1)) << kTS) |
         (j & (kT - 1));
}

// cell-relative slot -> node (i + dr, j + ds) of component comp (the
// pic_current_kernel mapping: Jx 2x3, Jy 2x2, Jz 3x2)
__device__ __forceinline__ void slot_node(int sl, int& comp, int& dr, int& ds) {
  if (sl < 6) {
    comp = 0;
    dr = sl >= 3 ? 1 : 0;
    ds = sl - 3 * dr - 1;
  } else if (sl < 10) {
    comp = 1;
    dr = (sl - 6) >> 1;
    ds = (sl - 6) & 1;
  } else {
    comp = 2;
    dr = ((sl - 10) >> 1) - 1;
    ds = (sl - 10) & 1;
  }
}

// every node a gather or deposit of cell (i, j) touches lies in the patch of
// the tile with origin (tz, tx)
__device__ __forceinline__ bool in_patch(int i, int j, int tz, int tx) {
  return (unsigned)(i - tz + kGd) <= (unsigned)(kT - 1 + 2 * kGd) &&
         (unsigned)(j - tx + kGd) <= (unsigned)(kT - 1 + 2 * kGd);
}

// local patch index of the padded node (P, Q)
__device__ __forceinline__ int patch_at(int P, int Q, int tz, int tx) {
  return (P - tz + kGd) * kPP + (Q - tx + kGd);
}

template <bool kFast = false>
__device__ __forceinline__ float gather_s(const float* s_f, int c, int i0, int j0, float fz,
                                          float fx, int tz, int tx) {
  const float* F = s_f + c * kPatch + patch_at(i0 + 1, j0 + 1, tz, tx);
  const float4 q = make_float4(F[0], F[1], F[kPP], F[kPP + 1]);
  return kFast ? cic_fast(q, fz, fx) : cic(q, fz, fx);
}

// Exact node sums from two fire-and-forget 32-bit shared atomics:
// v = (v >> 16) * 2^16 + (v & 0xffff); the low halves (< 2^16 each) cannot
// overflow int32 while a tile holds fewer than kSplitMax particles (each
// particle adds to a node at most once); denser tiles go global.
constexpr long long kSplitMax = 32768;
__device__ __forceinline__ void sadd_split(unsigned* lo, int* hi, int v) {
  atomicAdd(lo, (unsigned)(v & 0xffff));
  atomicAdd(hi, v >> 16);
}

__device__ __forceinline__ void enqueue_t(FlushEntry* e, const int v[kNodes], int i, int j) {
#pragma unroll
  for (int k = 0; k < kNodes / 4; ++k) e->v[k] = make_int4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  e->cell = i;
  e->m = (unsigned)j;
}

__device__ __forceinline__ void drain_tile(const PicParams& p, const FlushEntry* q, int count,
                                           int lane, unsigned* s_lo, int* s_hi, int tz, int tx,
                                           bool dense) {
  __syncwarp();
  const int node = lane & 15;
  int comp, dr, ds;
  slot_node(node, comp, dr, ds);
  for (int e0 = 0; e0 < count; e0 += 2) {
    const int e = e0 + (lane >> 4);
    if (e < count) {
      const int i = q[e].cell, j = (int)q[e].m;
      const int v = reinterpret_cast<const int*>(q[e].v)[node];
      if (v) {
        if (!dense && in_patch(i, j, tz, tx)) {
          const int o = comp * kPatch + patch_at(i + dr + 1, j + ds + 1, tz, tx);
          sadd_split(s_lo + o, s_hi + o, v);
        } else {
          red_add(p.Jn + comp * p.jn_stride + (long long)(i + dr + 1) * p.pitch + (j + ds + 1), v);
        }
      }
    }
  }
  __syncwarp();
}

// kG consecutive doubles, stored back only for particles of this tile:
// one vector store when the whole group is ours, else per particle.
__device__ __forceinline__ void stg_mask(double* a, long long i, long long lo, long long hi,
                                         const double v[kG]) {
  if (i >= lo && i + kG <= hi) {
    stg(a, i, hi, v);
  } else {
#pragma unroll
    for (int j = 0; j < kG; ++j)
      if (i + j >= lo && i + j < hi) __stcs(a + i + j, v[j]);
  }
}

// kFast: tolerance mode (LBX_PIC_FAST | LBX_PIC_TILED): fast_axis, FMA gathers,
// float32 Boris increment, float run sums (rounded to fixed point at the queue).
template <bool kClock, bool kFast = false>
__global__ void __launch_bounds__(kPB, LBX_PIC_MINB) pic_tile_kernel(PicParams p) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  FlushEntry* s_q = reinterpret_cast<FlushEntry*>(s_dyn) + (size_t)(threadIdx.x >> 5) * kQCapT;
  float* s_f = reinterpret_cast<float*>(s_dyn + (size_t)kPW * kQCapT * sizeof(FlushEntry));  // [6][kPatch]
  unsigned* s_lo = reinterpret_cast<unsigned*>(s_f + 6 * kPatch);                            // [3][kPatch]
  int* s_hi = reinterpret_cast<int*>(s_lo + 3 * kPatch);                                     // [3][kPatch]
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_hi + 3 * kPatch);                          // nb
  unsigned* s_clk = s_cnt + p.nb;                                                            // nb
  __shared__ long long s_n;
  __shared__ int s_box[4];
  __shared__ int s_last;
  __shared__ unsigned long long s_red[kPW];
  __shared__ long long s_min[kPW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_n = *((volatile long long*)&p.st->n);
    s_box[0] = INT_MAX;
    s_box[1] = INT_MIN;
    s_box[2] = INT_MAX;
    s_box[3] = INT_MIN;
  }
  for (int b = tid; b < p.nb; b += kPB) {
    s_cnt[b] = 0u;
    if (kClock) s_clk[b] = 0u;
  }
  __syncthreads();
  const long long n = s_n;
  const double ez = (double)p.nz, ex = (double)p.nx;
  const double h = 0.5 * p.qm * p.dt;
  unsigned removed = 0;                          // per lane: 32 bits (register pressure)
  long long first_out = LLONG_MAX;
  int err = 0;
  int bimin = INT_MAX, bimax = INT_MIN, bjmin = INT_MAX, bjmax = INT_MIN;

  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    // the ranges partition [0, n_sort); the last one is extended to n, so any
    // input (even one the ranges do not describe) is processed exactly once
    const long long lo = min((long long)p.tile_rd[tile], n);
    const long long hi = tile == p.ntiles - 1 ? n : min((long long)p.tile_rd[tile + 1], n);
    if (lo >= hi) continue;   // CTA-uniform
    const bool dense = hi - lo >= kSplitMax;
    const int tz = (tile / p.ntx) * kT, tx = (tile % p.ntx) * kT;
    const int P0 = tz - kGd, Q0 = tx - kGd;   // padded index of patch row / column 0
    __syncthreads();                          // the previous tile's patch and sums are done
    for (int o = tid; o < 6 * kPatch; o += kPB) {
      const int c = o / kPatch, rr = (o - c * kPatch) / kPP, cc = o - c * kPatch - rr * kPP;
      const int P = P0 + rr, Q = Q0 + cc;
      s_f[o] = (P >= 0 && P < p.nz + 2 && Q >= 0 && Q < p.nx + 2)
                   ? __ldg(p.F[c] + (long long)P * p.pitch + Q)
                   : 0.f;
    }
    for (int o = tid; o < 3 * kPatch; o += kPB) {
      s_lo[o] = 0u;
      s_hi[o] = 0;
    }
    __syncthreads();
    const long long a0 = lo & ~(long long)(kG - 1);   // group starts stay 32-byte aligned
    const int run = min(kRun, (int)(((hi - a0 + kPB - 1) / kPB + kG - 1) / kG) * kG);
    for (long long w = a0 + (long long)warp * 32 * run; w < hi; w += (long long)kPW * 32 * run) {
      const long long run0 = w + (long long)lane * run;
      int acc[kNodes];
      float accf[kNodes];
#pragma unroll
      for (int i = 0; i < kNodes; ++i) {
        acc[i] = 0;
        accf[i] = 0.f;
      }
      int cur = -1, cur_i = 0, cur_j = 0;
      int hb = -1;
      unsigned hn = 0;
      long long t_last = 0;
      if (kClock) t_last = clock64();
#pragma unroll 1
      for (int g = 0; g < run / kG; ++g) {
        const long long i0 = run0 + g * kG;
        if (__all_sync(kAll, i0 >= hi)) break;
        double pz[kG], px[kG], puz[kG], pux[kG], puy[kG];
        ldg(p.z, i0, hi, pz);
        ldg(p.x, i0, hi, px);
        ldg(p.uz, i0, hi, puz);
        ldg(p.ux, i0, hi, pux);
        ldg(p.uy, i0, hi, puy);
        bool keep[kG];
        int nkey[kG];
        float vsx[kG], vsy[kG], vsz[kG];
#pragma unroll
        for (int k = 0; k < kG; ++k) {
          const bool valid = i0 + k >= lo && i0 + k < hi;
          const Axis az = pic_axis<kFast>(pz[k]), ax = pic_axis<kFast>(px[k]);
          float Ex, Ey, Ez, Bx, By, Bz;
          if (in_patch(az.i, ax.i, tz, tx)) {
            Ex = gather_s<kFast>(s_f, 0, az.i, ax.ih, az.f, ax.fh, tz, tx);
            Ey = gather_s<kFast>(s_f, 1, az.i, ax.i, az.f, ax.f, tz, tx);
            Ez = gather_s<kFast>(s_f, 2, az.ih, ax.i, az.fh, ax.f, tz, tx);
            Bx = gather_s<kFast>(s_f, 3, az.ih, ax.i, az.fh, ax.f, tz, tx);
            By = gather_s<kFast>(s_f, 4, az.ih, ax.ih, az.fh, ax.fh, tz, tx);
            Bz = gather_s<kFast>(s_f, 5, az.i, ax.ih, az.f, ax.fh, tz, tx);
          } else {
            Ex = gather_c<false, kFast>(p, 0, az.i, ax.ih, az.f, ax.fh);
            Ey = gather_c<false, kFast>(p, 1, az.i, ax.i, az.f, ax.f);
            Ez = gather_c<false, kFast>(p, 2, az.ih, ax.i, az.fh, ax.f);
            Bx = gather_c<false, kFast>(p, 3, az.ih, ax.i, az.fh, ax.f);
            By = gather_c<false, kFast>(p, 4, az.ih, ax.ih, az.fh, ax.fh);
            Bz = gather_c<false, kFast>(p, 5, az.i, ax.ih, az.f, ax.fh);
          }
          if (kFast) {
            const float ig = boris_fast(pux[k], puy[k], puz[k], (float)h, Ex, Ey, Ez, Bx, By, Bz);
            const float dtg = (float)p.dt * ig;
            pz[k] = __dadd_rn(pz[k], (double)__fmul_rn(dtg, (float)puz[k]));
            px[k] = __dadd_rn(px[k], (double)__fmul_rn(dtg, (float)pux[k]));
            const int iz = __double2int_rz(pz[k]), ix = __double2int_rz(px[k]);
            keep[k] = valid && pz[k] >= 0.0 && px[k] >= 0.0 && iz < p.nz && ix < p.nx;
            nkey[k] = keep[k] ? iz * p.nx + ix : -1;
            const float qv = keep[k] ? __fmul_rn((float)p.qw * p.vscale, ig) : 0.f;
            vsx[k] = __fmul_rn(qv, (float)pux[k]);
            vsy[k] = __fmul_rn(qv, (float)puy[k]);
            vsz[k] = __fmul_rn(qv, (float)puz[k]);
          } else {
          // relativistic Boris (x, y, z order; oracle boris())
          const double hEx = __dmul_rn(h, (double)Ex), hEy = __dmul_rn(h, (double)Ey),
                       hEz = __dmul_rn(h, (double)Ez);
          const double mx = __dadd_rn(pux[k], hEx);
          const double my = __dadd_rn(puy[k], hEy);
          const double mz = __dadd_rn(puz[k], hEz);
          const double gg = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(mx, mx)),
                                                           __dmul_rn(my, my)), __dmul_rn(mz, mz)));
          const double ig = __drcp_rn(gg);
          const double tbx = __dmul_rn(__dmul_rn(h, (double)Bx), ig);
          const double tby = __dmul_rn(__dmul_rn(h, (double)By), ig);
          const double tbz = __dmul_rn(__dmul_rn(h, (double)Bz), ig);
          const double s2 = __dmul_rn(2.0, __drcp_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(tbx, tbx)),
                                                                         __dmul_rn(tby, tby)),
                                                               __dmul_rn(tbz, tbz))));
          const double qx = __dadd_rn(mx, __dsub_rn(__dmul_rn(my, tbz), __dmul_rn(mz, tby)));
          const double qy = __dadd_rn(my, __dsub_rn(__dmul_rn(mz, tbx), __dmul_rn(mx, tbz)));
          const double qz = __dadd_rn(mz, __dsub_rn(__dmul_rn(mx, tby), __dmul_rn(my, tbx)));
          pux[k] = __dadd_rn(__dadd_rn(mx, __dmul_rn(s2, __dsub_rn(__dmul_rn(qy, tbz), __dmul_rn(qz, tby)))), hEx);
          puy[k] = __dadd_rn(__dadd_rn(my, __dmul_rn(s2, __dsub_rn(__dmul_rn(qz, tbx), __dmul_rn(qx, tbz)))), hEy);
          puz[k] = __dadd_rn(__dadd_rn(mz, __dmul_rn(s2, __dsub_rn(__dmul_rn(qx, tby), __dmul_rn(qy, tbx)))), hEz);
          const double gam = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(pux[k], pux[k])),
                                                            __dmul_rn(puy[k], puy[k])),
                                                  __dmul_rn(puz[k], puz[k])));
          const double igam = __drcp_rn(gam);
          pz[k] = __dadd_rn(pz[k], __dmul_rn(__dmul_rn(p.dt, puz[k]), igam));
          px[k] = __dadd_rn(px[k], __dmul_rn(__dmul_rn(p.dt, pux[k]), igam));
          keep[k] = valid && pz[k] >= 0.0 && pz[k] < ez && px[k] >= 0.0 && px[k] < ex;
          nkey[k] = keep[k] ? (int)pz[k] * p.nx + (int)px[k] : -1;
          const double qwg = keep[k] ? p.qw : 0.0;
          vsx[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, pux[k]), igam)), p.vscale);
          vsy[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puy[k]), igam)), p.vscale);
          vsz[k] = __fmul_rn(__double2float_rn(__dmul_rn(__dmul_rn(qwg, puz[k]), igam)), p.vscale);
          }
          if (valid && !keep[k]) {
            ++removed;
            first_out = min(first_out, i0 + k);
            if (p.removed_list) {
              const unsigned long long slot = atomicAdd(&p.st->removed_count, 1ull);
              if ((long long)slot < p.removed_cap) p.removed_list[slot] = i0 + k;
            }
          }
        }
        stg_mask(p.oz, i0, lo, hi, pz);
        stg_mask(p.ox, i0, lo, hi, px);
        stg_mask(p.ouz, i0, lo, hi, puz);
        stg_mask(p.oux, i0, lo, hi, pux);
        stg_mask(p.ouy, i0, lo, hi, puy);
        // current: register runs -> warp queue -> shared (patch) / global
        const unsigned lt = (1u << lane) - 1u;
        int qn = 0;
#pragma unroll
        for (int k = 0; k < kG; ++k) {
          const bool dep = nkey[k] >= 0;
          const Axis az = pic_axis<kFast>(dep ? pz[k] : 0.5), ax = pic_axis<kFast>(dep ? px[k] : 0.5);
          const bool same = dep && nkey[k] == cur;
          const bool strag = dep && !same && cur >= 0 && k + 1 < kG && nkey[k + 1] != nkey[k];
          const bool swap = dep && !same && !strag;
          const bool need = strag || (swap && cur >= 0);
          const unsigned fm = __ballot_sync(kAll, need);
          if (kFast) {
            // float run sums, rounded to fixed point when queued
            if (need) {
              int qi[kNodes];
              if (strag) {
                float w[kNodes];
#pragma unroll
                for (int i = 0; i < kNodes; ++i) w[i] = 0.f;
                node_accum(az, ax, vsx[k], vsy[k], vsz[k], w);
#pragma unroll
                for (int i = 0; i < kNodes; ++i) qi[i] = __float2int_rn(w[i]);
                enqueue_t(s_q + qn + __popc(fm & lt), qi, az.i, ax.i);
              } else {
#pragma unroll
                for (int i = 0; i < kNodes; ++i) qi[i] = __float2int_rn(accf[i]);
                enqueue_t(s_q + qn + __popc(fm & lt), qi, cur_i, cur_j);
              }
            }
            qn += __popc(fm);
            if (kQCapT < 32 * kG && qn > kQCapT - 32) {
              drain_tile(p, s_q, qn, lane, s_lo, s_hi, tz, tx, dense);
              qn = 0;
            }
            if (__any_sync(kAll, swap)) {
              if (swap) {
#pragma unroll
                for (int i = 0; i < kNodes; ++i) accf[i] = 0.f;
                cur = nkey[k];
                cur_i = az.i;
                cur_j = ax.i;
              }
            }
            if (same || swap) node_accum(az, ax, vsx[k], vsy[k], vsz[k], accf);
          } else {
          int q[kNodes];
          node_values(az, ax, vsx[k], vsy[k], vsz[k], q);
          if (need) {
            if (strag) enqueue_t(s_q + qn + __popc(fm & lt), q, az.i, ax.i);
            else enqueue_t(s_q + qn + __popc(fm & lt), acc, cur_i, cur_j);
          }
          qn += __popc(fm);
          if (kQCapT < 32 * kG && qn > kQCapT - 32) {
            drain_tile(p, s_q, qn, lane, s_lo, s_hi, tz, tx, dense);
            qn = 0;
          }
          if (same) {
#pragma unroll
            for (int i = 0; i < kNodes; ++i) acc[i] += q[i];
          } else if (swap) {
#pragma unroll
            for (int i = 0; i < kNodes; ++i) acc[i] = q[i];
            cur = nkey[k];
            cur_i = az.i;
            cur_j = ax.i;
          }
          }
          if (!dep) continue;
          bimin = min(bimin, az.i);
          bimax = max(bimax, az.i);
          bjmin = min(bjmin, ax.i);
          bjmax = max(bjmax, ax.i);
          const int bz = az.i >> p.log2m, bx = ax.i >> p.log2m;
          if (bz >= p.nbz || bx >= p.nbx) {
            ++err;
          } else if (bz * p.nbx + bx == hb) {
            ++hn;
          } else {
            if (hb >= 0) {
              atomicAdd(s_cnt + hb, hn);
              if (kClock) {
                const long long t = clock64();
                atomicAdd(s_clk + hb, (unsigned)min((t - t_last) >> 4, (long long)(1u << 30)));
                t_last = t;
              }
            }
            hb = bz * p.nbx + bx;
            hn = 1;
          }
        }
        if (qn) drain_tile(p, s_q, qn, lane, s_lo, s_hi, tz, tx, dense);
      }
      {
        const unsigned fm = __ballot_sync(kAll, cur >= 0);
        if (kFast) {
#pragma unroll
          for (int i = 0; i < kNodes; ++i) acc[i] = __float2int_rn(accf[i]);
        }
        if (cur >= 0) enqueue_t(s_q + __popc(fm & ((1u << lane) - 1u)), acc, cur_i, cur_j);
        if (fm) drain_tile(p, s_q, __popc(fm), lane, s_lo, s_hi, tz, tx, dense);
      }
      unsigned tclk = 0;
      if (kClock && hb >= 0) tclk = (unsigned)min((clock64() - t_last) >> 4, (long long)(1u << 30));
      const int hb0 = __shfl_sync(kAll, hb, 0);
      if (__all_sync(kAll, hb == hb0)) {
        const unsigned tot = __reduce_add_sync(kAll, hn);
        const unsigned clk = kClock ? __reduce_add_sync(kAll, tclk) : 0u;
        if (lane == 0 && hb0 >= 0 && tot) {
          atomicAdd(s_cnt + hb0, tot);
          if (kClock) atomicAdd(s_clk + hb0, clk);
        }
      } else if (hb >= 0 && hn) {
        atomicAdd(s_cnt + hb, hn);
        if (kClock) atomicAdd(s_clk + hb, tclk);
      }
    }
    __syncthreads();
    for (int o = tid; o < 3 * kPatch; o += kPB) {   // the tile's node sums -> Jn
      const long long v = (long long)s_hi[o] * 65536 + (long long)s_lo[o];
      if (!v) continue;
      const int c = o / kPatch, rr = (o - c * kPatch) / kPP, cc = o - c * kPatch - rr * kPP;
      red_add(p.Jn + c * p.jn_stride + (long long)(P0 + rr) * p.pitch + (Q0 + cc), v);
    }
  }

  // ---- CTA totals, deposit box, histogram flush, epilogue (as pic_push_kernel) ----
  const unsigned long long wa = (unsigned long long)warp_sum((long long)removed);
  const long long wm = warp_min(first_out), we = warp_sum(err);
  const int wimin = __reduce_min_sync(kAll, bimin), wimax = __reduce_max_sync(kAll, bimax);
  const int wjmin = __reduce_min_sync(kAll, bjmin), wjmax = __reduce_max_sync(kAll, bjmax);
  if (lane == 0) {
    s_red[warp] = wa;
    s_min[warp] = wm;
    if (we) atomicAdd((unsigned long long*)&p.st->err, (unsigned long long)we);
    if (wimin <= wimax) {
      atomicMin(&s_box[0], wimin);
      atomicMax(&s_box[1], wimax);
      atomicMin(&s_box[2], wjmin);
      atomicMax(&s_box[3], wjmax);
    }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long ta = 0;
    long long tm = LLONG_MAX;
    for (int w2 = 0; w2 < kPW; ++w2) {
      ta += s_red[w2];
      tm = min(tm, s_min[w2]);
    }
    if (ta) {
      atomicAdd(&p.st->leavers, ta);
      atomicMin(&p.st->first_leaver, tm);
    }
    if (s_box[0] <= s_box[1]) {
      atomicMin(p.dep_box + 0, s_box[0]);
      atomicMax(p.dep_box + 1, s_box[1]);
      atomicMin(p.dep_box + 2, s_box[2]);
      atomicMax(p.dep_box + 3, s_box[3]);
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
  step_record<kClock>(p.g_cnt, p.g_clk, p.nb, p.counts_out, p.cost_out, p.clk_out, p.wp, p.wc,
                      p.cells, 4);
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

// Sorted mode, resynchronisation / periodic sort: particles per cell of the
// current positions.  A warp takes 32 consecutive particles (coalesced
// loads); each run of equal keys across the lanes adds its length with one
// RED (a lane-per-thread run of 64 particles read with a 512-byte stride
// between lanes: 2.1 GB fetched for 1.6 GB, 0.79 ms on C2 x128).
__global__ void pic_count_kernel(const double* __restrict__ z, const double* __restrict__ x,
                                 const DevState* st, unsigned* cell_cnt, int nx, int ntx = 0) {
  const long long n = st->n;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 < n;
       w += warps) {
    const long long i = w * 32 + lane;
    const bool live = i < n;
    int key = -1;
    if (live) {
      const int iz = (int)__ldcs(z + i), ix = (int)__ldcs(x + i);
      key = ntx ? tile_key(iz, ix, ntx) : iz * nx + ix;
    }
    const int prev = __shfl_up_sync(kAll, key, 1);
    const bool start = live && (lane == 0 || key != prev);
    const unsigned sm = __ballot_sync(kAll, start);
    const unsigned lm = __ballot_sync(kAll, live);
    if (start) {
      const unsigned later = sm & ~((2u << lane) - 1u);   // run starts after this lane
      const int end = later ? __ffs(later) - 1 : 32 - __clz(lm);
      red_add32(cell_cnt + key, (unsigned)(end - lane));
    }
  }
}
// Periodic re-sort (lbx_pic_sort): scatter the particles to their cell's
// slots.  A warp takes 32 consecutive particles (coalesced loads); lanes with
// the same cell share one cursor atomic (__match_any_sync) and write
// consecutive slots.
__global__ void pic_sort_scatter_kernel(const double* __restrict__ z, const double* __restrict__ x,
                                        const double* __restrict__ uz,
                                        const double* __restrict__ ux,
                                        const double* __restrict__ uy, double* oz, double* ox,
                                        double* ouz, double* oux, double* ouy, const DevState* st,
                                        unsigned* cursor, int nx, int ntx) {
  // kSG groups of 32 consecutive particles per warp iteration: every load
  // and every cursor atomic of the groups is in flight together (one group
  // per iteration left the warp waiting on each atomic's round trip: 0.66
  // of HBM on C2 x128)
  constexpr int kSG = 4;
  const long long n = st->n;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       w * 32 * kSG < n; w += warps) {
    double vz[kSG], vx[kSG], vuz[kSG], vux[kSG], vuy[kSG];
    int key[kSG];
    bool live[kSG];
#pragma unroll
    for (int g = 0; g < kSG; ++g) {
      const long long i = (w * kSG + g) * 32 + lane;
      live[g] = i < n;
      const long long j = live[g] ? i : n - 1;
      vz[g] = __ldcs(z + j);
      vx[g] = __ldcs(x + j);
      vuz[g] = __ldcs(uz + j);
      vux[g] = __ldcs(ux + j);
      vuy[g] = __ldcs(uy + j);
      key[g] = ntx ? tile_key((int)vz[g], (int)vx[g], ntx) : (int)vz[g] * nx + (int)vx[g];
    }
    unsigned base[kSG], grp[kSG];
#pragma unroll
    for (int g = 0; g < kSG; ++g) {
      const unsigned act = __ballot_sync(kAll, live[g]);
      grp[g] = __match_any_sync(kAll, live[g] ? key[g] : -1) & act;
      base[g] = 0;
      if (live[g] && lane == __ffs(grp[g]) - 1)
        base[g] = atomicAdd(cursor + key[g], (unsigned)__popc(grp[g]));
    }
#pragma unroll
    for (int g = 0; g < kSG; ++g) {
      const int leader = live[g] ? __ffs(grp[g]) - 1 : lane;
      const unsigned b = __shfl_sync(kAll, base[g], leader);
      if (!live[g]) continue;
      const long long d = (long long)b + __popc(grp[g] & ((1u << lane) - 1u));
      __stcs(oz + d, vz[g]);
      __stcs(ox + d, vx[g]);
      __stcs(ouz + d, vuz[g]);
      __stcs(oux + d, vux[g]);
      __stcs(ouy + d, vuy[g]);
    }
  }
}

// Exclusive scan of cell_cnt into cursor (the first slot of each cell), in
// two launches over kScanBlocks contiguous segments; cell_cnt is zeroed.
constexpr int kScanBlocks = 296;
constexpr int kScanThreads = 1024;

__global__ void pic_scan_reduce_kernel(const unsigned* __restrict__ cell_cnt, long long cells,
                                       unsigned* block_sum) {
  const long long seg = (cells + gridDim.x - 1) / gridDim.x;
  const long long a = blockIdx.x * seg, b = min(cells, a + seg);
  unsigned s = 0;
  for (long long c = a + threadIdx.x; c < b; c += blockDim.x) s += cell_cnt[c];
  s = __reduce_add_sync(kAll, s);
  __shared__ unsigned w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned v = threadIdx.x < (blockDim.x >> 5) ? w[threadIdx.x] : 0u;
    v = __reduce_add_sync(kAll, v);
    if (threadIdx.x == 0) block_sum[blockIdx.x] = v;
  }
}

__global__ void pic_scan_apply_kernel(unsigned* cell_cnt, long long cells,
                                      const unsigned* __restrict__ block_sum, unsigned* cursor,
                                      unsigned* tile_start = nullptr) {
  __shared__ unsigned w[32];
  __shared__ unsigned s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this segment's base: sum of the preceding segments' totals
  unsigned pre = 0;
  for (int i = threadIdx.x; i < (int)blockIdx.x; i += blockDim.x) pre += block_sum[i];
  pre = __reduce_add_sync(kAll, pre);
  if (lane == 0) w[warp] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
    s_base = t;
  }
  __syncthreads();
  unsigned base = s_base;
  const long long seg = (cells + gridDim.x - 1) / gridDim.x;
  const long long a = blockIdx.x * seg, b = min(cells, a + seg);
  for (long long c0 = a; c0 < b; c0 += blockDim.x) {
    const long long c = c0 + threadIdx.x;
    const unsigned v = c < b ? cell_cnt[c] : 0u;
    // block-wide exclusive scan of v
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(kAll, incl, o);
      if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned t = lane < (int)(blockDim.x >> 5) ? w[lane] : 0u;
      unsigned ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kAll, ti, o);
        if (lane >= o) ti += y;
      }
      w[lane] = ti - t;   // exclusive warp offsets
    }
    __syncthreads();
    const unsigned excl = base + w[warp] + incl - v;
    if (c < b) {
      cursor[c] = excl;
      cell_cnt[c] = 0u;
      if (tile_start) {   // tile-major keys: 2^kTileShift per tile; [ntiles] = total
        if ((c & ((1 << kTileShift) - 1)) == 0) tile_start[c >> kTileShift] = excl;
        if (c == cells - 1) tile_start[cells >> kTileShift] = excl + v;
      }
    }
    // next chunk's base = excl of the last thread + its v
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_base = excl + v;
    __syncthreads();
    base = s_base;
  }
}

// Sorted mode, O(removed) compaction of the absorbed slots: survivors from
// the tail [n_new, n_new + L) move into the holes below n_new (order within a
// cell is not kept anyway).  L = st->removed_count; when it exceeds the list
// capacity these kernels do nothing and the stable compaction runs instead.
__global__ void pic_fill_mark_kernel(DevState* st, const long long* __restrict__ removed,
                                     long long cap, long long* holes, long long* tail_flag) {
  const long long L = (long long)st->removed_count, n_new = st->n;
  if (L == 0 || L > cap) return;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < L;
       k += (long long)gridDim.x * blockDim.x) {
    const long long r = removed[k];
    if (r >= n_new) tail_flag[r - n_new] = 1;
    else holes[atomicAdd(&st->holes, 1ull)] = r;
  }
}

__global__ void pic_fill_move_kernel(DevState* st, long long cap, const long long* __restrict__ holes,
                                     long long* tail_flag, double* z, double* x, double* uz,
                                     double* ux, double* uy) {
  const long long L = (long long)st->removed_count, n_new = st->n;
  if (L == 0 || L > cap) return;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < L;
       j += (long long)gridDim.x * blockDim.x) {
    if (tail_flag[j]) {
      tail_flag[j] = 0;
      continue;
    }
    const long long src = n_new + j;
    const long long dst = holes[atomicAdd(&st->movers, 1ull)];
    z[dst] = z[src];
    x[dst] = x[src];
    uz[dst] = uz[src];
    ux[dst] = ux[src];
    uy[dst] = uy[src];
  }
}

__global__ void pic_fill_done_kernel(DevState* st, long long cap) {
  const long long L = (long long)st->removed_count;
  if (L > 0 && L <= cap) {   // compacted: nothing left for the stable pass
    st->leavers = 0ull;
    st->first_leaver = LLONG_MAX;
    st->n_old = st->n;
  }
  st->holes = 0ull;
  st->movers = 0ull;
  st->removed_count = 0ull;
}

// fields -> quads: Q[c][qi*(nx+1) + qj] = (F[qi][qj], F[qi][qj+1], F[qi+1][qj],
// F[qi+1][qj+1]) in padded indices, qi in [0, nz], qj in [0, nx]; also resets
// the deposit bounding box for this step's push.
__global__ void pic_quad_kernel(const float* __restrict__ F0, const float* __restrict__ F1,
                                const float* __restrict__ F2, const float* __restrict__ F3,
                                const float* __restrict__ F4, const float* __restrict__ F5,
                                float4* Q, long long quads, int qpitch, int pitch, int* dep_box,
                                int diff) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    dep_box[0] = INT_MAX;
    dep_box[1] = INT_MIN;
    dep_box[2] = INT_MAX;
    dep_box[3] = INT_MIN;
  }
  const float* F[6] = {F0, F1, F2, F3, F4, F5};
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < quads;
       o += (long long)gridDim.x * blockDim.x) {
    const int qi = (int)(o / qpitch), qj = (int)(o - (long long)qi * qpitch);
    const long long g = (long long)qi * pitch + qj;
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const float a = __ldg(F[c] + g), b = __ldg(F[c] + g + 1), d0 = __ldg(F[c] + g + pitch),
                  d1 = __ldg(F[c] + g + pitch + 1);
      // diff (LBX_PIC_FAST): (a, b - a, c - a, a - b - c + d) for cic_diff
      __stcg(Q + c * quads + o,
             diff ? make_float4(a, __fsub_rn(b, a), __fsub_rn(d0, a),
                                __fadd_rn(__fsub_rn(a, b), __fsub_rn(d1, d0)))
                  : make_float4(a, b, d0, d1));
    }
  }
}

// Jc (cell-centric node sums) -> J: node (i, j) collects the slots of the
// cells around it; J += float32(sum / scale) as the oracle's deposit.
__global__ void pic_current_kernel(const unsigned long long* __restrict__ Jc, const int* dep_box,
                                   float* Jx, float* Jy, float* Jz, int nz, int nx,
                                   double inv_scale) {
  const int bi0 = dep_box[0], bi1 = dep_box[1], bj0 = dep_box[2], bj1 = dep_box[3];
  if (bi0 > bi1) return;
  // receiving nodes: rows [bi0-1, bi1+1] x cols [bj0-1, bj1+1]
  const int r0 = bi0 - 1, c0 = bj0 - 1, R = bi1 - bi0 + 3, C = bj1 - bj0 + 3;
  const int pitch = nx + 2;
  const long long all = (long long)R * C;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < all;
       o += (long long)gridDim.x * blockDim.x) {
    const int i = r0 + (int)(o / C), j = c0 + (int)(o % C);
    if (i < -1 || i > nz || j < -1 || j > nx) continue;
    long long sx = 0, sy = 0, sz = 0;
#pragma unroll
    for (int r = -1; r <= 1; ++r) {
      const int ci = i - r;
      if (ci < 0 || ci >= nz) continue;
#pragma unroll
      for (int s = -1; s <= 1; ++s) {
        const int cj = j - s;
        if (cj < 0 || cj >= nx) continue;
        const unsigned long long* cell = Jc + ((long long)ci * nx + cj) * kNodes;
        if (r >= 0) sx += (long long)cell[r * 3 + s + 1];                       // Jx rows {0,1}
        if (r >= 0 && s >= 0) sy += (long long)cell[6 + r * 2 + s];              // Jy
        if (s >= 0) sz += (long long)cell[10 + (r + 1) * 2 + s];                 // Jz cols {0,1}
      }
    }
    const long long o2 = (long long)(i + 1) * pitch + (j + 1);
    if (sx) Jx[o2] = __fadd_rn(Jx[o2], (float)__dmul_rn((double)sx, inv_scale));
    if (sy) Jy[o2] = __fadd_rn(Jy[o2], (float)__dmul_rn((double)sy, inv_scale));
    if (sz) Jz[o2] = __fadd_rn(Jz[o2], (float)__dmul_rn((double)sz, inv_scale));
  }
}

// Clears the deposit bounding box of Jc (after pic_current_kernel).
__global__ void pic_zero_kernel(unsigned long long* Jc, const int* dep_box, int nx) {
  const int bi0 = dep_box[0], bi1 = dep_box[1], bj0 = dep_box[2], bj1 = dep_box[3];
  if (bi0 > bi1) return;
  const int C = bj1 - bj0 + 1;
  const long long all = (long long)(bi1 - bi0 + 1) * C * (kNodes / 2);
  ulonglong2* J2 = reinterpret_cast<ulonglong2*>(Jc);
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < all;
       o += (long long)gridDim.x * blockDim.x) {
    const long long cell = o / (kNodes / 2);
    const int i = bi0 + (int)(cell / C), j = bj0 + (int)(cell % C);
    J2[((long long)i * nx + j) * (kNodes / 2) + (o % (kNodes / 2))] = make_ulonglong2(0ull, 0ull);
  }
}

// Tiled mode: Jn (node-centric int64) -> J over the deposit box's nodes,
// clearing Jn; the same float32 rounding of the same integer node sums as
// pic_current_kernel.
__global__ void pic_current_node_kernel(unsigned long long* Jn, long long stride,
                                        const int* dep_box, float* Jx, float* Jy, float* Jz,
                                        int nz, int nx, double inv_scale) {
  const int bi0 = dep_box[0], bi1 = dep_box[1], bj0 = dep_box[2], bj1 = dep_box[3];
  if (bi0 > bi1) return;
  // nodes of cells [bi0, bi1] x [bj0, bj1]: padded rows bi0 .. bi1 + 2
  const int r0 = max(bi0, 0), r1 = min(bi1 + 2, nz + 1), c0 = max(bj0, 0), c1 = min(bj1 + 2, nx + 1);
  const int C = c1 - c0 + 1, pitch = nx + 2;
  const long long all = (long long)(r1 - r0 + 1) * C;
  float* J[3] = {Jx, Jy, Jz};
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < all;
       o += (long long)gridDim.x * blockDim.x) {
    const long long idx = (long long)(r0 + (int)(o / C)) * pitch + (c0 + (int)(o % C));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long v = (long long)Jn[c * stride + idx];
      if (v) {
        J[c][idx] = __fadd_rn(J[c][idx], (float)__dmul_rn((double)v, inv_scale));
        Jn[c * stride + idx] = 0ull;
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

// Jc -> J over the deposit box, clear Jc, Yee update (unless disabled).
// ---------------------------------------------------------------------------
// Charge-conserving PIC step (lbx_pic_args::shape_order K = 1..3): the
// paper's deposition (PAPER.md:235 -- third-order shapes; ~50 % of the
// walltime).  Per particle: K-order B-spline gather of every
// component at its stagger, Boris (float32 increment, boris_fast), move,
// absorb, then Esirkepov's decomposition on a common (K+2)^2 node window of
// the old and new positions (oracle/pic_oracle.py esirkepov_current):
// Jz / Jx as prefix sums of Wz / Wx along their axis, Jy from Wy; node
// values rounded to fixed point and added as integers into a padded
// node-centric int64 accumulator (kEskG guard nodes: every window of a
// kept particle fits).  A warp whose 32 consecutive particles share one
// window (dense, cell-sorted plasma) sums each node over the warp with
// redux.sync and issues one RED per node; otherwise every lane adds its own.
// pic_esk_current_kernel converts the sums (dropping nodes beyond the field
// arrays' one guard layer) and clears them; the Yee update follows.
constexpr int kEskG = 4;
constexpr int kEB = 256;
#ifndef LBX_ESK_RUN
#define LBX_ESK_RUN 16
#endif
constexpr int kEskRun = LBX_ESK_RUN;     // 32-particle iterations per warp chunk

// lowest node with a possibly nonzero weight: floor(v - (K+1)/2) + 1
template <int K>
__device__ __forceinline__ int shape_base(double v) {
  return __double2int_rd(v - 0.5 * (K + 1)) + 1;
}

// The K+1 nonzero weights of a position v, closed form: base = the lowest
// node (shape_base), u = frac(v - (K+1)/2) in [0, 1); w[k] = S_K(base + k - v)
// (K = 3: (1-u)^3/6, (3u^3 - 6u^2 + 4)/6, 1 - the others, u^3/6).  One
// evaluation per axis instead of one branchless piecewise polynomial per node.
template <int K>
__device__ __forceinline__ int bweights(double v, float w[K + 1]) {
  const double q = v - 0.5 * (K + 1);
  const double fl = floor(q);
  const float u = __double2float_rn(q - fl);
  if (K == 1) {
    w[0] = __fsub_rn(1.f, u);
    w[1] = u;
  } else if (K == 2) {
    const float h = __fsub_rn(u, 0.5f);
    w[0] = 0.5f * __fsub_rn(1.f, u) * __fsub_rn(1.f, u);
    w[1] = __fmaf_rn(-h, h, 0.75f);
    w[2] = 0.5f * u * u;
  } else {
    const float v1 = __fsub_rn(1.f, u), u2 = u * u, u3 = u2 * u;
    w[0] = v1 * v1 * v1 * (1.f / 6.f);
    w[1] = __fmaf_rn(u2, __fmaf_rn(0.5f, u, -1.f), 2.f / 3.f);
    w[3] = u3 * (1.f / 6.f);
    w[2] = __fsub_rn(__fsub_rn(__fsub_rn(1.f, w[0]), w[1]), w[3]);
  }
  return (int)fl + 1;
}

#ifndef LBX_ESK_F2
#define LBX_ESK_F2 0   // 1: Esirkepov gather / deposit arithmetic in packed f32x2 ops (measured slower per step, off)
#endif
// shared-memory adds of two nodes' values: two LDS, one FADD2, two STS
__device__ __forceinline__ void sadd2(float* a, int o1, float2 v) {
  const float2 t = __fadd2_rn(make_float2(a[0], a[o1]), v);
  a[0] = t.x;
  a[o1] = t.y;
}

// Row-quad gather: R[(r + 1) * rpitch + (c + 1)] = the padded field values
// (r, c .. c + 3) (zeros outside the array), so a shape-K gather is K + 1
// 16-byte loads instead of (K + 1)^2 scalar loads.
template <int K>
__device__ __forceinline__ float gather_rows(const float4* __restrict__ R, int rpitch, int bz,
                                             const float wz[K + 1], int bx,
                                             const float wx[K + 1]) {
  const float4* q = R + (long long)(bz + 2) * rpitch + (bx + 2);   // padded row bz + 1, col bx + 1
  float acc = 0.f;
  if constexpr (LBX_ESK_F2 && K % 2 == 1) {
    // two rows' sums per packed f32x2 op; each lane of an FFMA2 rounds as
    // the scalar FFMA does, and the row chain keeps its order: same bits
#pragma unroll
    for (int k = 0; k <= K; k += 2) {
      const float4 v = __ldg(q + (long long)k * rpitch), u = __ldg(q + (long long)(k + 1) * rpitch);
      float2 rs = __fmul2_rn(make_float2(wx[0], wx[0]), make_float2(v.x, u.x));
      rs = __ffma2_rn(make_float2(wx[1], wx[1]), make_float2(v.y, u.y), rs);
      if (K >= 2) rs = __ffma2_rn(make_float2(wx[2], wx[2]), make_float2(v.z, u.z), rs);
      if (K >= 3) rs = __ffma2_rn(make_float2(wx[3], wx[3]), make_float2(v.w, u.w), rs);
      acc = __fmaf_rn(wz[k], rs.x, acc);
      acc = __fmaf_rn(wz[k + 1], rs.y, acc);
    }
  } else {
#pragma unroll
    for (int k = 0; k <= K; ++k) {
      const float4 v = __ldg(q + (long long)k * rpitch);
      float rs = wx[0] * v.x;
      rs = __fmaf_rn(wx[1], v.y, rs);
      if (K >= 2) rs = __fmaf_rn(wx[2], v.z, rs);
      if (K >= 3) rs = __fmaf_rn(wx[3], v.w, rs);
      acc = __fmaf_rn(wz[k], rs, acc);
    }
  }
  return acc;
}

// Esirkepov's common-window shape of one position: its K+1 weights placed
// at window nodes o .. o + K (o = its base - the window base, 0 or 1).
template <int K>
__device__ __forceinline__ void window_shape(double v, int wbase, float S[K + 2]) {
  float w[K + 1];
  const int o = bweights<K>(v, w) - wbase;
#pragma unroll
  for (int k = 0; k < K + 2; ++k)
    S[k] = o ? (k >= 1 ? w[k - 1] : 0.f) : (k <= K ? w[k] : 0.f);
}

__global__ void esk_rows_kernel(const float* __restrict__ F0, const float* __restrict__ F1,
                                const float* __restrict__ F2, const float* __restrict__ F3,
                                const float* __restrict__ F4, const float* __restrict__ F5,
                                float4* R, int nz, int nx) {
  const int rp = nx + 5, pitch = nx + 2;
  const long long rows = (long long)(nz + 5) * rp;
  const float* F[6] = {F0, F1, F2, F3, F4, F5};
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < rows;
       o += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(o / rp) - 1, c = (int)(o % rp) - 1;   // padded field indices
    const bool rok = r >= 0 && r <= nz + 1;
#pragma unroll
    for (int comp = 0; comp < 6; ++comp) {
      float v[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int cc = c + l;
        v[l] = (rok && cc >= 0 && cc <= nx + 1) ? __ldg(F[comp] + (long long)r * pitch + cc) : 0.f;
      }
      __stcg(R + comp * rows + o, make_float4(v[0], v[1], v[2], v[3]));
    }
  }
}

// Where a deposit goes: passed BY VALUE to the out-of-line flush / direct
// paths (a reference to the kernel parameter would copy all of EskParams to
// the stack).
struct EskOut {
  unsigned long long* J;        // [3][stride] padded node sums (Jx, Jy, Jz)
  long long stride;
  int apitch;                   // nx + 2 kEskG
  float cz;                     // -(q w / dt) * scale  (Jz, Jx)
  float cy;                     // q w * scale          (Jy, times vy)
};

struct EskParams {
  PicParams b;                  // particles, fields F[], grid, boxes, status, outputs
  const float4* R[6];           // row-quad field copies [(nz+5) x (nx+5)]
  int rpitch;
  EskOut o;                     // the current sums (by value into the out-of-line paths)
};

// The held block of pic_esk_kernel: the window of the block origin plus one
// node below in x (always) and in z (kEskZE = 1): Jz (K+1+ZE) x (W+1),
// Jx (W+ZE) x (K+2), Jy (W+ZE) x (W+1) nodes, each [node][lane] floats.
#ifndef LBX_ESK_ZEXT
#define LBX_ESK_ZEXT 1
#endif
constexpr int kEskZE = LBX_ESK_ZEXT;
template <int K>
struct EskBlock {
  static constexpr int W = K + 2;
  static constexpr int ZC = W + 1, ZR = K + 1 + kEskZE;   // Jz
  static constexpr int XC = K + 2, XR = W + kEskZE;       // Jx
  static constexpr int YC = W + 1, YR = W + kEskZE;       // Jy
  static constexpr int NZ = ZR * ZC, NX = XR * XC, NY = YR * YC, NE = NZ + NX + NY;
};

// Add a warp's held block (pic_esk_kernel): node t's 32 lane sums (read
// rotated: conflict-free), zeroed, rounded to fixed point, one RED each.
// Out of line: the rare path keeps its registers off the particle loop.
template <int K>
__device__ __noinline__ void esk_flush(const EskOut e, float* acc, int hbz, int hbx, int lane) {
  using B = EskBlock<K>;
  constexpr int NE = B::NE;
  __syncwarp();
  const long long h0 = (long long)(hbz - kEskZE + kEskG) * e.apitch + (hbx - 1 + kEskG);
  for (int t = lane; t < NE; t += 32) {
    float sum = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      float* a = acc + t * 32 + ((k + lane) & 31);
      sum += *a;
      *a = 0.f;
    }
    int comp, di, dj;
    float scale;
    if (t < B::NZ) {
      comp = 2; di = t / B::ZC; dj = t % B::ZC; scale = e.cz;
    } else if (t < B::NZ + B::NX) {
      comp = 0; di = (t - B::NZ) / B::XC; dj = (t - B::NZ) % B::XC; scale = e.cz;
    } else {
      comp = 1; di = (t - B::NZ - B::NX) / B::YC; dj = (t - B::NZ - B::NX) % B::YC; scale = e.cy;
    }
    const long long v = __float2ll_rn(sum * scale);
    if (v) red_add(e.J + comp * e.stride + h0 + (long long)di * e.apitch + dj, v);
  }
  __syncwarp();
}

// One particle's fixed-point Esirkepov values straight to HBM (a lane
// outside its warp's held block).
template <int K>
__device__ __noinline__ void esk_direct(const EskOut e, int bz, int bx, const float* s0z,
                                        const float* dsz, const float* s0x, const float* dsx,
                                        float uyg) {
  constexpr int W = K + 2;
  const long long r0 = (long long)(bz + kEskG) * e.apitch + (bx + kEskG);
  const float cz = e.cz, cy = e.cy * uyg;
  for (int j = 0; j < W; ++j) {
    const float hx = __fmaf_rn(0.5f, dsx[j], s0x[j]);
    float a = 0.f;
    for (int ii = 0; ii <= K; ++ii) {
      a = __fmaf_rn(dsz[ii], hx, a);
      const int v = __float2int_rn(cz * a);
      if (v) red_add(e.J + 2 * e.stride + r0 + (long long)ii * e.apitch + j, v);
    }
  }
  for (int ii = 0; ii < W; ++ii) {
    const float hz = __fmaf_rn(0.5f, dsz[ii], s0z[ii]);
    float a = 0.f;
    for (int j = 0; j <= K; ++j) {
      a = __fmaf_rn(dsx[j], hz, a);
      const int v = __float2int_rn(cz * a);
      if (v) red_add(e.J + r0 + (long long)ii * e.apitch + j, v);
    }
  }
  for (int ii = 0; ii < W; ++ii) {
    const float a0 = __fmaf_rn(0.5f, dsz[ii], s0z[ii]);
    const float a1 = __fmaf_rn(1.f / 3.f, dsz[ii], 0.5f * s0z[ii]);
    for (int j = 0; j < W; ++j) {
      const int v = __float2int_rn(cy * __fmaf_rn(a1, dsx[j], a0 * s0x[j]));
      if (v) red_add(e.J + e.stride + r0 + (long long)ii * e.apitch + j, v);
    }
  }
}

template <int K, bool kClock>
#ifndef LBX_ESK_MINB
#define LBX_ESK_MINB 2
#endif
#ifndef LBX_ESK_PREFETCH
#define LBX_ESK_PREFETCH 1
#endif
__global__ void __launch_bounds__(kEB, LBX_ESK_MINB) pic_esk_kernel(EskParams e) {
  constexpr int W = K + 2;                 // window nodes per axis
  const PicParams& p = e.b;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_dyn);
  unsigned* s_clk = s_cnt + p.nb;
  __shared__ PushShared sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  push_prologue<kClock>(p, sh, s_cnt, s_clk);
  const long long n = sh.n;
  const double ez = (double)p.nz, ex = (double)p.nx;
  const float hf = (float)(0.5 * p.qm * p.dt), dtf = (float)p.dt;
  unsigned removed = 0;                          // per lane: 32 bits (register pressure)
  long long first_out = LLONG_MAX;
  int err = 0;
  // A warp takes chunks of kEskRun x 32 consecutive particles and holds a
  // node block in shared memory: every lane keeps its own float sums
  // (acc[node][lane], conflict-free) of the Esirkepov values of its
  // particles whose window base lies within one node below the held window
  // (the particles of a dense, cell-sorted plasma, incl. those that moved a
  // face down); the block is summed over the lanes, rounded to fixed point
  // and added to HBM only when most of the warp's particles leave it
  // (recentre) and at the end of the chunk.  Lanes outside it add their own
  // fixed-point values directly.  (Round 2; replaces a redux.sync per node
  // per particle: 1,000 of 1,600 instructions per particle, ncu.)
  using Blk = EskBlock<K>;
  constexpr int NE = Blk::NE;
  float* acc = reinterpret_cast<float*>(s_dyn + (size_t)p.nb * 8) + (size_t)warp * NE * 32;
  for (int t = lane; t < NE * 32; t += 32) acc[t] = 0.f;
  __syncwarp();
  int hbz = INT_MIN / 2, hbx = INT_MIN / 2;   // held window (block origin: hbz - 1, hbx - 1)
  auto flush = [&]() {
    if (hbz != INT_MIN / 2) esk_flush<K>(e.o, acc, hbz, hbx, lane);
  };
  const long long chunk = (long long)kEskRun * 32;
  // the next 32 particles' loads are issued before this iteration's work
  // (LBX_ESK_PREFETCH): their HBM latency hides behind the gather / deposit
  double nz0 = 0.0, nx0 = 0.0, nuz = 0.0, nux = 0.0, nuy = 0.0;
  auto load = [&](long long w) {
    // particle loads bypass L1 (the row-quad gathers live there)
    const long long ic = min(w + lane, n - 1);
    nz0 = ld_na(p.z + ic);
    nx0 = ld_na(p.x + ic);
    nuz = ld_na(p.uz + ic);
    nux = ld_na(p.ux + ic);
    nuy = ld_na(p.uy + ic);
  };
  for (long long c0 = ((long long)blockIdx.x * (kEB / 32) + warp) * chunk; c0 < n;
       c0 += (long long)gridDim.x * (kEB / 32) * chunk) {
  const long long wend = min(n, c0 + chunk);
  if (LBX_ESK_PREFETCH) load(c0);
  for (long long w0 = c0; w0 < wend; w0 += 32) {
    const long long i = w0 + lane;
    const bool valid = i < n;
    long long t0 = 0;
    if (kClock) t0 = clock64();
    if (!LBX_ESK_PREFETCH) load(w0);
    const double z0 = nz0, x0 = nx0;
    double uz = nuz, ux = nux, uy = nuy;
    if (LBX_ESK_PREFETCH && w0 + 32 < wend) load(w0 + 32);
    // staggers: (0, 1/2) Ex Bz | (0, 0) Ey | (1/2, 0) Ez Bx | (1/2, 1/2) By
    // weights of the four stagger positions, once each
    float wz0[K + 1], wzh[K + 1], wx0[K + 1], wxh[K + 1];
    const int bz0 = bweights<K>(z0, wz0), bzh = bweights<K>(z0 - 0.5, wzh);
    const int bx0 = bweights<K>(x0, wx0), bxh = bweights<K>(x0 - 0.5, wxh);
    const int rp = e.rpitch;
    const float Ex = gather_rows<K>(e.R[0], rp, bz0, wz0, bxh, wxh);
    const float Ey = gather_rows<K>(e.R[1], rp, bz0, wz0, bx0, wx0);
    const float Ez = gather_rows<K>(e.R[2], rp, bzh, wzh, bx0, wx0);
    const float Bx = gather_rows<K>(e.R[3], rp, bzh, wzh, bx0, wx0);
    const float By = gather_rows<K>(e.R[4], rp, bzh, wzh, bxh, wxh);
    const float Bz = gather_rows<K>(e.R[5], rp, bz0, wz0, bxh, wxh);
    const float ig = boris_fast(ux, uy, uz, hf, Ex, Ey, Ez, Bx, By, Bz);
    const float dtg = dtf * ig;
    const double z1 = __dadd_rn(z0, (double)__fmul_rn(dtg, (float)uz));
    const double x1 = __dadd_rn(x0, (double)__fmul_rn(dtg, (float)ux));
    const bool keep = valid && z1 >= 0.0 && z1 < ez && x1 >= 0.0 && x1 < ex;
    if (valid) {
      __stcs(p.oz + i, z1);
      __stcs(p.ox + i, x1);
      __stcs(p.ouz + i, uz);
      __stcs(p.oux + i, ux);
      __stcs(p.ouy + i, uy);
      if (!keep) {
        ++removed;
        first_out = min(first_out, i);
        if (p.removed_list) {
          const unsigned long long slot = atomicAdd(&p.st->removed_count, 1ull);
          if ((long long)slot < p.removed_cap) p.removed_list[slot] = i;
        }
      }
    }
    // ---- Esirkepov weights on the common window ----
    const int bz = shape_base<K>(fmin(z0, z1)), bx = shape_base<K>(fmin(x0, x1));
    float s0z[W], dsz[W], s0x[W], dsx[W];
    window_shape<K>(z0, bz, s0z);
    window_shape<K>(z1, bz, dsz);
    window_shape<K>(x0, bx, s0x);
    window_shape<K>(x1, bx, dsx);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      dsz[k] = __fsub_rn(dsz[k], s0z[k]);
      dsx[k] = __fsub_rn(dsx[k], s0x[k]);
    }
    const float uyg = __fmul_rn((float)uy, ig);     // Jy's velocity factor
    const unsigned km = __ballot_sync(kAll, keep);
    const int lead = km ? __ffs(km) - 1 : 0;
    bool inb = keep && (unsigned)(bz - hbz + kEskZE) <= (unsigned)kEskZE &&
               (unsigned)(bx - hbx + 1) <= 1u;
    if (km && 2 * __popc(__ballot_sync(kAll, inb)) < __popc(km)) {
      // most kept particles outside the held block: add it, hold the block
      // whose upper window is the warp's highest (covers that and one below)
      flush();
      hbz = __reduce_max_sync(kAll, keep ? bz : INT_MIN);
      hbx = __reduce_max_sync(kAll, keep ? bx : INT_MIN);
      inb = keep && (unsigned)(bz - hbz + kEskZE) <= (unsigned)kEskZE &&
            (unsigned)(bx - hbx + 1) <= 1u;
    }
    if (inb) {
      // unscaled values into this lane's slots at the block offset (oz, ox)
      const int oz = bz - hbz + kEskZE, ox = bx - hbx + 1;
      float* az = acc + (oz * Blk::ZC + ox) * 32 + lane;
      float* ax = acc + (Blk::NZ + oz * Blk::XC + ox) * 32 + lane;
      float* ay = acc + (Blk::NZ + Blk::NX + oz * Blk::YC + ox) * 32 + lane;
      if (LBX_ESK_F2) {
        // the same values, two window nodes per packed op (j pairs for Jz /
        // Jy, ii pairs for Jx); each lane of a pair rounds as before
        constexpr int WP = W & ~1;             // paired part; node W-1 alone when W is odd
#pragma unroll
        for (int j = 0; j < WP; j += 2) {
          const float2 hx = __ffma2_rn(make_float2(0.5f, 0.5f), make_float2(dsx[j], dsx[j + 1]),
                                       make_float2(s0x[j], s0x[j + 1]));
          float2 a = make_float2(0.f, 0.f);
#pragma unroll
          for (int ii = 0; ii <= K; ++ii) {
            a = __ffma2_rn(make_float2(dsz[ii], dsz[ii]), hx, a);
            sadd2(az + (ii * Blk::ZC + j) * 32, 32, a);
          }
        }
        if (W & 1) {
          const int j = W - 1;
          const float hx = __fmaf_rn(0.5f, dsx[j], s0x[j]);
          float a = 0.f;
#pragma unroll
          for (int ii = 0; ii <= K; ++ii) {
            a = __fmaf_rn(dsz[ii], hx, a);
            az[(ii * Blk::ZC + j) * 32] += a;
          }
        }
#pragma unroll
        for (int ii = 0; ii < WP; ii += 2) {
          const float2 hz = __ffma2_rn(make_float2(0.5f, 0.5f), make_float2(dsz[ii], dsz[ii + 1]),
                                       make_float2(s0z[ii], s0z[ii + 1]));
          float2 a = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j <= K; ++j) {
            a = __ffma2_rn(make_float2(dsx[j], dsx[j]), hz, a);
            sadd2(ax + (ii * Blk::XC + j) * 32, Blk::XC * 32, a);
          }
        }
        if (W & 1) {
          const int ii = W - 1;
          const float hz = __fmaf_rn(0.5f, dsz[ii], s0z[ii]);
          float a = 0.f;
#pragma unroll
          for (int j = 0; j <= K; ++j) {
            a = __fmaf_rn(dsx[j], hz, a);
            ax[(ii * Blk::XC + j) * 32] += a;
          }
        }
#pragma unroll
        for (int ii = 0; ii < W; ++ii) {
          // (a0, a1) = uyg * (s0z + dsz/2, s0z/2 + dsz/3)
          const float2 a01 = __fmul2_rn(make_float2(uyg, uyg),
                                        __ffma2_rn(make_float2(0.5f, 1.f / 3.f), make_float2(dsz[ii], dsz[ii]),
                                                   make_float2(s0z[ii], 0.5f * s0z[ii])));
#pragma unroll
          for (int j = 0; j < WP; j += 2) {
            const float2 t = __fmul2_rn(make_float2(a01.x, a01.x), make_float2(s0x[j], s0x[j + 1]));
            sadd2(ay + (ii * Blk::YC + j) * 32, 32,
                  __ffma2_rn(make_float2(a01.y, a01.y), make_float2(dsx[j], dsx[j + 1]), t));
          }
          if (W & 1) {
            const int j = W - 1;
            ay[(ii * Blk::YC + j) * 32] += __fmaf_rn(a01.y, dsx[j], a01.x * s0x[j]);
          }
        }
      } else {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const float hx = __fmaf_rn(0.5f, dsx[j], s0x[j]);
        float a = 0.f;
#pragma unroll
        for (int ii = 0; ii <= K; ++ii) {
          a = __fmaf_rn(dsz[ii], hx, a);
          az[(ii * Blk::ZC + j) * 32] += a;
        }
      }
#pragma unroll
      for (int ii = 0; ii < W; ++ii) {
        const float hz = __fmaf_rn(0.5f, dsz[ii], s0z[ii]);
        float a = 0.f;
#pragma unroll
        for (int j = 0; j <= K; ++j) {
          a = __fmaf_rn(dsx[j], hz, a);
          ax[(ii * Blk::XC + j) * 32] += a;
        }
      }
#pragma unroll
      for (int ii = 0; ii < W; ++ii) {
        const float a0 = __fmul_rn(uyg, __fmaf_rn(0.5f, dsz[ii], s0z[ii]));             // s0z + dsz/2
        const float a1 = __fmul_rn(uyg, __fmaf_rn(1.f / 3.f, dsz[ii], 0.5f * s0z[ii])); // s0z/2 + dsz/3
#pragma unroll
        for (int j = 0; j < W; ++j) ay[(ii * Blk::YC + j) * 32] += __fmaf_rn(a1, dsx[j], a0 * s0x[j]);
      }
      }
    } else if (keep) {   // outside the block: this particle's values straight to HBM
      esk_direct<K>(e.o, bz, bx, s0z, dsz, s0x, dsx, uyg);
    }
    // ---- per-box survivor counts (+ GpuClock: the particle's whole work) ----
    int box = -1;
    if (keep) {
      const int bzz = __double2int_rz(z1) >> p.log2m, bxx = __double2int_rz(x1) >> p.log2m;
      if (bzz >= p.nbz || bxx >= p.nbx) ++err;
      else box = bzz * p.nbx + bxx;
    }
    unsigned dt = 0;
    if (kClock) dt = (unsigned)min((clock64() - t0) >> 4, (long long)(1 << 26));
    const int b0 = __shfl_sync(kAll, box, lead);
    if (__all_sync(kAll, box < 0 || box == b0)) {
      const unsigned cnt = __popc(__ballot_sync(kAll, box >= 0));
      const unsigned ck = kClock ? __reduce_add_sync(kAll, box >= 0 ? dt : 0u) : 0u;
      if (lane == 0 && cnt) {
        atomicAdd(s_cnt + b0, cnt);
        if (kClock) atomicAdd(s_clk + b0, ck);
      }
    } else if (box >= 0) {
      atomicAdd(s_cnt + box, 1u);
      if (kClock) atomicAdd(s_clk + box, dt);
    }
  }
  }
  flush();
  push_epilogue<kClock>(p, sh, n, removed, first_out, err, INT_MAX, INT_MIN, INT_MAX, INT_MIN,
                        s_cnt, s_clk);
}

__global__ void pic_esk_current_kernel(unsigned long long* __restrict__ J, long long stride,
                                       int apitch, float* __restrict__ jx, float* __restrict__ jy,
                                       float* __restrict__ jz, int nz, int nx, double inv_scale) {
  const int pitch = nx + 2;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < stride;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / apitch), c = (int)(idx - (long long)r * apitch);
    const int i = r - kEskG, j = c - kEskG;                 // node (i, j)
    const bool stored = i >= -1 && i <= nz && j >= -1 && j <= nx;
    float* out[3] = {jx, jy, jz};
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const long long v = (long long)J[comp * stride + idx];
      if (v) J[comp * stride + idx] = 0ull;
      if (stored) out[comp][(i + 1) * pitch + (j + 1)] = (float)((double)v * inv_scale);
    }
  }
}

int pic_finish(lbx_ctx* ctx, const lbx_pic_args* a, cudaStream_t s, double jscale,
               bool tiled = false) {
  const long long cells = (long long)a->nz * a->nx;
  const int pitch = a->nx + 2;
  const unsigned cg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (cells + 255) / 256));
  if (tiled) {
    const int* box = reinterpret_cast<const int*>(ctx->pic_jn + 3 * ctx->pic_jn_stride);
    pic_current_node_kernel<<<cg, 256, 0, s>>>(ctx->pic_jn, ctx->pic_jn_stride, box, a->current[0],
                                               a->current[1], a->current[2], a->nz, a->nx,
                                               1.0 / jscale);
  } else {
    int* dep_box = reinterpret_cast<int*>(ctx->pic_acc + ctx->pic_cells * kNodes);
    pic_current_kernel<<<cg, 256, 0, s>>>(ctx->pic_acc, dep_box, a->current[0], a->current[1],
                                          a->current[2], a->nz, a->nx, 1.0 / jscale);
    pic_zero_kernel<<<cg, 256, 0, s>>>(ctx->pic_acc, dep_box, a->nx);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "current launch");
  if (a->flags & LBX_PIC_NO_FIELD_SOLVE) return LBX_OK;
  const unsigned fg = cg;
  pic_b_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->nz, a->nx, pitch, a->dt);
  pic_e_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->current[0], a->current[1],
                                  a->current[2], a->nz, a->nx, pitch, a->dt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "field solve launch");
  return LBX_OK;
}


int esk_finish(lbx_ctx* ctx, const lbx_pic_args* a, cudaStream_t s);

// Host side of the charge-conserving step (lbx_pic_args::shape_order > 0).
int pic_step_esirkepov(lbx_ctx* ctx, const lbx_pic_args* a, cudaStream_t s) {
  const int K = a->shape_order;
  if (a->out[0]) return set_error(LBX_EINVAL, "shape_order > 0 runs in place (no out[])");
  if (a->flags & LBX_PIC_TILED)
    return set_error(LBX_EINVAL, "shape_order > 0 does not support tiled steps");
  uintptr_t al = (uintptr_t)a->z | (uintptr_t)a->x | (uintptr_t)a->uz | (uintptr_t)a->ux |
                 (uintptr_t)a->uy;
  if (al & 7u) return set_error(LBX_EINVAL, "particle arrays must be 8-byte aligned");
  const int nbz = a->nz / a->box_size, nbx = a->nx / a->box_size, nb = nbz * nbx;
  if (nb > 4096) return set_error(LBX_EINVAL, "PIC step supports <= 4096 boxes");
  int rc = ensure_accumulators(ctx, nb);
  if (rc) return rc;
  rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  ctx->pic_sort_next = nullptr;
  ctx->pic_tiles_nz = ctx->pic_tiles_nx = 0;
  const int apitch = a->nx + 2 * kEskG;
  const long long stride = (long long)(a->nz + 2 * kEskG) * apitch;
  if (!ctx->pic_esk || ctx->pic_esk_elems != stride) {
    if (ctx->pic_esk) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_esk);
    }
    ctx->pic_esk = nullptr;
    const size_t bytes = (size_t)stride * 3 * 8 + 16;
    if (cudaMalloc(&ctx->pic_esk, bytes) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC Esirkepov current accumulators");
    cudaMemsetAsync(ctx->pic_esk, 0, bytes, s);
    ctx->pic_esk_elems = stride;
  }
  const long long rcap = std::max(1ll << 20, (long long)(ctx->n_upper / 64));
  const bool fill = !(a->flags & LBX_PIC_STABLE_ORDER);
  if (fill && (!ctx->pic_fill || ctx->pic_fill_cap < rcap)) {
    if (ctx->pic_fill) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_fill);
    }
    ctx->pic_fill = nullptr;
    if (cudaMalloc(&ctx->pic_fill, (size_t)rcap * 3 * 8) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC hole-filling lists");
    cudaMemsetAsync(ctx->pic_fill, 0, (size_t)rcap * 3 * 8, s);
    ctx->pic_fill_cap = rcap;
  }
  // fixed-point scale: a particle's largest node value, max(|q w| / dt, |q w|),
  // maps to <= 2^20 (warp sums of 32 fit int32)
  const double vmax = std::fabs(a->q_times_w) / std::min(a->dt, 1.0);
  int e2 = 0;
  std::frexp(1048576.0 / vmax, &e2);
  const double jscale = std::ldexp(1.0, e2 - 1);
  EskParams e{};
  PicParams& p = e.b;
  p.z = a->z;
  p.x = a->x;
  p.uz = a->uz;
  p.ux = a->ux;
  p.uy = a->uy;
  p.oz = a->z;
  p.ox = a->x;
  p.ouz = a->uz;
  p.oux = a->ux;
  p.ouy = a->uy;
  for (int c = 0; c < 6; ++c) p.F[c] = a->fields[c];
  p.pitch = a->nx + 2;
  p.dep_box = reinterpret_cast<int*>(ctx->pic_esk + 3 * stride);
  p.removed_list = fill ? ctx->pic_fill : nullptr;
  p.removed_cap = fill ? ctx->pic_fill_cap : 0;
  p.nz = a->nz;
  p.nx = a->nx;
  p.qm = a->q_over_m;
  p.qw = a->q_times_w;
  p.dt = a->dt;
  int l2 = 0;
  while ((1 << l2) < a->box_size) ++l2;
  p.log2m = l2;
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
  const long long rows = (long long)(a->nz + 5) * (a->nx + 5);
  if (!ctx->pic_quad || ctx->pic_quads < rows) {
    if (ctx->pic_quad) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_quad);
    }
    ctx->pic_quad = nullptr;
    if (cudaMalloc(&ctx->pic_quad, (size_t)rows * 6 * sizeof(float4)) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC row-quad field buffer");
    ctx->pic_quads = rows;
  }
  float4* R = static_cast<float4*>(ctx->pic_quad);
  for (int c = 0; c < 6; ++c) e.R[c] = R + c * rows;
  e.rpitch = a->nx + 5;
  {
    const unsigned rg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (rows + 255) / 256));
    esk_rows_kernel<<<rg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                       a->fields[4], a->fields[5], R, a->nz, a->nx);
  }
  e.o.J = ctx->pic_esk;
  e.o.stride = stride;
  e.o.apitch = apitch;
  e.o.cz = (float)(-(a->q_times_w / a->dt) * jscale);
  e.o.cy = (float)(a->q_times_w * jscale);
  const bool clock = (a->flags & LBX_STEP_CLOCK) != 0;
  void (*kern)(EskParams) = nullptr;
  switch (K) {
    case 1: kern = clock ? pic_esk_kernel<1, true> : pic_esk_kernel<1, false>; break;
    case 2: kern = clock ? pic_esk_kernel<2, true> : pic_esk_kernel<2, false>; break;
    case 3: kern = clock ? pic_esk_kernel<3, true> : pic_esk_kernel<3, false>; break;
    default: return set_error(LBX_EINVAL, "shape_order must be 0 (CIC direct) or 1, 2, 3");
  }
  const int NE = K == 1 ? EskBlock<1>::NE : (K == 2 ? EskBlock<2>::NE : EskBlock<3>::NE);
  const size_t smem = (size_t)nb * 8 + (size_t)(kEB / 32) * NE * 32 * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return cuda_fail(ea, "cudaFuncSetAttribute(esk)");
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEB, smem);
  long long grid = (long long)std::max(per_sm, 1) * ctx->num_sms;
  if (ctx->grid_override > 0) grid = ctx->grid_override;
  grid = std::max(1ll, std::min(grid, (long long)((ctx->n_upper + kEB - 1) / kEB)));
  kern<<<(unsigned)grid, kEB, smem, s>>>(e);
  cudaError_t er = cudaGetLastError();
  if (er != cudaSuccess) return cuda_fail(er, "pic_esk_kernel launch");
  if (fill) {
    const long long fc = ctx->pic_fill_cap;
    const unsigned fg2 = (unsigned)std::max(1, ctx->num_sms * 2);
    pic_fill_mark_kernel<<<fg2, 256, 0, s>>>(ctx->st, ctx->pic_fill, fc, ctx->pic_fill + fc,
                                             ctx->pic_fill + 2 * fc);
    pic_fill_move_kernel<<<fg2, 256, 0, s>>>(ctx->st, fc, ctx->pic_fill + fc, ctx->pic_fill + 2 * fc,
                                             a->z, a->x, a->uz, a->ux, a->uy);
    pic_fill_done_kernel<<<1, 1, 0, s>>>(ctx->st, fc);
  }
  rc = launch_compact(ctx, a->z, a->x, a->uz, a->ux, a->uy, nullptr, (double)a->nz, (double)a->nx, s);
  if (rc) return rc;
  if (a->flags & LBX_PIC_DEFER_CURRENT) return LBX_OK;   // multi-GPU: sums exchanged first
  return esk_finish(ctx, a, s);
}

// Esirkepov node sums -> current arrays (cleared), then the Yee update.
int esk_finish(lbx_ctx* ctx, const lbx_pic_args* a, cudaStream_t s) {
  const int apitch = a->nx + 2 * kEskG;
  const long long stride = (long long)(a->nz + 2 * kEskG) * apitch;
  if (!ctx->pic_esk || ctx->pic_esk_elems != stride)
    return set_error(LBX_EINVAL, "lbx_pic_finish without a deferred Esirkepov step on this grid");
  const double vmax = std::fabs(a->q_times_w) / std::min(a->dt, 1.0);
  int e2 = 0;
  std::frexp(1048576.0 / vmax, &e2);
  const double jscale = std::ldexp(1.0, e2 - 1);
  const unsigned cg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (stride + 255) / 256));
  pic_esk_current_kernel<<<cg, 256, 0, s>>>(ctx->pic_esk, stride, apitch, a->current[0],
                                            a->current[1], a->current[2], a->nz, a->nx,
                                            1.0 / jscale);
  cudaError_t er = cudaGetLastError();
  if (er != cudaSuccess) return cuda_fail(er, "current launch");
  if (a->flags & LBX_PIC_NO_FIELD_SOLVE) return LBX_OK;
  const int pitch = a->nx + 2;
  const long long cells = (long long)a->nz * a->nx;
  const unsigned fg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (cells + 255) / 256));
  pic_b_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->nz, a->nx, pitch, a->dt);
  pic_e_kernel<<<fg, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2], a->fields[3],
                                  a->fields[4], a->fields[5], a->current[0], a->current[1],
                                  a->current[2], a->nz, a->nx, pitch, a->dt);
  er = cudaGetLastError();
  if (er != cudaSuccess) return cuda_fail(er, "field solve launch");
  return LBX_OK;
}

}  // namespace
}  // namespace lbx

using namespace lbx;

extern "C" int lbx_pic_step(lbx_ctx* ctx, const lbx_pic_args* a, void* stream) {
  clear_error();
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  if (a->nz < 1 || a->nx < 1) return set_error(LBX_EINVAL, "grid must be at least 1x1");
  if ((long long)(a->nz + 1) * (a->nx + 1) >= (1ll << 31) / 16)
    return set_error(LBX_EINVAL, "PIC grid too large (quad index must fit 32 bits)");
  if (a->box_size < 1 || a->nz % a->box_size || a->nx % a->box_size ||
      (a->box_size & (a->box_size - 1)))
    return set_error(LBX_EINVAL, "PIC box_size must be a power of two dividing the grid");
  if (!(a->dt > 0.0 && a->dt < 0.7))
    return set_error(LBX_EINVAL, "dt must be in (0, 0.7) (2D CFL with unit cells)");
  for (int c = 0; c < 6; ++c)
    if (!a->fields[c]) return set_error(LBX_EINVAL, "NULL field array");
  for (int c = 0; c < 3; ++c)
    if (!a->current[c]) return set_error(LBX_EINVAL, "NULL current array");
  if (!(a->q_times_w != 0.0)) return set_error(LBX_EINVAL, "q_times_w must be nonzero");
  if (a->shape_order) return pic_step_esirkepov(ctx, a, (cudaStream_t)stream);
  const bool sorted = a->out[0] != nullptr;
  uintptr_t al = (uintptr_t)a->z | (uintptr_t)a->x | (uintptr_t)a->uz | (uintptr_t)a->ux |
                 (uintptr_t)a->uy;
  for (int c = 0; c < 5; ++c) {
    if (sorted && !a->out[c]) return set_error(LBX_EINVAL, "sorted mode needs all 5 output arrays");
    al |= (uintptr_t)a->out[c];
  }
  if (al & 31u) return set_error(LBX_EINVAL, "particle arrays must be 32-byte aligned");
  if (!(a->q_times_w != 0.0)) return set_error(LBX_EINVAL, "q_times_w must be nonzero");
  const bool tiled = (a->flags & LBX_PIC_TILED) != 0;
  if (tiled && sorted) return set_error(LBX_EINVAL, "LBX_PIC_TILED runs in place (no out[])");
  if ((a->flags & LBX_PIC_FAST) && sorted)
    return set_error(LBX_EINVAL, "LBX_PIC_FAST runs in place");
  if (tiled && (a->flags & LBX_PIC_DEFER_CURRENT))
    return set_error(LBX_EINVAL, "LBX_PIC_TILED does not support LBX_PIC_DEFER_CURRENT");
  if (tiled && (ctx->pic_tiles_nz != a->nz || ctx->pic_tiles_nx != a->nx))
    return set_error(LBX_EINVAL, "LBX_PIC_TILED needs lbx_pic_sort with LBX_PIC_TILED on this grid first");
  const int nbz = a->nz / a->box_size, nbx = a->nx / a->box_size, nb = nbz * nbx;
  if (nb > 4096) return set_error(LBX_EINVAL, "PIC step supports <= 4096 boxes");
  int rc = ensure_accumulators(ctx, nb);
  if (rc) return rc;
  rc = reserve_status(ctx, ctx->n_upper);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const long long cells = (long long)a->nz * a->nx;
  const long long quads = (long long)(a->nz + 1) * (a->nx + 1);
  if (!sorted) ctx->pic_sort_next = nullptr;   // an in-place step invalidates the cell slots
  const long long jn_stride = (long long)(a->nz + 2) * (a->nx + 2);
  if (tiled && (!ctx->pic_jn || ctx->pic_jn_stride != jn_stride)) {
    if (ctx->pic_jn) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_jn);
    }
    ctx->pic_jn = nullptr;
    const size_t bytes = (size_t)jn_stride * 3 * 8 + 16;
    if (cudaMalloc(&ctx->pic_jn, bytes) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC node current accumulators");
    cudaMemsetAsync(ctx->pic_jn, 0, bytes, s);
    ctx->pic_jn_stride = jn_stride;
  }
  if (!tiled && (!ctx->pic_acc || ctx->pic_cells < cells)) {
    if (ctx->pic_acc) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_acc);
    }
    ctx->pic_acc = nullptr;
    const size_t bytes = (size_t)cells * kNodes * 8 + 16;
    if (cudaMalloc(&ctx->pic_acc, bytes) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC current accumulators");
    cudaMemsetAsync(ctx->pic_acc, 0, bytes, s);
    ctx->pic_cells = cells;
  }
  if (!tiled && (!ctx->pic_quad || ctx->pic_quads < quads)) {
    if (ctx->pic_quad) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_quad);
    }
    ctx->pic_quad = nullptr;
    if (cudaMalloc(&ctx->pic_quad, (size_t)quads * 6 * sizeof(float4)) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC quad field buffer");
    ctx->pic_quads = quads;
  }
  if (sorted && (!ctx->pic_sortbuf || ctx->pic_sort_cells < cells)) {
    if (ctx->pic_sortbuf) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_sortbuf);
    }
    ctx->pic_sortbuf = nullptr;
    const size_t bytes = ((size_t)cells * 2 + kScanBlocks) * sizeof(unsigned);
    if (cudaMalloc(&ctx->pic_sortbuf, bytes) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC sort buffers");
    cudaMemsetAsync(ctx->pic_sortbuf, 0, bytes, s);
    ctx->pic_sort_cells = cells;
    ctx->pic_sort_next = nullptr;
  }
  const long long rcap = std::max(1ll << 20, (long long)(ctx->n_upper / 64));
  const bool fill = sorted || !(a->flags & LBX_PIC_STABLE_ORDER);
  if (fill && (!ctx->pic_fill || ctx->pic_fill_cap < rcap)) {
    if (ctx->pic_fill) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_fill);
    }
    ctx->pic_fill = nullptr;
    if (cudaMalloc(&ctx->pic_fill, (size_t)rcap * 3 * 8) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC hole-filling lists");
    cudaMemsetAsync(ctx->pic_fill, 0, (size_t)rcap * 3 * 8, s);
    ctx->pic_fill_cap = rcap;
  }
  float4* Q = static_cast<float4*>(ctx->pic_quad);
  unsigned* cell_cnt = sorted ? ctx->pic_sortbuf : nullptr;
  unsigned* cursor = sorted ? ctx->pic_sortbuf + cells : nullptr;
  unsigned* block_sum = sorted ? ctx->pic_sortbuf + 2 * cells : nullptr;
  int* dep_box = tiled ? reinterpret_cast<int*>(ctx->pic_jn + 3 * jn_stride)
                       : reinterpret_cast<int*>(ctx->pic_acc + ctx->pic_cells * kNodes);
  PicParams p{};
  p.z = a->z;
  p.x = a->x;
  p.uz = a->uz;
  p.ux = a->ux;
  p.uy = a->uy;
  double* out[5] = {a->z, a->x, a->uz, a->ux, a->uy};
  if (sorted)
    for (int c = 0; c < 5; ++c) out[c] = a->out[c];
  p.oz = out[0];
  p.ox = out[1];
  p.ouz = out[2];
  p.oux = out[3];
  p.ouy = out[4];
  p.cell_cnt = cell_cnt;
  p.cursor = cursor;
  p.removed_list = fill ? ctx->pic_fill : nullptr;
  p.removed_cap = fill ? ctx->pic_fill_cap : 0;
  for (int c = 0; c < 6; ++c) p.Q[c] = Q + c * quads;
  for (int c = 0; c < 6; ++c) p.F[c] = a->fields[c];
  p.pitch = a->nx + 2;
  p.Jc = ctx->pic_acc;
  p.dep_box = dep_box;
  int e2 = 0;
  std::frexp(1048576.0 / std::fabs(a->q_times_w), &e2);  // scale = 2^floor(log2(2^20/|qw|))
  const double jscale = std::ldexp(1.0, e2 - 1);
  p.vscale = (float)jscale;
  p.nz = a->nz;
  p.nx = a->nx;
  p.qpitch = a->nx + 1;
  p.qm = a->q_over_m;
  p.qw = a->q_times_w;
  p.dt = a->dt;
  int l2 = 0;
  while ((1 << l2) < a->box_size) ++l2;
  p.log2m = l2;
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
  const int pitch = a->nx + 2;
  const unsigned qg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8, (quads + 255) / 256));
  if (sorted && (ctx->pic_sort_next != a->z || (a->flags & LBX_PIC_RESYNC))) {
    // the slots of the input's cells are unknown: count them (cell_cnt is zero here)
    const unsigned ng = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8,
                                                         (long long)(ctx->n_upper / kRun + 255) / 256));
    pic_count_kernel<<<ng, 256, 0, s>>>(a->z, a->x, ctx->st, cell_cnt, a->nx);
    pic_scan_reduce_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, cells, block_sum);
    pic_scan_apply_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, cells, block_sum, cursor);
  }
  // quad copy when nodes are shared by many particles (dense plasma), else
  // direct gather (LBX_PIC_QUAD / LBX_PIC_DIRECT force either)
  bool quad = ctx->n_upper >= 16 * cells;
  if (a->flags & LBX_PIC_QUAD) quad = true;
  if ((a->flags & LBX_PIC_DIRECT) || tiled) quad = false;
  pic_quad_kernel<<<quad ? qg : 1, 256, 0, s>>>(a->fields[0], a->fields[1], a->fields[2],
                                                 a->fields[3], a->fields[4], a->fields[5], Q,
                                                 quad ? quads : 0, p.qpitch, pitch, dep_box,
                                                 (a->flags & LBX_PIC_FAST) ? 1 : 0);
  const bool clock = (a->flags & LBX_STEP_CLOCK) != 0;
  const bool fast = (a->flags & LBX_PIC_FAST) != 0;
  size_t smem = (size_t)kPW * kQCap * sizeof(FlushEntry) + (size_t)nb * 8;
  void (*kern)(PicParams);
  const int ntx = (a->nx + kT - 1) / kT, ntz = (a->nz + kT - 1) / kT;
  if (tiled) {
    smem = (size_t)kPW * kQCapT * sizeof(FlushEntry) + (size_t)6 * kPatch * 4 +
           (size_t)6 * kPatch * 4 + (size_t)nb * 8;
    kern = fast ? (clock ? pic_tile_kernel<true, true> : pic_tile_kernel<false, true>)
                : (clock ? pic_tile_kernel<true> : pic_tile_kernel<false>);
    p.tile_rd = ctx->pic_tiles;
    p.Jn = ctx->pic_jn;
    p.jn_stride = jn_stride;
    p.ntx = ntx;
    p.ntiles = ntz * ntx;
  } else if (quad && !sorted && LBX_PIC_PIPE) {
    smem = (size_t)kPW * sizeof(PipeWarp) + (size_t)nb * 8;
    kern = fast ? (clock ? pic_pipe_kernel<true, true> : pic_pipe_kernel<false, true>)
                : (clock ? pic_pipe_kernel<true, false> : pic_pipe_kernel<false, false>);
  } else if (fast)
    kern = clock ? (quad ? pic_push_kernel<true, false, true, true> : pic_push_kernel<true, false, false, true>)
                 : (quad ? pic_push_kernel<false, false, true, true> : pic_push_kernel<false, false, false, true>);
  else if (quad)
    kern = clock ? (sorted ? pic_push_kernel<true, true, true> : pic_push_kernel<true, false, true>)
                 : (sorted ? pic_push_kernel<false, true, true> : pic_push_kernel<false, false, true>);
  else
    kern = clock ? (sorted ? pic_push_kernel<true, true, false> : pic_push_kernel<true, false, false>)
                 : (sorted ? pic_push_kernel<false, true, false> : pic_push_kernel<false, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(pic)");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPB, smem);
  long long grid = (long long)std::max(per_sm, 1) * ctx->num_sms;
  if (ctx->grid_override > 0) grid = ctx->grid_override;
  const long long units = (ctx->n_upper + kUnitP - 1) / kUnitP;
  grid = std::max(1ll, std::min(grid, tiled ? (long long)ntz * ntx : (units + kPW - 1) / kPW));
  kern<<<(unsigned)grid, kPB, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pic_push_kernel launch");
  if (fill) {
    const long long fc = ctx->pic_fill_cap;
    const unsigned fg2 = (unsigned)std::max(1, ctx->num_sms * 2);
    pic_fill_mark_kernel<<<fg2, 256, 0, s>>>(ctx->st, ctx->pic_fill, fc, ctx->pic_fill + fc,
                                             ctx->pic_fill + 2 * fc);
    pic_fill_move_kernel<<<fg2, 256, 0, s>>>(ctx->st, fc, ctx->pic_fill + fc, ctx->pic_fill + 2 * fc,
                                             out[0], out[1], out[2], out[3], out[4]);
    pic_fill_done_kernel<<<1, 1, 0, s>>>(ctx->st, fc);
  }
  rc = launch_compact(ctx, out[0], out[1], out[2], out[3], out[4], nullptr, (double)a->nz,
                      (double)a->nx, stream);
  if (rc) return rc;
  if (sorted) {   // next step's slots: exclusive scan of this step's kept particles per cell
    pic_scan_reduce_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, cells, block_sum);
    pic_scan_apply_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, cells, block_sum, cursor);
    ctx->pic_sort_next = out[0];
  }
  if (sorted) ctx->pic_tiles_nz = ctx->pic_tiles_nx = 0;   // sort-on-write moved the particles
  if (a->flags & LBX_PIC_DEFER_CURRENT) return LBX_OK;
  return pic_finish(ctx, a, s, jscale, tiled);
}


extern "C" int lbx_pic_sort(lbx_ctx* ctx, const lbx_pic_args* a, void* stream) {
  clear_error();
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  if (a->nz < 1 || a->nx < 1) return set_error(LBX_EINVAL, "grid must be at least 1x1");
  if ((long long)a->nz * a->nx >= (1ll << 31))
    return set_error(LBX_EINVAL, "PIC grid too large (cell index must fit 32 bits)");
  const double* in[5] = {a->z, a->x, a->uz, a->ux, a->uy};
  for (int c = 0; c < 5; ++c)
    if (!in[c] || !a->out[c]) return set_error(LBX_EINVAL, "lbx_pic_sort needs the 5 arrays and out[]");
  cudaStream_t s = (cudaStream_t)stream;
  const bool tiled = (a->flags & LBX_PIC_TILED) != 0;
  const int ntx = (a->nx + kT - 1) / kT, ntz = (a->nz + kT - 1) / kT;
  const long long ntiles = (long long)ntz * ntx;
  // keys: row-major cells, or tile-major (2^kTileShift per tile, ragged tiles padded)
  const long long keys = tiled ? ntiles << kTileShift : (long long)a->nz * a->nx;
  if (!ctx->pic_sortbuf || ctx->pic_sort_cells < keys) {
    if (ctx->pic_sortbuf) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_sortbuf);
    }
    ctx->pic_sortbuf = nullptr;
    const size_t bytes = ((size_t)keys * 2 + kScanBlocks) * sizeof(unsigned);
    if (cudaMalloc(&ctx->pic_sortbuf, bytes) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC sort buffers");
    cudaMemsetAsync(ctx->pic_sortbuf, 0, bytes, s);
    ctx->pic_sort_cells = keys;
  }
  if (tiled && (!ctx->pic_tiles || ctx->pic_tiles_cap < ntiles + 1)) {
    if (ctx->pic_tiles) {
      cudaDeviceSynchronize();
      cudaFree(ctx->pic_tiles);
    }
    ctx->pic_tiles = nullptr;
    if (cudaMalloc(&ctx->pic_tiles, (size_t)(ntiles + 1) * sizeof(unsigned)) != cudaSuccess)
      return set_error(LBX_EOOM, "PIC tile ranges");
    ctx->pic_tiles_cap = ntiles + 1;
  }
  unsigned* cell_cnt = ctx->pic_sortbuf;
  unsigned* cursor = ctx->pic_sortbuf + keys;
  unsigned* block_sum = ctx->pic_sortbuf + 2 * keys;
  // sorted mode keeps its cursors in the same buffer at a row-major stride,
  // which a padded tile-major count range can overlap
  if (tiled) cudaMemsetAsync(cell_cnt, 0, (size_t)keys * sizeof(unsigned), s);
  const unsigned ng = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 8,
                                                       (long long)(ctx->n_upper / kRun + 255) / 256));
  pic_count_kernel<<<ng, 256, 0, s>>>(a->z, a->x, ctx->st, cell_cnt, a->nx, tiled ? ntx : 0);
  pic_scan_reduce_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, keys, block_sum);
  pic_scan_apply_kernel<<<kScanBlocks, kScanThreads, 0, s>>>(cell_cnt, keys, block_sum, cursor,
                                                             tiled ? ctx->pic_tiles : nullptr);
  const unsigned sg = (unsigned)std::max(1ll, std::min((long long)ctx->num_sms * 16,
                                                       (long long)(ctx->n_upper + 255) / 256));
  pic_sort_scatter_kernel<<<sg, 256, 0, s>>>(a->z, a->x, a->uz, a->ux, a->uy, a->out[0], a->out[1],
                                             a->out[2], a->out[3], a->out[4], ctx->st, cursor,
                                             a->nx, tiled ? ntx : 0);
  ctx->pic_sort_next = nullptr;   // the cursors were consumed
  ctx->pic_tiles_nz = tiled ? a->nz : 0;
  ctx->pic_tiles_nx = tiled ? a->nx : 0;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pic sort launch");
  return LBX_OK;
}

extern "C" int lbx_pic_finish(lbx_ctx* ctx, const lbx_pic_args* a, void* stream) {
  clear_error();
  if (!ctx || !a) return set_error(LBX_EINVAL, "NULL argument");
  if (a->shape_order) {
    if (!(a->q_times_w != 0.0)) return set_error(LBX_EINVAL, "q_times_w must be nonzero");
    return esk_finish(ctx, a, (cudaStream_t)stream);
  }
  if (!ctx->pic_acc || ctx->pic_cells != (long long)a->nz * a->nx)
    return set_error(LBX_EINVAL, "lbx_pic_finish without a deferred lbx_pic_step on this grid");
  if (!(a->q_times_w != 0.0)) return set_error(LBX_EINVAL, "q_times_w must be nonzero");
  int e2 = 0;
  std::frexp(1048576.0 / std::fabs(a->q_times_w), &e2);
  return pic_finish(ctx, a, (cudaStream_t)stream, std::ldexp(1.0, e2 - 1));
}

extern "C" int lbx_pic_esk_current_view(lbx_ctx* ctx, uint64_t** j, int64_t* stride,
                                        int32_t* guard) {
  clear_error();
  if (!ctx || !j || !stride || !guard) return set_error(LBX_EINVAL, "NULL argument");
  if (!ctx->pic_esk) return set_error(LBX_EINVAL, "no Esirkepov PIC step has run on this context");
  *j = reinterpret_cast<uint64_t*>(ctx->pic_esk);
  *stride = ctx->pic_esk_elems;
  *guard = kEskG;
  return LBX_OK;
}

extern "C" int lbx_pic_current_view(lbx_ctx* ctx, uint64_t** jc, int64_t* cells, int32_t** box) {
  clear_error();
  if (!ctx || !jc || !cells || !box) return set_error(LBX_EINVAL, "NULL argument");
  if (!ctx->pic_acc) return set_error(LBX_EINVAL, "no PIC step has run on this context");
  *jc = reinterpret_cast<uint64_t*>(ctx->pic_acc);
  *cells = ctx->pic_cells;
  *box = reinterpret_cast<int32_t*>(ctx->pic_acc + ctx->pic_cells * kNodes);
  return LBX_OK;
}
