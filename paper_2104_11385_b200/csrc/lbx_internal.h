// Internal declarations shared by the libLBX translation units.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <string>

#include "lbx.h"

namespace lbx {

// Thread-local last-error slot behind lbx_last_error().
int set_error(int code, const char* fmt, ...);
void clear_error();

// Device-resident step state (one per context).  Written only by the
// kernels' last CTA (epilogue) and by stream-ordered host memcpys.
struct DevState {
  unsigned long long ticket;  // next tile ticket (reset to 0 by the epilogue)
  unsigned int done;          // CTAs finished (reset to 0 by the epilogue)
  unsigned int epoch;         // look-back epoch tag, 1..2^22-1
  long long n;                // live particles (input count of the next step)
  long long err;              // cumulative out-of-grid survivors
  unsigned long long leavers; // absorbed this step (push -> compaction handoff)
  long long first_leaver;     // lowest index absorbed this step (LLONG_MAX: none)
  long long n_old;            // count before this step's push (compaction input)
  unsigned long long staged;  // emigrant records staged this call
  unsigned long long removed_count;  // removed indices listed this call
  unsigned long long holes;          // hole-fill cursors
  unsigned long long movers;
  unsigned int rot;           // GpuClock chunk-rotation counter (stream_kernel)
};

// Host-side model of the particle state's pushed-and-binned step.
struct StepLaunch {
  double *z, *x, *vz, *vx;
  double ez, ex, m;
  int nbz, nbx;
  double wp, wc, cells;
  bool clock;
  long long* counts_out;
  double* cost_out;
  unsigned long long* clk_out;
  long long* n_out;
  long long* err_out;
};

}  // namespace lbx

namespace lbx {
struct HostPipe;
void destroy_pipe(HostPipe* hp);
}  // namespace lbx

struct lbx_ctx {
  int device = 0;
  int num_sms = 0;
  int64_t l2_bytes = 0;               // cudaDevAttrL2CacheSize
  lbx::DevState* st = nullptr;        // device
  unsigned long long* status = nullptr;  // look-back tile status words
  int64_t status_tiles = 0;
  unsigned long long* acc = nullptr;  // per-box accumulators [2][acc_boxes]
  int32_t acc_boxes = 0;
  int64_t n_upper = 0;                // host upper bound on the live count
  int grid_override = 0;
  int64_t* host_scratch = nullptr;    // pinned
  lbx::HostPipe* pipe = nullptr;      // lbx_advance_bin_host lanes (lazy)
  unsigned long long* pic_acc = nullptr;  // PIC cell-centric fixed-point current [cells][16]
  int64_t pic_cells = 0;                  //   + 4 ints: deposit bounding box
  void* pic_quad = nullptr;               // PIC quad-expanded fields (float4) [6][quads]
  int64_t pic_quads = 0;
  unsigned* pic_sortbuf = nullptr;        // PIC sorted mode: cell counts, cursors, block sums
  int64_t pic_sort_cells = 0;
  const void* pic_sort_next = nullptr;    // z array whose cell slots are in the cursors
  long long* pic_fill = nullptr;          // sorted mode: removed list, holes, tail flags [3][cap]
  int64_t pic_fill_cap = 0;
  unsigned* pic_tiles = nullptr;          // tiled mode: slot ranges of the last tile-major sort
  int64_t pic_tiles_cap = 0;
  int pic_tiles_nz = 0, pic_tiles_nx = 0; //   grid they describe (0: none)
  unsigned long long* pic_jn = nullptr;   // tiled mode: node-centric current [3][(nz+2)(nx+2)] + box
  int64_t pic_jn_stride = 0;
  unsigned long long* pic_esk = nullptr;  // Esirkepov: padded node current [3][(nz+2G)(nx+2G)]
  int64_t pic_esk_elems = 0;
  long long* fill_scratch = nullptr;      // hole-fill: holes[cap] + tail flags[cap]
  int64_t fill_cap = 0;
  bool timing = false;                    // lbx_ctx_enable_timing
  void* ev0 = nullptr;                    // cudaEvent_t
  void* ev1 = nullptr;
};

#include <vector>

namespace lbx {
// Implemented in lbx_balancer.cpp.
double pairwise_sum(const double* a, int64_t n);
int efficiency(const double* cost, const int64_t* owner, int64_t n, int32_t R, double* eff,
               int32_t* degenerate, std::vector<double>& scratch);
int knapsack(const double* v, int64_t n, int32_t R, double cap_factor, int64_t* owner);
int sfc(const double* cost, const int64_t* curve, int64_t n, int32_t R, int64_t* owner);
int measured_cost(const double* work, int64_t n, double amplitude, uint64_t seed, uint64_t step,
                  double* out);
// Implemented in lbx_kernels.cu.
int launch_push_step(lbx_ctx* ctx, const StepLaunch& a, void* stream,
                     const lbx_exchange_args* ex = nullptr, bool push = true);
int ensure_accumulators(lbx_ctx* ctx, int32_t nboxes);
// In-place stable compaction of particles whose (z, x) left the domain, as
// recorded by the preceding push (st->leavers / first_leaver); carries up to
// four more per-particle arrays (a..d, each may be NULL).
int launch_compact(lbx_ctx* ctx, double* z, double* x, double* a, double* b, double* c,
                   double* d, double ez, double ex, void* stream);
int reserve_status(lbx_ctx* ctx, int64_t capacity);
// Resident multi-step kernel (lbx_resident.cu): device control block and
// launch description.  kResSlots must match the kernel's accumulator ring.
constexpr int kResSlots = 8;
struct ResCtl {
  unsigned long long recorded;              // steps recorded (last + 1)
  unsigned long long n_acc[kResSlots];      // live particles of the slot's step
  unsigned long long err_acc;               // out-of-grid survivors this run
  unsigned long long n_final;
  unsigned int arrive[kResSlots];           // CTAs done with the slot's step
  unsigned int done;
  unsigned int abort;
};
struct ResidentLaunch {
  double *z, *x, *vz, *vx, *kvz, *kvx;
  long long n, first, last, kick_step;
  double ez, ex, m;
  int pow2, nbz, nbx;
  double wp, wc, cells;
  bool clock;
  ResCtl* ctl;                              // device
  unsigned long long* acc;                  // device [kResSlots][2 * nb]
  unsigned char* rec;                       // mapped host record ring (device pointer)
  size_t rec_bytes;
  int H;
  unsigned long long* flags;                // mapped [H] (device pointer)
  const volatile unsigned long long* consumed;
  const volatile unsigned* abort_h;
  unsigned long long* trace;                // NULL, or [3][last - first] timestamps
};
// Largest particle count the resident kernel holds for nb boxes, and its grid.
int resident_capacity(lbx_ctx* ctx, int nb, long long* max_particles, int* grid);
int launch_resident(lbx_ctx* ctx, const ResidentLaunch& a, void* stream);
// Timers strategy helpers (lbx_kernels.cu): phase 0 = box ids + counts,
// phase 1 = scatter indices into per-box segments (offsets from the host).
int launch_timers_sort(const double* z, const double* x, long long n, double m, int nbz, int nbx,
                       int* box, unsigned long long* counts, unsigned long long* cursors,
                       int* perm, const unsigned long long* offsets_host, void* stream,
                       int phase);
int launch_timers_push(double* z, double* x, const double* vz, const double* vx, const int* idx,
                       long long cnt, void* stream);
// CUPTI activity-record timer (lbx_cupti.cpp).
int cupti_acquire();
void cupti_release();
int cupti_stream(void* stream, uint32_t* id);
int cupti_collect(uint32_t stream_id, int n, double* dur_ns);
}  // namespace lbx

#ifdef __CUDACC__
namespace lbx {
// Last CTA of a step kernel: per-box totals -> the step record (counts,
// heuristic cost w_p*count + w_c*cells, clock tally << clk_shift), and the
// accumulators cleared for the next launch.  Every other CTA fenced its
// atomics before taking the done ticket, so L2 loads (ld.cg) see the totals;
// four loads per thread are in flight at once instead of one returning
// atomic exchange per box (the serial tail of small steps).
template <bool kClock>
__device__ __forceinline__ void step_record(unsigned long long* g_cnt, unsigned long long* g_clk,
                                            int nb, long long* counts_out, double* cost_out,
                                            unsigned long long* clk_out, double wp, double wc,
                                            double cells, int clk_shift) {
  constexpr int kU = 4;
  for (int b0 = threadIdx.x; b0 < nb; b0 += kU * blockDim.x) {
    unsigned long long c[kU], k[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int b = b0 + u * (int)blockDim.x;
      c[u] = b < nb ? __ldcg(g_cnt + b) : 0ull;
      k[u] = (kClock && b < nb) ? __ldcg(g_clk + b) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int b = b0 + u * (int)blockDim.x;
      if (b >= nb) break;
      __stcg(g_cnt + b, 0ull);
      if (counts_out) counts_out[b] = (long long)c[u];
      if (cost_out)
        cost_out[b] = __dadd_rn(__dmul_rn(wp, (double)(long long)c[u]), __dmul_rn(wc, cells));
      if (kClock) {
        __stcg(g_clk + b, 0ull);
        if (clk_out) clk_out[b] = k[u] << clk_shift;
      }
    }
  }
}
}  // namespace lbx
#endif
