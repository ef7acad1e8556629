// libLBX native stepping runtime: the per-step loop of workload.py:388-470
// (run_simulation) without Python in it.
//
// Two layers:
//   lbx_lb   host half of a step, given the step's global per-box counts
//            (and GpuClock tally / device heuristic cost): provider cost
//            (workload.py:414), efficiency, should_attempt/attempt_rebalance
//            (balancer.py:258-304), adoption, and the walltime-model columns
//            of step_walltime (workload.py:314-363) -- all bit-exact with the
//            reference.  Used by lbx_sim below and by the multi-GPU driver
//            (parallel.py) after the per-box tallies are all-reduced.
//   lbx_sim  single-GPU loop: one fused kernel launch per step whose last CTA
//            writes the step record straight into a mapped pinned ring slot
//            (no memcpy enqueued); the host consumes records up to `ring`
//            steps behind the device (on one GPU the mapping never feeds
//            back into particle data).  Capacity runs (OOM can halt the run)
//            use a depth of 1 so the device never passes the halting step.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lbx_internal.h"

using namespace lbx;

struct lbx_lb {
  lbx_sim_config cfg{};
  int32_t nbz = 0, nbx = 0, nb = 0;
  int32_t nby = 1;       // 3D (extent_y > 0)
  double cells = 0.0;    // cells per box: M^2 (2D) or M^3 (3D)
  std::vector<int64_t> curve, face_a, face_b;
  std::vector<int64_t> owner, prop, prev;
  std::vector<double> work, scratch, rank_acc;
  std::vector<int64_t> faces_per_rank;
  std::vector<double> rank3;   // per-rank cost / work / particle sums [3][R]
  int64_t fmax = 0;            // most off-rank faces of a rank under `owner`
  bool faces_dirty = true;     // owner changed since fmax was counted
  // calibrated GpuClock: tallies summed over the LB window (the steps since
  // the previous attempt), reset after every attempt
  std::vector<uint64_t> clk_acc;
  int64_t acc_n = 0, acc_steps = 0;
};

struct ProposalPool;

struct lbx_sim {
  lbx_ctx* ctx = nullptr;
  lbx_lb* lb = nullptr;
  double *z = nullptr, *x = nullptr, *vz = nullptr, *vx = nullptr;
  double *kvz = nullptr, *kvx = nullptr;
  int ring = 0;
  size_t rec_bytes = 0;
  unsigned char* ring_h = nullptr;
  unsigned char* ring_d = nullptr;
  std::vector<cudaEvent_t> ev, t0, t1;  // completion / kernel timing events
  bool timing = false;
  // Timers strategy (cost_kind == LBX_COST_TIMERS)
  int64_t n_host = 0;
  int* box = nullptr;
  int* perm = nullptr;
  double* zero_v = nullptr;
  unsigned long long* d_counts = nullptr;
  unsigned long long* d_cursors = nullptr;
  unsigned long long* h_counts = nullptr;   // pinned
  unsigned long long* h_offsets = nullptr;  // pinned
  std::vector<cudaEvent_t> tb0, tb1;
  std::vector<double> timers;
  // CUPTI strategy (cost_kind == LBX_COST_CUPTI): same per-box launches
  bool cupti = false;
  void* stream = nullptr;
  std::vector<double> spans;
  // CUDA-graph replay of whole kCycle-step cycles (surrogate physics): the
  // loop's own stream, one graph per (ring half, kicked, timing), captured
  // on first use and replayed -- one launch per 16 steps instead of three.
  cudaStream_t gs = nullptr;
  cudaEvent_t join = nullptr;
  cudaGraphExec_t gexec[2][2][2] = {};
  bool graphs = false;   // eligible (ring of 2 cycles, surrogate, not disabled)
  bool warm = false;     // a per-step launch has run (allocations are done)
  bool capturing = false;
  long long graph_cycles = 0;
  // resident multi-step kernel (lbx_resident.cu): surrogate physics, particle
  // set within shared-memory capacity, no per-step kernel timing
  bool resident = false;            // eligible configuration
  long long resident_max = 0;       // particle capacity for this box grid
  ResCtl* rctl = nullptr;           // device
  unsigned long long* racc = nullptr;      // device [kResSlots][2 * nb]
  unsigned char* rctl_h = nullptr;         // mapped: flags[ring], consumed, abort
  unsigned char* rctl_d = nullptr;
  long long resident_runs = 0;
  ProposalPool* pool = nullptr;            // resident loop: remap proposals off-thread
  // PIC physics
  float* fields[6] = {};
  float* current[3] = {};
  double* uy = nullptr;
};

namespace {

struct Rec {
  int64_t* counts;
  double* cost;
  uint64_t* clk;
  int64_t* n;
  int64_t* err;
};

Rec rec_at(unsigned char* base, size_t rec_bytes, int slot, int nb) {
  unsigned char* p = base + (size_t)slot * rec_bytes;
  Rec r;
  r.counts = reinterpret_cast<int64_t*>(p);
  r.cost = reinterpret_cast<double*>(p + 8 * (size_t)nb);
  r.clk = reinterpret_cast<uint64_t*>(p + 16 * (size_t)nb);
  r.n = reinterpret_cast<int64_t*>(p + 24 * (size_t)nb);
  r.err = r.n + 1;
  return r;
}

bool should_attempt(const lbx_sim_config& c, int64_t step) {
  if (c.static_step >= 0 && step == c.static_step) return true;
  return c.interval <= c.total_steps && step % c.interval == 0;
}

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(LBX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int validate(const lbx_sim_config& c) {
  if (c.box_size < 1 || c.extent_z % c.box_size || c.extent_x % c.box_size)
    return set_error(LBX_EINVAL, "box_size %d must divide the extents", c.box_size);
  if (c.n_ranks < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1");
  if (c.total_steps < 1) return set_error(LBX_EINVAL, "total_steps must be >= 1");
  if (c.interval < 1) return set_error(LBX_EINVAL, "interval must be >= 1");
  if (c.cost_kind < 0 || c.cost_kind > LBX_COST_CUPTI)
    return set_error(LBX_EINVAL, "unknown cost kind %d", c.cost_kind);
  if (c.physics != LBX_PHYSICS_SURROGATE && c.physics != LBX_PHYSICS_PIC)
    return set_error(LBX_EINVAL, "unknown physics %d", c.physics);
  if (c.clock_mode != LBX_CLOCK_RAW && c.clock_mode != LBX_CLOCK_CALIBRATED)
    return set_error(LBX_EINVAL, "unknown clock mode %d", c.clock_mode);
  if (c.physics == LBX_PHYSICS_PIC &&
      (c.cost_kind == LBX_COST_TIMERS || c.cost_kind == LBX_COST_CUPTI))
    return set_error(LBX_EINVAL, "Timers strategies are implemented for the surrogate push only");
  return LBX_OK;
}

}  // namespace

namespace lbx {

// Host half of one step (see file comment), in two stages:
//  lb_cost    the step's cost row (o->cost_trace) and traces -- a function of
//             the step's record and of earlier records only (the GpuClock
//             window restarts at every attempt step, adopted or not), never
//             of the mapping, so a pipelined caller may run it ahead;
//  lb_decide  efficiency under the current mapping, the remap attempt
//             (proposal computed here, or handed in by a caller that ran the
//             knapsack / SFC ahead on the same cost row), gate, walltime.
// `device_cost` is the heuristic cost formed on the device (NULL: form it
// here from counts -- same separately rounded products).  `clk` is the
// GpuClock tally (NULL unless cost_kind is GPUCLOCK).
int lb_cost(lbx_lb* s, int64_t step, const int64_t* counts, const double* device_cost,
            const uint64_t* clk, lbx_sim_outputs* o, const double* timers = nullptr) {
  const lbx_sim_config& c = s->cfg;
  const int nb = s->nb;
  const double cells = s->cells;
  double* cost = o->cost_trace + (size_t)step * nb;
  switch (c.cost_kind) {
    case LBX_COST_HEURISTIC:
      if (device_cost) {
        std::memcpy(cost, device_cost, sizeof(double) * nb);
      } else {
        for (int b = 0; b < nb; ++b) cost[b] = c.w_particle * (double)counts[b] + c.w_cell * cells;
      }
      break;
    case LBX_COST_MEASURED:
    case LBX_COST_INSTRUMENTED:
      for (int b = 0; b < nb; ++b) s->work[b] = c.work_wp * (double)counts[b] + c.work_wc * cells;
      measured_cost(s->work.data(), nb, c.noise_amplitude, c.noise_seed, (uint64_t)step, cost);
      break;
    case LBX_COST_GPUCLOCK:
      if (!clk) return set_error(LBX_EINVAL, "GpuClock costs need the clock tally");
      if (c.clock_mode == LBX_CLOCK_CALIBRATED) {
        // cost.py calibrated_gpuclock_cost: the same operations in the same
        // order (integer sums over the window, one scale, mul then add)
        if ((int)s->clk_acc.size() != nb) s->clk_acc.assign(nb, 0);
        uint64_t tot = 0;
        int64_t np_ = 0;
        for (int b = 0; b < nb; ++b) {
          s->clk_acc[b] += clk[b];
          tot += s->clk_acc[b];
          np_ += counts[b];
        }
        s->acc_n += np_;
        s->acc_steps += 1;
        const double mean_n = (double)s->acc_n / (double)s->acc_steps;
        const double scale = tot ? c.w_particle * mean_n / (double)tot : 0.0;
        const double cell = c.w_cell * cells;
        for (int b = 0; b < nb; ++b) cost[b] = (double)s->clk_acc[b] * scale + cell;
        if (should_attempt(c, step)) {   // new LB window after every attempt
          std::fill(s->clk_acc.begin(), s->clk_acc.end(), 0ull);
          s->acc_n = s->acc_steps = 0;
        }
      } else {
        for (int b = 0; b < nb; ++b) cost[b] = (double)clk[b];
      }
      break;
    case LBX_COST_TIMERS:
    case LBX_COST_CUPTI:
      if (!timers) return set_error(LBX_EINVAL, "Timers costs need per-box kernel timings");
      std::memcpy(cost, timers, sizeof(double) * nb);
      break;
    default:
      return set_error(LBX_EINVAL, "unknown cost kind %d", c.cost_kind);
  }
  if (o->count_trace) std::memcpy(o->count_trace + (size_t)step * nb, counts, 8 * (size_t)nb);
  if (o->clock_trace && clk) std::memcpy(o->clock_trace + (size_t)step * nb, clk, 8 * (size_t)nb);
  return LBX_OK;
}

// Remap proposal for one cost row (knapsack or SFC, as configured).
int lb_propose(const lbx_lb* s, const double* cost, int64_t* prop) {
  const lbx_sim_config& c = s->cfg;
  return c.strategy == LBX_STRATEGY_KNAPSACK ? knapsack(cost, s->nb, c.n_ranks, c.cap_factor, prop)
                                             : sfc(cost, s->curve.data(), s->nb, c.n_ranks, prop);
}

int lb_decide(lbx_lb* s, int64_t step, const int64_t* counts, int64_t n_alive,
              lbx_sim_outputs* o, int* adopted_out, int* halt, const int64_t* ready_prop) {
  const lbx_sim_config& c = s->cfg;
  const int nb = s->nb;
  const int32_t R = c.n_ranks;
  const double cells = s->cells;
  const double* cost = o->cost_trace + (size_t)step * nb;
  for (int b = 0; b < nb; ++b) s->work[b] = c.work_wp * (double)counts[b] + c.work_wc * cells;
  if (o->n_alive) o->n_alive[step] = n_alive;

  // One pass over the boxes: per-rank cost (efficiency), true work (compute
  // max) and particles (occupancy) under the current mapping.  Each rank's
  // sums still run in box order (numpy's bincount / add order), three
  // independent chains instead of three passes.
  if ((int32_t)s->rank3.size() != 3 * R) s->rank3.assign(3 * (size_t)R, 0.0);
  double* lc = s->rank3.data();
  double* lw = lc + R;
  double* ln = lw + R;
  auto rank_sums = [&](const int64_t* own, bool with_cost) {
    std::fill(s->rank3.begin(), s->rank3.end(), 0.0);
    if (with_cost) {
      for (int b = 0; b < nb; ++b) {
        const int64_t r = own[b];
        lc[r] += cost[b];
        lw[r] += s->work[b];
        ln[r] += (double)counts[b];
      }
    } else {
      for (int b = 0; b < nb; ++b) {
        const int64_t r = own[b];
        lw[r] += s->work[b];
        ln[r] += (double)counts[b];
      }
    }
  };
  rank_sums(s->owner.data(), true);

  // balance (balancer.py:258-304); efficiency as lbx::efficiency (mean / max)
  double e_cur = 1.0;
  {
    double top = lc[0];
    for (int32_t r = 1; r < R; ++r) top = std::max(top, lc[r]);
    if (top != 0.0) e_cur = (pairwise_sum(lc, R) / (double)R) / top;
  }
  double e_after = e_cur;
  const bool attempted = should_attempt(c, step);
  bool adopted = false;
  int64_t moved_particles = 0;
  if (attempted) {
    o->n_attempts += 1;
    if (ready_prop) {
      std::memcpy(s->prop.data(), ready_prop, 8 * (size_t)nb);
    } else {
      int rc = lb_propose(s, cost, s->prop.data());
      if (rc) return rc;
    }
    double e_prop = 1.0;
    efficiency(cost, s->prop.data(), nb, R, &e_prop, nullptr, s->scratch);
    const double need = c.threshold_relative ? e_cur * (1.0 + c.improvement_threshold)
                                             : e_cur + c.improvement_threshold;
    adopted = e_prop >= need && e_prop >= e_cur;
    if (adopted && c.migration_ratio > 0.0) {
      // price the redistribution against the load saved over one interval
      std::vector<double> lpc(R, 0.0), lpp(R, 0.0);
      double total_cost = 0.0;
      int64_t total_n = 0, moved = 0;
      for (int b = 0; b < nb; ++b) {
        lpc[s->owner[b]] += cost[b];
        lpp[s->prop[b]] += cost[b];
        total_cost += cost[b];
        total_n += counts[b];
        if (s->prop[b] != s->owner[b]) moved += counts[b];
      }
      const double mc = *std::max_element(lpc.begin(), lpc.end());
      const double mp = *std::max_element(lpp.begin(), lpp.end());
      const double per_push = total_n > 0 ? total_cost / (double)total_n : 0.0;
      const double saved = (double)c.interval * (mc - mp);
      adopted = saved > c.migration_ratio * per_push * (double)moved;
    }
    if (adopted) {
      for (int b = 0; b < nb; ++b)
        if (s->prop[b] != s->owner[b]) moved_particles += counts[b];
      s->owner.swap(s->prop);
      s->faces_dirty = true;
      rank_sums(s->owner.data(), false);   // walltime under the adopted mapping
      e_after = e_prop;
      if (o->adopt_steps) o->adopt_steps[o->n_adoptions] = step;
      if (o->adopt_owners)
        std::memcpy(o->adopt_owners + (size_t)o->n_adoptions * nb, s->owner.data(),
                    8 * (size_t)nb);
      o->n_adoptions += 1;
    }
  }

  // walltime model (workload.py:314-363)
  double compute_max = lw[0];
  for (int r = 1; r < R; ++r) compute_max = std::max(compute_max, lw[r]);
  if (s->faces_dirty) {   // off-rank faces change only with the mapping
    std::fill(s->faces_per_rank.begin(), s->faces_per_rank.end(), 0);
    for (size_t f = 0; f < s->face_a.size(); ++f) {
      const int64_t ra = s->owner[s->face_a[f]], rb = s->owner[s->face_b[f]];
      if (ra != rb) {
        s->faces_per_rank[ra] += 1;
        s->faces_per_rank[rb] += 1;
      }
    }
    s->fmax = s->faces_per_rank[0];
    for (int r = 1; r < R; ++r) s->fmax = std::max(s->fmax, s->faces_per_rank[r]);
    s->faces_dirty = false;
  }
  double comm_max = (double)s->fmax * c.comm_per_face;
  double gather = attempted ? c.gather : 0.0;
  double redis = 0.0;
  if (adopted)
    redis = c.redistribute_latency + c.redistribute_per_particle * (double)moved_particles;
  double occ = ln[0];
  for (int r = 1; r < R; ++r) occ = std::max(occ, ln[r]);
  const int64_t mrp = (int64_t)occ;
  const bool oom = c.capacity_particles >= 0 && mrp > c.capacity_particles;
  const double ov = c.overhead_factor;
  compute_max *= ov;
  comm_max *= ov;
  gather *= ov;
  redis *= ov;
  o->eff_before[step] = e_cur;
  o->eff_after[step] = e_after;
  o->adopted[step] = adopted;
  o->attempted[step] = attempted;
  o->compute_max[step] = compute_max;
  o->comm_max[step] = comm_max;
  o->gather[step] = gather;
  o->redistribute[step] = redis;
  o->walltime[step] = compute_max + comm_max + gather + redis;
  o->max_rank_particles[step] = mrp;
  o->oom[step] = oom;
  o->completed_steps = step + 1;
  if (adopted_out) *adopted_out = adopted ? 1 : 0;
  *halt = oom ? 1 : 0;
  return LBX_OK;
}

int lb_step(lbx_lb* s, int64_t step, const int64_t* counts, const double* device_cost,
            const uint64_t* clk, int64_t n_alive, lbx_sim_outputs* o, int* adopted_out,
            int* halt, const double* timers = nullptr) {
  int rc = lb_cost(s, step, counts, device_cost, clk, o, timers);
  if (rc) return rc;
  return lb_decide(s, step, counts, n_alive, o, adopted_out, halt, nullptr);
}

}  // namespace lbx

namespace {

// Timers strategy: per-box push launches bracketed by CUDA events (the
// paper's CUPTI-style per-kernel timing).  Box-sorts the
// particle indices first (needs the per-box counts on the host), then the
// fused kernel runs with zero velocity to count survivors, form the
// heuristic record and compact the absorbed particles.
int timers_prepare(lbx_sim* s, const double* vz, const double* vx, cudaStream_t st) {
  const lbx_sim_config& c = s->lb->cfg;
  const int nb = s->lb->nb;
  const long long n = s->n_host;
  int rc = launch_timers_sort(s->z, s->x, n, (double)c.box_size, s->lb->nbz, s->lb->nbx, s->box,
                              s->d_counts, s->d_cursors, s->perm, nullptr, st, 0);
  if (rc) return rc;
  cudaMemcpyAsync(s->h_counts, s->d_counts, (size_t)nb * 8, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "timers histogram");
  unsigned long long acc = 0;
  for (int b = 0; b < nb; ++b) {
    s->h_offsets[b] = acc;
    acc += s->h_counts[b];
  }
  rc = launch_timers_sort(s->z, s->x, n, (double)c.box_size, s->lb->nbz, s->lb->nbx, s->box,
                          s->d_counts, s->d_cursors, s->perm, s->h_offsets, st, 1);
  if (rc) return rc;
  for (int b = 0; b < nb; ++b) {
    const long long cnt = (long long)s->h_counts[b];
    if (!cnt) continue;
    if (!s->cupti) cudaEventRecord(s->tb0[b], st);
    rc = launch_timers_push(s->z, s->x, vz, vx, s->perm + s->h_offsets[b], cnt, st);
    if (rc) return rc;
    if (!s->cupti) cudaEventRecord(s->tb1[b], st);
  }
  return LBX_OK;
}

// Stream event record that, under graph capture, becomes an event-record
// node the host can wait on (a plain record would be a capture-internal join).
cudaError_t record(const lbx_sim* s, cudaEvent_t ev, cudaStream_t st) {
  return s->capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                      : cudaEventRecord(ev, st);
}

int launch_step(lbx_sim* s, int64_t step, cudaStream_t st) {
  const int slot = (int)(step % s->ring);
  if (s->timing) record(s, s->t0[slot], st);
  Rec d = rec_at(s->ring_d, s->rec_bytes, slot, s->lb->nb);
  const lbx_sim_config& c = s->lb->cfg;
  const bool kicked = step >= c.kick_step && s->kvz != nullptr;
  const bool timers = c.cost_kind == LBX_COST_TIMERS || c.cost_kind == LBX_COST_CUPTI;
  if (c.physics == LBX_PHYSICS_PIC) {
    lbx_pic_args pa{};
    pa.z = s->z;
    pa.x = s->x;
    pa.uz = kicked ? s->kvz : s->vz;
    pa.ux = kicked ? s->kvx : s->vx;
    pa.uy = s->uy;
    for (int k = 0; k < 6; ++k) pa.fields[k] = s->fields[k];
    for (int k = 0; k < 3; ++k) pa.current[k] = s->current[k];
    pa.nz = c.extent_z;
    pa.nx = c.extent_x;
    pa.box_size = c.box_size;
    pa.q_over_m = c.pic_q_over_m;
    pa.q_times_w = c.pic_q_times_w;
    pa.dt = c.pic_dt;
    pa.w_particle = c.w_particle;
    pa.w_cell = c.w_cell;
    pa.flags = (c.cost_kind == LBX_COST_GPUCLOCK ? LBX_STEP_CLOCK : 0u) | LBX_PIC_STABLE_ORDER;
    pa.counts_out = d.counts;
    pa.cost_out = d.cost;
    pa.clk_out = d.clk;
    pa.n_out = d.n;
    pa.err_out = d.err;
    int rc = lbx_pic_step(s->ctx, &pa, st);
    if (rc) return rc;
    if (s->timing) record(s, s->t1[slot], st);
    cudaError_t e = record(s, s->ev[slot], st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    return LBX_OK;
  }
  if (timers) {
    int rc = timers_prepare(s, kicked ? s->kvz : s->vz, kicked ? s->kvx : s->vx, st);
    if (rc) return rc;
  }
  StepLaunch a{};
  a.z = s->z;
  a.x = s->x;
  a.vz = timers ? s->zero_v : kicked ? s->kvz : s->vz;
  a.vx = timers ? s->zero_v : kicked ? s->kvx : s->vx;
  a.ez = (double)c.extent_z;
  a.ex = (double)c.extent_x;
  a.m = (double)c.box_size;
  a.nbz = s->lb->nbz;
  a.nbx = s->lb->nbx;
  a.wp = c.w_particle;
  a.wc = c.w_cell;
  a.cells = (double)c.box_size * (double)c.box_size;
  a.clock = c.cost_kind == LBX_COST_GPUCLOCK;
  a.counts_out = reinterpret_cast<long long*>(d.counts);
  a.cost_out = d.cost;
  a.clk_out = a.clock ? reinterpret_cast<unsigned long long*>(d.clk) : nullptr;
  a.n_out = reinterpret_cast<long long*>(d.n);
  a.err_out = reinterpret_cast<long long*>(d.err);
  int rc = launch_push_step(s->ctx, a, st);
  if (rc) return rc;
  if (s->timing) record(s, s->t1[slot], st);
  cudaError_t e = record(s, s->ev[slot], st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  return LBX_OK;
}

constexpr int kCycle = 16;

void drop_graphs(lbx_sim* s) {
  for (auto& a : s->gexec)
    for (auto& b : a)
      for (auto& g : b)
        if (g) cudaGraphExecDestroy(g), g = nullptr;
}

bool kicked_at(const lbx_sim* s, int64_t step) {
  return step >= s->lb->cfg.kick_step && s->kvz != nullptr;
}

// Launches steps [step, step + kCycle) as one graph (captured the first time
// this (half, kicked, timing) combination is seen).  Returns false -- with
// nothing launched and graphs disabled for this sim -- if capture fails.
bool launch_cycle(lbx_sim* s, int64_t step, cudaStream_t st) {
  const int half = (int)((step / kCycle) & 1);
  const int kick = kicked_at(s, step) ? 1 : 0;
  cudaGraphExec_t& ge = s->gexec[half][kick][s->timing ? 1 : 0];
  if (!ge) {
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    s->capturing = ok;
    for (int j = 0; ok && j < kCycle; ++j) ok = launch_step(s, step + j, st) == LBX_OK;
    s->capturing = false;
    const cudaError_t ec = cudaStreamEndCapture(st, &g);
    ok = ok && ec == cudaSuccess && g != nullptr &&
         cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      if (std::getenv("LBX_GRAPH_DEBUG"))
        std::fprintf(stderr, "lbx: graph capture failed at step %lld: end=%s last=%s (%s)\n",
                     (long long)step, cudaGetErrorString(ec), cudaGetErrorString(cudaGetLastError()),
                     lbx_last_error());
      ge = nullptr;
      cudaGetLastError();   // clear the capture error; per-step launches from here on
      clear_error();
      s->graphs = false;
      return false;
    }
  }
  if (cudaGraphLaunch(ge, st) != cudaSuccess) {
    cudaGetLastError();
    s->graphs = false;
    return false;
  }
  ++s->graph_cycles;
  return true;
}

int process_step(lbx_sim* s, int64_t step, lbx_sim_outputs* o, int* halt) {
  const int slot = (int)(step % s->ring);
  cudaError_t e = cudaEventSynchronize(s->ev[slot]);
  if (e != cudaSuccess) return cuda_fail(e, "step kernel");
  Rec h = rec_at(s->ring_h, s->rec_bytes, slot, s->lb->nb);
  if (s->timing && o->kernel_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->t0[slot], s->t1[slot]);
    o->kernel_ms[step] = ms;
  }
  if (*h.err != 0)
    return set_error(LBX_ERANGE, "step %lld: %lld survivors fall outside the box grid",
                     (long long)step, (long long)*h.err);
  const bool clock = s->lb->cfg.cost_kind == LBX_COST_GPUCLOCK;
  const double* timers = nullptr;
  if (s->cupti) {
    int busy = 0;
    for (int b = 0; b < s->lb->nb; ++b) busy += s->h_counts[b] != 0;
    uint32_t sid = 0;
    int rc = cupti_stream(s->stream, &sid);
    if (!rc) rc = cupti_collect(sid, busy, s->spans.data());
    if (rc) return rc;
    for (int b = 0, k = 0; b < s->lb->nb; ++b)
      s->timers[b] = s->h_counts[b] ? s->spans[k++] / 1000.0 : 0.0;  // microseconds
    timers = s->timers.data();
    if (o->clock_trace)
      for (int b = 0; b < s->lb->nb; ++b)
        o->clock_trace[(size_t)step * s->lb->nb + b] = (uint64_t)(s->timers[b] * 1000.0);
  } else if (s->lb->cfg.cost_kind == LBX_COST_TIMERS) {
    for (int b = 0; b < s->lb->nb; ++b) {
      float ms = 0.f;
      if (s->h_counts[b]) cudaEventElapsedTime(&ms, s->tb0[b], s->tb1[b]);
      s->timers[b] = 1000.0 * (double)ms;  // microseconds
    }
    timers = s->timers.data();
    if (o->clock_trace)  // record the per-box launch times (ns) in the clock trace slot
      for (int b = 0; b < s->lb->nb; ++b)
        o->clock_trace[(size_t)step * s->lb->nb + b] = (uint64_t)(s->timers[b] * 1000.0);
  }
  s->n_host = *h.n;
  return lb_step(s->lb, step, h.counts, h.cost, clock ? h.clk : nullptr, *h.n, o, nullptr, halt,
                 timers);
}

}  // namespace

// Proposal pool of the resident loop: worker threads run the remap proposal
// (knapsack / SFC) of attempt steps whose cost rows the cost stage formed
// ahead of the decide stage.  One job per attempt step, at most H steps
// ahead (slot = step % H); the proposal is a pure function of the cost row,
// so it is the same mapping lb_decide would compute itself.
struct ProposalPool {
  struct Job {
    int64_t step = -1;
    const double* cost = nullptr;
    std::vector<int64_t> prop;
    int rc = 0;
    std::string err;
    std::atomic<int> state{0};   // 0 free, 1 queued / running, 2 done
  };
  const lbx_lb* lb;
  std::vector<Job> jobs;
  std::deque<Job*> queue;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::thread> th;
  bool stop = false;

  ProposalPool(const lbx_lb* l, int slots, int workers) : lb(l), jobs(slots) {
    for (auto& j : jobs) j.prop.assign(l->nb, 0);
    for (int w = 0; w < workers; ++w) th.emplace_back([this] { run(); });
  }
  ~ProposalPool() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  void run() {
    while (true) {
      Job* j = nullptr;
      {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [this] { return stop || !queue.empty(); });
        if (stop && queue.empty()) return;
        j = queue.front();
        queue.pop_front();
      }
      j->rc = lb_propose(lb, j->cost, j->prop.data());
      if (j->rc) j->err = lbx_last_error();
      j->state.store(2, std::memory_order_release);
    }
  }
  void submit(int64_t step, const double* cost) {
    Job& j = jobs[step % (int64_t)jobs.size()];
    j.step = step;
    j.cost = cost;
    j.rc = 0;
    j.state.store(1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(mu);
      queue.push_back(&j);
    }
    cv.notify_one();
  }
  int wait(int64_t step, const int64_t** prop) {
    Job& j = jobs[step % (int64_t)jobs.size()];
    if (j.step != step || j.state.load(std::memory_order_relaxed) == 0)
      return set_error(LBX_EINVAL, "no proposal queued for step %lld", (long long)step);
    while (j.state.load(std::memory_order_acquire) != 2) std::this_thread::yield();
    j.state.store(0, std::memory_order_relaxed);
    if (j.rc) return set_error(j.rc, "%s", j.err.c_str());
    *prop = j.prop.data();
    return LBX_OK;
  }
  void drain() {   // let queued / running jobs finish (their cost rows stay valid)
    for (auto& j : jobs)
      while (j.state.load(std::memory_order_acquire) == 1) std::this_thread::yield();
    for (auto& j : jobs) j.state.store(0, std::memory_order_relaxed);
  }
};

namespace {

// Resident path (lbx_resident.cu): one cooperative launch runs steps
// [first, last); the host follows the per-step ready flags the kernel raises
// in mapped memory, runs the host LB step on each record and reports its
// progress back (the kernel waits only when H steps ahead of the host).  The
// run ends with the look-back compaction of the CTA ranges' holes.
int run_resident(lbx_sim* s, int64_t first, int64_t last, lbx_sim_outputs* o, cudaStream_t st,
                 int* halt) {
  const lbx_sim_config& c = s->lb->cfg;
  const int nb = s->lb->nb;
  const int H = s->ring;
  volatile unsigned long long* flags = reinterpret_cast<unsigned long long*>(s->rctl_h);
  volatile unsigned long long* consumed = flags + H;
  volatile unsigned* abort_h = reinterpret_cast<volatile unsigned*>(flags + H + 1);
  for (int i = 0; i < H; ++i) flags[i] = 0ull;
  *consumed = (unsigned long long)first;
  *abort_h = 0u;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  const bool kick = s->kvz != nullptr;
  ResidentLaunch a{};
  a.z = s->z;
  a.x = s->x;
  a.vz = s->vz;
  a.vx = s->vx;
  a.kvz = s->kvz;
  a.kvx = s->kvx;
  a.n = s->n_host;
  a.first = first;
  a.last = last;
  a.kick_step = kick ? c.kick_step : LLONG_MAX;
  a.ez = (double)c.extent_z;
  a.ex = (double)c.extent_x;
  a.m = (double)c.box_size;
  a.pow2 = (c.box_size & (c.box_size - 1)) == 0;
  a.nbz = s->lb->nbz;
  a.nbx = s->lb->nbx;
  a.wp = c.w_particle;
  a.wc = c.w_cell;
  a.cells = (double)c.box_size * (double)c.box_size;
  a.clock = c.cost_kind == LBX_COST_GPUCLOCK;
  a.ctl = s->rctl;
  a.acc = s->racc;
  a.rec = s->ring_d;
  a.rec_bytes = s->rec_bytes;
  a.H = H;
  a.flags = reinterpret_cast<unsigned long long*>(s->rctl_d);
  a.consumed = reinterpret_cast<unsigned long long*>(s->rctl_d) + H;
  a.abort_h = reinterpret_cast<const unsigned*>(reinterpret_cast<unsigned long long*>(s->rctl_d) + H + 1);
#ifdef LBX_RES_TRACE
  unsigned long long* trace_d = nullptr;
  cudaMalloc(&trace_d, 3 * sizeof(unsigned long long) * (last - first));
  cudaMemset(trace_d, 0, 3 * sizeof(unsigned long long) * (last - first));
  a.trace = trace_d;
#endif
  int rc = launch_resident(s->ctx, a, st);
  if (rc) return rc;
  ++s->resident_runs;
  auto fail = [&](int code) {   // stop the kernel, reset its control state
    if (s->pool) s->pool->drain();
    *abort_h = 1u;
    cudaStreamSynchronize(st);
    cudaGetLastError();
    cudaMemsetAsync(s->rctl, 0, sizeof(ResCtl), st);
    cudaMemsetAsync(s->racc, 0, sizeof(unsigned long long) * 2 * kResSlots * nb, st);
    cudaStreamSynchronize(st);
    return code;
  };
  // Records are taken in two passes: the cost stage (lb_cost) runs ahead on
  // every record that has arrived, and hands each attempt step's cost row to
  // the proposal pool (the knapsack / SFC of the step, off this thread); the
  // decide stage (lb_decide) follows in step order and collects the proposal.
  ProposalPool* pool = s->pool;
  auto ready = [&](int64_t t) { return flags[t % H] == (unsigned long long)(t + 1); };
  int64_t ahead = first;   // next step for the cost stage
  for (int64_t step = first; step < last; ++step) {
    const int slot = (int)(step % H);
    unsigned spins = 0;
    while (!ready(step)) {
      if ((++spins & 4095u) == 0u) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q != cudaErrorNotReady && !ready(step)) {
          return fail(q == cudaSuccess ? set_error(LBX_ECUDA, "resident kernel ended before step %lld",
                                                   (long long)step)
                                       : cuda_fail(q, "resident kernel"));
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    while (ahead < last && ahead < step + H && (ahead == step || ready(ahead))) {
      std::atomic_thread_fence(std::memory_order_acquire);
      Rec r = rec_at(s->ring_h, s->rec_bytes, (int)(ahead % H), nb);
      if (*r.err != 0)
        return fail(set_error(LBX_ERANGE, "step %lld: %lld survivors fall outside the box grid",
                              (long long)ahead, (long long)*r.err));
      rc = lb_cost(s->lb, ahead, r.counts, nullptr, a.clock ? r.clk : nullptr, o);
      if (rc) return fail(rc);
      if (pool && should_attempt(c, ahead))
        pool->submit(ahead, o->cost_trace + (size_t)ahead * nb);
      ++ahead;
    }
    Rec h = rec_at(s->ring_h, s->rec_bytes, slot, nb);
    s->n_host = *h.n;
    const int64_t* prop = nullptr;
    if (pool && should_attempt(c, step)) {
      rc = pool->wait(step, &prop);
      if (rc) return fail(rc);
    }
    rc = lb_decide(s->lb, step, h.counts, *h.n, o, nullptr, halt, prop);
    if (rc) return fail(rc);
    std::atomic_thread_fence(std::memory_order_release);
    *consumed = (unsigned long long)(step + 1);
  }
  // holes -> stable compaction; velocities live in the kick arrays once kicked
  const bool kicked = kick && last > c.kick_step;
  rc = launch_compact(s->ctx, s->z, s->x, kicked ? s->kvz : s->vz, kicked ? s->kvx : s->vx,
                      (kick && !kicked) ? s->kvz : nullptr, (kick && !kicked) ? s->kvx : nullptr,
                      (double)c.extent_z, (double)c.extent_x, st);
  if (rc) return rc;
#ifdef LBX_RES_TRACE
  {
    const int64_t T = last - first;
    std::vector<unsigned long long> tr(3 * T);
    cudaStreamSynchronize(st);
    cudaMemcpy(tr.data(), trace_d, tr.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(trace_d);
    double per = T > 1 ? (double)(tr[T - 1] - tr[0]) / (T - 1) : 0, rec = 0, lag = 0;
    for (int64_t i = 0; i < T; ++i) {
      rec += (double)(tr[2 * T + i] - tr[T + i]);
      lag += (double)(tr[T + i] - tr[i]);
    }
    std::fprintf(stderr, "lbx resident trace: %lld steps, CTA0 step period %.0f ns, courier %.0f ns, "
                 "step start -> record start %.0f ns\n", (long long)T, per, rec / T, lag / T);
  }
#endif
  return LBX_OK;
}

}  // namespace

extern "C" {

int lbx_lb_create(lbx_lb** out, const lbx_sim_config* cfg, const int64_t* initial_owner) {
  clear_error();
  if (!out || !cfg) return set_error(LBX_EINVAL, "NULL argument");
  int rc = validate(*cfg);
  if (rc) return rc;
  const lbx_sim_config& c = *cfg;
  lbx_lb* s = new lbx_lb();
  s->cfg = c;
  s->nbz = c.extent_z / c.box_size;
  s->nbx = c.extent_x / c.box_size;
  const bool three_d = c.extent_y > 0;
  if (three_d) {
    if (c.extent_y % c.box_size) {
      delete s;
      return set_error(LBX_EINVAL, "box_size %d must divide the y-extent", c.box_size);
    }
    s->nby = c.extent_y / c.box_size;
  }
  s->nb = s->nbz * s->nby * s->nbx;
  s->cells = three_d ? (double)c.box_size * c.box_size * c.box_size
                     : (double)((int64_t)c.box_size * c.box_size);
  const int nb = s->nb;
  s->curve.resize(nb);
  if (three_d) lbx_morton_order_3d(s->nbz, s->nby, s->nbx, s->curve.data());
  else lbx_morton_order(s->nbz, s->nbx, s->curve.data());
  const int NY = s->nby, NX = s->nbx;
  auto id = [&](int bz, int by, int bx) { return ((int64_t)bz * NY + by) * NX + bx; };
  for (int bz = 0; bz + 1 < s->nbz; ++bz)   // z-neighbours first, then y, then x
    for (int by = 0; by < NY; ++by)
      for (int bx = 0; bx < NX; ++bx) {
        s->face_a.push_back(id(bz, by, bx));
        s->face_b.push_back(id(bz + 1, by, bx));
      }
  for (int bz = 0; bz < s->nbz; ++bz)
    for (int by = 0; by + 1 < NY; ++by)
      for (int bx = 0; bx < NX; ++bx) {
        s->face_a.push_back(id(bz, by, bx));
        s->face_b.push_back(id(bz, by + 1, bx));
      }
  for (int bz = 0; bz < s->nbz; ++bz)
    for (int by = 0; by < NY; ++by)
      for (int bx = 0; bx + 1 < NX; ++bx) {
        s->face_a.push_back(id(bz, by, bx));
        s->face_b.push_back(id(bz, by, bx + 1));
      }
  s->owner.assign(nb, 0);
  if (initial_owner) {
    for (int b = 0; b < nb; ++b) {
      if (initial_owner[b] < 0 || initial_owner[b] >= c.n_ranks) {
        delete s;
        return set_error(LBX_EINVAL, "owner entries must lie in [0, %d)", c.n_ranks);
      }
      s->owner[b] = initial_owner[b];
    }
  }
  s->prop.assign(nb, 0);
  s->prev.assign(nb, 0);
  s->work.assign(nb, 0.0);
  s->rank_acc.assign(c.n_ranks, 0.0);
  s->faces_per_rank.assign(c.n_ranks, 0);
  *out = s;
  return LBX_OK;
}

int lbx_lb_destroy(lbx_lb* lb) {
  delete lb;
  return LBX_OK;
}

int lbx_lb_step(lbx_lb* lb, int64_t step, const int64_t* counts, const uint64_t* clk,
                int64_t n_alive, lbx_sim_outputs* out, int32_t* adopted, int32_t* halt) {
  clear_error();
  if (!lb || !counts || !out || !halt) return set_error(LBX_EINVAL, "NULL argument");
  if (step < 0 || step >= lb->cfg.total_steps)
    return set_error(LBX_EINVAL, "step %lld outside [0, %lld)", (long long)step,
                     (long long)lb->cfg.total_steps);
  int a = 0, h = 0;
  int rc = lb_step(lb, step, counts, nullptr, clk, n_alive, out, &a, &h);
  if (adopted) *adopted = a;
  *halt = h;
  return rc;
}

int lbx_lb_set_migration_ratio(lbx_lb* lb, double ratio) {
  clear_error();
  if (!lb) return set_error(LBX_EINVAL, "NULL argument");
  if (!(ratio >= 0.0)) return set_error(LBX_EINVAL, "migration ratio must be >= 0");
  lb->cfg.migration_ratio = ratio;
  return LBX_OK;
}

int lbx_lb_owner(lbx_lb* lb, int64_t* owner) {
  clear_error();
  if (!lb || !owner) return set_error(LBX_EINVAL, "NULL argument");
  std::memcpy(owner, lb->owner.data(), 8 * (size_t)lb->nb);
  return LBX_OK;
}

int lbx_sim_create(lbx_sim** out, lbx_ctx* ctx, const lbx_sim_config* cfg) {
  clear_error();
  if (!out || !ctx || !cfg) return set_error(LBX_EINVAL, "NULL argument");
  if (cfg->extent_y > 0)
    return set_error(LBX_EINVAL, "3D runs use lbx_push_step_3d + lbx_lb (Simulation3D)");
  lbx_lb* lb = nullptr;
  int rc = lbx_lb_create(&lb, cfg, nullptr);
  if (rc) return rc;
  lbx_sim* s = new lbx_sim();
  s->ctx = ctx;
  s->lb = lb;
  const int nb = lb->nb;
  s->ring = (cfg->capacity_particles >= 0 || cfg->cost_kind == LBX_COST_TIMERS ||
             cfg->cost_kind == LBX_COST_CUPTI)
                ? 1
                : 2 * kCycle;
  if (s->ring > 1 && cfg->physics == LBX_PHYSICS_SURROGATE && !std::getenv("LBX_NO_GRAPHS")) {
    s->graphs = cudaStreamCreateWithFlags(&s->gs, cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming) == cudaSuccess;
    if (!s->graphs) cudaGetLastError();
  }
  if (cfg->cost_kind == LBX_COST_CUPTI) {
    rc = cupti_acquire();
    if (rc) {
      lbx_sim_destroy(s);
      return rc;
    }
    s->cupti = true;
    s->spans.assign(nb, 0.0);
  }
  s->rec_bytes = ((size_t)24 * nb + 16 + 255) & ~(size_t)255;
  cudaError_t e = cudaHostAlloc(&s->ring_h, s->rec_bytes * s->ring, cudaHostAllocMapped);
  if (e != cudaSuccess) {
    lbx_sim_destroy(s);
    return cuda_fail(e, "cudaHostAlloc(ring)");
  }
  std::memset(s->ring_h, 0, s->rec_bytes * s->ring);
  e = cudaHostGetDevicePointer((void**)&s->ring_d, s->ring_h, 0);
  if (e != cudaSuccess) {
    lbx_sim_destroy(s);
    return cuda_fail(e, "cudaHostGetDevicePointer");
  }
  s->ev.resize(s->ring);
  s->t0.resize(s->ring);
  s->t1.resize(s->ring);
  for (int i = 0; i < s->ring; ++i) {
    cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming);
    cudaEventCreate(&s->t0[i]);
    cudaEventCreate(&s->t1[i]);
  }
  rc = ensure_accumulators(ctx, nb);
  if (rc) {
    lbx_sim_destroy(s);
    return rc;
  }
  // resident multi-step kernel: the reference's surrogate step with an
  // on-device cost form (no Timers launches), no capacity halting (ring > 1)
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
  if (coop && s->ring > 1 && cfg->physics == LBX_PHYSICS_SURROGATE &&
      cfg->cost_kind != LBX_COST_TIMERS && cfg->cost_kind != LBX_COST_CUPTI && nb <= 8192 &&
      !std::getenv("LBX_NO_RESIDENT")) {
    int grid = 0;
    rc = resident_capacity(ctx, nb, &s->resident_max, &grid);
    const size_t ctl_bytes = sizeof(unsigned long long) * (s->ring + 2);
    bool ok = rc == LBX_OK &&
              cudaMalloc(&s->rctl, sizeof(ResCtl)) == cudaSuccess &&
              cudaMalloc(&s->racc, sizeof(unsigned long long) * 2 * kResSlots * nb) == cudaSuccess &&
              cudaHostAlloc(&s->rctl_h, ctl_bytes, cudaHostAllocMapped) == cudaSuccess &&
              cudaHostGetDevicePointer((void**)&s->rctl_d, s->rctl_h, 0) == cudaSuccess;
    if (ok) {
      cudaMemset(s->rctl, 0, sizeof(ResCtl));
      cudaMemset(s->racc, 0, sizeof(unsigned long long) * 2 * kResSlots * nb);
      std::memset(s->rctl_h, 0, ctl_bytes);
      s->resident = true;
      if (cfg->interval <= cfg->total_steps || cfg->static_step >= 0) {
        const char* e = std::getenv("LBX_LB_WORKERS");
        const int workers = e ? std::atoi(e) : 4;
        if (workers > 0) s->pool = new ProposalPool(lb, s->ring, workers);
      }
    } else {
      cudaGetLastError();
      clear_error();
    }
  }
  *out = s;
  return LBX_OK;
}

int lbx_sim_destroy(lbx_sim* s) {
  clear_error();
  if (!s) return LBX_OK;
  for (auto& ev : s->ev) cudaEventSynchronize(ev), cudaEventDestroy(ev);
  for (auto& ev : s->t0) cudaEventDestroy(ev);
  for (auto& ev : s->t1) cudaEventDestroy(ev);
  if (s->ring_h) cudaFreeHost(s->ring_h);
  for (auto& ev : s->tb0) cudaEventDestroy(ev);
  for (auto& ev : s->tb1) cudaEventDestroy(ev);
  if (s->gs) cudaStreamSynchronize(s->gs);
  drop_graphs(s);
  if (s->gs) cudaStreamDestroy(s->gs);
  if (s->join) cudaEventDestroy(s->join);
  if (s->cupti) cupti_release();
  delete s->pool;
  cudaFree(s->rctl);
  cudaFree(s->racc);
  if (s->rctl_h) cudaFreeHost(s->rctl_h);
  cudaFree(s->box);
  cudaFree(s->perm);
  cudaFree(s->zero_v);
  cudaFree(s->d_counts);
  cudaFree(s->d_cursors);
  cudaFreeHost(s->h_counts);
  cudaFreeHost(s->h_offsets);
  delete s->lb;
  delete s;
  return LBX_OK;
}

int lbx_sim_set_particles(lbx_sim* s, double* z, double* x, double* vz, double* vx,
                          double* kick_vz, double* kick_vx, int64_t n, void* stream) {
  clear_error();
  if (!s) return set_error(LBX_EINVAL, "sim is NULL");
  if (n < 0) return set_error(LBX_EINVAL, "n must be >= 0");
  if ((kick_vz == nullptr) != (kick_vx == nullptr))
    return set_error(LBX_EINVAL, "kick velocity buffers must be given together");
  s->z = z;
  s->x = x;
  s->vz = vz;
  s->vx = vx;
  s->kvz = kick_vz;
  s->kvx = kick_vx;
  s->n_host = n;
  drop_graphs(s);   // captured pointers and launch sizes change
  if (s->lb->cfg.cost_kind == LBX_COST_TIMERS || s->cupti) {
    if (n >= (1ll << 31)) return set_error(LBX_EINVAL, "Timers strategy supports < 2^31 particles");
    const int nb = s->lb->nb;
    cudaFree(s->box);
    cudaFree(s->perm);
    cudaFree(s->zero_v);
    s->box = s->perm = nullptr;
    s->zero_v = nullptr;
    bool ok = cudaMalloc(&s->box, (size_t)(n + 1) * 4) == cudaSuccess &&
              cudaMalloc(&s->perm, (size_t)(n + 1) * 4) == cudaSuccess &&
              cudaMalloc(&s->zero_v, (size_t)(n + 2) * 8) == cudaSuccess;
    if (ok && !s->d_counts) {
      ok = cudaMalloc(&s->d_counts, (size_t)nb * 8) == cudaSuccess &&
           cudaMalloc(&s->d_cursors, (size_t)nb * 8) == cudaSuccess &&
           cudaHostAlloc(&s->h_counts, (size_t)nb * 8, cudaHostAllocDefault) == cudaSuccess &&
           cudaHostAlloc(&s->h_offsets, (size_t)nb * 8, cudaHostAllocDefault) == cudaSuccess;
      s->tb0.resize(nb);
      s->tb1.resize(nb);
      for (int b = 0; b < nb; ++b) {
        cudaEventCreate(&s->tb0[b]);
        cudaEventCreate(&s->tb1[b]);
      }
      s->timers.assign(nb, 0.0);
    }
    if (!ok) return set_error(LBX_EOOM, "Timers buffers");
    cudaMemset(s->zero_v, 0, (size_t)(n + 2) * 8);
  }
  return lbx_ctx_set_count(s->ctx, n, stream);
}

int lbx_sim_set_fields(lbx_sim* s, float* const* fields, float* const* current, double* uy) {
  clear_error();
  if (!s || !fields || !current || !uy) return set_error(LBX_EINVAL, "NULL argument");
  for (int k = 0; k < 6; ++k) s->fields[k] = fields[k];
  for (int k = 0; k < 3; ++k) s->current[k] = current[k];
  s->uy = uy;
  return LBX_OK;
}

int lbx_sim_run(lbx_sim* s, int64_t first, int64_t last, lbx_sim_outputs* o, void* stream) {
  clear_error();
  if (!s || !o) return set_error(LBX_EINVAL, "NULL argument");
  const lbx_sim_config& c = s->lb->cfg;
  if (first < 0 || last > c.total_steps || first > last)
    return set_error(LBX_EINVAL, "step range [%lld, %lld) outside [0, %lld)", (long long)first,
                     (long long)last, (long long)c.total_steps);
  if (!s->z) return set_error(LBX_EINVAL, "particles not set");
  if (c.physics == LBX_PHYSICS_PIC && !s->uy)
    return set_error(LBX_EINVAL, "PIC physics needs lbx_sim_set_fields");
  if (first == 0) {
    std::memcpy(s->lb->owner.data(), o->owner, 8 * (size_t)s->lb->nb);
    s->lb->faces_dirty = true;
  }
  for (int b = 0; b < s->lb->nb; ++b)
    if (s->lb->owner[b] < 0 || s->lb->owner[b] >= c.n_ranks)
      return set_error(LBX_EINVAL, "owner entries must lie in [0, %d)", c.n_ranks);
  cudaStream_t caller = (cudaStream_t)stream;
  cudaStream_t st = caller;
  if (s->gs) {   // run on the loop's own (capturable) stream, ordered after the caller's work
    cudaEventRecord(s->join, caller);
    cudaStreamWaitEvent(s->gs, s->join, 0);
    st = s->gs;
  }
  s->stream = st;
  s->timing = o->kernel_ms != nullptr;
  int64_t launched = first, processed = first;
  int halt = 0;
  if (s->resident && !s->timing && last - first >= 2 && s->n_host > 0 &&
      s->n_host <= s->resident_max) {
    int rc = run_resident(s, first, last, o, st, &halt);
    if (rc) return rc;
    processed = launched = last;
  }
  while (processed < last && !halt) {
    while (launched < last && launched - processed < s->ring) {
      // whole cycle as one graph: aligned, one side of the kick; wait for
      // the ring half it writes to be processed
      if (s->graphs && s->warm && launched % kCycle == 0 && launched + kCycle <= last &&
          kicked_at(s, launched) == kicked_at(s, launched + kCycle - 1)) {
        if (launched - processed + kCycle > s->ring) break;
        if (launch_cycle(s, launched, st)) {
          launched += kCycle;
          continue;
        }
      }
      int rc = launch_step(s, launched, st);
      if (rc) return rc;
      s->warm = true;
      ++launched;
    }
    int rc = process_step(s, processed, o, &halt);
    if (rc) return rc;
    ++processed;
  }
  // Capacity runs use ring=1, so no step past a halting step was launched.
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "stream sync");
  if (s->gs) {
    cudaEventRecord(s->join, s->gs);
    cudaStreamWaitEvent(caller, s->join, 0);
  }
  std::memcpy(o->owner, s->lb->owner.data(), 8 * (size_t)s->lb->nb);
  return LBX_OK;
}

int lbx_sim_graph_cycles(lbx_sim* s, int64_t* cycles) {
  clear_error();
  if (!s || !cycles) return set_error(LBX_EINVAL, "NULL argument");
  *cycles = s->graph_cycles;
  return LBX_OK;
}

int lbx_sim_resident_runs(lbx_sim* s, int64_t* runs) {
  clear_error();
  if (!s || !runs) return set_error(LBX_EINVAL, "NULL argument");
  *runs = s->resident_runs;
  return LBX_OK;
}

int lbx_sim_particles(lbx_sim* s, int64_t* n, void* stream) {
  clear_error();
  if (!s || !n) return set_error(LBX_EINVAL, "NULL argument");
  return lbx_ctx_get_count(s->ctx, n, stream);
}

}  // extern "C"
