// libLBX native stepping runtime: the per-step loop of workload.py:388-470
// (run_simulation) without Python in it.
//
// Per step s:
//   device  fused push/absorb/compact/bin/heuristic/clock kernel (one launch);
//           its last CTA writes the step record (counts, heuristic cost,
//           clock tally, survivor count) straight into a mapped pinned ring
//           slot, so no memcpy is enqueued;
//   host    once slot s is complete: provider cost (workload.py:414), trace,
//           efficiency, should_attempt/attempt_rebalance (balancer.py:258-304),
//           adoption, and the walltime-model columns of step_walltime
//           (workload.py:314-363), all bit-exact with the reference.
// The host runs up to `ring` steps behind the device: on one GPU the mapping
// never feeds back into particle data, so nothing but the ring depth limits
// the overlap.  Runs with a particle capacity (OOM can stop the run) use a
// depth of 1 so the device never advances past the halting step.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "lbx_internal.h"

using namespace lbx;

struct lbx_sim {
  lbx_ctx* ctx = nullptr;
  lbx_sim_config cfg{};
  int32_t nbz = 0, nbx = 0, nb = 0;
  std::vector<int64_t> curve, face_a, face_b;
  double *z = nullptr, *x = nullptr, *vz = nullptr, *vx = nullptr;
  double *kvz = nullptr, *kvx = nullptr;
  // mapped pinned ring of step records
  int ring = 0;
  size_t rec_bytes = 0;
  unsigned char* ring_h = nullptr;
  unsigned char* ring_d = nullptr;
  std::vector<cudaEvent_t> ev, t0, t1;  // completion / kernel timing events
  bool timing = false;
  std::vector<int64_t> owner, prop, prev;
  std::vector<double> work, cost, scratch, rank_acc;
  std::vector<int64_t> faces_per_rank;
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

int launch_step(lbx_sim* s, int64_t step, cudaStream_t st) {
  const int tslot = (int)(step % s->ring);
  if (s->timing) cudaEventRecord(s->t0[tslot], st);
  const int slot = (int)(step % s->ring);
  Rec d = rec_at(s->ring_d, s->rec_bytes, slot, s->nb);
  const bool kicked = step >= s->cfg.kick_step && s->kvz != nullptr;
  StepLaunch a{};
  a.z = s->z;
  a.x = s->x;
  a.vz = kicked ? s->kvz : s->vz;
  a.vx = kicked ? s->kvx : s->vx;
  a.ez = (double)s->cfg.extent_z;
  a.ex = (double)s->cfg.extent_x;
  a.m = (double)s->cfg.box_size;
  a.nbz = s->nbz;
  a.nbx = s->nbx;
  a.wp = s->cfg.w_particle;
  a.wc = s->cfg.w_cell;
  a.cells = (double)s->cfg.box_size * (double)s->cfg.box_size;
  a.clock = s->cfg.cost_kind == LBX_COST_GPUCLOCK;
  a.counts_out = reinterpret_cast<long long*>(d.counts);
  a.cost_out = d.cost;
  a.clk_out = a.clock ? reinterpret_cast<unsigned long long*>(d.clk) : nullptr;
  a.n_out = reinterpret_cast<long long*>(d.n);
  a.err_out = reinterpret_cast<long long*>(d.err);
  int rc = launch_push_step(s->ctx, a, st);
  if (rc) return rc;
  if (s->timing) cudaEventRecord(s->t1[tslot], st);
  cudaError_t e = cudaEventRecord(s->ev[slot], st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  return LBX_OK;
}

// Host half of one step.  Returns 1 if the step hit OOM (run halts).
int process_step(lbx_sim* s, int64_t step, lbx_sim_outputs* o, int* halt) {
  const lbx_sim_config& c = s->cfg;
  const int nb = s->nb;
  const int32_t R = c.n_ranks;
  const int slot = (int)(step % s->ring);
  cudaError_t e = cudaEventSynchronize(s->ev[slot]);
  if (e != cudaSuccess) return cuda_fail(e, "step kernel");
  Rec h = rec_at(s->ring_h, s->rec_bytes, slot, nb);
  if (s->timing && o->kernel_ms) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->t0[slot], s->t1[slot]);
    o->kernel_ms[step] = ms;
  }
  if (*h.err != 0)
    return set_error(LBX_ERANGE, "step %lld: %lld survivors fall outside the box grid",
                     (long long)step, (long long)*h.err);

  // true work (workload.py:303-311) and provider cost (workload.py:414)
  const double cells = (double)((int64_t)c.box_size * c.box_size);
  for (int b = 0; b < nb; ++b) s->work[b] = c.work_wp * (double)h.counts[b] + c.work_wc * cells;
  double* cost = o->cost_trace + (size_t)step * nb;
  switch (c.cost_kind) {
    case LBX_COST_HEURISTIC:
      std::memcpy(cost, h.cost, sizeof(double) * nb);
      break;
    case LBX_COST_MEASURED:
    case LBX_COST_INSTRUMENTED:
      measured_cost(s->work.data(), nb, c.noise_amplitude, c.noise_seed, (uint64_t)step, cost);
      break;
    case LBX_COST_GPUCLOCK:
      for (int b = 0; b < nb; ++b) cost[b] = (double)h.clk[b];
      break;
    default:
      return set_error(LBX_EINVAL, "unknown cost kind %d", c.cost_kind);
  }
  if (o->count_trace) std::memcpy(o->count_trace + (size_t)step * nb, h.counts, 8 * (size_t)nb);
  if (o->clock_trace) std::memcpy(o->clock_trace + (size_t)step * nb, h.clk, 8 * (size_t)nb);
  o->n_alive[step] = *h.n;

  // balance (balancer.py:258-304)
  double e_cur = 1.0, e_after;
  efficiency(cost, s->owner.data(), nb, R, &e_cur, nullptr, s->scratch);
  e_after = e_cur;
  const bool attempted = should_attempt(c, step);
  bool adopted = false;
  s->prev = s->owner;
  if (attempted) {
    o->n_attempts += 1;
    int rc = c.strategy == LBX_STRATEGY_KNAPSACK
                 ? knapsack(cost, nb, R, c.cap_factor, s->prop.data())
                 : sfc(cost, s->curve.data(), nb, R, s->prop.data());
    if (rc) return rc;
    double e_prop = 1.0;
    efficiency(cost, s->prop.data(), nb, R, &e_prop, nullptr, s->scratch);
    const double need = c.threshold_relative ? e_cur * (1.0 + c.improvement_threshold)
                                             : e_cur + c.improvement_threshold;
    adopted = e_prop >= need && e_prop >= e_cur;
    if (adopted) {
      s->owner = s->prop;
      e_after = e_prop;
      o->adopt_steps[o->n_adoptions] = step;
      if (o->adopt_owners)
        std::memcpy(o->adopt_owners + (size_t)o->n_adoptions * nb, s->owner.data(),
                    8 * (size_t)nb);
      o->n_adoptions += 1;
    }
  }

  // walltime model (workload.py:314-363)
  std::fill(s->rank_acc.begin(), s->rank_acc.end(), 0.0);
  for (int b = 0; b < nb; ++b) s->rank_acc[s->owner[b]] += s->work[b];
  double compute_max = s->rank_acc[0];
  for (int r = 1; r < R; ++r) compute_max = std::max(compute_max, s->rank_acc[r]);
  std::fill(s->faces_per_rank.begin(), s->faces_per_rank.end(), 0);
  for (size_t f = 0; f < s->face_a.size(); ++f) {
    const int64_t ra = s->owner[s->face_a[f]], rb = s->owner[s->face_b[f]];
    if (ra != rb) {
      s->faces_per_rank[ra] += 1;
      s->faces_per_rank[rb] += 1;
    }
  }
  int64_t fmax = s->faces_per_rank[0];
  for (int r = 1; r < R; ++r) fmax = std::max(fmax, s->faces_per_rank[r]);
  double comm_max = (double)fmax * c.comm_per_face;
  double gather = attempted ? c.gather : 0.0;
  double redis = 0.0;
  if (adopted) {
    int64_t moved = 0;
    for (int b = 0; b < nb; ++b)
      if (s->owner[b] != s->prev[b]) moved += h.counts[b];
    redis = c.redistribute_latency + c.redistribute_per_particle * (double)moved;
  }
  std::fill(s->rank_acc.begin(), s->rank_acc.end(), 0.0);
  for (int b = 0; b < nb; ++b) s->rank_acc[s->owner[b]] += (double)h.counts[b];
  double occ = s->rank_acc[0];
  for (int r = 1; r < R; ++r) occ = std::max(occ, s->rank_acc[r]);
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
  *halt = oom ? 1 : 0;
  return LBX_OK;
}

}  // namespace

extern "C" {

int lbx_sim_create(lbx_sim** out, lbx_ctx* ctx, const lbx_sim_config* cfg) {
  clear_error();
  if (!out || !ctx || !cfg) return set_error(LBX_EINVAL, "NULL argument");
  const lbx_sim_config& c = *cfg;
  if (c.box_size < 1 || c.extent_z % c.box_size || c.extent_x % c.box_size)
    return set_error(LBX_EINVAL, "box_size %d must divide the extents", c.box_size);
  if (c.n_ranks < 1) return set_error(LBX_EINVAL, "n_ranks must be >= 1");
  if (c.total_steps < 1) return set_error(LBX_EINVAL, "total_steps must be >= 1");
  if (c.interval < 1) return set_error(LBX_EINVAL, "interval must be >= 1");
  if (c.cost_kind < 0 || c.cost_kind > LBX_COST_GPUCLOCK)
    return set_error(LBX_EINVAL, "unknown cost kind %d", c.cost_kind);
  lbx_sim* s = new lbx_sim();
  s->ctx = ctx;
  s->cfg = c;
  s->nbz = c.extent_z / c.box_size;
  s->nbx = c.extent_x / c.box_size;
  s->nb = s->nbz * s->nbx;
  const int nb = s->nb;
  s->curve.resize(nb);
  lbx_morton_order(s->nbz, s->nbx, s->curve.data());
  for (int bz = 0; bz + 1 < s->nbz; ++bz)
    for (int bx = 0; bx < s->nbx; ++bx) {
      s->face_a.push_back(bz * s->nbx + bx);
      s->face_b.push_back((bz + 1) * s->nbx + bx);
    }
  for (int bz = 0; bz < s->nbz; ++bz)
    for (int bx = 0; bx + 1 < s->nbx; ++bx) {
      s->face_a.push_back(bz * s->nbx + bx);
      s->face_b.push_back(bz * s->nbx + bx + 1);
    }
  s->owner.assign(nb, 0);
  s->prop.assign(nb, 0);
  s->prev.assign(nb, 0);
  s->work.assign(nb, 0.0);
  s->rank_acc.assign(c.n_ranks, 0.0);
  s->faces_per_rank.assign(c.n_ranks, 0);
  s->ring = c.capacity_particles >= 0 ? 1 : 16;
  s->rec_bytes = ((size_t)24 * nb + 16 + 255) & ~(size_t)255;
  cudaError_t e = cudaHostAlloc(&s->ring_h, s->rec_bytes * s->ring, cudaHostAllocMapped);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaHostAlloc(ring)");
  }
  std::memset(s->ring_h, 0, s->rec_bytes * s->ring);
  e = cudaHostGetDevicePointer((void**)&s->ring_d, s->ring_h, 0);
  if (e != cudaSuccess) {
    lbx_sim_destroy(s);
    return cuda_fail(e, "cudaHostGetDevicePointer");
  }
  s->ev.resize(s->ring);
  for (auto& ev : s->ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  s->t0.resize(s->ring);
  s->t1.resize(s->ring);
  for (int i = 0; i < s->ring; ++i) {
    cudaEventCreate(&s->t0[i]);
    cudaEventCreate(&s->t1[i]);
  }
  int rc = ensure_accumulators(ctx, nb);
  if (rc) {
    lbx_sim_destroy(s);
    return rc;
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
  return lbx_ctx_set_count(s->ctx, n, stream);
}

int lbx_sim_run(lbx_sim* s, int64_t first, int64_t last, lbx_sim_outputs* o, void* stream) {
  clear_error();
  if (!s || !o) return set_error(LBX_EINVAL, "NULL argument");
  if (first < 0 || last > s->cfg.total_steps || first > last)
    return set_error(LBX_EINVAL, "step range [%lld, %lld) outside [0, %lld)", (long long)first,
                     (long long)last, (long long)s->cfg.total_steps);
  if (!s->z) return set_error(LBX_EINVAL, "particles not set");
  if (first == 0) std::memcpy(s->owner.data(), o->owner, 8 * (size_t)s->nb);
  for (int b = 0; b < s->nb; ++b)
    if (s->owner[b] < 0 || s->owner[b] >= s->cfg.n_ranks)
      return set_error(LBX_EINVAL, "owner entries must lie in [0, %d)", s->cfg.n_ranks);
  cudaStream_t st = (cudaStream_t)stream;
  s->timing = o->kernel_ms != nullptr;
  int64_t launched = first, processed = first;
  int halt = 0;
  while (processed < last && !halt) {
    while (launched < last && launched - processed < s->ring) {
      int rc = launch_step(s, launched, st);
      if (rc) return rc;
      ++launched;
    }
    int rc = process_step(s, processed, o, &halt);
    if (rc) return rc;
    ++processed;
  }
  // Capacity runs use ring=1, so no step past a halting step was launched.
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "stream sync");
  std::memcpy(o->owner, s->owner.data(), 8 * (size_t)s->nb);
  return LBX_OK;
}

int lbx_sim_particles(lbx_sim* s, int64_t* n, void* stream) {
  clear_error();
  if (!s || !n) return set_error(LBX_EINVAL, "NULL argument");
  return lbx_ctx_get_count(s->ctx, n, stream);
}

}  // extern "C"
