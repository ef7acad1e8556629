/*
 * lbx.h -- C ABI of the B200-native in-situ cost assessment + load-balancing
 * path (libLBX, built from paper_2104_11385_b200/csrc/).
 *
 * Every entry point returns 0 on success or a nonzero LBX_E* code; the
 * message of the most recent failure on the calling thread is available from
 * lbx_last_error().  The Python host layer maps LBX_EINVAL to ValueError
 * (same message substrings the reference raises: "cap", "permutation",
 * "curve", "length", ...), LBX_ECUDA to RuntimeError and LBX_EOOM to
 * MemoryError.
 *
 * Ownership: the caller allocates every buffer (host or device) and keeps it
 * alive for the duration of the call (for stream-ordered device calls: until
 * the stream has drained).  The library never frees caller memory.  Opaque
 * contexts are created and destroyed by explicit calls.  Host functions are
 * reentrant; device functions are asynchronous on the caller's stream
 * (`stream` is a cudaStream_t passed as void*; NULL = legacy default stream).
 *
 * Reference interface each entry replaces is cited as file:line under
 * /root/reference/pkg/src/lbsim/.
 */
#ifndef LBX_H_
#define LBX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBX_OK 0
#define LBX_EINVAL 1   /* contract violation -> ValueError              */
#define LBX_ECUDA 2    /* CUDA runtime failure -> RuntimeError          */
#define LBX_EOOM 3     /* device allocation failure -> MemoryError      */
#define LBX_ERANGE 4   /* particle outside the box grid -> ValueError   */

/* Last error message of the calling thread ("" if none). */
const char* lbx_last_error(void);
/* Library version string and the compute capability it was built for. */
const char* lbx_version(void);

/* ------------------------------------------------------------------------
 * Device context: the look-back workspace and the device-resident step
 * state (tile ticket, finished-CTA counter, look-back epoch, live particle
 * count).  One context per device and stream of work.
 * ---------------------------------------------------------------------- */
typedef struct lbx_ctx lbx_ctx;

/* capacity = max particles any call on this context will process. */
int lbx_ctx_create(lbx_ctx** out, int device, int64_t capacity);
int lbx_ctx_destroy(lbx_ctx* ctx);
/* Grow the look-back workspace to at least `capacity` particles. */
int lbx_ctx_reserve(lbx_ctx* ctx, int64_t capacity);
/* Stream-ordered: set / read the device-resident live particle count. */
int lbx_ctx_set_count(lbx_ctx* ctx, int64_t n, void* stream);
/* Host-side upper bound on the live count (launch sizing) without touching
 * the device count -- for loops whose count changes on the device only. */
int lbx_ctx_set_upper(lbx_ctx* ctx, int64_t n_upper);
int lbx_ctx_get_count(lbx_ctx* ctx, int64_t* n_host, void* stream); /* syncs */
/* Persistent-grid size the step kernels launch with (0 = auto: resident
 * CTAs per SM x SMs). */
int lbx_ctx_set_grid(lbx_ctx* ctx, int ctas);
/* Kernel timing: when on, the main streaming kernel of each step call is
 * bracketed by CUDA events recorded immediately around its launch;
 * lbx_ctx_last_kernel_ms waits for the end event and returns milliseconds. */
int lbx_ctx_enable_timing(lbx_ctx* ctx, int on);
int lbx_ctx_last_kernel_ms(lbx_ctx* ctx, float* ms);

/* ------------------------------------------------------------------------
 * Drop-in kernels (reference plugin point 1, kernels.py:10-25).
 * Array-of-structs [n][2] float64 device buffers, exactly the reference's
 * argument layout.
 * ---------------------------------------------------------------------- */

/* Replaces _kernels.pyx:12-35 advance_particles (fallback
 * _kernels_py.py:13-22): out_pos[m] = pos+vel of survivors (0 <= p < extent
 * on both axes), out_vel[m] = their velocities, order preserved.  Single
 * pass (decoupled look-back stable compaction).  *m_dev (device int64)
 * receives m.  Buffers must not overlap. */
int lbx_advance_particles(lbx_ctx* ctx, const double* pos, const double* vel,
                          int64_t n, double extent_z, double extent_x,
                          double* out_pos, double* out_vel, int64_t* m_dev,
                          void* stream);

/* Replaces _kernels.pyx:38-47 bin_particles: counts[nbz*nbx] (device int64,
 * overwritten) of (int)(z/M)*nbx + (int)(x/M).  A position outside the grid
 * (UB in the reference) sets *err_dev (device int64, may be NULL) nonzero. */
int lbx_bin_particles(const double* pos, int64_t n, double box_size,
                      int32_t nbz, int32_t nbx, int64_t* counts,
                      int64_t* err_dev, void* stream);

/* The plugin path for HOST arrays (the reference calls advance_particles and
 * bin_particles on numpy arrays every step, workload.py:293-298): advance
 * [n][2] host pos/vel (pinned for full PCIe speed) into host out_pos/out_vel
 * (capacity n; survivors, order kept, *m_out of them) and, when counts !=
 * NULL, the per-box counts of the survivors and their heuristic cost (cost
 * may be NULL).  4 Mi-particle chunks rotate over three streams, each chunk
 * stream-ordered end to end (copy in, advance, bin, copy out) with no host
 * round trip, so both PCIe directions and the kernels overlap; a chunk's
 * survivors land at its own offset and gaps left by absorbed particles are
 * closed on the host afterwards.  Synchronous. */
int lbx_advance_bin_host(lbx_ctx* ctx, const double* pos, const double* vel, int64_t n,
                         double extent_z, double extent_x, double box_size,
                         int32_t nbz, int32_t nbx, double w_particle, double w_cell,
                         double* out_pos, double* out_vel, int64_t* counts,
                         double* cost, int64_t* m_out);

/* ------------------------------------------------------------------------
 * Fused device step (the hot path; replaces workload.py:286-300 advance +
 * workload.py:303-311 true_work counts + cost.py:83-95 heuristic_cost, and
 * adds the GpuClock tally of PAPER.md:170-173).
 *
 * Structure-of-arrays particle state z,x,vz,vx (float64, 16-byte aligned,
 * capacity >= n + 2), updated IN PLACE: push, absorb, stable compaction,
 * per-box counts of the survivors, heuristic cost, optional per-box clock64
 * tally -- one kernel launch.  n is the context's device-resident count and
 * is replaced by the survivor count.
 *
 * Outputs (device or mapped-pinned host pointers, any may be NULL):
 *   counts_out[nb] int64   survivors per box (== bin_particles of result)
 *   cost_out[nb]   double  wp*count + wc*cells, no FMA (cost.py:94)
 *   clk_out[nb]    uint64  GpuClock tally (SM cycles attributed per box);
 *                          requires flags & LBX_STEP_CLOCK
 *   n_out          int64   survivor count
 * ---------------------------------------------------------------------- */
#define LBX_STEP_CLOCK 1u   /* fused GpuClock instrumentation             */

typedef struct lbx_step_args {
  double* z;
  double* x;
  double* vz;
  double* vx;
  double extent_z, extent_x;
  double box_size;
  int32_t nbz, nbx;
  double w_particle, w_cell;   /* heuristic weights (cost.py:52-63)     */
  double cells_per_box;        /* BoxArray.cells_per_box (M*M)          */
  uint32_t flags;
  int64_t* counts_out;
  double* cost_out;
  uint64_t* clk_out;
  int64_t* n_out;
  int64_t* err_out;            /* out-of-grid survivors (should be 0)   */
} lbx_step_args;

int lbx_push_step(lbx_ctx* ctx, const lbx_step_args* args, void* stream);

/* 3D fused step (config C4, parity unpinned): SoA float64 z, y, x, vz, vy, vx
 * in place (72 B/particle), absorbing box [0,Ez)x[0,Ey)x[0,Ex), per-box
 * counts / heuristic cost / GpuClock into (nbz*nby*nbx) box vectors, stable
 * compaction.  box_size must be a power of two dividing the extents. */
typedef struct lbx_step3d_args {
  double *z, *y, *x, *vz, *vy, *vx;
  int32_t extent_z, extent_y, extent_x, box_size;
  double w_particle, w_cell;
  uint32_t flags;               /* LBX_STEP_CLOCK */
  int64_t* counts_out;
  double* cost_out;
  uint64_t* clk_out;
  int64_t* n_out;
  int64_t* err_out;
  int64_t* removed_list;        /* optional: list removed indices and skip the
                                   stable compaction (then lbx_fill_holes with
                                   z, x, y, vz, vy, vx in the six slots) */
  int64_t removed_cap;
} lbx_step3d_args;

int lbx_push_step_3d(lbx_ctx* ctx, const lbx_step3d_args* args, void* stream);


/* Replaces cost.py:83-95 heuristic_cost on device vectors:
 * cost[i] = w_particle*particles[i] + w_cell*cells[i], two separately
 * rounded products then one add (no FMA). */
int lbx_heuristic_cost(const double* particles, const double* cells, int64_t n,
                       double w_particle, double w_cell, double* cost,
                       void* stream);

/* ------------------------------------------------------------------------
 * Host balancer (pure, reentrant, bit-exact with the reference's numpy
 * arithmetic: sequential bincount sums, numpy pairwise sum for means and
 * the SFC target, lexsort/argmin tie rules, exact swap expressions).
 * owner/curve arrays are int64 box-indexed.
 * ---------------------------------------------------------------------- */

/* balancer.py:73-79 rank_loads: loads[R] = bincount(owner, weights=cost). */
int lbx_rank_loads(const double* cost, const int64_t* owner, int64_t n,
                   int32_t n_ranks, double* loads);
/* balancer.py:82-99 efficiency_flagged: mean/max; all-zero -> 1.0 + flag. */
int lbx_efficiency(const double* cost, const int64_t* owner, int64_t n,
                   int32_t n_ranks, double* eff, int32_t* degenerate);
/* balancer.py:102-179 knapsack_assign (LPT + cap + swap refinement). */
int lbx_knapsack(const double* cost, int64_t n, int32_t n_ranks,
                 double cap_factor, int64_t* owner);
/* balancer.py:182-219 sfc_assign (greedy split of the curve). */
int lbx_sfc(const double* cost, const int64_t* curve, int64_t n,
            int32_t n_ranks, int64_t* owner);
/* decomposition.py:137-168 morton_order (2D: axis 0 on even bits). */
int lbx_morton_order(int32_t nbz, int32_t nbx, int64_t* curve);
/* 3D extension (config C4; parity unpinned): axis 0 on bits 0,3,6,... */
int lbx_morton_order_3d(int32_t nb0, int32_t nb1, int32_t nb2, int64_t* curve);
/* decomposition.py:176-181 slab_mapping. */
int lbx_slab_mapping(int64_t n_boxes, int32_t n_ranks, int64_t* owner);
/* numpy pairwise float64 sum (used by .sum()/.mean(), balancer.py:93,199). */
double lbx_pairwise_sum(const double* a, int64_t n);
/* cost.py:98-113 measured_cost noise stream: out[i] = work[i]*(1+eps_i),
 * eps from numpy PCG64(SeedSequence((seed, 0x6D656173, step))).uniform. */
int lbx_measured_cost(const double* work, int64_t n, double amplitude,
                      uint64_t seed, uint64_t step, double* out);

/* ------------------------------------------------------------------------
 * Native stepping runtime (replaces workload.py:388-470 run_simulation's
 * per-step loop: advance -> assess -> should_attempt/attempt_rebalance ->
 * step_walltime).  The Python layer builds the scenario (numpy init,
 * kick velocities) and hands device buffers in; the loop then runs without
 * Python in it.  Results are left in caller-provided host arrays.
 * ---------------------------------------------------------------------- */
typedef struct lbx_sim lbx_sim;

#define LBX_COST_HEURISTIC 0     /* device counts -> heuristic cost          */
#define LBX_COST_MEASURED 1      /* modeled timer: true work x PCG64 noise   */
#define LBX_COST_INSTRUMENTED 2  /* same stream, overhead factor applied    */
#define LBX_COST_GPUCLOCK 3      /* fused clock64 tally (real device cost)   */
#define LBX_COST_TIMERS 4        /* per-box launches timed with CUDA events
                                    (the paper's CUPTI-style Timers); cost =
                                    microseconds per box                      */
#define LBX_COST_CUPTI 5         /* the same per-box launches timed by CUPTI
                                    kernel activity records (the paper's
                                    actual Timers mechanism, PAPER.md:174-178;
                                    libcupti is dlopen'ed on first use); cost
                                    = microseconds per box                   */

#define LBX_STRATEGY_KNAPSACK 0
#define LBX_STRATEGY_SFC 1

typedef struct lbx_sim_config {
  /* geometry */
  int32_t extent_z, extent_x, box_size, n_ranks;
  /* per-step scheduling */
  int64_t total_steps;
  int64_t kick_step;           /* step whose advance uses the kick velocity */
  /* balance policy (balancer.py:31-59) */
  int32_t strategy;            /* LBX_STRATEGY_*                              */
  int64_t interval;
  double improvement_threshold;
  int32_t threshold_relative;  /* 1 relative, 0 absolute                      */
  double cap_factor;
  int64_t static_step;         /* -1 = none                                   */
  /* cost provider (cost.py:153-215) */
  int32_t cost_kind;           /* LBX_COST_*                                  */
  double w_particle, w_cell;   /* provider heuristic weights                  */
  double noise_amplitude;
  uint64_t noise_seed;
  double overhead_factor;
  /* ground-truth work weights (workload.py:100) */
  double work_wp, work_wc;
  /* walltime model (workload.py:72-86, resolved) */
  double comm_per_face, gather, redistribute_per_particle, redistribute_latency;
  int64_t capacity_particles;  /* -1 = unlimited                              */
  /* per-step physics: LBX_PHYSICS_SURROGATE (the reference's ballistic
   * advance) or LBX_PHYSICS_PIC (lbx_pic_step; needs lbx_sim_set_fields) */
  int32_t physics;
  double pic_dt, pic_q_over_m, pic_q_times_w;
  /* 3D box decomposition (config C4; the reference is 2D only): extent_y > 0
   * makes the LB object 3D -- boxes (bz*nby + by)*nbx + bx, 3D Morton curve,
   * interior faces along z, y, x, M^3 cells per box. */
  int32_t extent_y;
  /* Migration-aware adoption (the paper's future work;
   * 0 = the reference's gate only).  When > 0 a proposal that passes the
   * efficiency gate is adopted only if the load it saves over one interval,
   * interval * (max rank load now - max rank load proposed), exceeds the
   * cost of moving the particles of every re-owned box, priced at
   * migration_ratio particle-pushes each (cost per push = total cost /
   * total particles of the step). */
  double migration_ratio;
  /* GpuClock cost form (cost_kind == LBX_COST_GPUCLOCK):
   *   LBX_CLOCK_RAW        cost_b = clock tally_b (the paper's thread-summed
   *                        cycles of the particle kernel);
   *   LBX_CLOCK_CALIBRATED cost_b = K_b * (w_particle * Nbar / sum K)
   *                        + w_cell * cells_b, K = the tallies summed over
   *                        the LB window (the steps since the previous
   *                        attempt, reset after each attempt), Nbar = mean
   *                        particles per step over the window: the measured
   *                        tally carries the particle work's distribution
   *                        over boxes, scaled to the heuristic's particle
   *                        units, plus the per-box field work, which no
   *                        particle kernel measures and which is identical
   *                        for equal-size boxes. */
  int32_t clock_mode;
} lbx_sim_config;

#define LBX_CLOCK_RAW 0
#define LBX_CLOCK_CALIBRATED 1

#define LBX_PHYSICS_SURROGATE 0
#define LBX_PHYSICS_PIC 1

/* Per-step outputs, host arrays of length total_steps (caller-owned). */
typedef struct lbx_sim_outputs {
  double* eff_before;
  double* eff_after;
  uint8_t* adopted;
  uint8_t* attempted;
  double* compute_max;
  double* comm_max;
  double* gather;
  double* redistribute;
  double* walltime;
  int64_t* max_rank_particles;
  uint8_t* oom;
  int64_t* n_alive;            /* survivors after the step                  */
  double* cost_trace;          /* [total_steps][n_boxes]                    */
  int64_t* count_trace;        /* [total_steps][n_boxes] or NULL            */
  uint64_t* clock_trace;       /* [total_steps][n_boxes] or NULL            */
  int64_t* owner;              /* [n_boxes] in: initial mapping; out: final */
  /* adoption snapshots: step index per adoption and owner rows */
  int64_t* adopt_steps;        /* [total_steps]                              */
  int64_t* adopt_owners;       /* [total_steps][n_boxes] or NULL            */
  double* kernel_ms;           /* [total_steps] fused-kernel time (CUDA events
                                  on the launch stream) or NULL             */
  int64_t n_adoptions;         /* out                                        */
  int64_t n_attempts;          /* out                                        */
  int64_t completed_steps;     /* out                                        */
} lbx_sim_outputs;

/* Host half of the loop alone (no device needed): provider cost, efficiency,
 * attempt/adopt, walltime-model columns for one step, given the step's GLOBAL
 * per-box survivor counts (and GpuClock tally).  The multi-GPU driver calls
 * it on every rank after all-reducing the tallies, so every rank takes the
 * same decision with no broadcast.  `out` arrays as for lbx_sim_run. */
typedef struct lbx_lb lbx_lb;
int lbx_lb_create(lbx_lb** out, const lbx_sim_config* cfg, const int64_t* initial_owner);
int lbx_lb_destroy(lbx_lb* lb);
int lbx_lb_step(lbx_lb* lb, int64_t step, const int64_t* counts, const uint64_t* clk,
                int64_t n_alive, lbx_sim_outputs* out, int32_t* adopted, int32_t* halt);
int lbx_lb_owner(lbx_lb* lb, int64_t* owner);
/* Replace the migration-aware gate's price (lbx_sim_config::migration_ratio,
 * particle-pushes per moved particle) -- the distributed loop feeds it the
 * MEASURED redistribution cost after every adoption. */
int lbx_lb_set_migration_ratio(lbx_lb* lb, double ratio);

int lbx_sim_create(lbx_sim** out, lbx_ctx* ctx, const lbx_sim_config* cfg);
int lbx_sim_destroy(lbx_sim* sim);
/* Particle buffers (device SoA, capacity >= n + 2); kick_vz/kick_vx replace
 * the velocity buffers at kick_step (pointer swap, no copy). */
int lbx_sim_set_particles(lbx_sim* sim, double* z, double* x, double* vz,
                          double* vx, double* kick_vz, double* kick_vx,
                          int64_t n, void* stream);
/* PIC physics: Yee field arrays (as lbx_pic_args) and the uy momentum array;
 * the velocity / kick buffers of lbx_sim_set_particles hold uz, ux. */
int lbx_sim_set_fields(lbx_sim* sim, float* const* fields, float* const* current, double* uy);
/* Run steps [first, last) of the loop; outputs indexed by absolute step.
 * The loop runs on its own stream, ordered after `stream`'s prior work and
 * before its later work.  Surrogate-physics runs whose particle set fits the
 * GPU's shared memory (~1 M particles on a B200; no capacity model, no
 * per-step kernel timing, no Timers strategy) run as ONE resident
 * cooperative kernel per call, the host following its per-step records
 * (env LBX_NO_RESIDENT disables); others replay each aligned 16-step cycle
 * as one CUDA graph (captured on first use; env LBX_NO_GRAPHS disables),
 * with per-step launches elsewhere -- identical results. */
int lbx_sim_run(lbx_sim* sim, int64_t first, int64_t last,
                lbx_sim_outputs* out, void* stream);
/* Number of 16-step cycles this sim has launched as CUDA graphs. */
int lbx_sim_graph_cycles(lbx_sim* sim, int64_t* cycles);
/* Number of lbx_sim_run calls this sim has run on the resident kernel. */
int lbx_sim_resident_runs(lbx_sim* sim, int64_t* runs);
/* Current device live count (syncs the stream). */
int lbx_sim_particles(lbx_sim* sim, int64_t* n, void* stream);

/* ------------------------------------------------------------------------
 * 2D3V electromagnetic PIC step (SURVEY 8a row a15 / north-star item 1; not
 * in the reference, parity unpinned -- checked bit-exactly against
 * oracle/pic_oracle.py).  Particles SoA float64 z, x, uz, ux, uy (u = gamma
 * v, c = 1, unit cells), 32-byte aligned, capacity >= n + 2, count in the
 * context as for lbx_push_step.  Fields float32 on a Yee grid with one zero
 * guard layer: arrays of (nz+2) x (nx+2), cell (i, j) at [(i+1)*(nx+2) + j+1];
 * fields[] = {Ex, Ey, Ez, Bx, By, Bz}, current[] = {Jx, Jy, Jz} (zero on
 * entry, consumed).  One call: field gather (quad-expanded copy of the
 * fields) + Boris push + absorb + current deposition (cell-relative
 * fixed-point nodes accumulated per lane over cell runs, integer atomics:
 * deterministic) + per-box counts / heuristic cost / GpuClock tally + stable
 * compaction + Yee field update.
 * ---------------------------------------------------------------------- */
#define LBX_PIC_NO_FIELD_SOLVE 2u  /* skip the Yee update (tests)         */
#define LBX_PIC_RESYNC 4u          /* sorted mode: recount the input cells   */
#define LBX_PIC_STABLE_ORDER 64u   /* in place: keep particle order (stable  */
                                   /* compaction of absorbed particles);     */
                                   /* default fills their slots from the     */
                                   /* tail, O(absorbed)                      */
#define LBX_PIC_QUAD 16u           /* gather from the quad-expanded copy     */
#define LBX_PIC_DIRECT 32u         /* gather from the fields (default: quad  */
                                   /* when >= 16 particles per cell)         */
#define LBX_PIC_DEFER_CURRENT 8u   /* stop after push + compaction: the      */
                                   /* cell accumulator stays for a cross-GPU */
                                   /* reduction, then lbx_pic_finish         */
#define LBX_PIC_TILED 128u         /* in place, one CTA per 16x16-cell tile: */
                                   /* field patch and current in shared      */
                                   /* memory, node-centric int64 current.    */
                                   /* Tile slot ranges come from the last    */
                                   /* lbx_pic_sort with this flag (stale     */
                                   /* ranges cost speed, never correctness). */
                                   /* Sparse plasmas; not with sorted mode   */
                                   /* or LBX_PIC_DEFER_CURRENT               */

#define LBX_PIC_FAST 256u          /* tolerance mode (in place, untiled):   */
                                   /* float32 Boris increment with FMA and  */
                                   /* MUFU rsqrt/rcp, FMA gathers; checked  */
                                   /* against the fp64 oracle at a stated   */
                                   /* tolerance, not bit-exact              */
typedef struct lbx_pic_args {
  double* z;
  double* x;
  double* uz;
  double* ux;
  double* uy;
  float* fields[6];
  float* current[3];
  int32_t nz, nx;             /* grid (cells) == particle domain            */
  int32_t box_size;           /* power of two dividing nz and nx            */
  double q_over_m, q_times_w; /* species charge/mass, charge x macro weight */
  double dt;                  /* < 1/sqrt(2)                                */
  double w_particle, w_cell;  /* heuristic weights for cost_out             */
  uint32_t flags;             /* LBX_STEP_CLOCK | LBX_PIC_NO_FIELD_SOLVE    */
  int64_t* counts_out;
  double* cost_out;
  uint64_t* clk_out;
  int64_t* n_out;
  int64_t* err_out;
  /* Sorted mode (all five non-NULL): results are written to out[] = {z, x,
   * uz, ux, uy} grouped by each particle's cell at the START of the step
   * (sort-on-write, no extra pass), so the next step's particles of a cell
   * are contiguous and their current is accumulated in registers.  The
   * caller swaps in/out after the call.  The library keeps the next step's
   * cell slots; passing any other input than the last call's out[] (or
   * LBX_PIC_RESYNC) recounts them.  The last output is recognised by its
   * address: a host that frees a state and may reuse its memory, or that
   * edits the particles between calls, must pass LBX_PIC_RESYNC (the
   * Python wrapper does, keyed on the state object and its version).  Absorbed particles' slots are filled
   * from the tail (O(absorbed)).  Order within a cell is not deterministic;
   * every computed value is.  NULL: in place (order kept with
   * LBX_PIC_STABLE_ORDER, else absorbed slots filled from the tail). */
  double* out[5];
  /* 0: the CIC step above (direct deposit at the new position).  1, 2, 3:
   * charge-conserving Esirkepov deposition with B-spline particle shapes of
   * that order (CIC / TSC / PQS; the paper runs order 3) and
   * the same-order gather at each component's stagger: in place, float32
   * weights (tolerance mode, oracle/pic_oracle.py esirkepov_current), node
   * current accumulated as int64 fixed point; not combinable with sorted /
   * tiled / deferred-current modes. */
  int32_t shape_order;
} lbx_pic_args;

int lbx_pic_step(lbx_ctx* ctx, const lbx_pic_args* args, void* stream);

/* Counting sort of the particles (z, x, uz, ux, uy; the context's device
 * count) by cell into out[] (order within a cell not kept; the caller swaps
 * in/out).  Run every few steps it keeps an in-place run at the speed of a
 * freshly cell-ordered input (the deposit's register runs follow cell
 * order) without sort-on-write's per-step cost.  With LBX_PIC_TILED in
 * flags the key is tile-major (16x16-cell tiles) and the tiles' slot ranges
 * are kept for LBX_PIC_TILED steps.  Fields and physics args are ignored. */
int lbx_pic_sort(lbx_ctx* ctx, const lbx_pic_args* args, void* stream);

/* Multi-GPU PIC (guard-cell current exchange): after a LBX_PIC_DEFER_CURRENT
 * step the context holds the step's current as exact integers, cell-centric
 * jc[cells][16] (16 cell-relative nodes, int64 two's complement) over the
 * deposit box box[4] = {row_min, row_max, col_min, col_max} (device).  Ranks
 * sum the rows of the cells along their shared faces into each other's rows
 * (integer sums: bit-identical to one GPU in any order), set box to their
 * region and call lbx_pic_finish (node gather into current[], clear, Yee
 * update with the same args). */
int lbx_pic_current_view(lbx_ctx* ctx, uint64_t** jc, int64_t* cells, int32_t** box);
/* The same for a deferred Esirkepov step (shape_order > 0): node-centric
 * fixed-point sums j[3][stride], stride = (nz + 2 guard) (nx + 2 guard),
 * node (i, j) of component c at j[c * stride + (i + guard) (nx + 2 guard)
 * + (j + guard)]; lbx_pic_finish with shape_order set converts them (all
 * nodes, cleared) and runs the Yee update.  Replaces the reference's
 * modelled guard-cell communication (workload.py:324-327) for the paper's
 * order-3 deposition. */
int lbx_pic_esk_current_view(lbx_ctx* ctx, uint64_t** j, int64_t* stride, int32_t* guard);
int lbx_pic_finish(lbx_ctx* ctx, const lbx_pic_args* args, void* stream);

/* ------------------------------------------------------------------------
 * Multi-GPU: box ownership -> GPU.  Each rank holds the particles
 * of the boxes it owns.  A particle whose new box belongs to another rank is
 * copied into the staging buffer as a 6-double record (z, x, vz, vx, kick_vz,
 * kick_vx) tagged with its destination and removed locally (in-place
 * compaction).  Every rank still bins ALL particles it pushed into the full
 * per-box vector, so an all-reduce(sum) of counts / clock tallies is exact.
 * Replaces the analytic comm/redistribution model of workload.py:324-337
 * with real traffic.
 * ---------------------------------------------------------------------- */
#define LBX_RECORD_DOUBLES 6

typedef struct lbx_exchange_args {
  const int32_t* owner;     /* device [nbz*nbx]: owning rank of each box       */
  int32_t rank, world;      /* this rank, number of ranks (<= 64)              */
  double* stage;            /* device [stage_cap][6] emigrant records          */
  int32_t* stage_dest;      /* device [stage_cap] destination rank             */
  int64_t stage_cap;
  int64_t* send_counts;     /* device [world] emigrants per destination; the
                               caller zeroes it before the call              */
  double* kick_vz;          /* pending kick velocities travelling with the
                               particles (NULL once the kick has happened)   */
  double* kick_vx;
  /* Optional O(removed) compaction: when removed_list != NULL, the indices of
   * every particle removed locally (absorbed or emigrated) are listed there
   * (removed_cap entries) and NO stable compaction runs; the caller then
   * calls lbx_fill_holes once it knows the count.  Local particle order is
   * not preserved (the multi-GPU path does not need it). */
  int64_t* removed_list;
  int64_t removed_cap;
  /* Peer-memory exchange (fused push + exchange over NVLink / NVSwitch):
   * when peer_recv != NULL the kernel writes each emigrant record straight
   * into its destination's receive buffer, peer_recv[dest] (device array of
   * `world` pointers to peer memory, lbx_peer_alloc / lbx_peer_open), at a
   * slot reserved with one remote atomic per (warp, destination) on
   * peer_cursor[dest] (u64 in the destination's memory); stage / stage_dest
   * are not used.  The destination learns its count from its own cursor
   * after any collective that orders it after the senders' kernels. */
  double* const* peer_recv;
  unsigned long long* const* peer_cursor;
  int64_t peer_recv_cap;
} lbx_exchange_args;

/* lbx_push_step + emigrant staging (per-step box-crossing exchange). */
int lbx_push_step_exchange(lbx_ctx* ctx, const lbx_step_args* args,
                           const lbx_exchange_args* ex, void* stream);
/* Adoption-time migration: stage every local particle whose box is owned
 * elsewhere under ex->owner (no push), compact the rest; *n_out (device) gets
 * the local count left. */
int lbx_partition(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx,
                  double extent_z, double extent_x, double box_size, int32_t nbz,
                  int32_t nbx, const lbx_exchange_args* ex, int64_t* n_out,
                  void* stream);
/* Multi-GPU 3D (Distributed3D; the 3D analogue of lbx_push_step_exchange,
 * not fused over peer memory): the same fused 3D step, and survivors in
 * boxes another rank owns (ex->owner, int32 [nbz*nby*nbx]) are staged as
 * 6-double (z, y, x, vz, vy, vx) records with their destination (still
 * counted in their box: per-rank counts sum to the global bin counts) and
 * removed locally.  ex->removed_list is required (lbx_fill_holes with z, y,
 * x, vz, vy, vx in the six slots compacts); no pending kick arrays, no peer
 * buffers.  lbx_group_by_dest / lbx_unpack (same six slots) move the records. */
int lbx_push_step_3d_exchange(lbx_ctx* ctx, const lbx_step3d_args* args,
                              const lbx_exchange_args* ex, void* stream);
/* Adoption-time 3D migration: stage and list every particle whose box
 * ex->owner gives to another rank (no push).  n_out (device int64[2]) =
 * {particles kept, error code}. */
int lbx_partition_3d(lbx_ctx* ctx, double* z, double* y, double* x, double* vz,
                     double* vy, double* vx, int32_t extent_z, int32_t extent_y,
                     int32_t extent_x, int32_t box_size, const lbx_exchange_args* ex,
                     int64_t* n_out, void* stream);
/* Unstable O(removed) compaction: the n_removed listed indices (any order)
 * are removed from [0, n_new + n_removed) by moving survivors from the tail
 * [n_new, n_new + n_removed) into the holes below n_new.  kick_vz/kick_vx may
 * be NULL.  Sets the context's live count to n_new. */
int lbx_fill_holes(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx,
                   double* kick_vz, double* kick_vx, const int64_t* removed,
                   int64_t n_removed, int64_t n_new, void* stream);
/* Device-count variants for a pipelined loop (no host round trip per step):
 * lbx_fill_holes_dev takes L = removals listed by the preceding exchange
 * push (<= removed_cap) and n_new from the device state, and recognises
 * removed tail slots by their position (outside the domain, or the emigrant
 * sentinel z = -1); lbx_unpack_peer_dev appends the records peers wrote
 * into `recv` (count = the rank's own cursor, then reset to 0) at the
 * device live count, bounded by `capacity` (overflow sets the error word). */
int lbx_fill_holes_dev(lbx_ctx* ctx, double* z, double* x, double* vz, double* vx,
                       double* kick_vz, double* kick_vx, const int64_t* removed,
                       int64_t removed_cap, double extent_z, double extent_x, void* stream);
int lbx_unpack_peer_dev(lbx_ctx* ctx, const double* recv, uint64_t* cursor, int64_t capacity,
                        double* z, double* x, double* vz, double* vx, double* kick_vz,
                        double* kick_vx, void* stream);
/* Group `count` staged records by destination into `send` ([count][6]);
 * cursors[world] (device) holds each destination's first slot on entry. */
int lbx_group_by_dest(const double* stage, const int32_t* stage_dest, int64_t count,
                      int32_t world, int64_t* cursors, double* send, void* stream);
/* Append n_recv received records at index `offset` of the SoA arrays
 * (kick_vz/kick_vx may be NULL). */
int lbx_unpack(const double* recv, int64_t n_recv, int64_t offset, double* z, double* x,
               double* vz, double* vx, double* kick_vz, double* kick_vx, void* stream);

/* Peer memory for the fused exchange.  lbx_peer_alloc: cudaMalloc'd device
 * buffer (zeroed) and its 64-byte IPC handle; lbx_peer_open maps another
 * process's buffer (NVLink / NVSwitch peer access enabled lazily; same-GPU
 * processes also work); lbx_peer_close / lbx_peer_free release them.
 * lbx_peer_can_access: 1 if device `dev` can access device `peer`. */
int lbx_peer_alloc(int64_t bytes, void** ptr, unsigned char handle[64]);
int lbx_peer_open(const unsigned char handle[64], void** ptr);
int lbx_peer_close(void* ptr);
int lbx_peer_free(void* ptr);
int lbx_peer_can_access(int32_t dev, int32_t peer, int32_t* yes);

#ifdef __cplusplus
}
#endif
#endif /* LBX_H_ */
