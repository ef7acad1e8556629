// Host LB step (lbx_lb_step) time per step on the C2 box grid, no Python: scripts/lb_host_bench.cpp
// build: g++ -O2 -Iinclude scripts/lb_host_bench.cpp -Lpaper_2104_11385_b200 -lLBX -Wl,-rpath,$PWD/paper_2104_11385_b200 -o /tmp/lbh
// run:   /tmp/lbh RANKS INTERVAL
#include <cstdlib>
#include "lbx.h"
#include <chrono>
#include <cstdio>
#include <vector>
#include <cstring>
int main(int argc, char** argv) {
  lbx_sim_config c{};
  c.extent_z = 960; c.extent_x = 960; c.box_size = 32; c.n_ranks = atoi(argv[1]);
  c.total_steps = 2000; c.kick_step = 0; c.strategy = LBX_STRATEGY_KNAPSACK; c.interval = atoi(argv[2]);
  c.improvement_threshold = 0.1; c.threshold_relative = 1; c.cap_factor = 1.5; c.static_step = -1;
  c.cost_kind = LBX_COST_HEURISTIC; c.w_particle = 0.75; c.w_cell = 0.25; c.work_wp = 1; c.work_wc = 0.1;
  c.capacity_particles = -1; c.overhead_factor = 1; c.physics = LBX_PHYSICS_SURROGATE; c.clock_mode = LBX_CLOCK_RAW;
  const int nb = 900, T = 2000;
  std::vector<int64_t> own(nb); for (int b = 0; b < nb; ++b) own[b] = (int64_t)b * c.n_ranks / nb;
  lbx_lb* lb; if (lbx_lb_create(&lb, &c, own.data())) { printf("%s\n", lbx_last_error()); return 1; }
  std::vector<double> d[7]; for (auto& v : d) v.assign(T, 0);
  std::vector<uint8_t> u[3]; for (auto& v : u) v.assign(T, 0);
  std::vector<int64_t> mrp(T), na(T), as(T), ao((size_t)T * nb);
  std::vector<double> ct((size_t)T * nb);
  lbx_sim_outputs o{};
  o.eff_before = d[0].data(); o.eff_after = d[1].data(); o.compute_max = d[2].data(); o.comm_max = d[3].data();
  o.gather = d[4].data(); o.redistribute = d[5].data(); o.walltime = d[6].data();
  o.adopted = u[0].data(); o.attempted = u[1].data(); o.oom = u[2].data();
  o.max_rank_particles = mrp.data(); o.n_alive = na.data(); o.cost_trace = ct.data(); o.owner = own.data();
  o.adopt_steps = as.data(); o.adopt_owners = ao.data();
  std::vector<int64_t> counts(nb); for (int b = 0; b < nb; ++b) counts[b] = (b * 7919) % 3000;
  int32_t a, h;
  auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < T; ++s) lbx_lb_step(lb, s, counts.data(), nullptr, 801499, &o, &a, &h);
  auto t1 = std::chrono::steady_clock::now();
  printf("R=%d interval=%d: %.2f us/step\n", c.n_ranks, (int)c.interval, std::chrono::duration<double, std::micro>(t1 - t0).count() / T);
}
