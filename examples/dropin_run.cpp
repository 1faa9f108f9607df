// dropin_run.cpp — the reference's own C++ API, switched to the GPU by namespace.
//
// Builds against the UNMODIFIED reference headers (/root/reference/proj/include)
// and include/enmf_gpu.hpp; runs config 1 (gen_lowrank 200x200 r=20 seed 1,
// random_init seed 2, e-ahals-hp3, 200 iterations) through enmf::run (CPU) and
// enmf::gpu::run (B200) and prints both final relative errors and the largest
// per-iteration deviation.  Build: make -C examples (needs /root/reference).
#include <cmath>
#include <cstdio>

#include <enmf/data.hpp>
#include <enmf/engine.hpp>

#include "enmf_gpu.hpp"

int main() {
  const enmf::DenseMatrix x = enmf::gen_lowrank(200, 200, 20, 1);
  const auto [w0, h0] = enmf::random_init(200, 200, 20, 2);
  enmf::SolverConfig cfg;
  cfg.inner_h = cfg.inner_w = enmf::InnerSolver::hals;
  cfg.hp = 3;
  cfg.beta0 = 0.5;
  cfg.gamma = 1.01;
  cfg.gamma_bar = 1.005;
  cfg.eta = 1.5;
  cfg.max_outer_iterations = 200;
  const enmf::RunRecord cpu = enmf::run(x, w0, h0, cfg, enmf::TimingMode::none);
  const enmf::RunRecord gpu = enmf::gpu::run(x, w0, h0, cfg, enmf::TimingMode::none);
  double worst = 0.0;
  int restart_mismatch = 0;
  for (std::size_t k = 0; k < cpu.iterations.size(); ++k) {
    const double a = cpu.iterations[k].error, b = gpu.iterations[k].error;
    worst = std::fmax(worst, std::fabs(a - b) / a);
    restart_mismatch += cpu.iterations[k].restarted != gpu.iterations[k].restarted;
  }
  std::printf("cpu final %.17g  gpu final %.17g  worst rel dev %.3e  restart mismatches %d\n",
              cpu.final_relative_error(), gpu.final_relative_error(), worst, restart_mismatch);
  return (worst <= 1e-9 && restart_mismatch == 0) ? 0 : 1;
}
