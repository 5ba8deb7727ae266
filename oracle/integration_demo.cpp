// TEST INFRASTRUCTURE ONLY — the INTEGRATION.md binding, compiled and run.
//
// Links the UNMODIFIED reference (oracle/_ref/obj/*.o) with
// integration/hexsem_b200_adapter.hpp and libhexsem_b200.so, then solves the
// same problem three ways through the reference's own public API:
//   ref   pcg(sys.operator_fn(), sys.preconditioner_fn(), b)   (all reference)
//   plug  pcg(b200_operator(plan), b200_preconditioner(plan), b) (reference loop,
//         B200 operators: the plug-in level)
//   solve b200_pcg(plan, b)                                     (solve level)
// and prints one JSON line (iterations, final residuals, max |dr_k|/r_0, ||u||).
// usage: integration_demo k order family(0..2) precond(0..3) [devices "0,0" | bitwise]
//   devices: a multi-GPU plan, one element slab per listed device
//   bitwise: the bitwise-reference plan (every difference must be exactly 0)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "hexsem_b200_adapter.hpp"

using namespace hexsem;

int main(int argc, char** argv)
{
  ProblemConfig cfg;
  cfg.k = argc > 1 ? std::atoi(argv[1]) : 8;
  cfg.order = argc > 2 ? std::atoi(argv[2]) : 4;
  cfg.family = static_cast<MeshFamily>(argc > 3 ? std::atoi(argv[3]) : 0);
  cfg.precond = static_cast<PrecondMode>(argc > 4 ? std::atoi(argv[4]) : 0);
  cfg.pcg.rel_tolerance = 1e-8;
  try {
    SemSystem sys = build_system(cfg);
    const Vector b = sys.assemble_load([](const std::array<Real, 3>&) { return Real(1); });  // problem.cpp:129
    const PcgResult ref = pcg(sys.operator_fn(), sys.preconditioner_fn(), b, cfg.pcg);
    const gid ne = sys.mesh.num_elements();
    std::vector<int> devices;
    bool bitwise = false;
    if (argc > 5) {
      const std::string mode = argv[5];
      if (mode == "bitwise") {
        bitwise = true;
      } else {
        std::size_t p = 0;
        while (p < mode.size()) {
          const std::size_t q = mode.find(',', p);
          devices.push_back(std::atoi(mode.substr(p, q == std::string::npos ? std::string::npos : q - p).c_str()));
          if (q == std::string::npos) break;
          p = q + 1;
        }
      }
    }
    hxb_plan* plan = make_b200_plan(sys.mesh, cfg.order, Vector(ne, cfg.kappa), Vector(ne, cfg.c), cfg.precond,
                                    cfg.coarse_solve, cfg.coarse_direct_threshold, OperatorVariant::stored, devices,
                                    bitwise);
    const PcgResult plug = pcg(b200_operator(plan), b200_preconditioner(plan), b, cfg.pcg);
    const PcgResult solve = b200_pcg(plan, b, cfg.pcg);
    hxb_plan_destroy(plan);
    auto dr = [&](const PcgResult& a) {
      double m = 0;
      const std::size_t n = std::min(a.residual_history.size(), ref.residual_history.size());
      for (std::size_t q = 0; q < n; ++q)
        m = std::fmax(m, std::fabs(a.residual_history[q] - ref.residual_history[q]));
      return m / ref.residual_history[0];
    };
    auto du = [&](const PcgResult& a) {
      double d = 0, n = 0;
      for (std::size_t q = 0; q < ref.u.size(); ++q) {
        d += (a.u[q] - ref.u[q]) * (a.u[q] - ref.u[q]);
        n += ref.u[q] * ref.u[q];
      }
      return std::sqrt(d / n);
    };
    std::printf("{\"N\": %d, \"n_gpus\": %d, \"ref_iterations\": %d, \"plug_iterations\": %d, \"solve_iterations\": %d, "
                "\"plug_max_dr_over_r0\": %.3e, \"solve_max_dr_over_r0\": %.3e, \"plug_u_rel\": %.3e, "
                "\"solve_u_rel\": %.3e, \"ref_status\": %d, \"plug_status\": %d, \"solve_status\": %d}\n",
                sys.maps.num_global, std::max<int>(1, static_cast<int>(devices.size())), ref.iterations, plug.iterations, solve.iterations, dr(plug), dr(solve), du(plug),
                du(solve), static_cast<int>(ref.status), static_cast<int>(plug.status),
                static_cast<int>(solve.status));
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
