// hexsem_b200_adapter.hpp — the reference-side binding.
//
// Drop next to proj/include/hexsem/problem.hpp in the reference tree and link
// paper_1506_05996_b200/libhexsem_b200.so: the B200 plan then supplies the
// bodies of the reference's own LinearOp plug-in points (krylov.hpp:32,
// SemSystem::operator_fn / preconditioner_fn, problem.cpp:28-36), or replaces
// pcg(...) as a whole (krylov.hpp:37-38). Only the C-ABI of
// include/hexsem_b200.h crosses the boundary (plain pointers and sizes).
#ifndef HEXSEM_B200_ADAPTER_HPP
#define HEXSEM_B200_ADAPTER_HPP

#include <stdexcept>
#include <vector>

#include "hexsem/problem.hpp"
#include "hexsem_b200.h"

namespace hexsem {

// build_system's mesh and per-element coefficients -> a device plan
// devices: empty = one GPU (device 0); several = a multi-GPU plan with one
// element slab per entry (hxb_options.n_gpus / devices, NCCL between distinct
// devices). bitwise: the reference-order verification mode
// (hxb_options.bitwise_reference), equal to this reference bit for bit.
inline hxb_plan* make_b200_plan(const HexMesh& mesh, int order, const Vector& kappa, const Vector& c, PrecondMode mode,
                                CoarseSolve coarse, gid direct_threshold,
                                OperatorVariant variant = OperatorVariant::stored,
                                const std::vector<int>& devices = {}, bool bitwise = false)
{
  std::vector<double> xyz(3 * mesh.vertices.size());
  for (std::size_t v = 0; v < mesh.vertices.size(); ++v)
    for (int d = 0; d < 3; ++d) xyz[3 * v + d] = mesh.vertices[v][d];
  std::vector<int32_t> conn(8 * mesh.elements.size());
  for (std::size_t e = 0; e < mesh.elements.size(); ++e)
    for (int q = 0; q < 8; ++q) conn[8 * e + q] = mesh.elements[e][q];
  std::vector<int32_t> be, bf;
  std::vector<uint8_t> bt;
  for (const auto& b : mesh.boundary_faces) {
    be.push_back(b.element);
    bf.push_back(b.face);
    bt.push_back(static_cast<uint8_t>(b.tag));
  }
  hxb_mesh m{mesh.num_vertices(), xyz.data(), mesh.num_elements(), conn.data(), static_cast<int32_t>(be.size()),
             be.data(),           bf.data(),  bt.data()};
  hxb_options opt;
  hxb_default_options(&opt);
  opt.precond_mode = static_cast<int>(mode);     // same enum order (precond.hpp:12)
  opt.coarse_solve = static_cast<int>(coarse);   // same enum order (coarse.hpp:28)
  opt.direct_threshold = direct_threshold;
  opt.variant = static_cast<int>(variant);       // same enum order (operator.hpp:14)
  opt.bitwise_reference = bitwise ? 1 : 0;
  if (devices.size() > HXB_MAX_GPUS) throw std::invalid_argument("at most HXB_MAX_GPUS devices");
  if (devices.size() == 1) opt.device = devices[0];
  if (devices.size() > 1) {
    opt.n_gpus = static_cast<int>(devices.size());
    for (std::size_t r = 0; r < devices.size(); ++r) opt.devices[r] = devices[r];
  }
  hxb_plan* plan = nullptr;
  if (int rc = hxb_plan_create(&m, order, kappa.data(), c.data(), &opt, &plan)) {
    if (rc == HXB_EINVAL) throw std::invalid_argument(hxb_last_error());
    throw std::runtime_error(hxb_last_error());
  }
  return plan;
}

inline LinearOp b200_operator(hxb_plan* plan)  // replaces SemSystem::operator_fn
{
  return [plan](std::span<const Real> u, std::span<Real> r) {
    if (hxb_apply_A(plan, u.data(), r.data())) throw std::runtime_error(hxb_last_error());
  };
}

inline LinearOp b200_preconditioner(hxb_plan* plan)  // replaces SemSystem::preconditioner_fn
{
  return [plan](std::span<const Real> r, std::span<Real> z) {
    if (hxb_apply_P(plan, r.data(), z.data())) throw std::runtime_error(hxb_last_error());
  };
}

// pcg(A, P, b, cfg) with the whole Krylov loop on the device (krylov.cpp:20-71)
inline PcgResult b200_pcg(hxb_plan* plan, std::span<const Real> b, const PcgConfig& cfg)
{
  hxb_plan_info info;
  if (hxb_plan_get_info(plan, &info)) throw std::runtime_error(hxb_last_error());
  hxb_pcg_config pc{cfg.rel_tolerance, cfg.max_iterations, cfg.record_history ? 1 : 0};
  PcgResult out;
  out.u.resize(static_cast<std::size_t>(info.num_global));
  std::vector<double> rh(cfg.max_iterations + 1), zh(cfg.max_iterations + 1);
  hxb_pcg_result res{};
  res.residual_history = rh.data();
  res.zr_history = zh.data();
  res.u = out.u.data();
  if (hxb_solve(plan, b.data(), &pc, &res)) throw std::runtime_error(hxb_last_error());
  out.status = static_cast<PcgStatus>(res.status);  // krylov.hpp:22
  out.iterations = res.iterations;
  out.residual_history.assign(rh.begin(), rh.begin() + res.num_residuals);
  out.zr_history.assign(zh.begin(), zh.begin() + res.num_zr);
  out.diagnostic = res.diagnostic;
  return out;
}

}  // namespace hexsem

#endif
