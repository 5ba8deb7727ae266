// Host setup driver: the B200 plan's counterpart of build_system
// (problem.cpp:73-108) up to, but excluding, the device upload.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "setup.hpp"

namespace hxb {

HexMesh mesh_from_arrays(int nv, const double* xyz, int ne, const std::int32_t* conn, int nbf, const std::int32_t* be,
                         const std::int32_t* bf, const std::uint8_t* bt)
{
  if (nv < 0 || ne < 0 || nbf < 0) throw HxbError(1, "negative mesh sizes");
  if ((nv > 0 && !xyz) || (ne > 0 && !conn) || (nbf > 0 && (!be || !bf || !bt)))
    throw HxbError(1, "mesh arrays must be non-null");
  HexMesh mesh;
  mesh.vertices.resize(nv);
  for (int v = 0; v < nv; ++v)
    for (int d = 0; d < 3; ++d) mesh.vertices[v][d] = xyz[3 * static_cast<std::size_t>(v) + d];
  mesh.elements.resize(ne);
  for (int e = 0; e < ne; ++e)
    for (int q = 0; q < 8; ++q) mesh.elements[e][q] = conn[8 * static_cast<std::size_t>(e) + q];
  for (int b = 0; b < nbf; ++b) {
    if (be[b] < 0 || be[b] >= ne || bf[b] < 0 || bf[b] > 5 || bt[b] > 1)
      throw HxbError(1, "boundary face out of range");
    mesh.boundary_faces.push_back({be[b], bf[b], bt[b]});
  }
  return mesh;
}

void setup_phase(const char* name)
{
  static const bool on = [] {
    const char* v = std::getenv("HXB_SETUP_TIMING");
    return v && *v && *v != '0';
  }();
  if (!on) return;
  using clk = std::chrono::steady_clock;
  static thread_local clk::time_point t0;
  static thread_local std::string cur;
  const auto now = clk::now();
  if (!cur.empty())
    std::fprintf(stderr, "[hxb setup] %-28s %8.3f s\n", cur.c_str(), std::chrono::duration<double>(now - t0).count());
  cur = name ? name : "";
  t0 = now;
}

void build_host_setup(HostSetup& hs, int order, const SetupOptions& opt)
{
  if (order < 1 || order > 10) throw HxbError(1, "order must lie in 1..10");
  if (opt.precond_mode < 0 || opt.precond_mode > 3) throw HxbError(1, "unknown precond mode");
  const int ne = hs.mesh.num_elements();
  if (static_cast<int>(hs.kappa.size()) != ne || static_cast<int>(hs.c.size()) != ne)
    throw HxbError(1, "kappa/c must hold one value per element");
  for (int e = 0; e < ne; ++e) {  // operator.cpp:69-75
    if (hs.kappa[e] < 0) throw HxbError(1, "kappa must be nonnegative");
    if (hs.c[e] < 0) throw HxbError(1, "c must be nonnegative");
  }
  hs.order = order;
  hs.do_fine = opt.precond_mode == 0 || opt.precond_mode == 1;
  hs.do_coarse = opt.precond_mode == 0 || opt.precond_mode == 2;
  if (hs.do_fine)
    for (int e = 0; e < ne; ++e)  // solve_subdomain precondition (fine.cpp:150-151)
      if (!(hs.kappa[e] > 0)) throw HxbError(1, "need kappa > 0, c >= 0");

  hs.basis = make_gll_basis(order);
  setup_phase("geometry");
  if (opt.geometry_hook) {  // device plans: factors computed on the GPU (kernels_setup.cuh)
    hs.geo = Geometry{};
    hs.geo.h = element_dimensions_all(hs.mesh);
    opt.geometry_hook(hs);
  } else {
    hs.geo = compute_geometry(hs.mesh, hs.basis, hs.kappa, opt.store_planes);  // throws on inverted elements
  }
  setup_phase("numbering");
  hs.num = build_numbering(hs.mesh, order);
  setup_phase("lumped mass");
  const int nloc = hs.basis.npts() * hs.basis.npts() * hs.basis.npts();
  if (!opt.device_lumped) {
    hs.lumped.assign(hs.num.num_global, 0.0);
    std::vector<gid> l2g(nloc);
    for (int e = 0; e < ne; ++e) {
      element_l2g(hs.num, ne, e, l2g.data());
      for (int l = 0; l < nloc; ++l) hs.lumped[l2g[l]] += hs.geo.mass[static_cast<std::size_t>(e) * nloc + l];
    }
  }
  hs.pencil = build_pencil(hs.basis);
  if (hs.do_coarse) {
    setup_phase("coarse matrix");
    hs.vmask = coarse_dirichlet_mask(hs.mesh);
    hs.Kc = assemble_coarse_matrix(hs.mesh, hs.kappa, hs.c, hs.vmask);
    hs.use_amg = opt.coarse_solve == 2 || (opt.coarse_solve == 0 && hs.Kc.n > opt.direct_threshold);
    setup_phase("amg setup");
    if (hs.use_amg) hs.amg = amg_setup(hs.Kc);
  }
  setup_phase("after host setup");
}

void export_index_maps(const HostSetup& hs, std::int32_t* l2g, std::int64_t* g2l_offsets, std::int32_t* g2l_elem,
                       std::int32_t* g2l_local, std::int32_t* sub_l2g, std::uint8_t* mask)
{
  const Numbering& num = hs.num;
  const int ne = hs.mesh.num_elements(), np = hs.order + 1, nloc = np * np * np, P = hs.order + 3;
  const int N = num.num_global;
  std::vector<gid> full(static_cast<std::size_t>(ne) * nloc);
  for (int e = 0; e < ne; ++e) element_l2g(num, ne, e, full.data() + static_cast<std::size_t>(e) * nloc);
  if (l2g) std::memcpy(l2g, full.data(), full.size() * sizeof(gid));
  if (g2l_offsets || g2l_elem || g2l_local) {
    std::vector<std::int64_t> off(static_cast<std::size_t>(N) + 1, 0);
    for (gid g : full) off[g + 1]++;
    for (int g = 0; g < N; ++g) off[g + 1] += off[g];
    if (g2l_offsets) std::memcpy(g2l_offsets, off.data(), off.size() * sizeof(std::int64_t));
    std::vector<std::int64_t> cur(off.begin(), off.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int l = 0; l < nloc; ++l) {
        const std::int64_t s = cur[full[static_cast<std::size_t>(e) * nloc + l]]++;
        if (g2l_elem) g2l_elem[s] = e;
        if (g2l_local) g2l_local[s] = l;
      }
  }
  if (sub_l2g) {
    const std::size_t nsub = static_cast<std::size_t>(P) * P * P;
    std::vector<gid> scratch(nloc);
    for (int e = 0; e < ne; ++e)
      for_each_sub_slot(num, ne, e, scratch.data(),
                        [&](gid g, int slot) { sub_l2g[static_cast<std::size_t>(e) * nsub + slot] = g; });
  }
  if (mask) std::memcpy(mask, num.dirichlet_mask.data(), num.dirichlet_mask.size());
}

}  // namespace hxb
