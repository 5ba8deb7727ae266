// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the UNMODIFIED reference library (hexsem, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load it; the product never links it.
//
// Every entry point forwards to the reference's own public API:
//   build_system / SemSystem           problem.hpp:68-85, problem.cpp:73-108
//   SemOperator::apply                 operator.cpp:255-287
//   TwoScalePreconditioner::apply      precond.cpp:27-67
//   FinePreconditioner::apply          fine.cpp:210-231
//   CoarsePreconditioner::apply etc.   coarse.cpp:138-208
//   pcg                                krylov.cpp:20-71
//   build_index_maps                   mesh.cpp:287-453
//   build_pencil                       fine.cpp:15-80
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "hexsem/mesh_io.hpp"
#include "hexsem/problem.hpp"

using namespace hexsem;

namespace {

thread_local std::string g_err;

// SemOperator & co. keep raw pointers into SemSystem (operator.hpp:78-80),
// so the system must be built in place, never moved.
struct RefSystem {
  ProblemConfig cfg;
  double build_seconds = 0;
  SemSystem sys;
};

template <class F>
int guard(F&& f)
{
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

// Mirrors ProblemConfig (problem.hpp:35-62); enums as ints in declaration order.
struct ref_config {
  int k, refine, family, boundary;      // MeshFamily, BoundaryTag
  int bar[3];
  double bar_size[3];
  int order;
  double kappa, c;
  int precond;                          // PrecondMode: two_scale, fine_only, coarse_only, none
  int variant;                          // OperatorVariant: stored, on_the_fly
  int coarse_solve;                     // CoarseSolve: automatic, direct, amg
  int coarse_direct_threshold;
  int concurrent_precond, fine_threads;
};

const char* ref_last_error() { return g_err.c_str(); }

static ProblemConfig to_cfg(const ref_config* c)
{
  ProblemConfig cfg;
  cfg.k = c->k;
  cfg.refine = c->refine;
  cfg.family = static_cast<MeshFamily>(c->family);
  cfg.boundary = static_cast<BoundaryTag>(c->boundary);
  for (int d = 0; d < 3; ++d) {
    cfg.bar[d] = c->bar[d];
    cfg.bar_size[d] = c->bar_size[d];
  }
  cfg.order = c->order;
  cfg.kappa = c->kappa;
  cfg.c = c->c;
  cfg.precond = static_cast<PrecondMode>(c->precond);
  cfg.variant = static_cast<OperatorVariant>(c->variant);
  cfg.coarse_solve = static_cast<CoarseSolve>(c->coarse_solve);
  cfg.coarse_direct_threshold = c->coarse_direct_threshold;
  cfg.concurrent_precond = c->concurrent_precond != 0;
  cfg.fine_threads = c->fine_threads;
  return cfg;
}

// build_system(config) — problem.cpp:73-108
int ref_create(const ref_config* c, void** out)
{
  return guard([&] {
    const ProblemConfig cfg = to_cfg(c);
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<RefSystem> h(new RefSystem{cfg, 0.0, build_system(cfg)});
    h->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
  });
}

// Same construction order as build_system (problem.cpp:73-108) but on a
// caller-supplied mesh with per-element kappa/c (the class constructors
// accept vectors: operator.hpp:49-55, fine.hpp:60-61, coarse.hpp:33-36).
int ref_create_mesh(int nv, const double* xyz, int ne, const int32_t* conn, int nbf,
                    const int32_t* bf_elem, const int32_t* bf_face, const uint8_t* bf_tag,
                    int order, const double* kappa_e, const double* c_e, const ref_config* c,
                    void** out)
{
  return guard([&] {
    auto h = std::make_unique<RefSystem>();
    h->cfg = to_cfg(c);
    h->cfg.order = order;
    const auto t0 = std::chrono::steady_clock::now();
    SemSystem& sys = h->sys;
    sys.mesh.vertices.resize(nv);
    for (int v = 0; v < nv; ++v)
      for (int d = 0; d < 3; ++d) sys.mesh.vertices[v][d] = xyz[3 * v + d];
    sys.mesh.elements.resize(ne);
    for (int e = 0; e < ne; ++e)
      for (int q = 0; q < 8; ++q) sys.mesh.elements[e][q] = conn[8 * e + q];
    for (int b = 0; b < nbf; ++b)
      sys.mesh.boundary_faces.push_back(
          {bf_elem[b], bf_face[b], static_cast<BoundaryTag>(bf_tag[b])});
    check_jacobians(sys.mesh);
    sys.basis = make_gll_basis(order);
    sys.maps = build_index_maps(sys.mesh, sys.basis);
    Vector kappa(kappa_e, kappa_e + ne), cc(c_e, c_e + ne);
    GeometricFactors factors = compute_factors(sys.mesh, sys.basis);
    const auto mode = h->cfg.precond;
    const bool need_fine = mode == PrecondMode::two_scale || mode == PrecondMode::fine_only;
    const bool need_coarse = mode == PrecondMode::two_scale || mode == PrecondMode::coarse_only;
    if (need_coarse)
      sys.coarse = std::make_unique<CoarsePreconditioner>(sys.mesh, sys.basis, sys.maps, factors,
                                                          kappa, cc, h->cfg.coarse_solve,
                                                          h->cfg.coarse_direct_threshold);
    if (need_fine)
      sys.fine = std::make_unique<FinePreconditioner>(sys.mesh, sys.basis, sys.maps, kappa, cc);
    sys.op = std::make_unique<SemOperator>(sys.mesh, sys.basis, sys.maps, std::move(factors),
                                           std::move(kappa), std::move(cc), h->cfg.variant);
    sys.precond = std::make_unique<TwoScalePreconditioner>(
        sys.maps, sys.fine.get(), sys.coarse.get(), mode, h->cfg.concurrent_precond,
        h->cfg.fine_threads);
    h->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
  });
}

void ref_destroy(void* h) { delete static_cast<RefSystem*>(h); }

// info[0..9] = N, NE, NV, order, coarse_n, coarse_amg, amg_levels, nbf, build_ms, has_fine
int ref_info(void* hp, int64_t* info)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const SemSystem& s = h->sys;
    info[0] = s.maps.num_global;
    info[1] = s.mesh.num_elements();
    info[2] = s.mesh.num_vertices();
    info[3] = s.basis.order;
    info[4] = s.coarse ? s.coarse->num_coarse() : 0;
    info[5] = s.coarse ? (s.coarse->uses_amg() ? 1 : 0) : 0;
    info[6] = (s.coarse && s.coarse->hierarchy()) ? s.coarse->hierarchy()->num_levels() : 0;
    info[7] = static_cast<int64_t>(s.mesh.boundary_faces.size());
    info[8] = static_cast<int64_t>(h->build_seconds * 1000.0);
    info[9] = s.fine ? 1 : 0;
  });
}

int ref_export_mesh(void* hp, double* xyz, int32_t* conn, int32_t* bf_elem, int32_t* bf_face,
                    uint8_t* bf_tag)
{
  return guard([&] {
    const HexMesh& m = static_cast<RefSystem*>(hp)->sys.mesh;
    for (std::size_t v = 0; v < m.vertices.size(); ++v)
      for (int d = 0; d < 3; ++d) xyz[3 * v + d] = m.vertices[v][d];
    for (std::size_t e = 0; e < m.elements.size(); ++e)
      for (int q = 0; q < 8; ++q) conn[8 * e + q] = m.elements[e][q];
    for (std::size_t b = 0; b < m.boundary_faces.size(); ++b) {
      bf_elem[b] = m.boundary_faces[b].element;
      bf_face[b] = m.boundary_faces[b].face;
      bf_tag[b] = static_cast<uint8_t>(m.boundary_faces[b].tag);
    }
  });
}

// IndexMaps (mesh.hpp:66-97); any output pointer may be NULL.
int ref_export_maps(void* hp, int32_t* l2g, int64_t* g2l_off, int32_t* g2l_elem,
                    int32_t* g2l_local, int32_t* sub_l2g, uint8_t* mask)
{
  return guard([&] {
    const IndexMaps& m = static_cast<RefSystem*>(hp)->sys.maps;
    if (l2g) std::memcpy(l2g, m.l2g.data(), m.l2g.size() * sizeof(int32_t));
    if (g2l_off)
      for (std::size_t i = 0; i < m.g2l_offsets.size(); ++i) g2l_off[i] = static_cast<int64_t>(m.g2l_offsets[i]);
    if (g2l_elem) std::memcpy(g2l_elem, m.g2l_elem.data(), m.g2l_elem.size() * sizeof(int32_t));
    if (g2l_local) std::memcpy(g2l_local, m.g2l_local.data(), m.g2l_local.size() * sizeof(int32_t));
    if (sub_l2g) std::memcpy(sub_l2g, m.sub_l2g.data(), m.sub_l2g.size() * sizeof(int32_t));
    if (mask) std::memcpy(mask, m.dirichlet_mask.data(), m.dirichlet_mask.size());
  });
}

int ref_apply_A(void* hp, const double* u, double* r)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const std::size_t n = h->sys.maps.num_global;
    h->sys.op->apply(std::span<const Real>(u, n), std::span<Real>(r, n));
  });
}

int ref_apply_P(void* hp, const double* r, double* z)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const std::size_t n = h->sys.maps.num_global;
    h->sys.precond->apply(std::span<const Real>(r, n), std::span<Real>(z, n));
  });
}

int ref_apply_fine(void* hp, const double* r, double* z)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const std::size_t n = h->sys.maps.num_global;
    if (!h->sys.fine) throw std::invalid_argument("system has no fine preconditioner");
    h->sys.fine->apply(std::span<const Real>(r, n), std::span<Real>(z, n));
  });
}

int ref_apply_coarse(void* hp, const double* r, double* z)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const std::size_t n = h->sys.maps.num_global;
    if (!h->sys.coarse) throw std::invalid_argument("system has no coarse preconditioner");
    h->sys.coarse->apply(std::span<const Real>(r, n), std::span<Real>(z, n));
  });
}

int ref_restrict(void* hp, const double* r, double* R)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    h->sys.coarse->restrict_residual(std::span<const Real>(r, h->sys.maps.num_global),
                                     std::span<Real>(R, h->sys.mesh.num_vertices()));
  });
}

int ref_prolongate(void* hp, const double* Z, double* z)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    h->sys.coarse->prolongate(std::span<const Real>(Z, h->sys.mesh.num_vertices()),
                              std::span<Real>(z, h->sys.maps.num_global));
  });
}

int ref_lumped_mass(void* hp, double* m)
{
  return guard([&] {
    const Vector& lm = static_cast<RefSystem*>(hp)->sys.op->lumped_mass();
    std::memcpy(m, lm.data(), lm.size() * sizeof(double));
  });
}

// b = m_N * 1 masked (problem.cpp:38-46, 129)
int ref_load_ones(void* hp, double* b)
{
  return guard([&] {
    const Vector v =
        static_cast<RefSystem*>(hp)->sys.assemble_load([](const std::array<Real, 3>&) { return Real(1); });
    std::memcpy(b, v.data(), v.size() * sizeof(double));
  });
}

// Coarse matrix CSR (coarse.cpp:21-87): sizes first (ptr may be NULL).
int ref_coarse_matrix(void* hp, int64_t* nnz, int64_t* ptr, int32_t* col, double* val)
{
  return guard([&] {
    const CsrMatrix& K = static_cast<RefSystem*>(hp)->sys.coarse->coarse_matrix();
    *nnz = static_cast<int64_t>(K.nnz());
    if (!ptr) return;
    for (std::size_t i = 0; i < K.ptr.size(); ++i) ptr[i] = static_cast<int64_t>(K.ptr[i]);
    std::memcpy(col, K.col.data(), K.col.size() * sizeof(int32_t));
    std::memcpy(val, K.val.data(), K.val.size() * sizeof(double));
  });
}

// AMG level l (amg.hpp:52-60): rows, nnz, and (if non-NULL) CSR + aggregates.
int ref_amg_level(void* hp, int l, int64_t* rows, int64_t* nnz, int64_t* ptr, int32_t* col,
                  double* val, int32_t* agg)
{
  return guard([&] {
    const AmgHierarchy* a = static_cast<RefSystem*>(hp)->sys.coarse->hierarchy();
    if (!a) throw std::invalid_argument("coarse solve is not AMG");
    const CsrMatrix& A = a->level_matrix(l);
    *rows = A.n;
    *nnz = static_cast<int64_t>(A.nnz());
    if (ptr) {
      for (std::size_t i = 0; i < A.ptr.size(); ++i) ptr[i] = static_cast<int64_t>(A.ptr[i]);
      std::memcpy(col, A.col.data(), A.col.size() * sizeof(int32_t));
      std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
    }
    if (agg && l + 1 < a->num_levels()) {
      const auto& g = a->aggregates(l);
      std::memcpy(agg, g.data(), g.size() * sizeof(int32_t));
    }
  });
}

// pcg(operator_fn, preconditioner_fn, b, cfg) — krylov.cpp:20-71. History
// buffers hold max_iterations+1 entries. status: 0 converged, 1 max, 2 breakdown.
int ref_pcg(void* hp, const double* b, double tol, int max_iterations, int* iterations,
            int* status, double* residual_history, double* zr_history, double* u,
            double* solve_seconds)
{
  return guard([&] {
    auto* h = static_cast<RefSystem*>(hp);
    const std::size_t n = h->sys.maps.num_global;
    PcgConfig pc;
    pc.rel_tolerance = tol;
    pc.max_iterations = max_iterations;
    pc.record_history = true;
    const auto t0 = std::chrono::steady_clock::now();
    PcgResult res = pcg(h->sys.operator_fn(), h->sys.preconditioner_fn(),
                        std::span<const Real>(b, n), pc);
    if (solve_seconds)
      *solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *iterations = res.iterations;
    *status = static_cast<int>(res.status);
    if (residual_history)
      std::memcpy(residual_history, res.residual_history.data(), res.residual_history.size() * sizeof(double));
    if (zr_history) std::memcpy(zr_history, res.zr_history.data(), res.zr_history.size() * sizeof(double));
    if (u) std::memcpy(u, res.u.data(), n * sizeof(double));
    if (!res.diagnostic.empty()) g_err = res.diagnostic;
  });
}

// GllBasis (gll.hpp:17-31)
int ref_gll(int n, double* nodes, double* weights, double* deriv, double* vdm)
{
  return guard([&] {
    const GllBasis b = make_gll_basis(n);
    std::memcpy(nodes, b.nodes.data(), b.nodes.size() * sizeof(double));
    std::memcpy(weights, b.weights.data(), b.weights.size() * sizeof(double));
    std::memcpy(deriv, b.deriv.data(), b.deriv.size() * sizeof(double));
    if (vdm) std::memcpy(vdm, b.coarse_vandermonde.data(), b.coarse_vandermonde.size() * sizeof(double));
  });
}

// PencilFactorization (fine.hpp:18-26)
int ref_pencil(int n, double* K, double* M, double* V, double* Vinv, double* lambda)
{
  return guard([&] {
    const PencilFactorization p = build_pencil(make_gll_basis(n));
    std::memcpy(K, p.K_ext.data(), p.K_ext.size() * sizeof(double));
    std::memcpy(M, p.M_ext.data(), p.M_ext.size() * sizeof(double));
    std::memcpy(V, p.V.data(), p.V.size() * sizeof(double));
    std::memcpy(Vinv, p.V_inv.data(), p.V_inv.size() * sizeof(double));
    std::memcpy(lambda, p.lambda.data(), p.lambda.size() * sizeof(double));
  });
}

// element h (geometry.cpp:76-103) for all elements, [NE][3]
int ref_element_h(void* hp, double* h3)
{
  return guard([&] {
    const HexMesh& m = static_cast<RefSystem*>(hp)->sys.mesh;
    for (gid e = 0; e < m.num_elements(); ++e) {
      const auto h = element_dimensions(m, e);
      for (int d = 0; d < 3; ++d) h3[3 * e + d] = h[d];
    }
  });
}

// solve_heat (problem.cpp:145-255) through the reference's own driver.
struct ref_heat {
  double dt;
  int steps;
  double rho, cp, q_power, source_radius;
  int has_source, auto_trajectory;
  double source_start[3], source_end[3];
  double initial_value;
};

int ref_solve_heat(const ref_config* c, const ref_heat* h, double tol, int max_iterations, int64_t n_cap,
                   int* num_steps, int* all_converged, int* iterations, double* residual, double* mean,
                   double* l2, double* source_integral, double* final_u, int64_t* n_out, double* seconds)
{
  return guard([&] {
    ProblemConfig cfg = to_cfg(c);
    cfg.pcg.rel_tolerance = tol;
    cfg.pcg.max_iterations = max_iterations;
    cfg.heat.dt = h->dt;
    cfg.heat.steps = h->steps;
    cfg.heat.rho = h->rho;
    cfg.heat.cp = h->cp;
    cfg.heat.q_power = h->q_power;
    cfg.heat.source_radius = h->source_radius;
    cfg.heat.has_source = h->has_source != 0;
    cfg.heat.auto_trajectory = h->auto_trajectory != 0;
    for (int d = 0; d < 3; ++d) {
      cfg.heat.source_start[d] = h->source_start[d];
      cfg.heat.source_end[d] = h->source_end[d];
    }
    cfg.heat.initial_value = h->initial_value;
    const HeatReport rep = solve_heat(cfg);
    *num_steps = static_cast<int>(rep.steps.size());
    *all_converged = rep.all_converged ? 1 : 0;
    for (std::size_t q = 0; q < rep.steps.size(); ++q) {
      iterations[q] = rep.steps[q].iterations;
      residual[q] = rep.steps[q].residual;
      mean[q] = rep.steps[q].mean_temperature;
      l2[q] = rep.steps[q].l2_norm;
      source_integral[q] = rep.steps[q].source_integral;
    }
    *n_out = static_cast<int64_t>(rep.final_field.size());
    if (final_u && n_cap >= *n_out) std::memcpy(final_u, rep.final_field.data(), rep.final_field.size() * sizeof(double));
    if (seconds) *seconds = rep.base.timings.solve_seconds;
  });
}

// Counter models (operator.cpp:20-37, fine.cpp:82-92)
unsigned long long ref_words_model(long long ne, int n, int variant)
{
  return KernelCounters::words_model(ne, n, static_cast<OperatorVariant>(variant));
}
unsigned long long ref_flops_model(long long ne, int n) { return KernelCounters::contraction_flops_model(ne, n); }
unsigned long long ref_fine_ops_model(long long ne, int n) { return FineCounters::ops_model(ne, n); }
unsigned long long ref_fine_words_model(long long ne, int n) { return FineCounters::words_model(ne, n); }

// Mesh files through the reference's own readers/writers (mesh_io.cpp): the
// cross-implementation fixtures for the mesh-format row.
static HexMesh mesh_of(int nv, const double* xyz, int ne, const int32_t* conn, int nbf, const int32_t* be,
                       const int32_t* bf, const uint8_t* bt)
{
  HexMesh m;
  m.vertices.resize(nv);
  for (int v = 0; v < nv; ++v)
    for (int d = 0; d < 3; ++d) m.vertices[v][d] = xyz[3 * v + d];
  m.elements.resize(ne);
  for (int e = 0; e < ne; ++e)
    for (int q = 0; q < 8; ++q) m.elements[e][q] = conn[8 * e + q];
  for (int b = 0; b < nbf; ++b) m.boundary_faces.push_back({be[b], bf[b], static_cast<BoundaryTag>(bt[b])});
  return m;
}

// format: 0 = by extension (write_mesh_file), 1 = write_msh, 2 = write_native
int ref_write_mesh(int nv, const double* xyz, int ne, const int32_t* conn, int nbf, const int32_t* be,
                   const int32_t* bf, const uint8_t* bt, const char* path, int format)
{
  return guard([&] {
    const HexMesh m = mesh_of(nv, xyz, ne, conn, nbf, be, bf, bt);
    if (format == 1)
      write_msh(m, path);
    else if (format == 2)
      write_native(m, path);
    else
      write_mesh_file(m, path);
  });
}

// format: 0 = read_mesh_file, 1 = read_msh, 2 = read_native
int ref_read_mesh(const char* path, int format, void** out)
{
  return guard([&] {
    auto m = std::make_unique<HexMesh>(format == 1 ? read_msh(path)
                                       : format == 2 ? read_native(path)
                                                     : read_mesh_file(path));
    *out = m.release();
  });
}

void ref_mesh_counts(void* m, int64_t* c)
{
  const HexMesh& h = *static_cast<HexMesh*>(m);
  c[0] = h.num_vertices();
  c[1] = h.num_elements();
  c[2] = static_cast<int64_t>(h.boundary_faces.size());
}

void ref_mesh_export(void* m, double* xyz, int32_t* conn, int32_t* be, int32_t* bf, uint8_t* bt)
{
  const HexMesh& h = *static_cast<HexMesh*>(m);
  for (std::size_t v = 0; v < h.vertices.size(); ++v)
    for (int d = 0; d < 3; ++d) xyz[3 * v + d] = h.vertices[v][d];
  for (std::size_t e = 0; e < h.elements.size(); ++e)
    for (int q = 0; q < 8; ++q) conn[8 * e + q] = h.elements[e][q];
  for (std::size_t b = 0; b < h.boundary_faces.size(); ++b) {
    be[b] = h.boundary_faces[b].element;
    bf[b] = h.boundary_faces[b].face;
    bt[b] = static_cast<uint8_t>(h.boundary_faces[b].tag);
  }
}

void ref_mesh_free(void* m) { delete static_cast<HexMesh*>(m); }

}  // extern "C"
