// Host-only part of the C-ABI (include/hexsem_b200.h): mesh generators,
// the GPU-free setup object used by the bit-exactness tests, counter models.
// Compiled with g++ (no CUDA); the device plan lives in plan.cu.
#include <cmath>
#include <cstring>
#include <memory>

#include "../../include/hexsem_b200.h"
#include "capi_common.hpp"

namespace hxb {

namespace {
thread_local std::string g_last_error;

struct MeshHolder {
  HexMesh mesh;
  std::vector<double> xyz;
  std::vector<std::int32_t> conn, be, bf;
  std::vector<std::uint8_t> bt;
};

hxb_mesh_buf* wrap_mesh(HexMesh&& m)
{
  auto h = std::make_unique<MeshHolder>();
  h->mesh = std::move(m);
  const HexMesh& mm = h->mesh;
  h->xyz.resize(3 * mm.vertices.size());
  for (std::size_t v = 0; v < mm.vertices.size(); ++v)
    for (int d = 0; d < 3; ++d) h->xyz[3 * v + d] = mm.vertices[v][d];
  h->conn.resize(8 * mm.elements.size());
  for (std::size_t e = 0; e < mm.elements.size(); ++e)
    for (int q = 0; q < 8; ++q) h->conn[8 * e + q] = mm.elements[e][q];
  for (const auto& b : mm.boundary_faces) {
    h->be.push_back(b.element);
    h->bf.push_back(b.face);
    h->bt.push_back(b.tag);
  }
  auto* out = new hxb_mesh_buf;
  out->view.num_vertices = static_cast<std::int32_t>(mm.vertices.size());
  out->view.xyz = h->xyz.data();
  out->view.num_elements = static_cast<std::int32_t>(mm.elements.size());
  out->view.conn = h->conn.data();
  out->view.num_boundary_faces = static_cast<std::int32_t>(h->be.size());
  out->view.bface_element = h->be.data();
  out->view.bface_face = h->bf.data();
  out->view.bface_tag = h->bt.data();
  out->impl = h.release();
  return out;
}

HexMesh view_to_mesh(const hxb_mesh* m)
{
  if (!m) throw HxbError(HXB_EINVAL, "mesh must be non-null");
  return mesh_from_arrays(m->num_vertices, m->xyz, m->num_elements, m->conn, m->num_boundary_faces,
                          m->bface_element, m->bface_face, m->bface_tag);
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

void export_amg_level(const HostSetup& hs, int level, std::int64_t* rows, std::int64_t* nnz, std::int64_t* ptr,
                      std::int32_t* col, double* val, std::int32_t* aggregate)
{
  if (!hs.use_amg) throw HxbError(HXB_EINVAL, "coarse solve is not AMG");
  const int L = static_cast<int>(hs.amg.levels.size());
  if (level < 0 || level > L) throw HxbError(HXB_EINVAL, "level out of range");
  const Csr& A = level < L ? hs.amg.levels[level].A : hs.amg.coarsest;
  *rows = A.n;
  *nnz = static_cast<std::int64_t>(A.nnz());
  if (ptr) {
    std::memcpy(ptr, A.ptr.data(), A.ptr.size() * sizeof(std::int64_t));
    std::memcpy(col, A.col.data(), A.col.size() * sizeof(std::int32_t));
    std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
  }
  if (aggregate && level < L)
    std::memcpy(aggregate, hs.amg.levels[level].aggregate.data(), hs.amg.levels[level].aggregate.size() * sizeof(std::int32_t));
}

void fill_amg_info(const HostSetup& hs, std::int32_t* levels, std::int64_t* rows, std::int64_t* nnz)
{
  *levels = 0;
  if (!hs.use_amg) return;
  const int L = static_cast<int>(hs.amg.levels.size());
  *levels = L + 1;
  for (int l = 0; l <= L && l < 16; ++l) {
    const Csr& A = l < L ? hs.amg.levels[l].A : hs.amg.coarsest;
    rows[l] = A.n;
    nnz[l] = static_cast<std::int64_t>(A.nnz());
  }
}

}  // namespace hxb

using namespace hxb;

extern "C" {

const char* hxb_last_error(void) { return g_last_error.c_str(); }

void hxb_default_options(hxb_options* opt)
{
  std::memset(opt, 0, sizeof(*opt));
  opt->precond_mode = HXB_PRECOND_TWO_SCALE;
  opt->coarse_solve = HXB_COARSE_AUTOMATIC;
  opt->direct_threshold = 64000;
  opt->variant = HXB_VARIANT_STORED;
  opt->device = 0;
  opt->n_gpus = 1;
  for (int r = 0; r < HXB_MAX_GPUS; ++r) opt->devices[r] = r;
  opt->nranks = 1;
}

int hxb_generate_cube_mesh(int k, int family, int boundary_tag, hxb_mesh_buf** out)
{
  return guarded([&] {
    if (family < 0 || family > 2) throw HxbError(HXB_EINVAL, "unknown mesh family");
    if (boundary_tag < 0 || boundary_tag > 1) throw HxbError(HXB_EINVAL, "unknown boundary tag");
    *out = wrap_mesh(generate_cube_mesh(k, static_cast<MeshFamily>(family), static_cast<std::uint8_t>(boundary_tag)));
  });
}

int hxb_generate_box_mesh(int kx, int ky, int kz, const double size[3], int boundary_tag, hxb_mesh_buf** out)
{
  return guarded([&] {
    if (boundary_tag < 0 || boundary_tag > 1) throw HxbError(HXB_EINVAL, "unknown boundary tag");
    *out = wrap_mesh(generate_box_mesh(kx, ky, kz, {size[0], size[1], size[2]}, static_cast<std::uint8_t>(boundary_tag)));
  });
}

int hxb_refine_uniform(const hxb_mesh* in, hxb_mesh_buf** out)
{
  return guarded([&] { *out = wrap_mesh(refine_uniform(view_to_mesh(in))); });
}

int hxb_read_mesh_file(const char* path, int format, hxb_mesh_buf** out)
{
  return guarded([&] {
    if (!path || !out) throw HxbError(HXB_EINVAL, "null argument");
    switch (format) {
      case HXB_MESHFILE_AUTO: *out = wrap_mesh(read_mesh_file(path)); break;
      case HXB_MESHFILE_MSH: *out = wrap_mesh(read_msh(path)); break;
      case HXB_MESHFILE_NATIVE: *out = wrap_mesh(read_native(path)); break;
      default: throw HxbError(HXB_EINVAL, "unknown mesh file format");
    }
  });
}

int hxb_write_mesh_file(const hxb_mesh* mesh, const char* path, int format)
{
  return guarded([&] {
    if (!path) throw HxbError(HXB_EINVAL, "null argument");
    const HexMesh m = view_to_mesh(mesh);
    switch (format) {
      case HXB_MESHFILE_AUTO: write_mesh_file(m, path); break;
      case HXB_MESHFILE_MSH: write_msh(m, path); break;
      case HXB_MESHFILE_NATIVE: write_native(m, path); break;
      default: throw HxbError(HXB_EINVAL, "unknown mesh file format");
    }
  });
}

void hxb_mesh_free(hxb_mesh_buf* m)
{
  if (!m) return;
  delete static_cast<MeshHolder*>(m->impl);
  delete m;
}

int hxb_setup_create(const hxb_mesh* mesh, int order, const double* kappa_e, const double* c_e, const hxb_options* opt,
                     hxb_setup** out)
{
  return guarded([&] {
    if (!out || !kappa_e || !c_e) throw HxbError(HXB_EINVAL, "null argument");
    hxb_options o;
    if (opt)
      o = *opt;
    else
      hxb_default_options(&o);
    auto hs = std::make_unique<HostSetup>();
    hs->mesh = view_to_mesh(mesh);
    const int ne = hs->mesh.num_elements();
    hs->kappa.assign(kappa_e, kappa_e + ne);
    hs->c.assign(c_e, c_e + ne);
    SetupOptions so;
    so.precond_mode = o.precond_mode;
    so.coarse_solve = o.coarse_solve;
    so.direct_threshold = o.direct_threshold;
    build_host_setup(*hs, order, so);
    *out = reinterpret_cast<hxb_setup*>(hs.release());
  });
}

void hxb_setup_destroy(hxb_setup* s) { delete reinterpret_cast<HostSetup*>(s); }

int hxb_setup_info(const hxb_setup* s, hxb_plan_info* info)
{
  return guarded([&] {
    const HostSetup* hs = reinterpret_cast<const HostSetup*>(s);
    if (!hs || !info) throw HxbError(HXB_EINVAL, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->num_global = hs->num.num_global;
    info->num_elements = hs->mesh.num_elements();
    info->num_vertices = hs->mesh.num_vertices();
    info->order = hs->order;
    info->coarse_uses_amg = hs->use_amg ? 1 : 0;
    info->coarse_n = hs->Kc.n;
    fill_amg_info(*hs, &info->amg_levels, info->amg_rows, info->amg_nnz);
  });
}

int hxb_setup_export_maps(const hxb_setup* s, int32_t* l2g, int64_t* g2l_offsets, int32_t* g2l_elem,
                          int32_t* g2l_local, int32_t* sub_l2g, uint8_t* dirichlet_mask)
{
  return guarded([&] {
    if (!s) throw HxbError(HXB_EINVAL, "null setup");
    export_index_maps(*reinterpret_cast<const HostSetup*>(s), l2g, g2l_offsets, g2l_elem, g2l_local, sub_l2g,
                      dirichlet_mask);
  });
}

int hxb_setup_amg_level(const hxb_setup* s, int level, int64_t* rows, int64_t* nnz, int64_t* ptr, int32_t* col,
                        double* val, int32_t* aggregate)
{
  return guarded([&] {
    if (!s) throw HxbError(HXB_EINVAL, "null setup");
    export_amg_level(*reinterpret_cast<const HostSetup*>(s), level, rows, nnz, ptr, col, val, aggregate);
  });
}

int hxb_setup_lumped_mass(const hxb_setup* s, double* m)
{
  return guarded([&] {
    const HostSetup* hs = reinterpret_cast<const HostSetup*>(s);
    if (!hs) throw HxbError(HXB_EINVAL, "null setup");
    std::memcpy(m, hs->lumped.data(), hs->lumped.size() * sizeof(double));
  });
}

int hxb_setup_export_geometry(const hxb_setup* s, double* mass, double* wg)
{
  return guarded([&] {
    const HostSetup* hs = reinterpret_cast<const HostSetup*>(s);
    if (!hs) throw HxbError(HXB_EINVAL, "null setup");
    if (mass) std::memcpy(mass, hs->geo.mass.data(), hs->geo.mass.size() * sizeof(double));
    if (wg) std::memcpy(wg, hs->geo.wg.data(), hs->geo.wg.size() * sizeof(double));
  });
}

int hxb_gll(int order, double* nodes, double* weights, double* deriv)
{
  return guarded([&] {
    const GllBasis b = make_gll_basis(order);
    std::memcpy(nodes, b.nodes.data(), b.nodes.size() * sizeof(double));
    std::memcpy(weights, b.weights.data(), b.weights.size() * sizeof(double));
    std::memcpy(deriv, b.deriv.data(), b.deriv.size() * sizeof(double));
  });
}

int hxb_pencil(int order, double* K, double* M, double* V, double* V_inv, double* lambda)
{
  return guarded([&] {
    const Pencil p = build_pencil(make_gll_basis(order));
    std::memcpy(K, p.K.data(), p.K.size() * sizeof(double));
    std::memcpy(M, p.M.data(), p.M.size() * sizeof(double));
    std::memcpy(V, p.V.data(), p.V.size() * sizeof(double));
    std::memcpy(V_inv, p.V_inv.data(), p.V_inv.size() * sizeof(double));
    std::memcpy(lambda, p.lambda.data(), p.lambda.size() * sizeof(double));
  });
}

uint64_t hxb_words_model(int64_t ne, int order, int variant)
{
  const uint64_t np = order + 1;
  return static_cast<uint64_t>(ne) * ((variant == HXB_VARIANT_STORED ? 10 : 3) * np * np * np + np * np + 2);
}
uint64_t hxb_flops_model(int64_t ne, int order)
{
  const uint64_t np = order + 1;
  return static_cast<uint64_t>(ne) * (12 * np * np * np * np + 18 * np * np * np);
}
uint64_t hxb_fine_ops_model(int64_t ne, int order)
{
  const uint64_t p = order + 3;
  return static_cast<uint64_t>(ne) * (6 * p * p * p * p + 15 * p * p * p);
}
uint64_t hxb_fine_words_model(int64_t ne, int order)
{
  const uint64_t p = order + 3;
  return static_cast<uint64_t>(ne) * (3 * p * p * p + 4 * p * p);
}


// Partition lists of rank `rank` of `nranks` (GPU-free; same code as the plan's).
// counts[6] = e0, e1, n_group0, n_up, n_down, total local surface nodes;
// nodes (may be NULL) receives the local node ids [group0 | up | down].
int hxb_setup_dist_lists(const hxb_setup* setup, int rank, int nranks, int64_t* counts, int32_t* nodes)
{
  return guarded([&] {
    if (!setup || !counts) throw HxbError(HXB_EINVAL, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw HxbError(HXB_EINVAL, "rank out of range");
    const HostSetup& hs = *reinterpret_cast<const HostSetup*>(setup);
    const int nsurfp = (surface_slot_count(hs.order + 1) + 3) & ~3;
    DistLists d = dist_partition(hs, rank, nranks, nsurfp);
    const int64_t v[6] = {d.e0, d.e1, d.n_grp0, d.n_up, d.n_down, static_cast<int64_t>(d.nodes.size())};
    std::memcpy(counts, v, sizeof(v));
    if (nodes) std::memcpy(nodes, d.nodes.data(), d.nodes.size() * sizeof(int32_t));
  });
}

// GPU-free check of the sparse direct coarse factor (setup_nd.cpp) on the
// setup's coupled coarse block: relative residual |A x - b| / |b| of a
// factor solve with b = 1, factor entries, separator-tree levels.
int hxb_setup_coarse_direct_check(const hxb_setup* setup, double* rel_residual, int64_t* factor_entries,
                                  int32_t* levels)
{
  return guarded([&] {
    const HostSetup& hs = *reinterpret_cast<const HostSetup*>(setup);
    if (!hs.do_coarse) throw HxbError(HXB_EINVAL, "setup has no coarse preconditioner");
    const Csr& K = hs.Kc;
    std::vector<int> pos(K.n, -1), coupled;
    for (int i = 0; i < K.n; ++i)
      for (std::int64_t q = K.ptr[i]; q < K.ptr[i + 1]; ++q)
        if (K.col[q] != i) {
          pos[i] = static_cast<int>(coupled.size());
          coupled.push_back(i);
          break;
        }
    Csr B;
    B.n = static_cast<gid>(coupled.size());
    B.ptr.assign(1, 0);
    for (int i : coupled) {
      for (std::int64_t q = K.ptr[i]; q < K.ptr[i + 1]; ++q) {
        B.col.push_back(pos[K.col[q]]);
        B.val.push_back(K.val[q]);
      }
      B.ptr.push_back(static_cast<std::int64_t>(B.col.size()));
    }
    std::vector<std::array<double, 3>> xyz(B.n);
    for (int q = 0; q < B.n; ++q) xyz[q] = hs.mesh.vertices[coupled[q]];
    const NdFactor F = nd_cholesky(B, xyz);
    std::vector<double> b(B.n, 1.0);
    const std::vector<double> x = nd_solve_host(F, b);
    double rn = 0, bn = 0;
    for (int i = 0; i < B.n; ++i) {
      double ax = 0;
      for (std::int64_t q = B.ptr[i]; q < B.ptr[i + 1]; ++q) ax += B.val[q] * x[B.col[q]];
      rn += (ax - b[i]) * (ax - b[i]);
      bn += b[i] * b[i];
    }
    if (rel_residual) *rel_residual = std::sqrt(rn / bn);
    std::int64_t e = 0;
    for (const NdSupernode& S : F.sn) e += static_cast<std::int64_t>(S.linv.size() + S.l21.size());
    if (factor_entries) *factor_entries = e;
    if (levels) *levels = F.levels;
  });
}

}  // extern "C"
