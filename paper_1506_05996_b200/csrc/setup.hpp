// Host-side setup for the B200 SEM-PCG plan (native C++, runs once per plan).
//
// Everything here re-derives, from the mesh alone, the data the reference
// builds in build_system (problem.cpp:73-108): the GLL basis (gll.cpp), the
// global numbering (mesh.cpp:287-453, reproduced bit-exactly by a closed-form
// entity ranking instead of the 72M-key sort), geometric factors
// (geometry.cpp:105-151), the FDM pencil (fine.cpp:15-80), the Q1 coarse
// matrix (coarse.cpp:21-87) and the aggregation-AMG hierarchy (amg.cpp:53-186).
// The device layouts these feed are described in DESIGN.md §3.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace hxb {

using gid = std::int32_t;

// mesh.hpp:24-29 — local face ids 0/1 = xi -/+, 2/3 = eta -/+, 4/5 = zeta -/+.
struct BoundaryFace {
  gid element = 0;
  int face = 0;
  std::uint8_t tag = 0;  // 0 dirichlet, 1 neumann (BoundaryTag)
};

// mesh.hpp:33 — Gmsh/VTK corner order from (xi,eta,zeta) bits.
inline constexpr int kHexCornerFromBits[8] = {0, 1, 3, 2, 4, 5, 7, 6};
inline int hex_corner(int bi, int bj, int bk) { return kHexCornerFromBits[bi + 2 * bj + 4 * bk]; }

struct HexMesh {  // mesh.hpp:38-45
  std::vector<std::array<double, 3>> vertices;
  std::vector<std::array<gid, 8>> elements;
  std::vector<BoundaryFace> boundary_faces;
  gid num_vertices() const { return static_cast<gid>(vertices.size()); }
  gid num_elements() const { return static_cast<gid>(elements.size()); }
};

enum class MeshFamily { uniform = 0, distorted_domain = 1, distorted_elements = 2 };

HexMesh generate_box_mesh(int kx, int ky, int kz, std::array<double, 3> size, std::uint8_t tag);
HexMesh generate_cube_mesh(int k, MeshFamily family, std::uint8_t tag);
HexMesh refine_uniform(const HexMesh& mesh);
const std::array<int, 4>& face_corners(int face);
void check_jacobians(const HexMesh& mesh);
// mesh_io.hpp:14-31 (setup_mesh_io.cpp)
HexMesh read_msh(const std::string& path);
void write_msh(const HexMesh& mesh, const std::string& path);
HexMesh read_native(const std::string& path);
void write_native(const HexMesh& mesh, const std::string& path);
HexMesh read_mesh_file(const std::string& path);
void write_mesh_file(const HexMesh& mesh, const std::string& path);

struct GllBasis {  // gll.hpp:17-31
  int order = 0;
  std::vector<double> nodes, weights, deriv, coarse_vandermonde;
  int npts() const { return order + 1; }
  double d(int i, int j) const { return deriv[static_cast<std::size_t>(i) * npts() + j]; }
};
GllBasis make_gll_basis(int order);

struct Jacobian {
  double j[9];
  double det;
};
// geometry.cpp:44-74 (same operation order); throws on det <= 0.
Jacobian jacobian(const HexMesh& mesh, gid e, double xi, double eta, double zeta);
std::array<double, 3> element_dimensions(const HexMesh& mesh, gid e);  // geometry.cpp:76-103
std::array<double, 3> trilinear_map(const HexMesh& mesh, gid e, double xi, double eta, double zeta);

// ---------------------------------------------------------------------------
// Numbering. Global ids follow the reference NodeKey order exactly:
// [referenced vertices | edge-interior | face-interior | element-interior].
// Element-surface local nodes therefore map below num_surface_global and
// element-interior local nodes are the contiguous block above it.
struct Numbering {
  int order = 0;
  gid num_global = 0;
  gid num_vertex_nodes = 0;    // NVu
  gid num_edges = 0;           // unique edges
  gid num_faces = 0;           // unique faces
  gid num_surface_global = 0;  // NVu + NEd(n-1) + NF(n-1)^2
  std::vector<gid> vertex_rank;  // vertex id -> global id (or -1 if unreferenced)
  // per element: global ids of its element-surface local nodes in ascending
  // local index order (the "surface slots"), NE * nsurf
  std::vector<gid> l2g_surf;
  std::vector<std::uint8_t> dirichlet_mask;  // per global node
  // face adjacency: for element e and face f, neighbor element (or -1) and its face
  std::vector<gid> face_nbr_elem;  // NE*6
  std::vector<std::int8_t> face_nbr_face;
  // per element and face: global ids of the neighbor's first interior layer
  // for the (n+1)^2 face slots (u fastest, mesh.cpp:419-450), or -1
  std::vector<gid> sub_face;  // NE*6*np^2
};

int surface_slot_count(int np);                // np^3 - (np-2)^3
int surface_slot_of(int np, int i, int j, int k);  // -1 for element-interior nodes
Numbering build_numbering(const HexMesh& mesh, int order);
// Full l2g for element e into out[nloc] (reference layout, mesh.hpp:73-74).
void element_l2g(const Numbering& num, int ne_total, gid e, gid* out);

// ---------------------------------------------------------------------------
struct Geometry {
  std::vector<double> mass;   // NE*nloc, rho_i rho_j rho_k det J
  std::vector<double> wg;     // 6 planes x NE*nloc : Gt_ab * (kappa_e * mass), operator.cpp:80-89
  std::vector<double> h;      // NE*3, element_dimensions
};
Geometry compute_geometry(const HexMesh& mesh, const GllBasis& basis, const std::vector<double>& kappa,
                          bool store_planes);
std::vector<double> element_dimensions_all(const HexMesh& mesh);  // NE*3

struct Pencil {  // fine.hpp:18-26
  int p = 0;
  std::vector<double> K, M, V, V_inv, lambda;
};
Pencil build_pencil(const GllBasis& basis);

// ---------------------------------------------------------------------------
struct Csr {  // amg.hpp:14-22
  gid n = 0;
  std::vector<std::int64_t> ptr;
  std::vector<gid> col;
  std::vector<double> val;
  std::size_t nnz() const { return val.size(); }
};

struct Triplet {
  gid r, c;
  double v;
};
Csr csr_from_triplets(gid n, std::vector<Triplet> t);                 // amg.cpp:22-40
std::vector<std::uint8_t> coarse_dirichlet_mask(const HexMesh& mesh);  // coarse.cpp:11-19
Csr assemble_coarse_matrix(const HexMesh& mesh, const std::vector<double>& kappa,
                           const std::vector<double>& c, const std::vector<std::uint8_t>& vmask);

struct AmgLevel {
  Csr A;
  std::vector<double> inv_diag;
  std::vector<gid> aggregate;  // row -> next-level row
  gid n_coarse = 0;
};
struct AmgSetup {
  std::vector<AmgLevel> levels;
  Csr coarsest;
};
AmgSetup amg_setup(Csr fine);  // amg.cpp:151-186

// Dense SPD inverse of the coupled block of a matrix whose remaining rows are
// decoupled (diagonal only). Used for the AMG coarsest level and the direct
// coarse solve (the reference's SimplicialLLT, coarse.cpp:117-127, amg.cpp:176-194).
struct DenseCoarse {
  gid n = 0;
  std::vector<gid> coupled;        // row ids of the coupled block, ascending
  std::vector<double> inv_diag;    // 1/a_ii for decoupled rows (0 for coupled)
  std::vector<double> ainv;        // coupled x coupled inverse, row-major (host-computed if small)
  std::vector<double> coupled_a;   // coupled block (dense, row-major), small blocks only
  // large blocks: the coupled block as CSR (coupled numbering) for the device factorization
  std::vector<std::int64_t> csr_ptr;
  std::vector<gid> csr_col;
  std::vector<double> csr_val;
};
DenseCoarse dense_coarse_setup(const Csr& A, int host_inverse_limit);
// Profile Cholesky of an SPD matrix after reverse Cuthill-McKee (SimplicialLLT
// as built for the reference here, coarse.cpp:117-127): row i of L holds
// columns [first[i], i] at env[start[i] ..]; P A P^T = L L^T with row i of the
// permuted matrix = row perm[i] of A.
struct EnvelopeFactor {
  gid n = 0;
  std::vector<std::int64_t> perm, first, start;
  std::vector<double> env;
};
EnvelopeFactor envelope_cholesky(const Csr& A);

// Nested-dissection supernodal Cholesky (setup_nd.cpp) of an SPD matrix whose
// rows carry vertex coordinates: P A P^T = L L^T, supernodes in postorder,
// supernode s owning permuted columns [c0, c1) and below-diagonal rows `rows`
// (permuted ids, ascending); linv = L11^-1 (m x m), l21 (r x m), row-major.
struct NdSupernode {
  std::vector<int> verts;     // original row ids (the separator or leaf)
  std::vector<int> children;
  int parent = -1, level = 0, c0 = 0, c1 = 0;
  std::vector<int> rows;
  std::vector<double> linv, l21;
};
struct NdFactor {
  int n = 0, levels = 0;
  std::vector<int> perm;      // permuted index -> original row
  std::vector<NdSupernode> sn;
};
NdFactor nd_cholesky(const Csr& A, const std::vector<std::array<double, 3>>& xyz);
std::vector<double> nd_solve_host(const NdFactor& F, const std::vector<double>& b);

// Setup phase timer: HXB_SETUP_TIMING=1 prints each phase's wall time to stderr.
void setup_phase(const char* name);  // closes the running phase, opens `name` (nullptr: close and print)

struct HxbError : std::runtime_error {
  int code;
  HxbError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

}  // namespace hxb

namespace hxb {

// Everything the plan needs, computed on the host from the mesh alone
// (build_system, problem.cpp:73-108, minus the GPU upload). Separate from the
// device plan so the bit-exact parts (numbering, aggregation) are testable
// without a GPU.
struct HostSetup;
struct SetupOptions {
  int precond_mode = 0;         // PrecondMode
  int coarse_solve = 0;         // CoarseSolve
  gid direct_threshold = 64000; // coarse.hpp:36
  bool store_planes = true;     // false for the on-the-fly operator variant (no kappa*m*Gt planes)
  // when set, replaces the host per-node geometry: must fill hs.geo.mass (all
  // elements); hs.geo.h is computed on the host either way (device plans)
  std::function<void(HostSetup&)> geometry_hook;
  bool device_lumped = false;  // the plan assembles the lumped mass on the device (hs.lumped filled later)
};

struct HostSetup {
  HexMesh mesh;
  int order = 0;
  std::vector<double> kappa, c;
  GllBasis basis;
  Geometry geo;
  Numbering num;
  std::vector<double> lumped;     // m_N (operator.cpp:90-91)
  Pencil pencil;
  bool do_fine = false, do_coarse = false, use_amg = false;
  std::vector<std::uint8_t> vmask;
  Csr Kc;
  AmgSetup amg;
};

void build_host_setup(HostSetup& hs, int order, const SetupOptions& opt);  // hs.mesh, kappa, c pre-filled

// Element-slab partition of the Ax assembly for rank `rank` of `nranks`
// (SURVEY §8e): owned elements [e0, e1); local surface nodes ordered
// [group 0 | up-interface | down-interface], each ascending global id;
// local Ax CSR (copies in (e,l) order) and the [e][2][nsurfp] surface map.
struct DistLists {
  int e0 = 0, e1 = 0;
  int n_grp0 = 0, n_up = 0, n_down = 0;
  std::vector<int> nodes;
  std::vector<unsigned> off;
  std::vector<int> idx;
  std::vector<int> smap;
};
DistLists dist_partition(const HostSetup& hs, int rank, int nranks, int nsurfp);

// The preconditioner side of the distributed solve (setup_dist.cpp):
//   finalised nodes = fin_surf (group 0 + down, local-list order) then the
//   owned interior range [ib0, ib1); fine CSR over them in (e, slot) order;
//   fine_pos[le][slot] >= 0 local sum position, -1 sentinel, <= -2 index
//   -2-q into this rank's send buffer [to down | to up]; frecv_* positions
//   for the neighbours' contributions in the order they send them;
//   ghost_from_* nodes whose r this rank receives, ghost_to_* it sends;
//   pr_* every copy (global e*nsurfp+slot, mass) of the finalised surface nodes.
struct DistPcgLists {
  int ib0 = 0, ib1 = 0;
  std::vector<int> fin_surf;
  std::vector<unsigned> fine_off;
  std::vector<int> fine_pos;
  int n_fsend_down = 0, n_fsend_up = 0;
  std::vector<int> frecv_down, frecv_up;
  std::vector<int> ghost_from_down, ghost_from_up, ghost_to_down, ghost_to_up;
  std::vector<unsigned> pr_off;
  std::vector<int> pr_idx;
  std::vector<double> pr_mass;
};
DistPcgLists dist_pcg_setup(const HostSetup& hs, const DistLists& d, int rank, int nranks);

// Physical coordinates of every global node, xyz[3g+d] (mesh.cpp:477-492).
std::vector<double> global_node_coords(const HostSetup& hs);
HexMesh mesh_from_arrays(int nv, const double* xyz, int ne, const std::int32_t* conn, int nbf,
                         const std::int32_t* be, const std::int32_t* bf, const std::uint8_t* bt);
// IndexMaps export in the reference layout (mesh.hpp:66-97); null pointers skipped.
void export_index_maps(const HostSetup& hs, std::int32_t* l2g, std::int64_t* g2l_offsets, std::int32_t* g2l_elem,
                       std::int32_t* g2l_local, std::int32_t* sub_l2g, std::uint8_t* mask);
// Visit every non-sentinel (n+3)^3 subdomain slot of element e in ascending
// slot order: fn(global id, slot index).
template <class F>
void for_each_sub_slot(const Numbering& num, int ne, gid e, gid* l2g_scratch, F&& fn)
{
  const int n = num.order, np = n + 1, P = n + 3;
  element_l2g(num, ne, e, l2g_scratch);
  const gid* sf = num.sub_face.data() + static_cast<std::size_t>(e) * 6 * np * np;
  for (int z = 0; z < P; ++z)
    for (int y = 0; y < P; ++y)
      for (int x = 0; x < P; ++x) {
        const int ii = x - 1, jj = y - 1, kk = z - 1;
        const bool ox = ii < 0 || ii > n, oy = jj < 0 || jj > n, oz = kk < 0 || kk > n;
        const int nout = ox + oy + oz;
        gid g = -1;
        if (nout == 0) {
          g = l2g_scratch[(kk * np + jj) * np + ii];
        } else if (nout == 1) {
          int f, u, w;
          if (ox) {
            f = ii < 0 ? 0 : 1;
            u = jj;
            w = kk;
          } else if (oy) {
            f = jj < 0 ? 2 : 3;
            u = kk;
            w = ii;
          } else {
            f = kk < 0 ? 4 : 5;
            u = ii;
            w = jj;
          }
          g = sf[(f * np + w) * np + u];
        }
        fn(g, (z * P + y) * P + x);
      }
}

}  // namespace hxb
