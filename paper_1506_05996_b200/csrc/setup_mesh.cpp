// Mesh generators, GLL basis and element geometry (host, native C++).
//
// These reproduce the reference's inputs bit-for-bit (same formulas in the
// same operation order) so the plan sees the identical mesh and factors:
//   generate_box_mesh / generate_cube_mesh / refine_uniform   mesh.cpp:67-234
//   legendre / gll_nodes_weights / derivation_matrix / coarse_vandermonde  gll.cpp:13-114
//   jacobian / element_dimensions / compute_factors            geometry.cpp:26-161
//   kappa*m*Gt premultiplied planes                            operator.cpp:77-89
#include <algorithm>
#include <cmath>
#include <span>
#include <unordered_map>

#include "setup.hpp"

namespace hxb {

namespace {

std::array<std::array<int, 4>, 6> make_face_corner_table()
{
  std::array<std::array<int, 4>, 6> t{};
  for (int f = 0; f < 6; ++f) {
    const int a = f / 2, s = f % 2;
    int idx = 0;
    for (int v = 0; v < 2; ++v)
      for (int u = 0; u < 2; ++u) {
        int bits[3];
        bits[a] = s;
        bits[(a + 1) % 3] = u;
        bits[(a + 2) % 3] = v;
        t[f][idx++] = hex_corner(bits[0], bits[1], bits[2]);
      }
  }
  return t;
}
const std::array<std::array<int, 4>, 6> kFaceCorners = make_face_corner_table();

std::uint64_t splitmix64(std::uint64_t& state)
{
  state += 0x9E3779B97F4A7C15ull;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double unit_double(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

struct KeyHash {
  template <std::size_t N>
  std::size_t operator()(const std::array<gid, N>& k) const
  {
    std::uint64_t h = 1469598103934665603ull;
    for (gid x : k) h = (h ^ static_cast<std::uint32_t>(x)) * 1099511628211ull;
    return static_cast<std::size_t>(h);
  }
};

}  // namespace

const std::array<int, 4>& face_corners(int face) { return kFaceCorners[face]; }

HexMesh generate_box_mesh(int kx, int ky, int kz, std::array<double, 3> size, std::uint8_t tag)
{
  if (kx < 1 || ky < 1 || kz < 1) throw HxbError(1, "box mesh needs k >= 1 per axis");
  HexMesh mesh;
  const int nvx = kx + 1, nvy = ky + 1, nvz = kz + 1;
  mesh.vertices.reserve(static_cast<std::size_t>(nvx) * nvy * nvz);
  for (int iz = 0; iz < nvz; ++iz)
    for (int iy = 0; iy < nvy; ++iy)
      for (int ix = 0; ix < nvx; ++ix)
        mesh.vertices.push_back({size[0] * ix / kx, size[1] * iy / ky, size[2] * iz / kz});
  auto vid = [&](int ix, int iy, int iz) {
    return static_cast<gid>((static_cast<std::size_t>(iz) * nvy + iy) * nvx + ix);
  };
  mesh.elements.reserve(static_cast<std::size_t>(kx) * ky * kz);
  for (int ez = 0; ez < kz; ++ez)
    for (int ey = 0; ey < ky; ++ey)
      for (int ex = 0; ex < kx; ++ex) {
        std::array<gid, 8> conn{};
        for (int c = 0; c < 8; ++c) {
          const int bi = c & 1, bj = (c >> 1) & 1, bk = (c >> 2) & 1;
          conn[hex_corner(bi, bj, bk)] = vid(ex + bi, ey + bj, ez + bk);
        }
        mesh.elements.push_back(conn);
      }
  for (int ez = 0; ez < kz; ++ez)
    for (int ey = 0; ey < ky; ++ey)
      for (int ex = 0; ex < kx; ++ex) {
        const gid e = static_cast<gid>((static_cast<std::size_t>(ez) * ky + ey) * kx + ex);
        if (ex == 0) mesh.boundary_faces.push_back({e, 0, tag});
        if (ex == kx - 1) mesh.boundary_faces.push_back({e, 1, tag});
        if (ey == 0) mesh.boundary_faces.push_back({e, 2, tag});
        if (ey == ky - 1) mesh.boundary_faces.push_back({e, 3, tag});
        if (ez == 0) mesh.boundary_faces.push_back({e, 4, tag});
        if (ez == kz - 1) mesh.boundary_faces.push_back({e, 5, tag});
      }
  return mesh;
}

HexMesh generate_cube_mesh(int k, MeshFamily family, std::uint8_t tag)
{
  HexMesh mesh = generate_box_mesh(k, k, k, {1.0, 1.0, 1.0}, tag);
  if (family == MeshFamily::distorted_domain) {
    const double a = 0.1;
    for (auto& v : mesh.vertices) {
      const double x = v[0], y = v[1], z = v[2];
      v[0] = x + a * std::sin(double(M_PI) * y);
      v[1] = y + a * std::sin(double(M_PI) * z);
      v[2] = z + a * std::sin(double(M_PI) * x);
    }
  } else if (family == MeshFamily::distorted_elements) {
    const double h = 1.0 / k;
    const int nv = k + 1;
    for (int iz = 1; iz < k; ++iz)
      for (int iy = 1; iy < k; ++iy)
        for (int ix = 1; ix < k; ++ix) {
          std::uint64_t state = 0x5DEECE66Dull ^ ((static_cast<std::uint64_t>(ix) << 42) |
                                                  (static_cast<std::uint64_t>(iy) << 21) |
                                                  static_cast<std::uint64_t>(iz));
          auto& v = mesh.vertices[(static_cast<std::size_t>(iz) * nv + iy) * nv + ix];
          for (int d = 0; d < 3; ++d) {
            const double u = unit_double(splitmix64(state));
            v[d] += (u - 0.5) * 0.5 * h;
          }
        }
  }
  check_jacobians(mesh);
  return mesh;
}

HexMesh refine_uniform(const HexMesh& mesh)
{
  HexMesh fine;
  fine.vertices = mesh.vertices;
  std::unordered_map<std::array<gid, 2>, gid, KeyHash> edge_mid;
  std::unordered_map<std::array<gid, 4>, gid, KeyHash> face_mid;
  edge_mid.reserve(mesh.elements.size() * 4);
  face_mid.reserve(mesh.elements.size() * 4);

  auto midpoint = [&](std::span<const gid> vs) {
    std::array<double, 3> p{0, 0, 0};
    for (gid v : vs)
      for (int d = 0; d < 3; ++d) p[d] += mesh.vertices[v][d];
    for (int d = 0; d < 3; ++d) p[d] /= static_cast<double>(vs.size());
    return p;
  };
  auto edge_vertex = [&](gid a, gid b) {
    std::array<gid, 2> key{std::min(a, b), std::max(a, b)};
    auto it = edge_mid.find(key);
    if (it != edge_mid.end()) return it->second;
    const gid id = fine.num_vertices();
    fine.vertices.push_back(midpoint(std::span<const gid>(key.data(), 2)));
    edge_mid.emplace(key, id);
    return id;
  };
  auto face_vertex = [&](std::array<gid, 4> vs) {
    std::sort(vs.begin(), vs.end());
    auto it = face_mid.find(vs);
    if (it != face_mid.end()) return it->second;
    const gid id = fine.num_vertices();
    fine.vertices.push_back(midpoint(std::span<const gid>(vs.data(), 4)));
    face_mid.emplace(vs, id);
    return id;
  };

  fine.elements.reserve(mesh.elements.size() * 8);
  for (gid e = 0; e < mesh.num_elements(); ++e) {
    const auto& conn = mesh.elements[e];
    gid lattice[3][3][3];
    for (int z = 0; z < 3; ++z)
      for (int y = 0; y < 3; ++y)
        for (int x = 0; x < 3; ++x) {
          const int odd = (x == 1) + (y == 1) + (z == 1);
          if (odd == 0) {
            lattice[x][y][z] = conn[hex_corner(x / 2, y / 2, z / 2)];
          } else if (odd == 1) {
            int lo[3] = {x / 2, y / 2, z / 2}, hi[3] = {x / 2, y / 2, z / 2};
            const int a = (x == 1) ? 0 : (y == 1) ? 1 : 2;
            lo[a] = 0;
            hi[a] = 1;
            lattice[x][y][z] = edge_vertex(conn[hex_corner(lo[0], lo[1], lo[2])],
                                           conn[hex_corner(hi[0], hi[1], hi[2])]);
          } else if (odd == 2) {
            const int a = (x != 1) ? 0 : (y != 1) ? 1 : 2;
            std::array<gid, 4> vs{};
            int idx = 0;
            for (int v = 0; v < 2; ++v)
              for (int u = 0; u < 2; ++u) {
                int bits[3];
                bits[a] = (a == 0 ? x : a == 1 ? y : z) / 2;
                bits[(a + 1) % 3] = u;
                bits[(a + 2) % 3] = v;
                vs[idx++] = conn[hex_corner(bits[0], bits[1], bits[2])];
              }
            lattice[x][y][z] = face_vertex(vs);
          } else {
            const gid id = fine.num_vertices();
            fine.vertices.push_back(midpoint(std::span<const gid>(conn.data(), 8)));
            lattice[x][y][z] = id;
          }
        }
    for (int oc = 0; oc < 8; ++oc) {
      const int ox = oc & 1, oy = (oc >> 1) & 1, oz = (oc >> 2) & 1;
      std::array<gid, 8> child{};
      for (int c = 0; c < 8; ++c) {
        const int bi = c & 1, bj = (c >> 1) & 1, bk = (c >> 2) & 1;
        child[hex_corner(bi, bj, bk)] = lattice[ox + bi][oy + bj][oz + bk];
      }
      fine.elements.push_back(child);
    }
  }
  for (const auto& bf : mesh.boundary_faces) {
    const int a = bf.face / 2, s = bf.face % 2;
    for (int oc = 0; oc < 8; ++oc) {
      const int bits[3] = {oc & 1, (oc >> 1) & 1, (oc >> 2) & 1};
      if (bits[a] == s) fine.boundary_faces.push_back({bf.element * 8 + oc, bf.face, bf.tag});
    }
  }
  check_jacobians(fine);
  return fine;
}

// ---------------------------------------------------------------------------
// GLL basis — gll.cpp:13-114

namespace {
std::pair<double, double> legendre(int n, double t)
{
  double pm1 = 1.0, p = t;
  if (n == 0) return {1.0, 0.0};
  for (int k = 2; k <= n; ++k) {
    const double pk = ((2.0 * k - 1.0) * t * p - (k - 1.0) * pm1) / k;
    pm1 = p;
    p = pk;
  }
  double dp;
  if (std::abs(1.0 - t * t) < 1e-14)
    dp = 0.5 * n * (n + 1.0) * (t > 0 ? 1.0 : ((n % 2 == 0) ? -1.0 : 1.0));
  else
    dp = n * (pm1 - t * p) / (1.0 - t * t);
  return {p, dp};
}
}  // namespace

GllBasis make_gll_basis(int n)
{
  if (n < 1) throw HxbError(1, "gll order must be >= 1, got " + std::to_string(n));
  GllBasis b;
  b.order = n;
  const int np = n + 1;
  std::vector<double> t(np, 0.0);
  t[0] = -1.0;
  t[n] = 1.0;
  for (int i = 1; i < n; ++i) {  // Newton on (1-t^2) P'_n from Chebyshev-Lobatto guesses
    double x = -std::cos(M_PI * i / n);
    for (int it = 0; it < 100; ++it) {
      const auto [p, dp] = legendre(n, x);
      const double f = (1.0 - x * x) * dp;
      const double df = -static_cast<double>(n) * (n + 1.0) * p;
      const double dx = f / df;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    t[i] = x;
  }
  for (int i = 0; i <= n / 2; ++i) {  // exact symmetry
    const double s = 0.5 * (t[i] - t[n - i]);
    t[i] = s;
    t[n - i] = -s;
  }
  b.nodes.resize(np);
  b.weights.resize(np);
  for (int i = 0; i <= n; ++i) {
    const auto [p, dp] = legendre(n, t[i]);
    (void)dp;
    b.nodes[i] = t[i];
    b.weights[i] = 2.0 / (n * (n + 1.0) * p * p);
  }
  b.deriv.assign(static_cast<std::size_t>(np) * np, 0.0);
  std::vector<double> ln(np);
  for (int i = 0; i < np; ++i) ln[i] = legendre(n, b.nodes[i]).first;
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j)
      if (i != j) b.deriv[static_cast<std::size_t>(i) * np + j] = ln[j] / (ln[i] * (b.nodes[j] - b.nodes[i]));
  b.deriv[0] = -0.25 * n * (n + 1.0);
  b.deriv[static_cast<std::size_t>(np) * np - 1] = 0.25 * n * (n + 1.0);
  const std::size_t nloc = static_cast<std::size_t>(np) * np * np;
  b.coarse_vandermonde.resize(8 * nloc);
  auto hat = [](int which, double tt) { return which == 0 ? 0.5 * (1 - tt) : 0.5 * (1 + tt); };
  for (int corner = 0; corner < 8; ++corner) {
    const int ci = corner & 1, cj = (corner >> 1) & 1, ck = (corner >> 2) & 1;
    std::size_t node = 0;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++node)
          b.coarse_vandermonde[corner * nloc + node] =
              hat(ci, b.nodes[i]) * hat(cj, b.nodes[j]) * hat(ck, b.nodes[k]);
  }
  return b;
}

// ---------------------------------------------------------------------------
// Geometry — geometry.cpp:26-161

namespace {
inline void corner_coords(const HexMesh& mesh, gid e, double xyz[8][3])
{
  for (int c = 0; c < 8; ++c) {
    const auto& v = mesh.vertices[mesh.elements[e][c]];
    xyz[c][0] = v[0];
    xyz[c][1] = v[1];
    xyz[c][2] = v[2];
  }
}
}  // namespace

std::array<double, 3> trilinear_map(const HexMesh& mesh, gid e, double xi, double eta, double zeta)
{
  double xyz[8][3];
  corner_coords(mesh, e, xyz);
  const double hx[2] = {0.5 * (1 - xi), 0.5 * (1 + xi)};
  const double hy[2] = {0.5 * (1 - eta), 0.5 * (1 + eta)};
  const double hz[2] = {0.5 * (1 - zeta), 0.5 * (1 + zeta)};
  std::array<double, 3> p{0, 0, 0};
  for (int bk = 0; bk < 2; ++bk)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) {
        const double w = hx[bi] * hy[bj] * hz[bk];
        const int c = hex_corner(bi, bj, bk);
        for (int d = 0; d < 3; ++d) p[d] += w * xyz[c][d];
      }
  return p;
}

Jacobian jacobian(const HexMesh& mesh, gid e, double xi, double eta, double zeta)
{
  double xyz[8][3];
  corner_coords(mesh, e, xyz);
  const double h[3][2] = {{0.5 * (1 - xi), 0.5 * (1 + xi)},
                          {0.5 * (1 - eta), 0.5 * (1 + eta)},
                          {0.5 * (1 - zeta), 0.5 * (1 + zeta)}};
  constexpr double dh[2] = {-0.5, 0.5};
  Jacobian out{};
  for (int bk = 0; bk < 2; ++bk)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) {
        const int c = hex_corner(bi, bj, bk);
        const double wx = dh[bi] * h[1][bj] * h[2][bk];
        const double wy = h[0][bi] * dh[bj] * h[2][bk];
        const double wz = h[0][bi] * h[1][bj] * dh[bk];
        for (int d = 0; d < 3; ++d) {
          out.j[d * 3 + 0] += wx * xyz[c][d];
          out.j[d * 3 + 1] += wy * xyz[c][d];
          out.j[d * 3 + 2] += wz * xyz[c][d];
        }
      }
  const double* j = out.j;
  out.det = j[0] * (j[4] * j[8] - j[5] * j[7]) - j[1] * (j[3] * j[8] - j[5] * j[6]) +
            j[2] * (j[3] * j[7] - j[4] * j[6]);
  if (!(out.det > 0))
    throw HxbError(2, "inverted element " + std::to_string(e) +
                          ": non-positive Jacobian determinant " + std::to_string(out.det));
  return out;
}

std::array<double, 3> element_dimensions(const HexMesh& mesh, gid e)
{
  double xyz[8][3];
  corner_coords(mesh, e, xyz);
  auto edge_len = [&](int ca, int cb) {
    double s = 0;
    for (int d = 0; d < 3; ++d) {
      const double t = xyz[cb][d] - xyz[ca][d];
      s += t * t;
    }
    return std::sqrt(s);
  };
  std::array<double, 3> h{0, 0, 0};
  for (int a = 0; a < 3; ++a) {
    double sum = 0;
    for (int v = 0; v < 2; ++v)
      for (int u = 0; u < 2; ++u) {
        int lo[3], hi[3];
        lo[a] = 0;
        hi[a] = 1;
        lo[(a + 1) % 3] = hi[(a + 1) % 3] = u;
        lo[(a + 2) % 3] = hi[(a + 2) % 3] = v;
        sum += edge_len(hex_corner(lo[0], lo[1], lo[2]), hex_corner(hi[0], hi[1], hi[2]));
      }
    h[a] = 0.25 * sum;
  }
  return h;
}

void check_jacobians(const HexMesh& mesh)
{
  for (gid e = 0; e < mesh.num_elements(); ++e)
    for (int k = -1; k <= 1; ++k)
      for (int j = -1; j <= 1; ++j)
        for (int i = -1; i <= 1; ++i)
          (void)jacobian(mesh, e, static_cast<double>(i), static_cast<double>(j), static_cast<double>(k));
}

std::vector<double> element_dimensions_all(const HexMesh& mesh)
{
  std::vector<double> h(static_cast<std::size_t>(mesh.num_elements()) * 3);
  for (gid e = 0; e < mesh.num_elements(); ++e) {
    const auto hh = element_dimensions(mesh, e);
    for (int d = 0; d < 3; ++d) h[3 * static_cast<std::size_t>(e) + d] = hh[d];
  }
  return h;
}

Geometry compute_geometry(const HexMesh& mesh, const GllBasis& basis, const std::vector<double>& kappa,
                          bool store_planes)
{
  const int np = basis.npts();
  const gid ne = mesh.num_elements();
  const std::size_t nloc = static_cast<std::size_t>(np) * np * np;
  const std::size_t total = static_cast<std::size_t>(ne) * nloc;
  Geometry g;
  g.mass.resize(total);
  if (store_planes) g.wg.resize(6 * total);
  g.h.resize(static_cast<std::size_t>(ne) * 3);
  for (gid e = 0; e < ne; ++e) {
    const auto hh = element_dimensions(mesh, e);
    for (int d = 0; d < 3; ++d) g.h[3 * static_cast<std::size_t>(e) + d] = hh[d];
    std::size_t node = 0;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++node) {
          const Jacobian jac = jacobian(mesh, e, basis.nodes[i], basis.nodes[j], basis.nodes[k]);
          const double* J = jac.j;
          double inv[9];
          inv[0] = (J[4] * J[8] - J[5] * J[7]) / jac.det;
          inv[1] = (J[2] * J[7] - J[1] * J[8]) / jac.det;
          inv[2] = (J[1] * J[5] - J[2] * J[4]) / jac.det;
          inv[3] = (J[5] * J[6] - J[3] * J[8]) / jac.det;
          inv[4] = (J[0] * J[8] - J[2] * J[6]) / jac.det;
          inv[5] = (J[2] * J[3] - J[0] * J[5]) / jac.det;
          inv[6] = (J[3] * J[7] - J[4] * J[6]) / jac.det;
          inv[7] = (J[1] * J[6] - J[0] * J[7]) / jac.det;
          inv[8] = (J[0] * J[4] - J[1] * J[3]) / jac.det;
          auto gt = [&](int r, int c) {
            return inv[r * 3 + 0] * inv[c * 3 + 0] + inv[r * 3 + 1] * inv[c * 3 + 1] +
                   inv[r * 3 + 2] * inv[c * 3 + 2];
          };
          const std::size_t at = static_cast<std::size_t>(e) * nloc + node;
          const double m = basis.weights[i] * basis.weights[j] * basis.weights[k] * jac.det;
          g.mass[at] = m;
          if (store_planes) {
            const double scale = kappa[e] * m;  // operator.cpp:83-87: wg *= kappa_e * mass
            g.wg[0 * total + at] = gt(0, 0) * scale;
            g.wg[1 * total + at] = gt(0, 1) * scale;
            g.wg[2 * total + at] = gt(0, 2) * scale;
            g.wg[3 * total + at] = gt(1, 1) * scale;
            g.wg[4 * total + at] = gt(1, 2) * scale;
            g.wg[5 * total + at] = gt(2, 2) * scale;
          }
        }
  }
  return g;
}

}  // namespace hxb
