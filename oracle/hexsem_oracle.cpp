// oracle/hexsem_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// Plain C++ CPU restatement of the reference solver path (hexsem,
// /root/reference/proj) used as the parity checker for the B200 kernels.
// It is NOT the product: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg may load it (through oracle/ctypes_oracle.py).
//
// Written from the reference's behaviour, function by function; every block
// cites the reference file:line it restates. It is deliberately simple and
// sequential (no threads, no tricks): sort-based global numbering, dense or
// envelope Cholesky, cyclic-Jacobi eigen-solve. Floating-point operations are
// kept in the reference's order so that, compiled like the reference (no
// FMA), results agree to the last bit except where the reference calls Eigen
// (pencil eigenvectors and the coarse Cholesky: rounding-level differences).
//
// Pinning: tests/test_oracle.py checks this restatement against (a) the
// reference's own known answers (test_mesh.cpp / test_operator.cpp /
// test_fine.cpp / test_output.txt goldens) and (b) the compiled
// reference oracle/_ref/libhexsem_ref.so on the same inputs.
//
// C-ABI: identical to oracle/ref_driver.cpp with the prefix orc_.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace orc {

using i32 = std::int32_t;
using i64 = std::int64_t;
using Vec = std::vector<double>;

struct BadInput : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// ---------------------------------------------------------------------------
// Mesh (mesh.hpp:19-45). Corner c with bits (bi,bj,bk) sits at connectivity
// slot kSlot[bi+2bj+4bk] (Gmsh order, mesh.hpp:31-33).
constexpr int kSlot[8] = {0, 1, 3, 2, 4, 5, 7, 6};
inline int slot_of(int bi, int bj, int bk) { return kSlot[bi + 2 * bj + 4 * bk]; }

struct Face {
  i32 elem;
  int face;  // 0/1 = xi -/+, 2/3 = eta -/+, 4/5 = zeta -/+
  int tag;   // 0 dirichlet, 1 neumann
};

struct Mesh {
  std::vector<std::array<double, 3>> X;
  std::vector<std::array<i32, 8>> E;
  std::vector<Face> bfaces;
  i32 nv() const { return static_cast<i32>(X.size()); }
  i32 ne() const { return static_cast<i32>(E.size()); }
};

// 4 connectivity slots of face f: bits[axis]=side, (u,v) on the two other
// axes in cyclic order, v outer (mesh.cpp:22-38).
std::array<int, 4> face_slots(int f)
{
  const int a = f / 2, s = f % 2;
  std::array<int, 4> out{};
  int q = 0;
  for (int v = 0; v < 2; ++v)
    for (int u = 0; u < 2; ++u) {
      int b[3];
      b[a] = s;
      b[(a + 1) % 3] = u;
      b[(a + 2) % 3] = v;
      out[q++] = slot_of(b[0], b[1], b[2]);
    }
  return out;
}

// ---------------------------------------------------------------------------
// Trilinear geometry (geometry.cpp:26-74)
struct Jac {
  double j[9];
  double det;
};

Jac jacobian_at(const Mesh& m, i32 e, double xi, double eta, double zeta)
{
  double c[8][3];
  for (int q = 0; q < 8; ++q)
    for (int d = 0; d < 3; ++d) c[q][d] = m.X[m.E[e][q]][d];
  const double h0[2] = {0.5 * (1 - xi), 0.5 * (1 + xi)};
  const double h1[2] = {0.5 * (1 - eta), 0.5 * (1 + eta)};
  const double h2[2] = {0.5 * (1 - zeta), 0.5 * (1 + zeta)};
  const double dh[2] = {-0.5, 0.5};
  Jac J{};
  for (int bk = 0; bk < 2; ++bk)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) {
        const int q = slot_of(bi, bj, bk);
        const double wx = dh[bi] * h1[bj] * h2[bk];
        const double wy = h0[bi] * dh[bj] * h2[bk];
        const double wz = h0[bi] * h1[bj] * dh[bk];
        for (int d = 0; d < 3; ++d) {
          J.j[3 * d + 0] += wx * c[q][d];
          J.j[3 * d + 1] += wy * c[q][d];
          J.j[3 * d + 2] += wz * c[q][d];
        }
      }
  const double* a = J.j;
  J.det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
          a[2] * (a[3] * a[7] - a[4] * a[6]);
  if (!(J.det > 0)) throw std::runtime_error("inverted element " + std::to_string(e));
  return J;
}

// inverse via adjugate / det, row-major (geometry.cpp:127-135)
void inverse(const Jac& J, double inv[9])
{
  const double* a = J.j;
  inv[0] = (a[4] * a[8] - a[5] * a[7]) / J.det;
  inv[1] = (a[2] * a[7] - a[1] * a[8]) / J.det;
  inv[2] = (a[1] * a[5] - a[2] * a[4]) / J.det;
  inv[3] = (a[5] * a[6] - a[3] * a[8]) / J.det;
  inv[4] = (a[0] * a[8] - a[2] * a[6]) / J.det;
  inv[5] = (a[2] * a[3] - a[0] * a[5]) / J.det;
  inv[6] = (a[3] * a[7] - a[4] * a[6]) / J.det;
  inv[7] = (a[1] * a[6] - a[0] * a[7]) / J.det;
  inv[8] = (a[0] * a[4] - a[1] * a[3]) / J.det;
}

// check_jacobians: 3x3x3 lattice per element (geometry.cpp:153-161)
void screen(const Mesh& m)
{
  for (i32 e = 0; e < m.ne(); ++e)
    for (int k = -1; k <= 1; ++k)
      for (int j = -1; j <= 1; ++j)
        for (int i = -1; i <= 1; ++i) jacobian_at(m, e, i, j, k);
}

std::array<double, 3> map_point(const Mesh& m, i32 e, double xi, double eta, double zeta)
{  // trilinear_map (geometry.cpp:26-42)
  const double h0[2] = {0.5 * (1 - xi), 0.5 * (1 + xi)};
  const double h1[2] = {0.5 * (1 - eta), 0.5 * (1 + eta)};
  const double h2[2] = {0.5 * (1 - zeta), 0.5 * (1 + zeta)};
  std::array<double, 3> p{0, 0, 0};
  for (int bk = 0; bk < 2; ++bk)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) {
        const double w = h0[bi] * h1[bj] * h2[bk];
        const auto& v = m.X[m.E[e][slot_of(bi, bj, bk)]];
        for (int d = 0; d < 3; ++d) p[d] += w * v[d];
      }
  return p;
}

// element_dimensions: mean of the 4 edges along each axis (geometry.cpp:76-103)
std::array<double, 3> elem_h(const Mesh& m, i32 e)
{
  std::array<double, 3> h{};
  for (int a = 0; a < 3; ++a) {
    double sum = 0;
    for (int v = 0; v < 2; ++v)
      for (int u = 0; u < 2; ++u) {
        int lo[3], hi[3];
        lo[a] = 0;
        hi[a] = 1;
        lo[(a + 1) % 3] = hi[(a + 1) % 3] = u;
        lo[(a + 2) % 3] = hi[(a + 2) % 3] = v;
        const auto& A = m.X[m.E[e][slot_of(lo[0], lo[1], lo[2])]];
        const auto& B = m.X[m.E[e][slot_of(hi[0], hi[1], hi[2])]];
        double s = 0;
        for (int d = 0; d < 3; ++d) {
          const double t = B[d] - A[d];
          s += t * t;
        }
        sum += std::sqrt(s);
      }
    h[a] = 0.25 * sum;
  }
  return h;
}

// ---------------------------------------------------------------------------
// Mesh generators (mesh.cpp:67-139)
Mesh box(int kx, int ky, int kz, const double size[3], int tag)
{
  if (kx < 1 || ky < 1 || kz < 1) throw BadInput("box mesh needs k >= 1 per axis");
  Mesh m;
  const int nx = kx + 1, ny = ky + 1, nz = kz + 1;
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) m.X.push_back({size[0] * x / kx, size[1] * y / ky, size[2] * z / kz});
  for (int ez = 0; ez < kz; ++ez)
    for (int ey = 0; ey < ky; ++ey)
      for (int ex = 0; ex < kx; ++ex) {
        std::array<i32, 8> c{};
        for (int q = 0; q < 8; ++q) {
          const int bi = q & 1, bj = (q >> 1) & 1, bk = q >> 2;
          c[slot_of(bi, bj, bk)] = static_cast<i32>(((ez + bk) * ny + (ey + bj)) * nx + ex + bi);
        }
        m.E.push_back(c);
      }
  for (int ez = 0; ez < kz; ++ez)
    for (int ey = 0; ey < ky; ++ey)
      for (int ex = 0; ex < kx; ++ex) {
        const i32 e = (ez * ky + ey) * kx + ex;
        if (ex == 0) m.bfaces.push_back({e, 0, tag});
        if (ex == kx - 1) m.bfaces.push_back({e, 1, tag});
        if (ey == 0) m.bfaces.push_back({e, 2, tag});
        if (ey == ky - 1) m.bfaces.push_back({e, 3, tag});
        if (ez == 0) m.bfaces.push_back({e, 4, tag});
        if (ez == kz - 1) m.bfaces.push_back({e, 5, tag});
      }
  return m;
}

std::uint64_t mix64(std::uint64_t& s)
{  // splitmix64 (mesh.cpp:40-47)
  s += 0x9E3779B97F4A7C15ull;
  std::uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

Mesh cube(int k, int family, int tag)
{
  const double one[3] = {1, 1, 1};
  Mesh m = box(k, k, k, one, tag);
  if (family == 1) {  // distorted_domain (mesh.cpp:113-120)
    for (auto& v : m.X) {
      const double x = v[0], y = v[1], z = v[2];
      v[0] = x + 0.1 * std::sin(M_PI * y);
      v[1] = y + 0.1 * std::sin(M_PI * z);
      v[2] = z + 0.1 * std::sin(M_PI * x);
    }
  } else if (family == 2) {  // distorted_elements: interior vertices jittered (mesh.cpp:121-136)
    const double h = 1.0 / k;
    const int nv = k + 1;
    for (int z = 1; z < k; ++z)
      for (int y = 1; y < k; ++y)
        for (int x = 1; x < k; ++x) {
          std::uint64_t st = 0x5DEECE66Dull ^ ((static_cast<std::uint64_t>(x) << 42) |
                                               (static_cast<std::uint64_t>(y) << 21) | static_cast<std::uint64_t>(z));
          auto& v = m.X[(static_cast<std::size_t>(z) * nv + y) * nv + x];
          for (int d = 0; d < 3; ++d) {
            const double u = static_cast<double>(mix64(st) >> 11) * 0x1.0p-53;
            v[d] += (u - 0.5) * 0.5 * h;
          }
        }
  }
  screen(m);
  return m;
}

// refine_uniform: 8 children through the trilinear midpoints, new vertices
// deduplicated by entity (edge / face / centre) (mesh.cpp:141-234)
Mesh refine(const Mesh& in)
{
  Mesh out;
  out.X = in.X;
  std::map<std::pair<i32, i32>, i32> emid;
  std::map<std::array<i32, 4>, i32> fmid;
  auto centroid = [&](const i32* ids, int cnt) {
    std::array<double, 3> p{0, 0, 0};
    for (int q = 0; q < cnt; ++q)
      for (int d = 0; d < 3; ++d) p[d] += in.X[ids[q]][d];
    for (int d = 0; d < 3; ++d) p[d] /= static_cast<double>(cnt);
    return p;
  };
  for (i32 e = 0; e < in.ne(); ++e) {
    const auto& c = in.E[e];
    i32 L[3][3][3];
    for (int z = 0; z < 3; ++z)
      for (int y = 0; y < 3; ++y)
        for (int x = 0; x < 3; ++x) {
          const int odd = (x == 1) + (y == 1) + (z == 1);
          const int xyz[3] = {x, y, z};
          if (odd == 0) {
            L[x][y][z] = c[slot_of(x / 2, y / 2, z / 2)];
          } else if (odd == 1) {
            const int a = x == 1 ? 0 : (y == 1 ? 1 : 2);
            int lo[3] = {x / 2, y / 2, z / 2}, hi[3] = {x / 2, y / 2, z / 2};
            lo[a] = 0;
            hi[a] = 1;
            const i32 va = c[slot_of(lo[0], lo[1], lo[2])], vb = c[slot_of(hi[0], hi[1], hi[2])];
            const std::pair<i32, i32> key(std::min(va, vb), std::max(va, vb));
            auto it = emid.find(key);
            if (it == emid.end()) {
              const i32 ids[2] = {key.first, key.second};
              it = emid.emplace(key, out.nv()).first;
              out.X.push_back(centroid(ids, 2));
            }
            L[x][y][z] = it->second;
          } else if (odd == 2) {
            const int a = x != 1 ? 0 : (y != 1 ? 1 : 2);
            std::array<i32, 4> vs{};
            int q = 0;
            for (int v = 0; v < 2; ++v)
              for (int u = 0; u < 2; ++u) {
                int b[3];
                b[a] = xyz[a] / 2;
                b[(a + 1) % 3] = u;
                b[(a + 2) % 3] = v;
                vs[q++] = c[slot_of(b[0], b[1], b[2])];
              }
            std::sort(vs.begin(), vs.end());
            auto it = fmid.find(vs);
            if (it == fmid.end()) {
              it = fmid.emplace(vs, out.nv()).first;
              out.X.push_back(centroid(vs.data(), 4));
            }
            L[x][y][z] = it->second;
          } else {
            L[x][y][z] = out.nv();
            out.X.push_back(centroid(c.data(), 8));
          }
        }
    for (int oc = 0; oc < 8; ++oc) {
      const int ox = oc & 1, oy = (oc >> 1) & 1, oz = oc >> 2;
      std::array<i32, 8> ch{};
      for (int q = 0; q < 8; ++q) {
        const int bi = q & 1, bj = (q >> 1) & 1, bk = q >> 2;
        ch[slot_of(bi, bj, bk)] = L[ox + bi][oy + bj][oz + bk];
      }
      out.E.push_back(ch);
    }
  }
  for (const Face& f : in.bfaces) {
    const int a = f.face / 2, s = f.face % 2;
    for (int oc = 0; oc < 8; ++oc) {
      const int b[3] = {oc & 1, (oc >> 1) & 1, oc >> 2};
      if (b[a] == s) out.bfaces.push_back({f.elem * 8 + oc, f.face, f.tag});
    }
  }
  screen(out);
  return out;
}

// ---------------------------------------------------------------------------
// GLL basis (gll.cpp:13-114)
std::pair<double, double> legendre(int n, double t)
{
  if (n == 0) return {1.0, 0.0};
  double prev = 1.0, cur = t;
  for (int k = 2; k <= n; ++k) {
    const double nxt = ((2.0 * k - 1.0) * t * cur - (k - 1.0) * prev) / k;
    prev = cur;
    cur = nxt;
  }
  double d;
  if (std::abs(1.0 - t * t) < 1e-14)
    d = 0.5 * n * (n + 1.0) * (t > 0 ? 1.0 : ((n % 2 == 0) ? -1.0 : 1.0));
  else
    d = n * (prev - t * cur) / (1.0 - t * t);
  return {cur, d};
}

struct Basis {
  int n = 0;
  Vec t, w, D, B;  // nodes, weights, D[i*np+j] = phi_i'(t_j), B[corner*nloc + node]
  int np() const { return n + 1; }
};

Basis make_basis(int n)
{
  if (n < 1) throw BadInput("gll order must be >= 1, got " + std::to_string(n));
  Basis b;
  b.n = n;
  const int np = n + 1;
  Vec t(np, 0.0);
  t[0] = -1.0;
  t[n] = 1.0;
  for (int i = 1; i < n; ++i) {  // Newton on (1-t^2) P_n' from Chebyshev-Lobatto guesses (gll.cpp:43-56)
    double x = -std::cos(M_PI * i / n);
    for (int it = 0; it < 100; ++it) {
      const auto pd = legendre(n, x);
      const double dx = ((1.0 - x * x) * pd.second) / (-static_cast<double>(n) * (n + 1.0) * pd.first);
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    t[i] = x;
  }
  for (int i = 0; i <= n / 2; ++i) {  // exact symmetry (gll.cpp:57-61)
    const double s = 0.5 * (t[i] - t[n - i]);
    t[i] = s;
    t[n - i] = -s;
  }
  b.t = t;
  b.w.resize(np);
  for (int i = 0; i < np; ++i) {
    const double p = legendre(n, t[i]).first;
    b.w[i] = 2.0 / (n * (n + 1.0) * p * p);
  }
  b.D.assign(static_cast<std::size_t>(np) * np, 0.0);  // gll.cpp:70-87
  Vec Pn(np);
  for (int i = 0; i < np; ++i) Pn[i] = legendre(n, t[i]).first;
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j)
      if (i != j) b.D[i * np + j] = Pn[j] / (Pn[i] * (t[j] - t[i]));
  b.D[0] = -0.25 * n * (n + 1.0);
  b.D[np * np - 1] = 0.25 * n * (n + 1.0);
  const int nloc = np * np * np;  // gll.cpp:89-104
  b.B.resize(8 * static_cast<std::size_t>(nloc));
  auto hat = [](int w, double x) { return w == 0 ? 0.5 * (1 - x) : 0.5 * (1 + x); };
  for (int cb = 0; cb < 8; ++cb) {
    int l = 0;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l)
          b.B[cb * nloc + l] = hat(cb & 1, t[i]) * hat((cb >> 1) & 1, t[j]) * hat(cb >> 2, t[k]);
  }
  return b;
}

// ---------------------------------------------------------------------------
// Global numbering (mesh.cpp:240-453): every GLL node gets a canonical key of
// the mesh entity that owns it; the global id is the rank of the key.
using Key = std::array<i64, 5>;

Key face_key_of(const i32 c[2][2], int p, int q, int n)
{  // min over the 8 symmetries of the square (mesh.cpp:260-281)
  Key best{};
  bool first = true;
  for (int x0 = 0; x0 < 2; ++x0)
    for (int y0 = 0; y0 < 2; ++y0)
      for (int sw = 0; sw < 2; ++sw) {
        const i32 o = c[x0][y0];
        const i32 xn = sw ? c[x0][1 - y0] : c[1 - x0][y0];
        const i32 yn = sw ? c[1 - x0][y0] : c[x0][1 - y0];
        const int pp = x0 ? n - p : p, qq = y0 ? n - q : q;
        const int s = sw ? qq : pp, t = sw ? pp : qq;
        const Key k = {2, o, xn, static_cast<i64>(yn) * (n + 1) + s, t};
        if (first || k < best) best = k;
        first = false;
      }
  return best;
}

struct Maps {
  int n = 0;
  i32 N = 0;
  std::vector<i32> l2g;
  std::vector<i64> g2l_off;
  std::vector<i32> g2l_elem, g2l_local;
  std::vector<i32> sub;  // sub_l2g
  std::vector<std::uint8_t> mask;
  int nloc() const { return (n + 1) * (n + 1) * (n + 1); }
  int nsub() const { return (n + 3) * (n + 3) * (n + 3); }
};

Maps number(const Mesh& m, int n)
{
  const int np = n + 1, nloc = np * np * np;
  const i32 ne = m.ne();
  Maps M;
  M.n = n;
  std::vector<std::pair<Key, i64>> keys;
  keys.reserve(static_cast<std::size_t>(ne) * nloc);
  auto cls = [&](int i) { return i == 0 ? 0 : (i == n ? 2 : 1); };
  for (i32 e = 0; e < ne; ++e) {
    const auto& c = m.E[e];
    int l = 0;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l) {
          const int ix[3] = {i, j, k};
          const int ps[3] = {cls(i), cls(j), cls(k)};
          const int inner = (ps[0] == 1) + (ps[1] == 1) + (ps[2] == 1);
          Key key{};
          if (inner == 0) {  // vertex
            key = {0, c[slot_of(i / n, j / n, k / n)], 0, 0, 0};
          } else if (inner == 1) {  // edge interior: (min, max, param from min)
            const int a = ps[0] == 1 ? 0 : (ps[1] == 1 ? 1 : 2);
            int lo[3] = {ix[0] / n, ix[1] / n, ix[2] / n}, hi[3] = {lo[0], lo[1], lo[2]};
            lo[a] = 0;
            hi[a] = 1;
            i32 va = c[slot_of(lo[0], lo[1], lo[2])], vb = c[slot_of(hi[0], hi[1], hi[2])];
            int par = ix[a];
            if (va > vb) {
              std::swap(va, vb);
              par = n - par;
            }
            key = {1, va, vb, par, 0};
          } else if (inner == 2) {  // face interior
            const int a = ps[0] != 1 ? 0 : (ps[1] != 1 ? 1 : 2);
            const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
            i32 cc[2][2];
            for (int u = 0; u < 2; ++u)
              for (int v = 0; v < 2; ++v) {
                int b[3];
                b[a] = ix[a] / n;
                b[a1] = u;
                b[a2] = v;
                cc[u][v] = c[slot_of(b[0], b[1], b[2])];
              }
            key = face_key_of(cc, ix[a1], ix[a2], n);
          } else {  // element interior
            key = {3, e, l, 0, 0};
          }
          keys.push_back({key, static_cast<i64>(e) * nloc + l});
        }
  }
  std::sort(keys.begin(), keys.end());
  M.l2g.assign(keys.size(), -1);
  i32 g = -1;
  for (std::size_t q = 0; q < keys.size(); ++q) {
    if (q == 0 || keys[q].first != keys[q - 1].first) ++g;
    M.l2g[keys[q].second] = g;
  }
  M.N = g + 1;
  // g2l CSR in (e, l) order (mesh.cpp:352-367)
  M.g2l_off.assign(M.N + 1, 0);
  for (i32 x : M.l2g) M.g2l_off[x + 1]++;
  for (i32 x = 0; x < M.N; ++x) M.g2l_off[x + 1] += M.g2l_off[x];
  M.g2l_elem.resize(M.l2g.size());
  M.g2l_local.resize(M.l2g.size());
  std::vector<i64> cur(M.g2l_off.begin(), M.g2l_off.end() - 1);
  for (i32 e = 0; e < ne; ++e)
    for (int l = 0; l < nloc; ++l) {
      const i64 s = cur[M.l2g[static_cast<i64>(e) * nloc + l]]++;
      M.g2l_elem[s] = e;
      M.g2l_local[s] = l;
    }
  // Dirichlet mask (mesh.cpp:369-383)
  M.mask.assign(M.N, 0);
  for (const Face& f : m.bfaces) {
    if (f.tag != 0) continue;
    const int a = f.face / 2, s = f.face % 2;
    for (int v = 0; v < np; ++v)
      for (int u = 0; u < np; ++u) {
        int ijk[3];
        ijk[a] = s ? n : 0;
        ijk[(a + 1) % 3] = u;
        ijk[(a + 2) % 3] = v;
        M.mask[M.l2g[static_cast<i64>(f.elem) * nloc + (ijk[2] * np + ijk[1]) * np + ijk[0]]] = 1;
      }
  }
  // sub_l2g (mesh.cpp:385-451): interior slots = l2g; face slots = the
  // face-neighbour's first interior layer; others kNoNode = -1
  const int p = n + 3, nsub = p * p * p;
  M.sub.assign(static_cast<std::size_t>(ne) * nsub, -1);
  auto sslot = [&](int i, int j, int k) { return ((k + 1) * p + (j + 1)) * p + (i + 1); };
  std::map<std::array<i32, 4>, std::vector<std::pair<i32, int>>> faces;
  auto fkey = [&](i32 e, int f) {
    std::array<i32, 4> k{};
    const auto sl = face_slots(f);
    for (int q = 0; q < 4; ++q) k[q] = m.E[e][sl[q]];
    std::sort(k.begin(), k.end());
    return k;
  };
  for (i32 e = 0; e < ne; ++e)
    for (int f = 0; f < 6; ++f) faces[fkey(e, f)].push_back({e, f});
  for (const auto& kv : faces)
    if (kv.second.size() > 2) throw std::runtime_error("non-conforming mesh: face shared by more than two elements");
  for (i32 e = 0; e < ne; ++e) {
    const i64 eb = static_cast<i64>(e) * nloc;
    for (int k = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i)
          M.sub[static_cast<i64>(e) * nsub + sslot(i, j, k)] = M.l2g[eb + (k * np + j) * np + i];
    for (int f = 0; f < 6; ++f) {
      i32 e2 = -1;
      int f2 = -1;
      for (const auto& of : faces[fkey(e, f)])
        if (of.first != e) {
          e2 = of.first;
          f2 = of.second;
        }
      if (e2 < 0) continue;
      const int a = f / 2, s = f % 2, a2 = f2 / 2, s2 = f2 % 2;
      for (int v = 0; v < np; ++v)
        for (int u = 0; u < np; ++u) {
          int ijk[3];
          ijk[a] = s ? n : 0;
          ijk[(a + 1) % 3] = u;
          ijk[(a + 2) % 3] = v;
          const i32 gg = M.l2g[eb + (ijk[2] * np + ijk[1]) * np + ijk[0]];
          int l2 = -1;  // first copy of gg in e2 (mesh.cpp:413-417)
          for (i64 q = M.g2l_off[gg]; q < M.g2l_off[gg + 1]; ++q)
            if (M.g2l_elem[q] == e2) {
              l2 = M.g2l_local[q];
              break;
            }
          if (l2 < 0) throw std::runtime_error("global node has no copy in expected neighbor element");
          int q2[3] = {l2 % np, (l2 / np) % np, l2 / (np * np)};
          q2[a2] += s2 ? -1 : 1;
          int sl[3];
          sl[a] = s ? n + 1 : -1;
          sl[(a + 1) % 3] = u;
          sl[(a + 2) % 3] = v;
          M.sub[static_cast<i64>(e) * nsub + sslot(sl[0], sl[1], sl[2])] =
              M.l2g[static_cast<i64>(e2) * nloc + (q2[2] * np + q2[1]) * np + q2[0]];
        }
    }
  }
  return M;
}

// gather in CSR (e, l) order (mesh.cpp:463-475)
void gather(const Maps& M, const Vec& loc, Vec& glob)
{
  const int nloc = M.nloc();
  glob.assign(M.N, 0.0);
  for (i32 g = 0; g < M.N; ++g) {
    double s = 0;
    for (i64 q = M.g2l_off[g]; q < M.g2l_off[g + 1]; ++q)
      s += loc[static_cast<i64>(M.g2l_elem[q]) * nloc + M.g2l_local[q]];
    glob[g] = s;
  }
}

// ---------------------------------------------------------------------------
// Dense / envelope Cholesky (stands in for Eigen SimplicialLLT, coarse.cpp:89-127,
// amg.cpp:176-194). Envelope storage on the natural ordering.
struct Csr {
  i32 n = 0;
  std::vector<i64> ptr;
  std::vector<i32> col;
  Vec val;
  void mul(const Vec& x, Vec& y) const
  {  // CsrMatrix::multiply (amg.cpp:13-20)
    for (i32 i = 0; i < n; ++i) {
      double s = 0;
      for (i64 k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * x[col[k]];
      y[i] = s;
    }
  }
};

Csr from_triplets(i32 n, const std::vector<std::tuple<i32, i32, double>>& t3)
{  // csr_from_triplets (amg.cpp:22-40): std::sort on (row, col) only, then sum
   // duplicates in the sorted order. std::sort's permutation depends only on
   // the comparison outcomes, so the same input order gives the reference's
   // summation order.
  std::vector<std::pair<std::pair<i32, i32>, double>> t;
  t.reserve(t3.size());
  for (const auto& x : t3) t.push_back({{std::get<0>(x), std::get<1>(x)}, std::get<2>(x)});
  std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  Csr A;
  A.n = n;
  A.ptr.assign(n + 1, 0);
  for (std::size_t i = 0; i < t.size();) {
    std::size_t j = i;
    double s = 0;
    while (j < t.size() && t[j].first == t[i].first) s += t[j++].second;
    A.ptr[t[i].first.first + 1]++;
    A.col.push_back(t[i].first.second);
    A.val.push_back(s);
    i = j;
  }
  for (i32 i = 0; i < n; ++i) A.ptr[i + 1] += A.ptr[i];
  return A;
}

struct Envelope {
  // Sparse Cholesky in envelope (profile) storage after a reverse
  // Cuthill-McKee ordering (refined meshes have scattered vertex ids).
  i32 n = 0;
  std::vector<i32> perm;   // new -> old
  std::vector<i32> first;  // first column of row i's envelope (permuted)
  std::vector<i64> start;  // offset of row i
  Vec L;
  double& at(i32 i, i32 j) { return L[start[i] + (j - first[i])]; }
  double get(i32 i, i32 j) const { return j < first[i] ? 0.0 : L[start[i] + (j - first[i])]; }

  static std::vector<i32> rcm(const Csr& A)
  {
    const i32 n = A.n;
    std::vector<int> deg(n);
    for (i32 i = 0; i < n; ++i) deg[i] = static_cast<int>(A.ptr[i + 1] - A.ptr[i]);
    std::vector<i32> order;
    order.reserve(n);
    std::vector<char> seen(n, 0);
    std::vector<i32> byDeg(n);
    for (i32 i = 0; i < n; ++i) byDeg[i] = i;
    std::stable_sort(byDeg.begin(), byDeg.end(), [&](i32 a, i32 b) { return deg[a] < deg[b]; });
    for (i32 root : byDeg) {
      if (seen[root]) continue;
      std::size_t head = order.size();
      order.push_back(root);
      seen[root] = 1;
      while (head < order.size()) {
        const i32 v = order[head++];
        std::vector<i32> nb;
        for (i64 k = A.ptr[v]; k < A.ptr[v + 1]; ++k)
          if (!seen[A.col[k]]) {
            seen[A.col[k]] = 1;
            nb.push_back(A.col[k]);
          }
        std::stable_sort(nb.begin(), nb.end(), [&](i32 a, i32 b) { return deg[a] < deg[b]; });
        order.insert(order.end(), nb.begin(), nb.end());
      }
    }
    std::reverse(order.begin(), order.end());
    return order;
  }

  void factor(const Csr& A)
  {
    n = A.n;
    perm = rcm(A);
    std::vector<i32> inv(n);
    for (i32 i = 0; i < n; ++i) inv[perm[i]] = i;
    first.assign(n, 0);
    for (i32 i = 0; i < n; ++i) first[i] = i;
    for (i32 r = 0; r < n; ++r)
      for (i64 k = A.ptr[r]; k < A.ptr[r + 1]; ++k) {
        const i32 i = inv[r], j = inv[A.col[k]];
        if (j < i) first[i] = std::min(first[i], j);
      }
    start.assign(n + 1, 0);
    for (i32 i = 0; i < n; ++i) start[i + 1] = start[i] + (i - first[i] + 1);
    L.assign(start[n], 0.0);
    for (i32 r = 0; r < n; ++r)
      for (i64 k = A.ptr[r]; k < A.ptr[r + 1]; ++k) {
        const i32 i = inv[r], j = inv[A.col[k]];
        if (j <= i) at(i, j) = A.val[k];
      }
    for (i32 i = 0; i < n; ++i) {
      for (i32 j = first[i]; j <= i; ++j) {
        double s = at(i, j);
        const i32 k0 = std::max(first[i], first[j]);
        const double* li = &L[start[i] + (k0 - first[i])];
        const double* lj = &L[start[j] + (k0 - first[j])];
        for (i32 k = 0; k < j - k0; ++k) s -= li[k] * lj[k];
        if (j < i) {
          at(i, j) = s / at(j, j);
        } else {
          if (!(s > 0)) throw std::runtime_error("coarse matrix Cholesky failed (matrix not SPD?)");
          at(i, i) = std::sqrt(s);
        }
      }
    }
  }
  void solve(const Vec& b, Vec& x) const
  {
    Vec y(n);
    for (i32 i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (i32 i = 0; i < n; ++i) {
      double s = y[i];
      for (i32 k = first[i]; k < i; ++k) s -= get(i, k) * y[k];
      y[i] = s / get(i, i);
    }
    for (i32 i = n - 1; i >= 0; --i) {
      y[i] /= get(i, i);
      for (i32 k = first[i]; k < i; ++k) y[k] -= get(i, k) * y[i];
    }
    x.assign(n, 0.0);
    for (i32 i = 0; i < n; ++i) x[perm[i]] = y[i];
  }
};

// ---------------------------------------------------------------------------
// AMG (amg.cpp:42-279): greedy aggregation (target 8), Galerkin, K-cycle.
struct Amg {
  struct Level {
    Csr A;
    Vec idiag;
    std::vector<i32> agg;
    i32 nc = 0;
  };
  std::vector<Level> lv;
  Csr coarsest;
  Envelope chol;

  static Vec inv_diag(const Csr& A)
  {
    Vec d(A.n, 0.0);
    for (i32 i = 0; i < A.n; ++i) {
      double v = 0;
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
        if (A.col[k] == i) v = A.val[k];
      if (!(v > 0)) throw std::runtime_error("amg: non-positive diagonal at row " + std::to_string(i));
      d[i] = 1 / v;
    }
    return d;
  }

  static i32 aggregate(const Csr& A, std::vector<i32>& grp)
  {  // aggregate_pass (amg.cpp:53-112)
    grp.assign(A.n, -1);
    std::vector<int> size;
    i32 next = 0;
    for (i32 i = 0; i < A.n; ++i) {
      if (grp[i] >= 0) continue;
      std::vector<std::pair<double, i32>> nb;
      bool clean = true;
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1] && clean; ++k) {
        const i32 j = A.col[k];
        if (j == i || A.val[k] == 0.0) continue;
        if (grp[j] >= 0) clean = false;
        else nb.push_back({-std::abs(A.val[k]), j});
      }
      if (!clean) continue;
      grp[i] = next;
      std::sort(nb.begin(), nb.end());
      int sz = 1;
      for (const auto& x : nb) {
        if (sz >= 8) break;
        grp[x.second] = next;
        ++sz;
      }
      size.push_back(sz);
      ++next;
    }
    for (i32 i = 0; i < A.n; ++i) {
      if (grp[i] >= 0) continue;
      i32 best = -1;
      double bv = 0;
      bool bsmall = false;
      for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const i32 j = A.col[k];
        if (j == i || grp[j] < 0 || A.val[k] == 0.0) continue;
        const double a = std::abs(A.val[k]);
        const bool small = size[grp[j]] < 8;
        if (best < 0 || (small && !bsmall) || (small == bsmall && a > bv)) {
          best = grp[j];
          bv = a;
          bsmall = small;
        }
      }
      if (best >= 0) {
        grp[i] = best;
        ++size[best];
      } else {
        grp[i] = next++;
        size.push_back(1);
      }
    }
    return next;
  }

  void setup(Csr A)
  {  // Impl::setup (amg.cpp:151-186)
    while (A.n > 64) {
      Level L;
      L.idiag = inv_diag(A);
      std::vector<i32> g;
      const i32 nc = aggregate(A, g);
      if (nc > static_cast<i32>(0.95 * A.n)) break;
      std::vector<std::tuple<i32, i32, double>> t;
      t.reserve(A.val.size());
      for (i32 i = 0; i < A.n; ++i)
        for (i64 k = A.ptr[i]; k < A.ptr[i + 1]; ++k) t.emplace_back(g[i], g[A.col[k]], A.val[k]);
      Csr C = from_triplets(nc, t);
      L.agg = std::move(g);
      L.nc = nc;
      L.A = std::move(A);
      A = std::move(C);
      lv.push_back(std::move(L));
    }
    coarsest = std::move(A);
    inv_diag(coarsest);
    chol.factor(coarsest);
  }

  void cycle(std::size_t l, const Vec& r, Vec& z) const
  {  // amg.cpp:198-227, omega = 2/3, 2 sweeps
    if (l == lv.size()) {
      chol.solve(r, z);
      return;
    }
    const Level& L = lv[l];
    const i32 n = L.A.n;
    const double w = 2.0 / 3.0;
    Vec tmp(n), rho(n);
    for (i32 i = 0; i < n; ++i) z[i] = w * L.idiag[i] * r[i];
    auto sweep = [&] {
      L.A.mul(z, tmp);
      for (i32 i = 0; i < n; ++i) z[i] += w * L.idiag[i] * (r[i] - tmp[i]);
    };
    sweep();
    L.A.mul(z, tmp);
    for (i32 i = 0; i < n; ++i) rho[i] = r[i] - tmp[i];
    Vec rc(L.nc, 0.0), ec(L.nc, 0.0);
    for (i32 i = 0; i < n; ++i) rc[L.agg[i]] += rho[i];
    ksolve(l + 1, rc, ec);
    for (i32 i = 0; i < n; ++i) z[i] += ec[L.agg[i]];
    sweep();
    sweep();
  }

  void ksolve(std::size_t l, const Vec& b, Vec& x) const
  {  // two PCG steps preconditioned by cycle(l) (amg.cpp:230-263)
    if (l == lv.size()) {
      chol.solve(b, x);
      return;
    }
    const Csr& A = lv[l].A;
    const i32 n = A.n;
    Vec r(b), z(n), p(n), f(n);
    std::fill(x.begin(), x.end(), 0.0);
    cycle(l, r, z);
    double zr = 0;
    for (i32 i = 0; i < n; ++i) zr += z[i] * r[i];
    p = z;
    for (int it = 0; it < 2; ++it) {
      A.mul(p, f);
      double pf = 0;
      for (i32 i = 0; i < n; ++i) pf += p[i] * f[i];
      if (!(pf > 0) || !(std::abs(zr) > 0)) return;
      const double alpha = zr / pf;
      for (i32 i = 0; i < n; ++i) {
        x[i] += alpha * p[i];
        r[i] -= alpha * f[i];
      }
      if (it == 1) break;
      cycle(l, r, z);
      double zn = 0;
      for (i32 i = 0; i < n; ++i) zn += z[i] * r[i];
      const double beta = zn / zr;
      zr = zn;
      for (i32 i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
  }
};

// ---------------------------------------------------------------------------
// Fine Schwarz pencil (fine.cpp:15-80) with a cyclic Jacobi eigen-solver.
struct Pencil {
  int p = 0;
  Vec K, M, V, Vi, lam;
};

void jacobi_eigen(int n, Vec S, Vec& lam, Vec& Q)
{  // S symmetric row-major; columns of Q are eigenvectors; ascending eigenvalues
  Q.assign(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) Q[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += S[i * n + j] * S[i * n + j];
    if (off < 1e-300) break;
    for (int pp = 0; pp < n; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        const double apq = S[pp * n + q];
        if (apq == 0.0) continue;
        const double theta = (S[q * n + q] - S[pp * n + pp]) / (2 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double a = S[k * n + pp], b = S[k * n + q];
          S[k * n + pp] = c * a - s * b;
          S[k * n + q] = s * a + c * b;
        }
        for (int k = 0; k < n; ++k) {
          const double a = S[pp * n + k], b = S[q * n + k];
          S[pp * n + k] = c * a - s * b;
          S[q * n + k] = s * a + c * b;
        }
        for (int k = 0; k < n; ++k) {
          const double a = Q[k * n + pp], b = Q[k * n + q];
          Q[k * n + pp] = c * a - s * b;
          Q[k * n + q] = s * a + c * b;
        }
      }
  }
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return S[a * n + a] < S[b * n + b]; });
  lam.resize(n);
  Vec Qs(static_cast<std::size_t>(n) * n);
  for (int c = 0; c < n; ++c) {
    lam[c] = S[ord[c] * n + ord[c]];
    for (int r = 0; r < n; ++r) Qs[r * n + c] = Q[r * n + ord[c]];
  }
  Q = Qs;
}

Pencil make_pencil(const Basis& b)
{
  const int n = b.n, np = n + 1, p = n + 3;
  Vec d(static_cast<std::size_t>(np) * np, 0.0);  // d_ij = sum_m D_im D_jm rho_m (fine.cpp:20-27)
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      double s = 0;
      for (int m = 0; m < np; ++m) s += b.D[i * np + m] * b.D[j * np + m] * b.w[m];
      d[i * np + j] = s;
    }
  Pencil P;
  P.p = p;
  P.K.assign(static_cast<std::size_t>(p) * p, 0.0);
  P.M.assign(p, 0.0);
  for (int o = -2; o <= 2; ++o)  // lattice assembly over nodes -1..n+1 (fine.cpp:36-50)
    for (int a = 0; a <= n; ++a) {
      const int pa = o * n + a;
      if (pa < -1 || pa > n + 1) continue;
      P.M[pa + 1] += b.w[a];
      for (int c = 0; c <= n; ++c) {
        const int pb = o * n + c;
        if (pb < -1 || pb > n + 1) continue;
        P.K[(pa + 1) * p + (pb + 1)] += d[a * np + c];
      }
    }
  Vec S(static_cast<std::size_t>(p) * p);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) S[i * p + j] = P.K[i * p + j] / std::sqrt(P.M[i] * P.M[j]);
  Vec Ssym(S.size());
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) Ssym[i * p + j] = 0.5 * (S[i * p + j] + S[j * p + i]);
  Vec Q;
  jacobi_eigen(p, Ssym, P.lam, Q);
  for (int i = 0; i < p; ++i)
    if (!(P.lam[i] > 0)) throw std::runtime_error("pencil eigenvalue not positive");
  P.V.resize(static_cast<std::size_t>(p) * p);
  P.Vi.resize(static_cast<std::size_t>(p) * p);
  for (int i = 0; i < p; ++i)  // V[i][j] = Q(j,i) sqrt(M_j), V^-1[i][j] = Q(i,j)/sqrt(M_i) (fine.cpp:72-78)
    for (int j = 0; j < p; ++j) {
      P.V[i * p + j] = Q[j * p + i] * std::sqrt(P.M[j]);
      P.Vi[i * p + j] = Q[i * p + j] / std::sqrt(P.M[i]);
    }
  return P;
}

// out[..d..] = sum_a mat[d*p+a] in[..a..] along one axis (fine.cpp:98-136)
void pass(int p, int axis, const Vec& mat, const double* in, double* out)
{
  for (int k = 0; k < p; ++k)
    for (int j = 0; j < p; ++j)
      for (int i = 0; i < p; ++i) {
        const int dd = axis == 0 ? i : (axis == 1 ? j : k);
        double s = 0;
        for (int a = 0; a < p; ++a) {
          const int src = axis == 0 ? (k * p + j) * p + a : (axis == 1 ? (k * p + a) * p + i : (a * p + j) * p + i);
          s += mat[dd * p + a] * in[src];
        }
        out[(k * p + j) * p + i] = s;
      }
}

// solve_subdomain (fine.cpp:140-185)
void subdomain_solve(const Pencil& P, const double* r, const std::array<double, 3>& h, double kap, double c,
                     double* z)
{
  const int p = P.p, ns = p * p * p;
  Vec w(ns), t(ns);
  const double svol = 8.0 / (h[0] * h[1] * h[2]);
  const double ix2 = 1.0 / (h[0] * h[0]), iy2 = 1.0 / (h[1] * h[1]), iz2 = 1.0 / (h[2] * h[2]);
  for (int k = 0, q = 0; k < p; ++k)
    for (int j = 0; j < p; ++j)
      for (int i = 0; i < p; ++i, ++q) w[q] = svol * r[q] / (P.M[i] * P.M[j] * P.M[k]);
  pass(p, 0, P.V, w.data(), t.data());
  pass(p, 1, P.V, t.data(), w.data());
  pass(p, 2, P.V, w.data(), t.data());
  for (int f = 0, q = 0; f < p; ++f)
    for (int e = 0; e < p; ++e)
      for (int d = 0; d < p; ++d, ++q) t[q] /= 4 * kap * (P.lam[d] * ix2 + P.lam[e] * iy2 + P.lam[f] * iz2) + c;
  pass(p, 0, P.Vi, t.data(), w.data());
  pass(p, 1, P.Vi, w.data(), t.data());
  pass(p, 2, P.Vi, t.data(), z);
}

// ---------------------------------------------------------------------------
// The system (problem.cpp:73-108 build_system)
struct System {
  int mode = 0;  // 0 two_scale, 1 fine_only, 2 coarse_only, 3 none
  int variant = 0;  // OperatorVariant: 0 stored, 1 on_the_fly (operator.hpp:14)
  Mesh mesh;
  Basis basis;
  Maps maps;
  Vec kappa, c;
  Vec mass;                     // NE*nloc
  std::array<Vec, 6> wg;        // kappa*m*Gt planes
  Vec lumped;
  // fine
  bool has_fine = false;
  Pencil pencil;
  std::vector<std::array<double, 3>> h;
  // coarse
  bool has_coarse = false, use_amg = false;
  std::vector<std::uint8_t> vmask;
  Csr Kc;
  Amg amg;
  Envelope direct;
  double build_seconds = 0;

  i32 N() const { return maps.N; }
};

void build(System& S, const int* ccfg_mode, int coarse_solve, int direct_threshold)
{
  const int n = S.basis.n, np = n + 1, nloc = np * np * np;
  const i32 ne = S.mesh.ne();
  S.mode = *ccfg_mode;
  S.maps = number(S.mesh, n);
  // compute_factors (geometry.cpp:105-151) + SemOperator ctor (operator.cpp:61-95)
  S.mass.resize(static_cast<std::size_t>(ne) * nloc);
  for (auto& g : S.wg) g.resize(S.mass.size());
  for (i32 e = 0; e < ne; ++e)
    for (int k = 0, l = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l) {
          const Jac J = jacobian_at(S.mesh, e, S.basis.t[i], S.basis.t[j], S.basis.t[k]);
          double v[9];
          inverse(J, v);
          auto gt = [&](int r, int cc) { return v[3 * r] * v[3 * cc] + v[3 * r + 1] * v[3 * cc + 1] + v[3 * r + 2] * v[3 * cc + 2]; };
          const std::size_t at = static_cast<std::size_t>(e) * nloc + l;
          const double m = S.basis.w[i] * S.basis.w[j] * S.basis.w[k] * J.det;
          S.mass[at] = m;
          const double g6[6] = {gt(0, 0), gt(0, 1), gt(0, 2), gt(1, 1), gt(1, 2), gt(2, 2)};
          for (int q = 0; q < 6; ++q) S.wg[q][at] = g6[q] * (S.kappa[e] * m);
        }
  for (i32 e = 0; e < ne; ++e)
    if (S.kappa[e] < 0 || S.c[e] < 0) throw BadInput("kappa/c must be nonnegative");
  gather(S.maps, S.mass, S.lumped);

  S.has_fine = S.mode == 0 || S.mode == 1;
  S.has_coarse = S.mode == 0 || S.mode == 2;
  if (S.has_coarse) {
    // coarse_dirichlet_mask + assemble_coarse_matrix (coarse.cpp:11-87)
    const i32 nv = S.mesh.nv();
    S.vmask.assign(nv, 0);
    for (const Face& f : S.mesh.bfaces)
      if (f.tag == 0)
        for (int sl : face_slots(f.face)) S.vmask[S.mesh.E[f.elem][sl]] = 1;
    std::vector<std::tuple<i32, i32, double>> t;
    for (i32 e = 0; e < ne; ++e) {
      double ke[8][8] = {};
      for (int qb = 0; qb < 8; ++qb) {
        const Jac J = jacobian_at(S.mesh, e, (qb & 1) ? 1.0 : -1.0, (qb & 2) ? 1.0 : -1.0, (qb & 4) ? 1.0 : -1.0);
        double v[9];
        inverse(J, v);
        const double hq[3][2] = {{(qb & 1) ? 0.0 : 1.0, (qb & 1) ? 1.0 : 0.0},
                                 {(qb & 2) ? 0.0 : 1.0, (qb & 2) ? 1.0 : 0.0},
                                 {(qb & 4) ? 0.0 : 1.0, (qb & 4) ? 1.0 : 0.0}};
        double gr[8][3];
        for (int ab = 0; ab < 8; ++ab) {
          const int bi = ab & 1, bj = (ab >> 1) & 1, bk = ab >> 2;
          const double dh[3] = {(bi ? 0.5 : -0.5) * hq[1][bj] * hq[2][bk], hq[0][bi] * (bj ? 0.5 : -0.5) * hq[2][bk],
                                hq[0][bi] * hq[1][bj] * (bk ? 0.5 : -0.5)};
          for (int d = 0; d < 3; ++d) gr[ab][d] = v[d] * dh[0] + v[3 + d] * dh[1] + v[6 + d] * dh[2];
        }
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b) {
            double s = S.kappa[e] * (gr[a][0] * gr[b][0] + gr[a][1] * gr[b][1] + gr[a][2] * gr[b][2]);
            if (a == b && a == qb) s += S.c[e];
            ke[a][b] += J.det * s;
          }
      }
      for (int a = 0; a < 8; ++a) {
        const i32 ga = S.mesh.E[e][kSlot[a]];
        for (int b = 0; b < 8; ++b) {
          const i32 gb = S.mesh.E[e][kSlot[b]];
          if (S.vmask[ga] || S.vmask[gb]) continue;
          t.emplace_back(ga, gb, ke[a][b]);
        }
      }
    }
    for (i32 v = 0; v < nv; ++v)
      if (S.vmask[v]) t.emplace_back(v, v, 1.0);
    S.Kc = from_triplets(nv, t);
    S.use_amg = coarse_solve == 2 || (coarse_solve == 0 && S.Kc.n > direct_threshold);
    if (S.use_amg)
      S.amg.setup(S.Kc);
    else
      S.direct.factor(S.Kc);
  }
  if (S.has_fine) {
    S.pencil = make_pencil(S.basis);
    S.h.resize(ne);
    for (i32 e = 0; e < ne; ++e) S.h[e] = elem_h(S.mesh, e);
  }
}

// otf_element_kernel geometry (operator.cpp:174-251): per node, the Jacobian
// from the 8 corners in (bk,bj,bi) order, its adjugate, det, and
// kappa rho^3/det adj adj^T, m = rho^3 det. Writes element-local planes.
void otf_geometry(const System& S, i32 e, std::array<Vec, 6>& wg, Vec& m)
{
  const int np = S.basis.np();
  const Vec& t = S.basis.t;
  const Vec& w = S.basis.w;
  double xyz[8][3];
  for (int cc = 0; cc < 8; ++cc)
    for (int d = 0; d < 3; ++d) xyz[cc][d] = S.mesh.X[S.mesh.E[e][cc]][d];
  const double kap = S.kappa[e];
  for (int k = 0, node = 0; k < np; ++k)
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i, ++node) {
        const double h[3][2] = {{0.5 * (1 - t[i]), 0.5 * (1 + t[i])},
                                {0.5 * (1 - t[j]), 0.5 * (1 + t[j])},
                                {0.5 * (1 - t[k]), 0.5 * (1 + t[k])}};
        const double dh[2] = {-0.5, 0.5};
        double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int bk = 0; bk < 2; ++bk)
          for (int bj = 0; bj < 2; ++bj)
            for (int bi = 0; bi < 2; ++bi) {
              const int cc = slot_of(bi, bj, bk);
              const double wx = dh[bi] * h[1][bj] * h[2][bk];
              const double wy = h[0][bi] * dh[bj] * h[2][bk];
              const double wz = h[0][bi] * h[1][bj] * dh[bk];
              for (int d = 0; d < 3; ++d) {
                J[d * 3 + 0] += wx * xyz[cc][d];
                J[d * 3 + 1] += wy * xyz[cc][d];
                J[d * 3 + 2] += wz * xyz[cc][d];
              }
            }
        double a[9];
        a[0] = J[4] * J[8] - J[5] * J[7];
        a[1] = J[2] * J[7] - J[1] * J[8];
        a[2] = J[1] * J[5] - J[2] * J[4];
        a[3] = J[5] * J[6] - J[3] * J[8];
        a[4] = J[0] * J[8] - J[2] * J[6];
        a[5] = J[2] * J[3] - J[0] * J[5];
        a[6] = J[3] * J[7] - J[4] * J[6];
        a[7] = J[1] * J[6] - J[0] * J[7];
        a[8] = J[0] * J[4] - J[1] * J[3];
        const double det = J[0] * a[0] + J[1] * a[3] + J[2] * a[6];
        if (!(det > 0)) throw std::runtime_error("inverted element in on-the-fly kernel");
        const double rho3 = w[i] * w[j] * w[k];
        const double scale = kap * rho3 / det;
        auto aat = [&](int r0, int c0) {
          return a[r0 * 3 + 0] * a[c0 * 3 + 0] + a[r0 * 3 + 1] * a[c0 * 3 + 1] + a[r0 * 3 + 2] * a[c0 * 3 + 2];
        };
        wg[0][node] = scale * aat(0, 0);
        wg[1][node] = scale * aat(0, 1);
        wg[2][node] = scale * aat(0, 2);
        wg[3][node] = scale * aat(1, 1);
        wg[4][node] = scale * aat(1, 2);
        wg[5][node] = scale * aat(2, 2);
        m[node] = rho3 * det;
      }
}

// SemOperator::apply (operator.cpp:124-163, 255-287), stored or on-the-fly geometry
void apply_A(const System& S, const double* u, double* r)
{
  const int np = S.basis.np(), nloc = np * np * np;
  const Maps& M = S.maps;
  const double* D = S.basis.D.data();
  Vec ul(nloc), fa(nloc), fb(nloc), fc(nloc), rl(static_cast<std::size_t>(S.mesh.ne()) * nloc);
  std::array<Vec, 6> wotf;
  Vec motf(S.variant ? nloc : 0);
  for (auto& v : wotf) v.resize(S.variant ? nloc : 0);
  for (i32 e = 0; e < S.mesh.ne(); ++e) {
    const std::size_t eb = static_cast<std::size_t>(e) * nloc;
    if (S.variant) otf_geometry(S, e, wotf, motf);
    const std::size_t gb = S.variant ? 0 : eb;  // plane offset of this element
    const std::array<const Vec*, 6> W = S.variant ? std::array<const Vec*, 6>{&wotf[0], &wotf[1], &wotf[2], &wotf[3], &wotf[4], &wotf[5]}
                                                  : std::array<const Vec*, 6>{&S.wg[0], &S.wg[1], &S.wg[2], &S.wg[3], &S.wg[4], &S.wg[5]};
    const double* mass = S.variant ? motf.data() : &S.mass[eb];
    for (int l = 0; l < nloc; ++l) {
      const i32 g = M.l2g[eb + l];
      ul[l] = M.mask[g] ? 0.0 : u[g];
    }
    for (int k = 0, l = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l) {
          double sx = 0, sy = 0, sz = 0;
          for (int m = 0; m < np; ++m) {
            sx += D[m * np + i] * ul[(k * np + j) * np + m];
            sy += D[m * np + j] * ul[(k * np + m) * np + i];
            sz += D[m * np + k] * ul[(m * np + j) * np + i];
          }
          const double* w[6] = {&(*W[0])[gb], &(*W[1])[gb], &(*W[2])[gb], &(*W[3])[gb], &(*W[4])[gb], &(*W[5])[gb]};
          fa[l] = w[0][l] * sx + w[1][l] * sy + w[2][l] * sz;
          fb[l] = w[1][l] * sx + w[3][l] * sy + w[4][l] * sz;
          fc[l] = w[2][l] * sx + w[4][l] * sy + w[5][l] * sz;
        }
    for (int k = 0, l = 0; k < np; ++k)
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i, ++l) {
          double s = 0;
          for (int m = 0; m < np; ++m) {
            s += D[i * np + m] * fa[(k * np + j) * np + m];
            s += D[j * np + m] * fb[(k * np + m) * np + i];
            s += D[k * np + m] * fc[(m * np + j) * np + i];
          }
          rl[eb + l] = s + (S.c[e] * ul[l]) * mass[l];
        }
  }
  Vec rg;
  gather(M, rl, rg);
  for (i32 g = 0; g < M.N; ++g) r[g] = M.mask[g] ? u[g] : rg[g];
}

// FinePreconditioner::apply (fine.cpp:210-231)
void apply_fine(const System& S, const double* r, double* z)
{
  const int p = S.pencil.p, ns = p * p * p;
  Vec rs(ns), zs(ns);
  std::fill(z, z + S.N(), 0.0);
  for (i32 e = 0; e < S.mesh.ne(); ++e) {
    const i32* sub = &S.maps.sub[static_cast<std::size_t>(e) * ns];
    for (int s = 0; s < ns; ++s) rs[s] = sub[s] < 0 ? 0.0 : r[sub[s]];
    subdomain_solve(S.pencil, rs.data(), S.h[e], S.kappa[e], S.c[e], zs.data());
    for (int s = 0; s < ns; ++s)
      if (sub[s] >= 0) z[sub[s]] += zs[s];
  }
}

// restrict_residual (coarse.cpp:138-162)
void restrict_res(const System& S, const double* r, Vec& R)
{
  const int nloc = S.maps.nloc();
  R.assign(S.mesh.nv(), 0.0);
  Vec y(nloc);
  for (i32 e = 0; e < S.mesh.ne(); ++e) {
    const std::size_t eb = static_cast<std::size_t>(e) * nloc;
    for (int l = 0; l < nloc; ++l) {
      const i32 g = S.maps.l2g[eb + l];
      y[l] = r[g] / S.lumped[g];
    }
    for (int cb = 0; cb < 8; ++cb) {
      double s = 0;
      for (int l = 0; l < nloc; ++l) s += S.basis.B[cb * nloc + l] * y[l] * S.mass[eb + l];
      R[S.mesh.E[e][kSlot[cb]]] += s;
    }
  }
}

// prolongate (coarse.cpp:164-186)
void prolong(const System& S, const Vec& Z, double* z)
{
  const int nloc = S.maps.nloc();
  Vec zl(static_cast<std::size_t>(S.mesh.ne()) * nloc);
  for (i32 e = 0; e < S.mesh.ne(); ++e) {
    double zc[8];
    for (int cb = 0; cb < 8; ++cb) zc[cb] = Z[S.mesh.E[e][kSlot[cb]]];
    const std::size_t eb = static_cast<std::size_t>(e) * nloc;
    for (int l = 0; l < nloc; ++l) {
      double s = 0;
      for (int cb = 0; cb < 8; ++cb) s += S.basis.B[cb * nloc + l] * zc[cb];
      zl[eb + l] = s * S.mass[eb + l];
    }
  }
  Vec zg;
  gather(S.maps, zl, zg);
  for (i32 g = 0; g < S.N(); ++g) z[g] = zg[g] / S.lumped[g];
}

// CoarsePreconditioner::apply (coarse.cpp:188-208)
void apply_coarse(const System& S, const double* r, double* z)
{
  Vec R, Z(S.mesh.nv(), 0.0);
  restrict_res(S, r, R);
  for (i32 v = 0; v < S.Kc.n; ++v)
    if (S.vmask[v]) R[v] = 0;
  if (S.use_amg) {
    S.amg.cycle(0, R, Z);
    Vec rho(S.Kc.n), dz(S.Kc.n, 0.0);
    S.Kc.mul(Z, rho);
    for (i32 v = 0; v < S.Kc.n; ++v) rho[v] = R[v] - rho[v];
    S.amg.cycle(0, rho, dz);
    for (i32 v = 0; v < S.Kc.n; ++v) Z[v] += dz[v];
  } else {
    S.direct.solve(R, Z);
  }
  prolong(S, Z, z);
}

// TwoScalePreconditioner::apply, sequential (precond.cpp:27-67)
void apply_P(const System& S, const double* r, double* z)
{
  const i32 N = S.N();
  if (S.mode == 3) {
    std::copy(r, r + N, z);
    return;
  }
  Vec rm(N), zf(N, 0.0), zc(N, 0.0);
  for (i32 g = 0; g < N; ++g) rm[g] = S.maps.mask[g] ? 0.0 : r[g];
  const bool f = S.mode != 2, c = S.mode != 1;
  if (f) apply_fine(S, rm.data(), zf.data());
  if (c) apply_coarse(S, rm.data(), zc.data());
  for (i32 g = 0; g < N; ++g) {
    if (S.maps.mask[g]) {
      z[g] = r[g];
    } else {
      double s = 0;
      if (f) s += zf[g];
      if (c) s += zc[g];
      z[g] = s;
    }
  }
}

// 0: the reference's sequential double accumulation (krylov.cpp:11-16);
// 1: correctly rounded (double-double compensated products and sums) — an
//    instrument for separating summation rounding from everything else
int g_dot_mode = 0;

double dot(const Vec& a, const Vec& b)
{
  if (g_dot_mode == 0) {  // krylov.cpp:11-16
    double s = 0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
  }
  double hi = 0, lo = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double p = a[i] * b[i];
    const double pe = std::fma(a[i], b[i], -p);  // exact product error
    const double t = hi + p;
    const double z = t - hi;
    lo += (hi - (t - z)) + (p - z) + pe;  // TwoSum error + product error
    hi = t;
  }
  return hi + lo;
}

// pcg with u0 = 0 (krylov.cpp:20-71)
void pcg(const System& S, const double* b, double tol, int maxit, int* iters, int* status, double* rh, double* zh,
         double* uo)
{
  if (!(tol > 0) || !(tol < 1)) throw BadInput("pcg: rel_tolerance must lie in (0,1)");
  if (maxit < 1) throw BadInput("pcg: max_iterations must be >= 1");
  const i32 N = S.N();
  Vec u(N, 0.0), r(b, b + N), z(N), p(N), f(N);
  int nr = 0, nz = 0;
  *iters = 0;
  *status = 0;
  const double r0 = std::sqrt(dot(r, r));
  rh[nr++] = r0;
  if (r0 != 0.0) {
    apply_P(S, r.data(), z.data());
    p = z;
    double zr = dot(z, r);
    *status = 1;
    for (int k = 0; k < maxit; ++k) {
      zh[nz++] = zr;
      apply_A(S, p.data(), f.data());
      const double pf = dot(p, f);
      if (!(pf > 0)) {
        *status = 2;
        break;
      }
      const double alpha = zr / pf;
      for (i32 i = 0; i < N; ++i) {
        u[i] += alpha * p[i];
        r[i] -= alpha * f[i];
      }
      *iters = k + 1;
      const double rn = std::sqrt(dot(r, r));
      rh[nr++] = rn;
      if (rn / r0 <= tol) {
        *status = 0;
        break;
      }
      apply_P(S, r.data(), z.data());
      const double zn = dot(z, r);
      const double beta = zn / zr;
      zr = zn;
      for (i32 i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
    }
  }
  if (uo) std::copy(u.begin(), u.end(), uo);
}

thread_local std::string g_err;

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

unsigned long long upow(unsigned long long b, int e)
{
  unsigned long long r = 1;
  while (e-- > 0) r *= b;
  return r;
}

}  // namespace orc

using namespace orc;

extern "C" {

// Same layout as ref_config (oracle/ref_driver.cpp) = ProblemConfig subset (problem.hpp:35-62).
struct orc_config {
  int k, refine, family, boundary;
  int bar[3];
  double bar_size[3];
  int order;
  double kappa, c;
  int precond, variant, coarse_solve, coarse_direct_threshold;
  int concurrent_precond, fine_threads;
};

const char* orc_last_error() { return g_err.c_str(); }

// Dot-product summation mode of the restated pcg (see orc::dot).
void orc_set_dot_mode(int mode) { g_dot_mode = mode; }

static void finish(System& S, const orc_config* c)
{
  const auto t0 = std::chrono::steady_clock::now();
  build(S, &c->precond, c->coarse_solve, c->coarse_direct_threshold);
  S.build_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int orc_create(const orc_config* c, void** out)
{
  return guard([&] {
    if (c->variant != 0 && c->variant != 1) throw BadInput("unknown operator variant");
    auto S = std::make_unique<System>();
    S->variant = c->variant;
    const auto t0 = std::chrono::steady_clock::now();
    if (c->bar[0] > 0)
      S->mesh = box(c->bar[0], c->bar[1], c->bar[2], c->bar_size, c->boundary);
    else
      S->mesh = cube(c->k, c->family, c->boundary);
    for (int q = 0; q < c->refine; ++q) S->mesh = refine(S->mesh);
    S->basis = make_basis(c->order);
    S->kappa.assign(S->mesh.ne(), c->kappa);
    S->c.assign(S->mesh.ne(), c->c);
    S->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    finish(*S, c);
    *out = S.release();
  });
}

int orc_create_mesh(int nv, const double* xyz, int ne, const int32_t* conn, int nbf, const int32_t* bf_elem,
                    const int32_t* bf_face, const uint8_t* bf_tag, int order, const double* kappa_e,
                    const double* c_e, const orc_config* c, void** out)
{
  return guard([&] {
    auto S = std::make_unique<System>();
    S->variant = c->variant;
    S->mesh.X.resize(nv);
    for (int v = 0; v < nv; ++v)
      for (int d = 0; d < 3; ++d) S->mesh.X[v][d] = xyz[3 * v + d];
    S->mesh.E.resize(ne);
    for (int e = 0; e < ne; ++e)
      for (int q = 0; q < 8; ++q) S->mesh.E[e][q] = conn[8 * e + q];
    for (int b = 0; b < nbf; ++b) S->mesh.bfaces.push_back({bf_elem[b], bf_face[b], bf_tag[b]});
    screen(S->mesh);
    S->basis = make_basis(order);
    S->kappa.assign(kappa_e, kappa_e + ne);
    S->c.assign(c_e, c_e + ne);
    finish(*S, c);
    *out = S.release();
  });
}

void orc_destroy(void* h) { delete static_cast<System*>(h); }

int orc_info(void* hp, int64_t* info)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    info[0] = S.N();
    info[1] = S.mesh.ne();
    info[2] = S.mesh.nv();
    info[3] = S.basis.n;
    info[4] = S.has_coarse ? S.Kc.n : 0;
    info[5] = S.use_amg ? 1 : 0;
    info[6] = S.use_amg ? static_cast<int64_t>(S.amg.lv.size()) + 1 : 0;
    info[7] = static_cast<int64_t>(S.mesh.bfaces.size());
    info[8] = static_cast<int64_t>(S.build_seconds * 1000.0);
    info[9] = S.has_fine ? 1 : 0;
  });
}

int orc_export_mesh(void* hp, double* xyz, int32_t* conn, int32_t* bf_elem, int32_t* bf_face, uint8_t* bf_tag)
{
  return guard([&] {
    const Mesh& m = static_cast<System*>(hp)->mesh;
    for (i32 v = 0; v < m.nv(); ++v)
      for (int d = 0; d < 3; ++d) xyz[3 * v + d] = m.X[v][d];
    for (i32 e = 0; e < m.ne(); ++e)
      for (int q = 0; q < 8; ++q) conn[8 * e + q] = m.E[e][q];
    for (std::size_t b = 0; b < m.bfaces.size(); ++b) {
      bf_elem[b] = m.bfaces[b].elem;
      bf_face[b] = m.bfaces[b].face;
      bf_tag[b] = static_cast<uint8_t>(m.bfaces[b].tag);
    }
  });
}

int orc_export_maps(void* hp, int32_t* l2g, int64_t* off, int32_t* ge, int32_t* gl, int32_t* sub, uint8_t* mask)
{
  return guard([&] {
    const Maps& M = static_cast<System*>(hp)->maps;
    if (l2g) std::memcpy(l2g, M.l2g.data(), M.l2g.size() * 4);
    if (off) std::memcpy(off, M.g2l_off.data(), M.g2l_off.size() * 8);
    if (ge) std::memcpy(ge, M.g2l_elem.data(), M.g2l_elem.size() * 4);
    if (gl) std::memcpy(gl, M.g2l_local.data(), M.g2l_local.size() * 4);
    if (sub) std::memcpy(sub, M.sub.data(), M.sub.size() * 4);
    if (mask) std::memcpy(mask, M.mask.data(), M.mask.size());
  });
}

int orc_apply_A(void* hp, const double* u, double* r)
{
  return guard([&] { apply_A(*static_cast<System*>(hp), u, r); });
}

int orc_apply_P(void* hp, const double* r, double* z)
{
  return guard([&] { apply_P(*static_cast<System*>(hp), r, z); });
}

int orc_apply_fine(void* hp, const double* r, double* z)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    if (!S.has_fine) throw BadInput("system has no fine preconditioner");
    apply_fine(S, r, z);
  });
}

int orc_apply_coarse(void* hp, const double* r, double* z)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    if (!S.has_coarse) throw BadInput("system has no coarse preconditioner");
    apply_coarse(S, r, z);
  });
}

int orc_restrict(void* hp, const double* r, double* R)
{
  return guard([&] {
    Vec out;
    restrict_res(*static_cast<System*>(hp), r, out);
    std::copy(out.begin(), out.end(), R);
  });
}

int orc_prolongate(void* hp, const double* Z, double* z)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    prolong(S, Vec(Z, Z + S.mesh.nv()), z);
  });
}

int orc_lumped_mass(void* hp, double* m)
{
  return guard([&] {
    const Vec& l = static_cast<System*>(hp)->lumped;
    std::copy(l.begin(), l.end(), m);
  });
}

// assemble_load with s = 1 (problem.cpp:38-46): b = m_N, 0 on the mask
int orc_load_ones(void* hp, double* b)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    for (i32 g = 0; g < S.N(); ++g) b[g] = S.maps.mask[g] ? 0.0 : S.lumped[g] * 1.0;
  });
}

int orc_coarse_matrix(void* hp, int64_t* nnz, int64_t* ptr, int32_t* col, double* val)
{
  return guard([&] {
    const Csr& K = static_cast<System*>(hp)->Kc;
    *nnz = static_cast<int64_t>(K.val.size());
    if (!ptr) return;
    std::memcpy(ptr, K.ptr.data(), K.ptr.size() * 8);
    std::memcpy(col, K.col.data(), K.col.size() * 4);
    std::memcpy(val, K.val.data(), K.val.size() * 8);
  });
}

int orc_amg_level(void* hp, int l, int64_t* rows, int64_t* nnz, int64_t* ptr, int32_t* col, double* val,
                  int32_t* agg)
{
  return guard([&] {
    const System& S = *static_cast<System*>(hp);
    if (!S.use_amg) throw BadInput("coarse solve is not AMG");
    const int L = static_cast<int>(S.amg.lv.size());
    if (l < 0 || l > L) throw BadInput("level out of range");
    const Csr& A = l < L ? S.amg.lv[l].A : S.amg.coarsest;
    *rows = A.n;
    *nnz = static_cast<int64_t>(A.val.size());
    if (ptr) {
      std::memcpy(ptr, A.ptr.data(), A.ptr.size() * 8);
      std::memcpy(col, A.col.data(), A.col.size() * 4);
      std::memcpy(val, A.val.data(), A.val.size() * 8);
    }
    if (agg && l < L) std::memcpy(agg, S.amg.lv[l].agg.data(), S.amg.lv[l].agg.size() * 4);
  });
}

int orc_pcg(void* hp, const double* b, double tol, int max_iterations, int* iterations, int* status,
            double* residual_history, double* zr_history, double* u, double* solve_seconds)
{
  return guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    pcg(*static_cast<System*>(hp), b, tol, max_iterations, iterations, status, residual_history, zr_history, u);
    if (solve_seconds) *solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int orc_gll(int n, double* nodes, double* weights, double* deriv, double* vdm)
{
  return guard([&] {
    const Basis b = make_basis(n);
    std::copy(b.t.begin(), b.t.end(), nodes);
    std::copy(b.w.begin(), b.w.end(), weights);
    std::copy(b.D.begin(), b.D.end(), deriv);
    if (vdm) std::copy(b.B.begin(), b.B.end(), vdm);
  });
}

int orc_pencil(int n, double* K, double* M, double* V, double* Vinv, double* lambda)
{
  return guard([&] {
    const Pencil P = make_pencil(make_basis(n));
    std::copy(P.K.begin(), P.K.end(), K);
    std::copy(P.M.begin(), P.M.end(), M);
    std::copy(P.V.begin(), P.V.end(), V);
    std::copy(P.Vi.begin(), P.Vi.end(), Vinv);
    std::copy(P.lam.begin(), P.lam.end(), lambda);
  });
}

int orc_element_h(void* hp, double* h3)
{
  return guard([&] {
    const Mesh& m = static_cast<System*>(hp)->mesh;
    for (i32 e = 0; e < m.ne(); ++e) {
      const auto h = elem_h(m, e);
      for (int d = 0; d < 3; ++d) h3[3 * e + d] = h[d];
    }
  });
}

// KernelCounters / FineCounters models (operator.cpp:20-37, fine.cpp:82-92)
unsigned long long orc_words_model(long long ne, int n, int variant)
{
  return static_cast<unsigned long long>(ne) * ((variant == 0 ? 10 : 3) * upow(n + 1, 3) + upow(n + 1, 2) + 2);
}
unsigned long long orc_flops_model(long long ne, int n)
{
  return static_cast<unsigned long long>(ne) * (12 * upow(n + 1, 4) + 18 * upow(n + 1, 3));
}
unsigned long long orc_fine_ops_model(long long ne, int n)
{
  return static_cast<unsigned long long>(ne) * (6 * upow(n + 3, 4) + 15 * upow(n + 3, 3));
}
unsigned long long orc_fine_words_model(long long ne, int n)
{
  return static_cast<unsigned long long>(ne) * (3 * upow(n + 3, 3) + 4 * upow(n + 3, 2));
}

}  // extern "C"
