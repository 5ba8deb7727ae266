// Sparse direct coarse solve: geometric nested dissection + supernodal
// (multifrontal) Cholesky of the coupled block of K_c, for the reference's
// direct path (SimplicialLLT, coarse.cpp:112-127 and 201-206, taken when the
// coarse grid has <= 64000 vertices). The factor is O(n^{4/3}) instead of
// the dense inverse's O(n^2) (12 GB at 54,872 unknowns), and the device
// triangular solves run level by level over the separator tree
// (kernels_coarse.cuh: nd_fwd_*/nd_bwd_*), every sum in a fixed order.
//
// Ordering: recursive median bisection of the vertex coordinates along the
// longest axis; the separator is the set of lower-half vertices with a
// neighbour in the upper half; leaves stop at kNdLeaf vertices. Supernodes
// are numbered in postorder (children first), each owning a contiguous
// column range of the permuted matrix.
// Numeric: for each supernode s (postorder) the front
//   F = [A_ss + upd ; A_ts + upd] over columns V_s and rows V_s u struct(s)
// is assembled (children's update matrices extend-added in child order),
// then L11 = chol(F11), L21 = F21 L11^-T, U_s = F22 - L21 L21^T. Stored for
// the device: L11^-1 (so each diagonal solve is a GEMV) and L21.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>

#include "setup.hpp"

namespace hxb {

namespace {

constexpr int kNdLeaf = 96;

struct NdBuilder {
  const std::vector<std::vector<int>>& adj;
  const std::vector<std::array<double, 3>>& xyz;
  std::vector<NdSupernode>& sn;
  std::vector<int> side;
  NdBuilder(const std::vector<std::vector<int>>& a, const std::vector<std::array<double, 3>>& x,
            std::vector<NdSupernode>& s)
      : adj(a), xyz(x), sn(s), side(a.size(), -1)
  {
  }

  // returns the supernode index; vertices listed in `verts` (original ids)
  int build(std::vector<int> verts, int depth)
  {
    if (static_cast<int>(verts.size()) <= kNdLeaf || depth > 40) {
      NdSupernode s;
      s.verts = std::move(verts);
      sn.push_back(std::move(s));
      return static_cast<int>(sn.size()) - 1;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int v : verts)
      for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], xyz[v][d]), hi[d] = std::max(hi[d], xyz[v][d]);
    int axis = 0;
    for (int d = 1; d < 3; ++d)
      if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
    const std::size_t half = verts.size() / 2;
    std::nth_element(verts.begin(), verts.begin() + half, verts.end(), [&](int a, int b) {
      return xyz[a][axis] < xyz[b][axis] || (xyz[a][axis] == xyz[b][axis] && a < b);
    });
    std::vector<int> left(verts.begin(), verts.begin() + half), right(verts.begin() + half, verts.end());
    for (int v : left) side[v] = 0;
    for (int v : right) side[v] = 1;
    std::vector<int> sep, lrest;
    for (int v : left) {
      bool touches = false;
      for (int w : adj[v])
        if (side[w] == 1) {
          touches = true;
          break;
        }
      (touches ? sep : lrest).push_back(v);
    }
    for (int v : verts) side[v] = -1;
    std::sort(sep.begin(), sep.end());
    const int a = build(std::move(lrest), depth + 1);
    const int b = build(std::move(right), depth + 1);
    NdSupernode s;
    s.verts = std::move(sep);
    s.children = {a, b};
    sn.push_back(std::move(s));
    return static_cast<int>(sn.size()) - 1;
  }
};

// dense Cholesky of the leading m x m block of F (row-major, ld f), lower
bool chol_inplace(double* F, int m, int f)
{
  for (int j = 0; j < m; ++j) {
    double* Fj = F + static_cast<std::size_t>(j) * f;
    double d = Fj[j];
    for (int k = 0; k < j; ++k) d -= Fj[k] * Fj[k];
    if (!(d > 0)) return false;
    const double ljj = std::sqrt(d);
    Fj[j] = ljj;
    const double inv = 1.0 / ljj;
    for (int i = j + 1; i < m; ++i) {
      double* Fi = F + static_cast<std::size_t>(i) * f;
      double s = Fi[j];
      for (int k = 0; k < j; ++k) s -= Fi[k] * Fj[k];
      Fi[j] = s * inv;
    }
  }
  return true;
}

}  // namespace

NdFactor nd_cholesky(const Csr& A, const std::vector<std::array<double, 3>>& xyz)
{
  const int n = A.n;
  NdFactor F;
  F.n = n;
  std::vector<std::vector<int>> adj(n);
  for (int i = 0; i < n; ++i)
    for (std::int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q)
      if (A.col[q] != i) adj[i].push_back(A.col[q]);
  {
    std::vector<int> all(n);
    std::iota(all.begin(), all.end(), 0);
    NdBuilder b(adj, xyz, F.sn);
    b.build(std::move(all), 0);
  }
  // postorder = creation order (children are created before their parent)
  const int ns = static_cast<int>(F.sn.size());
  F.perm.assign(n, -1);  // new index -> original row
  std::vector<int> inew(n, -1);
  int col = 0;
  for (int s = 0; s < ns; ++s) {
    NdSupernode& S = F.sn[s];
    S.c0 = col;
    for (int v : S.verts) {
      inew[v] = col;
      F.perm[col++] = v;
    }
    S.c1 = col;
    for (int c : S.children) F.sn[c].parent = s;
  }
  // symbolic: struct(s) = (A rows below + children's structs) beyond column c1
  for (int s = 0; s < ns; ++s) {
    NdSupernode& S = F.sn[s];
    std::vector<int> rows;
    for (int v : S.verts)
      for (int w : adj[v])
        if (inew[w] >= S.c1) rows.push_back(inew[w]);
    for (int c : S.children)
      for (int r : F.sn[c].rows)
        if (r >= S.c1) rows.push_back(r);
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
    S.rows = std::move(rows);
  }
  // levels (leaves 0): a supernode's level is 1 + max over its children
  F.levels = 0;
  for (int s = 0; s < ns; ++s) {
    int lv = 0;
    for (int c : F.sn[s].children) lv = std::max(lv, F.sn[c].level + 1);
    F.sn[s].level = lv;
    F.levels = std::max(F.levels, lv + 1);
  }
  // numeric multifrontal, one level at a time (supernodes of a level in parallel)
  std::vector<std::vector<double>> upd(ns);  // update matrix of each supernode (r x r, row-major, lower)
  std::vector<std::vector<int>> by_level(F.levels);
  for (int s = 0; s < ns; ++s) by_level[F.sn[s].level].push_back(s);
  bool ok = true;
  const int nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (int lv = 0; lv < F.levels && ok; ++lv) {
    const std::vector<int>& list = by_level[lv];
    std::vector<char> good(list.size(), 1);
    auto work = [&](int t) {
      for (std::size_t q = t; q < list.size(); q += nthreads) {
        const int s = list[q];
        NdSupernode& S = F.sn[s];
        const int m = S.c1 - S.c0, r = static_cast<int>(S.rows.size()), f = m + r;
        std::vector<double> Fr(static_cast<std::size_t>(f) * f, 0.0);
        auto pos = [&](int g) {  // front position of permuted row g (g >= c0)
          if (g < S.c1) return g - S.c0;
          return m + static_cast<int>(std::lower_bound(S.rows.begin(), S.rows.end(), g) - S.rows.begin());
        };
        for (int j = 0; j < m; ++j) {
          const int v = F.perm[S.c0 + j];
          for (std::int64_t k = A.ptr[v]; k < A.ptr[v + 1]; ++k) {
            const int g = inew[A.col[k]];
            if (g < S.c0 + j) continue;  // lower triangle: rows at or after this column
            Fr[static_cast<std::size_t>(pos(g)) * f + j] += A.val[k];
          }
        }
        for (int c : S.children) {  // extend-add, child order
          const NdSupernode& C = F.sn[c];
          const int rc = static_cast<int>(C.rows.size());
          std::vector<int> map(rc);
          for (int i = 0; i < rc; ++i) map[i] = pos(C.rows[i]);
          const std::vector<double>& U = upd[c];
          for (int i = 0; i < rc; ++i)
            for (int j = 0; j <= i; ++j) Fr[static_cast<std::size_t>(map[i]) * f + map[j]] += U[static_cast<std::size_t>(i) * rc + j];
        }
        for (int c : S.children) std::vector<double>().swap(upd[c]);
        if (!chol_inplace(Fr.data(), m, f)) {
          good[q] = 0;
          continue;
        }
        // L21 = F21 L11^-T (row by row forward substitution)
        for (int i = m; i < f; ++i) {
          double* Fi = Fr.data() + static_cast<std::size_t>(i) * f;
          for (int j = 0; j < m; ++j) {
            const double* Fj = Fr.data() + static_cast<std::size_t>(j) * f;
            double s2 = Fi[j];
            for (int k = 0; k < j; ++k) s2 -= Fi[k] * Fj[k];
            Fi[j] = s2 / Fj[j];
          }
        }
        // U = F22 - L21 L21^T (lower)
        std::vector<double>& U = upd[s];
        U.assign(static_cast<std::size_t>(r) * r, 0.0);
        for (int i = 0; i < r; ++i) {
          const double* Li = Fr.data() + static_cast<std::size_t>(m + i) * f;
          for (int j = 0; j <= i; ++j) {
            const double* Lj = Fr.data() + static_cast<std::size_t>(m + j) * f;
            double s2 = Fr[static_cast<std::size_t>(m + i) * f + m + j];
            for (int k = 0; k < m; ++k) s2 -= Li[k] * Lj[k];
            U[static_cast<std::size_t>(i) * r + j] = s2;
          }
        }
        // L11^-1 (lower) and L21, row-major
        S.linv.assign(static_cast<std::size_t>(m) * m, 0.0);
        for (int i = 0; i < m; ++i) {  // row i of X = L11^-1: (e_i - sum_k<i L_ik X_k) / L_ii, row axpys
          double* Xi = S.linv.data() + static_cast<std::size_t>(i) * m;
          const double* Fi = Fr.data() + static_cast<std::size_t>(i) * f;
          Xi[i] = 1.0;
          for (int k = 0; k < i; ++k) {
            const double lik = Fi[k];
            const double* Xk = S.linv.data() + static_cast<std::size_t>(k) * m;
            for (int c2 = 0; c2 <= k; ++c2) Xi[c2] -= lik * Xk[c2];
          }
          const double inv = 1.0 / Fi[i];
          for (int c2 = 0; c2 <= i; ++c2) Xi[c2] *= inv;
        }
        S.l21.resize(static_cast<std::size_t>(r) * m);
        for (int i = 0; i < r; ++i)
          std::copy(Fr.begin() + static_cast<std::size_t>(m + i) * f, Fr.begin() + static_cast<std::size_t>(m + i) * f + m,
                    S.l21.begin() + static_cast<std::size_t>(i) * m);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& t : th) t.join();
    for (char g : good) ok = ok && g;
  }
  if (!ok) throw HxbError(3, "coarse matrix Cholesky failed (matrix not SPD?)");
  return F;
}

// Host replay of the device solve (nd_* kernels): x = A^-1 b for the
// factored matrix, same recurrences, for GPU-free checks of the factor.
std::vector<double> nd_solve_host(const NdFactor& F, const std::vector<double>& b)
{
  const int n = F.n, ns = static_cast<int>(F.sn.size());
  std::vector<double> y(n), z(n), t(n), x(n);
  for (int i = 0; i < n; ++i) y[i] = b[F.perm[i]];
  std::vector<std::vector<double>> acc(ns);
  for (int s = 0; s < ns; ++s) {  // postorder = forward order
    const NdSupernode& S = F.sn[s];
    const int m = S.c1 - S.c0, r = static_cast<int>(S.rows.size());
    std::vector<double> ye(y.begin() + S.c0, y.begin() + S.c1);
    acc[s].assign(r, 0.0);
    for (int c : S.children) {
      const NdSupernode& C = F.sn[c];
      for (std::size_t i = 0; i < C.rows.size(); ++i) {
        const int g = C.rows[i];
        if (g < S.c1)
          ye[g - S.c0] -= acc[c][i];
        else
          acc[s][std::lower_bound(S.rows.begin(), S.rows.end(), g) - S.rows.begin()] += acc[c][i];
      }
    }
    for (int j = 0; j < m; ++j) {
      double v = 0;
      for (int k = 0; k <= j; ++k) v += S.linv[static_cast<std::size_t>(j) * m + k] * ye[k];
      z[S.c0 + j] = v;
    }
    for (int i = 0; i < r; ++i)
      for (int k = 0; k < m; ++k) acc[s][i] += S.l21[static_cast<std::size_t>(i) * m + k] * z[S.c0 + k];
  }
  for (int s = ns - 1; s >= 0; --s) {
    const NdSupernode& S = F.sn[s];
    const int m = S.c1 - S.c0, r = static_cast<int>(S.rows.size());
    for (int j = 0; j < m; ++j) {
      double v = z[S.c0 + j];
      for (int i = 0; i < r; ++i) v -= S.l21[static_cast<std::size_t>(i) * m + j] * x[S.rows[i]];
      t[S.c0 + j] = v;
    }
    for (int j = 0; j < m; ++j) {
      double v = 0;
      for (int k = j; k < m; ++k) v += S.linv[static_cast<std::size_t>(k) * m + j] * t[S.c0 + k];
      x[S.c0 + j] = v;
    }
  }
  std::vector<double> out(n);
  for (int i = 0; i < n; ++i) out[F.perm[i]] = x[i];
  return out;
}

}  // namespace hxb
