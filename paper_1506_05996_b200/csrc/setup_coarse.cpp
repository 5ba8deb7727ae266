// FDM pencil, Q1 coarse matrix and aggregation-AMG setup (host, native C++).
//
//   build_pencil                 fine.cpp:15-80 (own cyclic-Jacobi eigen-solve
//                                replaces Eigen::SelfAdjointEigenSolver)
//   csr_from_triplets            amg.cpp:22-40
//   coarse_dirichlet_mask        coarse.cpp:11-19
//   assemble_coarse_matrix       coarse.cpp:21-87
//   aggregate_pass / galerkin    amg.cpp:53-122
//   AmgHierarchy::Impl::setup    amg.cpp:151-186
//
// The AMG hierarchy must match the reference bit-for-bit (aggregation compares
// |a_ij| with ties broken by column), so triplet sums use the same container
// type, comparator and std::sort as the reference, giving the same order of
// duplicate summation.
#include <algorithm>
#include <cmath>

#include "setup.hpp"
#include "setup_parallel.hpp"

namespace hxb {

// ---------------------------------------------------------------------------
namespace {

// Cyclic Jacobi for a small symmetric matrix (row-major); eigenvalues
// ascending, eigenvectors as unit columns of Q (row-major q[r*n+c]).
void symmetric_eigen(int n, std::vector<double> A, std::vector<double>& lambda, std::vector<double>& Q)
{
  std::vector<double> V(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[static_cast<std::size_t>(i) * n + j]; };
  auto v = [&](int i, int j) -> double& { return V[static_cast<std::size_t>(i) * n + j]; };
  bool ok = false;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, diag = 0;
    for (int i = 0; i < n; ++i) {
      diag += a(i, i) * a(i, i);
      for (int j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
    }
    if (off <= 1e-34 * diag || off == 0.0) {
      ok = true;
      break;
    }
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  if (!ok) throw HxbError(3, "pencil eigen-solve did not converge");
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return a(x, x) < a(y, y); });
  lambda.resize(n);
  Q.assign(static_cast<std::size_t>(n) * n, 0.0);
  for (int c = 0; c < n; ++c) {
    lambda[c] = a(order[c], order[c]);
    for (int r = 0; r < n; ++r) Q[static_cast<std::size_t>(r) * n + c] = v(r, order[c]);
  }
}

}  // namespace

Pencil build_pencil(const GllBasis& basis)
{
  const int n = basis.order, np = n + 1, p = n + 3;
  std::vector<double> d(static_cast<std::size_t>(np) * np, 0.0);
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      double s = 0;
      for (int m = 0; m < np; ++m) s += basis.d(i, m) * basis.d(j, m) * basis.weights[m];
      d[static_cast<std::size_t>(i) * np + j] = s;
    }
  Pencil out;
  out.p = p;
  out.K.assign(static_cast<std::size_t>(p) * p, 0.0);
  out.M.assign(p, 0.0);
  for (int o = -2; o <= 2; ++o)
    for (int a = 0; a <= n; ++a) {
      const int pa = o * n + a;
      if (pa < -1 || pa > n + 1) continue;
      out.M[pa + 1] += basis.weights[a];
      for (int b = 0; b <= n; ++b) {
        const int pb = o * n + b;
        if (pb < -1 || pb > n + 1) continue;
        out.K[static_cast<std::size_t>(pa + 1) * p + (pb + 1)] += d[static_cast<std::size_t>(a) * np + b];
      }
    }
  std::vector<double> S(static_cast<std::size_t>(p) * p), Ssym(S.size());
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      S[static_cast<std::size_t>(i) * p + j] = out.K[static_cast<std::size_t>(i) * p + j] / std::sqrt(out.M[i] * out.M[j]);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      Ssym[static_cast<std::size_t>(i) * p + j] = 0.5 * (S[static_cast<std::size_t>(i) * p + j] + S[static_cast<std::size_t>(j) * p + i]);
  std::vector<double> Q;
  symmetric_eigen(p, Ssym, out.lambda, Q);
  for (int i = 0; i < p; ++i)
    if (!(out.lambda[i] > 0))
      throw HxbError(3, "pencil eigenvalue " + std::to_string(i) + " is not positive for order " + std::to_string(n));
  out.V.resize(static_cast<std::size_t>(p) * p);
  out.V_inv.resize(static_cast<std::size_t>(p) * p);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      out.V[static_cast<std::size_t>(i) * p + j] = Q[static_cast<std::size_t>(j) * p + i] * std::sqrt(out.M[j]);
      out.V_inv[static_cast<std::size_t>(i) * p + j] = Q[static_cast<std::size_t>(i) * p + j] / std::sqrt(out.M[i]);
    }
  return out;
}

// ---------------------------------------------------------------------------
namespace {
using RefTrip = std::pair<std::pair<gid, gid>, double>;

Csr csr_from_reftrips(gid n, std::vector<RefTrip> trips)
{
  // the reference's std::sort (amg.cpp:28), equal keys left in its order (setup_parallel.hpp)
  std_sort_threads(trips.begin(), trips.end(), [](const RefTrip& a, const RefTrip& b) { return a.first < b.first; });
  Csr m;
  m.n = n;
  m.ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  m.col.reserve(trips.size() / 2);
  m.val.reserve(trips.size() / 2);
  for (std::size_t i = 0; i < trips.size();) {
    std::size_t j = i;
    double s = 0;
    while (j < trips.size() && trips[j].first == trips[i].first) s += trips[j++].second;
    m.ptr[static_cast<std::size_t>(trips[i].first.first) + 1]++;
    m.col.push_back(trips[i].first.second);
    m.val.push_back(s);
    i = j;
  }
  for (gid i = 0; i < n; ++i) m.ptr[i + 1] += m.ptr[i];
  return m;
}
}  // namespace

Csr csr_from_triplets(gid n, std::vector<Triplet> t)
{
  std::vector<RefTrip> r(t.size());
  for (std::size_t i = 0; i < t.size(); ++i) r[i] = {{t[i].r, t[i].c}, t[i].v};
  return csr_from_reftrips(n, std::move(r));
}

std::vector<std::uint8_t> coarse_dirichlet_mask(const HexMesh& mesh)
{
  std::vector<std::uint8_t> mask(mesh.num_vertices(), 0);
  for (const auto& bf : mesh.boundary_faces) {
    if (bf.tag != 0) continue;
    for (int c : face_corners(bf.face)) mask[mesh.elements[bf.element][c]] = 1;
  }
  return mask;
}

Csr assemble_coarse_matrix(const HexMesh& mesh, const std::vector<double>& kappa, const std::vector<double>& c,
                           const std::vector<std::uint8_t>& vmask)
{
  const gid nv = mesh.num_vertices();
  const gid ne = mesh.num_elements();
  // element matrices on host threads (independent), then the triplets in
  // element order exactly as the reference's single loop appends them
  std::vector<double> kall(static_cast<std::size_t>(ne) * 64);
  parallel_for(ne, [&](gid e_begin, gid e_end) {
  for (gid e = e_begin; e < e_end; ++e) {
    double ke[8][8] = {};
    for (int qb = 0; qb < 8; ++qb) {
      const double xi = (qb & 1) ? 1.0 : -1.0;
      const double eta = (qb & 2) ? 1.0 : -1.0;
      const double zeta = (qb & 4) ? 1.0 : -1.0;
      const Jacobian jac = jacobian(mesh, e, xi, eta, zeta);
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
      double grad[8][3];
      const double hq[3][2] = {{(qb & 1) ? 0.0 : 1.0, (qb & 1) ? 1.0 : 0.0},
                               {(qb & 2) ? 0.0 : 1.0, (qb & 2) ? 1.0 : 0.0},
                               {(qb & 4) ? 0.0 : 1.0, (qb & 4) ? 1.0 : 0.0}};
      for (int ab = 0; ab < 8; ++ab) {
        const int bi = ab & 1, bj = (ab >> 1) & 1, bk = (ab >> 2) & 1;
        const double dhat[3] = {(bi ? 0.5 : -0.5) * hq[1][bj] * hq[2][bk],
                                hq[0][bi] * (bj ? 0.5 : -0.5) * hq[2][bk],
                                hq[0][bi] * hq[1][bj] * (bk ? 0.5 : -0.5)};
        for (int d = 0; d < 3; ++d)
          grad[ab][d] = inv[0 * 3 + d] * dhat[0] + inv[1 * 3 + d] * dhat[1] + inv[2 * 3 + d] * dhat[2];
      }
      const double mq = jac.det;
      for (int ab = 0; ab < 8; ++ab)
        for (int bb = 0; bb < 8; ++bb) {
          double s = kappa[e] * (grad[ab][0] * grad[bb][0] + grad[ab][1] * grad[bb][1] + grad[ab][2] * grad[bb][2]);
          if (ab == bb && ab == qb) s += c[e];
          ke[ab][bb] += mq * s;
        }
    }
    std::copy(&ke[0][0], &ke[0][0] + 64, kall.begin() + static_cast<std::size_t>(e) * 64);
  }
  });
  std::vector<RefTrip> trips;
  trips.reserve(static_cast<std::size_t>(ne) * 64);
  for (gid e = 0; e < ne; ++e) {
    const double* ke = kall.data() + static_cast<std::size_t>(e) * 64;
    for (int ab = 0; ab < 8; ++ab) {
      const gid ga = mesh.elements[e][hex_corner(ab & 1, (ab >> 1) & 1, (ab >> 2) & 1)];
      for (int bb = 0; bb < 8; ++bb) {
        const gid gb = mesh.elements[e][hex_corner(bb & 1, (bb >> 1) & 1, (bb >> 2) & 1)];
        if (vmask[ga] || vmask[gb]) continue;
        trips.push_back({{ga, gb}, ke[ab * 8 + bb]});
      }
    }
  }
  for (gid v = 0; v < nv; ++v)
    if (vmask[v]) trips.push_back({{v, v}, 1.0});
  return csr_from_reftrips(nv, std::move(trips));
}

// ---------------------------------------------------------------------------
namespace {
constexpr gid kCoarsestSize = 64;
constexpr int kAggregateTarget = 8;

gid aggregate_pass(const Csr& A, std::vector<gid>& group)
{
  group.assign(A.n, -1);
  gid next = 0;
  std::vector<int> agg_size;
  std::vector<std::pair<double, gid>> nbrs;
  for (gid i = 0; i < A.n; ++i) {
    if (group[i] >= 0) continue;
    bool clean = true;
    nbrs.clear();
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const gid j = A.col[k];
      if (j == i || A.val[k] == 0.0) continue;
      if (group[j] >= 0) {
        clean = false;
        break;
      }
      nbrs.push_back({-std::abs(A.val[k]), j});
    }
    if (!clean) continue;
    group[i] = next;
    std::sort(nbrs.begin(), nbrs.end());
    int size = 1;
    for (const auto& [neg, j] : nbrs) {
      if (size >= kAggregateTarget) break;
      group[j] = next;
      ++size;
    }
    agg_size.push_back(size);
    ++next;
  }
  for (gid i = 0; i < A.n; ++i) {
    if (group[i] >= 0) continue;
    gid best = -1;
    double best_val = 0;
    bool best_small = false;
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const gid j = A.col[k];
      if (j == i || group[j] < 0 || A.val[k] == 0.0) continue;
      const double a = std::abs(A.val[k]);
      const bool small = agg_size[group[j]] < kAggregateTarget;
      if (best < 0 || (small && !best_small) || (small == best_small && a > best_val)) {
        best = group[j];
        best_val = a;
        best_small = small;
      }
    }
    if (best >= 0) {
      group[i] = best;
      ++agg_size[best];
    } else {
      group[i] = next;
      agg_size.push_back(1);
      ++next;
    }
  }
  return next;
}

Csr galerkin(const Csr& A, const std::vector<gid>& agg, gid nc)
{
  std::vector<RefTrip> trips;
  trips.reserve(A.nnz());
  for (gid i = 0; i < A.n; ++i)
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) trips.push_back({{agg[i], agg[A.col[k]]}, A.val[k]});
  return csr_from_reftrips(nc, std::move(trips));
}

void check_diag(const Csr& A, std::vector<double>& inv_diag)
{
  inv_diag.assign(A.n, 0.0);
  for (gid i = 0; i < A.n; ++i) {
    double d = 0;
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] == i) d = A.val[k];
    if (!(d > 0)) throw HxbError(3, "amg: non-positive diagonal at row " + std::to_string(i));
    inv_diag[i] = 1 / d;
  }
}
}  // namespace

AmgSetup amg_setup(Csr fine)
{
  AmgSetup out;
  Csr A = std::move(fine);
  while (A.n > kCoarsestSize) {
    AmgLevel lvl;
    check_diag(A, lvl.inv_diag);
    std::vector<gid> agg;
    const gid nc = aggregate_pass(A, agg);
    if (nc > static_cast<gid>(0.95 * A.n)) break;
    Csr coarse = galerkin(A, agg, nc);
    lvl.aggregate = std::move(agg);
    lvl.n_coarse = nc;
    lvl.A = std::move(A);
    A = std::move(coarse);
    out.levels.push_back(std::move(lvl));
  }
  out.coarsest = std::move(A);
  std::vector<double> tmp;
  check_diag(out.coarsest, tmp);
  return out;
}

// ---------------------------------------------------------------------------
DenseCoarse dense_coarse_setup(const Csr& A, int host_inverse_limit)
{
  DenseCoarse dc;
  dc.n = A.n;
  dc.inv_diag.assign(A.n, 0.0);
  std::vector<gid> pos(A.n, -1);
  for (gid i = 0; i < A.n; ++i) {
    bool coupled = false;
    double d = 0;
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      if (A.col[k] == i)
        d = A.val[k];
      else
        coupled = true;
    }
    if (coupled) {
      pos[i] = static_cast<gid>(dc.coupled.size());
      dc.coupled.push_back(i);
    } else {
      if (!(d > 0)) throw HxbError(3, "coarse matrix Cholesky failed (matrix not SPD?)");
      dc.inv_diag[i] = 1.0 / d;
    }
  }
  const std::size_t m = dc.coupled.size();
  if (static_cast<long>(m) > host_inverse_limit) {
    // large block: hand its sparse rows to the device factorization (no m^2 host array)
    dc.csr_ptr.assign(1, 0);
    for (std::size_t r = 0; r < m; ++r) {
      const gid i = dc.coupled[r];
      for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const gid j = A.col[k];
        if (pos[j] < 0) throw HxbError(3, "coarse matrix is not structurally symmetric");
        dc.csr_col.push_back(pos[j]);
        dc.csr_val.push_back(A.val[k]);
      }
      dc.csr_ptr.push_back(static_cast<std::int64_t>(dc.csr_col.size()));
    }
    return dc;
  }
  dc.coupled_a.assign(m * m, 0.0);
  for (std::size_t r = 0; r < m; ++r) {
    const gid i = dc.coupled[r];
    for (std::int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const gid j = A.col[k];
      if (pos[j] < 0) throw HxbError(3, "coarse matrix is not structurally symmetric");
      dc.coupled_a[r * m + pos[j]] += A.val[k];
    }
  }
  if (static_cast<long>(m) <= host_inverse_limit) {
    // Cholesky A = L L^T then A^-1 = L^-T L^-1, all host-side, small m only.
    std::vector<double> L = dc.coupled_a;
    for (std::size_t j = 0; j < m; ++j) {
      double d = L[j * m + j];
      for (std::size_t k = 0; k < j; ++k) d -= L[j * m + k] * L[j * m + k];
      if (!(d > 0)) throw HxbError(3, "coarse matrix Cholesky failed (matrix not SPD?)");
      const double ljj = std::sqrt(d);
      L[j * m + j] = ljj;
      for (std::size_t i = j + 1; i < m; ++i) {
        double s = L[i * m + j];
        for (std::size_t k = 0; k < j; ++k) s -= L[i * m + k] * L[j * m + k];
        L[i * m + j] = s / ljj;
      }
    }
    // W = L^-1 (lower), then Ainv = W^T W
    std::vector<double> W(m * m, 0.0);
    for (std::size_t c = 0; c < m; ++c) {
      for (std::size_t i = c; i < m; ++i) {
        double s = (i == c) ? 1.0 : 0.0;
        for (std::size_t k = c; k < i; ++k) s -= L[i * m + k] * W[k * m + c];
        W[i * m + c] = s / L[i * m + i];
      }
    }
    dc.ainv.assign(m * m, 0.0);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j <= i; ++j) {
        double s = 0;
        for (std::size_t k = i; k < m; ++k) s += W[k * m + i] * W[k * m + j];
        dc.ainv[i * m + j] = s;
        dc.ainv[j * m + i] = s;
      }
  }
  return dc;
}

// ---------------------------------------------------------------------------
// Envelope (profile) Cholesky after a reverse Cuthill-McKee ordering: the
// factorisation behind the reference's SimplicialLLT direct coarse solves
// (coarse.cpp:117-127, amg.cpp:176-194) as built in this environment (Eigen is
// absent from the image and unpinned by the reference; the test build of the
// reference, oracle/_ref, links the profile-Cholesky SimplicialLLT of
// oracle/eigen_shim). Used by the bitwise-reference plans, whose device solve
// replays the same row-bordering recurrences in the same order.
EnvelopeFactor envelope_cholesky(const Csr& A)
{
  const std::int64_t n = A.n;
  EnvelopeFactor f;
  f.n = A.n;
  // graph of the strictly lower entries, both directions, sorted and unique
  std::vector<std::vector<std::int64_t>> nbr(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q)
      if (A.col[q] < i) {
        nbr[i].push_back(A.col[q]);
        nbr[A.col[q]].push_back(i);
      }
  for (auto& l : nbr) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  auto deg_less = [&](std::int64_t x, std::int64_t y) { return nbr[x].size() < nbr[y].size(); };
  // Cuthill-McKee from min-degree seeds (ties in index order), reversed
  std::vector<std::int64_t> seeds(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) seeds[i] = i;
  std::stable_sort(seeds.begin(), seeds.end(), deg_less);
  std::vector<char> seen(static_cast<std::size_t>(n), 0);
  f.perm.clear();
  f.perm.reserve(static_cast<std::size_t>(n));
  for (std::int64_t seed : seeds) {
    if (seen[seed]) continue;
    seen[seed] = 1;
    std::size_t head = f.perm.size();
    f.perm.push_back(seed);
    while (head < f.perm.size()) {
      const std::int64_t v = f.perm[head++];
      std::vector<std::int64_t> fresh;
      for (std::int64_t w : nbr[v])
        if (!seen[w]) {
          seen[w] = 1;
          fresh.push_back(w);
        }
      std::stable_sort(fresh.begin(), fresh.end(), deg_less);
      f.perm.insert(f.perm.end(), fresh.begin(), fresh.end());
    }
  }
  std::reverse(f.perm.begin(), f.perm.end());
  std::vector<std::int64_t> inv(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) inv[f.perm[i]] = i;
  // profile of the permuted lower triangle, then its values
  f.first.resize(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) f.first[i] = i;
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q)
      if (A.col[q] <= i) {
        const std::int64_t a = inv[i], b = inv[A.col[q]];
        const std::int64_t row = std::max(a, b);
        f.first[row] = std::min(f.first[row], std::min(a, b));
      }
  f.start.assign(static_cast<std::size_t>(n) + 1, 0);
  for (std::int64_t i = 0; i < n; ++i) f.start[i + 1] = f.start[i] + (i - f.first[i] + 1);
  f.env.assign(static_cast<std::size_t>(f.start[n]), 0.0);
  auto L = [&](std::int64_t i, std::int64_t j) -> double& { return f.env[f.start[i] + (j - f.first[i])]; };
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q)
      if (A.col[q] <= i) {
        const std::int64_t a = inv[i], b = inv[A.col[q]];
        L(std::max(a, b), std::min(a, b)) += A.val[q];
      }
  // row-bordering factorisation: L_ij = (a_ij - sum_k L_ik L_jk) / L_jj
  for (std::int64_t i = 0; i < n; ++i) {
    for (std::int64_t j = f.first[i]; j < i; ++j) {
      double s = L(i, j);
      for (std::int64_t k = std::max(f.first[i], f.first[j]); k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / L(j, j);
    }
    double d = L(i, i);
    for (std::int64_t k = f.first[i]; k < i; ++k) d -= L(i, k) * L(i, k);
    if (!(d > 0)) throw HxbError(3, "coarse matrix Cholesky failed (matrix not SPD?)");
    L(i, i) = std::sqrt(d);
  }
  return f;
}

}  // namespace hxb
