// Device-side setup: the geometric factors of the stored
// operator, compute_factors (geometry.cpp:105-151) + the kappa*mass scaling
// of the SemOperator constructor (operator.cpp:76-88), one thread per local
// node. Every operation is an explicitly rounded IEEE intrinsic in the
// reference's evaluation order (its Release build has no FMA contraction),
// so the planes and the mass are bit-identical to the host restatement and
// to the reference, while taking milliseconds instead of seconds.
#pragma once

#include "kernels_common.cuh"

namespace hxb {

struct GeoArgs {
  double hat0[kMaxNP], hat1[kMaxNP], w[kMaxNP];  // 0.5(1 -+ t_i) and GLL weights, host-computed
  const double* xyz;                             // nv*3
  const int* conn;                               // ne*8, Gmsh corner order
  const double* kappa;                           // ne
  double* mass;                                  // [ne][nloc] (all elements)
  double* wg;                                    // [e - e0][6][nlocp] for e in [e0, e0 + nel), or null
  int ne, e0, nel, nlocp;
  int* bad;                                      // min inverted element (init INT_MAX)
};

template <int NP>
__global__ void __launch_bounds__(256) geometry_kernel(const __grid_constant__ GeoArgs a)
{
  constexpr int NL = NP * NP * NP;
  constexpr int kSlot[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // corner bits (bi,bj,bk) -> connectivity slot (mesh.hpp:31-33)
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(a.ne) * NL) return;
  const int e = static_cast<int>(t / NL), node = static_cast<int>(t % NL);
  const int i = node % NP, j = (node / NP) % NP, k = node / (NP * NP);
  const double h[3][2] = {{a.hat0[i], a.hat1[i]}, {a.hat0[j], a.hat1[j]}, {a.hat0[k], a.hat1[k]}};
  const double dh[2] = {-0.5, 0.5};
  double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int bk = 0; bk < 2; ++bk)  // jacobian (geometry.cpp:43-64)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) {
        const int v = __ldg(a.conn + 8LL * e + kSlot[bi + 2 * bj + 4 * bk]);
        const double wx = __dmul_rn(__dmul_rn(dh[bi], h[1][bj]), h[2][bk]);
        const double wy = __dmul_rn(__dmul_rn(h[0][bi], dh[bj]), h[2][bk]);
        const double wz = __dmul_rn(__dmul_rn(h[0][bi], h[1][bj]), dh[bk]);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double x = __ldg(a.xyz + 3LL * v + d);
          J[d * 3 + 0] = __dadd_rn(J[d * 3 + 0], __dmul_rn(wx, x));
          J[d * 3 + 1] = __dadd_rn(J[d * 3 + 1], __dmul_rn(wy, x));
          J[d * 3 + 2] = __dadd_rn(J[d * 3 + 2], __dmul_rn(wz, x));
        }
      }
  auto cof = [](double p, double q, double r, double s) { return __dsub_rn(__dmul_rn(p, q), __dmul_rn(r, s)); };
  const double det = __dadd_rn(__dsub_rn(__dmul_rn(J[0], cof(J[4], J[8], J[5], J[7])),
                                         __dmul_rn(J[1], cof(J[3], J[8], J[5], J[6]))),
                               __dmul_rn(J[2], cof(J[3], J[7], J[4], J[6])));
  if (!(det > 0)) {
    atomicMin(a.bad, e);
    return;
  }
  double inv[9];  // compute_factors (geometry.cpp:122-131)
  inv[0] = __ddiv_rn(cof(J[4], J[8], J[5], J[7]), det);
  inv[1] = __ddiv_rn(cof(J[2], J[7], J[1], J[8]), det);
  inv[2] = __ddiv_rn(cof(J[1], J[5], J[2], J[4]), det);
  inv[3] = __ddiv_rn(cof(J[5], J[6], J[3], J[8]), det);
  inv[4] = __ddiv_rn(cof(J[0], J[8], J[2], J[6]), det);
  inv[5] = __ddiv_rn(cof(J[2], J[3], J[0], J[5]), det);
  inv[6] = __ddiv_rn(cof(J[3], J[7], J[4], J[6]), det);
  inv[7] = __ddiv_rn(cof(J[1], J[6], J[0], J[7]), det);
  inv[8] = __ddiv_rn(cof(J[0], J[4], J[1], J[3]), det);
  const double m = __dmul_rn(__dmul_rn(__dmul_rn(a.w[i], a.w[j]), a.w[k]), det);
  a.mass[static_cast<long long>(e) * NL + node] = m;
  if (a.wg && e >= a.e0 && e < a.e0 + a.nel) {
    auto gt = [&](int r, int c) {
      return __dadd_rn(__dadd_rn(__dmul_rn(inv[r * 3], inv[c * 3]), __dmul_rn(inv[r * 3 + 1], inv[c * 3 + 1])),
                       __dmul_rn(inv[r * 3 + 2], inv[c * 3 + 2]));
    };
    const double scale = __dmul_rn(__ldg(a.kappa + e), m);  // operator.cpp:83-87
    double* o = a.wg + static_cast<long long>(e - a.e0) * 6 * a.nlocp + node;
    o[0] = __dmul_rn(gt(0, 0), scale);
    o[a.nlocp] = __dmul_rn(gt(0, 1), scale);
    o[2 * a.nlocp] = __dmul_rn(gt(0, 2), scale);
    o[3 * a.nlocp] = __dmul_rn(gt(1, 1), scale);
    o[4 * a.nlocp] = __dmul_rn(gt(1, 2), scale);
    o[5 * a.nlocp] = __dmul_rn(gt(2, 2), scale);
  }
}

// Subdomain slot -> global node of every element's (n+3)^3 FDM subdomain
// (sub_l2g, mesh.cpp:385-451; for_each_sub_slot order): own nodes from the
// surface codes / closed-form interior ids, face slots from the face-neighbour
// table, edge and corner slots -1. Dirichlet codes (-g-2) decode to g.
template <int NP>
__global__ void sub_keys_kernel(const int* __restrict__ smap, int sstride, const int* __restrict__ sub_face,
                                int sfstride, int ne, int nsg, int* __restrict__ keys)
{
  constexpr int n = NP - 1, P = NP + 2, P3 = P * P * P, NI = (n - 1) * (n - 1) * (n - 1);
  auto dec = [](int c) { return c >= 0 ? c : (c <= -2 ? -c - 2 : -1); };
  const long long total = static_cast<long long>(ne) * P3;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(t / P3), slot = static_cast<int>(t % P3);
    const int x = slot % P, y = (slot / P) % P, z = slot / (P * P);
    const int ii = x - 1, jj = y - 1, kk = z - 1;
    const bool ox = ii < 0 || ii > n, oy = jj < 0 || jj > n, oz = kk < 0 || kk > n;
    const int nout = ox + oy + oz;
    int g = -1;
    if (nout == 0) {
      const int s = surface_slot(NP, ii, jj, kk);
      g = s >= 0 ? dec(__ldg(smap + static_cast<long long>(e) * sstride + s))
                 : nsg + e * NI + ((kk - 1) * (n - 1) + (jj - 1)) * (n - 1) + (ii - 1);
    } else if (nout == 1) {
      int f, u, w;
      if (ox) {
        f = ii < 0 ? 0 : 1, u = jj, w = kk;
      } else if (oy) {
        f = jj < 0 ? 2 : 3, u = kk, w = ii;
      } else {
        f = kk < 0 ? 4 : 5, u = ii, w = jj;
      }
      g = dec(__ldg(sub_face + static_cast<long long>(e) * sfstride + (f * NP + w) * NP + u));
    }
    keys[t] = g;
  }
}

// Surface map rows and the Ax gather CSR from the sorted surface copies:
// smap[e][0][q] = Dirichlet-encoded global id, smap[e][1][q] = the copy's CSR
// position; ax_idx[pos] = e*nsurfp + q (copies ascending in (e, q)).
__global__ void surface_map_kernel(const int* __restrict__ l2g_surf, const int* __restrict__ pos,
                                   const std::uint8_t* __restrict__ mask, int ne, int nsurf, int nsurfp,
                                   int* __restrict__ smap, int* __restrict__ ax_idx)
{
  const long long total = static_cast<long long>(ne) * nsurf;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(t / nsurf), q = static_cast<int>(t % nsurf);
    const int g = l2g_surf[t], p = pos[t];
    int* row = smap + static_cast<long long>(e) * 2 * nsurfp;
    row[q] = mask[g] ? encode_dirichlet(g) : g;
    row[nsurfp + q] = p;
    ax_idx[p] = e * nsurfp + q;
  }
}

// sub_face rows [e][6 np^2] -> padded [e][nfp], Dirichlet-encoded (-1: no neighbour)
__global__ void encode_sub_face_kernel(const int* __restrict__ raw, const std::uint8_t* __restrict__ mask, int ne,
                                       int nf, int nfp, int* __restrict__ enc)
{
  const long long n = static_cast<long long>(ne) * nfp;
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = p / nfp;
    const int q = static_cast<int>(p % nfp);
    int v = -1;
    if (q < nf) {
      const int g = raw[e * nf + q];
      v = g < 0 ? -1 : (mask[g] ? encode_dirichlet(g) : g);
    }
    enc[p] = v;
  }
}

__global__ void iota_kernel(int* __restrict__ v, int n)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) v[t] = t;
}
// cnt[t'] = copies of node perm[t'] (cnt[n] = 0 for the exclusive scan)
__global__ void perm_counts_kernel(const unsigned* __restrict__ off, const int* __restrict__ perm, int n,
                                   unsigned* __restrict__ cnt)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += gridDim.x * blockDim.x) {
    if (t == n) {
      cnt[t] = 0;
    } else {
      const int g = perm[t];
      cnt[t] = off[g + 1] - off[g];
    }
  }
}
// idx2 segments in permuted node order
__global__ void perm_segments_kernel(const unsigned* __restrict__ off, const int* __restrict__ idx,
                                     const int* __restrict__ perm, const unsigned* __restrict__ off2, int n,
                                     int* __restrict__ idx2)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int g = perm[t];
    const unsigned a = off[g], b = off[g + 1], d = off2[t];
    for (unsigned q = a; q < b; ++q) idx2[d + (q - a)] = idx[q];
  }
}

// b[g] = mask ? 0 : m_N * 1 (assemble_load with s = 1, problem.cpp:38-46)
__global__ void load_ones_kernel(const std::uint8_t* __restrict__ mask, const double* __restrict__ lumped, int n,
                                 double* __restrict__ b)
{
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x)
    b[g] = mask[g] ? 0.0 : lumped[g] * 1.0;
}

// Restriction weights of the surface slots, m_l / m_N (coarse.cpp:149, 157):
// the FDM's fused restriction reads one contiguous row per element instead of
// the scattered 1/m_N and the mass row (Dirichlet slots weigh 0)
__global__ void restrict_weights_kernel(const int* __restrict__ smap, int sstride, const double* __restrict__ mass,
                                        int nloc, const double* __restrict__ inv_lumped, const int* __restrict__ slot_l,
                                        int nsurf_raw, int nsurfp, int ne, double* __restrict__ cw)
{
  const long long n = static_cast<long long>(ne) * nsurfp;
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = p / nsurfp;
    const int q = static_cast<int>(p % nsurfp);
    double w = 0.0;
    if (q < nsurf_raw) {
      const int code = smap[e * sstride + q];
      if (code >= 0) w = mass[e * nloc + slot_l[q]] * inv_lumped[code];
    }
    cw[p] = w;
  }
}

// Lumped mass m_N = gather of the local masses (SemOperator ctor,
// operator.cpp:90-91): surface nodes sum their copies in the CSR's (e, l)
// order from 0, interior nodes have one copy (0 + m = m); and 1/m_N. Same
// additions in the same order as the host loop, so bitwise equal.
template <int NP>
__global__ void lumped_mass_kernel(const unsigned* __restrict__ off, const int* __restrict__ ax_idx,
                                   const double* __restrict__ mass, const int* __restrict__ slot_l, int nsurfp,
                                   int nsg, int n, double* __restrict__ lumped, double* __restrict__ inv_lumped)
{
  constexpr int nn = NP - 1, NI = (nn - 1) * (nn - 1) * (nn - 1), NL = NP * NP * NP;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (g < nsg) {
      for (unsigned q = __ldg(off + g); q < __ldg(off + g + 1); ++q) {
        const int x = __ldg(ax_idx + q);
        s += __ldg(mass + static_cast<long long>(x / nsurfp) * NL + __ldg(slot_l + x % nsurfp));
      }
    } else if constexpr (NI > 0) {
      const int t = g - nsg, l = t % NI;
      const long long e = t / NI;
      const int i = 1 + l % (nn - 1), j = 1 + (l / (nn - 1)) % (nn - 1), k = 1 + l / ((nn - 1) * (nn - 1));
      s += __ldg(mass + e * NL + (k * NP + j) * NP + i);
    }
    lumped[g] = s;
    inv_lumped[g] = 1.0 / s;
  }
}

// stable counting sort of a flat source stream by destination (see device_csr_by_key)
__global__ void iota_key_kernel(const int* __restrict__ keys, long long n, int nkeys, int* __restrict__ k2,
                                int* __restrict__ vals, unsigned* __restrict__ counts)
{
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = keys[i];
    k2[i] = k < 0 ? nkeys : k;
    vals[i] = static_cast<int>(i);
    if (k >= 0) atomicAdd(counts + k, 1u);
  }
}

__global__ void scatter_pos_kernel(const int* __restrict__ sorted_vals, long long n_valid, long long n,
                                   int* __restrict__ pos)
{
  for (long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<long long>(gridDim.x) * blockDim.x)
    pos[sorted_vals[p]] = p < n_valid ? static_cast<int>(p) : -1;
}

}  // namespace hxb
