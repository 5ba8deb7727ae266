// Coarse two-scale component on the device:
//   restrict_cw_kernel + vertex_gather_kernel CoarsePreconditioner::restrict_residual
//                                            (coarse.cpp:138-162) + R[mask]=0 (:191-192)
//   AMG K-cycle kernels                      AmgHierarchy cycle/ksolve (amg.cpp:198-263)
//   dense_solve_kernel                       coarsest / direct solve (Eigen LLT in the
//                                            reference, amg.cpp:188-194, coarse.cpp:201-206)
// All sums over shared entities use sorted member lists (no atomics).
#pragma once

#include "kernels_common.cuh"

namespace hxb {

constexpr double kJacobiOmega = 2.0 / 3.0;  // amg.cpp:44

// Restriction, warp per element (restrict_residual, coarse.cpp:138-162, on
// the masked residual, precond.cpp:35): R_cb(e) = sum_l B[cb][l] y_l m_l with
// y = r / m_N, using precomputed surface-slot weights cw = m_l / m_N
// (restrict_weights_kernel): w_l = r_l cw_l on surface slots, w_l = r_l on
// element-interior nodes (one copy: m_N = m_l). No mass or 1/m_N loads, so it
// runs as a cheap standalone pass before the FDM and the coarse solve can
// start concurrently with the fine solves.
//
// Warp per element, lanes over the element's nodes in storage order: surface
// slots first (codes and weights are contiguous rows, r gathered through the
// codes), then the interior block (contiguous ids). Every load of a warp
// instruction is coalesced; each lane spreads its node's weighted value over
// the 8 corners with hat_a(t_i) hat_b(t_j) hat_c(t_k) and the warp reduces the
// partials in a fixed tree (deterministic; the order differs from the
// reference's l-loop at rounding level only). Measured against the line-per-
// lane traversal it replaced (strided interior loads, 35 % of HBM): see
// DESIGN.md section 7.
#ifndef RESTRICT_MINB
#define RESTRICT_MINB 4
#endif
#ifndef RESTRICT_US
#define RESTRICT_US 4
#endif
template <int NP>
__global__ void __launch_bounds__(256, RESTRICT_MINB) restrict_cw_kernel(const double* __restrict__ r, const int* __restrict__ smap,
                                                          const double* __restrict__ cw, double* __restrict__ Rpart,
                                                          int ne, int sstride, int nsurfp, int nsg,
                                                          const int* __restrict__ order)
{
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1), NS = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2);
  constexpr int US = NP == 7 && RESTRICT_US > 3 && RESTRICT_MINB >= 4 ? 3 : RESTRICT_US;  // loads in flight per lane (NP = 7 spills at 4)
  __shared__ double h0[NP], h1[NP];
  // local (i, j, k) of every surface slot and element-interior index, packed i | j << 4 | k << 8
  __shared__ unsigned short lut_surf[NS], lut_int[NI > 0 ? NI : 1];
  if (threadIdx.x < NP) {
    h0[threadIdx.x] = c_tab[NP].hat0[threadIdx.x];
    h1[threadIdx.x] = c_tab[NP].hat1[threadIdx.x];
  }
  for (int q = threadIdx.x; q < NS; q += blockDim.x) {
    int i, j, k;
    surface_ijk<NP>(q, i, j, k);
    lut_surf[q] = static_cast<unsigned short>(i | (j << 4) | (k << 8));
  }
  for (int q = threadIdx.x; q < NI; q += blockDim.x)
    lut_int[q] = static_cast<unsigned short>((1 + q % (n - 1)) | ((1 + (q / (n - 1)) % (n - 1)) << 4) |
                                             ((1 + q / ((n - 1) * (n - 1))) << 8));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  auto spread = [&](double (&acc)[8], unsigned ijk, double w) {
    const int i = ijk & 15, j = (ijk >> 4) & 15, k = ijk >> 8;
    const double a0 = h0[i] * w, a1 = h1[i] * w;
    const double c00 = h0[j] * h0[k], c10 = h1[j] * h0[k], c01 = h0[j] * h1[k], c11 = h1[j] * h1[k];
    acc[0] += c00 * a0;
    acc[1] += c00 * a1;
    acc[2] += c10 * a0;
    acc[3] += c10 * a1;
    acc[4] += c01 * a0;
    acc[5] += c01 * a1;
    acc[6] += c11 * a0;
    acc[7] += c11 * a1;
  };
  // elements in Morton order (order[], the FDM's traversal): the face
  // neighbours that share a surface node run close in time, so its r is read
  // from L2
  for (int eo = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; eo < ne; eo += warps) {
    const int e = order ? __ldg(order + eo) : eo;
    const int* surf = smap + (long long)e * sstride;
    const double* we = cw + (long long)e * nsurfp;
    const double* ri = r + (long long)nsg + (long long)e * NI;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 1
    for (int s0 = 0; s0 < NS; s0 += 32 * US) {
      int code[US];
      double wt[US], v[US];
#pragma unroll
      for (int u = 0; u < US; ++u) {
        const int s = s0 + 32 * u + lane;
        code[u] = s < NS ? __ldg(surf + s) : -1;
        wt[u] = s < NS ? __ldg(we + s) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < US; ++u) v[u] = code[u] >= 0 ? __ldg(r + code[u]) : 0.0;  // Dirichlet: masked (precond.cpp:35)
#pragma unroll
      for (int u = 0; u < US; ++u) {
        const int s = s0 + 32 * u + lane;
        if (s < NS) spread(acc, lut_surf[s], v[u] * wt[u]);
      }
    }
    if constexpr (NI > 0) {
#pragma unroll 1
      for (int t0 = 0; t0 < NI; t0 += 32 * US) {
        double v[US];
#pragma unroll
        for (int u = 0; u < US; ++u) {
          const int t = t0 + 32 * u + lane;
          v[u] = t < NI ? __ldg(ri + t) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < US; ++u) {
          const int t = t0 + 32 * u + lane;
          if (t < NI) spread(acc, lut_int[t], v[u]);
        }
      }
    }
#pragma unroll
    for (int cb = 0; cb < 8; ++cb)
      for (int o = 16; o > 0; o >>= 1) acc[cb] += __shfl_xor_sync(0xffffffffu, acc[cb], o);
    if (lane < 8) {
      double v = acc[0];
#pragma unroll
      for (int cb = 1; cb < 8; ++cb)
        if (lane == cb) v = acc[cb];
      Rpart[8 * (long long)e + lane] = v;
    }
  }
}

// Zc[8e + cb] = Z[vertex of corner cb of e] (the 8 coarse values each element
// prolongates, coarse.cpp:170-171), so the fused combine reads one 64-byte
// block per element copy instead of 8 dependent gathers.
__global__ void corner_values_kernel(const double* __restrict__ Z, const int* __restrict__ conn,
                                     double* __restrict__ Zc, int ne)
{
  constexpr int kCorner[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // kHexCornerFromBits, mesh.hpp:33
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < 8LL * ne; q += (long long)gridDim.x * blockDim.x) {
    const long long e = q >> 3;
    const int cb = static_cast<int>(q & 7);
    Zc[q] = __ldg(Z + __ldg(conn + 8 * e + kCorner[cb]));
  }
}

// Dense coarse block on the device: scatter the CSR into a zeroed m x m array.
__global__ void dense_scatter_kernel(const long long* __restrict__ ptr, const int* __restrict__ col,
                                     const double* __restrict__ val, int m, double* __restrict__ A)
{
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x)
    for (long long k = ptr[r]; k < ptr[r + 1]; ++k) A[(std::size_t)r * m + col[k]] += val[k];
}
__global__ void dense_identity_kernel(double* __restrict__ A, int m)
{
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) A[(std::size_t)r * m + r] = 1.0;
}

// ---------------------------------------------------------------------------
// AMG level data (device pointers)
struct DevCsr {
  int n;
  const int* ptr;
  const int* col;
  const double* val;
};

__device__ __forceinline__ double csr_row_dot(const DevCsr& A, int i, const double* __restrict__ x)
{
  return csr_row_sum(A.ptr, A.col, A.val, i, [&](int c) { return __ldg(x + c); });
}

// z = z1 + w d (r - A z1), z1 = w d r computed on the fly (amg.cpp:212-213)
struct KScalars {
  double zr, pf, zr_next;
  int stopped;
  int pad;
};

// init (the K-solve's first cycle): also r_copy = r, x = 0, stopped = 0 (the
// K-solve's initialisation, folded into its first kernel)
__global__ void amg_jacobi2_kernel(DevCsr A, const double* __restrict__ dinv, const double* __restrict__ r,
                                   double* __restrict__ z, double* __restrict__ r_copy = nullptr,
                                   double* __restrict__ x_zero = nullptr, KScalars* ks_init = nullptr)
{
  if (ks_init && blockIdx.x == 0 && threadIdx.x == 0) ks_init->stopped = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
    if (r_copy) {
      r_copy[i] = __ldg(r + i);
      x_zero[i] = 0.0;
    }
    const double s = csr_row_sum(A.ptr, A.col, A.val, i,
                                 [&](int c) { return kJacobiOmega * __ldg(dinv + c) * __ldg(r + c); });
    const double z1 = kJacobiOmega * __ldg(dinv + i) * __ldg(r + i);
    z[i] = z1 + kJacobiOmega * __ldg(dinv + i) * (__ldg(r + i) - s);
  }
}

// rc[c] = sum over members i of aggregate c (ascending) of rho_i
// (rho = r - A z from amg_resid_kernel; amg.cpp:214-218)
__global__ void amg_agg_sum_kernel(const double* __restrict__ rho, const int* __restrict__ agg_ptr,
                                   const int* __restrict__ agg_mem, double* __restrict__ rc, int nc)
{
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = __ldg(agg_ptr + c); q < __ldg(agg_ptr + c + 1); ++q) s += __ldg(rho + __ldg(agg_mem + q));
    rc[c] = s;
  }
}

// zout = z3 + w d (r - A z3), z3 = zin + ec[agg] on the fly (amg.cpp:220-222)
__global__ void amg_prolong_smooth_kernel(DevCsr A, const double* __restrict__ dinv, const double* __restrict__ r,
                                          const double* __restrict__ zin, const double* __restrict__ ec,
                                          const int* __restrict__ agg, double* __restrict__ zout)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
    const double s = csr_row_sum(A.ptr, A.col, A.val, i,
                                 [&](int c) { return __ldg(zin + c) + __ldg(ec + __ldg(agg + c)); });
    const double z3 = __ldg(zin + i) + __ldg(ec + __ldg(agg + i));
    zout[i] = z3 + kJacobiOmega * __ldg(dinv + i) * (__ldg(r + i) - s);
  }
}

// zout = zin + w d (r - A zin)   (amg.cpp:204-208)
__global__ void amg_smooth_kernel(DevCsr A, const double* __restrict__ dinv, const double* __restrict__ r,
                                  const double* __restrict__ zin, double* __restrict__ zout)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
    const double s = csr_row_dot(A, i, zin);
    zout[i] = __ldg(zin + i) + kJacobiOmega * __ldg(dinv + i) * (__ldg(r + i) - s);
  }
}

// the same smoothing step with the K-solve's following z.r (and optional
// p = z) fused in: identical grid, loop and reduction as amg_dot_kernel, so
// the dot is bitwise the separate kernel's
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) amg_smooth_dot_kernel(DevCsr A, const double* __restrict__ dinv,
                                                              const double* __restrict__ r,
                                                              const double* __restrict__ zin, double* __restrict__ zout,
                                                              double* __restrict__ p, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  double acc = 0.0;
  for (int i = blockIdx.x * BLOCK + threadIdx.x; i < A.n; i += gridDim.x * BLOCK) {
    const double s = csr_row_dot(A, i, zin);
    const double ri = __ldg(r + i);
    const double zi = __ldg(zin + i) + kJacobiOmega * __ldg(dinv + i) * (ri - s);
    zout[i] = zi;
    if (p) p[i] = zi;
    acc += zi * ri;
  }
  dot_commit<BLOCK>(d, acc, red);
}

// ---------------------------------------------------------------------------
// K-cycle inner PCG (amg.cpp:230-263). Scalars of one ksolve invocation:

// f = A p; result = p.f
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) amg_spmv_dot_kernel(DevCsr A, const double* __restrict__ p,
                                                            double* __restrict__ f, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  double s = 0.0;
  for (int i = blockIdx.x * BLOCK + threadIdx.x; i < A.n; i += gridDim.x * BLOCK) {
    const double fi = csr_row_dot(A, i, p);
    f[i] = fi;
    s += p[i] * fi;
  }
  dot_commit<BLOCK>(d, s, red);
}

// if (!(pf > 0) || !(|zr| > 0)) stop; else x += a p, r -= a f  (amg.cpp:244-253).
// zr_is_next: the second step reads zr from zr_next (the value the separate
// shift kernel used to copy into zr after amg_kdir_kernel)
__global__ void amg_kupdate_kernel(const double* __restrict__ p, const double* __restrict__ f, double* __restrict__ x,
                                   double* __restrict__ r, int n, KScalars* ks, int zr_is_next)
{
  const double pf = ks->pf, zr = zr_is_next ? ks->zr_next : ks->zr;
  const bool stop = ks->stopped || !(pf > 0) || !(fabs(zr) > 0);
  if (stop) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) ks->stopped = 1;
    return;
  }
  const double alpha = zr / pf;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * f[i];
  }
}

// beta = zr_next/zr; zr = zr_next; p = z + beta p   (amg.cpp:256-260)
__global__ void amg_kdir_kernel(const double* __restrict__ z, double* __restrict__ p, int n, KScalars* ks)
{
  if (ks->stopped) return;
  const double beta = ks->zr_next / ks->zr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = z[i] + beta * p[i];
}

// rho = R - K Z
__global__ void amg_resid_kernel(DevCsr A, const double* __restrict__ R, const double* __restrict__ Z,
                                 double* __restrict__ rho)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x)
    rho[i] = __ldg(R + i) - csr_row_dot(A, i, Z);
}

__global__ void axpy1_kernel(double* __restrict__ y, const double* __restrict__ x, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] += x[i];
}

// Dense coarse solve: z[coupled[r]] = sum_c Ainv[r][c] b[coupled[c]]; z[i] = b[i]*inv_diag[i] otherwise.
// One warp per coupled row (coalesced row reads).
__global__ void dense_solve_kernel(const double* __restrict__ ainv, const int* __restrict__ coupled, int m,
                                   const double* __restrict__ inv_diag, const double* __restrict__ b,
                                   double* __restrict__ z, int n)
{
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int rr = warp; rr < m; rr += nwarps) {
    const double* row = ainv + (std::size_t)rr * m;
    double s = 0.0;
    for (int c = lane; c < m; c += 32) s += row[c] * __ldg(b + __ldg(coupled + c));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) z[__ldg(coupled + rr)] = s;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double di = __ldg(inv_diag + i);
    if (di != 0.0) z[i] = __ldg(b + i) * di;
  }
}

// ---------------------------------------------------------------------------
// Large direct coarse solve (coupled block m > 1500): the inverse is symmetric,
// so only its lower-triangle 64x64 tiles are stored (m^2/2 doubles: 12 GB
// instead of 24 GB at m = 54,872) and applied as y_I = sum_{J<=I} A_IJ x_J +
// sum_{I'>I} A_I'I^T x_I'. Each tile is read once; its row and column partial
// sums go to per-tile slots and a second kernel adds them in a fixed order
// (deterministic, no atomics).
constexpr int kDenseTile = 64;

__device__ __forceinline__ void tile_of(long long t, int& I, int& J)
{
  I = static_cast<int>((sqrt(8.0 * static_cast<double>(t) + 1.0) - 1.0) * 0.5);
  while (static_cast<long long>(I + 1) * (I + 2) / 2 <= t) ++I;
  while (static_cast<long long>(I) * (I + 1) / 2 > t) --I;
  J = static_cast<int>(t - static_cast<long long>(I) * (I + 1) / 2);
}

// tiles[t][64][64] from the full row-major inverse (zero padded past m)
__global__ void dense_pack_kernel(const double* __restrict__ full, int m, double* __restrict__ tiles, long long ntiles)
{
  constexpr int T = kDenseTile;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int I, J;
    tile_of(t, I, J);
    double* dst = tiles + t * T * T;
    for (int q = threadIdx.x; q < T * T; q += blockDim.x) {
      const int r = I * T + q / T, c = J * T + q % T;
      dst[q] = (r < m && c < m) ? full[static_cast<std::size_t>(r) * m + c] : 0.0;
    }
  }
}

// xg[c] = b[coupled[c]] (zero padded to nt*64)
__global__ void dense_gather_x_kernel(const double* __restrict__ b, const int* __restrict__ coupled, int m, int mp,
                                      double* __restrict__ xg)
{
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < mp; c += gridDim.x * blockDim.x)
    xg[c] = c < m ? __ldg(b + __ldg(coupled + c)) : 0.0;
}

// one 256-thread CTA per tile: coalesced tile load into padded shared memory,
// then 64 threads form the row sums and 64 the column sums (off-diagonal tiles)
__global__ void __launch_bounds__(256) dense_tile_gemv_kernel(const double* __restrict__ tiles,
                                                              const double* __restrict__ xg, long long ntiles,
                                                              double* __restrict__ rowpart, double* __restrict__ colpart)
{
  constexpr int T = kDenseTile, S = T + 1;
  __shared__ double a[T * S];
  __shared__ double xi[T], xj[T];
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int I, J;
    tile_of(t, I, J);
    const double* src = tiles + t * T * T;
#pragma unroll 4
    for (int q = threadIdx.x; q < T * T; q += 256) a[(q / T) * S + q % T] = __ldcs(src + q);
    if (threadIdx.x < T) {
      xj[threadIdx.x] = __ldg(xg + J * T + threadIdx.x);
      xi[threadIdx.x] = __ldg(xg + I * T + threadIdx.x);
    }
    __syncthreads();
    if (threadIdx.x < T) {  // row sums
      const int r = threadIdx.x;
      double s = 0.0;
#pragma unroll 8
      for (int c = 0; c < T; ++c) s += a[r * S + c] * xj[c];
      rowpart[t * T + r] = s;
    } else if (threadIdx.x < 2 * T && I != J) {  // column sums (transpose part)
      const int c = threadIdx.x - T;
      double s = 0.0;
#pragma unroll 8
      for (int r = 0; r < T; ++r) s += a[r * S + c] * xi[r];
      colpart[t * T + c] = s;
    }
    __syncthreads();
  }
}

// z[coupled[i]] = sum_{J<=I} rowpart(I,J)[i] + sum_{I'>I} colpart(I',I)[i]; decoupled rows b/a_ii
__global__ void dense_tile_reduce_kernel(const double* __restrict__ rowpart, const double* __restrict__ colpart, int m,
                                         int nt, const int* __restrict__ coupled, const double* __restrict__ inv_diag,
                                         const double* __restrict__ b, double* __restrict__ z, int n)
{
  constexpr int T = kDenseTile;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int I = i / T, il = i % T;
    const long long base = static_cast<long long>(I) * (I + 1) / 2;
    double s = 0.0;
    for (int J = 0; J <= I; ++J) s += __ldg(rowpart + (base + J) * T + il);
    for (int I2 = I + 1; I2 < nt; ++I2) s += __ldg(colpart + (static_cast<long long>(I2) * (I2 + 1) / 2 + I) * T + il);
    z[__ldg(coupled + i)] = s;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double di = __ldg(inv_diag + i);
    if (di != 0.0) z[i] = __ldg(b + i) * di;
  }
}

// ---------------------------------------------------------------------------
// Sparse direct coarse solve (setup_nd.cpp): nested-dissection supernodal
// factor P A P^T = L L^T of the coupled block, solved level by level over the
// separator tree. Per supernode s (columns [c0, c0+m), below-diagonal rows
// rows[0..r)):
//   forward   ye = y_s - (children's propagated L z contributions to V_s)
//             z_s = L11^-1 ye                                  (nd_fwd_diag)
//             acc_s = L21 z_s + (children's contributions to rows(s))  (nd_fwd_upd)
//   backward  t_s = z_s - L21^T x(rows(s))                      (nd_bwd_upd)
//             x_s = L11^-T t_s                                  (nd_bwd_diag)
// Each dot product is a warp reduction in a fixed tree; the children's
// contributions are summed in child order from per-position lists, so the
// solve is deterministic. One CTA handles one task (supernode, block of rows).
struct NdDev {
  int n = 0;                       // coupled unknowns
  const int* perm = nullptr;       // permuted index -> coupled index
  const int* c0 = nullptr;
  const int* m = nullptr;
  const int* r = nullptr;
  const long long* linv_off = nullptr;  // also the offsets of linvT (m x m each)
  const long long* l21_off = nullptr;   // also the offsets of l21T (r x m / m x r)
  const double *linv = nullptr, *linvT = nullptr, *l21 = nullptr, *l21T = nullptr;
  const long long* rows_off = nullptr;  // rows and acc of supernode s at rows_off[s]
  const int* rows = nullptr;
  const long long* inc_base = nullptr;  // position (s, p) -> inc_base[s] + p in inc_ptr
  const int* inc_ptr = nullptr;
  const int* inc_idx = nullptr;         // acc entries contributing to that position, child order
  double *y = nullptr, *z = nullptr, *t = nullptr, *x = nullptr, *acc = nullptr;
};
struct NdTask {
  int s, row0, nrows;
};
constexpr int kNdRowsPerTask = 32;
constexpr int kNdBlock = 256;

__device__ __forceinline__ double nd_warp_sum(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double nd_incoming(const NdDev& d, int s, int p)
{
  const long long q = d.inc_base[s] + p;
  double sum = 0.0;
  for (int k = d.inc_ptr[q]; k < d.inc_ptr[q + 1]; ++k) sum += d.acc[d.inc_idx[k]];
  return sum;
}

__global__ void __launch_bounds__(kNdBlock) nd_fwd_diag_kernel(NdDev d, const NdTask* __restrict__ tasks)
{
  extern __shared__ double ye[];
  const NdTask T = tasks[blockIdx.x];
  const int s = T.s, m = d.m[s], c0 = d.c0[s];
  for (int j = threadIdx.x; j < m; j += blockDim.x) ye[j] = d.y[c0 + j] - nd_incoming(d, s, j);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* L = d.linv + d.linv_off[s];
  for (int j = T.row0 + warp; j < T.row0 + T.nrows; j += kNdBlock / 32) {
    const double* row = L + static_cast<long long>(j) * m;
    double v = 0.0;
    for (int k = lane; k <= j; k += 32) v += row[k] * ye[k];
    v = nd_warp_sum(v);
    if (lane == 0) d.z[c0 + j] = v;
  }
}

__global__ void __launch_bounds__(kNdBlock) nd_fwd_upd_kernel(NdDev d, const NdTask* __restrict__ tasks)
{
  const NdTask T = tasks[blockIdx.x];
  const int s = T.s, m = d.m[s], c0 = d.c0[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* L = d.l21 + d.l21_off[s];
  for (int i = T.row0 + warp; i < T.row0 + T.nrows; i += kNdBlock / 32) {
    const double* row = L + static_cast<long long>(i) * m;
    double v = 0.0;
    for (int k = lane; k < m; k += 32) v += row[k] * d.z[c0 + k];
    v = nd_warp_sum(v);
    if (lane == 0) d.acc[d.rows_off[s] + i] = v + nd_incoming(d, s, m + i);
  }
}

__global__ void __launch_bounds__(kNdBlock) nd_bwd_upd_kernel(NdDev d, const NdTask* __restrict__ tasks)
{
  const NdTask T = tasks[blockIdx.x];
  const int s = T.s, m = d.m[s], r = d.r[s], c0 = d.c0[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* L = d.l21T + d.l21_off[s];
  const int* rows = d.rows + d.rows_off[s];
  for (int j = T.row0 + warp; j < T.row0 + T.nrows; j += kNdBlock / 32) {
    const double* row = L + static_cast<long long>(j) * r;
    double v = 0.0;
    for (int k = lane; k < r; k += 32) v += row[k] * d.x[rows[k]];
    v = nd_warp_sum(v);
    if (lane == 0) d.t[c0 + j] = d.z[c0 + j] - v;
  }
  (void)m;
}

__global__ void __launch_bounds__(kNdBlock) nd_bwd_diag_kernel(NdDev d, const NdTask* __restrict__ tasks)
{
  const NdTask T = tasks[blockIdx.x];
  const int s = T.s, m = d.m[s], c0 = d.c0[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* L = d.linvT + d.linv_off[s];  // row j of L11^-T: entries k >= j
  for (int j = T.row0 + warp; j < T.row0 + T.nrows; j += kNdBlock / 32) {
    const double* row = L + static_cast<long long>(j) * m;
    double v = 0.0;
    for (int k = j + lane; k < m; k += 32) v += row[k] * d.t[c0 + k];
    v = nd_warp_sum(v);
    if (lane == 0) d.x[c0 + j] = v;
  }
}

// y = P b on the coupled rows; decoupled rows solved directly (1/a_ii)
__global__ void nd_permute_in_kernel(const int* __restrict__ perm, const int* __restrict__ coupled, int m,
                                     const double* __restrict__ inv_diag, const double* __restrict__ b,
                                     double* __restrict__ y, double* __restrict__ out, int n)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n || i < m; i += gridDim.x * blockDim.x) {
    if (i < m) y[i] = b[coupled[perm[i]]];
    if (i < n && inv_diag[i] != 0.0) out[i] = b[i] * inv_diag[i];
  }
}

__global__ void nd_permute_out_kernel(const int* __restrict__ perm, const int* __restrict__ coupled, int m,
                                      const double* __restrict__ x, double* __restrict__ out)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) out[coupled[perm[i]]] = x[i];
}

}  // namespace hxb
