// PCG vector kernels (krylov.cpp:20-71) with the dot products fused into the
// passes that produce their operands. Iteration scalars live in device-side
// history arrays indexed by iteration, so no kernel ever rewrites a scalar
// another block may still be reading:
//   zr[k]  = z_k . r_k          (written by the combine kernel / init)
//   pf[k]  = p_k . A p_k        (written by the Ax gather epilogue)
//   res[k] = ||r_k||            (res[0] = ||b||)
//   alpha_k = zr[k]/pf[k], beta_k = zr[k+1]/zr[k]
#pragma once

#include "kernels_common.cuh"

namespace hxb {

// r = b, u = 0, sum b.b -> res2
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) pcg_init_kernel(const double* __restrict__ b, double* __restrict__ r,
                                                        double* __restrict__ u, int n, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  double s = 0.0;
  for (int i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
    const double bi = b[i];
    r[i] = bi;
    u[i] = 0.0;
    s += bi * bi;
  }
  dot_commit<BLOCK>(d, s, red);
}

// p = z, and zr = z.r
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) copy_dot_kernel(const double* __restrict__ z, const double* __restrict__ r,
                                                        double* __restrict__ p, int n, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  double s = 0.0;
  for (int i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
    const double zi = z[i];
    if (p) p[i] = zi;
    s += zi * r[i];
  }
  dot_commit<BLOCK>(d, s, red);
}

// alpha = zr[k]/pf[k]; r -= alpha f; sum r.r -> rn2 (krylov.cpp:52-58).
// Skips the update on breakdown (!(pf > 0)); the host reads pf[k] and stops.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) pcg_update_kernel(const double* __restrict__ f, double* __restrict__ r, int n,
                                                          const double* __restrict__ zr, const double* __restrict__ pf,
                                                          int k, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  const double pfk = pf[k];
  double s = 0.0;
  if (pfk > 0) {
    const double alpha = zr[k] / pfk;
    for (int i = blockIdx.x * BLOCK + threadIdx.x; i < n; i += gridDim.x * BLOCK) {
      const double ri = r[i] - alpha * f[i];
      r[i] = ri;
      s += ri * ri;
    }
  }
  dot_commit<BLOCK>(d, s, red);
}

// u += alpha_k p_k; p_{k+1} = z + beta_k p_k   (krylov.cpp:54, 63-66; the u
// update of iteration k is deferred to this pass so p is read once)
__global__ void pcg_dir_kernel(const double* __restrict__ z, double* __restrict__ p, double* __restrict__ u, int n,
                               const double* __restrict__ zr, const double* __restrict__ pf, int k)
{
  const double alpha = zr[k] / pf[k];
  const double beta = zr[k + 1] / zr[k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double pi = p[i];
    u[i] += alpha * pi;
    p[i] = z[i] + beta * pi;
  }
}

// p_{k+1} = z + beta_k p_k alone: u += alpha_k p_k already ran inside the
// fine half of the combine (in the shadow of the coarse solve)
__global__ void pcg_dir_p_kernel(const double* __restrict__ z, double* __restrict__ p, int n,
                                 const double* __restrict__ zr, int k)
{
  const double beta = zr[k + 1] / zr[k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = z[i] + beta * p[i];
}

// final u += alpha_k p_k
__global__ void pcg_final_kernel(const double* __restrict__ p, double* __restrict__ u, int n,
                                 const double* __restrict__ zr, const double* __restrict__ pf, int k)
{
  const double alpha = zr[k] / pf[k];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) u[i] += alpha * p[i];
}

// res[k] = sqrt(res2)
__global__ void sqrt_store_kernel(const double* __restrict__ src, double* __restrict__ dst)
{
  *dst = sqrt(*src);
}

// --- backward-Euler heat driver (problem.cpp:145-255) -------------------------
// b = mask ? 0 : m (u/dt + q), q = Q/(rho cp) inside the moving ball;
// source integral sum m q over free nodes -> dot
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) heat_rhs_kernel(const double* __restrict__ xyz, const double* __restrict__ m,
                                                        const std::uint8_t* __restrict__ mask,
                                                        const double* __restrict__ u, double* __restrict__ b, int n,
                                                        double cx, double cy, double cz, double r2, double qd,
                                                        double dt, int has_source, DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  double s = 0.0;
  for (int g = blockIdx.x * BLOCK + threadIdx.x; g < n; g += gridDim.x * BLOCK) {
    double dist2 = 0.0;
    const double dx = xyz[3 * (long long)g] - cx, dy = xyz[3 * (long long)g + 1] - cy, dz = xyz[3 * (long long)g + 2] - cz;
    dist2 += dx * dx;
    dist2 += dy * dy;
    dist2 += dz * dz;
    const double q = (has_source && dist2 <= r2) ? qd : 0.0;
    const bool fixed = mask[g] != 0;
    b[g] = fixed ? 0.0 : m[g] * (u[g] / dt + q);
    if (!fixed) s += m[g] * q;
  }
  dot_commit<BLOCK>(d, s, red);
}

// b -= A u (warm start residual, problem.cpp:211-212)
__global__ void sub_kernel(double* __restrict__ b, const double* __restrict__ au, int n)
{
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) b[g] -= au[g];
}

// u += du; partial sums of m u (slot 0) and m u^2 (slot 1) (problem.cpp:214-221)
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) heat_update_kernel(double* __restrict__ u, const double* __restrict__ du,
                                                           const double* __restrict__ m, int n, DotArgs d0, DotArgs d1)
{
  __shared__ double red[BLOCK / 32];
  double s0 = 0.0, s1 = 0.0;
  for (int g = blockIdx.x * BLOCK + threadIdx.x; g < n; g += gridDim.x * BLOCK) {
    const double v = u[g] + du[g];
    u[g] = v;
    s0 += m[g] * v;
    s1 += m[g] * v * v;
  }
  dot_commit<BLOCK>(d0, s0, red);
  dot_commit<BLOCK>(d1, s1, red);
}

// mode none: z = r, zr = z.r
// (precond.cpp:30-33)

}  // namespace hxb
