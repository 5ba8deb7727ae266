// Ax: matrix-free SEM stiffness + mass action, SemOperator::apply
// (operator.cpp:255-287) with the element contraction of
// contraction_kernel (operator.cpp:124-163), restructured for sm_100a.
//
// Each CTA works on EPB elements, each element an NP x NP thread tile (i,j)
// owning the k-column of its element. Per element:
//   A  gather u (masked) into registers (k-column) and two shared copies laid
//      out for x-line and y-line access
//   B  r- and s-derivatives as line contractions: thread -> one x-line and one
//      y-line (NP inputs in registers, NP outputs, in place); t-derivative on
//      the owner's register column. Loops run m-outer so each row D[m][*] is a
//      uniform constant load shared by all NP outputs.
//   C  owner combines with the six kappa*m*Gt planes (coalesced FP64 loads)
//      into fluxes fa, fb (shared, in place) and fc (registers)
//   D  adjoint line contractions of fa (x) and fb (y) in place, and of fc on
//      the owner column (rows of D^T)
//   E  owner sums the three adjoint parts + (c*u)*m and stores: element-interior
//      nodes straight into r (a unique copy, no assembly); element-surface
//      nodes into the surface E-vector, summed later by ax_gather in reference
//      (e,l) order (mesh.cpp:463-475).
// Shared layouts are bank-conflict free for all three access patterns at
// NP=8 (swizzled); other orders use odd padded strides.
#pragma once

#include "kernels_common.cuh"

namespace hxb {

template <int NP>
struct AxShape {
  static constexpr int kLocal = NP * NP;  // threads per element
  static constexpr int kEPB = NP <= 3 ? 8 : (NP <= 6 ? 4 : (NP <= 8 ? 2 : 1));
  static constexpr int kBlock = ((kLocal * kEPB + 31) / 32) * 32;
  static constexpr int kS = NP | 1;  // generic padded row stride
  // per-element shared doubles for the x-layout (sa) and y-layout (sb) buffers
  static constexpr int kBufA = NP == 8 ? 512 : NP * NP * kS;
  static constexpr int kBufB = NP == 8 ? 576 : NP * NP * kS;
  static constexpr int kSmemDoubles = (kBufA + kBufB) * kEPB;
  // register budget per thread (>= 20 resident warps per SM at NP=8)
  static constexpr int kRegs = NP >= 9 ? 128 : 96;
  static constexpr int kMinBlocks = 65536 / (kBlock * kRegs) > 0 ? 65536 / (kBlock * kRegs) : 1;
};

// x-layout: owner (i,j | k) and x-line (j,k | m) accesses conflict free
template <int NP>
__device__ __forceinline__ int lay_a(int k, int j, int i)
{
  if constexpr (NP == 8)
    return k * 64 + j * 8 + (i ^ ((j >> 1) | ((k & 1) << 2)));
  else
    return (k * NP + j) * AxShape<NP>::kS + i;
}
// y-layout: owner (i,j | k) and y-line (i,k | m) accesses conflict free
template <int NP>
__device__ __forceinline__ int lay_b(int k, int j, int i)
{
  if constexpr (NP == 8)
    return k * 72 + j * 8 + i;
  else
    return (k * NP + j) * AxShape<NP>::kS + i;
}

struct AxArgs {
  const double* u;          // N, input (p in PCG)
  const double* wg;         // 6 planes, plane stride = plane_stride
  std::size_t plane_stride; // NE * nloc
  const double* mass;       // NE * nloc
  const double* c_e;        // NE
  const int* l2g_surf;      // NE * nsurf, Dirichlet-encoded
  double* rsurf;            // NE * nsurf surface E-vector (output)
  double* r;                // N output (interior nodes written here)
  int ne;
  int nsurf;
  int num_surface_global;   // first element-interior global id
  DotArgs dot;              // optional: sum over interior nodes of u*r
};

// Three line contractions sharing one matrix, m-outer: each row M[m][*] is
// loaded once (uniform constant loads) and feeds 3*NP DFMAs; live state is the
// three output lines plus the owner column. m ascending = reference order
// (operator.cpp:135-140).
template <int NP, class FX, class FY>
__device__ __forceinline__ void contract3(const double* __restrict__ M, FX&& in_x, FY&& in_y,
                                          const double (&col)[NP], double (&ox)[NP], double (&oy)[NP],
                                          double (&oz)[NP])
{
  {
    const double x0 = in_x(0), y0 = in_y(0), z0 = col[0];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double d = M[q];
      ox[q] = d * x0;
      oy[q] = d * y0;
      oz[q] = d * z0;
    }
  }
#pragma unroll
  for (int m = 1; m < NP; ++m) {
    const double xm = in_x(m), ym = in_y(m), zm = col[m];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double d = M[m * NP + q];
      ox[q] += d * xm;
      oy[q] += d * ym;
      oz[q] += d * zm;
    }
  }
}

template <int NP>
__global__ void __launch_bounds__(AxShape<NP>::kBlock, AxShape<NP>::kMinBlocks) ax_elem_kernel(AxArgs a)
{
  using Sh = AxShape<NP>;
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  extern __shared__ double smem[];
  __shared__ double red[Sh::kBlock / 32];
  const double* D = c_tab[NP].D;
  const double* DT = c_tab[NP].DT;

  const int tid = threadIdx.x;
  const int el = tid / Sh::kLocal;
  const bool lane_ok = el < Sh::kEPB;
  const int loc = tid - el * Sh::kLocal;
  const int i = loc % NP, j = loc / NP;  // owner column; also x-line (j'=i,k'=j) and y-line (i'=i,k'=j)
  const int elc = lane_ok ? el : 0;
  double* sa = smem + elc * (Sh::kBufA + Sh::kBufB);
  double* sb = sa + Sh::kBufA;
  const int e = blockIdx.x * Sh::kEPB + el;
  const bool active = lane_ok && e < a.ne;
  const long long ibase = (long long)a.num_surface_global + (long long)e * NI;
  const int* surf = a.l2g_surf + (long long)e * a.nsurf;

  // ---- A: gather u (masked, operator.cpp:264-265) ---------------------------
  double ucol[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    double v = 0.0;
    if (active) {
      const int s = surface_slot(NP, i, j, k);
      v = s >= 0 ? load_masked(a.u, __ldg(surf + s))
                 : __ldg(a.u + ibase + ((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1));
    }
    ucol[k] = v;
    if (lane_ok) {
      sa[lay_a<NP>(k, j, i)] = v;
      sb[lay_b<NP>(k, j, i)] = v;
    }
  }
  __syncthreads();

  // ---- B: derivatives (operator.cpp:136-138): x-line, y-line, owner z-column
  double fz[NP];
  {
    double ox[NP], oy[NP];
    contract3<NP>(D, [&](int m) { return sa[lay_a<NP>(j, i, m)]; }, [&](int m) { return sb[lay_b<NP>(j, m, i)]; },
                  ucol, ox, oy, fz);
    __syncthreads();  // all lines read before any is overwritten
    if (lane_ok) {
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        sa[lay_a<NP>(j, i, q)] = ox[q];
        sb[lay_b<NP>(j, q, i)] = oy[q];
      }
    }
  }
  __syncthreads();

  // ---- C: metric fluxes (operator.cpp:142-144) ------------------------------
  if (active) {
    const std::size_t ps = a.plane_stride;
    const double* g0 = a.wg + (std::size_t)e * NP * NP * NP + j * NP + i;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double* gk = g0 + k * NP * NP;
      const double w0 = __ldg(gk), w1 = __ldg(gk + ps), w2 = __ldg(gk + 2 * ps);
      const double w3 = __ldg(gk + 3 * ps), w4 = __ldg(gk + 4 * ps), w5 = __ldg(gk + 5 * ps);
      const int pa = lay_a<NP>(k, j, i), pb = lay_b<NP>(k, j, i);
      const double sx = sa[pa], sy = sb[pb], sz = fz[k];
      sa[pa] = w0 * sx + w1 * sy + w2 * sz;
      sb[pb] = w1 * sx + w3 * sy + w4 * sz;
      fz[k] = w2 * sx + w4 * sy + w5 * sz;
    }
  }
  __syncthreads();

  // ---- D: adjoint contractions (operator.cpp:152-157), rows of D^T ------------
  double tz[NP];
  {
    double ox[NP], oy[NP];
    contract3<NP>(DT, [&](int m) { return sa[lay_a<NP>(j, i, m)]; }, [&](int m) { return sb[lay_b<NP>(j, m, i)]; },
                  fz, ox, oy, tz);
    __syncthreads();
    if (lane_ok) {
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        sa[lay_a<NP>(j, i, q)] = ox[q];
        sb[lay_b<NP>(j, q, i)] = oy[q];
      }
    }
  }
  __syncthreads();

  // ---- E: sum, mass term, store ---------------------------------------------
  double dot = 0.0;
  if (active) {
    const double ce = __ldg(a.c_e + e);
    const double* m0 = a.mass + (std::size_t)e * NP * NP * NP + j * NP + i;
    double* rs = a.rsurf + (long long)e * a.nsurf;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double r = (sa[lay_a<NP>(k, j, i)] + sb[lay_b<NP>(k, j, i)]) + tz[k];
      if (ce != 0.0) r += (ce * ucol[k]) * __ldg(m0 + k * NP * NP);  // operator.cpp:159
      const int s = surface_slot(NP, i, j, k);
      if (s >= 0) {
        rs[s] = r;
      } else {
        a.r[ibase + ((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1)] = r;
        dot += ucol[k] * r;
      }
    }
  }
  dot_commit<Sh::kBlock>(a.dot, dot, red);
}

}  // namespace hxb
