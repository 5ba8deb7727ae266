// Ax: matrix-free SEM stiffness + mass action, SemOperator::apply
// (operator.cpp:255-287) with the element contraction of
// contraction_kernel (operator.cpp:124-163), restructured for sm_100a.
//
// One CTA holds EPB elements; each element is an NP x NP thread tile (i,j)
// owning the k-column of its element. Per element:
//   A  load u (masked gather via the surface map / closed-form interior ids)
//      into registers (k-column) and shared memory
//   B  r- and s-derivatives as line contractions: thread -> one x-line and
//      one y-line, NP inputs in registers, NP outputs; D entries are
//      compile-time indices into constant memory (DFMA constant operands).
//      t-derivative stays in the owner's registers.
//   C  owner combines with the six kappa*m*Gt planes (coalesced FP64 loads)
//      into fluxes fa, fb (shared, in place) and fc (registers)
//   D  adjoint line contractions of fa (x-lines) and fb (y-lines) in place
//   E  owner sums x/y/z adjoint parts + (c*u)*m and writes: element-interior
//      nodes straight into r (unique owner, no assembly needed); element-
//      surface nodes into the surface E-vector, later summed by ax_gather in
//      reference (e,l) order (mesh.cpp:463-475).
// Shared rows are padded to an odd stride so every line access is
// bank-conflict free for FP64.
#pragma once

#include "kernels_common.cuh"

namespace hxb {

template <int NP>
struct AxShape {
  static constexpr int kLocal = NP * NP;                         // threads per element
  static constexpr int kEPB = NP <= 3 ? 8 : (NP <= 6 ? 4 : (NP <= 8 ? 2 : 1));
  static constexpr int kBlock = ((kLocal * kEPB + 31) / 32) * 32;
  static constexpr int kS = NP | 1;                              // padded row stride
  static constexpr int kBuf = NP * NP * kS;                      // one field per element
  static constexpr int kSmemDoubles = 3 * kBuf * kEPB;
};

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

template <int NP>
__global__ void __launch_bounds__(AxShape<NP>::kBlock) ax_elem_kernel(AxArgs a)
{
  using Sh = AxShape<NP>;
  constexpr int n = NP - 1, S = Sh::kS, B = Sh::kBuf;
  extern __shared__ double smem[];
  __shared__ double red[Sh::kBlock / 32];
  const double* D = c_tab[NP].D;

  const int tid = threadIdx.x;
  const int el = tid / Sh::kLocal;
  const int loc = tid - el * Sh::kLocal;
  const int i = loc % NP, j = loc / NP;
  const int e = blockIdx.x * Sh::kEPB + el;
  const bool active = (el < Sh::kEPB) && (e < a.ne);
  const int elc = el < Sh::kEPB ? el : 0;
  double* su = smem + elc * 3 * B;
  double* sa = su + B;
  double* sb = sa + B;

  // ---- A: gather u (masked) -------------------------------------------------
  double ucol[NP];
  const long long ebase_int = (long long)a.num_surface_global + (long long)e * (n - 1) * (n - 1) * (n - 1);
  const int* surf = a.l2g_surf + (long long)e * a.nsurf;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    double v = 0.0;
    if (active) {
      const int s = surface_slot(NP, i, j, k);
      if (s < 0)
        v = __ldg(a.u + ebase_int + ((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1));
      else
        v = load_masked(a.u, __ldg(surf + s));
    }
    ucol[k] = v;
    if (el < Sh::kEPB) su[(k * NP + j) * S + i] = v;
  }
  __syncthreads();

  // ---- B: x- and y-derivative lines; z in registers -------------------------
  if (el < Sh::kEPB) {
    const int la = loc % NP, lb = loc / NP;
    double line[NP];
    // x-line (j=la, k=lb): sx[ii] = sum_m D[m][ii] u[k][j][m]  (operator.cpp:136)
#pragma unroll
    for (int m = 0; m < NP; ++m) line[m] = su[(lb * NP + la) * S + m];
#pragma unroll
    for (int ii = 0; ii < NP; ++ii) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) s += D[m * NP + ii] * line[m];
      sa[(lb * NP + la) * S + ii] = s;
    }
    // y-line (i=la, k=lb): sy[jj] = sum_m D[m][jj] u[k][m][i]  (operator.cpp:137)
#pragma unroll
    for (int m = 0; m < NP; ++m) line[m] = su[(lb * NP + m) * S + la];
#pragma unroll
    for (int jj = 0; jj < NP; ++jj) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) s += D[m * NP + jj] * line[m];
      sb[(lb * NP + jj) * S + la] = s;
    }
  }
  // z-derivative on the owner's column (operator.cpp:138)
  double fz[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < NP; ++m) s += D[m * NP + k] * ucol[m];
    fz[k] = s;
  }
  __syncthreads();

  // ---- C: metric fluxes (operator.cpp:142-144) -------------------------------
  if (active) {
    const std::size_t ps = a.plane_stride;
    const double* g0 = a.wg + (std::size_t)e * NP * NP * NP + j * NP + i;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double* gk = g0 + k * NP * NP;
      const double w0 = __ldg(gk), w1 = __ldg(gk + ps), w2 = __ldg(gk + 2 * ps);
      const double w3 = __ldg(gk + 3 * ps), w4 = __ldg(gk + 4 * ps), w5 = __ldg(gk + 5 * ps);
      const int at = (k * NP + j) * S + i;
      const double sx = sa[at], sy = sb[at], sz = fz[k];
      sa[at] = w0 * sx + w1 * sy + w2 * sz;
      sb[at] = w1 * sx + w3 * sy + w4 * sz;
      fz[k] = w2 * sx + w4 * sy + w5 * sz;
    }
  }
  __syncthreads();

  // ---- D: adjoint contractions of fa (x) and fb (y), in place ---------------
  if (el < Sh::kEPB) {
    const int la = loc % NP, lb = loc / NP;
    double line[NP];
#pragma unroll
    for (int m = 0; m < NP; ++m) line[m] = sa[(lb * NP + la) * S + m];
#pragma unroll
    for (int ii = 0; ii < NP; ++ii) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) s += D[ii * NP + m] * line[m];
      sa[(lb * NP + la) * S + ii] = s;
    }
#pragma unroll
    for (int m = 0; m < NP; ++m) line[m] = sb[(lb * NP + m) * S + la];
#pragma unroll
    for (int jj = 0; jj < NP; ++jj) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) s += D[jj * NP + m] * line[m];
      sb[(lb * NP + jj) * S + la] = s;
    }
  }
  __syncthreads();

  // ---- E: assemble and store -------------------------------------------------
  double dot = 0.0;
  if (active) {
    const double ce = __ldg(a.c_e + e);
    const double* m0 = a.mass + (std::size_t)e * NP * NP * NP + j * NP + i;
    double* rs = a.rsurf + (long long)e * a.nsurf;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double tz = 0.0;
#pragma unroll
      for (int m = 0; m < NP; ++m) tz += D[k * NP + m] * fz[m];
      const int at = (k * NP + j) * S + i;
      double r = (sa[at] + sb[at]) + tz;
      if (ce != 0.0) r += (ce * ucol[k]) * __ldg(m0 + k * NP * NP);  // operator.cpp:159
      const int s = surface_slot(NP, i, j, k);
      if (s < 0) {
        a.r[ebase_int + ((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1)] = r;
        dot += ucol[k] * r;
      } else {
        rs[s] = r;
      }
    }
  }
  dot_commit<Sh::kBlock>(a.dot, dot, red);
}

// Surface assembly over element-surface copies, in ascending (e,l) order
// (gather, mesh.cpp:463-475), plus the Dirichlet identity rows
// (operator.cpp:279-280) and the optional fused p.Ap partial.
struct AxGatherArgs {
  const double* rsurf;
  const unsigned* off;   // num_surface_global + 1
  const int* idx;        // e*nsurf + slot, sorted per node
  const double* u;
  const std::uint8_t* mask;
  double* r;
  int num_surface_global;
  DotArgs dot;
};

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) ax_gather_kernel(AxGatherArgs a)
{
  __shared__ double red[BLOCK / 32];
  double dot = 0.0;
  for (int g = blockIdx.x * BLOCK + threadIdx.x; g < a.num_surface_global; g += gridDim.x * BLOCK) {
    const unsigned q0 = __ldg(a.off + g), q1 = __ldg(a.off + g + 1);
    double s = 0.0;
    for (unsigned q = q0; q < q1; ++q) s += __ldg(a.rsurf + __ldg(a.idx + q));
    const double ug = __ldg(a.u + g);
    if (__ldg(a.mask + g)) s = ug;
    a.r[g] = s;
    dot += ug * s;
  }
  dot_commit<BLOCK>(a.dot, dot, red);
}

}  // namespace hxb
