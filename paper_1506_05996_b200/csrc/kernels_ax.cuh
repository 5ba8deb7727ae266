// Ax: matrix-free SEM stiffness + mass action, SemOperator::apply
// (operator.cpp:255-287) with the element contraction of
// contraction_kernel (operator.cpp:124-163), restructured for sm_100a.
//
// Each CTA works on one element at a time, an NP x NP thread tile (i,j) with
// each thread owning the k-column of the element. Per element:
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
  static constexpr int kLocal = NP * NP;              // threads per element
  static constexpr int kBlock = ((kLocal + 31) / 32) * 32;
  static constexpr int kEPB = 1;                      // one element per CTA (persistent)
  static constexpr int kS = NP | 1;                   // generic padded row stride
  static constexpr int kNloc = NP * NP * NP;
  static constexpr int kNlocP = (kNloc + 1) & ~1;     // 16-byte aligned plane blocks
  static constexpr int kNsurf = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2);
  static constexpr int kNsurfP = (kNsurf + 3) & ~3;   // 16-byte aligned index blocks
  // per-element shared doubles for the x-layout (sa) and y-layout (sb) buffers
  static constexpr int kBufA = NP == 8 ? 512 : NP * NP * kS;
  static constexpr int kBufB = NP == 8 ? 576 : NP * NP * kS;
  static constexpr std::size_t kGBytes = 6ull * kNlocP * sizeof(double);
  static constexpr std::size_t kIdxBytes = kNsurfP * sizeof(int);  // Dirichlet-encoded codes
  static constexpr std::size_t kSmemBytes = kGBytes + (kBufA + kBufB + 2 * NP * NP) * sizeof(double) + kIdxBytes +
                                            2 * sizeof(unsigned long long);
  // register cap per resident-CTA target (cfg4 sweep, element kernel / HBM):
  // np = 6: 6 CTAs/SM 0.72, 8 0.76, 10 0.72; np = 7: 6 0.87, 8 0.88, 10 0.56;
  // np = 9: 2 0.67, 3 0.84, 4 0.87; np = 10: 2 0.69, 3 0.77 (4 spills);
  // np = 11: 2 0.86, 3 0.76
  static constexpr int kMinBlocks = NP <= 7 ? 8 : NP == 8 ? 6 : NP == 9 ? 4 : NP == 10 ? 3 : 2;
  // on-the-fly geometry: the planes are replaced by the element record (8
  // corners + kappa, TMA-staged) and two Jacobian-column tables
  static constexpr int kRecD = 26;                      // doubles per element record (16-byte multiple)
  static constexpr std::size_t kRecBytes = kRecD * sizeof(double);
  static constexpr int kOtfHeadD = 32 + 6 * NP * NP;    // record (padded) + T0 + T1
  static constexpr std::size_t kSmemOtfBytes = kOtfHeadD * sizeof(double) +
                                               (kBufA + kBufB + 2 * NP * NP) * sizeof(double) + kIdxBytes +
                                               2 * sizeof(unsigned long long);
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
  const double* wg;         // [e][6][nlocp]: kappa*m*Gt planes per element (TMA-staged)
  const double* erec;       // on-the-fly variant: [e][26] = corner xyz in (bi,bj,bk)-bit order, kappa_e, 0
  const double* mass;       // NE * nloc
  const double* c_e;        // NE
  const int* smap;          // [e][2][nsurfp]: row 0 Dirichlet-encoded global ids (TMA-staged)
  double* rsurf;            // [e][nsurfp] surface E-vector (output)
  double* r;                // N output (interior nodes written here)
  int ne;                   // one past the last element processed
  int num_surface_global;   // first element-interior global id
  int e_begin = 0;          // first element processed (chunked host-pointer apply)
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

// ---- on-the-fly geometry (SemOperator::otf_element_kernel, operator.cpp:174-253)
// The trilinear map's Jacobian columns are bilinear in the other two
// coordinates: dX/dxi depends on (eta_j, zeta_k) only, dX/deta on (xi_i,
// zeta_k), dX/dzeta on (xi_i, eta_j), so each is an NP^2 table per element
// instead of a 24-term sum per node. X[b*3+d] with b = bi + 2 bj + 4 bk.
__device__ __forceinline__ double hatv(const OrderTables& T, int b, int q) { return b ? T.hat1[q] : T.hat0[q]; }

// column c (0: d/dxi, 1: d/deta, 2: d/dzeta) at the two other coordinates' node indices (p, q)
__device__ __forceinline__ void jac_column(const OrderTables& T, const double* __restrict__ X, int c, int p, int q,
                                           double (&out)[3])
{
  const int sc = 1 << c, s1 = c == 0 ? 2 : 1, s2 = c == 2 ? 2 : 4;  // bit strides: varied axis, first/second other axis
  out[0] = out[1] = out[2] = 0.0;
#pragma unroll
  for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
    for (int b1 = 0; b1 < 2; ++b1) {
      const double h = hatv(T, b1, p) * hatv(T, b2, q);
      const int lo = b1 * s1 + b2 * s2, hi = lo + sc;
#pragma unroll
      for (int d = 0; d < 3; ++d) out[d] += h * (0.5 * (X[hi * 3 + d] - X[lo * 3 + d]));
    }
}

// 1/x to full FP64 precision: MUFU reciprocal seed + two Newton steps
// (5 FP64 instructions instead of the division sequence); within 1 ulp
__device__ __forceinline__ double fast_rcp(double x)
{
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Metric flux at one node straight from the adjugate A of its Jacobian:
// kappa m Gt s = kappa rho^3/det A A^T s, evaluated as A (A^T s) (18 FMAs
// instead of forming the six entries and applying them); m = rho^3 det.
__device__ __forceinline__ void otf_flux(const double (&jx)[3], const double (&jy)[3], const double (&jz)[3],
                                         double kap_rho3, double rho3, double sx, double sy, double sz,
                                         double& fa, double& fb, double& fc, double& m)
{
  const double J0 = jx[0], J1 = jy[0], J2 = jz[0], J3 = jx[1], J4 = jy[1], J5 = jz[1], J6 = jx[2], J7 = jy[2],
               J8 = jz[2];
  const double a0 = J4 * J8 - J5 * J7, a1 = J2 * J7 - J1 * J8, a2 = J1 * J5 - J2 * J4;
  const double a3 = J5 * J6 - J3 * J8, a4 = J0 * J8 - J2 * J6, a5 = J2 * J3 - J0 * J5;
  const double a6 = J3 * J7 - J4 * J6, a7 = J1 * J6 - J0 * J7, a8 = J0 * J4 - J1 * J3;
  const double det = J0 * a0 + J1 * a3 + J2 * a6;
  const double scale = kap_rho3 * fast_rcp(det);
  const double v0 = a0 * sx + a3 * sy + a6 * sz, v1 = a1 * sx + a4 * sy + a7 * sz, v2 = a2 * sx + a5 * sy + a8 * sz;
  fa = scale * (a0 * v0 + a1 * v1 + a2 * v2);
  fb = scale * (a3 * v0 + a4 * v1 + a5 * v2);
  fc = scale * (a6 * v0 + a7 * v1 + a8 * v2);
  m = rho3 * det;
}

// kappa*m*Gt (six symmetric entries) and m at one node from its Jacobian
// columns: m Gt = rho^3/det adj adj^T, m = rho^3 det (operator.cpp:226-250)
__device__ __forceinline__ void otf_metric(const double (&jx)[3], const double (&jy)[3], const double (&jz)[3],
                                           double kap_rho3, double rho3, double (&w)[6], double& m)
{
  const double J0 = jx[0], J1 = jy[0], J2 = jz[0], J3 = jx[1], J4 = jy[1], J5 = jz[1], J6 = jx[2], J7 = jy[2],
               J8 = jz[2];
  const double a0 = J4 * J8 - J5 * J7, a1 = J2 * J7 - J1 * J8, a2 = J1 * J5 - J2 * J4;
  const double a3 = J5 * J6 - J3 * J8, a4 = J0 * J8 - J2 * J6, a5 = J2 * J3 - J0 * J5;
  const double a6 = J3 * J7 - J4 * J6, a7 = J1 * J6 - J0 * J7, a8 = J0 * J4 - J1 * J3;
  const double det = J0 * a0 + J1 * a3 + J2 * a6;
  const double scale = kap_rho3 / det;
  w[0] = scale * (a0 * a0 + a1 * a1 + a2 * a2);
  w[1] = scale * (a0 * a3 + a1 * a4 + a2 * a5);
  w[2] = scale * (a0 * a6 + a1 * a7 + a2 * a8);
  w[3] = scale * (a3 * a3 + a4 * a4 + a5 * a5);
  w[4] = scale * (a3 * a6 + a4 * a7 + a5 * a8);
  w[5] = scale * (a6 * a6 + a7 * a7 + a8 * a8);
  m = rho3 * det;
}

// Persistent: CTA b processes elements b, b+grid, ... . The element's six
// metric planes (6*nloc FP64, the bulk of Ax traffic) and its surface index
// block are streamed into shared memory by TMA bulk copies issued one element
// ahead (planes for e' once phase C of e has consumed them, indices for e''
// once u(e') has been gathered), and u(e') is gathered into registers during
// phase D of e, so HBM traffic overlaps the contractions. D and D^T live in
// shared memory and are read as warp-uniform broadcasts, keeping registers
// low enough for 6 CTAs per SM.
//
// OTF (operator variant on_the_fly): instead of the planes, a 208-byte element
// record (corners + kappa) is staged the same way; phase B builds the
// Jacobian-column tables, phase C forms kappa*m*Gt per node in registers.
template <int NP, bool OTF = false>
__global__ void __launch_bounds__(AxShape<NP>::kBlock, AxShape<NP>::kMinBlocks) ax_elem_kernel(AxArgs a)
{
  using Sh = AxShape<NP>;
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1), NLP = Sh::kNlocP;
  constexpr std::size_t kStage = OTF ? Sh::kRecBytes : Sh::kGBytes;  // bar[0] transaction per element
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sG = reinterpret_cast<double*>(smem_raw);                  // [6][nlocp] | OTF: record, T0, T1
  double* sT0 = sG + 32;                                             // OTF: dX/dxi at (eta_j, zeta_k)
  double* sT1 = sT0 + 3 * NP * NP;                                   // OTF: dX/deta at (xi_i, zeta_k)
  const double* stage_src = OTF ? a.erec : a.wg;
  constexpr int kStageD = OTF ? Sh::kRecD : 6 * NLP;
  double* sa = sG + (OTF ? Sh::kOtfHeadD : 6 * NLP);
  double* sb = sa + Sh::kBufA;
  double* sD = sb + Sh::kBufB;                                       // D, then D^T
  double* sDT = sD + NP * NP;
  int* sidx = reinterpret_cast<int*>(sDT + NP * NP);                 // [nsurfp]
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sidx + Sh::kNsurfP);  // [0]=G, [1]=idx
  __shared__ double red[Sh::kBlock / 32];

  const int tid = threadIdx.x;
  const bool lane_ok = tid < Sh::kLocal;
  const int loc = lane_ok ? tid : 0;
  const int i = loc % NP, j = loc / NP;  // owner column; also x-line (j'=i,k'=j) and y-line (i'=i,k'=j)
  // node classification of this thread's column: surface slot, or -1-(interior offset)
  int code[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int s = surface_slot(NP, i, j, k);
    code[k] = s >= 0 ? s : -1 - (((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1));
  }

  int e = a.e_begin + blockIdx.x;
  for (int q = tid; q < NP * NP; q += Sh::kBlock) {
    sD[q] = c_tab[NP].D[q];
    sDT[q] = c_tab[NP].DT[q];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && e < a.ne) {
    mbar_expect_tx(&bar[1], Sh::kIdxBytes);
    bulk_g2s(sidx, a.smap + (long long)e * 2 * Sh::kNsurfP, Sh::kIdxBytes, &bar[1]);
    mbar_expect_tx(&bar[0], kStage);
    bulk_g2s(sG, stage_src + (long long)e * kStageD, kStage, &bar[0]);
  }
  // gather u for element ee (masked, operator.cpp:264-265) using the staged indices
  auto gather_u = [&](int ee, double (&dst)[NP]) {
    const long long ib = (long long)a.num_surface_global + (long long)ee * NI;
#pragma unroll
    for (int k = 0; k < NP; ++k)
      dst[k] = code[k] >= 0 ? load_masked(a.u, sidx[code[k]]) : __ldg(a.u + ib - 1 - code[k]);
  };
  double ucol[NP];
  double ce = 0.0;
  unsigned phase = 0;
  if (e < a.ne) {
    mbar_wait(&bar[1], 0);
    gather_u(e, ucol);
    ce = __ldg(a.c_e + e);
    __syncthreads();
    if (tid == 0 && e + (int)gridDim.x < a.ne) {
      fence_proxy_async_smem();  // every warp's sidx reads (gather_u) precede the overwrite
      mbar_expect_tx(&bar[1], Sh::kIdxBytes);
      bulk_g2s(sidx, a.smap + (long long)(e + gridDim.x) * 2 * Sh::kNsurfP, Sh::kIdxBytes, &bar[1]);
    }
  }
  double dot = 0.0;
  for (; e < a.ne; e += gridDim.x, phase ^= 1u) {
    const int en = e + gridDim.x;
    const long long ibase = (long long)a.num_surface_global + (long long)e * NI;

    // ---- A: u column -> shared (two layouts) ------------------------------------
    if (lane_ok) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        sa[lay_a<NP>(k, j, i)] = ucol[k];
        sb[lay_b<NP>(k, j, i)] = ucol[k];
      }
    }
    __syncthreads();

    // ---- B: derivatives (operator.cpp:136-138): x-line, y-line, owner z-column
    double fz[NP];
    double jz[3] = {0.0, 0.0, 0.0}, kap = 0.0;
    if constexpr (OTF) {  // Jacobian-column tables of element e (consumed in phase C)
      mbar_wait(&bar[0], phase);
      if (lane_ok) {
        const OrderTables& T = c_tab[NP];
        double t[3];
        jac_column(T, sG, 0, i, j, t);  // entry (k'=j, j'=i)
#pragma unroll
        for (int d = 0; d < 3; ++d) sT0[(j * NP + i) * 3 + d] = t[d];
        jac_column(T, sG, 1, i, j, t);  // entry (k'=j, i'=i)
#pragma unroll
        for (int d = 0; d < 3; ++d) sT1[(j * NP + i) * 3 + d] = t[d];
        jac_column(T, sG, 2, i, j, jz);
        kap = sG[24];
      }
    }
    {
      double ox[NP], oy[NP];
      contract3<NP>(sD, [&](int m) { return sa[lay_a<NP>(j, i, m)]; }, [&](int m) { return sb[lay_b<NP>(j, m, i)]; },
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

    // ---- C: metric fluxes (operator.cpp:142-144), planes from shared ----------
    double mk[OTF ? NP : 1];
    if constexpr (!OTF) mbar_wait(&bar[0], phase);
    if (lane_ok) {
      const double wij = OTF ? c_tab[NP].w[i] * c_tab[NP].w[j] : 0.0;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int pa = lay_a<NP>(k, j, i), pb = lay_b<NP>(k, j, i);
        const double sx = sa[pa], sy = sb[pb], sz = fz[k];
        if constexpr (OTF) {
          const double jx[3] = {sT0[(k * NP + j) * 3], sT0[(k * NP + j) * 3 + 1], sT0[(k * NP + j) * 3 + 2]};
          const double jy[3] = {sT1[(k * NP + i) * 3], sT1[(k * NP + i) * 3 + 1], sT1[(k * NP + i) * 3 + 2]};
          const double rho3 = wij * c_tab[NP].w[k];
          double f0, f1, f2;
          otf_flux(jx, jy, jz, kap * rho3, rho3, sx, sy, sz, f0, f1, f2, mk[k]);
          sa[pa] = f0;
          sb[pb] = f1;
          fz[k] = f2;
        } else {
          const int l = (k * NP + j) * NP + i;
          const double w0 = sG[l], w1 = sG[NLP + l], w2 = sG[2 * NLP + l];
          const double w3 = sG[3 * NLP + l], w4 = sG[4 * NLP + l], w5 = sG[5 * NLP + l];
          sa[pa] = w0 * sx + w1 * sy + w2 * sz;
          sb[pb] = w1 * sx + w3 * sy + w4 * sz;
          fz[k] = w2 * sx + w4 * sy + w5 * sz;
        }
      }
    }
    __syncthreads();  // sG consumed
    if (tid == 0 && en < a.ne) {
      fence_proxy_async_smem();
      mbar_expect_tx(&bar[0], kStage);
      bulk_g2s(sG, stage_src + (long long)en * kStageD, kStage, &bar[0]);
    }
    // prefetch u(e') and c(e') while the adjoint contractions run
    double unext[NP];
    double cnext = 0.0;
    if (en < a.ne) {
      mbar_wait(&bar[1], phase ^ 1u);
      gather_u(en, unext);
      cnext = __ldg(a.c_e + en);
    }

    // ---- D: adjoint contractions (operator.cpp:152-157), rows of D^T ------------
    double tz[NP];
    {
      double ox[NP], oy[NP];
      contract3<NP>(sDT, [&](int m) { return sa[lay_a<NP>(j, i, m)]; }, [&](int m) { return sb[lay_b<NP>(j, m, i)]; },
                    fz, ox, oy, tz);
      __syncthreads();  // lines read; sidx(e') consumed
      if (tid == 0 && en + (int)gridDim.x < a.ne) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar[1], Sh::kIdxBytes);
        bulk_g2s(sidx, a.smap + (long long)(en + gridDim.x) * 2 * Sh::kNsurfP, Sh::kIdxBytes, &bar[1]);
      }
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
    if (lane_ok) {
      const double* m0 = a.mass + (std::size_t)e * Sh::kNloc + j * NP + i;
      double* rs = a.rsurf + (long long)e * Sh::kNsurfP;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        double r = (sa[lay_a<NP>(k, j, i)] + sb[lay_b<NP>(k, j, i)]) + tz[k];
        if (ce != 0.0) {  // operator.cpp:159
          if constexpr (OTF)
            r += (ce * ucol[k]) * mk[k];
          else
            r += (ce * ucol[k]) * __ldg(m0 + k * NP * NP);
        }
        if (code[k] >= 0) {
          rs[code[k]] = r;
        } else {
          a.r[ibase - 1 - code[k]] = r;
          dot += ucol[k] * r;
        }
      }
    }
    __syncthreads();  // sa/sb reads done before the next element's phase A
#pragma unroll
    for (int k = 0; k < NP; ++k) ucol[k] = unext[k];
    ce = cnext;
  }
  dot_commit<Sh::kBlock>(a.dot, dot, red);
}

// ---------------------------------------------------------------------------
// Low orders (NP <= 3, nloc <= 27; dispatched by plan.cu): one thread per local node, EPB elements
// per 256-thread CTA, persistent. Each CTA keeps EPB elements' u and fluxes in
// shared memory; the per-node arithmetic is contraction_kernel's
// (operator.cpp:124-163) with phase 2 in the reference's interleaved order.
// The NP x NP-tile kernel above would leave most of every warp idle here.
template <int NP>
struct AxSmall {
  static constexpr int kNL = NP * NP * NP;
  static constexpr int kBlock = 256;
  static constexpr int kEPB = kBlock / kNL;
  static constexpr int kNlocP = (kNL + 1) & ~1;
  static constexpr int kNS = kNL - (NP - 2) * (NP - 2) * (NP - 2);
  static constexpr int kNSP = (kNS + 3) & ~3;
};

template <int NP, bool OTF = false>
__global__ void __launch_bounds__(256) ax_small_kernel(AxArgs a)
{
  using S = AxSmall<NP>;
  constexpr int NL = S::kNL, EPB = S::kEPB, n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  constexpr int RD = AxShape<NP>::kRecD;
  __shared__ double su[EPB][NL], fa[EPB][NL], fb[EPB][NL], fc[EPB][NL];
  __shared__ double srec[OTF ? EPB : 1][RD];
  __shared__ double sD[NP * NP];
  __shared__ double red[S::kBlock / 32];
  const int tid = threadIdx.x;
  for (int q = tid; q < NP * NP; q += S::kBlock) sD[q] = c_tab[NP].D[q];
  const int el = tid / NL, l = tid % NL;
  const int i = l % NP, j = (l / NP) % NP, k = l / (NP * NP);
  const int slot = surface_slot(NP, i, j, k);
  const int ioff = slot >= 0 ? 0 : ((k - 1) * (n - 1) + (j - 1)) * (n - 1) + (i - 1);
  const bool lane_ok = el < EPB;
  __syncthreads();
  double dot = 0.0;
  for (int eb = a.e_begin + blockIdx.x * EPB; eb < a.ne; eb += gridDim.x * EPB) {
    const int e = eb + el;
    const bool act = lane_ok && e < a.ne;
    double u = 0.0, w[6] = {0, 0, 0, 0, 0, 0}, mo = 0.0;
    if constexpr (OTF) {
      for (int q = tid; q < EPB * RD; q += S::kBlock) {
        const int qe = q / RD;
        srec[qe][q % RD] = eb + qe < a.ne ? __ldg(a.erec + (long long)(eb + qe) * RD + q % RD) : 1.0;
      }
    }
    if (act) {
      if (slot >= 0)
        u = load_masked(a.u, __ldg(a.smap + (long long)e * 2 * S::kNSP + slot));  // masked (operator.cpp:264)
      else
        u = __ldg(a.u + (long long)a.num_surface_global + (long long)e * NI + ioff);
      if constexpr (!OTF) {
        const double* wp = a.wg + (long long)e * 6 * S::kNlocP + l;
#pragma unroll
        for (int p = 0; p < 6; ++p) w[p] = __ldg(wp + p * S::kNlocP);
      }
      su[el][l] = u;
    }
    __syncthreads();
    if constexpr (OTF) {
      if (act) {
        const OrderTables& T = c_tab[NP];
        double jx[3], jy[3], jz[3];
        jac_column(T, srec[el], 0, j, k, jx);
        jac_column(T, srec[el], 1, i, k, jy);
        jac_column(T, srec[el], 2, i, j, jz);
        const double rho3 = T.w[i] * T.w[j] * T.w[k];
        otf_metric(jx, jy, jz, srec[el][24] * rho3, rho3, w, mo);
      }
    }
    if (act) {  // derivatives and metric fluxes (operator.cpp:135-144)
      double sx = 0, sy = 0, sz = 0;
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        sx += sD[m * NP + i] * su[el][(k * NP + j) * NP + m];
        sy += sD[m * NP + j] * su[el][(k * NP + m) * NP + i];
        sz += sD[m * NP + k] * su[el][(m * NP + j) * NP + i];
      }
      fa[el][l] = w[0] * sx + w[1] * sy + w[2] * sz;
      fb[el][l] = w[1] * sx + w[3] * sy + w[4] * sz;
      fc[el][l] = w[2] * sx + w[4] * sy + w[5] * sz;
    }
    __syncthreads();
    if (act) {  // adjoint contractions, one accumulator (operator.cpp:152-157)
      double s = 0;
#pragma unroll
      for (int m = 0; m < NP; ++m) {
        s += sD[i * NP + m] * fa[el][(k * NP + j) * NP + m];
        s += sD[j * NP + m] * fb[el][(k * NP + m) * NP + i];
        s += sD[k * NP + m] * fc[el][(m * NP + j) * NP + i];
      }
      const double ce = __ldg(a.c_e + e);
      if (ce != 0.0) s += (ce * u) * (OTF ? mo : __ldg(a.mass + (std::size_t)e * NL + l));  // operator.cpp:159
      if (slot >= 0) {
        a.rsurf[(long long)e * S::kNSP + slot] = s;
      } else {
        a.r[(long long)a.num_surface_global + (long long)e * NI + ioff] = s;
        dot += u * s;
      }
    }
    __syncthreads();
  }
  dot_commit<S::kBlock>(a.dot, dot, red);
}

}  // namespace hxb
