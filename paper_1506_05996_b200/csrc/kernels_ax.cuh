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
  static constexpr int kMinBlocks = NP <= 8 ? 6 : 2;  // caps registers; shared memory sets the real limit
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

// Persistent: CTA b processes elements b, b+grid, ... . The element's six
// metric planes (6*nloc FP64, the bulk of Ax traffic) and its surface index
// block are streamed into shared memory by TMA bulk copies issued one element
// ahead (planes for e' once phase C of e has consumed them, indices for e''
// once u(e') has been gathered), and u(e') is gathered into registers during
// phase D of e, so HBM traffic overlaps the contractions. D and D^T live in
// shared memory and are read as warp-uniform broadcasts, keeping registers
// low enough for 6 CTAs per SM.
template <int NP>
__global__ void __launch_bounds__(AxShape<NP>::kBlock, AxShape<NP>::kMinBlocks) ax_elem_kernel(AxArgs a)
{
  using Sh = AxShape<NP>;
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1), NLP = Sh::kNlocP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sG = reinterpret_cast<double*>(smem_raw);                  // [6][nlocp]
  double* sa = sG + 6 * NLP;
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
    mbar_expect_tx(&bar[0], Sh::kGBytes);
    bulk_g2s(sG, a.wg + (long long)e * 6 * NLP, Sh::kGBytes, &bar[0]);
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
    mbar_wait(&bar[0], phase);
    if (lane_ok) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int l = (k * NP + j) * NP + i;
        const double w0 = sG[l], w1 = sG[NLP + l], w2 = sG[2 * NLP + l];
        const double w3 = sG[3 * NLP + l], w4 = sG[4 * NLP + l], w5 = sG[5 * NLP + l];
        const int pa = lay_a<NP>(k, j, i), pb = lay_b<NP>(k, j, i);
        const double sx = sa[pa], sy = sb[pb], sz = fz[k];
        sa[pa] = w0 * sx + w1 * sy + w2 * sz;
        sb[pb] = w1 * sx + w3 * sy + w4 * sz;
        fz[k] = w2 * sx + w4 * sy + w5 * sz;
      }
    }
    __syncthreads();  // sG consumed
    if (tid == 0 && en < a.ne) {
      fence_proxy_async_smem();
      mbar_expect_tx(&bar[0], Sh::kGBytes);
      bulk_g2s(sG, a.wg + (long long)en * 6 * NLP, Sh::kGBytes, &bar[0]);
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
        if (ce != 0.0) r += (ce * ucol[k]) * __ldg(m0 + k * NP * NP);  // operator.cpp:159
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

template <int NP>
__global__ void __launch_bounds__(256) ax_small_kernel(AxArgs a)
{
  using S = AxSmall<NP>;
  constexpr int NL = S::kNL, EPB = S::kEPB, n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  __shared__ double su[EPB][NL], fa[EPB][NL], fb[EPB][NL], fc[EPB][NL];
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
    double u = 0.0, w[6] = {0, 0, 0, 0, 0, 0};
    if (act) {
      if (slot >= 0)
        u = load_masked(a.u, __ldg(a.smap + (long long)e * 2 * S::kNSP + slot));  // masked (operator.cpp:264)
      else
        u = __ldg(a.u + (long long)a.num_surface_global + (long long)e * NI + ioff);
      const double* wp = a.wg + (long long)e * 6 * S::kNlocP + l;
#pragma unroll
      for (int p = 0; p < 6; ++p) w[p] = __ldg(wp + p * S::kNlocP);
      su[el][l] = u;
    }
    __syncthreads();
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
      if (ce != 0.0) s += (ce * u) * __ldg(a.mass + (std::size_t)e * NL + l);  // operator.cpp:159
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
