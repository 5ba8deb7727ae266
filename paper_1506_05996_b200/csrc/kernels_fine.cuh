// Fine two-scale component: overlapping Schwarz subdomain solves by fast
// diagonalization (FinePreconditioner::apply, fine.cpp:210-231 with
// solve_subdomain, fine.cpp:140-185), and the combine kernel that assembles
// z = zf + zc in reference order (precond.cpp:57-66) with the coarse
// prolongation (coarse.cpp:164-186) fused into the same per-node pass.
//
// fdm_kernel: one CTA per element subdomain of P^3 = (n+3)^3 slots.
//   load  r' = svol * r / (M_i M_j M_k) for interior-region slots (own nodes,
//         masked) and face slots (neighbour's first interior layer, sub_face);
//         edge/corner slots read 0 (mesh.cpp:385-451)
//   6 line passes (V along x,y,z; pointwise 1/(4k(..)+c) fused into the z pass;
//         V^-1 along x,y,z): thread = one line, P inputs in registers, P outputs;
//         V/V^-1 entries are constant-memory operands (fully unrolled)
//   store z_sub[e*P^3 + slot] (every slot; sentinel slots are never gathered)
#pragma once

#include "kernels_common.cuh"

namespace hxb {

template <int NP>
struct FdmShape {
  static constexpr int kP = NP + 2;
  static constexpr int kLines = kP * kP;
  static constexpr int kBlock = ((kLines + 31) / 32) * 32;
  static constexpr int kS = kP | 1;
  static constexpr int kBuf = kP * kP * kS;
};

struct FdmArgs {
  const double* r;          // N (PCG residual; masked on read)
  const int* l2g_surf;      // NE*nsurf, Dirichlet-encoded
  const int* sub_face;      // NE*6*np^2, -1 none, Dirichlet-encoded
  const double* h3;         // NE*3 element dimensions
  const double* kappa_e;
  const double* c_e;
  double* zsub;             // NE*P^3
  int ne, nsurf, num_surface_global;
};

template <int NP>
__global__ void __launch_bounds__(FdmShape<NP>::kBlock) fdm_kernel(FdmArgs a)
{
  using Sh = FdmShape<NP>;
  constexpr int P = Sh::kP, S = Sh::kS, n = NP - 1;
  __shared__ double buf[Sh::kBuf];
  const OrderTables& T = c_tab[NP];
  const int e = blockIdx.x;
  const int tid = threadIdx.x;

  const double hx = __ldg(a.h3 + 3 * e), hy = __ldg(a.h3 + 3 * e + 1), hz = __ldg(a.h3 + 3 * e + 2);
  const double svol = 8.0 / (hx * hy * hz);  // fine.cpp:154

  // ---- load r' into the extended block (fine.cpp:221-222, 161-166) ----------
  const int* surf = a.l2g_surf + (long long)e * a.nsurf;
  const int* sf = a.sub_face + (long long)e * 6 * NP * NP;
  const long long ibase = (long long)a.num_surface_global + (long long)e * (n - 1) * (n - 1) * (n - 1);
  for (int q = tid; q < P * P * P; q += Sh::kBlock) {
    const int x = q % P, y = (q / P) % P, z = q / (P * P);
    const int ii = x - 1, jj = y - 1, kk = z - 1;
    const bool ox = (ii < 0 || ii > n), oy = (jj < 0 || jj > n), oz = (kk < 0 || kk > n);
    const int nout = ox + oy + oz;
    double v = 0.0;
    if (nout == 0) {
      const int s = surface_slot(NP, ii, jj, kk);
      if (s < 0)
        v = __ldg(a.r + ibase + ((kk - 1) * (n - 1) + (jj - 1)) * (n - 1) + (ii - 1));
      else
        v = load_masked(a.r, __ldg(surf + s));
    } else if (nout == 1) {
      int f, u, w;
      if (ox) {
        f = ii < 0 ? 0 : 1;
        u = jj;
        w = kk;
      } else if (oy) {
        f = jj < 0 ? 2 : 3;
        u = kk;
        w = ii;
      } else {
        f = kk < 0 ? 4 : 5;
        u = ii;
        w = jj;
      }
      const int code = __ldg(sf + (f * NP + w) * NP + u);
      v = load_masked(a.r, code);
    }
    buf[(z * P + y) * S + x] = svol * v / (T.M[x] * T.M[y] * T.M[z]);
  }
  __syncthreads();

  const int la = tid % P, lb = tid / P;
  const bool line_thread = tid < Sh::kLines;
  double line[P];

  // pass along x with matrix Mt (fine.cpp:98-112)
  auto pass_x = [&](const double* Mt) {
    if (line_thread) {
#pragma unroll
      for (int x = 0; x < P; ++x) line[x] = buf[(lb * P + la) * S + x];
#pragma unroll
      for (int d = 0; d < P; ++d) {
        double s = 0.0;
#pragma unroll
        for (int x = 0; x < P; ++x) s += Mt[d * P + x] * line[x];
        buf[(lb * P + la) * S + d] = s;
      }
    }
    __syncthreads();
  };
  auto pass_y = [&](const double* Mt) {  // fine.cpp:113-121
    if (line_thread) {
#pragma unroll
      for (int y = 0; y < P; ++y) line[y] = buf[(lb * P + y) * S + la];
#pragma unroll
      for (int d = 0; d < P; ++d) {
        double s = 0.0;
#pragma unroll
        for (int y = 0; y < P; ++y) s += Mt[d * P + y] * line[y];
        buf[(lb * P + d) * S + la] = s;
      }
    }
    __syncthreads();
  };

  pass_x(T.V);
  pass_y(T.V);
  // z pass with V, then the pointwise division (fine.cpp:172-177)
  if (line_thread) {
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy), ihz2 = 1.0 / (hz * hz);
    const double kappa4 = 4.0 * __ldg(a.kappa_e + e), ce = __ldg(a.c_e + e);
    const double lx = T.lam[la] * ihx2, ly = T.lam[lb] * ihy2;
#pragma unroll
    for (int z = 0; z < P; ++z) line[z] = buf[(z * P + lb) * S + la];
#pragma unroll
    for (int d = 0; d < P; ++d) {
      double s = 0.0;
#pragma unroll
      for (int z = 0; z < P; ++z) s += T.V[d * P + z] * line[z];
      buf[(d * P + lb) * S + la] = s / (kappa4 * (lx + ly + T.lam[d] * ihz2) + ce);
    }
  }
  __syncthreads();
  pass_x(T.Vi);
  pass_y(T.Vi);
  if (line_thread) {
#pragma unroll
    for (int z = 0; z < P; ++z) line[z] = buf[(z * P + lb) * S + la];
    double* out = a.zsub + (long long)e * P * P * P;
#pragma unroll
    for (int d = 0; d < P; ++d) {
      double s = 0.0;
#pragma unroll
      for (int z = 0; z < P; ++z) s += T.Vi[d * P + z] * line[z];
      out[(d * P + lb) * P + la] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Combine: z[g] = mask ? r : (0 + zf) + zc  (precond.cpp:57-66), with
//   zf = sum of z_sub over the node's subdomain slots in ascending
//        (e, slot) order (fine.cpp:224-227 accumulation order)
//   zc = (sum over copies (e,l) in (e,l) order of (sum_cb B[cb][l] Z[v_cb]) * m_l) / m_N
//        (coarse.cpp:164-186)
// and the fused z.r partial (krylov.cpp:37/62).
struct CombineArgs {
  const double* r;
  const std::uint8_t* mask;
  // fine
  const double* zsub;
  const unsigned* fine_off;   // N+1
  const int* fine_idx;        // e*P^3 + slot
  // coarse prolongation
  const double* Z;            // NV
  const int* conn;            // NE*8 (Gmsh corner order)
  const double* mass;         // NE*nloc
  const double* lumped;       // N
  const unsigned* ax_off;     // num_surface_global+1
  const int* ax_idx;          // e*nsurf + slot
  const short* surf_local;    // nsurf: slot -> local node index
  double* z;
  int N, num_surface_global, nsurf;
  int do_fine, do_coarse;
  DotArgs dot;
};

template <int NP>
__device__ __forceinline__ double prolong_copy(const CombineArgs& a, int e, int l)
{
  const OrderTables& T = c_tab[NP];
  const int i = l % NP, j = (l / NP) % NP, k = l / (NP * NP);
  const int* cn = a.conn + 8 * e;
  // B[cb][l] = hat(ci,t_i) hat(cj,t_j) hat(ck,t_k), gll.cpp:89-104
  const double hi[2] = {T.hat0[i], T.hat1[i]};
  const double hj[2] = {T.hat0[j], T.hat1[j]};
  const double hk[2] = {T.hat0[k], T.hat1[k]};
  double s = 0.0;
#pragma unroll
  for (int cb = 0; cb < 8; ++cb) {
    constexpr int kCorner[8] = {0, 1, 3, 2, 4, 5, 7, 6};
    const double b = hi[cb & 1] * hj[(cb >> 1) & 1] * hk[(cb >> 2) & 1];
    s += b * __ldg(a.Z + __ldg(cn + kCorner[cb]));
  }
  return s * __ldg(a.mass + (std::size_t)e * NP * NP * NP + l);
}

template <int NP, int BLOCK>
__global__ void __launch_bounds__(BLOCK) combine_kernel(CombineArgs a)
{
  constexpr int n = NP - 1, nint = (n - 1) * (n - 1) * (n - 1);
  __shared__ double red[BLOCK / 32];
  double dot = 0.0;
  for (int g = blockIdx.x * BLOCK + threadIdx.x; g < a.N; g += gridDim.x * BLOCK) {
    const double rg = __ldg(a.r + g);
    double zg;
    if (__ldg(a.mask + g)) {
      zg = rg;
    } else {
      double s = 0.0;
      if (a.do_fine) {
        double zf = 0.0;
        const unsigned q0 = __ldg(a.fine_off + g), q1 = __ldg(a.fine_off + g + 1);
        for (unsigned q = q0; q < q1; ++q) zf += __ldg(a.zsub + __ldg(a.fine_idx + q));
        s += zf;
      }
      if (a.do_coarse) {
        double zc = 0.0;
        if (g < a.num_surface_global) {
          const unsigned q0 = __ldg(a.ax_off + g), q1 = __ldg(a.ax_off + g + 1);
          for (unsigned q = q0; q < q1; ++q) {
            const int ent = __ldg(a.ax_idx + q);
            const int e = ent / a.nsurf;
            zc += prolong_copy<NP>(a, e, __ldg(a.surf_local + (ent - e * a.nsurf)));
          }
        } else {
          if constexpr (nint > 0) {
            const int q = g - a.num_surface_global;
            const int e = q / nint, rem = q - e * nint;
            const int ii = rem % (n - 1) + 1, jj = (rem / (n - 1)) % (n - 1) + 1, kk = rem / ((n - 1) * (n - 1)) + 1;
            zc = prolong_copy<NP>(a, e, (kk * NP + jj) * NP + ii);
          }
        }
        s += zc / __ldg(a.lumped + g);
      }
      zg = s;
    }
    a.z[g] = zg;
    dot += zg * rg;
  }
  dot_commit<BLOCK>(a.dot, dot, red);
}

}  // namespace hxb
