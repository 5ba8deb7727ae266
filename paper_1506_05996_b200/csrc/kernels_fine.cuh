// Fine two-scale component: overlapping Schwarz subdomain solves by fast
// diagonalization (FinePreconditioner::apply, fine.cpp:210-231 with
// solve_subdomain, fine.cpp:140-185). Assembly of the subdomain outputs is
// done by combine_kernel (kernels_gather.cuh).
//
// fdm_kernel: one CTA per element subdomain of P^3 = (n+3)^3 slots, one thread
// per line (P^2 lines per direction). Separable transform in 4 shared-memory
// round trips:
//   1  gather r along an x-line straight from HBM (own nodes via the surface
//      map / closed-form interior ids, face slots via sub_face, edge/corner
//      slots 0; mesh.cpp:385-451), scale to r' (fine.cpp:161-166), apply V
//   2  V along y
//   3  V along z, pointwise 1/(4k(lx+ly+lz)+c) (fine.cpp:172-177), V^-1 along z
//   4  V^-1 along y
//   5  V^-1 along x and store each slot's value at its CSR position (sorted
//      by destination node, so the combine kernel streams it)
// The transforms along different axes commute, so running V^-1 z-first is
// the reference's x,y,z order up to rounding. V/V^-1 rows are uniform
// constant loads (transposed tables), and the padded strides below were
// chosen by exhaustive search for the fewest shared-memory wavefronts over
// all three line directions.
#pragma once

#include "kernels_common.cuh"

namespace hxb {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem)
{
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// stage n ints (16-byte aligned source and destination when n4) with the CTA's threads
template <bool V16>
__device__ __forceinline__ void stage_ints(int* dst, const int* src, int n, int tid, int nthreads)
{
  if constexpr (V16) {
    for (int q = tid; q < n / 4; q += nthreads) cp_async16(dst + 4 * q, src + 4 * q);
  } else {
    for (int q = tid; q < n; q += nthreads) cp_async4(dst + q, src + q);
  }
}

#ifndef FDM_S10
#define FDM_S10 17
#define FDM_PS10 170
#endif
template <int P>
struct FdmLayout {  // (row stride S, plane stride PS) per pencil size
  static constexpr int S = P == 6 ? 9 : P == 8 ? 9 : P == 10 ? FDM_S10 : P == 12 ? 13 : P;
  static constexpr int PS = P == 4 ? 19 : P == 6 ? 54 : P == 8 ? 72 : P == 10 ? FDM_PS10 : P == 12 ? 156 : P * S;
};

#ifndef FDM_MIN_BLOCKS
#define FDM_MIN_BLOCKS 8
#endif
// resident CTAs per SM the register budget is sized for, per order: the high
// orders spill at 8 (P = 12: 48 registers + 88 B stack, P = 13: 40 + 168 B).
// Measured alone at cfg4 sizes (profiles/r02_ab_experiments.jsonl, A/B 29):
// n=8 (NP=9) 8: 0.451, 7: 0.441 ms; n=9 (NP=10) 8: 0.841, 7: 0.755, 6: 0.743,
// 5: 0.722 ms; n=10 (NP=11) 8: 0.597, 6: 0.439, 5: 0.398, 4: 0.407 ms.
#ifndef FDM_MB9
#define FDM_MB9 7
#endif
#ifndef FDM_MB10
#define FDM_MB10 5
#endif
#ifndef FDM_MB11
#define FDM_MB11 5
#endif
template <int NP>
constexpr int fdm_min_blocks()
{
  return NP == 9 ? FDM_MB9 : NP == 10 ? FDM_MB10 : NP == 11 ? FDM_MB11 : FDM_MIN_BLOCKS;
}
template <int NP>
struct FdmShape {
  static constexpr int kP = NP + 2;
  static constexpr int kLines = kP * kP;
  static constexpr int kBlock = ((kLines + 31) / 32) * 32;
  static constexpr int kS = FdmLayout<kP>::S;
  static constexpr int kPS = FdmLayout<kP>::PS;
  static constexpr int kBuf = kP * kPS;
  static constexpr int kMinBlocks = fdm_min_blocks<NP>();  // resident CTAs per SM the register budget is sized for
};

struct FdmArgs {
  const double* r;          // N (PCG residual; masked on read)
  const int* smap;          // [e][2][nsurfp]: row 0 Dirichlet-encoded global ids
  const int* sub_face;      // NE*6*np^2, -1 none, Dirichlet-encoded
  const double* h3;         // NE*3 element dimensions
  const double* kappa_e;
  const double* c_e;
  const int* pos;           // [e][P^3] CSR position of each slot's contribution (-1: sentinel)
  double* zsort;            // contributions in CSR order (combine streams them)
  // fused coarse restriction (restrict_residual, coarse.cpp:138-162): null Rpart = off
  const double* cw;         // [e][nsurfp] surface-slot weights m_l / m_N (0 on Dirichlet slots)
  double* Rpart;            // [e][8] corner partial sums
  double* fsend = nullptr;  // distributed plans: contributions finalised by a neighbour (pos <= -2)
  int ne, sstride, num_surface_global;
  int sfstride;             // per-element stride of sub_face (6 np^2 padded to 4 ints: TMA rows)
  const int* order = nullptr;  // optional CTA -> element map (L2-friendly traversal); results do not depend on it
};

// out[q] = sum_m MT[m*P+q] in[m] (dense, m ascending = tensor_pass order)
template <int P>
__device__ __forceinline__ void pencil_apply(const double* __restrict__ MT, const double (&in)[P], double (&out)[P])
{
#pragma unroll
  for (int q = 0; q < P; ++q) out[q] = MT[q] * in[0];
#pragma unroll
  for (int m = 1; m < P; ++m)
#pragma unroll
    for (int q = 0; q < P; ++q) out[q] += MT[m * P + q] * in[m];
}

// Forward transform out = V in with the even/odd split: the pencil is
// reflection symmetric, so row d of V is even (d even) or odd (d odd) and
// V in = [FE^T (in + flip in) ; FO^T (in - flip in)] at half the FMAs.
template <int P>
__device__ __forceinline__ void pencil_fwd_eo(const double* __restrict__ FE, const double* __restrict__ FO,
                                              const double (&in)[P], double (&out)[P])
{
  constexpr int h = P / 2, mid = P & 1, NE = (P + 1) / 2, NO = P / 2;
  double ev[h + mid], od[h];
#pragma unroll
  for (int x = 0; x < h; ++x) {
    ev[x] = in[x] + in[P - 1 - x];
    od[x] = in[x] - in[P - 1 - x];
  }
  if constexpr (mid) ev[h] = in[h];
  double oe[NE], oo[NO];
#pragma unroll
  for (int a = 0; a < NE; ++a) oe[a] = FE[a] * ev[0];
#pragma unroll
  for (int x = 1; x < h + mid; ++x)
#pragma unroll
    for (int a = 0; a < NE; ++a) oe[a] += FE[x * NE + a] * ev[x];
#pragma unroll
  for (int a = 0; a < NO; ++a) oo[a] = FO[a] * od[0];
#pragma unroll
  for (int x = 1; x < h; ++x)
#pragma unroll
    for (int a = 0; a < NO; ++a) oo[a] += FO[x * NO + a] * od[x];
#pragma unroll
  for (int a = 0; a < NE; ++a) out[2 * a] = oe[a];
#pragma unroll
  for (int a = 0; a < NO; ++a) out[2 * a + 1] = oo[a];
}

// Inverse transform out = V^-1 in with the split: columns of V^-1 are even/odd.
template <int P>
__device__ __forceinline__ void pencil_inv_eo(const double* __restrict__ IE, const double* __restrict__ IO,
                                              const double (&in)[P], double (&out)[P])
{
  constexpr int h = P / 2, mid = P & 1, NE = (P + 1) / 2, NO = P / 2;
  double E[h + mid], O[h];
#pragma unroll
  for (int x = 0; x < h + mid; ++x) E[x] = IE[x] * in[0];
#pragma unroll
  for (int a = 1; a < NE; ++a)
#pragma unroll
    for (int x = 0; x < h + mid; ++x) E[x] += IE[a * (h + mid) + x] * in[2 * a];
#pragma unroll
  for (int x = 0; x < h; ++x) O[x] = IO[x] * in[1];
#pragma unroll
  for (int a = 1; a < NO; ++a)
#pragma unroll
    for (int x = 0; x < h; ++x) O[x] += IO[a * h + x] * in[2 * a + 1];
#pragma unroll
  for (int x = 0; x < h; ++x) {
    out[x] = E[x] + O[x];
    out[P - 1 - x] = E[x] - O[x];
  }
  if constexpr (mid) out[h] = E[h];
}

// EPB subdomains per CTA: lines of consecutive elements packed into the same
// warps (P^2 lines per element: at P = 6 one element per CTA leaves 28 of
// 64 lanes idle). Used when the restriction is not fused (the Rpart/fsend
// paths reduce per element over whole warps and keep EPB = 1), and only where
// one subdomain per CTA leaves most lanes idle: measured at cfg4 sizes
// (profiles/r02_ab_experiments.jsonl, A/B 10), packing took n=3 (P=6) from
// 1.89 to 1.62 ms but lost at n=4..8 (e.g. n=7: 1.23 -> 1.34 ms), where the
// extra shared memory per CTA costs more occupancy than the idle lanes.
template <int NP>
struct FdmEPB {
  static constexpr int kP = NP + 2;
  static constexpr int value = (kP == 4 || kP == 6) ? 256 / (kP * kP) : 1;
};
template <int NP, int EPB>
struct FdmShapeE {
  static constexpr int kLines = (NP + 2) * (NP + 2);
  static constexpr int kBlock = ((EPB * kLines + 31) / 32) * 32;
  static constexpr int kMinBlocks =
      EPB == 1 ? fdm_min_blocks<NP>() : ((FDM_MIN_BLOCKS * 128) / kBlock > 0 ? (FDM_MIN_BLOCKS * 128) / kBlock : 1);
};

template <int NP, bool EO, int EPB = 1>
__global__ void __launch_bounds__(FdmShapeE<NP, EPB>::kBlock, FdmShapeE<NP, EPB>::kMinBlocks) fdm_kernel(FdmArgs a)
{
  using Sh = FdmShape<NP>;
  constexpr int kBlk = FdmShapeE<NP, EPB>::kBlock;
  constexpr int P = Sh::kP, S = Sh::kS, PS = Sh::kPS, n = NP - 1;
  constexpr int kTab = EO ? 1 : 2 * P * P;
  __shared__ double buf_all[EPB * Sh::kBuf];
  __shared__ double tab[kTab];  // dense fallback only: V^T, V^-T as warp-uniform broadcasts
  const OrderTables& T = c_tab[NP];
  const FdmConst& C = c_fdm[NP];  // even/odd tables, lambda, 1/M: constant bank
  const int tid = threadIdx.x;
  const int es = min(tid / (P * P), EPB - 1);  // this thread's subdomain in the CTA
  const int tl = tid - es * P * P;
  const long long eidx = static_cast<long long>(blockIdx.x) * EPB + es;
  const bool ev = eidx < a.ne;
  const int e = ev ? (a.order ? __ldg(a.order + eidx) : static_cast<int>(eidx)) : 0;
  const bool lt = tid < EPB * P * P && ev;
  const int la = tl % P, lb = tl / P;
  double* buf = buf_all + es * Sh::kBuf;
  auto at = [](int x, int y, int z) { return z * PS + y * S + x; };
  if constexpr (!EO) {
    for (int q = tid; q < P * P; q += kBlk) {
      tab[q] = T.VT[q];
      tab[P * P + q] = T.ViT[q];
    }
  }
  __shared__ double s_lam[P], s_invM[P];  // the per-thread (non-uniform) indices read these; uniform ones the constant bank
  for (int q = tid; q < P; q += kBlk) {
    s_lam[q] = C.lam[q];
    s_invM[q] = C.invM[q];
  }
  auto fwd = [&](const double (&in)[P], double (&out)[P]) {
    if constexpr (EO)
      pencil_fwd_eo<P>(C.FE, C.FO, in, out);
    else
      pencil_apply<P>(tab, in, out);
  };
  auto inv = [&](const double (&in)[P], double (&out)[P]) {
    if constexpr (EO)
      pencil_inv_eo<P>(C.IE, C.IO, in, out);
    else
      pencil_apply<P>(tab + P * P, in, out);
  };

  __shared__ double s_h0[NP], s_h1[NP];   // coarse hats 0.5(1 -+ t) (gll.cpp:92)
  __shared__ double s_red[kBlk / 32][8];
  for (int q = tid; q < NP; q += kBlk) {
    s_h0[q] = T.hat0[q];
    s_h1[q] = T.hat1[q];
  }
  // the element's surface codes and face-neighbour ids (needed first) and its
  // output positions (needed last) are staged by coalesced cp.async copies
  constexpr int NS = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2), NSP = (NS + 3) & ~3;
  constexpr int NF = (6 * NP * NP + 3) & ~3, P3 = P * P * P;
  __shared__ __align__(16) int s_code_all[EPB][NSP];
  __shared__ __align__(16) int s_sf_all[EPB][NF];
  // output positions, staged by 16-byte copies (a row stride padded for the
  // pass-5 reads needed 4-byte copies: measured 4.4M extra wavefronts per
  // launch at cfg2 against 1.4M from the 2-way read conflicts it removed)
  constexpr int PR = P;
  constexpr int P3P = ((P * P * PR) + 3) & ~3;
  __shared__ __align__(16) int s_pos_all[EPB][P3P];
  __shared__ __align__(16) double s_cw[EPB == 1 ? NSP : 2];
  const int* s_code = s_code_all[es];
  const int* s_sf = s_sf_all[es];
  const int* s_pos = s_pos_all[es];
#pragma unroll 1
  for (int q = 0; q < EPB; ++q) {  // every subdomain's rows, staged by the whole CTA
    const long long ei = static_cast<long long>(blockIdx.x) * EPB + q;
    if (ei >= a.ne) break;
    const int eq = a.order ? __ldg(a.order + ei) : static_cast<int>(ei);
    stage_ints<true>(s_code_all[q], a.smap + (long long)eq * a.sstride, NSP, tid, kBlk);
    stage_ints<true>(s_sf_all[q], a.sub_face + (long long)eq * a.sfstride, NF, tid, kBlk);
  }
  if constexpr (EPB == 1) {
    if (a.Rpart)
      for (int q = tid; q < NSP / 2; q += kBlk) cp_async16(s_cw + 2 * q, a.cw + (long long)e * NSP + 2 * q);
  }
  cp_async_commit();
#pragma unroll 1
  for (int q = 0; q < EPB; ++q) {
    const long long ei = static_cast<long long>(blockIdx.x) * EPB + q;
    if (ei >= a.ne) break;
    const int eq = a.order ? __ldg(a.order + ei) : static_cast<int>(ei);
    stage_ints<(P3 % 4) == 0>(s_pos_all[q], a.pos + (long long)eq * P3, P3, tid, kBlk);
  }
  cp_async_commit();
  const double hx = __ldg(a.h3 + 3 * e), hy = __ldg(a.h3 + 3 * e + 1), hz = __ldg(a.h3 + 3 * e + 2);
  const double svol = 8.0 / (hx * hy * hz);  // fine.cpp:154
  double in[P], out[P];
  double racc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cp_async_wait_1();
  __syncthreads();

  // ---- 1: gather + r' scaling + V along x (thread = x-line (y=la, z=lb)) -------
  if (lt) {
    const int y = la, z = lb, jj = y - 1, kk = z - 1;
    const bool iny = jj >= 0 && jj <= n, inz = kk >= 0 && kk <= n;
    const int* surf = s_code;
    const int* sf = s_sf;
    const long long ibase = (long long)a.num_surface_global + (long long)e * (n - 1) * (n - 1) * (n - 1);
#pragma unroll
    for (int x = 0; x < P; ++x) in[x] = 0.0;
    if (iny && inz) {
      in[0] = load_masked(a.r, sf[(0 * NP + kk) * NP + jj]);      // face 0 slot (u=jj, w=kk)
      in[P - 1] = load_masked(a.r, sf[(1 * NP + kk) * NP + jj]);  // face 1 slot
      int gl[NP];  // own-node ids of this x-line (-1: Dirichlet, reads as 0)
#pragma unroll
      for (int ii = 0; ii <= n; ++ii) {
        const int s = surface_slot(NP, ii, jj, kk);
        if (s >= 0) {
          const int code = surf[s];
          gl[ii] = code >= 0 ? code : -1;
        } else {
          gl[ii] = static_cast<int>(ibase + ((kk - 1) * (n - 1) + (jj - 1)) * (n - 1) + (ii - 1));
        }
      }
#pragma unroll
      for (int ii = 0; ii <= n; ++ii) in[ii + 1] = gl[ii] >= 0 ? __ldg(a.r + gl[ii]) : 0.0;
      if (EPB == 1 && a.Rpart) {
        // this line's share of the 8 corner sums R_cb = sum_l B[cb][l] (r/m_N)_l m_l.
        // An element-interior node has one copy, so m_N = m_l and its term is
        // r itself (to rounding): only surface nodes read 1/m_N and m_l.
        const bool line_interior = jj > 0 && jj < n && kk > 0 && kk < n;
        double w0 = 0.0, w1 = 0.0;
#pragma unroll
        for (int ii = 0; ii <= n; ++ii) {
          double w;
          if (line_interior && ii > 0 && ii < n)
            w = in[ii + 1];
          else
            w = in[ii + 1] * s_cw[surface_slot(NP, ii, jj, kk)];  // (r/m_N) m_l as r (m_l/m_N)
          w0 += s_h0[ii] * w;
          w1 += s_h1[ii] * w;
        }
        const double hj[2] = {s_h0[jj], s_h1[jj]}, hk[2] = {s_h0[kk], s_h1[kk]};
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) racc[cb] = (hj[(cb >> 1) & 1] * hk[cb >> 2]) * ((cb & 1) ? w1 : w0);
      }
    } else if (inz && (y == 0 || y == P - 1)) {  // faces 2/3: u=kk, w=ii
      const int f = y == 0 ? 2 : 3;
#pragma unroll
      for (int ii = 0; ii <= n; ++ii) in[ii + 1] = load_masked(a.r, sf[(f * NP + ii) * NP + kk]);
    } else if (iny && (z == 0 || z == P - 1)) {  // faces 4/5: u=ii, w=jj
      const int f = z == 0 ? 4 : 5;
#pragma unroll
      for (int ii = 0; ii <= n; ++ii) in[ii + 1] = load_masked(a.r, sf[(f * NP + jj) * NP + ii]);
    }
    // r' = 8/(hx hy hz) r / (M_i M_j M_k) (fine.cpp:161-166), as products of reciprocals
    const double syz = svol * s_invM[y] * s_invM[z];
#pragma unroll
    for (int x = 0; x < P; ++x) in[x] = in[x] * (syz * C.invM[x]);  // x uniform: constant-bank operand
    fwd(in, out);
#pragma unroll
    for (int x = 0; x < P; ++x) buf[at(x, y, z)] = out[x];
  }
  if (EPB == 1 && a.Rpart) {  // fixed-tree reduction of the corner sums over the CTA's lines
#pragma unroll
    for (int cb = 0; cb < 8; ++cb)
      for (int o = 16; o > 0; o >>= 1) racc[cb] += __shfl_xor_sync(0xffffffffu, racc[cb], o);
    if ((tid & 31) == 0)
#pragma unroll
      for (int cb = 0; cb < 8; ++cb) s_red[tid >> 5][cb] = racc[cb];
  }
  __syncthreads();
  if (EPB == 1 && a.Rpart && tid < 8) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kBlk / 32; ++w) v += s_red[w][tid];
    a.Rpart[8 * (long long)e + tid] = v;
  }

  // ---- 2: V along y (thread = y-line (x=la, z=lb)) ----------------------------
  if (lt) {
#pragma unroll
    for (int y = 0; y < P; ++y) in[y] = buf[at(la, y, lb)];
    fwd(in, out);
#pragma unroll
    for (int y = 0; y < P; ++y) buf[at(la, y, lb)] = out[y];
  }
  __syncthreads();

  // ---- 3: V along z, eigenvalue division, V^-1 along z (thread = (x=la, y=lb)) --
  if (lt) {
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy), ihz2 = 1.0 / (hz * hz);
    const double kappa4 = 4.0 * __ldg(a.kappa_e + e), ce = __ldg(a.c_e + e);
    const double lxy = s_lam[la] * ihx2 + s_lam[lb] * ihy2;
#pragma unroll
    for (int z = 0; z < P; ++z) in[z] = buf[at(la, lb, z)];
    fwd(in, out);
#pragma unroll
    for (int z = 0; z < P; ++z) out[z] = out[z] * __drcp_rn(kappa4 * (lxy + C.lam[z] * ihz2) + ce);
    inv(out, in);
#pragma unroll
    for (int z = 0; z < P; ++z) buf[at(la, lb, z)] = in[z];
  }
  __syncthreads();

  // ---- 4: V^-1 along y ----------------------------------------------------------
  if (lt) {
#pragma unroll
    for (int y = 0; y < P; ++y) in[y] = buf[at(la, y, lb)];
    inv(in, out);
#pragma unroll
    for (int y = 0; y < P; ++y) buf[at(la, y, lb)] = out[y];
  }
  cp_async_wait_all();  // output positions staged
  __syncthreads();

  // ---- 5: V^-1 along x, store --------------------------------------------------
  if (lt) {
#pragma unroll
    for (int x = 0; x < P; ++x) in[x] = buf[at(x, la, lb)];
    inv(in, out);
    const int* ps = s_pos + (lb * P + la) * PR;
#pragma unroll
    for (int x = 0; x < P; ++x) {
      const int q = ps[x];
      if (q >= 0)
        a.zsort[q] = out[x];
      else if (EPB == 1 && q <= -2)  // finalised by a neighbour rank (distributed plans)
        a.fsend[-2 - q] = out[x];
    }
  }
}

// ---------------------------------------------------------------------------
}  // namespace hxb
