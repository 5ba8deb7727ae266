// Deterministic gathers over sorted CSR lists (no atomics): the assembly
// step of every scatter-add in the reference, replayed in the reference's
// summation order (copies in ascending source index, mesh.cpp:463-475).
//
// warp_csr_sum: a warp owns 32 consecutive destination nodes. Their source
// lists are contiguous in idx[], so the warp loads the index segment
// coalesced, gathers all source values in parallel into a per-warp staging
// buffer (high memory-level parallelism), and each lane then sums its own
// node's entries sequentially from shared memory — the same left-to-right
// order as the reference loop.
#pragma once

#include "kernels_common.cuh"

namespace hxb {

constexpr int kGatherBlock = 256;
constexpr int kGatherCap = 320;  // staged values per warp (avg ~1.5-2.6 per node)


// Sums for a warp's 32 consecutive nodes of values scattered in an E-vector: src(idx[q]) gathered by the warp
// (coalesced index segment, parallel value loads), then per-lane sequential sums.
template <class Src>
__device__ __forceinline__ double warp_csr_sum(const unsigned* __restrict__ off, const int* __restrict__ idx, Src&& src,
                                               int g0, int n, double* __restrict__ stage)
{
  const int lane = threadIdx.x & 31;
  const int g = g0 + lane;
  const unsigned my0 = __ldg(off + min(g, n));
  const unsigned my1 = __ldg(off + min(g + 1, n));
  const unsigned base = __shfl_sync(0xffffffffu, my0, 0);
  const unsigned end = __shfl_sync(0xffffffffu, my1, 31);
  const unsigned cnt = end - base;
  double s = 0.0;
  if (cnt <= static_cast<unsigned>(kGatherCap)) {
#pragma unroll 4
    for (unsigned c = lane; c < cnt; c += 32) stage[c] = src(__ldg(idx + base + c));
    __syncwarp();
    for (unsigned q = my0 - base; q < my1 - base; ++q) s += stage[q];
    __syncwarp();
  } else {
    for (unsigned q = my0; q < my1; ++q) s += src(__ldg(idx + q));
  }
  return s;
}

// ---------------------------------------------------------------------------
// Ax surface assembly (gather, mesh.cpp:463-475) + Dirichlet identity rows
// (operator.cpp:279-280) + the optional fused p.Ap partial.
struct AxGatherArgs {
  const double* rsurf;   // [e][nsurfp] surface E-vector (ax_elem_kernel)
  const unsigned* off;   // num_surface_global + 1
  const int* idx;        // e*nsurfp + slot, ascending per node
  const double* u;
  const std::uint8_t* mask;
  double* r;
  int num_surface_global;  // one past the last node gathered (off has one more entry)
  const int* nodes;        // null: node t is global id t; else global id of local node t
  DotArgs dot;
  int t_begin = 0;         // first node gathered (a sub-range of the surface nodes)
};

__global__ void __launch_bounds__(kGatherBlock) ax_gather_kernel(AxGatherArgs a)
{
  __shared__ double red[kGatherBlock / 32];
  __shared__ double stage[kGatherBlock / 32][kGatherCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kGatherBlock / 32);
  double dot = 0.0;
  for (int g0 = a.t_begin + (blockIdx.x * (kGatherBlock / 32) + warp) * 32; g0 < a.num_surface_global;
       g0 += nwarps * 32) {
    const double s = warp_csr_sum(a.off, a.idx, [&](int q) { return __ldg(a.rsurf + q); }, g0,
                                  a.num_surface_global, stage[warp]);
    const int t = g0 + lane;
    if (t < a.num_surface_global) {
      const int g = a.nodes ? __ldg(a.nodes + t) : t;
      const double ug = __ldg(a.u + g);
      const double rg = __ldg(a.mask + g) ? ug : s;
      a.r[g] = rg;
      dot += ug * rg;
    }
  }
  dot_commit<kGatherBlock>(a.dot, dot, red);
}

// ---------------------------------------------------------------------------
// Distributed Ax (element-slab partition). A node shared by ranks
// r and r+1 has its copies in ascending element order, so rank r's copies
// come first: rank r sums them (partial), rank r+1 continues the same
// left-to-right sum with its own copies and finalises (mask), and returns the
// final value. The result is bit-identical to the single-plan gather.

// send[t] = sum of this rank's copies of up-interface node t (no mask: not final)
__global__ void dist_partial_kernel(const unsigned* __restrict__ off, const int* __restrict__ idx,
                                    const double* __restrict__ rsurf, int n, double* __restrict__ send)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (unsigned q = __ldg(off + t); q < __ldg(off + t + 1); ++q) s += __ldg(rsurf + __ldg(idx + q));
    send[t] = s;
  }
}

// down-interface node t: continue the lower rank's partial with this rank's
// copies, apply the Dirichlet identity, store and return the final value
__global__ void dist_continue_kernel(const unsigned* __restrict__ off, const int* __restrict__ idx,
                                     const double* __restrict__ rsurf, const int* __restrict__ nodes, int n,
                                     const double* __restrict__ u, const std::uint8_t* __restrict__ mask,
                                     const double* __restrict__ recv, double* __restrict__ r, double* __restrict__ send)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    double s = __ldg(recv + t);
    for (unsigned q = __ldg(off + t); q < __ldg(off + t + 1); ++q) s += __ldg(rsurf + __ldg(idx + q));
    const int g = __ldg(nodes + t);
    const double v = __ldg(mask + g) ? __ldg(u + g) : s;
    r[g] = v;
    send[t] = v;
  }
}

// --- distributed preconditioned CG helpers ----------------------------------
// x[list[t]] -> buf[t]
__global__ void dist_pack_kernel(const int* __restrict__ list, int n, const double* __restrict__ x, double* __restrict__ buf)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) buf[t] = __ldg(x + __ldg(list + t));
}
// buf[t] -> x[list[t]]
__global__ void dist_unpack_kernel(const int* __restrict__ list, int n, const double* __restrict__ buf, double* __restrict__ x)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) x[__ldg(list + t)] = __ldg(buf + t);
}
// local vector updates over the rank's nodes: surface list + interior range
//   mode 0: r = b, u = 0              (krylov.cpp:29-30)
//   mode 1: u += a p, r -= a f        (krylov.cpp:53-56)
//   mode 2: p = z + a p               (krylov.cpp:64-66)
//   mode 3: p = z                     (krylov.cpp:38)
// a_num/a_den (device scalars, optional): a = *a_num / *a_den, computed on the
// device (alpha = zr/pf, beta = zr_next/zr of krylov.cpp:53,64); mode 1 is a
// no-op when *a_den <= 0 (the breakdown exit of krylov.cpp:46-51 skips the update)
__global__ void dist_vec_kernel(int mode, const int* __restrict__ list, int nlist, int ib0, int ib1, double a,
                                const double* __restrict__ x0, const double* __restrict__ x1, double* __restrict__ y0,
                                double* __restrict__ y1, const double* __restrict__ a_num = nullptr,
                                const double* __restrict__ a_den = nullptr)
{
  if (a_num) {
    const double den = *a_den;
    if (mode == 1 && !(den > 0)) return;
    a = *a_num / den;
  }
  const int total = nlist + (ib1 - ib0);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int g = t < nlist ? __ldg(list + t) : ib0 + (t - nlist);
    if (mode == 0) {
      y0[g] = x0[g];
      y1[g] = 0.0;
    } else if (mode == 1) {
      y1[g] += a * x0[g];   // u (y1) += a p (x0)
      y0[g] -= a * x1[g];   // r (y0) -= a f (x1)
    } else if (mode == 2) {
      y0[g] = x0[g] + a * y0[g];
    } else {
      y0[g] = x0[g];
    }
  }
}
// partial dot over the rank's finalised nodes (each global node counted once)
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) dist_dot_kernel(const int* __restrict__ list, int nlist, int ib0, int ib1,
                                                        const double* __restrict__ x, const double* __restrict__ y,
                                                        DotArgs d)
{
  __shared__ double red[BLOCK / 32];
  const int total = nlist + (ib1 - ib0);
  double s = 0.0;
  for (int t = blockIdx.x * BLOCK + threadIdx.x; t < total; t += gridDim.x * BLOCK) {
    const int g = t < nlist ? __ldg(list + t) : ib0 + (t - nlist);
    s += __ldg(x + g) * __ldg(y + g);
  }
  dot_commit<BLOCK>(d, s, red);
}
// sum of the ranks' partial scalars in rank order (every rank computes the
// same value: the deterministic all-reduce of the in-process transport)
__global__ void sum_partials_kernel(const double* __restrict__ parts, int R, double* __restrict__ out)
{
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < R; ++q) s += parts[q];
    *out = s;
  }
}
// neighbours' fine contributions into their sum positions
__global__ void dist_fine_scatter_kernel(const int* __restrict__ pos, int n, const double* __restrict__ recv,
                                         double* __restrict__ zsort)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) zsort[__ldg(pos + t)] = __ldg(recv + t);
}

// up-interface node t: the final value computed by the upper rank
__global__ void dist_finish_kernel(const int* __restrict__ nodes, int n, const double* __restrict__ recv,
                                   double* __restrict__ r)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) r[__ldg(nodes + t)] = __ldg(recv + t);
}

// Two-scale combine with the coarse prolongation fused in (precond.cpp:57-66,
// prolongate coarse.cpp:164-186): per node g
//   zf = sum of its subdomain contributions in (e, slot) order (fine.cpp:224-227)
//   zc = (sum over its copies (e,l), in (e,l) order, of
//         (sum_cb B[cb][l] Zc[e][cb]) * m[e][l]) / m_N[g]
//   z  = mask ? r : (0 + zf) + zc ;  z.r partial
// Element-interior nodes have one copy whose (e,l) follows from g
// (interior ids are (e, local)-ordered, mesh.cpp:283); surface nodes walk
// their Ax gather list (ax_idx = e*nsurfp + slot).
struct CombineProlongArgs {
  const double* r;
  const std::uint8_t* mask;
  const double* zsort;
  const unsigned* fine_off;
  const unsigned* ax_off;
  const int* ax_idx;
  const double* Zc;
  const double* mass;      // [e][nloc] (element-interior copies)
  const double* mass_csr;  // surface copies, Ax-CSR order
  const double* lumped;
  const double* inv_lumped;
  double* z;
  int N, nsg;
  int do_fine, do_coarse;
  int fine_in_z = 0;  // the fine sums are already in z (combine_fine_kernel ran concurrently with the coarse solve)
  DotArgs dot;
  // item t -> node: t < nsg: surface node (surf_nodes ? surf_nodes[t] : t),
  // t >= nsg: interior node ibase + (t - nsg) of element (t - nsg)/NI + e0;
  // the distributed plan runs over its finalised nodes only
  const int* surf_nodes = nullptr;
  int ibase = 0;    // global id of the first interior item
  int e0 = 0;       // global id of the first element whose mass block is at `mass`
};

#ifndef COMBINE_MIN_BLOCKS
#define COMBINE_MIN_BLOCKS 6  // cfg2: 6 (40 regs, 100 B spills) 0.857 ms, 4 (64 regs) 0.937, 8 (32 regs) 1.024
#endif
template <int NP>
__global__ void __launch_bounds__(kGatherBlock, COMBINE_MIN_BLOCKS) combine_prolong_kernel(CombineProlongArgs a)
{
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  constexpr int NS = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2), NSP = (NS + 3) & ~3;
  __shared__ double red[kGatherBlock / 32];
  __shared__ double h0[NP], h1[NP];
  if (threadIdx.x < NP) {
    h0[threadIdx.x] = c_tab[NP].hat0[threadIdx.x];
    h1[threadIdx.x] = c_tab[NP].hat1[threadIdx.x];
  }
  __syncthreads();
  // prolongated value of copy (e; i,j,k) before the mass: sum_cb B[cb][l] Zc[e][cb] (coarse.cpp:176-179)
  auto pz = [&](long long e, int i, int j, int k) {
    const double2* zc2 = reinterpret_cast<const double2*>(a.Zc + 8 * e);
    const double2 c01 = __ldg(zc2), c23 = __ldg(zc2 + 1), c45 = __ldg(zc2 + 2), c67 = __ldg(zc2 + 3);
    const double zc[8] = {c01.x, c01.y, c23.x, c23.y, c45.x, c45.y, c67.x, c67.y};
    const double hi[2] = {h0[i], h1[i]}, hj[2] = {h0[j], h1[j]}, hk[2] = {h0[k], h1[k]};
    double s = 0.0;
#pragma unroll
    for (int cb = 0; cb < 8; ++cb) s += hi[cb & 1] * hj[(cb >> 1) & 1] * hk[cb >> 2] * zc[cb];
    return s;
  };
  double dot = 0.0;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < a.N; it += gridDim.x * blockDim.x) {
    const bool surf = it < a.nsg;
    const int g = surf ? (a.surf_nodes ? __ldg(a.surf_nodes + it) : it) : a.ibase + (it - a.nsg);
    const double rg = __ldg(a.r + g);
    double zg;
    if (surf && __ldg(a.mask + g)) {  // Dirichlet nodes are element-surface nodes
      zg = rg;
    } else {
      double s = 0.0;
      if (a.fine_in_z) {
        s = a.z[g];
      } else if (a.do_fine) {
        // up to 8 contributions loaded at once (predicated), summed in list order
        const unsigned q0 = __ldg(a.fine_off + it), q1 = __ldg(a.fine_off + it + 1);
        double v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) v[t] = q0 + t < q1 ? __ldcs(a.zsort + q0 + t) : 0.0;
        double zf = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (q0 + t < q1) zf += v[t];
        for (unsigned q = q0 + 8; q < q1; ++q) zf += __ldcs(a.zsort + q);
        s += zf;
      }
      if (a.do_coarse) {
        double zc = 0.0;
        if (!surf) {
          if constexpr (NI > 0) {
            const int t = it - a.nsg;  // interior ids are (e, local)-ordered (mesh.cpp:283)
            const long long el = t / NI;          // element relative to e0
            const int l = t % NI;
            const int i = 1 + l % (n - 1), j = 1 + (l / (n - 1)) % (n - 1), k = 1 + l / ((n - 1) * (n - 1));
            // single copy: (B zc) m / m_N with m_N = m is B zc to rounding (coarse.cpp:180, 185)
            zc = pz(el + a.e0, i, j, k);
          }
        } else {
          // face nodes (2 copies) dominate: the first two copies are evaluated
          // independently, the rest (edges 4, vertices 8+) in order after them
          const unsigned c0 = __ldg(a.ax_off + it), c1 = __ldg(a.ax_off + it + 1);
          const int x0 = __ldg(a.ax_idx + c0);
          const int x1 = c0 + 1 < c1 ? __ldg(a.ax_idx + c0 + 1) : x0;
          int i0, j0, k0, i1, j1, k1;
          surface_ijk<NP>(x0 % NSP, i0, j0, k0);
          surface_ijk<NP>(x1 % NSP, i1, j1, k1);
          const double m0 = __ldcs(a.mass_csr + c0);
          const double m1 = c0 + 1 < c1 ? __ldcs(a.mass_csr + c0 + 1) : 0.0;
          const double p0 = pz(x0 / NSP, i0, j0, k0) * m0;
          const double p1 = pz(x1 / NSP, i1, j1, k1) * m1;
          zc += p0;
          if (c0 + 1 < c1) zc += p1;
          for (unsigned q = c0 + 2; q < c1; ++q) {
            const int c = __ldg(a.ax_idx + q);
            int i, j, k;
            surface_ijk<NP>(c % NSP, i, j, k);
            zc += pz(c / NSP, i, j, k) * __ldcs(a.mass_csr + q);
          }
        }
        s += surf ? zc * __ldg(a.inv_lumped + g) : zc;  // /m_N (coarse.cpp:185) as a product with 1/m_N
      }
      zg = s;
    }
    a.z[g] = zg;
    dot += zg * rg;
  }
  dot_commit<kGatherBlock>(a.dot, dot, red);
}

// First half of the split combine: z[g] = sum of node g's fine contributions
// in list order (the do_fine branch of combine_prolong_kernel, same
// arithmetic). It runs while the coarse solve occupies a few SMs; the coarse
// half then reads z back (fine_in_z), so the result is bit-identical to the
// fused kernel. One item per thread, no persistent loop, so the coarse
// kernels on the high-priority stream are scheduled as soon as CTAs retire.

__global__ void __launch_bounds__(kGatherBlock) combine_fine_kernel(const double* __restrict__ zsort,
                                                                    const unsigned* __restrict__ fine_off,
                                                                    const int* __restrict__ surf_nodes, int nsg,
                                                                    int ibase, int n_items, double* __restrict__ z,
                                                                    PcgUArgs ua)
{
  const double alpha = ua.u ? ua.zr[ua.k] / ua.pf[ua.k] : 0.0;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += gridDim.x * blockDim.x) {
  const int g = it < nsg ? (surf_nodes ? __ldg(surf_nodes + it) : it) : ibase + (it - nsg);
  const unsigned q0 = __ldg(fine_off + it), q1 = __ldg(fine_off + it + 1);
  double v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) v[t] = q0 + t < q1 ? __ldcs(zsort + q0 + t) : 0.0;
  double zf = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (q0 + t < q1) zf += v[t];
  for (unsigned q = q0 + 8; q < q1; ++q) zf += __ldcs(zsort + q);
  z[g] = zf;
  if (ua.u) ua.u[g] += alpha * ua.p[g];
  }
}

// R[v] = vmask[v] ? 0 : sum of Rpart over (e,cb) incidences in ascending order
// (restrict_residual accumulation, coarse.cpp:155-160, then coarse.cpp:191-192)
__global__ void vertex_gather_kernel(const double* __restrict__ Rpart, const unsigned* __restrict__ off,
                                     const int* __restrict__ idx, const std::uint8_t* __restrict__ vmask,
                                     double* __restrict__ R, int nv)
{
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (unsigned q = __ldg(off + v); q < __ldg(off + v + 1); ++q) s += __ldg(Rpart + __ldg(idx + q));
    R[v] = __ldg(vmask + v) ? 0.0 : s;
  }
}

}  // namespace hxb
