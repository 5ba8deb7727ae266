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
//   zc = the Q1 prolongation of the coarse solution at g
//   z  = mask ? r : (0 + zf) + zc ;  z.r partial
// The reference forms zc as the mass-weighted average over g's copies,
// (sum_(e,l) (B Zc_e)_l m_l) / m_N. The Q1 interpolant is continuous across
// element faces (a shared face's values depend only on its four vertices), so
// every copy carries the same value to rounding and the average is that value
// to rounding: the combine evaluates it once, at the node's first copy (for an
// element-interior node, its only copy). That drops the per-copy mass and
// index streams (0.5 GB per apply at cfg2); the bitwise-reference mode
// (compat.cu) keeps the reference's weighted form.
//
// Warp per 32 consecutive nodes: their contribution lists are one contiguous
// zsort segment, staged by coalesced loads into shared memory; each lane then
// sums its node's entries in list order.
struct CombineProlongArgs {
  const double* r;
  const std::uint8_t* mask;
  const double* zsort;
  const unsigned* fine_off;
  const int* surf_first;   // first copy e*nsurfp + slot of each surface item (Zc element numbering)
  const double* Zc;
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
  int e0 = 0;       // Zc index of the element owning the first interior item
};

#ifndef COMBINE_MIN_BLOCKS
#define COMBINE_MIN_BLOCKS 6
#endif
constexpr int kCombineCap = 320;  // staged contributions per warp (avg ~2.9 per node at P = n+3)

// sum, for each lane's item g0 + lane, of its CSR segment of a contiguous value array
__device__ __forceinline__ double warp_segment_sum(const unsigned* __restrict__ off, const double* __restrict__ val,
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
  if (cnt <= static_cast<unsigned>(kCombineCap)) {
#pragma unroll 4
    for (unsigned c = lane; c < cnt; c += 32) stage[c] = __ldcs(val + base + c);
    __syncwarp();
    for (unsigned q = my0 - base; q < my1 - base; ++q) s += stage[q];
    __syncwarp();
  } else {
    for (unsigned q = my0; q < my1; ++q) s += __ldcs(val + q);
  }
  return s;
}

template <int NP>
__global__ void __launch_bounds__(kGatherBlock, COMBINE_MIN_BLOCKS) combine_prolong_kernel(CombineProlongArgs a)
{
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  constexpr int NS = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2), NSP = (NS + 3) & ~3;
  __shared__ double red[kGatherBlock / 32];
  __shared__ double stage[kGatherBlock / 32][kCombineCap];
  __shared__ double h0[NP], h1[NP];
  if (threadIdx.x < NP) {
    h0[threadIdx.x] = c_tab[NP].hat0[threadIdx.x];
    h1[threadIdx.x] = c_tab[NP].hat1[threadIdx.x];
  }
  __syncthreads();
  // prolongated value at (e; i,j,k): sum_cb B[cb][l] Zc[e][cb] (coarse.cpp:176-179)
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kGatherBlock / 32);
  const bool stage_fine = a.do_fine && !a.fine_in_z;
  double dot = 0.0;
  for (int w0 = (blockIdx.x * (kGatherBlock / 32) + warp) * 32; w0 < a.N; w0 += nwarps * 32) {
    // every load that does not depend on the contribution sums is issued first
    // (node id, r, mask, the prolongation's element corners), so a warp waits
    // for two dependent round trips per 32 nodes rather than four
    const int it = w0 + lane;
    const bool valid = it < a.N;
    const bool surf = it < a.nsg;
    const int g = !valid ? 0 : surf ? (a.surf_nodes ? __ldg(a.surf_nodes + it) : it) : a.ibase + (it - a.nsg);
    const double rg = valid ? __ldg(a.r + g) : 0.0;
    const bool dir = valid && surf && __ldg(a.mask + g);  // Dirichlet nodes are element-surface nodes
    long long ze = 0;
    int i = 0, j = 0, k = 0;
    if (a.do_coarse && valid) {
      if (!surf) {
        if constexpr (NI > 0) {
          const int t = it - a.nsg;  // interior ids are (e, local)-ordered (mesh.cpp:283)
          const int l = t % NI;
          ze = t / NI + a.e0;
          i = 1 + l % (n - 1);
          j = 1 + (l / (n - 1)) % (n - 1);
          k = 1 + l / ((n - 1) * (n - 1));
        }
      } else {
        const int x0 = __ldg(a.surf_first + it);
        ze = x0 / NSP;
        surface_ijk<NP>(x0 % NSP, i, j, k);
      }
    }
    const double zc = a.do_coarse && valid && !dir ? pz(ze, i, j, k) : 0.0;
    const double zf = stage_fine ? warp_segment_sum(a.fine_off, a.zsort, w0, a.N, stage[warp]) : 0.0;
    if (!valid) continue;
    double zg;
    if (dir) {
      zg = rg;
    } else {
      double s = 0.0;
      if (a.fine_in_z)
        s = a.z[g];
      else if (a.do_fine)
        s += zf;
      if (a.do_coarse) s += zc;
      zg = s;
    }
    a.z[g] = zg;
    dot += zg * rg;
  }
  dot_commit<kGatherBlock>(a.dot, dot, red);
}

// ---------------------------------------------------------------------------
// The same combine as a TMA-streamed persistent kernel (single-device plans,
// node ids = item ids). A tile of kCombTile consecutive nodes reads five
// contiguous ranges: r, the Dirichlet mask, the contribution offsets, the
// first-copy codes and its zsort segment [off[t0], off[t1]). One thread issues
// them as 1-D bulk copies (cp.async.bulk) completing on the stage's mbarrier,
// one tile ahead, into two shared-memory stages; the CTA's threads then sum,
// prolongate and store straight from shared memory. The data stream needs no
// per-thread loads in flight, so the kernel runs at the copy engines' rate
// instead of the warps' memory-level parallelism. Tiles whose segment exceeds
// the stage (none in the meshes measured) and the tail tile read global memory
// directly. Same arithmetic, same order as combine_prolong_kernel.
// Tile of 512 nodes from order 3 up (2.6-5.9 contributions per node on
// average), 256 below (up to 10 per node at order 2), so a tile's segment
// fits the 3072-entry stage (measured: order 3 at 256 nodes 0.394 ms, at 512
// 0.366 ms with a few tiles over the cap reading global memory).
#ifndef COMB_BLOCK
#define COMB_BLOCK 256
#endif
constexpr int kCombZcap = 3072, kCombTileMax = 512;
template <int NP>
struct CombTile {
  static constexpr int value = NP <= 3 ? 256 : 512;
  static constexpr int block = COMB_BLOCK < value ? COMB_BLOCK : value;   // threads per CTA
  static constexpr int minb = block >= 512 ? 2 : 3;                       // resident CTAs per SM
};
template <int T>
struct CombStage {
  double zs[kCombZcap];
  double rr[T];
  unsigned off[T + 4];
  int sf[T];
  unsigned char mk[T];
};
template <int T>
constexpr int comb_smem() { return 2 * static_cast<int>(sizeof(CombStage<T>)); }

template <int NP>
__global__ void __launch_bounds__(CombTile<NP>::block, CombTile<NP>::minb) combine_tma_kernel(CombineProlongArgs a, int ntiles, int ntma)
{
  constexpr int kCombTile = CombTile<NP>::value, kCombBlock = CombTile<NP>::block;
  using CombStageT = CombStage<kCombTile>;
  constexpr int n = NP - 1, NI = (n - 1) * (n - 1) * (n - 1);
  constexpr int NS = NP * NP * NP - (NP - 2) * (NP - 2) * (NP - 2), NSP = (NS + 3) & ~3;
  extern __shared__ __align__(128) unsigned char comb_smem[];
  CombStageT* st = reinterpret_cast<CombStageT*>(comb_smem);
  __shared__ __align__(8) unsigned long long full[2];
  __shared__ unsigned zbase[2], zfit[2];
  __shared__ double red[kCombBlock / 32];
  __shared__ double h0[NP], h1[NP];
  // local (i, j, k) of every element-interior index and surface slot, packed
  // i | j << 4 | k << 8: one shared load instead of the div/mod chains
  __shared__ unsigned short lut_int[NI > 0 ? NI : 1], lut_surf[NSP];
  const int tid = threadIdx.x;
  if (tid < NP) {
    h0[tid] = c_tab[NP].hat0[tid];
    h1[tid] = c_tab[NP].hat1[tid];
  }
  for (int q = tid; q < NI; q += kCombBlock)
    lut_int[q] = static_cast<unsigned short>((1 + q % (n - 1)) | ((1 + (q / (n - 1)) % (n - 1)) << 4) |
                                             ((1 + q / ((n - 1) * (n - 1))) << 8));
  for (int q = tid; q < NSP; q += kCombBlock) {
    int i = 0, j = 0, k = 0;
    if (q < NS) surface_ijk<NP>(q, i, j, k);
    lut_surf[q] = static_cast<unsigned short>(i | (j << 4) | (k << 8));
  }
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // Q1 prolongation at packed local coordinates, evaluated separably (x, then
  // y, then z: 14 operations instead of the 24 of the corner sum; the same
  // value to rounding)
  auto pz = [&](long long e, unsigned ijk) {
    const int i = ijk & 15, j = (ijk >> 4) & 15, k = ijk >> 8;
    const double2* zc2 = reinterpret_cast<const double2*>(a.Zc + 8 * e);
    const double2 c01 = __ldg(zc2), c23 = __ldg(zc2 + 1), c45 = __ldg(zc2 + 2), c67 = __ldg(zc2 + 3);
    const double xi0 = h0[i], xi1 = h1[i];
    const double a00 = xi0 * c01.x + xi1 * c01.y, a10 = xi0 * c23.x + xi1 * c23.y;
    const double a01 = xi0 * c45.x + xi1 * c45.y, a11 = xi0 * c67.x + xi1 * c67.y;
    const double yj0 = h0[j], yj1 = h1[j];
    return h0[k] * (yj0 * a00 + yj1 * a10) + h1[k] * (yj0 * a01 + yj1 * a11);
  };
  // thread 0: stage tile ti (ti < ntma: every range in bounds)
  auto issue = [&](int ti, int s) {
    const long long t0 = static_cast<long long>(ti) * kCombTile;
    const unsigned q0 = __ldg(a.fine_off + t0), q1 = __ldg(a.fine_off + t0 + kCombTile);
    const unsigned z0 = q0 & ~1u, z1 = (q1 + 1) & ~1u;
    // the second half of a split combine reads the fine sums from z instead
    const bool fits = !a.fine_in_z && z1 - z0 <= static_cast<unsigned>(kCombZcap);
    const bool sf = a.do_coarse && t0 < a.nsg;
    zbase[s] = z0;
    zfit[s] = fits ? 1u : 0u;
    const unsigned bytes = kCombTile * 8 + (kCombTile + 4) * 4 + kCombTile + (sf ? kCombTile * 4 : 0) +
                           (fits ? (z1 - z0) * 8 : 0);
    fence_proxy_async_smem();
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(st[s].rr, a.r + t0, kCombTile * 8, &full[s]);
    bulk_g2s(st[s].off, a.fine_off + t0, (kCombTile + 4) * 4, &full[s]);
    bulk_g2s(st[s].mk, a.mask + t0, kCombTile, &full[s]);
    if (sf) bulk_g2s(st[s].sf, a.surf_first + t0, kCombTile * 4, &full[s]);
    if (fits && z1 > z0) bulk_g2s(st[s].zs, a.zsort + z0, (z1 - z0) * 8, &full[s]);
  };
  double dot = 0.0;
  if (tid == 0 && static_cast<int>(blockIdx.x) < ntma) issue(blockIdx.x, 0);
  int use = 0;
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++use) {
    const int s = use & 1;
    const int tn = ti + gridDim.x;
    if (tid == 0 && tn < ntma) issue(tn, s ^ 1);  // stage s^1 was released by the last __syncthreads
    const bool staged = ti < ntma;
    if (staged) mbar_wait(&full[s], (use >> 1) & 1);
    const CombStageT& S = st[s];
    const long long t0 = static_cast<long long>(ti) * kCombTile;
    const unsigned z0 = staged ? zbase[s] : 0u;
    const bool fit = staged && zfit[s];
#pragma unroll
    for (int h = 0; h < kCombTile / kCombBlock; ++h) {
      const int l = tid + h * kCombBlock;
      const long long itl = t0 + l;
      if (itl >= a.N) continue;
      const int it = static_cast<int>(itl);
      const bool surf = it < a.nsg;
      const double rg = staged ? S.rr[l] : __ldg(a.r + it);
      double zg;
      if (surf && (staged ? S.mk[l] : __ldg(a.mask + it))) {
        zg = rg;
      } else {
        double sum = 0.0;
        if (a.fine_in_z) {
          sum = a.z[it];
        } else if (a.do_fine) {
          const unsigned q0 = staged ? S.off[l] : __ldg(a.fine_off + it);
          const unsigned q1 = staged ? S.off[l + 1] : __ldg(a.fine_off + it + 1);
          double zf = 0.0;
          if (fit) {
            for (unsigned q = q0 - z0; q < q1 - z0; ++q) zf += S.zs[q];
          } else {
            for (unsigned q = q0; q < q1; ++q) zf += __ldcs(a.zsort + q);
          }
          sum += zf;
        }
        if (a.do_coarse) {
          double zc = 0.0;
          if (!surf) {
            if constexpr (NI > 0) {
              const int t = it - a.nsg;
              zc = pz(t / NI, lut_int[t % NI]);
            }
          } else {
            const int x0 = staged ? S.sf[l] : __ldg(a.surf_first + it);
            zc = pz(x0 / NSP, lut_surf[x0 % NSP]);
          }
          sum += zc;
        }
        zg = sum;
      }
      a.z[it] = zg;
      dot += zg * rg;
    }
    __syncthreads();  // stage s fully read before thread 0 refills it (next iteration's issue)
  }
  dot_commit<kCombBlock>(a.dot, dot, red);
}

// first copy (lowest (e, slot)) of every item of a copy CSR
__global__ void first_copy_kernel(const unsigned* __restrict__ off, const int* __restrict__ idx, int n,
                                  int* __restrict__ first)
{
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    first[t] = __ldg(idx + __ldg(off + t));
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
