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

// Sum vals[off[g] .. off[g+1]) left to right for the warp's 32 consecutive
// nodes. The producers wrote each contribution at its CSR position, so the
// warp's whole segment is contiguous: one coalesced sweep into the staging
// buffer, then a sequential per-lane sum (reference order).
__device__ __forceinline__ double warp_seg_sum(const unsigned* __restrict__ off, const double* __restrict__ vals, int g0,
                                               int n, double* __restrict__ stage)
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
    for (unsigned c = lane; c < cnt; c += 32) stage[c] = __ldcs(vals + base + c);
    __syncwarp();
    for (unsigned q = my0 - base; q < my1 - base; ++q) s += stage[q];
    __syncwarp();
  } else {
    for (unsigned q = my0; q < my1; ++q) s += __ldcs(vals + q);
  }
  return s;
}

// Same, for values scattered in an E-vector: src(idx[q]) gathered by the warp
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
  int num_surface_global;
  DotArgs dot;
};

__global__ void __launch_bounds__(kGatherBlock) ax_gather_kernel(AxGatherArgs a)
{
  __shared__ double red[kGatherBlock / 32];
  __shared__ double stage[kGatherBlock / 32][kGatherCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kGatherBlock / 32);
  double dot = 0.0;
  for (int g0 = (blockIdx.x * (kGatherBlock / 32) + warp) * 32; g0 < a.num_surface_global; g0 += nwarps * 32) {
    const double s = warp_csr_sum(a.off, a.idx, [&](int q) { return __ldg(a.rsurf + q); }, g0,
                                  a.num_surface_global, stage[warp]);
    const int g = g0 + lane;
    if (g < a.num_surface_global) {
      const double ug = __ldg(a.u + g);
      const double rg = __ldg(a.mask + g) ? ug : s;
      a.r[g] = rg;
      dot += ug * rg;
    }
  }
  dot_commit<kGatherBlock>(a.dot, dot, red);
}

// ---------------------------------------------------------------------------
// Two-scale combine (precond.cpp:57-66): z = mask ? r : (0 + zf) + zc, with
//   zf = sum of the node's subdomain-slot values in ascending (e,slot) order
//        (FinePreconditioner accumulation, fine.cpp:224-227)
//   zc = (sum of the node's prolongated copies in (e,l) order) / m_N
//        (CoarsePreconditioner::prolongate, coarse.cpp:164-186; the per-copy
//        values come from prolong_elem_kernel)
// plus the fused z.r partial.
struct CombineArgs {
  const double* r;
  const std::uint8_t* mask;
  const double* zsort;       // fine subdomain outputs in CSR order (fdm_kernel)
  const unsigned* fine_off;  // N+1
  const double* psort;       // prolongated surface copies in CSR order (prolong_elem_kernel)
  const double* pint;        // prolongated element-interior nodes (N, [nsg,N) used)
  const unsigned* ax_off;    // nsg+1
  const double* lumped;      // m_N
  double* z;
  int N, nsg;
  int do_fine, do_coarse;
  DotArgs dot;
};

__global__ void __launch_bounds__(kGatherBlock, 4) combine_kernel(CombineArgs a)
{
  __shared__ double red[kGatherBlock / 32];
  __shared__ double stage[kGatherBlock / 32][kGatherCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kGatherBlock / 32);
  double dot = 0.0;
  for (int g0 = (blockIdx.x * (kGatherBlock / 32) + warp) * 32; g0 < a.N; g0 += nwarps * 32) {
    const int g = g0 + lane;
    double zf = 0.0, zc = 0.0;
    if (a.do_fine)
      zf = warp_seg_sum(a.fine_off, a.zsort, g0, a.N, stage[warp]);
    if (a.do_coarse) {
      if (g0 < a.nsg)
        zc = warp_seg_sum(a.ax_off, a.psort, g0, a.nsg, stage[warp]);
      if (g >= a.nsg && g < a.N) zc = __ldg(a.pint + g);
    }
    if (g < a.N) {
      const double rg = __ldg(a.r + g);
      double zg;
      if (__ldg(a.mask + g)) {
        zg = rg;
      } else {
        double s = 0.0;
        if (a.do_fine) s += zf;
        if (a.do_coarse) s += zc / __ldg(a.lumped + g);
        zg = s;
      }
      a.z[g] = zg;
      dot += zg * rg;
    }
  }
  dot_commit<kGatherBlock>(a.dot, dot, red);
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
