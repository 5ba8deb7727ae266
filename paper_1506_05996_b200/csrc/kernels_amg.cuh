// AMG K-cycle below the finest level in ONE thread-block-cluster kernel.
//
// AmgHierarchy::cycle / ksolve (amg.cpp:198-263) recurse through levels
// 1..L whose sizes collapse quickly (cfg2: 32,200 -> 17,336 -> 16,295 rows,
// of which only 15,974 / 1,110 / 69 are coupled). Launched as ~60 tiny
// kernels per K-cycle the coarse solve is launch-latency bound, so
// ksolve(1) runs here as one kernel on a cluster of CTAs that synchronise
// with cluster barriers (hundreds of ns) instead of kernel boundaries.
//
// Rows that are decoupled identity rows with a provably zero right-hand side
// (Dirichlet vertices, coarse.cpp:79-85, masked in R, coarse.cpp:191-192,
// and aggregates made only of them) carry exact zeros through every cycle
// and are dropped from levels >= 1 by the host (compact numbering); adding
// their zero terms to any sum changes nothing, so the arithmetic of the kept
// rows is the reference's.
//
// Dot products: per-thread partials over a fixed row->thread map, fixed
// warp/CTA trees, CTA partials summed in cluster-rank order through
// distributed shared memory -> deterministic and identical in every CTA.
// Vectors written inside the kernel are read with ld.global.cg (L2) after a
// cluster barrier, so no stale L1 line is ever consumed.
#pragma once

#include <cooperative_groups.h>

#include "kernels_coarse.cuh"
#include "kernels_common.cuh"

namespace hxb {

namespace cg = cooperative_groups;

constexpr int kAmgMaxLevels = 14;
constexpr int kAmgClusterBlock = 1024;
// ksolve subtrees whose top level has at most this many rows run inside CTA 0
// alone (block barriers, ~10x cheaper than cluster barriers); the other CTAs
// wait at one cluster barrier
constexpr int kAmgLocalRows = 4096;

// One compacted level (AMG level l >= 1), all indices compact.
struct CLev {
  int n = 0;                                       // kept rows
  const int* ptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  const double* dinv = nullptr;                    // 1/a_ii
  const int* agg = nullptr;                        // row -> next level's compact row
  const int* mptr = nullptr;                       // next level's rows: member lists (ascending)
  const int* mem = nullptr;
  int nc = 0;                                      // next level's kept rows
  double *zA = nullptr, *zB = nullptr, *rho = nullptr;      // cycle work
  double *kr = nullptr, *kz = nullptr, *kp = nullptr, *kf = nullptr;  // ksolve work
  double *b = nullptr, *x = nullptr;               // ksolve rhs / solution at this level
};

struct AmgClusterArgs {
  CLev lev[kAmgMaxLevels];
  int L = 0;                 // compact non-coarsest levels (lev[0] = AMG level 1); lev[L] = coarsest
  // coarsest solve: inverse of the coupled block (m x m, row-major, rows `coupled`)
  // plus 1/a_ii on the decoupled rows (inv_diag != 0 there)
  const double* ainv = nullptr;
  const int* coupled = nullptr;
  const double* inv_diag = nullptr;
  int m = 0;
};

struct ClusterCtx {
  cg::cluster_group cl;
  bool local;  // true: only this CTA participates (block-level sync and sums)
  int tid, nthr;
  double* part;  // __shared__ double[2]: this CTA's dot partial (double-buffered)
  double* bcast; // __shared__ double: broadcast of the reduced value
  double* wred;  // __shared__ double[32]
  int parity;
};

// barrier.cluster.arrive.release / wait.acquire: orders every memory access
// (global included) of the cluster's threads at cluster scope; mutable
// vectors are read with ld.global.cg, so no L1 line can be stale.
__device__ __forceinline__ void csync(ClusterCtx& c)
{
  if (c.local)
    __syncthreads();
  else
    c.cl.sync();
}

// Deterministic cluster-wide sum of one value per thread (also a cluster
// barrier that publishes every global write made before it).
__device__ double cluster_sum(ClusterCtx& c, double v)
{
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) c.wred[warp] = v;
  __syncthreads();
  double* slot = c.part + c.parity;
  c.parity ^= 1;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += c.wred[w];
    *slot = s;
    if (c.local) *c.bcast = s;
  }
  if (c.local) {
    __syncthreads();
    const double r = *c.bcast;
    __syncthreads();  // bcast may be rewritten by the next sum
    return r;
  }
  c.cl.sync();  // every CTA's partial is in its shared memory
  if (warp == 0) {
    const int ranks = (int)c.cl.num_blocks();
    double s = 0.0;
    if (lane < ranks) s = *c.cl.map_shared_rank(slot, lane);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) *c.bcast = s;
  }
  __syncthreads();
  return *c.bcast;
}

__device__ __forceinline__ double crow(const CLev& L, int i, const double* __restrict__ x)
{
  return csr_row_sum(L.ptr, L.col, L.val, i, [&](int j) { return __ldcg(x + j); });
}

__device__ void amg_ksolve(ClusterCtx& c, const AmgClusterArgs& a, int l, const double* b, double* x);

// x = Ainv b on the coarsest level (Eigen LLT solve in the reference, amg.cpp:188-194)
__device__ void amg_dense(ClusterCtx& c, const AmgClusterArgs& a, const double* b, double* x)
{
  const int lane = threadIdx.x & 31;
  const int gw = c.tid >> 5, nw = c.nthr >> 5;
  for (int r = gw; r < a.m; r += nw) {
    const double* row = a.ainv + (std::size_t)r * a.m;
    double s = 0.0;
    for (int q = lane; q < a.m; q += 32) s += __ldg(row + q) * __ldcg(b + __ldg(a.coupled + q));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) __stcg(x + __ldg(a.coupled + r), s);
  }
  const int n = a.lev[a.L].n;
  for (int i = c.tid; i < n; i += c.nthr) {
    const double di = __ldg(a.inv_diag + i);
    if (di != 0.0) __stcg(x + i, __ldcg(b + i) * di);
  }
  csync(c);
}

// One multigrid cycle at compact level l (amg.cpp:198-227); result in `out`.
__device__ void amg_cycle(ClusterCtx& c, const AmgClusterArgs& a, int l, const double* r, double* out)
{
  if (l == a.L) {
    amg_dense(c, a, r, out);
    return;
  }
  constexpr double w = kJacobiOmega;
  const CLev& L = a.lev[l];
  const CLev& N = a.lev[l + 1];
  // z = w d r; one Jacobi sweep (z1 formed on the fly for the neighbours)
  for (int i = c.tid; i < L.n; i += c.nthr) {
    const double s = csr_row_sum(L.ptr, L.col, L.val, i, [&](int j) { return w * __ldg(L.dinv + j) * __ldcg(r + j); });
    const double di = __ldg(L.dinv + i), ri = __ldcg(r + i);
    __stcg(L.zA + i, w * di * ri + w * di * (ri - s));
  }
  csync(c);
  // rho = r - A z
  for (int i = c.tid; i < L.n; i += c.nthr) __stcg(L.rho + i, __ldcg(r + i) - crow(L, i, L.zA));
  csync(c);
  // rc = sum over aggregate members (ascending) of rho
  for (int k = c.tid; k < N.n; k += c.nthr) {
    double s = 0.0;
    const int q1 = __ldg(L.mptr + k + 1);
    for (int q = __ldg(L.mptr + k); q < q1; ++q) s += __ldcg(L.rho + __ldg(L.mem + q));
    __stcg(N.b + k, s);
  }
  csync(c);
  amg_ksolve(c, a, l + 1, N.b, N.x);
  // z += ec[agg]; first post-smoothing sweep (z3 on the fly)
  for (int i = c.tid; i < L.n; i += c.nthr) {
    const double s = csr_row_sum(L.ptr, L.col, L.val, i,
                                 [&](int j) { return __ldcg(L.zA + j) + __ldcg(N.x + __ldg(L.agg + j)); });
    const double z3 = __ldcg(L.zA + i) + __ldcg(N.x + __ldg(L.agg + i));
    __stcg(L.zB + i, z3 + w * __ldg(L.dinv + i) * (__ldcg(r + i) - s));
  }
  csync(c);
  // second sweep
  for (int i = c.tid; i < L.n; i += c.nthr) {
    const double s = crow(L, i, L.zB);
    __stcg(out + i, __ldcg(L.zB + i) + w * __ldg(L.dinv + i) * (__ldcg(r + i) - s));
  }
  csync(c);
}

// Exactly two PCG steps on A_l x = b preconditioned by cycle(l) (amg.cpp:230-263).
__device__ void amg_ksolve(ClusterCtx& c, const AmgClusterArgs& a, int l, const double* b, double* x)
{
  if (!c.local && a.lev[l].n <= kAmgLocalRows) {
    // small subtree: CTA 0 alone (b was published by the caller's barrier)
    if (c.cl.block_rank() == 0) {
      ClusterCtx lc = c;
      lc.local = true;
      lc.tid = threadIdx.x;
      lc.nthr = blockDim.x;
      amg_ksolve(lc, a, l, b, x);
      c.parity = lc.parity;
    }
    c.cl.sync();
    return;
  }
  if (l == a.L) {
    amg_dense(c, a, b, x);
    return;
  }
  const CLev& L = a.lev[l];
  const int n = L.n;
  // r = b, x = 0: the first cycle reads b directly; r is materialised by the update
  amg_cycle(c, a, l, b, L.kz);
  double loc = 0.0;
  for (int i = c.tid; i < n; i += c.nthr) loc += __ldcg(L.kz + i) * __ldcg(b + i);
  double zr = cluster_sum(c, loc);
  const double* p = L.kz;  // p = z; copied into kp by the first f = A p sweep, since
  const double* rr = b;    // the next cycle overwrites kz
  for (int it = 0; it < 2; ++it) {
    loc = 0.0;
    for (int i = c.tid; i < n; i += c.nthr) {
      const double fi = crow(L, i, p);
      const double pi = __ldcg(p + i);
      __stcg(L.kf + i, fi);
      if (it == 0) __stcg(L.kp + i, pi);
      loc += pi * fi;
    }
    p = L.kp;
    const double pf = cluster_sum(c, loc);  // its barrier also publishes kf
    if (!(pf > 0) || !(fabs(zr) > 0)) {
      if (it == 0)  // x stays 0
        for (int i = c.tid; i < n; i += c.nthr) __stcg(x + i, 0.0);
      csync(c);
      return;
    }
    const double alpha = zr / pf;
    for (int i = c.tid; i < n; i += c.nthr) {
      const double pi = __ldcg(p + i);
      __stcg(x + i, it == 0 ? alpha * pi : __ldcg(x + i) + alpha * pi);  // x = 0 + alpha p
      if (it == 0) __stcg(L.kr + i, __ldcg(rr + i) - alpha * __ldcg(L.kf + i));
    }
    csync(c);
    if (it == 1) break;
    amg_cycle(c, a, l, L.kr, L.kz);
    loc = 0.0;
    for (int i = c.tid; i < n; i += c.nthr) loc += __ldcg(L.kz + i) * __ldcg(L.kr + i);
    const double zr_next = cluster_sum(c, loc);
    const double beta = zr_next / zr;
    zr = zr_next;
    for (int i = c.tid; i < n; i += c.nthr) __stcg(L.kp + i, __ldcg(L.kz + i) + beta * __ldcg(p + i));
    csync(c);
    p = L.kp;
    rr = L.kr;
  }
}

// ksolve(1, b, x) of the finest cycle: b = lev[0].b (compact level-1 rc), x = lev[0].x
// (or the coarsest dense solve when the hierarchy has a single level below 0).
__global__ void __launch_bounds__(kAmgClusterBlock, 1) amg_cluster_kernel(const __grid_constant__ AmgClusterArgs a, const double* b, double* x)
{
  __shared__ double part[2], bcast, wred[32];
  ClusterCtx c{cg::this_cluster(), false, 0, 0, part, &bcast, wred, 0};
  c.tid = (int)c.cl.block_rank() * (int)blockDim.x + (int)threadIdx.x;
  c.nthr = (int)c.cl.num_blocks() * (int)blockDim.x;
  amg_ksolve(c, a, 0, b, x);
}

// ksolve(l) of the compacted hierarchy by ONE CTA with block barriers: the
// small levels (<= kAmgLocalRows kept rows) of the default per-step K-cycle,
// where a kernel per step would be all launch latency (one launch instead of
// ~21 at cfg2).
__global__ void __launch_bounds__(kAmgClusterBlock, 1) amg_local_ksolve_kernel(const __grid_constant__ AmgClusterArgs a,
                                                                               int l, const double* b, double* x)
{
  __shared__ double part[2], bcast, wred[32];
  ClusterCtx c{cg::this_cluster(), true, (int)threadIdx.x, (int)blockDim.x, part, &bcast, wred, 0};
  amg_ksolve(c, a, l, b, x);
}

// ---------------------------------------------------------------------------
// Finest-level (level 0, full vertex numbering) glue kernels.

// b1[k] = sum over the members (ascending, level-0 ids) of kept level-1 row k of rho
__global__ void amg_agg_sum_compact_kernel(const double* __restrict__ rho, const int* __restrict__ mptr,
                                           const int* __restrict__ mem, double* __restrict__ b1, int n1)
{
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n1; k += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = __ldg(mptr + k); q < __ldg(mptr + k + 1); ++q) s += __ldg(rho + __ldg(mem + q));
    b1[k] = s;
  }
}

// zout = z3 + w d (r - A z3), z3 = zin + ec1[agg0c] (0 for dropped aggregates) (amg.cpp:220-222)
__global__ void amg_prolong_smooth_compact_kernel(DevCsr A, const double* __restrict__ dinv, const double* __restrict__ r,
                                                  const double* __restrict__ zin, const double* __restrict__ ec,
                                                  const int* __restrict__ aggc, double* __restrict__ zout)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
    const double s = csr_row_sum(A.ptr, A.col, A.val, i, [&](int c) {
      const int k = __ldg(aggc + c);
      return __ldg(zin + c) + (k >= 0 ? __ldg(ec + k) : 0.0);
    });
    const int ki = __ldg(aggc + i);
    const double z3 = __ldg(zin + i) + (ki >= 0 ? __ldg(ec + ki) : 0.0);
    zout[i] = z3 + kJacobiOmega * __ldg(dinv + i) * (__ldg(r + i) - s);
  }
}

}  // namespace hxb
