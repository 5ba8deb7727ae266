// Shared device helpers: constant-memory operator tables, deterministic
// reductions, index encodings. sm_100a, FP64 throughout.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hxb {

constexpr int kMaxNP = 11;         // orders 1..10
constexpr int kMaxP = kMaxNP + 2;  // FDM pencil size n+3

// Per-order operator tables (device global memory, ~6.5 KB per order). Index
// [NP] selects the order so plans of different orders coexist. Kernels copy
// the rows they contract with into shared memory once per CTA and read them
// as warp-uniform broadcasts (one LDS.128 feeds two DFMA columns), which on
// sm_100a is cheaper than staging FP64 constants through uniform registers.
struct OrderTables {
  double D[kMaxNP * kMaxNP];   // D[m*np+i] = phi'_m(t_i), gll.hpp:23-26
  double DT[kMaxNP * kMaxNP];  // DT[m*np+i] = D[i*np+m] (adjoint contractions read rows)
  double VT[kMaxP * kMaxP];    // pencil V transposed: VT[x*p+d] = V[d][x] (fine.hpp:22)
  double ViT[kMaxP * kMaxP];   // pencil V^-1 transposed (fine.hpp:23)
  double M[kMaxP];             // pencil lumped mass (fine.hpp:21)
  double invM[kMaxP];          // 1/M
  // even/odd split of the pencil transforms (eigenvectors of the reflection-
  // symmetric pencil are even (d even) or odd (d odd)); see fdm_kernel
  double FE[49], FO[36];       // forward: FE[x*NE+a] = V[2a][x], FO[x*NO+a] = V[2a+1][x]
  double IE[49], IO[36];       // inverse: IE[a*(h+mid)+x] = Vi[x][2a], IO[a*h+x] = Vi[x][2a+1]
  int eo_ok;                   // 1 when the split is exact to rounding (checked at setup)
  double lam[kMaxP];           // pencil eigenvalues (fine.hpp:24)
  double hat0[kMaxNP];         // 0.5*(1-t_i)  coarse hats (gll.cpp:92)
  double hat1[kMaxNP];         // 0.5*(1+t_i)
  double w[kMaxNP];            // GLL weights rho_i (gll.hpp:21), on-the-fly geometry
};
// Single translation unit (plan.cu) includes the kernels, so this is the definition.
__device__ OrderTables c_tab[kMaxNP + 1];

// FDM transform tables in the constant bank: with the order a template
// parameter every coefficient address is a compile-time immediate, so the
// kernels read them as LDCU.128 into uniform registers (one per warp, off
// the L1/shared path that the line transposes saturate).
struct FdmConst {
  double FE[49], FO[36], IE[49], IO[36];
  double lam[kMaxP], invM[kMaxP];
};
__constant__ FdmConst c_fdm[kMaxNP + 1];

// Global-id encodings in the gather/scatter maps:
//   v >= 0   free node v
//   v == -1  no node (sentinel slot, IndexMaps::kNoNode)
//   v <= -2  Dirichlet node (-v-2): reads as 0 (masked input, operator.cpp:264,
//            precond.cpp:35)
__host__ __device__ inline int encode_dirichlet(int g) { return -g - 2; }
__device__ __forceinline__ double load_masked(const double* __restrict__ x, int code)
{
  return code >= 0 ? __ldg(x + code) : 0.0;
}

// Rank of local node (i,j,k) among element-surface nodes in ascending local
// index, -1 for element-interior (mirrors setup_numbering.cpp). An
// entity-grouped rsurf order (vertices, edges, faces: contiguous runs per mesh
// edge/face) was measured at cfg2 three ways: the gather read
// 0.36 GB less (0.265 -> 0.215 ms) but the element kernel lost more, with
// scattered stores (0.76 -> 0.99 ms), a TMA bulk store of a shared-staged row
// (0.87 ms) or coalesced 16-byte stores of it (0.89 ms); this order stays.
__host__ __device__ __forceinline__ int surface_slot(int np, int i, int j, int k)
{
  const int n = np - 1, mid = 4 * np - 4;
  if (k == 0) return j * np + i;
  if (k == n) return np * np + (np - 2) * mid + j * np + i;
  const int base = np * np + (k - 1) * mid;
  if (j == 0) return base + i;
  if (j == n) return base + np + 2 * (np - 2) + i;
  if (i == 0) return base + np + 2 * (j - 1);
  if (i == n) return base + np + 2 * (j - 1) + 1;
  return -1;
}

// Inverse of surface_slot: local (i,j,k) of surface slot s.
template <int NP>
__device__ __forceinline__ void surface_ijk(int s, int& i, int& j, int& k)
{
  constexpr int n = NP - 1, mid = 4 * NP - 4, NN = NP * NP;
  if (s < NN) {
    k = 0;
    j = s / NP;
    i = s % NP;
    return;
  }
  const int t = s - NN;
  if (t >= (NP - 2) * mid) {
    const int u = t - (NP - 2) * mid;
    k = n;
    j = u / NP;
    i = u % NP;
    return;
  }
  k = 1 + t / mid;
  const int rem = t % mid;
  if (rem < NP) {
    j = 0;
    i = rem;
  } else if (rem >= NP + 2 * (NP - 2)) {
    j = n;
    i = rem - (NP + 2 * (NP - 2));
  } else {
    const int q = rem - NP;
    j = 1 + q / 2;
    i = (q & 1) ? n : 0;
  }
}

// optional u += alpha_k p_k of the PCG (krylov.cpp:54) riding along another pass
struct PcgUArgs {
  double* u = nullptr;
  const double* p = nullptr;
  const double* zr = nullptr;
  const double* pf = nullptr;
  int k = 0;
};

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, 1-D, no tensor map) completing on an
// mbarrier: global -> shared staging for streamed per-element data.
__device__ __forceinline__ unsigned smem_u32(const void* p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Orders this thread's (and, through a preceding __syncthreads, the whole
// CTA's) generic-proxy shared-memory accesses before its subsequent
// async-proxy (TMA) accesses: required before a bulk copy overwrites a buffer
// that other threads have just read with ordinary loads (WAR across proxies).
__device__ __forceinline__ void fence_proxy_async_smem()
{
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity)
{
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// CSR row sum s = sum_q val[q] * x(col[q]) in ascending q (CsrMatrix::multiply
// order, amg.cpp:13-20), with the loads of 8 entries issued before any of
// their products is summed: the row costs ~3 memory round trips instead of
// one per entry.
template <class XF>
__device__ __forceinline__ double csr_row_sum(const int* __restrict__ ptr, const int* __restrict__ col,
                                              const double* __restrict__ val, int i, XF&& xf)
{
  const int q0 = __ldg(ptr + i), q1 = __ldg(ptr + i + 1);
  double s = 0.0;
  for (int q = q0; q < q1; q += 8) {
    int c[8];
    double v[8], x[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool ok = q + t < q1;
      c[t] = ok ? __ldg(col + q + t) : 0;
      v[t] = ok ? __ldg(val + q + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = q + t < q1 ? xf(c[t]) : 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (q + t < q1) s += v[t] * x[t];
  }
  return s;
}

// ---------------------------------------------------------------------------
// Deterministic dot products. Each participating kernel block reduces its
// partial in a fixed tree and stores it at partials[offset + blockIdx.x]; the
// last block to finish (ticket) sums partials[0 .. offset+gridDim.x) in a
// fixed order. Results are bitwise reproducible run to run.
struct DotArgs {
  double* partials = nullptr;  // null: no dot requested
  unsigned* ticket = nullptr;
  double* result = nullptr;    // null: only store partials (a later kernel finalizes)
  int offset = 0;
};

template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* red)
{
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) s += red[w];
  }
  return s;  // valid in thread 0
}

// Must be called by every thread of the block (linear block of BLOCK threads).
template <int BLOCK>
__device__ void dot_commit(const DotArgs& d, double v, double* red)
{
  if (d.partials == nullptr) return;
  const double s = block_sum<BLOCK>(v, red);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    d.partials[d.offset + blockIdx.x] = s;
    last = false;
    if (d.result != nullptr) {
      __threadfence();
      const unsigned t = atomicAdd(d.ticket, 1u);
      last = (t == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int total = d.offset + gridDim.x;
  double acc = 0;
  for (int q = threadIdx.x; q < total; q += BLOCK) acc += __ldcg(d.partials + q);
  const double tot = block_sum<BLOCK>(acc, red);
  if (threadIdx.x == 0) {
    *d.result = tot;
    *d.ticket = 0;
  }
}

}  // namespace hxb
