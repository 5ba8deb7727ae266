// Bitwise-reference mode: see compat.hpp. Compiled with -fmad=false.
#include "compat.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

namespace hxb {

#define CX_CUDA(call)                                                                                 \
  do {                                                                                                \
    cudaError_t err__ = (call);                                                                       \
    if (err__ != cudaSuccess)                                                                         \
      throw HxbError(HXB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(err__));               \
  } while (0)

namespace {

constexpr int kCxBlock = 256;
constexpr double kOmega = 2.0 / 3.0;  // kJacobiOmega = Real(2) / 3 (amg.cpp:44)
constexpr int kSweeps = 2;            // kSmoothSweeps (amg.cpp:45)

int cx_grid(long long n) { return static_cast<int>(std::max(1LL, std::min((n + kCxBlock - 1) / kCxBlock, 148LL * 16))); }

// ---------------------------------------------------------------------------
// Operator (operator.cpp:124-287)

struct CxAxArgs {
  int np, nloc, nlocp, variant;
  const double* u_loc;
  double* r_loc;
  const double* D;
  const double* wg;
  const double* erec;
  const double* nodes;
  const double* weights;
  const double* mass;
  const double* c_e;
};

// One CTA per element: phase 1 (derivatives + metric fluxes), phase 2 (adjoint
// contractions, the interleaved sum of operator.cpp:152-157, + (c u) m).
__global__ void cx_ax_elem_kernel(CxAxArgs a)
{
  extern __shared__ double sh[];
  const int np = a.np, nloc = a.nloc;
  double* su = sh;
  double* fa = su + nloc;
  double* fb = fa + nloc;
  double* fc = fb + nloc;
  double* sD = fc + nloc;
  double* wge = sD + np * np;   // on-the-fly: 6 planes
  double* me = wge + 6 * nloc;  // on-the-fly: mass
  const long long e = blockIdx.x;
  for (int q = threadIdx.x; q < nloc; q += blockDim.x) su[q] = a.u_loc[e * nloc + q];
  for (int q = threadIdx.x; q < np * np; q += blockDim.x) sD[q] = a.D[q];
  if (a.variant == HXB_VARIANT_ON_THE_FLY) {  // otf_element_kernel geometry (operator.cpp:182-240)
    const double* rec = a.erec + e * 26;
    const double kap = rec[24];
    for (int node = threadIdx.x; node < nloc; node += blockDim.x) {
      const int i = node % np, j = (node / np) % np, k = node / (np * np);
      const double h[3][2] = {{0.5 * (1 - a.nodes[i]), 0.5 * (1 + a.nodes[i])},
                              {0.5 * (1 - a.nodes[j]), 0.5 * (1 + a.nodes[j])},
                              {0.5 * (1 - a.nodes[k]), 0.5 * (1 + a.nodes[k])}};
      const double dh[2] = {-0.5, 0.5};
      double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int bk = 0; bk < 2; ++bk)
        for (int bj = 0; bj < 2; ++bj)
          for (int bi = 0; bi < 2; ++bi) {
            const double* x = rec + 3 * (bi + 2 * bj + 4 * bk);  // corner hex_corner(bi, bj, bk)
            const double wx = dh[bi] * h[1][bj] * h[2][bk];
            const double wy = h[0][bi] * dh[bj] * h[2][bk];
            const double wz = h[0][bi] * h[1][bj] * dh[bk];
            for (int d = 0; d < 3; ++d) {
              J[d * 3 + 0] += wx * x[d];
              J[d * 3 + 1] += wy * x[d];
              J[d * 3 + 2] += wz * x[d];
            }
          }
      double adj[9];
      adj[0] = J[4] * J[8] - J[5] * J[7];
      adj[1] = J[2] * J[7] - J[1] * J[8];
      adj[2] = J[1] * J[5] - J[2] * J[4];
      adj[3] = J[5] * J[6] - J[3] * J[8];
      adj[4] = J[0] * J[8] - J[2] * J[6];
      adj[5] = J[2] * J[3] - J[0] * J[5];
      adj[6] = J[3] * J[7] - J[4] * J[6];
      adj[7] = J[1] * J[6] - J[0] * J[7];
      adj[8] = J[0] * J[4] - J[1] * J[3];
      const double det = J[0] * adj[0] + J[1] * adj[3] + J[2] * adj[6];
      const double rho3 = a.weights[i] * a.weights[j] * a.weights[k];
      const double scale = kap * rho3 / det;
      auto aat = [&](int r0, int c0) {
        return adj[r0 * 3 + 0] * adj[c0 * 3 + 0] + adj[r0 * 3 + 1] * adj[c0 * 3 + 1] + adj[r0 * 3 + 2] * adj[c0 * 3 + 2];
      };
      wge[0 * nloc + node] = scale * aat(0, 0);
      wge[1 * nloc + node] = scale * aat(0, 1);
      wge[2 * nloc + node] = scale * aat(0, 2);
      wge[3 * nloc + node] = scale * aat(1, 1);
      wge[4 * nloc + node] = scale * aat(1, 2);
      wge[5 * nloc + node] = scale * aat(2, 2);
      me[node] = rho3 * det;
    }
  }
  __syncthreads();
  const bool otf = a.variant == HXB_VARIANT_ON_THE_FLY;
  for (int node = threadIdx.x; node < nloc; node += blockDim.x) {
    const int i = node % np, j = (node / np) % np, k = node / (np * np);
    double sx = 0, sy = 0, sz = 0;
    for (int mm = 0; mm < np; ++mm) {
      sx += sD[mm * np + i] * su[(k * np + j) * np + mm];
      sy += sD[mm * np + j] * su[(k * np + mm) * np + i];
      sz += sD[mm * np + k] * su[(mm * np + j) * np + i];
    }
    double w[6];
    for (int g = 0; g < 6; ++g) w[g] = otf ? wge[g * nloc + node] : a.wg[(e * 6 + g) * a.nlocp + node];
    fa[node] = w[0] * sx + w[1] * sy + w[2] * sz;
    fb[node] = w[1] * sx + w[3] * sy + w[4] * sz;
    fc[node] = w[2] * sx + w[4] * sy + w[5] * sz;
  }
  __syncthreads();
  const double c = a.c_e[e];
  for (int node = threadIdx.x; node < nloc; node += blockDim.x) {
    const int i = node % np, j = (node / np) % np, k = node / (np * np);
    double s = 0;
    for (int mm = 0; mm < np; ++mm) {
      s += sD[i * np + mm] * fa[(k * np + j) * np + mm];
      s += sD[j * np + mm] * fb[(k * np + mm) * np + i];
      s += sD[k * np + mm] * fc[(mm * np + j) * np + i];
    }
    const double m = otf ? me[node] : a.mass[e * nloc + node];
    a.r_loc[e * nloc + node] = s + (c * su[node]) * m;
  }
}

// u_masked + scatter (operator.cpp:268-269, mesh.cpp:455-461)
__global__ void cx_scatter_kernel(const double* __restrict__ x, const std::uint8_t* __restrict__ mask,
                                  const int* __restrict__ l2g, long long n_loc, double* __restrict__ out)
{
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n_loc; q += (long long)gridDim.x * blockDim.x) {
    const int g = l2g[q];
    out[q] = (mask && mask[g]) ? 0.0 : x[g];
  }
}

// gather (mesh.cpp:463-475): sum = 0, copies in (e, l) order; optional
// Dirichlet identity rows (operator.cpp:279-280) or division by m_N
// (coarse.cpp:185)
__global__ void cx_gather_kernel(const double* __restrict__ loc, const unsigned* __restrict__ off,
                                 const int* __restrict__ idx, int n, const std::uint8_t* __restrict__ mask,
                                 const double* __restrict__ dirichlet_src, const double* __restrict__ divide_by,
                                 double* __restrict__ out)
{
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    double sum = 0;
    for (unsigned q = off[g]; q < off[g + 1]; ++q) sum += loc[idx[q]];
    if (divide_by) sum /= divide_by[g];
    if (mask && mask[g]) sum = dirichlet_src[g];
    out[g] = sum;
  }
}

// ---------------------------------------------------------------------------
// Fine preconditioner (fine.cpp:98-270)

struct CxFdmArgs {
  int P, nsub;
  const double* rin;
  const int* sub;
  const double* h3;
  const double* kappa_e;
  const double* c_e;
  const double* V;
  const double* Vinv;
  const double* lam;
  const double* M;
  const int* pos;
  double* zsort;
};

// tensor_pass (fine.cpp:98-136): out[.., d, ..] = sum_a mat[d*p+a] in[.., a, ..]
__device__ void cx_tensor_pass(int p, int axis, const double* mat, const double* in, double* out)
{
  const int n3 = p * p * p;
  for (int o = threadIdx.x; o < n3; o += blockDim.x) {
    const int x = o % p, y = (o / p) % p, z = o / (p * p);
    double s = 0;
    if (axis == 0) {
      const double* row = mat + x * p;
      const double* col = in + (z * p + y) * p;
      for (int a = 0; a < p; ++a) s += row[a] * col[a];
    } else if (axis == 1) {
      const double* row = mat + y * p;
      for (int a = 0; a < p; ++a) s += row[a] * in[(z * p + a) * p + x];
    } else {
      const double* row = mat + z * p;
      for (int a = 0; a < p; ++a) s += row[a] * in[(a * p + y) * p + x];
    }
    out[o] = s;
  }
  __syncthreads();
}

// solve_subdomain (fine.cpp:140-185) for one element per CTA; the outputs go
// to their (e, slot)-ordered accumulation positions (fine.cpp:224-227).
__global__ void cx_fdm_kernel(CxFdmArgs a)
{
  extern __shared__ double sh[];
  const int p = a.P, nsub = a.nsub;
  double* w = sh;
  double* t = w + nsub;
  double* sV = t + nsub;
  double* sVi = sV + p * p;
  const long long e = blockIdx.x;
  for (int q = threadIdx.x; q < p * p; q += blockDim.x) {
    sV[q] = a.V[q];
    sVi[q] = a.Vinv[q];
  }
  const double h0 = a.h3[3 * e], h1 = a.h3[3 * e + 1], h2 = a.h3[3 * e + 2];
  const double svol = 8.0 / (h0 * h1 * h2);
  const double ihx2 = 1.0 / (h0 * h0), ihy2 = 1.0 / (h1 * h1), ihz2 = 1.0 / (h2 * h2);
  const double kappa4 = 4 * a.kappa_e[e];
  const double c = a.c_e[e];
  for (int node = threadIdx.x; node < nsub; node += blockDim.x) {
    const int i = node % p, j = (node / p) % p, k = node / (p * p);
    const int g = a.sub[e * nsub + node];
    const double r = g < 0 ? 0.0 : a.rin[g];
    w[node] = svol * r / (a.M[i] * a.M[j] * a.M[k]);
  }
  __syncthreads();
  cx_tensor_pass(p, 0, sV, w, t);
  cx_tensor_pass(p, 1, sV, t, w);
  cx_tensor_pass(p, 2, sV, w, t);
  for (int node = threadIdx.x; node < nsub; node += blockDim.x) {
    const int dd = node % p, ee = (node / p) % p, ff = node / (p * p);
    t[node] /= kappa4 * (a.lam[dd] * ihx2 + a.lam[ee] * ihy2 + a.lam[ff] * ihz2) + c;
  }
  __syncthreads();
  cx_tensor_pass(p, 0, sVi, t, w);
  cx_tensor_pass(p, 1, sVi, w, t);
  cx_tensor_pass(p, 2, sVi, t, w);
  for (int node = threadIdx.x; node < nsub; node += blockDim.x) {
    const int q = a.pos[e * nsub + node];
    if (q >= 0) a.zsort[q] = w[node];
  }
}

// z_global[g] = 0 + contributions in (e, slot) order (fine.cpp:222-228)
__global__ void cx_sum_lists_kernel(const double* __restrict__ vals, const unsigned* __restrict__ off, int n,
                                    double* __restrict__ out)
{
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    double s = 0;
    for (unsigned q = off[g]; q < off[g + 1]; ++q) s += vals[q];
    out[g] = s;
  }
}

// ---------------------------------------------------------------------------
// Coarse preconditioner (coarse.cpp:138-208)

__global__ void cx_div_kernel(const double* __restrict__ x, const double* __restrict__ d, int n, double* __restrict__ y)
{
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) y[g] = x[g] / d[g];
}

// s_cb = sum_l B[cb][l] y[l] m[l] per (element, corner) (coarse.cpp:152-160)
__global__ void cx_restrict_kernel(const double* __restrict__ work, const int* __restrict__ l2g,
                                   const double* __restrict__ mass, const double* __restrict__ B, int nloc, int ne,
                                   double* __restrict__ Rpart)
{
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < 8LL * ne; q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / 8;
    const int cb = static_cast<int>(q % 8);
    const double* brow = B + cb * nloc;
    double s = 0;
    for (int l = 0; l < nloc; ++l) s += brow[l] * work[l2g[e * nloc + l]] * mass[e * nloc + l];
    Rpart[q] = s;
  }
}

// R[v] = 0 + the (e, cb) contributions in element order, then R[mask] = 0
// (coarse.cpp:158-160, 191-192)
__global__ void cx_vertex_kernel(const double* __restrict__ Rpart, const unsigned* __restrict__ off,
                                 const int* __restrict__ idx, const std::uint8_t* __restrict__ vmask, int nv,
                                 double* __restrict__ R)
{
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double s = 0;
    for (unsigned q = off[v]; q < off[v + 1]; ++q) s += Rpart[idx[q]];
    R[v] = vmask[v] ? 0.0 : s;
  }
}

// z_local[l] = (sum_cb B[cb][l] Z_cb) m[l] (coarse.cpp:172-181)
__global__ void cx_prolong_kernel(const double* __restrict__ Z, const int* __restrict__ conn,
                                  const double* __restrict__ B, const double* __restrict__ mass, int nloc, int ne,
                                  double* __restrict__ zl)
{
  const long long n = static_cast<long long>(ne) * nloc;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const long long e = q / nloc;
    const int l = static_cast<int>(q % nloc);
    double zc[8];
    for (int cb = 0; cb < 8; ++cb) zc[cb] = Z[conn[8 * e + (cb ^ ((cb >> 1) & 1))]];  // kHexCornerFromBits
    double s = 0;
    for (int cb = 0; cb < 8; ++cb) s += B[cb * nloc + l] * zc[cb];
    zl[q] = s * mass[q];
  }
}

// y = A x, row sums from 0 in stored order (CsrMatrix::multiply, amg.cpp:13-20)
__global__ void cx_spmv_kernel(const long long* __restrict__ ptr, const int* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ x, int n,
                               double* __restrict__ y)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0;
    for (long long q = ptr[i]; q < ptr[i + 1]; ++q) s += val[q] * x[col[q]];
    y[i] = s;
  }
}

// elementwise steps of cycle / ksolve / pcg / precond; op selects the formula
enum CxOp {
  kZeroY = 0,        // y = 0
  kCopy = 1,         // y = x0
  kJacobi0 = 2,      // y = omega d r            (amg.cpp:215)        x0 = d, x1 = r
  kJacobiUpd = 3,    // y += omega d (r - t)     (amg.cpp:212)        x0 = d, x1 = r, x2 = t
  kSubFrom = 4,      // y = x0 - x1
  kAxpy = 5,         // y += a x0
  kAxmy = 6,         // y -= a x0
  kXpay = 7,         // y = x0 + a y
  kAddAgg = 8,       // y += x0[agg[i]]           (amg.cpp:224)
  kMaskZero = 9,     // y = mask ? 0 : x0         (precond.cpp:35)
  kCombine = 10,     // y = mask ? x2 : (0 + [x0]) + [x1]  (precond.cpp:56-66)
  kAddTo = 11        // y += x0
};

struct CxVecArgs {
  int op, n;
  double a;
  const double *x0, *x1, *x2;
  const int* agg;
  const std::uint8_t* mask;
  int use0, use1;
  double* y;
};

__global__ void cx_vec_kernel(CxVecArgs v)
{
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.n; i += gridDim.x * blockDim.x) {
    switch (v.op) {
      case kZeroY: v.y[i] = 0; break;
      case kCopy: v.y[i] = v.x0[i]; break;
      case kJacobi0: v.y[i] = kOmega * v.x0[i] * v.x1[i]; break;
      case kJacobiUpd: v.y[i] += kOmega * v.x0[i] * (v.x1[i] - v.x2[i]); break;
      case kSubFrom: v.y[i] = v.x0[i] - v.x1[i]; break;
      case kAxpy: v.y[i] += v.a * v.x0[i]; break;
      case kAxmy: v.y[i] -= v.a * v.x0[i]; break;
      case kXpay: v.y[i] = v.x0[i] + v.a * v.y[i]; break;
      case kAddAgg: v.y[i] += v.x0[v.agg[i]]; break;
      case kMaskZero: v.y[i] = v.mask[i] ? 0.0 : v.x0[i]; break;
      case kCombine: {
        if (v.mask[i]) {
          v.y[i] = v.x2[i];
        } else {
          double s = 0;
          if (v.use0) s += v.x0[i];
          if (v.use1) s += v.x1[i];
          v.y[i] = s;
        }
        break;
      }
      case kAddTo: v.y[i] += v.x0[i]; break;
      default: break;
    }
  }
}

// aggregate sums rc[c] = 0 + rho over the members in ascending row order
// (amg.cpp:222: rc[agg[i]] += rho[i] for i ascending)
__global__ void cx_agg_sum_kernel(const double* __restrict__ rho, const int* __restrict__ aptr,
                                  const int* __restrict__ amem, int nc, double* __restrict__ rc)
{
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    double s = 0;
    for (int q = aptr[c]; q < aptr[c + 1]; ++q) s += rho[amem[q]];
    rc[c] = s;
  }
}

// dot (krylov.cpp:11-16): s += a_i b_i in index order. The products are
// independent (each rounded once, whoever computes it), so warps 1.. stage the
// next chunk of products in shared memory while thread 0 adds the current
// chunk in order: the only serial work left is the additions themselves.
constexpr int kDotChunk = 2048;
constexpr int kDotBlock = 512;
__global__ void __launch_bounds__(kDotBlock) cx_dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                           long long n, double* __restrict__ out)
{
  __shared__ double buf[2][kDotChunk];
  const int tid = threadIdx.x;
  for (int q = tid; q < kDotChunk && q < n; q += kDotBlock) buf[0][q] = a[q] * b[q];
  __syncthreads();
  double s = 0;
  for (long long base = 0; base < n; base += kDotChunk) {
    const int cur = static_cast<int>((base / kDotChunk) & 1);
    if (tid == 0) {
      const int m = static_cast<int>(n - base < kDotChunk ? n - base : kDotChunk);
      const double* v = buf[cur];
      for (int j = 0; j < m; ++j) s += v[j];
    } else if (tid >= 32) {
      const long long nb = base + kDotChunk;
      for (int q = tid - 32; q < kDotChunk && nb + q < n; q += kDotBlock - 32) buf[cur ^ 1][q] = a[nb + q] * b[nb + q];
    }
    __syncthreads();
  }
  if (tid == 0) *out = s;
}

// SimplicialLLT::solve as built for the reference (envelope factor after
// RCM): y = P b, L y' = y (row sweep), L^T x' = y' (column sweep), x = P^T x'.
// Row sweep: the products L_ik y_k of a row are independent (each rounded
// once), so the block forms them in shared memory and thread 0 subtracts
// them in k order. Column sweep: for a fixed i the updates of different y_k
// are independent, and each y_k still receives its updates in descending i.
constexpr int kEnvChunk = 2048;
__global__ void __launch_bounds__(256) cx_envelope_solve_kernel(CompatEnvelope f, const double* __restrict__ b,
                                                                double* __restrict__ x)
{
  __shared__ double prod[kEnvChunk];
  __shared__ double yi_s;
  const int tid = threadIdx.x;
  const long long n = f.n;
  double* y = f.y;
  for (long long i = tid; i < n; i += blockDim.x) y[i] = b[f.perm[i]];
  __syncthreads();
  for (long long i = 0; i < n; ++i) {
    const double* Li = f.env + f.start[i] - f.first[i];
    double s = 0;
    if (tid == 0) s = y[i];
    for (long long k0 = f.first[i]; k0 < i; k0 += kEnvChunk) {
      const int len = static_cast<int>(i - k0 < kEnvChunk ? i - k0 : kEnvChunk);
      for (int q = tid; q < len; q += blockDim.x) prod[q] = Li[k0 + q] * y[k0 + q];
      __syncthreads();
      if (tid == 0)
        for (int q = 0; q < len; ++q) s -= prod[q];
      __syncthreads();
    }
    if (tid == 0) y[i] = s / Li[i];
    __syncthreads();
  }
  for (long long i = n - 1; i >= 0; --i) {
    const double* Li = f.env + f.start[i] - f.first[i];
    if (tid == 0) {
      y[i] /= Li[i];
      yi_s = y[i];
    }
    __syncthreads();
    const double yi = yi_s;
    for (long long k = f.first[i] + tid; k < i; k += blockDim.x) y[k] -= Li[k] * yi;
    __syncthreads();
  }
  for (long long i = tid; i < n; i += blockDim.x) x[f.perm[i]] = y[i];
}

// ---------------------------------------------------------------------------
// host helpers

template <class T>
T* cx_upload(CompatPlan& c, const std::vector<T>& h)
{
  void* p = nullptr;
  CX_CUDA(cudaMalloc(&p, std::max<std::size_t>(1, h.size()) * sizeof(T)));
  c.owned.push_back(p);
  if (!h.empty()) CX_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return static_cast<T*>(p);
}

template <class T>
T* cx_alloc(CompatPlan& c, std::size_t n)
{
  void* p = nullptr;
  CX_CUDA(cudaMalloc(&p, std::max<std::size_t>(1, n) * sizeof(T)));
  c.owned.push_back(p);
  CX_CUDA(cudaMemset(p, 0, std::max<std::size_t>(1, n) * sizeof(T)));
  return static_cast<T*>(p);
}

CompatEnvelope upload_envelope(CompatPlan& c, const EnvelopeFactor& f)
{
  CompatEnvelope d;
  d.n = f.n;
  std::vector<long long> perm(f.perm.begin(), f.perm.end()), first(f.first.begin(), f.first.end()),
      start(f.start.begin(), f.start.end());
  d.perm = cx_upload(c, perm);
  d.first = cx_upload(c, first);
  d.start = cx_upload(c, start);
  d.env = cx_upload(c, f.env);
  d.y = cx_alloc<double>(c, f.n);
  return d;
}

void vec(cudaStream_t s, CxOp op, int n, double a, double* y, const double* x0 = nullptr, const double* x1 = nullptr,
         const double* x2 = nullptr, const int* agg = nullptr, const std::uint8_t* mask = nullptr, int use0 = 1,
         int use1 = 1)
{
  if (n <= 0) return;
  CxVecArgs v{op, n, a, x0, x1, x2, agg, mask, use0, use1, y};
  cx_vec_kernel<<<cx_grid(n), kCxBlock, 0, s>>>(v);
}

double dot(CompatPlan& c, cudaStream_t s, const double* a, const double* b, long long n)
{
  cx_dot_kernel<<<1, kDotBlock, 0, s>>>(a, b, n, c.scal);
  CX_CUDA(cudaMemcpyAsync(c.h_scal, c.scal, sizeof(double), cudaMemcpyDeviceToHost, s));
  CX_CUDA(cudaStreamSynchronize(s));
  return c.h_scal[0];
}

void spmv(cudaStream_t s, const CompatLevel& L, const double* x, double* y)
{
  cx_spmv_kernel<<<cx_grid(L.n), kCxBlock, 0, s>>>(L.ptr, L.col, L.val, x, L.n, y);
}

void direct_solve(CompatPlan& c, cudaStream_t s, const double* b, double* x)
{
  cx_envelope_solve_kernel<<<1, 256, 0, s>>>(c.coarsest, b, x);
}

void ksolve(CompatPlan& c, cudaStream_t s, std::size_t l, const double* b, double* x);

// AmgHierarchy::Impl::cycle (amg.cpp:199-228)
void cycle(CompatPlan& c, cudaStream_t s, std::size_t l, const double* r, double* z)
{
  if (l == c.lv.size()) {
    direct_solve(c, s, r, z);
    return;
  }
  CompatLevel& L = c.lv[l];
  const int n = L.n;
  vec(s, kJacobi0, n, 0, z, L.inv_diag, r);
  auto smooth = [&](int sweeps) {
    for (int q = 0; q < sweeps; ++q) {
      spmv(s, L, z, L.cy_tmp);
      vec(s, kJacobiUpd, n, 0, z, L.inv_diag, r, L.cy_tmp);
    }
  };
  smooth(kSweeps - 1);
  spmv(s, L, z, L.cy_tmp);
  vec(s, kSubFrom, n, 0, L.cy_rho, r, L.cy_tmp);
  cx_agg_sum_kernel<<<cx_grid(L.nc), kCxBlock, 0, s>>>(L.cy_rho, L.agg_ptr, L.agg_mem, L.nc, L.cy_rc);
  vec(s, kZeroY, L.nc, 0, L.cy_ec);
  ksolve(c, s, l + 1, L.cy_rc, L.cy_ec);
  vec(s, kAddAgg, n, 0, z, L.cy_ec, nullptr, nullptr, L.agg);
  smooth(kSweeps);
}

// AmgHierarchy::Impl::ksolve: exactly two PCG steps (amg.cpp:231-263)
void ksolve(CompatPlan& c, cudaStream_t s, std::size_t l, const double* b, double* x)
{
  if (l == c.lv.size()) {
    direct_solve(c, s, b, x);
    return;
  }
  CompatLevel& L = c.lv[l];
  const int n = L.n;
  vec(s, kCopy, n, 0, L.ks_r, b);
  vec(s, kZeroY, n, 0, x);
  cycle(c, s, l, L.ks_r, L.ks_z);
  double zr = dot(c, s, L.ks_z, L.ks_r, n);
  vec(s, kCopy, n, 0, L.ks_p, L.ks_z);
  for (int it = 0; it < 2; ++it) {
    spmv(s, L, L.ks_p, L.ks_f);
    const double pf = dot(c, s, L.ks_p, L.ks_f, n);
    if (!(pf > 0) || !(std::abs(zr) > 0)) return;
    const double alpha = zr / pf;
    vec(s, kAxpy, n, alpha, x, L.ks_p);
    vec(s, kAxmy, n, alpha, L.ks_r, L.ks_f);
    if (it == 1) break;
    cycle(c, s, l, L.ks_r, L.ks_z);
    const double zr_next = dot(c, s, L.ks_z, L.ks_r, n);
    const double beta = zr_next / zr;
    zr = zr_next;
    vec(s, kXpay, n, beta, L.ks_p, L.ks_z);
  }
}

// FinePreconditioner::apply(x) -> out (fine.cpp:210-231)
void fine_apply(CompatPlan& c, cudaStream_t s, const double* x, double* out)
{
  CxFdmArgs a{c.P, c.nsub, x, c.sub_l2g, c.h3, c.kappa_e, c.c_e, c.V, c.Vinv, c.lam, c.Mext, c.fine_pos, c.zsort};
  const std::size_t smem = sizeof(double) * (2 * static_cast<std::size_t>(c.nsub) + 2 * c.P * c.P);
  cx_fdm_kernel<<<c.ne, kCxBlock, smem, s>>>(a);
  cx_sum_lists_kernel<<<cx_grid(c.N), kCxBlock, 0, s>>>(c.zsort, c.fine_off, c.N, out);
}

// CoarsePreconditioner::apply(x) -> out (coarse.cpp:188-208)
void coarse_apply(CompatPlan& c, cudaStream_t s, const double* x, double* out)
{
  cx_div_kernel<<<cx_grid(c.N), kCxBlock, 0, s>>>(x, c.lumped, c.N, c.work);
  cx_restrict_kernel<<<cx_grid(8LL * c.ne), kCxBlock, 0, s>>>(c.work, c.l2g, c.mass, c.B, c.nloc, c.ne, c.Rpart);
  cx_vertex_kernel<<<cx_grid(c.nv), kCxBlock, 0, s>>>(c.Rpart, c.vtx_off, c.vtx_idx, c.vmask, c.nv, c.R);
  if (c.use_amg) {  // two composed K-cycles (coarse.cpp:193-200)
    cycle(c, s, 0, c.R, c.Z);
    CompatLevel K0{};
    K0.n = c.nv;
    K0.ptr = c.Kc_ptr;
    K0.col = c.Kc_col;
    K0.val = c.Kc_val;
    spmv(s, K0, c.Z, c.rho);
    vec(s, kSubFrom, c.nv, 0, c.rho, c.R, c.rho);
    cycle(c, s, 0, c.rho, c.dZ);
    vec(s, kAddTo, c.nv, 0, c.Z, c.dZ);
  } else {
    direct_solve(c, s, c.R, c.Z);
  }
  const long long nl = static_cast<long long>(c.ne) * c.nloc;
  cx_prolong_kernel<<<cx_grid(nl), kCxBlock, 0, s>>>(c.Z, c.conn, c.B, c.mass, c.nloc, c.ne, c.r_loc);
  cx_gather_kernel<<<cx_grid(c.N), kCxBlock, 0, s>>>(c.r_loc, c.g2l_off, c.g2l_idx, c.N, nullptr, nullptr, c.lumped,
                                                      out);
}

}  // namespace

CompatPlan::~CompatPlan()
{
  for (void* p : owned) cudaFree(p);
  if (h_scal) cudaFreeHost(h_scal);
}

void compat_init(CompatPlan& c, const HostSetup& hs)
{
  const Numbering& num = hs.num;
  c.np = hs.basis.npts();
  c.nloc = c.np * c.np * c.np;
  c.nlocp = (c.nloc + 1) & ~1;
  c.ne = hs.mesh.num_elements();
  c.N = num.num_global;
  c.P = c.np + 2;
  c.nsub = c.P * c.P * c.P;
  c.nv = hs.mesh.num_vertices();
  c.do_fine = hs.do_fine;
  c.do_coarse = hs.do_coarse;
  c.use_amg = hs.use_amg;
  const std::size_t nl = static_cast<std::size_t>(c.ne) * c.nloc;
  // full l2g and the g2l copy lists in (e, l) order (mesh.cpp:352-367)
  std::vector<int> l2g(nl);
  for (int e = 0; e < c.ne; ++e) element_l2g(num, c.ne, e, l2g.data() + static_cast<std::size_t>(e) * c.nloc);
  std::vector<unsigned> off(static_cast<std::size_t>(c.N) + 1, 0);
  for (int g : l2g) off[g + 1]++;
  for (int g = 0; g < c.N; ++g) off[g + 1] += off[g];
  std::vector<int> idx(nl);
  {
    std::vector<unsigned> cur(off.begin(), off.end() - 1);
    for (std::size_t q = 0; q < nl; ++q) idx[cur[l2g[q]]++] = static_cast<int>(q);
  }
  c.l2g = cx_upload(c, l2g);
  c.g2l_off = cx_upload(c, off);
  c.g2l_idx = cx_upload(c, idx);
  c.D = cx_upload(c, hs.basis.deriv);
  c.nodes = cx_upload(c, hs.basis.nodes);
  c.weights = cx_upload(c, hs.basis.weights);
  c.u_loc = cx_alloc<double>(c, nl);
  c.r_loc = cx_alloc<double>(c, nl);
  for (double** v : {&c.rm, &c.zf, &c.zc, &c.work, &c.u, &c.r, &c.z, &c.p, &c.f}) *v = cx_alloc<double>(c, c.N);
  c.scal = cx_alloc<double>(c, 8);
  CX_CUDA(cudaMallocHost(&c.h_scal, 8 * sizeof(double)));
  if (c.do_fine) {
    std::vector<int> sub(static_cast<std::size_t>(c.ne) * c.nsub, -1);
    std::vector<gid> scratch(c.nloc);
    for (int e = 0; e < c.ne; ++e)
      for_each_sub_slot(num, c.ne, e, scratch.data(),
                        [&](gid g, int slot) { sub[static_cast<std::size_t>(e) * c.nsub + slot] = g; });
    c.sub_l2g = cx_upload(c, sub);
    c.V = cx_upload(c, hs.pencil.V);
    c.Vinv = cx_upload(c, hs.pencil.V_inv);
    c.lam = cx_upload(c, hs.pencil.lambda);
    c.Mext = cx_upload(c, hs.pencil.M);
  }
  if (c.do_coarse) {
    c.B = cx_upload(c, hs.basis.coarse_vandermonde);
    c.Rpart = cx_alloc<double>(c, 8 * static_cast<std::size_t>(c.ne));
    for (double** v : {&c.R, &c.Z, &c.rho, &c.dZ}) *v = cx_alloc<double>(c, c.nv);
    std::vector<long long> kp(hs.Kc.ptr.begin(), hs.Kc.ptr.end());
    c.Kc_ptr = cx_upload(c, kp);
    c.Kc_col = cx_upload(c, hs.Kc.col);
    c.Kc_val = cx_upload(c, hs.Kc.val);
    if (c.use_amg) {
      for (const AmgLevel& h : hs.amg.levels) {
        CompatLevel L;
        L.n = h.A.n;
        L.nc = h.n_coarse;
        std::vector<long long> ptr(h.A.ptr.begin(), h.A.ptr.end());
        L.ptr = cx_upload(c, ptr);
        L.col = cx_upload(c, h.A.col);
        L.val = cx_upload(c, h.A.val);
        L.inv_diag = cx_upload(c, h.inv_diag);
        L.agg = cx_upload(c, h.aggregate);
        std::vector<int> aptr(static_cast<std::size_t>(L.nc) + 1, 0), amem(L.n);
        for (int i = 0; i < L.n; ++i) aptr[h.aggregate[i] + 1]++;
        for (int q = 0; q < L.nc; ++q) aptr[q + 1] += aptr[q];
        std::vector<int> cur(aptr.begin(), aptr.end() - 1);
        for (int i = 0; i < L.n; ++i) amem[cur[h.aggregate[i]]++] = i;
        L.agg_ptr = cx_upload(c, aptr);
        L.agg_mem = cx_upload(c, amem);
        for (double** v : {&L.cy_rho, &L.cy_tmp, &L.ks_r, &L.ks_z, &L.ks_p, &L.ks_f}) *v = cx_alloc<double>(c, L.n);
        L.cy_rc = cx_alloc<double>(c, L.nc);
        L.cy_ec = cx_alloc<double>(c, L.nc);
        c.lv.push_back(L);
      }
      c.coarsest = upload_envelope(c, envelope_cholesky(hs.amg.coarsest));
    } else {
      c.coarsest = upload_envelope(c, envelope_cholesky(hs.Kc));
    }
  }
  CX_CUDA(cudaDeviceSynchronize());
  c.ready = true;
}

void compat_apply_A(CompatPlan& c, const double* u, double* r, cudaStream_t s)
{
  const long long nl = static_cast<long long>(c.ne) * c.nloc;
  cx_scatter_kernel<<<cx_grid(nl), kCxBlock, 0, s>>>(u, c.mask, c.l2g, nl, c.u_loc);
  CxAxArgs a{c.np, c.nloc, c.nlocp, c.variant, c.u_loc, c.r_loc, c.D, c.wg, c.erec, c.nodes, c.weights, c.mass, c.c_e};
  std::size_t smem = sizeof(double) * (4 * static_cast<std::size_t>(c.nloc) + c.np * c.np);
  if (c.variant == HXB_VARIANT_ON_THE_FLY) smem += sizeof(double) * 7 * c.nloc;
  CX_CUDA(cudaFuncSetAttribute(cx_ax_elem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cx_ax_elem_kernel<<<c.ne, kCxBlock, smem, s>>>(a);
  cx_gather_kernel<<<cx_grid(c.N), kCxBlock, 0, s>>>(c.r_loc, c.g2l_off, c.g2l_idx, c.N, c.mask, u, nullptr, r);
  CX_CUDA(cudaGetLastError());
}

void compat_apply_P(CompatPlan& c, int precond_mode, int which, const double* r, double* z, cudaStream_t s)
{
  if (which == HXB_PRECOND_FINE_ONLY) {
    fine_apply(c, s, r, z);
  } else if (which == HXB_PRECOND_COARSE_ONLY) {
    coarse_apply(c, s, r, z);
  } else if (precond_mode == HXB_PRECOND_NONE) {  // TwoScalePreconditioner::apply (precond.cpp:27-67)
    vec(s, kCopy, c.N, 0, z, r);
  } else {
    vec(s, kMaskZero, c.N, 0, c.rm, r, nullptr, nullptr, nullptr, c.mask);
    if (c.do_fine) fine_apply(c, s, c.rm, c.zf);
    if (c.do_coarse) coarse_apply(c, s, c.rm, c.zc);
    vec(s, kCombine, c.N, 0, z, c.zf, c.zc, r, nullptr, c.mask, c.do_fine ? 1 : 0, c.do_coarse ? 1 : 0);
  }
  CX_CUDA(cudaGetLastError());
}

void compat_pcg(CompatPlan& c, int precond_mode, const double* b, const hxb_pcg_config& cfg, hxb_pcg_result* res,
                cudaStream_t s)
{
  if (!(cfg.rel_tolerance > 0) || !(cfg.rel_tolerance < 1))
    throw HxbError(HXB_EINVAL, "pcg: rel_tolerance must lie in (0,1)");
  if (cfg.max_iterations < 1) throw HxbError(HXB_EINVAL, "pcg: max_iterations must be >= 1");
  const int n = c.N;
  std::vector<double> rh, zh;
  vec(s, kCopy, n, 0, c.r, b);
  vec(s, kZeroY, n, 0, c.u);
  const double r0 = std::sqrt(dot(c, s, c.r, c.r, n));
  rh.push_back(r0);
  int status = HXB_PCG_CONVERGED, iterations = 0;
  std::string diag;
  if (r0 != 0.0) {
    compat_apply_P(c, precond_mode, -1, c.r, c.z, s);
    vec(s, kCopy, n, 0, c.p, c.z);
    double zr = dot(c, s, c.z, c.r, n);
    status = HXB_PCG_MAX_ITERATIONS;
    diag = "not converged within " + std::to_string(cfg.max_iterations) + " iterations";
    for (int k = 0; k < cfg.max_iterations; ++k) {
      zh.push_back(zr);
      compat_apply_A(c, c.p, c.f, s);
      const double pf = dot(c, s, c.p, c.f, n);
      if (!(pf > 0)) {
        status = HXB_PCG_BREAKDOWN;
        char buf[160];
        std::snprintf(buf, sizeof(buf), "indefinite operator: p.Ap = %f at iteration %d", pf, k);
        diag = buf;
        break;
      }
      const double alpha = zr / pf;
      vec(s, kAxpy, n, alpha, c.u, c.p);
      vec(s, kAxmy, n, alpha, c.r, c.f);
      iterations = k + 1;
      const double rn = std::sqrt(dot(c, s, c.r, c.r, n));
      rh.push_back(rn);
      if (rn / r0 <= cfg.rel_tolerance) {
        status = HXB_PCG_CONVERGED;
        diag.clear();
        break;
      }
      compat_apply_P(c, precond_mode, -1, c.r, c.z, s);
      const double zr_next = dot(c, s, c.z, c.r, n);
      const double beta = zr_next / zr;
      zr = zr_next;
      vec(s, kXpay, n, beta, c.p, c.z);
    }
  }
  CX_CUDA(cudaStreamSynchronize(s));
  res->status = status;
  res->iterations = iterations;
  res->num_residuals = cfg.record_history ? static_cast<int>(rh.size()) : 0;
  res->num_zr = cfg.record_history ? static_cast<int>(zh.size()) : 0;
  if (cfg.record_history) {
    if (res->residual_history) std::memcpy(res->residual_history, rh.data(), sizeof(double) * rh.size());
    if (res->zr_history && !zh.empty()) std::memcpy(res->zr_history, zh.data(), sizeof(double) * zh.size());
  }
  std::snprintf(res->diagnostic, sizeof(res->diagnostic), "%s", diag.c_str());
}

}  // namespace hxb
