// Device plan: setup upload, kernel orchestration, device-resident PCG, and
// the C-ABI declared in include/hexsem_b200.h.
//
// A plan is the B200 counterpart of the reference SemSystem
// (problem.hpp:68-85): built once from the mesh, it owns every device array;
// the PCG loop (krylov.cpp:20-71) runs entirely on the GPU with one 16-byte
// status read-back per iteration. The coarse correction runs on its own
// stream as a captured CUDA graph, concurrently with the fine FDM solves
// (the reference's std::async, precond.cpp:40-46).
#include <cuda.h>  // green-context types only: the functions come from cudaGetDriverEntryPointByVersion
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the functions are resolved by dlopen (NcclApi)

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/hexsem_b200.h"
#include "kernels_ax.cuh"
#include "kernels_coarse.cuh"
#include "kernels_setup.cuh"
#include "kernels_common.cuh"
#include "kernels_fine.cuh"
#include "kernels_gather.cuh"
#include "kernels_vec.cuh"
#include "capi_common.hpp"
#include "compat.hpp"
#include "setup.hpp"

namespace hxb {

namespace {


#define HXB_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t err__ = (call);                                                                     \
    if (err__ != cudaSuccess)                                                                       \
      throw HxbError(HXB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(err__));             \
  } while (0)

constexpr int kVecBlock = 256;
#ifndef COMBINE_TMA
#define COMBINE_TMA 1  // A/B: 0 = the warp-staged combine_prolong_kernel on single-device plans
#endif
#ifndef GATHER_FIRST_COPY_ORDER
#define GATHER_FIRST_COPY_ORDER 1  // A/B: 0 = the Ax gather walks surface nodes in global-id order
#endif
#ifndef ND_SPLIT_CTAS_PER_SM
#define ND_SPLIT_CTAS_PER_SM 2  // ND levels with fewer 32-row blocks than this many per SM use 8-row blocks
#endif
#ifndef COARSE_BLOCK
#define COARSE_BLOCK 256
#endif
constexpr int kCoarseBlock = COARSE_BLOCK;  // block of the coarse graph's vector kernels


int gather_grid(long long n)
{
  const long long b = (n + kGatherBlock - 1) / kGatherBlock;
  return static_cast<int>(std::max(1LL, std::min(b, 148LL * 8)));
}

// Grid for a grid-stride kernel: never more blocks than can be resident at
// once (one wave), so no block is left for a partial second wave.
int g_num_sms = 148;
template <class K>
int fill_grid(K kernel, int block, long long items)
{
  static thread_local std::vector<std::pair<const void*, int>> cache;
  const void* key = reinterpret_cast<const void*>(kernel);
  int per_sm = 0;
  for (const auto& kv : cache)
    if (kv.first == key) per_sm = kv.second;
  if (per_sm == 0) {
    HXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
    per_sm = std::max(per_sm, 1);
    cache.emplace_back(key, per_sm);
  }
  const long long need = (items + block - 1) / block;
  return static_cast<int>(std::max(1LL, std::min(need, static_cast<long long>(per_sm) * g_num_sms)));
}

int vec_grid(long long n)
{
  const long long b = (n + kVecBlock - 1) / kVecBlock;
  return static_cast<int>(std::max(1LL, std::min(b, 148LL * 4)));
}

// --- device memory tracking -------------------------------------------------
struct DeviceArena {
  std::vector<void*> ptrs;
  std::size_t bytes = 0;
  template <class T>
  T* alloc(std::size_t count)
  {
    if (count == 0) count = 1;
    void* p = nullptr;
    HXB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    ptrs.push_back(p);
    bytes += count * sizeof(T);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& h)
  {
    T* d = alloc<T>(h.size());
    if (!h.empty()) HXB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  ~DeviceArena()
  {
    for (void* p : ptrs) cudaFree(p);
  }
};

struct DevLevel {
  int n = 0, nc = 0;
  DevCsr A{};
  double* dinv = nullptr;
  int* agg = nullptr;
  int* agg_ptr = nullptr;
  int* agg_mem = nullptr;
  double *zA = nullptr, *zB = nullptr, *kr = nullptr, *kz = nullptr, *kp = nullptr, *kf = nullptr;
  double *b = nullptr, *x = nullptr;  // rc/ec targets from the finer level's cycle
  KScalars* ks = nullptr;
};

struct DevDense {
  // nested-dissection supernodal factor (large coupled blocks with vertex coordinates)
  bool nd = false;
  NdDev ndd;
  int nd_levels = 0, nd_max_m = 0;
  std::vector<std::pair<NdTask*, int>> nd_fwd_diag, nd_fwd_upd, nd_bwd_upd, nd_bwd_diag;  // per level
  std::int64_t nd_factor_bytes = 0;
  int n = 0, m = 0;
  double* ainv = nullptr;  // full row-major inverse (small blocks)
  int* coupled = nullptr;
  double* inv_diag = nullptr;
  // large blocks: lower-triangle 64x64 tiles of the inverse + partial-sum slots
  double* tiles = nullptr;
  long long ntiles = 0;
  int nt = 0;
  double *xg = nullptr, *rowpart = nullptr, *colpart = nullptr;
};

}  // namespace

struct Group;
void destroy_group(Group* g);
void destroy_green(CUgreenCtx g);

struct Plan {
  int device = 0;
  cudaStream_t s_main = nullptr, s_coarse = nullptr;  // s_coarse: highest priority
  bool split_combine = true;
  // restriction as its own pass before the FDM, so the coarse solve runs
  // concurrently with the fine solves and one combine follows (default for
  // single-device two-scale plans); false: restriction fused into the FDM and
  // the combine split around the coarse solve (hxb_options.restrict_in_fdm)
  bool restrict_first = false;
  bool fdm_one_per_cta = false;  // A/B (HXB_FDM_ONE_PER_CTA=1): one subdomain per FDM CTA at every order
  int* fdm_order = nullptr;  // FDM CTA -> element: Morton order of element centroids (neighbours close in time)
  bool host_lists = false;  // build the fine gather lists on the host (A/B checks of the device sort)
  bool bitwise = false;     // hxb_options.bitwise_reference: every apply/solve through compat.cu
  CompatPlan cx;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr, ev_a = nullptr;
  cudaGraphExec_t coarse_exec = nullptr;
  // SM partition (hxb_options.coarse_sms): s_coarse and s_fine are streams of
  // two green contexts splitting the SMs; null s_fine: no partition
  CUgreenCtx g_coarse = nullptr, g_fine = nullptr;
  cudaStream_t s_fine = nullptr;
  cudaEvent_t ev_fine = nullptr;
  int coarse_sms = 0;  // SMs of the coarse partition (0: none)
  DeviceArena mem;

  int order = 0, np = 0, nloc = 0, nsurf = 0, P = 0;
  int ne = 0, nv = 0, N = 0, nsg = 0;
  int num_sms = 148, ax_grid = 1;
  std::size_t n_ax_entries = 0;
  bool fdm_eo = false;
  int precond_mode = 0, variant = 0;
  bool do_fine = false, do_coarse = false, use_amg = false;
  double setup_seconds = 0;

  // host state kept for exports (planes dropped after upload); shared by the
  // ranks of a multi-GPU plan (built once, read-only afterwards)
  std::shared_ptr<HostSetup> hsp;
  HostSetup& hs;
  bool shared_setup = false;
  Group* group = nullptr;   // multi-GPU plan (hxb_options.n_gpus > 1): this Plan is only the handle
  Plan() : hsp(std::make_shared<HostSetup>()), hs(*hsp) {}
  explicit Plan(std::shared_ptr<HostSetup> shared) : hsp(std::move(shared)), hs(*hsp), shared_setup(true) {}
  gid coarse_n = 0;

  // device arrays
  double* wg = nullptr;
  double* erec = nullptr;  // on-the-fly variant: [e][26] corners + kappa
  double* mass = nullptr;
  double* c_e = nullptr;
  double* kappa_e = nullptr;
  double* h3 = nullptr;
  int* smap = nullptr;        // [e][2][nsurf]: encoded l2g codes, Ax CSR positions
  unsigned* ax_off = nullptr;
  std::uint8_t* mask = nullptr;
  double* d_lumped = nullptr;
  double* d_inv_lumped = nullptr;
  int* sub_face = nullptr;
  unsigned* fine_off = nullptr;
  int* fine_pos = nullptr;    // [e][P^3] CSR position (-1 sentinel)
  double* zsort = nullptr;
  int* conn = nullptr;
  unsigned* vtx_off = nullptr;
  int* vtx_idx = nullptr;
  std::uint8_t* vmask = nullptr;
  double *Rpart = nullptr, *R = nullptr, *Z = nullptr, *rho = nullptr, *dZ = nullptr;
  double* Zc = nullptr;       // [e][8] coarse corner values for the fused prolongation
  int* surf_first = nullptr;  // first copy of each surface item (combine's prolongation)
  double* cw = nullptr;       // [e][nsurf] restriction weights m_l / m_N of the surface slots (fused in the FDM)
  std::vector<DevLevel> lv;  // AMG levels 0..L (L = coarsest, uses dense)
  DevDense dense;
  DevCsr Kc{};               // K_c on the device (AMG mode: residual between the two K-cycles)
  std::uint8_t* zero_mask = nullptr;

  // PCG vectors
  double *u = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *f = nullptr, *b = nullptr, *rsurf = nullptr;
  int* ax_idx = nullptr;
  // scalars / reductions
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  double* cpartials = nullptr;
  unsigned* cticket = nullptr;
  double* zr_hist = nullptr;
  double* pf_hist = nullptr;
  double* res_hist = nullptr;
  double* res2 = nullptr;
  double* scratch = nullptr;
  double* h_status = nullptr;  // pinned
  int hist_cap = 0;

  // element-slab partition (distributed Ax); rank 0 of 1 = whole mesh
  int rank = 0, nranks = 1;
  int e0 = 0;                 // first owned element (global id); pl.ne counts owned elements
  int* ax_nodes = nullptr;    // local surface node -> global id (null: identity)
  // the Ax gather's own order (single-device plans): surface nodes sorted by
  // their first copy (e, slot), with the CSR permuted to match
  unsigned* gx_off = nullptr;
  int* gx_idx = nullptr;
  int* gx_nodes = nullptr;
  int n_loc_surf = 0;         // local surface nodes = [group0 | up | down]
  int n_grp0 = 0, n_up = 0, n_down = 0;
  int sfstride = 0;           // sub_face row stride (ints)
  int ne_total = 0;           // elements of the whole mesh
  // host-pointer Ax pipeline: copy streams and per-chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  // host-pointer Ax pipeline: surface-node id runs by the element chunk that
  // first needs them (H2D) and the chunk after which they are complete (D2H)
  struct IdRun {
    int g0, g1, chunk;
  };
  std::vector<IdRun> runs_in, runs_out;
  bool runs_ready = false;
  // distributed preconditioned CG (setup_dist.cpp)
  int* fin_surf = nullptr;    // finalised surface nodes (group 0 + down)
  int n_fin_surf = 0, ib0 = 0, ib1 = 0;
  int* frecv_pos = nullptr;   // [from down | from up] sum positions of the neighbours' contributions
  int n_frecv_down = 0, n_frecv_up = 0, n_fsend_down = 0, n_fsend_up = 0;
  int *g_from_down = nullptr, *g_from_up = nullptr, *g_to_down = nullptr, *g_to_up = nullptr;
  int n_g_from_down = 0, n_g_from_up = 0, n_g_to_down = 0, n_g_to_up = 0;
  int* loc_list = nullptr;    // local surface nodes (= ax_nodes) for vector updates
  double* fsend = nullptr;    // FDM contributions for the neighbours (caller buffer, set per call)
  std::vector<double> h_xyz;  // global node coordinates (heat driver), host copy
  double* d_xyz = nullptr;
  double* heat_u = nullptr;

  // live kernel timing (bench roofline): event pairs around tagged launches on s_main
  bool kt_on = false;
  std::vector<cudaEvent_t> kt_ev;
  std::vector<int> kt_tag;
  std::size_t kt_used = 0;
  long long launches = 0;      // kernels enqueued by the plan (graph nodes counted per launch)
  int coarse_graph_nodes = 0;

  ~Plan()
  {
    if (group) destroy_group(group);
    if (coarse_exec) cudaGraphExecDestroy(coarse_exec);
    for (cudaEvent_t e : {ev_fork, ev_join, ev_t0, ev_t1, ev_a})
      if (e) cudaEventDestroy(e);
    if (s_main) cudaStreamDestroy(s_main);
    if (s_coarse) cudaStreamDestroy(s_coarse);
    if (s_fine) cudaStreamDestroy(s_fine);
    if (ev_fine) cudaEventDestroy(ev_fine);
    destroy_green(g_coarse);
    destroy_green(g_fine);
    if (h_status) cudaFreeHost(h_status);
    for (cudaEvent_t e : kt_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
  }
};

namespace {

// --- template dispatch over the polynomial order --------------------------
#define HXB_DISPATCH_NP(np, F, ...)                         \
  switch (np) {                                             \
    case 2: F<2>(__VA_ARGS__); break;                       \
    case 3: F<3>(__VA_ARGS__); break;                       \
    case 4: F<4>(__VA_ARGS__); break;                       \
    case 5: F<5>(__VA_ARGS__); break;                       \
    case 6: F<6>(__VA_ARGS__); break;                       \
    case 7: F<7>(__VA_ARGS__); break;                       \
    case 8: F<8>(__VA_ARGS__); break;                       \
    case 9: F<9>(__VA_ARGS__); break;                       \
    case 10: F<10>(__VA_ARGS__); break;                     \
    case 11: F<11>(__VA_ARGS__); break;                     \
    default: throw HxbError(HXB_EINVAL, "order out of range 1..10"); \
  }

// tagged event pair around one launch (hxb_kernel_timing); no-op unless enabled
struct KtScope {
  Plan& pl;
  cudaStream_t s;
  bool on;
  KtScope(Plan& p, int tag, cudaStream_t st) : pl(p), s(st), on(p.kt_on && p.kt_used + 2 <= p.kt_ev.size())
  {
    if (on) {
      pl.kt_tag[pl.kt_used / 2] = tag;
      HXB_CUDA(cudaEventRecord(pl.kt_ev[pl.kt_used], s));
    }
  }
  ~KtScope()
  {
    if (on) {
      cudaEventRecord(pl.kt_ev[pl.kt_used + 1], s);
      pl.kt_used += 2;
    }
  }
};

DotArgs dot_args(Plan& pl, double* result, int offset = 0)
{
  DotArgs d;
  d.partials = pl.partials;
  d.ticket = pl.ticket;
  d.result = result;
  d.offset = offset;
  return d;
}

DotArgs cdot_args(Plan& pl, double* result)
{
  DotArgs d;
  d.partials = pl.cpartials;
  d.ticket = pl.cticket;
  d.result = result;
  d.offset = 0;
  return d;
}

#ifndef AX_SMALL_MAX_NP
#define AX_SMALL_MAX_NP 3  // thread-per-node Ax kernel up to this np (tile kernel above)
#endif
template <int NP, bool OTF>
int ax_persistent_grid_v(const Plan& pl)
{
  if constexpr (NP <= AX_SMALL_MAX_NP) {  // thread-per-node kernel for the low orders
    int per_sm = 0;
    HXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ax_small_kernel<NP, OTF>, AxSmall<NP>::kBlock, 0));
    per_sm = std::max(per_sm, 1);
    const int need = (pl.ne + AxSmall<NP>::kEPB - 1) / AxSmall<NP>::kEPB;
    return std::max(1, std::min(need, per_sm * pl.num_sms));
  }
  using Sh = AxShape<NP>;
  const int smem = static_cast<int>(OTF ? Sh::kSmemOtfBytes : Sh::kSmemBytes);
  HXB_CUDA(cudaFuncSetAttribute(ax_elem_kernel<NP, OTF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  HXB_CUDA(cudaFuncSetAttribute(ax_elem_kernel<NP, OTF>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  HXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ax_elem_kernel<NP, OTF>, Sh::kBlock, smem));
  per_sm = std::max(per_sm, 1);
  return std::max(1, std::min(pl.ne, per_sm * pl.num_sms));
}

template <int NP>
int ax_persistent_grid(const Plan& pl)
{
  return pl.variant == HXB_VARIANT_ON_THE_FLY ? ax_persistent_grid_v<NP, true>(pl) : ax_persistent_grid_v<NP, false>(pl);
}

template <int NP, bool OTF>
void launch_ax_kernel(const Plan& pl, const AxArgs& a, int grid, cudaStream_t s)
{
  if constexpr (NP <= AX_SMALL_MAX_NP)
    ax_small_kernel<NP, OTF><<<grid, AxSmall<NP>::kBlock, 0, s>>>(a);
  else
    ax_elem_kernel<NP, OTF><<<grid, AxShape<NP>::kBlock, OTF ? AxShape<NP>::kSmemOtfBytes : AxShape<NP>::kSmemBytes,
                              s>>>(a);
}

template <int NP>
void launch_ax_kernel(const Plan& pl, const AxArgs& a, int grid, cudaStream_t s)
{
  if (pl.variant == HXB_VARIANT_ON_THE_FLY)
    launch_ax_kernel<NP, true>(pl, a, grid, s);
  else
    launch_ax_kernel<NP, false>(pl, a, grid, s);
}

template <int NP>
void launch_ax_elem(Plan& pl, const double* u, double* r, DotArgs dot, cudaStream_t s)
{
  using Sh = AxShape<NP>;
  AxArgs a;
  a.u = u;
  a.wg = pl.wg;
  a.erec = pl.erec;
  a.mass = pl.mass;
  a.c_e = pl.c_e;
  a.smap = pl.smap;
  a.rsurf = pl.rsurf;
  a.r = r;
  a.ne = pl.ne;
  a.num_surface_global = pl.nsg + pl.e0 * (pl.order - 1) * (pl.order - 1) * (pl.order - 1);  // first owned interior id
  a.dot = dot;
  launch_ax_kernel<NP>(pl, a, pl.ax_grid, s);
}

// element range [e_begin, e_end) of the element kernel (host-pointer pipeline)
template <int NP>
void launch_ax_elem_range(Plan& pl, const double* u, double* r, int e_begin, int e_end, cudaStream_t s)
{
  using Sh = AxShape<NP>;
  AxArgs a;
  a.u = u;
  a.wg = pl.wg;
  a.erec = pl.erec;
  a.mass = pl.mass;
  a.c_e = pl.c_e;
  a.smap = pl.smap;
  a.rsurf = pl.rsurf;
  a.r = r;
  a.ne = e_end;
  a.e_begin = e_begin;
  a.num_surface_global = pl.nsg;
  a.dot = DotArgs{};
  int grid;
  if constexpr (NP <= AX_SMALL_MAX_NP)
    grid = std::max(1, std::min(pl.ax_grid, (e_end - e_begin + AxSmall<NP>::kEPB - 1) / AxSmall<NP>::kEPB));
  else
    grid = std::max(1, std::min(pl.ax_grid, e_end - e_begin));
  launch_ax_kernel<NP>(pl, a, grid, s);
}

template <int NP>
void init_ax_grid(Plan& pl)
{
  pl.ax_grid = ax_persistent_grid<NP>(pl);
}

int ax_elem_grid(const Plan& pl) { return pl.ax_grid; }

// f = A u (+ optional u.f into *dot_result)
void enqueue_ax(Plan& pl, const double* u, double* r, double* dot_result, cudaStream_t s)
{
  const int g_elem = ax_elem_grid(pl);
  DotArgs d1{}, d2{};
  if (dot_result) {
    d1 = dot_args(pl, nullptr, 0);
    d2 = dot_args(pl, dot_result, g_elem);
  }
  {
    KtScope kt(pl, HXB_KT_AX_ELEM, s);
    HXB_DISPATCH_NP(pl.np, launch_ax_elem, pl, u, r, d1, s);
  }
  AxGatherArgs g;
  g.rsurf = pl.rsurf;
  g.off = pl.ax_off;
  g.idx = pl.ax_idx;
  g.u = u;
  g.mask = pl.mask;
  g.r = r;
  g.num_surface_global = pl.nranks > 1 ? pl.n_grp0 : pl.nsg;  // distributed: interface nodes go through dist_*
  g.nodes = pl.ax_nodes;
  if (pl.gx_off) {  // first-copy order: rsurf rows are read while they are still in L2
    g.off = pl.gx_off;
    g.idx = pl.gx_idx;
    g.nodes = pl.gx_nodes;
  }
  g.dot = d2;
  {
    KtScope kt(pl, HXB_KT_AX_GATHER, s);
    ax_gather_kernel<<<fill_grid(ax_gather_kernel, kGatherBlock, g.num_surface_global), kGatherBlock, 0, s>>>(g);
  }
  pl.launches += 2;
}

template <int NP>
void launch_fdm(Plan& pl, cudaStream_t s)
{
  FdmArgs a;
  a.r = pl.r;
  a.smap = pl.smap;
  a.sub_face = pl.sub_face;
  a.h3 = pl.h3;
  a.kappa_e = pl.kappa_e;
  a.c_e = pl.c_e;
  a.pos = pl.fine_pos;
  a.zsort = pl.zsort;
  a.ne = pl.ne;
  a.sstride = 2 * pl.nsurf;
  a.num_surface_global = pl.nsg + pl.e0 * (pl.order - 1) * (pl.order - 1) * (pl.order - 1);  // first owned interior id
  a.cw = pl.cw;
  a.Rpart = pl.do_coarse && !pl.restrict_first ? pl.Rpart + 8LL * pl.e0 : nullptr;  // owned slab of the full Rpart
  a.fsend = pl.fsend;
  a.sfstride = pl.sfstride;
  a.order = pl.fdm_order;
  KtScope kt(pl, HXB_KT_FDM, s);
  pl.launches += 1;
  constexpr int EPB = FdmEPB<NP>::value;
  if (pl.fdm_eo && EPB > 1 && !a.Rpart && !a.fsend && !pl.fdm_one_per_cta)  // several subdomains per CTA
    fdm_kernel<NP, true, EPB><<<(pl.ne + EPB - 1) / EPB, FdmShapeE<NP, EPB>::kBlock, 0, s>>>(a);
  else if (pl.fdm_eo)
    fdm_kernel<NP, true><<<pl.ne, FdmShape<NP>::kBlock, 0, s>>>(a);
  else
    fdm_kernel<NP, false><<<pl.ne, FdmShape<NP>::kBlock, 0, s>>>(a);
}

template <int NP>
void launch_combine_np(Plan& pl, double* zr_result, cudaStream_t s, bool do_fine, bool do_coarse,
                       bool fine_in_z = false)
{
  CombineProlongArgs a;
  a.r = pl.r;
  a.mask = pl.mask;
  a.zsort = pl.zsort;
  a.fine_off = pl.fine_off;
  a.surf_first = pl.surf_first;
  a.Zc = pl.Zc;
  a.z = pl.z;
  if (pl.nranks > 1) {  // this rank's finalised nodes
    a.N = pl.n_fin_surf + (pl.ib1 - pl.ib0);
    a.nsg = pl.n_fin_surf;
    a.surf_nodes = pl.fin_surf;
    a.ibase = pl.ib0;
    a.e0 = pl.e0;
  } else {
    a.N = pl.N;
    a.nsg = pl.nsg;
    a.ibase = pl.nsg;
    a.e0 = 0;
  }
  a.do_fine = do_fine ? 1 : 0;
  a.do_coarse = do_coarse ? 1 : 0;
  a.fine_in_z = fine_in_z ? 1 : 0;
  a.dot = zr_result ? dot_args(pl, zr_result) : DotArgs{};
  if (COMBINE_TMA && pl.nranks == 1 && (do_fine || fine_in_z) && a.N > 0) {
    constexpr int kCombTile = CombTile<NP>::value, kCombSmem = comb_smem<kCombTile>();
    static bool attr = false;  // per NP instantiation
    if (!attr) {
      HXB_CUDA(cudaFuncSetAttribute(combine_tma_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCombSmem));
      attr = true;
    }
    const long long ntiles = (static_cast<long long>(a.N) + kCombTile - 1) / kCombTile;
    // tiles whose five ranges are in bounds: r/mask [t0, t0+T), fine_off [t0, t0+T+4)
    const long long span = static_cast<long long>(a.N) + 1 - kCombTile - 4;  // last in-bounds tile start
    const long long ntma = span < 0 ? 0 : span / kCombTile + 1;
    int per_sm = 0;
    constexpr int kCombBlock = CombTile<NP>::block;
    HXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, combine_tma_kernel<NP>, kCombBlock, kCombSmem));
    const int grid = static_cast<int>(std::max(1LL, std::min<long long>(ntiles, 1LL * std::max(per_sm, 1) * pl.num_sms)));
    combine_tma_kernel<NP><<<grid, kCombBlock, kCombSmem, s>>>(a, static_cast<int>(ntiles),
                                                                static_cast<int>(std::min(ntma, ntiles)));
    return;
  }
  combine_prolong_kernel<NP><<<fill_grid(combine_prolong_kernel<NP>, kGatherBlock, a.N), kGatherBlock, 0, s>>>(a);
}

void launch_combine(Plan& pl, double* zr_result, cudaStream_t s, bool do_fine, bool do_coarse,
                    bool fine_in_z = false)
{
  KtScope kt(pl, HXB_KT_COMBINE, s);
  pl.launches += 1;
  HXB_DISPATCH_NP(pl.np, launch_combine_np, pl, zr_result, s, do_fine, do_coarse, fine_in_z);
}

void launch_combine_fine(Plan& pl, cudaStream_t s, const PcgUArgs& ua = {})
{
  const bool dist = pl.nranks > 1;
  const int n_items = dist ? pl.n_fin_surf + (pl.ib1 - pl.ib0) : pl.N;
  const int nsg = dist ? pl.n_fin_surf : pl.nsg;
  const int ibase = dist ? pl.ib0 : pl.nsg;
  // one item per thread (a persistent grid leaves the coarse kernels no room: measured slower)
  combine_fine_kernel<<<std::max((n_items + kGatherBlock - 1) / kGatherBlock, 1), kGatherBlock, 0, s>>>(
      pl.zsort, pl.fine_off, dist ? pl.fin_surf : nullptr, nsg, ibase, n_items, pl.z, ua);
  pl.launches += 1;
}

// Zc = Z at each element's corners (interior copies, prolonged inside the
// combine) and the prolongated surface copies (coarse.cpp:164-181)
void launch_prolong(Plan& pl, cudaStream_t s)
{
  corner_values_kernel<<<vec_grid(8LL * pl.ne_total), kVecBlock, 0, s>>>(pl.Z, pl.conn, pl.Zc, pl.ne_total);
}

template <int NP>
void launch_restrict(Plan& pl, cudaStream_t s)
{
  if (!pl.cw) throw HxbError(HXB_EINVAL, "restriction weights missing (plan without a coarse branch)");
  const int grid = fill_grid(restrict_cw_kernel<NP>, 256, 32LL * pl.ne);
  restrict_cw_kernel<NP><<<grid, 256, 0, s>>>(pl.r, pl.smap, pl.cw, pl.Rpart, pl.ne, 2 * pl.nsurf, pl.nsurf, pl.nsg,
                                              pl.fdm_order);
}

// ---- AMG enqueue (captured into the coarse graph) --------------------------
void enqueue_nd(Plan& pl, const DevDense& d, const double* b, double* x, cudaStream_t s);

void enqueue_dense(Plan& pl, const double* b, double* x, cudaStream_t s)
{
  const DevDense& d = pl.dense;
  if (d.nd) {
    enqueue_nd(pl, d, b, x, s);
    return;
  }
  if (d.tiles) {  // packed symmetric tiles (large coupled block)
    const int mp = d.nt * kDenseTile;
    dense_gather_x_kernel<<<vec_grid(mp), kVecBlock, 0, s>>>(b, d.coupled, d.m, mp, d.xg);
    const unsigned grid = static_cast<unsigned>(std::min<long long>(d.ntiles, 8LL * pl.num_sms));
    dense_tile_gemv_kernel<<<grid, 256, 0, s>>>(d.tiles, d.xg, d.ntiles, d.rowpart, d.colpart);
    dense_tile_reduce_kernel<<<vec_grid(std::max(d.m, d.n)), kVecBlock, 0, s>>>(d.rowpart, d.colpart, d.m, d.nt,
                                                                                   d.coupled, d.inv_diag, b, x, d.n);
    return;
  }
  const int threads = 256;
  const int rows_per_block = threads / 32;
  int grid = std::max((d.m + rows_per_block - 1) / rows_per_block, (d.n + threads - 1) / threads);
  grid = std::max(1, std::min(grid, 148 * 8));
  dense_solve_kernel<<<grid, threads, 0, s>>>(d.ainv, d.coupled, d.m, d.inv_diag, b, x, d.n);
}

void enqueue_ksolve(Plan& pl, int l, const double* b, double* x, cudaStream_t s);

// grid of a coarse-graph kernel (grid-stride loops). Capping it so the
// graph's kernels need fewer CTA slots next to the concurrent FDM was measured
// slower at every cap (cfg2: 148 CTAs 4.44, 74 CTAs 4.60 ms per iteration
// against 4.35 uncapped, profiles/r02_ab_experiments.jsonl A/B 11).
int coarse_grid(const Plan& pl, long long n, int block = kCoarseBlock)
{
  (void)pl;
  return static_cast<int>(std::max(1LL, std::min((n + block - 1) / block, 148LL * 4)));
}

// Fusions used when the cycle runs inside ksolve(l): the K-solve's init
// (r_copy = r, x = 0) in the first kernel, its z.r (and p = z) in the last.
struct CycleFuse {
  double* r_copy = nullptr;
  double* x_zero = nullptr;
  KScalars* ks_init = nullptr;
  double* p_copy = nullptr;
  const DotArgs* dot = nullptr;
};

void enqueue_cycle(Plan& pl, int l, const double* r, double* zout, cudaStream_t s, const CycleFuse& fu = {})
{
  const int L = static_cast<int>(pl.lv.size()) - 1;
  if (l == L) {
    enqueue_dense(pl, r, zout, s);
    return;
  }
  DevLevel& v = pl.lv[l];
  DevLevel& c = pl.lv[l + 1];
  const int g = coarse_grid(pl, v.n);
  amg_jacobi2_kernel<<<g, kCoarseBlock, 0, s>>>(v.A, v.dinv, r, v.zA, fu.r_copy, fu.x_zero, fu.ks_init);
  amg_resid_kernel<<<g, kCoarseBlock, 0, s>>>(v.A, r, v.zA, v.kf);  // kf is free during the cycle
  amg_agg_sum_kernel<<<coarse_grid(pl, v.nc), kCoarseBlock, 0, s>>>(v.kf, v.agg_ptr, v.agg_mem, c.b, v.nc);
  enqueue_ksolve(pl, l + 1, c.b, c.x, s);
  amg_prolong_smooth_kernel<<<g, kCoarseBlock, 0, s>>>(v.A, v.dinv, r, v.zA, c.x, v.agg, v.zB);
  if (fu.dot)
    amg_smooth_dot_kernel<kCoarseBlock><<<g, kCoarseBlock, 0, s>>>(v.A, v.dinv, r, v.zB, zout, fu.p_copy, *fu.dot);
  else
    amg_smooth_kernel<<<g, kCoarseBlock, 0, s>>>(v.A, v.dinv, r, v.zB, zout);
}

void enqueue_ksolve(Plan& pl, int l, const double* b, double* x, cudaStream_t s)
{
  const int L = static_cast<int>(pl.lv.size()) - 1;
  if (l == L) {
    enqueue_dense(pl, b, x, s);
    return;
  }
  DevLevel& v = pl.lv[l];
  const int g = coarse_grid(pl, v.n);
  {  // init fused into the first cycle's Jacobi kernel, z.r and p = z into its last smoother
    const DotArgs d0 = cdot_args(pl, &v.ks->zr);
    CycleFuse fu;
    fu.r_copy = v.kr;
    fu.x_zero = x;
    fu.ks_init = v.ks;
    fu.p_copy = v.kp;
    fu.dot = &d0;
    enqueue_cycle(pl, l, b, v.kz, s, fu);
  }
  for (int it = 0; it < 2; ++it) {
    amg_spmv_dot_kernel<kCoarseBlock><<<g, kCoarseBlock, 0, s>>>(v.A, v.kp, v.kf, cdot_args(pl, &v.ks->pf));
    // amg.cpp:244-253; the second step reads zr from zr_next (the shift after kdir is folded in)
    amg_kupdate_kernel<<<g, kCoarseBlock, 0, s>>>(v.kp, v.kf, x, v.kr, v.n, v.ks, it);
    if (it == 1) break;
    const DotArgs d1 = cdot_args(pl, &v.ks->zr_next);
    CycleFuse fu;
    fu.dot = &d1;
    enqueue_cycle(pl, l, v.kr, v.kz, s, fu);
    amg_kdir_kernel<<<g, kCoarseBlock, 0, s>>>(v.kz, v.kp, v.n, v.ks);
  }
}

// Rpart -> R -> coarse solve -> Zc (coarse.cpp:188-206). Rpart comes from
// restrict_cw_kernel launched just before the graph (or, with
// restrict_in_fdm, from the FDM kernel's fused restriction).
void enqueue_coarse(Plan& pl, cudaStream_t s)
{
  vertex_gather_kernel<<<coarse_grid(pl, pl.nv), kCoarseBlock, 0, s>>>(pl.Rpart, pl.vtx_off, pl.vtx_idx, pl.vmask, pl.R, pl.nv);
  if (pl.use_amg) {
    enqueue_cycle(pl, 0, pl.R, pl.Z, s);
    // two composed K-cycles: Z = B R + B (R - K_c B R)  (coarse.cpp:193-200)
    const DevCsr K = pl.Kc;
    amg_resid_kernel<<<coarse_grid(pl, K.n), kCoarseBlock, 0, s>>>(K, pl.R, pl.Z, pl.rho);
    enqueue_cycle(pl, 0, pl.rho, pl.dZ, s);
    axpy1_kernel<<<coarse_grid(pl, K.n), kCoarseBlock, 0, s>>>(pl.Z, pl.dZ, K.n);
  } else {
    enqueue_dense(pl, pl.R, pl.Z, s);
  }
  launch_prolong(pl, s);
}

// ---- SM partition for the coarse solve (green contexts) -------------------
// The driver entry points are resolved through the runtime
// (cudaGetDriverEntryPointByVersion), so the library does not link libcuda.
struct GreenApi {
  CUresult (*dev_get)(CUdevice*, int) = nullptr;
  CUresult (*get_res)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned) = nullptr;
  CUresult (*gen_desc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*create)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*stream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  CUresult (*destroy)(CUgreenCtx) = nullptr;
  bool ok = false;
};

const GreenApi& green_api()
{
  static const GreenApi api = [] {
    GreenApi g;
    auto sym = [](const char* name, auto& fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPointByVersion(name, &p, CUDART_VERSION, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
      return fn != nullptr;
    };
    g.ok = sym("cuDeviceGet", g.dev_get) && sym("cuDeviceGetDevResource", g.get_res) &&
           sym("cuDevSmResourceSplitByCount", g.split) && sym("cuDevResourceGenerateDesc", g.gen_desc) &&
           sym("cuGreenCtxCreate", g.create) && sym("cuGreenCtxStreamCreate", g.stream) &&
           sym("cuGreenCtxDestroy", g.destroy);
    cudaGetLastError();
    return g;
  }();
  return api;
}

// SMs of the coarse partition when hxb_options.coarse_sms is 0
constexpr int kDefaultCoarseSms = -1;

// Split the device's SMs into a coarse partition of `want` SMs (rounded up to
// the hardware granularity) and the rest; s_coarse becomes a high-priority
// stream of the first, s_fine a stream of the second. The coarse graph is
// captured afterwards on s_coarse, so its replays stay on those SMs. Without
// driver support the plan keeps one shared SM pool (same results).
void make_sm_partition(Plan& pl, int want)
{
  const GreenApi& G = green_api();
  if (!G.ok) return;
  CUdevice dev = 0;
  CUdevResource all{}, part{}, rest{};
  unsigned nb = 1;
  if (G.dev_get(&dev, pl.device) != CUDA_SUCCESS || G.get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return;
  if (static_cast<unsigned>(want) >= all.sm.smCount ||
      G.split(&part, &nb, &all, &rest, 0, static_cast<unsigned>(want)) != CUDA_SUCCESS || nb != 1 ||
      rest.sm.smCount == 0)
    return;
  CUdevResourceDesc da = nullptr, db = nullptr;
  if (G.gen_desc(&da, &part, 1) != CUDA_SUCCESS || G.gen_desc(&db, &rest, 1) != CUDA_SUCCESS) return;
  CUgreenCtx ga = nullptr, gb = nullptr;
  if (G.create(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return;
  if (G.create(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    G.destroy(ga);
    return;
  }
  int lo = 0, hi = 0;
  HXB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CUstream sa = nullptr, sb = nullptr;
  if (G.stream(&sa, ga, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS ||
      G.stream(&sb, gb, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    if (sa) cudaStreamDestroy(sa);
    G.destroy(ga);
    G.destroy(gb);
    return;
  }
  HXB_CUDA(cudaStreamDestroy(pl.s_coarse));
  pl.s_coarse = sa;
  pl.s_fine = sb;
  pl.g_coarse = ga;
  pl.g_fine = gb;
  HXB_CUDA(cudaEventCreateWithFlags(&pl.ev_fine, cudaEventDisableTiming));
  pl.coarse_sms = static_cast<int>(part.sm.smCount);
}

}  // namespace

void destroy_green(CUgreenCtx g)
{
  if (g && green_api().ok) green_api().destroy(g);
}

namespace {

void capture_coarse_graph(Plan& pl)
{
  cudaGraph_t graph;
  HXB_CUDA(cudaStreamBeginCapture(pl.s_coarse, cudaStreamCaptureModeThreadLocal));
  enqueue_coarse(pl, pl.s_coarse);
  HXB_CUDA(cudaStreamEndCapture(pl.s_coarse, &graph));
  std::size_t nodes = 0;
  HXB_CUDA(cudaGraphGetNodes(graph, nullptr, &nodes));
  pl.coarse_graph_nodes = static_cast<int>(nodes);
  HXB_CUDA(cudaGraphInstantiate(&pl.coarse_exec, graph, 0));
  cudaGraphDestroy(graph);
}

// z = P r (reads pl.r, writes pl.z); optional z.r into *zr_result. With ua,
// the PCG's u += alpha_k p_k runs inside the fine half of the combine (in the
// shadow of the coarse solve); returns whether it did.
bool enqueue_precond(Plan& pl, double* zr_result, const PcgUArgs* ua = nullptr)
{
  cudaStream_t s = pl.s_main;
  if (pl.precond_mode == HXB_PRECOND_NONE) {
    copy_dot_kernel<kVecBlock><<<fill_grid(copy_dot_kernel<kVecBlock>, kVecBlock, pl.N), kVecBlock, 0, s>>>(pl.r, pl.r, pl.z, pl.N,
                                                                     zr_result ? dot_args(pl, zr_result) : DotArgs{});
    pl.launches += 1;
    return false;
  }
  if (pl.restrict_first) {
    // restriction pass, then the coarse solve (a latency-bound chain on a few
    // SMs, high-priority stream) concurrently with the fine solves; one
    // combine sums both, applies the mask and forms z.r
    HXB_DISPATCH_NP(pl.np, launch_restrict, pl, s);
    HXB_CUDA(cudaEventRecord(pl.ev_fork, s));
    HXB_CUDA(cudaStreamWaitEvent(pl.s_coarse, pl.ev_fork, 0));
    pl.launches += 1;
    {
      KtScope kt(pl, HXB_KT_COARSE, pl.s_coarse);
      HXB_CUDA(cudaGraphLaunch(pl.coarse_exec, pl.s_coarse));
    }
    pl.launches += pl.coarse_graph_nodes;
    HXB_CUDA(cudaEventRecord(pl.ev_join, pl.s_coarse));
    if (pl.s_fine) {  // SM partition: the fine solves on the other green context's SMs
      HXB_CUDA(cudaStreamWaitEvent(pl.s_fine, pl.ev_fork, 0));
      HXB_DISPATCH_NP(pl.np, launch_fdm, pl, pl.s_fine);
      HXB_CUDA(cudaEventRecord(pl.ev_fine, pl.s_fine));
      HXB_CUDA(cudaStreamWaitEvent(s, pl.ev_fine, 0));
    } else {
      HXB_DISPATCH_NP(pl.np, launch_fdm, pl, s);
    }
    HXB_CUDA(cudaStreamWaitEvent(s, pl.ev_join, 0));
    launch_combine(pl, zr_result, s, true, true);
    return false;
  }
  // fine FDM solves with the coarse restriction fused in (one pass over r),
  // then the coarse graph; the combine sums both and applies the mask
  if (pl.do_fine) {
    HXB_DISPATCH_NP(pl.np, launch_fdm, pl, s);
  } else if (pl.do_coarse) {
    HXB_DISPATCH_NP(pl.np, launch_restrict, pl, s);
    pl.launches += 1;
  }
  if (pl.do_fine && pl.do_coarse && pl.split_combine) {
    // the coarse solve (a latency-bound chain on a few SMs) on the
    // high-priority stream, concurrent with the fine half of the combine
    HXB_CUDA(cudaEventRecord(pl.ev_fork, s));
    HXB_CUDA(cudaStreamWaitEvent(pl.s_coarse, pl.ev_fork, 0));
    {
      KtScope kt(pl, HXB_KT_COARSE, pl.s_coarse);
      HXB_CUDA(cudaGraphLaunch(pl.coarse_exec, pl.s_coarse));
    }
    pl.launches += pl.coarse_graph_nodes;
    HXB_CUDA(cudaEventRecord(pl.ev_join, pl.s_coarse));
    const bool with_u = ua && pl.nranks == 1;
    {
      KtScope kt(pl, HXB_KT_COMBINE_FINE, s);
      launch_combine_fine(pl, s, with_u ? *ua : PcgUArgs{});
    }
    HXB_CUDA(cudaStreamWaitEvent(s, pl.ev_join, 0));
    launch_combine(pl, zr_result, s, false, true, true);
    return with_u;
  }
  if (pl.do_coarse) {
    KtScope kt(pl, HXB_KT_COARSE, s);
    HXB_CUDA(cudaGraphLaunch(pl.coarse_exec, s));
    pl.launches += pl.coarse_graph_nodes;
  }
  launch_combine(pl, zr_result, s, pl.do_fine, pl.do_coarse);
  return false;
}

// ---------------------------------------------------------------------------
// Setup

bool upload_tables(const GllBasis& basis, const Pencil& pencil)
{
  OrderTables t{};
  const int np = basis.npts();
  for (int q = 0; q < np * np; ++q) t.D[q] = basis.deriv[q];
  for (int m = 0; m < np; ++m)
    for (int i = 0; i < np; ++i) t.DT[m * np + i] = basis.deriv[i * np + m];
  for (int d = 0; d < pencil.p; ++d)
    for (int x = 0; x < pencil.p; ++x) {
      t.VT[x * pencil.p + d] = pencil.V[d * pencil.p + x];
      t.ViT[x * pencil.p + d] = pencil.V_inv[d * pencil.p + x];
    }
  for (int q = 0; q < pencil.p; ++q) {
    t.M[q] = pencil.M[q];
    t.invM[q] = 1.0 / pencil.M[q];
    t.lam[q] = pencil.lambda[q];
  }
  {  // even/odd split (fdm_kernel): eigenvector d must be even for even d, odd for odd d
    const int P = pencil.p, h = P / 2, mid = P & 1, NE = (P + 1) / 2, NO = P / 2;
    double vmax = 0;
    for (double v : pencil.V) vmax = std::max(vmax, std::fabs(v));
    double wmax = 0;
    for (double v : pencil.V_inv) wmax = std::max(wmax, std::fabs(v));
    bool ok = true;
    for (int d = 0; d < P; ++d) {
      const double sgn = (d % 2 == 0) ? 1.0 : -1.0;
      for (int x = 0; x < P; ++x) {
        if (std::fabs(pencil.V[d * P + x] - sgn * pencil.V[d * P + (P - 1 - x)]) > 1e-12 * vmax) ok = false;
        if (std::fabs(pencil.V_inv[x * P + d] - sgn * pencil.V_inv[(P - 1 - x) * P + d]) > 1e-12 * wmax) ok = false;
      }
    }
    t.eo_ok = ok ? 1 : 0;
    for (int x = 0; x < h + mid; ++x)
      for (int a = 0; a < NE; ++a) t.FE[x * NE + a] = pencil.V[(2 * a) * P + x];
    for (int x = 0; x < h; ++x)
      for (int a = 0; a < NO; ++a) t.FO[x * NO + a] = pencil.V[(2 * a + 1) * P + x];
    for (int a = 0; a < NE; ++a)
      for (int x = 0; x < h + mid; ++x) t.IE[a * (h + mid) + x] = pencil.V_inv[x * P + 2 * a];
    for (int a = 0; a < NO; ++a)
      for (int x = 0; x < h; ++x) t.IO[a * h + x] = pencil.V_inv[x * P + 2 * a + 1];
  }
  for (int i = 0; i < np; ++i) {
    t.hat0[i] = 0.5 * (1 - basis.nodes[i]);
    t.hat1[i] = 0.5 * (1 + basis.nodes[i]);
    t.w[i] = basis.weights[i];
  }
  HXB_CUDA(cudaMemcpyToSymbol(c_tab, &t, sizeof(OrderTables), sizeof(OrderTables) * np));
  FdmConst fc{};
  std::memcpy(fc.FE, t.FE, sizeof(fc.FE));
  std::memcpy(fc.FO, t.FO, sizeof(fc.FO));
  std::memcpy(fc.IE, t.IE, sizeof(fc.IE));
  std::memcpy(fc.IO, t.IO, sizeof(fc.IO));
  std::memcpy(fc.lam, t.lam, sizeof(fc.lam));
  std::memcpy(fc.invM, t.invM, sizeof(fc.invM));
  HXB_CUDA(cudaMemcpyToSymbol(c_fdm, &fc, sizeof(FdmConst), sizeof(FdmConst) * np));
  return t.eo_ok != 0;
}

// CSR by counting sort of a flat (already ascending) source index stream.
struct GatherCsr {
  std::vector<unsigned> off;
  std::vector<int> idx;
};

// Upload a nested-dissection factor of the coupled block (setup_nd.cpp) and
// its per-level task lists.
void nd_to_device(Plan& pl, DevDense& d, const NdFactor& F)
{
  DeviceArena& M = pl.mem;
  const int ns = static_cast<int>(F.sn.size());
  std::vector<int> c0(ns), mm(ns), rr(ns);
  std::vector<long long> linv_off(ns), l21_off(ns), rows_off(ns), inc_base(ns);
  long long nlinv = 0, nl21 = 0, nrows = 0, npos = 0;
  for (int s = 0; s < ns; ++s) {
    const NdSupernode& S = F.sn[s];
    c0[s] = S.c0;
    mm[s] = S.c1 - S.c0;
    rr[s] = static_cast<int>(S.rows.size());
    linv_off[s] = nlinv;
    l21_off[s] = nl21;
    rows_off[s] = nrows;
    inc_base[s] = npos;
    nlinv += static_cast<long long>(mm[s]) * mm[s];
    nl21 += static_cast<long long>(mm[s]) * rr[s];
    nrows += rr[s];
    npos += mm[s] + rr[s];
    d.nd_max_m = std::max(d.nd_max_m, mm[s]);
  }
  std::vector<double> linv(nlinv), linvT(nlinv), l21(nl21), l21T(nl21);
  std::vector<int> rows(nrows);
  for (int s = 0; s < ns; ++s) {
    const NdSupernode& S = F.sn[s];
    const int m = mm[s], r = rr[s];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        linv[linv_off[s] + static_cast<long long>(i) * m + j] = S.linv[static_cast<std::size_t>(i) * m + j];
        linvT[linv_off[s] + static_cast<long long>(j) * m + i] = S.linv[static_cast<std::size_t>(i) * m + j];
      }
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < m; ++j) {
        l21[l21_off[s] + static_cast<long long>(i) * m + j] = S.l21[static_cast<std::size_t>(i) * m + j];
        l21T[l21_off[s] + static_cast<long long>(j) * r + i] = S.l21[static_cast<std::size_t>(i) * m + j];
      }
    std::copy(S.rows.begin(), S.rows.end(), rows.begin() + rows_off[s]);
  }
  // incoming contributions of each front position: children's acc entries, child order
  std::vector<int> cnt(npos + 1, 0);
  std::vector<std::vector<std::pair<long long, int>>> lists(ns);
  for (int s = 0; s < ns; ++s) {
    const NdSupernode& S = F.sn[s];
    for (int c : S.children) {
      const NdSupernode& C = F.sn[c];
      for (int i = 0; i < rr[c]; ++i) {
        const int g = C.rows[i];
        int p;
        if (g < S.c1) {
          p = g - S.c0;
        } else {
          p = mm[s] + static_cast<int>(std::lower_bound(S.rows.begin(), S.rows.end(), g) - S.rows.begin());
        }
        lists[s].push_back({inc_base[s] + p, static_cast<int>(rows_off[c] + i)});
      }
    }
    for (const auto& e : lists[s]) cnt[e.first + 1]++;
  }
  for (long long q = 0; q < npos; ++q) cnt[q + 1] += cnt[q];
  std::vector<int> idx(cnt[npos]);
  {
    std::vector<int> cur(cnt.begin(), cnt.end() - 1);
    for (int s = 0; s < ns; ++s)
      for (const auto& e : lists[s]) idx[cur[e.first]++] = e.second;  // stable: child order, row order
  }
  NdDev& D = d.ndd;
  D.n = F.n;
  D.perm = M.upload(F.perm);
  D.c0 = M.upload(c0);
  D.m = M.upload(mm);
  D.r = M.upload(rr);
  D.linv_off = M.upload(linv_off);
  D.l21_off = M.upload(l21_off);
  D.linv = M.upload(linv);
  D.linvT = M.upload(linvT);
  D.l21 = M.upload(l21);
  D.l21T = M.upload(l21T);
  D.rows_off = M.upload(rows_off);
  D.rows = M.upload(rows);
  D.inc_base = M.upload(inc_base);
  D.inc_ptr = M.upload(cnt);
  D.inc_idx = M.upload(idx);
  for (double** v : {&D.y, &D.z, &D.t, &D.x}) *v = M.alloc<double>(std::max(1, F.n));
  D.acc = M.alloc<double>(std::max<long long>(1, nrows));
  d.nd_factor_bytes = static_cast<std::int64_t>(sizeof(double)) * 2 * (nlinv + nl21);
  // per-level task lists: blocks of kNdRowsPerTask rows, or of 8 rows (one
  // per warp) on the levels near the root, whose few large supernodes would
  // otherwise run on a few dozen CTAs (measured at 27^3, n=10: the root-side
  // backward updates took 35-42 us each on 21-45 CTAs)
  d.nd_levels = F.levels;
  std::vector<long long> lv_m(F.levels, 0), lv_r(F.levels, 0);
  for (int s = 0; s < ns; ++s) {
    lv_m[F.sn[s].level] += mm[s];
    lv_r[F.sn[s].level] += rr[s];
  }
  auto block_rows = [&](long long rows) {
    return rows / kNdRowsPerTask >= static_cast<long long>(ND_SPLIT_CTAS_PER_SM) * pl.num_sms ? kNdRowsPerTask : 8;
  };
  std::vector<std::vector<NdTask>> fd(F.levels), fu(F.levels), bu(F.levels), bd(F.levels);
  for (int s = 0; s < ns; ++s) {
    const int lv = F.sn[s].level;
    const int bm = block_rows(lv_m[lv]), br = block_rows(lv_r[lv]);
    for (int r0 = 0; r0 < mm[s]; r0 += bm) {
      const NdTask t{s, r0, std::min(bm, mm[s] - r0)};
      fd[lv].push_back(t);
      bu[lv].push_back(t);
      bd[lv].push_back(t);
    }
    for (int r0 = 0; r0 < rr[s]; r0 += br) fu[lv].push_back(NdTask{s, r0, std::min(br, rr[s] - r0)});
  }
  auto up = [&](const std::vector<std::vector<NdTask>>& v, std::vector<std::pair<NdTask*, int>>& out) {
    out.clear();
    for (const auto& l : v) out.push_back({l.empty() ? nullptr : M.upload(l), static_cast<int>(l.size())});
  };
  up(fd, d.nd_fwd_diag);
  up(fu, d.nd_fwd_upd);
  up(bu, d.nd_bwd_upd);
  up(bd, d.nd_bwd_diag);
  const int smem = static_cast<int>(sizeof(double) * std::max(1, d.nd_max_m));
  if (smem > 200 * 1024) throw HxbError(HXB_EINVAL, "coarse separator too large for the supernodal solve");
  HXB_CUDA(cudaFuncSetAttribute(nd_fwd_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  d.nd = true;
}

void enqueue_nd(Plan& pl, const DevDense& d, const double* b, double* x, cudaStream_t s)
{
  const NdDev& D = d.ndd;
  nd_permute_in_kernel<<<vec_grid(std::max(d.n, d.m)), kVecBlock, 0, s>>>(D.perm, d.coupled, d.m, d.inv_diag, b, D.y,
                                                                          x, d.n);
  const int smem = static_cast<int>(sizeof(double) * std::max(1, d.nd_max_m));
  for (int lv = 0; lv < d.nd_levels; ++lv) {
    if (d.nd_fwd_diag[lv].second)
      nd_fwd_diag_kernel<<<d.nd_fwd_diag[lv].second, kNdBlock, smem, s>>>(D, d.nd_fwd_diag[lv].first);
    if (d.nd_fwd_upd[lv].second)
      nd_fwd_upd_kernel<<<d.nd_fwd_upd[lv].second, kNdBlock, 0, s>>>(D, d.nd_fwd_upd[lv].first);
  }
  for (int lv = d.nd_levels - 1; lv >= 0; --lv) {
    if (d.nd_bwd_upd[lv].second)
      nd_bwd_upd_kernel<<<d.nd_bwd_upd[lv].second, kNdBlock, 0, s>>>(D, d.nd_bwd_upd[lv].first);
    if (d.nd_bwd_diag[lv].second)
      nd_bwd_diag_kernel<<<d.nd_bwd_diag[lv].second, kNdBlock, 0, s>>>(D, d.nd_bwd_diag[lv].first);
  }
  nd_permute_out_kernel<<<vec_grid(d.m), kVecBlock, 0, s>>>(D.perm, d.coupled, d.m, D.x, x);
  (void)pl;
}

DevDense dense_to_device(Plan& pl, const Csr& A, const std::vector<std::array<double, 3>>* coords = nullptr)
{
  DenseCoarse dc = dense_coarse_setup(A, 1500);
  DevDense d;
  d.n = dc.n;
  d.m = static_cast<int>(dc.coupled.size());
  d.coupled = pl.mem.upload(dc.coupled);
  d.inv_diag = pl.mem.upload(dc.inv_diag);
  const std::size_t mm = static_cast<std::size_t>(d.m) * d.m;
  if (!dc.ainv.empty() || d.m == 0) {
    d.ainv = pl.mem.upload(dc.ainv);
    return d;
  }
  if (coords && !std::getenv("HXB_DENSE_COARSE")) {  // sparse direct solve of the coupled block
    Csr B;
    B.n = d.m;
    B.ptr = dc.csr_ptr;
    B.col = dc.csr_col;
    B.val = dc.csr_val;
    std::vector<std::array<double, 3>> xyz(d.m);
    for (int q = 0; q < d.m; ++q) xyz[q] = (*coords)[dc.coupled[q]];
    setup_phase("coarse ND factor");
    const NdFactor F = nd_cholesky(B, xyz);
    nd_to_device(pl, d, F);
    return d;
  }
  // large coupled block: Cholesky on the device (64-bit cuSOLVER API: m^2 may
  // exceed 2^31) and the inverse from potrs against the identity; the
  // inverse is symmetric, so its column-major columns are the row-major rows
  const int m = d.m;
  double* L = nullptr;
  HXB_CUDA(cudaMalloc(&L, mm * sizeof(double)));
  HXB_CUDA(cudaMemset(L, 0, mm * sizeof(double)));
  {
    long long* dptr = nullptr;
    int* dcol = nullptr;
    double* dval = nullptr;
    HXB_CUDA(cudaMalloc(&dptr, dc.csr_ptr.size() * sizeof(long long)));
    HXB_CUDA(cudaMalloc(&dcol, std::max<std::size_t>(1, dc.csr_col.size()) * sizeof(int)));
    HXB_CUDA(cudaMalloc(&dval, std::max<std::size_t>(1, dc.csr_val.size()) * sizeof(double)));
    HXB_CUDA(cudaMemcpy(dptr, dc.csr_ptr.data(), dc.csr_ptr.size() * sizeof(long long), cudaMemcpyHostToDevice));
    HXB_CUDA(cudaMemcpy(dcol, dc.csr_col.data(), dc.csr_col.size() * sizeof(int), cudaMemcpyHostToDevice));
    HXB_CUDA(cudaMemcpy(dval, dc.csr_val.data(), dc.csr_val.size() * sizeof(double), cudaMemcpyHostToDevice));
    dense_scatter_kernel<<<vec_grid(m), kVecBlock>>>(dptr, dcol, dval, m, L);
    HXB_CUDA(cudaDeviceSynchronize());
    cudaFree(dptr);
    cudaFree(dcol);
    cudaFree(dval);
  }
  double* full = nullptr;  // the full inverse, packed into tiles below
  HXB_CUDA(cudaMalloc(&full, mm * sizeof(double)));
  d.ainv = full;
  HXB_CUDA(cudaMemset(d.ainv, 0, mm * sizeof(double)));
  dense_identity_kernel<<<vec_grid(m), kVecBlock>>>(d.ainv, m);
  cusolverDnHandle_t h;
  cusolverDnParams_t prm;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS || cusolverDnCreateParams(&prm) != CUSOLVER_STATUS_SUCCESS)
    throw HxbError(HXB_ECUDA, "cusolverDnCreate failed");
  std::size_t wdev = 0, whost = 0;
  cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, L, m, CUDA_R_64F, &wdev, &whost);
  void* work = nullptr;
  std::vector<unsigned char> hwork(std::max<std::size_t>(1, whost));
  int* info = nullptr;
  HXB_CUDA(cudaMalloc(&work, std::max<std::size_t>(1, wdev)));
  HXB_CUDA(cudaMalloc(&info, sizeof(int)));
  int hinfo = 0;
  cusolverStatus_t st = cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, L, m, CUDA_R_64F, work, wdev,
                                         hwork.data(), whost, info);
  HXB_CUDA(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
  if (st == CUSOLVER_STATUS_SUCCESS && hinfo == 0) {
    st = cusolverDnXpotrs(h, prm, CUBLAS_FILL_MODE_LOWER, m, m, CUDA_R_64F, L, m, CUDA_R_64F, d.ainv, m, info);
    HXB_CUDA(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
  }
  cudaFree(work);
  cudaFree(info);
  cudaFree(L);
  cusolverDnDestroyParams(prm);
  cusolverDnDestroy(h);
  if (st != CUSOLVER_STATUS_SUCCESS || hinfo != 0) {
    cudaFree(full);
    throw HxbError(HXB_ENUMERIC, "coarse matrix Cholesky failed (matrix not SPD?)");
  }
  d.nt = (m + kDenseTile - 1) / kDenseTile;
  d.ntiles = static_cast<long long>(d.nt) * (d.nt + 1) / 2;
  d.tiles = pl.mem.alloc<double>(static_cast<std::size_t>(d.ntiles) * kDenseTile * kDenseTile);
  dense_pack_kernel<<<static_cast<unsigned>(std::min<long long>(d.ntiles, 65535LL * 16)), 256>>>(full, m, d.tiles,
                                                                                                d.ntiles);
  HXB_CUDA(cudaDeviceSynchronize());
  cudaFree(full);
  d.ainv = nullptr;
  d.xg = pl.mem.alloc<double>(static_cast<std::size_t>(d.nt) * kDenseTile);
  d.rowpart = pl.mem.alloc<double>(static_cast<std::size_t>(d.ntiles) * kDenseTile);
  d.colpart = pl.mem.alloc<double>(static_cast<std::size_t>(d.ntiles) * kDenseTile);
  return d;
}

DevCsr csr_to_device(Plan& pl, const Csr& A)
{
  if (A.nnz() > 0x7fffffffULL) throw HxbError(HXB_EINVAL, "coarse matrix too large");
  std::vector<int> ptr(A.ptr.begin(), A.ptr.end());
  DevCsr d;
  d.n = A.n;
  d.ptr = pl.mem.upload(ptr);
  d.col = pl.mem.upload(A.col);
  d.val = pl.mem.upload(A.val);
  return d;
}

// Element-slab partition of the Ax gather. Rank r owns the
// elements [e0, e0+ne). Its surface nodes split into
//   group 0: all copies owned here            -> ax_gather_kernel
//   up:      copies also in rank r+1's slab     -> partial sum sent up
//   down:    copies also in rank r-1's slab     -> continue the partial received
// each group in ascending global id (the neighbour's matching list is the
// same set in the same order). A node spanning three ranks is rejected.
// Element-slab partition of the Ax gather, uploaded.
void build_dist_ax(Plan& pl, const HostSetup& hs, int /*nsurf_raw*/)
{
  DistLists d = dist_partition(hs, pl.rank, pl.nranks, pl.nsurf);
  pl.n_grp0 = d.n_grp0;
  pl.n_up = d.n_up;
  pl.n_down = d.n_down;
  pl.n_loc_surf = static_cast<int>(d.nodes.size());
  DeviceArena& M = pl.mem;
  pl.smap = M.upload(d.smap);
  pl.ax_off = M.upload(d.off);
  pl.ax_idx = M.upload(d.idx);
  pl.ax_nodes = M.upload(d.nodes);
  pl.n_ax_entries = d.off[pl.n_loc_surf];
}

// Stable counting sort of a flat source stream by destination on the device:
// keys[i] in [0, nkeys) or -1 (no destination). off = CSR offsets over the
// destinations; pos[i] = position of source i in its destination's list, in
// ascending i (the reference's accumulation order), -1 when skipped. Returns
// the number of entries. (The host equivalent is the two-pass counting sort.)
long long device_csr_by_key(const int* d_keys, long long n, int nkeys, unsigned* d_off, int* d_pos)
{
  if (n > 0x7fffffffLL) throw HxbError(HXB_EINVAL, "device_csr_by_key: too many entries");
  const int nn = static_cast<int>(n);
  int *k2 = nullptr, *vals = nullptr, *k2s = nullptr, *valss = nullptr;
  unsigned* counts = nullptr;
  HXB_CUDA(cudaMalloc(&k2, sizeof(int) * std::max(nn, 1)));
  HXB_CUDA(cudaMalloc(&vals, sizeof(int) * std::max(nn, 1)));
  HXB_CUDA(cudaMalloc(&k2s, sizeof(int) * std::max(nn, 1)));
  HXB_CUDA(cudaMalloc(&valss, sizeof(int) * std::max(nn, 1)));
  HXB_CUDA(cudaMalloc(&counts, sizeof(unsigned) * (static_cast<std::size_t>(nkeys) + 1)));
  HXB_CUDA(cudaMemset(counts, 0, sizeof(unsigned) * (static_cast<std::size_t>(nkeys) + 1)));
  iota_key_kernel<<<vec_grid(n), kVecBlock>>>(d_keys, n, nkeys, k2, vals, counts);
  HXB_CUDA(cudaGetLastError());
  std::size_t b1 = 0, b2 = 0;
  int bits = 1;
  while ((1LL << bits) <= nkeys) ++bits;
  HXB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b1, counts, d_off, nkeys + 1));
  HXB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, k2, k2s, vals, valss, nn, 0, bits));
  void* tmp = nullptr;
  HXB_CUDA(cudaMalloc(&tmp, std::max<std::size_t>({b1, b2, 1})));
  HXB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, b1, counts, d_off, nkeys + 1));
  HXB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b2, k2, k2s, vals, valss, nn, 0, bits));  // stable
  unsigned total = 0;
  HXB_CUDA(cudaMemcpy(&total, d_off + nkeys, sizeof(unsigned), cudaMemcpyDeviceToHost));
  scatter_pos_kernel<<<vec_grid(n), kVecBlock>>>(valss, total, n, d_pos);
  HXB_CUDA(cudaGetLastError());
  HXB_CUDA(cudaDeviceSynchronize());
  for (void* q : {static_cast<void*>(k2), static_cast<void*>(vals), static_cast<void*>(k2s), static_cast<void*>(valss),
                  static_cast<void*>(counts), tmp})
    cudaFree(q);
  return total;
}

// Ax gather order for single-device plans: surface nodes sorted by their
// first copy e*nsurf + slot (unique keys), the CSR rebuilt in that order. The
// gather then walks rsurf element by element (first copies contiguous, the
// other copies in neighbours handled a few rows later), instead of in
// global-id order, which revisits each rsurf sector from several faces after
// it may have left L2. Each node's own sum keeps its (e, l) order, so r is
// unchanged bit for bit; only the fused p.Ap's summation order moves.
void build_gather_order(Plan& pl)
{
  const int n = pl.nsg;
  DeviceArena tmp;
  int* key = tmp.alloc<int>(n);
  int* key2 = tmp.alloc<int>(n);
  int* val = tmp.alloc<int>(n);
  unsigned* cnt = tmp.alloc<unsigned>(static_cast<std::size_t>(n) + 1);
  pl.gx_nodes = pl.mem.alloc<int>(n);
  first_copy_kernel<<<vec_grid(n), kVecBlock>>>(pl.ax_off, pl.ax_idx, n, key);
  iota_kernel<<<vec_grid(n), kVecBlock>>>(val, n);
  int bits = 1;
  const long long maxkey = static_cast<long long>(pl.ne) * pl.nsurf;
  while ((1LL << bits) <= maxkey) ++bits;
  std::size_t b1 = 0, b2 = 0;
  HXB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, key, key2, val, pl.gx_nodes, n, 0, bits));
  pl.gx_off = pl.mem.alloc<unsigned>(static_cast<std::size_t>(n) + 1);
  HXB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, cnt, pl.gx_off, n + 1));
  void* work = tmp.alloc<unsigned char>(std::max<std::size_t>({b1, b2, 1}));
  HXB_CUDA(cub::DeviceRadixSort::SortPairs(work, b1, key, key2, val, pl.gx_nodes, n, 0, bits));
  perm_counts_kernel<<<vec_grid(n), kVecBlock>>>(pl.ax_off, pl.gx_nodes, n, cnt);
  HXB_CUDA(cub::DeviceScan::ExclusiveSum(work, b2, cnt, pl.gx_off, n + 1));
  pl.gx_idx = pl.mem.alloc<int>(std::max<std::size_t>(pl.n_ax_entries, 1));
  perm_segments_kernel<<<vec_grid(n), kVecBlock>>>(pl.ax_off, pl.ax_idx, pl.gx_nodes, pl.gx_off, n, pl.gx_idx);
  HXB_CUDA(cudaGetLastError());
  HXB_CUDA(cudaDeviceSynchronize());
}

template <int NP>
void launch_lumped(Plan& pl, const int* d_slot)
{
  lumped_mass_kernel<NP><<<vec_grid(pl.N), kVecBlock>>>(pl.ax_off, pl.ax_idx, pl.mass, d_slot, pl.nsurf, pl.nsg,
                                                          pl.N, pl.d_lumped, pl.d_inv_lumped);
}

template <int NP>
void launch_sub_keys(const Plan& pl, int* keys)
{
  sub_keys_kernel<NP><<<vec_grid(static_cast<long long>(pl.ne) * pl.P * pl.P * pl.P), kVecBlock>>>(
      pl.smap, 2 * pl.nsurf, pl.sub_face, pl.sfstride, pl.ne, pl.nsg, keys);
}

template <int NP>
void launch_geometry(const GeoArgs& a, long long n, cudaStream_t s)
{
  geometry_kernel<NP><<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a);
}

// compute_factors + kappa*mass scaling on the device: the
// stored planes go straight into their [e][6][nlocp] TMA layout, the mass is
// kept on the device and copied back once for the host-side consumers
// (lumped mass, coarse/prolongation lists).
void device_geometry(Plan& pl, HostSetup& hs, const hxb_options& opt)
{
  const int np = hs.basis.npts(), nloc = np * np * np, ne = hs.mesh.num_elements();
  const int nranks = std::max(1, opt.nranks), rank = nranks > 1 ? opt.rank : 0;
  const int e0 = static_cast<int>(static_cast<long long>(ne) * rank / nranks);
  const int e1 = static_cast<int>(static_cast<long long>(ne) * (rank + 1) / nranks);
  GeoArgs a{};
  for (int i = 0; i < np; ++i) {
    a.hat0[i] = 0.5 * (1 - hs.basis.nodes[i]);  // the jacobian's h (geometry.cpp:47-49)
    a.hat1[i] = 0.5 * (1 + hs.basis.nodes[i]);
    a.w[i] = hs.basis.weights[i];
  }
  std::vector<double> xyz(3 * static_cast<std::size_t>(hs.mesh.num_vertices()));
  for (std::size_t v = 0; v < hs.mesh.vertices.size(); ++v)
    for (int d = 0; d < 3; ++d) xyz[3 * v + d] = hs.mesh.vertices[v][d];
  std::vector<int> conn(8 * static_cast<std::size_t>(ne));
  for (int e = 0; e < ne; ++e)
    for (int q = 0; q < 8; ++q) conn[8 * static_cast<std::size_t>(e) + q] = hs.mesh.elements[e][q];
  DeviceArena tmp;
  a.xyz = tmp.upload(xyz);
  a.conn = tmp.upload(conn);
  a.kappa = tmp.upload(hs.kappa);
  a.ne = ne;
  a.e0 = e0;
  a.nel = e1 - e0;
  a.nlocp = (nloc + 1) & ~1;
  double* mass = (nranks == 1 ? pl.mem : tmp).alloc<double>(static_cast<std::size_t>(ne) * nloc);
  a.mass = mass;
  a.wg = opt.variant == HXB_VARIANT_STORED ? pl.mem.alloc<double>(static_cast<std::size_t>(e1 - e0) * 6 * a.nlocp)
                                           : nullptr;
  if (a.wg) HXB_CUDA(cudaMemset(a.wg, 0, static_cast<std::size_t>(e1 - e0) * 6 * a.nlocp * sizeof(double)));
  int* bad = tmp.alloc<int>(1);
  const int big = 0x7fffffff;
  HXB_CUDA(cudaMemcpy(bad, &big, sizeof(int), cudaMemcpyHostToDevice));
  a.bad = bad;
  HXB_DISPATCH_NP(np, launch_geometry, a, static_cast<long long>(ne) * nloc, cudaStream_t{});
  HXB_CUDA(cudaGetLastError());
  int first_bad = big;
  HXB_CUDA(cudaMemcpy(&first_bad, bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (first_bad != big)
    throw HxbError(HXB_EMESH, "inverted element " + std::to_string(first_bad) +
                                  ": non-positive Jacobian determinant at a GLL node");
  const bool device_lumped = std::max(1, opt.nranks) == 1 && opt.host_lists == 0;
  if (!device_lumped && !pl.shared_setup) {  // host consumers: lumped mass, host gather lists, distributed setup
    hs.geo.mass.resize(static_cast<std::size_t>(ne) * nloc);
    HXB_CUDA(cudaMemcpy(hs.geo.mass.data(), mass, hs.geo.mass.size() * sizeof(double), cudaMemcpyDeviceToHost));
  }
  pl.wg = a.wg;
  pl.mass = nranks == 1 ? mass : nullptr;
}

void build_plan(Plan& pl, const hxb_mesh* m, int order, const double* kappa_e, const double* c_e, const hxb_options& opt)
{
  const auto t0 = std::chrono::steady_clock::now();
  setup_phase("device init");
  if (!m) throw HxbError(HXB_EINVAL, "mesh must be non-null");
  if (m->num_elements <= 0) throw HxbError(HXB_EINVAL, "mesh has no hexahedra");  // cf. mesh_io.cpp:118
  if (opt.variant != HXB_VARIANT_STORED && opt.variant != HXB_VARIANT_ON_THE_FLY)
    throw HxbError(HXB_EINVAL, "unknown operator variant");
  pl.device = opt.device;
  HXB_CUDA(cudaSetDevice(pl.device));
  {
    cudaDeviceProp prop;
    HXB_CUDA(cudaGetDeviceProperties(&prop, pl.device));
    if (prop.major != 10) throw HxbError(HXB_ECUDA, "hexsem_b200 requires an sm_100 (B200) device");
    pl.num_sms = prop.multiProcessorCount;
    g_num_sms = prop.multiProcessorCount;
  }
  if (opt.bitwise_reference && (opt.nranks > 1 || opt.n_gpus > 1))
    throw HxbError(HXB_EINVAL, "bitwise_reference plans are single-device, single-rank");
  if (opt.bitwise_reference && opt.host_lists)
    throw HxbError(HXB_EINVAL, "bitwise_reference plans use the device fine lists");
  if (opt.nranks > 1) {  // validated before any setup work (the geometry hook reads them)
    if (opt.rank < 0 || opt.rank >= opt.nranks) throw HxbError(HXB_EINVAL, "rank out of range");
    if (opt.precond_mode != HXB_PRECOND_NONE && opt.precond_mode != HXB_PRECOND_TWO_SCALE)
      throw HxbError(HXB_EINVAL, "distributed plans support precond_mode two_scale or none");
    if (opt.nranks > m->num_elements) throw HxbError(HXB_EINVAL, "more ranks than elements");
  }
  HostSetup& hs = pl.hs;
  if (pl.shared_setup) {  // another rank of the multi-GPU plan built the host setup: only this slab's planes
    if (hs.order != order || hs.mesh.num_elements() != m->num_elements)
      throw HxbError(HXB_EINVAL, "shared host setup does not match the mesh");
    device_geometry(pl, hs, opt);
  } else {
    hs.mesh = mesh_from_arrays(m->num_vertices, m->xyz, m->num_elements, m->conn, m->num_boundary_faces,
                               m->bface_element, m->bface_face, m->bface_tag);
    const int ne0 = hs.mesh.num_elements();
    hs.kappa.assign(kappa_e, kappa_e + ne0);
    hs.c.assign(c_e, c_e + ne0);
    SetupOptions so;
    so.precond_mode = opt.precond_mode;
    so.coarse_solve = opt.coarse_solve;
    so.direct_threshold = opt.direct_threshold;
    so.store_planes = opt.variant == HXB_VARIANT_STORED;
    so.geometry_hook = [&pl, &opt](HostSetup& h) { device_geometry(pl, h, opt); };
    // single-device plan with device lists: the lumped mass is assembled on the
    // device after the surface CSR exists, so the masses never go back to the host
    so.device_lumped = std::max(1, opt.nranks) == 1 && opt.host_lists == 0;
    setup_phase("mesh + checks");
    build_host_setup(hs, order, so);
  }
  const int ne = hs.mesh.num_elements();
  setup_phase("device: streams, tables");
  const HexMesh& mesh = hs.mesh;
  const Numbering& num = hs.num;

  pl.order = order;
  pl.np = order + 1;
  pl.nloc = pl.np * pl.np * pl.np;
  const int nsurf_raw = surface_slot_count(pl.np);
  pl.nsurf = (nsurf_raw + 3) & ~3;  // padded element stride of every surface-slot array (16 B aligned)
  pl.P = order + 3;
  pl.nranks = std::max(1, opt.nranks);
  pl.rank = pl.nranks > 1 ? opt.rank : 0;
  pl.ne_total = ne;
  pl.e0 = static_cast<int>(static_cast<long long>(ne) * pl.rank / pl.nranks);
  pl.ne = static_cast<int>(static_cast<long long>(ne) * (pl.rank + 1) / pl.nranks) - pl.e0;
  pl.nv = mesh.num_vertices();
  pl.precond_mode = opt.precond_mode;
  pl.variant = opt.variant;
  pl.do_fine = hs.do_fine;
  pl.do_coarse = hs.do_coarse;
  pl.use_amg = hs.use_amg;
  pl.N = num.num_global;
  pl.nsg = num.num_surface_global;
  if (static_cast<std::size_t>(ne) * pl.nsurf > 0x7fffffffULL ||
      static_cast<std::size_t>(ne) * pl.P * pl.P * pl.P > 0x7fffffffULL)
    throw HxbError(HXB_EINVAL, "mesh too large for one device plan");

  pl.fdm_eo = upload_tables(hs.basis, hs.pencil);
  HXB_DISPATCH_NP(pl.np, init_ax_grid, pl);
  pl.split_combine = opt.fused_combine == 0;
  pl.host_lists = opt.host_lists != 0;

  HXB_CUDA(cudaStreamCreateWithFlags(&pl.s_main, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;
    HXB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    HXB_CUDA(cudaStreamCreateWithPriority(&pl.s_coarse, cudaStreamNonBlocking, hi));
  }
  for (cudaEvent_t* e : {&pl.ev_fork, &pl.ev_join}) HXB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&pl.ev_t0, &pl.ev_t1, &pl.ev_a}) HXB_CUDA(cudaEventCreate(e));

  DeviceArena& M = pl.mem;
  const int e0 = pl.e0, nel = pl.ne;  // owned elements [e0, e0 + nel)
  setup_phase("upload geometry");
  if (pl.variant == HXB_VARIANT_ON_THE_FLY) {  // element records: corners in (bi,bj,bk)-bit order, kappa
    constexpr int RD = 26;
    std::vector<double> rec(static_cast<std::size_t>(nel) * RD, 0.0);
    for (int le = 0; le < nel; ++le) {
      double* q = &rec[static_cast<std::size_t>(le) * RD];
      for (int b = 0; b < 8; ++b) {
        const auto& v = mesh.vertices[mesh.elements[e0 + le][hex_corner(b & 1, (b >> 1) & 1, b >> 2)]];
        for (int d = 0; d < 3; ++d) q[3 * b + d] = v[d];
      }
      q[24] = hs.kappa[e0 + le];
    }
    pl.erec = M.upload(rec);
  } else if (!pl.wg) {  // host planes regrouped per element: [e][6][nlocp] (one TMA stream per element)
    const int nlocp = (pl.nloc + 1) & ~1;
    const std::size_t total = static_cast<std::size_t>(ne) * pl.nloc;
    std::vector<double> wge(static_cast<std::size_t>(nel) * 6 * nlocp, 0.0);
    for (int le = 0; le < nel; ++le)
      for (int p = 0; p < 6; ++p)
        std::memcpy(&wge[(static_cast<std::size_t>(le) * 6 + p) * nlocp],
                    &hs.geo.wg[p * total + static_cast<std::size_t>(e0 + le) * pl.nloc], pl.nloc * sizeof(double));
    pl.wg = M.upload(wge);
  }
  if (!pl.shared_setup) {
    hs.geo.wg.clear();
    hs.geo.wg.shrink_to_fit();
  }
  auto slice = [&](const std::vector<double>& v, int per) {
    return std::vector<double>(v.begin() + static_cast<std::size_t>(e0) * per,
                               v.begin() + static_cast<std::size_t>(e0 + nel) * per);
  };
  if (!pl.mass) pl.mass = M.upload(pl.nranks > 1 ? slice(hs.geo.mass, pl.nloc) : hs.geo.mass);
  pl.c_e = M.upload(pl.nranks > 1 ? slice(hs.c, 1) : hs.c);
  pl.kappa_e = M.upload(pl.nranks > 1 ? slice(hs.kappa, 1) : hs.kappa);
  pl.h3 = M.upload(pl.nranks > 1 ? slice(hs.geo.h, 3) : hs.geo.h);
  pl.mask = M.upload(num.dirichlet_mask);
  pl.zero_mask = M.alloc<std::uint8_t>(pl.N);
  HXB_CUDA(cudaMemset(pl.zero_mask, 0, pl.N));
  if (!hs.lumped.empty()) {  // else assembled on the device once the surface CSR exists
    pl.d_lumped = M.upload(hs.lumped);
    std::vector<double> inv(hs.lumped.size());
    for (std::size_t g = 0; g < inv.size(); ++g) inv[g] = 1.0 / hs.lumped[g];
    pl.d_inv_lumped = M.upload(inv);
  }

  setup_phase("surface map + Ax CSR");
  // surface map [e][2][nsurf]: Dirichlet-encoded global ids and each copy's
  // position in the Ax surface CSR (copies of a node in ascending (e,l) order,
  // mesh.cpp:358-367) - producers write there, gathers stream contiguously
  if (pl.nranks == 1 && !pl.host_lists) {  // device sort of the surface copies by node
    const long long ncopy = static_cast<long long>(ne) * nsurf_raw;
    int* keys = nullptr;
    int* pos = nullptr;
    HXB_CUDA(cudaMalloc(&keys, sizeof(int) * std::max<long long>(1, ncopy)));
    HXB_CUDA(cudaMalloc(&pos, sizeof(int) * std::max<long long>(1, ncopy)));
    HXB_CUDA(cudaMemcpy(keys, num.l2g_surf.data(), sizeof(int) * ncopy, cudaMemcpyHostToDevice));
    pl.ax_off = M.alloc<unsigned>(static_cast<std::size_t>(pl.nsg) + 1);
    const long long total = device_csr_by_key(keys, ncopy, pl.nsg, pl.ax_off, pos);
    pl.n_ax_entries = static_cast<unsigned>(total);
    pl.smap = M.alloc<int>(static_cast<std::size_t>(ne) * 2 * pl.nsurf);
    HXB_CUDA(cudaMemset(pl.smap, 0, sizeof(int) * static_cast<std::size_t>(ne) * 2 * pl.nsurf));
    pl.ax_idx = M.alloc<int>(static_cast<std::size_t>(std::max<long long>(total, 1)));
    surface_map_kernel<<<vec_grid(ncopy), kVecBlock>>>(keys, pos, pl.mask, ne, nsurf_raw, pl.nsurf, pl.smap,
                                                        pl.ax_idx);
    HXB_CUDA(cudaGetLastError());
    pl.n_loc_surf = pl.n_grp0 = pl.nsg;
    if (hs.lumped.empty()) {  // lumped mass and 1/m_N from the device masses in CSR order
      std::vector<int> slot_l(nsurf_raw);
      for (int k = 0; k < pl.np; ++k)
        for (int j = 0; j < pl.np; ++j)
          for (int i = 0; i < pl.np; ++i) {
            const int sl = surface_slot(pl.np, i, j, k);
            if (sl >= 0) slot_l[sl] = (k * pl.np + j) * pl.np + i;
          }
      int* d_slot = M.upload(slot_l);
      pl.d_lumped = M.alloc<double>(pl.N);
      pl.d_inv_lumped = M.alloc<double>(pl.N);
      HXB_DISPATCH_NP(pl.np, launch_lumped, pl, d_slot);
      HXB_CUDA(cudaGetLastError());
      // the host copy (load vector, exports) is made on first use: host_lumped()
    }
    HXB_CUDA(cudaDeviceSynchronize());
    cudaFree(keys);
    cudaFree(pos);
  } else if (pl.nranks == 1) {
    std::vector<unsigned> off(static_cast<std::size_t>(pl.nsg) + 1, 0);
    for (gid g : num.l2g_surf) off[g + 1]++;
    for (int g = 0; g < pl.nsg; ++g) off[g + 1] += off[g];
    std::vector<unsigned> cur(off.begin(), off.end() - 1);
    std::vector<int> smap(static_cast<std::size_t>(ne) * 2 * pl.nsurf, 0);
    for (int e = 0; e < ne; ++e)
      for (int q = 0; q < nsurf_raw; ++q) {
        const gid g = num.l2g_surf[static_cast<std::size_t>(e) * nsurf_raw + q];
        int* row = &smap[static_cast<std::size_t>(e) * 2 * pl.nsurf];
        row[q] = num.dirichlet_mask[g] ? encode_dirichlet(g) : g;
        row[pl.nsurf + q] = static_cast<int>(cur[g]++);
      }
    pl.smap = M.upload(smap);
    pl.ax_off = M.upload(off);
    pl.n_ax_entries = off[pl.nsg];
    std::vector<int> idx(off[pl.nsg]);
    for (int e = 0; e < ne; ++e)
      for (int q = 0; q < nsurf_raw; ++q)
        idx[smap[static_cast<std::size_t>(e) * 2 * pl.nsurf + pl.nsurf + q]] = e * pl.nsurf + q;
    pl.ax_idx = M.upload(idx);
    pl.n_loc_surf = pl.n_grp0 = pl.nsg;
  } else {
    build_dist_ax(pl, hs, nsurf_raw);
  }
  pl.rsurf = M.alloc<double>(static_cast<std::size_t>(pl.ne) * pl.nsurf);
  if (pl.do_coarse && pl.nranks == 1 && pl.nsg > 0) {  // first copy of every surface node (combine's prolongation)
    // padded to whole combine tiles (combine_tma_kernel stages a tile's entries at once)
    const std::size_t padded = (static_cast<std::size_t>(pl.nsg) + kCombTileMax - 1) / kCombTileMax * kCombTileMax;
    pl.surf_first = M.alloc<int>(padded);
    HXB_CUDA(cudaMemset(pl.surf_first, 0, sizeof(int) * padded));
    first_copy_kernel<<<vec_grid(pl.nsg), kVecBlock>>>(pl.ax_off, pl.ax_idx, pl.nsg, pl.surf_first);
    HXB_CUDA(cudaGetLastError());
  }
  if (GATHER_FIRST_COPY_ORDER && pl.nranks == 1 && pl.nsg > 0) build_gather_order(pl);

  pl.restrict_first = pl.do_fine && pl.do_coarse && pl.nranks == 1 && opt.restrict_in_fdm == 0;
  if (pl.restrict_first && !pl.group) {
    const int want = opt.coarse_sms == 0 ? kDefaultCoarseSms : opt.coarse_sms;
    if (want > 0) make_sm_partition(pl, want);
  }
  if (const char* o = std::getenv("HXB_FDM_ONE_PER_CTA")) pl.fdm_one_per_cta = std::atoi(o) != 0;
  if (pl.do_coarse) {  // restriction weights m_l / m_N of the surface slots (restriction pass / fused in the FDM)
    std::vector<int> slot_l(nsurf_raw);
    for (int k = 0; k < pl.np; ++k)
      for (int j = 0; j < pl.np; ++j)
        for (int i = 0; i < pl.np; ++i) {
          const int sl = surface_slot(pl.np, i, j, k);
          if (sl >= 0) slot_l[sl] = (k * pl.np + j) * pl.np + i;
        }
    DeviceArena tmp;
    int* d_slot = tmp.upload(slot_l);
    pl.cw = M.alloc<double>(static_cast<std::size_t>(pl.ne) * pl.nsurf);
    restrict_weights_kernel<<<vec_grid(static_cast<long long>(pl.ne) * pl.nsurf), kVecBlock>>>(
        pl.smap, 2 * pl.nsurf, pl.mass, pl.nloc, pl.d_inv_lumped, d_slot, nsurf_raw, pl.nsurf, pl.ne, pl.cw);
    HXB_CUDA(cudaGetLastError());
    HXB_CUDA(cudaDeviceSynchronize());
  }
  setup_phase("fine lists");
  // fine: encoded sub_face and the subdomain gather CSR in (e, slot) order
  if (pl.do_fine) {
    const int nf = 6 * pl.np * pl.np, nfp = (nf + 3) & ~3;  // rows padded for 16-byte TMA copies
    pl.sfstride = nfp;
    // raw rows uploaded, Dirichlet-encoded and padded on the device
    DeviceArena tmp;
    const std::size_t nrow = static_cast<std::size_t>(pl.ne) * nf;
    int* raw = tmp.alloc<int>(nrow);
    HXB_CUDA(cudaMemcpy(raw, num.sub_face.data() + static_cast<std::size_t>(pl.e0) * nf, sizeof(int) * nrow,
                        cudaMemcpyHostToDevice));
    pl.sub_face = M.alloc<int>(static_cast<std::size_t>(pl.ne) * nfp);
    encode_sub_face_kernel<<<vec_grid(static_cast<long long>(pl.ne) * nfp), kVecBlock>>>(raw, pl.mask, pl.ne, nf, nfp,
                                                                                       pl.sub_face);
    HXB_CUDA(cudaGetLastError());
    HXB_CUDA(cudaDeviceSynchronize());
  }
  if (pl.do_fine && pl.nranks > 1) {
    const DistLists dl = dist_partition(hs, pl.rank, pl.nranks, pl.nsurf);
    const DistPcgLists d = dist_pcg_setup(hs, dl, pl.rank, pl.nranks);
    pl.fin_surf = M.upload(d.fin_surf);
    pl.n_fin_surf = static_cast<int>(d.fin_surf.size());
    pl.ib0 = d.ib0;
    pl.ib1 = d.ib1;
    pl.fine_off = M.upload(d.fine_off);
    pl.fine_pos = M.upload(d.fine_pos);
    pl.zsort = M.alloc<double>(std::max<std::size_t>(1, d.fine_off.back()));
    pl.n_fsend_down = d.n_fsend_down;
    pl.n_fsend_up = d.n_fsend_up;
    std::vector<int> fr(d.frecv_down);
    fr.insert(fr.end(), d.frecv_up.begin(), d.frecv_up.end());
    pl.frecv_pos = M.upload(fr);
    pl.n_frecv_down = static_cast<int>(d.frecv_down.size());
    pl.n_frecv_up = static_cast<int>(d.frecv_up.size());
    pl.g_from_down = M.upload(d.ghost_from_down);
    pl.g_from_up = M.upload(d.ghost_from_up);
    pl.g_to_down = M.upload(d.ghost_to_down);
    pl.g_to_up = M.upload(d.ghost_to_up);
    pl.n_g_from_down = static_cast<int>(d.ghost_from_down.size());
    pl.n_g_from_up = static_cast<int>(d.ghost_from_up.size());
    pl.n_g_to_down = static_cast<int>(d.ghost_to_down.size());
    pl.n_g_to_up = static_cast<int>(d.ghost_to_up.size());
    if (pl.n_fin_surf > 0) {  // first copy of every finalised surface node (combine's prolongation)
      DeviceArena tmp;
      const unsigned* d_off = tmp.upload(d.pr_off);
      const int* d_idx = tmp.upload(d.pr_idx);
      pl.surf_first = M.alloc<int>(pl.n_fin_surf);
      first_copy_kernel<<<vec_grid(pl.n_fin_surf), kVecBlock>>>(d_off, d_idx, pl.n_fin_surf, pl.surf_first);
      HXB_CUDA(cudaGetLastError());
      HXB_CUDA(cudaDeviceSynchronize());
    }
  } else if (pl.do_fine && !pl.host_lists) {
    // subdomain contributions' (e, slot)-ordered positions by a device sort
    const std::size_t nsub = static_cast<std::size_t>(pl.P) * pl.P * pl.P;
    int* keys = nullptr;
    HXB_CUDA(cudaMalloc(&keys, sizeof(int) * std::max<std::size_t>(1, ne * nsub)));
    HXB_DISPATCH_NP(pl.np, launch_sub_keys, pl, keys);
    HXB_CUDA(cudaGetLastError());
    pl.fine_off = M.alloc<unsigned>(static_cast<std::size_t>(pl.N) + 1);
    pl.fine_pos = M.alloc<int>(ne * nsub);
    const long long total = device_csr_by_key(keys, static_cast<long long>(ne * nsub), pl.N, pl.fine_off, pl.fine_pos);
    cudaFree(keys);
    pl.zsort = M.alloc<double>(static_cast<std::size_t>(std::max<long long>(total, 1)) + 2);  // +2: even-rounded tile copies
  } else if (pl.do_fine) {
    const std::size_t nsub = static_cast<std::size_t>(pl.P) * pl.P * pl.P;
    std::vector<unsigned> cnt(static_cast<std::size_t>(pl.N) + 1, 0);
    std::vector<gid> scratch(pl.nloc);
    for (int e = 0; e < ne; ++e)
      for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int) {
        if (g >= 0) cnt[g + 1]++;
      });
    for (int g = 0; g < pl.N; ++g) cnt[g + 1] += cnt[g];
    // each (e, slot) contribution's position in the per-node list, ascending
    // (e, slot) = the reference accumulation order (fine.cpp:224-227)
    std::vector<int> pos(static_cast<std::size_t>(ne) * nsub, -1);
    std::vector<unsigned> cur(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < ne; ++e)
      for_each_sub_slot(num, ne, e, scratch.data(), [&](gid g, int slot) {
        if (g >= 0) pos[static_cast<std::size_t>(e) * nsub + slot] = static_cast<int>(cur[g]++);
      });
    pl.fine_off = M.upload(cnt);
    pl.fine_pos = M.upload(pos);
    pl.zsort = M.alloc<double>(static_cast<std::size_t>(cnt[pl.N]) + 2);  // +2: even-rounded tile copies
  }
  if (pl.nranks > 1) {
    std::vector<int> nodes_host(pl.n_loc_surf);
    HXB_CUDA(cudaMemcpy(nodes_host.data(), pl.ax_nodes, sizeof(int) * pl.n_loc_surf, cudaMemcpyDeviceToHost));
    pl.loc_list = pl.ax_nodes;
    if (!pl.do_fine) {  // operator-only plan: finalised set still needed for dots
      std::vector<int> fs(nodes_host.begin(), nodes_host.begin() + pl.n_grp0);
      fs.insert(fs.end(), nodes_host.begin() + pl.n_grp0 + pl.n_up, nodes_host.end());
      pl.fin_surf = M.upload(fs);
      pl.n_fin_surf = static_cast<int>(fs.size());
      const long long NI = static_cast<long long>(pl.order - 1) * (pl.order - 1) * (pl.order - 1);
      pl.ib0 = static_cast<int>(pl.nsg + pl.e0 * NI);
      pl.ib1 = static_cast<int>(pl.nsg + (pl.e0 + pl.ne) * NI);
    }
  }

  if (pl.do_fine && pl.nranks == 1 && opt.fdm_element_order == 0) {
    // Morton (z-order) traversal of the element centroids for the FDM: the
    // face neighbours whose first layers a subdomain reads are processed
    // close in time, so their r values are still in L2
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    std::vector<std::array<double, 3>> cen(ne);
    for (int e = 0; e < ne; ++e) {
      std::array<double, 3> c{0, 0, 0};
      for (int q = 0; q < 8; ++q)
        for (int d = 0; d < 3; ++d) c[d] += 0.125 * mesh.vertices[mesh.elements[e][q]][d];
      cen[e] = c;
      for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], c[d]), hi[d] = std::max(hi[d], c[d]);
    }
    auto spread = [](std::uint64_t v) {  // 21 bits -> every third bit
      v &= 0x1fffff;
      v = (v | v << 32) & 0x1f00000000ffffULL;
      v = (v | v << 16) & 0x1f0000ff0000ffULL;
      v = (v | v << 8) & 0x100f00f00f00f00fULL;
      v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
      v = (v | v << 2) & 0x1249249249249249ULL;
      return v;
    };
    std::vector<std::pair<std::uint64_t, int>> key(ne);
    for (int e = 0; e < ne; ++e) {
      std::uint64_t m = 0;
      for (int d = 0; d < 3; ++d) {
        const double t = hi[d] > lo[d] ? (cen[e][d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
        m |= spread(static_cast<std::uint64_t>(t * 2097151.0)) << d;
      }
      key[e] = {m, e};
    }
    std::sort(key.begin(), key.end());
    std::vector<int> ord(ne);
    for (int e = 0; e < ne; ++e) ord[e] = key[e].second;
    pl.fdm_order = M.upload(ord);
  }
  setup_phase("coarse device");
  // coarse: connectivity, vertex incidence CSR (e, cb) order, coarse matrix, AMG / dense
  if (pl.do_coarse) {
    std::vector<int> conn(static_cast<std::size_t>(ne) * 8);
    for (int e = 0; e < ne; ++e)
      for (int q = 0; q < 8; ++q) conn[8 * static_cast<std::size_t>(e) + q] = mesh.elements[e][q];
    pl.conn = M.upload(conn);
    std::vector<unsigned> off(static_cast<std::size_t>(pl.nv) + 1, 0);
    for (int e = 0; e < ne; ++e)
      for (int cb = 0; cb < 8; ++cb) off[mesh.elements[e][kHexCornerFromBits[cb]] + 1]++;
    for (int v = 0; v < pl.nv; ++v) off[v + 1] += off[v];
    std::vector<int> idx(static_cast<std::size_t>(ne) * 8);
    std::vector<unsigned> cur(off.begin(), off.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int cb = 0; cb < 8; ++cb) idx[cur[mesh.elements[e][kHexCornerFromBits[cb]]]++] = 8 * e + cb;
    pl.vtx_off = M.upload(off);
    pl.vtx_idx = M.upload(idx);
    pl.vmask = M.upload(hs.vmask);
    pl.Rpart = M.alloc<double>(static_cast<std::size_t>(ne) * 8);
    pl.R = M.alloc<double>(pl.nv);
    pl.Z = M.alloc<double>(pl.nv);
    pl.rho = M.alloc<double>(pl.nv);
    pl.dZ = M.alloc<double>(pl.nv);
    pl.Zc = M.alloc<double>(static_cast<std::size_t>(ne) * 8);
    pl.coarse_n = hs.Kc.n;
    if (pl.use_amg) {
      const AmgSetup& amg = hs.amg;
      const int L = static_cast<int>(amg.levels.size());
      pl.lv.resize(L + 1);
      for (int l = 0; l < L; ++l) {
        const AmgLevel& h = amg.levels[l];
        DevLevel& v = pl.lv[l];
        v.n = h.A.n;
        v.nc = h.n_coarse;
        v.A = csr_to_device(pl, h.A);
        v.dinv = M.upload(h.inv_diag);
        v.agg = M.upload(h.aggregate);
        std::vector<int> aptr(static_cast<std::size_t>(v.nc) + 1, 0), amem(v.n);
        for (int i = 0; i < v.n; ++i) aptr[h.aggregate[i] + 1]++;
        for (int c = 0; c < v.nc; ++c) aptr[c + 1] += aptr[c];
        std::vector<int> cur2(aptr.begin(), aptr.end() - 1);
        for (int i = 0; i < v.n; ++i) amem[cur2[h.aggregate[i]]++] = i;
        v.agg_ptr = M.upload(aptr);
        v.agg_mem = M.upload(amem);
        for (double** b : {&v.zA, &v.zB, &v.kr, &v.kz, &v.kp, &v.kf}) *b = M.alloc<double>(v.n);
        v.ks = M.alloc<KScalars>(1);
      }
      pl.lv[L].n = amg.coarsest.n;
      for (int l = 1; l <= L; ++l) {
        pl.lv[l].b = M.alloc<double>(pl.lv[l].n);
        pl.lv[l].x = M.alloc<double>(pl.lv[l].n);
      }
      pl.dense = dense_to_device(pl, amg.coarsest);
      // rho = R - K_c Z reads the same matrix as AMG level 0 (amg.cpp:151-160): share it
      const Csr& A0 = amg.levels.empty() ? hs.Kc : amg.levels[0].A;
      if (!amg.levels.empty() && A0.n == hs.Kc.n && A0.ptr == hs.Kc.ptr && A0.col == hs.Kc.col && A0.val == hs.Kc.val)
        pl.Kc = pl.lv[0].A;
      else
        pl.Kc = csr_to_device(pl, hs.Kc);
    } else {
      pl.dense = dense_to_device(pl, hs.Kc, &mesh.vertices);  // K_c rows are mesh vertices
    }
  }

  setup_phase("vectors + graph");
  // PCG vectors and reduction scratch
  for (double** v : {&pl.u, &pl.r, &pl.z, &pl.p, &pl.f, &pl.b}) {
    *v = M.alloc<double>(pl.N);
    HXB_CUDA(cudaMemset(*v, 0, sizeof(double) * pl.N));
  }
  const int npart = ax_elem_grid(pl) + 64 * pl.num_sms;  // elem-kernel partials + any one-wave grid
  pl.partials = M.alloc<double>(npart);
  pl.ticket = M.alloc<unsigned>(1);
  pl.cpartials = M.alloc<double>(64 * pl.num_sms);
  pl.cticket = M.alloc<unsigned>(1);
  HXB_CUDA(cudaMemset(pl.ticket, 0, sizeof(unsigned)));
  HXB_CUDA(cudaMemset(pl.cticket, 0, sizeof(unsigned)));
  pl.scratch = M.alloc<double>(64);
  pl.res2 = pl.scratch;
  HXB_CUDA(cudaMallocHost(&pl.h_status, 64 * sizeof(double)));
  if (pl.do_coarse) capture_coarse_graph(pl);
  HXB_CUDA(cudaDeviceSynchronize());
  if (opt.bitwise_reference) {  // reference-order arithmetic (compat.cu) over the same device data
    setup_phase("bitwise-reference tables");
    CompatPlan& c = pl.cx;
    c.variant = pl.variant;
    c.wg = pl.wg;
    c.erec = pl.erec;
    c.mass = pl.mass;
    c.c_e = pl.c_e;
    c.kappa_e = pl.kappa_e;
    c.h3 = pl.h3;
    c.mask = pl.mask;
    c.lumped = pl.d_lumped;
    c.fine_pos = pl.fine_pos;
    c.fine_off = pl.fine_off;
    c.zsort = pl.zsort;
    c.conn = pl.conn;
    c.vtx_off = pl.vtx_off;
    c.vtx_idx = pl.vtx_idx;
    c.vmask = pl.vmask;
    compat_init(c, hs);
    pl.bitwise = true;
  }
  setup_phase(nullptr);
  pl.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ensure_hist(Plan& pl, int max_iterations)
{
  if (pl.hist_cap >= max_iterations + 2) return;
  const int cap = max_iterations + 2;
  pl.zr_hist = pl.mem.alloc<double>(cap);
  pl.pf_hist = pl.mem.alloc<double>(cap);
  pl.res_hist = pl.mem.alloc<double>(cap);
  pl.hist_cap = cap;
}

// Mirrors pcg (krylov.cpp:20-71) statement by statement; the vectors never
// leave the device.
void run_pcg(Plan& pl, const hxb_pcg_config& cfg, hxb_pcg_result* res)
{
  if (!(cfg.rel_tolerance > 0) || !(cfg.rel_tolerance < 1))
    throw HxbError(HXB_EINVAL, "pcg: rel_tolerance must lie in (0,1)");
  if (cfg.max_iterations < 1) throw HxbError(HXB_EINVAL, "pcg: max_iterations must be >= 1");
  ensure_hist(pl, cfg.max_iterations);
  cudaStream_t s = pl.s_main;
  const int n = pl.N;
  HXB_CUDA(cudaEventRecord(pl.ev_t0, s));
  pcg_init_kernel<kVecBlock><<<fill_grid(pcg_init_kernel<kVecBlock>, kVecBlock, n), kVecBlock, 0, s>>>(pl.b, pl.r, pl.u, n, dot_args(pl, pl.res2));
  sqrt_store_kernel<<<1, 1, 0, s>>>(pl.res2, pl.res_hist);
  pl.launches += 2;
  HXB_CUDA(cudaMemcpyAsync(pl.h_status, pl.res_hist, sizeof(double), cudaMemcpyDeviceToHost, s));
  HXB_CUDA(cudaStreamSynchronize(s));
  const double r0 = pl.h_status[0];
  int status = HXB_PCG_CONVERGED, iterations = 0;
  std::string diag;
  if (r0 != 0.0) {
    enqueue_precond(pl, nullptr);
    copy_dot_kernel<kVecBlock><<<fill_grid(copy_dot_kernel<kVecBlock>, kVecBlock, n), kVecBlock, 0, s>>>(pl.z, pl.r, pl.p, n, dot_args(pl, pl.zr_hist));
    pl.launches += 1;
    status = HXB_PCG_MAX_ITERATIONS;
    for (int k = 0; k < cfg.max_iterations; ++k) {
      enqueue_ax(pl, pl.p, pl.f, pl.pf_hist + k, s);
      pcg_update_kernel<kVecBlock><<<fill_grid(pcg_update_kernel<kVecBlock>, kVecBlock, n), kVecBlock, 0, s>>>(
          pl.f, pl.r, n, pl.zr_hist, pl.pf_hist, k, dot_args(pl, pl.res2));
      sqrt_store_kernel<<<1, 1, 0, s>>>(pl.res2, pl.res_hist + k + 1);
      pl.launches += 2;
      HXB_CUDA(cudaMemcpyAsync(pl.h_status, pl.pf_hist + k, sizeof(double), cudaMemcpyDeviceToHost, s));
      HXB_CUDA(cudaMemcpyAsync(pl.h_status + 1, pl.res_hist + k + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
      HXB_CUDA(cudaStreamSynchronize(s));
      const double pf = pl.h_status[0], rn = pl.h_status[1];
      if (!(pf > 0)) {
        status = HXB_PCG_BREAKDOWN;
        char buf[160];
        std::snprintf(buf, sizeof(buf), "indefinite operator: p.Ap = %f at iteration %d", pf, k);
        diag = buf;
        iterations = k;
        res->num_zr = k + 1;
        break;
      }
      iterations = k + 1;
      if (rn / r0 <= cfg.rel_tolerance) {
        status = HXB_PCG_CONVERGED;
        pcg_final_kernel<<<fill_grid(pcg_final_kernel, kVecBlock, n), kVecBlock, 0, s>>>(pl.p, pl.u, n, pl.zr_hist, pl.pf_hist, k);
        pl.launches += 1;
        break;
      }
      if (k + 1 == cfg.max_iterations) {
        pcg_final_kernel<<<fill_grid(pcg_final_kernel, kVecBlock, n), kVecBlock, 0, s>>>(pl.p, pl.u, n, pl.zr_hist, pl.pf_hist, k);
        pl.launches += 1;
        diag = "not converged within " + std::to_string(cfg.max_iterations) + " iterations";
        break;
      }
      PcgUArgs ua;
      ua.u = pl.u;
      ua.p = pl.p;
      ua.zr = pl.zr_hist;
      ua.pf = pl.pf_hist;
      ua.k = k;
      if (enqueue_precond(pl, pl.zr_hist + k + 1, &ua))
        pcg_dir_p_kernel<<<fill_grid(pcg_dir_p_kernel, kVecBlock, n), kVecBlock, 0, s>>>(pl.z, pl.p, n, pl.zr_hist, k);
      else
        pcg_dir_kernel<<<fill_grid(pcg_dir_kernel, kVecBlock, n), kVecBlock, 0, s>>>(pl.z, pl.p, pl.u, n, pl.zr_hist,
                                                                                      pl.pf_hist, k);
      pl.launches += 1;
    }
  }
  HXB_CUDA(cudaEventRecord(pl.ev_t1, s));
  HXB_CUDA(cudaEventSynchronize(pl.ev_t1));
  float ms = 0;
  HXB_CUDA(cudaEventElapsedTime(&ms, pl.ev_t0, pl.ev_t1));
  res->solve_seconds = ms / 1000.0;
  res->status = status;
  res->iterations = iterations;
  res->num_residuals = r0 == 0.0 ? 1 : iterations + 1;
  if (status != HXB_PCG_BREAKDOWN) res->num_zr = r0 == 0.0 ? 0 : iterations;
  if (!cfg.record_history) res->num_residuals = res->num_zr = 0;  // empty histories (krylov.cpp:36, 44, 55)
  std::snprintf(res->diagnostic, sizeof(res->diagnostic), "%s", diag.c_str());
  if (cfg.record_history) {
    if (res->residual_history)
      HXB_CUDA(cudaMemcpy(res->residual_history, pl.res_hist, sizeof(double) * res->num_residuals, cudaMemcpyDeviceToHost));
    if (res->zr_history && res->num_zr > 0)
      HXB_CUDA(cudaMemcpy(res->zr_history, pl.zr_hist, sizeof(double) * res->num_zr, cudaMemcpyDeviceToHost));
  }
  if (res->u) HXB_CUDA(cudaMemcpy(res->u, pl.u, sizeof(double) * n, cudaMemcpyDeviceToHost));
}

// Ordering against the caller's stream for the _device entry points. A NULL
// stream is the legacy default stream (torch's default stream has handle 0):
// the plan's non-blocking streams would not otherwise wait for work queued
// there (e.g. an NCCL receive that torch made the default stream wait on), so
// the plan waits on an event recorded on cudaStreamLegacy, and the call
// returns only when its own work is done.
void caller_stream_in(Plan& pl, void* stream)
{
  const cudaStream_t caller = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  HXB_CUDA(cudaEventRecord(pl.ev_a, caller));
  HXB_CUDA(cudaStreamWaitEvent(pl.s_main, pl.ev_a, 0));
}

void caller_stream_out(Plan& pl, void* stream)
{
  HXB_CUDA(cudaGetLastError());
  if (stream) {
    HXB_CUDA(cudaEventRecord(pl.ev_a, pl.s_main));
    HXB_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), pl.ev_a, 0));
  } else {
    HXB_CUDA(cudaStreamSynchronize(pl.s_main));
  }
}

Plan* as_plan(hxb_plan* p)
{
  if (!p) throw HxbError(HXB_EINVAL, "null plan");
  return reinterpret_cast<Plan*>(p);
}

// entry points that act on one device's vectors: not on a multi-GPU handle
Plan* as_device_plan(hxb_plan* p)
{
  Plan* pl = as_plan(p);
  if (pl->group)
    throw HxbError(HXB_EINVAL, "multi-GPU plans take host vectors (hxb_solve, hxb_apply_A); this entry point "
                               "acts on one device's memory");
  return pl;
}


}  // namespace
}  // namespace hxb

// ============================================================================
// Multi-GPU plan (hxb_options.n_gpus > 1): the mesh is cut into
// R contiguous element slabs, slab r on devices[r]. One host thread per GPU
// runs pcg (krylov.cpp:20-71) on its slab; the exchanges of the staged
// hxb_dist_* protocol (interface Ax partials and finals, ghost r, returned
// fine contributions, restriction partials, interface z finals) and the
// scalar all-reduces go over NCCL (ncclSend/ncclRecv/ncclAllReduce/
// ncclAllGather on the plan's stream, NVLink between the GPUs of one box) or,
// when ranks share a device, over device-to-device copies ordered by events.
// Scalars stay on the device: alpha and beta are formed by the vector
// kernels from device history arrays, so the only host read per iteration
// is the convergence check (rn, p.Ap), as in the single-GPU loop.
namespace hxb {

namespace {

// barrier for the rank threads; abort() releases everyone with an error
class RankBarrier {
 public:
  explicit RankBarrier(int n) : n_(n) {}
  void wait()
  {
    std::unique_lock<std::mutex> lk(m_);
    if (aborted_) throw HxbError(HXB_ECUDA, "multi-GPU solve aborted by another rank");
    const long long gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return gen_ != gen || aborted_; });
    if (aborted_) throw HxbError(HXB_ECUDA, "multi-GPU solve aborted by another rank");
  }
  void abort()
  {
    std::lock_guard<std::mutex> lk(m_);
    aborted_ = true;
    cv_.notify_all();
  }
  void reset()
  {
    std::lock_guard<std::mutex> lk(m_);
    aborted_ = false;
    count_ = 0;
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_, count_ = 0;
  long long gen_ = 0;
  bool aborted_ = false;
};

// NCCL is resolved at run time (dlopen), only when a multi-GPU plan with
// distinct devices is built: an NCCL already loaded into the process (e.g.
// torch's) is reused, and merely loading libhexsem_b200.so never pulls a
// second libnccl into a process that has its own.
struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api()
{
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto get = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp && err.empty()) err = std::string("NCCL symbol missing: ") + name;
    };
    get(api.CommInitAll, "ncclCommInitAll");
    get(api.CommDestroy, "ncclCommDestroy");
    get(api.GroupStart, "ncclGroupStart");
    get(api.GroupEnd, "ncclGroupEnd");
    get(api.Send, "ncclSend");
    get(api.Recv, "ncclRecv");
    get(api.AllReduce, "ncclAllReduce");
    get(api.AllGather, "ncclAllGather");
    get(api.GetErrorString, "ncclGetErrorString");
  });
  if (!err.empty()) throw HxbError(HXB_ENCCL, err);
  return api;
}

#define HXB_NCCL(call)                                                                              \
  do {                                                                                              \
    ncclResult_t res__ = (call);                                                                    \
    if (res__ != ncclSuccess) throw HxbError(HXB_ENCCL, std::string(#call) + ": " + nccl_api().GetErrorString(res__)); \
  } while (0)

struct RankBuf {
  double *send_up = nullptr, *recv_down = nullptr, *send_down = nullptr, *recv_up = nullptr;
  double *gsend_down = nullptr, *gsend_up = nullptr, *grecv_down = nullptr, *grecv_up = nullptr;
  double *fsend = nullptr, *frecv = nullptr, *zsend_down = nullptr, *zrecv_up = nullptr;
  double* gather = nullptr;  // NCCL all-gather of the restriction partials: R slabs of `cap`
  double* scal = nullptr;    // [0] r.r [1] z.r [2] p.f partials, [4, 4+R) pulled partials, [32] r.r sum
  double *hist_zr = nullptr, *hist_pf = nullptr;
  double* outbuf = nullptr;  // finalised surface values for the host
  double* h_scal = nullptr;  // pinned
  int hist_cap = 0;
  std::vector<int> fin_surf;  // host copy: finalised surface nodes of this rank
};

struct Mail {  // local transport: what each rank offers in the current exchange
  const double* down = nullptr;  // to rank r-1
  const double* up = nullptr;    // to rank r+1
  const double* scalar = nullptr;
};

}  // namespace

struct Group {
  int R = 0;
  std::vector<int> dev;
  std::vector<std::unique_ptr<Plan>> pl;
  std::vector<RankBuf> buf;
  bool nccl = false;
  std::vector<ncclComm_t> comm;
  std::unique_ptr<RankBarrier> bar;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<Mail> mail;
  int cap = 0;  // padded restriction slab (doubles)
  ~Group()
  {
    for (int r = 0; r < static_cast<int>(pl.size()); ++r) {
      cudaSetDevice(dev[r]);
      cudaDeviceSynchronize();
      if (r < static_cast<int>(ev_ready.size()) && ev_ready[r]) cudaEventDestroy(ev_ready[r]);
      if (r < static_cast<int>(ev_done.size()) && ev_done[r]) cudaEventDestroy(ev_done[r]);
      if (r < static_cast<int>(buf.size()) && buf[r].h_scal) cudaFreeHost(buf[r].h_scal);
    }
    for (ncclComm_t c : comm)
      if (c) nccl_api().CommDestroy(c);
  }
};

void destroy_group(Group* g) { delete g; }

// the host setup behind a plan (a multi-GPU handle's ranks share rank 0's)
const HostSetup& plan_hs(Plan* pl) { return pl->group ? pl->group->pl[0]->hs : pl->hs; }

// host copy of the lumped mass: single-device plans assemble it on the device
// and copy it back on first use (3 GB at cfg5, not needed by a device solve)
const std::vector<double>& host_lumped(Plan* pl)
{
  if (pl->group) return pl->group->pl[0]->hs.lumped;
  HostSetup& hs = pl->hs;
  if (hs.lumped.empty() && pl->N > 0) {
    if (!pl->d_lumped) throw HxbError(HXB_EINVAL, "plan has no lumped mass");
    HXB_CUDA(cudaSetDevice(pl->device));
    hs.lumped.resize(pl->N);
    HXB_CUDA(cudaMemcpy(hs.lumped.data(), pl->d_lumped, sizeof(double) * pl->N, cudaMemcpyDeviceToHost));
  }
  return hs.lumped;
}

namespace {

// ---- transport ---------------------------------------------------------------
// exchange with the neighbours: to_down/to_up go to ranks r-1/r+1, from_down/
// from_up arrive from them (counts pair up by construction of the lists)
void g_exchange(Group& G, int r, const double* to_down, int n_to_down, const double* to_up, int n_to_up,
                double* from_down, int n_from_down, double* from_up, int n_from_up)
{
  Plan& P = *G.pl[r];
  cudaStream_t s = P.s_main;
  if (G.nccl) {
    HXB_NCCL(nccl_api().GroupStart());
    if (r > 0) {
      if (n_to_down) HXB_NCCL(nccl_api().Send(to_down, n_to_down, ncclDouble, r - 1, G.comm[r], s));
      if (n_from_down) HXB_NCCL(nccl_api().Recv(from_down, n_from_down, ncclDouble, r - 1, G.comm[r], s));
    }
    if (r + 1 < G.R) {
      if (n_to_up) HXB_NCCL(nccl_api().Send(to_up, n_to_up, ncclDouble, r + 1, G.comm[r], s));
      if (n_from_up) HXB_NCCL(nccl_api().Recv(from_up, n_from_up, ncclDouble, r + 1, G.comm[r], s));
    }
    HXB_NCCL(nccl_api().GroupEnd());
    return;
  }
  // pull model: after everyone's sends are ready, each rank copies what it receives
  G.mail[r].down = to_down;
  G.mail[r].up = to_up;
  HXB_CUDA(cudaEventRecord(G.ev_ready[r], s));
  G.bar->wait();
  if (r > 0 && n_from_down) {
    HXB_CUDA(cudaStreamWaitEvent(s, G.ev_ready[r - 1], 0));
    HXB_CUDA(cudaMemcpyPeerAsync(from_down, G.dev[r], G.mail[r - 1].up, G.dev[r - 1], sizeof(double) * n_from_down, s));
  }
  if (r + 1 < G.R && n_from_up) {
    HXB_CUDA(cudaStreamWaitEvent(s, G.ev_ready[r + 1], 0));
    HXB_CUDA(cudaMemcpyPeerAsync(from_up, G.dev[r], G.mail[r + 1].down, G.dev[r + 1], sizeof(double) * n_from_up, s));
  }
  HXB_CUDA(cudaEventRecord(G.ev_done[r], s));
  G.bar->wait();
  if (r > 0) HXB_CUDA(cudaStreamWaitEvent(s, G.ev_done[r - 1], 0));
  if (r + 1 < G.R) HXB_CUDA(cudaStreamWaitEvent(s, G.ev_done[r + 1], 0));
}

// *sum = sum over ranks of *partial (device scalars; identical on every rank)
void g_allreduce(Group& G, int r, const double* partial, double* sum)
{
  Plan& P = *G.pl[r];
  cudaStream_t s = P.s_main;
  if (G.nccl) {
    HXB_NCCL(nccl_api().AllReduce(partial, sum, 1, ncclDouble, ncclSum, G.comm[r], s));
    return;
  }
  G.mail[r].scalar = partial;
  HXB_CUDA(cudaEventRecord(G.ev_ready[r], s));
  G.bar->wait();
  double* parts = G.buf[r].scal + 4;
  for (int q = 0; q < G.R; ++q) {
    HXB_CUDA(cudaStreamWaitEvent(s, G.ev_ready[q], 0));
    HXB_CUDA(cudaMemcpyPeerAsync(parts + q, G.dev[r], G.mail[q].scalar, G.dev[q], sizeof(double), s));
  }
  sum_partials_kernel<<<1, 32, 0, s>>>(parts, G.R, sum);
  P.launches += 1;
  HXB_CUDA(cudaEventRecord(G.ev_done[r], s));
  G.bar->wait();
  for (int q = 0; q < G.R; ++q) HXB_CUDA(cudaStreamWaitEvent(s, G.ev_done[q], 0));
}

// every rank's restriction partials (its slab of Rpart) into every rank's full Rpart
void g_allgather_rpart(Group& G, int r)
{
  Plan& P = *G.pl[r];
  cudaStream_t s = P.s_main;
  if (G.nccl) {
    double* mine = G.buf[r].gather + static_cast<std::size_t>(r) * G.cap;
    HXB_CUDA(cudaMemcpyAsync(mine, P.Rpart + 8LL * P.e0, sizeof(double) * 8 * P.ne, cudaMemcpyDeviceToDevice, s));
    HXB_NCCL(nccl_api().AllGather(mine, G.buf[r].gather, G.cap, ncclDouble, G.comm[r], s));
    for (int q = 0; q < G.R; ++q)
      if (q != r)
        HXB_CUDA(cudaMemcpyAsync(P.Rpart + 8LL * G.pl[q]->e0, G.buf[r].gather + static_cast<std::size_t>(q) * G.cap,
                                 sizeof(double) * 8 * G.pl[q]->ne, cudaMemcpyDeviceToDevice, s));
    return;
  }
  HXB_CUDA(cudaEventRecord(G.ev_ready[r], s));
  G.bar->wait();
  for (int q = 0; q < G.R; ++q)
    if (q != r) {
      const Plan& Q = *G.pl[q];
      HXB_CUDA(cudaStreamWaitEvent(s, G.ev_ready[q], 0));
      HXB_CUDA(cudaMemcpyPeerAsync(P.Rpart + 8LL * Q.e0, G.dev[r], Q.Rpart + 8LL * Q.e0, G.dev[q],
                                   sizeof(double) * 8 * Q.ne, s));
    }
  HXB_CUDA(cudaEventRecord(G.ev_done[r], s));
  G.bar->wait();
  for (int q = 0; q < G.R; ++q) HXB_CUDA(cudaStreamWaitEvent(s, G.ev_done[q], 0));
}

// ---- the staged steps (bodies of hxb_dist_*) on the plan's stream -----------
void r_vec(Plan& P, int mode, const double* x0, const double* x1, double* y0, double* y1, const double* num = nullptr,
           const double* den = nullptr)
{
  const int total = P.n_loc_surf + (P.ib1 - P.ib0);
  dist_vec_kernel<<<fill_grid(dist_vec_kernel, kVecBlock, total), kVecBlock, 0, P.s_main>>>(
      mode, P.loc_list, P.n_loc_surf, P.ib0, P.ib1, 0.0, x0, x1, y0, y1, num, den);
  P.launches += 1;
}

void r_dot(Plan& P, const double* x, const double* y, double* out)
{
  const int total = P.n_fin_surf + (P.ib1 - P.ib0);
  dist_dot_kernel<kVecBlock><<<fill_grid(dist_dot_kernel<kVecBlock>, kVecBlock, total), kVecBlock, 0, P.s_main>>>(
      P.fin_surf, P.n_fin_surf, P.ib0, P.ib1, x, y, dot_args(P, out));
  P.launches += 1;
}

void r_pack(Plan& P, const int* list, int n, const double* x, double* buf)
{
  if (n) dist_pack_kernel<<<vec_grid(n), kVecBlock, 0, P.s_main>>>(list, n, x, buf), P.launches += 1;
}

void r_unpack(Plan& P, const int* list, int n, const double* buf, double* x)
{
  if (n) dist_unpack_kernel<<<vec_grid(n), kVecBlock, 0, P.s_main>>>(list, n, buf, x), P.launches += 1;
}

// f = A p over the slabs (hxb_dist_apply_A_begin/_continue/_end)
void g_apply_A(Group& G, int r, const double* p, double* f)
{
  Plan& P = *G.pl[r];
  RankBuf& B = G.buf[r];
  cudaStream_t s = P.s_main;
  enqueue_ax(P, p, f, nullptr, s);
  if (P.n_up) {
    dist_partial_kernel<<<vec_grid(P.n_up), kVecBlock, 0, s>>>(P.ax_off + P.n_grp0, P.ax_idx, P.rsurf, P.n_up, B.send_up);
    P.launches += 1;
  }
  g_exchange(G, r, nullptr, 0, B.send_up, P.n_up, B.recv_down, P.n_down, nullptr, 0);
  if (P.n_down) {
    const int t0 = P.n_grp0 + P.n_up;
    dist_continue_kernel<<<vec_grid(P.n_down), kVecBlock, 0, s>>>(P.ax_off + t0, P.ax_idx, P.rsurf, P.ax_nodes + t0,
                                                                  P.n_down, p, P.mask, B.recv_down, f, B.send_down);
    P.launches += 1;
  }
  g_exchange(G, r, B.send_down, P.n_down, nullptr, 0, nullptr, 0, B.recv_up, P.n_up);
  if (P.n_up) {
    dist_finish_kernel<<<vec_grid(P.n_up), kVecBlock, 0, s>>>(P.ax_nodes + P.n_grp0, P.n_up, B.recv_up, f);
    P.launches += 1;
  }
}

// z = P r over the slabs (precond.cpp:27-67); *zr = global z.r on every rank
void g_precond(Group& G, int r, double* zr)
{
  Plan& P = *G.pl[r];
  RankBuf& B = G.buf[r];
  cudaStream_t s = P.s_main;
  if (!P.do_fine) {  // PrecondMode::none: z = r
    r_vec(P, 3, P.r, nullptr, P.z, nullptr);
    r_dot(P, P.z, P.r, B.scal + 1);
    g_allreduce(G, r, B.scal + 1, zr);
    return;
  }
  r_pack(P, P.g_to_down, P.n_g_to_down, P.r, B.gsend_down);
  r_pack(P, P.g_to_up, P.n_g_to_up, P.r, B.gsend_up);
  g_exchange(G, r, B.gsend_down, P.n_g_to_down, B.gsend_up, P.n_g_to_up, B.grecv_down, P.n_g_from_down, B.grecv_up,
             P.n_g_from_up);
  r_unpack(P, P.g_from_down, P.n_g_from_down, B.grecv_down, P.r);
  r_unpack(P, P.g_from_up, P.n_g_from_up, B.grecv_up, P.r);
  P.fsend = B.fsend;
  HXB_DISPATCH_NP(P.np, launch_fdm, P, s);
  P.fsend = nullptr;
  g_exchange(G, r, B.fsend, P.n_fsend_down, B.fsend + P.n_fsend_down, P.n_fsend_up, B.frecv, P.n_frecv_down,
             B.frecv + P.n_frecv_down, P.n_frecv_up);
  const int nrecv = P.n_frecv_down + P.n_frecv_up;
  if (nrecv) {
    dist_fine_scatter_kernel<<<vec_grid(nrecv), kVecBlock, 0, s>>>(P.frecv_pos, nrecv, B.frecv, P.zsort);
    P.launches += 1;
  }
  g_allgather_rpart(G, r);
  HXB_CUDA(cudaGraphLaunch(P.coarse_exec, s));  // replicated coarse solve: identical on every rank
  P.launches += P.coarse_graph_nodes;
  launch_combine(P, B.scal + 1, s, P.do_fine, P.do_coarse);
  g_allreduce(G, r, B.scal + 1, zr);
  // finals of the down-interface nodes to the lower rank
  r_pack(P, P.ax_nodes + P.n_grp0 + P.n_up, P.n_down, P.z, B.zsend_down);
  g_exchange(G, r, B.zsend_down, P.n_down, nullptr, 0, nullptr, 0, B.zrecv_up, P.n_up);
  r_unpack(P, P.ax_nodes + P.n_grp0, P.n_up, B.zrecv_up, P.z);
}

// this rank's finalised values of x (surface list + owned interior range) into host y
void g_output(Group& G, int r, const double* x, double* y)
{
  Plan& P = *G.pl[r];
  RankBuf& B = G.buf[r];
  cudaStream_t s = P.s_main;
  r_pack(P, P.fin_surf, P.n_fin_surf, x, B.outbuf);
  std::vector<double> surf(P.n_fin_surf);
  if (P.n_fin_surf)
    HXB_CUDA(cudaMemcpyAsync(surf.data(), B.outbuf, sizeof(double) * P.n_fin_surf, cudaMemcpyDeviceToHost, s));
  if (P.ib1 > P.ib0)
    HXB_CUDA(cudaMemcpyAsync(y + P.ib0, x + P.ib0, sizeof(double) * (P.ib1 - P.ib0), cudaMemcpyDeviceToHost, s));
  HXB_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < P.n_fin_surf; ++q) y[B.fin_surf[q]] = surf[q];
}

struct RankResult {
  int status = HXB_PCG_CONVERGED, iterations = 0;
  std::vector<double> res_hist, zr_hist;
  std::string diag;
  double solve_seconds = 0;
};

// pcg (krylov.cpp:20-71) on rank r; b already in P.b
void g_rank_pcg(Group& G, int r, const hxb_pcg_config& cfg, RankResult& out)
{
  Plan& P = *G.pl[r];
  RankBuf& B = G.buf[r];
  HXB_CUDA(cudaSetDevice(P.device));
  cudaStream_t s = P.s_main;
  if (B.hist_cap < cfg.max_iterations + 2) {
    B.hist_cap = cfg.max_iterations + 2;
    B.hist_zr = P.mem.alloc<double>(B.hist_cap);
    B.hist_pf = P.mem.alloc<double>(B.hist_cap);
  }
  HXB_CUDA(cudaEventRecord(P.ev_t0, s));
  r_vec(P, 0, P.b, nullptr, P.r, P.u);  // r = b, u = 0
  r_dot(P, P.r, P.r, B.scal + 0);
  g_allreduce(G, r, B.scal + 0, B.scal + 32);
  HXB_CUDA(cudaMemcpyAsync(B.h_scal, B.scal + 32, sizeof(double), cudaMemcpyDeviceToHost, s));
  HXB_CUDA(cudaStreamSynchronize(s));
  const double r0 = std::sqrt(B.h_scal[0]);
  out.res_hist.push_back(r0);
  out.status = HXB_PCG_CONVERGED;
  int k = 0;
  if (r0 != 0.0) {
    g_precond(G, r, B.hist_zr + 0);
    r_vec(P, 3, P.z, nullptr, P.p, nullptr);  // p = z
    out.status = HXB_PCG_MAX_ITERATIONS;
    for (k = 0; k < cfg.max_iterations; ++k) {
      g_apply_A(G, r, P.p, P.f);
      r_dot(P, P.p, P.f, B.scal + 2);
      g_allreduce(G, r, B.scal + 2, B.hist_pf + k);
      r_vec(P, 1, P.p, P.f, P.r, P.u, B.hist_zr + k, B.hist_pf + k);  // u += alpha p, r -= alpha f
      r_dot(P, P.r, P.r, B.scal + 0);
      g_allreduce(G, r, B.scal + 0, B.scal + 32);
      HXB_CUDA(cudaMemcpyAsync(B.h_scal, B.hist_pf + k, sizeof(double), cudaMemcpyDeviceToHost, s));
      HXB_CUDA(cudaMemcpyAsync(B.h_scal + 1, B.scal + 32, sizeof(double), cudaMemcpyDeviceToHost, s));
      HXB_CUDA(cudaStreamSynchronize(s));  // the one host read per iteration (convergence)
      const double pf = B.h_scal[0], rn = std::sqrt(B.h_scal[1]);
      if (!(pf > 0)) {
        out.status = HXB_PCG_BREAKDOWN;
        char msg[160];
        std::snprintf(msg, sizeof(msg), "indefinite operator: p.Ap = %f at iteration %d", pf, k);
        out.diag = msg;
        out.iterations = k;
        ++k;  // zr_k was recorded
        break;
      }
      out.iterations = k + 1;
      out.res_hist.push_back(rn);
      if (rn / r0 <= cfg.rel_tolerance) {
        out.status = HXB_PCG_CONVERGED;
        ++k;
        break;
      }
      if (k + 1 == cfg.max_iterations) {
        out.diag = "not converged within " + std::to_string(cfg.max_iterations) + " iterations";
        ++k;
        break;
      }
      g_precond(G, r, B.hist_zr + k + 1);
      r_vec(P, 2, P.z, nullptr, P.p, nullptr, B.hist_zr + k + 1, B.hist_zr + k);  // p = z + beta p
    }
  }
  HXB_CUDA(cudaEventRecord(P.ev_t1, s));
  HXB_CUDA(cudaEventSynchronize(P.ev_t1));
  float ms = 0;
  HXB_CUDA(cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1));
  out.solve_seconds = ms / 1000.0;
  const int nzr = r0 == 0.0 ? 0 : k;
  out.zr_hist.resize(nzr);
  if (nzr) HXB_CUDA(cudaMemcpy(out.zr_hist.data(), B.hist_zr, sizeof(double) * nzr, cudaMemcpyDeviceToHost));
}

// run fn(r) on one host thread per rank; the first error is rethrown
template <class F>
void g_run(Group& G, F&& fn)
{
  G.bar->reset();
  std::vector<std::exception_ptr> err(G.R);
  std::vector<std::thread> th;
  for (int r = 0; r < G.R; ++r)
    th.emplace_back([&, r] {
      try {
        HXB_CUDA(cudaSetDevice(G.dev[r]));
        fn(r);
      } catch (...) {
        err[r] = std::current_exception();
        G.bar->abort();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

void build_group(Plan& top, const hxb_mesh* m, int order, const double* kappa_e, const double* c_e,
                 const hxb_options& opt)
{
  const int R = opt.n_gpus;
  if (R < 2 || R > HXB_MAX_GPUS) throw HxbError(HXB_EINVAL, "n_gpus must lie in 2..8");
  if (!m || m->num_elements < R) throw HxbError(HXB_EINVAL, "more GPUs than elements");
  if (opt.nranks > 1) throw HxbError(HXB_EINVAL, "n_gpus and the staged rank/nranks are exclusive");
  if (opt.precond_mode != HXB_PRECOND_NONE && opt.precond_mode != HXB_PRECOND_TWO_SCALE)
    throw HxbError(HXB_EINVAL, "multi-GPU plans support precond_mode two_scale or none");
  int ndev = 0;
  HXB_CUDA(cudaGetDeviceCount(&ndev));
  auto G = std::make_unique<Group>();
  G->R = R;
  for (int r = 0; r < R; ++r) {
    if (opt.devices[r] < 0 || opt.devices[r] >= ndev) throw HxbError(HXB_EINVAL, "device ordinal out of range");
    G->dev.push_back(opt.devices[r]);
  }
  // rank 0 builds the host setup (numbering, coarse matrix, AMG) once; the
  // other ranks share it read-only and build their device slabs one after the
  // other (their graph captures must not overlap another thread's setup calls
  // on a shared device)
  auto rank_opt = [&](int r) {
    hxb_options o = opt;
    o.n_gpus = 1;
    o.rank = r;
    o.nranks = R;
    o.device = G->dev[r];
    return o;
  };
  G->pl.resize(R);
  {
    const hxb_options o = rank_opt(0);
    G->pl[0] = std::make_unique<Plan>();
    build_plan(*G->pl[0], m, order, kappa_e, c_e, o);
  }
  std::shared_ptr<HostSetup> hs = G->pl[0]->hsp;
  for (int r = 1; r < R; ++r) {
    const hxb_options o = rank_opt(r);
    G->pl[r] = std::make_unique<Plan>(hs);
    build_plan(*G->pl[r], m, order, kappa_e, c_e, o);
  }
  // exchange buffers, events
  int max_ne = 0;
  for (int r = 0; r < R; ++r) max_ne = std::max(max_ne, G->pl[r]->ne);
  G->cap = 8 * max_ne;
  bool distinct = true;
  for (int r = 0; r < R; ++r)
    for (int q = 0; q < r; ++q) distinct = distinct && G->dev[r] != G->dev[q];
  const char* tr = std::getenv("HXB_GROUP_TRANSPORT");
  G->nccl = distinct && !(tr && std::string(tr) == "local");
  G->buf.resize(R);
  G->ev_ready.assign(R, nullptr);
  G->ev_done.assign(R, nullptr);
  G->mail.resize(R);
  for (int r = 0; r < R; ++r) {
    Plan& P = *G->pl[r];
    RankBuf& B = G->buf[r];
    HXB_CUDA(cudaSetDevice(P.device));
    DeviceArena& M = P.mem;
    B.send_up = M.alloc<double>(P.n_up);
    B.recv_up = M.alloc<double>(P.n_up);
    B.zrecv_up = M.alloc<double>(P.n_up);
    B.send_down = M.alloc<double>(P.n_down);
    B.recv_down = M.alloc<double>(P.n_down);
    B.zsend_down = M.alloc<double>(P.n_down);
    B.gsend_down = M.alloc<double>(P.n_g_to_down);
    B.gsend_up = M.alloc<double>(P.n_g_to_up);
    B.grecv_down = M.alloc<double>(P.n_g_from_down);
    B.grecv_up = M.alloc<double>(P.n_g_from_up);
    B.fsend = M.alloc<double>(P.n_fsend_down + P.n_fsend_up);
    B.frecv = M.alloc<double>(P.n_frecv_down + P.n_frecv_up);
    B.scal = M.alloc<double>(64);
    HXB_CUDA(cudaMemset(B.scal, 0, 64 * sizeof(double)));
    B.outbuf = M.alloc<double>(P.n_fin_surf);
    if (G->nccl && P.do_coarse) B.gather = M.alloc<double>(static_cast<std::size_t>(R) * G->cap);
    HXB_CUDA(cudaMallocHost(&B.h_scal, 8 * sizeof(double)));
    B.fin_surf.resize(P.n_fin_surf);
    if (P.n_fin_surf)
      HXB_CUDA(cudaMemcpy(B.fin_surf.data(), P.fin_surf, sizeof(int) * P.n_fin_surf, cudaMemcpyDeviceToHost));
    HXB_CUDA(cudaEventCreateWithFlags(&G->ev_ready[r], cudaEventDisableTiming));
    HXB_CUDA(cudaEventCreateWithFlags(&G->ev_done[r], cudaEventDisableTiming));
    for (int q = 0; q < R; ++q)  // direct NVLink copies between distinct devices where possible
      if (G->dev[q] != P.device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, P.device, G->dev[q]);
        if (ok && cudaDeviceEnablePeerAccess(G->dev[q], 0) != cudaSuccess) cudaGetLastError();
      }
  }
  if (G->nccl) {
    G->comm.assign(R, nullptr);
    HXB_NCCL(nccl_api().CommInitAll(G->comm.data(), R, G->dev.data()));
  }
  G->bar = std::make_unique<RankBarrier>(R);
  for (int r = 0; r < R; ++r) HXB_CUDA(cudaDeviceSynchronize());
  // the handle: whole-mesh facts for hxb_plan_get_info
  Plan& P0 = *G->pl[0];
  top.device = G->dev[0];
  top.order = P0.order;
  top.np = P0.np;
  top.nloc = P0.nloc;
  top.N = P0.N;
  top.ne = P0.ne_total;
  top.ne_total = P0.ne_total;
  top.nv = P0.nv;
  top.use_amg = P0.use_amg;
  top.coarse_n = P0.coarse_n;
  top.precond_mode = P0.precond_mode;
  top.do_fine = P0.do_fine;
  top.do_coarse = P0.do_coarse;
  top.nranks = R;
  for (int r = 0; r < R; ++r) top.setup_seconds = std::max(top.setup_seconds, G->pl[r]->setup_seconds);
  top.group = G.release();
}

// hxb_solve on a multi-GPU plan: b (host, or NULL for the Poisson load) -> res
void group_solve(Plan& top, const double* b, const hxb_pcg_config& cfg, hxb_pcg_result* res)
{
  if (!(cfg.rel_tolerance > 0) || !(cfg.rel_tolerance < 1))
    throw HxbError(HXB_EINVAL, "pcg: rel_tolerance must lie in (0,1)");
  if (cfg.max_iterations < 1) throw HxbError(HXB_EINVAL, "pcg: max_iterations must be >= 1");
  Group& G = *top.group;
  const HostSetup& hs = G.pl[0]->hs;
  const int N = top.N;
  std::vector<double> bdef;
  if (!b) {
    bdef.resize(N);
    for (int g = 0; g < N; ++g) bdef[g] = hs.num.dirichlet_mask[g] ? 0.0 : hs.lumped[g] * 1.0;
    b = bdef.data();
  }
  std::vector<RankResult> out(G.R);
  const auto t0 = std::chrono::steady_clock::now();
  g_run(G, [&](int r) {
    Plan& P = *G.pl[r];
    HXB_CUDA(cudaMemcpyAsync(P.b, b, sizeof(double) * N, cudaMemcpyHostToDevice, P.s_main));
    g_rank_pcg(G, r, cfg, out[r]);
    if (res->u) g_output(G, r, P.u, res->u);
  });
  (void)t0;
  const RankResult& o = out[0];
  double secs = 0;
  for (const RankResult& q : out) secs = std::max(secs, q.solve_seconds);
  res->status = o.status;
  res->iterations = o.iterations;
  res->solve_seconds = secs;
  res->num_residuals = cfg.record_history ? static_cast<int>(o.res_hist.size()) : 0;
  res->num_zr = cfg.record_history ? static_cast<int>(o.zr_hist.size()) : 0;
  if (cfg.record_history) {
    if (res->residual_history) std::memcpy(res->residual_history, o.res_hist.data(), sizeof(double) * o.res_hist.size());
    if (res->zr_history && !o.zr_hist.empty())
      std::memcpy(res->zr_history, o.zr_hist.data(), sizeof(double) * o.zr_hist.size());
  }
  std::snprintf(res->diagnostic, sizeof(res->diagnostic), "%s", o.diag.c_str());
}

// hxb_apply_P on a multi-GPU plan (host vectors, TwoScalePreconditioner::apply)
void group_apply_P(Plan& top, const double* rin, double* z_out)
{
  Group& G = *top.group;
  const int N = top.N;
  g_run(G, [&](int r) {
    Plan& P = *G.pl[r];
    HXB_CUDA(cudaMemcpyAsync(P.r, rin, sizeof(double) * N, cudaMemcpyHostToDevice, P.s_main));
    g_precond(G, r, G.buf[r].scal + 33);
    g_output(G, r, P.z, z_out);
  });
}

// hxb_apply_A on a multi-GPU plan (host vectors)
void group_apply_A(Plan& top, const double* u, double* r_out)
{
  Group& G = *top.group;
  const int N = top.N;
  g_run(G, [&](int r) {
    Plan& P = *G.pl[r];
    HXB_CUDA(cudaMemcpyAsync(P.p, u, sizeof(double) * N, cudaMemcpyHostToDevice, P.s_main));
    g_apply_A(G, r, P.p, P.f);
    g_output(G, r, P.f, r_out);
  });
}

}  // namespace
}  // namespace hxb


using namespace hxb;

extern "C" {

int hxb_plan_create(const hxb_mesh* mesh, int order, const double* kappa_e, const double* c_e, const hxb_options* opt,
                    hxb_plan** out)
{
  return guarded([&] {
    if (!out) throw HxbError(HXB_EINVAL, "null output");
    if (!kappa_e || !c_e) throw HxbError(HXB_EINVAL, "kappa/c must hold one value per element");
    hxb_options o;
    if (opt)
      o = *opt;
    else
      hxb_default_options(&o);
    auto pl = std::make_unique<Plan>();
    if (o.n_gpus > 1)
      build_group(*pl, mesh, order, kappa_e, c_e, o);
    else
      build_plan(*pl, mesh, order, kappa_e, c_e, o);
    *out = reinterpret_cast<hxb_plan*>(pl.release());
  });
}

int hxb_plan_destroy(hxb_plan* plan)
{
  return guarded([&] {
    if (plan) {
      Plan* pl = as_plan(plan);
      cudaSetDevice(pl->device);
      cudaDeviceSynchronize();
      delete pl;
    }
  });
}

int hxb_plan_get_info(const hxb_plan* plan, hxb_plan_info* info)
{
  return guarded([&] {
    const Plan* pl = reinterpret_cast<const Plan*>(plan);
    if (!pl || !info) throw HxbError(HXB_EINVAL, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->num_global = pl->N;
    info->num_elements = pl->ne;
    info->num_vertices = pl->nv;
    info->order = pl->order;
    info->coarse_uses_amg = pl->use_amg ? 1 : 0;
    info->coarse_n = pl->coarse_n;
    info->precond_mode = pl->precond_mode;
    fill_amg_info(pl->group ? pl->group->pl[0]->hs : pl->hs, &info->amg_levels, info->amg_rows, info->amg_nnz);
    info->setup_seconds = pl->setup_seconds;
    info->device_bytes = static_cast<int64_t>(pl->mem.bytes);
    info->coarse_sms = pl->coarse_sms;
    if (pl->group)
      for (const auto& q : pl->group->pl) info->device_bytes += static_cast<int64_t>(q->mem.bytes);
  });
}

int hxb_apply_A_device(hxb_plan* plan, const double* d_u, double* d_r, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (pl->nranks > 1) throw HxbError(HXB_EINVAL, "distributed plans: use hxb_dist_apply_A_*");
    HXB_CUDA(cudaSetDevice(pl->device));
    caller_stream_in(*pl, stream);
    if (pl->bitwise)
      compat_apply_A(pl->cx, d_u, d_r, pl->s_main);
    else
      enqueue_ax(*pl, d_u, d_r, nullptr, pl->s_main);
    caller_stream_out(*pl, stream);
  });
}

// Host-pointer Ax (SemOperator::apply on host spans) as a copy/compute
// pipeline: element-interior values belong to one element each and are
// contiguous per element range, so after the surface part of u is on the
// device, chunk c's interior u (H2D stream), chunk c's element kernel (main
// stream) and chunk c-1's interior r (D2H stream) run concurrently; the
// surface gather and its D2H close the apply. PCIe is full duplex, so the
// in- and outbound copies overlap each other and the compute.
int hxb_apply_A(hxb_plan* plan, const double* u, double* r)
{
  return guarded([&] {
    Plan* pl = as_plan(plan);
    if (!u || !r) throw HxbError(HXB_EINVAL, "null argument");
    if (pl->group) {
      group_apply_A(*pl, u, r);
      return;
    }
    if (pl->nranks > 1) throw HxbError(HXB_EINVAL, "distributed plans: use hxb_dist_apply_A_*");
    HXB_CUDA(cudaSetDevice(pl->device));
    Plan& P = *pl;
    if (P.bitwise) {  // verification mode: plain copies around the reference-order operator
      HXB_CUDA(cudaMemcpyAsync(P.p, u, sizeof(double) * P.N, cudaMemcpyHostToDevice, P.s_main));
      compat_apply_A(P.cx, P.p, P.f, P.s_main);
      HXB_CUDA(cudaMemcpyAsync(r, P.f, sizeof(double) * P.N, cudaMemcpyDeviceToHost, P.s_main));
      HXB_CUDA(cudaStreamSynchronize(P.s_main));
      return;
    }
    constexpr int C = 8;  // measured at cfg2: 8 chunks 10.5 ms, 16 10.8 ms, 32 11.1 ms
    if (!P.s_in) {
      HXB_CUDA(cudaStreamCreateWithFlags(&P.s_in, cudaStreamNonBlocking));
      HXB_CUDA(cudaStreamCreateWithFlags(&P.s_out, cudaStreamNonBlocking));
      P.pipe_ev.resize(2 * C + 2);
      for (cudaEvent_t& e : P.pipe_ev) HXB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const long long NI = static_cast<long long>(P.order - 1) * (P.order - 1) * (P.order - 1);
    const std::size_t sbytes = sizeof(double) * P.nsg;
    cudaEvent_t ev_surf = P.pipe_ev[2 * C], ev_done = P.pipe_ev[2 * C + 1];
    if (!P.runs_ready) {  // surface nodes as id runs of equal first/last element chunk
      P.runs_ready = true;
      const int nsr = surface_slot_count(P.np);
      std::vector<int> lo(P.nsg, C), hi(P.nsg, -1);
      const auto& l2s = P.hs.num.l2g_surf;
      for (long long e = 0; e < P.ne; ++e) {
        int c = 0;
        while (c + 1 < C && static_cast<long long>(P.ne) * (c + 1) / C <= e) ++c;
        for (int q = 0; q < nsr; ++q) {
          const int g = l2s[e * nsr + q];
          lo[g] = std::min(lo[g], c);
          hi[g] = std::max(hi[g], c);
        }
      }
      // within each numbering class (vertices, edge nodes, face nodes: each
      // ordered roughly along the element order) send u by the suffix minimum
      // of the first-use chunk and r by the prefix maximum of the completion
      // chunk: both are monotone, so each class splits into <= C id runs
      const long long b1 = P.hs.num.num_vertex_nodes;
      const long long b2 = b1 + static_cast<long long>(P.hs.num.num_edges) * (P.order - 1);
      const long long bounds[4] = {0, b1, b2, P.nsg};
      for (int k = 0; k < 3; ++k) {
        const int s0 = static_cast<int>(bounds[k]), s1 = static_cast<int>(bounds[k + 1]);
        if (s1 <= s0) continue;
        std::vector<int> sm(s1 - s0), pm(s1 - s0);
        int m = C;
        for (int g = s1 - 1; g >= s0; --g) sm[g - s0] = m = std::min(m, lo[g]);
        m = -1;
        for (int g = s0; g < s1; ++g) pm[g - s0] = m = std::max(m, hi[g]);
        auto runs = [&](const std::vector<int>& key, std::vector<Plan::IdRun>& out) {
          for (int g = s0; g < s1;) {
            int h = g + 1;
            while (h < s1 && key[h - s0] == key[g - s0]) ++h;
            out.push_back({g, h, std::max(0, std::min(C - 1, key[g - s0]))});
            g = h;
          }
        };
        runs(sm, P.runs_in);
        runs(pm, P.runs_out);
      }
      auto by_chunk = [](const Plan::IdRun& a, const Plan::IdRun& b) { return a.chunk < b.chunk; };
      std::stable_sort(P.runs_in.begin(), P.runs_in.end(), by_chunk);
      std::stable_sort(P.runs_out.begin(), P.runs_out.end(), by_chunk);
    }
    if (!P.runs_in.empty()) {
      // surface u by first use, interior u per chunk (H2D); element kernel per chunk;
      // surface r gathered and sent as soon as every copy's element chunk is done (D2H)
      HXB_CUDA(cudaEventRecord(ev_done, P.s_main));
      HXB_CUDA(cudaStreamWaitEvent(P.s_in, ev_done, 0));
      std::size_t ri = 0, ro = 0;
      for (int c = 0; c < C; ++c) {
        for (; ri < P.runs_in.size() && P.runs_in[ri].chunk <= c; ++ri) {
          const auto& R = P.runs_in[ri];
          HXB_CUDA(cudaMemcpyAsync(P.p + R.g0, u + R.g0, sizeof(double) * (R.g1 - R.g0), cudaMemcpyHostToDevice,
                                   P.s_in));
        }
        const int e0 = static_cast<int>(static_cast<long long>(P.ne) * c / C);
        const int e1 = static_cast<int>(static_cast<long long>(P.ne) * (c + 1) / C);
        const long long g0 = P.nsg + e0 * NI, cnt = (e1 - e0) * NI;
        if (cnt > 0)
          HXB_CUDA(cudaMemcpyAsync(P.p + g0, u + g0, sizeof(double) * cnt, cudaMemcpyHostToDevice, P.s_in));
        HXB_CUDA(cudaEventRecord(P.pipe_ev[2 * c], P.s_in));
        HXB_CUDA(cudaStreamWaitEvent(P.s_main, P.pipe_ev[2 * c], 0));
        if (e1 > e0) HXB_DISPATCH_NP(P.np, launch_ax_elem_range, P, P.p, P.f, e0, e1, P.s_main);
        const std::size_t ro0 = ro;
        for (; ro < P.runs_out.size() && P.runs_out[ro].chunk <= c; ++ro) {
          AxGatherArgs g;  // surface assembly + Dirichlet rows (operator.cpp:278-280) of this run
          g.rsurf = P.rsurf;
          g.off = P.ax_off;
          g.idx = P.ax_idx;
          g.u = P.p;
          g.mask = P.mask;
          g.r = P.f;
          g.t_begin = P.runs_out[ro].g0;
          g.num_surface_global = P.runs_out[ro].g1;
          g.nodes = nullptr;
          g.dot = DotArgs{};
          const int n = P.runs_out[ro].g1 - P.runs_out[ro].g0;
          ax_gather_kernel<<<std::max(1, std::min(fill_grid(ax_gather_kernel, kGatherBlock, P.nsg),
                                                  (n + kGatherBlock - 1) / kGatherBlock)),
                             kGatherBlock, 0, P.s_main>>>(g);
          P.launches += 1;
        }
        HXB_CUDA(cudaEventRecord(P.pipe_ev[2 * c + 1], P.s_main));
        HXB_CUDA(cudaStreamWaitEvent(P.s_out, P.pipe_ev[2 * c + 1], 0));
        if (cnt > 0)
          HXB_CUDA(cudaMemcpyAsync(r + g0, P.f + g0, sizeof(double) * cnt, cudaMemcpyDeviceToHost, P.s_out));
        for (std::size_t q = ro0; q < ro; ++q) {
          const auto& R = P.runs_out[q];
          HXB_CUDA(cudaMemcpyAsync(r + R.g0, P.f + R.g0, sizeof(double) * (R.g1 - R.g0), cudaMemcpyDeviceToHost,
                                   P.s_out));
        }
        P.launches += 1;
      }
      HXB_CUDA(cudaGetLastError());
      HXB_CUDA(cudaStreamSynchronize(P.s_out));
      return;
    }
    HXB_CUDA(cudaEventRecord(ev_done, P.s_main));  // previous work on the plan's buffers is ordered first
    HXB_CUDA(cudaStreamWaitEvent(P.s_in, ev_done, 0));
    HXB_CUDA(cudaMemcpyAsync(P.p, u, sbytes, cudaMemcpyHostToDevice, P.s_in));
    HXB_CUDA(cudaEventRecord(ev_surf, P.s_in));
    for (int c = 0; c < C; ++c) {
      const int e0 = static_cast<int>(static_cast<long long>(P.ne) * c / C);
      const int e1 = static_cast<int>(static_cast<long long>(P.ne) * (c + 1) / C);
      const long long g0 = P.nsg + e0 * NI, cnt = (e1 - e0) * NI;
      if (cnt > 0)
        HXB_CUDA(cudaMemcpyAsync(P.p + g0, u + g0, sizeof(double) * cnt, cudaMemcpyHostToDevice, P.s_in));
      HXB_CUDA(cudaEventRecord(P.pipe_ev[2 * c], P.s_in));
      HXB_CUDA(cudaStreamWaitEvent(P.s_main, P.pipe_ev[2 * c], 0));
      if (e1 > e0) HXB_DISPATCH_NP(P.np, launch_ax_elem_range, P, P.p, P.f, e0, e1, P.s_main);
      HXB_CUDA(cudaEventRecord(P.pipe_ev[2 * c + 1], P.s_main));
      HXB_CUDA(cudaStreamWaitEvent(P.s_out, P.pipe_ev[2 * c + 1], 0));
      if (cnt > 0)
        HXB_CUDA(cudaMemcpyAsync(r + g0, P.f + g0, sizeof(double) * cnt, cudaMemcpyDeviceToHost, P.s_out));
    }
    AxGatherArgs g;  // surface assembly + Dirichlet rows (operator.cpp:278-280)
    g.rsurf = P.rsurf;
    g.off = P.ax_off;
    g.idx = P.ax_idx;
    g.u = P.p;
    g.mask = P.mask;
    g.r = P.f;
    g.num_surface_global = P.nsg;
    g.nodes = nullptr;
    g.dot = DotArgs{};
    ax_gather_kernel<<<fill_grid(ax_gather_kernel, kGatherBlock, P.nsg), kGatherBlock, 0, P.s_main>>>(g);
    P.launches += C + 1;
    HXB_CUDA(cudaGetLastError());
    HXB_CUDA(cudaEventRecord(ev_done, P.s_main));
    HXB_CUDA(cudaStreamWaitEvent(P.s_out, ev_done, 0));
    HXB_CUDA(cudaMemcpyAsync(r, P.f, sbytes, cudaMemcpyDeviceToHost, P.s_out));
    HXB_CUDA(cudaStreamSynchronize(P.s_out));
  });
}

static int apply_precond_host(hxb_plan* plan, const double* r, double* z, int mode)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    if (mode == HXB_PRECOND_FINE_ONLY && !pl->do_fine) throw HxbError(HXB_EINVAL, "system has no fine preconditioner");
    if (mode == HXB_PRECOND_COARSE_ONLY && !pl->do_coarse)
      throw HxbError(HXB_EINVAL, "system has no coarse preconditioner");
    const std::size_t bytes = sizeof(double) * pl->N;
    HXB_CUDA(cudaMemcpyAsync(pl->r, r, bytes, cudaMemcpyHostToDevice, pl->s_main));
    if (pl->bitwise) {
      compat_apply_P(pl->cx, pl->precond_mode, mode, pl->r, pl->z, pl->s_main);
    } else if (mode < 0) {
      enqueue_precond(*pl, nullptr);
    } else {
      // component-only applies (FinePreconditioner::apply / CoarsePreconditioner::apply):
      // run the requested branch and a combine without the mask/identity rows
      const bool f = mode == HXB_PRECOND_FINE_ONLY, c = mode == HXB_PRECOND_COARSE_ONLY;
      if (f) HXB_DISPATCH_NP(pl->np, launch_fdm, *pl, pl->s_main);
      if (c) {
        HXB_DISPATCH_NP(pl->np, launch_restrict, *pl, pl->s_main);
        HXB_CUDA(cudaGraphLaunch(pl->coarse_exec, pl->s_main));
      }
      // FinePreconditioner::apply / CoarsePreconditioner::apply have no mask
      // rows; emulate with a mask-free combine by temporarily pointing at a zero mask
      std::uint8_t* saved = pl->mask;
      pl->mask = pl->zero_mask;
      launch_combine(*pl, nullptr, pl->s_main, f, c);
      pl->mask = saved;
    }
    HXB_CUDA(cudaGetLastError());
    HXB_CUDA(cudaMemcpyAsync(z, pl->z, bytes, cudaMemcpyDeviceToHost, pl->s_main));
    HXB_CUDA(cudaStreamSynchronize(pl->s_main));
  });
}

int hxb_apply_P(hxb_plan* plan, const double* r, double* z)
{
  Plan* pl = plan ? reinterpret_cast<Plan*>(plan) : nullptr;
  if (pl && pl->group)
    return guarded([&] {
      if (!r || !z) throw HxbError(HXB_EINVAL, "null argument");
      group_apply_P(*pl, r, z);
    });
  return apply_precond_host(plan, r, z, -1);
}
int hxb_apply_fine(hxb_plan* plan, const double* r, double* z)
{
  return apply_precond_host(plan, r, z, HXB_PRECOND_FINE_ONLY);
}
int hxb_apply_coarse(hxb_plan* plan, const double* r, double* z)
{
  return apply_precond_host(plan, r, z, HXB_PRECOND_COARSE_ONLY);
}

int hxb_apply_P_device(hxb_plan* plan, const double* d_r, double* d_z, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    cudaStream_t s = pl->s_main;
    caller_stream_in(*pl, stream);
    if (pl->bitwise) {
      compat_apply_P(pl->cx, pl->precond_mode, -1, d_r, d_z, s);
    } else {
      if (d_r != pl->r) HXB_CUDA(cudaMemcpyAsync(pl->r, d_r, sizeof(double) * pl->N, cudaMemcpyDeviceToDevice, s));
      enqueue_precond(*pl, nullptr);
      if (d_z != pl->z) HXB_CUDA(cudaMemcpyAsync(d_z, pl->z, sizeof(double) * pl->N, cudaMemcpyDeviceToDevice, s));
    }
    caller_stream_out(*pl, stream);
  });
}

static void solve_dispatch(Plan& pl, const hxb_pcg_config& cfg, hxb_pcg_result* res)
{
  if (!pl.bitwise) {
    run_pcg(pl, cfg, res);
    return;
  }
  HXB_CUDA(cudaEventRecord(pl.ev_t0, pl.s_main));
  compat_pcg(pl.cx, pl.precond_mode, pl.b, cfg, res, pl.s_main);
  HXB_CUDA(cudaEventRecord(pl.ev_t1, pl.s_main));
  HXB_CUDA(cudaEventSynchronize(pl.ev_t1));
  float ms = 0;
  HXB_CUDA(cudaEventElapsedTime(&ms, pl.ev_t0, pl.ev_t1));
  res->solve_seconds = ms / 1000.0;
  if (res->u) HXB_CUDA(cudaMemcpy(res->u, pl.cx.u, sizeof(double) * pl.N, cudaMemcpyDeviceToHost));
}

// b = assemble_load(s = 1) (problem.cpp:38-46): m_N * 1 off the Dirichlet nodes, on the device
static void fill_default_b(Plan& pl)
{
  load_ones_kernel<<<vec_grid(pl.N), kVecBlock, 0, pl.s_main>>>(pl.mask, pl.d_lumped, pl.N, pl.b);
  HXB_CUDA(cudaGetLastError());
  HXB_CUDA(cudaStreamSynchronize(pl.s_main));
}

int hxb_solve(hxb_plan* plan, const double* b, const hxb_pcg_config* cfg, hxb_pcg_result* res)
{
  return guarded([&] {
    Plan* pl = as_plan(plan);
    if (!cfg || !res) throw HxbError(HXB_EINVAL, "null argument");
    if (pl->group) {
      group_solve(*pl, b, *cfg, res);
      return;
    }
    if (pl->nranks > 1) throw HxbError(HXB_EINVAL, "staged distributed plans: use hxb_dist_* (or a multi-GPU plan)");
    HXB_CUDA(cudaSetDevice(pl->device));
    if (b)
      HXB_CUDA(cudaMemcpy(pl->b, b, sizeof(double) * pl->N, cudaMemcpyHostToDevice));
    else
      fill_default_b(*pl);
    solve_dispatch(*pl, *cfg, res);
  });
}

int hxb_solve_device(hxb_plan* plan, const double* d_b, const hxb_pcg_config* cfg, hxb_pcg_result* res)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (pl->nranks > 1) throw HxbError(HXB_EINVAL, "distributed plans support the staged operator only");
    if (!cfg || !res) throw HxbError(HXB_EINVAL, "null argument");
    HXB_CUDA(cudaSetDevice(pl->device));
    if (d_b && d_b != pl->b)
      HXB_CUDA(cudaMemcpy(pl->b, d_b, sizeof(double) * pl->N, cudaMemcpyDeviceToDevice));
    else if (!d_b)
      fill_default_b(*pl);
    solve_dispatch(*pl, *cfg, res);
  });
}

static void ensure_coords(Plan& pl)
{
  if (pl.d_xyz) return;
  pl.h_xyz = global_node_coords(pl.hs);
  pl.d_xyz = pl.mem.upload(pl.h_xyz);
}

int hxb_node_coords(hxb_plan* plan, double* xyz)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!xyz) throw HxbError(HXB_EINVAL, "null argument");
    HXB_CUDA(cudaSetDevice(pl->device));
    ensure_coords(*pl);
    std::memcpy(xyz, pl->h_xyz.data(), sizeof(double) * pl->h_xyz.size());
  });
}

int hxb_solve_heat(hxb_plan* plan, const hxb_heat_config* hc, const hxb_pcg_config* pc, hxb_heat_step* steps_out,
                   int* num_steps, int* all_converged, double* final_u, double* solve_seconds)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!hc || !pc || !steps_out || !num_steps || !all_converged) throw HxbError(HXB_EINVAL, "null argument");
    if (!(hc->dt > 0)) throw HxbError(HXB_EINVAL, "heat: dt must be positive");
    if (pl->nranks > 1) throw HxbError(HXB_EINVAL, "distributed plans: use the staged API");
    // backward Euler needs c = 1/dt on every element (problem.cpp:149 enforces it)
    const double c_dt = 1 / hc->dt;
    for (double c : pl->hs.c)
      if (!(std::fabs(c - c_dt) <= 1e-12 * std::fabs(c_dt)))
        throw HxbError(HXB_EINVAL, "heat: the plan must carry c = 1/dt on every element (problem.cpp:149)");
    HXB_CUDA(cudaSetDevice(pl->device));
    Plan& P = *pl;
    const int n = P.N;
    ensure_coords(P);
    const std::vector<double>& xyz = P.h_xyz;
    // trajectory (problem.cpp:155-170)
    double lo[3] = {xyz.empty() ? 0.0 : xyz[0], xyz.empty() ? 0.0 : xyz[1], xyz.empty() ? 0.0 : xyz[2]};
    double hi[3] = {lo[0], lo[1], lo[2]};
    for (int g = 0; g < n; ++g)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], xyz[3 * static_cast<std::size_t>(g) + d]);
        hi[d] = std::max(hi[d], xyz[3 * static_cast<std::size_t>(g) + d]);
      }
    double s0[3], s1[3];
    for (int d = 0; d < 3; ++d) {
      s0[d] = hc->source_start[d];
      s1[d] = hc->source_end[d];
    }
    if (hc->auto_trajectory) {
      int axis = 0;
      for (int d = 1; d < 3; ++d)
        if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
      for (int d = 0; d < 3; ++d) s0[d] = s1[d] = 0.5 * (lo[d] + hi[d]);
      s0[axis] = lo[axis] + hc->source_radius;
      s1[axis] = hi[axis] - hc->source_radius;
    }
    const double qd = hc->q_power / (hc->rho * hc->cp);
    const double r2 = hc->source_radius * hc->source_radius;
    const double total_time = hc->dt * hc->steps;
    double mass_total = 0;
    const std::vector<double>& lumped = host_lumped(&P);
    for (int g = 0; g < n; ++g) mass_total += lumped[g];
    if (!P.heat_u) P.heat_u = P.mem.alloc<double>(n);
    {
      std::vector<double> u0(n);
      for (int g = 0; g < n; ++g) u0[g] = P.hs.num.dirichlet_mask[g] ? 0.0 : hc->initial_value;
      HXB_CUDA(cudaMemcpy(P.heat_u, u0.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    cudaStream_t s = P.s_main;
    std::vector<double> hist(static_cast<std::size_t>(pc->max_iterations) + 2);
    *all_converged = 1;
    *num_steps = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int step = 1; step <= hc->steps; ++step) {
      const double t = hc->dt * step;
      const double frac = total_time > 0 ? std::min(1.0, t / total_time) : 0.0;
      double c[3];
      for (int d = 0; d < 3; ++d) c[d] = s0[d] + frac * (s1[d] - s0[d]);
      heat_rhs_kernel<kVecBlock><<<fill_grid(heat_rhs_kernel<kVecBlock>, kVecBlock, n), kVecBlock, 0, s>>>(
          P.d_xyz, P.d_lumped, P.mask, P.heat_u, P.b, n, c[0], c[1], c[2], r2, qd, hc->dt, hc->has_source,
          dot_args(P, P.scratch + 2));
      enqueue_ax(P, P.heat_u, P.f, nullptr, s);  // warm start: b -= A u_prev
      sub_kernel<<<fill_grid(sub_kernel, kVecBlock, n), kVecBlock, 0, s>>>(P.b, P.f, n);
      P.launches += 2;
      hxb_pcg_result res{};
      res.residual_history = hist.data();
      run_pcg(P, *pc, &res);  // du in P.u
      heat_update_kernel<kVecBlock><<<fill_grid(heat_update_kernel<kVecBlock>, kVecBlock, n), kVecBlock, 0, s>>>(
          P.heat_u, P.u, P.d_lumped, n, dot_args(P, P.scratch + 3), cdot_args(P, P.scratch + 4));
      P.launches += 1;
      double sc[5];
      HXB_CUDA(cudaMemcpyAsync(sc, P.scratch, sizeof(sc), cudaMemcpyDeviceToHost, s));
      HXB_CUDA(cudaStreamSynchronize(s));
      hxb_heat_step& rec = steps_out[step - 1];
      rec.step = step;
      rec.iterations = res.iterations;
      rec.residual = res.num_residuals > 0 ? hist[res.num_residuals - 1] : 0.0;
      rec.mean_temperature = sc[3] / mass_total;
      rec.l2_norm = std::sqrt(sc[4]);
      rec.source_integral = sc[2];
      *num_steps = step;
      if (res.status != HXB_PCG_CONVERGED) {
        *all_converged = 0;
        break;
      }
    }
    if (solve_seconds) *solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (final_u) HXB_CUDA(cudaMemcpy(final_u, P.heat_u, sizeof(double) * n, cudaMemcpyDeviceToHost));
  });
}

int hxb_load_ones(hxb_plan* plan, double* b)
{
  return guarded([&] {
    Plan* pl = as_plan(plan);
    const HostSetup& hs = plan_hs(pl);
    const std::vector<double>& lumped = host_lumped(pl);
    for (int g = 0; g < pl->N; ++g) b[g] = hs.num.dirichlet_mask[g] ? 0.0 : lumped[g] * 1.0;
  });
}

int hxb_lumped_mass(hxb_plan* plan, double* m)
{
  return guarded([&] {
    Plan* pl = as_plan(plan);
    std::memcpy(m, host_lumped(pl).data(), sizeof(double) * pl->N);
  });
}

int hxb_export_geometry(hxb_plan* plan, double* mass, double* wg)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    const std::size_t nloc = pl->nloc, nlocp = (nloc + 1) & ~std::size_t{1}, nel = pl->ne;
    if (mass) HXB_CUDA(cudaMemcpy(mass, pl->mass, nel * nloc * sizeof(double), cudaMemcpyDeviceToHost));
    if (wg) {
      if (!pl->wg) throw HxbError(HXB_EINVAL, "plan holds no stored planes (on-the-fly variant)");
      std::vector<double> blk(nel * 6 * nlocp);
      HXB_CUDA(cudaMemcpy(blk.data(), pl->wg, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (std::size_t e = 0; e < nel; ++e)
        for (int p = 0; p < 6; ++p)
          std::memcpy(wg + p * nel * nloc + e * nloc, &blk[(e * 6 + p) * nlocp], nloc * sizeof(double));
    }
  });
}

int hxb_export_maps(hxb_plan* plan, int32_t* l2g, int64_t* g2l_offsets, int32_t* g2l_elem, int32_t* g2l_local,
                    int32_t* sub_l2g, uint8_t* dirichlet_mask)
{
  return guarded([&] { export_index_maps(plan_hs(as_plan(plan)), l2g, g2l_offsets, g2l_elem, g2l_local, sub_l2g, dirichlet_mask); });
}

int hxb_amg_level(hxb_plan* plan, int level, int64_t* rows, int64_t* nnz, int64_t* ptr, int32_t* col, double* val,
                  int32_t* aggregate)
{
  return guarded([&] { export_amg_level(plan_hs(as_plan(plan)), level, rows, nnz, ptr, col, val, aggregate); });
}

// Per-component device times (ms, CUDA events, warm caches, mean of reps):
// out[0] Ax element kernel, [1] Ax gather, [2] FDM subdomain solves,
// [3] coarse branch graph (restrict + solve + prolong), [4] combine,
// [5] full P apply (fine || coarse, combine), [6] PCG vector update,
// [7] PCG direction update.
int hxb_profile(hxb_plan* plan, int reps, double* out)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    cudaStream_t s = pl->s_main;
    auto timeit = [&](auto&& fn) {
      for (int w = 0; w < 2; ++w) fn();
      HXB_CUDA(cudaStreamSynchronize(s));
      HXB_CUDA(cudaEventRecord(pl->ev_t0, s));
      for (int q = 0; q < reps; ++q) fn();
      HXB_CUDA(cudaEventRecord(pl->ev_t1, s));
      HXB_CUDA(cudaEventSynchronize(pl->ev_t1));
      float ms = 0;
      HXB_CUDA(cudaEventElapsedTime(&ms, pl->ev_t0, pl->ev_t1));
      return static_cast<double>(ms) / reps;
    };
    for (int q = 0; q < 16; ++q) out[q] = 0;
    ensure_hist(*pl, 4);
    // realistic operands: r = p = m_N (the Poisson load before masking), so the
    // AMG K-cycles do their full work (a zero right-hand side exits early)
    HXB_CUDA(cudaMemcpyAsync(pl->r, pl->d_lumped, sizeof(double) * pl->N, cudaMemcpyDeviceToDevice, s));
    HXB_CUDA(cudaMemcpyAsync(pl->p, pl->d_lumped, sizeof(double) * pl->N, cudaMemcpyDeviceToDevice, s));
    if (pl->do_fine) HXB_DISPATCH_NP(pl->np, launch_fdm, *pl, s);
    out[0] = timeit([&] { HXB_DISPATCH_NP(pl->np, launch_ax_elem, *pl, pl->p, pl->f, DotArgs{}, s); });
    out[1] = timeit([&] { enqueue_ax(*pl, pl->p, pl->f, nullptr, s); }) - out[0];
    if (pl->do_fine) out[2] = timeit([&] { HXB_DISPATCH_NP(pl->np, launch_fdm, *pl, s); });
    if (pl->do_coarse) out[3] = timeit([&] { HXB_CUDA(cudaGraphLaunch(pl->coarse_exec, s)); });  // after Rpart
    out[4] = timeit([&] { launch_combine(*pl, pl->zr_hist, s, pl->do_fine, pl->do_coarse); });
    if (pl->do_fine) out[12] = timeit([&] { launch_combine(*pl, pl->zr_hist, s, true, false); });

    if (pl->do_coarse) out[13] = timeit([&] { launch_combine(*pl, pl->zr_hist, s, false, true); });
    out[5] = timeit([&] { enqueue_precond(*pl, pl->zr_hist); });
    HXB_CUDA(cudaMemcpy(pl->pf_hist, pl->zr_hist, sizeof(double), cudaMemcpyDeviceToDevice));
    out[6] = timeit([&] {
      pcg_update_kernel<kVecBlock><<<fill_grid(pcg_update_kernel<kVecBlock>, kVecBlock, pl->N), kVecBlock, 0, s>>>(pl->f, pl->r, pl->N, pl->zr_hist, pl->pf_hist,
                                                                         0, dot_args(*pl, pl->res2));
    });
    out[7] = timeit([&] {
      pcg_dir_kernel<<<fill_grid(pcg_dir_kernel, kVecBlock, pl->N), kVecBlock, 0, s>>>(pl->z, pl->p, pl->u, pl->N, pl->zr_hist, pl->pf_hist, 0);
    });
    if (pl->do_coarse) {
      // standalone restriction (used without a fine branch; fused into FDM otherwise)
      out[8] = timeit([&] { HXB_DISPATCH_NP(pl->np, launch_restrict, *pl, s); });
      out[9] = timeit([&] { launch_prolong(*pl, s); });
      out[10] = out[3] - out[9];  // vertex gather + AMG / dense solve
    }
    HXB_CUDA(cudaGetLastError());
  });
}

int hxb_bench_apply_A(hxb_plan* plan, int reps, double* ms_per_apply, double* ms_elem_kernel)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    cudaStream_t s = pl->s_main;
    for (int w = 0; w < 3; ++w) enqueue_ax(*pl, pl->p, pl->f, nullptr, s);
    HXB_CUDA(cudaStreamSynchronize(s));
    HXB_CUDA(cudaEventRecord(pl->ev_t0, s));
    for (int q = 0; q < reps; ++q) enqueue_ax(*pl, pl->p, pl->f, nullptr, s);
    HXB_CUDA(cudaEventRecord(pl->ev_t1, s));
    HXB_CUDA(cudaEventSynchronize(pl->ev_t1));
    float ms = 0;
    HXB_CUDA(cudaEventElapsedTime(&ms, pl->ev_t0, pl->ev_t1));
    *ms_per_apply = ms / reps;
    if (ms_elem_kernel) {
      HXB_CUDA(cudaEventRecord(pl->ev_t0, s));
      for (int q = 0; q < reps; ++q) HXB_DISPATCH_NP(pl->np, launch_ax_elem, *pl, pl->p, pl->f, DotArgs{}, s);
      HXB_CUDA(cudaEventRecord(pl->ev_t1, s));
      HXB_CUDA(cudaEventSynchronize(pl->ev_t1));
      HXB_CUDA(cudaEventElapsedTime(&ms, pl->ev_t0, pl->ev_t1));
      *ms_elem_kernel = ms / reps;
    }
    HXB_CUDA(cudaGetLastError());
  });
}

// ---- distributed Ax (element-slab partition) ---------------------------------
static void dist_stream_in(Plan* pl, void* stream) { caller_stream_in(*pl, stream); }
static void dist_stream_out(Plan* pl, void* stream) { caller_stream_out(*pl, stream); }

int hxb_dist_info(hxb_plan* plan, int64_t* info)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!info) throw HxbError(HXB_EINVAL, "null argument");
    const int64_t v[8] = {pl->rank, pl->nranks, pl->e0, pl->e0 + pl->ne, pl->n_up, pl->n_down, pl->n_grp0, pl->N};
    std::memcpy(info, v, sizeof(v));
  });
}

int hxb_dist_lists(hxb_plan* plan, int32_t* up_nodes, int32_t* down_nodes)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    if (pl->nranks == 1) return;
    if (up_nodes && pl->n_up)
      HXB_CUDA(cudaMemcpy(up_nodes, pl->ax_nodes + pl->n_grp0, sizeof(int) * pl->n_up, cudaMemcpyDeviceToHost));
    if (down_nodes && pl->n_down)
      HXB_CUDA(cudaMemcpy(down_nodes, pl->ax_nodes + pl->n_grp0 + pl->n_up, sizeof(int) * pl->n_down,
                          cudaMemcpyDeviceToHost));
  });
}

int hxb_dist_apply_A_begin(hxb_plan* plan, const double* d_u, double* d_r, double* d_send_up, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    enqueue_ax(*pl, d_u, d_r, nullptr, pl->s_main);  // owned elements + group-0 nodes
    if (pl->n_up) {
      dist_partial_kernel<<<vec_grid(pl->n_up), kVecBlock, 0, pl->s_main>>>(pl->ax_off + pl->n_grp0, pl->ax_idx, pl->rsurf,
                                                                             pl->n_up, d_send_up);
      pl->launches += 1;
    }
    dist_stream_out(pl, stream);
  });
}

int hxb_dist_apply_A_continue(hxb_plan* plan, const double* d_u, double* d_r, const double* d_recv_down,
                              double* d_send_down, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    if (pl->n_down) {
      const int t0 = pl->n_grp0 + pl->n_up;
      dist_continue_kernel<<<vec_grid(pl->n_down), kVecBlock, 0, pl->s_main>>>(
          pl->ax_off + t0, pl->ax_idx, pl->rsurf, pl->ax_nodes + t0, pl->n_down, d_u, pl->mask, d_recv_down, d_r,
          d_send_down);
      pl->launches += 1;
    }
    dist_stream_out(pl, stream);
  });
}

int hxb_dist_apply_A_end(hxb_plan* plan, double* d_r, const double* d_recv_up, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    if (pl->n_up) {
      dist_finish_kernel<<<vec_grid(pl->n_up), kVecBlock, 0, pl->s_main>>>(pl->ax_nodes + pl->n_grp0, pl->n_up, d_recv_up,
                                                                            d_r);
      pl->launches += 1;
    }
    dist_stream_out(pl, stream);
  });
}

// ---- distributed preconditioned CG (staged; Python/NCCL carries the messages)
int hxb_dist_pcg_info(hxb_plan* plan, int64_t* info)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!info) throw HxbError(HXB_EINVAL, "null argument");
    const int64_t v[16] = {pl->n_g_from_down, pl->n_g_from_up, pl->n_g_to_down, pl->n_g_to_up,
                           pl->n_fsend_down,  pl->n_fsend_up,  pl->n_frecv_down, pl->n_frecv_up,
                           pl->e0,           pl->e0 + pl->ne, pl->ne_total,    pl->do_fine ? 1 : 0,
                           pl->do_coarse ? 1 : 0, pl->n_up, pl->n_down, pl->N};
    std::memcpy(info, v, sizeof(v));
  });
}

int hxb_dist_vec(hxb_plan* plan, int mode, double a, const double* x0, const double* x1, double* y0, double* y1,
                 void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (mode < 0 || mode > 3) throw HxbError(HXB_EINVAL, "mode out of range");
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    const int total = pl->n_loc_surf + (pl->ib1 - pl->ib0);
    dist_vec_kernel<<<fill_grid(dist_vec_kernel, kVecBlock, total), kVecBlock, 0, pl->s_main>>>(
        mode, pl->loc_list, pl->n_loc_surf, pl->ib0, pl->ib1, a, x0, x1, y0, y1);
    pl->launches += 1;
    dist_stream_out(pl, stream);
  });
}

int hxb_dist_dot(hxb_plan* plan, const double* x, const double* y, double* d_out, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    const int total = pl->n_fin_surf + (pl->ib1 - pl->ib0);
    dist_dot_kernel<kVecBlock><<<fill_grid(dist_dot_kernel<kVecBlock>, kVecBlock, total), kVecBlock, 0, pl->s_main>>>(
        pl->fin_surf, pl->n_fin_surf, pl->ib0, pl->ib1, x, y, dot_args(*pl, d_out));
    pl->launches += 1;
    dist_stream_out(pl, stream);
  });
}

// which: 0 ghost r to the lower rank, 1 ghost r to the upper rank, 2 finals of the
// down-interface nodes (to the lower rank); unpack: 0/1 ghosts from lower/upper,
// 2 finals of the up-interface nodes (from the upper rank)
static void dist_list(Plan* pl, int which, bool pack, const int** list, int* n)
{
  if (which == 0) {
    *list = pack ? pl->g_to_down : pl->g_from_down;
    *n = pack ? pl->n_g_to_down : pl->n_g_from_down;
  } else if (which == 1) {
    *list = pack ? pl->g_to_up : pl->g_from_up;
    *n = pack ? pl->n_g_to_up : pl->n_g_from_up;
  } else if (which == 2) {
    *list = pack ? pl->ax_nodes + pl->n_grp0 + pl->n_up : pl->ax_nodes + pl->n_grp0;
    *n = pack ? pl->n_down : pl->n_up;
  } else {
    throw HxbError(HXB_EINVAL, "which out of range");
  }
}

int hxb_dist_pack(hxb_plan* plan, int which, const double* d_x, double* d_buf, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    const int* list;
    int n;
    dist_list(pl, which, true, &list, &n);
    dist_stream_in(pl, stream);
    if (n) dist_pack_kernel<<<vec_grid(n), kVecBlock, 0, pl->s_main>>>(list, n, d_x, d_buf), pl->launches += 1;
    dist_stream_out(pl, stream);
  });
}

int hxb_dist_unpack(hxb_plan* plan, int which, const double* d_buf, double* d_x, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    const int* list;
    int n;
    dist_list(pl, which, false, &list, &n);
    dist_stream_in(pl, stream);
    if (n) dist_unpack_kernel<<<vec_grid(n), kVecBlock, 0, pl->s_main>>>(list, n, d_buf, d_x), pl->launches += 1;
    dist_stream_out(pl, stream);
  });
}

// fine subdomain solves of the owned elements on residual d_r (ghosts filled):
// local contributions to the sum buffer, the others to d_fsend [to lower | to
// upper], and the owned slab of the coarse restriction partials
int hxb_dist_fine(hxb_plan* plan, const double* d_r, double* d_fsend, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!pl->do_fine) throw HxbError(HXB_EINVAL, "plan has no fine preconditioner");
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    double* keep = pl->r;
    pl->r = const_cast<double*>(d_r);
    pl->fsend = d_fsend;
    HXB_DISPATCH_NP(pl->np, launch_fdm, *pl, pl->s_main);
    pl->r = keep;
    pl->fsend = nullptr;
    dist_stream_out(pl, stream);
  });
}

int hxb_dist_fine_recv(hxb_plan* plan, const double* d_frecv, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    const int n = pl->n_frecv_down + pl->n_frecv_up;
    if (n) dist_fine_scatter_kernel<<<vec_grid(n), kVecBlock, 0, pl->s_main>>>(pl->frecv_pos, n, d_frecv, pl->zsort),
        pl->launches += 1;
    dist_stream_out(pl, stream);
  });
}

// Rpart slab (direction 0: owned slab -> d_buf) or full array (1: d_buf -> plan)
int hxb_dist_rpart(hxb_plan* plan, int direction, double* d_buf, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!pl->do_coarse) throw HxbError(HXB_EINVAL, "plan has no coarse preconditioner");
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    if (direction == 0)
      HXB_CUDA(cudaMemcpyAsync(d_buf, pl->Rpart + 8LL * pl->e0, sizeof(double) * 8 * pl->ne, cudaMemcpyDeviceToDevice,
                               pl->s_main));
    else
      HXB_CUDA(cudaMemcpyAsync(pl->Rpart, d_buf, sizeof(double) * 8 * pl->ne_total, cudaMemcpyDeviceToDevice,
                               pl->s_main));
    dist_stream_out(pl, stream);
  });
}

// coarse solve over the full Rpart (replicated on every rank, identical results)
int hxb_dist_coarse(hxb_plan* plan, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!pl->do_coarse) throw HxbError(HXB_EINVAL, "plan has no coarse preconditioner");
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    HXB_CUDA(cudaGraphLaunch(pl->coarse_exec, pl->s_main));
    pl->launches += pl->coarse_graph_nodes;
    dist_stream_out(pl, stream);
  });
}

// z = P r on the finalised nodes (mask rows, fine + coarse sums); partial z.r -> d_zr
int hxb_dist_combine(hxb_plan* plan, const double* d_r, double* d_z, double* d_zr, void* stream)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    dist_stream_in(pl, stream);
    double* kr = pl->r;
    double* kz = pl->z;
    pl->r = const_cast<double*>(d_r);
    pl->z = d_z;
    launch_combine(*pl, d_zr, pl->s_main, pl->do_fine, pl->do_coarse);
    pl->r = kr;
    pl->z = kz;
    dist_stream_out(pl, stream);
  });
}

int hxb_kernel_timing(hxb_plan* plan, int enable, int max_launches)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    HXB_CUDA(cudaSetDevice(pl->device));
    if (enable) {
      if (max_launches < 1) throw HxbError(HXB_EINVAL, "max_launches must be >= 1");
      const std::size_t want = 2 * static_cast<std::size_t>(max_launches);
      while (pl->kt_ev.size() < want) {
        cudaEvent_t e;
        HXB_CUDA(cudaEventCreate(&e));
        pl->kt_ev.push_back(e);
      }
      pl->kt_tag.assign(pl->kt_ev.size() / 2, -1);
      pl->kt_used = 0;
    }
    pl->kt_on = enable != 0;
  });
}

int hxb_kernel_timing_read(hxb_plan* plan, int tag, double* total_ms, int* count)
{
  return guarded([&] {
    Plan* pl = as_device_plan(plan);
    if (!total_ms || !count) throw HxbError(HXB_EINVAL, "null argument");
    HXB_CUDA(cudaSetDevice(pl->device));
    HXB_CUDA(cudaStreamSynchronize(pl->s_main));
    double ms = 0;
    int c = 0;
    for (std::size_t i = 0; 2 * i + 1 < pl->kt_used; ++i) {
      if (pl->kt_tag[i] != tag) continue;
      float m = 0;
      HXB_CUDA(cudaEventElapsedTime(&m, pl->kt_ev[2 * i], pl->kt_ev[2 * i + 1]));
      ms += m;
      ++c;
    }
    *total_ms = ms;
    *count = c;
  });
}

int hxb_launch_count(hxb_plan* plan, int64_t* launches)
{
  return guarded([&] {
    Plan* pl = as_plan(plan);
    if (!launches) throw HxbError(HXB_EINVAL, "null argument");
    *launches = pl->launches;
    if (pl->group)
      for (const auto& q : pl->group->pl) *launches += q->launches;
  });
}

}  // extern "C"
