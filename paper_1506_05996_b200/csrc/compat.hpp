// Bitwise-reference mode (hxb_options.bitwise_reference): the solver path
// evaluated in the reference's exact floating-point order, so Ax, P and the
// whole PCG history equal the reference bit for bit.
//
// compat.cu is compiled with -fmad=false (the reference's Release build has no
// FMA contraction: x86-64 without -march, oracle/Makefile) and mirrors, loop
// for loop:
//   SemOperator::apply + contraction_kernel / otf_element_kernel
//                                          operator.cpp:124-287
//   scatter / gather                       mesh.cpp:455-475
//   FinePreconditioner::apply(+_parallel), solve_subdomain, tensor_pass
//                                          fine.cpp:98-270
//   restrict_residual / prolongate / CoarsePreconditioner::apply
//                                          coarse.cpp:138-208
//   AmgHierarchy cycle / ksolve / direct_solve, CsrMatrix::multiply
//                                          amg.cpp:13-20, 188-263
//   TwoScalePreconditioner::apply          precond.cpp:27-67
//   dot / norm2 / pcg                      krylov.cpp:11-71
// Reductions whose order matters (dot products, the envelope triangular
// solves) run sequentially on one thread; everything else is parallel over
// independent outputs, each output computed by the reference's own sequence
// of operations. It is a verification mode: correct, deterministic, slow.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/hexsem_b200.h"
#include "setup.hpp"

namespace hxb {

struct CompatLevel {  // one AmgHierarchy level (amg.cpp:46-52)
  int n = 0, nc = 0;
  const long long* ptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  const double* inv_diag = nullptr;
  const int* agg = nullptr;
  const int* agg_ptr = nullptr;  // members of each aggregate, ascending row
  const int* agg_mem = nullptr;
  // scratch: cycle (rho, tmp, rc, ec) and ksolve (r, z, p, f) at this level
  double *cy_rho = nullptr, *cy_tmp = nullptr, *cy_rc = nullptr, *cy_ec = nullptr;
  double *ks_r = nullptr, *ks_z = nullptr, *ks_p = nullptr, *ks_f = nullptr;
};

struct CompatEnvelope {  // EnvelopeFactor on the device
  int n = 0;
  const long long *perm = nullptr, *first = nullptr, *start = nullptr;
  const double* env = nullptr;
  double* y = nullptr;
};

struct CompatPlan {
  bool ready = false;
  int np = 0, nloc = 0, nlocp = 0, ne = 0, N = 0, P = 0, nsub = 0, nv = 0, variant = 0;
  bool do_fine = false, do_coarse = false, use_amg = false;
  // borrowed from the plan (device)
  const double* wg = nullptr;      // stored planes [e][6][nlocp]
  const double* erec = nullptr;    // on-the-fly records [e][26]: corners (bi,bj,bk bits) + kappa
  const double* mass = nullptr;    // [e][nloc]
  const double* c_e = nullptr;
  const double* kappa_e = nullptr;
  const double* h3 = nullptr;      // [e][3] element_dimensions
  const std::uint8_t* mask = nullptr;
  const double* lumped = nullptr;
  const int* fine_pos = nullptr;   // [e][nsub] position in the (e, slot)-ordered per-node list, -1 sentinel
  const unsigned* fine_off = nullptr;
  double* zsort = nullptr;
  const int* conn = nullptr;       // [e][8] mesh corners (Gmsh order)
  const unsigned* vtx_off = nullptr;  // (e, cb) incidences per vertex, ascending
  const int* vtx_idx = nullptr;
  const std::uint8_t* vmask = nullptr;
  // owned (compat-only uploads)
  int* l2g = nullptr;              // [e][nloc]
  unsigned* g2l_off = nullptr;     // [N+1]
  int* g2l_idx = nullptr;          // copies e*nloc+l in (e, l) order
  int* sub_l2g = nullptr;          // [e][nsub], -1 = kNoNode
  double *D = nullptr, *nodes = nullptr, *weights = nullptr, *B = nullptr;
  double *V = nullptr, *Vinv = nullptr, *lam = nullptr, *Mext = nullptr;
  long long* Kc_ptr = nullptr;
  int* Kc_col = nullptr;
  double* Kc_val = nullptr;
  std::vector<CompatLevel> lv;     // AMG levels; coarsest solved by `coarsest`
  CompatEnvelope coarsest;         // AMG coarsest or the whole K_c (direct path)
  // scratch
  double *u_loc = nullptr, *r_loc = nullptr, *rm = nullptr, *zf = nullptr, *zc = nullptr, *work = nullptr;
  double *Rpart = nullptr, *R = nullptr, *Z = nullptr, *rho = nullptr, *dZ = nullptr;
  double *u = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *f = nullptr;
  double* scal = nullptr;          // device scalars
  double* h_scal = nullptr;        // pinned mirror
  std::vector<void*> owned;
  ~CompatPlan();
};

// Upload the compat-only tables from the host setup (the borrowed pointers
// must already be set).
void compat_init(CompatPlan& c, const HostSetup& hs);

// SemOperator::apply: r = A u (device vectors of length N).
void compat_apply_A(CompatPlan& c, const double* u, double* r, cudaStream_t s);
// mode -1: TwoScalePreconditioner::apply; HXB_PRECOND_FINE_ONLY:
// FinePreconditioner::apply; HXB_PRECOND_COARSE_ONLY: CoarsePreconditioner::apply.
void compat_apply_P(CompatPlan& c, int precond_mode, int which, const double* r, double* z, cudaStream_t s);
// pcg(A, P, b, cfg) with u0 = 0 (krylov.cpp:20-71); u left in c.u.
void compat_pcg(CompatPlan& c, int precond_mode, const double* b, const hxb_pcg_config& cfg, hxb_pcg_result* res,
                cudaStream_t s);

}  // namespace hxb
