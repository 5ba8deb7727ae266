/*
 * hexsem_b200.h — C-ABI of the B200-native matrix-free SEM PCG solve.
 *
 * Drop-in boundary for the reference hexsem solver path (/root/reference/proj):
 * plain pointers and sizes, no C++ or torch types, no exceptions across the
 * ABI. Every entry point names the reference interface it replaces.
 *
 * Reference plug-in surface being replaced:
 *   using LinearOp = std::function<void(span<const Real>, span<Real>)>   krylov.hpp:32
 *   PcgResult pcg(const LinearOp& A, const LinearOp& P, span<const Real> b,
 *                 const PcgConfig&)                                       krylov.hpp:37-38
 *   SemSystem build_system(const ProblemConfig&)                          problem.hpp:81
 *   PoissonResult solve_poisson(const ProblemConfig&)                     problem.hpp:93
 *   SemOperator::apply                                                    operator.hpp:57
 *   TwoScalePreconditioner::apply                                         precond.hpp:24
 *   IndexMaps build_index_maps(const HexMesh&, const GllBasis&)           mesh.hpp:99
 *
 * Errors: every function returns HXB_OK (0) or an error code; the message is
 * available from hxb_last_error() (thread-local). Non-convergence is NOT an
 * error: it is reported in hxb_pcg_result.status (PcgStatus, krylov.hpp:22).
 */
#ifndef HEXSEM_B200_H
#define HEXSEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (reference exception classes they replace). */
enum {
  HXB_OK = 0,
  HXB_EINVAL = 1,   /* std::invalid_argument: bad sizes/params (operator.cpp:69-75, krylov.cpp:23-25) */
  HXB_EMESH = 2,    /* std::runtime_error: inverted element (geometry.cpp:70-72), non-conforming (mesh.cpp:402-403) */
  HXB_ENUMERIC = 3, /* std::runtime_error: Cholesky / AMG diagonal / pencil failure (coarse.cpp:126, amg.cpp:145) */
  HXB_ECUDA = 4,    /* CUDA runtime failure or no sm_100 device */
  HXB_ENCCL = 5,    /* NCCL failure (multi-GPU plans) */
  HXB_EIO = 6       /* std::runtime_error from the mesh readers/writers (mesh_io.cpp:53,112,127,190-193,214) */
};

/* PrecondMode (precond.hpp:12) */
enum { HXB_PRECOND_TWO_SCALE = 0, HXB_PRECOND_FINE_ONLY = 1, HXB_PRECOND_COARSE_ONLY = 2, HXB_PRECOND_NONE = 3 };
/* CoarseSolve (coarse.hpp:28) */
enum { HXB_COARSE_AUTOMATIC = 0, HXB_COARSE_DIRECT = 1, HXB_COARSE_AMG = 2 };
/* OperatorVariant (operator.hpp:14) */
enum { HXB_VARIANT_STORED = 0, HXB_VARIANT_ON_THE_FLY = 1 };
/* MeshFamily (mesh.hpp:47) */
enum { HXB_MESH_UNIFORM = 0, HXB_MESH_DISTORTED_DOMAIN = 1, HXB_MESH_DISTORTED_ELEMENTS = 2 };
/* BoundaryTag (mesh.hpp:19) */
enum { HXB_TAG_DIRICHLET = 0, HXB_TAG_NEUMANN = 1 };
/* PcgStatus (krylov.hpp:22) */
enum { HXB_PCG_CONVERGED = 0, HXB_PCG_MAX_ITERATIONS = 1, HXB_PCG_BREAKDOWN = 2 };

/* HexMesh (mesh.hpp:38-45): vertices xyz[3*nv]; conn[8*ne] in Gmsh corner
 * order (mesh.hpp:31-33); boundary faces as parallel arrays (mesh.hpp:24-29).
 * Borrowed: hxb_plan_create copies what it needs. */
typedef struct hxb_mesh {
  int32_t num_vertices;
  const double* xyz;
  int32_t num_elements;
  const int32_t* conn;
  int32_t num_boundary_faces;
  const int32_t* bface_element;
  const int32_t* bface_face;
  const uint8_t* bface_tag;
} hxb_mesh;

/* Owned mesh returned by the generators (generate_cube_mesh etc.). */
typedef struct hxb_mesh_buf {
  hxb_mesh view;
  void* impl;
} hxb_mesh_buf;

/* ProblemConfig solver knobs (problem.hpp:44-53) plus the B200 plan layout. */
#define HXB_MAX_GPUS 8
typedef struct hxb_options {
  int precond_mode;            /* HXB_PRECOND_* (default two_scale) */
  int coarse_solve;            /* HXB_COARSE_* (default automatic) */
  int32_t direct_threshold;    /* vertices; default 64000 (coarse.hpp:36) */
  int variant;                 /* HXB_VARIANT_* (default stored) */
  int device;                  /* CUDA device ordinal of a single-GPU plan */
  /* Verification mode: every floating-point operation in the reference's
   * order and rounding (no FMA contraction, sequential dot products as
   * krylov.cpp:11-16, the interleaved phase-2 sum of operator.cpp:152-157,
   * the full x->y->z pencil passes of fine.cpp:169-182 with true divisions,
   * the envelope Cholesky of the direct coarse solve). hxb_apply_* and
   * hxb_solve then equal the reference bit for bit; the kernels are simple
   * and slow (one thread per element / sequential reductions). */
  int bitwise_reference;
  /* Multi-GPU plan: n_gpus > 1 partitions the mesh into n_gpus
   * contiguous element slabs, one per device (devices[r], default r), each
   * driven by its own host thread; halos and PCG scalars move over NCCL
   * (distinct devices) or device-to-device copies (ranks sharing a device).
   * hxb_solve / hxb_apply_A work unchanged on such a plan. */
  int n_gpus;
  int devices[HXB_MAX_GPUS];
  /* Staged distributed plan: this plan is rank `rank` of `nranks` element
   * slabs and the caller carries the messages (hxb_dist_*). nranks <= 1: whole mesh. */
  int rank;
  int nranks;
  /* A/B switches kept for measurement and bitwise cross-checks (0 = default):
   * fused_combine: one combine after the coarse solve instead of its fine
   *   half running concurrently with the coarse graph;
   * fdm_element_order: FDM subdomains in element order instead of Morton order;
   * host_lists: fine-solve gather lists by the host counting sort instead of
   *   the device radix sort;
   * restrict_in_fdm: coarse restriction fused into the FDM kernel and the
   *   coarse solve overlapped with the fine half of a split combine, instead
   *   of a restriction pass first and the coarse solve concurrent with the FDM. */
  int fused_combine;
  int fdm_element_order;
  int host_lists;
  int restrict_in_fdm;
  /* SM partition of a single-GPU two-scale plan: the coarse solve runs on
   * coarse_sms SMs of its own (a green context) while the fine solves run on
   * the others, so the coarse solve's chain of small kernels never waits for
   * SMs held by the fine solves. 0: the library default; -1: no partition
   * (both share every SM, the coarse stream at high priority); > 0: that many
   * SMs (rounded to the hardware's granularity of 8). */
  int coarse_sms;
  int reserved[2];
} hxb_options;

/* PcgConfig (krylov.hpp:15-19) */
typedef struct hxb_pcg_config {
  double rel_tolerance;        /* (0,1), default 1e-6 */
  int max_iterations;          /* >= 1, default 500 */
  int record_history;
} hxb_pcg_config;

/* PcgResult (krylov.hpp:24-30). History/solution buffers are caller-owned:
 * residual_history and zr_history hold max_iterations+1 doubles, u holds N.
 * Any of them may be NULL. */
typedef struct hxb_pcg_result {
  int status;                  /* HXB_PCG_* */
  int iterations;
  int num_residuals;           /* entries written to residual_history */
  int num_zr;                  /* entries written to zr_history */
  double* residual_history;
  double* zr_history;
  double* u;
  double solve_seconds;        /* device-timed solve (CUDA events) */
  char diagnostic[256];
} hxb_pcg_result;

/* Plan facts (SolveReport fields, report.hpp:26-46). */
typedef struct hxb_plan_info {
  int64_t num_global;          /* N */
  int64_t num_elements;        /* N_E */
  int64_t num_vertices;
  int32_t order;
  int32_t coarse_uses_amg;
  int64_t coarse_n;
  int32_t amg_levels;          /* including the coarsest */
  int32_t precond_mode;
  int64_t amg_rows[16];
  int64_t amg_nnz[16];
  double setup_seconds;        /* host setup + upload */
  int64_t device_bytes;        /* device memory held by the plan */
  int32_t coarse_sms;          /* SMs of the coarse solve's partition (0: all SMs shared) */
  int32_t pad_;
} hxb_plan_info;

typedef struct hxb_plan hxb_plan;

const char* hxb_last_error(void);
void hxb_default_options(hxb_options* opt);

/* Mesh sources: generate_box_mesh / generate_cube_mesh / refine_uniform (mesh.hpp:49-62). */
int hxb_generate_cube_mesh(int k, int family, int boundary_tag, hxb_mesh_buf** out);
int hxb_generate_box_mesh(int kx, int ky, int kz, const double size[3], int boundary_tag, hxb_mesh_buf** out);
int hxb_refine_uniform(const hxb_mesh* in, hxb_mesh_buf** out);
void hxb_mesh_free(hxb_mesh_buf* m);

/* Mesh files (mesh_io.hpp:14-31): Gmsh MSH 2.2 ASCII (read_msh/write_msh,
 * mesh_io.cpp:49-145) and the native "HXSM0001" binary (read_native/
 * write_native, mesh_io.cpp:147-218). HXB_MESHFILE_AUTO dispatches on the
 * ".msh" extension like read_mesh_file/write_mesh_file (mesh_io.cpp:220-232).
 * Readers check every element's Jacobian (HXB_EMESH on an inverted one). */
enum { HXB_MESHFILE_AUTO = 0, HXB_MESHFILE_MSH = 1, HXB_MESHFILE_NATIVE = 2 };
int hxb_read_mesh_file(const char* path, int format, hxb_mesh_buf** out);
int hxb_write_mesh_file(const hxb_mesh* mesh, const char* path, int format);

/* build_system (problem.cpp:73-108) on a caller mesh with per-element kappa/c
 * (operator.hpp:49-55). Uploads everything once; all vectors stay on the GPU. */
int hxb_plan_create(const hxb_mesh* mesh, int order, const double* kappa_e, const double* c_e,
                    const hxb_options* opt, hxb_plan** out);
int hxb_plan_destroy(hxb_plan* plan);
int hxb_plan_get_info(const hxb_plan* plan, hxb_plan_info* info);

/* Host-pointer plug-ins: each is a drop-in LinearOp body (krylov.hpp:32). */
int hxb_apply_A(hxb_plan* plan, const double* u, double* r);          /* SemOperator::apply */
int hxb_apply_P(hxb_plan* plan, const double* r, double* z);          /* TwoScalePreconditioner::apply */
int hxb_apply_fine(hxb_plan* plan, const double* r, double* z);       /* FinePreconditioner::apply */
int hxb_apply_coarse(hxb_plan* plan, const double* r, double* z);     /* CoarsePreconditioner::apply */

/* Device-pointer variants (inputs/outputs already in HBM; stream = cudaStream_t or NULL). */
int hxb_apply_A_device(hxb_plan* plan, const double* d_u, double* d_r, void* stream);
int hxb_apply_P_device(hxb_plan* plan, const double* d_r, double* d_z, void* stream);

/* pcg(A, P, b, cfg) with u0 = 0 (krylov.cpp:20-71), entirely on the device.
 * b = NULL uses the Poisson load b = m_N * 1, masked (problem.cpp:129, 38-46). */
int hxb_solve(hxb_plan* plan, const double* b, const hxb_pcg_config* cfg, hxb_pcg_result* res);
int hxb_solve_device(hxb_plan* plan, const double* d_b, const hxb_pcg_config* cfg, hxb_pcg_result* res);

/* HeatConfig (problem.hpp:18-31): backward Euler on rho cp du/dt - div(kappa grad u) = Q
 * inside a ball moving along a straight trajectory. */
typedef struct hxb_heat_config {
  double dt;                   /* > 0; the plan must carry c = 1/dt per element (problem.cpp:149) */
  int steps;
  double rho, cp, q_power, source_radius;
  int has_source;
  int auto_trajectory;         /* straight line along the longest bounding-box axis */
  double source_start[3], source_end[3];
  double initial_value;
} hxb_heat_config;

/* HeatStep (report.hpp:57-64) */
typedef struct hxb_heat_step {
  int step, iterations;
  double residual, mean_temperature, l2_norm, source_integral;
} hxb_heat_step;

/* solve_heat (problem.cpp:145-255) on the device: per step the load, the
 * warm-start residual b - A u, a PCG solve for the correction and the
 * update all stay in HBM. steps_out holds cfg->steps records; final_u (may
 * be NULL) receives N values. */
int hxb_solve_heat(hxb_plan* plan, const hxb_heat_config* cfg, const hxb_pcg_config* pcg, hxb_heat_step* steps_out,
                   int* num_steps, int* all_converged, double* final_u, double* solve_seconds);

/* Physical coordinates of the global nodes, xyz[3N] (global_node_coords, mesh.cpp:477-492). */
int hxb_node_coords(hxb_plan* plan, double* xyz);

/* assemble_load(s = 1) and lumped_mass (problem.cpp:38-46, operator.hpp:60). */
int hxb_load_ones(hxb_plan* plan, double* b);
int hxb_lumped_mass(hxb_plan* plan, double* m);
/* Geometric factors of the plan's elements (compute_factors, geometry.cpp:105-151,
 * computed on the device): mass[NE*nloc] = rho^3 det J and, stored variant
 * only, wg[6][NE*nloc] = kappa*mass*Gt planes (operator.cpp:76-88). NULL skips. */
int hxb_export_geometry(hxb_plan* plan, double* mass, double* wg);

/* IndexMaps export for the bit-exact numbering check (mesh.hpp:66-97).
 * Any pointer may be NULL. Sizes: l2g/g2l_elem/g2l_local NE*(n+1)^3,
 * g2l_offsets N+1, sub_l2g NE*(n+3)^3, mask N. */
int hxb_export_maps(hxb_plan* plan, int32_t* l2g, int64_t* g2l_offsets, int32_t* g2l_elem,
                    int32_t* g2l_local, int32_t* sub_l2g, uint8_t* dirichlet_mask);

/* AMG level export for the bit-exact aggregation check (amg.hpp:52-60). */
int hxb_amg_level(hxb_plan* plan, int level, int64_t* rows, int64_t* nnz, int64_t* ptr, int32_t* col,
                  double* val, int32_t* aggregate);

/* GPU-free host setup (the build_system work minus the device upload): the
 * numbering, coarse matrix and AMG aggregation are exported for the
 * bit-exactness checks against the reference on machines without a GPU. */
typedef struct hxb_setup hxb_setup;
int hxb_setup_create(const hxb_mesh* mesh, int order, const double* kappa_e, const double* c_e,
                     const hxb_options* opt, hxb_setup** out);
void hxb_setup_destroy(hxb_setup* setup);
int hxb_setup_info(const hxb_setup* setup, hxb_plan_info* info);
int hxb_setup_export_maps(const hxb_setup* setup, int32_t* l2g, int64_t* g2l_offsets, int32_t* g2l_elem,
                          int32_t* g2l_local, int32_t* sub_l2g, uint8_t* dirichlet_mask);
int hxb_setup_amg_level(const hxb_setup* setup, int level, int64_t* rows, int64_t* nnz, int64_t* ptr,
                        int32_t* col, double* val, int32_t* aggregate);
int hxb_setup_lumped_mass(const hxb_setup* setup, double* m);
int hxb_setup_export_geometry(const hxb_setup* setup, double* mass, double* wg);  /* host restatement */
/* GPU-free partition lists of the distributed operator (see hxb_dist_*):
 * counts[6] = e0, e1, n_group0, n_up, n_down, local surface nodes; nodes
 * (optional) = local node ids [group0 | up | down]. */
int hxb_setup_dist_lists(const hxb_setup* setup, int rank, int nranks, int64_t* counts, int32_t* nodes);

/* GPU-free check of the sparse direct coarse factor (nested dissection +
 * supernodal Cholesky of the coupled block of K_c, the device replacement of
 * SimplicialLLT, coarse.cpp:112-127): relative residual of a solve with b = 1,
 * number of stored factor entries, separator-tree levels. */
int hxb_setup_coarse_direct_check(const hxb_setup* setup, double* rel_residual, int64_t* factor_entries,
                                  int32_t* levels);

/* GllBasis (gll.hpp:17-31) and PencilFactorization (fine.hpp:18-26) tables. */
int hxb_gll(int order, double* nodes, double* weights, double* deriv);
int hxb_pencil(int order, double* K, double* M, double* V, double* V_inv, double* lambda);

/* Time `reps` back-to-back device Ax applications of the plan's p vector with
 * CUDA events; returns mean ms per apply (kernel-level bench helper). */
int hxb_bench_apply_A(hxb_plan* plan, int reps, double* ms_per_apply, double* ms_elem_kernel);

/* Per-component device timings (ms), out[16]: Ax element, Ax gather, FDM,
 * coarse branch, combine, full P, PCG update, PCG direction, restrict,
 * prolong, AMG solve, one AMG cluster kernel, combine fine-only, combine
 * coarse-only. */
int hxb_profile(hxb_plan* plan, int reps, double* out);

/* Distributed Ax over an element-slab partition (one plan per
 * GPU, rank r of R owning elements [r*NE/R, (r+1)*NE/R), created with
 * options.rank = r, options.nranks = R and precond_mode none). Vectors are
 * global-length device arrays; a rank reads/writes only the nodes of its
 * elements. Interface nodes are summed in the reference's (e,l) order across
 * ranks (SemOperator::apply + gather, operator.cpp:255-287, mesh.cpp:463-475):
 *   begin:    element kernel, local gather, partial sums for the upper neighbour -> send_up[n_up]
 *   (send_up of rank r -> recv_down of rank r+1)
 *   continue: continue rank r-1's partials, Dirichlet rows, finals -> send_down[n_down]
 *   (send_down of rank r -> recv_up of rank r-1)
 *   end:      write the finals received from the upper neighbour
 * The result equals the single-plan hxb_apply_A bit for bit.
 * info[8] = rank, nranks, e0, e1, n_up, n_down, n_group0, N. */
int hxb_dist_info(hxb_plan* plan, int64_t* info);
int hxb_dist_lists(hxb_plan* plan, int32_t* up_nodes, int32_t* down_nodes);
int hxb_dist_apply_A_begin(hxb_plan* plan, const double* d_u, double* d_r, double* d_send_up, void* stream);
int hxb_dist_apply_A_continue(hxb_plan* plan, const double* d_u, double* d_r, const double* d_recv_down,
                              double* d_send_down, void* stream);
int hxb_dist_apply_A_end(hxb_plan* plan, double* d_r, const double* d_recv_up, void* stream);

/* Distributed two-scale PCG, staged (same slab plans, options.rank/nranks;
 * the caller carries the messages, see paper_1506_05996_b200/dist.py). Per
 * iteration of krylov.cpp:20-71: vector updates over the rank's nodes
 * (hxb_dist_vec: 0 r=b,u=0  1 u+=a p, r-=a f  2 p=z+a p  3 p=z), partial dots
 * over its finalised nodes (hxb_dist_dot -> device scalar, then all-reduce),
 * and the preconditioner:
 *   ghost r exchange (pack/unpack which 0/1), hxb_dist_fine -> fsend
 *   [to lower | to upper] + Rpart slab, exchange, hxb_dist_fine_recv,
 *   Rpart slab out (hxb_dist_rpart 0) -> all-gather -> full in (1),
 *   hxb_dist_coarse (replicated AMG), hxb_dist_combine (z on finalised
 *   nodes + partial z.r), finals of the down-interface to the lower rank
 *   (pack/unpack which 2).
 * info[16] = ghost from lower/upper, ghost to lower/upper, fine send to
 * lower/upper, fine recv from lower/upper, e0, e1, NE, has fine, has coarse,
 * n_up, n_down, N. */
int hxb_dist_pcg_info(hxb_plan* plan, int64_t* info);
int hxb_dist_vec(hxb_plan* plan, int mode, double a, const double* x0, const double* x1, double* y0, double* y1,
                 void* stream);
int hxb_dist_dot(hxb_plan* plan, const double* x, const double* y, double* d_out, void* stream);
int hxb_dist_pack(hxb_plan* plan, int which, const double* d_x, double* d_buf, void* stream);
int hxb_dist_unpack(hxb_plan* plan, int which, const double* d_buf, double* d_x, void* stream);
int hxb_dist_fine(hxb_plan* plan, const double* d_r, double* d_fsend, void* stream);
int hxb_dist_fine_recv(hxb_plan* plan, const double* d_frecv, void* stream);
int hxb_dist_rpart(hxb_plan* plan, int direction, double* d_buf, void* stream);
int hxb_dist_coarse(hxb_plan* plan, void* stream);
int hxb_dist_combine(hxb_plan* plan, const double* d_r, double* d_z, double* d_zr, void* stream);

/* Live kernel timing for the bench roofline: while enabled, the plan brackets
 * each tagged launch on its main stream with a CUDA event pair (up to
 * max_launches launches). _read sums the durations of one tag. The reference
 * equivalent is the wall-clock counter of SemOperator::apply
 * (operator.cpp:262,285-286), per kernel instead of per apply. */
enum { HXB_KT_AX_ELEM = 0, HXB_KT_AX_GATHER = 1, HXB_KT_FDM = 2, HXB_KT_COMBINE = 3, HXB_KT_COARSE = 4,
       HXB_KT_COMBINE_FINE = 5 };
int hxb_kernel_timing(hxb_plan* plan, int enable, int max_launches);
int hxb_kernel_timing_read(hxb_plan* plan, int tag, double* total_ms, int* count);
/* Kernels the plan has enqueued since creation (coarse-graph nodes counted per launch). */
int hxb_launch_count(hxb_plan* plan, int64_t* launches);

/* Counter models (operator.cpp:20-37, fine.cpp:82-92). */
uint64_t hxb_words_model(int64_t ne, int order, int variant);
uint64_t hxb_flops_model(int64_t ne, int order);
uint64_t hxb_fine_ops_model(int64_t ne, int order);
uint64_t hxb_fine_words_model(int64_t ne, int order);

#ifdef __cplusplus
}
#endif

#endif /* HEXSEM_B200_H */
