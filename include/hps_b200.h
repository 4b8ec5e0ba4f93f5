/* hps_b200 — B200-native HPS-multigrid hot path (arXiv 2511.00735), C ABI.
 *
 * Drop-in boundary for the reference hps2d C++ entry points on the hot path
 * (paths relative to the reference root):
 *   local ItI build   ElementOperators(rule, h, eta, coeff)  proj/include/hps/element.hpp:63-64
 *                     source_to_outgoing                     proj/include/hps/element.hpp:82
 *                     build_elements(mesh, rule)             proj/include/hps/mesh.hpp:44
 *   skeleton          assemble_skeleton                      proj/include/hps/skeleton.hpp:74-75
 *                     BlockMatrix::apply (interface matvec)  proj/include/hps/block_matrix.hpp:39
 *   merge             merge_pair                             proj/include/hps/dissection.hpp:30-31
 *                     eliminate_level / build_hierarchy      proj/include/hps/dissection.hpp:64-72
 *   preconditioner    build_preconditioner / apply           proj/include/hps/multigrid.hpp:34-50
 *   GMRES             gmres / fgmres / gmres_fixed_steps      proj/include/hps/krylov.hpp:39-51
 *
 * Conventions (the reference's):
 *   - complex values are interleaved (re, im) doubles (std::complex<double>);
 *   - matrices are column-major (Eigen default);
 *   - element id = ey * n + ex; tensor node (i, j) -> i * (N + 1) + j;
 *   - element boundary order left | right | bottom | top, ascending along a side;
 *   - skeleton vector = face blocks in elimination order, each 2 (N - 1) wide,
 *     slot 0 = data incoming to e2, slot 1 = data incoming to e1.
 * Errors never cross the ABI as exceptions: every call returns an
 * hpsb_status, and hpsb_last_error() holds a thread-local message
 * (proj/src/capi.cpp:13-24, proj/include/hps/hps.h:24-30,96-97).
 * Pointers are HOST pointers unless the function name ends in _dev.
 * Objects are immutable after build and owned by the library behind opaque
 * handles with create/destroy pairs; calls on one context are serialised on
 * that context's CUDA stream (several contexts may live on one host thread).
 * Destroy every object before the context it was built on.  There is no CPU
 * fallback: without a usable sm_100 device every compute call returns
 * HPSB_INTERNAL.
 */
#ifndef HPS_B200_H
#define HPS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hpsb_status {
  HPSB_OK = 0,
  HPSB_INVALID_ARGUMENT = 1,
  HPSB_NO_CONVERGENCE = 2,
  HPSB_IO = 3,
  HPSB_INTERNAL = 4
} hpsb_status;

typedef struct hpsb_context_s* hpsb_context;
typedef struct hpsb_elements_s* hpsb_elements;
typedef struct hpsb_skeleton_s* hpsb_skeleton;
typedef struct hpsb_hierarchy_s* hpsb_hierarchy;
typedef struct hpsb_precond_s* hpsb_precond;

/* MgConfig (proj/include/hps/multigrid.hpp:12-18; reference defaults
 * depth 2, gamma 1, coarse_iters 4, exact_coarse 0). */
typedef struct hpsb_mg_config {
  int depth;        /* number of hierarchy levels used (2 <= depth <= built depth) */
  int gamma;        /* coarse calls per intermediate level (1 = V-cycle; > 1: host-recursive cycle, single-RHS applies) */
  int coarse_iters; /* unpreconditioned GMRES steps at the deepest level (<= 512) */
  int exact_coarse; /* dense inverse of M_depth instead of coarse GMRES; gamma and
                       coarse_iters are then ignored */
} hpsb_mg_config;

/* KrylovConfig (proj/include/hps/krylov.hpp:15-21; reference defaults
 * restart 60, tol 1e-8, max_iters 2000, record_history 1, reorthogonalize 0). */
typedef struct hpsb_krylov_config {
  int restart;
  double tol;
  int max_iters;
  int record_history;  /* residual history (hpsb_context_residual_history) and
                          basis_orthogonality, single right-hand side */
  int reorthogonalize; /* 0: one modified Gram-Schmidt pass per Arnoldi step
                          (krylov.cpp:98-102); != 0: two passes, run as two
                          classical passes (CGS2, one kernel each) */
} hpsb_krylov_config;

/* SolveReport (proj/include/hps/krylov.hpp:23-34), device-timed. */
typedef struct hpsb_solve_report {
  int iterations;
  int converged;
  double final_residual;
  double seconds;             /* CUDA-event time of the solve */
  double precond_seconds;     /* reserved (0) */
  double matvec_seconds;      /* reserved (0) */
  double wall_build;          /* device build time of the preconditioner's hierarchy (s), 0 without */
  double wall_solve;          /* = seconds */
  int64_t precond_memory;     /* device bytes of the preconditioner (MgPreconditioner::memory_bytes) */
  double basis_orthogonality; /* max ||<V_a,V_b>| - delta_ab| per cycle (with record_history) */
} hpsb_solve_report;

/* ---------------------------------------------------------------- library */
const char* hpsb_last_error(void);
const char* hpsb_version(void);

/* Context on one CUDA device (one stream). */
hpsb_status hpsb_context_create(int device, hpsb_context* out);
hpsb_status hpsb_context_destroy(hpsb_context ctx);
hpsb_status hpsb_context_synchronize(hpsb_context ctx);

/* ------------------------------------------------------ host-side structure
 * Integer structure, bit-exact with the reference (no device needed).       */
/* GLL rule (proj/src/spectral.cpp:26-87): nodes[N+1], weights[N+1], diff[(N+1)^2]. */
hpsb_status hpsb_gll_rule(int order, double* nodes, double* weights, double* diff);
/* IndexSets (proj/src/element.cpp:22-55): left|right|bottom|top|interior|noncorner|comp_of_full. */
hpsb_status hpsb_index_sets(int order, int* out);
/* FaceGraph (proj/src/skeleton.cpp:20-78): faces[6F] (e1,e2,s1,s2,level,group),
 * level_range[2L], face_of_element[4 n^2]. */
hpsb_status hpsb_face_graph(int n, int* faces, int* level_range, int* face_of_element);

/* Seeded BASELINE.json problem samples (shared conventions).
 * kind: 0 reference bump, 1 reference plane wave, 2 BASELINE config `config`.
 * n / order (and kappa for kind 2) override the config's mesh / wavenumber
 * when > 0 (hpsb_problem_dims reports the config's own wavenumber).  coeff[n^2][(N+1)^2] real,
 * source[n^2][(N-1)^2] complex, tside[nrhs][n^2][4][N-1] complex.          */
hpsb_status hpsb_problem_dims(int kind, int config, int n, int order, int* n_out, int* order_out,
                              int* nrhs_out, double* kappa_out, int* restart_out, double* tol_out);
hpsb_status hpsb_problem_sample(int kind, int config, uint64_t seed, int n, int order, double kappa,
                                double* coeff, double* source, double* tside, int* source_zero);

/* ----------------------------------------------------------- element stage
 * Batched local ItI build: ElementOperators + source_to_outgoing for all n^2
 * elements (proj/src/element.cpp:127-174, proj/src/mesh.cpp:36-109).
 * coeff = c = kappa^2 (1 - b) at every tensor node (real, as mesh.cpp:62),
 * source = s at the interior nodes (unweighted; the kernel applies the
 * tensor quadrature weights as mesh.cpp:89-103), or NULL for s = 0.
 * The call returns once the stage is enqueued on the context's stream (the
 * caller goes on to hpsb_skeleton_create / hpsb_hierarchy_build while the
 * device works): device inputs of hpsb_elements_build_dev must stay valid
 * until the stage completes (hpsb_elements_fallbacks or
 * hpsb_context_synchronize waits for it; host inputs are copied before the
 * call returns).  A singular element -- the reference's exception from
 * build_elements (mesh.cpp:82-84) -- is reported with its element id by the
 * first call that waits for the stage: hpsb_elements_get, hpsb_hierarchy_build
 * or any skeleton call other than hpsb_skeleton_create*.                   */
hpsb_status hpsb_elements_build(hpsb_context ctx, int n, int order, double eta,
                                const double* coeff, const double* source, hpsb_elements* out);
hpsb_status hpsb_elements_build_dev(hpsb_context ctx, int n, int order, double eta,
                                    const double* coeff_dev, const double* source_dev,
                                    hpsb_elements* out);
hpsb_status hpsb_elements_destroy(hpsb_elements el);
/* Waits for the element stage; *count = elements whose interior block was
 * not positive definite and went through the pivoted-LU fallback.          */
hpsb_status hpsb_elements_fallbacks(hpsb_elements el, int* count);
/* T[e] (4(N-1))^2 complex col-major and H[e] 4(N-1) complex, for e in [e0, e0+count). */
hpsb_status hpsb_elements_get(hpsb_elements el, int e0, int count, double* T, double* H);

/* ------------------------------------------------------------ skeleton
 * assemble_skeleton (proj/src/skeleton.cpp:88-137): the interface operator
 * M = I + sum_e scatter(T_e) and rhs = -H - sum_phys T t.  tside as from
 * hpsb_problem_sample (nrhs right-hand sides).                              */
hpsb_status hpsb_skeleton_create(hpsb_elements el, const double* tside, int nrhs,
                                 hpsb_skeleton* out);
/* Same, with t given on the physical boundary only, as boundary_side_data
 * produces it (proj/src/mesh.cpp:111-139): tbnd[nrhs][4][n][N-1] complex,
 * domain sides x=0, x=1, y=0, y=1, each with its n elements in ascending
 * order (y for the vertical sides, x for the horizontal ones) and the N-1
 * side nodes ascending.  Moves 4n(N-1) values per right-hand side instead of
 * n^2 4(N-1).                                                               */
hpsb_status hpsb_skeleton_create_boundary(hpsb_elements el, const double* tbnd, int nrhs,
                                          hpsb_skeleton* out);
hpsb_status hpsb_skeleton_destroy(hpsb_skeleton sk);
int64_t hpsb_skeleton_dim(hpsb_skeleton sk);
hpsb_status hpsb_skeleton_rhs(hpsb_skeleton sk, int r, double* rhs);
/* y = M x (BlockMatrix::apply, proj/src/block_matrix.cpp:23-31). */
hpsb_status hpsb_skeleton_apply(hpsb_skeleton sk, const double* x, double* y);
hpsb_status hpsb_skeleton_apply_dev(hpsb_skeleton sk, const double* x_dev, double* y_dev);
/* recover_solution(mesh, elements, graph, g) (proj/src/problems.cpp:60-92):
 * the field on every element's corner-free nodes from the skeleton solution
 * x (dim complex) of right-hand side r.  field: n^2 x ((N+1)^2 - 4) complex,
 * element-major, nodes in the compressed order of element.cpp:47-53.       */
hpsb_status hpsb_recover(hpsb_skeleton sk, const double* x, int r, double* field);
hpsb_status hpsb_recover_dev(hpsb_skeleton sk, const double* x_dev, int r, double* field_dev);

/* ----------------------------------------------------------- merges
 * build_hierarchy(system, depth, factor_coarse) (proj/src/dissection.cpp:200-227):
 * level-by-level Schur elimination of the merge tree, batched per level.
 * depth = 0 means all levels.  factor_coarse != 0 also factors M_depth
 * (dense inverse, dissection.cpp:225) for hpsb_direct_solve.              */
hpsb_status hpsb_hierarchy_build(hpsb_skeleton sk, int depth, int factor_coarse,
                                 hpsb_hierarchy* out);
hpsb_status hpsb_hierarchy_destroy(hpsb_hierarchy h);
hpsb_status hpsb_hierarchy_info(hpsb_hierarchy h, int* depth, int* total_levels,
                                int64_t* device_bytes, double* build_seconds);
/* Export level l's system M_l in the reference's bs x bs block layout
 * (HierarchyLevel::M, proj/include/hps/dissection.hpp:35-41).  First call
 * with keys == NULL to get the number of structurally non-zero blocks.     */
hpsb_status hpsb_hierarchy_level_blocks(hpsb_hierarchy h, int level, int* nblocks, int* first_face,
                                        int* keys, double* data);
/* y = M_l x for level l's system (HierarchyLevel::M.apply on the level
 * system over faces [first_face(l), total), proj/src/block_matrix.cpp:23-31,
 * proj/include/hps/dissection.hpp:35-41): x, y of length
 * (faces - first_face(l)) * 2 (N - 1), host pointers.  Single-GPU hierarchies. */
hpsb_status hpsb_hierarchy_level_apply(hpsb_hierarchy h, int level, const double* x, double* y);
/* Two-element merge (merge_pair, proj/src/dissection.cpp:23-82). */
hpsb_status hpsb_merge_pair(hpsb_context ctx, int side_len, const double* T1, const double* H1,
                            const double* T2, const double* H2, int alpha, int beta, double* T,
                            double* H);

/* ---------------------------------------------------- preconditioner / GMRES */
hpsb_status hpsb_precond_create(hpsb_hierarchy h, hpsb_mg_config cfg, hpsb_precond* out);
hpsb_status hpsb_precond_destroy(hpsb_precond p);
/* z = MG(v) (MgPreconditioner::apply, proj/src/multigrid.cpp:30-100). */
hpsb_status hpsb_precond_apply(hpsb_precond p, const double* v, double* z);
hpsb_status hpsb_precond_apply_dev(hpsb_precond p, const double* v_dev, double* z_dev);
/* direct_solve(hierarchy, rhs) (proj/src/dissection.cpp:240-292): forward
 * elimination through every level, the coarse solve, back substitution.
 * Needs a full-depth hierarchy built with factor_coarse != 0 (the dense
 * coarse factor of dissection.cpp:225); else HPSB_INVALID_ARGUMENT.       */
hpsb_status hpsb_direct_solve(hpsb_hierarchy h, const double* rhs, double* x);
hpsb_status hpsb_direct_solve_dev(hpsb_hierarchy h, const double* rhs_dev, double* x_dev);

/* Restarted (F)GMRES on the skeleton system (proj/src/krylov.cpp:45-178).
 * precond == NULL runs unpreconditioned GMRES.  Returns HPSB_NO_CONVERGENCE
 * (report still filled, x still written) when the tolerance is not met.     */
hpsb_status hpsb_fgmres(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                        hpsb_krylov_config cfg, hpsb_solve_report* report);
hpsb_status hpsb_fgmres_dev(hpsb_skeleton sk, hpsb_precond precond, const double* rhs_dev,
                            double* x_dev, hpsb_krylov_config cfg, hpsb_solve_report* report);
/* gmres(op, rhs, cfg, right_precond) (proj/src/krylov.cpp:180-186): restarted
 * GMRES with an optional FIXED right preconditioner (NULL: unpreconditioned).  */
hpsb_status hpsb_gmres(hpsb_skeleton sk, hpsb_precond right_precond, const double* rhs, double* x,
                       hpsb_krylov_config cfg, hpsb_solve_report* report);
hpsb_status hpsb_gmres_dev(hpsb_skeleton sk, hpsb_precond right_precond, const double* rhs_dev,
                           double* x_dev, hpsb_krylov_config cfg, hpsb_solve_report* report);

/* Multi-RHS (nrhs <= 32, single GPU): the R vectors are stored column-wise
 * (vector b at offset b * dim).  The operators are applied to all R at once
 * (one pass over the stored maps per application, FP64 tensor-core GEMMs);
 * FGMRES runs R independent solves in lockstep with per-RHS Arnoldi,
 * restarts and convergence (reports[b] per right-hand side).                */
hpsb_status hpsb_skeleton_apply_batch_dev(hpsb_skeleton sk, const double* x_dev, double* y_dev,
                                          int nrhs);
hpsb_status hpsb_precond_apply_batch_dev(hpsb_precond p, const double* v_dev, double* z_dev,
                                         int nrhs);
hpsb_status hpsb_fgmres_batch(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                              int nrhs, hpsb_krylov_config cfg, hpsb_solve_report* reports);
hpsb_status hpsb_fgmres_batch_dev(hpsb_skeleton sk, hpsb_precond precond, const double* rhs_dev,
                                  double* x_dev, int nrhs, hpsb_krylov_config cfg,
                                  hpsb_solve_report* reports);

/* Device pointer of the skeleton's right-hand side r (for _dev solves). */
const double* hpsb_skeleton_rhs_dev(hpsb_skeleton sk, int r);

/* Number of library kernels launched on this context so far (bench evidence). */
int64_t hpsb_context_launches(hpsb_context ctx);

/* Residual history (|g_{j+1}| / ||b|| per iteration, krylov.cpp:118) of the
 * last single-RHS hpsb_fgmres[_dev] run with record_history != 0.  Copies up
 * to cap values into out (may be NULL); returns the history length.       */
int64_t hpsb_context_residual_history(hpsb_context ctx, double* out, int64_t cap);

/* Device timer on the context stream (CUDA events): start, then stop returns
 * the elapsed seconds between the two event records.                       */
hpsb_status hpsb_context_timer_start(hpsb_context ctx);
hpsb_status hpsb_context_timer_stop(hpsb_context ctx, double* seconds);

/* Per-kernel CUDA-event profiling.  enable != 0 brackets every launch with
 * events (adds overhead: use outside timed regions); entries aggregate by
 * kernel name: launches, total ms, algorithmic bytes and flops.            */
hpsb_status hpsb_context_profile(hpsb_context ctx, int enable);
int hpsb_context_profile_count(hpsb_context ctx);
hpsb_status hpsb_context_profile_entry(hpsb_context ctx, int i, char* name, int name_len,
                                       int64_t* launches, double* ms, double* bytes,
                                       double* flops);
hpsb_status hpsb_context_profile_reset(hpsb_context ctx);

/* Algorithmic operator bytes one preconditioner apply streams (roofline). */
int64_t hpsb_precond_bytes(hpsb_precond p);

/* Pinned algorithmic work of SURVEY.md §8(d) (the roofline numerators):
 * setup flops = sum_e (ni^3/3 + 2 ni^2 nb + 8 nb^3)
 *             + sum_merges 8 [(8/3) s^3 + 4 s^2 (p1+p2) + s (p1+p2)^2];
 * operator bytes per outer FGMRES iteration =
 *   16 [nnz(M_1) + sum_{l<depth} (2 (2s)^2 + 2 s (p1+p2)) + ci nnz(M_depth)]
 * (sub-block entries without identities; vector traffic excluded).          */
hpsb_status hpsb_hierarchy_pinned_flops(hpsb_hierarchy h, double* element_flops,
                                        double* merge_flops);
double hpsb_precond_pinned_bytes(hpsb_precond p);

/* ------------------------------------------------------------ multi-GPU
 * Quadtree-subtree sharding over G = 2^g ranks, one per GPU.
 * Attach a communicator to a context BEFORE building objects on it; every
 * object built on that context is then sharded: each rank builds the
 * elements and merge levels 1..L-g of its own subtree; each merge of the
 * top levels runs on one rank (owner-computes, the other child's box map
 * arrives by NCCL send / recv) and the coarse level is replicated.  The
 * solvers keep distributed vectors (a rank's subtree rows plus the few
 * global rows), exchange only the global rows between levels and in the
 * matvec, and sum the Krylov inner products with an NCCL allreduce.
 * Vectors at the ABI stay full length (replicated) on every rank.           */
typedef struct hpsb_local_group_s* hpsb_local_group;
/* NCCL (one process per GPU): rank 0 makes the id, all ranks attach. */
hpsb_status hpsb_nccl_unique_id(unsigned char id[128]);
hpsb_status hpsb_context_attach_nccl(hpsb_context ctx, const unsigned char id[128], int rank,
                                     int world);
/* Single-process emulation of `world` ranks (one host thread + context per
 * rank, host barriers; used to test the sharded path on one GPU).          */
hpsb_status hpsb_local_group_create(int world, hpsb_local_group* out);
hpsb_status hpsb_local_group_destroy(hpsb_local_group g);
hpsb_status hpsb_context_attach_local(hpsb_context ctx, hpsb_local_group g, int rank);
hpsb_status hpsb_context_comm_info(hpsb_context ctx, int* rank, int* world);
/* Host-only: the sharding plan (element owner per element, face owner per
 * face with -1 on the shared top-level faces) and the last local level.    */
hpsb_status hpsb_partition(int n, int world, int rank, int* elem_owner, int* face_owner,
                           int* last_local_level);
/* Host-only: owners[g] = the rank that runs merge (group) g of `level`
 * (owner-computes: the rank holding the merge's first child box; the
 * elements' owners at level 1).  Levels above the subtrees spread their
 * merges over the ranks; the coarse (last built) level is replicated.     */
hpsb_status hpsb_merge_owners(int n, int world, int level, int* owners);

#ifdef __cplusplus
}
#endif
#endif /* HPS_B200_H */
