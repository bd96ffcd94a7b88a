/*
 * gmt.h -- C ABI of libgmt: the matrix-free voxel geometric-multigrid hot
 * path of GMT (arXiv 2604.26518) on NVIDIA B200 (sm_100a).
 *
 * The library solves the periodic cell problems of PAPER.md Sec. 3.1
 * (Eq. 1-3) for every load case at once -- linear elasticity (3 dof/node,
 * the 6 unit strains of App. F1) or steady heat conduction (1 dof/node, the
 * 3 unit gradients of App. F2) -- with the matrix-free element-by-element
 * (EBE) GMG V-cycle of Sec. 3.2 Alg. 1 / Sec. 4.4 Alg. 2 / Sec. 4.6, and
 * evaluates the effective tensor C^H (App. F1/F2 "Effective Property
 * Calculation").  Every arithmetic step runs in the library's own CUDA
 * kernels; there is no CPU fallback.
 *
 * Conventions:
 *  - Voxel grid of N^3 unit-cube trilinear hexahedra on the periodic torus
 *    (Eq. 2); lengths in voxel units, |Omega| = N^3.
 *  - Material field: N^3 per-voxel scales s_e >= 0 in [z][y][x] order
 *    (x fastest).  s_e = 0 is void, 1 is the base material, other values
 *    scale it (App. F3 Eq. C_e = (rho_min + rho^p) C_0 evaluated by the
 *    caller).  GMT_U8 input is occupancy: byte != 0 -> s = 1.
 *  - Nodal vectors at level l (resolution n_l = N / 2^l, l = 0 finest):
 *    float32 component planes [m][c][z][y][x], m = load case (6 elastic /
 *    3 thermal), c = component (3 / 1); NRHS * DPN * n_l^3 floats,
 *    contiguous (value (m,c) of node i at index (m*DPN + c) * n_l^3 + i,
 *    node i = x + n_l (y + n_l z)).
 *  - Voigt order (11,22,33,23,13,12), engineering shear.
 *  - Inactive nodes (every incident voxel void) are outside the active set
 *    (Sec. 4.1.1): they carry no unknowns; gmt_get_solution returns 0 there.
 *
 * Ownership: the library owns all memory it allocates; every pointer the
 * caller passes is borrowed for the duration of the call only.  Pointers
 * flagged GMT_DEVICE must be device pointers on the problem's device;
 * GMT_HOST pointers may be pageable or pinned host memory.
 *
 * Asynchrony: compute entry points enqueue work on the problem's CUDA stream
 * and return; entry points that return host values (norms, C^H, solution to
 * host) synchronise that stream first.  gmt_sync() waits explicitly.
 *
 * Errors: every int-returning function returns GMT_OK (0) or a negative
 * GMT_ERR_* code; gmt_last_error() returns a thread-local message.  A CUDA
 * error inside a call is reported as GMT_ERR_CUDA and leaves the problem
 * in an unspecified numeric state (destroy it).
 */
#ifndef GMT_H_
#define GMT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GMT_API __attribute__((visibility("default")))
#else
#define GMT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GMT_ABI_VERSION 1

#define GMT_OK 0
#define GMT_ERR_ARG (-1)     /* invalid argument */
#define GMT_ERR_CUDA (-2)    /* CUDA runtime / launch error */
#define GMT_ERR_STATE (-3)   /* call not valid in the problem's state */
#define GMT_ERR_NOMEM (-4)   /* device allocation failed */
#define GMT_ERR_NCCL (-5)    /* NCCL failure (distributed problems) */

#define GMT_PHYSICS_ELASTIC 0 /* App. F1: 3 dof/node, 6 load cases */
#define GMT_PHYSICS_THERMAL 1 /* App. F2: 1 dof/node, 3 load cases */

#define GMT_F32 0 /* float32 scales */
#define GMT_U8 1  /* uint8 occupancy */

#define GMT_HOST 0
#define GMT_DEVICE 1

typedef struct gmt_problem_s* gmt_problem;

typedef struct gmt_config {
  int physics;        /* GMT_PHYSICS_* */
  int res;            /* N_res voxels per axis; divisible by 2^(levels-1) */
  int levels;         /* L >= 1 grid levels (Sec. 3.2); 0 = default: coarsest n >= 4 */
  double E, nu;       /* base isotropic material (elastic); E > 0, -1 < nu < 0.5 */
  double kappa;       /* base conductivity (thermal), > 0 */
  double omega;       /* damped-Jacobi factor; 0 = default (0.45 elastic, 0.6 thermal) */
  int pre_sweeps;     /* It^l pre-smoothing sweeps (Alg. 1 line 3); default 2 (App. A1) */
  int post_sweeps;    /* It^l post-smoothing sweeps (Alg. 1 line 11); default 2 */
  int coarse_sweeps;  /* It^L sweeps on the coarsest level (Alg. 1 line 8); default 16 */
  int device;         /* CUDA device ordinal */
  void* stream;       /* cudaStream_t to run on, or NULL: the library creates one */
  int use_graphs;     /* 1 = replay V-cycles from a captured CUDA graph (default 1) */
} gmt_config;

/* Fill *cfg with defaults for the physics and resolution.  Returns GMT_ERR_ARG
 * for unknown physics or res < 2. */
GMT_API int gmt_default_config(gmt_config* cfg, int physics, int res);

/* gmt_create -- the problem statement of PAPER.md Sec. 3.1: resolution,
 * voxel material field and base material (E/nu or kappa).  Allocates the
 * level hierarchy on cfg->device, uploads the material and builds the
 * Galerkin coarse operators K^{l+1} = R K^l P (Sec. 3.2 "Operator
 * Consistency", Sec. 4.6 Eq. 17).  The initial guess is zero.
 *   material: N^3 voxel values [z][y][x] of material_dtype at material_location.
 * Errors: GMT_ERR_ARG (bad config / null material), GMT_ERR_NOMEM, GMT_ERR_CUDA. */
GMT_API int gmt_create(const gmt_config* cfg, const void* material, int material_dtype,
               int material_location, gmt_problem* out);

/* Replace the material field (same resolution) and rebuild the coarse
 * operators; the solution is reset to zero. */
GMT_API int gmt_set_material(gmt_problem p, const void* material, int dtype, int location);

/* Alg. 2 line 1: u^1 <- u_hat^1.  u: finest-level vector (layout above) or
 * NULL for zero.  Only active nodes (nodes touching a nonzero voxel, Sec.
 * 4.1.1) carry unknowns: values of u at inactive nodes are ignored (a device
 * buffer is copied at active nodes only; gmt_get_solution reports inactive
 * nodes as 0).  The upload is stream-ordered; the caller keeps u valid until
 * the next call that synchronises (gmt_homogenize, gmt_residual_norms,
 * gmt_get_solution to host, gmt_sync).  Errors: GMT_ERR_ARG, GMT_ERR_CUDA. */
GMT_API int gmt_set_initial_guess(gmt_problem p, const float* u, int location);

/* Alg. 2 line 6: u^{l} <- e_hat^{l} instead of 0 for level l in [1, L-1]
 * during the NEXT gmt_vcycle call only.  e: level-l vector or NULL to clear. */
GMT_API int gmt_inject_correction(gmt_problem p, int level, const float* e, int location);

/* Run ncycles V-cycles (Alg. 1 with damped-Jacobi smoothing) on the current
 * solution for all load cases.  Asynchronous. */
GMT_API int gmt_vcycle(gmt_problem p, int ncycles);

/* Relative residual of Sec. 5.2, r_m = ||f_m - K u_m||_2 / ||f_m||_2, for each
 * load case m of the current finest-level solution.  rel, abs_r, abs_f are
 * host arrays of NRHS doubles (abs_r / abs_f may be NULL).  Synchronises. */
GMT_API int gmt_residual_norms(gmt_problem p, double* rel, double* abs_r, double* abs_f);

/* Mixed-precision iterative refinement.  The level-0
 * solution is fp32 and |u| grows like N in voxel units, so plain fp32 cycles
 * stall at a relative residual of roughly N * 2^-24 (8e-5 at 512^3).  In
 * refinement the solution is held as an unevaluated pair hi + lo of fp32
 * arrays; each gmt_vcycle computes the defect f - K hi - K lo (difference-form
 * kernels), runs one V-cycle on the fp32 correction from zero with the defect
 * as right-hand side, and adds it with an error-free two-sum -- in exact
 * arithmetic the same V-cycle.  mode: 0 = auto (default: gmt_solve switches
 * when a cycle reduces the residual by less than 30 %), 1 = off (also leaves
 * refinement, u = fp32(hi + lo)), 2 = on now.  gmt_get_solution returns
 * fp32(hi + lo), gmt_homogenize evaluates C^H at hi (C^H is stationary at the
 * solution), gmt_residual_norms the residual of hi + lo.  gmt_set_material /
 * gmt_set_initial_guess leave refinement.  Slab-partitioned problems refine
 * the same way (the hi / lo ghost planes are exchanged for the defect). */
GMT_API int gmt_set_refinement(gmt_problem p, int mode);
/* Level-0 sweep implementation (rows A1-A3): 0 = k_l0, CUDA-core
 * sum-factorised stencil (default); 1 = k_l0_tc, the tensor-core variant
 * named by the north star: Sec. 4.6 Eq. 14 as batched element contractions
 * U_e K_e^T on tcgen05 (kind::tf32, 3xTF32 split for fp32 accuracy, TMEM
 * accumulators).  Same results to rounding; kept for the A/B measurement
 * (DESIGN.md "Tensor cores").  Synchronises the stream; drops the captured
 * V-cycle graph.  Errors: GMT_ERR_ARG. */
GMT_API int gmt_set_level0_kernel(gmt_problem p, int kind);

/* 1 while the problem is in refinement, 0 otherwise. */
GMT_API int gmt_refinement_active(gmt_problem p);

/* Repeat V-cycles until max_m r_m <= rel_tol or max_cycles cycles ran.
 * *cycles_done / *final_rel (max over load cases) may be NULL; history, if
 * non-NULL, receives (max_cycles+1)*NRHS doubles: per-cycle residuals,
 * history[0..NRHS) being the initial one.  Synchronises.  Returns GMT_OK
 * also when the tolerance was not reached (check *final_rel). */
GMT_API int gmt_solve(gmt_problem p, double rel_tol, int max_cycles, int* cycles_done,
              double* final_rel, double* history);

/* App. F1/F2 effective tensor of the current solution:
 *   C^H_ij = 1/|Omega| sum_e (x_0^i - u_e^i)^T (s_e K_e) (x_0^j - u_e^j)
 * written row-major to CH (NRHS x NRHS host doubles: 6x6 C^H or 3x3 kappa^H).
 * Synchronises. */
GMT_API int gmt_homogenize(gmt_problem p, double* CH);

/* Copy the finest-level solution to u (layout above).  zero_mean != 0
 * applies the Sec. 4.5 gauge sum_i u_i = 0 per load case and component over
 * the active nodes (to the copy only).  Synchronises when location==GMT_HOST. */
GMT_API int gmt_get_solution(gmt_problem p, float* u, int location, int zero_mean);

/* Compact active-node I/O (Sec. 4.1.1 "sparse voxels": the paper's input and
 * network output live on the active nodes only).  The active set of the
 * current material is the sorted list of level-0 nodes i = x + n (y + n z)
 * touching a nonzero voxel; a compact vector holds NRHS * DPN * A floats,
 * layout [m][c][k] (k = position in the list, k fastest).
 *   gmt_active_count: A (>= 0), or a negative GMT_ERR_* code.
 *   gmt_active_nodes: writes the A node indices (int32) to `nodes`.
 *   gmt_set_initial_guess_compact: Alg. 2 line 1 from a compact vector (the
 *     same semantics as gmt_set_initial_guess, a fraction of the bytes).
 *   gmt_get_solution_compact: the finest-level solution at the active nodes
 *     (zero_mean as in gmt_get_solution).  Synchronises for GMT_HOST.
 * Single-device problems only (GMT_ERR_STATE on slab-partitioned ones). */
GMT_API long long gmt_active_count(gmt_problem p);
GMT_API int gmt_active_nodes(gmt_problem p, int32_t* nodes, int location);
GMT_API int gmt_set_initial_guess_compact(gmt_problem p, const float* u_active, int location);
GMT_API int gmt_get_solution_compact(gmt_problem p, float* u_active, int location, int zero_mean);

/* Batches of independent problems on one GPU (BASELINE configs[2]:
 * high-throughput screening of many unit cells, Sec. 7.1 / App. C).  A batch
 * borrows `count` single-device problems created on the same device (they
 * must outlive it and are still usable on their own).  gmt_batch_vcycle runs
 * one V-cycle of every problem per cycle as ONE CUDA-graph launch: the
 * problems' V-cycles are captured side by side (one graph branch per
 * problem stream) and replayed concurrently; the graph is re-captured when a
 * problem's operators change shape.  It is ordered after all work already
 * enqueued on the problems' streams and before work enqueued later.
 * Problems in iterative refinement or with a pending injection are cycled
 * one by one instead.  gmt_batch_homogenize / gmt_batch_residual_norms
 * write count * NRHS^2 (C^H, row-major per problem) / count * NRHS (relative
 * residuals) host doubles with one synchronisation.  Errors: GMT_ERR_ARG
 * (empty batch, slab problems, mixed devices), GMT_ERR_CUDA. */
typedef struct gmt_batch_s* gmt_batch;
GMT_API int gmt_batch_create(gmt_problem* problems, int count, gmt_batch* out);
GMT_API int gmt_batch_vcycle(gmt_batch b, int ncycles);
GMT_API int gmt_batch_homogenize(gmt_batch b, double* CH);
GMT_API int gmt_batch_residual_norms(gmt_batch b, double* rel);
GMT_API void gmt_batch_destroy(gmt_batch b);

/* Problem properties. */
GMT_API int gmt_num_levels(gmt_problem p);
GMT_API int gmt_level_res(gmt_problem p, int level);      /* n_l */
GMT_API int gmt_nrhs(gmt_problem p);                      /* 6 or 3 */
GMT_API int gmt_dpn(gmt_problem p);                       /* 3 or 1 */
GMT_API void* gmt_stream(gmt_problem p);                  /* the problem's cudaStream_t */
GMT_API size_t gmt_device_bytes(gmt_problem p);           /* device memory held */
GMT_API int gmt_sync(gmt_problem p);
GMT_API void gmt_destroy(gmt_problem p);
GMT_API const char* gmt_last_error(void);
GMT_API int gmt_abi_version(void);

/* ---- Live profiling (bench instrumentation) ----------------------------------
 * Kernel classes: 0 level-0 damped-Jacobi sweep, 1 level-0 residual, 2 level-0
 * prolongation+correction, 3 restriction 0->1, 4 all level>=1 operator /
 * transfer kernels, 5 coarsest solve, 6 Galerkin setup, 7 C^H reduction.
 * gmt_profile_enable(p, mask): bracket every launch of the classes in `mask`
 * (bit c = class c) with CUDA events on the problem stream (also inside the
 * captured V-cycle graph).  gmt_profile_collect synchronises and accumulates
 * the elapsed times of all brackets recorded since the previous collect;
 * gmt_profile_read returns the accumulated milliseconds and launch count of
 * one class.  gmt_kernel_launches counts every libgmt kernel launch executed
 * (graph replays included). */
GMT_API int gmt_profile_enable(gmt_problem p, unsigned mask);
GMT_API int gmt_profile_collect(gmt_problem p);
GMT_API int gmt_profile_read(gmt_problem p, int cls, double* total_ms, long long* launches, int reset);
GMT_API long long gmt_kernel_launches(gmt_problem p);

/* ---- Row-level entry points (one step of the hot path each) ------------------
 * Device pointers only (GMT_DEVICE); vectors in the level layout above;
 * asynchronous on the problem's stream.  They use the problem's material and
 * Galerkin operators but never touch its solution state. */

/* Sec. 4.6 Eq. 14: y = K^l u (level 0: EBE from the material; l >= 1: the
 * Galerkin operator). */
GMT_API int gmt_op_apply(gmt_problem p, int level, const float* u, float* y);
/* Alg. 1 line 4: r = f - K^l u; f == NULL at level 0 means the load vector. */
GMT_API int gmt_op_residual(gmt_problem p, int level, const float* u, const float* f, float* r);
/* One damped-Jacobi sweep: u_out = u + omega D^{-1} (f - K^l u) on active
 * dofs, u_out = u elsewhere; f == NULL at level 0 means the load vector. */
GMT_API int gmt_op_jacobi(gmt_problem p, int level, const float* u, const float* f, float* u_out);
/* App. E2 restriction R = P^T: f_c (level+1) = R r (level). */
GMT_API int gmt_op_restrict(gmt_problem p, int level, const float* r, float* fc);
/* App. E2 prolongation + correction: u (level) += P e (level+1) on active
 * fine nodes. */
GMT_API int gmt_op_prolong_add(gmt_problem p, int level, const float* e, float* u);
/* Eq. 3 load vector f = sum_e A_e^T s_e f_e at level 0. */
GMT_API int gmt_op_loads(gmt_problem p, float* f);
/* diag(K^l), layout [c][z][y][x] (DPN * n_l^3 floats). */
GMT_API int gmt_op_diagonal(gmt_problem p, int level, float* d);
/* The assembled Galerkin operator of level l >= 1 as a 27-point block
 * stencil: S[((d*DPN + a)*DPN + b) * n_l^3 + node], d = (dx+1) + 3(dy+1) +
 * 9(dz+1): coupling of dof a at node i to dof b at node i + d. */
GMT_API int gmt_op_stencil(gmt_problem p, int level, float* S);
/* C^H of an arbitrary finest-level field u (device); CH host NRHS^2 doubles. */
GMT_API int gmt_op_effective_tensor(gmt_problem p, const float* u, double* CH);

/* ---- Slab-partitioned problems (data parallelism, Sec. 3.2 / Sec. 4.6) -------
 * The grid is cut into P slabs of N/P z-planes.  Levels l < Ld (the
 * "partitioned" levels, n_l/P >= 2 planes per slab, Ld >= 3 required) keep one
 * slab per part plus one ghost plane on each side, refreshed by halo
 * exchanges before every kernel that reads across a slab face; levels
 * l >= Ld are small and replicated on every part (each part restricts its
 * region into level Ld, then an all-gather completes it).  Dot products
 * (residual norms, C^H, the zero-mean gauge) are summed over parts.  Results
 * equal those of the single-device problem up to float rounding order.
 * Row-level entry points and gmt_inject_correction return GMT_ERR_STATE on
 * partitioned problems; every other entry point accepts them.
 *
 * Vectors/materials passed to a partitioned problem use the layout above
 * restricted to the planes the handle holds: all N planes for
 * gmt_create_slabs, this rank's N/P planes [z0, z0 + N/P) for gmt_create_dist
 * (z0 = rank * N/P).  Components stay contiguous: value (m,c) of local node i
 * is at (m*DPN + c) * (N^2 * nz_held) + i. */

/* Geometry of slab `rank` of `nslabs`: info[0] = z0 (first plane), info[1] =
 * N/P planes, info[2] = Ld (number of partitioned levels; L when nslabs==1),
 * info[3] = L.  Host only.  GMT_ERR_ARG if the partition is not possible. */
GMT_API int gmt_slab_layout(int res, int levels, int nslabs, int rank, int* info);

/* The ghost-plane exchange part `rank` of `nslabs` takes part in (row A11):
 * the list the NCCL transport issues inside one ncclGroupStart/End (and the
 * local transport resolves to device copies) for a vector view of nz owned
 * planes, ncomp components `cstride` elements apart and `plane` elements per
 * plane, with `lo` ghost planes below and `hi` above (periodic ring of parts;
 * lo, hi in {0, 1, 2}).  Entry i: send (is_send[i] = 1) or receive of
 * count[i] elements at element offset offset[i] from the view base (plane 0
 * of component 0; ghost planes at plane indices -lo .. -1 and nz .. nz+hi-1)
 * to / from part peer[i].  The sends and receives of a pair of parts match
 * in issue order (NCCL's rule).  Returns the number of entries (at most cap
 * are written; call with cap = 0 to size), negative on bad arguments.  Host
 * only, no device work. */
GMT_API int gmt_halo_schedule(int nslabs, int rank, int nz, int ncomp, long long cstride, long long plane, int lo,
                              int hi, int* peer, int* is_send, long long* offset, long long* count, int cap);

/* P slabs on one device (cfg->device), exchanging ghost planes by device
 * copies on one stream: the partitioned algorithm without a second GPU.
 * material: the full N^3 field.  The returned handle owns all slabs. */
GMT_API int gmt_create_slabs(const gmt_config* cfg, const void* material, int material_dtype,
                             int material_location, int nslabs, gmt_problem* out);

/* NCCL unique id for gmt_create_dist (call on one rank, broadcast the bytes).
 * id: host buffer of len >= 128 bytes.  GMT_ERR_NCCL if libnccl.so.2 cannot
 * be loaded (NCCL is dlopen'ed at first use). */
GMT_API int gmt_nccl_unique_id(void* id, size_t len);

/* Slab `rank` of an `nranks`-process job, one process per GPU (cfg->device).
 * Halo planes travel by ncclSend/ncclRecv, the replicated level by
 * ncclAllGather, dot products by ncclAllReduce, all on the problem stream.
 * Collective: every rank must call it (and every later entry point) in the
 * same order.  material_slab: this rank's N/P planes. */
GMT_API int gmt_create_dist(const gmt_config* cfg, const void* material_slab, int material_dtype,
                            int material_location, int rank, int nranks, const void* nccl_id,
                            gmt_problem* out);

/* Number of slabs of the problem (1 for gmt_create). */
GMT_API int gmt_num_slabs(gmt_problem p);

#ifdef __cplusplus
}
#endif
#endif /* GMT_H_ */
