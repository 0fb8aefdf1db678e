/*
 * tomesh.h — C ABI of the B200 (sm_100a) hot path of
 *   Wang, de Sturler & Paulino, "Dynamic Adaptive Mesh Refinement for
 *   Topology Optimization", arXiv:1009.4975 (reference text: PAPER.md).
 *
 * What the calls compute (citations are PAPER.md line : section / equation):
 *
 *   tomesh_upload   the FE mesh of the current adaptive quadtree/octree
 *                   (:564-571 §6; hanging-node interpolation P of Eq. 6,
 *                   :653-663), Dirichlet region Omega_0 (Eq. 1, :300-301),
 *                   loads f (Eq. 1) and the filter neighbourhoods (Eq. 4,
 *                   :600-609), copied to the device.
 *   tosolve_cg      u solving K(x) u = f (Eq. 1, :296-304) with the SIMP
 *                   modulus E_min + x^p (E0 - E_min) (Eq. 2, :322-324), via
 *                   the projected system with unit diagonal on constrained
 *                   DOFs (Eq. 8, :678-682), Dirichlet DOFs eliminated
 *                   symmetrically, solved by CG on the diagonally rescaled
 *                   system D^-1/2 A D^-1/2 (:511-523) = Jacobi-PCG, then the
 *                   recovery u = [I 0; P 0] u_hat (Eq. 9, :683-686).
 *   to_sensitivity  dc_e = -p x_e^(p-1) (E0 - E_min) u_e^T K0(h_e) u_e
 *                   (sensitivity analysis, :343-346; formula per north_star,
 *                   DESIGN.md reading R2) and optionally c = f^T u (Eq. 1).
 *   to_filter       Eq. 5 (:613-616), Stainko's volume-weighted Sigmund
 *                   filter, with H_de of Eq. 4; or its density variant
 *                   (reading R10).
 *   to_oc_update    the design update of the Fig. 1 loop (:350-354 §3, "we
 *                   use Optimality Criteria (OC)"; formula not printed, read
 *                   as Bendsoe's heuristic OC step, reading R18)
 *                   with the volume constraint of Eq. 1 (:296-304) met by a
 *                   bisection on its multiplier, entirely on the device.
 *   to_amr_mark     the refinement/derefinement marks of the dynamic AMR
 *                   strategy (:458-463 §4); the mesh update itself is host
 *                   code (tomesh_host_adapt in tomesh_host.h).
 *   to_apply_A / to_jacobi_diag / to_project_rhs / to_recover
 *                   the individual operators of Eqs. 7-9, exposed for
 *                   operator-level parity checks.
 *
 * Conventions shared by every call
 *   - dim = 2 (Q4 plane stress, unit thickness) or 3 (H8).  Local corner of
 *     an element c = cx + 2 cy + 4 cz, local DOF = dim*c + component; global
 *     DOF = dim*node + component.  Vectors over DOFs have
 *     length dim*n_node and keep hanging and fixed DOFs.
 *   - All floating point is IEEE fp64.
 *   - Device pointers are raw CUDA device addresses on the handle's device
 *     (e.g. torch.Tensor.data_ptr() of a contiguous float64 CUDA tensor).
 *     They stay owned by the caller; the library never frees or retains them.
 *   - cuda_stream is a cudaStream_t (NULL = legacy default stream).  Calls
 *     that fill host outputs synchronise that stream before returning; the
 *     others are asynchronous with respect to the host.
 *   - Errors: every call returns a status (0 = OK, >0 = result usable with a
 *     warning, <0 = failure).  No exception or abort crosses the ABI.  The
 *     thread-local message of the last failure is to_last_error().
 *   - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef TOMESH_H
#define TOMESH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct to_mesh to_mesh;

enum {
  TO_OK = 0,
  TO_NOT_CONVERGED = 1,   /* max_iter reached above rtol; stats and u filled   */
  TO_EINVAL = -1,         /* bad argument (NULL pointer, bad size, x <= 0 ...) */
  TO_ECUDA = -2,          /* CUDA runtime error                                */
  TO_ENOMEM = -3,         /* device allocation failed                          */
  TO_EMESH = -4,          /* inconsistent mesh arrays (see to_last_error)      */
  TO_ENAN = -5,           /* NaN/Inf appeared in the CG recurrences            */
  TO_EBREAKDOWN = -6,     /* p^T A p <= 0                                      */
  TO_ENONPOS_DIAG = -7    /* a free DOF has a non-positive diagonal            */
};

/* tosolve_cg flags */
enum {
  TO_WARM = 1,            /* u_dev holds the initial guess  */
  TO_FIXED_ITERS = 2,     /* run exactly max_iter iterations, ignore rtol      */
  TO_HISTORY = 4,         /* record ||r_k||/||b|| into the handle's history    */
  TO_NO_TRUE_RES = 8,     /* skip the extra matvec for relres_true             */
  TO_PROFILE = 16,        /* time every iteration kernel with CUDA events      */
  TO_PROFILE_LOOP = 32    /* one event pair around all iteration launches      */
};

/* to_filter modes */
enum { TO_FILTER_SENS = 0, TO_FILTER_DENS = 1 };

/* Mesh description (host memory; copied by tomesh_upload).
 * Lattice: finest level L = max_level, lattice unit h_L = h0 / 2^L; a leaf
 * with level l has edge s = 2^(L-l) lattice units, anchor = its minimum
 * corner in lattice units.  Arrays must follow the canonical contract of
 * SURVEY.md §8(b) C1-C9 (Morton element and node order, ascending hanging and
 * fixed lists, ascending parents per hanging node). */
typedef struct {
  int32_t dim;                 /* 2 or 3                                         */
  int32_t max_level;           /* L >= 0                                         */
  double  h0;                  /* level-0 cell edge (physical length)            */
  int64_t n_elem, n_node;
  const int32_t *elem_node;    /* [n_elem][2^dim] node ids, C4 corner order      */
  const int32_t *elem_anchor;  /* [n_elem][dim]  lattice anchors                 */
  const int8_t  *elem_level;   /* [n_elem]                                       */
  int64_t n_hang;              /* hanging nodes (Eq. 6 "constrained DOFs")       */
  const int32_t *hang_node;    /* [n_hang] ascending node ids                    */
  const int32_t *hang_ptr;     /* [n_hang+1]                                     */
  const int32_t *hang_parent;  /* [hang_ptr[n_hang]] ascending within a row      */
  const double  *hang_weight;  /* [hang_ptr[n_hang]] rows sum to 1 (1/2 or 1/4)  */
  int64_t n_fixed;
  const int64_t *fixed_dof;    /* [n_fixed] ascending DOF ids, no hanging DOF;
                                  prescribed value u0 = 0                        */
  const double  *load;         /* [dim*n_node] consistent nodal loads f, before
                                  the projection C^T (hanging loads allowed)     */
  double E0, Emin, nu;         /* SIMP E_min + x^p (E0 - E_min); Poisson ratio   */
  double rmin;                 /* filter radius (physical); 0 = no filter        */
  int64_t filt_nnz;
  const int64_t *filt_ptr;     /* [n_elem+1] or NULL when rmin == 0              */
  const int32_t *filt_idx;     /* [filt_nnz] neighbours with |c_d-c_e| < rmin,
                                  ascending, self included (C9)                  */
  uint32_t options;            /* TO_UPLOAD_* bits below (0 = defaults)          */
  int32_t  n_owned;            /* 0: every node is this handle's.  > 0: a rank's
                                  local mesh of a general-path shard group
                                  (to_gshard_attach): nodes [0, n_owned) are
                                  owned, the rest ghosts / hanging; the
                                  operator is built for the owned nodes only
                                  (forces the general path)                      */
} to_mesh_desc;

/* to_mesh_desc.options.  The operator, and therefore u, is the same on every
 * path; these only choose the device code that applies it.
 *   TO_UPLOAD_GENERAL        keep a uniform H8 box on the general (canonical
 *                            Morton order) path instead of the structured
 *                            one; tosolve_minres with TO_PC_IC0 needs it.
 *   TO_UPLOAD_LAUNCHED       general path: launch one kernel per PCG iteration
 *                            even for the smallest meshes (by default a mesh
 *                            that one thread-block cluster of at most 16
 *                            CTAs holds, e.g. c1 and c2, runs the whole loop
 *                            in that cluster with the CG state in shared
 *                            memory; failing that, a mesh of at most 32
 *                            operator blocks runs it in one cooperative
 *                            kernel).
 *   TO_UPLOAD_NO_CLUSTER     general path: do not use the cluster-resident
 *                            solver (the cooperative kernel, or one kernel
 *                            per iteration, instead).
 *   TO_UPLOAD_EP             general path: run tosolve_cg's iterations on the
 *                            element-partitioned blocks (every element once,
 *                            partial sums of shared nodes in per-block slots,
 *                            Chronopoulos-Gear form of the same PCG);
 *                            the default for large meshes where enabled.
 *   TO_UPLOAD_NO_EP          general path: never use it. */
enum { TO_UPLOAD_GENERAL = 1, TO_UPLOAD_LAUNCHED = 2, TO_UPLOAD_NO_CLUSTER = 4, TO_UPLOAD_EP = 8,
       TO_UPLOAD_NO_EP = 16 };

typedef struct {
  int32_t iters;               /* CG iterations performed                        */
  int32_t status;              /* same code as the return value                  */
  double  relres;              /* recurrence ||r_k||_2 / ||b||_2                 */
  double  relres_true;         /* ||b - A x||_2 / ||b||_2 at exit (-1 if skipped)*/
  double  ms;                  /* device time of the whole call (CUDA events)    */
  double  bnorm;               /* ||b||_2                                        */
} to_cg_stats;

typedef struct {
  int32_t dim, structured;     /* structured = 1: uniform-grid fast path chosen  */
  int64_t n_elem, n_node, n_dof, n_hang, n_fixed, filt_nnz;
  int64_t grid[3];             /* element grid when structured                   */
  int64_t device_bytes;        /* device memory held by the handle               */
  int32_t kernel_launches;     /* kernels launched by the last tosolve_cg        */
  int32_t matvec_variant;      /* CG iteration path: 1 structured H8 (one
                                  kernel per iteration), 3 general, whole
                                  loop in one cooperative kernel, 4 general
                                  one kernel per iteration, 5 general, whole
                                  loop in one thread-block cluster, 6 general
                                  element-partitioned, one kernel per
                                  iteration                                    */
  int64_t launches_total;      /* kernels launched by every call on this handle
                                  since upload (monotone counter)               */
  int32_t gen_blocks;          /* general path: owner-computes blocks (CTAs per
                                  iteration launch; 0 when structured)         */
  int32_t gen_smem_bytes;      /* general path: dynamic shared memory per CTA  */
  int32_t gen_max_loc, gen_max_el;   /* largest local node / element count of
                                  a block (they size the shared memory)       */
  int64_t gen_local_el;        /* sum over blocks of the staged elements (the
                                  element recompute is gen_local_el / n_elem) */
  int64_t gen_local_nodes;     /* sum over blocks of owned + halo + virtual
                                  node slots                                    */
} to_mesh_info;

/* Validate, copy to `device`, derive device encodings, allocate the CG
 * workspace.  Rejects with TO_EMESH: out-of-range indices, a constraint
 * parent that is itself hanging, a hanging DOF listed as fixed, hanging
 * weights not summing to 1, unsorted lists.  On success *out owns all device
 * memory until tomesh_free. */
int  tomesh_upload(const to_mesh_desc *desc, int device, void *cuda_stream, to_mesh **out);
void tomesh_free(to_mesh *m);
int  tomesh_get_info(const to_mesh *m, to_mesh_info *info);

/* Solve A u_hat = b (Eq. 8 + Dirichlet rows) by Jacobi-PCG and write
 * u = C u_hat (Eq. 9) to u_dev[dim*n_node] (fixed DOFs = 0).
 *   penal      SIMP exponent p (> 0; continuation is the caller's business)
 *   x_dev      [n_elem] densities in (0, 1]
 *   u_dev      [dim*n_node] output; input guess when flags & TO_WARM
 *   rtol       stop when ||r_k||/||b|| <= rtol (ignored with TO_FIXED_ITERS)
 *   max_iter   iteration cap (exact count with TO_FIXED_ITERS)
 *   st         nullable host stats
 * Synchronises cuda_stream.  Returns TO_NOT_CONVERGED (> 0) if the cap was
 * reached, TO_EBREAKDOWN / TO_ENAN / TO_ENONPOS_DIAG on numerical failure. */
int  tosolve_cg(to_mesh *m, double penal, const double *x_dev, double *u_dev,
                double rtol, int32_t max_iter, uint32_t flags, to_cg_stats *st,
                void *cuda_stream);

/* The paper's own solver (§5): MINRES (Paige-Saunders) on
 * the explicitly rescaled system K~ = D^-1/2 A D^-1/2 (:511-523), either with
 * the rescaling alone (TO_PC_JACOBI) or preconditioned by a zero-fill
 * incomplete Cholesky factor of K~ (TO_PC_IC0, :524-530; shifted on
 * breakdown, reading R24).  Krylov recycling (RMINRES) is not
 * implemented.  Starts from u = 0; stops when the M^-1-norm of the residual,
 * |eta|, falls to rtol times its initial value, or after max_iter steps
 * (TO_NOT_CONVERGED).  flags: TO_NO_TRUE_RES only.  Synchronises the stream. */
enum { TO_PC_JACOBI = 0, TO_PC_IC0 = 1 };
typedef struct {
  int32_t iters, status;
  double  eta_rel;             /* |eta_final| / |eta_0|                          */
  double  relres_true;         /* ||b - A u||_2 / ||b||_2 (-1 if skipped)         */
  double  ms;                  /* device time of the call                        */
  double  ic0_shift;           /* shift a of the IC(0) factor of K~ + a I (-1: none) */
  int32_t ic0_levels[2];       /* dependency levels of the forward / backward solves */
} to_minres_stats;
int  tosolve_minres(to_mesh *m, double penal, const double *x_dev, double *u_dev, double rtol,
                    int32_t max_iter, int32_t precond, uint32_t flags, to_minres_stats *st,
                    void *cuda_stream);

/* Residual history of the last TO_HISTORY solve: copies min(n, iters)
 * values of ||r_k||/||b|| (k = 1..iters) to host `out`; returns the count. */
int  tosolve_history(const to_mesh *m, double *out, int32_t n);

/* Per-kernel device time of the last TO_PROFILE solve, in ms, summed over
 * its iterations: out[0] operator apply (q = A p, with p.q), out[1] the
 * alpha reduction (0 when fused into the apply), out[2] r update + (r.z,
 * r.r), out[3] x/p update, out[4] number of iterations profiled; with
 * n >= 6, out[5] = the device time from the first to the last iteration
 * launch of a TO_PROFILE_LOOP solve (one event pair, no per-launch events). */
int  tosolve_profile(const to_mesh *m, double *out, int32_t n);

/* dc_dev[n_elem] = -p x^(p-1) (E0-Emin) u_e^T K0(h_e) u_e with u_e the element
 * gather of u_dev (already recovered, hanging values included).  If
 * compliance_host != NULL also computes f^T u and synchronises. */
int  to_sensitivity(to_mesh *m, double penal, const double *x_dev, const double *u_dev,
                    double *dc_dev, double *compliance_host, void *cuda_stream);

/* TO_FILTER_SENS: out_e = sum_d x_d H_de V_d in_d / (x_e sum_d H_de V_d)  (Eq. 5)
 * TO_FILTER_DENS: out_e = sum_d H_de V_d in_d / sum_d H_de V_d
 * H_de = rmin - |c_d - c_e| over the uploaded neighbour lists (Eq. 4).
 * out_dev must not alias in_dev or x_dev.  Asynchronous. */
int  to_filter(to_mesh *m, int32_t mode, const double *x_dev, const double *in_dev,
               double *out_dev, void *cuda_stream);

/* OC design update (reading R18), element-wise with V_e = (2^(L-l_e) h_L)^dim:
 *   x_new_e(lam) = min(min(1, x_e + move), max(max(rho_o, x_e - move),
 *                      x_e (max(-dc_e, 0) / (lam V_e))^eta))
 * with lam >= 0 such that sum_e V_e x_new_e = volfrac sum_e V_e: lam = 0 when
 * even the lam -> 0+ limit stays within the budget ("inactive"); else the
 * bracket [0, 1e9] (upper end widened x1e3 while still too much volume, up
 * to 1e300; if that never suffices: "infeasible", lam = the last upper end)
 * is bisected until l2 - l1 <= 1e-12 (l1 + l2) or 200 bisections.
 *   x_dev, dc_dev  [n_elem] densities (in [rho_o, 1]) and filtered
 *                  sensitivities (<= 0; positive values act as 0)
 *   volfrac        V0 in (0, 1]; move >= 0; eta > 0; rho_o in (0, 1)
 *   x_new_dev      [n_elem] output; may alias x_dev, must not alias dc_dev
 *   st             nullable; filled after synchronising cuda_stream
 * Returns TO_EINVAL for bad arguments, TO_ENAN if x or dc holds NaN/Inf. */
typedef struct {
  double  lambda;              /* volume multiplier (0 when inactive)            */
  double  volume;              /* sum V x_new / sum V                            */
  double  change;              /* max |x_new - x| (Condition 1)*/
  double  ms;                  /* device time of the call (CUDA events)          */
  int32_t steps;               /* bracket widenings + bisections                 */
  int32_t state;               /* 0 active, 1 inactive, 2 infeasible             */
  int32_t passes;              /* passes over the elements (grid-wide sums)      */
} to_oc_stats;
int  to_oc_update(to_mesh *m, const double *x_dev, const double *dc_dev, double volfrac,
                  double move, double eta, double rho_o, double *x_new_dev,
                  to_oc_stats *st, void *cuda_stream);

/* Dynamic AMR marking (§4, reading R21), one
 * int8 per element into marks_dev (device memory, [n_elem]):
 *   +1  a solid element (x_d >= rho_s) lies within r_amr of e (centre
 *       distance < r_amr, e itself included) and e is below max_level;
 *   -1  no solid element within r_amr and e is above level 0;
 *    0  otherwise.
 * r_amr is the handle's filter radius rmin ("we use rmin = r_amr",
 * PAPER.md:606-607), evaluated on the same neighbour lists / stencil as
 * to_filter; rmin = 0 means the element alone.  The marks feed
 * tomesh_host_adapt (include/tomesh_host.h).  Asynchronous. */
int  to_amr_mark(to_mesh *m, const double *x_dev, double rho_s, int8_t *marks_dev, void *cuda_stream);

/* The Fig. 1 optimization loop on the uploaded (fixed) mesh:
 * per step  tosolve_cg (warm-started from the previous u, :541-543) ->
 * to_sensitivity (+ compliance) -> to_filter SENS (Eq. 5, if filter and
 * rmin > 0) -> to_oc_update written in place into x_dev.  p-continuation
 * (:331-333, reading R19): p starts at penal0 and rises by
 * penal_step (capped at penal_max) after a step whose design change is
 * < change_tol (Condition 1, :431-434) or after stage_steps steps at the
 * current p.  With stop_on_converge the loop ends after the first step at
 * p = penal_max with change < change_tol.  Mesh adaptation (Fig. 1's
 * refine/derefine branch) is not part of this call.
 *   x_dev      [n_elem] in: initial design; out: the final design
 *   u_dev      [dim*n_node] out: displacement of the last solve
 *   hist       nullable [n_steps] per-step record; *steps_done = steps run
 *   state      nullable continuation / adaptation state carried across calls
 *              (NULL: start at penal0 with fresh counters)
 * The first solve of a call starts from zero (after an adaptation the mesh
 * changed); later ones are warm-started.  Synchronises cuda_stream every step.  Returns the first failing status of
 * a step (< 0), TO_NOT_CONVERGED if some solve hit max_iter, else TO_OK. */
typedef struct {
  double  volfrac, move, eta, rho_o;        /* to_oc_update (reading R18)        */
  double  penal0, penal_max, penal_step;    /* continuation (reading R19)        */
  int32_t stage_steps, stop_on_converge;
  double  change_tol;                       /* Condition 1 (0.01)                */
  double  rtol;                             /* per solve                         */
  int32_t max_iter, filter;                 /* filter = 1: Eq. 5 on dc           */
  int32_t adapt_min_steps, adapt_max_steps; /* > 0: stop after the step at which
                                               the AMR trigger fires (PAPER.md:
                                               421-446, reading R23): change <
                                               change_tol and >= min steps since
                                               the last adaptation, or >= max   */
} to_opt_params;
typedef struct {
  double  penal;          /* in/out: current SIMP exponent                       */
  int32_t at_stage;       /* in/out: steps taken at the current exponent         */
  int32_t since_adapt;    /* in/out: steps since the last mesh adaptation        */
  int32_t adapt_due;      /* out: 1 = stopped because the AMR trigger fired      */
  int32_t converged;      /* out: 1 = stopped by stop_on_converge                */
} to_opt_state;
typedef struct {
  double  compliance;          /* f^T u at the design entering the step          */
  double  penal, volume, change, lambda;
  double  solve_ms, oc_ms;     /* device times (CUDA events)                     */
  int32_t cg_iters, status;    /* solve iterations and status                    */
} to_opt_step;
int  to_optimize(to_mesh *m, const to_opt_params *params, int32_t n_steps, double *x_dev,
                 double *u_dev, to_opt_step *hist, int32_t *steps_done, to_opt_state *state,
                 void *cuda_stream);

/* ---- z-slab sharding of the structured path (one handle per
 * slab and per GPU) -----------------------------------------------
 * The path shards with "one exchange step per matvec plus scalar reductions":
 * the mesh is cut into slabs of node planes along z; rank r OWNS the global
 * node planes [a_r, b_r) and its handle is uploaded (tomesh_upload) with the
 * uniform sub-box of element layers [a_r - 2, b_r + 1) (clipped to the mesh),
 * i.e. two ghost node planes on each interior side, its loads and Dirichlet
 * DOFs sliced from the global problem.  The exchange is fused into the
 * iteration kernel (the owners of the boundary planes store r, p and q into
 * the neighbour's ghost plane: NVLink peer stores when the neighbour is
 * another GPU) and every scalar reduction is a device-side all-reduce (each
 * rank pushes its partials into every rank's slots, flags with release
 * semantics, the ranks sum the slots in rank order), so every rank takes the
 * same alpha, beta and stop decision and no host sync is added.
 *
 * to_shard_buffers  fills this handle's exchange buffers (device addresses on
 *                   its device; allocates the slots on first use).  Share them
 *                   with the other ranks: directly within one process, through
 *                   to_ipc_export / to_ipc_open across processes.
 * to_shard_attach   makes the handle rank `rank` of `nranks` (<= TO_SHARD_MAX):
 *                   gz_lo[r] = global node plane of rank r's local plane 0,
 *                   [own_lo, own_hi) = this rank's owned LOCAL planes (>= 2;
 *                   rank 0 starts at 0, the last rank ends at its last plane,
 *                   interior sides need two ghost planes), peers[r] = rank r's
 *                   buffers as addressable from this handle's device (peers[rank]
 *                   = its own).  Peer access is enabled to every other device a
 *                   peer buffer lives on (one process, several GPUs).  TO_EINVAL
 *                   on any inconsistency.  Synchronises.
 * tosolve_cg_group  tosolve_cg on n attached handles of one group in
 *                   lockstep (n = nranks in one process: several GPUs, or all
 *                   slabs on one GPU; n = 1 per process when each rank runs in
 *                   its own process).  Every rank of the group must make the
 *                   same sequence of group calls.  x_dev[i] are the local
 *                   element densities, u_dev[i] receives the local u: owned
 *                   planes and the ghost planes the sensitivities and filter of
 *                   the owned elements need (a-1, b, b+1).  flags: TO_FIXED_ITERS,
 *                   TO_HISTORY, TO_PROFILE_LOOP, TO_NO_TRUE_RES (the true residual is
 *                   not computed: relres_true = -1).  A rank that waits ~20 s
 *                   for a peer fails with TO_ECUDA instead of hanging.
 *                   Synchronises every stream.  st[i] per handle (identical
 *                   iteration counts and residuals on every rank).
 * After a group solve, to_sensitivity and to_filter on each handle are exact on
 * its owned elements (the element layers [a_r, b_r)), and to_sensitivity's
 * compliance_host is this rank's partial sum of f.u over its owned DOFs (the
 * compliance is the sum over ranks). */
#define TO_SHARD_MAX 16
typedef struct {
  double *rb[2], *pb[2], *qb[2];   /* internal CG vectors (ping-pong)                  */
  double *x;                       /* internal iterate                                 */
  double *slots;                   /* [4][TO_SHARD_MAX][8] all-reduce slots            */
  unsigned long long *flags;       /* [4][TO_SHARD_MAX] sequence flags                 */
  int32_t nx, ny, nz;              /* node box of the handle (0: general handle)        */
  int32_t pad;
  int64_t plane_doubles;           /* doubles per internal node plane (0: general)     */
  double *dinv;                    /* Jacobi inverse diagonal (general handles)         */
} to_shard_bufs;
int  to_shard_buffers(to_mesh *m, to_shard_bufs *out, void *cuda_stream);

/* ---- Morton node-range sharding of the general (AMR) path ------
 * Rank r's handle is uploaded with its local mesh (paper_1009_4975_b200/
 * amr_shard.py): its owned nodes first (to_mesh_desc.n_owned), then the ghosts
 * (the other corners of its elements and the parents of its hanging corners),
 * then its non-owned hanging nodes; every element contributing to an owned
 * node (directly or through a hanging corner, Eq. 6).  The iteration kernel
 * computes the owned nodes; after it, every rank stores r_k, p_k, q_k of the
 * nodes its peers hold as ghosts into their buffers (peer stores) and pushes
 * its partial dots (the same slot / flag all-reduce as the z-slab path), so
 * the next iteration reads complete ghosts and every rank takes the same step.
 * Jacobi diagonal and b at the ghosts come from their owners once per solve,
 * and x after it (sensitivities of every local element are then exact).
 * to_gshard_attach  makes a general handle rank `rank` of `nranks`: send
 *                   entry i stores this rank's owned local node send_local[i]
 *                   into ghost node send_remote[i] of rank send_rank[i];
 *                   peers[r] = rank r's to_shard_buffers.  Synchronises.
 * tosolve_cg_group drives attached general handles the same way as slabs; the
 * filter is not sharded (handles are uploaded with rmin = 0), and
 * to_sensitivity's compliance_host is the rank's partial over owned DOFs. */
int  to_gshard_attach(to_mesh *m, int32_t rank, int32_t nranks, const to_shard_bufs *peers, int64_t n_send,
                      const int32_t *send_rank, const int32_t *send_local, const int32_t *send_remote,
                      void *cuda_stream);
int  to_shard_attach(to_mesh *m, int32_t rank, int32_t nranks, const int32_t *gz_lo, int32_t own_lo,
                     int32_t own_hi, const to_shard_bufs *peers, void *cuda_stream);
int  tosolve_cg_group(to_mesh *const *ms, int32_t n, double penal, const double *const *x_dev,
                      double *const *u_dev, double rtol, int32_t max_iter, uint32_t flags,
                      to_cg_stats *st, void *const *cuda_streams);
/* CUDA IPC of a device buffer of the handle (any address inside one of its
 * allocations): 64-byte handle + byte offset; to_ipc_open maps it on `device`
 * (peer access enabled lazily) and returns the address of the same byte;
 * to_ipc_close unmaps (pass the opened address minus the offset). */
int  to_ipc_export(to_mesh *m, const void *dev_ptr, void *handle64, uint64_t *offset);
int  to_ipc_open(int device, const void *handle64, uint64_t offset, void **dev_ptr);
int  to_ipc_close(int device, void *base_ptr);

/* Operator-level entry points (parity and diagnostics; asynchronous).
 * to_apply_A:      q = A v,  A = Pi_F C^T K(x) C Pi_F + (I - Pi_F)  (Eq. 8)
 * to_jacobi_diag:  d = diag(A)  (1 on hanging and fixed DOFs)
 * to_project_rhs:  b = Pi_F C^T f  (Eq. 7 right-hand side)
 * to_recover:      u = C v  (Eq. 9); in place allowed (u_dev == v_dev) */
int  to_apply_A(to_mesh *m, double penal, const double *x_dev, const double *v_dev,
                double *q_dev, void *cuda_stream);
int  to_jacobi_diag(to_mesh *m, double penal, const double *x_dev, double *d_dev,
                    void *cuda_stream);
int  to_project_rhs(to_mesh *m, double *b_dev, void *cuda_stream);
int  to_recover(to_mesh *m, const double *v_dev, double *u_dev, void *cuda_stream);

/* Host-only diagnostics (no GPU needed): the unit element matrix K0 the
 * kernels use (E = 1, h = 1, closed form of csrc/element.cpp), dim*2^dim
 * square, row-major, local DOF = dim*corner + component; and, for dim = 3,
 * its Hadamard factorisation (diag[3][8], off[3][3][8], see csrc/element.h).
 * Returns 0, or the number of entries violating the factorisation pattern. */
int  to_element_matrix(int32_t dim, double nu, double *K_host);
int  to_element_hadamard(double nu, double *diag_host, double *off_host);

/* Thread-local message describing the last failure ("" if none). */
const char *to_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TOMESH_H */
