/*
 * bspde_b200.h -- C ABI of the B200 (sm_100a) tensor B-spline heat/elliptic
 * solve path.  Plain pointers, sizes and a cudaStream_t passed as void*;
 * no torch types.  Every entry point returns 0 on success and a nonzero
 * BSPDE_ERR_* code on failure; bspde_last_error() returns the message of the
 * calling thread's last failure.
 *
 * The reference (arxiv/paper_1904_03057, package `bspde`, pure Python) has
 * no FFI; these entry points replace the numeric calls of its operator
 * protocol and solver.  Each declaration names the reference interface it
 * replaces (paths relative to /root/reference/pkg/src/bspde/).
 *
 * Device field layout ("ghosted slab"): a field of the local extended
 * coefficient grid (nz owned z-planes, ny rows, nx columns; reference array
 * axes (axis0, axis1, axis2) = (z, y, x), x contiguous) is stored as
 *     double buf[nz + 2*ghost][ny][pitch_y]     (pitch_z = ny * pitch_y)
 * with ghost == degree.  Owned plane k lives at buffer plane k + ghost.
 * Ghost planes hold the neighbouring slab's planes (multi-GPU z-slabs) or
 * zeros at a physical domain end; they are read, never written, by the
 * kernels.  pitch_y is even (16-byte rows, a TMA requirement); columns
 * nx..pitch_y-1 are ignored.  All pointers passed below are the buffer base
 * (first ghost plane), 16-byte aligned, device memory.
 */
#ifndef BSPDE_B200_H
#define BSPDE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CG search directions live in a ring of R ghosted-slab fields (one
 * contiguous allocation, field after field; R = bspde_cg_config.p_ring, 2 or
 * BSPDE_P_RING): iteration k reads p_{k-1} from field (k-1) % R and writes
 * p_k to field k % R.  Pass A of iteration k also applies x += alpha_{k-1}
 * p_{k-1} (it stages p_{k-1} anyway), in the reference's rounding order
 * (solver.py:94); the last iteration's update is applied at the end of a
 * solve (bspde_cg_flush_x).  R = 2 suffices (the default). */
#define BSPDE_P_RING 4

#define BSPDE_OK 0
#define BSPDE_ERR_ARG 1      /* invalid argument (ValidationError) */
#define BSPDE_ERR_CUDA 2     /* CUDA runtime / driver failure */
#define BSPDE_ERR_STATE 3    /* API misuse */

/* CG status codes (bspde_cg_report.status) */
#define BSPDE_CG_RUNNING 0
#define BSPDE_CG_CONVERGED 1
#define BSPDE_CG_MAXITER 2
#define BSPDE_CG_INDEFINITE 3 /* IndefiniteOperatorError, solver.py:88-92 */
#define BSPDE_CG_DIVERGED 4   /* DivergenceError, solver.py:105-108 */
#define BSPDE_CG_ZERO_RHS 5   /* early return, solver.py:63-67 */

typedef struct bspde_plan bspde_plan; /* opaque */

/*
 * Operator description.  Replaces the data an OnTheFlyOperator reads from
 * SystemData (assembly.py:342-389) for constant D / mu on a box domain with
 * Neumann faces:
 *   A = Mz(x)(My(x)(c_mass Mx + c_stiff[2] Kx) + c_stiff[1] Ky(x)Mx)
 *       + c_stiff[0] Kz(x)My(x)Mx
 * with c_mass = vol*mu and c_stiff[a] = vol*D/h_a^2 (assembly.py:426-433).
 * Per axis a (0=z, 1=y, 2=x) the banded Gram factor is given in class form:
 * table[c*(2p+1) + k+p] = G[i, i+k] for rows i of class c, classes
 * 0..ew-1 = first rows, ew = interior (Toeplitz), ew+1..2ew = last rows.
 * inv_diag_table[(cz*NCy + cy)*NCx + cx] (NCa = 2*ew[a]+1) is the Jacobi
 * preconditioner 1/diag (1 where diag == 0, solver.py:69-73) per class triple.
 * Box-face Robin / penalty terms (assembly.py:201-232) arrive folded into
 * the edge-row classes of stiff_table (the interior row must stay the
 * Toeplitz taps: the kernels use compile-time interior taps).
 */
typedef struct {
  int32_t device;       /* CUDA device ordinal the plan (and its launches) use */
  int32_t degree;       /* p in 1..5 */
  int32_t nz, ny, nx;   /* local extents: owned z planes, rows, columns */
  int32_t nz_global;    /* global extended z extent */
  int32_t z_offset;     /* global z index of owned plane 0 */
  int32_t ew[3];        /* edge rows per axis end (z, y, x) */
  int64_t pitch_y;      /* elements between rows (even, >= nx) */
  const double* mass_table[3];  /* host, (2ew+1)*(2p+1) each */
  const double* stiff_table[3]; /* host, same shape */
  const double* inv_diag_table; /* host, NCz*NCy*NCx */
  double c_mass;
  double c_stiff[3];
} bspde_plan_desc;

typedef struct {
  double tol;
  int32_t max_iter;
  int32_t record_history;
  int32_t has_x0;       /* 0: x0 = None (x is zeroed), 1: x holds x0 */
  int32_t poll_every;   /* iterations per CUDA-graph chunk between host polls (<=0: default 8) */
  int32_t p_ring;       /* search-direction ring length R: 2 or 4 (0: 2) */
} bspde_cg_config;

typedef struct {
  int32_t iterations;
  int32_t status;       /* BSPDE_CG_* */
  double relative_residual;
  double residual;
  double residual0;
  double rhs_norm;
  double last_pAp;      /* curvature at failure (indefinite) */
} bspde_cg_report;

/* ---- library ---------------------------------------------------------- */
const char* bspde_last_error(void);
int bspde_version(void);
/* 1 if CUDA device `device` exists and has compute capability 10.x, else 0. */
int bspde_device_ok(int device);

/* ---- plan: replaces make_operator(data, strategy) (operator.py:407-414) */
int bspde_plan_create(const bspde_plan_desc* desc, bspde_plan** out);
int bspde_plan_destroy(bspde_plan* plan);
/* Bytes of device scratch (CG scalar state, per-CTA partials, counters). */
int64_t bspde_scratch_bytes(const bspde_plan* plan);
/* Number of kernel launches issued by this plan since creation. */
int64_t bspde_launch_count(const bspde_plan* plan);

/* out = A c.  Replaces OnTheFlyOperator.apply (operator.py:217-229). */
int bspde_apply(bspde_plan* plan, const double* c, double* out, void* stream);

/* out = cm * (Mz(x)My(x)Mx) c + a * f   (f may be NULL).
 * Replaces assembled_rhs(data, n_s=p, q) * (operator.py:417-441) for a box
 * with Neumann faces (cm = vol), and the heat RHS  M u_prev + dt F. */
int bspde_mass_apply(bspde_plan* plan, const double* c, const double* f,
                     double cm, double a, double* out, void* stream);

/* out = diag(A) on the owned region.
 * Replaces _OperatorBase.jacobi_diagonal (operator.py:156-171). */
int bspde_jacobi_diagonal(bspde_plan* plan, const double* diag_table,
                          double* out, void* stream);

/* Full Jacobi-PCG on one device.  Replaces pcg(operator, rhs, config, x0)
 * (solver.py:51-117): identical recurrence, stopping rule (recursive
 * ||r||/||b|| <= tol or max_iter), indefinite and divergence guards.
 * b, x, r, ap are ghosted-slab fields, p_ring cfg->p_ring of them back to
 * back (the search directions); b may alias ap (b is only read by the
 * initial residual, before the first Ap is written); x holds x0 on entry when
 * cfg->has_x0, the solution on exit.  scratch: bspde_scratch_bytes bytes.
 * history: device array of max_iter+1 doubles or NULL. */
int bspde_pcg_solve(bspde_plan* plan, const double* b, double* x, double* r,
                    double* p_ring, double* ap, void* scratch, double* history,
                    const bspde_cg_config* cfg, bspde_cg_report* report,
                    void* stream);

/* One implicit-Euler heat step: solves (M + dt K) u_new = cm M u + a f with
 * x0 = u (Jacobi-PCG as bspde_pcg_solve), u updated in place.  The right-hand
 * side is never formed: the first residual r0 = (cm M u + a f) - A u and its
 * sums come from one fused kernel (the mass apply rides along as a second
 * z ring; b = cm M u + a f is rounded as bspde_mass_apply rounds it).
 * f may be NULL (no source).  cfg->has_x0 must be 1.  Replaces the
 * composition b = M.apply(u) + dt F; pcg(A, b, cfg, x0 = u) of the heat
 * oracle (solver.py:51-117). */
int bspde_heat_step(bspde_plan* plan, double* u, const double* f, double cm, double a,
                    double* r, double* p_ring, double* ap, void* scratch, double* history,
                    const bspde_cg_config* cfg, bspde_cg_report* report, void* stream);
/* The fused first residual alone (step-wise / tests): r = (cm M u + a f) - A u,
 * sums = {<b,b>, <r,D^-1 r>, <r,r>} of that b (kind 0). */
int bspde_heat_residual(bspde_plan* plan, const double* u, const double* f, double cm,
                        double a, double* r, void* scratch, int fuse, void* stream);

/* ---- step-wise CG for the multi-GPU driver (z-slabs, one rank per GPU).
 * fuse = 1: the kernel's last CTA reduces the per-CTA partials and runs the
 * scalar update (single device).  fuse = 0: it only writes this rank's sums
 * as double-double pairs (the first 64 bytes of scratch: 4 hi, then 4 lo);
 * one rank calls bspde_cg_finalize(kind), N ranks all-gather those 64 bytes
 * and call bspde_cg_finalize_gathered(kind) -- the scalars, hence the
 * iterates, are then bit-identical to the single-device solve. */
int bspde_cg_setup(bspde_plan* plan, void* scratch, double* history,
                   const bspde_cg_config* cfg, void* stream);
/* r = b - A x (x = x0 or zero), sums = {<b,b>, <r,D^-1 r>, <r,r>}   kind 0 */
int bspde_cg_residual(bspde_plan* plan, const double* b, const double* x,
                      double* r, void* scratch, int fuse, void* stream);
/* p_k = D^-1 r + beta p_{k-1} on the fly (written to p_out at owned
 * points); ap = A p_k; sums = {<p,Ap>}; and, for k >= 1, x += alpha_{k-1}
 * p_{k-1} at the owned points (solver.py:94; p_in = p_{k-1})       kind 1
 * p_in / p_out ping-pong between iterations (they must differ); at k = 0
 * (beta = 0) p_in only needs finite values (the drivers pass r). */
int bspde_cg_pass_a(bspde_plan* plan, double* x, const double* r, const double* p_in,
                    double* p_out, double* ap, void* scratch, int fuse,
                    void* stream);
/* Pass A restricted to the owned output planes [z_begin, z_begin + z_count)
 * (local indices; it streams the p planes either side).  accumulate = 1 adds
 * the range's <p,Ap> to the sums instead of overwriting them.  The z-slab
 * driver runs the interior range [p, nz - p) -- which reads no ghost plane --
 * while the NCCL halo exchange is in flight, then the two boundary ranges
 * (overlap the halo with the interior apply).  The reference
 * analogue is a worker's window of blocks (operator.py:61-74). */
int bspde_cg_pass_a_range(bspde_plan* plan, double* x, const double* r,
                          const double* p_in, double* p_out, double* ap, void* scratch,
                          int z_begin, int z_count, int accumulate, int fuse,
                          void* stream);
/* r -= alpha Ap; sums = {<r,D^-1 r>, <r,r>} (solver.py:95-101; x moves in
 * the next pass A).  Iteration k's pass A must read ring field (k-1) % R and
 * write field k % R (R = the p_ring given to bspde_cg_setup).        kind 2 */
int bspde_cg_pass_b(bspde_plan* plan, double* r, const double* ap, void* scratch,
                    int fuse, void* stream);
/* Apply the pending x update (x += alpha_j p_j for the last iteration,
 * which no further pass A applies).  bspde_pcg_solve does this itself;
 * step-wise drivers call it once after their loop (idempotent). */
int bspde_cg_flush_x(bspde_plan* plan, double* x, const double* p_ring,
                     void* scratch, void* stream);
/* kind 0/1/2: scalar update after residual / pass A / pass B (skipped when
 * inactive); kind 3 is used internally by bspde_cg_flush_x. */
int bspde_cg_finalize(bspde_plan* plan, void* scratch, int kind, void* stream);
/* N-rank scalar update: `gathered` = the rank-major all-gather (world x 8
 * doubles) of every rank's first 64 scratch bytes; the pairs are summed in
 * rank order in double-double and rounded once (kind 0..2). */
int bspde_cg_finalize_gathered(bspde_plan* plan, void* scratch, const void* gathered,
                               int world, int kind, void* stream);
/* ---- z-slab peer halos (NVLink peer memory / CUDA IPC) ------------------
 * With peers set, the step-wise pass B stores the new r of its first / last
 * p owned planes into the lower / upper neighbour's r ghost planes, and the
 * preceding pass A's p_k of those planes into the neighbours' ghost planes
 * of the same ring field (k % R): the compute kernels carry the halo
 * exchange (no separate transfer per iteration).  The scalar all-gather
 * after pass B orders those stores before the neighbours' next pass A.  The
 * reference analogue is the worker windows' halo (operator.py:61-74). */
typedef struct {
  const double* ring;        /* this rank's p ring: ring_len fields, ring_stride doubles apart */
  const double* r;           /* this rank's r */
  long long ring_stride;
  int ring_len;
  int lo_nz;                 /* owned planes of the lower neighbour */
  double* lo_ring;           /* lower neighbour (NULL: none) */
  long long lo_ring_stride;
  double* lo_r;
  double* hi_ring;           /* upper neighbour (NULL: none) */
  long long hi_ring_stride;
  double* hi_r;
} bspde_slab_peers;
/* NULL clears. */
int bspde_slab_set_peers(bspde_plan* plan, const bspde_slab_peers* peers);
/* CUDA IPC of a device pointer inside a cudaMalloc'd block: 64-byte handle of
 * the block + the pointer's offset; import maps it (peer access enabled
 * lazily) and returns the pointer; close unmaps. */
int bspde_ipc_export(const void* ptr, void* handle64, uint64_t* offset);
int bspde_ipc_import(const void* handle64, uint64_t offset, void** ptr);
int bspde_ipc_close(void* ptr);
/* Copy the scalar state to the host (synchronizes the stream). */
int bspde_cg_read_report(bspde_plan* plan, const void* scratch,
                         bspde_cg_report* report, int32_t* active, void* stream);

/* ---- B-spline field transforms (setup / I/O; plan-free) ------------------
 * Direct transform (node samples -> coefficients) of lines of a strided
 * 3-D array, in place: line (a, b) starts at data + a*sa + b*sb and has n
 * elements at the given stride; a varies fastest across threads.  Replaces
 * _prefilter_lines (bspline.py:168-211) with its rounding order.  poles /
 * gain as compute_poles(degree) (bspline.py:140-155, np.roots values);
 * extension 0 = mirror, 1 = replicate, 2 = zero (direct_transform's
 * policies).  npoles = 0 (degree <= 1) is a no-op. */
int bspde_prefilter_lines(double* data, int32_t n, int64_t stride, int32_t na,
                          int32_t nb, int64_t sa, int64_t sb, const double* poles,
                          int32_t npoles, double gain, int32_t extension,
                          void* stream);
/* np.pad(..., ext, mode="reflect") along one axis of a 3-D array whose inner
 * region [ext, dims[axis]-ext) is filled (transform_field, problem.py:178-194). */
int bspde_reflect_pad(double* data, const int32_t* dims, const int64_t* strides,
                      int32_t axis, int32_t ext, void* stream);
/* In place along lines (same addressing as bspde_prefilter_lines): solve the
 * banded system L U x = x with DEVICE factors lb[n][m] (L[i, i-k], unit
 * diagonal) and ub[n][m+1] (U[i, i+k]) -- the mirror-folded Gram system of the
 * "l2" prefilter (_l2_project_axis, problem.py:142-175); m <= 8. */
int bspde_banded_solve_lines(double* data, int32_t n, int64_t stride, int32_t na, int32_t nb,
                             int64_t sa, int64_t sb, const double* lb, const double* ub,
                             int32_t m, void* stream);
/* out[.., i, ..] = sum_t w[i*ntaps + t] * in[.., idx[i*ntaps + t], ..] along
 * one axis (idx, w: DEVICE arrays, extension policy folded into idx): the
 * spline evaluation of indirect_transform (bspline.py:245-310) on a lattice of
 * points, one axis per call; ntaps <= 11. */
int bspde_resample_axis(const double* in, const int64_t* in_strides, double* out,
                        const int32_t* out_dims, const int64_t* out_strides, int32_t axis,
                        const int32_t* idx, const double* w, int32_t ntaps, void* stream);
/* out[q] = sum_{a,b,k} wz[q,a] wy[q,b] wx[q,k] c[iz[q,a], iy[q,b], ix[q,k]] for
 * npts scattered points (indirect_transform, bspline.py:253-310): idx / w are
 * DEVICE arrays [3][npts][ntaps] (axis 0, 1, 2; extension folded into idx),
 * c a 3-D array with the given element strides; ntaps <= 11. */
int bspde_eval_points(const double* c, const int64_t* strides, int64_t npts, int32_t ntaps,
                      const int32_t* idx, const double* w, double* out, void* stream);
/* out[i] = sum_t taps[t] * in[i + offset + t] along one axis (sample_solution,
 * problem.py:330-348; accumulated in the reference's order), ntaps <= 11. */
int bspde_fir_axis(const double* in, const int64_t* in_strides, double* out,
                   const int32_t* out_dims, const int64_t* out_strides, int32_t axis,
                   int32_t offset, const double* taps, int32_t ntaps, void* stream);

/* ---- variable-coefficient operator ---------------
 * The reference's on-the-fly operator for spline-valued diffusion D(x) and
 * absorption mu(x) fields (operator.py:217-229, stencil_block
 * assembly.py:460-472): per node l the (2p+1)^3 stencil
 *   P[a, l] = sum_b [ D[l+b] (sz Tz'Ty Tx + sy Tz Ty' Tx + sx Tz Ty Tx')[a, b]
 *                   + mu[l+b] sm (Tz Ty Tx)[a, b] ]
 * from per-axis trilinear tables (kernels.py:158-173, edge rows
 * assembly.py:83-108), assembled once into HBM and applied as
 * t_l = sum_a P[a, l] c[l + a].  Box domains in 1-3 D (unit axes, see
 * `degenerate`), optional Robin /
 * penalty face terms.
 * Fields are dense (z, y, x) arrays (x fastest) on the device. */
typedef struct bspde_stencil bspde_stencil;

typedef struct {
  int32_t device;
  int32_t degree;        /* n_b in 1..5 */
  int32_t param_degree;  /* n_p in 0..5 (degree of the D / mu fields) */
  int32_t nz, ny, nx;    /* coefficient (extended) extents */
  int32_t pz, py, px;    /* parameter-field (extended) extents */
  int32_t ext, ext_p;    /* basis_extension(n_b), basis_extension(n_p) */
  int32_t ew[3];         /* edge rows per axis end */
  /* host: per axis, [0] = value/value, [1] = derivative/derivative trilinear
   * class tables, (2ew+1) x (2n_b+1) x (2mw+1), mw = (n_b+n_p+1)/2 */
  const double* tables[3][2];
  double scale_stiff[3]; /* vol / h_a^2 */
  double scale_mass;     /* vol */
  /* box-face Robin / penalty terms (make_face_term, assembly.py:201-232):
   * P += weight * (v v^T)_axis (x) (h M)_other axes */
  int32_t nfaces;        /* 0..6 */
  int32_t face_axis[6], face_side[6];
  double face_weight[6];
  const double* face_values;  /* host, ew values of the low face (high face mirrored) */
  const double* mass_gram;    /* host, unit mass Gram class table (2ew+1) x (2n_b+1) */
  double step[3];
  /* 1-D / 2-D problems ride as 3-D with unit leading axes: degenerate[a] = 1
   * marks such an axis (extent 1, no extension, tables the identity factor:
   * value class table 1 at (a = 0, b = 0), derivative table 0, step 1) */
  int32_t degenerate[3];
} bspde_stencil_desc;

int bspde_stencil_create(const bspde_stencil_desc* desc, bspde_stencil** plan);
int bspde_stencil_destroy(bspde_stencil* plan);
/* number of doubles of the stencil array P ((2p+1)^3 * rows) */
int64_t bspde_stencil_entries(const bspde_stencil* plan);
/* Compact mode (mask domains): store and iterate only the nact active rows
 * (device array of their dense indices, ascending, kept alive by the caller)
 * -- P[a * nact + k]; the vectors stay dense and their inactive entries are
 * never written (inactive entries of a right-hand side must be zero, as the
 * reference's _mask_rhs_fixup makes them, operator.py:444-459).  Call before
 * bspde_stencil_assemble; the 600 x 600 x 2400 leg needs ~40 GB instead of
 * 187 GB of stencil. */
int bspde_stencil_set_rows(bspde_stencil* plan, const int64_t* rows, int64_t nact);
int64_t bspde_stencil_launch_count(const bspde_stencil* plan);
/* P <- stencils of all nodes from the parameter fields (device, dense) */
int bspde_stencil_assemble(bspde_stencil* plan, const double* dfield,
                           const double* mfield, double* P, void* stream);
/* out = A c (OnTheFlyOperator.apply) */
int bspde_stencil_apply(bspde_stencil* plan, const double* P, const double* c,
                        double* out, void* stream);
/* out = diag(A) (_diagonal_from_bands) */
int bspde_stencil_diagonal(bspde_stencil* plan, const double* P, double* out,
                           void* stream);
/* Jacobi-PCG (solver.py:51-117; precond 1 = jacobi, 0 = none) on dense
 * fields; scratch: bspde_scratch_bytes-sized (any plan). */
int bspde_stencil_pcg(bspde_stencil* plan, const double* P, const double* b,
                      double* x, double* r, double* p, double* ap, void* scratch,
                      double* history, const bspde_cg_config* cfg,
                      bspde_cg_report* report, int32_t precond, void* stream);

/* ---- matrix-free ("on-the-fly") variable-coefficient operator -------------
 * The reference's OnTheFlyOperator (operator.py:217-229; stencil_block /
 * term_stencil, assembly.py:280-297, :460-472) without any stored stencil:
 * a sum-factorised z-streaming kernel rebuilds every node's stencil action
 * from the D / mu fields and the trilinear tables on each apply (32 B/DoF of
 * HBM traffic, no (2p+1)^3 per-node array).  3-D boxes, no face terms,
 * n_b = n_p <= 3 (bspde_otf_supported); the plan is a bspde_stencil plan.
 * prepare: keeps the device field pointers (dense parameter-grid arrays,
 * alive while the plan is used) and writes the Jacobi diagonal into diag
 * (N doubles, kept and used by the PCG). */
int bspde_otf_supported(const bspde_stencil* plan);
int bspde_otf_prepare(bspde_stencil* plan, const double* dfield, const double* mfield,
                      double* diag, void* stream);
/* out = A c.  Replaces OnTheFlyOperator.apply (operator.py:217-229). */
int bspde_otf_apply(bspde_stencil* plan, const double* c, double* out, void* stream);
/* Jacobi-PCG with the matrix-free apply (same recurrence and state as
 * bspde_stencil_pcg).  Replaces pcg over OnTheFlyOperator (solver.py:51-117). */
int bspde_otf_pcg(bspde_stencil* plan, const double* b, double* x, double* r, double* p,
                  double* ap, void* scratch, double* history, const bspde_cg_config* cfg,
                  bspde_cg_report* report, int32_t precond, void* stream);

/* ---- mask (voxel) domains ------------------------
 * Replaces the reference's boundary-stencil machinery for MaskDomain
 * systems: _attach_mask_boundary (assembly.py:538-637), the exposed-face
 * surface terms _attach_mask_surface (:657-737) and the row patch
 * _patch_boundary_rows (operator.py:142-154).  After bspde_stencil_assemble
 * with free-space tables (ew = 0), bspde_stencil_mask_patch zeroes the rows
 * of inactive nodes and rebuilds the rows of boundary nodes from the
 * occupied cells of their support:
 *   P[a, l] = sum_{occupied c} sum_b f[c+b] (per-axis cell tables)[l+a-c, l-c, b]
 *           + weight * sum_{exposed faces} (v v)_normal (x) R_tangential.
 * All pointers in the desc are DEVICE pointers except where noted. */
typedef struct {
  const uint8_t* occupancy;   /* cells (cz, cy, cx), nonzero = occupied */
  int32_t cells[3];           /* cz, cy, cx (= node extents - 1) */
  const uint8_t* node_class;  /* nz*ny*nx: 0 inactive, 1 interior, 2 boundary */
  const int64_t* brows;       /* flat extended indices of the boundary nodes */
  int64_t nbrows;
  const int64_t* brows_k;     /* compact plans: each boundary row's slot in the active-row list */
  int32_t jlo, nj;            /* cell_node_offsets(n_b) = jlo .. jlo+nj-1 */
  int32_t blo, nbp;           /* cell_node_offsets(n_p) */
  const double* cell_tri;     /* [2][nj][nj][nbp]: value / derivative cell tables */
  const double* cell_bil;     /* [nj][nj] cell bilinear (n_b, n_b) */
  const double* cell_single;  /* [nj] single-spline cell integrals */
  const double* face_vals;    /* [2fc-1] spline values at a cell face */
  int32_t fc;                 /* first_clean_position(n_b) */
  int32_t has_surface;        /* exposed-face terms with one global weight */
  double surface_weight;
  int32_t degenerate[3];      /* unit axes of a 1-D / 2-D mask (one cell layer) */
} bspde_mask_desc;

int bspde_stencil_mask_patch(bspde_stencil* plan, const bspde_mask_desc* mask,
                             const double* dfield, const double* mfield, double* P,
                             void* stream);
/* out[l] += value * weight * (exposed-face single integrals) on boundary rows
 * (the surface_rhs_entries of assembly.py:728-737) */
int bspde_stencil_mask_surface_rhs(bspde_stencil* plan, const bspde_mask_desc* mask,
                                   double value, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BSPDE_B200_H */
