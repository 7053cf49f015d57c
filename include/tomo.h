/*
 * tomo.h — C ABI of libtomo: the exact-gradient evaluation of arXiv 2104.12282 (ONSG)
 * on one B200 (sm_100a).
 *
 * The paper's ONSG method exists to skip this evaluation: "to compute the gradient g^(k),
 * one needs to first solve u^(k) through K(z^(k))u - f = 0, which is very computationally
 * expensive ... Iterative solvers such as preconditioned conjugate gradient (PCG) ... are
 * typically used" (§"ONSG for Computational Morphogenesis", Eq. 5);
 * "The standard optimizer uses the PCG method with the Jacobi preconditioner" (PAPER.md
 * l.240). One evaluation = Jacobi-PCG solve of K(rho)u = f on a structured grid of 8-node
 * trilinear hexahedra (SIMP: E = Emin + rho^p (E0 - Emin)), compliance c = f^T u (Eq. 4,
 * PAPER.md l.175), sensitivity dc_e = -p rho_e^(p-1) (E0-Emin) u_e^T KE u_e (Eq. 5, PAPER.md
 * l.181-183), the density filter P / P^T and the optimality-criteria
 * (OC) update. Interpretations of what the paper leaves open are the
 * readings A1-A23 listed in DESIGN.md §3.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Grid      nelx x nely x nelz unit hexahedra of edge h; x is the beam axis, z vertical.
 *            Node (i,j,k) -> n = i + (nelx+1)*(j + (nely+1)*k); element (i,j,k) ->
 *            e = i + nelx*(j + nely*k) (x fastest). N_n = (nelx+1)(nely+1)(nelz+1),
 *            N_dof = 3*N_n, N_e = nelx*nely*nelz.
 *  Vectors   displacement-like vectors are fp64 arrays of N_dof, array-of-structs:
 *            dof 3n+c holds component c (0=x,1=y,2=z) of node n. Element fields are fp64
 *            arrays of N_e in element order.
 *  Corners   element corner a in order (0,0,0),(1,0,0),(1,1,0),(0,1,0),(0,0,1),(1,0,1),
 *            (1,1,1),(0,1,1); element DOF list = [3*n_a + c].
 *  Fixed     fixed DOFs act as identity rows and columns of K_hat (reading A7).
 *  Pointers  "d_" = device pointer (owned by the caller, normally a torch tensor), 8-byte
 *            aligned; "h_" = host pointer. The library never allocates device memory: all
 *            scratch lives in the caller's workspace given to tomo_bind().
 *  Streams   every call is enqueued on the stream given to tomo_bind(). Calls that return
 *            a host value (tomo_solve, tomo_compliance, tomo_sensitivity with energy_out,
 *            tomo_oc_update, tomo_evaluate*) synchronise that stream before returning.
 *  Errors    every int-returning call returns TOMO_OK (0) or a negative tomo_status
 *            (tomo_solve returns the iteration count >= 0 on success). A message is
 *            available from tomo_last_error(). No C++ exception crosses the ABI.
 *  Threads   a context is not thread-safe; use one context per problem / per thread.
 */
#ifndef TOMO_H
#define TOMO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tomo_ctx tomo_ctx; /* opaque */

typedef enum {
  TOMO_OK = 0,
  TOMO_EINVAL = -1,        /* bad argument (NULL, misaligned pointer, bad parameter)     */
  TOMO_EDOMAIN = -2,       /* a density outside [0,1]                    */
  TOMO_ESIZE = -3,         /* a length does not match the context's grid */
  TOMO_EBREAKDOWN = -4,    /* PCG: p^T K p <= 0                          */
  TOMO_EPRECOND = -5,      /* Jacobi diagonal <= 0 at a free DOF         */
  TOMO_ENAN = -6,          /* NaN/Inf met in a reduction                                 */
  TOMO_EBRACKET = -7,      /* OC: NaN in the bisection                   */
  TOMO_ECUDA = -8,         /* a CUDA runtime error; see tomo_last_error                  */
  TOMO_ENOWORKSPACE = -9   /* call needs tomo_bind() first, or workspace too small        */
} tomo_status;

typedef struct {
  int nelx, nely, nelz; /* elements per axis, each >= 1                   */
  double h;             /* element edge length > 0; KE scales as h (3D elasticity)       */
} tomo_grid;

typedef enum {
  TOMO_BC_CANTILEVER = 1, /* x=0 face clamped; load_total in -z... (sign in load_total)
                             spread in equal parts over nodes (nelx, j, 0), j=0..nely
                             (BASELINE.json configs[0]; reading A8)       */
  TOMO_BC_MBB_HALF = 2,   /* u_x=0 on x=0 face, u_z=0 on nodes (nelx, j, 0), u_y=0 at node
                             (nelx,0,0); load_total in z spread equally over nodes (0, j,
                             nelz) (BASELINE.json configs[2]; readings A9, A10)           */
  TOMO_BC_EXPLICIT = 3    /* fixed_dofs / load_dofs / load_vals as given                  */
} tomo_bc_kind;

typedef struct {
  int kind;                 /* tomo_bc_kind                                               */
  double load_total;        /* presets: total z force (e.g. -1.0)                         */
  const int64_t* fixed_dofs; int64_t n_fixed;              /* EXPLICIT only (host)        */
  const int64_t* load_dofs; const double* load_vals; int64_t n_loads; /* EXPLICIT (host)  */
} tomo_bc;

typedef struct {
  int iterations;           /* number of K_hat p products in the PCG loop (reading A11)   */
  int converged;            /* 1: ||r_k|| <= tol ||f|| (recursive) and the true residual
                               ||f - K_hat u|| <= tol ||f||; 2: the recursive residual met
                               tol but the true one did not (fp64 floor at high contrast);
                               0: max_iters reached (not an error)          */
  double rel_res_recursive; /* ||r_k|| / ||f||                                            */
  double rel_res_true;      /* ||f - K_hat u|| / ||f|| recomputed at exit                 */
} tomo_solve_info;

/* ---------------------------------------------------------------- lifetime
 * tomo_create: host-only; validates (nel* >= 1, h > 0, 0 < Emin < E0, 0 < nu < 0.5, p >= 1,
 * rmin > 0; EXPLICIT dofs in range and no loaded DOF fixed) and
 * builds the host tables: KE (24x24, 2x2x2 Gauss quadrature of B^T C B)
 * and its Walsh-basis coefficients, the BC mask and load list, the filter taps
 * {d in Z^3 : rmin - |d| > 0} (reading A15). No device work.     */
int tomo_create(tomo_ctx** out, const tomo_grid* g, double E0, double Emin, double nu,
                double penal, double rmin, const tomo_bc* bc);
/* bytes of device workspace tomo_bind needs (all PCG vectors, E, Jacobi, filter sums)   */
size_t tomo_workspace_bytes(const tomo_ctx* ctx);
/* binds a caller-owned device workspace (>= tomo_workspace_bytes, 256-B aligned) and a
 * stream (cudaStream_t passed as void*; NULL = legacy default stream). Uploads tables and
 * computes the device-side mask, filter sums Hs and neighbour counts. Synchronises.      */
int tomo_bind(tomo_ctx* ctx, void* d_workspace, size_t bytes, void* stream);
void tomo_destroy(tomo_ctx* ctx);
const char* tomo_last_error(const tomo_ctx* ctx);
/* sizes: out[0]=N_e, out[1]=N_n, out[2]=N_dof, out[3]=n_loads, out[4]=n_taps            */
int tomo_sizes(const tomo_ctx* ctx, int64_t out[5]);

/* ---------------------------------------------------------------- operator
 * y = K_hat(rho) u (SPEC.md l.123-131 [OP apply_stiffness]; "K(z)u - f"):
 * y = sum_e E_e S_e^T KE S_e (u with fixed entries zeroed), then y_i = u_i at fixed DOFs.
 * d_rho: N_e densities in [0,1] (else TOMO_EDOMAIN); d_u, d_y: N_dof, must not alias.    */
int tomo_apply(tomo_ctx* ctx, const double* d_rho, int64_t n_e, const double* d_u,
               double* d_y, int64_t n_dof);

/* Jacobi-PCG solve K_hat(rho) u = f:
 * d_u in: x0 (fixed entries are zeroed), out: u. Stops when ||r_k||_2 <= tol ||f||_2 on
 * the recursive residual or after max_iters products (converged = 0, not an error,
 * SPEC.md l.172). f = 0 gives u = 0 and 0 iterations. Returns iterations >= 0 or status.
 * info may be NULL.                                                                      */
int tomo_solve(tomo_ctx* ctx, const double* d_rho, int64_t n_e, double* d_u, int64_t n_dof,
               double tol, int max_iters, tomo_solve_info* info);

/* c = f^T u (Eq. 4), to host *c_out.                 */
int tomo_compliance(tomo_ctx* ctx, const double* d_u, int64_t n_dof, double* c_out);

/* Eq. 5 (reading A5):
 * ce_e = u_e^T KE u_e (u zeroed at fixed DOFs), dc_e = -p rho_e^(p-1) (E0-Emin) ce_e.
 * d_ce and energy_out (host, sum_e E_e ce_e = u^T K u) may be NULL.                      */
int tomo_sensitivity(tomo_ctx* ctx, const double* d_rho, const double* d_u, double* d_dc,
                     double* d_ce, double* energy_out);

/* density filter ("P is the density filter matrix"):
 * transpose = 0: out = P in,   (P x)_i = sum_j w_ij x_j / Hs_i
 * transpose = 1: out = P^T in, (P^T v)_j = sum_i w_ij v_i / Hs_i   ("filtered dc")
 * w_ij = rmin - |c_i - c_j| > 0 over element centroids (element units), domain-truncated.
 * d_in and d_out must not alias.                                                          */
int tomo_filter(tomo_ctx* ctx, const double* d_in, double* d_out, int64_t n_e, int transpose);

/* dV/dz = P^T v with v = 1 (reading A16) into d_dv[N_e].                 */
int tomo_volume_grad(tomo_ctx* ctx, double* d_dv, int64_t n_e);

/* OC update (reading A17). With B_e(l) = max(0,-g_e) /
 * (dv_e l): x_new_e(l) = clamp(x_e sqrt(B_e) [eta=0.5; B^eta otherwise],
 *                              max(0, x_e - move), min(1, x_e + move)).
 * Device bisection l1=1e-30, l2=1e30, lm = sqrt(l1 l2) while l2 > l1(1+1e-15) (<= 200
 * steps): dv^T x_new(lm) > volfrac N_e ? l1 = lm : l2 = lm. Writes x_new(l2), *lambda_out
 * = l2, *steps_out = steps, negated when the target is unreachable within the move limits
 * (not an error). d_dv = P^T 1 from tomo_volume_grad.                                    */
int tomo_oc_update(tomo_ctx* ctx, const double* d_x, const double* d_g, const double* d_dv,
                   int64_t n_e, double volfrac, double move, double eta, double* d_xnew,
                   double* lambda_out, int* steps_out);

/* One exact-gradient evaluation (the metric unit): tomo_solve(rho, u)
 * then c = f^T u, dc (Eq. 5), dcf = P^T dc. All arrays device; d_u in: x0, out: u.
 * d_dc may be NULL (kept in workspace). Returns iterations >= 0 or a status.             */
int tomo_evaluate(tomo_ctx* ctx, const double* d_rho, double* d_u, double* d_dc,
                  double* d_dcf, double tol, int max_iters, double* c_out,
                  tomo_solve_info* info);
/* The same with HOST arrays (h_rho in; h_u, h_dcf out; h_u may be NULL): copies in and
 * out through the workspace's staging vectors inside the call (the e2e measurement).     */
int tomo_evaluate_host(tomo_ctx* ctx, const double* h_rho, double* h_u, double* h_dcf,
                       double tol, int max_iters, double* c_out, tomo_solve_info* info);

/* ---------------------------------------------------------------- two-scale coarse path
 * ("coarse-grained design variable vector z_C ... each of
 * its component is the averaged value of z in each subset", l.184-186 "3D blocks of
 * uniform dimensions N_B x N_B x N_B ... K_C(z_C)u_C - f_C = 0", Alg. 1 lines 3-4;
 * SPEC.md l.364-391). nb must divide nelx, nely and nelz (else TOMO_EINVAL).
 * tomo_create_coarse: host-only; a new context for the coarse problem: grid nelx/nb x nely/nb x nelz/nb, edge
 * nb*h, the fine material, and the fine BCs restricted per SPEC.md l.374-382 (reading R4):
 * a coarse DOF is fixed iff a fine node whose nearest coarse node it is (per axis
 * I = floor(i/nb + 1/2)) has that DOF fixed; fine loads are summed onto that node. The
 * result is solved with the ordinary tomo_solve on its own bound workspace.
 * tomo_coarsen: z_C[b] = mean of z over block b (element order on both grids), on the fine
 * context's stream; d_z: N_e fine, d_zc: N_e / nb^3.                                    */
int tomo_create_coarse(tomo_ctx** out, const tomo_ctx* fine, int nb);
int tomo_coarsen(tomo_ctx* fine, const double* d_z, int nb, double* d_zc, int64_t n_ec);

/* ---------------------------------------------------------------- multigrid-preconditioned CG
 * ("Iterative solvers such as preconditioned conjugate
 * gradient (PCG) and multi-grid methods are typically used"). Optional solver; the metric
 * path is the Jacobi-PCG of tomo_solve. Levels l = 1..levels-1 halve the grid (each
 * dimension must be divisible by 2^(levels-1)); their E is the mean of the 8 children's E,
 * their BCs those of tomo_create_coarse(nb = 2). Preconditioner: one V-cycle with `nu`
 * damped-Jacobi sweeps (weight omega) before and after the coarse correction, full-weighting
 * restriction = transpose of trilinear prolongation, the coarsest level solved by the fused
 * Jacobi-PCG to coarse_tol (at most coarse_iters launches). Outer loop: flexible CG
 * (Polak-Ribiere beta) from x0 = 0 with its scalars on the device, stopped on ||r_k|| <= tol
 * ||f||; the whole loop is one CUDA graph with a conditional WHILE node (host-batched
 * iterations under tomo_set_graph(ctx, 0)); returns iterations >= 0 or a status.
 * tomo_mg_workspace_bytes is host-only (builds the level contexts); tomo_mg_bind binds a
 * caller-owned device workspace of that size (256-B aligned) on the context's stream.     */
size_t tomo_mg_workspace_bytes(tomo_ctx* ctx, int levels);
int tomo_mg_bind(tomo_ctx* ctx, int levels, void* d_workspace, size_t bytes);
int tomo_mg_params(tomo_ctx* ctx, int nu, double omega, int coarse_iters, double coarse_tol);
int tomo_solve_mg(tomo_ctx* ctx, const double* d_rho, int64_t n_e, double* d_u, int64_t n_dof,
                  double tol, int max_iters, tomo_solve_info* info);

/* ---------------------------------------------------------------- introspection (tests)
 * Integer tables produced by the same device index code the kernels use, for bit-exact
 * parity with the oracle (BASELINE.json north_star: "DOF maps, filter neighbour lists,
 * BC masks ... must match bit-exactly").                                                 */
int tomo_get_ke(const tomo_ctx* ctx, double* h_out576);        /* KE row-major, host      */
int tomo_get_fixed_mask(tomo_ctx* ctx, uint8_t* d_mask);       /* N_dof bytes, device     */
int tomo_get_load(const tomo_ctx* ctx, int64_t* h_dofs, double* h_vals, int64_t* n_inout);
int tomo_get_filter_taps(const tomo_ctx* ctx, int* h_offsets /* 3*n */, double* h_w,
                         int* n_inout);
int tomo_get_element_dofs(tomo_ctx* ctx, int64_t* d_map /* 24*N_e */);
int tomo_get_neighbor_counts(tomo_ctx* ctx, int* d_counts /* N_e */);
int tomo_get_jacobi(tomo_ctx* ctx, const double* d_rho, double* d_dinv /* N_n */);
/* kernel launches enqueued by this context so far (all kinds), for bench bookkeeping    */
int64_t tomo_launch_count(const tomo_ctx* ctx);

/* ---------------------------------------------------------------- microbenchmarks
 * sustained FP64 FMA rate (GFLOP/s, FMA = 2 flop) and the per-launch mean time of the
 * PCG kernels of the last tomo_solve measured with CUDA events on the bound stream.      */
int tomo_bench_dfma(tomo_ctx* ctx, double* gflops_out, double* ms_out);
/* Residual history of the next solves (diagnostics): while set, launch k of
 * every PCG solve writes d_hist[k] = r_k^T r_k (k < n; the relative residual is
 * sqrt(d_hist[k]) / ||f||). d_hist: caller-owned device buffer of n doubles; n = 0 stops.  */
int tomo_set_history(tomo_ctx* ctx, double* d_hist, int n);
/* PCG beta (default 0): 0 = the single-pass recurrence (reading R1: beta from
 * the predicted r_{k+1}.z_{k+1}, one pass per iteration); 1 = textbook beta from the explicit
 * r_{k+1}, one extra reduction pass over r, q, D^-1 per iteration.         */
int tomo_set_pcg_exact_beta(tomo_ctx* ctx, int on);
/* PCG loop execution (default 1): 1 = the whole loop as one CUDA graph with a conditional
 * WHILE node (one launch and one read-back per solve); 0 = host-batched launches of the
 * same kernels (what ncu can profile: kernels inside conditional graphs are not captured).
 * Either way an iteration is one fused operator pass (k_op<OP_PCG>) and, with programmatic
 * dependent launch and single-pass beta, a one-block control kernel (k_pcg_red: grid totals,
 * stop test, alpha, beta) chained to it; the iterates do not depend on the form.          */
int tomo_set_graph(tomo_ctx* ctx, int on);
/* times[0] = mean ms per fused PCG launch, times[1] = 0 (no separate K_B kernel), times[2]
 * = number of launches timed. Requires tomo_set_profiling(ctx, 1) before the solve.      */
int tomo_set_profiling(tomo_ctx* ctx, int on);
/* K_hat u throughput: E from d_rho, then `reps` back-to-back launches of the operator
 * kernel on the workspace's internal (padded) u, timed with CUDA events on the bound stream;
 * *ms_out = mean ms per application.                                                    */
int tomo_bench_apply(tomo_ctx* ctx, const double* d_rho, int reps, double* ms_out);
int tomo_profile_times(const tomo_ctx* ctx, double* times3);

#ifdef __cplusplus
}
#endif
#endif /* TOMO_H */
