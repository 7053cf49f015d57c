// Internal declarations shared by the libtomo host code (api.cu) and the kernels
// (kernels.cu). Not part of the ABI; see include/tomo.h.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tomo {

// Checked build (-DTOMO_CHECKED=1, scripts/build_variants.py checked:TOMO_CHECKED=1): device
// asserts on shared-memory and global indices of the operator, filter and sensitivity kernels
// (the memory-safety net in place of compute-sanitizer, which is closed on this pool). A
// failed check traps, so the launch returns an error instead of reading out of bounds.
#ifndef TOMO_CHECKED
#define TOMO_CHECKED 0
#endif
#if TOMO_CHECKED
#define TCHECK(cond) \
  do {               \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define TCHECK(cond) \
  do {               \
  } while (0)
#endif

// Structured grid of nx*ny*nz hexahedra; (nx+1)(ny+1)(nz+1) nodes.
// The ABI vectors are dense AoS (DOF 3n+c, node n = i + nnx(j + nny k)). The solver's
// internal vectors are PADDED ROW-SoA (dof_pad): a node row (j, k) is three component
// sub-rows of nnx_pad (even) doubles, so every sub-row is a multiple of 16 bytes (a TMA
// requirement) and a warp's 32 consecutive nodes of one component are 256 contiguous
// bytes; element fields use rows of nx_pad (even); the per-node fixed mask uses byte rows
// of mp (multiple of 16).
struct Grid {
  int nx, ny, nz;     // elements per axis
  int nnx, nny, nnz;  // nodes per axis
  int nnx_pad, nx_pad, mp;
  long long nn, ne, ndof;          // dense counts
  long long nn_pad, ne_pad, ndof_pad, mask_bytes;
};

__host__ __device__ inline long long node_pad(const Grid& g, int i, int j, int k) {
  return (long long)i + (long long)g.nnx_pad * (j + (long long)g.nny * k);
}
// internal (padded row-SoA) index of DOF c of node (i, j, k)
__host__ __device__ inline long long dof_pad(const Grid& g, int i, int j, int k, int c) {
  return (long long)i + (long long)g.nnx_pad * (c + 3 * (j + (long long)g.nny * k));
}
__host__ __device__ inline long long node_dense(const Grid& g, int i, int j, int k) {
  return (long long)i + (long long)g.nnx * (j + (long long)g.nny * k);
}
__host__ __device__ inline long long mask_index(const Grid& g, int i, int j, int k) {
  return (long long)i + (long long)g.mp * (j + (long long)g.nny * k);
}
__host__ __device__ inline long long elem_pad(const Grid& g, int i, int j, int k) {
  return (long long)i + (long long)g.nx_pad * (j + (long long)g.ny * k);
}

// The E=1 element stiffness KE written in the (unnormalised, +-1) tensor-Walsh basis of
// corner values: D = T KE T^T / 64 has 45 non-zeros out of 576, described by these seven
// numbers (derived and checked entry by entry in api.cu: walsh_coefficients()).
//   normal strains : v_x0 = amb w_x0 + b (w_x0 + w_y1 + w_z2)   (and cyclic)
//   shear          : v_x1 = v_y0 = g (w_x1 + w_y0)              (and xz, yz)
//   bilinear modes : v_xy0 = c1 w_xy0 + c2 w_yz2, ...,  v_xy2 = c3 (s + w_xy2), s = w_xy2+w_xz1+w_yz0
//   trilinear mode : v_xyz_c = c4 w_xyz_c
struct Walsh {
  double amb, b, g, c1, c2, c3, c4;
};

// Device-side scalar state of one PCG solve (read/written only by kernels, except the
// host reads it back once per batch of iterations). Single-pass PCG:
// launch k forms r_k = r_{k-1} - alpha_{k-1} q_{k-1}, p_k = D^-1 r_k + beta_{k-1} p_{k-1},
// u_k = u_{k-1} + alpha_{k-1} p_{k-1}, q_k = K p_k and reduces p.q, r.z, r.r, z.q, q.D^-1 q.
struct Scal {
  double alpha;       // alpha_{k-1} for the next launch
  double beta;        // beta_{k-1} for the next launch
  double rz;          // r_k^T D^-1 r_k (exact, from the explicit r_k)
  double rr;          // r_k^T r_k
  double pq;          // p_k^T K p_k
  double rr_true;     // ||f - K u||^2 at exit
  double tol_fnorm;   // tol * ||f||
  double energy;      // sum_e E_e ce_e (sensitivity)
  double comp;        // f^T u
  int k;              // index of the next PCG launch
  int iters;          // products that contributed to u (standard PCG count)
  int done;           // 0 running, 1 converged, 2 max_iters, 3 error
  int status;         // tomo_status of an error
  int max_iters;
  int domain_bad;     // a density outside [0,1] / NaN met by k_simp
  unsigned cntA, cntB, cntR;  // last-block counters (reset by the last block)
  int hist_n;         // length of hist (0: no residual history)
  double* hist;       // optional device buffer: hist[k] = r_k^T r_k of launch k (tomo_set_history)
};

// Device scalars of the MG-preconditioned flexible CG (mg.cu k_fcg_*; api.cu tomo_solve_mg)
struct FcgScal {
  double rz, rr, alpha, beta, stop;
  int k, done, status, max_iters;  // done: 0 running, 1 converged, 2 max_iters, 3 error
  unsigned cnt;                    // last-block counter
  int pad;
};
enum FcgMode { FCG_INIT = 0, FCG_ALPHA = 1, FCG_BETA = 2 };

enum OpMode { OP_APPLY = 0, OP_PCG = 1 };

// Operator tile: 32 x OP_BY threads. Warp w stages node rows w and w+1 of the tile (OP_BY+1
// node rows j0-1 .. j0+OP_BY-1, the shared row staged by both warps), computes element row
// w (element column i0-1+tx in lane tx; lane 31 is outside the tile) and outputs node row
// w+1 (OP_OY = OP_BY-1 output rows j0 .. j0+OP_BY-2, OP_OX = 30 output columns i0 .. i0+29).
// x-neighbours are exchanged with warp shuffles; the only cross-warp exchange is the
// bottom-face contribution of element row w+1 to node row w+1 (one barrier per plane).
// A block marches along z through a chunk of node planes.
#ifndef TOMO_OP_BY
#define TOMO_OP_BY 8
#endif
constexpr int OP_BY = TOMO_OP_BY;
constexpr int OP_MINB = OP_BY >= 16 ? 1 : 2;  // resident blocks per SM the tile is sized for
constexpr int OP_TX = 32;           // threads per tile row (lane tx <-> node / element column i0-1+tx)
constexpr int OP_OX = 30;           // output nodes per tile along x
constexpr int OP_OY = OP_BY - 1;    // output nodes per tile along y
#ifndef TOMO_OP_NS
#define TOMO_OP_NS 2
#endif
constexpr int OP_NS = TOMO_OP_NS;   // TMA pipeline stages (node planes in flight)
#ifndef TOMO_OP_MINB_APPLY
#define TOMO_OP_MINB_APPLY 2
#endif
constexpr int OP_MINB_APPLY = TOMO_OP_MINB_APPLY;  // resident blocks per SM of the K_hat u kernel
#ifndef TOMO_GSREG_APPLY
#define TOMO_GSREG_APPLY 1
#endif
#ifndef TOMO_GSREG_PCG
#define TOMO_GSREG_PCG 0
#endif
// carry the top face of the last element in registers (1) or shared memory (0)
constexpr int OP_GSREG_APPLY = TOMO_GSREG_APPLY, OP_GSREG_PCG = TOMO_GSREG_PCG;
#ifndef TOMO_PINGPONG_PCG
#define TOMO_PINGPONG_PCG 0
#endif
constexpr bool OP_PINGPONG_PCG = TOMO_PINGPONG_PCG != 0;
#ifndef TOMO_ACQREL_ARRIVE
#define TOMO_ACQREL_ARRIVE 0  // A/B: last-block arrival as one acq_rel atomic (kernels.cu arrive_last)
#endif
#ifndef TOMO_SEP_EARLY
#define TOMO_SEP_EARLY 0  // A/B: k_pcg_red lets the next launch be scheduled before it waits
#endif
#ifndef TOMO_OP_NS_APPLY
#define TOMO_OP_NS_APPLY 6
#endif
#ifndef TOMO_APPLY_RAWLDG
#define TOMO_APPLY_RAWLDG 0  // A/B: K_hat u re-reads the raw u of fixed DOFs at the output (no carry)
#endif
#ifndef TOMO_GS_TMEM
#define TOMO_GS_TMEM 0  // A/B: the PCG kernel's top-face carry in tensor memory instead of shared memory
#endif
#ifndef TOMO_EARLY_REFILL
#define TOMO_EARLY_REFILL 0  // A/B: PCG stage refill issued mid-step behind an "empty" mbarrier
#endif
constexpr int OP_NS_APPLY = TOMO_OP_NS_APPLY;  // stages of the K_hat u kernel (smaller stages)
// (an L2 prefetch of planes 2-6 ahead measured slower at every distance: 82.5-106.5 vs 79.8 us)

struct OpArgs {
  CUtensorMap tm_in;    // APPLY: u ; PCG: r_{k-1} (box 98 x (BY+1) doubles)
  CUtensorMap tm_qold;  // PCG: q_{k-1}            (box 98 x (BY+1))
  CUtensorMap tm_pold;  // PCG: p_{k-1}            (box 98 x (BY+1))
  CUtensorMap tm_uown;  // PCG: u, owned box   (box 90 x BY-1)
  CUtensorMap tm_dinv;  // PCG: Jacobi, per node (box 32 x (BY+1))
  CUtensorMap tm_mask;  // fixed mask bytes     (box 32 x (BY+1))
  CUtensorMap tm_E;     // element modulus      (box 32 x BY)
  Grid g;
  Walsh w;
  double* rnew;         // PCG: r_k (owned nodes written)
  double* pnew;         // PCG: p_k (owned nodes written)
  double* u;            // PCG: u (owned nodes: u += alpha_{k-1} p_{k-1}) ; APPLY: the input vector
  double* out;          // APPLY: y (raw u at fixed DOFs) ; PCG: q
  double* partials;     // PCG: five per block
  Scal* s;              // PCG
  int ntiles;           // x-y tiles
  int zchunks;          // 0: persistent balanced schedule; > 0: block = (tile, z-chunk)
  unsigned long long cond;  // PCG in a CUDA graph: WHILE-node handle cleared when done (0: none)
  int sep;              // PCG: 1 = the grid reduction / control runs in k_pcg_red after each launch
};

// launch helpers (kernels.cu). All enqueue on `st`; return the launch error.
int op_tiles(const Grid& g);
size_t op_smem(int mode);
int op_occupancy(int mode);
cudaError_t launch_op(int mode, const OpArgs& a, int nblocks, cudaStream_t st, bool pdl = false);
// kernel node of one PCG launch (args copied into the node)
cudaError_t add_pcg_node(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* deps,
                         size_t ndeps, const OpArgs& a, int nblocks);
// the one-block control kernel after a PCG launch (OpArgs::sep), launched / as a graph node
// after `prev` with a programmatic edge
cudaError_t launch_pcg_red(const OpArgs& a, int nblocks, cudaStream_t st, bool pdl);
cudaError_t add_pcg_red_node(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphNode_t prev,
                             const OpArgs& a, int nblocks);
// the same node after `prev` with a programmatic-dependent-launch edge (prev may be null)
cudaError_t add_pcg_node_pdl(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphNode_t prev,
                             const OpArgs& a, int nblocks);
cudaError_t launch_simp(const Grid& g, const double* rho, double* E, double E0, double Emin,
                        double penal, Scal* s, cudaStream_t st);
cudaError_t launch_jacobi(const Grid& g, const double* E, double ke_diag, double* dinv,
                          cudaStream_t st);
// dense ABI vector <-> padded internal vector (in: fixed entries zeroed)
cudaError_t launch_pack(const Grid& g, const double* dense, double* pad, const uint8_t* mask,
                        cudaStream_t st);
cudaError_t launch_unpack(const Grid& g, const double* pad, double* dense, cudaStream_t st);
cudaError_t launch_scal_init(Scal* s, double tol_fnorm, int max_iters, cudaStream_t st);
// r = -q + f (sparse f at padded DOF indices)
cudaError_t launch_resid(const Grid& g, const double* q, double* r, const int64_t* ldofs_pad,
                         const double* lvals, int nloads, cudaStream_t st);
// exact-beta variant: beta_k from the explicit r_{k+1} (after each PCG launch)
cudaError_t launch_beta(const Grid& g, const double* r, const double* q, const double* dinv,
                        Scal* s, double* partials, int nblocks, cudaStream_t st);
cudaError_t add_beta_node(cudaGraph_t gr, cudaGraphNode_t* node, const cudaGraphNode_t* deps,
                          size_t ndeps, const Grid& g, const double* r, const double* q,
                          const double* dinv, Scal* s, double* partials, int nblocks);
cudaError_t launch_norm2(const Grid& g, const double* r, Scal* s, double* partials,
                         int nblocks, cudaStream_t st);
cudaError_t launch_compliance(const double* u, const int64_t* ldofs, const double* lvals,
                              int nloads, Scal* s, cudaStream_t st);
cudaError_t launch_sens(const Grid& g, const Walsh& w, const double* rho, const double* u,
                        const uint8_t* mask, double penal, double dE, double Emin,
                        double* dc, double* ce, double* partials, int max_blocks, Scal* s,
                        int want_energy, cudaStream_t st);
cudaError_t launch_filter_sums(const Grid& g, const int* taps, const double* w, int ntaps,
                               double* Hs, double* iHs, int* counts, cudaStream_t st);
cudaError_t launch_filter(const Grid& g, const int* taps, const double* w, int ntaps,
                          const double* Hs, const double* in, double* out, int transpose,
                          cudaStream_t st);
cudaError_t launch_filter_tiled(const Grid& g, int R, int M, const double* wd2, const double* hw,
                                const double* iHs, const double* in, double* out, int transpose,
                                int sms, cudaStream_t st);
cudaError_t launch_oc(int ne, const double* x, const double* g, const double* dv,
                      double* xnew, double target, double move, double eta,
                      double* partials, double* out2, int grid_blocks, cudaStream_t st);
int oc_max_blocks();
cudaError_t launch_edofs(const Grid& g, long long* map, cudaStream_t st);
cudaError_t launch_mask_dofs(const Grid& g, const uint8_t* mask, uint8_t* out,
                             cudaStream_t st);
cudaError_t launch_dinv_dense(const Grid& g, const double* dinv_pad, double* out,
                              cudaStream_t st);
cudaError_t launch_coarsen(const Grid& g, int nb, const double* z, double* zc, cudaStream_t st);
cudaError_t launch_dfma(double* out, int blocks, int iters, cudaStream_t st);
cudaError_t launch_set_tol(Scal* s, double tol, cudaStream_t st);
// multigrid (mg.cu)
cudaError_t launch_jacobi_smooth(const Grid& g, double omega, const double* b, const double* kx,
                                 const double* dinv, const uint8_t* mask, double* x, cudaStream_t st);
cudaError_t launch_residual(const Grid& g, const double* b, const double* kx, const uint8_t* mask,
                            double* r, cudaStream_t st);
cudaError_t launch_restrict(const Grid& gf, const Grid& gc, const double* rf, const uint8_t* maskc,
                            double* rc, cudaStream_t st);
cudaError_t launch_prolong_add(const Grid& gf, const Grid& gc, const double* xc,
                               const uint8_t* maskf, double* xf, cudaStream_t st);
cudaError_t launch_coarsen_E(const Grid& gf, const Grid& gc, const double* Ef, double* Ec,
                             int mode, cudaStream_t st);

cudaError_t launch_fcg_dot(long long n, const double* a, const double* b, const double* c,
                           double* partials, int nblocks, FcgScal* s, int mode,
                           unsigned long long cond, cudaStream_t st);
cudaError_t launch_fcg_axpy2(long long n, const FcgScal* s, const double* P, double* U,
                             const double* Q, double* R, cudaStream_t st);
cudaError_t launch_fcg_xpby(long long n, const FcgScal* s, const double* Z, double* P,
                            cudaStream_t st);
cudaError_t launch_fcg_init(FcgScal* s, double stop, int max_iters, cudaStream_t st);

}  // namespace tomo
