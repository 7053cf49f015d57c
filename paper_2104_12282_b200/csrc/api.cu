// libtomo host side: the C ABI of include/tomo.h.
//
// Host-only work at tomo_create (KE by quadrature and its Walsh-basis core, BC mask and
// load list, filter taps); device work is enqueued on the stream bound by tomo_bind into
// the caller's workspace. tomo_bind also encodes the TMA tensor maps of the internal
// (padded) PCG vectors. The PCG driver launches one fused single-pass PCG kernel per
// iteration (kernels.cu, k_op<OP_PCG>), either as one CUDA graph with a conditional WHILE
// node (default) or in host batches (tomo_set_graph(ctx, 0)), and reads the device
// scalars back once per graph launch / batch. Consecutive PCG launches are chained by
// programmatic dependent launch (graph edges / launch attribute): a launch's blocks are
// scheduled while its predecessor finishes and wait inside for its completion.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for profilers

#include "../../include/tomo.h"
#include "tomo_internal.h"

using namespace tomo;

struct tomo_ctx {
  Grid g{};
  double h = 1, E0 = 1, Emin = 1e-9, nu = 0.3, penal = 3, rmin = 1.5;
  double KE[576];
  Walsh w{};
  double ke_diag = 0;
  std::vector<uint8_t> mask;       // dense per node, bit c = DOF 3n+c fixed
  std::vector<int64_t> load_dofs;  // dense DOF indices, distinct, insertion order
  std::vector<int64_t> load_dofs_pad;
  std::vector<double> load_vals;
  double fnorm = 0;
  std::vector<int> taps;  // 3 per tap
  std::vector<double> tap_w;
  int filt_R = 0, filt_M = 0;     // taps = {d : |d|^2 <= filt_M}, R = floor(sqrt(M))
  std::vector<double> wd2;        // weight by |d|^2 (3 R^2 + 1 entries)
  std::string err;
  // workspace
  bool bound = false;
  cudaStream_t st = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  size_t off_E, off_dinv, off_Hs, off_iHs, off_t0, off_t1, off_t2, off_u, off_r0, off_r1, off_p0, off_p1, off_q0, off_q1, off_us,
      off_mask, off_cnt, off_ld, off_ldp, off_lv, off_taps, off_tw, off_wd2, off_part, off_scal, off_oc,
      off_end;
  size_t n_part = 0;
  int op_blocks = 1;   // fused PCG kernel grid
  int op_zchunks = 0;
  int ap_blocks = 1;   // K_hat u kernel grid (its own occupancy)
  int ap_zchunks = 0;
  int nb_b = 1, nb_s = 1, nb_oc = 1;
  int64_t launches = 0;
  int sms = 148;
  // operator launch variants (tensor maps bound to workspace buffers)
  OpArgs op_apply_u{}, op_apply_p0{}, op_pcg[2];  // op_pcg[k & 1] for launch k
  cudaAccessPolicyWindow l2win{};  // TOMO_L2_PERSIST (A/B): persisting window of the PCG launches; num_bytes 0 = none
  cudaGraph_t pcg_graph = nullptr;        // WHILE(not done) { launch even; launch odd }
  bool use_graph = true;                  // tomo_set_graph: graph (1) or host batches (0)
  bool exact_beta = false;                // tomo_set_pcg_exact_beta: textbook beta (extra pass)
  bool pdl = true;                        // programmatic dependent launch between PCG launches
  int body_launches = 2;                  // PCG launches per WHILE body of the graph
  cudaGraphExec_t pcg_exec = nullptr;
  // multigrid hierarchy (tomo_mg_*): levels 1..L-1 are coarse contexts bound to the caller's
  // MG workspace; the outer flexible-CG vectors of the fine level live there too
  std::vector<tomo_ctx*> mg;
  char* mg_ws = nullptr;
  size_t mg_off_U = 0, mg_off_R = 0, mg_off_P = 0, mg_off_Q = 0, mg_off_Z = 0, mg_off_Zo = 0,
         mg_off_part = 0, mg_off_fs = 0, mg_end = 0;
  cudaGraph_t mg_graph = nullptr;        // WHILE(not done) { one flexible-CG iteration }
  cudaGraphExec_t mg_exec = nullptr;
  std::vector<size_t> mg_level_off;
  OpArgs op_apply_P{}, op_apply_Z{};
  bool mg_bound = false;
  int mg_nu = 2;              // pre- and post-smoothing sweeps
  double mg_omega = 0.3;      // damped Jacobi (0.45 diverges at cfg3's 1e9 contrast)
  int mg_coarse_iters = 30;   // coarsest level: fused Jacobi-PCG, loose tolerance
  double mg_coarse_tol = 1e-2;
  int mg_emode = std::getenv("TOMO_MG_EMODE") ? std::atoi(std::getenv("TOMO_MG_EMODE")) : 0;
  // profiling
  bool prof = false;
  double prof_a_ms = 0, prof_b_ms = 0;
  int64_t prof_n = 0;
  std::vector<cudaEvent_t> ev;

  template <class T>
  T* P(size_t off) const { return reinterpret_cast<T*>(ws + off); }
  double* E() const { return P<double>(off_E); }
  double* dinv() const { return P<double>(off_dinv); }
  double* Hs() const { return P<double>(off_Hs); }
  double* iHs() const { return P<double>(off_iHs); }
  double* t0() const { return P<double>(off_t0); }
  double* t1() const { return P<double>(off_t1); }
  double* t2() const { return P<double>(off_t2); }
  double* u() const { return P<double>(off_u); }
  double* r(int i) const { return P<double>(i ? off_r1 : off_r0); }
  double* p(int i) const { return P<double>(i ? off_p1 : off_p0); }
  double* q(int i) const { return P<double>(i ? off_q1 : off_q0); }
  double* us() const { return P<double>(off_us); }
  uint8_t* dmask() const { return P<uint8_t>(off_mask); }
  int* cnt() const { return P<int>(off_cnt); }
  int64_t* ld() const { return P<int64_t>(off_ld); }
  int64_t* ldp() const { return P<int64_t>(off_ldp); }
  double* lv() const { return P<double>(off_lv); }
  int* dtaps() const { return P<int>(off_taps); }
  double* tw() const { return P<double>(off_tw); }
  double* wd2v() const { return P<double>(off_wd2); }
  double* part() const { return P<double>(off_part); }
  Scal* scal() const { return P<Scal>(off_scal); }
  double* ocout() const { return P<double>(off_oc); }
};

namespace {

// NVTX range for the duration of a C-ABI call (ncu --nvtx --nvtx-include "tomo_solve/" ...)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

int fail(tomo_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(tomo_ctx* c, cudaError_t e, const char* where) {
  return fail(c, TOMO_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, expr)                                        \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
  } while (0)

#define LAUNCH(ctx, expr) \
  do {                    \
    CK(ctx, (expr));      \
    ++(ctx)->launches;    \
  } while (0)

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// ---------------------------------------------------------------- KE by quadrature
// KE = sum over the 2x2x2 Gauss points of w |J| B^T C B on a cube of edge h (SPEC.md
// l.105-113): trilinear shape functions N_a = prod_d (x_d if corner_d else 1 - x_d) on
// [0,1]^3, C isotropic (E = 1, nu), engineering shear strains. 2-point Gauss is exact here.
void build_ke(double nu, double h, double* KE) {
  static const int corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                   {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
  const double lam = nu / ((1 + nu) * (1 - 2 * nu)), mu = 1 / (2 * (1 + nu));
  double C[6][6] = {};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) C[a][b] = lam + (a == b ? 2 * mu : 0.0);
  for (int a = 3; a < 6; ++a) C[a][a] = mu;
  const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  const double wdet = 0.125 * h * h * h;
  std::memset(KE, 0, sizeof(double) * 576);
  for (int p0 = 0; p0 < 2; ++p0)
    for (int p1 = 0; p1 < 2; ++p1)
      for (int p2 = 0; p2 < 2; ++p2) {
        const double xi[3] = {gp[p0], gp[p1], gp[p2]};
        double B[6][24] = {};
        for (int a = 0; a < 8; ++a) {
          double f[3], s[3];
          for (int d = 0; d < 3; ++d) {
            f[d] = corner[a][d] ? xi[d] : 1 - xi[d];
            s[d] = corner[a][d] ? 1.0 : -1.0;
          }
          const double gx = s[0] * f[1] * f[2] / h, gy = f[0] * s[1] * f[2] / h,
                       gz = f[0] * f[1] * s[2] / h;
          B[0][3 * a] = gx;
          B[1][3 * a + 1] = gy;
          B[2][3 * a + 2] = gz;
          B[3][3 * a] = gy; B[3][3 * a + 1] = gx;          // gamma_xy
          B[4][3 * a + 1] = gz; B[4][3 * a + 2] = gy;      // gamma_yz
          B[5][3 * a] = gz; B[5][3 * a + 2] = gx;          // gamma_zx
        }
        double CB[6][24];
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 24; ++j) {
            double acc = 0;
            for (int k = 0; k < 6; ++k) acc += C[i][k] * B[k][j];
            CB[i][j] = acc;
          }
        for (int i = 0; i < 24; ++i)
          for (int j = 0; j < 24; ++j) {
            double acc = 0;
            for (int k = 0; k < 6; ++k) acc += B[k][i] * CB[k][j];
            KE[24 * i + j] += wdet * acc;
          }
      }
}

// D = T KE T^T / 64 in the +-1 Walsh basis (mode m = mx + 2 my + 4 mz, sign +1 on the
// corner side of each "difference" axis); extract the 7 coefficients and check that the
// pattern reproduces all 576 entries.
bool walsh_coefficients(const double* KE, Walsh* W, double* maxdev) {
  static const int corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                   {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
  double T[8][8];
  for (int m = 0; m < 8; ++m)
    for (int a = 0; a < 8; ++a) {
      double s = 1;
      for (int d = 0; d < 3; ++d)
        if ((m >> d) & 1) s *= corner[a][d] ? 1.0 : -1.0;
      T[m][a] = s;
    }
  double D[24][24];  // local: tomo_create may run concurrently on several threads
  for (int m = 0; m < 8; ++m)
    for (int c = 0; c < 3; ++c)
      for (int n = 0; n < 8; ++n)
        for (int e = 0; e < 3; ++e) {
          double acc = 0;
          for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b) acc += T[m][a] * KE[24 * (3 * a + c) + 3 * b + e] * T[n][b];
          D[3 * m + c][3 * n + e] = acc / 64.0;
        }
  auto at = [&](int m, int c, int n, int e) { return D[3 * m + c][3 * n + e]; };
  const int mx = 1, my = 2, mz = 4, mxy = 3, mxz = 5, myz = 6, mxyz = 7;
  W->b = at(mx, 0, my, 1);
  W->amb = at(mx, 0, mx, 0) - W->b;
  W->g = at(mx, 1, mx, 1);
  W->c1 = at(mxy, 0, mxy, 0);
  W->c2 = at(mxy, 0, myz, 2);
  W->c3 = at(mxy, 2, mxz, 1);
  W->c4 = at(mxyz, 0, mxyz, 0);
  double R[24][24] = {};
  auto set = [&](int m, int c, int n, int e, double v) { R[3 * m + c][3 * n + e] += v; };
  const int nm[3] = {mx, my, mz};
  for (int c = 0; c < 3; ++c) {  // normal strains
    for (int e = 0; e < 3; ++e) set(nm[c], c, nm[e], e, W->b);
    set(nm[c], c, nm[c], c, W->amb);
  }
  for (int c = 0; c < 3; ++c)  // shear: v_{m_c, e} = v_{m_e, c} = g (w_{m_c,e} + w_{m_e,c})
    for (int e = 0; e < 3; ++e)
      if (c != e) {
        set(nm[c], e, nm[c], e, W->g);
        set(nm[c], e, nm[e], c, W->g);
      }
  // bilinear modes
  set(mxy, 0, mxy, 0, W->c1); set(mxy, 0, myz, 2, W->c2);
  set(mxy, 1, mxy, 1, W->c1); set(mxy, 1, mxz, 2, W->c2);
  set(mxz, 0, mxz, 0, W->c1); set(mxz, 0, myz, 1, W->c2);
  set(mxz, 2, mxz, 2, W->c1); set(mxz, 2, mxy, 1, W->c2);
  set(myz, 1, myz, 1, W->c1); set(myz, 1, mxz, 0, W->c2);
  set(myz, 2, myz, 2, W->c1); set(myz, 2, mxy, 0, W->c2);
  const int sm[3] = {mxy, mxz, myz}, sc[3] = {2, 1, 0};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) set(sm[i], sc[i], sm[j], sc[j], W->c3);
    set(sm[i], sc[i], sm[i], sc[i], W->c3);
  }
  for (int c = 0; c < 3; ++c) set(mxyz, c, mxyz, c, W->c4);
  double mx_abs = 0, dev = 0;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) {
      mx_abs = std::fmax(mx_abs, std::fabs(D[i][j]));
      dev = std::fmax(dev, std::fabs(D[i][j] - R[i][j]));
    }
  *maxdev = dev / mx_abs;
  return dev <= 1e-13 * mx_abs;
}

inline long long node_id(const Grid& g, int i, int j, int k) {
  return (long long)i + (long long)g.nnx * (j + (long long)g.nny * k);
}

bool check_ptr(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 7) == 0; }

// ---------------------------------------------------------------- TMA tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D tiled map over a [d2][d1][d0] array with byte pitches pitch1 (row) and pitch2 (plane)
int make_map(tomo_ctx* c, CUtensorMap* tm, CUtensorMapDataType dt, void* base, uint64_t d0,
             uint64_t d1, uint64_t d2, uint64_t pitch1, uint64_t pitch2, uint32_t b0,
             uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return fail(c, TOMO_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {pitch1, pitch2};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  // A/B knob TOMO_TMA_L2PROMO = 0 (none) | 1 (64 B) | 2 (128 B, default) | 3 (256 B)
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (const char* e = getenv("TOMO_TMA_L2PROMO")) {
    const int v = atoi(e);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
            : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
            : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
  CUresult r = fn(tm, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, TOMO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return TOMO_OK;
}

}  // namespace

// ====================================================================== lifetime
extern "C" int tomo_create(tomo_ctx** out, const tomo_grid* gr, double E0, double Emin,
                           double nu, double penal, double rmin, const tomo_bc* bc) {
  if (!out || !gr || !bc) return TOMO_EINVAL;
  *out = nullptr;
  tomo_ctx* c = new (std::nothrow) tomo_ctx();
  if (!c) return TOMO_EINVAL;
  auto bad = [&](const char* m) {
    c->err = m;
    *out = c;  // returned so tomo_last_error works; caller must destroy
    return TOMO_EINVAL;
  };
  if (gr->nelx < 1 || gr->nely < 1 || gr->nelz < 1) return bad("nel* must be >= 1 (SPEC.md l.39)");
  if (!(gr->h > 0)) return bad("h must be > 0");
  if (!(Emin > 0 && Emin < E0)) return bad("need 0 < Emin < E0 (SPEC.md l.97)");
  if (!(nu > 0 && nu < 0.5)) return bad("need 0 < nu < 0.5 (SPEC.md l.97)");
  if (!(penal >= 1)) return bad("need penal >= 1 (SPEC.md l.97)");
  if (!(rmin > 0)) return bad("need rmin > 0");
  Grid& g = c->g;
  g.nx = gr->nelx; g.ny = gr->nely; g.nz = gr->nelz;
  g.nnx = g.nx + 1; g.nny = g.ny + 1; g.nnz = g.nz + 1;
  g.nnx_pad = g.nnx + (g.nnx & 1);
  g.nx_pad = g.nx + (g.nx & 1);
  g.mp = (g.nnx + 15) & ~15;
  g.nn = (long long)g.nnx * g.nny * g.nnz;
  g.ne = (long long)g.nx * g.ny * g.nz;
  g.ndof = 3 * g.nn;
  g.nn_pad = (long long)g.nnx_pad * g.nny * g.nnz;
  g.ne_pad = (long long)g.nx_pad * g.ny * g.nz;
  g.ndof_pad = 3 * g.nn_pad;
  g.mask_bytes = (long long)g.mp * g.nny * g.nnz;
  if (g.ndof_pad >= (1LL << 31) - 64) return bad("grid too large (internal DOF index is 32-bit)");
  c->h = gr->h; c->E0 = E0; c->Emin = Emin; c->nu = nu; c->penal = penal; c->rmin = rmin;
  build_ke(nu, gr->h, c->KE);
  double dev = 0;
  if (!walsh_coefficients(c->KE, &c->w, &dev)) return bad("KE Walsh pattern check failed");
  c->ke_diag = c->KE[0];
  for (int i = 0; i < 24; ++i)
    if (std::fabs(c->KE[25 * i] - c->ke_diag) > 1e-13 * c->ke_diag)
      return bad("KE diagonal not constant");

  // boundary conditions
  c->mask.assign((size_t)g.nn, 0);
  std::vector<std::pair<int64_t, double>> loads;
  if (bc->kind == TOMO_BC_CANTILEVER) {
    for (int k = 0; k <= g.nz; ++k)
      for (int j = 0; j <= g.ny; ++j) c->mask[node_id(g, 0, j, k)] = 7;
    for (int j = 0; j <= g.ny; ++j)
      loads.push_back({3 * node_id(g, g.nx, j, 0) + 2, bc->load_total / (g.ny + 1)});
  } else if (bc->kind == TOMO_BC_MBB_HALF) {
    for (int k = 0; k <= g.nz; ++k)
      for (int j = 0; j <= g.ny; ++j) c->mask[node_id(g, 0, j, k)] |= 1;
    for (int j = 0; j <= g.ny; ++j) c->mask[node_id(g, g.nx, j, 0)] |= 4;
    c->mask[node_id(g, g.nx, 0, 0)] |= 2;
    for (int j = 0; j <= g.ny; ++j)
      loads.push_back({3 * node_id(g, 0, j, g.nz) + 2, bc->load_total / (g.ny + 1)});
  } else if (bc->kind == TOMO_BC_EXPLICIT) {
    if (bc->n_fixed < 0 || bc->n_loads < 0) return bad("negative BC list length");
    if ((bc->n_fixed && !bc->fixed_dofs) || (bc->n_loads && (!bc->load_dofs || !bc->load_vals)))
      return bad("NULL BC list");
    for (int64_t i = 0; i < bc->n_fixed; ++i) {
      const int64_t d = bc->fixed_dofs[i];
      if (d < 0 || d >= g.ndof) return bad("fixed DOF out of range");
      c->mask[d / 3] |= (uint8_t)(1u << (d % 3));
    }
    for (int64_t i = 0; i < bc->n_loads; ++i) {
      const int64_t d = bc->load_dofs[i];
      if (d < 0 || d >= g.ndof) return bad("load DOF out of range");
      loads.push_back({d, bc->load_vals[i]});
    }
  } else {
    return bad("unknown BC kind");
  }
  for (auto& l : loads) {
    if ((c->mask[l.first / 3] >> (l.first % 3)) & 1) return bad("a load sits on a fixed DOF (SPEC.md l.31)");
    bool merged = false;
    for (size_t i = 0; i < c->load_dofs.size(); ++i)
      if (c->load_dofs[i] == l.first) { c->load_vals[i] += l.second; merged = true; break; }
    if (!merged) { c->load_dofs.push_back(l.first); c->load_vals.push_back(l.second); }
  }
  for (int64_t d : c->load_dofs) {
    const long long n = d / 3;
    const int i = (int)(n % g.nnx), j = (int)((n / g.nnx) % g.nny), k = (int)(n / ((long long)g.nnx * g.nny));
    c->load_dofs_pad.push_back(dof_pad(g, i, j, k, (int)(d % 3)));
  }
  double ff = 0;
  for (double v : c->load_vals) ff += v * v;
  c->fnorm = std::sqrt(ff);

  // filter taps {d : rmin - |d| > 0}, order dz, dy, dx ascending (reading A15)
  const int R = (int)std::ceil(rmin);
  for (int dz = -R; dz <= R; ++dz)
    for (int dy = -R; dy <= R; ++dy)
      for (int dx = -R; dx <= R; ++dx) {
        const double w = rmin - std::sqrt((double)(dx * dx + dy * dy + dz * dz));
        if (w > 0) {
          c->taps.push_back(dx); c->taps.push_back(dy); c->taps.push_back(dz);
          c->tap_w.push_back(w);
        }
      }

  // the tap set is a ball {|d|^2 <= M} (rmin - sqrt(d2) > 0 is monotone in d2): the tiled
  // filter kernel indexes the weights by |d|^2
  for (size_t t = 0; t < c->tap_w.size(); ++t) {
    const int d2 = c->taps[3 * t] * c->taps[3 * t] + c->taps[3 * t + 1] * c->taps[3 * t + 1] +
                   c->taps[3 * t + 2] * c->taps[3 * t + 2];
    c->filt_M = std::max(c->filt_M, d2);
  }
  c->filt_R = (int)std::floor(std::sqrt((double)c->filt_M) + 1e-9);
  c->wd2.assign((size_t)(3 * c->filt_R * c->filt_R + 1), 0.0);
  for (size_t t = 0; t < c->tap_w.size(); ++t) {
    const int d2 = c->taps[3 * t] * c->taps[3 * t] + c->taps[3 * t + 1] * c->taps[3 * t + 1] +
                   c->taps[3 * t + 2] * c->taps[3 * t + 2];
    c->wd2[d2] = c->tap_w[t];
  }

  // workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  const size_t vp = sizeof(double) * (size_t)g.ndof_pad, ve = sizeof(double) * (size_t)g.ne;
  c->off_E = take(sizeof(double) * (size_t)g.ne_pad);
  c->off_dinv = take(sizeof(double) * (size_t)g.nn_pad);
  c->off_u = take(vp);  // next to E and D^-1: one contiguous L2 access-policy window (tomo_bind)
  c->off_Hs = take(ve);
  c->off_iHs = take(ve);
  c->off_t0 = take(ve);
  c->off_t1 = take(ve);
  c->off_t2 = take(ve);
  c->off_r0 = take(vp);
  c->off_r1 = take(vp);
  c->off_p0 = take(vp);
  c->off_p1 = take(vp);
  c->off_q0 = take(vp);
  c->off_q1 = take(vp);
  c->off_us = take(sizeof(double) * (size_t)g.ndof);
  c->off_mask = take((size_t)g.mask_bytes);
  c->off_cnt = take(sizeof(int) * (size_t)g.ne);
  c->off_ld = take(sizeof(int64_t) * (c->load_dofs.size() + 1));
  c->off_ldp = take(sizeof(int64_t) * (c->load_dofs.size() + 1));
  c->off_lv = take(sizeof(double) * (c->load_dofs.size() + 1));
  c->off_taps = take(sizeof(int) * (c->taps.size() + 3));
  c->off_tw = take(sizeof(double) * (c->tap_w.size() + 1));
  c->off_wd2 = take(sizeof(double) * c->wd2.size());
  c->n_part = 8192 * 5;
  c->off_part = take(sizeof(double) * c->n_part);
  c->off_scal = take(sizeof(Scal));
  c->off_oc = take(sizeof(double) * 4);
  c->off_end = o;
  *out = c;
  return TOMO_OK;
}

extern "C" size_t tomo_workspace_bytes(const tomo_ctx* c) { return c ? c->off_end : 0; }

extern "C" void tomo_destroy(tomo_ctx* c) {
  if (!c) return;
  for (auto* l : c->mg) tomo_destroy(l);
  if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
  if (c->pcg_graph) cudaGraphDestroy(c->pcg_graph);
  if (c->mg_exec) cudaGraphExecDestroy(c->mg_exec);
  if (c->mg_graph) cudaGraphDestroy(c->mg_graph);
  for (auto e : c->ev) cudaEventDestroy(e);
  delete c;
}

extern "C" const char* tomo_last_error(const tomo_ctx* c) {
  return c ? c->err.c_str() : "null context";
}

extern "C" int tomo_sizes(const tomo_ctx* c, int64_t out[5]) {
  if (!c || !out) return TOMO_EINVAL;
  out[0] = c->g.ne; out[1] = c->g.nn; out[2] = c->g.ndof;
  out[3] = (int64_t)c->load_dofs.size(); out[4] = (int64_t)c->tap_w.size();
  return TOMO_OK;
}

namespace {
// operator launch variants: maps over the padded internal vectors
// the PCG control in the separate one-block kernel k_pcg_red (with PDL, single-pass beta;
// TOMO_NO_SEP_RED: the last block of each launch does it, as before)
int pcg_sep(const tomo_ctx* c) {
  return c->pdl && !c->exact_beta && !std::getenv("TOMO_NO_SEP_RED") ? 1 : 0;
}

int build_op_args(tomo_ctx* c) {
  const Grid& g = c->g;
  // row-SoA vectors: a 3-D map over (x, 3 * y + component, z), sub-row pitch 8 nnx_pad bytes
  const uint64_t rowv = 8ull * g.nnx_pad, planev = 3 * rowv * g.nny;
  const uint64_t rown = 8ull * g.nnx_pad, planen = rown * g.nny;
  const uint64_t rowm = (uint64_t)g.mp, planem = rowm * g.nny;
  const uint64_t rowe = 8ull * g.nx_pad, planee = rowe * g.ny;
  const CUtensorMapDataType F64 = CU_TENSOR_MAP_DATA_TYPE_FLOAT64, U8 = CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const uint32_t inw = OP_TX + 2, inh = OP_BY + 1;  // boxes widened: aligned starts
  CUtensorMap tm_u, tm_uown, tm_r[2], tm_q[2], tm_p[2], tm_dinv, tm_mask, tm_E;
  int rc;
  auto vec = [&](CUtensorMap* tm, double* base, uint32_t b0, uint32_t rows) {
    return make_map(c, tm, F64, base, g.nnx, 3ull * g.nny, g.nnz, rowv, planev, b0, 3 * rows);
  };
  if ((rc = vec(&tm_u, c->u(), inw, inh))) return rc;
  if ((rc = vec(&tm_uown, c->u(), inw, OP_OY))) return rc;
  for (int i = 0; i < 2; ++i) {
    if ((rc = vec(&tm_r[i], c->r(i), inw, inh))) return rc;
    if ((rc = vec(&tm_q[i], c->q(i), inw, inh))) return rc;
    if ((rc = vec(&tm_p[i], c->p(i), inw, inh))) return rc;
  }
  if ((rc = make_map(c, &tm_dinv, F64, c->dinv(), g.nnx, g.nny, g.nnz, rown, planen, inw, inh))) return rc;
  if ((rc = make_map(c, &tm_mask, U8, c->dmask(), g.nnx, g.nny, g.nnz, rowm, planem, 48, inh))) return rc;
  if ((rc = make_map(c, &tm_E, F64, c->E(), g.nx, g.ny, g.nz, rowe, planee, 32, OP_BY))) return rc;
  OpArgs base{};
  base.tm_uown = tm_uown;
  base.tm_dinv = tm_dinv;
  base.tm_mask = tm_mask;
  base.tm_E = tm_E;
  base.g = g;
  base.w = c->w;
  base.partials = c->part();
  base.s = c->scal();
  base.ntiles = op_tiles(g);
  base.zchunks = c->op_zchunks;
  c->op_apply_u = base;
  c->op_apply_u.zchunks = c->ap_zchunks;
  c->op_apply_u.tm_in = tm_u;
  c->op_apply_u.out = c->q(0);
  c->op_apply_u.u = c->u();      // APPLY: the input vector itself (raw values at fixed DOFs)
  c->op_apply_p0 = base;
  c->op_apply_p0.zchunks = c->ap_zchunks;
  c->op_apply_p0.tm_in = tm_p[0];
  c->op_apply_p0.out = c->q(0);
  c->op_apply_p0.u = c->p(0);
  // launch k reads the "old" buffers (k & 1) ^ 1 and writes the "new" ones k & 1
  for (int par = 0; par < 2; ++par) {
    const int o = par ^ 1, n = par;
    OpArgs& a = c->op_pcg[par];
    a = base;
    a.tm_in = tm_r[o];
    a.tm_qold = tm_q[o];
    a.tm_pold = tm_p[o];
    a.rnew = c->r(n);
    a.pnew = c->p(n);
    a.out = c->q(n);
    a.u = c->u();
    a.sep = pcg_sep(c);
  }
  return TOMO_OK;
}
}  // namespace

#ifndef TOMO_PDL_UNROLL
#define TOMO_PDL_UNROLL 16
#endif
namespace {
// The whole PCG loop as one graph: a conditional WHILE node whose body is the even and the
// odd launch; the last block of a launch that sets `done` clears the condition. Launches
// after convergence inside the body exit at their first instruction.
// TOMO_L2_PERSIST: the persisting window on a PCG kernel node of the graph (no-op otherwise)
cudaError_t l2_node(tomo_ctx* c, cudaGraphNode_t n) {
  if (!c->l2win.num_bytes) return cudaSuccess;
  cudaKernelNodeAttrValue v = {};
  v.accessPolicyWindow = c->l2win;
  return cudaGraphKernelNodeSetAttribute(n, cudaKernelNodeAttributeAccessPolicyWindow, &v);
}

int build_pcg_graph(tomo_ctx* c) {
  if (c->pcg_exec) { cudaGraphExecDestroy(c->pcg_exec); c->pcg_exec = nullptr; }
  if (c->pcg_graph) { cudaGraphDestroy(c->pcg_graph); c->pcg_graph = nullptr; }
  if (!c->use_graph) return TOMO_OK;  // host-batched launches (tomo_set_graph(ctx, 0))
  CK(c, cudaGraphCreate(&c->pcg_graph, 0));
  cudaGraphConditionalHandle h;
  CK(c, cudaGraphConditionalHandleCreate(&h, c->pcg_graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CK(c, cudaGraphAddNode(&cnode, c->pcg_graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  OpArgs a0 = c->op_pcg[0], a1 = c->op_pcg[1];
  a0.cond = h;
  a1.cond = h;
  cudaGraphNode_t n0, n1;
  c->body_launches = 2;
  if (c->pdl && !c->exact_beta) {
    // U launches per body chained by programmatic edges: launch i+1's blocks are scheduled
    // while launch i finishes (its last block's reduction, the kernel boundary) and wait in
    // griddepcontrol.wait for its completion. A WHILE-iteration boundary is an ordinary
    // dependency, so the body is unrolled; launches after the one that sets `done` exit at
    // their first instructions.
    // With OpArgs::sep each PCG launch is followed by the one-block control kernel
    // k_pcg_red (programmatic edges both ways): launch i+1 is scheduled once launch i is
    // complete and issues its first TMA loads while k_pcg_red sums launch i's partials.
    const int U = TOMO_PDL_UNROLL;
    cudaGraphNode_t prev = nullptr;
    for (int i = 0; i < U; ++i) {
      cudaGraphNode_t n;
      const OpArgs& ai = (i & 1) ? a1 : a0;
      CK(c, add_pcg_node_pdl(body, &n, prev, ai, c->op_blocks));
      CK(c, l2_node(c, n));
      prev = n;
      if (ai.sep) {
        CK(c, add_pcg_red_node(body, &n, prev, ai, c->op_blocks));
        prev = n;
      }
    }
    c->body_launches = U;
  } else {
  CK(c, add_pcg_node(body, &n0, nullptr, 0, a0, c->op_blocks));
  CK(c, l2_node(c, n0));
  if (c->exact_beta) {
    cudaGraphNode_t b0, b1;
    CK(c, add_beta_node(body, &b0, &n0, 1, c->g, c->r(0), c->q(0), c->dinv(), c->scal(), c->part(), c->nb_b));
    CK(c, add_pcg_node(body, &n1, &b0, 1, a1, c->op_blocks));
    CK(c, l2_node(c, n1));
    CK(c, add_beta_node(body, &b1, &n1, 1, c->g, c->r(1), c->q(1), c->dinv(), c->scal(), c->part(), c->nb_b));
  } else {
    CK(c, add_pcg_node(body, &n1, &n0, 1, a1, c->op_blocks));
    CK(c, l2_node(c, n1));
  }
  }
  CK(c, cudaGraphInstantiate(&c->pcg_exec, c->pcg_graph, 0));
  return TOMO_OK;
}
}  // namespace

namespace {
// Operator grid for `occ` resident blocks per SM. Synchronised schedule: block = (tile,
// z-chunk) with equal chunks, so the blocks of a wave march the same planes together and
// neighbouring tiles share their halo rows through L2 (cfg3: DRAM reads 227 -> 171 MB per
// PCG launch). The chunk count minimises waves x steps per block, waves = ceil(blocks /
// resident slots), steps = planes per chunk + 2 (pipeline fill; the first chunk skips the
// warm-up on plane -1 and takes one plane more): cfg3 2 chunks (one wave),
// 192x96x96 3 chunks, 256x128x128 5 chunks (three waves; measured 261 -> 191 us per PCG
// launch against the persistent balanced schedule used before). The balanced schedule
// (one block per slot, an equal contiguous share of the (tile, plane) list) remains for
// grids with more tiles than the partials buffer holds blocks.
void op_schedule(const Grid& g, int occ, int sms, int max_blocks, int* blocks, int* zchunks) {
  if (occ < 1) occ = 1;
  const long long tiles = op_tiles(g), slots = (long long)occ * sms;
  const long long units = tiles * g.nnz;
  *blocks = (int)std::max<long long>(1, std::min<long long>(slots, units));
  *zchunks = 0;
  const char* sc = std::getenv("TOMO_SCHED");  // A/B knob: "balanced" | "sync"
  if ((sc && std::strcmp(sc, "balanced") == 0) || tiles > max_blocks) return;
  int ch = 1;
  long long best = -1;
  for (int c = 1; c <= g.nnz && tiles * c <= max_blocks; ++c) {
    const long long waves = (tiles * c + slots - 1) / slots;
    // steps of the longest chunk (the kernel's split: z_q = 1 + q (nnz - 1) / chunks, the
    // first chunk skips the warm-up step on plane -1)
    long long steps = 0;
    auto zq = [&](int q) { return q == 0 ? 0 : std::min(g.nnz, 1 + (q * (g.nnz - 1)) / c); };
    for (int q = 0; q < c; ++q) {
      const int z0 = zq(q), z1 = zq(q + 1);
      steps = std::max<long long>(steps, z1 - z0 + 2 - (q == 0 ? 1 : 0));
    }
    const long long cost = waves * steps;
    if (best < 0 || cost < best) { best = cost; ch = c; }
  }
  if (const char* zc = std::getenv("TOMO_ZCHUNKS"))  // A/B knob
    ch = (int)std::max(1LL, std::min<long long>(std::min(g.nnz, std::atoi(zc)), max_blocks / tiles));
  *zchunks = ch;
  *blocks = (int)(tiles * ch);
}
}  // namespace

extern "C" int tomo_bind(tomo_ctx* c, void* d_ws, size_t bytes, void* stream) {
  if (!c) return TOMO_EINVAL;
  if (!d_ws || (reinterpret_cast<uintptr_t>(d_ws) & 255)) return fail(c, TOMO_EINVAL, "workspace must be 256-B aligned");
  if (bytes < c->off_end) return fail(c, TOMO_ENOWORKSPACE, "workspace too small");
  c->ws = static_cast<char*>(d_ws);
  c->ws_bytes = bytes;
  c->st = static_cast<cudaStream_t>(stream);
  if (std::getenv("TOMO_NO_GRAPH")) c->use_graph = false;  // A/B knob, same as tomo_set_graph(ctx, 0)
  if (std::getenv("TOMO_NO_PDL")) c->pdl = false;           // A/B knob: plain launch-to-launch order
  const Grid& g = c->g;
  int dev = 0;
  CK(c, cudaGetDevice(&dev));
  CK(c, cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
  // zero everything once: pad entries of the internal vectors must read as 0
  CK(c, cudaMemsetAsync(c->ws, 0, c->off_end, c->st));
  std::vector<uint8_t> mpad((size_t)g.mask_bytes, 0);
  for (int k = 0; k < g.nnz; ++k)
    for (int j = 0; j < g.nny; ++j)
      for (int i = 0; i < g.nnx; ++i) mpad[mask_index(g, i, j, k)] = c->mask[node_id(g, i, j, k)];
  CK(c, cudaMemcpyAsync(c->dmask(), mpad.data(), mpad.size(), cudaMemcpyHostToDevice, c->st));
  if (!c->load_dofs.empty()) {
    CK(c, cudaMemcpyAsync(c->ld(), c->load_dofs.data(), sizeof(int64_t) * c->load_dofs.size(), cudaMemcpyHostToDevice, c->st));
    CK(c, cudaMemcpyAsync(c->ldp(), c->load_dofs_pad.data(), sizeof(int64_t) * c->load_dofs.size(), cudaMemcpyHostToDevice, c->st));
    CK(c, cudaMemcpyAsync(c->lv(), c->load_vals.data(), sizeof(double) * c->load_vals.size(), cudaMemcpyHostToDevice, c->st));
  }
  if (!c->tap_w.empty()) {
    CK(c, cudaMemcpyAsync(c->dtaps(), c->taps.data(), sizeof(int) * c->taps.size(), cudaMemcpyHostToDevice, c->st));
    CK(c, cudaMemcpyAsync(c->tw(), c->tap_w.data(), sizeof(double) * c->tap_w.size(), cudaMemcpyHostToDevice, c->st));
    CK(c, cudaMemcpyAsync(c->wd2v(), c->wd2.data(), sizeof(double) * c->wd2.size(), cudaMemcpyHostToDevice, c->st));
  }
  LAUNCH(c, launch_filter_sums(g, c->dtaps(), c->tw(), (int)c->tap_w.size(), c->Hs(), c->iHs(), c->cnt(), c->st));
  op_schedule(g, op_occupancy(OP_PCG), c->sms, (int)(c->n_part / 5), &c->op_blocks, &c->op_zchunks);
  op_schedule(g, op_occupancy(OP_APPLY), c->sms, (int)(c->n_part / 5), &c->ap_blocks, &c->ap_zchunks);
  c->nb_b = (int)std::min<long long>((g.ndof_pad / 2 + 255) / 256, (long long)c->sms * 4);
  c->nb_s = (int)std::min<long long>((g.ne + 255) / 256, (long long)c->sms * 8);
  c->nb_oc = std::min(oc_max_blocks(), (int)std::max<long long>(1, (g.ne + 255) / 256));
  if ((size_t)c->nb_oc * 2 > c->n_part) c->nb_oc = (int)(c->n_part / 2);
  if (int rc = build_op_args(c)) return rc;
  c->l2win = cudaAccessPolicyWindow{};
  if (std::getenv("TOMO_L2_PERSIST")) {
    // A/B experiment: E and D^-1 (adjacent in the workspace, read by every PCG launch) as a
    // persisting L2 access-policy window of the stream and of the graph's PCG kernel nodes
    // (TOMO_L2_PERSIST=2: and u, which follows them: read and rewritten by every launch)
    const bool with_u = atoi(std::getenv("TOMO_L2_PERSIST")) >= 2;
    const size_t bytes = with_u ? (size_t)(c->off_u - c->off_E) + sizeof(double) * (size_t)g.ndof_pad
                                : (size_t)(c->off_u - c->off_E);
    int dev = 0, maxp = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(bytes + (4u << 20), (size_t)maxp));
    fprintf(stderr, "[tomo] L2 persisting window %.1f MB (device max %.1f MB)\n", bytes / 1e6, maxp / 1e6);
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = c->E();
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)maxp / (double)bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(c, cudaStreamSetAttribute(c->st, cudaStreamAttributeAccessPolicyWindow, &v));
    c->l2win = v.accessPolicyWindow;  // the graph's PCG kernel nodes get the same window
  }
  if (int rc = build_pcg_graph(c)) return rc;
  CK(c, cudaStreamSynchronize(c->st));
  c->bound = true;
  return TOMO_OK;
}

// ====================================================================== helpers
namespace {

int need_bound(tomo_ctx* c) {
  if (!c) return TOMO_EINVAL;
  if (!c->bound) return fail(c, TOMO_ENOWORKSPACE, "call tomo_bind first");
  return TOMO_OK;
}

// density filter (P or P^T): the tiled kernel for tap balls up to R = 8, else the per-tap
// gather kernel
cudaError_t run_filter(tomo_ctx* c, const double* in, double* out, int transpose) {
  if (!std::getenv("TOMO_FILTER_GATHER")) {  // A/B knob: force the per-tap gather kernel
    const cudaError_t e = launch_filter_tiled(c->g, c->filt_R, c->filt_M, c->wd2v(), c->wd2.data(), c->iHs(), in, out,
                                              transpose, c->sms, c->st);
    if (e != cudaErrorNotSupported) return e;
  }
  return launch_filter(c->g, c->dtaps(), c->tw(), (int)c->tap_w.size(), c->Hs(), in, out, transpose,
                       c->st);
}

// E = SIMP(rho) and D^-1 into the workspace; checks rho in [0,1]
int prepare_modulus(tomo_ctx* c, const double* d_rho, bool jacobi) {
  const Grid& g = c->g;
  CK(c, cudaMemsetAsync(&c->scal()->domain_bad, 0, sizeof(int), c->st));
  LAUNCH(c, launch_simp(g, d_rho, c->E(), c->E0, c->Emin, c->penal, c->scal(), c->st));
  if (jacobi) LAUNCH(c, launch_jacobi(g, c->E(), c->ke_diag, c->dinv(), c->st));
  int badv = 0;
  CK(c, cudaMemcpyAsync(&badv, &c->scal()->domain_bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  if (badv) return fail(c, TOMO_EDOMAIN, "density outside [0,1] (SPEC.md l.118)");
  return TOMO_OK;
}

// The PCG launches (graph or host batches) until the device sets `done`; *hs_out = final
// scalars. The scalars, r_{-1}, q_{-1}, p_{-1} and u must be initialised by the caller.
int run_pcg_loop(tomo_ctx* c, int max_iters, Scal* hs_out) {
  Scal& hs = *hs_out;
  hs = Scal{};
  int k = 0;  // launches issued
  int batch = 8;
  const bool prof = c->prof;
  if (c->pcg_exec && (!prof || !std::getenv("TOMO_PROFILE_PER_LAUNCH"))) {
    // the whole loop on the device: one graph launch, one read-back. Profiling brackets the
    // graph launch with two events (no perturbation of the loop): device time / launches.
    if (prof) {
      while (c->ev.size() < 2) {
        cudaEvent_t e;
        CK(c, cudaEventCreate(&e));
        c->ev.push_back(e);
      }
      CK(c, cudaEventRecord(c->ev[0], c->st));
    }
    CK(c, cudaGraphLaunch(c->pcg_exec, c->st));
    if (prof) CK(c, cudaEventRecord(c->ev[1], c->st));
    CK(c, cudaMemcpyAsync(&hs, c->scal(), sizeof(Scal), cudaMemcpyDeviceToHost, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    const int U = c->body_launches;
    const int nodes = U * ((hs.iters + U) / U) * (c->op_pcg[0].sep ? 2 : 1);  // whole bodies
    c->launches += nodes;
    if (prof) {
      float ms = 0;
      CK(c, cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
      // the launch after the one that set `done` (odd count) exits at its first instruction
      c->prof_a_ms += ms;
      c->prof_n += hs.iters + 1;
    }
  } else {
  if (prof) {
    while (c->ev.size() < 2 * 257) {
      cudaEvent_t e;
      CK(c, cudaEventCreate(&e));
      c->ev.push_back(e);
    }
  }
  for (;;) {
    const int nb = std::min(batch, max_iters + 1 - k);
    if (nb <= 0) break;
    for (int i = 0; i < nb; ++i) {
      if (prof && i < 256) CK(c, cudaEventRecord(c->ev[2 * i], c->st));
      LAUNCH(c, launch_op(OP_PCG, c->op_pcg[(k + i) & 1], c->op_blocks, c->st,
                          c->pdl && !c->exact_beta && i > 0));
      if (c->op_pcg[0].sep) LAUNCH(c, launch_pcg_red(c->op_pcg[(k + i) & 1], c->op_blocks, c->st, true));
      if (c->exact_beta) {
        const int par = (k + i) & 1;
        LAUNCH(c, launch_beta(c->g, c->r(par), c->q(par), c->dinv(), c->scal(), c->part(), c->nb_b, c->st));
      }
      if (prof && i < 256) CK(c, cudaEventRecord(c->ev[2 * i + 1], c->st));
    }
    const int k_before = hs.k;
    k += nb;
    CK(c, cudaMemcpyAsync(&hs, c->scal(), sizeof(Scal), cudaMemcpyDeviceToHost, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    if (prof) {
      // launches that did work: up to and including the one that set `done`
      const int real = std::min(nb, hs.done ? hs.iters - k_before + 1 : nb);
      for (int i = 0; i < real && i < 256; ++i) {
        float ta = 0;
        CK(c, cudaEventElapsedTime(&ta, c->ev[2 * i], c->ev[2 * i + 1]));
        c->prof_a_ms += ta;
        ++c->prof_n;
      }
    }
    if (hs.done) break;
    if (batch < 128) batch *= 2;
  }
  }
  return TOMO_OK;
}

// Single-pass Jacobi-PCG on the bound workspace: E / dinv ready; c->u()
// holds x0 (padded, masked). One fused launch per iteration; launch k checks r_k.
int pcg_internal(tomo_ctx* c, double tol, int max_iters, tomo_solve_info* info) {
  const Grid& g = c->g;
  const int nl = (int)c->load_dofs.size();
  const size_t vb = sizeof(double) * (size_t)g.ndof_pad;
  Scal hs{};
  LAUNCH(c, launch_scal_init(c->scal(), tol * c->fnorm, max_iters, c->st));
  // r_{-1} := r0 = f - K u0 in r[1]; q_{-1} = p_{-1} = 0
  LAUNCH(c, launch_op(OP_APPLY, c->op_apply_u, c->ap_blocks, c->st));
  LAUNCH(c, launch_resid(g, c->q(0), c->r(1), c->ldp(), c->lv(), nl, c->st));
  CK(c, cudaMemsetAsync(c->q(1), 0, vb, c->st));
  CK(c, cudaMemsetAsync(c->p(1), 0, vb, c->st));
  if (int rc = run_pcg_loop(c, max_iters, &hs)) return rc;
  if (hs.done == 3) {
    return fail(c, hs.status ? hs.status : TOMO_EBREAKDOWN,
                hs.status == TOMO_ENAN ? "NaN/Inf in PCG" : "PCG breakdown: p^T K p <= 0 (SPEC.md l.173)");
  }
  // true residual ||f - K u||
  LAUNCH(c, launch_op(OP_APPLY, c->op_apply_u, c->ap_blocks, c->st));
  LAUNCH(c, launch_resid(g, c->q(0), c->r(0), c->ldp(), c->lv(), nl, c->st));
  LAUNCH(c, launch_norm2(g, c->r(0), c->scal(), c->part(), c->nb_b, c->st));
  CK(c, cudaMemcpyAsync(&hs, c->scal(), sizeof(Scal), cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  if (info) {
    info->iterations = hs.iters;
    // 1: recursive AND true residual <= tol; 2: the recursive residual met tol but the true
    // residual recomputed at exit did not (the fp64 floor of a high-contrast problem)
    info->converged = hs.done != 1 ? 0 : (std::sqrt(hs.rr_true) <= tol * c->fnorm ? 1 : 2);
    info->rel_res_recursive = c->fnorm > 0 ? std::sqrt(hs.rr) / c->fnorm : 0.0;
    info->rel_res_true = c->fnorm > 0 ? std::sqrt(hs.rr_true) / c->fnorm : 0.0;
  }
  return hs.iters;
}

}  // namespace

// ====================================================================== operator / solve
extern "C" int tomo_apply(tomo_ctx* c, const double* d_rho, int64_t n_e, const double* d_u,
                          double* d_y, int64_t n_dof) {
  Range nvtx_range("tomo_apply");
  if (int rc = need_bound(c)) return rc;
  if (n_e != c->g.ne || n_dof != c->g.ndof) return fail(c, TOMO_ESIZE, "length mismatch (SPEC.md l.127)");
  if (!check_ptr(d_rho) || !check_ptr(d_u) || !check_ptr(d_y)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (d_u == d_y) return fail(c, TOMO_EINVAL, "u and y must not alias");
  if (int rc = prepare_modulus(c, d_rho, false)) return rc;
  LAUNCH(c, launch_pack(c->g, d_u, c->p(0), nullptr, c->st));
  LAUNCH(c, launch_op(OP_APPLY, c->op_apply_p0, c->ap_blocks, c->st));
  LAUNCH(c, launch_unpack(c->g, c->q(0), d_y, c->st));
  return TOMO_OK;
}

extern "C" int tomo_solve(tomo_ctx* c, const double* d_rho, int64_t n_e, double* d_u,
                          int64_t n_dof, double tol, int max_iters, tomo_solve_info* info) {
  Range nvtx_range("tomo_solve");
  if (int rc = need_bound(c)) return rc;
  if (n_e != c->g.ne || n_dof != c->g.ndof) return fail(c, TOMO_ESIZE, "length mismatch (SPEC.md l.127)");
  if (!check_ptr(d_rho) || !check_ptr(d_u)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (!(tol >= 0) || max_iters < 0) return fail(c, TOMO_EINVAL, "bad tol / max_iters");
  if (c->fnorm == 0.0) {  // f = 0: u = 0, no iterations
    CK(c, cudaMemsetAsync(d_u, 0, sizeof(double) * (size_t)n_dof, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    if (info) *info = tomo_solve_info{0, 1, 0.0, 0.0};
    return 0;
  }
  if (int rc = prepare_modulus(c, d_rho, true)) return rc;
  LAUNCH(c, launch_pack(c->g, d_u, c->u(), c->dmask(), c->st));
  const int it = pcg_internal(c, tol, max_iters, info);
  if (it < 0) return it;
  LAUNCH(c, launch_unpack(c->g, c->u(), d_u, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return it;
}

extern "C" int tomo_compliance(tomo_ctx* c, const double* d_u, int64_t n_dof, double* c_out) {
  if (int rc = need_bound(c)) return rc;
  if (n_dof != c->g.ndof) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_u) || !c_out) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  LAUNCH(c, launch_compliance(d_u, c->ld(), c->lv(), (int)c->load_dofs.size(), c->scal(), c->st));
  CK(c, cudaMemcpyAsync(c_out, &c->scal()->comp, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_sensitivity(tomo_ctx* c, const double* d_rho, const double* d_u,
                                double* d_dc, double* d_ce, double* energy_out) {
  Range nvtx_range("tomo_sensitivity");
  if (int rc = need_bound(c)) return rc;
  if (!check_ptr(d_rho) || !check_ptr(d_u) || !check_ptr(d_dc) || (d_ce && !check_ptr(d_ce)))
    return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  LAUNCH(c, launch_sens(c->g, c->w, d_rho, d_u, c->dmask(), c->penal, c->E0 - c->Emin, c->Emin,
                        d_dc, d_ce, c->part(), (int)c->n_part, c->scal(), energy_out ? 1 : 0, c->st));
  if (energy_out) {
    CK(c, cudaMemcpyAsync(energy_out, &c->scal()->energy, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(c, cudaStreamSynchronize(c->st));
  }
  return TOMO_OK;
}

extern "C" int tomo_filter(tomo_ctx* c, const double* d_in, double* d_out, int64_t n_e,
                           int transpose) {
  Range nvtx_range("tomo_filter");
  if (int rc = need_bound(c)) return rc;
  if (n_e != c->g.ne) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_in) || !check_ptr(d_out)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (d_in == d_out) return fail(c, TOMO_EINVAL, "in and out must not alias");
  LAUNCH(c, run_filter(c, d_in, d_out, transpose ? 1 : 0));
  return TOMO_OK;
}

extern "C" int tomo_volume_grad(tomo_ctx* c, double* d_dv, int64_t n_e) {
  if (int rc = need_bound(c)) return rc;
  if (n_e != c->g.ne) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_dv)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  // ones into t1, then P^T
  std::vector<double> ones((size_t)n_e, 1.0);
  CK(c, cudaMemcpyAsync(c->t1(), ones.data(), sizeof(double) * (size_t)n_e, cudaMemcpyHostToDevice, c->st));
  LAUNCH(c, run_filter(c, c->t1(), d_dv, 1));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_oc_update(tomo_ctx* c, const double* d_x, const double* d_g,
                              const double* d_dv, int64_t n_e, double volfrac, double move,
                              double eta, double* d_xnew, double* lambda_out, int* steps_out) {
  Range nvtx_range("tomo_oc_update");
  if (int rc = need_bound(c)) return rc;
  if (n_e != c->g.ne) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_x) || !check_ptr(d_g) || !check_ptr(d_dv) || !check_ptr(d_xnew))
    return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (!(volfrac > 0 && volfrac <= 1) || !(move > 0) || !(eta > 0)) return fail(c, TOMO_EINVAL, "bad OC parameters");
  const double target = volfrac * (double)n_e;
  CK(c, cudaMemsetAsync(c->ocout(), 0, sizeof(double) * 4, c->st));
  CK(c, launch_oc((int)n_e, d_x, d_g, d_dv, d_xnew, target, move, eta, c->part(), c->ocout(), c->nb_oc, c->st));
  ++c->launches;
  double o[3];
  CK(c, cudaMemcpyAsync(o, c->ocout(), sizeof(o), cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  if (o[2] != 0.0) return fail(c, TOMO_ENAN, "NaN/Inf in x, g or dv (SPEC.md l.322 \"NaN in gradients -> error\")");
  if (std::isnan(o[0])) return fail(c, TOMO_EBRACKET, "NaN in OC bisection (SPEC.md l.322)");
  if (lambda_out) *lambda_out = o[0];
  if (steps_out) *steps_out = (int)o[1];
  return TOMO_OK;
}

// ====================================================================== evaluation
namespace {
int evaluate_dev(tomo_ctx* c, const double* d_rho, double* d_u, double* d_dc, double* d_dcf,
                 double tol, int max_iters, double* c_out, tomo_solve_info* info) {
  const int it = tomo_solve(c, d_rho, c->g.ne, d_u, c->g.ndof, tol, max_iters, info);
  if (it < 0) return it;
  double* dc = d_dc ? d_dc : c->t0();
  LAUNCH(c, launch_compliance(d_u, c->ld(), c->lv(), (int)c->load_dofs.size(), c->scal(), c->st));
  // the solve left u in the workspace in the padded row-SoA layout (zero at fixed DOFs):
  // the sensitivity reads that copy (coalesced, no mask bytes) instead of the dense d_u
  // (not when f = 0: tomo_solve then returns u = 0 without touching the workspace copy)
  const bool pad_u = c->fnorm != 0.0 && !getenv("TOMO_SENS_DENSE");  // A/B knob
  LAUNCH(c, launch_sens(c->g, c->w, d_rho, pad_u ? c->u() : d_u, pad_u ? nullptr : c->dmask(), c->penal,
                        c->E0 - c->Emin, c->Emin, dc, nullptr, c->part(), (int)c->n_part, c->scal(), 0, c->st));
  LAUNCH(c, run_filter(c, dc, d_dcf, 1));
  if (c_out) {
    CK(c, cudaMemcpyAsync(c_out, &c->scal()->comp, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  }
  CK(c, cudaStreamSynchronize(c->st));
  return it;
}
}  // namespace

extern "C" int tomo_evaluate(tomo_ctx* c, const double* d_rho, double* d_u, double* d_dc,
                             double* d_dcf, double tol, int max_iters, double* c_out,
                             tomo_solve_info* info) {
  Range nvtx_range("tomo_evaluate");
  if (int rc = need_bound(c)) return rc;
  if (!check_ptr(d_rho) || !check_ptr(d_u) || !check_ptr(d_dcf) || (d_dc && !check_ptr(d_dc)))
    return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  return evaluate_dev(c, d_rho, d_u, d_dc, d_dcf, tol, max_iters, c_out, info);
}

extern "C" int tomo_evaluate_host(tomo_ctx* c, const double* h_rho, double* h_u, double* h_dcf,
                                  double tol, int max_iters, double* c_out,
                                  tomo_solve_info* info) {
  Range nvtx_range("tomo_evaluate_host");
  if (int rc = need_bound(c)) return rc;
  if (!h_rho || !h_dcf) return fail(c, TOMO_EINVAL, "NULL host pointer");
  const size_t be = sizeof(double) * (size_t)c->g.ne, bd = sizeof(double) * (size_t)c->g.ndof;
  // staging: rho -> t1, u -> us (x0 = 0), dc -> t0, dcf -> t2
  CK(c, cudaMemcpyAsync(c->t1(), h_rho, be, cudaMemcpyHostToDevice, c->st));
  CK(c, cudaMemsetAsync(c->us(), 0, bd, c->st));
  double* dcf = c->t2();
  const int it = evaluate_dev(c, c->t1(), c->us(), nullptr, dcf, tol, max_iters, c_out, info);
  if (it < 0) return it;
  CK(c, cudaMemcpyAsync(h_dcf, dcf, be, cudaMemcpyDeviceToHost, c->st));
  if (h_u) CK(c, cudaMemcpyAsync(h_u, c->us(), bd, cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return it;
}

// ====================================================================== introspection
extern "C" int tomo_get_ke(const tomo_ctx* c, double* out) {
  if (!c || !out) return TOMO_EINVAL;
  std::memcpy(out, c->KE, sizeof(c->KE));
  return TOMO_OK;
}

extern "C" int tomo_get_fixed_mask(tomo_ctx* c, uint8_t* d_mask) {
  if (int rc = need_bound(c)) return rc;
  if (!d_mask) return fail(c, TOMO_EINVAL, "NULL pointer");
  LAUNCH(c, launch_mask_dofs(c->g, c->dmask(), d_mask, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_get_load(const tomo_ctx* c, int64_t* dofs, double* vals, int64_t* n) {
  if (!c || !n) return TOMO_EINVAL;
  const int64_t m = (int64_t)c->load_dofs.size();
  if (dofs && vals) {
    if (*n < m) return TOMO_ESIZE;
    std::memcpy(dofs, c->load_dofs.data(), sizeof(int64_t) * m);
    std::memcpy(vals, c->load_vals.data(), sizeof(double) * m);
  }
  *n = m;
  return TOMO_OK;
}

extern "C" int tomo_get_filter_taps(const tomo_ctx* c, int* off, double* w, int* n) {
  if (!c || !n) return TOMO_EINVAL;
  const int m = (int)c->tap_w.size();
  if (off && w) {
    if (*n < m) return TOMO_ESIZE;
    std::memcpy(off, c->taps.data(), sizeof(int) * 3 * m);
    std::memcpy(w, c->tap_w.data(), sizeof(double) * m);
  }
  *n = m;
  return TOMO_OK;
}

extern "C" int tomo_get_element_dofs(tomo_ctx* c, int64_t* d_map) {
  if (int rc = need_bound(c)) return rc;
  if (!check_ptr(d_map)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  LAUNCH(c, launch_edofs(c->g, reinterpret_cast<long long*>(d_map), c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_get_neighbor_counts(tomo_ctx* c, int* d_counts) {
  if (int rc = need_bound(c)) return rc;
  if (!d_counts) return fail(c, TOMO_EINVAL, "NULL pointer");
  CK(c, cudaMemcpyAsync(d_counts, c->cnt(), sizeof(int) * (size_t)c->g.ne, cudaMemcpyDeviceToDevice, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_get_jacobi(tomo_ctx* c, const double* d_rho, double* d_dinv) {
  if (int rc = need_bound(c)) return rc;
  if (!check_ptr(d_rho) || !check_ptr(d_dinv)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (int rc = prepare_modulus(c, d_rho, true)) return rc;
  LAUNCH(c, launch_dinv_dense(c->g, c->dinv(), d_dinv, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int64_t tomo_launch_count(const tomo_ctx* c) { return c ? c->launches : -1; }

extern "C" int tomo_bench_dfma(tomo_ctx* c, double* gflops_out, double* ms_out) {
  if (int rc = need_bound(c)) return rc;
  const int blocks = c->sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  CK(c, cudaEventCreate(&e0));
  CK(c, cudaEventCreate(&e1));
  LAUNCH(c, launch_dfma(c->part(), blocks, 64, c->st));  // warm-up
  CK(c, cudaEventRecord(e0, c->st));
  LAUNCH(c, launch_dfma(c->part(), blocks, iters, c->st));
  CK(c, cudaEventRecord(e1, c->st));
  CK(c, cudaEventSynchronize(e1));
  float ms = 0;
  CK(c, cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8 * 8 * (double)iters * 256.0 * blocks;
  if (gflops_out) *gflops_out = flops / (ms * 1e-3) / 1e9;
  if (ms_out) *ms_out = ms;
  return TOMO_OK;
}

extern "C" int tomo_set_history(tomo_ctx* c, double* d_hist, int n) {
  if (int rc = need_bound(c)) return rc;
  if (n < 0 || (n > 0 && !check_ptr(d_hist))) return fail(c, TOMO_EINVAL, "bad history buffer");
  Scal* s = c->scal();
  double* h = n > 0 ? d_hist : nullptr;
  CK(c, cudaMemcpyAsync(&s->hist, &h, sizeof(h), cudaMemcpyHostToDevice, c->st));
  CK(c, cudaMemcpyAsync(&s->hist_n, &n, sizeof(n), cudaMemcpyHostToDevice, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TOMO_OK;
}

extern "C" int tomo_set_pcg_exact_beta(tomo_ctx* c, int on) {
  if (!c) return TOMO_EINVAL;
  c->exact_beta = on != 0;
  c->op_pcg[0].sep = c->op_pcg[1].sep = pcg_sep(c);
  if (c->bound) return build_pcg_graph(c);
  return TOMO_OK;
}

extern "C" int tomo_set_graph(tomo_ctx* c, int on) {
  if (!c) return TOMO_EINVAL;
  c->use_graph = on != 0;
  if (!c->bound) return TOMO_OK;  // built at tomo_bind
  if (c->use_graph && !c->pcg_exec) return build_pcg_graph(c);
  if (!c->use_graph) {
    if (c->pcg_exec) { cudaGraphExecDestroy(c->pcg_exec); c->pcg_exec = nullptr; }
    if (c->pcg_graph) { cudaGraphDestroy(c->pcg_graph); c->pcg_graph = nullptr; }
  }
  return TOMO_OK;
}

extern "C" int tomo_set_profiling(tomo_ctx* c, int on) {
  if (!c) return TOMO_EINVAL;
  c->prof = on != 0;
  c->prof_a_ms = c->prof_b_ms = 0;
  c->prof_n = 0;
  return TOMO_OK;
}

extern "C" int tomo_profile_times(const tomo_ctx* c, double* t) {
  if (!c || !t) return TOMO_EINVAL;
  t[0] = c->prof_n ? c->prof_a_ms / c->prof_n : 0.0;
  t[1] = 0.0;  // single-pass PCG: there is no separate K_B kernel
  t[2] = (double)c->prof_n;
  return TOMO_OK;
}

extern "C" int tomo_bench_apply(tomo_ctx* c, const double* d_rho, int reps, double* ms_out) {
  if (int rc = need_bound(c)) return rc;
  if (!check_ptr(d_rho) || reps < 1) return fail(c, TOMO_EINVAL, "bad argument");
  if (int rc = prepare_modulus(c, d_rho, false)) return rc;
  cudaEvent_t e0, e1;
  CK(c, cudaEventCreate(&e0));
  CK(c, cudaEventCreate(&e1));
  LAUNCH(c, launch_op(OP_APPLY, c->op_apply_u, c->ap_blocks, c->st));  // warm-up
  CK(c, cudaEventRecord(e0, c->st));
  // back-to-back applications chained by programmatic dependent launch (each waits for the
  // previous one's completion before it reads; TOMO_NO_PDL: launch-to-launch order)
  for (int i = 0; i < reps; ++i)
    LAUNCH(c, launch_op(OP_APPLY, c->op_apply_u, c->ap_blocks, c->st, c->pdl && i > 0));
  CK(c, cudaEventRecord(e1, c->st));
  CK(c, cudaEventSynchronize(e1));
  float ms = 0;
  CK(c, cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ms_out) *ms_out = ms / reps;
  return TOMO_OK;
}

// ====================================================================== two-scale coarse path
extern "C" int tomo_create_coarse(tomo_ctx** out, const tomo_ctx* f, int nb) {
  if (!out || !f) return TOMO_EINVAL;
  *out = nullptr;
  const Grid& g = f->g;
  if (nb < 1 || g.nx % nb || g.ny % nb || g.nz % nb) return TOMO_EINVAL;
  const int cx = g.nx / nb, cy = g.ny / nb, cz = g.nz / nb;
  // per-axis nearest coarse index, ties up (reading R4): I = floor((2 i + nb) / (2 nb))
  auto near = [nb](int i) { return (2 * i + nb) / (2 * nb); };
  auto cnode = [&](long long n) {
    const int i = (int)(n % g.nnx), j = (int)((n / g.nnx) % g.nny), k = (int)(n / ((long long)g.nnx * g.nny));
    return (long long)near(i) + (long long)(cx + 1) * (near(j) + (long long)(cy + 1) * near(k));
  };
  const long long nnc = (long long)(cx + 1) * (cy + 1) * (cz + 1);
  std::vector<uint8_t> mc((size_t)nnc, 0);
  for (long long n = 0; n < g.nn; ++n)
    if (f->mask[n]) mc[cnode(n)] |= f->mask[n];
  std::vector<int64_t> fixed;
  for (long long n = 0; n < nnc; ++n)
    for (int c = 0; c < 3; ++c)
      if ((mc[n] >> c) & 1) fixed.push_back(3 * n + c);
  std::vector<double> fc((size_t)(3 * nnc), 0.0);
  for (size_t l = 0; l < f->load_dofs.size(); ++l) {
    const int64_t d = f->load_dofs[l];
    fc[3 * cnode(d / 3) + d % 3] += f->load_vals[l];
  }
  std::vector<int64_t> ld;
  std::vector<double> lv;
  for (long long d = 0; d < 3 * nnc; ++d)
    if (fc[d] != 0.0) { ld.push_back(d); lv.push_back(fc[d]); }
  tomo_grid gc{cx, cy, cz, f->h * nb};
  tomo_bc bc{TOMO_BC_EXPLICIT, 0.0, fixed.data(), (int64_t)fixed.size(), ld.data(), lv.data(),
             (int64_t)ld.size()};
  return tomo_create(out, &gc, f->E0, f->Emin, f->nu, f->penal, f->rmin, &bc);
}

extern "C" int tomo_coarsen(tomo_ctx* c, const double* d_z, int nb, double* d_zc, int64_t n_ec) {
  if (int rc = need_bound(c)) return rc;
  const Grid& g = c->g;
  if (nb < 1 || g.nx % nb || g.ny % nb || g.nz % nb) return fail(c, TOMO_EINVAL, "nb must divide the grid (SPEC.md l.386)");
  if (n_ec != (int64_t)(g.nx / nb) * (g.ny / nb) * (g.nz / nb)) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_z) || !check_ptr(d_zc)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  LAUNCH(c, launch_coarsen(g, nb, d_z, d_zc, c->st));
  return TOMO_OK;
}

// ====================================================================== multigrid
namespace {

int mg_levels_possible(const Grid& g) {
  int L = 1;
  int x = g.nx, y = g.ny, z = g.nz;
  while (x % 2 == 0 && y % 2 == 0 && z % 2 == 0 && x >= 2 && y >= 2 && z >= 2) {
    x /= 2; y /= 2; z /= 2;
    ++L;
  }
  return L;
}

// APPLY with an arbitrary (padded, fine-level) input buffer: maps built at tomo_mg_bind
int mg_build_maps(tomo_ctx* c) {
  const Grid& g = c->g;
  const uint64_t rowv = 8ull * g.nnx_pad, planev = 3 * rowv * g.nny;  // row-SoA (dof_pad)
  const uint32_t inw = OP_TX + 2, inh = 3 * (OP_BY + 1);
  CUtensorMap tP, tZ;
  auto P = [&](size_t off) { return reinterpret_cast<double*>(c->mg_ws + off); };
  if (int rc = make_map(c, &tP, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, P(c->mg_off_P), g.nnx, 3ull * g.nny, g.nnz, rowv, planev, inw, inh)) return rc;
  if (int rc = make_map(c, &tZ, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, P(c->mg_off_Z), g.nnx, 3ull * g.nny, g.nnz, rowv, planev, inw, inh)) return rc;
  c->op_apply_P = c->op_apply_u;
  c->op_apply_P.tm_in = tP;
  c->op_apply_P.out = P(c->mg_off_Q);
  c->op_apply_P.u = P(c->mg_off_P);
  c->op_apply_Z = c->op_apply_u;
  c->op_apply_Z.tm_in = tZ;
  c->op_apply_Z.out = c->q(0);
  c->op_apply_Z.u = P(c->mg_off_Z);
  return TOMO_OK;
}

double* mgv(tomo_ctx* c, size_t off) { return reinterpret_cast<double*>(c->mg_ws + off); }

// Jacobi-PCG on context c with the right-hand side already in r(1) (padded): relative
// tolerance tol on ||b||, from u = 0 - the coarsest level of the V-cycle. At most `launches`
// fused PCG launches are issued without reading anything back (launches after convergence
// exit at their first instruction): no host synchronisation, so the V-cycle can be captured
// into a CUDA graph.
int pcg_rhs_fixed(tomo_ctx* c, double tol, int launches) {
  const Grid& g = c->g;
  const size_t vb = sizeof(double) * (size_t)g.ndof_pad;
  LAUNCH(c, launch_scal_init(c->scal(), 0.0, launches, c->st));
  LAUNCH(c, launch_norm2(g, c->r(1), c->scal(), c->part(), c->nb_b, c->st));
  LAUNCH(c, launch_set_tol(c->scal(), tol, c->st));
  CK(c, cudaMemsetAsync(c->u(), 0, vb, c->st));
  CK(c, cudaMemsetAsync(c->q(1), 0, vb, c->st));
  CK(c, cudaMemsetAsync(c->p(1), 0, vb, c->st));
  for (int k = 0; k <= launches; ++k) {
    LAUNCH(c, launch_op(OP_PCG, c->op_pcg[k & 1], c->op_blocks, c->st));
    if (c->op_pcg[0].sep) LAUNCH(c, launch_pcg_red(c->op_pcg[k & 1], c->op_blocks, c->st, false));
  }
  return TOMO_OK;
}

// x = V-cycle(b) on level l (l = 0: the fine context with outer buffers b = R, x = Z).
int mg_vcycle(tomo_ctx* f, int l, const double* b, double* x) {
  tomo_ctx* c = l == 0 ? f : f->mg[l - 1];
  const Grid& g = c->g;
  const int L = (int)f->mg.size() + 1;
  const size_t vb = sizeof(double) * (size_t)g.ndof_pad;
  if (l == L - 1) {  // coarsest: approximate solve by Jacobi-PCG
    if (b != c->r(1)) CK(c, cudaMemcpyAsync(c->r(1), b, vb, cudaMemcpyDeviceToDevice, c->st));
    if (int rc = pcg_rhs_fixed(c, f->mg_coarse_tol, f->mg_coarse_iters)) return rc;
    if (x != c->u()) CK(c, cudaMemcpyAsync(x, c->u(), vb, cudaMemcpyDeviceToDevice, c->st));
    return TOMO_OK;
  }
  const OpArgs& ax = l == 0 ? f->op_apply_Z : c->op_apply_u;  // K x -> c->q(0)
  const double om = f->mg_omega;
  // pre-smoothing from x = 0: the first sweep is x = omega D^-1 b
  CK(c, cudaMemsetAsync(x, 0, vb, c->st));
  CK(c, cudaMemsetAsync(c->q(0), 0, vb, c->st));
  for (int s = 0; s < f->mg_nu; ++s) {
    if (s > 0) LAUNCH(c, launch_op(OP_APPLY, ax, c->ap_blocks, c->st));
    LAUNCH(c, launch_jacobi_smooth(g, om, b, c->q(0), c->dinv(), c->dmask(), x, c->st));
  }
  // residual, restriction, coarse correction, prolongation
  tomo_ctx* n = f->mg[l];
  LAUNCH(c, launch_op(OP_APPLY, ax, c->ap_blocks, c->st));
  LAUNCH(c, launch_residual(g, b, c->q(0), c->dmask(), c->r(1), c->st));
  const bool coarsest_next = (l + 1 == L - 1);
  double* bn = coarsest_next ? n->r(1) : n->r(0);
  LAUNCH(c, launch_restrict(g, n->g, c->r(1), n->dmask(), bn, c->st));
  if (int rc = mg_vcycle(f, l + 1, bn, n->u())) return rc;
  LAUNCH(c, launch_prolong_add(g, n->g, n->u(), c->dmask(), x, c->st));
  // post-smoothing (same sweeps: symmetric cycle)
  for (int s = 0; s < f->mg_nu; ++s) {
    LAUNCH(c, launch_op(OP_APPLY, ax, c->ap_blocks, c->st));
    LAUNCH(c, launch_jacobi_smooth(g, om, b, c->q(0), c->dinv(), c->dmask(), x, c->st));
  }
  return TOMO_OK;
}

}  // namespace

extern "C" size_t tomo_mg_workspace_bytes(tomo_ctx* c, int levels) {
  if (!c || levels < 2 || levels > mg_levels_possible(c->g)) return 0;
  if ((int)c->mg.size() != levels - 1) {
    for (auto* l : c->mg) tomo_destroy(l);
    c->mg.clear();
    c->mg_bound = false;
    const tomo_ctx* prev = c;
    for (int l = 1; l < levels; ++l) {
      tomo_ctx* n = nullptr;
      if (tomo_create_coarse(&n, prev, 2) != TOMO_OK) {
        if (n) tomo_destroy(n);
        for (auto* x : c->mg) tomo_destroy(x);
        c->mg.clear();
        return 0;
      }
      c->mg.push_back(n);
      prev = n;
    }
  }
  size_t o = 0;
  c->mg_level_off.clear();
  for (auto* l : c->mg) {
    c->mg_level_off.push_back(o);
    o = align_up(o + l->off_end);
  }
  const size_t vp = sizeof(double) * (size_t)c->g.ndof_pad;
  c->mg_off_U = o; o = align_up(o + vp);
  c->mg_off_R = o; o = align_up(o + vp);
  c->mg_off_P = o; o = align_up(o + vp);
  c->mg_off_Q = o; o = align_up(o + vp);
  c->mg_off_Z = o; o = align_up(o + vp);
  c->mg_off_Zo = o; o = align_up(o + vp);
  c->mg_off_part = o; o = align_up(o + sizeof(double) * 3 * 4 * 1024);
  c->mg_off_fs = o; o = align_up(o + sizeof(FcgScal));
  c->mg_end = o;
  return o;
}

extern "C" int tomo_mg_bind(tomo_ctx* c, int levels, void* d_ws, size_t bytes) {
  if (int rc = need_bound(c)) return rc;
  const size_t need = tomo_mg_workspace_bytes(c, levels);
  if (!need) return fail(c, TOMO_EINVAL, "levels must be >= 2 and the grid divisible by 2^(levels-1)");
  if (!d_ws || (reinterpret_cast<uintptr_t>(d_ws) & 255)) return fail(c, TOMO_EINVAL, "MG workspace must be 256-B aligned");
  if (bytes < need) return fail(c, TOMO_ENOWORKSPACE, "MG workspace too small");
  c->mg_ws = static_cast<char*>(d_ws);
  CK(c, cudaMemsetAsync(c->mg_ws, 0, need, c->st));
  for (size_t l = 0; l < c->mg.size(); ++l) {
    if (int rc = tomo_bind(c->mg[l], c->mg_ws + c->mg_level_off[l], c->mg[l]->off_end, c->st))
      return fail(c, rc, std::string("binding MG level: ") + tomo_last_error(c->mg[l]));
  }
  if (int rc = mg_build_maps(c)) return rc;
  if (c->mg_exec) { cudaGraphExecDestroy(c->mg_exec); c->mg_exec = nullptr; }
  if (c->mg_graph) { cudaGraphDestroy(c->mg_graph); c->mg_graph = nullptr; }
  c->mg_bound = true;
  return TOMO_OK;
}

extern "C" int tomo_solve_mg(tomo_ctx* c, const double* d_rho, int64_t n_e, double* d_u,
                             int64_t n_dof, double tol, int max_iters, tomo_solve_info* info) {
  Range nvtx_range("tomo_solve_mg");
  if (int rc = need_bound(c)) return rc;
  if (!c->mg_bound) return fail(c, TOMO_ENOWORKSPACE, "call tomo_mg_bind first");
  if (n_e != c->g.ne || n_dof != c->g.ndof) return fail(c, TOMO_ESIZE, "length mismatch");
  if (!check_ptr(d_rho) || !check_ptr(d_u)) return fail(c, TOMO_EINVAL, "NULL or misaligned pointer");
  if (c->fnorm == 0.0) {
    CK(c, cudaMemsetAsync(d_u, 0, sizeof(double) * (size_t)n_dof, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    if (info) *info = tomo_solve_info{0, 1, 0.0, 0.0};
    return 0;
  }
  const Grid& g = c->g;
  const long long n = g.ndof_pad;
  const size_t vb = sizeof(double) * (size_t)n;
  if (int rc = prepare_modulus(c, d_rho, true)) return rc;
  // coarse levels: E averaged over the 8 children, their own Jacobi diagonals
  const tomo_ctx* prev = c;
  for (auto* l : c->mg) {
    LAUNCH(c, launch_coarsen_E(prev->g, l->g, prev->E(), l->E(), c->mg_emode, c->st));
    LAUNCH(c, launch_jacobi(l->g, l->E(), l->ke_diag, l->dinv(), c->st));
    prev = l;
  }
  double *U = mgv(c, c->mg_off_U), *R = mgv(c, c->mg_off_R), *Pv = mgv(c, c->mg_off_P),
         *Q = mgv(c, c->mg_off_Q), *Z = mgv(c, c->mg_off_Z), *Zo = mgv(c, c->mg_off_Zo);
  FcgScal* fs = reinterpret_cast<FcgScal*>(c->mg_ws + c->mg_off_fs);
  double* part = mgv(c, c->mg_off_part);
  const int nb = std::min(c->sms * 4, 4 * 1024);
  // x0 = 0, r0 = f (the flexible CG runs from a cold start, reading A12); scalars on the device
  CK(c, cudaMemsetAsync(U, 0, vb, c->st));
  CK(c, cudaMemsetAsync(c->q(0), 0, vb, c->st));
  LAUNCH(c, launch_resid(g, c->q(0), R, c->ldp(), c->lv(), (int)c->load_dofs.size(), c->st));
  if (int rc = mg_vcycle(c, 0, R, Z)) return rc;
  CK(c, cudaMemcpyAsync(Pv, Z, vb, cudaMemcpyDeviceToDevice, c->st));
  LAUNCH(c, launch_fcg_init(fs, tol * c->fnorm, max_iters, c->st));
  LAUNCH(c, launch_fcg_dot(n, R, Z, nullptr, part, nb, fs, FCG_INIT, 0, c->st));
  // one outer iteration: Q = K P, alpha, U/R update, Z = V-cycle(R), beta + stop test, P update
  auto iteration = [&](unsigned long long cond) -> int {
    LAUNCH(c, launch_op(OP_APPLY, c->op_apply_P, c->ap_blocks, c->st));
    LAUNCH(c, launch_fcg_dot(n, Pv, Q, nullptr, part, nb, fs, FCG_ALPHA, 0, c->st));
    LAUNCH(c, launch_fcg_axpy2(n, fs, Pv, U, Q, R, c->st));
    CK(c, cudaMemcpyAsync(Zo, Z, vb, cudaMemcpyDeviceToDevice, c->st));
    if (int rc = mg_vcycle(c, 0, R, Z)) return rc;
    LAUNCH(c, launch_fcg_dot(n, R, Z, Zo, part, nb, fs, FCG_BETA, cond, c->st));
    LAUNCH(c, launch_fcg_xpby(n, fs, Z, Pv, c->st));
    return TOMO_OK;
  };
  FcgScal hf{};
  if (c->use_graph) {
    // the whole loop as one graph: a conditional WHILE node whose body is one iteration,
    // captured from the stream; the beta/stop reduction clears the condition
    if (!c->mg_exec) {
      CK(c, cudaGraphCreate(&c->mg_graph, 0));
      cudaGraphConditionalHandle h;
      CK(c, cudaGraphConditionalHandleCreate(&h, c->mg_graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t cnode;
      CK(c, cudaGraphAddNode(&cnode, c->mg_graph, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      // capture on a private stream (the bound one may be the legacy default stream, which
      // cannot capture); every level's launches are redirected to it meanwhile
      cudaStream_t cs = nullptr;
      CK(c, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      std::vector<tomo_ctx*> all{c};
      for (auto* l : c->mg) all.push_back(l);
      const cudaStream_t bound = c->st;
      for (auto* x : all) x->st = cs;
      cudaError_t ec = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
      int rc = TOMO_OK;
      if (ec == cudaSuccess) {
        rc = iteration(h);
        cudaGraph_t captured = nullptr;
        ec = cudaStreamEndCapture(cs, &captured);
      }
      for (auto* x : all) x->st = bound;
      cudaStreamDestroy(cs);
      if (rc) return rc;
      CK(c, ec);
      CK(c, cudaGraphInstantiate(&c->mg_exec, c->mg_graph, 0));
    }
    CK(c, cudaGraphLaunch(c->mg_exec, c->st));
    CK(c, cudaMemcpyAsync(&hf, fs, sizeof(hf), cudaMemcpyDeviceToHost, c->st));
    CK(c, cudaStreamSynchronize(c->st));
  } else {
    for (;;) {  // host-batched iterations, the scalars read back every 8
      for (int i = 0; i < 8; ++i)
        if (int rc = iteration(0)) return rc;
      CK(c, cudaMemcpyAsync(&hf, fs, sizeof(hf), cudaMemcpyDeviceToHost, c->st));
      CK(c, cudaStreamSynchronize(c->st));
      if (hf.done) break;
    }
  }
  if (hf.done == 3)
    return fail(c, hf.status ? hf.status : TOMO_EBREAKDOWN,
                hf.status == TOMO_ENAN ? "NaN/Inf in MG-CG" : "MG-CG breakdown: p^T K p <= 0");
  const int k = hf.k;
  const bool conv = hf.done == 1;
  const double rr = hf.rr, stop = tol * c->fnorm;
  // true residual, then u out
  CK(c, cudaMemcpyAsync(c->u(), U, vb, cudaMemcpyDeviceToDevice, c->st));
  LAUNCH(c, launch_op(OP_APPLY, c->op_apply_u, c->ap_blocks, c->st));
  LAUNCH(c, launch_resid(g, c->q(0), c->r(0), c->ldp(), c->lv(), (int)c->load_dofs.size(), c->st));
  LAUNCH(c, launch_norm2(g, c->r(0), c->scal(), c->part(), c->nb_b, c->st));
  LAUNCH(c, launch_unpack(g, U, d_u, c->st));
  double rrt = 0;
  CK(c, cudaMemcpyAsync(&rrt, &c->scal()->rr_true, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  if (info) {
    info->iterations = k;
    info->converged = !conv ? 0 : (std::sqrt(rrt) <= stop ? 1 : 2);  // as tomo_solve (tomo.h)
    info->rel_res_recursive = std::sqrt(rr) / c->fnorm;
    info->rel_res_true = std::sqrt(rrt) / c->fnorm;
  }
  return k;
}

extern "C" int tomo_mg_params(tomo_ctx* c, int nu, double omega, int coarse_iters, double coarse_tol) {
  if (!c || nu < 1 || !(omega > 0 && omega < 2) || coarse_iters < 1 || !(coarse_tol > 0)) return TOMO_EINVAL;
  if (c->mg_exec) { cudaGraphExecDestroy(c->mg_exec); c->mg_exec = nullptr; }
  if (c->mg_graph) { cudaGraphDestroy(c->mg_graph); c->mg_graph = nullptr; }
  c->mg_nu = nu;
  c->mg_omega = omega;
  c->mg_coarse_iters = coarse_iters;
  c->mg_coarse_tol = coarse_tol;
  return TOMO_OK;
}
