// libtomo multigrid kernels ("Iterative solvers such
// as preconditioned conjugate gradient (PCG) and multi-grid methods are typically used").
//
// Geometric multigrid on the structured grid, used as the preconditioner of a flexible CG:
//   level l+1 = level l coarsened by 2 per axis, element edge 2h, E averaged over the 8
//   children (rediscretisation), BCs restricted by tomo_create_coarse (reading R4);
//   V-cycle: damped Jacobi smoothing (the same operator kernel), full-weighting restriction
//   R = P^T, trilinear prolongation P; fixed DOFs are zero in every correction.
// All vectors are in the padded internal layout of their level (tomo_internal.h).
#include "tomo_internal.h"

namespace tomo {
namespace {

inline unsigned nblk(long long n, int bs, int cap) {
  long long b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

__device__ __forceinline__ void node_of(const Grid& g, long long n, int& i, int& j, int& k) {
  i = (int)(n % g.nnx);
  j = (int)((n / g.nnx) % g.nny);
  k = (int)(n / ((long long)g.nnx * g.nny));
}

// x += omega D^-1 (b - Kx) on free DOFs (Kx: the operator applied to x)
__global__ void k_jacobi_smooth(Grid g, double omega, const double* __restrict__ b,
                                const double* __restrict__ kx, const double* __restrict__ dinv,
                                const uint8_t* __restrict__ mask, double* __restrict__ x) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    int i, j, k;
    node_of(g, n, i, j, k);
    const unsigned m = mask[mask_index(g, i, j, k)];
    const double w = omega * dinv[node_pad(g, i, j, k)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long p = dof_pad(g, i, j, k, c);
      x[p] = ((m >> c) & 1u) ? 0.0 : fma(w, b[p] - kx[p], x[p]);
    }
  }
}

// r = b - Kx on free DOFs (0 at fixed DOFs)
__global__ void k_residual(Grid g, const double* __restrict__ b, const double* __restrict__ kx,
                           const uint8_t* __restrict__ mask, double* __restrict__ r) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    int i, j, k;
    node_of(g, n, i, j, k);
    const unsigned m = mask[mask_index(g, i, j, k)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long p = dof_pad(g, i, j, k, c);
      r[p] = ((m >> c) & 1u) ? 0.0 : b[p] - kx[p];
    }
  }
}

// 1-D trilinear weight of fine index f for coarse index C (f = 2C + d, |d| <= 1)
__device__ __forceinline__ double w1(int f, int C) {
  const int d = f - 2 * C;
  return d == 0 ? 1.0 : ((d == 1 || d == -1) ? 0.5 : 0.0);
}

// rc = P^T rf (full weighting: 27 fine nodes around 2C with weights prod (1 - |d|/2));
// zero at coarse fixed DOFs. Fixed summation order dz, dy, dx.
__global__ void k_restrict(Grid gf, Grid gc, const double* __restrict__ rf,
                           const uint8_t* __restrict__ maskc, double* __restrict__ rc) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < gc.nn; n += stride) {
    int I, J, K;
    node_of(gc, n, I, J, K);
    double s[3] = {0.0, 0.0, 0.0};
    for (int dz = -1; dz <= 1; ++dz) {
      const int k = 2 * K + dz;
      if (k < 0 || k > gf.nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int j = 2 * J + dy;
        if (j < 0 || j > gf.ny) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int i = 2 * I + dx;
          if (i < 0 || i > gf.nx) continue;
          const double w = w1(i, I) * w1(j, J) * w1(k, K);
#pragma unroll
          for (int c = 0; c < 3; ++c) s[c] = fma(w, rf[dof_pad(gf, i, j, k, c)], s[c]);
        }
      }
    }
    const unsigned m = maskc[mask_index(gc, I, J, K)];
#pragma unroll
    for (int c = 0; c < 3; ++c) rc[dof_pad(gc, I, J, K, c)] = ((m >> c) & 1u) ? 0.0 : s[c];
  }
}

// xf += P xc (trilinear interpolation from the coarse nodes around f/2); zero at fine fixed
__global__ void k_prolong_add(Grid gf, Grid gc, const double* __restrict__ xc,
                              const uint8_t* __restrict__ maskf, double* __restrict__ xf) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < gf.nn; n += stride) {
    int i, j, k;
    node_of(gf, n, i, j, k);
    double s[3] = {0.0, 0.0, 0.0};
    for (int K = k >> 1; K <= (k + 1) >> 1; ++K) {
      if (K > gc.nz) continue;
      const double wz = w1(k, K);
      for (int J = j >> 1; J <= (j + 1) >> 1; ++J) {
        if (J > gc.ny) continue;
        const double wy = wz * w1(j, J);
        for (int I = i >> 1; I <= (i + 1) >> 1; ++I) {
          if (I > gc.nx) continue;
          const double w = wy * w1(i, I);
#pragma unroll
          for (int c = 0; c < 3; ++c) s[c] = fma(w, xc[dof_pad(gc, I, J, K, c)], s[c]);
        }
      }
    }
    const unsigned m = maskf[mask_index(gf, i, j, k)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long p = dof_pad(gf, i, j, k, c);
      xf[p] = ((m >> c) & 1u) ? 0.0 : xf[p] + s[c];
    }
  }
}

// coarse E from the 8 child elements' E (padded element layouts on both levels):
// mode 0 arithmetic mean, 1 geometric mean, 2 harmonic mean
__global__ void k_coarsen_E(Grid gf, Grid gc, const double* __restrict__ Ef, double* __restrict__ Ec,
                            int mode) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < gc.ne; e += stride) {
    const int I = (int)(e % gc.nx), J = (int)((e / gc.nx) % gc.ny), K = (int)(e / ((long long)gc.nx * gc.ny));
    double s = 0.0;
    for (int k = 2 * K; k < 2 * K + 2; ++k)
      for (int j = 2 * J; j < 2 * J + 2; ++j)
        for (int i = 2 * I; i < 2 * I + 2; ++i) {
          const double v = Ef[elem_pad(gf, i, j, k)];
          s += mode == 0 ? v : (mode == 1 ? log(v) : 1.0 / v);
        }
    Ec[elem_pad(gc, I, J, K)] = mode == 0 ? 0.125 * s : (mode == 1 ? exp(0.125 * s) : 8.0 / s);
  }
}

// ---- flexible-CG vector kernels (flat over padded vectors; pads are 0) -----------------
}  // namespace

cudaError_t launch_jacobi_smooth(const Grid& g, double omega, const double* b, const double* kx,
                                 const double* dinv, const uint8_t* mask, double* x, cudaStream_t st) {
  k_jacobi_smooth<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, omega, b, kx, dinv, mask, x);
  return cudaGetLastError();
}
cudaError_t launch_residual(const Grid& g, const double* b, const double* kx, const uint8_t* mask,
                            double* r, cudaStream_t st) {
  k_residual<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, b, kx, mask, r);
  return cudaGetLastError();
}
cudaError_t launch_restrict(const Grid& gf, const Grid& gc, const double* rf, const uint8_t* maskc,
                            double* rc, cudaStream_t st) {
  k_restrict<<<nblk(gc.nn, 256, 148 * 16), 256, 0, st>>>(gf, gc, rf, maskc, rc);
  return cudaGetLastError();
}
cudaError_t launch_prolong_add(const Grid& gf, const Grid& gc, const double* xc,
                               const uint8_t* maskf, double* xf, cudaStream_t st) {
  k_prolong_add<<<nblk(gf.nn, 256, 148 * 16), 256, 0, st>>>(gf, gc, xc, maskf, xf);
  return cudaGetLastError();
}
cudaError_t launch_coarsen_E(const Grid& gf, const Grid& gc, const double* Ef, double* Ec,
                             int mode, cudaStream_t st) {
  k_coarsen_E<<<nblk(gc.ne, 256, 148 * 16), 256, 0, st>>>(gf, gc, Ef, Ec, mode);
  return cudaGetLastError();
}

namespace {
// ---------------------------------------------------------------- device-resident flexible CG
// The MG-preconditioned flexible CG with its scalars on the device (no host round trip per
// iteration), so that a whole outer iteration can be captured into a CUDA graph.
// k_fcg_dot: block partials of up to three dots of one pass; the last block sums them in
// block order (deterministic) and applies the step `mode`:
//   FCG_INIT  (a = R, b = Z):       rz = R.Z, rr = R.R; done if ||R|| <= stop
//   FCG_ALPHA (a = P, b = Q):       alpha = rz / P.Q  (breakdown / NaN -> done = 3)
//   FCG_BETA  (a = R, b = Z, c = Zo): rr = R.R; done = 1 if ||R|| <= stop, = 2 at max_iters;
//                                   else beta = (R.Z - R.Zo) / rz (Polak-Ribiere), rz = R.Z
// and clears the graph's WHILE condition when done. Every kernel of the iteration returns at
// once when `done` is set.
__device__ __forceinline__ double fcg_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) k_fcg_dot(long long n, const double* __restrict__ a,
                                                 const double* __restrict__ b,
                                                 const double* __restrict__ c, double* partials,
                                                 FcgScal* s, int mode, unsigned long long cond) {
  __shared__ double red[3][8];
  __shared__ int last;
  if (mode != FCG_INIT && *(volatile int*)&s->done) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n; d += stride) {
    const double av = a[d];
    s0 = fma(av, b[d], s0);
    if (c) s1 = fma(av, c[d], s1);
    s2 = fma(av, av, s2);
  }
  s0 = fcg_warp_sum(s0);
  s1 = fcg_warp_sum(s1);
  s2 = fcg_warp_sum(s2);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[0][w] = s0; red[1][w] = s1; red[2][w] = s2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { t0 += red[0][i]; t1 += red[1][i]; t2 += red[2][i]; }
    partials[3 * blockIdx.x] = t0;
    partials[3 * blockIdx.x + 1] = t1;
    partials[3 * blockIdx.x + 2] = t2;
    __threadfence();
    last = atomicAdd(&s->cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  double d0 = 0.0, d1 = 0.0, d2 = 0.0;
  for (unsigned i = 0; i < gridDim.x; ++i) {
    d0 += __ldcg(partials + 3 * i);
    d1 += __ldcg(partials + 3 * i + 1);
    d2 += __ldcg(partials + 3 * i + 2);
  }
  s->cnt = 0;
  if (mode == FCG_INIT) {
    s->rz = d0;
    s->rr = d2;
    s->k = 0;
    s->done = sqrt(d2) <= s->stop ? 1 : 0;
  } else if (mode == FCG_ALPHA) {
    if (!(d0 > 0.0) || !isfinite(d0)) {
      s->done = 3;
      s->status = isnan(d0) ? -6 : -4;  // TOMO_ENAN / TOMO_EBREAKDOWN
    } else {
      s->alpha = s->rz / d0;
    }
  } else {
    s->k += 1;
    s->rr = d2;
    if (!isfinite(d2)) {
      s->done = 3;
      s->status = -6;
    } else if (sqrt(d2) <= s->stop) {
      s->done = 1;
    } else if (s->k >= s->max_iters) {
      s->done = 2;
    } else {
      s->beta = (d0 - d1) / s->rz;
      s->rz = d0;
    }
  }
  __threadfence();
  if (cond && s->done) cudaGraphSetConditional(cond, 0u);
}

// U += alpha P ; R -= alpha Q (alpha from the device scalars)
__global__ void k_fcg_axpy2(long long n, const FcgScal* s, const double* __restrict__ P,
                            double* __restrict__ U, const double* __restrict__ Q,
                            double* __restrict__ R) {
  if (*(volatile const int*)&s->done) return;
  const double a = s->alpha;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n; d += stride) {
    U[d] = fma(a, P[d], U[d]);
    R[d] = fma(-a, Q[d], R[d]);
  }
}

// P = Z + beta P
__global__ void k_fcg_xpby(long long n, const FcgScal* s, const double* __restrict__ Z,
                           double* __restrict__ P) {
  if (*(volatile const int*)&s->done) return;
  const double b = s->beta;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n; d += stride)
    P[d] = fma(b, P[d], Z[d]);
}

__global__ void k_fcg_init(FcgScal* s, double stop, int max_iters) {
  s->rz = s->rr = s->alpha = s->beta = 0.0;
  s->stop = stop;
  s->k = 0;
  s->done = 0;
  s->status = 0;
  s->max_iters = max_iters;
  s->cnt = 0;
}

}  // namespace

cudaError_t launch_fcg_dot(long long n, const double* a, const double* b, const double* c,
                           double* partials, int nblocks, FcgScal* s, int mode,
                           unsigned long long cond, cudaStream_t st) {
  k_fcg_dot<<<nblocks, 256, 0, st>>>(n, a, b, c, partials, s, mode, cond);
  return cudaGetLastError();
}
cudaError_t launch_fcg_axpy2(long long n, const FcgScal* s, const double* P, double* U,
                             const double* Q, double* R, cudaStream_t st) {
  k_fcg_axpy2<<<nblk(n, 256, 148 * 8), 256, 0, st>>>(n, s, P, U, Q, R);
  return cudaGetLastError();
}
cudaError_t launch_fcg_xpby(long long n, const FcgScal* s, const double* Z, double* P,
                            cudaStream_t st) {
  k_fcg_xpby<<<nblk(n, 256, 148 * 8), 256, 0, st>>>(n, s, Z, P);
  return cudaGetLastError();
}
cudaError_t launch_fcg_init(FcgScal* s, double stop, int max_iters, cudaStream_t st) {
  k_fcg_init<<<1, 1, 0, st>>>(s, stop, max_iters);
  return cudaGetLastError();
}

}  // namespace tomo
