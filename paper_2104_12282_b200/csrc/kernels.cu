// libtomo kernels for sm_100a: the exact-gradient evaluation of arXiv 2104.12282.
//
//   k_op<OP_APPLY>  y = K_hat(rho) u
//   k_op<OP_PCG>    one single-pass Jacobi-PCG iteration: r = r_old - alpha q_old,
//                   p = D^-1 r + beta p_old, u += alpha p_old, q = K_hat p, and the block
//                   partials of p.q, r.z, r.r (+ the beta prediction terms); the last block
//                   sets alpha, beta and the stop flag
//   k_simp/k_jacobi SIMP modulus and Jacobi diagonal
//   k_sens          Eq. 5 sensitivity
//   k_filter        density filter P / P^T
//   k_oc            OC update with device bisection
//
// Operator design. KE is never stored: in the tensor-Walsh basis of corner
// values the 24x24 KE has 45 non-zeros. The operator takes the 2-D Walsh transform of every
// node plane once per element column (shared by the two elements stacked on it), applies
// the 7-coefficient core scaled by E_e, transforms back, and accumulates the top face of
// one element with the bottom face of the next. A 32 x 8 block owns a 30 x 7 column of
// output nodes and marches along z through a chunk of node planes. Every input plane tile
// (vector incl. halo, Jacobi, mask bytes, E, owned u) is fetched by ONE thread with TMA
// (cp.async.bulk.tensor, OOB zero fill gives the domain boundary for free) into an
// OP_NS-stage (PCG) / OP_NS_APPLY-stage (K_hat u) mbarrier pipeline.
// All reductions are two-stage and deterministic (fixed partition, fixed-order final sum
// by the last block); there are no floating-point atomics.
#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>

#include "tomo_internal.h"

namespace cg = cooperative_groups;

namespace tomo {
namespace {

constexpr int TX = 32;
constexpr int BY = OP_BY;
constexpr int NT = TX * BY;            // threads per operator block
constexpr int OX = OP_OX;              // output nodes per tile along x
constexpr int OY = OP_OY;              // output nodes per tile along y
constexpr int NS = OP_NS;              // pipeline stages
constexpr int NR = BY + 1;             // node rows per tile (warp w stages rows w, w+1)
constexpr int ER = BY;                 // element rows per tile (one per warp)
// Internal vectors are row-SoA (tomo_internal.h dof_pad): a node row is 3 component
// sub-rows of nnx_pad doubles, so lane tx <-> node i0-1+tx reads and writes one component
// of 32 consecutive nodes per instruction (coalesced global stores, conflict-free smem).
// TMA boxes. The innermost box start must be 16-byte aligned (measured on this B200: an
// 8-byte-aligned start faults with "illegal instruction"), so every box starts at the
// aligned-down coordinate and is widened; smem reads add the per-block offset.
constexpr int VB_W = TX + 2;           // 34 doubles per component sub-row (start offset 0..1)
constexpr int VB_R = 3 * NR;           // 27 sub-rows: node rows j0-1 .. j0+BY-1, 3 components
constexpr int UB_R = 3 * OY;           // 21 sub-rows: owned node rows j0 .. j0+OY-1 (u, PCG)
constexpr int DB_W = TX + 2;           // 34 doubles: Jacobi rows (start offset 0..1)
constexpr int MB_W = 48;               // 48 bytes: mask rows (start offset 0..15)
constexpr int E_W = 32;                // element box width (start offset 0..1, 31 used)
constexpr int GSN = 12;                // top face carried as Walsh face modes
// stage layout in doubles, every piece 128-byte aligned
constexpr int al16(int n) { return (n + 15) & ~15; }  // doubles -> multiple of 128 B
constexpr int R_OFF = 0;                                       // r_{k-1} (APPLY: u)
constexpr int QO_OFF = R_OFF + al16(VB_W * VB_R);              // q_{k-1}
constexpr int PO_OFF = QO_OFF + al16(VB_W * VB_R);             // p_{k-1}
constexpr int UO_OFF = PO_OFF + al16(VB_W * VB_R);             // u, owned rows
constexpr int DI_OFF = UO_OFF + al16(VB_W * UB_R);             // D^-1
constexpr int EE_OFF = DI_OFF + al16(DB_W * NR);               // E
constexpr int MK_OFF = EE_OFF + al16(E_W * ER);                // mask bytes
constexpr int STAGE = MK_OFF + al16((MB_W * NR + 7) / 8);
constexpr unsigned BYTES_PCG =
    8u * (3 * VB_W * VB_R + VB_W * UB_R + DB_W * NR + E_W * ER) + MB_W * NR;
constexpr unsigned BYTES_APPLY = 8u * (VB_W * VB_R + E_W * ER) + MB_W * NR;
// APPLY stages hold only u, E and the mask (9.7 KB): more of them fit, and they are needed
// because a stage carries too few bytes to cover DRAM latency with two
constexpr int NS_A = OP_NS_APPLY;
constexpr int EE_OFF_A = al16(VB_W * VB_R);
constexpr int MK_OFF_A = EE_OFF_A + al16(E_W * ER);
constexpr int STAGE_A = MK_OFF_A + al16((MB_W * NR + 7) / 8);

// per-mode pipeline geometry
template <int MODE> struct Lay {
  static constexpr int ns = NS, stage = STAGE, ee = EE_OFF, mk = MK_OFF;
  static constexpr unsigned bytes = BYTES_PCG;
};
template <> struct Lay<OP_APPLY> {
  static constexpr int ns = NS_A, stage = STAGE_A, ee = EE_OFF_A, mk = MK_OFF_A;
  static constexpr unsigned bytes = BYTES_APPLY;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Tensor memory as thread-private storage (TOMO_GS_TMEM, A/B): shape 32x32b = lane l of warp w
// reads/writes its own 32-bit cells at TMEM lane 32 (w % 4) + l, columns col .. col + 7
__device__ __forceinline__ void tmem_ld8(unsigned taddr, unsigned (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(unsigned taddr, const unsigned (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum; result valid in every thread. `red` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int t = threadIdx.x + blockDim.x * threadIdx.y;
  const int nt = blockDim.x * blockDim.y;
  v = warp_sum(v);
  __syncthreads();
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (t < 32) {
    r = (t < (nt >> 5)) ? red[t] : 0.0;
    r = warp_sum(r);
    if (t == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  return r;
}

// Two-stage reduction: block partials, then the last block to arrive sums all partials in
// block order (the result does not depend on which block is last).
__device__ __forceinline__ bool arrive_last(unsigned* cnt, unsigned nblocks, int* s_flag) {
  const int t = threadIdx.x + blockDim.x * threadIdx.y;
  __syncthreads();
  if (t == 0) {
#if TOMO_ACQREL_ARRIVE
    // one acq_rel atomic: releases this block's partials, and the last block acquires all
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
#else
    __threadfence();
    unsigned prev = atomicAdd(cnt, 1u);
#endif
    *s_flag = (prev == nblocks - 1);
  }
  __syncthreads();
  return *s_flag != 0;
}

__device__ __forceinline__ double sum_partials(const double* p, int n, int stride, int off,
                                               double* red) {
  const int t = threadIdx.x + blockDim.x * threadIdx.y;
  const int nt = blockDim.x * blockDim.y;
  double acc = 0.0;
  for (int i = t; i < n; i += nt) acc += __ldcg(p + (long long)i * stride + off);
  return block_sum(acc, red);
}

// Five deterministic block sums at once (one pass of barriers); result in every thread.
__device__ __forceinline__ void block_sum5(double (&v)[5], double* red) {
  const int t = threadIdx.x + blockDim.x * threadIdx.y;
  const int nw = (blockDim.x * blockDim.y) >> 5;
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if ((t & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 5; ++i) red[i * 32 + (t >> 5)] = v[i];
  }
  __syncthreads();
  if (t < 32) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      double r = (t < nw) ? red[i * 32 + t] : 0.0;
      r = warp_sum(r);
      if (t == 0) red[160 + i] = r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = red[160 + i];
  __syncthreads();
}

// ------------------------------------------------------------------ Walsh element core
// Face transform of the 4 corner nodes (X..X+1, Y..Y+1) of one node plane, per component:
// modes 00 (sum), 10 (x difference), 01 (y difference), 11 (xy). F[m*3 + c].
__device__ __forceinline__ void face_from(double a00, double a10, double a01, double a11,
                                          double* F, int c) {
  const double s0 = a00 + a10, d0 = a10 - a00, s1 = a01 + a11, d1 = a11 - a01;
  F[0 + c] = s0 + s1;
  F[3 + c] = d0 + d1;
  F[6 + c] = s1 - s0;
  F[9 + c] = d1 - d0;
}

// v = E * D * w for one element, w built from the faces below (lo) and above (hi); returns
// the per-face inverse transforms Gb (z = 0 corners) and Gt (z = 1 corners).
__device__ __forceinline__ void element_core(const double (&Flo)[12], const double (&Fhi)[12],
                                             double E, const Walsh& W, double (&Gb)[12],
                                             double (&Gt)[12]) {
  double wx[3], wy[3], wz[3], wxy[3], wxz[3], wyz[3], wxyz[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    wx[c] = Flo[3 + c] + Fhi[3 + c];
    wy[c] = Flo[6 + c] + Fhi[6 + c];
    wz[c] = Fhi[0 + c] - Flo[0 + c];
    wxy[c] = Flo[9 + c] + Fhi[9 + c];
    wxz[c] = Fhi[3 + c] - Flo[3 + c];
    wyz[c] = Fhi[6 + c] - Flo[6 + c];
    wxyz[c] = Fhi[9 + c] - Flo[9 + c];
  }
  const double A = E * W.amb, B = E * W.b, G = E * W.g;
  const double C1 = E * W.c1, C2 = E * W.c2, C3 = E * W.c3, C4 = E * W.c4;
  double vx[3], vy[3], vz[3], vxy[3], vxz[3], vyz[3], vxyz[3];
  const double Bt = B * (wx[0] + wy[1] + wz[2]);
  vx[0] = fma(A, wx[0], Bt);
  vy[1] = fma(A, wy[1], Bt);
  vz[2] = fma(A, wz[2], Bt);
  const double sxy = G * (wx[1] + wy[0]);
  const double sxz = G * (wx[2] + wz[0]);
  const double syz = G * (wy[2] + wz[1]);
  vx[1] = sxy; vy[0] = sxy;
  vx[2] = sxz; vz[0] = sxz;
  vy[2] = syz; vz[1] = syz;
  const double s = wxy[2] + wxz[1] + wyz[0];
  vxy[2] = C3 * (s + wxy[2]);
  vxz[1] = C3 * (s + wxz[1]);
  vyz[0] = C3 * (s + wyz[0]);
  vxy[0] = fma(C1, wxy[0], C2 * wyz[2]);
  vxy[1] = fma(C1, wxy[1], C2 * wxz[2]);
  vxz[0] = fma(C1, wxz[0], C2 * wyz[1]);
  vxz[2] = fma(C1, wxz[2], C2 * wxy[1]);
  vyz[1] = fma(C1, wyz[1], C2 * wxz[0]);
  vyz[2] = fma(C1, wyz[2], C2 * wxy[0]);
#pragma unroll
  for (int c = 0; c < 3; ++c) vxyz[c] = C4 * wxyz[c];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    Gb[0 + c] = -vz[c];
    Gt[0 + c] = vz[c];
    Gb[3 + c] = vx[c] - vxz[c];
    Gt[3 + c] = vx[c] + vxz[c];
    Gb[6 + c] = vy[c] - vyz[c];
    Gt[6 + c] = vy[c] + vyz[c];
    Gb[9 + c] = vxy[c] - vxyz[c];
    Gt[9 + c] = vxy[c] + vxyz[c];
  }
}

// u_e^T KE u_e = w^T D w for one element (E = 1 core).
__device__ __forceinline__ double element_energy(const double (&Flo)[12],
                                                 const double (&Fhi)[12], const Walsh& W) {
  double wx[3], wy[3], wz[3], wxy[3], wxz[3], wyz[3], wxyz[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    wx[c] = Flo[3 + c] + Fhi[3 + c];
    wy[c] = Flo[6 + c] + Fhi[6 + c];
    wz[c] = Fhi[0 + c] - Flo[0 + c];
    wxy[c] = Flo[9 + c] + Fhi[9 + c];
    wxz[c] = Fhi[3 + c] - Flo[3 + c];
    wyz[c] = Fhi[6 + c] - Flo[6 + c];
    wxyz[c] = Fhi[9 + c] - Flo[9 + c];
  }
  const double t = wx[0] + wy[1] + wz[2];
  double e = W.amb * (wx[0] * wx[0] + wy[1] * wy[1] + wz[2] * wz[2]) + W.b * t * t;
  const double sxy = wx[1] + wy[0], sxz = wx[2] + wz[0], syz = wy[2] + wz[1];
  e += W.g * (sxy * sxy + sxz * sxz + syz * syz);
  const double s = wxy[2] + wxz[1] + wyz[0];
  e += W.c3 * (s * s + wxy[2] * wxy[2] + wxz[1] * wxz[1] + wyz[0] * wyz[0]);
  e += W.c1 * (wxy[0] * wxy[0] + wxy[1] * wxy[1] + wxz[0] * wxz[0] + wxz[2] * wxz[2] +
               wyz[1] * wyz[1] + wyz[2] * wyz[2]);
  e += 2.0 * W.c2 * (wxy[0] * wyz[2] + wxy[1] * wxz[2] + wxz[0] * wyz[1]);
  e += W.c4 * (wxyz[0] * wxyz[0] + wxyz[1] * wxyz[1] + wxyz[2] * wxyz[2]);
  return e;
}

// Corner a of element (i,j,k): order (0,0,0),(1,0,0),(1,1,0),(0,1,0),(0,0,1),(1,0,1),
// (1,1,1),(0,1,1). Shared by k_sens and k_edofs.
__device__ __forceinline__ void corner_offset(int a, int& ax, int& ay, int& az) {
  ax = ((a + 1) >> 1) & 1;  // 0,1,1,0
  ay = (a >> 1) & 1;        // 0,0,1,1
  az = a >> 2;
}

// ------------------------------------------------------------------ operator / K_A
// box starts (aligned down) of one block's tiles; offsets are the smem shifts
struct TileOrigin {
  int xv, xm, xe;  // aligned starts: vector / Jacobi (doubles), mask (bytes), element
  int ov, om, oe;  // offsets of node i0-1 (element i0-1) inside the boxes
};

__device__ __forceinline__ TileOrigin tile_origin(int i0) {
  TileOrigin o;
  const int sn = i0 - 1;
  o.xv = sn & ~1; o.ov = sn - o.xv;
  o.xm = sn & ~15; o.om = sn - o.xm;
  o.xe = sn & ~1; o.oe = sn - o.xe;
  return o;
}

template <int MODE>
__device__ __forceinline__ void issue_plane(const OpArgs& a, double* stg, uint64_t* bar,
                                            const TileOrigin& o, int i0, int j0, int kq) {
  using L = Lay<MODE>;
  mbar_expect_tx(bar, L::bytes);
  // vector boxes: sub-rows 3 (j0-1) .. 3 (j0+BY) - 1 (row -3..-1 = node row -1: OOB, zeros)
  tma_load_3d(stg + R_OFF, &a.tm_in, o.xv, 3 * (j0 - 1), kq, bar);
  if (MODE == OP_PCG) {
    tma_load_3d(stg + QO_OFF, &a.tm_qold, o.xv, 3 * (j0 - 1), kq, bar);
    tma_load_3d(stg + PO_OFF, &a.tm_pold, o.xv, 3 * (j0 - 1), kq, bar);
    tma_load_3d(stg + UO_OFF, &a.tm_uown, o.xv, 3 * j0, kq, bar);
    tma_load_3d(stg + DI_OFF, &a.tm_dinv, o.xv, j0 - 1, kq, bar);
  }
  tma_load_3d(stg + L::mk, &a.tm_mask, o.xm, j0 - 1, kq, bar);
  tma_load_3d(stg + L::ee, &a.tm_E, o.xe, j0 - 1, kq - 1, bar);  // element plane kq-1
}

// per-thread state carried from one node plane to the next
struct Carry {
  double F[12];        // Walsh face of the node plane (the next element's lower face)
  double G[12];        // top face of the last element (when carried in registers)
  double pv[3], pz[3]; // output node: p and z (PCG) / masked and raw u (APPLY)
  double pdi;          // output node: D^-1 (PCG)
  unsigned pm;         // output node: fixed bits
};

#ifdef TOMO_EXP_TIMELINE  // timing experiment only: per-block globaltimer stamps of PCG launches
__device__ unsigned long long g_tl[2][4096][7];  // [launch parity][block]: entry, loop end, exit, smid
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int MODE>
__global__ void __launch_bounds__(NT, MODE == OP_PCG ? OP_MINB : OP_MINB_APPLY)
    k_op(const __grid_constant__ OpArgs a) {
#ifdef TOMO_EXP_TIMELINE
  const unsigned long long tl0 = gtimer();
#endif
  using L = Lay<MODE>;
  constexpr int NS = L::ns, STAGE = L::stage;
  extern __shared__ __align__(128) double smem[];
  double* stages = smem;                     // [NS][STAGE]
  double* CD = stages + NS * STAGE;          // [2][3][NT] bottom-face contributions (by parity)
  double* GS = CD + 6 * NT;                  // [GSN][NT] thread-private: top face of the last element
  double* red = GS + GSN * NT;               // [168]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 168);  // [NS] full (TMA bytes landed)
  uint64_t* ebars = bars + NS;                              // [NS] empty (every warp has read the stage)
  int* s_flag = reinterpret_cast<int*>(ebars + NS);
  constexpr bool kEarly = MODE == OP_PCG && TOMO_EARLY_REFILL;

  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * TX + tx;
  const Grid& g = a.g;

  double beta = 0.0, alpha_prev = 0.0;
  // K_hat u launched programmatically after another K_hat u (tomo_bench_apply): its blocks may
  // be resident before the previous grid completes; nothing is read before it has (no-op
  // for ordinary launches)
  if (MODE == OP_APPLY) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (MODE == OP_PCG && (!a.sep || TOMO_SEP_EARLY)) {
    // programmatic dependent launch: this grid may have been scheduled while the previous
    // PCG launch was finishing; everything below reads its results (no-op without PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (*(volatile int*)&a.s->done) return;
    beta = *(volatile double*)&a.s->beta;
    alpha_prev = *(volatile double*)&a.s->alpha;
  }

  // 32-bit offsets into the padded vectors (ndof_pad < 2^31 is checked at create)
  const int rowd = 3 * g.nnx_pad;
  const int planed = rowd * g.nny;
  // persistent, balanced schedule: block b owns work units [ub, ue) of the list
  // (tile, node plane), tile-major; it processes them as z-segments split at tile edges
  const int tiles_x = (g.nnx + OX - 1) / OX;
  int ub, ue;
  if (a.zchunks > 0) {
    // synchronised schedule: block = (tile, z-chunk), equal chunks, so every block marches
    // the same planes at the same time and neighbouring tiles share their halos through L2
    const int tile = blockIdx.x % a.ntiles, ch = blockIdx.x / a.ntiles;
    // chunk c = node planes [z_c, z_{c+1}), z_c = 1 + c (nnz - 1) / chunks: the first chunk
    // gets one plane more because it skips the warm-up step on plane -1 (below), so every
    // chunk costs the same number of steps (cfg3: 30 and 30 instead of 30 and 31)
    auto zc = [&](int c) { return c == 0 ? 0 : min(g.nnz, 1 + (c * (g.nnz - 1)) / a.zchunks); };
    ub = tile * g.nnz + zc(ch);
    ue = tile * g.nnz + zc(ch + 1);
  } else {
    const long long units = (long long)a.ntiles * g.nnz;
    ub = (int)((units * blockIdx.x) / gridDim.x);
    ue = (int)((units * (blockIdx.x + 1)) / gridDim.x);
  }

  if (t == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&bars[s], 1); mbar_init(&ebars[s], BY); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  constexpr bool kGsTmem = MODE == OP_PCG && TOMO_GS_TMEM;
  unsigned* s_tmem = reinterpret_cast<unsigned*>(s_flag + 1);
  if (kGsTmem && ty == 0) {  // warp 0 allocates 64 TMEM columns (48 used: 2 warps per lane quarter x 24)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (kGsTmem) asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (kGsTmem) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tm_base = kGsTmem ? *s_tmem : 0u;
  const unsigned tm_gs = tm_base + ((unsigned)((ty & 3) * 32) << 16) + (unsigned)(ty >> 2) * 24u;
  auto tmem_free = [&]() {
    if (kGsTmem) {
      __syncthreads();
      if (ty == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tm_base) : "memory");
    }
  };
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // p.q, r.z, r.r, z.q, q.D^-1.q

  int git = 0;  // global step counter (mbarrier phase)
  for (int u0 = ub; u0 < ue;) {
  const int tile = u0 / g.nnz;
  const int kbeg = u0 - tile * g.nnz;
  const int kend = min(g.nnz, kbeg + (ue - u0));
  u0 += kend - kbeg;
  const int i0 = (tile % tiles_x) * OX, j0 = (tile / tiles_x) * OY;
  const int nit = kend - kbeg + 2;
  // step it stages node plane kbeg - 1 + it; plane -1 is all zeros (TMA out-of-bounds fill),
  // and so is the state it would hand on, so a segment starting at plane 0 begins at step 1
  const int it0 = kbeg == 0 ? 1 : 0;
  const TileOrigin org = tile_origin(i0);
  if (t == 0) {
    for (int s = 0; s < NS && it0 + s < nit; ++s)
      issue_plane<MODE>(a, stages + ((git + s) % NS) * STAGE, &bars[(git + s) % NS], org, i0, j0,
                        kbeg - 1 + it0 + s);
  }
  if (MODE == OP_PCG && a.sep && !TOMO_SEP_EARLY && u0 - (kend - kbeg) == ub) {
    // separate reduction (OpArgs::sep): this grid was scheduled after the previous PCG
    // launch completed (the reduction kernel between them triggers it only then), so the
    // loads above already read final data while that kernel sums the partials; its alpha,
    // beta and stop flag are read once it has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (*(volatile int*)&a.s->done) {
      if (t == 0)  // no bulk copy may be in flight at exit
        for (int s = 0; s < NS && it0 + s < nit; ++s)
          mbar_wait(&bars[(git + s) % NS], (unsigned)((git + s) / NS) & 1u);
      tmem_free();
      return;
    }
    beta = *(volatile double*)&a.s->beta;
    alpha_prev = *(volatile double*)&a.s->alpha;
  }

  // output node (i0-1+tx, j0+ty) = top node of this warp's element row
  const int gi = i0 - 1 + tx, gj = j0 + ty;
  const bool own_row = ty < OY && gj <= g.ny;
  const bool mine = own_row && tx >= 1 && tx <= OX && gi <= g.nx;
  const int g_own = gi + rowd * gj;                      // node (gi, gj), component 0, plane 0
  // smem offsets: component-0 sub-row of node rows ty (b) and ty+1 (o) in the vector box,
  // lane tx at node i0-1+tx; component c adds c * VB_W
  const int fvb = 3 * ty * VB_W + org.ov + tx;
  const int fvo = fvb + 3 * VB_W;
  const int fuo = 3 * ty * VB_W + org.ov + tx;           // node row ty+1 in the owned-u box
  const int fdb = ty * DB_W + org.ov + tx, fdo = fdb + DB_W;
  const int fmb = ty * MB_W + org.om + tx, fmo = fmb + MB_W;
  // element (tx, ty); lane 31's element lies outside the tile and its result is never read:
  // it reads lane 30's modulus instead of one past the box (the checked build found this)
  const int fe = ty * E_W + org.oe + min(tx, TX - 2);
  // every stage index this thread will read lies inside its piece of the stage
  TCHECK(fvb >= 0 && fvo + 2 * VB_W < VB_W * VB_R && (ty >= OY || fuo + 2 * VB_W < VB_W * UB_R));
  TCHECK(fdo < DB_W * NR && fmo < MB_W * NR && fe < E_W * ER && org.om + TX <= MB_W);

  // state carried from one node plane to the next; K_hat u uses the two copies ping-pong (the
  // loop unrolled by two) so that nothing is copied between registers at the end of a step
  constexpr bool kGsReg = MODE == OP_APPLY ? OP_GSREG_APPLY != 0 : OP_GSREG_PCG != 0;
  Carry c0, c1;
#pragma unroll
  for (int i = 0; i < 12; ++i) c0.F[i] = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) { c0.pv[c] = 0.0; c0.pz[c] = 0.0; }
  c0.pdi = 0.0;
  c0.pm = 0;

  // one node plane kn = kbeg - 1 + it: P = state of plane kn - 1, N = state of plane kn
  auto step = [&](const int it, const Carry& P, Carry& N) {
    const int s = git % NS;
    double* stg = stages + s * STAGE;
    double* CDn = CD + (it & 1) * 3 * NT;
    const int kn = kbeg - 1 + it;
    mbar_wait(&bars[s], (unsigned)(git / NS) & 1u);
    ++git;
    // ---- stage node rows b = ty and o = ty+1: p = D^-1 r + beta p_old with
    //      r = r_old - alpha q_old (PCG), or masked u (APPLY). PCG needs no masking here:
    //      r_{-1}, q_{-1}, p_{-1} and u are zero at fixed DOFs (tomo_create rejects loads on
    //      fixed DOFs, u0 is packed with the mask) and every launch writes r, p, q = 0 there
    //      (q is masked at the output), so the staged values are already zero.
    const unsigned char* MKb = reinterpret_cast<const unsigned char*>(stg + L::mk);
    N.pm = MKb[fmo];
    double vb[3], vo[3];
    if (MODE == OP_PCG) {
      const double dib = stg[DI_OFF + fdb];
      N.pdi = stg[DI_OFF + fdo];
      double pold_o[3], ro[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int cb = fvb + c * VB_W, co = fvo + c * VB_W;
        const double rb = fma(-alpha_prev, stg[QO_OFF + cb], stg[R_OFF + cb]);
        vb[c] = fma(beta, stg[PO_OFF + cb], dib * rb);
        ro[c] = fma(-alpha_prev, stg[QO_OFF + co], stg[R_OFF + co]);
        N.pz[c] = N.pdi * ro[c];
        pold_o[c] = stg[PO_OFF + co];
        vo[c] = fma(beta, pold_o[c], N.pz[c]);
      }
      // owned updates of node row o (r_k, p_k, u_k): one component of 30 consecutive nodes
      // per store instruction (row-SoA layout)
      if (mine && kn >= kbeg && kn < kend) {
        const int go = g_own + planed * kn;
        TCHECK(go >= 0 && go + 2 * g.nnx_pad < g.ndof_pad && gi < g.nnx_pad);
        double rz = 0.0, rr = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#ifndef TOMO_EXP_NO_COMMIT_STORE  // timing experiment only
          a.rnew[go + c * g.nnx_pad] = ro[c];
          a.pnew[go + c * g.nnx_pad] = vo[c];
          a.u[go + c * g.nnx_pad] = fma(alpha_prev, pold_o[c], stg[UO_OFF + fuo + c * VB_W]);
#endif
          rz = fma(N.pz[c], ro[c], rz);
          rr = fma(ro[c], ro[c], rr);
        }
        acc[1] += rz;
        acc[2] += rr;
      }
    } else {
      const unsigned mb = MKb[fmb];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        vb[c] = ((mb >> c) & 1u) ? 0.0 : stg[R_OFF + fvb + c * VB_W];
#if TOMO_APPLY_RAWLDG
        // (raw u of a fixed DOF is re-read from global memory at the output instead of carried)
        vo[c] = ((N.pm >> c) & 1u) ? 0.0 : stg[R_OFF + fvo + c * VB_W];
#else
        N.pz[c] = stg[R_OFF + fvo + c * VB_W];  // raw u (identity rows at fixed DOFs)
        vo[c] = ((N.pm >> c) & 1u) ? 0.0 : N.pz[c];
#endif
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) N.pv[c] = vo[c];
    const double Ecur = stg[L::ee + fe];  // lane 31: a column outside the tile (unused)
    if (kEarly) {
      // the stage's last read is above: release it (one arrival per warp) so that its refill
      // can be issued in the middle of this step instead of after the plane barrier
      __syncwarp();
      if (tx == 0) mbar_arrive(&ebars[s]);
    }

    // ---- element row ty between node rows b and o (lane 31's results are never read;
    // skipping out-of-domain rows of edge tiles measured slower: 79.8 vs 78.4 us)
    // this plane's face (= the next element's lower face): the y butterfly of the lane's own
    // node column first, then the x butterfly with the next lane's (6 DADD per component
    // instead of the 8 of face_from, same shuffle count)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double sg = vb[c] + vo[c], dl = vo[c] - vb[c];
      const double sgn = __shfl_down_sync(0xffffffffu, sg, 1);
      const double dln = __shfl_down_sync(0xffffffffu, dl, 1);
      N.F[0 + c] = sg + sgn;
      N.F[3 + c] = sgn - sg;
      N.F[6 + c] = dl + dln;
      N.F[9 + c] = dln - dl;
    }
    if (kEarly && t == 0 && it + NS < nit) {
      mbar_wait(&ebars[s], (unsigned)((git - 1) / NS) & 1u);  // all BY warps have read stage s
      issue_plane<MODE>(a, stg, &bars[s], org, i0, j0, kn + NS);
    }
    double cup[3] = {0.0, 0.0, 0.0};
    if (it >= 1) {
      double Gb[12], Gt[12];
#ifdef TOMO_EXP_NO_CORE  // timing experiment only: bypass the element core
#pragma unroll
      for (int i = 0; i < 12; ++i) { Gb[i] = P.F[i] * Ecur; Gt[i] = N.F[i] * Ecur; }
#else
      element_core(P.F, N.F, Ecur, a.w, Gb, Gt);
#endif
      if (it >= 2) {
        if (kGsTmem) tmem_wait_st();  // the previous step's top face is in tensor memory
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          // previous element's top face + this element's bottom face, in face modes
          double g00, g10, g01, g11;
          if (kGsTmem) {
            unsigned r[8];
            tmem_ld8(tm_gs + 8u * c, r);
            tmem_wait_ld();
            g00 = __hiloint2double((int)r[1], (int)r[0]);
            g10 = __hiloint2double((int)r[3], (int)r[2]);
            g01 = __hiloint2double((int)r[5], (int)r[4]);
            g11 = __hiloint2double((int)r[7], (int)r[6]);
          } else {
            g00 = kGsReg ? P.G[0 + c] : GS[(0 + c) * NT + t];
            g10 = kGsReg ? P.G[3 + c] : GS[(3 + c) * NT + t];
            g01 = kGsReg ? P.G[6 + c] : GS[(6 + c) * NT + t];
            g11 = kGsReg ? P.G[9 + c] : GS[(9 + c) * NT + t];
          }
          const double m00 = g00 + Gb[0 + c];
          const double m10 = g10 + Gb[3 + c];
          const double m01 = g01 + Gb[6 + c];
          const double m11 = g11 + Gb[9 + c];
          // inverse transform: the x butterfly first (corner x = 1 of element tx-1 comes from
          // the lane below), then the y butterfly of the node column (8 DADD per component)
          const double L0 = m00 - m10, L1 = m01 - m11, R0 = m00 + m10, R1 = m01 + m11;
          const double c0 = L0 + __shfl_up_sync(0xffffffffu, R0, 1);
          const double c1 = L1 + __shfl_up_sync(0xffffffffu, R1, 1);
          cup[c] = c0 + c1;            // -> node row o (mine)
          CDn[c * NT + t] = c0 - c1;   // -> node row b
        }
      }
      if (kGsTmem) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          unsigned r[8];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            r[2 * m] = (unsigned)__double2loint(Gt[3 * m + c]);
            r[2 * m + 1] = (unsigned)__double2hiint(Gt[3 * m + c]);
          }
          tmem_st8(tm_gs + 8u * c, r);
        }
      } else {
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        if (kGsReg) N.G[i] = Gt[i];
        else GS[i * NT + t] = Gt[i];
      }
      }
    }
    __syncthreads();  // CD of this plane complete; stage s consumed by every warp
    // (issuing from warp BY-1, which has no owned row, measured the same: 71.8 vs 71.4 us)
    if (!kEarly && t == 0 && it + NS < nit) issue_plane<MODE>(a, stg, &bars[s], org, i0, j0, kn + NS);
    // (a segment's last NS steps issue nothing, so the next segment starts with free stages)

    if (it >= 2 && mine) {
      const int gb = g_own + planed * (kn - 1);  // output node plane kn - 1
      TCHECK(gb >= 0 && gb + 2 * g.nnx_pad < g.ndof_pad);
      double pq = 0.0, zq = 0.0, qdq = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double qv = cup[c] + CDn[c * NT + t + TX];  // + bottom face of element row ty+1
        const bool fixed = (P.pm >> c) & 1u;
        if (MODE == OP_PCG) {
          qv = fixed ? 0.0 : qv;
#ifndef TOMO_EXP_NO_Q_STORE  // timing experiment only
          a.out[gb + c * g.nnx_pad] = qv;
#endif
          pq = fma(P.pv[c], qv, pq);
          zq = fma(P.pz[c], qv, zq);
          qdq = fma(P.pdi * qv, qv, qdq);
        } else {
#if TOMO_APPLY_RAWLDG
          a.out[gb + c * g.nnx_pad] = fixed ? __ldg(a.u + gb + c * g.nnx_pad) : qv;
#else
          a.out[gb + c * g.nnx_pad] = fixed ? P.pz[c] : qv;
#endif
        }
      }
      acc[0] += pq;
      acc[3] += zq;
      acc[4] += qdq;
    }
  };

  if (MODE == OP_APPLY || OP_PINGPONG_PCG) {
    int it = it0;
    for (; it + 1 < nit; it += 2) {
      step(it, c0, c1);
      step(it + 1, c1, c0);
    }
    if (it < nit) step(it, c0, c1);
  } else {
    // (ping-pong measured slower for the fused PCG kernel: 76.9 vs 71.7 us at cfg3)
    for (int it = it0; it < nit; ++it) {
      step(it, c0, c1);
      c0 = c1;
    }
  }
  __syncthreads();  // segment done: CD / GS / stages may be reused by the next segment
  }
  // the next PCG launch may be scheduled now (it waits for this grid's completion before it
  // reads anything): its blocks take the slots of blocks that have finished their planes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tmem_free();
#ifdef TOMO_EXP_TIMELINE
  const unsigned long long tl1 = gtimer();
  const int tl_par = MODE == OP_PCG ? (*(volatile int*)&a.s->k) & 1 : 0;
#endif

  if (MODE == OP_PCG && a.sep) {
    // the grid totals, the stop test and alpha, beta are k_pcg_red's (the next kernel)
    block_sum5(acc, red);
    if (t < 5) a.partials[5 * blockIdx.x + t] = acc[t];
  } else if (MODE == OP_PCG) {
    const unsigned nb = gridDim.x;
    const unsigned b = blockIdx.x;
    block_sum5(acc, red);
    if (t < 5) a.partials[5 * b + t] = acc[t];
    if (arrive_last(&a.s->cntA, nb, s_flag)) {
      double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (unsigned i = t; i < nb; i += NT) {
#pragma unroll
        for (int q = 0; q < 5; ++q) tot[q] += __ldcg(a.partials + 5 * (size_t)i + q);
      }
      block_sum5(tot, red);
      if (t == 0) {
        Scal* s = a.s;
        const int k = s->k;
        const double pq = tot[0], rz = tot[1], rr = tot[2], zq = tot[3], qdq = tot[4];
        s->pq = pq;
        s->rz = rz;
        s->rr = rr;
        if (k < s->hist_n) s->hist[k] = rr;
#ifdef TOMO_EXP_NOSTOP  // timing experiments: run exactly max_iters launches whatever the values
        if (k >= s->max_iters) { s->done = 2; s->iters = k; } else { s->alpha = 0.5; s->beta = 0.5; s->k = k + 1; }
        if (false) {
#else
        if (!isfinite(pq) || !isfinite(rz) || !isfinite(rr) || !isfinite(zq) || !isfinite(qdq)) {
#endif
          s->status = -6;  // TOMO_ENAN
          s->done = 3;
          s->iters = k;
        } else if (sqrt(rr) <= s->tol_fnorm) {
          s->done = 1;  // r_k converged: u_k (written by this launch) is the solution
          s->iters = k;
        } else if (k >= s->max_iters) {
          s->done = 2;
          s->iters = k;
        } else if (!(pq > 0.0)) {
          s->status = -4;  // TOMO_EBREAKDOWN
          s->done = 3;
          s->iters = k;
        } else {
          // r_{k+1}^T z_{k+1} = r.z - 2 alpha z.q + alpha^2 q.D^-1.q (exact algebra; the
          // next launch recomputes r.z from the explicit r_{k+1}, so nothing accumulates)
          const double alpha = rz / pq;
          const double rz_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, zq, rz));
          s->alpha = alpha;
          s->beta = rz_next / rz;
          s->k = k + 1;
        }
        s->cntA = 0;
        __threadfence();
        if (a.cond && s->done) cudaGraphSetConditional(a.cond, 0u);  // end the graph's loop
      }
    }
  }
#ifdef TOMO_EXP_TIMELINE
  if (MODE == OP_PCG && t == 0 && blockIdx.x < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    auto& G = g_tl[tl_par][blockIdx.x];
    G[0] = tl0; G[1] = tl1; G[2] = gtimer(); G[3] = smid;
  }
#endif
}

// The control of PCG iteration k in its own one-block kernel (OpArgs::sep): after launch k
// of k_op<OP_PCG> has completed, sum its block partials in the fixed order of k_op's last
// block (same thread count, same loop, same block_sum5: the same totals bit for bit), test
// convergence / max_iters / breakdown / NaN and set alpha_k, beta_k - the same decision as
// the last-block path. It lets launch k+1 be scheduled as soon as launch k is complete, so
// launch k+1's first TMA loads overlap this reduction.
__global__ void __launch_bounds__(NT) k_pcg_red(const double* __restrict__ partials, int nb, Scal* s,
                                                unsigned long long cond) {
  __shared__ double red[168];
#if TOMO_SEP_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // launch k+1 may be scheduled
  asm volatile("griddepcontrol.wait;" ::: "memory");               // launch k complete
#else
  asm volatile("griddepcontrol.wait;" ::: "memory");               // launch k complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // launch k+1 may start
#endif
  if (*(volatile int*)&s->done) return;
  const int t = threadIdx.x;
  double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (unsigned i = t; i < (unsigned)nb; i += NT) {
#pragma unroll
    for (int q = 0; q < 5; ++q) tot[q] += __ldcg(partials + 5 * (size_t)i + q);
  }
  block_sum5(tot, red);
  if (t == 0) {
    const int k = s->k;
    const double pq = tot[0], rz = tot[1], rr = tot[2], zq = tot[3], qdq = tot[4];
    s->pq = pq;
    s->rz = rz;
    s->rr = rr;
    if (k < s->hist_n) s->hist[k] = rr;
#ifdef TOMO_EXP_NOSTOP  // timing experiments: run exactly max_iters launches whatever the values
    if (k >= s->max_iters) { s->done = 2; s->iters = k; } else { s->alpha = 0.5; s->beta = 0.5; s->k = k + 1; }
    if (false) {
#else
    if (!isfinite(pq) || !isfinite(rz) || !isfinite(rr) || !isfinite(zq) || !isfinite(qdq)) {
#endif
      s->status = -6;  // TOMO_ENAN
      s->done = 3;
      s->iters = k;
    } else if (sqrt(rr) <= s->tol_fnorm) {
      s->done = 1;  // r_k converged: u_k (written by launch k) is the solution
      s->iters = k;
    } else if (k >= s->max_iters) {
      s->done = 2;
      s->iters = k;
    } else if (!(pq > 0.0)) {
      s->status = -4;  // TOMO_EBREAKDOWN
      s->done = 3;
      s->iters = k;
    } else {
      const double alpha = rz / pq;
      const double rz_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, zq, rz));
      s->alpha = alpha;
      s->beta = rz_next / rz;
      s->k = k + 1;
    }
    __threadfence();
    if (cond && s->done) cudaGraphSetConditional(cond, 0u);  // end the graph's loop
  }
}

// ------------------------------------------------------------------ solve-level reductions and vector kernels
// ||r||^2 over a padded vector (pad entries are 0): the true residual at exit.
__global__ void __launch_bounds__(256) k_norm2(Grid g, const double* __restrict__ r, Scal* s,
                                               double* partials) {
  __shared__ double red[32];
  __shared__ int s_flag;
  double rr = 0.0;
  const int n2 = (int)(g.ndof_pad / 2);
  const int stride = gridDim.x * blockDim.x;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 v = r2[i];
    rr = fma(v.x, v.x, rr);
    rr = fma(v.y, v.y, rr);
  }
  const double b = block_sum(rr, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
  if (arrive_last(&s->cntB, gridDim.x, &s_flag)) {
    const double tot = sum_partials(partials, gridDim.x, 1, 0, red);
    if (threadIdx.x == 0) {
      s->rr_true = tot;
      s->cntB = 0;
      __threadfence();
    }
  }
}

// Exact-beta variant (tomo_set_pcg_exact_beta; the textbook recurrence of SURVEY §8 a4):
// after launch k, r_{k+1}^T z_{k+1} from the explicit r_{k+1} = r_k - alpha_k q_k over all
// nodes, so beta_k = r_{k+1}.z_{k+1} / r_k.z_k replaces the single-pass prediction. One more
// pass over r, q and D^-1 per iteration (the vectors are not written: the next launch forms
// r_{k+1} again). Deterministic two-stage reduction; skipped once the solve has stopped.
__global__ void __launch_bounds__(256) k_beta(Grid g, const double* __restrict__ r,
                                              const double* __restrict__ q,
                                              const double* __restrict__ dinv, Scal* s,
                                              double* partials) {
  __shared__ double red[32];
  __shared__ int s_flag;
  if (*(volatile int*)&s->done) return;
  const double alpha = *(volatile double*)&s->alpha;
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long plane = (long long)g.nnx_pad * g.nny;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn_pad; n += stride) {
    const long long i = n % g.nnx_pad, jk = n / g.nnx_pad;  // padded node, row jk = j + nny k
    const double d = dinv[n];
    const long long base = i + 3 * g.nnx_pad * jk;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double rn = fma(-alpha, q[base + c * g.nnx_pad], r[base + c * g.nnx_pad]);
      acc = fma(d * rn, rn, acc);
    }
  }
  (void)plane;
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
  if (arrive_last(&s->cntB, gridDim.x, &s_flag)) {
    const double tot = sum_partials(partials, gridDim.x, 1, 0, red);
    if (threadIdx.x == 0) {
      s->beta = tot / s->rz;
      s->cntB = 0;
      __threadfence();
    }
  }
}

__global__ void k_scal_init(Scal* s, double tol_fnorm, int max_iters) {
  s->alpha = 0.0; s->beta = 0.0; s->rz = 0.0; s->rr = 0.0; s->pq = 0.0;
  s->rr_true = 0.0; s->tol_fnorm = tol_fnorm; s->energy = 0.0; s->comp = 0.0;
  s->k = 0; s->iters = 0; s->done = 0; s->status = 0; s->max_iters = max_iters;
  s->domain_bad = 0; s->cntA = 0; s->cntB = 0; s->cntR = 0;
  // hist / hist_n are set by the host (tomo_set_history) and kept across solves
}

// r = -q (padded), then r[load dof] += f (loads are distinct DOFs)
__global__ void k_resid(long long n, const double* __restrict__ q, double* __restrict__ r) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n; d += stride)
    r[d] = -q[d];
}
__global__ void k_add_loads(double* r, const int64_t* dofs, const double* vals, int n) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x)
    r[dofs[i]] += vals[i];
}

// dense ABI vector (AoS) -> padded row-SoA internal vector, fixed entries zeroed
__global__ void k_pack(Grid g, const double* __restrict__ dense, double* __restrict__ pad,
                       const uint8_t* __restrict__ mask) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    const int i = (int)(n % g.nnx);
    const int j = (int)((n / g.nnx) % g.nny);
    const int k = (int)(n / ((long long)g.nnx * g.nny));
    const unsigned m = mask ? mask[mask_index(g, i, j, k)] : 0u;  // NULL: no masking
#pragma unroll
    for (int c = 0; c < 3; ++c) pad[dof_pad(g, i, j, k, c)] = ((m >> c) & 1u) ? 0.0 : dense[3 * n + c];
  }
}
__global__ void k_unpack(Grid g, const double* __restrict__ pad, double* __restrict__ dense) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    const int i = (int)(n % g.nnx);
    const int j = (int)((n / g.nnx) % g.nny);
    const int k = (int)(n / ((long long)g.nnx * g.nny));
#pragma unroll
    for (int c = 0; c < 3; ++c) dense[3 * n + c] = pad[dof_pad(g, i, j, k, c)];
  }
}

// ------------------------------------------------------------------ SIMP and Jacobi
// E (padded element rows) from the caller's dense rho; flags rho outside [0,1] or NaN.
__global__ void k_simp(Grid g, const double* __restrict__ rho, double* __restrict__ E,
                       double E0, double Emin, double penal, Scal* s) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.ne; e += stride) {
    const int i = (int)(e % g.nx);
    const int j = (int)((e / g.nx) % g.ny);
    const int k = (int)(e / ((long long)g.nx * g.ny));
    const double r = rho[e];
    bad |= !(r >= -1e-12 && r <= 1.0 + 1e-12);  // SPEC.md l.118 with reading R3 (rounding)
    E[elem_pad(g, i, j, k)] = Emin + pow(r, penal) * (E0 - Emin);
  }
  if (bad) s->domain_bad = 1;
}

// diag(K) at node n = KE_dd * sum of E over the (up to 8) elements around n; all 24
// diagonal entries of the cube KE are equal, so D^-1 is one scalar per node (padded).
__global__ void k_jacobi(Grid g, const double* __restrict__ E, double ke_diag,
                         double* __restrict__ dinv) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    const int i = (int)(n % g.nnx);
    const int j = (int)((n / g.nnx) % g.nny);
    const int k = (int)(n / ((long long)g.nnx * g.nny));
    double sE = 0.0;
    for (int dk = -1; dk <= 0; ++dk)
      for (int dj = -1; dj <= 0; ++dj)
        for (int di = -1; di <= 0; ++di) {
          const int ei = i + di, ej = j + dj, ek = k + dk;
          if (ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny && ek >= 0 && ek < g.nz)
            sE += E[elem_pad(g, ei, ej, ek)];
        }
    dinv[node_pad(g, i, j, k)] = 1.0 / (ke_diag * sE);
  }
}

// ------------------------------------------------------------------ compliance, sensitivity
__global__ void k_compliance(const double* u, const int64_t* dofs, const double* vals, int n,
                             Scal* s) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = fma(vals[i], u[dofs[i]], acc);
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) s->comp = tot;
}

// Sensitivity (Eq. 5) by element columns: a 32 x 8 block, lane tx <-> node column i0+tx of
// node rows j and j+1 (j = j0 + ty), marching along z through a chunk of node planes. Each
// node plane is loaded once per thread (6 values, masked), the x-neighbour's corners come
// by warp shuffle and the lower face is carried from the previous plane, so an element
// costs 6 loads instead of 24 gathers; lane 31 only supplies corners. ce = w^T D w.
// mask == nullptr: u is the workspace's padded row-SoA solution (coalesced, no mask bytes).
constexpr int SENS_X = 31, SENS_BY = 8;
// 4 resident blocks per SM (62 registers, no spills) and z chunks from the resident slots:
// cfg3 28.0 -> 26.3 us, 192x96x96 39.8 -> 29.5, 256x128x128 127.8 -> 69.8 us
// (scripts/explore/sens_ab.sh; TOMO_SENS_MINB=1 / TOMO_SENS_OLDCHUNK=1 restore the old build)
#ifndef TOMO_SENS_PREFETCH
#define TOMO_SENS_PREFETCH 0  // A/B: node-plane loads issued one plane ahead of use
#endif
#ifndef TOMO_SENS_MINB
#define TOMO_SENS_MINB 4
#endif
__global__ void __launch_bounds__(256, TOMO_SENS_MINB) k_sens(Grid g, Walsh W, const double* __restrict__ rho,
                                              const double* __restrict__ u,
                                              const uint8_t* __restrict__ mask, double penal,
                                              double dE, double Emin, double* __restrict__ dc,
                                              double* __restrict__ ce_out, double* partials,
                                              Scal* s, int want_energy, int zchunk) {
  __shared__ double red[32];
  __shared__ int s_flag;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tiles_x = (g.nx + SENS_X - 1) / SENS_X, tiles = tiles_x * ((g.ny + SENS_BY - 1) / SENS_BY);
  const int tile = blockIdx.x % tiles, ch = blockIdx.x / tiles;
  const int i0 = (tile % tiles_x) * SENS_X, j = (tile / tiles_x) * SENS_BY + ty;
  const int k0 = ch * zchunk, k1 = min(g.nz, k0 + zchunk);  // elements k0 .. k1-1
  const int in = i0 + tx;                                    // this lane's node column
  const bool node_ok = in <= g.nx && j < g.ny;
  const bool elem_ok = tx < SENS_X && in < g.nx && j < g.ny;
  const int ipen = (penal == (double)(int)penal && penal >= 1.0 && penal <= 8.0) ? (int)penal : 0;
  double energy = 0.0;
  double Flo[12], Fhi[12];
  // raw corner values of node plane k: this lane's node column, rows j and j+1
  auto load = [&](int k, double (&a0)[3], double (&a1)[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) { a0[c] = 0.0; a1[c] = 0.0; }
    if (node_ok && mask == nullptr) {
      // u in the internal padded row-SoA layout (zero at fixed DOFs): one component of 32
      // consecutive nodes per load instruction, no mask bytes (tomo_evaluate's path)
      const long long b0 = dof_pad(g, in, j, k, 0);
      TCHECK(b0 >= 0 && b0 + 5LL * g.nnx_pad < g.ndof_pad && k <= g.nz);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a0[c] = __ldg(u + b0 + (long long)c * g.nnx_pad);
        a1[c] = __ldg(u + b0 + (long long)(3 + c) * g.nnx_pad);
      }
    } else if (node_ok) {
      const long long n0 = node_dense(g, in, j, k), n1 = node_dense(g, in, j + 1, k);
      TCHECK(n0 >= 0 && n1 < g.nn && k <= g.nz);
      const unsigned m0 = __ldg(mask + mask_index(g, in, j, k));
      const unsigned m1 = __ldg(mask + mask_index(g, in, j + 1, k));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a0[c] = ((m0 >> c) & 1u) ? 0.0 : __ldg(u + 3 * n0 + c);
        a1[c] = ((m1 >> c) & 1u) ? 0.0 : __ldg(u + 3 * n1 + c);
      }
    }
  };
  auto face = [&](const double (&a0)[3], const double (&a1)[3], double (&F)[12]) {  // Walsh face
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double b0 = __shfl_down_sync(0xffffffffu, a0[c], 1);
      const double b1 = __shfl_down_sync(0xffffffffu, a1[c], 1);
      face_from(a0[c], b0, a1[c], b1, F, c);
    }
  };
  double A0[3], A1[3];
  load(k0, A0, A1);
  face(A0, A1, Flo);
#if TOMO_SENS_PREFETCH
  load(k0 + 1, A0, A1);  // k0 + 1 <= nz
#endif
  for (int k = k0; k < k1; ++k) {
#if TOMO_SENS_PREFETCH
    // plane k+1 was loaded one step earlier; the loads of plane k+2 fly during this element
    double B0[3], B1[3];
    if (k + 1 < k1) load(k + 2, B0, B1);
    face(A0, A1, Fhi);
#else
    load(k + 1, A0, A1);
    face(A0, A1, Fhi);
#endif
    if (elem_ok) {
      const long long e = in + (long long)g.nx * (j + (long long)g.ny * k);
      const double ce = element_energy(Flo, Fhi, W);
      const double r = rho[e];
      // r^(p-1): repeated products for integer p (the configs' p = 3; a DP pow costs ~100
      // instructions), pow otherwise
      double rp1;
      if (ipen > 0) {
        rp1 = 1.0;
        for (int q = 1; q < ipen; ++q) rp1 *= r;
      } else {
        rp1 = pow(r, penal - 1.0);
      }
      dc[e] = -penal * rp1 * dE * ce;  // Eq. 5 with dE = E0 - Emin (A5)
      if (ce_out) ce_out[e] = ce;
      if (want_energy) energy = fma(Emin + rp1 * r * dE, ce, energy);
    }
#pragma unroll
    for (int q = 0; q < 12; ++q) Flo[q] = Fhi[q];
#if TOMO_SENS_PREFETCH
    if (k + 1 < k1) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { A0[c] = B0[c]; A1[c] = B1[c]; }
    }
#endif
  }
  if (!want_energy) return;
  const double bs = block_sum(energy, red);
  const int b = blockIdx.x;
  if (threadIdx.x == 0 && threadIdx.y == 0) partials[b] = bs;
  if (arrive_last(&s->cntR, gridDim.x, &s_flag)) {
    const double tot = sum_partials(partials, gridDim.x, 1, 0, red);
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      s->energy = tot;
      s->cntR = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ density filter
// taps: 3 ints (dx, dy, dz) + weight each, order dz, dy, dx ascending (reading A15)
__global__ void k_filter_sums(Grid g, const int* __restrict__ taps,
                              const double* __restrict__ w, int ntaps, double* Hs, double* iHs,
                              int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.ne; e += stride) {
    const int i = (int)(e % g.nx);
    const int j = (int)((e / g.nx) % g.ny);
    const int k = (int)(e / ((long long)g.nx * g.ny));
    double acc = 0.0;
    int cnt = 0;
    for (int t = 0; t < ntaps; ++t) {
      const int ii = i + taps[3 * t], jj = j + taps[3 * t + 1], kk = k + taps[3 * t + 2];
      if (ii >= 0 && ii < g.nx && jj >= 0 && jj < g.ny && kk >= 0 && kk < g.nz) {
        acc += w[t];
        ++cnt;
      }
    }
    Hs[e] = acc;
    iHs[e] = 1.0 / acc;
    counts[e] = cnt;
  }
}

__global__ void __launch_bounds__(256) k_filter(Grid g, const int* __restrict__ taps,
                                                const double* __restrict__ w, int ntaps,
                                                const double* __restrict__ Hs,
                                                const double* __restrict__ in,
                                                double* __restrict__ out, int transpose) {
  extern __shared__ double fsm[];
  double* sw = fsm;
  int* so = reinterpret_cast<int*>(sw + ntaps);
  for (int t = threadIdx.x; t < ntaps; t += blockDim.x) {
    sw[t] = w[t];
    so[3 * t] = taps[3 * t];
    so[3 * t + 1] = taps[3 * t + 1];
    so[3 * t + 2] = taps[3 * t + 2];
  }
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long pe = (long long)g.nx * g.ny;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.ne; e += stride) {
    const int i = (int)(e % g.nx);
    const int j = (int)((e / g.nx) % g.ny);
    const int k = (int)(e / pe);
    double acc = 0.0;
    for (int t = 0; t < ntaps; ++t) {
      const int ii = i + so[3 * t], jj = j + so[3 * t + 1], kk = k + so[3 * t + 2];
      if (ii >= 0 && ii < g.nx && jj >= 0 && jj < g.ny && kk >= 0 && kk < g.nz) {
        const long long e2 = ii + (long long)g.nx * jj + pe * kk;
        const double v = transpose ? __ldg(in + e2) / __ldg(Hs + e2) : __ldg(in + e2);
        acc = fma(sw[t], v, acc);
      }
    }
    out[e] = transpose ? acc : acc / Hs[e];
  }
}

// Tiled density filter for a ball-shaped tap set {d in Z^3 : |d|^2 <= M} (every cone filter
// w = rmin - |d| > 0 is one: sqrt is monotone). A block of FT_X x FT_Y / ROWS threads owns
// FT_X x FT_Y output columns (each thread ROWS adjacent rows for radii R <= 3, one row beyond)
// and marches along z through a chunk of planes. Each input plane (tile + R halo, zero outside the domain; multiplied by
// 1/Hs in transpose mode: P^T v = H (v / Hs)) is staged once in shared memory, double
// buffered with the next plane's global loads issued before the current plane's FMAs, and
// scattered into 2R+1 register accumulators per output row, acc[j] = output plane zi - R + j.
// Weights wd2[|d|^2] live in registers (specialised tap sets) or shared memory (runtime M).
// Per output: about (2R+1)(2R+2)/2 shared loads per input plane and one FMA per tap. Forward
// mode multiplies the finished output by 1/Hs (P x = H x / Hs).
#ifndef TOMO_FT_SHELL
#define TOMO_FT_SHELL 1  // specialised radii: shell sums (A/B knob: 0 = one FMA per tap)
#endif
#ifndef TOMO_FT_ROWS
#define TOMO_FT_ROWS 2  // output rows per thread for radii R <= 3 (A/B knob: 1, 2, 4; 2 adjacent rows measured best)
#endif
#ifndef TOMO_FT_ADJ
// ROWS > 1: a thread's output rows are adjacent (y, y+1: they share 2R of their 2R+1 tap rows, so
// the shared loads per output drop from (2R+1)^2 to (2R+1)(2R+2)/2) instead of FT_Y/ROWS apart
// (no sharing). cfg3, 93 taps: 1 row 23.4 us, 2 rows FT_Y/2 apart 33.5, 2 adjacent rows 21.2,
// 4 adjacent rows 25.3 (64-thread blocks: too few warps) (scripts/explore/filter_ab.sh)
#define TOMO_FT_ADJ 1
#endif
#ifndef TOMO_FT_ZMIN_R
#define TOMO_FT_ZMIN_R 4  // z chunks are at least ZMIN_R * R + 4 planes thick (halo FMA waste)
#endif
#ifndef TOMO_FT_BLOCKS_PER_SM
#define TOMO_FT_BLOCKS_PER_SM 3  // target resident blocks per SM when choosing z chunks
#endif
constexpr int FT_X = 32, FT_Y = 8;  // output tile; ROWS output rows per thread (1, 2 or 4)

// shell bookkeeping of the tiled filter (constant-folded once the tap loops are unrolled):
// is (dx, dy) the first tap of its shell dx^2 + dy^2 in (dy, dx) order; has shell m a tap
__host__ __device__ constexpr bool ft_first_in_shell(int dx, int dy, int R) {
  for (int y = -R; y <= R; ++y)
    for (int x = -R; x <= R; ++x) {
      if (y == dy && x == dx) return true;
      if (x * x + y * y == dx * dx + dy * dy) return false;
    }
  return true;
}
__host__ __device__ constexpr bool ft_shell_nonempty(int m, int R) {
  for (int y = -R; y <= R; ++y)
    for (int x = -R; x <= R; ++x)
      if (x * x + y * y == m) return true;
  return false;
}

// cone weights by |d|^2 as a by-value kernel parameter: constant-bank operands of the FMAs
struct FtW {
  double w[64];
};

template <int R, int MM, int ROWS>
__global__ void __launch_bounds__(FT_X * FT_Y / ROWS) k_filter_t(Grid g, const __grid_constant__ FtW fw,
                                                  const double* __restrict__ wd2, int M,
                                                  const double* __restrict__ iHs,
                                                  const double* __restrict__ in,
                                                  double* __restrict__ out, int transpose,
                                                  int zchunk) {
  constexpr int FT_YT = FT_Y / ROWS, FT_T = FT_X * FT_YT;
  constexpr int RSTEP = TOMO_FT_ADJ ? 1 : FT_YT;  // distance between a thread's output rows
  constexpr int PX = FT_X + 2 * R, PY = FT_Y + 2 * R, NA = 2 * R + 1, DMAX = 3 * R * R;
  constexpr int NL = (PX * PY + FT_T - 1) / FT_T;  // staged values per thread and plane
  __shared__ double pl[2][PY * PX];
  __shared__ double sw[MM >= 0 ? 1 : DMAX + 1];  // runtime-M weights (broadcast reads)
  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * FT_X + tx;
  const int ry = TOMO_FT_ADJ ? ty * ROWS : ty;     // the thread's first output row in the tile
  const int tiles_x = (g.nx + FT_X - 1) / FT_X, tiles = tiles_x * ((g.ny + FT_Y - 1) / FT_Y);
  const int tile = blockIdx.x % tiles, ch = blockIdx.x / tiles;
  const int x0 = (tile % tiles_x) * FT_X, y0 = (tile / tiles_x) * FT_Y;
  const int z0 = ch * zchunk, z1 = min(g.nz, z0 + zchunk);
  const int Mr = MM >= 0 ? MM : M;
  constexpr int WN = MM >= 0 && !(R <= 3 && TOMO_FT_SHELL) ? MM + 1 : 1;
  double w[WN];  // specialised tap sets without shells: weights in registers
#pragma unroll
  for (int d = 0; d < WN; ++d) w[d] = wd2[d];
  if (MM < 0)
    for (int d = t; d <= DMAX; d += FT_T) sw[d] = d <= Mr ? wd2[d] : 0.0;
  double acc[ROWS][NA];
#pragma unroll
  for (int h = 0; h < ROWS; ++h)
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[h][j] = 0.0;
  const long long pe = (long long)g.nx * g.ny;
  // raw loads only (the transpose scaling by 1/Hs happens at staging time), so that the
  // loads stay in flight while the FMAs of the current plane run
  struct Pf { double a[NL], b[NL]; };
  auto fetch = [&](Pf& pf, int zi) {  // this thread's staging slots of plane zi
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int q = t + l * FT_T;
      const int xx = x0 - R + q % PX, yy = y0 - R + q / PX;
      double va = 0.0, vb = 0.0;
      if (q < PX * PY && xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zi < g.nz) {
        const long long e = xx + (long long)g.nx * yy + pe * zi;
        va = __ldg(in + e);
        if (transpose) vb = __ldg(iHs + e);
      }
      pf.a[l] = va;
      pf.b[l] = vb;
    }
  };
  auto stage = [&](int b, const Pf& pf) {
#pragma unroll
    for (int l = 0; l < NL; ++l)
      if (t + l * FT_T < PX * PY) pl[b][t + l * FT_T] = transpose ? pf.a[l] * pf.b[l] : pf.a[l];
  };
  const int zb = max(0, z0 - R), ze = min(g.nz, z1 + R);  // input planes that exist
  const int x = x0 + tx;
  // output plane z is complete once input plane z + R is in (or the domain ends); forward
  // mode scales by 1/Hs of the output (ih, loaded at the start of the step)
  auto flush = [&](int z, const double (&ih)[ROWS]) {
#pragma unroll
    for (int h = 0; h < ROWS; ++h) {
      const int y = y0 + ry + h * RSTEP;
      if (x < g.nx && y < g.ny && z >= z0 && z < z1) {
        const long long e = x + (long long)g.nx * y + pe * z;
        out[e] = transpose ? acc[h][0] : acc[h][0] * ih[h];
      }
#pragma unroll
      for (int j = 0; j + 1 < NA; ++j) acc[h][j] = acc[h][j + 1];
      acc[h][NA - 1] = 0.0;
    }
  };
  auto load_ih = [&](int z, double (&ih)[ROWS]) {
#pragma unroll
    for (int h = 0; h < ROWS; ++h) {
      const int y = y0 + ry + h * RSTEP;
      ih[h] = (!transpose && x < g.nx && y < g.ny && z >= z0 && z < z1)
                  ? __ldg(iHs + x + (long long)g.nx * y + pe * z) : 0.0;
    }
  };
  // input plane zi from smem buffer b; the loads of plane zi + 2 go to F while the FMAs run,
  // plane zi + 1 (fetched one step earlier into S) is staged into the other buffer at the end
  auto step = [&](int zi, int b, Pf& F, const Pf& S) {
    if (zi + 2 < ze) fetch(F, zi + 2);
    double ih[ROWS];
    load_ih(zi - R, ih);
    const double* P = pl[b];
    if constexpr (MM >= 0 && R <= 3 && TOMO_FT_SHELL) {
      // shell sums: the weight depends on |d|^2 = m + dz^2 only, so the taps of one input
      // plane are first summed over each 2-D shell m = dx^2 + dy^2 (one DADD per tap), and
      // every output plane dz takes one FMA per shell (cfg3, rmin 3: 19 DADD + 24 DFMA per
      // element and input plane instead of 93 DFMA: 25.1 -> 23.2 us). The loops unroll
      // completely, so S[] indices are constants. Not for rmin 7.2: its ~30 live shell sums
      // take the kernel to 204 registers and one block per SM (1323 vs 214 us measured).
#pragma unroll
      for (int h = 0; h < ROWS; ++h) {
        double S[MM + 1];
#pragma unroll
        for (int dy = -R; dy <= R; ++dy) {
#pragma unroll
          for (int dx = -R; dx <= R; ++dx) {
            const int m = dx * dx + dy * dy;
            if (m > MM) continue;
            TCHECK((ry + h * RSTEP + R + dy) * PX + tx + R + dx < PX * PY);
            const double v = P[(ry + h * RSTEP + R + dy) * PX + tx + R + dx];
            if (ft_first_in_shell(dx, dy, R)) S[m] = v;
            else S[m] += v;
          }
        }
#pragma unroll
        for (int m = 0; m <= MM; ++m) {
          if (!ft_shell_nonempty(m, R)) continue;
#pragma unroll
          for (int j = 0; j < NA; ++j) {
            const int dz = R - j;
            if (m + dz * dz <= MM) acc[h][j] = fma(fw.w[m + dz * dz], S[m], acc[h][j]);
          }
        }
      }
    } else {
#pragma unroll
    for (int dy = -R; dy <= R + (ROWS - 1) * RSTEP; ++dy) {
#pragma unroll
      for (int dx = -R; dx <= R; ++dx) {
        // column (dx, dy) of row 0 is column (dx, dy - FT_YT) of row 1
        bool rh[ROWS], any = false;
#pragma unroll
        for (int h = 0; h < ROWS; ++h) {
          const int dyh = dy - h * RSTEP;
          rh[h] = dyh >= -R && dyh <= R && dx * dx + dyh * dyh <= (MM >= 0 ? MM : DMAX);
          any |= rh[h];
        }
        if (!any) continue;
        TCHECK((ry + R + dy) * PX + tx + R + dx < PX * PY);
        const double v = P[(ry + R + dy) * PX + tx + R + dx];
#pragma unroll
        for (int h = 0; h < ROWS; ++h) {
          if (!rh[h]) continue;
          const int dyh = dy - h * RSTEP;
#pragma unroll
          for (int j = 0; j < NA; ++j) {
            const int dz = R - j, d2 = dx * dx + dyh * dyh + dz * dz;
            if (d2 <= (MM >= 0 ? MM : DMAX)) {
              if (MM >= 0) acc[h][j] = fma(w[MM >= 0 ? d2 : 0], v, acc[h][j]);
              else if (d2 <= Mr) acc[h][j] = fma(sw[d2], v, acc[h][j]);
            }
          }
        }
      }
    }
    }
    flush(zi - R, ih);
    if (zi + 1 == ze)  // drain: outputs whose remaining input planes lie outside the domain
      for (int z = zi - R + 1; z < z1; ++z) {
        load_ih(z, ih);
        flush(z, ih);
      }
    if (zi + 1 < ze) {
      stage(b ^ 1, S);
      __syncthreads();
    }
  };
  Pf pa, pb;
  fetch(pa, zb);
  fetch(pb, zb + 1);
  stage(0, pa);
  __syncthreads();
  for (int zi = zb; zi < ze; zi += 2) {
    step(zi, 0, pa, pb);
    if (zi + 1 < ze) step(zi + 1, 1, pb, pa);
  }
}

// ------------------------------------------------------------------ OC (cooperative)
__device__ __forceinline__ double oc_xnew(double x, double gg, double dv, double lam,
                                          double move, double eta) {
  const double B = fmax(0.0, -gg) / (dv * lam);
  const double sc = (eta == 0.5) ? sqrt(B) : pow(B, eta);
  const double lo = fmax(0.0, x - move), hi = fmin(1.0, x + move);
  return fmin(fmax(x * sc, lo), hi);
}

__global__ void __launch_bounds__(256) k_oc(int ne, const double* __restrict__ x,
                                            const double* __restrict__ gv,
                                            const double* __restrict__ dv,
                                            double* __restrict__ xnew, double target,
                                            double move, double eta, double* partials,
                                            double* out2) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  const int G = gridDim.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double l1 = 1e-30, l2 = 1e30;
  const double lo0 = l1, hi0 = l2;
  int steps = 0;
  // SPEC.md l.322 "NaN in gradients -> error": flag non-finite x, g, dv (out2[2], zeroed by
  // the host before the launch; every writer stores the same value)
  bool bad = false;
  for (long long e = g0; e < ne; e += stride)
    bad |= !isfinite(x[e]) || !isfinite(gv[e]) || !isfinite(dv[e]);
  if (bad) *(volatile double*)(out2 + 2) = 1.0;
  while (l2 > l1 * (1.0 + 1e-15) && steps < 200) {
    const double lm = sqrt(l1 * l2);
    double v = 0.0;
    for (long long e = g0; e < ne; e += stride)
      v = fma(dv[e], oc_xnew(x[e], gv[e], dv[e], lm, move, eta), v);
    const double bs = block_sum(v, red);
    double* part = partials + (steps & 1) * G;
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    grid.sync();
    const double tot = sum_partials(part, G, 1, 0, red);
    if (tot > target) l1 = lm;
    else l2 = lm;
    ++steps;
  }
  for (long long e = g0; e < ne; e += stride) xnew[e] = oc_xnew(x[e], gv[e], dv[e], l2, move, eta);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const bool unreachable = (l2 == hi0) || (l1 == lo0);
    out2[0] = l2;
    out2[1] = unreachable ? -(double)steps : (double)steps;
  }
}

// ------------------------------------------------------------------ two-scale coarse path
// z_C[b] = mean of z over the nb^3 fine elements of block b (fixed summation order k, j, i)
__global__ void k_coarsen(Grid g, int nb, const double* __restrict__ z, double* __restrict__ zc) {
  const int cx = g.nx / nb, cy = g.ny / nb;
  const long long nc = (long long)cx * cy * (g.nz / nb);
  const double inv = 1.0 / ((double)nb * nb * nb);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nc; b += stride) {
    const int I = (int)(b % cx), J = (int)((b / cx) % cy), K = (int)(b / ((long long)cx * cy));
    double s = 0.0;
    for (int k = K * nb; k < K * nb + nb; ++k)
      for (int j = J * nb; j < J * nb + nb; ++j)
        for (int i = I * nb; i < I * nb + nb; ++i)
          s += z[i + (long long)g.nx * (j + (long long)g.ny * k)];
    zc[b] = s * inv;
  }
}

// ------------------------------------------------------------------ introspection, bench
__global__ void k_edofs(Grid g, long long* map) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.ne; e += stride) {
    const int i = (int)(e % g.nx);
    const int j = (int)((e / g.nx) % g.ny);
    const int k = (int)(e / ((long long)g.nx * g.ny));
    for (int a = 0; a < 8; ++a) {
      int ax, ay, az;
      corner_offset(a, ax, ay, az);
      const long long n = node_dense(g, i + ax, j + ay, k + az);
      for (int c = 0; c < 3; ++c) map[24 * e + 3 * a + c] = 3 * n + c;
    }
  }
}

__global__ void k_mask_dofs(Grid g, const uint8_t* mask, uint8_t* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    const int i = (int)(n % g.nnx);
    const int j = (int)((n / g.nnx) % g.nny);
    const int k = (int)(n / ((long long)g.nnx * g.nny));
    const unsigned m = mask[mask_index(g, i, j, k)];
    for (int c = 0; c < 3; ++c) out[3 * n + c] = (m >> c) & 1u;
  }
}

__global__ void k_dinv_dense(Grid g, const double* dinv_pad, double* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.nn; n += stride) {
    const int i = (int)(n % g.nnx);
    const int j = (int)((n / g.nnx) % g.nny);
    const int k = (int)(n / ((long long)g.nnx * g.nny));
    out[n] = dinv_pad[node_pad(g, i, j, k)];
  }
}

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // never true; defeats dead-code elimination
}

inline unsigned nblk(long long n, int bs, int cap) {
  long long b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

}  // namespace

// ================================================================== launch helpers
int op_tiles(const Grid& g) {
  return ((g.nnx + OX - 1) / OX) * ((g.nny + OY - 1) / OY);
}

size_t op_smem(int mode) {
  const size_t ns = mode == OP_PCG ? NS : NS_A, st = mode == OP_PCG ? STAGE : STAGE_A;
  return sizeof(double) * (ns * st + (6 + GSN) * NT + 168) + sizeof(uint64_t) * 2 * ns + 16;
}

// The dynamic shared memory opt-in is a per-device function attribute: set it once per
// device (several contexts may live on several GPUs of one process).
static std::mutex g_attr_mu;
static void op_attr() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaFuncSetAttribute(k_op<OP_PCG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)op_smem(1));
  cudaFuncSetAttribute(k_op<OP_APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)op_smem(0));
  done[dev] = true;
}

cudaError_t launch_op(int mode, const OpArgs& a, int nblocks, cudaStream_t st, bool pdl) {
  op_attr();
  if (pdl) {
    // programmatic dependent launch after the previous launch of the same kernel on this stream
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(TX, BY);
    cfg.dynamicSmemBytes = op_smem(mode);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return mode == OP_PCG ? cudaLaunchKernelEx(&cfg, k_op<OP_PCG>, a) : cudaLaunchKernelEx(&cfg, k_op<OP_APPLY>, a);
  }
  if (mode == OP_PCG) k_op<OP_PCG><<<nblocks, dim3(TX, BY), op_smem(1), st>>>(a);
  else k_op<OP_APPLY><<<nblocks, dim3(TX, BY), op_smem(0), st>>>(a);
  return cudaGetLastError();
}

cudaError_t add_pcg_node(cudaGraph_t g, cudaGraphNode_t* node, const cudaGraphNode_t* deps,
                         size_t ndeps, const OpArgs& a, int nblocks) {
  op_attr();
  cudaKernelNodeParams kp = {};
  void* args[] = {const_cast<OpArgs*>(&a)};
  kp.func = reinterpret_cast<void*>(k_op<OP_PCG>);
  kp.gridDim = dim3(nblocks);
  kp.blockDim = dim3(TX, BY);
  kp.sharedMemBytes = (unsigned)op_smem(1);
  kp.kernelParams = args;
  return cudaGraphAddKernelNode(node, g, deps, ndeps, &kp);
}

cudaError_t launch_pcg_red(const OpArgs& a, int nblocks, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(NT);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_pcg_red, (const double*)a.partials, nblocks, a.s, 0ull);
}

cudaError_t add_pcg_red_node(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphNode_t prev,
                             const OpArgs& a, int nblocks) {
  cudaKernelNodeParams kp = {};
  const double* part = a.partials;
  Scal* sc = a.s;
  unsigned long long cond = a.cond;
  void* args[] = {(void*)&part, &nblocks, &sc, &cond};
  kp.func = reinterpret_cast<void*>(k_pcg_red);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(NT);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  cudaError_t e = cudaGraphAddKernelNode(node, g, nullptr, 0, &kp);
  if (e != cudaSuccess || !prev) return e;
  cudaGraphEdgeData ed = {};
  ed.from_port = cudaGraphKernelNodePortProgrammatic;
  ed.type = cudaGraphDependencyTypeProgrammatic;
  return cudaGraphAddDependencies_v2(g, &prev, node, &ed, 1);
}

cudaError_t add_pcg_node_pdl(cudaGraph_t g, cudaGraphNode_t* node, cudaGraphNode_t prev,
                             const OpArgs& a, int nblocks) {
  cudaError_t e = add_pcg_node(g, node, nullptr, 0, a, nblocks);
  if (e != cudaSuccess || !prev) return e;
  // programmatic edge: the node may launch once every block of `prev` has triggered
  // (griddepcontrol.launch_dependents after its planes); it waits for prev's completion
  // (griddepcontrol.wait) before reading anything
  cudaGraphEdgeData ed = {};
  ed.from_port = cudaGraphKernelNodePortProgrammatic;
  ed.type = cudaGraphDependencyTypeProgrammatic;
  return cudaGraphAddDependencies_v2(g, &prev, node, &ed, 1);
}

int op_occupancy(int mode) {
  op_attr();
  int nb = 0;
  if (mode == OP_PCG)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_op<OP_PCG>, NT, op_smem(1));
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_op<OP_APPLY>, NT, op_smem(0));
  return nb;
}

cudaError_t launch_simp(const Grid& g, const double* rho, double* E, double E0, double Emin,
                        double penal, Scal* s, cudaStream_t st) {
  k_simp<<<nblk(g.ne, 256, 148 * 16), 256, 0, st>>>(g, rho, E, E0, Emin, penal, s);
  return cudaGetLastError();
}
cudaError_t launch_jacobi(const Grid& g, const double* E, double ke_diag, double* dinv,
                          cudaStream_t st) {
  k_jacobi<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, E, ke_diag, dinv);
  return cudaGetLastError();
}
cudaError_t launch_pack(const Grid& g, const double* dense, double* pad, const uint8_t* mask,
                        cudaStream_t st) {
  k_pack<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, dense, pad, mask);
  return cudaGetLastError();
}
cudaError_t launch_unpack(const Grid& g, const double* pad, double* dense, cudaStream_t st) {
  k_unpack<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, pad, dense);
  return cudaGetLastError();
}
cudaError_t launch_scal_init(Scal* s, double tol_fnorm, int max_iters, cudaStream_t st) {
  k_scal_init<<<1, 1, 0, st>>>(s, tol_fnorm, max_iters);
  return cudaGetLastError();
}
cudaError_t launch_resid(const Grid& g, const double* q, double* r, const int64_t* ldofs,
                         const double* lvals, int nloads, cudaStream_t st) {
  k_resid<<<nblk(g.ndof_pad, 256, 148 * 16), 256, 0, st>>>(g.ndof_pad, q, r);
  if (nloads > 0) k_add_loads<<<nblk(nloads, 256, 64), 256, 0, st>>>(r, ldofs, lvals, nloads);
  return cudaGetLastError();
}
cudaError_t launch_beta(const Grid& g, const double* r, const double* q, const double* dinv,
                        Scal* s, double* partials, int nblocks, cudaStream_t st) {
  k_beta<<<nblocks, 256, 0, st>>>(g, r, q, dinv, s, partials);
  return cudaGetLastError();
}
cudaError_t add_beta_node(cudaGraph_t gr, cudaGraphNode_t* node, const cudaGraphNode_t* deps,
                          size_t ndeps, const Grid& g, const double* r, const double* q,
                          const double* dinv, Scal* s, double* partials, int nblocks) {
  cudaKernelNodeParams kp = {};
  Grid gg = g;
  void* args[] = {&gg, (void*)&r, (void*)&q, (void*)&dinv, &s, &partials};
  kp.func = reinterpret_cast<void*>(k_beta);
  kp.gridDim = dim3(nblocks);
  kp.blockDim = dim3(256);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  return cudaGraphAddKernelNode(node, gr, deps, ndeps, &kp);
}
cudaError_t launch_norm2(const Grid& g, const double* r, Scal* s, double* partials,
                         int nblocks, cudaStream_t st) {
  k_norm2<<<nblocks, 256, 0, st>>>(g, r, s, partials);
  return cudaGetLastError();
}
cudaError_t launch_compliance(const double* u, const int64_t* ldofs, const double* lvals,
                              int nloads, Scal* s, cudaStream_t st) {
  k_compliance<<<1, 256, 0, st>>>(u, ldofs, lvals, nloads, s);
  return cudaGetLastError();
}
cudaError_t launch_sens(const Grid& g, const Walsh& w, const double* rho, const double* u,
                        const uint8_t* mask, double penal, double dE, double Emin,
                        double* dc, double* ce, double* partials, int max_blocks, Scal* s,
                        int want_energy, cudaStream_t st) {
  const int tiles = ((g.nx + SENS_X - 1) / SENS_X) * ((g.ny + SENS_BY - 1) / SENS_BY);
  // z-chunk length from the resident slots: minimise waves x (planes per chunk + 1)
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sens, 32 * SENS_BY, 0);
  const long long slots = (long long)std::max(1, occ) * sms;
  int zchunk = g.nz, chunks = 1;
  long long best = -1;
#if TOMO_SENS_OLDCHUNK
  chunks = std::max(1, std::min(g.nz, (4 * 148 + tiles - 1) / tiles));
  chunks = std::max(1, std::min(chunks, max_blocks / std::max(1, tiles)));
  zchunk = (g.nz + chunks - 1) / chunks;
  chunks = (g.nz + zchunk - 1) / zchunk;
  const bool search = false;
#else
  const bool search = true;
#endif
  for (int c = 1; search && c <= g.nz; ++c) {
    const int zc = (g.nz + c - 1) / c, cc = (g.nz + zc - 1) / zc;
    const long long nb = (long long)tiles * cc;
    if (want_energy && nb > max_blocks) break;
    const long long cost = ((nb + slots - 1) / slots) * (zc + 1);
    if (best < 0 || cost < best) { best = cost; zchunk = zc; chunks = cc; }
  }
  if (want_energy && tiles * chunks > max_blocks) return cudaErrorInvalidValue;  // partials
  k_sens<<<tiles * chunks, dim3(32, SENS_BY), 0, st>>>(g, w, rho, u, mask, penal, dE, Emin, dc, ce,
                                                       partials, s, want_energy, zchunk);
  return cudaGetLastError();
}
cudaError_t launch_filter_sums(const Grid& g, const int* taps, const double* w, int ntaps,
                               double* Hs, double* iHs, int* counts, cudaStream_t st) {
  k_filter_sums<<<nblk(g.ne, 256, 148 * 16), 256, 0, st>>>(g, taps, w, ntaps, Hs, iHs, counts);
  return cudaGetLastError();
}
cudaError_t launch_filter(const Grid& g, const int* taps, const double* w, int ntaps,
                          const double* Hs, const double* in, double* out, int transpose,
                          cudaStream_t st) {
  const size_t sm = (size_t)ntaps * (sizeof(double) + 3 * sizeof(int));
  if (sm > 48 * 1024) {  // per device (as op_attr); cheap enough to set on every such launch
    std::lock_guard<std::mutex> lk(g_attr_mu);
    cudaFuncSetAttribute(k_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  }
  k_filter<<<nblk(g.ne, 256, 148 * 16), 256, sm, st>>>(g, taps, w, ntaps, Hs, in, out,
                                                       transpose);
  return cudaGetLastError();
}
// tiled filter launch for a ball of radius^2 M (R = floor(sqrt(M))): specialised tap sets of
// the configs (rmin 1.5, 2, 3 and the paper's 7.2) and a runtime-M kernel per R up to 8;
// returns cudaErrorNotSupported when R > 8 (the caller falls back to k_filter)
cudaError_t launch_filter_tiled(const Grid& g, int R, int M, const double* wd2, const double* hw,
                                const double* iHs, const double* in, double* out, int transpose,
                                int sms, cudaStream_t st) {
  const int tiles = ((g.nx + FT_X - 1) / FT_X) * ((g.ny + FT_Y - 1) / FT_Y);
  // z chunks: aim at >= 3 blocks per SM, but no chunk thinner than 4R + 4 planes (the 2R
  // halo planes of a chunk cost FMAs)
  int chunks = std::max(1, (TOMO_FT_BLOCKS_PER_SM * sms + tiles - 1) / tiles);
  chunks = std::min(chunks, std::max(1, g.nz / (TOMO_FT_ZMIN_R * R + 4)));
  const int zchunk = (g.nz + chunks - 1) / chunks;
  chunks = (g.nz + zchunk - 1) / zchunk;
  const dim3 grid(tiles * chunks);
  // two output rows per thread halve the shared loads per FMA where loads would bound (small
  // R); one row per thread for large R (FMA-bound, and the unrolled body stays in registers)
  FtW fw{};
  for (int d = 0; d <= M && d < 64; ++d) fw.w[d] = hw[d];
#define TOMO_FT(RR, MMM)                                                                  \
  k_filter_t<RR, MMM, (RR <= 3 ? TOMO_FT_ROWS : 1)>                                         \
      <<<grid, dim3(FT_X, FT_Y / (RR <= 3 ? TOMO_FT_ROWS : 1)), 0, st>>>(g, fw, wd2, M, iHs, in, out, \
                                                                     transpose, zchunk)
  if (R == 1 && M == 2) TOMO_FT(1, 2);
  else if (R == 1 && M == 3) TOMO_FT(1, 3);
  else if (R == 2 && M == 8) TOMO_FT(2, 8);
  else if (R == 7 && M == 51) TOMO_FT(7, 51);
  else if (R == 0) TOMO_FT(0, 0);
  else if (R == 1) TOMO_FT(1, -1);
  else if (R == 2) TOMO_FT(2, -1);
  else if (R == 3) TOMO_FT(3, -1);
  else if (R == 4) TOMO_FT(4, -1);
  else if (R == 5) TOMO_FT(5, -1);
  else if (R == 6) TOMO_FT(6, -1);
  else if (R == 7) TOMO_FT(7, -1);
  else if (R == 8) TOMO_FT(8, -1);
  else return cudaErrorNotSupported;
#undef TOMO_FT
  return cudaGetLastError();
}

int oc_max_blocks() {
  int nb = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_oc, 256, 0);
  if (nb > 4) nb = 4;
  return nb * sms;
}
cudaError_t launch_oc(int ne, const double* x, const double* g, const double* dv,
                      double* xnew, double target, double move, double eta,
                      double* partials, double* out2, int grid_blocks, cudaStream_t st) {
  void* args[] = {(void*)&ne,    (void*)&x,      (void*)&g,        (void*)&dv,
                  (void*)&xnew,  (void*)&target, (void*)&move,     (void*)&eta,
                  (void*)&partials, (void*)&out2};
  return cudaLaunchCooperativeKernel((void*)k_oc, dim3(grid_blocks), dim3(256), args, 0, st);
}
cudaError_t launch_edofs(const Grid& g, long long* map, cudaStream_t st) {
  k_edofs<<<nblk(g.ne, 256, 148 * 16), 256, 0, st>>>(g, map);
  return cudaGetLastError();
}
cudaError_t launch_mask_dofs(const Grid& g, const uint8_t* mask, uint8_t* out,
                             cudaStream_t st) {
  k_mask_dofs<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, mask, out);
  return cudaGetLastError();
}
cudaError_t launch_dinv_dense(const Grid& g, const double* dinv_pad, double* out,
                              cudaStream_t st) {
  k_dinv_dense<<<nblk(g.nn, 256, 148 * 16), 256, 0, st>>>(g, dinv_pad, out);
  return cudaGetLastError();
}
cudaError_t launch_coarsen(const Grid& g, int nb, const double* z, double* zc, cudaStream_t st) {
  const long long nc = (long long)(g.nx / nb) * (g.ny / nb) * (g.nz / nb);
  k_coarsen<<<nblk(nc, 256, 148 * 16), 256, 0, st>>>(g, nb, z, zc);
  return cudaGetLastError();
}
__global__ void k_set_tol(Scal* s, double tol) { s->tol_fnorm = tol * sqrt(s->rr_true); }
cudaError_t launch_set_tol(Scal* s, double tol, cudaStream_t st) {
  k_set_tol<<<1, 1, 0, st>>>(s, tol);
  return cudaGetLastError();
}
cudaError_t launch_dfma(double* out, int blocks, int iters, cudaStream_t st) {
  k_dfma<<<blocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace tomo

#ifdef TOMO_EXP_TIMELINE  // timing experiment only: copy the per-block stamps of the last two PCG launches
extern "C" int tomo_exp_timeline(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, tomo::g_tl, sizeof(tomo::g_tl));
}
#endif
