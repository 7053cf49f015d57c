// Probe: parameterised 2-D/3-D tiled TMA load. argv: rank d0 d1 d2 b0 b1 x y z dyn
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct A { CUtensorMap tm; double* out; int x, y, z, rank, n; };
template <int DYN>
__global__ void k(const __grid_constant__ A a) {
  __shared__ __align__(128) double ssm[DYN ? 1 : 4096];
  extern __shared__ __align__(128) double dsm[];
  double* sm = DYN ? dsm : ssm;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(s32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(&bar)), "r"(a.n * 8) : "memory");
    if (a.rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" :: "r"(s32(sm)), "l"((unsigned long long)&a.tm), "r"(a.x), "r"(a.y), "r"(s32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" :: "r"(s32(sm)), "l"((unsigned long long)&a.tm), "r"(a.x), "r"(a.y), "r"(a.z), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" :: "r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) a.out[i] = sm[i];
}
int main(int argc, char** argv) {
  int rank = atoi(argv[1]); unsigned long long d0 = atoll(argv[2]), d1 = atoll(argv[3]), d2 = atoll(argv[4]);
  unsigned b0 = atoi(argv[5]), b1 = atoi(argv[6]); int x = atoi(argv[7]), y = atoi(argv[8]), z = atoi(argv[9]), dyn = atoi(argv[10]);
  size_t p1 = ((d0 * 8 + 15) / 16) * 16, p2 = p1 * d1;
  double *g, *o; cudaMalloc(&g, p2 * d2 + 4096); cudaMalloc(&o, 1 << 16);
  std::vector<double> h((p2 * d2) / 8); for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  cudaMemcpy(g, h.data(), p2 * d2, cudaMemcpyHostToDevice);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  A a{}; a.out = o; a.x = x; a.y = y; a.z = z; a.rank = rank; a.n = b0 * b1;
  cuuint64_t dims[3] = {d0, d1, d2}, str[2] = {p1, p2}; cuuint32_t box[3] = {b0, b1, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, g, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (dyn) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); k<1><<<1, 128, 64 * 1024>>>(a); }
  else k<0><<<1, 128>>>(a);
  cudaError_t e = cudaDeviceSynchronize();
  double rr[3] = {-1, -1, -1}; if (e == cudaSuccess) cudaMemcpy(rr, o, 24, cudaMemcpyDeviceToHost);
  printf("rank %d dims %llu %llu %llu box %u %u at %d %d %d dyn %d: enc %d %s  %g %g %g\n", rank, d0, d1, d2, b0, b1, x, y, z, dyn, (int)r, cudaGetErrorString(e), rr[0], rr[1], rr[2]);
  return 0;
}
