// Probe: plain (non-tensor) bulk async copy global->shared, and 1-D/2-D tensor maps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct A2 { CUtensorMap tm; double* out; };
__global__ void bulk(const double* src, double* out, int n) {
  __shared__ __align__(128) double sm[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(s32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(&bar)), "r"(n * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(s32(sm)), "l"(src), "r"(n * 8), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" :: "r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}
__global__ void tma2(const __grid_constant__ A2 a, int n) {
  __shared__ __align__(128) double sm[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(s32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(&bar)), "r"(n * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" :: "r"(s32(sm)), "l"((unsigned long long)&a.tm), "r"(0), "r"(0), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" :: "r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) a.out[i] = sm[i];
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  double *g, *o; cudaMalloc(&g, 1 << 20); cudaMalloc(&o, 1 << 16);
  std::vector<double> h(1 << 17); for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  cudaMemcpy(g, h.data(), 1 << 20, cudaMemcpyHostToDevice);
  if (mode == 0) { bulk<<<1, 128>>>(g, o, 512); }
  else {
    void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    A2 a{}; a.out = o;
    cuuint64_t dims[2] = {256, 64}, str[1] = {2048}; cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
    CUresult r = enc(&a.tm, mode == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    tma2<<<1, 128>>>(a, mode == 1 ? 256 : 128);
  }
  cudaError_t e = cudaDeviceSynchronize();
  double r[4] = {0}; if (e == cudaSuccess) cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
  printf("mode %d: %s  %g %g %g\n", mode, cudaGetErrorString(e), r[0], r[1], r[2]);
  return e != cudaSuccess;
}
