// Standalone probe of the TMA path used by k_op (debug aid; not part of libtomo).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>

struct Args { CUtensorMap tm; int x, y, z; double* out; };

__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ CUtensorMap gtm_storage;
template <int V>
__global__ void probe(const __grid_constant__ Args a, int n, const CUtensorMap* gtm) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(s32(&bar)));
    if (V == 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const CUtensorMap* tmp = (V == 4) ? gtm : &a.tm;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(&bar)), "r"(n * 8) : "memory");
    if (V == 3)
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   :: "r"(s32(sm)), "l"((unsigned long long)tmp), "r"(a.x), "r"(a.y), "r"(a.z), "r"(s32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   :: "r"(s32(sm)), "l"((unsigned long long)tmp), "r"(a.x), "r"(a.y), "r"(a.z), "r"(s32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" :: "r"(s32(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) a.out[i] = sm[i];
}

int main(int argc, char** argv) {
  int ci = atoi(argv[1]), var = atoi(argv[2]); int dt = argc > 3 ? atoi(argv[3]) : 0; int prom = argc > 4 ? atoi(argv[4]) : 1;
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  printf("entry point %p q=%d\n", fnp, (int)q);
  struct Case { const char* name; unsigned long long d0, d1, d2; unsigned b0, b1; int x, y, z; int v; };
  Case cases[] = {
    {"inside, box<=dim", 300, 20, 10, 96, 9, 3, 2, 1, 1},
    {"inside, fence.proxy", 300, 20, 10, 96, 9, 3, 2, 1, 2},
    {"negative coords", 300, 20, 10, 96, 9, -3, -1, -1, 1},
    {"box > dim0", 75, 13, 13, 96, 9, -3, -1, 0, 1},
    {"fully OOB z", 300, 20, 10, 96, 9, 0, 0, 12, 1},
  };
  { auto& c = cases[ci]; c.v = var;
    size_t pitch1 = ((c.d0 * 8 + 15) / 16) * 16, pitch2 = pitch1 * c.d1;
    double* g; cudaMalloc(&g, pitch2 * c.d2);
    std::vector<double> h(pitch2 * c.d2 / 8);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    cudaMemcpy(g, h.data(), pitch2 * c.d2, cudaMemcpyHostToDevice);
    Args a{}; a.x = c.x; a.y = c.y; a.z = c.z;
    cuuint64_t dims[3] = {c.d0, c.d1, c.d2}, str[2] = {pitch1, pitch2};
    cuuint32_t box[3] = {c.b0, c.b1, 1}, es[3] = {1, 1, 1};
    CUtensorMapDataType dts[4] = {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_DATA_TYPE_UINT8};
    int esz[4] = {8, 8, 4, 1};
    dims[0] = c.d0 * 8 / esz[dt]; box[0] = c.b0 * 8 / esz[dt];
    if (box[0] > 256) { box[0] = 256; }
    CUresult r = enc(&a.tm, dts[dt], 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("dt=%d prom=%d box0=%u\n", dt, prom, box[0]);
    int n = box[0] * esz[dt] / 8 * c.b1;
    cudaMalloc(&a.out, n * 8);
    cudaError_t e;
    CUtensorMap* dtm; cudaMalloc(&dtm, sizeof(CUtensorMap)); cudaMemcpy(dtm, &a.tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    switch (c.v) {
      case 1: cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); probe<1><<<1, 128, 64 * 1024>>>(a, n, dtm); break;
      case 2: cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); probe<2><<<1, 128, 64 * 1024>>>(a, n, dtm); break;
      case 3: cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); probe<3><<<1, 128, 64 * 1024>>>(a, n, dtm); break;
      default: cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); probe<4><<<1, 128, 64 * 1024>>>(a, n, dtm); break;
    }
    e = cudaDeviceSynchronize();
    std::vector<double> o(n);
    if (e == cudaSuccess) cudaMemcpy(o.data(), a.out, n * 8, cudaMemcpyDeviceToHost);
    printf("v%d %-22s encode=%d kernel=%s  out[0]=%g out[1]=%g out[%d]=%g\n", c.v, c.name, (int)r, cudaGetErrorString(e), o[0], o[1], c.b0, o[c.b0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
