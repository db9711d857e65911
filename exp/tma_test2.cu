// bisecting TMA box shapes (development aid)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int n, int rank, int c0, int fence) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (fence) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(&bar)), "r"(n * 8) : "memory");
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                   ::"r"(sa(sm)), "l"((uint64_t)&tm), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                   ::"r"(sa(sm)), "l"((uint64_t)&tm), "r"(c0), "r"(c0 ? 3 : 0), "r"(0), "r"(c0 ? 1 : 0), "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar)) : "memory");
  for (int q = threadIdx.x; q < n; q += blockDim.x) out[q] = sm[q];
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int cfg = atoi(argv[1]);
  std::vector<double> h(1 << 20);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  int rank, n;
  CUresult r;
  const cuuint32_t es[4] = {1, 1, 1, 1};
  if (cfg == 0) {  // 2D 64 x 64, box 16 x 8
    rank = 2; const cuuint64_t dims[2] = {64, 64}; const cuuint64_t str[1] = {64 * 8}; const cuuint32_t box[2] = {16, 8};
    n = 128;
    r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    rank = 4;
    const cuuint64_t dims[4] = {32, 8, 170, 6};
    const cuuint64_t str[3] = {32 * 8, 32 * 8 * 8, 32 * 8 * 170 * 8};
    cuuint32_t box[4] = {16, 1, 8, 1};
    if (cfg == 2) box[2] = 170;
    if (cfg == 3) box[0] = 18;
    if (cfg == 4) { box[0] = 18; box[2] = 170; }
    n = box[0] * box[1] * box[2] * box[3];
    r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, (argc > 2 && atoi(argv[2])) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("cfg %d encode %d n %d\n", cfg, (int)r, n);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<1, 128, 100000>>>(tm, o, n, rank, argc > 3 ? atoi(argv[3]) : 0, argc > 4 ? atoi(argv[4]) : 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("cfg %d: %s\n", cfg, cudaGetErrorString(e));
  std::vector<double> ho(n);
  cudaMemcpy(ho.data(), o, n * 8, cudaMemcpyDeviceToHost);
  printf("first %g %g %g\n", ho[0], ho[1], ho[n - 1]);
  return 0;
}
