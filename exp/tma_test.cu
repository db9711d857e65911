// standalone check of a 4-D FP64 TMA box load into shared memory with an mbarrier (development aid)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
               ::"r"(d), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b) : "memory");
}

template <int BX, int BY, int BF, int BZ>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0, int z0, int mode) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BX * BY * BF * BZ);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (mode >= 1) mbar_expect_tx(bar, sizeof(double) * BX * BY * BF * BZ);
    if (mode >= 2) tma_load_4d(sm, &tm, bar, x0, y0, 0, z0);
  }
  __syncthreads();
  if (mode >= 1) mbar_wait(bar, 0);
  for (int q = threadIdx.x; q < BX * BY * BF * BZ; q += blockDim.x) out[q] = sm[q];
}

int main(int argc, char** argv) {
  const int nx = 32, ny = 8, nf = 170, nz = 6;
  std::vector<double> h((size_t)nx * ny * nf * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  constexpr int BX = 18, BY = 1, BF = 170, BZ = 1;
  cudaMalloc(&o, sizeof(double) * BX * BY * BF * BZ);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[4] = {nx, ny, nf, nz};
  const cuuint64_t str[3] = {nx * 8, (cuuint64_t)nx * ny * 8, (cuuint64_t)nx * ny * nf * 8};
  const cuuint32_t box[4] = {BX, BY, BF, BZ};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const int dtv = argc > 1 ? atoi(argv[1]) : 0;
  const CUtensorMapDataType dty = dtv == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : (dtv == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_INT64);
  CUresult r = encode(&tm, dty, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  size_t smem = sizeof(double) * BX * BY * BF * BZ + 16;
  cudaFuncSetAttribute(k<BX, BY, BF, BZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  setvbuf(stdout, nullptr, _IONBF, 0);
  for (int mode = 0; mode <= 2; mode += 2) {
    k<BX, BY, BF, BZ><<<1, 128, smem>>>(tm, o, 3, 2, 1, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  std::vector<double> ho(BX * BY * BF * BZ);
  cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int f = 0; f < BF; ++f)
    for (int x = 0; x < BX; ++x) {
      double want = (x + 3 < nx) ? h[(((size_t)1 * nf + f) * ny + 2) * nx + x + 3] : 0.0;
      if (ho[f * BX + x] != want) ++bad;
    }
  printf("mismatches %d\n", bad);
  return 0;
}
