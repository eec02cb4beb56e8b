// Probe 2: isolate the failing piece of the TMA path.
// mode 0: mbarrier arrive/try_wait only (no async copy)
// mode 1: cp.async.bulk (non-tensor, 1-D) global->shared + mbarrier
// mode 2: TMA with the tensor map in GLOBAL memory (runtime entry point encode)
// mode 3: TMA with __grid_constant__ map encoded by libcuda's cuTensorMapEncodeTiled (-lcuda)
// mode 4: TMA with __grid_constant__ map (runtime entry point encode) -- the failing baseline
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait0(uint64_t* bar) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sa(bar)), "r"(0)
        : "memory");
}
__device__ __forceinline__ void init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__global__ void k_mbar(double* out) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
  wait0(&bar);
  if (threadIdx.x == 0) out[0] = 42.0;
}
__global__ void k_bulk(const double* src, double* out, int n) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm)),
                 "l"(src), "r"(n * 8), "r"(sa(&bar))
                 : "memory");
  }
  wait0(&bar);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}
__device__ __forceinline__ void tma3(double* dst, const void* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          sa(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(sa(bar))
      : "memory");
}
__global__ void k_tma_global(const CUtensorMap* tm, double* out, int bytes) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    tma3(sm, tm, 0, 0, 2, &bar);
  }
  wait0(&bar);
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = sm[i];
}
__global__ void k_tma_param(const __grid_constant__ CUtensorMap tm, double* out, int bytes) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    tma3(sm, &tm, 0, 0, 2, &bar);
  }
  wait0(&bar);
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = sm[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  const int nx = 64, ny = 64, nz = 10, bw = 32;
  std::vector<double> h((size_t)nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 64 * 64 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap m;
  memset(&m, 0, sizeof(m));
  cuuint64_t dims[3] = {nx, ny, nz};
  cuuint64_t str[2] = {nx * 8, (cuuint64_t)nx * ny * 8};
  cuuint32_t box[3] = {bw, bw, 1}, es[3] = {1, 1, 1};
  CUresult rc = CUDA_SUCCESS;
  if (mode == 3) {
    rc = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (mode >= 2) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    rc = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int bytes = bw * bw * 8;
  cudaFuncSetAttribute((const void*)k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (mode == 0) k_mbar<<<1, 128>>>(o);
  if (mode == 1) k_bulk<<<1, 128, bytes>>>(d + 2 * nx * ny, o, bw * bw);
  if (mode == 2) {
    CUtensorMap* gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    k_tma_global<<<1, 128, bytes>>>(gm, o, bytes);
  }
  if (mode >= 3) k_tma_param<<<1, 128, bytes>>>(m, o, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = -1;
  if (e == cudaSuccess && mode >= 1) {
    std::vector<double> r(bw * bw);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int yy = 0; yy < bw; ++yy)
      for (int xx = 0; xx < bw; ++xx) {
        double want = mode == 1 ? h[(size_t)2 * nx * ny + yy * bw + xx] : h[(size_t)2 * nx * ny + yy * nx + xx];
        if (r[yy * bw + xx] != want) ++bad;
      }
  }
  int drv = 0;
  cudaDriverGetVersion(&drv);
  printf("mode=%d encode=%d driver=%d -> %s mismatches=%d\n", mode, (int)rc, drv, cudaGetErrorString(e), bad);
  return 0;
}
