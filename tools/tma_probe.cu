// Minimal probe: one TMA 3-D tile load through a __grid_constant__ tensor map.
// argv: fence(0=mbarrier_init,1=proxy,2=none) tile(0/1) dtype(0=f64,1=u64,2=f32x2) boxw smem_offset
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int FENCE, int TILE>
__global__ void probe(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0, int z0,
                      int bytes, int off) {
  extern __shared__ __align__(1024) unsigned char raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw);
  double* sm = reinterpret_cast<double*>(raw + off);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
    if (FENCE == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (FENCE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes)
                 : "memory");
    if (TILE)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              sa(sm)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(z0), "r"(sa(bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              sa(sm)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(z0), "r"(sa(bar))
          : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(sa(bar)), "r"(0)
        : "memory");
  }
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = sm[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int fence = atoi(argv[1]), tile = atoi(argv[2]), dt = atoi(argv[3]), bw = atoi(argv[4]),
      off = atoi(argv[5]);
  int st = argc > 6 ? atoi(argv[6]) : -3;
  const int nx = 64, ny = 64, nz = 10;
  std::vector<double> h((size_t)nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 64 * 64 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  CUtensorMapDataType t = dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                  : (dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  int mult = dt == 2 ? 2 : 1;
  cuuint64_t dims[3] = {(cuuint64_t)nx * mult, ny, nz};
  cuuint64_t str[2] = {nx * 8, (cuuint64_t)nx * ny * 8};
  cuuint32_t box[3] = {(cuuint32_t)(bw * mult), (cuuint32_t)bw, 1}, es[3] = {1, 1, 1};
  CUresult rc = ((Enc)fn)(&m, t, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = bw * bw * 8;
  auto k = fence == 0 ? (tile ? probe<0, 1> : probe<0, 0>)
                      : fence == 1 ? (tile ? probe<1, 1> : probe<1, 0>) : (tile ? probe<2, 1> : probe<2, 0>);
  cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<1, 128, bytes + off + 64>>>(m, o, st * mult, st, 2, bytes, off);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = -1;
  if (e == cudaSuccess) {
    std::vector<double> r(bw * bw);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int yy = 0; yy < bw; ++yy)
      for (int xx = 0; xx < bw; ++xx) {
        int gx = xx + st, gy = yy + st;
        double want = (gx < 0 || gy < 0) ? 0.0 : h[(size_t)2 * nx * ny + gy * nx + gx];
        if (r[yy * bw + xx] != want) ++bad;
      }
  }
  printf("st=%d fence=%d tile=%d dtype=%d boxw=%d off=%d encode=%d -> %s mismatches=%d\n", st, fence, tile, dt,
         bw, off, (int)rc, cudaGetErrorString(e), bad);
  return 0;
}
