// Which 3D fp64 TMA boxes / start coordinates does sm_100a accept?  One load per process.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu
//   ./tma_probe bx by cx cy
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void k(const __grid_constant__ CUtensorMap m, int cx, int cy, unsigned bytes, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            (unsigned)__cvta_generic_to_shared(sm)),
        "l"((unsigned long long)&m), "r"(cx), "r"(cy), "r"(0), "r"(b)
        : "memory");
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(b));
    out[0] = sm[0];
  }
}

int main(int argc, char** argv) {
  int bx = atoi(argv[1]), by = atoi(argv[2]), cx = atoi(argv[3]), cy = atoi(argv[4]);
  int nx = 64, ny = 64, nz = 4;
  double* g;
  cudaMalloc(&g, sizeof(double) * nx * ny * nz);
  double* out;
  cudaMalloc(&out, 8);
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t str[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  size_t smem = (size_t)bx * by * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<1, 32, smem>>>(m, cx, cy, (unsigned)smem, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("box %3d x %3d  start (%3d,%3d)  bytes %6zu (%%128=%3zu)  encode=%d  run=%s\n", bx, by, cx, cy, smem, smem % 128,
         (int)r, cudaGetErrorString(e));
  return 0;
}
