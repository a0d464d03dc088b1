// dmma_mix_probe.cu -- resolves the DMMA throughput question left by fp64_probe (0.44 DMMA/cycle/SM
// at 32 warps) vs dmma_rate_probe (0.25): W warps per SM, of which the first WM run DMMA chains
// (CH accumulators, A operand distinct per chain when DIST, else shared) and the rest DFMA chains
// (8 per thread).  Each warp records its own cycles; the block's span is max(t1) - min(t0).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_mix_probe tools/dmma_mix_probe.cu
#include <cstdio>
#include <vector>

constexpr int ITERS = 2048;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CH, bool DIST>
__global__ void probe(int wm, double* out, long long* span, double s) {
  __shared__ long long t0s, t1s;
  if (threadIdx.x == 0) { t0s = 0x7fffffffffffffffLL; t1s = 0; }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double a[CH], d[2 * CH], f[8];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = DIST ? 1e-3 * threadIdx.x + c + 1 : 1e-3 * threadIdx.x + 1;
#pragma unroll
  for (int c = 0; c < 2 * CH; ++c) d[c] = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = 1e-3 * threadIdx.x + k;
  const long long t0 = clock64();
  if (warp < wm) {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int c = 0; c < CH; ++c) dmma(d[2 * c], d[2 * c + 1], a[c], s);
    }
  } else {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = fma(f[k], s, 1e-12);
    }
  }
  const long long t1 = clock64();
  atomicMin(&t0s, t0);
  atomicMax(&t1s, t1);
  __syncthreads();
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 2 * CH; ++c) acc += d[c];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) span[blockIdx.x] = t1s - t0s;
}

template <int CH, bool DIST>
void run(int sms, int warps, int wm) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * warps * 32);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  probe<CH, DIST><<<sms, warps * 32>>>(wm, out, cyc, 0.999999);
  probe<CH, DIST><<<sms, warps * 32>>>(wm, out, cyc, 0.999999);
  cudaDeviceSynchronize();
  std::vector<long long> h(sms);
  cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (long long c : h) mean += (double)c;
  mean /= sms;
  const double dm = (double)wm * ITERS * CH, df = (double)(warps - wm) * ITERS * 8;
  printf("warps %2d (DMMA %2d, CH %d, %s A): DMMA %.3f/cyc  DFMA %.3f/cyc  -> %6.1f FMA/cycle/SM (%.0f cycles)\n",
         warps, wm, CH, DIST ? "distinct" : "shared", dm / mean, df / mean, (256 * dm + 32 * df) / mean, mean);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16, 32}) {
    run<4, true>(sms, w, w);
    run<4, false>(sms, w, w);
    run<1, true>(sms, w, w);
  }
  for (int w : {8, 16, 32}) {
    run<4, true>(sms, w, w / 2);
    run<4, true>(sms, w, w / 4);
    run<2, true>(sms, w, w / 2);
  }
  run<4, true>(sms, 16, 0);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
