// dmma_rate_probe.cu -- DMMA.8x8x4 latency and throughput vs. warps per SM and independent
// accumulator chains per warp, plus the cost of feeding it from shared memory (one LDS.64 A
// fragment per DMMA, or one per two) and of running DFMA chains beside it.  Results in SM
// cycles (clock64), one CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_rate_probe tools/dmma_rate_probe.cu
#include <cstdio>
#include <vector>

constexpr int ITERS = 1024;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// CH independent chains; LD: 0 = register operands, 1 = one LDS per DMMA, 2 = one LDS per 2 DMMA;
// DF: DFMA instructions per DMMA issued by the same warp (independent chains)
template <int CH, int LD, int DF>
__global__ void probe(double* out, long long* cyc, double s) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double d[2 * CH];
#pragma unroll
  for (int k = 0; k < 2 * CH; ++k) d[k] = 0.0;
  double f[4] = {threadIdx.x * 1e-3, 1.0, 2.0, 3.0};
  const double a0 = threadIdx.x * 1e-3;
  const double* p = sm + (threadIdx.x & 31) + 32 * ((threadIdx.x >> 5) & 7);
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double a = a0;
      if (LD == 1 || (LD == 2 && (c & 1) == 0)) a = p[((it * CH + c) * 256) & 4095];
      dmma(d[2 * c], d[2 * c + 1], a, s);
#pragma unroll
      for (int q = 0; q < DF; ++q) f[q & 3] = fma(f[q & 3], s, 1e-12);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double acc = f[0] + f[1] + f[2] + f[3];
#pragma unroll
  for (int k = 0; k < 2 * CH; ++k) acc += d[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH, int LD, int DF>
void run(int sms, int warps, const char* what) {
  const int threads = warps * 32;
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  probe<CH, LD, DF><<<sms, threads>>>(out, cyc, 0.999999);
  probe<CH, LD, DF><<<sms, threads>>>(out, cyc, 0.999999);
  cudaDeviceSynchronize();
  std::vector<long long> h(sms);
  cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (long long c : h) mean += (double)c;
  mean /= sms;
  const double dmmas = (double)warps * ITERS * CH;
  printf("%-22s warps %2d chains %d: %6.3f DMMA/cycle/SM (%5.1f FMA/cyc), %6.1f cycles per DMMA per warp-chain\n",
         what, warps, CH, dmmas / mean, 256.0 * dmmas / mean + 32.0 * DF * dmmas / mean, mean / (ITERS));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 0, 0>(sms, 1, "latency");
  for (int w : {4, 8, 16, 32}) {
    run<1, 0, 0>(sms, w, "reg operands");
    run<2, 0, 0>(sms, w, "reg operands");
    run<4, 0, 0>(sms, w, "reg operands");
    run<8, 0, 0>(sms, w, "reg operands");
  }
  for (int w : {8, 16}) {
    run<4, 1, 0>(sms, w, "LDS per DMMA");
    run<4, 2, 0>(sms, w, "LDS per 2 DMMA");
    run<4, 0, 2>(sms, w, "+2 DFMA per DMMA");
    run<4, 0, 4>(sms, w, "+4 DFMA per DMMA");
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
