// fp64_probe.cu -- FP64 issue rates on this B200: DFMA (CUDA cores), DMMA m8n8k4 (tensor
// cores), both at once, and DFMA with a shared-memory load per FMA (the blur's x/y-pass shape).
// Each kernel runs a fixed amount of independent work per warp and reads the SM cycle counter,
// so the result is in operations per SM per cycle, independent of the clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <vector>

constexpr int ITERS = 2048;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// mode 0: DFMA only (8 independent chains per thread)
// mode 1: DMMA only (4 independent accumulators per warp)
// mode 2: even warps DFMA, odd warps DMMA
// mode 3: DFMA with an LDS.64 operand per FMA (x-pass shape)
__global__ void probe(int mode, double* out, long long* cyc, double s) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t0 = clock64();
  const bool do_mma = mode == 1 || (mode == 2 && (warp & 1));
  if (do_mma) {
    for (int it = 0; it < ITERS; ++it) {
      dmma(d[0], d[1], a[0], s);
      dmma(d[2], d[3], a[1], s);
      dmma(d[4], d[5], a[2], s);
      dmma(d[6], d[7], a[3], s);
    }
  } else if (mode == 3) {
    const double* p = sm + (threadIdx.x & 1023);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(p[(k * 37 + it) & 2047], s, a[k]);
    }
  } else {
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], s, 1e-12);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += a[k] + d[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"DFMA", "DMMA m8n8k4", "DFMA + DMMA (half the warps each)", "DFMA with LDS operand"};
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 4; ++mode) {
      double* out;
      long long* cyc;
      cudaMalloc(&out, sizeof(double) * sms * threads);
      cudaMalloc(&cyc, sizeof(long long) * sms);
      probe<<<sms, threads>>>(mode, out, cyc, 0.999999);  // warm-up
      probe<<<sms, threads>>>(mode, out, cyc, 0.999999);
      cudaDeviceSynchronize();
      std::vector<long long> h(sms);
      cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (long long c : h) mean += (double)c;
      mean /= sms;
      const int warps = threads / 32;
      double fma_per_sm = 0, instr_per_sm = 0;
      if (mode == 0 || mode == 3) {
        instr_per_sm = (double)warps * ITERS * 8;
        fma_per_sm = instr_per_sm * 32;
      } else if (mode == 1) {
        instr_per_sm = (double)warps * ITERS * 4;
        fma_per_sm = instr_per_sm * 256;
      } else {
        const double fi = (double)(warps / 2) * ITERS * 8, mi = (double)(warps / 2) * ITERS * 4;
        instr_per_sm = fi + mi;
        fma_per_sm = fi * 32 + mi * 256;
      }
      printf("%-36s threads/SM %4d: %7.2f FMA/cycle/SM, %.3f warp-instr/cycle/SM (%.0f cycles)\n", names[mode],
             threads, fma_per_sm / mean, instr_per_sm / mean, mean);
      cudaFree(out);
      cudaFree(cyc);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
