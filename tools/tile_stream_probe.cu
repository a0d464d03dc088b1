// tile_stream_probe.cu -- DRAM bandwidth of the fused blur's access pattern without its arithmetic:
// persistent CTAs (one per SM) walk (z chunk, TX x TY column tile) items round-robin like blur3d_mma
// and, per plane, read a TX x TY tile of `in` and of `old` and write a TX x TY tile of `out`
// (plain coalesced loads / stores, 512 threads).  Compared with a flat streaming copy of the same
// bytes, it tells whether the tile shape (256-byte row pieces at a 4 KB stride) caps the blur.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_stream_probe tools/tile_stream_probe.cu
#include <cstdio>
#include <vector>

template <int TX, int TY, bool OLD>
__global__ void __launch_bounds__(512, 1) tiles(const double* __restrict__ in, const double* __restrict__ old,
                                                double* __restrict__ out, int n, int zchunk, int items) {
  const int tiles_x = n / TX, tiles_n = tiles_x * (n / TY);
  const size_t nxy = (size_t)n * n;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int t = item % tiles_n;
    const int z0 = (item / tiles_n) * zchunk, z1 = min(n, z0 + zchunk);
    const int x0 = (t % tiles_x) * TX, y0 = (t / tiles_x) * TY;
    // four planes in flight per thread (the blur keeps several planes in flight through its rings)
    for (int zb = z0; zb < z1; zb += 4) {
      constexpr int PER = TX * TY / 512;
      double v[4][PER];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int k = threadIdx.x + 512 * j, z = zb + u;
          const size_t i = (size_t)z * nxy + (size_t)(y0 + k / TX) * n + x0 + k % TX;
          v[u][j] = z < z1 ? __ldcs(in + i) + (OLD ? __ldcs(old + i) : 0.0) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int k = threadIdx.x + 512 * j, z = zb + u;
          const size_t i = (size_t)z * nxy + (size_t)(y0 + k / TX) * n + x0 + k % TX;
          if (z < z1) __stcs(out + i, v[u][j]);
        }
    }
  }
}

__global__ void flat(const double* __restrict__ in, const double* __restrict__ old, double* __restrict__ out,
                     size_t N) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __ldcs(in + i) + __ldcs(old + i);
}

template <int TX, int TY, bool OLD>
void run(const double* in, const double* old, double* out, int n, int sms) {
  const int tiles_n = (n / TX) * (n / TY);
  int zchunk = n;
  long best = -1;
  for (int zc = 1; zc <= n; ++zc) {
    const long items = (long)tiles_n * ((n + zc - 1) / zc);
    const long g = items < sms ? items : sms;
    const long cost = (items + g - 1) / g * (zc + 12);
    if (best < 0 || cost < best) best = cost, zchunk = zc;
  }
  const int items = tiles_n * ((n + zchunk - 1) / zchunk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) tiles<TX, TY, OLD><<<sms, 512>>>(in, old, out, n, zchunk, items);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) tiles<TX, TY, OLD><<<sms, 512>>>(in, old, out, n, zchunk, items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 10;
  const double bytes = 8.0 * n * n * n * (OLD ? 3 : 2);
  printf("tiles TX %3d TY %3d old %d zchunk %3d: %.3f ms  %.0f GB/s\n", TX, TY, (int)OLD, zchunk, ms, bytes / ms / 1e6);
}

int main() {
  const int n = 512;
  const size_t N = (size_t)n * n * n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *in, *old, *out;
  cudaMalloc(&in, 8 * N);
  cudaMalloc(&old, 8 * N);
  cudaMalloc(&out, 8 * N);
  cudaMemset(in, 0, 8 * N);
  cudaMemset(old, 0, 8 * N);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) flat<<<sms * 4, 512>>>(in, old, out, N);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) flat<<<sms * 4, 512>>>(in, old, out, N);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("flat (in + old -> out): %.3f ms  %.0f GB/s\n", ms / 10, 24.0 * N / (ms / 10) / 1e6);
  run<32, 32, true>(in, old, out, n, sms);
  run<32, 32, false>(in, old, out, n, sms);
  run<64, 16, true>(in, old, out, n, sms);
  run<64, 32, true>(in, old, out, n, sms);
  run<128, 8, true>(in, old, out, n, sms);
  run<128, 16, true>(in, old, out, n, sms);
  run<256, 8, true>(in, old, out, n, sms);
  run<512, 2, true>(in, old, out, n, sms);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
