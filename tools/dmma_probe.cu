// dmma_probe.cu -- what rounding does the FP64 tensor-core MMA (mma.sync m8n8k4 f64) perform?
// Compares D = A(8x4) B(4x8) + C on the device with host models of the k-sum:
//   seq  : fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))   (an fma chain in ascending k)
//   rev  : the same chain in descending k
//   exact: the exact sum rounded once (long double / two-sum emulation)
// Inputs are drawn with wide exponent spread so that the models disagree often.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o dmma_probe tools/dmma_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__global__ void dmma_kernel(const double* A, const double* B, const double* C, double* D, int reps) {
  // fragment layout for m8n8k4 f64 (row.col): lane l holds A[l/4][l%4], B[l%4][l/4],
  // C/D: two elements D[l/4][2*(l%4) + {0,1}]
  const int l = threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    const double* a = A + r * 32;
    const double* b = B + r * 32;
    const double* c = C + r * 64;
    double* d = D + r * 64;
    const double av = a[(l / 4) * 4 + (l % 4)];
    const double bv = b[(l % 4) * 8 + (l / 4)];
    const double c0 = c[(l / 4) * 8 + 2 * (l % 4)], c1 = c[(l / 4) * 8 + 2 * (l % 4) + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(av), "d"(bv), "d"(c0), "d"(c1));
    d[(l / 4) * 8 + 2 * (l % 4)] = d0;
    d[(l / 4) * 8 + 2 * (l % 4) + 1] = d1;
  }
}

int main() {
  const int reps = 20000;
  std::vector<double> A(reps * 32), B(reps * 32), C(reps * 64), D(reps * 64);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1, 1);
  std::uniform_int_distribution<int> e(-30, 30);
  for (auto& x : A) x = std::ldexp(u(g), e(g));
  for (auto& x : B) x = std::ldexp(u(g), e(g));
  for (auto& x : C) x = std::ldexp(u(g), e(g) * 2);
  double *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, A.size() * 8);
  cudaMalloc(&dB, B.size() * 8);
  cudaMalloc(&dC, C.size() * 8);
  cudaMalloc(&dD, D.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  dmma_kernel<<<1, 32>>>(dA, dB, dC, dD, reps);
  cudaError_t err = cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
  if (err != cudaSuccess) {
    printf("cuda error %s\n", cudaGetErrorString(err));
    return 1;
  }
  long seq = 0, rev = 0, exact = 0, total = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        const double* a = &A[r * 32 + i * 4];
        double bb[4];
        for (int k = 0; k < 4; ++k) bb[k] = B[r * 32 + k * 8 + j];
        const double c = C[r * 64 + i * 8 + j];
        const double d = D[r * 64 + i * 8 + j];
        double s = c;
        for (int k = 0; k < 4; ++k) s = std::fma(a[k], bb[k], s);
        double t = c;
        for (int k = 3; k >= 0; --k) t = std::fma(a[k], bb[k], t);
        __float128 q = (__float128)c;
        for (int k = 0; k < 4; ++k) q += (__float128)a[k] * (__float128)bb[k];
        const double x = (double)q;
        seq += d == s;
        rev += d == t;
        exact += d == x;
        ++total;
      }
  printf("DMMA m8n8k4 f64 vs models over %ld outputs: seq-fma %ld, rev-fma %ld, exact-once %ld\n", total, seq, rev,
         exact);
  return 0;
}
