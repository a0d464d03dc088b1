// vec.cuh -- device-side pieces shared by the operator / stencil / solver kernels.
#pragma once

#include "internal.cuh"

namespace mlsqr_b200 {

// POD copy of Epi passed by value to kernels
struct EpiArgs {
  const double* sx;
  const double* old;
  const double* so;
  const double* coef;
  double* seg;
  const int* gate;
};

inline EpiArgs to_args(const Epi& e) { return {e.sx, e.old, e.so, e.coef, e.seg, e.gate}; }

// xpby (kernels_scalar.cpp:19-21): out = a + coef * (old * so)
__device__ __forceinline__ double epilogue(double a, const EpiArgs& e, size_t i) {
  if (!e.old) return a;
  double o = e.old[i];
  if (e.so) o = o * *e.so;
  return a + *e.coef * o;
}

// cp.async (LDGSTS) helpers: src-size 0 zero-fills the destination
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// L2 prefetch (no register cost): z-marching kernels touch plane z + k early so the
// one-plane-ahead register loads hit L2 instead of waiting on HBM
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Three tree-32 levels over in[0 .. 32768) (zero padded past J); result in thread 0.
// Requires blockDim.x == 1024.  Thread t forms level 1 of group t (in[32t .. 32t+31]) with the
// serial emulation of tree32 (32 independent loads, 31 adds with ILP 16/8/4/2/1), the warp's
// shuffle tree forms level 2 over its 32 consecutive groups, warp 0 level 3 -- the canonical
// order, without the 32 dependent shuffle chains per warp of a warp-per-group level 1.
__device__ __forceinline__ double block_reduce3(const double* __restrict__ in, size_t J) {
  __shared__ double wres[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t base = (size_t)threadIdx.x * 32;
  double v[32];
  if (base + 32 <= J && !(reinterpret_cast<uintptr_t>(in + base) & 15)) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 q = *reinterpret_cast<const double2*>(in + base + 2 * k);
      v[2 * k] = q.x;
      v[2 * k + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = base + k < J ? in[base + k] : 0.0;
  }
  double keep = tree32_serial(v);
  keep = tree32(keep);
  if (lane == 0) wres[w] = keep;
  __syncthreads();
  double r = 0.0;
  if (w == 0) r = tree32(wres[lane]);
  __syncthreads();
  return r;
}

// Final canonical pass (<= 1024 partials, one warp: thread-serial level + shuffle level) fused
// with the scalar step that consumes the result: thread 0 writes *out, then runs fin() -- also
// when the reduction itself is gated off (the scalar steps test their own flags), exactly as the
// separate reduce + fin kernels did.
template <class F>
__global__ void __launch_bounds__(32) reduce_final_fin(const double* __restrict__ in, size_t J,
                                                       double* __restrict__ out, const int* gate, F fin) {
  const int lane = threadIdx.x;
  if (!(gate && *gate == 0)) {
    const size_t base = (size_t)lane * 32;
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = base + j < J ? in[base + j] : 0.0;
    const double r = tree32(tree32_serial(v));
    if (lane == 0) *out = r;
  }
  if (lane == 0) fin();
}

template <class F>
void reduce_segments_fin(Ctx* c, const double* seg, size_t nseg, double* scratch, double* out, const int* gate,
                         F fin) {
  size_t J = 0;
  const double* cur = reduce_segments_to_warp(c, seg, nseg, scratch, gate, &J);
  reduce_final_fin<F><<<1, 32, 0, c->stream>>>(cur, J, out, gate, fin);
  c->count();
  c->check_launch();
}

}  // namespace mlsqr_b200
