// vec.cuh -- device-side pieces shared by the operator / stencil / solver kernels.
#pragma once

#include <cooperative_groups.h>

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

// one reduce2_kernel pass (vec.cu): J values -> K = ceil(J / 1024)
void reduce2_pass(Ctx* c, const double* in, size_t J, size_t K, double* out, const int* gate);

// The last two-level pass, when it leaves at most 64 values (at most 8 blocks of reduce2_kernel),
// fused with the final one-warp pass in ONE launch: the blocks form a thread-block cluster, each
// warp's level-2 value goes straight into block 0's shared memory (DSMEM), a cluster barrier
// (release / acquire), then block 0's first warp runs reduce_final_fin's pass over them and the
// scalar step.  The same values meet the same trees in the same order, so the result is
// bit-identical; one launch per reduction fewer (four per LSQR iteration).
template <class F>
__global__ void __launch_bounds__(256) reduce2_final_fin(const double* __restrict__ in, size_t J, size_t K,
                                                         double* __restrict__ out, const int* gate, F fin) {
  namespace cg = cooperative_groups;
  __shared__ double part[64];
  cg::cluster_group cl = cg::this_cluster();
  const bool live = !(gate && *gate == 0);
  const int lane = threadIdx.x & 31;
  const size_t k = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (live && k < K) {  // reduce2_kernel's warp
    const size_t base = k * 1024 + (size_t)lane * 32;
    double v[32];
    if (base + 32 <= J && !(reinterpret_cast<uintptr_t>(in + base) & 15)) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double2 q = *reinterpret_cast<const double2*>(in + base + 2 * j);
        v[2 * j] = q.x;
        v[2 * j + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = base + j < J ? in[base + j] : 0.0;
    }
    const double r = tree32(tree32_serial(v));
    if (lane == 0) cl.map_shared_rank(part, 0)[k] = r;
  }
  cl.sync();
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // reduce_final_fin over the K values
    if (live) {
      const size_t base = (size_t)lane * 32;
      double v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = base + j < K ? part[base + j] : 0.0;
      const double r = tree32(tree32_serial(v));
      if (lane == 0) *out = r;
    }
    if (lane == 0) fin();
  }
}

template <class F>
void reduce_segments_fin(Ctx* c, const double* seg, size_t nseg, double* scratch, double* out, const int* gate,
                         F fin) {
  // MLSQR_CLUSTER_FIN=0: the last pass and the final pass as two launches
  static const bool fused = !(getenv("MLSQR_CLUSTER_FIN") && getenv("MLSQR_CLUSTER_FIN")[0] == '0');
  if (fused && nseg > 1024) {
    const double* cur = seg;
    size_t J = nseg;
    double* s = scratch;
    while (J > 64 * 1024) {
      const size_t K = (J + 1023) / 1024;
      reduce2_pass(c, cur, J, K, s, gate);
      cur = s;
      s += K;
      J = K;
    }
    if (J > 1024) {
      const size_t K = (J + 1023) / 1024;
      const unsigned nb = (unsigned)((K + 7) / 8);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(nb);
      cfg.blockDim = dim3(256);
      cfg.stream = c->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = nb;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      MLSQR_CUDA(cudaLaunchKernelEx(&cfg, reduce2_final_fin<F>, cur, J, K, out, gate, fin));
    } else {
      reduce_final_fin<F><<<1, 32, 0, c->stream>>>(cur, J, out, gate, fin);
    }
    c->count();
    c->check_launch();
    return;
  }
  size_t J = 0;
  const double* cur = reduce_segments_to_warp(c, seg, nseg, scratch, gate, &J);
  reduce_final_fin<F><<<1, 32, 0, c->stream>>>(cur, J, out, gate, fin);
  c->count();
  c->check_launch();
}

}  // namespace mlsqr_b200
