// gather_peak.cu -- microbenchmarks for the bounds the FAST-BCC kernels hit
// (DESIGN.md §3): random 4-byte gathers (the w gather, finds, label/record
// lookups) and dependent pointer chasing (list-ranking walks).  Measurement
// tooling only; not part of the product library.
//
//   gp_gather_stream: 8 consecutive indices per thread from a streamed index
//     array (two 16-byte loads, as the arc-balanced kernels read adj), one
//     4-byte gather arr[idx] each, min/max folded into one store per thread.
//   gp_gather_hash: 8 independent gathers per thread at hashed indices (no
//     index stream at all).
//   gp_chase: K independent chains over a random cyclic permutation; every
//     step is one dependent 4-byte load (the walk0 critical path).
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU;
  x ^= x >> 15; x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256, 8) k_gather_stream(const uint32_t* __restrict__ idx, int64_t nchunks,
                                                          const int* __restrict__ arr, int* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nchunks; q += (int64_t)gridDim.x * blockDim.x) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(idx) + 2 * q);
    const int4 y = __ldg(reinterpret_cast<const int4*>(idx) + 2 * q + 1);
    const uint32_t w[8] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w,
                           (uint32_t)y.x, (uint32_t)y.y, (uint32_t)y.z, (uint32_t)y.w};
    int m1 = 0x7fffffff, m2 = -1;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int f = __ldg(arr + w[i]);
      m1 = min(m1, f);
      m2 = max(m2, f);
    }
    out[q] = m1 ^ m2;
  }
}

__global__ void __launch_bounds__(256, 8) k_gather_hash(const int* __restrict__ arr, uint32_t nelem, int iters,
                                                        int* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0;
  for (int it = 0; it < iters; it++) {
    int v[8];
#pragma unroll
    for (int i = 0; i < 8; i++) v[i] = __ldg(arr + hash32(t * 8u + i + (uint32_t)it * 0x9E3779B1u) % nelem);
#pragma unroll
    for (int i = 0; i < 8; i++) acc += v[i];
  }
  out[t] = acc;
}

__global__ void k_perm_next(const uint32_t* __restrict__ perm, uint32_t n, int* __restrict__ nxt) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    nxt[perm[i]] = (int)perm[(i + 1) % n];
}

__global__ void __launch_bounds__(256) k_chase(const int* __restrict__ nxt, int chains, uint32_t n, int steps,
                                               int* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= chains) return;
  int e = (int)(hash32((uint32_t)j) % n);
  for (int s = 0; s < steps; s++) e = __ldg(nxt + e);
  out[j] = e;
}

static float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

extern "C" {

// mode 0: streamed indices (idx: count uint32 values < nelem, count % 8 == 0)
// mode 1: hashed indices (count gathers)
// Returns the best-of-reps gathers per second (< 0 on a CUDA error).
double gp_gather(int mode, const int* arr, uint32_t nelem, const uint32_t* idx, int64_t count, int* out, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  const int grid = 148 * 8;
  int iters = (int)(count / ((int64_t)grid * 256 * 8));
  if (iters < 1) iters = 1;
  if (mode != 0) count = (int64_t)iters * grid * 256 * 8;  // gathers actually issued
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a);
    if (mode == 0) {
      k_gather_stream<<<grid, 256>>>(idx, count / 8, arr, out);
    } else {
      k_gather_hash<<<grid, 256>>>(arr, nelem, iters, out);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    const double s = elapsed(a, b) * 1e-3;
    if (s > 0 && count / s > best) best = count / s;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// dependent chains over the cyclic permutation perm[0..n) (nxt: n ints of
// scratch): returns the mean nanoseconds per step of one chain.
double gp_chase(const uint32_t* perm, uint32_t n, int* nxt, int chains, int steps, int* out) {
  k_perm_next<<<148 * 8, 256>>>(perm, n, nxt);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_chase<<<(chains + 255) / 256, 256>>>(nxt, chains, n, 16, out);  // warm
  cudaEventRecord(a);
  k_chase<<<(chains + 255) / 256, 256>>>(nxt, chains, n, steps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  const double ns = elapsed(a, b) * 1e6 / steps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? ns : -1.0;
}
}
