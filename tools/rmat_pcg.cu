// rmat_pcg.cu -- config-5 RMAT edge pairs on the GPU, bit-identical to
// workloads.rmat / _rmat_pairs (numpy Generator(PCG64(seed)).random draws,
// level-major per chunk).  Test/bench input generation only (the numpy path
// takes ~3 minutes for 5.4e8 edges); not part of the product library.
//
// numpy's PCG64 is PCG XSL-RR 128/64: state = state * MULT + inc, output
// rotr64(hi ^ lo, hi >> 58) of the new state; random() = (out >> 11) * 2^-53.
// Draw j of the stream is reached by the O(log j) LCG jump-ahead.
#include <cstdint>

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ u128 advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_m = 1, acc_p = 0, cur_m = mult(), cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  return acc_m * s + acc_p;
}

__device__ __forceinline__ uint64_t out(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64 - r) & 63));
}

// one chunk of k edges; `base` = draws consumed before the chunk
__global__ void gen_rmat(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t base, int64_t k,
                       int scale, int per, int64_t* u, int64_t* v) {
  const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * per;
  if (i0 >= k) return;
  const int64_t i1 = i0 + per < k ? i0 + per : k;
  for (int64_t i = i0; i < i1; i++) { u[i] = 0; v[i] = 0; }
  for (int lvl = 0; lvl < scale; lvl++) {
    u128 s = advance(s0, inc, base + (uint64_t)lvl * (uint64_t)k + (uint64_t)i0);
    const int64_t bit = (int64_t)1 << (scale - 1 - lvl);
    for (int64_t i = i0; i < i1; i++) {
      s = s * mult() + inc;
      const double r = (double)(out(s) >> 11) * (1.0 / 9007199254740992.0);
      if (r >= 0.76) u[i] |= bit;
      if ((r >= 0.57 && r < 0.76) || r >= 0.95) v[i] |= bit;
    }
  }
}

extern "C" int rmat_pairs_chunk(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint64_t base, int64_t k,
                                int scale, int64_t* u, int64_t* v, void* stream) {
  const int per = 256, B = 128;
  const int64_t threads = (k + per - 1) / per;
  const int grid = (int)((threads + B - 1) / B);
  gen_rmat<<<grid, B, 0, (cudaStream_t)stream>>>(s_hi, s_lo, i_hi, i_lo, base, k, scale, per, u, v);
  return (int)cudaGetLastError();
}
