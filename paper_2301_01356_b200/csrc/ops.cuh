// ops.cuh -- stand-alone operations (ops.cu), called by the C ABI in api.cu.
#pragma once

#include "kernels.cuh"

namespace fbcc {

size_t op_list_ranking_bytes(int64_t L);
int op_list_ranking(const int* nxt, int64_t L, const int* heads, int64_t H, int* ranks, void* ws, Scalars* sc,
                    cudaStream_t st);

size_t op_symmetrize_bytes(int64_t k);
int op_symmetrize(const int64_t* u, const int64_t* v, int64_t k, int64_t n, int64_t* off, uint32_t* edges,
                  void* ws, Scalars* sc, cudaStream_t st);

size_t op_extract_bytes(int64_t n);
int op_extract_bccs(const int* label, const int* head, int64_t n, int* block_off, int* block_vtx, void* ws,
                    Scalars* sc, cudaStream_t st);

// dry = true: only report the workspace need
int op_build_euler_tour(int64_t n, const int2* pairs, int64_t k, const int* labels, int* parent, int* first,
                        int* last, void* ws, size_t ws_bytes, Scalars* sc, cudaStream_t st, bool dry, size_t* need);
int op_compute_tags(const Graph& g, const int* parent, const int* first, const int* last, int* w1, int* w2, int* low,
                    int* high, void* ws, size_t ws_bytes, cudaStream_t st, bool dry, size_t* need);

int op_classify_edges(const Graph& g, const int* parent, const int* first, const int* last, const int* low,
                      const int* high, int8_t* cls, Scalars* sc, cudaStream_t st);

}  // namespace fbcc
