// Shared GEMM argument block and epilogue (SIMT fp32 path and tcgen05 bf16 path).
#pragma once
#include <cuda.h>

#include "nnt_internal.h"

namespace nnt {

struct GemmArgs {
  int ta, tb;
  int64_t M, N, K;
  int64_t batch0, batch1;
  float alpha, beta;
  const void* A;
  int64_t lda, sa0, sa1;
  const void* B;
  int64_t ldb, sb0, sb1;
  void* C;
  int64_t ldc, sc0, sc1;
  int c_dtype;
  int in_dtype;
  // epilogue
  const float* bias;
  const float* residual;
  int64_t ld_res;
  int act;
  void* aux;
  int64_t ld_aux;
  int causal;
  void* workspace;  // split-K partials (optional)
  size_t workspace_bytes;
  float* row_stats;  // fused softmax subroutine 1: per (row, 32-column tile) (max, sumexp)
  int64_t ld_stats;  // pairs per row
  const float* rowvec;  // NNT_ACT_SOFTMAX_BWD: D per row
  float rowscale;
  float* a_rowsum;  // R27: beta * a_rowsum + alpha * sum_k op(A)[i][k] (bias gradient of dW GEMMs)
  // R35 tensor-parallel row scatter: row i -> scat[i / scat_rows] + (scat_rank * scat_rows + i % scat_rows) * ldc
  int scat_R, scat_rank;
  int64_t scat_rows;
  float* scat[NNT_TP_MAX];
};

// Base pointer for row i of C under the R35 row scatter (row i's address = base + i * ldc), or Cb.
template <typename TC>
__device__ __forceinline__ TC* scatter_row_base(const GemmArgs& g, TC* Cb, int64_t i) {
  if (!g.scat_R) return Cb;
  const int64_t o = i / g.scat_rows;
  return reinterpret_cast<TC*>(g.scat[o]) + ((int64_t)g.scat_rank - o) * g.scat_rows * g.ldc;
}

nnt_status gemm_simt_launch(const GemmArgs& a, cudaStream_t s);
// *kernels (optional) receives the number of kernels launched (2 with a split-K reduce).
nnt_status gemm_tc_launch(const GemmArgs& a, cudaStream_t s, int* kernels = nullptr);
int64_t gemm_tc_splits(const GemmArgs& a);  // split-K factor the tcgen05 path would use
// split-K workspace bytes for `splits` (partials + a_rowsum partials + the in-kernel reduce's
// arrival counters; 0 when splits == 1)
size_t splitk_workspace_bytes(const GemmArgs& a, int64_t splits);
// stream-K workspace bytes (partial slots + flag zone; shape independent) and whether the
// stream-K schedule is enabled (NNT_GEMM_SK != 0)
size_t sk_workspace_bytes();
bool sk_on();
// 4-D TMA tensor map (dims {inner, outer, batch1, batch0}, SWIZZLE_128B, box {box_inner, box_outer,
// 1, 1}; es = element bytes, ld / s1 / s0 in elements)
nnt_status make_tma_map_4d(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t inner,
                           int64_t outer, int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_inner,
                           int box_outer);

// 5-D "blocked" TMA map of an [outer][mn] operand (row stride ld) as {64, outer, mn / 64, b1, b0}:
// one box {64, box_outer, nblk} stages nblk consecutive 64-element blocks of a row range, blocks
// 64 * box_outer * es bytes apart in shared memory (the SW128 layout of nblk separate 2-D boxes).
// mn % 64 == 0 only.  Returns false when not applicable or rejected (NNT_GEMM_BLOCKED=0: always).
bool make_tma_map_blocked(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t mn,
                          int64_t outer, int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_outer,
                          int nblk);

// Epilogue for one element: acc is sum_k op(A) op(B) of batch item (p,q), row i, col j.
template <typename TC>
__device__ __forceinline__ void epilogue_store(const GemmArgs& g, TC* __restrict__ Cb, TC* __restrict__ auxb,
                                               int64_t i, int64_t j, float acc) {
  float pre = g.alpha * acc;
  if (g.bias) pre += __ldg(g.bias + j);
  if (g.beta != 0.f) pre += g.beta * to_f32(Cb[i * g.ldc + j]);
  if (g.residual) pre += g.residual[i * g.ld_res + j];
  float out = pre;
  if (g.act == NNT_ACT_GELU) {
    auxb[i * g.ld_aux + j] = from_f32<TC>(pre);
    out = gelu_f(pre);
  } else if (g.act == NNT_ACT_GELU_BWD) {
    out = pre * gelu_grad_f(to_f32(auxb[i * g.ld_aux + j]));
  }
  scatter_row_base(g, Cb, i)[i * g.ldc + j] = from_f32<TC>(out);
}

}  // namespace nnt
