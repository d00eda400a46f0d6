// Deterministic column merge of row-chunk partials: out[c] (+)= sum_k part[k][c],
// k ascending within each of kMergeWarps contiguous k-ranges, then the range sums
// in ascending order.  A fixed association (no atomics), so results are bitwise
// reproducible; 32 columns per CTA (coalesced 128 B rows), the warps split k.
#pragma once
#include "nnt_internal.h"

namespace nnt {

constexpr int kMergeWarps = 32;

// blockIdx.y selects one of up to three independent merges (part + y * group_stride -> out[y]),
// so the LayerNorm reductions (dgamma, dbeta and optionally sum_t dx) take one launch.
static __global__ void __launch_bounds__(32 * kMergeWarps)
    column_merge_kernel(const float* __restrict__ part_base, int64_t chunks, int64_t N, float* __restrict__ out0,
                        int accumulate, int64_t group_stride, float* __restrict__ out1, float* __restrict__ out2) {
  NNT_PDL_ENTRY();
  __shared__ float red[kMergeWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* __restrict__ part = part_base + blockIdx.y * group_stride;
  float* __restrict__ out = blockIdx.y == 0 ? out0 : (blockIdx.y == 1 ? out1 : out2);
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  const int64_t per = (chunks + kMergeWarps - 1) / kMergeWarps;
  const int64_t k0 = w * per, k1 = min(chunks, k0 + per);
  float s = 0.f;
  if (c < N) {
    int64_t k = k0;
    for (; k + 4 <= k1; k += 4) {
      float a = part[k * N + c], b = part[(k + 1) * N + c], d = part[(k + 2) * N + c], e = part[(k + 3) * N + c];
      s += a;
      s += b;
      s += d;
      s += e;
    }
    for (; k < k1; ++k) s += part[k * N + c];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kMergeWarps; ++i) t += red[i][lane];
    out[c] = accumulate ? out[c] + t : t;
  }
}

static inline void launch_column_merge(const float* part, int64_t chunks, int64_t N, float* out, int accumulate,
                                cudaStream_t s) {
  ::nnt::launch(column_merge_kernel, dim3((unsigned)((N + 31) / 32), 1), 32 * kMergeWarps, 0, s, part, chunks, N, out, accumulate,
                                                                                    0, out, out);
}
// two merges in one launch: part0 -> out0 and part0 + group_stride -> out1
static inline void launch_column_merge2(const float* part0, int64_t group_stride, int64_t chunks, int64_t N,
                                        float* out0, float* out1, int accumulate, cudaStream_t s) {
  ::nnt::launch(column_merge_kernel, dim3((unsigned)((N + 31) / 32), 2), 32 * kMergeWarps, 0, s, part0, chunks, N, out0,
                                                                                    accumulate, group_stride, out1, out1);
}

// three merges in one launch: part0 + y * group_stride -> out_y, y = 0, 1, 2
static inline void launch_column_merge3(const float* part0, int64_t group_stride, int64_t chunks, int64_t N,
                                        float* out0, float* out1, float* out2, int accumulate, cudaStream_t s) {
  ::nnt::launch(column_merge_kernel, dim3((unsigned)((N + 31) / 32), 3), 32 * kMergeWarps, 0, s, part0, chunks, N,
                out0, accumulate, group_stride, out1, out2);
}

}  // namespace nnt
