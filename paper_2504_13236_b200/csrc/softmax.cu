// Attention softmax as the paper's two subroutines plus its
// backward.  One warp per slice (row of keys); the row is held in registers as
// float4 chunks (128 columns per chunk, 4 per lane), reductions by warp
// shuffle.  Causal rows touch only their valid prefix k <= q (about half of the
// S x S bytes), and the probability row is zero-filled only up to the next
// NNT_CAUSAL_ALIGN boundary that the tensor-core GEMMs read.
#include <math_constants.h>

#include "nnt_internal.h"

namespace nnt {
namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerBlock = kThreads / 32;
constexpr int kMaxChunks = 16;  // cols <= 2048 in registers
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) { return exp2f(x); }

// merge (m,s) (+) (m2,s2); (-inf, 0) is the identity (R10)
__device__ __forceinline__ void mse_merge(float& m, float& s, float m2, float s2) {
  float M = fmaxf(m, m2);
  if (M == -CUDART_INF_F) return;  // both empty
  float a = (m == -CUDART_INF_F) ? 0.f : s * ex2((m - M) * kLog2e);
  float b = (m2 == -CUDART_INF_F) ? 0.f : s2 * ex2((m2 - M) * kLog2e);
  m = M;
  s = a + b;
}

__device__ __forceinline__ int64_t valid_cols(int64_t row, int64_t cols, int causal, int64_t seq_q) {
  if (!causal) return cols;
  int64_t q = row % seq_q;
  return min(cols, q + 1);
}
__device__ __forceinline__ int64_t write_cols(int64_t row, int64_t cols, int causal, int64_t seq_q) {
  if (!causal) return cols;
  int64_t q = row % seq_q;
  int64_t w = ((q + 1 + NNT_CAUSAL_ALIGN - 1) / NNT_CAUSAL_ALIGN) * NNT_CAUSAL_ALIGN;
  return min(cols, w);
}

template <typename T>
__device__ __forceinline__ float4 load4(const T* p);
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 lo = *reinterpret_cast<__nv_bfloat162*>(&u.x), hi = *reinterpret_cast<__nv_bfloat162*>(&u.y);
  float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
  return make_float4(a.x, a.y, b.x, b.y);
}
template <typename T>
__device__ __forceinline__ void store4(T* p, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = pk;
}

__device__ __forceinline__ float comp(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// ------------------------------------------------------------------ subroutine 1
template <int NC>
__global__ void __launch_bounds__(kThreads) maxsumexp_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                             int64_t ldx, int64_t tile_k, int causal, int64_t seq_q,
                                                             float* __restrict__ stats, int accumulate) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t nvalid = valid_cols(row, cols, causal, seq_q);
  const float* xr = x + row * ldx;
  float4 v[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int64_t col = (int64_t)c * 128 + lane * 4;
    v[c] = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
    if (col < nvalid) {
      float4 t = *reinterpret_cast<const float4*>(xr + col);
      v[c].x = t.x;
      v[c].y = (col + 1 < nvalid) ? t.y : -CUDART_INF_F;
      v[c].z = (col + 2 < nvalid) ? t.z : -CUDART_INF_F;
      v[c].w = (col + 3 < nvalid) ? t.w : -CUDART_INF_F;
    }
  }
  float M = -CUDART_INF_F, S = 0.f;
  if (tile_k >= nvalid) {
    // one key tile covers the slice: (m, s) straight from registers (masked entries are -inf -> 0)
    float mj = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < NC; ++c) mj = fmaxf(fmaxf(mj, fmaxf(v[c].x, v[c].y)), fmaxf(v[c].z, v[c].w));
    mj = warp_max(mj);
    float sj = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c * 128 < nvalid)  // warp-uniform: skip chunks entirely past the causal prefix
        sj += (ex2((v[c].x - mj) * kLog2e) + ex2((v[c].y - mj) * kLog2e)) +
              (ex2((v[c].z - mj) * kLog2e) + ex2((v[c].w - mj) * kLog2e));
    sj = warp_sum(sj);
    M = mj;
    S = sj;
  }
  // per key tile [t0, t0 + tile_k): partial (m_j, s_j), merged in ascending order
  for (int64_t t0 = 0; tile_k < nvalid && t0 < nvalid; t0 += tile_k) {
    const int64_t t1 = min(t0 + tile_k, nvalid);
    float mj = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t col = (int64_t)c * 128 + lane * 4 + i;
        if (col >= t0 && col < t1) mj = fmaxf(mj, comp(v[c], i));
      }
    mj = warp_max(mj);
    const float mjv = mj;
    float sj = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t col = (int64_t)c * 128 + lane * 4 + i;
        if (col >= t0 && col < t1) sj += ex2((comp(v[c], i) - mjv) * kLog2e);
      }
    sj = warp_sum(sj);
    mse_merge(M, S, mj, sj);
  }
  if (lane == 0) {
    if (accumulate) {
      float m0 = stats[2 * row], s0 = stats[2 * row + 1];
      mse_merge(m0, s0, M, S);
      M = m0;
      S = s0;
    }
    stats[2 * row] = M;
    stats[2 * row + 1] = S;
  }
}

// ------------------------------------------------------------------ aggregation of subroutine 1
// One thread per slice: merges its key-tile partials in ascending tile order (R10).
__global__ void __launch_bounds__(kThreads) maxsumexp_merge_kernel(const float2* __restrict__ part, int64_t rows,
                                                                   int64_t nparts, int64_t ld, int64_t part_cols,
                                                                   int causal, int64_t seq_q,
                                                                   float2* __restrict__ stats) {
  NNT_PDL_ENTRY();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  int64_t n = nparts;
  if (causal) n = min(n, (row % seq_q) / part_cols + 1);
  const float2* pr = part + row * ld;
  float M = -CUDART_INF_F, S = 0.f;
  for (int64_t gi = 0; gi < n; ++gi) {
    const float2 p = pr[gi];
    mse_merge(M, S, p.x, p.y);
  }
  stats[row] = make_float2(M, S);
}

// ------------------------------------------------------------------ D = rowdot(dO, O) per (b, head, s)
// One thread per (b, s, head): h contiguous elements of dO and O (16-byte loads when
// h*sizeof(T) % 16 == 0); output index (b*H + n)*S + s.
template <typename T>
__global__ void __launch_bounds__(kThreads) attn_rowdot_kernel(const T* __restrict__ dO, const T* __restrict__ O,
                                                               int64_t B, int64_t S, int64_t H, int64_t h,
                                                               float* __restrict__ D) {
  NNT_PDL_ENTRY();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // ((b*S + s)*H + n)
  if (idx >= B * S * H) return;
  const int64_t n = idx % H, bs = idx / H, b = bs / S, s = bs % S;
  const T* a = dO + bs * H * h + n * h;
  const T* o = O + bs * H * h + n * h;
  float acc = 0.f;
  constexpr int V = 16 / sizeof(T);
  if ((h * sizeof(T)) % 16 == 0) {
    for (int64_t i = 0; i < h; i += V) {
      uint4 ua = *reinterpret_cast<const uint4*>(a + i), uo = *reinterpret_cast<const uint4*>(o + i);
      const T* ea = reinterpret_cast<const T*>(&ua);
      const T* eo = reinterpret_cast<const T*>(&uo);
#pragma unroll
      for (int j = 0; j < V; ++j) acc = fmaf(to_f32(ea[j]), to_f32(eo[j]), acc);
    }
  } else {
    for (int64_t i = 0; i < h; ++i) acc = fmaf(to_f32(a[i]), to_f32(o[i]), acc);
  }
  D[(b * H + n) * S + s] = acc;
}

// Lane-cooperative form: L lanes per (token, head) row, one 16-byte vector each (h = L x 16 B),
// so every warp load instruction reads 32 / L whole rows contiguously; the L partial dot
// products are combined by an xor tree (fixed order).  Used whenever h x sizeof(T) / 16 is a
// power of two <= 32 (GPT-2: h = 64 bf16 -> L = 8); otherwise the thread-per-row kernel above.
template <typename T, int L>
__global__ void __launch_bounds__(kThreads) attn_rowdot_lanes_kernel(const T* __restrict__ dO,
                                                                     const T* __restrict__ O, int64_t B, int64_t S,
                                                                     int64_t H, float* __restrict__ D) {
  NNT_PDL_ENTRY();
  constexpr int V = 16 / sizeof(T);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t idx = t / L;  // ((b*S + s)*H + n); rows are h = L*V elements, contiguous
  const int part = (int)(t % L);
  float acc = 0.f;
  if (idx < B * S * H) {
    const uint4 ua = __ldg(reinterpret_cast<const uint4*>(dO) + t), uo = __ldg(reinterpret_cast<const uint4*>(O) + t);
    const T* ea = reinterpret_cast<const T*>(&ua);
    const T* eo = reinterpret_cast<const T*>(&uo);
#pragma unroll
    for (int j = 0; j < V; ++j) acc = fmaf(to_f32(ea[j]), to_f32(eo[j]), acc);
  }
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (part == 0 && idx < B * S * H) {
    const int64_t n = idx % H, bs = idx / H, b = bs / S, s = bs % S;
    D[(b * H + n) * S + s] = acc;
  }
}

// ------------------------------------------------------------------ subroutine 2
template <typename TO>
__global__ void __launch_bounds__(kThreads) softmax_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                           int64_t ldx, int causal, int64_t seq_q,
                                                           const float* __restrict__ stats, TO* __restrict__ y,
                                                           int64_t ldy) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t nvalid = valid_cols(row, cols, causal, seq_q);
  const int64_t nwrite = write_cols(row, cols, causal, seq_q);
  const float M = stats[2 * row], inv_s = 1.0f / stats[2 * row + 1];
  const float* xr = x + row * ldx;
  TO* yr = y + row * ldy;
  for (int64_t col = lane * 4; col < nwrite; col += 128) {
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < nvalid) {
      float4 t = *reinterpret_cast<const float4*>(xr + col);
      o.x = ex2((t.x - M) * kLog2e) * inv_s;
      o.y = (col + 1 < nvalid) ? ex2((t.y - M) * kLog2e) * inv_s : 0.f;
      o.z = (col + 2 < nvalid) ? ex2((t.z - M) * kLog2e) * inv_s : 0.f;
      o.w = (col + 3 < nvalid) ? ex2((t.w - M) * kLog2e) * inv_s : 0.f;
    }
    store4<TO>(yr + col, o);
  }
}

// ------------------------------------------------------------------ backward
template <typename TP, typename TO, int NC>
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(const TP* __restrict__ p, int64_t ldp,
                                                               const float* __restrict__ dp, int64_t lddp,
                                                               int64_t rows, int64_t cols, int causal, int64_t seq_q,
                                                               float scale, TO* __restrict__ da, int64_t ldda) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t nvalid = valid_cols(row, cols, causal, seq_q);
  const int64_t nwrite = write_cols(row, cols, causal, seq_q);
  const TP* pr = p + row * ldp;
  const float* dr = dp + row * lddp;
  float4 pv[NC], dv[NC];
  float d = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int64_t col = (int64_t)c * 128 + lane * 4;
    pv[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    dv[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < nvalid) {
      float4 a = load4<TP>(pr + col);
      float4 b = *reinterpret_cast<const float4*>(dr + col);
      pv[c].x = a.x; dv[c].x = b.x;
      if (col + 1 < nvalid) { pv[c].y = a.y; dv[c].y = b.y; }
      if (col + 2 < nvalid) { pv[c].z = a.z; dv[c].z = b.z; }
      if (col + 3 < nvalid) { pv[c].w = a.w; dv[c].w = b.w; }
      d += (pv[c].x * dv[c].x + pv[c].y * dv[c].y) + (pv[c].z * dv[c].z + pv[c].w * dv[c].w);
    }
  }
  d = warp_sum(d);
  TO* orow = da + row * ldda;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int64_t col = (int64_t)c * 128 + lane * 4;
    if (col < nwrite) {
      float4 o;
      o.x = scale * pv[c].x * (dv[c].x - d);
      o.y = scale * pv[c].y * (dv[c].y - d);
      o.z = scale * pv[c].z * (dv[c].z - d);
      o.w = scale * pv[c].w * (dv[c].w - d);
      store4<TO>(orow + col, o);
    }
  }
}

inline unsigned row_blocks(int64_t rows) { return (unsigned)((rows + kRowsPerBlock - 1) / kRowsPerBlock); }

int chunks_for(int64_t cols) {
  int64_t c = (cols + 127) / 128;
  const int opts[] = {1, 2, 4, 8, 16};
  for (int o : opts)
    if (o >= c) return o;
  return -1;
}

}  // namespace
}  // namespace nnt

using namespace nnt;

static nnt_status check_rows(const char* who, int64_t rows, int64_t cols, int64_t ld, int causal, int64_t seq_q) {
  NNT_REQUIRE(rows > 0 && cols > 0 && ld >= cols, NNT_ERR_SHAPE, "%s: rows=%lld cols=%lld ld=%lld", who,
              (long long)rows, (long long)cols, (long long)ld);
  NNT_REQUIRE(!causal || seq_q > 0, NNT_ERR_SHAPE, "%s: causal needs seq_q > 0", who);
  NNT_REQUIRE(cols % 4 == 0 && ld % 4 == 0, NNT_ERR_ALIGN, "%s: cols and ld must be multiples of 4", who);
  NNT_REQUIRE(chunks_for(cols) > 0, NNT_ERR_UNSUPPORTED, "%s: cols=%lld > 2048", who, (long long)cols);
  return NNT_OK;
}

extern "C" {

nnt_status nnt_maxsumexp(const float* x, int64_t rows, int64_t cols, int64_t ldx, int64_t tile_k, int causal,
                         int64_t seq_q, float* stats, int accumulate, nnt_stream_t stream) {
  NNT_REQUIRE(x && stats, NNT_ERR_NULL, "nnt_maxsumexp: NULL pointer");
  NNT_TRY(check_rows("nnt_maxsumexp", rows, cols, ldx, causal, seq_q));
  NNT_REQUIRE(tile_k > 0, NNT_ERR_TILE, "nnt_maxsumexp: tile_k=%lld", (long long)tile_k);
  NNT_REQUIRE(aligned16(x), NNT_ERR_ALIGN, "nnt_maxsumexp: x not 16B aligned");
  double frac = causal ? 0.5 * (1.0 + 1.0 / (double)cols) : 1.0;
  LaunchScope sc(NNT_K_MAXSUMEXP, stream, 4.0 * rows * cols * frac + 8.0 * rows, 0);
  int nc = chunks_for(cols);
#define NNT_MSE(N)                                                                                         \
  case N:                                                                                                  \
    ::nnt::launch(maxsumexp_kernel<N>, row_blocks(rows), kThreads, 0, stream, x, rows, cols, ldx, tile_k, causal, seq_q, \
                                                                   stats, accumulate);                     \
    break;
  switch (nc) { NNT_MSE(1) NNT_MSE(2) NNT_MSE(4) NNT_MSE(8) NNT_MSE(16) }
#undef NNT_MSE
  return check_launch("maxsumexp");
}

nnt_status nnt_attn_rowdot(const void* dO, const void* O, int dtype, int64_t B, int64_t S, int64_t H, int64_t h,
                           float* D, nnt_stream_t stream) {
  NNT_REQUIRE(dO && O && D, NNT_ERR_NULL, "nnt_attn_rowdot: NULL pointer");
  NNT_REQUIRE(B > 0 && S > 0 && H > 0 && h > 0, NNT_ERR_SHAPE, "nnt_attn_rowdot: bad shape");
  NNT_REQUIRE(valid_dtype(dtype), NNT_ERR_DTYPE, "nnt_attn_rowdot: dtype %d", dtype);
  NNT_REQUIRE(aligned16(dO) && aligned16(O), NNT_ERR_ALIGN, "nnt_attn_rowdot: pointers must be 16-byte aligned");
  const int64_t n = B * S * H;
  LaunchScope sc(NNT_K_MISC, stream, 2.0 * dtype_size(dtype) * n * h + 4.0 * n, 2.0 * n * h);
  const int64_t lanes = (h * (int64_t)dtype_size(dtype)) % 16 == 0 ? h * (int64_t)dtype_size(dtype) / 16 : 0;
  if (lanes == 2 || lanes == 4 || lanes == 8 || lanes == 16 || lanes == 32) {
    const unsigned g = (unsigned)((n * lanes + kThreads - 1) / kThreads);
#define NNT_RDL(T, LN)                                                                                         \
  case LN:                                                                                                     \
    ::nnt::launch(attn_rowdot_lanes_kernel<T, LN>, g, kThreads, 0, stream, (const T*)dO, (const T*)O, B, S, H, D); \
    break;
    if (dtype == NNT_BF16) {
      switch (lanes) { NNT_RDL(__nv_bfloat16, 2) NNT_RDL(__nv_bfloat16, 4) NNT_RDL(__nv_bfloat16, 8)
                       NNT_RDL(__nv_bfloat16, 16) NNT_RDL(__nv_bfloat16, 32) }
    } else {
      switch (lanes) { NNT_RDL(float, 2) NNT_RDL(float, 4) NNT_RDL(float, 8) NNT_RDL(float, 16) NNT_RDL(float, 32) }
    }
#undef NNT_RDL
    return check_launch("attn_rowdot");
  }
  const unsigned grid = (unsigned)((n + kThreads - 1) / kThreads);
  if (dtype == NNT_BF16)
    ::nnt::launch(attn_rowdot_kernel<__nv_bfloat16>, grid, kThreads, 0, stream, (const __nv_bfloat16*)dO,
                                                                     (const __nv_bfloat16*)O, B, S, H, h, D);
  else
    ::nnt::launch(attn_rowdot_kernel<float>, grid, kThreads, 0, stream, (const float*)dO, (const float*)O, B, S, H, h, D);
  return check_launch("attn_rowdot");
}

nnt_status nnt_maxsumexp_merge(const float* part, int64_t rows, int64_t nparts, int64_t ld_parts, int64_t part_cols,
                               int causal, int64_t seq_q, float* stats, nnt_stream_t stream) {
  NNT_REQUIRE(part && stats, NNT_ERR_NULL, "nnt_maxsumexp_merge: NULL pointer");
  NNT_REQUIRE(rows > 0 && nparts > 0 && ld_parts >= nparts, NNT_ERR_SHAPE,
              "nnt_maxsumexp_merge: rows=%lld nparts=%lld ld=%lld", (long long)rows, (long long)nparts,
              (long long)ld_parts);
  NNT_REQUIRE(part_cols > 0, NNT_ERR_TILE, "nnt_maxsumexp_merge: part_cols=%lld", (long long)part_cols);
  NNT_REQUIRE(!causal || seq_q > 0, NNT_ERR_SHAPE, "nnt_maxsumexp_merge: causal needs seq_q > 0");
  NNT_REQUIRE((reinterpret_cast<uintptr_t>(part) & 7u) == 0 && (reinterpret_cast<uintptr_t>(stats) & 7u) == 0,
              NNT_ERR_ALIGN, "nnt_maxsumexp_merge: pointers must be 8-byte aligned");
  LaunchScope sc(NNT_K_MAXSUMEXP, stream, 8.0 * rows * (causal ? 0.5 : 1.0) * nparts + 8.0 * rows, 0);
  ::nnt::launch(maxsumexp_merge_kernel, (unsigned)((rows + kThreads - 1) / kThreads), kThreads, 0, stream, 
      (const float2*)part, rows, nparts, ld_parts, part_cols, causal, seq_q, (float2*)stats);
  return check_launch("maxsumexp_merge");
}

nnt_status nnt_softmax(const float* x, int64_t rows, int64_t cols, int64_t ldx, int64_t tile_k, int causal,
                       int64_t seq_q, const float* stats, void* y, int y_dtype, int64_t ldy, nnt_stream_t stream) {
  NNT_REQUIRE(x && stats && y, NNT_ERR_NULL, "nnt_softmax: NULL pointer");
  NNT_TRY(check_rows("nnt_softmax", rows, cols, ldx, causal, seq_q));
  NNT_REQUIRE(ldy >= cols && ldy % 4 == 0, NNT_ERR_SHAPE, "nnt_softmax: ldy=%lld", (long long)ldy);
  NNT_REQUIRE(tile_k > 0, NNT_ERR_TILE, "nnt_softmax: tile_k=%lld", (long long)tile_k);
  NNT_REQUIRE(valid_dtype(y_dtype), NNT_ERR_DTYPE, "nnt_softmax: dtype %d", y_dtype);
  NNT_REQUIRE(aligned16(x) && aligned16(y), NNT_ERR_ALIGN, "nnt_softmax: pointers not 16B aligned");
  double frac = causal ? 0.5 * (1.0 + 1.0 / (double)cols) : 1.0;
  LaunchScope sc(NNT_K_SOFTMAX, stream, (4.0 + dtype_size(y_dtype)) * rows * cols * frac + 8.0 * rows, 0);
  if (y_dtype == NNT_F32)
    ::nnt::launch(softmax_kernel<float>, row_blocks(rows), kThreads, 0, stream, x, rows, cols, ldx, causal, seq_q, stats,
                                                                     (float*)y, ldy);
  else
    ::nnt::launch(softmax_kernel<__nv_bfloat16>, row_blocks(rows), kThreads, 0, stream, x, rows, cols, ldx, causal, seq_q,
                                                                             stats, (__nv_bfloat16*)y, ldy);
  return check_launch("softmax");
}

nnt_status nnt_softmax_bwd(const void* p, int p_dtype, int64_t ldp, const float* dp, int64_t lddp, int64_t rows,
                           int64_t cols, int causal, int64_t seq_q, float scale, void* da, int da_dtype,
                           int64_t ldda, nnt_stream_t stream) {
  NNT_REQUIRE(p && dp && da, NNT_ERR_NULL, "nnt_softmax_bwd: NULL pointer");
  NNT_TRY(check_rows("nnt_softmax_bwd", rows, cols, lddp, causal, seq_q));
  NNT_REQUIRE(ldp >= cols && ldda >= cols && ldp % 4 == 0 && ldda % 4 == 0, NNT_ERR_SHAPE,
              "nnt_softmax_bwd: leading dims");
  NNT_REQUIRE(valid_dtype(p_dtype) && valid_dtype(da_dtype), NNT_ERR_DTYPE, "nnt_softmax_bwd: dtype");
  NNT_REQUIRE(aligned16(p) && aligned16(dp) && aligned16(da), NNT_ERR_ALIGN, "nnt_softmax_bwd: alignment");
  double frac = causal ? 0.5 * (1.0 + 1.0 / (double)cols) : 1.0;
  LaunchScope sc(NNT_K_SOFTMAX_BWD, stream,
                 (dtype_size(p_dtype) + 4.0 + dtype_size(da_dtype)) * rows * cols * frac, 0);
  int nc = chunks_for(cols);
  unsigned g = row_blocks(rows);
#define NNT_SMB(TP, TO, N)                                                                               \
  case N:                                                                                                \
    ::nnt::launch(softmax_bwd_kernel<TP, TO, N>, g, kThreads, 0, stream, (const TP*)p, ldp, dp, lddp, rows, cols,    \
                                                              causal, seq_q, scale, (TO*)da, ldda);      \
    break;
#define NNT_SMB_ALL(TP, TO) \
  switch (nc) { NNT_SMB(TP, TO, 1) NNT_SMB(TP, TO, 2) NNT_SMB(TP, TO, 4) NNT_SMB(TP, TO, 8) NNT_SMB(TP, TO, 16) }
  if (p_dtype == NNT_F32 && da_dtype == NNT_F32) {
    NNT_SMB_ALL(float, float)
  } else if (p_dtype == NNT_BF16 && da_dtype == NNT_BF16) {
    NNT_SMB_ALL(__nv_bfloat16, __nv_bfloat16)
  } else if (p_dtype == NNT_F32 && da_dtype == NNT_BF16) {
    NNT_SMB_ALL(float, __nv_bfloat16)
  } else {
    NNT_SMB_ALL(__nv_bfloat16, float)
  }
#undef NNT_SMB_ALL
#undef NNT_SMB
  return check_launch("softmax_bwd");
}

}  // extern "C"
