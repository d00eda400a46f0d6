// GPT-2 shell: the embedding layer and the cross-entropy loss
// built from the two SoftMax subroutines.  The tied LM head itself is
// two nnt_tile_gemm calls made by the driver.
//
//   nnt_embedding_fwd  x[t] = wte[ids[t]] + wpe[t mod S]           (warp per token, float4)
//   nnt_embedding_bwd  dwte[v] (+)= sum of dx over the tokens with id v, in token order;
//                      dwpe[s] (+)= sum_b dx[b, s]
//                      deterministic without atomics on floats: a counting sort of the token
//                      positions by id (integer histogram, one-CTA exclusive scan, stable rank
//                      = number of earlier tokens with the same id), then one warp per
//                      vocabulary row sums its bucket in token order
//   nnt_cross_entropy  per row: subroutine 1 (per-thread running (max, sumexp) over its
//                      16-byte vocabulary tiles, merged in fixed order, R10) then loss =
//                      log S + M - x[label] and, fused with subroutine 2, the gradient
//                      scale * (e^{x - M} / S - onehot(label)) written over the logits
#include "nnt_internal.h"

namespace nnt {
namespace {

constexpr int kT = 256;

// ------------------------------------------------------------------ embedding forward
__global__ void __launch_bounds__(kT) embed_fwd_kernel(const int32_t* __restrict__ ids, int64_t T, int64_t S,
                                                       const float* __restrict__ wte, int64_t V,
                                                       const float* __restrict__ wpe, int E,
                                                       float* __restrict__ x) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kT / 32);
  for (int64_t t = (int64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); t < T; t += warps) {
    int64_t id = __ldg(ids + t);
    id = id < 0 ? 0 : (id >= V ? V - 1 : id);  // out-of-range ids are clamped (documented)
    const float4* a = reinterpret_cast<const float4*>(wte + id * E);
    const float4* b = reinterpret_cast<const float4*>(wpe + (t % S) * E);
    float4* o = reinterpret_cast<float4*>(x + t * E);
    for (int i = lane; i < E / 4; i += 32) {
      const float4 u = __ldg(a + i), w = __ldg(b + i);
      o[i] = make_float4(u.x + w.x, u.y + w.y, u.z + w.z, u.w + w.w);
    }
  }
}

// ------------------------------------------------------------------ embedding backward
// scratch layout (ints): hist[V + 1] | rank[T] | offs[V + 1] | order[T]
__global__ void __launch_bounds__(kT) embed_hist_kernel(const int32_t* __restrict__ ids, int64_t T, int64_t V,
                                                        int* __restrict__ hist) {
  NNT_PDL_ENTRY();
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < T; t += (int64_t)gridDim.x * kT) {
    int64_t id = ids[t];
    id = id < 0 ? 0 : (id >= V ? V - 1 : id);
    atomicAdd(hist + id, 1);  // integer counts: order-independent
  }
}

__global__ void __launch_bounds__(kT) zero_ints_kernel(int* __restrict__ p, int64_t n) {
  NNT_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) p[i] = 0;
}

// offs[v] = sum_{u < v} hist[u] for v < n (one CTA): the counts are staged in shared memory with
// coalesced loads, each thread scans a contiguous chunk there, the chunk sums are scanned
// across the CTA, and the offsets leave through shared memory with coalesced stores.
constexpr int kScanMax = 54 * 1024;  // ints staged in shared memory (216 KB, + 4 KB static)
__global__ void __launch_bounds__(1024) embed_scan_kernel(const int* __restrict__ hist, int64_t n,
                                                          int* __restrict__ offs) {
  NNT_PDL_ENTRY();
  extern __shared__ int buf[];  // [n]
  __shared__ int part[1024];
  for (int64_t i = threadIdx.x; i < n; i += 1024) buf[i] = hist[i];
  __syncthreads();
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
  int s = 0;
  for (int64_t i = b; i < e; ++i) s += buf[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // inclusive Hillis-Steele scan of the chunk sums
    const int v = threadIdx.x >= d ? part[threadIdx.x - d] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = b; i < e; ++i) {
    const int h = buf[i];
    buf[i] = run;
    run += h;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += 1024) offs[i] = buf[i];
}

// rank[t] = #{t' < t : ids[t'] == ids[t]} (stable position inside the id's bucket).  CTA (x, y)
// compares its kT tokens with the earlier tokens of chunk y (kRankChunk ids staged in shared
// memory) and adds its counts with integer atomics (order-independent, exact).
constexpr int kRankChunk = 1024;
__global__ void __launch_bounds__(kT) embed_rank_kernel(const int32_t* __restrict__ ids, int64_t T, int64_t V,
                                                        int* __restrict__ rank) {
  NNT_PDL_ENTRY();
  __shared__ int tile[kRankChunk];
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.y * kRankChunk;
  if (c0 >= (int64_t)blockIdx.x * kT + kT || c0 >= T) return;  // chunk entirely after this CTA's tokens
  for (int i = threadIdx.x; i < kRankChunk; i += kT) {
    const int64_t j = c0 + i;
    int64_t v = j < T ? ids[j] : -2;
    if (j < T) v = v < 0 ? 0 : (v >= V ? V - 1 : v);
    tile[i] = (int)v;
  }
  __syncthreads();
  if (t >= T) return;
  int64_t my = ids[t];
  my = my < 0 ? 0 : (my >= V ? V - 1 : my);
  const int64_t lim64 = t - c0 < kRankChunk ? t - c0 : kRankChunk;
  const int lim = lim64 > 0 ? (int)lim64 : 0;
  int r = 0;
  for (int k = 0; k < lim; ++k) r += tile[k] == (int)my;
  if (r) atomicAdd(rank + t, r);
}

__global__ void __launch_bounds__(kT) embed_place_kernel(const int32_t* __restrict__ ids, int64_t T, int64_t V,
                                                         const int* __restrict__ offs, const int* __restrict__ rank,
                                                         int* __restrict__ order) {
  NNT_PDL_ENTRY();
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < T; t += (int64_t)gridDim.x * kT) {
    int64_t my = ids[t];
    my = my < 0 ? 0 : (my >= V ? V - 1 : my);
    order[offs[my] + rank[t]] = (int)t;
  }
}

// dwte[v] (+)= sum over the bucket of v in token order; one warp per vocabulary row
__global__ void __launch_bounds__(kT) embed_bucket_kernel(const int* __restrict__ offs, const int* __restrict__ order,
                                                          const float* __restrict__ dx, int E, int64_t V,
                                                          float* __restrict__ dwte, int accumulate) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5);
  if (v >= V) return;
  const int b = offs[v], e = offs[v + 1];
  if (b == e && accumulate) return;
  float4* o = reinterpret_cast<float4*>(dwte + v * E);
  for (int i = lane; i < E / 4; i += 32) {
    float4 s = accumulate ? o[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = b; k < e; ++k) {
      const float4 d = __ldg(reinterpret_cast<const float4*>(dx + (int64_t)order[k] * E) + i);
      s.x += d.x; s.y += d.y; s.z += d.z; s.w += d.w;
    }
    o[i] = s;
  }
}

// dwpe[s] (+)= sum_b dx[b, s] (b ascending)
__global__ void __launch_bounds__(kT) embed_pos_kernel(const float* __restrict__ dx, int64_t B, int64_t S, int E,
                                                       float* __restrict__ dwpe, int accumulate) {
  NNT_PDL_ENTRY();
  const int64_t n4 = S * (E / 4);
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kT) {
    float4 s = accumulate ? reinterpret_cast<float4*>(dwpe)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t b = 0; b < B; ++b) {
      const float4 d = __ldg(reinterpret_cast<const float4*>(dx) + b * n4 + i);
      s.x += d.x; s.y += d.y; s.z += d.z; s.w += d.w;
    }
    reinterpret_cast<float4*>(dwpe)[i] = s;
  }
}

// ------------------------------------------------------------------ cross-entropy
template <typename T>
__device__ __forceinline__ void load8(const T* p, float* f);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);  // plain load: dlogits may alias the logits
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* f) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float* f);
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float* f) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 t = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&t);
  }
  *reinterpret_cast<uint4*>(p) = u;
}
template <>
__device__ __forceinline__ void store8<float>(float* p, const float* f) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}

// running (max, sumexp) merge of R10: (m,s) + (m',s') = (M, s e^{m-M} + s' e^{m'-M}); (-inf, 0) is the identity
__device__ __forceinline__ void mse_merge(float& m, float& s, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s = s2;
    return;
  }
  const float M = fmaxf(m, m2);
  s = s * __expf(m - M) + s2 * __expf(m2 - M);
  m = M;
}

// One CTA per row.  Thread i owns the 8-element vectors i, i + kT, ... of the row (and the
// scalar tail elements i, i + kT, ... beyond the last full vector).
template <typename T>
__global__ void __launch_bounds__(kT) cross_entropy_kernel(const T* logits, int64_t rows, int64_t V, int64_t ld,
                                                           const int32_t* __restrict__ labels, float scale,
                                                           float* __restrict__ loss_rows, float* __restrict__ stats,
                                                           T* dlogits, int64_t ld_d) {
  NNT_PDL_ENTRY();
  __shared__ float sm[kT], ss[kT];
  __shared__ float red_m, red_s;
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const T* x = logits + r * ld;
  const int64_t nv = V / 8;
  // subroutine 1: per-thread (max, sumexp) over its tiles, then the fixed-order merge
  float m = -INFINITY, s = 0.f;
  for (int64_t i = threadIdx.x; i < nv; i += kT) {
    float f[8];
    load8<T>(x + 8 * i, f);
    float tm = f[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) tm = fmaxf(tm, f[k]);
    float ts = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) ts += __expf(f[k] - tm);
    mse_merge(m, s, tm, ts);
  }
  for (int64_t k = 8 * nv + threadIdx.x; k < V; k += kT) mse_merge(m, s, to_f32(x[k]), 1.f);
  sm[threadIdx.x] = m;
  ss[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    for (int i = 0; i < kT; ++i) mse_merge(M, S, sm[i], ss[i]);  // ascending thread order
    red_m = M;
    red_s = S;
    int64_t c = labels[r];
    c = c < 0 ? 0 : (c >= V ? V - 1 : c);
    if (loss_rows) loss_rows[r] = logf(S) + M - to_f32(x[c]);
    if (stats) {
      stats[2 * r] = M;
      stats[2 * r + 1] = S;
    }
  }
  __syncthreads();
  if (dlogits == nullptr) return;
  // subroutine 2 fused with the gradient: scale * (e^{x - M} / S - onehot(label))
  const float M = red_m, inv = scale / red_s;
  int64_t c = labels[r];
  c = c < 0 ? 0 : (c >= V ? V - 1 : c);
  T* d = dlogits + r * ld_d;
  for (int64_t i = threadIdx.x; i < nv; i += kT) {
    float f[8];
    load8<T>(x + 8 * i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = __expf(f[k] - M) * inv - (8 * i + k == c ? scale : 0.f);
    store8<T>(d + 8 * i, f);
  }
  for (int64_t k = 8 * nv + threadIdx.x; k < V; k += kT)
    d[k] = from_f32<T>(__expf(to_f32(x[k]) - M) * inv - (k == c ? scale : 0.f));
}

inline int grid_cap(int64_t items, int per_cta) {
  int64_t g = (items + per_cta - 1) / per_cta;
  const int64_t cap = 8LL * num_sms();
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_embedding_fwd(const int32_t* ids, int64_t T, int64_t S, const float* wte, int64_t V,
                             const float* wpe, int64_t E, float* x, nnt_stream_t stream) {
  NNT_REQUIRE(ids && wte && wpe && x, NNT_ERR_NULL, "nnt_embedding_fwd: NULL pointer");
  NNT_REQUIRE(T > 0 && S > 0 && T % S == 0 && V > 0 && E > 0, NNT_ERR_SHAPE,
              "nnt_embedding_fwd: T=%lld S=%lld V=%lld E=%lld", (long long)T, (long long)S, (long long)V, (long long)E);
  NNT_REQUIRE(E % 4 == 0 && aligned16(wte) && aligned16(wpe) && aligned16(x), NNT_ERR_ALIGN,
              "nnt_embedding_fwd: E %% 4 and 16-byte alignment required");
  LaunchScope sc(NNT_K_MISC, stream, 12.0 * T * E + 4.0 * T, 0);
  NNT_CUDA_TRY(::nnt::launch(embed_fwd_kernel, dim3(grid_cap(T, kT / 32)), dim3(kT), 0, (cudaStream_t)stream, ids, T,
                             S, wte, V, wpe, (int)E, x));
  return NNT_OK;
}

size_t nnt_embedding_bwd_scratch_bytes(int64_t T, int64_t V) {
  if (T <= 0 || V <= 0) return 0;
  return (size_t)(2 * (V + 1) + 2 * T) * sizeof(int);
}

nnt_status nnt_embedding_bwd(const int32_t* ids, int64_t T, int64_t S, const float* dx, int64_t E, float* dwte,
                             int64_t V, float* dwpe, int accumulate, void* scratch, size_t scratch_bytes,
                             nnt_stream_t stream) {
  NNT_REQUIRE(ids && dx && dwte && dwpe && scratch, NNT_ERR_NULL, "nnt_embedding_bwd: NULL pointer");
  NNT_REQUIRE(T > 0 && S > 0 && T % S == 0 && V > 0 && E > 0 && T < (1ll << 31) && V < (1ll << 30), NNT_ERR_SHAPE,
              "nnt_embedding_bwd: T=%lld S=%lld V=%lld E=%lld", (long long)T, (long long)S, (long long)V, (long long)E);
  NNT_REQUIRE(E % 4 == 0 && aligned16(dx) && aligned16(dwte) && aligned16(dwpe), NNT_ERR_ALIGN,
              "nnt_embedding_bwd: E %% 4 and 16-byte alignment required");
  NNT_REQUIRE(scratch_bytes >= nnt_embedding_bwd_scratch_bytes(T, V), NNT_ERR_WORKSPACE,
              "nnt_embedding_bwd: scratch %zu < %zu", scratch_bytes, nnt_embedding_bwd_scratch_bytes(T, V));
  cudaStream_t s = (cudaStream_t)stream;
  int* hist = (int*)scratch;  // hist[V + 1] then rank[T] (zeroed together)
  int* rank = hist + (V + 1);
  int* offs = rank + T;
  int* order = offs + (V + 1);
  LaunchScope sc(NNT_K_MISC, s, 8.0 * T * E + 8.0 * V * 4 + 4.0 * V * E, 0, 7);
  static const size_t scan_smem = [] {
    cudaFuncSetAttribute(embed_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kScanMax * sizeof(int)));
    return (size_t)kScanMax * sizeof(int);
  }();
  NNT_REQUIRE(V + 1 <= kScanMax, NNT_ERR_UNSUPPORTED, "nnt_embedding_bwd: V=%lld > %d", (long long)V,
              kScanMax - 1);
  NNT_CUDA_TRY(::nnt::launch(zero_ints_kernel, dim3(grid_cap(V + 1 + T, kT)), dim3(kT), 0, s, hist, V + 1 + T));
  NNT_CUDA_TRY(::nnt::launch(embed_hist_kernel, dim3(grid_cap(T, kT)), dim3(kT), 0, s, ids, T, V, hist));
  NNT_CUDA_TRY(::nnt::launch(embed_scan_kernel, dim3(1), dim3(1024), (size_t)(V + 1) * sizeof(int), s,
                             (const int*)hist, V + 1, offs));
  (void)scan_smem;
  NNT_CUDA_TRY(::nnt::launch(embed_rank_kernel,
                             dim3((unsigned)((T + kT - 1) / kT), (unsigned)((T + kRankChunk - 1) / kRankChunk)),
                             dim3(kT), 0, s, ids, T, V, rank));
  NNT_CUDA_TRY(::nnt::launch(embed_place_kernel, dim3(grid_cap(T, kT)), dim3(kT), 0, s, ids, T, V,
                             (const int*)offs, (const int*)rank, order));
  NNT_CUDA_TRY(::nnt::launch(embed_bucket_kernel, dim3((unsigned)((V + kT / 32 - 1) / (kT / 32))), dim3(kT), 0, s,
                             (const int*)offs, (const int*)order, dx, (int)E, V, dwte, accumulate));
  NNT_CUDA_TRY(::nnt::launch(embed_pos_kernel, dim3(grid_cap(S * E / 4, kT)), dim3(kT), 0, s, dx, T / S, S, (int)E,
                             dwpe, accumulate));
  return NNT_OK;
}

nnt_status nnt_cross_entropy(const void* logits, int dtype, int64_t rows, int64_t V, int64_t ld,
                             const int32_t* labels, float scale, float* loss_rows, float* stats, void* dlogits,
                             int64_t ld_d, nnt_stream_t stream) {
  NNT_REQUIRE(logits && labels, NNT_ERR_NULL, "nnt_cross_entropy: NULL pointer");
  NNT_REQUIRE(rows > 0 && V > 0 && ld >= V && (!dlogits || ld_d >= V) && rows < (1ll << 31), NNT_ERR_SHAPE,
              "nnt_cross_entropy: rows=%lld V=%lld ld=%lld", (long long)rows, (long long)V, (long long)ld);
  NNT_REQUIRE(valid_dtype(dtype), NNT_ERR_DTYPE, "nnt_cross_entropy: dtype %d", dtype);
  const size_t es = dtype_size(dtype);
  NNT_REQUIRE(aligned16(logits) && (ld * es) % 16 == 0 && (!dlogits || (aligned16(dlogits) && (ld_d * es) % 16 == 0)),
              NNT_ERR_ALIGN, "nnt_cross_entropy: 16-byte aligned rows required");
  LaunchScope sc(NNT_K_SOFTMAX, stream, (double)rows * V * es * (dlogits ? 3.0 : 1.0) + 16.0 * rows, 0);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == NNT_BF16)
    NNT_CUDA_TRY(::nnt::launch(cross_entropy_kernel<__nv_bfloat16>, dim3((unsigned)rows), dim3(kT), 0, s,
                               (const __nv_bfloat16*)logits, rows, V, ld, labels, scale, loss_rows, stats,
                               (__nv_bfloat16*)dlogits, ld_d));
  else
    NNT_CUDA_TRY(::nnt::launch(cross_entropy_kernel<float>, dim3((unsigned)rows), dim3(kT), 0, s,
                               (const float*)logits, rows, V, ld, labels, scale, loss_rows, stats, (float*)dlogits,
                               ld_d));
  return NNT_OK;
}

}  // extern "C"
