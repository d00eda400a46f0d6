// GPT-2 shell: the embedding layer and the cross-entropy loss
// built from the two SoftMax subroutines.  The tied LM head itself is
// two nnt_tile_gemm calls made by the driver.
//
//   nnt_embedding_fwd  x[t] = wte[ids[t]] + wpe[t mod S]           (warp per token, float4)
//   nnt_embedding_bwd  dwte[v] (+)= sum of dx over the tokens with id v, in token order;
//                      dwpe[s] (+)= sum_b dx[b, s]
//                      deterministic without atomics on floats: a counting sort of the token
//                      positions by id (integer histogram, one-CTA exclusive scan; the bucket
//                      order from a sort of the unique (id, t) keys), then one warp per
//                      vocabulary row sums its bucket in token order
//   nnt_cross_entropy  per row: subroutine 1 (the row's (max, sumexp), R10) then loss =
//                      log S + M - x[label] and, fused with subroutine 2, the gradient
//                      scale * (e^{x - M} / S - onehot(label)) written over the logits.
//                      bf16 rows up to 104 KB: persistent CTAs, rows double-buffered in shared
//                      memory by cp.async.bulk (logits read from HBM once, written once);
//                      rows up to 200 KB: one CTA per row staged in shared memory; longer rows:
//                      the re-reading kernel (per-thread running (max, sumexp), fixed-order merge)
#include <cstdlib>

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
// scratch layout: hist[V + 1] | offs[V + 1] | order[T] (ints) | keys[2][T] (uint64, 8-byte aligned)
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

// The bucket order: the token positions sorted by the key (id, t) -- keys are unique, so ANY sort
// yields the one order "by id, then ascending t" (the stable counting sort's order) and
// order[p] = t of the p-th smallest key lands each token at offs[id] + (number of earlier tokens
// with its id).  A chunk of kSortChunk keys is bitonic-sorted in shared memory per CTA, then
// merge passes double the sorted run length (merge path: a key's output position is its index
// in its own run plus the number of smaller keys in the partner run, by binary search).
// O(T log^2 kSortChunk + T log T) work over all SMs.
constexpr int kSortChunk = 2048;
__device__ __forceinline__ uint64_t embed_key(const int32_t* ids, int64_t t, int64_t V) {
  int64_t v = ids[t];
  v = v < 0 ? 0 : (v >= V ? V - 1 : v);
  return ((uint64_t)v << 32) | (uint64_t)t;
}
__global__ void __launch_bounds__(1024) embed_sort_chunk_kernel(const int32_t* __restrict__ ids, int64_t T, int64_t V,
                                                                uint64_t* __restrict__ keys) {
  NNT_PDL_ENTRY();
  __shared__ uint64_t k[kSortChunk];
  const int64_t c0 = (int64_t)blockIdx.x * kSortChunk;
  for (int i = threadIdx.x; i < kSortChunk; i += 1024)
    k[i] = c0 + i < T ? embed_key(ids, c0 + i, V) : ~0ull;  // padding sorts last
  __syncthreads();
  for (int size = 2; size <= kSortChunk; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < kSortChunk / 2; i += 1024) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;  // the pair (lo, hi) of this step
        const bool up = (lo & size) == 0;
        const uint64_t a = k[lo], b = k[hi];
        if ((a > b) == up) {
          k[lo] = b;
          k[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kSortChunk; i += 1024)
    if (c0 + i < T) keys[c0 + i] = k[i];
}
// Merge the sorted runs [2jL, 2jL + L) and [2jL + L, 2(j+1)L) of src into dst (runs cut at T).
__global__ void __launch_bounds__(kT) embed_merge_kernel(const uint64_t* __restrict__ src, int64_t T, int64_t L,
                                                         uint64_t* __restrict__ dst) {
  NNT_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < T; i += (int64_t)gridDim.x * kT) {
    const int64_t base = i / (2 * L) * (2 * L);
    const bool first = i - base < L;
    const int64_t own0 = first ? base : base + L;
    const int64_t o0 = min(T, first ? base + L : base), o1 = min(T, o0 + L);  // the partner run (may be empty)
    const uint64_t key = src[i];
    int64_t lo = o0, hi = o1;  // count the partner's smaller keys (keys are unique)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (src[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    dst[base + (i - own0) + (lo - o0)] = key;
  }
}
__global__ void __launch_bounds__(kT) embed_order_kernel(const uint64_t* __restrict__ keys, int64_t T,
                                                         int* __restrict__ order) {
  NNT_PDL_ENTRY();
  for (int64_t p = (int64_t)blockIdx.x * kT + threadIdx.x; p < T; p += (int64_t)gridDim.x * kT)
    order[p] = (int)(keys[p] & 0xffffffffu);
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

// Row-staged variant (the product path for bf16 logits): one CTA per row copies the row's full
// 16-byte vectors into shared memory once while taking the row maximum, so the logits are read
// from HBM exactly once and written once (the re-reading kernel above touches them twice).
//   pass A  global -> smem, per-thread max, block max M (fixed xor-tree order)
//   pass B  S = sum_k e^{x_k - M} from smem (per-thread in vector order, then the fixed tree)
//   pass C  smem -> global: scale * (e^{x - M} / S - onehot(label))
// Subroutine 1's (max, sumexp) is thus taken as max first, then the sum relative to it — the
// same pair the running merge of R10 produces, with one exponential per element per pass.
constexpr int kCeT = 512;
constexpr size_t kCeSmemMax = 200 * 1024;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool kMax, int NT = kCeT>
__device__ __forceinline__ float ce_block_reduce(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, w) : v + w;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = lane < NT / 32 ? red[lane] : (kMax ? -INFINITY : 0.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, w) : v + w;
  }
  __syncthreads();  // red[] is reused by the next reduction
  return v;
}

template <typename T>
__global__ void __launch_bounds__(kCeT, 2)
    cross_entropy_staged_kernel(const T* logits, int64_t rows, int64_t V, int64_t ld,
                                const int32_t* __restrict__ labels, float scale, float* __restrict__ loss_rows,
                                float* __restrict__ stats, T* dlogits, int64_t ld_d) {
  NNT_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char ce_smem[];
  T* row = reinterpret_cast<T*>(ce_smem);
  __shared__ float red[kCeT / 32];
  __shared__ float tail[8];
  __shared__ float xlabel;
  const int64_t r = blockIdx.x;
  const T* x = logits + r * ld;
  const int nv = (int)(V / 8), ntail = (int)(V - 8 * (int64_t)nv);
  int64_t c = labels[r];
  c = c < 0 ? 0 : (c >= V ? V - 1 : c);
  // pass A: stage the row, running max (4 vectors in flight per thread)
  float m = -INFINITY;
  int i = threadIdx.x;
  for (; i + 3 * kCeT < nv; i += 4 * kCeT) {
    float f[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) load8<T>(x + 8 * (int64_t)(i + u * kCeT), f[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      store8<T>(row + 8 * (i + u * kCeT), f[u]);
#pragma unroll
      for (int k = 0; k < 8; ++k) m = fmaxf(m, f[u][k]);
    }
  }
  for (; i < nv; i += kCeT) {
    float f[8];
    load8<T>(x + 8 * (int64_t)i, f);
    store8<T>(row + 8 * i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) m = fmaxf(m, f[k]);
  }
  if (threadIdx.x < ntail) {
    const float t = to_f32(x[8 * (int64_t)nv + threadIdx.x]);
    tail[threadIdx.x] = t;
    m = fmaxf(m, t);
  }
  if (threadIdx.x == 0) xlabel = to_f32(x[c]);
  const float M = ce_block_reduce<true>(m, red);  // its barriers also publish row[], tail[], xlabel
  const float ML = M * kLog2e;
  // pass B: S = sum e^{x - M}
  float s = 0.f;
  for (int j = threadIdx.x; j < nv; j += kCeT) {
    float f[8];
    load8<T>(row + 8 * j, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += ex2f(fmaf(f[k], kLog2e, -ML));
  }
  if (threadIdx.x < ntail) s += ex2f(fmaf(tail[threadIdx.x], kLog2e, -ML));
  const float S = ce_block_reduce<false>(s, red);
  if (threadIdx.x == 0) {
    if (loss_rows) loss_rows[r] = logf(S) + M - xlabel;
    if (stats) {
      stats[2 * r] = M;
      stats[2 * r + 1] = S;
    }
  }
  if (dlogits == nullptr) return;
  // pass C: subroutine 2 fused with the gradient, written over the logits when they alias
  const float inv = scale / S;
  T* d = dlogits + r * ld_d;
  for (int j = threadIdx.x; j < nv; j += kCeT) {
    float f[8];
    load8<T>(row + 8 * j, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = ex2f(fmaf(f[k], kLog2e, -ML)) * inv;
    store8<T>(d + 8 * (int64_t)j, f);
  }
  if (c < 8 * (int64_t)nv && threadIdx.x == (int)((c >> 3) % kCeT))  // - onehot(label), same thread
    d[c] = from_f32<T>(ex2f(fmaf(xlabel, kLog2e, -ML)) * inv - scale);
  if (threadIdx.x < ntail) {
    const int64_t k = 8 * (int64_t)nv + threadIdx.x;
    d[k] = from_f32<T>(ex2f(fmaf(tail[threadIdx.x], kLog2e, -ML)) * inv - (k == c ? scale : 0.f));
  }
}

// Persistent, double-buffered variant (bf16 GPT-2 vocabulary: 2 x 100.5 KB rows per SM): one
// CTA per SM walks rows r = blockIdx.x + k * gridDim.x; while it runs the three passes over row
// k from shared memory, a bulk async copy (cp.async.bulk, completion on an mbarrier) brings row
// k + 1 into the other buffer, so the HBM read stream never waits for the exponentials.
// Same arithmetic as cross_entropy_staged_kernel, pass A reading the staged row.
constexpr int kCePT = 1024;
constexpr uint32_t kCeChunk = 32768;

__device__ __forceinline__ uint32_t ce_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ce_mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
// one thread: expect `bytes` on `bar`, then copy them global -> shared in kCeChunk pieces
__device__ __forceinline__ void ce_fetch_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of dst first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  for (uint32_t o = 0; o < bytes; o += kCeChunk) {
    const uint32_t n = bytes - o < kCeChunk ? bytes - o : kCeChunk;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst + o), "l"(reinterpret_cast<const char*>(src) + o), "r"(n), "r"(bar)
                 : "memory");
  }
}

template <typename T>
__global__ void __launch_bounds__(kCePT, 1)
    cross_entropy_pipe_kernel(const T* logits, int64_t rows, int64_t V, int64_t ld,
                              const int32_t* __restrict__ labels, float scale, float* __restrict__ loss_rows,
                              float* __restrict__ stats, T* dlogits, int64_t ld_d) {
  NNT_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char ce_smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ float red[kCePT / 32];
  const int nv = (int)(V / 8), ntail = (int)(V - 8 * (int64_t)nv);
  const uint32_t row_bytes = (uint32_t)nv * 8u * (uint32_t)sizeof(T);
  const uint32_t buf0 = ce_smem_u32(ce_smem);
  const uint32_t bar0 = ce_smem_u32(&bar[0]), bar1 = ce_smem_u32(&bar[1]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (row_bytes && (int64_t)blockIdx.x < rows)
      ce_fetch_row(buf0, logits + (int64_t)blockIdx.x * ld, row_bytes, bar0);
  }
  __syncthreads();
  int k = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++k) {
    const int b = k & 1;
    // every thread is past row k-1's pass C (its last read of buf[b^1]): refill that buffer
    if (threadIdx.x == 0 && row_bytes && r + gridDim.x < rows)
      ce_fetch_row(buf0 + (uint32_t)(b ^ 1) * row_bytes, logits + (r + gridDim.x) * ld, row_bytes, b ? bar0 : bar1);
    const T* x = logits + r * ld;
    int64_t c = labels[r];
    c = c < 0 ? 0 : (c >= V ? V - 1 : c);
    const float xc = to_f32(x[c]);  // read before this row's pass C may overwrite it
    const float xt = threadIdx.x < ntail ? to_f32(x[8 * (int64_t)nv + threadIdx.x]) : -INFINITY;
    if (row_bytes) ce_mbar_wait(b ? bar1 : bar0, (uint32_t)(k >> 1) & 1u);
    const T* row = reinterpret_cast<const T*>(ce_smem + (size_t)b * row_bytes);
    // pass A: max
    float m = xt;
    for (int j = threadIdx.x; j < nv; j += kCePT) {
      float f[8];
      load8<T>(row + 8 * j, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) m = fmaxf(m, f[q]);
    }
    const float M = ce_block_reduce<true, kCePT>(m, red);
    const float ML = M * kLog2e;
    // pass B: S = sum e^{x - M}
    float sum = threadIdx.x < ntail ? ex2f(fmaf(xt, kLog2e, -ML)) : 0.f;
    for (int j = threadIdx.x; j < nv; j += kCePT) {
      float f[8];
      load8<T>(row + 8 * j, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) sum += ex2f(fmaf(f[q], kLog2e, -ML));
    }
    const float S = ce_block_reduce<false, kCePT>(sum, red);
    if (threadIdx.x == 0) {
      if (loss_rows) loss_rows[r] = logf(S) + M - xc;
      if (stats) {
        stats[2 * r] = M;
        stats[2 * r + 1] = S;
      }
    }
    if (dlogits != nullptr) {
      // pass C: subroutine 2 fused with the gradient
      const float inv = scale / S;
      T* d = dlogits + r * ld_d;
      for (int j = threadIdx.x; j < nv; j += kCePT) {
        float f[8];
        load8<T>(row + 8 * j, f);
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = ex2f(fmaf(f[q], kLog2e, -ML)) * inv;
        store8<T>(d + 8 * (int64_t)j, f);
      }
      // - onehot(label): the thread that stored the label's vector rewrites that one element
      if (c < 8 * (int64_t)nv && threadIdx.x == (int)((c >> 3) % kCePT))
        d[c] = from_f32<T>(ex2f(fmaf(xc, kLog2e, -ML)) * inv - scale);
      if (threadIdx.x < ntail) {
        const int64_t q = 8 * (int64_t)nv + threadIdx.x;
        d[q] = from_f32<T>(ex2f(fmaf(xt, kLog2e, -ML)) * inv - (q == c ? scale : 0.f));
      }
    }
    __syncthreads();  // buf[b] is refilled at the top of iteration k + 1
  }
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
  const size_t ints = (size_t)(2 * (V + 1) + T);
  return (ints * sizeof(int) + 7) / 8 * 8 + (size_t)2 * T * sizeof(uint64_t);
}

nnt_status nnt_embedding_bwd(const int32_t* ids, int64_t T, int64_t S, const float* dx, int64_t E, float* dwte,
                             int64_t V, float* dwpe, int accumulate_wte, int accumulate_wpe, void* scratch,
                             size_t scratch_bytes, nnt_stream_t stream) {
  NNT_REQUIRE(ids && dx && dwte && dwpe && scratch, NNT_ERR_NULL, "nnt_embedding_bwd: NULL pointer");
  NNT_REQUIRE(T > 0 && S > 0 && T % S == 0 && V > 0 && E > 0 && T < (1ll << 31) && V < (1ll << 30), NNT_ERR_SHAPE,
              "nnt_embedding_bwd: T=%lld S=%lld V=%lld E=%lld", (long long)T, (long long)S, (long long)V, (long long)E);
  NNT_REQUIRE(E % 4 == 0 && aligned16(dx) && aligned16(dwte) && aligned16(dwpe), NNT_ERR_ALIGN,
              "nnt_embedding_bwd: E %% 4 and 16-byte alignment required");
  NNT_REQUIRE(scratch_bytes >= nnt_embedding_bwd_scratch_bytes(T, V), NNT_ERR_WORKSPACE,
              "nnt_embedding_bwd: scratch %zu < %zu", scratch_bytes, nnt_embedding_bwd_scratch_bytes(T, V));
  cudaStream_t s = (cudaStream_t)stream;
  int* hist = (int*)scratch;
  int* offs = hist + (V + 1);
  int* order = offs + (V + 1);
  uint64_t* keys = reinterpret_cast<uint64_t*>(scratch) + ((2 * (V + 1) + T) * sizeof(int) + 7) / 8;
  uint64_t* keys2 = keys + T;
  LaunchScope sc(NNT_K_MISC, s, 8.0 * T * E + 8.0 * V * 4 + 4.0 * V * E, 0, 7);
  NNT_CUDA_TRY(set_max_dyn_smem(embed_scan_kernel, (int)(kScanMax * sizeof(int))));
  NNT_REQUIRE(V + 1 <= kScanMax, NNT_ERR_UNSUPPORTED, "nnt_embedding_bwd: V=%lld > %d", (long long)V,
              kScanMax - 1);
  NNT_REQUIRE(aligned16(scratch), NNT_ERR_ALIGN, "nnt_embedding_bwd: scratch must be 16-byte aligned");
  NNT_CUDA_TRY(::nnt::launch(zero_ints_kernel, dim3(grid_cap(V + 1, kT)), dim3(kT), 0, s, hist, V + 1));
  NNT_CUDA_TRY(::nnt::launch(embed_hist_kernel, dim3(grid_cap(T, kT)), dim3(kT), 0, s, ids, T, V, hist));
  NNT_CUDA_TRY(::nnt::launch(embed_scan_kernel, dim3(1), dim3(1024), (size_t)(V + 1) * sizeof(int), s,
                             (const int*)hist, V + 1, offs));
  NNT_CUDA_TRY(::nnt::launch(embed_sort_chunk_kernel, dim3((unsigned)((T + kSortChunk - 1) / kSortChunk)), dim3(1024),
                             0, s, ids, T, V, keys));
  for (int64_t L = kSortChunk; L < T; L *= 2) {
    NNT_CUDA_TRY(::nnt::launch(embed_merge_kernel, dim3(grid_cap(T, kT)), dim3(kT), 0, s, (const uint64_t*)keys, T, L,
                               keys2));
    uint64_t* tmp = keys;
    keys = keys2;
    keys2 = tmp;
    sc.add_kernels(1);
  }
  NNT_CUDA_TRY(::nnt::launch(embed_order_kernel, dim3(grid_cap(T, kT)), dim3(kT), 0, s, (const uint64_t*)keys, T,
                             order));
  NNT_CUDA_TRY(::nnt::launch(embed_bucket_kernel, dim3((unsigned)((V + kT / 32 - 1) / (kT / 32))), dim3(kT), 0, s,
                             (const int*)offs, (const int*)order, dx, (int)E, V, dwte, accumulate_wte));
  NNT_CUDA_TRY(::nnt::launch(embed_pos_kernel, dim3(grid_cap(S * E / 4, kT)), dim3(kT), 0, s, dx, T / S, S, (int)E,
                             dwpe, accumulate_wpe));
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
  // algorithmic bytes: the logits read once, the gradient written once (whatever the kernel re-reads)
  LaunchScope sc(NNT_K_SOFTMAX, stream, (double)rows * V * es * (dlogits ? 2.0 : 1.0) + 16.0 * rows, 0);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t row_bytes = (size_t)(V / 8) * 8 * es;
  static const bool restream = [] {  // NNT_CE_RESTREAM=1: the two-read kernel (A/B runs)
    const char* e = getenv("NNT_CE_RESTREAM");
    return e && e[0] == '1';
  }();
  if (2 * row_bytes <= kCeSmemMax + 8192 && dtype == NNT_BF16 && !restream) {
    NNT_CUDA_TRY(set_max_dyn_smem(cross_entropy_pipe_kernel<__nv_bfloat16>, (int)(kCeSmemMax + 8192)));
    const int64_t grid = rows < num_sms() ? rows : num_sms();
    NNT_CUDA_TRY(::nnt::launch(cross_entropy_pipe_kernel<__nv_bfloat16>, dim3((unsigned)grid), dim3(kCePT),
                               2 * row_bytes, s, (const __nv_bfloat16*)logits, rows, V, ld, labels, scale, loss_rows,
                               stats, (__nv_bfloat16*)dlogits, ld_d));
    return NNT_OK;
  }
  if (row_bytes <= kCeSmemMax && !restream) {
    if (dtype == NNT_BF16) {
      NNT_CUDA_TRY(set_max_dyn_smem(cross_entropy_staged_kernel<__nv_bfloat16>, (int)kCeSmemMax));
      NNT_CUDA_TRY(::nnt::launch(cross_entropy_staged_kernel<__nv_bfloat16>, dim3((unsigned)rows), dim3(kCeT),
                                 row_bytes, s, (const __nv_bfloat16*)logits, rows, V, ld, labels, scale, loss_rows,
                                 stats, (__nv_bfloat16*)dlogits, ld_d));
    } else {
      NNT_CUDA_TRY(set_max_dyn_smem(cross_entropy_staged_kernel<float>, (int)kCeSmemMax));
      NNT_CUDA_TRY(::nnt::launch(cross_entropy_staged_kernel<float>, dim3((unsigned)rows), dim3(kCeT), row_bytes, s,
                                 (const float*)logits, rows, V, ld, labels, scale, loss_rows, stats, (float*)dlogits,
                                 ld_d));
    }
    return NNT_OK;
  }
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
