// Elementwise / streaming kernels: GELU fwd/bwd, Adam,
// bias-gradient column sums, dtype conversion and the probe-loss dot product.
// All are HBM-bound: 128-bit vector access, grid-stride loops sized in
// multiples of the SM count, deterministic (ordered) reductions, no atomics.
#include "reduce.cuh"

namespace nnt {
namespace {

constexpr int kThreads = 256;
constexpr int kPartitionSMs = 148;  // fixed so workspace sizes do not depend on the device

inline int grid_for(int64_t work_items, int per_sm = 8) {
  int64_t g = (work_items + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ------------------------------------------------------------------ GELU
template <typename T, bool kBwd>
__global__ void __launch_bounds__(kThreads) gelu_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                        T* __restrict__ y, int64_t n, bool vec_ok) {
  NNT_PDL_ENTRY();
  constexpr int V = 16 / sizeof(T);
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t nv = vec_ok ? n / V : 0;
  for (int64_t i = tid; i < nv; i += stride) {
    uint4 xv = reinterpret_cast<const uint4*>(x)[i];
    uint4 dv;
    if (kBwd) dv = reinterpret_cast<const uint4*>(dy)[i];
    const T* xe = reinterpret_cast<const T*>(&xv);
    const T* de = reinterpret_cast<const T*>(&dv);
    uint4 ov;
    T* oe = reinterpret_cast<T*>(&ov);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float u = to_f32(xe[j]);
      float r = kBwd ? to_f32(de[j]) * gelu_grad_f(u) : gelu_f(u);
      oe[j] = from_f32<T>(r);
    }
    reinterpret_cast<uint4*>(y)[i] = ov;
  }
  for (int64_t i = nv * V + tid; i < n; i += stride) {
    float u = to_f32(x[i]);
    float r = kBwd ? to_f32(dy[i]) * gelu_grad_f(u) : gelu_f(u);
    y[i] = from_f32<T>(r);
  }
}

// ------------------------------------------------------------------ Adam
__global__ void __launch_bounds__(kThreads) adam_kernel(int64_t n, float* __restrict__ w,
                                                        const float* __restrict__ g, float* __restrict__ m,
                                                        float* __restrict__ v, __nv_bfloat16* __restrict__ w16,
                                                        nnt_adam_hparams hp, bool vec_ok) {
  NNT_PDL_ENTRY();
  const float b1 = hp.beta1, b2 = hp.beta2;
  const float c1 = hp.one_minus_beta1 != 0.f ? hp.one_minus_beta1 : 1.f - hp.beta1;
  const float c2 = hp.one_minus_beta2 != 0.f ? hp.one_minus_beta2 : 1.f - hp.beta2;
  const float bc1 = hp.bias_corr_dev ? __ldg(hp.bias_corr_dev) : hp.bias_corr1;
  const float bc2 = hp.bias_corr_dev ? __ldg(hp.bias_corr_dev + 1) : hp.bias_corr2;
  const float inv_bc1 = 1.f / bc1, inv_bc2 = 1.f / bc2;
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float lr_wd = -hp.lr * hp.weight_decay;
  // explicit roundings / FMAs: the vector and scalar loops (and any alignment of a range)
  // give bitwise the same update
  auto upd = [&](float& wi, float gi, float& mi, float& vi) {
    gi = __fmul_rn(gi, hp.grad_scale);
    mi = fmaf(b1, mi, __fmul_rn(c1, gi));
    vi = fmaf(b2, vi, __fmul_rn(__fmul_rn(c2, gi), gi));
    const float mhat = __fmul_rn(mi, inv_bc1);
    const float vhat = __fmul_rn(vi, inv_bc2);
    const float wold = wi;
    wi = __fsub_rn(wi, __fdiv_rn(__fmul_rn(hp.lr, mhat), __fadd_rn(sqrtf(vhat), hp.eps)));
    if (hp.weight_decay != 0.f) wi = fmaf(lr_wd, wold, wi);
  };
  int64_t nv = vec_ok ? n / 4 : 0;
  for (int64_t i = tid; i < nv; i += stride) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 mv = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    upd(wv.x, gv.x, mv.x, vv.x);
    upd(wv.y, gv.y, mv.y, vv.y);
    upd(wv.z, gv.z, mv.z, vv.z);
    upd(wv.w, gv.w, mv.w, vv.w);
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (w16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(wv.z, wv.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(w16)[i] = pk;
    }
  }
  for (int64_t i = nv * 4 + tid; i < n; i += stride) {
    float wi = w[i], mi = m[i], vi = v[i];
    upd(wi, g[i], mi, vi);
    w[i] = wi;
    m[i] = mi;
    v[i] = vi;
    if (w16) w16[i] = __float2bfloat16_rn(wi);
  }
}

__global__ void __launch_bounds__(kThreads) sgd_kernel(int64_t n, float* __restrict__ w,
                                                       const float* __restrict__ g, float* __restrict__ buf,
                                                       __nv_bfloat16* __restrict__ w16, float lr, float mom, float wd,
                                                       bool vec_ok) {
  NNT_PDL_ENTRY();
  auto upd = [&](float& wi, float gi, float& bi) {
    const float d = wd != 0.f ? fmaf(wd, wi, gi) : gi;
    bi = fmaf(mom, bi, d);
    wi = fmaf(-lr, bi, wi);
  };
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = vec_ok ? n / 4 : 0;
  for (int64_t i = tid; i < nv; i += stride) {
    float4 wv = reinterpret_cast<float4*>(w)[i], bv = reinterpret_cast<float4*>(buf)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    upd(wv.x, gv.x, bv.x);
    upd(wv.y, gv.y, bv.y);
    upd(wv.z, gv.z, bv.z);
    upd(wv.w, gv.w, bv.w);
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(buf)[i] = bv;
    if (w16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y), hi = __floats2bfloat162_rn(wv.z, wv.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(w16)[i] = pk;
    }
  }
  for (int64_t i = nv * 4 + tid; i < n; i += stride) {
    float wi = w[i], bi = buf[i];
    upd(wi, g[i], bi);
    w[i] = wi;
    buf[i] = bi;
    if (w16) w16[i] = __float2bfloat16_rn(wi);
  }
}

__global__ void adam_tick_kernel(double beta1, double beta2, int64_t* t, float* bc) {
  NNT_PDL_ENTRY();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t s = t[0] + 1;
    t[0] = s;
    bc[0] = (float)(1.0 - pow(beta1, (double)s));
    bc[1] = (float)(1.0 - pow(beta2, (double)s));
  }
}

// ------------------------------------------------------------------ convert
template <typename TI, typename TO>
__global__ void __launch_bounds__(kThreads) convert_kernel(const TI* __restrict__ x, TO* __restrict__ y, int64_t n) {
  NNT_PDL_ENTRY();
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) y[i] = from_f32<TO>(to_f32(x[i]));
}

__global__ void __launch_bounds__(kThreads) scale_kernel(const float* x, float alpha, float* y, int64_t n, bool vec_ok) {
  NNT_PDL_ENTRY();
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t nv = vec_ok ? n / 4 : 0;
  for (int64_t i = tid; i < nv; i += stride) {
    float4 v = reinterpret_cast<const float4*>(x)[i];
    reinterpret_cast<float4*>(y)[i] = make_float4(alpha * v.x, alpha * v.y, alpha * v.z, alpha * v.w);
  }
  for (int64_t i = nv * 4 + tid; i < n; i += stride) y[i] = alpha * x[i];
}

// ------------------------------------------------------------------ bias grad
// Column partial sums over row chunks: block (strip, chunk) sums rows
// [chunk*rows_per, ...) of a 128-column strip (lane -> 4 columns, 8 warps stride
// over rows), reduces warps in fixed order, writes partial[chunk][col].
struct ColsumPlan {
  int64_t chunks, rows_per;
};
inline ColsumPlan colsum_plan(int64_t T, int64_t N) {
  int64_t strips = (N + 127) / 128;
  int64_t want = (4 * kPartitionSMs + strips - 1) / strips;
  int64_t chunks = want;
  int64_t max_chunks = (T + 31) / 32;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  int64_t rows_per = (T + chunks - 1) / chunks;
  chunks = (T + rows_per - 1) / rows_per;
  return {chunks, rows_per};
}

__device__ __forceinline__ float4 load4f(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 load4f(const __nv_bfloat16* p) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads) colsum_partial_kernel(const T* __restrict__ dy, int64_t T_, int64_t N,
                                                                  int64_t ld, int64_t rows_per,
                                                                  float* __restrict__ partial,
                                                                  __nv_bfloat16* __restrict__ copy16) {
  NNT_PDL_ENTRY();
  __shared__ float red[8][128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col0 = (int64_t)blockIdx.x * 128 + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  int64_t r1 = r0 + rows_per;
  if (r1 > T_) r1 = T_;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (VEC) {
    if (col0 < N) {
#pragma unroll 4
      for (int64_t r = r0 + warp; r < r1; r += 8) {
        float4 v = load4f(dy + r * ld + col0);
        acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
        if (copy16) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(copy16 + r * ld + col0) = pk;
        }
      }
    }
  } else {
    for (int64_t r = r0 + warp; r < r1; r += 8) {
      const T* row = dy + r * ld;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t c = col0 + j;
        if (c < N) {
          float v = to_f32(row[c]);
          acc[j] += v;
          if (copy16) copy16[r * ld + c] = __float2bfloat16_rn(v);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[warp][lane * 4 + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 128) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    int64_t c = (int64_t)blockIdx.x * 128 + threadIdx.x;
    if (c < N) partial[(int64_t)blockIdx.y * N + c] = s;
  }
}

// ------------------------------------------------------------------ dot
constexpr int kDotBlocks = 2 * kPartitionSMs;
__global__ void __launch_bounds__(kThreads) dot_partial_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                               int64_t n, double* __restrict__ partial) {
  NNT_PDL_ENTRY();
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (double)a[i] * (double)b[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// one warp: lane l sums partials l, l + 32, ... in order, then a fixed xor tree (was one thread
// walking all 2 x 148 partials: a dependent chain of loads and fp64 adds, ~15 us)
__global__ void dot_merge_kernel(const double* __restrict__ partial, int n, float scale, float* out) {
  NNT_PDL_ENTRY();
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) t += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) out[0] = (float)(t * (double)scale);
}

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_gelu_fwd(const void* x, void* y, int dtype, int64_t n, nnt_stream_t stream) {
  NNT_REQUIRE(x && y, NNT_ERR_NULL, "nnt_gelu_fwd: NULL pointer");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_gelu_fwd: n=%lld", (long long)n);
  NNT_REQUIRE(valid_dtype(dtype), NNT_ERR_DTYPE, "nnt_gelu_fwd: dtype %d", dtype);
  if (n == 0) return NNT_OK;
  bool vec = aligned16(x) && aligned16(y);
  size_t es = dtype_size(dtype);
  LaunchScope sc(NNT_K_GELU, stream, 2.0 * es * n, 0);
  if (dtype == NNT_F32)
    ::nnt::launch(gelu_kernel<float, false>, grid_for(n / 4 + 1), kThreads, 0, stream, (const float*)x, nullptr, (float*)y, n, vec);
  else
    ::nnt::launch(gelu_kernel<__nv_bfloat16, false>, grid_for(n / 8 + 1), kThreads, 0, stream, 
        (const __nv_bfloat16*)x, nullptr, (__nv_bfloat16*)y, n, vec);
  return check_launch("gelu_fwd");
}

nnt_status nnt_gelu_bwd(const void* x, const void* dy, void* dx, int dtype, int64_t n, nnt_stream_t stream) {
  NNT_REQUIRE(x && dy && dx, NNT_ERR_NULL, "nnt_gelu_bwd: NULL pointer");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_gelu_bwd: n=%lld", (long long)n);
  NNT_REQUIRE(valid_dtype(dtype), NNT_ERR_DTYPE, "nnt_gelu_bwd: dtype %d", dtype);
  if (n == 0) return NNT_OK;
  bool vec = aligned16(x) && aligned16(dy) && aligned16(dx);
  size_t es = dtype_size(dtype);
  LaunchScope sc(NNT_K_GELU, stream, 3.0 * es * n, 0);
  if (dtype == NNT_F32)
    ::nnt::launch(gelu_kernel<float, true>, grid_for(n / 4 + 1), kThreads, 0, stream, (const float*)x, (const float*)dy,
                                                                          (float*)dx, n, vec);
  else
    ::nnt::launch(gelu_kernel<__nv_bfloat16, true>, grid_for(n / 8 + 1), kThreads, 0, stream, 
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (__nv_bfloat16*)dx, n, vec);
  return check_launch("gelu_bwd");
}

nnt_status nnt_adam_step(int64_t n, float* w, const float* g, float* m, float* v, void* w_bf16,
                         const nnt_adam_hparams* hp, nnt_stream_t stream) {
  NNT_REQUIRE(w && g && m && v && hp, NNT_ERR_NULL, "nnt_adam_step: NULL pointer");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_adam_step: n=%lld", (long long)n);
  NNT_REQUIRE(hp->bias_corr_dev || (hp->bias_corr1 > 0.f && hp->bias_corr2 > 0.f), NNT_ERR_ARG,
              "nnt_adam_step: bias corrections must be > 0 (t >= 1)");
  if (n == 0) return NNT_OK;
  bool vec = aligned16(w) && aligned16(g) && aligned16(m) && aligned16(v) &&
             (w_bf16 == nullptr || (reinterpret_cast<uintptr_t>(w_bf16) & 7u) == 0);
  LaunchScope sc(NNT_K_ADAM, stream, (28.0 + (w_bf16 ? 2.0 : 0.0)) * n, 0);
  ::nnt::launch(adam_kernel, grid_for(n / 4 + 1), kThreads, 0, stream, n, w, g, m, v, (__nv_bfloat16*)w_bf16, *hp, vec);
  return check_launch("adam");
}

nnt_status nnt_sgd_step(int64_t n, float* w, const float* g, float* buf, void* w_bf16, float lr, float momentum,
                        float weight_decay, nnt_stream_t stream) {
  NNT_REQUIRE(w && g && buf, NNT_ERR_NULL, "nnt_sgd_step: NULL pointer");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_sgd_step: n=%lld", (long long)n);
  if (n == 0) return NNT_OK;
  const bool vec = aligned16(w) && aligned16(g) && aligned16(buf) &&
                   (w_bf16 == nullptr || (reinterpret_cast<uintptr_t>(w_bf16) & 7u) == 0);
  LaunchScope sc(NNT_K_ADAM, stream, (20.0 + (w_bf16 ? 2.0 : 0.0)) * n, 0);
  ::nnt::launch(sgd_kernel, grid_for(n / 4 + 1), kThreads, 0, stream, n, w, g, buf, (__nv_bfloat16*)w_bf16, lr,
                momentum, weight_decay, vec);
  return check_launch("sgd");
}

nnt_status nnt_adam_tick(double beta1, double beta2, int64_t* t_dev, float* bias_corr_dev, nnt_stream_t stream) {
  NNT_REQUIRE(t_dev && bias_corr_dev, NNT_ERR_NULL, "nnt_adam_tick: NULL pointer");
  NNT_REQUIRE(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0, NNT_ERR_ARG, "nnt_adam_tick: beta");
  LaunchScope sc(NNT_K_ADAM, stream, 16.0, 0);
  ::nnt::launch(adam_tick_kernel, 1, 32, 0, stream, beta1, beta2, t_dev, bias_corr_dev);
  return check_launch("adam_tick");
}

nnt_status nnt_convert(const void* x, int x_dtype, void* y, int y_dtype, int64_t n, nnt_stream_t stream) {
  NNT_REQUIRE(x && y, NNT_ERR_NULL, "nnt_convert: NULL pointer");
  NNT_REQUIRE(valid_dtype(x_dtype) && valid_dtype(y_dtype), NNT_ERR_DTYPE, "nnt_convert: dtype");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_convert: n=%lld", (long long)n);
  if (n == 0) return NNT_OK;
  LaunchScope sc(NNT_K_MISC, stream, (double)(dtype_size(x_dtype) + dtype_size(y_dtype)) * n, 0);
  int grid = grid_for(n);
  if (x_dtype == NNT_F32 && y_dtype == NNT_BF16)
    ::nnt::launch(convert_kernel<float, __nv_bfloat16>, grid, kThreads, 0, stream, (const float*)x, (__nv_bfloat16*)y, n);
  else if (x_dtype == NNT_BF16 && y_dtype == NNT_F32)
    ::nnt::launch(convert_kernel<__nv_bfloat16, float>, grid, kThreads, 0, stream, (const __nv_bfloat16*)x, (float*)y, n);
  else if (x_dtype == NNT_F32)
    ::nnt::launch(convert_kernel<float, float>, grid, kThreads, 0, stream, (const float*)x, (float*)y, n);
  else
    ::nnt::launch(convert_kernel<__nv_bfloat16, __nv_bfloat16>, grid, kThreads, 0, stream, (const __nv_bfloat16*)x,
                                                                                  (__nv_bfloat16*)y, n);
  return check_launch("convert");
}

nnt_status nnt_scale(const float* x, float alpha, float* y, int64_t n, nnt_stream_t stream) {
  NNT_REQUIRE(x && y, NNT_ERR_NULL, "nnt_scale: NULL pointer");
  NNT_REQUIRE(n >= 0, NNT_ERR_SHAPE, "nnt_scale: n=%lld", (long long)n);
  if (n == 0) return NNT_OK;
  LaunchScope sc(NNT_K_MISC, stream, 8.0 * n, (double)n);
  ::nnt::launch(scale_kernel, grid_for(n / 4 + 1), kThreads, 0, stream, x, alpha, y, n, aligned16(x) && aligned16(y));
  return check_launch("scale");
}

size_t nnt_bias_grad_scratch_bytes(int64_t T, int64_t N) {
  if (T <= 0 || N <= 0) return 0;
  ColsumPlan p = colsum_plan(T, N);
  return (size_t)p.chunks * (size_t)N * sizeof(float);
}

nnt_status nnt_bias_grad(const void* dy, int dy_dtype, int64_t T, int64_t N, int64_t lddy, float* db,
                         int accumulate, void* dy_bf16_out, void* scratch, size_t scratch_bytes,
                         nnt_stream_t stream) {
  NNT_REQUIRE(dy && db && scratch, NNT_ERR_NULL, "nnt_bias_grad: NULL pointer");
  NNT_REQUIRE(T > 0 && N > 0 && lddy >= N, NNT_ERR_SHAPE, "nnt_bias_grad: T=%lld N=%lld ld=%lld",
              (long long)T, (long long)N, (long long)lddy);
  NNT_REQUIRE(valid_dtype(dy_dtype), NNT_ERR_DTYPE, "nnt_bias_grad: dtype %d", dy_dtype);
  NNT_REQUIRE(dy_bf16_out == nullptr || dy_dtype == NNT_F32, NNT_ERR_DTYPE,
              "nnt_bias_grad: bf16 copy requires fp32 dy");
  NNT_REQUIRE(scratch_bytes >= nnt_bias_grad_scratch_bytes(T, N), NNT_ERR_WORKSPACE,
              "nnt_bias_grad: scratch %zu < %zu", scratch_bytes, nnt_bias_grad_scratch_bytes(T, N));
  ColsumPlan p = colsum_plan(T, N);
  double bytes = (double)T * N * dtype_size(dy_dtype) + (dy_bf16_out ? 2.0 * T * N : 0.0) + 4.0 * N;
  LaunchScope sc(NNT_K_BIAS_GRAD, stream, bytes, 0, 2);
  dim3 grid((unsigned)((N + 127) / 128), (unsigned)p.chunks);
  const size_t es = dtype_size(dy_dtype);
  const bool vec = N % 4 == 0 && lddy % 4 == 0 && (reinterpret_cast<uintptr_t>(dy) % (4 * es)) == 0 &&
                   (!dy_bf16_out || (reinterpret_cast<uintptr_t>(dy_bf16_out) & 7u) == 0);
  __nv_bfloat16* c16 = (__nv_bfloat16*)dy_bf16_out;
  if (dy_dtype == NNT_F32) {
    if (vec)
      ::nnt::launch(colsum_partial_kernel<float, true>, grid, kThreads, 0, stream, (const float*)dy, T, N, lddy, p.rows_per,
                                                                        (float*)scratch, c16);
    else
      ::nnt::launch(colsum_partial_kernel<float, false>, grid, kThreads, 0, stream, (const float*)dy, T, N, lddy, p.rows_per,
                                                                         (float*)scratch, c16);
  } else {
    if (vec)
      ::nnt::launch(colsum_partial_kernel<__nv_bfloat16, true>, grid, kThreads, 0, stream, 
          (const __nv_bfloat16*)dy, T, N, lddy, p.rows_per, (float*)scratch, nullptr);
    else
      ::nnt::launch(colsum_partial_kernel<__nv_bfloat16, false>, grid, kThreads, 0, stream, 
          (const __nv_bfloat16*)dy, T, N, lddy, p.rows_per, (float*)scratch, nullptr);
  }
  NNT_TRY(check_launch("bias_grad partial"));
  launch_column_merge((const float*)scratch, p.chunks, N, db, accumulate, stream);
  return check_launch("bias_grad merge");
}

size_t nnt_dot_scratch_bytes(int64_t n) { return (size_t)kDotBlocks * sizeof(double); }

nnt_status nnt_dot(const float* y, const float* r, int64_t n, float scale, float* out, void* scratch,
                   size_t scratch_bytes, nnt_stream_t stream) {
  NNT_REQUIRE(y && r && out && scratch, NNT_ERR_NULL, "nnt_dot: NULL pointer");
  NNT_REQUIRE(n > 0, NNT_ERR_SHAPE, "nnt_dot: n=%lld", (long long)n);
  NNT_REQUIRE(scratch_bytes >= nnt_dot_scratch_bytes(n), NNT_ERR_WORKSPACE, "nnt_dot: scratch too small");
  LaunchScope sc(NNT_K_MISC, stream, 8.0 * n, 2.0 * n, 2);
  ::nnt::launch(dot_partial_kernel, kDotBlocks, kThreads, 0, stream, y, r, n, (double*)scratch);
  NNT_TRY(check_launch("dot partial"));
  ::nnt::launch(dot_merge_kernel, 1, 32, 0, stream, (const double*)scratch, kDotBlocks, scale, out);
  return check_launch("dot merge");
}

}  // extern "C"
