// LayerNorm forward / backward.  HBM-bound row kernels: one
// 128-thread CTA per token row, the row held in registers (128-bit loads),
// block reductions by warp shuffle + a 4-entry shared array.  The backward's
// dgamma/dbeta are per-row-chunk column partials merged in ascending chunk
// order (deterministic, no atomics).
#include "nnt_internal.h"

namespace nnt {
namespace {

constexpr int kT = 128;          // threads per CTA
constexpr int kMaxNV = 16;       // float4 per thread -> E <= 8192
constexpr int kBwdRowsPer = 16;  // rows per dgamma/dbeta partial chunk

__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < kT / 32; ++i) t += sh[i];  // fixed order
  return t;
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

// Forward: steps 1-3 of P:162 for one row.  Column index of (thread, j) is
// 4*(tid + j*kT); shifted sums with c = x[row][0] (R9); tile_e partials are
// merged in ascending tile order by summation, which is what the block
// reduction computes (fixed order).
template <typename TO, int NV>
__global__ void __launch_bounds__(kT) ln_fwd_kernel(const float* __restrict__ x, int64_t E, int64_t ldx,
                                                    const float* __restrict__ gamma, const float* __restrict__ beta,
                                                    float eps, TO* __restrict__ y, int64_t ldy,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  __shared__ float sh[kT / 32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * ldx;
  const float c = __ldg(xr);
  float4 v[NV];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
    if (col < E) {
      v[j] = __ldg(reinterpret_cast<const float4*>(xr + col));
      float d0 = v[j].x - c, d1 = v[j].y - c, d2 = v[j].z - c, d3 = v[j].w - c;
      s1 += (d0 + d1) + (d2 + d3);
      s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
  }
  s1 = block_sum(s1, sh);
  s2 = block_sum(s2, sh);
  const float inv_e = 1.0f / (float)E;
  const float ms = s1 * inv_e;
  const float var = fmaxf(s2 * inv_e - ms * ms, 0.f);
  const float mu = c + ms;
  const float rs = rsqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
  TO* yr = y + row * ldy;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
    if (col < E) {
      float4 g = __ldg(reinterpret_cast<const float4*>(gamma + col));
      float4 b = __ldg(reinterpret_cast<const float4*>(beta + col));
      float4 o;
      o.x = g.x * ((v[j].x - mu) * rs) + b.x;
      o.y = g.y * ((v[j].y - mu) * rs) + b.y;
      o.z = g.z * ((v[j].z - mu) * rs) + b.z;
      o.w = g.w * ((v[j].w - mu) * rs) + b.w;
      store4<TO>(yr + col, o);
    }
  }
}

// Backward for a chunk of kBwdRowsPer rows; dgamma/dbeta partial of the chunk.
template <int NV>
__global__ void __launch_bounds__(kT) ln_bwd_kernel(const float* __restrict__ dy, int64_t lddy,
                                                    const float* __restrict__ x, int64_t ldx,
                                                    const float* __restrict__ mean, const float* __restrict__ rstd,
                                                    const float* __restrict__ gamma, int64_t T, int64_t E,
                                                    const float* dres, float* dx, int64_t lddx,
                                                    __nv_bfloat16* __restrict__ dx16,
                                                    float* __restrict__ pg, float* __restrict__ pb) {
  __shared__ float sh[kT / 32];
  float4 accg[NV], accb[NV], g4[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    accg[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    accb[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
    if (col < E) g4[j] = __ldg(reinterpret_cast<const float4*>(gamma + col));
  }
  const int64_t r0 = (int64_t)blockIdx.x * kBwdRowsPer;
  const int64_t r1 = min(r0 + kBwdRowsPer, T);
  const float inv_e = 1.0f / (float)E;
  for (int64_t row = r0; row < r1; ++row) {
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    float4 xh[NV], dxh[NV];
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
      if (col < E) {
        float4 xv = __ldg(reinterpret_cast<const float4*>(x + row * ldx + col));
        float4 d = __ldg(reinterpret_cast<const float4*>(dy + row * lddy + col));
        xh[j] = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        dxh[j] = make_float4(d.x * g4[j].x, d.y * g4[j].y, d.z * g4[j].z, d.w * g4[j].w);
        sa += (dxh[j].x + dxh[j].y) + (dxh[j].z + dxh[j].w);
        sb += (dxh[j].x * xh[j].x + dxh[j].y * xh[j].y) + (dxh[j].z * xh[j].z + dxh[j].w * xh[j].w);
        accg[j].x += d.x * xh[j].x; accg[j].y += d.y * xh[j].y;
        accg[j].z += d.z * xh[j].z; accg[j].w += d.w * xh[j].w;
        accb[j].x += d.x; accb[j].y += d.y; accb[j].z += d.z; accb[j].w += d.w;
      }
    }
    sa = block_sum(sa, sh) * inv_e;
    sb = block_sum(sb, sh) * inv_e;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
      if (col < E) {
        float4 o;
        o.x = rs * (dxh[j].x - sa - xh[j].x * sb);
        o.y = rs * (dxh[j].y - sa - xh[j].y * sb);
        o.z = rs * (dxh[j].z - sa - xh[j].z * sb);
        o.w = rs * (dxh[j].w - sa - xh[j].w * sb);
        if (dres) {
          float4 r = *reinterpret_cast<const float4*>(dres + row * lddx + col);
          o.x += r.x; o.y += r.y; o.z += r.z; o.w += r.w;
        }
        *reinterpret_cast<float4*>(dx + row * lddx + col) = o;
        if (dx16) store4<__nv_bfloat16>(dx16 + row * lddx + col, o);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
    if (col < E) {
      *reinterpret_cast<float4*>(pg + (int64_t)blockIdx.x * E + col) = accg[j];
      *reinterpret_cast<float4*>(pb + (int64_t)blockIdx.x * E + col) = accb[j];
    }
  }
}

__global__ void ln_param_merge_kernel(const float* __restrict__ pg, const float* __restrict__ pb, int64_t chunks,
                                      int64_t E, float* dgamma, float* dbeta, int accumulate) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= E) return;
  float sg = 0.f, sb = 0.f;
  for (int64_t k = 0; k < chunks; ++k) {
    sg += pg[k * E + c];
    sb += pb[k * E + c];
  }
  dgamma[c] = accumulate ? dgamma[c] + sg : sg;
  dbeta[c] = accumulate ? dbeta[c] + sb : sb;
}

template <typename TO>
nnt_status launch_fwd(int nv, const float* x, int64_t T, int64_t E, int64_t ldx, const float* g, const float* b,
                      float eps, TO* y, int64_t ldy, float* mean, float* rstd, cudaStream_t s) {
#define NNT_LNF(NVV) \
  case NVV: ln_fwd_kernel<TO, NVV><<<(unsigned)T, kT, 0, s>>>(x, E, ldx, g, b, eps, y, ldy, mean, rstd); break;
  switch (nv) {
    NNT_LNF(1) NNT_LNF(2) NNT_LNF(3) NNT_LNF(4) NNT_LNF(6) NNT_LNF(8) NNT_LNF(12) NNT_LNF(16)
    default: return fail(NNT_ERR_UNSUPPORTED, "layernorm: unsupported E");
  }
#undef NNT_LNF
  return check_launch("layernorm_fwd");
}

int pick_nv(int64_t E) {
  int64_t need = (E / 4 + kT - 1) / kT;
  const int opts[] = {1, 2, 3, 4, 6, 8, 12, 16};
  for (int o : opts)
    if (o >= need) return o;
  return -1;
}

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_layernorm_fwd(const float* x, int64_t T, int64_t E, int64_t ldx, int64_t tile_e, const float* gamma,
                             const float* beta, float eps, void* y, int y_dtype, int64_t ldy, float* mean,
                             float* rstd, nnt_stream_t stream) {
  NNT_REQUIRE(x && gamma && beta && y && mean && rstd, NNT_ERR_NULL, "nnt_layernorm_fwd: NULL pointer");
  NNT_REQUIRE(T > 0 && E > 0 && ldx >= E && ldy >= E, NNT_ERR_SHAPE, "nnt_layernorm_fwd: T=%lld E=%lld",
              (long long)T, (long long)E);
  NNT_REQUIRE(tile_e > 0, NNT_ERR_TILE, "nnt_layernorm_fwd: tile_e=%lld", (long long)tile_e);
  NNT_REQUIRE(valid_dtype(y_dtype), NNT_ERR_DTYPE, "nnt_layernorm_fwd: dtype %d", y_dtype);
  NNT_REQUIRE(E % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned16(x) && aligned16(gamma) &&
                  aligned16(beta) && aligned16(y),
              NNT_ERR_ALIGN, "nnt_layernorm_fwd: E, ld must be multiples of 4 and pointers 16B aligned");
  int nv = pick_nv(E);
  NNT_REQUIRE(nv > 0, NNT_ERR_UNSUPPORTED, "nnt_layernorm_fwd: E=%lld > 8192", (long long)E);
  LaunchScope sc(NNT_K_LN_FWD, stream, (double)T * E * (4 + dtype_size(y_dtype)) + 8.0 * T, 0);
  if (y_dtype == NNT_F32) return launch_fwd<float>(nv, x, T, E, ldx, gamma, beta, eps, (float*)y, ldy, mean, rstd, stream);
  return launch_fwd<__nv_bfloat16>(nv, x, T, E, ldx, gamma, beta, eps, (__nv_bfloat16*)y, ldy, mean, rstd, stream);
}

size_t nnt_layernorm_bwd_scratch_bytes(int64_t T, int64_t E) {
  if (T <= 0 || E <= 0) return 0;
  int64_t chunks = (T + kBwdRowsPer - 1) / kBwdRowsPer;
  return (size_t)(2 * chunks * E) * sizeof(float);
}

nnt_status nnt_layernorm_bwd(const float* dy, int64_t lddy, const float* x, int64_t ldx, const float* mean,
                             const float* rstd, const float* gamma, int64_t T, int64_t E, const float* dres,
                             float* dx, int64_t lddx, void* dx_bf16, float* dgamma, float* dbeta,
                             int accumulate_params, void* scratch, size_t scratch_bytes, nnt_stream_t stream) {
  NNT_REQUIRE(dy && x && mean && rstd && gamma && dx && dgamma && dbeta && scratch, NNT_ERR_NULL,
              "nnt_layernorm_bwd: NULL pointer");
  NNT_REQUIRE(T > 0 && E > 0 && lddy >= E && ldx >= E && lddx >= E, NNT_ERR_SHAPE,
              "nnt_layernorm_bwd: T=%lld E=%lld", (long long)T, (long long)E);
  NNT_REQUIRE(E % 4 == 0 && lddy % 4 == 0 && ldx % 4 == 0 && lddx % 4 == 0 && aligned16(dy) && aligned16(x) &&
                  aligned16(dx) && aligned16(gamma) && (!dres || aligned16(dres)) &&
                  (!dx_bf16 || (reinterpret_cast<uintptr_t>(dx_bf16) & 7u) == 0),
              NNT_ERR_ALIGN, "nnt_layernorm_bwd: alignment");
  NNT_REQUIRE(scratch_bytes >= nnt_layernorm_bwd_scratch_bytes(T, E), NNT_ERR_WORKSPACE,
              "nnt_layernorm_bwd: scratch %zu < %zu", scratch_bytes, nnt_layernorm_bwd_scratch_bytes(T, E));
  int nv = pick_nv(E);
  NNT_REQUIRE(nv > 0, NNT_ERR_UNSUPPORTED, "nnt_layernorm_bwd: E=%lld > 8192", (long long)E);
  int64_t chunks = (T + kBwdRowsPer - 1) / kBwdRowsPer;
  float* pg = (float*)scratch;
  float* pb = pg + chunks * E;
  double bytes = (double)T * E * (4 + 4 + 4 + (dres ? 4 : 0) + (dx_bf16 ? 2 : 0)) + 8.0 * T;
  LaunchScope sc(NNT_K_LN_BWD, stream, bytes, 0, 2);
#define NNT_LNB(NVV)                                                                                        \
  case NVV:                                                                                                 \
    ln_bwd_kernel<NVV><<<(unsigned)chunks, kT, 0, stream>>>(dy, lddy, x, ldx, mean, rstd, gamma, T, E, dres, \
                                                            dx, lddx, (__nv_bfloat16*)dx_bf16, pg, pb);      \
    break;
  switch (nv) {
    NNT_LNB(1) NNT_LNB(2) NNT_LNB(3) NNT_LNB(4) NNT_LNB(6) NNT_LNB(8) NNT_LNB(12) NNT_LNB(16)
    default: return fail(NNT_ERR_UNSUPPORTED, "layernorm_bwd: unsupported E");
  }
#undef NNT_LNB
  NNT_TRY(check_launch("layernorm_bwd"));
  ln_param_merge_kernel<<<(unsigned)((E + 255) / 256), 256, 0, stream>>>(pg, pb, chunks, E, dgamma, dbeta,
                                                                          accumulate_params);
  return check_launch("layernorm_bwd merge");
}

}  // extern "C"
