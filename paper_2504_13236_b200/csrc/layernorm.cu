// LayerNorm forward / backward.  HBM-bound row kernels.
//   E <= 1024: one WARP per token row (row in registers as float4, reductions by
//              warp shuffle only); forward warps stride over rows with the next row
//              prefetched, backward CTAs own a block of rows (single pass);
//   E  > 1024: forward one 128-thread CTA per row (shuffle + 4-entry shared array; the ring-fed
//              4-warp-group variant, NNT_LN_FWD_RING=1, measured slower);
//              backward a group of 4 or 8 warps per row, persistent CTAs (ln_bwd_groups).
// The backward's dgamma/dbeta are per-CTA column partials (rows of a CTA are
// accumulated in a fixed order) merged by the deterministic column merge
// (reduce.cuh): bitwise reproducible, no atomics.
#include <cstdlib>

#include "reduce.cuh"
#include "tc_ptx.cuh"

namespace nnt {
namespace {

constexpr int kWarpRowsPerCta = 8;   // warp kernels: 8 warps
constexpr int kT = 128;              // CTA-per-row kernels: threads
constexpr int kCtaBwdRows = 16;      // backward kernels: at least this many rows per partial

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

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

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

// Normalise + affine of one float4 (steps 2 and 3 of P:162).
__device__ __forceinline__ float4 affine(float4 v, float4 g, float4 b, float mu, float rs) {
  return make_float4(g.x * ((v.x - mu) * rs) + b.x, g.y * ((v.y - mu) * rs) + b.y, g.z * ((v.z - mu) * rs) + b.z,
                     g.w * ((v.w - mu) * rs) + b.w);
}

// ------------------------------------------------------------------ forward, warp per row
// Step 1 with shifted sums (c = x[row][0], R9); E-tile partials are merged by
// summation, which is what the (fixed-order) shuffle reduction computes.
// Warps stride over rows (row = warp id + k * total warps) with the next row's loads issued
// before the current row's reduction, so reads and writes of neighbouring rows overlap.
template <typename TO, int NV>
__global__ void __launch_bounds__(32 * kWarpRowsPerCta)
    ln_fwd_warp(const float* __restrict__ x, int64_t T, int E, int64_t ldx, const float* __restrict__ gamma,
                const float* __restrict__ beta, float eps, TO* __restrict__ y, int64_t ldy,
                float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  NNT_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * kWarpRowsPerCta;
  int64_t row = (int64_t)blockIdx.x * kWarpRowsPerCta + (threadIdx.x >> 5);
  if (row >= T) return;
  const float inv_e = 1.0f / (float)E;
  float4 v[NV], nx[NV];
  float c = __ldg(x + row * ldx), cn = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (4 * (lane + 32 * j) < E) v[j] = ldg4(x + row * ldx + 4 * (lane + 32 * j));
  for (; row < T; row += stride) {
    const int64_t nrow = row + stride;
    if (nrow < T) {  // next row in flight while this one is reduced and stored
      cn = __ldg(x + nrow * ldx);
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (4 * (lane + 32 * j) < E) nx[j] = ldg4(x + nrow * ldx + 4 * (lane + 32 * j));
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if (4 * (lane + 32 * j) < E) {
        float d0 = v[j].x - c, d1 = v[j].y - c, d2 = v[j].z - c, d3 = v[j].w - c;
        s1 += (d0 + d1) + (d2 + d3);
        s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float ms = s1 * inv_e;
    const float var = fmaxf(s2 * inv_e - ms * ms, 0.f);
    const float mu = c + ms, rs = rsqrtf(var + eps);
    if (lane == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
    TO* yr = y + row * ldy;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int col = 4 * (lane + 32 * j);
      if (col < E) store4<TO>(yr + col, affine(v[j], ldg4(gamma + col), ldg4(beta + col), mu, rs));
    }
    c = cn;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = nx[j];
  }
}

// ------------------------------------------------------------------ forward, CTA per row
template <typename TO, int NV>
__global__ void __launch_bounds__(kT) ln_fwd_cta(const float* __restrict__ x, int64_t E, int64_t ldx,
                                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                                 float eps, TO* __restrict__ y, int64_t ldy,
                                                 float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  NNT_PDL_ENTRY();
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
      v[j] = ldg4(xr + col);
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
  const float mu = c + ms, rs = rsqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
  TO* yr = y + row * ldy;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int64_t col = 4 * ((int64_t)threadIdx.x + j * kT);
    if (col < E) store4<TO>(yr + col, affine(v[j], ldg4(gamma + col), ldg4(beta + col), mu, rs));
  }
}

// ------------------------------------------------------------------ backward helpers
struct RowGrad {
  float4 xh, dxh;
};

// dx of one float4 given the row means sa = mean(dxhat), sb = mean(dxhat*xhat)
__device__ __forceinline__ float4 dx_of(const RowGrad& r, float rs, float sa, float sb) {
  return make_float4(rs * (r.dxh.x - sa - r.xh.x * sb), rs * (r.dxh.y - sa - r.xh.y * sb),
                     rs * (r.dxh.z - sa - r.xh.z * sb), rs * (r.dxh.w - sa - r.xh.w * sb));
}

// ------------------------------------------------------------------ backward, warp per row, single pass
// One warp per row in a CTA of kRowsWarps warps that owns `rows_per_cta` consecutive rows: x,
// dy and the residual gradient of a row are loaded once (all loads of a row in flight
// together), xhat and dxhat stay in registers for the dx pass, and the lane's dgamma/dbeta
// columns accumulate in registers over the CTA's rows.  The CTA's warps are combined in fixed
// order at the end into one partial row (deterministic, no atomics).  Two 192-thread CTAs per
// SM leave 168 registers per thread: no spills at E = 768.
constexpr int kRowsWarps = 6;

// SUM: also the column sums of the output dx (a third partial row: the bias gradient of the
// linear layer whose output this LayerNorm's input is, e.g. the previous block's projection).
template <int NV, bool SUM>
__global__ void __launch_bounds__(32 * kRowsWarps, 2)
    ln_bwd_rows(const float* __restrict__ dy, int64_t lddy, const float* __restrict__ x, int64_t ldx,
                const float* __restrict__ mean, const float* __restrict__ rstd, const float* __restrict__ gamma,
                int64_t T, int E, int64_t rows_per_cta, const float* __restrict__ dres, float* __restrict__ dx,
                int64_t lddx, __nv_bfloat16* __restrict__ dx16, float* __restrict__ pg, float* __restrict__ pb,
                float* __restrict__ ps) {
  NNT_PDL_ENTRY();
  extern __shared__ float4 red[];  // [kRowsWarps][2 + SUM][E/4], used once at the end
  constexpr int NP = SUM ? 3 : 2;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int E4 = E / 4;
  const float inv_e = 1.0f / (float)E;
  float4 ag[NV], ab[NV], as[SUM ? NV : 1];
#pragma unroll
  for (int j = 0; j < NV; ++j) ag[j] = ab[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (SUM)
#pragma unroll
    for (int j = 0; j < (SUM ? NV : 1); ++j) as[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(r0 + rows_per_cta, T);
  for (int64_t row = r0 + w; row < r1; row += kRowsWarps) {
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    float4 xh[NV], dh[NV], rr[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * j;
      if (i4 < E4) {
        xh[j] = ldg4(x + row * ldx + 4 * i4);
        dh[j] = ldg4(dy + row * lddy + 4 * i4);
        rr[j] = dres ? ldg4(dres + row * lddx + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * j;
      if (i4 < E4) {
        const float4 g = ldg4(gamma + 4 * i4), d = dh[j];
        float4& h = xh[j];
        h = make_float4((h.x - mu) * rs, (h.y - mu) * rs, (h.z - mu) * rs, (h.w - mu) * rs);
        ag[j].x += d.x * h.x; ag[j].y += d.y * h.y; ag[j].z += d.z * h.z; ag[j].w += d.w * h.w;
        ab[j].x += d.x; ab[j].y += d.y; ab[j].z += d.z; ab[j].w += d.w;
        const float4 e = make_float4(d.x * g.x, d.y * g.y, d.z * g.z, d.w * g.w);  // dxhat
        dh[j] = e;
        sa += (e.x + e.y) + (e.z + e.w);
        sb += (e.x * h.x + e.y * h.y) + (e.z * h.z + e.w * h.w);
      }
    }
    sa = warp_sum(sa) * inv_e;
    sb = warp_sum(sb) * inv_e;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * j;
      if (i4 < E4) {
        RowGrad rg{xh[j], dh[j]};
        float4 o = dx_of(rg, rs, sa, sb);
        o.x += rr[j].x; o.y += rr[j].y; o.z += rr[j].z; o.w += rr[j].w;
        *reinterpret_cast<float4*>(dx + row * lddx + 4 * i4) = o;
        if (dx16) store4<__nv_bfloat16>(dx16 + row * lddx + 4 * i4, o);
        if constexpr (SUM) {
          as[j].x += o.x; as[j].y += o.y; as[j].z += o.z; as[j].w += o.w;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i4 = lane + 32 * j;
    if (i4 < E4) {
      red[(size_t)(NP * w) * E4 + i4] = ag[j];
      red[(size_t)(NP * w + 1) * E4 + i4] = ab[j];
      if constexpr (SUM) red[(size_t)(NP * w + 2) * E4 + i4] = as[j];
    }
  }
  __syncthreads();
  for (int i4 = threadIdx.x; i4 < E4; i4 += 32 * kRowsWarps) {
    float4 sg = make_float4(0.f, 0.f, 0.f, 0.f), s4 = make_float4(0.f, 0.f, 0.f, 0.f),
           ss = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < kRowsWarps; ++k) {  // fixed warp order
      const float4 a = red[(size_t)(NP * k) * E4 + i4], b = red[(size_t)(NP * k + 1) * E4 + i4];
      sg.x += a.x; sg.y += a.y; sg.z += a.z; sg.w += a.w;
      s4.x += b.x; s4.y += b.y; s4.z += b.z; s4.w += b.w;
      if constexpr (SUM) {
        const float4 c = red[(size_t)(NP * k + 2) * E4 + i4];
        ss.x += c.x; ss.y += c.y; ss.z += c.z; ss.w += c.w;
      }
    }
    reinterpret_cast<float4*>(pg + (int64_t)blockIdx.x * E)[i4] = sg;
    reinterpret_cast<float4*>(pb + (int64_t)blockIdx.x * E)[i4] = s4;
    if constexpr (SUM) reinterpret_cast<float4*>(ps + (int64_t)blockIdx.x * E)[i4] = ss;
  }
}

// ------------------------------------------------------------------ backward, warp groups per row
// E > 1024: a row is split over a group of G warps (float4 column i4 = lane + 32 (k + G j) for
// warp k of the group, so each warp streams contiguous 512-byte pieces); the CTA's 8 warps form
// 8 / G groups that stride over the CTA's rows.  The next row's x / dy / residual-gradient loads
// are issued before the current row's reductions (double-buffered registers), the per-row sums
// sa, sb cross the group's warps through double-buffered shared slots with one named barrier per
// row, and dgamma / dbeta (/ sum_t dx) accumulate in registers over the group's rows; the groups
// are combined in fixed order at the end into one partial row per CTA (deterministic, merged by
// the column merge like the row kernel).  One CTA per SM, persistent over rows.
constexpr int kGrpWarps = 8;

template <int NV, int G, bool SUM>
__global__ void __launch_bounds__(32 * kGrpWarps, 1)
    ln_bwd_groups(const float* __restrict__ dy, int64_t lddy, const float* __restrict__ x, int64_t ldx,
                  const float* __restrict__ mean, const float* __restrict__ rstd, const float* __restrict__ gamma,
                  int64_t T, int E, int64_t rows_per_cta, const float* __restrict__ dres, float* __restrict__ dx,
                  int64_t lddx, __nv_bfloat16* __restrict__ dx16, float* __restrict__ pg, float* __restrict__ pb,
                  float* __restrict__ ps) {
  NNT_PDL_ENTRY();
  constexpr int NG = kGrpWarps / G;  // row groups per CTA
  constexpr int NP = SUM ? 3 : 2;
  extern __shared__ float4 red[];    // [NG][NP][E/4] at the end
  __shared__ float2 xs[2][NG][G];    // per-row (sa, sb) of each warp, double-buffered
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = w / G, k = w % G;
  const int E4 = E / 4;
  const float inv_e = 1.0f / (float)E;
  // NV <= 4: the next row prefetched and gamma held in registers; NV > 4 (E > 4096): neither
  // (register budget of one 256-thread CTA per SM)
  constexpr bool PREF = NV <= 4;
  float4 ag[NV], ab[NV], as[SUM ? NV : 1], gm[PREF ? NV : 1];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    ag[j] = ab[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (SUM) as[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int i4 = lane + 32 * (k + G * j);
    if constexpr (PREF) gm[j] = i4 < E4 ? ldg4(gamma + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(r0 + rows_per_cta, T);
  float4 xv[NV], dv[NV], rv[NV];
  auto load = [&](int64_t row, float4 (&a)[NV], float4 (&b)[NV], float4 (&c)[NV]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + G * j);
      if (i4 < E4) {
        a[j] = ldg4(x + row * ldx + 4 * i4);
        b[j] = ldg4(dy + row * lddy + 4 * i4);
        c[j] = dres ? ldg4(dres + row * lddx + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  int64_t row = r0 + grp;
  float mu = 0.f, rs = 0.f;  // this row's statistics, loaded with its data (a late load stalls every use)
  if (row < r1) {
    load(row, xv, dv, rv);
    mu = __ldg(mean + row);
    rs = __ldg(rstd + row);
  }
  int buf = 0;
  for (; row < r1; row += NG, buf ^= 1) {
    float4 xn[PREF ? NV : 1], dn[PREF ? NV : 1], rn[PREF ? NV : 1];
    float mun = 0.f, rsn = 0.f;
    const int64_t nrow = row + NG;
    if (nrow < r1) {
      mun = __ldg(mean + nrow);
      rsn = __ldg(rstd + nrow);
      if constexpr (PREF) load(nrow, xn, dn, rn);  // next row in flight during this one's reductions
    }
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + G * j);
      if (i4 < E4) {
        const float4 d = dv[j];
        float4& h = xv[j];
        h = make_float4((h.x - mu) * rs, (h.y - mu) * rs, (h.z - mu) * rs, (h.w - mu) * rs);
        ag[j].x += d.x * h.x; ag[j].y += d.y * h.y; ag[j].z += d.z * h.z; ag[j].w += d.w * h.w;
        ab[j].x += d.x; ab[j].y += d.y; ab[j].z += d.z; ab[j].w += d.w;
        float4 gj;
        if constexpr (PREF)
          gj = gm[j];
        else
          gj = ldg4(gamma + 4 * i4);
        const float4 e = make_float4(d.x * gj.x, d.y * gj.y, d.z * gj.z, d.w * gj.w);  // dxhat
        dv[j] = e;
        sa += (e.x + e.y) + (e.z + e.w);
        sb += (e.x * h.x + e.y * h.y) + (e.z * h.z + e.w * h.w);
      }
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) xs[buf][grp][k] = make_float2(sa, sb);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * G) : "memory");
    sa = 0.f;
    sb = 0.f;
#pragma unroll
    for (int i = 0; i < G; ++i) {  // fixed warp order
      const float2 t = xs[buf][grp][i];
      sa += t.x;
      sb += t.y;
    }
    sa *= inv_e;
    sb *= inv_e;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + G * j);
      if (i4 < E4) {
        RowGrad rg{xv[j], dv[j]};
        float4 o = dx_of(rg, rs, sa, sb);
        o.x += rv[j].x; o.y += rv[j].y; o.z += rv[j].z; o.w += rv[j].w;
        *reinterpret_cast<float4*>(dx + row * lddx + 4 * i4) = o;
        if (dx16) store4<__nv_bfloat16>(dx16 + row * lddx + 4 * i4, o);
        if constexpr (SUM) {
          as[j].x += o.x; as[j].y += o.y; as[j].z += o.z; as[j].w += o.w;
        }
      }
    }
    if constexpr (PREF) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        xv[j] = xn[j];
        dv[j] = dn[j];
        rv[j] = rn[j];
      }
    } else if (nrow < r1) {
      load(nrow, xv, dv, rv);
    }
    mu = mun;
    rs = rsn;
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i4 = lane + 32 * (k + G * j);
    if (i4 < E4) {
      red[(size_t)(NP * grp) * E4 + i4] = ag[j];
      red[(size_t)(NP * grp + 1) * E4 + i4] = ab[j];
      if constexpr (SUM) red[(size_t)(NP * grp + 2) * E4 + i4] = as[j];
    }
  }
  __syncthreads();
  for (int i4 = threadIdx.x; i4 < E4; i4 += 32 * kGrpWarps) {
    float4 sg = make_float4(0.f, 0.f, 0.f, 0.f), s4 = make_float4(0.f, 0.f, 0.f, 0.f),
           ss = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < NG; ++q) {  // fixed group order
      const float4 a = red[(size_t)(NP * q) * E4 + i4], b = red[(size_t)(NP * q + 1) * E4 + i4];
      sg.x += a.x; sg.y += a.y; sg.z += a.z; sg.w += a.w;
      s4.x += b.x; s4.y += b.y; s4.z += b.z; s4.w += b.w;
      if constexpr (SUM) {
        const float4 c = red[(size_t)(NP * q + 2) * E4 + i4];
        ss.x += c.x; ss.y += c.y; ss.z += c.z; ss.w += c.w;
      }
    }
    reinterpret_cast<float4*>(pg + (int64_t)blockIdx.x * E)[i4] = sg;
    reinterpret_cast<float4*>(pb + (int64_t)blockIdx.x * E)[i4] = s4;
    if constexpr (SUM) reinterpret_cast<float4*>(ps + (int64_t)blockIdx.x * E)[i4] = ss;
  }
}

// ------------------------------------------------------------------ backward, row ring (1024 < E <= 2048)
// The group kernel above keeps one row in flight per group beyond the one being reduced (register
// prefetch: 220 registers, 8 warps per SM), so each group waits about one DRAM latency per row
// (ncu: 47 % of DRAM bandwidth at E = 1600, long-scoreboard stalls).  Here each group of 4 warps
// owns a ring of kRing shared-memory slots; one elected thread streams the group's rows into it
// with 1-D bulk copies (x, dy and the residual gradient of a row: 3 E floats, completing on the
// slot's mbarrier), kRing rows ahead of the row being reduced.  The arithmetic, the per-row
// cross-warp sums and the fixed-order column partials are those of ln_bwd_groups.
constexpr int kRing = 4, kRingGroups = 2, kRingG = 4;
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int NV, bool SUM>
__global__ void __launch_bounds__(32 * kRingG * kRingGroups, 1)
    ln_bwd_ring(const float* __restrict__ dy, int64_t lddy, const float* __restrict__ x, int64_t ldx,
                const float* __restrict__ mean, const float* __restrict__ rstd, const float* __restrict__ gamma,
                int64_t T, int E, int64_t rows_per_cta, const float* __restrict__ dres, float* __restrict__ dx,
                int64_t lddx, __nv_bfloat16* __restrict__ dx16, float* __restrict__ pg, float* __restrict__ pb,
                float* __restrict__ ps) {
  NNT_PDL_ENTRY();
  constexpr int NP = SUM ? 3 : 2;
  extern __shared__ __align__(1024) uint8_t ring_smem[];  // [kRingGroups][kRing] slots of {x, dy, dres} rows
  __shared__ float2 xs[2][kRingGroups][kRingG];
  __shared__ __align__(8) uint64_t fullb[kRingGroups][kRing];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = w / kRingG, k = w % kRingG;
  const int E4 = E / 4;
  const float inv_e = 1.0f / (float)E;
  const int nin = dres ? 3 : 2;
  const uint32_t row_bytes = (uint32_t)E * 4u;
  float4* const slots = reinterpret_cast<float4*>(ring_smem) + (size_t)grp * kRing * 3 * E4;
  if (k == 0 && lane == 0)
    for (int i = 0; i < kRing; ++i) mbar_init(smem_u32(&fullb[grp][i]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(r0 + rows_per_cta, T);
  // the group's rows: r0 + grp, r0 + grp + kRingGroups, ...; row index n of the group -> slot n % kRing
  auto issue = [&](int64_t n) {  // elected thread: bulk copies of the group's n-th row
    const int64_t row = r0 + grp + n * kRingGroups;
    if (row >= r1) return;
    const int sl = (int)(n % kRing);
    const uint32_t bar = smem_u32(&fullb[grp][sl]);
    const uint32_t dst = smem_u32(slots + (size_t)sl * 3 * E4);
    mbar_expect_tx(bar, row_bytes * (uint32_t)nin);
    bulk_g2s(dst, x + row * ldx, row_bytes, bar);
    bulk_g2s(dst + row_bytes, dy + row * lddy, row_bytes, bar);
    if (dres) bulk_g2s(dst + 2 * row_bytes, dres + row * lddx, row_bytes, bar);
  };
  if (k == 0 && lane == 0)
    for (int n = 0; n < kRing; ++n) issue(n);
  float4 ag[NV], ab[NV], as[SUM ? NV : 1], gm[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    ag[j] = ab[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (SUM) as[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int i4 = lane + 32 * (k + kRingG * j);
    gm[j] = i4 < E4 ? ldg4(gamma + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  int64_t row = r0 + grp;
  float mu = 0.f, rs = 0.f;
  if (row < r1) {
    mu = __ldg(mean + row);
    rs = __ldg(rstd + row);
  }
  int buf = 0;
  for (int64_t n = 0; row < r1; ++n, row += kRingGroups, buf ^= 1) {
    const int sl = (int)(n % kRing);
    float mun = 0.f, rsn = 0.f;
    if (row + kRingGroups < r1) {
      mun = __ldg(mean + row + kRingGroups);
      rsn = __ldg(rstd + row + kRingGroups);
    }
    mbar_wait(smem_u32(&fullb[grp][sl]), (uint32_t)((n / kRing) & 1));
    const float4* xr = slots + (size_t)sl * 3 * E4;
    float4 xv[NV], dv[NV], rv[NV];
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + kRingG * j);
      if (i4 < E4) {
        float4 h = xr[i4];
        const float4 d = xr[E4 + i4];
        rv[j] = dres ? xr[2 * E4 + i4] : make_float4(0.f, 0.f, 0.f, 0.f);
        h = make_float4((h.x - mu) * rs, (h.y - mu) * rs, (h.z - mu) * rs, (h.w - mu) * rs);
        xv[j] = h;
        ag[j].x += d.x * h.x; ag[j].y += d.y * h.y; ag[j].z += d.z * h.z; ag[j].w += d.w * h.w;
        ab[j].x += d.x; ab[j].y += d.y; ab[j].z += d.z; ab[j].w += d.w;
        const float4 gj = gm[j];
        const float4 e = make_float4(d.x * gj.x, d.y * gj.y, d.z * gj.z, d.w * gj.w);  // dxhat
        dv[j] = e;
        sa += (e.x + e.y) + (e.z + e.w);
        sb += (e.x * h.x + e.y * h.y) + (e.z * h.z + e.w * h.w);
      }
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) xs[buf][grp][k] = make_float2(sa, sb);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * kRingG) : "memory");  // also: the slot is read
    if (k == 0 && lane == 0) issue(n + kRing);  // refill the slot kRing rows ahead
    sa = 0.f;
    sb = 0.f;
#pragma unroll
    for (int i = 0; i < kRingG; ++i) {  // fixed warp order
      const float2 t = xs[buf][grp][i];
      sa += t.x;
      sb += t.y;
    }
    sa *= inv_e;
    sb *= inv_e;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + kRingG * j);
      if (i4 < E4) {
        RowGrad rg{xv[j], dv[j]};
        float4 o = dx_of(rg, rs, sa, sb);
        o.x += rv[j].x; o.y += rv[j].y; o.z += rv[j].z; o.w += rv[j].w;
        *reinterpret_cast<float4*>(dx + row * lddx + 4 * i4) = o;
        if (dx16) store4<__nv_bfloat16>(dx16 + row * lddx + 4 * i4, o);
        if constexpr (SUM) {
          as[j].x += o.x; as[j].y += o.y; as[j].z += o.z; as[j].w += o.w;
        }
      }
    }
    mu = mun;
    rs = rsn;
  }
  __syncthreads();  // the ring is free: reuse it for the group partials
  float4* red = reinterpret_cast<float4*>(ring_smem);  // [kRingGroups][NP][E/4]
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i4 = lane + 32 * (k + kRingG * j);
    if (i4 < E4) {
      red[(size_t)(NP * grp) * E4 + i4] = ag[j];
      red[(size_t)(NP * grp + 1) * E4 + i4] = ab[j];
      if constexpr (SUM) red[(size_t)(NP * grp + 2) * E4 + i4] = as[j];
    }
  }
  __syncthreads();
  for (int i4 = threadIdx.x; i4 < E4; i4 += 32 * kRingG * kRingGroups) {
    float4 sg = make_float4(0.f, 0.f, 0.f, 0.f), s4 = make_float4(0.f, 0.f, 0.f, 0.f),
           ss = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < kRingGroups; ++q) {  // fixed group order
      const float4 a = red[(size_t)(NP * q) * E4 + i4], b = red[(size_t)(NP * q + 1) * E4 + i4];
      sg.x += a.x; sg.y += a.y; sg.z += a.z; sg.w += a.w;
      s4.x += b.x; s4.y += b.y; s4.z += b.z; s4.w += b.w;
      if constexpr (SUM) {
        const float4 c = red[(size_t)(NP * q + 2) * E4 + i4];
        ss.x += c.x; ss.y += c.y; ss.z += c.z; ss.w += c.w;
      }
    }
    reinterpret_cast<float4*>(pg + (int64_t)blockIdx.x * E)[i4] = sg;
    reinterpret_cast<float4*>(pb + (int64_t)blockIdx.x * E)[i4] = s4;
    if constexpr (SUM) reinterpret_cast<float4*>(ps + (int64_t)blockIdx.x * E)[i4] = ss;
  }
}

// NNT_LN_BWD_RING=0: the register-prefetch group kernel for 1024 < E <= 2048 too (A/B runs)
bool ln_bwd_ring_on() {
  const char* e = getenv("NNT_LN_BWD_RING");
  return !(e && e[0] == '0');
}

// warps per row and float4s per lane of the group kernel (E > 1024): G = 4 up to E = 2048, 8 above
void pick_groups(int64_t E, int* G, int* NV) {
  const int64_t E4 = E / 4;
  *G = E4 <= 4 * 32 * 4 ? 4 : 8;
  *NV = (int)((E4 + 32 * *G - 1) / (32 * *G));
}

int pick_nv_cta(int64_t E) {
  int64_t need = (E / 4 + kT - 1) / kT;
  const int opts[] = {1, 2, 3, 4, 6, 8, 12, 16};
  for (int o : opts)
    if (o >= need) return o;
  return -1;
}
int pick_nv_warp(int64_t E) {
  if (E > 1024) return -1;
  int64_t need = (E / 4 + 31) / 32;
  const int opts[] = {1, 2, 4, 6, 8};
  for (int o : opts)
    if (o >= need) return o;
  return -1;
}

// ------------------------------------------------------------------ forward, row ring (1024 < E <= 2048)
// The forward counterpart of ln_bwd_ring: groups of 4 warps, each with a ring of kRing x rows
// streamed by bulk copies (kRing rows ahead), CTAs persistent over a block of rows; the row's
// shifted sums (c = x[row][0], R9) cross the group's warps through double-buffered shared slots
// (fixed warp order).  Same arithmetic as ln_fwd_cta up to the order of the shifted sums.
template <typename TO, int NV>
__global__ void __launch_bounds__(32 * kRingG * kRingGroups)
    ln_fwd_ring(const float* __restrict__ x, int64_t T, int E, int64_t ldx, int64_t rows_per_cta,
                const float* __restrict__ gamma, const float* __restrict__ beta, float eps, TO* __restrict__ y,
                int64_t ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  NNT_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t ring_smem[];  // [kRingGroups][kRing] x rows
  __shared__ float2 xs[2][kRingGroups][kRingG];
  __shared__ __align__(8) uint64_t fullb[kRingGroups][kRing];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = w / kRingG, k = w % kRingG;
  const int E4 = E / 4;
  const float inv_e = 1.0f / (float)E;
  const uint32_t row_bytes = (uint32_t)E * 4u;
  float4* const slots = reinterpret_cast<float4*>(ring_smem) + (size_t)grp * kRing * E4;
  if (k == 0 && lane == 0)
    for (int i = 0; i < kRing; ++i) mbar_init(smem_u32(&fullb[grp][i]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(r0 + rows_per_cta, T);
  auto issue = [&](int64_t n) {  // elected thread: the group's n-th row into slot n % kRing
    const int64_t row = r0 + grp + n * kRingGroups;
    if (row >= r1) return;
    const int sl = (int)(n % kRing);
    const uint32_t bar = smem_u32(&fullb[grp][sl]);
    mbar_expect_tx(bar, row_bytes);
    bulk_g2s(smem_u32(slots + (size_t)sl * E4), x + row * ldx, row_bytes, bar);
  };
  if (k == 0 && lane == 0)
    for (int n = 0; n < kRing; ++n) issue(n);
  float4 gm[NV], bt[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int i4 = lane + 32 * (k + kRingG * j);
    gm[j] = i4 < E4 ? ldg4(gamma + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
    bt[j] = i4 < E4 ? ldg4(beta + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  int buf = 0;
  int64_t row = r0 + grp;
  for (int64_t n = 0; row < r1; ++n, row += kRingGroups, buf ^= 1) {
    const int sl = (int)(n % kRing);
    mbar_wait(smem_u32(&fullb[grp][sl]), (uint32_t)((n / kRing) & 1));
    const float4* xr = slots + (size_t)sl * E4;
    const float c = reinterpret_cast<const float*>(xr)[0];
    float4 v[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + kRingG * j);
      if (i4 < E4) {
        v[j] = xr[i4];
        const float d0 = v[j].x - c, d1 = v[j].y - c, d2 = v[j].z - c, d3 = v[j].w - c;
        s1 += (d0 + d1) + (d2 + d3);
        s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) xs[buf][grp][k] = make_float2(s1, s2);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * kRingG) : "memory");  // also: the slot is read
    if (k == 0 && lane == 0) issue(n + kRing);
    s1 = 0.f;
    s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kRingG; ++i) {  // fixed warp order
      const float2 t = xs[buf][grp][i];
      s1 += t.x;
      s2 += t.y;
    }
    const float ms = s1 * inv_e;
    const float var = fmaxf(s2 * inv_e - ms * ms, 0.f);
    const float mu = c + ms, rs = rsqrtf(var + eps);
    if (k == 0 && lane == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
    TO* yr = y + row * ldy;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i4 = lane + 32 * (k + kRingG * j);
      if (i4 < E4) store4<TO>(yr + 4 * i4, affine(v[j], gm[j], bt[j], mu, rs));
    }
  }
}

// NNT_LN_FWD_RING=1 selects the ring forward for 1024 < E <= 2048; off by default: measured slower
// than the one-CTA-per-row kernel (E = 1600: 14.1 vs 11.5 us, E = 1280: 9.6 vs 9.3 us)
bool ln_fwd_ring_on() {
  const char* e = getenv("NNT_LN_FWD_RING");
  return e && e[0] == '1';
}

template <typename TO>
nnt_status launch_fwd(const float* x, int64_t T, int64_t E, int64_t ldx, const float* g, const float* b, float eps,
                      TO* y, int64_t ldy, float* mean, float* rstd, cudaStream_t s) {
  int nvw = pick_nv_warp(E);
  if (nvw > 0) {
    int64_t g64 = (T + kWarpRowsPerCta - 1) / kWarpRowsPerCta;  // warps stride over rows: 2 CTAs per SM
    if (g64 > 2 * num_sms()) g64 = 2 * num_sms();
    unsigned grid = (unsigned)g64;
#define NNT_LNFW(N) \
  case N: ::nnt::launch(ln_fwd_warp<TO, N>, grid, 32 * kWarpRowsPerCta, 0, s, x, T, (int)E, ldx, g, b, eps, y, ldy, mean, rstd); break;
    switch (nvw) { NNT_LNFW(1) NNT_LNFW(2) NNT_LNFW(4) NNT_LNFW(6) NNT_LNFW(8) }
#undef NNT_LNFW
    return check_launch("layernorm_fwd");
  }
  if (E <= 2048 && ln_fwd_ring_on() && (ldx * 4) % 16 == 0 && aligned16(x)) {
    // rows streamed into shared-memory rings; persistent CTAs, 4 per SM
    const int nvr = (int)((E / 4 + 32 * kRingG - 1) / (32 * kRingG));
    const int64_t resident = 4 * (int64_t)num_sms();
    int64_t rows_per = (T + resident - 1) / resident;
    if (rows_per < kRingGroups) rows_per = kRingGroups;
    const int64_t grid = (T + rows_per - 1) / rows_per;
    const size_t smem_ring = (size_t)kRingGroups * kRing * E * sizeof(float);  // <= 64 KB
    auto run = [&](auto kern) -> nnt_status {
      NNT_CUDA_TRY(set_max_dyn_smem(kern, (int)smem_ring));
      NNT_CUDA_TRY(::nnt::launch(kern, dim3((unsigned)grid), dim3(32 * kRingG * kRingGroups), smem_ring, s, x, T,
                                 (int)E, ldx, rows_per, g, b, eps, y, ldy, mean, rstd));
      return NNT_OK;
    };
    if (nvr == 3)
      NNT_TRY(run(ln_fwd_ring<TO, 3>));
    else
      NNT_TRY(run(ln_fwd_ring<TO, 4>));
    return check_launch("layernorm_fwd");
  }
  int nv = pick_nv_cta(E);
#define NNT_LNF(N) \
  case N: ::nnt::launch(ln_fwd_cta<TO, N>, (unsigned)T, kT, 0, s, x, E, ldx, g, b, eps, y, ldy, mean, rstd); break;
  switch (nv) {
    NNT_LNF(1) NNT_LNF(2) NNT_LNF(3) NNT_LNF(4) NNT_LNF(6) NNT_LNF(8) NNT_LNF(12) NNT_LNF(16)
    default: return fail(NNT_ERR_UNSUPPORTED, "layernorm: unsupported E");
  }
#undef NNT_LNF
  return check_launch("layernorm_fwd");
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
  NNT_REQUIRE(pick_nv_cta(E) > 0, NNT_ERR_UNSUPPORTED, "nnt_layernorm_fwd: E=%lld > 8192", (long long)E);
  LaunchScope sc(NNT_K_LN_FWD, stream, (double)T * E * (4 + dtype_size(y_dtype)) + 8.0 * T, 0);
  if (y_dtype == NNT_F32) return launch_fwd<float>(x, T, E, ldx, gamma, beta, eps, (float*)y, ldy, mean, rstd, stream);
  return launch_fwd<__nv_bfloat16>(x, T, E, ldx, gamma, beta, eps, (__nv_bfloat16*)y, ldy, mean, rstd, stream);
}

size_t nnt_layernorm_bwd_scratch_bytes(int64_t T, int64_t E) {
  if (T <= 0 || E <= 0) return 0;
  int64_t chunks = (T + kCtaBwdRows - 1) / kCtaBwdRows;  // >= the warp kernel's chunk count
  return (size_t)(3 * chunks * E) * sizeof(float);  // dgamma, dbeta and (optional) sum_t dx partials
}

nnt_status nnt_layernorm_bwd(const float* dy, int64_t lddy, const float* x, int64_t ldx, const float* mean,
                             const float* rstd, const float* gamma, int64_t T, int64_t E, const float* dres,
                             float* dx, int64_t lddx, void* dx_bf16, float* dgamma, float* dbeta,
                             float* dx_colsum, int accumulate_params, void* scratch, size_t scratch_bytes,
                             nnt_stream_t stream) {
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
  NNT_REQUIRE(pick_nv_cta(E) > 0, NNT_ERR_UNSUPPORTED, "nnt_layernorm_bwd: E=%lld > 8192", (long long)E);
  const int nvw = pick_nv_warp(E);
  // single-pass kernels: rows per CTA so that the resident CTAs (two per SM for the row kernel,
  // one for the group kernel) cover T in one wave (>= 16 rows, so the partial count stays within
  // nnt_layernorm_bwd_scratch_bytes)
  const int64_t resident = (nvw > 0 ? 2 : 1) * (int64_t)num_sms();
  int64_t rows_per_cta = (T + resident - 1) / resident;
  if (rows_per_cta < kCtaBwdRows) rows_per_cta = kCtaBwdRows;
  const int64_t chunks = (T + rows_per_cta - 1) / rows_per_cta;
  float* pg = (float*)scratch;
  float* pb = pg + chunks * E;
  float* ps = pb + chunks * E;
  double bytes = (double)T * E * (4 + 4 + 4 + (dres ? 4 : 0) + (dx_bf16 ? 2 : 0)) + 8.0 * T;
  const bool sum = dx_colsum != nullptr;
  LaunchScope sc(NNT_K_LN_BWD, stream, bytes, 0, 2);
  __nv_bfloat16* d16 = (__nv_bfloat16*)dx_bf16;
  if (nvw > 0) {
    const size_t smem_red = (size_t)kRowsWarps * (sum ? 3 : 2) * E * sizeof(float);  // <= 72 KB (E <= 1024)
    auto run = [&](auto kern) -> nnt_status {
      if (smem_red > 48 * 1024)
        NNT_CUDA_TRY(set_max_dyn_smem(kern, (int)smem_red));
      NNT_CUDA_TRY(::nnt::launch(kern, dim3((unsigned)chunks), dim3(32 * kRowsWarps), smem_red, stream, dy, lddy, x,
                                 ldx, mean, rstd, gamma, T, (int)E, rows_per_cta, dres, dx, lddx, d16, pg, pb, ps));
      return NNT_OK;
    };
#define NNT_LNBR(N) \
  case N: NNT_TRY(sum ? run(ln_bwd_rows<N, true>) : run(ln_bwd_rows<N, false>)); break;
    switch (nvw) { NNT_LNBR(1) NNT_LNBR(2) NNT_LNBR(4) NNT_LNBR(6) NNT_LNBR(8) }
#undef NNT_LNBR
  } else if (E <= 2048 && ln_bwd_ring_on() && (ldx * 4) % 16 == 0 && (lddy * 4) % 16 == 0 && aligned16(x) &&
             aligned16(dy)) {
    // rows streamed into shared-memory rings by bulk copies (16-byte aligned rows)
    const int NV = (int)((E / 4 + 32 * kRingG - 1) / (32 * kRingG));
    const size_t smem_ring = (size_t)kRingGroups * kRing * 3 * E * sizeof(float);  // <= 192 KB
    auto run = [&](auto kern) -> nnt_status {
      NNT_CUDA_TRY(set_max_dyn_smem(kern, (int)smem_ring));
      NNT_CUDA_TRY(::nnt::launch(kern, dim3((unsigned)chunks), dim3(32 * kRingG * kRingGroups), smem_ring, stream, dy,
                                 lddy, x, ldx, mean, rstd, gamma, T, (int)E, rows_per_cta, dres, dx, lddx, d16, pg, pb,
                                 ps));
      return NNT_OK;
    };
    if (NV == 3)
      NNT_TRY(sum ? run(ln_bwd_ring<3, true>) : run(ln_bwd_ring<3, false>));
    else
      NNT_TRY(sum ? run(ln_bwd_ring<4, true>) : run(ln_bwd_ring<4, false>));
  } else {
    int G = 0, NV = 0;
    pick_groups(E, &G, &NV);
    const size_t smem_red = (size_t)(kGrpWarps / G) * (sum ? 3 : 2) * E * sizeof(float);  // <= 64 KB
    auto run = [&](auto kern) -> nnt_status {
      NNT_CUDA_TRY(set_max_dyn_smem(kern, (int)smem_red));
      NNT_CUDA_TRY(::nnt::launch(kern, dim3((unsigned)chunks), dim3(32 * kGrpWarps), smem_red, stream, dy, lddy, x,
                                 ldx, mean, rstd, gamma, T, (int)E, rows_per_cta, dres, dx, lddx, d16, pg, pb, ps));
      return NNT_OK;
    };
#define NNT_LNBG(GG, N)                                                                              \
  if (G == GG && NV == N) {                                                                          \
    NNT_TRY(sum ? run(ln_bwd_groups<N, GG, true>) : run(ln_bwd_groups<N, GG, false>));               \
  } else
    NNT_LNBG(4, 3) NNT_LNBG(4, 4) NNT_LNBG(8, 3) NNT_LNBG(8, 4) NNT_LNBG(8, 5) NNT_LNBG(8, 6) NNT_LNBG(8, 7)
    NNT_LNBG(8, 8)
    return fail(NNT_ERR_UNSUPPORTED, "nnt_layernorm_bwd: unsupported E");
#undef NNT_LNBG
  }
  NNT_TRY(check_launch("layernorm_bwd"));
  if (sum)
    launch_column_merge3(pg, chunks * E, chunks, E, dgamma, dbeta, dx_colsum, accumulate_params, stream);
  else
    launch_column_merge2(pg, chunks * E, chunks, E, dgamma, dbeta, accumulate_params, stream);
  return check_launch("layernorm_bwd merge");
}

}  // extern "C"
