// fp32 SIMT GEMM (the fp32 path, R15: true FFMA, not tf32 — tf32's 10-bit
// mantissa cannot meet rel 1e-4).  64x64x16 CTA tiles, 256 threads, 4x4
// outputs per thread, both operand majors via strided smem fills.  Causal
// block skipping per nnt_causal.  Used for the tiny parity config; the bf16
// path runs on tcgen05 (gemm_tc.cu).
#include "gemm_common.cuh"

namespace nnt {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <typename TC>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(GemmArgs g) {
  NNT_PDL_ENTRY();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int64_t bz = blockIdx.z;
  const int64_t p = bz / g.batch1, q = bz % g.batch1;
  const float* A = (const float*)g.A + p * g.sa0 + q * g.sa1;
  const float* B = (const float*)g.B + p * g.sb0 + q * g.sb1;
  TC* C = (TC*)g.C + p * g.sc0 + q * g.sc1;
  TC* aux = (TC*)g.aux;
  if (aux) aux += p * g.sc0 + q * g.sc1;  // aux shares C's batch strides
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (g.causal == NNT_CAUSAL_OUT_LOWER && n0 > m0 + BM - 1) return;
  int64_t k_begin = 0, k_end = g.K;
  if (g.causal == NNT_CAUSAL_A_LOWER) k_end = min(g.K, m0 + BM);
  if (g.causal == NNT_CAUSAL_A_UPPER) k_begin = min(g.K, m0);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int64_t k0 = k_begin; k0 < k_end; k0 += BK) {
    // A tile: op(A)[m0+mi][k0+ki]
    for (int e = threadIdx.x; e < BM * BK; e += NT) {
      int mi, ki;
      if (g.ta == NNT_NOTRANS) { ki = e % BK; mi = e / BK; } else { mi = e % BM; ki = e / BM; }
      int64_t gi = m0 + mi, gk = k0 + ki;
      float v = 0.f;
      if (gi < g.M && gk < k_end) v = g.ta == NNT_NOTRANS ? A[gi * g.lda + gk] : A[gk * g.lda + gi];
      As[ki][mi] = v;
    }
    for (int e = threadIdx.x; e < BN * BK; e += NT) {
      int ni, ki;
      if (g.tb == NNT_NOTRANS) { ni = e % BN; ki = e / BN; } else { ki = e % BK; ni = e / BK; }
      int64_t gj = n0 + ni, gk = k0 + ki;
      float v = 0.f;
      if (gj < g.N && gk < k_end) v = g.tb == NNT_NOTRANS ? B[gk * g.ldb + gj] : B[gj * g.ldb + gk];
      Bs[ki][ni] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int64_t i = m0 + ty * 4 + r, j = n0 + tx * 4 + c;
      if (i < g.M && j < g.N) epilogue_store<TC>(g, C, aux, i, j, acc[r][c]);
    }
}

}  // namespace

nnt_status gemm_simt_launch(const GemmArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM), (unsigned)(a.batch0 * a.batch1));
  NNT_REQUIRE(grid.y <= 65535 && grid.z <= 65535, NNT_ERR_UNSUPPORTED, "gemm_simt: grid too large");
  if (a.c_dtype == NNT_F32)
    ::nnt::launch(gemm_simt_kernel<float>, grid, NT, 0, s, a);
  else
    ::nnt::launch(gemm_simt_kernel<__nv_bfloat16>, grid, NT, 0, s, a);
  return check_launch("gemm_simt");
}

}  // namespace nnt
