// nnt_tile_gemm: argument validation and dispatch (P:150-153 linear layer,
// P:181 attention products).  fp32 operands -> SIMT fp32 path; bf16 operands
// -> tcgen05 tensor-core path.  There is no other route and no fallback.
#include "gemm_common.cuh"

using namespace nnt;

extern "C" size_t nnt_tile_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int c_dtype, int act, int causal,
                                                int64_t batch_items) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.c_dtype = c_dtype;
  g.act = act;
  g.causal = causal;
  g.batch0 = batch_items > 0 ? batch_items : 1;
  g.batch1 = 1;
  // split partials of C, of the a_rowsum row sums (R27), then the in-kernel reduce's counters;
  // or, for a GEMM the stream-K schedule can take, its partial slots and flags (the larger)
  const size_t split = splitk_workspace_bytes(g, gemm_tc_splits(g));
  const bool sk = sk_on() && g.batch0 == 1 && causal == NNT_CAUSAL_NONE &&
                  (act == NNT_ACT_NONE || act == NNT_ACT_GELU || act == NNT_ACT_GELU_BWD);
  const size_t skb = sk ? sk_workspace_bytes() : 0;
  return split > skb ? split : skb;
}

extern "C" nnt_status nnt_tile_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const int64_t* batch,
                                    float alpha, const void* A, int a_dtype, int64_t lda, const int64_t* stride_a,
                                    const void* B, int b_dtype, int64_t ldb, const int64_t* stride_b, float beta,
                                    void* C, int c_dtype, int64_t ldc, const int64_t* stride_c, const int64_t* tile,
                                    const nnt_epilogue* epi, nnt_stream_t stream) {
  const bool stats_only = epi && epi->act == NNT_ACT_ROWSTATS;  // C is not written
  NNT_REQUIRE(A && B && (C || stats_only), NNT_ERR_NULL, "nnt_tile_gemm: NULL operand");
  NNT_REQUIRE(!stats_only || !C, NNT_ERR_ARG, "nnt_tile_gemm: ROWSTATS writes no C (pass NULL)");
  NNT_REQUIRE(trans_a == NNT_NOTRANS || trans_a == NNT_TRANS, NNT_ERR_ARG, "nnt_tile_gemm: trans_a=%d", trans_a);
  NNT_REQUIRE(trans_b == NNT_NOTRANS || trans_b == NNT_TRANS, NNT_ERR_ARG, "nnt_tile_gemm: trans_b=%d", trans_b);
  NNT_REQUIRE(M > 0 && N > 0 && K > 0, NNT_ERR_SHAPE, "nnt_tile_gemm: M=%lld N=%lld K=%lld", (long long)M,
              (long long)N, (long long)K);
  NNT_REQUIRE(valid_dtype(a_dtype) && a_dtype == b_dtype && valid_dtype(c_dtype), NNT_ERR_DTYPE,
              "nnt_tile_gemm: dtypes A=%d B=%d C=%d (A and B must match)", a_dtype, b_dtype, c_dtype);
  int64_t b0 = batch ? batch[0] : 1, b1 = batch ? batch[1] : 1;
  NNT_REQUIRE(b0 > 0 && b1 > 0, NNT_ERR_SHAPE, "nnt_tile_gemm: batch {%lld,%lld}", (long long)b0, (long long)b1);
  NNT_REQUIRE(lda >= (trans_a == NNT_NOTRANS ? K : M), NNT_ERR_SHAPE, "nnt_tile_gemm: lda=%lld too small",
              (long long)lda);
  NNT_REQUIRE(ldb >= (trans_b == NNT_NOTRANS ? N : K), NNT_ERR_SHAPE, "nnt_tile_gemm: ldb=%lld too small",
              (long long)ldb);
  NNT_REQUIRE(stats_only || ldc >= N, NNT_ERR_SHAPE, "nnt_tile_gemm: ldc=%lld < N", (long long)ldc);
  if (tile) {
    NNT_REQUIRE(tile[0] > 0 && tile[1] > 0 && tile[2] > 0, NNT_ERR_TILE, "nnt_tile_gemm: tile must be positive");
  }
  GemmArgs g{};
  g.ta = trans_a;
  g.tb = trans_b;
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch0 = b0;
  g.batch1 = b1;
  g.alpha = alpha;
  g.beta = beta;
  g.A = A;
  g.lda = lda;
  g.sa0 = stride_a ? stride_a[0] : 0;
  g.sa1 = stride_a ? stride_a[1] : 0;
  g.B = B;
  g.ldb = ldb;
  g.sb0 = stride_b ? stride_b[0] : 0;
  g.sb1 = stride_b ? stride_b[1] : 0;
  g.C = C;
  g.ldc = ldc;
  g.sc0 = stride_c ? stride_c[0] : 0;
  g.sc1 = stride_c ? stride_c[1] : 0;
  g.c_dtype = c_dtype;
  g.in_dtype = a_dtype;
  g.causal = NNT_CAUSAL_NONE;
  if (epi) {
    NNT_REQUIRE(epi->act >= NNT_ACT_NONE && epi->act <= NNT_ACT_SOFTMAX, NNT_ERR_ARG, "nnt_tile_gemm: act=%d",
                epi->act);
    const bool sm = epi->act == NNT_ACT_ROWSTATS || epi->act == NNT_ACT_SOFTMAX;
    NNT_REQUIRE(!sm || (a_dtype == NNT_BF16 && epi->row_stats && !epi->bias && !epi->residual && beta == 0.f &&
                        alpha > 0.f &&
                        (epi->act == NNT_ACT_ROWSTATS || c_dtype == NNT_BF16) &&
                        (epi->causal == NNT_CAUSAL_NONE || epi->causal == NNT_CAUSAL_OUT_LOWER)),
                NNT_ERR_UNSUPPORTED,
                "nnt_tile_gemm: ROWSTATS/SOFTMAX epilogues need bf16 operands, row_stats, alpha > 0, no bias/residual/beta, "
                "bf16 C (SOFTMAX), causal NONE or OUT_LOWER");
    NNT_REQUIRE(epi->act != NNT_ACT_SOFTMAX_BWD || (a_dtype == NNT_BF16 && epi->rowvec && epi->aux),
                NNT_ERR_UNSUPPORTED, "nnt_tile_gemm: SOFTMAX_BWD epilogue needs bf16 operands, aux (P) and rowvec (D)");
    NNT_REQUIRE(epi->causal >= NNT_CAUSAL_NONE && epi->causal <= NNT_CAUSAL_A_UPPER, NNT_ERR_ARG,
                "nnt_tile_gemm: causal=%d", epi->causal);
    NNT_REQUIRE(epi->act == NNT_ACT_NONE || sm || epi->aux, NNT_ERR_NULL, "nnt_tile_gemm: GELU epilogue needs aux");
    NNT_REQUIRE(!epi->residual || epi->ld_residual >= N, NNT_ERR_SHAPE, "nnt_tile_gemm: ld_residual");
    NNT_REQUIRE(!epi->aux || epi->ld_aux >= N, NNT_ERR_SHAPE, "nnt_tile_gemm: ld_aux");
    NNT_REQUIRE((!epi->residual && (!epi->aux || epi->act == NNT_ACT_SOFTMAX_BWD)) || (b0 == 1 && b1 == 1),
                NNT_ERR_UNSUPPORTED, "nnt_tile_gemm: residual/GELU-aux epilogues are for unbatched GEMMs");
    g.bias = epi->bias;
    g.residual = epi->residual;
    g.ld_res = epi->ld_residual;
    g.act = epi->act;
    g.aux = epi->aux;
    g.ld_aux = epi->ld_aux;
    g.causal = epi->causal;
    g.workspace = epi->workspace;
    g.workspace_bytes = epi->workspace_bytes;
    g.row_stats = epi->row_stats;
    g.ld_stats = epi->ld_row_stats;
    g.rowvec = epi->rowvec;
    g.rowscale = epi->rowscale;
    g.a_rowsum = epi->a_rowsum;
    if (epi->scatter) {  // R35 tensor-parallel row scatter
      const nnt_tp_comm* cm = epi->scatter;
      NNT_REQUIRE(cm->R >= 1 && cm->R <= NNT_TP_MAX && cm->rank >= 0 && cm->rank < cm->R, NNT_ERR_ARG,
                  "nnt_tile_gemm: scatter R=%d rank=%d", cm->R, cm->rank);
      NNT_REQUIRE(c_dtype == NNT_F32 && b0 == 1 && b1 == 1 && M == cm->rows && N == cm->cols && ldc == N &&
                      beta == 0.f && epi->act == NNT_ACT_NONE && !epi->a_rowsum && !epi->row_stats,
                  NNT_ERR_UNSUPPORTED,
                  "nnt_tile_gemm: scatter needs fp32 C, unbatched, M == rows, N == ldc == cols, beta 0, no activation");
      g.scat_R = cm->R;
      g.scat_rank = cm->rank;
      g.scat_rows = (cm->rows + cm->R - 1) / cm->R;
      for (int o = 0; o < cm->R; ++o) {
        NNT_REQUIRE(cm->recv[o], NNT_ERR_NULL, "nnt_tile_gemm: scatter recv[%d] NULL", o);
        g.scat[o] = cm->recv[o];
      }
      g.workspace = nullptr;  // no split-K / stream-K partials
      g.workspace_bytes = 0;
    }
    NNT_REQUIRE(!epi->a_rowsum || (a_dtype == NNT_BF16 && b0 == 1 && b1 == 1 && epi->causal == NNT_CAUSAL_NONE &&
                                   epi->act == NNT_ACT_NONE && !epi->row_stats),
                NNT_ERR_UNSUPPORTED,
                "nnt_tile_gemm: a_rowsum needs bf16 operands, an unbatched non-causal GEMM, no activation");
    NNT_REQUIRE(!epi->row_stats || sm || (a_dtype == NNT_BF16 && c_dtype == NNT_F32 && epi->act == NNT_ACT_NONE &&
                                    epi->ld_row_stats >= (N + 31) / 32 &&
                                    (epi->causal == NNT_CAUSAL_NONE || epi->causal == NNT_CAUSAL_OUT_LOWER)),
                NNT_ERR_UNSUPPORTED,
                "nnt_tile_gemm: row_stats needs bf16 operands, fp32 C, no activation, ld >= ceil(N/32)");
  }
  const double frac = g.causal == NNT_CAUSAL_NONE ? 1.0 : 0.5;
  const double flops = 2.0 * (double)M * N * K * b0 * b1 * frac;
  const double es = (double)dtype_size(a_dtype);
  const double c_bytes = stats_only ? 0.0
                                    : (double)M * N * dtype_size(c_dtype) * b0 * b1 *
                                          (g.causal == NNT_CAUSAL_OUT_LOWER ? 0.5 : 1.0) * (beta != 0.f ? 2.0 : 1.0);
  const bool sm_act = g.act == NNT_ACT_ROWSTATS || g.act == NNT_ACT_SOFTMAX;
  const double bytes = ((double)M * K * es + (double)K * N * es) * b0 * b1 * (g.causal == NNT_CAUSAL_NONE ? 1.0 : 0.5) +
                       c_bytes + (g.residual ? 4.0 * M * N : 0.0) +
                       (g.aux ? (double)M * N * dtype_size(c_dtype) : 0.0) + (sm_act ? 8.0 * M * b0 * b1 : 0.0) +
                       (g.a_rowsum ? 4.0 * M * (beta != 0.f ? 2.0 : 1.0) : 0.0);
  if (a_dtype == NNT_F32) {
    LaunchScope sc(NNT_K_GEMM_SIMT, stream, bytes, flops);
    return gemm_simt_launch(g, stream);
  }
  LaunchScope sc(b0 * b1 > 1 ? NNT_K_GEMM_TC_ATTN : NNT_K_GEMM_TC, stream, bytes, flops);
  int kernels = 1;
  const nnt_status st = gemm_tc_launch(g, stream, &kernels);
  if (kernels > 1) sc.add_kernels(kernels - 1);
  return st;
}
