// nnt_block_fwd / nnt_block_bwd: execute the lowered tile-task DAG of one
// pre-LN GPT-2 block (reading R1) on one stream.  Every launch group of the
// plan (dag.cpp) maps to one kernel launch that executes all of that group's
// tile tasks.  Workspace layout ("saved" per layer, "scratch" shared) is
// computed here; the caller owns the memory.
#include <cmath>

#include "dag.h"
#include "nnt_internal.h"

namespace nnt {
namespace {

struct Layout {
  // saved (per layer)
  size_t mean1, rstd1, h1, qkv, P, stats, O, x1, mean2, rstd2, h2, u, g, saved_bytes;
  // scratch
  size_t scores, dvec, dy16, du, dh, dx1, dx116, dO, dA, dqkv, colsum, colsum2, lnscr, gemm_ws, sk_ws, scratch_bytes;
  size_t colsum_bytes, lnscr_bytes, gemm_ws_bytes, sk_ws_bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// H, F: the heads and FFN width this block instance computes (all of them, or one tensor-parallel
// shard's, nnt_block_tp); Ea = H * Dh is its attention width.
Layout make_layout(const nnt_block_cfg& c, int64_t H_l, int64_t F_l) {
  const size_t T = c.B * c.S, E = c.E, F = F_l, H = H_l, S = c.S, B = c.B, Ea = H * (c.E / c.H);
  const size_t dt = c.dtype == NNT_BF16 ? 2 : 4;
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  L.mean1 = take(4 * T);
  L.rstd1 = take(4 * T);
  L.h1 = take(dt * T * E);
  L.qkv = take(dt * T * 3 * Ea);
  L.P = take(dt * B * H * S * S);
  L.stats = take(4 * 2 * B * H * S);
  L.O = take(dt * T * Ea);
  L.x1 = take(4 * T * E);
  L.mean2 = take(4 * T);
  L.rstd2 = take(4 * T);
  L.h2 = take(dt * T * E);
  L.u = take(dt * T * F);
  L.g = take(dt * T * F);
  L.saved_bytes = o;
  o = 0;
  // fp32 path: the materialised scores; the bf16 path keeps score tiles on chip (R26)
  L.scores = take(c.dtype == NNT_BF16 ? 0 : 4 * B * H * S * S);
  L.dvec = take(c.dtype == NNT_BF16 ? 4 * B * H * S : 0);  // D = rowdot(dO, O) (bf16 path)
  L.dy16 = take(dt * T * E);
  L.du = take(dt * T * F);
  L.dh = take(4 * T * E);
  L.dx1 = take(4 * T * E);
  L.dx116 = take(dt * T * E);
  L.dO = take(dt * T * Ea);
  L.dA = take(dt * B * H * S * S);
  L.dqkv = take(dt * T * 3 * Ea);
  L.colsum_bytes = 0;
  for (size_t n : {E, F, 3 * Ea}) {
    size_t cs = nnt_bias_grad_scratch_bytes(T, n);
    if (cs > L.colsum_bytes) L.colsum_bytes = cs;
  }
  L.colsum = take(L.colsum_bytes);
  L.colsum2 = take(L.colsum_bytes);  // the side stream's column sums (FC_DB, OUT_DB, QKV_DB)
  L.lnscr_bytes = nnt_layernorm_bwd_scratch_bytes(T, E);
  L.lnscr = take(L.lnscr_bytes);
  // split-K partials of the four dW GEMMs ([3E x E], [E x E], [4E x E], [E x 4E], K = T)
  L.gemm_ws_bytes = 0;
  if (c.dtype == NNT_BF16) {
    const size_t shapes[4][2] = {{3 * Ea, E}, {E, Ea}, {F, E}, {E, F}};
    for (auto& sh : shapes) {
      size_t b = nnt_tile_gemm_workspace_bytes((int64_t)sh[0], (int64_t)sh[1], (int64_t)T, NNT_F32, NNT_ACT_NONE,
                                               NNT_CAUSAL_NONE, 1);
      if (b > L.gemm_ws_bytes) L.gemm_ws_bytes = b;
    }
  }
  L.gemm_ws = take(L.gemm_ws_bytes);
  // the main stream's projection GEMMs (forward and dX): stream-K partial slots and flags (the dW
  // GEMMs, which may run concurrently on the side stream, keep gemm_ws)
  L.sk_ws_bytes = c.dtype == NNT_BF16 ? nnt_tile_gemm_workspace_bytes((int64_t)T, (int64_t)E, (int64_t)E, NNT_BF16,
                                                                      NNT_ACT_NONE, NNT_CAUSAL_NONE, 1)
                                      : 0;
  L.sk_ws = take(L.sk_ws_bytes);
  L.scratch_bytes = o;
  return L;
}

nnt_status check_cfg(const nnt_block_cfg* c) {
  NNT_REQUIRE(c, NNT_ERR_NULL, "block: NULL cfg");
  NNT_REQUIRE(c->E > 0 && c->H > 0 && c->S > 0 && c->B > 0 && c->E % c->H == 0, NNT_ERR_SHAPE,
              "block: bad shape E=%lld H=%lld S=%lld B=%lld", (long long)c->E, (long long)c->H, (long long)c->S,
              (long long)c->B);
  NNT_REQUIRE(c->tile_e > 0 && c->tile_f > 0 && c->tile_s > 0 && c->tile_t > 0, NNT_ERR_TILE,
              "block: tiles must be positive");
  NNT_REQUIRE(valid_dtype(c->dtype), NNT_ERR_DTYPE, "block: dtype %d", c->dtype);
  NNT_REQUIRE(c->E % 8 == 0 && c->S % 8 == 0 && (c->E / c->H) % 8 == 0, NNT_ERR_ALIGN,
              "block: E, S and head size must be multiples of 8");
  NNT_REQUIRE(c->S <= 2048, NNT_ERR_UNSUPPORTED, "block: S > 2048 unsupported (materialised softmax rows)");
  return NNT_OK;
}

struct Ctx {
  const nnt_block_cfg& c;
  int64_t T, E, F, H, S, B, Dh;
  int64_t Ea;     // attention width H * Dh (= E unless a tensor-parallel shard)
  bool add_bias;  // OUT / PROJ add the replicated bias and the residual (false on all but one TP shard)
  float* x1;      // the attention sub-block's output x1 (in `saved`, or the caller's for nnt_block_tp)
  float* dh;      // dL/dh2, then dL/dh1 (in `scratch`, or the caller's for nnt_block_tp)
  int dt;
  float inv_sqrt_dh;
  int64_t tile_lin[3];
  uint8_t* sv;
  uint8_t* sc;
  Layout L;
  cudaStream_t st;
  cudaStream_t side;  // nnt_block_bwd_streams: weight/bias-gradient ops run here (or NULL)
  const nnt_block_bwd_links* links;  // nnt_block_bwd_streams: fused cross-layer bias sums (or NULL)
  bool ln_rows;                      // the LayerNorm backward fuses the column sums of dx (every E)
  bool fused_attn;                   // bf16, h = 64, S % 128 == 0: the fused attention tile kernels (R33)
  const nnt_tp_comm* comm;           // nnt_block_tp with a comm: the partial-producing GEMMs scatter (R35)
  template <typename P>
  P* s(size_t off) const { return reinterpret_cast<P*>(sv + off); }
  template <typename P>
  P* k(size_t off) const { return reinterpret_cast<P*>(sc + off); }
};

nnt_status gemm(const Ctx& x, int ta, int tb, int64_t M, int64_t N, int64_t K, const int64_t* batch, float alpha,
                const void* A, int64_t lda, const int64_t* sa, const void* B, int64_t ldb, const int64_t* sb,
                float beta, void* C, int cdt, int64_t ldc, const int64_t* sc, const nnt_epilogue* epi) {
  nnt_epilogue e{};
  if (!batch && x.L.sk_ws_bytes && !(epi && epi->workspace)) {  // unbatched main-stream GEMM: stream-K slots
    if (epi) e = *epi;
    e.workspace = x.k<void>(x.L.sk_ws);
    e.workspace_bytes = x.L.sk_ws_bytes;
    epi = &e;
  }
  return nnt_tile_gemm(ta, tb, M, N, K, batch, alpha, A, x.dt, lda, sa, B, x.dt, ldb, sb, beta, C, cdt, ldc, sc,
                       x.tile_lin, epi, x.st);
}

nnt_status run_fwd_op(const Ctx& x, int op, const nnt_block_params* p, const float* xin, float* y) {
  const int64_t T = x.T, E = x.E, F = x.F, S = x.S, H = x.H, B = x.B, Dh = x.Dh, Ea = x.Ea;
  const int dt = x.dt;
  const int64_t batch[2] = {B, H};
  nnt_epilogue e{};
  switch (op) {
    case NNT_OP_LN1:
      return nnt_layernorm_fwd(xin, T, E, E, x.c.tile_e, p->ln1_g, p->ln1_b, x.c.ln_eps, x.s<void>(x.L.h1), dt, E,
                               x.s<float>(x.L.mean1), x.s<float>(x.L.rstd1), x.st);
    case NNT_OP_QKV:
      e.bias = p->b_qkv;
      return gemm(x, NNT_NOTRANS, NNT_TRANS, T, 3 * Ea, E, nullptr, 1.f, x.s<void>(x.L.h1), E, nullptr, p->w_qkv, E,
                  nullptr, 0.f, x.s<void>(x.L.qkv), dt, 3 * Ea, nullptr, &e);
    case NNT_OP_SCORES: {
      const size_t es = dt == NNT_BF16 ? 2 : 4;
      const int64_t sq[2] = {S * 3 * Ea, Dh}, ssc[2] = {H * S * S, S * S};
      e.causal = x.c.causal ? NNT_CAUSAL_OUT_LOWER : NNT_CAUSAL_NONE;
      uint8_t* q = x.s<uint8_t>(x.L.qkv);
      if (x.fused_attn && nnt_attention_stats_enabled())  // R26 in the fused attention pipeline
        return nnt_attention_stats(x.s<void>(x.L.qkv), B, S, H, Dh, x.inv_sqrt_dh, x.c.causal, x.s<float>(x.L.stats),
                                   x.st);
      if (dt == NNT_BF16) {
        // R26: the score tiles stay on chip; subroutine 1 and its aggregation over all key tiles
        // of a row run in the GEMM epilogue, producing the slice stats directly
        e.act = NNT_ACT_ROWSTATS;
        e.row_stats = x.s<float>(x.L.stats);
        return gemm(x, NNT_NOTRANS, NNT_TRANS, S, S, Dh, batch, x.inv_sqrt_dh, q, 3 * Ea, sq, q + es * Ea, 3 * Ea,
                    sq, 0.f, nullptr, NNT_F32, S, ssc, &e);
      }
      return gemm(x, NNT_NOTRANS, NNT_TRANS, S, S, Dh, batch, x.inv_sqrt_dh, q, 3 * Ea, sq, q + es * Ea, 3 * Ea, sq,
                  0.f, x.k<float>(x.L.scores), NNT_F32, S, ssc, &e);
    }
    case NNT_OP_MAXSUMEXP:  // fp32 path only (the bf16 path fuses it into NNT_OP_SCORES)
      return nnt_maxsumexp(x.k<float>(x.L.scores), B * H * S, S, S, x.c.tile_s, x.c.causal, S,
                           x.s<float>(x.L.stats), 0, x.st);
    case NNT_OP_SOFTMAX:
      if (x.fused_attn)  // R33: subroutine 2 and P V in one tile pass; P stored once, never re-read
        return nnt_attention_fwd_pv(x.s<void>(x.L.qkv), B, S, H, Dh, x.inv_sqrt_dh, x.c.causal, x.s<float>(x.L.stats),
                                    x.s<void>(x.L.P), x.s<void>(x.L.O), x.st);
      if (dt == NNT_BF16) {
        // R26: subroutine 2 on recomputed score tiles (same MMA order as the stats pass), P in bf16
        const int64_t sq[2] = {S * 3 * Ea, Dh}, sp[2] = {H * S * S, S * S};
        e.causal = x.c.causal ? NNT_CAUSAL_OUT_LOWER : NNT_CAUSAL_NONE;
        e.act = NNT_ACT_SOFTMAX;
        e.row_stats = x.s<float>(x.L.stats);
        uint8_t* q = x.s<uint8_t>(x.L.qkv);
        return gemm(x, NNT_NOTRANS, NNT_TRANS, S, S, Dh, batch, x.inv_sqrt_dh, q, 3 * Ea, sq, q + 2 * Ea, 3 * Ea, sq,
                    0.f, x.s<void>(x.L.P), dt, S, sp, &e);
      }
      return nnt_softmax(x.k<float>(x.L.scores), B * H * S, S, S, x.c.tile_s, x.c.causal, S, x.s<float>(x.L.stats),
                         x.s<void>(x.L.P), dt, S, x.st);
    case NNT_OP_PV: {
      if (x.fused_attn) return NNT_OK;  // formed with P in NNT_OP_SOFTMAX
      const size_t es = dt == NNT_BF16 ? 2 : 4;
      const int64_t sp[2] = {H * S * S, S * S}, sv[2] = {S * 3 * Ea, Dh}, so[2] = {S * Ea, Dh};
      e.causal = x.c.causal ? NNT_CAUSAL_A_LOWER : NNT_CAUSAL_NONE;
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, S, Dh, S, batch, 1.f, x.s<void>(x.L.P), S, sp,
                  x.s<uint8_t>(x.L.qkv) + es * 2 * Ea, 3 * Ea, sv, 0.f, x.s<void>(x.L.O), dt, Ea, so, &e);
    }
    case NNT_OP_OUT:
      if (x.add_bias) {
        e.bias = p->b_o;
        e.residual = xin;
        e.ld_residual = E;
      }
      e.scatter = x.comm;  // tensor-parallel partial x1 -> its owners' receive slots (R35)
      return gemm(x, NNT_NOTRANS, NNT_TRANS, T, E, Ea, nullptr, 1.f, x.s<void>(x.L.O), Ea, nullptr, p->w_o, Ea,
                  nullptr, 0.f, x.x1, NNT_F32, E, nullptr, &e);
    case NNT_OP_LN2:
      return nnt_layernorm_fwd(x.x1, T, E, E, x.c.tile_e, p->ln2_g, p->ln2_b, x.c.ln_eps,
                               x.s<void>(x.L.h2), dt, E, x.s<float>(x.L.mean2), x.s<float>(x.L.rstd2), x.st);
    case NNT_OP_FC:
      e.bias = p->b_fc;
      e.act = NNT_ACT_GELU;
      e.aux = x.s<void>(x.L.u);
      e.ld_aux = F;
      return gemm(x, NNT_NOTRANS, NNT_TRANS, T, F, E, nullptr, 1.f, x.s<void>(x.L.h2), E, nullptr, p->w_fc, E,
                  nullptr, 0.f, x.s<void>(x.L.g), dt, F, nullptr, &e);
    case NNT_OP_PROJ:
      if (x.add_bias) {
        e.bias = p->b_pr;
        e.residual = x.x1;
        e.ld_residual = E;
      }
      e.scatter = x.comm;
      return gemm(x, NNT_NOTRANS, NNT_TRANS, T, E, F, nullptr, 1.f, x.s<void>(x.L.g), F, nullptr, p->w_pr, F,
                  nullptr, 0.f, y, NNT_F32, E, nullptr, &e);
  }
  return fail(NNT_ERR_ARG, "block fwd: unexpected op in plan");
}

nnt_status run_bwd_op(const Ctx& x, int op, const nnt_block_params* p, const float* xin, const float* dy, float* dx,
                      const nnt_block_grads* g, int acc) {
  const int64_t T = x.T, E = x.E, F = x.F, S = x.S, H = x.H, B = x.B, Dh = x.Dh, Ea = x.Ea;
  const int dt = x.dt;
  const bool bf = dt == NNT_BF16;
  const size_t es = bf ? 2 : 4;
  const int64_t batch[2] = {B, H};
  const float beta = acc ? 1.f : 0.f;
  // GEMM operand views of dy and dx1 (bf16 copies on the bf16 path)
  // the layer above's LayerNorm already made sum_t dy (into g->b_pr) and the bf16 copy of dy
  const bool dy_done = x.links && x.links->dy_colsum_done && (!bf || x.links->dy_bf16);
  const void* dyA = bf ? (dy_done ? x.links->dy_bf16 : x.k<void>(x.L.dy16)) : (const void*)dy;
  const void* dx1A = bf ? x.k<void>(x.L.dx116) : x.k<void>(x.L.dx1);
  nnt_epilogue e{};
  nnt_epilogue ws{};  // dW GEMMs: split-K partials in the shared scratch
  ws.workspace = x.L.gemm_ws_bytes ? x.k<void>(x.L.gemm_ws) : nullptr;
  ws.workspace_bytes = x.L.gemm_ws_bytes;
  switch (op) {
    case NNT_OP_PROJ_DB:
      if (dy_done) return NNT_OK;  // fused into the layer above's LayerNorm backward
      return nnt_bias_grad(dy, NNT_F32, T, E, E, g->b_pr, acc, bf ? x.k<void>(x.L.dy16) : nullptr,
                           x.k<void>(x.L.colsum), x.L.colsum_bytes, x.st);
    case NNT_OP_PROJ_DW:
      return gemm(x, NNT_TRANS, NNT_NOTRANS, E, F, T, nullptr, 1.f, dyA, E, nullptr, x.s<void>(x.L.g), F, nullptr,
                  beta, g->w_pr, NNT_F32, F, nullptr, &ws);
    case NNT_OP_PROJ_DX:
      e.act = NNT_ACT_GELU_BWD;
      e.aux = x.s<void>(x.L.u);
      e.ld_aux = F;
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, T, F, E, nullptr, 1.f, dyA, E, nullptr, p->w_pr, F, nullptr, 0.f,
                  x.k<void>(x.L.du), dt, F, nullptr, &e);
    case NNT_OP_FC_DB:
      return nnt_bias_grad(x.k<void>(x.L.du), dt, T, F, F, g->b_fc, acc, nullptr, x.k<void>(x.L.colsum2),
                           x.L.colsum_bytes, x.st);
    case NNT_OP_FC_DW:
      return gemm(x, NNT_TRANS, NNT_NOTRANS, F, E, T, nullptr, 1.f, x.k<void>(x.L.du), F, nullptr,
                  x.s<void>(x.L.h2), E, nullptr, beta, g->w_fc, NNT_F32, E, nullptr, &ws);
    case NNT_OP_FC_DX:
      e.scatter = x.comm;  // tensor-parallel partial dL/dh2 (R35)
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, T, E, F, nullptr, 1.f, x.k<void>(x.L.du), F, nullptr, p->w_fc, E,
                  nullptr, 0.f, x.dh, NNT_F32, E, nullptr, x.comm ? &e : nullptr);
    case NNT_OP_LN2_BWD:
      // b_o's gradient sum_t dx1 is the column sum of this LayerNorm's output: fused
      return nnt_layernorm_bwd(x.dh, E, x.x1, E, x.s<float>(x.L.mean2),
                               x.s<float>(x.L.rstd2), p->ln2_g, T, E, dy, x.k<float>(x.L.dx1), E,
                               bf ? x.k<void>(x.L.dx116) : nullptr, g->ln2_g, g->ln2_b, x.ln_rows ? g->b_o : nullptr,
                               acc, x.k<void>(x.L.lnscr), x.L.lnscr_bytes, x.st);
    case NNT_OP_OUT_DB:
      if (x.ln_rows) return NNT_OK;  // fused into NNT_OP_LN2_BWD
      return nnt_bias_grad(x.k<float>(x.L.dx1), NNT_F32, T, E, E, g->b_o, acc, nullptr, x.k<void>(x.L.colsum2),
                           x.L.colsum_bytes, x.st);
    case NNT_OP_OUT_DW:
      return gemm(x, NNT_TRANS, NNT_NOTRANS, E, Ea, T, nullptr, 1.f, dx1A, E, nullptr, x.s<void>(x.L.O), Ea, nullptr,
                  beta, g->w_o, NNT_F32, Ea, nullptr, &ws);
    case NNT_OP_OUT_DX:
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, T, Ea, E, nullptr, 1.f, dx1A, E, nullptr, p->w_o, Ea, nullptr, 0.f,
                  x.k<void>(x.L.dO), dt, Ea, nullptr, nullptr);
    case NNT_OP_ATT_DP: {
      if (x.fused_attn)  // R33: dA (keys-major), dK and dV in one pass over the P tiles
        return nnt_attention_bwd_kv(x.s<void>(x.L.qkv), x.k<void>(x.L.dO), x.s<void>(x.L.P), x.k<float>(x.L.dvec),
                                    B, S, H, Dh, x.inv_sqrt_dh, x.c.causal, x.k<void>(x.L.dA), x.k<void>(x.L.dqkv),
                                    x.st);
      const int64_t so[2] = {S * Ea, Dh}, sv[2] = {S * 3 * Ea, Dh}, sp[2] = {H * S * S, S * S};
      e.causal = x.c.causal ? NNT_CAUSAL_OUT_LOWER : NNT_CAUSAL_NONE;
      if (bf) {  // softmax backward in the epilogue: dA = P * (dO V^T - D) / sqrt(h), straight to bf16
        e.act = NNT_ACT_SOFTMAX_BWD;
        e.aux = x.s<void>(x.L.P);
        e.ld_aux = S;
        e.rowvec = x.k<float>(x.L.dvec);
        e.rowscale = x.inv_sqrt_dh;
        return gemm(x, NNT_NOTRANS, NNT_TRANS, S, S, Dh, batch, 1.f, x.k<void>(x.L.dO), Ea, so,
                    x.s<uint8_t>(x.L.qkv) + es * 2 * Ea, 3 * Ea, sv, 0.f, x.k<void>(x.L.dA), dt, S, sp, &e);
      }
      return gemm(x, NNT_NOTRANS, NNT_TRANS, S, S, Dh, batch, 1.f, x.k<void>(x.L.dO), Ea, so,
                  x.s<uint8_t>(x.L.qkv) + es * 2 * Ea, 3 * Ea, sv, 0.f, x.k<float>(x.L.scores), NNT_F32, S, sp, &e);
    }
    case NNT_OP_ATT_DV: {
      if (x.fused_attn) return NNT_OK;  // formed in NNT_OP_ATT_DP
      const int64_t sp[2] = {H * S * S, S * S}, so[2] = {S * Ea, Dh}, sq[2] = {S * 3 * Ea, Dh};
      e.causal = x.c.causal ? NNT_CAUSAL_A_UPPER : NNT_CAUSAL_NONE;
      return gemm(x, NNT_TRANS, NNT_NOTRANS, S, Dh, S, batch, 1.f, x.s<void>(x.L.P), S, sp, x.k<void>(x.L.dO), Ea, so,
                  0.f, x.k<uint8_t>(x.L.dqkv) + es * 2 * Ea, dt, 3 * Ea, sq, &e);
    }
    case NNT_OP_SOFTMAX_BWD:
      if (bf)  // the reduction D = sum_k P dP via the dO.O identity; dA is formed in the dP GEMM
        return nnt_attn_rowdot(x.k<void>(x.L.dO), x.s<void>(x.L.O), dt, B, S, H, Dh, x.k<float>(x.L.dvec), x.st);
      return nnt_softmax_bwd(x.s<void>(x.L.P), dt, S, x.k<float>(x.L.scores), S, B * H * S, S, x.c.causal, S,
                             x.inv_sqrt_dh, x.k<void>(x.L.dA), dt, S, x.st);
    case NNT_OP_ATT_DQ: {
      const int64_t sp[2] = {H * S * S, S * S}, sq[2] = {S * 3 * Ea, Dh};
      e.causal = x.c.causal ? NNT_CAUSAL_A_LOWER : NNT_CAUSAL_NONE;
      // dQ = dA K (dA query-major, from nnt_attention_bwd_kv or the dP GEMM's softmax-backward epilogue)
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, S, Dh, S, batch, 1.f, x.k<void>(x.L.dA), S, sp,
                  x.s<uint8_t>(x.L.qkv) + es * Ea, 3 * Ea, sq, 0.f, x.k<void>(x.L.dqkv), dt, 3 * Ea, sq, &e);
    }
    case NNT_OP_ATT_DK: {
      if (x.fused_attn) return NNT_OK;  // formed in NNT_OP_ATT_DP
      const int64_t sp[2] = {H * S * S, S * S}, sq[2] = {S * 3 * Ea, Dh};
      e.causal = x.c.causal ? NNT_CAUSAL_A_UPPER : NNT_CAUSAL_NONE;
      return gemm(x, NNT_TRANS, NNT_NOTRANS, S, Dh, S, batch, 1.f, x.k<void>(x.L.dA), S, sp, x.s<void>(x.L.qkv),
                  3 * Ea, sq, 0.f, x.k<uint8_t>(x.L.dqkv) + es * Ea, dt, 3 * Ea, sq, &e);
    }
    case NNT_OP_QKV_DB:
      return nnt_bias_grad(x.k<void>(x.L.dqkv), dt, T, 3 * Ea, 3 * Ea, g->b_qkv, acc, nullptr, x.k<void>(x.L.colsum2),
                           x.L.colsum_bytes, x.st);
    case NNT_OP_QKV_DW:
      return gemm(x, NNT_TRANS, NNT_NOTRANS, 3 * Ea, E, T, nullptr, 1.f, x.k<void>(x.L.dqkv), 3 * Ea, nullptr,
                  x.s<void>(x.L.h1), E, nullptr, beta, g->w_qkv, NNT_F32, E, nullptr, &ws);
    case NNT_OP_QKV_DX:
      e.scatter = x.comm;  // tensor-parallel partial dL/dh1 (R35)
      return gemm(x, NNT_NOTRANS, NNT_NOTRANS, T, E, 3 * Ea, nullptr, 1.f, x.k<void>(x.L.dqkv), 3 * Ea, nullptr,
                  p->w_qkv, E, nullptr, 0.f, x.dh, NNT_F32, E, nullptr, x.comm ? &e : nullptr);
    case NNT_OP_LN1_BWD:
      return nnt_layernorm_bwd(x.dh, E, xin, E, x.s<float>(x.L.mean1), x.s<float>(x.L.rstd1), p->ln1_g,
                               T, E, x.k<float>(x.L.dx1), dx, E, x.links ? x.links->dx_bf16 : nullptr, g->ln1_g,
                               g->ln1_b, x.links && x.ln_rows ? x.links->dx_colsum : nullptr, acc,
                               x.k<void>(x.L.lnscr), x.L.lnscr_bytes, x.st);
  }
  return fail(NNT_ERR_ARG, "block bwd: unexpected op in plan");
}

Ctx make_ctx(const nnt_block_cfg& c, void* saved, void* scratch, cudaStream_t st, const nnt_block_tp* tp = nullptr) {
  Ctx x{c};
  x.T = c.B * c.S;
  x.E = c.E;
  x.F = tp ? tp->ffn : 4 * c.E;
  x.H = tp ? tp->heads : c.H;
  x.S = c.S;
  x.B = c.B;
  x.Dh = c.E / c.H;
  x.dt = c.dtype;
  x.inv_sqrt_dh = (float)(1.0 / std::sqrt((double)x.Dh));
  x.tile_lin[0] = c.tile_t;
  x.tile_lin[1] = c.tile_e;
  x.tile_lin[2] = c.tile_e;
  x.sv = (uint8_t*)saved;
  x.sc = (uint8_t*)scratch;
  x.Ea = x.H * x.Dh;
  x.add_bias = tp ? tp->add_bias != 0 : true;
  x.comm = tp ? tp->comm : nullptr;
  x.L = make_layout(c, x.H, x.F);
  x.x1 = reinterpret_cast<float*>(x.sv + x.L.x1);
  x.dh = reinterpret_cast<float*>(x.sc + x.L.dh);
  x.st = st;
  x.side = nullptr;
  x.links = nullptr;
  x.ln_rows = true;
  const char* attn_e = getenv("NNT_ATTN_FUSED");  // =0: the unfused GEMM sequence (A/B runs, tests)
  const bool attn_env = !(attn_e && attn_e[0] == '0');
  x.fused_attn = attn_env && c.dtype == NNT_BF16 && nnt_attention_fused_supported(c.S, x.Dh);
  return x;
}

// Each op must form exactly one launch group (all its tile tasks independent).
nnt_status check_plan(const BlockPlan* plan) {
  int seen[NNT_OP_COUNT] = {0};
  for (auto& gr : plan->groups) {
    NNT_REQUIRE(++seen[gr.op] == 1, NNT_ERR_UNSUPPORTED, "block plan: op %s spans several levels",
                nnt_op_name(gr.op));
  }
  return NNT_OK;
}

nnt_status check_tp(const nnt_block_cfg* c, const nnt_block_tp* tp) {
  NNT_TRY(check_cfg(c));
  NNT_REQUIRE(tp, NNT_ERR_NULL, "nnt_block_tp: NULL shard descriptor");
  NNT_REQUIRE(tp->heads > 0 && tp->heads <= c->H && tp->ffn > 0 && tp->ffn <= 4 * c->E, NNT_ERR_SHAPE,
              "nnt_block_tp: shard heads=%lld (H=%lld) ffn=%lld (4E=%lld)", (long long)tp->heads, (long long)c->H,
              (long long)tp->ffn, (long long)(4 * c->E));
  NNT_REQUIRE(tp->ffn % 8 == 0, NNT_ERR_ALIGN, "nnt_block_tp: shard ffn width must be a multiple of 8");
  NNT_REQUIRE(tp->add_bias == 0 || tp->add_bias == 1, NNT_ERR_ARG, "nnt_block_tp: add_bias must be 0 or 1");
  NNT_REQUIRE(!tp->comm || (tp->comm->rows == c->B * c->S && tp->comm->cols == c->E), NNT_ERR_SHAPE,
              "nnt_block_tp: comm reduces %lld x %lld, the block's activations are %lld x %lld",
              (long long)(tp->comm ? tp->comm->rows : 0), (long long)(tp->comm ? tp->comm->cols : 0),
              (long long)(c->B * c->S), (long long)c->E);
  return NNT_OK;
}

// The tensor-parallel stages (nnt.h, nnt_block_tp_*): the ops between two reductions over the
// shard group, in an order that respects every dependency of the block DAG.
const int kTpFwd[2][8] = {{NNT_OP_LN1, NNT_OP_QKV, NNT_OP_SCORES, NNT_OP_MAXSUMEXP, NNT_OP_SOFTMAX, NNT_OP_PV,
                           NNT_OP_OUT, -1},
                          {NNT_OP_LN2, NNT_OP_FC, NNT_OP_PROJ, -1}};
const int kTpBwd[3][14] = {{NNT_OP_PROJ_DB, NNT_OP_PROJ_DW, NNT_OP_PROJ_DX, NNT_OP_FC_DB, NNT_OP_FC_DW, NNT_OP_FC_DX,
                            -1},
                           {NNT_OP_LN2_BWD, NNT_OP_OUT_DB, NNT_OP_OUT_DW, NNT_OP_OUT_DX, NNT_OP_SOFTMAX_BWD,
                            NNT_OP_ATT_DP, NNT_OP_SOFTMAX_BWD, NNT_OP_ATT_DV, NNT_OP_ATT_DQ, NNT_OP_ATT_DK,
                            NNT_OP_QKV_DB, NNT_OP_QKV_DW, NNT_OP_QKV_DX, -1},
                           {NNT_OP_LN1_BWD, -1}};

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_block_workspace_size(const nnt_block_cfg* cfg, size_t* saved_bytes, size_t* scratch_bytes) {
  NNT_TRY(check_cfg(cfg));
  NNT_REQUIRE(saved_bytes && scratch_bytes, NNT_ERR_NULL, "nnt_block_workspace_size: NULL output");
  Layout L = make_layout(*cfg, cfg->H, 4 * cfg->E);
  *saved_bytes = L.saved_bytes;
  *scratch_bytes = L.scratch_bytes;
  return NNT_OK;
}

nnt_status nnt_block_tp_workspace_size(const nnt_block_cfg* cfg, const nnt_block_tp* tp, size_t* saved_bytes,
                                      size_t* scratch_bytes) {
  NNT_TRY(check_tp(cfg, tp));
  NNT_REQUIRE(saved_bytes && scratch_bytes, NNT_ERR_NULL, "nnt_block_tp_workspace_size: NULL output");
  Layout L = make_layout(*cfg, tp->heads, tp->ffn);
  *saved_bytes = L.saved_bytes;
  *scratch_bytes = L.scratch_bytes;
  return NNT_OK;
}

nnt_status nnt_block_tp_fwd(const nnt_block_cfg* cfg, const nnt_block_tp* tp, const nnt_block_params* p, int stage,
                            const float* x, float* x1, float* y, void* saved, void* scratch, nnt_stream_t stream) {
  NNT_TRY(check_tp(cfg, tp));
  NNT_REQUIRE(stage == 0 || stage == 1, NNT_ERR_ARG, "nnt_block_tp_fwd: stage %d", stage);
  NNT_REQUIRE(p && x && x1 && saved && scratch && (stage == 0 || y), NNT_ERR_NULL, "nnt_block_tp_fwd: NULL argument");
  Ctx c = make_ctx(*cfg, saved, scratch, stream, tp);
  c.x1 = x1;
  const bool bf = cfg->dtype == NNT_BF16;
  for (const int* op = kTpFwd[stage]; *op >= 0; ++op) {
    if (*op == NNT_OP_MAXSUMEXP && bf) continue;  // fused into the score GEMM on the bf16 path (R26)
    NNT_TRY(run_fwd_op(c, *op, p, x, y));
  }
  return NNT_OK;
}

nnt_status nnt_block_tp_bwd(const nnt_block_cfg* cfg, const nnt_block_tp* tp, const nnt_block_params* p, int stage,
                            const float* x, const float* x1, const void* saved, void* scratch, const float* dy,
                            float* dh, float* dx, const nnt_block_grads* g, int accumulate_grads,
                            nnt_stream_t stream) {
  NNT_TRY(check_tp(cfg, tp));
  NNT_REQUIRE(stage >= 0 && stage <= 2, NNT_ERR_ARG, "nnt_block_tp_bwd: stage %d", stage);
  NNT_REQUIRE(p && x && x1 && saved && scratch && dy && dh && g && (stage < 2 || dx), NNT_ERR_NULL,
              "nnt_block_tp_bwd: NULL argument");
  Ctx c = make_ctx(*cfg, const_cast<void*>(saved), scratch, stream, tp);
  c.x1 = const_cast<float*>(x1);
  c.dh = dh;
  const bool bf = cfg->dtype == NNT_BF16;
  bool seen_dp = false;
  for (const int* op = kTpBwd[stage]; *op >= 0; ++op) {
    if (*op == NNT_OP_ATT_DP) seen_dp = true;
    // softmax backward: before the dP GEMM on the bf16 path (D feeds its epilogue), after it on fp32
    if (*op == NNT_OP_SOFTMAX_BWD && seen_dp == bf) continue;
    NNT_TRY(run_bwd_op(c, *op, p, x, dy, dx, g, accumulate_grads));
  }
  return NNT_OK;
}

nnt_status nnt_block_fwd(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x, float* y, void* saved,
                         void* scratch, nnt_stream_t stream) {
  NNT_TRY(check_cfg(cfg));
  NNT_REQUIRE(p && x && y && saved && scratch, NNT_ERR_NULL, "nnt_block_fwd: NULL argument");
  NNT_REQUIRE(p->ln1_g && p->ln1_b && p->ln2_g && p->ln2_b && p->w_qkv && p->w_o && p->w_fc && p->w_pr && p->b_qkv &&
                  p->b_o && p->b_fc && p->b_pr,
              NNT_ERR_NULL, "nnt_block_fwd: NULL parameter");
  const BlockPlan* plan = block_plan(*cfg, 0);
  NNT_REQUIRE(plan != nullptr, NNT_ERR_SHAPE, "nnt_block_fwd: %s", nnt_last_error());
  NNT_TRY(check_plan(plan));
  Ctx c = make_ctx(*cfg, saved, scratch, stream);
  for (const auto& gr : plan->groups) NNT_TRY(run_fwd_op(c, gr.op, p, x, y));
  return NNT_OK;
}

nnt_status nnt_block_bwd(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x, const void* saved,
                         void* scratch, const float* dy, float* dx, const nnt_block_grads* g, int accumulate_grads,
                         nnt_event_t* grad_ready, nnt_stream_t stream) {
  return nnt_block_bwd_streams(cfg, p, x, saved, scratch, dy, dx, g, accumulate_grads, grad_ready, stream, nullptr,
                               nullptr);
}

nnt_status nnt_block_bwd_streams(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x,
                                 const void* saved, void* scratch, const float* dy, float* dx,
                                 const nnt_block_grads* g, int accumulate_grads, nnt_event_t* grad_ready,
                                 nnt_stream_t stream, nnt_stream_t side_stream, const nnt_block_bwd_links* links) {
  NNT_TRY(check_cfg(cfg));
  NNT_REQUIRE(p && x && saved && scratch && dy && dx && g, NNT_ERR_NULL, "nnt_block_bwd: NULL argument");
  NNT_REQUIRE(g->ln1_g && g->ln1_b && g->ln2_g && g->ln2_b && g->w_qkv && g->w_o && g->w_fc && g->w_pr && g->b_qkv &&
                  g->b_o && g->b_fc && g->b_pr,
              NNT_ERR_NULL, "nnt_block_bwd: NULL gradient");
  NNT_REQUIRE(side_stream == nullptr || side_stream != stream, NNT_ERR_ARG,
              "nnt_block_bwd_streams: side stream must differ from the main stream");
  const BlockPlan* plan = block_plan(*cfg, 1);
  NNT_REQUIRE(plan != nullptr, NNT_ERR_SHAPE, "nnt_block_bwd: %s", nnt_last_error());
  NNT_TRY(check_plan(plan));
  Ctx c = make_ctx(*cfg, const_cast<void*>(saved), scratch, stream);
  NNT_REQUIRE(!links || !links->dx_bf16 || cfg->dtype == NNT_BF16, NNT_ERR_DTYPE,
              "nnt_block_bwd_streams: links.dx_bf16 is for the bf16 path");
  c.links = links;
  cudaStream_t side = (cudaStream_t)side_stream;
  // Ops that only produce weight / bias gradients leave the critical dX chain: with a side
  // stream they run there, each after everything enqueued on the main stream so far (one
  // fork event per batch of side ops), and the main stream joins the side stream at the end.
  // They write disjoint gradients and read buffers the main stream does not overwrite within
  // this call (the side column sums use their own scratch), so results are bitwise unchanged.
  // Which ops: the DAG's sinks that write only parameter gradients (LaunchGroup::side_ok, dag.cpp):
  // the dW GEMMs and the bias column sums that make no copy for a later op.
  auto on_side = [&](const LaunchGroup& gr) { return side != nullptr && gr.side_ok; };
  // fork / join events, one pair per device (events belong to the device current at creation)
  static thread_local cudaEvent_t ev_pool[kMaxDevices][2] = {};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (side) {
    int dev = 0;
    NNT_CUDA_TRY(cudaGetDevice(&dev));
    NNT_REQUIRE(dev >= 0 && dev < kMaxDevices, NNT_ERR_UNSUPPORTED, "nnt_block_bwd_streams: device %d", dev);
    if (!ev_pool[dev][0]) {
      NNT_CUDA_TRY(cudaEventCreateWithFlags(&ev_pool[dev][0], cudaEventDisableTiming));
      NNT_CUDA_TRY(cudaEventCreateWithFlags(&ev_pool[dev][1], cudaEventDisableTiming));
    }
    ev_fork = ev_pool[dev][0];
    ev_join = ev_pool[dev][1];
  }
  Ctx cs = c;
  cs.st = side;
  bool main_advanced = true;  // main-stream work not yet visible to the side stream
  // Gradient sets for the DP events: each fires once every op that writes the set's
  // gradients OR reads the set's weights has been enqueued, so an optimizer step
  // on another stream after the event cannot race with this backward pass.
  static const int sets[4][4] = {{NNT_OP_PROJ_DB, NNT_OP_PROJ_DW, NNT_OP_PROJ_DX, -1},
                                 {NNT_OP_FC_DB, NNT_OP_FC_DW, NNT_OP_FC_DX, NNT_OP_LN2_BWD},
                                 {NNT_OP_OUT_DB, NNT_OP_OUT_DW, NNT_OP_OUT_DX, -1},
                                 {NNT_OP_QKV_DB, NNT_OP_QKV_DW, NNT_OP_QKV_DX, NNT_OP_LN1_BWD}};
  int remaining[4];
  for (int k = 0; k < 4; ++k) remaining[k] = sets[k][3] < 0 ? 3 : 4;
  const bool lagged = side && links && links->side_done;
  for (const auto& gr : plan->groups) {
    if (gr.op == NNT_OP_LN1_BWD && side && links && links->wait_before_dx)  // the layer above's side ops
      NNT_CUDA_TRY(cudaStreamWaitEvent(stream, (cudaEvent_t)links->wait_before_dx, 0));  // read dy
    if (on_side(gr)) {
      if (main_advanced) {
        NNT_CUDA_TRY(cudaEventRecord(ev_fork, stream));
        NNT_CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
        main_advanced = false;
      }
      NNT_TRY(run_bwd_op(cs, gr.op, p, x, dy, dx, g, accumulate_grads));
    } else {
      NNT_TRY(run_bwd_op(c, gr.op, p, x, dy, dx, g, accumulate_grads));
      main_advanced = true;
    }
    if (!grad_ready) continue;
    for (int k = 0; k < 4; ++k)
      for (int j = 0; j < 4; ++j) {
        if (sets[k][j] != gr.op || --remaining[k] != 0 || !grad_ready[k]) continue;
        if (!side) {
          NNT_CUDA_TRY(cudaEventRecord((cudaEvent_t)grad_ready[k], stream));
          continue;
        }
        // the set's ops are split over both streams: bring the side stream past the main
        // stream's work so far (side ops enqueued later would fork from a later point anyway),
        // then the event on the side stream covers both -- each bucket fires as soon as its own
        // set is done, not at the end of the layer
        if (main_advanced) {
          NNT_CUDA_TRY(cudaEventRecord(ev_fork, stream));
          NNT_CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
          main_advanced = false;
        }
        NNT_CUDA_TRY(cudaEventRecord((cudaEvent_t)grad_ready[k], side));
      }
  }
  if (lagged) {  // the caller joins later (links.side_done); its next call alternates scratch
    NNT_CUDA_TRY(cudaEventRecord((cudaEvent_t)links->side_done, side));
  } else if (side) {  // join: the main stream continues only after the side stream's work
    NNT_CUDA_TRY(cudaEventRecord(ev_join, side));
    NNT_CUDA_TRY(cudaStreamWaitEvent(stream, ev_join, 0));
  }
  return NNT_OK;
}

}  // extern "C"
