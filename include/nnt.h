/*
 * nnt.h — C ABI of libnnt.so, the B200 (sm_100a) hot path of NNTile's
 * data-parallel GPT-2 block (arXiv 2504.13236).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n
 * (interfaces/test ideas only); "Rk" = reading k in DESIGN.md §Readings.
 *
 * General conventions (apply to every entry point unless stated otherwise)
 * -----------------------------------------------------------------------
 *  - C linkage, no exceptions cross the ABI.  Every call returns nnt_status.
 *    On failure the thread-local nnt_last_error() holds a one-line message.
 *  - Validation happens before any launch: a call that returns an error has
 *    enqueued NOTHING.  Fail fast, first error wins.
 *  - Ownership: the caller owns all memory.  Pointers marked "device" must be
 *    device memory of the current CUDA device; pointers marked "host" are host
 *    memory.  The library never allocates or frees device memory on the hot
 *    path; scratch/saved workspaces are caller-provided and sized by the
 *    *_bytes / *_size functions.
 *  - Asynchrony: every device-touching call is asynchronous on the given
 *    stream (a cudaStream_t; NULL = legacy default stream) and does not
 *    synchronise the host.
 *  - Layout: row-major; leading dimensions ("ld") and strides in ELEMENTS.
 *    Tensors that feed the tensor-core path need 16-byte aligned base
 *    pointers and leading dimensions / batch strides whose byte size is a
 *    multiple of 16 (TMA requirement) — else NNT_ERR_ALIGN.
 *  - dtypes: NNT_F32 (fp32 path: SIMT FFMA, true fp32) and NNT_BF16 (bf16
 *    operands on tcgen05 tensor cores, fp32 accumulation) (R15).
 *  - Tiles: tensors are split into tiles with a tile shape; a
 *    tile larger than its dimension is clamped; tile <= 0 is
 *    NNT_ERR_TILE.  Logical tiles define the tile-task grid (nnt_block_dag_*);
 *    one kernel launch executes every independent tile task of a level, so
 *    results do not depend on the tile shape beyond floating-point rounding
 *    order (tile invariance, tests/test_gpu_*).
 */
#ifndef NNT_H_
#define NNT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNT_ABI_VERSION 1

/* Causal write/read alignment of attention-probability rows (see nnt_softmax). */
#define NNT_CAUSAL_ALIGN 128

typedef struct CUstream_st* nnt_stream_t; /* == cudaStream_t */
typedef struct CUevent_st* nnt_event_t;   /* == cudaEvent_t  */

typedef enum {
  NNT_OK = 0,
  NNT_ERR_NULL = 1,        /* required pointer is NULL                        */
  NNT_ERR_SHAPE = 2,       /* non-positive or inconsistent dimension          */
  NNT_ERR_TILE = 3,        /* non-positive tile size                          */
  NNT_ERR_DTYPE = 4,       /* unsupported dtype / dtype combination           */
  NNT_ERR_ALIGN = 5,       /* pointer / leading-dimension alignment violated  */
  NNT_ERR_UNSUPPORTED = 6, /* valid request outside what the library implements */
  NNT_ERR_WORKSPACE = 7,   /* caller workspace too small                      */
  NNT_ERR_CUDA = 8,        /* a CUDA runtime/driver call failed               */
  NNT_ERR_ARG = 9          /* other invalid argument (enum out of range, ...) */
} nnt_status;

typedef enum { NNT_F32 = 0, NNT_BF16 = 1 } nnt_dtype;
typedef enum { NNT_NOTRANS = 0, NNT_TRANS = 1 } nnt_trans;

/* ------------------------------------------------------------------------- */
/* Library / device                                                           */
/* ------------------------------------------------------------------------- */
int nnt_abi_version(void);
const char* nnt_last_error(void);
/* NNT_OK iff `device` is compute capability 10.0 (sm_100a SASS in this library). */
nnt_status nnt_device_check(int device);

/* ------------------------------------------------------------------------- */
/* Tile bookkeeping (host only, integer, bit-exact) — P:72-75          */
/* ------------------------------------------------------------------------- */
/* grid[d] = ceil(shape[d] / min(tile[d], shape[d])).  host arrays of length ndim. */
nnt_status nnt_tile_grid(int ndim, const int64_t* shape, const int64_t* tile, int64_t* grid);
/* offset / extent of tile `idx` along one axis: extent = min(t, dim - idx*t), t = min(tile, dim). */
nnt_status nnt_tile_extent(int64_t dim, int64_t tile, int64_t idx, int64_t* offset, int64_t* extent);
/* Batch tiles owned by rank r of R: [floor(r n / R), floor((r+1) n / R)). */
nnt_status nnt_partition(int64_t n_units, int n_ranks, int rank, int64_t* begin, int64_t* end);

/* ------------------------------------------------------------------------- */
/* Tiled GEMM — linear layer Y = W X +. b, attention products     */
/* (P:181).                                                                   */
/* ------------------------------------------------------------------------- */
typedef enum {
  NNT_CAUSAL_NONE = 0,
  /* Only C[i][j] with j <= i is required; C entries with j > i may be left
   * untouched or hold arbitrary finite values (attention scores, dP).       */
  NNT_CAUSAL_OUT_LOWER = 1,
  /* op(A) is lower triangular (op(A)[i][k] == 0 for k > i): the kernel may
   * skip the zero K-blocks.  Result = the full product (P·V, dA·K).         */
  NNT_CAUSAL_A_LOWER = 2,
  /* op(A) is upper triangular (op(A)[i][k] == 0 for k < i): zero K-blocks
   * may be skipped (P^T·dO, dA^T·Q).                                         */
  NNT_CAUSAL_A_UPPER = 3
} nnt_causal;

typedef enum {
  NNT_ACT_NONE = 0,
  NNT_ACT_GELU = 1,     /* aux <- pre ; C <- gelu(pre)           (R11) */
  NNT_ACT_GELU_BWD = 2, /* C <- pre * gelu'(aux)                  (R18)          */
  /* Softmax backward fused into the dP = dO V^T GEMM (R18 with D from the dO.O identity):
   * C <- rowscale * aux * (pre - rowvec[item*M + i]); aux = P (same dtype, batch strides and
   * ld as C), rowvec = D (fp32), rowscale = 1/sqrt(h).  bf16 path only. */
  NNT_ACT_SOFTMAX_BWD = 3,
  /* SoftMax subroutine 1 over whole rows, fused into the score GEMM (R26):
   * x = alpha*acc is never stored (C must be NULL); row_stats[(p*batch1 + q)*M + i] receives
   * (max_j x_ij, sum_j e^{x_ij - max}) over the row's valid columns (j <= i when causal ==
   * NNT_CAUSAL_OUT_LOWER).  One task owns all key tiles of a 128-row block, so the per-tile
   * partials are aggregated on chip.  bf16 operands, alpha > 0; no bias / residual / beta. */
  NNT_ACT_ROWSTATS = 4,
  /* SoftMax subroutine 2 fused into a recomputation of the score GEMM (R26):
   * C = e^{alpha*acc - M_i} / S_i with (M_i, S_i) = row_stats[(p*batch1 + q)*M + i] (input, as
   * written by NNT_ACT_ROWSTATS).  causal == NNT_CAUSAL_OUT_LOWER: entries j > i are written
   * as 0 up to column roundup(i+1, NNT_CAUSAL_ALIGN) and not written beyond (nnt_softmax's
   * extents).  bf16 operands, bf16 C; no bias / residual / beta. */
  NNT_ACT_SOFTMAX = 5
} nnt_act;

/* Tensor-parallel reduction over peer memory (reading R35).
 * A group of R ranks SUMs an fp32 [rows][cols] tensor of which each rank holds a partial.  Rows
 * are owned in blocks of rows_per = ceil(rows / R): owner o holds rows [o rows_per, (o+1) rows_per).
 * All pointers are device addresses usable by this rank's kernels: its own buffers and the
 * peers' buffers mapped into its address space (symmetric memory over NVLink; on one GPU, plain
 * allocations standing for the ranks).  Ownership stays with the caller.
 *   recv[o]:  owner o's receive buffer, [R][rows_per][cols] fp32: slot w holds writer w's partial
 *             of o's rows.  A GEMM with nnt_epilogue.scatter = comm writes its output rows
 *             straight into these slots (the reduce-scatter's send, fused into the epilogue).
 *   flags[q]: rank q's flag words, [2][NNT_TP_MAX] uint32, zero-initialised once; a reduction
 *             is identified by a caller-chosen epoch (increasing, never 0). */
#define NNT_TP_MAX 8
typedef struct {
  int R;                           /* group size, 1..NNT_TP_MAX */
  int rank;                        /* this rank, 0..R-1         */
  int64_t rows, cols;              /* the reduced tensor: rows x cols fp32 (row-major, ld = cols) */
  float* recv[NNT_TP_MAX];
  uint32_t* flags[NNT_TP_MAX];
} nnt_tp_comm;

typedef struct {
  const float* bias;      /* device fp32 [N] added to every row, or NULL          */
  const float* residual;  /* device fp32 [M][ld_residual] added, or NULL (may alias C
                             only when C is fp32 with ldc == ld_residual)          */
  int64_t ld_residual;
  int act;                /* nnt_act                                               */
  void* aux;              /* device, same dtype as C, [M][ld_aux]: GELU pre-activation
                             (written by NNT_ACT_GELU, read by NNT_ACT_GELU_BWD)    */
  int64_t ld_aux;
  int causal;             /* nnt_causal (applies per batch item)                   */
  void* workspace;        /* device scratch for split-K partials, or NULL (no split);
                             see nnt_tile_gemm_workspace_bytes                     */
  size_t workspace_bytes;
  /* SoftMax subroutine 1 fused into the epilogue, bf16 path with fp32 C:
   * for every output row and every 32-column key tile g the partial
   * (m_g, s_g) = (max, sum e^{x - m_g}) of x = alpha*acc over the tile's valid columns
   * (col <= row when causal == NNT_CAUSAL_OUT_LOWER; (-inf, 0) if none) is written to
   * row_stats[((p*batch1 + q)*M + row)*ld_row_stats + g] as two floats.  Merged by
   * nnt_maxsumexp_merge.  NULL = off.
   * With act NNT_ACT_ROWSTATS / NNT_ACT_SOFTMAX: one (max, sumexp) pair per output row (output /
   * input respectively, see nnt_act); ld_row_stats is ignored. */
  float* row_stats;
  int64_t ld_row_stats;   /* in (max, sumexp) pairs, >= ceil(N / 32) */
  const float* rowvec;    /* NNT_ACT_SOFTMAX_BWD: per-row D, indexed (p*batch1 + q)*M + i */
  float rowscale;         /* NNT_ACT_SOFTMAX_BWD: output scale                            */
  /* Row sums of op(A), fused into the GEMM (R27): a_rowsum[i] = beta * a_rowsum[i] +
   * alpha * sum_k op(A)[i][k], device fp32 [M], or NULL = off.  With A = dY^T (the dW = dY^T X
   * GEMM of a linear layer) this is the bias gradient db = sum over tokens of dY,
   * computed by the tensor cores against a ones vector from the bf16 operand the GEMM already
   * stages.  bf16 operands, unbatched, non-causal, no activation; it uses the GEMM's split-K
   * workspace when the GEMM splits K (nnt_tile_gemm_workspace_bytes includes its slices). */
  float* a_rowsum;
  /* Tensor-parallel row scatter (R35), or NULL: output row i is stored to
   * scatter->recv[i / rows_per] slot scatter->rank instead of C (C is not written).  fp32 C,
   * unbatched, M == scatter->rows, N == ldc == scatter->cols; no split-K / stream-K. */
  const nnt_tp_comm* scatter;
} nnt_epilogue;

/* Workspace bytes that let nnt_tile_gemm split K for this shape (bf16 path; 0 when it would
 * not split).  Splitting applies to fp32 C without activation or causal mode (the dW GEMMs):
 * split s writes alpha * (its K-range partial) to workspace slice s and an ordered reduce
 * forms C = beta*C + sum_s partial_s (+bias, +residual), splits added in ascending order (R25).
 * The reduce runs inside the GEMM: the last split to finish each output region adds the
 * partials; the arrival counters it uses sit in the last 16 KB of the workspace (as sized by the
 * caller's workspace_bytes, which must stay the same for a buffer; GEMMs of different shapes may
 * share one workspace sized for the largest).
 * CONTRACT: that zone must be ZERO before the first use (e.g. torch.zeros for the whole buffer);
 * every call leaves it zero again.  A smaller workspace that still holds the partials is accepted
 * and reduces with a separate kernel launch instead. */
size_t nnt_tile_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int c_dtype, int act, int causal,
                                     int64_t batch_items);

/*
 * C = epilogue( alpha * op(A) · op(B) ),  for each of batch[0]*batch[1] items.
 *   pre = alpha * sum_k op(A)[i][k] op(B)[k][j]  (+ bias[j]) (+ beta * C_old[i][j])
 *         (+ residual[i][j]);  C = act(pre).
 * op(A) is M x K: A is stored [M][lda] if trans_a == NNT_NOTRANS, [K][lda] if NNT_TRANS.
 * op(B) is K x N: B is stored [K][ldb] if trans_b == NNT_NOTRANS, [N][ldb] if NNT_TRANS.
 * Batch item (p, q) uses A + p*stride_a[0] + q*stride_a[1] (elements), likewise B, C
 * (strides may be 0; batch/strides may be NULL for a single item).  This is how
 * attention's (N_b, N_h) views of the fused [N_b, N_s, 3, N_h, h] QKV buffer are
 * addressed without copies.
 * dtypes: (A,B) both NNT_F32 (SIMT fp32 path) or both NNT_BF16 (tcgen05 path);
 * C NNT_F32 or NNT_BF16.  Accumulation is fp32 over K in ascending order, i.e. the
 * K-tile Reduce of the tiled GEMM in a fixed, deterministic order.
 * tile: host int64[3] logical tile (tile_m, tile_n, tile_k); NULL = untiled.
 */
nnt_status nnt_tile_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                         const int64_t* batch,
                         float alpha,
                         const void* A, int a_dtype, int64_t lda, const int64_t* stride_a,
                         const void* B, int b_dtype, int64_t ldb, const int64_t* stride_b,
                         float beta,
                         void* C, int c_dtype, int64_t ldc, const int64_t* stride_c,
                         const int64_t* tile, const nnt_epilogue* epi, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* SoftMax as two subroutines                                     */
/* ------------------------------------------------------------------------- */
/*
 * Subroutine 1: for every slice (row) r of x (device fp32 [rows][ldx])
 * over columns [0, cols): per key tile of tile_k columns the partial
 * (m_j = max, s_j = sum e^{x - m_j}), merged in ascending tile order with
 * (m,s)(+)(m',s') = (M, s e^{m-M} + s' e^{m'-M}); (-inf, 0) is the identity (R10).
 * causal != 0: row r is query q = r % seq_q and columns k > q are excluded (R2).
 * stats: device fp32 [rows][2] = (max, sumexp).  accumulate != 0 merges the
 * result into the existing stats instead of overwriting (one call per key tile).
 */
nnt_status nnt_maxsumexp(const float* x, int64_t rows, int64_t cols, int64_t ldx,
                         int64_t tile_k, int causal, int64_t seq_q,
                         float* stats, int accumulate, nnt_stream_t stream);

/*
 * Aggregation of subroutine 1 ("aggregates them"): merges per-key-tile partials
 * part[r][g] = (m_g, s_g) (device fp32 pairs, row pitch ld_parts pairs, tile width
 * part_cols) in ascending g into stats[r] = (M, S); with causal != 0 only the tiles holding
 * a valid column (g*part_cols <= q, q = r % seq_q) are read.  Same merge rule as
 * nnt_maxsumexp.
 */
nnt_status nnt_maxsumexp_merge(const float* part, int64_t rows, int64_t nparts, int64_t ld_parts,
                               int64_t part_cols, int causal, int64_t seq_q, float* stats,
                               nnt_stream_t stream);

/*
 * Subroutine 2: y[r][k] = e^{x[r][k] - M_r} / S_r with (M_r, S_r) = stats[r].
 * y is device fp32 or bf16 [rows][ldy].  causal != 0: entries with k > q are written
 * as 0 for k < min(cols, roundup(q+1, NNT_CAUSAL_ALIGN)) and not written beyond;
 * x entries with k > q are never read.
 */
nnt_status nnt_softmax(const float* x, int64_t rows, int64_t cols, int64_t ldx, int64_t tile_k,
                       int causal, int64_t seq_q, const float* stats,
                       void* y, int y_dtype, int64_t ldy, nnt_stream_t stream);

/*
 * Softmax backward (R18): da = scale * P ⊙ (dP − D), D[r] = sum_k P[r][k] dP[r][k].
 * p: device fp32/bf16 [rows][ldp]; dp: device fp32 [rows][lddp]; da: device
 * fp32/bf16 [rows][ldda].  causal: same read/write extents as nnt_softmax
 * (masked entries written as exact 0; dP above the diagonal is never read).
 */
nnt_status nnt_softmax_bwd(const void* p, int p_dtype, int64_t ldp,
                           const float* dp, int64_t lddp,
                           int64_t rows, int64_t cols, int causal, int64_t seq_q, float scale,
                           void* da, int da_dtype, int64_t ldda, nnt_stream_t stream);

/*
 * D for the softmax backward through the identity sum_k P[q][k] dP[q][k] = sum_i dO[q][i] O[q][i]
 * (dP = dO V^T and O = P V; pinned in tests/test_oracle_pins.py):
 *   D[(b*H + n)*S + s] = sum_{i<h} dO[b][s][n*h + i] * O[b][s][n*h + i]
 * dO, O: device bf16 or fp32 [B][S][H*h] (`dtype`); D: device fp32 [B*H*S].
 */
nnt_status nnt_attn_rowdot(const void* dO, const void* O, int dtype, int64_t B, int64_t S, int64_t H,
                           int64_t h, float* D, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Fused attention tiles (bf16 path, readings R20, R26, R33)       */
/* ------------------------------------------------------------------------- */
/* Pipeline trace of the fused attention kernels (tools/attn_trace.py): enable != 0 makes CTA 0
 * of the following launches record %globaltimer at 6 events of each of its first 256 iterations
 * (fwd: K/V loads issued, S MMA issued, S ready in the epilogue, P staged, P seen by the MMA
 * issuer, O MMA issued); host_out (nullable, up to cap entries of [2][6][256] uint64) receives the
 * last recorded values (index 0 forward, 1 backward).  Debug only; off by default. */
nnt_status nnt_attention_trace(int enable, uint64_t* host_out, int64_t cap);

/* 1 when the fused attention kernels below cover (S, h): head size 64 and S % 128 == 0. */
int nnt_attention_fused_supported(int64_t S, int64_t h);

/*
 * Softmax subroutine 2 and the value product of B = V SoftMax(K^T Q / sqrt(h)),
 * per (batch b, head n), 128 x 128 tile by tile:
 *   P[b][n][q][k] = e^{scale * q_q . k_k - M} / S_sum   (k <= q when causal, else 0 in the
 *                   diagonal tile; tiles above the diagonal are not written)
 *   O[b][q][n*h + i] = sum_k P[b][n][q][k] V[b][k][n*h + i]
 * with (M, S_sum) the row statistics of softmax subroutine 1 (the ROWSTATS score GEMM, R26).
 * Each P tile is staged in shared memory once: stored to HBM (the backward reads it) and fed to
 * the P V tensor-core product from there.
 * qkv: device bf16 [B][S][3][H][h] (Q | K | V thirds, row pitch 3*H*h); stats: device fp32
 * [B*H*S][2] = (M in scaled-score units, S_sum); P: device bf16 [B][H][S][S]; O: device bf16
 * [B][S][H*h].  h == 64, S % 128 == 0 (else NNT_ERR_UNSUPPORTED); 16-byte aligned.
 */
/* Softmax subroutine 1 of the bf16 attention, per (b, n, query q): the score row
 * x[k] = scale * sum_i Q[q][i] K[k][i] over keys k (k <= q when causal) is formed tile by tile on
 * the tensor cores and reduced on chip -- never stored (R26) -- to stats[(b*H + n)*S + q] =
 * (M, S) = (max_k x[k], sum_k e^{x[k] - M}) as two floats (the input nnt_attention_fwd_pv reads).
 * qkv as above; stats: device fp32 [B][H][S][2].  Same conditions (h = 64, S % 128 == 0). */
nnt_status nnt_attention_stats(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t h, float scale, int causal,
                               float* stats, nnt_stream_t stream);
/* 1 unless NNT_ATTN_STATS=0 in the environment: the block uses nnt_attention_stats for the row
 * statistics (else the NNT_ACT_ROWSTATS score GEMM). */
int nnt_attention_stats_enabled(void);

nnt_status nnt_attention_fwd_pv(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t h, float scale,
                                int causal, const float* stats, void* P, void* O, nnt_stream_t stream);

/*
 * Softmax backward with the dK / dV products (R18, R20), per (b, n) and 128-key block kb over the
 * query blocks qb (>= kb when causal):
 *   dA[b][n][q][k] = scale * P[q][k] * (sum_i dO[q][i] V[k][i] - D[q])      (stored query-major)
 *   dK[k][n*h + i] = sum_q dA[q][k] Q[q][i]              dV[k][n*h + i] = sum_q P[q][k] dO[q][i]
 * D = rowdot(dO, O) (nnt_attn_rowdot).  Each P tile is read once and each dA tile written once
 * (formed over the P tile in shared memory); dK and dV accumulate on chip over the query blocks.
 * dQ = dA K is the GEMM nnt_tile_gemm(NNT_NOTRANS, NNT_NOTRANS, S, h, S, {B, H}, 1, dA, S,
 * {H*S*S, S*S}, K, ..., causal NNT_CAUSAL_A_LOWER) (entries with k > q are zero; blocks with
 * kb > qb are not written and not read).
 * qkv, P, D as above; dO: device bf16 [B][S][H*h]; dA: device bf16 [B][H][S][S]; dqkv: device
 * bf16 [B][S][3][H][h] -- its K and V thirds are written, the Q third untouched.
 */
nnt_status nnt_attention_bwd_kv(const void* qkv, const void* dO, const void* P, const float* D, int64_t B,
                                int64_t S, int64_t H, int64_t h, float scale, int causal, void* dA,
                                void* dqkv, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* LayerNorm in three steps                                       */
/* ------------------------------------------------------------------------- */
/*
 * For every token row t of x (device fp32 [T][ldx]) over E columns:
 *   step 1, per E-tile of tile_e columns: shifted sums S1 = sum (x - c), S2 = sum (x - c)^2
 *           with c = x[t][0]; merged over tiles in ascending order (R9);
 *           mean = c + S1/E, var = max(S2/E - (S1/E)^2, 0), rstd = 1/sqrt(var + eps);
 *   step 2: xhat = (x - mean) * rstd;   step 3: y = gamma * xhat + beta.
 * y: device fp32/bf16 [T][ldy]; mean, rstd: device fp32 [T] (saved for backward).
 */
nnt_status nnt_layernorm_fwd(const float* x, int64_t T, int64_t E, int64_t ldx, int64_t tile_e,
                             const float* gamma, const float* beta, float eps,
                             void* y, int y_dtype, int64_t ldy,
                             float* mean, float* rstd, nnt_stream_t stream);

/* Scratch bytes nnt_layernorm_bwd needs for its ordered dgamma/dbeta partials. */
size_t nnt_layernorm_bwd_scratch_bytes(int64_t T, int64_t E);

/*
 * LayerNorm backward (R18):
 *   dxhat = dy * gamma;  dx = dres + rstd * (dxhat - mean_e dxhat - xhat * mean_e(dxhat xhat))
 *   dgamma (+)= sum_t dy * xhat;  dbeta (+)= sum_t dy   (column partials over row
 *   chunks, merged in ascending chunk order: deterministic).
 * dy: device fp32 [T][lddy]; x, mean, rstd, gamma as in the forward; dres: device
 * fp32 [T][lddx] or NULL (residual-stream gradient added to dx; may alias dx);
 * dx: device fp32 [T][lddx]; dx_bf16: device bf16 [T][lddx] copy of dx or NULL;
 * dgamma, dbeta: device fp32 [E]; dx_colsum: NULL or device fp32 [E] (+)= sum_t dx, the
 * bias gradient of the linear layer that produced this LayerNorm's input; accumulate_params
 * != 0 adds into dgamma / dbeta / dx_colsum.  E <= 8192.
 */
nnt_status nnt_layernorm_bwd(const float* dy, int64_t lddy, const float* x, int64_t ldx,
                             const float* mean, const float* rstd, const float* gamma,
                             int64_t T, int64_t E,
                             const float* dres, float* dx, int64_t lddx, void* dx_bf16,
                             float* dgamma, float* dbeta, float* dx_colsum, int accumulate_params,
                             void* scratch, size_t scratch_bytes, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Elementwise GELU (R11 tanh form)                                */
/* ------------------------------------------------------------------------- */
/* y[i] = gelu(x[i]); x, y device arrays of n elements of `dtype`. */
nnt_status nnt_gelu_fwd(const void* x, void* y, int dtype, int64_t n, nnt_stream_t stream);
/* dx[i] = dy[i] * gelu'(x[i]). */
nnt_status nnt_gelu_bwd(const void* x, const void* dy, void* dx, int dtype, int64_t n,
                        nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Bias gradient: column sums db[j] (+)= sum_t dy[t][j] (R18)                 */
/* ------------------------------------------------------------------------- */
size_t nnt_bias_grad_scratch_bytes(int64_t T, int64_t N);
/* dy: device fp32/bf16 [T][lddy]; db device fp32 [N]; dy_bf16_out: optional device
 * bf16 [T][lddy] copy of dy (cast fused into the same pass; fp32 dy only). */
nnt_status nnt_bias_grad(const void* dy, int dy_dtype, int64_t T, int64_t N, int64_t lddy,
                         float* db, int accumulate, void* dy_bf16_out,
                         void* scratch, size_t scratch_bytes, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Adam / AdamW per tile (R12)                                     */
/* ------------------------------------------------------------------------- */
typedef struct {
  float lr, beta1, beta2, eps;
  float weight_decay; /* 0 = Adam; > 0 = AdamW decoupled decay w -= lr*wd*w_old */
  float bias_corr1;   /* 1 - beta1^t, computed by the caller in fp64, t >= 1    */
  float bias_corr2;   /* 1 - beta2^t                                            */
  float grad_scale;   /* g is multiplied by this first (1 = none)               */
  /* device fp32 [2] = {bias_corr1, bias_corr2}, read by the kernel instead of the two
   * scalars above when non-NULL (lets a captured CUDA graph advance the step count) */
  const float* bias_corr_dev;
  /* 1 - beta1 and 1 - beta2 rounded to fp32 from the caller's fp64 values (R23: 1.0f - 0.999f is
   * off by 1.3e-5 relative from fp32(1 - 0.999)); 0 = derive them in fp32 from beta1 / beta2 */
  float one_minus_beta1, one_minus_beta2;
} nnt_adam_hparams;

/* m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; w -= lr (m/bc1) / (sqrt(v/bc2) + eps).
 * w, g, m, v: device fp32 [n] (one flat tile range); w_bf16: optional device bf16 [n]
 * shadow written as round-to-nearest-even(w_new); hp: host struct. */
nnt_status nnt_adam_step(int64_t n, float* w, const float* g, float* m, float* v, void* w_bf16,
                         const nnt_adam_hparams* hp, nnt_stream_t stream);

/* Advances a device step counter and writes the Adam bias corrections for it:
 * t_dev[0] += 1;  bias_corr_dev = {1 - beta1^t, 1 - beta2^t} computed in fp64 (R12).
 * t_dev: device int64 [1]; bias_corr_dev: device fp32 [2] (pass it as
 * nnt_adam_hparams.bias_corr_dev).  One thread; usable inside a captured CUDA graph. */
nnt_status nnt_adam_tick(double beta1, double beta2, int64_t* t_dev, float* bias_corr_dev, nnt_stream_t stream);

/* SGD with momentum ("a weighted sum of the input vector, gradient, and momentum
 * term"): buf = momentum * buf + (g + weight_decay * w); w -= lr * buf (buf starts at 0).
 * w, g, buf: device fp32 [n]; w_bf16: nullable bf16 shadow of w, refreshed in the same pass. */
nnt_status nnt_sgd_step(int64_t n, float* w, const float* g, float* buf, void* w_bf16, float lr, float momentum,
                        float weight_decay, nnt_stream_t stream);

/* fp32 -> bf16 (round to nearest even) or bf16 -> fp32 conversion of n elements. */
nnt_status nnt_convert(const void* x, int x_dtype, void* y, int y_dtype, int64_t n,
                       nnt_stream_t stream);

/* y[i] = alpha * x[i] (fp32, n elements; y may alias x).  Used for dy = r / T_global (R13). */
nnt_status nnt_scale(const float* x, float alpha, float* y, int64_t n, nnt_stream_t stream);

/* Block-only loss (R13): out[0] = scale * sum_i y[i] r[i] (deterministic order). */
size_t nnt_dot_scratch_bytes(int64_t n);
nnt_status nnt_dot(const float* y, const float* r, int64_t n, float scale, float* out,
                   void* scratch, size_t scratch_bytes, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* GPT-2 shell: embedding layer and cross-entropy loss       */
/* ------------------------------------------------------------------------- */
/* Embedding layer (learned positions, reading R29):
 *   x[t] = wte[ids[t]] + wpe[t mod S]  for t < T (T = B*S tokens, row-major [B][S]).
 * ids: device int32 [T] in [0, V) (out-of-range ids are clamped); wte: device fp32 [V][E];
 * wpe: device fp32 [>= S][E]; x: device fp32 [T][E].  E % 4 == 0, 16-byte aligned. */
nnt_status nnt_embedding_fwd(const int32_t* ids, int64_t T, int64_t S, const float* wte, int64_t V,
                             const float* wpe, int64_t E, float* x, nnt_stream_t stream);

/* Scratch bytes of nnt_embedding_bwd (a counting sort of the T token positions by id). */
size_t nnt_embedding_bwd_scratch_bytes(int64_t T, int64_t V);

/* Adjoint of nnt_embedding_fwd: dwte[v] (+)= sum over tokens t with ids[t] == v of dx[t]
 * (added in ascending t), dwpe[s] (+)= sum_b dx[b*S + s] (ascending b).  accumulate_wte != 0
 * adds into dwte (rows of dwte whose id does not occur are then untouched; the tied LM head
 * writes its half of the gradient there first), 0 overwrites; accumulate_wpe likewise for dwpe
 * (separate flags: the two tables have separate producers).
 * Deterministic (integer counting sort, no floating-point atomics).  dx: device fp32 [T][E];
 * dwte: [V][E]; dwpe: [>= S][E] (rows >= S untouched). */
nnt_status nnt_embedding_bwd(const int32_t* ids, int64_t T, int64_t S, const float* dx, int64_t E,
                             float* dwte, int64_t V, float* dwpe, int accumulate_wte, int accumulate_wpe,
                             void* scratch, size_t scratch_bytes, nnt_stream_t stream);

/* Cross-entropy through the two SoftMax subroutines (R13): per row r of
 * the logits x (device fp32/bf16 [rows][ld], V classes), subroutine 1 gives (M_r, S_r) =
 * (max_k x, sum_k e^{x - M}) (R10 merge, fixed order) and
 *   loss_rows[r] = log S_r + M_r - x[r][labels[r]]            (if loss_rows != NULL)
 *   stats[r]     = (M_r, S_r)                                 (if stats != NULL, fp32 [rows][2])
 *   dlogits[r][k] = scale * (e^{x[r][k] - M_r} / S_r - [k == labels[r]])   (if dlogits != NULL;
 *                   same dtype as x, row pitch ld_d, may alias x)
 * labels: device int32 [rows] (clamped to [0, V)).  Rows 16-byte aligned. */
nnt_status nnt_cross_entropy(const void* logits, int dtype, int64_t rows, int64_t V, int64_t ld,
                             const int32_t* labels, float scale, float* loss_rows, float* stats,
                             void* dlogits, int64_t ld_d, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* GPT-2 block (pre-LN, R1) forward / backward on one GPU's batch tiles        */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t E;       /* N_e embedding size                     */
  int64_t H;       /* N_h heads, h = E / H                   */
  int64_t S;       /* N_s sequence length                    */
  int64_t B;       /* N_b sequences on this GPU              */
  int64_t tile_e;  /* logical tile along embedding axes      */
  int64_t tile_f;  /* logical tile along the MLP hidden axis */
  int64_t tile_s;  /* logical tile along the sequence axis   */
  int64_t tile_t;  /* logical tile along tokens (rows)       */
  int dtype;       /* NNT_F32 or NNT_BF16 compute path       */
  float ln_eps;    /* LayerNorm epsilon (R9: 1e-5)           */
  int causal;      /* 1 = GPT-2 causal mask (R2)             */
} nnt_block_cfg;

/* Parameters of one block.  LayerNorm and bias vectors are fp32 masters; the four
 * weight matrices are in cfg.dtype (bf16 shadows on the bf16 path).
 * Shapes: w_qkv [3E][E] (q, k, v row blocks), w_o [E][E], w_fc [4E][E], w_pr [E][4E]. */
typedef struct {
  const float *ln1_g, *ln1_b, *b_qkv, *b_o, *ln2_g, *ln2_b, *b_fc, *b_pr;
  const void *w_qkv, *w_o, *w_fc, *w_pr;
} nnt_block_params;

/* fp32 gradients, same shapes as the parameters. */
typedef struct {
  float *ln1_g, *ln1_b, *w_qkv, *b_qkv, *w_o, *b_o, *ln2_g, *ln2_b, *w_fc, *b_fc, *w_pr, *b_pr;
} nnt_block_grads;

/* Bytes of the per-block `saved` activation workspace (kept from fwd to bwd, one per
 * layer) and of the shared `scratch` workspace (reusable across layers).  `scratch` holds the
 * dW GEMMs' split-K workspace: ZERO-FILL it before its first use (see
 * nnt_tile_gemm_workspace_bytes); the block calls leave that part zero again. */
nnt_status nnt_block_workspace_size(const nnt_block_cfg* cfg, size_t* saved_bytes,
                                    size_t* scratch_bytes);

/* y = block(x).  x, y: device fp32 [B][S][E]; saved/scratch: device workspaces.
 * Executes the block's lowered tile-task DAG (nnt_block_dag_describe) in order. */
nnt_status nnt_block_fwd(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x,
                         float* y, void* saved, void* scratch, nnt_stream_t stream);

/* Backward of nnt_block_fwd.  x: the same input; dy: device fp32 [B][S][E]; dx: device
 * fp32 [B][S][E] (may alias dy); g: fp32 gradients (accumulate_grads != 0 adds into
 * them).  grad_ready: NULL or 4 events recorded on `stream` when the gradients of
 * {mlp.proj, mlp.fc+ln2, attn.out, attn.qkv+ln1} are final (for overlapped DP
 * all-reduce). */
nnt_status nnt_block_bwd(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x,
                         const void* saved, void* scratch, const float* dy, float* dx,
                         const nnt_block_grads* g, int accumulate_grads,
                         nnt_event_t* grad_ready, nnt_stream_t stream);

/* nnt_block_bwd with a second stream: the ops that only produce weight / bias gradients
 * (the four dW GEMMs, the FC / out / QKV bias column sums) run on `side_stream`, forked
 * from `stream` after the ops they depend on and joined back into `stream` before the call
 * returns, so they fill the gaps of the dX chain.  Same results bit for bit.  side_stream
 * NULL = nnt_block_bwd.  grad_ready events (if given) are recorded on `stream` after the
 * join.  NNT_ERR_ARG if side_stream == stream.  links (nullable): the projection-bias column
 * sum and the bf16 copy of dy / dx are made by the LayerNorm backward of the layer above /
 * this layer instead of a separate pass over dy (consecutive blocks of a stack chain them). */
typedef struct {
  const void* dy_bf16;  /* bf16 copy of dy made by the caller (the layer above's dx_bf16), or NULL */
  int dy_colsum_done;   /* != 0: g->b_pr already holds (+)= sum_t dy (the layer above's dx_colsum) */
  float* dx_colsum;     /* NULL or [E]: (+)= sum_t dx, the output-projection bias gradient of the
                           layer below (follows accumulate_grads) */
  void* dx_bf16;        /* NULL or bf16 [T][E]: copy of dx for the layer below (bf16 path) */
  /* Lagged join of the side stream (with a side stream only): the side stream's ops of one layer
   * may still run while the main stream does the layer below, when the caller alternates two
   * scratch workspaces between layers and gives these events (NULL: join at the end of the call).
   *   side_done:      recorded on the side stream after this call's side ops (no join);
   *   wait_before_dx: the main stream waits on it before the LayerNorm-1 backward writes dx and
   *                   dx_bf16 -- the previous call's side_done (its side ops read the dy and the
   *                   bf16 copy of dy that this call's dx overwrites). */
  nnt_event_t side_done;
  nnt_event_t wait_before_dx;
} nnt_block_bwd_links;
nnt_status nnt_block_bwd_streams(const nnt_block_cfg* cfg, const nnt_block_params* p, const float* x,
                                 const void* saved, void* scratch, const float* dy, float* dx,
                                 const nnt_block_grads* g, int accumulate_grads,
                                 nnt_event_t* grad_ready, nnt_stream_t stream,
                                 nnt_stream_t side_stream, const nnt_block_bwd_links* links);

/* ------------------------------------------------------------------------- */
/* Tensor-parallel block shards ("split entire data  */
/* into tiles across embedding dimension", reading R31)                          */
/* ------------------------------------------------------------------------- */
/* One shard of a block split over a group of R GPUs along its inner dimensions: the shard
 * owns `heads` attention heads (the q/k/v rows of w_qkv / b_qkv for those heads, in the
 * order q-rows, k-rows, v-rows: w_qkv [3*heads*h][E]; the matching columns of w_o:
 * [E][heads*h]) and `ffn` hidden units (rows of w_fc / b_fc: [ffn][E]; columns of w_pr:
 * [E][ffn]).  LayerNorm parameters, b_o and b_pr are replicated.  Activations along E
 * (x, x1, y, dy, dx) are replicated; the shard's contributions to x1, y, dL/dh2 and dL/dh1
 * are partial sums that the caller reduces over the group (SUM) between stages.  With
 * heads = H, ffn = 4E, add_bias = 1 a single shard is the whole block. */
typedef struct {
  int64_t heads;  /* attention heads of this shard (1..H); heads * h a multiple of 8 */
  int64_t ffn;    /* MLP hidden units of this shard (1..4E), a multiple of 8           */
  int add_bias;   /* 1 on exactly one shard of the group: it adds b_o, b_pr and the residuals */
  const nnt_tp_comm* comm;  /* NULL: the stages write their partial sums locally (x1 / y / dh) and
                               the caller reduces them (e.g. NCCL); else the partial-producing
                               GEMM of each stage scatters its rows into comm->recv (R35) and the
                               caller completes the SUM with nnt_tp_signal / nnt_tp_reduce_gather /
                               nnt_tp_wait, which write x1 / y / dh on every rank */
} nnt_block_tp;

/* Workspace bytes of one shard (as nnt_block_workspace_size). */
nnt_status nnt_block_tp_workspace_size(const nnt_block_cfg* cfg, const nnt_block_tp* tp,
                                       size_t* saved_bytes, size_t* scratch_bytes);

/* Forward stages of a shard (p: the shard's parameter pointers, shapes above).
 *   stage 0: LN1(x) -> QKV -> attention over the shard's heads -> out-projection:
 *            x1 := this shard's partial of x + attn(x) (the bias and x only if add_bias).
 *   stage 1: (x1 now the group SUM) LN2(x1) -> FC + GELU -> projection:
 *            y := this shard's partial of x1 + mlp(x1).
 * x, x1, y: device fp32 [B][S][E]; x1 must stay untouched until the backward. */
nnt_status nnt_block_tp_fwd(const nnt_block_cfg* cfg, const nnt_block_tp* tp, const nnt_block_params* p,
                            int stage, const float* x, float* x1, float* y, void* saved, void* scratch,
                            nnt_stream_t stream);

/* Backward stages of a shard (dy replicated; g: the shard's gradients; replicated
 * parameters' gradients come out identical on every shard).
 *   stage 0: dy -> projection / FC gradients of the shard -> dh := partial dL/dh2.
 *   stage 1: (dh now the group SUM) LN2 backward (+ dy) -> dx1 (kept in scratch) ->
 *            out-projection / attention / QKV gradients -> dh := partial dL/dh1.
 *   stage 2: (dh now the group SUM) LN1 backward (+ dx1) -> dx.
 * dh: device fp32 [B][S][E], caller-owned; scratch must not be reused between stages. */
nnt_status nnt_block_tp_bwd(const nnt_block_cfg* cfg, const nnt_block_tp* tp, const nnt_block_params* p,
                            int stage, const float* x, const float* x1, const void* saved, void* scratch,
                            const float* dy, float* dh, float* dx, const nnt_block_grads* g,
                            int accumulate_grads, nnt_stream_t stream);

/* The rest of a tensor-parallel SUM after the GEMMs have scattered their partials (R35).  A rank
 * calls, on its stream, in this order:
 *   nnt_tp_signal(comm, epoch, 0)        tell every owner this rank's partials are in place;
 *   nnt_tp_reduce_gather(comm, out, epoch) wait for the R writers of this rank's rows, sum the R
 *                                        partials of each row in rank order (the same fixed
 *                                        association on every rank: replicas stay bitwise
 *                                        identical), write the sums into every rank's out[q]
 *                                        (out[q]: rank q's [rows][cols] destination);
 *   nnt_tp_signal(comm, epoch, 1)        tell every rank this rank's rows are gathered;
 *   nnt_tp_wait(comm, epoch)             wait until every owner's rows have arrived here.
 * After nnt_tp_wait the rank may read its out and reuse the recv buffers.  (On one GPU, ranks
 * standing in one process may issue all signals before the reduce-gathers.) */
nnt_status nnt_tp_signal(const nnt_tp_comm* comm, uint32_t epoch, int which, nnt_stream_t stream);
nnt_status nnt_tp_reduce_gather(const nnt_tp_comm* comm, float* const* out, uint32_t epoch, nnt_stream_t stream);
nnt_status nnt_tp_wait(const nnt_tp_comm* comm, uint32_t epoch, nnt_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Tile-task DAG (STF rules S:46)                               */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t op;        /* nnt_block_op                                        */
  int32_t level;     /* topological level (longest dependency chain)        */
  int64_t tile[3];   /* tile coordinates of the task within the op's grid   */
  int32_t n_deps;    /* number of predecessor tasks                          */
  int32_t group;     /* index of the launch group executing this task       */
} nnt_task;

typedef struct {
  int32_t op;
  int32_t level;
  int64_t n_tasks;
  int32_t side_stream_ok;  /* 1: no task of another op depends on this op and it writes only
                              parameter gradients (a sink of the pass): nnt_block_bwd_streams runs
                              it on the side stream */
} nnt_launch_group;

/* Ops of the block DAG, in submission (program) order. */
typedef enum {
  NNT_OP_LN1 = 0, NNT_OP_QKV, NNT_OP_SCORES, NNT_OP_MAXSUMEXP, NNT_OP_SOFTMAX, NNT_OP_PV,
  NNT_OP_OUT, NNT_OP_LN2, NNT_OP_FC, NNT_OP_PROJ,
  /* backward */
  NNT_OP_PROJ_DB, NNT_OP_PROJ_DW, NNT_OP_PROJ_DX, NNT_OP_FC_DB, NNT_OP_FC_DW, NNT_OP_FC_DX,
  NNT_OP_LN2_BWD, NNT_OP_OUT_DB, NNT_OP_OUT_DW, NNT_OP_OUT_DX, NNT_OP_ATT_DP, NNT_OP_ATT_DV,
  NNT_OP_SOFTMAX_BWD, NNT_OP_ATT_DQ, NNT_OP_ATT_DK, NNT_OP_QKV_DB, NNT_OP_QKV_DW,
  NNT_OP_QKV_DX, NNT_OP_LN1_BWD,
  NNT_OP_COUNT
} nnt_block_op;

const char* nnt_op_name(int op);

/* Builds (or returns the cached) tile-task DAG of one block pass (pass 0 = forward,
 * 1 = backward) from STF submission of per-tile tasks with R/W/RW/Reduce accesses,
 * and its lowering into launch groups: one group per op, launched at the highest
 * level its tasks reach (every dependency edge crosses launch levels; ops that
 * share a launch level are independent).  Writes up to
 * task_cap tasks / group_cap groups (host arrays, may be NULL with cap 0) and the
 * full counts. */
nnt_status nnt_block_dag_describe(const nnt_block_cfg* cfg, int pass,
                                  nnt_task* tasks, int64_t task_cap, int64_t* n_tasks,
                                  nnt_launch_group* groups, int64_t group_cap, int64_t* n_groups);

/* The STF graph builder the block plans use ("inserts tasks into the graph one by one";
 * dependency rules S:46: R->R none, R->W/RW edge, W/RW->anything edge, Reduce->Reduce none,
 * Reduce<->R/W/RW edge), on an arbitrary program: n_tasks tasks submitted in order over handles
 * 0..n_handles-1; task t has n_acc[t] accesses, taken in order from acc_handle / acc_mode
 * (nnt_access_mode: 0 R, 1 W, 2 RW, 3 Reduce; a handle at most once per task).  Outputs (host
 * arrays): level[n_tasks] (longest dependency chain), dep_offsets[n_tasks + 1] and the
 * predecessor lists dep_ids[dep_offsets[t] .. dep_offsets[t+1]) (at most dep_cap entries;
 * NNT_ERR_WORKSPACE with dep_offsets filled when dep_cap is too small).  Host-only, for tests. */
nnt_status nnt_stf_build(int64_t n_handles, int64_t n_tasks, const int32_t* n_acc, const int64_t* acc_handle,
                         const int32_t* acc_mode, int32_t* level, int64_t* dep_offsets, int32_t* dep_ids,
                         int64_t dep_cap);

/* ------------------------------------------------------------------------- */
/* Kernel timing (bench.py roofline): CUDA events around every launch.         */
/* ------------------------------------------------------------------------- */
typedef enum {
  NNT_K_GEMM_TC = 0, NNT_K_GEMM_TC_ATTN, NNT_K_GEMM_SIMT, NNT_K_MAXSUMEXP, NNT_K_SOFTMAX, NNT_K_SOFTMAX_BWD,
  NNT_K_LN_FWD, NNT_K_LN_BWD, NNT_K_GELU, NNT_K_BIAS_GRAD, NNT_K_ADAM, NNT_K_MISC,
  NNT_K_COUNT
} nnt_kernel_class;

/* enable != 0 starts recording (clears previous records). */
nnt_status nnt_timing_enable(int enable);
/* Synchronises the recorded events and returns, per kernel class, the summed
 * device time in ms, the launch count and the summed algorithmic bytes and flops
 * (host arrays of length NNT_K_COUNT; any may be NULL). */
nnt_status nnt_timing_read(double* ms, int64_t* launches, double* bytes, double* flops);
/* The recorded launch scopes in issue order: kclass[i] (nnt_kernel_class) and
 * kernels[i] (kernels the scope launched, e.g. 2 for a split-K GEMM + its ordered
 * reduce), for i < min(cap, *n); *n receives the total count.  Host arrays, may be
 * NULL when cap == 0.  Lets a profiler's per-kernel list (ncu) be attributed to
 * kernel classes. */
nnt_status nnt_timing_trace(int32_t* kclass, int32_t* kernels, int64_t cap, int64_t* n);
/* Number of kernels this library launched since load (all classes). */
int64_t nnt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NNT_H_ */
