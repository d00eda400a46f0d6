// bf16 tensor-core GEMM for sm_100a: tcgen05.mma (kind::f16, fp32 accumulate in
// TMEM), operands staged by TMA (SWIZZLE_128B) through an mbarrier ring,
// warp-specialised persistent CTAs:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9  epilogue: tcgen05.ld TMEM -> registers -> bias / beta*C /
//               residual / GELU / GELU' -> swizzled smem staging -> TMA bulk
//               tensor store; two warps per TMEM lane quadrant take alternating
//               128-byte column chunks; TMEM accumulators are double-buffered so
//               the epilogue of tile i overlaps the MMAs of tile i+1.
// Both operand majors are native (instruction-descriptor major bits + the
// canonical K-major / MN-major SW128 shared-memory layouts), so dX = dY W,
// dW = dY^T X and the six attention products run without transposes.  Batch
// items (b, head) are the two outer dimensions of 4-D TMA tensor maps.
//
// Tile width BN in {64, 128, 192, 256} is chosen per GEMM from a wave model
// (tiles per 148 SMs).  Causal GEMMs enumerate only the lower-triangular output
// tiles (OUT_LOWER) or order tiles heaviest-K-range first (A_LOWER / A_UPPER)
// so the static persistent schedule stays balanced.
//
// Split-K (small output grids with long K: the dW GEMMs), when the caller passes a
// workspace: split s writes alpha * (its K-range partial) to workspace slice s;
// a reduce kernel then forms C = beta*C + sum_s partial_s (+bias +residual) with
// the splits added in ascending order — one fixed association, bitwise
// reproducible.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm_common.cuh"
#include "tc_ptx.cuh"

namespace nnt {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;        // 64 bf16 = 128 B = one SW128 row
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStageBytesPerWarp = 4096;  // 32 rows x 128 B, SW128 staging for one TMA store box
constexpr int kStageBufs = 2;             // staging ring per epilogue warp (one store in flight while refilling)
constexpr int kMaxSmem = 232448;          // 227 KB opt-in dynamic shared memory per CTA
// mbarriers: full/empty per stage (<= 8 each), TMEM full/empty (2 each), per epilogue warp
// and staging buffer an epilogue-input TMA barrier (kEpiWarps * kStageBufs), the TMEM slot;
// then (at kOnesOff) the all-ones B tile of the a_rowsum MMA (R27): 16 x 16 bf16, K-major,
// no swizzle (4 core matrices of 8 rows x 16 B).
constexpr int kOnesOff = 512;
constexpr int kOnesBytes = 512;
constexpr int kBarBytes = kOnesOff + kOnesBytes;

// Epilogue specialisations (separate instantiations keep each one small and branch-light):
//   EPI_GENERIC  bias / beta*C / residual / GELU / GELU' / split-K partials
//   EPI_SCORES   fp32 C = alpha*acc (attention scores) + optional fused per-32-key-tile
//                (max, sumexp) (softmax subroutine 1)
//   EPI_DA       bf16 C = rowscale * P * (acc - D[row]) (softmax backward), P staged by TMA a
//                task ahead
//   EPI_ROWSTATS per-row (max, sumexp) over all key tiles of a row block (ORDER_ROWS tasks),
//                no C (softmax subroutine 1 with on-chip aggregation, R26)
//   EPI_SOFTMAX  bf16 C = e^{alpha*acc - M} / S from the row's stats (subroutine 2, R26)
enum EpiMode {
  EPI_GENERIC = 0, EPI_SCORES = 1, EPI_DA = 2, EPI_ROWSTATS = 3, EPI_SOFTMAX = 4, EPI_GENERIC_RS = 5, EPI_SPLITK = 6
};
// EPI_SPLITK: the generic epilogue of a split-K GEMM (fp32 C) with the in-kernel ordered reduce;
// its own instantiation, so the reduce's registers do not weigh on the unsplit GEMMs.
// EPI_GENERIC_RS: the generic epilogue plus the a_rowsum ones-vector MMAs (R27).  A separate
// instantiation: even predicated off, the extra tcgen05.mma issue sequences in the MMA loop cost
// ~30% of the single-thread issue rate (measured 422 -> 286 ns per K-block of a lone tile).
constexpr bool generic_epi(int e) { return e == EPI_GENERIC || e == EPI_GENERIC_RS || e == EPI_SPLITK; }

// CG = CTAs per MMA (tcgen05 cta_group): 1, or 2 = an SM pair computing a 256 x BN tile
// (each CTA stages its 128 A rows and half of the BN B rows; the leader issues M=256 MMAs).
// CTAS = CTAs resident per SM: the softmax passes (K = 64: one K block per tile, MUFU/latency-
// bound epilogues) run two CTAs per SM for twice the epilogue warps, in <= 113 KB each with
// fewer stages and one staging buffer per warp.
template <int BN, int CG = 1, int EPI = EPI_GENERIC>
struct Cfg {
  static constexpr int CTAS = (EPI == EPI_ROWSTATS || EPI == EPI_SOFTMAX) ? 2 : 1;
  static constexpr int BUFS = CTAS == 2 ? 1 : kStageBufs;  // staging buffers per epilogue warp
  static constexpr int SMEM_LIMIT = CTAS == 2 ? 113 * 1024 : kMaxSmem;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = BN / CG;             // B rows (N) this CTA stages
  static constexpr int B_BLKS = (B_ROWS + 63) / 64;  // MN-major B: whole 64-element blocks (a
  // 96-row pair half loads two; the MMA reads the first 96 columns)
  static constexpr int B_BYTES_K = B_ROWS * BK * 2;  // K-major B bytes per stage
  static constexpr int B_BYTES = B_BLKS * 64 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // ROWSTATS: no C staging, only the half-merge exchange slots (2 x BM float2)
  static constexpr int EPI_BYTES = EPI == EPI_ROWSTATS ? 2 * BM * 8 : kEpiWarps * BUFS * kStageBytesPerWarp;
  static constexpr int STAGES_FIT = (SMEM_LIMIT - EPI_BYTES - 1024 - kBarBytes) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  // generic epilogue with BN <= 192: 32 more columns hold the a_rowsum accumulators (R27), 16 per
  // TMEM accumulator buffer
  static constexpr bool ROWSUM = EPI == EPI_GENERIC_RS && 2 * BN + 32 <= 512;
  static constexpr int TCOLS = 2 * BN + (ROWSUM ? 32 : 0);
  static constexpr int TMEM_COLS = TCOLS <= 32 ? 32 : (TCOLS <= 64 ? 64 : (TCOLS <= 128 ? 128 : (TCOLS <= 256 ? 256 : 512)));
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int SMEM_BYTES = EPI_OFF + EPI_BYTES + 1024 /*align*/ + kBarBytes;
  static_assert(STAGES >= 2 && SMEM_BYTES <= SMEM_LIMIT, "shared memory budget");
  static_assert(CTAS * TMEM_COLS <= 512, "TMEM columns per SM");
};

// ORDER_N_OUTER: consecutive tiles walk down M for one N column (B tile shared, A streamed);
// ORDER_M_OUTER: consecutive tiles walk along N for one M row block (A shared, B streamed) -- the
// concurrent wave then reads each block of the larger operand once instead of once per wave
enum TileOrder {
  ORDER_N_OUTER = 0, ORDER_TRI = 1, ORDER_HEAVY_LOW_M = 2, ORDER_HEAVY_HIGH_M = 3, ORDER_ROWS = 4, ORDER_M_OUTER = 5
};

// n / d and n % d for a runtime divisor d >= 1 and n < 2^31 with a multiply-high and a shift
// (round-up multiplier method).  The single-thread TMA producer and MMA issuer decode a tile per
// task; with 64-bit division subroutines that decode cost ~2k cycles, more than the MMAs of a
// K = 64 attention tile.
struct FastDiv {
  uint32_t d, mul, shr;
  void init(int64_t div) {
    d = (uint32_t)(div < 1 ? 1 : div);
    shr = 0;
    while (shr < 32 && (1ull << shr) < d) ++shr;
    mul = (uint32_t)(((1ull << 32) * ((1ull << shr) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shr; }
  __device__ __forceinline__ uint32_t mod(uint32_t n, uint32_t q) const { return n - q * d; }
};

struct TcParams {
  GemmArgs g;
  int64_t mt, nt, tiles_per_batch, num_tiles, num_tasks;
  int64_t splits, kb_per_split;
  FastDiv f_splits, f_tpb, f_mt, f_nt, f_nbat, f_level, f_b1;  // divisors of the task decode
  // split-K tasks split-major (task = split * num_tiles + tile): a wave runs many tiles of ONE K
  // range, so it shares that range of both operands, instead of every K range of a few tiles
  // (which streamed all of the narrow operand once per wave); tile-major with NNT_GEMM_SPLITMAJOR=0
  int split_major;
  FastDiv f_tiles;
  uint32_t idesc;
  uint32_t idesc_ones;  // a_rowsum MMA: N = 16, B (ones) K-major
  int rowsum;           // a_rowsum requested (R27)
  int a_kmajor, b_kmajor;
  // MN-major operand through a 5-D map (make_map_blocked): all its 64-element blocks of a stage in
  // one TMA request instead of one request per block
  int a_blk, b_blk;
  int tma_store;  // epilogue stores through TMA (C / aux / workspace maps valid)
  int order;      // TileOrder
  int ws_mode;    // split partials go to the workspace map; bias/beta/residual applied by the reduce
  int in_kind;    // InKind: the epilogue input prefetched a chunk ahead (generic epilogue)
  // ws_mode with the in-kernel ordered reduce: per (tile, CTA of the pair, epilogue warp) an
  // arrival counter in the workspace; the last split to arrive adds all partials of its region
  // in split order and stores C (no reduce kernel)
  int fused_reduce;
  uint32_t* counters;
  // Stream-K (sk = 1; generic epilogue, unbatched, non-causal, splits == 1): tiles [0, sk_dp_tiles)
  // run whole (tile k*G + unit), the remaining tiles' K-block iterations (sk_iters in all) are
  // cut into G equal contiguous ranges, one per unit, so the last wave is not quantised.  A tile
  // covered by several units is finished by the unit holding its last K-block: it adds the other
  // units' fp32 partials (sk_part slots, one per unit and CTA) in a fixed order, behind per-warp
  // flags in the counter zone.
  int sk;
  int64_t sk_dp_tiles, sk_iters, nkb;
  float* sk_part;
  // Narrow tail tiles (generic epilogues, N % BN != 0): the last N column of tiles (n0 == tail_n0)
  // runs its MMAs with N = tail_n (the column remainder rounded up to 32) instead of BN, the CTAs
  // of a pair staging tail_n / 2 B rows each, so no tensor-core cycles go to the zero-filled
  // columns; with tail_last (ORDER_M_OUTER) those cheap tiles are enumerated after every full
  // tile, so they fill the persistent schedule's last round.  tail_n0 = -1: off.
  int64_t tail_n0;
  int tail_n, tail_last;
  uint32_t idesc_tail;
  FastDiv f_ntf;  // nt - 1 (tail_last)
};

// Stream-K roles of a unit's work item
enum SkRole { SK_FULL = 0, SK_WRITER = 1, SK_FINISHER = 2 };

// PTX helpers (mbarrier, TMA, tcgen05 MMA / TMEM, smem descriptors): tc_ptx.cuh

// Output tiles per task: 1, or (ORDER_ROWS) the key tiles of the task's row block.
__device__ __forceinline__ int64_t task_subtiles(const TcParams& P, int64_t t, int bn) {
  if (P.order != ORDER_ROWS) return 1;
  const int64_t mb = P.mt - 1 - (int64_t)P.f_nbat.div((uint32_t)t);  // splits == 1
  if (P.g.causal == NNT_CAUSAL_OUT_LOWER) return min(P.nt, ((mb + 1) * BM + bn - 1) / bn);
  return P.nt;
}

// The static persistent schedule, walked identically by the producer, MMA and epilogue roles:
// CTA (pair) c of G takes task k*G + c in even rounds k and k*G + G-1-c in odd rounds
// (boustrophedon), which balances the heaviest-first causal orders; ORDER_ROWS tasks are
// walked tile by tile (sub).
struct TaskIter {
  int64_t c, G, k, t, sub;
  __device__ __forceinline__ TaskIter(int64_t c_, int64_t G_) : c(c_), G(G_), k(0), t(c_), sub(0) {}
  __device__ __forceinline__ static int64_t at(int64_t c, int64_t G, int64_t k) {
    return k * G + ((k & 1) ? (G - 1 - c) : c);
  }
  __device__ __forceinline__ int64_t next_task() const { return at(c, G, k + 1); }
  __device__ __forceinline__ void next(const TcParams& P, int bn) {
    if (++sub >= task_subtiles(P, t, bn)) {
      sub = 0;
      ++k;
      t = at(c, G, k);
    }
  }
};

// Which tile a task computes and which K-blocks it covers (nnt_causal semantics + split-K).
struct TileInfo {
  int64_t tile, bz, m0, n0, kb_begin, kb_end, split;
  int p, q;  // batch item (bz = p * batch1 + q)
};
// bm_tile: output rows per task (BM, or 2*BM for a CTA pair); row_off: this CTA's first row
// within the task's tile (CTA-pair rank * BM).  Causal orders are single-CTA only.
// ORDER_ROWS: a task is one (batch item, row block) and owns all its key tiles; j = key tile.
// 32-bit index math with precomputed divisors (host guarantees num_tasks < 2^31).
__device__ __forceinline__ TileInfo decode_task(const TcParams& P, int64_t t, int bn, int bm_tile = BM,
                                                int row_off = 0, int64_t j = 0) {
  TileInfo ti;
  const uint32_t tt = (uint32_t)t;
  uint32_t tile;
  if (P.split_major) {
    ti.split = P.f_tiles.div(tt);
    tile = P.f_tiles.mod(tt, (uint32_t)ti.split);
  } else {
    tile = P.f_splits.div(tt);
    ti.split = P.f_splits.mod(tt, tile);
  }
  ti.tile = tile;
  uint32_t mb, nb, bz;
  if (P.order == ORDER_ROWS) {
    // heaviest row blocks first (causal: row block mb holds mb+1 key tiles)
    const uint32_t level = P.f_nbat.div(tile);
    bz = P.f_nbat.mod(tile, level);
    mb = (uint32_t)P.mt - 1 - level;
    nb = (uint32_t)j;
  } else if (P.order == ORDER_TRI) {
    // compact lower-triangular enumeration (BN == BM, square grid): row mb holds mb+1 tiles
    bz = P.f_tpb.div(tile);
    const uint32_t r = P.f_tpb.mod(tile, bz);
    mb = (uint32_t)((sqrtf(8.0f * (float)r + 1.0f) - 1.0f) * 0.5f);
    while ((mb + 1) * (mb + 2) / 2 <= r) ++mb;
    while (mb * (mb + 1) / 2 > r) --mb;
    nb = r - mb * (mb + 1) / 2;
  } else if (P.order == ORDER_N_OUTER) {
    bz = P.f_tpb.div(tile);
    const uint32_t r = P.f_tpb.mod(tile, bz);
    nb = P.f_mt.div(r);
    mb = P.f_mt.mod(r, nb);
  } else if (P.order == ORDER_M_OUTER) {
    bz = P.f_tpb.div(tile);
    const uint32_t r = P.f_tpb.mod(tile, bz);
    const uint32_t full = P.tail_last ? (uint32_t)(P.mt * (P.nt - 1)) : 0xffffffffu;
    if (r >= full) {  // the narrow tail column, after every full tile; the last row blocks first
      // (their A blocks are the ones the concurrent full tiles are streaming / most recently used)
      mb = (uint32_t)P.mt - 1 - (r - full);
      nb = (uint32_t)P.nt - 1;
    } else if (P.tail_last) {
      mb = P.f_ntf.div(r);
      nb = P.f_ntf.mod(r, mb);
    } else {
      mb = P.f_nt.div(r);
      nb = P.f_nt.mod(r, mb);
    }
  } else {
    // heaviest K-range first: the m-block level is outermost, (batch, n) inner
    const uint32_t level = P.f_level.div(tile), r = P.f_level.mod(tile, level);
    mb = P.order == ORDER_HEAVY_HIGH_M ? (uint32_t)P.mt - 1 - level : level;
    bz = P.f_nt.div(r);
    nb = P.f_nt.mod(r, bz);
  }
  ti.bz = bz;
  ti.p = (int)P.f_b1.div(bz);
  ti.q = (int)P.f_b1.mod(bz, (uint32_t)ti.p);
  ti.m0 = (int64_t)mb * bm_tile + row_off;
  ti.n0 = (int64_t)nb * bn;
  int64_t k_begin = 0, k_end = P.g.K;
  if (P.g.causal == NNT_CAUSAL_A_LOWER) k_end = min(P.g.K, ti.m0 + BM);
  if (P.g.causal == NNT_CAUSAL_A_UPPER) k_begin = min(P.g.K, ti.m0);
  const int64_t kb0 = k_begin / BK, kb1 = (k_end + BK - 1) / BK;
  ti.kb_begin = min(kb1, kb0 + ti.split * P.kb_per_split);
  ti.kb_end = min(kb1, ti.kb_begin + P.kb_per_split);
  return ti;
}

// A unit's (CTA or CTA pair's) work list, walked identically by the producer, MMA and epilogue
// roles: the static task schedule (TaskIter), or with P.sk the stream-K list
//   [writer segment] [whole data-parallel tiles] [whole stream-K tiles] [finisher segment]
// Unit c owns iterations [s0, s1) = [c I / G, (c+1) I / G) of the stream-K tiles' (tile-major,
// K-block-minor) iteration space.  Its segment in the tile holding s1 - 1 ends before that tile's
// last K-block when s1 is not a tile boundary: a WRITER segment, processed first (its partial is
// stored early).  Its segment in the tile holding s0 starts after that tile's first K-block when s0
// is not a boundary: a FINISHER segment (it holds the tile's last K-block), processed last; the
// units it waits for are lower-numbered and wrote their partial as their first item, so the waits
// always point at work that never waits (no deadlock; launched in index order).
struct Walk {
  TaskIter it;
  int64_t j, n, s0, s1, n_dp, tf0, tf1;
  int has_w, has_f;
  __device__ __forceinline__ Walk(const TcParams& P, int64_t c, int64_t G) : it(c, G), j(0), n(0) {
    if (!P.sk) return;
    const int64_t I = P.sk_iters, nkb = P.nkb;
    s0 = c * I / G;
    s1 = (c + 1) * I / G;
    n_dp = P.sk_dp_tiles > c ? (P.sk_dp_tiles - c + G - 1) / G : 0;
    has_w = has_f = 0;
    tf0 = tf1 = 0;
    if (s1 > s0) {
      has_w = (s1 % nkb) != 0;
      has_f = (s0 % nkb) != 0 && !(s0 / nkb == (s1 - 1) / nkb && has_w);
      tf0 = (s0 + nkb - 1) / nkb;
      tf1 = s1 / nkb;
      if (tf1 < tf0) tf1 = tf0;
    }
    n = has_w + n_dp + (tf1 - tf0) + has_f;
  }
  __device__ __forceinline__ bool ok(const TcParams& P) const { return P.sk ? j < n : it.t < P.num_tasks; }
  __device__ __forceinline__ void next(const TcParams& P, int bn) {
    if (P.sk)
      ++j;
    else
      it.next(P, bn);
  }
  __device__ __forceinline__ TileInfo info(const TcParams& P, int bn, int bm_tile, int row_off, int& role) const {
    if (!P.sk) {
      role = SK_FULL;
      return decode_task(P, it.t, bn, bm_tile, row_off, it.sub);
    }
    const int64_t nkb = P.nkb, dp = P.sk_dp_tiles;
    int64_t jj = j, tile, kb0 = 0, kb1 = nkb;
    role = SK_FULL;
    if (jj < has_w) {
      const int64_t t1 = (s1 - 1) / nkb;
      tile = dp + t1;
      kb0 = (s0 > t1 * nkb ? s0 : t1 * nkb) - t1 * nkb;
      kb1 = s1 - t1 * nkb;
      role = SK_WRITER;
    } else if ((jj -= has_w) < n_dp) {
      tile = jj * it.G + it.c;
    } else if ((jj -= n_dp) < tf1 - tf0) {
      tile = dp + tf0 + jj;
    } else {
      const int64_t t0 = s0 / nkb;
      tile = dp + t0;
      kb0 = s0 - t0 * nkb;
      role = SK_FINISHER;
    }
    TileInfo ti = decode_task(P, tile, bn, bm_tile, row_off, 0);
    ti.kb_begin = kb0;
    ti.kb_end = kb1;
    return ti;
  }
};

// Stream-K partial slot of (unit, CTA rank): [BN/4][BM][4] fp32 -- a warp's float4 accesses for
// one column quad cover 32 consecutive rows (512 contiguous bytes)
__device__ __forceinline__ float* sk_slot(const TcParams& P, int64_t unit, uint32_t rank, int cg, int bn) {
  return P.sk_part + ((size_t)unit * cg + rank) * (size_t)BM * bn;
}
__device__ __forceinline__ uint32_t* sk_flag(const TcParams& P, int64_t unit, uint32_t rank, int cg, int epi_warp) {
  return P.counters + ((size_t)unit * cg + rank) * kEpiWarps + epi_warp;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ epilogue math
template <bool kFast>
__device__ __forceinline__ float tanh_f(float x) {
  if (kFast) {  // bf16 outputs: tanh.approx (rel err ~2^-11) is below bf16 rounding
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  return tanhf(x);  // fp32 outputs: accurate tanh (R15)
}
template <bool kFast>
__device__ __forceinline__ float gelu_e(float u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  return 0.5f * u * (1.0f + tanh_f<kFast>(c * (u + a * u * u * u)));
}
template <bool kFast>
__device__ __forceinline__ float gelu_grad_e(float u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float t = tanh_f<kFast>(c * (u + a * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * c * (1.0f + 3.0f * a * u * u);
}

// Packed fp32x2 forms (sm_100 FFMA2/FMUL2/FADD2: two lanes of fp32 math per instruction) of
// the epilogue activations, for bf16 outputs (tanh.approx): same formulas as gelu_e / gelu_grad_e
// up to fp32 rounding order.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 tanh2_approx(float2 z) { return make_float2(tanh_f<true>(z.x), tanh_f<true>(z.y)); }
__device__ __forceinline__ float2 gelu2(float2 u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float2 u2 = __fmul2_rn(u, u);
  const float2 z = __fmul2_rn(__fmul2_rn(u, f2(c)), __ffma2_rn(u2, f2(a), f2(1.f)));  // c u (1 + a u^2)
  const float2 hu = __fmul2_rn(u, f2(0.5f));
  return __ffma2_rn(hu, tanh2_approx(z), hu);  // u/2 (1 + t)
}
__device__ __forceinline__ float2 gelu_grad2(float2 u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float2 u2 = __fmul2_rn(u, u);
  const float2 z = __fmul2_rn(__fmul2_rn(u, f2(c)), __ffma2_rn(u2, f2(a), f2(1.f)));
  const float2 t = tanh2_approx(z);
  const float2 ne = __fmul2_rn(u, __ffma2_rn(u2, f2(-3.f * a * c), f2(-c)));  // -u c (1 + 3 a u^2)
  const float2 m = __ffma2_rn(t, t, f2(-1.f));                                // t^2 - 1
  const float2 h = __ffma2_rn(ne, m, t);                                      // t + u c (1+3au^2)(1-t^2)
  return __ffma2_rn(h, f2(0.5f), f2(0.5f));
}

template <typename T>
__device__ __forceinline__ float ld_elem(const T* p) { return to_f32(*p); }
// C may have been written by TMA stores of this kernel's earlier launches: bypass L1.
__device__ __forceinline__ float ld_c(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float ld_c(const __nv_bfloat16* p) {
  unsigned short u = __ldcg(reinterpret_cast<const unsigned short*>(p));
  return __bfloat162float(__ushort_as_bfloat16(u));
}

// 8 consecutive values as floats (one 16-byte load for bf16, two for fp32)
__device__ __forceinline__ void ld8(const float* p, float* o, bool cg) {
  float4 a = cg ? __ldcg(reinterpret_cast<const float4*>(p)) : *reinterpret_cast<const float4*>(p);
  float4 b = cg ? __ldcg(reinterpret_cast<const float4*>(p) + 1) : *(reinterpret_cast<const float4*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* o, bool cg) {
  uint4 u = cg ? __ldcg(reinterpret_cast<const uint4*>(p)) : *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float2 f = __bfloat1622float2(h[t]);
    o[2 * t] = f.x;
    o[2 * t + 1] = f.y;
  }
}

// The streamed (prefetched) epilogue input of a GEMM: at most one, element type = C's.
// IN_AUX_SMEM: the aux chunk is TMA-loaded into the chunk's staging buffer at tile start
// (before the accumulator wait) and read from shared memory; the output overwrites it in place.
// IN_RES_SMEM: the same for an fp32 residual, with more chunks per warp and tile than staging
// buffers: the first kStageBufs chunks load at tile start, chunk i + kStageBufs into buffer
// i % kStageBufs once chunk i's store has read it.
enum InKind { IN_NONE = 0, IN_AUX = 1, IN_RESIDUAL = 2, IN_COLD = 3, IN_AUX_SMEM = 4, IN_RES_SMEM = 5 };

// The W pre-activation outputs of one row chunk (GELU is applied by the caller after
// staging the pre-activation).  vec: operands 16-byte aligned with 16-byte pitches.
// raw: the prefetched chunk of input `in_kind` (valid when vec and the chunk is full).
template <typename TC, int W>
__device__ __forceinline__ void epi_math(const GemmArgs& g, const TC* Cb, const TC* auxb, int64_t row, int64_t col0,
                                         bool extras, bool vec, float dval, int in_kind, const Raw8& raw,
                                         float (&v)[W], bool with_alpha = true) {
  constexpr bool kFast = sizeof(TC) == 2;
  if (with_alpha && g.alpha != 1.f) {
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      const float2 x = __fmul2_rn(make_float2(v[j], v[j + 1]), f2(g.alpha));
      v[j] = x.x;
      v[j + 1] = x.y;
    }
  }
  if (!extras) return;  // split-K partial: bias/beta/residual belong to the reduce
  if (g.act == NNT_ACT_SOFTMAX_BWD) {
    // dA = scale * P * (dP - D): aux holds P with C's layout, dval = D of this row
    if (row < g.M) {
      const TC* ar = auxb + row * g.ld_aux + col0;
      if (vec && col0 + W <= g.N) {
        float t[8];
#pragma unroll
        for (int j = 0; j < W; j += 8) {
          ld8(ar + j, t, false);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[j + i] = g.rowscale * t[i] * (v[j + i] - dval);
        }
      } else {
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = col0 + j < g.N ? g.rowscale * ld_elem(ar + j) * (v[j] - dval) : 0.f;
      }
    }
    return;
  }
  if (vec && row < g.M && col0 + W <= g.N) {
    float t[8];
    auto add8 = [&](int j) {  // v[j..j+8) += t, two lanes per FADD2
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const float2 x = __fadd2_rn(make_float2(v[j + i], v[j + i + 1]), make_float2(t[i], t[i + 1]));
        v[j + i] = x.x;
        v[j + i + 1] = x.y;
      }
    };
    if (g.bias) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        ld8(g.bias + col0 + j, t, false);
        add8(j);
      }
    }
    if (g.beta != 0.f) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        if (in_kind == IN_COLD)
          unpack8<TC>(raw, j, t);
        else
          ld8(Cb + row * g.ldc + col0 + j, t, true);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[j + i] += g.beta * t[i];
      }
    }
    if (g.residual) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        if (in_kind == IN_RESIDUAL)
          unpack8<float>(raw, j, t);
        else
          ld8(g.residual + row * g.ld_res + col0 + j, t, false);
        add8(j);
      }
    }
    if (g.act == NNT_ACT_GELU_BWD) {
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        if (in_kind == IN_AUX)
          unpack8<TC>(raw, j, t);
        else
          ld8(auxb + row * g.ld_aux + col0 + j, t, false);
        if constexpr (kFast) {
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float2 x = __fmul2_rn(make_float2(v[j + i], v[j + i + 1]), gelu_grad2(make_float2(t[i], t[i + 1])));
            v[j + i] = x.x;
            v[j + i + 1] = x.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[j + i] *= gelu_grad_e<kFast>(t[i]);
        }
      }
    }
  } else if (row < g.M) {
    const bool full = col0 + W <= g.N;
    if (g.bias) {
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] += __ldg(g.bias + col0 + j);
    }
    if (g.beta != 0.f) {
      const TC* cr = Cb + row * g.ldc + col0;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] += g.beta * ld_c(cr + j);
    }
    if (g.residual) {
      const float* rr = g.residual + row * g.ld_res + col0;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] += rr[j];
    }
    if (g.act == NNT_ACT_GELU_BWD) {
      const TC* ar = auxb + row * g.ld_aux + col0;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] *= gelu_grad_e<kFast>(ld_elem(ar + j));
    }
  }
}

template <typename TC, int W>
__device__ __forceinline__ void direct_store(int64_t M, int64_t N, int64_t ld, TC* base, int64_t row, int64_t col0,
                                             const float (&v)[W]) {
  if (row >= M) return;
  TC* dst = base + row * ld + col0;
  if (col0 + W <= N && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {  // 16-byte vector stores
#pragma unroll
    for (int j = 0; j < W; j += 16 / (int)sizeof(TC)) {
      uint4 u;
      if (sizeof(TC) == 4) {
        u = make_uint4(__float_as_uint(v[j]), __float_as_uint(v[j + 1]), __float_as_uint(v[j + 2]),
                       __float_as_uint(v[j + 3]));
      } else {
        __nv_bfloat162 t0 = __floats2bfloat162_rn(v[j], v[j + 1]), t1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]), t3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
        u = make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                       *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
      }
      *reinterpret_cast<uint4*>(dst + j) = u;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (col0 + j < N) dst[j] = from_f32<TC>(v[j]);
}

// ------------------------------------------------------------------ kernel

// CG = 2: launched as clusters of 2 CTAs (an SM pair).  Task = 256 x BN output tile; rank r
// stages A rows [m0 + 128 r, +128) and B rows [n0 + r BN/2, +BN/2) and drains its own TMEM
// (rows m0 + 128 r ..); the leader (rank 0) waits for both halves on its full barrier
// (expect_tx of both CTAs' bytes) and issues the M=256 MMAs; the peer's epilogue warps arrive
// on the leader's TMEM-empty barrier.
template <int BN, typename TC, int EPI, int CG = 1>
__global__ void __launch_bounds__(kThreads, (Cfg<BN, CG, EPI>::CTAS))
    gemm_tc_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmAux) {
  static_assert(CG == 1 || (CG == 2 && generic_epi(EPI) && (BN / 2) % 32 == 0), "CTA-pair configuration");
  using C = Cfg<BN, CG, EPI>;
  static_assert(EPI != EPI_DA || C::BUFS == 2, "EPI_DA double-buffers P");
  constexpr int W = 128 / (int)sizeof(TC);  // columns per 128-byte staging row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::EPI_OFF + C::EPI_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;  // [kEpiWarps][kStageBufs]: epilogue-input TMA loads (IN_AUX_SMEM)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inbar + kEpiWarps * kStageBufs);
  static_assert((2 * 8 + 4 + kEpiWarps * kStageBufs) * 8 + 4 <= kOnesOff, "barrier area");
  uint8_t* const ones = reinterpret_cast<uint8_t*>(bars) + kOnesOff;  // a_rowsum B operand (R27)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GemmArgs& g = P.g;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int row_off = (int)rank * BM;
  const int64_t task0 = blockIdx.x / CG, task_step = gridDim.x / CG;

  if constexpr (C::ROWSUM) {
    if (P.rowsum && warp == 2) {  // bf16 ones (0x3F80), visible to the tensor cores (async proxy)
      reinterpret_cast<uint4*>(ones)[lane] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
      fence_async_smem();
    }
  }

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), kEpiWarps * CG);
    }
    for (int s = 0; s < kEpiWarps * kStageBufs; ++s) mbar_init(smem_u32(&inbar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrive / complete_tx
    __syncthreads();     // (also a CTA barrier for the TMEM-address slot: racecheck does not model the cluster one)
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: everything above (barrier init, TMEM allocation, tensor-map prefetch) overlapped the
  // previous kernel's tail; inputs are read only after it has completed
  NNT_PDL_ENTRY();

  if (warp == 0) {
    // ===================== TMA producer (warp-wide, elected issue)
    {
      int stage = 0;
      uint32_t phase = 0;
      for (Walk wk(P, task0, task_step); wk.ok(P); wk.next(P, BN)) {
        int role;
        TileInfo ti = wk.info(P, BN, BM * CG, row_off, role);
        const int p = ti.p, q = ti.q;
        // this CTA's B rows (a narrow tail tile: tail_n / CG rows per CTA, the MMA's N / 2 each)
        const int nb0 = (int)ti.n0 + (int)rank * ((ti.n0 == P.tail_n0 ? P.tail_n : BN) / CG);
        for (int64_t kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
          const int k0 = (int)(kb * BK);
          const uint32_t stage_tx = C::A_BYTES + (P.b_kmajor ? C::B_BYTES_K : C::B_BYTES);
          if constexpr (CG == 2) {
            const uint32_t fb_local = smem_u32(&full[stage]);
            if (rank == 0) mbar_expect_tx_w(fb_local, CG * stage_tx);
            const uint32_t fb = map_to_rank(fb_local, 0);
            if (P.a_kmajor) {
              tma_load_4d_pair_w(sa, &tmA, fb, k0, (int)ti.m0, q, p);
            } else if (P.a_blk) {
              tma_load_5d_pair_w(sa, &tmA, fb, 0, k0, (int)ti.m0 / 64, q, p);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_4d_pair_w(sa + j * 8192, &tmA, fb, (int)ti.m0 + 64 * j, k0, q, p);
            }
            if (P.b_kmajor) {
              tma_load_4d_pair_w(sb, &tmB, fb, k0, nb0, q, p);
            } else if (P.b_blk) {
              tma_load_5d_pair_w(sb, &tmB, fb, 0, k0, nb0 / 64, q, p);
            } else {
#pragma unroll
              for (int j = 0; j < C::B_BLKS; ++j) tma_load_4d_pair_w(sb + j * 8192, &tmB, fb, nb0 + 64 * j, k0, q, p);
            }
          } else {
            const uint32_t fb = smem_u32(&full[stage]);
            mbar_expect_tx_w(fb, stage_tx);
            if (P.a_kmajor) {
              tma_load_4d_w(sa, &tmA, fb, k0, (int)ti.m0, q, p);
            } else if (P.a_blk) {
              tma_load_5d_w(sa, &tmA, fb, 0, k0, (int)ti.m0 / 64, q, p);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_4d_w(sa + j * 8192, &tmA, fb, (int)ti.m0 + 64 * j, k0, q, p);
            }
            if (P.b_kmajor) {
              tma_load_4d_w(sb, &tmB, fb, k0, (int)ti.n0, q, p);
            } else if (P.b_blk) {
              tma_load_5d_w(sb, &tmB, fb, 0, k0, (int)ti.n0 / 64, q, p);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_4d_w(sb + j * 8192, &tmB, fb, (int)ti.n0 + 64 * j, k0, q, p);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // every operand load of this CTA is issued: with PDL the next kernel on the stream may be
      // scheduled now (its CTAs wait in griddepcontrol.wait until this grid completes), hiding its
      // launch behind this CTA's last MMAs and epilogue
      pdl_trigger();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (CTA pair: the leader only)
    if (rank == 0) {  // warp-wide loop, elected issue
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart; +32 B per UMMA_K=16.
      // MN-major SW128: 64-element MN blocks LBO = 8 KB apart, 8-row K groups SBO = 1 KB
      // apart; +2 KB per UMMA_K=16.
      const uint32_t a_lbo = P.a_kmajor ? 16u : 8192u, b_lbo = P.b_kmajor ? 16u : 8192u;
      const uint32_t a_step = P.a_kmajor ? 32u : 2048u, b_step = P.b_kmajor ? 32u : 2048u;
      for (Walk wk(P, task0, task_step); wk.ok(P); wk.next(P, BN)) {
        int role;
        TileInfo ti = wk.info(P, BN, BM * CG, row_off, role);
        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        // narrow tail tile: N = tail_n (the epilogue reads past it only into clipped columns >= N)
        const uint32_t idesc = ti.n0 == P.tail_n0 ? P.idesc_tail : P.idesc;
        for (int64_t kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t ad = make_sdesc(sa + kk * a_step, a_lbo, 1024u);
            uint64_t bd = make_sdesc(sb + kk * b_step, b_lbo, 1024u);
            if constexpr (CG == 2)
              mma_bf16_pair_w(tmem_d, ad, bd, idesc, (kb > ti.kb_begin || kk > 0) ? 1u : 0u);
            else
              mma_bf16_w(tmem_d, ad, bd, idesc, (kb > ti.kb_begin || kk > 0) ? 1u : 0u);
            if constexpr (C::ROWSUM) {
              // R27: sum_k op(A)[i][k] = op(A) x ones, into 16 columns past the two accumulators
              // (the first N tile of each row block only)
              if (P.rowsum && ti.n0 == 0) {
                const uint64_t od = make_sdesc_noswz(smem_u32(ones), 128u, 256u);
                const uint32_t tr = tmem_base + (uint32_t)(2 * BN + acc * 16);
                if constexpr (CG == 2)
                  mma_bf16_pair_w(tr, ad, od, P.idesc_ones, (kb > ti.kb_begin || kk > 0) ? 1u : 0u);
                else
                  mma_bf16_w(tr, ad, od, P.idesc_ones, (kb > ti.kb_begin || kk > 0) ? 1u : 0u);
              }
            }
          }
          if constexpr (CG == 2)
            mma_commit_pair_w(smem_u32(&empty[stage]));
          else
            mma_commit_w(smem_u32(&empty[stage]));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2)
          mma_commit_pair_w(smem_u32(&tfull[acc]));
        else
          mma_commit_w(smem_u32(&tfull[acc]));
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if constexpr (!generic_epi(EPI)) {
    // ===================== specialised epilogues (attention score-type GEMMs)
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    uint8_t* const stage_base = smem + C::EPI_OFF + (warp - 2) * C::BUFS * kStageBytesPerWarp;
    int ring = 0;
    const float L2E = 1.4426950408889634f;
    int acc = 0;
    uint32_t acc_phase = 0;
    // EPI_ROWSTATS: running (max, sumexp) of this lane's row over this half's columns of the
    // task's key tiles (online merge rule of R10); the quadrant's two halves combine at task end
    float m_run = -INFINITY, l_run = 0.f;
    int xbuf = 0;
    const float sc_c = g.alpha * L2E;  // EPI_ROWSTATS / EPI_SOFTMAX: e^{alpha*a} = 2^{a*sc_c}
    // columns per chunk: a 128-byte staging row of C, or (ROWSTATS, no C) 64 columns so one
    // wait covers two TMEM loads and the exp chain has twice the independent work
    constexpr int WE = EPI == EPI_ROWSTATS ? 64 : W;
    static_assert(EPI != EPI_DA || BN == 2 * W, "EPI_DA: one P chunk per epilogue warp and task");
    // EPI_DA: P chunk loads (TMA, aux map) into this warp's staging buffer b
    int da_buf = 0;
    uint32_t da_phase = 0;
    auto da_load = [&](const TileInfo& tt, int b) {
      const uint32_t bar = smem_u32(&inbar[(warp - 2) * kStageBufs + b]);
      mbar_expect_tx(bar, kStageBytesPerWarp);
      tma_load_4d(smem_u32(stage_base + b * kStageBytesPerWarp), &tmAux, bar, (int)tt.n0 + half * W,
                  (int)tt.m0 + quad * 32, tt.q, tt.p);
    };
    if constexpr (EPI == EPI_DA) {
      if (lane == 0 && task0 < P.num_tasks) da_load(decode_task(P, task0, BN), 0);
    }
    for (TaskIter it(task0, task_step); it.t < P.num_tasks; it.next(P, BN)) {
      const int64_t t = it.t, sub = it.sub;
      TileInfo ti = decode_task(P, t, BN, BM, 0, sub);
      const int p = ti.p, q = ti.q;
      const int row_in = (int)ti.m0 + quad * 32 + lane;  // row of this lane within the batch item
      const bool row_ok = row_in < g.M;
      const int cy = (int)ti.m0 + quad * 32;
      const int c_first = half * WE;
      // EPI_DA: this warp's P chunk of the task (BN == 2W: one chunk per warp) arrives by TMA in
      // staging buffer da_buf, loaded during the previous task; the next task's chunk is
      // prefetched into the other buffer now, once the store that last used it has read it
      Raw8 raw;
      float dval = 0.f;
      if constexpr (EPI == EPI_DA) {
        if (lane == 0) {
          bulk_wait_read0();
          const int64_t tn = it.next_task();  // (EPI_DA tasks are single tiles)
          if (tn < P.num_tasks) da_load(decode_task(P, tn, BN), da_buf ^ 1);
        }
        __syncwarp();
        dval = row_ok ? __ldg(g.rowvec + ti.bz * g.M + row_in) : 0.f;
      }
      // EPI_SOFTMAX: the row's (M, S) from the statistics pass
      float sm_ml = 0.f, sm_inv = 0.f;
      if constexpr (EPI == EPI_SOFTMAX) {
        if (row_ok) {
          const float2 rs = __ldg(reinterpret_cast<const float2*>(g.row_stats) + ti.bz * g.M + row_in);
          sm_ml = rs.x * L2E;
          sm_inv = 1.f / rs.y;
        }
      }
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const bool has_k = ti.kb_end > ti.kb_begin;
#pragma unroll 1
      for (int c = c_first; c < BN; c += 2 * WE) {
        if (ti.n0 + c >= g.N) break;  // warp-uniform
        const int col0 = (int)ti.n0 + c;
        float v[WE];
        if (has_k) {
          tmem_ld_cols<WE / 32>(tmem_base + (uint32_t)(acc * BN + c) + ((uint32_t)(quad * 32) << 16), v);
        } else {
#pragma unroll
          for (int j = 0; j < WE; ++j) v[j] = 0.f;
        }
        if constexpr (EPI == EPI_SCORES) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] *= g.alpha;
          if (g.row_stats != nullptr && row_ok) {
            // softmax subroutine 1 on this 32-key tile; warp-uniform fast path when every lane's
            // row sees all 32 columns (causal: col0 + 31 <= smallest row of the warp)
            const bool all_valid = (col0 + 32 <= g.N) && (g.causal != NNT_CAUSAL_OUT_LOWER || col0 + 31 <= cy);
            float m, s = 0.f;
            if (all_valid) {
              float m0 = fmaxf(v[0], v[1]), m1 = fmaxf(v[2], v[3]);
#pragma unroll
              for (int j = 4; j < 32; j += 4) {
                m0 = fmaxf(m0, fmaxf(v[j], v[j + 1]));
                m1 = fmaxf(m1, fmaxf(v[j + 2], v[j + 3]));
              }
              m = fmaxf(m0, m1);
              const float ml = m * L2E;
              float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                s0 += exp2f(fmaf(v[j], L2E, -ml));
                s1 += exp2f(fmaf(v[j + 1], L2E, -ml));
                s2 += exp2f(fmaf(v[j + 2], L2E, -ml));
                s3 += exp2f(fmaf(v[j + 3], L2E, -ml));
              }
              s = (s0 + s1) + (s2 + s3);
            } else {
              int lim = g.N - col0;
              if (g.causal == NNT_CAUSAL_OUT_LOWER && row_in - col0 + 1 < lim) lim = row_in - col0 + 1;
              m = -INFINITY;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < lim) m = fmaxf(m, v[j]);
              if (m != -INFINITY) {
                const float ml = m * L2E;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j < lim) s += exp2f(fmaf(v[j], L2E, -ml));
              }
            }
            reinterpret_cast<float2*>(g.row_stats)[(ti.bz * g.M + row_in) * g.ld_stats + col0 / 32] =
                make_float2(m, s);
          }
        } else if constexpr (EPI == EPI_ROWSTATS) {
          // subroutine 1 on this 32-key chunk, merged into the running (m, l): no C store.
          // (per-lane branch only: the next chunk's tcgen05.ld is warp-collective)
          // m_run is kept in accumulator units (alpha > 0: max(alpha*acc) = alpha*max(acc)
          // exactly); e^{alpha*acc - alpha*m} = 2^{acc*c - m*c} with c = alpha*log2(e)
          int lim = row_ok ? g.N - col0 : 0;
          if (g.causal == NNT_CAUSAL_OUT_LOWER && row_in - col0 + 1 < lim) lim = row_in - col0 + 1;
          if (lim > 0) {
            if (lim < WE) {
#pragma unroll
              for (int j = 0; j < WE; ++j)
                if (j >= lim) v[j] = -INFINITY;
            }
            float mx[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) mx[i] = fmaxf(v[i], v[i + 4]);
#pragma unroll
            for (int j = 8; j < WE; j += 8)
#pragma unroll
              for (int i = 0; i < 4; ++i) mx[i] = fmaxf(mx[i], fmaxf(v[j + i], v[j + 4 + i]));
            const float m_new = fmaxf(m_run, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])));  // finite
            const float mc = m_new * sc_c;
            float2 s[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) s[i] = f2(0.f);
#pragma unroll
            for (int j = 0; j < WE; j += 8)  // 2^{-inf} = 0 for the masked columns
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 x = __ffma2_rn(make_float2(v[j + 2 * i], v[j + 2 * i + 1]), f2(sc_c), f2(-mc));
                s[i] = __fadd2_rn(s[i], make_float2(ex2_approx(x.x), ex2_approx(x.y)));
              }
            const float st = ((s[0].x + s[0].y) + (s[1].x + s[1].y)) + ((s[2].x + s[2].y) + (s[3].x + s[3].y));
            l_run = fmaf(l_run, ex2_approx((m_run - m_new) * sc_c), st);
            m_run = m_new;
          }
          continue;
        } else if constexpr (EPI == EPI_SOFTMAX) {
          // subroutine 2: P = e^{x - M} / S on the recomputed scores; masked entries 0
          int lim = g.N - col0;
          if (g.causal == NNT_CAUSAL_OUT_LOWER && row_in - col0 + 1 < lim) lim = row_in - col0 + 1;
          if (!row_ok) lim = 0;
          if (lim >= W) {
#pragma unroll
            for (int j = 0; j < W; j += 2) {
              const float2 x = __ffma2_rn(make_float2(v[j], v[j + 1]), f2(sc_c), f2(-sm_ml));
              const float2 y = __fmul2_rn(make_float2(ex2_approx(x.x), ex2_approx(x.y)), f2(sm_inv));
              v[j] = y.x;
              v[j + 1] = y.y;
            }
          } else {
#pragma unroll
            for (int j = 0; j < W; ++j) v[j] = j < lim ? ex2_approx(fmaf(v[j], sc_c, -sm_ml)) * sm_inv : 0.f;
          }
        } else {
          // dA = rowscale * P * (dP - D) with P from staging buffer da_buf (zero-filled past M / N;
          // those outputs are clipped by the TMA store)
          mbar_wait(smem_u32(&inbar[(warp - 2) * kStageBufs + da_buf]), (da_phase >> da_buf) & 1u);
          da_phase ^= 1u << da_buf;
          unstage_row(raw, stage_base + da_buf * kStageBytesPerWarp, lane);
          float t[8];
#pragma unroll
          for (int j = 0; j < W; j += 8) {
            unpack8<TC>(raw, j, t);
#pragma unroll
            for (int i = 0; i < 8; i += 2) {  // (rowscale * P) * (dP - D), same rounding order
              const float2 d = __fadd2_rn(make_float2(v[j + i], v[j + i + 1]), f2(-dval));
              const float2 y = __fmul2_rn(__fmul2_rn(make_float2(t[i], t[i + 1]), f2(g.rowscale)), d);
              v[j + i] = y.x;
              v[j + i + 1] = y.y;
            }
          }
          ring = da_buf;  // the output overwrites P in place
        }
        if constexpr (EPI != EPI_ROWSTATS) {  // (ROWSTATS has no C)
          // stage + TMA store (2-buffer ring per warp)
          uint8_t* buf = stage_base + ring * kStageBytesPerWarp;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::BUFS - 1) : "memory");
          __syncwarp();
          stage_row<TC, W>(buf, lane, v);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmC, smem_u32(buf), col0, cy, q, p);
            bulk_commit();
          }
          ring = ring + 1 == C::BUFS ? 0 : ring + 1;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if constexpr (EPI == EPI_DA) da_buf ^= 1;
      if constexpr (EPI == EPI_ROWSTATS) {
        if (sub + 1 == task_subtiles(P, t, BN)) {
          // task end: half 1 publishes its (m, l); half 0 merges both and writes the row's stats
          // (double-buffered exchange slot: the next task's write waits behind this barrier)
          float2* xch = reinterpret_cast<float2*>(smem + C::EPI_OFF) + xbuf * BM + quad * 32 + lane;
          if (half == 1) *xch = make_float2(m_run, l_run);
          asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
          if (half == 0 && row_ok) {
            const float2 o = *xch;
            const float M = fmaxf(m_run, o.x);  // accumulator units
            float S = 0.f;
            if (M != -INFINITY) S = l_run * ex2_approx((m_run - M) * sc_c) + o.y * ex2_approx((o.x - M) * sc_c);
            reinterpret_cast<float2*>(g.row_stats)[ti.bz * g.M + row_in] = make_float2(M * g.alpha, S);
          }
          xbuf ^= 1;
          m_run = -INFINITY;
          l_run = 0.f;
        }
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ===================== epilogue: warps 2..9; TMEM lane quadrant = warp % 4 (tcgen05.ld rule),
    // the two warps of a quadrant take alternating 128-byte column chunks
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    uint8_t* const stage_base = smem + C::EPI_OFF + (warp - 2) * C::BUFS * kStageBytesPerWarp;
    int ring = 0;
    // Stage one 32-row x 128-byte chunk and issue its TMA store; before refilling a buffer,
    // at most kStageBufs-1 earlier stores (those reading the other buffers) may be in flight.
    auto stage_and_store = [&](const CUtensorMap* map, const auto& vals, bool as_f32, int c0, int c1, int c2,
                               int c3) {
      uint8_t* buf = stage_base + ring * kStageBytesPerWarp;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::BUFS - 1) : "memory");
      __syncwarp();
      if (as_f32)
        stage_row<float, W>(buf, lane, vals);
      else
        stage_row<TC, W>(buf, lane, vals);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d(map, smem_u32(buf), c0, c1, c2, c3);
        bulk_commit();
      }
      ring = ring + 1 == C::BUFS ? 0 : ring + 1;
    };
    const size_t cs = sizeof(TC);
    auto a16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
    const bool vec = a16(g.C) && (g.ldc * cs) % 16 == 0 && (!g.bias || a16(g.bias)) &&
                     (!g.residual || (a16(g.residual) && g.ld_res % 4 == 0)) &&
                     (!g.aux || (a16(g.aux) && (g.ld_aux * cs) % 16 == 0)) && (g.sc0 * cs) % 16 == 0 &&
                     (g.sc1 * cs) % 16 == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t in_phase = 0;  // IN_AUX_SMEM: bit i = phase of this warp's input barrier i
    for (Walk wk(P, task0, task_step); wk.ok(P); wk.next(P, BN)) {
      int role;
      TileInfo ti = wk.info(P, BN, BM * CG, row_off, role);
      const int64_t p = ti.p, q = ti.q;
      TC* Cb = (TC*)g.C + p * g.sc0 + q * g.sc1;
      TC* auxb = g.aux ? (TC*)g.aux + p * g.sc0 + q * g.sc1 : nullptr;
      const int64_t row = ti.m0 + quad * 32 + lane;
      // the streamed input (residual / GELU' aux / beta*C) of a chunk, prefetched one chunk ahead
      auto in_ptr = [&](int c) -> const void* {
        const int64_t col0 = ti.n0 + c;
        if (P.in_kind == IN_AUX) return auxb + row * g.ld_aux + col0;
        if (P.in_kind == IN_RESIDUAL) return g.residual + row * g.ld_res + col0;
        return Cb + row * g.ldc + col0;
      };
      // (fp32 C only: a bf16 chunk already holds 64 live values, a prefetch buffer would spill)
      auto can_stream = [&](int c) {
        return sizeof(TC) == 4 && P.in_kind != IN_NONE && P.in_kind != IN_RES_SMEM && vec && row < g.M && c < BN &&
               ti.n0 + c + W <= g.N && role != SK_WRITER;
      };
      Raw8 raw;
      if (can_stream(half * W)) raw_load(raw, in_ptr(half * W));  // overlaps the wait for the MMAs
      // IN_*_SMEM: this warp's input chunk c of the tile -> staging buffer b (TMA, inbar[b])
      auto in_load = [&](int c, int b) {
        const uint32_t bar = smem_u32(&inbar[(warp - 2) * kStageBufs + b]);
        mbar_expect_tx(bar, kStageBytesPerWarp);
        tma_load_4d(smem_u32(stage_base + b * kStageBytesPerWarp), &tmAux, bar, (int)(ti.n0 + c),
                    (int)(ti.m0 + quad * 32), (int)q, (int)p);
      };
      const bool in_smem = (P.in_kind == IN_AUX_SMEM || P.in_kind == IN_RES_SMEM) && role != SK_WRITER;
      if (P.in_kind == IN_RES_SMEM && role != SK_WRITER) {
        // the first kStageBufs residual chunks of the tile, before the accumulator wait
        if (lane == 0) {
          bulk_wait_read0();  // earlier TMA stores have finished reading the buffers
          int i = 0;
          for (int c = half * W; c < BN && ti.n0 + c < g.N && i < kStageBufs; c += 2 * W, ++i) in_load(c, i);
        }
        __syncwarp();
        ring = 0;
      }
      if (P.in_kind == IN_AUX_SMEM && role != SK_WRITER) {
        // TMA-load this warp's aux chunks of the tile into its staging buffers (chunk i ->
        // buffer i) before the accumulator wait, so the loads overlap the MMAs
        if (lane == 0) {
          bulk_wait_read0();  // earlier TMA stores have finished reading the buffers
          int i = 0;
          for (int c = half * W; c < BN && ti.n0 + c < g.N; c += 2 * W, ++i) {
            const uint32_t bar = smem_u32(&inbar[(warp - 2) * kStageBufs + i]);
            mbar_expect_tx(bar, kStageBytesPerWarp);
            tma_load_4d(smem_u32(stage_base + i * kStageBytesPerWarp), &tmAux, bar, (int)(ti.n0 + c),
                        (int)(ti.m0 + quad * 32), (int)q, (int)p);
          }
        }
        __syncwarp();
        ring = 0;
      }
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const bool has_k = ti.kb_end > ti.kb_begin;
      const float dval =
          (g.act == NNT_ACT_SOFTMAX_BWD && row < g.M) ? __ldg(g.rowvec + ti.bz * g.M + row) : 0.f;
      // stream-K: this warp's partial slot region (writer), or the first / last unit whose partial
      // of this tile the finisher adds (units w_lo..w_hi, all below this one)
      const int rrow = quad * 32 + lane;  // row within this CTA's 128
      int64_t w_lo = 0, w_hi = -1;
      if (role == SK_FINISHER) {
        const int64_t t_start = (ti.tile - P.sk_dp_tiles) * P.nkb;  // the tile's first iteration
        w_hi = wk.it.c - 1;
        w_lo = w_hi;
        while (w_lo > 0 && (w_lo * P.sk_iters) / wk.it.G > t_start) --w_lo;  // unit w_lo starts at or before
        if (lane == 0) {
          for (int64_t w = w_lo; w <= w_hi; ++w) {
            uint32_t* f = sk_flag(P, w, rank, CG, warp - 2);
            while (ld_acquire_u32(f) == 0u) __nanosleep(64);
            *f = 0u;  // consumed: every launch leaves the flags zero (the workspace contract)
          }
        }
        __syncwarp();
      }
      int ci = 0;  // chunk index within the tile (IN_AUX_SMEM: its staging buffer)
#pragma unroll 1
      for (int c = half * W; c < BN; c += 2 * W, ++ci) {
        if (ti.n0 + c >= g.N) break;  // warp-uniform
        float v[W];
#pragma unroll
        for (int h = 0; h < W / 32; ++h) {
          if (has_k) {
            tmem_ld32(tmem_base + (uint32_t)(acc * BN + c + 32 * h) + ((uint32_t)(quad * 32) << 16), v + 32 * h);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[32 * h + j] = 0.f;
          }
        }
        const int cx = (int)(ti.n0 + c), cy = (int)(ti.m0 + quad * 32);
        if (role == SK_WRITER) {  // raw fp32 partial -> this unit's slot (alpha and extras at the finisher)
          float4* sl = reinterpret_cast<float4*>(sk_slot(P, wk.it.c, rank, CG, BN)) + (size_t)(c / 4) * BM + rrow;
#pragma unroll
          for (int j = 0; j < W / 4; ++j)
            __stcg(sl + (size_t)j * BM, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
          continue;
        }
        if (role == SK_FINISHER) {  // own partial + the lower units' partials, in descending unit order
#pragma unroll 1
          for (int64_t w = w_hi; w >= w_lo; --w) {
            const float4* sl =
                reinterpret_cast<const float4*>(sk_slot(P, w, rank, CG, BN)) + (size_t)(c / 4) * BM + rrow;
#pragma unroll
            for (int j = 0; j < W / 4; ++j) {
              const float4 t = __ldcg(sl + (size_t)j * BM);
              v[4 * j] += t.x;
              v[4 * j + 1] += t.y;
              v[4 * j + 2] += t.z;
              v[4 * j + 3] += t.w;
            }
          }
        }
        if (EPI == EPI_SPLITK || P.ws_mode) {
          // split-K partial (fp32) -> workspace slice ti.split; C is formed by the reduce
          epi_math<TC, W>(g, Cb, auxb, row, ti.n0 + c, false, vec, 0.f, IN_NONE, raw, v);
          stage_and_store(&tmAux, v, true, cx, cy, (int)ti.split, 0);
          continue;
        }
        int kind = can_stream(c) ? P.in_kind : IN_NONE;
        const int ib = ci % kStageBufs;  // IN_*_SMEM: the chunk's staging buffer (== ring)
        if (in_smem) {  // the input chunk landed in staging buffer ib
          mbar_wait(smem_u32(&inbar[(warp - 2) * kStageBufs + ib]), (in_phase >> ib) & 1u);
          in_phase ^= 1u << ib;
          unstage_row(raw, stage_base + ib * kStageBytesPerWarp, lane);
          kind = P.in_kind == IN_AUX_SMEM ? IN_AUX : IN_RESIDUAL;
        }
        epi_math<TC, W>(g, Cb, auxb, row, ti.n0 + c, true, vec, dval, kind, raw, v);
        if (can_stream(c + 2 * W)) raw_load(raw, in_ptr(c + 2 * W));  // next chunk's input, in flight meanwhile
        if (g.row_stats != nullptr && row < g.M) {
          // fused softmax subroutine 1: (max, sumexp) of this row over the chunk's
          // valid columns (W = 32 for fp32 C: one 32-column key tile)
          const int64_t col0 = ti.n0 + c;
          int64_t lim = g.N - col0;
          if (g.causal == NNT_CAUSAL_OUT_LOWER && row - col0 + 1 < lim) lim = row - col0 + 1;
          float m = -INFINITY, s = 0.f;
#pragma unroll
          for (int j = 0; j < W; ++j)
            if (j < lim) m = fmaxf(m, v[j]);
          if (m != -INFINITY) {
#pragma unroll
            for (int j = 0; j < W; ++j)
              if (j < lim) s += exp2f((v[j] - m) * 1.4426950408889634f);
          }
          *reinterpret_cast<float2*>(g.row_stats + 2 * ((ti.bz * g.M + row) * g.ld_stats + col0 / 32)) =
              make_float2(m, s);
        }
        auto stage_store = [&](const CUtensorMap* map) { stage_and_store(map, v, false, cx, cy, (int)q, (int)p); };
        if (g.act == NNT_ACT_GELU) {  // pre-activation -> aux, then gelu in place -> C
          if (P.tma_store)
            stage_store(&tmAux);
          else
            direct_store<TC, W>(g.M, g.N, g.ld_aux, auxb, row, ti.n0 + c, v);
          if constexpr (sizeof(TC) == 2) {
#pragma unroll
            for (int j = 0; j < W; j += 2) {
              const float2 x = gelu2(make_float2(v[j], v[j + 1]));
              v[j] = x.x;
              v[j + 1] = x.y;
            }
          } else {
#pragma unroll
            for (int j = 0; j < W; ++j) v[j] = gelu_e<false>(v[j]);
          }
        }
        if (P.tma_store)
          stage_store(&tmC);
        else
          direct_store<TC, W>(g.M, g.N, g.ldc, scatter_row_base(g, Cb, row), row, ti.n0 + c, v);
        if (in_smem && P.in_kind == IN_RES_SMEM) {
          // refill buffer ib with chunk ci + kStageBufs once this chunk's store has read it
          const int cn = c + 2 * W * kStageBufs;
          if (lane == 0 && cn < BN && ti.n0 + cn < g.N) {
            bulk_wait_read0();
            in_load(cn, ib);
          }
          __syncwarp();
        }
      }
      if constexpr (C::ROWSUM) {
        // R27: this row's sum of op(A) over the task's K range (one warp per lane quadrant)
        if (P.rowsum && ti.n0 == 0 && half == 0) {
          float rv = has_k ? tmem_ld1(tmem_base + (uint32_t)(2 * BN + acc * 16) + ((uint32_t)(quad * 32) << 16)) : 0.f;
          if (row < g.M) {
            rv *= g.alpha;
            if (P.ws_mode)  // split partial, after the C partials; the reduce adds them in split order
              ((float*)g.workspace)[P.splits * g.M * g.N + ti.split * g.M + row] = rv;
            else
              g.a_rowsum[row] = g.beta != 0.f ? fmaf(g.beta, g.a_rowsum[row], rv) : rv;
          }
        }
      }
      tc_fence_before();
      if (role == SK_WRITER) __threadfence();  // this lane's partial stores before the flag
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(map_to_rank(smem_u32(&tempty[acc]), 0));  // the leader's MMA waits on it
        else
          mbar_arrive(smem_u32(&tempty[acc]));
        if (role == SK_WRITER) st_release_u32(sk_flag(P, wk.it.c, rank, CG, warp - 2), 1u);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if constexpr (EPI == EPI_SPLITK) {
      if (P.fused_reduce) {
        // Ordered split-K reduction in the kernel (R25): this warp's region of the tile (its
        // lane quadrant's 32 rows x its column chunks) gets one arrival per split; the split that
        // arrives last adds the partials of all splits in ascending split order -- the same fixed
        // association whichever CTA that is -- applies beta*C / bias / residual and stores C.
        uint32_t* cnt = P.counters + ((uint32_t)ti.tile * CG + rank) * kEpiWarps + (uint32_t)(warp - 2);
        int last = 0;
        if (lane == 0) {
          bulk_wait0();  // this warp's partial stores (async proxy) have completed
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          last = atomicAdd(cnt, 1u) == (uint32_t)(P.splits - 1) ? 1 : 0;
          if (last) {
            *cnt = 0u;  // every launch leaves its counters zero (the workspace contract)
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
#pragma unroll 1
          for (int c = half * W; c < BN; c += 2 * W) {
            if (ti.n0 + c >= g.N) break;  // warp-uniform
            const int cx = (int)(ti.n0 + c), cy = (int)(ti.m0 + quad * 32);
            // partial s of this chunk -> staging buffer s & 1 (TMA, 32 rows x 128 B), one ahead
            auto ld_part = [&](int64_t sp) {
              const int b = (int)(sp & 1);
              const uint32_t bar = smem_u32(&inbar[(warp - 2) * kStageBufs + b]);
              mbar_expect_tx(bar, kStageBytesPerWarp);
              tma_load_4d(smem_u32(stage_base + b * kStageBytesPerWarp), &tmAux, bar, cx, cy, (int)sp, 0);
            };
            if (lane == 0) {
              bulk_wait_read0();  // earlier stores have read the staging buffers
              ld_part(0);
            }
            __syncwarp();
            float v[W];
            Raw8 raw;
#pragma unroll 1
            for (int64_t sp = 0; sp < P.splits; ++sp) {
              const int b = (int)(sp & 1);
              if (lane == 0 && sp + 1 < P.splits) ld_part(sp + 1);
              mbar_wait(smem_u32(&inbar[(warp - 2) * kStageBufs + b]), (in_phase >> b) & 1u);
              in_phase ^= 1u << b;
              unstage_row(raw, stage_base + b * kStageBytesPerWarp, lane);
              __syncwarp();  // every lane has read buffer b before it is refilled
              float t[8];
#pragma unroll
              for (int j = 0; j < W; j += 8) {
                unpack8<float>(raw, j, t);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[j + i] = sp == 0 ? t[i] : v[j + i] + t[i];
              }
            }
            epi_math<TC, W>(g, Cb, auxb, row, ti.n0 + c, true, vec, 0.f, IN_NONE, raw, v, false);
            ring = 0;
            stage_and_store(&tmC, v, false, cx, cy, (int)q, (int)p);
          }
        }
      }
      }
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync_all();  // neither CTA frees TMEM / exits while the pair's MMAs or arrivals are pending
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
  }
}

// C = beta*C + sum_s ws[s] (+bias) (+residual), splits added in ascending order (fp32 C).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int64_t splits, int64_t M,
                                                            int64_t N, float* C, int64_t ldc, float beta,
                                                            const float* __restrict__ bias,
                                                            const float* __restrict__ residual, int64_t ld_res,
                                                            float* __restrict__ rowsum) {
  NNT_PDL_ENTRY();
  const int64_t nq = N / 4;  // N % 4 == 0 (checked on the host)
  const int64_t total = M * nq;
  if (rowsum) {  // R27: a_rowsum = beta * a_rowsum + sum_s partial_s (slices after the C partials)
    const float* wsr = ws + splits * M * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
      float s = __ldcg(wsr + i);
      for (int64_t k = 1; k < splits; ++k) s += __ldcg(wsr + k * M + i);
      rowsum[i] = beta != 0.f ? fmaf(beta, rowsum[i], s) : s;
    }
  }
  if (ldc == N && (!residual || ld_res == N) && !bias) {
    // dense C (the dW GEMMs): flat float4 index, two independent elements per thread in flight
    const float4* w4 = reinterpret_cast<const float4*>(ws);
    float4* c4 = reinterpret_cast<float4*>(C);
    const float4* r4 = reinterpret_cast<const float4*>(residual);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += 2 * stride) {
      const int64_t j = i + stride;
      const bool two = j < total;
      float4 s0 = __ldcg(w4 + i), s1 = two ? __ldcg(w4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t k = 1; k < splits; ++k) {
        const float4 t0 = __ldcg(w4 + k * total + i);
        s0.x += t0.x; s0.y += t0.y; s0.z += t0.z; s0.w += t0.w;
        if (two) {
          const float4 t1 = __ldcg(w4 + k * total + j);
          s1.x += t1.x; s1.y += t1.y; s1.z += t1.z; s1.w += t1.w;
        }
      }
      if (beta != 0.f) {
        const float4 o0 = c4[i];
        s0.x += beta * o0.x; s0.y += beta * o0.y; s0.z += beta * o0.z; s0.w += beta * o0.w;
        if (two) {
          const float4 o1 = c4[j];
          s1.x += beta * o1.x; s1.y += beta * o1.y; s1.z += beta * o1.z; s1.w += beta * o1.w;
        }
      }
      if (residual) {
        const float4 o0 = r4[i];
        s0.x += o0.x; s0.y += o0.y; s0.z += o0.z; s0.w += o0.w;
        if (two) {
          const float4 o1 = r4[j];
          s1.x += o1.x; s1.y += o1.y; s1.z += o1.z; s1.w += o1.w;
        }
      }
      c4[i] = s0;
      if (two) c4[j] = s1;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nq, c = (i % nq) * 4;
    float4 s = __ldcg(reinterpret_cast<const float4*>(ws + r * N + c));
    for (int64_t k = 1; k < splits; ++k) {
      float4 t = __ldcg(reinterpret_cast<const float4*>(ws + (k * M + r) * N + c));
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    if (bias) {
      float4 b = *reinterpret_cast<const float4*>(bias + c);
      s.x += b.x; s.y += b.y; s.z += b.z; s.w += b.w;
    }
    float4* cp = reinterpret_cast<float4*>(C + r * ldc + c);
    if (beta != 0.f) {
      float4 o = *cp;
      s.x += beta * o.x; s.y += beta * o.y; s.z += beta * o.z; s.w += beta * o.w;
    }
    if (residual) {
      float4 o = *reinterpret_cast<const float4*>(residual + r * ld_res + c);
      s.x += o.x; s.y += o.y; s.z += o.z; s.w += o.w;
    }
    *cp = s;
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

nnt_status get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  NNT_REQUIRE(g_encode != nullptr, NNT_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  return NNT_OK;
}

// 4-D tensor map: dims {inner, outer, batch1, batch0}; es = element bytes.
nnt_status make_map(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t inner, int64_t outer,
                    int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_inner, int box_outer) {
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)b1, (cuuint64_t)b0};
  // size-1 batch dims get a harmless valid stride
  int64_t st1 = b1 > 1 ? s1 : ld * outer;
  int64_t st0 = b0 > 1 ? s0 : st1 * b1;
  cuuint64_t strides[3] = {(cuuint64_t)(ld * es), (cuuint64_t)(st1 * es), (cuuint64_t)(st0 * es)};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  NNT_REQUIRE(r == CUDA_SUCCESS, NNT_ERR_CUDA,
              "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld s1=%lld s0=%lld", (int)r,
              (long long)inner, (long long)outer, (long long)ld, (long long)s1, (long long)s0);
  return NNT_OK;
}

// One TMA request per MN-major operand stage (make_map_blocked; NNT_GEMM_BLOCKED=0: one per
// 64-element block, A/B runs)
bool blocked_off() {
  const char* e = getenv("NNT_GEMM_BLOCKED");
  return e && e[0] == '0';
}

// MN-major operand [K][MN] (row stride ld) as {64, K, MN / 64, b1, b0}: dim 2 steps 64 elements
// (128 B) along MN, so one box {64, box_k, nblk} stages nblk consecutive 64-element MN blocks of a
// SW128 operand, blocks 64 * box_k * es bytes apart in shared memory.  MN % 64 == 0 only (dim 0 is
// never clipped: a ragged MN edge could not be zero-filled).  Returns false if the driver rejects
// the map (the caller keeps the one-request-per-block 4-D map).
bool make_map_blocked(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t mn, int64_t k,
                      int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_k, int nblk) {
  if (mn % 64 != 0 || nblk < 1 || nblk > 256 || blocked_off()) return false;
  cuuint64_t dims[5] = {64, (cuuint64_t)k, (cuuint64_t)(mn / 64), (cuuint64_t)b1, (cuuint64_t)b0};
  int64_t st1 = b1 > 1 ? s1 : ld * k;
  int64_t st0 = b0 > 1 ? s0 : st1 * b1;
  cuuint64_t strides[4] = {(cuuint64_t)(ld * es), (cuuint64_t)(64 * es), (cuuint64_t)(st1 * es),
                           (cuuint64_t)(st0 * es)};
  cuuint32_t box[5] = {64, (cuuint32_t)box_k, (cuuint32_t)nblk, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(map, dt, 5, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

nnt_status make_tma_map_4d(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t inner,
                           int64_t outer, int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_inner,
                           int box_outer) {
  NNT_TRY(get_encoder());
  return make_map(map, dt, es, base, inner, outer, ld, b1, s1, b0, s0, box_inner, box_outer);
}

bool make_tma_map_blocked(CUtensorMap* map, CUtensorMapDataType dt, size_t es, const void* base, int64_t mn,
                          int64_t outer, int64_t ld, int64_t b1, int64_t s1, int64_t b0, int64_t s0, int box_outer,
                          int nblk) {
  if (get_encoder() != NNT_OK) return false;
  return make_map_blocked(map, dt, es, base, mn, outer, ld, b1, s1, b0, s0, box_outer, nblk);
}

// Split-K factor for a GEMM: fp32 C, no activation, unbatched, non-causal, an output grid
// that leaves SMs idle and a K long enough to cut (>= 8 K-blocks per split).
namespace {
int64_t long_k_splits(const GemmArgs& a);
}

int64_t gemm_tc_splits(const GemmArgs& a) {
  if (a.c_dtype != NNT_F32 || a.act != NNT_ACT_NONE || a.causal != NNT_CAUSAL_NONE || a.batch0 * a.batch1 != 1 ||
      a.N % 4 != 0)
    return 1;
  const int64_t tiles = cdiv(a.M, BM) * cdiv(a.N, 256);
  const int64_t nkb = cdiv(a.K, BK);
  const int64_t sms = num_sms();
  if (tiles * 2 > sms) return long_k_splits(a);
  int64_t s = sms / tiles;
  if (s > nkb / 8) s = nkb / 8;
  if (s > 8) s = 8;
  return s < 1 ? 1 : s;
}

namespace {

// C (and the GELU aux) can be written by TMA tensor stores
bool c_tma_ok(const GemmArgs& a, size_t es) {
  auto ok16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  return !a.scat_R && ok16(a.C) && (a.ldc * es) % 16 == 0 && (a.batch1 <= 1 || (a.sc1 > 0 && (a.sc1 * es) % 16 == 0)) &&
         (a.batch0 <= 1 || (a.sc0 > 0 && (a.sc0 * es) % 16 == 0)) &&
         (a.act != NNT_ACT_GELU || (ok16(a.aux) && (a.ld_aux * es) % 16 == 0));
}

// Persistent CTA-pair grid: as many clusters of 2 as can be co-resident at one CTA per SM
// (pairs are formed within a GPC, so fewer than num_sms/2 when GPCs hold odd SM counts).  A
// pair that is not resident would run its whole static task list after the others finish.
int64_t pair_units() {
  static int64_t units = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    using Cq = Cfg<256, 2>;
    auto kern = gemm_tc_kernel<256, float, EPI_GENERIC, 2>;
    int n = 0;
    if (set_max_dyn_smem(kern, (int)Cq::SMEM_BYTES) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3((unsigned)(num_sms() / 2 * 2));
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = Cq::SMEM_BYTES;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      q.attrs = attr;
      q.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) n = 0;
    }
    (void)cudaGetLastError();
    units = n > 0 ? n : num_sms() / 2;
    if (getenv("NNT_DEBUG_GEMM")) fprintf(stderr, "gemm_tc: %lld co-resident CTA pairs (query %d)\n", (long long)units, n);
  });
  return units;
}

}  // namespace

// Split-K workspace: partials [splits][M][N] and a_rowsum partials [splits][M] from the start;
// the arrival counters of the in-kernel reduce in a fixed zone of kSplitCounters words at the END
// of the workspace as the caller sizes it (16-byte aligned down), so GEMMs of different shapes
// sharing one workspace (the block's four dW GEMMs) all find their counters in the same zone,
// never under another shape's partials.  One counter per (tile, CTA of a pair, epilogue warp).
constexpr int64_t kSplitCounters = 4096;
size_t splitk_partial_bytes(const GemmArgs& a, int64_t splits) {
  const size_t b = (size_t)splits * ((size_t)a.M * (size_t)a.N + (size_t)a.M) * sizeof(float);
  return (b + 15) / 16 * 16;
}
size_t splitk_workspace_bytes(const GemmArgs& a, int64_t splits) {
  return splits > 1 ? splitk_partial_bytes(a, splits) + (size_t)kSplitCounters * sizeof(uint32_t) : 0;
}
uint32_t* splitk_counters(const GemmArgs& a) {
  const uintptr_t end = (reinterpret_cast<uintptr_t>(a.workspace) + a.workspace_bytes) & ~uintptr_t(15);
  return reinterpret_cast<uint32_t*>(end - (size_t)kSplitCounters * sizeof(uint32_t));
}
// The reduce runs in the GEMM when the workspace holds partials + counter zone, the tile grid's
// counters fit the zone (split GEMMs use 256-wide tiles), C is TMA-storable and no a_rowsum is
// requested (that keeps the separate ordered reduce kernel).
// Off by default: measured in the GPT-2 small step (4 interleaved runs) the separate
// reduce kernels, which run on the backward's side stream under the main-stream work, cost less
// than the in-kernel reduction's serial tail (gemm class 7.41 vs 7.72 ms/step).  NNT_SPLITK_FUSED=1
// turns it on.
bool fused_reduce_on() {  // read per call (tests switch it within one process)
  const char* e = getenv("NNT_SPLITK_FUSED");
  return e && e[0] == '1';
}
bool fused_reduce_ok(const GemmArgs& a, int64_t splits) {
  if (!fused_reduce_on()) return false;
  const int64_t regions = (cdiv(a.M, BM) + 1) * cdiv(a.N, 256) * kEpiWarps;
  return splits > 1 && !a.a_rowsum && a.workspace_bytes >= splitk_workspace_bytes(a, splits) &&
         regions <= kSplitCounters && c_tma_ok(a, sizeof(float)) && a.batch0 * a.batch1 == 1;
}

bool split_major_on() {  // NNT_GEMM_SPLITMAJOR=0: split-K tasks tile-major (A/B runs)
  const char* e = getenv("NNT_GEMM_SPLITMAJOR");
  return !(e && e[0] == '0');
}

// fp32 residual chunks staged by TMA (IN_RES_SMEM; NNT_GEMM_RES_SMEM=0: register prefetch, A/B runs)
bool res_smem_on() {
  const char* e = getenv("NNT_GEMM_RES_SMEM");
  return !(e && e[0] == '0');
}

// Narrow tail tiles (P.tail_n0; NNT_GEMM_TAIL=0: full-width MMAs on the last N column, A/B runs)
bool tail_on() {  // read per call
  const char* e = getenv("NNT_GEMM_TAIL");
  return !(e && e[0] == '0');
}

// Tile raster (NNT_GEMM_ORDER=0: always N-outer, the round-1 order; A/B runs)
bool m_outer_on() {  // read per call
  const char* e = getenv("NNT_GEMM_ORDER");
  return !(e && e[0] == '0');
}

// Stream-K (P.sk): off by default, NNT_GEMM_SK=1 enables it; NNT_GEMM_SK_EFF sets the wave
// efficiency (tiles / (waves x units)) below which a GEMM is scheduled stream-K (default 0.82).
// Measured on the GPT-2 XL step (4 interleaved runs): the GEMM class 77.0 -> 75.5 ms
// but the step 106.1 -> 106.9 ms (lower SM clock under the power cap, side-stream overlap).
bool sk_on() {  // read per call (tests switch it within one process)
  const char* e = getenv("NNT_GEMM_SK");
  return e && e[0] == '1';
}
double sk_eff() {
  const char* e = getenv("NNT_GEMM_SK_EFF");
  return e ? atof(e) : 0.82;
}
// Partial slots: one BM x 256 fp32 region per CTA of the widest grid, then the flag zone (the
// split-K counter zone at the workspace end: one flag per CTA and epilogue warp).
size_t sk_workspace_bytes() {
  return (size_t)num_sms() * BM * 256 * sizeof(float) + 16 + (size_t)kSplitCounters * sizeof(uint32_t);
}
// A GEMM the stream-K schedule can take: generic epilogue, unbatched, non-causal, no a_rowsum,
// and a workspace holding the slots and flags.
bool sk_possible(const GemmArgs& a) {
  const bool generic = a.act == NNT_ACT_NONE || a.act == NNT_ACT_GELU || a.act == NNT_ACT_GELU_BWD;
  return sk_on() && generic && !a.row_stats && !a.a_rowsum && a.batch0 * a.batch1 == 1 &&
         a.causal == NNT_CAUSAL_NONE && a.workspace && (reinterpret_cast<uintptr_t>(a.workspace) & 15u) == 0 &&
         a.workspace_bytes >= sk_workspace_bytes() && num_sms() * kEpiWarps <= kSplitCounters;
}
// Worth it (measured on the GPT-2 XL shapes, tools/gemm_bench.py): the last
// data-parallel wave is at most ~80 % full, K is long (>= 64 K-blocks: the fp32 partial written and
// read back is small against a tile's main loop) and at least two whole waves stay data-parallel.
// With fewer whole waves, or short K, the units' desynchronised K offsets cost more L2 operand
// traffic than the balanced last wave saves (XL QKV-dW 131 -> 143 us, QKV 93 -> 100 us, small
// FC+GELU 52 -> 65 us).  Every unit then also gets >= 1 tile of K-blocks (no empty unit range,
// whose finisher would wait for a flag nobody sets).
bool sk_pays(int64_t tiles, int64_t nkb, int64_t units) {
  const int64_t waves = (tiles + units - 1) / units;
  const double eff = (double)tiles / (double)(waves * units);
  return eff < sk_eff() && nkb >= 64 && tiles / units >= 2;
}

namespace {

template <int BN, typename TC, int EPI, int CG = 1>
nnt_status launch_bn(const GemmArgs& a, cudaStream_t s, int64_t splits, bool sk_allowed = false) {
  using C = Cfg<BN, CG, EPI>;
  const cudaError_t attr_err = set_max_dyn_smem(gemm_tc_kernel<BN, TC, EPI, CG>, (int)C::SMEM_BYTES);
  NNT_REQUIRE(attr_err == cudaSuccess, NNT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
  NNT_TRY(get_encoder());
  TcParams P;
  P.g = a;
  P.a_kmajor = a.ta == NNT_NOTRANS;
  P.b_kmajor = a.tb == NNT_TRANS;
  P.mt = cdiv(a.M, BM * CG);
  P.nt = cdiv(a.N, BN);
  if (EPI == EPI_ROWSTATS) {
    P.order = ORDER_ROWS;  // task = (batch item, row block) with all its key tiles
    P.tiles_per_batch = P.mt;
  } else if (a.causal == NNT_CAUSAL_OUT_LOWER && BN == BM && P.mt == P.nt) {
    P.order = ORDER_TRI;
    P.tiles_per_batch = P.mt * (P.mt + 1) / 2;
  } else {
    P.order = a.causal == NNT_CAUSAL_A_LOWER ? ORDER_HEAVY_HIGH_M
                                             : (a.causal == NNT_CAUSAL_A_UPPER ? ORDER_HEAVY_LOW_M : ORDER_N_OUTER);
    // non-causal: keep the LARGER operand's blocks shared by the concurrently running tiles
    if (P.order == ORDER_N_OUTER && m_outer_on() && a.M > a.N) P.order = ORDER_M_OUTER;
    P.tiles_per_batch = P.mt * P.nt;
  }
  P.num_tiles = P.tiles_per_batch * a.batch0 * a.batch1;
  const int64_t nkb = cdiv(a.K, BK);
  P.splits = splits;
  P.kb_per_split = cdiv(nkb, P.splits);
  P.num_tasks = P.num_tiles * P.splits;
  NNT_REQUIRE(!P.fused_reduce || P.num_tiles * CG * kEpiWarps <= kSplitCounters, NNT_ERR_UNSUPPORTED,
              "gemm(bf16): split-K counters");
  NNT_REQUIRE(P.num_tasks < (1ll << 31), NNT_ERR_UNSUPPORTED, "gemm(bf16): %lld tile tasks (> 2^31)",
              (long long)P.num_tasks);
  P.f_splits.init(P.splits);
  P.split_major = P.splits > 1 && split_major_on() ? 1 : 0;
  P.f_tiles.init(P.num_tiles);
  P.f_tpb.init(P.tiles_per_batch);
  P.f_mt.init(P.mt);
  P.f_nt.init(P.nt);
  P.f_nbat.init(a.batch0 * a.batch1);
  P.f_level.init(P.num_tiles / P.mt);
  P.f_b1.init(a.batch1);
  P.ws_mode = splits > 1 ? 1 : 0;
  P.fused_reduce = EPI == EPI_SPLITK ? 1 : 0;
  P.counters = P.fused_reduce ? splitk_counters(a) : nullptr;
  // stream-K when the data-parallel waves would leave a partly empty last wave
  const int64_t G_units = CG == 1 ? num_sms() * C::CTAS : pair_units();
  P.sk = 0;
  P.sk_dp_tiles = P.sk_iters = 0;
  P.nkb = nkb;
  P.sk_part = nullptr;
  if (sk_allowed && EPI == EPI_GENERIC && splits == 1 && (P.order == ORDER_N_OUTER || P.order == ORDER_M_OUTER) &&
      !a.a_rowsum &&
      sk_pays(P.num_tiles, nkb, G_units)) {
    const int64_t full_waves = P.num_tiles / G_units;
    P.sk = 1;
    P.sk_dp_tiles = full_waves >= 1 ? (full_waves - 1) * G_units : 0;
    P.sk_iters = (P.num_tiles - P.sk_dp_tiles) * nkb;
    P.sk_part = reinterpret_cast<float*>(a.workspace);
    P.counters = splitk_counters(a);
    if (getenv("NNT_DEBUG_GEMM"))
      fprintf(stderr, "gemm_tc stream-K %lldx%lldx%lld: BN %d CG %d tiles %lld units %lld dp %lld iters %lld\n",
              (long long)a.M, (long long)a.N, (long long)a.K, BN, CG, (long long)P.num_tiles, (long long)G_units,
              (long long)P.sk_dp_tiles, (long long)P.sk_iters);
  }
  // the one epilogue input streamed (prefetched) per chunk; element size must equal C's
  if (P.ws_mode || !generic_epi(EPI))
    P.in_kind = IN_NONE;
  else if (a.act == NNT_ACT_GELU_BWD)
    P.in_kind = sizeof(TC) == 2 && c_tma_ok(a, sizeof(TC)) && aligned16(a.aux) &&
                        (a.ld_aux * (int64_t)sizeof(TC)) % 16 == 0
                    ? IN_AUX_SMEM  // bf16: the register prefetch would spill; stage it through smem
                    : IN_AUX;
  else if (a.residual && sizeof(TC) == 4)
    P.in_kind = res_smem_on() && c_tma_ok(a, sizeof(TC)) && aligned16(a.residual) && a.ld_res % 4 == 0 &&
                        a.batch0 * a.batch1 == 1
                    ? IN_RES_SMEM  // TMA-staged residual chunks (NNT_GEMM_RES_SMEM=0: register prefetch)
                    : IN_RESIDUAL;
  else if (a.beta != 0.f)
    P.in_kind = IN_COLD;
  else
    P.in_kind = IN_NONE;
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((P.a_kmajor ? 0u : 1u) << 15) | ((P.b_kmajor ? 0u : 1u) << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
  P.idesc_ones = (1u << 4) | (1u << 7) | (1u << 10) | ((P.a_kmajor ? 0u : 1u) << 15) | ((uint32_t)(16 >> 3) << 17) |
                 ((uint32_t)((BM * CG) >> 4) << 24);
  P.tail_n0 = -1;
  P.tail_n = BN;
  P.tail_last = 0;
  P.idesc_tail = P.idesc;
  if (generic_epi(EPI) && tail_on() && a.N % BN != 0) {
    // K-major B: the remainder rounded up to 32 (a CTA pair stages tn / 2 rows per CTA, a multiple
    // of 16); MN-major B: to 64 per CTA, so the pair's second half starts on a 64-element (128-byte)
    // block of the TMA box (measured: 32-element offsets split every box row over two lines)
    const int gran = P.b_kmajor ? 32 : 64 * CG;
    const int tn = (int)(((a.N % BN) + gran - 1) / gran * gran);
    if (tn < BN) {
      P.tail_n0 = (P.nt - 1) * BN;
      P.tail_n = tn;
      P.idesc_tail = (P.idesc & ~(0x3Fu << 17)) | ((uint32_t)(tn >> 3) << 17);
      // tail tiles last only with a K-major A: the dW GEMMs' (MN-major A) tail tiles re-read their
      // A blocks from DRAM when they run apart from their row block (measured slower)
      P.tail_last = (P.order == ORDER_M_OUTER && !P.sk && P.nt > 1 && P.a_kmajor) ? 1 : 0;
    }
  }
  P.f_ntf.init(P.nt > 1 ? P.nt - 1 : 1);
  P.rowsum = a.a_rowsum != nullptr ? 1 : 0;
  NNT_REQUIRE(!P.rowsum || C::ROWSUM, NNT_ERR_UNSUPPORTED, "gemm(bf16): a_rowsum needs a tile width <= 192");
  CUtensorMap tmA, tmB, tmC, tmAux;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  P.a_blk = P.b_blk = 0;
  if (P.a_kmajor)
    NNT_TRY(make_map(&tmA, bf, 2, a.A, a.K, a.M, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, BK, BM));
  else if (make_map_blocked(&tmA, bf, 2, a.A, a.M, a.K, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, BK, BM / 64))
    P.a_blk = 1;
  else
    NNT_TRY(make_map(&tmA, bf, 2, a.A, a.M, a.K, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, 64, BK));
  // (MN-major B blocked only when every CTA's first B row is 64-aligned: pair halves and the
  // narrow tail's halves are multiples of 64 then)
  if (P.b_kmajor)
    NNT_TRY(make_map(&tmB, bf, 2, a.B, a.K, a.N, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, BK, BN / CG));
  else if ((BN / CG) % 64 == 0 && (P.tail_n0 < 0 || (P.tail_n / CG) % 64 == 0) &&
           make_map_blocked(&tmB, bf, 2, a.B, a.N, a.K, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, BK, C::B_BLKS))
    P.b_blk = 1;
  else
    NNT_TRY(make_map(&tmB, bf, 2, a.B, a.N, a.K, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, 64, BK));
  const size_t es = sizeof(TC);
  const CUtensorMapDataType cdt = sizeof(TC) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : bf;
  const int W = (int)(128 / es);
  auto ok16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  memset(&tmC, 0, sizeof(tmC));
  memset(&tmAux, 0, sizeof(tmAux));
  if (P.ws_mode) {
    // workspace [splits][M][N] fp32; the aux map slot carries it
    P.tma_store = 1;
    NNT_TRY(make_map(&tmAux, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.workspace, a.N, a.M, a.N, splits, a.M * a.N, 1, 0,
                     32, 32));
    if (P.fused_reduce)  // C (fp32) stored by the last split of each region
      NNT_TRY(make_map(&tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.C, a.N, a.M, a.ldc, 1, 0, 1, 0, 32, 32));
  } else if (EPI == EPI_ROWSTATS) {
    P.tma_store = 0;  // no C
  } else {
    const bool tma_ok = c_tma_ok(a, es);
    NNT_REQUIRE(generic_epi(EPI) || tma_ok, NNT_ERR_ALIGN, "gemm(bf16): specialised epilogue needs TMA-able C");
    (void)ok16;
    P.tma_store = tma_ok ? 1 : 0;  // (direct 16-byte stores measured 1.5x slower than TMA stores)
    if (tma_ok) {
      NNT_TRY(make_map(&tmC, cdt, es, a.C, a.N, a.M, a.ldc, a.batch1, a.sc1, a.batch0, a.sc0, W, 32));
      if (a.act == NNT_ACT_GELU || P.in_kind == IN_AUX_SMEM || EPI == EPI_DA)  // GELU out / GELU', P in
        NNT_TRY(make_map(&tmAux, cdt, es, a.aux, a.N, a.M, a.ld_aux, a.batch1, a.sc1, a.batch0, a.sc0, W, 32));
      if (P.in_kind == IN_RES_SMEM)  // the fp32 residual, staged chunk by chunk
        NNT_TRY(make_map(&tmAux, cdt, es, a.residual, a.N, a.M, a.ld_res, 1, 0, 1, 0, W, 32));
    }
  }
  if constexpr (CG == 1) {
    const int64_t units = num_sms() * C::CTAS;  // persistent: C::CTAS CTAs per SM
    int64_t grid = P.sk ? units : (P.num_tasks < units ? P.num_tasks : units);
    if (grid < 1) grid = 1;
    ::nnt::launch(gemm_tc_kernel<BN, TC, EPI, 1>, (unsigned)grid, kThreads, C::SMEM_BYTES, s, P, tmA, tmB, tmC, tmAux);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const int64_t max_clusters = pair_units();
    int64_t grid = P.sk ? max_clusters : (P.num_tasks < max_clusters ? P.num_tasks : max_clusters);
    if (grid < 1) grid = 1;
    cfg.gridDim = dim3((unsigned)(grid * CG));
    NNT_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, TC, EPI, CG>, P, tmA, tmB, tmC, tmAux));
  }
  NNT_TRY(check_launch("gemm_tc"));
  if (getenv("NNT_DEBUG_GEMM"))
    fprintf(stderr, "gemm_tc launch %lldx%lldx%lld batch %lld: BN %d CG %d EPI %d splits %lld sk %d tiles %lld tail %d%s\n",
            (long long)a.M, (long long)a.N, (long long)a.K, (long long)(a.batch0 * a.batch1), BN, CG, EPI,
            (long long)splits, P.sk, (long long)P.num_tiles, P.tail_n0 >= 0 ? P.tail_n : 0, P.tail_last ? " last" : "");
  if (P.ws_mode && !P.fused_reduce) {
    const int64_t total = a.M * (a.N / 4);
    int64_t blocks = cdiv(total, 256);
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    ::nnt::launch(splitk_reduce_kernel, (unsigned)blocks, 256, 0, s, (const float*)a.workspace, splits, a.M, a.N, (float*)a.C,
                                                          a.ldc, a.beta, a.bias, a.residual, a.ld_res,
                                                          P.rowsum ? a.a_rowsum : nullptr);
    NNT_TRY(check_launch("gemm_tc splitk reduce"));
  }
  return NNT_OK;
}

// Tile shape from a two-term roofline per round of the persistent schedule.  Per SM, a tile
// costs max(MMA cycles, L2 cycles): the tensor core retires 8192 bf16 FLOP per cycle
// (128 x BN x K tile = BN*K/32 cycles), and the SM's operand + epilogue traffic,
//   (128 + BN/CG) * K * 2 bytes (a CTA pair stages half of B per SM) + 128 * BN * epilogue bytes,
// shares the L2 slice throughput (~5200 B per SM cycle chip-wide at 1965 MHz, calibrated on the
// K = 768 / 3072 projection GEMMs; B300_MICROARCH: LTS cap ~6300 B/cyc at locked clocks) with
// every SM busy in that round; the epilogue term below bounds a round from the other side.
// Small-K projection GEMMs are L2-bound with 128-row tiles, which is why the 256-row CTA-pair
// tiles (half the operand bytes per FLOP) usually win.
double l2_bytes_per_cycle() {
  static const double v = [] {
    const char* e = getenv("NNT_GEMM_L2");
    return e ? atof(e) : 5200.0;
  }();
  return v;
}

double tile_cost(const GemmArgs& a, int bn, int cg, int64_t units, size_t es_c, bool sk = false) {
  const int64_t nb = a.batch0 * a.batch1;
  const int64_t tiles = cdiv(a.M, (int64_t)BM * cg) * cdiv(a.N, bn) * nb;
  const double kp = (double)(cdiv(a.K, BK) * BK);
  const double mma = bn * kp / 32.0;
  double epi = (double)es_c;                                    // C
  if (a.act == NNT_ACT_GELU || a.act == NNT_ACT_GELU_BWD) epi += (double)es_c;  // aux out / in
  if (a.residual) epi += 4.0;
  if (a.beta != 0.f) epi += (double)es_c;
  const double bytes_sm = (BM + (double)bn / cg) * kp * 2.0 + (double)BM * bn * epi;
  const double l2 = l2_bytes_per_cycle();
  // the epilogue drains ~12 B of output + input per SM cycle (measured: TMEM -> registers ->
  // SW128 staging -> TMA store); it overlaps the next tile's MMAs, the last tile's is exposed
  const double t_epi = (double)BM * bn * epi / 12.0;
  const int64_t full = tiles / units, rem = tiles % units;
  if (sk && rem && sk_pays(tiles, (int64_t)(kp / BK), units)) {
    // stream-K: fractional waves, plus a partial tile written and read back (fp32) per unit
    const double wave = fmax(fmax(mma, (double)units * cg * bytes_sm / l2), t_epi);
    return (double)tiles / (double)units * wave + t_epi + 2.0 * BM * bn * 4.0 / 12.0;
  }
  double cost = (double)full * fmax(fmax(mma, (double)units * cg * bytes_sm / l2), t_epi);
  if (rem) cost += fmax(fmax(mma, (double)rem * cg * bytes_sm / l2), t_epi);
  return cost + t_epi;
}

int choose_bn(const GemmArgs& a, size_t es_c, double* cost_out = nullptr, bool sk = false) {
  if (cost_out) *cost_out = 1e300;
  if (a.N <= 64) return 64;
  if (a.causal == NNT_CAUSAL_OUT_LOWER) return 128;
  const int cands[3] = {256, 192, 128};
  int best = 256;
  double best_cost = 1e300;
  for (int bn : cands) {
    const double cost = tile_cost(a, bn, 1, num_sms(), es_c, sk);
    if (cost < best_cost * 0.97) {  // near-ties (within the model's error) go to the wider tile
      best_cost = cost;
      best = bn;
    }
  }
  if (cost_out) *cost_out = best_cost;
  return best;
}

// CTA pairs (cta_group::2, 256-row tiles) for the plain projection-type GEMMs: unbatched,
// non-causal, generic epilogue.  NNT_GEMM_CG=1 in the environment forces single-CTA tiles,
// NNT_GEMM_CG=2 forces pairs wherever they are legal.
int forced_cg() {
  static const int forced = [] {
    const char* e = getenv("NNT_GEMM_CG");
    return e ? atoi(e) : 0;
  }();
  return forced;
}
// The out-projection-type GEMM (fp32 residual, K < 2048) with the TMA-staged residual and a narrow
// last N column (N % 256 in (0, 128]: GPT-2 XL's N = 1600) runs fastest on 256-wide CTA pairs:
// 47.5 us vs 52.6 (single-CTA 192) and 62 (the tile model's 128-wide pairs, which do not see the
// narrow tail); with N a multiple of 256 (small N = 768) single-CTA tiles stay ahead (measured).
bool out_proj_pair256(const GemmArgs& a) {
  const char* e = getenv("NNT_GEMM_OUT_PAIR");  // NNT_GEMM_OUT_PAIR=0: the tile model's choice (A/B runs)
  if (e && e[0] == '0') return false;
  return forced_cg() != 1 && a.residual && a.K < 2048 && a.c_dtype == NNT_F32 && res_smem_on() && tail_on() &&
         a.N % 256 != 0 && a.N % 256 <= 128 && a.act == NNT_ACT_NONE && a.batch0 * a.batch1 == 1 &&
         a.causal == NNT_CAUSAL_NONE && a.M >= 2 * BM && !a.a_rowsum && c_tma_ok(a, sizeof(float)) &&
         aligned16(a.residual) && a.ld_res % 4 == 0 && num_sms() >= 2;
}
bool use_pair(const GemmArgs& a) {
  if (forced_cg() == 1) return false;
  // measured exception to the model: a streamed fp32 residual with a short K (the attention
  // out-projection, K = E) runs 15% faster on single-CTA 192-wide tiles than on any pair tile
  if (forced_cg() != 2 && a.residual && a.K < 2048) return false;
  return a.batch0 * a.batch1 == 1 && a.causal == NNT_CAUSAL_NONE && a.M >= 2 * BM && a.N > 64 &&
         num_sms() >= 2;
}

// Pair widths whose half is a whole 64-column MN-major block.
int choose_bn_pair(const GemmArgs& a, size_t es_c, double* cost_out, bool sk = false) {
  // (192-wide pair tiles -- N = 1600 as 9 x 192 instead of 7 x 256 with a nearly empty last round
  // -- ran 2-4 % slower on every GPT-2 XL shape: these GEMMs are bound by the L2 -> SM operand
  // stream, which narrower tiles increase per FLOP; DESIGN §7.1.  NNT_GEMM_192=1 re-enables them.)
  const int cands[3] = {256, 128, getenv("NNT_GEMM_192") ? 192 : 128};
  if (const char* f = getenv("NNT_GEMM_BN")) {  // A/B override of the tile model
    *cost_out = 0;
    return atoi(f);
  }
  // Measured exception: a K-major B whose 256-wide pair tiles fill their rounds badly (< 70 %: GPT-2
  // small's N = 768 projection, 96 tiles on 74 pairs) takes 192-wide pairs (128 tiles: 86 %): small
  // proj 54 -> 47 us.  Not for MN-major B (a 96-row half over-fetches a 64-column block) nor for the
  // milder XL case (N = 1600: 76 %, measured slower).  NNT_GEMM_192_EXC=0 disables it.
  if (a.tb == NNT_TRANS && a.batch0 * a.batch1 == 1 && a.N % 192 == 0 && !getenv("NNT_GEMM_192")) {
    const char* e = getenv("NNT_GEMM_192_EXC");
    const int64_t units = pair_units(), t256 = cdiv(a.M, 2 * BM) * cdiv(a.N, 256), t192 = cdiv(a.M, 2 * BM) * (a.N / 192);
    const double eff256 = (double)t256 / (double)(cdiv(t256, units) * units);
    const double eff192 = (double)t192 / (double)(cdiv(t192, units) * units);
    if (!(e && e[0] == '0') && eff256 < 0.7 && eff192 > 0.8) {
      *cost_out = tile_cost(a, 192, 2, units, es_c, sk);
      return 192;
    }
  }
  int best = 256;
  double best_cost = 1e300;
  for (int bn : cands) {
    const double cost = tile_cost(a, bn, 2, pair_units(), es_c, sk);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = bn;
    }
  }
  *cost_out = best_cost;
  return best;
}

// Very long K with a grid of CTA-pair tiles that fills its last round badly (the LM head's
// dh = dlogits wte: 96 tiles of K = 50257 on 74 pairs): splitting K evens the rounds.  Chosen by
// the tile model plus the ordered reduce's traffic (~3300 B per SM cycle of HBM).
int64_t long_k_splits(const GemmArgs& a) {
  if (a.K < 16384 || !use_pair(a)) return 1;
  const int64_t units = pair_units();
  int64_t best = 1;
  double best_cost = tile_cost(a, 256, 2, units, 4);
  for (int64_t sp = 2; sp <= 4; ++sp) {
    GemmArgs b = a;
    b.K = cdiv(a.K, sp);
    b.batch0 = sp;  // sp independent K ranges of the same tile grid
    b.batch1 = 1;
    const double reduce = (double)a.M * a.N * 4.0 * (sp + 1) / 3300.0;
    const double cost = tile_cost(b, 256, 2, units, 4) + reduce;
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

template <typename TC>
nnt_status launch_tc(const GemmArgs& a, cudaStream_t s, int64_t splits, bool sk = false) {
  const bool tma_ok = splits == 1 && c_tma_ok(a, sizeof(TC));
  if constexpr (sizeof(TC) == 2) {
    if (tma_ok && a.act == NNT_ACT_SOFTMAX_BWD && aligned16(a.aux) && (a.ld_aux * 2) % 16 == 0)
      return launch_bn<128, TC, EPI_DA>(a, s, 1);  // P staged by TMA a task ahead
    if (a.act == NNT_ACT_SOFTMAX) return launch_bn<128, TC, EPI_SOFTMAX>(a, s, 1);
  } else {
    if (tma_ok && a.act == NNT_ACT_NONE && !a.bias && !a.residual && a.beta == 0.f &&
        (a.row_stats || a.causal == NNT_CAUSAL_OUT_LOWER))
      return launch_bn<128, TC, EPI_SCORES>(a, s, 1);
  }
  if (a.a_rowsum) {  // R27: tiles <= 192 wide leave TMEM columns for the row-sum accumulators
    if (use_pair(a)) return launch_bn<128, TC, EPI_GENERIC_RS, 2>(a, s, splits);
    switch (choose_bn(a, sizeof(TC))) {
      case 64: return launch_bn<64, TC, EPI_GENERIC_RS>(a, s, splits);
      case 128: return launch_bn<128, TC, EPI_GENERIC_RS>(a, s, splits);
      default: return launch_bn<192, TC, EPI_GENERIC_RS>(a, s, splits);
    }
  }
  if (splits == 1 && !sk && !getenv("NNT_GEMM_BN") && out_proj_pair256(a))
    return launch_bn<256, TC, EPI_GENERIC, 2>(a, s, 1, false);
  if (use_pair(a)) {
    double cost_pair = 0, cost_single = 0;
    const int bnp = choose_bn_pair(a, sizeof(TC), &cost_pair, sk);
    const int bns = choose_bn(a, sizeof(TC), &cost_single, sk);
    if (getenv("NNT_DEBUG_GEMM"))
      fprintf(stderr, "gemm_tc %lldx%lldx%lld: pair BN %d cost %.0f, single BN %d cost %.0f\n", (long long)a.M,
              (long long)a.N, (long long)a.K, bnp, cost_pair, bns, cost_single);
    if constexpr (sizeof(TC) == 4) {
      if (splits > 1 && fused_reduce_ok(a, splits)) return launch_bn<256, TC, EPI_SPLITK, 2>(a, s, splits);
    }
    if (splits > 1 || forced_cg() == 2 || cost_pair <= cost_single) {  // ties go to pairs
      if (bnp == 256 || splits > 1) return launch_bn<256, TC, EPI_GENERIC, 2>(a, s, splits, sk);
      if (bnp == 192) return launch_bn<192, TC, EPI_GENERIC, 2>(a, s, splits, sk);
      return launch_bn<128, TC, EPI_GENERIC, 2>(a, s, splits, sk);
    }
  }
  if constexpr (sizeof(TC) == 4) {
    if (splits > 1 && fused_reduce_ok(a, splits)) return launch_bn<256, TC, EPI_SPLITK, 1>(a, s, splits);
  }
  switch (splits > 1 ? 256 : choose_bn(a, sizeof(TC), nullptr, sk)) {
    case 64: return launch_bn<64, TC, EPI_GENERIC>(a, s, splits, sk);
    case 128: return launch_bn<128, TC, EPI_GENERIC>(a, s, splits, sk);
    case 192: return launch_bn<192, TC, EPI_GENERIC>(a, s, splits, sk);
    default: return launch_bn<256, TC, EPI_GENERIC>(a, s, splits, sk);
  }
}

}  // namespace

nnt_status gemm_tc_launch(const GemmArgs& a, cudaStream_t s, int* kernels) {
  // TMA: 16-byte aligned base, 16-byte multiple strides (bf16: multiples of 8 elements).
  NNT_REQUIRE(aligned16(a.A) && aligned16(a.B), NNT_ERR_ALIGN, "gemm(bf16): A/B must be 16-byte aligned");
  NNT_REQUIRE(a.lda % 8 == 0 && a.ldb % 8 == 0, NNT_ERR_ALIGN, "gemm(bf16): lda/ldb must be multiples of 8");
  NNT_REQUIRE((a.batch1 <= 1 || (a.sa1 % 8 == 0 && a.sb1 % 8 == 0 && a.sa1 > 0 && a.sb1 > 0)) &&
                  (a.batch0 <= 1 || (a.sa0 % 8 == 0 && a.sb0 % 8 == 0 && a.sa0 > 0 && a.sb0 > 0)),
              NNT_ERR_ALIGN, "gemm(bf16): batch strides must be positive multiples of 8");
  NNT_REQUIRE(a.M < (1ll << 31) && a.N < (1ll << 31) && a.K < (1ll << 31), NNT_ERR_UNSUPPORTED,
              "gemm(bf16): dims must fit int32 TMA coordinates");
  int64_t splits = gemm_tc_splits(a);  // the workspace is sized for this split count
  if (a.a_rowsum && splits > 1) {
    // row-sum GEMMs run 128-wide tiles (pairs when M >= 256): refit the split to that grid
    const bool pair = use_pair(a);
    const int64_t units = pair ? pair_units() : num_sms();
    const int64_t tiles = cdiv(a.M, BM * (pair ? 2 : 1)) * cdiv(a.N, 128);
    int64_t s2 = units / tiles;
    splits = s2 < 1 ? 1 : (s2 < splits ? s2 : splits);
  }
  const bool ws_ok = a.workspace && (reinterpret_cast<uintptr_t>(a.workspace) & 15u) == 0 &&
                     a.workspace_bytes >= (size_t)splits * (a.M * a.N + (a.a_rowsum ? a.M : 0)) * sizeof(float) &&
                     (reinterpret_cast<uintptr_t>(a.C) & 15u) == 0 && a.ldc % 4 == 0 &&
                     (!a.residual || ((reinterpret_cast<uintptr_t>(a.residual) & 15u) == 0 && a.ld_res % 4 == 0)) &&
                     (!a.bias || (reinterpret_cast<uintptr_t>(a.bias) & 15u) == 0);
  if (!ws_ok) splits = 1;
  // stream-K (a workspace big enough for its slots) replaces split-K: no partial round trip
  // through HBM for the whole tile grid and no reduce launch
  const bool sk = sk_possible(a) && !a.scat_R;
  if (sk || a.scat_R) splits = 1;
  if (kernels) *kernels = splits > 1 && !fused_reduce_ok(a, splits) ? 2 : 1;
  if (a.act == NNT_ACT_ROWSTATS) return launch_bn<128, float, EPI_ROWSTATS>(a, s, 1);
  if (a.c_dtype == NNT_F32) return launch_tc<float>(a, s, splits, sk);
  return launch_tc<__nv_bfloat16>(a, s, splits, sk);
}

}  // namespace nnt
