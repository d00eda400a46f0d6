// Fused attention tile kernels of the bf16 path (readings R20, R26, R33).
//
// The paper's attention is B = V SoftMax(K^T Q / sqrt(h)) per (batch, head) with the
// softmax built from the maxsumexp subroutine and a normalise subroutine.  The bf16
// path runs subroutine 1 (the row statistics) in the score GEMM's epilogue (R26); these two
// kernels then run every remaining attention product tile by tile, each key / query tile pair
// touched once:
//
//   nnt_attention_fwd_pv  (subroutine 2 + the value product) -- task = (b, h, query block):
//       for each key block kb <= qb:  S = Q K_kb^T (tcgen05, TMEM)  ->  P = e^{S - M} / S_sum
//       (epilogue, from the row statistics)  ->  P stored to HBM (the backward reads it) AND
//       staged in shared memory as the A operand of  O += P V_kb  (tcgen05, TMEM);  O stored once.
//       P is read back from HBM zero times (the unfused path re-read it for P V).
//   nnt_attention_bwd_kv  (softmax backward + dV + dK) -- task = (b, h, key block):
//       for each query block qb >= kb:  dP = dO_qb V_kb^T (tcgen05) and dV += P^T dO_qb straight
//       from the TMA-loaded P tile  ->  dA = P (dP - D) / sqrt(h) (epilogue, written over the P
//       tile in shared memory)  ->  dA stored (for dQ = dA K) and used in place as the A operand
//       of  dK += dA^T Q_qb.  dK, dV accumulate in TMEM over the query blocks and are stored
//       once.  Each P tile is read once, each dA tile written once (the unfused path read P three
//       times and dA twice).
//
// Warp roles as in the GEMM (gemm_tc.cu): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2..17 epilogue (TMEM lane quadrant = warp % 4; the four warps of a quadrant take
// the four 32-column groups of a 128 x 128 tile: the epilogues are latency- and MUFU-bound, so
// they get more warps than the GEMM's).  Persistent CTAs, static heaviest-first task
// order with a boustrophedon assignment.  Head size h = 64 and S % 128 == 0 (the configurations
// of BASELINE.json); the block falls back to the unfused GEMM sequence otherwise.
#include <cuda.h>

#include <cstdlib>

#include "gemm_common.cuh"
#include "tc_ptx.cuh"

namespace nnt {
namespace {

constexpr int kEW = 16;                      // epilogue warps: 4 per TMEM lane quadrant
constexpr int kAThreads = 64 + 32 * kEW;
constexpr int TB = 128;     // query / key block
constexpr int HD = 64;      // head size
constexpr int TILE16 = 16384;  // one 128-row x 128-byte SW128 tile (64 bf16 per row)
constexpr int PIECE = 4096;    // one epilogue warp's 32-row x 128-byte staging piece

struct AttnParams {
  int B, H, S, nblk, num_tasks, causal;
  float scale;          // 1 / sqrt(h)
  const float* stats;   // fwd: (M, S_sum) per (b, h, query) as float2, M in scaled-score units
  const float* D;       // bwd: D = rowdot(dO, O) per (b, h, query)
  unsigned long long* trace;  // nnt_attention_trace: CTA 0's per-iteration event times, or NULL
  int l2hints;                // L2 policies on the TMA traffic: 0 none, 1 evict_last on the re-read tiles and
                              // evict_first on the P / dA streams, 2 (default) evict_first on the streams only
  int p_blk;                  // backward: the P map is blocked (make_tma_map_blocked): a 128 x 128 P tile's two
                              // 64-key halves in one TMA request
  int bgroup;                 // backward: key-block levels interleaved per (b, h) in groups of bgroup (1: level-major)
};

// Pipeline trace (nnt_attention_trace, tools): CTA 0 records %globaltimer at kTraceEv events of
// each of its first kTraceIt iterations.
constexpr int kTraceIt = 256, kTraceEv = 6;
__device__ unsigned long long g_attn_trace[2][kTraceEv][kTraceIt];
__device__ __forceinline__ void trace_ev(const AttnParams& P, int ev, int64_t g) {
  if (P.trace && blockIdx.x == 0 && g < kTraceIt) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[ev * kTraceIt + g] = t;
  }
}

// idesc: fp32 accumulate, bf16 A / B, the operands' majors, N, M = 128
__host__ __device__ constexpr uint32_t idesc_of(bool a_mn, bool b_mn, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TB >> 4) << 24);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier (one elected lane)
__device__ __forceinline__ void bulk_load_w(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("{\n\t.reg .pred e;\n\t" NNT_ELECT
               "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// 32 values (bf16) -> one half (16-byte chunks 4 sub .. 4 sub + 3) of this lane's 128-byte row of
// an SW128 staging piece; the other half is written by the partner warp
__device__ __forceinline__ void stage_half_row(uint8_t* piece, int lane, int sub, const float (&v)[32]) {
  uint8_t* rowp = piece + lane * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 u;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
    __nv_bfloat162 t1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
    __nv_bfloat162 t3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
    u.x = *reinterpret_cast<uint32_t*>(&t0);
    u.y = *reinterpret_cast<uint32_t*>(&t1);
    u.z = *reinterpret_cast<uint32_t*>(&t2);
    u.w = *reinterpret_cast<uint32_t*>(&t3);
    *reinterpret_cast<uint4*>(rowp + (((sub * 4 + j) ^ (lane & 7)) << 4)) = u;
  }
}
// the two warps of a (quadrant, 64-column chunk) pair: named barrier 1 + pair (64 threads)
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
}

__device__ __forceinline__ int64_t task_at(int64_t c, int64_t G, int64_t k) {
  return k * G + ((k & 1) ? (G - 1 - c) : c);
}

__device__ __forceinline__ void tmem_alloc512(uint32_t slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(slot) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free512(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

// ============================================================================ forward
// smem: Q[2] (task parity) | K ring[3] | V ring[3] | P staging[2] (32 KB: half h at +16 KB,
// quadrant rows at +4 KB) | O staging[2] (16 KB each) | barriers.  TMEM: S[3] at columns 0 / 128 /
// 256, O[2] at 384 / 448.
constexpr int F_STAGES = 3;  // K ring and V ring, 3 tiles each
constexpr int F_Q = 0, F_K = 2 * TILE16, F_V = F_K + F_STAGES * TILE16, F_P = F_V + F_STAGES * TILE16;
constexpr int F_O = F_P + 2 * 2 * TILE16;
constexpr int kAThreadsF = kAThreads + 32;  // + the V producer warp (warp 18)
constexpr int F_BAR = F_O + 2 * TILE16;
constexpr int F_SMEM = F_BAR + 256 + 1024;

__global__ void __launch_bounds__(kAThreadsF, 1)
    attn_fwd_pv_kernel(const __grid_constant__ AttnParams P, const __grid_constant__ CUtensorMap mQ,
                       const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV,
                       const __grid_constant__ CUtensorMap mPst, const __grid_constant__ CUtensorMap mO) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint64_t* full = bars;                  // [3] K tile landed
  uint64_t* empty = bars + 3;             // [3] K tile consumed (its S MMA done)
  uint64_t* qfull = bars + 6;             // [2] Q of a task landed
  uint64_t* qempty = bars + 8;            // [2] the task's last S MMA done
  uint64_t* sfull = bars + 10;            // [3] S accumulator ready
  uint64_t* sempty = bars + 13;           // [3] S accumulator drained (8 warps)
  uint64_t* pfull = bars + 16;            // [2] P staging written (8 warps)
  uint64_t* pempty = bars + 18;           // [2] P staging consumed by MMA O
  uint64_t* ofull = bars + 20;            // [2] O accumulator of a task complete
  uint64_t* oempty = bars + 22;           // [2] O accumulator drained (4 warps)
  uint64_t* vfull = bars + 24;            // [3] V tile landed
  uint64_t* vempty = bars + 27;           // [3] V tile consumed (its O MMA done)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = P.B * P.H;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), kEW / 2);  // one ping-pong group per use
      mbar_init(smem_u32(&vfull[i]), 1);
      mbar_init(smem_u32(&vempty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&qfull[i]), 1);
      mbar_init(smem_u32(&qempty[i]), 1);
      mbar_init(smem_u32(&pfull[i]), kEW / 2);
      mbar_init(smem_u32(&pempty[i]), 1);
      mbar_init(smem_u32(&ofull[i]), 1);
      mbar_init(smem_u32(&oempty[i]), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NNT_PDL_ENTRY();
  // task t (heaviest first): level = t / BH -> query block qb = nblk - 1 - level; bh = t % BH
  auto decode = [&](int64_t t, int& qb, int& b, int& h) {  // (bgroup: levels interleaved per (b, h))
    const int g = P.bgroup;
    const int level = (int)(t / ((int64_t)g * BH)) * g + (int)(t % g), bh = (int)((t / g) % BH);
    qb = P.nblk - 1 - level;
    b = bh / P.H;
    h = bh % P.H;
  };
  const int64_t c0 = blockIdx.x, G = gridDim.x;
  const uint64_t pol_keep = P.l2hints == 1 ? l2_policy_evict_last() : l2_policy_evict_normal();
  const uint64_t pol_stream = P.l2hints ? l2_policy_evict_first() : l2_policy_evict_normal();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: Q and the K ring
    int stage = 0;
    uint32_t phase = 0;
    int tl = 0;
    int64_t it_p = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int qs = tl & 1;
      mbar_wait(smem_u32(&qempty[qs]), ((tl >> 1) & 1) ^ 1);
      mbar_expect_tx_w(smem_u32(&qfull[qs]), TILE16);
      tma_load_4d_w(smem_u32(smem + F_Q + qs * TILE16), &mQ, smem_u32(&qfull[qs]), 0, qb * TB, h, b);
      const int nk = P.causal ? qb + 1 : P.nblk;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        mbar_expect_tx_w(smem_u32(&full[stage]), TILE16);
        tma_load_4d_w_hint(smem_u32(smem + F_K + stage * TILE16), &mK, smem_u32(&full[stage]), 0, kb * TB, h, b,
                           pol_keep);  // K_kb: re-read by the (b, h)'s other query-block tasks
        if (lane == 0) trace_ev(P, 0, it_p);
        ++it_p;
        if (++stage == F_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    pdl_trigger();
  } else if (warp == 2 + kEW) {
    // ------------------------------------------------ TMA producer: the V ring (its tiles are
    // released by the O MMAs, later than the K tiles by the S MMAs: separate rings and producers
    // let the K loads run ahead)
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t k = 0;; ++k) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int nk = P.causal ? qb + 1 : P.nblk;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(&vempty[stage]), phase ^ 1);
        mbar_expect_tx_w(smem_u32(&vfull[stage]), TILE16);
        tma_load_4d_w_hint(smem_u32(smem + F_V + stage * TILE16), &mV, smem_u32(&vfull[stage]), 0, kb * TB, h, b,
                           pol_keep);
        if (++stage == F_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // A flat stream of iterations g over this CTA's tasks (S buffer g % 3, P buffer g % 2, stage
    // g % 3): the S MMAs run two iterations ahead of the O MMA of iteration g (which waits for the
    // epilogue's P), across task boundaries too, so each ping-pong epilogue group finds its next
    // S tile ready when it finishes a P tile.
    const uint32_t id_s = idesc_of(false, false, TB);  // S = Q K^T: both K-major, N = 128
    const uint32_t id_o = idesc_of(false, true, HD);   // O += P V: P K-major, V MN-major, N = 64
    struct Cur {
      int64_t k;  // task index in this CTA's schedule
      int tl, i, nk;
      bool ok;
    };
    auto first = [&]() {
      Cur c{0, 0, 0, 0, false};
      const int64_t t = task_at(c0, G, 0);
      if (t < P.num_tasks) {
        int qb, b, h;
        decode(t, qb, b, h);
        c.nk = P.causal ? qb + 1 : P.nblk;
        c.ok = true;
      }
      return c;
    };
    auto next = [&](Cur c) {
      if (++c.i < c.nk) return c;
      const int64_t t = task_at(c0, G, c.k + 1);
      if (t >= P.num_tasks) {
        c.ok = false;
        return c;
      }
      int qb, b, h;
      decode(t, qb, b, h);
      ++c.k;
      ++c.tl;
      c.i = 0;
      c.nk = P.causal ? qb + 1 : P.nblk;
      return c;
    };
    // S(g) can be issued without blocking: its Q, S buffer and K tile are there
    auto s_ready = [&](int64_t g, const Cur& c) {
      const int sb = (int)(g % 3), stg = (int)(g % F_STAGES), qs = c.tl & 1;
      return (c.i != 0 || mbar_test(smem_u32(&qfull[qs]), (c.tl >> 1) & 1)) &&
             mbar_test(smem_u32(&sempty[sb]), (uint32_t)(((g / 3) & 1) ^ 1)) &&
             mbar_test(smem_u32(&full[stg]), (uint32_t)((g / F_STAGES) & 1));
    };
    auto issue_s = [&](int64_t g, const Cur& c) {
      const int sb = (int)(g % 3), stg = (int)(g % F_STAGES), qs = c.tl & 1;
      if (c.i == 0) mbar_wait(smem_u32(&qfull[qs]), (c.tl >> 1) & 1);
      mbar_wait(smem_u32(&sempty[sb]), (uint32_t)(((g / 3) & 1) ^ 1));
      mbar_wait(smem_u32(&full[stg]), (uint32_t)((g / F_STAGES) & 1));
      tc_fence_after();
      const uint32_t sq = smem_u32(smem + F_Q + qs * TILE16);
      const uint32_t sk = smem_u32(smem + F_K + stg * TILE16);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        mma_bf16_w(tmem + sb * TB, make_sdesc(sq + kk * 32, 16, 1024), make_sdesc(sk + kk * 32, 16, 1024), id_s,
                   kk > 0 ? 1u : 0u);
      mma_commit_w(smem_u32(&sfull[sb]));
      mma_commit_w(smem_u32(&empty[stg]));  // the K tile is free
      if (lane == 0) trace_ev(P, 1, g);
      if (c.i == c.nk - 1) mma_commit_w(smem_u32(&qempty[qs]));  // the task's last S MMA: Q may be reloaded
    };
    Cur cur = first(), ahead1 = cur, ahead2 = cur;
    if (cur.ok) {
      issue_s(0, cur);
      ahead1 = next(cur);
      if (ahead1.ok) issue_s(1, ahead1);
      ahead2 = ahead1.ok ? next(ahead1) : ahead1;
    }
    for (int64_t g = 0; cur.ok; ++g) {
      // S(g + 2) now if nothing blocks it, else after O(g): O(g) never waits behind a K load
      bool s_pending = ahead2.ok;
      if (s_pending && s_ready(g + 2, ahead2)) {
        issue_s(g + 2, ahead2);
        s_pending = false;
      }
      // O += P V for iteration g
      const int os = cur.tl & 1, pb = (int)(g & 1), stg = (int)(g % F_STAGES);
      if (cur.i == 0) mbar_wait(smem_u32(&oempty[os]), ((cur.tl >> 1) & 1) ^ 1);
      mbar_wait(smem_u32(&vfull[stg]), (uint32_t)((g / F_STAGES) & 1));
      mbar_wait(smem_u32(&pfull[pb]), (uint32_t)((g >> 1) & 1));
      if (lane == 0) trace_ev(P, 4, g);
      tc_fence_after();
      const uint32_t sp = smem_u32(smem + F_P + pb * 2 * TILE16);
      const uint32_t sv = smem_u32(smem + F_V + stg * TILE16);
#pragma unroll
      for (int kk = 0; kk < TB / 16; ++kk)  // K = 128 keys: P chunk kk/4 (+16 KB), V rows +2 KB
        mma_bf16_w(tmem + 384 + os * HD, make_sdesc(sp + (kk >> 2) * TILE16 + (kk & 3) * 32, 16, 1024),
                   make_sdesc(sv + kk * 2048, 8192, 1024), id_o, (cur.i > 0 || kk > 0) ? 1u : 0u);
      mma_commit_w(smem_u32(&pempty[pb]));
      mma_commit_w(smem_u32(&vempty[stg]));
      if (lane == 0) trace_ev(P, 5, g);
      if (cur.i == cur.nk - 1) mma_commit_w(smem_u32(&ofull[os]));
      if (s_pending) issue_s(g + 2, ahead2);
      cur = ahead1;
      ahead1 = ahead2;
      if (ahead2.ok) ahead2 = next(ahead2);
    }
  } else if (warp < 2 + kEW) {
    // ------------------------------------------------ epilogue warps 2..17: two ping-pong groups
    // Group grp = (warp - 2) / 8 takes the iterations g with g % 2 == grp (S buffer, P staging
    // buffer grp), so each group has two iterations' time for its P tile: the epilogue's per-tile
    // latency chain (TMEM load, exponentials, staging, proxy fence, barrier, store) overlaps the
    // other group's.  Inside a group: TMEM lane quadrant quad (rows), 64-column chunk hc (two
    // 32-column halves in turn); each warp writes whole 128-byte staging rows and stores its piece.
    const int grp = (warp - 2) >> 3, quad = warp & 3, hc = ((warp - 2) >> 2) & 1;
    const float L2E = 1.4426950408889634f;
    const float sc = P.scale * L2E;
    int it = 0, tl = 0;
    // the row statistics of this lane's query row, loaded one task ahead
    auto stats_of = [&](int64_t tt) {
      if (tt >= P.num_tasks) return make_float2(0.f, 1.f);
      int qb_, b_, h_;
      decode(tt, qb_, b_, h_);
      return __ldg(reinterpret_cast<const float2*>(P.stats) +
                   ((int64_t)(b_ * P.H + h_) * P.S + qb_ * TB + quad * 32 + lane));
    };
    float2 st_next = stats_of(task_at(c0, G, 0));
    // O = P V of a finished task -> bf16 -> TMA store, by the 4 chunk-0 warps of the group that
    // owns the NEXT task's first iteration, after that iteration's P tile (O is double-buffered
    // in TMEM, so its completion and store overlap P work); O staging buffer grp
    auto o_epilogue = [&](int tlo, int qbo, int bo, int ho) {
      if (hc != 0) return;
      const int os = tlo & 1;
      mbar_wait(smem_u32(&ofull[os]), (tlo >> 1) & 1);
      tc_fence_after();
      float v[64];
      tmem_ld_cols<2>(tmem + 384 + os * HD + ((uint32_t)(quad * 32) << 16), v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&oempty[os]));
      uint8_t* piece = smem + F_O + grp * TILE16 + quad * PIECE;
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      stage_row<__nv_bfloat16, 64>(piece, lane, v);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d(&mO, smem_u32(piece), 0, qbo * TB + quad * 32, ho, bo);
        bulk_commit();
      }
    };
    int pq = -1, pb_ = 0, ph = 0;  // the task whose O epilogue is pending
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int q = qb * TB + quad * 32 + lane;  // this lane's query row
      const float2 st = st_next;
      st_next = stats_of(task_at(c0, G, k + 1));
      const float ml = st.x * L2E, inv = rcp_approx(st.y);
      const int nk = P.causal ? qb + 1 : P.nblk;
      for (int i = 0; i < nk; ++i, ++it) {
        if ((it & 1) != grp) continue;
        const int sb = it % 3, pbuf = it & 1;  // S buffer, P staging buffer (== grp)
        mbar_wait(smem_u32(&sfull[sb]), (uint32_t)((it / 3) & 1));
        if (warp == 2 && lane == 0) trace_ev(P, 2, it);
        tc_fence_after();
        // P staging buffer grp: free once MMA O of iteration it-2 (pempty) and this warp's store
        // of it (its most recent bulk group) are done
        mbar_wait(smem_u32(&pempty[pbuf]), ((it >> 1) & 1) ^ 1);
        uint8_t* piece = smem + F_P + pbuf * 2 * TILE16 + hc * TILE16 + quad * PIECE;
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          float v[32];
          tmem_ld32(tmem + sb * TB + hc * 64 + sub * 32 + ((uint32_t)(quad * 32) << 16), v);
          if (sub == 1) {  // the S buffer is free once both halves are in registers
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&sempty[sb]));
          }
          const int key0 = i * TB + hc * 64 + sub * 32;
          int lim = 32;  // causal: keys <= q
          if (P.causal && key0 + 31 > q) lim = q - key0 + 1;
          if (lim >= 32) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float2 x = __ffma2_rn(make_float2(v[j], v[j + 1]), make_float2(sc, sc), make_float2(-ml, -ml));
              const float2 y = __fmul2_rn(make_float2(ex2_approx(x.x), ex2_approx(x.y)), make_float2(inv, inv));
              v[j] = y.x;
              v[j + 1] = y.y;
            }
          } else if (lim > 0) {  // diagonal tile: keys > q masked (-> 0)
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = ex2_approx(j < lim ? fmaf(v[j], sc, -ml) : -INFINITY) * inv;
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          stage_half_row(piece, lane, sub, v);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(smem_u32(&pfull[pbuf]));
          if (warp == 2) trace_ev(P, 3, it);
          tma_store_4d_hint(&mPst, smem_u32(piece), i * TB + hc * 64, qb * TB + quad * 32, h, b, pol_stream);
          bulk_commit();
        }
        if (i == 0 && pq >= 0) o_epilogue(tl - 1, pq, pb_, ph);  // the previous task's O
      }
      pq = qb;
      pb_ = b;
      ph = h;
    }
    if (pq >= 0 && (it & 1) == grp) o_epilogue(tl - 1, pq, pb_, ph);
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem);
  }
}

// ============================================================================ row statistics
// Softmax subroutine 1 on the score tiles of one (b, h, query block) task, formed on
// the tensor cores and never stored (R26): per query row the running (max, sumexp) over the key
// tiles, merged with the rule of R10.  The pipeline of the forward kernel without the value
// product: warp 0 streams Q (per task) and the K tiles (3-stage ring), warp 1 issues S = Q K^T
// into three TMEM buffers, two ping-pong groups of 8 epilogue warps (iterations g % 2) reduce a
// tile's 32-key halves into per-lane running pairs, and at the end of a task each epilogue warp
// deposits its pair in a shared-memory slot; warp 18 merges the 4 pairs of each row (group 0 /
// 1 x key half 0 / 1, fixed order) and writes (M, S) -- M in scaled-score units, S = sum
// e^{scale x - M} -- the format of the NNT_ACT_ROWSTATS GEMM epilogue.
constexpr int R_STAGES = 3;
constexpr int R_Q = 0, R_K = 2 * TILE16, R_X = R_K + R_STAGES * TILE16;  // X: [2][4 quad][4][32] float2
constexpr int R_BAR = R_X + 2 * 4 * 4 * 32 * 8;
constexpr int R_SMEM = R_BAR + 256 + 1024;
constexpr int kAThreadsR = kAThreads + 32;  // + the merge warp (warp 18)

__global__ void __launch_bounds__(kAThreadsR, 1)
    attn_stats_kernel(const __grid_constant__ AttnParams P, const __grid_constant__ CUtensorMap mQ,
                      const __grid_constant__ CUtensorMap mK, float* __restrict__ stats) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + R_BAR);
  uint64_t* full = bars;        // [3] K tile landed
  uint64_t* empty = bars + 3;   // [3] K tile consumed (its S MMA done)
  uint64_t* qfull = bars + 6;   // [2]
  uint64_t* qempty = bars + 8;  // [2] the task's last S MMA done
  uint64_t* sfull = bars + 10;  // [3] S accumulator ready
  uint64_t* sempty = bars + 13; // [3] drained (8 warps)
  uint64_t* xfull = bars + 16;  // [2] a task's 16 per-warp pairs deposited (16 warps)
  uint64_t* xempty = bars + 18; // [2] merged (warp 18)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
  float2* xs = reinterpret_cast<float2*>(smem + R_X);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = P.B * P.H;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), kEW / 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&qfull[i]), 1);
      mbar_init(smem_u32(&qempty[i]), 1);
      mbar_init(smem_u32(&xfull[i]), kEW);
      mbar_init(smem_u32(&xempty[i]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NNT_PDL_ENTRY();
  auto decode = [&](int64_t t, int& qb, int& b, int& h) {  // heaviest first, as the forward
    const int g = P.bgroup;
    const int level = (int)(t / ((int64_t)g * BH)) * g + (int)(t % g), bh = (int)((t / g) % BH);
    qb = P.nblk - 1 - level;
    b = bh / P.H;
    h = bh % P.H;
  };
  const int64_t c0 = blockIdx.x, G = gridDim.x;
  const uint64_t pol_keep = P.l2hints == 1 ? l2_policy_evict_last() : l2_policy_evict_normal();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: Q and the K ring
    int stage = 0;
    uint32_t phase = 0;
    int tl = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int qs = tl & 1;
      mbar_wait(smem_u32(&qempty[qs]), ((tl >> 1) & 1) ^ 1);
      mbar_expect_tx_w(smem_u32(&qfull[qs]), TILE16);
      tma_load_4d_w(smem_u32(smem + R_Q + qs * TILE16), &mQ, smem_u32(&qfull[qs]), 0, qb * TB, h, b);
      const int nk = P.causal ? qb + 1 : P.nblk;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        mbar_expect_tx_w(smem_u32(&full[stage]), TILE16);
        tma_load_4d_w_hint(smem_u32(smem + R_K + stage * TILE16), &mK, smem_u32(&full[stage]), 0, kb * TB, h, b,
                           pol_keep);
        if (++stage == R_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    pdl_trigger();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer: S(g) = Q K_kb^T into buffer g % 3
    const uint32_t id_s = idesc_of(false, false, TB);
    int tl = 0;
    int64_t g = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int qs = tl & 1, nk = P.causal ? qb + 1 : P.nblk;
      mbar_wait(smem_u32(&qfull[qs]), (tl >> 1) & 1);
      for (int i = 0; i < nk; ++i, ++g) {
        const int sb = (int)(g % 3), stg = (int)(g % R_STAGES);
        mbar_wait(smem_u32(&sempty[sb]), (uint32_t)(((g / 3) & 1) ^ 1));
        mbar_wait(smem_u32(&full[stg]), (uint32_t)((g / R_STAGES) & 1));
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + R_Q + qs * TILE16), sk = smem_u32(smem + R_K + stg * TILE16);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_w(tmem + sb * TB, make_sdesc(sq + kk * 32, 16, 1024), make_sdesc(sk + kk * 32, 16, 1024), id_s,
                     kk > 0 ? 1u : 0u);
        mma_commit_w(smem_u32(&sfull[sb]));
        mma_commit_w(smem_u32(&empty[stg]));
        if (i == nk - 1) mma_commit_w(smem_u32(&qempty[qs]));
      }
    }
  } else if (warp < 2 + kEW) {
    // ------------------------------------------------ epilogue warps 2..17
    const int grp = (warp - 2) >> 3, quad = warp & 3, hc = ((warp - 2) >> 2) & 1;
    const float sc = P.scale * 1.4426950408889634f;  // log2-scaled scores: y = x * scale * log2(e)
    int it = 0, tl = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int q = qb * TB + quad * 32 + lane;  // this lane's query row
      const int nk = P.causal ? qb + 1 : P.nblk;
      float m = -INFINITY, l = 0.f;  // running (max, sumexp) in log2 units over this warp's keys
      for (int i = 0; i < nk; ++i, ++it) {
        if ((it & 1) != grp) continue;
        const int sb = it % 3;
        mbar_wait(smem_u32(&sfull[sb]), (uint32_t)((it / 3) & 1));
        tc_fence_after();
        float v[64];
        tmem_ld_cols<2>(tmem + sb * TB + hc * 64 + ((uint32_t)(quad * 32) << 16), v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sempty[sb]));
        const int key0 = i * TB + hc * 64;
        int lim = 64;  // causal: keys <= q
        if (P.causal && key0 + 63 > q) lim = q - key0 + 1;
        if (lim >= 64) {
          float m0 = fmaxf(v[0], v[1]), m1 = fmaxf(v[2], v[3]);
#pragma unroll
          for (int j = 4; j < 64; j += 4) {
            m0 = fmaxf(m0, fmaxf(v[j], v[j + 1]));
            m1 = fmaxf(m1, fmaxf(v[j + 2], v[j + 3]));
          }
          const float mn = fmaxf(m, fmaxf(m0, m1) * sc);
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int j = 0; j < 64; j += 4) {
            s0 += ex2_approx(fmaf(v[j], sc, -mn));
            s1 += ex2_approx(fmaf(v[j + 1], sc, -mn));
            s2 += ex2_approx(fmaf(v[j + 2], sc, -mn));
            s3 += ex2_approx(fmaf(v[j + 3], sc, -mn));
          }
          l = l * ex2_approx(m - mn) + ((s0 + s1) + (s2 + s3));
          m = mn;
        } else if (lim > 0) {  // diagonal tile: keys > q masked
          float mx = -INFINITY;
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < lim) mx = fmaxf(mx, v[j]);
          const float mn = fmaxf(m, mx * sc);
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j < lim) s += ex2_approx(fmaf(v[j], sc, -mn));
          l = (m == -INFINITY ? 0.f : l * ex2_approx(m - mn)) + s;
          m = mn;
        }
      }
      // this warp's pair for the task -> slot (task parity, quad, grp * 2 + hc, lane)
      const int xs_ = tl & 1;
      mbar_wait(smem_u32(&xempty[xs_]), ((tl >> 1) & 1) ^ 1);
      xs[((xs_ * 4 + quad) * 4 + grp * 2 + hc) * 32 + lane] = make_float2(m, l);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&xfull[xs_]));
    }
  } else {
    // ------------------------------------------------ warp 18: merge the 4 pairs of each row
    int tl = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int qb, b, h;
      decode(t, qb, b, h);
      const int xs_ = tl & 1;
      mbar_wait(smem_u32(&xfull[xs_]), (tl >> 1) & 1);
      float2* out = reinterpret_cast<float2*>(stats) + ((int64_t)(b * P.H + h) * P.S + qb * TB);
#pragma unroll 1
      for (int quad = 0; quad < 4; ++quad) {
        float2 pr[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) pr[w] = xs[((xs_ * 4 + quad) * 4 + w) * 32 + lane];
        float M = fmaxf(fmaxf(pr[0].x, pr[1].x), fmaxf(pr[2].x, pr[3].x));
        float S = 0.f;
        if (M != -INFINITY) {
#pragma unroll
          for (int w = 0; w < 4; ++w)  // fixed order: (group 0, half 0), (0, 1), (1, 0), (1, 1)
            if (pr[w].x != -INFINITY) S += pr[w].y * ex2_approx(pr[w].x - M);
        }
        out[quad * 32 + lane] = make_float2(M * 0.6931471805599453f, S);  // (scaled-score max, sumexp)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&xempty[xs_]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem);
  }
}

// ============================================================================ backward
// smem: V[2] (task parity) | 3 stages of {dO_qb, Q_qb, P tile (2 x 16 KB)} | D slots [3] | barriers.
// TMEM: dP[2] at columns 0 / 128, {dV, dK}[2] at 256 / 384 (+64 for dK).
// Iteration g (a query block of a task) uses stage g % 3 and dP buffer g % 2, and is processed by
// epilogue group g % 2.  dP = dO V^T puts the tile's queries on the TMEM lanes, so an epilogue lane
// owns one query row: it reads that row of P as 16-byte chunks, forms dA = P (dP - D) / sqrt(h)
// and writes it back IN PLACE over P (the dV MMA that read P is committed with dP, so it has
// completed when the epilogue sees dP); the tile then serves as the A operand of dK += dA^T Q (the
// same MN-major view dV uses for P^T) and is stored by TMA (query-major dA, for dQ = dA K).  No
// separate dA staging: the freed 64 KB hold a third operand stage.
constexpr int B_STAGES = 3;
constexpr int B_D_BYTES = TB * 4;                    // D of the stage's query block (bulk copy)
constexpr int B_STAGE_TX = 4 * TILE16 + B_D_BYTES;   // bytes landing per stage
constexpr int B_STAGE_BYTES = 4 * TILE16;
constexpr int B_V = 0, B_ST = 2 * TILE16, B_D = B_ST + B_STAGES * B_STAGE_BYTES;
constexpr int B_BAR = B_D + B_STAGES * B_D_BYTES;
constexpr int B_SMEM = B_BAR + 256 + 1024;
static_assert(B_SMEM <= 232448, "backward shared memory budget");

__global__ void __launch_bounds__(kAThreads, 1)
    attn_bwd_kv_kernel(const __grid_constant__ AttnParams P, const __grid_constant__ CUtensorMap mV,
                       const __grid_constant__ CUtensorMap mdO, const __grid_constant__ CUtensorMap mQ,
                       const __grid_constant__ CUtensorMap mP, const __grid_constant__ CUtensorMap mdA,
                       const __grid_constant__ CUtensorMap mdK, const __grid_constant__ CUtensorMap mdV) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + B_BAR);
  uint64_t* full = bars;           // [3] stage dO, Q, P, D landed
  uint64_t* empty = bars + 3;      // [3] stage released: MMA dK committed + the 8 warps of its group (dA stored)
  uint64_t* vfull = bars + 6;      // [2]
  uint64_t* vempty = bars + 8;     // [2] the task's last dP MMA done
  uint64_t* tfull = bars + 10;     // [2] dP accumulator ready (and the iteration's dV MMA done)
  uint64_t* tempty = bars + 12;    // [2] drained (8 warps)
  uint64_t* dafull = bars + 14;    // [2] dA of group g written over P (8 warps)
  uint64_t* afull = bars + 16;     // [2] dV, dK of a task complete
  uint64_t* aempty = bars + 18;    // [2] drained (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BH = P.B * P.H;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < B_STAGES; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1 + kEW / 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&vfull[i]), 1);
      mbar_init(smem_u32(&vempty[i]), 1);
      mbar_init(smem_u32(&tfull[i]), 1);
      mbar_init(smem_u32(&tempty[i]), kEW / 2);
      mbar_init(smem_u32(&dafull[i]), kEW / 2);
      mbar_init(smem_u32(&afull[i]), 1);
      mbar_init(smem_u32(&aempty[i]), kEW / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NNT_PDL_ENTRY();
  // task t (heaviest first): level = t / BH -> key block kb = level (causal: nblk - kb query blocks)
  // bgroup g > 1: levels [j g, (j+1) g) of one (b, h) are consecutive tasks, so they run at the same
  // time and share their dO / Q tiles in L2 (level-major: a (b, h)'s next level runs ~1.4 rounds later)
  auto decode = [&](int64_t t, int& kb, int& b, int& h) {
    const int g = P.bgroup;
    const int level = (int)(t / ((int64_t)g * BH)) * g + (int)(t % g), bh = (int)((t / g) % BH);
    kb = level;
    b = bh / P.H;
    h = bh % P.H;
  };
  auto q_first = [&](int kb) { return P.causal ? kb : 0; };
  const int64_t c0 = blockIdx.x, G = gridDim.x;
  const uint64_t pol_keep = P.l2hints == 1 ? l2_policy_evict_last() : l2_policy_evict_normal();
  const uint64_t pol_stream = P.l2hints ? l2_policy_evict_first() : l2_policy_evict_normal();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    int tl = 0;
    int64_t it_p = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int kb, b, h;
      decode(t, kb, b, h);
      const int vs = tl & 1;
      mbar_wait(smem_u32(&vempty[vs]), ((tl >> 1) & 1) ^ 1);
      mbar_expect_tx_w(smem_u32(&vfull[vs]), TILE16);
      tma_load_4d_w(smem_u32(smem + B_V + vs * TILE16), &mV, smem_u32(&vfull[vs]), 0, kb * TB, h, b);
      for (int qb = q_first(kb); qb < P.nblk; ++qb) {
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        const uint32_t st = smem_u32(smem + B_ST + stage * B_STAGE_BYTES);
        const uint32_t fb = smem_u32(&full[stage]);
        mbar_expect_tx_w(fb, B_STAGE_TX);
        bulk_load_w(smem_u32(smem + B_D + stage * B_D_BYTES), P.D + ((int64_t)(b * P.H + h) * P.S + qb * TB),
                    B_D_BYTES, fb);
        // dO_qb / Q_qb are re-read by the (b, h)'s other key-block tasks (kept in L2); P is read once
        tma_load_4d_w_hint(st, &mdO, fb, 0, qb * TB, h, b, pol_keep);
        tma_load_4d_w_hint(st + TILE16, &mQ, fb, 0, qb * TB, h, b, pol_keep);
        if (P.p_blk) {  // both 64-key halves of the P tile in one request
          tma_load_5d_w_hint(st + 2 * TILE16, &mP, fb, 0, qb * TB, kb * (TB / 64), h, b, pol_stream);
        } else {
          tma_load_4d_w_hint(st + 2 * TILE16, &mP, fb, kb * TB, qb * TB, h, b, pol_stream);       // keys kb*128 + 0..63
          tma_load_4d_w_hint(st + 3 * TILE16, &mP, fb, kb * TB + 64, qb * TB, h, b, pol_stream);  // keys + 64..127
        }
        if (lane == 0) trace_ev(P, 0, it_p);
        ++it_p;
        if (++stage == B_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    pdl_trigger();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // A flat stream of iterations g over this CTA's tasks.  issue_dp(g) = dP of g (dO V^T) then dV
    // += P^T dO of g, one commit: the epilogue may overwrite P once dP is visible.  The dP / dV of
    // iteration g + 1 is issued as soon as nothing blocks it -- before the dK MMA of iteration g if
    // possible (which waits for the epilogue's dA), else right after it.
    const uint32_t id_dp = idesc_of(false, false, TB);  // dP = dO V^T: both K-major, N = 128 keys
    const uint32_t id_pt = idesc_of(true, true, HD);    // dV += P^T dO, dK += dA^T Q: both MN-major
    struct Cur {
      int64_t k;
      int tl, i, nq;
      bool ok;
    };
    auto nq_of = [&](int64_t t) {
      int kb, b, h;
      decode(t, kb, b, h);
      return P.nblk - q_first(kb);
    };
    auto next = [&](Cur c) {
      if (++c.i < c.nq) return c;
      const int64_t t = task_at(c0, G, c.k + 1);
      if (t >= P.num_tasks) {
        c.ok = false;
        return c;
      }
      ++c.k;
      ++c.tl;
      c.i = 0;
      c.nq = nq_of(t);
      return c;
    };
    auto dp_ready = [&](int64_t g, const Cur& c) {
      const uint32_t tp = (uint32_t)((c.tl >> 1) & 1);
      return (c.i != 0 || (mbar_test(smem_u32(&vfull[c.tl & 1]), tp) && mbar_test(smem_u32(&aempty[c.tl & 1]), tp ^ 1))) &&
             mbar_test(smem_u32(&tempty[g & 1]), (uint32_t)(((g >> 1) & 1) ^ 1)) &&
             mbar_test(smem_u32(&full[g % B_STAGES]), (uint32_t)((g / B_STAGES) & 1));
    };
    auto issue_dp = [&](int64_t g, const Cur& c) {
      const int tb = (int)(g & 1), stg = (int)(g % B_STAGES), vs = c.tl & 1;
      if (c.i == 0) {
        mbar_wait(smem_u32(&vfull[vs]), (c.tl >> 1) & 1);
        mbar_wait(smem_u32(&aempty[vs]), ((c.tl >> 1) & 1) ^ 1);  // the task's dV / dK buffer drained
      }
      mbar_wait(smem_u32(&tempty[tb]), (uint32_t)(((g >> 1) & 1) ^ 1));
      mbar_wait(smem_u32(&full[stg]), (uint32_t)((g / B_STAGES) & 1));
      tc_fence_after();
      const uint32_t sv = smem_u32(smem + B_V + vs * TILE16);
      const uint32_t st = smem_u32(smem + B_ST + stg * B_STAGE_BYTES);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        mma_bf16_w(tmem + tb * TB, make_sdesc(st + kk * 32, 16, 1024), make_sdesc(sv + kk * 32, 16, 1024), id_dp,
                   kk > 0 ? 1u : 0u);
      // dV += P^T dO (both operands in the stage): K = 128 queries
      const uint32_t tdv = tmem + 256 + vs * 128;
#pragma unroll
      for (int kk = 0; kk < TB / 16; ++kk)
        mma_bf16_w(tdv, make_sdesc(st + 2 * TILE16 + kk * 2048, TILE16, 1024), make_sdesc(st + kk * 2048, 8192, 1024),
                   id_pt, (c.i > 0 || kk > 0) ? 1u : 0u);
      mma_commit_w(smem_u32(&tfull[tb]));
      if (lane == 0) trace_ev(P, 1, g);
      if (c.i == c.nq - 1) mma_commit_w(smem_u32(&vempty[vs]));  // the task's last dP MMA: V may be reloaded
    };
    Cur cur{0, 0, 0, 0, false};
    {
      const int64_t t0 = task_at(c0, G, 0);
      if (t0 < P.num_tasks) {
        cur.nq = nq_of(t0);
        cur.ok = true;
      }
    }
    if (cur.ok) issue_dp(0, cur);
    for (int64_t g = 0; cur.ok; ++g) {
      const int as = cur.tl & 1, stg = (int)(g % B_STAGES), db = (int)(g & 1);
      const uint32_t st = smem_u32(smem + B_ST + stg * B_STAGE_BYTES);
      const uint32_t tdk = tmem + 256 + as * 128 + HD;
      const Cur nxt = next(cur);
      bool pending = nxt.ok;
      if (pending && dp_ready(g + 1, nxt)) {
        issue_dp(g + 1, nxt);
        pending = false;
      }
      // dK += dA^T Q once group g % 2 has written dA over the stage's P tile
      mbar_wait(smem_u32(&dafull[db]), (uint32_t)((g >> 1) & 1));
      if (lane == 0) trace_ev(P, 4, g);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < TB / 16; ++kk)
        mma_bf16_w(tdk, make_sdesc(st + 2 * TILE16 + kk * 2048, TILE16, 1024),
                   make_sdesc(st + TILE16 + kk * 2048, 8192, 1024), id_pt, (cur.i > 0 || kk > 0) ? 1u : 0u);
      if (lane == 0) trace_ev(P, 5, g);
      mma_commit_w(smem_u32(&empty[stg]));
      if (cur.i == cur.nq - 1) mma_commit_w(smem_u32(&afull[as]));
      if (pending) issue_dp(g + 1, nxt);
      cur = nxt;
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..17: two ping-pong groups
    // Group grp = (warp - 2) / 8 takes the iterations g with g % 2 == grp.  Inside a group: TMEM
    // lane quadrant quad (query rows quad*32 ..), key half hc (P box hc: keys hc*64 .. +63, the
    // lane's 128-byte row of it).  The group that ran a task's last iteration then drains its dK
    // (hc 0) / dV (hc 1) through its own dA piece of the stage.
    const int grp = (warp - 2) >> 3, quad = warp & 3, hc = ((warp - 2) >> 2) & 1;
    const int qrow = quad * 32 + lane;  // this lane's query row of the tile
    int it = 0, tl = 0;
    for (int64_t k = 0;; ++k, ++tl) {
      const int64_t t = task_at(c0, G, k);
      if (t >= P.num_tasks) break;
      int kb, b, h;
      decode(t, kb, b, h);
      const int q0 = q_first(kb);
      for (int qb = q0; qb < P.nblk; ++qb, ++it) {
        if ((it & 1) != grp) continue;
        const int stg = it % B_STAGES;
        mbar_wait(smem_u32(&tfull[grp]), (it >> 1) & 1);
        if (warp == 2 && lane == 0) trace_ev(P, 2, it);
        tc_fence_after();
        mbar_wait(smem_u32(&full[stg]), (uint32_t)((it / B_STAGES) & 1));  // P and D of this stage
        uint8_t* const box = smem + B_ST + stg * B_STAGE_BYTES + 2 * TILE16 + hc * TILE16;
        uint8_t* const prow = box + qrow * 128;
        uint8_t* const piece = box + quad * PIECE;  // this warp's 32 rows of the box
        const float dq = reinterpret_cast<const float*>(smem + B_D + stg * B_D_BYTES)[qrow];
#pragma unroll 1
        for (int sub = 0; sub < 2; ++sub) {
          float v[32];  // dP[query = qrow][key = hc * 64 + sub * 32 + j]
          tmem_ld32(tmem + grp * TB + hc * 64 + sub * 32 + ((uint32_t)(quad * 32) << 16), v);
          if (sub == 1) {  // the dP buffer is free once both halves are in registers
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty[grp]));
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {  // 16-byte chunk sub * 4 + c of the row: keys 8 (sub*4+c) ..
            uint4* ptr = reinterpret_cast<uint4*>(prow + (((sub * 4 + c) ^ (qrow & 7)) << 4));
            uint4 u = *ptr;
            uint32_t* wd = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 pp = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wd[e]));
              const float a0 = (pp.x * P.scale) * (v[8 * c + 2 * e] - dq);  // dA = P (dP - D) / sqrt(h)  (R20)
              const float a1 = (pp.y * P.scale) * (v[8 * c + 2 * e + 1] - dq);
              __nv_bfloat162 r = __floats2bfloat162_rn(a0, a1);
              wd[e] = *reinterpret_cast<uint32_t*>(&r);
            }
            *ptr = u;
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(smem_u32(&dafull[grp]));
          if (warp == 2) trace_ev(P, 3, it);
          tma_store_4d_hint(&mdA, smem_u32(piece), kb * TB + hc * 64, qb * TB + quad * 32, h, b, pol_stream);
          bulk_commit();
        }
        if (qb == P.nblk - 1) {
          // dK (hc 0) / dV (hc 1) of the key block -> bf16 -> TMA store, staged in this warp's dA
          // piece (afull: the task's dK MMAs, the last readers of the stage, are done; the dA
          // store has read the piece)
          const int as = tl & 1;
          mbar_wait(smem_u32(&afull[as]), (tl >> 1) & 1);
          tc_fence_after();
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            float v[32];
            tmem_ld32(tmem + 256 + as * 128 + (hc == 0 ? HD : 0) + sub * 32 + ((uint32_t)(quad * 32) << 16), v);
            stage_half_row(piece, lane, sub, v);
          }
          tc_fence_before();
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(smem_u32(&aempty[as]));
            tma_store_4d(hc == 0 ? &mdK : &mdV, smem_u32(piece), 0, kb * TB + quad * 32, h, b);
            bulk_commit();
          }
        }
        if (lane == 0) {  // the stage may be refilled once this warp's stores have read it
          bulk_wait_read0();
          mbar_arrive(smem_u32(&empty[stg]));
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem);
  }
}

int64_t persistent_grid(int64_t tasks) { return tasks < num_sms() ? tasks : num_sms(); }

bool g_trace_on = false;
// key / query-block levels interleaved per (b, h) in groups of g (attention kernels' task order;
// NNT_ATTN_FGROUP: forward / statistics, NNT_ATTN_BGROUP: backward; 1 = level-major)
int attn_group(const char* var, int64_t nblk) {
  const char* e = getenv(var);
  const int g = e ? atoi(e) : 1;
  return (g > 1 && nblk % g == 0) ? g : 1;
}

int l2hints_on() {  // read per call (A/B runs switch it within one process)
  const char* e = getenv("NNT_ATTN_L2HINT");
  return e ? atoi(e) : 2;
}
unsigned long long* trace_ptr(int which) {
  if (!g_trace_on) return nullptr;
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_attn_trace) != cudaSuccess) return nullptr;
  return reinterpret_cast<unsigned long long*>(p) + (size_t)which * kTraceEv * kTraceIt;
}

nnt_status check_attn(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t Dh, const char* what) {
  NNT_REQUIRE(qkv, NNT_ERR_NULL, "%s: NULL pointer", what);
  NNT_REQUIRE(B > 0 && H > 0 && S > 0 && B * H * S < (1ll << 31), NNT_ERR_SHAPE, "%s: B=%lld S=%lld H=%lld", what,
              (long long)B, (long long)S, (long long)H);
  NNT_REQUIRE(Dh == HD && S % TB == 0, NNT_ERR_UNSUPPORTED, "%s: needs head size 64 and S %% 128 == 0 (Dh=%lld S=%lld)",
              what, (long long)Dh, (long long)S);
  NNT_REQUIRE(aligned16(qkv), NNT_ERR_ALIGN, "%s: 16-byte alignment", what);
  return NNT_OK;
}

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_attention_trace(int enable, uint64_t* host_out, int64_t cap) {
  g_trace_on = enable != 0;
  if (host_out && cap > 0) {
    const int64_t n = cap < 2 * kTraceEv * kTraceIt ? cap : 2 * kTraceEv * kTraceIt;
    NNT_CUDA_TRY(cudaMemcpyFromSymbol(host_out, g_attn_trace, (size_t)n * sizeof(uint64_t)));
  }
  return NNT_OK;
}

int nnt_attention_fused_supported(int64_t S, int64_t Dh) { return Dh == HD && S > 0 && S % TB == 0 ? 1 : 0; }

// NNT_ATTN_STATS=0: the row statistics by the NNT_ACT_ROWSTATS score GEMM (A/B runs)
int nnt_attention_stats_enabled() {
  const char* e = getenv("NNT_ATTN_STATS");
  return e && e[0] == '0' ? 0 : 1;
}

nnt_status nnt_attention_stats(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t Dh, float scale, int causal,
                               float* stats, nnt_stream_t stream) {
  NNT_TRY(check_attn(qkv, B, S, H, Dh, "nnt_attention_stats"));
  NNT_REQUIRE(stats, NNT_ERR_NULL, "nnt_attention_stats: NULL stats");
  NNT_REQUIRE(aligned16(stats), NNT_ERR_ALIGN, "nnt_attention_stats: alignment");
  const int64_t Ea = H * Dh, nblk = S / TB;
  AttnParams prm{(int)B, (int)H, (int)S, (int)nblk, (int)(B * H * nblk), causal ? 1 : 0, scale, nullptr, nullptr,
                 nullptr, l2hints_on(), 0, attn_group("NNT_ATTN_FGROUP", nblk)};
  CUtensorMap mQ, mK;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const __nv_bfloat16* q = (const __nv_bfloat16*)qkv;
  NNT_TRY(make_tma_map_4d(&mQ, bf, 2, q, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mK, bf, 2, q + Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  // algorithmic bytes: Q and K read once, the (max, sumexp) pairs written
  const double ptiles = (double)B * H * (causal ? nblk * (nblk + 1) / 2 : nblk * nblk);
  LaunchScope sc(NNT_K_GEMM_TC_ATTN, stream, 2.0 * B * S * Ea * 2 + 8.0 * B * H * S, ptiles * 2.0 * TB * TB * HD);
  NNT_CUDA_TRY(set_max_dyn_smem(attn_stats_kernel, R_SMEM));
  NNT_CUDA_TRY(::nnt::launch(attn_stats_kernel, dim3((unsigned)persistent_grid(prm.num_tasks)), dim3(kAThreadsR),
                             (size_t)R_SMEM, (cudaStream_t)stream, prm, mQ, mK, stats));
  return check_launch("attn_stats");
}

nnt_status nnt_attention_fwd_pv(const void* qkv, int64_t B, int64_t S, int64_t H, int64_t Dh, float scale,
                                int causal, const float* stats, void* P, void* O, nnt_stream_t stream) {
  NNT_TRY(check_attn(qkv, B, S, H, Dh, "nnt_attention_fwd_pv"));
  NNT_REQUIRE(stats && P && O, NNT_ERR_NULL, "nnt_attention_fwd_pv: NULL pointer");
  NNT_REQUIRE(aligned16(P) && aligned16(O) && aligned16(stats), NNT_ERR_ALIGN, "nnt_attention_fwd_pv: alignment");
  const int64_t Ea = H * Dh, nblk = S / TB;
  AttnParams prm{(int)B, (int)H, (int)S, (int)nblk, (int)(B * H * nblk), causal ? 1 : 0, scale, stats, nullptr,
                 trace_ptr(0), l2hints_on(), 0, attn_group("NNT_ATTN_FGROUP", nblk)};
  CUtensorMap mQ, mK, mV, mPst, mO;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const __nv_bfloat16* q = (const __nv_bfloat16*)qkv;
  NNT_TRY(make_tma_map_4d(&mQ, bf, 2, q, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mK, bf, 2, q + Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mV, bf, 2, q + 2 * Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mPst, bf, 2, P, S, S, S, H, S * S, B, H * S * S, 64, 32));
  NNT_TRY(make_tma_map_4d(&mO, bf, 2, O, Dh, S, Ea, H, Dh, B, S * Ea, 64, 32));
  // algorithmic bytes: P written once (causal: the lower-triangular 128 x 128 tiles), O written,
  // Q / K / V read once each
  const double ptiles = (double)B * H * (causal ? nblk * (nblk + 1) / 2 : nblk * nblk);
  LaunchScope sc(NNT_K_GEMM_TC_ATTN, stream, ptiles * TB * TB * 2 + 4.0 * B * S * Ea * 2,
                 ptiles * 4.0 * TB * TB * HD);
  NNT_CUDA_TRY(set_max_dyn_smem(attn_fwd_pv_kernel, F_SMEM));
  NNT_CUDA_TRY(::nnt::launch(attn_fwd_pv_kernel, dim3((unsigned)persistent_grid(prm.num_tasks)), dim3(kAThreadsF),
                             (size_t)F_SMEM, (cudaStream_t)stream, prm, mQ, mK, mV, mPst, mO));
  return check_launch("attn_fwd_pv");
}

nnt_status nnt_attention_bwd_kv(const void* qkv, const void* dO, const void* P, const float* D, int64_t B, int64_t S,
                                int64_t H, int64_t Dh, float scale, int causal, void* dA, void* dqkv,
                                nnt_stream_t stream) {
  NNT_TRY(check_attn(qkv, B, S, H, Dh, "nnt_attention_bwd_kv"));
  NNT_REQUIRE(dO && P && D && dA && dqkv, NNT_ERR_NULL, "nnt_attention_bwd_kv: NULL pointer");
  NNT_REQUIRE(aligned16(dO) && aligned16(P) && aligned16(D) && aligned16(dA) && aligned16(dqkv), NNT_ERR_ALIGN,
              "nnt_attention_bwd_kv: alignment");
  const int64_t Ea = H * Dh, nblk = S / TB;
  AttnParams prm{(int)B, (int)H, (int)S, (int)nblk, (int)(B * H * nblk), causal ? 1 : 0, scale, nullptr, D,
                 trace_ptr(1), l2hints_on(), 0, 1};
  CUtensorMap mV, mdO, mQ, mP, mdA, mdK, mdV;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const __nv_bfloat16* q = (const __nv_bfloat16*)qkv;
  __nv_bfloat16* dq = (__nv_bfloat16*)dqkv;
  NNT_TRY(make_tma_map_4d(&mV, bf, 2, q + 2 * Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mQ, bf, 2, q, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, TB));
  NNT_TRY(make_tma_map_4d(&mdO, bf, 2, dO, Dh, S, Ea, H, Dh, B, S * Ea, 64, TB));
  prm.bgroup = attn_group("NNT_ATTN_BGROUP", nblk);
  // NNT_ATTN_PBLK=1: one blocked request per P tile instead of two 4-D ones (measured neutral: the
  // kernel is DRAM-bound; off by default)
  const char* pb = getenv("NNT_ATTN_PBLK");
  if ((pb && pb[0] == '1') && make_tma_map_blocked(&mP, bf, 2, P, S, S, S, H, S * S, B, H * S * S, TB, TB / 64))
    prm.p_blk = 1;
  else
    NNT_TRY(make_tma_map_4d(&mP, bf, 2, P, S, S, S, H, S * S, B, H * S * S, 64, TB));
  NNT_TRY(make_tma_map_4d(&mdA, bf, 2, dA, S, S, S, H, S * S, B, H * S * S, 64, 32));
  NNT_TRY(make_tma_map_4d(&mdK, bf, 2, dq + Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, 32));
  NNT_TRY(make_tma_map_4d(&mdV, bf, 2, dq + 2 * Ea, Dh, S, 3 * Ea, H, Dh, B, S * 3 * Ea, 64, 32));
  // algorithmic bytes: P read once, dA written once, Q / V / dO read, dK / dV written
  const double ptiles = (double)B * H * (causal ? nblk * (nblk + 1) / 2 : nblk * nblk);
  LaunchScope sc(NNT_K_GEMM_TC_ATTN, stream, ptiles * TB * TB * 2 * 2 + 5.0 * B * S * Ea * 2,
                 ptiles * 6.0 * TB * TB * HD);
  NNT_CUDA_TRY(set_max_dyn_smem(attn_bwd_kv_kernel, B_SMEM));
  NNT_CUDA_TRY(::nnt::launch(attn_bwd_kv_kernel, dim3((unsigned)persistent_grid(prm.num_tasks)), dim3(kAThreads),
                             (size_t)B_SMEM, (cudaStream_t)stream, prm, mV, mdO, mQ, mP, mdA, mdK, mdV));
  return check_launch("attn_bwd_kv");
}

}  // extern "C"
