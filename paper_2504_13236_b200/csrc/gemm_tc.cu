// bf16 tensor-core GEMM for sm_100a: tcgen05.mma (kind::f16, fp32 accumulate in
// TMEM), operands staged by TMA (SWIZZLE_128B) through an mbarrier ring,
// warp-specialised persistent CTAs:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> bias / beta*C /
//               residual / GELU / GELU' -> swizzled smem staging -> TMA bulk
//               tensor store (coalesced, asynchronous); double-buffered TMEM
//               accumulators so the epilogue of tile i overlaps tile i+1's MMAs.
// Both operand majors are native (instruction-descriptor major bits + the
// canonical K-major / MN-major SW128 shared-memory layouts), so dX = dY W,
// dW = dY^T X and the six attention products run without transposes.  Batch
// items (b, head) are the two outer dimensions of 4-D TMA tensor maps.
//
// Split-K (small output grids with long K, i.e. the dW GEMMs): the K range of a
// tile is cut into `splits` contiguous pieces computed by different CTAs; their
// fp32 partial tiles are accumulated into C in ascending split order through a
// per-tile semaphore (split s waits until split s-1 has stored), so the sum
// has one fixed association and results are bitwise reproducible.  Split-K
// GEMMs on one device must not run concurrently (they share the semaphores);
// the block executor issues them on one stream.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm_common.cuh"

namespace nnt {

__device__ unsigned int g_tile_sem[65536];  // split-K semaphores (zero at load, reset by the last split)

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SW128 row
constexpr int kThreads = 192;
constexpr int kEpiWarps = 4;
constexpr int kStageBytesPerWarp = 4096;  // 32 rows x 128 B, SW128 staging for one TMA store box
constexpr int kMaxSemTiles = 65536;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_BYTES = kEpiWarps * 2 * kStageBytesPerWarp;  // C + aux staging per warp
  static constexpr int SMEM_BYTES = EPI_OFF + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcParams {
  GemmArgs g;
  int64_t mt, nt, tiles_per_batch, num_tiles, num_tasks;
  int64_t splits, kb_per_split;
  uint32_t idesc;
  int a_kmajor, b_kmajor;
  int tma_store;  // epilogue stores through TMA (C and aux maps valid)
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// SW128 shared-memory matrix descriptor (sm_100 "version 1" format).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Which tiles exist and which K-blocks each task covers (nnt_causal semantics + split-K).
struct TileInfo {
  int64_t tile, bz, m0, n0, kb_begin, kb_end, split;
  bool skip;
};
__device__ __forceinline__ TileInfo decode_task(const TcParams& P, int64_t t, int bn) {
  TileInfo ti;
  ti.split = t % P.splits;
  ti.tile = t / P.splits;
  ti.bz = ti.tile / P.tiles_per_batch;
  int64_t r = ti.tile % P.tiles_per_batch;
  int64_t nb = r / P.mt, mb = r % P.mt;
  ti.m0 = mb * BM;
  ti.n0 = nb * bn;
  int64_t k_begin = 0, k_end = P.g.K;
  if (P.g.causal == NNT_CAUSAL_A_LOWER) k_end = min(P.g.K, ti.m0 + BM);
  if (P.g.causal == NNT_CAUSAL_A_UPPER) k_begin = min(P.g.K, ti.m0);
  int64_t kb0 = k_begin / BK, kb1 = (k_end + BK - 1) / BK;
  ti.kb_begin = min(kb1, kb0 + ti.split * P.kb_per_split);
  ti.kb_end = min(kb1, ti.kb_begin + P.kb_per_split);
  ti.skip = (P.g.causal == NNT_CAUSAL_OUT_LOWER) && (ti.n0 > ti.m0 + BM - 1);
  return ti;
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

template <typename T>
__device__ __forceinline__ float ld_elem(const T* p) { return to_f32(*p); }
// C is re-read after other CTAs (split-K) or TMA stores wrote it: bypass L1.
__device__ __forceinline__ float ld_c(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float ld_c(const __nv_bfloat16* p) {
  unsigned short u = __ldcg(reinterpret_cast<const unsigned short*>(p));
  return __bfloat162float(__ushort_as_bfloat16(u));
}

// Computes the W outputs of one row chunk in registers.  pre-activation kept in `pre`.
template <typename TC, int W>
__device__ __forceinline__ void epi_math(const GemmArgs& g, const TC* Cb, const TC* auxb, int64_t row, int64_t col0,
                                         float beta, bool first, float (&v)[W], float (&pre)[W]) {
  constexpr bool kFast = sizeof(TC) == 2;
  const bool full = (row < g.M) && (col0 + W <= g.N);
#pragma unroll
  for (int j = 0; j < W; ++j) v[j] *= g.alpha;
  if (row < g.M) {
    if (first && g.bias) {
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] += __ldg(g.bias + col0 + j);
    }
    if (beta != 0.f) {
      const TC* cr = Cb + row * g.ldc + col0;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (full || col0 + j < g.N) v[j] += beta * ld_c(cr + j);
    }
    if (first && g.residual) {
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
  if (g.act == NNT_ACT_GELU) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
      pre[j] = v[j];
      v[j] = gelu_e<kFast>(v[j]);
    }
  }
}

// Writes a 128-byte row chunk to SW128-swizzled staging (row = lane, 8 x 16 B pieces).
template <typename TC, int W>
__device__ __forceinline__ void stage_row(uint8_t* buf, int lane, const float (&v)[W]) {
  uint8_t* rowp = buf + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint4 u;
    if (sizeof(TC) == 4) {
      u.x = __float_as_uint(v[4 * j]);
      u.y = __float_as_uint(v[4 * j + 1]);
      u.z = __float_as_uint(v[4 * j + 2]);
      u.w = __float_as_uint(v[4 * j + 3]);
    } else {
      __nv_bfloat162 t0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
      __nv_bfloat162 t1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
      __nv_bfloat162 t2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
      __nv_bfloat162 t3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
      u.x = *reinterpret_cast<uint32_t*>(&t0);
      u.y = *reinterpret_cast<uint32_t*>(&t1);
      u.z = *reinterpret_cast<uint32_t*>(&t2);
      u.w = *reinterpret_cast<uint32_t*>(&t3);
    }
    *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = u;
  }
}

template <typename TC, int W>
__device__ __forceinline__ void direct_store(const GemmArgs& g, TC* Cb, TC* auxb, int64_t row, int64_t col0,
                                             const float (&v)[W], const float (&pre)[W]) {
  if (row >= g.M) return;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if (col0 + j < g.N) {
      Cb[row * g.ldc + col0 + j] = from_f32<TC>(v[j]);
      if (g.act == NNT_ACT_GELU) auxb[row * g.ld_aux + col0 + j] = from_f32<TC>(pre[j]);
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int BN, typename TC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmAux) {
  using C = Cfg<BN>;
  constexpr int W = 128 / (int)sizeof(TC);  // columns per 128-byte staging row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::EPI_OFF + C::EPI_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GemmArgs& g = P.g;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < P.num_tasks; t += gridDim.x) {
        TileInfo ti = decode_task(P, t, BN);
        if (ti.skip) continue;
        const int p = (int)(ti.bz / g.batch1), q = (int)(ti.bz % g.batch1);
        for (int64_t kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_expect_tx(fb, C::STAGE_BYTES);
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
          const int k0 = (int)(kb * BK);
          if (P.a_kmajor) {
            tma_load_4d(sa, &tmA, fb, k0, (int)ti.m0, q, p);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_4d(sa + j * 8192, &tmA, fb, (int)ti.m0 + 64 * j, k0, q, p);
          }
          if (P.b_kmajor) {
            tma_load_4d(sb, &tmB, fb, k0, (int)ti.n0, q, p);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_4d(sb + j * 8192, &tmB, fb, (int)ti.n0 + 64 * j, k0, q, p);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart; +32 B per UMMA_K=16.
      // MN-major SW128: 64-element MN blocks LBO = 8 KB apart, 8-row K groups SBO = 1 KB
      // apart; +2 KB per UMMA_K=16.
      const uint32_t a_lbo = P.a_kmajor ? 16u : 8192u, b_lbo = P.b_kmajor ? 16u : 8192u;
      const uint32_t a_step = P.a_kmajor ? 32u : 2048u, b_step = P.b_kmajor ? 32u : 2048u;
      for (int64_t t = blockIdx.x; t < P.num_tasks; t += gridDim.x) {
        TileInfo ti = decode_task(P, t, BN);
        if (ti.skip) continue;
        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int64_t kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t ad = make_sdesc(sa + kk * a_step, a_lbo, 1024u);
            uint64_t bd = make_sdesc(sb + kk * b_step, b_lbo, 1024u);
            mma_bf16(tmem_d, ad, bd, P.idesc, (kb > ti.kb_begin || kk > 0) ? 1u : 0u);
          }
          mma_commit(smem_u32(&empty[stage]));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(smem_u32(&tfull[acc]));
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5 -> TMEM lane quadrants 2,3,0,1)
    const int quad = warp & 3;
    uint8_t* stage_c = smem + C::EPI_OFF + quad * 2 * kStageBytesPerWarp;
    uint8_t* stage_a = stage_c + kStageBytesPerWarp;
    const uint32_t stage_c_u32 = smem_u32(stage_c), stage_a_u32 = smem_u32(stage_a);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < P.num_tasks; t += gridDim.x) {
      TileInfo ti = decode_task(P, t, BN);
      if (ti.skip) continue;
      const int64_t p = ti.bz / g.batch1, q = ti.bz % g.batch1;
      TC* Cb = (TC*)g.C + p * g.sc0 + q * g.sc1;
      TC* auxb = g.aux ? (TC*)g.aux + p * g.sc0 + q * g.sc1 : nullptr;
      const bool first = ti.split == 0;
      const float beta = first ? g.beta : 1.0f;  // later splits accumulate onto the stored partial sum
      if (P.splits > 1 && !first) {
        // ordered split-K: wait until split (s-1) of this tile has stored its partial sum
        if (warp == 2 && lane == 0) {
          const unsigned int want = (unsigned int)ti.split;
          unsigned int cur;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&g_tile_sem[ti.tile]) : "memory");
          } while (cur != want);
        }
        epi_bar();
      }
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const int64_t row = ti.m0 + quad * 32 + lane;
      const bool has_k = ti.kb_end > ti.kb_begin;
#pragma unroll 1
      for (int c = 0; c < BN; c += W) {
        if (ti.n0 + c >= g.N) break;  // warp-uniform
        float v[W], pre[W];
#pragma unroll
        for (int h = 0; h < W / 32; ++h) {
          if (has_k) {
            tmem_ld32(tmem_base + (uint32_t)(acc * BN + c + 32 * h) + ((uint32_t)(quad * 32) << 16), v + 32 * h);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[32 * h + j] = 0.f;
          }
        }
        epi_math<TC, W>(g, Cb, auxb, row, ti.n0 + c, beta, first, v, pre);
        if (P.tma_store) {
          if (lane == 0) bulk_wait_read0();  // staging buffers free again
          __syncwarp();
          stage_row<TC, W>(stage_c, lane, v);
          if (g.act == NNT_ACT_GELU) stage_row<TC, W>(stage_a, lane, pre);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int cx = (int)(ti.n0 + c), cy = (int)(ti.m0 + quad * 32);
            tma_store_4d(&tmC, stage_c_u32, cx, cy, (int)q, (int)p);
            if (g.act == NNT_ACT_GELU) tma_store_4d(&tmAux, stage_a_u32, cx, cy, (int)q, (int)p);
            bulk_commit();
          }
        } else {
          direct_store<TC, W>(g, Cb, auxb, row, ti.n0 + c, v, pre);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (P.splits > 1) {
        // publish: this split's sum is in C (stores complete and visible), then signal split s+1
        if (lane == 0 && P.tma_store) bulk_wait0();
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        epi_bar();
        if (warp == 2 && lane == 0) {
          const unsigned int next = (ti.split + 1 == P.splits) ? 0u : (unsigned int)(ti.split + 1);
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&g_tile_sem[ti.tile]), "r"(next) : "memory");
        }
      }
    }
    if (lane == 0 && P.tma_store) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)C::TMEM_COLS)
                 : "memory");
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

// Split-K factor: only for fp32 C without activation (the dW GEMMs) whose output grid
// leaves most SMs idle and whose K is long enough to cut.
int64_t choose_splits(const GemmArgs& a, int64_t tiles, int64_t nkb) {
  if (a.c_dtype != NNT_F32 || a.act != NNT_ACT_NONE || a.causal != NNT_CAUSAL_NONE || a.batch0 * a.batch1 != 1)
    return 1;
  const int64_t sms = num_sms();
  if (tiles * 2 > sms || tiles > kMaxSemTiles) return 1;
  int64_t s = sms / tiles;
  if (s > nkb / 8) s = nkb / 8;  // keep >= 8 K-blocks per split
  if (s > 16) s = 16;
  return s < 1 ? 1 : s;
}

template <int BN, typename TC>
nnt_status launch_bn(const GemmArgs& a, cudaStream_t s) {
  using C = Cfg<BN>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_tc_kernel<BN, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    C::SMEM_BYTES);
  });
  NNT_REQUIRE(attr_err == cudaSuccess, NNT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
  NNT_TRY(get_encoder());
  TcParams P;
  P.g = a;
  P.a_kmajor = a.ta == NNT_NOTRANS;
  P.b_kmajor = a.tb == NNT_TRANS;
  P.mt = (a.M + BM - 1) / BM;
  P.nt = (a.N + BN - 1) / BN;
  P.tiles_per_batch = P.mt * P.nt;
  P.num_tiles = P.tiles_per_batch * a.batch0 * a.batch1;
  const int64_t nkb = (a.K + BK - 1) / BK;
  P.splits = choose_splits(a, P.num_tiles, nkb);
  P.kb_per_split = (nkb + P.splits - 1) / P.splits;
  P.splits = (nkb + P.kb_per_split - 1) / P.kb_per_split;  // no empty splits
  P.num_tasks = P.num_tiles * P.splits;
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((P.a_kmajor ? 0u : 1u) << 15) | ((P.b_kmajor ? 0u : 1u) << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  CUtensorMap tmA, tmB, tmC, tmAux;
  const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (P.a_kmajor)
    NNT_TRY(make_map(&tmA, bf, 2, a.A, a.K, a.M, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, BK, BM));
  else
    NNT_TRY(make_map(&tmA, bf, 2, a.A, a.M, a.K, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, 64, BK));
  if (P.b_kmajor)
    NNT_TRY(make_map(&tmB, bf, 2, a.B, a.K, a.N, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, BK, BN));
  else
    NNT_TRY(make_map(&tmB, bf, 2, a.B, a.N, a.K, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, 64, BK));
  // epilogue through TMA stores when C (and aux) satisfy the tensor-map rules
  const size_t es = sizeof(TC);
  const CUtensorMapDataType cdt = sizeof(TC) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : bf;
  const int W = (int)(128 / es);
  auto ok16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool tma_ok = ok16(a.C) && (a.ldc * es) % 16 == 0 && (a.batch1 <= 1 || (a.sc1 > 0 && (a.sc1 * es) % 16 == 0)) &&
                (a.batch0 <= 1 || (a.sc0 > 0 && (a.sc0 * es) % 16 == 0)) &&
                (a.act != NNT_ACT_GELU || (ok16(a.aux) && (a.ld_aux * es) % 16 == 0));
  P.tma_store = tma_ok ? 1 : 0;
  memset(&tmC, 0, sizeof(tmC));
  memset(&tmAux, 0, sizeof(tmAux));
  if (tma_ok) {
    NNT_TRY(make_map(&tmC, cdt, es, a.C, a.N, a.M, a.ldc, a.batch1, a.sc1, a.batch0, a.sc0, W, 32));
    if (a.act == NNT_ACT_GELU)
      NNT_TRY(make_map(&tmAux, cdt, es, a.aux, a.N, a.M, a.ld_aux, a.batch1, a.sc1, a.batch0, a.sc0, W, 32));
  }
  int64_t grid = P.num_tasks < num_sms() ? P.num_tasks : num_sms();
  if (grid < 1) grid = 1;
  gemm_tc_kernel<BN, TC><<<(unsigned)grid, kThreads, C::SMEM_BYTES, s>>>(P, tmA, tmB, tmC, tmAux);
  return check_launch("gemm_tc");
}

template <typename TC>
nnt_status launch_tc(const GemmArgs& a, cudaStream_t s) {
  if (a.N <= 64) return launch_bn<64, TC>(a, s);
  if (a.N <= 128 || a.causal == NNT_CAUSAL_OUT_LOWER) return launch_bn<128, TC>(a, s);
  return launch_bn<256, TC>(a, s);
}

}  // namespace

nnt_status gemm_tc_launch(const GemmArgs& a, cudaStream_t s) {
  // TMA: 16-byte aligned base, 16-byte multiple strides (bf16: multiples of 8 elements).
  NNT_REQUIRE(aligned16(a.A) && aligned16(a.B), NNT_ERR_ALIGN, "gemm(bf16): A/B must be 16-byte aligned");
  NNT_REQUIRE(a.lda % 8 == 0 && a.ldb % 8 == 0, NNT_ERR_ALIGN, "gemm(bf16): lda/ldb must be multiples of 8");
  NNT_REQUIRE((a.batch1 <= 1 || (a.sa1 % 8 == 0 && a.sb1 % 8 == 0 && a.sa1 > 0 && a.sb1 > 0)) &&
                  (a.batch0 <= 1 || (a.sa0 % 8 == 0 && a.sb0 % 8 == 0 && a.sa0 > 0 && a.sb0 > 0)),
              NNT_ERR_ALIGN, "gemm(bf16): batch strides must be positive multiples of 8");
  NNT_REQUIRE(a.M < (1ll << 31) && a.N < (1ll << 31) && a.K < (1ll << 31), NNT_ERR_UNSUPPORTED,
              "gemm(bf16): dims must fit int32 TMA coordinates");
  if (a.c_dtype == NNT_F32) return launch_tc<float>(a, s);
  return launch_tc<__nv_bfloat16>(a, s);
}

}  // namespace nnt
