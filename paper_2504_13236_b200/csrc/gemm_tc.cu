// bf16 tensor-core GEMM for sm_100a: tcgen05.mma (kind::f16, fp32 accumulate in
// TMEM), operands staged by TMA (SWIZZLE_128B) through an mbarrier ring,
// warp-specialised persistent CTAs:
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> bias / residual /
//               GELU / GELU' -> global, double-buffered accumulators so the
//               epilogue of tile i overlaps the MMAs of tile i+1.
// Both operand majors are supported natively (instruction-descriptor major
// bits + the canonical K-major / MN-major SW128 shared-memory layouts), so
// dX = dY W, dW = dY^T X and all six attention products run without transposes.
// Batch items (b, head) are the two outer dimensions of 4-D TMA tensor maps.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm_common.cuh"

namespace nnt {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SW128 row
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcParams {
  GemmArgs g;
  int64_t mt, nt, tiles_per_batch, num_tiles;
  uint32_t idesc;
  int a_kmajor, b_kmajor;
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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
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

// Which tiles exist and which K range each covers (nnt_causal semantics).
struct TileInfo {
  int64_t bz, m0, n0, kb_begin, kb_end;
  bool skip;
};
__device__ __forceinline__ TileInfo decode_tile(const TcParams& P, int64_t t, int bn) {
  TileInfo ti;
  ti.bz = t / P.tiles_per_batch;
  int64_t r = t % P.tiles_per_batch;
  int64_t nb = r / P.mt, mb = r % P.mt;
  ti.m0 = mb * BM;
  ti.n0 = nb * bn;
  int64_t k_begin = 0, k_end = P.g.K;
  if (P.g.causal == NNT_CAUSAL_A_LOWER) k_end = min(P.g.K, ti.m0 + BM);
  if (P.g.causal == NNT_CAUSAL_A_UPPER) k_begin = min(P.g.K, ti.m0);
  ti.kb_begin = k_begin / BK;
  ti.kb_end = (k_end + BK - 1) / BK;
  ti.skip = (P.g.causal == NNT_CAUSAL_OUT_LOWER) && (ti.n0 > ti.m0 + BM - 1);
  return ti;
}

// ------------------------------------------------------------------ epilogue
template <typename TC>
__device__ __forceinline__ void store32(TC* dst, const float (&v)[32]);
template <>
__device__ __forceinline__ void store32<float>(float* dst, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
}
template <>
__device__ __forceinline__ void store32<__nv_bfloat16>(__nv_bfloat16* dst, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    uint4 u;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(v[j], v[j + 1]), t1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]), t3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
    u.x = *reinterpret_cast<uint32_t*>(&t0);
    u.y = *reinterpret_cast<uint32_t*>(&t1);
    u.z = *reinterpret_cast<uint32_t*>(&t2);
    u.w = *reinterpret_cast<uint32_t*>(&t3);
    *reinterpret_cast<uint4*>(dst + j) = u;
  }
}
template <typename TC>
__device__ __forceinline__ void load32(const TC* src, float (&v)[32]);
template <>
__device__ __forceinline__ void load32<float>(const float* src, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 4) {
    float4 t = *reinterpret_cast<const float4*>(src + j);
    v[j] = t.x; v[j + 1] = t.y; v[j + 2] = t.z; v[j + 3] = t.w;
  }
}
template <>
__device__ __forceinline__ void load32<__nv_bfloat16>(const __nv_bfloat16* src, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    uint4 u = *reinterpret_cast<const uint4*>(src + j);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float2 f = __bfloat1622float2(h[t]);
      v[j + 2 * t] = f.x;
      v[j + 2 * t + 1] = f.y;
    }
  }
}

template <typename TC>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& g, TC* Cb, TC* auxb, int64_t row, int64_t col0,
                                               const uint32_t (&r)[32], bool vec_ok) {
  if (row >= g.M) return;
  if (vec_ok && col0 + 32 <= g.N) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = g.alpha * __uint_as_float(r[j]);
    if (g.bias) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 b = __ldg(reinterpret_cast<const float4*>(g.bias + col0 + j));
        v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
      }
    }
    if (g.beta != 0.f) {
      float o[32];
      load32<TC>(Cb + row * g.ldc + col0, o);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += g.beta * o[j];
    }
    if (g.residual) {
      float o[32];
      load32<float>(g.residual + row * g.ld_res + col0, o);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += o[j];
    }
    if (g.act == NNT_ACT_GELU) {
      store32<TC>(auxb + row * g.ld_aux + col0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
    } else if (g.act == NNT_ACT_GELU_BWD) {
      float u[32];
      load32<TC>(auxb + row * g.ld_aux + col0, u);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(u[j]);
    }
    store32<TC>(Cb + row * g.ldc + col0, v);
  } else {
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {
      int64_t col = col0 + j;
      if (col < g.N) epilogue_store<TC>(g, Cb, auxb, row, col, __uint_as_float(r[j]));
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int BN, typename TC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
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
      mbar_init(smem_u32(&tempty[s]), 4);
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
      for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
        TileInfo ti = decode_tile(P, t, BN);
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
      for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
        TileInfo ti = decode_tile(P, t, BN);
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
    int acc = 0;
    uint32_t acc_phase = 0;
    const size_t cs = sizeof(TC);
    const bool vec_ok = ((g.ldc * cs) % 16 == 0) && ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0) &&
                        (!g.residual || (g.ld_res % 4 == 0 && (reinterpret_cast<uintptr_t>(g.residual) & 15) == 0)) &&
                        (!g.aux || ((g.ld_aux * cs) % 16 == 0 && (reinterpret_cast<uintptr_t>(g.aux) & 15) == 0)) &&
                        (!g.bias || (reinterpret_cast<uintptr_t>(g.bias) & 15) == 0) &&
                        ((g.sc0 * cs) % 16 == 0) && ((g.sc1 * cs) % 16 == 0);
    for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
      TileInfo ti = decode_tile(P, t, BN);
      if (ti.skip) continue;
      const int64_t p = ti.bz / g.batch1, q = ti.bz % g.batch1;
      TC* Cb = (TC*)g.C + p * g.sc0 + q * g.sc1;
      TC* auxb = g.aux ? (TC*)g.aux + p * g.sc0 + q * g.sc1 : nullptr;
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const int64_t row = ti.m0 + quad * 32 + lane;
      const bool has_k = ti.kb_end > ti.kb_begin;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        if (has_k) {
          tmem_ld32(tmem_base + (uint32_t)(acc * BN + c) + ((uint32_t)(quad * 32) << 16), r);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        if (ti.n0 + c < g.N) epilogue_chunk<TC>(g, Cb, auxb, row, ti.n0 + c, r, vec_ok);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
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

// 4-D bf16 tensor map: dims {inner, outer, batch1, batch0}.
nnt_status make_map(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int64_t ld, int64_t b1,
                    int64_t s1, int64_t b0, int64_t s0, int box_inner, int box_outer) {
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)b1, (cuuint64_t)b0};
  // size-1 batch dims get a harmless valid stride
  int64_t st1 = b1 > 1 ? s1 : ld * outer;
  int64_t st0 = b0 > 1 ? s0 : st1 * b1;
  cuuint64_t strides[3] = {(cuuint64_t)(ld * 2), (cuuint64_t)(st1 * 2), (cuuint64_t)(st0 * 2)};
  cuuint32_t box[4] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  NNT_REQUIRE(r == CUDA_SUCCESS, NNT_ERR_CUDA,
              "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld s1=%lld s0=%lld", (int)r,
              (long long)inner, (long long)outer, (long long)ld, (long long)s1, (long long)s0);
  return NNT_OK;
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
  P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((P.a_kmajor ? 0u : 1u) << 15) | ((P.b_kmajor ? 0u : 1u) << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  CUtensorMap tmA, tmB;
  if (P.a_kmajor)
    NNT_TRY(make_map(&tmA, a.A, a.K, a.M, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, BK, BM));
  else
    NNT_TRY(make_map(&tmA, a.A, a.M, a.K, a.lda, a.batch1, a.sa1, a.batch0, a.sa0, 64, BK));
  if (P.b_kmajor)
    NNT_TRY(make_map(&tmB, a.B, a.K, a.N, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, BK, BN));
  else
    NNT_TRY(make_map(&tmB, a.B, a.N, a.K, a.ldb, a.batch1, a.sb1, a.batch0, a.sb0, 64, BK));
  int64_t grid = P.num_tiles < num_sms() ? P.num_tiles : num_sms();
  if (grid < 1) grid = 1;
  gemm_tc_kernel<BN, TC><<<(unsigned)grid, kThreads, C::SMEM_BYTES, s>>>(P, tmA, tmB);
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
