// Internal helpers shared by the libnnt translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/nnt.h"

namespace nnt {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
inline nnt_status fail(nnt_status s, const char* msg) {
  set_error("%s", msg);
  return s;
}

#define NNT_REQUIRE(cond, status, ...)      \
  do {                                      \
    if (!(cond)) {                          \
      ::nnt::set_error(__VA_ARGS__);        \
      return (status);                      \
    }                                       \
  } while (0)

#define NNT_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::nnt::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                       __FILE__, __LINE__);                                       \
      return NNT_ERR_CUDA;                                                        \
    }                                                                             \
  } while (0)

#define NNT_TRY(expr)                 \
  do {                                \
    nnt_status _s = (expr);           \
    if (_s != NNT_OK) return _s;      \
  } while (0)

// Checks the launch that was just enqueued.
inline nnt_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("launch of %s failed: %s", what, cudaGetErrorString(e));
    return NNT_ERR_CUDA;
  }
  return NNT_OK;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t dtype_size(int dt) { return dt == NNT_BF16 ? 2 : 4; }
inline bool valid_dtype(int dt) { return dt == NNT_F32 || dt == NNT_BF16; }

// ---------------------------------------------------------------- timing
// RAII scope recording CUDA events around one launch when timing is enabled.
struct LaunchScope {
  LaunchScope(int kclass, cudaStream_t s, double bytes, double flops, int kernels = 1);
  ~LaunchScope();
  void add_kernels(int k);  // the scope launched k more kernels than declared (decided inside)
  int kclass_;
  cudaStream_t s_;
  int slot_;
};

int num_sms();

// Per-process state is kept per device where CUDA ties it to one (events, function attributes):
// one process may drive several GPUs.
constexpr int kMaxDevices = 64;
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, bytes).
cudaError_t set_max_dyn_smem(const void* fn, int bytes);
template <typename F>
inline cudaError_t set_max_dyn_smem(F* fn, int bytes) {
  return set_max_dyn_smem(reinterpret_cast<const void*>(fn), bytes);
}

// ---------------------------------------------------------------- launches
// Every libnnt kernel is launched with programmatic dependent launch (PDL) allowed: the next
// kernel on the stream may be scheduled while this one drains, its CTAs run their prologue
// (smem carve-up, barrier init, TMEM allocation) and then block in griddepcontrol.wait until
// the previous grid has completed and its writes are visible (NNT_PDL_ENTRY at the top of
// every kernel).  Inside a CUDA graph this becomes a programmatic edge, hiding the per-kernel
// launch gap of the ~430-launch training step.  On by default; NNT_PDL=0 disables it.
bool pdl_enabled();

#if defined(__CUDACC__)
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

#if defined(__CUDACC__)
// ---------------------------------------------------------------- PDL (see launch())
// Wait until the previous grid on the stream has completed (its memory visible), then allow
// the next grid to be scheduled.  A no-op when the kernel was launched without PDL.
// The early trigger is issued only where a kernel knows its remaining work is a tail (the
// persistent GEMM once its last operand load is issued, pdl_trigger); elsewhere the dependents
// are released as the CTAs exit.  (Triggering at every kernel's entry let dependent CTAs take
// SM slots from the still-running grid: measured slower.)
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define NNT_PDL_ENTRY() ::nnt::pdl_entry()

// ---------------------------------------------------------------- device math
__device__ __forceinline__ float bf16_to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f32_to_bf16(float v) { return __float2bfloat16_rn(v); }

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// GELU tanh form (R11).  tanhf (not tanh.approx) keeps the fp32 path within 1e-6.
__device__ __forceinline__ float gelu_f(float u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  return 0.5f * u * (1.0f + tanhf(c * (u + a * u * u * u)));
}
__device__ __forceinline__ float gelu_grad_f(float u) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float t = tanhf(c * (u + a * u * u * u));
  return 0.5f * (1.0f + t) + 0.5f * u * (1.0f - t * t) * c * (1.0f + 3.0f * a * u * u);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

#endif  // __CUDACC__

}  // namespace nnt
