// Tensor-parallel SUM over peer memory ("tiles across the
// embedding dimension" on different GPUs; readings R31, R35).
//
// The partial-producing GEMM of a shard's stage (out-projection, projection, FC-dX, QKV-dX)
// writes each output row straight into the row's owner's receive slot (nnt_epilogue.scatter:
// the reduce-scatter's send, fused into the GEMM epilogue, over NVLink when the owner is a peer).
// The owner then sums the R slots of each of its rows in rank order and writes the sums into
// every rank's destination (the all-gather), also over peer memory.  Flags: rank q's words
// [0][w] = the epoch in which writer w's partials reached q's receive buffer, [1][o] = the epoch
// in which owner o's reduced rows reached q.  Stores to flags are release at system scope after
// a system fence; waits are acquire at system scope.
#include "nnt_internal.h"

namespace nnt {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct Comm {  // the ABI descriptor, by value (kernel parameter)
  int R, rank;
  int64_t rows, cols, rows_per;
  float* recv[NNT_TP_MAX];
  uint32_t* flags[NNT_TP_MAX];
  float* out[NNT_TP_MAX];
};

// which = 0: flags[o][0][rank] for every owner o; which = 1: flags[q][1][rank] for every rank q
__global__ void tp_signal_kernel(Comm c, uint32_t epoch, int which) {
  NNT_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  __threadfence_system();  // this rank's stores (the scattered partials / the gathered rows) first
  for (int q = 0; q < c.R; ++q) st_release_sys(c.flags[q] + which * NNT_TP_MAX + c.rank, epoch);
}

__global__ void tp_wait_kernel(Comm c, uint32_t epoch) {
  NNT_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  for (int o = 0; o < c.R; ++o)
    while (ld_acquire_sys(c.flags[c.rank] + NNT_TP_MAX + o) != epoch) __nanosleep(100);
  __threadfence_system();
}

// This rank's rows [rank*rows_per, ...): sum of the R slots in rank order -> every out[q].
__global__ void __launch_bounds__(kT) tp_reduce_gather_kernel(Comm c, uint32_t epoch) {
  NNT_PDL_ENTRY();
  if (threadIdx.x == 0) {
    for (int w = 0; w < c.R; ++w)
      while (ld_acquire_sys(c.flags[c.rank] + w) != epoch) __nanosleep(100);
  }
  __syncthreads();
  const int64_t r0 = (int64_t)c.rank * c.rows_per;
  const int64_t nr = c.rows - r0 < c.rows_per ? c.rows - r0 : c.rows_per;
  if (nr <= 0) return;
  const int64_t n4 = nr * c.cols / 4;  // cols % 4 == 0 (checked on the host)
  const float4* slot0 = reinterpret_cast<const float4*>(c.recv[c.rank]);
  const int64_t slot4 = c.rows_per * c.cols / 4;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kT) {
    float4 s = __ldcv(slot0 + i);  // writer 0's partial (written by other kernels / peers: volatile load)
    for (int w = 1; w < c.R; ++w) {
      const float4 t = __ldcv(slot0 + (int64_t)w * slot4 + i);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    for (int q = 0; q < c.R; ++q) reinterpret_cast<float4*>(c.out[q] + r0 * c.cols)[i] = s;
  }
}

nnt_status to_comm(const nnt_tp_comm* cm, Comm* c, const char* what) {
  NNT_REQUIRE(cm, NNT_ERR_NULL, "%s: NULL comm", what);
  NNT_REQUIRE(cm->R >= 1 && cm->R <= NNT_TP_MAX && cm->rank >= 0 && cm->rank < cm->R && cm->rows > 0 && cm->cols > 0,
              NNT_ERR_ARG, "%s: R=%d rank=%d rows=%lld cols=%lld", what, cm->R, cm->rank, (long long)cm->rows,
              (long long)cm->cols);
  NNT_REQUIRE(cm->cols % 4 == 0, NNT_ERR_ALIGN, "%s: cols %% 4", what);
  *c = Comm{};
  c->R = cm->R;
  c->rank = cm->rank;
  c->rows = cm->rows;
  c->cols = cm->cols;
  c->rows_per = (cm->rows + cm->R - 1) / cm->R;
  for (int q = 0; q < cm->R; ++q) {
    NNT_REQUIRE(cm->recv[q] && cm->flags[q], NNT_ERR_NULL, "%s: recv / flags of rank %d NULL", what, q);
    NNT_REQUIRE(aligned16(cm->recv[q]), NNT_ERR_ALIGN, "%s: recv[%d] 16-byte alignment", what, q);
    c->recv[q] = cm->recv[q];
    c->flags[q] = cm->flags[q];
  }
  return NNT_OK;
}

}  // namespace
}  // namespace nnt

using namespace nnt;

extern "C" {

nnt_status nnt_tp_signal(const nnt_tp_comm* comm, uint32_t epoch, int which, nnt_stream_t stream) {
  Comm c;
  NNT_TRY(to_comm(comm, &c, "nnt_tp_signal"));
  NNT_REQUIRE(epoch != 0 && (which == 0 || which == 1), NNT_ERR_ARG, "nnt_tp_signal: epoch %u which %d", epoch, which);
  LaunchScope sc(NNT_K_MISC, stream, 0, 0);
  NNT_CUDA_TRY(::nnt::launch(tp_signal_kernel, 1, 32, 0, (cudaStream_t)stream, c, epoch, which));
  return NNT_OK;
}

nnt_status nnt_tp_reduce_gather(const nnt_tp_comm* comm, float* const* out, uint32_t epoch, nnt_stream_t stream) {
  Comm c;
  NNT_TRY(to_comm(comm, &c, "nnt_tp_reduce_gather"));
  NNT_REQUIRE(epoch != 0 && out, NNT_ERR_ARG, "nnt_tp_reduce_gather: epoch 0 or NULL out");
  for (int q = 0; q < c.R; ++q) {
    NNT_REQUIRE(out[q] && aligned16(out[q]), NNT_ERR_ALIGN, "nnt_tp_reduce_gather: out[%d] NULL or unaligned", q);
    c.out[q] = out[q];
  }
  // algorithmic bytes: R slots of this rank's rows read, R copies of them written
  const double bytes = 8.0 * c.R * (double)c.rows_per * c.cols;
  LaunchScope sc(NNT_K_MISC, stream, bytes, (double)c.R * c.rows_per * c.cols);
  int64_t blocks = (c.rows_per * c.cols / 4 + kT - 1) / kT;
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  if (blocks < 1) blocks = 1;
  NNT_CUDA_TRY(::nnt::launch(tp_reduce_gather_kernel, (unsigned)blocks, kT, 0, (cudaStream_t)stream, c, epoch));
  return NNT_OK;
}

nnt_status nnt_tp_wait(const nnt_tp_comm* comm, uint32_t epoch, nnt_stream_t stream) {
  Comm c;
  NNT_TRY(to_comm(comm, &c, "nnt_tp_wait"));
  NNT_REQUIRE(epoch != 0, NNT_ERR_ARG, "nnt_tp_wait: epoch 0");
  LaunchScope sc(NNT_K_MISC, stream, 0, 0);
  NNT_CUDA_TRY(::nnt::launch(tp_wait_kernel, 1, 32, 0, (cudaStream_t)stream, c, epoch));
  return NNT_OK;
}

}  // extern "C"
