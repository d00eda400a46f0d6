// Library plumbing: errors, version/device checks, tile bookkeeping (P:72-75,
// P:231) and the per-launch CUDA-event timer used by bench.py's roofline.
#include <cstdlib>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "nnt_internal.h"

namespace nnt {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t set_max_dyn_smem(const void* fn, int bytes) {
  // cudaFuncSetAttribute acts on the current device's context: cache per (function, device)
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(fn, dev, bytes);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    // on by default since the early trigger moved to the GEMM's last operand load (interleaved
    // A/B: 11.71 -> 11.64 ms/step); NNT_PDL=0 launches without the attribute
    const char* e = getenv("NNT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ---------------------------------------------------------------- timing
namespace {
struct TimingRecord {
  int kclass;
  cudaEvent_t start, stop;
  double bytes, flops;
  int kernels;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<TimingRecord> g_records;
std::vector<cudaEvent_t> g_event_pool;
std::atomic<int64_t> g_launches{0};

// Inside a stream capture a plain cudaEventRecord only expresses a dependency; an
// external record makes it an event-record node that timestamps every graph replay.
void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

LaunchScope::LaunchScope(int kclass, cudaStream_t s, double bytes, double flops, int kernels)
    : kclass_(kclass), s_(s), slot_(-1) {
  g_launches.fetch_add(kernels, std::memory_order_relaxed);
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  TimingRecord r{kclass, take_event(), take_event(), bytes, flops, kernels};
  record(r.start, s);
  slot_ = (int)g_records.size();
  g_records.push_back(r);
}

void LaunchScope::add_kernels(int k) {
  g_launches.fetch_add(k, std::memory_order_relaxed);
  if (slot_ < 0) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  g_records[slot_].kernels += k;
}

LaunchScope::~LaunchScope() {
  if (slot_ < 0) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  record(g_records[slot_].stop, s_);
}

}  // namespace nnt

using namespace nnt;

extern "C" {

int nnt_abi_version(void) { return NNT_ABI_VERSION; }

const char* nnt_last_error(void) { return g_last_error; }

nnt_status nnt_device_check(int device) {
  int major = 0, minor = 0;
  NNT_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  NNT_CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  NNT_REQUIRE(major == 10 && minor == 0, NNT_ERR_UNSUPPORTED,
              "device %d is sm_%d%d; libnnt carries sm_100a SASS only", device, major, minor);
  return NNT_OK;
}

nnt_status nnt_tile_grid(int ndim, const int64_t* shape, const int64_t* tile, int64_t* grid) {
  NNT_REQUIRE(shape && tile && grid, NNT_ERR_NULL, "nnt_tile_grid: NULL argument");
  NNT_REQUIRE(ndim > 0, NNT_ERR_SHAPE, "nnt_tile_grid: ndim=%d", ndim);
  for (int d = 0; d < ndim; ++d) {
    NNT_REQUIRE(shape[d] > 0, NNT_ERR_SHAPE, "nnt_tile_grid: shape[%d]=%lld", d, (long long)shape[d]);
    NNT_REQUIRE(tile[d] > 0, NNT_ERR_TILE, "nnt_tile_grid: tile[%d]=%lld", d, (long long)tile[d]);
  }
  for (int d = 0; d < ndim; ++d) {
    int64_t t = tile[d] < shape[d] ? tile[d] : shape[d];
    grid[d] = (shape[d] + t - 1) / t;
  }
  return NNT_OK;
}

nnt_status nnt_tile_extent(int64_t dim, int64_t tile, int64_t idx, int64_t* offset, int64_t* extent) {
  NNT_REQUIRE(offset && extent, NNT_ERR_NULL, "nnt_tile_extent: NULL argument");
  NNT_REQUIRE(dim > 0, NNT_ERR_SHAPE, "nnt_tile_extent: dim=%lld", (long long)dim);
  NNT_REQUIRE(tile > 0, NNT_ERR_TILE, "nnt_tile_extent: tile=%lld", (long long)tile);
  int64_t t = tile < dim ? tile : dim;
  int64_t n = (dim + t - 1) / t;
  NNT_REQUIRE(idx >= 0 && idx < n, NNT_ERR_ARG, "nnt_tile_extent: idx %lld outside grid %lld",
              (long long)idx, (long long)n);
  *offset = idx * t;
  *extent = (dim - idx * t) < t ? (dim - idx * t) : t;
  return NNT_OK;
}

nnt_status nnt_partition(int64_t n_units, int n_ranks, int rank, int64_t* begin, int64_t* end) {
  NNT_REQUIRE(begin && end, NNT_ERR_NULL, "nnt_partition: NULL argument");
  NNT_REQUIRE(n_units >= 0 && n_ranks > 0, NNT_ERR_SHAPE, "nnt_partition: n=%lld R=%d",
              (long long)n_units, n_ranks);
  NNT_REQUIRE(rank >= 0 && rank < n_ranks, NNT_ERR_ARG, "nnt_partition: rank %d of %d", rank, n_ranks);
  *begin = ((int64_t)rank * n_units) / n_ranks;
  *end = ((int64_t)(rank + 1) * n_units) / n_ranks;
  return NNT_OK;
}

nnt_status nnt_timing_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto& r : g_records) {
    g_event_pool.push_back(r.start);
    g_event_pool.push_back(r.stop);
  }
  g_records.clear();
  g_timing = enable != 0;
  return NNT_OK;
}

nnt_status nnt_timing_read(double* ms, int64_t* launches, double* bytes, double* flops) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (int k = 0; k < NNT_K_COUNT; ++k) {
    if (ms) ms[k] = 0;
    if (launches) launches[k] = 0;
    if (bytes) bytes[k] = 0;
    if (flops) flops[k] = 0;
  }
  for (auto& r : g_records) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.stop);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.start, r.stop);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();  // do not leave it for the next launch check
      set_error("nnt_timing_read: %s", cudaGetErrorString(e));
      return NNT_ERR_CUDA;
    }
    if (ms) ms[r.kclass] += t;
    if (launches) launches[r.kclass] += 1;
    if (bytes) bytes[r.kclass] += r.bytes;
    if (flops) flops[r.kclass] += r.flops;
  }
  return NNT_OK;
}

nnt_status nnt_timing_trace(int32_t* kclass, int32_t* kernels, int64_t cap, int64_t* n) {
  NNT_REQUIRE(n, NNT_ERR_NULL, "nnt_timing_trace: NULL count");
  NNT_REQUIRE(cap >= 0 && (cap == 0 || (kclass && kernels)), NNT_ERR_NULL, "nnt_timing_trace: NULL arrays");
  std::lock_guard<std::mutex> lk(g_tmu);
  *n = (int64_t)g_records.size();
  for (int64_t i = 0; i < cap && i < *n; ++i) {
    kclass[i] = g_records[i].kclass;
    kernels[i] = g_records[i].kernels;
  }
  return NNT_OK;
}

int64_t nnt_launch_count(void) { return g_launches.load(); }

}  // extern "C"
