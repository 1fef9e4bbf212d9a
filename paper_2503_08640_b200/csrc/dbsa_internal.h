// dbsa_internal.h -- host-side helpers shared by the C-ABI translation units:
// thread-local error reporting and the cuTensorMapEncodeTiled driver entry.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

namespace dbsa {

// Record a formatted error message for dbsa_last_error() and return `code`.
int set_error(int code, const char *fmt, ...);

// cuTensorMapEncodeTiled for a bf16 tensor (resolved through
// cudaGetDriverEntryPoint, so the library does not link libcuda directly).
bool encode_tiled_bf16(CUtensorMap *map, const void *base, int rank, const cuuint64_t *dims,
                       const cuuint64_t *strides_bytes, const cuuint32_t *box, const cuuint32_t *elem_strides,
                       CUtensorMapSwizzle swizzle);

inline int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(6, "%s: %s", what, cudaGetErrorString(e));
  return 0;
}

// Programmatic dependent launch (PDL).  A kernel launched with pdl = true may
// start while its stream predecessor is still running; it must execute
// pdl_wait() before touching anything the predecessor writes (and every CTA
// waits before it exits, so completion stays transitive along the stream).
// pdl_trigger() in a predecessor lets its dependents launch before it exits.
// Without the launch attribute pdl_wait() returns at once.  DBSA_PDL=0 turns
// the attribute off (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("DBSA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// L2 residency for small, repeatedly re-read activations (the residual stream
// of a batch-1 forward): a launch may mark one buffer persisting, so the
// per-layer weight streams (hundreds of MB) do not evict it between layers.
// The device's persisting carve-out is set once (DBSA_L2_PERSIST_MB, default 16;
// 0 disables).
constexpr size_t kPersistMaxBytes = 8u << 20;     // activations kept resident (the residual stream)
constexpr size_t kWindowMaxBytes = 128u << 20;     // cudaDevAttrMaxAccessPolicyWindowSize on B200
inline bool l2_persist_ready(cudaStream_t s) {
  // set once, outside any stream capture (a device-wide call there could
  // invalidate the capture); until then launches go without the window
  static std::atomic<int> state{0};  // 0 not yet, 1 set, -1 off / failed
  if (state.load() == 0) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return false;
    const char *e = getenv("DBSA_L2_PERSIST_MB");
    const size_t mb = e ? (size_t)atoi(e) : 16;
    const bool ok = mb && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, mb << 20) == cudaSuccess;
    if (!ok) cudaGetLastError();  // clear a failed call's error
    state.store(ok ? 1 : -1);
  }
  return state.load() > 0;
}

struct Persist {
  const void *base = nullptr;
  size_t bytes = 0;
};

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kp(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                             Persist keep, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl && pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (keep.base && keep.bytes && keep.bytes <= kWindowMaxBytes && l2_persist_ready(s)) {
    at[n].id = cudaLaunchAttributeAccessPolicyWindow;
    at[n].val.accessPolicyWindow.base_ptr = const_cast<void *>(keep.base);
    at[n].val.accessPolicyWindow.num_bytes = keep.bytes;
    at[n].val.accessPolicyWindow.hitRatio = 1.f;
    at[n].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[n].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++n;
  }
  cfg.attrs = n ? at : nullptr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args &&...args) {
  return launch_kp(kern, grid, block, smem, s, pdl, Persist{}, std::forward<Args>(args)...);
}

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

}  // namespace dbsa
