// dbsa_internal.h -- host-side helpers shared by the C-ABI translation units:
// thread-local error reporting and the cuTensorMapEncodeTiled driver entry.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

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

}  // namespace dbsa
