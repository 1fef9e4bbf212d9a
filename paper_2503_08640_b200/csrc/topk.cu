// topk.cu -- K4: anchor-first top-k group selection + ordering, bit-exact with
// retrieval.select (retrieval.py:352-374) and retrieval.order (retrieval.py:377-388).
//
// select: picked = [0] + sorted(1..n-1, key=(-score, id))[:budget-1].
// Under that total order a candidate's rank is the number of candidates that
// precede it, so selection and the output permutation are both computed by
// counting comparisons -- no floating-point arithmetic, only f64 compares, so
// the result is identical to Python's sort.  One CTA per query; the score row
// is staged in shared memory and each warp counts with ballot/popc.
#include <cuda_runtime.h>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"

namespace dbsa {

__device__ __forceinline__ bool before_desc(double sa, int a, double sb, int b) {
  // (-sa, a) < (-sb, b)
  return sa > sb || (sa == sb && a < b);
}

__global__ void topk_kernel(const double *scores, int64_t n_units, int64_t budget, int ordering, int32_t *out) {
  extern __shared__ double sh[];
  double *s = sh;                                               // [n_units]
  int32_t *sel = reinterpret_cast<int32_t *>(s + n_units);      // [budget-1]
  const int64_t q = blockIdx.x;
  const double *row = scores + q * n_units;
  for (int64_t u = threadIdx.x; u < n_units; u += blockDim.x) s[u] = row[u];
  __syncthreads();
  const int k = (int)budget - 1;
  const int lane = threadIdx.x & 31;
  // rank every candidate u in 1..n-1; a warp handles 32 candidates at a time
  for (int64_t base = 1 + (threadIdx.x & ~31); base < n_units; base += blockDim.x) {
    const int64_t u = base + lane;
    const bool active = u < n_units;
    const double su = active ? s[u] : 0.0;
    int rank = 0;
    for (int64_t v0 = 1; v0 < n_units; v0 += 32) {
      const int64_t v = v0 + lane;
      const double sv = v < n_units ? s[v] : 0.0;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const double svj = __shfl_sync(0xffffffffu, sv, j);
        const int64_t vj = v0 + j;
        if (active && vj < n_units && before_desc(svj, (int)vj, su, (int)u)) ++rank;
      }
    }
    if (active && rank < k) sel[rank] = (int32_t)u;
  }
  __syncthreads();
  int32_t *o = out + q * budget;
  if (threadIdx.x == 0) o[0] = 0;
  // order the picked units (anchor pinned first)
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int id = sel[i];
    const double si = s[id];
    int pos = 0;
    for (int j = 0; j < k; ++j) {
      const int jd = sel[j];
      bool b;
      if (ordering == 0) b = jd < id;                                  // in-order: ascending id
      else if (ordering == 1) b = s[jd] < si || (s[jd] == si && jd < id);  // low-to-high: (score, id)
      else b = jd > id;                                                // reverse: descending id
      pos += b;
    }
    o[1 + pos] = id;
  }
}

}  // namespace dbsa

extern "C" int dbsa_topk_select(const double *scores, int64_t n_queries, int64_t n_units, int64_t budget,
                                int32_t ordering, int32_t *out_ids, void *stream) {
  using namespace dbsa;
  if (n_queries < 0 || n_units < 1) return set_error(DBSA_ERR_VALIDATION, "topk: need n_units >= 1");
  if (budget < 1 || budget > n_units) return set_error(DBSA_ERR_VALIDATION, "topk: budget %lld outside [1, %lld]",
                                                       (long long)budget, (long long)n_units);
  if (ordering < 0 || ordering > 2) return set_error(DBSA_ERR_VALIDATION, "topk: unknown ordering %d", ordering);
  if (n_queries == 0) return DBSA_OK;
  const size_t smem = n_units * sizeof(double) + budget * sizeof(int32_t);
  if (smem > 200 * 1024) return set_error(DBSA_ERR_SHAPE, "topk: %lld units exceed the shared-memory stage", (long long)n_units);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (smem > 48 * 1024) cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  topk_kernel<<<(unsigned)n_queries, 128, smem, s>>>(scores, n_units, budget, ordering, out_ids);
  return check_launch("topk_select");
}
