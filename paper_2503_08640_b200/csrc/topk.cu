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

// ---------------------------------------------------------------------------
// Large unit counts (example granularity: thousands of demonstrations): a
// radix select instead of the O(n^2) comparison count.  The (-score, id)
// order is a 64-bit key per candidate -- the score's bits made order-
// preserving and complemented (larger score = smaller key; -0.0 folded onto
// +0.0, which Python's sort treats as equal), with the id breaking ties --
// so the budget-1 best candidates are those with key < T plus the lowest-id
// ones with key == T, where T (the (k-1)-th smallest key) is found by eight
// 8-bit MSB-first histogram passes.  Compaction in ascending id order gives
// in-order (and, reversed, reverse) directly; low-to-high ranks the k picked
// units by (score, id) by counting.  Only integer operations on the score
// bits: identical to the reference's sort.
__device__ __forceinline__ unsigned long long desc_key(double d) {
  unsigned long long b = __double_as_longlong(d == 0.0 ? 0.0 : d);
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending in d
  return ~b;                                         // descending in d
}

constexpr int kTopkThreads = 512;
constexpr int64_t kTopkCountMax = 256;    // up to here the O(n^2) shared-memory count is faster
constexpr int64_t kTopkSortMax = 16384;   // low-to-high: picked units sorted in shared memory

__global__ void __launch_bounds__(kTopkThreads) topk_radix_kernel(const double *scores, int64_t n_units,
                                                                  int64_t budget, int ordering, int32_t *out,
                                                                  int sort_pow2) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_kk;
  __shared__ long long s_less[kTopkThreads], s_eq[kTopkThreads];
  const int64_t q = blockIdx.x;
  const double *row = scores + q * n_units;
  int32_t *o = out + q * budget;
  const long long k = budget - 1;  // candidates to pick among ids 1..n-1
  if (threadIdx.x == 0) {
    o[0] = 0;
    s_prefix = 0ull;
    s_kk = k - 1;  // 0-based rank of T among the remaining candidates
  }
  if (k == 0) return;
  __syncthreads();
  unsigned long long mask = 0ull;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    for (int64_t u = 1 + threadIdx.x; u < n_units; u += blockDim.x) {
      const unsigned long long key = desc_key(row[u]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // one warp finds the digit holding rank kk
      const long long kk = s_kk;
      unsigned int c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) tot += (c[j] = hist[threadIdx.x * 8 + j]);
      unsigned int incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned int v = __shfl_up_sync(0xffffffffu, incl, off);
        if ((int)threadIdx.x >= off) incl += v;
      }
      unsigned int before = incl - tot;
      const bool mine = before <= (unsigned long long)kk && (unsigned long long)kk < incl;
      if (mine) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((unsigned long long)kk < before + c[j]) {
            s_prefix = prefix | ((unsigned long long)(threadIdx.x * 8 + j) << shift);
            s_kk = kk - before;
            break;
          }
          before += c[j];
        }
      }
    }
    mask |= 255ull << shift;
    __syncthreads();
  }
  const unsigned long long T = s_prefix;
  const long long need = s_kk + 1;  // candidates with key == T to take, lowest ids first
  // ordered compaction: thread t owns the contiguous id range [lo, hi)
  const int64_t per = (n_units - 1 + blockDim.x - 1) / blockDim.x;
  const int64_t lo = 1 + threadIdx.x * per, hi = min(n_units, lo + per);
  long long n_less = 0, n_eq = 0;
  for (int64_t u = lo; u < hi; ++u) {
    const unsigned long long key = desc_key(row[u]);
    n_less += key < T;
    n_eq += key == T;
  }
  s_less[threadIdx.x] = n_less;
  s_eq[threadIdx.x] = n_eq;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scans (512 entries, once per query)
    long long a = 0, b = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const long long x = s_less[t], y = s_eq[t];
      s_less[t] = a;
      s_eq[t] = b;
      a += x;
      b += y;
    }
  }
  __syncthreads();
  __shared__ long long s_last_tie;  // id of the last tie taken (ties up to it are picked)
  long long less_before = s_less[threadIdx.x], eq_before = s_eq[threadIdx.x];
  for (int64_t u = lo; u < hi; ++u) {
    const unsigned long long key = desc_key(row[u]);
    const bool take = key < T || (key == T && eq_before < need);
    if (take) {
      const long long pos = less_before + (eq_before < need ? eq_before : need);  // rank in ascending id
      if (ordering == 2) o[k - pos] = (int32_t)u;
      else o[1 + pos] = (int32_t)u;  // in-order; low-to-high sorts these below
      if (key == T && eq_before == need - 1) s_last_tie = u;
    }
    less_before += key < T;
    eq_before += key == T;
  }
  if (ordering != 1) return;
  __syncthreads();
  if (sort_pow2 > 0) {
    // low-to-high: bitonic sort of the k picked units by (score, id) ascending
    // in shared memory (k <= kTopkSortMax)
    extern __shared__ unsigned long long dyn[];
    unsigned long long *sk = dyn;                                   // [sort_pow2] ascending-score keys
    int32_t *sid = reinterpret_cast<int32_t *>(sk + sort_pow2);     // [sort_pow2] ids
    for (int i = threadIdx.x; i < sort_pow2; i += blockDim.x) {
      if (i < k) {
        const int32_t id = o[1 + i];
        sk[i] = ~desc_key(row[id]);
        sid[i] = id;
      } else {
        sk[i] = ~0ull;
        sid[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    for (int size = 2; size <= sort_pow2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < sort_pow2; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const bool gt = sk[i] > sk[j] || (sk[i] == sk[j] && sid[i] > sid[j]);
            if (gt == up) {
              const unsigned long long tk = sk[i];
              sk[i] = sk[j];
              sk[j] = tk;
              const int32_t ti = sid[i];
              sid[i] = sid[j];
              sid[j] = ti;
            }
          }
        }
        __syncthreads();
      }
    }
    for (long long i = threadIdx.x; i < k; i += blockDim.x) o[1 + i] = sid[i];
    return;
  }
  // low-to-high past the shared-memory sort: rank each picked unit by (score,
  // id) ascending among the picked set {key < T} + {key == T, id <= last tie},
  // by counting over the row
  const long long last_tie = s_last_tie;
  for (int64_t u = lo; u < hi; ++u) {
    const unsigned long long ku = desc_key(row[u]);
    if (!(ku < T || (ku == T && u <= last_tie))) continue;
    long long pos = 0;
    for (int64_t v = 1; v < n_units; ++v) {
      const unsigned long long kv = desc_key(row[v]);
      const bool picked = kv < T || (kv == T && v <= last_tie);
      // ascending score == descending desc_key
      pos += picked && (kv > ku || (kv == ku && v < u));
    }
    o[1 + pos] = (int32_t)u;
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
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n_units > kTopkCountMax) {  // O(n) radix select (example granularity)
    int pow2 = 0;
    if (ordering == 1 && budget - 1 <= kTopkSortMax) {
      pow2 = 1;
      while (pow2 < budget - 1) pow2 <<= 1;
    }
    const size_t smem = (size_t)pow2 * (sizeof(unsigned long long) + sizeof(int32_t));
    if (smem > 32 * 1024)  // dynamic + the kernel's ~10 KB of static shared memory past the 48 KB default
      cudaFuncSetAttribute(topk_radix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    topk_radix_kernel<<<(unsigned)n_queries, kTopkThreads, smem, s>>>(scores, n_units, budget, ordering, out_ids,
                                                                      pow2);
    return check_launch("topk_select");
  }
  const size_t smem = n_units * sizeof(double) + budget * sizeof(int32_t);
  if (smem > 48 * 1024) cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  topk_kernel<<<(unsigned)n_queries, 128, smem, s>>>(scores, n_units, budget, ordering, out_ids);
  return check_launch("topk_select");
}
