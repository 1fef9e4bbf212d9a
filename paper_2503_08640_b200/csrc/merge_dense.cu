// merge_dense.cu -- K3m LSE merge of split partials, plus the small fused
// dense-path kernels of the pre-norm block (RMSNorm, SiLU gate) and the
// label log-prob gather of score_label.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"

namespace dbsa {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per (group, row): lse = log sum_s exp(lse_s); O = sum_s exp(lse_s - lse) O_s.
// This is the split form of the single softmax of kernels._softmax64 (kernels.py:52-56).
template <bool BF16>
__global__ void lse_merge_kernel(DbsaMergeArgs a) {
  const DbsaMergeGroup g = a.groups[blockIdx.y];
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= g.rows) return;
  const int hd = a.head_dim, gs = a.n_heads / a.n_kv_heads;
  const int64_t sstride = a.split_stride > 0 ? a.split_stride : g.rows;
  float mx = -INFINITY;
  for (int s = lane; s < g.n_splits; s += 32) mx = fmaxf(mx, a.part_lse[g.part_row0 + (int64_t)s * sstride + r]);
  mx = warp_max(mx);
  float tot = 0.f;
  for (int s = lane; s < g.n_splits; s += 32) {
    const float l = a.part_lse[g.part_row0 + (int64_t)s * sstride + r];
    tot += l == -INFINITY ? 0.f : __expf(l - mx);
  }
  tot = warp_sum(tot);
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
  __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * hd;
  for (int d0 = 0; d0 < hd; d0 += 32 * 4) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < g.n_splits; ++s) {
      const float l = a.part_lse[g.part_row0 + (int64_t)s * sstride + r];
      if (l == -INFINITY) continue;
      const float wgt = __expf(l - mx) * inv;
      const int64_t off = (g.part_row0 + (int64_t)s * sstride + r) * hd;
      if constexpr (BF16) {
        const __nv_bfloat16 *src = reinterpret_cast<const __nv_bfloat16 *>(a.part_o) + off;
        if ((hd & 3) == 0 && d0 + lane * 4 + 3 < hd) {
          const uint2 v = *reinterpret_cast<const uint2 *>(src + d0 + lane * 4);
          const __nv_bfloat162 v0 = *reinterpret_cast<const __nv_bfloat162 *>(&v.x);
          const __nv_bfloat162 v1 = *reinterpret_cast<const __nv_bfloat162 *>(&v.y);
          acc[0] += wgt * __low2float(v0);
          acc[1] += wgt * __high2float(v0);
          acc[2] += wgt * __low2float(v1);
          acc[3] += wgt * __high2float(v1);
        } else {
          for (int i = 0; i < 4; ++i)
            if (d0 + lane * 4 + i < hd) acc[i] += wgt * __bfloat162float(src[d0 + lane * 4 + i]);
        }
      } else {
        const float *src = reinterpret_cast<const float *>(a.part_o) + off;
        if ((hd & 3) == 0 && d0 + lane * 4 + 3 < hd) {
          const float4 v = *reinterpret_cast<const float4 *>(src + d0 + lane * 4);
          acc[0] += wgt * v.x;
          acc[1] += wgt * v.y;
          acc[2] += wgt * v.z;
          acc[3] += wgt * v.w;
        } else {
          for (int i = 0; i < 4; ++i)
            if (d0 + lane * 4 + i < hd) acc[i] += wgt * src[d0 + lane * 4 + i];
        }
      }
    }
    for (int i = 0; i < 4; ++i)
      if (d0 + lane * 4 + i < hd) dst[d0 + lane * 4 + i] = __float2bfloat16(acc[i]);
  }
}

// x fp32 [rows, dim] -> bf16 x * rsqrt(mean(x^2) + eps) * w (kernels.rms_norm, kernels.py:103-112).
__global__ void rmsnorm_kernel(const float *x, const float *w, __nv_bfloat16 *out, int64_t dim, float eps) {
  const int64_t row = blockIdx.x;
  const float *xr = x + row * dim;
  float ss = 0.f;
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) ss += xr[i] * xr[i];
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)dim + eps);
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) out[row * dim + i] = __float2bfloat16(xr[i] * inv * w[i]);
}

// gate_up bf16 [rows, 2*ffn] (gate | up) -> silu(gate) * up (kernels.silu_gate, kernels.py:115-123).
__global__ void silu_mul_kernel(const __nv_bfloat16 *gu, __nv_bfloat16 *out, int64_t rows, int64_t ffn) {
  const int64_t n = rows * ffn;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / ffn, c = idx % ffn;
    const float g = __bfloat162float(gu[r * 2 * ffn + c]);
    const float u = __bfloat162float(gu[r * 2 * ffn + ffn + c]);
    out[idx] = __float2bfloat16(g / (1.f + __expf(-g)) * u);
  }
}

// logprob[r] = logits[r, target[r]] - logsumexp(logits[r, :]) (model.log_softmax_rows, model.py:414-417).
__global__ void label_logprob_kernel(const float *logits, int64_t vocab, const int32_t *target, float *out) {
  const int64_t row = blockIdx.x;
  const float *lr = logits + row * vocab;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) mx = fmaxf(mx, lr[i]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) s += __expf(lr[i] - mx);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[row] = lr[target[row]] - mx - logf(v);
  }
}

}  // namespace dbsa

extern "C" int dbsa_lse_merge(const DbsaMergeArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_lse_merge: null args");
  const DbsaMergeArgs &a = *args;
  if (a.n_groups <= 0 || a.max_rows <= 0) return DBSA_OK;
  dim3 grid((a.max_rows + 3) / 4, a.n_groups);
  if (a.part_bf16)
    lse_merge_kernel<true><<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  else
    lse_merge_kernel<false><<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("lse_merge");
}

extern "C" int dbsa_rmsnorm(const float *x, const float *weight, void *out, int64_t rows, int64_t dim, float eps,
                            void *stream) {
  using namespace dbsa;
  if (rows <= 0) return DBSA_OK;
  const int threads = dim >= 1024 ? 256 : (dim >= 256 ? 128 : 64);
  rmsnorm_kernel<<<(unsigned)rows, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, weight, reinterpret_cast<__nv_bfloat16 *>(out), dim, eps);
  return check_launch("rmsnorm");
}

extern "C" int dbsa_silu_mul(const void *gate_up, void *out, int64_t rows, int64_t ffn, void *stream) {
  using namespace dbsa;
  if (rows <= 0) return DBSA_OK;
  const int64_t n = rows * ffn;
  const int blocks = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  silu_mul_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16 *>(gate_up), reinterpret_cast<__nv_bfloat16 *>(out), rows, ffn);
  return check_launch("silu_mul");
}

extern "C" int dbsa_label_logprob(const float *logits, int64_t rows, int64_t vocab, const int32_t *target, float *out,
                                  void *stream) {
  using namespace dbsa;
  if (rows <= 0) return DBSA_OK;
  label_logprob_kernel<<<(unsigned)rows, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(logits, vocab, target, out);
  return check_launch("label_logprob");
}
