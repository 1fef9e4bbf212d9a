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
// Lanes first own splits (max, sum, per-split weights), then own 4 head dims
// each: the weights are broadcast by shuffle and 8 splits' partial rows are
// loaded before they are accumulated, so the loads of a row are in flight together.
template <bool BF16>
__device__ __forceinline__ void load4(const void *base, int64_t off, float (&v)[4]) {
  if constexpr (BF16) {
    const uint2 u = *reinterpret_cast<const uint2 *>(reinterpret_cast<const __nv_bfloat16 *>(base) + off);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&u.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162 *>(&u.y);
    v[0] = __low2float(a), v[1] = __high2float(a), v[2] = __low2float(b), v[3] = __high2float(b);
  } else {
    const float4 f = *reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(base) + off);
    v[0] = f.x, v[1] = f.y, v[2] = f.z, v[3] = f.w;
  }
}
template <bool BF16>
__device__ __forceinline__ float load1(const void *base, int64_t off) {
  if constexpr (BF16)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(base)[off]);
  else
    return reinterpret_cast<const float *>(base)[off];
}

// Partial row of split 0, row r of group g (DbsaMergeArgs.part_tok_layout).
// Element offset of (partial row, dim d) -- row-major, or the 16-column chunk
// layout of DbsaMergeArgs.part_chunk_rows (d a multiple of 4 keeps a float4 /
// 4-element load inside one chunk).
__device__ __forceinline__ int64_t part_off(const DbsaMergeArgs &a, int64_t row, int d) {
  return a.part_chunk_rows > 0 ? ((int64_t)(d >> 4) * a.part_chunk_rows + row) * 16 + (d & 15)
                               : row * a.head_dim + d;
}
__device__ __forceinline__ int64_t merge_row0(const DbsaMergeArgs &a, const DbsaMergeGroup &g, int r, int gs) {
  return a.part_tok_layout ? (int64_t)(g.q_tok0 + r / gs) * a.n_heads + g.kv_head * gs + r % gs
                           : g.part_row0 + r;
}
// Partial-out mode (DbsaMergeArgs.out_lse): the merged row's natural-log LSE.
__device__ __forceinline__ void merge_store_lse(const DbsaMergeArgs &a, int t, int head, float mx, float tot) {
  a.out_lse[(int64_t)t * a.n_heads + head] = tot > 0.f ? mx + __logf(tot) : -INFINITY;
}

template <bool BF16, bool LATENCY>
__global__ void lse_merge_kernel(DbsaMergeArgs a) {
  pdl_wait();
  const DbsaMergeGroup g = a.groups[blockIdx.y];
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= g.rows) return;
  const int hd = a.head_dim, gs = a.n_heads / a.n_kv_heads;
  const int64_t sstride = a.split_stride > 0 ? a.split_stride : g.rows;
  const int64_t row0 = merge_row0(a, g, r, gs);
  constexpr int kFast = 24;
  if (LATENCY && hd <= 128 && (hd & 3) == 0 && g.n_splits <= kFast) {
    // latency path (few rows, e.g. one query): every split's partial row is
    // loaded before the LSE reduction (the loads do not depend on it), so the
    // row costs ~two memory round trips; large merges keep the lean path below
    // (its lower register count keeps more rows in flight)
    const int dl = lane * 4 + 3 < hd ? lane * 4 : 0;
    float v[kFast][4];
#pragma unroll
    for (int s = 0; s < kFast; ++s)
      if (s < g.n_splits) load4<BF16>(a.part_o, part_off(a, row0 + (int64_t)s * sstride, dl), v[s]);
    const float l = lane < g.n_splits ? a.part_lse[row0 + (int64_t)lane * sstride] : -INFINITY;
    const float mx = warp_max(l);
    const float e = l == -INFINITY ? 0.f : __expf(l - mx);
    const float tot = warp_sum(e);
    const float wl = tot > 0.f ? e / tot : 0.f;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < kFast; ++s) {
      const float ws = __shfl_sync(0xffffffffu, wl, s);
      if (s < g.n_splits && ws != 0.f) {  // an empty split (LSE -inf) may hold garbage: 0 * NaN
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += ws * v[s][i];
      }
    }
    if (a.out_lse && lane == 0) merge_store_lse(a, g.q_tok0 + r / gs, g.kv_head * gs + r % gs, mx, tot);
    if (lane * 4 + 3 < hd) {
      const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
      __nv_bfloat16 *dst =
          reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * hd + lane * 4;
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc[0], acc[1]), hi = __floats2bfloat162_rn(acc[2], acc[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t *>(&lo);
      u.y = *reinterpret_cast<uint32_t *>(&hi);
      *reinterpret_cast<uint2 *>(dst) = u;
    }
    return;
  }
  // one read of each split's LSE: lane s holds split s (a second pass only past 32 splits)
  const float l_own = lane < g.n_splits ? a.part_lse[row0 + (int64_t)lane * sstride] : -INFINITY;
  float mx = l_own;
  for (int s = lane + 32; s < g.n_splits; s += 32) mx = fmaxf(mx, a.part_lse[row0 + (int64_t)s * sstride]);
  mx = warp_max(mx);
  float tot = l_own == -INFINITY ? 0.f : __expf(l_own - mx);
  for (int s = lane + 32; s < g.n_splits; s += 32) {
    const float l = a.part_lse[row0 + (int64_t)s * sstride];
    tot += l == -INFINITY ? 0.f : __expf(l - mx);
  }
  tot = warp_sum(tot);
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
  if (a.out_lse && lane == 0) merge_store_lse(a, t, head, mx, tot);
  __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * hd;
  const bool vec = (hd & 3) == 0;
  for (int d0 = 0; d0 < hd; d0 += 128) {
    const int d = d0 + lane * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < g.n_splits; s0 += 32) {
      const int cnt = min(32, g.n_splits - s0);
      float wl = 0.f;
      if (lane < cnt) {
        const float l = s0 == 0 ? l_own : a.part_lse[row0 + (int64_t)(s0 + lane) * sstride];
        wl = l == -INFINITY ? 0.f : __expf(l - mx) * inv;
      }
      int k = 0;
      if (vec) {  // warp-uniform: lanes past the head read column 0 and drop it
        const int dl = d + 3 < hd ? d : 0;
        for (; k + 8 <= cnt; k += 8) {
          float v[8][4];
#pragma unroll
          for (int u = 0; u < 8; ++u) load4<BF16>(a.part_o, part_off(a, row0 + (int64_t)(s0 + k + u) * sstride, dl), v[u]);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float wu = __shfl_sync(0xffffffffu, wl, k + u);
            if (wu != 0.f) {
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[i] += wu * v[u][i];
            }
          }
        }
        for (; k < cnt; ++k) {
          float v[4];
          load4<BF16>(a.part_o, part_off(a, row0 + (int64_t)(s0 + k) * sstride, dl), v);
          const float wu = __shfl_sync(0xffffffffu, wl, k);
          if (wu != 0.f) {
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += wu * v[i];
          }
        }
      } else {
        for (; k < cnt; ++k) {
          const float wu = __shfl_sync(0xffffffffu, wl, k);
          if (wu == 0.f) continue;
          const int64_t off = (row0 + (int64_t)(s0 + k) * sstride) * hd + d;
          for (int i = 0; i < 4; ++i)
            if (d + i < hd) acc[i] += wu * load1<BF16>(a.part_o, off + i);
        }
      }
    }
    if (vec && d + 3 < hd) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc[0], acc[1]), hi = __floats2bfloat162_rn(acc[2], acc[3]);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t *>(&lo);
      u.y = *reinterpret_cast<uint32_t *>(&hi);
      *reinterpret_cast<uint2 *>(dst + d) = u;
    } else {
      for (int i = 0; i < 4; ++i)
        if (d + i < hd) dst[d + i] = __float2bfloat16(acc[i]);
    }
  }
}

// Throughput form for the chunk-major batch (bf16 partials, head_dim 128): a
// quarter-warp per row, 32-byte loads (16 dims per lane), the row's split LSEs
// spread over the quarter-warp 8 at a time, 8 partial rows in flight.
__device__ __forceinline__ uint32_t pack2_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}
__global__ void lse_merge_bf16_h128_kernel(DbsaMergeArgs a) {
  pdl_wait();
  // a quarter-warp (8 lanes) per row, 32-byte loads (16 dims per lane)
  const int qw = threadIdx.x >> 3, ql = threadIdx.x & 7;
  const int r = blockIdx.x * (blockDim.x >> 3) + qw;
  const bool live = r < a.groups[blockIdx.y].rows;
  const DbsaMergeGroup g = a.groups[blockIdx.y];
  const int gs = a.n_heads / a.n_kv_heads;
  const int64_t sstride = a.split_stride > 0 ? a.split_stride : g.rows;
  const int64_t row0 = merge_row0(a, g, live ? r : 0, gs);
  const int n = g.n_splits;
  const unsigned full = 0xffffffffu;
  float mx = -INFINITY;
  for (int s = ql; s < n; s += 8) mx = fmaxf(mx, a.part_lse[row0 + (int64_t)s * sstride]);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(full, mx, o));
  float tot = 0.f;
  for (int s = ql; s < n; s += 8) {
    const float l = a.part_lse[row0 + (int64_t)s * sstride];
    tot += l == -INFINITY ? 0.f : __expf(l - mx);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) tot += __shfl_xor_sync(full, tot, o);
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  // this lane's 16 dims of split 0's row, and the distance between splits
  const bool chunked = a.part_chunk_rows > 0;
  const __nv_bfloat16 *base = reinterpret_cast<const __nv_bfloat16 *>(a.part_o) +
                              (chunked ? ((int64_t)ql * a.part_chunk_rows + row0) * 16 : row0 * 128 + ql * 16);
  const int64_t split_elems = chunked ? sstride * 16 : sstride * 128;
  const int src0 = threadIdx.x & 24;  // lane 0 of this quarter-warp
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int c0 = 0; c0 < n; c0 += 8) {
    const int sl = c0 + ql;
    const float l = sl < n ? a.part_lse[row0 + (int64_t)sl * sstride] : -INFINITY;
    const float wl = l == -INFINITY ? 0.f : __expf(l - mx) * inv;
    uint32_t v[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c0 + u < n)
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                       "=r"(v[u][6]), "=r"(v[u][7])
                     : "l"(base + (int64_t)(c0 + u) * split_elems));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float wgt = __shfl_sync(full, wl, src0 + u);
      if (c0 + u < n && wgt != 0.f) {  // skip empty splits (LSE -inf): their rows may be unwritten
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&v[u][i]));
          acc[2 * i] += wgt * f.x;
          acc[2 * i + 1] += wgt * f.y;
        }
      }
    }
  }
  if (live) {
    const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
    if (a.out_lse && ql == 0) merge_store_lse(a, t, head, mx, tot);
    __nv_bfloat16 *dst =
        reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * 128 + ql * 16;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = pack2_bf16(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// Chunk-layout form (DbsaMergeArgs.part_chunk_rows, bf16): a thread per row,
// so one 32-byte load of column chunk c from 32 consecutive rows is 1 KB of
// contiguous partials (the layout's point: K3's epilogue stores the same way).
// The row's split weights exp(lse_s - max) / sum go to shared memory once;
// then per chunk, 8 splits' loads are in flight before they are used.
constexpr int kChunkMergeThreads = 64, kChunkMergeMaxSplits = 64;
__global__ void __launch_bounds__(kChunkMergeThreads) lse_merge_chunked_kernel(DbsaMergeArgs a) {
  __shared__ float wsm[kChunkMergeMaxSplits][kChunkMergeThreads];
  pdl_wait();
  const DbsaMergeGroup g = a.groups[blockIdx.y];
  const int r = blockIdx.x * kChunkMergeThreads + threadIdx.x;
  if (r >= g.rows) return;  // no block-wide sync below: a thread's weights are its own
  const int gs = a.n_heads / a.n_kv_heads, hd = a.head_dim;
  const int64_t sstride = a.split_stride > 0 ? a.split_stride : g.rows;
  const int64_t row0 = merge_row0(a, g, r, gs);
  const int n = g.n_splits;
  // one pass of online (max, sum) over the row's split LSEs, then the weights
  float mx = -INFINITY, tot = 0.f;
  for (int s = 0; s < n; ++s) {
    const float l = a.part_lse[row0 + (int64_t)s * sstride];
    if (l == -INFINITY) continue;
    if (l > mx) {
      tot = tot * __expf(mx - l) + 1.f;
      mx = l;
    } else {
      tot += __expf(l - mx);
    }
  }
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  for (int s = 0; s < n && s < kChunkMergeMaxSplits; ++s) {
    const float l = a.part_lse[row0 + (int64_t)s * sstride];
    wsm[s][threadIdx.x] = l == -INFINITY ? 0.f : __expf(l - mx) * inv;
  }
  auto weight = [&](int s) {  // splits past the shared table (rare) recompute theirs
    if (s < kChunkMergeMaxSplits) return wsm[s][threadIdx.x];
    const float l = a.part_lse[row0 + (int64_t)s * sstride];
    return l == -INFINITY ? 0.f : __expf(l - mx) * inv;
  };
  const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
  if (a.out_lse) merge_store_lse(a, t, head, mx, tot);
  const __nv_bfloat16 *base = reinterpret_cast<const __nv_bfloat16 *>(a.part_o) + row0 * 16;
  const int64_t cstride = a.part_chunk_rows * 16, s_el = sstride * 16;
  __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * hd;
  for (int c = 0; c < hd / 16; ++c) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    const __nv_bfloat16 *bc = base + c * cstride;
    for (int s0 = 0; s0 < n; s0 += 8) {
      uint32_t v[8][8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < n)
          asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                         "=r"(v[u][6]), "=r"(v[u][7])
                       : "l"(bc + (int64_t)(s0 + u) * s_el));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float wgt = s0 + u < n ? weight(s0 + u) : 0.f;
        if (wgt != 0.f) {  // an empty split (LSE -inf) may hold garbage: 0 * NaN
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&v[u][i]));
            acc[2 * i] += wgt * f.x;
            acc[2 * i + 1] += wgt * f.y;
          }
        }
      }
    }
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = pack2_bf16(acc[2 * i], acc[2 * i + 1]);
    *reinterpret_cast<uint4 *>(dst + c * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4 *>(dst + c * 16 + 8) = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// Chunk layout, wide form: a block is 32 rows x (head_dim / 16) column chunks,
// thread (row, chunk).  A warp reads one column chunk of 32 consecutive rows
// (1 KB contiguous per split).  The rows' split LSEs are loaded once per block,
// all in flight, into shared memory; each thread then streams its 32-byte
// pieces kCM2Batch splits at a time.  Eight threads per row and four
// resident blocks per SM keep more bytes in flight than the thread-per-row
// form above (chunk-major C3: 0.118 ms -> 0.094 ms; 10 splits per batch at
// 2 blocks / SM: 0.109, 5 at 3: 0.098, 20 at 1: 0.170).
#ifndef DBSA_CM2_BATCH
#define DBSA_CM2_BATCH 4
#endif
#ifndef DBSA_CM2_MINB
#define DBSA_CM2_MINB 4
#endif
#ifndef DBSA_CM2_MIN_ROWS
#define DBSA_CM2_MIN_ROWS 128
#endif
constexpr int kCM2MaxSplits = 64, kCM2Batch = DBSA_CM2_BATCH;
__global__ void __launch_bounds__(256, DBSA_CM2_MINB) lse_merge_chunked2_kernel(DbsaMergeArgs a) {
  __shared__ float lse_s[kCM2MaxSplits][32];
  pdl_wait();
  const DbsaMergeGroup g = a.groups[blockIdx.y];
  const int rl = threadIdx.x, c = threadIdx.y, nch = blockDim.y;
  const int r = blockIdx.x * 32 + rl;
  const bool ok = r < g.rows;
  const int gs = a.n_heads / a.n_kv_heads, hd = a.head_dim;
  const int64_t sstride = a.split_stride > 0 ? a.split_stride : g.rows;
  const int64_t row0 = ok ? merge_row0(a, g, r, gs) : 0;
  const int n = g.n_splits;
  for (int s = c; s < n && s < kCM2MaxSplits; s += nch)
    lse_s[s][rl] = ok ? a.part_lse[row0 + (int64_t)s * sstride] : -INFINITY;
  __syncthreads();
  if (!ok) return;
  auto lse_at = [&](int s) {  // splits past the shared table (rare) read theirs again
    return s < kCM2MaxSplits ? lse_s[s][rl] : a.part_lse[row0 + (int64_t)s * sstride];
  };
  float mx = -INFINITY;
  for (int s = 0; s < n; ++s) mx = fmaxf(mx, lse_at(s));
  float tot = 0.f;
  for (int s = 0; s < n; ++s) {
    const float l = lse_at(s);
    tot += l == -INFINITY ? 0.f : __expf(l - mx);
  }
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  const int t = g.q_tok0 + r / gs, head = g.kv_head * gs + r % gs;
  if (a.out_lse && c == 0) merge_store_lse(a, t, head, mx, tot);
  const __nv_bfloat16 *bc = reinterpret_cast<const __nv_bfloat16 *>(a.part_o) + row0 * 16 + c * a.part_chunk_rows * 16;
  const int64_t s_el = sstride * 16;
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int s0 = 0; s0 < n; s0 += kCM2Batch) {
    uint32_t v[kCM2Batch][8];
#pragma unroll
    for (int u = 0; u < kCM2Batch; ++u)
      if (s0 + u < n)
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]), "=r"(v[u][5]),
                       "=r"(v[u][6]), "=r"(v[u][7])
                     : "l"(bc + (int64_t)(s0 + u) * s_el));
#pragma unroll
    for (int u = 0; u < kCM2Batch; ++u) {
      const float l = s0 + u < n ? lse_at(s0 + u) : -INFINITY;
      if (l != -INFINITY) {  // an empty split (LSE -inf) may hold garbage: 0 * NaN
        const float wgt = __expf(l - mx) * inv;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&v[u][i]));
          acc[2 * i] += wgt * f.x;
          acc[2 * i + 1] += wgt * f.y;
        }
      }
    }
  }
  if (c * 16 >= hd) return;
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = pack2_bf16(acc[2 * i], acc[2 * i + 1]);
  __nv_bfloat16 *dst =
      reinterpret_cast<__nv_bfloat16 *>(a.out) + (int64_t)t * a.out_tok_stride + (int64_t)head * hd + c * 16;
  *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4 *>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
}

// x fp32 [rows, dim] -> bf16 x * rsqrt(mean(x^2) + eps) * w (kernels.rms_norm, kernels.py:103-112).
// ADD: first x += delta in place -- the residual add of model.py:352-359 fused
// with the norm that reads the same row.  float4 path: each thread keeps its
// VPT float4 of the row in registers between the sum and the scale pass.
template <bool ADD, int VPT>
__global__ void rmsnorm4_kernel(float *x, const float *delta, const float *w, __nv_bfloat16 *out, int64_t dim,
                                float eps) {
  const int64_t row = blockIdx.x;
  float4 *xr = reinterpret_cast<float4 *>(x + row * dim);
  const int n4 = (int)(dim >> 2);
  float4 v[VPT], ww[VPT];
  pdl_wait();
  // the weight loads go out with the row's (not after the reduction), so
  // they are in registers by the scale pass
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < n4) ww[k] = __ldg(reinterpret_cast<const float4 *>(w) + i);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < n4) {
      v[k] = xr[i];
      if constexpr (ADD) {
        const float4 d = reinterpret_cast<const float4 *>(delta + row * dim)[i];
        v[k].x += d.x, v[k].y += d.y, v[k].z += d.z, v[k].w += d.w;
        xr[i] = v[k];
      }
      ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)dim + eps);
  uint2 *orow = reinterpret_cast<uint2 *>(out + row * dim);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < n4) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(v[k].x * inv * ww[k].x, v[k].y * inv * ww[k].y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(v[k].z * inv * ww[k].z, v[k].w * inv * ww[k].w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t *>(&lo);
      u.y = *reinterpret_cast<uint32_t *>(&hi);
      orow[i] = u;
    }
  }
}

template <bool ADD>
__global__ void rmsnorm_kernel(float *x, const float *delta, const float *w, __nv_bfloat16 *out, int64_t dim,
                               float eps) {
  pdl_wait();
  const int64_t row = blockIdx.x;
  float *xr = x + row * dim;
  float ss = 0.f;
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) {
    float v = xr[i];
    if constexpr (ADD) {
      v += delta[row * dim + i];
      xr[i] = v;
    }
    ss += v * v;
  }
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

template <bool ADD>
static int launch_rmsnorm(float *x, const float *delta, const float *weight, void *out, int64_t rows, int64_t dim,
                          float eps, cudaStream_t st) {
  if (rows <= 0) return DBSA_OK;
  __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(out);
  const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(weight) |
                    reinterpret_cast<uintptr_t>(out) | (ADD ? reinterpret_cast<uintptr_t>(delta) : 0)) & 15) == 0;
  // the residual stream x is re-read by the next norm one projection / FFN
  // later: keep it in L2 across the weight streams (small batches only)
  const size_t xbytes = (size_t)rows * dim * sizeof(float);
  const Persist keep{x, ADD && xbytes <= kPersistMaxBytes ? xbytes : 0};
  if (dim % 4 == 0 && al && dim <= 4 * 256 * 8) {
    const int n4 = (int)(dim / 4);
    if (n4 <= 256 * 4)
      launch_kp(rmsnorm4_kernel<ADD, 4>, dim3((unsigned)rows), dim3(256), 0, st, true, keep, x, delta, weight, o, dim,
                eps);
    else
      launch_kp(rmsnorm4_kernel<ADD, 8>, dim3((unsigned)rows), dim3(256), 0, st, true, keep, x, delta, weight, o, dim,
                eps);
  } else {
    const int threads = dim >= 1024 ? 256 : (dim >= 256 ? 128 : 64);
    launch_kp(rmsnorm_kernel<ADD>, dim3((unsigned)rows), dim3(threads), 0, st, true, keep, x, delta, weight, o, dim,
              eps);
  }
  return check_launch("rmsnorm");
}

// gate_up bf16 [rows, 2*ffn] (gate | up) -> silu(gate) * up (kernels.silu_gate, kernels.py:115-123).
__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }
__global__ void silu_mul_kernel(const __nv_bfloat16 *gu, __nv_bfloat16 *out, int64_t rows, int64_t ffn) {
  pdl_wait();
  const int64_t n = rows * ffn;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / ffn, c = idx % ffn;
    const float g = __bfloat162float(gu[r * 2 * ffn + c]);
    const float u = __bfloat162float(gu[r * 2 * ffn + ffn + c]);
    out[idx] = __float2bfloat16(silu_f(g) * u);
  }
}
// 8 columns per thread (16-byte loads of gate and up), one CTA row-strip per y.
__global__ void silu_mul8_kernel(const uint4 *gu, uint4 *out, int64_t rows, int64_t ffn8) {
  pdl_wait();
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const uint4 *gr = gu + r * 2 * ffn8;
    uint4 *orow = out + r * ffn8;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ffn8; c += (int64_t)gridDim.x * blockDim.x) {
      const uint4 g4 = gr[c], u4 = gr[ffn8 + c];
      const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&g4);
      const __nv_bfloat162 *u2 = reinterpret_cast<const __nv_bfloat162 *>(&u4);
      uint4 o4;
      __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(&o4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 g = __bfloat1622float2(g2[i]), u = __bfloat1622float2(u2[i]);
        o2[i] = __floats2bfloat162_rn(silu_f(g.x) * u.x, silu_f(g.y) * u.y);
      }
      orow[c] = o4;
    }
  }
}

// logprob[r] = logits[r, target[r]] - logsumexp(logits[r, :]) (model.log_softmax_rows, model.py:414-417).
// One pass over the row: each thread keeps an online (max, sum) over float4
// reads, merged across the block.
__device__ __forceinline__ void lse_combine(float &m, float &s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}
__global__ void label_logprob_kernel(const float *logits, int64_t vocab, const int32_t *target, float *out) {
  const int64_t row = blockIdx.x;
  const float *lr = logits + row * vocab;
  float m = -INFINITY, sum = 0.f;
  auto add = [&](float v) {
    if (v > m) {
      sum = (m == -INFINITY ? 0.f : sum * __expf(m - v)) + 1.f;
      m = v;
    } else {
      sum += __expf(v - m);
    }
  };
  if ((vocab & 3) == 0 && (reinterpret_cast<uintptr_t>(lr) & 15) == 0) {
    const float4 *l4 = reinterpret_cast<const float4 *>(lr);
    for (int64_t i = threadIdx.x; i < vocab / 4; i += blockDim.x) {
      const float4 v = l4[i];
      const float vm = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
      if (vm > m) {
        sum = m == -INFINITY ? 0.f : sum * __expf(m - vm);
        m = vm;
      }
      sum += __expf(v.x - m) + __expf(v.y - m) + __expf(v.z - m) + __expf(v.w - m);
    }
  } else {
    for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) add(lr[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    lse_combine(m, sum, m2, s2);
  }
  __shared__ float sm[32], ss[32];
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x >> 5] = m;
    ss[threadIdx.x >> 5] = sum;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool ok = threadIdx.x < (blockDim.x >> 5);
    m = ok ? sm[threadIdx.x] : -INFINITY;
    sum = ok ? ss[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      lse_combine(m, sum, m2, s2);
    }
    if (threadIdx.x == 0) out[row] = lr[target[row]] - m - logf(sum);
  }
}

// Per query (one warp): label score = sum of its tokens' log-probs (rows
// label_row0[o] .. label_row0[o+1] of output o = q * n_labels + l, summed in
// order), then the strict-> argmax over the labels (the first maximum wins:
// pipeline.py:376-382 over the sorted labels).
__global__ void label_reduce_kernel(const float *lp, const int32_t *label_row0, int64_t n_queries, int n_labels,
                                    float *scores, int64_t *best) {
  const int64_t q = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= n_queries) return;
  float sc = -INFINITY;
  int idx = 0x7fffffff;
  for (int l = lane; l < n_labels; l += 32) {
    const int64_t o = q * n_labels + l;
    float acc = 0.f;
    for (int r = label_row0[o]; r < label_row0[o + 1]; ++r) acc += lp[r];
    scores[o] = acc;
    if (acc > sc) {
      sc = acc;
      idx = l;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float s2 = __shfl_xor_sync(0xffffffffu, sc, off);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, off);
    if (s2 > sc || (s2 == sc && i2 < idx)) {
      sc = s2;
      idx = i2;
    }
  }
  if (lane == 0) best[q] = idx == 0x7fffffff ? 0 : idx;
}

}  // namespace dbsa

extern "C" int dbsa_lse_merge(const DbsaMergeArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_lse_merge: null args");
  const DbsaMergeArgs &a = *args;
  if (a.n_groups <= 0 || a.max_rows <= 0) return DBSA_OK;
  if (a.part_chunk_rows > 0 && (!a.part_bf16 || a.part_tok_layout || a.head_dim % 16))
    return set_error(DBSA_ERR_CONFIG, "part_chunk_rows needs bf16 row-indexed partials and head_dim %% 16 == 0");
  dim3 grid((a.max_rows + 3) / 4, a.n_groups);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool small = (int64_t)a.n_groups * a.max_rows <= 16384;
  // the chunk layout: a thread per row (the latency form for small merges reads it through part_off)
  static const bool wide = [] {
    const char *e = getenv("DBSA_MERGE_WIDE");
    return !(e && e[0] == '0');
  }();
  // the wide form wins on tall groups (GQA: rows = tokens x group size; C3 K3m
  // 0.118 -> 0.109 ms) and loses on short ones (MHA C4, 44 rows: 0.037 -> 0.056)
  if (a.part_chunk_rows > 0 && !small && wide && a.max_rows >= DBSA_CM2_MIN_ROWS && a.head_dim % 16 == 0 && a.head_dim <= 256) {
    launch_k(lse_merge_chunked2_kernel, dim3((a.max_rows + 31) / 32, a.n_groups), dim3(32, a.head_dim / 16), 0, st,
             true, a);
    return check_launch("lse_merge");
  }
  if (a.part_chunk_rows > 0 && !small) {
    launch_k(lse_merge_chunked_kernel, dim3((a.max_rows + kChunkMergeThreads - 1) / kChunkMergeThreads, a.n_groups),
             dim3(kChunkMergeThreads), 0, st, true, a);
    return check_launch("lse_merge");
  }
  if (a.part_bf16 && a.head_dim == 128 && !small) {
    launch_k(lse_merge_bf16_h128_kernel, dim3((a.max_rows + 15) / 16, a.n_groups), dim3(128), 0, st, true, a);
    return check_launch("lse_merge");
  }
  if (a.part_bf16) {
    if (small)
      launch_k(lse_merge_kernel<true, true>, grid, dim3(128), 0, st, true, a);
    else
      launch_k(lse_merge_kernel<true, false>, grid, dim3(128), 0, st, true, a);
  } else {
    if (small)
      launch_k(lse_merge_kernel<false, true>, grid, dim3(128), 0, st, true, a);
    else
      launch_k(lse_merge_kernel<false, false>, grid, dim3(128), 0, st, true, a);
  }
  return check_launch("lse_merge");
}

extern "C" int dbsa_rmsnorm(const float *x, const float *weight, void *out, int64_t rows, int64_t dim, float eps,
                            void *stream) {
  return dbsa::launch_rmsnorm<false>(const_cast<float *>(x), nullptr, weight, out, rows, dim, eps,
                                     reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int dbsa_add_rmsnorm(float *x, const float *delta, const float *weight, void *out, int64_t rows, int64_t dim,
                                float eps, void *stream) {
  return dbsa::launch_rmsnorm<true>(x, delta, weight, out, rows, dim, eps, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int dbsa_silu_mul(const void *gate_up, void *out, int64_t rows, int64_t ffn, void *stream) {
  using namespace dbsa;
  if (rows <= 0) return DBSA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (ffn % 8 == 0 && (reinterpret_cast<uintptr_t>(gate_up) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const int64_t ffn8 = ffn / 8;
    const int bx = (int)((ffn8 + 255) / 256);
    const int by = (int)(rows < 65535 ? rows : 65535);
    launch_k(silu_mul8_kernel, dim3(bx, by), dim3(256), 0, st, true, reinterpret_cast<const uint4 *>(gate_up),
             reinterpret_cast<uint4 *>(out), rows, ffn8);
    return check_launch("silu_mul");
  }
  const int64_t n = rows * ffn;
  const int blocks = (int)((n + 255) / 256 < 148 * 32 ? (n + 255) / 256 : 148 * 32);
  silu_mul_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16 *>(gate_up),
                                          reinterpret_cast<__nv_bfloat16 *>(out), rows, ffn);
  return check_launch("silu_mul");
}

extern "C" int dbsa_label_logprob(const float *logits, int64_t rows, int64_t vocab, const int32_t *target, float *out,
                                  void *stream) {
  using namespace dbsa;
  if (rows <= 0) return DBSA_OK;
  label_logprob_kernel<<<(unsigned)rows, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(logits, vocab, target, out);
  return check_launch("label_logprob");
}

extern "C" int dbsa_label_reduce(const float *lp, const int32_t *label_row0, int64_t n_queries, int32_t n_labels,
                                 float *scores, int64_t *best, void *stream) {
  using namespace dbsa;
  if (n_queries <= 0) return DBSA_OK;
  if (n_labels <= 0) return set_error(DBSA_ERR_VALIDATION, "n_labels must be positive");
  const int per_block = 4;  // warps (queries) per block
  label_reduce_kernel<<<(unsigned)((n_queries + per_block - 1) / per_block), 32 * per_block, 0,
                        reinterpret_cast<cudaStream_t>(stream)>>>(lp, label_row0, n_queries, n_labels, scores, best);
  return check_launch("label_reduce");
}
