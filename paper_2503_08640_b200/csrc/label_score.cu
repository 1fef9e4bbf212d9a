// label_score.cu -- K5, the fused label-scoring epilogue of stage 2.
//
// The reference scores a label by materialising the logits of every scored
// row (model.logits_from_hidden, model.py:393-397), taking log_softmax_rows
// (model.py:414-417) and gathering the label token (model.py:441-443).  Here
// the logits never leave the SM: a persistent tcgen05 GEMM over x @ lm_head
// (x: the final-normed scored rows, lm_head K-major [vocab, d]) holds a
// 256-row x 256-vocab fp32 tile in TMEM (two M tiles of 128 lanes x 256
// columns = all 512 columns), and the epilogue warpgroups fold each row's 256
// logits into a running (max, sum of 2^x) before the next tile overwrites the
// accumulator.  A second small launch combines a row's per-tile partials into
// its LSE and subtracts it from the target logit.
//
//   warp 0: TMA producer (x and lm_head K slices of 64, 128B swizzle)
//   warp 1: MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M128 N256 K16, SS)
//   warp 2: TMEM allocator
//   warps 4-11: epilogue, one warpgroup per accumulator slot, one row per thread
// Batch-1 shapes (rows <= 128, one M tile) use the narrow form: N = 128 vocab
// tiles (twice the works, a shorter last wave), a 6-deep ring of one-M-tile
// stages, x loaded for its real rows only, and the two TMEM slots alternating
// between works so one slot's epilogue overlaps the next work's MMAs.
//
// Work = (pair of M tiles, vocab tile), M-pair fastest, so the CTAs running
// at the same time share vocab tiles and lm_head is read from HBM about once
// per launch (x, a few MB, stays in L2).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"
#include "sm100_ptx.cuh"

namespace dbsa {

constexpr int kLsBK = 64;                          // K per stage: one 128-byte swizzle row of bf16
constexpr int kLsMBytes = 128 * kLsBK * 2;         // one M tile's K slice (16 KB)
constexpr int kLsABytes = 2 * kLsMBytes;           // two M tiles
constexpr int kLsHalf = 128;                       // workspace granularity: one (max, sum) per 128 vocab columns
constexpr int kLsThreads = 384;

// BN vocab columns per tile (one N = BN MMA): 256 for batches, 128 when the
// rows fit one M tile (batch 1), so the vocab splits into twice as many works
// and the last wave of the persistent grid is shorter.  Deeper ring for BN 128.
template <int BN, bool NARROW>
struct LsCfg {
  static constexpr int ABytes = NARROW ? kLsMBytes : kLsABytes;  // the narrow form has one M tile
  static constexpr int BBytes = BN * kLsBK * 2;
  static constexpr int StageBytes = ABytes + BBytes;
  static constexpr int Stages = (200 * 1024) / StageBytes > 8 ? 8 : (200 * 1024) / StageBytes;
  static constexpr int Smem = Stages * StageBytes + 1024 + 1024;
};

struct LsParams {
  int64_t rows, rows_pad, vocab;
  int m_tiles, m_pairs, n_tiles, k_steps, n_work, x_box_rows;
  float2 *part;  // [vocab / 128][rows_pad]: (max, sum of 2^(x - max)) of x = logit * log2(e)
};

// Accumulator slots: a work with two M tiles uses TMEM slots 0 and 1 (one per
// M tile); a work with one M tile (batch 1, or the odd last tile) takes slot
// 0 / 1 alternately, so the next work's MMAs run while the other epilogue
// warpgroup drains the previous one.  Every role walks the same work list and
// derives the same slots.
struct LsSlots {
  int n_single = 0;
  __device__ __forceinline__ int first(int nm) {  // slot of M tile 0 of the next work (nm M tiles)
    return nm == 2 ? 0 : (n_single++ & 1);
  }
};

template <int BN, bool NARROW>
__global__ void __launch_bounds__(kLsThreads, 1)
    label_lse_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                     const LsParams p) {
  using C = LsCfg<BN, NARROW>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::Stages * C::StageBytes);
  uint64_t *full = bars;                   // [stages] K slice landed
  uint64_t *empty = full + C::Stages;      // [stages] K slice consumed by the MMAs
  uint64_t *acc_full = empty + C::Stages;  // [2] accumulator slot complete
  uint64_t *acc_empty = acc_full + 2;      // [2] accumulator slot read by the epilogue
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int m = 0; m < 2; ++m) {
      mbar_init(&acc_full[m], 1);
      mbar_init(&acc_empty[m], 128);
    }
    fence_mbar_init();
    tma_prefetch(&tm_x);
    tma_prefetch(&tm_w);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int wk = blockIdx.x; wk < p.n_work; wk += gridDim.x) {
        const int m0 = (wk % p.m_pairs) * 2, nt = wk / p.m_pairs;
        const int nm = min(2, p.m_tiles - m0);
        // narrow: only the x box rows (p.x_box_rows, the real rows rounded to 16) are
        // loaded; the stale rows below them in the A tile only feed accumulator rows the
        // epilogue never stores (row r of D depends on row r of A alone)
        const uint32_t bytes = nm * (uint32_t)p.x_box_rows * (kLsBK * 2) + C::BBytes;
        for (int k = 0; k < p.k_steps; ++k, ++it) {
          const int s = it % C::Stages;
          if (it >= C::Stages) mbar_wait(&empty[s], ((it / C::Stages) & 1) ^ 1);
          uint8_t *st = smem + s * C::StageBytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          for (int m = 0; m < nm; ++m) tma_load_2d(st + m * kLsMBytes, &tm_x, &full[s], k * kLsBK, (m0 + m) * 128);
          tma_load_2d(st + C::ABytes, &tm_w, &full[s], k * kLsBK, nt * BN);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
    const bool leader = elect_one();
    int it = 0;
    int cnt[2] = {0, 0};  // tiles accumulated per slot (acc_full / acc_empty phases)
    LsSlots sl;
    for (int wk = blockIdx.x; wk < p.n_work; wk += gridDim.x) {
      const int m0 = (wk % p.m_pairs) * 2;
      const int nm = min(2, p.m_tiles - m0);
      const int s0 = sl.first(nm);
      for (int m = 0; m < nm; ++m)
        if (cnt[s0 + m] > 0) mbar_wait(&acc_empty[s0 + m], (cnt[s0 + m] - 1) & 1);  // the epilogue drained it
      tc_fence_after();
      for (int k = 0; k < p.k_steps; ++k, ++it) {
        const int s = it % C::Stages;
        mbar_wait(&full[s], (it / C::Stages) & 1);
        tc_fence_after();
        if (leader) {
          const uint32_t sa = smem_u32(smem + s * C::StageBytes), sb = sa + C::ABytes;
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            if (m < nm) {
#pragma unroll
              for (int kk = 0; kk < kLsBK / 16; ++kk)
                umma_bf16_ss(tbase + (s0 + m) * 256, umma_desc_kmajor(sa + m * kLsMBytes + kk * 32, 128),
                             umma_desc_kmajor(sb + kk * 32, 128), idesc, (k | kk) != 0 ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (leader)
        for (int m = 0; m < nm; ++m) umma_commit(&acc_full[s0 + m]);
      __syncwarp();
      for (int m = 0; m < nm; ++m) ++cnt[s0 + m];
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue: row LSE partials
    const int e = (warp - 4) >> 2, q4 = warp & 3;  // this warpgroup drains accumulator slot e
    const int trow = q4 * 32 + lane;
    const uint32_t t_acc = tbase + ((uint32_t)(q4 * 32) << 16) + e * 256;
    constexpr float kLog2e = 1.4426950408889634f;
    int cnt = 0;
    LsSlots sl;
    for (int wk = blockIdx.x; wk < p.n_work; wk += gridDim.x) {
      const int m0 = (wk % p.m_pairs) * 2, nt = wk / p.m_pairs;
      const int nm = min(2, p.m_tiles - m0);
      const int s0 = sl.first(nm);
      if (e < s0 || e >= s0 + nm) continue;
      const int m = m0 + (e - s0);  // the M tile in this slot
      mbar_wait(&acc_full[e], cnt & 1);
      tc_fence_after();
      const int64_t col0 = (int64_t)nt * BN;
      const int valid = p.vocab - col0 < BN ? (int)(p.vocab - col0) : BN;  // columns past the vocab are TMA zero fill
      const int64_t row = (int64_t)m * 128 + trow;
      float mx = -INFINITY, sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN; c += 64) {
        float v[64];
        tmem_ld32(t_acc + c, *reinterpret_cast<float(*)[32]>(&v[0]));
        tmem_ld32(t_acc + c + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
        tmem_wait_ld();
        if (c + 64 >= BN) {  // the tile is in registers: hand the accumulator back
          tc_fence_before();
          mbar_arrive(&acc_empty[e]);
        }
        float cm = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          v[i] = c + i < valid ? v[i] * kLog2e : -INFINITY;
          cm = fmaxf(cm, v[i]);
        }
        const float mn = fmaxf(mx, cm);
        if (mn != -INFINITY) {
          float acc = mx == -INFINITY ? 0.f : sum * exp2f(mx - mn);
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            float ex;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"(v[i] - mn));
            acc += ex;
          }
          sum = acc;
          mx = mn;
        }
        if ((c + 64) % kLsHalf == 0) {  // one partial per 128 vocab columns
          const int64_t h0 = col0 + c + 64 - kLsHalf;  // first column of this half (halves past the vocab are not stored)
          if (row < p.rows && h0 < p.vocab) p.part[h0 / kLsHalf * p.rows_pad + row] = make_float2(mx, sum);
          mx = -INFINITY;
          sum = 0.f;
        }
      }
      ++cnt;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tbase, 512);
}

// One CTA per scored (row, target) pair: the row's LSE (natural log) from its
// per-128-column partials (each thread folds a strided share, then warp and
// block combines), and the target logit as a dot product of the same bf16
// operands with fp32 accumulation; out = logit - LSE.  A whole CTA per pair
// keeps the ~1,000 partial loads of a Llama-vocab row in flight together
// (a warp per pair took ~15 us at batch 1, latency-bound).
__device__ __forceinline__ void lse_fold(float &m, float &s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn != -INFINITY) {
    s = (m == -INFINITY ? 0.f : s * exp2f(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * exp2f(m2 - mn));
    m = mn;
  }
}

__global__ void __launch_bounds__(256) label_pair_logprob_kernel(const float2 *part, int n_tiles, int64_t rows_pad,
                                                                 const __nv_bfloat16 *x, const __nv_bfloat16 *w,
                                                                 int64_t d, const int64_t *pair_row,
                                                                 const int32_t *pair_target, int64_t n_pairs,
                                                                 float *out) {
  __shared__ float red_m[8], red_s[8], red_dot[8];
  const int64_t i = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row = pair_row[i];
  const int64_t tgt = pair_target[i];
  float m = -INFINITY, s = 0.f;
  for (int j = threadIdx.x; j < n_tiles; j += blockDim.x) {
    const float2 q = part[(int64_t)j * rows_pad + row];
    lse_fold(m, s, q.x, q.y);
  }
  const __nv_bfloat16 *xr = x + row * d, *wr = w + tgt * d;
  float acc = 0.f;
  for (int64_t c = (int64_t)threadIdx.x * 8; c < d; c += (int64_t)blockDim.x * 8) {
    const uint4 a = *reinterpret_cast<const uint4 *>(xr + c), b = *reinterpret_cast<const uint4 *>(wr + c);
    const __nv_bfloat162 *a2 = reinterpret_cast<const __nv_bfloat162 *>(&a);
    const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fa = __bfloat1622float2(a2[k]), fb = __bfloat1622float2(b2[k]);
      acc = fmaf(fa.x, fb.x, acc);
      acc = fmaf(fa.y, fb.y, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lse_fold(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
  }
  if (lane == 0) red_m[wid] = m, red_s[wid] = s, red_dot[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = -INFINITY, ss = 0.f, dot = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      lse_fold(mm, ss, red_m[k], red_s[k]);
      dot += red_dot[k];
    }
    out[i] = dot - (mm + log2f(ss)) * 0.69314718055994531f;
  }
}

static int num_sms_ls() {
  static thread_local int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, bool NARROW>
static int launch_lse(int grid, const CUtensorMap *maps, const LsParams &p, cudaStream_t s) {
  using C = LsCfg<BN, NARROW>;
  static thread_local bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(label_lse_kernel<BN, NARROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::Smem);
    if (e != cudaSuccess) return set_error(DBSA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  label_lse_kernel<BN, NARROW><<<grid, kLsThreads, C::Smem, s>>>(maps[0], maps[1], p);
  return check_launch("label_lse");
}

}  // namespace dbsa

extern "C" int dbsa_label_score(const DbsaLabelScoreArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_label_score: null args");
  const DbsaLabelScoreArgs &a = *args;
  if (a.n_pairs < 0 || a.rows < 0) return set_error(DBSA_ERR_VALIDATION, "dbsa_label_score: negative size");
  if (a.n_pairs == 0) return DBSA_OK;
  if (a.rows == 0 || a.vocab <= 0) return set_error(DBSA_ERR_VALIDATION, "dbsa_label_score: pairs without rows");
  if (a.d <= 0 || a.d % 8)  // 16-byte TMA row strides; the K tail of the last 64-slice is TMA zero fill
    return set_error(DBSA_ERR_CONFIG, "dbsa_label_score: d %lld not a multiple of 8", (long long)a.d);
  if (!a.x || !a.w || !a.workspace || !a.pair_row || !a.pair_target || !a.out)
    return set_error(DBSA_ERR_VALIDATION, "dbsa_label_score: null pointer argument");
  LsParams p;
  p.rows = a.rows;
  p.m_tiles = (int)((a.rows + 127) / 128);
  p.rows_pad = (int64_t)p.m_tiles * 128;
  p.m_pairs = (p.m_tiles + 1) / 2;
  p.vocab = a.vocab;
  // batch-1 shapes (one M tile): 128-column vocab tiles, a one-M-tile stage
  // layout with a deeper ring, and x loaded only for its real rows
  const bool narrow = p.m_tiles == 1;
  const int bn = narrow ? 128 : 256;
  p.n_tiles = (int)((a.vocab + bn - 1) / bn);
  p.k_steps = (int)((a.d + kLsBK - 1) / kLsBK);
  p.n_work = p.m_pairs * p.n_tiles;
  p.part = reinterpret_cast<float2 *>(a.workspace);
  CUtensorMap maps[2];
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)a.rows};
    cuuint64_t strides[1] = {(cuuint64_t)a.d * 2};
    p.x_box_rows = narrow ? (int)((a.rows + 15) / 16 * 16) : 128;
    cuuint32_t box[2] = {(cuuint32_t)kLsBK, (cuuint32_t)p.x_box_rows};
    cuuint32_t estr[2] = {1, 1};
    if (!encode_tiled_bf16(&maps[0], a.x, 2, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B))
      return DBSA_ERR_CUDA;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)a.vocab};
    cuuint64_t strides[1] = {(cuuint64_t)a.d * 2};
    cuuint32_t box[2] = {(cuuint32_t)kLsBK, (cuuint32_t)bn};
    cuuint32_t estr[2] = {1, 1};
    if (!encode_tiled_bf16(&maps[1], a.w, 2, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B))
      return DBSA_ERR_CUDA;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = p.n_work < num_sms_ls() ? p.n_work : num_sms_ls();
  if (int rc = narrow ? launch_lse<128, true>(grid, maps, p, s) : launch_lse<256, false>(grid, maps, p, s)) return rc;
  label_pair_logprob_kernel<<<(unsigned)a.n_pairs, 256, 0, s>>>(
      p.part, (int)((a.vocab + kLsHalf - 1) / kLsHalf), p.rows_pad, reinterpret_cast<const __nv_bfloat16 *>(a.x),
      reinterpret_cast<const __nv_bfloat16 *>(a.w), a.d, a.pair_row, a.pair_target, a.n_pairs, a.out);
  return check_launch("label_pair_logprob");
}
