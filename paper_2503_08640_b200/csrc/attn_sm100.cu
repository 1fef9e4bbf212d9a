// attn_sm100.cu -- K1 (stage-1 block-sparse prefill) and K3 (stage-2 split-KV
// query attention) of DBSA as ONE warp-specialised tcgen05/TMEM/TMA kernel.
//
// Reference semantics: kernels.masked_attention (kernels.py:73-100) called per
// (layer, kv head) from model._forward (model.py:327-351): q rotated at its own
// position and scaled by 1/sqrt(hd), softmax over the allowed keys only
// (masked entries exactly 0), then P.V.  Here a CTA owns up to 128*NUM_M query
// rows of one kv head (GQA heads packed token-major, the stacking of
// model.py:338-342) and streams the keys of a SEGMENT LIST through an online
// softmax, so the block-sparse mask of masks.block_mask_rows (masks.py:164-177)
// is never materialised:
//   stage 1: segments = [sink, prev-j groups] (FULL) + the group itself (SELF,
//            causal)                       -- pipeline.encode_blocks (pipeline.py:203-229)
//   stage 2: segments = selected chunks (FULL, each with its query-side RoPE
//            shift) + the query/label tokens (SELF, causal tree)
//                                          -- Runner.infer / score_label (pipeline.py:410-421, model.py:420-443)
//
// Roles (warp-specialised, one CTA per work item; FA4-style ping-pong):
//   warp 0      TMA producer: K tile [128 keys x HDP] into a K ring, V^T tile
//               [HDP x 128 keys] into a V ring (K runs one tile ahead of V)
//   warp 1      MMA warp (converged; one elected lane issues): per M tile m,
//               O(m) += P(m, j-1) V(j-1)  (A = P from TMEM)  then
//               S(m) = Q(m) K(j)^T        (A = Q from smem)
//   warp 2      TMEM allocator
//   warps 4..   softmax warpgroups, one per 128-row M tile, one row per thread:
//               Q prologue (load + RoPE + per-segment shift, swizzled
//               st.shared), S from TMEM, online softmax with lazy O rescale,
//               P (bf16) back into TMEM over S, epilogue.
// With two M tiles the tensor pipe works on tile m' while the softmax warps
// of tile m run, and vice versa.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"
#include "sm100_ptx.cuh"

namespace dbsa {

constexpr int kBN = 128;  // keys per tile
// lazy O rescale: only when a row's max grows by more than 2^DBSA_RESCALE_LOG2
// (P <= 2^DBSA_RESCALE_LOG2 stays exact in bf16's exponent range)
// Q staging: load iterations batched per round trip (1 = one at a time)
#ifndef DBSA_EPI_COLS
#define DBSA_EPI_COLS 128  // O columns per epilogue TMEM round trip
#endif
// one exp2 pair in four on the FMA pipe (polynomial) instead of MUFU (1)
#ifndef DBSA_POLY_EXP
#define DBSA_POLY_EXP 1
#endif
#ifndef DBSA_QSTAGE_BATCH
#define DBSA_QSTAGE_BATCH 8
#endif
#ifndef DBSA_RESCALE_LOG2
#define DBSA_RESCALE_LOG2 8.f
#endif

// Profiling build only (-DDBSA_STAMPS, tools/build_variant.py + tools/stamps.py):
// per-tile clock stamps of CTA 0 for the first 256 key tiles of the two-tile
// kernel, read back with dbsa_debug_stamps.
#ifdef DBSA_STAMPS
#ifndef DBSA_STAMP_CTA
#define DBSA_STAMP_CTA 0
#endif
__device__ long long g_stamps[256 * 12];
__device__ long long g_wstamps[256 * 12];  // per work of CTA 0: m*4 + {softmax done, Q staged, O full, epilogue done}
#define WSTAMP(slot, w)                                                       \
  do {                                                                        \
    if (blockIdx.x == DBSA_STAMP_CTA && (w) < 256) g_wstamps[(w) * 12 + (slot)] = clock64(); \
  } while (0)
#define STAMP(slot, j)                                                         \
  do {                                                                         \
    if (blockIdx.x == DBSA_STAMP_CTA && (j) < 256) g_stamps[(j) * 12 + (slot)] = clock64(); \
  } while (0)
// per-CTA globaltimer (ns) milestones of the last launch: 0 entry, 1 setup done,
// 2 first Q staged (m0), 3 MMA saw the first K tile, 4 last O committed,
// 5 / 6 last epilogue done (m0 / m1), 7 exit
__device__ unsigned long long g_cta[1024 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CSTAMP(slot)                                                    \
  do {                                                                  \
    if (blockIdx.x < 1024) g_cta[blockIdx.x * 8 + (slot)] = gtimer(); \
  } while (0)
#else
#define CSTAMP(slot) \
  do {               \
  } while (0)
#define STAMP(slot, j) \
  do {               \
  } while (0)
#define WSTAMP(slot, w) \
  do {                \
  } while (0)
#endif

template <int HDP, int NUM_M>
struct AttnCfg {
  static constexpr int QSW = HDP >= 64 ? 128 : HDP * 2;  // swizzle width of Q / K rows (bytes)
  static constexpr int KATOM = HDP >= 64 ? 64 : HDP;     // head-dim elements per K atom column
  static constexpr int NATOM = HDP / KATOM;              // atom columns along head_dim
  static constexpr int Q_BYTES = 128 * HDP * 2;
  static constexpr int K_BYTES = kBN * HDP * 2;
  static constexpr int V_BYTES = HDP * kBN * 2;  // V^T: HDP rows, 2 atoms of 64 keys (128B swizzle)
  static constexpr int FIXED = NUM_M * Q_BYTES;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int AVAIL = 232448 - 1024 /*align slack*/ - BAR_BYTES - FIXED;
  static constexpr int PAIRS = AVAIL / (K_BYTES + V_BYTES) > 4 ? 4 : AVAIL / (K_BYTES + V_BYTES);
  static constexpr int KST = PAIRS + ((AVAIL - PAIRS * (K_BYTES + V_BYTES)) >= K_BYTES ? 1 : 0);
  static constexpr int VST = PAIRS;
  static constexpr int SMEM = FIXED + KST * K_BYTES + VST * V_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 128 + 128 * NUM_M;
  static constexpr int REG_CTRL = 56, REG_SOFTMAX = 224;  // 128*56 + 256*224 <= 64K (NUM_M == 2)
  static constexpr int TMEM_NEED = NUM_M * (HDP + kBN);  // O(m) + S/P(m)
  static constexpr int TMEM_COLS =
      TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(PAIRS >= 2, "not enough shared memory for a 2-stage pipeline");
};

struct AttnParams {
  const __nv_bfloat16 *q;
  int64_t q_tok_stride;
  const int32_t *tok_pos;
  const int32_t *tok_lo;
  const float2 *rope;
  const __half2 *rope_h;  // optional fp16 copy of rope: the Q staging's rotation table
  int64_t rope_rows;
  int32_t n_heads, n_kv_heads, head_dim, gs;
  uint32_t gs_magic;  // ceil(2^32 / gs) for gs > 1 (0 for gs == 1): row / gs by one IMAD.HI (rows < 2^16)
  float scale_log2;
  const DbsaAttnWork *works;
  int32_t n_works;
  const DbsaAttnSeg *segs;
  __nv_bfloat16 *out;
  int64_t out_tok_stride;
  void *part_o;  // fp32, or bf16 if part_bf16
  float *part_lse;
  const DbsaRowMap *row_map;
  int part_bf16;  // out_mode DBSA_OUT_MAPPED works: q_tok0 indexes this map
  int dbg;  // profiling switches (DBSA_DEBUG_MODE): 1 = skip softmax math, 2 = skip MMAs, 4 = skip TMA loads,
            // 8 = skip epilogue stores, 16 = skip Q staging (two-tile kernel)
  unsigned long long *pair_count;  // optional: (row, key) pairs that entered the softmax (all heads)
  const int32_t *cta_works;        // optional: CTA b runs works [cta_works[b], cta_works[b+1])
  int64_t part_chunk_rows;         // > 0: bf16 partials in 16-column chunks (DbsaAttnArgs.part_chunk_rows)
  int pdl_early;                   // DbsaAttnArgs.pdl_early_q: only the producer waits for the predecessor
};

// This CTA's works: [begin, end) with stride `step` (round-robin over the grid,
// or the host-packed contiguous range of AttnParams.cta_works).
struct WorkRange {
  int begin, end, step;
};
__device__ __forceinline__ WorkRange cta_work_range(const AttnParams &p) {
  if (p.cta_works) return {p.cta_works[blockIdx.x], p.cta_works[blockIdx.x + 1], 1};
  return {(int)blockIdx.x, p.n_works, (int)gridDim.x};
}

// Pair counter (DbsaAttnArgs.pair_count): the unmasked entries of the S row a
// thread just masked, i.e. exactly the keys its softmax takes in.
__device__ __forceinline__ uint32_t count_visible(const float (&x)[kBN]) {
  uint32_t n = 0;
#pragma unroll
  for (int c = 0; c < kBN; ++c) n += x[c] != -INFINITY ? 1u : 0u;
  return n;
}
__device__ __forceinline__ void flush_pair_count(unsigned long long *dst, uint32_t n) {
  unsigned long long v = n;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Bits i of a 32-bit word with lo <= i < hi (lo, hi clamped to [0, 32]).
__device__ __forceinline__ uint32_t range_bits(int lo, int hi) {
  lo = min(max(lo, 0), 32);
  hi = min(max(hi, 0), 32);
  const uint32_t below_hi = hi >= 32 ? 0xffffffffu : (1u << hi) - 1u;
  const uint32_t below_lo = lo >= 32 ? 0xffffffffu : (1u << lo) - 1u;
  return below_hi & ~below_lo;
}

// 2^x for a pair on the FMA/ALU pipes (FA4's MUFU offload): round to the
// nearest integer with the 1.5*2^23 trick, a cubic for 2^f on f in [-0.5, 0.5]
// (rel. error < 7e-4, below bf16's 2^-8 resolution of P), integer part added
// to the exponent field.  Inputs are clamped at -126 (masked -inf -> ~1e-38).
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = fadd2(x, magic);
  const float2 r = fadd2(t, make_float2(-12582912.f, -12582912.f));  // round(x)
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);              // x - round(x)
  float2 q = ffma2(f, make_float2(0.0555041087f, 0.0555041087f), make_float2(0.2402265070f, 0.2402265070f));
  q = ffma2(q, f, make_float2(0.6931471806f, 0.6931471806f));
  q = ffma2(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Rotate this thread's query row (token t, head) at rope position `pos`,
// composed with the optional per-segment shift, and write it zero-padded to
// HDP into the swizzled K-major Q tile.  (model.rope_rotate_heads,
// model.py:222-239: pair (x_i, x_{i+hd/2}).)  Vector path: 16-byte loads of
// 8 bf16 from each half plus the matching (cos, sin) pairs, all issued before
// use so one row costs a few memory round trips, not one per element.
template <int HDP>
__device__ __forceinline__ void load_q_row(const AttnParams &p, uint8_t *q_tile, int row, bool valid,
                                           int t, int head, int rope_row) {
  constexpr int QSW = AttnCfg<HDP, 1>::QSW;
  const int hd = p.head_dim, half = hd >> 1;
  auto put = [&](int c, const float (&o)[8]) {
    const int atom = c / (QSW / 16), cc = c % (QSW / 16);
    uint4 *d = reinterpret_cast<uint4 *>(q_tile + atom * 128 * QSW + swz_offset(row, cc, QSW));
    *d = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
  };
  if (!valid) {
    const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < HDP / 8; ++c) put(c, z);
    return;
  }
  const __nv_bfloat16 *src = p.q + (int64_t)t * p.q_tok_stride + (int64_t)head * hd;
  const float2 *rp = p.rope + (int64_t)rope_row * half;
  if (HDP >= 32 && hd == HDP && (p.q_tok_stride & 7) == 0) {
    // fast path: full-width head, every 8-element chunk lies in one half, 16-byte
    // aligned rows.  Two passes, each issuing all of its loads before any use.
    constexpr int NCH = HDP / 16;           // 8-pair chunks per half
    constexpr int PASS = NCH >= 4 ? NCH / 2 : NCH;
#pragma unroll
    for (int c0 = 0; c0 < NCH; c0 += PASS) {
      uint4 lo4[PASS], hi4[PASS];
      float4 cs4[PASS][4];
#pragma unroll
      for (int u = 0; u < PASS; ++u) {
        const int i0 = (c0 + u) * 8;  // pair index of this chunk
        lo4[u] = *reinterpret_cast<const uint4 *>(src + i0);
        hi4[u] = *reinterpret_cast<const uint4 *>(src + half + i0);
#pragma unroll
        for (int v = 0; v < 4; ++v) cs4[u][v] = reinterpret_cast<const float4 *>(rp + i0)[v];
      }
#pragma unroll
      for (int u = 0; u < PASS; ++u) {
        const __nv_bfloat16 *lo = reinterpret_cast<const __nv_bfloat16 *>(&lo4[u]);
        const __nv_bfloat16 *hi = reinterpret_cast<const __nv_bfloat16 *>(&hi4[u]);
        const float *cs = reinterpret_cast<const float *>(cs4[u]);
        float a[8], b[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float c = cs[2 * j], sn = cs[2 * j + 1];
          const float x = __bfloat162float(lo[j]), y = __bfloat162float(hi[j]);
          a[j] = x * c - y * sn;
          b[j] = x * sn + y * c;
        }
        put(c0 + u, a);
        put(NCH + c0 + u, b);
      }
    }
    return;
  }
#pragma unroll 1
  for (int c = 0; c < HDP / 8; ++c) {
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = c * 8 + j;
      float val = 0.f;
      if (e < hd) {
        const int i = e < half ? e : e - half;
        const float lo = __bfloat162float(src[i]);
        const float hi = __bfloat162float(src[i + half]);
        const float2 cs = rp[i];
        val = e < half ? (lo * cs.x - hi * cs.y) : (lo * cs.y + hi * cs.x);
      }
      o[j] = val;
    }
    put(c, o);
  }
}

// Where row r of work w comes from and where its result goes.  Rows are
// token-major GQA packing: work-local token r / gs, head r % gs of the work's
// kv head.  Plain works read tokens q_tok0.. and rotate at tok_pos - shift of
// the current segment; DBSA_OUT_MAPPED works (chunk-major stage 2: rows of many
// queries against ONE chunk) take token, rope row and partial slot from the
// row map, so each query row carries its own re-positioning delta.
struct RowRef {
  bool valid;
  int t, head, rope_row;
  int64_t part_row;
};
// r / gs and r % gs for a row index r < 2^16 (exact: the magic's error term
// r * (magic * gs - 2^32) / 2^32 stays below 1 / gs)
__device__ __forceinline__ int gs_div(const AttnParams &p, int r) {
  return p.gs_magic ? (int)__umulhi((uint32_t)r, p.gs_magic) : r;
}
__device__ __forceinline__ RowRef row_ref(const AttnParams &p, const DbsaAttnWork &w, int r) {
  RowRef x;
  x.valid = r < w.n_tok * p.gs;
  const int q = gs_div(p, r);
  const int i = x.valid ? q : 0, hl = x.valid ? r - q * p.gs : 0;
  x.head = w.kv_head * p.gs + hl;
  if (w.out_mode == DBSA_OUT_MAPPED) {
    const DbsaRowMap e = p.row_map[w.q_tok0 + i];
    x.t = e.tok;
    x.rope_row = e.rope_row;
    x.part_row = w.part_row0 + (int64_t)e.part_tok * p.gs + hl;
  } else {
    x.t = w.q_tok0 + i;
    x.rope_row = p.tok_pos[x.t] - (w.seg_end > w.seg_begin ? p.segs[w.seg_begin].shift : 0);
    x.part_row = w.part_row0 + r;
  }
  return x;
}

// Columns [c0, c0 + CW) of one epilogue row, normalised by 1/l: bf16 into
// out, or a bf16 / fp32 partial.  32-byte stores (st.global.v8, whole
// sectors) on full-width aligned rows, element stores otherwise.
template <int HDP, int CW, bool CM = false>
__device__ __forceinline__ void epilogue_cols(const AttnParams &p, const float (&o)[CW], int c0, int t, int head,
                                              int out_mode, int64_t part_row, float inv_l) {
  const int hd = p.head_dim;
  const bool full = hd == HDP;
  if (CM || (out_mode != DBSA_OUT_BF16 && p.part_chunk_rows > 0)) {
    // 16-column chunk layout: this row's chunk k at ((c0/16 + k) * chunk_rows + part_row) * 16
    __nv_bfloat16 *base = reinterpret_cast<__nv_bfloat16 *>(p.part_o) + part_row * 16;
    const float2 il = make_float2(inv_l, inv_l);
#pragma unroll
    for (int c = 0; c < CW; c += 16) {
      if (c0 + c >= hd) break;
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 v = fmul2(make_float2(o[c + 2 * i], o[c + 2 * i + 1]), il);
        w[i] = pack_bf16(v.x, v.y);
      }
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(
                       base + (int64_t)((c0 + c) >> 4) * p.part_chunk_rows * 16),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                   : "memory");
    }
    return;
  }
  if (out_mode == DBSA_OUT_BF16 || p.part_bf16) {
    __nv_bfloat16 *dst = out_mode == DBSA_OUT_BF16
                             ? p.out + (int64_t)t * p.out_tok_stride + (int64_t)head * hd + c0
                             : reinterpret_cast<__nv_bfloat16 *>(p.part_o) + part_row * (int64_t)hd + c0;
    if (CW >= 16 && full && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
      const float2 il = make_float2(inv_l, inv_l);
#pragma unroll
      for (int c = 0; c < CW; c += 16) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 v = fmul2(make_float2(o[c + 2 * i], o[c + 2 * i + 1]), il);
          w[i] = pack_bf16(v.x, v.y);
        }
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + c), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
      }
      return;
    }
#pragma unroll
    for (int c = 0; c < CW; c += 8) {
      if (c0 + c + 8 <= hd && (hd & 7) == 0) {
        *reinterpret_cast<uint4 *>(dst + c) =
            make_uint4(pack_bf16(o[c] * inv_l, o[c + 1] * inv_l), pack_bf16(o[c + 2] * inv_l, o[c + 3] * inv_l),
                       pack_bf16(o[c + 4] * inv_l, o[c + 5] * inv_l), pack_bf16(o[c + 6] * inv_l, o[c + 7] * inv_l));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (c0 + c + i < hd) dst[c + i] = __float2bfloat16(o[c + i] * inv_l);
      }
    }
    return;
  }
  float *dst = reinterpret_cast<float *>(p.part_o) + part_row * (int64_t)hd + c0;
  if (CW >= 8 && full && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
    for (int c = 0; c < CW; c += 8)
      asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + c), "f"(o[c] * inv_l),
                   "f"(o[c + 1] * inv_l), "f"(o[c + 2] * inv_l), "f"(o[c + 3] * inv_l), "f"(o[c + 4] * inv_l),
                   "f"(o[c + 5] * inv_l), "f"(o[c + 6] * inv_l), "f"(o[c + 7] * inv_l)
                   : "memory");
    return;
  }
#pragma unroll
  for (int c = 0; c < CW; c += 4) {
    if (c0 + c + 4 <= hd && (hd & 3) == 0) {
      *reinterpret_cast<float4 *>(dst + c) =
          make_float4(o[c] * inv_l, o[c + 1] * inv_l, o[c + 2] * inv_l, o[c + 3] * inv_l);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (c0 + c + i < hd) dst[c + i] = o[c + i] * inv_l;
    }
  }
}

// Epilogue of one row (thread = TMEM lane = row): the O row from TMEM in
// chunks of DBSA_EPI_COLS columns (default the whole row: one round trip),
// normalised by 1/l, then either bf16 into out or a partial + natural-log LSE.
// Warp-collective (tcgen05.ld): every lane calls it, invalid rows store nothing.
template <int HDP, bool CM = false>
__device__ __forceinline__ void epilogue_row(const AttnParams &p, uint32_t t_o, bool valid, int t, int head,
                                             int out_mode, int64_t part_row, float l_sum, float m_used) {
  constexpr int CW = HDP > DBSA_EPI_COLS ? DBSA_EPI_COLS : HDP;
  const bool store = valid && (CM || !(p.dbg & 8));
  const bool empty = !(l_sum > 0.f);  // no visible key (e.g. a shard without chunks): O = 0, LSE = -inf
  const float inv_l = empty ? 0.f : 1.f / l_sum;
#pragma unroll
  for (int c0 = 0; c0 < HDP; c0 += CW) {
    float o[CW];
    if constexpr (CW >= 32) {
#pragma unroll
      for (int c = 0; c < CW; c += 32) tmem_ld32(t_o + c0 + c, *reinterpret_cast<float(*)[32]>(&o[c]));
    } else {
      tmem_ld16(t_o + c0, *reinterpret_cast<float(*)[16]>(&o[0]));
    }
    tmem_wait_ld();
    if (store) epilogue_cols<HDP, CW, CM>(p, o, c0, t, head, out_mode, part_row, inv_l);
  }
  // natural-log LSE of the scaled scores: (m + log2 l) * ln 2
  if (store && out_mode != DBSA_OUT_BF16)
    p.part_lse[part_row] = empty ? -INFINITY : (m_used + log2f(l_sum)) * 0.69314718055994531f;
}

// Row refs of the coop Q staging: lane (c, rsub) of warp q4 stages rows
// q4 * 32 + it * RPI + rsub, it < NIT, of M tile m.
template <int HDP>
struct QRefs {
  static constexpr int NCH = HDP / 16;  // chunk pairs per row == lanes per row
  static constexpr int RPI = 32 / NCH;  // rows per warp instruction
  static constexpr int NIT = 32 / RPI;  // iterations for the warp's 32 rows
  int tok[NIT], rrow[NIT];
  int head0;  // first query head of the work's kv head; row r is head head0 + r % gs
};

// Phase A of the coop staging: every iteration's (token, head, rope row), so
// the row-map / tok_pos round trip is paid once, not once per iteration.  The
// work boundary issues it before the epilogue so its latency hides there.
template <int HDP>
__device__ __forceinline__ void stage_refs_coop(const AttnParams &p, const DbsaAttnWork &w, int m, int q4, int lane,
                                                bool restage, int shift, QRefs<HDP> &x) {
  constexpr int NCH = QRefs<HDP>::NCH, RPI = QRefs<HDP>::RPI, NIT = QRefs<HDP>::NIT;
  const int rsub = lane / NCH;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const RowRef rr = row_ref(p, w, m * 128 + q4 * 32 + it * RPI + rsub);
    x.tok[it] = rr.valid ? rr.t : -1;
    x.rrow[it] = rr.rope_row;
  }
  x.head0 = w.kv_head * p.gs;
  if (restage) {
#pragma unroll
    for (int it = 0; it < NIT; ++it)
      if (x.tok[it] >= 0) x.rrow[it] = p.tok_pos[x.tok[it]] - shift;
  }
}

// Phase B: q chunk pairs + their (cos, sin), rotate, swizzled 16-byte stores
// into the Q tile.  HALF: the fp16 rotation table (AttnParams.rope_h).
template <int HDP, bool HALF, int QBATCH = DBSA_QSTAGE_BATCH>
__device__ __forceinline__ void stage_load_coop(const AttnParams &p, uint8_t *q_tile, int m, int q4, int lane,
                                                const QRefs<HDP> &x, int sw = -1) {
  constexpr int QSW = AttnCfg<HDP, 1>::QSW;
  constexpr int NCH = QRefs<HDP>::NCH, RPI = QRefs<HDP>::RPI, NIT = QRefs<HDP>::NIT;
  const int c = lane % NCH, rsub = lane / NCH, half = HDP / 2;
  const int(&tok)[NIT] = x.tok;
  const int(&rrow)[NIT] = x.rrow;
  int head[NIT];
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int rr = m * 128 + q4 * 32 + it * RPI + rsub;
    head[it] = x.head0 + rr - gs_div(p, rr) * p.gs;
  }
#if DBSA_QSTAGE_BATCH > 1
  // phase B, batched: the loads of QB iterations are issued before any of
  // them is used, so QB round trips overlap (QB x 24 registers in flight)
  constexpr int QB = QBATCH < NIT ? QBATCH : NIT;
  static_assert(NIT % QB == 0, "DBSA_QSTAGE_BATCH must divide the staging iterations");
#pragma unroll
  for (int i0 = 0; i0 < NIT; i0 += QB) {
    uint4 lo4[QB], hi4[QB];
    float4 cs4[QB][4];  // float32 table: (cos, sin) of 8 pairs
    uint4 rh4[QB][2];   // fp16 table
#pragma unroll
    for (int k = 0; k < QB; ++k) {
      const int it = i0 + k;
      const int tk = tok[it] >= 0 ? tok[it] : tok[0] >= 0 ? tok[0] : 0;  // invalid rows read a safe row
      const int hk = tok[it] >= 0 ? head[it] : 0, rk = tok[it] >= 0 ? rrow[it] : 0;
      const __nv_bfloat16 *src = p.q + (int64_t)tk * p.q_tok_stride + (int64_t)hk * HDP + c * 8;
      const float4 *rp = reinterpret_cast<const float4 *>(p.rope + (int64_t)rk * half + c * 8);
      lo4[k] = __ldg(reinterpret_cast<const uint4 *>(src));
      hi4[k] = __ldg(reinterpret_cast<const uint4 *>(src + half));
      if constexpr (HALF) {
        // fp16 (cos, sin) of the chunk's 8 pairs: 32 contiguous bytes
        const uint4 *rh = reinterpret_cast<const uint4 *>(p.rope_h + (int64_t)rk * half + c * 8);
        rh4[k][0] = __ldg(rh);
        rh4[k][1] = __ldg(rh + 1);
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) cs4[k][v] = __ldg(rp + v);
      }
    }
#ifdef DBSA_STAMPS
    if (sw >= 0 && m == 0 && q4 == 0 && lane == 0 && i0 == 0) {  // the first batch's loads are back
      asm volatile("" ::"r"(lo4[0].x), "r"(hi4[0].x), "r"(rh4[0][0].x), "r"(rh4[0][1].x));
      WSTAMP(11, sw);
    }
#endif
#pragma unroll
    for (int k = 0; k < QB; ++k) {
      const int it = i0 + k;
      const int row = q4 * 32 + it * RPI + rsub;
      const __nv_bfloat16 *lo = reinterpret_cast<const __nv_bfloat16 *>(&lo4[k]);
      const __nv_bfloat16 *hi = reinterpret_cast<const __nv_bfloat16 *>(&hi4[k]);
      float cs[16];
      if constexpr (HALF) {
        const __half2 *h2 = reinterpret_cast<const __half2 *>(rh4[k]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 f = __half22float2(h2[j]);
          cs[2 * j] = f.x;
          cs[2 * j + 1] = f.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) cs[j] = reinterpret_cast<const float *>(cs4[k])[j];
      }
      // rotate two pairs per FFMA2 / FMUL2.  A row past the work's rows keeps
      // the (finite) q of the safe row it read: its scores feed only its own
      // softmax row, whose O is never stored
      float a[8], b[8];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 xl = make_float2(__bfloat162float(lo[j]), __bfloat162float(lo[j + 1]));
        const float2 yh = make_float2(__bfloat162float(hi[j]), __bfloat162float(hi[j + 1]));
        const float2 cc = make_float2(cs[2 * j], cs[2 * j + 2]), sn = make_float2(cs[2 * j + 1], cs[2 * j + 3]);
        const float2 av = ffma2(xl, cc, fmul2(yh, make_float2(-sn.x, -sn.y)));
        const float2 bv = ffma2(xl, sn, fmul2(yh, cc));
        a[j] = av.x;
        a[j + 1] = av.y;
        b[j] = bv.x;
        b[j + 1] = bv.y;
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float(&o)[8] = hh ? b : a;
        const int ch = hh * NCH + c;
        const int atom = ch / (QSW / 16), cc = ch % (QSW / 16);
        uint4 *d = reinterpret_cast<uint4 *>(q_tile + atom * 128 * QSW + swz_offset(row, cc, QSW));
        *d = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
      }
    }
  }
#else
  // phase B: q chunk pair + its (cos, sin), rotate, swizzled 16-byte stores
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int row = q4 * 32 + it * RPI + rsub;
    float a[8], b[8];
    if (tok[it] >= 0) {
      const __nv_bfloat16 *src = p.q + (int64_t)tok[it] * p.q_tok_stride + (int64_t)head[it] * HDP + c * 8;
      const float4 *rp = reinterpret_cast<const float4 *>(p.rope + (int64_t)rrow[it] * half + c * 8);
      const uint4 lo4 = *reinterpret_cast<const uint4 *>(src);
      const uint4 hi4 = *reinterpret_cast<const uint4 *>(src + half);
      float4 cs4[4];
      if constexpr (HALF) {
        const __half2 *h2 = p.rope_h + (int64_t)rrow[it] * half + c * 8;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float2 f0 = __half22float2(h2[2 * v]), f1 = __half22float2(h2[2 * v + 1]);
          cs4[v] = make_float4(f0.x, f0.y, f1.x, f1.y);
        }
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) cs4[v] = rp[v];
      }
      const __nv_bfloat16 *lo = reinterpret_cast<const __nv_bfloat16 *>(&lo4);
      const __nv_bfloat16 *hi = reinterpret_cast<const __nv_bfloat16 *>(&hi4);
      const float *cs = reinterpret_cast<const float *>(cs4);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float cc = cs[2 * j], sn = cs[2 * j + 1];
        const float xl = __bfloat162float(lo[j]), yh = __bfloat162float(hi[j]);
        a[j] = xl * cc - yh * sn;
        b[j] = xl * sn + yh * cc;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = b[j] = 0.f;
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float(&o)[8] = hh ? b : a;
      const int ch = hh * NCH + c;
      const int atom = ch / (QSW / 16), cc = ch % (QSW / 16);
      uint4 *d = reinterpret_cast<uint4 *>(q_tile + atom * 128 * QSW + swz_offset(row, cc, QSW));
      *d = make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
    }
  }
#endif
}

// Stage the 128-row Q tile m of work w cooperatively: a row's 16-byte chunk
// pairs (c, c + HDP/16) -- the two rotary halves -- go to HDP/16 consecutive
// lanes, so one warp instruction reads whole 128-byte lines of q and of the
// rope table for 32 / (HDP/16) rows instead of one 16-byte piece of 32
// different rows (the thread-per-row form costs ~32 L1 wavefronts per
// instruction).  restage: rope row tok_pos - shift (a plain work's next
// segment); otherwise the row's own (row_ref) rope row.  Full-width heads only
// (hd == HDP, 16-byte aligned rows); the caller falls back to load_q_row.
template <int HDP, bool HALF, int QBATCH = DBSA_QSTAGE_BATCH>
__device__ __forceinline__ void stage_q_coop(const AttnParams &p, const DbsaAttnWork &w, int m, uint8_t *q_tile,
                                             int q4, int lane, bool restage, int shift, int sw = -1) {
  QRefs<HDP> x;
  stage_refs_coop<HDP>(p, w, m, q4, lane, restage, shift, x);
#ifdef DBSA_STAMPS
  if (sw >= 0 && m == 0 && q4 == 0 && lane == 0) {  // the row refs are back
    asm volatile("" ::"r"(x.tok[0]), "r"(x.rrow[0]));
    WSTAMP(10, sw);
  }
#endif
  stage_load_coop<HDP, HALF, QBATCH>(p, q_tile, m, q4, lane, x, sw);
}

// CM: the chunk-major specialisation (DbsaAttnArgs.one_seg_partials): every work
// has one segment and writes a partial, partials are bf16 in the 16-column chunk
// layout, Q is staged cooperatively with the fp16 rotation table, no pair
// counter and no profiling switches.  The paths it cannot take are compiled
// out, which leaves a third of the generic kernel's code to fetch at every
// work boundary (chunk-major C3 K3 1.184 -> 1.158 ms, C4 0.604 -> 0.582).
template <int HDP, int NUM_M, bool CM = false>
__global__ void __launch_bounds__(AttnCfg<HDP, NUM_M>::THREADS, 1)
    dbsa_attn_kernel(const __grid_constant__ CUtensorMap tm_k0, const __grid_constant__ CUtensorMap tm_v0,
                     const __grid_constant__ CUtensorMap tm_k1, const __grid_constant__ CUtensorMap tm_v1,
                     const AttnParams p) {
  // Persistent: CTA b runs works b, b + gridDim.x, ...  The K/V rings, TMEM and
  // every barrier carry over from one work to the next, so the next work's
  // K/V loads and first QK overlap this work's epilogue.
  using C = AttnCfg<HDP, NUM_M>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array, so the
  // compiler keeps the shared address space (STS for the Q tile, not generic ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = smem;                         // NUM_M x Q_BYTES
  uint8_t *sK = sQ + NUM_M * C::Q_BYTES;      // KST x K_BYTES
  uint8_t *sV = sK + C::KST * C::K_BYTES;     // VST x V_BYTES
  uint64_t *bars = reinterpret_cast<uint64_t *>(sV + C::VST * C::V_BYTES);
  uint64_t *k_full = bars;                    // [KST]
  uint64_t *k_empty = k_full + C::KST;        // [KST]
  uint64_t *v_full = k_empty + C::KST;        // [VST]
  uint64_t *v_empty = v_full + C::VST;        // [VST]
  uint64_t *q_full = v_empty + C::VST;        // [NUM_M]  Q(m) staged for the next work
  uint64_t *s_full = q_full + NUM_M;          // [NUM_M]  S(m, j) in TMEM
  uint64_t *p_full = s_full + NUM_M;          // [NUM_M]  P(m, j) in TMEM (S consumed)
  uint64_t *o_full = p_full + NUM_M;          // [NUM_M]  O(m) of a work complete
  uint64_t *q_ready = o_full + NUM_M;         // [NUM_M]  Q(m) re-staged for a new RoPE shift
  uint64_t *o_free = q_ready + NUM_M;         // [NUM_M]  O(m) read by the epilogue (TMEM reusable)
  uint64_t *p_half = o_free + NUM_M;          // [NUM_M]  first 64 keys of P(m, j) in TMEM
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(p_half + NUM_M);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WorkRange wr = cta_work_range(p);
  if (threadIdx.x == 0) CSTAMP(0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int m = 0; m < NUM_M; ++m) {
      mbar_init(&q_full[m], 128);
      mbar_init(&s_full[m], 1);
      mbar_init(&p_full[m], 128);
      mbar_init(&o_full[m], 1);
      mbar_init(&q_ready[m], 128);
      mbar_init(&o_free[m], 128);
      mbar_init(&p_half[m], 128);
    }
    fence_mbar_init();
    tma_prefetch(&tm_k0);
    tma_prefetch(&tm_v0);
    tma_prefetch(&tm_k1);
    tma_prefetch(&tm_v1);
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if (threadIdx.x == 0) CSTAMP(1);
  // Programmatic dependent launch: by default nothing runs past this point
  // before the stream predecessor completed.  With pdl_early (q and the tables
  // predate the predecessor, which writes only K/V pages) the softmax warps
  // stage the first Q while it runs; the producer waits before its first TMA
  // load, and since the CTA cannot exit before the producer, completion stays
  // ordered behind the predecessor.
  if (!p.pdl_early) pdl_wait();
  // The control warpgroup hands registers to the two softmax warpgroups; each
  // role's code sits inside the branch of its setmaxnreg so ptxas allocates
  // it under that budget.
  if (warp < 4) {
  if constexpr (NUM_M == 2) regs_dec<C::REG_CTRL>();
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      if (p.pdl_early) pdl_wait();
      // K(t) is issued one tile ahead of V(t - 1): QK needs K early, P.V needs V late.
      int kj = 0, vj = 0;
      int pend_src = 0, pend_layer = 0, pend_kv = 0, pend_row = -1;
      auto load_v = [&]() {
        const int st = vj % C::VST;
        if (vj >= C::VST) mbar_wait(&v_empty[st], ((vj / C::VST) & 1) ^ 1);
        if (!CM && (p.dbg & 4)) {
          mbar_arrive(&v_full[st]);
        } else {
          const CUtensorMap *tv = pend_src ? &tm_v1 : &tm_v0;
          mbar_arrive_expect_tx(&v_full[st], C::V_BYTES);
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_4d(sV + st * C::V_BYTES + a * HDP * 128, tv, &v_full[st], pend_row + a * 64, 0, pend_kv,
                        pend_layer);
        }
        ++vj;
      };
      for (int wi = wr.begin; wi < wr.end; wi += wr.step) {
        const DbsaAttnWork w = p.works[wi];
        for (int si = w.seg_begin; si < w.seg_end; ++si) {
          const DbsaAttnSeg sg = p.segs[si];
          const int off = sg.row0 & 63;  // tiles start on 64-row page boundaries
          const int nt = (off + sg.n_tok + kBN - 1) / kBN;
          const CUtensorMap *tk = sg.src ? &tm_k1 : &tm_k0;
          for (int tt = 0; tt < nt; ++tt) {
            const int row = sg.row0 - off + tt * kBN;
            const int st = kj % C::KST;
            if (kj >= C::KST) mbar_wait(&k_empty[st], ((kj / C::KST) & 1) ^ 1);
            if (!CM && (p.dbg & 4)) {
              mbar_arrive(&k_full[st]);
            } else {
              mbar_arrive_expect_tx(&k_full[st], C::K_BYTES);
#pragma unroll
              for (int a = 0; a < C::NATOM; ++a)
                tma_load_4d(sK + st * C::K_BYTES + a * kBN * C::QSW, tk, &k_full[st], a * C::KATOM, row, w.kv_head,
                            sg.layer);
            }
            ++kj;
            if (pend_row >= 0) load_v();
            pend_src = sg.src;
            pend_layer = sg.layer;
            pend_kv = w.kv_head;
            pend_row = row;
          }
        }
      }
      if (pend_row >= 0) load_v();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA warp
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, kBN);
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, HDP);
    const uint32_t sQa = smem_u32(sQ), sKa = smem_u32(sK), sVa = smem_u32(sV);
    const bool leader = elect_one();
    auto qk = [&](int m, int jg) {  // S(m) = Q(m) K(jg)^T, K = head_dim
      const int st = jg % C::KST;
      const uint32_t d = tbase + NUM_M * HDP + m * kBN;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < HDP / 16; ++kk) {
          const int a = (kk * 16) / C::KATOM;
          const int off = ((kk * 16) % C::KATOM) * 2;
          const uint64_t ad = umma_desc_kmajor(sQa + m * C::Q_BYTES + a * 128 * C::QSW + off, C::QSW);
          const uint64_t bd = umma_desc_kmajor(sKa + st * C::K_BYTES + a * kBN * C::QSW + off, C::QSW);
          if (CM || !(p.dbg & 2)) umma_bf16_ss(d, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[m]);
      }
      __syncwarp();
    };
    // O(m) (+)= P(m, jg) V(jg) over keys 64 hf .. 64 hf + 63, P from TMEM: the
    // first half is issued as soon as the softmax has written it (p_half), so
    // it runs on the tensor pipe while the softmax computes the second half
    auto pv = [&](int m, int jg, bool first, int hf) {
      const int st = jg % C::VST;
      const uint32_t d = tbase + m * HDP;
      const uint32_t pa = tbase + NUM_M * HDP + m * kBN;
      if (leader) {
#pragma unroll
        for (int kk = hf * kBN / 32; kk < (hf + 1) * kBN / 32; ++kk) {
          const int a = kk / 4;
          const int off = (kk % 4) * 32;
          const uint64_t bd = umma_desc_kmajor(sVa + st * C::V_BYTES + a * HDP * 128 + off, 128);
          if (CM || !(p.dbg & 2)) umma_bf16_ts(d, pa + kk * 8, bd, idesc_o, (!first || kk > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t *bar) {
      if (leader) umma_commit(bar);
      __syncwarp();
    };
    int jg = 0;        // global tile counter (ring slots and per-tile barrier phases)
    int n_bound = 0;   // RoPE-shift boundaries seen (q_ready phases)
    int wk = 0;        // works done by this CTA (q_full / o_full / o_free phases)
    for (int wi = wr.begin; wi < wr.end; wi += wr.step, ++wk) {
      const DbsaAttnWork w = p.works[wi];
      int n_tiles = 0;
      for (int si = w.seg_begin; si < w.seg_end; ++si)
        n_tiles += ((p.segs[si].row0 & 63) + p.segs[si].n_tok + kBN - 1) / kBN;
      for (int m = 0; m < NUM_M; ++m) mbar_wait(&q_full[m], wk & 1);
      tc_fence_after();
      if (n_tiles > 0) {
        // segment iterator: tile j is a "shift boundary" when it opens a segment
        // whose RoPE shift differs from the previous segment's -- QK(m, j) must
        // then wait for the softmax warps to re-stage Q(m) (q_ready), while
        // P.V(m, j-1) does not.
        int it_seg = w.seg_begin, it_tt = 0;
        int it_nt = ((p.segs[it_seg].row0 & 63) + p.segs[it_seg].n_tok + kBN - 1) / kBN;
        for (int j = 0; j < n_tiles; ++j) {
          bool boundary = false;
          if (it_tt == it_nt) {
            const int prev_shift = p.segs[it_seg].shift;
            ++it_seg;
            it_tt = 0;
            it_nt = ((p.segs[it_seg].row0 & 63) + p.segs[it_seg].n_tok + kBN - 1) / kBN;
            boundary = p.segs[it_seg].shift != prev_shift;
          }
          ++it_tt;
          const int t = jg + j;
          mbar_wait(&k_full[t % C::KST], (t / C::KST) & 1);
          tc_fence_after();
          if (t == 0 && lane == 0) CSTAMP(3);
          for (int m = 0; m < NUM_M; ++m) {
            if (j > 0) {
              // P(m, j-1) ready (and S(m) free): accumulate it, then reuse S(m) for tile j
              mbar_wait(&p_half[m], (t - 1) & 1);
              if (m == 0) mbar_wait(&v_full[(t - 1) % C::VST], ((t - 1) / C::VST) & 1);
              if (j == 1 && wk > 0) mbar_wait(&o_free[m], (wk - 1) & 1);  // previous work's O was read
              tc_fence_after();
              pv(m, t - 1, j == 1, 0);
              mbar_wait(&p_full[m], (t - 1) & 1);
              if (lane == 0) STAMP(10 + m, t - 1);
              tc_fence_after();
              pv(m, t - 1, false, 1);
              if (m == NUM_M - 1) commit(&v_empty[(t - 1) % C::VST]);
            }
            if (boundary) {
              mbar_wait(&q_ready[m], n_bound & 1);
              tc_fence_after();
            }
            qk(m, t);
          }
          n_bound += boundary;
          commit(&k_empty[t % C::KST]);
        }
        const int t = jg + n_tiles - 1;
        for (int m = 0; m < NUM_M; ++m) {
          mbar_wait(&p_half[m], t & 1);
          if (m == 0) mbar_wait(&v_full[t % C::VST], (t / C::VST) & 1);
          if (n_tiles == 1 && wk > 0) mbar_wait(&o_free[m], (wk - 1) & 1);
          tc_fence_after();
          pv(m, t, n_tiles == 1, 0);
          mbar_wait(&p_full[m], t & 1);
          tc_fence_after();
          pv(m, t, false, 1);
          commit(&o_full[m]);
        }
        if (lane == 0) CSTAMP(4);
        commit(&v_empty[t % C::VST]);
        jg += n_tiles;
      } else {
        for (int m = 0; m < NUM_M; ++m) {
          if (wk > 0) mbar_wait(&o_free[m], (wk - 1) & 1);
          commit(&o_full[m]);
        }
      }
    }
  }
  } else {
    if constexpr (NUM_M == 2) regs_inc<C::REG_SOFTMAX>();
    // ------------------------------------------------------------ softmax warpgroups
    const int m = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int trow = q4 * 32 + lane;  // row inside the M tile == TMEM lane
    const int r = m * 128 + trow;     // row inside the work
    uint8_t *q_tile = sQ + m * C::Q_BYTES;
    const uint32_t lane_base = tbase + ((uint32_t)(q4 * 32) << 16);
    const uint32_t t_s = lane_base + NUM_M * HDP + m * kBN;
    const uint32_t t_o = lane_base + m * HDP;
    const float sl2 = p.scale_log2;
    int jg = 0, wk = 0;
    uint32_t n_pairs = 0;  // pair counter (p.pair_count)

    const bool coop = CM || (HDP >= 16 && p.head_dim == HDP && (p.q_tok_stride & 7) == 0);
    auto stage_q = [&](const DbsaAttnWork &wq, bool restage, int shift, int sw = -1) {
      if (!CM && (p.dbg & 16)) return;  // profiling: keep whatever Q the tile holds
      if (CM || (coop && p.rope_h)) {
        // the specialised instance stages 4 iterations per batch (C3 K3 -0.5 %;
        // the generic kernel keeps 8: K1 +0.8 % and spills at 4)
        stage_q_coop<HDP, true, CM ? 4 : DBSA_QSTAGE_BATCH>(p, wq, m, q_tile, q4, lane, restage, shift, sw);
      } else if (coop) {
        stage_q_coop<HDP, false>(p, wq, m, q_tile, q4, lane, restage, shift);
      } else {
        const RowRef xq = row_ref(p, wq, r);
        load_q_row<HDP>(p, q_tile, trow, xq.valid, xq.t, xq.head, restage ? p.tok_pos[xq.t] - shift : xq.rope_row);
      }
    };
    // This thread's row of the next work (its descriptor, row refs, tree-mask
    // bound and first RoPE shift), loaded one work ahead: at a work boundary
    // the loads are issued before the epilogue, so their latency hides there.
    RowRef x_nx;
    DbsaAttnWork w_nx;
    int lo_nx = 0, rot_nx = 0;
    auto load_row = [&](const DbsaAttnWork &wq) {
      x_nx = row_ref(p, wq, r);
      lo_nx = (p.tok_lo && x_nx.valid) ? p.tok_lo[x_nx.t] : 0;
      rot_nx = wq.seg_end > wq.seg_begin ? p.segs[wq.seg_begin].shift : 0;
    };
    if (wr.begin < wr.end) {  // stage Q of the first work
      w_nx = p.works[wr.begin];
      load_row(w_nx);
      stage_q(w_nx, false, 0);
      fence_proxy_async_smem();
      mbar_arrive(&q_full[m]);
      if (m == 0 && trow == 0) CSTAMP(2);
    }
    for (int wi = wr.begin; wi < wr.end; wi += wr.step, ++wk) {
      const DbsaAttnWork w = w_nx;  // read at the previous boundary
      const RowRef xr = x_nx;
      const bool valid = xr.valid;
      const int t = xr.t, head = xr.head;
      const int rl = t - w.self_tok0;
      const int lo = lo_nx;
      int cur_rot = rot_nx;
      // Online softmax in the log2 domain; the scale is folded into the exp2
      // FFMA: p = 2^(x * scale_log2 - m_used).
      if (trow == 0 && m == 0 && w.seg_begin != 0x7fffffff) WSTAMP(8, wk);
      const bool warp_dead = __all_sync(0xffffffffu, !valid);
      float m_used = -INFINITY, l_sum = 0.f;
      int j = 0;
      for (int si = w.seg_begin; si < w.seg_end; ++si) {
        const DbsaAttnSeg sg = p.segs[si];
        if (trow == 0 && m == 0 && si == w.seg_begin && sg.n_tok != 0x7fffffff) WSTAMP(9, wk);
        const int off = sg.row0 & 63;
        const int nt = (off + sg.n_tok + kBN - 1) / kBN;
        const bool is_self = sg.kind == DBSA_SEG_SELF;
        // visible local keys of this row: [0, vis_hi) minus the band [band_lo, band_hi)
        int vis_hi = valid ? sg.n_tok : 0;
        int band_lo = 0, band_hi = 0;
        if (is_self) {
          vis_hi = min(vis_hi, rl + 1);
          band_lo = w.prefix;
          band_hi = lo;
        }
        for (int tt = 0; tt < nt; ++tt, ++j) {
          const int k0 = tt * kBN - off;  // local key index of tile column 0
          const int c_lo = max(0, -k0), c_hi = min(kBN, vis_hi - k0);
          const int b_lo = band_lo - k0, b_hi = band_hi - k0;
          // invalid rows (beyond the work's rows) count as full: their S is Q=0 . K = 0
          // and their P only feeds their own (never stored) O rows
          const bool full = !valid || (c_lo == 0 && c_hi == kBN && (b_hi <= 0 || b_lo >= kBN || b_lo >= b_hi));
          const bool restage = !CM && tt == nt - 1 && si + 1 < w.seg_end && p.segs[si + 1].shift != cur_rot;
          if (trow == 0) STAMP(m * 5 + 0, jg + j);
          mbar_wait(&s_full[m], (jg + j) & 1);
          tc_fence_after();
          if (trow == 0) STAMP(m * 5 + 1, jg + j);
          if (warp_dead || (!CM && (p.dbg & 1))) {  // no valid row: its P rows only feed its own (discarded) O rows
            if (restage) {
              cur_rot = p.segs[si + 1].shift;
              mbar_arrive(&q_ready[m]);  // nothing to re-stage for invalid rows
            }
            tc_fence_before();
            mbar_arrive(&p_half[m]);
            mbar_arrive(&p_full[m]);
            continue;
          }
          float x[kBN];
#pragma unroll
          for (int c = 0; c < kBN; c += 32) tmem_ld32(t_s + c, *reinterpret_cast<float(*)[32]>(&x[c]));
          tmem_wait_ld();
          if (trow == 0) STAMP(m * 5 + 2, jg + j);
          if (!__all_sync(0xffffffffu, full)) {
            // visible columns as four 32-bit words, then one bit test per column
            // (R2P + FSEL instead of two compares per column)
            uint32_t keep[kBN / 32];
#pragma unroll
            for (int wd = 0; wd < kBN / 32; ++wd) {
              keep[wd] = range_bits(c_lo - 32 * wd, c_hi - 32 * wd);
              if (is_self) keep[wd] &= ~range_bits(b_lo - 32 * wd, b_hi - 32 * wd);
            }
#pragma unroll
            for (int c = 0; c < kBN; ++c) x[c] = (keep[c >> 5] >> (c & 31)) & 1u ? x[c] : -INFINITY;
          }
          if (!CM && p.pair_count && valid) n_pairs += count_visible(x);
          float mx[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = fmax3(x[i], x[i + 8], x[i + 16]);
#pragma unroll
          for (int c = 24; c + 16 < kBN; c += 16)
#pragma unroll
            for (int i = 0; i < 8; ++i) mx[i] = fmax3(mx[i], x[c + i], x[c + 8 + i]);
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], x[kBN - 8 + i]);
          const float tmax =
              fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7])) * sl2;
          const float m_new = fmaxf(m_used, tmax);
          if (trow == 0) STAMP(m * 5 + 3, jg + j);
          // Lazy rescale (threshold 2^8).  S(m, j) being complete implies P.V(m, j-1)
          // retired (issued before QK(m, j) on the in-order tensor pipe), so O(m)
          // is quiescent here.  tcgen05.ld/st are warp-wide: the decision is warp-uniform.
          const bool need = (m_used != -INFINITY) && (m_new > m_used + DBSA_RESCALE_LOG2);
          float alpha = 1.f;
          if (__any_sync(0xffffffffu, need)) {
            if (m_used != -INFINITY) alpha = fast_exp2(m_used - m_new);
            m_used = m_new;
#pragma unroll 1
            for (int c0 = 0; c0 < HDP; c0 += 16) {
              float o[16];
              tmem_ld16(t_o + c0, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= alpha;
              tmem_st16(t_o + c0, o);
            }
          } else if (m_used == -INFINITY) {
            m_used = m_new;  // first finite max: O row holds nothing yet
          }
          l_sum *= alpha;
          const float msub = m_used == -INFINITY ? 0.f : m_used;
          // exp2 of (x * scale_log2 - m) two lanes at a time (FFMA2 / FADD2); one
          // pair in four goes through the FMA-pipe exp2 so the MUFU pipe
          // (16/clk/SM) does not bound the tile.
          const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-msub, -msub);
          float2 ps[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float2 a = ffma2(make_float2(x[h * 64 + c], x[h * 64 + c + 1]), sl2v, nmv);
              const float2 e = DBSA_POLY_EXP && ((c >> 1) & 3) == 3 ? exp2_fma2(a)
                                                                      : make_float2(fast_exp2(a.x), fast_exp2(a.y));
              ps[(c >> 1) & 1] = fadd2(ps[(c >> 1) & 1], e);
              pk[c >> 1] = pack_bf16(e.x, e.y);
            }
            tmem_st32(t_s + h * 32, pk);  // P(j): keys 64h..64h+63 over S columns 32h..32h+31
            if (h == 0) {
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&p_half[m]);  // P.V(m, j) over keys 0..63 may start
            }
          }
          const float2 pss = fadd2(ps[0], ps[1]);
          l_sum += pss.x + pss.y;
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&p_full[m]);  // P.V(m, j) may start now
          if (trow == 0) STAMP(m * 5 + 4, jg + j);
          if (restage) {  // QK(m, j) retired (S read); QK(m, j+1) waits for q_ready(m)
            cur_rot = p.segs[si + 1].shift;
            stage_q(w, true, cur_rot);
            fence_proxy_async_smem();
            mbar_arrive(&q_ready[m]);
          }
        }
      }
      jg += j;
      if (trow == 0) WSTAMP(m * 4 + 0, wk);
      // Work boundary.  The last QK(m) of this work has retired (its S was
      // read), so the next work's Q(m) is staged now and its first QK overlaps
      // this epilogue.  A work without key tiles read no S, so nothing yet
      // proves the MMA warp consumed this work's q_full phase: wait for its
      // o_full first, or the next arrival could complete a second q_full phase
      // before the first was observed.  This thread's own row of the next work
      // is loaded first: its latency hides under the staging and the epilogue.
      if (j == 0) mbar_wait(&o_full[m], wk & 1);
      const int wn = wi + wr.step;
      if (wn < wr.end) {
        w_nx = p.works[wn];
        load_row(w_nx);
        stage_q(w_nx, false, 0, wk);
        fence_proxy_async_smem();
        mbar_arrive(&q_full[m]);
      }
      if (trow == 0) WSTAMP(m * 4 + 1, wk);
      // ---------------------------------------------------------- epilogue
      mbar_wait(&o_full[m], wk & 1);
      tc_fence_after();
      if (trow == 0) WSTAMP(m * 4 + 2, wk);
      epilogue_row<HDP, CM>(p, t_o, valid, t, head, w.out_mode, xr.part_row, l_sum, m_used);
      tc_fence_before();
      mbar_arrive(&o_free[m]);  // O(m) may be overwritten by the next work's first P.V
      if (trow == 0) WSTAMP(m * 4 + 3, wk);
      if (trow == 0) CSTAMP(5 + m);
    }
    if (!CM && p.pair_count) flush_pair_count(p.pair_count, n_pairs);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) CSTAMP(7);
  if (warp == 2) tmem_dealloc(tbase, C::TMEM_COLS);
}

// ============================================================================
// Single-M-tile variant (num_m == 1): one 128-row M tile per CTA, Q held in
// TMEM (QK is a TS MMA too, so smem carries only K/V and the rings are deep),
// and S / P double-buffered in TMEM so QK(j+1) runs on the tensor pipe while
// the softmax warpgroup works on tile j: the softmax never waits for its own
// next S, which is the chain that bounds the two-tile kernel.
//   TMEM: O [0, HDP) | S0 [HDP, HDP+128) | S1 [HDP+128, HDP+256) | Q [HDP+256, +HDP/2)
// ============================================================================
template <int HDP>
struct Attn1Cfg {
  static constexpr int K_BYTES = kBN * HDP * 2;
  static constexpr int V_BYTES = HDP * kBN * 2;
  static constexpr int QSW = HDP >= 64 ? 128 : HDP * 2;
  static constexpr int KATOM = HDP >= 64 ? 64 : HDP;
  static constexpr int NATOM = HDP / KATOM;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int AVAIL = 232448 - 1024 - BAR_BYTES;
  static constexpr int PAIRS = AVAIL / (K_BYTES + V_BYTES) > 4 ? 4 : AVAIL / (K_BYTES + V_BYTES);
  static constexpr int KST = PAIRS + ((AVAIL - PAIRS * (K_BYTES + V_BYTES)) >= K_BYTES ? 1 : 0);
  static constexpr int VST = PAIRS;
  static constexpr int SMEM = KST * K_BYTES + VST * V_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 256;
  static constexpr int T_S0 = HDP, T_Q = HDP + 2 * kBN;
  static constexpr int TMEM_COLS = 512;
  static_assert(T_Q + HDP / 2 <= 512, "TMEM budget");
  static_assert(PAIRS >= 2, "not enough shared memory for a 2-stage pipeline");
};

// Rotate this thread's query row at rope row (tok_pos - shift) and store it
// into the TMEM Q columns (row = lane, two bf16 per 32-bit column: the
// A-operand layout of the TS MMA).
template <int HDP>
__device__ __forceinline__ void q_row_to_tmem(const AttnParams &p, uint32_t tq, bool valid, int t, int head,
                                              int rope_row) {
  const int hd = p.head_dim, half = hd >> 1;
  uint32_t pk[HDP / 2];
  if (!valid) {
#pragma unroll
    for (int i = 0; i < HDP / 2; ++i) pk[i] = 0u;
  } else {
    const __nv_bfloat16 *src = p.q + (int64_t)t * p.q_tok_stride + (int64_t)head * hd;
    const float2 *rp = p.rope + (int64_t)rope_row * half;
    if (HDP >= 32 && hd == HDP && (p.q_tok_stride & 7) == 0) {
      constexpr int NCH = HDP / 16;  // 8-pair chunks per half of the head
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint4 lo4 = *reinterpret_cast<const uint4 *>(src + c * 8);
        const uint4 hi4 = *reinterpret_cast<const uint4 *>(src + HDP / 2 + c * 8);
        float4 cs4[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) cs4[v] = reinterpret_cast<const float4 *>(rp + c * 8)[v];
        const __nv_bfloat16 *lo = reinterpret_cast<const __nv_bfloat16 *>(&lo4);
        const __nv_bfloat16 *hi = reinterpret_cast<const __nv_bfloat16 *>(&hi4);
        const float *cs = reinterpret_cast<const float *>(cs4);
        float a[8], b[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float cc = cs[2 * jj], sn = cs[2 * jj + 1];
          const float x = __bfloat162float(lo[jj]), y = __bfloat162float(hi[jj]);
          a[jj] = x * cc - y * sn;
          b[jj] = x * sn + y * cc;
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          pk[c * 4 + jj] = pack_bf16(a[2 * jj], a[2 * jj + 1]);
          pk[HDP / 4 + c * 4 + jj] = pack_bf16(b[2 * jj], b[2 * jj + 1]);
        }
      }
    } else {
#pragma unroll
      for (int e2 = 0; e2 < HDP / 2; ++e2) {
        float o2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = 2 * e2 + u;
          float val = 0.f;
          if (e < hd) {
            const int i = e < half ? e : e - half;
            const float lo = __bfloat162float(src[i]);
            const float hi = __bfloat162float(src[i + half]);
            const float2 cs = rp[i];
            val = e < half ? (lo * cs.x - hi * cs.y) : (lo * cs.y + hi * cs.x);
          }
          o2[u] = val;
        }
        pk[e2] = pack_bf16(o2[0], o2[1]);
      }
    }
  }
  if constexpr (HDP / 2 >= 32) {
#pragma unroll
    for (int c = 0; c < HDP / 2; c += 32) tmem_st32(tq + c, *reinterpret_cast<const uint32_t(*)[32]>(&pk[c]));
  } else if constexpr (HDP / 2 == 16) {
    tmem_st16u(tq, *reinterpret_cast<const uint32_t(*)[16]>(&pk[0]));
  } else {
    tmem_st8u(tq, *reinterpret_cast<const uint32_t(*)[8]>(&pk[0]));
  }
  tmem_wait_st();
}

template <int HDP>
__global__ void __launch_bounds__(256, 1)
    dbsa_attn1_kernel(const __grid_constant__ CUtensorMap tm_k0, const __grid_constant__ CUtensorMap tm_v0,
                      const __grid_constant__ CUtensorMap tm_k1, const __grid_constant__ CUtensorMap tm_v1,
                      const AttnParams p) {
  using C = Attn1Cfg<HDP>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array, so the
  // compiler keeps the shared address space (STS for the Q tile, not generic ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sK = smem;                      // KST x K_BYTES
  uint8_t *sV = sK + C::KST * C::K_BYTES;  // VST x V_BYTES
  uint64_t *bars = reinterpret_cast<uint64_t *>(sV + C::VST * C::V_BYTES);
  uint64_t *k_full = bars;
  uint64_t *k_empty = k_full + C::KST;
  uint64_t *v_full = k_empty + C::KST;
  uint64_t *v_empty = v_full + C::VST;
  uint64_t *s_full = v_empty + C::VST;  // [2] S(j) in buffer j & 1
  uint64_t *p_full = s_full + 2;        // [2] P(j) over S buffer j & 1
  uint64_t *q_full = p_full + 2;        // Q staged in TMEM (initially and after each shift change)
  uint64_t *pv_done = q_full + 1;       // P.V(j) retired (O may be rescaled)
  uint64_t *o_full = pv_done + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const DbsaAttnWork w = p.works[blockIdx.x];
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
    }
    mbar_init(q_full, 128);
    mbar_init(pv_done, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
    tma_prefetch(&tm_k0);
    tma_prefetch(&tm_v0);
    tma_prefetch(&tm_k1);
    tma_prefetch(&tm_v1);
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int kj = 0, vj = 0;
      auto load_v = [&](const DbsaAttnSeg &sg, int row) {
        const int st = vj % C::VST;
        if (vj >= C::VST) mbar_wait(&v_empty[st], ((vj / C::VST) & 1) ^ 1);
        if (p.dbg & 4) {
          mbar_arrive(&v_full[st]);
        } else {
          const CUtensorMap *tv = sg.src ? &tm_v1 : &tm_v0;
          mbar_arrive_expect_tx(&v_full[st], C::V_BYTES);
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_4d(sV + st * C::V_BYTES + a * HDP * 128, tv, &v_full[st], row + a * 64, 0, w.kv_head, sg.layer);
        }
        ++vj;
      };
      DbsaAttnSeg pend_sg{};
      int pend_row = -1;
      for (int si = w.seg_begin; si < w.seg_end; ++si) {
        const DbsaAttnSeg sg = p.segs[si];
        const int off = sg.row0 & 63;
        const int nt = (off + sg.n_tok + kBN - 1) / kBN;
        const CUtensorMap *tk = sg.src ? &tm_k1 : &tm_k0;
        for (int tt = 0; tt < nt; ++tt) {
          const int row = sg.row0 - off + tt * kBN;
          const int st = kj % C::KST;
          if (kj >= C::KST) mbar_wait(&k_empty[st], ((kj / C::KST) & 1) ^ 1);
          if (p.dbg & 4) {
            mbar_arrive(&k_full[st]);
          } else {
            mbar_arrive_expect_tx(&k_full[st], C::K_BYTES);
#pragma unroll
            for (int a = 0; a < C::NATOM; ++a)
              tma_load_4d(sK + st * C::K_BYTES + a * kBN * C::QSW, tk, &k_full[st], a * C::KATOM, row, w.kv_head,
                          sg.layer);
          }
          ++kj;
          if (pend_row >= 0) load_v(pend_sg, pend_row);
          pend_sg = sg;
          pend_row = row;
        }
      }
      if (pend_row >= 0) load_v(pend_sg, pend_row);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA warp
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, kBN);
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, HDP);
    const uint32_t sKa = smem_u32(sK), sVa = smem_u32(sV);
    int n_tiles = 0;
    for (int si = w.seg_begin; si < w.seg_end; ++si)
      n_tiles += ((p.segs[si].row0 & 63) + p.segs[si].n_tok + kBN - 1) / kBN;
    const bool leader = elect_one();
    auto commit = [&](uint64_t *bar) {
      if (leader) umma_commit(bar);
      __syncwarp();
    };
    auto qk = [&](int j) {  // S(j & 1) = Q K(j)^T: A = Q from TMEM, B = K tile (K-major smem)
      const int st = j % C::KST;
      const uint32_t d = tbase + C::T_S0 + (j & 1) * kBN;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < HDP / 16; ++kk) {
          const int a = (kk * 16) / C::KATOM;
          const int off = ((kk * 16) % C::KATOM) * 2;
          const uint64_t bd = umma_desc_kmajor(sKa + st * C::K_BYTES + a * kBN * C::QSW + off, C::QSW);
          if (!(p.dbg & 2)) umma_bf16_ts(d, tbase + C::T_Q + kk * 8, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto pv = [&](int j) {  // O += P(j) V(j): A = P in S buffer j & 1
      const int st = j % C::VST;
      const uint32_t pa = tbase + C::T_S0 + (j & 1) * kBN;
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const int a = kk / 4, off = (kk % 4) * 32;
          const uint64_t bd = umma_desc_kmajor(sVa + st * C::V_BYTES + a * HDP * 128 + off, 128);
          if (!(p.dbg & 2)) umma_bf16_ts(tbase, pa + kk * 8, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    if (n_tiles > 0) {
      // segment iterator for QK(t): a "shift boundary" tile opens a segment whose
      // RoPE shift differs from the previous one; its QK waits for the re-staged Q
      int it_seg = w.seg_begin, it_tt = 0;
      int it_nt = ((p.segs[it_seg].row0 & 63) + p.segs[it_seg].n_tok + kBN - 1) / kBN;
      int q_phase = 0;
      auto issue_qk = [&](int t) {
        bool boundary = false;
        if (it_tt == it_nt) {
          const int prev_shift = p.segs[it_seg].shift;
          ++it_seg;
          it_tt = 0;
          it_nt = ((p.segs[it_seg].row0 & 63) + p.segs[it_seg].n_tok + kBN - 1) / kBN;
          boundary = p.segs[it_seg].shift != prev_shift;
        }
        ++it_tt;
        if (boundary || t == 0) {
          mbar_wait(q_full, q_phase & 1);
          ++q_phase;
        }
        mbar_wait(&k_full[t % C::KST], (t / C::KST) & 1);
        tc_fence_after();
        qk(t);
        commit(&s_full[t & 1]);
        commit(&k_empty[t % C::KST]);
      };
      issue_qk(0);
      for (int j = 0; j < n_tiles; ++j) {
        // QK(j+1) into the other S buffer: its previous P(j-1) was consumed by
        // P.V(j-1), issued in the last iteration (in-order tensor pipe)
        if (j + 1 < n_tiles) issue_qk(j + 1);
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        mbar_wait(&v_full[j % C::VST], (j / C::VST) & 1);
        tc_fence_after();
        pv(j);
        commit(pv_done);
        commit(&v_empty[j % C::VST]);
      }
    }
    commit(o_full);
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax warpgroup
    const int q4 = warp & 3;
    const int trow = q4 * 32 + lane;
    const RowRef xr = row_ref(p, w, trow);
    const bool valid = xr.valid;
    const int t = xr.t, head = xr.head;
    const int rl = t - w.self_tok0;
    const int lo = (p.tok_lo && valid) ? p.tok_lo[t] : 0;
    const uint32_t lane_base = tbase + ((uint32_t)(q4 * 32) << 16);
    const uint32_t t_o = lane_base;
    const uint32_t t_q = lane_base + C::T_Q;

    int cur_rot = w.seg_end > w.seg_begin ? p.segs[w.seg_begin].shift : 0;
    q_row_to_tmem<HDP>(p, t_q, valid, t, head, xr.rope_row);
    tc_fence_before();
    mbar_arrive(q_full);

    const float sl2 = p.scale_log2;
    const bool warp_dead = __all_sync(0xffffffffu, !valid);
    float m_used = -INFINITY, l_sum = 0.f;
    uint32_t n_pairs = 0;  // pair counter (p.pair_count)
    int j = 0;
    for (int si = w.seg_begin; si < w.seg_end; ++si) {
      const DbsaAttnSeg sg = p.segs[si];
      const int off = sg.row0 & 63;
      const int nt = (off + sg.n_tok + kBN - 1) / kBN;
      const bool is_self = sg.kind == DBSA_SEG_SELF;
      int vis_hi = valid ? sg.n_tok : 0;
      int band_lo = 0, band_hi = 0;
      if (is_self) {
        vis_hi = min(vis_hi, rl + 1);
        band_lo = w.prefix;
        band_hi = lo;
      }
      for (int tt = 0; tt < nt; ++tt, ++j) {
        const int k0 = tt * kBN - off;
        const int c_lo = max(0, -k0), c_hi = min(kBN, vis_hi - k0);
        const int b_lo = band_lo - k0, b_hi = band_hi - k0;
        const bool full = !valid || (c_lo == 0 && c_hi == kBN && (b_hi <= 0 || b_lo >= kBN || b_lo >= b_hi));
        const bool restage = tt == nt - 1 && si + 1 < w.seg_end && p.segs[si + 1].shift != cur_rot;
        const uint32_t t_s = lane_base + C::T_S0 + (j & 1) * kBN;
        mbar_wait(&s_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        if (restage) {
          // QK(j) retired (S(j) ready), QK(j+1) waits for q_full: re-stage Q now so
          // the next tile's QK overlaps this tile's softmax
          cur_rot = p.segs[si + 1].shift;
          q_row_to_tmem<HDP>(p, t_q, valid, t, head, p.tok_pos[t] - cur_rot);
          tc_fence_before();
          mbar_arrive(q_full);
        }
        if (warp_dead || (p.dbg & 1)) {
          tc_fence_before();
          mbar_arrive(&p_full[j & 1]);
          continue;
        }
        float x[kBN];
#pragma unroll
        for (int c = 0; c < kBN; c += 32) tmem_ld32(t_s + c, *reinterpret_cast<float(*)[32]>(&x[c]));
        tmem_wait_ld();
        if (!__all_sync(0xffffffffu, full)) {
          uint32_t keep[kBN / 32];
#pragma unroll
          for (int wd = 0; wd < kBN / 32; ++wd)
            keep[wd] = range_bits(c_lo - 32 * wd, c_hi - 32 * wd) & ~range_bits(b_lo - 32 * wd, b_hi - 32 * wd);
#pragma unroll
          for (int c = 0; c < kBN; ++c) x[c] = (keep[c >> 5] >> (c & 31)) & 1u ? x[c] : -INFINITY;
        }
        if (p.pair_count && valid) n_pairs += count_visible(x);
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = fmax3(x[i], x[i + 8], x[i + 16]);
#pragma unroll
        for (int c = 24; c + 16 < kBN; c += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = fmax3(mx[i], x[c + i], x[c + 8 + i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], x[kBN - 8 + i]);
        const float tmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7])) * sl2;
        const float m_new = fmaxf(m_used, tmax);
        const bool need = (m_used != -INFINITY) && (m_new > m_used + DBSA_RESCALE_LOG2);
        float alpha = 1.f;
        if (__any_sync(0xffffffffu, need)) {
          // O is accumulated by P.V(j-1), issued once P(j-1) arrived: wait for it
          if (j > 0) mbar_wait(pv_done, (j - 1) & 1);
          tc_fence_after();
          if (m_used != -INFINITY) alpha = fast_exp2(m_used - m_new);
          m_used = m_new;
#pragma unroll 1
          for (int c0 = 0; c0 < HDP; c0 += 16) {
            float o[16];
            tmem_ld16(t_o + c0, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] *= alpha;
            tmem_st16(t_o + c0, o);
          }
          tmem_wait_st();
        } else if (m_used == -INFINITY) {
          m_used = m_new;
        }
        l_sum *= alpha;
        const float msub = m_used == -INFINITY ? 0.f : m_used;
        const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-msub, -msub);
        float2 ps[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 a = ffma2(make_float2(x[hh * 64 + c], x[hh * 64 + c + 1]), sl2v, nmv);
            const float2 e = ((c >> 1) & 3) == 3 ? exp2_fma2(a) : make_float2(fast_exp2(a.x), fast_exp2(a.y));
            ps[(c >> 1) & 1] = fadd2(ps[(c >> 1) & 1], e);
            pk[c >> 1] = pack_bf16(e.x, e.y);
          }
          tmem_st32(t_s + hh * 32, pk);
        }
        const float2 pss = fadd2(ps[0], ps[1]);
        l_sum += pss.x + pss.y;
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[j & 1]);
      }
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(o_full, 0);
    tc_fence_after();
    epilogue_row<HDP>(p, t_o, valid, t, head, w.out_mode, xr.part_row, l_sum, m_used);
    if (p.pair_count) flush_pair_count(p.pair_count, n_pairs);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tbase, C::TMEM_COLS);
}

// ---------------------------------------------------------------- host side

static bool encode_plane_maps(const DbsaAttnArgs &a, const void *k, const void *v, int64_t rows, int layers,
                              CUtensorMap *tk, CUtensorMap *tv) {
  const int HDP = a.hd_pad;
  const int qsw = HDP >= 64 ? 128 : HDP * 2;
  const int katom = HDP >= 64 ? 64 : HDP;
  CUtensorMapSwizzle ksw = qsw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                           : qsw == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_32B;
  {
    cuuint64_t dims[4] = {(cuuint64_t)HDP, (cuuint64_t)rows, (cuuint64_t)a.n_kv_heads, (cuuint64_t)layers};
    cuuint64_t strides[3] = {(cuuint64_t)HDP * 2, (cuuint64_t)rows * HDP * 2,
                             (cuuint64_t)a.n_kv_heads * rows * HDP * 2};
    cuuint32_t box[4] = {(cuuint32_t)katom, (cuuint32_t)kBN, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (!encode_tiled_bf16(tk, k, 4, dims, strides, box, estr, ksw)) return false;
  }
  {
    cuuint64_t dims[4] = {(cuuint64_t)rows, (cuuint64_t)HDP, (cuuint64_t)a.n_kv_heads, (cuuint64_t)layers};
    cuuint64_t strides[3] = {(cuuint64_t)rows * 2, (cuuint64_t)HDP * rows * 2,
                             (cuuint64_t)a.n_kv_heads * HDP * rows * 2};
    cuuint32_t box[4] = {64u, (cuuint32_t)HDP, 1, 1};  // one 64-key atom column of the V^T tile
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (!encode_tiled_bf16(tv, v, 4, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  }
  return true;
}

template <int HDP>
static int launch_attn1(const DbsaAttnArgs &a, const AttnParams &p, const CUtensorMap *maps, cudaStream_t s) {
  using C = Attn1Cfg<HDP>;
  auto kern = dbsa_attn1_kernel<HDP>;
  static thread_local bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_error(DBSA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  kern<<<a.n_works, C::THREADS, C::SMEM, s>>>(maps[0], maps[1], maps[2], maps[3], p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DBSA_ERR_CUDA, "attention launch: %s", cudaGetErrorString(e));
  return DBSA_OK;
}

static int num_sms() {
  static thread_local int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int HDP, int NUM_M, bool CM = false>
static int launch_attn(const DbsaAttnArgs &a, const AttnParams &p, const CUtensorMap *maps, cudaStream_t s) {
  using C = AttnCfg<HDP, NUM_M>;
  auto kern = dbsa_attn_kernel<HDP, NUM_M, CM>;
  static thread_local bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_error(DBSA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  // persistent: one CTA per SM (1 CTA fits per SM), striding over the works or
  // running the host-packed ranges of cta_works
  const int grid = a.cta_works ? a.n_ctas : a.n_works < num_sms() ? a.n_works : num_sms();
  // programmatic dependent launch only when Q staging may overlap the
  // predecessor (pdl_early_q): a batch launch gains nothing from it, and its
  // early-resident CTAs would hold every SM through the K2w boundary
  launch_k(kern, dim3(grid), dim3(C::THREADS), C::SMEM, s, p.pdl_early != 0, maps[0], maps[1], maps[2], maps[3], p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DBSA_ERR_CUDA, "attention launch: %s", cudaGetErrorString(e));
  return DBSA_OK;
}

}  // namespace dbsa

#ifdef DBSA_STAMPS
extern "C" int dbsa_debug_stamps(long long *host, int n) {
  return cudaMemcpyFromSymbol(host, dbsa::g_stamps, sizeof(long long) * (n < 256 * 12 ? n : 256 * 12)) == cudaSuccess
             ? 0
             : DBSA_ERR_CUDA;
}
extern "C" int dbsa_debug_cta(unsigned long long *host, int n) {
  return cudaMemcpyFromSymbol(host, dbsa::g_cta, sizeof(unsigned long long) * (n < 1024 * 8 ? n : 1024 * 8)) ==
                 cudaSuccess
             ? 0
             : DBSA_ERR_CUDA;
}
extern "C" int dbsa_debug_wstamps(long long *host, int n) {
  return cudaMemcpyFromSymbol(host, dbsa::g_wstamps, sizeof(long long) * (n < 256 * 12 ? n : 256 * 12)) == cudaSuccess
             ? 0
             : DBSA_ERR_CUDA;
}
#endif

extern "C" int dbsa_attention(const DbsaAttnArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_attention: null args");
  const DbsaAttnArgs &a = *args;
  if (a.n_works < 0) return set_error(DBSA_ERR_VALIDATION, "n_works < 0");
  if (a.n_works == 0) return DBSA_OK;
  if (a.head_dim <= 0 || a.head_dim % 2 || a.head_dim > a.hd_pad)
    return set_error(DBSA_ERR_CONFIG, "head_dim %d invalid for hd_pad %d", a.head_dim, a.hd_pad);
  if (!(a.hd_pad == 16 || a.hd_pad == 32 || a.hd_pad == 64 || a.hd_pad == 128))
    return set_error(DBSA_ERR_CONFIG, "hd_pad must be 16/32/64/128, got %d", a.hd_pad);
  if (a.n_kv_heads <= 0 || a.n_heads % a.n_kv_heads)
    return set_error(DBSA_ERR_CONFIG, "n_heads %d not a multiple of n_kv_heads %d", a.n_heads, a.n_kv_heads);
  if (a.num_m != 1 && a.num_m != 2) return set_error(DBSA_ERR_CONFIG, "num_m must be 1 or 2");
  if (a.pool_rows % 64 || a.aux_rows % 64) return set_error(DBSA_ERR_SHAPE, "plane rows must be multiples of 64");
  if (!a.q || !a.tok_pos || !a.rope_table || !a.k_pool || !a.v_pool || !a.works || !a.segs)
    return set_error(DBSA_ERR_VALIDATION, "dbsa_attention: null pointer argument");

  CUtensorMap maps[4];
  if (!encode_plane_maps(a, a.k_pool, a.v_pool, a.pool_rows, a.pool_layers, &maps[0], &maps[1]))
    return DBSA_ERR_CUDA;
  const void *ka = a.k_aux ? a.k_aux : a.k_pool;
  const void *va = a.v_aux ? a.v_aux : a.v_pool;
  const int64_t ar = a.k_aux ? a.aux_rows : a.pool_rows;
  const int al = a.k_aux ? a.aux_layers : a.pool_layers;
  if (!encode_plane_maps(a, ka, va, ar, al, &maps[2], &maps[3])) return DBSA_ERR_CUDA;

  AttnParams p;
  p.q = reinterpret_cast<const __nv_bfloat16 *>(a.q);
  p.q_tok_stride = a.q_tok_stride;
  p.tok_pos = a.tok_pos;
  p.tok_lo = a.tok_lo;
  p.rope = reinterpret_cast<const float2 *>(a.rope_table);
  p.rope_h = reinterpret_cast<const __half2 *>(a.rope_f16);
  p.rope_rows = a.rope_rows;
  p.n_heads = a.n_heads;
  p.n_kv_heads = a.n_kv_heads;
  p.head_dim = a.head_dim;
  p.gs = a.n_heads / a.n_kv_heads;
  p.gs_magic = p.gs > 1 ? (uint32_t)((0x100000000ull + (uint64_t)p.gs - 1) / (uint64_t)p.gs) : 0u;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.works = a.works;
  p.n_works = a.n_works;
  p.segs = a.segs;
  p.out = reinterpret_cast<__nv_bfloat16 *>(a.out);
  p.out_tok_stride = a.out_tok_stride;
  p.part_o = a.part_o;
  p.part_lse = a.part_lse;
  p.row_map = a.row_map;
  p.part_bf16 = a.part_bf16;
  p.pair_count = a.pair_count;
  p.cta_works = a.cta_works;
  p.pdl_early = a.pdl_early_q;
  p.part_chunk_rows = a.part_chunk_rows;
  if (a.part_chunk_rows > 0 && (!a.part_bf16 || a.head_dim % 16))
    return set_error(DBSA_ERR_CONFIG, "part_chunk_rows needs bf16 partials and head_dim %% 16 == 0");
  if (a.cta_works && (a.num_m != 2 || a.n_ctas <= 0 || a.n_ctas > num_sms()))
    return set_error(DBSA_ERR_CONFIG, "cta_works needs num_m == 2 and 0 < n_ctas <= %d, got num_m %d n_ctas %d",
                     num_sms(), a.num_m, a.n_ctas);
  {
    // profiling switches, read once per process (not on every launch)
    static const int dbg = [] {
      const char *e = getenv("DBSA_DEBUG_MODE");
      return e ? atoi(e) : 0;
    }();
    p.dbg = dbg;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // num_m 1 runs the single-M-tile kernel (Q in TMEM, double-buffered S) unless
  // DBSA_ATTN1=0 selects the one-tile instance of the two-tile kernel
  static const bool attn1 = [] {
    const char *e = getenv("DBSA_ATTN1");
    return !(e && e[0] == '0');
  }();
  if (a.num_m == 1 && !attn1) {
    switch (a.hd_pad) {
      case 16: return launch_attn<16, 1>(a, p, maps, s);
      case 32: return launch_attn<32, 1>(a, p, maps, s);
      case 64: return launch_attn<64, 1>(a, p, maps, s);
      case 128: return launch_attn<128, 1>(a, p, maps, s);
    }
  }
  // the chunk-major specialisation: the caller vouches that every work has one
  // segment and writes a partial (one_seg_partials); the launcher checks the rest
  const bool cm = a.one_seg_partials && a.num_m == 2 && a.part_bf16 && a.part_chunk_rows > 0 &&
                  !a.pair_count && !p.dbg && a.rope_f16 && a.head_dim == a.hd_pad && a.hd_pad >= 16 &&
                  (a.q_tok_stride & 7) == 0;
  if (cm) {
    switch (a.hd_pad) {
      case 16: return launch_attn<16, 2, true>(a, p, maps, s);
      case 32: return launch_attn<32, 2, true>(a, p, maps, s);
      case 64: return launch_attn<64, 2, true>(a, p, maps, s);
      case 128: return launch_attn<128, 2, true>(a, p, maps, s);
    }
  }
  switch (a.hd_pad * 10 + a.num_m) {
    case 161: return launch_attn1<16>(a, p, maps, s);
    case 162: return launch_attn<16, 2>(a, p, maps, s);
    case 321: return launch_attn1<32>(a, p, maps, s);
    case 322: return launch_attn<32, 2>(a, p, maps, s);
    case 641: return launch_attn1<64>(a, p, maps, s);
    case 642: return launch_attn<64, 2>(a, p, maps, s);
    case 1281: return launch_attn1<128>(a, p, maps, s);
    case 1282: return launch_attn<128, 2>(a, p, maps, s);
  }
  return set_error(DBSA_ERR_CONFIG, "unsupported attention variant");
}
