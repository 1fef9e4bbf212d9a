// kv_pages.cu -- K2w page write (rotated K rows + transposed V) and the
// float64-derived rotary table.
//
// Reference: SegmentedKVCache.append_block stores per-block pre-rotation K/V
// (kvstore.py:70-106); stage 1 re-rotates context blocks at their ORIGINAL
// positions before every use (pipeline.py:191-200).  The pool stores K already
// rotated at the original positions (so stage 1 reads it as-is) and stage 2
// moves the re-positioning to the query side (attn_sm100.cu).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/dbsa_b200.h"
#include "dbsa_internal.h"
#include "sm100_ptx.cuh"

namespace dbsa {

// grid (n_pages, n_kv_heads, 2: K | V), 256 threads.  K: [L][Hkv][rows][HDP]; V^T: [L][Hkv][HDP][rows].
// Full-width heads (hd == HDP, 16-byte aligned rows) take the vector path:
// a K item is one row's rotary chunk pair (elements 8c.. and HDP/2 + 8c..)
// read as two 16-byte loads with its 8 (cos, sin) pairs; V goes through a
// shared-memory [64 tokens][HDP] tile so both the loads (along d) and the V^T
// stores (along the token axis) are 16 bytes wide.
__global__ void kv_write_kernel(DbsaKvWriteArgs a) {
  // the attention launch that follows (pdl_early_q) may start now: it stages
  // Q meanwhile and waits for this grid before loading any K/V tile
  pdl_trigger();
  __shared__ __align__(16) __nv_bfloat16 vt[DBSA_PAGE_TOKENS * 128];
  const DbsaPage pg = a.pages[blockIdx.x];
  const int head = blockIdx.y;
  const int hd = a.head_dim, half = hd >> 1, HDP = a.hd_pad;
  const __nv_bfloat16 *ks = reinterpret_cast<const __nv_bfloat16 *>(a.k_src);
  const __nv_bfloat16 *vs = reinterpret_cast<const __nv_bfloat16 *>(a.v_src);
  const float2 *rope = reinterpret_cast<const float2 *>(a.rope_table);
  const int64_t plane = (int64_t)a.layer * a.n_kv_heads + head;
  __nv_bfloat16 *kd = reinterpret_cast<__nv_bfloat16 *>(a.k_dst) + plane * a.dst_rows * HDP;
  __nv_bfloat16 *vd = reinterpret_cast<__nv_bfloat16 *>(a.v_dst) + plane * a.dst_rows * HDP;
  const bool vec = hd == HDP && HDP >= 16 && (a.src_tok_stride & 7) == 0;

  const bool do_k = blockIdx.z == 0, do_v = blockIdx.z == 1;
  if (vec) {
    // K rows: item = (row i, chunk pair cp), rotated at tok_pos (model.py:222-239).
    const int ncp = HDP / 16;
    for (int it = threadIdx.x; do_k && it < DBSA_PAGE_TOKENS * ncp; it += blockDim.x) {
      const int i = it / ncp, cp = it % ncp;
      float lo_o[8], hi_o[8];
      if (i < pg.n_tok) {
        const int t = pg.tok0 + i;
        const __nv_bfloat16 *src = ks + (int64_t)t * a.src_tok_stride + (int64_t)head * hd + cp * 8;
        const uint4 l4 = *reinterpret_cast<const uint4 *>(src);
        const uint4 h4 = *reinterpret_cast<const uint4 *>(src + half);
        const float4 *rp = reinterpret_cast<const float4 *>(rope + (int64_t)a.tok_pos[t] * half + cp * 8);
        float cs[16];
#pragma unroll
        for (int v = 0; v < 4; ++v) *reinterpret_cast<float4 *>(&cs[4 * v]) = rp[v];
        const __nv_bfloat16 *l = reinterpret_cast<const __nv_bfloat16 *>(&l4);
        const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&h4);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float x = __bfloat162float(l[j]), y = __bfloat162float(h[j]);
          lo_o[j] = x * cs[2 * j] - y * cs[2 * j + 1];
          hi_o[j] = x * cs[2 * j + 1] + y * cs[2 * j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) lo_o[j] = hi_o[j] = 0.f;
      }
      __nv_bfloat16 *dst = kd + (int64_t)(pg.row0 + i) * HDP + cp * 8;
      *reinterpret_cast<uint4 *>(dst) = make_uint4(pack_bf16(lo_o[0], lo_o[1]), pack_bf16(lo_o[2], lo_o[3]),
                                                   pack_bf16(lo_o[4], lo_o[5]), pack_bf16(lo_o[6], lo_o[7]));
      *reinterpret_cast<uint4 *>(dst + half) = make_uint4(pack_bf16(hi_o[0], hi_o[1]), pack_bf16(hi_o[2], hi_o[3]),
                                                          pack_bf16(hi_o[4], hi_o[5]), pack_bf16(hi_o[6], hi_o[7]));
    }
    if (!do_v) return;
    // V: [64 tokens][HDP] into shared memory (zero past n_tok), then V^T rows.
    const int nch = HDP / 8;
    for (int it = threadIdx.x; it < DBSA_PAGE_TOKENS * nch; it += blockDim.x) {
      const int i = it / nch, c = it % nch;
      uint4 v4 = make_uint4(0u, 0u, 0u, 0u);
      if (i < pg.n_tok)
        v4 = *reinterpret_cast<const uint4 *>(vs + (int64_t)(pg.tok0 + i) * a.src_tok_stride + (int64_t)head * hd +
                                              c * 8);
      *reinterpret_cast<uint4 *>(&vt[i * HDP + c * 8]) = v4;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < HDP * (DBSA_PAGE_TOKENS / 8); it += blockDim.x) {
      const int d = it / (DBSA_PAGE_TOKENS / 8), ic = it % (DBSA_PAGE_TOKENS / 8);
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat16 a0 = vt[(ic * 8 + 2 * j) * HDP + d], a1 = vt[(ic * 8 + 2 * j + 1) * HDP + d];
        w[j] = (uint32_t)__bfloat16_as_ushort(a0) | ((uint32_t)__bfloat16_as_ushort(a1) << 16);
      }
      *reinterpret_cast<uint4 *>(vd + (int64_t)d * a.dst_rows + pg.row0 + ic * 8) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }

  // generic path (head_dim < HDP or unaligned rows): item = (row i, 8-element chunk c)
  const int kchunks = HDP / 8;
  for (int it = threadIdx.x; do_k && it < DBSA_PAGE_TOKENS * kchunks; it += blockDim.x) {
    const int i = it / kchunks, c = it % kchunks;
    float o[8];
    if (i < pg.n_tok) {
      const int t = pg.tok0 + i;
      const __nv_bfloat16 *src = ks + (int64_t)t * a.src_tok_stride + (int64_t)head * hd;
      const float2 *rp = rope + (int64_t)a.tok_pos[t] * half;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = c * 8 + j;
        float val = 0.f;
        if (e < hd) {
          const int pi = e < half ? e : e - half;
          const float lo = __bfloat162float(src[pi]), hi = __bfloat162float(src[pi + half]);
          const float2 cs = rp[pi];
          val = e < half ? lo * cs.x - hi * cs.y : lo * cs.y + hi * cs.x;
        }
        o[j] = val;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = 0.f;
    }
    *reinterpret_cast<uint4 *>(kd + (int64_t)(pg.row0 + i) * HDP + c * 8) =
        make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
  }
  // V^T columns: item = (dim d, 8-token chunk ic), 16-byte coalesced stores along the token axis.
  for (int it = threadIdx.x; do_v && it < HDP * (DBSA_PAGE_TOKENS / 8); it += blockDim.x) {
    const int d = it / (DBSA_PAGE_TOKENS / 8), ic = it % (DBSA_PAGE_TOKENS / 8);
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = ic * 8 + j;
      o[j] = (i < pg.n_tok && d < hd)
                 ? __bfloat162float(vs[(int64_t)(pg.tok0 + i) * a.src_tok_stride + (int64_t)head * hd + d])
                 : 0.f;
    }
    *reinterpret_cast<uint4 *>(vd + (int64_t)d * a.dst_rows + pg.row0 + ic * 8) =
        make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
  }
}

// K2r: page read-back for serialisation -- the inverse of K2w.  For every
// token of the given pages: K un-rotated at tok_pos (x c + y s, -x s + y c)
// and V, both fp32, token-major [t][kvh][d] (the reference's segment layout,
// kvstore.py:59-60).  grid (n_pages, n_kv_heads), 128 threads.
__global__ void kv_read_kernel(DbsaKvReadArgs a) {
  const DbsaPage pg = a.pages[blockIdx.x];
  const int head = blockIdx.y;
  const int hd = a.head_dim, half = hd >> 1, HDP = a.hd_pad;
  const float2 *rope = reinterpret_cast<const float2 *>(a.rope_table);
  const int64_t plane = (int64_t)a.layer * a.n_kv_heads + head;
  const __nv_bfloat16 *ks = reinterpret_cast<const __nv_bfloat16 *>(a.k_src) + plane * a.src_rows * HDP;
  const __nv_bfloat16 *vs = reinterpret_cast<const __nv_bfloat16 *>(a.v_src) + plane * a.src_rows * HDP;
  for (int it = threadIdx.x; it < pg.n_tok * half; it += blockDim.x) {
    const int i = it / half, e = it % half;
    const int t = pg.tok0 + i;
    const __nv_bfloat16 *kr = ks + (int64_t)(pg.row0 + i) * HDP;
    const float x = __bfloat162float(kr[e]), y = __bfloat162float(kr[e + half]);
    const float2 cs = rope[(int64_t)a.tok_pos[t] * half + e];
    float *kd = a.k_dst + ((int64_t)t * a.n_kv_heads + head) * hd;
    kd[e] = x * cs.x + y * cs.y;
    kd[e + half] = y * cs.x - x * cs.y;
  }
  for (int it = threadIdx.x; it < pg.n_tok * hd; it += blockDim.x) {
    const int i = it % pg.n_tok, d = it / pg.n_tok;  // token-fastest: coalesced V^T reads
    a.v_dst[((int64_t)(pg.tok0 + i) * a.n_kv_heads + head) * hd + d] =
        __bfloat162float(vs[(int64_t)d * a.src_rows + pg.row0 + i]);
  }
}

// table[p][i] = (cos, sin)((pos0 + p) * inv_freq[i]), angle formed in float64
// (model.rope_angles, model.py:205-209), rounded once to float32.
__global__ void rope_table_kernel(float2 *table, int64_t rows, const double *inv_freq, int half, int64_t pos0) {
  const int64_t n = rows * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / half;
    const int i = (int)(idx % half);
    const double ang = (double)(pos0 + p) * inv_freq[i];
    double s, c;
    sincos(ang, &s, &c);
    table[idx] = make_float2((float)c, (float)s);
  }
}

// The same angles rounded once from float64 to fp16 (cos, sin): the query
// rotation table of the two-tile attention kernel's Q staging.
__global__ void rope_table_f16_kernel(__half2 *table, int64_t rows, const double *inv_freq, int half, int64_t pos0) {
  const int64_t n = rows * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / half;
    const int i = (int)(idx % half);
    const double ang = (double)(pos0 + p) * inv_freq[i];
    double s, c;
    sincos(ang, &s, &c);
    table[idx] = __halves2half2(__double2half(c), __double2half(s));
  }
}

}  // namespace dbsa

extern "C" int dbsa_kv_write(const DbsaKvWriteArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_kv_write: null args");
  const DbsaKvWriteArgs &a = *args;
  if (a.n_pages < 0) return set_error(DBSA_ERR_VALIDATION, "n_pages < 0");
  if (a.n_pages == 0) return DBSA_OK;
  if (!(a.hd_pad == 16 || a.hd_pad == 32 || a.hd_pad == 64 || a.hd_pad == 128) || a.head_dim > a.hd_pad ||
      a.head_dim % 2)
    return set_error(DBSA_ERR_CONFIG, "bad head_dim %d / hd_pad %d", a.head_dim, a.hd_pad);
  if (a.dst_rows % DBSA_PAGE_TOKENS) return set_error(DBSA_ERR_SHAPE, "dst_rows must be a multiple of 64");
  if (a.layer < 0 || a.layer >= a.dst_layers) return set_error(DBSA_ERR_VALIDATION, "layer out of range");
  dim3 grid(a.n_pages, a.n_kv_heads, 2);
  kv_write_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("kv_write");
}

extern "C" int dbsa_kv_read(const DbsaKvReadArgs *args, void *stream) {
  using namespace dbsa;
  if (!args) return set_error(DBSA_ERR_VALIDATION, "dbsa_kv_read: null args");
  const DbsaKvReadArgs &a = *args;
  if (a.n_pages < 0) return set_error(DBSA_ERR_VALIDATION, "n_pages < 0");
  if (a.n_pages == 0) return DBSA_OK;
  if (!(a.hd_pad == 16 || a.hd_pad == 32 || a.hd_pad == 64 || a.hd_pad == 128) || a.head_dim > a.hd_pad ||
      a.head_dim % 2)
    return set_error(DBSA_ERR_CONFIG, "bad head_dim %d / hd_pad %d", a.head_dim, a.hd_pad);
  if (a.layer < 0 || a.layer >= a.src_layers) return set_error(DBSA_ERR_VALIDATION, "layer out of range");
  dim3 grid(a.n_pages, a.n_kv_heads);
  kv_read_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("kv_read");
}

extern "C" int dbsa_rope_table(float *table, int64_t rows, const double *inv_freq, int32_t half, int64_t pos0,
                               void *stream) {
  using namespace dbsa;
  if (rows <= 0 || half <= 0) return set_error(DBSA_ERR_VALIDATION, "rope table: empty");
  const int64_t n = rows * half;
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  rope_table_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(reinterpret_cast<float2 *>(table),
                                                                                  rows, inv_freq, half, pos0);
  return check_launch("rope_table");
}

extern "C" int dbsa_rope_table_f16(void *table, int64_t rows, const double *inv_freq, int32_t half, int64_t pos0,
                                   void *stream) {
  using namespace dbsa;
  if (rows <= 0 || half <= 0) return set_error(DBSA_ERR_VALIDATION, "rope table: empty");
  const int64_t n = rows * half;
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  rope_table_f16_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<__half2 *>(table), rows, inv_freq, half, pos0);
  return check_launch("rope_table_f16");
}
