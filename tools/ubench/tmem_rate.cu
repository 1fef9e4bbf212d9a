// TMEM read/write throughput: NW warps each issue tcgen05.ld.32x32b.x32 (4 KB per
// warp) back to back; reports bytes/clk per SM.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2503_08640_b200/csrc/sm100_ptx.cuh"
using namespace dbsa;

template <int NW, bool ST>
__global__ void kern(long long *out, float *sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float a[32], b[32], c[32], d[32];
    const uint32_t col = (i * 128) & 511;
    if (ST) {
      uint32_t v[32];
      for (int k = 0; k < 32; ++k) v[k] = i + k;
      tmem_st32(tb + col, v);
      tmem_st32(tb + ((col + 32) & 511), v);
      tmem_st32(tb + ((col + 64) & 511), v);
      tmem_st32(tb + ((col + 96) & 511), v);
      tmem_wait_st();
    } else {
      tmem_ld32(tb + col, a);
      tmem_ld32(tb + ((col + 32) & 511), b);
      tmem_ld32(tb + ((col + 64) & 511), c);
      tmem_ld32(tb + ((col + 96) & 511), d);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += (a[k] + b[k]) * (c[k] + d[k]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int NW, bool ST>
void run() {
  long long *d; float *s;
  cudaMalloc(&d, 8 * 148); cudaMalloc(&s, 4 * 148 * 32 * NW);
  int iters = 4000;
  kern<NW, ST><<<148, 32 * NW>>>(d, s, 10);
  kern<NW, ST><<<148, 32 * NW>>>(d, s, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  double bytes = (double)iters * NW * 4 * 32 * 32 * 4;  // 4 x (32 lanes x 32 cols x 4 B) per warp per iter
  printf("%s %2d warps: %.1f B/clk per SM (%.1f clk per 16 KB warp-batch)\n", ST ? "STTM" : "LDTM", NW, bytes / h,
         (double)h / iters);
}

int main() {
  run<4, false>(); run<8, false>(); run<12, false>(); run<16, false>();
  run<4, true>(); run<8, true>();
  return 0;
}
