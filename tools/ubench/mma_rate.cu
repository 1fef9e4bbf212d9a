// Microbenchmark: cycles per tcgen05.mma for (M=128, N, K=16) bf16 with A
// from smem (SS) or TMEM (TS); one issuing thread, back-to-back, one commit
// at the end.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2503_08640_b200/csrc/sm100_ptx.cuh"
using namespace dbsa;

template <int N, bool TS, int CEVERY>
__global__ void kern(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = umma_desc_kmajor(sb + kk * 32, 128);
        if (TS) umma_bf16_ts(tb, tb + 256 + kk * 8, bd, idesc, 1u);
        else umma_bf16_ss(tb, umma_desc_kmajor(sa + kk * 32, 128), bd, idesc, 1u);
        if (CEVERY && (kk % CEVERY) == CEVERY - 1) umma_commit(&bar2[kk & 3]);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <int N, bool TS, int CE = 0>
void run(int blocks) {
  long long *d; cudaMalloc(&d, blocks * 8);
  int iters = 2000;
  cudaFuncSetAttribute(kern<N, TS, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  kern<N, TS, CE><<<blocks, 128, 65536>>>(d, 10);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<N, TS, CE><<<blocks, 128, 65536>>>(d, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[1]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  double mmas = (double)iters * 8;
  double flops = 2.0 * 128 * N * 16 * mmas * blocks;
  printf("commit every %d: ", CE);
  printf("M=128 N=%3d K=16 %s blocks=%d: %.1f clk/MMA (block 0), %.1f TFLOP/s aggregate\n", N, TS ? "TS" : "SS", blocks,
         h[0] / mmas, flops / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  printf("start\n"); fflush(stdout);
  run<64, false>(148); run<128, false>(148);
  run<64, true>(148); run<128, true>(148);
  run<64, false, 1>(148); run<64, false, 4>(148); run<64, false, 8>(148);
  run<128, true, 1>(148); run<128, true, 4>(148);
  return 0;
}
