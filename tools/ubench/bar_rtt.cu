// Round-trip latency of the K1/K3 handshake without any math:
//   thread A: tcgen05.commit(s_full)  (or mbarrier.arrive)  -> 128 waiter threads
//   waiters:  wait s_full, arrive p_full (count 128)         -> thread A waits p_full
// Reports cycles per round trip for commit-based and arrive-based signalling.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2503_08640_b200/csrc/sm100_ptx.cuh"
using namespace dbsa;

template <bool COMMIT, int NW>
__global__ void kern(long long *out, int iters) {
  __shared__ uint64_t s_full, p_full;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&s_full, 1); mbar_init(&p_full, NW * 32); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        if (COMMIT) umma_commit(&s_full); else mbar_arrive(&s_full);
        mbar_wait(&p_full, i & 1);
      }
      out[blockIdx.x] = (clock64() - t0) / iters;
    }
  } else if (warp >= 4 && warp < 4 + NW) {
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&s_full, i & 1);
      mbar_arrive(&p_full);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 32);
}

template <bool C, int NW>
void run() {
  long long *d; cudaMalloc(&d, 8 * 148);
  kern<C, NW><<<148, 128 + 32 * NW>>>(d, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%s, %d waiter warps: %lld cycles per round trip\n", C ? "tcgen05.commit" : "mbarrier.arrive", NW, h);
}

int main() {
  run<false, 1>(); run<false, 4>(); run<false, 8>();
  run<true, 1>(); run<true, 4>(); run<true, 8>();
  return 0;
}
