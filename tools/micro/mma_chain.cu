// Microbenchmark: round-trip latency of a short tcgen05.mma chain as the attention
// kernel uses it -- one thread issues `reps` M128 x N64 x K16 TS MMAs (one tile's QK is
// 24), commits to an mbarrier, and the same warp waits for that phase; averaged over
// many rounds.  The difference to reps x 32 clk is the issue + commit + wake overhead
// paid once per tile on the S-buffer chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2501_15383_b200/csrc \
//        tools/micro/mma_chain.cu -o /tmp/mma_chain
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace lcx;

__global__ void chain(long long* out, int reps, int rounds) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int x = threadIdx.x; x < 64 * 64 * 2 / 16 * 4; x += blockDim.x)
    reinterpret_cast<uint4*>(smem)[x] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async();
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint64_t db = tc::sdesc_sw128(tc::smem_u32(smem));
    constexpr uint32_t idesc = tc::idesc_f16(128, 64, 1, 1);
    long long t0 = 0;
    for (int rd = 0; rd < rounds + 4; ++rd) {
      if (rd == 4) t0 = clock64();  // 4 warm-up rounds
      for (int r = 0; r < reps; ++r)
        tc::mma_f16_ts_warp(tmem, tmem + 256 + (r & 3) * 8, db + ((r & 3) * 32 >> 4), idesc,
                            r > 0);
      tc::mma_commit_warp(&bar);
      tc::mbar_wait(&bar, rd & 1);
      tc::tc_fence_after();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  const int smem = 64 * 64 * 2 * 4 + 1024;
  cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 2000;
  for (int reps : {1, 4, 8, 24, 48}) {
    chain<<<148, 128, smem>>>(d, reps, rounds);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148.0 * rounds;
    printf("reps=%2d: %.0f clk per issue+commit+wait round (%.0f beyond %d x 32)\n", reps, avg,
           avg - 32.0 * reps, reps);
  }
  return 0;
}
