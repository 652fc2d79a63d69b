// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion throughput for M=128 and
// N in {64, 128, 256}, A from shared memory (SS) or tensor memory (TS).  One CTA per SM,
// one thread issues `reps` MMAs into one accumulator, commit + wait, clock64 around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2501_15383_b200/csrc \
//        tools/micro/mma_rate.cu -o /tmp/mma_rate -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace lcx;

template <int N, bool TS>
__global__ void bench(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  // zero operands
  for (int x = threadIdx.x; x < (128 + N) * 64 * 2 / 16; x += blockDim.x)
    reinterpret_cast<uint4*>(smem)[x] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::fence_proxy_async();
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint64_t da = tc::sdesc_sw128(tc::smem_u32(smem));
    const uint64_t db = tc::sdesc_sw128(tc::smem_u32(smem + 128 * 128));
    constexpr uint32_t idesc = tc::idesc_f16(128, N, 1, 1);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (TS)
        tc::mma_f16_ts_warp(tmem, tmem + 256 + (r & 3) * 8, db + ((r & 3) * 32 >> 4), idesc, r > 0);
      else
        tc::mma_f16_ss_warp(tmem, da + ((r & 3) * 32 >> 4), db + ((r & 3) * 32 >> 4), idesc, r > 0);
    }
    tc::mma_commit_warp(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int reps = 4096;
  const int smem = (128 + 256) * 128 * 2 + 1024;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, TS><<<sms, 128, smem>>>(d, reps);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("N=%3d %s: %.1f clk per M128xN%dxK16 MMA (theory %d) err=%s\n", N, TS ? "TS" : "SS",
         avg / reps, N, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int sms : {1, 148}) {
    printf("grid %d\n", sms);
    run<64, false>(sms); run<64, true>(sms);
    run<128, false>(sms); run<128, true>(sms);
    run<256, false>(sms); run<256, true>(sms);
  }
  return 0;
}
