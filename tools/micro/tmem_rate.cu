// Microbenchmark: tcgen05.ld / tcgen05.st throughput and latency from 1, 4 and 8 warps
// (the attention kernel reads each 128 x 64 fp32 S tile -- 32 KB -- out of TMEM and
// writes P back over it).  One CTA per SM; every warp loops `reps` times over
// ld.32x32b.x32 (+ wait::ld) or st.32x32b.x16 (+ wait::st) on its own lane quadrant;
// clock64 around the loop, max over warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2501_15383_b200/csrc \
//        tools/micro/tmem_rate.cu -o /tmp/tmem_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace lcx;

template <bool LD>
__global__ void bench(long long* out, int reps, int nwarps, float* sink) {
  __shared__ uint32_t slot;
  __shared__ long long tmax;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) tmax = 0;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  if (warp < nwarps) {
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    float v[32];
    uint32_t w[16];
    for (int x = 0; x < 16; ++x) w[x] = threadIdx.x + x;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (LD) {
        tc::tmem_ld32_wait(base + (r & 1) * 32, v);
        acc += v[0] + v[17] + v[31];
      } else {
        tc::tmem_st16(base + (r & 3) * 16, w);
        tc::tmem_wait_st();
      }
    }
    const long long t1 = clock64();
    atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(t1 - t0));
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) out[blockIdx.x] = tmax;
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(float));
  const int reps = 4096;
  for (int ld = 1; ld >= 0; --ld) {
    for (int nw : {1, 4, 8}) {
      for (int it = 0; it < 2; ++it) {
        if (ld) bench<true><<<148, 256>>>(d_out, reps, nw, sink);
        else bench<false><<<148, 256>>>(d_out, reps, nw, sink);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int b = 0; b < 148; ++b) mx = h[b] > mx ? h[b] : mx;
      const double per = double(mx) / reps;               // clk per op per warp
      const double bytes = ld ? 32.0 * 32 * 4 : 32.0 * 16 * 4;  // per warp op
      printf("%s x%d warps=%d: %.1f clk per op per warp, %.1f B/clk per SM\n",
             ld ? "ld.32x32b.x32+wait" : "st.32x32b.x16+wait", ld ? 32 : 16, nw, per,
             bytes * nw / per);
    }
  }
  return 0;
}
