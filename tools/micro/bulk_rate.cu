// Microbenchmark: per-SM ingest rate of 1-D bulk copies (cp.async.bulk) global -> shared
// with an S-stage ring of 48 KB tiles (the tcgen05 attention kernel's K hi + K lo + V^T
// tile), one CTA per SM, source footprint `foot` bytes (L2-resident or not), tiles
// visited in a per-CTA pseudo-random or sequential order.  Prints B/clk/SM and TB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2501_15383_b200/csrc \
//        tools/micro/bulk_rate.cu -o /tmp/bulk_rate -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace lcx;

constexpr uint32_t kTile = 48 * 1024;

template <int S>
__global__ void bench(const uint8_t* src, long long ntiles_src, int iters, int pieces, int rnd,
                      long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) tc::mbar_init(full + s, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  auto next_tile = [&](int t) -> long long {
    if (!rnd) return (int64_t(blockIdx.x) * iters + t) % ntiles_src;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    return (long long)(x % uint64_t(ntiles_src));
  };
  const uint32_t piece = kTile / pieces;
  auto issue = [&](int t) {
    const int s = t % S;
    const long long tile = next_tile(t);
    tc::mbar_expect_tx(full + s, kTile);
    for (int k = 0; k < pieces; ++k)
      tc::bulk_load(smem + s * kTile + k * piece, src + tile * kTile + k * piece, piece, full + s);
  };
  for (int t = 0; t < S && t < iters; ++t) issue(t);
  long long t0 = clock64();
  for (int t = 0; t < iters; ++t) {
    tc::mbar_wait(full + (t % S), (t / S) & 1);
    if (t + S < iters) issue(t + S);
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
}

template <int S>
void run(const uint8_t* src, long long foot, int pieces, int rnd) {
  const int iters = 2000;
  long long* d_out;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  const size_t smem = S * kTile + 1024;
  cudaFuncSetAttribute(bench<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const long long nt = foot / kTile;
  bench<S><<<148, 32, smem>>>(src, nt, 200, pieces, rnd, d_out);  // warm
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<S><<<148, 32, smem>>>(src, nt, iters, pieces, rnd, d_out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = double(kTile) * iters;
  printf("stages %d pieces %d foot %7.1f MB %s: %6.1f B/clk/SM (slowest CTA), %6.2f TB/s\n", S,
         pieces, foot / 1e6, rnd ? "random" : "seq   ", bytes / mx, bytes * 148 / (ms * 1e9));
  cudaFree(d_out);
}

int main() {
  uint8_t* src;
  const long long big = 3ll << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  for (long long foot : {32ll << 20, 96ll << 20, big})
    for (int rnd : {0, 1}) {
      run<4>(src, foot, 3, rnd);
      run<4>(src, foot, 6, rnd);
    }
  run<2>(src, 32ll << 20, 3, 1);
  run<3>(src, 32ll << 20, 3, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
