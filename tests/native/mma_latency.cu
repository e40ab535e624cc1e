// Round-trip latency of the tensor-core step of the 7L kernels on B200: one tile group of 128
// threads (4 warps) per CTA repeats { named barrier; one elected thread issues K/16 tcgen05.mma kind::f16
// (M = 128, N, bf16, A from TMEM, B from a SWIZZLE_128B shared-memory tile) + tcgen05.commit; every thread waits on
// the mbarrier; tcgen05.ld of 32 accumulator columns + wait::ld } and reports clk per iteration.  Runs 1 CTA
// per SM on all SMs (as the 7L kernel's tile groups would, without their epilogues).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2302_05170_b200/csrc -o mma_lat tests/native/mma_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sl7_tc.cuh"

using namespace sl7;

template <int N, int KSTEPS, int LD>
__global__ void __launch_bounds__(128, 1) rt_kernel(long long* cyc, int iters, int groups_per_cta) {
  __shared__ __align__(1024) uint8_t btile[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_sh;
  for (int i = threadIdx.x; i < 64 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(btile)[i] = 0x3f803f80u;
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase_sh, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tbase_sh, acc = tb, a = tb + 64;
  const uint32_t lane_off = (uint32_t)((threadIdx.x >> 5) * 32) << 16;
  {
    uint32_t w[16];
    for (int k = 0; k < 16; ++k) w[k] = 0x3f803f80u;
    tc::tmem_st_32x32b_x16(a + lane_off, w);
    tc::tmem_st_32x32b_x16(a + lane_off + 16, w);
    tc::wait_st();
  }
  constexpr uint32_t idesc = tc::idesc_bf16_f32(128, N);
  const uint64_t bdesc = tc::smem_desc_sw128(tc::smem_u32(btile));
  uint32_t phase = 0;
  uint32_t sink = 0;
  long long t0 = 0;
  for (int it = -4; it < iters; ++it) {
    if (it == 0) t0 = clock64();
    tc::fence_before();
    tc::named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
      tc::fence_after();
#pragma unroll
      for (int k = 0; k < KSTEPS; ++k) tc::mma_bf16_ts(acc, a + 8u * (k & 3), bdesc + 2u * (k & 3), idesc, k > 0 ? 1u : 0u);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1u;
    tc::fence_after();
    if (LD == 1) {   // one 32-column load + wait
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(acc + lane_off, v);
      tc::wait_ld();
      sink += v[threadIdx.x & 31];
    } else if (LD == 2) {   // two 32-column loads, each followed by its wait (the kernel's halves)
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(acc + lane_off, v);
      tc::wait_ld();
      sink += v[threadIdx.x & 31];
      tc::tmem_ld_32x32b_x32(acc + lane_off + 32, v);
      tc::wait_ld();
      sink += v[(threadIdx.x + 1) & 31];
    } else if (LD == 3) {   // a load long after the MMA finished: is the latency the load's or the hand-over's?
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(acc + lane_off, v);
      tc::wait_ld();
      sink += v[threadIdx.x & 31];
      for (int d = 0; d < 64; ++d) sink = sink * 1664525u + 1013904223u;
      const long long tl = clock64();
      tc::tmem_ld_32x32b_x32(acc + lane_off + 32, v);
      tc::wait_ld();
      sink += v[(threadIdx.x + 1) & 31] + (uint32_t)(clock64() - tl);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0);
  if (sink == 0xdeadbeefu) cyc[blockIdx.x] = 0;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tb, 128);
}

template <int N, int KSTEPS, int LD>
void run(const char* name, int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int iters = 2000;
  rt_kernel<N, KSTEPS, LD><<<sms, 128>>>(d, iters, 1);
  cudaError_t e = cudaDeviceSynchronize();
  long long* h = new long long[sms];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += (double)h[i];
  printf("{\"case\": \"%s\", \"err\": \"%s\", \"clk_per_round_trip\": %.1f}\n", name, cudaGetErrorString(e),
         s / sms / iters);
  delete[] h;
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 4, 1>("hidden layer: N=64, K=64 (4 MMAs) + commit + mbarrier + tcgen05.ld x32", sms);
  run<64, 4, 2>("hidden layer + two x32 loads, each with its wait (the kernel's halves)", sms);
  run<64, 4, 0>("hidden layer without the accumulator load", sms);
  run<16, 4, 1>("output layer: N=16, K=64 (4 MMAs) + ld", sms);
  run<64, 1, 0>("one MMA (N=64, K=16) + commit + mbarrier", sms);
  run<64, 12, 0>("SPLIT layer: 12 MMAs (N=64) + commit + mbarrier", sms);
  return 0;
}
