// Pipe microbenchmarks: measured issue rates of the instructions the step kernels
// are built from, to replace the assumed 16 MUFU/clk/SM and 128 FFMA/clk/SM with B200 measurements.
// Each thread runs 8 independent dependency chains; results are op/clk/SM using clock64() deltas.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes_bench pipes_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CH 8
constexpr int ITERS = 4096;

template <int OP>
__device__ __forceinline__ float op(float x) {
  float r;
  if constexpr (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  if constexpr (OP == 1) {  // rcp(rcp(x)) would be folded by ptxas: interleave a cheap FMA-pipe op
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    r = r * 1.0001f;
  }
  if constexpr (OP == 2) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  if constexpr (OP == 3) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  if constexpr (OP == 4) asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  if constexpr (OP == 5) asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  if constexpr (OP == 6) r = fmaf(x, 0.999f, 0.0001f);
  if constexpr (OP == 7) {  // ex2.approx.bf16x2: one instruction, two results
    uint32_t u = __float_as_uint(x), v;
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(v) : "r"(u));
    r = __uint_as_float(v);
  }
  if constexpr (OP == 8) {
    uint32_t u = __float_as_uint(x), v;
    asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(v) : "r"(u));
    r = __uint_as_float(v);
  }
  if constexpr (OP == 9) r = __uint_as_float(__float_as_uint(x) ^ 0x5a5a5a5au);  // LOP3 (ALU pipe)
  return r;
}

template <int OP>
__global__ void pipe_kernel(float* out, long long* cycles) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = 0.5f + 0.01f * (threadIdx.x + c);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = op<OP>(v[c]);
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms, int threads, float* d_out, long long* d_cyc) {
  pipe_kernel<OP><<<sms, threads>>>(d_out, d_cyc);
  pipe_kernel<OP><<<sms, threads>>>(d_out, d_cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)h[i];
  avg /= sms;
  const double ops = (double)threads * ITERS * CH;
  printf("{\"op\": \"%s\", \"threads_per_sm\": %d, \"thread_ops_per_clk_per_sm\": %.2f}\n", name, threads, ops / avg);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, sizeof(float) * sms * 1024);
  cudaMalloc(&d_cyc, sizeof(long long) * sms);
  for (int threads : {512, 1024}) {
    run<0>("MUFU.EX2 (ex2.approx.f32)", sms, threads, d_out, d_cyc);
    run<1>("MUFU.RCP (rcp.approx.f32)", sms, threads, d_out, d_cyc);
    run<2>("MUFU.LG2 (lg2.approx.f32)", sms, threads, d_out, d_cyc);
    run<3>("MUFU.TANH (tanh.approx.f32)", sms, threads, d_out, d_cyc);
    run<4>("MUFU.RSQ (rsqrt.approx.f32)", sms, threads, d_out, d_cyc);
    run<5>("MUFU.SIN (sin.approx.f32)", sms, threads, d_out, d_cyc);
    run<6>("FFMA", sms, threads, d_out, d_cyc);
    run<7>("ex2.approx.bf16x2 (2 results/instr)", sms, threads, d_out, d_cyc);
    run<8>("tanh.approx.bf16x2 (2 results/instr)", sms, threads, d_out, d_cyc);
    run<9>("LOP3 (ALU)", sms, threads, d_out, d_cyc);
  }
  return 0;
}
