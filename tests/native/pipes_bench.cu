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
  if constexpr (OP == 12) {  // ex2.approx.f16x2: one instruction, two fp16 results
    uint32_t u = __float_as_uint(x), v;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(v) : "r"(u));
    r = __uint_as_float(v);
  }
  if constexpr (OP == 13) {
    uint32_t u = __float_as_uint(x), v;
    asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(v) : "r"(u));
    r = __uint_as_float(v);
  }
  if constexpr (OP == 14) {  // IMAD.WIDE.U32 (Philox's multiply): low word feeds the chain, high word kept live
    uint32_t u = __float_as_uint(x);
    unsigned long long w;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(u), "r"(0xD2511F53u));
    r = __uint_as_float((uint32_t)w ^ (uint32_t)(w >> 32));
  }
  if constexpr (OP == 16) {  // mul.lo.u32 by an immediate (IMAD)
    uint32_t u = __float_as_uint(x), w;
    asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(w) : "r"(u), "n"(0xD2511F53u));
    r = __uint_as_float(w);
  }
  if constexpr (OP == 17) {  // mul.hi.u32 by an immediate (IMAD.HI)
    uint32_t u = __float_as_uint(x), w;
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(w) : "r"(u), "n"(0xD2511F53u));
    r = __uint_as_float(w | 0x3f000000u);
  }
  if constexpr (OP == 18) {  // mul.wide.u32 by an immediate, both halves consumed by one LOP3-free add
    uint32_t u = __float_as_uint(x);
    unsigned long long w;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(u), "n"(0xD2511F53u));
    r = __uint_as_float((uint32_t)w + (uint32_t)(w >> 32));
  }
  if constexpr (OP == 15) {  // FFMA with all-register operands (no immediate)
    float m = __uint_as_float(__float_as_uint(x) | 1u), c;
    asm volatile("mov.b32 %0, 0x38d1b717;" : "=f"(c));
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(x), "f"(m), "f"(c));
  }
  return r;
}

// Packed fp32 (sm_100a FFMA2: fma.rn.f32x2, two fp32 FMAs per lane per instruction).  B = 0: all three
// operands packed registers; B = 1: the multiplier is a scalar register broadcast to both halves.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
template <int B>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, float s) {
  unsigned long long r;
  if constexpr (B == 0) {
    const unsigned long long m = pk2(0.999f, 0.998f), c = pk2(1e-4f, 2e-4f);
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(m), "l"(c));
  } else {
    const unsigned long long m = pk2(s, s), c = pk2(1e-4f, 2e-4f);
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(m), "l"(c));
  }
  return r;
}

// OP 10 / 11: FFMA2 (packed / broadcast), CH independent chains of packed pairs: 2 thread-FMAs per op.
template <int OP>
__global__ void pipe2_kernel(float* out, long long* cycles, float s) {
  unsigned long long v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = pk2(0.5f + 0.01f * (threadIdx.x + c), 0.25f + 0.01f * c);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = ffma2<OP - 10>(v[c], s);
  }
  __syncthreads();
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc += __uint_as_float((uint32_t)v[c]) + __uint_as_float((uint32_t)(v[c] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// Mix: per iteration NM MUFU.EX2 chains and NF FFMA2 chains (independent): measures whether the MUFU and
// the packed FMA pipe overlap (co-issue limit) -- the budget of a softplus epilogue that puts the log1p
// polynomial on FFMA2 next to the MUFU ex2.
template <int NM, int NF>
__global__ void mix_kernel(float* out, long long* cycles, float s) {
  float m[NM > 0 ? NM : 1];
  unsigned long long f[NF > 0 ? NF : 1];
#pragma unroll
  for (int c = 0; c < NM; ++c) m[c] = 0.5f + 0.01f * (threadIdx.x + c);
#pragma unroll
  for (int c = 0; c < NF; ++c) f[c] = pk2(0.5f + 0.01f * c, 0.25f);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NM; ++c) m[c] = op<0>(m[c]);
#pragma unroll
    for (int c = 0; c < NF; ++c) f[c] = ffma2<1>(f[c], s);
  }
  __syncthreads();
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < NM; ++c) acc += m[c];
#pragma unroll
  for (int c = 0; c < NF; ++c) acc += __uint_as_float((uint32_t)f[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// Issue cost of FFMA2 against FFMA at equal FLOPs, next to other pipes: per iteration NA ALU LOP3 chains
// (asm volatile, not foldable) and NM MUFU.EX2 chains plus either 2*NF FFMA (P = 0) or NF FFMA2 (P = 1).
// If FFMA2 took one issue slot its 64-lane work would leave the next slot to another pipe.
template <int NM, int NA, int NF, int P>
__global__ void mix2_kernel(float* out, long long* cycles, float s) {
  float m[NM > 0 ? NM : 1];
  uint32_t a[NA > 0 ? NA : 1];
  float f[NF > 0 ? 2 * NF : 1];
  unsigned long long g[NF > 0 ? NF : 1];
#pragma unroll
  for (int c = 0; c < NM; ++c) m[c] = 0.5f + 0.01f * (threadIdx.x + c);
#pragma unroll
  for (int c = 0; c < NA; ++c) a[c] = threadIdx.x * 2654435761u + c;
#pragma unroll
  for (int c = 0; c < 2 * NF; ++c) f[c] = 0.5f + 0.01f * c;
#pragma unroll
  for (int c = 0; c < NF; ++c) g[c] = pk2(0.5f + 0.01f * c, 0.25f);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NM; ++c) m[c] = op<0>(m[c]);
#pragma unroll
    for (int c = 0; c < NA; ++c)
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(a[(c + 1) % (NA > 0 ? NA : 1)]), "r"(i));
    if constexpr (P == 0) {
#pragma unroll
      for (int c = 0; c < 2 * NF; ++c) asm volatile("fma.rn.f32 %0, %0, %1, 0f38D1B717;" : "+f"(f[c]) : "f"(s));
    } else {
#pragma unroll
      for (int c = 0; c < NF; ++c) g[c] = ffma2<1>(g[c], s);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < NM; ++c) acc += m[c];
#pragma unroll
  for (int c = 0; c < NA; ++c) acc += __uint_as_float(a[c]);
#pragma unroll
  for (int c = 0; c < 2 * NF; ++c) acc += f[c];
#pragma unroll
  for (int c = 0; c < NF; ++c) acc += __uint_as_float((uint32_t)g[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// HBM: store-only (16-byte st.global.v4, grid-stride, one wave of 148 x 4 CTAs) and copy (v4 load + v4 store)
__global__ void store_kernel(float4* dst, size_t n4, float v) {
  const float4 q = make_float4(v, v, v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = q;
}
__global__ void copy_kernel(float4* dst, const float4* src, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
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

template <int OP>
void run2(const char* name, int sms, int threads, float* d_out, long long* d_cyc) {
  pipe2_kernel<OP><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  pipe2_kernel<OP><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)h[i];
  avg /= sms;
  const double instr = (double)threads * ITERS * CH;
  printf("{\"op\": \"%s\", \"threads_per_sm\": %d, \"thread_instr_per_clk_per_sm\": %.2f, "
         "\"fp32_fma_per_clk_per_sm\": %.2f}\n", name, threads, instr / avg, 2 * instr / avg);
}

template <int NM, int NF>
void runmix(int sms, int threads, float* d_out, long long* d_cyc) {
  mix_kernel<NM, NF><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  mix_kernel<NM, NF><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)h[i];
  avg /= sms;
  const double it = (double)threads * ITERS;
  printf("{\"op\": \"mix MUFU.EX2 x %d + FFMA2 x %d\", \"threads_per_sm\": %d, \"mufu_per_clk_per_sm\": %.2f, "
         "\"ffma2_instr_per_clk_per_sm\": %.2f, \"clk_per_thread_iter_x128\": %.3f}\n",
         NM, NF, threads, NM * it / avg, NF * it / avg, avg / it * 128.0);
}

template <int NM, int NA, int NF, int P>
void runmix2(int sms, int threads, float* d_out, long long* d_cyc) {
  mix2_kernel<NM, NA, NF, P><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  mix2_kernel<NM, NA, NF, P><<<sms, threads>>>(d_out, d_cyc, 0.999f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)h[i];
  avg /= sms;
  const double it = (double)threads * ITERS;
  printf("{\"op\": \"mix2 MUFU x %d + LOP3 x %d + %s\", \"threads_per_sm\": %d, "
         "\"clk_per_warp_iter_per_smsp\": %.3f}\n", NM, NA, P ? (NF == 4 ? "FFMA2 x 4" : NF == 8 ? "FFMA2 x 8" : "FFMA2 x 2")
         : (NF == 4 ? "FFMA x 8" : NF == 8 ? "FFMA x 16" : "FFMA x 4"), threads, avg / it * 128.0);
}

void run_hbm(int sms) {
  const size_t bytes = (size_t)8 << 30;   // 8 GiB >> 126 MB L2
  float4 *a = nullptr, *b = nullptr;
  if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&b, bytes) != cudaSuccess) {
    printf("{\"hbm\": \"alloc failed\"}\n");
    return;
  }
  const size_t n4 = bytes / 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int cta_per_sm : {2, 4, 8}) {
    const int grid = sms * cta_per_sm;
    float best_st = 1e30f, best_cp = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      store_kernel<<<grid, 256>>>(a, n4, 1.0f + r);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best_st) best_st = ms;
      cudaEventRecord(e0);
      copy_kernel<<<grid, 256>>>(b, a, n4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best_cp) best_cp = ms;
    }
    printf("{\"hbm\": \"v4 grid-stride, %d CTAs x 256 thr\", \"bytes\": %zu, \"store_only_GBps\": %.1f, "
           "\"copy_rw_GBps\": %.1f}\n", grid, bytes, bytes / (best_st * 1e6), 2.0 * bytes / (best_cp * 1e6));
  }
  cudaFree(a);
  cudaFree(b);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, sizeof(float) * sms * 1024);
  cudaMalloc(&d_cyc, sizeof(long long) * sms);
  for (int threads : {512, 1024}) {
    runmix2<0, 0, 8, 0>(sms, threads, d_out, d_cyc);
    runmix2<0, 0, 8, 1>(sms, threads, d_out, d_cyc);
    runmix2<0, 8, 4, 0>(sms, threads, d_out, d_cyc);
    runmix2<0, 8, 4, 1>(sms, threads, d_out, d_cyc);
    runmix2<0, 4, 4, 0>(sms, threads, d_out, d_cyc);
    runmix2<0, 4, 4, 1>(sms, threads, d_out, d_cyc);
    runmix2<1, 0, 4, 0>(sms, threads, d_out, d_cyc);
    runmix2<1, 0, 4, 1>(sms, threads, d_out, d_cyc);
    runmix2<1, 0, 2, 0>(sms, threads, d_out, d_cyc);
    runmix2<1, 0, 2, 1>(sms, threads, d_out, d_cyc);
    runmix2<1, 4, 2, 0>(sms, threads, d_out, d_cyc);
    runmix2<1, 4, 2, 1>(sms, threads, d_out, d_cyc);
    runmix2<0, 8, 0, 0>(sms, threads, d_out, d_cyc);
    run2<10>("FFMA2 (fma.rn.f32x2, packed operands)", sms, threads, d_out, d_cyc);
    run2<11>("FFMA2 (fma.rn.f32x2, scalar broadcast multiplier)", sms, threads, d_out, d_cyc);
    runmix<1, 0>(sms, threads, d_out, d_cyc);
    runmix<1, 2>(sms, threads, d_out, d_cyc);
    runmix<1, 4>(sms, threads, d_out, d_cyc);
    runmix<1, 6>(sms, threads, d_out, d_cyc);
    runmix<1, 8>(sms, threads, d_out, d_cyc);
    runmix<2, 8>(sms, threads, d_out, d_cyc);
    runmix<0, 8>(sms, threads, d_out, d_cyc);
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
    run<12>("ex2.approx.f16x2 (2 results/instr)", sms, threads, d_out, d_cyc);
    run<13>("tanh.approx.f16x2 (2 results/instr)", sms, threads, d_out, d_cyc);
    run<14>("mul.wide.u32 + LOP3 (IMAD.WIDE)", sms, threads, d_out, d_cyc);
    run<15>("FFMA all-register operands (+ LOP3)", sms, threads, d_out, d_cyc);
    run<16>("mul.lo.u32 imm (IMAD)", sms, threads, d_out, d_cyc);
    run<17>("mul.hi.u32 imm (IMAD.HI) + LOP3", sms, threads, d_out, d_cyc);
    run<18>("mul.wide.u32 imm (IMAD.WIDE) + IADD3", sms, threads, d_out, d_cyc);
  }
  run_hbm(sms);
  return 0;
}
