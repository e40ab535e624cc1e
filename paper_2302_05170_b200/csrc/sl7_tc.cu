// sl7_tc.cu -- the tensor-core step kernel of the Seven-League path generator (sm_100a, tcgen05).
//
// Algorithm I steps 3-8 for tiles of 128 paths, all n_steps inside one launch:
//   layer 1 (rank 1 in Y after folding dt, theta)     : FFMA + activation, fp32, CUDA cores
//   hidden layers 2..L and the output layer            : tcgen05.mma kind::f16, bf16 x bf16 -> fp32
//                                                        [128 paths x 64] x [64 x 64] (output: x 16)
//   bias + activation epilogue                         : tcgen05.ld -> FADD + MUFU -> bf16 -> tcgen05.st
//   Philox/Box-Muller normal, barycentric g_m, store   : CUDA cores, as in the fp32 kernels
//
// CTA = NG independent "tile groups" of 4 warps (128 threads).  Thread t of a group owns path t of
// the group's current tile AND TMEM lane t: the MMA's M dimension is the path index, so every
// accumulator row a thread reads with tcgen05.ld.32x32b is its own path's pre-activations, and the
// activations it writes back with tcgen05.st become the A operand (A-from-TMEM) of the next MMA.
// No activation ever touches shared or global memory.  While one group waits for its MMA (mbarrier
// signalled by tcgen05.commit), the other groups run their MUFU-bound epilogues, which is where the
// time goes (the XU pipe binds, the tensor pipe has >= 5x slack).
//
// TMEM per group (128 columns): [0,64) hidden accumulator fp32, [64,80) output accumulator fp32,
// [96,128) A operand (64 bf16 packed two per 32-bit column).  Shared memory: bf16 weight tiles in the
// SWIZZLE_128B K-major layout (staged once per CTA), the histogram, barriers.
#include <cuda_runtime.h>

#include "sl7_device.cuh"
#include "sl7_tc.cuh"

namespace sl7 {

namespace {
constexpr int kGroupThreads = 128;
constexpr uint32_t kColsPerGroup = 128;
constexpr uint32_t kAccCol = 0, kOutCol = 64, kACol = 96;
}  // namespace

template <int ACT, int H>
__device__ __forceinline__ void act_pack_32(const uint32_t (&v)[32], int col0, const float* bias, uint32_t (&pk)[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c0 = col0 + 2 * k, c1 = c0 + 1;
    const float a = (c0 < H) ? activate<ACT>(__uint_as_float(v[2 * k]) + bias[c0]) : 0.0f;
    const float b = (c1 < H) ? activate<ACT>(__uint_as_float(v[2 * k + 1]) + bias[c1]) : 0.0f;
    pk[k] = tc::pack_bf16x2(a, b);
  }
}

template <int NG, int H, int MR, bool RT_M, int ACT>
__global__ void __launch_bounds__(NG * kGroupThreads, 1)
    ann_tc_step_kernel(const __grid_constant__ RunParams p, const __grid_constant__ TcParams t) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mbar[NG];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[8];

  const int warp = threadIdx.x >> 5;
  const int g = warp >> 2;                 // tile group
  const int wq = warp & 3;                 // warp within the group -> TMEM lanes [32 wq, 32 wq + 32)
  const int tid_g = threadIdx.x & (kGroupThreads - 1);

  // ---- one-time CTA setup: weights -> smem (1024-aligned for the 128B swizzle), barriers, TMEM
  const uint32_t sbase = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* wsm = smem_raw + (sbase - tc::smem_u32(smem_raw));
  const int nL = t.n_mma_hidden;
  const int wbytes = nL * kTcTileBytes + kTcOutBytes;
  uint32_t* hist = reinterpret_cast<uint32_t*>(wsm + wbytes);
  {
    const uint4* src = reinterpret_cast<const uint4*>(t.wimg);
    uint4* dst = reinterpret_cast<uint4*>(wsm);
    for (int i = threadIdx.x; i < wbytes / 16; i += blockDim.x) dst[i] = src[i];
  }
  hist_init(p, hist);
  tc::fence_proxy_async_smem();            // generic-proxy smem writes -> visible to the tensor core
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NG; ++k) tc::mbar_init(&mbar[k], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base_sh, NG <= 2 ? 256u : 512u);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t gcol = tbase + (uint32_t)g * kColsPerGroup;
  const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
  const uint32_t acc_t = gcol + kAccCol, out_t = gcol + kOutCol, a_t = gcol + kACol;
  constexpr uint32_t idesc_h = tc::idesc_bf16_f32(128, kTcN);
  constexpr uint32_t idesc_o = tc::idesc_bf16_f32(128, kTcNOut);
  uint64_t* bar = &mbar[g];
  uint32_t phase = 0;

  StatAcc acc;
  const uint64_t n_tiles = (p.n_paths + kGroupThreads - 1) / kGroupThreads;
  for (uint64_t tile = (uint64_t)blockIdx.x * NG + g; tile < n_tiles; tile += (uint64_t)gridDim.x * NG) {
    const uint64_t q = tile * kGroupThreads + tid_g;
    const bool valid = q < p.n_paths;
    const uint64_t gp = p.path_offset + (valid ? q : 0);
    float Y = p.y0;
    if (valid && p.out_mode == kFull) p.out[q] = Y;
    RefState rs;
    ref_init(rs, p);
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    for (int i = 0; i < p.n_steps; ++i) {
      if ((i & 3) == 0) normals4(p.key0, p.key1, gp, (uint32_t)(i >> 2), z0, z1, z2, z3);
      const float Z = z0;
      z0 = z1; z1 = z2; z2 = z3;

      // ---- layer 1 (fp32) -> A operand in TMEM
      {
        uint32_t pk[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int c0 = 2 * k, c1 = 2 * k + 1;
          const float a = (c0 < H) ? activate<ACT>(fmaf(p.l1w[c0], Y, p.l1b[c0])) : 0.0f;
          const float b = (c1 < H) ? activate<ACT>(fmaf(p.l1w[c1], Y, p.l1b[c1])) : 0.0f;
          pk[k] = tc::pack_bf16x2(a, b);
        }
        tc::tmem_st_32x32b_x32(a_t + lane_off, pk);
        tc::wait_st();
      }
      // ---- layers 2..L+1 on the tensor cores
      float y[MR];
      for (int l = 0; l <= nL; ++l) {
        const bool last = (l == nL);
        tc::fence_before();
        tc::named_bar_sync(1 + g, kGroupThreads);
        if (tid_g == 0) {
          tc::fence_after();
          const uint64_t bdesc = tc::smem_desc_sw128(sbase + (uint32_t)l * kTcTileBytes);
          const uint32_t d = last ? out_t : acc_t;
          const uint32_t id = last ? idesc_o : idesc_h;
#pragma unroll
          for (int k = 0; k < kTcN / 16; ++k)   // K = 64 = 4 x 16; +32 bytes per K step inside the swizzle atom
            tc::mma_bf16_ts(d, a_t + 8u * k, bdesc + 2u * k, id, k > 0 ? 1u : 0u);
          tc::mma_commit(bar);
        }
        tc::mbar_wait(bar, phase);
        phase ^= 1u;
        tc::fence_after();
        if (!last) {
          uint32_t pk[32];
          {
            uint32_t v[32];
            tc::tmem_ld_32x32b_x32(acc_t + lane_off, v);
            tc::wait_ld();
            uint32_t h[16];
            act_pack_32<ACT, H>(v, 0, t.bias[l], h);
#pragma unroll
            for (int k = 0; k < 16; ++k) pk[k] = h[k];
          }
          if (H > 32) {
            uint32_t v[32];
            tc::tmem_ld_32x32b_x32(acc_t + lane_off + 32, v);
            tc::wait_ld();
            uint32_t h[16];
            act_pack_32<ACT, H>(v, 32, t.bias[l], h);
#pragma unroll
            for (int k = 0; k < 16; ++k) pk[16 + k] = h[k];
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) pk[16 + k] = 0u;
          }
          tc::tmem_st_32x32b_x32(a_t + lane_off, pk);
          tc::wait_st();
        } else {
          uint32_t v[16];
          tc::tmem_ld_32x32b_x16(out_t + lane_off, v);
          tc::wait_ld();
#pragma unroll
          for (int j = 0; j < MR; ++j) y[j] = fmaf(__uint_as_float(v[j]) + t.bout[j], p.out_scale[j], p.out_shift[j]);
        }
      }
      // ---- steps 5-6: Y_{i+1} = g_m(X_hat)
      Y = gm_eval<MR, RT_M>(p, Z, y);
      ref_step(rs, p, Z);
      if (valid && p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q] = Y;
    }
    if (valid) {
      if (p.out_mode == kTerminal) p.out[q] = Y;
      if (p.has_stats) stat_add(acc, p, Y, ref_final(rs, p), hist);
    }
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, NG <= 2 ? 256u : 512u);
}

namespace {

template <int NG, int H, int MR, bool RT, int ACT>
cudaError_t launch_tc_t(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  auto kernel = ann_tc_step_kernel<NG, H, MR, RT, ACT>;
  const size_t hist = (p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0;
  const size_t smem = 1024 + (size_t)t.n_mma_hidden * kTcTileBytes + kTcOutBytes + hist;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint64_t tiles = (p.n_paths + kGroupThreads - 1) / kGroupThreads;
  const uint64_t need = (tiles + NG - 1) / NG;
  const unsigned grid = (unsigned)(need < (uint64_t)num_sms ? need : (uint64_t)num_sms);
  kernel<<<grid, NG * kGroupThreads, smem, st>>>(p, t);
  return cudaGetLastError();
}

template <int ACT>
cudaError_t launch_tc_act(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  constexpr int NG = 4;
  if (p.width == 50 && p.m == 5) return launch_tc_t<NG, 50, 5, false, ACT>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 7) return launch_tc_t<NG, 50, 7, false, ACT>(p, t, st, num_sms);
  return launch_tc_t<NG, 64, kMaxM, true, ACT>(p, t, st, num_sms);
}

}  // namespace

int launch_tc_kernel(const RunParams& p, const TcParams& t, void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return (int)(p.act == SL7_ACT_TANH ? launch_tc_act<SL7_ACT_TANH>(p, t, st, num_sms)
                                     : launch_tc_act<SL7_ACT_SOFTPLUS>(p, t, st, num_sms));
}

}  // namespace sl7
