// sl7_tc.cu -- the tensor-core step kernel of the Seven-League path generator (sm_100a, tcgen05).
//
// Algorithm I steps 3-8 for tiles of 128 paths, all n_steps inside one launch:
//   layer 1 (rank 1 in Y after folding dt, theta)     : FFMA + activation, fp32, CUDA cores
//   hidden layers 2..L and the output layer            : tcgen05.mma kind::f16 (BF16: bf16 x bf16; SPLIT: three
//                                                        fp16 products of two-part operands) or kind::tf32,
//                                                        fp32 accumulate; [128 paths x 64] x [64 x 64] (output x 16)
//   bias + activation epilogue                         : tcgen05.ld -> MUFU.TANH (BF16 tanh), softplus pairs on
//                                                        MUFU ex2 + FFMA2 log1p polynomial / MUFU lg2, or the
//                                                        accurate FFMA2 pairs (SPLIT, TF32) -> pack -> tcgen05.st
//   Philox/Box-Muller normal, barycentric g_m, stats   : CUDA cores, as in the fp32 kernels
//
// CTA = NG independent "tile groups" of 4 warps (128 threads).  Thread t of a group owns path t of
// the group's current tile AND TMEM lane t: the MMA's M dimension is the path index, so every
// accumulator row a thread reads with tcgen05.ld.32x32b is its own path's pre-activations, and the
// activations it writes back with tcgen05.st become the A operand (A-from-TMEM) of the next MMA.
// No activation ever touches shared or global memory.  While one group waits for its MMA (mbarrier
// signalled by tcgen05.commit), the other groups run their MUFU-bound epilogues, which is where the
// time goes (the XU pipe binds, the tensor pipe has >= 5x slack).
//
// TMEM per group: [0,64) hidden accumulator fp32 (the [128 x 16] output accumulator reuses [0,16)), then the
// A operand: BF16 [64,96) (64 bf16 packed two per 32-bit column) -> 96 columns, 5 groups per SM; SPLIT two
// fp16 parts [64,128) and TF32 64 columns -> 128 columns, 4 groups.  Shared memory: the weight tiles in the
// SWIZZLE_128B K-major layout (staged once per CTA), the histogram, the per-thread statistics, barriers.
// (Experiment builds also hold the AS variants: the A operand, or SPLIT's lo part, in shared memory.)
#include <cuda_runtime.h>

#include "sl7_device.cuh"
#include "sl7_tc.cuh"

namespace sl7 {

namespace {
constexpr int kGroupThreads = 128;
constexpr uint32_t kColsPerGroup = 96;     // acc fp32 [0,64) (output layer reuses [0,16)), A bf16 [64,96)
constexpr uint32_t kAccCol = 0, kACol = 64;
}  // namespace

// 1/s for s in [1, 2] on the FMA pipe: quadratic seed (rel. error 1.7%) + 2 Newton steps (8e-8).
// Used to move part of the MUFU load (rcp) onto the FMA pipe (the XU pipe binds).
__device__ __forceinline__ float rcp12_newton(float s) {
  float r = fmaf(fmaf(0.30153724f, s, -1.39582404f), s, 2.08733358f);
  r = fmaf(r, fmaf(-s, r, 1.0f), r);
  r = fmaf(r, fmaf(-s, r, 1.0f), r);
  return r;
}

// Internal activation code of the TC kernel: tanh on the MUFU.TANH unit (tanh.approx.f32; measured on
// B200 at <= 9.9e-6 relative, 7.9e-6 absolute, far below the bf16 / tf32 rounding of the activation that
// follows), argument unscaled (act_scale 1).  The default tanh epilogue of the BF16 / TF32 modes.
constexpr int kActTanhX = 2;
__device__ __forceinline__ float tanh_mufu(float z) {
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(z));
  return r;
}

// Activation of the TC epilogue.  The argument is u = z * scale with scale = 2 log2(e) (tanh) or 1
// (softplus), folded on the host into layer 1 and into the biases.
//   tanh, 2 MUFU:      tanh = 1 - 2 / (2^u + 1)          (2^u -> 0 / inf gives -1 / 1 exactly)
//   tanh, 1 MUFU:      tanh|z| = (1 - e) / (1 + e), e = 2^-|u| in (0,1]: the denominator is in [1,2],
//                      so its reciprocal is rcp12_newton on the FMA pipe; sign restored by copysign
//   softplus, 2 MUFU:  max(z, 0) + ln2 log2(1 + 2^(-|z| log2 e))
// Absolute error <= ~2e-7 in every variant.
template <int ACT>
__device__ __forceinline__ float tc_act_u(float u, bool newton) {
  if constexpr (ACT == kActTanhX) {
    return tanh_mufu(u);
  } else if constexpr (ACT == SL7_ACT_TANH) {
    if (newton) {   // compile-time after unrolling
      const float e = ex2_approx(-fabsf(u));
      const float r = rcp12_newton(1.0f + e);
      return copysignf(fmaf(-e, r, r), u);
    }
    return fmaf(-2.0f, rcp_approx(ex2_approx(u) + 1.0f), 1.0f);
  } else {
    const float e = ex2_approx(fabsf(u) * -1.4426950408889634f);
    if (newton) {
      // log1p(e), e in (0, 1], as a degree-8 polynomial on the FMA pipe (abs. error 1.4e-7 in fp32)
      float lp = -6.301349960e-03f;
      lp = fmaf(lp, e, 3.544928879e-02f);
      lp = fmaf(lp, e, -9.422647208e-02f);
      lp = fmaf(lp, e, 1.666473895e-01f);
      lp = fmaf(lp, e, -2.402127683e-01f);
      lp = fmaf(lp, e, 3.316470385e-01f);
      lp = fmaf(lp, e, -4.998508692e-01f);
      lp = fmaf(lp, e, 9.999948740e-01f);
      lp = fmaf(lp, e, 2.928694798e-08f);
      return fmaxf(u, 0.0f) + lp;
    }
    return fmaf(0.69314718055994531f, lg2_approx(1.0f + e), fmaxf(u, 0.0f));
  }
}

// NMASK bit (unit % 8) set: this unit's second transcendental runs on the FMA pipe (tanh: reciprocal
// by Newton; softplus: log1p by polynomial), trading one MUFU op for ~6 FMA-pipe instructions.
template <int ACT, unsigned NMASK>
__device__ __forceinline__ bool use_newton(int c) {
  return (NMASK >> (c & 7)) & 1u;
}

// ---- paired softplus (kActSoftplusPair): two units per FFMA2 (fma.rn.f32x2, sm_100a).  FFMA2 has the
// FFMA FLOP rate at half the instructions and co-issues with MUFU better than FFMA (profiles/r02_pipes.md:
// 1 MUFU + 2 FFMA2 per warp-iteration 8.2 clk, 1 MUFU + 4 FFMA 10.1 clk; the MUFU bound is 8), so a pair
// whose log1p runs as a polynomial costs 1 MUFU per unit and ~9 FMA-pipe cycles, a pair on MUFU lg2 2 MUFU.
// NMASK bit (pair index % 8) selects the polynomial pairs.
constexpr int kActSoftplusPair = 4;

constexpr int kActTanhPair = 5;
constexpr int kActSoftplusPairS = 6;   // softplus pairs with a scaled accumulator (SPLIT: 2^-s)

__host__ __device__ constexpr bool is_pair_act(int act) {
  return act == kActSoftplusPair || act == kActTanhPair || act == kActSoftplusPairS;
}
__host__ __device__ constexpr int base_act(int act) {
  return act == kActTanhPair ? SL7_ACT_TANH : (is_pair_act(act) ? SL7_ACT_SOFTPLUS : act);
}

// one pair of units (c0, c0 + 1); NMASK bit (pair index % 8): polynomial log1p / Newton reciprocal.
// Softplus NMASK bit 8: the degree-7 log1p (BF16 only; the fp32-class modes keep degree 8).
template <int ACT, unsigned NMASK>
__device__ __forceinline__ void act_pair(float u0, float u1, int c0, float& h0, float& h1) {
  const bool alt = (NMASK >> ((c0 >> 1) & 7)) & 1u;
  if constexpr (ACT == kActTanhPair) {
    if (alt) tanh_pair<true>(u0, u1, h0, h1);
    else tanh_pair<false>(u0, u1, h0, h1);
  } else {
    if (alt) softplus_pair<true, (NMASK & 0x100u) != 0>(u0, u1, h0, h1);
    else softplus_pair<false>(u0, u1, h0, h1);
  }
}

// the pre-activation of a pair unit: BF16 softplus takes the accumulator as is (the host folds no scale);
// the others multiply by the layer's accumulator scale (FOLD) or add the scaled bias
template <int ACT, bool FOLD>
__device__ __forceinline__ float pair_u(float acc, float scale, const float* bs, int c) {
  if constexpr (ACT == kActSoftplusPair) return FOLD ? acc : acc + bs[c];
  else return FOLD ? acc * scale : fmaf(acc, scale, bs[c]);
}

// Pack two activations: NP = 1: bf16(h) (SL7_PREC_BF16).  NP = 2 (SL7_PREC_SPLIT): two fp16 parts,
// h0 = fp16(h), h1 = fp16(h - h0): h = h0 + h1 to 2^-22 relative (absolute 2^-25 where h1 falls into the
// binary16 subnormals), the fp32-class A operand of the three-product split MMA.
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void unpack_f16x2(uint32_t w, float& lo, float& hi) {
  asm("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\tcvt.f32.f16 %0, a;\n\tcvt.f32.f16 %1, b;\n\t}"
      : "=f"(lo), "=f"(hi) : "r"(w));
}

template <int NP, int NW>
__device__ __forceinline__ void split_pack(float a, float b, uint32_t (&pk)[NP][NW], int k) {
  static_assert(NP == 1 || NP == 2, "bf16 (1) or fp16 two-part (2)");
  if constexpr (NP == 1) {
    pk[0][k] = tc::pack_bf16x2(a, b);
  } else {
    const uint32_t w = pack_f16x2(a, b);
    float a0, b0;
    unpack_f16x2(w, a0, b0);
    pk[0][k] = w;
    pk[1][k] = pack_f16x2(a - a0, b - b0);
  }
}

// FOLD: the hidden bias rides in the MMA (K columns H, H+1, H+2 of A hold 1.0, the weight tile holds
// the bias split into three bf16 terms), so u = acc * scale.  Otherwise u = acc * scale + bias_scaled.
template <int ACT, int H, unsigned NMASK, bool FOLD, int NP, int NC = 32>
__device__ __forceinline__ void act_pack_32(const uint32_t (&v)[NC], int col0, float scale, const float* bs,
                                            uint32_t (&pk)[NP][NC / 2]) {
#pragma unroll
  for (int k = 0; k < NC / 2; ++k) {
    float h[2];
    const int c0 = col0 + 2 * k;
    if (is_pair_act(ACT) && c0 + 1 < H) {
      act_pair<ACT, NMASK>(pair_u<ACT, FOLD>(__uint_as_float(v[2 * k]), scale, bs, c0),
                           pair_u<ACT, FOLD>(__uint_as_float(v[2 * k + 1]), scale, bs, c0 + 1), c0, h[0], h[1]);
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = c0 + q;
        if (c < H) {
          const float acc = __uint_as_float(v[2 * k + q]);
          if constexpr (is_pair_act(ACT)) {
            h[q] = tc_act_u<base_act(ACT)>(pair_u<ACT, FOLD>(acc, scale, bs, c), true);
          } else {
            const float u = FOLD ? (ACT == kActTanhX ? acc : acc * scale) : fmaf(acc, scale, bs[c]);
            h[q] = tc_act_u<ACT>(u, use_newton<ACT, NMASK>(c));
          }
        } else {
          h[q] = (FOLD && c < H + 3) ? 1.0f : 0.0f;
        }
      }
    }
    split_pack<NP>(h[0], h[1], pk, k);
  }
}

// SL7_PREC_TF32: activations rounded to tf32 with cvt.rna (ties away, reading A-15), one 32-bit TMEM
// column per unit (the A operand of kind::tf32 is K-major fp32-width).
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

template <int ACT, int H, unsigned NMASK, bool FOLD>
__device__ __forceinline__ void act_tf32_32(const uint32_t (&v)[32], int col0, float scale, const float* bs,
                                            uint32_t (&w)[32]) {
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const int c0 = col0 + k;
    float h[2];
    if (is_pair_act(ACT) && c0 + 1 < H) {
      act_pair<ACT, NMASK>(pair_u<ACT, FOLD>(__uint_as_float(v[k]), scale, bs, c0),
                           pair_u<ACT, FOLD>(__uint_as_float(v[k + 1]), scale, bs, c0 + 1), c0, h[0], h[1]);
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = c0 + q;
        if (c < H) {
          const float acc = __uint_as_float(v[k + q]);
          if constexpr (is_pair_act(ACT)) {
            h[q] = tc_act_u<base_act(ACT)>(pair_u<ACT, FOLD>(acc, scale, bs, c), true);
          } else {
            const float u = FOLD ? (ACT == kActTanhX ? acc : acc * scale) : fmaf(acc, scale, bs[c]);
            h[q] = tc_act_u<ACT>(u, use_newton<ACT, NMASK>(c));
          }
        } else {
          h[q] = (FOLD && c < H + 3) ? 1.0f : 0.0f;
        }
      }
    }
    w[k] = tf32_rna(h[0]);
    w[k + 1] = tf32_rna(h[1]);
  }
}

// kind::tf32 MMA issue for one layer: K = 64 as 8 instructions of K = 8 (32 bytes of each K-major row).
// The weight tile is two SWIZZLE_128B K-blocks of [N rows][128 B] (K 0..31, then K 32..63), so K-step k
// reads block k / 4 at byte offset 32 (k % 4); the A operand advances 8 TMEM columns per K-step.
__device__ __forceinline__ void issue_layer_tf32(uint32_t acc_t, uint32_t a_t, uint32_t b_base, uint32_t n_rows,
                                                 uint32_t idesc) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint64_t bdesc = tc::smem_desc_sw128(b_base + (uint32_t)(k >> 2) * n_rows * 128u) + 2u * (uint32_t)(k & 3);
    tc::mma_tf32_ts(acc_t, a_t + 8u * k, bdesc, idesc, k > 0 ? 1u : 0u);
  }
}

// MMA issue for one layer: sum over (A part, B part) pairs of [128 x 64] x [64 x N] with K = 4 x 16.
// NP = 1: bf16 x bf16.  NP = 2 (fp16 parts): h0 W0 + h0 W1 + h1 W0 -- the dropped h1 W1 is 2^-22 of the
// leading product, so the layer is fp32-class from three f16 tensor-core products.
template <int NP>
__device__ __forceinline__ void issue_layer(uint32_t acc_t, uint32_t a_t, uint32_t b_base, uint32_t b_part_bytes,
                                            uint32_t idesc) {
  constexpr int NPAIR = (NP == 1) ? 1 : 3;
  constexpr int PA[3] = {0, 0, 1};
  constexpr int PB[3] = {0, 1, 0};
#pragma unroll
  for (int pr = 0; pr < NPAIR; ++pr) {
    const uint64_t bdesc = tc::smem_desc_sw128(b_base + (uint32_t)PB[pr] * b_part_bytes);
    const uint32_t a = a_t + 32u * PA[pr];
#pragma unroll
    for (int k = 0; k < kTcN / 16; ++k)   // +32 bytes per K step inside the 128-byte swizzle atom
      tc::mma_bf16_ts(acc_t, a + 8u * k, bdesc + 2u * k, idesc, (pr > 0 || k > 0) ? 1u : 0u);
  }
}

// AS (A operand in shared memory): thread row r of the group's [128 x 64] bf16 A tile, SWIZZLE_128B K-major
// (the layout of the weight tiles): row r at (r / 8) 1024 + (r % 8) 128 bytes, its 16-byte chunk c (columns
// 8c .. 8c+7) at chunk position c ^ (r % 8).  NW packed words = NW / 4 chunks starting at chunk c0.
template <int NW>
__device__ __forceinline__ void st_a_row(uint32_t row_base, uint32_t r7, int c0, const uint32_t (&w)[NW]) {
#pragma unroll
  for (int q = 0; q < NW / 4; ++q)
    tc::st_shared_v4(row_base + ((((uint32_t)(c0 + q)) ^ r7) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

template <int NG, int H, int MR, bool RT_M, int ACT, unsigned NMASK, int NP = 1, bool SKIPMMA = false, bool TF32 = false,
          bool AS = false>
__global__ void __launch_bounds__(NG * kGroupThreads, 1)
    ann_tc_step_kernel(const __grid_constant__ RunParams p, const __grid_constant__ TcParams t) {
  // epilogue in quarters of 16 columns (paired softplus, NMASK bit 9); the A columns of a quarter that is
  // not stored keep the layer-1 values (all such columns are zero padding: the same on every layer)
  constexpr bool QUARTERS = (ACT == kActSoftplusPair) && (NMASK & 0x200u) && !TF32;
  // NMASK bit 10 (with QUARTERS): software-pipelined quarters -- the TMEM load of quarter q+1 is issued before
  // quarter q's activations are computed, so its latency hides behind them (two 16-value buffers live)
  constexpr bool QPIPE = QUARTERS && (NMASK & 0x400u);
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mbar[NG];   // per group: MMA completion (tcgen05.commit)
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[8];

  const int warp = threadIdx.x >> 5;
  const int g = warp >> 2;                 // tile group
  const int wq = warp & 3;                 // warp within the group -> TMEM lanes [32 wq, 32 wq + 32)
  const int tid_g = threadIdx.x & (kGroupThreads - 1);
  static_assert(!TF32 || NP == 1, "TF32 has one operand part");
  static_assert(!AS || !TF32, "A in shared memory: the 16-bit kernels");
  // acc fp32 [0,64) + A (NP 16-bit parts | tf32) in TMEM.  AS: the LAST 16-bit part lives in shared memory (BF16:
  // the only part, TMEM holds the accumulator alone; SPLIT: part 0 stays in TMEM, part 1 moves out -> 96 columns)
  constexpr int NPT = AS ? NP - 1 : NP;   // operand parts in TMEM
  constexpr uint32_t kCols = kAccCol + 64u + (TF32 ? 64u : 32u * NPT);
  constexpr uint32_t kTileB = TF32 ? 2u * kTcTileBytes : (uint32_t)kTcTileBytes;   // bytes per weight tile part
  constexpr uint32_t kOutB = TF32 ? 2u * kTcOutBytes : (uint32_t)kTcOutBytes;
  constexpr uint32_t kTmemCols = NG * kCols <= 256 ? 256u : 512u;
  static_assert(NG * kCols <= 512, "TMEM: 512 columns per SM");
  constexpr bool FOLD = (H <= kTcN - 3);   // biases ride in spare K columns (host image must match)

  // ---- one-time CTA setup: weights -> smem (1024-aligned for the 128B swizzle), barriers, TMEM
  const uint32_t sbase = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* wsm = smem_raw + (sbase - tc::smem_u32(smem_raw));
  const int nL = t.n_mma_hidden;
  const int wbytes = NP * (nL * (int)kTileB + (int)kOutB);
  constexpr int kATileBytes = 128 * 128;   // AS: [128 rows][64 bf16] per group
  const int abytes = AS ? NG * kATileBytes : 0;
  uint32_t* hist = reinterpret_cast<uint32_t*>(wsm + wbytes + abytes);
  // per-thread running sums of the statistics live in shared memory ([8][threads], SoA), not in registers:
  // they change once per tile, and the 12 registers they would pin are worth more to the epilogue
  const int hist_words = (p.has_stats && p.n_bins > 0) ? ((p.n_bins + 2 + 1) & ~1) : 0;
  double* sst = reinterpret_cast<double*>(hist + hist_words);
  constexpr int kThreads = NG * kGroupThreads;
  if (p.has_stats)
    for (int k = 0; k < 8; ++k) sst[k * kThreads + threadIdx.x] = 0.0;
  {
    const uint4* src = reinterpret_cast<const uint4*>(TF32 ? t.wimg_tf32 : (NP == 1 ? t.wimg : t.wimg_split));
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
  if (warp == 0) tc::tmem_alloc(&tmem_base_sh, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t gcol = tbase + (uint32_t)g * kCols;
  const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
  const uint32_t acc_t = gcol + kAccCol, a_t = gcol + kACol;
  constexpr uint32_t idesc_h = TF32 ? tc::idesc_tf32_f32(128, kTcN)
                                    : (NP == 2 ? tc::idesc_f16_f32(128, kTcN) : tc::idesc_bf16_f32(128, kTcN));
  constexpr uint32_t idesc_o = TF32 ? tc::idesc_tf32_f32(128, kTcNOut)
                                    : (NP == 2 ? tc::idesc_f16_f32(128, kTcNOut) : tc::idesc_bf16_f32(128, kTcNOut));
  uint64_t* bar = &mbar[g];
  uint32_t phase = 0;
  // AS: the group's A tile (1024-aligned: the weight image is a multiple of 1024 bytes) and this thread's row
  const uint32_t a_s = sbase + (uint32_t)wbytes + (uint32_t)g * kATileBytes;
  const uint32_t a_row = a_s + ((uint32_t)tid_g >> 3) * 1024u + ((uint32_t)tid_g & 7u) * 128u;
  const uint32_t a_r7 = (uint32_t)tid_g & 7u;

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
      // BF16 / TF32 draw X_hat with the fast Box-Muller (|dX| <= 2e-6 (1 + |X|), far below the operand
      // rounding of these modes); SPLIT (fp32-class) keeps the libm one
      if ((i & 3) == 0) normals4_rk<(NP == 1)>(p, gp, (uint32_t)(i >> 2), z0, z1, z2, z3);
      const float Z = z0;
      z0 = z1; z1 = z2; z2 = z3;

      // ---- layer 1 (fp32, rank 1 in Y) -> A operand in TMEM, two 32-unit halves
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float h[32];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int c0 = 32 * half + k;
          if (is_pair_act(ACT) && c0 + 1 < H) {
            act_pair<ACT, NMASK>(fmaf(Y, t.l1w[c0], t.l1b[c0]), fmaf(Y, t.l1w[c0 + 1], t.l1b[c0 + 1]), c0, h[k],
                                 h[k + 1]);
          } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int c = c0 + q;
              h[k + q] = (c < H) ? tc_act_u<base_act(ACT)>(fmaf(Y, t.l1w[c], t.l1b[c]),
                                                           is_pair_act(ACT) || use_newton<ACT, NMASK>(c))
                                 : ((FOLD && c < H + 3) ? 1.0f : 0.0f);
            }
          }
        }
        if constexpr (TF32) {
          uint32_t w[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) w[k] = tf32_rna(h[k]);
          tc::tmem_st_32x32b_x32(a_t + lane_off + 32u * half, w);
        } else {
          uint32_t pk[NP][16];
#pragma unroll
          for (int k = 0; k < 16; ++k) split_pack<NP>(h[2 * k], h[2 * k + 1], pk, k);
#pragma unroll
          for (int part = 0; part < NPT; ++part)
            tc::tmem_st_32x32b_x16(a_t + 32u * part + lane_off + 16u * half, pk[part]);
          if constexpr (AS) st_a_row<16>(a_row, a_r7, 4 * half, pk[NP - 1]);
        }
      }
      if constexpr (AS) tc::fence_proxy_async_smem();
      if constexpr (NPT > 0 || TF32) tc::wait_st();
      // ---- layers 2..L+1 on the tensor cores; the Lagrange basis at Z (independent of the MLP)
      //      is computed while the first MMA runs
      float lb[MR], den = 1.0f, y[MR];
      for (int l = 0; l <= nL; ++l) {
        const bool last = (l == nL);
        tc::fence_before();
        tc::named_bar_sync(1 + g, kGroupThreads);
        if (tid_g == 0) {
          tc::fence_after();
          // weight image: NP parts of each hidden tile (8 KB), then NP parts of the output tile (2 KB).
          // (Issuing the hidden layers as two N = 32 halves with separate commits, to overlap the
          // epilogue of columns 0..31 with the MMAs of 32..63, measured slower: 1.38e10 vs 1.41e10.)
          if (SKIPMMA) {
            // timing experiment only (SL7_TC_VARIANT=9): same synchronisation, no tensor work
          } else if (TF32) {
            if (last) issue_layer_tf32(acc_t, a_t, sbase + (uint32_t)(nL * kTileB), kTcNOut, idesc_o);
            else issue_layer_tf32(acc_t, a_t, sbase + (uint32_t)(l * kTileB), kTcN, idesc_h);
          } else if (AS && NP == 1) {
            const uint64_t adesc = tc::smem_desc_sw128(a_s);
            const uint64_t bdesc = tc::smem_desc_sw128(sbase + (uint32_t)((last ? nL : l) * kTcTileBytes));
            const uint32_t idesc = last ? idesc_o : idesc_h;
#pragma unroll
            for (int k = 0; k < kTcN / 16; ++k)
              tc::mma_bf16_ss(acc_t, adesc + 2u * k, bdesc + 2u * k, idesc, k > 0 ? 1u : 0u);
          } else if (AS) {
            // SPLIT: h0 W0 + h0 W1 from the TMEM part, h1 W0 from the shared-memory part
            const uint32_t b0 = sbase + (uint32_t)(NP * (last ? nL : l) * kTcTileBytes);
            const uint32_t pb = last ? (uint32_t)kTcOutBytes : (uint32_t)kTcTileBytes;
            const uint32_t idesc = last ? idesc_o : idesc_h;
            const uint64_t bd0 = tc::smem_desc_sw128(b0), bd1 = tc::smem_desc_sw128(b0 + pb);
            const uint64_t ad1 = tc::smem_desc_sw128(a_s);
#pragma unroll
            for (int k = 0; k < kTcN / 16; ++k) tc::mma_bf16_ts(acc_t, a_t + 8u * k, bd0 + 2u * k, idesc, k > 0 ? 1u : 0u);
#pragma unroll
            for (int k = 0; k < kTcN / 16; ++k) tc::mma_bf16_ts(acc_t, a_t + 8u * k, bd1 + 2u * k, idesc, 1u);
#pragma unroll
            for (int k = 0; k < kTcN / 16; ++k) tc::mma_bf16_ss(acc_t, ad1 + 2u * k, bd0 + 2u * k, idesc, 1u);
          } else if (last) {
            issue_layer<NP>(acc_t, a_t, sbase + (uint32_t)(NP * nL * kTcTileBytes), kTcOutBytes, idesc_o);
          } else {
            issue_layer<NP>(acc_t, a_t, sbase + (uint32_t)(NP * l * kTcTileBytes), kTcTileBytes, idesc_h);
          }
          tc::mma_commit(bar);
        }
        if (l == 0) den = gm_basis<MR, RT_M>(p, Z, lb);
        tc::mbar_wait(bar, phase);
        phase ^= 1u;
        tc::fence_after();
        if (!last) {
          if constexpr (QPIPE) {
            constexpr int NQ = ((FOLD ? H + 3 : H) + 15) / 16;   // quarters holding live columns
            uint32_t va[16], vb[16];
            tc::tmem_ld_32x32b_x16(acc_t + lane_off, va);
            tc::wait_ld();
#pragma unroll
            for (int qt = 0; qt < NQ; ++qt) {
              uint32_t (&cur)[16] = (qt & 1) ? vb : va;
              uint32_t (&nxt)[16] = (qt & 1) ? va : vb;
              if (qt + 1 < NQ) tc::tmem_ld_32x32b_x16(acc_t + lane_off + 16u * (qt + 1), nxt);
              uint32_t pk[NP][8];
              act_pack_32<ACT, H, NMASK, FOLD, NP, 16>(cur, 16 * qt, t.lscale[l], t.bias[l], pk);
#pragma unroll
              for (int part = 0; part < NPT; ++part)
                tc::tmem_st_32x32b_x8(a_t + 32u * part + lane_off + 8u * qt, pk[part]);
              if constexpr (AS) st_a_row<8>(a_row, a_r7, 2 * qt, pk[NP - 1]);
              if (qt + 1 < NQ) tc::wait_ld();
            }
          } else if constexpr (QUARTERS) {
            // 16 columns at a time (fewer live registers: more pairs of the epilogue in flight); the
            // quarters past the last unit (and its 3 bias columns) are not loaded
#pragma unroll
            for (int qt = 0; qt < 4; ++qt) {
              if (16 * qt < (FOLD ? H + 3 : H)) {
                uint32_t v[16];
                tc::tmem_ld_32x32b_x16(acc_t + lane_off + 16u * qt, v);
                tc::wait_ld();
                uint32_t pk[NP][8];
                act_pack_32<ACT, H, NMASK, FOLD, NP, 16>(v, 16 * qt, t.lscale[l], t.bias[l], pk);
#pragma unroll
                for (int part = 0; part < NPT; ++part)
                  tc::tmem_st_32x32b_x8(a_t + 32u * part + lane_off + 8u * qt, pk[part]);
                if constexpr (AS) st_a_row<8>(a_row, a_r7, 2 * qt, pk[NP - 1]);
              }
            }
          } else {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tc::tmem_ld_32x32b_x32(acc_t + lane_off + 32u * half, v);
            tc::wait_ld();
            if constexpr (TF32) {
              uint32_t w[32];
              act_tf32_32<ACT, H, NMASK, FOLD>(v, 32 * half, t.lscale[l], t.bias[l], w);
              tc::tmem_st_32x32b_x32(a_t + lane_off + 32u * half, w);
            } else {
              uint32_t pk[NP][16];
              act_pack_32<ACT, H, NMASK, FOLD, NP>(v, 32 * half, t.lscale[l], t.bias[l], pk);
#pragma unroll
              for (int part = 0; part < NPT; ++part)
                tc::tmem_st_32x32b_x16(a_t + 32u * part + lane_off + 16u * half, pk[part]);
              if constexpr (AS) st_a_row<16>(a_row, a_r7, 4 * half, pk[NP - 1]);
            }
          }
          }
          if constexpr (AS) tc::fence_proxy_async_smem();
          if constexpr (NPT > 0 || TF32) tc::wait_st();
        } else {
          uint32_t v[16];
          tc::tmem_ld_32x32b_x16(acc_t + lane_off, v);
          tc::wait_ld();
#pragma unroll
          for (int j = 0; j < MR; ++j) {
            const float acc = (NP == 2) ? __uint_as_float(v[j]) * t.oscale : __uint_as_float(v[j]);
            y[j] = fmaf(p.res_y, Y, fmaf(FOLD ? acc : acc + t.bout[j], p.out_scale[j], p.out_shift[j]));
          }
        }
      }
      // ---- steps 5-6: Y_{i+1} = g_m(X_hat)
      Y = gm_combine<MR>(lb, den, y);
      ref_step(rs, p, Z);
      if (valid && p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q] = Y;
    }
    if (valid) {
      if (p.out_mode == kTerminal) p.out[q] = Y;
      if (p.has_stats) {
        StatAcc a;
        stat_add(a, p, Y, ref_final(rs, p), hist);
        const double v[8] = {a.s1, a.s2, a.s3, a.s4, a.e1, a.e2, (double)a.n, (double)a.nnf};
#pragma unroll
        for (int k = 0; k < 8; ++k) sst[k * kThreads + threadIdx.x] += v[k];
      }
    }
  }
  if (p.has_stats) {
    StatAcc acc;
    acc.s1 = sst[0 * kThreads + threadIdx.x];
    acc.s2 = sst[1 * kThreads + threadIdx.x];
    acc.s3 = sst[2 * kThreads + threadIdx.x];
    acc.s4 = sst[3 * kThreads + threadIdx.x];
    acc.e1 = sst[4 * kThreads + threadIdx.x];
    acc.e2 = sst[5 * kThreads + threadIdx.x];
    acc.n = (uint32_t)sst[6 * kThreads + threadIdx.x];
    acc.nnf = (uint32_t)sst[7 * kThreads + threadIdx.x];
    stat_flush(acc, p, hist, red);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, kTmemCols);
}

namespace {

template <int NG, int H, int MR, bool RT, int ACT, unsigned NMASK = 0u, int NP = 1, bool SKIP = false, bool TF32 = false,
          bool AS = false>
cudaError_t launch_tc_t(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  auto kernel = ann_tc_step_kernel<NG, H, MR, RT, ACT, NMASK, NP, SKIP, TF32, AS>;
  const size_t hist = (p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)((p.n_bins + 2 + 1) & ~1) : 0;
  const size_t sst = p.has_stats ? sizeof(double) * 8 * NG * kGroupThreads : 0;
  const size_t tile_b = TF32 ? 2 * kTcTileBytes : kTcTileBytes, out_b = TF32 ? 2 * kTcOutBytes : kTcOutBytes;
  const size_t smem = 1024 + (size_t)NP * ((size_t)t.n_mma_hidden * tile_b + out_b) + (AS ? (size_t)NG * 128 * 128 : 0) +
                      hist + sst;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint64_t tiles = (p.n_paths + kGroupThreads - 1) / kGroupThreads;
  const uint64_t need = (tiles + NG - 1) / NG;
  const unsigned grid = (unsigned)(need < (uint64_t)num_sms ? need : (uint64_t)num_sms);
  kernel<<<grid, NG * kGroupThreads, smem, st>>>(p, t);
  return cudaGetLastError();
}

// Tile groups per CTA and the split of tanh units between the MUFU reciprocal and the FMA-pipe
// reciprocal (NMASK bit (unit % 8)), chosen by measurement on B200 (cfg1, 4 groups,
// half of the units on the FMA pipe: 1.45e10 path-steps/s vs 1.30e10 all-MUFU).
constexpr int kTcGroups = 4;
constexpr unsigned kTanhNewtonMask = 0x55u;
constexpr unsigned kSoftplusPolyMask = 0x55u;

// SL7_PREC_SPLIT: two fp16 parts per operand (TMEM 64 + 2 x 32 = 128 columns per group -> 4 groups).
constexpr int kTcGroupsSplit = 4;

// softplus (2 MUFU ops per unit on half of the units): 5 groups per SM, as for tanh (cfg2: 1.03e10 vs 9.4e9)
constexpr int kTcGroupsSoftplus = 5;

template <int ACT>
cudaError_t launch_tc_act(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms);

// softplus, BF16: paired epilogue; polynomial log1p on the pairs of kSoftplusPairMask (bit = pair index % 8)
constexpr unsigned kSoftplusPairMask = 0x15Fu;

template <unsigned PM>
cudaError_t launch_sp_pair(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  constexpr int NG = kTcGroupsSoftplus;
  if (p.width == 50 && p.m == 5) return launch_tc_t<NG, 50, 5, false, kActSoftplusPair, PM>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 7) return launch_tc_t<NG, 50, 7, false, kActSoftplusPair, PM>(p, t, st, num_sms);
  return launch_tc_t<NG, 64, kMaxM, true, kActSoftplusPair, PM>(p, t, st, num_sms);
}

cudaError_t launch_softplus_bf16(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
#ifdef SL7_AB_HOOKS
  switch (t.variant) {   // A/B hook (SL7_TC_VARIANT): share of polynomial pairs, or the r01 epilogue
    case 20: return launch_sp_pair<0x00u>(p, t, st, num_sms);
    case 21: return launch_sp_pair<0x55u>(p, t, st, num_sms);
    case 22: return launch_sp_pair<0x77u>(p, t, st, num_sms);
    case 23: return launch_sp_pair<0x7Fu>(p, t, st, num_sms);
    case 24: return launch_sp_pair<0xFFu>(p, t, st, num_sms);
    case 25: return launch_tc_act<SL7_ACT_SOFTPLUS>(p, t, st, num_sms);
    case 26: return launch_sp_pair<0x177u>(p, t, st, num_sms);
    case 27: return launch_sp_pair<0x17Fu>(p, t, st, num_sms);
    case 28: return launch_sp_pair<0x1FFu>(p, t, st, num_sms);
    case 29: return launch_sp_pair<0x15Fu>(p, t, st, num_sms);
    case 30: return launch_sp_pair<0x13Fu>(p, t, st, num_sms);
    case 31: return launch_sp_pair<0x1DFu>(p, t, st, num_sms);
    case 32: return launch_sp_pair<0x15Bu>(p, t, st, num_sms);
    case 33: return launch_sp_pair<0x1F7u>(p, t, st, num_sms);
    case 34: return launch_sp_pair<0x35Fu>(p, t, st, num_sms);
    case 35: return launch_sp_pair<0x377u>(p, t, st, num_sms);
    case 36: return launch_sp_pair<0x3FFu>(p, t, st, num_sms);
    case 37: return launch_tc_t<kTcGroupsSoftplus, 50, 7, false, kActSoftplusPair, 0x15Fu, 1, true>(p, t, st, num_sms);
    case 38: return launch_tc_t<4, 50, 7, false, kActSoftplusPair, 0x15Fu>(p, t, st, num_sms);
    // A operand in shared memory: 64 TMEM columns per tile, 6 / 7 tile groups per SM
    case 48: return launch_sp_pair<0x75Fu>(p, t, st, num_sms);   // pipelined quarters
    case 49: return launch_sp_pair<0x777u>(p, t, st, num_sms);
    case 50: return launch_sp_pair<0x77Fu>(p, t, st, num_sms);
    case 51: return launch_sp_pair<0x71Fu>(p, t, st, num_sms);
    case 39: return launch_tc_t<6, 50, 7, false, kActSoftplusPair, 0x15Fu, 1, false, false, true>(p, t, st, num_sms);
    case 44: return launch_tc_t<7, 50, 7, false, kActSoftplusPair, 0x15Fu, 1, false, false, true>(p, t, st, num_sms);
    case 45: return launch_tc_t<5, 50, 7, false, kActSoftplusPair, 0x15Fu, 1, false, false, true>(p, t, st, num_sms);
    case 46: return launch_tc_t<6, 50, 7, false, kActSoftplusPair, 0x35Fu, 1, false, false, true>(p, t, st, num_sms);
    case 47: return launch_tc_t<7, 50, 7, false, kActSoftplusPair, 0x35Fu, 1, false, false, true>(p, t, st, num_sms);
    default: break;
  }
#endif
  return launch_sp_pair<kSoftplusPairMask>(p, t, st, num_sms);
}

// SL7_PREC_SPLIT / TF32: accurate activations in FFMA2 pairs; NMASK bit (pair % 8) = Newton reciprocal
// (tanh) / polynomial log1p (softplus, degree 8) on that pair, the others on MUFU
constexpr unsigned kSplitTanhMask = 0x77u;
constexpr unsigned kSplitSoftplusMask = 0x7Fu;

template <int NG, int PACT, unsigned PM, int NP, bool TF32>
cudaError_t launch_pairs(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  if (p.width == 50 && p.m == 5) return launch_tc_t<NG, 50, 5, false, PACT, PM, NP, false, TF32>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 7) return launch_tc_t<NG, 50, 7, false, PACT, PM, NP, false, TF32>(p, t, st, num_sms);
  return launch_tc_t<NG, 64, kMaxM, true, PACT, PM, NP, false, TF32>(p, t, st, num_sms);
}

template <int NG, int NP, bool TF32>
cudaError_t launch_accurate(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  const bool tanh = (p.act == SL7_ACT_TANH);
#ifdef SL7_AB_HOOKS
  switch (t.variant) {   // A/B hook: share of Newton / polynomial pairs
    case 40: return tanh ? launch_pairs<NG, kActTanhPair, 0x55u, NP, TF32>(p, t, st, num_sms)
                         : launch_pairs<NG, kActSoftplusPairS, 0x55u, NP, TF32>(p, t, st, num_sms);
    case 41: return tanh ? launch_pairs<NG, kActTanhPair, 0x7Fu, NP, TF32>(p, t, st, num_sms)
                         : launch_pairs<NG, kActSoftplusPairS, 0x7Fu, NP, TF32>(p, t, st, num_sms);
    case 42: return tanh ? launch_pairs<NG, kActTanhPair, 0xFFu, NP, TF32>(p, t, st, num_sms)
                         : launch_pairs<NG, kActSoftplusPairS, 0xFFu, NP, TF32>(p, t, st, num_sms);
    case 43: return tanh ? launch_pairs<NG, kActTanhPair, 0x5Fu, NP, TF32>(p, t, st, num_sms)
                         : launch_pairs<NG, kActSoftplusPairS, 0x5Fu, NP, TF32>(p, t, st, num_sms);
    case 55:   // SPLIT with the lo part in shared memory: 96 TMEM columns per group, 5 groups
      if constexpr (NP == 2 && !TF32) {
        if (p.width == 50 && p.m == 7)
          return tanh ? launch_tc_t<5, 50, 7, false, kActTanhPair, kSplitTanhMask, 2, false, false, true>(p, t, st, num_sms)
                      : launch_tc_t<5, 50, 7, false, kActSoftplusPairS, kSplitSoftplusMask, 2, false, false, true>(p, t, st, num_sms);
      }
      break;
    case 56:   // the same with 4 groups (the cost of the shared-memory part alone)
      if constexpr (NP == 2 && !TF32) {
        if (p.width == 50 && p.m == 7)
          return tanh ? launch_tc_t<4, 50, 7, false, kActTanhPair, kSplitTanhMask, 2, false, false, true>(p, t, st, num_sms)
                      : launch_tc_t<4, 50, 7, false, kActSoftplusPairS, kSplitSoftplusMask, 2, false, false, true>(p, t, st, num_sms);
      }
      break;
    default: break;
  }
#endif
  return tanh ? launch_pairs<NG, kActTanhPair, kSplitTanhMask, NP, TF32>(p, t, st, num_sms)
              : launch_pairs<NG, kActSoftplusPairS, kSplitSoftplusMask, NP, TF32>(p, t, st, num_sms);
}

template <int ACT>
cudaError_t launch_tc_act(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  constexpr int NG = (ACT == SL7_ACT_SOFTPLUS) ? kTcGroupsSoftplus : kTcGroups;
  constexpr unsigned NM = (ACT == SL7_ACT_TANH) ? kTanhNewtonMask : kSoftplusPolyMask;
  if (t.split) return launch_accurate<kTcGroupsSplit, 2, false>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 5) return launch_tc_t<NG, 50, 5, false, ACT, NM>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 7) {
    switch (t.variant) {   // A/B hook (SL7_TC_VARIANT): fraction of units with the FMA-pipe transcendental
      case 1: return launch_tc_t<NG, 50, 7, false, ACT, 0x00u>(p, t, st, num_sms);
      case 2: return launch_tc_t<NG, 50, 7, false, ACT, 0x25u>(p, t, st, num_sms);
      case 3: return launch_tc_t<NG, 50, 7, false, ACT, 0x77u>(p, t, st, num_sms);
#ifdef SL7_AB_HOOKS
      case 9: return launch_tc_t<NG, 50, 7, false, ACT, NM, 1, true>(p, t, st, num_sms);   // timing only
#endif
      default: return launch_tc_t<NG, 50, 7, false, ACT, NM>(p, t, st, num_sms);
    }
  }
  return launch_tc_t<NG, 64, kMaxM, true, ACT, NM>(p, t, st, num_sms);
}

// tanh on MUFU.TANH (kActTanhX): all units on the MUFU unit.  The epilogue is short, so the share of time
// a group waits for its MMA grows; 5 groups per SM (480 of 512 TMEM columns, <= 96 registers) keep the MUFU
// unit fed better than 4 (cfg1: 2.28e10 vs 2.18e10 path-steps/s).
constexpr int kTcGroupsTanhX = 5;

cudaError_t launch_tc_act_x(const RunParams& p, const TcParams& t, cudaStream_t st, int num_sms) {
  constexpr int NG = kTcGroupsTanhX;
  constexpr unsigned NM = 0x00u;
  // (SPLIT never takes MUFU.TANH: the host clears tanh_mufu for it)
  if (p.width == 50 && p.m == 5) return launch_tc_t<NG, 50, 5, false, kActTanhX, NM>(p, t, st, num_sms);
  if (p.width == 50 && p.m == 7) return launch_tc_t<NG, 50, 7, false, kActTanhX, NM>(p, t, st, num_sms);
  return launch_tc_t<NG, 64, kMaxM, true, kActTanhX, NM>(p, t, st, num_sms);
}

}  // namespace

// SL7_PREC_TF32: TMEM 64 + 64 columns per group -> 4 groups (512 columns)
constexpr int kTcGroupsTf32 = 4;


int launch_tc_kernel(const RunParams& p, const TcParams& t, void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // TF32 takes its rna rounding decisions on an accurate tanh (ex2 + reciprocal, ~2e-7 absolute): MUFU.TANH's
  // 1e-5 flips a few tf32 roundings of the one shared step-0 evaluation, which shifts every path's points
  // together (reading R-15), so the tf32 moments would not match O6 on the identical path set (T-4)
  if (t.tf32) return (int)launch_accurate<kTcGroupsTf32, 1, true>(p, t, st, num_sms);
  if (p.act == SL7_ACT_TANH && t.tanh_mufu) {
    return (int)launch_tc_act_x(p, t, st, num_sms);
  }
  if (p.act == SL7_ACT_SOFTPLUS && !t.split) return (int)launch_softplus_bf16(p, t, st, num_sms);
  return (int)(p.act == SL7_ACT_TANH ? launch_tc_act<SL7_ACT_TANH>(p, t, st, num_sms)
                                     : launch_tc_act<SL7_ACT_SOFTPLUS>(p, t, st, num_sms));
}

}  // namespace sl7
