// sl7_kernels.cu -- CUDA-core step kernels for sm_100a:
//   * exact-collocation kernel (GBM / OU closed-form H_j, BASELINE north_star + Eq. 6.6)
//   * ANN-FP32 kernel ("exact mode" MLP on the FMA pipe, weights staged in shared memory)
//   * RNG verification kernels (raw Philox words, normals)
//
// Persistent grid-stride design: one thread owns one path for ALL n_steps (Algorithm I steps 3-8
// run without leaving the kernel: state Y in a register, no host round trip per step, no HBM
// traffic except the optional path output).  Consecutive threads own consecutive paths, so a
// FULL-mode store of step i by a warp is one contiguous 128-byte segment of row i.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sl7_device.cuh"

namespace sl7 {

// ------------------------------------------------------------------------------------------------
// Exact-collocation step kernel.  y_j = H_j(Y) in closed form, then g_m(Z).
// ------------------------------------------------------------------------------------------------
// SPECIAL (SL7_FLAG_SPECIALIZED): same interpolant through the exact points, evaluated in closed form:
// GBM g_m(Z) = Y * Q(Z) with Q in monomial form (Horner, MR-1 FFMA); OU g_m(Z) = mean + std * Z.
// FAST (SL7_FLAG_FAST_NORMALS): MUFU Box-Muller.  With both, a path-step is ~30 instructions and the
// FULL-output kernel approaches the HBM store roofline (4 B per path-step).
template <int MR, bool RT_M, int COLLOC, bool FAST = false, bool SPECIAL = false>
__global__ void __launch_bounds__(256) exact_step_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  hist_init(p, hist);
  __syncthreads();
  StatAcc acc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_paths; q += stride) {
    const uint64_t gp = p.path_offset + q;
    float Y = p.y0;
    if (p.out_mode == kFull) p.out[q] = Y;
    RefState rs;
    ref_init(rs, p);
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    for (int i = 0; i < p.n_steps; ++i) {
      if ((i & 3) == 0) normals4<FAST>(p.key0, p.key1, gp, (uint32_t)(i >> 2), z0, z1, z2, z3);
      const float Z = z0;
      z0 = z1; z1 = z2; z2 = z3;
      if constexpr (SPECIAL) {
        if constexpr (COLLOC == kExactGbm) {
          float qz = p.q[MR - 1];
#pragma unroll
          for (int k = MR - 2; k >= 0; --k) qz = fmaf(qz, Z, p.q[k]);
          Y *= qz;
        } else {
          Y = fmaf(p.ou_s, Z, fmaf(p.ou_a, Y, p.ou_b));
        }
      } else {
        float y[MR];
        if constexpr (COLLOC == kExactGbm) {
#pragma unroll
          for (int j = 0; j < MR; ++j) y[j] = Y * p.c[j];
        } else {
          const float mean = fmaf(p.ou_a, Y, p.ou_b);
#pragma unroll
          for (int j = 0; j < MR; ++j) y[j] = mean + p.c[j];
        }
        Y = gm_eval<MR, RT_M>(p, Z, y);
      }
      ref_step(rs, p, Z);
      if (p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q] = Y;
    }
    if (p.out_mode == kTerminal) p.out[q] = Y;
    if (p.has_stats) stat_add(acc, p, Y, ref_final(rs, p), hist);
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

// Throughput form of the specialised exact kernel (the HBM-store-bound FULL mode of cfg3): steps are
// processed in Philox blocks of 4 (no per-step rotation of the buffered normals), the output pointer
// advances by one row per step, the key schedule comes from the constant bank, and the strong-error
// reference is compiled in only when requested (REF_ON).
template <int MR, int COLLOC>
__device__ __forceinline__ float special_step(const RunParams& p, float Y, float Z) {
  if constexpr (COLLOC == kExactGbm) {
    float qz = p.q[MR - 1];
#pragma unroll
    for (int k = MR - 2; k >= 0; --k) qz = fmaf(qz, Z, p.q[k]);
    return Y * qz;
  } else {
    return fmaf(p.ou_s, Z, fmaf(p.ou_a, Y, p.ou_b));
  }
}

template <int MR, int COLLOC, bool FAST, bool REF_ON>
__global__ void __launch_bounds__(256) exact_special_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  hist_init(p, hist);
  __syncthreads();
  StatAcc acc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool full = (p.out_mode == kFull);
  const int nfull = p.n_steps >> 2, rem = p.n_steps & 3;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_paths; q += stride) {
    const uint64_t gp = p.path_offset + q;
    float Y = p.y0;
    float* o = p.out + q;
    if (full) *o = Y;
    RefState rs;
    if (REF_ON) ref_init(rs, p);
    for (int b = 0; b < nfull; ++b) {
      float z[4];
      normals4_rk<FAST>(p, gp, (uint32_t)b, z[0], z[1], z[2], z[3]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        Y = special_step<MR, COLLOC>(p, Y, z[k]);
        if (REF_ON) ref_step(rs, p, z[k]);
        if (full) {
          o += p.n_paths;
          *o = Y;
        }
      }
    }
    if (rem) {
      float z[4];
      normals4_rk<FAST>(p, gp, (uint32_t)nfull, z[0], z[1], z[2], z[3]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (k < rem) {
          Y = special_step<MR, COLLOC>(p, Y, z[k]);
          if (REF_ON) ref_step(rs, p, z[k]);
          if (full) {
            o += p.n_paths;
            *o = Y;
          }
        }
      }
    }
    if (p.out_mode == kTerminal) p.out[q] = Y;
    if (p.has_stats) stat_add(acc, p, Y, REF_ON ? ref_final(rs, p) : 0.0, hist);
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

// FULL-output form for the HBM-store-bound cfg3 (§8(a7)): each thread carries FOUR consecutive paths
// through all steps and writes each step's row segment as one 16-byte store (st.global.cs.v4: the 52 GB
// path tensor is written once and never re-read by the kernel, so it is marked evict-first).  A warp's
// store is 512 contiguous bytes of row i.  The arithmetic of two paths at a time runs in FFMA2
// (fma.rn.f32x2): the fast Box-Muller of box_muller_fast and the closed-form Horner of special_step,
// operation for operation (bit-identical results, fewer issue slots).  Needs n_paths % 4 == 0 and a
// 16-byte aligned output (the launcher falls back to exact_special_kernel otherwise).
namespace {
__device__ __forceinline__ uint64_t f2pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2up(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2c(float c) { return f2pk(c, c); }
// (2 (r >> 9) + 1) 2^-24 exactly: the float 1 + (r >> 9) 2^-23, minus (1 - 2^-24)
__device__ __forceinline__ float unit_bits(uint32_t r) { return __uint_as_float(0x3F800000u | (r >> 9)); }

// box_muller_fast for two (ra, rb) word pairs at once (paths p and q); returns W = -Z (the sign is folded
// into the Horner coefficients of the caller): Wa = rad cos(a), Wb = rad sin(a)
__device__ __forceinline__ void box_muller_fast_x2(uint32_t rap, uint32_t rbp, uint32_t raq, uint32_t rbq,
                                                   uint64_t& Wa, uint64_t& Wb) {
  const uint64_t UA = f2fma(f2pk(unit_bits(rap), unit_bits(raq)), f2c(1.0f), f2c(-0.99999994039535522f));
  const uint64_t UB = f2fma(f2pk(unit_bits(rbp), unit_bits(rbq)), f2c(1.0f), f2c(-0.99999994039535522f));
  const uint64_t V = f2fma(UA, f2c(-1.0f), f2c(1.0f));
  uint64_t P = f2fma(V, f2c(0.2f), f2c(0.25f));
  P = f2fma(P, V, f2c(0.33333333f));
  P = f2fma(P, V, f2c(0.5f));
  P = f2fma(P, V, f2c(1.0f));
  const uint64_t SER = f2fma(f2fma(V, f2c(2.0f), f2c(0.0f)), P, f2c(0.0f));
  float uap, uaq, vp, vq, sp, sq;
  f2up(UA, uap, uaq);
  const uint64_t LG = f2fma(f2pk(lg2_fast(uap), lg2_fast(uaq)), f2c(-1.3862943611198906f), f2c(0.0f));
  float lp, lq;
  f2up(V, vp, vq);
  f2up(SER, sp, sq);
  f2up(LG, lp, lq);
  float rp, rq;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rp) : "f"((vp < 0.0625f) ? sp : lp));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"((vq < 0.0625f) ? sq : lq));
  float ap, aq;
  f2up(f2fma(f2fma(UB, f2c(1.0f), f2c(-0.5f)), f2c(6.2831853071795865f), f2c(0.0f)), ap, aq);
  float snp, snq, csp, csq;
  asm("sin.approx.f32 %0, %1;" : "=f"(snp) : "f"(ap));
  asm("cos.approx.f32 %0, %1;" : "=f"(csp) : "f"(ap));
  asm("sin.approx.f32 %0, %1;" : "=f"(snq) : "f"(aq));
  asm("cos.approx.f32 %0, %1;" : "=f"(csq) : "f"(aq));
  const uint64_t RAD = f2pk(rp, rq);
  Wa = f2fma(RAD, f2pk(csp, csq), f2c(0.0f));
  Wb = f2fma(RAD, f2pk(snp, snq), f2c(0.0f));
}

// The same fast Box-Muller with fewer FMA-pipe operations (the FULL kernel is bound by the FMA pipe: Philox's
// IMAD.WIDE and these FFMA2, profiles/r02_exact_full4x2_ncu.md), returning the normal in units of
// s = sqrt(2 ln 2): W' = -Z / s = sqrt(-log2 u) cos(a).  The factor -2 ln 2 of ln u moves out of the radius (the
// sqrt takes -log2 u through its operand's negation), the series branch carries 1/(2 ln 2) in its coefficients
// (v P(v) / ln 2 with P(v) = 1 + v/2 + v^2/3 + v^3/4 + v^4/5 ~ -ln(1 - v) / v), and the reduced angle
// 2 pi (u_b - 1/2) = 2 pi ((bits_b - 3/2) + 2^-24) is two FFMA2 from the mantissa bits (bits_b - 3/2 exact).
// The caller scales its Horner coefficients by s^j.  Same inputs and accuracy as box_muller_fast.
__device__ __forceinline__ void box_muller_fast_x2s(uint32_t rap, uint32_t rbp, uint32_t raq, uint32_t rbq,
                                                    uint64_t& Wa, uint64_t& Wb) {
  constexpr float kInvLn2 = 1.4426950408889634f;
  const uint64_t UA = f2fma(f2pk(unit_bits(rap), unit_bits(raq)), f2c(1.0f), f2c(-0.99999994039535522f));
  const uint64_t V = f2fma(UA, f2c(-1.0f), f2c(1.0f));
  uint64_t P = f2fma(V, f2c(0.2f * kInvLn2), f2c(0.25f * kInvLn2));
  P = f2fma(P, V, f2c(0.33333333f * kInvLn2));
  P = f2fma(P, V, f2c(0.5f * kInvLn2));
  P = f2fma(P, V, f2c(kInvLn2));
  const uint64_t SER = f2fma(V, P, f2c(0.0f));   // -log2(u) for v < 1/16
  float uap, uaq, vp, vq, sp, sq;
  f2up(UA, uap, uaq);
  f2up(V, vp, vq);
  f2up(SER, sp, sq);
  float rp, rq;
  const float lp = lg2_fast(uap), lq = lg2_fast(uaq);
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rp) : "f"((vp < 0.0625f) ? sp : -lp));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"((vq < 0.0625f) ? sq : -lq));
  const uint64_t D = f2fma(f2pk(unit_bits(rbp), unit_bits(rbq)), f2c(1.0f), f2c(-1.5f));
  float ap, aq;
  f2up(f2fma(D, f2c(6.2831853071795865f), f2c(6.2831853071795865f * 0x1p-24f)), ap, aq);
  float snp, snq, csp, csq;
  asm("sin.approx.f32 %0, %1;" : "=f"(snp) : "f"(ap));
  asm("cos.approx.f32 %0, %1;" : "=f"(csp) : "f"(ap));
  asm("sin.approx.f32 %0, %1;" : "=f"(snq) : "f"(aq));
  asm("cos.approx.f32 %0, %1;" : "=f"(csq) : "f"(aq));
  const uint64_t RAD = f2pk(rp, rq);
  Wa = f2fma(RAD, f2pk(csp, csq), f2c(0.0f));
  Wb = f2fma(RAD, f2pk(snp, snq), f2c(0.0f));
}
}  // namespace

template <int MR, int COLLOC, bool FAST, bool REF_ON, bool CS, int MINB = 1, bool SCALED = true>
__global__ void __launch_bounds__(256, MINB) exact_full4_kernel(const __grid_constant__ RunParams p) {
  static_assert(COLLOC == kExactGbm && FAST, "FFMA2 full-output kernel: GBM closed form, fast normals");
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  hist_init(p, hist);
  __syncthreads();
  StatAcc acc;
  // Horner in W = -Z: q'_j = (-1)^(MR-1-j) q_j gives qz' = (-1)^(MR-1) qz, rounding for rounding
  // SCALED: the normals arrive as W' = W / s (box_muller_fast_x2s), so coefficient j carries s^j
  constexpr float kS = 1.1774100225154747f;   // sqrt(2 ln 2)
  uint64_t QC[MR];
  float sj = 1.0f;
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const float c = ((MR - 1 - j) & 1) ? -p.q[j] : p.q[j];
    QC[j] = f2c(SCALED ? c * sj : c);
    sj *= kS;
  }
  constexpr float kSign = ((MR - 1) & 1) ? -1.0f : 1.0f;
  const uint64_t n4 = p.n_paths >> 2, stride = (uint64_t)gridDim.x * blockDim.x;
  const int nb = (p.n_steps + 3) >> 2;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n4; g += stride) {
    const uint64_t gp = p.path_offset + 4 * g;
    uint64_t Y01 = f2c(p.y0), Y23 = f2c(p.y0);
    float4* o = reinterpret_cast<float4*>(p.out) + g;
    auto put = [&](float4* a) {
      float4 v;
      f2up(Y01, v.x, v.y);
      f2up(Y23, v.z, v.w);
      if constexpr (CS) __stcs(a, v);
      else *a = v;
    };
    put(o);
    RefState rs[4];
    if (REF_ON)
#pragma unroll
      for (int u = 0; u < 4; ++u) ref_init(rs[u], p);
    for (int b = 0; b < nb; ++b) {
      uint4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = philox_path_block_rk(p.rk0, p.rk1, gp + u, (uint32_t)b);
      // W[k][pair]: step k of the block for paths (0,1) and (2,3)
      uint64_t W[4][2];
      if constexpr (SCALED) {
        box_muller_fast_x2s(r[0].x, r[0].y, r[1].x, r[1].y, W[0][0], W[1][0]);
        box_muller_fast_x2s(r[2].x, r[2].y, r[3].x, r[3].y, W[0][1], W[1][1]);
        box_muller_fast_x2s(r[0].z, r[0].w, r[1].z, r[1].w, W[2][0], W[3][0]);
        box_muller_fast_x2s(r[2].z, r[2].w, r[3].z, r[3].w, W[2][1], W[3][1]);
      } else {
        box_muller_fast_x2(r[0].x, r[0].y, r[1].x, r[1].y, W[0][0], W[1][0]);
        box_muller_fast_x2(r[2].x, r[2].y, r[3].x, r[3].y, W[0][1], W[1][1]);
        box_muller_fast_x2(r[0].z, r[0].w, r[1].z, r[1].w, W[2][0], W[3][0]);
        box_muller_fast_x2(r[2].z, r[2].w, r[3].z, r[3].w, W[2][1], W[3][1]);
      }
      const int ns = (p.n_steps - 4 * b < 4) ? p.n_steps - 4 * b : 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < ns) {
          uint64_t q01 = QC[MR - 1], q23 = QC[MR - 1];
#pragma unroll
          for (int j = MR - 2; j >= 0; --j) {
            q01 = f2fma(q01, W[k][0], QC[j]);
            q23 = f2fma(q23, W[k][1], QC[j]);
          }
          Y01 = f2fma(Y01, q01, f2c(0.0f));
          Y23 = f2fma(Y23, q23, f2c(0.0f));
          if constexpr (kSign < 0.0f) {
            Y01 = f2fma(Y01, f2c(-1.0f), f2c(0.0f));
            Y23 = f2fma(Y23, f2c(-1.0f), f2c(0.0f));
          }
          if (REF_ON) {
            const float zs = SCALED ? -kS : -1.0f;
            float w0, w1, w2, w3;
            f2up(W[k][0], w0, w1);
            f2up(W[k][1], w2, w3);
            ref_step(rs[0], p, zs * w0);
            ref_step(rs[1], p, zs * w1);
            ref_step(rs[2], p, zs * w2);
            ref_step(rs[3], p, zs * w3);
          }
          o += n4;
          put(o);
        }
      }
    }
    if (p.has_stats) {
      float y[4];
      f2up(Y01, y[0], y[1]);
      f2up(Y23, y[2], y[3]);
#pragma unroll
      for (int u = 0; u < 4; ++u) stat_add(acc, p, y[u], REF_ON ? ref_final(rs[u], p) : 0.0, hist);
    }
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

// ------------------------------------------------------------------------------------------------
// ANN-FP32 step kernel.  Layer 1 folded (pre_k = l1w_k Y + l1b_k, constant bank); hidden and output
// layers read from shared memory as float4 broadcasts (all lanes of a warp read the same row), one
// FFMA per weight with the activation vector held in registers.
// ------------------------------------------------------------------------------------------------
template <int H, int HS, int MR, bool RT_M, int ACT, int PP>
__global__ void __launch_bounds__(128) ann_f32_step_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  __shared__ double red[8];
  const int L = p.n_hidden;
  const size_t nw = f32_weight_floats(H, HS, L, MR);
  float* gs = sw + ((nw + 3) & ~size_t(3));                  // [H][PP][blockDim] activation scratch
  uint32_t* hist = reinterpret_cast<uint32_t*>(gs + (size_t)H * PP * blockDim.x);
  for (size_t k = threadIdx.x; k < nw; k += blockDim.x) sw[k] = p.wdev[k];
  hist_init(p, hist);
  __syncthreads();
  const float* wout = sw + (size_t)(L - 1) * f32_layer_floats(H, HS);
  const float* bout = wout + MR * HS;

  // PP paths per thread (paths base + tid and base + blockDim + tid): every weight broadcast from shared
  // memory feeds PP FFMAs.  With one path per thread the kernel was bound by shared-memory wavefronts
  // (81% busy: a warp-wide broadcast LDS.128 costs two wavefronts per four weights).
  StatAcc acc;
  const uint64_t tile = (uint64_t)PP * blockDim.x;
  const uint64_t stride = (uint64_t)gridDim.x * tile;
  for (uint64_t base = (uint64_t)blockIdx.x * tile; base < p.n_paths; base += stride) {
    uint64_t q[PP], gp[PP];
    bool ok[PP];
    float Y[PP], z[PP][4];
    RefState rs[PP];
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      q[pp] = base + (uint64_t)pp * blockDim.x + threadIdx.x;
      ok[pp] = q[pp] < p.n_paths;
      gp[pp] = p.path_offset + (ok[pp] ? q[pp] : 0);
      Y[pp] = p.y0;
      if (ok[pp] && p.out_mode == kFull) p.out[q[pp]] = Y[pp];
      ref_init(rs[pp], p);
#pragma unroll
      for (int r = 0; r < 4; ++r) z[pp][r] = 0.f;
    }
    for (int i = 0; i < p.n_steps; ++i) {
      float Z[PP];
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) {
        if ((i & 3) == 0) normals4(p.key0, p.key1, gp[pp], (uint32_t)(i >> 2), z[pp][0], z[pp][1], z[pp][2], z[pp][3]);
        Z[pp] = z[pp][0];
        z[pp][0] = z[pp][1]; z[pp][1] = z[pp][2]; z[pp][2] = z[pp][3];
      }
      // step 3 (Eq. 6.4): y_hat = H_hat(Y_i, dt, theta)
      float h[PP][H];
#pragma unroll
      for (int pp = 0; pp < PP; ++pp)
#pragma unroll
        for (int k = 0; k < H; ++k) h[pp][k] = activate<ACT>(fmaf(p.l1w[k], Y[pp], p.l1b[k]));
      for (int l = 0; l < L - 1; ++l) {
        const float* W = sw + (size_t)l * f32_layer_floats(H, HS);
        const float* b = W + H * HS;
        // output neurons in a rolled loop (a fully unrolled 50 x 50 body overflows the instruction
        // cache: ncu showed "no_instructions" as the top stall); each neuron's activation goes to the
        // thread's own column of a shared-memory scratch and is read back into registers afterwards
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
          const float4* row = reinterpret_cast<const float4*>(W + j * HS);
          float a0[PP], a1[PP];
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) { a0[pp] = b[j]; a1[pp] = 0.f; }
#pragma unroll
          for (int kk = 0; kk < HS / 4; ++kk) {
            const float4 wv = row[kk];
#pragma unroll
            for (int pp = 0; pp < PP; ++pp) {
              if (4 * kk + 0 < H) a0[pp] = fmaf(wv.x, h[pp][4 * kk + 0], a0[pp]);
              if (4 * kk + 1 < H) a1[pp] = fmaf(wv.y, h[pp][4 * kk + 1], a1[pp]);
              if (4 * kk + 2 < H) a0[pp] = fmaf(wv.z, h[pp][4 * kk + 2], a0[pp]);
              if (4 * kk + 3 < H) a1[pp] = fmaf(wv.w, h[pp][4 * kk + 3], a1[pp]);
            }
          }
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) gs[(j * PP + pp) * blockDim.x + threadIdx.x] = activate<ACT>(a0[pp] + a1[pp]);
        }
#pragma unroll
        for (int pp = 0; pp < PP; ++pp)
#pragma unroll
          for (int k = 0; k < H; ++k) h[pp][k] = gs[(k * PP + pp) * blockDim.x + threadIdx.x];
      }
      float y[PP][MR];
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const float4* row = reinterpret_cast<const float4*>(wout + j * HS);
        float a0[PP], a1[PP];
#pragma unroll
        for (int pp = 0; pp < PP; ++pp) { a0[pp] = bout[j]; a1[pp] = 0.f; }
#pragma unroll
        for (int kk = 0; kk < HS / 4; ++kk) {
          const float4 wv = row[kk];
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) {
            if (4 * kk + 0 < H) a0[pp] = fmaf(wv.x, h[pp][4 * kk + 0], a0[pp]);
            if (4 * kk + 1 < H) a1[pp] = fmaf(wv.y, h[pp][4 * kk + 1], a1[pp]);
            if (4 * kk + 2 < H) a0[pp] = fmaf(wv.z, h[pp][4 * kk + 2], a0[pp]);
            if (4 * kk + 3 < H) a1[pp] = fmaf(wv.w, h[pp][4 * kk + 3], a1[pp]);
          }
        }
#pragma unroll
        for (int pp = 0; pp < PP; ++pp)
          y[pp][j] = fmaf(p.res_y, Y[pp], fmaf(a0[pp] + a1[pp], p.out_scale[j], p.out_shift[j]));
      }
      // steps 5-6: Y_{i+1} = g_m(X_hat)
#pragma unroll
      for (int pp = 0; pp < PP; ++pp) {
        Y[pp] = gm_eval<MR, RT_M>(p, Z[pp], y[pp]);
        ref_step(rs[pp], p, Z[pp]);
        if (ok[pp] && p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q[pp]] = Y[pp];
      }
    }
#pragma unroll
    for (int pp = 0; pp < PP; ++pp) {
      if (!ok[pp]) continue;
      if (p.out_mode == kTerminal) p.out[q[pp]] = Y[pp];
      if (p.has_stats) stat_add(acc, p, Y[pp], ref_final(rs[pp], p), hist);
    }
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

// Packed form of the ANN-FP32 kernel: two paths per thread held as fp32 pairs, every weight (a scalar from
// the shared-memory float4 broadcast) feeds ONE FFMA2 (fma.rn.f32x2 with the weight broadcast to both
// halves) for the two paths -- the FFMA work is unchanged, the instruction count of the contractions
// halves (the r01 kernel was issue-bound at ~8000 instructions per path-step, 5350 of them FFMA).
// Activations of the two paths in pairs on MUFU (ex2 + rcp / ex2 + lg2: the FMA pipe is the bound here).
template <int ACT>
__device__ __forceinline__ uint64_t act_f32_pair(uint64_t U) {
  float u0, u1, h0, h1;
  up2(U, u0, u1);
  if constexpr (ACT == SL7_ACT_TANH) {
    // tanh z = (1 - e) / (1 + e) with e = 2^-2|z|log2(e): the pair form of act_tanh (argument scaled here)
    tanh_pair<false>(u0 * 2.8853900817779268f, u1 * 2.8853900817779268f, h0, h1);
  } else {
    softplus_pair<false>(u0, u1, h0, h1);
  }
  return pk2(h0, h1);
}

// NJ output neurons of one hidden layer at a time for the pair of paths, two accumulator chains each (2 NJ
// independent FFMA2 chains per thread: the r02 kernel with NJ = 2 stalled on FFMA2 latency at 2 warps per
// scheduler); the NJ weight rows are read as float4 broadcasts, each weight feeds one FFMA2.
template <int H, int HS, int NJ>
__device__ __forceinline__ void f32x2_neurons(const float* W, const float* b, const uint64_t (&h)[H], int j,
                                              uint64_t (&out)[NJ]) {
  uint64_t a0[NJ], a1[NJ];
#pragma unroll
  for (int u = 0; u < NJ; ++u) {
    a0[u] = pk2(b[j + u], b[j + u]);
    a1[u] = pk2(0.f, 0.f);
  }
#pragma unroll
  for (int kk = 0; kk < HS / 4; ++kk) {
    float4 wv[NJ];
#pragma unroll
    for (int u = 0; u < NJ; ++u) wv[u] = reinterpret_cast<const float4*>(W + (j + u) * HS)[kk];
#pragma unroll
    for (int u = 0; u < NJ; ++u) {
      if (4 * kk + 0 < H) a0[u] = fma2(h[4 * kk + 0], pk2(wv[u].x, wv[u].x), a0[u]);
      if (4 * kk + 1 < H) a1[u] = fma2(h[4 * kk + 1], pk2(wv[u].y, wv[u].y), a1[u]);
      if (4 * kk + 2 < H) a0[u] = fma2(h[4 * kk + 2], pk2(wv[u].z, wv[u].z), a0[u]);
      if (4 * kk + 3 < H) a1[u] = fma2(h[4 * kk + 3], pk2(wv[u].w, wv[u].w), a1[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < NJ; ++u) out[u] = fma2(a0[u], pk2(1.f, 1.f), a1[u]);
}

template <int H, int HS, int MR, int ACT, int MINB = 1, int NJ = 0>
__global__ void __launch_bounds__(128, MINB) ann_f32x2_step_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  __shared__ double red[8];
  const int L = p.n_hidden;
  const size_t nw = f32_weight_floats(H, HS, L, MR);
  uint64_t* gs = reinterpret_cast<uint64_t*>(sw + ((nw + 3) & ~size_t(3)));   // [H][blockDim] pair scratch
  uint32_t* hist = reinterpret_cast<uint32_t*>(gs + (size_t)H * blockDim.x);
  for (size_t k = threadIdx.x; k < nw; k += blockDim.x) sw[k] = p.wdev[k];
  hist_init(p, hist);
  __syncthreads();
  const float* wout = sw + (size_t)(L - 1) * f32_layer_floats(H, HS);
  const float* bout = wout + MR * HS;
  StatAcc acc;
  const uint64_t tile = 2ull * blockDim.x;
  const uint64_t stride = (uint64_t)gridDim.x * tile;
  for (uint64_t base = (uint64_t)blockIdx.x * tile; base < p.n_paths; base += stride) {
    uint64_t q[2], gp[2];
    bool ok[2];
    float z[2][4];
    RefState rs[2];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      q[pp] = base + (uint64_t)pp * blockDim.x + threadIdx.x;
      ok[pp] = q[pp] < p.n_paths;
      gp[pp] = p.path_offset + (ok[pp] ? q[pp] : 0);
      if (ok[pp] && p.out_mode == kFull) p.out[q[pp]] = p.y0;
      ref_init(rs[pp], p);
#pragma unroll
      for (int r = 0; r < 4; ++r) z[pp][r] = 0.f;
    }
    uint64_t Y = pk2(p.y0, p.y0);
    for (int i = 0; i < p.n_steps; ++i) {
      float Z[2];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        if ((i & 3) == 0) normals4(p.key0, p.key1, gp[pp], (uint32_t)(i >> 2), z[pp][0], z[pp][1], z[pp][2], z[pp][3]);
        Z[pp] = z[pp][0];
        z[pp][0] = z[pp][1]; z[pp][1] = z[pp][2]; z[pp][2] = z[pp][3];
      }
      uint64_t h[H];
#pragma unroll
      for (int k = 0; k < H; ++k) h[k] = act_f32_pair<ACT>(fma2(Y, pk2(p.l1w[k], p.l1w[k]), pk2(p.l1b[k], p.l1b[k])));
      for (int l = 0; l < L - 1; ++l) {
        const float* W = sw + (size_t)l * f32_layer_floats(H, HS);
        const float* b = W + H * HS;
        if constexpr (NJ > 0) {
          int j = 0;
#pragma unroll 1
          for (; j + NJ <= H; j += NJ) {
            uint64_t a[NJ];
            f32x2_neurons<H, HS, NJ>(W, b, h, j, a);
#pragma unroll
            for (int u = 0; u < NJ; ++u) gs[(size_t)(j + u) * blockDim.x + threadIdx.x] = act_f32_pair<ACT>(a[u]);
          }
#pragma unroll 1
          for (; j < H; ++j) {
            uint64_t a[1];
            f32x2_neurons<H, HS, 1>(W, b, h, j, a);
            gs[(size_t)j * blockDim.x + threadIdx.x] = act_f32_pair<ACT>(a[0]);
          }
        } else {
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
          const float4* row = reinterpret_cast<const float4*>(W + j * HS);
          uint64_t a0 = pk2(b[j], b[j]), a1 = pk2(0.f, 0.f);
#pragma unroll
          for (int kk = 0; kk < HS / 4; ++kk) {
            const float4 wv = row[kk];
            if (4 * kk + 0 < H) a0 = fma2(h[4 * kk + 0], pk2(wv.x, wv.x), a0);
            if (4 * kk + 1 < H) a1 = fma2(h[4 * kk + 1], pk2(wv.y, wv.y), a1);
            if (4 * kk + 2 < H) a0 = fma2(h[4 * kk + 2], pk2(wv.z, wv.z), a0);
            if (4 * kk + 3 < H) a1 = fma2(h[4 * kk + 3], pk2(wv.w, wv.w), a1);
          }
          gs[(size_t)j * blockDim.x + threadIdx.x] = act_f32_pair<ACT>(fma2(a0, pk2(1.f, 1.f), a1));
        }
        }
#pragma unroll
        for (int k = 0; k < H; ++k) h[k] = gs[(size_t)k * blockDim.x + threadIdx.x];
      }
      float y[2][MR];
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const float4* row = reinterpret_cast<const float4*>(wout + j * HS);
        uint64_t a0 = pk2(bout[j], bout[j]), a1 = pk2(0.f, 0.f);
#pragma unroll
        for (int kk = 0; kk < HS / 4; ++kk) {
          const float4 wv = row[kk];
          if (4 * kk + 0 < H) a0 = fma2(h[4 * kk + 0], pk2(wv.x, wv.x), a0);
          if (4 * kk + 1 < H) a1 = fma2(h[4 * kk + 1], pk2(wv.y, wv.y), a1);
          if (4 * kk + 2 < H) a0 = fma2(h[4 * kk + 2], pk2(wv.z, wv.z), a0);
          if (4 * kk + 3 < H) a1 = fma2(h[4 * kk + 3], pk2(wv.w, wv.w), a1);
        }
        float s0, s1, y0, y1;
        up2(fma2(a0, pk2(1.f, 1.f), a1), s0, s1);
        up2(Y, y0, y1);
        y[0][j] = fmaf(p.res_y, y0, fmaf(s0, p.out_scale[j], p.out_shift[j]));
        y[1][j] = fmaf(p.res_y, y1, fmaf(s1, p.out_scale[j], p.out_shift[j]));
      }
      float yn[2];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        yn[pp] = gm_eval<MR, false>(p, Z[pp], y[pp]);
        ref_step(rs[pp], p, Z[pp]);
        if (ok[pp] && p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q[pp]] = yn[pp];
      }
      Y = pk2(yn[0], yn[1]);
    }
    float yT[2];
    up2(Y, yT[0], yT[1]);
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      if (!ok[pp]) continue;
      if (p.out_mode == kTerminal) p.out[q[pp]] = yT[pp];
      if (p.has_stats) stat_add(acc, p, yT[pp], ref_final(rs[pp], p), hist);
    }
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

// ------------------------------------------------------------------------------------------------
// RNG verification kernels (same device functions as the step kernels).
// ------------------------------------------------------------------------------------------------
__global__ void philox_u32_kernel(uint32_t k0, uint32_t k1, uint64_t off, uint64_t n, uint32_t block, uint32_t* out) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox_path_block(k0, k1, off + q, block);
    out[q] = r.x;
    out[n + q] = r.y;
    out[2 * n + q] = r.z;
    out[3 * n + q] = r.w;
  }
}

template <bool FAST>
__global__ void normals_kernel(uint32_t k0, uint32_t k1, uint64_t off, uint64_t n, int n_steps, float* out) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    for (int i = 0; i < n_steps; ++i) {
      if ((i & 3) == 0) normals4<FAST>(k0, k1, off + q, (uint32_t)(i >> 2), z0, z1, z2, z3);
      out[(uint64_t)i * n + q] = z0;
      z0 = z1; z1 = z2; z2 = z3;
    }
  }
}

__global__ void zero_kernel(double* p, size_t n) {
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) p[k] = 0.0;
}

// ------------------------------------------------------------------------------------------------
// Launchers
// ------------------------------------------------------------------------------------------------
namespace {

template <typename K>
cudaError_t launch_persistent(K kernel, int threads, size_t smem, const RunParams& p, cudaStream_t st, int num_sms,
                              int paths_per_cta = 0) {
  cudaError_t e;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t per_cta = (uint64_t)(paths_per_cta > 0 ? paths_per_cta : threads);
  const uint64_t need = (p.n_paths + per_cta - 1) / per_cta;
  const uint64_t full = (uint64_t)per_sm * (uint64_t)num_sms;
  const unsigned grid = (unsigned)(need < full ? need : full);
  kernel<<<grid, threads, smem, st>>>(p);
  return cudaGetLastError();
}

size_t hist_bytes(const RunParams& p) {
  return (p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0;
}

template <int COLLOC, bool FAST, bool REF_ON>
cudaError_t launch_exact_special_r(const RunParams& p, cudaStream_t st, int num_sms, size_t smem) {
  // OU: the closed form does not depend on m; GBM: Horner of degree m-1 (m <= 8, zero padded)
  if (COLLOC == kExactOu || (p.m != 5 && p.m != 7))
    return launch_persistent(exact_special_kernel<8, COLLOC, FAST, REF_ON>, 256, smem, p, st, num_sms);
  if (p.m == 5) return launch_persistent(exact_special_kernel<5, COLLOC, FAST, REF_ON>, 256, smem, p, st, num_sms);
  return launch_persistent(exact_special_kernel<7, COLLOC, FAST, REF_ON>, 256, smem, p, st, num_sms);
}

template <int COLLOC, bool FAST, bool REF_ON, bool CS, int MINB = 1, bool SC = true>
cudaError_t launch_exact_full4_r(const RunParams& p, cudaStream_t st, int num_sms, size_t smem) {
  if (p.m != 5 && p.m != 7)
    return launch_persistent(exact_full4_kernel<8, COLLOC, FAST, REF_ON, CS, MINB, SC>, 256, smem, p, st, num_sms, 1024);
  if (p.m == 5)
    return launch_persistent(exact_full4_kernel<5, COLLOC, FAST, REF_ON, CS, MINB, SC>, 256, smem, p, st, num_sms, 1024);
  return launch_persistent(exact_full4_kernel<7, COLLOC, FAST, REF_ON, CS, MINB, SC>, 256, smem, p, st, num_sms, 1024);
}

template <int COLLOC, bool FAST>
cudaError_t launch_exact_special(const RunParams& p, cudaStream_t st, int num_sms, size_t smem) {
  const bool v4 = COLLOC == kExactGbm && FAST && p.out_mode == kFull && (p.n_paths & 3) == 0 &&
                  (reinterpret_cast<uintptr_t>(p.out) & 15) == 0;
  int variant = 0;
#ifdef SL7_AB_HOOKS
  if (const char* v = std::getenv("SL7_TC_VARIANT")) variant = std::atoi(v);   // 50: one path per thread
#endif
  if constexpr (COLLOC == kExactGbm && FAST) {
    if (v4 && variant != 50) {
      const bool ref = p.ref != kRefNone && p.has_stats;
      if (variant == 51) return ref ? launch_exact_full4_r<COLLOC, FAST, true, false>(p, st, num_sms, smem)
                                    : launch_exact_full4_r<COLLOC, FAST, false, false>(p, st, num_sms, smem);
      if (variant == 52) return ref ? launch_exact_full4_r<COLLOC, FAST, true, true, 4>(p, st, num_sms, smem)
                                    : launch_exact_full4_r<COLLOC, FAST, false, true, 4>(p, st, num_sms, smem);
      if (variant == 53) return ref ? launch_exact_full4_r<COLLOC, FAST, true, true, 3>(p, st, num_sms, smem)
                                    : launch_exact_full4_r<COLLOC, FAST, false, true, 3>(p, st, num_sms, smem);
      if (variant == 54) return ref ? launch_exact_full4_r<COLLOC, FAST, true, true, 4, false>(p, st, num_sms, smem)
                                    : launch_exact_full4_r<COLLOC, FAST, false, true, 4, false>(p, st, num_sms, smem);
      // 4 CTAs of 256 per SM (<= 64 registers): 9.0e11 vs 8.8e11 path-steps/s at 3 (cfg3, B200)
      return ref ? launch_exact_full4_r<COLLOC, FAST, true, true, 4>(p, st, num_sms, smem)
                 : launch_exact_full4_r<COLLOC, FAST, false, true, 4>(p, st, num_sms, smem);
    }
  }
  return (p.ref != kRefNone && p.has_stats) ? launch_exact_special_r<COLLOC, FAST, true>(p, st, num_sms, smem)
                                            : launch_exact_special_r<COLLOC, FAST, false>(p, st, num_sms, smem);
}

template <int COLLOC, bool FAST>
cudaError_t launch_exact_general(const RunParams& p, cudaStream_t st, int num_sms, size_t smem) {
  switch (p.m) {
    case 5: return launch_persistent(exact_step_kernel<5, false, COLLOC, FAST>, 256, smem, p, st, num_sms);
    case 7: return launch_persistent(exact_step_kernel<7, false, COLLOC, FAST>, 256, smem, p, st, num_sms);
    default: return launch_persistent(exact_step_kernel<kMaxM, true, COLLOC, FAST>, 256, smem, p, st, num_sms);
  }
}

template <int COLLOC>
cudaError_t launch_exact(const RunParams& p, cudaStream_t st, int num_sms) {
  const size_t smem = hist_bytes(p);
  const bool fast = p.flags & SL7_FLAG_FAST_NORMALS, special = p.flags & SL7_FLAG_SPECIALIZED;
  if (special) return fast ? launch_exact_special<COLLOC, true>(p, st, num_sms, smem)
                           : launch_exact_special<COLLOC, false>(p, st, num_sms, smem);
  return fast ? launch_exact_general<COLLOC, true>(p, st, num_sms, smem)
              : launch_exact_general<COLLOC, false>(p, st, num_sms, smem);
}

template <int H, int HS, int MR, bool RT, int ACT, int PP>
cudaError_t launch_ann_f32_t(const RunParams& p, cudaStream_t st, int num_sms) {
  const size_t nw = f32_weight_floats(H, HS, p.n_hidden, MR);
  const size_t smem = (((nw + 3) & ~size_t(3)) + (size_t)H * PP * 128) * sizeof(float) + hist_bytes(p);
  return launch_persistent(ann_f32_step_kernel<H, HS, MR, RT, ACT, PP>, 128, smem, p, st, num_sms, 128 * PP);
}

template <int H, int HS, int MR, int ACT, int MINB = 1, int NJ = 0>
cudaError_t launch_ann_f32x2_t(const RunParams& p, cudaStream_t st, int num_sms) {
  const size_t nw = f32_weight_floats(H, HS, p.n_hidden, MR);
  const size_t smem = (((nw + 3) & ~size_t(3)) + (size_t)H * 2 * 128) * sizeof(float) + hist_bytes(p);
  return launch_persistent(ann_f32x2_step_kernel<H, HS, MR, ACT, MINB, NJ>, 128, smem, p, st, num_sms, 256);
}

template <int ACT>
cudaError_t launch_ann_f32(const RunParams& p, cudaStream_t st, int num_sms) {
  int variant = 0;
#ifdef SL7_AB_HOOKS
  if (const char* v = std::getenv("SL7_TC_VARIANT")) variant = std::atoi(v);   // 60: the r01 FFMA kernel
#endif
  if (variant == 61) {
    if (p.width == 50 && p.m == 5) return launch_ann_f32x2_t<50, 52, 5, ACT, 3>(p, st, num_sms);
    if (p.width == 50 && p.m == 7) return launch_ann_f32x2_t<50, 52, 7, ACT, 3>(p, st, num_sms);
  }
  if (variant >= 63 && variant <= 66) {   // NJ neurons per iteration (2 chains each), MINB
    if (p.width == 50 && p.m == 7) {
      if (variant == 63) return launch_ann_f32x2_t<50, 52, 7, ACT, 1, 4>(p, st, num_sms);
      if (variant == 64) return launch_ann_f32x2_t<50, 52, 7, ACT, 2, 4>(p, st, num_sms);
      if (variant == 65) return launch_ann_f32x2_t<50, 52, 7, ACT, 1, 3>(p, st, num_sms);
      return launch_ann_f32x2_t<50, 52, 7, ACT, 1, 2>(p, st, num_sms);
    }
  }
  if (variant == 62) {
    if (p.width == 50 && p.m == 5) return launch_ann_f32x2_t<50, 52, 5, ACT, 4>(p, st, num_sms);
    if (p.width == 50 && p.m == 7) return launch_ann_f32x2_t<50, 52, 7, ACT, 4>(p, st, num_sms);
  }
  if (variant == 67) {   // the r02 first version: neurons in a rolled loop unrolled by 2 (the compiler's chains)
    if (p.width == 50 && p.m == 5) return launch_ann_f32x2_t<50, 52, 5, ACT>(p, st, num_sms);
    if (p.width == 50 && p.m == 7) return launch_ann_f32x2_t<50, 52, 7, ACT>(p, st, num_sms);
  }
  if (variant != 60) {
    // two neurons per iteration with two FFMA2 chains each, written out (cfg1: 3.49e9 -> 3.79e9 path-steps/s;
    // four neurons per iteration 3.78e9)
    if (p.width == 50 && p.m == 5) return launch_ann_f32x2_t<50, 52, 5, ACT, 1, 2>(p, st, num_sms);
    if (p.width == 50 && p.m == 7) return launch_ann_f32x2_t<50, 52, 7, ACT, 1, 2>(p, st, num_sms);
  }
  if (p.width == 50 && p.m == 5) return launch_ann_f32_t<50, 52, 5, false, ACT, 2>(p, st, num_sms);
  if (p.width == 50 && p.m == 7) return launch_ann_f32_t<50, 52, 7, false, ACT, 2>(p, st, num_sms);
  if (p.width == 64) return launch_ann_f32_t<64, 64, kMaxM, true, ACT, 1>(p, st, num_sms);
  return cudaErrorInvalidValue;
}

}  // namespace

int launch_step_kernel(const RunParams& p, int prec, void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  (void)prec;
  switch (p.colloc) {
    case kExactGbm: return (int)launch_exact<kExactGbm>(p, st, num_sms);
    case kExactOu: return (int)launch_exact<kExactOu>(p, st, num_sms);
    case kExactCir: return launch_exact_cir(p, stream, num_sms);
    default:
      return (int)(p.act == SL7_ACT_TANH ? launch_ann_f32<SL7_ACT_TANH>(p, st, num_sms)
                                         : launch_ann_f32<SL7_ACT_SOFTPLUS>(p, st, num_sms));
  }
}

int launch_philox_u32(uint64_t seed, uint64_t off, uint64_t n, uint32_t block, uint32_t* out, void* stream) {
  const unsigned grid = (unsigned)((n + 255) / 256 < 65535 ? (n + 255) / 256 : 65535);
  philox_u32_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (uint32_t)seed, (uint32_t)(seed >> 32), off, n, block, out);
  return (int)cudaGetLastError();
}

int launch_normals(uint64_t seed, uint64_t off, uint64_t n, int n_steps, bool fast, float* out, void* stream) {
  const unsigned grid = (unsigned)((n + 255) / 256 < 65535 ? (n + 255) / 256 : 65535);
  auto kernel = fast ? normals_kernel<true> : normals_kernel<false>;
  kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (uint32_t)seed, (uint32_t)(seed >> 32), off, n, n_steps, out);
  return (int)cudaGetLastError();
}

int launch_zero_stats(double* stats, size_t n, void* stream) {
  const unsigned grid = (unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  zero_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(stats, n);
  return (int)cudaGetLastError();
}

}  // namespace sl7
