// sl7_device.cuh -- device building blocks of the Seven-League step kernels (sm_100a).
//
//   a1  normals:       Philox4x32-10 + Box-Muller keyed by (seed, global path, step block)
//   a5/a6 g_m:         product form of the normalised barycentric Lagrange formula
//   a7  statistics:    shifted power sums, strong error, histogram; per-thread -> warp -> CTA -> global
//   activations:       MUFU-based tanh / softplus with absolute error ~2e-7
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sl7_internal.h"

namespace sl7 {

// ------------------------------------------------------------------------------------------------
// a1.  Philox4x32-10 (Salmon et al. SC'11): 10 rounds of two 32x32->64 multiplies (IMAD.HI + IMAD),
// key schedule (W0, W1).  counter = (block, 0, path_lo, path_hi), key = (seed_lo, seed_hi):
// identical to cuRAND curand4() after curand_init(seed, path, 4*block) (checked on the box).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += W0; k.y += W1; }
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ uint4 philox_path_block(uint32_t key0, uint32_t key1, uint64_t path, uint32_t block) {
  return philox4x32_10(make_uint4(block, 0u, (uint32_t)path, (uint32_t)(path >> 32)), make_uint2(key0, key1));
}

// The same generator with the key schedule precomputed on the host (round keys rk = key + r (W0, W1)
// live in the kernel-parameter constant bank and feed the LOP3s directly: no per-call key adds).
__device__ __forceinline__ uint4 philox_path_block_rk(const uint32_t* rk0, const uint32_t* rk1, uint64_t path,
                                                      uint32_t block) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint4 c = make_uint4(block, 0u, (uint32_t)path, (uint32_t)(path >> 32));
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ rk0[r], lo1, hi0 ^ c.w ^ rk1[r], lo0);
  }
  return c;
}

// u = (2 (r >> 9) + 1) 2^-24: exact in fp32, in [2^-24, 1 - 2^-24], never 0 or 1.
__device__ __forceinline__ float u32_to_unit(uint32_t r) {
  return __uint2float_rn(((r >> 9) << 1) | 1u) * 0x1p-24f;
}

// Box-Muller with accurate libm logf/sincospif (1-2 ulp everywhere, including u -> 1 where
// MUFU lg2.approx would lose the relative accuracy of ln u).
__device__ __forceinline__ void box_muller(uint32_t ra, uint32_t rb, float& za, float& zb) {
  const float ua = u32_to_unit(ra), ub = u32_to_unit(rb);
  const float rad = sqrtf(-2.0f * logf(ua));
  float s, c;
  sincospif(2.0f * ub, &s, &c);
  za = rad * c;
  zb = rad * s;
}

__device__ __forceinline__ float lg2_fast(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Fast Box-Muller on the MUFU pipe (exact-collocation, EM and CDC kernels under SL7_FLAG_FAST_NORMALS,
// where the RNG dominates the cost).  -2 ln u: MUFU lg2 has ~2^-22 ABSOLUTE error (measured on B200:
// relative error 0.86 at u = 1 - 2^-24), so for v = 1 - u < 2^-4 (v exact) the log is the series
// 2 (v + v^2/2 + v^3/3 + v^4/4 + v^5/5) (truncation <= 1.6e-7 relative); elsewhere lg2 is relatively
// accurate to <= 3e-7.  The angle: 2 pi u = 2 pi (u - 1/2) + pi with u - 1/2 exact, so MUFU sin/cos see
// (-pi, pi) (4e-7 absolute there) and the + pi flips both signs.  |Z_fast - Z| <= 2e-6 (1 + |Z|).
__device__ __forceinline__ void box_muller_fast(uint32_t ra, uint32_t rb, float& za, float& zb) {
  const float ua = u32_to_unit(ra), ub = u32_to_unit(rb);
  const float v = 1.0f - ua;
  const float ser = 2.0f * v * fmaf(v, fmaf(v, fmaf(v, fmaf(v, 0.2f, 0.25f), 0.33333333f), 0.5f), 1.0f);
  const float lg = -1.3862943611198906f * lg2_fast(ua);       // -2 ln2 log2(u)
  const float t = (v < 0.0625f) ? ser : lg;
  float rad;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rad) : "f"(t));
  // angle 2 pi u = 2 pi (u - 1/2) + pi: the reduced argument lies in (-pi, pi), where MUFU sin/cos are
  // accurate to 4e-7 absolute (measured, profiles/r01_pipes.md); the + pi flips both signs
  const float a = (ub - 0.5f) * 6.2831853071795865f;
  float s, c;
  asm("sin.approx.f32 %0, %1;" : "=f"(s) : "f"(a));
  asm("cos.approx.f32 %0, %1;" : "=f"(c) : "f"(a));
  za = -rad * c;
  zb = -rad * s;
}

template <bool FAST = false>
__device__ __forceinline__ void normals4_rk(const RunParams& p, uint64_t path, uint32_t block, float& z0, float& z1,
                                            float& z2, float& z3) {
  const uint4 r = philox_path_block_rk(p.rk0, p.rk1, path, block);
  if constexpr (FAST) {
    box_muller_fast(r.x, r.y, z0, z1);
    box_muller_fast(r.z, r.w, z2, z3);
  } else {
    box_muller(r.x, r.y, z0, z1);
    box_muller(r.z, r.w, z2, z3);
  }
}

template <bool FAST = false>
__device__ __forceinline__ void normals4(uint32_t key0, uint32_t key1, uint64_t path, uint32_t block,
                                         float& z0, float& z1, float& z2, float& z3) {
  const uint4 r = philox_path_block(key0, key1, path, block);
  if constexpr (FAST) {
    box_muller_fast(r.x, r.y, z0, z1);
    box_muller_fast(r.z, r.w, z2, z3);
  } else {
    box_muller(r.x, r.y, z0, z1);
    box_muller(r.z, r.w, z2, z3);
  }
}

// ------------------------------------------------------------------------------------------------
// a5/a6.  g_m(Z) = sum_j y_j l_j(Z) / sum_j l_j(Z), l_j(Z) = w_j prod_{k != j}(Z - x_k)
// (barycentric, PAPER.md:48 / ref [8]).  sum_j l_j == 1 exactly, so the division only removes the
// rounding of the fp32 weights (no poles, no node-hit branch).  d_k = (Z - xhi_k) - xlo_k keeps the
// node to ~2^-48 relative.  Prefix/suffix products: 3(M-1) FMUL + 2M FFMA/FADD + 1 rcp.
// MR = compile-time slot count; m_rt < MR means runtime m with padded slots (w = 0, d = 1).
// ------------------------------------------------------------------------------------------------
// Split form for kernels that overlap the basis with other latency: gm_basis fills
// l_j = w_j prod_{k != j}(Z - x_k) and returns sum_j l_j; gm_combine returns sum_j y_j l_j / sum_j l_j.
template <int MR, bool RUNTIME_M = false>
__device__ __forceinline__ float gm_basis(const RunParams& p, float Z, float (&lb)[MR]) {
  float d[MR];
#pragma unroll
  for (int k = 0; k < MR; ++k) {
    const float dk = (Z - p.xhi[k]) - p.xlo[k];
    d[k] = (RUNTIME_M && k >= p.m) ? 1.0f : dk;
  }
  float pre[MR];
  pre[0] = 1.0f;
#pragma unroll
  for (int k = 1; k < MR; ++k) pre[k] = pre[k - 1] * d[k - 1];
  float suf = 1.0f, den = 0.0f;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    lb[j] = p.w[j] * (pre[j] * suf);
    den += lb[j];
    suf *= d[j];
  }
  return den;
}

template <int MR>
__device__ __forceinline__ float gm_combine(const float (&lb)[MR], float den, const float (&y)[MR]) {
  float num = 0.0f;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) num = fmaf(lb[j], y[j], num);
  return __fdividef(num, den);
}

template <int MR, bool RUNTIME_M = false>
__device__ __forceinline__ float gm_eval(const RunParams& p, float Z, const float (&y)[MR]) {
  float d[MR];
#pragma unroll
  for (int k = 0; k < MR; ++k) {
    const float dk = (Z - p.xhi[k]) - p.xlo[k];
    d[k] = (RUNTIME_M && k >= p.m) ? 1.0f : dk;
  }
  float pre[MR];
  pre[0] = 1.0f;
#pragma unroll
  for (int k = 1; k < MR; ++k) pre[k] = pre[k - 1] * d[k - 1];
  float suf = 1.0f, num = 0.0f, den = 0.0f;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const float l = p.w[j] * (pre[j] * suf);
    num = fmaf(l, y[j], num);
    den += l;
    suf *= d[j];
  }
  return __fdividef(num, den);
}

// ------------------------------------------------------------------------------------------------
// Activations (PAPER.md:85 Softplus; tanh for BASELINE configs 0,1,3).  Two MUFU ops each.
// tanh(z) = sign(z) (1 - 2 / (e^{2|z|} + 1)),  |z| clamped at 15 (tanh(15) rounds to 1 in fp32).
// softplus(z) = max(z, 0) + ln 2 * log2(1 + e^{-|z|}).   Absolute error <= ~2.5e-7 for both.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float act_tanh(float z) {
  const float a = fminf(fabsf(z), 15.0f);
  const float e = ex2_approx(a * 2.8853900817779268f);  // e^{2a}
  const float t = fmaf(-2.0f, rcp_approx(e + 1.0f), 1.0f);
  return copysignf(t, z);
}

__device__ __forceinline__ float act_softplus(float z) {
  const float t = ex2_approx(fabsf(z) * -1.4426950408889634f);  // e^{-|z|}
  return fmaf(0.69314718055994531f, lg2_approx(1.0f + t), fmaxf(z, 0.0f));
}

template <int ACT>
__device__ __forceinline__ float activate(float z) {
  if constexpr (ACT == SL7_ACT_TANH) return act_tanh(z);
  else return act_softplus(z);
}

// ------------------------------------------------------------------------------------------------
// Packed fp32 pairs (sm_100a FFMA2, fma.rn.f32x2): two units / two paths per instruction.  FFMA2 has the
// FFMA FLOP rate at half the instructions and co-issues with MUFU better than FFMA (profiles/r02_pipes.md).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fma2s(uint64_t a, float b, float c) { return fma2(a, pk2(b, b), pk2(c, c)); }

// softplus of a pair.  POLY: log1p(e), e = 2^(-|u| log2 e) in (0, 1], as e q(e) with q the degree-7
// minimax polynomial of log1p(e)/e on [0, 1] (absolute error 2.5e-8 in exact arithmetic, 1.6e-7 after fp32
// Horner rounding, mean -1.4e-8 over e^-|u|, u ~ N(0, 2)); the last Horner step adds max(u, 0):
//   h = e q(e) + max(u, 0)   (8 FFMA2 per pair).
// Otherwise: h = ln 2 lg2(1 + e) + max(u, 0) with MUFU lg2 (FADD2 / FFMA2 for the pair).
template <bool POLY, bool DEG7 = false>
__device__ __forceinline__ void softplus_pair(float u0, float u1, float& h0, float& h1) {
  const float e0 = ex2_approx(fabsf(u0) * -1.4426950408889634f);
  const float e1 = ex2_approx(fabsf(u1) * -1.4426950408889634f);
  const uint64_t mx = pk2(fmaxf(u0, 0.0f), fmaxf(u1, 0.0f));
  const uint64_t E = pk2(e0, e1);
  uint64_t r;
  if constexpr (POLY && DEG7) {
    // degree-6 q (total degree 7): minimax error 1.8e-7, 3.4e-7 after fp32 rounding, mean -3.3e-8
    uint64_t q = fma2s(E, 1.081165298819542e-02f, -5.5391568690538406e-02f);
    q = fma2(q, E, pk2(1.351390779018402e-01f, 1.351390779018402e-01f));
    q = fma2(q, E, pk2(-2.263084203004837e-01f, -2.263084203004837e-01f));
    q = fma2(q, E, pk2(3.284189999103546e-01f, 3.284189999103546e-01f));
    q = fma2(q, E, pk2(-4.995054006576538e-01f, -4.995054006576538e-01f));
    q = fma2(q, E, pk2(9.99983012676239e-01f, 9.99983012676239e-01f));
    r = fma2(q, E, mx);
  } else if constexpr (POLY) {
    uint64_t q = fma2s(E, -6.678603123873472e-03f, 3.697235882282257e-02f);
    q = fma2(q, E, pk2(-9.672726690769196e-02f, -9.672726690769196e-02f));
    q = fma2(q, E, pk2(1.6879309713840485e-01f, 1.6879309713840485e-01f));
    q = fma2(q, E, pk2(-2.412412464618683e-01f, -2.412412464618683e-01f));
    q = fma2(q, E, pk2(3.3191972970962524e-01f, 3.3191972970962524e-01f));
    q = fma2(q, E, pk2(-4.998879134654999e-01f, -4.998879134654999e-01f));
    q = fma2(q, E, pk2(9.999969601631165e-01f, 9.999969601631165e-01f));
    r = fma2(q, E, mx);
  } else {
    float a0, a1;
    up2(fma2(E, pk2(1.0f, 1.0f), pk2(1.0f, 1.0f)), a0, a1);   // 1 + e
    r = fma2(pk2(lg2_approx(a0), lg2_approx(a1)), pk2(0.69314718055994531f, 0.69314718055994531f), mx);
  }
  up2(r, h0, h1);
}

// ---- accurate tanh of a pair (kActTanhPair; SPLIT and TF32): u = z 2 log2(e) (the scale is folded into
// the accumulator scale), tanh|z| = 2 r - 1 with r = 1 / (1 + e), e = 2^-|u| in (0, 1]: absolute error
// ~1.2e-7 (the same form as the MUFU ex2 + rcp epilogue).  NEWTON: r by a quadratic seed on [1, 2]
// (1.7%) and two Newton steps (8e-8) in FFMA2 (8 FFMA2 per pair, 1 MUFU per unit); otherwise MUFU rcp.
template <bool NEWTON>
__device__ __forceinline__ void tanh_pair(float u0, float u1, float& h0, float& h1) {
  const uint64_t E = pk2(ex2_approx(-fabsf(u0)), ex2_approx(-fabsf(u1)));
  uint64_t R;
  if constexpr (NEWTON) {
    const uint64_t NS = fma2(E, pk2(-1.0f, -1.0f), pk2(-1.0f, -1.0f));        // -(1 + e)
    R = fma2(fma2s(NS, 0.30153724f, 1.39582404f), NS, pk2(2.08733358f, 2.08733358f));
    R = fma2(R, fma2(NS, R, pk2(1.0f, 1.0f)), R);
    R = fma2(R, fma2(NS, R, pk2(1.0f, 1.0f)), R);
  } else {
    float s0, s1;
    up2(fma2(E, pk2(1.0f, 1.0f), pk2(1.0f, 1.0f)), s0, s1);
    R = pk2(rcp_approx(s0), rcp_approx(s1));
  }
  float t0, t1;
  up2(fma2(R, pk2(2.0f, 2.0f), pk2(-1.0f, -1.0f)), t0, t1);
  h0 = copysignf(t0, u0);
  h1 = copysignf(t1, u1);
}

// ------------------------------------------------------------------------------------------------
// a7.  Fused statistics of the terminal values.
// ------------------------------------------------------------------------------------------------
struct StatAcc {
  double s1 = 0, s2 = 0, s3 = 0, s4 = 0, e1 = 0, e2 = 0;
  uint32_t n = 0, nnf = 0;
};

__device__ __forceinline__ void stat_add(StatAcc& a, const RunParams& p, float y, double ref, uint32_t* hist) {
  if (isfinite(y)) {
    const double yd = (double)y;
    const double d = yd - p.shift, d2 = d * d;
    a.s1 += d;
    a.s2 += d2;
    a.s3 += d2 * d;
    a.s4 += d2 * d2;
    a.n += 1;
    if (p.ref != kRefNone) {
      const double e = yd - ref;
      a.e1 += fabs(e);
      a.e2 += e * e;
    }
    if (p.n_bins > 0) {
      const double t = (yd - p.hist_lo) * p.hist_scale;
      int bin;
      if (yd < p.hist_lo) bin = 0;
      else if (t >= (double)p.n_bins) bin = p.n_bins + 1;
      else bin = 1 + (int)t;
      atomicAdd(&hist[bin], 1u);
    }
  } else {
    a.nnf += 1;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Call by ALL threads of the CTA (contains __syncthreads).  red: 8 doubles of shared memory.
__device__ __forceinline__ void stat_flush(const StatAcc& a, const RunParams& p, uint32_t* hist, double* red) {
  const int tid = threadIdx.x;
  if (tid < 8) red[tid] = 0.0;
  __syncthreads();
  double v[8] = {(double)a.n, (double)a.nnf, a.s1, a.s2, a.s3, a.s4, a.e1, a.e2};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double s = warp_sum(v[k]);
    if ((tid & 31) == 0 && s != 0.0) atomicAdd(&red[k], s);
  }
  __syncthreads();
  if (tid < 8 && red[tid] != 0.0) atomicAdd(&p.stats[tid], red[tid]);
  if (p.n_bins > 0) {
    for (int b = tid; b < p.n_bins + 2; b += blockDim.x) {
      const uint32_t c = hist[b];
      if (c) atomicAdd(&p.stats[kStatsHead + b], (double)c);
    }
  }
}

__device__ __forceinline__ void hist_init(const RunParams& p, uint32_t* hist) {
  if (p.has_stats && p.n_bins > 0)
    for (int b = threadIdx.x; b < p.n_bins + 2; b += blockDim.x) hist[b] = 0u;
}

// ------------------------------------------------------------------------------------------------
// Order statistics by radix select (7L-CDC marginal points, training-set labels): the order-preserving
// 32-bit key of an fp32 value (negative: all bits flipped; non-negative: sign bit set), so unsigned key
// order = float order (-0 < +0; NaNs are excluded by the callers).  Two targets per quantile level.
// ------------------------------------------------------------------------------------------------
constexpr int kCdcMaxT = 2 * kMaxM;

__device__ __forceinline__ uint32_t f2key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// Path-wise exact reference state on the same normals.
struct RefState {
  double r;   // GBM: sum of Z; OU: exact state
};

__device__ __forceinline__ void ref_init(RefState& s, const RunParams& p) {
  s.r = (p.ref == kRefOu) ? p.y0_d : 0.0;
}
__device__ __forceinline__ void ref_step(RefState& s, const RunParams& p, float Z) {
  if (p.ref == kRefGbm) s.r += (double)Z;
  else if (p.ref == kRefOu) s.r = fma(p.ref_a, s.r, p.ref_b) + p.ref_s * (double)Z;
}
__device__ __forceinline__ double ref_final(const RefState& s, const RunParams& p) {
  if (p.ref == kRefGbm) return p.y0_d * exp(p.ref_drift_T + p.ref_vol * s.r);
  return s.r;
}

}  // namespace sl7
