// sl7_cir.cu -- exact-collocation CIR on sm_100a: the 7L step with the
// conditional collocation points of the CIR transition itself instead of the ANN.
//
// The CIR transition Y(t + dt) | Y(t) = c * chi'^2(d, lam) with c = sigma^2 (1 - e^{-kappa dt}) / (4 kappa),
// d = 4 kappa Ybar / sigma^2, lam = Y+ e^{-kappa dt} / c (Y+ = max(Y, 0), reading R-24), so
//     y_j = c * F^{-1}_{d,lam}(Phi(x_j))                                         (Eq. 6.3)
// per path and step, then Y_{i+1} = g_m(X_hat) exactly as in the other exact modes.
//
// F is evaluated in float64 as its Poisson mixture F(x) = sum_k w_k P(d/2 + k, x/2),
// w_k = e^{-mu} mu^k / k!, mu = lam/2, P the regularised lower incomplete gamma: P is computed once at
// the Poisson mode (series for y < a + 1, otherwise Legendre's continued fraction for Q by the Wallis
// recurrences of its convergents) and carried to the other k by the exact recurrences
// P(a+1, y) = P(a, y) - G(a), G(a) = y^a e^{-y} / Gamma(a+1) (forward) and P(a, y) = P(a+1, y) + G(a) (backward), the weights by w_{k+1} = w_k mu / (k+1); the density comes
// from the same terms.  The quantile is a bracketed Newton iteration from the Patnaik (scaled central
// chi-square) + Wilson-Hilferty starting point, which takes the normal quantile x_j directly.
// The work is float64 special-function evaluation (~4 Newton steps x ~2 (sqrt(mu) + ...) terms x m nodes
// per path-step): a reference generator, not a throughput path.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "sl7_device.cuh"

namespace sl7 {

namespace {

struct Ncx2 {
  double a_m;    // d/2 + k_mode
  double lg_m;   // lgamma(a_m + 1)
  double mu;     // lam / 2
  double w_m;    // Poisson weight at the mode
  int k_m;       // Poisson mode floor(mu)
};

// regularised lower incomplete gamma P(a, y), y > 0, given lgamma(a + 1)
__device__ double gamma_p(double a, double y, double lg_a1) {
  const double lpre = a * log(y) - y - lg_a1;   // log(y^a e^{-y} / Gamma(a + 1))
  if (y < a + 1.0) {
    // two series terms per float64 reciprocal: y/(a+n) and y/(a+n+1) from 1/((a+n)(a+n+1))
    double term = 1.0, sum = 1.0, ap = a;
    for (int n = 0; n < 1000; ++n) {
      const double a1 = ap + 1.0, a2 = ap + 2.0, r = y / (a1 * a2);
      ap = a2;
      term *= a2 * r;
      sum += term;
      term *= a1 * r;
      sum += term;
      if (term < sum * 1e-17) break;
    }
    return exp(lpre) * sum;
  }
  // Q(a, y) = e^{-y} y^a / Gamma(a) / K with Legendre's continued fraction
  //   K = b_0 + a_1/(b_1 + a_2/(b_2 + ...)),  b_n = y + 2n + 1 - a,  a_n = -n (n - a),
  // evaluated by the fundamental (Wallis) recurrences of its convergents P_n / R_n:
  //   P_n = b_n P_{n-1} + a_n P_{n-2},  R_n = b_n R_{n-1} + a_n R_{n-2}  (P_{-1} = 1, R_{-1} = 0, R_0 = 1),
  // rescaled whenever the numerators grow large; 1/K = R_n / P_n.
  double pm = 1.0, p0 = y + 1.0 - a, rm = 0.0, r0 = 1.0;
  double h = r0 / p0;
  for (int n = 1; n < 2000; ++n) {
    const double an = -(double)n * ((double)n - a), bn = y + 2.0 * n + 1.0 - a;
    const double p1 = fma(bn, p0, an * pm), r1 = fma(bn, r0, an * rm);
    pm = p0; p0 = p1; rm = r0; r0 = r1;
    if (fabs(p0) > 1e150) {
      const double sc = 1.0 / fabs(p0);
      pm *= sc; p0 *= sc; rm *= sc; r0 *= sc;
    }
    const double hn = r0 / p0;
    const bool done = fabs(hn - h) <= 1e-16 * fabs(hn);
    h = hn;
    if (done) break;
  }
  return 1.0 - exp(lpre + log(a)) * h;
}

// F(x), dF/dx and d2F/dx2 of the noncentral chi-square (the density of term k is w_k G(a_k) a_k / (2y) with
// a_k = d/2 + k; its derivative multiplies it by (a_k - 1)/x - 1/2)
__device__ void ncx2_cdf_pdf(const Ncx2& n, double x, double& F, double& f, double& df) {
  const double y = 0.5 * x;
  if (!(y > 0.0)) {
    F = 0.0;
    f = 0.0;
    df = 0.0;
    return;
  }
  const double P = gamma_p(n.a_m, y, n.lg_m);
  const double G = exp(n.a_m * log(y) - y - n.lg_m);
  double Fs = n.w_m * P, fs = n.w_m * G * n.a_m, fs2 = fs * (n.a_m - 1.0);
  {
    double Pk = P, Gk = G, wk = n.w_m, ak = n.a_m;
    for (int k = n.k_m + 1; k < n.k_m + 100000; ++k) {
      Pk = fmax(Pk - Gk, 0.0);
      // y / (a + 1) and mu / k from one float64 reciprocal of (a + 1) k
      const double a1 = ak + 1.0, kd = (double)k, r = 1.0 / (a1 * kd);
      Gk *= y * kd * r;
      ak = a1;
      wk *= n.mu * a1 * r;
      Fs += wk * Pk;
      const double t = wk * Gk * ak;
      fs += t;
      fs2 = fma(t, ak - 1.0, fs2);
      if (wk < 1e-17) break;
    }
  }
  {
    double Pk = P, Gk = G, wk = n.w_m, ak = n.a_m;
    const double ry = 1.0 / y, rmu = 1.0 / n.mu;   // loop invariants: two float64 divisions per term saved
    for (int k = n.k_m - 1; k >= 0; --k) {
      Gk *= ak * ry;
      ak -= 1.0;
      Pk += Gk;
      wk *= (double)(k + 1) * rmu;
      Fs += wk * Pk;
      const double t = wk * Gk * ak;
      fs += t;
      fs2 = fma(t, ak - 1.0, fs2);
      if (wk < 1e-17) break;
    }
  }
  F = Fs;
  f = 0.5 * fs / y;
  df = (0.5 / y) * (fs2 / x - 0.5 * fs);
}

// F^{-1}(p) with z = Phi^{-1}(p) for the starting point (Sankaran's normal approximation of a power of the
// noncentral chi-square, a few 1e-3 relative), then bracketed Halley steps (cubic convergence: two or
// three evaluations); lo: a known lower bracket (F(lo) <= p)
__device__ double ncx2_quantile(const Ncx2& n, double p, double z, double d, double lam, double lo) {
  const double s1 = d + lam, s2 = d + 2.0 * lam, s3 = d + 3.0 * lam;
  const double h = 1.0 - (2.0 / 3.0) * s1 * s3 / (s2 * s2);
  const double pp = s2 / (s1 * s1), mm = (h - 1.0) * (1.0 - 3.0 * h);
  const double mu = 1.0 + h * pp * (h - 1.0 - 0.5 * (2.0 - h) * mm * pp);
  const double sd = h * sqrt(2.0 * pp * (1.0 + 0.5 * mm * pp));
  const double base = fmax(mu + sd * z, 1e-3);
  double x = fmax(s1 * pow(base, 1.0 / h), lo);
  double hi = CUDART_INF;
  for (int it = 0; it < 100; ++it) {
    double F, f, df;
    ncx2_cdf_pdf(n, x, F, f, df);
    const double g = F - p;
    if (g < 0.0) lo = x; else hi = x;
    if (g == 0.0) break;
    const double den = 2.0 * f * f - g * df;
    double xn = (den > 0.0) ? x - 2.0 * g * f / den : x - g / f;   // Halley, Newton if the curvature term misbehaves
    if (!(f > 0.0) || !(xn > lo && xn < hi)) xn = (hi < CUDART_INF) ? 0.5 * (lo + hi) : 2.0 * x + 1.0;
    const bool done = fabs(xn - x) <= 1e-13 * xn;
    x = xn;
    if (done) break;
  }
  return x;
}

template <int MR, bool RT_M, bool FAST>
__global__ void __launch_bounds__(256) exact_cir_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  hist_init(p, hist);
  __syncthreads();
  StatAcc acc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int m = RT_M ? p.m : MR;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_paths; q += stride) {
    const uint64_t gp = p.path_offset + q;
    float Y = p.y0;
    if (p.out_mode == kFull) p.out[q] = Y;
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    for (int i = 0; i < p.n_steps; ++i) {
      if ((i & 3) == 0) normals4<FAST>(p.key0, p.key1, gp, (uint32_t)(i >> 2), z0, z1, z2, z3);
      const float Z = z0;
      z0 = z1; z1 = z2; z2 = z3;
      // conditional law of the step: c chi'^2(d, lam(Y+))
      const double lam = fmax((double)Y, 0.0) * p.cir_lscale;
      Ncx2 n;
      n.mu = 0.5 * lam;
      n.k_m = (int)floor(n.mu);
      n.a_m = 0.5 * p.cir_d + (double)n.k_m;
      n.lg_m = lgamma(n.a_m + 1.0);
      n.w_m = (n.mu > 0.0) ? exp(-n.mu + (double)n.k_m * log(n.mu) - lgamma((double)n.k_m + 1.0)) : 1.0;
      float y[MR];
      double lo = 0.0;
#pragma unroll 1
      for (int j = 0; j < m; ++j) {
        const double xq = ncx2_quantile(n, p.cir_p[j], p.cir_x[j], p.cir_d, lam, lo);
        lo = xq;   // quantiles increase with j
        y[j] = (float)(p.cir_c * xq);
      }
      if (RT_M)
        for (int j = m; j < MR; ++j) y[j] = 0.0f;
      Y = gm_eval<MR, RT_M>(p, Z, y);
      if (p.out_mode == kFull) p.out[(uint64_t)(i + 1) * p.n_paths + q] = Y;
    }
    if (p.out_mode == kTerminal) p.out[q] = Y;
    if (p.has_stats) stat_add(acc, p, Y, 0.0, hist);
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

template <int MR, bool RT_M, bool FAST>
cudaError_t launch_cir_t(const RunParams& p, cudaStream_t st, int num_sms) {
  auto kernel = exact_cir_kernel<MR, RT_M, FAST>;
  const size_t smem = (p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0;
  cudaError_t e;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t need = (p.n_paths + 255) / 256, full = (uint64_t)per_sm * (uint64_t)num_sms;
  kernel<<<(unsigned)(need < full ? need : full), 256, smem, st>>>(p);
  return cudaGetLastError();
}

template <bool FAST>
cudaError_t launch_cir_f(const RunParams& p, cudaStream_t st, int num_sms) {
  switch (p.m) {
    case 5: return launch_cir_t<5, false, FAST>(p, st, num_sms);
    case 7: return launch_cir_t<7, false, FAST>(p, st, num_sms);
    default: return launch_cir_t<kMaxM, true, FAST>(p, st, num_sms);
  }
}

}  // namespace

int launch_exact_cir(const RunParams& p, void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return (int)((p.flags & SL7_FLAG_FAST_NORMALS) ? launch_cir_f<true>(p, st, num_sms)
                                                 : launch_cir_f<false>(p, st, num_sms));
}

}  // namespace sl7
