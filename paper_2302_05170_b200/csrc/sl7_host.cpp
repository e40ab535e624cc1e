// sl7_host.cpp -- host runtime of the C ABI (include/sl7.h): validation, host setup, weight blob
// parsing and folding, per-run constants, launches, host-buffer staging, statistics summary.
//
// Host setup (Algorithm I step 2 prerequisites, done in double, rounded once to fp32):
//   * Gauss-Hermite nodes (probabilists' reading): eigenvalues of the symmetric
//     tridiagonal Jacobi matrix (0 diagonal, sqrt(k) off-diagonal) by our own implicit QL
//     iteration (no LAPACK), polished by Newton on the He_m three-term recurrence, symmetrised.
//   * barycentric weights w_j = 1 / prod_{k != j}(x_j - x_k) (ref [8]).
//   * fp32 hi/lo split of the nodes: x = xhi + xlo.
//   * ANN layer 1 folding: dt and theta are constant per run, so
//     W1 (f - in_shift)/in_scale + b1 = l1w * Y + l1b with l1w, l1b computed in double here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sl7_internal.h"

using namespace sl7;

namespace {

thread_local std::string g_err = "";

}  // namespace

struct sl7_ctx_s {
  int device = 0;
  int m = 0;
  int act = 0;
  std::vector<int> dims;   // empty: exact-only context
  double x[kMaxM] = {0}, w[kMaxM] = {0};
  // network (host copy, as loaded)
  bool has_net = false;
  std::vector<std::vector<float>> W, b;
  bool has_norm = false;
  bool residual = false;          // blob flags bit 1: H_j = Y + sqrt(dt) (out_j out_scale_j + out_shift_j)
  std::vector<float> in_shift, in_scale, out_shift, out_scale;
  std::vector<float> dom_lo, dom_hi;   // blob flags bit 2: the feature box the network was fitted on
  // device images
  int width = 0;           // hidden width used by the FP32 kernel (50 or 64 padded)
  float* d_wf32 = nullptr;
  void* d_wtc = nullptr;   // bf16 SWIZZLE_128B operand image for the tcgen05 kernel
  void* d_wtc_split = nullptr;   // W 2^s split into two fp16 parts per layer (SL7_PREC_SPLIT)
  void* d_wtc_tf32 = nullptr;    // tf32 operand image (SL7_PREC_TF32)
  TcParams tcp;            // biases + image pointer for the tcgen05 kernel
  int num_sms = 148;
  // host-mode staging
  float* d_out_scratch = nullptr;
  size_t out_cap = 0;
  double* d_stats_scratch = nullptr;
  size_t stats_cap = 0;
  // sl7_simulate_host_async: two device staging slots used alternately, D2H on a context-owned stream
  struct Staging {
    float* d_out = nullptr;
    size_t out_cap = 0;
    double* d_stats = nullptr;
    size_t stats_cap = 0;
    cudaEvent_t copied = nullptr;   // D2H of this slot's last call finished
    bool used = false;
  } stage[2];
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t computed = nullptr;
  int next_stage = 0;
  // training-set generator: feature rows and terminal-value scratch
  EmRow* d_rows = nullptr;
  size_t rows_cap = 0;
  float* d_term_scratch = nullptr;
  size_t term_cap = 0;
  // sharded 7L-CDC run in progress (sl7_cdc_*)
  RunParams cdc_p;
  CdcLevels cdc_lv;
  std::vector<CdcHorizon> cdc_hz;   // SL7_SCHEME_CDC_PRED: per-step predictor constants of the last call
  void* cdc_stream = nullptr;
  bool cdc_ready = false;
  // 7L-CDC scratch (selection histograms + table) and state buffer for STATS-only runs
  void* d_cdc = nullptr;
  void* d_cdc_tabs = nullptr;   // SL7_SCHEME_CDC_PRED fused kernel: per-step tables
  int32_t cdc_tab_cap = 0;
  float* d_state = nullptr;
  size_t state_cap = 0;
  std::string err;
};

namespace {

sl7_status fail(sl7_ctx ctx, sl7_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  if (ctx) ctx->err = buf;
  return s;
}

sl7_status cuda_fail(sl7_ctx ctx, cudaError_t e, const char* what) {
  return fail(ctx, SL7_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; return; }
    ok = (prev == dev) || (cudaSetDevice(dev) == cudaSuccess);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ---- Gauss-Hermite nodes (the x_j are the roots of the probabilists' He_m) ----
// The three-term recurrence He_0 = 1, He_1 = x, He_{k+1} = x He_k - k He_{k-1} is the sequence of leading
// principal minors det(x I - J_k) of the Jacobi matrix J (zero diagonal, off-diagonal sqrt(k)), hence a
// Sturm sequence: the number of sign changes of He_0(x), ..., He_m(x) is the number of roots below x.  Each
// root is isolated by bisection on that count (the ratios q_k = He_k / He_{k-1} keep it overflow-free) and
// then polished by Newton on He_m with He_m' = m He_{m-1}.  All roots lie in |x| < sqrt(4m + 2).

// number of roots of He_m below x: m minus the sign changes of the Sturm sequence (counted on its ratios)
int hermite_roots_below(int m, double x) {
  int changes = 0;
  double q = x;                       // He_1 / He_0
  for (int k = 1;; ++k) {
    if (q == 0.0) q = -1e-300;        // a zero minor: the sign the sequence has just right of x
    if (q < 0.0) ++changes;
    if (k == m) break;
    q = x - (double)k / q;            // He_{k+1} / He_k
  }
  return m - changes;
}

// He_m(x) and He_{m-1}(x) by the recurrence
void hermite_pair(int m, double x, double& hm, double& hm1) {
  double a = 1.0, b = x;  // He_0, He_1
  if (m == 0) { hm = 1.0; hm1 = 0.0; return; }
  for (int k = 1; k < m; ++k) {
    const double c = x * b - k * a;
    a = b;
    b = c;
  }
  hm = b;
  hm1 = a;
}

void gh_grid(int m, double* x, double* w) {
  std::vector<double> r(m);
  const double bound = std::sqrt(4.0 * m + 2.0);
  for (int j = 0; j < m; ++j) {
    // the (j+1)-th smallest root lies in [lo, hi): roots_below(lo) <= j < roots_below(hi)
    double lo = -bound, hi = bound;
    for (int it = 0; it < 200 && hi - lo > 1e-15 * (1.0 + std::fabs(lo)); ++it) {
      const double mid = 0.5 * (lo + hi);
      if (hermite_roots_below(m, mid) > j) hi = mid; else lo = mid;
    }
    double xj = 0.5 * (lo + hi);
    for (int it = 0; it < 3; ++it) {  // Newton polish
      double hm, hm1;
      hermite_pair(m, xj, hm, hm1);
      if (hm1 == 0.0) break;
      xj -= hm / (m * hm1);
    }
    r[j] = xj;
  }
  for (int j = 0; j < m; ++j) x[j] = 0.5 * (r[j] - r[m - 1 - j]);  // exact symmetry
  for (int j = 0; j < m; ++j) {
    double p = 1.0;
    for (int k = 0; k < m; ++k)
      if (k != j) p *= (x[j] - x[k]);
    w[j] = 1.0 / p;
  }
}

bool finite_all(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

uint32_t rd_u32(const unsigned char* p) {
  uint32_t v;
  std::memcpy(&v, p, 4);
  return v;
}

// OU conditional std factor sqrt((1 - e^{-2 lam dt}) / (2 lam)), series for lam dt < 1e-6 (Eq. 6.6)
double ou_std(double lam, double sigma, double dt) {
  const double a = lam * dt;
  const double vf = (a < 1e-6) ? dt * (1.0 - a + (2.0 / 3.0) * a * a) : -std::expm1(-2.0 * a) / (2.0 * lam);
  return sigma * std::sqrt(vf);
}

sl7_status build_f32_image(sl7_ctx c) {
  const int L = (int)c->dims.size() - 2;   // hidden layers
  const int M = c->m;
  bool all50 = true;
  for (int l = 1; l <= L; ++l) all50 = all50 && c->dims[l] == 50;
  const int H = (all50 && (M == 5 || M == 7)) ? 50 : 64;
  const int HS = (H == 50) ? 52 : 64;
  const int MR = (H == 50) ? M : kMaxM;
  c->width = H;
  std::vector<float> img(f32_weight_floats(H, HS, L, MR), 0.0f);
  size_t off = 0;
  for (int l = 1; l < L; ++l) {  // blob layer l maps hidden l -> hidden l+1
    const int fi = c->dims[l], fo = c->dims[l + 1];
    for (int j = 0; j < fo; ++j)
      for (int k = 0; k < fi; ++k) img[off + (size_t)j * HS + k] = c->W[l][(size_t)j * fi + k];
    off += (size_t)H * HS;
    for (int j = 0; j < fo; ++j) img[off + j] = c->b[l][j];
    off += (size_t)((H + 3) & ~3);
  }
  {
    const int fi = c->dims[L];
    for (int j = 0; j < M; ++j)
      for (int k = 0; k < fi; ++k) img[off + (size_t)j * HS + k] = c->W[L][(size_t)j * fi + k];
    off += (size_t)MR * HS;
    for (int j = 0; j < M; ++j) img[off + j] = c->b[L][j];
  }
  if (c->d_wf32) cudaFree(c->d_wf32);
  c->d_wf32 = nullptr;
  cudaError_t e = cudaMalloc(&c->d_wf32, img.size() * sizeof(float));
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(weights)");
  e = cudaMemcpy(c->d_wf32, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemcpy(weights)");
  return SL7_OK;
}

uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// fp16 (binary16) round-to-nearest-even of a finite |v| < 65504, and its value (SL7_PREC_SPLIT operands)
uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  const uint32_t ax = x & 0x7FFFFFFFu;
  if (ax >= 0x38800000u) {                 // |f| >= 2^-14: normal binary16
    uint32_t r = ax - 0x38000000u;         // exponent rebias 127 -> 15
    r += 0xFFFu + ((r >> 13) & 1u);        // round the 23-bit mantissa to 10 bits, ties to even
    return (uint16_t)(sign | (r >> 13));
  }
  // subnormal binary16: multiples of 2^-24 (the scaling by 2^24 is exact; nearbyint rounds ties to even)
  return (uint16_t)(sign | (uint16_t)std::nearbyint(std::fabs((double)f) * 16777216.0));
}
float f16_value(uint16_t h) {
  const int e = (h >> 10) & 0x1F, m = h & 0x3FF;
  const double v = e ? std::ldexp(1024.0 + m, e - 25) : std::ldexp((double)m, -24);
  return (float)((h & 0x8000u) ? -v : v);
}

// bf16 operand image of the MMA layers (layout: TcParams in sl7_internal.h) + fp32 biases.
sl7_status build_tc_image(sl7_ctx c) {
  const int L = (int)c->dims.size() - 2;
  const int nL = L - 1;
  auto bf = [](float v) {   // value of the bf16 (RNE) rounding of v
    uint32_t u = (uint32_t)f32_to_bf16_rne(v) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  };
  // np = 1: W rounded to bf16 (SL7_PREC_BF16).  np = 2 (SL7_PREC_SPLIT): W 2^s_l = W0 + W1 split into two
  // fp16 parts (W0 = fp16(W 2^s), W1 = fp16(W 2^s - W0): 22 significant bits), s_l a per-layer power of two
  // that puts max |W|, |b| of the layer at <= 2^14, so W1 stays out of the binary16 subnormals for all but
  // the layer's smallest weights; part p of hidden tile l at (np (l-1) + p) * 8 KB, output part p after them.
  auto layer_exp = [&](int l) {
    const int fi = c->dims[l], fo = c->dims[l + 1];
    double mx = 0.0;
    for (int i = 0; i < fi * fo; ++i) mx = std::max(mx, (double)std::fabs(c->W[l][(size_t)i]));
    for (int n = 0; n < fo; ++n) mx = std::max(mx, (double)std::fabs(c->b[l][n]));
    if (!(mx > 0.0)) return 0;
    int e;
    std::frexp(mx, &e);                     // mx in [2^(e-1), 2^e)
    return std::max(-60, std::min(60, 14 - e));
  };
  auto build = [&](int np) {
    std::vector<uint16_t> img((size_t)np * (nL * kTcTileBytes + kTcOutBytes) / 2, 0);
    auto put = [&](size_t tile_off_bytes, int n, int k, uint16_t v) {
      const size_t byte =
          tile_off_bytes + (size_t)n * 128 + (size_t)((((k * 2) >> 4) ^ (n & 7)) << 4) + (size_t)((k * 2) & 15);
      img[byte / 2] = v;
    };
    for (int l = 1; l <= L; ++l) {   // blob layer l: hidden l -> hidden l+1 (l < L) or -> output (l == L)
      const int fi = c->dims[l], fo = c->dims[l + 1];
      const size_t part_bytes = (l < L) ? kTcTileBytes : kTcOutBytes;
      const size_t base = (l < L) ? (size_t)np * (l - 1) * kTcTileBytes : (size_t)np * nL * kTcTileBytes;
      const int se = (np == 2) ? layer_exp(l) : 0;
      c->tcp.split_exp[l - 1] = se;
      for (int n = 0; n < fo; ++n)
        for (int k = 0; k < fi; ++k) {
          const float w = c->W[l][(size_t)n * fi + k];
          if (np == 1) {
            put(base, n, k, f32_to_bf16_rne(w));
          } else {
            const float ws = std::ldexp(w, se);            // exact (power of two)
            const uint16_t h0 = f32_to_f16_rne(ws);
            put(base, n, k, h0);
            put(base + part_bytes, n, k, f32_to_f16_rne(ws - f16_value(h0)));
          }
        }
      if (c->width == 50) {
        // the width-50 kernel (FOLD) feeds A = 1.0 in K columns 50..52 (part 0 only): the bias enters
        // the fp32 accumulation as three terms whose sum reproduces the fp32 bias (hi + mid + lo)
        for (int n = 0; n < fo; ++n) {
          if (np == 1) {
            const float b = c->b[l][n];
            const float hi = bf(b), mid = bf(b - hi), lo = bf(b - hi - mid);
            put(base, n, 50, f32_to_bf16_rne(hi));
            put(base, n, 51, f32_to_bf16_rne(mid));
            put(base, n, 52, f32_to_bf16_rne(lo));
          } else {
            const float b = std::ldexp(c->b[l][n], se);
            const uint16_t hi = f32_to_f16_rne(b);
            const uint16_t mid = f32_to_f16_rne(b - f16_value(hi));
            const uint16_t lo = f32_to_f16_rne(b - f16_value(hi) - f16_value(mid));
            put(base, n, 50, hi);
            put(base, n, 51, mid);
            put(base, n, 52, lo);
          }
        }
      }
    }
    return img;
  };
  std::memset(&c->tcp, 0, sizeof c->tcp);
  for (int l = 1; l <= L; ++l)
    for (int n = 0; n < c->dims[l + 1]; ++n) {
      if (l < L) c->tcp.bias[l - 1][n] = c->b[l][n];
      else c->tcp.bout[n] = c->b[l][n];
    }
  c->tcp.n_mma_hidden = nL;
  for (int np : {1, 2}) {
    const std::vector<uint16_t> img = build(np);
    void*& d = (np == 1) ? c->d_wtc : c->d_wtc_split;
    if (d) cudaFree(d);
    d = nullptr;
    cudaError_t e = cudaMalloc(&d, img.size() * 2);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(tc weights)");
    e = cudaMemcpy(d, img.data(), img.size() * 2, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemcpy(tc weights)");
  }
  // SL7_PREC_TF32 image: each tile = two SWIZZLE_128B K-blocks [N rows][128 B = 32 tf32] (K 0..31, 32..63),
  // values rounded with cvt.rna semantics (ties away from zero), the width-50 bias as three tf32 terms
  {
    auto rna = [](float v) {
      uint32_t u;
      std::memcpy(&u, &v, 4);
      u = (u + 0x1000u) & 0xFFFFE000u;
      float f;
      std::memcpy(&f, &u, 4);
      return f;
    };
    const size_t tile_b = 2 * (size_t)kTcTileBytes, out_b = 2 * (size_t)kTcOutBytes;
    std::vector<float> img((nL * tile_b + out_b) / 4, 0.0f);
    auto put = [&](size_t off, int nrows, int n, int k, float v) {
      const size_t byte = off + (size_t)(k >> 5) * nrows * 128 + (size_t)n * 128 +
                          (size_t)(((((k & 31) * 4) >> 4) ^ (n & 7)) << 4) + (size_t)(((k & 31) * 4) & 15);
      img[byte / 4] = v;
    };
    for (int l = 1; l <= L; ++l) {
      const int fi = c->dims[l], fo = c->dims[l + 1];
      const int nrows = (l < L) ? kTcN : kTcNOut;
      const size_t base = (l < L) ? (size_t)(l - 1) * tile_b : (size_t)nL * tile_b;
      for (int n = 0; n < fo; ++n)
        for (int k = 0; k < fi; ++k) put(base, nrows, n, k, rna(c->W[l][(size_t)n * fi + k]));
      if (c->width == 50)
        for (int n = 0; n < fo; ++n) {
          const float b = c->b[l][n];
          const float hi = rna(b), mid = rna(b - hi), lo = rna(b - hi - mid);
          put(base, nrows, n, 50, hi);
          put(base, nrows, n, 51, mid);
          put(base, nrows, n, 52, lo);
        }
    }
    if (c->d_wtc_tf32) cudaFree(c->d_wtc_tf32);
    c->d_wtc_tf32 = nullptr;
    cudaError_t e = cudaMalloc(&c->d_wtc_tf32, img.size() * 4);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(tf32 weights)");
    e = cudaMemcpy(c->d_wtc_tf32, img.data(), img.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemcpy(tf32 weights)");
  }
  c->tcp.wimg = c->d_wtc;
  c->tcp.wimg_split = c->d_wtc_split;
  c->tcp.wimg_tf32 = c->d_wtc_tf32;
  return SL7_OK;
}

// Part of RunParams common to every path kernel (7L, CDC, Euler-Maruyama): RNG, grid, outputs,
// statistics and the strong-error reference (evaluated on steps of ref_dt, ref_steps of them).
// Validates the arguments it consumes; the caller has validated dt and n_steps.
sl7_status prepare_base(sl7_ctx c, double Y0, int32_t n_steps, double ref_dt, int64_t ref_steps, uint64_t n_paths, uint64_t seed,
                        sl7_out out_mode, const sl7_run_opts* o, RunParams& p, bool have_out, bool have_stats) {
  if (n_paths < 1) return fail(c, SL7_EINVAL, "n_paths must be >= 1");
  if (o->path_offset + (n_paths - 1) < o->path_offset) return fail(c, SL7_EINVAL, "path_offset + n_paths - 1 overflows 2^64");
  if (!std::isfinite(Y0)) return fail(c, SL7_EINVAL, "Y0 must be finite");
  if (out_mode != SL7_OUT_FULL && out_mode != SL7_OUT_TERMINAL && out_mode != SL7_OUT_STATS)
    return fail(c, SL7_EINVAL, "out_mode");
  if (out_mode != SL7_OUT_STATS && !have_out) return fail(c, SL7_EINVAL, "d_out is NULL for a FULL/TERMINAL run");
  if (out_mode == SL7_OUT_STATS && !have_stats) return fail(c, SL7_EINVAL, "d_stats is NULL for a STATS run");
  if (have_stats) {
    if (o->n_bins < 0 || o->n_bins > 16384) return fail(c, SL7_EINVAL, "n_bins must be in 0..16384");
    if (o->n_bins > 0 && !(o->hist_hi > o->hist_lo && std::isfinite(o->hist_lo) && std::isfinite(o->hist_hi)))
      return fail(c, SL7_EINVAL, "hist_lo/hist_hi");
    if (!std::isfinite(o->shift)) return fail(c, SL7_EINVAL, "shift");
  }
  if (o->ref != SL7_REF_NONE && o->ref != SL7_REF_GBM && o->ref != SL7_REF_OU) return fail(c, SL7_EINVAL, "ref");
  if (o->ref != SL7_REF_NONE && !finite_all(o->ref_theta, 3)) return fail(c, SL7_EINVAL, "ref_theta");
  if (o->ref == SL7_REF_OU && (o->ref_theta[1] < 0 || o->ref_theta[2] < 0)) return fail(c, SL7_EINVAL, "ref_theta (lam, sigma >= 0)");

  std::memset(&p, 0, sizeof p);
  p.m = c->m;
  p.n_steps = n_steps;
  p.out_mode = (int)out_mode;
  p.n_paths = n_paths;
  p.path_offset = o->path_offset;
  p.key0 = (uint32_t)seed;
  p.key1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {   // Philox4x32-10 key schedule: k += (W0, W1) between rounds
    p.rk0[r] = p.key0 + (uint32_t)r * 0x9E3779B9u;
    p.rk1[r] = p.key1 + (uint32_t)r * 0xBB67AE85u;
  }
  p.y0 = (float)Y0;
  p.y0_d = (double)(float)Y0;
  for (int j = 0; j < kMaxM; ++j) {
    if (j < c->m) {
      const float hi = (float)c->x[j];
      p.xhi[j] = hi;
      p.xlo[j] = (float)(c->x[j] - (double)hi);
      p.w[j] = (float)c->w[j];
    } else {
      p.xhi[j] = p.xlo[j] = p.w[j] = 0.0f;   // padded slot: w = 0 (no contribution)
    }
  }
  p.ref = (int)o->ref;
  if (o->ref == SL7_REF_GBM) {
    const double mu = o->ref_theta[0], s = o->ref_theta[1];
    p.ref_drift_T = (mu - 0.5 * s * s) * ref_dt * (double)ref_steps;
    p.ref_vol = s * std::sqrt(ref_dt);
  } else if (o->ref == SL7_REF_OU) {
    const double ybar = o->ref_theta[0], lam = o->ref_theta[1], s = o->ref_theta[2];
    const double e = std::exp(-lam * ref_dt);
    p.ref_a = e;
    p.ref_b = ybar * (1.0 - e);
    p.ref_s = ou_std(lam, s, ref_dt);
  }
  p.has_stats = have_stats ? 1 : 0;
  p.n_bins = have_stats ? o->n_bins : 0;
  p.shift = o->shift;
  p.hist_lo = o->hist_lo;
  p.hist_scale = (p.n_bins > 0) ? (double)p.n_bins / (o->hist_hi - o->hist_lo) : 0.0;
  return SL7_OK;
}

// Fill RunParams for one sl7_simulate call; all validation happens here (synchronously, before any launch).
sl7_status prepare(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta, int32_t n_theta,
                   uint64_t n_paths, uint64_t seed, sl7_out out_mode, const sl7_run_opts* o, RunParams& p,
                   bool have_out, bool have_stats) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!o) return fail(c, SL7_EINVAL, "opts is NULL");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, SL7_EINVAL, "dt must be finite and > 0");
  if (n_steps < 1) return fail(c, SL7_EINVAL, "n_steps must be >= 1");
  if (n_theta < 0 || n_theta > SL7_MAX_THETA || (n_theta > 0 && !theta)) return fail(c, SL7_EINVAL, "theta/n_theta");
  if (n_theta > 0 && !finite_all(theta, n_theta)) return fail(c, SL7_EINVAL, "theta must be finite");
  sl7_status st = prepare_base(c, Y0, n_steps, dt, n_steps, n_paths, seed, out_mode, o, p, have_out, have_stats);
  if (st != SL7_OK) return st;
  switch (o->colloc) {
    case SL7_COLLOC_EXACT_GBM: {
      if (n_theta != 2) return fail(c, SL7_EINVAL, "EXACT_GBM needs theta = (mu, sigma)");
      const double mu = theta[0], s = theta[1];
      if (s < 0) return fail(c, SL7_EINVAL, "theta: sigma >= 0");
      double cj[kMaxM];
      for (int j = 0; j < c->m; ++j) {
        cj[j] = std::exp((mu - 0.5 * s * s) * dt + s * std::sqrt(dt) * c->x[j]);
        p.c[j] = (float)cj[j];
      }
      if (o->flags & SL7_FLAG_SPECIALIZED) {
        if (c->m > 8) return fail(c, SL7_EUNSUPPORTED, "SL7_FLAG_SPECIALIZED needs m <= 8");
        // monomial coefficients of the interpolant of c_j: solve sum_k q_k x_j^k = c_j (Gauss, pivoting)
        const int m = c->m;
        double A[8][9];
        for (int j = 0; j < m; ++j) {
          double xp = 1.0;
          for (int k = 0; k < m; ++k) { A[j][k] = xp; xp *= c->x[j]; }
          A[j][m] = cj[j];
        }
        for (int col = 0; col < m; ++col) {
          int piv = col;
          for (int r = col + 1; r < m; ++r)
            if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
          for (int k = 0; k <= m; ++k) std::swap(A[col][k], A[piv][k]);
          for (int r = 0; r < m; ++r) {
            if (r == col) continue;
            const double f = A[r][col] / A[col][col];
            for (int k = col; k <= m; ++k) A[r][k] -= f * A[col][k];
          }
        }
        for (int k = 0; k < 8; ++k) p.q[k] = (k < m) ? (float)(A[k][m] / A[k][k]) : 0.0f;
      }
      p.colloc = kExactGbm;
      break;
    }
    case SL7_COLLOC_EXACT_OU: {
      if (n_theta != 3) return fail(c, SL7_EINVAL, "EXACT_OU needs theta = (Ybar, lam, sigma)");
      const double ybar = theta[0], lam = theta[1], s = theta[2];
      if (lam < 0 || s < 0) return fail(c, SL7_EINVAL, "theta: lam >= 0 and sigma >= 0");
      const double e = std::exp(-lam * dt), sd = ou_std(lam, s, dt);
      p.ou_a = (float)e;
      p.ou_b = (float)(ybar * (1.0 - e));
      p.ou_s = (float)sd;
      for (int j = 0; j < c->m; ++j) p.c[j] = (float)(sd * c->x[j]);
      p.colloc = kExactOu;
      break;
    }
    case SL7_COLLOC_EXACT_CIR: {
      if (n_theta != 3) return fail(c, SL7_EINVAL, "EXACT_CIR needs theta = (kappa, Ybar, sigma)");
      const double kappa = theta[0], ybar = theta[1], s = theta[2];
      if (!(kappa > 0) || !(ybar > 0) || !(s > 0)) return fail(c, SL7_EINVAL, "theta: kappa, Ybar, sigma > 0");
      if (o->flags & SL7_FLAG_SPECIALIZED) return fail(c, SL7_EUNSUPPORTED, "EXACT_CIR: SL7_FLAG_SPECIALIZED");
      if (o->scheme != SL7_SCHEME_7L) return fail(c, SL7_EUNSUPPORTED, "EXACT_CIR: scheme CDC");
      p.cir_c = s * s * (-std::expm1(-kappa * dt)) / (4.0 * kappa);
      p.cir_d = 4.0 * kappa * ybar / (s * s);
      p.cir_lscale = std::exp(-kappa * dt) / p.cir_c;
      for (int j = 0; j < kMaxM; ++j) {
        p.cir_x[j] = (j < c->m) ? c->x[j] : 0.0;
        p.cir_p[j] = (j < c->m) ? 0.5 * std::erfc(-c->x[j] / std::sqrt(2.0)) : 0.0;
      }
      p.colloc = kExactCir;
      break;
    }
    case SL7_COLLOC_ANN: {
      if (c->dims.empty()) return fail(c, SL7_ESTATE, "ANN mode on a context created without layer_dims");
      if (!c->has_net) return fail(c, SL7_ESTATE, "ANN mode before sl7_load_weights");
      const int d_in = c->dims[0];
      if (n_theta != d_in - 2) return fail(c, SL7_EINVAL, "n_theta must equal layer_dims[0] - 2");
      if (o->prec != SL7_PREC_FP32 && o->prec != SL7_PREC_BF16 && o->prec != SL7_PREC_SPLIT && o->prec != SL7_PREC_TF32)
        return fail(c, SL7_EINVAL, "prec");
      const int H1 = c->dims[1];
      // features f = (Y, dt, theta...); normalised f' = (f - in_shift) / in_scale
      std::vector<double> f(d_in), sh(d_in, 0.0), sc(d_in, 1.0);
      f[0] = 0.0;
      f[1] = dt;
      for (int t = 0; t < n_theta; ++t) f[2 + t] = theta[t];
      if (c->has_norm)
        for (int k = 0; k < d_in; ++k) { sh[k] = c->in_shift[k]; sc[k] = c->in_scale[k]; }
      for (int k = 0; k < kMaxW; ++k) { p.l1w[k] = 0.0f; p.l1b[k] = 0.0f; }
      for (int k = 0; k < H1; ++k) {
        const float* Wr = &c->W[0][(size_t)k * d_in];
        double bias = c->b[0][k] - (double)Wr[0] * sh[0] / sc[0];
        for (int q = 1; q < d_in; ++q) bias += (double)Wr[q] * (f[q] - sh[q]) / sc[q];
        p.l1w[k] = (float)((double)Wr[0] / sc[0]);
        p.l1b[k] = (float)bias;
        p.l1w_d[k] = (double)Wr[0] / sc[0];
        p.l1b_d[k] = bias;
      }
      const double rs = c->residual ? std::sqrt(dt) : 1.0;
      for (int j = 0; j < kMaxM; ++j) {
        const double sc_j = (j < c->m && c->has_norm) ? c->out_scale[j] : (j < c->m ? 1.0 : 0.0);
        const double sh_j = (j < c->m && c->has_norm) ? c->out_shift[j] : 0.0;
        p.out_scale[j] = (float)(rs * sc_j);
        p.out_shift[j] = (float)(rs * sh_j);
      }
      p.res_y = c->residual ? 1.0f : 0.0f;
      p.act = c->act;
      p.n_hidden = (int)c->dims.size() - 2;
      p.width = c->width;
      p.wdev = c->d_wf32;
      p.colloc = kAnn;
      break;
    }
    default:
      return fail(c, SL7_EINVAL, "colloc");
  }
  if (o->flags & ~(SL7_FLAG_FAST_NORMALS | SL7_FLAG_SPECIALIZED)) return fail(c, SL7_EINVAL, "flags");
  if (o->scheme != SL7_SCHEME_7L && o->scheme != SL7_SCHEME_CDC && o->scheme != SL7_SCHEME_CDC_PRED)
    return fail(c, SL7_EINVAL, "scheme");
  if (o->scheme != SL7_SCHEME_7L) {
    if (o->ref != SL7_REF_NONE) return fail(c, SL7_EUNSUPPORTED, "scheme CDC: ref must be SL7_REF_NONE");
    if (o->flags & ~SL7_FLAG_FAST_NORMALS)
      return fail(c, SL7_EUNSUPPORTED, "scheme CDC: flags may only hold SL7_FLAG_FAST_NORMALS");
    if (p.colloc == kAnn && o->prec != SL7_PREC_FP32)
      return fail(c, SL7_EUNSUPPORTED, "scheme CDC: the m-row table runs in fp32 (prec must be SL7_PREC_FP32)");
  }
  p.flags = (p.colloc == kAnn && o->scheme == SL7_SCHEME_7L) ? 0u : o->flags;
  return SL7_OK;
}

// Euler-Maruyama constants of one (model, theta, dtau); shared by sl7_simulate_em and sl7_training_set so
// that a training row and the equivalent EM call use bit-identical coefficients.
sl7_status em_constants(sl7_ctx c, int model, const double* theta, int32_t n_theta, double dtau, float& a, float& s,
                        float& ybar) {
  if (model != SL7_MODEL_GBM && model != SL7_MODEL_OU && model != SL7_MODEL_CIR) return fail(c, SL7_EINVAL, "model");
  const int need = (model == SL7_MODEL_GBM) ? 2 : 3;
  if (n_theta != need || !theta) return fail(c, SL7_EINVAL, "theta: model %d needs %d parameters", model, need);
  if (!finite_all(theta, need)) return fail(c, SL7_EINVAL, "theta must be finite");
  const double sq = std::sqrt(dtau);
  if (model == SL7_MODEL_GBM) {
    if (theta[1] < 0) return fail(c, SL7_EINVAL, "theta: sigma >= 0");
    a = (float)(theta[0] * dtau);
    s = (float)(theta[1] * sq);
    ybar = 0.0f;
  } else {
    // OU (Ybar, lam, sigma); CIR (kappa, Ybar, sigma)
    const double rate = (model == SL7_MODEL_OU) ? theta[1] : theta[0];
    const double mean = (model == SL7_MODEL_OU) ? theta[0] : theta[1];
    if (rate < 0 || theta[2] < 0) return fail(c, SL7_EINVAL, "theta: rate >= 0 and sigma >= 0");
    a = (float)(rate * dtau);
    s = (float)(theta[2] * sq);
    ybar = (float)mean;
  }
  return SL7_OK;
}

sl7_status prepare_em(sl7_ctx c, int model, double Y0, double dt, int32_t n_steps, int32_t substeps, const double* theta,
                      int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode, const sl7_run_opts* o,
                      RunParams& p, bool have_out, bool have_stats) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!o) return fail(c, SL7_EINVAL, "opts is NULL");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(c, SL7_EINVAL, "dt must be finite and > 0");
  if (n_steps < 1) return fail(c, SL7_EINVAL, "n_steps must be >= 1");
  if (substeps < 1) return fail(c, SL7_EINVAL, "substeps must be >= 1");
  if ((int64_t)n_steps * substeps > (int64_t)1 << 31) return fail(c, SL7_EINVAL, "n_steps * substeps > 2^31");
  if (o->flags & ~SL7_FLAG_FAST_NORMALS) return fail(c, SL7_EINVAL, "flags (EM: SL7_FLAG_FAST_NORMALS only)");
  const double dtau = dt / substeps;
  float a, s, yb;
  sl7_status st = em_constants(c, model, theta, n_theta, dtau, a, s, yb);
  if (st != SL7_OK) return st;
  st = prepare_base(c, Y0, n_steps, dtau, (int64_t)n_steps * substeps, n_paths, seed, out_mode, o, p, have_out, have_stats);
  if (st != SL7_OK) return st;
  p.em_model = model;
  p.em_K = substeps;
  p.em_a = a;
  p.em_s = s;
  p.em_ybar = yb;
  p.flags = o->flags;
  p.colloc = -1;
  return SL7_OK;
}

sl7_status run(sl7_ctx c, RunParams& p, const sl7_run_opts* o, float* d_out, double* d_stats) {
  p.out = d_out;
  p.stats = d_stats;
  if (d_stats && !o->accumulate) {
    const int e = launch_zero_stats(d_stats, sl7_stats_elems(o->n_bins), o->stream);
    if (e) return cuda_fail(c, (cudaError_t)e, "zero stats");
  }
  int e;
  if (p.em_model != 0) {
    e = launch_em(p, o->stream, c->num_sms);
  } else if (o->scheme == SL7_SCHEME_CDC || o->scheme == SL7_SCHEME_CDC_PRED) {
    // 7L-CDC: states in HBM between steps (FULL rows, the TERMINAL output, or context scratch)
    if (!c->d_cdc) {
      cudaError_t ce = cudaMalloc(&c->d_cdc, cdc_scratch_bytes());
      if (ce != cudaSuccess) return cuda_fail(c, ce, "cudaMalloc(cdc scratch)");
    }
    e = cdc_init_scratch(c->d_cdc, o->stream);
    if (e) return cuda_fail(c, (cudaError_t)e, "cdc scratch init");
    // the fused CDC_PRED kernel (m = 5, 7) keeps every path's state in registers through all steps: no
    // state buffer in STATS mode
    const bool pred_fused = o->scheme == SL7_SCHEME_CDC_PRED && (c->m == 5 || c->m == 7) &&
                            p.n_steps <= kCdcFusedMaxSteps;
    std::vector<float*> rows;
    if (p.out_mode == kFull) {
      for (int i = 0; i <= p.n_steps; ++i) rows.push_back(d_out + (size_t)i * p.n_paths);
    } else if (p.out_mode == kTerminal) {
      rows.push_back(d_out);
    } else if (pred_fused) {
      rows.push_back(nullptr);
    } else {
      if (c->state_cap < p.n_paths) {
        if (c->d_state) cudaFree(c->d_state);
        c->d_state = nullptr;
        c->state_cap = 0;
        cudaError_t ce = cudaMalloc(&c->d_state, p.n_paths * sizeof(float));
        if (ce != cudaSuccess) return cuda_fail(c, ce, "cudaMalloc(cdc state)");
        c->state_cap = p.n_paths;
      }
      rows.push_back(c->d_state);
    }
    CdcLevels lv;
    for (int k = 0; k < kMaxM; ++k) lv.p[k] = (k < c->m) ? 0.5 * std::erfc(-c->x[k] / std::sqrt(2.0)) : 0.0;
    if (o->scheme == SL7_SCHEME_CDC_PRED) {
      if (c->cdc_hz.size() != (size_t)p.n_steps)
        return fail(c, SL7_ESTATE, "CDC_PRED horizons not prepared for this call (internal)");
      void* tabs = nullptr;
      if (pred_fused) {   // fused all-steps kernel
        if (c->cdc_tab_cap < p.n_steps) {
          if (c->d_cdc_tabs) cudaFree(c->d_cdc_tabs);
          c->d_cdc_tabs = nullptr;
          c->cdc_tab_cap = 0;
          cudaError_t ce = cudaMalloc(&c->d_cdc_tabs, (size_t)p.n_steps * cdc_table_bytes());
          if (ce != cudaSuccess) return cuda_fail(c, ce, "cudaMalloc(cdc tables)");
          c->cdc_tab_cap = p.n_steps;
        }
        tabs = c->d_cdc_tabs;
      }
      e = launch_cdc_pred(p, c->cdc_hz.data(), c->d_cdc, rows.data(), (int)rows.size(), o->stream, c->num_sms, tabs);
    }
    else
      e = launch_cdc(p, lv, c->d_cdc, rows.data(), (int)rows.size(), o->stream, c->num_sms);
  } else if (p.colloc == kAnn && (o->prec == SL7_PREC_BF16 || o->prec == SL7_PREC_SPLIT || o->prec == SL7_PREC_TF32)) {
    // per-run part of the TC parameters: layer 1 folded (as in RunParams) and pre-scaled in double
    TcParams t = c->tcp;
#ifdef SL7_AB_HOOKS
    // experiment builds only (-DSL7_AB_HOOKS): SL7_TC_VARIANT selects the epilogue variants timed in
    // DESIGN.md §6; variant 9 skips the MMAs (timing only, wrong results).  Product builds ignore it.
    const char* v = std::getenv("SL7_TC_VARIANT");
    t.variant = v ? std::atoi(v) : 0;
#else
    t.variant = 0;
#endif
    t.split = (o->prec == SL7_PREC_SPLIT) ? 1 : 0;
    t.tf32 = (o->prec == SL7_PREC_TF32) ? 1 : 0;
    // tanh on MUFU.TANH in BF16 mode (SL7_TC_VARIANT 1..9 select the ex2 + rcp epilogues of DESIGN.md §6 for
    // A/B timing); SPLIT and TF32 keep the accurate epilogue (their rounding decisions must follow O3 / O6)
    const bool ab_hook = (t.variant >= 1 && t.variant <= 9);
    t.tanh_mufu = (c->act == SL7_ACT_TANH && !t.split && !t.tf32 && !ab_hook) ? 1 : 0;
    const double sc = (c->act == SL7_ACT_TANH && !t.tanh_mufu) ? 2.0 / std::log(2.0) : 1.0;
    t.act_scale = (float)sc;
    for (int k = 0; k < kTcN; ++k) {
      t.l1w[k] = (float)(p.l1w_d[k] * sc);
      t.l1b[k] = (float)(p.l1b_d[k] * sc);
    }
    for (int l = 0; l < t.n_mma_hidden; ++l)
      for (int k = 0; k < kTcN; ++k) t.bias[l][k] = (float)((double)c->tcp.bias[l][k] * sc);
    // the SPLIT image holds W 2^s_l: its accumulators are scaled back by 2^-s_l (exact) in the epilogue
    for (int l = 0; l < t.n_mma_hidden; ++l) t.lscale[l] = (float)std::ldexp(sc, t.split ? -c->tcp.split_exp[l] : 0);
    t.oscale = (float)std::ldexp(1.0, t.split ? -c->tcp.split_exp[t.n_mma_hidden] : 0);
    e = launch_tc_kernel(p, t, o->stream, c->num_sms);
  } else {
    e = launch_step_kernel(p, (int)o->prec, o->stream, c->num_sms);
  }
  if (e) return cuda_fail(c, (cudaError_t)e, "step kernel launch");
  return SL7_OK;
}

}  // namespace

extern "C" {

int32_t sl7_abi_version(void) { return SL7_ABI_VERSION; }

const char* sl7_status_str(sl7_status s) {
  switch (s) {
    case SL7_OK: return "SL7_OK";
    case SL7_EINVAL: return "SL7_EINVAL";
    case SL7_ESTATE: return "SL7_ESTATE";
    case SL7_EFORMAT: return "SL7_EFORMAT";
    case SL7_ENOMEM: return "SL7_ENOMEM";
    case SL7_ECUDA: return "SL7_ECUDA";
    case SL7_ENONFINITE: return "SL7_ENONFINITE";
    case SL7_EUNSUPPORTED: return "SL7_EUNSUPPORTED";
  }
  return "SL7_?";
}

const char* sl7_last_error(sl7_ctx ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

size_t sl7_out_elems(int32_t n_steps, uint64_t n_paths, sl7_out mode) {
  if (mode == SL7_OUT_FULL) return (size_t)(n_steps + 1) * (size_t)n_paths;
  if (mode == SL7_OUT_TERMINAL) return (size_t)n_paths;
  return 0;
}

size_t sl7_stats_elems(int32_t n_bins) { return (size_t)kStatsHead + (size_t)(n_bins > 0 ? n_bins : 0) + 2; }

sl7_status sl7_gh_grid(int32_t m, double* x, double* w) {
  if (m < 1 || m > kMaxM) return fail(nullptr, SL7_EINVAL, "m must be in 1..%d", kMaxM);
  if (!x || !w) return fail(nullptr, SL7_EINVAL, "x/w NULL");
  gh_grid(m, x, w);
  return SL7_OK;
}

sl7_status sl7_create(int32_t m, const int32_t* layer_dims, int32_t n_dims, sl7_act act, int32_t device, sl7_ctx* out) {
  if (!out) return fail(nullptr, SL7_EINVAL, "out is NULL");
  *out = nullptr;
  if (m < 1 || m > kMaxM) return fail(nullptr, SL7_EINVAL, "m must be in 1..%d", kMaxM);
  if (act != SL7_ACT_TANH && act != SL7_ACT_SOFTPLUS) return fail(nullptr, SL7_EINVAL, "act");
  if (n_dims != 0) {
    if (!layer_dims) return fail(nullptr, SL7_EINVAL, "layer_dims is NULL");
    const int L = n_dims - 2;
    if (L < 1 || L > kMaxHidden) return fail(nullptr, SL7_EINVAL, "layer_dims: 1..%d hidden layers", kMaxHidden);
    if (layer_dims[n_dims - 1] != m) return fail(nullptr, SL7_EINVAL, "layer_dims: last entry must equal m");
    if (layer_dims[0] < 2 || layer_dims[0] > 2 + SL7_MAX_THETA) return fail(nullptr, SL7_EINVAL, "layer_dims: d_in = 2 + n_theta");
    for (int l = 1; l <= L; ++l)
      if (layer_dims[l] < 1 || layer_dims[l] > kMaxW) return fail(nullptr, SL7_EINVAL, "layer_dims: hidden width 1..%d", kMaxW);
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(nullptr, SL7_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(nullptr, SL7_EINVAL, "device %d out of range", device);
  sl7_ctx c = new (std::nothrow) sl7_ctx_s();
  if (!c) return fail(nullptr, SL7_ENOMEM, "context allocation");
  c->device = device;
  c->m = m;
  c->act = (int)act;
  for (int i = 0; i < n_dims; ++i) c->dims.push_back(layer_dims[i]);
  gh_grid(m, c->x, c->w);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    c->num_sms = prop.multiProcessorCount;
    if (prop.major != 10) {
      delete c;
      return fail(nullptr, SL7_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major, prop.minor);
    }
  }
  *out = c;
  return SL7_OK;
}

sl7_status sl7_load_weights(sl7_ctx c, const void* blob, size_t nbytes) {
  if (!c) return fail(nullptr, SL7_EINVAL, "ctx is NULL");
  if (c->dims.empty()) return fail(c, SL7_ESTATE, "context created without layer_dims");
  if (!blob) return fail(c, SL7_EINVAL, "blob is NULL");
  const unsigned char* p = static_cast<const unsigned char*>(blob);
  size_t off = 0;
  auto need = [&](size_t k) { return off + k <= nbytes; };
  if (!need(12) || std::memcmp(p, "SL7W", 4) != 0) return fail(c, SL7_EFORMAT, "magic");
  if (rd_u32(p + 4) != 1) return fail(c, SL7_EFORMAT, "version");
  const uint32_t nd = rd_u32(p + 8);
  off = 12;
  if (nd != c->dims.size() || !need(4 * (size_t)nd + 8)) return fail(c, SL7_EFORMAT, "layer_dims (n_dims)");
  for (uint32_t i = 0; i < nd; ++i)
    if ((int)rd_u32(p + off + 4 * i) != c->dims[i]) return fail(c, SL7_EFORMAT, "layer_dims[%u]", i);
  off += 4 * (size_t)nd;
  if ((int)rd_u32(p + off) != c->act) return fail(c, SL7_EFORMAT, "act");
  const uint32_t flags = rd_u32(p + off + 4);
  off += 8;
  std::vector<std::vector<float>> W, b;
  for (uint32_t l = 0; l + 1 < nd; ++l) {
    const size_t fi = c->dims[l], fo = c->dims[l + 1];
    if (!need(4 * (fo * fi + fo))) return fail(c, SL7_EFORMAT, "size (layer %u)", l);
    W.emplace_back(fo * fi);
    std::memcpy(W.back().data(), p + off, 4 * fo * fi);
    off += 4 * fo * fi;
    b.emplace_back(fo);
    std::memcpy(b.back().data(), p + off, 4 * fo);
    off += 4 * fo;
  }
  if (flags & ~7u) return fail(c, SL7_EFORMAT, "flags (bit0 has_norm, bit1 residual, bit2 has_domain)");
  const bool has_norm = flags & 1u;
  std::vector<float> ish, isc, osh, osc, dlo, dhi;
  if (has_norm) {
    const size_t d_in = c->dims[0], m = c->m;
    if (!need(4 * (2 * d_in + 2 * m))) return fail(c, SL7_EFORMAT, "size (normalisation)");
    auto take = [&](std::vector<float>& v, size_t n) {
      v.resize(n);
      std::memcpy(v.data(), p + off, 4 * n);
      off += 4 * n;
    };
    take(ish, d_in);
    take(isc, d_in);
    take(osh, m);
    take(osc, m);
    for (float s : isc)
      if (!(s != 0.0f) || !std::isfinite(s)) return fail(c, SL7_EFORMAT, "in_scale");
  }
  if (flags & 4u) {
    const size_t d_in = c->dims[0];
    if (!need(8 * d_in)) return fail(c, SL7_EFORMAT, "size (domain)");
    dlo.resize(d_in);
    dhi.resize(d_in);
    std::memcpy(dlo.data(), p + off, 4 * d_in);
    std::memcpy(dhi.data(), p + off + 4 * d_in, 4 * d_in);
    off += 8 * d_in;
    for (size_t k = 0; k < d_in; ++k)
      if (!(dlo[k] <= dhi[k])) return fail(c, SL7_EFORMAT, "domain[%zu]: lo > hi or not a number", k);
  }
  if (off != nbytes) return fail(c, SL7_EFORMAT, "size (%zu bytes, expected %zu)", nbytes, off);
  for (auto& v : W)
    for (float x : v)
      if (!std::isfinite(x)) return fail(c, SL7_EFORMAT, "non-finite weight");
  c->W = std::move(W);
  c->b = std::move(b);
  c->has_norm = has_norm;
  c->residual = (flags & 2u) != 0;
  c->in_shift = ish;
  c->in_scale = isc;
  c->out_shift = osh;
  c->out_scale = osc;
  c->dom_lo = dlo;
  c->dom_hi = dhi;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  sl7_status s = build_f32_image(c);
  if (s != SL7_OK) return s;
  s = build_tc_image(c);
  if (s != SL7_OK) return s;
  c->has_net = true;
  return SL7_OK;
}

// SL7_SCHEME_CDC_PRED: the predictor's constants at each horizon t_i = i dt (reading R-26), folded by the
// same code as the run's own (prepare with dt -> t_i); step 0 needs none (every path at Y0).  Every entry
// point that can run the scheme (sl7_simulate, sl7_simulate_host, sl7_simulate_host_async) calls this after
// its own prepare(), so run() always sees the horizons of the current call.  No-op for other schemes.
static sl7_status prepare_cdc_horizons(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta,
                                int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                                const sl7_run_opts* opts, bool has_out, bool has_stats) {
  if (opts->scheme != SL7_SCHEME_CDC_PRED) return SL7_OK;
  if (opts->colloc == SL7_COLLOC_ANN && !c->dom_hi.empty()) {
    // the predictor is read at (Y0, t_i) for t_i up to (n_steps - 1) dt: outside the fitted box it extrapolates
    const double t_max = dt * (double)(n_steps - 1), tol = 1e-6;
    if (n_steps > 1 && (t_max > (double)c->dom_hi[1] * (1.0 + tol) || dt < (double)c->dom_lo[1] * (1.0 - tol)))
      return fail(c, SL7_EINVAL, "CDC_PRED horizons [%g, %g] leave the network's fitted dt range [%g, %g]", dt, t_max,
                  (double)c->dom_lo[1], (double)c->dom_hi[1]);
    if (Y0 < (double)c->dom_lo[0] || Y0 > (double)c->dom_hi[0])
      return fail(c, SL7_EINVAL, "CDC_PRED: Y0 = %g outside the network's fitted range [%g, %g]", Y0,
                  (double)c->dom_lo[0], (double)c->dom_hi[0]);
  }
  c->cdc_hz.assign((size_t)n_steps, CdcHorizon{});
  for (int32_t i = 1; i < n_steps; ++i) {
    RunParams q;
    sl7_status s = prepare(c, Y0, dt * (double)i, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, q, has_out,
                           has_stats);
    if (s != SL7_OK) return s;
    CdcHorizon& h = c->cdc_hz[(size_t)i];
    std::memcpy(h.l1b, q.l1b, sizeof h.l1b);
    std::memcpy(h.osc, q.out_scale, sizeof h.osc);
    std::memcpy(h.osh, q.out_shift, sizeof h.osh);
    std::memcpy(h.c, q.c, sizeof h.c);
    h.ou_a = q.ou_a;
    h.ou_b = q.ou_b;
  }
  return SL7_OK;
}

sl7_status sl7_simulate(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta, int32_t n_theta,
                        uint64_t n_paths, uint64_t seed, sl7_out out_mode, const sl7_run_opts* opts, float* d_out,
                        double* d_stats) {
  RunParams p;
  sl7_status s = prepare(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, p, d_out != nullptr,
                         d_stats != nullptr);
  if (s != SL7_OK) return s;
  s = prepare_cdc_horizons(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, d_out != nullptr,
                           d_stats != nullptr);
  if (s != SL7_OK) return s;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  return run(c, p, opts, out_mode == SL7_OUT_STATS ? nullptr : d_out, d_stats);
}

sl7_status sl7_simulate_em(sl7_ctx c, sl7_model model, double Y0, double dt, int32_t n_steps, int32_t substeps,
                           const double* theta, int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                           const sl7_run_opts* opts, float* d_out, double* d_stats) {
  RunParams p;
  sl7_status s = prepare_em(c, (int)model, Y0, dt, n_steps, substeps, theta, n_theta, n_paths, seed, out_mode, opts, p,
                            d_out != nullptr, d_stats != nullptr);
  if (s != SL7_OK) return s;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  return run(c, p, opts, out_mode == SL7_OUT_STATS ? nullptr : d_out, d_stats);
}

sl7_status sl7_training_set(sl7_ctx c, sl7_model model, const double* F, uint64_t n_rows, uint32_t M, double dtau,
                            uint64_t seed, const sl7_run_opts* o, float* d_term, double* d_labels) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!o) return fail(c, SL7_EINVAL, "opts is NULL");
  if (model != SL7_MODEL_GBM && model != SL7_MODEL_OU && model != SL7_MODEL_CIR) return fail(c, SL7_EINVAL, "model");
  if (!F) return fail(c, SL7_EINVAL, "h_features is NULL");
  if (n_rows < 1) return fail(c, SL7_EINVAL, "n_rows must be >= 1");
  if (M < (uint32_t)c->m) return fail(c, SL7_EINVAL, "n_inner must be >= m");
  if (!(dtau > 0.0) || !std::isfinite(dtau)) return fail(c, SL7_EINVAL, "dtau must be finite and > 0");
  if (!d_labels) return fail(c, SL7_EINVAL, "d_labels is NULL");
  if (o->flags & ~SL7_FLAG_FAST_NORMALS) return fail(c, SL7_EINVAL, "flags (SL7_FLAG_FAST_NORMALS only)");
  if (n_rows > UINT64_MAX / M || o->path_offset + (n_rows * M - 1) < o->path_offset)
    return fail(c, SL7_EINVAL, "path_offset + n_rows * n_inner - 1 overflows 2^64");
  const int nt = (model == SL7_MODEL_GBM) ? 2 : 3, nf = 2 + nt;
  std::vector<EmRow> rows(n_rows);
  for (uint64_t r = 0; r < n_rows; ++r) {
    const double* f = F + r * nf;
    if (!std::isfinite(f[0])) return fail(c, SL7_EINVAL, "features[%llu]: y_start must be finite", (unsigned long long)r);
    if (!(f[1] > 0.0) || !std::isfinite(f[1])) return fail(c, SL7_EINVAL, "features[%llu]: dt must be finite and > 0", (unsigned long long)r);
    const double K = std::max(1.0, std::ceil(f[1] / dtau));
    if (K > 2147483648.0) return fail(c, SL7_EINVAL, "features[%llu]: ceil(dt / dtau) > 2^31", (unsigned long long)r);
    EmRow& er = rows[r];
    sl7_status st = em_constants(c, (int)model, f + 2, nt, f[1] / K, er.a, er.s, er.ybar);
    if (st != SL7_OK) return fail(c, st, "features[%llu]: %s", (unsigned long long)r, c->err.c_str());
    er.y0 = (float)f[0];
    er.K = (int32_t)K;
  }
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  RunParams p;
  std::memset(&p, 0, sizeof p);
  p.key0 = (uint32_t)seed;
  p.key1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.rk0[r] = p.key0 + (uint32_t)r * 0x9E3779B9u;
    p.rk1[r] = p.key1 + (uint32_t)r * 0xBB67AE85u;
  }
  p.path_offset = o->path_offset;
  p.em_model = (int)model;
  p.flags = o->flags;
  CdcLevels lv;
  for (int k = 0; k < kMaxM; ++k) lv.p[k] = (k < c->m) ? 0.5 * std::erfc(-c->x[k] / std::sqrt(2.0)) : 0.0;
  // rows per chunk: all of them into d_terminal, else a 1 GiB scratch; at most 2^31 - 1 blocks per launch
  const uint64_t tpr = (M + 255u) / 256u;
  uint64_t chunk = d_term ? n_rows : std::max<uint64_t>(1, std::min<uint64_t>(n_rows, (256ull << 20) / M));
  chunk = std::min<uint64_t>(chunk, 0x7FFFFFFFull / tpr);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(o->stream);
  cudaError_t e;
  if (c->rows_cap < chunk) {
    if (c->d_rows) cudaFree(c->d_rows);
    c->d_rows = nullptr;
    c->rows_cap = 0;
    e = cudaMalloc(&c->d_rows, chunk * sizeof(EmRow));
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(feature rows)");
    c->rows_cap = chunk;
  }
  if (!d_term && c->term_cap < chunk * M) {
    if (c->d_term_scratch) cudaFree(c->d_term_scratch);
    c->d_term_scratch = nullptr;
    c->term_cap = 0;
    e = cudaMalloc(&c->d_term_scratch, chunk * M * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(terminal scratch)");
    c->term_cap = chunk * M;
  }
  std::vector<EmRow> part;
  for (uint64_t start = 0; start < n_rows; start += chunk) {
    const uint64_t nr = std::min(chunk, n_rows - start);
    part.assign(rows.begin() + start, rows.begin() + start + nr);
    for (uint64_t r = 0; r < nr; ++r) part[r].row = (uint32_t)r;
    // longest rows first: the block scheduler then fills the tail with short rows
    std::stable_sort(part.begin(), part.end(), [](const EmRow& a, const EmRow& b) { return a.K > b.K; });
    e = cudaMemcpyAsync(c->d_rows, part.data(), nr * sizeof(EmRow), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D feature rows");
    float* term = d_term ? d_term + start * M : c->d_term_scratch;
    int k = launch_em_rows(p, c->d_rows, (uint32_t)nr, M, start, term, o->stream);
    if (k) return cuda_fail(c, (cudaError_t)k, "training-set EM kernel");
    k = launch_row_quantiles(term, (uint32_t)nr, M, c->m, lv, d_labels + start * c->m, o->stream);
    if (k) return cuda_fail(c, (cudaError_t)k, "training-set quantile kernel");
  }
  return SL7_OK;
}

size_t sl7_cdc_hist_elems(void) { return (size_t)2 * kMaxM * 256; }

sl7_status sl7_cdc_init(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta, int32_t n_theta,
                        uint64_t n_paths, uint64_t seed, const sl7_run_opts* opts, float* d_state) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!opts) return fail(c, SL7_EINVAL, "opts is NULL");
  if (!d_state) return fail(c, SL7_EINVAL, "d_state is NULL");
  c->cdc_ready = false;
  sl7_run_opts o = *opts;
  o.scheme = SL7_SCHEME_CDC;
  RunParams p;
  sl7_status s = prepare(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, SL7_OUT_STATS, &o, p, false, true);
  if (s != SL7_OK) return s;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  if (!c->d_cdc) {
    cudaError_t ce = cudaMalloc(&c->d_cdc, cdc_scratch_bytes());
    if (ce != cudaSuccess) return cuda_fail(c, ce, "cudaMalloc(cdc scratch)");
  }
  int e = cdc_init_scratch(c->d_cdc, o.stream);
  if (e) return cuda_fail(c, (cudaError_t)e, "cdc scratch init");
  e = cdc_fill(d_state, n_paths, p.y0, o.stream, c->num_sms);
  if (e) return cuda_fail(c, (cudaError_t)e, "cdc state init");
  for (int k = 0; k < kMaxM; ++k) c->cdc_lv.p[k] = (k < c->m) ? 0.5 * std::erfc(-c->x[k] / std::sqrt(2.0)) : 0.0;
  p.out_mode = kStatsOnly;
  c->cdc_p = p;
  c->cdc_stream = o.stream;
  c->cdc_ready = true;
  return SL7_OK;
}

sl7_status sl7_cdc_hist(sl7_ctx c, const float* d_state, int32_t pass, uint64_t* d_hist) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!c->cdc_ready) return fail(c, SL7_ESTATE, "sl7_cdc_hist before sl7_cdc_init");
  if (!d_state || !d_hist) return fail(c, SL7_EINVAL, "d_state/d_hist is NULL");
  if (pass < 0 || pass > 3) return fail(c, SL7_EINVAL, "pass must be 0..3");
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  const int e = cdc_hist(c->cdc_p, c->d_cdc, d_state, pass, reinterpret_cast<unsigned long long*>(d_hist), true,
                         c->cdc_stream, c->num_sms);
  return e ? cuda_fail(c, (cudaError_t)e, "cdc histogram") : SL7_OK;
}

sl7_status sl7_cdc_select(sl7_ctx c, int32_t pass, const uint64_t* d_hist) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!c->cdc_ready) return fail(c, SL7_ESTATE, "sl7_cdc_select before sl7_cdc_init");
  if (!d_hist) return fail(c, SL7_EINVAL, "d_hist is NULL");
  if (pass < 0 || pass > 3) return fail(c, SL7_EINVAL, "pass must be 0..3");
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  const int e = cdc_select(c->cdc_p, c->cdc_lv, c->d_cdc, pass,
                           const_cast<unsigned long long*>(reinterpret_cast<const unsigned long long*>(d_hist)), false,
                           c->cdc_stream);
  return e ? cuda_fail(c, (cudaError_t)e, "cdc select") : SL7_OK;
}

sl7_status sl7_cdc_step(sl7_ctx c, int32_t step, const float* d_in, float* d_out, double* d_stats) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!c->cdc_ready) return fail(c, SL7_ESTATE, "sl7_cdc_step before sl7_cdc_init");
  if (!d_in || !d_out) return fail(c, SL7_EINVAL, "d_in/d_out is NULL");
  if (step < 0 || step >= c->cdc_p.n_steps) return fail(c, SL7_EINVAL, "step must be in 0..n_steps-1");
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  RunParams p = c->cdc_p;
  p.stats = d_stats;
  p.has_stats = d_stats ? 1 : 0;
  const int e = cdc_advance(p, c->d_cdc, d_in, d_out, step, d_stats != nullptr, c->cdc_stream,
                            c->num_sms);
  return e ? cuda_fail(c, (cudaError_t)e, "cdc step") : SL7_OK;
}

sl7_status sl7_simulate_host(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta, int32_t n_theta,
                             uint64_t n_paths, uint64_t seed, sl7_out out_mode, const sl7_run_opts* opts, float* h_out,
                             double* h_stats, uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  RunParams p;
  sl7_status s = prepare(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, p, h_out != nullptr,
                         h_stats != nullptr);
  if (s != SL7_OK) return s;
  s = prepare_cdc_horizons(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, h_out != nullptr,
                           h_stats != nullptr);
  if (s != SL7_OK) return s;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(opts->stream);
  const size_t n_out = sl7_out_elems(n_steps, n_paths, out_mode);
  const size_t n_st = h_stats ? sl7_stats_elems(opts->n_bins) : 0;
  cudaError_t e;
  if (n_out > c->out_cap) {
    if (c->d_out_scratch) cudaFree(c->d_out_scratch);
    c->d_out_scratch = nullptr;
    c->out_cap = 0;
    e = cudaMalloc(&c->d_out_scratch, n_out * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(out scratch)");
    c->out_cap = n_out;
  }
  if (n_st > c->stats_cap) {
    if (c->d_stats_scratch) cudaFree(c->d_stats_scratch);
    c->d_stats_scratch = nullptr;
    c->stats_cap = 0;
    e = cudaMalloc(&c->d_stats_scratch, n_st * sizeof(double));
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(stats scratch)");
    c->stats_cap = n_st;
  }
  uint64_t up = 0, down = 0;
  sl7_run_opts o = *opts;
  if (h_stats && opts->accumulate) {
    e = cudaMemcpyAsync(c->d_stats_scratch, h_stats, n_st * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D stats");
    up += n_st * sizeof(double);
  }
  s = run(c, p, &o, n_out ? c->d_out_scratch : nullptr, h_stats ? c->d_stats_scratch : nullptr);
  if (s != SL7_OK) return s;
  if (n_out) {
    e = cudaMemcpyAsync(h_out, c->d_out_scratch, n_out * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H out");
    down += n_out * sizeof(float);
  }
  if (n_st) {
    e = cudaMemcpyAsync(h_stats, c->d_stats_scratch, n_st * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H stats");
    down += n_st * sizeof(double);
  }
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(c, e, "stream synchronize");
  // kernel parameters (RunParams) travel host->device with the launch
  up += sizeof(RunParams);
  if (h2d_bytes) *h2d_bytes = up;
  if (d2h_bytes) *d2h_bytes = down;
  return SL7_OK;
}

sl7_status sl7_simulate_host_async(sl7_ctx c, double Y0, double dt, int32_t n_steps, const double* theta,
                                   int32_t n_theta, uint64_t n_paths, uint64_t seed, sl7_out out_mode,
                                   const sl7_run_opts* opts, float* h_out, double* h_stats, uint64_t* h2d_bytes,
                                   uint64_t* d2h_bytes) {
  RunParams p;
  sl7_status s = prepare(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, p, h_out != nullptr,
                         h_stats != nullptr);
  if (s != SL7_OK) return s;
  s = prepare_cdc_horizons(c, Y0, dt, n_steps, theta, n_theta, n_paths, seed, out_mode, opts, h_out != nullptr,
                           h_stats != nullptr);
  if (s != SL7_OK) return s;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(opts->stream);
  cudaError_t e;
  if (!c->copy_stream) {
    e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(c, e, "copy stream");
    e = cudaEventCreateWithFlags(&c->computed, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(c, e, "event");
    for (auto& sg : c->stage) {
      e = cudaEventCreateWithFlags(&sg.copied, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(c, e, "event");
    }
  }
  auto& sg = c->stage[c->next_stage];
  const size_t n_out = sl7_out_elems(n_steps, n_paths, out_mode);
  const size_t n_st = h_stats ? sl7_stats_elems(opts->n_bins) : 0;
  // this slot's previous D2H must be done before its buffers are rewritten (and before reallocation)
  if (sg.used) {
    e = cudaStreamWaitEvent(st, sg.copied, 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "wait for staging slot");
  }
  if (n_out > sg.out_cap || n_st > sg.stats_cap) {
    if (sg.used) {
      e = cudaEventSynchronize(sg.copied);
      if (e != cudaSuccess) return cuda_fail(c, e, "staging slot");
    }
    if (n_out > sg.out_cap) {
      if (sg.d_out) cudaFree(sg.d_out);
      sg.d_out = nullptr;
      sg.out_cap = 0;
      e = cudaMalloc(&sg.d_out, n_out * sizeof(float));
      if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(staging out)");
      sg.out_cap = n_out;
    }
    if (n_st > sg.stats_cap) {
      if (sg.d_stats) cudaFree(sg.d_stats);
      sg.d_stats = nullptr;
      sg.stats_cap = 0;
      e = cudaMalloc(&sg.d_stats, n_st * sizeof(double));
      if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc(staging stats)");
      sg.stats_cap = n_st;
    }
  }
  uint64_t up = 0, down = 0;
  sl7_run_opts o = *opts;
  if (h_stats && opts->accumulate) {
    e = cudaMemcpyAsync(sg.d_stats, h_stats, n_st * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D stats");
    up += n_st * sizeof(double);
  }
  s = run(c, p, &o, n_out ? sg.d_out : nullptr, h_stats ? sg.d_stats : nullptr);
  if (s != SL7_OK) return s;
  // results leave on the copy stream, so the next call's kernels (on opts->stream) overlap this D2H
  e = cudaEventRecord(c->computed, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->copy_stream, c->computed, 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "copy ordering");
  if (n_out) {
    e = cudaMemcpyAsync(h_out, sg.d_out, n_out * sizeof(float), cudaMemcpyDeviceToHost, c->copy_stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H out");
    down += n_out * sizeof(float);
  }
  if (n_st) {
    e = cudaMemcpyAsync(h_stats, sg.d_stats, n_st * sizeof(double), cudaMemcpyDeviceToHost, c->copy_stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H stats");
    down += n_st * sizeof(double);
  }
  e = cudaEventRecord(sg.copied, c->copy_stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "event record");
  sg.used = true;
  c->next_stage ^= 1;
  up += sizeof(RunParams);
  if (h2d_bytes) *h2d_bytes = up;
  if (d2h_bytes) *d2h_bytes = down;
  return SL7_OK;
}

sl7_status sl7_sync(sl7_ctx c) {
  if (!c) return fail(c, SL7_EINVAL, "ctx is NULL");
  if (!c->copy_stream) return SL7_OK;
  DeviceGuard g(c->device);
  if (!g.ok) return fail(c, SL7_ECUDA, "cudaSetDevice(%d)", c->device);
  const cudaError_t e = cudaStreamSynchronize(c->copy_stream);
  return e == cudaSuccess ? SL7_OK : cuda_fail(c, e, "sl7_sync");
}

sl7_status sl7_stats(const double* v, const sl7_run_opts* o, sl7_summary* out) {
  if (!v || !o || !out) return fail(nullptr, SL7_EINVAL, "NULL argument");
  if (o->n_bins < 0 || o->n_bins > 16384) return fail(nullptr, SL7_EINVAL, "n_bins");
  if (out->n_q > 0 && (!out->q_levels || !out->q_values)) return fail(nullptr, SL7_EINVAL, "q_levels/q_values");
  const double n = v[0];
  out->n = (uint64_t)n;
  out->n_nonfinite = (uint64_t)v[1];
  if (!(n > 0)) return fail(nullptr, SL7_EINVAL, "no finite terminal values (n == 0)");
  const double a1 = v[2] / n, a2 = v[3] / n, a3 = v[4] / n, a4 = v[5] / n;
  const double var = a2 - a1 * a1;
  const double m3 = a3 - 3 * a1 * a2 + 2 * a1 * a1 * a1;
  const double m4 = a4 - 4 * a1 * a3 + 6 * a1 * a1 * a2 - 3 * a1 * a1 * a1 * a1;
  out->mean = o->shift + a1;
  out->var = var;
  out->skew = var > 0 ? m3 / std::pow(var, 1.5) : 0.0;
  out->exkurt = var > 0 ? m4 / (var * var) - 3.0 : 0.0;
  out->strong_err = v[6] / n;
  out->rms_err = std::sqrt(v[7] / n);
  // quantiles from the histogram CDF, plotting position (k - 0.5)/M, uniform spread inside a bin
  const int B = o->n_bins;
  for (int q = 0; q < out->n_q; ++q) {
    double res = std::nan("");
    const double lev = out->q_levels[q];
    if (B > 0 && lev > 0.0 && lev < 1.0) {
      const double target = lev * n + 0.5 - 0.5;   // counts strictly below the quantile point
      const double w = (o->hist_hi - o->hist_lo) / B;
      double cum = v[kStatsHead];                   // underflow
      if (target >= cum) {
        for (int k = 0; k < B; ++k) {
          const double ck = v[kStatsHead + 1 + k];
          if (target < cum + ck || (k == B - 1 && target <= cum + ck)) {
            const double frac = ck > 0 ? (target - cum) / ck : 0.0;
            res = o->hist_lo + (k + frac) * w;
            break;
          }
          cum += ck;
        }
      }
    }
    out->q_values[q] = res;
  }
  if (out->n_nonfinite > 0) return fail(nullptr, SL7_ENONFINITE, "%llu non-finite terminal values", (unsigned long long)out->n_nonfinite);
  return SL7_OK;
}

sl7_status sl7_philox_u32(uint64_t seed, uint64_t off, uint64_t n, uint32_t block, uint32_t* d_out, void* stream) {
  if (!d_out || n == 0) return fail(nullptr, SL7_EINVAL, "d_out/n_paths");
  if (off + (n - 1) < off) return fail(nullptr, SL7_EINVAL, "path_offset + n_paths - 1 overflows 2^64");
  const int e = launch_philox_u32(seed, off, n, block, d_out, stream);
  return e ? cuda_fail(nullptr, (cudaError_t)e, "philox kernel") : SL7_OK;
}

sl7_status sl7_normals(uint64_t seed, uint64_t off, uint64_t n, int32_t n_steps, uint32_t flags, float* d_out,
                       void* stream) {
  if (!d_out || n == 0 || n_steps < 1) return fail(nullptr, SL7_EINVAL, "d_out/n_paths/n_steps");
  if (off + (n - 1) < off) return fail(nullptr, SL7_EINVAL, "path_offset + n_paths - 1 overflows 2^64");
  if (flags & ~SL7_FLAG_FAST_NORMALS) return fail(nullptr, SL7_EINVAL, "flags");
  const int e = launch_normals(seed, off, n, n_steps, (flags & SL7_FLAG_FAST_NORMALS) != 0, d_out, stream);
  return e ? cuda_fail(nullptr, (cudaError_t)e, "normals kernel") : SL7_OK;
}

void sl7_destroy(sl7_ctx c) {
  if (!c) return;
  int dev = -1;
  if (cudaGetDevice(&dev) == cudaErrorCudartUnloading) {   // process exit: the runtime is gone, so is the memory
    delete c;
    return;
  }
  {
    DeviceGuard g(c->device);
    if (c->d_wf32) cudaFree(c->d_wf32);
    if (c->d_wtc) cudaFree(c->d_wtc);
    if (c->d_wtc_split) cudaFree(c->d_wtc_split);
    if (c->d_wtc_tf32) cudaFree(c->d_wtc_tf32);
    if (c->d_cdc) cudaFree(c->d_cdc);
    if (c->d_cdc_tabs) cudaFree(c->d_cdc_tabs);
    if (c->d_state) cudaFree(c->d_state);
    if (c->d_out_scratch) cudaFree(c->d_out_scratch);
    if (c->d_stats_scratch) cudaFree(c->d_stats_scratch);
    if (c->d_rows) cudaFree(c->d_rows);
    if (c->d_term_scratch) cudaFree(c->d_term_scratch);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    for (auto& sg : c->stage) {
      if (sg.d_out) cudaFree(sg.d_out);
      if (sg.d_stats) cudaFree(sg.d_stats);
      if (sg.copied) cudaEventDestroy(sg.copied);
    }
    if (c->computed) cudaEventDestroy(c->computed);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  }
  delete c;
}

}  // extern "C"
