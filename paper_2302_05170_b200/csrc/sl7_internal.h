// sl7_internal.h -- structures shared by the host runtime (sl7_host.cpp) and the sm_100a kernels.
// Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/sl7.h"

namespace sl7 {

constexpr int kMaxM = SL7_MAX_M;
constexpr int kMaxW = SL7_MAX_WIDTH;
constexpr int kMaxHidden = SL7_MAX_HIDDEN;
constexpr int kStatsHead = SL7_STATS_HEAD;

enum Colloc : int { kAnn = 0, kExactGbm = 1, kExactOu = 2, kExactCir = 3 };
enum Ref : int { kRefNone = 0, kRefGbm = 1, kRefOu = 2 };
enum OutMode : int { kFull = 0, kTerminal = 1, kStatsOnly = 2 };

// Everything one launch of a step kernel needs, passed by value as a __grid_constant__ parameter
// (kernel parameters live in the constant bank: uniform, broadcast, no global loads).
struct RunParams {
  // ---- problem ----
  int m;                 // nodes
  int n_steps;
  int out_mode;          // OutMode
  int colloc;            // Colloc
  uint64_t n_paths;
  uint64_t path_offset;  // global id of path 0 of this launch
  uint32_t key0, key1;   // Philox key = (seed_lo, seed_hi)
  uint32_t rk0[10], rk1[10];   // Philox round keys key + r (W0, W1), r = 0..9
  float y0;
  // ---- interpolation grid (Algorithm I step 5): nodes split x = xhi + xlo, barycentric w ----
  float xhi[kMaxM], xlo[kMaxM], w[kMaxM];
  // ---- exact collocation: GBM y_j = Y*c[j]; OU y_j = ou_a*Y + ou_b + c[j] (c[j] = std*x_j) ----
  float c[kMaxM];
  float ou_a, ou_b;
  // ---- SL7_FLAG_SPECIALIZED: GBM g_m(Z) = Y * sum_k q[k] Z^k (monomial form, m <= 8);
  //      OU g_m(Z) = ou_a Y + ou_b + ou_s Z
  float q[8];
  float ou_s;
  uint32_t flags;
  // ---- exact CIR: Y' | Y = cir_c chi'^2(cir_d, Y+ cir_lscale); quantile levels cir_p[j] = Phi(cir_x[j])
  double cir_c, cir_d, cir_lscale;
  double cir_p[kMaxM], cir_x[kMaxM];
  // ---- strong-error reference on the same normals ----
  int ref;               // Ref
  double ref_drift_T;    // GBM: (mu - s^2/2) T
  double ref_vol;        // GBM: s sqrt(dt)
  double ref_a, ref_b, ref_s;   // OU: R <- a R + b + s Z
  double y0_d;
  // ---- statistics ----
  int has_stats;
  int n_bins;
  double shift, hist_lo, hist_scale;   // bin = floor((Y - lo) * scale)
  float* out;
  double* stats;
  // ---- ANN (layer 1 folded: pre_k = l1w[k] * Y + l1b[k]) ----
  int act;               // sl7_act
  int n_hidden;          // L
  int width;             // padded hidden width used by the kernel
  float l1w[kMaxW], l1b[kMaxW];
  double l1w_d[kMaxW], l1b_d[kMaxW];   // host-side double copies (not read by kernels)
  float out_scale[kMaxM], out_shift[kMaxM];   // residual blobs: already multiplied by sqrt(dt)
  float res_y;                               // 1 for residual blobs (y_j = Y + ...), else 0
  const float* wdev;     // FP32 kernel: hidden + output weights (layout: WeightLayoutF32)
  const void* wtc;       // TC kernel: packed bf16 operand images (layout: sl7_tc.cu)
  const float* btc;      // TC kernel: fp32 biases [(L-1)][64] + out bias [16]
  // ---- Euler-Maruyama (sl7_simulate_em): Y <- Y + a(Y) dtau + b(Y) sqrt(dtau) Z, K sub-steps per step
  int em_model;          // sl7_model
  int em_K;
  float em_a, em_s, em_ybar;   // GBM: a = mu dtau, s = sigma sqrt(dtau); OU / CIR: a = lam dtau, s, ybar
};

// One feature row of the training-set generator (sl7_training_set), constants as in RunParams.
struct EmRow {
  float y0, a, s, ybar;
  int32_t K;      // Euler sub-steps of dt / K
  uint32_t row;   // output row within the chunk
};

// FP32-kernel weight image: for hidden layer l = 1..L-1: W[H][HS] then b[H] padded to a multiple of 4
// floats (HS = row stride, multiple of 4; every row starts 16-byte aligned), then Wout[M][HS], bout[M].
// Zero padded.
#ifdef __CUDACC__
#define SL7_HD __host__ __device__
#else
#define SL7_HD
#endif
SL7_HD inline size_t f32_layer_floats(int H, int HS) { return (size_t)H * HS + (size_t)((H + 3) & ~3); }
SL7_HD inline size_t f32_weight_floats(int H, int HS, int L, int M) {
  return (size_t)(L - 1) * f32_layer_floats(H, HS) + (size_t)M * HS + (size_t)((M + 3) & ~3);
}

// Tensor-core (tcgen05) kernel extras: fp32 biases of the MMA layers and the bf16 operand image.
// Image: for each hidden->hidden layer a [64 n][64 k] bf16 tile (8 KB), then the output layer as a
// [16 n][64 k] tile (2 KB); each tile in the K-major SWIZZLE_128B layout (row n = 128 bytes, the 16-byte
// chunk c of row n stored at chunk c ^ (n % 8)), weights rounded to bf16 with round-to-nearest-even.
constexpr int kTcN = 64;       // hidden width on the tensor cores (zero padded)
constexpr int kTcNOut = 16;    // output width (m padded)
constexpr int kTcTileBytes = kTcN * kTcN * 2;
constexpr int kTcOutBytes = kTcNOut * kTcN * 2;
struct TcParams {
  float act_scale;                    // tanh: 2 log2(e) (argument of 2^u); softplus: 1
  float l1w[kTcN], l1b[kTcN];         // layer 1 folded and scaled by act_scale
  float bias[kMaxHidden - 1][kTcN];   // hidden biases scaled by act_scale
  float bout[kTcNOut];
  // accumulator scale of each hidden MMA layer (act_scale, times 2^-s_l for SL7_PREC_SPLIT whose weight
  // image is W 2^s_l) and of the output layer (1, or 2^-s_out)
  float lscale[kMaxHidden - 1];
  float oscale;
  int split_exp[kMaxHidden];   // SL7_PREC_SPLIT: s_l of the MMA layers (hidden 0..L-2, then the output)
  const void* wimg;
  const void* wimg_split;   // SL7_PREC_SPLIT: per tile the two fp16 parts of W 2^s = W0 + W1 in turn
  const void* wimg_tf32;    // SL7_PREC_TF32: tf32 (cvt.rna) tiles, two SWIZZLE_128B K-blocks [N][128 B] each
  int n_mma_hidden;   // L - 1
  int variant;        // activation variant (experiment hook, SL7_TC_VARIANT)
  int split;          // 1: SL7_PREC_SPLIT
  int tanh_mufu;      // tanh on MUFU.TANH (argument unscaled: act_scale = 1)
  int tf32;           // 1: SL7_PREC_TF32
};

// 7L-CDC: quantile levels Phi(x_k) of the marginal collocation points (host, double).
struct CdcLevels {
  double p[kMaxM];
};
// SL7_SCHEME_CDC_PRED: the horizon-dependent constants of the predictor at (Y0, t_i = i dt), folded on
// the host exactly as RunParams folds the run's dt (layer-1 bias, residual output scale; exact modes'
// c_j and OU coefficients).  One per step, passed by value to the table kernel.
struct CdcHorizon {
  float l1b[kMaxW];
  float osc[kMaxM], osh[kMaxM];
  float c[kMaxM];
  float ou_a, ou_b;
};
// tables: device buffer of n_steps * cdc_table_bytes() (the fused all-steps kernel, m = 5 or 7), or NULL
// for the per-step path (table kernel + step kernel per step, any m)
int launch_cdc_pred(const RunParams& p, const CdcHorizon* hz, void* scratch, float* const* rows, int nrows,
                    void* stream, int num_sms, void* tables);
size_t cdc_table_bytes();
constexpr int kCdcFusedMaxSteps = 160;   // 160 x 464 B of step tables + the histogram: 2 CTAs per SM
size_t cdc_scratch_bytes();
int cdc_init_scratch(void* scratch, void* stream);
// rows: nrows == 1 -> one in-place state buffer; nrows == n_steps + 1 -> FULL output rows.
int launch_cdc(const RunParams& p, const CdcLevels& lv, void* scratch, float* const* rows, int nrows, void* stream,
               int num_sms);
// the pieces of one CDC step, for runs whose paths are sharded over ranks (sl7_cdc_*): the caller sums the
// pass histograms ([2 SL7_MAX_M][256] u64) over ranks between cdc_hist and cdc_select.
int cdc_fill(float* y, uint64_t n, float v, void* stream, int num_sms);
int cdc_hist(const RunParams& p, void* scratch, const float* y, int pass, unsigned long long* hist, bool zero,
             void* stream, int num_sms);
int cdc_select(const RunParams& p, const CdcLevels& lv, void* scratch, int pass, unsigned long long* hist, bool clear,
               void* stream);
int cdc_advance(const RunParams& p, void* scratch, const float* yin, float* yout, int step, bool stats, void* stream,
                int num_sms, unsigned long long* next_hist = nullptr);

// launchers (sl7_kernels.cu / sl7_tc.cu); return cudaError_t as int
int launch_step_kernel(const RunParams& p, int prec, void* stream, int num_sms);
int launch_tc_kernel(const RunParams& p, const TcParams& t, void* stream, int num_sms);
int launch_philox_u32(uint64_t seed, uint64_t off, uint64_t n, uint32_t block, uint32_t* out, void* stream);
int launch_normals(uint64_t seed, uint64_t off, uint64_t n, int n_steps, bool fast, float* out, void* stream);
int launch_zero_stats(double* stats, size_t n, void* stream);
// sl7_cir.cu
int launch_exact_cir(const RunParams& p, void* stream, int num_sms);
// sl7_em.cu
int launch_em(const RunParams& p, void* stream, int num_sms);
int launch_em_rows(const RunParams& p, const EmRow* d_rows, uint32_t n_rows, uint32_t M, uint64_t row_base,
                   float* term, void* stream);
int launch_row_quantiles(const float* term, uint32_t n_rows, uint32_t M, int m, const CdcLevels& lv,
                         double* labels, void* stream);

}  // namespace sl7
