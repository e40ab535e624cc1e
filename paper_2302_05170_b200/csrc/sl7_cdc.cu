// sl7_cdc.cu -- the 7L-CDC variant on sm_100a.
//
// Per large step i (readings R-18..R-20):
//   1. marginal collocation points z_k = empirical quantiles of the current states of ALL paths at
//      the levels Phi(x_k) (plotting position (k - 0.5)/M, linear interpolation between order
//      statistics).  The 2m order statistics are found EXACTLY by a 4-pass radix select on the
//      order-preserving 32-bit key of the fp32 state (8 bits per pass): each pass histograms the next
//      digit of the elements whose higher digits match a target's prefix (shared-memory histograms,
//      one per distinct prefix), then one small kernel walks the histograms to fix each target's digit.
//   2. table C[k][.] = H(z_k): m predictor calls (exact closed forms, or the MLP in fp32);
//   3. per path: y_j = Lagrange interpolant of k -> C[k][j] on the nodes z_k at the path's own state
//      (normalised barycentric product form), then Y_{i+1} = g_m(X_hat) on the Gauss-Hermite grid.
// Repeated z_k (step 0: every path at Y0) fall back to the nearest row (ties: lowest k).
// The states live in HBM between steps (the quantiles couple all paths), so a CDC step is a short
// sequence of launches on the caller's stream; HBM traffic per path-step: 4 selection reads + 1 read
// + 1 write of 4 bytes.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "sl7_device.cuh"

namespace sl7 {

// Device-side scratch of the CDC pipeline (context-owned).
// kCdcBiv: tables of m <= kCdcBiv also carry the step as ONE bivariate polynomial (CdcTable::D below)
constexpr int kCdcBiv = 8;

struct CdcScratch {
  unsigned long long hist[kCdcMaxT][256];   // per-slot digit histograms of the current pass
  unsigned long long rank[kCdcMaxT];        // residual rank of each target within its prefix
  uint32_t prefix[kCdcMaxT];                // key bits fixed so far (in the high bits)
  int slot_of[kCdcMaxT];                    // target -> histogram slot
  uint32_t slot_prefix[kCdcMaxT];           // distinct prefixes, ascending
  int nslot;
  unsigned long long M;                     // number of finite states
  double frac[kMaxM];                       // interpolation weight of the upper order statistic
  // the table the step kernel consumes
  float z[kMaxM], zlo[kMaxM], v[kMaxM], C[kMaxM][kMaxM];   // z + zlo = the double marginal point
  float sinv;   // 1 / half-range of the z_k: the interpolation works on (Y - z_k) * sinv (no fp32 under/overflow)
  int degenerate;
  double zd[kMaxM];
  float D[kCdcBiv][kCdcBiv];   // the step as a bivariate polynomial, as CdcTable::D
  float shinv, sc;
};

// One step's CDC_PRED table (the fused kernel stages all steps' tables; same fields as CdcScratch's).
struct CdcTable {
  float z[kMaxM], zlo[kMaxM], v[kMaxM], C[kMaxM][kMaxM];
  float sinv;
  int degenerate;
  double zd[kMaxM];
  // Y' = sum_j l_j(X) sum_k L_k(Yb) C[k][j] (g_m of the table interpolated at the clamped state, R-19/R-26) is a
  // polynomial of degree m-1 in each of s = (Yb - c) / h (c, h: centre and half-width of the hull) and X:
  // Y' = sum_a sum_b D[a][b] s^a X^b with D = A^T C B, A / B the monomial coefficients of the Lagrange bases
  // on the s-nodes of the z_k and on the Gauss-Hermite nodes (built in double by the table kernel)
  float D[kCdcBiv][kCdcBiv];
  float shinv, sc;   // s = Yb * shinv + sc
};

// From the double marginal points s->zd[0..m): the fp32 hi/lo split, the scaled barycentric weights and
// the degenerate flag the step kernel reads (one thread).
template <class T>
__device__ void cdc_finalize_marginals(T* s, int m, int degen) {
  s->degenerate = degen;
  for (int k = 0; k < m; ++k) {
    s->z[k] = (float)s->zd[k];
    s->zlo[k] = (float)(s->zd[k] - (double)s->z[k]);
    // barycentric weights of the nodes scaled to O(1) spacing: the normalised formula is invariant to a
    // common scale of all (Y - z_k), and for m up to 16 nodes the unscaled products under/overflow fp32
    const double sc = (!degen && m > 1) ? 0.5 * (s->zd[m - 1] - s->zd[0]) : 1.0;
    double w = 1.0;
    if (!degen)
      for (int l = 0; l < m; ++l)
        if (l != k) w *= (s->zd[k] - s->zd[l]) / sc;
    s->v[k] = degen ? 0.0f : (float)(1.0 / w);
    if (k == 0) s->sinv = (float)(1.0 / sc);
  }
}

// ---- pass p: histogram of digit p (bits [24 - 8p, 32 - 8p)) of the elements matching a slot prefix.
// The states of one step are concentrated in a few digit bins, so the shared-memory increments are
// warp-aggregated (__match_any_sync: one atomic per distinct bin per warp) instead of one per element.
__device__ __forceinline__ void warp_hist_add(uint32_t* h, int bin) {   // bin < 0: nothing (all lanes call)
  if (!__any_sync(0xffffffffu, bin >= 0)) return;   // later passes: most warps hold no candidate at all
  const unsigned peers = __match_any_sync(0xffffffffu, bin);
  if (bin >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
}

// Slot lookup: the elements of a pass that count are those whose key prefix (the 8 p bits fixed so far)
// equals one of the <= 2m slot prefixes.  Instead of a per-element binary search (the targets span the
// 0.01%..99.99% quantiles, so nearly every element is inside the prefix range and searched), the block
// builds a table in shared memory: pass 1 indexes the 8-bit prefix directly; pass 2 the 16-bit prefix
// (64 KB of one-byte slot ids); pass 3 maps the top 16 bits to a group of slots and then the next 8 bits
// within that group.  Entries hold slot + 1 (0: no slot).
constexpr int kCdcLutBytes = 65536 + kCdcMaxT * 256;

// PASS is a template parameter: with a runtime pass the per-element code carried every pass's branches
// (and their divergence bookkeeping) for each element.
template <int U, int PASS>
__global__ void __launch_bounds__(256) cdc_hist_kernel(const float* __restrict__ y, uint64_t n,
                                                       const CdcScratch* s, unsigned long long* __restrict__ hist) {
  constexpr int pass = PASS;
  extern __shared__ uint4 lut4[];
  uint8_t* lut16 = reinterpret_cast<uint8_t*>(lut4);        // [65536] (pass 1 uses the first 256)
  uint8_t* lut3 = lut16 + 65536;                             // [groups][256] (pass 3)
  __shared__ uint32_t h[kCdcMaxT * 256];
  const int nslot = s->nslot;
  for (int i = threadIdx.x; i < nslot * 256; i += blockDim.x) h[i] = 0u;
  if constexpr (PASS > 0) {
    const int words = (pass == 1) ? 256 / 16 : kCdcLutBytes / 16;
    for (int i = threadIdx.x; i < words; i += blockDim.x) lut4[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (pass < 3) {
        for (int k = 0; k < nslot; ++k) lut16[s->slot_prefix[k]] = (uint8_t)(k + 1);   // 8- or 16-bit prefixes
      } else {
        int ng = 0;   // slot prefixes are ascending, so equal top-16 parts are adjacent
        uint32_t last = 0xFFFFFFFFu;
        for (int k = 0; k < nslot; ++k) {
          const uint32_t sp = s->slot_prefix[k];
          if ((sp >> 8) != last) {
            last = sp >> 8;
            lut16[last] = (uint8_t)(++ng);
          }
          lut3[(ng - 1) * 256 + (sp & 255u)] = (uint8_t)(k + 1);
        }
      }
    }
  }
  __syncthreads();
  const int shift = 24 - 8 * pass;
  const int lane = threadIdx.x & 31;
  // the bin of one element (-1: not counted in this pass)
  auto bin_of = [&](float x) -> int {
    if (!isfinite(x)) return -1;
    const uint32_t key = f2key(x);
    const int digit = (int)((key >> shift) & 255u);
    if constexpr (PASS == 0) return digit;
    int slot;
    if constexpr (PASS < 3) {
      slot = (int)lut16[key >> (shift + 8)] - 1;
    } else {
      const int g = (int)lut16[key >> 16];
      slot = g ? (int)lut3[(g - 1) * 256 + ((key >> 8) & 255u)] - 1 : -1;
    }
    return slot >= 0 ? slot * 256 + digit : -1;
  };
  auto count = [&](int bin) {   // all lanes of the warp call it (pass 0 aggregates per warp)
    if constexpr (PASS == 0) warp_hist_add(h, bin);
    else if (bin >= 0) atomicAdd(&h[bin], 1u);
  };
  if ((reinterpret_cast<uintptr_t>(y) & 15u) == 0) {
    // 16-byte loads: each thread takes U/4 float4 per chunk (a warp reads 512 contiguous bytes per load),
    // so the per-element index arithmetic and bounds checks are amortised over four elements
    constexpr int V = (U + 3) / 4;
    const float4* y4 = reinterpret_cast<const float4*>(y);
    const uint64_t n4 = n >> 2;
    const uint64_t wstride = (uint64_t)gridDim.x * blockDim.x * V;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * V; base < n4; base += wstride) {
      float4 v[V];
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const uint64_t q = base + 32 * u + lane;
        const float inf = __int_as_float(0x7F800000);   // +inf: skipped
        v[u] = (q < n4) ? y4[q] : make_float4(inf, inf, inf, inf);
      }
#pragma unroll
      for (int u = 0; u < V; ++u) {
        count(bin_of(v[u].x));
        count(bin_of(v[u].y));
        count(bin_of(v[u].z));
        count(bin_of(v[u].w));
      }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {   // the n % 4 tail, one warp (all lanes call count)
      const uint64_t q = (n4 << 2) + lane;
      count(q < n ? bin_of(y[q]) : -1);
    }
  } else {
    // each warp takes chunks of 32 U consecutive elements: U coalesced loads in flight per thread (the LUT
    // passes run at 2 blocks per SM, so they need the deeper chunks to keep HBM busy)
    const uint64_t wstride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * U; base < n; base += wstride) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t q = base + 32 * u + lane;
        v[u] = (q < n) ? y[q] : __int_as_float(0x7F800000);   // +inf: skipped below
      }
#pragma unroll
      for (int u = 0; u < U; ++u) count(bin_of(v[u]));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslot * 256; i += blockDim.x) {
    const uint32_t c = h[i];
    if (c) atomicAdd(&hist[i], (unsigned long long)c);
  }
}

// ---- after pass p: fix each target's digit; set up the next pass.  One block of 1024 threads: warp t
// finds target t's bin with a warp scan over the slot's 256 counts (lane l owns bins 8l..8l+7).
// hist: [slot][256] counts of this pass over ALL paths of the run (summed over ranks for a sharded run);
// clear: zero it afterwards (the single-call path reuses the scratch histogram).
__global__ void __launch_bounds__(1024) cdc_scan_kernel(int pass, int m, CdcScratch* s, const __grid_constant__ CdcLevels lv,
                                                        unsigned long long* hist, int clear) {
  const int T = 2 * m, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (pass == 0) {
    if (warp == 0) {
      unsigned long long M = 0;
      for (int b = lane; b < 256; b += 32) M += hist[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M += __shfl_xor_sync(0xffffffffu, M, o);
      if (lane == 0) s->M = M;
      if (lane < m) {
        // target order statistics (0-based) of the plotting-position quantile (as the oracle:
        // pos = p M + 0.5 clamped to [1, M], k = floor(pos), f = pos - k, ranks k - 1 and min(k, M - 1))
        double f = 0.0;
        unsigned long long r0 = 0ull, r1 = 0ull;   // no finite state: every target at rank 0 (z = NaN below)
        if (M > 0) {
          double pos = __dadd_rn(__dmul_rn(lv.p[lane], (double)M), 0.5);
          pos = fmin(fmax(pos, 1.0), (double)M);
          const double kk = floor(pos);
          f = pos - kk;
          r0 = (unsigned long long)kk - 1ull;
          r1 = ((unsigned long long)kk < M) ? (unsigned long long)kk : M - 1ull;
        }
        s->frac[lane] = f;
        s->rank[2 * lane] = r0;
        s->rank[2 * lane + 1] = r1;
        s->prefix[2 * lane] = s->prefix[2 * lane + 1] = 0u;
      }
    }
    __syncthreads();
  }
  if (warp < T && s->M > 0) {
    const int t = warp, sl = (pass == 0) ? 0 : s->slot_of[t];
    const unsigned long long r = s->rank[t];
    const unsigned long long* hs = hist + 256 * sl;
    unsigned long long c[8], sum = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      c[u] = hs[lane * 8 + u];
      sum += c[u];
    }
    unsigned long long inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long nb = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += nb;
    }
    const unsigned long long exc = inc - sum;
    if (r >= exc && r < inc) {
      unsigned long long below = exc;
      int b = lane * 8;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (below + c[u] > r) {
          b = lane * 8 + u;
          break;
        }
        below += c[u];
      }
      s->rank[t] = r - below;
      s->prefix[t] = (s->prefix[t] << 8) | (uint32_t)b;
    }
  } else if (warp < T && lane == 0) {
    s->prefix[warp] <<= 8;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pass < 3) {
      // distinct prefixes, ascending.  The targets are NOT always in rank order: levels clamped to the
      // extreme order statistics repeat the pair (0, 1) (or (M-2, M-1)), e.g. 0, 1, 0, 1, ...
      int ns = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t v = s->prefix[t];
        int a = 0;
        while (a < ns && s->slot_prefix[a] < v) ++a;
        if (a == ns || s->slot_prefix[a] != v) {
          for (int b = ns; b > a; --b) s->slot_prefix[b] = s->slot_prefix[b - 1];
          s->slot_prefix[a] = v;
          ++ns;
        }
      }
      for (int t = 0; t < T; ++t) {
        int a = 0;
        while (s->slot_prefix[a] != s->prefix[t]) ++a;
        s->slot_of[t] = a;
      }
      s->nslot = ns;
    } else {
      // full keys known: marginal points in double (as the oracle: y_lo (1 - f) + y_hi f)
      int degen = 0;
      for (int k = 0; k < m; ++k) {
        const double a = (double)key2f(s->prefix[2 * k]), b = (double)key2f(s->prefix[2 * k + 1]);
        const double f = s->frac[k];
        s->zd[k] = (s->M > 0) ? __dadd_rn(__dmul_rn(a, 1.0 - f), __dmul_rn(b, f))
                              : __longlong_as_double(0x7FF8000000000000ll);
        if (k > 0 && !(s->zd[k] > s->zd[k - 1])) degen = 1;   // repeated (or NaN) marginal points
      }
      cdc_finalize_marginals(s, m, degen);
    }
  }
  __syncthreads();
  // clear the histograms for the next pass
  if (clear)
    for (int i = threadIdx.x; i < kCdcMaxT * 256; i += blockDim.x) hist[i] = 0ull;
  if (pass == 3 && threadIdx.x == 0) {   // reset the selection for the next step
    s->nslot = 1;
    s->slot_prefix[0] = 0u;
  }
}

// Monomial coefficients of the Lagrange basis on n[0..m): A[k][a] = coefficient of t^a in
// prod_{k' != k} (t - n_k') / (n_k - n_k'), in double (one thread).
__device__ void lagrange_monomial(const double* n, int m, double (*A)[kCdcBiv]) {
  for (int k = 0; k < m; ++k) {
    double q[kCdcBiv] = {1.0};
    double den = 1.0;
    int deg = 0;
    for (int k2 = 0; k2 < m; ++k2) {
      if (k2 == k) continue;
      for (int a = deg + 1; a >= 0; --a) q[a] = (a > 0 ? q[a - 1] : 0.0) - n[k2] * (a <= deg ? q[a] : 0.0);
      ++deg;
      den *= n[k] - n[k2];
    }
    for (int a = 0; a < m; ++a) A[k][a] = q[a] / den;
  }
}

// D = A^T C B of the step's table (CdcTable::D); skipped for repeated / unordered points (nearest-row rule)
template <class T>
__device__ void cdc_bivariate(const RunParams& p, T* s, int m) {
  if (s->degenerate || m < 2) return;
  const double c = 0.5 * (s->zd[0] + s->zd[m - 1]), h = 0.5 * (s->zd[m - 1] - s->zd[0]);
  if (!(h > 0.0) || !isfinite(h)) {   // marginal points at +-inf (a diverged run): the step yields NaN, as the
    for (int a = 0; a < kCdcBiv; ++a)   // Lagrange form would, and the paths are counted as non-finite
      for (int b = 0; b < kCdcBiv; ++b) s->D[a][b] = CUDART_NAN_F;
    s->shinv = 0.0f;
    s->sc = CUDART_NAN_F;
    return;
  }
  double sn[kCdcBiv], xn[kCdcBiv], A[kCdcBiv][kCdcBiv], B[kCdcBiv][kCdcBiv];
  for (int k = 0; k < m; ++k) {
    sn[k] = (s->zd[k] - c) / h;
    xn[k] = (double)p.xhi[k] + (double)p.xlo[k];
  }
  lagrange_monomial(sn, m, A);
  lagrange_monomial(xn, m, B);
  double CB[kCdcBiv][kCdcBiv];
  for (int k = 0; k < m; ++k)
    for (int b = 0; b < m; ++b) {
      double a = 0.0;
      for (int j = 0; j < m; ++j) a += (double)s->C[k][j] * B[j][b];
      CB[k][b] = a;
    }
  for (int a = 0; a < kCdcBiv; ++a)
    for (int b = 0; b < kCdcBiv; ++b) {
      double v = 0.0;
      if (a < m && b < m)
        for (int k = 0; k < m; ++k) v += A[k][a] * CB[k][b];
      s->D[a][b] = (float)v;
    }
  s->shinv = (float)(1.0 / h);
  s->sc = (float)(-c / h);
}

// ---- table rows C[k][.] = H(z_k)
__global__ void cdc_table_exact_kernel(const __grid_constant__ RunParams p, CdcScratch* s) {
  const int k = threadIdx.x / kMaxM, j = threadIdx.x % kMaxM;
  if (k < p.m && j < p.m) {
    const float zk = s->z[k];
    s->C[k][j] = (p.colloc == kExactGbm) ? zk * p.c[j] : fmaf(p.ou_a, zk, p.ou_b) + p.c[j];
  }
  __syncthreads();
  if (threadIdx.x == 0 && p.m <= kCdcBiv) cdc_bivariate(p, s, p.m);
}

// MLP on `rows` states zin[0..rows), fp32 with the accurate activations of the FP32 kernel, layer 1 folded
// with the bias l1b (the horizon's dt and theta); out[k][j] = res_y zin[k] + a_j osc_j + osh_j.  The weight
// image is the FP32 kernel's (hidden layers W[H][HS] + b, then output rows).  Block-wide (all threads call).
template <int ACT>
__device__ void cdc_mlp_rows(const RunParams& p, const float* l1b, const float* osc, const float* osh,
                             const float* zin, int rows, float (*out)[kMaxM]) {
  __shared__ float h[kMaxM][kMaxW], g[kMaxM][kMaxW];
  const int m = p.m, H = p.width, HS = (H == 50) ? 52 : 64, L = p.n_hidden;
  const int MR = (H == 50) ? m : kMaxM;
  __syncthreads();
  for (int i = threadIdx.x; i < rows * kMaxW; i += blockDim.x) {
    const int k = i / kMaxW, u = i % kMaxW;
    h[k][u] = (u < H) ? activate<ACT>(fmaf(p.l1w[u], zin[k], l1b[u])) : 0.0f;
  }
  __syncthreads();
  for (int l = 0; l < L - 1; ++l) {
    const float* W = p.wdev + (size_t)l * f32_layer_floats(H, HS);
    const float* b = W + (size_t)H * HS;
    for (int i = threadIdx.x; i < rows * kMaxW; i += blockDim.x) {
      const int k = i / kMaxW, u = i % kMaxW;
      float a = 0.0f;
      if (u < H) {
        a = b[u];
        for (int v = 0; v < H; ++v) a = fmaf(W[(size_t)u * HS + v], h[k][v], a);
        a = activate<ACT>(a);
      }
      g[k][u] = a;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < rows * kMaxW; i += blockDim.x) h[i / kMaxW][i % kMaxW] = g[i / kMaxW][i % kMaxW];
    __syncthreads();
  }
  const float* Wo = p.wdev + (size_t)(L - 1) * f32_layer_floats(H, HS);
  const float* bo = Wo + (size_t)MR * HS;
  for (int i = threadIdx.x; i < rows * m; i += blockDim.x) {
    const int k = i / m, j = i % m;
    float a = bo[j];
    for (int v = 0; v < H; ++v) a = fmaf(Wo[(size_t)j * HS + v], h[k][v], a);
    out[k][j] = fmaf(p.res_y, zin[k], fmaf(a, osc[j], osh[j]));
  }
  __syncthreads();
}

// table rows C[k][.] = H(z_k) with the network (the run's dt)
template <int ACT>
__global__ void __launch_bounds__(256) cdc_table_mlp_kernel(const __grid_constant__ RunParams p, CdcScratch* s) {
  cdc_mlp_rows<ACT>(p, p.l1b, p.out_scale, p.out_shift, s->z, p.m, s->C);   // ends with a block barrier
  if (threadIdx.x == 0 && p.m <= kCdcBiv) cdc_bivariate(p, s, p.m);
}

// SL7_SCHEME_CDC_PRED (reading R-26): the marginal collocation points of Y(t_i) are the predictor's at
// (Y0, t_i = i dt, theta) -- the horizon's folded constants hz -- instead of quantiles of the paths
// (t_0: every path at Y0, a degenerate table); then the table rows as above.  One block.

template <int ACT, class T>
__device__ void cdc_pred_table_body(const RunParams& p, const CdcHorizon& hz, T* s, int step) {
  __shared__ float zr[1][kMaxM];
  const int m = p.m;
  if (step > 0 && p.colloc == kAnn) {
    cdc_mlp_rows<ACT>(p, hz.l1b, hz.osc, hz.osh, &p.y0, 1, zr);
  } else if (threadIdx.x < m) {
    const int j = threadIdx.x;
    zr[0][j] = (step == 0) ? p.y0
             : (p.colloc == kExactGbm) ? p.y0 * hz.c[j] : fmaf(hz.ou_a, p.y0, hz.ou_b) + hz.c[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int degen = 0;
    for (int k = 0; k < m; ++k) {
      s->zd[k] = (double)zr[0][k];
      if (k > 0 && !(s->zd[k] > s->zd[k - 1])) degen = 1;   // repeated, unordered or NaN points
    }
    cdc_finalize_marginals(s, m, degen);
  }
  __syncthreads();
  if (p.colloc == kAnn) {
    cdc_mlp_rows<ACT>(p, p.l1b, p.out_scale, p.out_shift, s->z, m, s->C);
  } else {
    for (int i = threadIdx.x; i < m * m; i += blockDim.x) {
      const int k = i / m, j = i % m;
      const float zk = s->z[k];
      s->C[k][j] = (p.colloc == kExactGbm) ? zk * p.c[j] : fmaf(p.ou_a, zk, p.ou_b) + p.c[j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && m <= kCdcBiv) cdc_bivariate(p, s, m);
}

template <int ACT, class T>
__global__ void __launch_bounds__(256) cdc_table_pred_kernel(const __grid_constant__ RunParams p,
                                                             const __grid_constant__ CdcHorizon hz, T* s, int step) {
  cdc_pred_table_body<ACT>(p, hz, s, step);
}

// the tables of up to kCdcHzPack steps in one launch (block b: step first + b), horizons in the parameters
constexpr int kCdcHzPack = 32;
struct CdcHorizonPack {
  CdcHorizon h[kCdcHzPack];
};
template <int ACT>
__global__ void __launch_bounds__(256) cdc_tables_pred_kernel(const __grid_constant__ RunParams p,
                                                              const __grid_constant__ CdcHorizonPack hz,
                                                              CdcTable* tb, int first) {
  cdc_pred_table_body<ACT>(p, hz.h[blockIdx.x], tb + first + blockIdx.x, first + (int)blockIdx.x);
}

// ---- per-path CDC step: conditional points by interpolation in the state, then g_m(X_hat)
template <int MR, bool RT_M, bool FAST = false>
__global__ void __launch_bounds__(256) cdc_step_kernel(const __grid_constant__ RunParams p, const CdcScratch* s,
                                                       const float* yin, float* yout,   // may alias (in place)
                                                       int step, int last, unsigned long long* next_hist,
                                                       int clamp_hull) {
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  __shared__ float sz[kMaxM], szlo[kMaxM], sv[kMaxM], sC[kMaxM][kMaxM], ssinv;
  __shared__ int sdeg;
  // m <= kCdcBiv at compile time: the non-degenerate step is ONE bivariate polynomial in s = Y shinv + sc and X
  // (CdcScratch::D, built by the table kernel) instead of the basis in the state, the contraction and g_m
  constexpr bool BIV = !RT_M && MR <= kCdcBiv;
  __shared__ float sD[kCdcBiv][kCdcBiv], sshinv, ssc;
  __shared__ uint32_t nh[256];   // pass-0 digit histogram of the new states (next step's selection)
  if (next_hist)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) nh[i] = 0u;
  for (int i = threadIdx.x; i < kMaxM * kMaxM; i += blockDim.x) {
    const int k = i / kMaxM, j = i % kMaxM;
    sC[k][j] = (k < p.m && j < p.m) ? s->C[k][j] : 0.0f;
  }
  if (threadIdx.x < kMaxM) {
    sz[threadIdx.x] = (threadIdx.x < p.m) ? s->z[threadIdx.x] : 0.0f;
    sv[threadIdx.x] = (threadIdx.x < p.m) ? s->v[threadIdx.x] : 0.0f;
    szlo[threadIdx.x] = (threadIdx.x < p.m) ? s->zlo[threadIdx.x] : 0.0f;
    if (threadIdx.x == 0) ssinv = s->sinv;
  }
  if (threadIdx.x == 0) sdeg = s->degenerate;
  if (BIV) {
    for (int i = threadIdx.x; i < kCdcBiv * kCdcBiv; i += blockDim.x) sD[i / kCdcBiv][i % kCdcBiv] = s->D[i / kCdcBiv][i % kCdcBiv];
    if (threadIdx.x == 0) {
      sshinv = s->shinv;
      ssc = s->sc;
    }
  }
  if (last) hist_init(p, hist);
  __syncthreads();
  const int m = p.m;
  // the m x m table in registers when m is a compile-time constant (49 for m = 7): it is the same for every
  // path, and reading it from shared memory cost one LDS per FFMA of the contraction below
  float Cr[RT_M || BIV ? 1 : MR][RT_M || BIV ? 1 : MR];
  if constexpr (!RT_M && !BIV) {
#pragma unroll
    for (int k = 0; k < MR; ++k)
#pragma unroll
      for (int j = 0; j < MR; ++j) Cr[k][j] = sC[k][j];
  }
  float Dr[BIV ? MR : 1][BIV ? MR : 1];
  if constexpr (BIV) {
#pragma unroll
    for (int a = 0; a < MR; ++a)
#pragma unroll
      for (int b = 0; b < MR; ++b) Dr[a][b] = sD[a][b];
  }
  const float shinv = sshinv, sc = ssc;
  StatAcc acc;
  uint32_t ncl = 0;   // CDC_PRED: clamped path-steps of this step (stats E1)
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the fused histogram's __match_any_sync needs every lane)
  // the state of the next path is loaded one iteration ahead: at ~25% occupancy the load latency of Y was
  // the top stall (the first use of Y), not the arithmetic
  const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  float Ynext = (first + lane < p.n_paths) ? yin[first + lane] : 0.0f;
  for (uint64_t base = first; base < p.n_paths; base += stride) {
    const uint64_t q = base + lane;
    const float Y = Ynext;
    if (q + stride < p.n_paths) Ynext = yin[q + stride];   // yin may alias yout: a different path's slot
    int nbin = -1;
    if (q < p.n_paths) {
    float y[MR], sst = 0.0f;
    if (sdeg) {
      int kb = 0;
      float db = fabsf(Y - sz[0]);
      for (int k = 1; k < m; ++k) {
        const float d = fabsf(Y - sz[k]);
        if (d < db) { db = d; kb = k; }
      }
#pragma unroll
      for (int j = 0; j < MR; ++j) y[j] = sC[kb][j];
    } else {
      // Lagrange basis in the state on the marginal nodes (normalised barycentric product form)
      float d[MR], pre[MR];
#pragma unroll
      // Y - z_k with the marginal point carried as z + zlo (double-accurate nodes, as the GH grid's hi/lo)
      // CDC_PRED (R-26): the state clamped to the marginal hull (zlo = 0 there: the points are fp32); NaN stays
      const float Yb = !clamp_hull ? Y : (Y < sz[0]) ? sz[0] : (Y > sz[m - 1]) ? sz[m - 1] : Y;
      ncl += (clamp_hull && (Y < sz[0] || Y > sz[m - 1])) ? 1u : 0u;
      if constexpr (BIV) {
        sst = fmaf(Yb, shinv, sc);
      } else {
      for (int k = 0; k < MR; ++k) d[k] = (RT_M && k >= m) ? 1.0f : ((Yb - sz[k]) - szlo[k]) * ssinv;
      pre[0] = 1.0f;
#pragma unroll
      for (int k = 1; k < MR; ++k) pre[k] = pre[k - 1] * d[k - 1];
      float suf = 1.0f, den = 0.0f, lk[MR];
#pragma unroll
      for (int k = MR - 1; k >= 0; --k) {
        lk[k] = sv[k] * (pre[k] * suf);
        den += lk[k];
        suf *= d[k];
      }
      const float rden = __fdividef(1.0f, den);
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        float a = 0.0f;
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          if constexpr (RT_M) a = fmaf(lk[k], sC[k][j], a);
          else a = fmaf(lk[k], Cr[k][j], a);
        }
        y[j] = a * rden;
      }
      }
    }
    // X_hat for (path, step): the Philox block of the step, then only the Box-Muller pair that holds it
    const uint64_t gp = p.path_offset + q;
    const uint4 rr = philox_path_block_rk(p.rk0, p.rk1, gp, (uint32_t)(step >> 2));
    const int r = step & 3;
    float za, zb;
    if constexpr (FAST) box_muller_fast((r < 2) ? rr.x : rr.z, (r < 2) ? rr.y : rr.w, za, zb);
    else box_muller((r < 2) ? rr.x : rr.z, (r < 2) ? rr.y : rr.w, za, zb);
    const float Z = (r & 1) ? zb : za;
    float Yn;
    if (BIV && !sdeg) {
      float acc = 0.0f;
#pragma unroll
      for (int b = MR - 1; b >= 0; --b) {
        float qv = Dr[MR - 1][b];
#pragma unroll
        for (int a = MR - 2; a >= 0; --a) qv = fmaf(qv, sst, Dr[a][b]);
        acc = (b == MR - 1) ? qv : fmaf(acc, Z, qv);
      }
      Yn = acc;
    } else {
      Yn = gm_eval<MR, RT_M>(p, Z, y);
    }
    yout[q] = Yn;
    if (last && p.has_stats) stat_add(acc, p, Yn, 0.0, hist);
    nbin = isfinite(Yn) ? (int)(f2key(Yn) >> 24) : -1;
    }
    if (next_hist) warp_hist_add(nh, nbin);   // one call site, all lanes
  }
  if (last && p.has_stats) {
    acc.e1 += (double)ncl;
    stat_flush(acc, p, hist, red);
  } else if (p.has_stats && clamp_hull) {
    const double c = warp_sum((double)ncl);
    if (lane == 0 && c != 0.0) atomicAdd(&p.stats[6], c);
  }
  if (next_hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (nh[i]) atomicAdd(&next_hist[i], (unsigned long long)nh[i]);
  }
}

// ---- CDC_PRED fused over all steps: the tables do not depend on the paths, so each thread carries P paths
// through every step in registers (no state round trip through HBM, one launch), draws each Philox block once
// per 4 steps (all four normals used, where the per-step kernel draws a block per step and keeps one), and
// reads a step's table into registers once for its P paths.  All steps' tables are staged in shared memory.
template <int MR>
struct CdcSTab {
  float C[MR][MR];
  float D[MR][MR];   // the step as a bivariate polynomial (CdcTable::D)
  float z[MR], v[MR];
  float sinv, shinv, sc;
  int deg;
};
constexpr int kCdcFusedP = 4;

// nclamp: +1 when the state lies outside the marginal hull and is clamped (reported in the stats vector's E1 slot)
template <int MR, bool FAST>
__device__ __forceinline__ float cdc_pred_path_step(const RunParams& p, const CdcSTab<MR>& T, const float (&Cr)[MR][MR],
                                                    const float (&zr)[MR], const float (&vr)[MR], float sinv,
                                                    float Y, float Z, uint32_t& nclamp) {
  float y[MR];
  if (T.deg) {   // repeated / unordered marginal points (step 0): the nearest row, ties -> lowest k (R-20)
    int kb = 0;
    float db = fabsf(Y - zr[0]);
#pragma unroll
    for (int k = 1; k < MR; ++k) {
      const float d = fabsf(Y - zr[k]);
      if (d < db) { db = d; kb = k; }
    }
#pragma unroll
    for (int j = 0; j < MR; ++j) y[j] = T.C[kb][j];
  } else {
    const float Yb = (Y < zr[0]) ? zr[0] : (Y > zr[MR - 1]) ? zr[MR - 1] : Y;   // hull clamp (R-26); NaN stays
    nclamp += (Y < zr[0] || Y > zr[MR - 1]) ? 1u : 0u;
    float d[MR], pre[MR], lk[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) d[k] = (Yb - zr[k]) * sinv;
    pre[0] = 1.0f;
#pragma unroll
    for (int k = 1; k < MR; ++k) pre[k] = pre[k - 1] * d[k - 1];
    float suf = 1.0f, den = 0.0f;
#pragma unroll
    for (int k = MR - 1; k >= 0; --k) {
      lk[k] = vr[k] * (pre[k] * suf);
      den += lk[k];
      suf *= d[k];
    }
    const float rden = __fdividef(1.0f, den);
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      float a = 0.0f;
#pragma unroll
      for (int k = 0; k < MR; ++k) a = fmaf(lk[k], Cr[k][j], a);
      y[j] = a * rden;
    }
  }
  return gm_eval<MR, false>(p, Z, y);
}

template <int MR, bool FAST, bool BIV = true, bool ESTRIN = false>
__global__ void __launch_bounds__(256, 2) cdc_pred_fused_kernel(const __grid_constant__ RunParams p,
                                                             const CdcTable* __restrict__ tabs, float* __restrict__ out) {
  constexpr int P = kCdcFusedP;
  extern __shared__ __align__(16) unsigned char smem[];
  CdcSTab<MR>* st = reinterpret_cast<CdcSTab<MR>*>(smem);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + sizeof(CdcSTab<MR>) * (size_t)p.n_steps);
  __shared__ double red[8];
  const int n = p.n_steps;
  for (int i = threadIdx.x; i < n * MR * MR; i += blockDim.x) {
    const int t = i / (MR * MR), r = i % (MR * MR);
    st[t].C[r / MR][r % MR] = tabs[t].C[r / MR][r % MR];
    st[t].D[r / MR][r % MR] = tabs[t].D[r / MR][r % MR];
  }
  for (int i = threadIdx.x; i < n * MR; i += blockDim.x) {
    const int t = i / MR, k = i % MR;
    st[t].z[k] = tabs[t].z[k];
    st[t].v[k] = tabs[t].v[k];
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    st[t].sinv = tabs[t].sinv;
    st[t].shinv = tabs[t].shinv;
    st[t].sc = tabs[t].sc;
    st[t].deg = tabs[t].degenerate;
  }
  hist_init(p, hist);
  __syncthreads();
  const bool full = (p.out_mode == kFull);
  const uint64_t N = p.n_paths, chunk = (uint64_t)blockDim.x * P;
  StatAcc acc;
  uint32_t ncl = 0;   // clamped path-steps of this thread's valid paths
  for (uint64_t base = (uint64_t)blockIdx.x * chunk; base < N; base += (uint64_t)gridDim.x * chunk) {
    float Y[P], zn[P][4];
    bool ok[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const uint64_t q = base + (uint64_t)u * blockDim.x + threadIdx.x;
      ok[u] = q < N;
      Y[u] = p.y0;
      if (full && ok[u]) out[q] = p.y0;
    }
    for (int i0 = 0; i0 < n; i0 += 4) {
      // one Philox block per path gives the normals of steps i0..i0+3 (Z_{4b+r}, cos before sin)
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const uint64_t q = base + (uint64_t)u * blockDim.x + threadIdx.x;
        const uint4 rr = philox_path_block_rk(p.rk0, p.rk1, p.path_offset + q, (uint32_t)(i0 >> 2));
        if constexpr (FAST) {
          box_muller_fast(rr.x, rr.y, zn[u][0], zn[u][1]);
          box_muller_fast(rr.z, rr.w, zn[u][2], zn[u][3]);
        } else {
          box_muller(rr.x, rr.y, zn[u][0], zn[u][1]);
          box_muller(rr.z, rr.w, zn[u][2], zn[u][3]);
        }
      }
      // not unrolled over r (the normal is picked by selects): 4 copies of the step body instead of 16 keep the
      // kernel inside the instruction cache (ncu: 15% no_instructions stalls with the 16-copy version)
#pragma unroll 1
      for (int r = 0; r < 4; ++r) {
        const int i = i0 + r;
        if (i >= n) break;
        const CdcSTab<MR>& T = st[i];
        if (BIV && !T.deg) {
          // Y' = sum_b X^b P_b(s), P_b(s) = sum_a D[a][b] s^a: two paths per FFMA2 with D broadcast
          const float zlo = T.z[0], zhi = T.z[MR - 1], shinv = T.shinv, sc = T.sc;
#pragma unroll
          for (int u = 0; u < P; u += 2) {
            float Zp[2], Sp[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const float Yv = Y[u + v];
              Zp[v] = (r == 0) ? zn[u + v][0] : (r == 1) ? zn[u + v][1] : (r == 2) ? zn[u + v][2] : zn[u + v][3];
              const float Yb = (Yv < zlo) ? zlo : (Yv > zhi) ? zhi : Yv;   // hull clamp (R-26); NaN stays
              ncl += (ok[u + v] && (Yv < zlo || Yv > zhi)) ? 1u : 0u;
              Sp[v] = fmaf(Yb, shinv, sc);
            }
            const uint64_t S = pk2(Sp[0], Sp[1]), X = pk2(Zp[0], Zp[1]);
            uint64_t acc = 0;
            if constexpr (ESTRIN) {
              // the same polynomial in Estrin's order (pairs (c_2i + c_2i+1 t), then powers t^2, t^4): the same
              // FMA count as Horner, a dependence chain of ~log2(m) + 1 instead of m - 1
              const uint64_t z0 = pk2(0.0f, 0.0f);
              const uint64_t S2 = fma2(S, S, z0), X2 = fma2(X, X, z0);
              uint64_t P[MR];
#pragma unroll
              for (int b = 0; b < MR; ++b) {
                uint64_t e[(MR + 1) / 2];
#pragma unroll
                for (int i = 0; i < (MR + 1) / 2; ++i)
                  e[i] = (2 * i + 1 < MR) ? fma2(S, pk2(T.D[2 * i + 1][b], T.D[2 * i + 1][b]), pk2(T.D[2 * i][b], T.D[2 * i][b]))
                                          : pk2(T.D[2 * i][b], T.D[2 * i][b]);
                uint64_t q = e[(MR + 1) / 2 - 1];
#pragma unroll
                for (int i = (MR + 1) / 2 - 2; i >= 0; --i) q = fma2(q, S2, e[i]);
                P[b] = q;
              }
              uint64_t f[(MR + 1) / 2];
#pragma unroll
              for (int i = 0; i < (MR + 1) / 2; ++i) f[i] = (2 * i + 1 < MR) ? fma2(X, P[2 * i + 1], P[2 * i]) : P[2 * i];
              acc = f[(MR + 1) / 2 - 1];
#pragma unroll
              for (int i = (MR + 1) / 2 - 2; i >= 0; --i) acc = fma2(acc, X2, f[i]);
            } else {
#pragma unroll
            for (int b = MR - 1; b >= 0; --b) {
              uint64_t q = pk2(T.D[MR - 1][b], T.D[MR - 1][b]);
#pragma unroll
              for (int a = MR - 2; a >= 0; --a) q = fma2(q, S, pk2(T.D[a][b], T.D[a][b]));
              acc = (b == MR - 1) ? q : fma2(acc, X, q);
            }
            }
            up2(acc, Y[u], Y[u + 1]);
#pragma unroll
            for (int v = 0; v < 2; ++v)
              if (full && ok[u + v]) out[(uint64_t)(i + 1) * N + base + (uint64_t)(u + v) * blockDim.x + threadIdx.x] = Y[u + v];
          }
        } else {
        float Cr[MR][MR], zr[MR], vr[MR];
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          zr[k] = T.z[k];
          vr[k] = T.v[k];
#pragma unroll
          for (int j = 0; j < MR; ++j) Cr[k][j] = T.C[k][j];
        }
        const float sinv = T.sinv;
#pragma unroll
        for (int u = 0; u < P; ++u) {
          const float Z = (r == 0) ? zn[u][0] : (r == 1) ? zn[u][1] : (r == 2) ? zn[u][2] : zn[u][3];
          uint32_t c = 0;
          Y[u] = cdc_pred_path_step<MR, FAST>(p, T, Cr, zr, vr, sinv, Y[u], Z, c);
          ncl += ok[u] ? c : 0u;
          if (full && ok[u]) out[(uint64_t)(i + 1) * N + base + (uint64_t)u * blockDim.x + threadIdx.x] = Y[u];
        }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!ok[u]) continue;
      const uint64_t q = base + (uint64_t)u * blockDim.x + threadIdx.x;
      if (p.out_mode == kTerminal) out[q] = Y[u];
      if (p.has_stats) stat_add(acc, p, Y[u], 0.0, hist);
    }
  }
  if (p.has_stats) {
    acc.e1 += (double)ncl;   // E1 of a CDC_PRED run: clamped path-steps (no strong-error reference, include/sl7.h)
    stat_flush(acc, p, hist, red);
  }
}

__global__ void fill_kernel(float* y, uint64_t n, float v) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x)
    y[q] = v;
}

// ------------------------------------------------------------------------------------------------
size_t cdc_scratch_bytes() { return sizeof(CdcScratch); }

int cdc_init_scratch(void* scratch, void* stream) {
  CdcScratch h;
  memset(&h, 0, sizeof h);
  h.nslot = 1;
  return (int)cudaMemcpyAsync(scratch, &h, sizeof h, cudaMemcpyHostToDevice, (cudaStream_t)stream);
}

namespace {

unsigned cdc_grid(uint64_t n, int num_sms) {
  return (unsigned)(((n + 255) / 256) < (uint64_t)num_sms * 8 ? (n + 255) / 256 : (uint64_t)num_sms * 8);
}

}  // namespace

int cdc_fill(float* y, uint64_t n, float v, void* stream, int num_sms) {
  fill_kernel<<<cdc_grid(n, num_sms), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(y, n, v);
  return (int)cudaGetLastError();
}

int cdc_hist(const RunParams& p, void* scratch, const float* y, int pass, unsigned long long* hist, bool zero,
             void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (zero) {
    const cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * kCdcMaxT * 256, st);
    if (e != cudaSuccess) return (int)e;
  }
  const CdcScratch* sc = reinterpret_cast<const CdcScratch*>(scratch);
  const unsigned grid = cdc_grid(p.n_paths, num_sms);
  if (pass == 0) {
    cdc_hist_kernel<4, 0><<<grid, 256, 0, st>>>(y, p.n_paths, sc, hist);
  } else if (pass == 1) {
    cdc_hist_kernel<4, 1><<<grid, 256, 256, st>>>(y, p.n_paths, sc, hist);
  } else {
    auto k = (pass == 2) ? cdc_hist_kernel<16, 2> : cdc_hist_kernel<16, 3>;
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kCdcLutBytes);
    if (e != cudaSuccess) return (int)e;
    k<<<grid, 256, kCdcLutBytes, st>>>(y, p.n_paths, sc, hist);
  }
  return (int)cudaGetLastError();
}

int cdc_select(const RunParams& p, const CdcLevels& lv, void* scratch, int pass, unsigned long long* hist, bool clear,
               void* stream) {
  cdc_scan_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(pass, p.m, reinterpret_cast<CdcScratch*>(scratch),
                                                                          lv, hist, clear ? 1 : 0);
  return (int)cudaGetLastError();
}

int cdc_advance(const RunParams& p, void* scratch, const float* yin, float* yout, int step, bool stats, void* stream,
                int num_sms, unsigned long long* next_hist) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CdcScratch* s = reinterpret_cast<CdcScratch*>(scratch);
  if (p.colloc == kAnn) {
    if (p.act == SL7_ACT_TANH) cdc_table_mlp_kernel<SL7_ACT_TANH><<<1, 256, 0, st>>>(p, s);
    else cdc_table_mlp_kernel<SL7_ACT_SOFTPLUS><<<1, 256, 0, st>>>(p, s);
  } else {
    cdc_table_exact_kernel<<<1, kMaxM * kMaxM, 0, st>>>(p, s);
  }
  const size_t hist = (stats && p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0;
  const bool fast = p.flags & SL7_FLAG_FAST_NORMALS;
  auto step_k = (p.m == 5) ? (fast ? cdc_step_kernel<5, false, true> : cdc_step_kernel<5, false>)
              : (p.m == 7) ? (fast ? cdc_step_kernel<7, false, true> : cdc_step_kernel<7, false>)
                           : (fast ? cdc_step_kernel<kMaxM, true, true> : cdc_step_kernel<kMaxM, true>);
  if (hist > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(step_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist);
    if (e != cudaSuccess) return (int)e;
  }
  step_k<<<cdc_grid(p.n_paths, num_sms), 256, hist, st>>>(p, s, yin, yout, step, stats ? 1 : 0, next_hist, 0);
  return (int)cudaGetLastError();
}

// Runs all n_steps of the CDC scheme on one device (the selection histograms live in the scratch).
int launch_cdc(const RunParams& p, const CdcLevels& lv, void* scratch, float* const* rows, int nrows, void* stream,
               int num_sms) {
  CdcScratch* s = reinterpret_cast<CdcScratch*>(scratch);
  unsigned long long* hist = &s->hist[0][0];
  int e = cdc_fill(rows[0], p.n_paths, p.y0, stream, num_sms);   // row 0 = Y0
  if (e) return e;
  for (int i = 0; i < p.n_steps; ++i) {
    const float* yin = rows[(nrows == 1) ? 0 : i];
    float* yout = rows[(nrows == 1) ? 0 : i + 1];
    for (int pass = 0; pass < 4; ++pass) {
      if (pass > 0 || i == 0) {   // pass 0 of steps >= 1: histogrammed by the previous step kernel
        e = cdc_hist(p, scratch, yin, pass, hist, false, stream, num_sms);
        if (e) return e;
      }
      e = cdc_select(p, lv, scratch, pass, hist, true, stream);
      if (e) return e;
    }
    const bool last = (i == p.n_steps - 1);
    e = cdc_advance(p, scratch, yin, yout, i, last && p.has_stats, stream, num_sms, last ? nullptr : hist);
    if (e) return e;
  }
  return 0;
}

// SL7_SCHEME_CDC_PRED: per step the predicted-marginal table, then the (unchanged) per-path step kernel.
// No selection passes: paths are coupled only through the table, which is the same for any path set.
size_t cdc_table_bytes() { return sizeof(CdcTable); }

int launch_cdc_pred(const RunParams& p, const CdcHorizon* hz, void* scratch, float* const* rows, int nrows,
                    void* stream, int num_sms, void* tables) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CdcScratch* s = reinterpret_cast<CdcScratch*>(scratch);
  if (tables && (p.m == 5 || p.m == 7)) {
    // fused path: the n_steps tables (one block each, up to 32 per launch), then one kernel over all steps
    CdcTable* tb = reinterpret_cast<CdcTable*>(tables);
    for (int first = 0; first < p.n_steps; first += kCdcHzPack) {
      const int cnt = (p.n_steps - first < kCdcHzPack) ? p.n_steps - first : kCdcHzPack;
      CdcHorizonPack pack;
      std::memcpy(pack.h, hz + first, sizeof(CdcHorizon) * (size_t)cnt);
      if (p.act == SL7_ACT_TANH) cdc_tables_pred_kernel<SL7_ACT_TANH><<<cnt, 256, 0, st>>>(p, pack, tb, first);
      else cdc_tables_pred_kernel<SL7_ACT_SOFTPLUS><<<cnt, 256, 0, st>>>(p, pack, tb, first);
    }
    const bool fast = p.flags & SL7_FLAG_FAST_NORMALS;
    auto k = (p.m == 5) ? (fast ? cdc_pred_fused_kernel<5, true> : cdc_pred_fused_kernel<5, false>)
                        : (fast ? cdc_pred_fused_kernel<7, true> : cdc_pred_fused_kernel<7, false>);
#ifdef SL7_AB_HOOKS
    if (const char* v = std::getenv("SL7_TC_VARIANT"))
      if (std::atoi(v) == 70)   // the r01/r02 step: conditional points by Lagrange in the state, then g_m
        k = (p.m == 5) ? (fast ? cdc_pred_fused_kernel<5, true, false> : cdc_pred_fused_kernel<5, false, false>)
                       : (fast ? cdc_pred_fused_kernel<7, true, false> : cdc_pred_fused_kernel<7, false, false>);
      else if (std::atoi(v) == 71)   // Estrin order
        k = (p.m == 5) ? (fast ? cdc_pred_fused_kernel<5, true, true, true> : cdc_pred_fused_kernel<5, false, true, true>)
                       : (fast ? cdc_pred_fused_kernel<7, true, true, true> : cdc_pred_fused_kernel<7, false, true, true>);
#endif
    const size_t tab = (p.m == 5 ? sizeof(CdcSTab<5>) : sizeof(CdcSTab<7>)) * (size_t)p.n_steps;
    const size_t smem = tab + ((p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0);
    const cudaError_t ce = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ce != cudaSuccess) return (int)ce;
    const uint64_t groups = (p.n_paths + 256 * kCdcFusedP - 1) / (256 * kCdcFusedP);
    const unsigned grid = (unsigned)(groups < (uint64_t)num_sms * 2 * 8 ? groups : (uint64_t)num_sms * 2 * 8);
    k<<<grid, 256, smem, st>>>(p, tb, rows[0]);
    return (int)cudaGetLastError();
  }
  int e = cdc_fill(rows[0], p.n_paths, p.y0, stream, num_sms);   // row 0 = Y0
  if (e) return e;
  const size_t hist = (p.has_stats && p.n_bins > 0) ? sizeof(uint32_t) * (size_t)(p.n_bins + 2) : 0;
  const bool fast = p.flags & SL7_FLAG_FAST_NORMALS;
  auto step_k = (p.m == 5) ? (fast ? cdc_step_kernel<5, false, true> : cdc_step_kernel<5, false>)
              : (p.m == 7) ? (fast ? cdc_step_kernel<7, false, true> : cdc_step_kernel<7, false>)
                           : (fast ? cdc_step_kernel<kMaxM, true, true> : cdc_step_kernel<kMaxM, true>);
  if (hist > 48 * 1024) {
    const cudaError_t ce = cudaFuncSetAttribute(step_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist);
    if (ce != cudaSuccess) return (int)ce;
  }
  for (int i = 0; i < p.n_steps; ++i) {
    if (p.act == SL7_ACT_TANH) cdc_table_pred_kernel<SL7_ACT_TANH><<<1, 256, 0, st>>>(p, hz[i], s, i);
    else cdc_table_pred_kernel<SL7_ACT_SOFTPLUS><<<1, 256, 0, st>>>(p, hz[i], s, i);
    const float* yin = rows[(nrows == 1) ? 0 : i];
    float* yout = rows[(nrows == 1) ? 0 : i + 1];
    const bool last = (i == p.n_steps - 1);
    step_k<<<cdc_grid(p.n_paths, num_sms), 256, last ? hist : 0, st>>>(p, s, yin, yout, i, last && p.has_stats ? 1 : 0,
                                                                       nullptr, 1);
    e = (int)cudaGetLastError();
    if (e) return e;
  }
  return 0;
}

}  // namespace sl7
