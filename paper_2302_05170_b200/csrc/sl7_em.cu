// sl7_em.cu -- Euler-Maruyama comparator and offline training-set generation on sm_100a
// (SURVEY.md §8(f) rows 2-3).
//
//   em_kernel            Eq. 6.2 for GBM / OU / CIR with K sub-steps per large step,
//                        fine step k of path p on normal Z_{p,k} of the path generator's RNG (a1), the
//                        same outputs and fused statistics as the 7L kernels (strong error against the
//                        exact solution on the same fine normals).
//   em_rows_kernel       Algorithm I step 1: per feature row r, M inner EM paths of
//                        K_r = ceil(dt_r / dtau) sub-steps, global path id path_offset + r M + q; rows
//                        are launched longest-first (K descending) so the block scheduler balances them.
//   row_quantiles_kernel the labels: empirical quantiles of each row's M terminal values at the levels
//                        Phi(x_j) (plotting position (k - 0.5)/M, linear interpolation, reading R-18),
//                        one 1024-thread CTA per row, exact order statistics by a 4-pass 8-bit radix
//                        select with shared-memory histograms (the row is re-read from L2 per pass);
//                        warp t fixes target t's digit with a warp scan.
// The work per fine path-step is one normal (Philox/4 + Box-Muller/2) plus 2-4 FP32 ops, so both EM
// kernels are issue-bound on the RNG, like the exact-collocation kernels.
#include <cuda_runtime.h>

#include "sl7_device.cuh"

namespace sl7 {

// Eq. 6.2 for the three models; CIR with full truncation Y+ = max(Y, 0) in drift and diffusion (R-22).
template <int MODEL>
__device__ __forceinline__ float em_step(float Y, float Z, float a, float s, float ybar) {
  if constexpr (MODEL == SL7_MODEL_GBM) {
    return fmaf(Y, fmaf(s, Z, a), Y);                       // Y + Y (mu dtau + sigma sqrt(dtau) Z)
  } else if constexpr (MODEL == SL7_MODEL_OU) {
    return fmaf(s, Z, fmaf(a, ybar - Y, Y));                // Y + lam dtau (ybar - Y) + sigma sqrt(dtau) Z
  } else {
    const float yp = fmaxf(Y, 0.0f);
    return fmaf(s * sqrtf(yp), Z, fmaf(a, ybar - yp, Y));   // ... + sigma sqrt(Y+) sqrt(dtau) Z
  }
}

template <int MODEL, bool FAST, bool REF_ON>
__global__ void __launch_bounds__(256) em_kernel(const __grid_constant__ RunParams p) {
  extern __shared__ uint32_t hist[];
  __shared__ double red[8];
  hist_init(p, hist);
  __syncthreads();
  StatAcc acc;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool full = (p.out_mode == kFull);
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p.n_paths; q += stride) {
    const uint64_t gp = p.path_offset + q;
    float Y = p.y0;
    float* o = p.out + q;
    if (full) *o = Y;
    RefState rs;
    if (REF_ON) ref_init(rs, p);
    if ((p.em_K & 3) == 0) {
      // K a multiple of 4: each large step is K/4 whole Philox blocks (no per-step rotation)
      uint32_t blk = 0;
      for (int i = 0; i < p.n_steps; ++i) {
        for (int b = 0; b < (p.em_K >> 2); ++b, ++blk) {
          float z[4];
          normals4_rk<FAST>(p, gp, blk, z[0], z[1], z[2], z[3]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            Y = em_step<MODEL>(Y, z[u], p.em_a, p.em_s, p.em_ybar);
            if (REF_ON) ref_step(rs, p, z[u]);
          }
        }
        if (full) {
          o += p.n_paths;
          *o = Y;
        }
      }
    } else {
      float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
      uint32_t j = 0;   // fine step
      for (int i = 0; i < p.n_steps; ++i) {
        for (int k = 0; k < p.em_K; ++k, ++j) {
          if ((j & 3u) == 0u) normals4_rk<FAST>(p, gp, j >> 2, z0, z1, z2, z3);
          const float Z = z0;
          z0 = z1; z1 = z2; z2 = z3;
          Y = em_step<MODEL>(Y, Z, p.em_a, p.em_s, p.em_ybar);
          if (REF_ON) ref_step(rs, p, Z);
        }
        if (full) {
          o += p.n_paths;
          *o = Y;
        }
      }
    }
    if (p.out_mode == kTerminal) p.out[q] = Y;
    if (p.has_stats) stat_add(acc, p, Y, REF_ON ? ref_final(rs, p) : 0.0, hist);
  }
  if (p.has_stats) stat_flush(acc, p, hist, red);
}

template <int MODEL, bool FAST>
__global__ void __launch_bounds__(256) em_rows_kernel(const __grid_constant__ RunParams p, const EmRow* __restrict__ rows,
                                                      uint32_t M, uint32_t tiles_per_row, uint64_t row_base,
                                                      float* __restrict__ term) {
  const uint32_t rank = blockIdx.x / tiles_per_row, tile = blockIdx.x - rank * tiles_per_row;
  const EmRow r = rows[rank];
  const uint32_t q = tile * blockDim.x + threadIdx.x;
  if (q >= M) return;
  const uint64_t gp = p.path_offset + (row_base + r.row) * (uint64_t)M + q;
  float Y = r.y0;
  // fine steps in Philox blocks of four (no per-step buffer rotation or block test), then the remainder
  const uint32_t nb = (uint32_t)r.K >> 2, rem = (uint32_t)r.K & 3u;
  float z[4];
  for (uint32_t b = 0; b < nb; ++b) {
    normals4_rk<FAST>(p, gp, b, z[0], z[1], z[2], z[3]);
#pragma unroll
    for (int u = 0; u < 4; ++u) Y = em_step<MODEL>(Y, z[u], r.a, r.s, r.ybar);
  }
  if (rem) {
    normals4_rk<FAST>(p, gp, nb, z[0], z[1], z[2], z[3]);
#pragma unroll
    for (int u = 0; u < 3; ++u)
      if ((uint32_t)u < rem) Y = em_step<MODEL>(Y, z[u], r.a, r.s, r.ybar);
  }
  term[(size_t)r.row * M + q] = Y;
}

__global__ void __launch_bounds__(1024) row_quantiles_kernel(const float* __restrict__ term, uint32_t M, int m,
                                                             const __grid_constant__ CdcLevels lv,
                                                             double* __restrict__ labels) {
  __shared__ uint32_t h[kCdcMaxT][256];
  __shared__ uint32_t sp[kCdcMaxT];       // distinct prefixes of the current pass, ascending
  __shared__ int slot_of[kCdcMaxT];
  __shared__ uint32_t rnk[kCdcMaxT], pre[kCdcMaxT];
  __shared__ double frac[kMaxM];
  __shared__ int nslot;
  __shared__ uint32_t Mf;
  const float* y = term + (size_t)blockIdx.x * M;
  const int T = 2 * m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    nslot = 1;
    sp[0] = 0u;
  }
  __syncthreads();
  for (int pass = 0; pass < 4; ++pass) {
    const int ns = nslot;
    for (int i = tid; i < ns * 256; i += blockDim.x) h[i >> 8][i & 255] = 0u;
    __syncthreads();
    const int shift = 24 - 8 * pass;
    const uint32_t lo = sp[0], hi = sp[ns - 1];
    for (uint32_t q = tid; q < M; q += blockDim.x) {
      const float v = y[q];
      if (!isfinite(v)) continue;
      const uint32_t key = f2key(v);
      int slot = 0;
      if (pass > 0) {
        const uint32_t pf = key >> (shift + 8);
        if (pf < lo || pf > hi) continue;
        int a = 0, b = ns - 1;
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (sp[mid] < pf) a = mid + 1; else b = mid;
        }
        if (sp[a] != pf) continue;
        slot = a;
      }
      atomicAdd(&h[slot][(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (pass == 0) {
      if (warp == 0) {
        uint32_t s = 0;
        for (int b = lane; b < 256; b += 32) s += h[0][b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) Mf = s;
      }
      __syncthreads();
      if (tid < m) {
        // target order statistics (0-based) of the plotting-position quantile, as the oracle:
        // pos = p M + 0.5 clamped to [1, M], k = floor(pos), f = pos - k, ranks k - 1 and min(k, M - 1)
        const uint32_t n = Mf;
        double f = 0.0;
        uint32_t r0 = 0u, r1 = 0u;
        if (n > 0) {
          double pos = __dadd_rn(__dmul_rn(lv.p[tid], (double)n), 0.5);
          pos = fmin(fmax(pos, 1.0), (double)n);
          const double kk = floor(pos);
          f = pos - kk;
          r0 = (uint32_t)kk - 1u;
          r1 = ((uint32_t)kk < n) ? (uint32_t)kk : n - 1u;
        }
        frac[tid] = f;
        rnk[2 * tid] = r0;
        rnk[2 * tid + 1] = r1;
        pre[2 * tid] = pre[2 * tid + 1] = 0u;
      }
      __syncthreads();
    }
    if (Mf > 0 && warp < T) {
      // warp t: find the bin holding target t's residual rank (lane l owns bins 8l..8l+7)
      const int t = warp, sl = (pass == 0) ? 0 : slot_of[t];
      const uint32_t r = rnk[t];
      uint32_t c[8], s = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        c[u] = h[sl][lane * 8 + u];
        s += c[u];
      }
      uint32_t inc = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
      }
      const uint32_t exc = inc - s;
      __syncwarp();
      if (r >= exc && r < inc) {
        uint32_t below = exc;
        int b = lane * 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (below + c[u] > r) {
            b = lane * 8 + u;
            break;
          }
          below += c[u];
        }
        rnk[t] = r - below;
        pre[t] = (pre[t] << 8) | (uint32_t)b;
      }
    }
    __syncthreads();
    if (tid == 0 && pass < 3) {
      // distinct prefixes, ascending (levels clamped to the extreme order statistics repeat rank pairs out
      // of order, e.g. 0, 1, 0, 1, ...)
      int n = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t v = pre[t];
        int a = 0;
        while (a < n && sp[a] < v) ++a;
        if (a == n || sp[a] != v) {
          for (int b = n; b > a; --b) sp[b] = sp[b - 1];
          sp[a] = v;
          ++n;
        }
      }
      for (int t = 0; t < T; ++t) {
        int a = 0;
        while (sp[a] != pre[t]) ++a;
        slot_of[t] = a;
      }
      nslot = n;
    }
    __syncthreads();
  }
  if (tid < m) {
    double out = __longlong_as_double(0x7FF8000000000000ll);   // no finite terminal value: NaN
    if (Mf > 0) {
      const double a = (double)key2f(pre[2 * tid]), b = (double)key2f(pre[2 * tid + 1]), f = frac[tid];
      out = __dadd_rn(__dmul_rn(a, 1.0 - f), __dmul_rn(b, f));
    }
    labels[(size_t)blockIdx.x * m + tid] = out;
  }
}

// ------------------------------------------------------------------------------------------------
namespace {

template <int MODEL, bool FAST, bool REF_ON>
cudaError_t launch_em_t(const RunParams& p, cudaStream_t st, int num_sms) {
  auto kernel = em_kernel<MODEL, FAST, REF_ON>;
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

template <int MODEL>
cudaError_t launch_em_m(const RunParams& p, cudaStream_t st, int num_sms) {
  const bool fast = p.flags & SL7_FLAG_FAST_NORMALS, ref = (p.ref != kRefNone && p.has_stats);
  if (fast) return ref ? launch_em_t<MODEL, true, true>(p, st, num_sms) : launch_em_t<MODEL, true, false>(p, st, num_sms);
  return ref ? launch_em_t<MODEL, false, true>(p, st, num_sms) : launch_em_t<MODEL, false, false>(p, st, num_sms);
}

template <int MODEL, bool FAST>
cudaError_t launch_rows_t(const RunParams& p, const EmRow* rows, uint32_t n_rows, uint32_t M, uint64_t row_base,
                          float* term, cudaStream_t st) {
  const uint32_t tpr = (M + 255u) / 256u;
  const uint64_t blocks = (uint64_t)tpr * n_rows;
  if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
  em_rows_kernel<MODEL, FAST><<<(unsigned)blocks, 256, 0, st>>>(p, rows, M, tpr, row_base, term);
  return cudaGetLastError();
}

template <int MODEL>
cudaError_t launch_rows_m(const RunParams& p, const EmRow* rows, uint32_t n_rows, uint32_t M, uint64_t row_base,
                          float* term, cudaStream_t st) {
  return (p.flags & SL7_FLAG_FAST_NORMALS) ? launch_rows_t<MODEL, true>(p, rows, n_rows, M, row_base, term, st)
                                           : launch_rows_t<MODEL, false>(p, rows, n_rows, M, row_base, term, st);
}

}  // namespace

int launch_em(const RunParams& p, void* stream, int num_sms) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (p.em_model) {
    case SL7_MODEL_GBM: return (int)launch_em_m<SL7_MODEL_GBM>(p, st, num_sms);
    case SL7_MODEL_OU: return (int)launch_em_m<SL7_MODEL_OU>(p, st, num_sms);
    case SL7_MODEL_CIR: return (int)launch_em_m<SL7_MODEL_CIR>(p, st, num_sms);
  }
  return (int)cudaErrorInvalidValue;
}

int launch_em_rows(const RunParams& p, const EmRow* d_rows, uint32_t n_rows, uint32_t M, uint64_t row_base,
                   float* term, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (p.em_model) {
    case SL7_MODEL_GBM: return (int)launch_rows_m<SL7_MODEL_GBM>(p, d_rows, n_rows, M, row_base, term, st);
    case SL7_MODEL_OU: return (int)launch_rows_m<SL7_MODEL_OU>(p, d_rows, n_rows, M, row_base, term, st);
    case SL7_MODEL_CIR: return (int)launch_rows_m<SL7_MODEL_CIR>(p, d_rows, n_rows, M, row_base, term, st);
  }
  return (int)cudaErrorInvalidValue;
}

int launch_row_quantiles(const float* term, uint32_t n_rows, uint32_t M, int m, const CdcLevels& lv, double* labels,
                         void* stream) {
  row_quantiles_kernel<<<n_rows, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(term, M, m, lv, labels);
  return (int)cudaGetLastError();
}

}  // namespace sl7
