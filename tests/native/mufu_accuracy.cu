// Accuracy probe of the MUFU approximations a fast Box-Muller would use (run on the box):
//   lg2.approx.f32 on u = 1 - j 2^-24 (the relative accuracy of log near 1 decides the tail normals)
//   lg2.approx.f32 on (0, 1) (absolute error)
//   sin.approx / cos.approx on (-pi, pi) (absolute error)
//   tanh.approx.f32 (MUFU.TANH) on (-12, 12) (absolute and relative error; the TC kernel's tanh)
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_tanh(int n, float* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float z = -12.0f + 24.0f * ((float)i + 0.5f) / (float)n;
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(z));
  out[i] = r;
}

__global__ void probe(int n, float* lg_near1, float* lg_any, float* s, float* c) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float u = 1.0f - (float)(i + 1) * 0x1p-24f;
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(u));
  lg_near1[i] = r;
  float x = ((float)i + 0.5f) / (float)n;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  lg_any[i] = r;
  float a = (x - 0.5f) * 6.283185307179586f;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  s[i] = r;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  c[i] = r;
}

int main() {
  const int n = 1 << 22;
  float *d[4], *h = new float[(size_t)4 * n];
  for (int k = 0; k < 4; ++k) cudaMalloc(&d[k], sizeof(float) * n);
  probe<<<(n + 255) / 256, 256>>>(n, d[0], d[1], d[2], d[3]);
  for (int k = 0; k < 4; ++k) cudaMemcpy(h + (size_t)k * n, d[k], sizeof(float) * n, cudaMemcpyDeviceToHost);
  double m_rel_near1 = 0, m_abs_any = 0, m_sin = 0, m_cos = 0;
  int worst_j = 0;
  for (int i = 0; i < n; ++i) {
    double u = 1.0 - (double)(i + 1) * std::ldexp(1.0, -24);
    double ref = std::log2(u);
    double rel = std::fabs((h[i] - ref) / ref);
    if (rel > m_rel_near1) { m_rel_near1 = rel; worst_j = i + 1; }
    double x = ((double)(float)(((float)i + 0.5f) / (float)n));
    m_abs_any = std::fmax(m_abs_any, std::fabs(h[n + i] - std::log2(x)));
    double a = (double)(float)(((float)(x) - 0.5f) * 6.283185307179586f);
    m_sin = std::fmax(m_sin, std::fabs(h[2 * (size_t)n + i] - std::sin(a)));
    m_cos = std::fmax(m_cos, std::fabs(h[3 * (size_t)n + i] - std::cos(a)));
  }
  printf("{\"lg2_near1_max_rel\": %.3g, \"worst_j\": %d, \"lg2_abs_any\": %.3g, \"sin_abs\": %.3g, \"cos_abs\": %.3g}\n",
         m_rel_near1, worst_j, m_abs_any, m_sin, m_cos);
  {
    probe_tanh<<<(n + 255) / 256, 256>>>(n, d[0]);
    cudaMemcpy(h, d[0], sizeof(float) * n, cudaMemcpyDeviceToHost);
    double m_abs = 0, m_rel = 0, z_abs = 0, z_rel = 0, sum_err = 0;
    for (int i = 0; i < n; ++i) {
      const double z = (double)(-12.0f + 24.0f * ((float)i + 0.5f) / (float)n);
      const double ref = std::tanh(z), e = (double)h[i] - ref;
      sum_err += e;
      if (std::fabs(e) > m_abs) { m_abs = std::fabs(e); z_abs = z; }
      if (ref != 0 && std::fabs(e / ref) > m_rel) { m_rel = std::fabs(e / ref); z_rel = z; }
    }
    printf("{\"tanh_approx_max_abs\": %.3g, \"at\": %.4g, \"max_rel\": %.3g, \"at_rel\": %.4g, \"mean_err\": %.3g}\n",
           m_abs, z_abs, m_rel, z_rel, sum_err / n);
  }
  // relative error of lg2 for j = 1, 2, 4, ..., 2^22
  for (int j = 1; j <= (1 << 22); j <<= 2) {
    double u = 1.0 - (double)j * std::ldexp(1.0, -24);
    printf("  j=%8d u=1-j*2^-24 lg2_rel_err=%.3g\n", j, std::fabs((h[j - 1] - std::log2(u)) / std::log2(u)));
  }
  return 0;
}
