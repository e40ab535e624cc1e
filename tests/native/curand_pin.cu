// Library pin for the path generator's RNG (test infrastructure only, not linked into libsl7.so):
// cuRAND's Philox4_32_10 device generator.  curand_init(seed, subsequence = path, offset = 4*block)
// puts the counter at (block, 0, path_lo, path_hi) with key (seed_lo, seed_hi)
// (curand_kernel.h: curand_init / Philox_State_Incr_hi / Philox_State_Incr), so curand4() must
// return exactly the words sl7_philox_u32 returns.
#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <stdint.h>

__global__ void curand_pin_kernel(unsigned long long seed, unsigned long long off, unsigned long long n,
                                  unsigned block, uint32_t* out) {
  const unsigned long long q = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, off + q, 4ull * block, &st);
  const uint4 r = curand4(&st);
  out[q] = r.x;
  out[n + q] = r.y;
  out[2 * n + q] = r.z;
  out[3 * n + q] = r.w;
}

extern "C" int curand_pin_u32(unsigned long long seed, unsigned long long off, unsigned long long n, unsigned block,
                              uint32_t* d_out, void* stream) {
  curand_pin_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(seed, off, n, block, d_out);
  return (int)cudaGetLastError();
}
