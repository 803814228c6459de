// Bit-for-bit check of ff_div2 and ff_div2_pair (csrc/device/ff_exact.cuh: two quotients sharing one
// reciprocal, the 3-D projection's c_x / c_w, c_y / c_w; the pair form through FFMA2 / FMUL2) against
// div.rn.f32 (tests/test_gpu_division.py).
// Operands come from a counter-based hash, per mode:
//   0  random bit patterns inside the fast box (d in [2^-60, 2^60], |n| in [2^-40, 2^64))
//   1  random bit patterns over all floats (inf, NaN, zeros, denormals included; d > 0 forced)
//   2  the box edges: exponents at the bounds +-1, mantissas at 0 / all-ones / random
//   3  the projection's range: |n| <= 2^12, d in [2^-12, 2^12], mantissas random
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "../../paper_1505_00344_b200/csrc/device/ff_exact.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float with_exp(uint32_t r, int e) {   // sign from r, biased exponent e
  return __uint_as_float((r & 0x807fffffu) | ((uint32_t)e << 23));
}
__device__ void operands(int mode, uint64_t i, uint64_t seed, float& nx, float& ny, float& d) {
  const uint64_t h0 = mix(seed ^ (i * 3)), h1 = mix(seed ^ (i * 3 + 1)), h2 = mix(seed ^ (i * 3 + 2));
  const uint32_t a = (uint32_t)h0, b = (uint32_t)(h0 >> 32), c = (uint32_t)h1, s = (uint32_t)(h1 >> 32);
  if (mode == 0) {
    d = fabsf(with_exp(a, 67 + (int)(b % 121u)));             // 2^-60 .. 2^60
    nx = with_exp(c, 87 + (int)(s % 104u));                    // 2^-40 .. 2^63
    ny = with_exp((uint32_t)h2, 87 + (int)((h2 >> 32) % 104u));
  } else if (mode == 1) {
    d = fabsf(__uint_as_float(a));
    nx = __uint_as_float(c);
    ny = __uint_as_float((uint32_t)h2);
  } else if (mode == 2) {
    const int de[6] = {66, 67, 68, 186, 187, 188}, ne[6] = {86, 87, 88, 189, 190, 191};
    uint32_t m = (s & 3u) == 0 ? 0u : (s & 3u) == 1 ? 0x7fffffu : (a & 0x7fffffu);
    d = __uint_as_float(((uint32_t)de[b % 6u] << 23) | m);
    m = ((s >> 2) & 3u) == 0 ? 0u : ((s >> 2) & 3u) == 1 ? 0x7fffffu : (c & 0x7fffffu);
    nx = __uint_as_float((c & 0x80000000u) | ((uint32_t)ne[(b >> 8) % 6u] << 23) | m);
    ny = with_exp((uint32_t)h2, ne[(b >> 16) % 6u]);
  } else {
    d = fabsf(with_exp(a, 115 + (int)(b % 25u)));             // 2^-12 .. 2^12
    nx = with_exp(c, 100 + (int)(s % 40u));                    // up to 2^12
    ny = with_exp((uint32_t)h2, 100 + (int)((h2 >> 32) % 40u));
  }
}
__device__ __forceinline__ bool same(float x, float y) {   // bitwise, any NaN equal to any NaN
  return __float_as_uint(x) == __float_as_uint(y) || (x != x && y != y);
}
// fast[0]: scalar fast-path operands, fast[1]: pairs that took the packed fast path
__global__ void k_check(int mode, uint64_t n, uint64_t seed, unsigned long long* bad, unsigned long long* fast,
                        float* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float nx, ny, d;
    operands(mode, i, seed, nx, ny, d);
    if (!(d > 0.0f)) continue;   // the projection divides only when c_w > 0
    float qx, qy;
    ff_div2(nx, ny, d, qx, qy);
    const float rx = ieee_div(nx, d), ry = ieee_div(ny, d);
    const uint32_t md = __float_as_uint(d);
    if (md - 0x21800000u <= 0x5D800000u - 0x21800000u && ff_div_num_ok(nx) && ff_div_num_ok(ny)) atomicAdd(fast, 1ull);
    if (!same(qx, rx) || !same(qy, ry)) {
      if (atomicAdd(bad, 1ull) == 0ull) { first[0] = nx; first[1] = ny; first[2] = d; }
    }
    // the packed pair (ff_div2_pair): lane 0 = these operands, lane 1 = those of index i + n
    float nx1, ny1, d1;
    operands(mode, i + n, seed, nx1, ny1, d1);
    if (!(d1 > 0.0f)) continue;
    float2 px, py;
    if (ff_div2_pair(make_float2(nx, nx1), make_float2(ny, ny1), make_float2(d, d1), make_float2(1.0f, 1.0f), px, py)) {
      atomicAdd(fast + 1, 1ull);
      if (!same(px.x, rx) || !same(py.x, ry) || !same(px.y, ieee_div(nx1, d1)) || !same(py.y, ieee_div(ny1, d1))) {
        if (atomicAdd(bad, 1ull) == 0ull) { first[0] = nx1; first[1] = ny1; first[2] = d1; }
      }
    }
  }
}
extern "C" int div_check(int mode, unsigned long long n, unsigned long long seed, unsigned long long* out) {
  unsigned long long* dv;
  float* f;
  if (cudaMalloc(&dv, 3 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  if (cudaMalloc(&f, 3 * sizeof(float)) != cudaSuccess) return 1;
  cudaMemset(dv, 0, 3 * sizeof(unsigned long long));
  cudaMemset(f, 0, 3 * sizeof(float));
  k_check<<<148 * 8, 256>>>(mode, n, seed, dv, dv + 1, f);
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  float hf[3];
  unsigned long long cnt[3];
  cudaMemcpy(cnt, dv, sizeof cnt, cudaMemcpyDeviceToHost);
  out[0] = cnt[0]; out[1] = cnt[1]; out[5] = cnt[2];
  cudaMemcpy(hf, f, sizeof hf, cudaMemcpyDeviceToHost);
  for (int k = 0; k < 3; ++k) { uint32_t u; memcpy(&u, &hf[k], 4); out[2 + k] = u; }
  cudaFree(dv);
  cudaFree(f);
  return 0;
}
