// Do histogram REDs overlap with state streaming? (the S = 1 frame.) 8.4 M "particles":
// stream 3 x float2 per thread-pair in and out (201 MB, like the Lorenz state) and/or issue one
// red.relaxed.gpu.add per particle to a pseudo-random word of an 8 MiB image (2 M words, L2-resident).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o red_stream tools/ubench/red_stream.cu && ./red_stream
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_add(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
// mode bit 0: stream the state; bit 1: one RED per particle (2 per thread)
__global__ void k(float2* s0, float2* s1, float2* s2, unsigned* img, long long npairs, unsigned words, int mode,
                  unsigned salt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npairs; i += (long long)gridDim.x * blockDim.x) {
    if (mode & 1) {
      float2 a = __ldcs(s0 + i), b = __ldcs(s1 + i), c = __ldcs(s2 + i);
      a.x += 1.0f; b.y += 1.0f; c.x += a.y;
      __stcs(s0 + i, a); __stcs(s1 + i, b); __stcs(s2 + i, c);
    }
    if (mode & 2) {
      red_add(img + hash((unsigned)(2 * i) ^ salt) % words, 1u);
      red_add(img + hash((unsigned)(2 * i + 1) ^ salt) % words, 1u);
    }
  }
}
int main() {
  const long long n = 1 << 23, npairs = n / 2;
  const unsigned words = 2u << 20;
  float2 *s0, *s1, *s2; unsigned* img; char* flush;
  cudaMalloc(&s0, npairs * 8); cudaMalloc(&s1, npairs * 8); cudaMalloc(&s2, npairs * 8);
  cudaMalloc(&img, words * 4ull); cudaMalloc(&flush, 256 << 20);
  cudaMemset(s0, 0, npairs * 8); cudaMemset(s1, 0, npairs * 8); cudaMemset(s2, 0, npairs * 8); cudaMemset(img, 0, words * 4ull);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[4] = {"", "stream only", "REDs only  ", "stream+REDs"};
  for (int blocks_per_sm : {8, 16}) {
    for (int mode = 1; mode <= 3; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 10; ++rep) {
        cudaMemset(flush, rep, 256 << 20);   // evict the state from L2
        cudaEventRecord(e0);
        k<<<nsm * blocks_per_sm, 128>>>(s0, s1, s2, img, npairs, words, mode, rep * 7919u);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 1 && ms < best) best = ms;
      }
      printf("%2d blocks/SM x 128: %s %7.1f us   (%.3g REDs/s, %.0f GB/s state)\n", blocks_per_sm, names[mode],
             best * 1e3, (mode & 2) ? n / (best * 1e-3) : 0.0, (mode & 1) ? 48.0 * npairs / (best * 1e-3) / 1e9 : 0.0);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
