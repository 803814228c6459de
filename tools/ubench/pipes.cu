// Pipe-throughput microbenchmarks for B200 (sm_100a), SURVEY.md Appendix B items B1-B5.
// One CTA of 1024 threads per SM (grid = #SMs), so ops / SM-cycle of one CTA is the
// per-SM rate. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int ITERS = 4096;
constexpr int NACC = 8;

__global__ void k_ffma_reg(const float* __restrict__ in, float* out, long long* cyc) {
  float b = in[0], c = in[1];
  float a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = in[2 + i] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = fmaf(a[i], b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Each accumulator uses its own multiplier/addend registers: 3 distinct regs per FFMA.
__global__ void k_ffma_reg3(const float* __restrict__ in, float* out, long long* cyc) {
  float a[NACC], b[NACC], c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { a[i] = in[2 + i] + threadIdx.x; b[i] = in[i & 1] + i * 1e-7f; c[i] = in[1 - (i & 1)] * (1.f + i * 1e-7f); }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = fmaf(a[i], b[i], c[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(const float* __restrict__ in, float* out, long long* cyc) {
  float2 b = make_float2(in[0], in[0] * 1.0000001f), c = make_float2(in[1], in[1] * 0.9999999f);
  float2 a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = make_float2(in[2 + i] + threadIdx.x, in[2 + i] - threadIdx.x);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = __ffma2_rn(a[i], b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_fadd(const float* __restrict__ in, float* out, long long* cyc) {
  float b = in[0];
  float a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = in[2 + i] + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = a[i] + b;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcp(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

// 32 x 32 -> 64-bit multiply (IMAD.WIDE.U32) + 3-input XOR: one Philox4x32 half-round, the reset
// redraw's inner loop (what a reset costs)
__global__ void k_imadwide(const float* __restrict__ in, float* out, long long* cyc) {
  unsigned a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = __float_as_uint(in[2 + i]) + threadIdx.x * 7919u + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const unsigned long long p = (unsigned long long)a[i] * 0xD2511F53ull;
      a[i] = (unsigned)(p >> 32) ^ (unsigned)p ^ 0x9E3779B9u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2(const float* __restrict__ in, float* out, long long* cyc) {
  float a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = in[2 + i] * 1e-3f + threadIdx.x * 1e-6f;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = ex2(a[i]) ;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_rcp(const float* __restrict__ in, float* out, long long* cyc) {
  float a[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = in[2 + i] + 1.f + threadIdx.x * 1e-6f;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    // rcp(rcp(a)) = a let ptxas drop the whole chain (r01 printed ~4e6 lane-ops/clk); one FFMA per
    // reciprocal keeps it a chain (the FMA pipe has 8x the MUFU's throughput, so MUFU still binds)
    for (int i = 0; i < NACC; ++i) a[i] = rcp(fmaf(a[i], 0.5f, 1.0f));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// FFMA and EX2 interleaved 4:1 -- do the pipes overlap?
__global__ void k_mix(const float* __restrict__ in, float* out, long long* cyc) {
  float b = in[0], c = in[1];
  float a[NACC], e[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { a[i] = in[2 + i] + threadIdx.x; e[i] = in[2 + i] * 1e-3f; }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      a[i] = fmaf(a[i], b, c); a[i] = fmaf(a[i], b, c); a[i] = fmaf(a[i], b, c); a[i] = fmaf(a[i], b, c);
      e[i] = ex2(e[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i] + e[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Global atomics: every thread adds 1 to bin (gid % nbins) * stride, `reps` times.
__global__ void k_red(unsigned* img, int nbins, int reps, int aggregate) {
  long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    unsigned bin = (unsigned)((gid * 2654435761ull + r * 97) % nbins);
    if (aggregate) {
      unsigned peers = __match_any_sync(0xffffffffu, bin);
      int leader = __ffs(peers) - 1;
      if ((int)(threadIdx.x & 31) == leader) atomicAdd(img + bin, (unsigned)__popc(peers));
    } else {
      atomicAdd(img + bin, 1u);
    }
  }
}


// Packed FP32 with per-accumulator operands (no shared registers): does operand-register read
// bandwidth limit FFMA2 / FADD2 / FMUL2 the way it limits FFMA(3reg)?
#define PACKED_KERNEL(NAME, INIT, BODY)                                                             \
  __global__ void NAME(const float* __restrict__ in, float* out, long long* cyc) {                  \
    float2 a[NACC], b[NACC], c[NACC];                                                             \
    _Pragma("unroll") for (int i = 0; i < NACC; ++i) {                                             \
      a[i] = make_float2(in[2 + i] + threadIdx.x, in[2 + i] - threadIdx.x);                        \
      b[i] = make_float2(in[0] * (1.f + i * 1e-7f), in[0] * (1.f - i * 1e-7f));                    \
      c[i] = make_float2(in[1] * (1.f + i * 1e-7f), in[1] * (1.f - i * 1e-7f));                    \
      INIT;                                                                                        \
    }                                                                                              \
    __syncthreads();                                                                               \
    long long t0 = clock64();                                                                      \
    _Pragma("unroll 4") for (int it = 0; it < ITERS; ++it) {                                       \
      _Pragma("unroll") for (int i = 0; i < NACC; ++i) BODY;                                       \
    }                                                                                              \
    __syncthreads();                                                                               \
    long long t1 = clock64();                                                                      \
    float s = 0.f;                                                                                 \
    _Pragma("unroll") for (int i = 0; i < NACC; ++i) s += a[i].x + a[i].y;                         \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                                \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                               \
  }
PACKED_KERNEL(k_ffma2_3reg, (void)0, a[i] = __ffma2_rn(a[i], b[i], c[i]))
PACKED_KERNEL(k_ffma2_2reg, (void)0, a[i] = __ffma2_rn(a[i], b[i], make_float2(0.5f, 0.5f)))
PACKED_KERNEL(k_fadd2_2reg, c[i] = make_float2(-c[i].x * 1e-9f, c[i].y * 1e-9f), a[i] = __fadd2_rn(a[i], c[i]))
// scalar broadcast operand from a per-thread register (R.F32) vs a kernel parameter (UR / constant)
PACKED_KERNEL(k_ffma2_rscalar, b[i] = make_float2(1.0f + threadIdx.x * 1e-9f + i * 1e-8f, 0.f),
              a[i] = __ffma2_rn(make_float2(b[i].x, b[i].x), a[i], c[i]))
PACKED_KERNEL(k_fmul2_2reg, b[i] = make_float2(1.0000001f, 0.9999999f), a[i] = __fmul2_rn(a[i], b[i]))
// operand kinds of the HH ring loop: one pair + a per-thread register scalar + an
// immediate (c1 v + c2 with c1 in a register), one pair + two register scalars (q-table constants
// that ptxas kept in registers), two pairs + a register scalar per accumulator
PACKED_KERNEL(k_ffma2_p1r1k, b[i] = make_float2(0.999f + threadIdx.x * 1e-9f + i * 1e-8f, 0.f),
              a[i] = __ffma2_rn(a[i], make_float2(b[i].x, b[i].x), make_float2(0.25f, 0.25f)))
PACKED_KERNEL(k_ffma2_p1r2, (b[i] = make_float2(0.999f + threadIdx.x * 1e-9f + i * 1e-8f, 0.f),
                             c[i] = make_float2(0.25f + threadIdx.x * 1e-9f, 0.f)),
              a[i] = __ffma2_rn(a[i], make_float2(b[i].x, b[i].x), make_float2(c[i].x, c[i].x)))

typedef void (*kfn)(const float*, float*, long long*);

static double run(const char* name, kfn k, double ops_per_thread_iter, int iters, int nsm, int threads,
                  float* din, float* dout, long long* dcyc) {
  k<<<nsm, threads>>>(din, dout, dcyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<nsm, threads>>>(din, dout, dcyc);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = (long long*)malloc(sizeof(long long) * nsm);
  CK(cudaMemcpy(h, dcyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
  double mean = 0; long long mx = 0;
  for (int i = 0; i < nsm; ++i) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
  mean /= nsm;
  double per_sm_clk = threads * (double)iters * ops_per_thread_iter / mean;
  double total = (double)nsm * threads * iters * ops_per_thread_iter;
  printf("%-12s lane-ops/clk/SM = %7.1f   wall %.3f ms  -> %.3e lane-ops/s  (implied clk %.0f MHz)\n",
         name, per_sm_clk, ms, total / (ms * 1e-3), mean / (ms * 1e-3) / 1e6);
  free(h);
  return per_sm_clk;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0, l2 = 0, smemoptin = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&smemoptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int drv = 0, rt = 0; cudaDriverGetVersion(&drv); cudaRuntimeGetVersion(&rt);
  printf("device %s cc %d.%d SMs %d clockRate %d kHz memClock %d kHz L2 %d B smemOptin %d B regs/SM %d driver %d runtime %d\n",
         p.name, p.major, p.minor, p.multiProcessorCount, clk, memclk, l2, smemoptin, p.regsPerMultiprocessor, drv, rt);
  int nsm = p.multiProcessorCount;
  float hin[16]; for (int i = 0; i < 16; ++i) hin[i] = 0.999f + 1e-4f * i;
  hin[0] = 0.9999999f; hin[1] = 1e-7f;
  float *din, *dout; long long* dcyc;
  CK(cudaMalloc(&din, 64)); CK(cudaMalloc(&dout, sizeof(float) * nsm * 1024)); CK(cudaMalloc(&dcyc, sizeof(long long) * nsm));
  CK(cudaMemcpy(din, hin, 64, cudaMemcpyHostToDevice));
  for (int rep = 0; rep < 2; ++rep) {
    run("FFMA(b,c)", k_ffma_reg, NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA(3reg)", k_ffma_reg3, NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2", k_ffma2, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FADD", k_fadd, NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2(3reg)", k_ffma2_3reg, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2(2reg+k)", k_ffma2_2reg, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FADD2(2reg)", k_fadd2_2reg, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FMUL2(2reg)", k_fmul2_2reg, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2(Rscal)", k_ffma2_rscalar, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2(p1r1k)", k_ffma2_p1r1k, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("FFMA2(p1r2)", k_ffma2_p1r2, 2 * NACC, ITERS, nsm, 1024, din, dout, dcyc);
    run("MUFU.EX2", k_ex2, NACC, ITERS / 4, nsm, 1024, din, dout, dcyc);
    run("IMAD.WIDE", k_imadwide, NACC, ITERS / 4, nsm, 1024, din, dout, dcyc);
    run("MUFU.RCP", k_rcp, NACC, ITERS / 4, nsm, 1024, din, dout, dcyc);
    run("FFMA4+EX2", k_mix, 5 * NACC, ITERS / 4, nsm, 1024, din, dout, dcyc);
  }
  // atomics
  unsigned* img; size_t nimg = 1 << 22; CK(cudaMalloc(&img, nimg * 4));
  int nthreads = 8 << 20; int reps = 4;
  int bins_list[] = {1, 2, 64, 1 << 20, 1 << 22};
  for (int agg = 0; agg < 2; ++agg)
    for (int bi = 0; bi < 5; ++bi) {
      int nb = bins_list[bi];
      cudaMemset(img, 0, nimg * 4);
      k_red<<<nthreads / 256, 256>>>(img, nb, 1, agg);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_red<<<nthreads / 256, 256>>>(img, nb, reps, agg);
      cudaEventRecord(e1); CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("atomics agg=%d bins=%8d: %.3f ms for %d increments -> %.3e incr/s\n", agg, nb, ms, nthreads * reps,
             nthreads * (double)reps / (ms * 1e-3));
    }
  return 0;
}
