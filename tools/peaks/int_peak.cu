// Integer-pipe / FP64-pipe throughput microbenchmark for the limb-MAC roofline
// (SURVEY.md §8(d) "Peak P_int: measure it on the box").
//
// Each thread runs NACC independent multiply-accumulate chains for ITERS
// iterations; the grid covers every SM several times.  Reported: operations
// per second for
//   imad_wide_s32 : int64 += (int64)int32 * int32     (SASS IMAD.WIDE)
//   imad_wide_u32 : uint64 += (uint64)uint32 * uint32 (SASS IMAD.WIDE.U32)
//   imad_lo       : uint32 = a*b + c                  (SASS IMAD)
//   dfma          : double = a*b + c                  (SASS DFMA)
//   mix           : one IMAD.WIDE and one DFMA per step (do the pipes co-issue?)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NACC 8
__device__ __forceinline__ int64_t madw(int32_t a, int32_t b, int64_t c){ int64_t d; asm volatile("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c)); return d; }
#define ITERS 4096

__global__ void k_wide_s32(int64_t* out, int32_t b, int seed) {
  int64_t acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 131 + i + seed;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      acc[i] = madw((int32_t)acc[(i + 1) % NACC], b, acc[i]);
  }
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= acc[i];
  if (s == 0x1234567) out[0] = s;
}

__global__ void k_wide_u32(uint64_t* out, uint32_t b, int seed) {
  uint64_t acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 131 + i + seed;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      acc[i] = (uint64_t)(uint32_t)acc[(i + 1) % NACC] * (uint64_t)b + acc[i];
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= acc[i];
  if (s == 0x1234567) out[0] = s;
}

__global__ void k_lo(uint32_t* out, uint32_t b, int seed) {
  uint32_t acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 131 + i + seed;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = acc[(i + 1) % NACC] * b + acc[i];
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= acc[i];
  if (s == 0x1234567) out[0] = s;
}

__global__ void k_dfma(double* out, double b, int seed) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3 + i + seed;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fma(acc[(i + 1) % NACC], b, acc[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 0.123) out[0] = s;
}

__global__ void k_mix(double* out, int64_t* out2, double b, int32_t bi, int seed) {
  double acc[NACC];
  int64_t iacc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i] = threadIdx.x * 1e-3 + i + seed; iacc[i] = threadIdx.x + i + seed; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      acc[i] = fma(acc[(i + 1) % NACC], b, acc[i]);
      iacc[i] = madw((int32_t)iacc[(i + 1) % NACC], bi, iacc[i]);
    }
  }
  double s = 0; int64_t si = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) { s += acc[i]; si ^= iacc[i]; }
  if (s == 0.123) out[0] = s;
  if (si == 0x1234567) out2[0] = si;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  void* buf; cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256;
  const char* names[] = {"imad_wide_s32", "imad_wide_u32", "imad_lo", "dfma", "mix_imadwide_plus_dfma"};
  printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk);
  for (int kind = 0; kind < 5; kind++) {
    double best = 1e30;
    int blocks = sms * 8;
    for (int rep = 0; rep < 6; rep++) {
      cudaEventRecord(e0);
      switch (kind) {
        case 0: k_wide_s32<<<blocks, threads>>>((int64_t*)buf, 3, rep); break;
        case 1: k_wide_u32<<<blocks, threads>>>((uint64_t*)buf, 3u, rep); break;
        case 2: k_lo<<<blocks, threads>>>((uint32_t*)buf, 3u, rep); break;
        case 3: k_dfma<<<blocks, threads>>>((double*)buf, 1.0000001, rep); break;
        case 4: k_mix<<<blocks, threads>>>((double*)buf, (int64_t*)buf + 4, 1.0000001, 3, rep); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    double ops = (double)blocks * threads * ITERS * NACC * (kind == 4 ? 2 : 1);
    printf(", \"%s_ops_per_s\": %.4e, \"%s_ms\": %.4f", names[kind], ops / (best * 1e-3), names[kind], best);
  }
  cudaError_t err = cudaGetLastError();
  printf(", \"cuda_error\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
