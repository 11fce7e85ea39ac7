// tcgen05.mma kind::i8 issue-rate microbenchmark: MACs/s per SM for M = 128 and several N
// (one CTA per SM, one elected thread issues R MMAs back to back on the same smem tiles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

template <int N>
__global__ void __launch_bounds__(128) k_rate(int reps, unsigned long long* cyc) {
  __shared__ __align__(1024) int8_t sA[128 * 32];
  __shared__ __align__(1024) int8_t sB[256 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32; i += 128) sA[i] = (int8_t)(i & 7);
  for (int i = tid; i < 256 * 32; i += 128) sB[i] = (int8_t)(i & 5);
  constexpr int COLS = N < 32 ? 32 : N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    const uint64_t da = make_desc(smem_u32(sA), 128, 256), db = make_desc(smem_u32(sB), 128, 256);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t acc = r > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred done;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t@!done bra W_%=;\n\t}\n" ::"r"(smem_u32(&bar)));
    const long long t1 = clock64();
    atomicAdd(cyc, (unsigned long long)(t1 - t0));
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(COLS));
}

template <int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  const int reps = 20000, ctas = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_rate<N><<<ctas, 128>>>(100, d);
  cudaDeviceSynchronize();
  cudaMemset(d, 0, 8);
  cudaEventRecord(e0);
  k_rate<N><<<ctas, 128>>>(reps, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)ctas * reps * 128.0 * N * 32.0;
  printf("{\"M\": 128, \"N\": %d, \"K\": 32, \"err\": \"%s\", \"ms\": %.3f, \"macs_per_s\": %.4e, \"cycles_per_mma\": %.2f}\n", N,
         cudaGetErrorString(err), ms, macs / (ms * 1e-3), (double)c / ctas / reps);
  cudaFree(d);
}

int main() {
  run<8>();
  run<16>();
  run<32>();
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
