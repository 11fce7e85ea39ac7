// Stand-alone check of a tcgen05 int8 GEMM tile (kind::i8, K-major SWIZZLE_NONE operands in
// shared memory, s32 accumulator in TMEM) against a CPU reference.  Development tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8gemm_test i8gemm_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous); tile [row/8][k/16][row%8][16]
// LBO = byte distance of K-adjacent core matrices, SBO = of row-adjacent 8-row groups
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}
// instruction descriptor: dense, s32 accumulator (c_format 2), a/b signed int8 (format 1), K-major
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int TM = 128, TN = 128, TK = 32;

// C[M][N] (row-major int32) = A[M][K] (row-major int8) * B[N][K]^T (row-major int8)
__global__ void __launch_bounds__(128) k_i8gemm(const int8_t* A, const int8_t* B, int32_t* C, int M, int N, int K) {
  __shared__ __align__(1024) int8_t sA[TM * TK];
  __shared__ __align__(1024) int8_t sB[TN * TK];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(TM, TN);
  uint32_t phase = 0;
  for (int k0 = 0; k0 < K; k0 += TK) {
    // stage: element (row, k) -> [row/8][k/16][row%8][k%16]
    for (int i = tid; i < TM * TK; i += 128) {
      const int row = i / TK, k = i % TK;
      const int off = ((row >> 3) * 2 + (k >> 4)) * 128 + (row & 7) * 16 + (k & 15);
      sA[off] = (m0 + row < M) ? A[(size_t)(m0 + row) * K + k0 + k] : 0;
      sB[off] = (n0 + row < N) ? B[(size_t)(n0 + row) * K + k0 + k] : 0;
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint64_t da = make_desc(smem_u32(sA), 128, 256), db = make_desc(smem_u32(sB), 128, 256);
      const uint32_t acc = k0 > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMA before the shared tiles are overwritten
    asm volatile(
        "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(&bar)), "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n");
  }
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 8 columns per load
  for (int c0 = 0; c0 < TN; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    const int row = m0 + 32 * warp + lane;
    for (int j = 0; j < 8; ++j)
      if (row < M && n0 + c0 + j < N) C[(size_t)row * N + n0 + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TN));
}

int main() {
  const int M = 256, N = 256, K = 512;
  std::vector<int8_t> A((size_t)M * K), B((size_t)N * K);
  srand(7);
  for (auto& x : A) x = (int8_t)((rand() % 128) - 64);
  for (auto& x : B) x = (int8_t)((rand() % 128) - 64);
  int8_t *dA, *dB;
  int32_t* dC;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, (size_t)M * N * 4);
  k_i8gemm<<<dim3(N / TN, M / TM), 128>>>(dA, dB, dC, M, N, K);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> C((size_t)M * N);
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[(size_t)i * K + k] * B[(size_t)j * K + k];
      if (s != C[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): got %d want %ld\n", i, j, C[(size_t)i * N + j], s);
        ++bad;
      }
    }
  printf("mismatches: %ld of %d\n", bad, M * N);
  return bad != 0;
}
