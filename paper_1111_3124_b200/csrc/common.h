// Host-visible declarations shared by the translation units (capi.cu, state.cu,
// tier280.cu, tier512.cu).  Kernels are instantiated once per precision tier.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace mpsb {

constexpr int MAX_CHI = 256;
// then MPS_ENOCONV (a failed run reports MAX + 1 sweeps).  The oracle's textbook cyclic iteration
// stops at 60; the round-robin order needs up to ~1.3x its sweeps on
// strongly graded spectra (tests/test_gpu_graded.py: 53 vs 41, 56 vs 53), hence 120 here.
constexpr int JACOBI_MAX_SWEEPS = 120;
// precision tiers: L = radix-2^28 digits of the Jacobi format (W = 28L bits >= p),
// NL = u32 limbs of the scalar mpf format (one guard limb above the record width)
struct Tier280 { static constexpr int L = 10, NL = 10; };
struct Tier512 { static constexpr int L = 19, NL = 17; };

// Opt the kernel `kern` in to `bytes` of dynamic shared memory on the CURRENT device, once
// per (kernel, device, size); thread-safe.  The attribute is per device, so a process-wide
// "done" flag would leave a second device without it (its launches would then fail).
cudaError_t smem_optin(const void* kern, int bytes);
// Grow-only device scratch of the tensor-core GEMM path per (device, stream): GEMMs on
// different streams (the three-site side streams) never share it; null if cudaMalloc fails.
void* tc_scratch(size_t bytes, cudaStream_t st);
// the tensor-core GEMM path (tcgemm.cuh) is on unless MPS_TC=0 (A/B measurements)
bool tc_enabled();

inline int record_words(int p) { return 4 + (p + 31) / 32; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct BatchOut {  // device pointers (records unless stated)
  uint32_t* sigma; int* k; uint32_t* A_out; uint32_t* B_out; uint32_t* lam; int* sweeps;
  uint32_t* theta_dbg; int* status;
};

// Optional CUDA-event bracketing of individual kernels (bench.py roofline): which = kernel id.
enum { PROF_JACOBI = 0, PROF_CONTRACT = 1, PROF_FINALIZE = 2, PROF_PRECOND = 3, PROF_RECOVER = 4,
       PROF_JDB = 5,    // k_jacobi_db (inside PROF_PRECOND)
       PROF_XS = 6,     // refinement sweeps k_xs_params + k_xs_apply (inside PROF_PRECOND)
       PROF_TCMMA = 7,  // every k_tc_mma launch (inside the classes above)
       PROF_JSP = 8,    // binary32 phase of the block Jacobi + hand-over (inside PROF_PRECOND, R27)
       PROF_N = 9 };
// device counters of the profiling run (mps_profile_counts_n): [0] p-bit rotations, [1] pair
// evaluations, [2] norm-pass sweeps x M x N, [3] recovery N^2 M, [4] phase-U digit products x M,
// [5] certified stops, [6] algorithmic DFMA of k_jacobi_db, [7] int8 MACs issued by k_tc_mma
enum { CNT_JDB_DFMA = 6, CNT_TC_MAC = 7, CNT_JSP_FFMA = 8, CNT_N = 16 };
void prof_mark(int which, int begin, cudaStream_t st);
// device buffer of 4 running totals while profiling is on (else null), see k_accum_stats
unsigned long long* prof_counts();

template <class T>
int launch_update2_batch(int p, int chi, int chi_max, int batch, double thr, const uint32_t* A,
                         const uint32_t* B, const uint32_t* lam_l, const uint32_t* lam_m,
                         const uint32_t* lam_r, const uint32_t* U, const BatchOut& out, void* ws,
                         cudaStream_t st, std::vector<unsigned char>& hostdesc);
template <class T>
size_t update2_workspace(int chi, int batch);
template <class T>
size_t svd_workspace(int M, int N, int batch);
template <class T>
int run_svd_batch(int p, int M, int N, int batch, const uint32_t* dR, uint32_t* dsig, int* dsweeps, int* ddbg,
                  void* ws, cudaStream_t st, std::vector<unsigned char>& hd);
template <class T>
void run_debug_mpf(int p, int op, int n, const uint32_t* a, const uint32_t* b, uint32_t* out, cudaStream_t st);

}  // namespace mpsb
