// Mixed-precision preconditioning of the one-sided Jacobi SVD (R19).
//
//   Theta' (fixed point, p bits)  --k_fx_to_d-->  Theta_d (binary64, scaled by 2^-e)
//   one-sided block Jacobi on Theta_d, first in binary32, then in binary64 (R27)
//                                                -->  V_d  (unitary to ~1e-14)
//   X_0 = V_d (exact digits), Newton-Schulz in fixed point:
//       D_k = I - X_k^H X_k,   X_{k+1} = X_k + X_k D_k / 2        (quadratic: 2^-45 -> 2^-90 -> ...)
//   A_1 = Theta' X   (exactly unitary X to the working precision)
//   the p-bit Jacobi (k_jacobi) then starts from columns orthogonal to ~1e-14 and needs
//   ~4 sweeps instead of ~16.  V is recovered from Theta' as before (R16), or accumulated
//   starting from X (V = X W).
// The binary64 stage only chooses the starting basis; every p-bit quantity comes from exact
// fixed-point arithmetic, so the result is the p-bit SVD of Theta' (the oracle's, to tau).
#pragma once
#include <cstdint>

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace mpsb {

struct PreItem {
  int M, N;
  const int32_t* A0; const int64_t* eA0;  // Theta' (M x N, block exponent)
  double2* Ad;                            // [N][M] column-major complex binary64
  double2* Vd;                            // [N][N]
  unsigned long long* rowmax;             // max_r sum_c |Ad(r,c)|^2 as ordered bits (1)
  int* sweeps_d;                          // binary64 sweeps (1)
  int32_t* X;                             // N x N fixed, exponent 1 (output of k_d_to_fx)
  int64_t* eOne;                          // [2] = {1, 0}: exponents of X and of D/2
  int64_t* eA1;                           // exponent chosen for A_1 = Theta' X (1)
  int* anyflag;                           // [2] "some block pair rotated" per sweep parity (cluster mode)
  unsigned long long* offmax;             // [2] largest |gamma|^2 / (alpha_p alpha_q) per sweep parity (bits)
  // refinement sweep (xsweep.cuh, R22): X_1 (rotated in place), G = A_t^H A_t and its
  // exponent, the rotation records; X1 == nullptr: no refinement sweep for this item
  int32_t* X1; const int32_t* G; const int64_t* eG; int4* xs_rec;
  unsigned long long* cnt;  // profiling counters (CNT_*), or null
  // GEMM form of the refinement sweeps (R26): exponents {0, -1} of E and E/2; per sweep
  // the number of pairs applied as sequential exact rotations (the others enter E)
  int64_t* eXs; int* xs_big;
  // binary32 first phase of the block Jacobi (R27): As, Vs its matrices (null: no such
  // phase), V0 = binary64 copy of Vs, Rm = V0^H V0, Aj = Theta_d V_d (the binary64 phase then runs
  // on Aj with V preset in Vd), sweeps_s its sweep count
  float2* As; float2* Vs; double2* V0; double2* Rm; double2* Aj; int* sweeps_s;
  int* sp_bad;  // [1] set when the binary32 phase left a V that is not unitary to 1e-6 after one Newton-Schulz step
};

static __global__ void k_pre_init(const PreItem* items, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) *items[b].rowmax = 0ull;
}

// binary64 value of an L-digit fixed number times 2^-e (its top three digits)
template <int L>
__device__ __forceinline__ double fx_top_double(const int32_t* p, size_t ld) {
  const double t = (double)p[(size_t)(L - 1) * ld] * 72057594037927936.0 +  // 2^56
                   (double)p[(size_t)(L - 2) * ld] * 268435456.0 + (double)p[(size_t)(L - 3) * ld];
  return ldexp(t, -84);  // value * 2^-e = sum d_k 2^(28k - 28L)
}

template <int L>
__global__ void k_fx_to_d(const PreItem* items) {
  const PreItem it = items[blockIdx.y];
  const int M = it.M, N = it.N;
  if (N == 0) return;
  double rmax = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < N; ++c) {
      const int32_t* pr = it.A0 + ((size_t)(c * 2 + 0) * L) * M + r;
      const int32_t* pi = it.A0 + ((size_t)(c * 2 + 1) * L) * M + r;
      const double2 v = make_double2(fx_top_double<L>(pr, M), fx_top_double<L>(pi, M));
      it.Ad[(size_t)c * M + r] = v;
      s += v.x * v.x + v.y * v.y;
    }
    rmax = fmax(rmax, s);
  }
  atomicMax(it.rowmax, (unsigned long long)__double_as_longlong(rmax));
}

// all-reduce of four sums in 6 shuffles instead of 20: the first two levels exchange half of
// the values (each lane keeps the pair / the value its lane bits select), then a plain
// butterfly; finally every lane fetches the four totals from lanes 0..3
template <typename T>
__device__ __forceinline__ void warp_sum4_d(T& a, T& b, T& c, T& d) {
  const int lane = threadIdx.x & 31;
  const bool h16 = lane & 16, h8 = lane & 8;
  // level 16: keep (a, b) if bit 4 clear else (c, d)
  T x0 = h16 ? c : a, x1 = h16 ? d : b;
  const T y0 = h16 ? a : c, y1 = h16 ? b : d;
  x0 += __shfl_xor_sync(0xffffffffu, y0, 16);
  x1 += __shfl_xor_sync(0xffffffffu, y1, 16);
  // level 8: keep x0 if bit 3 clear else x1
  T z = h8 ? x1 : x0;
  z += __shfl_xor_sync(0xffffffffu, h8 ? x0 : x1, 8);
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
  // lane with bits (4, 3) = (i1, i0) holds total number 2 i1 + i0: a = 0, b = 1, c = 2, d = 3
  a = __shfl_sync(0xffffffffu, z, 0);
  b = __shfl_sync(0xffffffffu, z, 8);
  c = __shfl_sync(0xffffffffu, z, 16);
  d = __shfl_sync(0xffffffffu, z, 24);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// One-sided Jacobi in binary64 (V_d accumulated), blocked: one CTA (or cluster) per item;
// the columns are split into blocks of bs (16; 8 when M > 320; 4 when M > 640) and block pairs
// are visited round-robin; each block pair's 2bs columns are staged in shared memory and given
// one inner round-robin sweep of pair rotations accumulated in a 2bs x 2bs W, then
// A[:, block pair] and V[:, block pair] are multiplied by W.  HBM/L2 traffic per outer sweep is
// O(N M N/bs) instead of O(N^2 M) for a warp-per-pair kernel on global memory.
// Inner sweep, two forms (the rotation formula and the pair order are the same):
//  * Gram form (while the previous sweep still had a relative off-diagonal above JD_GRAM_OFF
//    and the block pair's column norms^2 are within 2^20 of each other): G = Ab^H Ab is formed
//    once (a 2bs x 2bs x M product) and the rotations are computed from and applied to G
//    (two-sided, G <- J^H G J) and W only; A's block columns are then Ab W.  The arithmetic
//    per pair drops from O(M) to O(bs), but G's rounding is relative to the largest column,
//    so the late sweeps (small off-diagonals) use
//  * the column form: every pair's dots are taken from the (rotated) columns in shared memory.
// Stops when a sweep rotates no pair (|gamma| > tol sqrt(alpha_p alpha_q), tol = 4 M 2^-53) —
// always decided on dots of the current columns (a Gram-form sweep that rotates nothing has
// not changed G, which equals those dots).  The binary64 stage only chooses the starting basis
// of the p-bit iteration (R19): no p-bit result depends on its rounding or on the form used.
// JD_BS_MAX caps the block size.  16 (default): 165 KB of shared memory, one CTA of 512 threads
// per SM.  8 keeps a CTA at 74 KB for M <= 320 (3 CTAs of 256 threads per SM overlap each other's
// barrier-bound inner steps) but doubles the inner steps: measured slower (configs[1] chi = 128:
// 132.7 vs 137.2 updates/s, preconditioner 2.78 vs 2.52 s per step; profiles/r02_jdb_bs8_ab.jsonl).
// The block size depends on M only, never on the batch, so a gate's result does not depend on
// which gates share its launch.
#ifndef JD_BS_MAX
#define JD_BS_MAX 16
#endif
__host__ __device__ inline int jd_bs(int M) {
  const int b = M <= 320 ? 16 : (M <= 640 ? 8 : 4);
  return b < JD_BS_MAX ? b : JD_BS_MAX;
}
constexpr int JD_THREADS = JD_BS_MAX >= 16 ? 512 : 256;  // the Gram phase needs bs (bs + 1) threads
constexpr int JD_MINB = JD_BS_MAX >= 16 ? 1 : 3;
#ifndef JD_TOL
#define JD_TOL (4.0 * M * 1.1102230246251565e-16)  // 4 M 2^-53 (1e-12 costs a p-bit sweep)
#endif  // one warp per pair of a block pair's inner step (bs <= 16)
#ifndef JD_CROSS  // 1: block pairs after the first step of a sweep rotate only their cross pairs
#define JD_CROSS 1
#endif
#ifndef JD_LAST_OFF
#define JD_LAST_OFF 1e-8  // a column-form sweep whose pairs were all below this is the last one
#endif
#ifndef JD_GRAM_OFF
#define JD_GRAM_OFF 1e-6  // Gram-form inner sweeps while max |gamma| / sqrt(alpha_p alpha_q) exceeds this
#endif
__host__ __device__ inline int jd_mp(int M) { return M | 1; }  // odd column stride: conflict-free Gram loads
// Gram phase: thread (tile, part) sums rows [part M / P, (part + 1) M / P) of one 2x2 tile of
// the bs (bs + 1) / 2 upper tiles; parts 1.. leave their partial sums in a scratch area
__host__ __device__ inline int jd_gram_parts(int bs) {
  const int TU = bs * (bs + 1) / 2, P = JD_THREADS / TU;
  return P < 1 ? 1 : (P > 4 ? 4 : P);
}
inline size_t jd_smem(int M, size_t el = 16) {  // el: bytes of a complex element (16 binary64, 8 binary32)
  const int bs = jd_bs(M), nc2 = 2 * bs;
  const size_t scr = (size_t)(jd_gram_parts(bs) - 1) * (bs * (bs + 1) / 2) * 4 * el;
  return (size_t)nc2 * jd_mp(M) * el + (size_t)nc2 * nc2 * el + (size_t)nc2 * (nc2 + 1) * el + scr + 64;
}

// MPS_JD_PROF=1 (debug): clock64 cycles of thread 0 per phase, summed over CTAs:
// [0] staging, [1] inner rotations, [2] A write-back, [3] V update, [4] block pairs, [5] sweeps,
// [6] block pairs in Gram form, [7] Gram products (cycles)
static __device__ unsigned long long jd_prof[8];
static __device__ int jd_prof_on;
static __device__ int jd_sp_maxsweeps = 40;  // debug (MPS_JD_SP_SWEEPS): cap of the binary32 phase

// Real type of the block Jacobi: binary64, or binary32 for the first phase (R27)
__device__ __forceinline__ double2 mk2(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ float2 mk2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double jd_rsqrt(double x) { return rsqrt(x); }
__device__ __forceinline__ float jd_rsqrt(float x) { return rsqrtf(x); }
// one complex element global -> shared (valid = 0: zero fill)
template <typename T2>
__device__ __forceinline__ void cp_async_el(void* smem, const void* gmem, bool valid) {
  if constexpr (sizeof(T2) == 16) {
    cp_async16(smem, gmem, valid ? 16 : 0);
  } else {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
  }
}
template <typename T> struct JdT;
template <> struct JdT<double> {
  using T2 = double2;
  static constexpr int MINB = JD_MINB;
  static constexpr double GRAM_OFF = JD_GRAM_OFF, STOP_OFF = 0.0, HUGE_ = 1.0e308, NORM_RATIO = 1048576.0;
  static __device__ __forceinline__ double2* A(const PreItem& it) { return it.Aj ? it.Aj : it.Ad; }
  static __device__ __forceinline__ double2* V(const PreItem& it) { return it.Vd; }
  static __device__ __forceinline__ double tol(int M) { return JD_TOL; }
  static __device__ __forceinline__ double thr(double tol, double sp, double sq) { return tol * tol * sp * sq; }
  static __device__ __forceinline__ bool ok(double, double) { return true; }
};
// binary32: Gram-form inner sweeps while a relative off-diagonal exceeds 2^-10 (G's rounding is
// 2^-24 of the largest column norm^2: norms^2 within 2^8; 2^10 measured slower: one more sweep), hand-over to binary64 once a whole sweep
// saw none above 2^-11 (its rotations leave ~2^-22, the binary32 floor eps sqrt(M) is ~2^-20)
template <> struct JdT<float> {
  using T2 = float2;
#ifndef JD_SP_MINB  // CTAs per SM of the binary32 phase (2: 64 registers per thread, 96 KB of shared memory each)
#define JD_SP_MINB 2
#endif
  static constexpr int MINB = JD_SP_MINB;
  #ifndef JD_SP_NORM_RATIO
#define JD_SP_NORM_RATIO 256.0f
#endif
  static constexpr float GRAM_OFF = 9.765625e-4f, STOP_OFF = 4.8828125e-4f, HUGE_ = 3.0e38f, NORM_RATIO = JD_SP_NORM_RATIO;
  static __device__ __forceinline__ float2* A(const PreItem& it) { return it.As; }
  static __device__ __forceinline__ float2* V(const PreItem& it) { return it.Vs; }
  static __device__ __forceinline__ float tol(int M) { return 4.0f * M * 5.9604645e-8f; }  // 4 M 2^-24
  static __device__ __forceinline__ float thr(float tol, float sp, float sq) { return (tol * sp) * (tol * sq); }
  // columns below 1e-15 of the largest (norms^2 below 1e-30 after k_d_to_s's scaling) are left to the
  // binary64 phase: their products underflow binary32
  static __device__ __forceinline__ bool ok(float sp, float sq) { return sp > 1e-30f && sq > 1e-30f; }
};

// dst[:, s_col[j]] = src (R rows, column stride ld, 2bs columns) x W  (thread: row r, half h)
template <typename T, typename T2>
__device__ __forceinline__ void jd_apply_w(const T2* src, int ld, T2* dst, int R, const T2* W, int bs,
                                           const int* s_col) {
  const int nc2 = 2 * bs;
  for (int t = threadIdx.x; t < 2 * R; t += blockDim.x) {
    const int r = t % R, h = t / R;
    T2 acc[JD_BS_MAX];
#pragma unroll
    for (int j = 0; j < JD_BS_MAX; ++j) acc[j] = mk2(T(0), T(0));
#pragma unroll 2
    for (int l = 0; l < nc2; ++l) {
      const T2 v = src[(size_t)l * ld + r];
#pragma unroll
      for (int j = 0; j < JD_BS_MAX; ++j) {
        if (j < bs) {
          const T2 w = W[(size_t)(h * bs + j) * nc2 + l];
          acc[j].x = fma(v.x, w.x, fma(-v.y, w.y, acc[j].x));
          acc[j].y = fma(v.x, w.y, fma(v.y, w.x, acc[j].y));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < JD_BS_MAX; ++j) {
      if (j < bs) {
        const int cj = s_col[h * bs + j];
        if (cj >= 0) dst[(size_t)cj * R + r] = acc[j];
      }
    }
  }
}

// rotation parameters of the oracle's formula (R17 form): d = alpha_q - alpha_p,
// r = sqrt(d^2 + 4|g|^2), c = sqrt((|d| + r) / 2r), s = sgn(d) g / (r c)
// (two reciprocal square roots, no division: 1/r, c^2 = (|d|/r + 1)/2, 1/c, s = sgn(d) g (1/r)(1/c))
template <typename T>
__device__ __forceinline__ void jd_rot(T sp, T sq, T gr, T gi, T g2, T& c, T& sr, T& si) {
  const T d = sq - sp;
  const T ir = jd_rsqrt(d * d + T(4) * g2);
  const T c2 = T(0.5) * fma(fabs(d), ir, T(1));
  const T ic = jd_rsqrt(c2);
  c = c2 * ic;
  const T sc = (d < 0 ? -ir : ir) * ic;
  sr = gr * sc;
  si = gi * sc;
}

// C CTAs (a thread-block cluster when C > 1) share one item: the block pairs of a step are
// dealt round-robin to the CTAs and the steps are separated by cluster barriers (few items in
// flight: an MPS layer).  The rotation sequence does not depend on C.
template <typename T>
__global__ void __launch_bounds__(JD_THREADS, JdT<T>::MINB) k_jacobi_blk(const PreItem* items, int C) {
  using T2 = typename JdT<T>::T2;
  constexpr bool SP = sizeof(T) == 4;  // the binary32 first phase (R27)
  namespace cg = cooperative_groups;
  const int crank = C > 1 ? (int)(blockIdx.x % C) : 0;
  const PreItem it = items[C > 1 ? blockIdx.x / C : blockIdx.x];
  auto csync = [&]() {
    if (C > 1) cg::this_cluster().sync();
    else __syncthreads();
  };
  const int M = it.M, N = it.N;
  if (N == 0) return;
  const int bs = jd_bs(M), nb = (N + bs - 1) / bs, nbe = nb + (nb & 1), nc2 = 2 * bs, MP = jd_mp(M);
  const int nh = bs;  // Gram: 2x2 tiles of entries (i, j), (i, j+bs), (i+bs, j), (i+bs, j+bs)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(16) unsigned char jds_raw[];
  T2* Ab = (T2*)jds_raw;              // [2bs][MP] block columns
  T2* W = Ab + (size_t)nc2 * MP;     // [2bs][2bs] column-major
  T2* G = W + (size_t)nc2 * nc2;      // [2bs][2bs + 1] row-major (Gram form)
  T2* Gs = G + (size_t)nc2 * (nc2 + 1);  // Gram partial sums of parts 1..P-1
  const int GL = nc2 + 1, lgc = __ffs(nc2) - 1;  // nc2 = 2^lgc
  __shared__ int s_any, s_rot, s_gram, s_col[32], s_ngram;
  __shared__ T s_c[16], s_sr[16], s_si[16];
  __shared__ int s_on[16], s_p[16], s_q[16];
  __shared__ unsigned long long s_off;  // max rel^2 = |g|^2 / (alpha_p alpha_q) of this CTA's sweep (bits)
  T2* A = JdT<T>::A(it);
  T2* V = JdT<T>::V(it);
  if (SP && A == nullptr) return;  // item without the binary32 phase
  if (SP || it.Aj == nullptr)      // (binary64 after a binary32 phase: V is preset, R27)
    for (int t = crank * blockDim.x + threadIdx.x; t < N * N; t += C * blockDim.x)
      V[t] = mk2((t % N) == (t / N) ? T(1) : T(0), T(0));
  const T tol = JdT<T>::tol(M);
  const bool prof = jd_prof_on && threadIdx.x == 0;
  long long tm = prof ? clock64() : 0;
  auto mark = [&](int k) {
    if (prof) {
      const long long t = clock64();
      atomicAdd(&jd_prof[k], (unsigned long long)(t - tm));
      tm = t;
    }
  };
  // 1.0 once this thread saw |g|^2 / (alpha_p alpha_q) > JD_GRAM_OFF^2 in the sweep (one atomic per
  // sweep; only that comparison is used, so no division on the rotation path)
  // (binary32 phase: 2.0 above its Gram-form threshold, 1.0 above the level it stops at)
  double off_t = 0.0;
  auto note_off = [&](T g2, T sp, T sq) {
    if (sp > 0 && sq > 0) {
      if (g2 > T(JdT<T>::GRAM_OFF * JdT<T>::GRAM_OFF) * (sp * sq)) off_t = SP ? 2.0 : 1.0;
      else if (SP && off_t < 1.0 && g2 > T(JdT<T>::STOP_OFF * JdT<T>::STOP_OFF) * (sp * sq)) off_t = 1.0;
      else if (!SP && off_t < 0.25 && g2 > T(JD_LAST_OFF * JD_LAST_OFF) * (sp * sq)) off_t = 0.25;
    }
  };
  int sweep = 0;
  const int maxsweeps = SP ? jd_sp_maxsweeps : 40;
  for (sweep = 1; sweep <= maxsweeps; ++sweep) {
    if (threadIdx.x == 0) { s_any = 0; s_off = 0ull; s_ngram = 0; }
    if (crank == 0 && threadIdx.x == 0) {
      *(volatile int*)&it.anyflag[sweep & 1] = 0;
      *(volatile unsigned long long*)&it.offmax[sweep & 1] = 0ull;
    }
    csync();
    // Gram-form sweep while the previous sweep's largest relative off-diagonal was big
    const bool gram_sweep =
        sweep == 1 || __longlong_as_double((long long)*(volatile unsigned long long*)&it.offmax[(sweep - 1) & 1]) >
                          (SP ? 1.5 : 0.5);  // flag levels of note_off
    for (int step = 0; step < nbe - 1; ++step) {
      for (int bp = crank; bp < nbe / 2; bp += C) {
        int I, J;
        rr_pair(nbe, step, bp, I, J);
        // local column l < bs: block I, l >= bs: block J; -1 = absent (ragged / dummy block)
        if (threadIdx.x < nc2) {
          const int l = threadIdx.x, blk = l < bs ? I : J, c = blk * bs + (l % bs);
          s_col[l] = (blk < nb && c < N) ? c : -1;
        }
        if (threadIdx.x == 0) { s_rot = 0; s_gram = 0; }
        // inner pair order: the first step of a sweep (its block pairs cover every block once)
        // visits all pairs of the 2bs columns (round-robin, 2bs - 1 steps), later steps only the
        // bs^2 cross pairs (i, bs + (i + s2) % bs), bs steps: every column pair is still met once
        // per sweep, the pairs inside a block are not re-rotated in each of its nbe - 1 visits
        const bool cross = JD_CROSS && step > 0;
        const int nin = cross ? bs : nc2 - 1;
        auto inner_pair = [&](int s2, int i, int& p, int& q) {
          if (cross) { p = i; q = bs + (i + s2) % bs; }
          else rr_pair(nc2, s2, i, p, q);
        };
        __syncthreads();
        for (int l = threadIdx.x / M, r = threadIdx.x % M; l < nc2;) {  // (l, r) advance by blockDim
          const int c = s_col[l];  // cp.async: all loads in flight at once (absent columns zero-filled)
          cp_async_el<T2>(Ab + (size_t)l * MP + r, c >= 0 ? (const void*)(A + (size_t)c * M + r) : (const void*)A, c >= 0);
          r += blockDim.x;
          while (r >= M) { r -= M; ++l; }
        }
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        mark(0);
        if (prof) atomicAdd(&jd_prof[4], 1ull);
        if (gram_sweep) {
          // G = Ab^H Ab, Hermitian: only the tiles ti <= tj (nh (nh + 1) / 2 of nh^2) are formed,
          // the others mirrored; thread (tile, part of the rows), parts 1.. sum through Gs
          const int t = threadIdx.x;
          const int TU = nh * (nh + 1) / 2, NP = jd_gram_parts(bs);
          T2 g[4] = {mk2(T(0), T(0)), mk2(T(0), T(0)), mk2(T(0), T(0)), mk2(T(0), T(0))};
          const int tile = t % TU, part = t / TU;
          int ti = 0, tj = tile;  // tile -> (ti, tj), ti <= tj (row ti holds nh - ti tiles)
          while (tj >= nh - ti) { tj -= nh - ti; ++ti; }
          tj += ti;
          if (t < NP * TU) {
            const int r0 = part * M / NP, r1 = (part + 1) * M / NP;
            const T2* a0 = Ab + (size_t)ti * MP;
            const T2* a1 = Ab + (size_t)(ti + bs) * MP;
            const T2* b0 = Ab + (size_t)tj * MP;
            const T2* b1 = Ab + (size_t)(tj + bs) * MP;
#pragma unroll 4
            for (int r = r0; r < r1; ++r) {
              const T2 x0 = a0[r], x1 = a1[r], y0 = b0[r], y1 = b1[r];
              // conj(x) y
              g[0].x = fma(x0.x, y0.x, fma(x0.y, y0.y, g[0].x)); g[0].y = fma(x0.x, y0.y, fma(-x0.y, y0.x, g[0].y));
              g[1].x = fma(x0.x, y1.x, fma(x0.y, y1.y, g[1].x)); g[1].y = fma(x0.x, y1.y, fma(-x0.y, y1.x, g[1].y));
              g[2].x = fma(x1.x, y0.x, fma(x1.y, y0.y, g[2].x)); g[2].y = fma(x1.x, y0.y, fma(-x1.y, y0.x, g[2].y));
              g[3].x = fma(x1.x, y1.x, fma(x1.y, y1.y, g[3].x)); g[3].y = fma(x1.x, y1.y, fma(-x1.y, y1.x, g[3].y));
            }
            if (part) {
#pragma unroll
              for (int k = 0; k < 4; ++k) Gs[((size_t)(part - 1) * TU + tile) * 4 + k] = g[k];
            }
          }
          __syncthreads();
          if (t < TU) {
            for (int pp = 1; pp < NP; ++pp) {  // parts in order: the sum does not depend on timing
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const T2 o = Gs[((size_t)(pp - 1) * TU + tile) * 4 + k];
                g[k].x += o.x;
                g[k].y += o.y;
              }
            }
            G[(size_t)ti * GL + tj] = g[0];
            G[(size_t)ti * GL + tj + bs] = g[1];
            G[(size_t)(ti + bs) * GL + tj] = g[2];
            G[(size_t)(ti + bs) * GL + tj + bs] = g[3];
            if (ti != tj) {  // G(b, a) = conj G(a, b)
              G[(size_t)tj * GL + ti] = mk2(g[0].x, -g[0].y);
              G[(size_t)(tj + bs) * GL + ti] = mk2(g[1].x, -g[1].y);
              G[(size_t)tj * GL + ti + bs] = mk2(g[2].x, -g[2].y);
              G[(size_t)(tj + bs) * GL + ti + bs] = mk2(g[3].x, -g[3].y);
            }
          }
          __syncthreads();
          if (warp == 0) {  // column norms^2 within 2^20: Gram form for this block pair (lane = column)
            T mx = 0, mn = JdT<T>::HUGE_;  // HUGE_: no valid column
            if (lane < nc2) {
              const T a = G[(size_t)lane * GL + lane].x;
              if (s_col[lane] >= 0 && a > 0) { mx = a; mn = a; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            }
            if (lane == 0) {
              s_gram = mn == JdT<T>::HUGE_ || mx <= mn * JdT<T>::NORM_RATIO;
              if (jac_trace_items > 1000 && blockIdx.x == 0) {
                s_ngram += s_gram;
                if (step == 1 && bp == 0) printf("    sweep %d step 1 block pair 0: norms^2 min %.3e max %.3e\n", sweep, (double)mn, (double)mx);
              }
            }
          }
        }
        for (int t = threadIdx.x; t < nc2 * nc2; t += blockDim.x)
          W[t] = mk2((t % nc2) == (t / nc2) ? T(1) : T(0), T(0));
        __syncthreads();
        if (prof && gram_sweep) {  // [7]: Gram products + mode decision (moved out of "inner")
          const long long t = clock64();
          atomicAdd(&jd_prof[7], (unsigned long long)(t - tm));
          tm = t;
        }
        if (s_gram) {
          if (prof) atomicAdd(&jd_prof[6], 1ull);
          for (int s2 = 0; s2 < nin; ++s2) {
            if (threadIdx.x < bs) {
              const int i = threadIdx.x;
              int p, q;
              inner_pair(s2, i, p, q);
              int on = 0;
              if (s_col[p] >= 0 && s_col[q] >= 0) {
                const T sp = G[(size_t)p * GL + p].x, sq = G[(size_t)q * GL + q].x;
                const T2 gg = G[(size_t)p * GL + q];
                const T g2 = gg.x * gg.x + gg.y * gg.y;
                note_off(g2, sp, sq);
                if (g2 > JdT<T>::thr(tol, sp, sq) && g2 != T(0) && JdT<T>::ok(sp, sq)) {
                  T c, sr, si;
                  jd_rot(sp, sq, gg.x, gg.y, g2, c, sr, si);
                  s_c[i] = c; s_sr[i] = sr; s_si[i] = si;
                  on = 1;
                  s_rot = 1;
                }
              }
              s_on[i] = on;
              s_p[i] = p;
              s_q[i] = q;
            }
            __syncthreads();
            // one pass: every 2x2 block (pairs a, b) of G becomes J_a^H G_ab J_b, and the
            // columns p, q of W of every rotating pair are rotated  (forming only the blocks a <= b of
            // the Hermitian G and mirroring them measured slower: k_jacobi_blk<double> 161 -> 168 ms)
            for (int t = threadIdx.x; t < bs * nc2; t += blockDim.x) {
              if (t < bs * bs) {
                const int a = t / bs, b = t % bs;
                const int pa = s_p[a], qa = s_q[a], pb = s_p[b], qb = s_q[b];
                T2 b00 = G[(size_t)pa * GL + pb], b01 = G[(size_t)pa * GL + qb];
                T2 b10 = G[(size_t)qa * GL + pb], b11 = G[(size_t)qa * GL + qb];
                if (s_on[b]) {  // columns:  x' = c x - conj(s) y,  y' = s x + c y
                  const T c = s_c[b], sr = s_sr[b], si = s_si[b];
                  T2 x = b00, y = b01;
                  b00 = mk2(c * x.x - (sr * y.x + si * y.y), c * x.y - (sr * y.y - si * y.x));
                  b01 = mk2(sr * x.x - si * x.y + c * y.x, sr * x.y + si * x.x + c * y.y);
                  x = b10; y = b11;
                  b10 = mk2(c * x.x - (sr * y.x + si * y.y), c * x.y - (sr * y.y - si * y.x));
                  b11 = mk2(sr * x.x - si * x.y + c * y.x, sr * x.y + si * x.x + c * y.y);
                }
                if (s_on[a]) {  // rows:  x' = c x - s y,  y' = conj(s) x + c y
                  const T c = s_c[a], sr = s_sr[a], si = s_si[a];
                  T2 x = b00, y = b10;
                  b00 = mk2(c * x.x - (sr * y.x - si * y.y), c * x.y - (sr * y.y + si * y.x));
                  b10 = mk2(sr * x.x + si * x.y + c * y.x, sr * x.y - si * x.x + c * y.y);
                  x = b01; y = b11;
                  b01 = mk2(c * x.x - (sr * y.x - si * y.y), c * x.y - (sr * y.y + si * y.x));
                  b11 = mk2(sr * x.x + si * x.y + c * y.x, sr * x.y - si * x.x + c * y.y);
                }
                if (s_on[a] | s_on[b]) {
                  G[(size_t)pa * GL + pb] = b00; G[(size_t)pa * GL + qb] = b01;
                  G[(size_t)qa * GL + pb] = b10; G[(size_t)qa * GL + qb] = b11;
                }
              }
              const int i = t >> lgc, k = t & (nc2 - 1);
              if (!s_on[i]) continue;
              const int p = s_p[i], q = s_q[i];
              const T c = s_c[i], sr = s_sr[i], si = s_si[i];
              T2* wp = W + (size_t)p * nc2 + k;
              T2* wq = W + (size_t)q * nc2 + k;
              const T2 x = *wp, y = *wq;
              *wp = mk2(c * x.x - (sr * y.x + si * y.y), c * x.y - (sr * y.y - si * y.x));
              *wq = mk2(sr * x.x - si * x.y + c * y.x, sr * x.y + si * x.x + c * y.y);
            }
            __syncthreads();
          }
        } else {
          for (int s2 = 0; s2 < nin; ++s2) {
            for (int i = warp; i < bs; i += JD_THREADS / 32) {
              int p, q;
              inner_pair(s2, i, p, q);
              if (s_col[p] < 0 || s_col[q] < 0) continue;
              T2* ap = Ab + (size_t)p * MP;
              T2* aq = Ab + (size_t)q * MP;
              T sp = 0, sq = 0, gr = 0, gi = 0;
              for (int r = lane; r < M; r += 32) {
                const T2 x = ap[r], y = aq[r];
                sp += x.x * x.x + x.y * x.y;
                sq += y.x * y.x + y.y * y.y;
                gr += x.x * y.x + x.y * y.y;
                gi += x.x * y.y - x.y * y.x;
              }
              warp_sum4_d(sp, sq, gr, gi);
              const T g2 = gr * gr + gi * gi;
              if (lane == 0) note_off(g2, sp, sq);
              if (!(g2 > JdT<T>::thr(tol, sp, sq)) || g2 == T(0) || !JdT<T>::ok(sp, sq)) continue;
              if (lane == 0) s_rot = 1;
              T c, sr, si;
              jd_rot(sp, sq, gr, gi, g2, c, sr, si);
              for (int r = lane; r < M; r += 32) {
                const T2 x = ap[r], y = aq[r];
                ap[r] = mk2(c * x.x - (sr * y.x + si * y.y), c * x.y - (sr * y.y - si * y.x));
                aq[r] = mk2(sr * x.x - si * x.y + c * y.x, sr * x.y + si * x.x + c * y.y);
              }
              T2* wp = W + (size_t)p * nc2;
              T2* wq = W + (size_t)q * nc2;
              for (int r = lane; r < nc2; r += 32) {
                const T2 x = wp[r], y = wq[r];
                wp[r] = mk2(c * x.x - (sr * y.x + si * y.y), c * x.y - (sr * y.y - si * y.x));
                wq[r] = mk2(sr * x.x - si * x.y + c * y.x, sr * x.y + si * x.x + c * y.y);
              }
            }
            __syncthreads();
          }
        }
        mark(1);
        if (it.cnt && threadIdx.x == 0) {  // algorithmic DFMA of this visit (bench.py roofline)
          const unsigned long long nc2u = nc2, Mu = M, Nu = N;
          unsigned long long f = 0;
          if (s_gram) f = 4ull * (nc2u * (nc2u + 1) / 2) * Mu + (unsigned long long)nin * (16ull * bs * bs + 8ull * bs * nc2u);
          else f = (unsigned long long)nin * bs * (16ull * Mu + 8ull * nc2u);
          if (s_rot) f += 4ull * nc2u * nc2u * (Mu + Nu);
          atomicAdd(&it.cnt[SP ? CNT_JSP_FFMA : CNT_JDB_DFMA], f);
        }
        if (s_rot) {  // block-uniform
          if (threadIdx.x == 0) s_any = 1;
          if (s_gram) {
            jd_apply_w<T, T2>(Ab, MP, A, M, W, bs, s_col);  // A[:, cols] = Ab W
          } else {
            for (int l = threadIdx.x / M, r = threadIdx.x % M; l < nc2;) {
              const int c = s_col[l];
              if (c >= 0) A[(size_t)c * M + r] = Ab[(size_t)l * MP + r];
              r += blockDim.x;
              while (r >= M) { r -= M; ++l; }
            }
          }
          __syncthreads();  // Ab is free now
          mark(2);
          // stage V[:, cols] (N <= M rows) in its place, then V[:, cols] = Vb W
          T2* Vb = Ab;  // [2bs][N]
          for (int l = threadIdx.x / N, r = threadIdx.x % N; l < nc2;) {
            const int c = s_col[l];
            cp_async_el<T2>(Vb + (size_t)l * N + r, c >= 0 ? (const void*)(V + (size_t)c * N + r) : (const void*)V, c >= 0);
            r += blockDim.x;
            while (r >= N) { r -= N; ++l; }
          }
          cp_commit();
          cp_wait<0>();
          __syncthreads();
          jd_apply_w<T, T2>(Vb, N, V, N, W, bs, s_col);
        }
        __syncthreads();
        mark(3);
      }
      csync();  // the next step's block pairs read columns this step wrote
    }
    if (off_t > 0) atomicMax(&s_off, (unsigned long long)__double_as_longlong(off_t));
    off_t = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_any) atomicOr(&it.anyflag[sweep & 1], 1);
      atomicMax(&it.offmax[sweep & 1], s_off);
    }
    csync();
    const int any = *(volatile int*)&it.anyflag[sweep & 1];
    if (jac_trace_items > 1000 && crank == 0 && threadIdx.x == 0 && (int)(blockIdx.x / C) == 0)
      printf("  block Jacobi (%s) sweep %d: %s form (%d block pairs), rotated %d, off flag %.1f\n", SP ? "binary32" : "binary64", sweep,
             gram_sweep ? "Gram" : "column", s_ngram, any, __longlong_as_double((long long)*(volatile unsigned long long*)&it.offmax[sweep & 1]));
    if (!any) break;
    // binary32 phase: every pair of this sweep was already below the hand-over level when it was
    // evaluated (its rotations leave ~ that level squared): the binary64 phase takes over
    if (SP && __longlong_as_double((long long)*(volatile unsigned long long*)&it.offmax[sweep & 1]) < 0.5) break;
    // binary64, column form: every pair of this sweep was below JD_LAST_OFF when it was evaluated, so its
    // rotations leave relative off-diagonals of order JD_LAST_OFF^2 / gap, below tol: the rotation-free
    // sweep that would confirm it is not run (the p-bit stages decide convergence, R19)
    if (!SP && !gram_sweep && __longlong_as_double((long long)*(volatile unsigned long long*)&it.offmax[sweep & 1]) < 0.2) break;
  }
  if (crank == 0 && threadIdx.x == 0) *(SP ? it.sweeps_s : it.sweeps_d) = sweep;
  if (jac_trace_items && crank == 0 && threadIdx.x == 0 && (int)(blockIdx.x / C) < jac_trace_items)
    printf("block Jacobi (%s) item %d M %d N %d: %d sweeps\n", SP ? "binary32" : "binary64", (int)(blockIdx.x / C), M, N, sweep);
  if (prof) atomicAdd(&jd_prof[5], (unsigned long long)sweep);
}

// ---------------------------------------------------------------------------- R27 hand-over
// binary32 phase -> binary64 phase: Vd = (binary64) Vs, then two Newton-Schulz steps in binary64,
// Rm = Vd^H Vd, V0 = Vd (3 I - Rm) / 2;  Rm = V0^H V0, Vd = V0 (3 I - Rm) / 2  (Vs is unitary to
// ~1e-5 only; the rotations of the binary64 phase keep whatever defect V starts with, and the
// fixed-point Newton-Schulz schedule (NsSched) expects a basis unitary to ~2^-45);  Aj = Theta_d Vd.
// binary32 copy of Theta_d for the first phase, scaled by a power of two so that its largest row
// norm is ~1 (the block exponent of Theta' may sit far above its entries: unscaled, the squared
// column norms of a circuit's Theta' reached 1e-14 and their products underflowed binary32)
static __global__ void __launch_bounds__(256) k_d_to_s(const PreItem* items) {
  const PreItem it = items[blockIdx.y];
  if (it.N == 0 || it.As == nullptr) return;
  const double rm = __longlong_as_double((long long)*it.rowmax);
  int ex = 0;
  if (rm > 0) frexp(rm, &ex);
  const double sc = ldexp(1.0, -(ex / 2));
  const size_t n = (size_t)it.M * it.N;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const double2 v = it.Ad[t];
    it.As[t] = make_float2((float)(v.x * sc), (float)(v.y * sc));
  }
}
static __global__ void __launch_bounds__(256) k_sp_to_dp(const PreItem* items) {
  const PreItem it = items[blockIdx.y];
  if (it.N == 0 || it.Vs == nullptr) return;
  const size_t n = (size_t)it.N * it.N;
  if (blockIdx.x == 0 && threadIdx.x == 0) *it.sp_bad = 0;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const float2 v = it.Vs[t];
    it.Vd[t] = make_double2((double)v.x, (double)v.y);
  }
}
// Batched complex binary64 GEMM for the hand-over, column-major, 64 x 64 tiles, 256 threads with a
// 4 x 4 register tile each.  which: 0: Rm = X^H X (N x N x N);  1: Y = 1.5 X - 0.5 X Rm, with
// (X, Y) = (Vd, V0) in Newton-Schulz step 0 and (V0, Vd) in step 1;  2: Aj = Ad Vd (M x N x N).
static __global__ void __launch_bounds__(256) k_zgemm_handover(const PreItem* items, int which, int nsstep) {
  const PreItem it = items[blockIdx.z];
  if (it.N == 0 || it.Vs == nullptr) return;
  const int N = it.N, M = it.M;
  const int rows = which == 2 ? M : N, cols = N, K = N;
  const double2* X = nsstep ? it.V0 : it.Vd;
  const double2* A = which == 2 ? it.Ad : X;
  const double2* B = which == 0 ? X : (which == 1 ? it.Rm : it.Vd);
  double2* C = which == 0 ? it.Rm : (which == 1 ? (nsstep ? it.Vd : it.V0) : it.Aj);
  const int lda = which == 2 ? M : N, ldb = N, ldc = rows;
  const bool conjA = which == 0;
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  if (r0 >= rows || c0 >= cols) return;
  __shared__ double2 As_[16][65], Bs_[16][65];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < K; k0 += 16) {
    __syncthreads();
    for (int w = threadIdx.x; w < 16 * 64; w += 256) {
      double2 va = make_double2(0.0, 0.0), vb = make_double2(0.0, 0.0);
      if (!conjA) {  // A(r, k) at A[k lda + r]: r fastest
        const int e = w % 64, kk = w / 64;
        if (r0 + e < rows && k0 + kk < K) va = A[(size_t)(k0 + kk) * lda + r0 + e];
        As_[kk][e] = va;
      } else {       // A^H(r, k) = conj A(k, r) at A[r lda + k]: k fastest
        const int kk = w % 16, e = w / 16;
        if (r0 + e < rows && k0 + kk < K) {
          va = A[(size_t)(r0 + e) * lda + k0 + kk];
          va.y = -va.y;
        }
        As_[kk][e] = va;
      }
      {              // B(k, c) at B[c ldb + k]: k fastest
        const int kk = w % 16, e = w / 16;
        if (c0 + e < cols && k0 + kk < K) vb = B[(size_t)(c0 + e) * ldb + k0 + kk];
        Bs_[kk][e] = vb;
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      double2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As_[kk][tx + 16 * i]; b[i] = Bs_[kk][ty + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, acc[i][j].x));
          acc[i][j].y = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, acc[i][j].y));
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + tx + 16 * i, c = c0 + ty + 16 * j;
      if (r >= rows || c >= cols) continue;
      double2 v = acc[i][j];
      if (which == 0 && nsstep == 1) {  // V after one step must be unitary to 1e-6 (NaN fails the test too)
        if (!(fabs(v.x - (r == c ? 1.0 : 0.0)) <= 1e-6) || !(fabs(v.y) <= 1e-6)) atomicOr(it.sp_bad, 1);
      }
      if (which == 1) {
        const double2 x = X[(size_t)c * N + r];
        v = make_double2(1.5 * x.x - 0.5 * v.x, 1.5 * x.y - 0.5 * v.y);
        if (nsstep == 1 && *it.sp_bad) v = make_double2(r == c ? 1.0 : 0.0, 0.0);  // binary64 phase from scratch
      }
      if (which == 2 && *it.sp_bad) v = it.Ad[(size_t)c * M + r];
      C[(size_t)c * ldc + r] = v;
    }
}

// debug (MPS_JACOBI_TRACE > 2000): defects of the hand-over / of the final binary64 pair (A, V) of item 0
static __global__ void k_dbg_pair(const PreItem* items, int stage) {
  const PreItem it = items[0];
  if (it.N == 0 || it.Aj == nullptr) return;
  const int N = it.N, M = it.M;
  __shared__ double s_u, s_a, s_m;
  if (threadIdx.x == 0) { s_u = 0; s_a = 0; s_m = 0; }
  __syncthreads();
  double eu = 0, ea = 0, am = 0;
  for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
    const int r = t % N, c = t / N;
    double2 acc = make_double2(r == c ? -1.0 : 0.0, 0.0);
    for (int k = 0; k < N; ++k) {
      const double2 x = it.Vd[(size_t)r * N + k], y = it.Vd[(size_t)c * N + k];
      acc.x += x.x * y.x + x.y * y.y;
      acc.y += x.x * y.y - x.y * y.x;
    }
    eu = fmax(eu, fmax(fabs(acc.x), fabs(acc.y)));
  }
  for (int t = threadIdx.x; t < M * N; t += blockDim.x) {
    const int r = t % M, c = t / M;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < N; ++k) {
      const double2 x = it.Ad[(size_t)k * M + r], y = it.Vd[(size_t)c * N + k];
      acc.x += x.x * y.x - x.y * y.y;
      acc.y += x.x * y.y + x.y * y.x;
    }
    const double2 z = it.Aj[(size_t)c * M + r];
    ea = fmax(ea, fmax(fabs(acc.x - z.x), fabs(acc.y - z.y)));
    am = fmax(am, fmax(fabs(z.x), fabs(z.y)));
  }
  atomicMax((unsigned long long*)&s_u, (unsigned long long)__double_as_longlong(eu));
  atomicMax((unsigned long long*)&s_a, (unsigned long long)__double_as_longlong(ea));
  atomicMax((unsigned long long*)&s_m, (unsigned long long)__double_as_longlong(am));
  __syncthreads();
  if (threadIdx.x == 0)
    printf("  hand-over check (%s) M %d N %d: max |V^H V - I| %.3e, max |A - Theta_d V| %.3e (max |A| %.3e)\n",
           stage ? "after the binary64 phase" : "before the binary64 phase", M, N, s_u, s_a, s_m);
}

// binary64 v (|v| <= 1) -> L balanced digits at exponent 1 (value = sum d_k 2^(28k) 2^(1-28L)), exact
template <int L>
__device__ __forceinline__ void double_to_fx(double v, int32_t (&d)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = 0;
  if (v == 0.0) return;
  const bool neg = v < 0;
  int ex;
  const double m = frexp(fabs(v), &ex);  // |v| = m 2^ex, m in [0.5, 1)
  const uint64_t M53 = (uint64_t)ldexp(m, 53);
  // integer I = |v| 2^(28L - 1) = M53 2^(ex - 53 + 28L - 1); s = bit position of M53's bit 0
  const int s = ex - 54 + 28 * L;
  if (s < -53) return;
  uint64_t lo = M53;
  int base = s;
  if (s < 0) { lo = M53 >> (-s); base = 0; }
  const int q = base / 28, r = base % 28;
  // lo << r spread over digits q, q+1, q+2 (53 + 27 bits at most)
  const unsigned __int128 w = (unsigned __int128)lo << r;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int j = k - q;
    if (j >= 0 && j < 3) d[k] = (int32_t)((w >> (28 * j)) & 0x0FFFFFFFu);
  }
  int32_t c = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int32_t x = d[k] + c;
    c = (x + (1 << 27)) >> 28;
    d[k] = x - (c << 28);
  }
  d[L - 1] += c << 28;
  if (neg) {
#pragma unroll
    for (int k = 0; k < L; ++k) d[k] = -d[k];
  }
}

// X_0 keeps only the top NS_X0_DIGITS digits of V_d (an error < 2^-110 in a starting basis that
// is unitary to ~2^-45 only): then every Newton-Schulz iterate X_k holds exactly lg[k-1]
// digits and the GEMMs skip the zero ones (NsSched::nz)
constexpr int NS_X0_DIGITS = 4;
template <int L>
__global__ void k_d_to_fx(const PreItem* items) {
  const PreItem it = items[blockIdx.y];
  const int N = it.N;
  if (N == 0) return;  // item without preconditioning
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    it.eOne[0] = 1; it.eOne[1] = 0;
    if (it.eXs) { it.eXs[0] = 0; it.eXs[1] = -1; }
  }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N * N; t += gridDim.x * blockDim.x) {
    const int r = t % N, c = t / N;
    const double2 v = it.Vd[(size_t)c * N + r];
    int32_t d[L];
    double_to_fx<L>(v.x, d);
#pragma unroll
    for (int k = 0; k < L - NS_X0_DIGITS; ++k) d[k] = 0;
    stfx<L>(it.X, N, c, 0, r, d);
    double_to_fx<L>(v.y, d);
#pragma unroll
    for (int k = 0; k < L - NS_X0_DIGITS; ++k) d[k] = 0;
    stfx<L>(it.X, N, c, 1, r, d);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // |A_1(r, c)| <= ||Theta'(r, :)|| ||x_c|| <= sqrt(rowmax) 2^e (1 + 2^-40): exponent
    // ceil(log2 sqrt(rowmax)) + 1 above e, so that |A_1| < 2^(eA1 - 1)
    const double rm = __longlong_as_double((long long)*it.rowmax);
    int64_t ea = *it.eA0;
    if (rm > 0) ea += (int64_t)ceil(0.5 * log2(rm) * (1 + 1e-12) + 1e-9) + 1;
    *it.eA1 = ea;
  }
}

// ---------------------------------------------------------------------------- GEMM
// C (rows x cols) = sgn * op(A) B (+ Cadd) (+ I), fixed-point complex with block exponents:
// op(A) = A (stored rows x K, column-major, ld lda) or A^H (A stored K x rows).  C is written
// at exponent *eCout (given); the digit sum is shifted by g = eC - eA - eB bits (-27..27).
// Precision schedule (template): only the top LG of the L stored digits of A and B take
// part (an LG-digit product, rounded to LG digits and stored as the top LG digits of C, the
// lower ones 0 (+ Cadd's)); the top Z of those digits of B are known to be 0 and skipped —
// zerr (if set) receives 1 when one is not (the caller then re-runs without the shortcut).
struct GemmT {
  const int32_t* A; int lda; const int64_t* eA;
  const int32_t* B; int ldb; const int64_t* eB;
  int32_t* C; int ldc; const int64_t* eCout;
  const int32_t* Cadd;  // same shape / exponent as C, or null
  int64_t* eCcols;      // if non-null: eCcols[c] = *eCout for every column (Jacobi layout)
  int rows, cols, K, conjA, neg, addI;
  int* zerr;
  // per-column mode (recovery of V, R16): B has column exponents eBcols[c]; column c of C is
  // (digit sum shifted by ghead bits) x colcoef[c] ((L+1)-digit coefficient), at exponent
  // eA + eBcols[c] + ghead + colexp[c], written to eCcols[c].  eCout is unused.
  const int64_t* eBcols; const int32_t* colcoef; const int64_t* colexp; int ghead;
  int herm;  // C is Hermitian (X^H X): only tiles on/above the diagonal are computed, mirrored
  int64_t* eCwrite;  // if non-null (block mode, eCout null): receives eC = eA + eB + ghead
  // column selection: logical column b < *ncols_dev is physical column colmap[b] of B and C
  // (the recovery of V computes only the columns kept by the truncation)
  const int* colmap; const int* ncols_dev;
  int upper;  // only entries r <= c are needed (tensor-core path: tiles below the diagonal skipped)
};

// per-column coefficient of the V recovery: 1/alpha_b = m 2^e, m in [0.5, 1) as L+1 digits
template <int NL>
struct RecItem {
  int N;
  const mpf<NL>* alpha;
  int32_t* coef;  // [N][L+1]
  int64_t* cexp;  // [N]
};
template <int L, int NL>
__global__ void k_recover_coef(const RecItem<NL>* items) {
  const RecItem<NL> it = items[blockIdx.y];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < it.N; b += gridDim.x * blockDim.x) {
    const mpf<NL> al = it.alpha[b];
    int32_t kd[L + 1];
    if (mpf_is_zero(al)) {
#pragma unroll
      for (int k = 0; k <= L; ++k) kd[k] = 0;
      it.cexp[b] = INT64_MIN;  // zero column of V
    } else {
      const mpf<NL> inv = mpf_recip(al);
      mpf_to_fixed<NL, L + 1>(mpf_ldexp(inv, -inv.e), 28, kd);
      it.cexp[b] = inv.e;
    }
#pragma unroll
    for (int k = 0; k <= L; ++k) it.coef[(size_t)b * (L + 1) + k] = kd[k];
  }
}

// round V 2^-g / 2^(28L) for any -27 <= g <= 27
template <int L>
__device__ __forceinline__ void tround_any(int64_t (&acc)[L + 2], int g, int32_t (&out)[L]) {
  if (g >= 0) {
    tround_sr<L>(acc, g, out);
    return;
  }
  tnorm2<L>(acc);
#pragma unroll
  for (int c = 0; c < L + 2; ++c) acc[c] *= ((int64_t)1 << (-g));
  tround2<L>(acc, out);
}

template <int L>
__device__ __forceinline__ void fx_balance(int32_t (&x)[L]) {
  int32_t c = 0;
#pragma unroll
  for (int k = 0; k < L - 1; ++k) {
    const int32_t v = x[k] + c;
    c = (v + (1 << 27)) >> 28;
    x[k] = v - (c << 28);
  }
  x[L - 1] += c;
}

// acc (LG+2 columns: LG-2 .. 2LG-1) += / -= x y, the top Z digits of y being zero and the
// low NZA digits of x / NZB digits of y too (the products skipped are exactly zero)
template <int LG, int Z, bool SUB, int NZA = 0, int NZB = 0>
__device__ __forceinline__ void tmul_z(int64_t (&acc)[LG + 2], const int32_t (&x)[LG], const int32_t (&y)[LG]) {
#pragma unroll
  for (int i = NZA; i < LG; ++i)
#pragma unroll
    for (int j = NZB; j < LG - Z; ++j)
      if (i + j >= LG - 2) acc[i + j - (LG - 2)] = madw(SUB ? -x[i] : x[i], y[j], acc[i + j - (LG - 2)]);
}

constexpr int GT_TILE = 16;
#ifndef GEMM_3M  // complex products of k_gemm_t in three real products
#define GEMM_3M 1
#endif
constexpr int GEMM_PLANES = GEMM_3M ? 3 : 2;

// Epilogue of one output entry (r, c) of a k_gemm_t-style GEMM: ar / ai are the exact sums of
// the real / imaginary parts as LG + 2 int64 digit columns (columns LG - 2 .. 2LG - 1 of the
// LG-digit frame); round by the head-room shift g, then the per-column coefficient, negation,
// + I, + Cadd, balancing, the known-zero top digit check (ZOUT), the store (mirrored for a
// Hermitian off-diagonal tile) and the column exponents.  Shared by k_gemm_t and the
// tensor-core path (tcgemm.cuh), so both write identical formats.
template <int L, int LG, int ZOUT>
__device__ __forceinline__ void gemm_t_store(const GemmT& it, int r, int c, int pc, int64_t (&ar)[LG + 2],
                                             int64_t (&ai)[LG + 2], int g, int64_t eC, bool percol, bool mirror,
                                             int& zbad) {
  constexpr int D0 = L - LG;
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    int32_t t[LG], o[L];
    tround_any<LG>(ri ? ai : ar, g, t);
#pragma unroll
    for (int j = 0; j < L; ++j) o[j] = j >= D0 ? t[j - D0] : 0;
    if (percol && it.colcoef) {  // x column coefficient (L+1 digits, fractional)
      int32_t K[L + 1];
#pragma unroll
      for (int k = 0; k <= L; ++k) K[k] = it.colcoef[(size_t)pc * (L + 1) + k];
      int64_t acc2[L + 2];
#pragma unroll
      for (int j = 0; j < L + 2; ++j) acc2[j] = 0;
      kmul_acc<L>(acc2, K, o, K[L] != 0);
      tround2<L>(acc2, o);
    }
    if (it.neg) {
#pragma unroll
      for (int j = 0; j < L; ++j) o[j] = -o[j];
    }
    if (it.addI && ri == 0 && r == c) o[L - 1] += 1 << (28 - (int)eC);  // + 1 at exponent eC (1)
    if (it.Cadd) {
      int32_t x[L];
      ldfx<L>(it.Cadd, it.ldc, c, ri, r, x);
#pragma unroll
      for (int j = 0; j < L; ++j) o[j] += x[j];
    }
    fx_balance<L>(o);
#pragma unroll
    for (int j = L - ZOUT; j < L; ++j)  // the consumer skips these digits: they must be 0
      if (o[j] != 0) zbad = 1;
    stfx<L>(it.C, it.ldc, pc, ri, r, o);
    if (mirror) {  // C(c, r) = conj C(r, c)
      if (ri) {
#pragma unroll
        for (int j = 0; j < L; ++j) o[j] = -o[j];
      }
      stfx<L>(it.C, it.ldc, r, ri, c, o);
    }
  }
  if (it.eCcols && r == 0) {
    if (!percol) it.eCcols[pc] = eC;
    else if (it.colexp && it.colexp[pc] == INT64_MIN) it.eCcols[pc] = 1;  // alpha = 0: zero column
    else it.eCcols[pc] = *it.eA + it.eBcols[pc] + it.ghead + (it.colexp ? it.colexp[pc] : 0);
  }
}

template <int L, int LG, int Z, int NZA = 0, int NZB = 0, int ZOUT = 0>
__global__ void __launch_bounds__(256, 2) k_gemm_t(const GemmT* items) {
  static_assert(LG <= L && Z < LG && NZA < LG && NZB + Z < LG && ZOUT < L, "precision schedule");
  // a truncated product forms only i + j >= LG - 2 with j < LG - Z, so digits i < Z - 1 of A
  // never take part either: A's digits below ALO are neither staged nor multiplied
  constexpr int ALO = NZA > Z - 1 ? NZA : (Z > 0 ? Z - 1 : 0);
  // k per staging round (16 measured no faster; 4 where 8 exceeds the 48 KB static limit)
  constexpr int GT_KB = (size_t)8 * GEMM_PLANES * LG * (GT_TILE + 1) * 4 * 2 > 48 * 1024 ? 4 : 8;
  // a staging round adds, per k, <= (LG - Z - NZB) products to a column, each < 2^56 except
  // the <= 2 that involve a top digit (digit sums up to 2^29: < 2^57 each, counted as 2 more
  // 2^56 units): (LG - Z - NZB + 2) GT_KB 2^56 <= 80 * 2^56 = 2^62.3 -> one normalisation
  // per round suffices
  constexpr bool NORM_ONCE = GEMM_3M && (LG - Z - NZB) * GT_KB <= 64;
  static_assert(!NORM_ONCE || (double)(LG - Z - NZB + 2) * GT_KB * 72057594037927936.0 + 268435456.0 <
                                  9223372036854775808.0, "k_gemm_t columns fit int64 within a staging round");
  constexpr int D0 = L - LG;  // first stored digit used
  const GemmT it = items[blockIdx.y];
  if (it.rows <= 0 || it.cols <= 0) return;  // item without this GEMM
  const int tilesR = (it.rows + GT_TILE - 1) / GT_TILE, tilesC = (it.cols + GT_TILE - 1) / GT_TILE;
  const int tx = threadIdx.x % GT_TILE, ty = threadIdx.x / GT_TILE;
  // planes: re, im, re + im (the last for the three-product complex multiply)
  __shared__ int32_t As[GT_KB][GEMM_PLANES][LG][GT_TILE + 1];  // +1: conflict-free k-fastest staging writes
  __shared__ int32_t Bs[GT_KB][GEMM_PLANES][LG][GT_TILE + 1];
  const bool percol = it.eBcols != nullptr;
  // block exponent: given (eCout), or eA + eB + ghead (head-room for K terms, eCwrite)
  const int64_t eC = percol ? 0 : (it.eCout ? *it.eCout : *it.eA + *it.eB + it.ghead);
  const int g = percol ? it.ghead : (int)(eC - (*it.eA + *it.eB));
  if (!percol && it.eCwrite && blockIdx.x == 0 && threadIdx.x == 0) *it.eCwrite = eC;
  int zbad = 0;
  const int ncols = it.ncols_dev ? min(*it.ncols_dev, it.cols) : it.cols;
  auto pcol = [&](int cc) { return it.colmap ? it.colmap[cc] : cc; };
  for (int tile = blockIdx.x; tile < tilesR * tilesC; tile += gridDim.x) {
    const int r0 = (tile % tilesR) * GT_TILE, c0 = (tile / tilesR) * GT_TILE;
    if (it.herm && c0 < r0) continue;  // block-uniform: the mirror tile writes these
    if (c0 >= ncols) continue;          // columns not selected
    const int r = r0 + tx, c = c0 + ty;
    int64_t ar[LG + 2], ai[LG + 2];
#pragma unroll
    for (int j = 0; j < LG + 2; ++j) ar[j] = ai[j] = 0;
#if GEMM_3M
    int64_t as[LG + 2];  // sum (xr + xi)(yr + yi)
#pragma unroll
    for (int j = 0; j < LG + 2; ++j) as[j] = 0;
#endif
    for (int k0 = 0; k0 < it.K; k0 += GT_KB) {
      __syncthreads();
      // stage the top LG digits of GT_KB x 16 elements of each operand (only the digits the
      // products use: A's [ALO, LG), B's [NZB, LG - Z)); the index order follows the
      // contiguous direction in global memory (rows of A, k of A^H and of B)
      constexpr int nA = LG - ALO, nB = LG - Z - NZB;
      for (int w = threadIdx.x; w < GT_KB * 2 * nA * GT_TILE; w += 256) {
        int32_t va = 0;
        if (!it.conjA) {
          const int e = w % GT_TILE, dg = ALO + (w / GT_TILE) % nA, ri = (w / (GT_TILE * nA)) % 2,
                    kk = w / (GT_TILE * nA * 2);
          const int k = k0 + kk, rr = r0 + e;
          if (k < it.K && rr < it.rows) va = it.A[((size_t)(k * 2 + ri) * L + D0 + dg) * it.lda + rr];
          As[kk][ri][dg][e] = va;
        } else {
          const int kk = w % GT_KB, dg = ALO + (w / GT_KB) % nA, ri = (w / (GT_KB * nA)) % 2, e = w / (GT_KB * nA * 2);
          const int k = k0 + kk, rr = r0 + e;
          if (k < it.K && rr < it.rows) {
            va = it.A[((size_t)(rr * 2 + ri) * L + D0 + dg) * it.lda + k];
            if (ri) va = -va;
          }
          As[kk][ri][dg][e] = va;
        }
      }
      for (int w = threadIdx.x; w < GT_KB * 2 * nB * GT_TILE; w += 256) {
        const int kk = w % GT_KB, dg = NZB + (w / GT_KB) % nB, ri = (w / (GT_KB * nB)) % 2, e = w / (GT_KB * nB * 2);
        const int k = k0 + kk, cc = c0 + e;
        int32_t vb = 0;
        if (k < it.K && cc < ncols) vb = it.B[((size_t)(pcol(cc) * 2 + ri) * L + D0 + dg) * it.ldb + k];
        Bs[kk][ri][dg][e] = vb;
      }
      __syncthreads();
#if GEMM_3M
      // (xr + i xi)(yr + i yi) = xr yr - xi yi + i [(xr + xi)(yr + yi) - xr yr - xi yi]: three
      // LG-digit products instead of four (digit sums |d| <= 2^29: products < 2^58, normalised
      // every 4 k so that no int64 column exceeds 2^62)
      for (int w = threadIdx.x; w < GT_KB * nA * GT_TILE; w += 256) {
        const int e = w % GT_TILE, dg = ALO + (w / GT_TILE) % nA, kk = w / (GT_TILE * nA);
        As[kk][2][dg][e] = As[kk][0][dg][e] + As[kk][1][dg][e];
      }
      for (int w = threadIdx.x; w < GT_KB * nB * GT_TILE; w += 256) {
        const int e = w % GT_TILE, dg = NZB + (w / GT_TILE) % nB, kk = w / (GT_TILE * nB);
        Bs[kk][2][dg][e] = Bs[kk][0][dg][e] + Bs[kk][1][dg][e];
      }
      __syncthreads();
#pragma unroll 1
      for (int kk = 0; kk < GT_KB; ++kk) {
        int32_t x[LG], y[LG];
#pragma unroll
        for (int j = 0; j < LG; ++j) { x[j] = As[kk][0][j][tx]; y[j] = Bs[kk][0][j][ty]; }
        tmul_z<LG, Z, false, ALO, NZB>(ar, x, y);
#pragma unroll
        for (int j = 0; j < LG; ++j) { x[j] = As[kk][1][j][tx]; y[j] = Bs[kk][1][j][ty]; }
        tmul_z<LG, Z, false, ALO, NZB>(ai, x, y);
#pragma unroll
        for (int j = 0; j < LG; ++j) { x[j] = As[kk][2][j][tx]; y[j] = Bs[kk][2][j][ty]; }
        tmul_z<LG, Z, false, ALO, NZB>(as, x, y);
        // a column receives <= LG - Z - NZB products (< 2^56 each: digit sums <= 2^28) per k:
        // normalise every 4 k unless a whole staging round cannot reach 2^62
        if (!NORM_ONCE && (kk & 3) == 3 && kk + 1 < GT_KB) { tnorm2<LG>(ar); tnorm2<LG>(ai); tnorm2<LG>(as); }
      }
      tnorm2<LG>(ar);
      tnorm2<LG>(ai);
      tnorm2<LG>(as);
#else
#pragma unroll 1
      for (int kk = 0; kk < GT_KB; ++kk) {
        int32_t xr[LG], xi[LG], yr[LG], yi[LG];
#pragma unroll
        for (int j = 0; j < LG; ++j) {
          xr[j] = As[kk][0][j][tx]; xi[j] = As[kk][1][j][tx];
          yr[j] = Bs[kk][0][j][ty]; yi[j] = Bs[kk][1][j][ty];
        }
        tmul_z<LG, Z, false, ALO, NZB>(ar, xr, yr);
        tmul_z<LG, Z, true, ALO, NZB>(ar, xi, yi);
        tmul_z<LG, Z, false, ALO, NZB>(ai, xr, yi);
        tmul_z<LG, Z, false, ALO, NZB>(ai, xi, yr);
        if ((kk & 7) == 7 && kk + 1 < GT_KB) { tnorm2<LG>(ar); tnorm2<LG>(ai); }  // <= 8 k per int64 column run
      }
      tnorm2<LG>(ar);
      tnorm2<LG>(ai);
#endif
    }
#if GEMM_3M
    // ar = sum xr yr, ai = sum xi yi, as = sum (xr + xi)(yr + yi) -> re = ar - ai, im = as - ar - ai
#pragma unroll
    for (int j = 0; j < LG + 2; ++j) {
      const int64_t t1 = ar[j], t2 = ai[j];
      ar[j] = t1 - t2;
      ai[j] = as[j] - t1 - t2;
    }
#endif
    if (r < it.rows && c < ncols) gemm_t_store<L, LG, ZOUT>(it, r, c, pcol(c), ar, ai, g, eC, percol, it.herm && c0 != r0, zbad);
  }
  if (zbad && it.zerr) atomicOr(it.zerr, 2);  // 2: re-run without the preconditioner
}

// Newton-Schulz precision schedule: iteration k computes D_k with LG digits and
// X_{k+1} = X_k + X_k D_k / 2 with LG digits skipping the Z top digits of D_k (zero since
// |D_k| ~ 2^(-45 * 2^k)); conservative by >= 1 digit, checked at run time (zerr).
// X_k (k >= 1) holds only lg[k-1] digits (the top ones: the update writes an lg[k-1]-digit
// product onto X_{k-1}, X_0 is cut to NS_X0_DIGITS), so in iteration k's lg[k]-digit frame its
// low nz[k] = lg[k] - lg[k-1] digits are zero by construction: D_k skips them in both operands,
// the update in X_k.  The skipped top Z digits of D_k are checked where D_k is written (ZOUT).
template <int L> struct NsSched;
template <> struct NsSched<10> {
  static_assert(NS_X0_DIGITS == 4, "lg[0]");
  static constexpr int n = 3;
  static constexpr int lg[3] = {4, 7, 10};
  static constexpr int z[3] = {1, 2, 5};
  static constexpr int nz[3] = {0, 3, 3};
};
template <> struct NsSched<19> {
  static constexpr int n = 4;
  static constexpr int lg[4] = {4, 7, 14, 19};
  static constexpr int z[4] = {1, 2, 5, 10};
  static constexpr int nz[4] = {0, 3, 7, 5};
};

template <int L, int K>
inline void launch_ns_iter(const GemmT* dD, const GemmT* dX, dim3 grid, cudaStream_t st) {
  constexpr int LG = NsSched<L>::lg[K], Z = NsSched<L>::z[K], NZ = NsSched<L>::nz[K];
  k_gemm_t<L, LG, 0, NZ, NZ, Z><<<grid, 256, 0, st>>>(dD);
  k_gemm_t<L, LG, Z, NZ, 0><<<grid, 256, 0, st>>>(dX);
}

}  // namespace mpsb
