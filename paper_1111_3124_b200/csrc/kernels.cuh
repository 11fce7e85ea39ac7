// sm_100a kernels of the MPS gate update.
// Every kernel works on a batch of independent "items" (gates or cfg2 matrices);
// per-item geometry and pointers live in small device descriptor arrays.
//
// Fixed-point matrix layout (the Jacobi working format):
//   digits  d[((col*2 + ri)*L + k)*ld + row]   (int32, balanced radix-2^28)
//   value   (sum_k d_k 2^(28k)) * 2^(e_col - 28L),  ri = 0 re / 1 im
// so a warp reading 32 consecutive rows of one digit plane issues one coalesced
// 128-byte transaction.  Store records are AoS (include/mps_b200.h format).
#pragma once
#include <cstdint>

#include <cooperative_groups.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "mp.cuh"

namespace mpsb {

constexpr int NTHR = 256;  // threads per CTA of the per-item kernels
constexpr int NWARP = NTHR / 32;
constexpr int MAX_SWEEPS = JACOBI_MAX_SWEEPS;
#ifndef JACOBI_STAGES_280
#define JACOBI_STAGES_280 2
#endif
#ifndef JACOBI_CTAS_280
#define JACOBI_CTAS_280 2
#endif

// ----------------------------------------------------------------------------
// item descriptors
// ----------------------------------------------------------------------------
// Build a fixed matrix from a site tensor G [2][da][db] (records):
//   mode 0: rows (i,a) = i*da + a, cols b      F = lamL(a) G^i(a,b) lamR(b)
//   mode 1: rows a, cols (i,b) = i*db + b      F = lamL(a) G^i(a,b) lamR(b)
struct PrepItem {
  const uint32_t* G;        // records
  const uint32_t* lamL;     // da records or null (= ones)
  const uint32_t* lamR;     // db records or null
  int da, db, mode;
  int32_t* F;               // digits, ld = rows
  int64_t* eF;              // block exponent (1 value)
};

// C = op(A) * B, op(A) = A or A^H ; block exponents; C rows x cols, inner K
struct GemmItem {
  const int32_t* A; int lda; const int64_t* eA;
  const int32_t* B; int ldb; const int64_t* eB;
  int32_t* C; int ldc; int64_t* eC;
  int rows, cols, K, conjA;  // conjA: A stored K x rows, use conj transpose
};

// Theta'(x-block) = sum_y U[x][y] Theta(y-block); rows = RB*chiL, cols = 2*chiR,
// x = 2*rowblock + colblock (qubit of the first site most significant).
// Output in Jacobi layout: A (M x N) with per-column exponents; trans -> A = Theta'^H.
struct MixItem {
  const int32_t* T; int ldt; const int64_t* eT;   // Theta (block exponent)
  const uint32_t* U;                              // D x D complex records
  int RB, chiL, chiR;                             // D = 2*RB
  int trans;
  int32_t* A; int64_t* eA; int M, N;              // output Jacobi matrix (M >= N)
};

template <int NL>
struct SvdItem {
  int M, N;                 // Jacobi matrix, N <= M, N even (padded)
  int32_t* A; int64_t* eA;  // [N][2][L][M], [N]
  int32_t* V;               // [N][2][L][N], exponent fixed = 1
  mpf<NL>* alpha;           // [N] squared column norms (output: final)
  mpf<NL>* gam;             // [N/2][2] scratch
  int32_t* coef;            // [N/2][33][L+1] scratch: 24 signed coefficient slots + 9 values (L+1 digits)
  int* dbg;                 // [64] rotations per sweep, or null
  int* rot;                 // [N/2] scratch
  int* negl;                // [N] scratch
  int* status;              // out: 0 / MPS_ENOCONV
  int* sweeps;              // out
  long long* rotations;     // out
  int* sync;                // scratch flag ("some pair rotated in this sweep")
  mpf<NL>* zbuf;            // scratch: negligible-column floor
  unsigned long long* phase_cycles;  // null, or [6]: D, R, U, norms, init, total (summed over CTAs)
  int32_t* A0;              // non-null: V is NOT accumulated; the input Theta' is kept here (M x N,
                            // block exponent eA0) and V is recovered after convergence (k_recover_v)
  int64_t* eA0;             // [1]
  int64_t* eV;              // [N] exponents of the recovered V columns
  int a0_ready;             // 1: A0 / eA0 were written by the producer (k_build_m2, k_mix), not copied here
  int v_preset;             // accumulating: V already holds the starting basis (preconditioner X), not I
  long long* uprod;         // null, or out: executed phase-U digit products per row (profiling)
  int* gexp;                // [2] scratch: max log2(|gamma|^2 / (alpha_p alpha_q)) of a sweep (by parity)
  int e2_hint;              // < 0: expected log2 of that ratio before sweep 1 (preconditioned); 0: none
  long long* evals;         // out: pair evaluations (gamma computed) over all sweeps
  int* cexp;                // null (MPS_NO_CERT=1: the paper's rotation-free stopping sweep), or [6]
                            // scratch of the certified stop (R21): by sweep parity [2k]
                            // max log2 bound of mu^2, [2k+1] of rho^2; [4] out: 1 = ended on it
  const int* done;          // null, or [1]: 1 = converged by the first-order finish (fo.cuh, R23)
};

// Sort / truncate / renormalise one SVD result and produce the split outputs.
template <int NL>
struct FinItem {
  int M, N, trans;          // Jacobi geometry; Theta' is (trans ? N x M : M x N)
  const int32_t* A; const int64_t* eA; const int32_t* V;
  const mpf<NL>* alpha;
  int chi_max;
  mpf<NL> thr;              // truncation threshold
  // scratch / outputs (device)
  int* ord;                 // [N] sorted column order
  mpf<NL>* inv_sig;         // [N] 1/sigma of sorted kept columns
  mpf<NL>* lam;             // [N] lambda' of kept (mpf)
  int* k_out;               // 1
  int* status;              // 1 (out: svd status if nonzero, else -4 when k = 0, else 0)
  const int* svd_status;    // the Jacobi status of this problem, or null
  const int64_t* eV;        // per-column exponents of V (recovered V), or null (= 1)
  uint32_t* sigma_rec;      // [nsig] records (sigma, descending) or null
  int nsig;                 // number of sigma records to write (<= N)
  uint32_t* lam_rec;        // [k] records or null
  // split outputs (records) — left: Gamma_L[i][a][b] = Ul[(i,a),b] / lamL(a)
  uint32_t* GL; int GL_ld;  // row stride (>= k) in complex records, or null
  const uint32_t* lamL;     // chiL records (null = ones)
  int chiL_out;             // rows of Ul = 2*chiL_out  (i, a)
  // right: Gamma_R[j][b][c] = conj(Wr[(j,c),b]) / lamR(c)
  uint32_t* GR; int GR_ld;  // GR[(j*GR_ld + b)*chiR + c]
  const uint32_t* lamR;     // chiR records (null = ones)
  int chiR_out;
  // optional M2 build (three-site): M2[(i,a),(j,b)] = Ul[(2i+j)chiL2 + a, b] * w_b
  int32_t* M2; int64_t* eM2; int M2_trans; int chiL2;
  int32_t* M2_A0; int64_t* M2_eA0;  // optional copy of M2 at one block exponent (V recovery of SVD#2)
  // V was recovered (eV != null): *redo = 1 when the kept spectrum spans more than 2^redo_bits
  // (sigma_1 / sigma_k), where the recovered V is not accurate enough (R16)
  int* redo; int redo_bits;
};

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void ldfx(const int32_t* base, int ld, int col, int ri, int row, int32_t (&x)[L]) {
  const int32_t* p = base + ((size_t)(col * 2 + ri) * L) * ld + row;
#pragma unroll
  for (int k = 0; k < L; ++k) x[k] = p[(size_t)k * ld];
}
template <int L>
__device__ __forceinline__ void stfx(int32_t* base, int ld, int col, int ri, int row, const int32_t (&x)[L]) {
  int32_t* p = base + ((size_t)(col * 2 + ri) * L) * ld + row;
#pragma unroll
  for (int k = 0; k < L; ++k) p[(size_t)k * ld] = x[k];
}

__device__ __forceinline__ int64_t rec_exp(const uint32_t* rec) { return rec_get_exp(rec); }

// keep-carry normalisation of L+2 accumulator columns (the last one absorbs)
template <int L>
__device__ __forceinline__ void tnorm2(int64_t (&acc)[L + 2]) {
  int64_t carry = 0;
#pragma unroll
  for (int c = 0; c <= L; ++c) {
    int64_t v = acc[c] + carry;
    carry = (v + HALF) >> RADIX;
    acc[c] = v - (carry << RADIX);
  }
  acc[L + 1] += carry;
}
template <int L>
__device__ __forceinline__ void tmul_acc2(int64_t (&acc)[L + 2], const int32_t (&x)[L], const int32_t (&y)[L]) {
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(x[i], y[j], acc[i + j - (L - 2)]);
}
template <int L>
__device__ __forceinline__ void tmul_sub2(int64_t (&acc)[L + 2], const int32_t (&x)[L], const int32_t (&y)[L]) {
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(-x[i], y[j], acc[i + j - (L - 2)]);
}

// Round sum V (acc columns L-2 .. 2L-1, acc[L+1] the top column) to
// round(V 2^(-g) / 2^(28L)) for 0 <= g <= 27 (used by the GEMMs for head-room).
template <int L>
__device__ __forceinline__ void tround_sr(int64_t (&acc)[L + 2], int g, int32_t (&out)[L]) {
  tnorm2<L>(acc);
  // multiply by 2^(28-g): digits <= 2^27 * 2^28 fits
  const int sh = 28 - g;
  int64_t ext[L + 3];
  int64_t carry = 0;
#pragma unroll
  for (int c = 0; c <= L + 1; ++c) {
    int64_t v = (acc[c] << sh) + carry;
    carry = (v + HALF) >> RADIX;
    ext[c] = v - (carry << RADIX);
  }
  ext[L + 2] = carry;
  // now V' = V 2^(28-g) with columns L-2 .. 2L ; result = round(V' / 2^(28(L+1)))
  // -> drop ext[0], ext[1], ext[2] (columns L-2, L-1, L); keep ext[3..L+2] (L digits)
  int64_t c0 = (ext[0] + HALF) >> RADIX;
  int64_t c1 = (ext[1] + c0 + HALF) >> RADIX;
  int64_t c2 = (ext[2] + c1 + HALF) >> RADIX;
  carry = c2;
#pragma unroll
  for (int j = 0; j < L - 1; ++j) {
    int64_t v = ext[j + 3] + carry;
    carry = (v + HALF) >> RADIX;
    out[j] = (int32_t)(v - (carry << RADIX));
  }
  out[L - 1] = (int32_t)(ext[L + 2] + carry);
}

// acc (L+2 columns: L-2 .. 2L-1) += K * x with K an (L+1)-digit coefficient
// (digit L = integer part, only formed when hasInt); x an L-digit number.
template <int L>
__device__ __forceinline__ void kmul_acc(int64_t (&acc)[L + 2], const int32_t (&K)[L + 1], const int32_t (&x)[L],
                                         bool hasInt) {
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(K[i], x[j], acc[i + j - (L - 2)]);
  if (hasInt) {
#pragma unroll
    for (int j = 0; j < L; ++j) acc[j + 2] = madw(K[L], x[j], acc[j + 2]);
  }
}
// acc += K x where the top Z fractional digits of K are known to be zero (late sweeps of a
// preconditioned Jacobi: s ~ 2^-46, 2^-92, 2^-184 and c = 1 - O(|s|^2)); digits of x that
// can only meet skipped digits of K are not loaded.  Same result as kmul_acc.
template <int L, int Z>
__device__ __forceinline__ void kmul_z(int64_t (&acc)[L + 2], const int32_t* Kp, const int32_t* xp, bool hasInt) {
  constexpr int J0 = Z >= 1 ? Z - 1 : 0;  // x digits j < J0 only pair with skipped K digits
  int32_t K[L + 1], x[L];
#pragma unroll
  for (int k = 0; k <= L; ++k) K[k] = (k < L - Z || k == L) ? Kp[k] : 0;
#pragma unroll
  for (int k = 0; k < L; ++k) x[k] = (k >= J0 || hasInt) ? xp[k * 32] : 0;
#pragma unroll
  for (int i = 0; i < L - Z; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(K[i], x[j], acc[i + j - (L - 2)]);
  if (hasInt) {
#pragma unroll
    for (int j = 0; j < L; ++j) acc[j + 2] = madw(K[L], x[j], acc[j + 2]);
  }
}
// round(V / 2^(28L)) of the L+2 accumulator columns (L-2 .. 2L-1) to L digits
template <int L>
__device__ __forceinline__ void tround2(int64_t (&acc)[L + 2], int32_t (&out)[L]) {
  tnorm2<L>(acc);
  int64_t c0 = (acc[0] + HALF) >> RADIX;
  int64_t carry = (acc[1] + c0 + HALF) >> RADIX;
#pragma unroll
  for (int j = 0; j < L - 1; ++j) {
    int64_t v = acc[j + 2] + carry;
    carry = (v + HALF) >> RADIX;
    out[j] = (int32_t)(v - (carry << RADIX));
  }
  out[L - 1] = (int32_t)(acc[L + 1] + carry);
}
// mpf -> (L+1)-digit coefficient at scale 1 (value = sum d_k 2^(28k) 2^(-28L)), |a| < 2^27
template <int NL, int L>
__device__ __forceinline__ void mpf_to_coef(const mpf<NL>& a, int32_t* out) {
  int32_t d[L + 1];
  mpf_to_fixed<NL, L + 1>(a, 28, d);  // L+1 digits at exponent 28: same digit weights as E = 0, one more digit
#pragma unroll
  for (int k = 0; k <= L; ++k) out[k] = d[k];
}

template <int L>
__device__ __forceinline__ void fx_to_cols(const int32_t (&x)[L], int64_t (&c)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) c[k] = x[k];
}

// log2 |a| as double (a != 0)
template <int NL>
__device__ __forceinline__ double mpf_log2(const mpf<NL>& a) {
  int64_t E;
  double f = fabs(mpf_frexp(a, &E));
  return (double)E + log2(f);
}

// 64-bit warp all-reduce (sum)
__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ void rr_pair(int N, int step, int i, int& p, int& q) {
  const int m = N - 1;
  if (i == 0) { p = step; q = m; }
  else { p = (step + i) % m; q = (step - i + m) % m; }
  if (p > q) { int t = p; p = q; q = t; }
}

// ----------------------------------------------------------------------------
// a1 preparation: scaled site tensor -> fixed matrix with a block exponent
// ----------------------------------------------------------------------------
static __global__ void k_init_exp(int64_t* e, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) e[i] = INT64_MIN;
}
// every PrepItem's block exponent <- INT64_MIN
static __global__ void k_init_prep(const PrepItem* items, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) *items[i].eF = INT64_MIN;
}
// *acc += *add ; if (*st == 0) *st = *st2
static __global__ void k_add_int(int* acc, const int* add, int* st, const int* st2) {
  *acc += *add;
  if (*st == 0) *st = *st2;
}
// eL, eR (first two int64 of each item's small area) <- INT64_MIN
static __global__ void k_init_exp_items(char* small0, size_t stride, int n) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) {
    int64_t* e = (int64_t*)(small0 + (size_t)b * stride);
    e[0] = INT64_MIN;
    e[1] = INT64_MIN;
  }
}

// pass 1: block exponent upper bound = max over entries of exp(lamL)+exp(G)+exp(lamR)
static __global__ void k_prep_exp(const PrepItem* items, int RB) {
  const PrepItem it = items[blockIdx.y];
  const int rb = RB;  // bytes per real record / 4
  const int n = 2 * it.da * it.db;
  int64_t best = INT64_MIN;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = t / (it.da * it.db), a = (t / it.db) % it.da, b = t % it.db;
    const uint32_t* g = it.G + (size_t)(2 * t) * rb;
    int64_t eg = max(rec_exp(g), rec_exp(g + rb));
    if (eg == INT64_MIN) continue;
    int64_t e = eg;
    if (it.lamL) { int64_t x = rec_exp(it.lamL + (size_t)a * rb); if (x == INT64_MIN) continue; e += x; }
    if (it.lamR) { int64_t x = rec_exp(it.lamR + (size_t)b * rb); if (x == INT64_MIN) continue; e += x; }
    (void)i;
    best = max(best, e);
  }
  // block reduce via atomics on the item exponent
  if (best != INT64_MIN) atomicMax((long long*)it.eF, (long long)best);
}

template <int L, int NL>
__global__ void k_prep_conv(const PrepItem* items, int RB) {
  const PrepItem it = items[blockIdx.y];
  const int rb = RB;
  const int n = 2 * it.da * it.db;
  int64_t E = *it.eF;
  if (E == INT64_MIN) E = 0;  // all-zero tensor
  const int rows = it.mode == 0 ? 2 * it.da : it.da;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = t / (it.da * it.db), a = (t / it.db) % it.da, b = t % it.db;
    const uint32_t* g = it.G + (size_t)(2 * t) * rb;
    mpf<NL> s = mpf_from_int<NL>(1);
    bool zero = false;
    if (it.lamL) s = mpf_from_record<NL>(it.lamL + (size_t)a * rb, rb - 4);
    if (it.lamR) s = mpf_mul(s, mpf_from_record<NL>(it.lamR + (size_t)b * rb, rb - 4));
    if (mpf_is_zero(s)) zero = true;
    int row, col;
    if (it.mode == 0) { row = i * it.da + a; col = b; }
    else { row = a; col = i * it.db + b; }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      int32_t d[L];
      mpf<NL> v = zero ? mpf_zero<NL>() : mpf_mul(s, mpf_from_record<NL>(g + ri * rb, rb - 4));
      mpf_to_fixed<NL, L>(v, E, d);
      stfx<L>(it.F, rows, col, ri, row, d);
    }
  }
}

// ----------------------------------------------------------------------------
// a1 contraction: batched complex fixed-point GEMM (one thread per C entry)
// ----------------------------------------------------------------------------
// Worst-case gain of one accumulator column of the truncated product (columns i + j >= L - 2)
// per k of the three-product contraction: the digit sums xr + xi, yr + yi are < 2^28 in
// magnitude except the top digit (index L - 1), which may reach 2^29 (top digits of a column
// with one integer digit of head-room reach 2^28), so a pair (i, j) adds < b(i) b(j) with
// b = 2^28, b(L - 1) = 2^29.  Column s = i + j collects min(s, 2L - 2 - s) + 1 pairs.
template <int L>
__host__ __device__ constexpr double gemm3m_col_gain() {
  double worst = 0;
  for (int s = L - 2; s <= 2 * L - 2; ++s) {
    double g = 0;
    for (int i = 0; i < L; ++i) {
      const int j = s - i;
      if (j < 0 || j >= L) continue;
      g += (i == L - 1 ? 536870912.0 : 268435456.0) * (j == L - 1 ? 536870912.0 : 268435456.0);
    }
    worst = g > worst ? g : worst;
  }
  return worst;
}
// k between normalisations: a column starts below 2^28 after tnorm2 and must stay below
// 2^63 - 2^32 (at most 8: beyond that the saved tnorm2 calls no longer matter).  L = 10:
// gain 12 * 2^56 per k -> 8; L = 19: 21 * 2^56 -> 6.
template <int L>
__host__ __device__ constexpr int gemm3m_norm_every() {
  const int n = (int)((9223372036854775808.0 - 4294967296.0) / gemm3m_col_gain<L>());
  return n > 8 ? 8 : n;
}
static_assert(gemm3m_norm_every<10>() == 8 && gemm3m_norm_every<19>() == 6, "contraction column bound");
static_assert(gemm3m_norm_every<19>() * gemm3m_col_gain<19>() + 268435456.0 < 9223372036854775808.0,
              "contraction columns fit int64 between normalisations");

template <int L>
__global__ void k_gemm(const GemmItem* items) {
  const GemmItem it = items[blockIdx.y];
  const int n = it.rows * it.cols;
  // head-room: sum of K complex products each |.| < 2^(eA+eB+1)
  int g = 1;
  while ((1 << (g - 1)) < it.K) ++g;  // 2^(g-1) >= K
  g += 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) *it.eC = *it.eA + *it.eB + g;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % it.rows, c = t / it.rows;
    // three real products per complex product: re = sum xr yr - sum xi yi,
    // im = sum (xr + xi)(yr + yi) - sum xr yr - sum xi yi; the columns are normalised every
    // gemm3m_norm_every<L>() k (worst-case column gain per k: gemm3m_col_gain, below)
    int64_t ar[L + 2], ai[L + 2], as[L + 2];
#pragma unroll
    for (int j = 0; j < L + 2; ++j) ar[j] = ai[j] = as[j] = 0;
    int cnt = 0;
    for (int k = 0; k < it.K; ++k) {
      int32_t xr[L], xi[L], yr[L], yi[L];
      if (it.conjA) {  // A stored K x rows: op(A)(r,k) = conj(A(k, r))
        ldfx<L>(it.A, it.lda, r, 0, k, xr);
        ldfx<L>(it.A, it.lda, r, 1, k, xi);
#pragma unroll
        for (int j = 0; j < L; ++j) xi[j] = -xi[j];
      } else {
        ldfx<L>(it.A, it.lda, k, 0, r, xr);
        ldfx<L>(it.A, it.lda, k, 1, r, xi);
      }
      ldfx<L>(it.B, it.ldb, c, 0, k, yr);
      ldfx<L>(it.B, it.ldb, c, 1, k, yi);
      tmul_acc2<L>(ar, xr, yr);
      tmul_acc2<L>(ai, xi, yi);
#pragma unroll
      for (int j = 0; j < L; ++j) { xr[j] += xi[j]; yr[j] += yi[j]; }
      tmul_acc2<L>(as, xr, yr);
      constexpr int NORM_EVERY = gemm3m_norm_every<L>();
      if (++cnt == NORM_EVERY) { cnt = 0; tnorm2<L>(ar); tnorm2<L>(ai); tnorm2<L>(as); }
    }
    tnorm2<L>(ar);
    tnorm2<L>(ai);
    tnorm2<L>(as);
#pragma unroll
    for (int j = 0; j < L + 2; ++j) {
      const int64_t t1 = ar[j], t2 = ai[j];
      ar[j] = t1 - t2;
      ai[j] = as[j] - t1 - t2;
    }
    int32_t o[L];
    tround_sr<L>(ar, g, o);
    stfx<L>(it.C, it.ldc, c, 0, r, o);
    tround_sr<L>(ai, g, o);
    stfx<L>(it.C, it.ldc, c, 1, r, o);
  }
}

// ----------------------------------------------------------------------------
// a2 gate application -> Jacobi layout (one thread per Theta' entry)
// ----------------------------------------------------------------------------
template <int L, int NL>
__global__ void k_mix(const MixItem* items, int RBr) {
  const MixItem it = items[blockIdx.y];
  const int D = 2 * it.RB;
  const int rows = it.RB * it.chiL, cols = 2 * it.chiR;
  const int n = rows * cols;
  // U as fixed digits at exponent 1 (|U_xy| <= 1 < 2^1) — staged in shared memory
  extern __shared__ int32_t su[];  // [D*D][2][L]
  for (int t = threadIdx.x; t < D * D; t += blockDim.x) {
    for (int ri = 0; ri < 2; ++ri) {
      mpf<NL> u = mpf_from_record<NL>(it.U + (size_t)(2 * t + ri) * RBr, RBr - 4);
      int32_t d[L];
      mpf_to_fixed<NL, L>(u, 1, d);
      for (int k = 0; k < L; ++k) su[(t * 2 + ri) * L + k] = d[k];
    }
  }
  __syncthreads();
  int g = 2;
  while ((1 << (g - 2)) < D) ++g;  // sum of D terms, |U| <= 1 (modulus < 2^0.5 per comp)
  const int64_t eOut = *it.eT + 1 + g;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % rows, c = t / rows;
    const int rb = r / it.chiL, a = r % it.chiL, cb = c / it.chiR, gg = c % it.chiR;
    const int x = 2 * rb + cb;
    int64_t ar[L + 2], ai[L + 2];
#pragma unroll
    for (int j = 0; j < L + 2; ++j) ar[j] = ai[j] = 0;
    for (int y = 0; y < D; ++y) {
      const int rr = (y >> 1) * it.chiL + a, cc = (y & 1) * it.chiR + gg;
      int32_t tr[L], ti[L], ur[L], ui[L];
      ldfx<L>(it.T, it.ldt, cc, 0, rr, tr);
      ldfx<L>(it.T, it.ldt, cc, 1, rr, ti);
#pragma unroll
      for (int k = 0; k < L; ++k) { ur[k] = su[((x * D + y) * 2 + 0) * L + k]; ui[k] = su[((x * D + y) * 2 + 1) * L + k]; }
      tmul_acc2<L>(ar, ur, tr);
      tmul_sub2<L>(ar, ui, ti);
      tmul_acc2<L>(ai, ur, ti);
      tmul_acc2<L>(ai, ui, tr);
    }
    int32_t o[L];
    if (!it.trans) {
      tround_sr<L>(ar, g, o); stfx<L>(it.A, it.M, c, 0, r, o);
      tround_sr<L>(ai, g, o); stfx<L>(it.A, it.M, c, 1, r, o);
      if (r == 0) it.eA[c] = eOut;
    } else {  // A = Theta'^H : A(c, r) = conj(Theta'(r, c))
      tround_sr<L>(ar, g, o); stfx<L>(it.A, it.M, r, 0, c, o);
      tround_sr<L>(ai, g, o);
#pragma unroll
      for (int k = 0; k < L; ++k) o[k] = -o[k];
      stfx<L>(it.A, it.M, r, 1, c, o);
      if (c == 0) it.eA[r] = eOut;
    }
  }
}

// fixed matrix (Jacobi layout with per-column exponents, or block exponent if eCol==null)
// -> column-major complex records (debug / theta output).  conjT: output (ThetaT)^H.
template <int L, int NL>
__global__ void k_fixed_to_records(const int32_t* F, int ld, const int64_t* eCol, const int64_t* eBlock,
                                   int rows, int cols, int conjT, uint32_t* out, int RBr, int p) {
  const int n = rows * cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % rows, c = t / rows;
    const int64_t E = eCol ? eCol[c] : *eBlock;
    for (int ri = 0; ri < 2; ++ri) {
      int32_t x[L];
      ldfx<L>(F, ld, c, ri, r, x);
      int64_t cols_[L];
      fx_to_cols<L>(x, cols_);
      mpf<NL> v = mpf_from_cols<NL, L>(cols_, E - 28 * (int64_t)L);
      if (conjT && ri == 1) v = mpf_neg(v);
      // output index: column-major of the (possibly transposed) matrix
      size_t o = conjT ? ((size_t)r * cols + c) : ((size_t)c * rows + r);
      mpf_to_record<NL>(v, out + (2 * o + ri) * (size_t)RBr, RBr - 4, p);
    }
  }
}

// ----------------------------------------------------------------------------
// a3 one-sided Jacobi SVD (one CTA per matrix, round-robin ordering)
// ----------------------------------------------------------------------------
template <int L, int NL>
__device__ void jac_norms(const SvdItem<NL>& it, bool set_negl, const mpf<NL>& z, int gw, int GW) {
  const int lane = threadIdx.x & 31;
  const int W = 28 * L;
  for (int j = gw; j < it.N; j += GW) {
    int64_t acc[L + 2];
#pragma unroll
    for (int c = 0; c < L + 2; ++c) acc[c] = 0;
    int cnt = 0;
    for (int r = lane; r < it.M; r += 32) {
      int32_t xr[L], xi[L];
      ldfx<L>(it.A, it.M, j, 0, r, xr);
      ldfx<L>(it.A, it.M, j, 1, r, xi);
      tmul_acc2<L>(acc, xr, xr);
      tmul_acc2<L>(acc, xi, xi);
      if (++cnt == 8) { cnt = 0; tnorm2<L>(acc); }
    }
    tnorm2<L>(acc);
#pragma unroll
    for (int c = 0; c < L + 2; ++c) acc[c] = warp_sum64(acc[c]);
    int64_t ej = it.eA[j];
    int shift = 0;
    if (lane == 0) {
      mpf<NL> a = mpf_from_cols<NL, L + 2>(acc, 28 * (int64_t)(L - 2) + 2 * ej - 2 * (int64_t)W);
      // renormalise: target exponent = ceil(log2 ||a||) + 1
      if (!mpf_is_zero(a)) {
        double lg = 0.5 * mpf_log2(a);
        int64_t target = (int64_t)ceil(lg + 1e-9) + 1;
        if (ej - target >= 2) {
          int64_t k = ej - target;
          if (k > 28 * L - 2) k = 28 * L - 2;
          shift = (int)k;
        }
      }
      it.alpha[j] = a;
      if (set_negl && (mpf_is_zero(a) || mpf_cmp(a, z) <= 0)) it.negl[j] = 1;
    }
    shift = __shfl_sync(0xffffffffu, shift, 0);
    if (shift) {
      const int q = shift / 28, rbit = shift % 28;
      for (int r = lane; r < it.M; r += 32) {
        for (int ri = 0; ri < 2; ++ri) {
          int32_t x[L];
          ldfx<L>(it.A, it.M, j, ri, r, x);
          int64_t y[L];
#pragma unroll
          for (int k = 0; k < L; ++k) y[k] = (k - q >= 0) ? ((int64_t)x[k - q] << rbit) : 0;
          int64_t carry = 0;
#pragma unroll
          for (int k = 0; k < L; ++k) {
            int64_t v = y[k] + carry;
            carry = (v + HALF) >> RADIX;
            x[k] = (int32_t)(v - (carry << RADIX));
          }
          x[L - 1] += (int32_t)(carry << RADIX);
          stfx<L>(it.A, it.M, j, ri, r, x);
        }
      }
      if (lane == 0) it.eA[j] = ej - shift;
    }
  }
}

// cp.async staging helpers (4-byte copies, zero-fill past the matrix edge)
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NW>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NW)); }

// 16-byte copy of `bytes` (0..16) valid bytes, the rest zero-filled (L2 only: streamed data)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// Stage rows [row0, row0+32) of the four operand columns (p re, p im, q re, q im) of a
// fixed matrix into buf[4][L][32] (one row per lane of the consumer).  When ld is a
// multiple of 4 words each lane moves 16 bytes (4 rows of one digit plane): lanes 8o..8o+7
// copy operand o, L copies per lane; otherwise one 4-byte copy per row and plane.
// LG (<= L): only the top LG digits of each value are staged, as buf[4][LG][32].
template <int L, int LG = L>
__device__ __forceinline__ void stage_rows(int32_t* buf, const int32_t* F, int ld, int p, int q, int row0, int rows,
                                          int lane) {
  if ((ld & 3) == 0) {
    const int op = lane >> 3, sub = lane & 7;
    const int col = op < 2 ? p : q, ri = op & 1;
    const int r = row0 + 4 * sub;
    int nv = rows - r;
    nv = nv < 0 ? 0 : (nv > 4 ? 4 : nv);
    const int32_t* g = F + ((size_t)(col * 2 + ri) * L + (L - LG)) * ld + (nv ? r : 0);
    int32_t* d = buf + op * LG * 32 + 4 * sub;
#pragma unroll
    for (int k = 0; k < LG; ++k) {
      cp_async16(d + k * 32, g, 4 * nv);
      g += ld;
    }
    return;
  }
  const int r = row0 + lane;
  const bool ok = r < rows;
  const int rr = ok ? r : 0;
#pragma unroll
  for (int op = 0; op < 4; ++op) {
    const int col = op < 2 ? p : q, ri = op & 1;
    const int32_t* g = F + ((size_t)(col * 2 + ri) * L + (L - LG)) * ld + rr;
#pragma unroll
    for (int k = 0; k < LG; ++k) cp_async4(buf + (op * LG + k) * 32 + lane, g + (size_t)k * ld, ok);
  }
}

// Per output o of (y_p.re, y_p.im, y_q.re, y_q.im): operand index of its three terms
// (0 x_p.re, 1 x_p.im, 2 x_q.re, 3 x_q.im); coefficients (sign folded) are stored as
// [mat][o][t] in the same order:
//   y_p.re = +Cp xrp - Psr xrq - Psi xiq     y_p.im = +Cp xip - Psr xiq + Psi xrq
//   y_q.re = +Cq xrq + Qsr xrp - Qsi xip     y_q.im = +Cq xiq + Qsr xip + Qsi xrp
// with Psr+iPsi = s 2^(eq-eo_p) (conj(s) multiplies x_q), Qsr+iQsi = s 2^(ep-eo_q),
// Cp = c 2^(ep-eo_p), Cq = c 2^(eq-eo_q); for V all scales are 1.
__constant__ int c_opidx[4][3] = {{0, 2, 3}, {1, 3, 2}, {2, 0, 1}, {3, 1, 0}};  // term 0: the c term
// slot u <- (+/-) vals[src & 15] of the 9 distinct values {Cp, Psr, Psi, Qsr, Qsi, Cq, c,
// sr, si}; bit 4 = negate
__constant__ int8_t c_coefsrc[24] = {0, 1 | 16, 2 | 16, 0, 1 | 16, 2, 5, 3, 4 | 16, 5, 3, 4,
                                     6, 7 | 16, 8 | 16, 6, 7 | 16, 8, 6, 7, 8 | 16, 6, 7, 8};

// Phase U for one 32-row chunk: the four outputs (y_p re/im, y_q re/im) of the staged rows,
// term 0 of each output being its c term.  ZC / ZS: known-zero top fractional digits of the
// c / s coefficients of this pair (U_VARIANTS, chosen in phase R from the actual digits).
template <int L, int ZC, int ZS>
__device__ __forceinline__ void u_chunk(int32_t* F, int rows, int p, int q, int r, int lane, const int32_t* b,
                                        const int32_t* wcoef, int mat, int flag) {
  constexpr int CW = L + 1;
#pragma unroll 1
  for (int o = 0; o < 4; ++o) {
    const int ib = 8 + (mat * 4 + o) * 3;  // integer-digit bits of this output's three slots
    int64_t acc[L + 2];
#pragma unroll
    for (int c = 0; c < L + 2; ++c) acc[c] = 0;
    const int32_t* Kp = wcoef + ((mat * 4 + o) * 3) * CW;
    kmul_z<L, ZC>(acc, Kp, b + c_opidx[o][0] * L * 32 + lane, (flag >> ib) & 1);
    kmul_z<L, ZS>(acc, Kp + CW, b + c_opidx[o][1] * L * 32 + lane, (flag >> (ib + 1)) & 1);
    kmul_z<L, ZS>(acc, Kp + 2 * CW, b + c_opidx[o][2] * L * 32 + lane, (flag >> (ib + 2)) & 1);
    int32_t out[L];
    tround2<L>(acc, out);
    if (r < rows) stfx<L>(F, rows, o < 2 ? p : q, o & 1, r, out);
  }
}
// Phase D for one pair: gamma = sum_r conj(a_p(r)) a_q(r) from the top LG digits of the
// columns (a truncated LG-digit product: absolute error ~2^-(28 LG - 6) ||a_p|| ||a_q||).
// LG < L in the sweeps where the off-diagonal is still large (R20); the sweep that
// ends the iteration always uses LG = L.
template <int L, int NL, int LG, int JST>
__device__ __forceinline__ void d_pair(const SvdItem<NL>& it, int32_t* wbuf, int p, int q, int i, int lane, int nchA) {
  constexpr int STAGE = 4 * L * 32;
  const int M = it.M;
  int64_t gr[LG + 2], gi[LG + 2];
#pragma unroll
  for (int c = 0; c < LG + 2; ++c) gr[c] = gi[c] = 0;
  stage_rows<L, LG>(wbuf, it.A, M, p, q, 0, M, lane);
  cp_commit();
  for (int ch = 0; ch < nchA; ++ch) {
    if (JST == 2 && ch + 1 < nchA) {
      stage_rows<L, LG>(wbuf + ((ch + 1) & 1) * STAGE, it.A, M, p, q, (ch + 1) * 32, M, lane);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncwarp();
    const int32_t* b = wbuf + (JST == 2 ? (ch & 1) * STAGE : 0);
    int32_t xa[LG], xb[LG];
    // rows past M were zero-filled: their products vanish
#pragma unroll
    for (int k = 0; k < LG; ++k) { xa[k] = b[(0 * LG + k) * 32 + lane]; xb[k] = b[(2 * LG + k) * 32 + lane]; }
    tmul_acc2<LG>(gr, xa, xb);  // xrp xrq
#pragma unroll
    for (int k = 0; k < LG; ++k) xb[k] = b[(3 * LG + k) * 32 + lane];
    tmul_acc2<LG>(gi, xa, xb);  // xrp xiq
#pragma unroll
    for (int k = 0; k < LG; ++k) xa[k] = b[(1 * LG + k) * 32 + lane];
    tmul_acc2<LG>(gr, xa, xb);  // xip xiq
#pragma unroll
    for (int k = 0; k < LG; ++k) xb[k] = b[(2 * LG + k) * 32 + lane];
    tmul_sub2<LG>(gi, xa, xb);  // - xip xrq
    if ((ch & 7) == 7) { tnorm2<LG>(gr); tnorm2<LG>(gi); }
    __syncwarp();
    if (JST == 1 && ch + 1 < nchA) {
      stage_rows<L, LG>(wbuf, it.A, M, p, q, (ch + 1) * 32, M, lane);
      cp_commit();
    }
  }
  tnorm2<LG>(gr);
  tnorm2<LG>(gi);
  // cross-lane column sums through shared memory (the staging buffer is free now):
  // lane l writes its 2(LG+2) columns, lanes 0..2(LG+2)-1 each sum one column over 32 lanes
  int64_t* red = (int64_t*)wbuf;  // [2(LG+2)][32]
  __syncwarp();
#pragma unroll
  for (int c = 0; c < LG + 2; ++c) { red[c * 32 + lane] = gr[c]; red[(LG + 2 + c) * 32 + lane] = gi[c]; }
  __syncwarp();
  int64_t sum[2] = {0, 0};  // 2(LG+2) columns over 32 lanes (two rounds when LG > 14)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (c < 2 * (LG + 2)) {
#pragma unroll 8
      for (int l = 0; l < 32; ++l) sum[h] += red[c * 32 + ((l + lane) & 31)];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (lane + 32 * h < 2 * (LG + 2)) red[lane + 32 * h] = sum[h];
  __syncwarp();
  // lane 0 converts gamma_re, lane 1 gamma_im (in parallel)
  if (lane < 2) {
    int64_t cols[LG + 2];
#pragma unroll
    for (int c = 0; c < LG + 2; ++c) cols[c] = red[lane * (LG + 2) + c];
    const int64_t E0 = 28 * (int64_t)(LG - 2) + it.eA[p] + it.eA[q] - 2 * 28 * (int64_t)LG;
    it.gam[2 * i + lane] = mpf_from_cols<NL, LG + 2>(cols, E0);
  }
  __syncwarp();
}

// variants (ZC, ZS), 280 bits: 0 = (0, 0), 1 = (3, 1), 2 = (6, 3), 3 = (10, 5); 512 bits: (0, 0),
// (3, 1), (10, 5), (19, 10).  After the refinement sweeps (R22) the p-bit sweeps rotate by
// |s| ~ 2^-155 (c = 1 - O(2^-310): no fractional digit) and, at 512 bits, then ~2^-310.
template <int L>
__host__ __device__ constexpr int u_var_zc(int v) { return v == 0 ? 0 : v == 1 ? 3 : v == 2 ? (L < 19 ? 6 : 10) : (L < 19 ? L : 19); }
template <int L>
__host__ __device__ constexpr int u_var_zs(int v) { return v == 0 ? 0 : v == 1 ? 1 : v == 2 ? (L < 19 ? 3 : 5) : (L < 19 ? 5 : 10); }

// Staging buffers per warp and resident CTAs per SM of k_jacobi.  280 bits: double
// buffering, 2 CTAs (16 warps, 128 registers).  The alternative of one buffer and 3 CTAs
// (24 warps, 80 registers with spills; -DJACOBI_STAGES_280=1 -DJACOBI_CTAS_280=3) measured
// 33.9 vs 34.3 updates/s per full wave and fits 1024 items worse (2.3 waves).  512 bits:
// double buffering, 1 CTA.
template <int L>
__host__ __device__ constexpr int jacobi_stages() { return L <= 10 ? JACOBI_STAGES_280 : 2; }
template <int L>
__host__ __device__ constexpr int jacobi_min_ctas() { return L <= 10 ? JACOBI_CTAS_280 : 1; }

// C CTAs (a thread-block cluster when C > 1) cooperate on one matrix: pairs, columns and
// rows are distributed over all C*NWARP warps, column state lives in global memory, and
// the phases are separated by cluster barriers.  The arithmetic of every pair is the same
// whatever C is, so results are bitwise independent of C.
// debug (MPS_JACOBI_TRACE=k): the first k matrices of a launch print, per sweep, the bounds of
// the certified stop (R21): log2 rho^2_max, log2 mu^2_max, rotations seen, certified
static __device__ int jac_trace_items;

template <int L, int NL>
__global__ void __launch_bounds__(NTHR, jacobi_min_ctas<L>()) k_jacobi(const SvdItem<NL>* items, int C) {
  namespace cg = cooperative_groups;
  const int crank = C > 1 ? (int)(blockIdx.x % C) : 0;
  const SvdItem<NL> it = items[C > 1 ? blockIdx.x / C : blockIdx.x];
  if (it.done && *it.done) return;  // converged by the first-order finish (R23): outputs written
  auto csync = [&]() {
    if (C > 1) cg::this_cluster().sync();
    else __syncthreads();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int gw = crank * NWARP + warp, GW = C * NWARP;       // global warp id / count
  const int gt = crank * NTHR + tid, GT = C * NTHR;          // global thread id / count
  const int M = it.M, N = it.N, NP = N / 2;
  const int W = 28 * L;
  constexpr int CW = L + 1;              // words per coefficient vector
  constexpr int STAGE = 4 * L * 32;      // words per staging buffer
  constexpr int JST = jacobi_stages<L>();
  extern __shared__ int32_t jsm[];
  int32_t* wbuf = jsm + warp * (JST * STAGE + 24 * CW);  // per warp: JST stage buffers + 24 coefficients
  int32_t* wcoef = wbuf + JST * STAGE;
  static_assert(2 * (L + 2) * 32 * 8 <= (JST * STAGE + 24 * CW) * 4, "phase-D column sums must fit the warp's buffers");
  __shared__ mpf<NL> s_red[1];

  if (crank == 0 && tid == 0) {
    *it.rotations = 0; *it.evals = 0;
    if (it.uprod) *it.uprod = 0;
    if (it.cexp) it.cexp[4] = 0;
  }
  const bool accV = it.A0 == nullptr;
  if (!accV && !it.a0_ready) {  // keep the input (block exponent from k_mix) for the recovery of V
    const size_t nw = (size_t)M * N * 2 * L;
    for (size_t t = gt; t < nw; t += GT) it.A0[t] = it.A[t];
    if (gt == 0) *it.eA0 = it.eA[0];
  }
  // V = I (exponent 1: 1 = 2^27 * 2^(28(L-1)) * 2^(1 - 28L))
  for (int t = gt; accV && !it.v_preset && t < N * N; t += GT) {
    const int r = t % N, c = t / N;
    int32_t x[L], z0[L];
#pragma unroll
    for (int k = 0; k < L; ++k) { x[k] = 0; z0[k] = 0; }
    if (r == c) x[L - 1] = 1 << 27;
    stfx<L>(it.V, N, c, 0, r, x);
    stfx<L>(it.V, N, c, 1, r, z0);
  }
  mpf<NL> z = mpf_zero<NL>();
  jac_norms<L, NL>(it, false, z, gw, GW);
  csync();
  // ||A||_F^2 and the negligible-column floor z = tol^2 ||A||_F^2 (CTA rank 0, warp 0)
  if (crank == 0 && warp == 0) {
    mpf<NL> s = mpf_zero<NL>();
    for (int j = lane; j < N; j += 32) s = mpf_add(s, it.alpha[j]);
    if (lane == 0) s_red[0] = mpf_zero<NL>();
    __syncwarp();
    for (int l = 0; l < 32; ++l) {
      if (lane == l) s_red[0] = mpf_add(s_red[0], s);
      __syncwarp();
    }
    if (lane == 0) {
      mpf<NL> tol2 = mpf_ldexp(mpf_from_int<NL>((int64_t)M * M), 4 - 2 * (int64_t)W);
      *it.zbuf = mpf_mul(tol2, s_red[0]);
    }
  }
  csync();
  z = *it.zbuf;
  for (int j = gt; j < N; j += GT) {
    const mpf<NL> a = it.alpha[j];
    it.negl[j] = (mpf_is_zero(a) || mpf_cmp(a, z) <= 0) ? 1 : 0;
  }
  csync();
  const mpf<NL> tol2 = mpf_ldexp(mpf_from_int<NL>((int64_t)M * M), 4 - 2 * (int64_t)W);  // tol = 4 M 2^-W
  const int nchA = (M + 31) / 32, nchV = (N + 31) / 32;

  int sweep = 0, conv = 0;
  long long nrot = 0, nev = 0, nup = 0;
  const bool prof = it.phase_cycles != nullptr && tid == 0;
  unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};
  long long t_start = clock64(), t_mark = t_start;
  auto mark = [&](int slot) {
    if (prof) {
      const long long t = clock64();
      pc[slot] += (unsigned long long)(t - t_mark);
      t_mark = t;
    }
  };
  mark(4);
  // digits of the dot products per sweep (R20): sweep k+1 needs gamma to ~eps_k^2 where
  // eps_k ~ (largest |gamma|/sqrt(alpha_p alpha_q) of sweep k)^2; a reduced sweep never ends
  // the iteration
  int e2prev = it.e2_hint;
  for (sweep = 1; sweep <= MAX_SWEEPS; ++sweep) {
    int lgd = L;
    // only the first two sweeps of a preconditioned iteration may be reduced (bounded: the
    // iteration then proceeds exactly as without R20)
    if (it.gexp && it.e2_hint < 0 && sweep <= 2 && e2prev > -100000) {  // INT_MIN: no evaluated pair
      const int64_t need = -2 * (int64_t)e2prev + 8;  // bits
      lgd = need <= 28 * 4 ? 4 : (need <= 28 * 7 ? 7 : L);
      if (lgd > L) lgd = L;
    }
    if (crank == 0 && tid == 0) {
      *(volatile int*)it.sync = 0;
      if (it.gexp) it.gexp[sweep & 1] = INT_MIN;
      if (it.cexp) { it.cexp[2 * (sweep & 1)] = INT_MIN; it.cexp[2 * (sweep & 1) + 1] = INT_MIN; }
    }
    int lmu = INT_MIN, lrho = INT_MIN;  // this thread's bounds for the certified stop (R21)
    csync();
    for (int step = 0; step < N - 1; ++step) {
      // ---- phase D: gamma = sum conj(a_p) a_q (warp per pair, lanes over rows, cp.async staging)
      for (int i = gw; i < NP; i += GW) {
        int p, q;
        rr_pair(N, step, i, p, q);
        if (it.negl[p] || it.negl[q]) continue;
        if (lgd == 4) d_pair<L, NL, 4, JST>(it, wbuf, p, q, i, lane, nchA);
        else if (lgd == 7) d_pair<L, NL, (L < 7 ? L : 7), JST>(it, wbuf, p, q, i, lane, nchA);
        else d_pair<L, NL, L, JST>(it, wbuf, p, q, i, lane, nchA);
      }
      csync();
      mark(0);
      // ---- phase R: rotation parameters (thread per pair)
      for (int i = gt; i < NP; i += GT) {
        int p, q;
        rr_pair(N, step, i, p, q);
        int flag = 0;
        if (!it.negl[p] && !it.negl[q]) {
          ++nev;
          mpf<NL> ap = it.alpha[p], aq = it.alpha[q];
          const mpf<NL> gr = it.gam[2 * i], gi = it.gam[2 * i + 1];
          const mpf<NL> g2 = mpf_add(mpf_mul(gr, gr), mpf_mul(gi, gi));
          if (it.gexp && !mpf_is_zero(g2) && !mpf_is_zero(ap) && !mpf_is_zero(aq) && !ap.neg && !aq.neg) {
            const int64_t e2 = g2.e - ap.e - aq.e + 2;  // >= log2(g2 / (ap aq))
            atomicMax(&it.gexp[sweep & 1], (int)(e2 < -100000 ? -100000 : (e2 > 100000 ? 100000 : e2)));
          }
          if (it.cexp && !mpf_is_zero(g2)) {  // rho^2 = |g|^2 / (alpha_p alpha_q) < 2^e2 (values in [2^(e-1), 2^e))
            const int64_t e2 = (mpf_is_zero(ap) || mpf_is_zero(aq) || ap.neg || aq.neg) ? 1000000
                               : g2.e - ap.e - aq.e + 2;
            lrho = max(lrho, (int)(e2 < -1000000 ? -1000000 : (e2 > 1000000 ? 1000000 : e2)));
          }
          if (!mpf_is_zero(g2) && mpf_cmp(g2, mpf_mul(tol2, mpf_mul(ap, aq))) > 0) {
            // The oracle's zeta = d/(2|g|), t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)),
            // c = 1/sqrt(1 + t^2), s = c t g/|g| (d = a_q - a_p, g = gamma), rewritten with
            // r = sqrt(d^2 + 4|g|^2) and c^2 = (|d| + r)/(2r) (no cancellation, both terms
            // >= 0) so that only two inverse square roots are needed:
            //   s = sgn(d) g / (r c),  t |g| = sgn(d) |g|^2 / (r c^2)      (R17)
            const mpf<NL> d = mpf_sub(aq, ap);
            const mpf<NL> w = mpf_add(mpf_mul(d, d), mpf_ldexp(g2, 2));
            const mpf<NL> rr = mpf_rsqrt(w);                       // 1/r
            const mpf<NL> c2 = mpf_ldexp(mpf_mul(mpf_add(mpf_abs(d), mpf_mul(w, rr)), rr), -1);
            const mpf<NL> ic = mpf_rsqrt(c2);                      // 1/c
            const mpf<NL> c = mpf_mul(c2, ic);
            mpf<NL> sc = mpf_mul(rr, ic);                          // 1/(r c)
            if (!mpf_is_zero(d) && d.neg) sc = mpf_neg(sc);
            const mpf<NL> sr = mpf_mul(sc, gr);
            const mpf<NL> si = mpf_mul(sc, gi);
            const mpf<NL> tg = mpf_mul(mpf_mul(g2, sc), ic);      // t |gamma|
            if (it.cexp) {  // mu^2 = |s|^2 max(alpha_p, alpha_q) / min(alpha_p, alpha_q), |s| = |g| |sc|
              const int64_t da = ap.e > aq.e ? ap.e - aq.e : aq.e - ap.e;
              const int64_t em = g2.e + 2 * sc.e + da + 1;
              lmu = max(lmu, (int)(em < -1000000 ? -1000000 : (em > 1000000 ? 1000000 : em)));
            }
            // a reduced-precision gamma (R20) leaves the new norms uncertain by up to
            // 2 |s| |gamma error| <= 2^-(28 lgd - 7) sqrt(alpha_p alpha_q): exponent of its square root
            const int64_t e_slack = lgd < L ? (ap.e + aq.e) / 4 - (28 * (int64_t)lgd - 8) / 2 + 2 : INT64_MIN / 4;
            ap = mpf_sub(ap, tg);
            aq = mpf_add(aq, tg);
            const int64_t ep = it.eA[p], eq = it.eA[q];
            const int64_t eb = (ep > eq ? ep : eq) + 1;  // bound of every term's exponent
            // Output exponents: tight from the predicted norms (slack for rounding), but no
            // lower than (largest term exponent) - 26 so that every scaled coefficient
            // |coef| 2^(e_in - e_out) stays < 2^26 (one integer digit).  A term's exponent is
            // e_in + e(coef) with |coef| < 2^e(coef); only genuine cancellation (output much
            // smaller than its terms) leaves a column under-normalised, as in floating point.
            const int64_t ec = mpf_is_zero(c) ? INT64_MIN / 4 : c.e;
            const int64_t es = (mpf_is_zero(sr) && mpf_is_zero(si)) ? INT64_MIN / 4
                               : (mpf_is_zero(sr) ? si.e : (mpf_is_zero(si) ? sr.e : (sr.e > si.e ? sr.e : si.e)));
            const int64_t tmax[2] = {(ep + ec > eq + es ? ep + ec : eq + es) + 1,
                                     (ep + es > eq + ec ? ep + es : eq + ec) + 1};
            int64_t eo[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const mpf<NL>& a = u ? aq : ap;
              int64_t enew = tmax[u] - W + 14;
              if (!mpf_is_zero(a) && !a.neg) {
                int64_t e1 = (int64_t)ceil(0.5 * mpf_log2(a) + 1e-9) + 1;
                if (e1 > enew) enew = e1;
              }
              if (e_slack + 1 > enew) enew = e_slack + 1;
              if (enew < tmax[u] - 26) enew = tmax[u] - 26;
              if (enew > eb) enew = eb;
              eo[u] = enew;
            }
            // 24 signed coefficient vectors [mat][o][t] (layout: see c_opidx)
            int32_t* cf = it.coef + (size_t)i * 33 * CW;
            // 9 distinct values {Cp, Psr, Psi, Qsr, Qsi, Cq, c, sr, si}:
            //   Cp = c 2^(ep-eo_p), Psr + i Psi = s 2^(eq-eo_p), Qsr + i Qsi = s 2^(ep-eo_q),
            //   Cq = c 2^(eq-eo_q), and c, sr, si unscaled (V);
            // the U warp expands them into the 24 signed slots (c_coefsrc)
            int vint = 0;
#pragma unroll 1
            for (int v = 0; v < 9; ++v) {  // one copy of the conversion code (i-cache)
              const mpf<NL> base = (v == 0 || v == 5 || v == 6) ? c : ((v == 1 || v == 3 || v == 7) ? sr : si);
              const int64_t sc = v == 0 ? ep - eo[0] : v == 1 || v == 2 ? eq - eo[0] : v == 3 || v == 4 ? ep - eo[1]
                                 : v == 5 ? eq - eo[1] : 0;
              int32_t dg[L + 1];
              mpf_to_fixed<NL, L + 1>(mpf_ldexp(base, sc), 28, dg);  // coefficient digits (scale 1)
#pragma unroll
              for (int k = 0; k <= L; ++k) cf[v * CW + k] = dg[k];
              if (dg[L]) vint |= 1 << v;
            }
            int ints = 0;  // bit u: slot u's coefficient has an integer digit
            for (int u = 0; u < 24; ++u)
              if ((vint >> (c_coefsrc[u] & 15)) & 1) ints |= 1 << u;
            // the signed slots [mat][o][t] in the order phase U reads them (slots 9.. of the
            // pair's area): phase U then copies them without index arithmetic or negation
#pragma unroll 1
            for (int u = 0; u < (accV ? 24 : 12); ++u) {
              const int src = c_coefsrc[u];
              const int32_t* from = cf + (src & 15) * CW;
              int32_t* to = cf + (9 + u) * CW;
#pragma unroll
              for (int k = 0; k <= L; ++k) to[k] = (src & 16) ? -from[k] : from[k];
            }
            // zero top fractional digits of each value -> the U variant of A (values 0..5) and V (6..8)
            int zv[9];
            for (int v = 0; v < 9; ++v) {
              int z = 0;
              while (z < L && cf[v * CW + L - 1 - z] == 0) ++z;
              zv[v] = z;
            }
            int varA = 0, varV = 0;
            {
              const int zc = min(zv[0], zv[5]), zs = min(min(zv[1], zv[2]), min(zv[3], zv[4]));
              const int zcv = zv[6], zsv = min(zv[7], zv[8]);
              for (int v = 3; v >= 1; --v)
                if (u_var_zc<L>(v) <= zc && u_var_zs<L>(v) <= zs) { varA = v; break; }
              for (int v = 3; v >= 1; --v)
                if (u_var_zc<L>(v) <= zcv && u_var_zs<L>(v) <= zsv) { varV = v; break; }
            }
            if (it.phase_cycles) {  // debug: digit products a leading-zero-aware U would need
              unsigned long long full = 0, need = 0;
              for (int u = 0; u < 12; ++u) {
                const int32_t* kv = cf + (c_coefsrc[u] & 15) * CW;
                int top = -1;
                for (int k = L - 1; k >= 0; --k)
                  if (top < 0 && kv[k]) top = k;
                for (int i = 0; i < L; ++i) {
                  const int nj = i >= L - 2 ? L : i + 2;
                  full += nj;
                  if (i <= top) need += nj;
                }
                full += L;
                if (kv[L]) need += L;
              }
              const int sw = sweep < 63 ? sweep : 63;
              atomicAdd(&it.phase_cycles[6 + 2 * sw], full);
              atomicAdd(&it.phase_cycles[7 + 2 * sw], need);
            }
            it.alpha[p] = ap;
            it.alpha[q] = aq;
            it.eA[p] = eo[0];
            it.eA[q] = eo[1];
            // No negligible flag from these incremental norms: a column whose norm collapses
            // by cancellation has an incremental alpha with absolute error ~2^-W alpha_old,
            // which could mark a still-significant column negligible for good.  The flag is
            // only set from exact norms (jac_norms at the end of the sweep).
            flag = 1 | (varA << 1) | (varV << 3) | (ints << 8);  // bits 8..31: slot integer digits
            if (it.uprod) {  // digit products phase U will execute per row (kmul_z counts)
              auto P = [](int Z) {
                int c = 0;
                for (int i = 0; i < L - Z; ++i) c += (i >= L - 2) ? L : i + 2;
                return c;
              };
              for (int mat = 0; mat < (accV ? 2 : 1); ++mat) {
                const int v = mat ? varV : varA;
                for (int o = 0; o < 4; ++o)
                  nup += P(u_var_zc<L>(v)) + 2 * P(u_var_zs<L>(v)) + L * __popc((ints >> ((mat * 4 + o) * 3)) & 7);
              }
            }
            if (it.phase_cycles) atomicAdd(&it.phase_cycles[6 + 128 + (sweep < 15 ? sweep : 15) * 4 + varA], 1ull);
            *(volatile int*)it.sync = 1;
            ++nrot;
            if (it.dbg) atomicAdd(&it.dbg[sweep < 63 ? sweep : 63], 1);
          }
        }
        it.rot[i] = flag;
      }
      csync();
      mark(1);
      // ---- phase U: apply the rotations to columns p, q of A and V
      for (int i = gw; i < NP; i += GW) {
        const int flag = it.rot[i];
        if (!(flag & 1)) continue;
        int p, q;
        rr_pair(N, step, i, p, q);
        const int32_t* cfg = it.coef + (size_t)i * 33 * CW + 9 * CW;  // signed slots (phase R)
        for (int w = lane; w < (accV ? 24 : 12) * CW; w += 32) wcoef[w] = cfg[w];
        __syncwarp();
        for (int mat = 0; mat < (accV ? 2 : 1); ++mat) {
          int32_t* F = mat ? it.V : it.A;
          const int rows = mat ? N : M;
          const int nch = mat ? nchV : nchA;
          stage_rows<L>(wbuf, F, rows, p, q, 0, rows, lane);
          cp_commit();
          for (int ch = 0; ch < nch; ++ch) {
            if (JST == 2 && ch + 1 < nch) {
              stage_rows<L>(wbuf + ((ch + 1) & 1) * STAGE, F, rows, p, q, (ch + 1) * 32, rows, lane);
              cp_commit();
              cp_wait<1>();
            } else {
              cp_wait<0>();
            }
            __syncwarp();
            const int32_t* b = wbuf + (JST == 2 ? (ch & 1) * STAGE : 0);
            const int r = ch * 32 + lane;
            const int var = (flag >> (1 + 2 * mat)) & 3;  // zero-digit variant (U_VARIANTS)
            if (var == 0) u_chunk<L, 0, 0>(F, rows, p, q, r, lane, b, wcoef, mat, flag);
            else if (var == 1) u_chunk<L, u_var_zc<L>(1), u_var_zs<L>(1)>(F, rows, p, q, r, lane, b, wcoef, mat, flag);
            else if (var == 2) u_chunk<L, u_var_zc<L>(2), u_var_zs<L>(2)>(F, rows, p, q, r, lane, b, wcoef, mat, flag);
            else u_chunk<L, u_var_zc<L>(3), u_var_zs<L>(3)>(F, rows, p, q, r, lane, b, wcoef, mat, flag);
            __syncwarp();
            if (JST == 1 && ch + 1 < nch) {
              stage_rows<L>(wbuf, F, rows, p, q, (ch + 1) * 32, rows, lane);
              cp_commit();
            }
          }
        }
      }
      csync();
      mark(2);
    }
    // refresh exact column norms (and renormalise columns) for the next sweep / the result
    const bool any = *(volatile int*)it.sync != 0 || lgd < L;
    if (it.gexp) e2prev = *(volatile int*)&it.gexp[sweep & 1];
    if (it.cexp) {
      if (lmu > INT_MIN) atomicMax(&it.cexp[2 * (sweep & 1)], lmu);
      if (lrho > INT_MIN) atomicMax(&it.cexp[2 * (sweep & 1) + 1], lrho);
    }
    // exact norms; the negligible-column rule (R3b) is re-evaluated on them
    jac_norms<L, NL>(it, true, z, gw, GW);
    csync();
    mark(3);
    // Certified stop (R21): a pair evaluated in this sweep ends it with
    // rho <= max(rho at its evaluation if not rotated (<= tol), rotation residual) plus at most
    // 2(N-2) later rotations touching p or q, each adding <= mu * (largest rho of the sweep)
    // (x2 for off-diagonals not yet evaluated, x2 for norm drift).  When that sum is below
    // tol / 256 the rotation-free sweep the stopping rule asks for is not run.
    bool cert = false;
    if (it.cexp && any && lgd == L) {
      const int emu = *(volatile int*)&it.cexp[2 * (sweep & 1)];
      const int erho = *(volatile int*)&it.cexp[2 * (sweep & 1) + 1];
      const int lg2N = 32 - __clz(2 * N - 1);                 // ceil(log2 2N)
      const int64_t etol2 = 2 * (int64_t)(31 - __clz(M)) + 4 - 2 * (int64_t)W;  // <= log2 tol^2
      cert = emu > INT_MIN && erho > INT_MIN && emu <= -2 * (lg2N + 3) &&
             2 * (int64_t)lg2N + emu + erho + 6 <= etol2 - 16;
    }
    if (jac_trace_items && crank == 0 && tid == 0 && (int)(C > 1 ? blockIdx.x / C : blockIdx.x) < jac_trace_items)
      printf("jacobi item %d N %d sweep %d lgd %d erho2 %d emu2 %d any %d cert %d\n", (int)(C > 1 ? blockIdx.x / C : blockIdx.x),
             N, sweep, lgd, it.cexp ? *(volatile int*)&it.cexp[2 * (sweep & 1) + 1] : 0,
             it.cexp ? *(volatile int*)&it.cexp[2 * (sweep & 1)] : 0, (int)any, (int)cert);
    if (!any || cert) {
      conv = 1;
      if (cert && crank == 0 && tid == 0) it.cexp[4] = 1;
      break;
    }
  }
  atomicAdd((unsigned long long*)it.rotations, (unsigned long long)nrot);
  atomicAdd((unsigned long long*)it.evals, (unsigned long long)nev);
  if (it.uprod) atomicAdd((unsigned long long*)it.uprod, (unsigned long long)nup);
  if (prof) {
    pc[5] = (unsigned long long)(clock64() - t_start);
    for (int i = 0; i < 6; ++i) atomicAdd(&it.phase_cycles[i], pc[i]);
  }
  if (crank == 0 && tid == 0) {
    *it.sweeps = conv ? sweep : MAX_SWEEPS + 1;
    *it.status = conv ? 0 : -3;
  }
}

template <int L>
constexpr size_t jacobi_smem_bytes() { return (size_t)NWARP * (jacobi_stages<L>() * 4 * L * 32 + 24 * (L + 1)) * 4; }

// Launch n items with C CTAs each (a cluster of C when C > 1).
template <int L, int NL>
inline void launch_jacobi(const SvdItem<NL>* d_items, int n, int C, cudaStream_t st);

// opt in to > 48 KB of dynamic shared memory (once per instantiation)
inline void jacobi_trace_init() {
  static int tr = -1;
  if (tr < 0) {
    const char* e = getenv("MPS_JACOBI_TRACE");
    tr = e ? atoi(e) : 0;
    if (tr > 0) cudaMemcpyToSymbol(jac_trace_items, &tr, sizeof(int));
  }
}
template <int L, int NL>
inline void jacobi_prepare() {
  smem_optin((const void*)k_jacobi<L, NL>, (int)jacobi_smem_bytes<L>());
  jacobi_trace_init();
}

template <int L, int NL>
inline void launch_jacobi(const SvdItem<NL>* d_items, int n, int C, cudaStream_t st) {
  jacobi_prepare<L, NL>();
  if (C <= 1) {
    k_jacobi<L, NL><<<n, NTHR, jacobi_smem_bytes<L>(), st>>>(d_items, 1);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n * C, 1, 1);
  cfg.blockDim = dim3(NTHR, 1, 1);
  cfg.dynamicSmemBytes = jacobi_smem_bytes<L>();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_jacobi<L, NL>, d_items, C);
}

// CTAs per matrix: fill ~2 CTAs per SM when few matrices are in flight, at least one pair
// per warp, power of two, at most 8 (portable cluster size).
// MPS_JACOBI_MAX_CLUSTER (env, default 8) caps C; tests use it to compare C = 1 and C > 1.
// Many matrices (more than one wave of `slots` resident CTAs): one CTA per matrix leaves the
// last wave partly empty (1024 items at chi = 128: 3.46 waves of 296 -> 4); C = 2 halves the
// quantum at a measured per-matrix overhead of ~4.5% (cluster barriers; C = 4: 18%), so C is
// chosen by waves(C) * overhead(C) / C (measured at N = 256, 280 bits: C = 2 gives 113.6 vs
// 108.3 updates/s; profiles/r01_cluster_ab_v24.jsonl).
inline int jacobi_cluster_size(int n_items, int min_N, int slots = 2 * 148) {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("MPS_JACOBI_MAX_CLUSTER");
    cap = e ? atoi(e) : 8;
    if (cap < 1) cap = 1;
    if (cap > 8) cap = 8;
  }
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("MPS_JACOBI_CLUSTER");  // A/B: force C (power of two <= 8)
    force = e ? atoi(e) : 0;
  }
  int C = 1;
  if (force > 1) {
    while (C < force && C < 8 && (C * 2) * NWARP <= min_N / 2) C *= 2;
    return C;
  }
  while (C < cap && n_items * C * 2 <= 2 * 148 && (C * 2) * NWARP <= min_N / 2) C *= 2;
  if (C == 1 && n_items > slots && min_N >= 256 && cap >= 2) {
    const double over[3] = {1.0, 1.045, 1.18};
    double best = 1e300;
    for (int c = 1, i = 0; c <= 4 && c <= cap && c * NWARP <= min_N / 2; c *= 2, ++i) {
      const double cost = (double)((n_items * c + slots - 1) / slots) * over[i] / c;
      if (cost < best - 1e-9) { best = cost; C = c; }
    }
  }
  return C;
}

// per-item counters -> running totals (profiling): [0] rotations, [1] pair evaluations,
// [2] sum over items of sweeps * M * N (norm passes), [3] sum of N*N*M (recovery GEMMs),
// [4] phase-U digit products x M, [5] items that ended on the certified stop (R21)
template <int NL>
__global__ void k_accum_stats(const SvdItem<NL>* items, int n, unsigned long long* tot) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    const SvdItem<NL>& it = items[b];
    atomicAdd(&tot[0], (unsigned long long)*it.rotations);
    atomicAdd(&tot[1], (unsigned long long)*it.evals);
    atomicAdd(&tot[2], (unsigned long long)(*it.sweeps + 1) * it.M * it.N);
    if (it.A0) atomicAdd(&tot[3], (unsigned long long)it.N * it.N * it.M);
    if (it.uprod) atomicAdd(&tot[4], (unsigned long long)*it.uprod * it.M);
    if (it.cexp) atomicAdd(&tot[5], (unsigned long long)it.cexp[4]);
  }
}

// ----------------------------------------------------------------------------
// a3' recovery of the right factor: V(c,b) = sum_r conj(A0(r,c)) A(r,b) / alpha_b
// (A = A0 V with A's columns a_b = sigma_b x_b, so V = A0^H A diag(1/sigma^2)).  A0 has one
// block exponent, A per-column exponents; column b of V gets its own exponent
// eV[b] = e0 + e_b + g + e(1/alpha_b) and the digits are scaled by the mantissa of 1/alpha_b.
template <int L, int NL>
__global__ void k_recover_v(const SvdItem<NL>* items) {
  const SvdItem<NL> it = items[blockIdx.y];
  if (!it.A0) return;
  const int M = it.M, N = it.N, W = 28 * L;
  int g = 1;
  while ((1 << (g - 1)) < M) ++g;
  g += 1;  // sum of M complex products, each |.| < 2^(e0 + e_b + 1)
  const int64_t e0 = *it.eA0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N * N; t += gridDim.x * blockDim.x) {
    const int c = t % N, b = t / N;
    const mpf<NL> al = it.alpha[b];
    int32_t o[L];
    if (mpf_is_zero(al)) {
#pragma unroll
      for (int k = 0; k < L; ++k) o[k] = 0;
      stfx<L>(it.V, N, b, 0, c, o);
      stfx<L>(it.V, N, b, 1, c, o);
      if (c == 0) it.eV[b] = 1;
      continue;
    }
    int64_t ar[L + 2], ai[L + 2];
#pragma unroll
    for (int j = 0; j < L + 2; ++j) ar[j] = ai[j] = 0;
    int cnt = 0;
    for (int r = 0; r < M; ++r) {
      int32_t xr[L], xi[L], yr[L], yi[L];
      ldfx<L>(it.A0, M, c, 0, r, xr);
      ldfx<L>(it.A0, M, c, 1, r, xi);
      ldfx<L>(it.A, M, b, 0, r, yr);
      ldfx<L>(it.A, M, b, 1, r, yi);
      tmul_acc2<L>(ar, xr, yr);  // conj(x) y: re = xr yr + xi yi, im = xr yi - xi yr
      tmul_acc2<L>(ar, xi, yi);
      tmul_acc2<L>(ai, xr, yi);
      tmul_sub2<L>(ai, xi, yr);
      if (++cnt == 8) { cnt = 0; tnorm2<L>(ar); tnorm2<L>(ai); }
    }
    // 1/alpha_b = m 2^ei, m in [0.5, 1): digits x m as a fractional coefficient
    const mpf<NL> inv = mpf_recip(al);
    const int64_t ei = inv.e;
    int32_t kd[L + 1];
    mpf_to_coef<NL, L>(mpf_ldexp(inv, -ei), kd);
    const int64_t eOut = e0 + it.eA[b] + g + ei;
    for (int ri = 0; ri < 2; ++ri) {
      int32_t d[L];
      tround_sr<L>(ri ? ai : ar, g, d);
      int64_t acc[L + 2];
#pragma unroll
      for (int j = 0; j < L + 2; ++j) acc[j] = 0;
      kmul_acc<L>(acc, kd, d, kd[L] != 0);
      tround2<L>(acc, o);
      stfx<L>(it.V, N, b, ri, c, o);
    }
    if (c == 0) it.eV[b] = eOut;
  }
}

// ----------------------------------------------------------------------------
// a4 order / truncate / renormalise (one CTA per item)
// ----------------------------------------------------------------------------
template <int L, int NL>
__global__ void __launch_bounds__(NTHR) k_finalize(const FinItem<NL>* items, int RBr, int p) {
  const FinItem<NL> it = items[blockIdx.x];
  const int N = it.N, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ unsigned char fsm[];
  mpf<NL>* sig = (mpf<NL>*)fsm;  // [N]
  __shared__ int s_cnt, s_k;
  __shared__ mpf<NL> s_sum[NWARP], s_all, s_kept, s_nu;
  for (int j = tid; j < N; j += NTHR) sig[j] = mpf_sqrt(it.alpha[j]);
  __syncthreads();
  // stable descending rank
  for (int j = tid; j < N; j += NTHR) {
    int rank = 0;
    for (int i = 0; i < N; ++i) {
      int c = mpf_cmp(sig[i], sig[j]);
      if (c > 0 || (c == 0 && i < j)) ++rank;
    }
    it.ord[rank] = j;
  }
  __syncthreads();
  // sum of all sigma^2 (= alpha)
  mpf<NL> s = mpf_zero<NL>();
  for (int j = tid; j < N; j += NTHR) s = mpf_add(s, it.alpha[j]);
  for (int l = 0; l < 32; ++l) {  // warp serial reduction
    mpf<NL> o;
    o.e = __shfl_sync(0xffffffffu, s.e, l);
    o.neg = __shfl_sync(0xffffffffu, s.neg, l);
#pragma unroll
    for (int k = 0; k < NL; ++k) o.m[k] = __shfl_sync(0xffffffffu, s.m[k], l);
    if (lane == 0 && l > 0) s = mpf_add(s, o);
  }
  if (lane == 0) s_sum[warp] = s;
  __syncthreads();
  if (tid == 0) {
    mpf<NL> a = s_sum[0];
    for (int w = 1; w < NWARP; ++w) a = mpf_add(a, s_sum[w]);
    s_all = a;
    const mpf<NL> cut = mpf_mul(it.thr, mpf_sqrt(a));
    int cnt = 0;
    while (cnt < N && !mpf_is_zero(sig[it.ord[cnt]]) && mpf_cmp(sig[it.ord[cnt]], cut) >= 0) ++cnt;
    int k = cnt < it.chi_max ? cnt : it.chi_max;
    s_k = k;
    mpf<NL> kept = mpf_zero<NL>();
    for (int b = 0; b < k; ++b) kept = mpf_add(kept, it.alpha[it.ord[b]]);
    s_kept = kept;
    s_nu = mpf_sqrt(kept);
    *it.k_out = k;
    if (it.redo && it.eV && k > 0) {
      const mpf<NL>& smax = sig[it.ord[0]];
      const mpf<NL>& smin = sig[it.ord[k - 1]];
      if (!mpf_is_zero(smin) && smax.e - smin.e > it.redo_bits) atomicOr(it.redo, 1);  // 1: accumulate V
    }
    const int js = it.svd_status ? *it.svd_status : 0;
    *it.status = js ? js : (k == 0 ? -4 : 0);
  }
  __syncthreads();
  const int k = s_k;
  const mpf<NL> inv_nu = k ? mpf_recip(s_nu) : mpf_zero<NL>();
  for (int b = tid; b < N; b += NTHR) {
    const int j = it.ord[b];
    if (it.sigma_rec && b < it.nsig) mpf_to_record<NL>(sig[j], it.sigma_rec + (size_t)b * RBr, RBr - 4, p);
    if (b < k) {
      mpf<NL> lam = mpf_mul(sig[j], inv_nu);
      it.lam[b] = lam;
      it.inv_sig[b] = mpf_recip(sig[j]);
      if (it.lam_rec) mpf_to_record<NL>(lam, it.lam_rec + (size_t)b * RBr, RBr - 4, p);
    }
  }
}

// a5 split outputs: Gamma_L[i][a][b] = Ul[(i,a),b] / lamL(a), Gamma_R[j][b][c] = conj(Wr[(j,c),b]) / lamR(c)
// Ul = X (= A col / sigma) or V (trans); Wr = V or X (trans). grid.x blocks over entries, grid.y items.
template <int L, int NL>
__global__ void k_split(const FinItem<NL>* items, int RBr, int p) {
  const FinItem<NL> it = items[blockIdx.y];
  const int k = *it.k_out;
  if (k <= 0) return;
  const int W = 28 * L;
  const int nL = it.GL ? 2 * it.chiL_out * k : 0;
  const int nR = it.GR ? 2 * it.chiR_out * k : 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nL + nR; t += gridDim.x * blockDim.x) {
    const bool left = t < nL;
    const int u = left ? t : t - nL;
    const int b = u % k, row = u / k;  // row = (i,a) or (j,c) index into the factor rows
    const int j = it.ord[b];
    // which stored matrix: X (A with exponent eA, scaled by 1/sigma) or V (exponent 1)
    const bool fromA = left ? !it.trans : it.trans;
    const int32_t* F = fromA ? it.A : it.V;
    const int ld = fromA ? it.M : it.N;
    const int64_t E = fromA ? it.eA[j] : (it.eV ? it.eV[j] : 1);
    mpf<NL> scale = fromA ? it.inv_sig[b] : mpf_from_int<NL>(1);
    const int chi = left ? it.chiL_out : it.chiR_out;
    const uint32_t* lam = left ? it.lamL : it.lamR;
    const int a = row % chi;
    if (lam) scale = mpf_mul(scale, mpf_recip(mpf_from_record<NL>(lam + (size_t)a * RBr, RBr - 4)));
    for (int ri = 0; ri < 2; ++ri) {
      int32_t x[L];
      ldfx<L>(F, ld, j, ri, row, x);
      int64_t cc[L];
      fx_to_cols<L>(x, cc);
      mpf<NL> v = mpf_mul(mpf_from_cols<NL, L>(cc, E - (int64_t)W), scale);
      // trans: the left factor V (resp. right factor X) of Theta'^H relates by
      // Theta' = V S X^H, so no extra conjugation is needed beyond Gamma_R's conj.
      if (!left && ri == 1) v = mpf_neg(v);  // conj for Gamma_R
      uint32_t* out;
      if (left) {
        const int i = row / it.chiL_out;
        out = it.GL + ((size_t)(i * it.chiL_out + a) * it.GL_ld + b) * 2 * RBr;
      } else {
        const int jj = row / it.chiR_out;
        out = it.GR + ((size_t)(jj * it.GR_ld + b) * it.chiR_out + a) * 2 * RBr;
      }
      mpf_to_record<NL>(v, out + ri * RBr, RBr - 4, p);
    }
  }
}

// three-site: M2[(i,a),(j,b)] = Ul[(2i+j) chiL2 + a, b] * w_b with w_b = lambda'_b/sigma_b
// (Ul = X = A/sigma) or lambda'_b (Ul = V); written in Jacobi layout (trans -> M2^H).
// Output exponent per column: E_b = E_src(b) + e(w_b); transposed, all columns share
// E_max = max_b E_b (set by k_finalize in *eM2max) and entries are scaled by
// kappa = w_b 2^(E_src - E_out) <= 1 (one truncated product per real).
template <int NL>
__device__ __forceinline__ void m2_weight(const FinItem<NL>& it, int b, mpf<NL>& w, int64_t& Es) {
  const bool fromA = !it.trans;
  const int j = it.ord[b];
  w = fromA ? mpf_mul(it.lam[b], it.inv_sig[b]) : it.lam[b];
  Es = fromA ? it.eA[j] : (it.eV ? it.eV[j] : 1);
}

template <int L, int NL>
__global__ void k_m2_exp(const FinItem<NL>* items, int64_t* eM2max) {
  const FinItem<NL> it = items[blockIdx.x];
  const int k = *it.k_out;
  __shared__ long long s_max;
  if (threadIdx.x == 0) s_max = INT64_MIN;
  __syncthreads();
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    mpf<NL> w; int64_t Es;
    m2_weight<NL>(it, b, w, Es);
    atomicMax(&s_max, (long long)(Es + w.e));
  }
  __syncthreads();
  if (threadIdx.x == 0) eM2max[blockIdx.x] = s_max;
}

template <int L, int NL>
__global__ void k_build_m2(const FinItem<NL>* items, const int64_t* eM2max) {
  const FinItem<NL> it = items[blockIdx.y];
  const int k = *it.k_out;
  if (k <= 0) return;
  const int chiL = it.chiL2;
  const int rows = 2 * chiL, cols = 2 * k;  // M2 geometry
  const int n = rows * cols;
  const bool fromA = !it.trans;
  const int trans = it.M2_trans;
  const int Mrows = trans ? cols : rows;  // Jacobi matrix rows
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % rows, c = t / rows;
    const int i = r / chiL, a = r % chiL, jj = c / k, b = c % k;
    const int j = it.ord[b];
    const int srow = (2 * i + jj) * chiL + a;
    const int32_t* F = fromA ? it.A : it.V;
    const int ld = fromA ? it.M : it.N;
    mpf<NL> w; int64_t Es;
    m2_weight<NL>(it, b, w, Es);
    const int64_t Eout = trans ? eM2max[blockIdx.y] : Es + w.e;
    int32_t wd[L];
    mpf_to_fixed<NL, L>(mpf_ldexp(w, Es - Eout), 0, wd);
    for (int ri = 0; ri < 2; ++ri) {
      int32_t x[L], o[L];
      ldfx<L>(F, ld, j, ri, srow, x);
      int64_t acc[L + 1];
#pragma unroll
      for (int q = 0; q <= L; ++q) acc[q] = 0;
      tmul_acc<L>(acc, wd, x);
      tround<L>(acc, 0, o);
      if (!trans) {
        stfx<L>(it.M2, Mrows, c, ri, r, o);
      } else {  // M2^H: row c, column r, conjugated
        if (ri == 1) {
#pragma unroll
          for (int q = 0; q < L; ++q) o[q] = -o[q];
        }
        stfx<L>(it.M2, Mrows, r, ri, c, o);
      }
    }
    if (it.M2_A0) {  // the same entries at the block exponent eM2max (input kept for V recovery)
      const int64_t E0 = eM2max[blockIdx.y];
      int32_t wd0[L];
      mpf_to_fixed<NL, L>(mpf_ldexp(w, Es - E0), 0, wd0);
      for (int ri = 0; ri < 2; ++ri) {
        int32_t x[L], o[L];
        ldfx<L>(F, ld, j, ri, srow, x);
        int64_t acc[L + 1];
#pragma unroll
        for (int q = 0; q <= L; ++q) acc[q] = 0;
        tmul_acc<L>(acc, wd0, x);
        tround<L>(acc, 0, o);
        if (!trans) {
          stfx<L>(it.M2_A0, Mrows, c, ri, r, o);
        } else {
          if (ri == 1) {
#pragma unroll
            for (int q = 0; q < L; ++q) o[q] = -o[q];
          }
          stfx<L>(it.M2_A0, Mrows, r, ri, c, o);
        }
      }
      if (t == 0) *it.M2_eA0 = E0;
    }
    if (!trans) { if (r == 0) it.eM2[c] = Eout; }
    else { if (c == 0) it.eM2[r] = Eout; }
  }
}

}  // namespace mpsb
