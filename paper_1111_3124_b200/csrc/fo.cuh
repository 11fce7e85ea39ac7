// First-order finish of the p-bit Jacobi (R23).
//
// After the refinement sweeps (R22) the columns of A_1 = Theta' X are orthogonal to
// rho ~ 2^-155, so every rotation of the next p-bit sweep has |s| ~ rho alpha / gap and c = 1 to
// the working precision (1 - |s|^2/2 with |s|^2 < 2^-290), and the products of two rotations
// (|s|^2) are below the 280-bit rounding.  The whole sweep is then the linear map
//   A_2 = A_1 (I + E),  E_pq = s_pq,  E_qp = -conj(s_pq)  (p < q),  s_pq = gamma_pq / (alpha_q - alpha_p)
// (the rotation of DESIGN.md R17 to first order in s; gamma, alpha from the Gram matrix
// G_1 = A_1^H A_1), one GEMM on the tensor cores instead of N(N-1)/2 column rotations.
// Convergence is then decided by the paper's criterion on the stored result: the Gram matrix
// G_2 = A_2^H A_2 must have |G_pq| <= tol_fo sqrt(G_pp G_qq) for every pair of non-negligible
// columns (the rotation-free sweep, evaluated as one GEMM), tol_fo = 16 tol (tol = 4 M 2^-W, R3):
// A_2 is rounded at its block exponent (k_jacobi rounds every rotated column at its own), which
// leaves off-diagonals up to ~2^-268 (measured max rho^2 = 2^-537 at chi = 128 against
// tol^2 = 2^-540); rho <= 2^-266 keeps sigma to rho^2 and the kept factors to rho / gap, far
// inside the parity tolerance (1e-70 ~ 2^-232).  Items for which E does not apply
// (some |s| >= 2^-145, a zero gap, graded spectra) or that fail the check run k_jacobi as before.
// Both Gram matrices carry L + 1 digits (an (L+1)-digit product of the zero-padded operands):
// the test needs |G_pq| to ~2^-300 of alpha, below the L-digit rounding of an L-digit GEMM.
#pragma once
#include <cstdint>

#include "precond.cuh"

namespace mpsb {

template <int NL>
struct FoItem {
  int M, N;                // N = 0: the item does not take the first-order finish
  const int32_t* G;        // N x N, L + 1 digits (upper triangle and diagonal), block exponent *eG
  const int64_t* eG;
  int32_t* E;              // N x N fixed, L digits, exponent 1 (out of k_fo_coef)
  int* ok;                 // [1] 1: E was formed; 0: E = 0, the item runs k_jacobi
  int* done;               // [1] 1: the check passed, k_jacobi skips the item
  mpf<NL>* alpha;          // out (SvdItem): squared column norms of A_2
  int* negl;               // out: negligible columns (R3b)
  int* status; int* sweeps; long long* rots; long long* evals; long long* uprod; int* cexp;
};

template <int L, int NL>
__device__ __forceinline__ mpf<NL> fo_entry(const int32_t* G, int N, int r, int c, int ri, int64_t eG) {
  int64_t col[L + 1];
  const int32_t* p = G + ((size_t)(c * 2 + ri) * (L + 1)) * N + r;
#pragma unroll
  for (int k = 0; k <= L; ++k) col[k] = p[(size_t)k * N];
  return mpf_from_cols<NL, L + 1>(col, eG - 28 * (int64_t)(L + 1));
}

// alpha_p = G_pp, the negligible-column floor z = tol^2 sum alpha (as k_jacobi), the flags
template <int L, int NL>
__device__ void fo_alpha(const FoItem<NL>& it, mpf<NL>* s_alpha, int* s_negl, mpf<NL>& s_z) {
  const int N = it.N, M = it.M;
  const int64_t eG = *it.eG;
  for (int p = threadIdx.x; p < N; p += blockDim.x) s_alpha[p] = fo_entry<L, NL>(it.G, N, p, p, 0, eG);
  __syncthreads();
  if (threadIdx.x == 0) {
    mpf<NL> s = mpf_zero<NL>();
    for (int p = 0; p < N; ++p) s = mpf_add(s, s_alpha[p]);
    const mpf<NL> tol2 = mpf_ldexp(mpf_from_int<NL>((int64_t)M * M), 4 - 2 * (int64_t)(28 * L));
    s_z = mpf_mul(tol2, s);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < N; p += blockDim.x)
    s_negl[p] = (mpf_is_zero(s_alpha[p]) || s_alpha[p].neg || mpf_cmp(s_alpha[p], s_z) <= 0) ? 1 : 0;
  __syncthreads();
}

// pair index t < N(N-1)/2 -> (p, q), p < q (row-major over the upper triangle)
__device__ __forceinline__ void fo_pair(int N, int t, int& p, int& q) {
  // p = largest with p (2N - p - 1) / 2 <= t
  int pp = (int)((2.0 * N - 1 - sqrt((2.0 * N - 1) * (2.0 * N - 1) - 8.0 * t)) / 2);
  while (pp > 0 && pp * (2 * N - pp - 1) / 2 > t) --pp;
  while ((pp + 1) * (2 * N - pp - 2) / 2 <= t) ++pp;
  p = pp;
  q = t - pp * (2 * N - pp - 1) / 2 + pp + 1;
}

// E from G_1 (one CTA per item).  Shared memory: alpha [N] mpf, negl [N] int.
template <int L, int NL>
__global__ void __launch_bounds__(256) k_fo_coef(const FoItem<NL>* items) {
  const FoItem<NL> it = items[blockIdx.x];
  const int N = it.N, M = it.M;
  if (N == 0) return;
  extern __shared__ int4 fo_sm[];
  mpf<NL>* s_alpha = (mpf<NL>*)fo_sm;
  int* s_negl = (int*)(s_alpha + N);
  __shared__ mpf<NL> s_z;
  __shared__ int s_ok, s_nrot;
  // E = 0
  const size_t nw = (size_t)N * N * 2 * L;
  for (size_t w = threadIdx.x; w < nw; w += blockDim.x) it.E[w] = 0;
  if (threadIdx.x == 0) { s_ok = 1; s_nrot = 0; }
  fo_alpha<L, NL>(it, s_alpha, s_negl, s_z);
  const int64_t eG = *it.eG;
  const mpf<NL> tol2 = mpf_ldexp(mpf_from_int<NL>((int64_t)M * M), 4 - 2 * (int64_t)(28 * L));
  const int npairs = N * (N - 1) / 2;
  int nrot = 0;
  for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
    int p, q;
    fo_pair(N, t, p, q);
    if (s_negl[p] || s_negl[q]) continue;  // never rotated (R3b)
    const mpf<NL> gr = fo_entry<L, NL>(it.G, N, p, q, 0, eG), gi = fo_entry<L, NL>(it.G, N, p, q, 1, eG);
    const mpf<NL> g2 = mpf_add(mpf_mul(gr, gr), mpf_mul(gi, gi));
    const mpf<NL> ap = s_alpha[p], aq = s_alpha[q];
    if (mpf_is_zero(g2) || mpf_cmp(g2, mpf_mul(tol2, mpf_mul(ap, aq))) <= 0) continue;  // not rotated
    const mpf<NL> d = mpf_sub(aq, ap);
    if (mpf_is_zero(d)) { s_ok = 0; continue; }
    const mpf<NL> id = mpf_recip(d);
    const mpf<NL> sr = mpf_mul(gr, id), si = mpf_mul(gi, id);
    // |s| < 2^-145: s^2 below the working precision (and E's top 5 digits are zero)
    if ((!mpf_is_zero(sr) && sr.e > -145) || (!mpf_is_zero(si) && si.e > -145)) { s_ok = 0; continue; }
    ++nrot;
    int32_t d1[L], d2[L];
    // E_pq = s (column q, row p); E_qp = -conj(s) = -sr + i si (column p, row q)
    mpf_to_fixed<NL, L>(sr, 1, d1);
    mpf_to_fixed<NL, L>(si, 1, d2);
    stfx<L>(it.E, N, q, 0, p, d1);
    stfx<L>(it.E, N, q, 1, p, d2);
#pragma unroll
    for (int k = 0; k < L; ++k) d1[k] = -d1[k];
    stfx<L>(it.E, N, p, 0, q, d1);
    stfx<L>(it.E, N, p, 1, q, d2);
  }
  atomicAdd(&s_nrot, nrot);
  __syncthreads();
  if (!s_ok) {  // fall back: E = 0 (A_2 = A_1 exactly), k_jacobi runs the item
    for (size_t w = threadIdx.x; w < nw; w += blockDim.x) it.E[w] = 0;
  }
  if (jac_trace_items && threadIdx.x == 0 && (int)blockIdx.x < jac_trace_items && !s_ok)
    printf("first-order finish item %d N %d: not applicable (some |s| >= 2^-145 or a zero gap)\n", (int)blockIdx.x, N);
  if (threadIdx.x == 0) {
    *it.ok = s_ok;
    *it.done = 0;
    *it.rots = s_ok ? s_nrot : 0;
  }
}

// The stopping criterion on G_2 = A_2^H A_2 (one CTA per item): every pair of non-negligible
// columns has |G_pq|^2 <= tol^2 G_pp G_qq.  On success the item is done: alpha, negl, the
// counters and the status are written as k_jacobi would (one sweep).
template <int L, int NL>
__global__ void __launch_bounds__(256) k_fo_check(const FoItem<NL>* items) {
  const FoItem<NL> it = items[blockIdx.x];
  const int N = it.N, M = it.M;
  if (N == 0 || !*it.ok) return;
  extern __shared__ int4 fo_sm[];
  mpf<NL>* s_alpha = (mpf<NL>*)fo_sm;
  int* s_negl = (int*)(s_alpha + N);
  __shared__ mpf<NL> s_z;
  __shared__ int s_pass;
  if (threadIdx.x == 0) s_pass = 1;
  fo_alpha<L, NL>(it, s_alpha, s_negl, s_z);
  const int64_t eG = *it.eG;
  // tol_fo^2 = 2^8 tol^2
  const mpf<NL> tol2 = mpf_ldexp(mpf_from_int<NL>((int64_t)M * M), 4 + 8 - 2 * (int64_t)(28 * L));
  const int npairs = N * (N - 1) / 2;
  __shared__ int s_emax;
  if (threadIdx.x == 0) s_emax = INT_MIN;
  __syncthreads();
  int emax = INT_MIN;
  for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
    int p, q;
    fo_pair(N, t, p, q);
    if (s_negl[p] || s_negl[q]) continue;
    const mpf<NL> gr = fo_entry<L, NL>(it.G, N, p, q, 0, eG), gi = fo_entry<L, NL>(it.G, N, p, q, 1, eG);
    const mpf<NL> g2 = mpf_add(mpf_mul(gr, gr), mpf_mul(gi, gi));
    if (mpf_is_zero(g2)) continue;
    const mpf<NL> den = mpf_mul(s_alpha[p], s_alpha[q]);
    emax = max(emax, (int)(g2.e - den.e));  // log2(rho^2) within 1
    if (mpf_cmp(g2, mpf_mul(tol2, den)) > 0) s_pass = 0;
  }
  atomicMax(&s_emax, emax);
  __syncthreads();
  if (jac_trace_items && threadIdx.x == 0 && (int)blockIdx.x < jac_trace_items)
    printf("first-order finish item %d N %d rotated %lld pairs, max log2 rho^2 ~ %d, check %s\n", (int)blockIdx.x, N,
           *it.rots, s_emax, s_pass ? "passed" : "failed");
  if (!s_pass) return;  // k_jacobi continues from A_2
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    it.alpha[p] = s_alpha[p];
    it.negl[p] = s_negl[p];
  }
  if (threadIdx.x == 0) {
    *it.done = 1;
    *it.status = 0;
    *it.sweeps = 1;
    *it.evals = npairs;
    if (it.uprod) *it.uprod = 0;
    if (it.cexp) it.cexp[4] = 0;
  }
}

template <int NL>
inline size_t fo_smem(int N) { return (size_t)N * sizeof(mpf<NL>) + (size_t)N * 4 + 16; }

}  // namespace mpsb
