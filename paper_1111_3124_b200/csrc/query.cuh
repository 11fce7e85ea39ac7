// Kernels on the MPS store outside the two/three-site update: one-site gates (a7),
// amplitudes (Eq. 1 contraction), transfer-matrix norm / expectation, and the
// unitarity check of gate matrices.  All arithmetic in the scalar mpf format.
#pragma once
#include "common.h"
#include "kernels.cuh"

namespace mpsb {

template <int NL>
struct cmpf {
  mpf<NL> re, im;
};

template <int NL>
__device__ __forceinline__ cmpf<NL> cm_zero() { return {mpf_zero<NL>(), mpf_zero<NL>()}; }
template <int NL>
__device__ __forceinline__ cmpf<NL> cm_mul(const cmpf<NL>& a, const cmpf<NL>& b) {
  return {mpf_sub(mpf_mul(a.re, b.re), mpf_mul(a.im, b.im)), mpf_add(mpf_mul(a.re, b.im), mpf_mul(a.im, b.re))};
}
template <int NL>
__device__ __forceinline__ cmpf<NL> cm_conjmul(const cmpf<NL>& a, const cmpf<NL>& b) {  // conj(a) b
  return {mpf_add(mpf_mul(a.re, b.re), mpf_mul(a.im, b.im)), mpf_sub(mpf_mul(a.re, b.im), mpf_mul(a.im, b.re))};
}
template <int NL>
__device__ __forceinline__ cmpf<NL> cm_add(const cmpf<NL>& a, const cmpf<NL>& b) {
  return {mpf_add(a.re, b.re), mpf_add(a.im, b.im)};
}
template <int NL>
__device__ __forceinline__ cmpf<NL> cm_scale(const mpf<NL>& s, const cmpf<NL>& a) {
  return {mpf_mul(s, a.re), mpf_mul(s, a.im)};
}
template <int NL>
__device__ __forceinline__ cmpf<NL> cm_from_rec(const uint32_t* rec, int RBr) {
  return {mpf_from_record<NL>(rec, RBr - 4), mpf_from_record<NL>(rec + RBr, RBr - 4)};
}
template <int NL>
__device__ __forceinline__ void cm_to_rec(const cmpf<NL>& a, uint32_t* rec, int RBr, int p) {
  mpf_to_record<NL>(a.re, rec, RBr - 4, p);
  mpf_to_record<NL>(a.im, rec + RBr, RBr - 4, p);
}

// a7: G'[i][a][b] = sum_j U[i][j] G[j][a][b]
template <int NL>
__global__ void k_onesite(const uint32_t* G, uint32_t* Gout, const uint32_t* U, int nab, int RBr, int p) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nab; t += gridDim.x * blockDim.x) {
    const cmpf<NL> g0 = cm_from_rec<NL>(G + (size_t)(2 * t) * RBr, RBr);
    const cmpf<NL> g1 = cm_from_rec<NL>(G + (size_t)(2 * (nab + t)) * RBr, RBr);
    for (int i = 0; i < 2; ++i) {
      const cmpf<NL> u0 = cm_from_rec<NL>(U + (size_t)(2 * (2 * i + 0)) * RBr, RBr);
      const cmpf<NL> u1 = cm_from_rec<NL>(U + (size_t)(2 * (2 * i + 1)) * RBr, RBr);
      cm_to_rec<NL>(cm_add(cm_mul(u0, g0), cm_mul(u1, g1)), Gout + (size_t)(2 * (i * nab + t)) * RBr, RBr, p);
    }
  }
}

// Amplitudes c(b) = G_0^{b0} lam_0 G_1^{b1} ... (Eq. 1), one CTA per basis state (grid-stride),
// vector ping-pong in global scratch (2 * maxchi cmpf per CTA).  Block form (site-sharded
// state): the chain starts from v_in (dims[0] complex records, null = [1]) and lam[s] is the
// Schmidt vector left of local site s (lam[0] = the external left bond or null); the output
// per state is the dims[n]-vector (the amplitude itself for a whole chain).
template <int NL>
__global__ void k_amplitudes(const uint32_t* const* G, const uint32_t* const* lam, const int* dims, int n,
                             const uint8_t* bits, long long nstates, int maxchi, cmpf<NL>* scratch,
                             const uint32_t* v_in, uint32_t* out, int RBr, int p) {
  for (long long st = blockIdx.x; st < nstates; st += gridDim.x) {
    cmpf<NL>* v0 = scratch + (size_t)blockIdx.x * 2 * maxchi;
    cmpf<NL>* v1 = v0 + maxchi;
    const uint8_t* b = bits + st * n;
    for (int a = threadIdx.x; a < dims[0]; a += blockDim.x)
      v0[a] = v_in ? cm_from_rec<NL>(v_in + (size_t)(2 * a) * RBr, RBr)
                   : cmpf<NL>{mpf_from_int<NL>(1), mpf_zero<NL>()};
    __syncthreads();
    for (int s = 0; s < n; ++s) {
      const int dl = dims[s], drs = dims[s + 1];
      const uint32_t* g = G[s] + (size_t)(2 * b[s] * dl * drs) * RBr;
      for (int c = threadIdx.x; c < drs; c += blockDim.x) {
        cmpf<NL> acc = cm_zero<NL>();
        for (int a = 0; a < dl; ++a) {
          const cmpf<NL> w = lam[s] ? cm_scale(mpf_from_record<NL>(lam[s] + (size_t)a * RBr, RBr - 4), v0[a]) : v0[a];
          acc = cm_add(acc, cm_mul(w, cm_from_rec<NL>(g + (size_t)(2 * (a * drs + c)) * RBr, RBr)));
        }
        v1[c] = acc;
      }
      __syncthreads();
      cmpf<NL>* t = v0; v0 = v1; v1 = t;
    }
    for (int c = threadIdx.x; c < dims[n]; c += blockDim.x)
      cm_to_rec<NL>(v0[c], out + (size_t)(2 * (st * dims[n] + c)) * RBr, RBr, p);
    __syncthreads();
  }
}

// T[i][b][c] = lam(b) G^i(b, c)   (lam null = 1), cmpf row-major
template <int NL>
__global__ void k_tmat(const uint32_t* G, const uint32_t* lam, int dl, int dr, cmpf<NL>* T, int RBr) {
  const int n = 2 * dl * dr;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int b = (t / dr) % dl;
    cmpf<NL> g = cm_from_rec<NL>(G + (size_t)(2 * t) * RBr, RBr);
    if (lam) g = cm_scale(mpf_from_record<NL>(lam + (size_t)b * RBr, RBr - 4), g);
    T[t] = g;
  }
}

// C[r][c] (+)= sum_k op(A)(r,k) B[k][c];  op(A)(r,k) = A[r*lda+k] or conj(A[k*lda+r]); row-major
template <int NL>
__global__ void k_cgemm_mpf(const cmpf<NL>* A, int lda, int conjT, const cmpf<NL>* B, int ldb, cmpf<NL>* C, int ldc,
                            int rows, int cols, int K, int accumulate) {
  const int n = rows * cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t / cols, c = t % cols;
    cmpf<NL> acc = accumulate ? C[(size_t)r * ldc + c] : cm_zero<NL>();
    for (int k = 0; k < K; ++k) {
      const cmpf<NL>& b = B[(size_t)k * ldb + c];
      if (conjT) acc = cm_add(acc, cm_conjmul(A[(size_t)k * lda + r], b));
      else acc = cm_add(acc, cm_mul(A[(size_t)r * lda + k], b));
    }
    C[(size_t)r * ldc + c] = acc;
  }
}

// Y (+)= s X with s a complex record (O matrix entry)
template <int NL>
__global__ void k_caxpy_rec(const uint32_t* s, const cmpf<NL>* X, cmpf<NL>* Y, int n, int accumulate, int RBr) {
  const cmpf<NL> a = cm_from_rec<NL>(s, RBr);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    cmpf<NL> v = cm_mul(a, X[t]);
    Y[t] = accumulate ? cm_add(Y[t], v) : v;
  }
}

// rho(a, b) = E_(b,a) / sum_x E_(x,x) ; E_j are 1x1 at stride X
template <int NL>
__global__ void k_rdo_out(const cmpf<NL>* E, int X, int D, uint32_t* out, int RBr, int p) {
  __shared__ mpf<NL> s_inv;
  if (threadIdx.x == 0) {
    mpf<NL> tr = mpf_zero<NL>();
    for (int x = 0; x < D; ++x) tr = mpf_add(tr, E[(size_t)(x * D + x) * X].re);
    s_inv = mpf_recip(tr);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < D * D; t += blockDim.x) {
    const int a = t / D, b = t % D;
    cm_to_rec<NL>(cm_scale(s_inv, E[(size_t)(b * D + a) * X]), out + (size_t)(2 * t) * RBr, RBr, p);
  }
}

template <int NL>
__global__ void k_set_one(cmpf<NL>* E) {
  E[0] = {mpf_from_int<NL>(1), mpf_zero<NL>()};
}

// out = num / den (complex / real part of den), plus raw num, den records
template <int NL>
__global__ void k_ratio(const cmpf<NL>* num, const cmpf<NL>* den, uint32_t* out, uint32_t* den_out, int RBr, int p) {
  const mpf<NL> inv = mpf_recip(den->re);
  if (out) cm_to_rec<NL>(cm_scale(inv, *num), out, RBr, p);
  if (den_out) mpf_to_record<NL>(den->re, den_out, RBr - 4, p);
}

// ||U^H U - I||_max <= 2^(-p+16) -> *bad = 1 otherwise (one CTA)
template <int NL>
__global__ void k_unitary(const uint32_t* U, int d, int p, int* bad, int RBr) {
  const mpf<NL> tol = mpf_ldexp(mpf_from_int<NL>(1), 16 - (int64_t)p);
  for (int t = threadIdx.x; t < d * d; t += blockDim.x) {
    const int a = t / d, b = t % d;
    cmpf<NL> acc = cm_zero<NL>();
    for (int r = 0; r < d; ++r)
      acc = cm_add(acc, cm_conjmul(cm_from_rec<NL>(U + (size_t)(2 * (r * d + a)) * RBr, RBr),
                                   cm_from_rec<NL>(U + (size_t)(2 * (r * d + b)) * RBr, RBr)));
    if (a == b) acc.re = mpf_sub(acc.re, mpf_from_int<NL>(1));
    if (mpf_cmp_abs(acc.re, tol) > 0 || mpf_cmp_abs(acc.im, tol) > 0) atomicExch(bad, 1);
  }
}

}  // namespace mpsb

namespace mpsb {

// -------------------------------------------------------------------- host drivers
template <class T>
void run_onesite(int p, const uint32_t* G, uint32_t* Gout, const uint32_t* U, int nab, cudaStream_t st) {
  k_onesite<T::NL><<<std::max(1, std::min(256, (nab + 127) / 128)), 128, 0, st>>>(G, Gout, U, nab, record_words(p), p);
}

template <class T>
size_t amp_scratch_bytes(int maxchi, int nblocks) { return sizeof(cmpf<T::NL>) * 2 * (size_t)maxchi * nblocks; }

template <class T>
void run_amplitudes(int p, const uint32_t* const* G, const uint32_t* const* lam, const int* dims, int n,
                    const uint8_t* bits, long long nstates, int maxchi, void* scratch, int nblocks,
                    const uint32_t* v_in, uint32_t* out, cudaStream_t st) {
  k_amplitudes<T::NL><<<nblocks, 128, 0, st>>>(G, lam, dims, n, bits, nstates, maxchi, (cmpf<T::NL>*)scratch, v_in,
                                              out, record_words(p), p);
}

template <class T>
void run_unitary(int p, const uint32_t* U, int d, int* bad, cudaStream_t st) {
  k_unitary<T::NL><<<1, 64, 0, st>>>(U, d, p, bad, record_words(p));
}

template <class T>
size_t transfer_scratch_bytes(int maxchi) { return sizeof(cmpf<T::NL>) * (size_t)maxchi * maxchi * 24 + 4096; }

// <Psi|O|Psi> (O on window s0..s0+k-1, or O == null for <Psi|Psi>) and <Psi|Psi>; writes
// out = num/den (complex record) and den_out (real record), either may be null.
template <class T>
int run_transfer(int p, int n, const uint32_t* const* Gh, const uint32_t* const* lamh, const int* dims,
                 const uint32_t* O, int s0, int k, void* scratch, int maxchi, uint32_t* out, uint32_t* den_out,
                 cudaStream_t st) {
  constexpr int NL = T::NL;
  using C = cmpf<NL>;
  const int RBr = record_words(p);
  const size_t X = (size_t)maxchi * maxchi;
  C* base = (C*)scratch;
  C* E = base;            // current environment
  C* E2 = base + X;       // next environment
  C* Tm = base + 2 * X;   // [2][dl][dr]
  C* F = base + 4 * X;    // [2][dl][dr]
  C* Psi = base + 6 * X;  // [8][dl][dr] window tensors
  C* OPsi = base + 14 * X;
  C* tmp = base + 22 * X;
  int nl = 0;
  auto blocks = [](size_t m) { return (int)std::max<size_t>(1, std::min<size_t>(1184, (m + 127) / 128)); };
  auto gemm = [&](const C* A, int lda, int conjT, const C* B, int ldb, C* Cc, int ldc, int rows, int cols, int K,
                  int acc) {
    k_cgemm_mpf<NL><<<blocks((size_t)rows * cols), 128, 0, st>>>(A, lda, conjT, B, ldb, Cc, ldc, rows, cols, K, acc);
    ++nl;
  };
  // plain site transfer: E' = sum_i T_i^H (E T_i)
  auto site = [&](int s, C*& Ecur, C*& Enext) {
    const int dl = dims[s], dr = dims[s + 1];
    k_tmat<NL><<<blocks(2 * (size_t)dl * dr), 128, 0, st>>>(Gh[s], s ? lamh[s - 1] : nullptr, dl, dr, Tm, RBr);
    ++nl;
    for (int i = 0; i < 2; ++i) gemm(Ecur, dl, 0, Tm + (size_t)i * dl * dr, dr, F + (size_t)i * dl * dr, dr, dl, dr, dl, 0);
    for (int i = 0; i < 2; ++i)
      gemm(Tm + (size_t)i * dl * dr, dr, 1, F + (size_t)i * dl * dr, dr, Enext, dr, dr, dr, dl, i);
    C* t = Ecur; Ecur = Enext; Enext = t;
  };
  k_set_one<NL><<<1, 1, 0, st>>>(E); ++nl;
  C* Ec = E;
  C* En = E2;
  // denominator first (plain chain), kept in tmp[0]
  for (int s = 0; s < n; ++s) site(s, Ec, En);
  cudaMemcpyAsync(tmp, Ec, sizeof(C), cudaMemcpyDeviceToDevice, st);
  C* num = tmp;
  if (O) {
    k_set_one<NL><<<1, 1, 0, st>>>(Ec); ++nl;
    for (int s = 0; s < s0; ++s) site(s, Ec, En);
    const int D = 1 << k, dl = dims[s0], dr = dims[s0 + k];
    // Psi_x = T_{s0}^{x0} T_{s0+1}^{x1} ... (x0 = MSB)
    for (int x = 0; x < D; ++x) {
      C* P = Psi + (size_t)x * maxchi * maxchi;
      int cl = dims[s0];
      for (int t = 0; t < k; ++t) {
        const int s = s0 + t, bit = (x >> (k - 1 - t)) & 1;
        const int sl = dims[s], sr = dims[s + 1];
        k_tmat<NL><<<blocks(2 * (size_t)sl * sr), 128, 0, st>>>(Gh[s], s ? lamh[s - 1] : nullptr, sl, sr, Tm, RBr);
        ++nl;
        const C* Ti = Tm + (size_t)bit * sl * sr;
        if (t == 0) {
          cudaMemcpyAsync(P, Ti, sizeof(C) * sl * sr, cudaMemcpyDeviceToDevice, st);
        } else {
          gemm(P, sl, 0, Ti, sr, F, sr, cl, sr, sl, 0);
          cudaMemcpyAsync(P, F, sizeof(C) * cl * sr, cudaMemcpyDeviceToDevice, st);
        }
      }
    }
    // OPsi_x = sum_y O[x][y] Psi_y ; E' = sum_x Psi_x^H E OPsi_x
    for (int x = 0; x < D; ++x) {
      C* Q = OPsi + (size_t)x * maxchi * maxchi;
      for (int y = 0; y < D; ++y) {
        k_caxpy_rec<NL><<<blocks((size_t)dl * dr), 128, 0, st>>>(O + (size_t)2 * (x * D + y) * RBr,
                                                                Psi + (size_t)y * maxchi * maxchi, Q, dl * dr, y > 0, RBr);
        ++nl;
      }
    }
    for (int x = 0; x < D; ++x) {
      gemm(Ec, dl, 0, OPsi + (size_t)x * maxchi * maxchi, dr, F, dr, dl, dr, dl, 0);
      gemm(Psi + (size_t)x * maxchi * maxchi, dr, 1, F, dr, En, dr, dr, dr, dl, x);
    }
    { C* t = Ec; Ec = En; En = t; }
    for (int s = s0 + k; s < n; ++s) site(s, Ec, En);
    num = Ec;
  }
  k_ratio<NL><<<1, 1, 0, st>>>(num, tmp, out, den_out, RBr, p); ++nl;
  return nl;
}

}  // namespace mpsb

namespace mpsb {

// Reduced density operator of the kept sites (ascending, k <= 6) by transfer contraction
// (P:322-341 RDO_block / RDO): environments E_{(x,x')}(b,b') = sum conj(A_x(b)) A_{x'}(b')
// over the open kept multi-indices; traced sites apply sum_i T_i^H E T_i, kept sites split
// every environment into its 4 children conj(T_i)^T E T_i'.  rho(a,b) = E_{(b,a)} / trace.
template <class T>
int run_rdo(int p, int n, const uint32_t* const* Gh, const uint32_t* const* lamh, const int* dims,
            const int* keep, int k, void* scratch, int maxchi, uint32_t* out, cudaStream_t st) {
  constexpr int NL = T::NL;
  using C = cmpf<NL>;
  const int RBr = record_words(p);
  const size_t X = (size_t)maxchi * maxchi;
  const int D = 1 << k, NE = D * D;   // final number of environments
  C* base = (C*)scratch;
  C* Ea = base;                 // NE environments (ping)
  C* Eb = base + NE * X;        // NE environments (pong)
  C* Tm = base + 2 * NE * X;    // [2][dl][dr]
  C* F = Tm + 2 * X;            // work
  int nl = 0;
  auto blocks = [](size_t m) { return (int)std::max<size_t>(1, std::min<size_t>(1184, (m + 127) / 128)); };
  auto gemm = [&](const C* A, int lda, int conjT, const C* B, int ldb, C* Cc, int ldc, int rows, int cols, int K,
                  int acc) {
    k_cgemm_mpf<NL><<<blocks((size_t)rows * cols), 128, 0, st>>>(A, lda, conjT, B, ldb, Cc, ldc, rows, cols, K, acc);
    ++nl;
  };
  k_set_one<NL><<<1, 1, 0, st>>>(Ea); ++nl;
  int ne = 1, kk = 0;  // current number of environments, kept sites so far
  for (int s = 0; s < n; ++s) {
    const int dl = dims[s], dr = dims[s + 1];
    k_tmat<NL><<<blocks(2 * (size_t)dl * dr), 128, 0, st>>>(Gh[s], s ? lamh[s - 1] : nullptr, dl, dr, Tm, RBr); ++nl;
    const bool kept = kk < k && keep[kk] == s;
    if (!kept) {
      for (int e = 0; e < ne; ++e) {
        for (int i = 0; i < 2; ++i) gemm(Ea + e * X, dl, 0, Tm + (size_t)i * dl * dr, dr, F + (size_t)i * X, dr, dl, dr, dl, 0);
        for (int i = 0; i < 2; ++i) gemm(Tm + (size_t)i * dl * dr, dr, 1, F + (size_t)i * X, dr, Eb + e * X, dr, dr, dr, dl, i);
      }
    } else {
      // child (x i, x' i') of environment (x, x'): index ((x*2+i)*(2D') + (x'*2+i')) with D' = 2^(kk+1)
      const int Dold = 1 << kk, Dnew = Dold * 2;
      for (int x = 0; x < Dold; ++x)
        for (int xp = 0; xp < Dold; ++xp) {
          const C* E = Ea + (x * Dold + xp) * X;
          for (int ip = 0; ip < 2; ++ip) gemm(E, dl, 0, Tm + (size_t)ip * dl * dr, dr, F + (size_t)ip * X, dr, dl, dr, dl, 0);
          for (int i = 0; i < 2; ++i)
            for (int ip = 0; ip < 2; ++ip)
              gemm(Tm + (size_t)i * dl * dr, dr, 1, F + (size_t)ip * X, dr,
                   Eb + ((x * 2 + i) * Dnew + (xp * 2 + ip)) * X, dr, dr, dr, dl, 0);
        }
      ne = Dnew * Dnew;
      ++kk;
    }
    C* t = Ea; Ea = Eb; Eb = t;
  }
  // trace and output rho(a, b) = E_(b,a) / trace
  k_rdo_out<NL><<<1, 64, 0, st>>>(Ea, (int)X, D, out, RBr, p); ++nl;
  return nl;
}

}  // namespace mpsb
