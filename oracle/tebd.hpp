// ORACLE — test infrastructure only (see mp.hpp header).
// Plain, slow, step-by-step implementation of the ZKCM_QC time-dependent MPS
// method (§3.1, Eq. 1 at P:240-247, Eq. 2 at P:268-271, gate update
// P:275-284) with every step in the order and notation of SURVEY.md §8(c) O3.
#pragma once
#include <vector>

#include "mp.hpp"

namespace orc {

// Status codes (same numeric values as include/mps_b200.h, defined independently).
enum {
  ORC_OK = 0, ORC_EINVAL = -1, ORC_ENOTUNITARY = -2, ORC_ENOCONV = -3, ORC_EZEROBOND = -4,
  ORC_EOVERLAP = -5, ORC_EUNSUPPORTED = -6, ORC_ENOMEM = -7, ORC_ETOOBIG = -10
};

using CVec = std::vector<Cplx>;
using RVec = std::vector<Real>;

// Dense column-major M x N complex matrix: a[col*M + row].
struct CMat;
// Theta' = U (lam_l G_s lam_m G_{s+1} lam_r) of the two-site update, O3 steps 1-2.

struct CMat {
  int M = 0, N = 0;
  CVec a;
  CMat() {}
  CMat(int m, int n) : M(m), N(n), a((size_t)m * n) {}
  Cplx& at(int r, int c) { return a[(size_t)c * M + r]; }
  const Cplx& at(int r, int c) const { return a[(size_t)c * M + r]; }
};

struct SvdResult {
  int status = ORC_OK;
  int sweeps = 0;       // sweeps executed, the final check-only sweep included
  long rotations = 0;
  RVec sigma;           // N values, column order (unsorted)
  CMat X;               // M x N, a_j / sigma_j (sigma_j > 0), else the raw column
  CMat A;               // M x N, the rotated columns a_j (before normalisation)
  CMat V;               // N x N accumulated rotations
};

// Cyclic one-sided Jacobi SVD of A (M x N, N <= M), SURVEY §8(c) O3 step 4-5.
SvdResult jacobi_svd(const CMat& A, int max_sweeps = 60, long max_pairs = -1);

// Left/right factorisation Theta = Ul diag(s) Wr^H, handling N > M by working on Theta^H
// (O3 step 3).  Returns sorted (descending, ties by index) and truncated factors.
struct Split {
  int status = ORC_OK;
  int sweeps = 0;
  long rotations = 0;
  int k = 0;            // kept
  RVec sigma_sorted;    // all min(M,N) singular values, descending
  RVec lam;             // k renormalised Schmidt values sigma/nu
  CMat Ul;              // M x k left factor  (columns X_b)
  CMat Wr;              // N x k right factor (columns V_b), Theta ~ Ul diag(sigma) Wr^H
  Real sum_sigma2;      // sum of all sigma^2
  Real nu;              // sqrt(sum kept sigma^2)
};
Split svd_truncate(const CMat& Theta, int chi_max, const Real& thr);

// Two-site update on window (s, s+1) -- SURVEY §8(c) O3 steps 1-8.
// Gamma tensors are [i][a][b] row-major, lam_* are the bond vectors (size = bond dim).
struct Update2 {
  int status = ORC_OK;
  int sweeps = 0;
  long rotations = 0;
  int k = 0;
  CVec GL, GR;          // new Gamma_s [2][chi_l][k], Gamma_{s+1} [2][k][chi_r]
  RVec lam;             // new lambda_s [k]
  RVec sigma_sorted;    // all singular values of Theta', descending
  CMat Theta;           // Theta' (2chi_l x 2chi_r) as contracted
};
struct CMat contract_two_site(const CVec& GL, const CVec& GR, const RVec& lam_l, const RVec& lam_m,
                              const RVec& lam_r, int chi_l, int chi_m, int chi_r, const CVec& U4);
Update2 update_two_site(const CVec& GL, const CVec& GR, const RVec& lam_l, const RVec& lam_m,
                        const RVec& lam_r, int chi_l, int chi_m, int chi_r, const CVec& U4,
                        int chi_max, const Real& thr);

// Three-site update on (s, s+1, s+2) with U(8), right-first split.
struct Update3 {
  int status = ORC_OK;
  int sweeps = 0;
  long rotations = 0;
  int k1 = 0, k2 = 0;
  CVec G0, G1, G2;      // [2][chi_l][k2], [2][k2][k1], [2][k1][chi_r]
  RVec lam1, lam2;      // new lambda_s [k2], lambda_{s+1} [k1]
  RVec sigma1, sigma2;  // all singular values of SVD#1, SVD#2 (descending)
};
Update3 update_three_site(const CVec& G0, const CVec& G1, const CVec& G2, const RVec& lam_l,
                          const RVec& lam_1, const RVec& lam_2, const RVec& lam_r, int chi_l,
                          int chi_1, int chi_2, int chi_r, const CVec& U8, int chi_max,
                          const Real& thr);

// The MPS of Eq. 1 in Vidal Gamma-lambda form.
struct Mps {
  int n = 0, chi_max = 1;
  Real thr;
  std::vector<CVec> G;      // G[s]: [2][m_{s-1}][m_s]
  std::vector<RVec> lam;    // lam[s], s = 0..n-2
  std::vector<int> m;       // bond dims m[s], s = 0..n-2
  long sweeps_total = 0;
  long gates = 0;
  int dl(int s) const { return s == 0 ? 1 : m[s - 1]; }
  int dr(int s) const { return s == n - 1 ? 1 : m[s]; }
};
int mps_init(Mps& st, int n, int chi_max, const Real& thr);
// Apply a d x d gate (row-major CVec, d = 2^k) on ascending sites; a two-qubit gate
// on (s, s+2) is embedded into U(8) with identity on s+1.
int mps_apply(Mps& st, const CVec& U, const int* sites, int k);
Cplx mps_amplitude(const Mps& st, const unsigned char* bits);
Real mps_norm2(const Mps& st);
Cplx mps_expect_raw(const Mps& st, const CVec& O, int s0, int k);  // <Psi|O|Psi>, no division

// Dense 2^n state-vector simulator (qubit 0 = MSB of the basis index).
struct Dense {
  int n = 0;
  CVec psi;
};
void dense_init(Dense& d, int n);
int dense_apply(Dense& d, const CVec& U, const int* sites, int k);

}  // namespace orc
