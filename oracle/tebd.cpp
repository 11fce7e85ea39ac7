// ORACLE — test infrastructure only (see mp.hpp header).
// Step-by-step ZKCM_QC MPS gate update following SURVEY.md §8(c) O3, whose steps
// restate PAPER.md §3.1 (Eq. 1; Schmidt form Eq. 2; the
// update touches only Q_s, V_s, Q_{s+1}; truncation of small Schmidt
// coefficients; U(8) gates as elementary gates).
#include "tebd.hpp"

#include <algorithm>
#include <numeric>

namespace orc {

static Real one() { return from_int(1); }
static Cplx czero() { return Cplx(); }
static Cplx cone() { Cplx c; c.re = one(); return c; }
static Real dsum_abs2(const CMat& A, int col) {  // sum_r |a_r|^2, RN after each row (O1)
  Real acc;
  for (int r = 0; r < A.M; ++r) {
    const Cplx& x = A.at(r, col);
    acc = fsum3(exact(acc), exact_mul(x.re, x.re), exact_mul(x.im, x.im));
  }
  return acc;
}

// ---------------------------------------------------------------- Jacobi SVD
// cyclic order p = 0..N-2, q = p+1..N-1, V = I_N,
// tol = M * 2^-p, skip when alpha_p = 0, alpha_q = 0 or |gamma| <= tol sqrt(alpha_p alpha_q)
// (tested squared: |gamma|^2 <= tol^2 alpha_p alpha_q), or when either column is
// negligible (alpha <= tol^2 ||A||_F^2, reading R3b), at most max_sweeps sweeps;
// a sweep without any rotation means convergence (it is counted).
SvdResult jacobi_svd(const CMat& A0, int max_sweeps, long max_pairs) {
  SvdResult r;
  const int M = A0.M, N = A0.N;
  r.A = A0;
  r.V = CMat(N, N);
  for (int j = 0; j < N; ++j) r.V.at(j, j) = cone();
  CMat& A = r.A;
  CMat& V = r.V;
  const Real tol2 = ldexp_r(from_int((int64_t)M * M), -2 * (int64_t)prec());
  const Real ONE = one();
  // Negligible-column rule (reading R3b): a column with alpha_j <= tol^2 ||A||_F^2
  // is rounding noise of the matrix and is never rotated (else a rank-deficient A keeps
  // re-orthogonalising its noise columns at ever smaller scales and never converges).
  Real fro2;
  for (int j = 0; j < N; ++j) fro2 = add(fro2, dsum_abs2(A, j));
  const Real zcol = mul(tol2, fro2);
  bool converged = false;
  long pairs_seen = 0;  // bounded-sample timing only (bench.py cpu_baseline): stop early
  for (int sweep = 1; sweep <= max_sweeps; ++sweep) {
    r.sweeps = sweep;
    bool rotated = false;
    for (int p = 0; p < N - 1; ++p) {
      for (int q = p + 1; q < N; ++q) {
        if (max_pairs >= 0 && pairs_seen++ >= max_pairs) { r.status = ORC_ENOCONV; r.rotations = pairs_seen - 1; return r; }
        // (4.1) alpha_p, alpha_q, gamma = sum conj(a_p) a_q
        Real ap = dsum_abs2(A, p), aq = dsum_abs2(A, q);
        Cplx g;
        for (int row = 0; row < M; ++row) cfma_conj(g, A.at(row, p), A.at(row, q));
        // (4.2) skip test
        if (ap.zero || aq.zero || cmp(ap, zcol) <= 0 || cmp(aq, zcol) <= 0) continue;
        Real g2 = cabs2(g);
        if (g2.zero) continue;
        Real rhs = mul(tol2, mul(ap, aq));
        if (cmp(g2, rhs) <= 0) continue;
        // (4.3) zeta, t, c, s
        Real gabs = sqrt_r(g2);
        Real zeta = div(sub(aq, ap), ldexp_r(gabs, 1));
        Real sq = sqrt_r(add(ONE, mul(zeta, zeta)));
        Real num = sign(zeta) < 0 ? neg(ONE) : ONE;  // sgn(0) = +1
        Real t = div(num, add(absr(zeta), sq));
        Real c = div(ONE, sqrt_r(add(ONE, mul(t, t))));
        Real ct = mul(c, t);
        Cplx s;
        s.re = mul(ct, div(g.re, gabs));
        s.im = mul(ct, div(g.im, gabs));
        // (4.4) a_p <- c a_p - conj(s) a_q ; a_q <- s a_p + c a_q (same on V)
        auto rot = [&](CMat& B) {
          for (int row = 0; row < B.M; ++row) {
            const Cplx P = B.at(row, p), Q = B.at(row, q);
            Cplx np, nq;
            np.re = fsum3(exact_mul(c, P.re), exact_neg(exact_mul(s.re, Q.re)),
                          exact_neg(exact_mul(s.im, Q.im)));
            np.im = fsum3(exact_mul(c, P.im), exact_neg(exact_mul(s.re, Q.im)),
                          exact_mul(s.im, Q.re));
            nq.re = fsum3(exact_mul(s.re, P.re), exact_neg(exact_mul(s.im, P.im)),
                          exact_mul(c, Q.re));
            nq.im = fsum3(exact_mul(s.re, P.im), exact_mul(s.im, P.re), exact_mul(c, Q.im));
            B.at(row, p) = np;
            B.at(row, q) = nq;
          }
        };
        rot(A);
        rot(V);
        rotated = true;
        ++r.rotations;
      }
    }
    if (!rotated) { converged = true; break; }
  }
  if (!converged) r.status = ORC_ENOCONV;
  // (5) sigma_j = sqrt(alpha_j), X_j = a_j / sigma_j
  r.sigma.resize(N);
  r.X = CMat(M, N);
  for (int j = 0; j < N; ++j) {
    Real al = dsum_abs2(A, j);
    r.sigma[j] = sqrt_r(al);
    for (int row = 0; row < M; ++row)
      r.X.at(row, j) = r.sigma[j].zero ? A.at(row, j) : cdivr(A.at(row, j), r.sigma[j]);
  }
  return r;
}

// ---------------------------------------------------------------- sort / truncate
// work on Theta^H when N > M; stable descending
// order (ties by ascending column index); k = min(chi_max, #{sigma >= thr*||sigma||_2});
// lambda' = sigma / sqrt(sum_kept sigma^2).
Split svd_truncate(const CMat& Theta, int chi_max, const Real& thr) {
  Split sp;
  const bool trans = Theta.N > Theta.M;
  CMat A;
  if (!trans) {
    A = Theta;
  } else {
    A = CMat(Theta.N, Theta.M);
    for (int r = 0; r < Theta.M; ++r)
      for (int c = 0; c < Theta.N; ++c) A.at(c, r) = cconj(Theta.at(r, c));
  }
  SvdResult svd = jacobi_svd(A);
  sp.sweeps = svd.sweeps;
  sp.rotations = svd.rotations;
  if (svd.status != ORC_OK) { sp.status = svd.status; return sp; }
  const int N = A.N;
  std::vector<int> ord(N);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(),
                   [&](int a, int b) { return cmp(svd.sigma[a], svd.sigma[b]) > 0; });
  sp.sigma_sorted.resize(N);
  for (int b = 0; b < N; ++b) sp.sigma_sorted[b] = svd.sigma[ord[b]];
  Real sum_all;
  for (int b = 0; b < N; ++b) sum_all = fsum2(exact(sum_all), exact_mul(sp.sigma_sorted[b], sp.sigma_sorted[b]));
  sp.sum_sigma2 = sum_all;
  Real cut = mul(thr, sqrt_r(sum_all));
  int cnt = 0;
  while (cnt < N && !sp.sigma_sorted[cnt].zero && cmp(sp.sigma_sorted[cnt], cut) >= 0) ++cnt;
  int k = std::min(chi_max, cnt);
  if (k == 0) { sp.status = ORC_EZEROBOND; return sp; }
  sp.k = k;
  Real kept;
  for (int b = 0; b < k; ++b) kept = fsum2(exact(kept), exact_mul(sp.sigma_sorted[b], sp.sigma_sorted[b]));
  sp.nu = sqrt_r(kept);
  sp.lam.resize(k);
  for (int b = 0; b < k; ++b) sp.lam[b] = div(sp.sigma_sorted[b], sp.nu);
  // Theta = X S V^H (no transpose)  or  Theta = V S X^H (transposed)
  const CMat& L = trans ? svd.V : svd.X;
  const CMat& R = trans ? svd.X : svd.V;
  sp.Ul = CMat(L.M, k);
  sp.Wr = CMat(R.M, k);
  for (int b = 0; b < k; ++b) {
    for (int r = 0; r < L.M; ++r) sp.Ul.at(r, b) = L.at(r, ord[b]);
    for (int r = 0; r < R.M; ++r) sp.Wr.at(r, b) = R.at(r, ord[b]);
  }
  return sp;
}

static inline const Cplx& T3(const CVec& g, int i, int a, int b, int da, int db) {
  return g[((size_t)i * da + a) * db + b];
}

// ---------------------------------------------------------------- two-site update
CMat contract_two_site(const CVec& GL, const CVec& GR, const RVec& lam_l, const RVec& lam_m,
                       const RVec& lam_r, int chi_l, int chi_m, int chi_r, const CVec& U4) {
  // (1) L^i(a,b) = RN(RN(lam_l(a) G_s^i(a,b)) lam_m(b));  R^j(b,c) = RN(G_{s+1}^j(b,c) lam_r(c))
  CVec Lt((size_t)2 * chi_l * chi_m), Rt((size_t)2 * chi_m * chi_r);
  for (int i = 0; i < 2; ++i)
    for (int a = 0; a < chi_l; ++a)
      for (int b = 0; b < chi_m; ++b)
        Lt[((size_t)i * chi_l + a) * chi_m + b] =
            cscale(lam_m[b], cscale(lam_l[a], T3(GL, i, a, b, chi_l, chi_m)));
  for (int j = 0; j < 2; ++j)
    for (int b = 0; b < chi_m; ++b)
      for (int c = 0; c < chi_r; ++c)
        Rt[((size_t)j * chi_m + b) * chi_r + c] = cscale(lam_r[c], T3(GR, j, b, c, chi_m, chi_r));
  // Theta[(i,a),(j,c)] = sum_b L^i(a,b) R^j(b,c), b in order
  const int M = 2 * chi_l, N = 2 * chi_r;
  CMat Th(M, N);
  for (int i = 0; i < 2; ++i)
    for (int a = 0; a < chi_l; ++a)
      for (int j = 0; j < 2; ++j)
        for (int c = 0; c < chi_r; ++c) {
          Cplx acc;
          for (int b = 0; b < chi_m; ++b)
            cfma(acc, Lt[((size_t)i * chi_l + a) * chi_m + b], Rt[((size_t)j * chi_m + b) * chi_r + c]);
          Th.at(i * chi_l + a, j * chi_r + c) = acc;
        }
  // (2) Theta'[(i,a),(j,c)] = sum_{i'j'} U[2i+j, 2i'+j'] Theta[(i',a),(j',c)], order 00,01,10,11
  CMat Tp(M, N);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int a = 0; a < chi_l; ++a)
        for (int c = 0; c < chi_r; ++c) {
          Cplx acc;
          for (int ip = 0; ip < 2; ++ip)
            for (int jp = 0; jp < 2; ++jp)
              cfma(acc, U4[(size_t)(2 * i + j) * 4 + (2 * ip + jp)], Th.at(ip * chi_l + a, jp * chi_r + c));
          Tp.at(i * chi_l + a, j * chi_r + c) = acc;
        }
  return Tp;
}

Update2 update_two_site(const CVec& GL, const CVec& GR, const RVec& lam_l, const RVec& lam_m,
                        const RVec& lam_r, int chi_l, int chi_m, int chi_r, const CVec& U4,
                        int chi_max, const Real& thr) {
  Update2 out;
  CMat Tp = contract_two_site(GL, GR, lam_l, lam_m, lam_r, chi_l, chi_m, chi_r, U4);
  out.Theta = Tp;
  // (3)-(7)
  Split sp = svd_truncate(Tp, chi_max, thr);
  out.sweeps = sp.sweeps;
  out.rotations = sp.rotations;
  out.sigma_sorted = sp.sigma_sorted;
  if (sp.status != ORC_OK) { out.status = sp.status; return out; }
  const int k = sp.k;
  out.k = k;
  out.lam = sp.lam;
  // (8) Gamma_s'^i(a,b) = X[(i,a),b] / lam_l(a);  Gamma_{s+1}'^j(b,c) = conj(V[(j,c),b]) / lam_r(c)
  out.GL.resize((size_t)2 * chi_l * k);
  out.GR.resize((size_t)2 * k * chi_r);
  for (int i = 0; i < 2; ++i)
    for (int a = 0; a < chi_l; ++a)
      for (int b = 0; b < k; ++b)
        out.GL[((size_t)i * chi_l + a) * k + b] = cdivr(sp.Ul.at(i * chi_l + a, b), lam_l[a]);
  for (int j = 0; j < 2; ++j)
    for (int b = 0; b < k; ++b)
      for (int c = 0; c < chi_r; ++c)
        out.GR[((size_t)j * k + b) * chi_r + c] = cdivr(cconj(sp.Wr.at(j * chi_r + c, b)), lam_r[c]);
  return out;
}

// ---------------------------------------------------------------- three-site update
Update3 update_three_site(const CVec& G0, const CVec& G1, const CVec& G2, const RVec& lam_l,
                          const RVec& lam_1, const RVec& lam_2, const RVec& lam_r, int chi_l,
                          int chi_1, int chi_2, int chi_r, const CVec& U8, int chi_max,
                          const Real& thr) {
  Update3 out;
  // L^i = lam_l G0^i lam_1 ; Mj = G1^j lam_2 ; R^k = G2^k lam_r
  CVec Lt((size_t)2 * chi_l * chi_1), Mt((size_t)2 * chi_1 * chi_2), Rt((size_t)2 * chi_2 * chi_r);
  for (int i = 0; i < 2; ++i)
    for (int a = 0; a < chi_l; ++a)
      for (int b = 0; b < chi_1; ++b)
        Lt[((size_t)i * chi_l + a) * chi_1 + b] =
            cscale(lam_1[b], cscale(lam_l[a], T3(G0, i, a, b, chi_l, chi_1)));
  for (int j = 0; j < 2; ++j)
    for (int b = 0; b < chi_1; ++b)
      for (int c = 0; c < chi_2; ++c)
        Mt[((size_t)j * chi_1 + b) * chi_2 + c] = cscale(lam_2[c], T3(G1, j, b, c, chi_1, chi_2));
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < chi_2; ++c)
      for (int d = 0; d < chi_r; ++d)
        Rt[((size_t)k * chi_2 + c) * chi_r + d] = cscale(lam_r[d], T3(G2, k, c, d, chi_2, chi_r));
  // T^{ij}(a,c) = sum_b L^i(a,b) M^j(b,c)
  CVec Tt((size_t)4 * chi_l * chi_2);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int a = 0; a < chi_l; ++a)
        for (int c = 0; c < chi_2; ++c) {
          Cplx acc;
          for (int b = 0; b < chi_1; ++b)
            cfma(acc, Lt[((size_t)i * chi_l + a) * chi_1 + b], Mt[((size_t)j * chi_1 + b) * chi_2 + c]);
          Tt[((size_t)(2 * i + j) * chi_l + a) * chi_2 + c] = acc;
        }
  // Theta[(i,j,a),(k,d)] = sum_c T^{ij}(a,c) R^k(c,d)
  const int M = 4 * chi_l, N = 2 * chi_r;
  CMat Th(M, N);
  for (int ij = 0; ij < 4; ++ij)
    for (int a = 0; a < chi_l; ++a)
      for (int k = 0; k < 2; ++k)
        for (int d = 0; d < chi_r; ++d) {
          Cplx acc;
          for (int c = 0; c < chi_2; ++c)
            cfma(acc, Tt[((size_t)ij * chi_l + a) * chi_2 + c], Rt[((size_t)k * chi_2 + c) * chi_r + d]);
          Th.at(ij * chi_l + a, k * chi_r + d) = acc;
        }
  // Theta' = U(8) on the physical triple, index 4i+2j+k, primed order 000..111
  CMat Tp(M, N);
  for (int x = 0; x < 8; ++x)
    for (int a = 0; a < chi_l; ++a)
      for (int d = 0; d < chi_r; ++d) {
        Cplx acc;
        for (int y = 0; y < 8; ++y)
          cfma(acc, U8[(size_t)x * 8 + y], Th.at((y >> 1) * chi_l + a, (y & 1) * chi_r + d));
        Tp.at((x >> 1) * chi_l + a, (x & 1) * chi_r + d) = acc;
      }
  // SVD#1 (splits off site s+2): new lambda_{s+1}, Gamma_{s+2}
  Split s1 = svd_truncate(Tp, chi_max, thr);
  out.sweeps += s1.sweeps;
  out.rotations += s1.rotations;
  out.sigma1 = s1.sigma_sorted;
  if (s1.status != ORC_OK) { out.status = s1.status; return out; }
  const int k1 = s1.k;
  out.k1 = k1;
  out.lam2 = s1.lam;
  out.G2.resize((size_t)2 * k1 * chi_r);
  for (int k = 0; k < 2; ++k)
    for (int b = 0; b < k1; ++b)
      for (int d = 0; d < chi_r; ++d)
        out.G2[((size_t)k * k1 + b) * chi_r + d] = cdivr(cconj(s1.Wr.at(k * chi_r + d, b)), lam_r[d]);
  // M2[(i,a),(j,b)] = RN(X1[(2i+j) chi_l + a, b] * lambda'_{s+1}(b))   (2chi_l x 2k1)
  CMat M2(2 * chi_l, 2 * k1);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int a = 0; a < chi_l; ++a)
        for (int b = 0; b < k1; ++b)
          M2.at(i * chi_l + a, j * k1 + b) = cscale(s1.lam[b], s1.Ul.at((2 * i + j) * chi_l + a, b));
  Split s2 = svd_truncate(M2, chi_max, thr);
  out.sweeps += s2.sweeps;
  out.rotations += s2.rotations;
  out.sigma2 = s2.sigma_sorted;
  if (s2.status != ORC_OK) { out.status = s2.status; return out; }
  const int k2 = s2.k;
  out.k2 = k2;
  out.lam1 = s2.lam;
  out.G0.resize((size_t)2 * chi_l * k2);
  out.G1.resize((size_t)2 * k2 * k1);
  for (int i = 0; i < 2; ++i)
    for (int a = 0; a < chi_l; ++a)
      for (int c = 0; c < k2; ++c)
        out.G0[((size_t)i * chi_l + a) * k2 + c] = cdivr(s2.Ul.at(i * chi_l + a, c), lam_l[a]);
  for (int j = 0; j < 2; ++j)
    for (int c = 0; c < k2; ++c)
      for (int b = 0; b < k1; ++b)
        out.G1[((size_t)j * k2 + c) * k1 + b] = cdivr(cconj(s2.Wr.at(j * k1 + b, c)), s1.lam[b]);
  return out;
}

// ---------------------------------------------------------------- MPS state
int mps_init(Mps& st, int n, int chi_max, const Real& thr) {
  if (n < 1 || chi_max < 1) return ORC_EINVAL;
  st.n = n;
  st.chi_max = chi_max;
  st.thr = thr;
  st.G.assign(n, CVec(2));
  for (int s = 0; s < n; ++s) { st.G[s][0] = cone(); st.G[s][1] = czero(); }
  st.lam.assign(n > 1 ? n - 1 : 0, RVec(1, one()));
  st.m.assign(n > 1 ? n - 1 : 0, 1);
  return ORC_OK;
}

static RVec ones(int d) { return RVec(d, one()); }
static RVec lam_left(const Mps& st, int s) { return s == 0 ? ones(1) : st.lam[s - 1]; }
static RVec lam_right(const Mps& st, int s) { return s == st.n - 1 ? ones(1) : st.lam[s]; }

// ||U^H U - I||_max <= 2^(-p+16)
static bool is_unitary(const CVec& U, int d) {
  Real tol = ldexp_r(one(), 16 - (int64_t)prec());
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      Cplx acc;
      for (int r = 0; r < d; ++r) cfma_conj(acc, U[(size_t)r * d + a], U[(size_t)r * d + b]);
      if (a == b) acc.re = sub(acc.re, one());
      if (cmp(absr(acc.re), tol) > 0 || cmp(absr(acc.im), tol) > 0) return false;
    }
  return true;
}

// One gate on ascending sites spanning at most three consecutive sites.
static int apply_local(Mps& st, const CVec& U, const int* sites, int k) {
  st.gates++;
  const int s = sites[0];
  if (k == 1) {
    const int dl = st.dl(s), dr = st.dr(s);
    CVec G((size_t)2 * dl * dr);
    for (int i = 0; i < 2; ++i)
      for (int a = 0; a < dl; ++a)
        for (int b = 0; b < dr; ++b) {
          Cplx acc;
          for (int j = 0; j < 2; ++j) cfma(acc, U[(size_t)i * 2 + j], st.G[s][((size_t)j * dl + a) * dr + b]);
          G[((size_t)i * dl + a) * dr + b] = acc;
        }
    st.G[s] = G;
    return ORC_OK;
  }
  if (k == 2 && sites[1] == s + 1) {
    Update2 u = update_two_site(st.G[s], st.G[s + 1], lam_left(st, s), st.lam[s], lam_right(st, s + 1),
                                st.dl(s), st.m[s], st.dr(s + 1), U, st.chi_max, st.thr);
    st.sweeps_total += u.sweeps;
    if (u.status != ORC_OK) return u.status;
    st.G[s] = u.GL;
    st.G[s + 1] = u.GR;
    st.lam[s] = u.lam;
    st.m[s] = u.k;
    return ORC_OK;
  }
  CVec U8;
  if (k == 2) {
    if (sites[1] != s + 2) return ORC_EINVAL;  // routed by mps_apply
    // U8[4i+2m+k, 4i'+2m'+k'] = U[2i+k, 2i'+k'] delta(m, m')
    U8.assign(64, Cplx());
    for (int x = 0; x < 8; ++x)
      for (int y = 0; y < 8; ++y) {
        int mi = (x >> 1) & 1, mj = (y >> 1) & 1;
        if (mi != mj) continue;
        int a = ((x >> 2) << 1) | (x & 1), b = ((y >> 2) << 1) | (y & 1);
        U8[(size_t)x * 8 + y] = U[(size_t)a * 4 + b];
      }
  } else {
    if (sites[1] != s + 1 || sites[2] != s + 2) return ORC_EINVAL;
    U8 = U;
  }
  Update3 u = update_three_site(st.G[s], st.G[s + 1], st.G[s + 2], lam_left(st, s), st.lam[s],
                                st.lam[s + 1], lam_right(st, s + 2), st.dl(s), st.m[s], st.m[s + 1],
                                st.dr(s + 2), U8, st.chi_max, st.thr);
  st.sweeps_total += u.sweeps;
  if (u.status != ORC_OK) return u.status;
  st.G[s] = u.G0;
  st.G[s + 1] = u.G1;
  st.G[s + 2] = u.G2;
  st.lam[s] = u.lam1;
  st.lam[s + 1] = u.lam2;
  st.m[s] = u.k2;
  st.m[s + 1] = u.k1;
  return ORC_OK;
}

// General placement (R18; the paper's applyU on "chosen qubits", §3.2,
// and the n factor of O(g n m^3)): a gate on k distinct qubits in any order is
// first written on ascending sites (its index bits permuted), and a gate whose sites do not
// fit three consecutive sites is routed with exact SWAPs: the far qubits are moved next to
// the lowest one, the gate acts on consecutive sites, and the SWAPs are undone in reverse.
int mps_apply(Mps& st, const CVec& U, const int* sites, int k) {
  if (k < 1 || k > 3) return ORC_EINVAL;
  for (int i = 0; i < k; ++i) {
    if (sites[i] < 0 || sites[i] >= st.n) return ORC_EINVAL;
    for (int j = 0; j < i; ++j)
      if (sites[j] == sites[i]) return ORC_EINVAL;
  }
  const int d = 1 << k;
  if ((int)U.size() != d * d) return ORC_EINVAL;
  if (!is_unitary(U, d)) return ORC_ENOTUNITARY;
  if (k == 1) return apply_local(st, U, sites, 1);
  // pos[t] = index into `sites` of the t-th smallest site
  int pos[3] = {0, 1, 2};
  for (int a = 0; a < k; ++a)
    for (int b = a + 1; b < k; ++b)
      if (sites[pos[b]] < sites[pos[a]]) std::swap(pos[a], pos[b]);
  int q[3];
  for (int t = 0; t < k; ++t) q[t] = sites[pos[t]];
  // W[x][y] = U[x_orig][y_orig]: bit t of x (MSB first) is bit pos[t] of x_orig
  auto to_orig = [&](int x) {
    int r = 0;
    for (int t = 0; t < k; ++t)
      if ((x >> (k - 1 - t)) & 1) r |= 1 << (k - 1 - pos[t]);
    return r;
  };
  CVec W((size_t)d * d);
  for (int x = 0; x < d; ++x)
    for (int y = 0; y < d; ++y) W[(size_t)x * d + y] = U[(size_t)to_orig(x) * d + to_orig(y)];
  if ((k == 2 && q[1] - q[0] <= 2) || (k == 3 && q[2] == q[0] + 2)) return apply_local(st, W, q, k);
  // SWAP = [[1,0,0,0],[0,0,1,0],[0,1,0,0],[0,0,0,1]]
  CVec S(16, Cplx());
  S[0] = cone(); S[6] = cone(); S[9] = cone(); S[15] = cone();
  int rc = ORC_OK;
  auto swp = [&](int t) {
    const int pr[2] = {t - 1, t};
    return apply_local(st, S, pr, 2);
  };
  const int a = q[0];
  if (k == 2) {
    for (int t = q[1]; t > a + 1 && !rc; --t) rc = swp(t);
    if (rc) return rc;
    const int pr[2] = {a, a + 1};
    if ((rc = apply_local(st, W, pr, 2))) return rc;
    for (int t = a + 2; t <= q[1] && !rc; ++t) rc = swp(t);
    return rc;
  }
  for (int t = q[1]; t > a + 1 && !rc; --t) rc = swp(t);
  for (int t = q[2]; t > a + 2 && !rc; --t) rc = swp(t);
  if (rc) return rc;
  const int tr[3] = {a, a + 1, a + 2};
  if ((rc = apply_local(st, W, tr, 3))) return rc;
  for (int t = a + 3; t <= q[2] && !rc; ++t) rc = swp(t);
  for (int t = a + 2; t <= q[1] && !rc; ++t) rc = swp(t);
  return rc;
}

// c(b) = Gamma_0^{b0} lam_0 Gamma_1^{b1} lam_1 ... Gamma_{n-1}^{b_{n-1}}, left to right (Eq. 1)
Cplx mps_amplitude(const Mps& st, const unsigned char* bits) {
  int d = st.dr(0);
  CVec v(d);
  for (int b = 0; b < d; ++b) v[b] = st.G[0][(size_t)bits[0] * d + b];
  for (int s = 1; s < st.n; ++s) {
    const int dl = st.dl(s), dr = st.dr(s);
    CVec w(dl), nv(dr);
    for (int b = 0; b < dl; ++b) w[b] = cscale(st.lam[s - 1][b], v[b]);
    for (int c = 0; c < dr; ++c) {
      Cplx acc;
      for (int b = 0; b < dl; ++b) cfma(acc, w[b], st.G[s][((size_t)bits[s] * dl + b) * dr + c]);
      nv[c] = acc;
    }
    v = nv;
  }
  return v[0];
}

// T_s^i(b,c) = lam_{s-1}(b) Gamma_s^i(b,c), lam_{-1} = 1
static CVec tmat(const Mps& st, int s) {
  const int dl = st.dl(s), dr = st.dr(s);
  CVec T((size_t)2 * dl * dr);
  for (int i = 0; i < 2; ++i)
    for (int b = 0; b < dl; ++b)
      for (int c = 0; c < dr; ++c) {
        const Cplx& g = st.G[s][((size_t)i * dl + b) * dr + c];
        T[((size_t)i * dl + b) * dr + c] = s == 0 ? g : cscale(st.lam[s - 1][b], g);
      }
  return T;
}

// E'(c,c') = sum_x sum_b conj(K_x(b,c)) sum_b' E(b,b') L_x(b',c')
static CVec transfer(const CVec& E, int dl, int dr, const std::vector<CVec>& K, const std::vector<CVec>& Lx) {
  CVec En((size_t)dr * dr);
  for (size_t x = 0; x < K.size(); ++x) {
    CVec F((size_t)dl * dr);
    for (int b = 0; b < dl; ++b)
      for (int c = 0; c < dr; ++c) {
        Cplx acc;
        for (int bp = 0; bp < dl; ++bp) cfma(acc, E[(size_t)b * dl + bp], Lx[x][(size_t)bp * dr + c]);
        F[(size_t)b * dr + c] = acc;
      }
    for (int c = 0; c < dr; ++c)
      for (int cp = 0; cp < dr; ++cp) {
        Cplx& acc = En[(size_t)c * dr + cp];
        for (int b = 0; b < dl; ++b) cfma_conj(acc, K[x][(size_t)b * dr + c], F[(size_t)b * dr + cp]);
      }
  }
  return En;
}

static CVec site_transfer(const Mps& st, int s, const CVec& E) {
  CVec T = tmat(st, s);
  const int dl = st.dl(s), dr = st.dr(s);
  std::vector<CVec> K(2);
  for (int i = 0; i < 2; ++i) K[i].assign(T.begin() + (size_t)i * dl * dr, T.begin() + (size_t)(i + 1) * dl * dr);
  return transfer(E, dl, dr, K, K);
}

Real mps_norm2(const Mps& st) {
  CVec E(1, cone());
  for (int s = 0; s < st.n; ++s) E = site_transfer(st, s, E);
  return E[0].re;
}

Cplx mps_expect_raw(const Mps& st, const CVec& O, int s0, int k) {
  CVec E(1, cone());
  for (int s = 0; s < s0; ++s) E = site_transfer(st, s, E);
  // window tensors Psi_x = T_{s0}^{x0} ... T_{s0+k-1}^{x_{k-1}}, x0 = MSB
  const int D = 1 << k;
  const int dl = st.dl(s0), dr = st.dr(s0 + k - 1);
  std::vector<CVec> Psi(D);
  for (int x = 0; x < D; ++x) {
    CVec cur;
    int cl = dl, cr = 0;
    for (int t = 0; t < k; ++t) {
      const int s = s0 + t, bit = (x >> (k - 1 - t)) & 1;
      CVec T = tmat(st, s);
      const int sl = st.dl(s), sr = st.dr(s);
      CVec Ti(T.begin() + (size_t)bit * sl * sr, T.begin() + (size_t)(bit + 1) * sl * sr);
      if (t == 0) { cur = Ti; cr = sr; continue; }
      CVec nx((size_t)cl * sr);
      for (int a = 0; a < cl; ++a)
        for (int c = 0; c < sr; ++c) {
          Cplx acc;
          for (int b = 0; b < cr; ++b) cfma(acc, cur[(size_t)a * cr + b], Ti[(size_t)b * sr + c]);
          nx[(size_t)a * sr + c] = acc;
        }
      cur = nx;
      cr = sr;
    }
    Psi[x] = cur;
  }
  std::vector<CVec> OPsi(D, CVec((size_t)dl * dr));
  for (int x = 0; x < D; ++x)
    for (size_t e = 0; e < (size_t)dl * dr; ++e) {
      Cplx acc;
      for (int y = 0; y < D; ++y) cfma(acc, O[(size_t)x * D + y], Psi[y][e]);
      OPsi[x][e] = acc;
    }
  E = transfer(E, dl, dr, Psi, OPsi);
  for (int s = s0 + k; s < st.n; ++s) E = site_transfer(st, s, E);
  return E[0];
}

// ---------------------------------------------------------------- dense simulator
void dense_init(Dense& d, int n) {
  d.n = n;
  d.psi.assign((size_t)1 << n, Cplx());
  d.psi[0] = cone();
}

// psi'[x] = sum_{y'} U[y, y'] psi[x with the target bits := y'], sites[0] = MSB of y
int dense_apply(Dense& d, const CVec& U, const int* sites, int k) {
  const int n = d.n, D = 1 << k;
  for (int i = 0; i < k; ++i)
    if (sites[i] < 0 || sites[i] >= n) return ORC_EINVAL;
  CVec out(d.psi.size());
  for (size_t x = 0; x < d.psi.size(); ++x) {
    int y = 0;
    size_t base = x;
    for (int t = 0; t < k; ++t) {
      int bitpos = n - 1 - sites[t];
      y = (y << 1) | (int)((x >> bitpos) & 1);
      base &= ~((size_t)1 << bitpos);
    }
    Cplx acc;
    for (int yp = 0; yp < D; ++yp) {
      size_t xp = base;
      for (int t = 0; t < k; ++t)
        if ((yp >> (k - 1 - t)) & 1) xp |= (size_t)1 << (n - 1 - sites[t]);
      cfma(acc, U[(size_t)y * D + yp], d.psi[xp]);
    }
    out[x] = acc;
  }
  d.psi = out;
  return ORC_OK;
}

}  // namespace orc
