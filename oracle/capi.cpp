// ORACLE — test infrastructure only (see mp.hpp header).
// extern "C" entry points of liboracle.so, loaded by tests/ (via oracle/__init__.py),
// __graft_entry__.smoke() and bench.py's CPU baseline.  All numbers cross this
// boundary as interchange records (format restated in mp.hpp), complex = re record
// then im record, tensors row-major [i][a][b], matrices column-major where stated.
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tebd.hpp"

using namespace orc;
typedef unsigned char uchar;

static thread_local std::string g_err;

#define GUARD_BEGIN try {
#define GUARD_END                        \
  }                                      \
  catch (const std::exception& e) {      \
    g_err = e.what();                    \
    return -99;                          \
  }

static size_t RB() { return record_bytes(prec()); }
static size_t CB() { return 2 * record_bytes(prec()); }
static CVec read_c(const uchar* p, size_t n) {
  CVec v(n);
  for (size_t i = 0; i < n; ++i) v[i] = cfrom_record(p + i * CB());
  return v;
}
static RVec read_r(const uchar* p, size_t n) {
  RVec v(n);
  for (size_t i = 0; i < n; ++i) v[i] = from_record(p + i * RB());
  return v;
}
static void write_c(const CVec& v, uchar* p) {
  for (size_t i = 0; i < v.size(); ++i) cto_record(v[i], p + i * CB());
}
static void write_r(const RVec& v, uchar* p) {
  for (size_t i = 0; i < v.size(); ++i) to_record(v[i], p + i * RB());
}

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
size_t orc_record_bytes(int p) { return record_bytes(p); }

// Elementwise correctly rounded ops on n records (pins against mpmath / IEEE):
// op 0 add, 1 sub, 2 mul, 3 div, 4 sqrt(a), 5 round(a) (re-round a record to p bits),
// 6 complex mul (a, b, out are complex records), 7 fsum: out = RN(a*b + c) with c in out.
int orc_arith(int p, int op, int n, const uchar* a, const uchar* b, uchar* out) {
  GUARD_BEGIN
  set_prec(p);
  const size_t rb = RB();
  for (int i = 0; i < n; ++i) {
    if (op == 6) {
      Cplx x = cfrom_record(a + i * 2 * rb), y = cfrom_record(b + i * 2 * rb);
      cto_record(cmul(x, y), out + i * 2 * rb);
      continue;
    }
    Real x = from_record(a + i * rb), y, r;
    if (op <= 3 || op == 7) y = from_record(b + i * rb);
    switch (op) {
      case 0: r = add(x, y); break;
      case 1: r = sub(x, y); break;
      case 2: r = mul(x, y); break;
      case 3: r = div(x, y); break;
      case 4: r = sqrt_r(x); break;
      case 5: r = x; break;
      case 7: { Real c = from_record(out + i * rb); r = fsum2(exact_mul(x, y), exact(c)); break; }
      default: g_err = "bad op"; return ORC_EINVAL;
    }
    to_record(r, out + i * rb);
  }
  return 0;
  GUARD_END
}

// One-sided Jacobi SVD of a column-major M x N complex matrix (N <= M).
// sigma: N reals (column order, unsorted); X: M*N (a_j/sigma_j); V: N*N; both column-major.
int orc_svd(int p, int M, int N, const uchar* A, uchar* sigma, uchar* X, uchar* V, int* sweeps) {
  GUARD_BEGIN
  set_prec(p);
  if (N > M || M < 1 || N < 1) return ORC_EINVAL;
  CMat a(M, N);
  a.a = read_c(A, (size_t)M * N);
  SvdResult r = jacobi_svd(a);
  if (sweeps) *sweeps = r.sweeps;
  if (sigma) write_r(r.sigma, sigma);
  if (X) write_c(r.X.a, X);
  if (V) write_c(r.V.a, V);
  return r.status;
  GUARD_END
}

// Batched two-site gate update (kernel-level parity entry, mirrors mps_bench_update_batch).
// Per item b: GL [2][chi_l][chi_m], GR [2][chi_m][chi_r], lam_* (NULL = ones), U [4][4].
// Outputs per item: sigma_out (min(2chi_l,2chi_r) sorted), k_out, GL_out [2][chi_l][chi_max]
// (first k columns valid, stride chi_max), GR_out [2][chi_max][chi_r], lam_out [chi_max],
// theta_out (NULL or column-major (2chi_l) x (2chi_r)), sweeps_out.
// Theta' = U (lam_l G_L lam_m G_R lam_r) only (contract_two_site, lambda = 1 when null), for
// full-size samples where the SVD would take minutes.  Layout as orc_update2_batch's theta_out.
int orc_theta2(int p, int chi_l, int chi_m, int chi_r, const uchar* GL, const uchar* GR, const uchar* U,
               uchar* theta_out) {
  GUARD_BEGIN
  set_prec(p);
  CVec gl = read_c(GL, (size_t)2 * chi_l * chi_m);
  CVec gr = read_c(GR, (size_t)2 * chi_m * chi_r);
  CVec u = read_c(U, 16);
  RVec ll(chi_l, from_int(1)), lm(chi_m, from_int(1)), lr(chi_r, from_int(1));
  CMat T = contract_two_site(gl, gr, ll, lm, lr, chi_l, chi_m, chi_r, u);
  write_c(T.a, theta_out);
  return ORC_OK;
  GUARD_END
}

int orc_update2_batch(int p, int batch, int chi_l, int chi_m, int chi_r, int chi_max, double thr,
                      const uchar* GL, const uchar* GR, const uchar* lam_l, const uchar* lam_m,
                      const uchar* lam_r, const uchar* U, uchar* sigma_out, int* k_out,
                      uchar* GL_out, uchar* GR_out, uchar* lam_out, uchar* theta_out,
                      int* sweeps_out, int nthreads) {
  GUARD_BEGIN
  set_prec(p);
  const size_t rb = RB(), cb = CB();
  const int nsig = std::min(2 * chi_l, 2 * chi_r);
  std::atomic<int> next(0), status(0);
  std::string err;
  auto work = [&]() {
    set_prec(p);
    try {
      for (int b; (b = next++) < batch;) {
        CVec gl = read_c(GL + (size_t)b * 2 * chi_l * chi_m * cb, (size_t)2 * chi_l * chi_m);
        CVec gr = read_c(GR + (size_t)b * 2 * chi_m * chi_r * cb, (size_t)2 * chi_m * chi_r);
        RVec ll = lam_l ? read_r(lam_l + (size_t)b * chi_l * rb, chi_l) : RVec(chi_l, from_int(1));
        RVec lm = lam_m ? read_r(lam_m + (size_t)b * chi_m * rb, chi_m) : RVec(chi_m, from_int(1));
        RVec lr = lam_r ? read_r(lam_r + (size_t)b * chi_r * rb, chi_r) : RVec(chi_r, from_int(1));
        CVec u = read_c(U + (size_t)b * 16 * cb, 16);
        Update2 r = update_two_site(gl, gr, ll, lm, lr, chi_l, chi_m, chi_r, u, chi_max, from_double(thr));
        if (sweeps_out) sweeps_out[b] = r.sweeps;
        if (k_out) k_out[b] = r.k;
        if (theta_out) write_c(r.Theta.a, theta_out + (size_t)b * 4 * chi_l * chi_r * cb);
        if (sigma_out) write_r(r.sigma_sorted, sigma_out + (size_t)b * nsig * rb);
        if (r.status != ORC_OK) { status = r.status; continue; }
        const int k = r.k;
        if (GL_out)
          for (int i = 0; i < 2; ++i)
            for (int a = 0; a < chi_l; ++a)
              for (int c = 0; c < k; ++c)
                cto_record(r.GL[((size_t)i * chi_l + a) * k + c],
                           GL_out + (((size_t)b * 2 * chi_l + i * chi_l + a) * chi_max + c) * cb);
        if (GR_out)
          for (int j = 0; j < 2; ++j)
            for (int c = 0; c < k; ++c)
              for (int g = 0; g < chi_r; ++g)
                cto_record(r.GR[((size_t)j * k + c) * chi_r + g],
                           GR_out + (((size_t)b * 2 * chi_max + j * chi_max + c) * chi_r + g) * cb);
        if (lam_out)
          for (int c = 0; c < k; ++c) to_record(r.lam[c], lam_out + ((size_t)b * chi_max + c) * rb);
      }
    } catch (const std::exception& e) {
      err = e.what();
      status = -99;
    }
  };
  int nt = std::max(1, std::min(nthreads, batch));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(work);
  for (auto& t : th) t.join();
  if (status == -99) g_err = err;
  return status;
  GUARD_END
}

// Bounded-sample timing of the two-site update (bench.py cpu_baseline / --impl reference):
// thread t takes item t (inputs as orc_update2_batch, lambda = 1), times the contraction
// (O3 steps 1-2) and the first max_pairs Jacobi pair evaluations (step 4).  Per-thread
// seconds are returned; nothing is tuned for this.
int orc_bench_update2(int p, int nthreads, int chi, long max_pairs, const uchar* GL, const uchar* GR,
                      const uchar* U, double* t_contract, double* t_pairs, long* pairs_done) {
  GUARD_BEGIN
  set_prec(p);
  const size_t cb = CB();
  std::vector<std::thread> th;
  std::string err;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t]() {
      try {
        set_prec(p);
        CVec gl = read_c(GL + (size_t)t * 2 * chi * chi * cb, (size_t)2 * chi * chi);
        CVec gr = read_c(GR + (size_t)t * 2 * chi * chi * cb, (size_t)2 * chi * chi);
        CVec u = read_c(U + (size_t)t * 16 * cb, 16);
        RVec ones(chi, from_int(1));
        auto t0 = std::chrono::steady_clock::now();
        CMat Tp = contract_two_site(gl, gr, ones, ones, ones, chi, chi, chi, u);
        auto t1 = std::chrono::steady_clock::now();
        SvdResult r = jacobi_svd(Tp, 60, max_pairs);
        auto t2 = std::chrono::steady_clock::now();
        t_contract[t] = std::chrono::duration<double>(t1 - t0).count();
        t_pairs[t] = std::chrono::duration<double>(t2 - t1).count();
        pairs_done[t] = max_pairs;
        (void)r;
      } catch (const std::exception& e) {
        err = e.what();
      }
    });
  for (auto& x : th) x.join();
  if (!err.empty()) { g_err = err; return -99; }
  return 0;
  GUARD_END
}

// ---------------------------------------------------------------- MPS handle
struct OrcMps {
  int p;
  Mps st;
};

int orc_mps_new(int n, int p, int chi_max, double thr, void** out) {
  GUARD_BEGIN
  set_prec(p);
  auto* h = new OrcMps();
  h->p = p;
  int rc = mps_init(h->st, n, chi_max, from_double(thr));
  if (rc) { delete h; return rc; }
  *out = h;
  return 0;
  GUARD_END
}
void orc_mps_free(void* h) { delete (OrcMps*)h; }

int orc_mps_apply(void* hv, const uchar* U, const int* sites, int k) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (k < 1 || k > 3) return ORC_EINVAL;
  const int d = 1 << k;
  return mps_apply(h->st, read_c(U, (size_t)d * d), sites, k);
  GUARD_END
}

// A layer of pairwise-disjoint gates: the updates (pure functions of the current tensors)
// are computed in parallel threads and committed in gate order; the arithmetic of every
// gate is exactly mps_apply's (parallelism over disjoint gates only).
int orc_mps_apply_layer(void* hv, int ng, const uchar* const* U, const int* sites_flat, const int* k, int nthreads) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  Mps& st = h->st;
  std::vector<int> off(ng + 1, 0), used(st.n, 0);
  for (int g = 0; g < ng; ++g) {
    off[g + 1] = off[g] + k[g];
    const int* s = sites_flat + off[g];
    if (k[g] < 1 || k[g] > 3) return ORC_EINVAL;
    int lo = st.n, hi = -1;
    for (int i = 0; i < k[g]; ++i) {
      if (s[i] < 0 || s[i] >= st.n) return ORC_EINVAL;
      for (int j = 0; j < i; ++j) if (s[j] == s[i]) return ORC_EINVAL;
      lo = std::min(lo, s[i]);
      hi = std::max(hi, s[i]);
    }
    for (int q = lo; q <= hi; ++q) if (used[q]++) return ORC_EOVERLAP;  // whole span
  }
  // plain adjacent two-site and consecutive three-site gates run in parallel; the rest
  // (one-site, span-3 two-site, reordered or routed gates) sequentially through mps_apply
  std::vector<int> par;
  for (int g = 0; g < ng; ++g) {
    const int* s = sites_flat + off[g];
    bool adj2 = k[g] == 2 && s[1] == s[0] + 1, adj3 = k[g] == 3 && s[1] == s[0] + 1 && s[2] == s[0] + 2;
    if (adj2 || adj3) par.push_back(g);
  }
  std::vector<Update2> r2(ng);
  std::vector<Update3> r3(ng);
  std::vector<CVec> Us(ng);
  for (int g = 0; g < ng; ++g) Us[g] = read_c(U[g], (size_t)1 << (2 * k[g]));
  std::atomic<int> next(0);
  std::string err;
  auto lamL = [&](int s) { return s == 0 ? RVec(1, from_int(1)) : st.lam[s - 1]; };
  auto lamR = [&](int s) { return s == st.n - 1 ? RVec(1, from_int(1)) : st.lam[s]; };
  auto work = [&]() {
    set_prec(h->p);
    try {
      for (int j; (j = next++) < (int)par.size();) {
        const int g = par[j];
        const int s = sites_flat[off[g]];
        if (k[g] == 2)
          r2[g] = update_two_site(st.G[s], st.G[s + 1], lamL(s), st.lam[s], lamR(s + 1), st.dl(s), st.m[s],
                                  st.dr(s + 1), Us[g], st.chi_max, st.thr);
        else
          r3[g] = update_three_site(st.G[s], st.G[s + 1], st.G[s + 2], lamL(s), st.lam[s], st.lam[s + 1],
                                    lamR(s + 2), st.dl(s), st.m[s], st.m[s + 1], st.dr(s + 2), Us[g], st.chi_max,
                                    st.thr);
      }
    } catch (const std::exception& e) {
      err = e.what();
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < std::max(1, nthreads); ++t) th.emplace_back(work);
  for (auto& t : th) t.join();
  if (!err.empty()) { g_err = err; return -99; }
  int rc = 0;
  for (int g = 0; g < ng && !rc; ++g) {
    const int* s = sites_flat + off[g];
    const int q = s[0];
    bool adj2 = k[g] == 2 && s[1] == s[0] + 1, adj3 = k[g] == 3 && s[1] == s[0] + 1 && s[2] == s[0] + 2;
    if (adj2) {
      Update2& u = r2[g];
      st.sweeps_total += u.sweeps;
      st.gates++;
      if (u.status) { rc = u.status; break; }
      st.G[q] = u.GL; st.G[q + 1] = u.GR; st.lam[q] = u.lam; st.m[q] = u.k;
    } else if (adj3) {
      Update3& u = r3[g];
      st.sweeps_total += u.sweeps;
      st.gates++;
      if (u.status) { rc = u.status; break; }
      st.G[q] = u.G0; st.G[q + 1] = u.G1; st.G[q + 2] = u.G2;
      st.lam[q] = u.lam1; st.lam[q + 1] = u.lam2; st.m[q] = u.k2; st.m[q + 1] = u.k1;
    } else {
      rc = mps_apply(st, Us[g], s, k[g]);
    }
  }
  return rc;
  GUARD_END
}

int orc_mps_amplitude(void* hv, const uint8_t* bits, uchar* out) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  cto_record(mps_amplitude(h->st, bits), out);
  return 0;
  GUARD_END
}

int orc_mps_to_dense(void* hv, uchar* out) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  const int n = h->st.n;
  if (n > 20) return ORC_ETOOBIG;
  std::vector<unsigned char> bits(n);
  for (size_t x = 0; x < ((size_t)1 << n); ++x) {
    for (int q = 0; q < n; ++q) bits[q] = (x >> (n - 1 - q)) & 1;
    cto_record(mps_amplitude(h->st, bits.data()), out + x * CB());
  }
  return 0;
  GUARD_END
}

int orc_mps_bond_dims(void* hv, int* out) {
  auto* h = (OrcMps*)hv;
  for (int s = 0; s + 1 < h->st.n; ++s) out[s] = h->st.m[s];
  return 0;
}
long orc_mps_sweeps(void* hv) { return ((OrcMps*)hv)->st.sweeps_total; }

int orc_mps_schmidt(void* hv, int bond, uchar* out, int* m) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (bond < 0 || bond >= h->st.n - 1) return ORC_EINVAL;
  *m = h->st.m[bond];
  if (out) write_r(h->st.lam[bond], out);
  return 0;
  GUARD_END
}

int orc_mps_get_site(void* hv, int site, uchar* out, int* ml, int* mr) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (site < 0 || site >= h->st.n) return ORC_EINVAL;
  *ml = h->st.dl(site);
  *mr = h->st.dr(site);
  if (out) write_c(h->st.G[site], out);
  return 0;
  GUARD_END
}

// set_schmidt may change the bond dimension; the caller then sets both neighbouring sites.
int orc_mps_set_schmidt(void* hv, int bond, const uchar* in, int m) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (bond < 0 || bond >= h->st.n - 1 || m < 1) return ORC_EINVAL;
  h->st.m[bond] = m;
  h->st.lam[bond] = read_r(in, m);
  return 0;
  GUARD_END
}

int orc_mps_set_site(void* hv, int site, const uchar* in, int ml, int mr) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (site < 0 || site >= h->st.n) return ORC_EINVAL;
  if (ml != h->st.dl(site) || mr != h->st.dr(site)) return ORC_EINVAL;
  h->st.G[site] = read_c(in, (size_t)2 * ml * mr);
  return 0;
  GUARD_END
}

int orc_mps_norm2(void* hv, uchar* out) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  to_record(mps_norm2(h->st), out);
  return 0;
  GUARD_END
}

// <Psi|O|Psi> / <Psi|Psi> (ratio, complex) and the raw numerator; sites contiguous ascending.
int orc_mps_expect(void* hv, const uchar* O, const int* sites, int k, uchar* out, uchar* raw) {
  GUARD_BEGIN
  auto* h = (OrcMps*)hv;
  set_prec(h->p);
  if (k < 1 || k > 3) return ORC_EINVAL;
  for (int i = 0; i < k; ++i)
    if (sites[i] != sites[0] + i || sites[i] < 0 || sites[i] >= h->st.n) return ORC_EINVAL;
  const int d = 1 << k;
  Cplx num = mps_expect_raw(h->st, read_c(O, (size_t)d * d), sites[0], k);
  Real den = mps_norm2(h->st);
  if (raw) cto_record(num, raw);
  if (out) cto_record(cdivr(num, den), out);
  return 0;
  GUARD_END
}

// ---------------------------------------------------------------- dense handle
struct OrcDense {
  int p;
  Dense d;
};
int orc_dense_new(int n, int p, void** out) {
  GUARD_BEGIN
  set_prec(p);
  if (n < 1 || n > 22) return ORC_EINVAL;
  auto* h = new OrcDense();
  h->p = p;
  dense_init(h->d, n);
  *out = h;
  return 0;
  GUARD_END
}
void orc_dense_free(void* h) { delete (OrcDense*)h; }
int orc_dense_apply(void* hv, const uchar* U, const int* sites, int k) {
  GUARD_BEGIN
  auto* h = (OrcDense*)hv;
  set_prec(h->p);
  const int d = 1 << k;
  return dense_apply(h->d, read_c(U, (size_t)d * d), sites, k);
  GUARD_END
}
int orc_dense_get(void* hv, uchar* out) {
  GUARD_BEGIN
  auto* h = (OrcDense*)hv;
  set_prec(h->p);
  write_c(h->d.psi, out);
  return 0;
  GUARD_END
}

}  // extern "C"
