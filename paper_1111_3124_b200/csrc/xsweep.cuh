// Low-precision refinement sweeps of the preconditioner's basis (R22).
//
// After the first Newton-Schulz iteration the basis X_1 (N x N, its top 4 digits, unitary to
// ~2^-92) makes the columns of Theta' X_1 orthogonal only to ~1e-13 (the binary64 Jacobi's
// stopping level).  A Jacobi sweep at 4 digits (112 bits) moves that to ~2^-78, a second one at
// 7 digits (after Newton-Schulz iteration 1, on X_2) to ~2^-155: the p-bit iteration (k_jacobi)
// then starts where its second / third sweep used to and needs two sweeps fewer.  Per sweep:
//
//   A_t = Theta' X              (XD-digit GEMM, tensor cores)
//   G   = A_t^H A_t             (XD-digit GEMM)
//   k_xs_params: one round-robin sweep of rotation parameters computed from G alone (the dot
//     products gamma_pq = G_pq as they stand at the start of the sweep, the column norms alpha
//     updated incrementally), in double-double arithmetic, each rotation rounded to the
//     XD-digit grid with c = sqrt(1 - |s|^2) so that it is unitary to ~2^-(28 XD)
//   k_xs_apply: X <- X R_1 R_2 ... (every row of X independently: a CTA keeps R rows of X in
//     shared memory and applies the whole sequence of rotations, one barrier per step)
//
// GEMM form (R26, default; MPS_XS_GEMM=0 applies every rotation sequentially as above):
// the rotations of a refinement sweep are tiny (|s| ~ 2^-41 / 2^-78) and their parameters all
// come from the Gram matrix at the start of the sweep, so their product is exp(E) up to
// commutators of order |s|^2 |gamma|, E_pq = s_pq, E_qp = -conj(s_pq): k_xs_params writes E, and
//   F = E + E E / 2,   X <- X + X F      (two XD-digit tensor-core GEMMs, k_xs_copy)
// replaces k_xs_apply's N(N-1)/2 sequential row rotations.  I + F is unitary to |E|^3, below the
// 2^-92 / 2^-184 the basis is unitary to; the columns of Theta' X end as orthogonal as after the
// sequential sweep (both are first-order in the stale gamma).  Pairs with |s| >= 2^-32 (4
// digits) / 2^-64 (7 digits) -- near-degenerate column norms -- are left out of E and applied
// afterwards by k_xs_apply as exact rotations (items without such pairs exit at once).
//
// The sweeps only choose a better starting basis: X stays unitary to the level the next
// Newton-Schulz iteration needs, and every p-bit quantity is still computed exactly from
// Theta' by the later stages, whose stopping rule decides convergence (as for R19).
#pragma once
#include <cstdint>

#include "precond.cuh"

namespace mpsb {

// Per item (PreItem fields): X1 (= Xb) and X (= Xa) = N x N fixed (L stored digits, the top XD
// significant), exponent 1, rotated in place; G = N x N fixed (top XD digits), Hermitian, block
// exponent *eG; xs_rec = [N - 1][N / 2] rotation records (k_xs_params).
// records of the widest sweep (7 digits: 112 bytes per pair; 6 digits use the same padding)
inline size_t xs_rec_bytes(int N) { return align_up((size_t)112 * (N / 2) * (N > 1 ? N - 1 : 0)); }

// ---------------------------------------------------------------------------- double-double
struct dd { double hi, lo; };
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_norm(double hi, double lo) {
  const double s = hi + lo;
  return {s, lo - (s - hi)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  return dd_norm(s.hi, s.lo + a.lo + b.lo);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  dd s = dd_two_sum(a.hi, b);
  return dd_norm(s.hi, s.lo + a.lo);
}
__device__ __forceinline__ dd dd_mul_dd_d(double a, double b) {  // exact product
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  // r = a - q1 b
  dd p = dd_mul_dd_d(q1, b.hi);
  p.lo = fma(q1, b.lo, p.lo);
  dd r = dd_add(a, {-p.hi, -p.lo});
  const double q2 = r.hi / b.hi;
  return dd_norm(q1, q2);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {  // a > 0
  const double s = sqrt(a.hi);
  dd sq = dd_mul_dd_d(s, s);
  dd r = dd_add(a, {-sq.hi, -sq.lo});
  return dd_norm(s, r.hi / (2.0 * s));
}

__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = dd_mul_dd_d(a.hi, b.hi);
  return dd_norm(p.hi, p.lo + fma(a.hi, b.lo, a.lo * b.hi));
}
__device__ __forceinline__ dd dd_scale(dd a, int e) { return {ldexp(a.hi, e), ldexp(a.lo, e)}; }

// per-precision constants: XD digits padded to P (int4 multiples); a rotation record holds cf,
// sr, si (P ints each) and a flag word (4 ints); the "typical" zero-digit variant (ZC top
// fractional digits of c - 1 and ZS of s known to be zero: |s| ~ rho ~ 2^-40 / 2^-78)
template <int XD> struct XsT {
  static constexpr int P = (XD + 3) / 4 * 4;
  static constexpr int REC = 3 * P + 4;
  static constexpr int ZC = XD == 4 ? 3 : 5;  // |c - 1| ~ 2^-86 (4 digits), ~2^-141 (6, 7 digits)
  static constexpr int ZS = XD == 4 ? 1 : 2;  // |s| ~ 2^-40, ~2^-70
  // GEMM form: E (exponent 0) and F = E + E E / 2 have ZE zero top digits; pairs with
  // |Re s| or |Im s| >= 2^-EBIG stay sequential rotations
  static constexpr int ZE = XD == 4 ? 1 : 2;
  static constexpr int EBIG = XD == 4 ? 32 : 64;  // |s|^3 below 2^-92 / 2^-184
};

// the GEMM form of the refinement sweeps (R26) is on unless MPS_XS_GEMM=0
inline bool xs_gemm_form() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_XS_GEMM");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0;
}

// add the integer-valued double x (|x| < 2^(28 XD)) to the digit columns D (28-bit weights)
template <int XD>
__device__ __forceinline__ void xs_add_int(double x, int64_t (&D)[XD + 3]) {
  if (x == 0.0) return;
  int ex;
  const double m = frexp(fabs(x), &ex);
  uint64_t M53 = (uint64_t)ldexp(m, 53);  // |x| = M53 2^(ex - 53)
  int sh = ex - 53;
  if (sh < 0) { M53 >>= -sh; sh = 0; }     // exact: x is an integer
  const int q = sh / 28, r = sh % 28;
  const unsigned __int128 w = (unsigned __int128)M53 << r;
  const int64_t sg = x < 0 ? -1 : 1;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int64_t v = (int64_t)((w >> (28 * j)) & (j < 2 ? 0x0FFFFFFFull : 0xFFFFFFFFFFull));
    if (q + j < XD + 3) D[q + j] += sg * v;
  }
}
// Round v (|v| < 1) to the grid 2^(-28 XD): the rounded value (exact, as dd) and its XD
// balanced digits at scale 1 (value = sum K_k 2^(28k - 28 XD))
template <int XD>
__device__ __forceinline__ dd xs_round_grid(dd v, int32_t (&K)[XD]) {
  constexpr int S = 28 * XD;
  const double h = ldexp(v.hi, S), l = ldexp(v.lo, S);
  double hr, lr;
  if (fabs(h) >= 4503599627370496.0) { hr = h; lr = rint(l); }  // |h| >= 2^52: integer-valued
  else { hr = rint(h + l); lr = 0.0; }
  int64_t D[XD + 3];
#pragma unroll
  for (int k = 0; k < XD + 3; ++k) D[k] = 0;
  xs_add_int<XD>(hr, D);
  xs_add_int<XD>(lr, D);
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < XD; ++k) {
    const int64_t x = D[k] + c;
    c = (x + (1 << 27)) >> 28;
    K[k] = (int32_t)(x - (c << 28));
  }
  K[XD - 1] += (int32_t)(c << 28);  // (c is 0 for |v| < 1 - 2^-29)
  return dd_norm(ldexp(hr, -S), ldexp(lr, -S));
}

// value (in units of 2^eG) of a G entry from its top XD stored digits, as dd (digit L - 1 has
// weight 2^-28)
template <int L, int XD>
__device__ __forceinline__ dd xs_g_dd(const int32_t* p, size_t ld) {
  dd s = {0.0, 0.0};
#pragma unroll
  for (int j = 0; j < XD; ++j) s = dd_add_d(s, ldexp((double)p[(size_t)(L - 1 - j) * ld], -28 * (j + 1)));
  return s;
}

// Rotation records of one sweep: one CTA per item, thread per pair, one step at a time
// (the column norms alpha, double-double in shared memory, change with every rotation).
// The parameters follow DESIGN.md R17 in double-double: r = sqrt(d^2 + 4|g|^2),
// c^2 = (|d| + r)/(2r), s = sgn(d) g/(r c), t|g| = sgn(d)|g|^2/(r c^2) (d = alpha_q - alpha_p,
// g = G_pq); s is rounded to the XD-digit grid and c - 1 = -|s|^2 / (1 + sqrt(1 - |s|^2))
// computed from the rounded s, so that the rotation is unitary to ~2^-(28 XD).
// sel: 0 rotates PreItem::X1 (after Newton-Schulz iteration 0), 1 PreItem::X (iteration 1).
// (Sequential form only, MPS_XS_GEMM=0; the GEMM form computes its coefficients in k_xs_emat.)
template <int L, int XD>
__global__ void k_xs_params(const PreItem* items) {
  using T = XsT<XD>;
  const PreItem it = items[blockIdx.x];
  const int N = it.N, NP = N / 2;
  if (N < 2 || it.X1 == nullptr) return;
  extern __shared__ dd xs_alpha[];  // [N]
  __shared__ double s_tr;
  __shared__ int s_nrot, s_emax;
  if (threadIdx.x == 0) s_emax = -9999;
  for (int p = threadIdx.x; p < N; p += blockDim.x) xs_alpha[p] = xs_g_dd<L, XD>(it.G + ((size_t)(p * 2) * L) * N + p, N);
  if (threadIdx.x == 0) s_nrot = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int p = 0; p < N; ++p) t += fmax(xs_alpha[p].hi, 0.0);
    s_tr = t;
  }
  __syncthreads();
  // a pair is rotated only when G resolves its dot product to 2^-50 of sqrt(alpha_p alpha_q)
  // (G's entries carry 28 XD bits below 2^eG), its columns are not negligible and it is not
  // already orthogonal to 2^-(14 XD + 44)
  const double floor2 = ldexp(1.0, -2 * (28 * XD - 50));
  const double negl = ldexp(s_tr, -400);
  const double thr2 = ldexp(1.0, -2 * (14 * XD + 44));
  for (int step = 0; step < N - 1; ++step) {
    for (int i = threadIdx.x; i < NP; i += blockDim.x) {
      int p, q;
      rr_pair(N, step, i, p, q);
      int4* rec = it.xs_rec + ((size_t)step * NP + i) * (T::REC / 4);
      int flag = 0;
      const dd ap = xs_alpha[p], aq = xs_alpha[q];
      const double pa = ap.hi * aq.hi;
      if (ap.hi > negl && aq.hi > negl && pa > floor2) {
        const int32_t* gp = it.G + ((size_t)(q * 2) * L) * N + p;  // G(p, q), column q
        const dd gr = xs_g_dd<L, XD>(gp, N), gi = xs_g_dd<L, XD>(gp + (size_t)L * N, N);
        const dd g2 = dd_add(dd_mul(gr, gr), dd_mul(gi, gi));
        const dd d = dd_add(aq, dd_neg(ap));
        if (g2.hi > thr2 * pa) {
          const dd ad = d.hi < 0 ? dd_neg(d) : d;
          const dd r = dd_sqrt(dd_add(dd_mul(d, d), dd_scale(g2, 2)));
          const dd c = dd_sqrt(dd_div(dd_add(ad, r), dd_scale(r, 1)));
          dd sc = dd_div({1.0, 0.0}, dd_mul(r, c));
          if (d.hi < 0) sc = dd_neg(sc);
          int32_t Kc[XD], Kr[XD], Ki[XD];
          const dd sr = xs_round_grid<XD>(dd_mul(sc, gr), Kr);
          const dd si = xs_round_grid<XD>(dd_mul(sc, gi), Ki);
          const dd u = dd_add(dd_mul(sr, sr), dd_mul(si, si));
          xs_round_grid<XD>(dd_neg(dd_div(u, dd_add_d(dd_sqrt(dd_add_d(dd_neg(u), 1.0)), 1.0))), Kc);
          bool zc = true, zs = true;
#pragma unroll
          for (int k = 0; k < T::ZC; ++k) zc = zc && Kc[XD - 1 - k] == 0;
#pragma unroll
          for (int k = 0; k < T::ZS; ++k) zs = zs && Kr[XD - 1 - k] == 0 && Ki[XD - 1 - k] == 0;
          int32_t w[3 * T::P];
#pragma unroll
          for (int k = 0; k < T::P; ++k) {
            w[k] = k < XD ? Kc[k] : 0;
            w[T::P + k] = k < XD ? Kr[k] : 0;
            w[2 * T::P + k] = k < XD ? Ki[k] : 0;
          }
#pragma unroll
          for (int k = 0; k < 3 * T::P / 4; ++k) rec[k] = make_int4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
          flag = 1 | ((zc && zs) ? 2 : 0);
          if (jac_trace_items) {
            atomicAdd(&s_nrot, 1);
            int ex;
            frexp(fmax(fabs(sr.hi), fabs(si.hi)), &ex);
            atomicMax(&s_emax, ex);
          }
          const dd tg = dd_div(dd_mul(g2, sc), c);  // t |g| (signed like d)
          xs_alpha[p] = dd_add(ap, dd_neg(tg));
          xs_alpha[q] = dd_add(aq, tg);
        }
      }
      rec[3 * T::P / 4] = make_int4(flag, 0, 0, 0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && it.xs_big) *it.xs_big = -1;  // k_xs_apply applies every record
  if (jac_trace_items && threadIdx.x == 0 && (int)blockIdx.x < jac_trace_items)
    printf("xsweep(%d digits, sequential) item %d N %d rotated %d of %d pairs, max |s| < 2^%d, alpha0 %.6e trace %.6e\n",
           XD, (int)blockIdx.x, N, s_nrot, NP * (N - 1), s_emax, xs_alpha[0].hi, s_tr);
}

// GEMM form (R26), parallel over the pairs: every pair's coefficient comes from the Gram matrix as
// it stands at the start of the sweep, diagonal included (k_xs_params updates the column norms
// rotation by rotation, a change of relative order |s|^2 in alpha_q - alpha_p), so no pair waits
// for another: thread t = (step, i) of the round-robin order, record slot t.  Small pairs go to E,
// the others get a rotation record (R17 in full) for k_xs_apply and are counted in *xs_big
// (zeroed by k_xs_zero).
template <int L, int XD>
__global__ void __launch_bounds__(256) k_xs_emat(const PreItem* items, int sel) {
  using T = XsT<XD>;
  const PreItem it = items[blockIdx.y];
  const int N = it.N, NP = N / 2;
  if (N < 2 || it.X1 == nullptr) return;
  int32_t* E = sel ? it.X1 : it.X;
  extern __shared__ dd xs_alpha[];  // [N]
  __shared__ double s_tr;
  __shared__ int s_nbig, s_nrot, s_emax;
  for (int p = threadIdx.x; p < N; p += blockDim.x) xs_alpha[p] = xs_g_dd<L, XD>(it.G + ((size_t)(p * 2) * L) * N + p, N);
  if (threadIdx.x == 0) { s_nbig = 0; s_nrot = 0; s_emax = -9999; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int p = 0; p < N; ++p) t += fmax(xs_alpha[p].hi, 0.0);  // (in this order in every CTA)
    s_tr = t;
  }
  __syncthreads();
  const double floor2 = ldexp(1.0, -2 * (28 * XD - 50));
  const double negl = ldexp(s_tr, -400);
  const double thr2 = ldexp(1.0, -2 * (14 * XD + 44));
  const int npairs = NP * (N - 1);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < npairs; t += gridDim.x * blockDim.x) {
    const int step = t / NP, i = t % NP;
    int p, q;
    rr_pair(N, step, i, p, q);
    int4* rec = it.xs_rec + (size_t)t * (T::REC / 4);
    int flag = 0;
    const dd ap = xs_alpha[p], aq = xs_alpha[q];
    const double pa = ap.hi * aq.hi;
    if (ap.hi > negl && aq.hi > negl && pa > floor2) {
      const int32_t* gp = it.G + ((size_t)(q * 2) * L) * N + p;  // G(p, q), column q
      const dd gr = xs_g_dd<L, XD>(gp, N), gi = xs_g_dd<L, XD>(gp + (size_t)L * N, N);
      const dd g2 = dd_add(dd_mul(gr, gr), dd_mul(gi, gi));
      if (g2.hi > thr2 * pa) {
        const dd d = dd_add(aq, dd_neg(ap));
        int32_t Kr[XD], Ki[XD];
        dd sr = {0.0, 0.0}, si = {0.0, 0.0};
        bool small = false;
        if (g2.hi <= 8.673617379884035e-19 * (d.hi * d.hi)) {  // |gamma|^2 <= 2^-60 d^2: s = gamma / d
          const dd inv = dd_div({1.0, 0.0}, d);
          sr = xs_round_grid<XD>(dd_mul(inv, gr), Kr);
          si = xs_round_grid<XD>(dd_mul(inv, gi), Ki);
          small = fabs(sr.hi) < ldexp(1.0, -T::EBIG) && fabs(si.hi) < ldexp(1.0, -T::EBIG);
        }
        if (small) {
          flag = 4;
          int32_t* e1 = E + ((size_t)(q * 2) * L + (L - XD)) * N + p;
          int32_t* e2 = E + ((size_t)(p * 2) * L + (L - XD)) * N + q;
#pragma unroll
          for (int k = 0; k < XD; ++k) {
            e1[(size_t)k * N] = Kr[k];
            e1[(size_t)(L + k) * N] = Ki[k];
            e2[(size_t)k * N] = -Kr[k];
            e2[(size_t)(L + k) * N] = Ki[k];
          }
        } else {  // a sequential exact rotation (R17), as k_xs_params
          const dd ad = d.hi < 0 ? dd_neg(d) : d;
          const dd r = dd_sqrt(dd_add(dd_mul(d, d), dd_scale(g2, 2)));
          const dd c = dd_sqrt(dd_div(dd_add(ad, r), dd_scale(r, 1)));
          dd sc = dd_div({1.0, 0.0}, dd_mul(r, c));
          if (d.hi < 0) sc = dd_neg(sc);
          int32_t Kc[XD];
          sr = xs_round_grid<XD>(dd_mul(sc, gr), Kr);
          si = xs_round_grid<XD>(dd_mul(sc, gi), Ki);
          const dd u = dd_add(dd_mul(sr, sr), dd_mul(si, si));
          xs_round_grid<XD>(dd_neg(dd_div(u, dd_add_d(dd_sqrt(dd_add_d(dd_neg(u), 1.0)), 1.0))), Kc);
          int32_t w[3 * T::P];
#pragma unroll
          for (int k = 0; k < T::P; ++k) {
            w[k] = k < XD ? Kc[k] : 0;
            w[T::P + k] = k < XD ? Kr[k] : 0;
            w[2 * T::P + k] = k < XD ? Ki[k] : 0;
          }
#pragma unroll
          for (int k = 0; k < 3 * T::P / 4; ++k) rec[k] = make_int4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
          flag = 1;
          atomicAdd(&s_nbig, 1);
        }
        if (jac_trace_items) {
          atomicAdd(&s_nrot, 1);
          int ex;
          frexp(fmax(fabs(sr.hi), fabs(si.hi)), &ex);
          atomicMax(&s_emax, ex);
        }
      }
    }
    rec[3 * T::P / 4] = make_int4(flag, 0, 0, 0);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_nbig) atomicAdd(it.xs_big, s_nbig);
  if (jac_trace_items && threadIdx.x == 0 && (int)blockIdx.y < jac_trace_items && blockIdx.x == 0)
    printf("xsweep(%d digits, GEMM form) item %d N %d: CTA 0 rotated %d pairs (%d as sequential rotations), max |s| < 2^%d, trace %.6e\n",
           XD, (int)blockIdx.y, N, s_nrot, s_nbig, s_emax, s_tr);
}

// GEMM form: zero E (all L digits) before k_xs_params scatters the rotation coefficients into it
template <int L>
__global__ void __launch_bounds__(256) k_xs_zero(const PreItem* items, int sel) {
  const PreItem it = items[blockIdx.y];
  if (it.N < 2 || it.X1 == nullptr) return;
  int4* E = (int4*)(sel ? it.X1 : it.X);
  if (blockIdx.x == 0 && threadIdx.x == 0 && it.xs_big) *it.xs_big = 0;
  const size_t n4 = (size_t)it.N * it.N * 2 * L / 4;  // N even: a multiple of 4 ints
  for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < n4; w += (size_t)gridDim.x * blockDim.x)
    E[w] = make_int4(0, 0, 0, 0);
}
// GEMM form: X <- X + X F was written into G's buffer; copy it back over X
template <int L>
__global__ void __launch_bounds__(256) k_xs_copy(const PreItem* items, int sel) {
  const PreItem it = items[blockIdx.y];
  if (it.N < 2 || it.X1 == nullptr) return;
  int4* X = (int4*)(sel ? it.X : it.X1);
  const int4* S = (const int4*)it.G;
  const size_t n4 = (size_t)it.N * it.N * 2 * L / 4;
  for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < n4; w += (size_t)gridDim.x * blockDim.x) X[w] = S[w];
}

// acc (XD + 2 columns: digit products XD - 2 .. 2 XD - 1) +/-= K x, truncated like tmul_acc2,
// the top ZK digits of K known to be zero
template <int XD, int ZK, bool SUB>
__device__ __forceinline__ void xs_mul(int64_t (&acc)[XD + 2], const int32_t* K, const int32_t* x) {
#pragma unroll
  for (int i = 0; i < XD - ZK; ++i)
#pragma unroll
    for (int j = 0; j < XD; ++j)
      if (i + j >= XD - 2) acc[i + j - (XD - 2)] = madw(SUB ? -K[i] : K[i], x[j], acc[i + j - (XD - 2)]);
}

// Rotation of one row entry pair with Gauss's three-product complex multiplies:
//   y_p = c x_p - conj(s) x_q:  re = x_rp + cf x_rp - T1 - si (x_rq + x_iq)
//                               im = x_ip + cf x_ip - T1 - sr (x_iq - x_rq),   T1 = x_rq (sr - si)
//   y_q = c x_q + s x_p:        re = x_rq + cf x_rq + T2 - si (x_rp + x_ip)
//                               im = x_iq + cf x_iq + T2 + sr (x_ip - x_rp),   T2 = x_rp (sr + si)
// (c = 1 + cf; rc = [cf | sr | si]).  Digit-wise sums and differences stay below 2^28 (products
// below 2^56) and keep the known-zero top digits of s.
template <int XD, int ZC>
__device__ __forceinline__ void xs_out(int64_t (&acc)[XD + 2], const int64_t (&T)[XD + 2], bool Tneg,
                                       const int32_t* cf, const int32_t* x0, int32_t* y) {
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) acc[c] = Tneg ? acc[c] - T[c] : acc[c] + T[c];
#pragma unroll
  for (int j = 0; j < XD; ++j) acc[j + 2] += x0[j];  // 1 * x0 (the integer digit of c)
  xs_mul<XD, ZC, false>(acc, cf, x0);
  int32_t o[XD];
  tround2<XD>(acc, o);
#pragma unroll
  for (int j = 0; j < XD; ++j) y[j] = o[j];
}

template <int XD, int ZC, int ZS>
__device__ __forceinline__ void xs_rotate(const int32_t* rc, int32_t* xrp, int32_t* xip, int32_t* xrq, int32_t* xiq) {
  constexpr int P = XsT<XD>::P;
  const int32_t *cf = rc, *sr = rc + P, *si = rc + 2 * P;
  int32_t smi[XD], spl[XD], sq[XD], dq[XD], sp[XD], dp[XD];
#pragma unroll
  for (int k = 0; k < XD; ++k) {
    smi[k] = sr[k] - si[k];
    spl[k] = sr[k] + si[k];
    sq[k] = xrq[k] + xiq[k];
    dq[k] = xiq[k] - xrq[k];
    sp[k] = xrp[k] + xip[k];
    dp[k] = xip[k] - xrp[k];
  }
  int32_t yrp[XD], yip[XD], yrq[XD], yiq[XD];
  int64_t T[XD + 2], acc[XD + 2];
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) T[c] = 0;
  xs_mul<XD, ZS, false>(T, smi, xrq);  // T1
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) acc[c] = 0;
  xs_mul<XD, ZS, true>(acc, si, sq);
  xs_out<XD, ZC>(acc, T, true, cf, xrp, yrp);
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) acc[c] = 0;
  xs_mul<XD, ZS, true>(acc, sr, dq);
  xs_out<XD, ZC>(acc, T, true, cf, xip, yip);
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) T[c] = 0;
  xs_mul<XD, ZS, false>(T, spl, xrp);  // T2
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) acc[c] = 0;
  xs_mul<XD, ZS, true>(acc, si, sp);
  xs_out<XD, ZC>(acc, T, false, cf, xrq, yrq);
#pragma unroll
  for (int c = 0; c < XD + 2; ++c) acc[c] = 0;
  xs_mul<XD, ZS, false>(acc, sr, dp);
  xs_out<XD, ZC>(acc, T, false, cf, xiq, yiq);
#pragma unroll
  for (int j = 0; j < XD; ++j) { xrp[j] = yrp[j]; xip[j] = yip[j]; xrq[j] = yrq[j]; xiq[j] = yiq[j]; }
}

template <int P>
__device__ __forceinline__ void xs_ld(const int4* s, int hs, int32_t* v) {
#pragma unroll
  for (int k = 0; k < P / 4; ++k) {
    const int4 t = s[(size_t)k * hs];
    v[4 * k] = t.x; v[4 * k + 1] = t.y; v[4 * k + 2] = t.z; v[4 * k + 3] = t.w;
  }
}
template <int P>
__device__ __forceinline__ void xs_st(int4* s, int hs, const int32_t* v) {
#pragma unroll
  for (int k = 0; k < P / 4; ++k) s[(size_t)k * hs] = make_int4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
// shared-memory column stride (int4) of k_xs_apply: entry (c, re/im, row r) at c CS + ri R + r,
// its k-th group of 4 digits at + k N CS.  With 2 groups (XD = 7, R = 4 rows) a warp's 16-byte
// phase of 8 lanes covers two pairs of 4 rows; a column stride of 192 bytes puts consecutive
// columns 64 bytes apart modulo 128, so the two pairs hit different banks.
template <int XD, int R>
__host__ __device__ constexpr int xs_cs() { return 2 * R + (XsT<XD>::P > 4 ? 4 : 0); }

// Apply the sweep's rotations to rows [R blockIdx.x, + R) of X (sel: see k_xs_params): the rows
// stay in shared memory, entry (col c, re/im, row r) as P ints (its top XD digits, xs_cs
// layout); per step, task t = (pair t / R, row t % R).
template <int L, int XD, int R>
__global__ void __launch_bounds__(256) k_xs_apply(const PreItem* items, int sel) {
  using T = XsT<XD>;
  constexpr int P = T::P, Q = P / 4;
  const PreItem it = items[blockIdx.y];
  const int N = it.N, NP = N / 2;
  if (N < 2 || it.X1 == nullptr) return;
  if (it.xs_big && *it.xs_big == 0) return;  // GEMM form: every rotation of the sweep went into E
  int32_t* X = sel ? it.X : it.X1;
  const int r0 = blockIdx.x * R;
  if (r0 >= N) return;
  extern __shared__ int4 xs_rows[];  // [Q][N][CS]
  constexpr int CS = xs_cs<XD, R>();
  const int HS = N * CS;
  for (int t = threadIdx.x; t < N * 2 * R; t += blockDim.x) {
    const int r = t % R, ri = (t / R) % 2, c = t / (2 * R);
    int32_t v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) v[k] = 0;
    if (r0 + r < N) {
      const int32_t* g = X + ((size_t)(c * 2 + ri) * L + (L - XD)) * N + r0 + r;
#pragma unroll
      for (int k = 0; k < XD; ++k) v[k] = g[(size_t)k * N];
    }
    xs_st<P>(xs_rows + (size_t)c * CS + ri * R + r, HS, v);
  }
  __syncthreads();
  for (int step = 0; step < N - 1; ++step) {
    const int4* rs = it.xs_rec + (size_t)step * NP * (T::REC / 4);
    for (int t = threadIdx.x; t < NP * R; t += blockDim.x) {
      const int i = t / R, r = t % R;
      const int4* rr = rs + (size_t)i * (T::REC / 4);
      const int flag = __ldg(&rr[3 * Q].x);
      if (!(flag & 1)) continue;
      int p, q;
      rr_pair(N, step, i, p, q);
      int32_t rc[3 * P];
#pragma unroll
      for (int k = 0; k < 3 * Q; ++k) {
        const int4 u = __ldg(&rr[k]);
        rc[4 * k] = u.x; rc[4 * k + 1] = u.y; rc[4 * k + 2] = u.z; rc[4 * k + 3] = u.w;
      }
      int4* sp = xs_rows + (size_t)p * CS + r;
      int4* sq = xs_rows + (size_t)q * CS + r;
      int32_t xrp[P], xip[P], xrq[P], xiq[P];
      xs_ld<P>(sp, HS, xrp);
      xs_ld<P>(sp + R, HS, xip);
      xs_ld<P>(sq, HS, xrq);
      xs_ld<P>(sq + R, HS, xiq);
      if (flag & 2) xs_rotate<XD, T::ZC, T::ZS>(rc, xrp, xip, xrq, xiq);
      else xs_rotate<XD, 0, 0>(rc, xrp, xip, xrq, xiq);
      xs_st<P>(sp, HS, xrp);
      xs_st<P>(sp + R, HS, xip);
      xs_st<P>(sq, HS, xrq);
      xs_st<P>(sq + R, HS, xiq);
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < N * 2 * R; t += blockDim.x) {
    const int r = t % R, ri = (t / R) % 2, c = t / (2 * R);
    if (r0 + r >= N) continue;
    int32_t v[P];
    xs_ld<P>(xs_rows + (size_t)c * CS + ri * R + r, HS, v);
    int32_t* g = X + ((size_t)(c * 2 + ri) * L + (L - XD)) * N + r0 + r;
#pragma unroll
    for (int k = 0; k < XD; ++k) g[(size_t)k * N] = v[k];
    for (int k = 1; k <= L - XD; ++k) g[-(ptrdiff_t)k * N] = 0;  // digits below the sweep's (X_2's 7th)
  }
}

template <int XD, int R>
constexpr size_t xs_apply_smem(int N) { return (size_t)N * xs_cs<XD, R>() * XsT<XD>::P * 4; }

// the two kernels of one refinement sweep at XD digits for n items (descriptors on the
// device); sel: which X (see k_xs_params); launch count
template <int L, int XD>
inline int launch_xs_apply(const PreItem* d, int n, int maxN, int sel, cudaStream_t st) {
  constexpr int R = XD <= 4 ? 8 : 4;  // 64 KB of rows at N = 256
  const size_t sm = xs_apply_smem<XD, R>(maxN);
  smem_optin((const void*)k_xs_apply<L, XD, R>, (int)sm);
  k_xs_apply<L, XD, R><<<dim3((maxN + R - 1) / R, n), 256, sm, st>>>(d, sel);
  return 1;
}
template <int L, int XD>
inline int launch_xsweep(const PreItem* d, int n, int maxN, int sel, cudaStream_t st) {
  if (n <= 0 || maxN < 2) return 0;
  jacobi_trace_init();
  const int thr = std::min(1024, std::max(32, ((maxN / 2 + 31) / 32) * 32));
  k_xs_params<L, XD><<<n, thr, (size_t)maxN * sizeof(dd), st>>>(d);
  return 1 + launch_xs_apply<L, XD>(d, n, maxN, sel, st);
}
// GEMM form, first half: E from G (the caller then runs the two GEMMs, k_xs_copy and launch_xs_apply)
template <int L, int XD>
inline int launch_xs_emat(const PreItem* d, int n, int maxN, int sel, cudaStream_t st) {
  if (n <= 0 || maxN < 2) return 0;
  jacobi_trace_init();
  k_xs_zero<L><<<dim3(32, n), 256, 0, st>>>(d, sel);
  const int npairs = (maxN / 2) * (maxN - 1);
  k_xs_emat<L, XD><<<dim3(std::max(1, std::min(64, (npairs + 255) / 256)), n), 256, (size_t)maxN * sizeof(dd), st>>>(d, sel);
  return 2;
}

}  // namespace mpsb
