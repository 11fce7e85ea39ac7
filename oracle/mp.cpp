// ORACLE — test infrastructure only (see mp.hpp header).  Correctly rounded
// (RNE) multiprecision arithmetic written from the definitions.
#include "mp.hpp"

#include <algorithm>
#include <climits>
#include <cmath>

namespace orc {

static thread_local int g_prec = 256;
int prec() { return g_prec; }
void set_prec(int p) {
  if (p < 2 || p > MAXP) throw std::runtime_error("oracle: precision out of range");
  g_prec = p;
}
static inline int nlimbs() { return (g_prec + 63) / 64; }

// ------------------------------------------------------------------ limb helpers
static int bitlen(const u64* d, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (d[i]) return i * 64 + (64 - __builtin_clzll(d[i]));
  return 0;
}
static inline int getbit(const u64* d, int n, long b) {
  if (b < 0) return 0;
  long li = b / 64;
  if (li >= n) return 0;
  return (int)((d[li] >> (b % 64)) & 1);
}
static bool any_below(const u64* d, int n, long b) {  // any bit at position < b
  if (b <= 0) return false;
  long full = b / 64;
  for (long i = 0; i < full && i < n; ++i)
    if (d[i]) return true;
  if (full < n && (b % 64)) {
    u64 mask = (((u64)1) << (b % 64)) - 1;
    if (d[full] & mask) return true;
  }
  return false;
}
// dst[0..dn) = src >> s  (logical), src has sn limbs
static void shr(u64* dst, int dn, const u64* src, int sn, long s) {
  long q = s / 64;
  int r = (int)(s % 64);
  for (int i = 0; i < dn; ++i) {
    long j = i + q;
    u64 lo = (j < sn) ? src[j] : 0;
    u64 hi = (j + 1 < sn) ? src[j + 1] : 0;
    dst[i] = r ? ((lo >> r) | (hi << (64 - r))) : lo;
  }
}
// dst[0..dn) = src << s, src has sn limbs
static void shl(u64* dst, int dn, const u64* src, int sn, long s) {
  long q = s / 64;
  int r = (int)(s % 64);
  for (int i = 0; i < dn; ++i) {
    long j = i - q;
    u64 lo = (j >= 0 && j < sn) ? src[j] : 0;
    u64 lo2 = (j - 1 >= 0 && j - 1 < sn) ? src[j - 1] : 0;
    dst[i] = r ? ((lo << r) | (lo2 >> (64 - r))) : lo;
  }
}

// Round the exact non-negative integer mag[0..n) * 2^lo to p bits, RNE.
static Real round_mag(const u64* mag, int n, int64_t lo, bool neg) {
  Real r;
  const int p = g_prec, nl = nlimbs();
  int b = bitlen(mag, n);
  if (b == 0) return r;  // exact zero (+0)
  r.zero = false;
  r.neg = neg;
  if (b <= p) {
    shl(r.m, nl, mag, n, p - b);
    r.e = lo - (p - b);
    return r;
  }
  long sh = b - p;
  shr(r.m, nl, mag, n, sh);
  int half = getbit(mag, n, sh - 1);
  bool sticky = any_below(mag, n, sh - 1);
  if (half && (sticky || (r.m[0] & 1))) {
    // increment
    bool carry_out = true;
    for (int i = 0; i < nl; ++i) {
      if (++r.m[i] != 0) { carry_out = false; break; }
    }
    // overflow to 2^p ?  (carry out of the top limb when p is a multiple of 64)
    if (carry_out || bitlen(r.m, nl) > p) {
      std::memset(r.m, 0, sizeof(u64) * nl);
      r.m[(p - 1) / 64] = ((u64)1) << ((p - 1) % 64);
      sh += 1;
    }
  }
  r.e = lo + sh;
  return r;
}

// ------------------------------------------------------------------ basics
Real from_int(int64_t v) {
  Exact x;
  if (v == 0) return Real();
  x.neg = v < 0;
  u64 a = v < 0 ? (u64)(-(v + 1)) + 1 : (u64)v;
  x.n = 1; x.d[0] = a; x.e = 0;
  const Exact* t[1] = {&x};
  return round_sum(t, 1);
}

Real from_double(double v) {
  if (v == 0.0) return Real();
  if (!std::isfinite(v)) throw std::runtime_error("oracle: non-finite double");
  int k;
  double f = std::frexp(std::fabs(v), &k);  // f in [0.5,1)
  u64 mant = (u64)std::ldexp(f, 53);        // exact
  Exact x;
  x.neg = v < 0; x.n = 1; x.d[0] = mant; x.e = (int64_t)k - 53;
  const Exact* t[1] = {&x};
  return round_sum(t, 1);
}

double to_double(const Real& x) {
  if (x.zero) return 0.0;
  const int nl = nlimbs();
  int b = bitlen(x.m, nl);
  u64 top[1];
  long sh = b > 64 ? b - 64 : 0;
  shr(top, 1, x.m, nl, sh);
  double d = std::ldexp((double)top[0], (int)(x.e + sh));
  return x.neg ? -d : d;
}

Real neg(const Real& x) { Real r = x; if (!r.zero) r.neg = !r.neg; return r; }
Real absr(const Real& x) { Real r = x; r.neg = false; return r; }
int sign(const Real& x) { return x.zero ? 0 : (x.neg ? -1 : 1); }

int cmp_abs(const Real& a, const Real& b) {
  if (a.zero && b.zero) return 0;
  if (a.zero) return -1;
  if (b.zero) return 1;
  // both normalised to exactly p bits: compare exponents, then mantissas
  if (a.e != b.e) return a.e < b.e ? -1 : 1;
  for (int i = nlimbs() - 1; i >= 0; --i)
    if (a.m[i] != b.m[i]) return a.m[i] < b.m[i] ? -1 : 1;
  return 0;
}
int cmp(const Real& a, const Real& b) {
  int sa = sign(a), sb = sign(b);
  if (sa != sb) return sa < sb ? -1 : 1;
  if (sa == 0) return 0;
  int c = cmp_abs(a, b);
  return sa > 0 ? c : -c;
}
Real ldexp_r(const Real& x, int64_t k) { Real r = x; if (!r.zero) r.e += k; return r; }

// ------------------------------------------------------------------ exact values
Exact exact(const Real& x) {
  Exact r;
  if (x.zero) return r;
  r.neg = x.neg; r.e = x.e; r.n = nlimbs();
  std::memcpy(r.d, x.m, sizeof(u64) * r.n);
  return r;
}
Exact exact_mul(const Real& a, const Real& b) {
  Exact r;
  if (a.zero || b.zero) return r;
  const int n = nlimbs();
  r.neg = a.neg != b.neg;
  r.e = a.e + b.e;
  r.n = 2 * n;
  std::memset(r.d, 0, sizeof(u64) * r.n);
  for (int i = 0; i < n; ++i) {
    u64 carry = 0;
    for (int j = 0; j < n; ++j) {
      u128 t = (u128)a.m[i] * b.m[j] + r.d[i + j] + carry;
      r.d[i + j] = (u64)t;
      carry = (u64)(t >> 64);
    }
    r.d[i + n] = carry;
  }
  return r;
}
Exact exact_neg(Exact x) { x.neg = !x.neg; return x; }

// Correctly rounded sum of exact terms: align every term exactly on a common
// two's-complement integer buffer (no truncation at all), then round once.
Real round_sum(const Exact* const* t, int k) {
  int64_t lo = INT64_MAX, hi = INT64_MIN;
  int live = 0;
  for (int i = 0; i < k; ++i) {
    int b = bitlen(t[i]->d, t[i]->n);
    if (b == 0) continue;
    ++live;
    lo = std::min(lo, t[i]->e);
    hi = std::max(hi, t[i]->e + b);
  }
  if (!live) return Real();
  int64_t span = hi - lo;
  int nb = (int)(span / 64) + 3;  // +sign/carry head-room
  if (nb > BIGL) throw std::runtime_error("oracle: exponent gap exceeds exact-sum buffer");
  u64 acc[BIGL];
  std::memset(acc, 0, sizeof(u64) * nb);
  u64 sh[BIGL];
  for (int i = 0; i < k; ++i) {
    const Exact& x = *t[i];
    if (bitlen(x.d, x.n) == 0) continue;
    int64_t off = x.e - lo;
    int q = (int)(off / 64), r = (int)(off % 64);
    int m = x.n + 1;
    // shifted limbs of x by r bits
    for (int j = 0; j < m; ++j) {
      u64 cur = j < x.n ? x.d[j] : 0;
      u64 prev = j > 0 ? x.d[j - 1] : 0;
      sh[j] = r ? ((cur << r) | (prev >> (64 - r))) : cur;
    }
    if (!x.neg) {
      u64 c = 0;
      for (int j = q; j < nb; ++j) {
        u64 v = (j - q < m) ? sh[j - q] : 0;
        u128 s = (u128)acc[j] + v + c;
        acc[j] = (u64)s;
        c = (u64)(s >> 64);
        if (j - q >= m && c == 0) break;
      }
    } else {
      u64 bor = 0;
      for (int j = q; j < nb; ++j) {
        u64 v = (j - q < m) ? sh[j - q] : 0;
        u128 s = (u128)acc[j] - v - bor;
        acc[j] = (u64)s;
        bor = (u64)(s >> 64) ? 1 : 0;
        if (j - q >= m && bor == 0) break;
      }
    }
  }
  bool negres = (acc[nb - 1] >> 63) & 1;
  if (negres) {  // two's complement negate
    u64 c = 1;
    for (int j = 0; j < nb; ++j) {
      u128 s = (u128)(~acc[j]) + c;
      acc[j] = (u64)s;
      c = (u64)(s >> 64);
    }
  }
  return round_mag(acc, nb, lo, negres);
}

Real fsum2(const Exact& a, const Exact& b) { const Exact* t[2] = {&a, &b}; return round_sum(t, 2); }
Real fsum3(const Exact& a, const Exact& b, const Exact& c) {
  const Exact* t[3] = {&a, &b, &c};
  return round_sum(t, 3);
}

Real add(const Real& a, const Real& b) { return fsum2(exact(a), exact(b)); }
Real sub(const Real& a, const Real& b) { return fsum2(exact(a), exact_neg(exact(b))); }
Real mul(const Real& a, const Real& b) {
  Exact x = exact_mul(a, b);
  const Exact* t[1] = {&x};
  return round_sum(t, 1);
}

// ------------------------------------------------------------------ division
// q = floor(num / den), rem != 0 flag; num has nn limbs, den has dn limbs.
// Restoring bit-serial long division (one quotient bit per step).
static void divmod_bits(const u64* num, int nn, const u64* den, int dn, u64* q, int qn, bool* rem_nz) {
  const int rn = dn + 1;
  u64 R[2 * RL + 4];
  std::memset(R, 0, sizeof(u64) * rn);
  std::memset(q, 0, sizeof(u64) * qn);
  int nb = bitlen(num, nn);
  for (int b = nb - 1; b >= 0; --b) {
    // R = 2R + bit
    u64 c = (u64)getbit(num, nn, b);
    for (int j = 0; j < rn; ++j) {
      u64 nc = R[j] >> 63;
      R[j] = (R[j] << 1) | c;
      c = nc;
    }
    // compare R >= den
    bool ge = true;
    for (int j = rn - 1; j >= 0; --j) {
      u64 dj = j < dn ? den[j] : 0;
      if (R[j] != dj) { ge = R[j] > dj; break; }
    }
    if (ge) {
      u64 bor = 0;
      for (int j = 0; j < rn; ++j) {
        u64 dj = j < dn ? den[j] : 0;
        u128 s = (u128)R[j] - dj - bor;
        R[j] = (u64)s;
        bor = (u64)(s >> 64) ? 1 : 0;
      }
      if (b / 64 < qn) q[b / 64] |= ((u64)1) << (b % 64);
    }
  }
  *rem_nz = bitlen(R, rn) != 0;
}

Real div(const Real& a, const Real& b) {
  if (b.zero) throw std::runtime_error("oracle: division by zero");
  if (a.zero) return Real();
  const int p = g_prec, n = nlimbs();
  // num = ma << (p+1); quotient in [2^p, 2^(p+2)) has >= p+1 bits
  u64 num[2 * RL + 2];
  const int nn = 2 * n + 1;
  shl(num, nn, a.m, n, p + 1);
  u64 q[2 * RL + 2];
  const int qn = n + 2;
  bool rem;
  divmod_bits(num, nn, b.m, n, q, qn, &rem);
  // append sticky bit below the quotient
  Exact x;
  x.neg = a.neg != b.neg;
  x.n = qn + 1;
  shl(x.d, x.n, q, qn, 1);
  x.d[0] |= rem ? 1 : 0;
  x.e = a.e - b.e - (p + 1) - 1;
  const Exact* t[1] = {&x};
  return round_sum(t, 1);
}

// ------------------------------------------------------------------ square root
Real sqrt_r(const Real& a) {
  if (a.zero) return Real();
  if (a.neg) throw std::runtime_error("oracle: sqrt of negative");
  const int p = g_prec, n = nlimbs();
  // N = ma << s, (a.e - s) even, N has >= 2p+2 bits so isqrt(N) has >= p+1 bits
  int64_t s = p + 2;
  if (((a.e - s) % 2 + 2) % 2) s += 1;
  const int W = 2 * n + 2;
  u64 N[2 * RL + 4];
  shl(N, W, a.m, n, s);
  // restoring integer square root: res = floor(sqrt(N)), remainder N - res^2
  u64 res[2 * RL + 4], bit[2 * RL + 4], tmp[2 * RL + 4];
  std::memset(res, 0, sizeof(u64) * W);
  std::memset(bit, 0, sizeof(u64) * W);
  int nb = bitlen(N, W);
  int top = (nb - 1) & ~1;  // highest even bit position <= msb
  bit[top / 64] = ((u64)1) << (top % 64);
  while (bitlen(bit, W) != 0) {
    // tmp = res + bit
    u64 c = 0;
    for (int j = 0; j < W; ++j) {
      u128 t = (u128)res[j] + bit[j] + c;
      tmp[j] = (u64)t; c = (u64)(t >> 64);
    }
    bool ge = true;
    for (int j = W - 1; j >= 0; --j)
      if (N[j] != tmp[j]) { ge = N[j] > tmp[j]; break; }
    // res >>= 1
    u64 r2[2 * RL + 4];
    shr(r2, W, res, W, 1);
    if (ge) {
      u64 bor = 0;
      for (int j = 0; j < W; ++j) {
        u128 t = (u128)N[j] - tmp[j] - bor;
        N[j] = (u64)t; bor = (u64)(t >> 64) ? 1 : 0;
      }
      c = 0;
      for (int j = 0; j < W; ++j) {
        u128 t = (u128)r2[j] + bit[j] + c;
        r2[j] = (u64)t; c = (u64)(t >> 64);
      }
    }
    std::memcpy(res, r2, sizeof(u64) * W);
    u64 b2[2 * RL + 4];
    shr(b2, W, bit, W, 2);
    std::memcpy(bit, b2, sizeof(u64) * W);
  }
  bool rem = bitlen(N, W) != 0;
  Exact x;
  x.neg = false;
  x.n = n + 3;  // res has ~p+2 bits
  shl(x.d, x.n, res, W, 1);
  x.d[0] |= rem ? 1 : 0;
  x.e = (a.e - s) / 2 - 1;
  const Exact* t[1] = {&x};
  return round_sum(t, 1);
}

// ------------------------------------------------------------------ complex
Cplx cadd(const Cplx& a, const Cplx& b) { return {add(a.re, b.re), add(a.im, b.im)}; }
Cplx csub(const Cplx& a, const Cplx& b) { return {sub(a.re, b.re), sub(a.im, b.im)}; }
Cplx cmul(const Cplx& a, const Cplx& b) {
  Real re = fsum2(exact_mul(a.re, b.re), exact_neg(exact_mul(a.im, b.im)));
  Real im = fsum2(exact_mul(a.re, b.im), exact_mul(a.im, b.re));
  return {re, im};
}
Cplx cconj(const Cplx& a) { return {a.re, neg(a.im)}; }
Cplx cscale(const Real& s, const Cplx& a) { return {mul(s, a.re), mul(s, a.im)}; }
Cplx cdivr(const Cplx& a, const Real& s) { return {div(a.re, s), div(a.im, s)}; }
void cfma(Cplx& acc, const Cplx& x, const Cplx& y) {
  Real re = fsum3(exact(acc.re), exact_mul(x.re, y.re), exact_neg(exact_mul(x.im, y.im)));
  Real im = fsum3(exact(acc.im), exact_mul(x.re, y.im), exact_mul(x.im, y.re));
  acc.re = re; acc.im = im;
}
void cfma_conj(Cplx& acc, const Cplx& x, const Cplx& y) {
  // conj(x)*y = (xr yr + xi yi) + i (xr yi - xi yr)
  Real re = fsum3(exact(acc.re), exact_mul(x.re, y.re), exact_mul(x.im, y.im));
  Real im = fsum3(exact(acc.im), exact_mul(x.re, y.im), exact_neg(exact_mul(x.im, y.re)));
  acc.re = re; acc.im = im;
}
Real cabs2(const Cplx& a) { return fsum2(exact_mul(a.re, a.re), exact_mul(a.im, a.im)); }

// ------------------------------------------------------------------ records
size_t record_bytes(int p) { return 16 + 4 * (size_t)((p + 31) / 32); }

Real from_record(const unsigned char* rec) {
  int64_t ex; uint32_t sg;
  std::memcpy(&ex, rec, 8);
  std::memcpy(&sg, rec + 8, 4);
  const int L = (g_prec + 31) / 32;
  u64 limbs64[RL + 1] = {0};
  for (int k = 0; k < L; ++k) {
    uint32_t w; std::memcpy(&w, rec + 16 + 4 * k, 4);
    limbs64[k / 2] |= ((u64)w) << (32 * (k % 2));
  }
  if (ex == INT64_MIN || bitlen(limbs64, (L + 1) / 2) == 0) return Real();
  Exact x;
  x.neg = sg != 0;
  x.n = (L + 1) / 2;
  std::memcpy(x.d, limbs64, sizeof(u64) * x.n);
  x.e = ex - 32 * (int64_t)L;
  const Exact* t[1] = {&x};
  return round_sum(t, 1);  // exact when the record holds <= p bits
}

void to_record(const Real& x, unsigned char* rec) {
  const int L = (g_prec + 31) / 32;
  std::memset(rec, 0, record_bytes(g_prec));
  if (x.zero) {
    int64_t ex = INT64_MIN;
    std::memcpy(rec, &ex, 8);
    return;
  }
  const int p = g_prec, n = nlimbs();
  u64 M[RL + 1];
  shl(M, (L + 1) / 2, x.m, n, 32 * (int64_t)L - p);
  int64_t ex = x.e + p;
  uint32_t sg = x.neg ? 1 : 0;
  std::memcpy(rec, &ex, 8);
  std::memcpy(rec + 8, &sg, 4);
  for (int k = 0; k < L; ++k) {
    uint32_t w = (uint32_t)(M[k / 2] >> (32 * (k % 2)));
    std::memcpy(rec + 16 + 4 * k, &w, 4);
  }
}
Cplx cfrom_record(const unsigned char* rec) {
  Cplx c;
  c.re = from_record(rec);
  c.im = from_record(rec + record_bytes(g_prec));
  return c;
}
void cto_record(const Cplx& x, unsigned char* rec) {
  to_record(x.re, rec);
  to_record(x.im, rec + record_bytes(g_prec));
}

}  // namespace orc
