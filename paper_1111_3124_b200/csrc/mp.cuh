// Device multiprecision arithmetic for the MPS gate update (sm_100a).
//
// Two number formats:
//
//  * mpf<NL>  — scalar floating point: value = (-1)^neg * m * 2^(e - 32*NL), m an
//    NL-limb u32 integer with its top bit set (normalised), int64 exponent
//    (BASELINE.json north_star: "64-bit exponent"); zero <=> e == MPF_ZERO.
//    Used only on the O(N)-per-step scalar path: rotation parameters, norms,
//    conversions, sorting/truncation.  One guard limb beyond the record width.
//
//  * fixed-point signed digits ("fx") — the bulk format of the Jacobi matrix:
//    value = sum_{k<L} d_k 2^(28k) * 2^(E - 28L), d_k balanced int32 digits
//    (|d_k| <= 2^27 after normalisation), one exponent E per matrix column.
//    A product of two digit vectors is accumulated column-wise in int64 with
//    one IMAD.WIDE (signed 32x32+64) per digit pair and NO carry handling
//    (|d_i d_j| <= 2^54, so 512 terms fit an int64 column); carries are resolved
//    once per result.  Only product columns >= L-2 are formed ("truncated
//    product", the low part only ever influences bits 2^-25 ulp below the result).
#pragma once
#include <cstdint>

#define MPF_ZERO INT64_MIN

namespace mpsb {

// ----------------------------------------------------------------------------
// fixed-point digit helpers
// ----------------------------------------------------------------------------
constexpr int RADIX = 28;
constexpr int64_t HALF = (int64_t)1 << 27;

__device__ __forceinline__ int64_t madw(int32_t a, int32_t b, int64_t c) {
  int64_t d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// acc[c] (c = 0..L) holds product column k = c + L - 2.
template <int L>
__device__ __forceinline__ void tmul_acc(int64_t (&acc)[L + 1], const int32_t (&x)[L], const int32_t (&y)[L]) {
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(x[i], y[j], acc[i + j - (L - 2)]);
}
// acc -= x*y
template <int L>
__device__ __forceinline__ void tmul_sub(int64_t (&acc)[L + 1], const int32_t (&x)[L], const int32_t (&y)[L]) {
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (i + j >= L - 2) acc[i + j - (L - 2)] = madw(-x[i], y[j], acc[i + j - (L - 2)]);
}

// Balanced carry normalisation of the L+1 accumulator columns; returns the carry
// out of the top column (column 2L-1).
template <int L>
__device__ __forceinline__ int64_t tnorm(int64_t (&acc)[L + 1]) {
  int64_t carry = 0;
#pragma unroll
  for (int c = 0; c <= L; ++c) {
    int64_t v = acc[c] + carry;
    carry = (v + HALF) >> RADIX;
    acc[c] = v - (carry << RADIX);
  }
  return carry;
}

// Round the accumulated product sum V (columns L-2..2L-2 in acc) to
// round(2^k V / 2^(28L)) as L balanced digits, 0 <= k <= 24.
template <int L>
__device__ __forceinline__ void tround(int64_t (&acc)[L + 1], int k, int32_t (&out)[L]) {
  int64_t top = tnorm<L>(acc);  // digits acc[0..L] balanced, top = column 2L-1
  if (k) {
    // shift every digit left by k and renormalise (digits <= 2^51, no overflow)
    int64_t carry = 0;
#pragma unroll
    for (int c = 0; c <= L; ++c) {
      int64_t v = (acc[c] << k) + carry;
      carry = (v + HALF) >> RADIX;
      acc[c] = v - (carry << RADIX);
    }
    top = (top << k) + carry;
  }
  // rounding: columns L-2 (acc[0]) and L-1 (acc[1]) are dropped
  int64_t c0 = (acc[0] + HALF) >> RADIX;
  int64_t v1 = acc[1] + c0;
  int64_t carry = (v1 + HALF) >> RADIX;  // round to nearest unit of 2^(28L)
#pragma unroll
  for (int j = 0; j < L - 1; ++j) {
    int64_t v = acc[j + 2] + carry;
    carry = (v + HALF) >> RADIX;
    out[j] = (int32_t)(v - (carry << RADIX));
  }
  out[L - 1] = (int32_t)(top + carry);
}

// ----------------------------------------------------------------------------
// register-only word shifters (runtime shift counts without runtime array indices,
// which would put the arrays in local memory): log2(N) passes of selects
// ----------------------------------------------------------------------------
// w[i] <- w[i - s] (zeros shifted in), s >= 0
template <int N>
__device__ __forceinline__ void words_up(uint32_t (&w)[N], int s) {
  const bool all = s >= N;
#pragma unroll
  for (int b = 1; b < N; b <<= 1) {
    const bool on = (s & b) != 0;
#pragma unroll
    for (int i = N - 1; i >= 0; --i) w[i] = on ? (i >= b ? w[i - b] : 0u) : w[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = all ? 0u : w[i];
}
// w[i] <- w[i + s] (zeros shifted in), s >= 0
template <int N>
__device__ __forceinline__ void words_down(uint32_t (&w)[N], int s) {
  const bool all = s >= N;
#pragma unroll
  for (int b = 1; b < N; b <<= 1) {
    const bool on = (s & b) != 0;
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = on ? (i + b < N ? w[i + b] : 0u) : w[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = all ? 0u : w[i];
}

// ----------------------------------------------------------------------------
// mpf: scalar multiprecision floating point
// ----------------------------------------------------------------------------
template <int NL>
struct mpf {
  uint32_t m[NL];
  int64_t e;
  int neg;
};

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_zero() {
  mpf<NL> r;
#pragma unroll
  for (int i = 0; i < NL; ++i) r.m[i] = 0;
  r.e = MPF_ZERO;
  r.neg = 0;
  return r;
}
template <int NL>
__device__ __forceinline__ bool mpf_is_zero(const mpf<NL>& a) { return a.e == MPF_ZERO; }

// normalise an NL+1 limb magnitude t (t[NL] top) with exponent e (value = t * 2^(e - 32*(NL+1)))
// into a (round to nearest on the dropped limb).
template <int NL>
__device__ __forceinline__ mpf<NL> mpf_pack(uint32_t (&t)[NL + 1], int64_t e, int neg) {
  mpf<NL> r;
  // find the top non-zero limb
  int top = -1;
#pragma unroll
  for (int i = NL; i >= 0; --i)
    if (top < 0 && t[i]) top = i;
  if (top < 0) return mpf_zero<NL>();
  // shift left by whole limbs so that t[NL] != 0
  const int ls = NL - top;
  words_up<NL + 1>(t, ls);
  e -= 32 * (int64_t)ls;
  int sh = __clz(t[NL]);
  if (sh) {
#pragma unroll
    for (int i = NL; i > 0; --i) t[i] = (t[i] << sh) | (t[i - 1] >> (32 - sh));
    t[0] <<= sh;
    e -= sh;
  }
  // round on the guard limb t[0]
  uint32_t carry = t[0] >> 31;
#pragma unroll
  for (int i = 1; i <= NL; ++i) {
    uint32_t v = t[i] + carry;
    carry = (carry && v == 0) ? 1u : 0u;
    r.m[i - 1] = v;
  }
  if (carry) {  // rounded up to 2^(32NL)
#pragma unroll
    for (int i = 0; i < NL; ++i) r.m[i] = 0;
    r.m[NL - 1] = 0x80000000u;
    e += 1;
  }
  r.e = e;
  r.neg = neg;
  return r;
}

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_neg(mpf<NL> a) { a.neg ^= 1; return a; }
template <int NL>
__device__ __forceinline__ mpf<NL> mpf_abs(mpf<NL> a) { a.neg = 0; return a; }

// |a| vs |b|
template <int NL>
__device__ __forceinline__ int mpf_cmp_abs(const mpf<NL>& a, const mpf<NL>& b) {
  bool az = mpf_is_zero(a), bz = mpf_is_zero(b);
  if (az || bz) return az && bz ? 0 : (az ? -1 : 1);
  if (a.e != b.e) return a.e < b.e ? -1 : 1;
#pragma unroll
  for (int i = NL - 1; i >= 0; --i)
    if (a.m[i] != b.m[i]) return a.m[i] < b.m[i] ? -1 : 1;
  return 0;
}
template <int NL>
__device__ __forceinline__ int mpf_cmp(const mpf<NL>& a, const mpf<NL>& b) {
  int sa = mpf_is_zero(a) ? 0 : (a.neg ? -1 : 1);
  int sb = mpf_is_zero(b) ? 0 : (b.neg ? -1 : 1);
  if (sa != sb) return sa < sb ? -1 : 1;
  if (sa == 0) return 0;
  int c = mpf_cmp_abs(a, b);
  return sa > 0 ? c : -c;
}

// a * b.  Partial products a_i b_j with i + j < NL - 2 are skipped: their sum (and the
// carries they would send up) is < NL^2/2 units of limb NL-1, the guard limb that
// mpf_pack rounds on, so the result is faithful to ~2^-(32 NL - 6) relative.
template <int NL>
__device__ __noinline__ mpf<NL> mpf_mul(mpf<NL> a, mpf<NL> b) {
  if (mpf_is_zero(a) || mpf_is_zero(b)) return mpf_zero<NL>();
  constexpr int LO = NL > 2 ? NL - 2 : 0;  // lowest product column kept
  uint32_t p[2 * NL];
#pragma unroll
  for (int i = 0; i < 2 * NL; ++i) p[i] = 0;
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    uint64_t carry = 0;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      if (i + j < LO) continue;
      uint64_t t = (uint64_t)a.m[i] * b.m[j] + p[i + j] + carry;
      p[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    p[i + NL] = (uint32_t)carry;
  }
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i <= NL; ++i) t[i] = p[NL - 1 + i];
  // value = p * 2^(ea + eb - 64NL) = t * 2^(ea + eb - 64NL + 32(NL-1)) ; t has NL+1 limbs
  int64_t e = a.e + b.e - 64 * (int64_t)NL + 32 * (int64_t)(NL - 1) + 32 * (int64_t)(NL + 1);
  return mpf_pack<NL>(t, e, a.neg ^ b.neg);
}

// precision change: the top K limbs (truncation) / zero extension
template <int K, int NL>
__device__ __forceinline__ mpf<K> mpf_resize(const mpf<NL>& a) {
  mpf<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int src = NL - K + i;
    r.m[i] = src >= 0 ? a.m[src] : 0u;
  }
  r.e = a.e;
  r.neg = a.neg;
  return r;
}

// a + b
template <int NL>
__device__ __noinline__ mpf<NL> mpf_add(mpf<NL> a, mpf<NL> b) {
  if (mpf_is_zero(a)) return b;
  if (mpf_is_zero(b)) return a;
  if (mpf_cmp_abs(a, b) < 0) { mpf<NL> t = a; a = b; b = t; }
  int64_t d = a.e - b.e;  // >= 0
  if (d > 32 * (NL + 1)) return a;
  // a and b as NL+1 limbs (one guard limb at the bottom); tb = (b << 32 guard) >> d
  uint32_t ta[NL + 1], tb[NL + 1];
  ta[0] = 0;
  tb[0] = 0;
#pragma unroll
  for (int i = 0; i < NL; ++i) { ta[i + 1] = a.m[i]; tb[i + 1] = b.m[i]; }
  const int q = (int)(d >> 5), r = (int)(d & 31);
  words_down<NL + 1>(tb, q);
#pragma unroll
  for (int i = 0; i <= NL; ++i) tb[i] = __funnelshift_r(tb[i], i < NL ? tb[i + 1] : 0u, r);
  uint32_t t[NL + 1];
  int64_t e = a.e + 32;  // t[NL] top limb has the weight of a.m[NL-1]*2^32...
  if (a.neg == b.neg) {
    uint32_t carry = 0;
#pragma unroll
    for (int i = 0; i <= NL; ++i) {
      uint64_t s = (uint64_t)ta[i] + tb[i] + carry;
      t[i] = (uint32_t)s;
      carry = (uint32_t)(s >> 32);
    }
    if (carry) {  // shift right one limb, dropping the guard limb
#pragma unroll
      for (int i = 0; i < NL; ++i) t[i] = t[i + 1];
      t[NL] = carry;
      e += 32;
    }
  } else {
    uint32_t borrow = 0;
#pragma unroll
    for (int i = 0; i <= NL; ++i) {
      uint64_t s = (uint64_t)ta[i] - tb[i] - borrow;
      t[i] = (uint32_t)s;
      borrow = (uint32_t)(s >> 63);
    }
  }
  // value = t * 2^(a.e - 32NL - 32) with t of NL+1 limbs -> mpf_pack wants 2^(E - 32(NL+1))
  return mpf_pack<NL>(t, e - 32, a.neg);
}

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_sub(const mpf<NL>& a, const mpf<NL>& b) { return mpf_add(a, mpf_neg(b)); }

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_ldexp(mpf<NL> a, int64_t k) {
  if (!mpf_is_zero(a)) a.e += k;
  return a;
}

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_from_int(int64_t v) {
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i <= NL; ++i) t[i] = 0;
  uint64_t a = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
  t[NL] = (uint32_t)(a >> 32);
  t[NL - 1] = (uint32_t)a;
  // value = a = t * 2^(E - 32(NL+1)) with t = a * 2^(32(NL-1)) -> E = 64
  return mpf_pack<NL>(t, 64, v < 0);
}

// (f, E) with |a| ~= f * 2^E, f in [0.5, 1) as double (diagnostics / Newton seeds)
template <int NL>
__device__ __forceinline__ double mpf_frexp(const mpf<NL>& a, int64_t* E) {
  if (mpf_is_zero(a)) { *E = 0; return 0.0; }
  double f = ((double)a.m[NL - 1] * 4294967296.0 + (double)a.m[NL - 2]) * (1.0 / 18446744073709551616.0);
  *E = a.e;
  return a.neg ? -f : f;
}
template <int NL>
__device__ __forceinline__ mpf<NL> mpf_from_frexp(double f, int64_t E) {
  if (f == 0.0) return mpf_zero<NL>();
  int neg = f < 0;
  f = fabs(f);
  int k;
  f = frexp(f, &k);  // f in [0.5,1)
  uint64_t man = (uint64_t)ldexp(f, 64);
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i <= NL; ++i) t[i] = 0;
  t[NL] = (uint32_t)(man >> 32);
  t[NL - 1] = (uint32_t)man;
  return mpf_pack<NL>(t, E + k, neg);
}

// Newton iterations with precision doubling: the iteration that takes b correct bits to
// 2b runs with K limbs, K the smallest of 4, 7, 13, ... (2K-1) that holds 2b bits, and the
// last one with all NL limbs (53 -> ~100 -> ~200 -> ~400 bits).
template <int K, int NL>
struct NewtonNext {
  static constexpr int value = (2 * K - 1 < NL) ? 2 * K - 1 : NL;
};

// 1/b: y <- y + y(1 - b y)
template <int NL, int K>
__device__ __forceinline__ mpf<NL> recip_chain(const mpf<NL>& b, mpf<K> y) {
  const mpf<K> bk = mpf_resize<K>(b);
  const mpf<K> r = mpf_sub(mpf_from_int<K>(1), mpf_mul(bk, y));
  y = mpf_add(y, mpf_mul(y, r));
  if constexpr (K == NL) {
    return y;
  } else {
    constexpr int K2 = NewtonNext<K, NL>::value;
    return recip_chain<NL, K2>(b, mpf_resize<K2>(y));
  }
}
template <int NL>
__device__ __noinline__ mpf<NL> mpf_recip(const mpf<NL>& b) {
  int64_t E;
  double f = mpf_frexp(b, &E);
  constexpr int K0 = NL < 4 ? NL : 4;
  return recip_chain<NL, K0>(b, mpf_from_frexp<K0>(1.0 / f, -E));
}

// 1/sqrt(x), x > 0: y <- y + y(1 - x y^2)/2
template <int NL, int K>
__device__ __forceinline__ mpf<NL> rsqrt_chain(const mpf<NL>& x, mpf<K> y) {
  const mpf<K> xk = mpf_resize<K>(x);
  const mpf<K> r = mpf_sub(mpf_from_int<K>(1), mpf_mul(xk, mpf_mul(y, y)));
  y = mpf_add(y, mpf_ldexp(mpf_mul(y, r), -1));
  if constexpr (K == NL) {
    return y;
  } else {
    constexpr int K2 = NewtonNext<K, NL>::value;
    return rsqrt_chain<NL, K2>(x, mpf_resize<K2>(y));
  }
}
template <int NL>
__device__ __noinline__ mpf<NL> mpf_rsqrt(const mpf<NL>& x) {
  int64_t E;
  double f = mpf_frexp(x, &E);  // x = f 2^E
  if (E & 1) { f *= 0.5; E += 1; }
  constexpr int K0 = NL < 4 ? NL : 4;
  return rsqrt_chain<NL, K0>(x, mpf_from_frexp<K0>(1.0 / sqrt(f), -E / 2));
}
template <int NL>
__device__ __forceinline__ mpf<NL> mpf_sqrt(const mpf<NL>& x) {
  if (mpf_is_zero(x)) return x;
  return mpf_mul(x, mpf_rsqrt(x));
}
template <int NL>
__device__ __forceinline__ mpf<NL> mpf_div(const mpf<NL>& a, const mpf<NL>& b) {
  return mpf_mul(a, mpf_recip(b));
}

// ----------------------------------------------------------------------------
// conversions
// ----------------------------------------------------------------------------
// Interchange record (include/mps_b200.h): int64 exp; u32 sign; u32 res; u32 limb[RL]
// value = (-1)^sign * limbs * 2^(exp - 32 RL).
// records are only 4-byte aligned (16 + 4L bytes): the int64 exponent is read/written as two words
__device__ __forceinline__ int64_t rec_get_exp(const uint32_t* rec) {
  return (int64_t)(((uint64_t)rec[1] << 32) | (uint64_t)rec[0]);
}
__device__ __forceinline__ void rec_set_exp(uint32_t* rec, int64_t e) {
  rec[0] = (uint32_t)(uint64_t)e;
  rec[1] = (uint32_t)((uint64_t)e >> 32);
}

template <int NL>
__device__ __forceinline__ mpf<NL> mpf_from_record(const uint32_t* rec, int RL) {
  int64_t ex = rec_get_exp(rec);
  if (ex == MPF_ZERO) return mpf_zero<NL>();
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i <= NL; ++i) t[i] = 0;
  // place the RL record limbs at the top of t
#pragma unroll
  for (int i = 0; i <= NL; ++i) {
    int src = i - (NL + 1 - RL);
    if (src >= 0 && src < RL) t[i] = rec[4 + src];
  }
  // value = limbs * 2^(ex - 32RL) = t * 2^(ex - 32RL - 32(NL+1-RL)) = t * 2^(ex - 32(NL+1))
  return mpf_pack<NL>(t, ex, rec[2] != 0);
}

// Round a (NL limbs) to p significant bits (round half up) and write a record with RL limbs.
template <int NL>
__device__ __forceinline__ void mpf_to_record(const mpf<NL>& a, uint32_t* rec, int RL, int p) {
  if (mpf_is_zero(a)) {
    rec_set_exp(rec, MPF_ZERO);
    rec[2] = 0; rec[3] = 0;
    for (int i = 0; i < RL; ++i) rec[4 + i] = 0;
    return;
  }
  // keep the top p bits of m (NL*32 bits) : add half at bit (32NL - p - 1)
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i < NL; ++i) t[i] = a.m[i];
  t[NL] = 0;
  int drop = 32 * NL - p;  // >= 32 (one guard limb at least)
  int q = (drop - 1) >> 5, r = (drop - 1) & 31;
  // add 2^(drop-1)
  uint32_t carry = 0;
#pragma unroll
  for (int i = 0; i <= NL; ++i) {
    uint32_t add = (i == q) ? (1u << r) : 0u;
    uint64_t s = (uint64_t)t[i] + add + carry;
    t[i] = (uint32_t)s;
    carry = (uint32_t)(s >> 32);
  }
  int64_t e = a.e;
  if (t[NL]) {  // overflow to 2^(32NL): mantissa becomes 1000..0
#pragma unroll
    for (int i = 0; i < NL; ++i) t[i] = 0;
    t[NL - 1] = 0x80000000u;
    e += 1;
  }
  // clear the dropped bits
  int qd = drop >> 5, rd = drop & 31;
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    if (i < qd) t[i] = 0;
    else if (i == qd && rd) t[i] &= ~((1u << rd) - 1u);
  }
  // record limbs = top RL limbs of t[0..NL-1]; value = t * 2^(e - 32NL) = limbs * 2^(e - 32RL)
  rec_set_exp(rec, e);
  rec[2] = a.neg ? 1u : 0u;
  rec[3] = 0;
  for (int i = 0; i < RL; ++i) rec[4 + i] = t[NL - RL + i];
}

// fixed digits (value = sum d_k 2^(28k) * 2^(E - 28L)) -> mpf.
// Digits may be unnormalised (any int64 column values); cols = number of digit columns.
template <int NL, int NC>
__device__ __forceinline__ mpf<NL> mpf_from_cols(const int64_t (&col)[NC], int64_t E_of_col0) {
  // value = sum_c col[c] 2^(28c) * 2^(E_of_col0).  Resolve carries into a two's-complement
  // integer of 32-bit words, then take sign and magnitude.
  constexpr int NW = (28 * NC + 64) / 32 + 2;
  uint32_t w[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = 0;
  // add each column (sign-extended) at bit offset 28c
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    int64_t v = col[c];
    int bit = 28 * c;
    int q = bit >> 5, r = bit & 31;
    // 96-bit sign-extended shifted value: v << r spread over words q, q+1, q+2
    uint64_t lo = (uint64_t)v << r;
    uint64_t hi = r ? (uint64_t)(v >> (64 - r)) : (uint64_t)(v >> 63);  // arithmetic
    uint32_t parts[3] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi};
    uint32_t ext = (v < 0) ? 0xFFFFFFFFu : 0u;
    uint32_t carry = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      if (i < q) continue;
      uint32_t add = (i - q < 3) ? parts[i - q] : ext;
      uint64_t s = (uint64_t)w[i] + add + carry;
      w[i] = (uint32_t)s;
      carry = (uint32_t)(s >> 32);
    }
  }
  int neg = (w[NW - 1] >> 31) & 1;
  if (neg) {
    uint32_t carry = 1;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint64_t s = (uint64_t)(~w[i]) + carry;
      w[i] = (uint32_t)s;
      carry = (uint32_t)(s >> 32);
    }
  }
  // take the top NL+1 words starting from the highest non-zero word
  int top = -1;
#pragma unroll
  for (int i = NW - 1; i >= 0; --i)
    if (top < 0 && w[i]) top = i;
  if (top < 0) return mpf_zero<NL>();
  // bring word `top` to index NW-1, then take the NL+1 words below it
  words_up<NW>(w, NW - 1 - top);
  uint32_t t[NL + 1];
#pragma unroll
  for (int i = 0; i <= NL; ++i) {
    const int src = NW - 1 - NL + i;
    t[i] = src >= 0 ? w[src] : 0u;
  }
  // value = w * 2^E0 ; t[NL] = w[top] -> value ~= t * 2^(E0 + 32(top - NL))
  //   mpf_pack expects value = t * 2^(E - 32(NL+1))  =>  E = E0 + 32(top - NL) + 32(NL+1)
  return mpf_pack<NL>(t, E_of_col0 + 32 * (int64_t)(top - NL) + 32 * (int64_t)(NL + 1), neg);
}

// mpf -> L fixed digits at column exponent E (value = sum d_k 2^(28k) 2^(E - 28L)),
// rounded to nearest; requires |a| < 2^E (else the top digit is simply large).
template <int NL, int L>
__device__ __forceinline__ void mpf_to_fixed(const mpf<NL>& a, int64_t E, int32_t (&d)[L]) {
#pragma unroll
  for (int k = 0; k < L; ++k) d[k] = 0;
  if (mpf_is_zero(a)) return;
  // integer X = round(m * 2^s), s = a.e - 32NL - E + 28L; digit k = bits [28k + sh, 28k + sh + 28)
  // of m (sh = -s), the rounding bit is bit sh - 1.  Y = m >> (sh - 1) (bits outside m are 0):
  // Y bit 0 = rounding bit, digit k = Y bits [1 + 28k, 29 + 28k).
  const int64_t sh = -(a.e - 32 * (int64_t)NL - E + 28 * (int64_t)L);
  if (sh >= 32 * (int64_t)NL + 1) return;  // rounds to zero
  constexpr int NY = (1 + 28 * L + 31) / 32 + 1;
  constexpr int OFF = NY + 1;
  constexpr int NE = OFF + NL + 1;
  const int64_t s1 = sh - 1;
  const int64_t qw = s1 >> 5;  // floor
  const int r = (int)(s1 & 31);
  int64_t sw = qw + OFF;       // E'[i] = E[i + sw] = m[i + qw]
  uint32_t Ex[NE];
#pragma unroll
  for (int j = 0; j < NE; ++j) Ex[j] = (j >= OFF && j < OFF + NL) ? a.m[j - OFF] : 0u;
  if (sw < 0) sw = NE;         // |a| far above 2^E: outside the contract, digits 0
  words_down<NE>(Ex, (int)(sw > NE ? NE : sw));
  uint32_t Y[NY];
#pragma unroll
  for (int i = 0; i < NY; ++i) Y[i] = __funnelshift_r(Ex[i], Ex[i + 1], r);
  uint32_t carry = Y[0] & 1u;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int bit = 1 + 28 * k, w = bit >> 5, b = bit & 31;
    const uint32_t hi = (w + 1 < NY) ? Y[w + 1] : 0u;
    const uint32_t v = __funnelshift_r(Y[w], hi, b) & 0x0FFFFFFFu;
    const uint32_t sum = v + carry;
    carry = sum >> 28;
    d[k] = (int32_t)(sum & 0x0FFFFFFFu);
  }
  d[L - 1] += (int32_t)(carry << 28);
  // balance digits: d in [0, 2^28) -> [-2^27, 2^27)
  int32_t c = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    int32_t v = d[k] + c;
    c = (v + (1 << 27)) >> 28;
    d[k] = v - (c << 28);
  }
  d[L - 1] += c << 28;
  if (a.neg) {
#pragma unroll
    for (int k = 0; k < L; ++k) d[k] = -d[k];
  }
}

}  // namespace mpsb
