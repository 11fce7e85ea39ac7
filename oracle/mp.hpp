// ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this code.  It shares
// no code with paper_1111_3124_b200/ (the CUDA product path) and never calls it.
//
// Plain multiprecision binary floating point, written from the definitions:
//   * a Real holds exactly p significant bits (MPFR-style precision p, SURVEY §8(c)
//     ledger #9: "280-bit" means exactly 280 significant bits), an int64 exponent
//     and a sign (BASELINE.json north_star: "280–512-bit mantissa, 64-bit exponent");
//   * every operation (+ − × ÷ √) returns the correctly rounded result of the
//     exact operation, round-to-nearest, ties-to-even ("Rounding mode:
//     round-to-nearest-even everywhere");
//   * "fused" sums of several exact products are rounded ONCE (SURVEY §8(c) O1:
//     complex re = RN(ac − bd), im = RN(ad + bc); dots acc ← RN(acc + exact(x·y))).
// Implementation: sign-magnitude, u64 limbs, schoolbook products with
// unsigned __int128, exact aligned integer sums, bit-by-bit restoring division
// and square root.  Nothing is blocked, approximated or reordered.
#pragma once
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using u64 = uint64_t;
using u128 = unsigned __int128;

constexpr int MAXP = 640;                 // largest supported precision in bits
constexpr int RL = (MAXP + 63) / 64;      // limbs of a Real mantissa
constexpr int BIGL = 300;                 // limbs of an exact sum buffer (19200 bits)

// Working precision of the calling thread (bits).  Set by every oracle entry point.
int prec();
void set_prec(int p);

// value = (neg ? -1 : +1) * m * 2^e,  m in [2^(p-1), 2^p) (exactly p bits), or zero.
struct Real {
  bool zero = true;
  bool neg = false;
  int64_t e = 0;
  u64 m[RL] = {0};
};

// An exact (unrounded) value: (neg ? -1 : 1) * d[0..n) * 2^e, arbitrary width <= BIGL/2.
struct Exact {
  bool neg = false;
  int n = 0;            // number of limbs in use (0 => zero)
  int64_t e = 0;
  u64 d[2 * RL + 2];
};

// ---- construction / conversion ----
Real from_int(int64_t v);
Real from_double(double v);               // exact (double has <= 53 bits; p >= 53 assumed)
double to_double(const Real& x);          // nearest-ish double, for diagnostics only
Real neg(const Real& x);
Real absr(const Real& x);
int cmp_abs(const Real& a, const Real& b);
int cmp(const Real& a, const Real& b);    // -1, 0, +1
inline bool is_zero(const Real& x) { return x.zero; }
int sign(const Real& x);                   // -1, 0, +1
Real ldexp_r(const Real& x, int64_t k);   // exact scaling by 2^k

// ---- exact intermediate values ----
Exact exact(const Real& x);
Exact exact_mul(const Real& a, const Real& b);
Exact exact_neg(Exact x);

// Correctly rounded value (RNE, p bits) of the exact sum of k exact terms.
Real round_sum(const Exact* const* t, int k);

// ---- correctly rounded operations ----
Real add(const Real& a, const Real& b);
Real sub(const Real& a, const Real& b);
Real mul(const Real& a, const Real& b);
Real div(const Real& a, const Real& b);
Real sqrt_r(const Real& a);
// RN(a*b + c*d) and friends (one rounding)
Real fsum2(const Exact& a, const Exact& b);
Real fsum3(const Exact& a, const Exact& b, const Exact& c);

// ---- complex (componentwise one rounding from exact products) ----
struct Cplx { Real re, im; };
Cplx cadd(const Cplx& a, const Cplx& b);
Cplx csub(const Cplx& a, const Cplx& b);
Cplx cmul(const Cplx& a, const Cplx& b);          // re=RN(ac-bd), im=RN(ad+bc)
Cplx cconj(const Cplx& a);
Cplx cscale(const Real& s, const Cplx& a);         // componentwise RN(s*x)
Cplx cdivr(const Cplx& a, const Real& s);          // componentwise RN(x/s)
// acc <- RN(acc + exact(x*y)) per component
void cfma(Cplx& acc, const Cplx& x, const Cplx& y);
// acc <- RN(acc + exact(conj(x)*y)) per component
void cfma_conj(Cplx& acc, const Cplx& x, const Cplx& y);
Real cabs2(const Cplx& a);                         // RN(re^2 + im^2)

// ---- interchange records (include/mps_b200.h format, re-implemented here) ----
// record: int64 exp; u32 sign; u32 reserved; u32 limb[L], L = ceil(p/32);
// value = (-1)^sign * (sum limb[k] 2^(32k)) * 2^(exp - 32L); zero: limbs 0, exp = INT64_MIN.
size_t record_bytes(int p);
Real from_record(const unsigned char* rec);        // uses prec(); input must have <= p bits
void to_record(const Real& x, unsigned char* rec); // uses prec()
Cplx cfrom_record(const unsigned char* rec);       // re record then im record
void cto_record(const Cplx& x, unsigned char* rec);


}  // namespace orc
