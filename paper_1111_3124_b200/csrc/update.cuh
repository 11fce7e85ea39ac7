// Generic (per-item dimensions) drivers of the two-site and three-site gate updates.
// Used by the MPS state (mps_apply_gate / mps_apply_layer: a layer of disjoint gates is
// one batched launch per kernel class) and by the configs[1] batch entry.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "precond.cuh"
#include "tcgemm.cuh"
#include "xsweep.cuh"
#include "fo.cuh"

namespace mpsb {

// host construction of an mpf from a double (exact)
template <int NL>
inline mpf<NL> mpf_host_from_double(double v) {
  mpf<NL> r;
  std::memset(&r, 0, sizeof(r));
  if (v == 0.0) { r.e = MPF_ZERO; return r; }
  int k;
  double f = std::frexp(std::fabs(v), &k);
  uint64_t man = (uint64_t)std::ldexp(f, 64);
  r.m[NL - 1] = (uint32_t)(man >> 32);
  r.m[NL - 2] = (uint32_t)man;
  r.e = k;
  r.neg = v < 0;
  return r;
}

// Scratch of one Jacobi problem (M x N, N even) + finalize bookkeeping
template <int L, int NL>
struct SvdScratch {
  int64_t* eA; mpf<NL>* alpha; mpf<NL>* gam; mpf<NL>* inv_sig; mpf<NL>* lam; int32_t* coef;
  int* rot; int* negl; int* ord; int* status; int* sweeps; int* fstatus; int* k; long long* rots;
  int64_t* e_misc;  // 4 spare exponents
  long long* uprod; // executed digit products of phase U per row (profiling)
  int* gexp;        // [2] per-sweep max gamma ratio exponent (precision schedule of phase D)
  int* cexp;        // [6] certified stop of the Jacobi iteration (R21)
  int* sync;
  mpf<NL>* zbuf;
  static size_t bytes(int N) {
    return align_up(8 * (size_t)N + 64) + align_up(sizeof(mpf<NL>) * (size_t)N * 4) +
           align_up(4 * (size_t)N / 2 * 33 * (L + 1)) + align_up(4 * (size_t)N * 3) + 256 + 256;
  }
  static SvdScratch carve(char* p, int N) {
    SvdScratch s;
    s.eA = (int64_t*)p;
    char* q = p + align_up(8 * (size_t)N + 64);
    s.alpha = (mpf<NL>*)q;
    s.gam = s.alpha + N;
    s.inv_sig = s.gam + N;
    s.lam = s.inv_sig + N;
    q += align_up(sizeof(mpf<NL>) * (size_t)N * 4);
    s.coef = (int32_t*)q;
    q += align_up(4 * (size_t)N / 2 * 33 * (L + 1));
    s.rot = (int*)q;
    s.negl = s.rot + N / 2;
    s.ord = s.negl + N;
    q += align_up(4 * (size_t)N * 3);
    s.status = (int*)q;
    s.sweeps = s.status + 1;
    s.fstatus = s.status + 2;
    s.k = s.status + 3;
    s.rots = (long long*)(q + 16);
    s.e_misc = (int64_t*)(q + 32);
    s.sync = (int*)(q + 64);
    s.uprod = (long long*)(q + 72);
    s.gexp = (int*)(q + 80);
    s.cexp = (int*)(q + 96);  // 6 ints, below zbuf
    s.zbuf = (mpf<NL>*)(q + 128);
    return s;
  }
};

inline size_t mat_bytes(int rows, int cols, int L) { return align_up((size_t)rows * cols * 2 * L * 4); }

// MPS_JACOBI_PHASES=1 (debug): per-phase cycle counters of the batched Jacobi, printed to
// stderr after each launch_update2 (D, R, U, norms, init, total; summed over CTAs).
// MPS_ACCUMULATE_V=1 (debug): accumulate V in every SVD instead of recovering it (R16).
inline bool force_accumulate_v() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_ACCUMULATE_V");
    on = e && atoi(e) ? 1 : 0;
  }
  return on != 0;
}

inline unsigned long long* phase_dbg() {
  static unsigned long long* d = nullptr;
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_JACOBI_PHASES");
    on = e && atoi(e) ? 1 : 0;
    if (on) {
      cudaMalloc(&d, (6 + 128 + 64) * sizeof(unsigned long long));
      cudaMemset(d, 0, (6 + 128 + 64) * sizeof(unsigned long long));
    }
  }
  return on ? d : nullptr;
}

// ---------------------------------------------------------------------------- two-site
struct Upd2Args {
  int chiL, chiM, chiR, chi_max;
  const uint32_t *GL, *GR, *lamL, *lamM, *lamR, *U;  // device records (lamL / lamR may be null)
  uint32_t *GL_out, *GR_out, *lam_out, *sigma_out;    // GL_out [2][chiL][ld], GR_out [2][ld][chiR]
  int out_ld;
  int *k_out, *sweeps_out, *status_out;               // device ints (may be null)
  uint32_t* theta_dbg;                                // column-major Theta' records or null
  int accumulate_v;                                   // 1: accumulate V (else recover it, R16)
  int no_precond;                                     // 1: no binary64 preconditioning (R19)
};

// kept-spectrum range (bits) above which a recovered V is replaced by an accumulated one:
// the recovered V_b carries ~2^-W (sigma_1 / sigma_b)^2 (A's column b has absolute error
// ~2^-W sigma_1 after the rotations, divided by sigma_b^2), and its loss of orthonormality
// propagates through later updates (measured: configs[3] amplitudes 2^13 worse than with
// accumulated V for kept ranges < 2^12).  At 280 bits (W = p, no guard digits) the budget is
// small: R = 4 (<= 2^8 amplification); at 512 bits (20 guard bits) R = 16.
template <int L>
constexpr int redo_bits() { return L <= 10 ? 4 : 16; }

// MPS_NO_PRECOND=1 (debug / A-B): run the p-bit Jacobi on Theta' itself (no binary64
// preconditioning, R19).
// MPS_REDUCED_D=1 (experimental, off): the first two sweeps of a preconditioned iteration
// compute the dot products from the top 4 / 7 digits (R20).  +3.5% at chi=128, but it failed
// the 512-bit echo pin (2^-220 instead of 2^-465): the truncated dot is accurate relative to
// the column exponents, not to the norms of columns collapsing inside a sweep.
inline bool use_reduced_d() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_REDUCED_D");
    on = (e && atoi(e)) ? 1 : 0;
  }
  return on != 0;
}
// MPS_NO_CERT=1 (debug): end every Jacobi iteration with the paper's rotation-free sweep
// instead of the certified stop (R21)
inline bool use_cert() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_NO_CERT");
    on = (e && atoi(e)) ? 0 : 1;
  }
  return on != 0;
}
inline bool use_precond() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_NO_PRECOND");
    on = (e && atoi(e)) ? 0 : 1;
  }
  return on != 0;
}
template <int L>
constexpr int ns_iters() { return NsSched<L>::n; }  // Newton-Schulz: 2^-45 -> 2^-360 / 2^-720
// GEMM descriptors per item: 2 per Newton-Schulz iteration, A_1 (X route), P and A_1 (P route),
// A_t = Theta' X and G = A_t^H A_t of the two refinement sweeps (R22), F = E + E E / 2 and
// X + X F of their GEMM form (R26)
template <int L>
constexpr int pre_slots() { return 2 * ns_iters<L>() + 11; }
// the refinement sweep (xsweep.cuh, R22) is on unless MPS_XSWEEP=0
inline bool use_xsweep() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_XSWEEP");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0;
}
constexpr int XS_MIN_N = 16;  // smaller items: no refinement sweep
#ifndef XS2_D
#define XS2_D 7  // digits of the second refinement sweep (6 measured: G resolves gamma to ~2^-156 of alpha only,
               // the sweep then ends at rho ~ 2^-140 and the first-order finish does not apply)
#endif
// the first-order finish (fo.cuh, R23) is on unless MPS_FO=0; it needs the refinement
// sweeps and the tensor-core GEMMs (its Gram matrices are (L+1)-digit products), 280-bit tier
inline bool use_fo() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_FO");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0 && use_xsweep() && tc_enabled();
}
// per-item buffers of the first-order finish: A_1 (M x N), G (N x N, L + 1 digits), flags
template <int L>
inline size_t fo_bytes(int M, int N) {
  return mat_bytes(M, N, L) + align_up((size_t)N * N * 2 * (L + 1) * 4) + 256;
}
// Gram matrix of the first-order finish: (L+1)-digit product of the zero-padded operands,
// upper triangle (tensor cores only; -1 if their scratch cannot be allocated)
template <int L>
inline int run_gram_ext(const GemmT* d, int n, int maxM, int maxN, cudaStream_t st) {
  return launch_gemm_tc<L, L + 1, 0, 1, 1, 0, L + 1>(d, n, maxN, maxN, maxM, st);
}
template <int NL>
static __global__ void k_fo_fail(const FoItem<NL>* items, int n, int L) {
  // the Gram GEMM could not run: E = 0 (A_2 = A_1), every item falls back to k_jacobi
  const FoItem<NL> it = items[blockIdx.y];
  if (it.N == 0) return;
  const size_t nw = (size_t)it.N * it.N * 2 * L;
  for (size_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) it.E[w] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) { *it.ok = 0; *it.done = 0; }
}

// the binary32 first phase of the block Jacobi (R27) is on unless MPS_JD_SP=0
inline bool use_jd_sp() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_JD_SP");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0;
}
constexpr int JD_SP_MIN_N = 32;  // smaller items: binary64 only

// preconditioner buffers of one item: Ad, Vd (binary64), X_a, X_b, D (fixed N x N; for a square
// item the last X buffer also holds P = A0 X_{n-1}), eMix[N], scalars
template <int L>
inline size_t pre_bytes(int M, int N) {
  return align_up(16 * (size_t)M * N) + align_up(16 * (size_t)N * N) + 3 * mat_bytes(N, N, L) + align_up(8 * (size_t)N) +
         256 + align_up(4 * (size_t)N * (L + 1)) + align_up(8 * (size_t)N) +  // + recovery coefficients
         xs_rec_bytes(N) +                                                     // + refinement sweep records
         align_up(16 * (size_t)M * N) + 2 * align_up(16 * (size_t)N * N);      // + Aj (As), V0, Rm (Vs) of R27
}

// preconditioner buffers carved from q (layout of pre_bytes)
template <int L>
struct PreBufs {
  double2 *Ad, *Vd;
  int32_t *Xa, *Xb, *Dm;
  int64_t* eMix;
  unsigned long long* rowmax;
  int* sweeps_d;
  int64_t *eOne, *eA1;
  int* anyflag;
  unsigned long long* offmax;
  int32_t* rcoef;
  int64_t* rexp;
  int64_t* eG;   // exponent of G (refinement sweep)
  int4* xs_rec;  // refinement sweep records
  int64_t* eXs;  // [2] = {0, -1}: exponents of E and E / 2 (GEMM form of the refinement sweeps)
  int* xs_big;   // pairs of the current refinement sweep applied as sequential rotations
  double2 *Aj, *V0, *Rm;  // R27: Theta_d V_d (the binary32 A aliases it), V0, V0^H V0 (the binary32 V aliases it)
  int *sweeps_s, *sp_bad;
  int32_t* Xfin() const { return (ns_iters<L>() % 2) ? Xb : Xa; }
};
template <int L>
inline PreBufs<L> carve_pre(char* q, int M, int N) {
  PreBufs<L> b;
  b.Ad = (double2*)q; q += align_up(16 * (size_t)M * N);
  b.Vd = (double2*)q; q += align_up(16 * (size_t)N * N);
  b.Xa = (int32_t*)q; q += mat_bytes(N, N, L);
  b.Xb = (int32_t*)q; q += mat_bytes(N, N, L);
  b.Dm = (int32_t*)q; q += mat_bytes(N, N, L);
  b.eMix = (int64_t*)q; q += align_up(8 * (size_t)N);
  b.rowmax = (unsigned long long*)q;
  b.sweeps_d = (int*)(q + 8);
  b.eOne = (int64_t*)(q + 16);
  b.eA1 = (int64_t*)(q + 32);
  b.anyflag = (int*)(q + 40);
  b.offmax = (unsigned long long*)(q + 64);
  b.rcoef = (int32_t*)(q + 256);
  b.rexp = (int64_t*)((char*)b.rcoef + align_up(4 * (size_t)N * (L + 1)));
  b.eG = (int64_t*)(q + 96);
  b.eXs = (int64_t*)(q + 112);
  b.xs_big = (int*)(q + 128);
  b.xs_rec = (int4*)((char*)b.rexp + align_up(8 * (size_t)N));
  b.Aj = (double2*)((char*)b.xs_rec + xs_rec_bytes(N));
  b.V0 = (double2*)((char*)b.Aj + align_up(16 * (size_t)M * N));
  b.Rm = (double2*)((char*)b.V0 + align_up(16 * (size_t)N * N));
  b.sweeps_s = (int*)(q + 136);
  b.sp_bad = (int*)(q + 140);
  return b;
}
// descriptors of one item's preconditioner (gt[k * stride], k = 0 .. 2 ns_iters): the
// input A0 (M x N, block exponent eA0) -> Af = A0 X with column exponents eAcols.
// p_route (V is recovered, so X itself is not needed): the last Newton-Schulz update is
// folded into A_1 = P + P D/2 with P = A0 X_{n-1} (X_{n-1} has nz zero low digits, so P costs
// fewer digit products than A0 X_n, and the N x N update of X disappears)
template <int L>
inline void pre_descs(const PreBufs<L>& pb, int M, int N, const int32_t* A0, const int64_t* eA0, int32_t* Af,
                      int64_t* eAcols, int* zerr, PreItem* pi, GemmT* gt, size_t stride, bool p_route = false) {
  constexpr int NSIT = ns_iters<L>();
  *pi = PreItem{M, N, A0, eA0, pb.Ad, pb.Vd, pb.rowmax, pb.sweeps_d, pb.Xa, pb.eOne, pb.eA1, pb.anyflag, pb.offmax,
                nullptr, nullptr, nullptr, nullptr, prof_counts()};
  if (use_jd_sp() && N >= JD_SP_MIN_N) {  // a per-item choice
    pi->As = (float2*)pb.Aj; pi->Vs = (float2*)pb.Rm; pi->V0 = pb.V0; pi->Rm = pb.Rm; pi->Aj = pb.Aj;
  }
  pi->sweeps_s = pb.sweeps_s;
  pi->sp_bad = pb.sp_bad;
  for (int k = 0; k < NSIT; ++k) {
    int32_t* Xc = (k % 2) ? pb.Xb : pb.Xa;
    int32_t* Xn = (k % 2) ? pb.Xa : pb.Xb;
    // D = I - X^H X (exponent 1, Hermitian);  X' = X + X (D/2)  (D read at exponent 0 = D/2)
    GemmT gd = GemmT{Xc, N, pb.eOne, Xc, N, pb.eOne, pb.Dm, N, pb.eOne, nullptr, nullptr, N, N, N, 1, 1, 1, zerr};
    gd.herm = 1;
    gt[(2 * k) * stride] = gd;
    gt[(2 * k + 1) * stride] =
        GemmT{Xc, N, pb.eOne, pb.Dm, N, pb.eOne + 1, Xn, N, pb.eOne, Xc, nullptr, N, N, N, 0, 0, 0, zerr};
  }
  // A_1 = A0 X at the exponent bounded by A0's largest row norm
  gt[(2 * NSIT) * stride] = GemmT{A0, M, eA0, pb.Xfin(), N, pb.eOne, Af, M, pb.eA1, nullptr, eAcols, M, N, N, 0, 0, 0, nullptr};
  const GemmT none{nullptr, 1, pb.eOne, nullptr, 1, pb.eOne, nullptr, 1, pb.eOne, nullptr, nullptr, 0, 0, 0, 0, 0, 0, nullptr};
  gt[(2 * NSIT + 1) * stride] = none;
  gt[(2 * NSIT + 2) * stride] = none;
  if (p_route && M == N) {  // a per-item choice (results must not depend on how items are batched);
                            // square items only: P lives in the N x N buffer of X_n
    constexpr int k = NSIT - 1;
    int32_t* Xc = (k % 2) ? pb.Xb : pb.Xa;
    int32_t* P = (k % 2) ? pb.Xa : pb.Xb;  // M x N, in place of X_n
    gt[(2 * k + 1) * stride] = none;
    gt[(2 * NSIT) * stride] = none;
    gt[(2 * NSIT + 1) * stride] = GemmT{A0, M, eA0, Xc, N, pb.eOne, P, M, pb.eA1, nullptr, nullptr, M, N, N, 0, 0, 0, nullptr};
    gt[(2 * NSIT + 2) * stride] = GemmT{P, M, pb.eA1, pb.Dm, N, pb.eOne + 1, Af, M, pb.eA1, P, eAcols, M, N, N, 0, 0, 0, zerr};
  }
  // refinement sweeps (R22): at 4 digits between Newton-Schulz iterations 0 and 1 on X_1 (the
  // output of iteration 0, in Xn = Xb), at 7 digits between iterations 1 and 2 on X_2 (in Xa):
  // A_t = Theta' X into Af at A_1's exponent, G = A_t^H A_t into D's buffer (free between the
  // iterations); each sweep rotates its X in place
  for (int k = 3; k < 11; ++k) gt[(2 * NSIT + k) * stride] = none;
  if (use_xsweep() && N >= XS_MIN_N) {
    int32_t* X1 = pb.Xb;
    int gh = 1;
    while ((1 << (gh - 1)) < M) ++gh;
    for (int w = 0; w < 2; ++w) {
      gt[(2 * NSIT + 3 + 2 * w) * stride] =
          GemmT{A0, M, eA0, w ? pb.Xa : X1, N, pb.eOne, Af, M, pb.eA1, nullptr, nullptr, M, N, N, 0, 0, 0, nullptr};
      GemmT g{Af, M, pb.eA1, Af, M, pb.eA1, pb.Dm, N, nullptr, nullptr, nullptr, N, N, M, 1, 0, 0, nullptr};
      g.ghead = gh + 1;  // sum of M products, each |.| < 2^(2 eA1 - 2)
      g.eCwrite = pb.eG;
      g.upper = 1;  // k_xs_params reads the diagonal and G(p, q), p < q
      gt[(2 * NSIT + 4 + 2 * w) * stride] = g;
      // GEMM form (R26): E in the X buffer the sweep does not rotate (exponent 0),
      // F = E + E (E / 2) into Af (A_t is dead once G is formed), X + X F into G's buffer
      int32_t* Xr = w ? pb.Xa : X1;
      int32_t* E = w ? X1 : pb.Xa;
      gt[(2 * NSIT + 7 + 2 * w) * stride] = GemmT{E, N, pb.eXs, E, N, pb.eXs + 1, Af, N, pb.eXs, E, nullptr, N, N, N, 0, 0, 0, nullptr};
      gt[(2 * NSIT + 8 + 2 * w) * stride] = GemmT{Xr, N, pb.eOne, Af, N, pb.eXs, pb.Dm, N, pb.eOne, Xr, nullptr, N, N, N, 0, 0, 0, nullptr};
    }
    pi->eXs = pb.eXs;
    pi->xs_big = pb.xs_big;
    pi->X1 = X1;
    pi->G = pb.Dm;
    pi->eG = pb.eG;
    pi->xs_rec = pb.xs_rec;
  }
}
template <int L>
inline void pre_skip_descs(const PreBufs<L>& pb, PreItem* pi, GemmT* gt, size_t stride) {
  *pi = PreItem{0, 0, nullptr, nullptr, nullptr, nullptr, pb.rowmax, pb.sweeps_d, nullptr, pb.eOne, pb.eA1, pb.anyflag, pb.offmax,
                nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < pre_slots<L>(); ++k)
    gt[k * stride] = GemmT{nullptr, 1, pb.eOne, nullptr, 1, pb.eOne, nullptr, 1, pb.eOne, nullptr, nullptr, 0, 0, 0, 0, 0, 0, nullptr};
}
// One GemmT launch over n items: the tensor-core path (tcgemm.cuh; LG <= TC_MAX_LG digits: with
// the staged pipeline any slice count fits, at 19 digits a slice-weight group sums <= 68 pairs x
// K <= 512 products < 2^14, below 2^30) unless MPS_TC=0, else (or when its scratch cannot be
// allocated) the IMAD.WIDE kernel.  Launch count.
#ifndef TC_MAX_LG
#define TC_MAX_LG 19
#endif
template <int L, int LG, int Z, int NZA = 0, int NZB = 0, int ZOUT = 0>
inline int run_gemm(const GemmT* d, int n, int maxR, int maxC, int maxK, dim3 grid, cudaStream_t st) {
  if constexpr (LG <= TC_MAX_LG) {
    if (tc_enabled() && maxR > 0 && maxC > 0 && maxK > 0) {
      const int nl = launch_gemm_tc<L, LG, Z, NZA, NZB, ZOUT>(d, n, maxR, maxC, maxK, st);
      if (nl >= 0) return nl;
    }
  }
  k_gemm_t<L, LG, Z, NZA, NZB, ZOUT><<<grid, 256, 0, st>>>(d);
  return 1;
}

// Newton-Schulz iteration K (precond.cuh NsSched): D_k = I - X_k^H X_k, X_{k+1} = X_k + X_k D_k / 2.
// On the tensor cores D_k is formed in full (no mirrored half: its two triangles are exact
// conjugates before the identical rounding).  Launch count.
template <int L, int K>
inline int run_ns_iter(const GemmT* dD, const GemmT* dX, int n, int maxN, dim3 grid, cudaStream_t st) {
  constexpr int LG = NsSched<L>::lg[K], Z = NsSched<L>::z[K], NZ = NsSched<L>::nz[K];
  return run_gemm<L, LG, 0, NZ, NZ, Z>(dD, n, maxN, maxN, maxN, grid, st) +
         run_gemm<L, LG, Z, NZ, 0>(dX, n, maxN, maxN, maxN, grid, st);
}

// One refinement sweep at XD digits from G (R22): sequential row rotations, or (R26, default) E,
// F = E + E E / 2, X + X F as two GEMMs (dF: their descriptors, n apart), the copy back, and the
// sequential rotations of the few pairs left out of E.  Launch count.
template <int L, int XD>
inline int run_xsweep(const PreItem* dpre, const GemmT* dF, int n, int maxN, int sel, dim3 gNN, cudaStream_t st) {
  int nl = 0;
  if (!xs_gemm_form()) {
    prof_mark(PROF_XS, 1, st);
    nl += launch_xsweep<L, XD>(dpre, n, maxN, sel, st);
    prof_mark(PROF_XS, 0, st);
    return nl;
  }
  constexpr int ZE = XsT<XD>::ZE;
  prof_mark(PROF_XS, 1, st);
  nl += launch_xs_emat<L, XD>(dpre, n, maxN, sel, st);
  prof_mark(PROF_XS, 0, st);
  nl += run_gemm<L, XD, ZE>(dF, n, maxN, maxN, maxN, gNN, st);
  nl += run_gemm<L, XD, ZE>(dF + (size_t)n, n, maxN, maxN, maxN, gNN, st);
  prof_mark(PROF_XS, 1, st);
  k_xs_copy<L><<<dim3(32, n), 256, 0, st>>>(dpre, sel); ++nl;
  nl += launch_xs_apply<L, XD>(dpre, n, maxN, sel, st);
  prof_mark(PROF_XS, 0, st);
  return nl;
}

// the preconditioner kernels for n items (descriptors already on the device); launch count
template <int L>
inline int launch_pre(const PreItem* dpre, const GemmT* dgt, int n, int maxM, int maxN, cudaStream_t st) {
  constexpr int NSIT = ns_iters<L>();
  int nl = 0;
  jacobi_trace_init();
  k_pre_init<<<(n + 255) / 256, 256, 0, st>>>(dpre, n); ++nl;
  k_fx_to_d<L><<<dim3(std::max(1, (maxM + 255) / 256), n), 256, 0, st>>>(dpre); ++nl;
  {
    // few items (an MPS layer): C CTAs per item share its block pairs (cluster barriers per step)
    // shared memory for the largest staging of any item: the block size depends on M, and
    // jd_smem is not monotone in M (bs halves above M = 320 and M = 640)
    auto smem_for = [&](size_t el) {
      return std::max(std::max(jd_smem(std::min(maxM, 320), el), jd_smem(std::min(maxM, 640), el)), jd_smem(maxM, el));
    };
    static int jprof = -1;
    if (jprof < 0) {
      const char* e = getenv("MPS_JD_PROF");
      jprof = e && atoi(e) ? 1 : 0;
      if (jprof) {
        const int one = 1;
        cudaMemcpyToSymbol(jd_prof_on, &one, sizeof(int));
      }
    }
    int C = 1;
    const int bpairs = ((maxN + jd_bs(maxM) - 1) / jd_bs(maxM) + 1) / 2;
    while (C < 8 && n * C * 2 <= 148 && C * 2 <= bpairs) C *= 2;
    auto run_phase = [&](auto kernel, size_t smem, const char* name) {
      smem_optin((const void*)kernel, (int)smem);
      if (jprof) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbolAsync(jd_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
      }
      if (C == 1) {
        kernel<<<n, JD_THREADS, smem, st>>>(dpre, 1);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n * C, 1, 1);
        cfg.blockDim = dim3(JD_THREADS, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kernel, dpre, C);
      }
      ++nl;
      if (jprof) {
        unsigned long long h[8];
        cudaMemcpyFromSymbolAsync(h, jd_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "%s cycles (thread 0, sum over CTAs): stage %.4e gram %.4e inner %.4e write %.4e vupd %.4e  block pairs %llu (Gram form %llu) sweeps %llu (items %d)\n",
                name, (double)h[0], (double)h[7], (double)h[1], (double)h[2], (double)h[3], h[4], h[6], h[5], n);
      }
    };
    static int spcap = -2;
    if (spcap == -2) {
      const char* e = getenv("MPS_JD_SP_SWEEPS");
      spcap = e ? atoi(e) : -1;
      if (spcap >= 0) cudaMemcpyToSymbol(jd_sp_maxsweeps, &spcap, sizeof(int));
    }
    if (use_jd_sp() && maxN >= JD_SP_MIN_N) {  // binary32 first phase and the hand-over (R27); items
                                               // without it (As == nullptr) exit at once
      prof_mark(PROF_JSP, 1, st);
      k_d_to_s<<<dim3(32, n), 256, 0, st>>>(dpre); ++nl;
      run_phase(k_jacobi_blk<float>, smem_for(8), "k_jacobi_blk<float>");
      k_sp_to_dp<<<dim3(32, n), 256, 0, st>>>(dpre); ++nl;
      const dim3 gN((maxN + 63) / 64, (maxN + 63) / 64, n), gM((maxM + 63) / 64, (maxN + 63) / 64, n);
      for (int nsstep = 0; nsstep < 2; ++nsstep) {
        k_zgemm_handover<<<gN, 256, 0, st>>>(dpre, 0, nsstep); ++nl;
        k_zgemm_handover<<<gN, 256, 0, st>>>(dpre, 1, nsstep); ++nl;
      }
      k_zgemm_handover<<<gM, 256, 0, st>>>(dpre, 2, 0); ++nl;
      prof_mark(PROF_JSP, 0, st);
    }
    static const bool dbgpair = getenv("MPS_JACOBI_TRACE") && atoi(getenv("MPS_JACOBI_TRACE")) > 2000;
    if (dbgpair) k_dbg_pair<<<1, 512, 0, st>>>(dpre, 0);
    prof_mark(PROF_JDB, 1, st);
    run_phase(k_jacobi_blk<double>, smem_for(16), "k_jacobi_blk<double>");
    prof_mark(PROF_JDB, 0, st);
    if (dbgpair) k_dbg_pair<<<1, 512, 0, st>>>(dpre, 1);
  }
  k_d_to_fx<L><<<dim3(std::max(1, std::min(64, (maxN * maxN + 255) / 256)), n), 256, 0, st>>>(dpre); ++nl;
  const int tNN = ((maxN + GT_TILE - 1) / GT_TILE) * ((maxN + GT_TILE - 1) / GT_TILE);
  const int tMN = ((maxM + GT_TILE - 1) / GT_TILE) * ((maxN + GT_TILE - 1) / GT_TILE);
  const dim3 gNN(std::min(tNN, 1024), n);
  const dim3 gMN(std::min(tMN, 1024), n);
  constexpr int KL = NSIT - 1;  // last iteration: lg = L
  static_assert(NsSched<L>::lg[KL] == L, "the last Newton-Schulz iteration is at full precision");
  nl += run_ns_iter<L, 0>(dgt, dgt + (size_t)n, n, maxN, gNN, st);
  const bool xs = use_xsweep() && maxN >= XS_MIN_N;  // refinement sweeps (R22); items without them
                                                       // have empty descriptors
  if (xs) {
    nl += run_gemm<L, 4, 0>(dgt + (size_t)(2 * NSIT + 3) * n, n, maxM, maxN, maxN, gMN, st);
    nl += run_gemm<L, 4, 0>(dgt + (size_t)(2 * NSIT + 4) * n, n, maxN, maxN, maxM, gNN, st);
    nl += run_xsweep<L, 4>(dpre, dgt + (size_t)(2 * NSIT + 7) * n, n, maxN, 0, gNN, st);
  }
  nl += run_ns_iter<L, 1>(dgt + (size_t)2 * n, dgt + (size_t)3 * n, n, maxN, gNN, st);
  if (xs) {
    // X_2 holds 7 digits; the sweep works on its top XS2_D (its 7th is dropped: X_2 then stays
    // unitary to 2^-168, which the last Newton-Schulz iteration squares away)
    static_assert(NsSched<L>::lg[1] == 7 && XS2_D <= 7, "X_2 holds 7 digits");
    nl += run_gemm<L, XS2_D, 0>(dgt + (size_t)(2 * NSIT + 5) * n, n, maxM, maxN, maxN, gMN, st);
    nl += run_gemm<L, XS2_D, 0>(dgt + (size_t)(2 * NSIT + 6) * n, n, maxN, maxN, maxM, gNN, st);
    nl += run_xsweep<L, XS2_D>(dpre, dgt + (size_t)(2 * NSIT + 9) * n, n, maxN, 1, gNN, st);
  }
  if constexpr (NSIT > 3) nl += run_ns_iter<L, 2>(dgt + (size_t)4 * n, dgt + (size_t)5 * n, n, maxN, gNN, st);
  const GemmT* dD = dgt + (size_t)(2 * KL) * n;
  const GemmT* dX = dgt + (size_t)(2 * KL + 1) * n;
  const GemmT* dA1 = dgt + (size_t)(2 * NSIT) * n;
  // X route: X_n = X_{n-1} + X_{n-1} D / 2, A_1 = A0 X_n; P route (items whose V is recovered):
  // P = A0 X_{n-1} (its nz zero low digits skipped), A_1 = P + P D / 2.  Items without a route
  // have empty descriptors in the other route's launches.
  nl += run_ns_iter<L, KL>(dD, dX, n, maxN, gNN, st);
  nl += run_gemm<L, L, 0>(dA1, n, maxM, maxN, maxN, gMN, st);
  {
    constexpr int Z = NsSched<L>::z[KL], NZ = NsSched<L>::nz[KL];
    nl += run_gemm<L, L, 0, 0, NZ>(dA1 + (size_t)n, n, maxM, maxN, maxN, gMN, st);
    nl += run_gemm<L, L, Z>(dA1 + (size_t)2 * n, n, maxM, maxN, maxN, gMN, st);
  }
  return nl;
}

template <int L, int NL>
inline size_t upd2_item_bytes(const Upd2Args& a) {
  const int M = 2 * std::max(a.chiL, a.chiR), N = 2 * std::min(a.chiL, a.chiR);
  size_t lr = mat_bytes(2 * a.chiL, a.chiM, L) + mat_bytes(a.chiM, 2 * a.chiR, L);
  size_t r1 = std::max(lr, mat_bytes(M, N, L));
  return r1 + mat_bytes(2 * a.chiL, 2 * a.chiR, L) + mat_bytes(N, N, L) + mat_bytes(M, N, L) +
         SvdScratch<L, NL>::bytes(N) + 8 * (size_t)N + 512 + pre_bytes<L>(M, N) + 256 + fo_bytes<L>(M, N);
}

// descriptor region of launch_update2 (the redo flags follow it)
template <int L, int NL>
inline size_t upd2_desc_bytes(int n) {
  return align_up(sizeof(PrepItem) * 2 * n) + align_up(sizeof(GemmItem) * n) + align_up(sizeof(MixItem) * n) +
         align_up(sizeof(SvdItem<NL>) * n) + align_up(sizeof(FinItem<NL>) * n) + align_up(sizeof(PreItem) * n) +
         align_up(sizeof(GemmT) * pre_slots<L>() * n) + align_up(sizeof(RecItem<NL>) * n) +
         align_up(sizeof(GemmT) * n) + align_up(sizeof(GemmT) * n) + align_up(sizeof(FoItem<NL>) * n) +
         align_up(sizeof(GemmT) * 3 * n);
}

template <class T>
size_t upd2_workspace(const Upd2Args* a, int n) {
  constexpr int L = T::L, NL = T::NL;
  size_t s = upd2_desc_bytes<L, NL>(n) + align_up(4 * (size_t)n) + 4096;
  for (int i = 0; i < n; ++i) s += align_up(upd2_item_bytes<L, NL>(a[i]));
  return s;
}

// Launch the update of n independent items (one batched launch per kernel class).
template <class T>
int launch_update2(int p, double thr, const Upd2Args* a, int n, void* ws, cudaStream_t st,
                   std::vector<unsigned char>& hd) {
  constexpr int L = T::L, NL = T::NL;
  const int RBr = record_words(p);
  const size_t cplx = 2 * (size_t)RBr;
  char* base = (char*)ws;
  const size_t d_prep = 0, d_gemm = align_up(sizeof(PrepItem) * 2 * n),
               d_mix = d_gemm + align_up(sizeof(GemmItem) * n), d_svd = d_mix + align_up(sizeof(MixItem) * n),
               d_fin = d_svd + align_up(sizeof(SvdItem<NL>) * n), d_pre = d_fin + align_up(sizeof(FinItem<NL>) * n),
               d_gt = d_pre + align_up(sizeof(PreItem) * n),
               d_rec = d_gt + align_up(sizeof(GemmT) * pre_slots<L>() * n),
               d_rg = d_rec + align_up(sizeof(RecItem<NL>) * n), d_gc = d_rg + align_up(sizeof(GemmT) * n),
               d_fo = d_gc + align_up(sizeof(GemmT) * n), d_fogt = d_fo + align_up(sizeof(FoItem<NL>) * n),
               d_end = upd2_desc_bytes<L, NL>(n);
  constexpr int NSIT = ns_iters<L>();
  const bool pre = use_precond();
  int* redo = (int*)(base + d_end);  // [n] flags (run_update2)
  hd.assign(d_end, 0);
  PreItem* hpre = (PreItem*)(hd.data() + d_pre);
  GemmT* hgt = (GemmT*)(hd.data() + d_gt);  // [2 NSIT + 1][n]: D_k, X_k+1 per iteration, then A_1
  RecItem<NL>* hrec = (RecItem<NL>*)(hd.data() + d_rec);
  GemmT* hrg = (GemmT*)(hd.data() + d_rg);  // V = Theta'^H A_final diag(1/alpha) (tiled GEMM)
  GemmT* hgc = (GemmT*)(hd.data() + d_gc);  // a1 contraction Theta = L R (tiled GEMM)
  FoItem<NL>* hfo = (FoItem<NL>*)(hd.data() + d_fo);  // first-order finish (R23)
  GemmT* hfg = (GemmT*)(hd.data() + d_fogt);          // [3][n]: G_1, A_2 = A_1 (I + E), G_2
  int n_fo = 0;
  PrepItem* hp = (PrepItem*)(hd.data() + d_prep);
  GemmItem* hg = (GemmItem*)(hd.data() + d_gemm);
  MixItem* hm = (MixItem*)(hd.data() + d_mix);
  SvdItem<NL>* hs = (SvdItem<NL>*)(hd.data() + d_svd);
  FinItem<NL>* hf = (FinItem<NL>*)(hd.data() + d_fin);
  const mpf<NL> thr_m = mpf_host_from_double<NL>(thr);
  char* items = base + d_end + align_up(4 * (size_t)n);
  int maxMN = 0, maxLR = 0, maxOut = 0;
  bool any_dbg = false;
  std::vector<int64_t*> einit;
  size_t off = 0;
  for (int b = 0; b < n; ++b) {
    const Upd2Args& g = a[b];
    const int chiL = g.chiL, chiM = g.chiM, chiR = g.chiR;
    const bool trans = chiR > chiL;
    const int M = 2 * std::max(chiL, chiR), N = 2 * std::min(chiL, chiR);
    char* ib = items + off;
    off += align_up(upd2_item_bytes<L, NL>(g));
    int32_t* Lf = (int32_t*)ib;
    int32_t* Rf = (int32_t*)(ib + mat_bytes(2 * chiL, chiM, L));
    int32_t* Af = (int32_t*)ib;
    size_t lr = mat_bytes(2 * chiL, chiM, L) + mat_bytes(chiM, 2 * chiR, L);
    char* p2 = ib + std::max(lr, mat_bytes(M, N, L));
    int32_t* Tf = (int32_t*)p2;
    int32_t* Vf = (int32_t*)(p2 + mat_bytes(2 * chiL, 2 * chiR, L));
    int32_t* A0f = (int32_t*)((char*)Vf + mat_bytes(N, N, L));
    char* sp = (char*)A0f + mat_bytes(M, N, L);
    auto S = SvdScratch<L, NL>::carve(sp, N);
    int64_t* eV = (int64_t*)align_up((size_t)sp + SvdScratch<L, NL>::bytes(N), 16);
    const PreBufs<L> PB = carve_pre<L>((char*)align_up((size_t)eV + 8 * (size_t)N, 256), M, N);
    int64_t* eMix = PB.eMix;
    int32_t* Xfin = PB.Xfin();
    int32_t* rcoef = PB.rcoef;
    int64_t* rexp = PB.rexp;
    const bool pb = pre && !g.no_precond;
    // first-order finish (R23): 280-bit tier, preconditioned with refinement sweeps, V recovered
    const bool fo = L == 10 && pb && use_fo() && N >= XS_MIN_N && !force_accumulate_v() && !g.accumulate_v;
    char* fob = (char*)PB.xs_rec + xs_rec_bytes(N);
    fob = (char*)align_up((size_t)fob, 256);
    int32_t* A1x = (int32_t*)fob;
    int32_t* Gx = (int32_t*)(fob + mat_bytes(M, N, L));
    int* foflags = (int*)(fob + mat_bytes(M, N, L) + align_up((size_t)N * N * 2 * (L + 1) * 4));  // ok, done
    int64_t* eGx = (int64_t*)(foflags + 4);
    int64_t* eL = S.e_misc;
    int64_t* eR = S.e_misc + 1;
    int64_t* eT = S.e_misc + 2;
    einit.push_back(eL);
    einit.push_back(eR);
    hp[2 * b] = PrepItem{g.GL, g.lamL, g.lamM, chiL, chiM, 0, Lf, eL};
    hp[2 * b + 1] = PrepItem{g.GR, nullptr, g.lamR, chiM, chiR, 1, Rf, eR};
    hg[b] = GemmItem{Lf, 2 * chiL, eL, Rf, chiM, eR, Tf, 2 * chiL, eT, 2 * chiL, 2 * chiR, chiM, 0};
    {
      GemmT gc = GemmT{Lf, 2 * chiL, eL, Rf, chiM, eR, Tf, 2 * chiL, nullptr, nullptr, nullptr, 2 * chiL, 2 * chiR, chiM,
                       0, 0, 0, nullptr};
      int gh = 1;
      while ((1 << (gh - 1)) < chiM) ++gh;
      gc.ghead = gh + 1;  // as k_gemm: sum of chiM complex products, each |.| < 2^(eA + eB + 1)
      gc.eCwrite = eT;
      hgc[b] = gc;
    }
    hm[b] = MixItem{Tf, 2 * chiL, eT, g.U, 2, chiL, chiR, trans ? 1 : 0, pb ? A0f : Af, pb ? eMix : S.eA, M, N};
    if (pre && !pb) pre_skip_descs<L>(PB, hpre + b, hgt + b, n);  // this item skips the preconditioner
    if (pb)  // V recovered: the last X update is folded into A_1 (P route); R23 items: A_1 into A1x
      pre_descs<L>(PB, M, N, A0f, eMix, fo ? A1x : Af, fo ? nullptr : S.eA, redo + b, hpre + b, hgt + b, n,
                   !force_accumulate_v() && !g.accumulate_v);
    {
      const GemmT none{nullptr, 1, PB.eOne, nullptr, 1, PB.eOne, nullptr, 1, PB.eOne, nullptr, nullptr, 0, 0, 0, 0, 0, 0, nullptr};
      FoItem<NL> fi{};
      hfg[b] = hfg[n + b] = hfg[2 * n + b] = none;
      if (fo) {
        int gh = 1;
        while ((1 << (gh - 1)) < M) ++gh;
        for (int w = 0; w < 2; ++w) {  // G_1 = A_1^H A_1, G_2 = A_2^H A_2 (upper triangle)
          GemmT gg{w ? Af : A1x, M, PB.eA1, w ? Af : A1x, M, PB.eA1, Gx, N, nullptr, nullptr, nullptr, N, N, M, 1, 0, 0, nullptr};
          gg.ghead = gh + 1;
          gg.eCwrite = eGx;
          gg.upper = 1;
          hfg[(2 * w) * n + b] = gg;
        }
        // A_2 = A_1 + A_1 E (E: the X buffer the preconditioner no longer needs, exponent 1)
        int32_t* E = PB.Xfin() == PB.Xa ? PB.Xb : PB.Xa;
        hfg[n + b] = GemmT{A1x, M, PB.eA1, E, N, PB.eOne, Af, M, PB.eA1, A1x, S.eA, M, N, N, 0, 0, 0, nullptr};
        fi.M = M; fi.N = N; fi.G = Gx; fi.eG = eGx; fi.E = E; fi.ok = foflags; fi.done = foflags + 1;
        fi.alpha = S.alpha; fi.negl = S.negl; fi.status = S.status;
        fi.sweeps = g.sweeps_out ? g.sweeps_out : S.sweeps; fi.rots = S.rots; fi.evals = S.rots + 1;
        fi.uprod = S.uprod; fi.cexp = use_cert() ? S.cexp : nullptr;
        ++n_fo;
      }
      hfo[b] = fi;
    }
    SvdItem<NL> si = {};
    si.M = M; si.N = N; si.A = Af; si.eA = S.eA; si.V = Vf; si.alpha = S.alpha; si.gam = S.gam; si.coef = S.coef;
    si.dbg = nullptr; si.rot = S.rot; si.negl = S.negl; si.status = S.status;
    si.sweeps = g.sweeps_out ? g.sweeps_out : S.sweeps; si.rotations = S.rots;
    si.sync = S.sync; si.zbuf = S.zbuf; si.phase_cycles = phase_dbg();
    const bool recover = !force_accumulate_v() && !g.accumulate_v;
    si.uprod = S.uprod;
    si.gexp = use_reduced_d() ? S.gexp : nullptr;
    si.cexp = use_cert() ? S.cexp : nullptr;
    si.e2_hint = pb ? -44 : 0;  // binary64 basis: |gamma|^2 / (alpha_p alpha_q) ~ 2^-44 at sweep 1 (1e-13)
    si.A0 = recover ? A0f : nullptr; si.eA0 = pb ? eMix : S.e_misc + 3; si.eV = eV; si.evals = S.rots + 1;
    si.a0_ready = pb ? 1 : 0;
    si.done = fo ? foflags + 1 : nullptr;
    if (pb && !recover) { si.V = Xfin; si.v_preset = 1; }  // V = X W
    {
      int gh = 1;
      while ((1 << (gh - 1)) < M) ++gh;
      gh += 1;  // sum of M complex products, each |.| < 2^(e0 + e_b + 1)
      hrec[b] = RecItem<NL>{recover ? N : 0, S.alpha, rcoef, rexp};
      hrg[b] = recover ? GemmT{A0f, M, si.eA0, Af, M, nullptr, Vf, N, nullptr, nullptr, eV, N, N, M, 1, 0, 0, nullptr,
                               S.eA, rcoef, rexp, gh, 0, nullptr, S.ord, g.k_out ? g.k_out : S.k}
                       : GemmT{nullptr, 1, nullptr, nullptr, 1, nullptr, nullptr, 1, nullptr, nullptr, nullptr, 0, 0, 0,
                               0, 0, 0, nullptr, nullptr, nullptr, nullptr, 0};
    }
    hs[b] = si;
    FinItem<NL> fi;
    std::memset(&fi, 0, sizeof(fi));
    fi.M = M; fi.N = N; fi.trans = trans ? 1 : 0; fi.A = Af; fi.eA = S.eA; fi.V = si.V; fi.alpha = S.alpha;
    fi.chi_max = g.chi_max; fi.thr = thr_m; fi.ord = S.ord; fi.inv_sig = S.inv_sig; fi.lam = S.lam;
    fi.k_out = g.k_out ? g.k_out : S.k; fi.status = g.status_out ? g.status_out : S.fstatus;
    fi.svd_status = S.status;
    fi.eV = recover ? eV : nullptr;
    fi.redo = recover ? redo + b : nullptr; fi.redo_bits = redo_bits<L>();
    fi.sigma_rec = g.sigma_out; fi.nsig = N; fi.lam_rec = g.lam_out;
    fi.GL = g.GL_out; fi.GL_ld = g.out_ld; fi.lamL = g.lamL; fi.chiL_out = chiL;
    fi.GR = g.GR_out; fi.GR_ld = g.out_ld; fi.lamR = g.lamR; fi.chiR_out = chiR;
    hf[b] = fi;
    maxMN = std::max(maxMN, M * N);
    maxLR = std::max(maxLR, 2 * std::max(chiL, chiR) * chiM);
    maxOut = std::max(maxOut, 2 * std::max(chiL, chiR) * std::min(g.chi_max, N));
    any_dbg |= g.theta_dbg != nullptr;
  }
  cudaMemcpyAsync(base, hd.data(), d_end, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(redo, 0, 4 * (size_t)n, st);
  int nl = 0;
  prof_mark(PROF_CONTRACT, 1, st);
  k_init_prep<<<(2 * n + 255) / 256, 256, 0, st>>>((const PrepItem*)(base + d_prep), 2 * n); ++nl;
  dim3 gp(std::max(1, std::min(64, (maxLR + 255) / 256)), 2 * n);
  k_prep_exp<<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep), RBr); ++nl;
  k_prep_conv<L, NL><<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep), RBr); ++nl;
  dim3 gg(std::max(1, std::min(128, (maxMN + 127) / 128)), n);
  // a1 contraction: the thread-per-element k_gemm measured 10% faster than the tiled
  // k_gemm_t at K = chi (92.7 vs 102.5 ms for 296 chi=128 items; with the three-product
  // k_gemm_t still 1.5% slower per bench step, v26); hgc stays as the tiled form
  if (L <= TC_MAX_LG && tc_enabled()) {  // on the tensor cores (tcgemm.cuh), as the GemmT form hgc
    int mr = 0, mc = 0, mk = 0;
    for (int b = 0; b < n; ++b) {
      mr = std::max(mr, hgc[b].rows);
      mc = std::max(mc, hgc[b].cols);
      mk = std::max(mk, hgc[b].K);
    }
    const int tC = ((mr + GT_TILE - 1) / GT_TILE) * ((mc + GT_TILE - 1) / GT_TILE);
    nl += run_gemm<L, L, 0>((const GemmT*)(base + d_gc), n, mr, mc, mk, dim3(std::max(1, std::min(tC, 1024)), n), st);
  } else {
    k_gemm<L><<<gg, 128, 0, st>>>((const GemmItem*)(base + d_gemm)); ++nl;
  }
  k_mix<L, NL><<<gg, 128, 16 * 2 * L * 4, st>>>((const MixItem*)(base + d_mix), RBr); ++nl;
  prof_mark(PROF_CONTRACT, 0, st);
  if (pre && !any_dbg) {
    prof_mark(PROF_PRECOND, 1, st);
    int maxM = 0, maxN = 0;
    for (int b = 0; b < n; ++b) { maxM = std::max(maxM, hs[b].M); maxN = std::max(maxN, hs[b].N); }
    nl += launch_pre<L>((const PreItem*)(base + d_pre), (const GemmT*)(base + d_gt), n, maxM, maxN, st);
    if (n_fo > 0) {  // first-order finish (R23)
      const FoItem<NL>* dfo = (const FoItem<NL>*)(base + d_fo);
      const GemmT* dfg = (const GemmT*)(base + d_fogt);
      const size_t fsm = fo_smem<NL>(maxN);
      smem_optin((const void*)k_fo_coef<L, NL>, (int)fsm);
      smem_optin((const void*)k_fo_check<L, NL>, (int)fsm);
      const int tMN = ((maxM + GT_TILE - 1) / GT_TILE) * ((maxN + GT_TILE - 1) / GT_TILE);
      const int g1 = run_gram_ext<L>(dfg, n, maxM, maxN, st);
      if (g1 >= 0) {
        nl += g1;
        k_fo_coef<L, NL><<<n, 256, fsm, st>>>(dfo); ++nl;
      } else {
        k_fo_fail<NL><<<dim3(64, n), 256, 0, st>>>(dfo, n, L); ++nl;
      }
      nl += run_gemm<L, L, 5>(dfg + n, n, maxM, maxN, maxN, dim3(std::min(tMN, 1024), n), st);
      if (g1 >= 0) {
        const int g2 = run_gram_ext<L>(dfg + 2 * n, n, maxM, maxN, st);
        if (g2 >= 0) {
          nl += g2;
          k_fo_check<L, NL><<<n, 256, fsm, st>>>(dfo); ++nl;
        }
      }
    }
    if (getenv("MPS_NS_FORCE_ZERR")) {  // test hook: as if every Newton-Schulz zero-digit check failed
      std::vector<int> two(n, 2);
      cudaMemcpyAsync(redo, two.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st);
      cudaStreamSynchronize(st);
    }
    prof_mark(PROF_PRECOND, 0, st);
  }
  if (any_dbg) {
    for (int b = 0; b < n; ++b) {
      if (!a[b].theta_dbg) continue;
      const MixItem& mi = hm[b];
      k_fixed_to_records<L, NL><<<64, 256, 0, st>>>(mi.A, mi.M, mi.eA, nullptr, mi.M, mi.N, mi.trans,
                                                    a[b].theta_dbg, RBr, p);
      ++nl;
    }
    return nl;
  }
  prof_mark(PROF_JACOBI, 1, st);
  {
    int minN = 1 << 30;
    for (int b = 0; b < n; ++b) minN = std::min(minN, hs[b].N);
    // when most items took the first-order finish (R23) only the few that failed its check run
    // here: size the clusters for a handful of active items (the finished ones exit at once)
    const int n_active = n_fo * 2 >= n ? std::max(1, (n - n_fo) + n_fo / 32) : n;
    launch_jacobi<L, NL>((const SvdItem<NL>*)(base + d_svd), n, jacobi_cluster_size(n_active, minN, jacobi_min_ctas<L>() * 148),
                         st);
    ++nl;
  }
  {
    int maxNN = 0;
    for (int b = 0; b < n; ++b) maxNN = std::max(maxNN, hs[b].N * hs[b].N);
    if (unsigned long long* pc = prof_counts()) {
      k_accum_stats<NL><<<(n + 127) / 128, 128, 0, st>>>((const SvdItem<NL>*)(base + d_svd), n, pc);
      ++nl;
    }
  }
  prof_mark(PROF_JACOBI, 0, st);
  if (unsigned long long* pd = phase_dbg()) {
    unsigned long long h[6 + 128 + 64];
    cudaMemcpyAsync(h, pd, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "jacobi phase cycles (sum over CTAs): D %.4e R %.4e U %.4e norms %.4e init %.4e total %.4e\n",
            (double)h[0], (double)h[1], (double)h[2], (double)h[3], (double)h[4], (double)h[5]);
    for (int sw = 1; sw < 64; ++sw)
      if (h[6 + 2 * sw])
        fprintf(stderr, "  sweep %2d: U digit products per row %.4e, needed with leading-zero skipping %.4e (%.3f)\n", sw,
                (double)h[6 + 2 * sw], (double)h[7 + 2 * sw], (double)h[7 + 2 * sw] / (double)h[6 + 2 * sw]);
    for (int sw = 1; sw < 16; ++sw) {
      const unsigned long long* v = h + 6 + 128 + 4 * sw;
      if (v[0] + v[1] + v[2] + v[3])
        fprintf(stderr, "  sweep %2d: rotations by U variant (0,0) %llu (3,1) %llu (6,3) %llu (10,6) %llu\n", sw, v[0], v[1],
                v[2], v[3]);
    }
    cudaMemsetAsync(pd, 0, sizeof(h), st);
  }
  prof_mark(PROF_FINALIZE, 1, st);
  int maxN = 0;
  for (int b = 0; b < n; ++b) maxN = std::max(maxN, hs[b].N);
  k_finalize<L, NL><<<n, NTHR, sizeof(mpf<NL>) * (size_t)maxN, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p);
  ++nl;
  prof_mark(PROF_FINALIZE, 0, st);
  {
    // V = Theta'^H A_final diag(1/alpha) for the columns the truncation keeps (ord[0..k)), after
    // k_finalize has ordered and counted them (R16)
    prof_mark(PROF_RECOVER, 1, st);
    int maxNr = 0;
    for (int b = 0; b < n; ++b) maxNr = std::max(maxNr, hs[b].N);
    k_recover_coef<L, NL><<<dim3(std::max(1, (maxNr + 127) / 128), n), 128, 0, st>>>((const RecItem<NL>*)(base + d_rec));
    ++nl;
    int maxMr = 0;
    for (int b = 0; b < n; ++b) maxMr = std::max(maxMr, hs[b].M);
    const int tR = ((maxNr + GT_TILE - 1) / GT_TILE) * ((maxNr + GT_TILE - 1) / GT_TILE);
    nl += run_gemm<L, L, 0>((const GemmT*)(base + d_rg), n, maxNr, maxNr, maxMr,
                            dim3(std::max(1, std::min(tR, 1024)), n), st);
    prof_mark(PROF_RECOVER, 0, st);
  }
  prof_mark(PROF_FINALIZE, 1, st);
  dim3 gs(std::max(1, std::min(64, (2 * maxOut + 255) / 256)), n);
  k_split<L, NL><<<gs, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p); ++nl;
  prof_mark(PROF_FINALIZE, 0, st);
  (void)cplx;
  return nl;
}

// launch_update2, then (synchronously) re-run with accumulated V every item whose kept
// spectrum was too wide for the recovered V (FinItem::redo).  Returns the launch count.
template <class T>
int run_update2(int p, double thr, const Upd2Args* a, int n, void* ws, cudaStream_t st,
                std::vector<unsigned char>& hd) {
  constexpr int NL = T::NL;
  int nl = launch_update2<T>(p, thr, a, n, ws, st, hd);
  if (force_accumulate_v()) return nl;
  const size_t d_end = upd2_desc_bytes<T::L, NL>(n);
  std::vector<int> redo(n, 0);
  cudaMemcpyAsync(redo.data(), (char*)ws + d_end, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  std::vector<Upd2Args> sub;
  for (int b = 0; b < n; ++b)
    if (redo[b]) {
      Upd2Args c = a[b];
      c.accumulate_v = 1;
      if (redo[b] & 2) c.no_precond = 1;
      sub.push_back(c);
    }
  if (getenv("MPS_DEBUG_REDO")) {
    int acc = 0;
    for (int b = 0; b < n; ++b) acc += a[b].accumulate_v;
    fprintf(stderr, "two-site batch of %d: %d accumulate V (predicted), %d re-run\n", n, acc, (int)sub.size());
  }
  if (!sub.empty()) {
    std::vector<unsigned char> hd2;
    nl += launch_update2<T>(p, thr, sub.data(), (int)sub.size(), ws, st, hd2);
    cudaStreamSynchronize(st);
  }
  return nl;
}

// ---------------------------------------------------------------------------- three-site
// Theta (4chiL x 2chiR) = U8 (lamL G0 lam1 G1 lam2 G2 lamR); SVD#1 splits off site s+2
// (lambda_{s+1}', Gamma_{s+2}'), M2 = X1 lambda' reshaped (2chiL x 2k1), SVD#2 gives
// lambda_s', Gamma_s', Gamma_{s+1}' (right site first).
struct Upd3Args {
  int chiL, chi1, chi2, chiR, chi_max;
  const uint32_t *G0, *G1, *G2, *lamL, *lam1, *lam2, *lamR, *U;  // lamL/lamR may be null
  // outputs (device): G0_out [2][chiL][ld], G1_out [2][ld][ld] (k2 x k1), G2_out [2][ld][chiR]
  uint32_t *G0_out, *G1_out, *G2_out, *lam1_out, *lam2_out;      // lam1 = lambda_s' (k2), lam2 = lambda_{s+1}' (k1)
  int ld;
  int *k1, *k2, *sweeps, *status;  // device
  int* redo;                        // device flag (one int) or null: recovered V too inaccurate
  int accumulate_v;                 // 1: accumulate V in this stage (the re-run)
  int s1_accumulated;               // stage 2: stage 1 ran with accumulated V (its V exponent is 1)
  int no_precond;                   // 1: this stage without the binary64 preconditioner (R19)
};

// workspace of one three-site update (bounded by the capacities: k1 <= min(chi_max, 2chiR, 4chiL))
template <int L, int NL>
inline size_t upd3_item_bytes(const Upd3Args& a) {
  const int M1 = std::max(4 * a.chiL, 2 * a.chiR), N1 = std::min(4 * a.chiL, 2 * a.chiR);
  const int k1max = std::min(a.chi_max, N1);
  const int M2 = std::max(2 * a.chiL, 2 * k1max), N2 = std::min(2 * a.chiL, 2 * k1max);
  size_t s = mat_bytes(2 * a.chiL, a.chi1, L) + mat_bytes(a.chi1, 2 * a.chi2, L) + mat_bytes(a.chi2, 2 * a.chiR, L) +
             mat_bytes(2 * a.chiL, 2 * a.chi2, L) + mat_bytes(4 * a.chiL, a.chi2, L) + mat_bytes(4 * a.chiL, 2 * a.chiR, L) +
             mat_bytes(M1, N1, L) + mat_bytes(N1, N1, L) + mat_bytes(M2 + 2, N2 + 2, L) + mat_bytes(N2 + 2, N2 + 2, L) +
             SvdScratch<L, NL>::bytes(N1) + SvdScratch<L, NL>::bytes(N2 + 2) + 1024;
  // V recovery (R16): the inputs of both SVDs and the per-column exponents of V
  s += mat_bytes(M1, N1, L) + mat_bytes(M2 + 2, N2 + 2, L) + align_up(8 * (size_t)N1) + align_up(8 * (size_t)(N2 + 2)) +
       256;
  s += pre_bytes<L>(M1, N1) + pre_bytes<L>(M2 + 2, N2 + 2) + 512;  // preconditioners of both SVDs (R19)
  return s;
}

// V-recovery buffers of a three-site update, after everything stage 1 and stage 2 carve
template <int L, int NL>
struct Upd3Rec {
  int32_t *A0a, *A0b;
  int64_t *eVa, *eVb, *eA0a, *eA0b;
  Upd3Rec(char* base_end, const Upd3Args& a) {
    const int M1 = std::max(4 * a.chiL, 2 * a.chiR), N1 = std::min(4 * a.chiL, 2 * a.chiR);
    const int k1max = std::min(a.chi_max, N1);
    const int M2 = std::max(2 * a.chiL, 2 * k1max), N2 = std::min(2 * a.chiL, 2 * k1max);
    char* q = base_end + mat_bytes(2 * a.chiL, a.chi1, L) + mat_bytes(a.chi1, 2 * a.chi2, L) +
              mat_bytes(a.chi2, 2 * a.chiR, L) + mat_bytes(2 * a.chiL, 2 * a.chi2, L) +
              mat_bytes(4 * a.chiL, a.chi2, L) + mat_bytes(4 * a.chiL, 2 * a.chiR, L) + mat_bytes(M1, N1, L) +
              mat_bytes(N1, N1, L) + SvdScratch<L, NL>::bytes(N1) + mat_bytes(M2 + 2, N2 + 2, L) +
              mat_bytes(N2 + 2, N2 + 2, L) + SvdScratch<L, NL>::bytes(N2 + 2);
    A0a = (int32_t*)q; q += mat_bytes(M1, N1, L);
    A0b = (int32_t*)q; q += mat_bytes(M2 + 2, N2 + 2, L);
    eVa = (int64_t*)q; q += align_up(8 * (size_t)N1);
    eVb = (int64_t*)q; q += align_up(8 * (size_t)(N2 + 2));
    eA0a = (int64_t*)q;
    eA0b = eA0a + 1;
    q += 256;
    pre1 = (char*)align_up((size_t)q, 256);
    pre2 = pre1 + pre_bytes<L>(M1, N1);
    M1_ = M1; N1_ = N1; M2_ = M2 + 2; N2_ = N2 + 2;
  }
  char *pre1, *pre2;
  int M1_, N1_, M2_, N2_;
  PreBufs<L> P1() const { return carve_pre<L>(pre1, M1_, N1_); }
  PreBufs<L> P2() const { return carve_pre<L>(pre2, M2_, N2_); }
};

// T (2chiL x 2chi2) -> T' (4chiL x chi2): T'[(2i+j)chiL + a, g] = T[(i chiL + a), (j chi2 + g)]
template <int L>
__global__ void k_relayout_T(const int32_t* T, int32_t* Tp, int chiL, int chi2) {
  const int n = 4 * chiL * chi2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % (4 * chiL), g = t / (4 * chiL);
    const int ij = r / chiL, a = r % chiL, i = ij >> 1, j = ij & 1;
    for (int ri = 0; ri < 2; ++ri) {
      int32_t x[L];
      ldfx<L>(T, 2 * chiL, j * chi2 + g, ri, i * chiL + a, x);
      stfx<L>(Tp, 4 * chiL, g, ri, r, x);
    }
  }
}

template <class T>
size_t upd3_workspace(const Upd3Args& a) {
  return upd3_item_bytes<T::L, T::NL>(a) + 6 * 4096;
}

// Stage 1: contraction, SVD#1, truncation, Gamma_{s+2}' and lambda_{s+1}'.  k1 lands in *a.k1.
template <class T>
int launch_update3_stage1(int p, double thr, const Upd3Args& a, void* ws, cudaStream_t st,
                          std::vector<unsigned char>& hd) {
  constexpr int L = T::L, NL = T::NL;
  const int RBr = record_words(p);
  char* base = (char*)ws;
  const size_t d_prep = 0, d_gemm = 1024, d_mix = 2048, d_svd = 2560, d_fin = 4096, d_end = 6 * 4096;
  hd.assign(d_end, 0);
  char* q = base + d_end;
  const int M1 = std::max(4 * a.chiL, 2 * a.chiR), N1 = std::min(4 * a.chiL, 2 * a.chiR);
  const bool trans1 = 2 * a.chiR > 4 * a.chiL;
  int32_t* Lf = (int32_t*)q; q += mat_bytes(2 * a.chiL, a.chi1, L);
  int32_t* Mf = (int32_t*)q; q += mat_bytes(a.chi1, 2 * a.chi2, L);
  int32_t* Rf = (int32_t*)q; q += mat_bytes(a.chi2, 2 * a.chiR, L);
  int32_t* Tf = (int32_t*)q; q += mat_bytes(2 * a.chiL, 2 * a.chi2, L);
  int32_t* Tp = (int32_t*)q; q += mat_bytes(4 * a.chiL, a.chi2, L);
  int32_t* Th = (int32_t*)q; q += mat_bytes(4 * a.chiL, 2 * a.chiR, L);
  int32_t* A1 = (int32_t*)q; q += mat_bytes(M1, N1, L);
  int32_t* V1 = (int32_t*)q; q += mat_bytes(N1, N1, L);
  auto S1 = SvdScratch<L, NL>::carve(q, N1);
  int64_t* e = S1.e_misc;  // eL, eM, eR, eT ; eTh in S1.e_misc[3]
  PrepItem* hp = (PrepItem*)(hd.data() + d_prep);
  hp[0] = PrepItem{a.G0, a.lamL, a.lam1, a.chiL, a.chi1, 0, Lf, e + 0};
  hp[1] = PrepItem{a.G1, nullptr, a.lam2, a.chi1, a.chi2, 1, Mf, e + 1};
  hp[2] = PrepItem{a.G2, nullptr, a.lamR, a.chi2, a.chiR, 1, Rf, e + 2};
  GemmItem* hg = (GemmItem*)(hd.data() + d_gemm);
  static thread_local int64_t dummy;
  (void)dummy;
  hg[0] = GemmItem{Lf, 2 * a.chiL, e + 0, Mf, a.chi1, e + 1, Tf, 2 * a.chiL, e + 3, 2 * a.chiL, 2 * a.chi2, a.chi1, 0};
  // GEMM2 output exponent goes to S1.e_misc... reuse e+0 after GEMM1 consumed it? keep separate: use eA[N1] region
  int64_t* eTh = S1.eA + N1;  // spare slot after the column exponents (64 bytes of slack)
  hg[1] = GemmItem{Tp, 4 * a.chiL, e + 3, Rf, a.chi2, e + 2, Th, 4 * a.chiL, eTh, 4 * a.chiL, 2 * a.chiR, a.chi2, 0};
  MixItem* hm = (MixItem*)(hd.data() + d_mix);
  const Upd3Rec<L, NL> rec(base + d_end, a);
  const bool pb1 = use_precond() && !a.no_precond;
  const PreBufs<L> PB1 = rec.P1();
  hm[0] = MixItem{Th, 4 * a.chiL, eTh, a.U, 4, a.chiL, a.chiR, trans1 ? 1 : 0, pb1 ? rec.A0a : A1, pb1 ? PB1.eMix : S1.eA,
                  M1, N1};
  const size_t d_pre1 = 16384, d_gt1 = 16640;
  static_assert(16384 + sizeof(PreItem) <= 16640 && 16640 + sizeof(GemmT) * pre_slots<L>() <= 20480, "stage-1 descriptors");
  const bool p_route1 = !force_accumulate_v() && !a.accumulate_v;  // V recovered: fold the last X update
  if (pb1) pre_descs<L>(PB1, M1, N1, rec.A0a, PB1.eMix, A1, S1.eA, a.redo, (PreItem*)(hd.data() + d_pre1),
                        (GemmT*)(hd.data() + d_gt1), 1, p_route1);
  SvdItem<NL>* hs = (SvdItem<NL>*)(hd.data() + d_svd);
  SvdItem<NL> si = {};
  si.M = M1; si.N = N1; si.A = A1; si.eA = S1.eA; si.V = V1; si.alpha = S1.alpha; si.gam = S1.gam;
  si.coef = S1.coef; si.dbg = nullptr; si.rot = S1.rot; si.negl = S1.negl; si.status = S1.status;
  si.sweeps = S1.sweeps; si.rotations = S1.rots; si.sync = S1.sync; si.zbuf = S1.zbuf; si.phase_cycles = nullptr;
  const bool recover = !force_accumulate_v() && !a.accumulate_v;
  si.uprod = S1.uprod;
  si.A0 = recover ? rec.A0a : nullptr; si.eA0 = pb1 ? PB1.eMix : rec.eA0a; si.eV = rec.eVa; si.evals = S1.rots + 1;
  si.a0_ready = pb1 ? 1 : 0;
  if (pb1 && !recover) { si.V = PB1.Xfin(); si.v_preset = 1; }
  hs[0] = si;
  FinItem<NL>* hf = (FinItem<NL>*)(hd.data() + d_fin);
  FinItem<NL> fi;
  std::memset(&fi, 0, sizeof(fi));
  fi.M = M1; fi.N = N1; fi.trans = trans1 ? 1 : 0; fi.A = A1; fi.eA = S1.eA; fi.V = V1; fi.alpha = S1.alpha;
  fi.chi_max = a.chi_max; fi.thr = mpf_host_from_double<NL>(thr); fi.ord = S1.ord; fi.inv_sig = S1.inv_sig;
  fi.lam = S1.lam; fi.k_out = a.k1; fi.status = a.status; fi.sigma_rec = nullptr; fi.nsig = 0;
  fi.svd_status = S1.status;
  fi.lam_rec = a.lam2_out; fi.GL = nullptr;
  fi.GR = a.G2_out; fi.GR_ld = a.ld; fi.lamR = a.lamR; fi.chiR_out = a.chiR;
  fi.chiL2 = a.chiL;
  fi.eV = recover ? rec.eVa : nullptr;
  fi.redo = recover ? a.redo : nullptr; fi.redo_bits = redo_bits<L>();
  hf[0] = fi;
  cudaMemcpyAsync(base, hd.data(), d_end, cudaMemcpyHostToDevice, st);
  int nl = 0;
  k_init_exp<<<1, 32, 0, st>>>(e, 3); ++nl;
  dim3 gp(std::max(1, std::min(64, (2 * a.chi1 * std::max(a.chiL, a.chi2) + 255) / 256)), 1);
  for (int i = 0; i < 3; ++i) {
    k_prep_exp<<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep) + i, RBr); ++nl;
    k_prep_conv<L, NL><<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep) + i, RBr); ++nl;
  }
  dim3 g1(std::max(1, std::min(128, (4 * a.chiL * a.chi2 + 127) / 128)), 1);
  k_gemm<L><<<g1, 128, 0, st>>>((const GemmItem*)(base + d_gemm)); ++nl;
  k_relayout_T<L><<<64, 256, 0, st>>>(Tf, Tp, a.chiL, a.chi2); ++nl;
  dim3 g2(std::max(1, std::min(128, (8 * a.chiL * a.chiR + 127) / 128)), 1);
  k_gemm<L><<<g2, 128, 0, st>>>((const GemmItem*)(base + d_gemm) + 1); ++nl;
  k_mix<L, NL><<<g2, 128, 64 * 2 * L * 4, st>>>((const MixItem*)(base + d_mix), RBr); ++nl;
  if (pb1) nl += launch_pre<L>((const PreItem*)(base + d_pre1), (const GemmT*)(base + d_gt1), 1, M1, N1, st);
  launch_jacobi<L, NL>((const SvdItem<NL>*)(base + d_svd), 1, jacobi_cluster_size(1, N1), st); ++nl;
  if (pb1 && !recover)  // V = X W was accumulated in the preconditioner's buffer; stage 2 reads V1
    cudaMemcpyAsync(V1, PB1.Xfin(), mat_bytes(N1, N1, L), cudaMemcpyDeviceToDevice, st);
  k_recover_v<L, NL><<<dim3(std::max(1, std::min(64, (N1 * N1 + 127) / 128)), 1), 128, 0, st>>>(
      (const SvdItem<NL>*)(base + d_svd)); ++nl;
  k_finalize<L, NL><<<1, NTHR, sizeof(mpf<NL>) * (size_t)N1, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p); ++nl;
  dim3 gs(std::max(1, std::min(64, (2 * a.chiR * N1 + 255) / 256)), 1);
  k_split<L, NL><<<gs, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p); ++nl;
  // sweeps of SVD#1 accumulate into *a.sweeps by the host (stage 2 reads S1.sweeps)
  cudaMemcpyAsync(a.sweeps, S1.sweeps, sizeof(int), cudaMemcpyDeviceToDevice, st);
  return nl;
}

// Stage 2 (k1 known on the host): M2 from SVD#1's left factor, SVD#2, split into G0', G1'.
template <class T>
int launch_update3_stage2(int p, double thr, const Upd3Args& a, int k1, void* ws, cudaStream_t st,
                          std::vector<unsigned char>& hd) {
  constexpr int L = T::L, NL = T::NL;
  const int RBr = record_words(p);
  char* base = (char*)ws;
  const size_t d_fin = 4096, d_svd2 = 8192, d_fin2 = 12288, d_end = 6 * 4096;
  // recover the stage-1 layout
  char* q = base + d_end;
  const int M1 = std::max(4 * a.chiL, 2 * a.chiR), N1 = std::min(4 * a.chiL, 2 * a.chiR);
  const int k1max = std::min(a.chi_max, N1);
  q += mat_bytes(2 * a.chiL, a.chi1, L) + mat_bytes(a.chi1, 2 * a.chi2, L) + mat_bytes(a.chi2, 2 * a.chiR, L) +
       mat_bytes(2 * a.chiL, 2 * a.chi2, L) + mat_bytes(4 * a.chiL, a.chi2, L) + mat_bytes(4 * a.chiL, 2 * a.chiR, L) +
       mat_bytes(M1, N1, L) + mat_bytes(N1, N1, L);
  auto S1 = SvdScratch<L, NL>::carve(q, N1);
  q += SvdScratch<L, NL>::bytes(N1);
  const int rows2 = 2 * a.chiL, cols2 = 2 * k1;
  const bool trans2 = cols2 > rows2;
  const int M2 = std::max(rows2, cols2), N2 = std::min(rows2, cols2);
  const int M2c = std::max(2 * a.chiL, 2 * k1max), N2c = std::min(2 * a.chiL, 2 * k1max);
  int32_t* A2 = (int32_t*)q; q += mat_bytes(M2c + 2, N2c + 2, L);
  int32_t* V2 = (int32_t*)q; q += mat_bytes(N2c + 2, N2c + 2, L);
  auto S2 = SvdScratch<L, NL>::carve(q, N2c + 2);
  hd.assign(d_end, 0);
  // the FinItem of SVD#1 (re-sent with the M2 target filled in)
  FinItem<NL>* hf1 = (FinItem<NL>*)(hd.data() + d_fin);
  {
    FinItem<NL> fi;
    std::memset(&fi, 0, sizeof(fi));
    const int32_t* A1 = (const int32_t*)(base + d_end + mat_bytes(2 * a.chiL, a.chi1, L) +
                                         mat_bytes(a.chi1, 2 * a.chi2, L) + mat_bytes(a.chi2, 2 * a.chiR, L) +
                                         mat_bytes(2 * a.chiL, 2 * a.chi2, L) + mat_bytes(4 * a.chiL, a.chi2, L) +
                                         mat_bytes(4 * a.chiL, 2 * a.chiR, L));
    fi.M = M1; fi.N = N1; fi.trans = 2 * a.chiR > 4 * a.chiL; fi.A = A1; fi.eA = S1.eA;
    fi.V = (const int32_t*)((const char*)A1 + mat_bytes(M1, N1, L));
    fi.alpha = S1.alpha; fi.ord = S1.ord; fi.inv_sig = S1.inv_sig; fi.lam = S1.lam; fi.k_out = a.k1;
    fi.status = a.status; fi.chiL2 = a.chiL; fi.M2 = A2; fi.eM2 = S2.eA; fi.M2_trans = trans2 ? 1 : 0;
    const Upd3Rec<L, NL> r1(base + d_end, a);
    fi.eV = (force_accumulate_v() || a.s1_accumulated) ? nullptr : r1.eVa;  // M2 from V1 when trans
    fi.M2_A0 = r1.A0b; fi.M2_eA0 = r1.eA0b;
    hf1[0] = fi;
  }
  SvdItem<NL>* hs = (SvdItem<NL>*)(hd.data() + d_svd2);
  SvdItem<NL> si = {};
  si.M = M2; si.N = N2; si.A = A2; si.eA = S2.eA; si.V = V2; si.alpha = S2.alpha; si.gam = S2.gam;
  si.coef = S2.coef; si.dbg = nullptr; si.rot = S2.rot; si.negl = S2.negl; si.status = S2.status;
  const Upd3Rec<L, NL> rec(base + d_end, a);
  si.sweeps = S2.sweeps; si.rotations = S2.rots; si.sync = S2.sync; si.zbuf = S2.zbuf; si.phase_cycles = nullptr;
  const bool recover = !force_accumulate_v() && !a.accumulate_v;
  si.uprod = S2.uprod;
  si.A0 = recover ? rec.A0b : nullptr; si.eA0 = rec.eA0b; si.eV = rec.eVb; si.evals = S2.rots + 1; si.a0_ready = 1;
  const bool pb2 = use_precond() && !a.no_precond;
  const PreBufs<L> PB2 = rec.P2();
  if (pb2 && !recover) { si.V = PB2.Xfin(); si.v_preset = 1; }
  const size_t d_pre2 = 20480, d_gt2 = 20736;
  static_assert(20480 + sizeof(PreItem) <= 20736 && 20736 + sizeof(GemmT) * pre_slots<L>() <= 24576, "stage-2 descriptors");
  if (pb2) pre_descs<L>(PB2, M2, N2, rec.A0b, rec.eA0b, A2, S2.eA, a.redo, (PreItem*)(hd.data() + d_pre2),
                        (GemmT*)(hd.data() + d_gt2), 1);
  hs[0] = si;
  FinItem<NL>* hf = (FinItem<NL>*)(hd.data() + d_fin2);
  FinItem<NL> fi;
  std::memset(&fi, 0, sizeof(fi));
  fi.M = M2; fi.N = N2; fi.trans = trans2 ? 1 : 0; fi.A = A2; fi.eA = S2.eA; fi.V = si.V; fi.alpha = S2.alpha;
  fi.chi_max = a.chi_max; fi.thr = mpf_host_from_double<NL>(thr); fi.ord = S2.ord; fi.inv_sig = S2.inv_sig;
  fi.lam = S2.lam; fi.k_out = a.k2; fi.status = S2.fstatus; fi.sigma_rec = nullptr; fi.nsig = 0;
  fi.svd_status = S2.status;
  fi.lam_rec = a.lam1_out;
  fi.GL = a.G0_out; fi.GL_ld = a.ld; fi.lamL = a.lamL; fi.chiL_out = a.chiL;
  fi.GR = a.G1_out; fi.GR_ld = a.ld; fi.lamR = a.lam2_out; fi.chiR_out = k1;
  fi.eV = recover ? rec.eVb : nullptr;
  fi.redo = recover ? a.redo : nullptr; fi.redo_bits = redo_bits<L>();
  hf[0] = fi;
  cudaMemcpyAsync(base + d_fin, hd.data() + d_fin, d_end - d_fin, cudaMemcpyHostToDevice, st);
  int nl = 0;
  k_m2_exp<L, NL><<<1, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin), S2.e_misc); ++nl;
  dim3 gb(std::max(1, std::min(64, (rows2 * cols2 + 255) / 256)), 1);
  k_build_m2<L, NL><<<gb, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin), S2.e_misc); ++nl;
  if (pb2) nl += launch_pre<L>((const PreItem*)(base + d_pre2), (const GemmT*)(base + d_gt2), 1, M2, N2, st);
  launch_jacobi<L, NL>((const SvdItem<NL>*)(base + d_svd2), 1, jacobi_cluster_size(1, N2), st); ++nl;
  k_recover_v<L, NL><<<dim3(std::max(1, std::min(64, (N2 * N2 + 127) / 128)), 1), 128, 0, st>>>(
      (const SvdItem<NL>*)(base + d_svd2)); ++nl;
  k_finalize<L, NL><<<1, NTHR, sizeof(mpf<NL>) * (size_t)N2, st>>>((const FinItem<NL>*)(base + d_fin2), RBr, p); ++nl;
  dim3 gs(std::max(1, std::min(64, (2 * std::max(a.chiL, k1) * N2 + 255) / 256)), 1);
  k_split<L, NL><<<gs, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin2), RBr, p); ++nl;
  k_add_int<<<1, 1, 0, st>>>(a.sweeps, S2.sweeps, a.status, S2.fstatus); ++nl;
  return nl;
}

}  // namespace mpsb
