// Tensor-core multiprecision GEMM: every GemmT product of the update (the contraction, the
// Newton-Schulz iterations, the refinement-sweep GEMMs, A_1 = Theta' X / P = Theta' X_{n-1} /
// A_1 = P + P D/2, the Gram matrices and A_1 (I + E) of the first-order finish, the recovery of
// V) on the 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM) instead of
// the IMAD.WIDE pipe (DESIGN.md §4 "Tensor cores").
//
// Every p-bit operand value of the LG-digit frame (balanced radix-2^28 int32 digits) is
// re-sliced EXACTLY into S = floor((7 LG + 1) / 2) + 1 balanced base-256 slices of the whole
// value, x = sum_s u_s 2^(8s), u_s in [-128, 127] (TC_SLICE_BITS = 7 keeps the first version:
// four 7-bit slices per digit).  A real product of two values is then sum_{s,t} u_s v_t 2^(8(s+t)),
// and a real GEMM C = A B is, per slice-weight group d = s + t, the int8 GEMM
// sum_{s+t=d} A_s B_t with exact int32 accumulation (each term <= 2^14, K <= 512, <= 68 pairs per
// group at 19 digits: < 2^30).  Groups of weight >= 2^(28 (LG - 2)) are formed (a superset of the
// digit pairs i + j >= LG - 2 the IMAD path keeps, so the truncated product is at least as
// accurate); the epilogue combines them into the int64 digit columns of the IMAD path and runs
// the same rounding / store code (gemm_t_store).  Complex: Re C = Ar Br + Ai (-Bi),
// Im C = Ar Bi + Ai Br (4 real products, accumulated in TMEM).
//
// Kernels per scratch chunk of items: k_tc_slice_a / k_tc_slice_b (digits -> int8 slice tiles in
// the UMMA K-major no-swizzle layout, so that staging is a straight bulk copy), k_tc_mma (one CTA
// per 128 x TC_N output tile and plane: TC_GCH groups at a time in TMEM; a producer warp streams
// stages of TC_SBK A-slice tiles and the B-slice tiles they meet into TC_NSTG shared-memory
// buffers with cp.async.bulk + mbarrier transaction counts, TC_WARPS warps issue the MMAs of
// their group and drain the chunk sums with tcgen05.ld), k_tc_epi (one thread per output entry).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <tuple>

#include "precond.cuh"

namespace mpsb {

#ifndef TC_N_   // tile shape switches (development A/B builds)
#define TC_N_ 128
#endif
#ifndef TC_GCH_
#define TC_GCH_ (512 / TC_N_)
#endif
#ifndef TC_WARPS_
#define TC_WARPS_ 4
#endif
#ifndef TC_SBK_
#define TC_SBK_ 6
#endif
#ifndef TC_NSTG_
#define TC_NSTG_ 3
#endif
#ifndef TC_PACKED  // 1: the drain combines the groups of a chunk into one int64 per entry (half the scratch traffic)
#define TC_PACKED 1
#endif
#ifndef TC_PRODUCER  // 1: a fifth warp streams the stage tiles; the MMA warps never wait for a buffer to drain
#define TC_PRODUCER 1
#endif
constexpr int TC_M = 128;  // output rows per CTA = MMA M = TMEM lanes
constexpr int TC_N = TC_N_;   // output columns per CTA = MMA N
constexpr int TC_K = 32;   // k per MMA instruction (kind::i8)
constexpr int TC_GCH = TC_GCH_;   // slice-weight groups per chunk: TC_GCH accumulators x TC_N columns = 512 TMEM columns
constexpr int TC_WARPS = TC_WARPS_;  // warps of k_tc_mma: warp w issues the MMAs of groups d0 + w (TC_GCH / TC_WARPS each)
constexpr int TC_SBK = TC_SBK_;  // A slices per pipeline stage (with the <= TC_SBK + TC_GCH - 1 B slices they meet)
constexpr int TC_THREADS = (TC_WARPS_ + (TC_PRODUCER ? 1 : 0)) * 32;
constexpr int TC_LOADER = TC_PRODUCER ? TC_WARPS_ : 0;  // the warp that issues the bulk copies
constexpr int TC_NSTG = TC_NSTG_;  // shared-memory stage buffers (bulk copies run TC_NSTG - 1 stages ahead of the MMAs)
static_assert(TC_GCH * TC_N <= 512 && TC_GCH % TC_WARPS == 0 && TC_WARPS % 4 == 0, "TMEM columns / warp roles");
constexpr int TC_STAGE = TC_SBK * 4096 + (TC_SBK + TC_GCH - 1) * TC_N * 32;  // bytes of one stage buffer
constexpr int TC_ATILE = TC_M * TC_K;  // bytes of one A slice tile
constexpr int TC_BTILE = TC_N * TC_K;  // bytes of one B slice tile

// Slice width: TC_SLICE_BITS = 7 (four slices per 28-bit digit) or 8 (balanced base-256 slices of
// the whole value: 7 slices per two digits, ~20% fewer slice pairs per product).
#ifndef TC_SLICE_BITS
#define TC_SLICE_BITS 8
#endif
constexpr int TC_SB = TC_SLICE_BITS;
static_assert(TC_SB == 7 || TC_SB == 8, "slice width");
// slices per LG-digit value (the last one the carry out of the top), the lowest slice-weight
// group formed (weight 2^(TC_SB d) >= 2^(28 (LG - 2)), the lowest digit column the IMAD path keeps),
// the highest group, the group count
template <int LG> __host__ __device__ constexpr int tc_ns() { return TC_SB == 7 ? 4 * LG + 1 : (7 * LG + 1) / 2 + 1; }
template <int LG> __host__ __device__ constexpr int tc_dlo() { return TC_SB == 7 ? 4 * (LG - 2) : (7 * (LG - 2) + 1) / 2; }
template <int LG> __host__ __device__ constexpr int tc_dhi() { return 2 * (tc_ns<LG>() - 1); }
template <int LG> __host__ __device__ constexpr int tc_ng() { return tc_dhi<LG>() - tc_dlo<LG>() + 1; }
// first slice that can be nonzero when the nz lowest digits are zero; one past the last slice
// that can be nonzero when the top z digits are zero
__host__ __device__ constexpr int tc_slice_lo(int nz) { return TC_SB == 7 ? 4 * nz : (7 * nz) / 2; }
template <int LG> __host__ __device__ constexpr int tc_slice_hi(int z) {
  return z <= 0 ? tc_ns<LG>() : (TC_SB == 7 ? 4 * (LG - z) : ((7 * (LG - z) + 1) / 2 + 1 < tc_ns<LG>() ? (7 * (LG - z) + 1) / 2 + 1 : tc_ns<LG>()));
}

struct TcDims {
  int tilesR, tilesC, kb;  // output row tiles (128), column tiles (32), k blocks (32), max over items
  size_t a_item, b_item, g_item;  // scratch bytes per item
  int8_t* A;                     // [item][plane 2][S][tilesR][kb][4096]
  int8_t* B;                     // [item][plane 3: re, im, -im][S][tilesC][kb][1024]
  int32_t* G;                    // [item][plane 2][NG][tilesC * TC_N][tilesR * 128] group sums, or (TC_PACKED)
                                 // int64 [item][plane 2][NCH][tilesC * TC_N][tilesR * 128] chunk sums
  int bisect;                    // debug (MPS_TC_BISECT): bit 0 no MMA, bit 1 no drain, bit 2 no staging
  unsigned long long* cnt;       // profiling counters (CNT_TC_MAC), or null
};

// byte offset of element (x, k) inside a K-major no-swizzle UMMA tile: core matrices of 8 rows
// x 16 bytes, [x / 8][k / 16][x % 8][k % 16] (32 k per tile)
__device__ __forceinline__ int tc_off(int x, int k) { return (((x >> 3) * 2 + (k >> 4)) << 7) + ((x & 7) << 4) + (k & 15); }

// next balanced 7-bit slice of v (v <- (v - u) / 128)
__device__ __forceinline__ int tc_bal7(int32_t& v) {
  const int32_t u = ((v + 64) & 127) - 64;
  v = (v - u) >> 7;
  return u;
}

// the four slices of digit v (+ the carry from the digit below): three balanced 7-bit slices and
// a fourth that keeps the rest when it fits int8 (always for balanced digits, so a zero digit
// gives zero slices and no carry), else balanced with a carry into the next digit
__device__ __forceinline__ void tc_digit(int32_t v, int32_t& carry, int (&u)[4]) {
  v += carry;
  u[0] = tc_bal7(v);
  u[1] = tc_bal7(v);
  u[2] = tc_bal7(v);
  if (v >= -128 && v <= 127) {
    u[3] = v;
    carry = 0;
  } else {
    u[3] = tc_bal7(v);
    carry = v;
  }
}

// base-256 slicing (TC_SB = 8): acc holds (x_{<=j} - emitted slices) / 2^(8 s); digit j enters at
// bit 28 j - 8 s in {0, 4}; slices s with 8 (s + 1) <= 28 (j + 1) are final after digit j (later
// digits only touch higher bits); balanced slices in [-128, 127] (the unique balanced base-256
// representation of x, so -x is sliced separately, never negated slice by slice)
__device__ __forceinline__ int tc_bal8(int64_t& acc) {
  const int u = (int)(((acc + 128) & 255) - 128);
  acc = (acc - u) >> 8;
  return u;
}
__device__ __forceinline__ void tc_add_digit8(int64_t& acc, int32_t d, int j) { acc += (int64_t)d << (28 * j - 8 * ((7 * j) / 2)); }

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// descriptor of a K-major no-swizzle tile: LBO = 128 B (k-adjacent core matrices), SBO = 256 B
// (8-row groups), sm100 descriptor version 1
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// instruction descriptor: dense, s32 accumulator, signed int8 A and B, K-major, M x N
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#if TC_SLICE_BITS == 7
// ---------------------------------------------------------------------------- slicing
// Operand A of the item (rows x K): plane ri of op(A)(r, k) in the LG-digit frame (digits
// D0 .. L-1 of the stored value).  conjA: A is stored K x rows, op(A) = A^H.
// Block (tile r, k block) of 128 x 32 entries; 256 threads.
template <int L, int LG>
__global__ void __launch_bounds__(256) k_tc_slice_a(const GemmT* items, int first, TcDims dm) {
  constexpr int S = tc_ns<LG>(), D0 = L - LG;
  const int item = first + blockIdx.z;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const int ri = blockIdx.y, rt = blockIdx.x % dm.tilesR, kbk = blockIdx.x / dm.tilesR;
  if (rt * TC_M >= it.rows || kbk * TC_K >= it.K) return;  // tiles no MMA reads
  int8_t* out = dm.A + blockIdx.z * dm.a_item + (size_t)ri * S * dm.tilesR * dm.kb * TC_ATILE +
                ((size_t)rt * dm.kb + kbk) * TC_ATILE;
  const size_t sstride = (size_t)dm.tilesR * dm.kb * TC_ATILE;  // between slices
  __shared__ int32_t T[TC_K][TC_M + 1];
  // element e = t + 256 i: k = e % 32 (fastest: coalesced tile bytes), x = e / 32
  int32_t carry[16];
  int64_t acc8[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { carry[i] = 0; acc8[i] = 0; }
  for (int j = 0; j < LG; ++j) {
    if (!it.conjA) {  // digits contiguous along rows: stage [k][x] through shared memory
      __syncthreads();
      for (int e = threadIdx.x; e < TC_M * TC_K; e += 256) {
        const int x = e % TC_M, k = e / TC_M;
        const int r = rt * TC_M + x, kk = kbk * TC_K + k;
        T[k][x] = (r < it.rows && kk < it.K && D0 + j >= 0) ? it.A[((size_t)(kk * 2 + ri) * L + D0 + j) * it.lda + r] : 0;
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = threadIdx.x + 256 * i, k = e & 31, x = e >> 5;
      int32_t v;
      if (!it.conjA) {
        v = T[k][x];
      } else {  // A stored K x rows, digits contiguous along k: op(A)(r, k) = conj A(k, r)
        const int r = rt * TC_M + x, kk = kbk * TC_K + k;
        v = (r < it.rows && kk < it.K && D0 + j >= 0) ? it.A[((size_t)(r * 2 + ri) * L + D0 + j) * it.lda + kk] : 0;
        if (ri) v = -v;
      }
      const int o = tc_off(x, k);
      if (TC_SB == 7) {
        int uu[4];
        tc_digit(v, carry[i], uu);
#pragma unroll
        for (int u = 0; u < 4; ++u) out[(size_t)(4 * j + u) * sstride + o] = (int8_t)uu[u];
      } else {
        tc_add_digit8(acc8[i], v, j);
        for (int sl = (7 * j) / 2; sl < (7 * (j + 1)) / 2; ++sl) out[(size_t)sl * sstride + o] = (int8_t)tc_bal8(acc8[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = threadIdx.x + 256 * i, k = e & 31, x = e >> 5;
    if (TC_SB == 7) {
      out[(size_t)(S - 1) * sstride + tc_off(x, k)] = (int8_t)carry[i];
    } else {
      for (int sl = (7 * LG) / 2; sl < S - 1; ++sl) out[(size_t)sl * sstride + tc_off(x, k)] = (int8_t)tc_bal8(acc8[i]);
      out[(size_t)(S - 1) * sstride + tc_off(x, k)] = (int8_t)acc8[i];
    }
  }
}

// Operand B (K x cols), logical column c = physical column colmap[c] (c < ncols): planes
// 0 re, 1 im, 2 -im.  Block (tile c, k block) of TC_N x 32 entries; 256 threads.
template <int L, int LG>
__global__ void __launch_bounds__(256) k_tc_slice_b(const GemmT* items, int first, TcDims dm) {
  constexpr int S = tc_ns<LG>(), D0 = L - LG;
  const int item = first + blockIdx.z;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const int ri = blockIdx.y, ct = blockIdx.x % dm.tilesC, kbk = blockIdx.x / dm.tilesC;
  const int ncols = it.ncols_dev ? min(*it.ncols_dev, it.cols) : it.cols;
  if (ct * TC_N >= ncols || kbk * TC_K >= it.K) return;  // tiles no MMA reads
  const size_t sstride = (size_t)dm.tilesC * dm.kb * TC_BTILE;
  const size_t pstride = (size_t)S * sstride;
  int8_t* out = dm.B + blockIdx.z * dm.b_item + (size_t)ri * pstride + ((size_t)ct * dm.kb + kbk) * TC_BTILE;
#pragma unroll
  for (int i = 0; i < TC_N * TC_K / 256; ++i) {
    const int e = threadIdx.x + 256 * i, k = e & 31, x = e >> 5;
    const int c = ct * TC_N + x, kk = kbk * TC_K + k;
    const bool ok = c < ncols && kk < it.K;
    const int pc = ok ? (it.colmap ? it.colmap[c] : c) : 0;
    const int o = tc_off(x, k);
    int32_t carry = 0;
    int64_t ap = 0, an = 0;  // TC_SB = 8: slicing of v and of -v (plane 2)
#pragma unroll
    for (int j = 0; j < LG; ++j) {
      const int32_t v = (ok && D0 + j >= 0) ? it.B[((size_t)(pc * 2 + ri) * L + D0 + j) * it.ldb + kk] : 0;
      if (TC_SB == 7) {
        int uu[4];
        tc_digit(v, carry, uu);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          out[(size_t)(4 * j + u) * sstride + o] = (int8_t)uu[u];
          if (ri) out[pstride + (size_t)(4 * j + u) * sstride + o] = (int8_t)(-uu[u]);  // plane 2: -im
        }
      } else {
        tc_add_digit8(ap, v, j);
        if (ri) tc_add_digit8(an, -v, j);
#pragma unroll
        for (int sl = (7 * j) / 2; sl < (7 * (j + 1)) / 2; ++sl) {
          out[(size_t)sl * sstride + o] = (int8_t)tc_bal8(ap);
          if (ri) out[pstride + (size_t)sl * sstride + o] = (int8_t)tc_bal8(an);
        }
      }
    }
    if (TC_SB == 7) {
      out[(size_t)(S - 1) * sstride + o] = (int8_t)carry;
      if (ri) out[pstride + (size_t)(S - 1) * sstride + o] = (int8_t)(-carry);
    } else {
      for (int sl = (7 * LG) / 2; sl < S - 1; ++sl) {
        out[(size_t)sl * sstride + o] = (int8_t)tc_bal8(ap);
        if (ri) out[pstride + (size_t)sl * sstride + o] = (int8_t)tc_bal8(an);
      }
      out[(size_t)(S - 1) * sstride + o] = (int8_t)ap;
      if (ri) out[pstride + (size_t)(S - 1) * sstride + o] = (int8_t)an;
    }
  }
}

#else
// ---------------------------------------------------------------------------- slicing (8-bit)
// A thread owns 16 consecutive k of one row x of a tile (half a tile row: one 16-byte line of a
// core matrix), keeps their running values in 16 int64 and writes every finished slice as ONE
// 16-byte store; the 8 lanes of consecutive x fill a 128-byte core matrix.  (The first version
// wrote single bytes, 16 useful bytes per 32-byte sector: the slicing kernels took half as long
// as the MMAs, profiles/r02_launches_v56.csv.)
struct TcAcc16 { int64_t a[16]; };
__device__ __forceinline__ uint4 tc_emit16(TcAcc16& t, bool last) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t u = last ? (uint32_t)(t.a[i] & 255) : (uint32_t)(tc_bal8(t.a[i]) & 255);
    w[i >> 2] |= u << (8 * (i & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// 16 consecutive ints p[0..15] (the first nv valid, the rest 0); vector loads when aligned
__device__ __forceinline__ void tc_load16(const int32_t* p, int nv, bool neg, int32_t (&v)[16]) {
  if (nv == 16 && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 t = __ldg((const int4*)p + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i < nv ? __ldg(p + i) : 0;
  }
  if (neg) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = -v[i];
  }
}
// byte offset of the 16-byte line (x, k group kg) of a tile
__device__ __forceinline__ int tc_line(int x, int kg) { return (((x >> 3) * 2 + kg) << 7) + ((x & 7) << 4); }

// digit j of 16 values enters the running values; the slices it completes are stored
template <int LG, bool NEG2>
__device__ __forceinline__ void tc_slice_digit(int j, const int32_t (&v)[16], TcAcc16& ap, TcAcc16& an, int8_t* o1, int8_t* o2,
                                               size_t sstride) {
  const int sh = 28 * j - 8 * ((7 * j) / 2);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    ap.a[i] += (int64_t)v[i] << sh;
    if (NEG2) an.a[i] += (int64_t)(-v[i]) << sh;
  }
  for (int sl = (7 * j) / 2; sl < (7 * (j + 1)) / 2; ++sl) {
    *(uint4*)(o1 + (size_t)sl * sstride) = tc_emit16(ap, false);
    if (NEG2) *(uint4*)(o2 + (size_t)sl * sstride) = tc_emit16(an, false);
  }
}
template <int LG, bool NEG2>
__device__ __forceinline__ void tc_slice_tail(TcAcc16& ap, TcAcc16& an, int8_t* o1, int8_t* o2, size_t sstride) {
  constexpr int S = tc_ns<LG>();
  for (int sl = (7 * LG) / 2; sl < S; ++sl) {
    *(uint4*)(o1 + (size_t)sl * sstride) = tc_emit16(ap, sl == S - 1);
    if (NEG2) *(uint4*)(o2 + (size_t)sl * sstride) = tc_emit16(an, sl == S - 1);
  }
}

// Operand A of the item (rows x K): plane ri of op(A)(r, k) in the LG-digit frame (digits
// D0 .. L-1 of the stored value).  conjA: A is stored K x rows, op(A) = A^H.
// Block (tile r, k block) of 128 x 32 entries; 256 threads = 128 rows x 2 k groups.
template <int L, int LG>
__global__ void __launch_bounds__(256) k_tc_slice_a(const GemmT* items, int first, TcDims dm) {
  constexpr int S = tc_ns<LG>(), D0 = L - LG;
  const int item = first + blockIdx.z;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const int ri = blockIdx.y, rt = blockIdx.x % dm.tilesR, kbk = blockIdx.x / dm.tilesR;
  if (rt * TC_M >= it.rows || kbk * TC_K >= it.K) return;  // tiles no MMA reads
  const size_t sstride = (size_t)dm.tilesR * dm.kb * TC_ATILE;  // between slices
  const int x = threadIdx.x % TC_M, kg = threadIdx.x / TC_M;
  int8_t* out = dm.A + blockIdx.z * dm.a_item + (size_t)ri * S * sstride + ((size_t)rt * dm.kb + kbk) * TC_ATILE + tc_line(x, kg);
  const int r = rt * TC_M + x, k0 = kbk * TC_K + 16 * kg;
  const int nv = r < it.rows ? max(0, min(16, it.K - k0)) : 0;
  TcAcc16 ap, an;
#pragma unroll
  for (int i = 0; i < 16; ++i) ap.a[i] = 0;
#pragma unroll 1
  for (int j = 0; j < LG; ++j) {
    int32_t v[16];
    if (D0 + j < 0 || nv == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0;
    } else if (!it.conjA) {  // op(A)(r, k) = A(r, k): rows contiguous (coalesced across the lanes)
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < nv ? __ldg(it.A + ((size_t)((k0 + i) * 2 + ri) * L + D0 + j) * it.lda + r) : 0;
    } else {                 // op(A)(r, k) = conj A(k, r): k contiguous
      tc_load16(it.A + ((size_t)(r * 2 + ri) * L + D0 + j) * it.lda + k0, nv, ri != 0, v);
    }
    tc_slice_digit<LG, false>(j, v, ap, an, out, out, sstride);
  }
  tc_slice_tail<LG, false>(ap, an, out, out, sstride);
}

// Operand B (K x cols), logical column c = physical column colmap[c] (c < ncols): planes
// 0 re, 1 im, 2 -im.  Block (tile c, k block) of TC_N x 32 entries; thread = (column, k group).
template <int L, int LG>
__global__ void __launch_bounds__(256) k_tc_slice_b(const GemmT* items, int first, TcDims dm) {
  constexpr int S = tc_ns<LG>(), D0 = L - LG;
  const int item = first + blockIdx.z;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const int ri = blockIdx.y, ct = blockIdx.x % dm.tilesC, kbk = blockIdx.x / dm.tilesC;
  const int ncols = it.ncols_dev ? min(*it.ncols_dev, it.cols) : it.cols;
  if (ct * TC_N >= ncols || kbk * TC_K >= it.K) return;  // tiles no MMA reads
  const size_t sstride = (size_t)dm.tilesC * dm.kb * TC_BTILE;
  const size_t pstride = (size_t)S * sstride;
  for (int e = threadIdx.x; e < TC_N * 2; e += 256) {
    const int x = e % TC_N, kg = e / TC_N;
    int8_t* out = dm.B + blockIdx.z * dm.b_item + (size_t)ri * pstride + ((size_t)ct * dm.kb + kbk) * TC_BTILE + tc_line(x, kg);
    const int c = ct * TC_N + x, k0 = kbk * TC_K + 16 * kg;
    const int nv = c < ncols ? max(0, min(16, it.K - k0)) : 0;
    const int pc = nv ? (it.colmap ? it.colmap[c] : c) : 0;
    TcAcc16 ap, an;
#pragma unroll
    for (int i = 0; i < 16; ++i) { ap.a[i] = 0; an.a[i] = 0; }
#pragma unroll 1
    for (int j = 0; j < LG; ++j) {
      int32_t v[16];
      if (D0 + j < 0 || nv == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0;
      } else {
        tc_load16(it.B + ((size_t)(pc * 2 + ri) * L + D0 + j) * it.ldb + k0, nv, false, v);
      }
      if (ri) tc_slice_digit<LG, true>(j, v, ap, an, out, out + pstride, sstride);   // plane 2: -im
      else tc_slice_digit<LG, false>(j, v, ap, an, out, out, sstride);
    }
    if (ri) tc_slice_tail<LG, true>(ap, an, out, out + pstride, sstride);
    else tc_slice_tail<LG, false>(ap, an, out, out, sstride);
  }
}

#endif
// ---------------------------------------------------------------------------- MMA
// 1 in exactly one lane of the (converged) warp
__device__ __forceinline__ uint32_t tc_elect() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(e));
  return e;
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tTCW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra TCW_%=;\n\t}\n" ::"r"(bar), "r"(parity));
}

// One CTA per 128 x TC_N output tile and plane (re / im of C = Re / Im sum of 2 real products).
// Slice-weight groups d = s + t in [DLO, 8 LG] are accumulated TC_GCH at a time in TMEM
// (a chunk).  The MMAs of a chunk are cut into stages (term, k block, block of TC_SBK A slices
// with the B slices they meet); thread 0 streams the stage tiles into two shared-memory buffers
// with bulk copies (mbarrier transaction counts) one stage ahead and issues the stage's MMAs,
// whose tcgen05.commit frees the buffer (the next stage is loaded right after a stage's MMAs are
// issued, into the buffer the previous stage's MMAs release); after a chunk all warps drain its accumulators to the
// group-sum scratch (tcgen05.ld).  Slice ranges: A s in [SA0, S), B t in [SB0, SB1).
template <int LG, int SA0, int SB0, int SB1>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tc_mma(const GemmT* items, int first, TcDims dm) {
  constexpr int S = tc_ns<LG>(), DLO = tc_dlo<LG>(), NG = tc_ng<LG>(), DHI = tc_dhi<LG>();
  constexpr int NCH = (NG + TC_GCH - 1) / TC_GCH;
  constexpr uint32_t IDESC = tc_idesc(TC_M, TC_N);
  const int item = first + blockIdx.y;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const int plane = blockIdx.x & 1, rest = blockIdx.x >> 1;
  const int rt = rest % dm.tilesR, ct = rest / dm.tilesR;
  const int ncols = it.ncols_dev ? min(*it.ncols_dev, it.cols) : it.cols;
  if (rt * TC_M >= it.rows || ct * TC_N >= ncols) return;  // CTA-uniform
  if (it.upper && ct * TC_N + TC_N <= rt * TC_M) return;      // entirely below the diagonal
  const int nkb = (it.K + TC_K - 1) / TC_K;
  extern __shared__ __align__(1024) int8_t tcs[];  // [TC_NSTG][TC_STAGE]
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar_full[TC_NSTG], bar_empty[TC_NSTG];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc_smem(&tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int b = 0; b < TC_NSTG; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(tc_smem(&bar_full[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tc_smem(&bar_empty[b])), "n"(TC_WARPS));  // one commit per warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const size_t a_s = (size_t)dm.tilesR * dm.kb * TC_ATILE, b_s = (size_t)dm.tilesC * dm.kb * TC_BTILE;
  const int8_t* Ab = dm.A + blockIdx.y * dm.a_item;
  const int8_t* Bb = dm.B + blockIdx.y * dm.b_item;
  int32_t* Gb = (int32_t*)((char*)dm.G + blockIdx.y * dm.g_item);
  const int RRr = dm.tilesR * TC_M, RCc = dm.tilesC * TC_N;
  // stage enumeration (thread 0): chunk ch, term, k block, A block [s0, s1], B range [t0, t1]
  struct Stage { int ch, term, kbk, s0, s1, t0, t1; };
  auto chunk_range = [&](int ch, int& d0, int& d1, int& slo, int& shi) {
    d0 = DLO + ch * TC_GCH;
    d1 = min(d0 + TC_GCH - 1, DHI);
    slo = max(SA0, d0 - (SB1 - 1));
    shi = min(S - 1, d1 - SB0);
  };
  auto chunk_empty = [&](int ch) {  // no slice pair reaches the chunk's groups
    int d0, d1, slo, shi;
    chunk_range(ch, d0, d1, slo, shi);
    return slo > shi;
  };
  auto set_ranges = [&](Stage& g) {
    int d0, d1, slo, shi;
    chunk_range(g.ch, d0, d1, slo, shi);
    g.s1 = min(g.s0 + TC_SBK - 1, shi);
    g.t0 = max(SB0, d0 - g.s1);
    g.t1 = min(SB1 - 1, d1 - g.s0);
  };
  // first stage of the first non-empty chunk at or after ch (false: none)
  auto chunk_start = [&](Stage& g, int ch) -> bool {
    while (ch < NCH && chunk_empty(ch)) ++ch;
    if (ch >= NCH) return false;
    int d0, d1, slo, shi;
    chunk_range(ch, d0, d1, slo, shi);
    g.ch = ch; g.term = 0; g.kbk = 0; g.s0 = slo;
    set_ranges(g);
    return true;
  };
  // advance a stage cursor; returns false past the last stage
  auto next_stage = [&](Stage& g) -> bool {
    int d0, d1, slo, shi;
    chunk_range(g.ch, d0, d1, slo, shi);
    g.s0 += TC_SBK;
    if (g.s0 > shi) {
      g.s0 = slo;
      if (++g.kbk >= nkb) {
        g.kbk = 0;
        if (++g.term >= 2) return chunk_start(g, g.ch + 1);
      }
    }
    set_ranges(g);
    return true;
  };
  // bulk copies of stage g into buffer b (A tiles at [0, 64 KB), B tiles after)
  auto load_stage = [&](const Stage& g, int b) {
    const int ap = g.term, bp = plane == 0 ? (g.term == 0 ? 0 : 2) : (g.term == 0 ? 1 : 0);
    const int8_t* Ap = Ab + (size_t)ap * S * a_s + ((size_t)rt * dm.kb + g.kbk) * TC_ATILE;
    const int8_t* Bp = Bb + (size_t)bp * S * b_s + ((size_t)ct * dm.kb + g.kbk) * TC_BTILE;
    const uint32_t bytes = (uint32_t)((g.s1 - g.s0 + 1) * TC_ATILE + (g.t1 - g.t0 + 1) * TC_BTILE);
    const uint32_t fb = tc_smem(&bar_full[b]);
    if (warp != TC_LOADER || !tc_elect()) return;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(bytes));
    int8_t* buf = tcs + (size_t)b * TC_STAGE;
    for (int s = g.s0; s <= g.s1; ++s)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       tc_smem(buf + (size_t)(s - g.s0) * TC_ATILE)),
                   "l"(Ap + (size_t)s * a_s), "n"(TC_ATILE), "r"(fb)
                   : "memory");
    int8_t* bbuf = buf + TC_SBK * TC_ATILE;
    for (int t = g.t0; t <= g.t1; ++t)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       tc_smem(bbuf + (size_t)(t - g.t0) * TC_BTILE)),
                   "l"(Bp + (size_t)t * b_s), "n"(TC_BTILE), "r"(fb)
                   : "memory");
  };
  Stage cur, nxt;        // cur: the stage whose MMAs are issued next; nxt: the next stage to load
  int i = 0;             // index of cur
  int nld = 0;           // stages loaded so far (index of nxt)
  bool more = false;     // nxt valid
  uint32_t started = 0;  // bit j: group d0 + j of the current chunk received an MMA
  unsigned long long nmma = 0;  // MMAs this warp issued (profiling)
  // every warp follows the stage sequence (warp-uniform values, elect.sync-predicated issue): warp 0
  // also streams the tiles, TC_NSTG - 1 stages ahead; warp w issues the MMAs of its groups of the chunk
  auto consumer_sync = [&]() {  // the MMA warps only (the producer warp runs on its own)
    if (TC_PRODUCER) asm volatile("bar.sync 1, %0;\n" ::"n"(TC_WARPS * 32) : "memory");
    else __syncthreads();
  };
  if (TC_PRODUCER && warp == TC_LOADER) {
    // producer warp: keeps TC_NSTG stages in flight; a buffer is refilled as soon as the MMAs of
    // the stage that used it have completed (tcgen05.commit of every MMA warp on its "empty" barrier)
    if (chunk_start(nxt, 0)) {
      more = true;
      while (more) {
        if (nld >= TC_NSTG) tc_mbar_wait(tc_smem(&bar_empty[nld % TC_NSTG]), ((nld - TC_NSTG) / TC_NSTG) & 1);
        load_stage(nxt, nld % TC_NSTG);
        ++nld;
        more = next_stage(nxt);
      }
    }
    return;
  }
  const bool have = chunk_start(cur, 0);
  if (!TC_PRODUCER && have) {
    nxt = cur;
    more = true;
    for (int k = 0; k < TC_NSTG - 1 && more; ++k) {
      load_stage(nxt, nld % TC_NSTG);
      ++nld;
      more = next_stage(nxt);
    }
  }
  for (int ch = 0; ch < NCH; ++ch) {
    int d0, d1, slo, shi;
    chunk_range(ch, d0, d1, slo, shi);
    started = 0;
    __shared__ uint32_t s_started;
    if (tid == 0) s_started = 0;
    if (slo <= shi) {
      while (true) {
        const int b = i % TC_NSTG;
        tc_mbar_wait(tc_smem(&bar_full[b]), (i / TC_NSTG) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int8_t* buf = tcs + (size_t)b * TC_STAGE;
        const int8_t* bbuf = buf + TC_SBK * TC_ATILE;
        for (int s = cur.s0; s <= cur.s1; ++s) {
          const uint64_t da = tc_desc(tc_smem(buf + (size_t)(s - cur.s0) * TC_ATILE));
          const int dlo = max(d0 + warp * (TC_GCH / TC_WARPS), s + cur.t0),
                    dhi = min(min(d1, d0 + (warp + 1) * (TC_GCH / TC_WARPS) - 1), s + cur.t1);
          for (int d = dlo; d <= dhi; ++d) {
            const int t = d - s;
            const uint32_t acc_addr = tmem + (uint32_t)((d - d0) * TC_N);
            const uint64_t db = tc_desc(tc_smem(bbuf + (size_t)(t - cur.t0) * TC_BTILE));
            const uint32_t acc = (started >> (d - d0)) & 1u;
            if (!(dm.bisect & 1))
              asm volatile(
                  "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                  "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(acc_addr),
                  "l"(da), "l"(db), "r"(IDESC), "r"(acc));
            started |= 1u << (d - d0);
            ++nmma;
          }
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                tc_smem(&bar_empty[b])));
        // prefetch stage i + TC_NSTG - 1 into the buffer of stage i - 1 once that stage's MMAs released
        // it (the MMAs of stage i are queued behind them, so the tensor pipe does not drain)
        if (!TC_PRODUCER && more) {
          if (nld >= TC_NSTG) tc_mbar_wait(tc_smem(&bar_empty[nld % TC_NSTG]), ((nld - TC_NSTG) / TC_NSTG) & 1);
          load_stage(nxt, nld % TC_NSTG);
          ++nld;
          more = next_stage(nxt);
        }
        Stage tmp = cur;
        const bool has_next = next_stage(tmp);
        const bool last_of_chunk = !has_next || tmp.ch != ch;
        ++i;
        if (has_next) cur = tmp;
        if (last_of_chunk) {
          tc_mbar_wait(tc_smem(&bar_empty[b]), ((i - 1) / TC_NSTG) & 1);  // every MMA of the chunk is done
          break;
        }
      }
    }
    if (lane == 0) atomicOr(&s_started, started);
    consumer_sync();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t stg = s_started;
    if constexpr (TC_PACKED) {
      // drain: warp w owns TMEM lanes 32 w .. + 31 (rows); the chunk's groups are combined into
      // sum_j g_j 2^(8 j) (|g_j| < 2^30, TC_GCH <= 4: below 2^55) and stored as one int64 per entry
      static_assert(TC_WARPS == 4 && TC_GCH <= 4 && TC_SB == 8, "packed drain: one owner per entry, 32-bit span");
      const int row = rt * TC_M + 32 * warp + lane;
      int64_t* g64 = (int64_t*)Gb + (((size_t)plane * NCH + ch) * RCc + (size_t)ct * TC_N) * RRr + row;
#pragma unroll 1
      for (int h = 0; h < TC_N / 32; ++h) {
        int64_t acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0;
        for (int d = d0; d <= d1; ++d) {
          if (!(((stg >> (d - d0)) & 1u) && !(dm.bisect & 2))) continue;  // warp-uniform
          uint32_t v[32];
          const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)((d - d0) * TC_N + 32 * h);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(addr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n");
          const int sh = 8 * (d - d0);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] += (int64_t)(int32_t)v[j] << sh;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) g64[(size_t)(32 * h + j) * RRr] = acc[j];
      }
    } else {
    // drain: warp w reads TMEM lanes 32 (w % 4) .. + 31 (rows) of groups d0 + w / 4, + 2, ...
    const int row = rt * TC_M + 32 * (warp & 3) + lane;
    for (int d = d0 + (warp >> 2); d <= d1; d += TC_WARPS / 4) {
      int32_t* g = Gb + (((size_t)plane * NG + (d - DLO)) * RCc + (size_t)ct * TC_N) * RRr + row;
#pragma unroll
      for (int h = 0; h < TC_N / 32; ++h) {
        uint32_t v[32];
        if (((stg >> (d - d0)) & 1u) && !(dm.bisect & 2)) {
          const uint32_t addr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((d - d0) * TC_N + 32 * h);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(addr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) g[(size_t)(32 * h + j) * RRr] = (int32_t)v[j];
      }
    }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    consumer_sync();  // the next chunk's MMAs overwrite the accumulators
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
  if (dm.cnt && lane == 0 && nmma) atomicAdd(&dm.cnt[CNT_TC_MAC], nmma * (unsigned long long)(TC_M * TC_N * TC_K));
}

// ---------------------------------------------------------------------------- epilogue
// One thread per output entry: group sums -> LG + 2 int64 digit columns (column d / 4 of the
// product, shifted by 7 (d % 4) bits) -> gemm_t_store (the IMAD path's rounding and store).
template <int L, int LG, int ZOUT, int LOUT>
__global__ void __launch_bounds__(256) k_tc_epi(const GemmT* items, int first, TcDims dm) {
  constexpr int DLO = tc_dlo<LG>(), NG = tc_ng<LG>();
  const int item = first + blockIdx.y;
  const GemmT it = items[item];
  if (it.rows <= 0 || it.cols <= 0) return;
  const bool percol = it.eBcols != nullptr;
  const int64_t eC = percol ? 0 : (it.eCout ? *it.eCout : *it.eA + *it.eB + it.ghead);
  const int g = percol ? it.ghead : (int)(eC - (*it.eA + *it.eB));
  if (!percol && it.eCwrite && blockIdx.x == 0 && threadIdx.x == 0) *it.eCwrite = eC;
  const int ncols = it.ncols_dev ? min(*it.ncols_dev, it.cols) : it.cols;
  const int RRr = dm.tilesR * TC_M, RCc = dm.tilesC * TC_N;
  const int32_t* Gb = (int32_t*)((char*)dm.G + blockIdx.y * dm.g_item);
  int zbad = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < it.rows * ncols; t += gridDim.x * blockDim.x) {
    const int r = t % it.rows, c = t / it.rows;
    if (it.upper && r > c) continue;
    int64_t acc[2][LG + 4];
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
#pragma unroll
      for (int j = 0; j < LG + 4; ++j) acc[ri][j] = 0;
      if constexpr (TC_PACKED) {
        // chunk sums v = sum_j g_j 2^(8 j) at bit 8 d0 of the product: low 28 bits and the rest
        // go to two adjacent digit columns (each term < 2^55 after its shift of < 28 bits)
        constexpr int NCH = (NG + TC_GCH - 1) / TC_GCH;
        const int64_t* G64 = (const int64_t*)Gb;
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
          const int bit = 8 * (DLO + q * TC_GCH), col = bit / 28 - (LG - 2), sh = bit - 28 * (bit / 28);
          const int64_t v = G64[(((size_t)ri * NCH + q) * RCc + c) * RRr + r];
          const int64_t hi = v >> 28, lo = v - (hi << 28);
          acc[ri][col] += lo << sh;
          acc[ri][col + 1] += hi << sh;
        }
        acc[ri][LG + 2] += acc[ri][LG + 3] * ((int64_t)1 << 28);
      } else {
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const int d = DLO + q;
          const int64_t v = Gb[(((size_t)ri * NG + q) * RCc + c) * RRr + r];
          if (TC_SB == 7) acc[ri][d / 4 - (LG - 2)] += v * ((int64_t)1 << (7 * (d % 4)));
          else acc[ri][(8 * d) / 28 - (LG - 2)] += v * ((int64_t)1 << (8 * d - 28 * ((8 * d) / 28)));
        }
      }
      acc[ri][LG + 1] += acc[ri][LG + 2] * ((int64_t)1 << 28);  // column 2LG (the top slices' carry)
    }
    int64_t ar[LG + 2], ai[LG + 2];
#pragma unroll
    for (int j = 0; j < LG + 2; ++j) { ar[j] = acc[0][j]; ai[j] = acc[1][j]; }
    gemm_t_store<LOUT, LG, ZOUT>(it, r, c, it.colmap ? it.colmap[c] : c, ar, ai, g, eC, percol, false, zbad);
  }
  if (zbad && it.zerr) atomicOr(it.zerr, 2);
}

// ---------------------------------------------------------------------------- launch

template <int LG, int SA0, int SB0, int SB1>
constexpr size_t tc_mma_smem() { return (size_t)TC_NSTG * TC_STAGE; }

// C = op(A) B for n items (GemmT on the device) on the tensor cores.  Z / NZA / NZB: known-zero
// top digits of B / low digits of A / low digits of B (their slices are not multiplied).
// Returns the number of kernel launches, or -1 when the scratch cannot be allocated (the
// caller then runs the IMAD kernel).
// LG > L: the operands' LG - L digits below the stored ones are zero (then NZA, NZB >= LG - L);
// LOUT: digits of C (default L; LOUT = LG keeps the product's full LG-digit rounding).
template <int L, int LG, int Z, int NZA, int NZB, int ZOUT, int LOUT = L>
inline int launch_gemm_tc(const GemmT* d_items, int n, int maxR, int maxC, int maxK, cudaStream_t st) {
  static_assert(LG <= L || (NZA >= LG - L && NZB >= LG - L), "zero-padded digits must be skipped");
  static_assert(LOUT >= LG || LOUT == L, "output digits");
  constexpr int S = tc_ns<LG>(), NG = tc_ng<LG>();
  constexpr int SA0 = tc_slice_lo(NZA), SB0 = tc_slice_lo(NZB), SB1 = tc_slice_hi<LG>(Z);
  TcDims dm;
  static const int bis = getenv("MPS_TC_BISECT") ? atoi(getenv("MPS_TC_BISECT")) : 0;
  dm.bisect = bis;
  dm.cnt = prof_counts();
  dm.tilesR = (maxR + TC_M - 1) / TC_M;
  dm.tilesC = (maxC + TC_N - 1) / TC_N;
  dm.kb = (maxK + TC_K - 1) / TC_K;
  dm.a_item = align_up((size_t)2 * S * dm.tilesR * dm.kb * TC_ATILE);
  dm.b_item = align_up((size_t)3 * S * dm.tilesC * dm.kb * TC_BTILE);
  dm.g_item = TC_PACKED ? align_up((size_t)2 * ((NG + TC_GCH - 1) / TC_GCH) * dm.tilesC * TC_N * dm.tilesR * TC_M * 8)
                        : align_up((size_t)2 * NG * dm.tilesC * TC_N * dm.tilesR * TC_M * 4);
  const size_t per = dm.a_item + dm.b_item + dm.g_item;
  const size_t budget = (size_t)3 << 30;
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>(n, budget / per));
  char* scr = (char*)tc_scratch(per * chunk, st);
  if (!scr) return -1;
  dm.A = (int8_t*)scr;
  dm.B = (int8_t*)(scr + dm.a_item * chunk);
  dm.G = (int32_t*)(scr + (dm.a_item + dm.b_item) * chunk);
  constexpr size_t smem = tc_mma_smem<LG, SA0, SB0, SB1>();
  smem_optin((const void*)k_tc_mma<LG, SA0, SB0, SB1>, (int)smem);
  static const bool dbg = getenv("MPS_TC_DEBUG") != nullptr;  // sync + check after every launch
  auto check = [&](const char* what) {
    if (!dbg) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "tc L=%d LG=%d Z=%d NZA=%d NZB=%d: %s n=%d chunk=%d R=%d C=%d K=%d: %s\n", L, LG, Z, NZA, NZB, what, n,
            chunk, maxR, maxC, maxK, cudaGetErrorString(e));
  };
  int nl = 0;
  for (int f = 0; f < n; f += chunk) {
    const int cnt = std::min(chunk, n - f);
    k_tc_slice_a<L, LG><<<dim3(dm.tilesR * dm.kb, 2, cnt), 256, 0, st>>>(d_items, f, dm);
    check("slice_a");
    k_tc_slice_b<L, LG><<<dim3(dm.tilesC * dm.kb, 2, cnt), 256, 0, st>>>(d_items, f, dm);
    check("slice_b");
    prof_mark(PROF_TCMMA, 1, st);
    k_tc_mma<LG, SA0, SB0, SB1><<<dim3(dm.tilesR * dm.tilesC * 2, cnt), TC_THREADS, smem, st>>>(d_items, f, dm);
    prof_mark(PROF_TCMMA, 0, st);
    check("mma");
    const int ne = dm.tilesR * TC_M * dm.tilesC * TC_N;
    k_tc_epi<L, LG, ZOUT, LOUT><<<dim3(std::min(1024, (ne + 255) / 256), cnt), 256, 0, st>>>(d_items, f, dm);
    check("epi");
    nl += 4;
  }
  return nl;
}

}  // namespace mpsb
