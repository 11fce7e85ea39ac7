// Host-side driver of the batched two-site gate update (BASELINE configs[1]):
// descriptors, workspace carving and the launch sequence
//   init -> prep_exp -> prep_conv -> gemm -> mix -> jacobi -> finalize -> split
// All launches go to one stream; nothing synchronises (the caller does).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "common.h"
#include "kernels.cuh"

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


// per-item workspace of one two-site update with bond dims (chi, chi, chi)
template <class T>
struct Ws2 {
  static constexpr int L = T::L, NL = T::NL;
  size_t o_LR, o_T, o_V, o_small, per_item;
  int chi, M, N;
  explicit Ws2(int chi_) : chi(chi_) {
    M = 2 * chi; N = 2 * chi;
    size_t mat = (size_t)M * N * 2 * L * 4;  // complex digits of an M x N matrix
    o_LR = 0;                                 // L (2chi x chi) + R (chi x 2chi) ; later A
    o_T = align_up(o_LR + mat);
    o_V = align_up(o_T + mat);
    o_small = align_up(o_V + mat);
    per_item = align_up(o_small + small_bytes());
  }
  size_t small_bytes() const {
    return 8 * 4 + 8 * (size_t)N /*eA*/ + sizeof(mpf<NL>) * (size_t)N * 4 /*alpha,gam,inv_sig,lam*/ +
           4 * (size_t)N / 2 * 9 * (L + 1) /*coef*/ + 4 * (size_t)N * 3 /*rot,negl,ord*/ + 512;
  }
};


// Launch the whole batched update for items [0, batch) using workspace ws (device)
// of size batch * Ws2::per_item + descriptor space.  Returns launches issued.
template <class T>
int launch_update2_batch(int p, int chi, int chi_max, int batch, double thr, const uint32_t* A,
                         const uint32_t* B, const uint32_t* lam_l, const uint32_t* lam_m,
                         const uint32_t* lam_r, const uint32_t* U, const BatchOut& out, void* ws,
                         cudaStream_t st, std::vector<unsigned char>& hostdesc) {
  constexpr int L = T::L, NL = T::NL;
  Ws2<T> w(chi);
  const int RBr = record_words(p);
  const int M = w.M, N = w.N;
  char* base = (char*)ws;
  // descriptor area at the front
  const size_t d_prep = 0;
  const size_t d_gemm = align_up(d_prep + sizeof(PrepItem) * 2 * batch);
  const size_t d_mix = align_up(d_gemm + sizeof(GemmItem) * batch);
  const size_t d_svd = align_up(d_mix + sizeof(MixItem) * batch);
  const size_t d_fin = align_up(d_svd + sizeof(SvdItem<NL>) * batch);
  const size_t d_end = align_up(d_fin + sizeof(FinItem<NL>) * batch);
  char* items = base + d_end;
  hostdesc.assign(d_end, 0);
  PrepItem* hp = (PrepItem*)(hostdesc.data() + d_prep);
  GemmItem* hg = (GemmItem*)(hostdesc.data() + d_gemm);
  MixItem* hm = (MixItem*)(hostdesc.data() + d_mix);
  SvdItem<NL>* hs = (SvdItem<NL>*)(hostdesc.data() + d_svd);
  FinItem<NL>* hf = (FinItem<NL>*)(hostdesc.data() + d_fin);
  const size_t cplx_rec = 2 * (size_t)RBr;  // words per complex record
  const mpf<NL> thr_m = mpf_host_from_double<NL>(thr);
  std::vector<int64_t*> eblocks;
  for (int b = 0; b < batch; ++b) {
    char* ib = items + (size_t)b * w.per_item;
    int32_t* Lf = (int32_t*)(ib + w.o_LR);
    int32_t* Rf = Lf + (size_t)2 * chi * chi * 2 * L;
    int32_t* Tf = (int32_t*)(ib + w.o_T);
    int32_t* Af = (int32_t*)(ib + w.o_LR);  // A reuses the L/R space (dead after the GEMM)
    int32_t* Vf = (int32_t*)(ib + w.o_V);
    char* sm = ib + w.o_small;
    int64_t* eL = (int64_t*)sm;
    int64_t* eR = eL + 1;
    int64_t* eT = eL + 2;
    long long* rots = (long long*)(eL + 3);
    int* ip = (int*)(sm + 32);
    int* status = ip;
    int* sweeps = ip + 1;
    int* fstatus = ip + 2;
    int* kscr = ip + 3;
    int64_t* eA = (int64_t*)(sm + 64);
    mpf<NL>* alpha = (mpf<NL>*)align_up((size_t)(eA + N), 16);
    mpf<NL>* gam = alpha + N;
    mpf<NL>* inv_sig = gam + N;
    mpf<NL>* lamm = inv_sig + N;
    int32_t* coef = (int32_t*)(lamm + N);
    int* rot = coef + (size_t)N / 2 * 9 * (L + 1);
    int* negl = rot + N / 2;
    int* ord = negl + N;
    const uint32_t* Ab = A + (size_t)b * 2 * chi * chi * cplx_rec;
    const uint32_t* Bb = B + (size_t)b * 2 * chi * chi * cplx_rec;
    const uint32_t* ll = lam_l ? lam_l + (size_t)b * chi * RBr : nullptr;
    const uint32_t* lm = lam_m ? lam_m + (size_t)b * chi * RBr : nullptr;
    const uint32_t* lr = lam_r ? lam_r + (size_t)b * chi * RBr : nullptr;
    hp[2 * b] = PrepItem{Ab, ll, lm, chi, chi, 0, Lf, eL};
    hp[2 * b + 1] = PrepItem{Bb, nullptr, lr, chi, chi, 1, Rf, eR};
    hg[b] = GemmItem{Lf, 2 * chi, eL, Rf, chi, eR, Tf, 2 * chi, eT, 2 * chi, 2 * chi, chi, 0};
    hm[b] = MixItem{Tf, 2 * chi, eT, U + (size_t)b * 16 * cplx_rec, 2, chi, chi, 0, Af, eA, M, N};
    SvdItem<NL> si;
    si.M = M; si.N = N; si.A = Af; si.eA = eA; si.V = Vf; si.alpha = alpha; si.gam = gam;
    si.coef = coef; si.rot = rot; si.negl = negl; si.status = status; si.sweeps = out.sweeps ? out.sweeps + b : sweeps;
    si.rotations = rots;
    si.dbg = nullptr;
    hs[b] = si;
    FinItem<NL> fi;
    std::memset(&fi, 0, sizeof(fi));
    fi.M = M; fi.N = N; fi.trans = 0; fi.A = Af; fi.eA = eA; fi.V = Vf; fi.alpha = alpha;
    fi.chi_max = chi_max; fi.thr = thr_m; fi.ord = ord; fi.inv_sig = inv_sig; fi.lam = lamm;
    fi.k_out = out.k ? out.k + b : kscr; fi.status = fstatus;
    fi.sigma_rec = out.sigma ? out.sigma + (size_t)b * N * RBr : nullptr;
    fi.nsig = N;
    fi.lam_rec = out.lam ? out.lam + (size_t)b * chi_max * RBr : nullptr;
    fi.GL = out.A_out ? out.A_out + (size_t)b * 2 * chi * chi_max * cplx_rec : nullptr;
    fi.GL_ld = chi_max; fi.lamL = ll; fi.chiL_out = chi;
    fi.GR = out.B_out ? out.B_out + (size_t)b * 2 * chi_max * chi * cplx_rec : nullptr;
    fi.GR_ld = chi_max; fi.lamR = lr; fi.chiR_out = chi;
    hf[b] = fi;
    eblocks.push_back(eL);
  }
  cudaMemcpyAsync(base, hostdesc.data(), d_end, cudaMemcpyHostToDevice, st);
  int nl = 0;
  prof_mark(PROF_CONTRACT, 1, st);
  k_init_exp_items<<<(batch + 255) / 256, 256, 0, st>>>(items + w.o_small, w.per_item, batch); ++nl;
  dim3 gp(std::max(1, std::min(64, (2 * chi * chi + 255) / 256)), 2 * batch);
  k_prep_exp<<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep), RBr); ++nl;
  k_prep_conv<L, NL><<<gp, 256, 0, st>>>((const PrepItem*)(base + d_prep), RBr); ++nl;
  dim3 gg(std::max(1, std::min(128, (4 * chi * chi + 127) / 128)), batch);
  k_gemm<L><<<gg, 128, 0, st>>>((const GemmItem*)(base + d_gemm)); ++nl;
  k_mix<L, NL><<<gg, 128, 16 * 2 * L * 4, st>>>((const MixItem*)(base + d_mix), RBr); ++nl;
  if (out.theta_dbg) {
    // emit Theta' of every item (column-major records) and stop
    for (int b = 0; b < batch; ++b) {
      const MixItem& mi = hm[b];
      k_fixed_to_records<L, NL><<<64, 256, 0, st>>>(mi.A, M, mi.eA, nullptr, M, N, 0,
                                                    out.theta_dbg + (size_t)b * M * N * cplx_rec, RBr, p);
      ++nl;
    }
    return nl;
  }
  prof_mark(PROF_CONTRACT, 0, st);
  prof_mark(PROF_JACOBI, 1, st);
  k_jacobi<L, NL><<<batch, NTHR, 0, st>>>((const SvdItem<NL>*)(base + d_svd)); ++nl;
  prof_mark(PROF_JACOBI, 0, st);
  prof_mark(PROF_FINALIZE, 1, st);
  size_t fsm = sizeof(mpf<NL>) * (size_t)N;
  k_finalize<L, NL><<<batch, NTHR, fsm, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p); ++nl;
  if (out.A_out || out.B_out) {
    dim3 gs(std::max(1, std::min(64, (4 * chi * chi_max + 255) / 256)), batch);
    k_split<L, NL><<<gs, 256, 0, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p); ++nl;
  }
  prof_mark(PROF_FINALIZE, 0, st);
  return nl;
}

template <class T>
size_t update2_workspace(int chi, int batch) {
  Ws2<T> w(chi);
  constexpr int NL = T::NL;
  size_t desc = align_up(sizeof(PrepItem) * 2 * batch) + align_up(sizeof(GemmItem) * batch) +
                align_up(sizeof(MixItem) * batch) + align_up(sizeof(SvdItem<NL>) * batch) +
                align_up(sizeof(FinItem<NL>) * batch) + 4096;
  return desc + (size_t)batch * w.per_item;
}

}  // namespace mpsb
