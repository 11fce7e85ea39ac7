// configs[1] batch entry: every item is a two-site update with bond dims (chi, chi, chi),
// delegated to the generic driver of update.cuh.
#pragma once
#include "update.cuh"

namespace mpsb {

inline std::vector<Upd2Args> batch_args(int p, int chi, int chi_max, int batch, const uint32_t* A, const uint32_t* B,
                                        const uint32_t* lam_l, const uint32_t* lam_m, const uint32_t* lam_r,
                                        const uint32_t* U, const BatchOut& out) {
  const int RBr = record_words(p);
  const size_t cplx = 2 * (size_t)RBr;
  std::vector<Upd2Args> v(batch);
  for (int b = 0; b < batch; ++b) {
    Upd2Args g;
    std::memset(&g, 0, sizeof(g));
    g.chiL = g.chiM = g.chiR = chi;
    g.chi_max = chi_max;
    g.GL = A + (size_t)b * 2 * chi * chi * cplx;
    g.GR = B + (size_t)b * 2 * chi * chi * cplx;
    g.lamL = lam_l ? lam_l + (size_t)b * chi * RBr : nullptr;
    g.lamM = lam_m ? lam_m + (size_t)b * chi * RBr : nullptr;
    g.lamR = lam_r ? lam_r + (size_t)b * chi * RBr : nullptr;
    g.U = U + (size_t)b * 16 * cplx;
    g.GL_out = out.A_out ? out.A_out + (size_t)b * 2 * chi * chi_max * cplx : nullptr;
    g.GR_out = out.B_out ? out.B_out + (size_t)b * 2 * chi_max * chi * cplx : nullptr;
    g.out_ld = chi_max;
    g.lam_out = out.lam ? out.lam + (size_t)b * chi_max * RBr : nullptr;
    g.sigma_out = out.sigma ? out.sigma + (size_t)b * 2 * chi * RBr : nullptr;
    g.k_out = out.k ? out.k + b : nullptr;
    g.sweeps_out = out.sweeps ? out.sweeps + b : nullptr;
    g.status_out = out.status ? out.status + b : nullptr;
    g.theta_dbg = out.theta_dbg ? out.theta_dbg + (size_t)b * 4 * chi * chi * cplx : nullptr;
    v[b] = g;
  }
  return v;
}

template <class T>
int launch_update2_batch(int p, int chi, int chi_max, int batch, double thr, const uint32_t* A,
                         const uint32_t* B, const uint32_t* lam_l, const uint32_t* lam_m,
                         const uint32_t* lam_r, const uint32_t* U, const BatchOut& out, void* ws,
                         cudaStream_t st, std::vector<unsigned char>& hostdesc) {
  std::vector<Upd2Args> v = batch_args(p, chi, chi_max, batch, A, B, lam_l, lam_m, lam_r, U, out);
  return run_update2<T>(p, thr, v.data(), batch, ws, st, hostdesc);
}

template <class T>
size_t update2_workspace(int chi, int batch) {
  Upd2Args g;
  std::memset(&g, 0, sizeof(g));
  g.chiL = g.chiM = g.chiR = chi;
  g.chi_max = chi;
  std::vector<Upd2Args> v(batch, g);
  return upd2_workspace<T>(v.data(), batch);
}

}  // namespace mpsb
