// Kernel-level test surface: batched SVD of given matrices and elementwise device
// multiprecision ops (include/mps_b200.h "kernel test surface").  Same kernels as the
// gate update; only the input conversion differs.
#pragma once
#include "common.h"
#include "update.cuh"

namespace mpsb {

// column-major M x N complex records -> Jacobi layout (trans: A = Theta^H), block exponent
struct MatItem {
  const uint32_t* R;  // records
  int M, N, trans;    // source geometry
  int32_t* A; int64_t* eA; int64_t* eblk;
};

__global__ static void k_mat_exp(const MatItem* items, int RBr) {
  const MatItem it = items[blockIdx.y];
  const int n = it.M * it.N * 2;
  long long best = INT64_MIN;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    int64_t e = rec_get_exp(it.R + (size_t)t * RBr);
    if (e != INT64_MIN && e > best) best = e;
  }
  if (best != INT64_MIN) atomicMax((long long*)it.eblk, best);
}

template <int L, int NL>
__global__ void k_mat_conv(const MatItem* items, int RBr) {
  const MatItem it = items[blockIdx.y];
  const int n = it.M * it.N;
  int64_t E = *it.eblk;
  if (E == INT64_MIN) E = 0;
  const int Mj = it.trans ? it.N : it.M;  // Jacobi rows
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % it.M, c = t / it.M;
    for (int ri = 0; ri < 2; ++ri) {
      mpf<NL> v = mpf_from_record<NL>(it.R + (size_t)(2 * t + ri) * RBr, RBr - 4);
      int32_t d[L];
      mpf_to_fixed<NL, L>(v, E, d);
      if (!it.trans) {
        stfx<L>(it.A, Mj, c, ri, r, d);
      } else {
        if (ri == 1)
          for (int k = 0; k < L; ++k) d[k] = -d[k];
        stfx<L>(it.A, Mj, r, ri, c, d);
      }
    }
    if (!it.trans && r == 0) it.eA[c] = E;
    if (it.trans && c == 0) it.eA[r] = E;
  }
}

// Elementwise device mpf ops on records (unit tests of the scalar format against the oracle)
template <int L, int NL>
__global__ void k_debug_mpf(int op, int n, const uint32_t* a, const uint32_t* b, uint32_t* out, int RBr, int p) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    mpf<NL> x = mpf_from_record<NL>(a + (size_t)t * RBr, RBr - 4);
    mpf<NL> y = b ? mpf_from_record<NL>(b + (size_t)t * RBr, RBr - 4) : mpf_zero<NL>();
    mpf<NL> r;
    switch (op) {
      case 0: r = mpf_add(x, y); break;
      case 1: r = mpf_sub(x, y); break;
      case 2: r = mpf_mul(x, y); break;
      case 3: r = mpf_div(x, y); break;
      case 4: r = mpf_sqrt(x); break;
      case 5: r = mpf_rsqrt(x); break;
      case 6: r = mpf_recip(x); break;
      case 7: r = x; break;
      default: {  // 8: through the fixed-point format (exponent = x.e + 1) and back
        int32_t d[L];
        int64_t E = mpf_is_zero(x) ? 0 : x.e + 1;
        mpf_to_fixed<NL, L>(x, E, d);
        int64_t c[L];
        for (int k = 0; k < L; ++k) c[k] = d[k];
        r = mpf_from_cols<NL, L>(c, E - 28 * (int64_t)L);
      }
    }
    mpf_to_record<NL>(r, out + (size_t)t * RBr, RBr - 4, p);
  }
}

}  // namespace mpsb

namespace mpsb {

template <class T>
size_t svd_workspace(int M, int N, int batch) {
  constexpr int L = T::L, NL = T::NL;
  const int Mj = M >= N ? M : N, Nj0 = M >= N ? N : M;
  const int Nj = Nj0 + (Nj0 & 1);
  size_t per = align_up((size_t)Mj * Nj * 2 * L * 4) + align_up((size_t)Nj * Nj * 2 * L * 4) +
               align_up(8 * (size_t)Nj + 64) + align_up(sizeof(mpf<NL>) * (size_t)Nj * 4) +
               align_up(4 * (size_t)Nj / 2 * 33 * (L + 1)) + align_up(4 * (size_t)Nj * 3 + 64) + 512;
  return align_up(sizeof(MatItem) * batch) + align_up(sizeof(SvdItem<NL>) * batch) +
         align_up(sizeof(FinItem<NL>) * batch) + (size_t)batch * per + 4096;
}

// sigma: batch * min(M,N) records, descending.  dbg: batch*64 ints (rotations per sweep) or null.
template <class T>
int run_svd_batch(int p, int M, int N, int batch, const uint32_t* dR, uint32_t* dsig, int* dsweeps, int* ddbg,
                  void* ws, cudaStream_t st, std::vector<unsigned char>& hd) {
  constexpr int L = T::L, NL = T::NL;
  const int RBr = record_words(p);
  const bool trans = N > M;
  const int Mj = trans ? N : M, Nj0 = trans ? M : N;
  const int Nj = Nj0 + (Nj0 & 1);  // round-robin needs an even column count: pad a zero column
  char* base = (char*)ws;
  const size_t d_mat = 0, d_svd = align_up(sizeof(MatItem) * batch),
               d_fin = d_svd + align_up(sizeof(SvdItem<NL>) * batch),
               d_end = d_fin + align_up(sizeof(FinItem<NL>) * batch);
  hd.assign(d_end, 0);
  MatItem* hm = (MatItem*)(hd.data() + d_mat);
  SvdItem<NL>* hs = (SvdItem<NL>*)(hd.data() + d_svd);
  FinItem<NL>* hf = (FinItem<NL>*)(hd.data() + d_fin);
  char* items = base + d_end;
  const size_t per = (svd_workspace<T>(M, N, batch) - d_end - 4096) / batch;
  cudaMemsetAsync(items, 0, per * batch, st);
  for (int b = 0; b < batch; ++b) {
    char* ib = items + (size_t)b * per;
    int32_t* A = (int32_t*)ib;
    int32_t* V = (int32_t*)(ib + align_up((size_t)Mj * Nj * 2 * L * 4));
    char* sm = (char*)V + align_up((size_t)Nj * Nj * 2 * L * 4);
    int64_t* eA = (int64_t*)sm;
    int64_t* eblk = eA + Nj;
    int* ip = (int*)(eblk + 1);
    long long* rots = (long long*)(eblk + 4);
    mpf<NL>* alpha = (mpf<NL>*)(sm + align_up(8 * (size_t)Nj + 64));
    mpf<NL>* gam = alpha + Nj;
    mpf<NL>* inv_sig = gam + Nj;
    mpf<NL>* lam = inv_sig + Nj;
    int32_t* coef = (int32_t*)((char*)alpha + align_up(sizeof(mpf<NL>) * (size_t)Nj * 4));
    int* rot = (int*)((char*)coef + align_up(4 * (size_t)Nj / 2 * 33 * (L + 1)));
    int* negl = rot + Nj / 2;
    int* ord = negl + Nj;
    int* syncp = (int*)align_up((size_t)(ord + Nj) + 64, 16);
    mpf<NL>* zbuf = (mpf<NL>*)(syncp + 16);
    hm[b] = MatItem{dR + (size_t)b * M * N * 2 * RBr, M, N, trans ? 1 : 0, A, eA, eblk};
    SvdItem<NL> si = {};
    si.M = Mj; si.N = Nj; si.A = A; si.eA = eA; si.V = V; si.alpha = alpha; si.gam = gam; si.coef = coef;
    si.dbg = ddbg ? ddbg + 64 * b : nullptr;
    si.rot = rot; si.negl = negl; si.status = ip; si.sweeps = dsweeps + b; si.rotations = rots;
    si.sync = syncp; si.zbuf = zbuf; si.phase_cycles = nullptr; si.A0 = nullptr; si.eA0 = nullptr; si.eV = nullptr; si.evals = rots + 1;
    si.cexp = use_cert() ? syncp + 4 : nullptr;  // syncp[4..9] (zbuf at syncp + 16)
    hs[b] = si;
    FinItem<NL> fi;
    std::memset(&fi, 0, sizeof(fi));
    fi.M = Mj; fi.N = Nj; fi.trans = trans; fi.A = A; fi.eA = eA; fi.V = V; fi.alpha = alpha;
    fi.chi_max = Nj; fi.thr = mpf_host_from_double<NL>(0.0); fi.ord = ord; fi.inv_sig = inv_sig; fi.lam = lam;
    fi.k_out = ip + 1; fi.status = ip + 2; fi.svd_status = ip; fi.sigma_rec = dsig + (size_t)b * Nj0 * RBr; fi.nsig = Nj0;
    hf[b] = fi;
  }
  cudaMemcpyAsync(base, hd.data(), d_end, cudaMemcpyHostToDevice, st);
  int nl = 0;
  // eblk = INT64_MIN: eA[Nj] slot follows eA; set via the exponent-init kernel on each item
  for (int b = 0; b < batch; ++b) {
    k_init_exp<<<1, 32, 0, st>>>(hm[b].eblk, 1);
    ++nl;
  }
  dim3 g(std::max(1, std::min(64, (M * N + 255) / 256)), batch);
  k_mat_exp<<<g, 256, 0, st>>>((const MatItem*)(base + d_mat), RBr); ++nl;
  k_mat_conv<L, NL><<<g, 256, 0, st>>>((const MatItem*)(base + d_mat), RBr); ++nl;
  launch_jacobi<L, NL>((const SvdItem<NL>*)(base + d_svd), batch, jacobi_cluster_size(batch, Nj, jacobi_min_ctas<L>() * 148), st); ++nl;
  // the sigma records of the padded zero column are not part of the output
  k_finalize<L, NL><<<batch, NTHR, sizeof(mpf<NL>) * (size_t)Nj, st>>>((const FinItem<NL>*)(base + d_fin), RBr, p);
  ++nl;
  return nl;
}

template <class T>
void run_debug_mpf(int p, int op, int n, const uint32_t* a, const uint32_t* b, uint32_t* out, cudaStream_t st) {
  k_debug_mpf<T::L, T::NL><<<std::max(1, std::min(1024, (n + 127) / 128)), 128, 0, st>>>(op, n, a, b, out, record_words(p), p);
}

}  // namespace mpsb
