// C ABI (include/mps_b200.h): validation, tier dispatch, host<->device marshalling.
// Every computation of the method runs in the kernels of kernels.cuh; this file only
// moves records, checks arguments and sequences launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <tuple>
#include <mutex>
#include <vector>

#include "../../include/mps_b200.h"
#include "common.h"

using namespace mpsb;

static thread_local int g_last_launches = 0;

// ---- kernel event profiling (bench.py): accumulated ms per kernel class
namespace {
struct Prof {
  bool on = false;
  unsigned long long* counts = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[PROF_N];
  std::vector<cudaEvent_t> pending_begin[PROF_N];
} g_prof;
}  // namespace

cudaError_t mpsb::smem_optin(const void* kern, int bytes) {
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, int>> done;  // (kernel, device, bytes)
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& d : done)
    if (std::get<0>(d) == kern && std::get<1>(d) == dev && std::get<2>(d) >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(kern, dev, bytes);
  return e;
}

void* mpsb::tc_scratch(size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  struct Buf { int dev; cudaStream_t st; void* p; size_t n; };
  static std::vector<Buf> bufs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  for (auto& b : bufs) {
    if (b.dev != dev || b.st != st) continue;
    if (b.n >= bytes) return b.p;
    cudaStreamSynchronize(st);  // the previous buffer may still be in use on this stream
    cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    b.n = bytes;
    return b.p;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  bufs.push_back({dev, st, p, bytes});
  return p;
}

bool mpsb::tc_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MPS_TC");
    on = e ? (atoi(e) != 0) : 1;
  }
  return on != 0;
}

unsigned long long* mpsb::prof_counts() { return g_prof.on ? g_prof.counts : nullptr; }

void mpsb::prof_mark(int which, int begin, cudaStream_t st) {
  if (!g_prof.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  if (begin) {
    g_prof.pending_begin[which].push_back(e);
  } else if (!g_prof.pending_begin[which].empty()) {
    g_prof.ev[which].push_back({g_prof.pending_begin[which].back(), e});
    g_prof.pending_begin[which].pop_back();
  }
}

extern "C" {

size_t mps_record_bytes(int p) { return 16 + 4 * (size_t)((p + 31) / 32); }

const char* mps_strerror(int s) {
  switch (s) {
    case MPS_OK: return "ok";
    case MPS_EINVAL: return "invalid argument";
    case MPS_ENOTUNITARY: return "gate is not unitary at working precision";
    case MPS_ENOCONV: return "Jacobi SVD did not converge";
    case MPS_EZEROBOND: return "all Schmidt coefficients below the truncation floor";
    case MPS_EOVERLAP: return "gates of a layer overlap";
    case MPS_EUNSUPPORTED: return "unsupported precision or size";
    case MPS_ENOMEM: return "out of device memory";
    case MPS_ECUDA: return "CUDA error (or no CUDA device)";
    case MPS_ENCCL: return "NCCL error";
    case MPS_ETOOBIG: return "state too large";
    default: return "unknown status";
  }
}

int mps_max_chi(void) { return MAX_CHI; }

int mps_profile_enable(int on) {
  for (int k = 0; k < PROF_N; ++k) {
    for (auto& pr : g_prof.ev[k]) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (auto& e : g_prof.pending_begin[k]) cudaEventDestroy(e);
    g_prof.ev[k].clear();
    g_prof.pending_begin[k].clear();
  }
  g_prof.on = on != 0;
  if (g_prof.on) {
    if (!g_prof.counts && cudaMalloc(&g_prof.counts, CNT_N * sizeof(unsigned long long)) != cudaSuccess) return MPS_ENOMEM;
    cudaMemset(g_prof.counts, 0, CNT_N * sizeof(unsigned long long));
  }
  return MPS_OK;
}

int mps_profile_counts_n(long long* out, int n) {
  if (!out || n < 1 || n > CNT_N || !g_prof.counts) return MPS_EINVAL;
  cudaDeviceSynchronize();
  unsigned long long h[CNT_N];
  if (cudaMemcpy(h, g_prof.counts, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return MPS_ECUDA;
  for (int i = 0; i < n; ++i) out[i] = (long long)h[i];
  return MPS_OK;
}
int mps_profile_counts(long long* out4) {
  if (!out4 || !g_prof.counts) return MPS_EINVAL;
  cudaDeviceSynchronize();
  unsigned long long h[4];
  if (cudaMemcpy(h, g_prof.counts, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return MPS_ECUDA;
  for (int i = 0; i < 4; ++i) out4[i] = (long long)h[i];
  return MPS_OK;
}

int mps_profile_query(int which, double* total_ms, int* launches) {
  if (which < 0 || which >= PROF_N || !total_ms || !launches) return MPS_EINVAL;
  double tot = 0;
  for (auto& pr : g_prof.ev[which]) {
    if (cudaEventSynchronize(pr.second) != cudaSuccess) return MPS_ECUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    tot += ms;
  }
  *total_ms = tot;
  *launches = (int)g_prof.ev[which].size();
  return MPS_OK;
}
int mps_last_launch_count(void) { return g_last_launches; }

size_t mps_update_batch_workspace(int p, int chi, int batch) {
  if (p < 64 || p > 512 || chi < 1 || chi > MAX_CHI || batch < 1) return 0;
  return p <= 280 ? update2_workspace<Tier280>(chi, batch) : update2_workspace<Tier512>(chi, batch);
}

int mps_update_batch_device(int p, int chi, int chi_max, int batch, double thr, const void* dA,
                            const void* dB, const void* dlam_l, const void* dlam_m, const void* dlam_r,
                            const void* dU, void* dsigma, int* dk_out, void* dA_out, void* dB_out,
                            void* dlam_out, int* dsweeps, void* dws, void* stream) {
  if (p < 64 || p > 512 || chi < 1 || chi > MAX_CHI || batch < 1 || chi_max < 1 || !dA || !dB || !dU || !dws)
    return MPS_EINVAL;
  if (thr <= 0) thr = std::ldexp(1.0, -((p + 1) / 2));
  BatchOut o{(uint32_t*)dsigma, dk_out, (uint32_t*)dA_out, (uint32_t*)dB_out, (uint32_t*)dlam_out, dsweeps, nullptr, nullptr};
  std::vector<unsigned char> hd;
  cudaStream_t st = (cudaStream_t)stream;
  int nl;
  if (p <= 280)
    nl = launch_update2_batch<Tier280>(p, chi, chi_max, batch, thr, (const uint32_t*)dA, (const uint32_t*)dB,
                                       (const uint32_t*)dlam_l, (const uint32_t*)dlam_m, (const uint32_t*)dlam_r,
                                       (const uint32_t*)dU, o, dws, st, hd);
  else
    nl = launch_update2_batch<Tier512>(p, chi, chi_max, batch, thr, (const uint32_t*)dA, (const uint32_t*)dB,
                                       (const uint32_t*)dlam_l, (const uint32_t*)dlam_m, (const uint32_t*)dlam_r,
                                       (const uint32_t*)dU, o, dws, st, hd);
  // the host descriptor buffer must outlive the async copy
  cudaError_t e = cudaGetLastError();  // launch errors first (not sticky)
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  else cudaStreamSynchronize(st);
  g_last_launches = nl;
  return e == cudaSuccess ? MPS_OK : MPS_ECUDA;
}

int mps_bench_update_batch(int p, int chi, int chi_max, int batch, double thr, const void* A, const void* B,
                           const void* lam_l, const void* lam_m, const void* lam_r, const void* U, void* sigma,
                           int* k_out, void* A_out, void* B_out, void* lam_out, int* sweeps, void* theta_debug,
                           void* stream) {
  if (p < 64 || p > 512 || chi < 1 || chi > MAX_CHI || batch < 1 || chi_max < 1 || !A || !B || !U)
    return MPS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MPS_ECUDA;
  if (thr <= 0) thr = std::ldexp(1.0, -((p + 1) / 2));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t rb = mps_record_bytes(p), cb = 2 * rb;
  const size_t nA = (size_t)batch * 2 * chi * chi * cb;
  const size_t nLam = (size_t)batch * chi * rb;
  const size_t nU = (size_t)batch * 16 * cb;
  const size_t nSig = (size_t)batch * 2 * chi * rb;
  const size_t nAo = (size_t)batch * 2 * chi * chi_max * cb;
  const size_t nLo = (size_t)batch * chi_max * rb;
  const size_t nTh = (size_t)batch * 4 * chi * chi * cb;
  // The batch is processed in chunks so that the host<->device copies of one chunk overlap the
  // kernels of another (copy-in stream -> compute on st -> copy-out stream, ordered by events):
  // chunks of 592 items (four waves of the one-CTA-per-SM kernels on 148 SMs, two of the
  // two-CTA-per-SM ones), so the chunked launches fill the same number of waves as one launch of the
  // whole batch (1024 = 592 + 432: 4 + 3 waves); smaller chunks overlap more of the copies but run
  // the kernels less efficiently (296-item chunks: 1.39 instead of 1.28 ms per item, measured).  One workspace,
  // sized for the largest chunk, serves all chunks (they compute one after the other on st).
  // MPS_E2E_CHUNK=<items> overrides the chunk size (0: one chunk).
  static const int chunk_env = getenv("MPS_E2E_CHUNK") ? atoi(getenv("MPS_E2E_CHUNK")) : -1;
  int chunk = chunk_env > 0 ? chunk_env : (chunk_env == 0 || batch <= 592 || theta_debug ? batch : 592);
  chunk = std::min(chunk, batch);
  const int nchunks = (batch + chunk - 1) / chunk;
  const size_t ws = mps_update_batch_workspace(p, chi, chunk);
  size_t tot = 0;
  auto slot = [&](size_t n) { size_t o = tot; tot += align_up(n); return o; };
  size_t oA = slot(nA), oB = slot(nA), oll = slot(lam_l ? nLam : 0), olm = slot(lam_m ? nLam : 0),
         olr = slot(lam_r ? nLam : 0), oU = slot(nU), oS = slot(nSig), oK = slot(4 * (size_t)batch),
         oAo = slot(nAo), oBo = slot(nAo), oLo = slot(nLo), oSw = slot(4 * (size_t)batch),
         oTh = slot(theta_debug ? nTh : 0), oWs = slot(ws);
  // one grow-only device arena reused across calls (a cudaMalloc / cudaFree of tens of GB per
  // call cost ~1 s of the end-to-end time); calls are serialised by the mutex
  static std::mutex arena_mu;
  static char* arena = nullptr;
  static size_t arena_sz = 0;
  static cudaStream_t s_in = nullptr, s_out = nullptr;
  std::lock_guard<std::mutex> lock(arena_mu);
  if (arena_sz < tot) {
    if (arena) cudaFree(arena);
    arena = nullptr;
    arena_sz = 0;
    if (cudaMalloc(&arena, tot) != cudaSuccess) return MPS_ENOMEM;
    arena_sz = tot;
  }
  if (nchunks > 1 && !s_in) {
    if (cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking) != cudaSuccess)
      return MPS_ECUDA;
  }
  char* d = arena;
  // per-item sizes (the arrays are item-major)
  const size_t iA = nA / batch, iLam = nLam / batch, iU = nU / batch, iSig = nSig / batch, iAo = nAo / batch,
               iLo = nLo / batch, iTh = nTh / batch;
  static const bool e2e_trace = getenv("MPS_E2E_TRACE") != nullptr;  // debug: per-chunk event times
  const unsigned evflags = e2e_trace ? cudaEventDefault : cudaEventDisableTiming;
  std::vector<cudaEvent_t> ev_in(nchunks), ev_done(nchunks), ev_out(nchunks);
  cudaStream_t cin = nchunks > 1 ? s_in : st, cout_ = nchunks > 1 ? s_out : st;
  cudaEvent_t ev_start = nullptr;
  if (nchunks > 1) {  // the copies start after the work already queued on st
    cudaEventCreateWithFlags(&ev_start, evflags);
    cudaEventRecord(ev_start, st);
    cudaStreamWaitEvent(cin, ev_start, 0);
    cudaStreamWaitEvent(cout_, ev_start, 0);
  }
  for (int c = 0; c < nchunks; ++c) {  // every host -> device copy is queued first
    const size_t f = (size_t)c * chunk, cnt = std::min<size_t>(chunk, batch - f);
    cudaMemcpyAsync(d + oA + f * iA, (const char*)A + f * iA, cnt * iA, cudaMemcpyHostToDevice, cin);
    cudaMemcpyAsync(d + oB + f * iA, (const char*)B + f * iA, cnt * iA, cudaMemcpyHostToDevice, cin);
    if (lam_l) cudaMemcpyAsync(d + oll + f * iLam, (const char*)lam_l + f * iLam, cnt * iLam, cudaMemcpyHostToDevice, cin);
    if (lam_m) cudaMemcpyAsync(d + olm + f * iLam, (const char*)lam_m + f * iLam, cnt * iLam, cudaMemcpyHostToDevice, cin);
    if (lam_r) cudaMemcpyAsync(d + olr + f * iLam, (const char*)lam_r + f * iLam, cnt * iLam, cudaMemcpyHostToDevice, cin);
    cudaMemcpyAsync(d + oU + f * iU, (const char*)U + f * iU, cnt * iU, cudaMemcpyHostToDevice, cin);
    if (nchunks > 1) {
      cudaEventCreateWithFlags(&ev_in[c], evflags);
      cudaEventCreateWithFlags(&ev_done[c], evflags);
      cudaEventCreateWithFlags(&ev_out[c], evflags);
      cudaEventRecord(ev_in[c], cin);
    }
  }
  std::vector<unsigned char> hd;
  int nl = 0;
  for (int c = 0; c < nchunks; ++c) {
    const size_t f = (size_t)c * chunk, cnt = std::min<size_t>(chunk, batch - f);
    if (nchunks > 1) cudaStreamWaitEvent(st, ev_in[c], 0);
    BatchOut o{(uint32_t*)(d + oS + f * iSig), (int*)(d + oK) + f, (uint32_t*)(d + oAo + f * iAo),
               (uint32_t*)(d + oBo + f * iAo), (uint32_t*)(d + oLo + f * iLo), (int*)(d + oSw) + f,
               theta_debug ? (uint32_t*)(d + oTh + f * iTh) : nullptr, nullptr};
    cudaMemsetAsync(d + oAo + f * iAo, 0, cnt * iAo, st);
    cudaMemsetAsync(d + oBo + f * iAo, 0, cnt * iAo, st);
    const uint32_t* ll = lam_l ? (const uint32_t*)(d + oll + f * iLam) : nullptr;
    const uint32_t* lm = lam_m ? (const uint32_t*)(d + olm + f * iLam) : nullptr;
    const uint32_t* lr = lam_r ? (const uint32_t*)(d + olr + f * iLam) : nullptr;
    if (p <= 280)
      nl += launch_update2_batch<Tier280>(p, chi, chi_max, (int)cnt, thr, (const uint32_t*)(d + oA + f * iA),
                                          (const uint32_t*)(d + oB + f * iA), ll, lm, lr,
                                          (const uint32_t*)(d + oU + f * iU), o, d + oWs, st, hd);
    else
      nl += launch_update2_batch<Tier512>(p, chi, chi_max, (int)cnt, thr, (const uint32_t*)(d + oA + f * iA),
                                          (const uint32_t*)(d + oB + f * iA), ll, lm, lr,
                                          (const uint32_t*)(d + oU + f * iU), o, d + oWs, st, hd);
    if (nchunks > 1) {
      cudaEventRecord(ev_done[c], st);
      cudaStreamWaitEvent(cout_, ev_done[c], 0);
    }
    if (theta_debug) cudaMemcpyAsync((char*)theta_debug + f * iTh, d + oTh + f * iTh, cnt * iTh, cudaMemcpyDeviceToHost, cout_);
    if (sigma) cudaMemcpyAsync((char*)sigma + f * iSig, d + oS + f * iSig, cnt * iSig, cudaMemcpyDeviceToHost, cout_);
    if (k_out) cudaMemcpyAsync(k_out + f, (int*)(d + oK) + f, 4 * cnt, cudaMemcpyDeviceToHost, cout_);
    if (A_out) cudaMemcpyAsync((char*)A_out + f * iAo, d + oAo + f * iAo, cnt * iAo, cudaMemcpyDeviceToHost, cout_);
    if (B_out) cudaMemcpyAsync((char*)B_out + f * iAo, d + oBo + f * iAo, cnt * iAo, cudaMemcpyDeviceToHost, cout_);
    if (lam_out) cudaMemcpyAsync((char*)lam_out + f * iLo, d + oLo + f * iLo, cnt * iLo, cudaMemcpyDeviceToHost, cout_);
    if (sweeps) cudaMemcpyAsync(sweeps + f, (int*)(d + oSw) + f, 4 * cnt, cudaMemcpyDeviceToHost, cout_);
    if (nchunks > 1) cudaEventRecord(ev_out[c], cout_);
  }
  g_last_launches = nl;
  cudaError_t e = cudaGetLastError();  // launch errors first (not sticky)
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && nchunks > 1) e = cudaStreamSynchronize(cout_);
  if (e == cudaSuccess && nchunks > 1) e = cudaStreamSynchronize(cin);
  if (nchunks > 1) {
    if (e2e_trace && e == cudaSuccess)
      for (int c = 0; c < nchunks; ++c) {
        float a = 0, b = 0, o = 0;
        cudaEventElapsedTime(&a, ev_start, ev_in[c]);
        cudaEventElapsedTime(&b, ev_start, ev_done[c]);
        cudaEventElapsedTime(&o, ev_start, ev_out[c]);
        fprintf(stderr, "e2e chunk %d: inputs on the device at %.1f ms, computed at %.1f ms, outputs on the host at %.1f ms\n", c, a, b, o);
      }
    for (int c = 0; c < nchunks; ++c) { cudaEventDestroy(ev_in[c]); cudaEventDestroy(ev_done[c]); cudaEventDestroy(ev_out[c]); }
    cudaEventDestroy(ev_start);
  }
  if (e != cudaSuccess) {
    fprintf(stderr, "mps_b200: CUDA error %s\n", cudaGetErrorString(e));
    return MPS_ECUDA;
  }
  if (!theta_debug && k_out) {
    for (int b = 0; b < batch; ++b)
      if (k_out[b] == 0) return MPS_EZEROBOND;
  }
  if (!theta_debug && sweeps) {
    for (int b = 0; b < batch; ++b)
      if (sweeps[b] > JACOBI_MAX_SWEEPS) return MPS_ENOCONV;
  }
  return MPS_OK;
}

int mps_svd_batch(int p, int M, int N, int batch, const void* A, void* sigma, int* sweeps, int* rot_per_sweep) {
  if (p < 64 || p > 512 || M < 1 || N < 1 || batch < 1 || !A || !sigma || std::min(M, N) > 2 * MAX_CHI ||
      std::max(M, N) > 4 * MAX_CHI)
    return MPS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MPS_ECUDA;
  const size_t rb = mps_record_bytes(p);
  const size_t nA = (size_t)batch * M * N * 2 * rb, nS = (size_t)batch * std::min(M, N) * rb;
  const size_t ws = p <= 280 ? svd_workspace<Tier280>(M, N, batch) : svd_workspace<Tier512>(M, N, batch);
  size_t tot = 0;
  auto slot = [&](size_t n) { size_t o = tot; tot += align_up(n); return o; };
  size_t oA = slot(nA), oS = slot(nS), oSw = slot(4 * (size_t)batch), oD = slot(256 * (size_t)batch), oW = slot(ws);
  char* d = nullptr;
  if (cudaMalloc(&d, tot) != cudaSuccess) return MPS_ENOMEM;
  cudaStream_t st = 0;
  cudaMemcpyAsync(d + oA, A, nA, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d + oD, 0, 256 * (size_t)batch, st);
  std::vector<unsigned char> hd;
  int nl = p <= 280 ? run_svd_batch<Tier280>(p, M, N, batch, (const uint32_t*)(d + oA), (uint32_t*)(d + oS),
                                             (int*)(d + oSw), (int*)(d + oD), d + oW, st, hd)
                    : run_svd_batch<Tier512>(p, M, N, batch, (const uint32_t*)(d + oA), (uint32_t*)(d + oS),
                                             (int*)(d + oSw), (int*)(d + oD), d + oW, st, hd);
  g_last_launches = nl;
  std::vector<int> sw(batch);
  cudaMemcpyAsync(sigma, d + oS, nS, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(sw.data(), d + oSw, 4 * (size_t)batch, cudaMemcpyDeviceToHost, st);
  if (rot_per_sweep) cudaMemcpyAsync(rot_per_sweep, d + oD, 256 * (size_t)batch, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaGetLastError();  // launch errors first (not sticky)
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    fprintf(stderr, "mps_b200: CUDA error %s\n", cudaGetErrorString(e));
    return MPS_ECUDA;
  }
  if (sweeps) std::memcpy(sweeps, sw.data(), 4 * (size_t)batch);
  for (int b = 0; b < batch; ++b)
    if (sw[b] > JACOBI_MAX_SWEEPS) return MPS_ENOCONV;
  return MPS_OK;
}

int mps_debug_mpf(int p, int op, int n, const void* a, const void* b, void* out) {
  if (p < 64 || p > 512 || n < 1 || op < 0 || op > 8 || !a || !out) return MPS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MPS_ECUDA;
  const size_t nb = (size_t)n * mps_record_bytes(p);
  char* d = nullptr;
  if (cudaMalloc(&d, 3 * align_up(nb)) != cudaSuccess) return MPS_ENOMEM;
  cudaMemcpy(d, a, nb, cudaMemcpyHostToDevice);
  if (b) cudaMemcpy(d + align_up(nb), b, nb, cudaMemcpyHostToDevice);
  uint32_t* o = (uint32_t*)(d + 2 * align_up(nb));
  if (p <= 280)
    run_debug_mpf<Tier280>(p, op, n, (const uint32_t*)d, b ? (const uint32_t*)(d + align_up(nb)) : nullptr, o, 0);
  else
    run_debug_mpf<Tier512>(p, op, n, (const uint32_t*)d, b ? (const uint32_t*)(d + align_up(nb)) : nullptr, o, 0);
  cudaError_t e = cudaMemcpy(out, o, nb, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? MPS_OK : MPS_ECUDA;
}

}  // extern "C"
