// The MPS state behind include/mps_b200.h (mps_init ... mps_stats): the on-device store
// of Eq. 1 in Vidal Gamma-lambda form and the host sequencing of gate updates.
// Every arithmetic step runs in the sm_100a kernels (update.cuh, query.cuh); this file only
// validates arguments, moves records and repacks updated tensors into the store.
//
// Store layout (device): site s holds [2][m_{s-1}][m_s] complex records packed at the
// current dims inside a buffer of capacity 2 cap_{s-1} cap_s; bond b holds m_b reals in a
// buffer of capacity cap_b = min(chi_max, 2^min(b+1, n-b-1)) (the Schmidt-rank bound).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mps_b200.h"
#include "common.h"
#include "tierops.h"
#include "update.cuh"

using namespace mpsb;

struct mps_state {
  int n = 0, p = 0, chi_max = 0, RBr = 0;
  // block (site-sharded) state: local sites are global [lo, lo+n) of ntot; the bonds
  // outside the block (lo-1 and lo+n-1) are external, with their Schmidt vectors mirrored
  int lo = 0, ntot = 0;
  bool has_l = false, has_r = false;
  int m_el = 1, m_er = 1, cap_el = 1, cap_er = 1;
  uint32_t* lam_el = nullptr;
  uint32_t* lam_er = nullptr;
  size_t rb = 0, cb = 0;
  double thr = 0;
  cudaStream_t st = 0;
  int sticky = MPS_OK;
  std::vector<int> m, cap;
  std::vector<uint32_t*> G, lam;
  const TierOps* ops = nullptr;
  void* ws = nullptr;
  size_t ws_sz = 0;
  char* tmp = nullptr;
  size_t tmp_sz = 0;
  int* dint = nullptr;  // 256 device ints
  std::vector<cudaStream_t> sub;  // side streams of batched three-site layers (created lazily)
  long long gates = 0, sweeps_total = 0;
  int last_sweeps = 0;
  int dl(int s) const { return s == 0 ? (has_l ? m_el : 1) : m[s - 1]; }
  int dr(int s) const { return s == n - 1 ? (has_r ? m_er : 1) : m[s]; }
  int capl(int s) const { return s == 0 ? (has_l ? cap_el : 1) : cap[s - 1]; }
  int capr(int s) const { return s == n - 1 ? (has_r ? cap_er : 1) : cap[s]; }
  // Schmidt vector left of site s / right of site s (null = the trivial [1] of a chain end)
  const uint32_t* lamL(int s) const { return s > 0 ? lam[s - 1] : (has_l ? lam_el : nullptr); }
  const uint32_t* lamR(int s) const { return s < n - 1 ? lam[s] : (has_r ? lam_er : nullptr); }
  int capR(int s) const { return s < n - 1 ? cap[s] : cap_er; }  // capacity of the bond right of s
};

namespace {

int cuda_ok(mps_state* s, cudaError_t e) {
  if (e == cudaSuccess) return MPS_OK;
  fprintf(stderr, "mps_b200: CUDA error %s\n", cudaGetErrorString(e));
  if (s) s->sticky = MPS_ECUDA;
  return MPS_ECUDA;
}

// Launch errors (a bad configuration, a missing shared-memory opt-in, a cluster that cannot
// be placed) are not sticky in the CUDA context and a later stream synchronisation does not
// report them: check cudaGetLastError before synchronising, and make either error sticky.
int sync_ok(mps_state* s, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_ok(s, e);
}

bool grow(void** buf, size_t* sz, size_t need) {
  if (*sz >= need) return true;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *sz = 0;
  if (cudaMalloc(buf, need) != cudaSuccess) return false;
  *sz = need;
  return true;
}

// host record of +1 / 0 at precision p
void host_record(int p, int one, std::vector<uint32_t>& out) {
  const int L = (p + 31) / 32;
  out.assign(4 + L, 0);
  int64_t e = one ? 1 : INT64_MIN;
  std::memcpy(out.data(), &e, 8);
  if (one) out[3 + L] = 0x80000000u;  // value = 2^31 2^(32(L-1)) 2^(1-32L) = 1
}

// sites: k distinct qubits in range, any order (general placement, R18)
int check_sites(const mps_state* s, const int* sites, int k) {
  if (!sites || k < 1 || k > 3) return MPS_EINVAL;
  for (int i = 0; i < k; ++i) {
    if (sites[i] < 0 || sites[i] >= s->n) return MPS_EINVAL;
    for (int j = 0; j < i; ++j)
      if (sites[j] == sites[i]) return MPS_EINVAL;
  }
  return MPS_OK;
}

// Reorder a k-qubit gate given on `sites` (sites[0] = most significant bit of the gate
// index, any order) to ascending sites: ss = sorted sites, Us[x'][y'] = U[x][y] where x' has
// bit t (MSB first) equal to bit idx[t] of x and ss[t] = sites[idx[t]].
void sort_gate(const unsigned char* U, size_t cb, int k, const int* sites, int* ss, std::vector<unsigned char>& Us) {
  int idx[3] = {0, 1, 2};
  std::sort(idx, idx + k, [&](int a, int b) { return sites[a] < sites[b]; });
  for (int t = 0; t < k; ++t) ss[t] = sites[idx[t]];
  const int D = 1 << k;
  auto orig = [&](int xs) {  // sorted-order index -> original-order index
    int x = 0;
    for (int t = 0; t < k; ++t)
      if ((xs >> (k - 1 - t)) & 1) x |= 1 << (k - 1 - idx[t]);
    return x;
  };
  Us.resize((size_t)D * D * cb);
  for (int xs = 0; xs < D; ++xs)
    for (int ys = 0; ys < D; ++ys)
      std::memcpy(Us.data() + ((size_t)xs * D + ys) * cb, U + ((size_t)orig(xs) * D + orig(ys)) * cb, cb);
}

// exact SWAP gate (4 x 4 complex records)
void swap_gate(int p, size_t cb, std::vector<unsigned char>& S) {
  std::vector<uint32_t> z, o;
  host_record(p, 0, z);
  host_record(p, 1, o);
  S.assign(16 * cb, 0);
  const int perm[4] = {0, 2, 1, 3};
  for (int x = 0; x < 4; ++x)
    for (int y = 0; y < 4; ++y) {
      unsigned char* dst = S.data() + (size_t)(x * 4 + y) * cb;
      std::memcpy(dst, (perm[x] == y ? o : z).data(), cb / 2);
      std::memcpy(dst + cb / 2, z.data(), cb / 2);
    }
}

// U(4) on (s, s+2) -> U(8) on (s, s+1, s+2) with identity on s+1
void embed_u8(const unsigned char* U4, size_t cb, std::vector<unsigned char>& U8, int p) {
  std::vector<uint32_t> z;
  host_record(p, 0, z);
  U8.assign(64 * cb, 0);
  for (int x = 0; x < 8; ++x)
    for (int y = 0; y < 8; ++y) {
      unsigned char* dst = U8.data() + (size_t)(x * 8 + y) * cb;
      int mi = (x >> 1) & 1, mj = (y >> 1) & 1;
      if (mi != mj) {
        std::memcpy(dst, z.data(), cb / 2);
        std::memcpy(dst + cb / 2, z.data(), cb / 2);
        continue;
      }
      int a = ((x >> 2) << 1) | (x & 1), b = ((y >> 2) << 1) | (y & 1);
      std::memcpy(dst, U4 + (size_t)(a * 4 + b) * cb, cb);
    }
}

// Upload U (d x d complex records) and check unitarity on the device.
int upload_gate(mps_state* s, const void* U, int d, uint32_t* dU) {
  cudaMemcpyAsync(dU, U, (size_t)d * d * s->cb, cudaMemcpyHostToDevice, s->st);
  cudaMemsetAsync(s->dint, 0, sizeof(int), s->st);
  s->ops->unitary(s->p, dU, d, s->dint, s->st);
  int bad = 0;
  cudaMemcpyAsync(&bad, s->dint, sizeof(int), cudaMemcpyDeviceToHost, s->st);
  if (int rc = sync_ok(s, s->st)) return rc;
  return bad ? MPS_ENOTUNITARY : MPS_OK;
}

// copy the packed sub-block [rows][k] of a [rows][ld] record matrix into dst
void repack_rows(mps_state* s, uint32_t* dst, const uint32_t* src, int rows, int k, int ld) {
  cudaMemcpy2DAsync(dst, (size_t)k * s->cb, src, (size_t)ld * s->cb, (size_t)k * s->cb, rows,
                    cudaMemcpyDeviceToDevice, s->st);
}
// [2][ld][cols] -> [2][k][cols]
void repack_blocks(mps_state* s, uint32_t* dst, const uint32_t* src, int k, int ld, int cols) {
  cudaMemcpy2DAsync(dst, (size_t)k * cols * s->cb, src, (size_t)ld * cols * s->cb, (size_t)k * cols * s->cb, 2,
                    cudaMemcpyDeviceToDevice, s->st);
}

// Range (bits) of a stored Schmidt vector (descending records): log2(lam_0 / lam_{m-1}).
// Used to predict whether an update's kept spectrum will be too wide for the recovered V (R16);
// a wrong guess is caught by the device check (FinItem::redo) and re-run.
int lam_range_bits(mps_state* s, const uint32_t* lam, int m) {
  if (!lam || m <= 1) return 0;
  int64_t e0 = 0, e1 = 0;
  cudaMemcpyAsync(&e0, lam, 8, cudaMemcpyDeviceToHost, s->st);
  cudaMemcpyAsync(&e1, (const char*)lam + (size_t)(m - 1) * s->rb, 8, cudaMemcpyDeviceToHost, s->st);
  cudaStreamSynchronize(s->st);
  if (e1 == INT64_MIN) return 1 << 20;
  return (int)std::min<int64_t>(e0 - e1, 1 << 20);
}
int recover_bits(const mps_state* s) { return s->ops->L <= 10 ? redo_bits<10>() : redo_bits<19>(); }

struct TwoSitePlan {
  int s, ld;
  uint32_t *GL, *GR, *lam, *sig;
  int* ints;  // k, sweeps, status
};

}  // namespace

extern "C" {

// global bond b capacity: Schmidt rank <= min(2^(b+1), 2^(N-b-1)), and <= chi_max
static int gcap(int b, int N, int chi_max) {
  int e = std::min(b + 1, N - b - 1);
  long long c = e >= 30 ? (1LL << 30) : (1LL << e);
  return (int)std::min<long long>(chi_max, c);
}

int mps_init_block(mps_state** out, int ntot, int lo, int hi, int p, int chi_max, double thr) {
  if (!out) return MPS_EINVAL;
  *out = nullptr;
  if (ntot < 1 || chi_max < 1 || lo < 0 || hi > ntot || hi <= lo) return MPS_EINVAL;
  if (p < 64 || p > 512 || chi_max > MAX_CHI) return MPS_EUNSUPPORTED;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MPS_ECUDA;
  const int n = hi - lo;
  auto* s = new mps_state();
  s->n = n;
  s->lo = lo;
  s->ntot = ntot;
  s->has_l = lo > 0;
  s->has_r = hi < ntot;
  s->p = p;
  s->chi_max = chi_max;
  s->RBr = record_words(p);
  s->rb = 4 * (size_t)s->RBr;
  s->cb = 2 * s->rb;
  s->thr = thr > 0 ? thr : std::ldexp(1.0, -((p + 1) / 2));
  s->ops = &tier_ops(p);
  s->m.assign(n > 1 ? n - 1 : 0, 1);
  s->cap.resize(n > 1 ? n - 1 : 0);
  for (int b = 0; b + 1 < n; ++b) s->cap[b] = gcap(lo + b, ntot, chi_max);
  if (s->has_l) s->cap_el = gcap(lo - 1, ntot, chi_max);
  if (s->has_r) s->cap_er = gcap(hi - 1, ntot, chi_max);
  std::vector<uint32_t> one, zero;
  host_record(p, 1, one);
  host_record(p, 0, zero);
  s->G.assign(n, nullptr);
  s->lam.assign(n > 1 ? n - 1 : 0, nullptr);
  bool ok = cudaMalloc(&s->dint, 256 * sizeof(int)) == cudaSuccess;
  for (int i = 0; ok && i < n; ++i) {
    ok = cudaMalloc(&s->G[i], (size_t)2 * s->capl(i) * s->capr(i) * s->cb) == cudaSuccess;
    if (!ok) break;
    // Gamma^0 = [1], Gamma^1 = [0]
    std::vector<uint32_t> g;
    g.insert(g.end(), one.begin(), one.end());
    g.insert(g.end(), zero.begin(), zero.end());
    g.insert(g.end(), zero.begin(), zero.end());
    g.insert(g.end(), zero.begin(), zero.end());
    cudaMemcpy(s->G[i], g.data(), 2 * s->cb, cudaMemcpyHostToDevice);
  }
  for (int b = 0; ok && b + 1 < n; ++b) {
    ok = cudaMalloc(&s->lam[b], (size_t)s->cap[b] * s->rb) == cudaSuccess;
    if (ok) cudaMemcpy(s->lam[b], one.data(), s->rb, cudaMemcpyHostToDevice);
  }
  if (ok && s->has_l) {
    ok = cudaMalloc(&s->lam_el, (size_t)s->cap_el * s->rb) == cudaSuccess;
    if (ok) cudaMemcpy(s->lam_el, one.data(), s->rb, cudaMemcpyHostToDevice);
  }
  if (ok && s->has_r) {
    ok = cudaMalloc(&s->lam_er, (size_t)s->cap_er * s->rb) == cudaSuccess;
    if (ok) cudaMemcpy(s->lam_er, one.data(), s->rb, cudaMemcpyHostToDevice);
  }
  if (!ok) {
    mps_free(s);
    return MPS_ENOMEM;
  }
  *out = s;
  return MPS_OK;
}

int mps_init(mps_state** out, int n, int p, int chi_max, double thr) {
  return mps_init_block(out, n, 0, n, p, chi_max, thr);
}

void mps_free(mps_state* s) {
  if (!s) return;
  for (auto* g : s->G) cudaFree(g);
  for (auto* l : s->lam) cudaFree(l);
  if (s->lam_el) cudaFree(s->lam_el);
  if (s->lam_er) cudaFree(s->lam_er);
  if (s->ws) cudaFree(s->ws);
  if (s->tmp) cudaFree(s->tmp);
  if (s->dint) cudaFree(s->dint);
  for (auto st : s->sub) cudaStreamDestroy(st);
  delete s;
}

int mps_set_stream(mps_state* s, void* stream) {
  if (!s) return MPS_EINVAL;
  s->st = (cudaStream_t)stream;
  return MPS_OK;
}

int mps_sync(mps_state* s) {
  if (!s) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  return sync_ok(s, s->st);
}

int mps_n_qubits(mps_state* s) { return s ? s->n : MPS_EINVAL; }

int mps_bond_dims(mps_state* s, int* out) {
  if (!s || !out) return MPS_EINVAL;
  for (int b = 0; b + 1 < s->n; ++b) out[b] = s->m[b];
  return s->sticky;
}

// ---------------------------------------------------------------- gates
static int apply_two_site_batch(mps_state* s, const std::vector<int>& first, const std::vector<const void*>& Us) {
  const int ng = (int)first.size();
  // temp layout per gate: U (16 cplx), GL out [2][dl][ld], GR out [2][ld][dr], lam [ld], sigma [N]
  std::vector<size_t> off(ng + 1, 0);
  for (int g = 0; g < ng; ++g) {
    const int q = first[g], ld = s->capR(q);
    const int dl = s->dl(q), dr = s->dr(q + 1);
    size_t need = align_up(16 * s->cb) + align_up((size_t)2 * dl * ld * s->cb) + align_up((size_t)2 * ld * dr * s->cb) +
                  align_up((size_t)ld * s->rb) + align_up((size_t)2 * std::max(dl, dr) * s->rb);
    off[g + 1] = off[g] + need;
  }
  if (!grow((void**)&s->tmp, &s->tmp_sz, off[ng] + 4096)) return s->sticky = MPS_ENOMEM;
  std::vector<Upd2Args> args(ng);
  for (int g = 0; g < ng; ++g) {
    const int q = first[g], ld = s->capR(q);
    const int dl = s->dl(q), dr = s->dr(q + 1);
    char* b = s->tmp + off[g];
    uint32_t* dU = (uint32_t*)b;
    if (int rc = upload_gate(s, Us[g], 4, dU)) return rc;
    Upd2Args a;
    std::memset(&a, 0, sizeof(a));
    a.chiL = dl; a.chiM = s->m[q]; a.chiR = dr; a.chi_max = s->chi_max;
    a.GL = s->G[q]; a.GR = s->G[q + 1];
    a.lamL = s->lamL(q);
    a.lamM = s->lam[q];
    a.lamR = s->lamR(q + 1);
    a.U = dU;
    b += align_up(16 * s->cb);
    a.GL_out = (uint32_t*)b; b += align_up((size_t)2 * dl * ld * s->cb);
    a.GR_out = (uint32_t*)b; b += align_up((size_t)2 * ld * dr * s->cb);
    a.lam_out = (uint32_t*)b; b += align_up((size_t)ld * s->rb);
    a.sigma_out = (uint32_t*)b;
    a.out_ld = ld;
    a.k_out = s->dint + 3 * g; a.sweeps_out = s->dint + 3 * g + 1; a.status_out = s->dint + 3 * g + 2;
    a.accumulate_v = lam_range_bits(s, s->lam[q], s->m[q]) > recover_bits(s) ? 1 : 0;
    args[g] = a;
  }
  if (3 * ng > 256) return MPS_EINVAL;
  size_t need = s->ops->upd2_ws(args.data(), ng);
  if (!grow(&s->ws, &s->ws_sz, need)) return s->sticky = MPS_ENOMEM;
  std::vector<unsigned char> hd;
  s->ops->upd2(s->p, s->thr, args.data(), ng, s->ws, s->st, hd);
  std::vector<int> res(3 * ng);
  cudaMemcpyAsync(res.data(), s->dint, sizeof(int) * 3 * ng, cudaMemcpyDeviceToHost, s->st);
  if (int rc = sync_ok(s, s->st)) return rc;
  for (int g = 0; g < ng; ++g) {
    const int k = res[3 * g], sw = res[3 * g + 1], stt = res[3 * g + 2];
    s->sweeps_total += sw;
    s->last_sweeps = sw;
    s->gates++;
    if (stt) return s->sticky = stt;
    const int q = first[g], ld = s->capR(q);
    const int dl = s->dl(q), dr = s->dr(q + 1);
    repack_rows(s, s->G[q], args[g].GL_out, 2 * dl, k, ld);
    repack_blocks(s, s->G[q + 1], args[g].GR_out, k, ld, dr);
    cudaMemcpyAsync(s->lam[q], args[g].lam_out, (size_t)k * s->rb, cudaMemcpyDeviceToDevice, s->st);
    s->m[q] = k;
  }
  return sync_ok(s, s->st);
}

static int apply_three_site(mps_state* s, int q, const void* U8) {
  const int dl = s->dl(q), d1 = s->m[q], d2 = s->m[q + 1], dr = s->dr(q + 2);
  const int ld = std::max(s->cap[q], s->cap[q + 1]);
  size_t o_U = 0, o_G0 = align_up(64 * s->cb), o_G1 = o_G0 + align_up((size_t)2 * dl * ld * s->cb),
         o_G2 = o_G1 + align_up((size_t)2 * ld * ld * s->cb), o_l1 = o_G2 + align_up((size_t)2 * ld * dr * s->cb),
         o_l2 = o_l1 + align_up((size_t)ld * s->rb), o_end = o_l2 + align_up((size_t)ld * s->rb);
  if (!grow((void**)&s->tmp, &s->tmp_sz, o_end + 4096)) return s->sticky = MPS_ENOMEM;
  uint32_t* dU = (uint32_t*)(s->tmp + o_U);
  if (int rc = upload_gate(s, U8, 8, dU)) return rc;
  Upd3Args a;
  std::memset(&a, 0, sizeof(a));
  a.chiL = dl; a.chi1 = d1; a.chi2 = d2; a.chiR = dr; a.chi_max = s->chi_max;
  a.G0 = s->G[q]; a.G1 = s->G[q + 1]; a.G2 = s->G[q + 2];
  a.lamL = s->lamL(q);
  a.lam1 = s->lam[q];
  a.lam2 = s->lam[q + 1];
  a.lamR = s->lamR(q + 2);
  a.U = dU;
  a.G0_out = (uint32_t*)(s->tmp + o_G0);
  a.G1_out = (uint32_t*)(s->tmp + o_G1);
  a.G2_out = (uint32_t*)(s->tmp + o_G2);
  a.lam1_out = (uint32_t*)(s->tmp + o_l1);
  a.lam2_out = (uint32_t*)(s->tmp + o_l2);
  a.ld = ld;
  a.k1 = s->dint; a.k2 = s->dint + 1; a.sweeps = s->dint + 2; a.status = s->dint + 3;
  size_t need = s->ops->upd3_ws(a);
  if (!grow(&s->ws, &s->ws_sz, need)) return s->sticky = MPS_ENOMEM;
  a.redo = s->dint + 4;
  std::vector<unsigned char> hd1, hd2;
  // each stage recovers V unless its kept spectrum is too wide; then it is re-run with
  // accumulated V (R16)
  int r1[5];
  const int rb1 = lam_range_bits(s, s->lam[q + 1], s->m[q + 1]), rb2 = lam_range_bits(s, s->lam[q], s->m[q]);
  for (int pass = rb1 > recover_bits(s) ? 1 : 0; pass < 2; ++pass) {
    a.accumulate_v = pass;
    cudaMemsetAsync(s->dint, 0, 5 * sizeof(int), s->st);
    s->ops->upd3_s1(s->p, s->thr, a, s->ws, s->st, hd1);
    cudaMemcpyAsync(r1, s->dint, sizeof(r1), cudaMemcpyDeviceToHost, s->st);
    if (int rc = sync_ok(s, s->st)) return rc;
    if (!r1[4] || r1[3]) break;
    if (r1[4] & 2) a.no_precond = 1;  // a Newton-Schulz zero-digit check failed: no preconditioner
    if (getenv("MPS_DEBUG_REDO")) fprintf(stderr, "three-site stage 1 at %d: re-run with accumulated V\n", q);
  }
  a.no_precond = 0;
  if (r1[3]) { s->sweeps_total += r1[2]; return s->sticky = r1[3]; }
  const int k1 = r1[0];
  a.s1_accumulated = a.accumulate_v;
  int r2[5];
  for (int pass = rb2 > recover_bits(s) ? 1 : 0; pass < 2; ++pass) {
    a.accumulate_v = pass;
    cudaMemcpyAsync(s->dint + 2, &r1[2], sizeof(int), cudaMemcpyHostToDevice, s->st);  // stage-1 sweeps
    cudaMemsetAsync(s->dint + 4, 0, sizeof(int), s->st);
    s->ops->upd3_s2(s->p, s->thr, a, k1, s->ws, s->st, hd2);
    cudaMemcpyAsync(r2, s->dint, sizeof(r2), cudaMemcpyDeviceToHost, s->st);
    if (int rc = sync_ok(s, s->st)) return rc;
    if (!r2[4] || r2[3]) break;
    if (r2[4] & 2) a.no_precond = 1;
    if (getenv("MPS_DEBUG_REDO")) fprintf(stderr, "three-site stage 2 at %d: re-run with accumulated V\n", q);
  }
  s->sweeps_total += r2[2];
  s->last_sweeps = r2[2];
  s->gates++;
  if (r2[3]) return s->sticky = r2[3];
  const int k2 = r2[1];
  repack_rows(s, s->G[q], a.G0_out, 2 * dl, k2, ld);
  repack_blocks(s, s->G[q + 1], a.G1_out, k2, ld, k1);
  repack_blocks(s, s->G[q + 2], a.G2_out, k1, ld, dr);
  cudaMemcpyAsync(s->lam[q], a.lam1_out, (size_t)k2 * s->rb, cudaMemcpyDeviceToDevice, s->st);
  cudaMemcpyAsync(s->lam[q + 1], a.lam2_out, (size_t)k1 * s->rb, cudaMemcpyDeviceToDevice, s->st);
  s->m[q] = k2;
  s->m[q + 1] = k1;
  return sync_ok(s, s->st);
}

// Disjoint three-site gates of a layer (U8 host records, sites qs[g]..qs[g]+2): the updates run
// concurrently on side streams (each stage is a chain of one-item kernels), with one host
// synchronisation per stage for all gates.  Arithmetic per gate = apply_three_site.
static int apply_three_site_batch(mps_state* s, const std::vector<int>& qs, const std::vector<const void*>& Us) {
  const int n = (int)qs.size();
  if (n == 0) return MPS_OK;
  if (n == 1) return apply_three_site(s, qs[0], Us[0]);
  constexpr int NS = 8, DI = 8;  // side streams; device ints per gate
  if (n * DI > 256) {            // chunk
    const int h = n / 2;
    if (int rc = apply_three_site_batch(s, std::vector<int>(qs.begin(), qs.begin() + h),
                                        std::vector<const void*>(Us.begin(), Us.begin() + h)))
      return rc;
    return apply_three_site_batch(s, std::vector<int>(qs.begin() + h, qs.end()),
                                  std::vector<const void*>(Us.begin() + h, Us.end()));
  }
  while ((int)s->sub.size() < NS) {
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return s->sticky = MPS_ECUDA;
    s->sub.push_back(st);
  }
  std::vector<Upd3Args> A(n);
  std::vector<size_t> off(n + 1, 0), woff(n + 1, 0);
  std::vector<int> ldv(n);
  for (int g = 0; g < n; ++g) {
    const int q = qs[g];
    const int dl = s->dl(q), dr = s->dr(q + 2), ld = std::max(s->cap[q], s->cap[q + 1]);
    ldv[g] = ld;
    off[g + 1] = off[g] + align_up(64 * s->cb) + align_up((size_t)2 * dl * ld * s->cb) +
                 align_up((size_t)2 * ld * ld * s->cb) + align_up((size_t)2 * ld * dr * s->cb) +
                 2 * align_up((size_t)ld * s->rb);
  }
  if (!grow((void**)&s->tmp, &s->tmp_sz, off[n] + 4096)) return s->sticky = MPS_ENOMEM;
  for (int g = 0; g < n; ++g) {
    const int q = qs[g];
    const int dl = s->dl(q), d1 = s->m[q], d2 = s->m[q + 1], dr = s->dr(q + 2), ld = ldv[g];
    char* b = s->tmp + off[g];
    uint32_t* dU = (uint32_t*)b;
    if (int rc = upload_gate(s, Us[g], 8, dU)) return rc;
    Upd3Args& a = A[g];
    std::memset(&a, 0, sizeof(a));
    a.chiL = dl; a.chi1 = d1; a.chi2 = d2; a.chiR = dr; a.chi_max = s->chi_max;
    a.G0 = s->G[q]; a.G1 = s->G[q + 1]; a.G2 = s->G[q + 2];
    a.lamL = s->lamL(q); a.lam1 = s->lam[q]; a.lam2 = s->lam[q + 1]; a.lamR = s->lamR(q + 2);
    a.U = dU;
    b += align_up(64 * s->cb);
    a.G0_out = (uint32_t*)b; b += align_up((size_t)2 * dl * ld * s->cb);
    a.G1_out = (uint32_t*)b; b += align_up((size_t)2 * ld * ld * s->cb);
    a.G2_out = (uint32_t*)b; b += align_up((size_t)2 * ld * dr * s->cb);
    a.lam1_out = (uint32_t*)b; b += align_up((size_t)ld * s->rb);
    a.lam2_out = (uint32_t*)b;
    a.ld = ld;
    int* di = s->dint + DI * g;
    a.k1 = di; a.k2 = di + 1; a.sweeps = di + 2; a.status = di + 3; a.redo = di + 4;
    woff[g + 1] = woff[g] + align_up(s->ops->upd3_ws(a));
  }
  if (!grow(&s->ws, &s->ws_sz, woff[n])) return s->sticky = MPS_ENOMEM;
  // side streams start after everything queued on the handle's stream
  cudaEvent_t ev0;
  cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
  cudaEventRecord(ev0, s->st);
  for (int i = 0; i < NS; ++i) cudaStreamWaitEvent(s->sub[i], ev0, 0);
  auto stream_of = [&](int g) { return s->sub[g % NS]; };
  auto sync_all = [&]() -> int {
    if (int rc = cuda_ok(s, cudaGetLastError())) return rc;  // launch errors (not sticky)
    for (int i = 0; i < NS; ++i)
      if (cudaError_t e = cudaStreamSynchronize(s->sub[i])) return cuda_ok(s, e);
    return MPS_OK;
  };
  std::vector<std::vector<unsigned char>> hd(2 * n);
  std::vector<int> r(DI * n, 0), k1(n, 0);
  // stage 1 (first pass with the predicted mode, at most one re-run per gate)
  std::vector<char> todo(n, 1);
  for (int g = 0; g < n; ++g) {
    const int q = qs[g];
    A[g].accumulate_v = lam_range_bits(s, s->lam[q + 1], s->m[q + 1]) > recover_bits(s) ? 1 : 0;
  }
  for (int pass = 0; pass < 2; ++pass) {
    for (int g = 0; g < n; ++g) {
      if (!todo[g]) continue;
      cudaMemsetAsync(s->dint + DI * g, 0, 5 * sizeof(int), stream_of(g));
      s->ops->upd3_s1(s->p, s->thr, A[g], (char*)s->ws + woff[g], stream_of(g), hd[2 * g]);
    }
    if (int rc = sync_all()) return rc;
    cudaMemcpy(r.data(), s->dint, sizeof(int) * DI * n, cudaMemcpyDeviceToHost);
    bool again = false;
    for (int g = 0; g < n; ++g) {
      todo[g] = 0;
      const int* rg = r.data() + DI * g;
      if (pass == 0 && rg[4] && !rg[3] && !A[g].accumulate_v) {
        A[g].accumulate_v = 1;
        if (rg[4] & 2) A[g].no_precond = 1;
        todo[g] = 1;
        again = true;
      }
    }
    if (!again) break;
  }
  for (int g = 0; g < n; ++g) {
    const int* rg = r.data() + DI * g;
    if (rg[3]) { s->sweeps_total += rg[2]; return s->sticky = rg[3]; }
    k1[g] = rg[0];
    A[g].s1_accumulated = A[g].accumulate_v;
    A[g].no_precond = 0;
    const int q = qs[g];
    A[g].accumulate_v = lam_range_bits(s, s->lam[q], s->m[q]) > recover_bits(s) ? 1 : 0;
    todo[g] = 1;
  }
  std::vector<int> r1 = r;
  for (int pass = 0; pass < 2; ++pass) {
    for (int g = 0; g < n; ++g) {
      if (!todo[g]) continue;
      cudaMemcpyAsync(s->dint + DI * g + 2, &r1[DI * g + 2], sizeof(int), cudaMemcpyHostToDevice, stream_of(g));
      cudaMemsetAsync(s->dint + DI * g + 4, 0, sizeof(int), stream_of(g));
      s->ops->upd3_s2(s->p, s->thr, A[g], k1[g], (char*)s->ws + woff[g], stream_of(g), hd[2 * g + 1]);
    }
    if (int rc = sync_all()) return rc;
    cudaMemcpy(r.data(), s->dint, sizeof(int) * DI * n, cudaMemcpyDeviceToHost);
    bool again = false;
    for (int g = 0; g < n; ++g) {
      todo[g] = 0;
      const int* rg = r.data() + DI * g;
      if (pass == 0 && rg[4] && !rg[3] && !A[g].accumulate_v) {
        A[g].accumulate_v = 1;
        if (rg[4] & 2) A[g].no_precond = 1;
        todo[g] = 1;
        again = true;
      }
    }
    if (!again) break;
  }
  cudaEventDestroy(ev0);
  for (int g = 0; g < n; ++g) {
    const int* rg = r.data() + DI * g;
    s->sweeps_total += rg[2];
    s->last_sweeps = rg[2];
    s->gates++;
    if (rg[3]) return s->sticky = rg[3];
  }
  for (int g = 0; g < n; ++g) {
    const int q = qs[g], dl = s->dl(q), dr = s->dr(q + 2), ld = ldv[g];
    const int k2 = r[DI * g + 1];
    const Upd3Args& a = A[g];
    repack_rows(s, s->G[q], a.G0_out, 2 * dl, k2, ld);
    repack_blocks(s, s->G[q + 1], a.G1_out, k2, ld, k1[g]);
    repack_blocks(s, s->G[q + 2], a.G2_out, k1[g], ld, dr);
    cudaMemcpyAsync(s->lam[q], a.lam1_out, (size_t)k2 * s->rb, cudaMemcpyDeviceToDevice, s->st);
    cudaMemcpyAsync(s->lam[q + 1], a.lam2_out, (size_t)k1[g] * s->rb, cudaMemcpyDeviceToDevice, s->st);
    s->m[q] = k2;
    s->m[q + 1] = k1[g];
  }
  return sync_ok(s, s->st);
}

static int apply_one(mps_state* s, const void* U, const int* sites, int k) {
  const int q = sites[0];
  if (k == 1) {
    const int nab = s->dl(q) * s->dr(q);
    size_t o_G = align_up(4 * s->cb);
    if (!grow((void**)&s->tmp, &s->tmp_sz, o_G + (size_t)2 * nab * s->cb + 4096)) return s->sticky = MPS_ENOMEM;
    uint32_t* dU = (uint32_t*)s->tmp;
    if (int rc = upload_gate(s, U, 2, dU)) return rc;
    uint32_t* out = (uint32_t*)(s->tmp + o_G);
    s->ops->onesite(s->p, s->G[q], out, dU, nab, s->st);
    cudaMemcpyAsync(s->G[q], out, (size_t)2 * nab * s->cb, cudaMemcpyDeviceToDevice, s->st);
    s->gates++;
    return sync_ok(s, s->st);
  }
  if (k == 2 && sites[1] == q + 1) return apply_two_site_batch(s, {q}, {U});
  if (k == 2) {
    std::vector<unsigned char> U8;
    embed_u8((const unsigned char*)U, s->cb, U8, s->p);
    return apply_three_site(s, q, U8.data());
  }
  return apply_three_site(s, q, U);
}

// General placement (R18): sort the sites (permuting U), then a gate that spans
// more than three consecutive sites is routed with exact SWAP gates: the far qubits are
// moved next to the first one, the gate is applied on consecutive sites, and the SWAPs are
// undone in reverse order.  A two-qubit gate on (s, s+2) keeps the U(8) embedding.
static int apply_general(mps_state* s, const void* U, const int* sites, int k) {
  if (k == 1) return apply_one(s, U, sites, k);
  int ss[3];
  std::vector<unsigned char> Us;
  sort_gate((const unsigned char*)U, s->cb, k, sites, ss, Us);
  const int a = ss[0];
  if ((k == 2 && ss[1] - a <= 2) || (k == 3 && ss[2] == a + 2)) return apply_one(s, Us.data(), ss, k);
  std::vector<unsigned char> S;
  swap_gate(s->p, s->cb, S);
  auto sw = [&](int t) {  // SWAP on (t-1, t)
    const int q[2] = {t - 1, t};
    return apply_one(s, S.data(), q, 2);
  };
  int rc = MPS_OK;
  if (k == 2) {
    const int b = ss[1];
    for (int t = b; t > a + 1 && !rc; --t) rc = sw(t);  // qubit b -> a+1
    if (rc) return rc;
    const int q[2] = {a, a + 1};
    if ((rc = apply_one(s, Us.data(), q, 2))) return rc;
    for (int t = a + 2; t <= b && !rc; ++t) rc = sw(t);  // back to b
    return rc;
  }
  const int b = ss[1], c = ss[2];
  for (int t = b; t > a + 1 && !rc; --t) rc = sw(t);  // qubit b -> a+1
  for (int t = c; t > a + 2 && !rc; --t) rc = sw(t);  // qubit c -> a+2
  if (rc) return rc;
  const int q[3] = {a, a + 1, a + 2};
  if ((rc = apply_one(s, Us.data(), q, 3))) return rc;
  for (int t = a + 3; t <= c && !rc; ++t) rc = sw(t);  // a+2 -> c
  for (int t = a + 2; t <= b && !rc; ++t) rc = sw(t);  // a+1 -> b
  return rc;
}

int mps_apply_gate(mps_state* s, const void* U, const int* sites, int k) {
  if (!s || !U) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  if (int rc = check_sites(s, sites, k)) return rc;
  return apply_general(s, U, sites, k);
}

int mps_apply_layer(mps_state* s, int ng, const void* const* U, const int* sites_flat, const int* k) {
  if (!s || ng < 0 || (ng && (!U || !sites_flat || !k))) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  std::vector<int> used(s->n, 0);
  int o = 0;
  for (int g = 0; g < ng; ++g) {
    if (int rc = check_sites(s, sites_flat + o, k[g])) return rc;
    const int lo = *std::min_element(sites_flat + o, sites_flat + o + k[g]);
    const int hi = *std::max_element(sites_flat + o, sites_flat + o + k[g]);
    for (int q = lo; q <= hi; ++q)  // the whole span (routed gates swap through it)
      if (used[q]++) return MPS_EOVERLAP;
    o += k[g];
  }
  // batched launch of every adjacent two-site gate, the rest one by one
  std::vector<int> first;
  std::vector<const void*> us;
  o = 0;
  for (int g = 0; g < ng; ++g) {
    if (k[g] == 2 && sites_flat[o + 1] == sites_flat[o] + 1) {
      first.push_back(sites_flat[o]);
      us.push_back(U[g]);
    }
    o += k[g];
  }
  for (size_t i = 0; i < first.size(); i += 64) {
    std::vector<int> f(first.begin() + i, first.begin() + std::min(first.size(), i + 64));
    std::vector<const void*> u(us.begin() + i, us.begin() + std::min(us.size(), i + 64));
    if (int rc = apply_two_site_batch(s, f, u)) return rc;
  }
  // three-site gates (ascending consecutive triples, and two-site gates on (s, s+2) embedded
  // into U(8)) run as one concurrent batch; the rest one by one
  std::vector<int> tq;
  std::vector<const void*> tu;
  std::vector<std::vector<unsigned char>> emb;
  emb.reserve(ng);
  o = 0;
  for (int g = 0; g < ng; ++g) {
    const int* st_ = sites_flat + o;
    if (k[g] == 3 && st_[1] == st_[0] + 1 && st_[2] == st_[0] + 2) {
      tq.push_back(st_[0]);
      tu.push_back(U[g]);
    } else if (k[g] == 2 && st_[1] == st_[0] + 2) {
      emb.emplace_back();
      embed_u8((const unsigned char*)U[g], s->cb, emb.back(), s->p);
      tq.push_back(st_[0]);
      tu.push_back(emb.back().data());
    }
    o += k[g];
  }
  if (int rc = apply_three_site_batch(s, tq, tu)) return rc;
  o = 0;
  for (int g = 0; g < ng; ++g) {
    const int* st_ = sites_flat + o;
    const bool adj2 = k[g] == 2 && st_[1] == st_[0] + 1;
    const bool tri = (k[g] == 3 && st_[1] == st_[0] + 1 && st_[2] == st_[0] + 2) || (k[g] == 2 && st_[1] == st_[0] + 2);
    if (!adj2 && !tri)
      if (int rc = apply_general(s, U[g], sites_flat + o, k[g])) return rc;
    o += k[g];
  }
  return MPS_OK;
}

// ---------------------------------------------------------------- queries
// amplitude chains of nstates bit strings over the local sites; v_in (host, dl(0) complex
// records) or null; out receives dr(n-1) complex records per state
static int amplitudes(mps_state* s, const uint8_t* bits_host, long long nstates, const void* v_in, void* out) {
  const int n = s->n;
  int maxchi = std::max(s->dl(0), s->dr(n - 1));
  for (int b = 0; b + 1 < n; ++b) maxchi = std::max(maxchi, s->m[b]);
  const int nblocks = (int)std::min<long long>(nstates, 1184);
  std::vector<int> dims(n + 1);
  for (int q = 0; q < n; ++q) dims[q] = s->dl(q);
  dims[n] = s->dr(n - 1);
  const size_t o_ptr = 0, o_lam = align_up(8 * (size_t)n), o_dims = o_lam + align_up(8 * (size_t)n),
               o_vin = o_dims + align_up(4 * (size_t)(n + 1)), o_bits = o_vin + align_up((size_t)dims[0] * s->cb),
               o_out = o_bits + align_up((size_t)nstates * n),
               o_scr = o_out + align_up((size_t)nstates * dims[n] * s->cb),
               o_end = o_scr + s->ops->amp_scratch(maxchi, nblocks);
  if (!grow((void**)&s->tmp, &s->tmp_sz, o_end)) return MPS_ENOMEM;
  std::vector<const uint32_t*> lam(n);
  for (int q = 0; q < n; ++q) lam[q] = s->lamL(q);
  cudaMemcpyAsync(s->tmp + o_ptr, s->G.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, s->st);
  cudaMemcpyAsync(s->tmp + o_lam, lam.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, s->st);
  cudaMemcpyAsync(s->tmp + o_dims, dims.data(), 4 * (size_t)(n + 1), cudaMemcpyHostToDevice, s->st);
  if (v_in) cudaMemcpyAsync(s->tmp + o_vin, v_in, (size_t)dims[0] * s->cb, cudaMemcpyHostToDevice, s->st);
  cudaMemcpyAsync(s->tmp + o_bits, bits_host, (size_t)nstates * n, cudaMemcpyHostToDevice, s->st);
  s->ops->amplitudes(s->p, (const uint32_t* const*)(s->tmp + o_ptr), (const uint32_t* const*)(s->tmp + o_lam),
                     (const int*)(s->tmp + o_dims), n, (const uint8_t*)(s->tmp + o_bits), nstates, maxchi,
                     s->tmp + o_scr, nblocks, v_in ? (const uint32_t*)(s->tmp + o_vin) : nullptr,
                     (uint32_t*)(s->tmp + o_out), s->st);
  cudaMemcpyAsync(out, s->tmp + o_out, (size_t)nstates * dims[n] * s->cb, cudaMemcpyDeviceToHost, s->st);
  return sync_ok(s, s->st);
}

int mps_amplitude(mps_state* s, const uint8_t* bits, void* out) {
  if (!s || !bits || !out) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  if (s->has_l || s->has_r) return MPS_EINVAL;  // block states: mps_amplitude_block
  for (int q = 0; q < s->n; ++q)
    if (bits[q] > 1) return MPS_EINVAL;
  return amplitudes(s, bits, 1, nullptr, out);
}

int mps_to_dense(mps_state* s, void* out) {
  if (!s || !out) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  if (s->has_l || s->has_r) return MPS_EINVAL;
  if (s->n > 24) return MPS_ETOOBIG;
  const long long ns = 1LL << s->n;
  std::vector<uint8_t> bits((size_t)ns * s->n);
  for (long long x = 0; x < ns; ++x)
    for (int q = 0; q < s->n; ++q) bits[(size_t)x * s->n + q] = (x >> (s->n - 1 - q)) & 1;
  return amplitudes(s, bits.data(), ns, nullptr, out);
}

static int transfer(mps_state* s, const void* O, const int* sites, int k, void* out, void* den_out) {
  if (s->has_l || s->has_r) return MPS_EINVAL;
  const int n = s->n;
  int maxchi = 1;
  for (int b = 0; b + 1 < n; ++b) maxchi = std::max(maxchi, s->m[b]);
  std::vector<int> dims(n + 1);
  dims[0] = 1;
  for (int q = 1; q < n; ++q) dims[q] = s->m[q - 1];
  dims[n] = 1;
  const size_t o_O = 0, o_res = align_up(64 * s->cb), o_scr = o_res + align_up(2 * s->cb),
               o_end = o_scr + s->ops->transfer_scratch(maxchi);
  if (!grow((void**)&s->tmp, &s->tmp_sz, o_end)) return MPS_ENOMEM;
  const int D = O ? (1 << k) : 0;
  if (O) cudaMemcpyAsync(s->tmp + o_O, O, (size_t)D * D * s->cb, cudaMemcpyHostToDevice, s->st);
  std::vector<const uint32_t*> G(s->G.begin(), s->G.end()), lam(s->lam.begin(), s->lam.end());
  uint32_t* res = (uint32_t*)(s->tmp + o_res);
  s->ops->transfer(s->p, n, G.data(), lam.data(), dims.data(), O ? (const uint32_t*)(s->tmp + o_O) : nullptr,
                   O ? sites[0] : 0, k, s->tmp + o_scr, maxchi, out ? res : nullptr,
                   den_out ? (uint32_t*)((char*)res + s->cb) : nullptr, s->st);
  if (out) cudaMemcpyAsync(out, res, s->cb, cudaMemcpyDeviceToHost, s->st);
  if (den_out) cudaMemcpyAsync(den_out, (char*)res + s->cb, s->rb, cudaMemcpyDeviceToHost, s->st);
  return sync_ok(s, s->st);
}

// Reduced density operator of ascending sites (P:322-341 RDO_block / RDO), normalised by its trace.
int mps_rdo(mps_state* s, const int* sites, int k, void* out) {
  if (!s || !sites || !out || k < 1 || k > 6) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  if (s->has_l || s->has_r) return MPS_EINVAL;
  for (int i = 0; i < k; ++i)
    if (sites[i] < 0 || sites[i] >= s->n || (i && sites[i] <= sites[i - 1])) return MPS_EINVAL;
  const int n = s->n, D = 1 << k;
  int maxchi = 1;
  for (int b = 0; b + 1 < n; ++b) maxchi = std::max(maxchi, s->m[b]);
  std::vector<int> dims(n + 1);
  dims[0] = 1;
  for (int q = 1; q < n; ++q) dims[q] = s->m[q - 1];
  dims[n] = 1;
  const size_t X = (size_t)maxchi * maxchi;
  const size_t cm = s->ops->transfer_scratch(1) / 24;  // sizeof(cmpf) (scratch of 24 1x1 matrices, minus slack)
  (void)cm;
  const size_t scr = s->ops->transfer_scratch(maxchi) / 24 * (2 * (size_t)D * D + 6) + 4096;
  const size_t o_res = 0, o_scr = align_up((size_t)D * D * s->cb), o_end = o_scr + scr;
  if (!grow((void**)&s->tmp, &s->tmp_sz, o_end)) return MPS_ENOMEM;
  std::vector<const uint32_t*> G(s->G.begin(), s->G.end()), lam(s->lam.begin(), s->lam.end());
  s->ops->rdo(s->p, n, G.data(), lam.data(), dims.data(), sites, k, s->tmp + o_scr, maxchi,
              (uint32_t*)(s->tmp + o_res), s->st);
  cudaMemcpyAsync(out, s->tmp + o_res, (size_t)D * D * s->cb, cudaMemcpyDeviceToHost, s->st);
  (void)X;
  return sync_ok(s, s->st);
}

int mps_norm2(mps_state* s, void* out) {
  if (!s || !out) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  return transfer(s, nullptr, nullptr, 0, nullptr, out);
}

int mps_expect(mps_state* s, const void* O, const int* sites, int k, void* out) {
  if (!s || !O || !out || !sites || k < 1 || k > 3) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  for (int i = 0; i < k; ++i)
    if (sites[i] != sites[0] + i || sites[i] < 0 || sites[i] >= s->n) return MPS_EINVAL;
  return transfer(s, O, sites, k, out, nullptr);
}

// ---------------------------------------------------------------- site-sharded blocks
int mps_amplitude_block(mps_state* s, const uint8_t* bits, const void* v_in, void* v_out) {
  if (!s || !bits || !v_out || (s->has_l && !v_in)) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  for (int q = 0; q < s->n; ++q)
    if (bits[q] > 1) return MPS_EINVAL;
  return amplitudes(s, bits, 1, s->has_l ? v_in : nullptr, v_out);
}

int mps_block_dims(mps_state* s, int* lo, int* n, int* m_ext_l, int* m_ext_r) {
  if (!s) return MPS_EINVAL;
  if (lo) *lo = s->lo;
  if (n) *n = s->n;
  if (m_ext_l) *m_ext_l = s->dl(0);
  if (m_ext_r) *m_ext_r = s->dr(s->n - 1);
  return s->sticky;
}

int mps_block_export_first(mps_state* s, void* dG, void* dlam, int* m_l, int* m_r) {
  if (!s || !dG || !m_l || !m_r || !s->has_l) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  *m_l = s->dl(0);
  *m_r = s->dr(0);
  cudaMemcpyAsync(dG, s->G[0], (size_t)2 * *m_l * *m_r * s->cb, cudaMemcpyDeviceToDevice, s->st);
  const uint32_t* lr = s->lamR(0);
  if (dlam && lr) cudaMemcpyAsync(dlam, lr, (size_t)*m_r * s->rb, cudaMemcpyDeviceToDevice, s->st);
  return sync_ok(s, s->st);
}

int mps_block_boundary_apply(mps_state* s, const void* U, const void* dG_halo, int m_h, const void* dlam_h,
                             void* dG_halo_out, void* dlam_mid_out, int* k_out) {
  if (!s || !U || !dG_halo || !dG_halo_out || !dlam_mid_out || !k_out || !s->has_r || m_h < 1) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  const int q = s->n - 1, ld = s->cap_er, dl = s->dl(q), dm = s->m_er;
  const size_t o_U = 0, o_GL = align_up(16 * s->cb), o_GR = o_GL + align_up((size_t)2 * dl * ld * s->cb),
               o_lam = o_GR + align_up((size_t)2 * ld * m_h * s->cb), o_end = o_lam + align_up((size_t)ld * s->rb);
  if (!grow((void**)&s->tmp, &s->tmp_sz, o_end + 4096)) return s->sticky = MPS_ENOMEM;
  uint32_t* dU = (uint32_t*)(s->tmp + o_U);
  if (int rc = upload_gate(s, U, 4, dU)) return rc;
  Upd2Args a;
  std::memset(&a, 0, sizeof(a));
  a.chiL = dl; a.chiM = dm; a.chiR = m_h; a.chi_max = s->chi_max;
  a.GL = s->G[q]; a.GR = (const uint32_t*)dG_halo;
  a.lamL = s->lamL(q); a.lamM = s->lam_er; a.lamR = (const uint32_t*)dlam_h;
  a.U = dU;
  a.GL_out = (uint32_t*)(s->tmp + o_GL);
  a.GR_out = (uint32_t*)(s->tmp + o_GR);
  a.lam_out = (uint32_t*)(s->tmp + o_lam);
  a.out_ld = ld;
  a.k_out = s->dint; a.sweeps_out = s->dint + 1; a.status_out = s->dint + 2;
  if (!grow(&s->ws, &s->ws_sz, s->ops->upd2_ws(&a, 1))) return s->sticky = MPS_ENOMEM;
  std::vector<unsigned char> hd;
  s->ops->upd2(s->p, s->thr, &a, 1, s->ws, s->st, hd);
  int res[3];
  cudaMemcpyAsync(res, s->dint, sizeof(res), cudaMemcpyDeviceToHost, s->st);
  if (int rc = sync_ok(s, s->st)) return rc;
  s->sweeps_total += res[1];
  s->last_sweeps = res[1];
  s->gates++;
  if (res[2]) return s->sticky = res[2];
  const int k = res[0];
  repack_rows(s, s->G[q], a.GL_out, 2 * dl, k, ld);
  repack_blocks(s, (uint32_t*)dG_halo_out, a.GR_out, k, ld, m_h);
  cudaMemcpyAsync(s->lam_er, a.lam_out, (size_t)k * s->rb, cudaMemcpyDeviceToDevice, s->st);
  cudaMemcpyAsync(dlam_mid_out, a.lam_out, (size_t)k * s->rb, cudaMemcpyDeviceToDevice, s->st);
  s->m_er = k;
  *k_out = k;
  return sync_ok(s, s->st);
}

int mps_block_import_first(mps_state* s, const void* dG0, const void* dlam_mid, int k) {
  if (!s || !dG0 || !dlam_mid || !s->has_l || k < 1 || k > s->cap_el) return MPS_EINVAL;
  if (s->sticky) return s->sticky;
  s->m_el = k;
  cudaMemcpyAsync(s->G[0], dG0, (size_t)2 * k * s->dr(0) * s->cb, cudaMemcpyDeviceToDevice, s->st);
  cudaMemcpyAsync(s->lam_el, dlam_mid, (size_t)k * s->rb, cudaMemcpyDeviceToDevice, s->st);
  return sync_ok(s, s->st);
}

// Site / Schmidt-vector transfer: `out` / `in` may be host or device memory (unified
// addressing decides the copy direction); copies are ordered on the state's stream and
// complete when the call returns.  The SPMD driver (dist.py) moves site tensors between
// ranks through device buffers with these calls.
int mps_schmidt(mps_state* s, int bond, void* out, int* m) {
  if (!s || !m || bond < 0 || bond >= s->n - 1) return MPS_EINVAL;
  *m = s->m[bond];
  if (out) {
    cudaMemcpyAsync(out, s->lam[bond], (size_t)s->m[bond] * s->rb, cudaMemcpyDefault, s->st);
    if (int rc = sync_ok(s, s->st)) return rc;
  }
  return s->sticky;
}

int mps_get_site(mps_state* s, int site, void* out, int* ml, int* mr) {
  if (!s || !ml || !mr || site < 0 || site >= s->n) return MPS_EINVAL;
  *ml = s->dl(site);
  *mr = s->dr(site);
  if (out) {
    cudaMemcpyAsync(out, s->G[site], (size_t)2 * *ml * *mr * s->cb, cudaMemcpyDefault, s->st);
    if (int rc = sync_ok(s, s->st)) return rc;
  }
  return s->sticky;
}

int mps_set_schmidt(mps_state* s, int bond, const void* in, int m) {
  if (!s || !in || bond < 0 || bond >= s->n - 1 || m < 1 || m > s->cap[bond]) return MPS_EINVAL;
  s->m[bond] = m;
  cudaMemcpyAsync(s->lam[bond], in, (size_t)m * s->rb, cudaMemcpyDefault, s->st);
  return sync_ok(s, s->st);
}

int mps_set_site(mps_state* s, int site, const void* in, int ml, int mr) {
  if (!s || !in || site < 0 || site >= s->n) return MPS_EINVAL;
  if (ml != s->dl(site) || mr != s->dr(site)) return MPS_EINVAL;
  cudaMemcpyAsync(s->G[site], in, (size_t)2 * ml * mr * s->cb, cudaMemcpyDefault, s->st);
  return sync_ok(s, s->st);
}

int mps_stats(mps_state* s, char* json, size_t cap) {
  if (!s || !json || !cap) return MPS_EINVAL;
  std::string j = "{\"gates\": " + std::to_string(s->gates) + ", \"sweeps_total\": " + std::to_string(s->sweeps_total) +
                  ", \"last_sweeps\": " + std::to_string(s->last_sweeps) + ", \"bond_dims\": [";
  for (int b = 0; b + 1 < s->n; ++b) j += (b ? ", " : "") + std::to_string(s->m[b]);
  j += "], \"status\": " + std::to_string(s->sticky) + "}";
  std::snprintf(json, cap, "%s", j.c_str());
  return j.size() < cap ? MPS_OK : MPS_EINVAL;
}

}  // extern "C"
