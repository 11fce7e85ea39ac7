// Per-precision-tier function table used by the MPS state (state.cu); the tables are
// defined in tier280.cu / tier512.cu, where every kernel is instantiated.
#pragma once
#include "common.h"

namespace mpsb {

struct Upd2Args;
struct Upd3Args;

struct TierOps {
  int L, NL;
  size_t (*upd2_ws)(const Upd2Args* a, int n);
  int (*upd2)(int p, double thr, const Upd2Args* a, int n, void* ws, cudaStream_t st, std::vector<unsigned char>& hd);
  size_t (*upd3_ws)(const Upd3Args& a);
  int (*upd3_s1)(int p, double thr, const Upd3Args& a, void* ws, cudaStream_t st, std::vector<unsigned char>& hd);
  int (*upd3_s2)(int p, double thr, const Upd3Args& a, int k1, void* ws, cudaStream_t st,
                 std::vector<unsigned char>& hd);
  void (*onesite)(int p, const uint32_t* G, uint32_t* Gout, const uint32_t* U, int nab, cudaStream_t st);
  size_t (*amp_scratch)(int maxchi, int nblocks);
  void (*amplitudes)(int p, const uint32_t* const* G, const uint32_t* const* lam, const int* dims, int n,
                     const uint8_t* bits, long long nstates, int maxchi, void* scratch, int nblocks,
                     const uint32_t* v_in, uint32_t* out, cudaStream_t st);
  void (*unitary)(int p, const uint32_t* U, int d, int* bad, cudaStream_t st);
  size_t (*transfer_scratch)(int maxchi);
  int (*rdo)(int p, int n, const uint32_t* const* Gh, const uint32_t* const* lamh, const int* dims, const int* keep,
             int k, void* scratch, int maxchi, uint32_t* out, cudaStream_t st);
  int (*transfer)(int p, int n, const uint32_t* const* Gh, const uint32_t* const* lamh, const int* dims,
                  const uint32_t* O, int s0, int k, void* scratch, int maxchi, uint32_t* out, uint32_t* den_out,
                  cudaStream_t st);
};

extern const TierOps tier280_ops;
extern const TierOps tier512_ops;
inline const TierOps& tier_ops(int p) { return p <= 280 ? tier280_ops : tier512_ops; }

}  // namespace mpsb
