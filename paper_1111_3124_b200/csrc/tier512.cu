// Explicit instantiation of every kernel driver for the 512-bit tier.
#include "batch.cuh"
#include "query.cuh"
#include "svd.cuh"
#include "tierops.h"
#include "update.cuh"

namespace mpsb {
template int launch_update2_batch<Tier512>(int, int, int, int, double, const uint32_t*, const uint32_t*,
                                          const uint32_t*, const uint32_t*, const uint32_t*, const uint32_t*,
                                          const BatchOut&, void*, cudaStream_t, std::vector<unsigned char>&);
template size_t update2_workspace<Tier512>(int, int);
template size_t svd_workspace<Tier512>(int, int, int);
template int run_svd_batch<Tier512>(int, int, int, int, const uint32_t*, uint32_t*, int*, int*, void*, cudaStream_t,
                                   std::vector<unsigned char>&);
template void run_debug_mpf<Tier512>(int, int, int, const uint32_t*, const uint32_t*, uint32_t*, cudaStream_t);

const TierOps tier512_ops = {
    Tier512::L, Tier512::NL,
    &upd2_workspace<Tier512>, &run_update2<Tier512>,
    &upd3_workspace<Tier512>, &launch_update3_stage1<Tier512>, &launch_update3_stage2<Tier512>,
    &run_onesite<Tier512>, &amp_scratch_bytes<Tier512>, &run_amplitudes<Tier512>, &run_unitary<Tier512>,
    &transfer_scratch_bytes<Tier512>, &run_rdo<Tier512>, &run_transfer<Tier512>,
};
}  // namespace mpsb
