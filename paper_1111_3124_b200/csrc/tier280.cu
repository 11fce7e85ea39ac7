// Explicit instantiation of every kernel driver for the 280-bit tier.
#include "batch.cuh"
#include "query.cuh"
#include "svd.cuh"
#include "tierops.h"
#include "update.cuh"

namespace mpsb {
template int launch_update2_batch<Tier280>(int, int, int, int, double, const uint32_t*, const uint32_t*,
                                          const uint32_t*, const uint32_t*, const uint32_t*, const uint32_t*,
                                          const BatchOut&, void*, cudaStream_t, std::vector<unsigned char>&);
template size_t update2_workspace<Tier280>(int, int);
template size_t svd_workspace<Tier280>(int, int, int);
template int run_svd_batch<Tier280>(int, int, int, int, const uint32_t*, uint32_t*, int*, int*, void*, cudaStream_t,
                                   std::vector<unsigned char>&);
template void run_debug_mpf<Tier280>(int, int, int, const uint32_t*, const uint32_t*, uint32_t*, cudaStream_t);

const TierOps tier280_ops = {
    Tier280::L, Tier280::NL,
    &upd2_workspace<Tier280>, &run_update2<Tier280>,
    &upd3_workspace<Tier280>, &launch_update3_stage1<Tier280>, &launch_update3_stage2<Tier280>,
    &run_onesite<Tier280>, &amp_scratch_bytes<Tier280>, &run_amplitudes<Tier280>, &run_unitary<Tier280>,
    &transfer_scratch_bytes<Tier280>, &run_rdo<Tier280>, &run_transfer<Tier280>,
};
}  // namespace mpsb
