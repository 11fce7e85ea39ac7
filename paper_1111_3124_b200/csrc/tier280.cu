// Explicit instantiation of every kernel driver for the 280-bit tier.
#include "batch.cuh"
#include "svd.cuh"

namespace mpsb {
template int launch_update2_batch<Tier280>(int, int, int, int, double, const uint32_t*, const uint32_t*,
                                          const uint32_t*, const uint32_t*, const uint32_t*, const uint32_t*,
                                          const BatchOut&, void*, cudaStream_t, std::vector<unsigned char>&);
template size_t update2_workspace<Tier280>(int, int);
template size_t svd_workspace<Tier280>(int, int, int);
template int run_svd_batch<Tier280>(int, int, int, int, const uint32_t*, uint32_t*, int*, int*, void*, cudaStream_t,
                                   std::vector<unsigned char>&);
template void run_debug_mpf<Tier280>(int, int, int, const uint32_t*, const uint32_t*, uint32_t*, cudaStream_t);
}  // namespace mpsb
