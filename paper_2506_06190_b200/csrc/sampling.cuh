// Internal sampling entry shared by the MC sampler (a8) and the Poisson-disk candidates.
#pragma once
#include "nat_internal.cuh"

namespace nat {

// samples[6][M] (xyz, normal), sample_tri[M]: the a8 construction (reading R-mc-sample)
// with Philox counter (j, tag, stream_lo, stream_hi); tag 0 = boundary samples, 2 =
// Poisson-disk candidates.  Arguments are validated by the callers.
nat_status mc_sample_tagged(const nat_mesh* mesh, const nat_geom* geom, int64_t M, uint64_t seed,
                            uint64_t stream_id, uint32_t tag, double* samples, int32_t* sample_tri,
                            cudaStream_t stream);

}  // namespace nat
