// k3d_perks.cu — variant (c) PERKS for 3D stencils (partially cached plane streaming).
// Placeholder plan until the kernel lands: reports "not planned" so AUTO picks PERSISTENT.
#include "internal.h"

namespace perks {

Plan plan_perks3d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  (void)p;
  pl.why = "perks3d: not built yet";
  return pl;
}

cudaError_t run_perks3d(const Problem &, const Plan &, const void *, void *, void *, int64_t,
                        cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace perks
