// Register-tiled specialised kernels (filled in by the optimisation pass).
#include "launch.h"

namespace nlemk {

bool admm_fast_supported(const AdmmLaunch&) { return false; }
cudaError_t launch_admm_fast(const AdmmLaunch&, cudaStream_t) { return cudaErrorNotSupported; }
bool nlem_fast_supported(const NlemLaunch&) { return false; }
cudaError_t launch_nlem_fast(const NlemLaunch&, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace nlemk
