// Second build of the low-rank NLEM kernel (kernels_nlem_lr.cu) for the small-mu regime: with
// lambda = w / mu >= ||p|| (the reference's default mu = 1e-3) the prox scales saturate at 1 and no
// history term decays, so the ring has to hold every sweep.  R = 12 covers T <= 12; the point
// state grows to 16 fields (32 tensor-memory columns per point pair, 256 per pixel), so 8
// pixel-warps share an SM instead of 16.  Launched by the ABI after the R = 4 launch when the
// small-mu probe ran and 4 < T <= 12 (abi.cu); beyond 12 sweeps the exact tile kernel serves.
#define NLEM_LR_R 12
#define NLEM_LR_WARPS 8
#define NLEM_LR_NAME nlem_pixels_lr_r12
#define NLEM_LR_SECONDARY 1
#include "kernels_nlem_lr.cu"
