// cutmax_warp_variants.cu — instantiations of the warp-per-row kernel
// (cutmax_warp_kernel.cuh): elements per lane E for fp64 and fp32, p = 3
// everywhere (analytic normaliser) and the runtime-schedule flow, rows that
// fill the 32 x E slots exactly (no phantom predicates) or not.
#include "cutmax_warp_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_WV(T, B, E)                                                                                 \
  {B, E,                                                                                                \
   {{(const void*)cutmax_warp_kernel<T, E, 0, false>, (const void*)cutmax_warp_kernel<T, E, 3, false>}, \
    {(const void*)cutmax_warp_kernel<T, E, 0, true>, (const void*)cutmax_warp_kernel<T, E, 3, true>}}}

const WarpVariant kWarpVariants[] = {
    PAM_WV(double, 8, 4),  PAM_WV(double, 8, 8),  PAM_WV(double, 8, 16), PAM_WV(double, 8, 32), PAM_WV(double, 8, 48),
    PAM_WV(float, 4, 8),   PAM_WV(float, 4, 16),  PAM_WV(float, 4, 32),  PAM_WV(float, 4, 64),  PAM_WV(float, 4, 96),
};
const int kNumWarpVariants = sizeof(kWarpVariants) / sizeof(kWarpVariants[0]);

}  // namespace pam
