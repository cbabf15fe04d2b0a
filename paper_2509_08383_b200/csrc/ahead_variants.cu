// ahead_variants.cu — instantiations of cutmax_ahead_kernel<NTG, E> (fp64, p = 3).
// Per-CTA capacity NTG*E elements.
#include "cutmax_ahead_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_AHEAD_VARIANT(NTG, E) \
  { NTG, E, (int)sizeof(AhCtl<NTG>), (const void*)cutmax_ahead_kernel<NTG, E> }

const AheadVariant kAheadVariants[] = {
    PAM_AHEAD_VARIANT(128, 8),  PAM_AHEAD_VARIANT(256, 8),  PAM_AHEAD_VARIANT(256, 16),
    PAM_AHEAD_VARIANT(512, 16), PAM_AHEAD_VARIANT(512, 24), PAM_AHEAD_VARIANT(512, 32),
    PAM_AHEAD_VARIANT(512, 34),
};
const int kNumAheadVariants = sizeof(kAheadVariants) / sizeof(kAheadVariants[0]);

}  // namespace pam
