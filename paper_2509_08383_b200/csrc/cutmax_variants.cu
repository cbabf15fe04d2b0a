// cutmax_variants.cu — instantiations of cutmax_rows_kernel<Elem, NT, E, P, TMA>.
// Per-CTA capacity NT*E elements; registers per thread ~ E*sizeof(Elem)/4 + ~30.
#include "cutmax_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_CUTMAX_VARIANT(ELEM, NTG, G, E)                                    \
  {                                                                           \
    (int)sizeof(ELEM), NTG, G, E, {                                           \
      (const void*)cutmax_rows_kernel<ELEM, NTG, G, E, 0>,                    \
          (const void*)cutmax_rows_kernel<ELEM, NTG, G, E, 3>                 \
    }                                                                         \
  }

// Per-group capacity NTG*E elements; registers per thread ~ E*sizeof(Elem)/4 + ~40.
const Variant kCutmaxVariants[] = {
    PAM_CUTMAX_VARIANT(double, 64, 1, 2),   PAM_CUTMAX_VARIANT(double, 128, 1, 4),
    PAM_CUTMAX_VARIANT(double, 128, 1, 8),  PAM_CUTMAX_VARIANT(double, 256, 1, 8),
    PAM_CUTMAX_VARIANT(double, 256, 1, 16), PAM_CUTMAX_VARIANT(double, 512, 1, 16),
    PAM_CUTMAX_VARIANT(double, 256, 1, 38), PAM_CUTMAX_VARIANT(double, 512, 1, 24),
    PAM_CUTMAX_VARIANT(double, 512, 1, 38),
    PAM_CUTMAX_VARIANT(double, 128, 2, 8),  PAM_CUTMAX_VARIANT(double, 256, 2, 16),
    PAM_CUTMAX_VARIANT(double, 256, 2, 24), PAM_CUTMAX_VARIANT(double, 256, 2, 38),
    PAM_CUTMAX_VARIANT(float, 64, 1, 4),    PAM_CUTMAX_VARIANT(float, 128, 1, 8),
    PAM_CUTMAX_VARIANT(float, 256, 1, 8),   PAM_CUTMAX_VARIANT(float, 256, 1, 16),
    PAM_CUTMAX_VARIANT(float, 512, 1, 16),  PAM_CUTMAX_VARIANT(float, 256, 1, 40),
    PAM_CUTMAX_VARIANT(float, 512, 1, 24),  PAM_CUTMAX_VARIANT(float, 512, 1, 40),
    PAM_CUTMAX_VARIANT(float, 256, 1, 76),
    PAM_CUTMAX_VARIANT(float, 256, 2, 16),  PAM_CUTMAX_VARIANT(float, 256, 2, 40),
    PAM_CUTMAX_VARIANT(float, 256, 2, 76),
};
const int kNumCutmaxVariants = sizeof(kCutmaxVariants) / sizeof(kCutmaxVariants[0]);

}  // namespace pam
