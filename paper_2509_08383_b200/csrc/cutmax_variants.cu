// cutmax_variants.cu — instantiations of cutmax_rows_kernel<Elem, NTG, E, P>.
// Per-CTA capacity NTG*E elements; registers per thread ~ E*sizeof(Elem)/4 + ~50.
#include "cutmax_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_CUTMAX_VARIANT_B(ELEM, NTG, E, MINB)                                          \
  {                                                                                       \
    (int)sizeof(ELEM), NTG, E, MINB, {                                                    \
      (const void*)cutmax_rows_kernel<ELEM, NTG, E, 0, MINB>,                             \
          (const void*)cutmax_rows_kernel<ELEM, NTG, E, 3, MINB>                          \
    }                                                                                     \
  }
#define PAM_CUTMAX_VARIANT(ELEM, NTG, E) PAM_CUTMAX_VARIANT_B(ELEM, NTG, E, 0)

const Variant kCutmaxVariants[] = {
    PAM_CUTMAX_VARIANT(double, 64, 2),   PAM_CUTMAX_VARIANT(double, 128, 4),  PAM_CUTMAX_VARIANT(double, 128, 8),
    PAM_CUTMAX_VARIANT(double, 256, 8),  PAM_CUTMAX_VARIANT(double, 256, 16), PAM_CUTMAX_VARIANT(double, 512, 16),
    PAM_CUTMAX_VARIANT(double, 256, 38), PAM_CUTMAX_VARIANT(double, 512, 24), PAM_CUTMAX_VARIANT(double, 512, 30),
    PAM_CUTMAX_VARIANT(double, 512, 34), PAM_CUTMAX_VARIANT(double, 512, 38),
    PAM_CUTMAX_VARIANT(double, 512, 32),  // exact fit: n = 32768 at C = 2
    PAM_CUTMAX_VARIANT_B(double, 256, 38, 2),  // two CTAs (two rows) per SM
    PAM_CUTMAX_VARIANT(float, 64, 4),    PAM_CUTMAX_VARIANT(float, 128, 8),   PAM_CUTMAX_VARIANT(float, 256, 8),
    PAM_CUTMAX_VARIANT(float, 256, 16),  PAM_CUTMAX_VARIANT(float, 512, 16),  PAM_CUTMAX_VARIANT(float, 256, 40),
    PAM_CUTMAX_VARIANT(float, 512, 24),  PAM_CUTMAX_VARIANT(float, 512, 40),  PAM_CUTMAX_VARIANT(float, 256, 76),
    PAM_CUTMAX_VARIANT_B(float, 256, 76, 2),
    PAM_CUTMAX_VARIANT(float, 256, 64),   PAM_CUTMAX_VARIANT_B(float, 256, 64, 2),  // exact fit: 32768 at C = 2
};
const int kNumCutmaxVariants = sizeof(kCutmaxVariants) / sizeof(kCutmaxVariants[0]);

}  // namespace pam
