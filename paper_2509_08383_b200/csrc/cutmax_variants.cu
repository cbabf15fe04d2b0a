// cutmax_variants.cu — instantiations of cutmax_rows_kernel<Elem, NT, E, P, TMA>.
// Per-CTA capacity NT*E elements; registers per thread ~ E*sizeof(Elem)/4 + ~30.
#include "cutmax_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_CUTMAX_VARIANT(ELEM, NT, E)                                                                      \
  {                                                                                                          \
    (int)sizeof(ELEM), NT, E, {                                                                              \
      {(const void*)cutmax_rows_kernel<ELEM, NT, E, 0, false>, (const void*)cutmax_rows_kernel<ELEM, NT, E, 0, true>}, \
          {(const void*)cutmax_rows_kernel<ELEM, NT, E, 3, false>,                                           \
           (const void*)cutmax_rows_kernel<ELEM, NT, E, 3, true>}                                            \
    }                                                                                                        \
  }

const Variant kCutmaxVariants[] = {
    PAM_CUTMAX_VARIANT(double, 64, 2),   PAM_CUTMAX_VARIANT(double, 128, 4),  PAM_CUTMAX_VARIANT(double, 128, 8),
    PAM_CUTMAX_VARIANT(double, 256, 8),  PAM_CUTMAX_VARIANT(double, 256, 16), PAM_CUTMAX_VARIANT(double, 512, 16),
    PAM_CUTMAX_VARIANT(double, 512, 24), PAM_CUTMAX_VARIANT(double, 512, 38),
    PAM_CUTMAX_VARIANT(float, 64, 4),    PAM_CUTMAX_VARIANT(float, 128, 8),   PAM_CUTMAX_VARIANT(float, 256, 8),
    PAM_CUTMAX_VARIANT(float, 256, 16),  PAM_CUTMAX_VARIANT(float, 512, 16),  PAM_CUTMAX_VARIANT(float, 512, 24),
    PAM_CUTMAX_VARIANT(float, 512, 40),
};
const int kNumCutmaxVariants = sizeof(kCutmaxVariants) / sizeof(kCutmaxVariants[0]);

}  // namespace pam
