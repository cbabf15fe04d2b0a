// cutmax_variants_f64.cu — fp64 instantiations of cutmax_rows_kernel<double, NTG, E, P, MINB, STOP>.
// Per-CTA capacity NTG*E elements; registers per thread ~ E*2 + ~60.
#include "cutmax_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_V(NTG, E, MINB, STOPFN)                                                                         \
  {                                                                                                         \
    8, NTG, E, MINB, {                                                                                      \
      (const void*)cutmax_rows_kernel<double, NTG, E, 0, MINB>,                                             \
          (const void*)cutmax_rows_kernel<double, NTG, E, 3, MINB>, STOPFN                                  \
    }                                                                                                       \
  }
// p = 3 only (the generic flow does not fit these register budgets)
#define PAM_W(NTG, E, MINB) \
  { 8, NTG, E, MINB, {nullptr, (const void*)cutmax_rows_kernel<double, NTG, E, 3, MINB>, nullptr} }
#define PAM_STOP(NTG, E, MINB) (const void*)cutmax_rows_kernel<double, NTG, E, 0, MINB, true>

const Variant kCutmaxVariantsF64[] = {
    PAM_V(64, 2, 0, PAM_STOP(64, 2, 0)),
    PAM_V(128, 4, 0, nullptr),
    PAM_V(128, 8, 0, PAM_STOP(128, 8, 0)),
    PAM_V(256, 8, 0, nullptr),
    PAM_V(256, 16, 0, PAM_STOP(256, 16, 0)),
    PAM_V(512, 16, 0, nullptr),
    PAM_V(256, 38, 0, nullptr),
    PAM_V(512, 24, 0, PAM_STOP(512, 24, 0)),
    PAM_V(512, 30, 0, nullptr),
    PAM_V(512, 34, 0, PAM_STOP(512, 34, 0)),
    PAM_V(512, 38, 0, nullptr),
    PAM_V(512, 32, 0, nullptr),  // exact fit: n = 32768 at C = 2
    PAM_V(256, 38, 2, nullptr),  // two CTAs (two rows) per SM
};
const int kNumCutmaxVariantsF64 = sizeof(kCutmaxVariantsF64) / sizeof(kCutmaxVariantsF64[0]);

}  // namespace pam
