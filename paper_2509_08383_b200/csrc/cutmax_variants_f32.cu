// cutmax_variants_f32.cu — fp32 instantiations of cutmax_rows_kernel<float, NTG, E, P, MINB, STOP>.
#include "cutmax_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_V(NTG, E, MINB, STOPFN)                                                                        \
  {                                                                                                        \
    4, NTG, E, MINB, {                                                                                     \
      (const void*)cutmax_rows_kernel<float, NTG, E, 0, MINB>,                                             \
          (const void*)cutmax_rows_kernel<float, NTG, E, 3, MINB>, STOPFN                                  \
    }                                                                                                      \
  }
#define PAM_STOP(NTG, E, MINB) (const void*)cutmax_rows_kernel<float, NTG, E, 0, MINB, true>

const Variant kCutmaxVariantsF32[] = {
    PAM_V(64, 4, 0, PAM_STOP(64, 4, 0)),
    PAM_V(128, 8, 0, nullptr),
    PAM_V(256, 8, 0, PAM_STOP(256, 8, 0)),
    PAM_V(256, 16, 0, nullptr),
    PAM_V(512, 16, 0, PAM_STOP(512, 16, 0)),
    PAM_V(256, 40, 0, nullptr),
    PAM_V(512, 24, 0, nullptr),
    PAM_V(512, 40, 0, PAM_STOP(512, 40, 0)),
    PAM_V(256, 76, 0, nullptr),
    PAM_V(256, 76, 2, nullptr),
    PAM_V(256, 64, 0, nullptr),  // exact fit: 32768 at C = 2
    PAM_V(256, 64, 2, nullptr),
};
const int kNumCutmaxVariantsF32 = sizeof(kCutmaxVariantsF32) / sizeof(kCutmaxVariantsF32[0]);

}  // namespace pam
