// cutmax_p3_variants_f32.cu — fp32 instantiations of the lean p = 3 kernel
// (cutmax_p3_kernel.cuh; fp32 storage and elementwise math, fp64 statistics)
// for the geometries of cutmax_variants_f32.cu.
#include "cutmax_p3_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_P3F(NTG, E, MINB) {4, NTG, E, MINB, 3, (const void*)cutmax_lean_kernel<float, NTG, E, MINB, 3>}

const LeanVariant kCutmaxP3F32[] = {
    PAM_P3F(128, 8, 0),  PAM_P3F(256, 8, 0),  PAM_P3F(256, 16, 0), PAM_P3F(512, 16, 0), PAM_P3F(256, 40, 0),
    PAM_P3F(512, 24, 0), PAM_P3F(512, 40, 0), PAM_P3F(256, 76, 0), PAM_P3F(256, 76, 2), PAM_P3F(256, 64, 0),
    PAM_P3F(256, 64, 2),
};
const int kNumCutmaxP3F32 = sizeof(kCutmaxP3F32) / sizeof(kCutmaxP3F32[0]);

}  // namespace pam
