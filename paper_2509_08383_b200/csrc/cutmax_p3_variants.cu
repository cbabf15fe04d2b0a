// cutmax_p3_variants.cu — fp64 instantiations of the lean p = 3 kernel
// (cutmax_p3_kernel.cuh) for the geometries of cutmax_variants_f64.cu.  The
// launcher takes one of these when p = 3 at every iteration, T >= 2 and the
// rows are 16-byte aligned; the geometry is the one the chooser picked for the
// general kernel of the same shape (matched on threads, elements, min blocks).
#include "cutmax_p3_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_P3(NTG, E, MINB) {8, NTG, E, MINB, 3, (const void*)cutmax_lean_kernel<double, NTG, E, MINB, 3>}

const LeanVariant kCutmaxP3F64[] = {
    PAM_P3(128, 8, 0),  PAM_P3(256, 16, 0), PAM_P3(512, 16, 0), PAM_P3(512, 24, 0),
    PAM_P3(512, 30, 0), PAM_P3(512, 32, 0), PAM_P3(512, 34, 0), PAM_P3(256, 38, 0),
};
const int kNumCutmaxP3F64 = sizeof(kCutmaxP3F64) / sizeof(kCutmaxP3F64[0]);

}  // namespace pam
