// cutmax_p3_variants.cu — instantiations of the lean p = 3 kernel
// (cutmax_p3_kernel.cuh) for the fp64 geometries of cutmax_variants_f64.cu.
// The launcher takes one of these when p = 3 at every iteration, T >= 2 and
// the rows are 16-byte aligned; the geometry (and its occupancy) is the one the
// chooser picked for the general kernel of the same shape.
#include "cutmax_p3_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_P3(NTG, E) {8, NTG, E, 0, (const void*)cutmax_p3_kernel<double, NTG, E>}

const LeanVariant kCutmaxP3F64[] = {
    PAM_P3(128, 8), PAM_P3(256, 16), PAM_P3(512, 16), PAM_P3(512, 24),
    PAM_P3(512, 30), PAM_P3(512, 32), PAM_P3(512, 34), PAM_P3(256, 38),
};
const int kNumCutmaxP3F64 = sizeof(kCutmaxP3F64) / sizeof(kCutmaxP3F64[0]);

}  // namespace pam
