// cutmax_pmix_variants.cu — the lean kernel (cutmax_p3_kernel.cuh) for mixed
// schedules p[t] (P = 0): the paper's HE schedule p = [16, 4, 4, 6]
// and any other per-iteration powers, fp64, at the geometries the
// chooser uses for n = 32768 and 151936.
#include "cutmax_p3_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_PM(NTG, E) {8, NTG, E, 0, 0, (const void*)cutmax_lean_kernel<double, NTG, E, 0, 0>}

const LeanVariant kCutmaxPMixF64[] = {PAM_PM(512, 34), PAM_PM(512, 32)};
const int kNumCutmaxPMixF64 = sizeof(kCutmaxPMixF64) / sizeof(kCutmaxPMixF64[0]);

}  // namespace pam
