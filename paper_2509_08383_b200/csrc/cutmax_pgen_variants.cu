// cutmax_pgen_variants.cu — the lean kernel (cutmax_p3_kernel.cuh) for the
// other fixed odd powers of the paper's Table 1 ((19,5) at
// T = 2, (19,27) at T = 3, (13,15) at T = 4, (9,15) at T = 5) and p = 5, fp64,
// at the geometries the chooser uses for n = 1024 .. 151936.
#include "cutmax_p3_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_PG(NTG, E, P) {8, NTG, E, 0, P, (const void*)cutmax_lean_kernel<double, NTG, E, 0, P>}
#define PAM_PG4(NTG, E) PAM_PG(NTG, E, 5), PAM_PG(NTG, E, 9), PAM_PG(NTG, E, 13), PAM_PG(NTG, E, 19)

const LeanVariant kCutmaxPGenF64[] = {
    PAM_PG4(512, 34), PAM_PG4(512, 32), PAM_PG4(512, 16), PAM_PG4(256, 16), PAM_PG4(256, 38),
};
const int kNumCutmaxPGenF64 = sizeof(kCutmaxPGenF64) / sizeof(kCutmaxPGenF64[0]);

}  // namespace pam
