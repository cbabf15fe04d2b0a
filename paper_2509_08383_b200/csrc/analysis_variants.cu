// analysis_variants.cu — instantiations of the analysis kernels (analysis_kernel.cuh).
#include "analysis_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_ANALYSIS_VARIANT(NT, E) \
  { NT, E, (const void*)trace_rows_kernel<NT, E>, (const void*)jvp_rows_kernel<NT, E> }

const AnalysisVariant kAnalysisVariants[] = {
    PAM_ANALYSIS_VARIANT(256, 2), PAM_ANALYSIS_VARIANT(512, 4), PAM_ANALYSIS_VARIANT(512, 8),
    PAM_ANALYSIS_VARIANT(512, 16), PAM_ANALYSIS_VARIANT(512, 20),
};
const int kNumAnalysisVariants = sizeof(kAnalysisVariants) / sizeof(kAnalysisVariants[0]);

}  // namespace pam
