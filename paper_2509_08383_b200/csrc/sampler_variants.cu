// sampler_variants.cu — instantiations of sampler_rows_kernel<NT, E, P, GUMBEL, STOP>.
#include "nucleus_kernel.cuh"
#include "pam_variants.h"

namespace pam {

#define PAM_SAMPLER_VARIANT(NT, E)                                                                             \
  {                                                                                                            \
    NT, E,                                                                                                     \
        {{(const void*)sampler_rows_kernel<NT, E, 0, false>, (const void*)sampler_rows_kernel<NT, E, 0, true>},  \
         {(const void*)sampler_rows_kernel<NT, E, 3, false>, (const void*)sampler_rows_kernel<NT, E, 3, true>}}, \
    {                                                                                                          \
      (const void*)sampler_rows_kernel<NT, E, 0, false, true>,                                                 \
          (const void*)sampler_rows_kernel<NT, E, 0, true, true>                                               \
    }                                                                                                          \
  }

const SamplerVariant kSamplerVariants[] = {
    PAM_SAMPLER_VARIANT(64, 2),   PAM_SAMPLER_VARIANT(128, 8),  PAM_SAMPLER_VARIANT(256, 8),
    PAM_SAMPLER_VARIANT(256, 16), PAM_SAMPLER_VARIANT(512, 16), PAM_SAMPLER_VARIANT(512, 20),
    PAM_SAMPLER_VARIANT(512, 24), PAM_SAMPLER_VARIANT(512, 32),  // exact fits: n = 16 x 9496+, 2 x 16384
    PAM_SAMPLER_VARIANT(512, 38),
};
const int kNumSamplerVariants = sizeof(kSamplerVariants) / sizeof(kSamplerVariants[0]);

}  // namespace pam
