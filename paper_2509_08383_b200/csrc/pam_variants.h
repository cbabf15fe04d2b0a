// pam_variants.h — the compiled kernel instantiations the launcher can pick
// from.  Each table lives in its own translation unit so nvcc builds them in
// parallel.
#pragma once

namespace pam {

struct Variant {
  int elem_bytes, ntg, e, minb;  // threads per CTA, elements per thread, launch-bounds min blocks (0: auto)
  const void* fn[2];          // [P==3]
};

// Analysis kernels (analysis_kernel.cuh): convergence trace and forward-mode JVP.
struct AnalysisVariant {
  int nt, e;
  const void* trace;
  const void* jvp;
};

struct SamplerVariant {
  int nt, e;
  const void* fn[2][2];  // [P==3][GUMBEL]
};

// Two-iterations-per-exchange fp64 p = 3 kernel (cutmax_ahead_kernel.cuh).
struct AheadVariant {
  int ntg, e;
  int ctl_bytes;  // sizeof(AhCtl<ntg>)
  const void* fn;
};

extern const Variant kCutmaxVariants[];
extern const AheadVariant kAheadVariants[];
extern const int kNumAheadVariants;
extern const int kNumCutmaxVariants;
extern const AnalysisVariant kAnalysisVariants[];
extern const int kNumAnalysisVariants;
extern const SamplerVariant kSamplerVariants[];
extern const int kNumSamplerVariants;

}  // namespace pam
