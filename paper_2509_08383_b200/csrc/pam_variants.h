// pam_variants.h — the compiled kernel instantiations the launcher can pick
// from.  Each table lives in its own translation unit so nvcc builds them in
// parallel; the launcher walks kCutmaxTables.
#pragma once

namespace pam {

// One CutMax geometry: threads per CTA, elements per thread, launch-bounds
// min blocks (0: auto), and its kernels:
//   fn[0] generic p (runtime schedule), fn[1] p = 3 everywhere (analytic
//   normaliser), fn[2] generic p with early stopping (eps_stop > 0; nullptr
//   when this geometry has no such instantiation).
struct Variant {
  int elem_bytes, ntg, e, minb;
  const void* fn[3];
};

struct VariantTable {
  const Variant* v;
  int count;
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
  const void* stop[2];   // generic p with early stopping, [GUMBEL]
};

// Lean p = 3 kernels (cutmax_p3_kernel.cuh), matched to a Variant by
// (elem_bytes, ntg, e, minb).
struct LeanVariant {
  int elem_bytes, ntg, e, minb, p;  // p: the odd power at every iteration
  const void* fn;
};
// Warp-per-row kernels (cutmax_warp_kernel.cuh): rows of n <= 32 * e elements.
struct WarpVariant {
  int elem_bytes, e;
  const void* fn[2][2];  // [n == 32 * e][p = 3 everywhere]
};
extern const WarpVariant kWarpVariants[];
extern const int kNumWarpVariants;

extern const LeanVariant kCutmaxP3F64[];
extern const int kNumCutmaxP3F64;
extern const LeanVariant kCutmaxP3F32[];
extern const int kNumCutmaxP3F32;
extern const LeanVariant kCutmaxPGenF64[];
extern const int kNumCutmaxPGenF64;
extern const LeanVariant kCutmaxPMixF64[];  // P = 0: per-iteration schedule p[t]
extern const int kNumCutmaxPMixF64;

extern const Variant kCutmaxVariantsF64[];
extern const int kNumCutmaxVariantsF64;
extern const Variant kCutmaxVariantsF32[];
extern const int kNumCutmaxVariantsF32;
extern const AnalysisVariant kAnalysisVariants[];
extern const int kNumAnalysisVariants;
extern const SamplerVariant kSamplerVariants[];
extern const int kNumSamplerVariants;

}  // namespace pam
