// polyargmax/polyargmax.hpp — drop-in C++ API of the B200 CutMax decoding core.
//
// Mirrors the reference's C++ entry points for the hot path (SPEC.md; the
// reference ships them as specifications only):
//   cutmax                 SPEC.md:60-69     (Alg. 1)
//   cutmaxStep
//   goldschmidtInv
//   goldschmidtInvSqrt
//   gumbelFromUniform
//   gumbelMaxSample
//   betaInverseCdf
//   nucleusAlpha
//   nucleusOneShotSample   SPEC.md:437-445   (Alg. 3)
// plus batch forms justified by the SPEC's concurrency model.
// Everything that touches a logit vector runs on the GPU through the C ABI
// (include/pam_c_api.h); errors are thrown as the types in errors.hpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "../pam_c_api.h"
#include "errors.hpp"

namespace polyargmax {

/// LogitVector: n >= 2 finite scores.
using LogitVector = std::vector<double>;

enum class ApproxMode { Exact = PAM_MODE_EXACT, Poly = PAM_MODE_POLY };
enum class Rescale { Auto = PAM_RESCALE_AUTO, Static = PAM_RESCALE_STATIC, None = PAM_RESCALE_NONE };

/// ApproxConfig.
struct ApproxConfig {
  int iterations = 5;
  double lo = 0.25, hi = 1.0;  // inputRange after rescaling
  int alphaBits = 7;
  Rescale rescale = Rescale::Auto;
  int scaleLog2 = 0;  // Rescale::Static: bound b = 2^scaleLog2

  /// Table 3 presets: invsqrt iterations 5/6/7/8 for alpha 7/9/11/13.
  static ApproxConfig invsqrtPreset(int alphaBits);
  /// Goldschmidt inverse preset on [1/2, 1) after AUTO rescaling.
  static ApproxConfig invPreset(int alphaBits);
};

/// CutMaxParams with the SPEC.md:121-127 decisions.
struct CutMaxParams {
  std::vector<int> p{3};       // odd >= 3, scalar or length-T schedule
  std::vector<double> c{5.0};  // > 0, scalar or length-T schedule
  int T = 4;
  bool checked = true;     // false = "unchecked" mode: even p allowed
  bool guarantee = false;  // require c > sqrt(n-1)
  bool normalize = true;   // false: return Y^(T+1) (used by cutmaxStep)
  double epsVar = 1e-24;
  double epsStop = 0.0;    // SPEC.md:126 (0 = off)
  ApproxMode invsqrtMode = ApproxMode::Exact;
  ApproxMode invMode = ApproxMode::Exact;
  std::vector<ApproxConfig> invsqrt{ApproxConfig::invsqrtPreset(7)};  // scalar or per iteration
  ApproxConfig inv = ApproxConfig::invPreset(7);

  /// Lower to the C ABI struct (broadcasting scalars to length T).
  pam_cutmax_params lower() const;
};

/// ScoreVector plus the argmax the kernel computes anyway and
/// the TieWarning (input top-2 gap < 1e-9; reported, not thrown).
struct ScoreVector {
  std::vector<double> values;
  bool normalized = true;
  int argmax = -1;
  bool tieWarning = false;
};

/// ResidualStats.
struct ResidualStats {
  double mu = 0, s2 = 0;
  std::vector<double> residuals;
  double dispersion = 0;
};

/// SamplerConfig.
struct SamplerConfig {
  double p = 0.9;
  double q = 0.9;
  double alpha = 0.0;  // <= 0: derive ln(1-q)/ln(p)
  std::uint64_t seed = 0;
  std::uint64_t draw = 0;
};

/// SampleOutcome plus the TieWarning of the perturbed vector x + G.
struct SampleOutcome {
  std::vector<double> onehot;
  int tokenIndex = -1;
  bool insideNucleus = false;
  bool tieWarning = false;
};

/// The top-p nucleus itself (smallest prefix of the descending
/// softmax with cumulative mass >= p, ties included): entry k is inside <=>
/// x[k] >= cutoff.  The ground truth of violationExperiment.
struct NucleusSet {
  double cutoff = 0.0;
  int size = 0;
  double mass = 0.0;
};

// ---- single-vector API (host vectors; GPU underneath) ----------------------
ScoreVector cutmax(const LogitVector& x, const CutMaxParams& params);
std::pair<std::vector<double>, ResidualStats> cutmaxStep(const std::vector<double>& y, int p, double c);
SampleOutcome nucleusOneShotSample(const LogitVector& x, const SamplerConfig& cfg, const CutMaxParams& params,
                                   std::uint64_t row_index = 0);
SampleOutcome gumbelMaxSample(const LogitVector& x, const CutMaxParams& params, std::uint64_t seed,
                              double nucleus_p = 0.9);
NucleusSet nucleusSet(const LogitVector& x, double p);

// ---- scalar API ------------------------------------------------------------
double goldschmidtInv(double x, const ApproxConfig& cfg);
double goldschmidtInvSqrt(double x, const ApproxConfig& cfg);
double nucleusAlpha(double p, double q);
double betaInverseCdf(double u, double alpha);
double gumbelFromUniform(double u);

// ---- batch API -------------------------------------------------------------
/// Host buffers (row-major B x n).  Throws on the first failing row.
void cutmax_batch(const double* X, std::size_t B, std::size_t n, const CutMaxParams& params, double* Z,
                  std::int32_t* argmax);
/// Device buffers, stream-ordered; per-row status lands in d_status (no throw
/// for data errors).  Throws only for invalid params / launch failures.
void cutmax_batch_device(const double* dX, std::size_t B, std::size_t n, std::size_t ld, const CutMaxParams& params,
                         double* dZ, std::int32_t* dArgmax, std::int32_t* dStatus, void* stream);
void nucleus_sample_batch_device(const double* dX, std::size_t B, std::size_t n, std::size_t ld,
                                 const SamplerConfig& cfg, const CutMaxParams& params, std::int32_t* dToken,
                                 std::uint8_t* dInside, std::int32_t* dStatus, void* stream);

// ---- analysis ---------------------------------------------------
/// One convergenceTrace entry: mu, s2, the non-top dispersion U
/// and the fraction of entries below the mean (Fig. 3).
struct TraceStep {
  double mu = 0.0, s2 = 0.0, dispersion = 0.0, fractionBelowMean = 0.0;
};
std::vector<TraceStep> convergenceTrace(const LogitVector& x, const CutMaxParams& params);
/// cutmaxJvp: forward-mode d cutmax(x)/dx . v on the GPU.
/// Throws SingularityError if s2 < epsVar anywhere on the path.
std::vector<double> cutmaxJvp(const LogitVector& x, const std::vector<double>& v, const CutMaxParams& params);
/// cutmaxJacobian: n JVPs with the basis directions, one batched launch.
/// Row-major n x n, J[i][j] = dZ_i / dx_j.
std::vector<double> cutmaxJacobian(const LogitVector& x, const CutMaxParams& params);

// ---- logit files -----------------------------------------
/// ingest: an LGT1 file (detected by its magic) or JSON lines.
/// Throws FormatError(byte offset) / NonFiniteError(vector index).
std::vector<LogitVector> ingest(const std::string& path);
/// LGT1 writer: values are stored as float32; ingest(write(v)) == v bit-exact for
/// float-representable inputs.
void writeLgt1(const std::string& path, const std::vector<LogitVector>& vectors);

/// Map a pam_status to the matching errors.hpp exception (no-op for PAM_OK).
/// `where` is the row / vector index, or the byte offset for PAM_ERR_FORMAT.
void throw_status(int status, std::size_t where = 0);

}  // namespace polyargmax
