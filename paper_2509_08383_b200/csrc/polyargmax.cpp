// polyargmax.cpp — the C++ API (include/polyargmax/polyargmax.hpp) over the C
// ABI.  Host vectors are staged to the GPU with the C ABI's host-buffer entry
// points; there is no CPU implementation of any vector operation here.
#include "../../include/polyargmax/polyargmax.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <string>

namespace polyargmax {

namespace {

struct DeviceBuffer {
  void* p = nullptr;
  explicit DeviceBuffer(std::size_t bytes) {
    if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw Error("cudaMalloc failed");
  }
  ~DeviceBuffer() {
    if (p) cudaFree(p);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void throw_status(int status, std::size_t row) {
  const int s = status & 0xff;
  const std::string msg = pam_status_string(s);
  switch (s) {
    case PAM_OK: return;
    case PAM_ERR_INVALID_PARAMS: throw InvalidParamsError(msg);
    case PAM_ERR_DEGENERATE_INPUT: throw DegenerateInputError(msg + " (row " + std::to_string(row) + ")");
    case PAM_ERR_RANGE: throw RangeError(msg + " (row " + std::to_string(row) + ")");
    case PAM_ERR_DOMAIN: throw DomainError(msg);
    case PAM_ERR_NON_FINITE: throw NonFiniteError(msg, row);
    case PAM_ERR_UNSUPPORTED: throw InvalidParamsError(msg);
    case PAM_ERR_BAD_ARGUMENT: throw InvalidParamsError(msg);
    case PAM_ERR_FORMAT: throw FormatError(msg, row);
    case PAM_ERR_SINGULAR: throw SingularityError(msg + " (row " + std::to_string(row) + ")");
    default: throw Error(msg + ": " + pam_last_cuda_error());
  }
}

std::vector<LogitVector> ingest(const std::string& path) {
  pam_ingest_info info;
  std::vector<LogitVector> out;
  int st = pam_lgt1_probe(path.c_str(), &info);
  if (st == PAM_OK) {
    std::vector<float> buf((size_t)(info.count * info.n));
    st = pam_lgt1_read(path.c_str(), buf.data(), (int64_t)buf.size(), &info);
    if (st == PAM_ERR_NON_FINITE) throw_status(st, (std::size_t)info.bad_vector);
    throw_status(st, (std::size_t)info.err_offset);
    for (int64_t r = 0; r < info.count; ++r)
      out.emplace_back(buf.begin() + r * info.n, buf.begin() + (r + 1) * info.n);
    return out;
  }
  if (st == PAM_ERR_FORMAT && info.err_offset == 0) {  // not LGT1 at all: JSON lines
    st = pam_jsonl_probe(path.c_str(), &info);
    if (st == PAM_OK) {
      std::vector<double> buf((size_t)(info.count * info.n));
      st = pam_jsonl_read(path.c_str(), buf.data(), (int64_t)buf.size(), &info);
      if (st == PAM_ERR_NON_FINITE) throw_status(st, (std::size_t)info.bad_vector);
      throw_status(st, 0);
      for (int64_t r = 0; r < info.count; ++r)
        out.emplace_back(buf.begin() + r * info.n, buf.begin() + (r + 1) * info.n);
      return out;
    }
  }
  throw_status(st, st == PAM_ERR_FORMAT ? (std::size_t)info.err_offset : 0);
  return out;
}

namespace {
using DevBuf = DeviceBuffer;
// JVPs of B directions (row-major B x n) at x; returns dZ row-major B x n
std::vector<double> jvp_rows(const LogitVector& x, const std::vector<double>& V, std::size_t B,
                             const CutMaxParams& params) {
  const std::size_t n = x.size();
  const pam_cutmax_params prm = params.lower();
  DevBuf dx(B * n * 8), dv(B * n * 8), ddz(B * n * 8), dst(B * 4);
  for (std::size_t r = 0; r < B; ++r)
    check_cuda(cudaMemcpy((double*)dx.p + r * n, x.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
  check_cuda(cudaMemcpy(dv.p, V.data(), B * n * 8, cudaMemcpyHostToDevice), "H2D");
  throw_status(pam_cutmax_jvp_batch_f64((const double*)dx.p, (const double*)dv.p, (int64_t)n, (int64_t)B,
                                        (int64_t)n, &prm, nullptr, (double*)ddz.p, (int64_t)n, (int32_t*)dst.p,
                                        nullptr));
  std::vector<double> dz(B * n);
  std::vector<int32_t> st(B);
  check_cuda(cudaMemcpy(dz.data(), ddz.p, B * n * 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(st.data(), dst.p, B * 4, cudaMemcpyDeviceToHost), "D2H");
  for (std::size_t r = 0; r < B; ++r) throw_status(st[r], r);
  return dz;
}
}  // namespace

std::vector<TraceStep> convergenceTrace(const LogitVector& x, const CutMaxParams& params) {
  const std::size_t n = x.size();
  const pam_cutmax_params prm = params.lower();
  DevBuf dx(n * 8), dout((std::size_t)prm.T * 4 * 8), dst(4);
  check_cuda(cudaMemcpy(dx.p, x.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
  throw_status(pam_convergence_trace_batch_f64((const double*)dx.p, (int64_t)n, 1, (int64_t)n, &prm,
                                               (double*)dout.p, (int32_t*)dst.p, nullptr));
  std::vector<double> out((std::size_t)prm.T * 4);
  int32_t st = 0;
  check_cuda(cudaMemcpy(out.data(), dout.p, out.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&st, dst.p, 4, cudaMemcpyDeviceToHost), "D2H");
  throw_status(st);
  std::vector<TraceStep> steps((std::size_t)prm.T);
  for (int t = 0; t < prm.T; ++t) steps[t] = {out[4 * t], out[4 * t + 1], out[4 * t + 2], out[4 * t + 3]};
  return steps;
}

std::vector<double> cutmaxJvp(const LogitVector& x, const std::vector<double>& v, const CutMaxParams& params) {
  if (v.size() != x.size()) throw InvalidParamsError("cutmaxJvp: v and x differ in length");
  return jvp_rows(x, v, 1, params);
}

std::vector<double> cutmaxJacobian(const LogitVector& x, const CutMaxParams& params) {
  const std::size_t n = x.size();
  std::vector<double> I(n * n, 0.0);
  for (std::size_t j = 0; j < n; ++j) I[j * n + j] = 1.0;
  const std::vector<double> cols = jvp_rows(x, I, n, params);  // row j = J e_j (column j of J)
  std::vector<double> J(n * n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) J[i * n + j] = cols[j * n + i];
  return J;
}

void writeLgt1(const std::string& path, const std::vector<LogitVector>& vectors) {
  const std::size_t n = vectors.empty() ? 0 : vectors[0].size();
  std::vector<float> buf;
  buf.reserve(vectors.size() * n);
  for (const auto& v : vectors) {
    if (v.size() != n) throw InvalidParamsError("writeLgt1: vectors of different lengths");
    for (double x : v) buf.push_back((float)x);
  }
  throw_status(pam_lgt1_write(path.c_str(), buf.data(), (int64_t)vectors.size(), (int64_t)n));
}

ApproxConfig ApproxConfig::invsqrtPreset(int alphaBits) {
  ApproxConfig c;
  c.alphaBits = alphaBits;
  c.iterations = alphaBits <= 7 ? 5 : alphaBits <= 9 ? 6 : alphaBits <= 11 ? 7 : 8;  // Table 3
  c.lo = 0.25;
  c.hi = 1.0;
  return c;
}

ApproxConfig ApproxConfig::invPreset(int alphaBits) {
  ApproxConfig c;
  c.alphaBits = alphaBits;
  // on [1/2,1) the error after d+1 factors is (1-x)^(2^(d+1)) <= 2^-(2^(d+1))
  int d = 0;
  while ((1 << (d + 1)) < alphaBits + 1) ++d;
  c.iterations = d < 2 ? 2 : d;
  c.lo = 0.5;
  c.hi = 1.0;
  return c;
}

static pam_approx_config lower_approx(const ApproxConfig& a) {
  pam_approx_config r{};
  r.iterations = a.iterations;
  r.alpha_bits = a.alphaBits;
  r.rescale = static_cast<int32_t>(a.rescale);
  r.scale_log2 = a.scaleLog2;
  r.lo = a.lo;
  r.hi = a.hi;
  return r;
}

pam_cutmax_params CutMaxParams::lower() const {
  if (T < 1 || T > PAM_MAX_T) throw InvalidParamsError("T must be in [1, 16] (SPEC.md:67)");
  auto pick = [&](auto const& v, int t) {
    if (v.empty()) throw InvalidParamsError("empty schedule");
    if (v.size() == 1) return v[0];
    if ((int)v.size() != T) throw InvalidParamsError("schedule length must be 1 or T (SPEC.md:124)");
    return v[t];
  };
  pam_cutmax_params r;
  pam_default_params(&r, T, 3, 5.0);
  r.flags = (checked ? 0 : PAM_F_UNCHECKED) | (guarantee ? PAM_F_GUARANTEE : 0) | (normalize ? 0 : PAM_F_NO_NORMALIZE);
  r.eps_var = epsVar;
  r.eps_stop = epsStop;
  r.invsqrt_mode = static_cast<int32_t>(invsqrtMode);
  r.inv_mode = static_cast<int32_t>(invMode);
  for (int t = 0; t < T; ++t) {
    r.p[t] = pick(p, t);
    r.c[t] = pick(c, t);
    r.invsqrt[t] = lower_approx(pick(invsqrt, t));
  }
  r.inv = lower_approx(inv);
  return r;
}

ScoreVector cutmax(const LogitVector& x, const CutMaxParams& params) {
  const pam_cutmax_params prm = params.lower();
  ScoreVector out;
  out.values.resize(x.size());
  out.normalized = params.normalize;
  std::int32_t am = -1, st = 0;
  const int rc = pam_cutmax_batch_host_f64(x.data(), 1, (int64_t)x.size(), &prm, out.values.data(), &am, &st);
  throw_status(rc, 0);
  throw_status(st, 0);
  out.argmax = am;
  out.tieWarning = (st & PAM_ROW_FLAG_TIE) != 0;
  return out;
}

std::pair<std::vector<double>, ResidualStats> cutmaxStep(const std::vector<double>& y, int p, double c) {
  CutMaxParams prm;
  prm.p = {p};
  prm.c = {c};
  prm.T = 1;
  prm.checked = false;
  prm.normalize = false;
  const pam_cutmax_params lp = prm.lower();
  const std::size_t n = y.size();
  DeviceBuffer dx(n * 8), dz(n * 8), ds(8), dst(16), dstat(16);
  check_cuda(cudaMemcpy(dx.p, y.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
  throw_status(pam_cutmax_batch_f64((const double*)dx.p, (int64_t)n, 1, (int64_t)n, &lp, (double*)dz.p, (int64_t)n,
                                    (int32_t*)ds.p, (int32_t*)dst.p, (double*)dstat.p, nullptr));
  std::vector<double> next(n);
  double stats[2];
  std::int32_t status = 0;
  check_cuda(cudaMemcpy(next.data(), dz.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(stats, dstat.p, 16, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&status, dst.p, 4, cudaMemcpyDeviceToHost), "D2H");
  throw_status(status, 0);
  ResidualStats rs;
  rs.mu = stats[0];
  rs.s2 = stats[1];
  // Residuals r_i = (y_i - mu)/s and the non-top dispersion U
  // are diagnostics of the SPEC's cutmaxStep contract, derived from the GPU's
  // mu and s2.
  const double inv_s = 1.0 / std::sqrt(rs.s2);
  std::size_t top = 0;
  for (std::size_t i = 1; i < n; ++i)
    if (y[i] > y[top]) top = i;
  rs.residuals.resize(n);
  double rsum = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    rs.residuals[i] = (y[i] - rs.mu) * inv_s;
    if (i != top) rsum += rs.residuals[i];
  }
  const double rbar = rsum / (double)(n - 1);
  for (std::size_t i = 0; i < n; ++i)
    if (i != top) rs.dispersion += (rs.residuals[i] - rbar) * (rs.residuals[i] - rbar);
  return {std::move(next), std::move(rs)};
}

static SampleOutcome sample_one(const LogitVector& x, const pam_sampler_cfg& cfg, const CutMaxParams& params,
                                bool gumbel, std::uint64_t row) {
  const pam_cutmax_params prm = params.lower();
  const std::size_t n = x.size();
  // The kernel keys the noise by seed ^ row_index; fold the requested row in.
  pam_sampler_cfg c2 = cfg;
  c2.seed = cfg.seed ^ row;
  DeviceBuffer dx(n * 8), dz(n * 8), dtok(4), dins(4), dst(4);
  check_cuda(cudaMemcpy(dx.p, x.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
  const int rc = gumbel ? pam_gumbel_sample_batch_f64((const double*)dx.p, (int64_t)n, 1, (int64_t)n, &c2, &prm,
                                                      (int32_t*)dtok.p, (uint8_t*)dins.p, (double*)dz.p,
                                                      (int64_t)n, (int32_t*)dst.p, nullptr)
                        : pam_nucleus_sample_batch_f64((const double*)dx.p, (int64_t)n, 1, (int64_t)n, &c2, &prm,
                                                       (int32_t*)dtok.p, (uint8_t*)dins.p, (double*)dz.p,
                                                       (int64_t)n, (int32_t*)dst.p, nullptr);
  throw_status(rc, 0);
  SampleOutcome out;
  out.onehot.resize(n);
  std::int32_t tok = -1, st = 0;
  std::uint8_t ins = 0;
  check_cuda(cudaMemcpy(out.onehot.data(), dz.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&tok, dtok.p, 4, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&ins, dins.p, 1, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&st, dst.p, 4, cudaMemcpyDeviceToHost), "D2H");
  throw_status(st, 0);
  out.tokenIndex = tok;
  out.insideNucleus = ins != 0;
  out.tieWarning = (st & PAM_ROW_FLAG_TIE) != 0;
  return out;
}

SampleOutcome nucleusOneShotSample(const LogitVector& x, const SamplerConfig& cfg, const CutMaxParams& params,
                                   std::uint64_t row_index) {
  pam_sampler_cfg c{cfg.p, cfg.q, cfg.alpha, cfg.seed, cfg.draw};
  return sample_one(x, c, params, false, row_index);
}

SampleOutcome gumbelMaxSample(const LogitVector& x, const CutMaxParams& params, std::uint64_t seed, double nucleus_p) {
  pam_sampler_cfg c{nucleus_p, nucleus_p, 0.0, seed, 0};
  return sample_one(x, c, params, true, 0);
}

NucleusSet nucleusSet(const LogitVector& x, double p) {
  const std::size_t n = x.size();
  DeviceBuffer dx(n * 8), dcut(8), dmass(8), dsize(4), dst(4);
  check_cuda(cudaMemcpy(dx.p, x.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
  throw_status(pam_nucleus_set_batch_f64((const double*)dx.p, (int64_t)n, 1, (int64_t)n, p, (double*)dcut.p,
                                         (int32_t*)dsize.p, (double*)dmass.p, (int32_t*)dst.p, nullptr),
               0);
  NucleusSet out;
  std::int32_t st = 0, size = 0;
  check_cuda(cudaMemcpy(&st, dst.p, 4, cudaMemcpyDeviceToHost), "D2H");
  throw_status(st, 0);
  check_cuda(cudaMemcpy(&out.cutoff, dcut.p, 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&out.mass, dmass.p, 8, cudaMemcpyDeviceToHost), "D2H");
  check_cuda(cudaMemcpy(&size, dsize.p, 4, cudaMemcpyDeviceToHost), "D2H");
  out.size = size;
  return out;
}

double goldschmidtInv(double x, const ApproxConfig& cfg) {
  const pam_approx_config c = lower_approx(cfg);
  double out = 0.0;
  throw_status(pam_goldschmidt_inv(x, &c, &out));
  return out;
}

double goldschmidtInvSqrt(double x, const ApproxConfig& cfg) {
  const pam_approx_config c = lower_approx(cfg);
  double out = 0.0;
  throw_status(pam_goldschmidt_invsqrt(x, &c, &out));
  return out;
}

double nucleusAlpha(double p, double q) {
  double out = 0.0;
  throw_status(pam_nucleus_alpha(p, q, &out));
  return out;
}

double betaInverseCdf(double u, double alpha) {
  if (!(u >= 0.0 && u <= 1.0) || !(alpha > 0.0)) throw DomainError("betaInverseCdf needs u in [0,1], alpha > 0");
  return pam_beta_inverse_cdf(u, alpha);
}

double gumbelFromUniform(double u) {
  double out = 0.0;
  throw_status(pam_gumbel_from_uniform(u, &out));
  return out;
}

void cutmax_batch(const double* X, std::size_t B, std::size_t n, const CutMaxParams& params, double* Z,
                  std::int32_t* argmax) {
  const pam_cutmax_params prm = params.lower();
  std::vector<std::int32_t> st(B);
  throw_status(pam_cutmax_batch_host_f64(X, (int64_t)B, (int64_t)n, &prm, Z, argmax, st.data()));
  for (std::size_t r = 0; r < B; ++r) throw_status(st[r], r);
}

void cutmax_batch_device(const double* dX, std::size_t B, std::size_t n, std::size_t ld, const CutMaxParams& params,
                         double* dZ, std::int32_t* dArgmax, std::int32_t* dStatus, void* stream) {
  const pam_cutmax_params prm = params.lower();
  throw_status(pam_cutmax_batch_f64(dX, (int64_t)ld, (int64_t)B, (int64_t)n, &prm, dZ, (int64_t)ld, dArgmax, dStatus,
                                    nullptr, stream));
}

void nucleus_sample_batch_device(const double* dX, std::size_t B, std::size_t n, std::size_t ld,
                                 const SamplerConfig& cfg, const CutMaxParams& params, std::int32_t* dToken,
                                 std::uint8_t* dInside, std::int32_t* dStatus, void* stream) {
  const pam_cutmax_params prm = params.lower();
  pam_sampler_cfg c{cfg.p, cfg.q, cfg.alpha, cfg.seed, cfg.draw};
  throw_status(pam_nucleus_sample_batch_f64(dX, (int64_t)ld, (int64_t)B, (int64_t)n, &c, &prm, dToken, dInside,
                                            nullptr, 0, dStatus, stream));
}

}  // namespace polyargmax
