// test_cpp_api.cpp — runtime test of the drop-in C++ API (include/polyargmax/polyargmax.hpp)
// as a C++20 consumer links it: every entry point a reference-side caller uses
// (SPEC.md:60-79 cutmax / cutmaxStep, 157-175 scalars, 397-445 samplers, the
// batch forms, 101-109 convergenceTrace, 491-506 JVP, 543-551 ingest), checked
// against the CPU oracle (oracle/liboracle.so, test infrastructure) and the SPEC's
// examples, plus every exception type the API can throw.
//
// Built by CMake (tests/cpp, target test_cpp_api) or tests/test_cpp_api.py; needs a GPU to run.
#include <polyargmax/polyargmax.hpp>

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

extern "C" {
#include "../../oracle/oracle.h"
}

namespace pa = polyargmax;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                                             \
  do {                                                               \
    if (cond) {                                                      \
      ++g_pass;                                                      \
    } else {                                                         \
      ++g_fail;                                                      \
      std::fprintf(stderr, "FAIL %s:%d: %s  ", __FILE__, __LINE__, #cond); \
      std::fprintf(stderr, __VA_ARGS__);                             \
      std::fprintf(stderr, "\n");                                    \
    }                                                                \
  } while (0)

static std::vector<double> gaussian(std::size_t n, unsigned seed, double sigma = 3.0) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> d(0.0, sigma);
  std::vector<double> x(n);
  for (auto& v : x) v = d(g);
  return x;
}

static double normwise(const double* a, const double* b, std::size_t n) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < n; ++i) {
    num = std::fmax(num, std::fabs(a[i] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return num / den;
}

template <typename E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void test_cutmax_vs_oracle() {
  const pa::CutMaxParams prm;  // p = 3, c = 5, T = 4
  const auto cp = prm.lower();
  for (std::size_t n : {2u, 1024u, 32768u, 151936u}) {
    const auto x = gaussian(n, 7 + (unsigned)n);
    const pa::ScoreVector sv = pa::cutmax(x, prm);
    std::vector<double> zr(n);
    int32_t amr = -1;
    const int st = orc_cutmax(x.data(), (int64_t)n, &cp, zr.data(), &amr, nullptr, nullptr);
    CHECK((st & 0xff) == 0, "oracle status %d", st);
    CHECK(sv.argmax == amr, "n=%zu argmax %d vs %d", n, sv.argmax, amr);
    const double e = normwise(sv.values.data(), zr.data(), n);
    CHECK(e <= 1e-12, "n=%zu normwise %.3e", n, e);
    double s = 0;
    for (double v : sv.values) s += v;
    CHECK(std::fabs(s - 1.0) <= 1e-9, "sum Z = %.17g", s);
    CHECK(sv.tieWarning == ((st & PAM_ROW_FLAG_TIE) != 0), "tie flag");
  }
  // x = [5, 2, 1], T = 1 -> argmax 0, sum 1
  pa::CutMaxParams p1;
  p1.T = 1;
  const auto sv = pa::cutmax({5.0, 2.0, 1.0}, p1);
  CHECK(sv.argmax == 0, "argmax %d", sv.argmax);
  CHECK(std::fabs(sv.values[0] + sv.values[1] + sv.values[2] - 1.0) <= 1e-12, "sum");
  // TieWarning: duplicated maximum
  auto x = gaussian(4096, 3);
  x[100] = x[4000] = 50.0;
  const auto tv = pa::cutmax(x, prm);
  CHECK(tv.tieWarning && tv.argmax == 100, "tie %d argmax %d", (int)tv.tieWarning, tv.argmax);
  // schedules and polynomial scalars (Table 1 / Table 3 settings)
  pa::CutMaxParams p2;
  p2.p = {13};
  p2.c = {15.0};
  p2.invsqrtMode = pa::ApproxMode::Poly;
  p2.invMode = pa::ApproxMode::Poly;
  const auto y = gaussian(32768, 11);
  const auto sv2 = pa::cutmax(y, p2);
  const auto cp2 = p2.lower();
  std::vector<double> zr(y.size());
  int32_t am2 = -1;
  orc_cutmax(y.data(), (int64_t)y.size(), &cp2, zr.data(), &am2, nullptr, nullptr);
  CHECK(sv2.argmax == am2, "p=13 argmax %d vs %d", sv2.argmax, am2);
  const double e2 = normwise(sv2.values.data(), zr.data(), y.size());
  CHECK(e2 <= 1e-12 * 13 * 13 * 13 * 13 / 81, "p=13 poly normwise %.3e", e2);
}

static void test_cutmax_step() {
  // y = [1, -1], c = 5, p = 3 -> residuals (1, -1), next = (1.728, 0.512)
  const auto [next, rs] = pa::cutmaxStep({1.0, -1.0}, 3, 5.0);
  CHECK(next.size() == 2 && std::fabs(next[0] - 1.728) < 1e-12 && std::fabs(next[1] - 0.512) < 1e-12,
        "next %.17g %.17g", next[0], next[1]);
  CHECK(std::fabs(rs.residuals[0] - 1.0) < 1e-12 && std::fabs(rs.residuals[1] + 1.0) < 1e-12, "residuals");
  // against the oracle on a longer vector
  const auto y = gaussian(20000, 5);
  const auto [nx, st] = pa::cutmaxStep(y, 3, 5.0);
  std::vector<double> nr(y.size()), rr(y.size());
  double mu, s2, disp;
  orc_cutmax_step(y.data(), (int64_t)y.size(), 3, 5.0, 1e-24, nr.data(), rr.data(), &mu, &s2, &disp);
  CHECK(normwise(nx.data(), nr.data(), y.size()) <= 1e-12, "step next");
  CHECK(std::fabs(st.mu - mu) <= 1e-12 * std::sqrt(s2) && std::fabs(st.s2 - s2) <= 1e-12 * s2, "step moments");
}

static void test_samplers() {
  const pa::CutMaxParams prm;
  const auto cp = prm.lower();
  const auto x = gaussian(32768, 21, 2.0);
  for (double p : {0.9, 0.95}) {
    pa::SamplerConfig cfg;
    cfg.p = p;
    cfg.seed = 2509;
    const auto so = pa::nucleusOneShotSample(x, cfg, prm, 3);
    pam_sampler_cfg sc{};
    sc.p = p;
    sc.q = cfg.q;
    sc.alpha = orc_nucleus_alpha(p, cfg.q);
    sc.seed = cfg.seed;
    sc.draw = 0;
    int32_t tok = -1;
    uint8_t ins = 0;
    const int st = orc_sample(x.data(), (int64_t)x.size(), &sc, &cp, 3, 0, &tok, &ins, nullptr);
    CHECK((st & 0xff) == 0, "oracle sample status %d", st);
    CHECK(so.tokenIndex == tok && so.insideNucleus == (ins != 0), "p=%.2f token %d vs %d", p, so.tokenIndex, tok);
    CHECK(so.onehot.size() == x.size() && so.onehot[so.tokenIndex] > 0.0, "one-hot");
  }
  const auto g = pa::gumbelMaxSample(x, prm, 77);
  pam_sampler_cfg sc{};
  sc.p = 0.9;
  sc.q = 0.9;
  sc.alpha = 1.0;
  sc.seed = 77;
  int32_t tok = -1;
  uint8_t ins = 0;
  orc_sample(x.data(), (int64_t)x.size(), &sc, &cp, 0, 1, &tok, &ins, nullptr);
  CHECK(g.tokenIndex == tok, "gumbel token %d vs %d", g.tokenIndex, tok);
  // the nucleus itself: bit-exact against the oracle's sort-and-walk
  for (double p : {0.9, 0.95}) {
    const pa::NucleusSet ns = pa::nucleusSet(x, p);
    double cut = 0, mass = 0;
    int32_t size = 0;
    orc_nucleus_set(x.data(), (int64_t)x.size(), p, &cut, &size, &mass);
    CHECK(ns.cutoff == cut && ns.size == size && ns.mass == mass, "nucleusSet p=%.2f size %d vs %d", p, ns.size, size);
  }
  CHECK(throws<pa::DomainError>([&] { pa::nucleusSet(x, 1.5); }), "nucleusSet p > 1");
}

static void test_scalars() {
  const auto gi = pa::ApproxConfig::invPreset(7);
  const auto gs = pa::ApproxConfig::invsqrtPreset(7);
  for (double v : {0.3, 0.55, 0.9, 3.0, 17.0}) {
    auto low = [](const pa::ApproxConfig& a) {
      pam_approx_config c{};
      c.iterations = a.iterations;
      c.alpha_bits = a.alphaBits;
      c.rescale = (int32_t)a.rescale;
      c.scale_log2 = a.scaleLog2;
      c.lo = a.lo;
      c.hi = a.hi;
      return c;
    };
    const pam_approx_config c1 = low(gi), c2 = low(gs);
    double r1 = 0, r2 = 0;
    orc_inv_cfg(v, &c1, &r1);
    orc_invsqrt_cfg(v, &c2, &r2);
    CHECK(pa::goldschmidtInv(v, gi) == r1, "inv(%g) %.17g vs %.17g", v, pa::goldschmidtInv(v, gi), r1);
    CHECK(pa::goldschmidtInvSqrt(v, gs) == r2, "invsqrt(%g)", v);
  }
  CHECK(pa::nucleusAlpha(0.9, 0.9) == orc_nucleus_alpha(0.9, 0.9), "alpha");
  CHECK(pa::betaInverseCdf(0.3, 21.85) == orc_beta_icdf(0.3, 21.85), "beta icdf");
  CHECK(pa::gumbelFromUniform(0.25) == orc_gumbel(0.25), "gumbel");
}

static void test_batches() {
  const pa::CutMaxParams prm;
  const auto cp = prm.lower();
  const std::size_t B = 96, n = 32768;
  std::vector<double> X(B * n);
  for (std::size_t r = 0; r < B; ++r) {
    const auto x = gaussian(n, 100 + (unsigned)r);
    std::copy(x.begin(), x.end(), X.begin() + r * n);
  }
  std::vector<double> Z(B * n), Zr(B * n);
  std::vector<int32_t> am(B), amr(B), str(B);
  pa::cutmax_batch(X.data(), B, n, prm, Z.data(), am.data());
  orc_cutmax_batch(X.data(), (int64_t)n, (int64_t)B, (int64_t)n, &cp, Zr.data(), (int64_t)n, amr.data(), str.data(), 0);
  double worst = 0;
  for (std::size_t r = 0; r < B; ++r) worst = std::fmax(worst, normwise(&Z[r * n], &Zr[r * n], n));
  CHECK(am == amr, "host batch argmax");
  CHECK(worst <= 1e-12, "host batch normwise %.3e", worst);
  // device buffers, stream-ordered
  double *dX = nullptr, *dZ = nullptr;
  int32_t *dA = nullptr, *dS = nullptr;
  cudaMalloc(&dX, B * n * 8);
  cudaMalloc(&dZ, B * n * 8);
  cudaMalloc(&dA, B * 4);
  cudaMalloc(&dS, B * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaMemcpyAsync(dX, X.data(), B * n * 8, cudaMemcpyHostToDevice, s);
  pa::cutmax_batch_device(dX, B, n, n, prm, dZ, dA, dS, s);
  std::vector<double> Zd(B * n);
  std::vector<int32_t> ad(B), sd(B);
  cudaMemcpyAsync(Zd.data(), dZ, B * n * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(ad.data(), dA, B * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(sd.data(), dS, B * 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  CHECK(ad == amr && sd == str, "device batch argmax/status");
  CHECK(Zd == Z, "device and host batch bit-identical");
  // sampler batch on device
  pa::SamplerConfig cfg;
  cfg.seed = 5;
  int32_t* dT = nullptr;
  uint8_t* dI = nullptr;
  cudaMalloc(&dT, B * 4);
  cudaMalloc(&dI, B);
  pa::nucleus_sample_batch_device(dX, B, n, n, cfg, prm, dT, dI, dS, s);
  std::vector<int32_t> tok(B), tokr(B), sr(B);
  std::vector<uint8_t> ins(B), insr(B);
  cudaMemcpyAsync(tok.data(), dT, B * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(ins.data(), dI, B, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  pam_sampler_cfg sc{};
  sc.p = cfg.p;
  sc.q = cfg.q;
  sc.alpha = orc_nucleus_alpha(cfg.p, cfg.q);
  sc.seed = cfg.seed;
  orc_sample_batch(X.data(), (int64_t)n, (int64_t)B, (int64_t)n, &sc, &cp, 0, tokr.data(), insr.data(), sr.data(), 0);
  CHECK(tok == tokr && ins == insr, "device sampler batch tokens");
  cudaFree(dX);
  cudaFree(dZ);
  cudaFree(dA);
  cudaFree(dS);
  cudaFree(dT);
  cudaFree(dI);
  cudaStreamDestroy(s);
}

static void test_analysis() {
  const pa::CutMaxParams prm;
  const auto cp = prm.lower();
  const auto x = gaussian(1024, 9);
  const auto tr = pa::convergenceTrace(x, prm);
  std::vector<double> out(4 * (std::size_t)prm.T);
  orc_convergence_trace(x.data(), (int64_t)x.size(), &cp, out.data());
  CHECK(tr.size() == (std::size_t)prm.T, "trace length");
  for (int t = 0; t < prm.T; ++t) {
    CHECK(std::fabs(tr[t].s2 - out[4 * t + 1]) <= 1e-12 * out[4 * t + 1], "trace s2 t=%d", t);
    CHECK(tr[t].fractionBelowMean == out[4 * t + 3], "trace fraction t=%d", t);
  }
  // two-level input -> dispersion 0 at every iteration
  std::vector<double> two(64, 1.0);
  two[7] = 3.0;
  for (const auto& st : pa::convergenceTrace(two, prm)) CHECK(st.dispersion <= 1e-20, "two-level dispersion");
  // JVP against the oracle's forward mode
  const auto v = gaussian(1024, 10, 1.0);
  const auto dz = pa::cutmaxJvp(x, v, prm);
  std::vector<double> zr(1024), dzr(1024);
  orc_cutmax_jvp(x.data(), v.data(), 1024, &cp, zr.data(), dzr.data());
  CHECK(normwise(dz.data(), dzr.data(), 1024) <= 1e-10, "jvp");
}

static void test_errors() {
  const pa::CutMaxParams prm;
  CHECK(throws<pa::DegenerateInputError>([&] { pa::cutmax(std::vector<double>(100, 2.0), prm); }), "degenerate");
  pa::CutMaxParams bad;
  bad.T = 0;
  CHECK(throws<pa::InvalidParamsError>([&] { pa::cutmax(gaussian(64, 1), bad); }), "T = 0");
  pa::CutMaxParams even;
  even.p = {4};
  CHECK(throws<pa::InvalidParamsError>([&] { pa::cutmax(gaussian(64, 1), even); }), "even p checked");
  auto xn = gaussian(64, 2);
  xn[5] = NAN;
  bool nf = false;
  try {
    pa::cutmax(xn, prm);
  } catch (const pa::NonFiniteError& e) {
    nf = true;
  }
  CHECK(nf, "non-finite");
  std::vector<double> X(3 * 64);
  for (std::size_t i = 0; i < X.size(); ++i) X[i] = std::sin(0.37 * (double)i);
  X[2 * 64 + 9] = INFINITY;
  std::vector<double> Z(X.size());
  std::vector<int32_t> am(3);
  std::size_t where = 0;
  try {
    pa::cutmax_batch(X.data(), 3, 64, prm, Z.data(), am.data());
  } catch (const pa::NonFiniteError& e) {
    where = e.vector_index();
  }
  CHECK(where == 2, "batch non-finite row index %zu", where);
  CHECK(throws<pa::DomainError>([] { pa::betaInverseCdf(-0.5, 2.0); }), "beta u<0");
  CHECK(throws<pa::DomainError>([] { pa::gumbelFromUniform(0.0); }), "gumbel u=0 (SPEC.md:401)");
  CHECK(throws<pa::DomainError>([] { pa::nucleusAlpha(1.5, 0.9); }), "alpha p>1");
  pa::ApproxConfig none = pa::ApproxConfig::invsqrtPreset(7);
  none.rescale = pa::Rescale::None;
  CHECK(throws<pa::RangeError>([&] { pa::goldschmidtInvSqrt(40.0, none); }), "invsqrt outside range");
  CHECK(throws<pa::SingularityError>([&] { pa::cutmaxJvp(std::vector<double>(32, 1.0), std::vector<double>(32, 1.0), prm); }),
        "jvp singular");
  const std::string path = "/tmp/pam_cpp_api_bad.jsonl";
  {
    std::ofstream f(path);
    f << "[1.0, 2.0, 3.0]\n[1.0, oops]\n";
  }
  std::size_t off = 0;
  try {
    pa::ingest(path);
  } catch (const pa::FormatError& e) {
    off = e.byte_offset();
  }
  CHECK(off > 15, "format error offset %zu", off);
  // every type derives from Error (errors.hpp)
  CHECK(throws<pa::Error>([&] { pa::cutmax(std::vector<double>(10, 0.0), prm); }), "Error base");
}

static void test_ingest_roundtrip() {
  std::vector<pa::LogitVector> vs{{1.5, -2.25, 3.0}, {0.0, 4.5, -1.0}};
  const std::string path = "/tmp/pam_cpp_api.lgt1";
  pa::writeLgt1(path, vs);
  const auto back = pa::ingest(path);
  CHECK(back == vs, "LGT1 round trip");
}

int main() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    std::fprintf(stderr, "no CUDA device\n");
    return 2;
  }
  test_cutmax_vs_oracle();
  test_cutmax_step();
  test_samplers();
  test_scalars();
  test_batches();
  test_analysis();
  test_errors();
  test_ingest_roundtrip();
  std::printf("test_cpp_api: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
