"""CPU: pin the oracle before trusting it.

1. SPEC known answers (tests/golden/spec_known_answers.json, SPEC.md line refs inline).
2. Golden CutMax vectors from an independent math.fsum restatement (cutmax_golden.npz).
3. Published Philox4x32-10 known-answer vectors (philox_kat.json).
4. SPEC invariants / properties.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import normwise

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(GOLD, "spec_known_answers.json")) as f:
        return json.load(f)


def params(pam, **kw):
    return pam.CutMaxParams(**kw).lower()


# ---------------------------------------------------------------- KATs -----
def test_spec67_three_vector(orc, pam, kat):
    st, z, am, _ = orc.cutmax(kat["spec67_x"], params(pam, p=3, c=5.0, T=1))
    assert st == 0 and am == kat["spec67_argmax"]
    assert abs(z.sum() - 1.0) <= 1e-12


def test_spec67_T0_invalid(orc, pam):
    prm = params(pam, T=1)
    prm.T = 0
    st, *_ = orc.cutmax([5.0, 2.0, 1.0], prm)
    assert st == 1  # InvalidParams


def test_spec77_two_level_residuals(orc, kat):
    st, _, r, *_ = orc.cutmax_step([0.9, 0.05, 0.05], 3, 5.0)
    assert st == 0
    np.testing.assert_allclose(r, kat["spec77_residuals_n3"], rtol=1e-14)


def test_spec78_step(orc, kat):
    st, nx, r, mu, s2, _ = orc.cutmax_step([1.0, -1.0], 3, 5.0)
    assert st == 0
    np.testing.assert_allclose(r, kat["spec78_residuals"], rtol=1e-15)
    np.testing.assert_allclose(nx, kat["spec78_next"], rtol=1e-15)


def test_spec79_scale_invariance(orc):
    y = np.random.default_rng(0).normal(0, 1, 50)
    _, _, r1, *_ = orc.cutmax_step(y, 3, 5.0)
    _, _, r2, *_ = orc.cutmax_step(7.5 * y, 3, 5.0)
    np.testing.assert_allclose(r1, r2, rtol=1e-12, atol=1e-14)


def test_spec84_88_fixed_point(orc, pam, kat):
    st, vec, s = orc.fixed_point_target(3, 3, 5.0)
    assert st == 0 and abs(s - kat["spec88_sstar_n3_p3_c5"]) <= 1e-15
    st, _, s2 = orc.fixed_point_target(2, 3, 5.0)
    assert abs(s2 - kat["spec87_sstar_n2_p3_c5"]) <= 1e-15
    for sv in (0.4, 0.6, 0.9):  # SPEC.md:88 (s > 1/n; SURVEY App. A10 on s=0.2)
        st, z, _, _ = orc.cutmax([sv, (1 - sv) / 2, (1 - sv) / 2], params(pam, p=3, c=5.0, T=1))
        assert abs(z[0] - s) <= 1e-12
    assert orc.fixed_point_target(3, 3, 1.0)[0] == 1  # c <= sqrt(n-1) -> InvalidParams
    # c -> infinity: s* -> 1/n
    assert abs(orc.fixed_point_target(5, 3, 1e9)[2] - 0.2) < 1e-6


def test_spec66_onehot_is_two_level(orc, pam, kat):
    """SPEC.md:66 claims Z_7 > 0.99; the input is already two-level, so the
    correct answer is s*(8,3,5) = 0.3927 at every T."""
    x = np.zeros(8)
    x[7] = 1.0
    for T in (1, 2, 4):
        st, z, am, _ = orc.cutmax(x, params(pam, p=3, c=5.0, T=T))
        assert am == 7 and abs(z[7] - kat["spec66_two_level_n8_sstar"]) <= 1e-12


def test_spec97_kappa(orc, kat):
    st, k = orc.contraction_factor(2, 3, 10.0)
    assert st == 0 and abs(k - kat["spec97_kappa_n2_p3_c10"]) <= 1e-15 * k
    ks = [orc.contraction_factor(n, 3, 40.0)[1] for n in (2, 4, 16, 64, 256)]
    assert all(a > b for a, b in zip(ks, ks[1:]))  # SPEC.md:98 monotone in n


def test_spec163_175_polyapprox(orc, pam, kat):
    assert orc.scalar("goldschmidt_inv", 1.0, 5) == 1.0
    assert abs(orc.scalar("goldschmidt_inv", 0.5, 5) - kat["spec164_inv_0p5"]) <= kat["spec_inv_tol"]
    assert abs(orc.scalar("goldschmidt_inv", 1.5, 5) - kat["spec165_inv_1p5"]) <= kat["spec_inv_tol"]
    assert orc.scalar("invsqrt_newton", 1.0, 5) == 1.0
    for d in (3, 4, 5):
        assert abs(orc.scalar("invsqrt_newton", 0.25, d) - kat["spec174_invsqrt_0p25"]) <= 2 ** -7
    # Table 3 presets: iterations / depth (2 mults per Newton step)
    for ab, it in kat["table3_invsqrt_iters"].items():
        cfg = pam.ApproxConfig.invsqrtPreset(int(ab))
        assert cfg.iterations == it and 2 * cfg.iterations == {5: 10, 6: 12, 7: 14, 8: 16}[it]


def test_spec198_error_envelope(orc, pam):
    """alphaBits=7 presets: max error <= 2^-7 over 10^4 samples of the guaranteed domain."""
    rng = np.random.default_rng(7)
    inv_cfg = pam.ApproxConfig(iterations=5, lo=0.5, hi=1.5, rescale="none").lower()
    isq_cfg = pam.ApproxConfig(iterations=5, lo=2 ** -4, hi=1.0, rescale="none").lower()
    for x in rng.uniform(2 ** -4 + 1e-9, 1.0, 10000):
        st, v = orc.approx_cfg(x, isq_cfg, inv=False)
        assert st == 0 and abs(v - 1 / math.sqrt(x)) <= 2 ** -7
    for x in rng.uniform(0.5, 1.5, 10000):
        st, v = orc.approx_cfg(x, inv_cfg, inv=True)
        assert st == 0 and abs(v - 1 / x) <= 2 ** -7
    # out of domain -> RangeError
    assert orc.approx_cfg(3.0, inv_cfg, inv=True)[0] == 3
    assert orc.approx_cfg(-1.0, isq_cfg, inv=False)[0] == 3


def test_auto_rescale_is_exact_power_of_two(orc, pam):
    """AUTO rescaling by 4^k: invsqrt(4^k x) == invsqrt(x) / 2^k bit for bit (pin A4)."""
    cfg = pam.ApproxConfig(iterations=6).lower()
    for x in (0.3, 0.7, 0.26):
        for k in (-20, -3, 0, 5, 40):
            a = orc.approx_cfg(x * 4.0 ** k, cfg, inv=False)[1]
            b = orc.approx_cfg(x, cfg, inv=False)[1]
            assert a == b / 2.0 ** k


def test_spec403_gumbel(orc, kat):
    for u, g in (kat["spec403_gumbel_u_e-1"], kat["spec404_gumbel_u_e-e"]):
        assert abs(orc.scalar("gumbel", u) - g) <= 1e-15
    us = np.linspace(0.01, 0.99, 99)
    gs = [orc.scalar("gumbel", u) for u in us]
    assert all(a < b for a, b in zip(gs, gs[1:]))  # monotone


def test_spec421_beta_and_alpha(orc, kat):
    assert orc.scalar("beta_icdf", 1.0, 3.0) == 1.0
    assert orc.scalar("beta_icdf", 0.0, 3.0) == 0.0
    for u in (0.1, 0.5, 0.9):
        assert orc.scalar("beta_icdf", u, 1.0) == u  # alpha=1: identity
    a = orc.scalar("nucleus_alpha", 0.9, 0.9)
    assert abs(a - kat["spec434_alpha_p0.9"]) <= 1e-14 * a
    assert abs(1 - 0.9 ** a - 0.9) <= 1e-12  # self-consistency
    assert orc.scalar("nucleus_alpha", 0.5, 0.5) == 1.0
    assert math.isnan(orc.scalar("nucleus_alpha", 1.0, 0.5))  # DomainError boundary


def test_philox_published_kat(orc):
    with open(os.path.join(GOLD, "philox_kat.json")) as f:
        for e in json.load(f):
            assert orc.philox(e["ctr"], e["key"]) == e["out"]


def test_exp_log_accuracy(orc):
    rng = np.random.default_rng(3)
    for x in np.concatenate([rng.uniform(-700, 700, 3000), rng.uniform(-1, 1, 3000)]):
        assert abs(orc.scalar("exp", x) - math.exp(x)) <= 2.3e-16 * 2 * math.exp(x)
    for x in np.concatenate([10 ** rng.uniform(-300, 300, 3000), rng.uniform(0.5, 2, 3000)]):
        ref = math.log(x)
        assert abs(orc.scalar("log", x) - ref) <= 2.3e-16 * 2 * max(abs(ref), 1e-300) + 1e-300
    assert orc.scalar("exp", 0.0) == 1.0 and orc.scalar("log", 1.0) == 0.0


# -------------------------------------------------------- golden vectors ---
def test_cutmax_golden_vectors(orc, pam):
    g = np.load(os.path.join(GOLD, "cutmax_golden.npz"))
    for i in range(int(g["count"])):
        ps, cs = list(g[f"p{i}"]), list(g[f"c{i}"])
        prm = params(pam, p=ps, c=cs, T=len(ps))
        st, z, am, _ = orc.cutmax(g[f"x{i}"], prm)
        assert st == 0
        assert am == int(g["argmax"][i])
        assert normwise(z, g[f"z{i}"]) <= 1e-13, f"case {i}"


# -------------------------------------------------------------- properties --
def test_argmax_invariance_property(orc, pam):
    """argmax preserved for unique maximisers when c > sqrt(n-1);
    2000 random vectors, mixed distributions, near-ties with gap >= 1e-6."""
    rng = np.random.default_rng(11)
    for trial in range(2000):
        n = int(rng.integers(2, 600))
        kind = trial % 3
        if kind == 0:
            x = rng.normal(0, 1, n)
        elif kind == 1:
            x = rng.standard_t(2, n)
        else:
            x = rng.normal(0, 1, n)
            j = int(np.argmax(x))
            x[j] = np.max(np.delete(x, j)) + 1e-6 * (1 + rng.random())
        c = 1.5 * math.sqrt(n - 1) + 1.0
        prm = params(pam, p=3, c=c, T=3, guarantee=True)
        st, z, am, _ = orc.cutmax(x, prm)
        assert st == 0 and am == int(np.argmax(x))
        assert abs(z.sum() - 1) <= 1e-9
        assert np.all(z > 0)


def test_standardization_identities_and_bound(orc):
    """SPEC.md:114-115 / 609: sum r = 0, mean r^2 = 1, max|r| <= sqrt(n-1)."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        n = int(rng.integers(2, 300))
        y = rng.standard_t(3, n)
        st, _, r, *_ = orc.cutmax_step(y, 3, 5.0)
        assert abs(r.sum()) <= 1e-9 and abs((r * r).mean() - 1) <= 1e-9
        assert np.max(np.abs(r)) <= math.sqrt(n - 1) + 1e-9


def test_contraction_theorem(orc, pam):
    """Theorem 1, acceptance #2: n in {3,8,64},
    p in {3,5}, c = 2 sqrt(n-1), 1000 random inputs each.

    What Step 4 of the proof actually bounds is the raw
    dispersion of the NORMALISED next state's non-top entries,
    sum_{j != i*} (F(y)_j - mean)^2 <= kappa * U(y), with U(y) in residual space.
    The residual-space reading U(F(y)) <= kappa U(y) does not hold
    in general (counter-examples at n=3), so the proven form is tested and the
    defect is recorded in DESIGN.md."""
    rng = np.random.default_rng(13)
    for n in (3, 8, 64):
        for p in (3, 5):
            c = 2.0 * math.sqrt(n - 1)
            st, kappa = orc.contraction_factor(n, p, c)
            assert st == 0
            for _ in range(1000):
                y = rng.random(n) + 0.1
                y /= y.sum()
                _, nx, _, _, _, d0 = orc.cutmax_step(y, p, c)
                nx /= nx.sum()
                top = int(np.argmax(nx))
                nt = np.delete(nx, top)
                raw = float(((nt - nt.mean()) ** 2).sum())
                assert raw <= kappa * d0 * (1 + 1e-9) + 1e-300


def test_convergence_trace(orc, pam):
    """two-level input has U = 0; normal input fraction below mean > 0.5."""
    st, tr = orc.convergence_trace([0.9, 0.05, 0.05], params(pam, p=3, c=5.0, T=3))
    assert st == 0 and np.all(np.abs(tr[:, 2]) <= 1e-20)
    x = np.random.default_rng(14).normal(0, 1, 1024)
    st, tr = orc.convergence_trace(x, params(pam, p=3, c=40.0, T=3, guarantee=True))
    assert tr[1, 3] > 0.5
    assert np.all(np.diff(tr[:, 2]) <= 1e-12)


def test_errors(orc, pam):
    prm = params(pam)
    assert orc.cutmax(np.full(10, 3.0), prm)[0] == 2       # DegenerateInput
    x = np.arange(10.0)
    x[4] = np.nan
    assert orc.cutmax(x, prm)[0] == 5                        # NonFinite
    assert orc.cutmax([1.0], prm)[0] == 1                    # n >= 2
    bad = params(pam, p=4)
    assert orc.cutmax([1.0, 2.0], bad)[0] == 1               # even p rejected in checked mode
    assert orc.cutmax([1.0, 2.0], params(pam, p=4, checked=False))[0] == 0
    assert orc.cutmax(np.arange(100.0), params(pam, c=5.0, guarantee=True))[0] == 1


def test_tie_warning(orc):
    assert orc.tie_warning([1.0, 2.0, 2.0 - 1e-12]) == 0x100
    assert orc.tie_warning([1.0, 2.0, 1.5]) == 0


def test_beta_tail_identity(orc):
    """Lemma 2 / Observation 1: P(G > p) = q within 3 sigma,
    with the pinned Philox uniforms (2e5 draws per case here)."""
    N = 200000
    for p, q in ((0.9, 0.9), (0.9, 0.95), (0.5, 0.5)):
        a = orc.scalar("nucleus_alpha", p, q)
        hits = sum(orc.scalar("beta_icdf", orc.scalar("uniform", 99, 0, 0, i), a) > p for i in range(N))
        sd = math.sqrt(q * (1 - q) / N)
        assert abs(hits / N - q) <= 3 * sd


def test_gumbel_fidelity(orc, pam):
    """Lemma 1: Gumbel-max through CutMax samples softmax;
    n=10, 20000 draws, TV <= 0.03 (scaled from 1e5 draws / 0.02)."""
    rng = np.random.default_rng(15)
    x = np.log(rng.dirichlet(np.ones(10)))
    prm = params(pam, p=3, c=5.0, T=4)
    X = np.repeat(x[None, :], 20000, axis=0)
    cfg = pam.SamplerConfig(p=0.9, seed=2024).lower()
    tok, _, st = orc.sample_batch(X, cfg, prm, gumbel=True)
    assert np.all(st == 0)
    freq = np.bincount(tok, minlength=10) / len(tok)
    soft = np.exp(x - x.max())
    soft /= soft.sum()
    assert 0.5 * np.abs(freq - soft).sum() <= 0.03


def test_nucleus_membership_rule(orc):
    """smallest prefix with mass >= p, ties included."""
    x = np.log(np.array([0.5, 0.3, 0.15, 0.05]))
    assert orc.nucleus_inside(x, 0.9, 0) and orc.nucleus_inside(x, 0.9, 2)
    assert not orc.nucleus_inside(x, 0.9, 3)
    assert orc.nucleus_inside(x, 0.75, 1) and not orc.nucleus_inside(x, 0.75, 2)
    xt = np.log(np.array([0.4, 0.3, 0.3]))  # tie at the boundary: both tied tokens inside
    assert orc.nucleus_inside(xt, 0.6, 1) and orc.nucleus_inside(xt, 0.6, 2)
    u = np.zeros(10)  # uniform logits, p=0.9 -> nucleus = 9 tokens -> ties: all 10
    assert all(orc.nucleus_inside(u, 0.9, i) for i in range(10))


def test_beta_cut_zero_violations_peaked(orc, pam):
    """Fig. 4 / acceptance #10, desk scale: peaked logits,
    20 prompts x 100 draws: beta-cut violation rate 0, Gumbel-max > 0."""
    rng = np.random.default_rng(16)
    prm = params(pam, p=3, c=5.0, T=4)
    beta_v = gum_v = 0
    for prompt in range(20):
        n = 2048
        x = rng.permutation(-1.1 * np.log(np.arange(1, n + 1)) + rng.normal(0, 0.3, n))
        X = np.repeat(x[None, :], 100, axis=0)
        cfg = pam.SamplerConfig(p=0.9, seed=1000 + prompt).lower()
        _, ins, st = orc.sample_batch(X, cfg, prm)
        assert np.all(st == 0)
        beta_v += int((ins == 0).sum())
        _, ins_g, _ = orc.sample_batch(X, cfg, prm, gumbel=True)
        gum_v += int((ins_g == 0).sum())
    assert beta_v == 0 and gum_v > 0


def test_cutmax_jvp_oracle(orc, pam):
    """cutmaxJvp (§8f rank 4): v = 0 -> 0, v = 1 -> 0 (shift
    invariance), linear in v, and central finite differences (h = 1e-5) within
    1e-4 relative on random (x, v), n <= 64."""
    rng = np.random.default_rng(21)
    prm = params(pam, p=3, c=5.0, T=4)
    for trial in range(40):
        n = int(rng.integers(2, 65))
        x = rng.normal(0, 2, n)
        st, z, dz = orc.cutmax_jvp(x, np.zeros(n), prm)
        assert st == 0 and np.all(dz == 0.0)
        st, _, dz1 = orc.cutmax_jvp(x, np.ones(n), prm)
        assert st == 0 and np.max(np.abs(dz1)) < 1e-11
        v1, v2 = rng.normal(size=n), rng.normal(size=n)
        _, _, a = orc.cutmax_jvp(x, v1, prm)
        _, _, b = orc.cutmax_jvp(x, v2, prm)
        _, _, ab = orc.cutmax_jvp(x, 2.0 * v1 - 3.0 * v2, prm)
        assert np.max(np.abs(ab - (2.0 * a - 3.0 * b))) <= 1e-10 * max(1.0, np.max(np.abs(ab)))
        h = 1e-5
        zp, _, _ = orc.cutmax_batch((x + h * v1)[None, :], prm)
        zm, _, _ = orc.cutmax_batch((x - h * v1)[None, :], prm)
        fd = (zp[0] - zm[0]) / (2 * h)
        # relative 1e-4 above the finite-difference noise floor ~eps/h
        assert np.max(np.abs(fd - a)) <= 1e-4 * np.max(np.abs(a)) + 1e-9
    st, _, _ = orc.cutmax_jvp(np.full(8, 2.5), np.ones(8), prm)
    assert st == pam._abi.PAM_ERR_SINGULAR


def test_table_log_exp_accuracy(orc):
    """The sampler's table-driven log / exp (oracle orc_log_t / orc_exp_t, the
    kernel's pam_scalar.h log_t / exp_t): <= 2 ulp against libm on the
    sampler's domains (uniforms in (0,1), the Gumbel inner values, Beta
    exponents in [-700, 0], nucleus exponents x - max <= 0) and beyond."""
    import numpy as np

    rng = np.random.default_rng(7)
    us = np.concatenate([rng.random(20000), 1.0 - rng.random(2000) * 1e-12, rng.random(2000) * 1e-300,
                         np.exp(rng.uniform(-36.7, 0.0, 4000)), rng.uniform(1.0, 1e6, 2000)])
    for u in us:
        if u <= 0.0:
            continue
        ref = math.log(u)
        got = orc.scalar("log_t", float(u))
        assert abs(got - ref) <= 2 * math.ulp(ref) + 1e-300, (u, got, ref)
    xs = np.concatenate([rng.uniform(-700.0, 0.0, 20000), rng.uniform(-1e-3, 1e-3, 2000),
                         rng.uniform(0.0, 709.0, 2000)])
    for x in xs:
        ref = math.exp(x)
        got = orc.scalar("exp_t", float(x))
        assert abs(got - ref) <= 2 * math.ulp(ref), (x, got, ref)
    assert orc.scalar("exp_t", 0.0) == 1.0 and orc.scalar("log_t", 1.0) == 0.0
    assert orc.scalar("exp_t", -800.0) == 0.0 and math.isinf(orc.scalar("exp_t", 800.0))
