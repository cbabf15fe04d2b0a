"""GPU tests of the SPEC decisions the boundary must honour beyond plain parity:
TieWarning, early stopping, the sampler's token
rule (argmax of Y^(T+1) before the normalisation, pin A7), and the C5 sweep at
its full batch size with every row checked against the oracle.

Every case compares the CUDA path (through the C ABI) with the CPU oracle on
the same seeded inputs; tolerances as tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

from conftest import normwise
from paper_2509_08383_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5
TIE = 0x100


def run_gpu(cuda, pam, x, prm):
    torch = cuda
    xt = torch.as_tensor(np.ascontiguousarray(x), device="cuda")
    z, am, st = pam.cutmax_batch_device(xt, prm)
    torch.cuda.synchronize()
    return z.cpu().numpy(), am.cpu().numpy(), st.cpu().numpy()


def check(z, am, st, zr, amr, str_, tol):
    assert np.array_equal(st, str_), f"status mismatch rows {np.nonzero(st != str_)[0][:8]}: {st[st != str_][:8]} vs {str_[st != str_][:8]}"
    ok = (st & 0xFF) == 0
    assert np.array_equal(am[ok], amr[ok]), f"argmax mismatch rows {np.nonzero(am != amr)[0][:8]}"
    worst = max((normwise(z[r], zr[r]) for r in np.nonzero(ok)[0]), default=0.0)
    print(f"worst normwise {worst:.3e} (tol {tol:.1e})")
    assert worst <= tol, f"normwise {worst:.3e} > {tol:.0e}"


# ----------------------------------------------------------- TieWarning ----
def tie_rows(B, n, seed, dtype=np.float64):
    """Rows with a planted top-2 gap: exact duplicates of the maximum, gaps just
    below and above 1e-9, and ordinary rows; both index orders of the pair."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 3.0, size=(B, n)).astype(dtype)
    gaps = [0.0, 0.0, 5e-10, 9.9e-10, 1.01e-9, 4e-9, None]
    for r in range(B):
        g = gaps[r % len(gaps)]
        if g is None:
            continue
        i, j = rng.choice(n, size=2, replace=False)
        top = dtype(x[r].max() + 1.0)
        x[r, i] = top
        x[r, j] = dtype(np.float64(top) - g)
    return x


@pytest.mark.parametrize("n,geom", [(1024, None), (32768, None), (151936, None), (9000, (256, 38, 1)),
                                    (9000, (128, 8, 9))])
def test_tie_warning_f64(cuda, pam, orc, n, geom):
    """PAM_ROW_FLAG_TIE on exactly the rows the oracle flags (status compared
    bit for bit), with the lowest index winning exact ties; single-CTA and
    cluster geometries and the pipelined rows of a many-rows-per-cluster launch."""
    B = 70 if n <= 32768 else 21
    x = tie_rows(B, n, seed=n)
    prm = pam.CutMaxParams()
    if geom is None:
        z, am, st = run_gpu(cuda, pam, x, prm)
    else:
        with pam.geometry_override(8, *geom):
            z, am, st = run_gpu(cuda, pam, x, prm)
    zr, amr, str_ = orc.cutmax_batch(x, prm.lower())
    assert np.count_nonzero(str_ & TIE) >= B // 3
    check(z, am, st, zr, amr, str_, TOL64)
    for r in range(B):  # flag == oracle's restated rule on the input itself
        assert bool(st[r] & TIE) == bool(orc.tie_warning(x[r]))


def test_tie_warning_undecided_overflow(cuda, pam, orc):
    """The fp64 screen works on 32-bit order keys (sign, exponent, 20 mantissa
    bits); rows whose top-2 keys straddle the 1e-9 threshold are settled by an
    exact re-scan at the end of the kernel from a 16-entry queue per cluster, or
    by re-scanning every row of the cluster when the queue overflows.  Every
    row here is undecided (duplicated maxima, sub-ulp-of-key gaps on both sides
    of 1e-9), ~20 per cluster at n = 151936."""
    torch = cuda
    B, n = 300, 151936
    rng = np.random.default_rng(77)
    x = rng.normal(0.0, 3.0, size=(B, n))
    gaps = [0.0, 5e-10, 9.99e-10, 1.001e-9, 3e-9, 0.0]
    for r in range(B):
        i, j = rng.choice(n, size=2, replace=False)
        top = x[r].max() + 1.0
        x[r, i] = top
        x[r, j] = top - gaps[r % len(gaps)]
    xt = torch.as_tensor(x, device="cuda")
    with pam.geometry_override(8, 512, 34, 9):  # 15 clusters: 20 rows each
        z, am, st = pam.cutmax_batch_device(xt, pam.CutMaxParams())
        info = pam.launch_info(8, B, n, pam.CutMaxParams())
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert np.all((st & 0xFF) == 0)
    want = np.array([orc.tie_warning(x[r]) for r in range(B)])
    assert np.array_equal((st & TIE) != 0, want != 0)
    assert np.array_equal(am.cpu().numpy(), x.argmax(axis=1))
    assert B / info["clusters"] > 16


def test_tie_warning_f32_and_generic_p(cuda, pam, orc):
    x = tie_rows(56, 32768, seed=5, dtype=np.float32)
    prm = pam.CutMaxParams()
    z, am, st = run_gpu(cuda, pam, x, prm)
    zr, amr, str_ = orc.cutmax_batch(x, prm.lower())
    check(z, am, st, zr, amr, str_, TOL32)
    x64 = tie_rows(42, 20000, seed=6)
    prm5 = pam.CutMaxParams(p=5, c=12.0, T=3)  # generic-p flow
    z, am, st = run_gpu(cuda, pam, x64, prm5)
    zr, amr, str_ = orc.cutmax_batch(x64, prm5.lower())
    check(z, am, st, zr, amr, str_, TOL64 * 125 / 81)
    assert np.count_nonzero(st & TIE) >= 12


def test_tie_warning_front_end(cuda, pam):
    """cutmax() reports the TieWarning (warnings module) and on the ScoreVector."""
    x = np.linspace(-1.0, 1.0, 4096)
    x[100] = x[-1]
    with pytest.warns(pam.TieWarning):
        sv = pam.cutmax(x)
    assert sv.tieWarning and sv.argmax == 100


# ------------------------------------------------------------ early stop ----
# The top mass only approaches 1 for the paper's larger powers (Table 1,
# (T, p, c) = (4, 13, 15), (5, 9, 15)); with p = 3 CutMax
# settles on its two-level fixed point (top mass s* < 1) and never stops.
def tol_for(ps, dtype, n):
    """1e-12 (fp64) / 1e-5 (fp32) scaled by prod(p)/81 as in test_gpu_parity,
    and never below the oracle's own summation error on rows where one term
    dominates sum Y: its sequential loop drops every term below half an ulp of
    the running total, up to n * 2^-53 relative (the kernel's tree sums keep them)."""
    base = 1e-12 if dtype == np.float64 else 1e-5
    return max(base * max(1.0, float(np.prod(ps)) / 81.0), 2.0 * n * 2.0 ** -53)


@pytest.mark.parametrize("eps", [1e-2, 1e-6])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_eps_stop_matches_oracle(cuda, pam, orc, eps, dtype):
    """SPEC.md:126 early stopping: the row stops after the iteration whose top
    mass max Y / sum Y reaches 1 - eps; Z, argmax and status match the oracle,
    and the rows really stop early (their Z differs from the full-T result)."""
    x = W.zipf_logits(40, 8192, seed=21).astype(dtype)
    prm = pam.CutMaxParams(p=13, c=15.0, T=6, epsStop=eps)
    z, am, st = run_gpu(cuda, pam, x, prm)
    zr, amr, str_ = orc.cutmax_batch(x, prm.lower())
    check(z, am, st, zr, amr, str_, tol_for([13] * 2, dtype, 8192))
    zfull, _, _ = orc.cutmax_batch(x, pam.CutMaxParams(p=13, c=15.0, T=6).lower())
    stopped = [r for r in range(len(x)) if not np.array_equal(zr[r], zfull[r])]
    assert len(stopped) >= 20


def test_eps_stop_cluster_and_sampler(cuda, pam, orc):
    """Early stop on a cluster geometry (n = 151936: the decision is taken by
    every CTA from identical exchanged sums) and inside the Beta-cut sampler."""
    torch = cuda
    x = W.zipf_logits(8, 151936, seed=9)
    prm = pam.CutMaxParams(p=9, c=15.0, T=6, epsStop=1e-6)
    z, am, st = run_gpu(cuda, pam, x, prm)
    zr, amr, str_ = orc.cutmax_batch(x, prm.lower())
    check(z, am, st, zr, amr, str_, tol_for([9] * 2, np.float64, 151936))
    xs = W.zipf_logits(32, 32768, seed=10)
    cfg = pam.SamplerConfig(p=0.9, seed=77)
    prm_s = pam.CutMaxParams(p=13, c=15.0, T=6, epsStop=1e-3)
    tok, ins, sts = pam.nucleus_sample_batch_device(torch.as_tensor(xs, device="cuda"), cfg, prm_s)
    tr, ir, sr = orc.sample_batch(xs, cfg.lower(), prm_s.lower())
    assert np.array_equal(sts.cpu().numpy(), sr)
    assert np.array_equal(tok.cpu().numpy(), tr) and np.array_equal(ins.cpu().numpy(), ir)


# ------------------------------------------------------ sampler token rule ---
def near_tie_rows(orc, x, seed, alpha, gaps):
    """Plant in every row a pair (i, j) whose perturbed logits x~ = x + G sit
    `gap` apart at the top (gap < 0 puts j above i; gap == 'ulp' one ulp apart),
    computing G exactly as the sampler does (Philox uniform -> Beta inverse CDF)."""
    rng = np.random.default_rng(seed + 1)
    B, n = x.shape
    pairs = []
    for r in range(B):
        i, j = (int(v) for v in rng.choice(n, size=2, replace=False))
        gi = orc.scalar("beta_icdf", orc.scalar("uniform", seed, r, 0, i), alpha)
        gj = orc.scalar("beta_icdf", orc.scalar("uniform", seed, r, 0, j), alpha)
        xi = 40.0 + rng.random()
        x[r, i] = xi
        ti = xi + gi
        g = gaps[r % len(gaps)]
        target = np.nextafter(ti, np.inf if r % 2 else -np.inf) if g == "ulp" else ti - g
        xj = target - gj
        for _ in range(16):  # land x_j + g_j exactly on target
            s_ = xj + gj
            if s_ == target:
                break
            xj = np.nextafter(xj, np.inf if s_ < target else -np.inf)
        x[r, j] = xj
        pairs.append((i, j, xi + gi, xj + gj))
    return pairs


def test_sampler_token_on_y_near_ties(cuda, pam, orc):
    """Near-ties at the top of x~ = x + G, below the 1e-9 TieWarning threshold
    and in both index orders.  The token is the argmax of Y^(T+1) before the
    normalisation (pin A7, as oracle.c orc_cutmax; a token taken on Z = Y *
    inv(sum Y) could merge the pair by rounding): token, flag and TieWarning
    must match the oracle exactly and pick the true maximiser of x~.

    Gaps of 2e-11 and 3e-12 are far above the pipeline's rounding noise
    (~1e-14 relative after p^T = 81 amplification), so the order is determined.
    At a ONE-ulp gap two correct fp64 evaluation orders (oracle: textbook
    loops; kernel: shifted moments, fma) may order the pair differently; such a
    row is a tie by SPEC.md:122 (flagged) and ties "can be broken arbitrarily"
    (PAPER.md:464), so there the test asserts the flag and that the token is
    one of the pair."""
    torch = cuda
    n, B, seed = 32768, 64, 4242
    cfg = pam.SamplerConfig(p=0.9, seed=seed)
    alpha = pam.nucleusAlpha(0.9)
    prm = pam.CutMaxParams()
    x = W.zipf_logits(B, n, seed=11)
    pairs = near_tie_rows(orc, x, seed, alpha, [2e-11, -2e-11, 3e-12, -3e-12])
    tok, ins, st = pam.nucleus_sample_batch_device(torch.as_tensor(x, device="cuda"), cfg, prm)
    tr, ir, sr = orc.sample_batch(x, cfg.lower(), prm.lower())
    assert np.array_equal(st.cpu().numpy(), sr)
    assert np.all(sr & TIE)
    assert np.array_equal(tok.cpu().numpy(), tr) and np.array_equal(ins.cpu().numpy(), ir)
    truth = np.array([i if ti > tj else j for i, j, ti, tj in pairs])
    assert np.array_equal(tr, truth)
    # one-ulp pairs: flagged ties, token within the pair on both sides
    x1 = W.zipf_logits(16, n, seed=12)
    pairs1 = near_tie_rows(orc, x1, seed, alpha, ["ulp"])
    tok1, _, st1 = pam.nucleus_sample_batch_device(torch.as_tensor(x1, device="cuda"), cfg, prm)
    tr1, _, sr1 = orc.sample_batch(x1, cfg.lower(), prm.lower())
    assert np.array_equal(st1.cpu().numpy(), sr1) and np.all(sr1 & TIE)
    for r, (i, j, _, _) in enumerate(pairs1):
        assert int(tok1[r]) in (i, j) and int(tr1[r]) in (i, j)


# -------------------------------------------------- C5 at full batch size ---
@pytest.mark.parametrize("n", [1024, 32768, 151936])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_c5_full_batch_every_row(cuda, pam, orc, n, dtype):
    """C5 at B = 4096 (the bench geometry at n = 151936: 512x34 C=9 with ~273
    rows per cluster; the exact-fit 512x32 C=2 at 32768; 740 C=1 clusters at
    1024): every row against the oracle, in 512-row chunks to bound host RAM."""
    torch = cuda
    B = 4096
    xg = W.torch_gaussian(B, n, seed=5000 + n, device="cuda")
    xt = xg if dtype == np.float64 else xg.float()
    prm = pam.CutMaxParams()
    z, am, st = pam.cutmax_batch_device(xt, prm)
    torch.cuda.synchronize()
    tol = TOL64 if dtype == np.float64 else TOL32
    for r0 in range(0, B, 512):
        xh = xt[r0:r0 + 512].cpu().numpy()
        zr, amr, str_ = orc.cutmax_batch(xh, prm.lower())
        check(z[r0:r0 + 512].cpu().numpy(), am[r0:r0 + 512].cpu().numpy(), st[r0:r0 + 512].cpu().numpy(),
              zr, amr, str_, tol)
        assert np.array_equal(amr, np.argmax(xh, axis=1))


# ---------------------------------------------------- SPEC acceptance #1 ----
@pytest.mark.parametrize("n", [50257, 151936])
def test_acceptance_argmax_recovery_table1(cuda, pam, orc, n):
    """SPEC.md:606 (acceptance #1; Table 1): on 100 peaked
    LLM-like fixtures (workloads.peaked_logits: log Zipf(1.1) + N(0, 0.5^2),
    permuted, top-1 margin >= 0.05 nats; the paper's QWEN logits are
    unavailable) cutmax with (T, p, c) = (4, 13, 15) and (5, 9, 15)
    recovers the argmax in 100/100 rows, with mean top mass >= 0.999 (T = 4) and
    >= 1 - 1e-6 (T = 5), in < 10 s.  On the raw Zipf rows (near-ties allowed)
    the argmax is still recovered 100/100; their top mass is lower on the
    near-tie rows and equals the oracle's.  8 rows per setting are checked
    against the oracle (tolerance 1e-12 * p^T / 81)."""
    import time

    torch = cuda
    for peaked in (True, False):
        x = W.peaked_logits(100, n, seed=606) if peaked else W.zipf_logits(100, n, seed=606)
        xt = torch.as_tensor(x, device="cuda")
        for T, p, c, mass in ((4, 13, 15.0, 0.999), (5, 9, 15.0, 1.0 - 1e-6)):
            prm = pam.CutMaxParams(T=T, p=p, c=c)
            t0 = time.perf_counter()
            z, am, st = pam.cutmax_batch_device(xt, prm)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert dt < 10.0
            st = st.cpu().numpy()
            assert np.all((st & 0xFF) == 0)
            assert np.array_equal(am.cpu().numpy(), x.argmax(axis=1)), "argmax recovery < 100/100"
            top = z.max(dim=1).values.cpu().numpy()
            print(f"n={n} peaked={peaked} (T,p,c)=({T},{p},{c}): mean top mass {top.mean():.9f}, "
                  f"min {top.min():.9f}, {dt * 1e3:.1f} ms")
            if peaked:
                assert top.mean() >= mass
            zr, amr, sr = orc.cutmax_batch(x[:8], prm.lower())
            check(z[:8].cpu().numpy(), am[:8].cpu().numpy(), st[:8], zr, amr, sr, TOL64 * p ** T / 81)
