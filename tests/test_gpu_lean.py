"""The lean p = 3 kernel (csrc/cutmax_p3_kernel.cuh) against the general CutMax
kernel (csrc/cutmax_kernel.cuh, p = 3 flow): same algebra, exchanges and
rounding, so Z, argmax, status (TieWarning included) and the per-iteration
stats must be bit-identical.  The oracle parity of the product path (which is
the lean kernel for these parameters) is covered by test_gpu_parity.py and
test_gpu_features.py; this file pins the A/B equivalence on the edge cases.
"""
import numpy as np
import pytest

from paper_2509_08383_b200 import workloads as W

pytestmark = pytest.mark.gpu


def both(torch, pam, x, prm, stats=False, tol=1e-14):
    """Run both kernels.  They share the algebra and the exchanges; the lean
    kernel accumulates a row's input sums in one (sum, sum of squares) pair
    where the general kernel interleaves two, so results agree to the last
    few bits (1e-14 normwise here, against the 1e-12 oracle bar) with argmax,
    status and TieWarning identical.  The lean kernel itself must not depend on
    whether a row is its cluster's first row: checked in
    test_lean_row_position_independent."""
    outs = []
    for general in (False, True):
        B, n = x.shape
        z = torch.empty_like(x)
        am = torch.empty(B, dtype=torch.int32, device=x.device)
        st = torch.empty(B, dtype=torch.int32, device=x.device)
        sv = torch.empty((B, prm.T, 2), dtype=torch.float64, device=x.device) if stats else None
        if general:
            with pam.general_p3_kernel():
                pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st, stats=sv)
                kid = pam.launch_info(x.element_size(), B, n, prm)["kernel_id"]
            assert kid < 1000
        else:
            pam.cutmax_batch_device(x, prm, z=z, argmax=am, status=st, stats=sv)
            kid = pam.launch_info(x.element_size(), B, n, prm)["kernel_id"]
            assert 1000 <= kid < 2000, "lean kernel not selected"
        torch.cuda.synchronize()
        outs.append((z, am, st, sv))
    (z0, a0, s0, v0), (z1, a1, s1, v1) = outs
    assert torch.equal(s0, s1), f"status differs: {(s0 != s1).nonzero()[:5].flatten().tolist()}"
    assert torch.equal(a0, a1), f"argmax differs: {(a0 != a1).nonzero()[:5].flatten().tolist()}"
    ok = (s0 & 0xFF) == 0
    if bool(ok.any()):
        err = ((z0[ok].double() - z1[ok].double()).abs().amax(1) / z1[ok].double().abs().amax(1)).max().item()
        assert err <= tol, err
    if stats and bool(ok.any()):  # mu to 1e-12 sigma (means sit near 0), s2 to 1e-12 relative
        a, b = v0[ok], v1[ok]
        sig = b[..., 1].clamp_min(0).sqrt()
        assert bool(((a[..., 0] - b[..., 0]).abs() <= 1e-12 * sig).all())
        assert bool(((a[..., 1] - b[..., 1]).abs() <= 1e-12 * b[..., 1].abs()).all())
    return z0, a0, s0


@pytest.mark.parametrize("B,n,T", [(64, 151936, 4), (40, 151936, 2), (33, 151936, 3), (256, 32768, 4),
                                   (200, 32768, 3), (37, 9000, 4), (5, 50000, 5)])
def test_lean_equals_general_gaussian(cuda, pam, B, n, T):
    torch = cuda
    x = W.torch_gaussian(B, n, seed=B + n + T)
    _, am, st = both(torch, pam, x, pam.CutMaxParams(p=3, c=5.0, T=T), stats=True)
    assert int(((st & 0xFF) != 0).sum()) == 0
    assert torch.equal(am.long(), x.argmax(dim=1))


def test_lean_equals_general_edge_rows(cuda, pam):
    """Planted ties / near-ties (TieWarning screen and its exact fallback),
    shifted rows that trip the one-pass cancellation guard, degenerate and
    non-finite rows, a Zipf row and polynomial-mode scalars."""
    torch = cuda
    B, n = 48, 151936
    rng = np.random.default_rng(5)
    x = rng.normal(0.0, 3.0, size=(B, n))
    for r in range(0, 12):  # duplicated max / gaps around 1e-9
        i, j = rng.choice(n, size=2, replace=False)
        top = x[r].max() + 1.0
        x[r, i] = top
        x[r, j] = top - [0.0, 5e-10, 9.99e-10, 1.001e-9, 2e-9, 1e-3][r % 6]
    x[12:18] += 1e6  # |mean| / sigma ~ 3e5: one-pass moments cancel -> exact second pass
    x[18] = 7.0  # degenerate
    x[19, 5] = np.nan
    x[20, 77] = np.inf
    x[21] = W.zipf_logits(1, n, seed=3)[0]
    x[22] = np.linspace(-1.0, 1.0, n)  # two-level-ish tails, exact duplicates nowhere
    xt = torch.as_tensor(x, device="cuda")
    both(torch, pam, xt, pam.CutMaxParams(), stats=True)
    both(torch, pam, xt, pam.CutMaxParams(T=3, c=7.0), stats=True)
    both(torch, pam, xt, pam.CutMaxParams(normalize=False), stats=True)


def test_lean_poly_mode(cuda, pam):
    torch = cuda
    x = W.torch_gaussian(64, 32768, seed=9)
    both(torch, pam, x, pam.CutMaxParams(invsqrtMode="poly", invMode="poly"), stats=True)


def test_lean_row_position_independent(cuda, pam):
    """A row gives bit-identical results whether it is the first row of its
    cluster (input sums from the prologue) or a pipelined one (input sums from
    the previous row's swap): run the same rows as the whole batch and as
    single-row launches."""
    torch = cuda
    B, n = 300, 151936
    x = W.torch_gaussian(B, n, seed=21)
    prm = pam.CutMaxParams()
    with pam.geometry_override(8, 512, 34, 9):  # same slicing for both launches
        z, am, st = pam.cutmax_batch_device(x, prm)
        assert pam.launch_info(8, B, n, prm)["kernel_id"] >= 1000
        for r in (0, 17, 150, 299):
            z1, a1, s1 = pam.cutmax_batch_device(x[r:r + 1].contiguous(), prm)
            torch.cuda.synchronize()
            assert torch.equal(z1[0], z[r]) and int(a1[0]) == int(am[r]) and int(s1[0]) == int(st[r])


@pytest.mark.parametrize("B,n", [(64, 151936), (300, 32768), (40, 9000)])
def test_lean_fp32_equals_general(cuda, pam, orc, B, n):
    """fp32 rows (fp32 storage and elementwise math, fp64 statistics) on the lean
    kernel vs the general one (2e-5 normwise: fp32 rounding of the two
    accumulation orders: each is within the fp32 bar 1e-5 of the oracle, so
    they agree to 2e-5), and 6 rows against the oracle at 1e-5."""
    torch = cuda
    x = W.torch_gaussian(B, n, seed=B + n, dtype=torch.float32)
    z, am, st = both(torch, pam, x, pam.CutMaxParams(), tol=2e-5)
    xs = x[:6].cpu().numpy()
    zr, amr, sr = orc.cutmax_batch(xs, pam.CutMaxParams().lower())
    zz = z[:6].cpu().numpy()
    assert np.array_equal(am[:6].cpu().numpy(), amr) and np.array_equal(st[:6].cpu().numpy(), sr)
    assert max(float(np.max(np.abs(zz[r] - zr[r])) / np.max(np.abs(zr[r]))) for r in range(6)) <= 1e-5


@pytest.mark.parametrize("n", [151936, 32768])
@pytest.mark.parametrize("T,p,c", [(2, 19, 5.0), (3, 19, 27.0), (4, 13, 15.0), (5, 9, 15.0), (3, 5, 12.0)])
def test_lean_table1_powers_vs_oracle(cuda, pam, orc, n, T, p, c):
    """The lean kernel at the paper's Table-1 settings and
    p = 5: explicit sum of Y^(T+1) instead of the p = 3 closed form.  Against the
    oracle: argmax and status exact, Z within 1e-12 * p^T / 81 normwise (the
    rounding amplification of test_gpu_parity.py)."""
    torch = cuda
    B = 24
    x = W.zipf_logits(B, n, seed=T * 100 + p)
    prm = pam.CutMaxParams(T=T, p=p, c=c)
    xt = torch.as_tensor(x, device="cuda")
    z, am, st = pam.cutmax_batch_device(xt, prm)
    torch.cuda.synchronize()
    assert 1000 <= pam.launch_info(8, B, n, prm)["kernel_id"] < 2000, "lean kernel not selected"
    zr, amr, sr = orc.cutmax_batch(x, prm.lower())
    st = st.cpu().numpy()
    assert np.array_equal(st, sr)
    ok = (st & 0xFF) == 0
    assert np.array_equal(am.cpu().numpy()[ok], amr[ok])
    zz = z.cpu().numpy()
    tol = 1e-12 * max(1.0, p ** T / 81)
    worst = max(float(np.max(np.abs(zz[r] - zr[r])) / np.max(np.abs(zr[r]))) for r in np.nonzero(ok)[0])
    assert worst <= tol, worst


@pytest.mark.parametrize("n", [151936, 32768])
@pytest.mark.parametrize("sched", [
    dict(p=[16, 4, 4, 6], c=[5.0, 3.0, 3.0, 3.0], T=4, checked=False),  # the HE schedule
    dict(p=[3, 5, 3], c=[5.0, 8.0, 5.0], T=3),                          # mixed odd powers (ipow loop)
    dict(p=4, c=6.0, T=3, checked=False),                                 # one even power everywhere
    dict(p=7, c=10.0, T=3),                                               # an odd power with no fixed-P kernel
    dict(p=[8, 2], c=[6.0, 4.0], T=2, checked=False),
])
def test_lean_mixed_schedule_vs_oracle(cuda, pam, orc, n, sched):
    """The mixed-schedule lean kernel (P = 0: per-iteration powers, unrolled
    square-and-multiply for the even powers of the HE schedule, ipow's loop for
    the rest) against the oracle and against the general kernel."""
    torch = cuda
    B = 100
    x = W.gaussian(B, n, seed=n % 97 + len(str(sched)))
    prm = pam.CutMaxParams(**sched)
    xt = torch.as_tensor(x, device="cuda")
    z, am, st = pam.cutmax_batch_device(xt, prm)
    torch.cuda.synchronize()
    assert 1000 <= pam.launch_info(8, B, n, prm)["kernel_id"] < 2000, "lean kernel not selected"
    with pam.general_p3_kernel():
        zg, amg, stg = pam.cutmax_batch_device(xt, prm)
        assert pam.launch_info(8, B, n, prm)["kernel_id"] < 1000
    torch.cuda.synchronize()
    zr, amr, sr = orc.cutmax_batch(x[:24], prm.lower())
    st_, am_ = st.cpu().numpy(), am.cpu().numpy()
    assert np.array_equal(st_[:24], sr) and np.array_equal(st_, stg.cpu().numpy())
    ok = (st_ & 0xFF) == 0
    assert bool(ok.any())
    assert np.array_equal(am_[:24][ok[:24]], amr[ok[:24]]) and np.array_equal(am_[ok], amg.cpu().numpy()[ok])
    ps = sched["p"] if isinstance(sched["p"], list) else [sched["p"]] * sched["T"]
    tol = 1e-12 * max(1.0, float(np.prod(ps)) / 81.0)
    zz = z.cpu().numpy()
    worst = max(float(np.max(np.abs(zz[r] - zr[r])) / np.max(np.abs(zr[r]))) for r in np.nonzero(ok[:24])[0])
    assert worst <= tol, worst
    zg_ = zg.cpu().numpy()
    worst_g = max(float(np.max(np.abs(zz[r] - zg_[r])) / np.max(np.abs(zg_[r]))) for r in np.nonzero(ok)[0])
    assert worst_g <= tol, worst_g
