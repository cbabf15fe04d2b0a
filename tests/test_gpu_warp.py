"""The warp-per-row kernel (csrc/cutmax_warp_kernel.cuh: aligned rows with
n <= 1536 fp64 / 3072 fp32) against the CPU oracle: argmax and status
(TieWarning included) exact, Z within 1e-12 (fp64) / 1e-5 (fp32) normwise,
tolerances scaled by prod(p)/81 for other schedules as in test_gpu_parity.py.
Covers rows that fill the 32 x E slots exactly and rows that do not, n down to
2, T = 1, generic p, polynomial scalars, the per-iteration stats, degenerate,
non-finite, shifted (one-pass cancellation) and tied rows, and checks that
unaligned rows go to the cluster kernel instead.
"""
import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu

TIE = 0x100


def run(torch, pam, x, prm, stats=False):
    xt = torch.as_tensor(np.ascontiguousarray(x), device="cuda")
    B = x.shape[0]
    sv = torch.empty((B, prm.T, 2), dtype=torch.float64, device="cuda") if stats else None
    z, am, st = pam.cutmax_batch_device(xt, prm, stats=sv)
    torch.cuda.synchronize()
    kid = pam.launch_info(x.dtype.itemsize, B, x.shape[1], prm)["kernel_id"]
    return z.cpu().numpy(), am.cpu().numpy(), st.cpu().numpy(), (sv.cpu().numpy() if stats else None), kid


def check(pam, orc, x, prm, tol, stats=False, want_warp=True):
    import torch

    z, am, st, sv, kid = run(torch, pam, x, prm, stats)
    assert (kid >= 2000) == want_warp, kid
    zr, amr, sr = orc.cutmax_batch(x, prm.lower())
    assert np.array_equal(st, sr), f"status {st[st != sr][:5]} vs {sr[st != sr][:5]}"
    ok = (st & 0xFF) == 0
    assert np.array_equal(am[ok], amr[ok])
    worst = max((normwise(z[r], zr[r]) for r in np.nonzero(ok)[0]), default=0.0)
    assert worst <= tol, worst
    if stats:  # mu within 1e-11 sigma, s2 within 1e-11 relative, against the fp64 oracle
        for r in np.nonzero(ok)[0][:8]:
            _, _, _, ref = orc.cutmax(x[r], prm.lower())
            assert np.all(np.abs(sv[r, :, 0] - ref[:, 0]) <= 1e-11 * np.sqrt(ref[:, 1]))
            assert np.all(np.abs(sv[r, :, 1] - ref[:, 1]) <= 1e-11 * ref[:, 1])
    return st


@pytest.mark.parametrize("n", [2, 3, 31, 64, 256, 1000, 1024, 1536])
@pytest.mark.parametrize("T", [1, 2, 4])
def test_warp_fp64_gaussian(cuda, pam, orc, n, T):
    B = 37
    x = np.random.default_rng(n * 10 + T).normal(0.0, 3.0, size=(B, n))
    check(pam, orc, x, pam.CutMaxParams(T=T), 1e-12, stats=(T == 4))


@pytest.mark.parametrize("n", [64, 1000, 1024, 3072])
def test_warp_fp32(cuda, pam, orc, n):
    x = np.random.default_rng(n).normal(0.0, 3.0, size=(64, n)).astype(np.float32)
    check(pam, orc, x, pam.CutMaxParams(), 1e-5)


def test_warp_generic_p_poly_and_unnormalised(cuda, pam, orc):
    x = np.random.default_rng(3).normal(0.0, 3.0, size=(48, 1024))
    check(pam, orc, x, pam.CutMaxParams(p=5, c=12.0, T=3), 1e-12 * 125 / 81)
    check(pam, orc, x, pam.CutMaxParams(p=[3, 5, 3], c=[5.0, 9.0, 5.0], T=3), 1e-12 * 45 / 81)
    check(pam, orc, x, pam.CutMaxParams(invsqrtMode="poly", invMode="poly"), 1e-12)
    check(pam, orc, x, pam.CutMaxParams(normalize=False), 1e-12)


def test_warp_edge_rows(cuda, pam, orc):
    """Degenerate, NaN, Inf, shifted with an outlier as the shift point (exact second pass),
    duplicated maxima and sub-1e-9 gaps (TieWarning screen + exact re-scan),
    a one-hot row; 1000 rows so every warp runs several rows."""
    rng = np.random.default_rng(11)
    B, n = 1000, 1024
    x = rng.normal(0.0, 3.0, size=(B, n))
    x[5] = 2.5
    x[6, 100] = np.nan
    x[7, 3] = -np.inf
    x[8:20] += 3e4  # |mean| / sigma ~ 1e4 (conditioning limit of the 1e-12 bar)
    x[8:20, 0] += 40.0  # K0 = x[0] ~ 13 sigma off the mean: the one-pass moments cancel -> exact second pass
    for r in range(20, 60):
        i, j = rng.choice(n, size=2, replace=False)
        top = x[r].max() + 1.0
        x[r, i] = top
        x[r, j] = top - [0.0, 5e-10, 9.99e-10, 1.001e-9, 3e-9][r % 5]
    x[60] = 0.0
    x[60, 777] = 1.0
    st = check(pam, orc, x, pam.CutMaxParams(), 1e-12)
    assert st[5] & 0xFF and st[6] & 0xFF and st[7] & 0xFF
    assert np.count_nonzero(st[20:60] & TIE) >= 24


def test_warp_unaligned_goes_to_cluster_kernel(cuda, pam, orc):
    import torch

    x = np.random.default_rng(4).normal(0.0, 3.0, size=(16, 1025))
    base = torch.as_tensor(x, device="cuda")
    xv = base[:, 1:]  # rows 16-byte misaligned, n = 1024 odd leading dimension
    prm = pam.CutMaxParams()
    z, am, st = pam.cutmax_batch_device(xv, prm)
    torch.cuda.synchronize()
    zr, amr, sr = orc.cutmax_batch(np.ascontiguousarray(x[:, 1:]), prm.lower())
    assert np.array_equal(st.cpu().numpy(), sr) and np.array_equal(am.cpu().numpy(), amr)
    zz = z.cpu().numpy()
    assert max(normwise(zz[r], zr[r]) for r in range(16)) <= 1e-12
