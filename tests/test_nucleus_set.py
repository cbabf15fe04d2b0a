"""The top-p nucleus itself: cutoff logit, size
and mass.  CPU: the oracle's sort-and-walk (oracle.c orc_nucleus_set) against
hand cases, a float64 numpy restatement and the membership predicate of
orc_nucleus_inside.  GPU: the cluster histogram scan (csrc/nucleus_set.cu)
against the oracle -- bit-exact, because the masses are fixed-point integers."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2509_08383_b200 import workloads as W


def np_nucleus(x, p):
    """float64 restatement: sort descending, walk the tie groups."""
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(x - x.max())
    order = np.argsort(-x, kind="stable")
    xs, es = x[order], e[order]
    total = es.sum()
    above, size, cutoff = 0.0, 0, None
    i = 0
    while i < len(xs):
        j = i
        while j < len(xs) and xs[j] == xs[i]:
            j += 1
        if not above < p * total:
            break
        cutoff, size = xs[i], j
        above += es[i:j].sum()
        i = j
    return cutoff, size, above / total


def test_oracle_hand_cases():
    # one dominant logit: mass > p alone -> nucleus = {that token}
    x = np.array([0.0, 10.0, 1.0, -2.0])
    cut, size, mass, st = orc.nucleus_set_batch(x, 0.9)
    assert st[0] == 0 and cut[0] == 10.0 and size[0] == 1 and mass[0] > 0.9
    # uniform logits: every entry ties with the cutoff; SPEC.md:464 includes ties,
    # so all n are inside (SPEC.md:444's "9 of 10" contradicts :464)
    cut, size, mass, st = orc.nucleus_set_batch(np.full(10, 0.25), 0.9)
    assert cut[0] == 0.25 and size[0] == 10 and mass[0] == 1.0
    # probabilities 0.5, 0.3, 0.2
    x = np.log(np.array([0.2, 0.5, 0.3]))
    for p, want in ((0.4, 1), (0.55, 2), (0.79, 2), (0.81, 3)):
        cut, size, mass, st = orc.nucleus_set_batch(x, p)
        assert size[0] == want, (p, size[0])
        assert cut[0] == np.sort(x)[::-1][want - 1]
    # -0.0 and +0.0 are one tie group; the cutoff comes back as +0.0
    cut, size, _, _ = orc.nucleus_set_batch(np.array([-0.0, 0.0, -5.0]), 0.5)
    assert size[0] == 2 and cut[0] == 0.0 and not np.signbit(cut[0])
    # errors
    _, _, _, st = orc.nucleus_set_batch(np.array([1.0, np.inf]), 0.9)
    assert st[0] == 5  # PAM_ERR_NON_FINITE
    _, _, _, st = orc.nucleus_set_batch(np.array([1.0, 2.0]), 1.5)
    assert st[0] != 0


@pytest.mark.parametrize("seed,n,p", [(1, 1000, 0.9), (2, 32768, 0.9), (3, 32768, 0.95), (4, 5000, 0.5), (5, 777, 0.99)])
def test_oracle_matches_float_restatement_and_membership(seed, n, p):
    x = W.zipf_logits(1, n, seed=seed)[0] if seed % 2 else W.gaussian(1, n, seed=seed)[0]
    cut, size, mass, st = orc.nucleus_set_batch(x, p)
    c2, s2, m2 = np_nucleus(x, p)
    assert st[0] == 0
    # the fixed-point masses move the boundary by < n * 2^-41 in mass: away from an
    # exact boundary the float restatement agrees entry for entry
    assert cut[0] == c2 and size[0] == s2
    assert abs(mass[0] - m2) < 1e-9
    assert size[0] == int((x >= cut[0]).sum())
    # membership predicate of the sampler (orc_nucleus_inside) <=> x_k >= cutoff
    rng = np.random.default_rng(seed)
    srt = np.argsort(-x)
    probe = list(rng.integers(0, n, 20)) + [int(srt[size[0] - 1])] + ([int(srt[size[0]])] if size[0] < n else [])
    for k in probe:
        assert orc.nucleus_inside(x, p, int(k)) == bool(x[k] >= cut[0])


def _gpu_vs_oracle(torch, pam, x, p):
    xt = torch.as_tensor(x, device="cuda")
    cut, size, mass, st = pam.nucleus_set_batch_device(xt, p)
    torch.cuda.synchronize()
    rc, rs, rm, rst = orc.nucleus_set_batch(x, p)
    assert np.array_equal(st.cpu().numpy(), rst)
    ok = rst == 0
    assert np.array_equal(size.cpu().numpy()[ok], rs[ok])
    assert np.array_equal(cut.cpu().numpy()[ok].view(np.uint64), rc[ok].view(np.uint64)), "cutoff bits differ"
    assert np.array_equal(mass.cpu().numpy()[ok].view(np.uint64), rm[ok].view(np.uint64)), "mass bits differ"
    return cut, size, mass, st


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0.9, 0.95])
def test_gpu_c4_shape(cuda, pam, p):
    """BASELINE C4: 128 x 32768 Zipf(1.1)-shaped logits (4-CTA clusters)."""
    x = W.zipf_logits(128, 32768, seed=11)
    cut, size, _, _ = _gpu_vs_oracle(cuda, pam, x, p)
    assert int(size.min()) >= 1
    # consistent with the fused sampler's membership flag
    cfg = pam.SamplerConfig(p=p, seed=99)
    tok, ins, st = pam.nucleus_sample_batch_device(cuda.as_tensor(x, device="cuda"), cfg, pam.CutMaxParams())
    xt = cuda.as_tensor(x, device="cuda")
    want = xt.gather(1, tok.long()[:, None])[:, 0] >= cut
    assert bool((want == ins.bool()).all())


@pytest.mark.gpu
@pytest.mark.parametrize("B,n,p", [(3, 10, 0.9), (40, 1024, 0.9), (33, 11264, 0.5), (20, 11266, 0.99), (9, 22528, 0.7),
                                   (17, 50257, 0.9), (24, 151936, 0.9), (5, 180224, 0.95)])
def test_gpu_shapes(cuda, pam, B, n, p):
    """Every cluster size (1..16 CTAs), ragged last slices, odd n."""
    x = W.gaussian(B, n, seed=n % 1000) if n % 2 else W.zipf_logits(B, n, seed=n % 1000)
    _gpu_vs_oracle(cuda, pam, x, p)


@pytest.mark.gpu
def test_gpu_ties_and_edges(cuda, pam):
    rng = np.random.default_rng(5)
    n = 40000
    x = np.round(rng.normal(0, 3, (16, n)), 1)  # heavy ties: ~120 distinct values
    x[0] = 0.25                                 # uniform row: all inside
    x[1, :] = -30.0
    x[1, 777] = 5.0                             # one dominant logit
    x[2, 100] = np.nan
    x[3, :5] = -0.0
    x[4] *= 1e-3                                # near-uniform
    x[5] += 1e6                                 # large offset
    cut, size, mass, st = _gpu_vs_oracle(cuda, pam, x, 0.9)
    assert int(size[0]) == n and float(mass[0]) == 1.0
    assert int(size[1]) == 1 and float(cut[1]) == 5.0
    assert int(st[2]) == 5 and int(size[2]) == 0


@pytest.mark.gpu
def test_gpu_errors_and_strided(cuda, pam):
    x = cuda.as_tensor(W.gaussian(4, 1000, seed=1), device="cuda")
    with pytest.raises(pam.DomainError):
        pam.nucleus_set_batch_device(x, 1.0)
    big = cuda.zeros((2, 180226), dtype=cuda.float64, device="cuda")
    with pytest.raises(pam.Error):
        pam.nucleus_set_batch_device(big, 0.9)
    wide = cuda.as_tensor(W.gaussian(6, 4096, seed=2), device="cuda")
    view = wide[:, :3000]  # ld 4096, n 3000
    cut, size, mass, st = pam.nucleus_set_batch_device(view, 0.8)
    rc, rs, rm, rst = orc.nucleus_set_batch(np.ascontiguousarray(view.cpu().numpy()), 0.8)
    assert np.array_equal(size.cpu().numpy(), rs) and np.array_equal(cut.cpu().numpy(), rc)
    d = pam.nucleusSet(view[0].cpu().numpy(), 0.8)
    assert d["size"] == rs[0] and d["cutoff"] == rc[0]


@pytest.mark.gpu
def test_gpu_fuzz(cuda, pam):
    """Seeded random shapes, scales, tie densities and p: every cluster size, n
    down to 1, rows with a handful of distinct values."""
    rng = np.random.default_rng(20250918)
    for case in range(40):
        n = int(rng.choice([1, 2, 7, 100, 1000, 4097, 11264, 11265, 30000, 60000, 100003]))
        B = int(rng.integers(1, 9))
        kind = case % 4
        if kind == 0:
            x = rng.normal(0.0, float(rng.choice([1e-3, 1.0, 3.0, 30.0])), (B, n))
        elif kind == 1:
            x = np.round(rng.normal(0.0, 2.0, (B, n)), int(rng.integers(0, 3)))  # heavy ties
        elif kind == 2:
            x = -1.1 * np.log(rng.permuted(np.tile(np.arange(1, n + 1, dtype=np.float64), (B, 1)), axis=1)) \
                + rng.normal(0, 0.5, (B, n))
        else:
            x = rng.normal(0.0, 3.0, (B, n)) + float(rng.choice([-1e6, 0.0, 1e3]))
        p = float(rng.choice([0.01, 0.3, 0.5, 0.9, 0.95, 0.999]))
        _gpu_vs_oracle(cuda, pam, np.ascontiguousarray(x), p)
