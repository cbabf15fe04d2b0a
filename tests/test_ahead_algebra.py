"""CPU check of the algebra behind cutmax_ahead_kernel (DESIGN.md §4 K1b):
the moments of the next iterate y' = (a + k v)^3 from the power sums of v,

    sum y'^q = sum_j C(3q, j) a^(3q-j) k^j S_j,   q = 1, 2, 3,

reproduce the two-pass statistics of two CutMax iterations and the analytic
normaliser, so one cluster exchange can serve two iterations.  Checked
against the oracle (fsum-exact Python restatement of Alg. 1) on the BASELINE
distributions; the kernel's own results are compared with the C oracle in
tests/test_gpu_parity.py::test_ahead_kernel_*."""
import math

import numpy as np
import pytest

from paper_2509_08383_b200 import workloads as W


def exact(x, T=4, p=3, c=5.0):
    y = np.array(x, dtype=np.float64)
    n = len(y)
    for _ in range(T):
        mu = math.fsum(y) / n
        s2 = math.fsum((y - mu) ** 2) / n
        y = ((y - mu) / (c * math.sqrt(s2)) + 1.0) ** p
    return y / math.fsum(y)


def power_sums(v, m):
    out = [float(len(v))]
    w = np.ones_like(v)
    for _ in range(m):
        w = w * v
        out.append(float(np.sum(w)))
    return out


def expand(S, a, k, m):
    return sum(math.comb(m, j) * a ** (m - j) * k ** j * S[j] for j in range(m + 1))


def ahead(x, c=5.0):
    """T = 4 in two stages, the way the kernel schedules it."""
    n = len(x)
    kp = 1.0 + 3.0 / c ** 2
    K0 = float(np.mean(x[[(j * n) // 8 for j in range(8)]]))  # the kernel's input shift
    v = x - K0
    S = power_sums(v, 6)                                        # exchange 1: S_1..S_6
    dm = S[1] / n
    s2 = S[2] / n - dm * dm
    k1 = 1.0 / (c * math.sqrt(s2))
    a1 = 1.0 - dm * k1
    E3, E6 = expand(S, a1, k1, 3) / n, expand(S, a1, k1, 6) / n
    k2 = 1.0 / (c * math.sqrt(E6 - E3 * E3))
    b2 = 1.0 - E3 * k2
    v3 = (((v * k1 + a1) ** 3) * k2 + b2) ** 3 - kp                # pass: y2, y3 (shifted)
    S = power_sums(v3, 9)                                        # exchange 2: S_1..S_9
    dm = S[1] / n
    s2 = S[2] / n - dm * dm
    k3 = 1.0 / (c * math.sqrt(s2))
    a3 = 1.0 - dm * k3
    P3, P6, P9 = (expand(S, a3, k3, m) / n for m in (3, 6, 9))
    k4 = 1.0 / (c * math.sqrt(P6 - P3 * P3))
    b4 = 1.0 - P3 * k4
    SY = n * (b4 ** 3 + 3 * b4 * b4 * k4 * P3 + 3 * b4 * k4 * k4 * P6 + k4 ** 3 * P9)  # analytic normaliser
    y5 = (((v3 * k3 + a3) ** 3) * k4 + b4) ** 3                  # last pass: y4, y5
    return y5 / SY


@pytest.mark.parametrize("name", ["gauss", "zipf", "planted", "offset"])
def test_two_iterations_per_exchange_match_exact(name):
    if name == "gauss":
        X = W.gaussian(4, 32768, seed=81)
    elif name == "zipf":
        X = W.zipf_logits(3, 32768, seed=82)
    elif name == "planted":
        X, _, _ = W.planted(4, 32768, seed=83)
    else:
        X = W.gaussian(3, 8192, seed=84) + 1.0e3
    for x in X:
        z, zr = ahead(x), exact(x)
        assert int(np.argmax(z)) == int(np.argmax(zr))
        assert np.max(np.abs(z - zr)) / np.max(np.abs(zr)) <= 1e-12


def test_binomial_expansion_identity():
    rng = np.random.default_rng(85)
    v = rng.normal(0.0, 1.0, 1000)
    S = power_sums(v, 9)
    for m in (3, 6, 9):
        for a, k in ((0.9, 0.2), (1.1, -0.3)):
            direct = float(np.sum((a + k * v) ** m))
            assert abs(expand(S, a, k, m) - direct) <= 1e-12 * abs(direct)
