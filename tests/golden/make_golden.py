"""Generate the committed golden fixtures for the oracle pin.

The reference ships no implementation and no fixtures, so
the golden vectors come from two independent sources:

1. The SPEC's own known answers (spec_known_answers.json), evaluated here from
   their closed forms with exactly-rounded sums (math.fsum) — SPEC.md:67, 77,
   78, 79, 84-88, 97, 163-165, 173-175, 403-404, 421-425, 433-435.
2. A second, independent restatement of Alg. 1 in pure Python
   with math.fsum reductions (cutmax_golden.npz): small vectors and their
   CutMax outputs, which the C oracle must reproduce to 1e-13 normwise with the
   identical argmax.
3. Published Philox4x32-10 known-answer vectors (Salmon et al., SC'11,
   Random123 kat_vectors) for the pinned RNG (philox_kat.json).

Run:  python tests/golden/make_golden.py   (rewrites the fixtures; deterministic)
"""
import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def ipow(z, p):
    acc, sq, have = None, z, False
    while p > 0:
        if p & 1:
            acc = sq if not have else acc * sq
            have = True
        p >>= 1
        if p:
            sq = sq * sq
    return acc if have else 1.0


def cutmax_ref(x, ps, cs):
    """Alg. 1 with exactly-rounded (fsum) mean/variance; textbook standardisation."""
    y = [float(v) for v in x]
    n = len(y)
    for p, c in zip(ps, cs):
        mu = math.fsum(y) / n
        s2 = math.fsum((v - mu) ** 2 for v in y) / n
        k = (1.0 / math.sqrt(s2)) * (1.0 / c)
        y = [ipow((v - mu) * k + 1.0, p) for v in y]
    tot = math.fsum(y)
    r = 1.0 / tot
    z = [v * r for v in y]
    am = max(range(n), key=lambda i: (z[i], -i))
    return np.array(z), am


def s_star(n, p, c):
    a = (1 + math.sqrt(n - 1) / c) ** p
    b = (1 - 1 / (c * math.sqrt(n - 1))) ** p
    return a / (a + (n - 1) * b)


def main():
    kat = {
        "spec67_x": [5.0, 2.0, 1.0], "spec67_argmax": 0,
        "spec77_residuals_n3": [math.sqrt(2.0), -1 / math.sqrt(2.0), -1 / math.sqrt(2.0)],
        "spec78_next": [1.2 ** 3, 0.8 ** 3],
        "spec78_residuals": [1.0, -1.0],
        "spec88_sstar_n3_p3_c5": s_star(3, 3, 5.0),
        "spec87_sstar_n2_p3_c5": (1 + 1 / 5) ** 3 / ((1 + 1 / 5) ** 3 + (1 - 1 / 5) ** 3),
        "spec97_kappa_n2_p3_c10": (0.09 * 1.1 ** 4) / (4 * 0.9 ** 6),
        "spec164_inv_0p5": 2.0, "spec165_inv_1p5": 2.0 / 3.0, "spec_inv_tol": 2.0 ** -7,
        "spec174_invsqrt_0p25": 2.0,
        "spec175_invsqrt_preset_alpha7": [5, 10],
        "table3_invsqrt_iters": {"7": 5, "9": 6, "11": 7, "13": 8},
        "spec403_gumbel_u_e-1": [math.exp(-1.0), 0.0],
        "spec404_gumbel_u_e-e": [math.exp(-math.e), -1.0],
        "spec434_alpha_p0.9": math.log(0.1) / math.log(0.9),
        "alpha_p0.95": math.log(0.05) / math.log(0.95),
        "spec66_two_level_n8_sstar": s_star(8, 3, 5.0),
    }
    with open(os.path.join(HERE, "spec_known_answers.json"), "w") as f:
        json.dump(kat, f, indent=1, sort_keys=True)

    rng = np.random.default_rng(20250908)
    cases = []
    for i, (n, dist, ps, cs) in enumerate([
        (2, "normal", [3], [5.0]),
        (3, "normal", [3, 3], [5.0, 5.0]),
        (8, "onehot", [3, 3, 3, 3], [5.0] * 4),
        (64, "normal", [3] * 4, [5.0] * 4),
        (257, "zipf", [3] * 4, [5.0] * 4),
        (1000, "normal", [13] * 4, [15.0] * 4),
        (1000, "zipf", [9] * 5, [15.0] * 5),
        (2048, "normal", [19] * 3, [27.0] * 3),
        (4096, "zipf", [3] * 3, [5.0] * 3),
    ]):
        if dist == "normal":
            x = rng.normal(0, 3, n)
        elif dist == "onehot":
            x = np.zeros(n)
            x[-1] = 1.0
        else:
            x = rng.permutation(-1.1 * np.log(np.arange(1, n + 1)) + rng.normal(0, 0.5, n))
        z, am = cutmax_ref(x, ps, cs)
        cases.append((x, np.array(ps), np.array(cs), z, am))
    np.savez(os.path.join(HERE, "cutmax_golden.npz"),
             **{f"x{i}": c[0] for i, c in enumerate(cases)},
             **{f"p{i}": c[1] for i, c in enumerate(cases)},
             **{f"c{i}": c[2] for i, c in enumerate(cases)},
             **{f"z{i}": c[3] for i, c in enumerate(cases)},
             argmax=np.array([c[4] for c in cases]), count=np.array(len(cases)))

    philox = [  # (ctr, key, expected) — Random123 kat_vectors, philox4x32 10 rounds
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    with open(os.path.join(HERE, "philox_kat.json"), "w") as f:
        json.dump([{"ctr": a, "key": b, "out": c} for a, b, c in philox], f, indent=1)


if __name__ == "__main__":
    main()
