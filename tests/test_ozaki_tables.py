"""CPU check of the CRT tables behind the INT8-emulated FP64 GEMM
(paper_2209_08722_b200/ozaki_tables.py -> csrc/skb_ozaki.cu): with the
kernel's own split-double arithmetic, random integers |C| < P/4 are recovered
from their symmetric residues to fp64 accuracy, and the two leading partial
sums are exact."""

import math
import random
from fractions import Fraction

import numpy as np

from paper_2209_08722_b200 import ozaki_tables as T


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _reconstruct(n, residues):
    bits, s2, rows = T.table(n)
    q = 0.0
    for l in range(n):
        q = _fma(residues[l], rows[l][2], q)
    q = float(np.rint(q))
    t1 = t2 = t3 = 0.0
    for l in range(n):
        t1 = _fma(residues[l], rows[l][3], t1)
        t2 = _fma(residues[l], rows[l][4], t2)
        t3 = _fma(residues[l], rows[l][5], t3)
    P = rows[n]
    t1 = _fma(-q, P[3], t1)
    t2 = _fma(-q, P[4], t2)
    t3 = _fma(-q, P[5], t3)
    # the first two sums are integers below 2^53: exact in fp64
    assert abs(t1) < 2 ** 53 and abs(t2) < 2 ** 53
    return math.ldexp(_fma(t1, 2.0 ** 40, t2) + t3, s2)


def test_moduli_pairwise_coprime_and_int8():
    T._check_coprime()
    assert all(p <= 256 for p in T.MODULI)
    assert T.table(16)[0] >= 2 * 53 + math.log2(131071) + 2  # the kernel's K <= 131071


def test_crt_reconstruction_accuracy():
    rng = random.Random(7)
    for n in (16, 17):
        P = math.prod(T.MODULI[:n])
        for t in range(400):
            C = rng.randrange(-P // 4, P // 4) if t % 2 else rng.randrange(-2 ** 60, 2 ** 60)
            res = []
            for p in T.MODULI[:n]:
                r = C % p
                if r > p // 2:
                    r -= p
                res.append(float(r))
            assert all(abs(r) <= 128 for r in res)
            got = _reconstruct(n, res)
            s2 = T.table(n)[1]
            err = abs(Fraction(got) - C)
            assert err <= Fraction(abs(C), 2 ** 51) + 2 ** (s2 + 2), (n, C, float(err))
