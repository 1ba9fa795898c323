"""Host checks of the GPU value path's numerical building blocks, no GPU needed:
the generated 2^(j/256) table (paper_2602_23040_b200/csrc/exp2_table.h) is the correctly rounded
one, and the exp64 algorithm of contract.cuh (one-constant Cody-Waite reduction, table, degree-3
Taylor), emulated in numpy fp64, stays within 3e-13 relative of exp over the compositing range."""
import decimal
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _table():
    src = open(os.path.join(ROOT, "paper_2602_23040_b200", "csrc", "exp2_table.h")).read()
    return [float.fromhex(h) for h in re.findall(r"0x[0-9a-f.]+p[+-]\d+", src)]


def test_exp2_table_correctly_rounded():
    tab = _table()
    assert len(tab) == 256
    decimal.getcontext().prec = 60
    for j in (0, 1, 37, 128, 200, 255):
        exact = decimal.Decimal(2) ** (decimal.Decimal(j) / 256)
        assert tab[j] == float(exact)
        # the neighbours of the stored value are no closer to the exact value
        d = abs(decimal.Decimal(tab[j]) - exact)
        for nb in (math.nextafter(tab[j], 0.0), math.nextafter(tab[j], 2.0)):
            assert abs(decimal.Decimal(nb) - exact) >= d


def test_exp64_emulation_error():
    tab = np.array(_table())
    L = math.log(2) / 256
    x = np.linspace(-6.0, 0.0, 2_000_001)
    k = np.rint(x * (256 / math.log(2)))
    r = x - k * L
    p = 1 + r * (1 + r * (0.5 + r / 6))
    v = tab[(k.astype(np.int64) & 255)] * p * np.exp2(np.floor(k / 256))
    assert np.max(np.abs(v / np.exp(x) - 1)) < 3e-13
