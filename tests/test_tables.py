"""The CUDA path's constant tables (host-checkable, no GPU): each entry of the fill's 2^(j/2048)
table and of the 2^(j/64) table is the correctly rounded fp64 value (checked against exp(j ln2 / N) summed as a Taylor
series in 70-digit decimal arithmetic -- a different method from the generator's 2 ** (j / N)),
and the exp constants of h2_internal.cuh are the rounded
values of 2048/ln2 and ln2/2048."""
import math
import os
import re
from decimal import Decimal, getcontext

import pytest

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2206_01885_b200", "csrc")


def _table(name):
    text = open(os.path.join(CSRC, name)).read()
    body = text[text.index("{") + 1:text.rindex("}")]
    return [float.fromhex(x) for x in re.findall(r"0x[0-9a-fA-F.]+p[+-]?\d+", body)]


def _exp_taylor(x):
    """e^x for small Decimal x by its Taylor series (60 digits)."""
    term, total, k = Decimal(1), Decimal(1), 1
    while abs(term) > Decimal(10) ** -70:
        term = term * x / k
        total += term
        k += 1
    return total


def _ln2():
    # ln 2 = sum 1 / (k 2^k)
    getcontext().prec = 70
    return sum(Decimal(1) / (k * Decimal(2) ** k) for k in range(1, 240))


@pytest.mark.parametrize("name,N", [("exp_table2048.inc", 2048), ("exp_table.inc", 64)])
def test_exp2_tables_correctly_rounded(name, N):
    vals = _table(name)
    assert len(vals) == N
    ln2 = _ln2()
    for j in range(0, N, 1 if N <= 64 else 7):
        exact = _exp_taylor(ln2 * j / N)
        v = vals[j]
        # correctly rounded: |v - exact| <= half an ulp of v
        assert abs(Decimal(v) - exact) <= Decimal(math.ulp(v)) / 2, (j, v)


def test_fill_exp_constants():
    text = open(os.path.join(CSRC, "h2_internal.cuh")).read()
    blk = text[text.index("kFillC[5]"):]
    blk = blk[:blk.index("};")]
    consts = [float.fromhex(x) for x in re.findall(r"0x[0-9a-fA-F.]+p[+-]?\d+", blk)]
    ln2 = _ln2()
    assert consts[0] == float(Decimal(2048) / ln2)
    assert consts[1] == float(ln2 / 2048)
