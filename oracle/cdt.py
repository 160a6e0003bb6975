"""Oracle-side CDT table for the discrete Gaussian (TEST INFRASTRUCTURE).

sigma = 3.2, support [-T, T] with T = floor(6 sigma) = 19
(reading G17 in DESIGN.md).  Thresholds thr[k] = floor(2^64 * CDF(-T + k)) for
k = 0 .. 2T-1, computed with Python's decimal module at 60 significant digits.
The CUDA library ships its own table as data, generated independently by
tools/gen_cdt_table.py (binary fixed point); the two are compared for equality by
tests/test_gpu_parity.py::test_keygen_matches_oracle.
"""
from decimal import Decimal, getcontext


def cdt_table(sigma: float = 3.2, T: int = 19):
    getcontext().prec = 60
    s = Decimal(str(sigma))
    rho = [(-(Decimal(e) ** 2) / (2 * s * s)).exp() for e in range(-T, T + 1)]
    Z = sum(rho)
    out, acc = [], Decimal(0)
    two64 = Decimal(2) ** 64
    for k in range(2 * T):
        acc += rho[k]
        out.append(int((acc / Z * two64).to_integral_value(rounding="ROUND_FLOOR")))
    return out
