import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfdfb.so")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


TOY = {  # small parameter set for exhaustive oracle pins (N=16, n=4)
    "name": "toy", "N": 16, "n": 4, "Q": 12289, "log_q_lwe": 16, "lwe_key": "binary", "rlwe_key": "ternary",
    "logL_rgsw": 5, "ell_rgsw": 3, "logL_boot": 5, "ell_boot": 3, "logL_pk": 5, "ell_pk": 3,
    "logL_ks": 4, "ell_ks": 4, "logL_pack": 1, "ell_pack": 14, "t": 4, "sigma": 3.2, "batch": 4,
    "seeds": {"keys": 11, "msgs": 12, "lut": 13, "err": 14},
}


@pytest.fixture
def toy_cfg():
    return dict(TOY)
