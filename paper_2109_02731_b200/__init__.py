"""B200-native (sm_100a) FDFB hot path: batched blind rotation, SampleExt, LWE key
switching, BuildAcc/PubMux and the coefficient Shift over VectorPack
(arXiv 2109.02731).  The compute lives in libfdfb.so (csrc/, C-ABI in
include/fdfb.h); this package is the thin ctypes binding."""
from .fdfb import Context, FdfbError, lib, params_from_config  # noqa: F401
from .fdfb import KEY_BRK, KEY_BPK, KEY_KSK, KEY_PACK  # noqa: F401
