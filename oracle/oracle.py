"""ctypes driver for oracle/fdfb_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module.  Arrays are numpy uint64 in the canonical layouts documented at the
top of fdfb_oracle.c and in DESIGN.md.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from .cdt import cdt_table

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fdfb_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# parameter-vector indices (must match the enum in fdfb_oracle.c)
P_FIELDS = ["N", "n", "Q", "log_q_lwe", "lwe_key", "rlwe_key", "logL_rgsw", "ell_rgsw",
            "logL_boot", "ell_boot", "logL_pk", "ell_pk", "logL_ks", "ell_ks",
            "logL_pack", "ell_pack", "t", "noiseless"]


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle())
        thr = cdt_table()
        arr = (C.c_uint64 * len(thr))(*thr)
        _lib.or_set_cdt(arr, C.c_int(len(thr) // 2))
        _lib.or_lwe_phase.restype = C.c_uint64
        _lib.or_lwe_phase_q.restype = C.c_uint64
        _lib.or_mod_switch.restype = C.c_uint64
        _lib.or_mod_switch.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def u64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


def philox(ctr, key):
    out = np.zeros(4, dtype=np.uint64)
    lib().or_philox(_p(u64(ctr)), _p(u64(key)), _p(out))
    return out


def num_threads() -> int:
    return int(lib().or_num_threads())


class Oracle:
    """Plain CPU implementation of the paper's algorithms for one parameter set."""

    def __init__(self, cfg: dict, noiseless: bool = False):
        self.cfg = dict(cfg)
        self.N, self.n, self.Q = cfg["N"], cfg["n"], cfg["Q"]
        self.logq = cfg["log_q_lwe"]
        self.q_lwe = 1 << self.logq
        self.t = cfg["t"]
        self.u = 2 if cfg["lwe_key"] == "ternary" else 1
        self.noiseless = noiseless or cfg.get("sigma", 3.2) == 0
        vals = dict(cfg)
        vals["lwe_key"] = 1 if cfg["lwe_key"] == "ternary" else 0
        vals["rlwe_key"] = 1 if cfg["rlwe_key"] == "ternary" else 0
        vals["noiseless"] = 1 if self.noiseless else 0
        self.P = u64([vals[f] for f in P_FIELDS])
        self.L = {k: 1 << cfg["logL_" + k] for k in ("rgsw", "boot", "pk", "ks", "pack")}
        self.ell = {k: cfg["ell_" + k] for k in ("rgsw", "boot", "pk", "ks", "pack")}
        self.L_pack = self.L["pack"]
        lib()

    # ---------------------------------------------------------------- keys
    def keygen_secrets(self, seed):
        s = np.zeros(self.n, dtype=np.int8)
        S = np.zeros(self.N, dtype=np.int8)
        lib().or_keygen_secrets(_p(self.P), C.c_uint64(seed), _p(s), _p(S))
        return s, S

    def brk(self, seed, s, S):
        out = np.zeros((self.n, self.u, 2 * self.ell["rgsw"], 2, self.N), dtype=np.uint64)
        lib().or_brk_gen(_p(self.P), C.c_uint64(seed), _p(s), _p(S), _p(out))
        return out

    def bpk(self, seed, S):
        out = np.zeros((self.N, self.ell["pk"], 2, self.N), dtype=np.uint64)
        lib().or_bpk_gen(_p(self.P), C.c_uint64(seed), _p(S), _p(out))
        return out

    def ksk(self, seed, s, S):
        out = np.zeros((self.N, self.ell["ks"], self.n + 1), dtype=np.uint64)
        lib().or_ksk_gen(_p(self.P), C.c_uint64(seed), _p(s), _p(S), _p(out))
        return out

    def pack_key(self, seed, S):
        out = np.zeros((self.N, self.ell["pack"], self.L_pack, 2, self.N), dtype=np.uint64)
        lib().or_pack_gen(_p(self.P), C.c_uint64(seed), _p(S), _p(out))
        return out

    def pack_key_entry(self, seed, S, i, j, k0):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_pack_gen_entry(_p(self.P), C.c_uint64(seed), _p(S), C.c_int(i), C.c_int(j),
                                C.c_int(k0), _p(out))
        return out

    def keys(self, seed):
        s, S = self.keygen_secrets(seed)
        return dict(s=s, S=S, brk=self.brk(seed, s, S), bpk=self.bpk(seed, S), ksk=self.ksk(seed, s, S))

    # ---------------------------------------------------------------- encryption
    def lwe_encrypt(self, seed, s, msgs, exact=False):
        msgs = u64(msgs)
        out = np.zeros((len(msgs), self.n + 1), dtype=np.uint64)
        lib().or_lwe_encrypt_batch(_p(self.P), C.c_uint64(seed), _p(s), _p(msgs), C.c_int(len(msgs)),
                                   C.c_uint64(1 if exact else 0), _p(out))
        return out

    def rlwe_encrypt(self, seed, S, msgs):
        msgs = u64(msgs).reshape(-1, self.N)
        out = np.zeros((msgs.shape[0], 2, self.N), dtype=np.uint64)
        lib().or_rlwe_encrypt_batch(_p(self.P), C.c_uint64(seed), _p(S), _p(msgs),
                                    C.c_int(msgs.shape[0]), _p(out))
        return out

    def rlwe_encrypt_obj(self, seed, dom, i0, i1, i2, S, m):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_rlwe_encrypt(_p(self.P), C.c_uint64(seed), C.c_uint64(dom), C.c_uint64(i0),
                              C.c_uint64(i1), C.c_uint64(i2), _p(S), _p(u64(m)), _p(out))
        return out

    def lwe_phase(self, s, c, logq=None):
        logq = self.logq if logq is None else logq
        c = u64(c)
        return int(lib().or_lwe_phase(C.c_int(len(s)), C.c_int(logq), _p(s), _p(c)))

    def lwe_phase_q(self, s, c):
        c = u64(c)
        return int(lib().or_lwe_phase_q(C.c_int(len(s)), C.c_uint64(self.Q), _p(s), _p(c)))

    def rlwe_phase(self, S, c):
        c = u64(c)
        out = np.zeros(self.N, dtype=np.uint64)
        lib().or_rlwe_phase(C.c_int(self.N), C.c_uint64(self.Q), _p(S), _p(c), _p(out))
        return out

    def decode(self, phase, q, t):
        """round(t * phase / q) mod t (PAPER.md:1725 rounding)."""
        return ((int(phase) * t * 2 + q) // (2 * q)) % t

    # ---------------------------------------------------------------- ring / primitives
    def ring_mul(self, a, b, N=None, Q=None):
        N = self.N if N is None else N
        Q = self.Q if Q is None else Q
        out = np.zeros(N, dtype=np.uint64)
        lib().or_ring_mul(C.c_int(N), C.c_uint64(Q), _p(u64(a)), _p(u64(b)), _p(out))
        return out

    def monomial_mul(self, a, e, N=None, Q=None):
        N = self.N if N is None else N
        Q = self.Q if Q is None else Q
        out = np.zeros(N, dtype=np.uint64)
        lib().or_monomial_mul(C.c_int(N), C.c_uint64(Q), _p(u64(a)), C.c_int64(int(e)), _p(out))
        return out

    def decomp(self, x, logL, ell):
        out = np.zeros(ell, dtype=np.uint64)
        lib().or_decomp(C.c_uint64(int(x)), C.c_int(logL), C.c_int(ell), _p(out))
        return out

    def ext_prod(self, Cm, d):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_ext_prod(C.c_int(self.N), C.c_uint64(self.Q), C.c_int(self.cfg["logL_rgsw"]),
                          C.c_int(self.ell["rgsw"]), _p(u64(Cm)), _p(u64(d)), _p(out))
        return out

    def cmux(self, Cm, g, h):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_cmux(C.c_int(self.N), C.c_uint64(self.Q), C.c_int(self.cfg["logL_rgsw"]),
                      C.c_int(self.ell["rgsw"]), _p(u64(Cm)), _p(u64(g)), _p(u64(h)), _p(out))
        return out

    def blind_rotate(self, brk, acc, abar, n_steps=None):
        acc = u64(acc).copy()
        abar = np.ascontiguousarray(np.asarray(abar, dtype=np.uint32))
        n_steps = self.n if n_steps is None else n_steps
        lib().or_blind_rotate(_p(self.P), _p(u64(brk)), _p(acc), _p(abar), C.c_int(n_steps))
        return acc

    def mod_switch(self, x, Qfrom, qto):
        return int(lib().or_mod_switch(int(x), int(Qfrom), int(qto)))

    def sample_extract(self, ct, k):
        out = np.zeros(self.N + 1, dtype=np.uint64)
        lib().or_sample_extract(C.c_int(self.N), C.c_uint64(self.Q), _p(u64(ct)), C.c_int(k), _p(out))
        return out

    def keyswitch_lwe(self, ksk, c):
        out = np.zeros(self.n + 1, dtype=np.uint64)
        lib().or_keyswitch_lwe(_p(self.P), _p(u64(ksk)), _p(u64(c)), _p(out))
        return out

    def keyswitch_rlwe(self, bpk, c):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_keyswitch_rlwe(_p(self.P), _p(u64(bpk)), _p(u64(c)), _p(out))
        return out

    def pubmux(self, accR, p0, p1):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_pubmux(_p(self.P), _p(u64(accR)), _p(u64(p0)), _p(u64(p1)), _p(out))
        return out

    # ---------------------------------------------------------------- LUT / bootstrap
    def bootsmap(self, f, t_out=None):
        """BootsMap[x] = Delta_{Q,t'} * f(x) with Delta = round(Q/t')."""
        t_out = self.t if t_out is None else t_out
        delta = (2 * self.Q + t_out) // (2 * t_out)
        return u64([(delta * int(v)) % self.Q for v in f])

    def setup_polynomial(self, bootsmap):
        p0 = np.zeros(self.N, dtype=np.uint64)
        p1 = np.zeros(self.N, dtype=np.uint64)
        lib().or_setup_polynomial(_p(self.P), _p(u64(bootsmap)), _p(p0), _p(p1))
        return p0, p1

    def bootstrap(self, keys, rotp, cts):
        cts = u64(cts).reshape(-1, self.n + 1)
        out = np.zeros_like(cts)
        lib().or_bootstrap(_p(self.P), _p(u64(keys["brk"])), _p(u64(keys["bpk"])), _p(u64(keys["ksk"])),
                           _p(u64(rotp[0])), _p(u64(rotp[1])), _p(cts), C.c_int(cts.shape[0]), _p(out))
        return out

    def bootstrap_tfhe(self, keys, rotp0, cts):
        """TFHE half-domain bootstrap (Fig. PAPER.md:3070-3090, output order of reading c.3)."""
        cts = u64(cts).reshape(-1, self.n + 1)
        out = np.zeros_like(cts)
        lib().or_bootstrap_tfhe(_p(self.P), _p(u64(keys["brk"])), _p(u64(keys["ksk"])), _p(u64(rotp0)), _p(cts),
                                C.c_int(cts.shape[0]), _p(out))
        return out

    def blind_rotate_shift(self, brk, pk, acc, abar, n_steps=None):
        """BlindRotate_Shift (reading S1); abar already in Z_N."""
        acc = u64(acc).copy()
        abar = np.ascontiguousarray(np.asarray(abar, dtype=np.uint32))
        n_steps = self.n if n_steps is None else n_steps
        lib().or_blind_rotate_shift(_p(self.P), _p(u64(brk)), _p(u64(pk)), _p(acc), _p(abar), C.c_int(n_steps))
        return acc

    def bootstrap_shift(self, keys, pk, rotp, cts, n_steps=None):
        """Shift-based bootstrap (readings S1-S3, output order of c.3).
        rotp: one plaintext polynomial (N coefficients in [0, Q))."""
        cts = u64(cts).reshape(-1, self.n + 1)
        out = np.zeros_like(cts)
        n_steps = self.n if n_steps is None else n_steps
        lib().or_bootstrap_shift(_p(self.P), _p(u64(keys["brk"])), _p(u64(pk)), _p(u64(keys["ksk"])),
                                 _p(u64(rotp)), _p(cts), C.c_int(cts.shape[0]), C.c_int(n_steps), _p(out))
        return out

    # ---------------------------------------------------------------- packing / shift
    def pack(self, pk, c, d):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_pack(_p(self.P), _p(u64(pk)), _p(u64(c)), C.c_int(d), _p(out))
        return out

    def vector_pack(self, pk, v):
        v = u64(v).reshape(-1, self.N + 1)
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_vector_pack(_p(self.P), _p(u64(pk)), _p(v), C.c_int(v.shape[0]), _p(out))
        return out

    def shift(self, pk, ct, d, force_branch2=False):
        out = np.zeros((2, self.N), dtype=np.uint64)
        lib().or_shift(_p(self.P), _p(u64(pk)), _p(u64(ct)), C.c_int(int(d)),
                       C.c_int(1 if force_branch2 else 0), _p(out))
        return out

    def permute(self, pk, ct, perm, literal=False):
        """Permute(ct, pK, pi) (reading P1); perm[i-1] = pi(i), 1-based."""
        out = np.zeros((2, self.N), dtype=np.uint64)
        perm = np.ascontiguousarray(np.asarray(perm, dtype=np.uint32))
        lib().or_permute(_p(self.P), _p(u64(pk)), _p(u64(ct)), _p(perm), C.c_int(1 if literal else 0), _p(out))
        return out

    def permute_batch(self, pk, cts, perms):
        cts = u64(cts).reshape(-1, 2, self.N)
        perms = np.ascontiguousarray(np.asarray(perms, dtype=np.uint32)).reshape(-1, self.N)
        out = np.zeros_like(cts)
        lib().or_permute_batch(_p(self.P), _p(u64(pk)), _p(cts), _p(perms), C.c_int(cts.shape[0]), _p(out))
        return out

    def shift_batch(self, pk, cts, ds):
        cts = u64(cts).reshape(-1, 2, self.N)
        ds = np.ascontiguousarray(np.asarray(ds, dtype=np.uint32))
        out = np.zeros_like(cts)
        lib().or_shift_batch(_p(self.P), _p(u64(pk)), _p(cts), _p(ds), C.c_int(cts.shape[0]), _p(out))
        return out
