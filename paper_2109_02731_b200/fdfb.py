"""Thin ctypes binding of libfdfb.so (include/fdfb.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libfdfb.so.  torch is used for device memory and streams.  There is NO CPU
fallback: if the shared library is missing or no CUDA device is present the
calls raise.
"""
import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfdfb.so")

KEY_BRK, KEY_BPK, KEY_KSK, KEY_PACK, KEY_SK_LWE, KEY_SK_RLWE = 1, 2, 3, 4, 5, 6


class fdfb_params(C.Structure):
    _fields_ = [("N", C.c_uint32), ("n", C.c_uint32), ("Q", C.c_uint64), ("log_q_lwe", C.c_uint32),
                ("lwe_key", C.c_uint32), ("rlwe_key", C.c_uint32),
                ("logL_rgsw", C.c_uint32), ("ell_rgsw", C.c_uint32), ("logL_boot", C.c_uint32),
                ("ell_boot", C.c_uint32), ("logL_pk", C.c_uint32), ("ell_pk", C.c_uint32),
                ("logL_ks", C.c_uint32), ("ell_ks", C.c_uint32), ("logL_pack", C.c_uint32),
                ("ell_pack", C.c_uint32), ("t", C.c_uint32), ("sigma_milli", C.c_uint32)]


class fdfb_sizes_t(C.Structure):
    _fields_ = [(k, C.c_size_t) for k in ("sk_lwe", "sk_rlwe", "brk", "bpk", "ksk", "pack",
                                           "canon_brk", "canon_bpk", "canon_ksk", "canon_pack")]


class FdfbError(RuntimeError):
    pass


_lib = None
_EXPORTS = ["fdfb_ctx_create", "fdfb_ctx_destroy", "fdfb_sizes", "fdfb_workspace_bootstrap", "fdfb_workspace_shift",
            "fdfb_workspace_vector_pack", "fdfb_keygen", "fdfb_keygen_canonical", "fdfb_key_import",
            "fdfb_lwe_encrypt", "fdfb_rlwe_encrypt", "fdfb_setup_lut", "fdfb_bootstrap_batch",
            "fdfb_bootstrap_batch_host", "fdfb_blind_rotate", "fdfb_sample_extract", "fdfb_lwe_keyswitch",
            "fdfb_vector_pack", "fdfb_shift", "fdfb_poly_mul", "fdfb_cdt_table", "fdfb_launch_count",
            "fdfb_status_string", "fdfb_last_cuda_error", "fdfb_timing_enable", "fdfb_timing_read",
            "fdfb_pack", "fdfb_device_status", "fdfb_key_export", "fdfb_shift_streaming",
            "fdfb_workspace_keyswitch", "fdfb_workspace_bootstrap_multi", "fdfb_bootstrap_multi_batch",
            "fdfb_bootstrap_tfhe_batch", "fdfb_workspace_permute", "fdfb_permute",
            "fdfb_workspace_bootstrap_shift", "fdfb_bootstrap_shift_batch", "fdfb_lwe_decrypt", "fdfb_rlwe_phase",
            "fdfb_gemm_i8", "fdfb_workspace_keygen", "fdfb_workspace_keygen_canonical",
            "fdfb_workspace_rlwe_encrypt", "fdfb_workspace_poly_mul", "fdfb_workspace_rlwe_phase",
            "fdfb_timing_read_union"]
KCLASS = {"blind_rotate": 0, "keyswitch_rlwe": 1, "keyswitch_lwe": 2, "shift": 3, "shift_gemm": 4}


def lib():
    """Load libfdfb.so (no fallback: raises if absent)."""
    global _lib
    if _lib is None:
        from . import build as _build
        if _build.is_stale():                      # missing or built from other sources: rebuild (nvcc)
            try:
                _build.build()
            except Exception as e:  # no nvcc / compile error: fail loudly, there is no CPU path
                raise FdfbError("libfdfb.so missing or stale and the build failed: %s" % e)
        if not os.path.exists(LIB_PATH) or _build.is_stale():
            raise FdfbError("libfdfb.so not built (run __graft_entry__.build()); no CPU fallback exists")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_size_t
        L.fdfb_ctx_create.argtypes = [C.POINTER(fdfb_params), C.c_int, C.POINTER(vp)]
        L.fdfb_ctx_destroy.argtypes = [vp]
        L.fdfb_ctx_destroy.restype = None
        L.fdfb_sizes.argtypes = [vp, C.POINTER(fdfb_sizes_t)]
        L.fdfb_workspace_bootstrap.argtypes = [vp, u32]
        L.fdfb_workspace_bootstrap.restype = sz
        L.fdfb_workspace_shift.argtypes = [vp, u32]
        L.fdfb_workspace_shift.restype = sz
        L.fdfb_workspace_vector_pack.argtypes = [vp, u32, u32]
        L.fdfb_workspace_vector_pack.restype = sz
        L.fdfb_keygen.argtypes = [vp, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.fdfb_keygen_canonical.argtypes = [vp, u64, C.c_int, vp, vp, vp, u32, vp, vp, vp]
        for f, a in (("fdfb_workspace_keygen", [vp]), ("fdfb_workspace_keygen_canonical", [vp, u32]),
                     ("fdfb_workspace_rlwe_encrypt", [vp, u32]), ("fdfb_workspace_poly_mul", [vp, u32]),
                     ("fdfb_workspace_rlwe_phase", [vp, u32])):
            getattr(L, f).argtypes = a
            getattr(L, f).restype = sz
        L.fdfb_key_import.argtypes = [vp, C.c_int, vp, vp, vp]
        L.fdfb_lwe_encrypt.argtypes = [vp, u64, vp, vp, u32, u32, u64, vp, vp]
        L.fdfb_rlwe_encrypt.argtypes = [vp, u64, vp, vp, u32, u64, vp, vp, vp]
        L.fdfb_setup_lut.argtypes = [vp, vp, u32, vp, vp]
        L.fdfb_bootstrap_batch.argtypes = [vp, vp, vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_bootstrap_batch_host.argtypes = [vp, vp, vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_blind_rotate.argtypes = [vp, vp, vp, vp, u32, u32, vp]
        L.fdfb_sample_extract.argtypes = [vp, vp, vp, vp, u32, vp]
        L.fdfb_lwe_keyswitch.argtypes = [vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_workspace_bootstrap_multi.argtypes = [vp, u32, u32]
        L.fdfb_workspace_bootstrap_multi.restype = sz
        L.fdfb_bootstrap_multi_batch.argtypes = [vp, vp, vp, vp, vp, u32, vp, vp, u32, vp, vp]
        L.fdfb_bootstrap_tfhe_batch.argtypes = [vp, vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_workspace_bootstrap_shift.argtypes = [vp, u32]
        L.fdfb_workspace_bootstrap_shift.restype = sz
        L.fdfb_bootstrap_shift_batch.argtypes = [vp, vp, vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_lwe_decrypt.argtypes = [vp, vp, vp, u32, u32, vp, vp, vp]
        L.fdfb_rlwe_phase.argtypes = [vp, vp, vp, u32, vp, vp, vp]
        L.fdfb_workspace_permute.argtypes = [vp, u32]
        L.fdfb_workspace_permute.restype = sz
        L.fdfb_permute.argtypes = [vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_workspace_keyswitch.argtypes = [vp, u32]
        L.fdfb_workspace_keyswitch.restype = sz
        L.fdfb_vector_pack.argtypes = [vp, vp, vp, u32, vp, u32, vp, vp]
        L.fdfb_shift.argtypes = [vp, vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_shift_streaming.argtypes = [vp, vp, vp, vp, vp, u32, vp]
        L.fdfb_poly_mul.argtypes = [vp, vp, vp, vp, u32, vp, vp]
        L.fdfb_gemm_i8.argtypes = [vp, vp, vp, u32, u32, u32, vp, vp]
        L.fdfb_cdt_table.argtypes = [vp, vp, C.POINTER(C.c_int)]
        L.fdfb_launch_count.argtypes = [vp]
        L.fdfb_launch_count.restype = u64
        L.fdfb_status_string.argtypes = [C.c_int]
        L.fdfb_status_string.restype = C.c_char_p
        L.fdfb_last_cuda_error.restype = C.c_char_p
        L.fdfb_timing_enable.argtypes = [vp, C.c_int]
        L.fdfb_key_export.argtypes = [vp, C.c_int, vp, vp, vp]
        L.fdfb_pack.argtypes = [vp, vp, vp, vp, vp, u32, vp]
        L.fdfb_device_status.argtypes = [vp, C.c_int]
        L.fdfb_timing_read.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(u64)]
        L.fdfb_timing_read_union.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(u64)]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        L = lib()
        msg = L.fdfb_status_string(rc).decode()
        if rc == -8:
            msg += ": " + L.fdfb_last_cuda_error().decode()
        raise FdfbError("fdfb error %d: %s" % (rc, msg))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise FdfbError("tensor must be contiguous")
        if not t.is_cuda and t.numel() and not t.is_pinned():
            raise FdfbError("host tensors must be pinned (device entry points take CUDA tensors)")
        return C.c_void_p(t.data_ptr())
    return t


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _keep(stream, *tensors):
    """Tensors allocated on the current stream but used by kernels enqueued on `stream`:
    tell the caching allocator, so their memory is not handed out again before `stream`
    has finished with it (temporaries dropped on return, outputs freed later)."""
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            t.record_stream(stream)


def params_from_config(cfg: dict, noiseless: bool = False) -> fdfb_params:
    p = fdfb_params()
    for k in ("N", "n", "Q", "log_q_lwe", "logL_rgsw", "ell_rgsw", "logL_boot", "ell_boot", "logL_pk", "ell_pk",
              "logL_ks", "ell_ks", "logL_pack", "ell_pack", "t"):
        setattr(p, k, int(cfg[k]))
    p.lwe_key = 1 if cfg["lwe_key"] == "ternary" else 0
    p.rlwe_key = 1 if cfg["rlwe_key"] == "ternary" else 0
    p.sigma_milli = 0 if (noiseless or cfg.get("sigma", 3.2) == 0) else int(round(cfg.get("sigma", 3.2) * 1000))
    return p


class Context:
    """One parameter set on one device.  Methods mirror the C-ABI names."""

    def __init__(self, cfg: dict, device: int = 0, noiseless: bool = False):
        if not torch.cuda.is_available():
            raise FdfbError("no CUDA device: the FDFB library has no CPU path")
        self.cfg = dict(cfg)
        self.device = torch.device("cuda", device)
        self.p = params_from_config(cfg, noiseless)
        h = C.c_void_p()
        _check(lib().fdfb_ctx_create(C.byref(self.p), device, C.byref(h)))
        self.h = h
        self.N, self.n, self.Q = cfg["N"], cfg["n"], cfg["Q"]
        self.u = 2 if cfg["lwe_key"] == "ternary" else 1
        s = fdfb_sizes_t()
        _check(lib().fdfb_sizes(self.h, C.byref(s)))
        self.sizes = {k: getattr(s, k) for k, _ in fdfb_sizes_t._fields_}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().fdfb_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ---------------------------------------------------------------- buffers
    def _u64(self, *shape):
        return torch.empty(shape, dtype=torch.uint64, device=self.device)

    def _bytes(self, n):
        return torch.empty(max(int(n), 8), dtype=torch.uint8, device=self.device)

    def launch_count(self) -> int:
        return int(lib().fdfb_launch_count(self.h))

    def timing_enable(self, on: bool = True):
        _check(lib().fdfb_timing_enable(self.h, 1 if on else 0))

    def timing_read(self, kclass: str, union: bool = False):
        """(device ms, launches) of one kernel class since the last read: summed durations, or with
        union=True the span the launches cover (launches on two streams may overlap)."""
        ms, cnt = C.c_double(), C.c_uint64()
        f = lib().fdfb_timing_read_union if union else lib().fdfb_timing_read
        _check(f(self.h, KCLASS[kclass], C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    # ---------------------------------------------------------------- keys
    def keygen(self, seed: int, which: int = 0x0F, sk=None, stream=None):
        """fdfb_keygen: returns dict of device tensors (secrets + opaque keys)."""
        if sk is None:
            sk = (torch.empty(self.n, dtype=torch.int8, device=self.device),
                  torch.empty(self.N, dtype=torch.int8, device=self.device))
            which |= 1
        keys = {"s": sk[0], "S": sk[1]}
        for bit, name in ((2, "brk"), (4, "bpk"), (8, "ksk"), (16, "pack")):
            keys[name] = self._bytes(self.sizes[name]) if which & bit else None
        ws = self._bytes(lib().fdfb_workspace_keygen(self.h)) if which & 30 else None
        _keep(stream, ws, *[v for v in keys.values() if v is not None])
        _check(lib().fdfb_keygen(self.h, C.c_uint64(seed), which, _ptr(keys["s"]), _ptr(keys["S"]),
                                 _ptr(keys["brk"]), _ptr(keys["bpk"]), _ptr(keys["ksk"]), _ptr(keys["pack"]),
                                 _ptr(ws), _stream(stream)))
        return keys

    def keygen_canonical(self, seed, kind, s, S, idx, stream=None):
        import numpy as np
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
        per = (self.n + 1) if kind == KEY_KSK else 2 * self.N
        out = self._u64(len(idx), per)
        ws = self._bytes(lib().fdfb_workspace_keygen_canonical(self.h, len(idx)))
        _keep(stream, out, ws)
        _check(lib().fdfb_keygen_canonical(self.h, C.c_uint64(seed), kind, _ptr(s), _ptr(S),
                                           idx.ctypes.data_as(C.c_void_p), len(idx), _ptr(out), _ptr(ws),
                                           _stream(stream)))
        return out

    def key_import(self, kind: int, canonical: torch.Tensor, stream=None):
        name = {KEY_BRK: "brk", KEY_BPK: "bpk", KEY_KSK: "ksk", KEY_PACK: "pack"}[kind]
        dev = self._bytes(self.sizes[name])
        canonical = canonical.contiguous()
        _keep(stream, dev, canonical)
        _check(lib().fdfb_key_import(self.h, kind, _ptr(canonical), _ptr(dev), _stream(stream)))
        return dev

    def key_export(self, kind: int, dev_key: torch.Tensor, stream=None):
        """Canonical (coefficient-domain) layout of a device key; BRK through inverse NTT + CRT."""
        name = {KEY_BRK: "canon_brk", KEY_BPK: "canon_bpk", KEY_KSK: "canon_ksk", KEY_PACK: "canon_pack"}[kind]
        out = self._u64(self.sizes[name] // 8)
        _keep(stream, out)
        _check(lib().fdfb_key_export(self.h, kind, _ptr(dev_key), _ptr(out), _stream(stream)))
        return out

    # ---------------------------------------------------------------- inputs / LUT
    def lwe_encrypt(self, seed, s, msgs: torch.Tensor, exact=False, first_index=0, stream=None):
        """LWE encryptions of msgs; ciphertext c is object first_index + c of the seed's stream
        (a shard passes its global offset and gets exactly the single-device ciphertexts)."""
        out = self._u64(msgs.numel(), self.n + 1)
        _keep(stream, out)
        _check(lib().fdfb_lwe_encrypt(self.h, C.c_uint64(seed), _ptr(s), _ptr(msgs), msgs.numel(),
                                      1 if exact else 0, C.c_uint64(first_index), _ptr(out), _stream(stream)))
        return out

    def lwe_decrypt(self, s, ct, t=None, stream=None):
        """Phase b - <a, s> mod q_lwe of every LWE ciphertext, and with t the decoded message
        round(t phase / q_lwe) mod t (fdfb_lwe_decrypt).  Returns (phase, msg or None)."""
        B = ct.shape[0]
        phase = self._u64(B)
        msg = self._u64(B) if t else None
        _keep(stream, phase, msg)
        _check(lib().fdfb_lwe_decrypt(self.h, _ptr(s), _ptr(ct), B, int(t or 0), _ptr(phase), _ptr(msg),
                                      _stream(stream)))
        return phase, msg

    def rlwe_phase(self, S, ct, stream=None):
        """b - a * S mod Q of every RLWE ciphertext [B, 2, N] (fdfb_rlwe_phase)."""
        B = ct.shape[0]
        out = self._u64(B, self.N)
        ws = self._bytes(lib().fdfb_workspace_rlwe_phase(self.h, B))
        _keep(stream, out, ws)
        _check(lib().fdfb_rlwe_phase(self.h, _ptr(S), _ptr(ct), B, _ptr(out), _ptr(ws), _stream(stream)))
        return out

    def rlwe_encrypt(self, seed, S, msgs: torch.Tensor, first_index=0, stream=None):
        cnt = msgs.shape[0]
        out = self._u64(cnt, 2, self.N)
        ws = self._bytes(lib().fdfb_workspace_rlwe_encrypt(self.h, cnt))
        _keep(stream, out, ws)
        _check(lib().fdfb_rlwe_encrypt(self.h, C.c_uint64(seed), _ptr(S), _ptr(msgs), cnt, C.c_uint64(first_index),
                                       _ptr(out), _ptr(ws), _stream(stream)))
        return out

    def setup_lut(self, lut, t_out=None, stream=None):
        import numpy as np
        lut = np.ascontiguousarray(np.asarray(lut, dtype=np.uint64))
        t_out = self.cfg["t"] if t_out is None else t_out
        rotp = self._u64(2, self.N)
        _keep(stream, rotp)
        _check(lib().fdfb_setup_lut(self.h, lut.ctypes.data_as(C.c_void_p), t_out, _ptr(rotp), _stream(stream)))
        return rotp

    # ---------------------------------------------------------------- hot path
    def workspace_bootstrap(self, B):
        return self._bytes(lib().fdfb_workspace_bootstrap(self.h, B))

    def bootstrap_batch(self, keys, rotp, ct_in, ct_out=None, workspace=None, stream=None):
        B = ct_in.shape[0]
        ct_out = self._u64(B, self.n + 1) if ct_out is None else ct_out
        ws = self.workspace_bootstrap(B) if workspace is None else workspace
        _keep(stream, ct_out, ws)
        _check(lib().fdfb_bootstrap_batch(self.h, _ptr(keys["brk"]), _ptr(keys["bpk"]), _ptr(keys["ksk"]),
                                          _ptr(rotp), _ptr(ct_in), _ptr(ct_out), B, _ptr(ws), _stream(stream)))
        return ct_out

    def bootstrap_multi(self, keys, rotps, ct_in, workspace=None, stream=None):
        """k LUTs on the same inputs (rotps: [k, 2, N] device tensor); returns [k, B, n+1]."""
        B, k = ct_in.shape[0], rotps.shape[0]
        out = self._u64(k, B, self.n + 1)
        ws = self._bytes(lib().fdfb_workspace_bootstrap_multi(self.h, B, k)) if workspace is None else workspace
        rotps = rotps.contiguous()
        _keep(stream, out, ws, rotps)
        _check(lib().fdfb_bootstrap_multi_batch(self.h, _ptr(keys["brk"]), _ptr(keys["bpk"]), _ptr(keys["ksk"]),
                                                _ptr(rotps), k, _ptr(ct_in), _ptr(out), B, _ptr(ws),
                                                _stream(stream)))
        return out

    def bootstrap_tfhe(self, keys, rotp, ct_in, workspace=None, stream=None):
        """TFHE half-domain bootstrap with rotP_0 of rotp ([2, N] from setup_lut)."""
        B = ct_in.shape[0]
        out = self._u64(B, self.n + 1)
        ws = self.workspace_bootstrap(B) if workspace is None else workspace
        _keep(stream, out, ws)
        _check(lib().fdfb_bootstrap_tfhe_batch(self.h, _ptr(keys["brk"]), _ptr(keys["ksk"]), _ptr(rotp), _ptr(ct_in),
                                               _ptr(out), B, _ptr(ws), _stream(stream)))
        return out

    def workspace_bootstrap_shift(self, B):
        return self._bytes(lib().fdfb_workspace_bootstrap_shift(self.h, B))

    def bootstrap_shift(self, keys, pack, rotp, ct_in, workspace=None, stream=None):
        """Shift-based bootstrap: rotp is ONE plaintext polynomial [N] in [0, Q)."""
        B = ct_in.shape[0]
        out = self._u64(B, self.n + 1)
        ws = self.workspace_bootstrap_shift(B) if workspace is None else workspace
        _keep(stream, out, ws)
        _check(lib().fdfb_bootstrap_shift_batch(self.h, _ptr(keys["brk"]), _ptr(pack), _ptr(keys["ksk"]), _ptr(rotp),
                                                _ptr(ct_in), _ptr(out), B, _ptr(ws), _stream(stream)))
        return out

    def bootstrap_batch_host(self, keys, rotp, ct_in_host, ct_out_host, workspace, stream=None):
        B = ct_in_host.shape[0]
        _check(lib().fdfb_bootstrap_batch_host(self.h, _ptr(keys["brk"]), _ptr(keys["bpk"]), _ptr(keys["ksk"]),
                                               _ptr(rotp), _ptr(ct_in_host), _ptr(ct_out_host), B, _ptr(workspace),
                                               _stream(stream)))
        return ct_out_host

    def blind_rotate(self, brk, acc, abar, acc_per_ct=1, stream=None):
        _check(lib().fdfb_blind_rotate(self.h, _ptr(brk), _ptr(acc), _ptr(abar), acc.shape[0], acc_per_ct,
                                       _stream(stream)))
        return acc

    def sample_extract(self, rlwe, k, stream=None):
        B = rlwe.shape[0]
        out = self._u64(B, self.N + 1)
        _keep(stream, out)
        _check(lib().fdfb_sample_extract(self.h, _ptr(rlwe), _ptr(k), _ptr(out), B, _stream(stream)))
        return out

    def lwe_keyswitch(self, ksk, lwe, gemm=True, stream=None):
        """KeySwitch N -> n; gemm=True: int8 tensor-core GEMM path, False: CUDA-core kernel."""
        B = lwe.shape[0]
        out = self._u64(B, self.n + 1)
        ws = self._bytes(lib().fdfb_workspace_keyswitch(self.h, B)) if gemm else None
        _keep(stream, out, ws)
        _check(lib().fdfb_lwe_keyswitch(self.h, _ptr(ksk), _ptr(lwe), _ptr(out), B, _ptr(ws), _stream(stream)))
        return out

    def vector_pack(self, pack, lwe, stream=None):
        B, m = lwe.shape[0], lwe.shape[1]
        out = self._u64(B, 2, self.N)
        ws = self._bytes(lib().fdfb_workspace_vector_pack(self.h, m, B))
        _keep(stream, out, ws)
        _check(lib().fdfb_vector_pack(self.h, _ptr(pack), _ptr(lwe), m, _ptr(out), B, _ptr(ws), _stream(stream)))
        return out

    def pack(self, pack, lwe, d, stream=None):
        B = lwe.shape[0]
        out = self._u64(B, 2, self.N)
        _keep(stream, out)
        _check(lib().fdfb_pack(self.h, _ptr(pack), _ptr(lwe), _ptr(d), _ptr(out), B, _stream(stream)))
        return out

    def device_status(self, clear=True):
        """Raise FdfbError if a kernel flagged an out-of-range k / d since the last clear."""
        _check(lib().fdfb_device_status(self.h, 1 if clear else 0))

    def workspace_shift(self, B):
        return self._bytes(lib().fdfb_workspace_shift(self.h, B))

    def shift(self, pack, rlwe, d, out=None, workspace=None, stream=None):
        B = rlwe.shape[0]
        out = self._u64(B, 2, self.N) if out is None else out
        ws = self.workspace_shift(B) if workspace is None else workspace
        _keep(stream, out, ws)
        _check(lib().fdfb_shift(self.h, _ptr(pack), _ptr(rlwe), _ptr(d), _ptr(out), B, _ptr(ws), _stream(stream)))
        return out

    def permute(self, pack, rlwe, perm, out=None, stream=None):
        """Permute slots: out encrypts sum_i m_{perm[i-1]} X^{i-1} (perm: [B, N] uint32, 1-based)."""
        B = rlwe.shape[0]
        out = self._u64(B, 2, self.N) if out is None else out
        n = lib().fdfb_workspace_permute(self.h, B)
        ws = self._bytes(n) if n else None
        _keep(stream, out, ws)
        _check(lib().fdfb_permute(self.h, _ptr(pack), _ptr(rlwe), _ptr(perm), _ptr(out), B, _ptr(ws),
                                  _stream(stream)))
        return out

    def shift_streaming(self, pack, rlwe, d, out=None, stream=None):
        B = rlwe.shape[0]
        out = self._u64(B, 2, self.N) if out is None else out
        _keep(stream, out)
        _check(lib().fdfb_shift_streaming(self.h, _ptr(pack), _ptr(rlwe), _ptr(d), _ptr(out), B, _stream(stream)))
        return out

    def poly_mul(self, a, b, stream=None):
        out = torch.empty_like(a)
        ws = self._bytes(lib().fdfb_workspace_poly_mul(self.h, a.shape[0]))
        _keep(stream, out, ws)
        _check(lib().fdfb_poly_mul(self.h, _ptr(a), _ptr(b), _ptr(out), a.shape[0], _ptr(ws), _stream(stream)))
        return out

    def gemm_i8(self, A, B, stream=None):
        """D = A @ B.T exactly (int8 x int8 -> int32) on the tcgen05 kernel (fdfb_gemm_i8)."""
        M, K = A.shape
        Nc = B.shape[0]
        D = torch.empty((M, Nc), dtype=torch.int32, device=self.device)
        _keep(stream, D)
        _check(lib().fdfb_gemm_i8(self.h, _ptr(A), _ptr(B), M, Nc, K, _ptr(D), _stream(stream)))
        return D

    def cdt_table(self):
        import numpy as np
        T = C.c_int()
        _check(lib().fdfb_cdt_table(self.h, None, C.byref(T)))
        out = np.zeros(2 * T.value, dtype=np.uint64)
        _check(lib().fdfb_cdt_table(self.h, out.ctypes.data_as(C.c_void_p), C.byref(T)))
        return out
