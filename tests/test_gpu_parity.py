"""GPU parity: the CUDA path (through the C-ABI binding) vs the CPU oracle, bit-exact.

All arithmetic on the path is exact modular integer arithmetic, so the bar is
byte equality (no tolerance).  Keys for the hot-path parity tests are generated
by the ORACLE and imported into the device format (fdfb_key_import); the GPU
keygen is checked separately against the oracle keygen.
"""
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle.oracle import Oracle, num_threads  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_02731_b200 import KEY_BPK, KEY_BRK, KEY_KSK, Context  # noqa: E402
from paper_2109_02731_b200 import KEY_PACK  # noqa: E402

DEV = torch.device("cuda", 0)

# Oracle sample sizes of the full-size tests.  The oracle's cost is fixed per item (schoolbook
# products: ~400 core-seconds per Large bootstrap or per Config-4 Shift with m ~ N/2), so the
# default sizes (up to 6 Large bootstraps, 3 Shift items) keep the whole `-m gpu` suite near 10 minutes
# on a 16-core host, half of the driver's 20-minute test step;
# FDFB_PARITY_FULL=1 takes the larger samples (>= 16 Large bootstraps, every forced Shift item;
# ~20 minutes; the log of such a run is kept under profiles/).
FULL = os.environ.get("FDFB_PARITY_FULL") == "1"


def per_item(fn, items, *args):
    """Run an oracle batch function over `items`: one call when there are at least as many items
    as host threads (the oracle parallelises over items), else one call per item (the oracle then
    parallelises inside the item: the ring products of an extProd, terms of VectorPack).  Scheduling only."""
    if len(items) >= num_threads():
        return fn(items, *args)
    return np.concatenate([fn(items[i:i + 1], *[a[i:i + 1] for a in args]) for i in range(len(items))])


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def H(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


_cache = {}


def setup(name, noiseless=False):
    key = (name, noiseless)
    if key not in _cache:
        cfg = synth.load_config(name)
        orc = Oracle(cfg, noiseless=noiseless)
        K = orc.keys(cfg["seeds"]["keys"])
        ctx = Context(cfg, 0, noiseless=noiseless)
        dk = {"brk": ctx.key_import(KEY_BRK, T(K["brk"].reshape(-1))),
              "bpk": ctx.key_import(KEY_BPK, T(K["bpk"].reshape(-1))),
              "ksk": ctx.key_import(KEY_KSK, T(K["ksk"].reshape(-1)))}
        _cache[key] = (cfg, orc, K, ctx, dk)
    return _cache[key]


# ----------------------------------------------------------------------------- NTT / ring
@pytest.mark.parametrize("name", ["tiny", "fhew", "large"])
def test_ntt_ring_product_matches_schoolbook(name):
    cfg = synth.load_config(name)
    orc = Oracle(cfg)
    ctx = Context(cfg, 0)
    rng = np.random.default_rng(5)
    Q, N = cfg["Q"], cfg["N"]
    a = rng.integers(0, Q, (5, N), dtype=np.uint64)
    b = rng.integers(0, Q, (5, N), dtype=np.uint64)
    a[0] = Q - 1; b[0] = Q - 1                                 # overflow canary: max operands
    a[1] = 0; a[1, N - 1] = 1; b[1] = 0; b[1, 1] = 1           # X^{N-1} * X = -1
    got = H(ctx.poly_mul(T(a), T(b)))
    for i in range(5):
        assert np.array_equal(got[i], orc.ring_mul(a[i], b[i])), i


# ----------------------------------------------------------------------------- keygen
@pytest.mark.parametrize("name", ["tiny", "large"])
def test_keygen_matches_oracle(name):
    cfg = synth.load_config(name)
    orc = Oracle(cfg)
    ctx = Context(cfg, 0)
    seed = cfg["seeds"]["keys"]
    s, S = orc.keygen_secrets(seed)
    keys = ctx.keygen(seed, which=1)
    assert np.array_equal(H(keys["s"]), s) and np.array_equal(H(keys["S"]), S)
    # independently computed CDT tables (library: data from tools/gen_cdt_table.py, exact binary
    # fixed point with a verified floor margin; oracle: 60-digit decimal) are equal
    from oracle.cdt import cdt_table
    lib_t = [int(x) for x in ctx.cdt_table()]
    assert len(lib_t) == 38 and lib_t == cdt_table()
    rng = np.random.default_rng(1)
    u, ell = orc.u, cfg["ell_rgsw"]
    n_brk = cfg["n"] * u * 2 * ell
    idx = np.unique(np.concatenate([[0, n_brk - 1], rng.integers(0, n_brk, 6)]))
    got = H(ctx.keygen_canonical(seed, KEY_BRK, keys["s"], keys["S"], idx))
    if name == "tiny":
        full = orc.brk(seed, s, S).reshape(-1, 2, cfg["N"])
        for r, i in enumerate(idx):
            assert np.array_equal(got[r].reshape(2, -1), full[i])
        bpk = orc.bpk(seed, S).reshape(-1, 2 * cfg["N"])
        ksk = orc.ksk(seed, s, S).reshape(-1, cfg["n"] + 1)
        ib = np.arange(bpk.shape[0])
        assert np.array_equal(H(ctx.keygen_canonical(seed, KEY_BPK, keys["s"], keys["S"], ib)), bpk)
        ik = np.arange(ksk.shape[0])
        assert np.array_equal(H(ctx.keygen_canonical(seed, KEY_KSK, keys["s"], keys["S"], ik)), ksk)
    # sampled pack-key entries (PackSetup) for every config
    L = 1 << cfg["logL_pack"]
    ip = [0, 5 * cfg["ell_pack"] * L + 1, cfg["N"] * cfg["ell_pack"] * L - 1]
    gp = H(ctx.keygen_canonical(seed, KEY_PACK, keys["s"], keys["S"], ip))
    for r, flat in enumerate(ip):
        k0 = flat % L; j = (flat // L) % cfg["ell_pack"]; i = flat // (L * cfg["ell_pack"])
        assert np.array_equal(gp[r].reshape(2, -1), orc.pack_key_entry(seed, S, i, j, k0))


def test_full_keygen_bootstraps_like_imported_keys():
    cfg, orc, K, ctx, dk = setup("tiny")
    keys = ctx.keygen(cfg["seeds"]["keys"])
    for name in ("brk", "bpk", "ksk"):
        assert torch.equal(keys[name], dk[name]), name


@pytest.mark.parametrize("name", ["tiny", "fhew", "large"])
def test_brk_export_is_canonical(name):
    """fdfb_key_export(BRK): inverse RNS NTTs + CRT of the device key give back the canonical
    BRKeyGen rows that were imported, for 1-, 2- and 3-prime contexts."""
    cfg, orc, K, ctx, dk = setup(name)
    got = H(ctx.key_export(KEY_BRK, dk["brk"]))
    assert np.array_equal(got, K["brk"].reshape(-1))


# ----------------------------------------------------------------------------- primitives
def test_sample_extract_all_k():
    cfg, orc, K, ctx, dk = setup("tiny")
    rng = np.random.default_rng(2)
    N = cfg["N"]
    ct = rng.integers(0, cfg["Q"], (N, 2, N), dtype=np.uint64)
    ks = np.arange(1, N + 1, dtype=np.uint32)
    got = H(ctx.sample_extract(T(ct), T(ks)))
    for i, k in enumerate(ks):
        assert np.array_equal(got[i], orc.sample_extract(ct[i], int(k)))


def test_sample_extract_invalid_k_flagged():
    """k outside 1..N: a zero row and the device status flag (include/fdfb.h), valid rows exact."""
    cfg, orc, K, ctx, dk = setup("tiny")
    N = cfg["N"]
    ct = np.random.default_rng(6).integers(0, cfg["Q"], (4, 2, N), dtype=np.uint64)
    ks = np.array([0, 1, N + 1, N], dtype=np.uint32)
    got = H(ctx.sample_extract(T(ct), T(ks)))
    with pytest.raises(Exception):
        ctx.device_status()
    assert not got[0].any() and not got[2].any()
    assert np.array_equal(got[1], orc.sample_extract(ct[1], 1))
    assert np.array_equal(got[3], orc.sample_extract(ct[3], N))
    ctx.device_status()                                            # cleared by the read


@pytest.mark.parametrize("name", ["tiny", "large"])
def test_decryption_helpers_match_oracle(name):
    """fdfb_lwe_decrypt (phase and decoded message) and fdfb_rlwe_phase vs the oracle's phase
    definitions and decode rounding (1725)."""
    cfg, orc, K, ctx, dk = setup(name)
    rng = np.random.default_rng(12)
    B, t = 37, cfg["t"]
    cts = rng.integers(0, 1 << cfg["log_q_lwe"], (B, cfg["n"] + 1), dtype=np.uint64)
    ph, msg = ctx.lwe_decrypt(T(K["s"]), T(cts), t=t)
    ph, msg = H(ph), H(msg)
    for c in range(B):
        want = orc.lwe_phase(K["s"], cts[c])
        assert int(ph[c]) == want and int(msg[c]) == orc.decode(want, 1 << cfg["log_q_lwe"], t), c
    rl = rng.integers(0, cfg["Q"], (3, 2, cfg["N"]), dtype=np.uint64)
    got = H(ctx.rlwe_phase(T(K["S"]), T(rl)))
    for c in range(3):
        assert np.array_equal(got[c], orc.rlwe_phase(K["S"], rl[c])), c


@pytest.mark.parametrize("name", ["tiny", "large"])
def test_lwe_keyswitch(name):
    cfg, orc, K, ctx, dk = setup(name)
    rng = np.random.default_rng(3)
    B = 37                                                      # ragged vs the 16-row tile
    c = rng.integers(0, 1 << cfg["log_q_lwe"], (B, cfg["N"] + 1), dtype=np.uint64)
    got = H(ctx.lwe_keyswitch(dk["ksk"], T(c)))                 # int8 tensor-core GEMM path
    for i in range(0, B, 1 if name == "tiny" else 12):
        assert np.array_equal(got[i], orc.keyswitch_lwe(K["ksk"], c[i]))
    assert np.array_equal(H(ctx.lwe_keyswitch(dk["ksk"], T(c), gemm=False)), got)   # CUDA-core kernel


@pytest.mark.parametrize("name,count", [("tiny", 1), ("tiny", 7), ("fhew", 3)])
def test_blind_rotate_matches_oracle(name, count):
    cfg, orc, K, ctx, dk = setup(name)
    rng = np.random.default_rng(4)
    N, n = cfg["N"], cfg["n"]
    acc = rng.integers(0, cfg["Q"], (count, 2, N), dtype=np.uint64)
    abar = rng.integers(0, 2 * N, (count, n)).astype(np.uint32)
    abar[0, :3] = 0                                              # zero rotations (d = 0)
    got = H(ctx.blind_rotate(dk["brk"], T(acc), T(abar)))
    for i in range(count):
        steps = n if name == "tiny" else 40
        if steps == n:
            ref = orc.blind_rotate(K["brk"], acc[i], abar[i])
            assert np.array_equal(got[i], ref), i
    if name == "fhew":   # truncated run: GPU with only the first 40 coefficients nonzero
        a2 = abar.copy(); a2[:, 40:] = 0
        got2 = H(ctx.blind_rotate(dk["brk"], T(acc), T(a2)))
        ref = orc.blind_rotate(K["brk"], acc[0], a2[0], n_steps=40)
        # steps with abar = 0 leave acc unchanged exactly, so the truncated oracle run is the full result
        assert np.array_equal(got2[0], ref)


@pytest.mark.parametrize("logL,ell", [(5, 6), (18, 2), (27, 1)])
def test_blind_rotate_generic_gadgets(logL, ell):
    """Gadgets outside the kernel's packed-digit form (logL > 16 or ell > 4: the u64 digit path)
    and a single digit (odd ell), Tiny ring with ternary u, bit-exact with the oracle."""
    cfg = dict(synth.load_config("tiny"), logL_rgsw=logL, ell_rgsw=ell, lwe_key="ternary", n=8,
               name="tiny_g%d" % logL)
    orc = Oracle(cfg)
    K = orc.keys(cfg["seeds"]["keys"])
    ctx = Context(cfg, 0)
    brk = ctx.key_import(KEY_BRK, T(K["brk"].reshape(-1)))
    rng = np.random.default_rng(logL)
    N, n = cfg["N"], cfg["n"]
    acc = rng.integers(0, cfg["Q"], (3, 2, N), dtype=np.uint64)
    abar = rng.integers(0, 2 * N, (3, n)).astype(np.uint32)
    got = H(ctx.blind_rotate(brk, T(acc), T(abar)))
    for i in range(3):
        assert np.array_equal(got[i], orc.blind_rotate(K["brk"], acc[i], abar[i])), i


@pytest.mark.parametrize("name", ["fhew", "large", "shift512"])
def test_blind_rotate_cluster_path_equals_batched_kernel(name, monkeypatch):
    """The small-batch cluster kernel (one RNS prime per CTA, CRT terms combined through
    distributed shared memory) gives the batched kernel's bytes; both are pinned to the oracle
    elsewhere (the FHEW-like parity tests run on the cluster path)."""
    cfg = SHIFT512 if name == "shift512" else synth.load_config(name)   # N = 512 with 3 primes
    outs = []
    for mode in ("0", "2", "3"):                                    # batched, clusters of NP, of 2 NP
        monkeypatch.setenv("FDFB_BR_CLUSTER", mode)
        ctx = Context(cfg, 0)
        keys = ctx.keygen(cfg["seeds"]["keys"], which=0x03)
        g = torch.Generator(device="cuda").manual_seed(3)
        acc = torch.randint(0, cfg["Q"], (5, 2, cfg["N"]), device="cuda", generator=g).to(torch.uint64)
        abar = torch.randint(0, 2 * cfg["N"], (5, cfg["n"]), device="cuda", generator=g).to(torch.uint32)
        outs.append(H(ctx.blind_rotate(keys["brk"], acc, abar)))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


# ----------------------------------------------------------------------------- bootstrap
@pytest.mark.parametrize("B", [1, 5, 16])
def test_bootstrap_tiny_bit_exact(B):
    cfg, orc, K, ctx, dk = setup("tiny")
    f = synth.lut(cfg)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    rot = ctx.setup_lut(f)
    assert np.array_equal(H(rot), np.stack(rotp))
    msgs = synth.messages(cfg, B, seed=100 + B)
    cts = orc.lwe_encrypt(200 + B, K["s"], msgs)
    got = H(ctx.bootstrap_batch(dk, rot, T(cts)))
    assert np.array_equal(got, orc.bootstrap(K, rotp, cts))


def test_bootstrap_noiseless_full_domain_tiny():
    cfg, orc, K, ctx, dk = setup("tiny", noiseless=True)
    for seed in (1, 2):
        f = synth.lut(cfg, seed=seed)
        rot = ctx.setup_lut(f)
        msgs = np.arange(cfg["t"], dtype=np.uint64)
        cts = orc.lwe_encrypt(7, K["s"], msgs, exact=True)
        got = H(ctx.bootstrap_batch(dk, rot, T(cts)))
        dec = [orc.decode(orc.lwe_phase(K["s"], c), orc.q_lwe, orc.t) for c in got]
        assert dec == [int(f[m]) for m in msgs]
        rotp = orc.setup_polynomial(orc.bootsmap(f))
        assert np.array_equal(got[:4], orc.bootstrap(K, rotp, cts[:4]))


@pytest.mark.slow
def test_bootstrap_fhew_sampled():
    cfg, orc, K, ctx, dk = setup("fhew")
    f = synth.lut(cfg)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    B = cfg["batch"]
    msgs = synth.messages(cfg, B)
    cts = orc.lwe_encrypt(cfg["seeds"]["err"], K["s"], msgs)
    got = H(ctx.bootstrap_batch(dk, ctx.setup_lut(f), T(cts)))
    # seeded random subsample (the oracle runs the items in parallel over the host cores)
    pick = np.sort(np.random.default_rng(101).choice(B, 32, replace=False))
    ref = orc.bootstrap(K, rotp, cts[pick])
    for r, i in enumerate(pick):
        assert np.array_equal(got[i], ref[r]), int(i)


# ----------------------------------------------------------------------------- Pack / VectorPack / Shift
SHIFT512 = {  # mid-size Shift case on the BIN (L_pK = 2, ell = 54) path at 54-bit Q
    "name": "shift512", "N": 512, "n": 64, "Q": 18014398509404161, "log_q_lwe": 52, "lwe_key": "ternary",
    "rlwe_key": "ternary", "logL_rgsw": 14, "ell_rgsw": 4, "logL_boot": 8, "ell_boot": 7, "logL_pk": 14,
    "ell_pk": 4, "logL_ks": 4, "ell_ks": 13, "logL_pack": 1, "ell_pack": 54, "t": 256, "sigma": 3.2,
    "batch": 16, "seeds": {"keys": 9001, "msgs": 9002, "lut": 9003, "err": 9004}}

_pcache = {}


def pack_setup(name):
    """Oracle PackSetup key (canonical) imported into the device format."""
    if name not in _pcache:
        cfg = SHIFT512 if name == "shift512" else synth.load_config(name)
        orc = Oracle(cfg)
        s, S = orc.keygen_secrets(cfg["seeds"]["keys"])
        pk = orc.pack_key(cfg["seeds"]["keys"], S)
        ctx = Context(cfg, 0)
        dpk = ctx.key_import(KEY_PACK, T(pk.reshape(-1)))
        _pcache[name] = (cfg, orc, s, S, pk, ctx, dpk)
    return _pcache[name]


def test_pack_key_device_format_from_keygen_equals_import():
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("tiny_shift")
    keys = ctx.keygen(cfg["seeds"]["keys"], which=0x11)
    assert np.array_equal(H(keys["S"]), S)
    assert torch.equal(keys["pack"], dpk)                       # canonical part and suffix sums
    assert np.array_equal(H(ctx.key_export(KEY_PACK, dpk)), pk.reshape(-1))


@pytest.mark.parametrize("name", ["tiny_shift", "shift512"])
def test_vector_pack_and_pack(name):
    cfg, orc, s, S, pk, ctx, dpk = pack_setup(name)
    N, Q = cfg["N"], cfg["Q"]
    rng = np.random.default_rng(21)
    for m in (1, 3, N if name == "tiny_shift" else 9):
        v = rng.integers(0, Q, (2, m, N + 1), dtype=np.uint64)
        got = H(ctx.vector_pack(dpk, T(v)))
        for b in range(2):
            assert np.array_equal(got[b], orc.vector_pack(pk, v[b])), (m, b)
    c = rng.integers(0, Q, (4, N + 1), dtype=np.uint64)
    d = np.array([1, 2, N // 2, N], dtype=np.uint32)
    got = H(ctx.pack(dpk, T(c), T(d)))
    for b in range(4):
        assert np.array_equal(got[b], orc.pack(pk, c[b], int(d[b]))), b


def test_shift_tiny_every_d_bit_exact():
    """Every d in [1, N-1] (both branches, the d = N/2 tie) on the Tiny Shift config."""
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("tiny_shift")
    N = cfg["N"]
    msg = synth.rlwe_messages(cfg, 1)
    ct = orc.rlwe_encrypt(cfg["seeds"]["err"], S, msg)[0]
    ds = np.arange(1, N, dtype=np.uint32)
    cts = np.repeat(ct[None], len(ds), axis=0)
    got = H(ctx.shift(dpk, T(cts), T(ds)))
    ctx.device_status()
    ref = orc.shift_batch(pk, cts, ds)
    assert np.array_equal(got, ref)
    for d in cfg["shift_d"]:                                    # the config's named cases decrypt to the rotation
        assert np.array_equal((orc.rlwe_phase(S, got[d - 1]) - np.roll(msg[0], d).astype(np.int64)
                               ).astype(np.int64).__abs__().max() < 2 ** 26, True)


def test_shift_bin_path_bit_exact():
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("shift512")
    N = cfg["N"]
    msg = synth.rlwe_messages(cfg, 13)
    cts = orc.rlwe_encrypt(cfg["seeds"]["err"], S, msg)
    ds = np.array([1, 2, 3, 100, 255, 256, 257, 300, 509, 510, 511, 17, 490], dtype=np.uint32)   # 13: ragged tile
    got = H(ctx.shift(dpk, T(cts), T(ds)))
    ctx.device_status()
    assert np.array_equal(got, orc.shift_batch(pk, cts, ds))


def test_shift_gemm_path_equals_streaming_kernel():
    """The two device evaluations of Shift (int8 GEMM and CUDA-core streaming) agree byte for byte."""
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("shift512")
    N = cfg["N"]
    msg = synth.rlwe_messages(cfg, 21, seed=3)
    cts = T(orc.rlwe_encrypt(9, S, msg))
    ds = T(synth.shift_amounts(cfg, 21, seed=4))
    a = H(ctx.shift(dpk, cts, ds))
    b = H(ctx.shift_streaming(dpk, cts, ds))
    assert np.array_equal(a, b)
    bad = T(np.array([0, 3, N], np.uint32))
    z = H(ctx.shift(dpk, cts[:3], bad))
    with pytest.raises(Exception):
        ctx.device_status()
    assert not z[0].any() and not z[2].any() and z[1].any()


def test_shift_out_of_range_d_flagged():
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("tiny_shift")
    N = cfg["N"]
    cts = np.zeros((3, 2, N), np.uint64)
    got = H(ctx.shift(dpk, T(cts), T(np.array([0, 5, N], np.uint32))))
    with pytest.raises(Exception):
        ctx.device_status()
    assert not got[0].any() and not got[2].any()
    ctx.device_status()                                          # cleared


# ----------------------------------------------------------------------------- full-size (bench launch configuration)
@pytest.mark.slow
def test_bootstrap_large_full_batch_sampled_bit_exact():
    """Large configuration at the bench's batch (B = 4096: the ladder launch rotates B ell_boot =
    20480 accumulators on 296 persistent CTAs, the final launch 4096): up to 6 outputs (16 with
    FDFB_PARITY_FULL=1) bit-exact with
    the oracle -- a seeded random subsample plus items whose ladder accumulators fall in the
    last, partial wave of the ladder launch (accumulators >= 296 * 69, i.e. ciphertexts >= 4085)
    and in the last wave of the final launch.  The oracle computes them in parallel over the
    host cores (schoolbook products, ~0.5 min of CPU per item per core-group)."""
    cfg, orc, K, ctx, dk = setup("large")
    f = synth.lut(cfg)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    B = cfg["batch"]
    msgs = synth.messages(cfg, B)
    cts = orc.lwe_encrypt(cfg["seeds"]["err"], K["s"], msgs)
    got = H(ctx.bootstrap_batch(dk, ctx.setup_lut(f), T(cts)))
    rng = np.random.default_rng(202)
    tail = rng.choice(np.arange(4085, B), 3, replace=False)             # last ladder wave
    rest = rng.choice(np.setdiff1d(np.arange(B), tail), 13, replace=False)
    if FULL:
        pick = np.sort(np.concatenate([tail, rest]))
        ref = per_item(lambda c: orc.bootstrap(K, rotp, c), cts[pick])
        for r, i in enumerate(pick):
            assert np.array_equal(got[i], ref[r]), int(i)
        return
    # default: up to 6 items, one oracle call each (tail and random items alternating); a slow
    # host stops after the first 3 once 180 s of oracle time are spent (40-60 s per item measured)
    order = [tail[0], rest[0], tail[1], rest[1], tail[2], rest[2]]
    t0, done = time.perf_counter(), 0
    for i in order:
        ref = orc.bootstrap(K, rotp, cts[i:i + 1])[0]
        assert np.array_equal(got[i], ref), int(i)
        done += 1
        if done >= 3 and time.perf_counter() - t0 > 180.0:
            break
    print("large full-batch parity: %d items in %.0f s" % (done, time.perf_counter() - t0))


def test_bootstrap_large_full_batch_noiseless_full_domain():
    """Property at full size: noiseless keys and mod-switch-exact inputs -> every one of the
    4096 outputs decrypts exactly to f(m) (Thm), all 256 messages."""
    cfg = synth.load_config("large")
    ctx = Context(cfg, 0, noiseless=True)
    keys = ctx.keygen(cfg["seeds"]["keys"])
    f = synth.lut(cfg, seed=77)
    B = cfg["batch"]
    msgs = np.arange(B, dtype=np.uint64) % cfg["t"]
    cts = ctx.lwe_encrypt(5, keys["s"], T(msgs), exact=True)
    out = H(ctx.bootstrap_batch(keys, ctx.setup_lut(f), cts))
    s = H(keys["s"]).astype(np.int64).astype(np.uint64)
    q = 1 << cfg["log_q_lwe"]
    ph = (out[:, 0] - (out[:, 1:] * s[None, :]).sum(axis=1)) & np.uint64(q - 1)
    dec = ((ph.astype(object) * cfg["t"] * 2 + q) // (2 * q)) % cfg["t"]
    assert [int(x) for x in dec] == [int(f[int(m)]) for m in msgs]


@pytest.mark.slow
def test_shift_config4_full_batch():
    """Shift/VectorPack configuration at the bench's batch (1024 RLWE, d ~ U[1, 2047]) with the
    oracle's PackSetup key: three items forced to d = 1023, 1024 (= N/2, the tie -> branch 1)
    and 1025 (branch 2), i.e. the largest packs m ~ N/2, plus two seeded random items; of these
    d = 1024, d = 1025 and one random item (all five with FDFB_PARITY_FULL=1) are compared
    bit-exactly with the oracle; and every output decrypts to roll(m, d) within the lemma's bound."""
    cfg = synth.load_config("shift")
    orc = Oracle(cfg)
    s, S = orc.keygen_secrets(cfg["seeds"]["keys"])
    pk = orc.pack_key(cfg["seeds"]["keys"], S)                      # ~7.25 GB, ~1.5 min on 16 threads
    ctx = Context(cfg, 0)
    dpk = ctx.key_import(KEY_PACK, T(pk.reshape(-1)))
    N, Q, B = cfg["N"], cfg["Q"], cfg["batch"]
    msg = synth.rlwe_messages(cfg, B)
    ds = synth.shift_amounts(cfg, B)
    rng = np.random.default_rng(404)
    forced = rng.choice(B, 3, replace=False)
    ds[forced] = [N // 2 - 1, N // 2, N // 2 + 1]
    others = rng.choice(np.setdiff1d(np.arange(B), forced), 2, replace=False)
    cts = orc.rlwe_encrypt(cfg["seeds"]["err"], S, msg)
    d_cts = T(cts)
    d_got = ctx.shift(dpk, d_cts, T(ds))
    got = H(d_got)
    ctx.device_status()
    # default: the tie d = N/2 (branch 1, m = N/2, the largest pack), d = N/2 + 1 (branch 2,
    # m = N/2 - 1) and one random item; FULL adds d = N/2 - 1 and a second random item
    pick = np.concatenate([forced, others]) if FULL else np.concatenate([forced[1:], others[:1]])
    ref = per_item(lambda c, d: orc.shift_batch(pk, c, d), cts[pick], ds[pick])
    for r, i in enumerate(pick):
        assert np.array_equal(got[i], ref[r]), (int(i), int(ds[i]))
    # every output decrypts to roll(m, d): phases by fdfb_rlwe_phase (itself checked against the
    # oracle's phase at this ring in test_decryption_helpers_match_oracle[large]); the first four
    # items also by a plain numpy phase, which must agree with it
    Qu = np.uint64(Q)
    ph_all = H(ctx.rlwe_phase(T(S), d_got))
    for c in range(4):
        ph = got[c, 0].copy()
        a = got[c, 1]
        for i in np.nonzero(S)[0]:
            r = np.concatenate([(Qu - a[N - i:]) % Qu, a[:N - i]]) if i else a.copy()
            if S[i] < 0:
                r = (Qu - r) % Qu
            ph = np.where(ph >= r, ph - r, ph + Qu - r)
        assert np.array_equal(ph, ph_all[c]), c
    rolled = np.stack([np.roll(msg[c], int(ds[c])) for c in range(B)])
    e = (ph_all + Qu - rolled) % Qu
    e = np.minimum(e, Qu - e)
    worst = int(e.max())
    assert worst < Q // 1024, worst


# ----------------------------------------------------------------------------- NEXT rows: multi-LUT, TFHE
@pytest.mark.parametrize("B", [1, 6])
def test_bootstrap_multi_lut_equals_single_lut_oracle(B):
    """k LUTs sharing the ladder: output kk is byte-identical to the oracle's
    single-LUT bootstrap under LUT kk (the reused acc_{c,i} are the same values)."""
    cfg, orc, K, ctx, dk = setup("tiny")
    luts = [synth.lut(cfg, seed=50 + kk) for kk in range(3)]
    rot = torch.stack([ctx.setup_lut(f) for f in luts])
    msgs = synth.messages(cfg, B, seed=300 + B)
    cts = orc.lwe_encrypt(400 + B, K["s"], msgs)
    got = H(ctx.bootstrap_multi(dk, rot, T(cts)))
    for kk, f in enumerate(luts):
        rotp = orc.setup_polynomial(orc.bootsmap(f))
        assert np.array_equal(got[kk], orc.bootstrap(K, rotp, cts)), kk


def test_bootstrap_multi_lut_k1_and_ragged():
    """k = 1 is the single-LUT bootstrap; k = 5 on a ragged batch of 3 matches per LUT."""
    cfg, orc, K, ctx, dk = setup("tiny")
    msgs = synth.messages(cfg, 3, seed=41)
    cts = T(orc.lwe_encrypt(42, K["s"], msgs))
    luts = [synth.lut(cfg, seed=70 + kk) for kk in range(5)]
    rot = torch.stack([ctx.setup_lut(f) for f in luts])
    one = H(ctx.bootstrap_multi(dk, rot[:1], cts))
    assert np.array_equal(one[0], H(ctx.bootstrap_batch(dk, rot[0], cts)))
    five = H(ctx.bootstrap_multi(dk, rot, cts))
    for kk in range(5):
        assert np.array_equal(five[kk], H(ctx.bootstrap_batch(dk, rot[kk], cts))), kk


def test_bootstrap_multi_lut_large_equals_single():
    cfg, orc, K, ctx, dk = setup("large")
    luts = [synth.lut(cfg, seed=60 + kk) for kk in range(2)]
    rot = torch.stack([ctx.setup_lut(f) for f in luts])
    msgs = synth.messages(cfg, 150, seed=7)
    cts = T(orc.lwe_encrypt(8, K["s"], msgs))
    got = H(ctx.bootstrap_multi(dk, rot, cts))
    for kk in range(2):
        assert np.array_equal(got[kk], H(ctx.bootstrap_batch(dk, rot[kk], cts))), kk


@pytest.mark.parametrize("name,B", [("tiny", 5), ("fhew", 2)])
def test_bootstrap_tfhe_bit_exact(name, B):
    cfg, orc, K, ctx, dk = setup(name)
    f = synth.lut(cfg, seed=9)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    rot = ctx.setup_lut(f)
    msgs = synth.messages(cfg, B, seed=11)
    cts = orc.lwe_encrypt(12, K["s"], msgs)
    got = H(ctx.bootstrap_tfhe(dk, rot, T(cts)))
    assert np.array_equal(got, orc.bootstrap_tfhe(K, rotp[0], cts))


@pytest.mark.slow
def test_bootstrap_tfhe_large_sampled_bit_exact():
    """TFHE bootstrap at the Large set (one blind rotation of 2048 CMux steps) for a batch of 300
    (the batched kernel), 16 sampled outputs (seeded, incl. the last) bit-exact with the oracle; and the same inputs at
    B = 3 (the small-batch cluster path) give the same bytes."""
    cfg, orc, K, ctx, dk = setup("large")
    f = synth.lut(cfg, seed=19)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    rot = ctx.setup_lut(f)
    msgs = synth.messages(cfg, 300, seed=20)
    cts = orc.lwe_encrypt(21, K["s"], msgs)
    got = H(ctx.bootstrap_tfhe(dk, rot, T(cts)))
    small = H(ctx.bootstrap_tfhe(dk, rot, T(cts[:3])))
    assert np.array_equal(small, got[:3])
    pick = np.sort(np.concatenate([[299], np.random.default_rng(303).choice(299, 15, replace=False)]))
    ref = orc.bootstrap_tfhe(K, rotp[0], cts[pick])
    for r, i in enumerate(pick):
        assert np.array_equal(got[i], ref[r]), int(i)


def test_bootstrap_tfhe_negacyclic_contrast_large():
    """Noiseless keys, mod-switch-exact inputs, Large: TFHE returns F(m) on the lower half and
    -F(m - t/2) on the upper half, FDFB returns F(m) everywhere (SPEC.md acceptance 2)."""
    cfg = synth.load_config("large")
    ctx = Context(cfg, 0, noiseless=True)
    keys = ctx.keygen(cfg["seeds"]["keys"])
    f = synth.lut(cfg, seed=13)
    t = cfg["t"]
    msgs = np.arange(t, dtype=np.uint64)
    cts = ctx.lwe_encrypt(14, keys["s"], T(msgs), exact=True)
    rot = ctx.setup_lut(f)
    s = H(keys["s"]).astype(np.int64).astype(np.uint64)
    q = 1 << cfg["log_q_lwe"]

    def dec(out):
        ph = (out[:, 0] - (out[:, 1:] * s[None, :]).sum(axis=1)) & np.uint64(q - 1)
        return [int(x) for x in ((ph.astype(object) * t * 2 + q) // (2 * q)) % t]

    tf, fd = dec(H(ctx.bootstrap_tfhe(keys, rot, cts))), dec(H(ctx.bootstrap_batch(keys, rot, cts)))
    assert fd == [int(f[m]) for m in range(t)]
    assert tf == [int(f[m]) if m < t // 2 else (-int(f[m - t // 2])) % t for m in range(t)]


# ----------------------------------------------------------------------------- Permute (NEXT #3)
@pytest.mark.parametrize("name", ["tiny_shift", "shift512"])
def test_permute_bit_exact(name):
    """Permute (reading P1) on the definition path (L = 512) and the int8 GEMM
    path (L = 2, ell = 54): identity, a transposition, a rotation and random permutations."""
    cfg, orc, s, S, pk, ctx, dpk = pack_setup(name)
    N = cfg["N"]
    rng = np.random.default_rng(23)
    perms = [np.arange(1, N + 1), np.roll(np.arange(1, N + 1), 5)]
    p2 = np.arange(1, N + 1); p2[[0, N - 1]] = p2[[N - 1, 0]]
    perms += [p2, rng.permutation(N) + 1, rng.permutation(N) + 1]
    perms = np.stack(perms).astype(np.uint32)
    msg = synth.rlwe_messages(cfg, len(perms), seed=24)
    cts = orc.rlwe_encrypt(25, S, msg)
    got = H(ctx.permute(dpk, T(cts), T(perms)))
    ctx.device_status()
    assert np.array_equal(got, orc.permute_batch(pk, cts, perms))
    ph = orc.rlwe_phase(S, got[3])                       # decrypts to the permuted message
    e = (ph.astype(object) - msg[3][perms[3] - 1].astype(object)) % cfg["Q"]
    assert max(min(int(x), cfg["Q"] - int(x)) for x in e) < cfg["Q"] // 1024


def test_permute_invalid_entries_are_fixed_points():
    """A permutation entry outside 1..N is treated as a fixed point and raises the status flag
    (include/fdfb.h): invalid entries on slots that are fixed points of a permutation give that
    permutation's result, exactly as the oracle computes it."""
    cfg, orc, s, S, pk, ctx, dpk = pack_setup("shift512")
    N = cfg["N"]
    rng = np.random.default_rng(27)
    perm = (rng.permutation(N) + 1).astype(np.uint32)
    for slot in (4, 101):                                           # make slots 4 and 101 fixed points
        other = int(np.nonzero(perm == slot)[0][0])
        perm[other], perm[slot - 1] = perm[slot - 1], slot
    bad = perm.copy()
    bad[[3, 100]] = [0, N + 7]                                      # invalid entries -> treated as fixed
    ref_perm = perm
    msg = synth.rlwe_messages(cfg, 1, seed=28)
    ct = orc.rlwe_encrypt(29, S, msg)
    got = H(ctx.permute(dpk, T(ct), T(bad[None])))
    with pytest.raises(Exception):
        ctx.device_status()
    assert np.array_equal(got[0], orc.permute(pk, ct[0], ref_perm))


@pytest.mark.parametrize("name", ["tiny", "fhew"])
def test_bootstrap_cuda_graph_capture_and_replay(name):
    """The bootstrap path is stream-ordered with no host synchronisation, so it can be captured
    into a CUDA graph once and replayed: replays on new inputs equal direct calls (FHEW-like at
    B = 7 runs its blind rotations on the cluster kernel and its key switches as cuBLASLt GEMMs)."""
    cfg, orc, K, ctx, dk = setup(name)
    rot = ctx.setup_lut(synth.lut(cfg, seed=81))
    a = T(orc.lwe_encrypt(82, K["s"], synth.messages(cfg, 7, seed=83)))
    b = T(orc.lwe_encrypt(84, K["s"], synth.messages(cfg, 7, seed=85)))
    ws = ctx.workspace_bootstrap(7)
    static_in = a.clone()
    out = torch.empty_like(a)
    ctx.bootstrap_batch(dk, rot, static_in, out, ws)              # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.bootstrap_batch(dk, rot, static_in, out, ws)
    for x in (a, b):
        static_in.copy_(x)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ctx.bootstrap_batch(dk, rot, x))


def test_bootstrap_host_buffers_api():
    """fdfb_bootstrap_batch_host (pinned host in/out, copies on the stream) == the device call."""
    cfg, orc, K, ctx, dk = setup("tiny")
    f = synth.lut(cfg, seed=71)
    rot = ctx.setup_lut(f)
    cts = orc.lwe_encrypt(72, K["s"], synth.messages(cfg, 9, seed=73))
    h_in = torch.from_numpy(cts).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    ctx.bootstrap_batch_host(dk, rot, h_in, h_out, ctx.workspace_bootstrap(9))
    assert np.array_equal(h_out.numpy(), H(ctx.bootstrap_batch(dk, rot, T(cts))))


# ----------------------------------------------------------------------------- shift-based bootstrap (NEXT #4)
SHIFTBOOT256 = {  # shift-based bootstrap on the int8-GEMM Shift path (L_pK = 2), ternary u, small n
    "name": "shiftboot256", "N": 256, "n": 16, "Q": 134215681, "log_q_lwe": 32, "lwe_key": "ternary",
    "rlwe_key": "ternary", "logL_rgsw": 9, "ell_rgsw": 3, "logL_boot": 9, "ell_boot": 3, "logL_pk": 9,
    "ell_pk": 3, "logL_ks": 4, "ell_ks": 8, "logL_pack": 1, "ell_pack": 27, "t": 16, "sigma": 3.2,
    "batch": 5, "seeds": {"keys": 9101, "msgs": 9102, "lut": 9103, "err": 9104}}


def _shiftboot_inputs(cfg, orc, s, B, seed):
    """Random-phase LWE inputs (a few with zero mask coefficients: the identity steps of
    reading S1) and a random plaintext rotP = Delta g, g: Z_N -> Z_t."""
    rng = np.random.default_rng(seed)
    N, q, t, Q = cfg["N"], 1 << cfg["log_q_lwe"], cfg["t"], cfg["Q"]
    cts = orc.lwe_encrypt(seed, s, rng.integers(0, t, B).astype(np.uint64))
    cts[:, 0] = (cts[:, 0] + rng.integers(0, q, B, dtype=np.uint64)) % np.uint64(q)
    cts[0, 1:5] = 0
    if B > 1:
        cts[1, 1:] = np.uint64(q // N) * np.uint64(N - 1)        # every a~_i = N - 1
    g = rng.integers(0, t, N)
    delta = (2 * Q + t) // (2 * t)
    rotp = np.array([(delta * int(v)) % Q for v in g], np.uint64)
    return cts, g, rotp


@pytest.mark.parametrize("name,B", [("tiny_shift", 3), ("shiftboot256", 5)])
def test_bootstrap_shift_bit_exact(name, B):
    """Shift-based bootstrap bit-exact with the oracle: the streaming Shift
    (L_pK = 512, binary u) and the int8-GEMM Shift (L_pK = 2, ternary u, ragged batch)."""
    cfg = SHIFTBOOT256 if name == "shiftboot256" else synth.load_config(name)
    orc = Oracle(cfg)
    K = orc.keys(cfg["seeds"]["keys"])
    pk = orc.pack_key(cfg["seeds"]["keys"], K["S"])
    ctx = Context(cfg, 0)
    dk = {"brk": ctx.key_import(KEY_BRK, T(K["brk"].reshape(-1))),
          "ksk": ctx.key_import(KEY_KSK, T(K["ksk"].reshape(-1)))}
    dpk = ctx.key_import(KEY_PACK, T(pk.reshape(-1)))
    cts, g, rotp = _shiftboot_inputs(cfg, orc, K["s"], B, seed=31)
    got = H(ctx.bootstrap_shift(dk, dpk, T(rotp), T(cts)))
    ctx.device_status()
    assert np.array_equal(got, orc.bootstrap_shift(K, pk, rotp, cts))


@pytest.mark.slow
def test_bootstrap_shift_large_noisy_full_domain():
    """Shift configuration (N = 2048, n = 1024 ternary, L_pK = 2, sigma = 3.2 keys from the GPU
    keygen): every output decrypts to g((-y) mod N), y the phase of ModSwitch(ct, q, N) -- the
    full Z_N domain with no negacyclic restriction (Thm)."""
    cfg = synth.load_config("shift")
    ctx = Context(cfg, 0)
    keys = ctx.keygen(cfg["seeds"]["keys"], which=0x1B)        # s, S, brK, ksK, pack
    orc = Oracle(cfg)
    s = H(keys["s"])
    B = 24
    cts_h, g, rotp = _shiftboot_inputs(cfg, orc, s, B, seed=41)
    out = H(ctx.bootstrap_shift(keys, keys["pack"], T(rotp), T(cts_h)))
    ctx.device_status()
    N, t, q = cfg["N"], cfg["t"], 1 << cfg["log_q_lwe"]
    s64 = s.astype(np.int64)
    ms = ((cts_h.astype(object) * 2 * N + q) // (2 * q)) % N              # ModSwitch(ct, q, N)
    y = [(int(ms[c, 0]) - int(np.dot(ms[c, 1:].astype(np.int64), s64))) % N for c in range(B)]
    su = s64.astype(np.uint64)
    ph = (out[:, 0] - (out[:, 1:] * su[None, :]).sum(axis=1)) & np.uint64(q - 1)
    dec = [int(x) for x in ((ph.astype(object) * t * 2 + q) // (2 * q)) % t]
    assert dec == [int(g[(-yy) % N]) for yy in y]


# ----------------------------------------------------------------------------- empty batches
def test_empty_batches_are_noops():
    """B = 0 (empty tensors, NULL data pointers) is FDFB_OK and launches nothing on every batched
    entry point (include/fdfb.h conventions)."""
    cfg, orc, K, ctx, dk = setup("tiny")
    rot = ctx.setup_lut(synth.lut(cfg))
    e_lwe = torch.empty((0, cfg["n"] + 1), dtype=torch.uint64, device=DEV)
    e_rlwe = torch.empty((0, 2, cfg["N"]), dtype=torch.uint64, device=DEV)
    e_u32 = torch.empty(0, dtype=torch.uint32, device=DEV)
    torch.cuda.synchronize()
    n0 = ctx.launch_count()
    assert ctx.bootstrap_batch(dk, rot, e_lwe).shape == (0, cfg["n"] + 1)
    assert ctx.bootstrap_tfhe(dk, rot, e_lwe).shape[0] == 0
    assert ctx.bootstrap_multi(dk, torch.stack([rot, rot]), e_lwe).numel() == 0
    assert ctx.sample_extract(e_rlwe, e_u32).shape[0] == 0
    ctx.blind_rotate(dk["brk"], e_rlwe, e_u32)
    torch.cuda.synchronize()
    assert ctx.launch_count() == n0
    pcfg, porc, s, S, pk, pctx, dpk = pack_setup("tiny_shift")
    e_rlwe2 = torch.empty((0, 2, pcfg["N"]), dtype=torch.uint64, device=DEV)
    n1 = pctx.launch_count()
    assert pctx.shift(dpk, e_rlwe2, e_u32).shape[0] == 0
    assert pctx.permute(dpk, e_rlwe2, torch.empty((0, pcfg["N"]), dtype=torch.uint32, device=DEV)).shape[0] == 0
    torch.cuda.synchronize()
    assert pctx.launch_count() == n1
    pctx.device_status()


def test_bootstrap_two_part_split_equals_one_part_and_oracle(monkeypatch):
    """B >= 64 single-LUT batches run as two stream-overlapped halves (helper stream forked and
    joined with events): bytes equal the one-part run (FDFB_BOOT_SPLIT=0) and the oracle on a
    seeded sample, also when the split call is captured into a CUDA graph and replayed."""
    cfg, orc, K, ctx, dk = setup("tiny")
    f = synth.lut(cfg, seed=91)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    rot = ctx.setup_lut(f)
    B = 201                                                     # odd: halves of 100 and 101
    cts = orc.lwe_encrypt(92, K["s"], synth.messages(cfg, B, seed=93))
    got = H(ctx.bootstrap_batch(dk, rot, T(cts)))
    monkeypatch.setenv("FDFB_BOOT_SPLIT", "0")
    one = Context(cfg, 0)
    dk1 = {"brk": one.key_import(KEY_BRK, T(K["brk"].reshape(-1))),
           "bpk": one.key_import(KEY_BPK, T(K["bpk"].reshape(-1))),
           "ksk": one.key_import(KEY_KSK, T(K["ksk"].reshape(-1)))}
    assert np.array_equal(got, H(one.bootstrap_batch(dk1, one.setup_lut(f), T(cts))))
    pick = np.sort(np.random.default_rng(94).choice(B, 12, replace=False))
    assert np.array_equal(got[pick], orc.bootstrap(K, rotp, cts[pick]))
    ws = ctx.workspace_bootstrap(B)
    static_in = T(cts)
    out = torch.empty_like(static_in)
    ctx.bootstrap_batch(dk, rot, static_in, out, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.bootstrap_batch(dk, rot, static_in, out, ws)
    other = orc.lwe_encrypt(95, K["s"], synth.messages(cfg, B, seed=96))
    static_in.copy_(T(other))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ctx.bootstrap_batch(dk, rot, T(other)))


@pytest.mark.parametrize("pace", ["0", "8,4096,1000000", "32,160"])
def test_blind_rotate_key_pacing_changes_no_bytes(pace, monkeypatch):
    """Key-stream pacing of the persistent kernel (kernels_br.cuh pace_wait) only delays CTAs:
    with more accumulators than resident CTAs (several rounds per CTA) the bytes equal the
    oracle-checked unpaced run, also with a tight window that makes CTAs wait all the time."""
    cfg, orc, K, ctx, dk = setup("tiny")
    monkeypatch.setenv("FDFB_BR_CLUSTER", "0")
    g = torch.Generator(device="cuda").manual_seed(77)
    n_acc = 6000                                                 # > 148 x 16 resident CTAs at N = 256
    acc = torch.randint(0, cfg["Q"], (n_acc, 2, cfg["N"]), device="cuda", generator=g).to(torch.uint64)
    abar = torch.randint(0, 2 * cfg["N"], (n_acc, cfg["n"]), device="cuda", generator=g).to(torch.uint32)
    monkeypatch.setenv("FDFB_BR_PACE", "0")
    ref = H(Context(cfg, 0).blind_rotate(dk["brk"], acc.clone(), abar))
    monkeypatch.setenv("FDFB_BR_PACE", pace)
    got = H(Context(cfg, 0).blind_rotate(dk["brk"], acc.clone(), abar))
    assert np.array_equal(got, ref)
    A, ab = H(acc), H(abar)
    for i in (0, 2367, 5999):
        assert np.array_equal(got[i], orc.blind_rotate(K["brk"], A[i], ab[i]))


# the int8 key-switch GEMMs split each centred key coefficient into 7 balanced
# base-256 digits, exact for |v| <= 2^54, so validate() accepts Q < 2^55 and q_lwe <= 2^55.  This
# set sits at both limits: Q the largest prime below 2^55 with Q = 1 mod 2N, q_lwe = 2^55.
EDGE = dict(synth.load_config("tiny"), name="edge", Q=36028797018963457, log_q_lwe=55,
            logL_rgsw=14, ell_rgsw=4, logL_boot=11, ell_boot=5, logL_pk=14, ell_pk=4, logL_ks=5, ell_ks=11,
            logL_pack=12, ell_pack=5)


def test_edge_moduli_keyswitch_and_bootstrap_bit_exact():
    cfg = EDGE
    orc = Oracle(cfg)
    K = orc.keys(cfg["seeds"]["keys"])
    ctx = Context(cfg, 0)
    dk = {"brk": ctx.key_import(KEY_BRK, T(K["brk"].reshape(-1))),
          "bpk": ctx.key_import(KEY_BPK, T(K["bpk"].reshape(-1))),
          "ksk": ctx.key_import(KEY_KSK, T(K["ksk"].reshape(-1)))}
    ksk = K["ksk"].astype(object) % (1 << 55)
    cen = np.where(ksk >= (1 << 54), ksk - (1 << 55), ksk)
    assert int(np.abs(cen).max()) > (1 << 54) - (1 << 48)            # key coefficients at the digit limit
    rng = np.random.default_rng(11)
    c = rng.integers(0, 1 << 55, (21, cfg["N"] + 1), dtype=np.uint64)
    c[0, :] = (1 << 55) - 1                                         # every digit at its maximum
    got = H(ctx.lwe_keyswitch(dk["ksk"], T(c)))
    for i in range(21):
        assert np.array_equal(got[i], orc.keyswitch_lwe(K["ksk"], c[i])), i
    assert np.array_equal(H(ctx.lwe_keyswitch(dk["ksk"], T(c), gemm=False)), got)
    f = synth.lut(cfg, seed=12)
    rotp = orc.setup_polynomial(orc.bootsmap(f))
    cts = orc.lwe_encrypt(13, K["s"], synth.messages(cfg, 6, seed=14))
    got = H(ctx.bootstrap_batch(dk, ctx.setup_lut(f), T(cts)))     # BuildAcc switch with pK mod Q ~ 2^55
    assert np.array_equal(got, orc.bootstrap(K, rotp, cts))
