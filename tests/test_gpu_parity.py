"""GPU parity: the CUDA path (through the C-ABI binding) vs the CPU oracle, bit-exact.

All arithmetic on the path is exact modular integer arithmetic, so the bar is
byte equality (no tolerance).  Keys for the hot-path parity tests are generated
by the ORACLE and imported into the device format (fdfb_key_import); the GPU
keygen is checked separately against the oracle keygen.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_02731_b200 import KEY_BPK, KEY_BRK, KEY_KSK, Context  # noqa: E402
from paper_2109_02731_b200 import KEY_PACK  # noqa: E402

DEV = torch.device("cuda", 0)


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
    # independently computed CDT tables (library: long double; oracle: 60-digit decimal) agree to a
    # few units of 2^-64: a sample differs only if its 64-bit uniform hits that gap (p < 2^-60)
    from oracle.cdt import cdt_table
    lib_t = [int(x) for x in ctx.cdt_table()]
    assert len(lib_t) == 38 and max(abs(a - b) for a, b in zip(lib_t, cdt_table())) <= 4
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


@pytest.mark.parametrize("name", ["tiny", "large"])
def test_lwe_keyswitch(name):
    cfg, orc, K, ctx, dk = setup(name)
    rng = np.random.default_rng(3)
    B = 37                                                      # ragged vs the 16-row tile
    c = rng.integers(0, 1 << cfg["log_q_lwe"], (B, cfg["N"] + 1), dtype=np.uint64)
    got = H(ctx.lwe_keyswitch(dk["ksk"], T(c)))
    for i in range(0, B, 1 if name == "tiny" else 12):
        assert np.array_equal(got[i], orc.keyswitch_lwe(K["ksk"], c[i]))


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
    pick = [0, B - 1]
    assert np.array_equal(got[pick], orc.bootstrap(K, rotp, cts[pick]))
