"""Decryption-failure measurement of the FDFB bootstrap at the Large configuration for a
choice of L_boot (the config may use L_boot = 2^11 -- 6 instead of 8 blind
rotations per bootstrap -- if >= 1e5 noisy bootstraps show no failure).

    python tools/noise_large.py --logL-boot 11 --batches 25
Noisy keys (sigma = 3.2), mod-switch-exact inputs (so input rounding is not the failure
source), a fresh random LUT per batch; every output is decrypted with s (plain phase) and
compared with f(m); the output error (phase - Delta f(m), centred mod q_lwe) is summarised."""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_02731_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--logL-boot", type=int, default=11)
ap.add_argument("--batches", type=int, default=25)
ap.add_argument("--batch", type=int, default=4096)
a = ap.parse_args()
cfg = synth.load_config("large")
bits = (cfg["Q"] - 1).bit_length()
cfg["logL_boot"] = a.logL_boot
cfg["ell_boot"] = -(-bits // a.logL_boot)
ctx = Context(cfg, 0)
keys = ctx.keygen(cfg["seeds"]["keys"] + 1000 + a.logL_boot)
s = keys["s"].cpu().numpy().astype(np.int64).astype(np.uint64)
q, t = 1 << cfg["log_q_lwe"], cfg["t"]
delta = q // t
ws = ctx.workspace_bootstrap(a.batch)
fails, n_tot, errs_max, sq = 0, 0, 0, 0.0
t0 = time.time()
for bi in range(a.batches):
    rng = np.random.default_rng(10_000 + bi)
    f = rng.integers(0, t, t, dtype=np.uint64)
    msgs = rng.integers(0, t, a.batch, dtype=np.uint64)
    cts = ctx.lwe_encrypt(20_000 + bi, keys["s"], torch.from_numpy(msgs).cuda(), exact=True)
    out = ctx.bootstrap_batch(keys, ctx.setup_lut(f), cts, workspace=ws).cpu().numpy()
    ph = (out[:, 0] - (out[:, 1:] * s[None, :]).sum(axis=1)) & np.uint64(q - 1)
    e = (ph - (f[msgs] * np.uint64(delta))) & np.uint64(q - 1)
    e = e.astype(np.int64)
    e = np.where(e >= q // 2, e - q, e)
    dec = ((ph.astype(object) * t * 2 + q) // (2 * q)) % t
    fails += int(sum(int(x) != int(y) for x, y in zip(dec, f[msgs])))
    n_tot += a.batch
    errs_max = max(errs_max, int(np.abs(e).max()))
    sq += float((e.astype(np.float64) ** 2).sum())
sd = math.sqrt(sq / n_tot)
margin = delta / 2
res = {"logL_boot": a.logL_boot, "ell_boot": cfg["ell_boot"], "bootstraps": n_tot, "failures": fails,
       "output_error_sd_log2": math.log2(sd), "max_abs_error_log2": math.log2(max(errs_max, 1)),
       "margin_log2": math.log2(margin), "margin_over_sd": margin / sd,
       "gaussian_tail_p": math.erfc(margin / sd / math.sqrt(2)), "seconds": time.time() - t0}
print(json.dumps(res), flush=True)
