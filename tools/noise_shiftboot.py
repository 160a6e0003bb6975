"""Output noise of the shift-based bootstrap at the Shift configuration
(N = 2048, n = 1024 ternary, L_pK = 2, sigma = 3.2 keys from the GPU keygen).

    python tools/noise_shiftboot.py --batches 2 --batch 1024
Random-phase inputs, rotP = Delta g for a random g: Z_N -> Z_t; every output is decrypted
with s and compared with g((-y) mod N), y the phase of ModSwitch(ct, q, N) (plain numpy);
the output error (phase - (q/t) g, centred mod q_lwe) is summarised against the decoding
margin q / (2t).  One JSON line."""
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
ap.add_argument("--batches", type=int, default=2)
ap.add_argument("--batch", type=int, default=1024)
a = ap.parse_args()
cfg = synth.load_config("shift")
ctx = Context(cfg, 0)
keys = ctx.keygen(cfg["seeds"]["keys"] + 77, which=0x1B)
s = keys["s"].cpu().numpy().astype(np.int64)
N, q, t, Q = cfg["N"], 1 << cfg["log_q_lwe"], cfg["t"], cfg["Q"]
delta_q, delta_Q = q // t, (2 * Q + t) // (2 * t)
ws = ctx.workspace_bootstrap_shift(a.batch)
fails, n_tot, emax, sq = 0, 0, 0, 0.0
t0 = time.time()
for bi in range(a.batches):
    rng = np.random.default_rng(30_000 + bi)
    g = rng.integers(0, t, N)
    rotp = torch.from_numpy(np.array([(delta_Q * int(v)) % Q for v in g], np.uint64)).cuda()
    cts = ctx.lwe_encrypt(40_000 + bi, keys["s"], torch.from_numpy(rng.integers(0, t, a.batch).astype(np.uint64)).cuda())
    off = torch.from_numpy(rng.integers(0, q, a.batch, dtype=np.uint64)).cuda()
    cts[:, 0] = (cts[:, 0].view(torch.int64) + off.view(torch.int64)).view(torch.uint64)
    cts[:, 0] = (cts[:, 0].view(torch.int64) & (q - 1)).view(torch.uint64)
    out = ctx.bootstrap_shift(keys, keys["pack"], rotp, cts, workspace=ws).cpu().numpy()
    cin = cts.cpu().numpy()
    ms = ((cin.astype(object) * 2 * N + q) // (2 * q)) % N
    y = np.array([(int(ms[c, 0]) - int(np.dot(ms[c, 1:].astype(np.int64), s))) % N for c in range(a.batch)])
    want = g[(-y) % N].astype(np.uint64)
    ph = (out[:, 0] - (out[:, 1:] * s.astype(np.uint64)[None, :]).sum(axis=1)) & np.uint64(q - 1)
    e = ((ph - want * np.uint64(delta_q)) & np.uint64(q - 1)).astype(np.int64)
    e = np.where(e >= q // 2, e - q, e)
    dec = ((ph.astype(object) * t * 2 + q) // (2 * q)) % t
    fails += int(sum(int(x) != int(w) for x, w in zip(dec, want)))
    n_tot += a.batch
    emax = max(emax, int(np.abs(e).max()))
    sq += float((e.astype(np.float64) ** 2).sum())
sd = math.sqrt(sq / n_tot)
margin = delta_q / 2
print(json.dumps({"workload": "shiftboot", "N": N, "n": cfg["n"], "L_pack": 1 << cfg["logL_pack"],
                  "bootstraps": n_tot, "failures": fails, "output_error_sd_log2": math.log2(max(sd, 1)),
                  "max_abs_error_log2": math.log2(max(emax, 1)), "margin_log2": math.log2(margin),
                  "margin_over_sd": margin / max(sd, 1), "seconds": time.time() - t0}), flush=True)
