"""One blind-rotation launch at the Large configuration (for ncu --set full).

    python tools/prof_br.py [--acc 148] [--config large]
Runs fdfb_blind_rotate once on `acc` accumulators (full n-step rotation) after one
warm-up launch; the kernel is the one bench.py's step spends >90% of its time in."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_02731_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--acc", type=int, default=148)
ap.add_argument("--config", default="large")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = synth.load_config(a.config)
ctx = Context(cfg, 0)
keys = ctx.keygen(cfg["seeds"]["keys"], which=0x03)
g = torch.Generator(device="cuda").manual_seed(1)
acc = torch.randint(0, 1 << 53, (a.acc, 2, cfg["N"]), device="cuda", generator=g).to(torch.uint64)
abar = torch.randint(0, 2 * cfg["N"], (a.acc, cfg["n"]), device="cuda", generator=g).to(torch.uint32)
ctx.blind_rotate(keys["brk"], acc.clone(), abar)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(a.reps):
    x = acc.clone()
    s.record()
    ctx.blind_rotate(keys["brk"], x, abar)
    e.record()
    torch.cuda.synchronize()
    print("blind_rotate: %d accumulators x %d CMux in %.2f ms" % (a.acc, cfg["n"] * ctx.u, s.elapsed_time(e)))
