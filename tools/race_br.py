"""Short blind rotations for compute-sanitizer (racecheck / memcheck / synccheck).

    compute-sanitizer --tool racecheck python tools/race_br.py
Large ring parameters with n = 3 (6 ternary CMux steps), 3 accumulators, plus the Tiny
configuration; the GIN (shift-based) mode for one step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2109_02731_b200 import Context  # noqa: E402

for name in ("large", "tiny"):
    cfg = dict(synth.load_config(name))
    cfg["n"] = 3
    ctx = Context(cfg, 0)
    keys = ctx.keygen(7, which=0x03)
    g = torch.Generator(device="cuda").manual_seed(1)
    acc = torch.randint(0, cfg["Q"], (3, 2, cfg["N"]), device="cuda", generator=g).to(torch.uint64)
    abar = torch.randint(0, 2 * cfg["N"], (3, cfg["n"]), device="cuda", generator=g).to(torch.uint32)
    ctx.blind_rotate(keys["brk"], acc, abar)
    torch.cuda.synchronize()
    print(name, "ok", int(acc.view(torch.int64).sum().item()) & 0xffff)
