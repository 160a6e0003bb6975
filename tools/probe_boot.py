"""Quick timing probe of bootstrap_batch / blind_rotate on the GPU (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2109_02731_b200 import Context

name = sys.argv[1] if len(sys.argv) > 1 else "large"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 148
cfg = synth.load_config(name)
ctx = Context(cfg, 0)
t0 = time.time()
keys = ctx.keygen(cfg["seeds"]["keys"])
torch.cuda.synchronize()
print("keygen %.2fs" % (time.time() - t0), flush=True)
msgs = torch.from_numpy(synth.messages(cfg, B)).cuda()
cts = ctx.lwe_encrypt(cfg["seeds"]["err"], keys["s"], msgs)
rot = ctx.setup_lut(synth.lut(cfg))
ws = ctx.workspace_bootstrap(B)
out = ctx.bootstrap_batch(keys, rot, cts, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); out = ctx.bootstrap_batch(keys, rot, cts, workspace=ws); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print("%s B=%d bootstrap %.1f ms  -> %.1f bootstraps/s" % (name, B, ms, B / ms * 1e3), flush=True)
# BR alone on B*ell_boot accumulators
acc = torch.zeros(B * cfg["ell_boot"], 2, cfg["N"], dtype=torch.uint64, device="cuda")
abar = torch.randint(0, 2 * cfg["N"], (B, cfg["n"]), dtype=torch.int32, device="cuda").to(torch.uint32)
ctx.blind_rotate(keys["brk"], acc, abar, acc_per_ct=cfg["ell_boot"])
e0.record(); ctx.blind_rotate(keys["brk"], acc, abar, acc_per_ct=cfg["ell_boot"]); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ncmux = B * cfg["ell_boot"] * cfg["n"] * (2 if cfg["lwe_key"] == "ternary" else 1)
print("BR %d accs: %.1f ms, %.2f us/CMux-acc, %.3e CMux/s" % (B * cfg["ell_boot"], ms, ms * 1e3 / ncmux, ncmux / ms * 1e3))
