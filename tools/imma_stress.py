"""Stress / timing probe of the tcgen05 int8 GEMM (fdfb_gemm_i8) over tile counts and K, each
shape in a subprocess with a timeout (a hang shows as TIMEOUT instead of blocking the box).
Usage: python tools/imma_stress.py [shape ...]   shape = M,N,K"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = ["256,224,4096", "256,16576,4096", "256,66304,1024", "512,66304,1024", "2048,28672,8192",
          "2048,28672,65536", "2048,28672,223184"]


def child(M, N, K, check):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import synth
    from paper_2109_02731_b200 import Context
    ctx = Context(synth.load_config("tiny"), 0)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    A = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
    B = torch.randint(-128, 128, (N, K), dtype=torch.int8, device=dev, generator=g)
    D = ctx.gemm_i8(A, B)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D = ctx.gemm_i8(A, B)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = None
    if check:
        r = np.random.default_rng(0).integers(0, M, 4)
        c = np.random.default_rng(1).integers(0, N, 4)
        Ah = A[r].cpu().numpy().astype(np.int64)
        Bh = B[c].cpu().numpy().astype(np.int64)
        ok = bool(np.array_equal(D[r][:, c].cpu().numpy().astype(np.int64), Ah @ Bh.T))
    ms = min(ts)
    print(json.dumps({"M": M, "N": N, "K": K, "ms": ms, "tops": 2.0 * M * N * K / ms / 1e9, "ok": ok}))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        M, N, K = map(int, sys.argv[2].split(","))
        return child(M, N, K, True)
    shapes = sys.argv[1:] or SHAPES
    for s in shapes:
        t0 = time.time()
        try:
            r = subprocess.run([sys.executable, __file__, "--child", s], capture_output=True, text=True, timeout=60)
            out = (r.stdout.strip().splitlines() or ["rc=%d %s" % (r.returncode, r.stderr[-300:])])[-1]
        except subprocess.TimeoutExpired:
            out = "TIMEOUT"
        print(s, "cg=%s" % os.environ.get("FDFB_IMMA_CG", "2"), "%.1fs" % (time.time() - t0), out, flush=True)


if __name__ == "__main__":
    main()
