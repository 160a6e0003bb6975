"""bench.py -- throughput of the FDFB hot path on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fdfb|reference] [--config large]

One step = fdfb_bootstrap_batch over one per-GPU batch of the Large configuration
(N=2048, n=1024, 54-bit Q, B=4096 LWE ciphertexts of uniform 8-bit messages, one
seeded 256-entry LUT): ModSwitch -> ell_boot+1 batched blind rotations -> SampleExt
-> BuildAcc (LWE->RLWE key switch + PubMux) -> SampleExt -> ModSwitch -> LWE key
switch.  Keys are resident (generated once on rank 0, NCCL-broadcast for N > 1);
inputs are resident in HBM when the timed region starts.  Per-GPU work is fixed
(weak scaling); value = all ranks' ciphertexts / max-over-ranks device time.

--impl reference times the CPU oracle (oracle/, test infrastructure) on this box's
host cores on a bounded sample of the same workload (rank 0 only).

Other workloads (same JSON contract; not the driver's headline): --workload multilut
(k LUTs per input), tfhe, shift, permute, shiftboot; --box runs BASELINE's Box-scale
configuration (65536 ciphertexts sharded over the ranks, strong scaling); --config
tiny / fhew times the parity-only parameter sets.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# Integer-multiply roofline: every IMAD-class
# instruction issues on the fmaheavy pipe, 16 lanes/clk per SMSP = 64 lane-slots/clk/SM
# (guide: fma pipe rt_SMSP = 2; tools/intbench.cu measures 64-70 IMAD lanes/SM/clk and
# half that for IMAD.WIDE / IMAD.HI).  Peak = 148 SMs x 64 x 1965 MHz (max SM clock).
IMAD_PER_SM_CLK = 64
# Slots per lazy 54-bit Shoup modmul a*w - umulhi(a,w')*Q as compiled for sm_100a:
# 6 IMAD.WIDE (2 slots each) + 4 IMAD (1 slot) = 16 (SASS of tools/intbench.cu k_shoup64,
# whose measured rate, 4 modmul/SM/clk at nominal clock, confirms it).
IMAD_PER_MODMUL = 16


def imad_per_modmul(cfg):
    """Slots of the cheapest direct Shoup modmul at the configuration's modulus width:
    - Q < 2^31: 4 (IMAD.HI + 2 IMAD on 32-bit words; the result in [0, 2Q) fits 32 bits);
    - 2^31 <= Q < 2^32 (FHEW-like, Q = 2^32 - 10239): 6 -- [0, 2Q) no longer fits a 32-bit word,
      so a*w - q*Q is formed in 64 bits: IMAD.HI + 2 IMAD.WIDE (2 slots each);
    - otherwise 16 (the 54-bit Shoup above)."""
    if cfg["Q"] < (1 << 31):
        return 4
    return 6 if cfg["Q"] < (1 << 32) else IMAD_PER_MODMUL
# DRAM traffic of one bench step, measured: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum`
# over every launch of one step of this workload (tools/traffic_step.py; the summary JSON is
# committed under profiles/<round>/traffic_<workload>.json and read at run time).  None if absent.
TRAFFIC_FILES = [os.path.join(ROOT, "profiles", r, "traffic_%s.json") for r in ("r02", "r01")]


def measured_traffic(workload):
    for f in TRAFFIC_FILES:
        f = f % workload
        if os.path.exists(f):
            return json.load(open(f))
    return None


def parse():
    """CLI; --workload shift times fdfb_shift on the Shift/VectorPack configuration."""
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 3; 300 for --workload shift, whose step is ~10 ms, so that the "
                         "timed region spans seconds and the clock sampler sees it)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fdfb", choices=["fdfb", "reference"])
    ap.add_argument("--config", default=None, help="configs/<name>.json (default: large / shift)")
    ap.add_argument("--workload", default="bootstrap", choices=["bootstrap", "multilut", "tfhe", "shift", "permute",
                                                                 "shiftboot"])
    ap.add_argument("--luts", type=int, default=4, help="functions per input for --workload multilut")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the config's)")
    ap.add_argument("--box", action="store_true",
                    help="Box-scale: 65536 ciphertexts in total, sharded over the ranks (strong scaling)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="end-to-end steps (default: --steps)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (GPU box); gloo only for functional tests")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = 300 if (a.workload == "shift" and a.impl != "reference") else 3
    if a.config is None:
        a.config = "shift" if a.workload in ("shift", "permute", "shiftboot") else "large"
    return a


def algorithmic_work(cfg):
    """Per-bootstrap algorithmic modmul counts."""
    N, n, ell = cfg["N"], cfg["n"], cfg["ell_rgsw"]
    u = 2 if cfg["lwe_key"] == "ternary" else 1
    logN = N.bit_length() - 1
    ntt = (N // 2) * logN
    per_cmux = (2 * ell + 2) * ntt + 2 * ell * 2 * N
    cmux_per_bs = (cfg["ell_boot"] + 1) * n * u
    return per_cmux, cmux_per_bs


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(cfg, seconds):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload.

    Sample: one blind-rotation accumulator of the configuration stepped through as
    many CMux steps as fit in ~`seconds`; the oracle's
    schoolbook ring product parallelises over the host cores (OpenMP).  Throughput is
    scaled to bootstraps/s by the CMux count of one bootstrap ((ell_boot+1)*n*u); the
    remaining ~10% of a bootstrap (BuildAcc, key switches) is not charged, so the
    figure overstates the oracle.  brK entries are uniform mod Q: the oracle's CMux
    cost does not depend on key values."""
    import numpy as np
    from oracle.oracle import Oracle, num_threads
    orc = Oracle(cfg)
    N, n, u, ell = cfg["N"], cfg["n"], orc.u, cfg["ell_rgsw"]
    rng = np.random.default_rng(7)
    acc = rng.integers(0, cfg["Q"], (2, N), dtype=np.uint64)
    t0 = time.perf_counter()
    probe_steps = 1
    brk = rng.integers(0, cfg["Q"], (probe_steps, u, 2 * ell, 2, N), dtype=np.uint64)
    abar = rng.integers(1, 2 * N, probe_steps).astype(np.uint32)
    orc.blind_rotate(brk, acc, abar, n_steps=probe_steps)
    per = (time.perf_counter() - t0) / (probe_steps * u)
    steps = max(1, min(n, int(seconds / max(per, 1e-9) / u)))
    brk = rng.integers(0, cfg["Q"], (steps, u, 2 * ell, 2, N), dtype=np.uint64)
    abar = rng.integers(1, 2 * N, steps).astype(np.uint32)
    t0 = time.perf_counter()
    passes = 0
    while True:                                # repeat (at most 8 x) until ~`seconds` of CPU work
        orc.blind_rotate(brk, acc, abar, n_steps=steps)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= 0.8 * seconds or passes >= 8:
            break
    steps *= passes
    _, cmux_per_bs = algorithmic_work(cfg)
    cmux_s = steps * u / dt
    return {"value": cmux_s / cmux_per_bs, "unit": "bootstraps/s", "cores": num_threads(), "kind": "oracle",
            "sample": "%d CMux steps (of %d per bootstrap) of one N=%d accumulator in %.1f s on %d threads; "
                      "scaled by CMux count, BuildAcc/KS not charged" % (steps * u, cmux_per_bs, N, dt,
                                                                         num_threads()),
            "seconds": dt}


def bootstrap_config(cfg, B, world, box=False):
    """The config dict of the bootstrap workload line; both arms print exactly this."""
    return {"workload": cfg["name"] + ("-box65536" if box else ""), "N": cfg["N"], "n": cfg["n"],
            "Q_bits": cfg["Q"].bit_length(), "ell_boot": cfg["ell_boot"], "per_gpu_batch": B,
            "global_batch": B * world, "parallelism": "dp%d" % world,
            "l2": "flushed between timed steps (256 MB write)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, each step a bounded sample of the bootstrap
    workload (rank 0 only; under torchrun the other ranks exit without work).  ms_per_step is
    the measured duration of one sample step; value scales the sample to bootstraps/s."""
    if rank != 0:
        return
    if world > 1:   # torchrun pins OMP_NUM_THREADS=1 per rank; rank 0 alone runs the oracle here
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import synth
    cfg = synth.load_config(args.config)
    B = args.batch or cfg["batch"]
    if args.box:
        B = 65536 // world
    vals = []
    per_step_s = max(2.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(max(0, args.warmup)):       # untimed warm-up samples (page-in, thread pool), discarded
        cpu_oracle_sample(cfg, per_step_s)
    for _ in range(max(1, args.steps)):
        vals.append(cpu_oracle_sample(cfg, per_step_s))
    v = sum(x["value"] for x in vals) / len(vals)
    step_s = sum(x["seconds"] for x in vals) / len(vals)
    cb = dict(vals[-1])
    cb["value"] = v
    cb.pop("seconds", None)
    line = {"impl": "reference", "metric": "functional bootstraps/sec (N=%d)" % cfg["N"], "value": v,
            "unit": "bootstraps/s", "n_gpus": world, "steps": len(vals), "warmup": max(0, args.warmup),
            "ms_per_step": 1000.0 * step_s, "higher_is_better": True,
            "scaling": "strong" if args.box else "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": bootstrap_config(cfg, B, world, args.box),
            "step": "one bounded oracle sample (see cpu_baseline.sample), measured; value = sample scaled "
                    "to whole bootstraps by CMux count",
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "bootstraps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
class BootstrapWorkload:
    """fdfb_bootstrap_batch over B LWE ciphertexts of the Large configuration."""
    metric = "functional bootstraps/sec (N=2048)"
    unit = "bootstraps/s"
    kclass = "blind_rotate"
    kernel = "k_blind_rotate_p<2048,3>"

    def __init__(self, ctx, cfg, B, rank, world, dev, stream):
        import torch
        import synth
        from paper_2109_02731_b200.dist import broadcast_keys, shard_range
        self.ctx, self.cfg, self.B, self.stream = ctx, cfg, B, stream
        # labels follow the configuration (the class strings name the Large set the metric is quoted on);
        # RNS primes of the blind rotation: Q itself below 2^28, else 2 (32-bit Q) or 3 (54-bit Q) primes
        npr = 1 if cfg["Q"] < (1 << 28) else (2 if cfg["Q"] < (1 << 32) else 3)
        self.metric = self.metric.replace("N=2048", "N=%d" % cfg["N"])
        self.kernel = "k_blind_rotate_p<%d,%d>" % (cfg["N"], npr)
        t0 = time.perf_counter()
        if rank == 0:
            keys = ctx.keygen(cfg["seeds"]["keys"], which=0x0F)
        else:
            keys = {"s": torch.empty(ctx.n, dtype=torch.int8, device=dev),
                    "S": torch.empty(ctx.N, dtype=torch.int8, device=dev),
                    "brk": ctx._bytes(ctx.sizes["brk"]), "bpk": ctx._bytes(ctx.sizes["bpk"]),
                    "ksk": ctx._bytes(ctx.sizes["ksk"]), "pack": None}
        torch.cuda.synchronize()
        self.keygen_s = time.perf_counter() - t0
        self.bcast_s = 0.0
        if world > 1:                           # one NCCL broadcast of every key over NVLink
            t0 = time.perf_counter()
            broadcast_keys(keys)
            torch.cuda.synchronize()
            self.bcast_s = time.perf_counter() - t0
        self.keys = keys
        self.f = synth.lut(cfg)
        self.rotp = ctx.setup_lut(self.f)
        start, count = shard_range(B * world, world, rank)
        self.msgs = synth.messages(cfg, B * world)[start:start + count]
        # global object indices: a shard encrypts exactly what one device would for the whole batch
        self.ct_in = ctx.lwe_encrypt(cfg["seeds"]["err"], keys["s"], torch.from_numpy(self.msgs.copy()).to(dev),
                                     first_index=start)
        self.ct_out = torch.empty_like(self.ct_in)
        self.ws = ctx.workspace_bootstrap(B)
        self.io_bytes = B * (ctx.n + 1) * 8
        self.key_bytes = ctx.sizes["brk"] + ctx.sizes["bpk"] + ctx.sizes["ksk"]

    def step(self):
        self.ctx.bootstrap_batch(self.keys, self.rotp, self.ct_in, self.ct_out, self.ws, stream=self.stream)

    def host_buffers(self):
        import torch
        h_in = torch.empty(tuple(self.ct_in.shape), dtype=torch.uint64, pin_memory=True)
        h_in.copy_(self.ct_in.cpu())
        return h_in, torch.empty_like(h_in).pin_memory()

    def step_host(self, h_in, h_out):
        self.ctx.bootstrap_batch_host(self.keys, self.rotp, h_in, h_out, self.ws, stream=self.stream)

    def spot_check(self):
        """Decrypt 64 outputs with s (plain phase; no oracle) and count f(m) hits."""
        import numpy as np
        cfg = self.cfg
        s_h = self.keys["s"].cpu().numpy().astype(np.int64).astype(np.uint64)
        out_h = self.ct_out[:64].cpu().numpy()
        q = 1 << cfg["log_q_lwe"]
        ph = (out_h[:, 0] - (out_h[:, 1:] * s_h[None, :]).sum(axis=1)) & np.uint64(q - 1)
        dec = ((ph.astype(object) * cfg["t"] * 2 + q) // (2 * q)) % cfg["t"]
        ok = sum(int(a) == int(b) for a, b in zip(dec, self.f[self.msgs[:64]]))
        return {"lut_spot_check": "%d/64 outputs decrypt to f(m)" % ok}

    def roofline(self, kernel_ms_per_step, ms_step):
        per_cmux, cmux_per_bs = algorithmic_work(self.cfg)
        modmul_step = per_cmux * cmux_per_bs * self.B
        imad_s = modmul_step * imad_per_modmul(self.cfg) / (kernel_ms_per_step / 1e3)
        peak = 148 * IMAD_PER_SM_CLK * 1965e6
        hbm_peak = json.load(open(PEAKS_FILE))["hbm_gbs"] if os.path.exists(PEAKS_FILE) else 6549.8
        tr = measured_traffic("bootstrap") if self.B == 4096 else None
        traffic = tr["dram_bytes_per_step"] if tr else None
        hbm_gbs = traffic / (ms_step / 1e3) / 1e9 if traffic else None
        return {"kernel": self.kernel, "bound": "alu", "achieved": imad_s / 1e12, "peak": peak / 1e12,
                "unit": "T IMAD-slots/s", "frac": imad_s / peak,
                "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": hbm_peak,
                        "frac": hbm_gbs / hbm_peak if hbm_gbs else None,
                        "basis": "measured DRAM bytes of one step (ncu) / step time vs MEASURED_PEAKS.json hbm_gbs"},
                "traffic": traffic,
                "traffic_basis": (tr["how"] + "; " + tr["source"]) if tr else "not measured for this batch",
                "algorithmic_bytes_per_step": self.B * 2 * (self.cfg["n"] + 1) * 8 + self.key_bytes,
                "modmul_per_step": modmul_step, "imad_per_modmul": imad_per_modmul(self.cfg),
                "modmul_per_s": modmul_step / (kernel_ms_per_step / 1e3),
                "peak_basis": "fmaheavy pipe: 148 SM x 64 IMAD slots/clk x 1965 MHz; "
                              "16 slots per 54-bit Shoup modmul (6 for 2^31 <= Q < 2^32, 4 for Q < 2^31)"}

    def config(self):
        return bootstrap_config(self.cfg, self.B, self.world, self.box)


class ShiftWorkload:
    """fdfb_shift over B RLWE ciphertexts of the Shift/VectorPack configuration
    (N=2048, L_pK=2, ell_pK=54), d ~ U[1, N-1] per ciphertext."""
    metric = "shifts/sec (N=2048, L_pK=2, ell_pK=54)"
    unit = "shifts/s"
    kclass = ("shift", "shift_gemm")
    kernel = "k_shift_bits + k_imma<2> (tcgen05 int8 GEMM, recombining epilogue) + k_shift_gemm_finish"

    def __init__(self, ctx, cfg, B, rank, world, dev, stream):
        import torch
        import synth
        from paper_2109_02731_b200.dist import broadcast_keys, shard_range
        self.ctx, self.cfg, self.B, self.stream = ctx, cfg, B, stream
        t0 = time.perf_counter()
        if rank == 0:
            keys = ctx.keygen(cfg["seeds"]["keys"], which=0x11)
        else:
            keys = {"s": torch.empty(ctx.n, dtype=torch.int8, device=dev),
                    "S": torch.empty(ctx.N, dtype=torch.int8, device=dev), "pack": ctx._bytes(ctx.sizes["pack"])}
        torch.cuda.synchronize()
        self.keygen_s = time.perf_counter() - t0
        self.bcast_s = 0.0
        if world > 1:
            t0 = time.perf_counter()
            broadcast_keys(keys)
            torch.cuda.synchronize()
            self.bcast_s = time.perf_counter() - t0
        self.keys = keys
        start, count = shard_range(B * world, world, rank)
        self.msg = synth.rlwe_messages(cfg, B * world)[start:start + count]
        self.d = synth.shift_amounts(cfg, B * world)[start:start + count]
        self.ct_in = ctx.rlwe_encrypt(cfg["seeds"]["err"], keys["S"], torch.from_numpy(self.msg).to(dev),
                                      first_index=start)
        self.d_dev = torch.from_numpy(self.d.astype("uint32")).to(dev)
        self.ct_out = torch.empty_like(self.ct_in)
        self.ws = ctx.workspace_shift(B)
        self.io_bytes = B * 2 * ctx.N * 8
        self.key_bytes = ctx.sizes["pack"]

    def step(self):
        self.ctx.shift(self.keys["pack"], self.ct_in, self.d_dev, self.ct_out, workspace=self.ws, stream=self.stream)

    def host_buffers(self):
        import torch
        h_in = torch.empty(tuple(self.ct_in.shape), dtype=torch.uint64, pin_memory=True)
        h_in.copy_(self.ct_in.cpu())
        return h_in, torch.empty_like(h_in).pin_memory()

    def step_host(self, h_in, h_out):
        # host-buffer end to end through the public API: H2D, shift, D2H on the stream
        import torch
        with torch.cuda.stream(self.stream):
            self.ct_in.copy_(h_in, non_blocking=True)
            self.step()
            h_out.copy_(self.ct_out, non_blocking=True)
        self.stream.synchronize()

    def spot_check(self):
        """Phase of 4 outputs (b - a*S, negacyclic, S ternary; numpy) equals roll(m, d) up to noise."""
        import numpy as np
        Q, N = self.cfg["Q"], self.cfg["N"]
        Qu = np.uint64(Q)
        S = self.keys["S"].cpu().numpy().astype(np.int64)
        out = self.ct_out[:4].cpu().numpy()
        worst = 0
        for c in range(4):
            ph = out[c, 0].copy()
            a = out[c, 1]
            for i in np.nonzero(S)[0]:          # subtract S_i X^i a (X^N = -1)
                r = np.concatenate([(Qu - a[N - i:]) % Qu, a[:N - i]]) if i else a.copy()
                if S[i] < 0:
                    r = (Qu - r) % Qu
                ph = np.where(ph >= r, ph - r, ph + Qu - r)
            e = (ph.astype(object) - np.roll(self.msg[c], int(self.d[c])).astype(object)) % Q
            worst = max(worst, max(min(int(x), Q - int(x)) for x in e))
        return {"shift_spot_check": "max |phase - roll(m, d)| over 4 outputs = 2^%.1f (Q = 2^%.1f)"
                                    % (np.log2(max(worst, 1)), np.log2(Q))}

    def roofline(self, kernel_ms_per_step, ms_step):
        # The step is one exact int8 GEMM (M = 2B bit rows, K = ell(N-1) + N + ell N terms,
        # N_out = 7 digit planes x 2N) plus two O(B K) / O(B N) kernels: tensor-bound.  Peak:
        # dense int8 = 2 x the measured bf16 GEMM rate (guide's nominal 4.5 vs 2.25 PFLOP/s ratio).
        N, ell = self.cfg["N"], self.cfg["ell_pack"]
        K = ell * (N - 1) + N + ell * N
        ops = 2.0 * (2 * self.B) * K * (7 * 2 * N)
        tops = ops / (kernel_ms_per_step / 1e3) / 1e12
        pk = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
        # the burst peak for a short timed region, the sustained (power-capped) one for a long one
        sustained = getattr(self, "timed_ms", 0) > 1000.0 and "bf16_tflops_sustained" in pk
        bf16 = pk.get("bf16_tflops_sustained" if sustained else "bf16_tflops", 1590.0)
        peak = 2 * bf16
        # the suffix-sum route is ~4 N^2 ell bit-selected modular additions per shift;
        # on CUDA cores one 64-bit modular add is >= 5 ALU lane-ops (IADD3, IADD3.X, ISETP.EX x2, SEL)
        modadds = 4.0 * N * N * ell * self.B
        alu_peak = 148 * 64 * 1965e6 / 5
        return {"kernel": self.kernel, "bound": "tensor", "achieved": tops, "peak": peak, "unit": "TOP/s (int8)",
                "frac": tops / peak, "traffic": None, "gemm": {"M": 2 * self.B, "K": K, "N": 7 * 2 * N},
                "peak_basis": "2 x MEASURED_PEAKS.json %s (int8 = 2 x bf16 nominal)"
                              % ("bf16_tflops_sustained" if sustained else "bf16_tflops"),
                "algorithmic": {"modadds_per_step": modadds, "achieved_per_s": modadds / (kernel_ms_per_step / 1e3),
                                "cuda_core_peak_per_s": alu_peak,
                                "frac": modadds / (kernel_ms_per_step / 1e3) / alu_peak,
                                "basis": "SURVEY 8(d.3) suffix-sum route (4 N^2 ell modular adds per shift) vs "
                                         "148 SM x 64 ALU lanes x 1965 MHz / 5 lane-ops per 64-bit modular add; "
                                         "> 1 means the int8 GEMM form beats any CUDA-core evaluation of it"}}

    def config(self):
        cfg = self.cfg
        return {"workload": cfg["name"], "N": cfg["N"], "ell_pack": cfg["ell_pack"], "L_pack": 1 << cfg["logL_pack"],
                "d": "U[1, N-1] per ciphertext"}


class MultiLutWorkload(BootstrapWorkload):
    """fdfb_bootstrap_multi_batch: k LUTs on the same B inputs (ladder shared);
    the unit is one function evaluation (k per input)."""
    metric = "functional bootstrap outputs/sec, k LUTs per input (N=2048)"
    unit = "function evaluations/s"

    def __init__(self, ctx, cfg, B, rank, world, dev, stream, k=4):
        import torch
        import synth
        super().__init__(ctx, cfg, B, rank, world, dev, stream)
        self.k = k
        self.fs = [synth.lut(cfg, seed=1000 + i) for i in range(k)]
        self.rotps = torch.stack([ctx.setup_lut(f) for f in self.fs])
        from paper_2109_02731_b200.fdfb import lib
        self.ws = ctx._bytes(lib().fdfb_workspace_bootstrap_multi(ctx.h, B, k))
        self.ct_out = torch.empty((k, B, ctx.n + 1), dtype=torch.uint64, device=dev)
        self.units = k
        self.io_out_bytes = k * self.io_bytes

    def step(self):
        from paper_2109_02731_b200.fdfb import _check, _ptr, _stream, lib
        c = self.ctx
        _check(lib().fdfb_bootstrap_multi_batch(c.h, _ptr(self.keys["brk"]), _ptr(self.keys["bpk"]),
                                                _ptr(self.keys["ksk"]), _ptr(self.rotps), self.k, _ptr(self.ct_in),
                                                _ptr(self.ct_out), self.B, _ptr(self.ws), _stream(self.stream)))

    def step_host(self, h_in, h_out):
        import torch
        with torch.cuda.stream(self.stream):
            self.ct_in.copy_(h_in, non_blocking=True)
            self.step()
            h_out.copy_(self.ct_out, non_blocking=True)
        self.stream.synchronize()

    def host_buffers(self):
        import torch
        h_in = torch.empty(tuple(self.ct_in.shape), dtype=torch.uint64, pin_memory=True)
        h_in.copy_(self.ct_in.cpu())
        return h_in, torch.empty(tuple(self.ct_out.shape), dtype=torch.uint64, pin_memory=True)

    def spot_check(self):
        import numpy as np
        cfg = self.cfg
        s_h = self.keys["s"].cpu().numpy().astype(np.int64).astype(np.uint64)
        q = 1 << cfg["log_q_lwe"]
        ok = 0
        for kk, f in enumerate(self.fs):
            out_h = self.ct_out[kk, :16].cpu().numpy()
            ph = (out_h[:, 0] - (out_h[:, 1:] * s_h[None, :]).sum(axis=1)) & np.uint64(q - 1)
            dec = ((ph.astype(object) * cfg["t"] * 2 + q) // (2 * q)) % cfg["t"]
            ok += sum(int(a) == int(b) for a, b in zip(dec, f[self.msgs[:16]]))
        return {"lut_spot_check": "%d/%d outputs decrypt to f_k(m)" % (ok, 16 * self.k)}

    def roofline(self, kernel_ms_per_step, ms_step):
        per_cmux, _ = algorithmic_work(self.cfg)
        n, u = self.cfg["n"], 2 if self.cfg["lwe_key"] == "ternary" else 1
        modmul_step = per_cmux * n * u * self.B * (self.cfg["ell_boot"] + self.k)   # ell_boot + k rotations
        imad_s = modmul_step * imad_per_modmul(self.cfg) / (kernel_ms_per_step / 1e3)
        peak = 148 * IMAD_PER_SM_CLK * 1965e6
        return {"kernel": self.kernel, "bound": "alu", "achieved": imad_s / 1e12, "peak": peak / 1e12,
                "unit": "T IMAD-slots/s", "frac": imad_s / peak, "traffic": None,
                "blind_rotations_per_input": self.cfg["ell_boot"] + self.k}

    def config(self):
        d = super().config()
        d["luts_per_input"] = self.k
        return d


class TfheWorkload(BootstrapWorkload):
    """fdfb_bootstrap_tfhe_batch: the half-domain TFHE bootstrap (one blind rotation)."""
    metric = "TFHE half-domain bootstraps/sec (N=2048)"
    unit = "bootstraps/s"

    def step(self):
        self.ctx.bootstrap_tfhe(self.keys, self.rotp, self.ct_in, workspace=self.ws, stream=self.stream)

    def step_host(self, h_in, h_out):
        import torch
        with torch.cuda.stream(self.stream):
            self.ct_in.copy_(h_in, non_blocking=True)
            out = self.ctx.bootstrap_tfhe(self.keys, self.rotp, self.ct_in, workspace=self.ws, stream=self.stream)
            h_out.copy_(out, non_blocking=True)
        self.stream.synchronize()
        self.ct_out = out

    def spot_check(self):
        self.ct_out = self.ctx.bootstrap_tfhe(self.keys, self.rotp, self.ct_in, workspace=self.ws, stream=self.stream)
        return {"note": "half-domain: correct for m < t/2 only (negacyclic); checked by the parity tests"}

    def roofline(self, kernel_ms_per_step, ms_step):
        per_cmux, _ = algorithmic_work(self.cfg)
        n, u = self.cfg["n"], 2 if self.cfg["lwe_key"] == "ternary" else 1
        modmul_step = per_cmux * n * u * self.B
        imad_s = modmul_step * imad_per_modmul(self.cfg) / (kernel_ms_per_step / 1e3)
        peak = 148 * IMAD_PER_SM_CLK * 1965e6
        return {"kernel": self.kernel, "bound": "alu", "achieved": imad_s / 1e12, "peak": peak / 1e12,
                "unit": "T IMAD-slots/s", "frac": imad_s / peak, "traffic": None}


class PermuteWorkload(ShiftWorkload):
    """fdfb_permute over B RLWE ciphertexts with uniformly random permutations (Shift config keys)."""
    metric = "permutes/sec (N=2048, L_pK=2, ell_pK=54)"
    unit = "permutes/s"
    kernel = "k_perm_bits + k_imma<2> (tcgen05 int8 GEMM) + k_permute_partial/reduce"

    def __init__(self, ctx, cfg, B, rank, world, dev, stream):
        import numpy as np
        import torch
        super().__init__(ctx, cfg, B, rank, world, dev, stream)
        rng = np.random.default_rng(31 + rank)
        self.perm = np.stack([rng.permutation(ctx.N) + 1 for _ in range(B)]).astype(np.uint32)
        self.perm_dev = torch.from_numpy(self.perm).to(dev)
        from paper_2109_02731_b200.fdfb import lib
        self.ws = ctx._bytes(lib().fdfb_workspace_permute(ctx.h, B))

    def step(self):
        from paper_2109_02731_b200.fdfb import _check, _ptr, _stream, lib
        c = self.ctx
        _check(lib().fdfb_permute(c.h, _ptr(self.keys["pack"]), _ptr(self.ct_in), _ptr(self.perm_dev),
                                  _ptr(self.ct_out), self.B, _ptr(self.ws), _stream(self.stream)))

    def spot_check(self):
        import numpy as np
        self.d = np.zeros(self.B, np.int64)                     # reuse the phase check with a permutation
        Q, N = self.cfg["Q"], self.cfg["N"]
        Qu = np.uint64(Q)
        S = self.keys["S"].cpu().numpy().astype(np.int64)
        out = self.ct_out[:2].cpu().numpy()
        worst = 0
        for c in range(2):
            ph = out[c, 0].copy()
            a = out[c, 1]
            for i in np.nonzero(S)[0]:
                r = np.concatenate([(Qu - a[N - i:]) % Qu, a[:N - i]]) if i else a.copy()
                if S[i] < 0:
                    r = (Qu - r) % Qu
                ph = np.where(ph >= r, ph - r, ph + Qu - r)
            e = (ph + Qu - self.msg[c][self.perm[c] - 1]) % Qu
            worst = max(worst, int(np.minimum(e, Qu - e).max()))
        return {"permute_spot_check": "max |phase - m[pi]| over 2 outputs = 2^%.1f (Q = 2^%.1f)"
                                      % (np.log2(max(worst, 1)), np.log2(Q))}

    def roofline(self, kernel_ms_per_step, ms_step):
        N, ell = self.cfg["N"], self.cfg["ell_pack"]
        ops = 2.0 * (self.B * N) * (N * ell) * (14 * N)
        tops = ops / (kernel_ms_per_step / 1e3) / 1e12
        bf16 = json.load(open(PEAKS_FILE))["bf16_tflops"] if os.path.exists(PEAKS_FILE) else 1590.0
        return {"kernel": self.kernel, "bound": "tensor", "achieved": tops, "peak": 2 * bf16,
                "unit": "TOP/s (int8)", "frac": tops / (2 * bf16), "traffic": None,
                "gemm": {"M": self.B * N, "K": N * ell, "N": 14 * N}}


class ShiftBootWorkload:
    """fdfb_bootstrap_shift_batch: the shift-based bootstrap on the Shift
    configuration -- n u = 2048 sequential steps, each one batched Shift (int8 GEMM over the
    packing key) and one CMux per ciphertext; rotP = Delta g for a seeded g: Z_N -> Z_t."""
    metric = "shift-based bootstraps/sec (N=2048, L_pK=2)"
    unit = "bootstraps/s"
    kclass = "shift_gemm"
    kernel = "k_imma<2> tcgen05 int8 GEMM (Shift inside every CMux)"

    def __init__(self, ctx, cfg, B, rank, world, dev, stream):
        import numpy as np
        import torch
        import synth
        from paper_2109_02731_b200.dist import broadcast_keys, shard_range
        self.ctx, self.cfg, self.B, self.stream = ctx, cfg, B, stream
        t0 = time.perf_counter()
        if rank == 0:
            keys = ctx.keygen(cfg["seeds"]["keys"], which=0x1B)
        else:
            keys = {"s": torch.empty(ctx.n, dtype=torch.int8, device=dev),
                    "S": torch.empty(ctx.N, dtype=torch.int8, device=dev), "brk": ctx._bytes(ctx.sizes["brk"]),
                    "bpk": None, "ksk": ctx._bytes(ctx.sizes["ksk"]), "pack": ctx._bytes(ctx.sizes["pack"])}
        torch.cuda.synchronize()
        self.keygen_s = time.perf_counter() - t0
        self.bcast_s = 0.0
        if world > 1:
            t0 = time.perf_counter()
            broadcast_keys(keys)
            torch.cuda.synchronize()
            self.bcast_s = time.perf_counter() - t0
        self.keys = keys
        N, t, Q = cfg["N"], cfg["t"], cfg["Q"]
        rng = np.random.default_rng(cfg["seeds"]["lut"])
        self.g = rng.integers(0, t, N)
        delta = (2 * Q + t) // (2 * t)
        self.rotp = torch.from_numpy(np.array([(delta * int(v)) % Q for v in self.g], np.uint64)).to(dev)
        start, count = shard_range(B * world, world, rank)
        self.msgs = synth.messages(cfg, B * world)[start:start + count]
        # global object indices: a shard encrypts exactly what one device would for the whole batch
        self.ct_in = ctx.lwe_encrypt(cfg["seeds"]["err"], keys["s"], torch.from_numpy(self.msgs.copy()).to(dev),
                                     first_index=start)
        self.ct_out = torch.empty_like(self.ct_in)
        self.ws = ctx.workspace_bootstrap_shift(B)
        self.io_bytes = B * (ctx.n + 1) * 8
        self.key_bytes = ctx.sizes["brk"] + ctx.sizes["ksk"] + ctx.sizes["pack"]

    def step(self):
        self.ct_out = self.ctx.bootstrap_shift(self.keys, self.keys["pack"], self.rotp, self.ct_in,
                                               workspace=self.ws, stream=self.stream)

    def host_buffers(self):
        import torch
        h_in = torch.empty(tuple(self.ct_in.shape), dtype=torch.uint64, pin_memory=True)
        h_in.copy_(self.ct_in.cpu())
        return h_in, torch.empty_like(h_in).pin_memory()

    def step_host(self, h_in, h_out):
        import torch
        with torch.cuda.stream(self.stream):
            self.ct_in.copy_(h_in, non_blocking=True)
            self.step()
            h_out.copy_(self.ct_out, non_blocking=True)
        self.stream.synchronize()

    def spot_check(self):
        """64 outputs decrypt to g((-y) mod N), y the phase of ModSwitch(ct, q, N) (plain numpy)."""
        import numpy as np
        cfg = self.cfg
        N, t, q = cfg["N"], cfg["t"], 1 << cfg["log_q_lwe"]
        s = self.keys["s"].cpu().numpy().astype(np.int64)
        cin = self.ct_in[:64].cpu().numpy()
        out = self.ct_out[:64].cpu().numpy()
        ms = ((cin.astype(object) * 2 * N + q) // (2 * q)) % N
        y = [(int(ms[c, 0]) - int(np.dot(ms[c, 1:].astype(np.int64), s))) % N for c in range(len(cin))]
        ph = (out[:, 0] - (out[:, 1:] * s.astype(np.uint64)[None, :]).sum(axis=1)) & np.uint64(q - 1)
        dec = ((ph.astype(object) * t * 2 + q) // (2 * q)) % t
        ok = sum(int(d) == int(self.g[(-yy) % N]) for d, yy in zip(dec, y))
        return {"lut_spot_check": "%d/%d outputs decrypt to g(-y mod N)" % (ok, len(cin))}

    def roofline(self, kernel_ms_per_step, ms_step):
        N, ell = self.cfg["N"], self.cfg["ell_pack"]
        u = 2 if self.cfg["lwe_key"] == "ternary" else 1
        K = ell * (N - 1) + N + ell * N
        ops = 2.0 * (2 * self.B) * K * (7 * 2 * N) * self.cfg["n"] * u
        tops = ops / (kernel_ms_per_step / 1e3) / 1e12
        bf16 = json.load(open(PEAKS_FILE))["bf16_tflops"] if os.path.exists(PEAKS_FILE) else 1590.0
        return {"kernel": self.kernel, "bound": "tensor", "achieved": tops, "peak": 2 * bf16,
                "unit": "TOP/s (int8)", "frac": tops / (2 * bf16), "traffic": None,
                "gemm": {"M": 2 * self.B, "K": K, "N": 7 * 2 * N, "per_step": self.cfg["n"] * u},
                "peak_basis": "2 x MEASURED_PEAKS.json bf16_tflops (int8 = 2 x bf16 nominal)"}

    def config(self):
        cfg = self.cfg
        return {"workload": cfg["name"] + "-shiftboot", "N": cfg["N"], "n": cfg["n"], "ell_pack": cfg["ell_pack"],
                "L_pack": 1 << cfg["logL_pack"], "t": cfg["t"]}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import synth
    from paper_2109_02731_b200 import Context
    from paper_2109_02731_b200.dist import max_over_ranks

    # FDFB_SHARE_DEVICE=1 maps every rank to device 0: a functional test of the multi-rank path
    # on a one-GPU box (ranks never wait on each other inside kernels); not for measurements.
    if os.environ.get("FDFB_SHARE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    cfg = synth.load_config(args.config)
    B = args.batch or cfg["batch"]
    if args.box:                               # BASELINE Box-scale: 65536 over 1/2/4/8 GPUs
        if 65536 % world:
            raise SystemExit("--box needs a world size dividing 65536")
        B = 65536 // world
    ctx = Context(cfg, local)
    stream = torch.cuda.current_stream()
    if args.workload == "multilut":
        W = MultiLutWorkload(ctx, cfg, B, rank, world, dev, stream, k=args.luts)
    else:
        W = {"bootstrap": BootstrapWorkload, "tfhe": TfheWorkload, "shift": ShiftWorkload,
             "permute": PermuteWorkload, "shiftboot": ShiftBootWorkload}[args.workload](ctx, cfg, B, rank, world, dev, stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MB > 126 MB L2
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        W.step()
    torch.cuda.synchronize()
    extra = W.spot_check() if rank == 0 else {}

    # ------------------------------------------------------------------ timed region
    kcls = W.kclass if isinstance(W.kclass, tuple) else (W.kclass,)
    ctx.timing_enable(True)
    for kc in kcls:
        ctx.timing_read(kc)
    launches0 = ctx.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.5)                            # nvidia-smi needs a moment before its first sample
    for i in range(args.steps):
        flush.zero_()                          # L2 flush between timed steps (outside the events)
        evs[i][0].record(stream)
        W.step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    launches = ctx.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in evs)
    k_ms, k_launches = 0.0, 0
    for kc in kcls:
        a_ms, a_n = ctx.timing_read(kc, union=True)     # span covered (the halves' launches overlap)
        k_ms, k_launches = k_ms + a_ms, k_launches + a_n
    ctx.timing_enable(False)
    if world > 1:
        ms = max_over_ranks(ms, device=dev)
    ms_step = ms / args.steps
    value = B * world * getattr(W, "units", 1) / (ms_step / 1e3)

    # ------------------------------------------------------------------ end to end (host buffers)
    e2e_steps = args.e2e_steps or args.steps
    h_in, h_out = W.host_buffers()
    W.step_host(h_in, h_out)                   # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_ms = 0.0
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        W.step_host(h_in, h_out)
        b.record(stream)
        b.synchronize()
        e_ms += a.elapsed_time(b)
    if world > 1:
        e_ms = max_over_ranks(e_ms, device=dev)
    e2e_value = B * world * getattr(W, "units", 1) / (e_ms / e2e_steps / 1e3)
    e2e_ok = bool(torch.equal(h_out, W.ct_out.cpu()))

    if rank == 0:
        kms_step = k_ms / args.steps
        W.timed_ms = ms
        roof = W.roofline(kms_step, ms_step)
        roof.update({"kernel_ms_per_step": kms_step, "kernel_launches": k_launches,
                     "kernel_share_of_step": kms_step / ms_step})
        W.world, W.box = world, args.box
        cfgd = W.config()
        if "per_gpu_batch" not in cfgd:
            if args.box:
                cfgd["workload"] = cfgd.get("workload", "") + "-box65536"
            cfgd.update({"per_gpu_batch": B, "global_batch": B * world, "parallelism": "dp%d" % world,
                         "l2": "flushed between timed steps (256 MB write)"})
        line = {
            "metric": W.metric, "value": value, "unit": W.unit,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if args.box else "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": cfgd, "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": W.unit, "steps": e2e_steps,
                    "h2d_bytes_per_step": W.io_bytes, "d2h_bytes_per_step": getattr(W, "io_out_bytes", W.io_bytes),
                    "matches_device_path": e2e_ok},
            "roofline": roof, "clocks": clocks,
            "keygen_s": W.keygen_s, "key_broadcast_s": W.bcast_s, "keys_resident_bytes": W.key_bytes,
        }
        line.update(extra)
        if world == 1 and not args.no_cpu_baseline and args.workload == "bootstrap":
            cb = cpu_oracle_sample(cfg, args.cpu_seconds)
            cb.pop("seconds", None)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
