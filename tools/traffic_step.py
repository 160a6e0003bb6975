"""DRAM traffic of one bench step, for bench.py's roofline.traffic (run it under ncu on the GPU box).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/traffic.csv python tools/traffic_step.py [--workload bootstrap]
    python tools/traffic_step.py --summarise gpurun_out/traffic.csv > profiles/r02/traffic_bootstrap.json

The program builds bench.py's workload and runs two identical steps; the summary keeps the
launches of the second step (the first warms up) and sums dram__bytes_read + dram__bytes_write
over all kernels and over the blind-rotation kernels.  ncu serialises the launches (the
bootstrap's two halves do not overlap under it), which changes timing, not bytes."""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(workload, batch):
    import torch
    import bench
    import synth
    from paper_2109_02731_b200 import Context
    cfg = synth.load_config("shift" if workload in ("shift", "permute") else "large")
    B = batch or cfg["batch"]
    ctx = Context(cfg, 0)
    W = {"bootstrap": bench.BootstrapWorkload, "shift": bench.ShiftWorkload}[workload](
        ctx, cfg, B, 0, 1, torch.device("cuda", 0), torch.cuda.current_stream())
    for _ in range(2):
        W.step()
    torch.cuda.synchronize()


def summarise(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        d = per.setdefault(int(r[iid]), {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    ids = sorted(per)
    # the two steps launch the same kernels: keep the second half (the setup launches come first)
    names = [per[i]["name"] for i in ids]
    n = len(ids)
    step = None
    for L in range(1, n // 2 + 1):                # the longest repeated suffix = one step
        if names[n - 2 * L:n - L] == names[n - L:]:
            step = L
    keep = ids[n - step:] if step else ids
    unit = 1.0
    tot = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in keep)
    br = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in keep
             if "blind_rotate" in per[i]["name"])
    print(json.dumps({"launches_per_step": len(keep), "dram_bytes_per_step": tot * unit,
                      "br_dram_bytes_per_step": br * unit, "source": os.path.basename(path),
                      "how": "ncu dram__bytes_read.sum + dram__bytes_write.sum over the launches of one "
                             "bench step (tools/traffic_step.py)"}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bootstrap")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--summarise", default=None)
    a = ap.parse_args()
    if a.summarise:
        summarise(a.summarise)
    else:
        run(a.workload, a.batch)
