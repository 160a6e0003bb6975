"""Per-source-line warp-stall samples of one kernel from an ncu report (--import-source on).

    python tools/ncu_lines.py REPORT.ncu-rep MANGLED_KERNEL_NAME [TOP]
    (NCU_LINES_METRIC=<source-page column>, e.g. "Instructions Executed", sums that column instead)

Compiles csrc/fdfb_api.cu to a cubin with -lineinfo (same flags as the library), maps every
SASS offset of the kernel to its (file, line) with nvdisasm -g, and sums the report's
"Warp Stall Sampling (All Samples)" per line.  The report must come from the current sources.
"""
import collections
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, fn, top=40):
    cub = "/tmp/fdfb_lines.cubin"
    subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-cubin", "-o", cub,
                    os.path.join(ROOT, "paper_2109_02731_b200", "csrc", "fdfb_api.cu")], check=True)
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(dis) if l.startswith(".text." + fn + ":")][0]
    cur, off2line = None, {}
    for l in dis[start + 1:]:
        if l.startswith(".text.") or l.startswith("//-----"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = rows[1]
    ai, wi = h.index("Address"), h.index(os.environ.get("NCU_LINES_METRIC", "Warp Stall Sampling (All Samples)"))
    base, agg, tot = None, collections.Counter(), 0
    for r in rows[2:]:
        if len(r) <= wi:
            continue
        try:
            a, w = int(r[ai], 16), int(float(r[wi] or 0))
        except ValueError:
            continue
        base = a if base is None else base
        agg[off2line.get(a - base)] += w
        tot += w
    cache = {}
    for key, v in agg.most_common(top):
        if key is None:
            print("%5.2f%%  ?" % (100 * v / tot))
            continue
        f, ln = key
        if f not in cache:
            cache[f] = open(f).read().split("\n") if os.path.exists(f) else []
        txt = cache[f][ln - 1].strip()[:90] if ln - 1 < len(cache[f]) else ""
        print("%5.2f%%  %s:%d  %s" % (100 * v / tot, os.path.basename(f), ln, txt))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
