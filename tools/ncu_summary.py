"""Summarise an ncu --set full report (raw page) into the numbers DESIGN.md / profiles cite."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_shared.sum",
        "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__cluster_size",
        "launch__shared_mem_per_block_dynamic"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:80])
        for i, k in enumerate(h):
            if k in KEYS or ("warp_issue_stalled" in k and k.endswith("_per_issue_active.ratio")) or \
                    (k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")):
                try:
                    if float(v[i].replace(",", "")) == 0:
                        continue
                except ValueError:
                    pass
                print("  %-75s %s %s" % (k, v[i], u[i]))


if __name__ == "__main__":
    main(sys.argv[1])
