"""Pick the judged metrics out of an `ncu --page raw --csv` export (one row per launch).

    python tools/ncu_raw_pick.py gpurun_out/x_raw.csv
"""
import csv
import sys

WANT = ["Kernel Name", "launch__grid_size", "launch__block_size", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units = rows[h], rows[h + 1]
    col = {k: i for i, k in enumerate(hdr)}
    for n, r in enumerate(rows[h + 2:]):
        print(f"--- launch {n}")
        for k in WANT:
            if k in col and col[k] < len(r):
                v = r[col[k]]
                print(f"   {k} {v[:90]} {units[col[k]]}")


if __name__ == "__main__":
    main(sys.argv[1])
