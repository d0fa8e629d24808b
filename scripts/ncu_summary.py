"""Summarise an ncu --page raw --csv export: key timing, memory, occupancy and stall metrics of each kernel.
usage: ncu_summary.py raw.csv [more metric substrings...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__maximum_warps_per_active_cycle_pct", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_issue_stalled", "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "smsp__warp_issue_stalled"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
extra = sys.argv[2:]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")][:120])
    for i, h in enumerate(hdr):
        if any(h.startswith(k) for k in KEYS) or any(e in h for e in extra):
            if h.startswith("smsp__warp_issue_stalled") and not h.endswith("per_warp_active.pct"):
                continue
            print(f"  {h} = {r[i]} {units[i]}")
