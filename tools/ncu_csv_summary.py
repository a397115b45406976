"""Summarise an `ncu --page raw --csv` export (one row per launch): key
metrics, pipe utilisation and the warp-stall breakdown per launch.  Used on
the exports tools/gpu_round.sh writes on the GPU box.

    python tools/ncu_csv_summary.py RAW.csv [max_launches]
"""
import csv
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second"]

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for r in rows[2:2 + lim]:
    print("==", r[hdr.index("Kernel Name")][:110])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:64s} {r[i]:>18s} {units[i]}")
    st = []
    for i, n in enumerate(hdr):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v >= 0.05:
                st.append((v, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    if st:
        print("   warp stalls per issued instruction: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)))
