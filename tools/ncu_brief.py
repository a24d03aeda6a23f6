"""One-screen summary of an ncu report's raw page: time, DRAM bytes, throughputs, issue
activity and the top warp-stall reasons of every captured kernel.
usage: ncu -i rep --page raw --csv > raw.csv; python tools/ncu_brief.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        # tensor cores: tcgen05 pipe busy, executed UTCHMMA bf16 ops against the dense peak (the
        # 3xBF16 split executes 3x the algorithmic FLOPs), shared-memory wavefronts of the
        # operand reads, TMEM instructions
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print("==", r[col["Kernel Name"]][:90])
    for k in KEYS:
        if k in col:
            print(f"   {k:62s} {r[col[k]]:>14s} {units[col[k]]}")
    st = [(float(r[i] or 0), h) for h, i in col.items()
          if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
    st.sort(reverse=True)
    print("   stalls/issue:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st[:6]))
