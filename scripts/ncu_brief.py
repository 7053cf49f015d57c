"""Print the headline metrics and top stall reasons of every kernel in an ncu report.
    python scripts/ncu_brief.py report.ncu-rep [n_top_sass]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for v in rows[2:]:
    print("-----")
    for w in want:
        if w in h:
            print(f"  {w}: {v[h.index(w)]}")
    st = [(k, float(v[i])) for i, k in enumerate(h)
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and v[i] not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    print("  stalls/issue:", ", ".join(f"{k[34:-23]} {x:.2f}" for k, x in st[:8]))
if ntop:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hh = r[1]
    i_s, i_src = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    body = [x for x in r[2:] if len(x) > i_s and x[i_s].isdigit()]
    tot = sum(int(x[i_s]) for x in body)
    print("total stall samples", tot)
    for x in sorted(body, key=lambda x: -int(x[i_s]))[:ntop]:
        print(f"  {x[i_s]:>6} {x[0][-5:]} {x[i_src][:100]}")
