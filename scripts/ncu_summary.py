"""Summarise an ncu report (--set full) into JSON lines for profiles/: per kernel launch the
duration, DRAM bytes, achieved occupancy, issue utilisation, FP64 pipe use, top stall reasons.
    python scripts/ncu_summary.py report.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
out = []
for v in rows[2:]:
    d = dict(zip(hdr, v))

    def f(k):
        try:
            return float(d[k])
        except (KeyError, ValueError):
            return None
    stalls = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: f(k)
              for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio") and f(k)}
    top = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
    rr, ww = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    unit_scale = 1.0
    out.append({
        "kernel": d.get("Kernel Name"), "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
        "duration_us": f("gpu__time_duration.sum"),
        "dram_read_MB": rr, "dram_write_MB": ww,
        "dram_traffic_MB": (rr or 0) + (ww or 0),
        "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "registers": f("launch__registers_per_thread"),
        "smem_per_block": f("launch__shared_mem_per_block_dynamic"),
        "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "inst_executed": f("smsp__inst_executed.sum"),
        "dfma": f("sm__sass_thread_inst_executed_op_dfma_pred_on.sum"),
        "dadd": f("sm__sass_thread_inst_executed_op_dadd_pred_on.sum"),
        "dmul": f("sm__sass_thread_inst_executed_op_dmul_pred_on.sum"),
        "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "sm_ghz": f("smsp__cycles_elapsed.avg.per_second"),
        "top_stalls_cycles_per_issue": top,
    })
js = json.dumps(out, indent=1)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(js)
print(js)
