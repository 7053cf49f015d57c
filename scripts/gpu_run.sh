#!/bin/bash
# One parameterised gpurun driver (replaces the round-1 one-off s3_g*.sh scripts).
#   bash scripts/gpu_run.sh TAG STEP [STEP ...]
# steps: build | tests[:<pytest -k expr>] | smoke | bench | sweep | launches | ncu:<kernel regex>
#        | time:<python script args>        (outputs under gpurun_out/TAG_*)
TAG=$1; shift
O=gpurun_out; mkdir -p $O
DPM=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_gpu.txt 2>&1
for S in "$@"; do
  case "$S" in
    build) python -m paper_2104_12282_b200.build --force > $O/${TAG}_build.log 2>&1 || { tail -20 $O/${TAG}_build.log; exit 1; } ;;
    tests) timeout 1500 python -m pytest tests -m gpu -q -x -rs > $O/${TAG}_tests.log 2>&1; tail -4 $O/${TAG}_tests.log ;;
    tests:*) timeout 1500 python -m pytest tests -m gpu -q -rs -s -k "${S#tests:}" > $O/${TAG}_tests.log 2>&1; tail -4 $O/${TAG}_tests.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; tail -2 $O/${TAG}_smoke.log ;;
    bench) timeout 900 python bench.py > $O/${TAG}_bench.log 2>&1; tail -1 $O/${TAG}_bench.log | cut -c1-400 ;;
    benchq) timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench.log 2>&1; tail -1 $O/${TAG}_bench.log | cut -c1-400 ;;
    sweep) timeout 1200 python scripts/sweep_cfg4.py > $O/${TAG}_sweep.log 2>&1; tail -3 $O/${TAG}_sweep.log ;;
    launches) B="bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
      TOMO_NO_GRAPH=1 python $B > $O/${TAG}_plain.log 2>&1 && \
      TOMO_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -s 32000 -c 12000 --csv \
        --log-file $O/${TAG}_launches.csv python $B > $O/${TAG}_ncu_ll.log 2>&1; tail -2 $O/${TAG}_ncu_ll.log
      python scripts/launch_list_summary.py $O/${TAG}_launches.csv $O/${TAG}_launch_summary.json \
        "TOMO_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum -s 32000 -c 12000 $B" > /dev/null ;;
    report) timeout 1800 python tests/report_configs.py $O/${TAG}_configs_report.json > $O/${TAG}_report.log 2>&1; tail -2 $O/${TAG}_report.log ;;
    ncu:*) K=${S#ncu:}; TOMO_NO_GRAPH=1 python scripts/prof_step.py cfg3 12 > $O/${TAG}_plain.log 2>&1 && \
      TOMO_NO_GRAPH=1 ncu --set full --metrics $DPM --clock-control none --import-source on -k regex:"$K" -s 4 -c 2 \
        -o $O/${TAG}_prof python scripts/prof_step.py cfg3 12 > $O/${TAG}_ncu.log 2>&1; tail -2 $O/${TAG}_ncu.log ;;
    ncuall) TOMO_NO_GRAPH=1 python scripts/prof_step.py cfg3 6 > $O/${TAG}_plain.log 2>&1 && \
      TOMO_NO_GRAPH=1 ncu --set full --metrics $DPM --clock-control none --import-source on \
        -k regex:"k_op|k_sens|k_filter_t|k_oc" -c 12 -o $O/${TAG}_all python scripts/prof_step.py cfg3 6 \
        > $O/${TAG}_ncuall.log 2>&1; tail -2 $O/${TAG}_ncuall.log ;;
    checked) test -f paper_2104_12282_b200/lib/checked.so || python scripts/build_variants.py checked:TOMO_CHECKED=1 > /dev/null
      TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/checked.so timeout 1500 python -m pytest tests -m gpu -q -rs \
        -k "parity or edges or errors or twoscale or streams or schedule or cfg4_full or cfg2" > $O/${TAG}_checked.log 2>&1; tail -3 $O/${TAG}_checked.log ;;
    time:*) timeout 900 python ${S#time:} > $O/${TAG}_time.log 2>&1; tail -5 $O/${TAG}_time.log ;;
  esac
done
echo run-done
