#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list of one
# C2 generate, and `ncu --set full` captures of the top kernels.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [what...]'
# what ∈ {tests, smoke, bench, launches, full} (default: all). Outputs → gpurun_out/.
set -u
mkdir -p gpurun_out
WHAT="${*:-tests smoke bench launches full}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest rc=$?" | tee -a gpurun_out/summary.txt; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?" | tee -a gpurun_out/summary.txt; tail -2 gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.log 2>&1
      echo "bench rc=$?" | tee -a gpurun_out/summary.txt; tail -c 3000 gpurun_out/bench.log ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/launches.log 2>&1
      echo "launches rc=$?" | tee -a gpurun_out/summary.txt
      python scripts/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launches_summary.txt 2>&1
      head -30 gpurun_out/launches_summary.txt ;;
    full)
      # logits GEMM (the N=32000 launch) + HARS stage 1 + stage 2 + attention, one generate.
      timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
        -k regex:"tc_gemm|retrieve|hars_select|decoder_self_attention|cross_attention|layer_norm" \
        -s 116 -c 72 -o gpurun_out/prof_step -f python scripts/profile_step.py --steps 2 \
        > gpurun_out/full.log 2>&1
      echo "full rc=$?" | tee -a gpurun_out/summary.txt; tail -3 gpurun_out/full.log ;;
  esac
done
