#!/bin/bash
# Iteration check on the GPU box: all GPU tests, CUPTI timeline of one C2
# generate, bench line (PDL off / on).
set -u
mkdir -p gpurun_out
if [ -n "${PYTEST_K:-}" ]; then KARG=(-k "$PYTEST_K"); else KARG=(); fi
timeout 900 python -m pytest tests -q -m gpu -x "${KARG[@]}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/timeline.py bf16 > gpurun_out/timeline_bf16.txt 2>&1; echo "timeline rc=$?"; grep -v Warn gpurun_out/timeline_bf16.txt | grep -v warn
if [ "${BENCH:-1}" = 1 ]; then
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.log
FQ_PDL=1 timeout 600 python bench.py --no-cpu-baseline --no-micro > gpurun_out/bench_pdl.log 2>&1; echo "bench pdl rc=$?"; tail -c 400 gpurun_out/bench_pdl.log
fi
