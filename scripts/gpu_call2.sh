set -u
mkdir -p gpurun_out
timeout 300 python scripts/timeline.py bf16 > gpurun_out/timeline_bf16.txt 2>&1; echo "timeline rc=$?"
cat gpurun_out/timeline_bf16.txt
bash scripts/ncu_kernels.sh r1
