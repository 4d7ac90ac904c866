#!/bin/bash
# End-of-round ncu evidence (exact fp32 mode = the bench headline, plus the
# fp16 output layer): launch list of one C2 generate, the DRAM traffic of one
# decode step's 37 GEMM launches (CTA-pair and split-K kernels), and
# `--set full` captures of one steady-state (step 10) launch of each hot
# kernel. Usage: bash scripts/ncu_round2b.sh <tag>
set -u
T=${1:-r2b}
P=${PREC:-fp32}
mkdir -p gpurun_out
cap() {  # name regex skip [precision]
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k regex:"$2" -s "$3" -c 1 -o gpurun_out/${T}_$1 -f \
    python scripts/profile_step.py --precision ${4:-$P} --steps 40 > gpurun_out/${T}_$1.log 2>&1
  echo "$1 rc=$?"
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${T}_launches.csv python scripts/profile_step.py --precision $P > /dev/null 2>&1
echo "launches rc=$?"
# one decode step's GEMMs: skip the 25 encoder / cross-K/V GEMMs + 10 steps x 37
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,launch__grid_size \
  --clock-control none --profile-from-start off -k regex:gemm --csv \
  -s 395 -c 37 python scripts/profile_step.py --precision $P --steps 12 > gpurun_out/${T}_step_gemms.csv 2> gpurun_out/${T}_step_gemms.log
echo "gemms rc=$?"
# pair<96>: decode QKV only (6 / step); pair<128>: 13 encoder / cross-K/V, then
# per step 6 FFN1 + logits; split-K: 4 / layer / step (self-out, cross-q,
# cross-out, FFN2); tc_gemm_kernel: the encoder's N = 1024 GEMMs
cap qkv "xh_pair_gemm_kernel<.int.96" 60
cap ffn1 "xh_pair_gemm_kernel<.int.128" 83
cap logits "xh_pair_gemm_kernel<.int.128" 89
cap splitk "tc_gemm_splitk" 240
cap encgemm "tc_gemm_kernel" 1
cap selfattn "decoder_self_attention" 190
cap crossattn "cross_attention" 190
cap ln "layer_norm_slabs_row128" 540
cap harsstep "hars_step_item_kernel" 30
cap encattn "encoder_attention" 3
cap logits16 "tc_gemm_kernel<.int.224" 30 fp16
cap merge16 "hars_merge_step" 32 fp16
for f in qkv ffn1 logits splitk encgemm selfattn crossattn ln harsstep encattn logits16 merge16; do
  python scripts/ncu_summary.py gpurun_out/${T}_$f.ncu-rep 12 > gpurun_out/${T}_${f}_summary.txt 2>&1
  python scripts/ncu_ops.py gpurun_out/${T}_$f.ncu-rep 12 >> gpurun_out/${T}_${f}_summary.txt 2>&1
done
python scripts/launch_summary.py gpurun_out/${T}_launches.csv 30 > gpurun_out/${T}_launches_summary.txt 2>&1
rm -f gpurun_out/${T}_launches.csv gpurun_out/${T}_*.ncu-rep
python scripts/gemm_traffic_json.py gpurun_out/${T}_step_gemms.csv gpurun_out/${T}_ncu_gemm_traffic.json \
  "ncu (--clock-control none) of the GEMM launches of one C2 $P decode step (step 11 of a generate; scripts/ncu_round2b.sh ${T}): dram__bytes_read.sum + dram__bytes_write.sum per launch" \
  > gpurun_out/${T}_traffic.log 2>&1
ls -la gpurun_out | grep $T
