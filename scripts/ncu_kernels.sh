#!/bin/bash
# Targeted `ncu --set full` captures, one report per kernel family, of a
# steady-state C2 bf16 decode step (scripts/profile_step.py, 40 decode steps,
# kernels after the warm-up graph capture). Usage: bash scripts/ncu_kernels.sh [tag]
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
cap() {  # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"$2" -s "$3" -c "$4" -o gpurun_out/${TAG}_$1 -f \
    python scripts/profile_step.py --steps 40 > gpurun_out/${TAG}_$1.log 2>&1
  echo "$1 rc=$?"
}
# per decode step: 6 self-attn, 6 cross-attn, 1 retrieve, 1 select; 18 N=1024 GEMMs, ...
cap selfattn "decoder_self_attention" 190 1
cap crossattn "cross_attention" 190 1
cap retrieve "retrieve_kernel" 32 1
cap select "hars_select" 32 1
cap gemm32 "tc_gemm_kernel<32" 570 3
cap gemm128 "tc_gemm_kernel<128" 380 2
cap splitk "splitk" 190 1
cap logits "tc_gemm_kernel<256" 40 1
cap ln "layer_norm_row128" 570 1
ls -la gpurun_out
