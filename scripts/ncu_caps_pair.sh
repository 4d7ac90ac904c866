set -u
T=r2b; P=fp32
cap() {
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    --kernel-name-base demangled -k regex:"$2" -s "$3" -c 1 -o gpurun_out/${T}_$1 -f \
    python scripts/profile_step.py --precision ${4:-$P} --steps 40 > gpurun_out/${T}_$1.log 2>&1
  echo "$1 rc=$?"
}
cap qkv "xh_pair_gemm_kernel<.int.96" 60
cap ffn1 "xh_pair_gemm_kernel<.int.128" 83
cap logits "xh_pair_gemm_kernel<.int.128" 89
for f in qkv ffn1 logits; do
  python scripts/ncu_summary.py gpurun_out/${T}_$f.ncu-rep 12 > gpurun_out/${T}_${f}_summary.txt 2>&1
  python scripts/ncu_ops.py gpurun_out/${T}_$f.ncu-rep 12 >> gpurun_out/${T}_${f}_summary.txt 2>&1
done
rm -f gpurun_out/${T}_*.ncu-rep
