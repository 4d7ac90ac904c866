cd $GRAFT_REPO_ROOT
SHAPES=512x3072x1024 timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"tc_gemm_kernel" -s 6 -c 1 -o gpurun_out/epi_qkv python scripts/gemm_cta_anatomy.py > gpurun_out/ncu_epi.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_epi.log
