#!/bin/bash
# One `ncu --set full` capture + summary: bash scripts/ncu_cap_one.sh <tag> <name> <regex> <skip> [precision]
set -u
T=$1; N=$2; RX=$3; SK=$4; P=${5:-fp32}
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k regex:"$RX" -s "$SK" -c 1 -o gpurun_out/${T}_$N -f \
  python scripts/profile_step.py --precision $P --steps 40 > gpurun_out/${T}_$N.log 2>&1
echo "$N rc=$?"
python scripts/ncu_summary.py gpurun_out/${T}_$N.ncu-rep 12 > gpurun_out/${T}_${N}_summary.txt 2>&1
python scripts/ncu_ops.py gpurun_out/${T}_$N.ncu-rep 12 >> gpurun_out/${T}_${N}_summary.txt 2>&1
rm -f gpurun_out/${T}_$N.ncu-rep
