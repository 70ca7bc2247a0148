#!/bin/bash
# Usage (on the GPU box via gpurun): scripts/prof_kernels.sh <tag> [rows]
# 1) plain run of the profiled command (must exit 0), 2) per-launch list,
# 3) ncu --set full on the top kernels.  Outputs under gpurun_out/.
set -e
TAG=${1:-prof}; ROWS=${2:-1024}
CMD="python bench.py --rows $ROWS --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:"k_round_mac|k_tensor_intt|k_ntt32r_sel3|k_mac" -s 40 -c 4 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1 || true
ls -la gpurun_out/
