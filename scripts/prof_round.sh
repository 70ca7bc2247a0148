#!/bin/bash
# Round-end measurement on the GPU box (gpurun): tests, default bench line, the ncu launch list
# of the same bench command, and one ncu --set full capture of the hot kernels (4096-row run,
# same per-launch sizes as the full C4 answer).  Outputs under gpurun_out/<tag>_*.
TAG=${1:-r01}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || exit 1
python scripts/bench_brief.py bench < gpurun_out/${TAG}_bench.json
BCMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$BCMD > gpurun_out/${TAG}_launch_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $BCMD \
    > gpurun_out/${TAG}_launches.log 2>&1
CMD="python bench.py --rows 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$CMD > gpurun_out/${TAG}_full_plain.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_tensor_intt|k_round_tc|k_ntt32r_sel3|k_mac2|k_mac_tma" \
    -s 8 -c 4 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_full_ncu.log 2>&1
ls -la gpurun_out | grep ${TAG}
