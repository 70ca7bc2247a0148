#!/bin/bash
# Round-end measurement on the GPU box (gpurun): tests, default bench line, the ncu launch list
# of the same bench command, and one ncu --set full capture of the hot kernels (4096-row run,
# same per-launch sizes as the full C4 answer).  Everything is summarised on the box (the
# .ncu-rep files are too large to bring back); outputs under gpurun_out/<tag>_*.
TAG=${1:-r02}
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
    python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
fi
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err || exit 1
python scripts/bench_brief.py bench < gpurun_out/${TAG}_bench.json
BCMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$BCMD > gpurun_out/${TAG}_launch_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $BCMD \
    > gpurun_out/${TAG}_launches.log 2>&1
# the launch list covers 3 warm-up answers + 1 timed + 2 e2e (warm-up, timed) + 1 profiling pass = 7 answers
python scripts/ncu_launch_summary.py gpurun_out/${TAG}_launches.csv 7 > gpurun_out/${TAG}_launches.txt
gzip -f gpurun_out/${TAG}_launches.csv
CMD="python bench.py --rows 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$CMD > gpurun_out/${TAG}_full_plain.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_tensor_intt|k_round_tma|k_ntt_mac" \
    -s 6 -c 3 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_full_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_summary.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/${TAG}_full.ncu-rep C4 gpurun_out/${TAG}_ncu_traffic_C4.json > /dev/null 2>&1
for K in k_tensor_intt k_ntt_mac k_round_tma; do
    ncu -i gpurun_out/${TAG}_full.ncu-rep -k regex:$K --page source --csv --print-source sass \
        > gpurun_out/${TAG}_src_$K.csv 2>/dev/null
    python scripts/ncu_src_mix.py gpurun_out/${TAG}_src_$K.csv > gpurun_out/${TAG}_mix_$K.txt 2>&1
    rm -f gpurun_out/${TAG}_src_$K.csv
done
rm -f gpurun_out/${TAG}_full.ncu-rep
ls -la gpurun_out | grep ${TAG}
