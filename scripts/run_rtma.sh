mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_rtma.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rtma.txt
rm -f gpurun_out/rtma.txt
for F in 1 0; do
CWGPU_ROUND_TMA=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/rtma.err | tee gpurun_out/rtma_$F.json | python scripts/bench_brief.py RTMA=$F >> gpurun_out/rtma.txt
done
