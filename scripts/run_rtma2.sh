mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_rtma2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rtma2.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/rtma2.err | tee gpurun_out/rtma2.json | python scripts/bench_brief.py RTMA2 > gpurun_out/rtma2.txt
