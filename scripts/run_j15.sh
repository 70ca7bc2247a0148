mkdir -p gpurun_out
rm -f gpurun_out/j15.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_j15.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_j15.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/j15.err | tee gpurun_out/j15.json | python scripts/bench_brief.py J15 >> gpurun_out/j15.txt
