mkdir -p gpurun_out
rm -f gpurun_out/c5.txt
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "config5 or full_params" > gpurun_out/pytest_c5.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c5.txt
timeout 900 python bench.py --config C5 --rows 4096 --steps 2 --warmup 3 --no-cpu-baseline 2>>gpurun_out/c5.err | python scripts/bench_brief.py C5-4096rows >> gpurun_out/c5.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/c5.err | python scripts/bench_brief.py C4 >> gpurun_out/c5.txt
