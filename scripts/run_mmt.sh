mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "variants or full_params" > gpurun_out/pytest_mmt.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mmt.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/mmt.err | python scripts/bench_brief.py MMT > gpurun_out/mmt.txt
