mkdir -p gpurun_out
rm -f gpurun_out/ks32c.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "expand or substitute or relin" > gpurun_out/pytest_ks32c.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ks32c.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ks32c.err | tee gpurun_out/ks32c.json | python scripts/bench_brief.py KS32c >> gpurun_out/ks32c.txt
