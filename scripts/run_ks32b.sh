mkdir -p gpurun_out
rm -f gpurun_out/ks32b.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ks32b.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ks32b.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ks32b.err | tee gpurun_out/ks32b.json | python scripts/bench_brief.py KS32b >> gpurun_out/ks32b.txt
timeout 300 python bench.py --rows 8192 --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ks32b.err | tee gpurun_out/ks32b_8k.json | python scripts/bench_brief.py KS32b rows=8192 >> gpurun_out/ks32b.txt
