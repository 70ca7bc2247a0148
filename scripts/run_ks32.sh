mkdir -p gpurun_out
rm -f gpurun_out/ks32.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ks32.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ks32.txt
for F in 1 0; do
CWGPU_KS32=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ks32.err | tee gpurun_out/ks32_$F.json | python scripts/bench_brief.py KS32=$F >> gpurun_out/ks32.txt
CWGPU_KS32=$F timeout 300 python bench.py --rows 8192 --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/ks32.err | python scripts/bench_brief.py KS32=$F rows=8192 >> gpurun_out/ks32.txt
done
