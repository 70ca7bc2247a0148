mkdir -p gpurun_out
rm -f gpurun_out/g2.txt
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_golden.py -x -q -k "variants or full_params or answer_small or rounding_engines or exact_fallback or golden" > gpurun_out/pytest_g2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g2.txt
for F in 1 0; do
CWGPU_ROUND_G2=$F timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/g2.err | python scripts/bench_brief.py G2=$F >> gpurun_out/g2.txt
done
