mkdir -p gpurun_out
rm -f gpurun_out/shoup.txt
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "variants or full_params or answer_small or rounding_engines or golden" > gpurun_out/pytest_shoup.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shoup.txt
for F in 1 0; do
CWGPU_TENSOR_SHOUP=$F CWGPU_STREAMS=3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/shoup.err | python scripts/bench_brief.py SHOUP=$F >> gpurun_out/shoup.txt
done
