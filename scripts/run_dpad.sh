mkdir -p gpurun_out
rm -f gpurun_out/dpad.txt
CWGPU_DPAD=1 timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "variants or full_params or answer_small or rounding_engines or select" > gpurun_out/pytest_dpad.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dpad.txt
for it in 1 2; do for P in 0 1; do
CWGPU_DPAD=$P timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/dpad.err | python scripts/bench_brief.py DPAD=$P >> gpurun_out/dpad.txt
done; done
