mkdir -p gpurun_out
rm -f gpurun_out/persist.txt
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "full_params or answer_small or rounding_engines" > gpurun_out/pytest_persist.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_persist.txt
for F in 1 0; do
CWGPU_TENSOR_PERSIST=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/persist.err | tee gpurun_out/persist_$F.json | python scripts/bench_brief.py PERSIST=$F >> gpurun_out/persist.txt
done
