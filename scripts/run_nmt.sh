mkdir -p gpurun_out
rm -f gpurun_out/nmt.txt
CWGPU_FUSE_MAC=3 timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -k "full_params or answer_small or rounding_engines" > gpurun_out/pytest_nmt.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_nmt.txt
for F in 3 1; do
CWGPU_FUSE_MAC=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/nmt.err | tee gpurun_out/nmt_$F.json | python scripts/bench_brief.py FUSE=$F >> gpurun_out/nmt.txt
done
