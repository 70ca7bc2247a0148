mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "full_params" > gpurun_out/pytest_tir.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tir.txt
for F in 1 0; do
CWGPU_FUSE_TIR=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/tir.err | tee gpurun_out/tir_$F.json | python scripts/bench_brief.py TIR=$F >> gpurun_out/tir.txt
done
