mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for F in 1 2 0; do
CWGPU_FUSE_MAC=$F python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/fuse.err | tee gpurun_out/fuse_$F.json | python scripts/bench_brief.py FUSE=$F >> gpurun_out/fuse.txt
done
