mkdir -p gpurun_out
rm -f gpurun_out/smem.txt
for X in 0 92000 75000; do for S in 2 3; do
CWGPU_TENSOR_SMEM=$X CWGPU_STREAMS=$S timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/smem.err | python scripts/bench_brief.py SMEM=$X S=$S >> gpurun_out/smem.txt
done; done
