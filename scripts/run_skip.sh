mkdir -p gpurun_out
rm -f gpurun_out/skip.txt
for K in 0 1 2 3; do
CWGPU_DEBUG_SKIP=$K timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/skip.err | python scripts/bench_brief.py SKIP=$K >> gpurun_out/skip.txt
done
