mkdir -p gpurun_out
rm -f gpurun_out/rctas.txt
for RC in 1 2 3 4; do for S in 2 3; do
CWGPU_ROUND_CTAS=$RC CWGPU_STREAMS=$S timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/rctas.err | python scripts/bench_brief.py RC=$RC S=$S >> gpurun_out/rctas.txt
done; done
