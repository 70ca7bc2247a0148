set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s_default.json 2> gpurun_out/s_default.err
for R in 16 32 64; do for S in 2 4; do
CWGPU_TILE_ROWS=$R CWGPU_STREAMS=$S python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/sweep.err | python scripts/bench_brief.py R=$R S=$S >> gpurun_out/sweep.txt
done; done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline | python scripts/bench_brief.py default >> gpurun_out/sweep.txt
