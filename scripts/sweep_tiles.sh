# tile rows x tile streams sweep of the C4 bench (pipelined ms per answer); results -> gpurun_out/sweep.txt
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
for R in 0 128 256 364; do for S in 2 3 4; do
if [ "$R" = "0" ]; then unset CWGPU_TILE_ROWS; else export CWGPU_TILE_ROWS=$R; fi
CWGPU_STREAMS=$S timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/sweep.err | python scripts/bench_brief.py R=$R S=$S >> gpurun_out/sweep.txt
done; done
