# tile rows x tile streams sweep of the C4 bench (pipelined ms per answer); results -> gpurun_out/sweep.txt
# usage: scripts/sweep_tiles.sh "32 48 64 182" "2 3"
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
for R in ${1:-0 128 256 364}; do for S in ${2:-2 3 4}; do
timeout 300 python bench.py --opt tile_rows=$R --opt streams=$S --steps 3 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/sweep.err | python scripts/bench_brief.py R=$R S=$S >> gpurun_out/sweep.txt
done; done
cat gpurun_out/sweep.txt
