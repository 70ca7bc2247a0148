# C3 A/B of library options: scripts/ab_c3.sh "--opt mac_rows=0" "--opt mac_rows=1" ...
mkdir -p gpurun_out
rm -f gpurun_out/ab_c3.txt
for it in 1 2; do for O in "$@"; do
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-verify $O 2>>gpurun_out/ab.err | python scripts/bench_brief.py "$O" >> gpurun_out/ab_c3.txt
done; done
cat gpurun_out/ab_c3.txt
