# C5 (4096 rows) A/B of library options: scripts/ab_c5.sh "--opt ks_ci=4" "--opt ks_ci=2"
mkdir -p gpurun_out
for it in 1 2; do for O in "$@"; do
timeout 600 python bench.py --config C5 --rows 4096 --steps 2 --warmup 3 --no-cpu-baseline --no-verify $O 2>>gpurun_out/ab.err | python scripts/bench_brief.py "$O" >> gpurun_out/ab_c5.txt
done; done
cat gpurun_out/ab_c5.txt
