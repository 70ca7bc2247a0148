mkdir -p gpurun_out
rm -f gpurun_out/other.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline 2>>gpurun_out/other.err | python scripts/bench_brief.py C3 >> gpurun_out/other.txt
timeout 900 python bench.py --config C5 --rows 4096 --steps 2 --warmup 3 --no-cpu-baseline 2>>gpurun_out/other.err | python scripts/bench_brief.py C5-4096rows >> gpurun_out/other.txt
timeout 600 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/other.err | python scripts/bench_brief.py C1 >> gpurun_out/other.txt
