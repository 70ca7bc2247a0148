mkdir -p gpurun_out
python scripts/bench_ntt.py 0 1 13 18 19 20 > gpurun_out/ntt_micro2.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/bulk.err | tee gpurun_out/bulk.json | python scripts/bench_brief.py BULK > gpurun_out/bulk.txt
