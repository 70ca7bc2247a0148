mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded" > gpurun_out/pytest_shard.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shard.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/shard.err | python scripts/bench_brief.py SHARD-1gpu > gpurun_out/shard.txt
