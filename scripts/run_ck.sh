mkdir -p gpurun_out
rm -f gpurun_out/ck.txt
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "variants" > gpurun_out/pytest_ck.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ck.txt
for CK in 0 13 26 40; do
CWGPU_MAC_CK=$CK timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/ck.err | python scripts/bench_brief.py CK=$CK >> gpurun_out/ck.txt
done
