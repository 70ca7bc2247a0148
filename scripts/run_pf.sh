mkdir -p gpurun_out
rm -f gpurun_out/pf.txt
timeout 600 python -m pytest tests/test_gpu_configs.py -x -q -k "variants" > gpurun_out/pytest_pf.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pf.txt
for it in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/pf.err | python scripts/bench_brief.py PF=1 >> gpurun_out/pf.txt
cp paper_2202_07569_b200/libcwgpu.so /tmp/pf1.so; cp build/libcwgpu_nopf.so paper_2202_07569_b200/libcwgpu.so
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/pf.err | python scripts/bench_brief.py PF=0 >> gpurun_out/pf.txt
cp /tmp/pf1.so paper_2202_07569_b200/libcwgpu.so
done
