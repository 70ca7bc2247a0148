# same-box A/B of two builds: $1 = alternative .so (build/), labels $2 (in-tree) / $3 (alternative)
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for it in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/ab.err | python scripts/bench_brief.py $2 >> gpurun_out/ab.txt
cp paper_2202_07569_b200/libcwgpu.so /tmp/ab_main.so; cp $1 paper_2202_07569_b200/libcwgpu.so
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/ab.err | python scripts/bench_brief.py $3 >> gpurun_out/ab.txt
cp /tmp/ab_main.so paper_2202_07569_b200/libcwgpu.so
done
