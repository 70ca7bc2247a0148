mkdir -p gpurun_out
rm -f gpurun_out/dbg_tir3.txt
for R in 8192 65536; do for F in 1; do
CWGPU_FUSE_TIR=$F timeout 200 python bench.py --rows $R --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | python scripts/bench_brief.py R=$R TIR=$F >> gpurun_out/dbg_tir3.txt
done; done
