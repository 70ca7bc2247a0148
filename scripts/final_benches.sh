# Round-end bench lines for the other BASELINE configurations (one B200), each with the compiled
# reference timed on the box's host threads (cpu_baseline).  Outputs under gpurun_out/final/.
O=gpurun_out/final
mkdir -p $O
python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "batch or async or payload" 2>&1 | tail -2
for C in C3 C1 C2-k2 C2-k1 C2-k4; do
timeout 1500 python bench.py --config $C --steps 5 --warmup 3 > $O/bench_$C.json 2> $O/bench_$C.err
python scripts/bench_brief.py $C < $O/bench_$C.json
done
timeout 2400 python bench.py --config C5 --steps 2 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
python scripts/bench_brief.py C5 < $O/bench_C5.json
for C in C2-k8 C2-k16; do
timeout 1500 python bench.py --config $C --steps 3 --warmup 3 > $O/bench_$C.json 2> $O/bench_$C.err
python scripts/bench_brief.py $C < $O/bench_$C.json
done
