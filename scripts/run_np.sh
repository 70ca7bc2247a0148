mkdir -p gpurun_out
rm -f gpurun_out/np.txt
for NP in 2 1; do for S in 2 3; do
CWGPU_NTT_NP=$NP CWGPU_STREAMS=$S timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verify 2>>gpurun_out/np.err | python scripts/bench_brief.py NP=$NP S=$S >> gpurun_out/np.txt
done; done
