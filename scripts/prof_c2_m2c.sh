mkdir -p gpurun_out
CMD="python bench.py --config C2-k2 --steps 1 --warmup 1 --no-cpu-baseline --no-verify $*"
ncu --set full --import-source on --clock-control none -k regex:"k_mac_to_chain_tc" -s 2 -c 2 -o gpurun_out/c2m2c $CMD > gpurun_out/c2m2c_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/c2m2c.ncu-rep > gpurun_out/c2m2c_summary.txt 2>&1
python scripts/ncu_stalls.py gpurun_out/c2m2c.ncu-rep k_mac_to_chain_tc 30 >> gpurun_out/c2m2c_summary.txt 2>&1
cat gpurun_out/c2m2c_summary.txt
