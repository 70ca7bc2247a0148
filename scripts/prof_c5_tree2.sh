mkdir -p gpurun_out
CMD="python bench.py --config C5 --rows 2048 --steps 1 --warmup 1 --no-cpu-baseline --no-verify $*"
ncu --set full --import-source on --clock-control none -k regex:"k_mac_to_chain|k_lift_tc|k_arith|k_prep_factors|k_relin_add" -s 12 -c 8 -o gpurun_out/c5tree2 $CMD > gpurun_out/c5tree2_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/c5tree2.ncu-rep > gpurun_out/c5tree2_summary.txt 2>&1
for K in k_mac_to_chain k_lift_tc; do
echo "=== $K" >> gpurun_out/c5tree2_summary.txt
python scripts/ncu_stalls.py gpurun_out/c5tree2.ncu-rep $K 24 >> gpurun_out/c5tree2_summary.txt 2>&1
done
cat gpurun_out/c5tree2_summary.txt
