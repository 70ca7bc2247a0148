# ncu --set full of the tree-path kernels at C5 (4096 rows): k_mac_to_chain, k_ks_mac32s, k_lift_tc,
# k_decompose_t, k_ks_crt; summaries -> gpurun_out/c5tree_summary.txt
mkdir -p gpurun_out
CMD="python bench.py --config C5 --rows 2048 --steps 1 --warmup 1 --no-cpu-baseline --no-verify $*"
ncu --set full --import-source on --clock-control none -k regex:"k_mac_to_chain|k_ks_mac32s|k_lift_tc|k_decompose_t|k_ks_crt" -s 40 -c 14 -o gpurun_out/c5tree $CMD > gpurun_out/c5tree_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/c5tree.ncu-rep > gpurun_out/c5tree_summary.txt 2>&1
for K in k_mac_to_chain k_ks_mac32s k_decompose_t k_ks_crt; do
echo "=== $K" >> gpurun_out/c5tree_summary.txt
python scripts/ncu_stalls.py gpurun_out/c5tree.ncu-rep $K 16 >> gpurun_out/c5tree_summary.txt 2>&1
done
cat gpurun_out/c5tree_summary.txt
