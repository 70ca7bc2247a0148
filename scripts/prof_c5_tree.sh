# ncu --set full of the product-tree kernels at C5 (2,048 rows): the tensor-core conversions
# (k_lift_tc, k_mac_to_chain_tc, k_decompose_tc), the key-switch MAC / CRT (k_ks_mac32t, k_ks_crt3);
# summary -> gpurun_out/c5tree_summary.txt
mkdir -p gpurun_out
CMD="python bench.py --config C5 --rows 2048 --steps 1 --warmup 1 --no-cpu-baseline --no-verify $*"
rm -f gpurun_out/c5tree_summary.txt
for K in k_lift_tc k_mac_to_chain_tc k_decompose_tc k_ks_mac32t k_ks_crt3; do
ncu --set full --import-source on --clock-control none -k regex:"$K" -s 30 -c 1 -o gpurun_out/c5tree_$K $CMD > gpurun_out/c5tree_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/c5tree_$K.ncu-rep >> gpurun_out/c5tree_summary.txt 2>&1
python scripts/ncu_stalls.py gpurun_out/c5tree_$K.ncu-rep $K 0 >> gpurun_out/c5tree_summary.txt 2>&1
rm -f gpurun_out/c5tree_$K.ncu-rep
done
cat gpurun_out/c5tree_summary.txt
