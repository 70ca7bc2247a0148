mkdir -p gpurun_out
CMD="python bench.py --rows 2048 --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$CMD > gpurun_out/ntt_plain.json 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tensor_intt|k_ntt_mac|k_round_tma" -s 6 -c 3 -o gpurun_out/ntt_full $CMD > gpurun_out/ntt_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/ntt_full.ncu-rep > gpurun_out/ntt_summary.txt 2>&1
for K in k_tensor_intt k_ntt_mac k_round_tma; do
ncu -i gpurun_out/ntt_full.ncu-rep -k regex:$K --page source --csv --print-source sass > gpurun_out/src_$K.csv 2>/dev/null
gzip -f gpurun_out/src_$K.csv
done
rm -f gpurun_out/*.ncu-rep
