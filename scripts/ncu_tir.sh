mkdir -p gpurun_out
CMD="python bench.py --rows 2048 --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
$CMD > gpurun_out/tir_plain.json 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tir" -s 2 -c 1 -o gpurun_out/tir_full $CMD > gpurun_out/tir_ncu.log 2>&1
CWGPU_FUSE_TIR=0 timeout 600 ncu --set full --clock-control none -k regex:"k_tensor_intt|k_round_tc" -s 4 -c 2 -o gpurun_out/tir0_full $CMD > gpurun_out/tir0_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/tir_full.ncu-rep > gpurun_out/tir_summary.txt 2>&1
python scripts/ncu_summary.py gpurun_out/tir0_full.ncu-rep >> gpurun_out/tir_summary.txt 2>&1
ncu -i gpurun_out/tir_full.ncu-rep --page source --csv --print-source sass > gpurun_out/tir_source.csv 2>/dev/null
gzip -f gpurun_out/tir_source.csv
ls -la gpurun_out >> gpurun_out/tir_summary.txt
rm -f gpurun_out/*.ncu-rep
