# ncu of the C3 whole-row payload MAC (k_mac_rows), 4096 rows; summaries -> gpurun_out/c3rows_*
mkdir -p gpurun_out
CMD="python bench.py --config C3 --rows 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-verify $*"
$CMD > gpurun_out/c3rows_plain.json 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_mac_rows" -s 4 -c 2 -o gpurun_out/c3rows $CMD > gpurun_out/c3rows_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/c3rows.ncu-rep > gpurun_out/c3rows_summary.txt 2>&1
python scripts/ncu_stalls.py gpurun_out/c3rows.ncu-rep k_mac_rows 40 >> gpurun_out/c3rows_summary.txt 2>&1
cat gpurun_out/c3rows_summary.txt
