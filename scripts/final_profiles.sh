# Round-end evidence on one B200: full GPU test suite, the C4 headline bench line, the ncu launch
# list and ncu --set full summaries of the C4 hot kernels and of the C3 whole-row payload MAC.
# Outputs under gpurun_out/final/ (copied into profiles/ by hand).
O=gpurun_out/final
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python bench.py --steps 10 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err || exit 1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv $CMD > $O/ncu_launch.log 2>&1
python scripts/ncu_launch_summary.py $O/launches_C4.csv 7 > $O/ncu_launches_C4.txt 2>&1
gzip -f $O/launches_C4.csv
ncu --set full --import-source on --clock-control none -k regex:"k_tensor_intt_r|k_round_tma|k_ntt_mac" -s 60 -c 3 -o $O/full_C4 $CMD > $O/ncu_full.log 2>&1
python scripts/ncu_summary.py $O/full_C4.ncu-rep > $O/ncu_summary_C4_hot_kernels.txt 2>&1
for K in k_tensor_intt k_ntt_mac k_round_tma; do
echo "== per-opcode mix and stall samples: $K" >> $O/ncu_summary_C4_hot_kernels.txt
python scripts/ncu_stalls.py $O/full_C4.ncu-rep $K 0 >> $O/ncu_summary_C4_hot_kernels.txt 2>&1
done
python scripts/ncu_traffic.py $O/full_C4.ncu-rep C4 $O/ncu_traffic_C4.json > $O/ncu_traffic.log 2>&1
# C3 payload MAC (k_mac_rows) against HBM
CMD3="python bench.py --config C3 --rows 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-verify"
ncu --set full --import-source on --clock-control none -k regex:"k_mac_rows" -s 4 -c 2 -o $O/full_C3mac $CMD3 > $O/ncu_c3.log 2>&1
python scripts/ncu_summary.py $O/full_C3mac.ncu-rep > $O/ncu_summary_C3_payload_mac.txt 2>&1
python scripts/ncu_stalls.py $O/full_C3mac.ncu-rep k_mac_rows 0 >> $O/ncu_summary_C3_payload_mac.txt 2>&1
rm -f $O/full_C4.ncu-rep $O/full_C3mac.ncu-rep
tail -c 600 $O/bench_C4.json; cat $O/ncu_launches_C4.txt | head -8; cat $O/ncu_summary_C3_payload_mac.txt | head -8
