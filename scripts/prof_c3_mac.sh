# ncu of the C3 payload MAC kernels (4096 rows): k_mac_tma_q (3 slices / CTA, default) and
# k_mac_tma (mac_sg = 0); summaries -> gpurun_out/c3mac_*
mkdir -p gpurun_out
for V in 1 0; do
CMD="python bench.py --config C3 --rows 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-verify --opt mac_sg=$V"
$CMD > gpurun_out/c3mac_plain_$V.json 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_mac_tma" -s 4 -c 2 -o gpurun_out/c3mac_$V $CMD > gpurun_out/c3mac_ncu_$V.log 2>&1
python scripts/ncu_summary.py gpurun_out/c3mac_$V.ncu-rep > gpurun_out/c3mac_summary_$V.txt 2>&1
rm -f gpurun_out/c3mac_$V.ncu-rep
done
cat gpurun_out/c3mac_summary_*.txt
