# Final state check on one B200: smoke(), the full GPU suite, every config's bench line.
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.txt; cat $O/pytest_gpu.txt
python bench.py --steps 10 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err; python scripts/bench_brief.py C4 < $O/bench_C4.json
bash scripts/final_benches.sh
