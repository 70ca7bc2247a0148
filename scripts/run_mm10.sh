mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_mm10.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mm10.txt
bash scripts/run_ab.sh build/libcwgpu_old.so NEW OLD
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print(d['config'], d['verified_decrypt'])" >> gpurun_out/ab.txt
