mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "load_db_bytes" > gpurun_out/pytest_dbb.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbb.txt
